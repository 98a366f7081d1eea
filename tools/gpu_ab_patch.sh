mkdir -p gpurun_out; : > gpurun_out/patch.log
BMB_LIB=build/variants/patch1.so timeout 600 python -m pytest -q -m gpu tests/test_gpu_expand.py -x -k "quads" >> gpurun_out/patch.log 2>&1
for v in base patch1 base patch1; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/patch.log
  timeout 300 python tools/probe_lanes.py 1024 4 >> gpurun_out/patch.log 2>&1
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "expand_quad\|span\|eval_sub_kernel<2, true, 8" >> gpurun_out/patch.log
done
unset BMB_LIB
