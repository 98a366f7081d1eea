mkdir -p gpurun_out; : > gpurun_out/occ2.log
for v in base h2o26 h2o28 h2o30; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/occ2.log
  timeout 300 python tools/probe_lanes.py 1024 4 >> gpurun_out/occ2.log 2>&1
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "eval_sub_kernel<2\|span" >> gpurun_out/occ2.log
done
unset BMB_LIB
