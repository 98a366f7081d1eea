mkdir -p gpurun_out; : > gpurun_out/nb.log
for v in base nb64 nb128; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/nb.log
  timeout 300 python tools/probe_lanes.py 1024 4 >> gpurun_out/nb.log 2>&1
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "advance_kernel\|step_kernel\|span" >> gpurun_out/nb.log
done
unset BMB_LIB
