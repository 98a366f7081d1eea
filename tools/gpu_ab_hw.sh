mkdir -p gpurun_out; : > gpurun_out/hw.log
for v in base hw4 base hw4; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/hw.log
  timeout 300 python tools/probe_lanes.py 1024 4 >> gpurun_out/hw.log 2>&1
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "eval_sub\|span" >> gpurun_out/hw.log
done
unset BMB_LIB
