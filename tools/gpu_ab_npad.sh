mkdir -p gpurun_out; : > gpurun_out/npad.log
for v in base npad8 npad16; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/npad.log
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "advance_kernel\|step_kernel\|span" >> gpurun_out/npad.log
done
unset BMB_LIB
