mkdir -p gpurun_out; : > gpurun_out/seedab.log
for v in base seed48 seed40 base; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/seedab.log
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "seed_kernel\|span" >> gpurun_out/seedab.log
done
unset BMB_LIB
