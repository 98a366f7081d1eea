mkdir -p gpurun_out; : > gpurun_out/pm.log
for v in base pm3 pm1; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/pm.log
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "expand_quad\|span" >> gpurun_out/pm.log
done
unset BMB_LIB
