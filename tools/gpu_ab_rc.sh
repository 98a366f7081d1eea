mkdir -p gpurun_out; : > gpurun_out/rc.log
for v in base rc2 rc8; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/rc.log
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | head -8 >> gpurun_out/rc.log
done
unset BMB_LIB
