mkdir -p gpurun_out; : > gpurun_out/occ.log
for v in base o28 o24 oth28 oth20 base; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v" >> gpurun_out/occ.log
  timeout 300 python tools/probe_lanes.py 1024 4 >> gpurun_out/occ.log 2>&1
  timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "eval_sub\|span" >> gpurun_out/occ.log
done
unset BMB_LIB
