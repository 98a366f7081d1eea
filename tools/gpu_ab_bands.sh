# A/B of library variants on the single-lane band breakdown (tools/probe_bands.py):
#   gpurun -- 'bash tools/gpu_ab_bands.sh base minb2_3 ...'   (base = the in-tree build)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  for rep in 1 2; do
    echo "== $v rep $rep" >> gpurun_out/ab_bands.log
    timeout 300 python tools/probe_bands.py 256 2>&1 | grep -E "timed|^\{'expand|band [0-9]" >> gpurun_out/ab_bands.log
  done
done
unset BMB_LIB
