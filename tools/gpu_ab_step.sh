# A/B of library variants on the config-2 step time (tools/probe_lanes.py, 4 lanes):
#   gpurun -- 'bash tools/gpu_ab_step.sh base v1 v2 ...'
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  echo "== $v $(timeout 300 python tools/probe_lanes.py 1024 4 4 2>&1 | grep lanes | tr '\n' ' ')" >> gpurun_out/ab_step.log
done
unset BMB_LIB
