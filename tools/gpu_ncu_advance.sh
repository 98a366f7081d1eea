# ncu --set full of two large Newton rounds (advance_kernel) of a single-lane
# 1024-particle config-2 run (tools/probe_bands.py); the launches are whole-group
# lists of ~10^5 candidates.   gpurun -- 'bash tools/gpu_ncu_advance.sh tag'
TAG=${1:-r2}
mkdir -p gpurun_out
BMB_NO_WARMUP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel \
  --launch-skip 3 --launch-count 2 -o gpurun_out/advance_${TAG} python tools/probe_bands.py 1024 \
  > gpurun_out/ncu_advance_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_advance_${TAG}.log
