# ncu --set full of the first order-2 / order-0 evaluation launches of the main
# (64-particle) run in band L: skips the 8-particle warm-up's launches of the band.
L=${1:-16}; TAG=${2:-r2}; SKIP=${3:-400}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "bmb_band${L}/" \
  -k regex:eval_kernel --launch-skip ${SKIP} --launch-count 2 -o gpurun_out/evalbig_l${L}_${TAG} \
  python tools/probe_bands.py 64 > gpurun_out/ncu_evalbig_${L}_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_evalbig_${L}_${TAG}.log
