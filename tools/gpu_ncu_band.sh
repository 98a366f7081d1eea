# Band breakdown + ncu --set full of the first order-2 / order-0 evaluation launches
# of band L (NVTX range bmb_band<L>) in tools/probe_bands.py.
#   gpurun -- 'bash tools/gpu_ncu_band.sh 16 tag'
L=${1:-16}; TAG=${2:-r2}
mkdir -p gpurun_out
timeout 300 python tools/probe_bands.py 256 > gpurun_out/bands_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "bmb_band${L}/" \
  -k regex:"eval_kernel|eval_sub_kernel" --launch-count 2 -o gpurun_out/eval_l${L}_${TAG} python tools/probe_bands.py 64 \
  > gpurun_out/ncu_eval_${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_eval_${TAG}.log
