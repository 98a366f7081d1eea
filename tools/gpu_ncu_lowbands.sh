# ncu of the first band-4 and band-8 order-2 evaluation launches (8-lane jobs)
mkdir -p gpurun_out
export BMB_NO_WARMUP=1
for b in 4 8; do
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "bmb_band$b/" \
  -k regex:"eval_sub_kernel" --launch-count 2 -o gpurun_out/eval_l$b python tools/probe_bands.py 64 > gpurun_out/ncu_eval$b.log 2>&1; echo "ncu_eval$b=$?" >> gpurun_out/status_lowbands.txt
done
