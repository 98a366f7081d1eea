mkdir -p gpurun_out
set -x
python tools/probe_refine_l16.py 8 > gpurun_out/refine_l16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|expand_factored|compose_kernel" -c 4 -o gpurun_out/l16_full python tools/probe_refine_l16.py 8 > gpurun_out/ncu_l16.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
