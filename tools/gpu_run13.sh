mkdir -p gpurun_out
python tools/probe_refine_l16.py 32 > gpurun_out/refine_l16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"compose_kernel|accept_kernel|step_kernel|iter_begin" -c 6 -o gpurun_out/refine_misc python tools/probe_refine_l16.py 32 > gpurun_out/ncu_misc.log 2>&1; echo ncu=$? > gpurun_out/status.txt
