mkdir -p gpurun_out
python tools/bench_configs.py 3x > gpurun_out/cfg3x.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expand_factored -s 1 -c 1 -o gpurun_out/r1_expand python tools/bench_configs.py 3x > gpurun_out/ncu_a.log 2>&1
python tools/probe_refine_l16.py 64 > gpurun_out/refine_l16.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"eval_kernel|compose_kernel|step_kernel|accept_kernel" -c 5 -o gpurun_out/r1_refine python tools/probe_refine_l16.py 64 > gpurun_out/ncu_b.log 2>&1
python tools/bench_configs.py 4 > gpurun_out/cfg4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_sweep -s 1 -c 1 -o gpurun_out/r1_sweep python tools/bench_configs.py 4 > gpurun_out/ncu_c.log 2>&1
echo done > gpurun_out/status.txt
