mkdir -p gpurun_out
python tools/bench_configs.py 3x > gpurun_out/cfg3x.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expand_factored -s 1 -c 1 -o gpurun_out/expand64 python tools/bench_configs.py 3x > gpurun_out/ncu_exp.log 2>&1; echo ncu=$? > gpurun_out/status.txt
