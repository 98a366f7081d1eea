mkdir -p gpurun_out
python tools/probe_align.py 64 > gpurun_out/probe64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expand_factored -s 0 -c 1 -o gpurun_out/expand_bench python tools/probe_align.py 64 > gpurun_out/ncu_eb.log 2>&1; echo ncu=$? > gpurun_out/status.txt
