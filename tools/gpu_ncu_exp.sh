mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:expand_factored --launch-skip 1 --launch-count 1 -o gpurun_out/expand_cfg2 python tools/probe_bands.py 64 > gpurun_out/ncu_exp.log 2>&1; echo ncu=$? > gpurun_out/status.txt
