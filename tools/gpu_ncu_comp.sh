mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:compose_kernel --launch-skip 23 --launch-count 1 -o gpurun_out/compose_l16 python tools/probe_bands.py 64 > gpurun_out/ncu_comp.log 2>&1; echo ncu=$? > gpurun_out/status.txt
