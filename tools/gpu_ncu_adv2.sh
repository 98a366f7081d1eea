mkdir -p gpurun_out
export BMB_NO_WARMUP=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/advance2 python tools/probe_bands.py 1024 > gpurun_out/ncu_adv2.log 2>&1; echo ncu=$? > gpurun_out/status_adv2.txt
