# ncu of one config-2 seed launch
mkdir -p gpurun_out
export BMB_NO_WARMUP=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"seed_kernel" --launch-skip 1 --launch-count 1 -o gpurun_out/seed3 python tools/probe_bands.py 64 > gpurun_out/ncu_seed.log 2>&1; echo ncu_seed=$? > gpurun_out/status_ncu_seed.txt
