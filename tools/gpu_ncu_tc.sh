# ncu of one config-2 expansion launch, tensor-core phi-DFT kernel and the FP32-pipe pair kernel:
#   gpurun --timeout 1500 -- 'bash tools/gpu_ncu_tc.sh'
mkdir -p gpurun_out
export BMB_NO_WARMUP=1
BMB_EXPAND_TC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"expand_tc" --launch-skip 1 --launch-count 1 -o gpurun_out/expand_tc python tools/probe_bands.py 64 > gpurun_out/ncu_tc.log 2>&1; echo ncu_tc=$? > gpurun_out/status_ncu_tc.txt
BMB_EXPAND_TC=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"expand_pair" --launch-skip 1 --launch-count 1 -o gpurun_out/expand_pair python tools/probe_bands.py 64 > gpurun_out/ncu_pair.log 2>&1; echo ncu_pair=$? >> gpurun_out/status_ncu_tc.txt
