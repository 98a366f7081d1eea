mkdir -p gpurun_out
timeout 600 python tools/probe_lanes.py 1024 2 3 4 5 6 8 > gpurun_out/lanes.txt 2>&1
timeout 600 python tools/probe_bands.py 256 > gpurun_out/bands.txt 2>&1
