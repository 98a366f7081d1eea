mkdir -p gpurun_out
timeout 600 python tools/probe_lanes.py 1024 3 4 5 6 8 4 6 > gpurun_out/lanes2.txt 2>&1
