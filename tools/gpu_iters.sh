mkdir -p gpurun_out
BMB_DEBUG_ITERS=1 BMB_NO_WARMUP=1 timeout 600 python tools/probe_bands.py 256 > gpurun_out/iters.txt 2> gpurun_out/iters.err
