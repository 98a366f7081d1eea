mkdir -p gpurun_out; : > gpurun_out/fold.log
timeout 600 python -m pytest -q -m gpu tests/test_gpu_expand.py -x >> gpurun_out/fold.log 2>&1
timeout 300 python tools/probe_lanes.py 1024 4 >> gpurun_out/fold.log 2>&1
timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "expand_quad\|span" >> gpurun_out/fold.log
