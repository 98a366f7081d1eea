mkdir -p gpurun_out; : > gpurun_out/n2.log
timeout 900 python -m pytest -q -m gpu tests/test_gpu_align.py tests/test_gpu_average_generate.py -x >> gpurun_out/n2.log 2>&1
timeout 300 python tools/probe_lanes.py 1024 4 >> gpurun_out/n2.log 2>&1
timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | grep "advance_kernel\|step_kernel\|span" >> gpurun_out/n2.log
