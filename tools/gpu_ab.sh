mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
timeout 400 python tools/profile_kernels.py 512 1 > gpurun_out/prof1.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
