mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_align.py tests/test_gpu_average_generate.py tests/test_gpu_objective.py -x > gpurun_out/n_tests.log 2>&1; echo tests=$? > gpurun_out/n_status.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo "bench=$?" >> gpurun_out/n_status.txt
timeout 300 python tools/probe_lanes.py 1024 1 4 > gpurun_out/n_lanes.txt 2>&1
