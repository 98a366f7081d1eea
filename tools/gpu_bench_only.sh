mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_gpu_align.py tests/test_gpu_objective.py tests/test_gpu_eval.py -x > gpurun_out/s_tests.log 2>&1; echo tests=$? > gpurun_out/s_status.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err; echo "bench=$?" >> gpurun_out/s_status.txt
