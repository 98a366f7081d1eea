# quick check: expansion tests, config-2 bench (no CPU baseline), config 5
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_gpu_expand.py -x > gpurun_out/q_tests.log 2>&1; echo tests=$? > gpurun_out/q_status.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench=$?" >> gpurun_out/q_status.txt
timeout 600 python tools/bench_configs.py 5 > gpurun_out/q_cfg5.jsonl 2> gpurun_out/q_cfg5.err; echo "cfg5=$?" >> gpurun_out/q_status.txt
