mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_align.py tests/test_gpu_average_generate.py -x > gpurun_out/r_tests.log 2>&1; echo tests=$? > gpurun_out/r_status.txt
for c in 1 4 8; do
  BMB_ROUND_CHECK=$c timeout 300 python tools/probe_lanes.py 1024 1 4 > gpurun_out/round_check$c.txt 2>&1
done
