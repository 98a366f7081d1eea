# A/B of the tensor-core phi-DFT expansion (BMB_EXPAND_TC) on the expansion tests and the config-2 step:
#   gpurun --timeout 1200 -- 'bash tools/gpu_ab_tc.sh'
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_gpu_expand.py -x -k "tensor_dft or window_pairs" > gpurun_out/tc_tests.log 2>&1; echo tests=$? > gpurun_out/tc_status.txt
for tc in 0 1; do
  BMB_EXPAND_TC=$tc timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_tc$tc.json 2> gpurun_out/bench_tc$tc.err; echo "bench_tc$tc=$?" >> gpurun_out/tc_status.txt
done
