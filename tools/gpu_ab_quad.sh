# A/B of the quad-copy pair-list expansion (BMB_EXPAND_QUAD) on the expansion tests and the config-2 step:
#   gpurun --timeout 1200 -- 'bash tools/gpu_ab_quad.sh'
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_gpu_expand.py -x -k "quads or tensor_dft or pairs" > gpurun_out/quad_tests.log 2>&1; echo tests=$? > gpurun_out/quad_status.txt
for q in 0 1; do
  BMB_EXPAND_QUAD=$q timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quad$q.json 2> gpurun_out/bench_quad$q.err; echo "bench_quad$q=$?" >> gpurun_out/quad_status.txt
done
