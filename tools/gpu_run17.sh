mkdir -p gpurun_out
python -m pytest -q -m gpu tests -x -k "expand or align or average" > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/status.txt
for v in default minb3 minb4; do
  if [ $v = default ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  python tools/bench_configs.py 3x > gpurun_out/cfg3x_$v.log 2>&1
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
