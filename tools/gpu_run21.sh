mkdir -p gpurun_out
for v in default q0mb2 q0mb3 default; do
  if [ $v = default ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  python tools/bench_configs.py 4 > gpurun_out/cfg4_$v.jsonl 2>&1
done
