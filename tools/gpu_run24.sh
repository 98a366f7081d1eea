mkdir -p gpurun_out
for v in default nb32 nb256; do
  if [ $v = default ]; then unset BMB_LIB; else export BMB_LIB=build/variants/$v.so; fi
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
