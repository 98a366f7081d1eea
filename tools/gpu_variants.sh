# A/B of compile-time variants: CUPTI kernel profile (512 particles, one lane) per variant
mkdir -p gpurun_out; : > gpurun_out/variants.log
for n in base comp512 comp128 comp384; do
  echo "== $n" >> gpurun_out/variants.log
  if [ $n = base ]; then lib=""; else lib="BMB_LIB=build/variants/$n.so"; fi
  env $lib timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | head -7 >> gpurun_out/variants.log
done
