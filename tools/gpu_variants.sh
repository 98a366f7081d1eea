# A/B of variants: CUPTI kernel profile (512 particles, one lane) per variant.
# An entry is a variant .so name (build/variants/NAME.so), "base", or base with
# an environment setting (e.g. "env:BMB_EVAL_K0=2").
mkdir -p gpurun_out; : > gpurun_out/variants.log
for n in ${VARIANTS:-base}; do
  echo "== $n" >> gpurun_out/variants.log
  case $n in
    base) pre="" ;;
    env:*) pre="${n#env:}" ;;
    *) pre="BMB_LIB=build/variants/$n.so" ;;
  esac
  env $pre timeout 300 python tools/profile_kernels.py 512 1 2>&1 | grep -v arn | head -12 >> gpurun_out/variants.log
done
