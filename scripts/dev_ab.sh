# developer A/B of compile-time variants: warm per-kernel times of steady C3 steps per variant
set -x
for defs in "" "-DCW_ZT=2" "-DCW_ZT=8" "-DCW_ZT_MAC=1" "-DCW_ZT_MAC=4" "-DCW_ST_BY=16" "-DCW_ST_BY=4" ""; do
  tag=$(echo "x$defs" | tr -c 'a-zA-Z0-9=\n' '_')
  CW_NVCC_DEFS="$defs" python -m paper_2204_01117_b200.build --force > /dev/null 2>&1 && python scripts/dev_kernel_times.py 5 > gpurun_out/kt_$tag.$RANDOM.log 2>&1
done
