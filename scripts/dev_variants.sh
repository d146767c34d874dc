#!/bin/bash
# developer A/B of compile-time variants on the GPU box: for each CW_NVCC_DEFS
# string, rebuild and record warm per-kernel times of steady C3 steps plus the
# per-phase PCG probe.  Usage: bash scripts/dev_variants.sh "" "-DX=1" ...
mkdir -p gpurun_out
for defs in "$@"; do
  tag=$(echo "v$defs" | tr -c 'a-zA-Z0-9=\n' '_')
  echo "=== variant [$defs]"
  CW_NVCC_DEFS="$defs" python -m paper_2204_01117_b200.build --force > gpurun_out/build_$tag.log 2>&1 || { echo build failed; tail -5 gpurun_out/build_$tag.log; continue; }
  python scripts/dev_kernel_times.py 5 2>/dev/null | grep -E "${KT_GREP:-iterations|k_pcg|total}"
  python scripts/dev_probe_pcg.py 6 2>/dev/null | tail -1
done
