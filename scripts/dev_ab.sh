set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_ab.log 2>&1
for v in 1 0 1 0; do CW_PCG_PREFILL=$v python scripts/dev_kernel_times.py 5 > gpurun_out/kt_pf$v.$RANDOM.log 2>&1; done
for v in 1 0 1; do CW_PCG_PREFILL=$v python bench.py --no-cpu --no-design 2>/dev/null | tail -1 > gpurun_out/bench_pf$v.$RANDOM.json; done
CW_NVCC_DEFS="-DCW_MAC_PRED_MINB=6" python -m paper_2204_01117_b200.build --force > /dev/null 2>&1 && python scripts/dev_kernel_times.py 5 > gpurun_out/kt_pred6.log 2>&1
CW_NVCC_DEFS="-DCW_MAC_PRED_MINB=8 -DCW_MAC_CORR_MINB=6" python -m paper_2204_01117_b200.build --force > /dev/null 2>&1 && python scripts/dev_kernel_times.py 5 > gpurun_out/kt_pred8c6.log 2>&1
