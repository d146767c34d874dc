set -x
T=r1j
python bench.py > gpurun_out/bench_full_$T.log 2>&1; tail -1 gpurun_out/bench_full_$T.log > gpurun_out/bench_$T.json
python bench.py --impl reference > gpurun_out/bench_ref_full_$T.log 2>&1; tail -1 gpurun_out/bench_ref_full_$T.log > gpurun_out/bench_ref_$T.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_ll_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pcg --launch-skip 3 --launch-count 1 -o gpurun_out/k_pcg_$T -f python bench.py --steps 3 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_full_$T.log 2>&1
python scripts/dev_kernel_times.py 5 > gpurun_out/ktimes_$T.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stepk_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_stepk_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_mac --launch-skip 6 --launch-count 2 -o gpurun_out/k_mac_$T -f python bench.py --steps 3 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_mac_$T.log 2>&1
python scripts/dev_c5.py 5 > gpurun_out/c5_$T.log 2>&1
