# one round's evidence on the GPU box: tests, bench (both arms, the driver's
# K/W), the ncu launch list of the bench command, one ncu --set full capture
# of k_pcg, warm per-kernel times.  Usage: bash scripts/dev_profile_round.sh TAG
set -x
T=${1:-r2}
python -m pytest tests -m gpu -q > gpurun_out/gputests_$T.log 2>&1; tail -3 gpurun_out/gputests_$T.log
python __graft_entry__.py > gpurun_out/smoke_$T.log 2>&1; tail -1 gpurun_out/smoke_$T.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full_$T.log 2>&1; tail -1 gpurun_out/bench_full_$T.log > gpurun_out/bench_$T.json
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_full_$T.log 2>&1; tail -1 gpurun_out/bench_ref_full_$T.log > gpurun_out/bench_ref_$T.json
python scripts/dev_kernel_times.py 5 > gpurun_out/ktimes_$T.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_plain_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_ll_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pcg --launch-skip 3 --launch-count 1 -o gpurun_out/k_pcg_$T -f python bench.py --steps 3 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_full_$T.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stepk_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-design > gpurun_out/ncu_stepk_$T.log 2>&1
