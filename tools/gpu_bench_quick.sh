# bench line (no CPU baseline) + launch list of the timed steps
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "BENCH $?"
python tools/bench_brief.py gpurun_out/bench_q.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph --profile-timed > gpurun_out/plain_bench.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_q.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph --profile-timed > gpurun_out/ncu_launch.log 2>&1; echo "NCU LAUNCH $?"
