# GPU suite + a launch list of exactly the timed steps (bench.py --profile-timed under --profile-from-start off)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -ra -x > gpurun_out/gpu_tests.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
  --log-file gpurun_out/launches_timed.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
  --no-per-view --no-recon --no-graph --profile-timed > gpurun_out/ncu_launch_timed.log 2>&1; echo "NCU LAUNCH EXIT $?"
