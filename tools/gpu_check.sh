# GPU suite (all failures listed), smoke, a short bench line
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -ra > gpurun_out/gpu_tests.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE $?
tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "BENCH EXIT $?"
tail -2 gpurun_out/bench.log
