set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_windowed.py tests/test_gpu_shear.py tests/test_gpu_pwls.py tests/test_gpu_subsets.py tests/test_gpu_parity.py -q -ra -x > gpurun_out/t_win.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_win.log
tail -15 gpurun_out/t_win.log
timeout 600 python tools/shard_timing.py 1 > gpurun_out/shard_timing.json 2> gpurun_out/shard_timing.err; echo "SHARD EXIT $?"
cat gpurun_out/shard_timing.json; tail -5 gpurun_out/shard_timing.err
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "BENCH EXIT $?"
tail -c 4000 gpurun_out/bench.log
