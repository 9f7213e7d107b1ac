set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pwls.py tests/test_gpu_subsets.py -q -ra > gpurun_out/t_pwls.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_pwls.log
tail -5 gpurun_out/t_pwls.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "BENCH EXIT $?"
tail -c 6000 gpurun_out/bench.log; tail -20 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "REF EXIT $?"
tail -c 3000 gpurun_out/bench_ref.log
nproc; lscpu | head -20
