set -x
mkdir -p gpurun_out
timeout 900 python tools/hbm_kernels.py > gpurun_out/hbm_kernels.json 2> gpurun_out/hbm_kernels.err; echo "HBM EXIT $?"
cat gpurun_out/hbm_kernels.json; tail -3 gpurun_out/hbm_kernels.err
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "BENCH EXIT $?"
tail -c 5000 gpurun_out/bench.log; tail -5 gpurun_out/bench.err
