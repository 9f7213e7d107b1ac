# HBM-bound kernels at 256^3, per-rank shard timings, NEXT timings (current build)
mkdir -p gpurun_out
timeout 900 python tools/hbm_kernels.py > gpurun_out/hbm_kernels.json 2> gpurun_out/hbm_kernels.err; echo "HBM EXIT $?"
timeout 600 python tools/shard_timing.py 1 > gpurun_out/shard_timing.json 2> gpurun_out/shard_timing.err; echo "SHARD EXIT $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "REF EXIT $?"
