# quick GPU check: band_u / s-pass variants + full-size parity + a short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -k "band_u or s_pass" -x -q > gpurun_out/t_var.log 2>&1; echo "VAR EXIT $?"; tail -3 gpurun_out/t_var.log
LFM_DEBUG_TUNE=1 LFM_DEBUG=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-per-view > gpurun_out/bench_q.log 2> gpurun_out/bench_q.err; echo "BENCH EXIT $?"; tail -1 gpurun_out/bench_q.log
grep "autotune\|direct s\|collapsed forward" gpurun_out/bench_q.err | grep -v "xp_\|_s1 \|_s3 " | head -40
