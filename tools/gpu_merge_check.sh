mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/t_var.log 2>&1; echo "VAR EXIT $?"; tail -3 gpurun_out/t_var.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-per-view > gpurun_out/bench_m.log 2>&1; echo "BENCH EXIT $?"; tail -1 gpurun_out/bench_m.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:band_v --csv --log-file gpurun_out/bv.csv python tools/prof_pair.py 0 > gpurun_out/bv.log 2>&1; echo "NCU $?"
grep band_v gpurun_out/bv.csv | awk -F'","' '{print $5, $NF}' | head
