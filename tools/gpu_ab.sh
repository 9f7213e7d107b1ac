# A/B on one box: bench default vs the unfused rotation; shard timing; launch list of one bench pair
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_windowed.py tests/test_gpu_shear.py -q -ra -x > gpurun_out/t_win.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_win.log
tail -5 gpurun_out/t_win.log
for i in 1 2; do
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-per-view --no-recon > gpurun_out/bench_a$i.log 2>&1
LFM_NO_ROT_FUSE=1 timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-per-view --no-recon > gpurun_out/bench_b$i.log 2>&1
done
python - <<'PY'
import json
for n in ("a1","b1","a2","b2"):
    d=json.loads(open("gpurun_out/bench_%s.log"%n).read().strip().splitlines()[-1])
    k=d["kernels"]
    print(n, "%.1f pairs/s"%d["value"], {kk: round(v["ms"]*1e3,1) for kk,v in k.items()})
PY
timeout 600 python tools/shard_timing.py 1 > gpurun_out/shard_timing.json 2> gpurun_out/shard_timing.err; echo "SHARD EXIT $?"
cat gpurun_out/shard_timing.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph > gpurun_out/ncu_list.log 2>&1; echo "NCU EXIT $?"
