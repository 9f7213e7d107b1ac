set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_windowed.py tests/test_gpu_shear.py tests/test_gpu_pwls.py -q -ra -x > gpurun_out/t_win.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_win.log
tail -4 gpurun_out/t_win.log
for i in 1 2; do
timeout 300 python tools/ab_stage.py tools/ab/liblfm_r01.so paper_1812_03358_b200/liblfm.so >> gpurun_out/ab_stage.log 2>&1
done
cat gpurun_out/ab_stage.log
timeout 600 python tools/shard_timing.py 1 > gpurun_out/shard_timing.json 2> gpurun_out/shard_timing.err; echo "SHARD EXIT $?"
cat gpurun_out/shard_timing.json
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-per-view --no-recon > gpurun_out/bench_a.log 2>&1
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_a.log").read().strip().splitlines()[-1])
print("%.1f pairs/s"%d["value"], {kk: round(v["ms"]*1e3,1) for kk,v in d["kernels"].items()})
PY
