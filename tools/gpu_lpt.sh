set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_concurrent.py tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_windowed.py -q -ra -x > gpurun_out/t_lpt.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_lpt.log
tail -4 gpurun_out/t_lpt.log
rm -f gpurun_out/ab_lpt.log
for i in 1 2; do
timeout 300 python tools/ab_stage.py paper_1812_03358_b200/liblfm.so >> gpurun_out/ab_lpt.log 2>&1
LFM_NO_LPT=1 timeout 300 python tools/ab_stage.py paper_1812_03358_b200/liblfm.so >> gpurun_out/ab_lpt.log 2>&1
done
cat gpurun_out/ab_lpt.log
for v in "" 1; do
LFM_NO_LPT=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-per-view --no-recon > gpurun_out/bench_lpt$v.log 2>&1
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_lpt$v.log").read().strip().splitlines()[-1])
print("LPT_OFF=$v", "%.1f pairs/s"%d["value"], {kk: round(v["ms"]*1e3,1) for kk,v in d["kernels"].items() if "pass" in kk})
PY
done
