# 2xFP16 band_u: parity suites, then bench A/B against the 3xTF32 form (LFM_UMMA_TF32=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/f16_tests.log 2>&1; echo "TESTS EXIT $?"; tail -5 gpurun_out/f16_tests.log
for v in f16 tf32; do
  if [ $v = tf32 ]; then export LFM_UMMA_TF32=1; fi
  timeout 300 python bench.py --steps 200 --no-per-view --no-recon --no-cpu-baseline --no-e2e > gpurun_out/f16_bench_$v.log 2>&1; echo "BENCH $v EXIT $?"
  python - "$v" <<'PY'
import json, sys
l = [x for x in open("gpurun_out/f16_bench_%s.log" % sys.argv[1]) if x.startswith("{")]
d = json.loads(l[-1]); k = d.get("kernels", {})
print(sys.argv[1], "pairs/s %.1f" % d["value"], {n: round(v["ms"] * 1e3, 1) for n, v in k.items() if "pass" in n})
PY
done
