# bench line with the e2e legs (no CPU baseline / recon / per-view), twice
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --no-per-view --no-recon --no-cpu-baseline > gpurun_out/e2e.log 2>&1
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/e2e.log") if l.startswith("{")][-1])
print("pairs/s %.1f" % d["value"], "e2e %.1f" % d["e2e"]["value"], "roof %.1f frac %.3f" % (d["e2e"]["copy_roof"]["value"], d["e2e"]["copy_roof"]["frac"]), "grad %.1f" % d["e2e_gradient"]["value"])
PY
done
