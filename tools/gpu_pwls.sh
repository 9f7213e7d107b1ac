# PWLS kernels: parity tests, then HBM fractions at 256^3 and the 128^3 bench kernel table
timeout 600 python -m pytest tests/test_gpu_pwls.py tests/test_gpu_recon.py -q 2>&1 | tail -2
timeout 900 python tools/hbm_kernels.py > gpurun_out/hbm_kernels.json 2> gpurun_out/hbm_kernels.err; echo "HBM EXIT $?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/hbm_kernels.json"))
for k, v in d["kernels"].items(): print("%-24s %7.1f us %5.3f" % (k, v["us"], v["frac_measured"]))
PY
