# GPU parity suite + two bench lines (no CPU baseline / per-view; recon included)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/q_tests.log 2>&1; echo "TESTS EXIT $?"; tail -3 gpurun_out/q_tests.log
B="python bench.py --steps 300 --no-per-view --no-cpu-baseline --no-e2e"
for i in 1 2; do timeout 600 $B > gpurun_out/q_bench.log 2>&1; python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/q_bench.log") if l.startswith("{")][-1])
print("pairs/s %.1f" % d["value"], "recon ms/it %.4f" % d["recon"]["ms_per_iteration"], "OS %.4f" % d["recon"]["ordered_subsets"]["ms_per_subset_iteration"], "err %.4f" % d["recon"]["rel_error_vs_truth_after_50"])
PY
done
