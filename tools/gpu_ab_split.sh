# A/B: column-scaled one-kernel split of the adjoint input (default) vs global maxima + split (LFM_SPLIT_GLOBAL=1)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo "TESTS EXIT $?"; tail -3 gpurun_out/ab_tests.log
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2; do
  timeout 300 $B > gpurun_out/ab_cols.log 2>&1; python tools/bench_brief.py gpurun_out/ab_cols.log
  LFM_SPLIT_GLOBAL=1 timeout 300 $B > gpurun_out/ab_glob.log 2>&1; python tools/bench_brief.py gpurun_out/ab_glob.log
done
python tools/prof_stage.py adj > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/adj_stage.csv python tools/prof_stage.py adj > /dev/null 2>&1; echo "NCU $?"
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/adj_stage.csv")))
hdr=None
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print("%-40s %-28s %s"%(d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"]))
PY
