set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_windowed.py tests/test_gpu_parity.py -q -ra -x > gpurun_out/t_sk.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_sk.log
tail -4 gpurun_out/t_sk.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/win_launches.csv python tools/win_breakdown.py > gpurun_out/ncu_win.log 2>&1; echo "NCU EXIT $?"
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/win_launches.csv")))
hdr=None
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get("Metric Name")=="gpu__time_duration.sum": print("%-50s %8.1f"%(d["Kernel Name"][:50], float(d["Metric Value"].replace(",",""))/1e3))
PY
timeout 600 python tools/shard_timing.py 1 > gpurun_out/shard_timing.json 2> gpurun_out/shard_timing.err; echo "SHARD EXIT $?"
cat gpurun_out/shard_timing.json
timeout 900 python tools/next_timing.py > gpurun_out/next_timing.json 2> gpurun_out/next_timing.err; echo "NEXT EXIT $?"
cat gpurun_out/next_timing.json; tail -3 gpurun_out/next_timing.err
