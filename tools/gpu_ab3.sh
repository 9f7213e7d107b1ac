set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shear.py -q -ra -x > gpurun_out/t_shear.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_shear.log
tail -3 gpurun_out/t_shear.log
timeout 300 python tools/ab_stage.py paper_1812_03358_b200/liblfm.so > gpurun_out/ab3.log 2>&1
LFM_ROT_FUSE=0 timeout 300 python tools/ab_stage.py paper_1812_03358_b200/liblfm.so >> gpurun_out/ab3.log 2>&1
cat gpurun_out/ab3.log
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
