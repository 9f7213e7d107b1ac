# same-box A/B of the working tree's liblfm.so against liblfm_head.so (the last commit), interleaved; the GPU suite
# on the working tree first
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo "TESTS EXIT $?"; tail -2 gpurun_out/ab_tests.log
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2 3; do
  timeout 300 $B > gpurun_out/ab_new.log 2>&1; echo "new"; python tools/bench_brief.py gpurun_out/ab_new.log
  LFM_LIB=paper_1812_03358_b200/liblfm_head.so timeout 300 $B > gpurun_out/ab_head.log 2>&1; echo "head"; python tools/bench_brief.py gpurun_out/ab_head.log
done
for L in liblfm.so liblfm_head.so; do
LFM_LIB=paper_1812_03358_b200/$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/ab_$L.csv python tools/prof_pair.py 1 > /dev/null 2>&1; echo "NCU $L $?"
python - $L <<'PY'
import csv, sys
rows=list(csv.reader(open("gpurun_out/ab_%s.csv" % sys.argv[1])))
hdr=None; out={}
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); out.setdefault((d["ID"], d["Kernel Name"][:40]), {})[d["Metric Name"]]=float(d["Metric Value"].replace(",",""))
for (i,k),m in out.items(): print("%-40s %8.1f us %8.1f MB" % (k, m.get("gpu__time_duration.sum",0)/1e3, (m.get("dram__bytes_read.sum",0)+m.get("dram__bytes_write.sum",0))/1e6))
PY
done
