# band_v adjoint 2xFP16 K blocks of 64 (128-byte Z rows) vs 32 (LFM_VBK_A): parity, bench A/B, stage times under ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -k "block_width or stage_entry" -q -x -ra > gpurun_out/vbk_tests.log 2>&1; echo "TESTS EXIT $?"; tail -3 gpurun_out/vbk_tests.log
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2; do
  for bk in 32 64; do
    LFM_VBK_A=$bk timeout 300 $B > gpurun_out/ab_vbk$bk.log 2>&1; echo "VBK_A=$bk"; python tools/bench_brief.py gpurun_out/ab_vbk$bk.log
  done
done
for bk in 32 64; do
LFM_VBK_A=$bk timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:band_v --csv \
  --log-file gpurun_out/vbk_$bk.csv python tools/prof_pair.py 1 > /dev/null 2>&1; echo "NCU $bk $?"
python - $bk <<'PY'
import csv, sys
rows=list(csv.reader(open("gpurun_out/vbk_%s.csv" % sys.argv[1])))
hdr=None
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print("%-44s %-28s %s"%(d["Kernel Name"][:44], d["Metric Name"], d["Metric Value"]))
PY
done
