# band_u L2 prefetch distance sweep (LFM_U_PF): stage times and pairs/s
for p in 0 4 8 16; do
  export LFM_U_PF=$p
  echo "pf $p: $(python tools/prof_stage.py fwd 0 4 2>&1 | tail -1) $(python tools/prof_stage.py adj 0 4 2>&1 | tail -1)"
  timeout 300 python bench.py --steps 200 --no-per-view --no-recon --no-cpu-baseline --no-e2e > gpurun_out/pf_$p.log 2>&1
  python tools/bench_brief.py gpurun_out/pf_$p.log | cut -c 1-200
done
