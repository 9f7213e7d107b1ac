# 2xFP16 band_u drain-group sweep: stage times and the bench line per LFM_U16_GROUP
mkdir -p gpurun_out
for g in 8 12 16; do
  export LFM_U16_GROUP=$g
  python tools/prof_stage.py fwd 0 4 2>&1 | tail -1; python tools/prof_stage.py adj 0 4 2>&1 | tail -1
  timeout 300 python bench.py --steps 200 --no-per-view --no-recon --no-cpu-baseline --no-e2e > gpurun_out/g16_$g.log 2>&1
  python tools/bench_brief.py gpurun_out/g16_$g.log
done
