# same-box A/B of the working tree's liblfm.so against an experiment build liblfm_var.so (LFM_NVCC_DEFS), interleaved
mkdir -p gpurun_out
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2 3; do
  timeout 300 $B > gpurun_out/ab_new.log 2>&1; echo "default"; python tools/bench_brief.py gpurun_out/ab_new.log | cut -c1-200
  LFM_LIB=paper_1812_03358_b200/liblfm_var.so timeout 300 $B > gpurun_out/ab_var.log 2>&1; echo "variant"; python tools/bench_brief.py gpurun_out/ab_var.log | cut -c1-200
done
