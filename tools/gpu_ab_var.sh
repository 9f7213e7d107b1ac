# same-box A/B of the working tree's liblfm.so against an experiment build liblfm_var.so (LFM_NVCC_DEFS): parity
# of the variant first, then interleaved bench lines
mkdir -p gpurun_out
LFM_LIB=paper_1812_03358_b200/liblfm_var.so timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_windowed.py -q -x > gpurun_out/var_tests.log 2>&1; echo "VAR TESTS EXIT $?"; tail -2 gpurun_out/var_tests.log
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2 3; do
  timeout 300 $B > gpurun_out/ab_new.log 2>&1; echo "default"; python tools/bench_brief.py gpurun_out/ab_new.log | cut -c1-160
  LFM_LIB=paper_1812_03358_b200/liblfm_var.so timeout 300 $B > gpurun_out/ab_var.log 2>&1; echo "variant"; python tools/bench_brief.py gpurun_out/ab_var.log | cut -c1-160
done
