# weight images by tensor-map boxes instead of bulk copies (LFM_U_WTMA band_u, LFM_V_WTMA band_v): parity with both
# on, bench A/B, TMA rate microbenchmark
mkdir -p gpurun_out
timeout 60 ./tools/microbench/tma_rate.bin
LFM_U_WTMA=1 LFM_V_WTMA=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_windowed.py tests/test_gpu_variants.py -q -x > gpurun_out/w_tests.log 2>&1; echo "TESTS WTMA EXIT $?"; tail -3 gpurun_out/w_tests.log
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2; do
  timeout 300 $B > gpurun_out/w0.log 2>&1; echo "default"; python tools/bench_brief.py gpurun_out/w0.log
  LFM_U_WTMA=1 timeout 300 $B > gpurun_out/wu.log 2>&1; echo "U_WTMA"; python tools/bench_brief.py gpurun_out/wu.log
  LFM_V_WTMA=1 timeout 300 $B > gpurun_out/wv.log 2>&1; echo "V_WTMA"; python tools/bench_brief.py gpurun_out/wv.log
  LFM_U_WTMA=1 LFM_V_WTMA=1 timeout 300 $B > gpurun_out/wuv.log 2>&1; echo "UV_WTMA"; python tools/bench_brief.py gpurun_out/wuv.log
done
