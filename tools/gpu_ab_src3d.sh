# GPU suite on the default build; 3D-box band_u source loads (LFM_U_SRC3D=1): full-size parity + bench A/B;
# TMA rate microbenchmark (2D / bulk / 3D boxes)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3_tests.log 2>&1; echo "TESTS EXIT $?"; tail -3 gpurun_out/s3_tests.log
LFM_U_SRC3D=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_windowed.py -q -x > gpurun_out/s3_tests3d.log 2>&1; echo "TESTS 3D EXIT $?"; tail -3 gpurun_out/s3_tests3d.log
timeout 60 ./tools/microbench/tma_rate.bin
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2; do
  timeout 300 $B > gpurun_out/s3_def.log 2>&1; echo "default"; python tools/bench_brief.py gpurun_out/s3_def.log
  LFM_U_SRC3D=1 timeout 300 $B > gpurun_out/s3_3d.log 2>&1; echo "SRC3D"; python tools/bench_brief.py gpurun_out/s3_3d.log
done
