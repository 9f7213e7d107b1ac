set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_windowed.py tests/test_gpu_shear.py -q -ra > gpurun_out/t_hex.log 2>&1; echo "T EXIT $?" >> gpurun_out/t_hex.log
tail -25 gpurun_out/t_hex.log
