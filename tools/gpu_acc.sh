# float4 vol_accumulate: concurrent-pair tests, then the bench A/B against the previous build's number
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_concurrent.py tests/test_gpu_pwls.py tests/test_gpu_recon.py -x -q 2>&1 | tail -1
bash tools/gpu_ab.sh "LFM_SH_X4=4" "LFM_SH_X4=4" 2>&1 | grep -v "direct s"
