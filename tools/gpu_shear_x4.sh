# x-pass float4 kernel: rotation parity (forced on and off), warm rotation timing, bench A/B
mkdir -p gpurun_out
for v in 1 0; do
  echo "== LFM_SH_X4=$v"
  LFM_SH_X4=$v timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_oracle_rotation.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1
  LFM_SH_X4=$v timeout 300 python tools/part_timing.py 2>&1 | grep -i "rot" | head -4
done
bash tools/gpu_ab.sh "LFM_SH_X4=1" "LFM_SH_X4=0" "LFM_SH_X4=1" "LFM_SH_X4=0" 2>&1 | grep -v "direct s"
