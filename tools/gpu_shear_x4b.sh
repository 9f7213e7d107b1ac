# x4 shear z-chunk A/B (LFM_SH_X4 = 1: 8 z, 2: 4 z, 3: 16 z): rotation parity, warm rotation time, bench
mkdir -p gpurun_out
for v in 2 4 5; do
  echo "== LFM_SH_X4=$v"
  LFM_SH_X4=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
  LFM_SH_X4=$v timeout 300 python tools/part_timing.py 2>&1 | grep -i "rotate" | head -2
done
bash tools/gpu_ab.sh "LFM_SH_X4=2" "LFM_SH_X4=4" "LFM_SH_X4=5" "LFM_SH_X4=2" 2>&1 | grep -v "direct s"
