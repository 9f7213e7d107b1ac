# shear z-chunk A/B: rotation parity, warm piece timings and the bench for LFM_SH_ZC = 8 / 16 / 32
mkdir -p gpurun_out
for zc in 8 16 32; do
  echo "== LFM_SH_ZC=$zc"
  LFM_SH_ZC=$zc timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
  LFM_SH_ZC=$zc timeout 300 python tools/part_timing.py 2>&1 | grep -i "rot" | head -4
done
bash tools/gpu_ab.sh "LFM_SH_ZC=8" "LFM_SH_ZC=16" "LFM_SH_ZC=32" "LFM_SH_ZC=8" 2>&1 | grep -v "direct s"
