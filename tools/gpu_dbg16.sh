export CUDA_LAUNCH_BLOCKING=1
for v in "LFM_DBG_SKIP_V=1" "LFM_NO_X16=1"; do
  echo "== $v"; env $v timeout 120 python tools/dbg_f16.py small_two 2>&1 | grep -E "ok|Error|error" | head -6
done
