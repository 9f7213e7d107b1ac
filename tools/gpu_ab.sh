# A/B of environment settings on the bench: bash tools/gpu_ab.sh "ENV1=.. ENV2=.." "ENV3=.." ...
mkdir -p gpurun_out
for e in "$@"; do
  echo "== $e"
  env $e LFM_DEBUG_TUNE=1 LFM_DEBUG=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-per-view --no-e2e > gpurun_out/ab.log 2> gpurun_out/ab.err
  python -c "import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('pairs/s %.1f' % d['value'])"
  grep "direct s" gpurun_out/ab.err | head -2
done
