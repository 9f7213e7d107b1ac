# same-box A/B of a bench environment variable: tools/gpu_ab_env.sh "VAR=value" (interleaved, 3 rounds)
mkdir -p gpurun_out
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2 3; do
  timeout 300 $B > gpurun_out/ab0.log 2>&1; echo "default"; python tools/bench_brief.py gpurun_out/ab0.log | cut -c1-60
  env $1 timeout 300 $B > gpurun_out/ab1.log 2>&1; echo "$1"; python tools/bench_brief.py gpurun_out/ab1.log | cut -c1-60
done
