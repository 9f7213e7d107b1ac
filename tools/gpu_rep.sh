# repeatability: bench twice + stage times
for i in 1 2; do
  echo "$(python tools/prof_stage.py fwd 0 4 2>&1 | tail -1) $(python tools/prof_stage.py adj 0 4 2>&1 | tail -1)"
  timeout 300 python bench.py --steps 200 --no-per-view --no-recon --no-cpu-baseline --no-e2e > gpurun_out/rep_$i.log 2>&1
  python tools/bench_brief.py gpurun_out/rep_$i.log | cut -c 1-200
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pci.bus_id --format=csv
