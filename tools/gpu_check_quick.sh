# GPU parity suite + two bench lines (no CPU baseline / recon) + the PCIe copy roof of the e2e line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/q_tests.log 2>&1; echo "TESTS EXIT $?"; tail -3 gpurun_out/q_tests.log
B="python bench.py --steps 300 --no-per-view --no-recon --no-cpu-baseline --no-e2e"
for i in 1 2; do timeout 300 $B > gpurun_out/q_bench.log 2>&1; python tools/bench_brief.py gpurun_out/q_bench.log; done
timeout 120 python tools/pcie_roof.py > gpurun_out/pcie_roof.json 2>&1; cat gpurun_out/pcie_roof.json
