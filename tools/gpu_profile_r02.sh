# Round-2 evidence pass on one B200: GPU suite, smoke, bench line (+ reference arm), launch list of the timed
# steps, ncu --set full of the dominant kernels, per-kernel DRAM bytes (128^3 pair kernels and the 256^3 HBM-bound
# kernels), PCIe copy roof, shard / NEXT timings.  Summaries: tools/summarize_profiles.py r02 ... (here, after).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -ra > gpurun_out/gpu_tests.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE $?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err; echo "BENCH EXIT $?"
tail -c 400 gpurun_out/bench_final.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "REF EXIT $?"
timeout 120 python tools/pcie_roof.py > gpurun_out/pcie_roof.json 2>&1; echo "PCIE EXIT $?"
timeout 900 python tools/hbm_kernels.py > gpurun_out/hbm_kernels.json 2> gpurun_out/hbm_kernels.err; echo "HBM EXIT $?"
timeout 600 python tools/shard_timing.py 1 > gpurun_out/shard_timing.json 2> gpurun_out/shard_timing.err; echo "SHARD EXIT $?"
timeout 900 python tools/next_timing.py > gpurun_out/next_timing.json 2> gpurun_out/next_timing.err; echo "NEXT EXIT $?"
LC="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph --profile-timed"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches.csv $LC > gpurun_out/ncu_launch.log 2>&1; echo "NCU LAUNCH EXIT $?"
for st in fwd adj; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"band_u|split" -f \
    -o gpurun_out/prof_$st python tools/prof_stage.py $st > gpurun_out/ncu_$st.log 2>&1; echo "NCU $st EXIT $?"
done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:band_v -f \
  -o gpurun_out/prof_spass python tools/prof_pair.py 0 > gpurun_out/ncu_spass.log 2>&1; echo "NCU spass EXIT $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --profile-from-start off --log-file gpurun_out/pair_dram.csv python tools/prof_pair.py 1 > gpurun_out/ncu_pd.log 2>&1; echo "NCU PD EXIT $?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"shear|band_v|stats|reduce_final|reg26|fista|copy_scale|fill_kernel" -c 400 --log-file gpurun_out/hbm_dram.csv \
  python tools/hbm_kernels.py > gpurun_out/ncu_hd.log 2>&1; echo "NCU HD EXIT $?"
