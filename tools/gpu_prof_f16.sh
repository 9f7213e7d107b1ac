# 2xFP16 pipeline: launch list of the timed bench steps (time + DRAM bytes), full captures of band_u (fwd t pass)
# and the band_v pair
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph --profile-timed > gpurun_out/plain_bench.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_f16.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph --profile-timed > gpurun_out/ncu_launch.log 2>&1; echo "NCU LAUNCH $?"
python tools/prof_stage.py fwd > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:band_u -f \
    -o gpurun_out/prof_f16_fwd python tools/prof_stage.py fwd > gpurun_out/ncu_f16_fwd.log 2>&1; echo "NCU fwd $?"
python tools/prof_pair.py 0 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:band_v -f \
  -o gpurun_out/prof_f16_spass python tools/prof_pair.py 0 > gpurun_out/ncu_f16_spass.log 2>&1; echo "NCU spass $?"
