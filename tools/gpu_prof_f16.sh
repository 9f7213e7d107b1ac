# 2xFP16 band_u: plain stage timings, then the launch list of the timed bench steps and full captures of band_u
mkdir -p gpurun_out
python tools/prof_stage.py fwd 0 5 && python tools/prof_stage.py adj 0 5 > gpurun_out/stage_plain.log 2>&1; cat gpurun_out/stage_plain.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph --profile-timed > gpurun_out/plain_bench.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_f16.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-per-view --no-recon --no-graph --profile-timed > gpurun_out/ncu_launch.log 2>&1; echo "NCU LAUNCH $?"
for st in fwd adj; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:band_u -f \
    -o gpurun_out/prof_f16_$st python tools/prof_stage.py $st > gpurun_out/ncu_f16_$st.log 2>&1; echo "NCU $st $?"
done
