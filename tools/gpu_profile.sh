# Profiling pass (one GPU): tune cache -> bench line -> ncu launch list -> ncu --set full of both t-pass stages.
#   gpurun -- 'bash tools/gpu_profile.sh'      (results in gpurun_out/)
mkdir -p gpurun_out
export LFM_TUNE_FILE=/tmp/lfm_tune.txt
rm -f $LFM_TUNE_FILE
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1; echo "BENCH EXIT $?"
tail -1 gpurun_out/prof_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-per-view > gpurun_out/ncu_launch.log 2>&1; echo "NCU LAUNCH EXIT $?"
python tools/launches.py gpurun_out/launches.csv | head -20
for st in fwd adj; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o gpurun_out/prof_$st \
    python tools/prof_stage.py $st > gpurun_out/ncu_$st.log 2>&1; echo "NCU $st EXIT $?"
done
# the s passes (band_v, tcgen05): one forward and one adjoint launch
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:band_v -f \
  -o gpurun_out/prof_spass python tools/prof_pair.py 0 > gpurun_out/ncu_spass.log 2>&1; echo "NCU spass EXIT $?"
