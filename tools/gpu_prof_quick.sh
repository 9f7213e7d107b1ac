# ncu --set full (source-level) of the t passes (band_u fwd / adj stages) and the band_v pair, current build
mkdir -p gpurun_out
for st in fwd adj; do
  python tools/prof_stage.py $st > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"band_u|split" -f \
    -o gpurun_out/pq_$st python tools/prof_stage.py $st > gpurun_out/pq_$st.log 2>&1; echo "NCU $st $?"
done
python tools/prof_pair.py 0 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:band_v -f \
  -o gpurun_out/pq_spass python tools/prof_pair.py 0 > gpurun_out/pq_spass.log 2>&1; echo "NCU spass $?"
