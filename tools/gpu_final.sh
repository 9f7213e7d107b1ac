# end-of-session pass: GPU suite, bench line, smoke, then the profiling pass (tools/gpu_profile.sh)
bash tools/gpu_round.sh
bash tools/gpu_profile.sh
