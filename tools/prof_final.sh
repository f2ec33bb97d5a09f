bash tools/profile_round.sh gpurun_out/prof_r2
ls gpurun_out/prof_r2
