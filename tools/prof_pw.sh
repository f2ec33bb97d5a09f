./tools/dmma_probe > gpurun_out/r2_dmma_probe.jsonl 2>&1; cat gpurun_out/r2_dmma_probe.jsonl
python tools/passbench.py --n 30 --reps 1 > gpurun_out/r2_pw_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tma_turn_pw -s 1 -c 1 -o gpurun_out/r2_pw_prof python tools/passbench.py --n 30 --reps 1 > gpurun_out/r2_pw_ncu.log 2>&1; tail -3 gpurun_out/r2_pw_ncu.log
