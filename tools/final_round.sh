# round-end evidence on one B200: the bench line, the ncu launch list + full capture of the pass
# kernels (tools/profile_round.sh), and ncu of the DMMA-vs-butterfly probe
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_final_bench.json 2> gpurun_out/r2_final_bench.err; tail -c 300 gpurun_out/r2_final_bench.json
bash tools/profile_round.sh gpurun_out/prof_r2b
./tools/dmma_probe > gpurun_out/r2_dmma_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor.sum,smsp__inst_executed.sum \
    -k regex:"bfly_kernel|dmma_kernel" -s 1 -c 3 --csv --log-file gpurun_out/r2_dmma_ncu.csv ./tools/dmma_probe > gpurun_out/r2_dmma_ncu.log 2>&1; tail -3 gpurun_out/r2_dmma_ncu.log
