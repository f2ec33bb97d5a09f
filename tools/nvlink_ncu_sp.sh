# NVLink + DRAM counters of the moving passes with the spatial split (2 GPUs, one process): run
# once without ncu, then the ncu launch list with the counters (tools/nvlink_ncu.py)
timeout 300 python tools/nvlink_ncu.py --n 31 --p 2 > gpurun_out/r2_nvlink_sp_plain.log 2>&1 || { tail -5 gpurun_out/r2_nvlink_sp_plain.log; exit 1; }
tail -2 gpurun_out/r2_nvlink_sp_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:tma_pass --csv --log-file gpurun_out/r2_nvlink_ncu_sp.csv python tools/nvlink_ncu.py --n 31 --p 2 > gpurun_out/r2_nvlink_ncu_sp.log 2>&1
tail -3 gpurun_out/r2_nvlink_ncu_sp.log; wc -l gpurun_out/r2_nvlink_ncu_sp.csv
