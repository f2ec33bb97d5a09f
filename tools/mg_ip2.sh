TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
QSIM_SWAP_INPLACE=1 timeout 600 $TR --master-port 29524 tools/mgpu_prof.py --nlocal 30 --p 8 --tag ip 2>&1 | grep "{"
timeout 1200 $TR --master-port 29525 tools/mgpu_prof.py --nlocal 33 --p 4 --tag ip33 2>&1 | grep -E "{|rror"
timeout 900 $TR --master-port 29526 bench.py --gpus 2 --steps 3 --warmup 3 --no-extras > gpurun_out/r2_bench_n2b.json 2>&1; grep "^{" gpurun_out/r2_bench_n2b.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['sec_per_layer'], d['nvlink'])"
python tools/nvlink_ncu.py --n 31 --p 2 > gpurun_out/r2_nvl_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:tma_pass --csv --log-file gpurun_out/r2_nvlink_ncu.csv python tools/nvlink_ncu.py --n 31 --p 2 > gpurun_out/r2_nvl_ncu.log 2>&1; tail -2 gpurun_out/r2_nvl_plain.log gpurun_out/r2_nvl_ncu.log
