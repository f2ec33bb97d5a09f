# multi-GPU bench lines (N from $NG) for profiles/
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1"
mkdir -p gpurun_out/mgb
timeout 400 $T --master-port 29551 bench.py --gpus ${NG:-2} --steps 3 --warmup 3 > gpurun_out/mgb/bench_${NG:-2}.log 2>&1
timeout 300 $T --master-port 29552 tools/mgpu_prof.py --tag final > gpurun_out/mgb/prof_${NG:-2}.log 2>&1
