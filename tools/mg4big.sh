# n = 35 on 4 GPUs: 137 GB shard per GPU (the per-GPU shape of n = 36 on 8 GPUs): the second shard
# buffer does not fit, so the swap runs in place through the bounded staging ring (NCCL)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
mkdir -p gpurun_out/big4
timeout 1200 $T --master-port 29601 tools/mgpu_check.py --qubits 35 --p 2 > gpurun_out/big4/check.log 2>&1; echo check=$? >> gpurun_out/big4/check.log
timeout 900 $T --master-port 29602 bench.py --gpus 4 --nlocal 33 --p 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/big4/bench.log 2>&1; echo bench=$? >> gpurun_out/big4/bench.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/big4/check.log
