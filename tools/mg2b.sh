T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
mkdir -p gpurun_out/mg2b
timeout 900 $T --master-port 29591 tools/mgpu_check.py --qubits 24 31 --p 3 > gpurun_out/mg2b/check.log 2>&1; echo check=$? >> gpurun_out/mg2b/check.log
timeout 400 $T --master-port 29592 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/mg2b/bench.log 2>&1
for w in 1,0.8,1.2 1.2,1,0.8 1,1.2,0.8; do QSIM_SPLIT_W=$w timeout 300 $T --master-port 29593 tools/mgpu_prof.py --tag w_$w >> gpurun_out/mg2b/prof.log 2>&1; done
