# 4-GPU per-pass profile of the top-bit split-swap weights (boundary, R1, S0)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
mkdir -p gpurun_out/mg4
for w in ${WEIGHTS:-default}; do
  if [ "$w" = default ]; then timeout 300 $T --master-port 29541 tools/mgpu_prof.py --tag w_default >> gpurun_out/mg4/prof.log 2>&1
  else QSIM_SPLIT_W=$w timeout 300 $T --master-port 29541 tools/mgpu_prof.py --tag w_$w >> gpurun_out/mg4/prof.log 2>&1; fi
done
timeout 300 $T --master-port 29542 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/mg4/bench.log 2>&1
