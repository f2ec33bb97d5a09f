# 2-GPU per-pass profile of the top-bit split-swap weights (boundary, R1, S0)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
mkdir -p gpurun_out/mg2w
for w in ${WEIGHTS:-default}; do
  if [ "$w" = default ]; then timeout 300 $T --master-port 29581 tools/mgpu_prof.py --tag w_default >> gpurun_out/mg2w/prof.log 2>&1
  else QSIM_SPLIT_W=$w timeout 300 $T --master-port 29581 tools/mgpu_prof.py --tag w_$w >> gpurun_out/mg2w/prof.log 2>&1; fi
done
