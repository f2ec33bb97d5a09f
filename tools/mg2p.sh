# 2-GPU per-pass profile of the multi-GPU layer for several schedules
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
mkdir -p gpurun_out/mg2
for sh in ${SHARES:-0.5}; do
QSIM_LS_SHARE=$sh timeout 300 $T --master-port 29531 tools/mgpu_prof.py --tag low_$sh >> gpurun_out/mg2/prof.log 2>&1
done
QSIM_LOWSWAP=0 timeout 300 $T --master-port 29532 tools/mgpu_prof.py --tag old >> gpurun_out/mg2/prof.log 2>&1
