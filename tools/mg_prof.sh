# per-pass timing of the multi-GPU layer (NG GPUs): split swap off / default / weight variants
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1"
QSIM_SPLIT_SWAP=0 timeout 300 $T --master-port 29511 tools/mgpu_prof.py --tag nosplit
timeout 300 $T --master-port 29512 tools/mgpu_prof.py --tag split_default
for w in $WEIGHTS; do QSIM_SPLIT_W=$w timeout 300 $T --master-port 29513 tools/mgpu_prof.py --tag split_$w; done
