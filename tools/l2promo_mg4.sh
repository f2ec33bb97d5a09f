# L2 promotion of the run sets' maps on 4 GPUs (n = 32, fused split + spatial split)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for v in 256 128 256 128; do
  QSIM_L2PROMO=$v timeout 600 $TR --master-port 29581 tools/mgpu_prof.py --nlocal 30 --p 8 --tag g4oop$v 2>&1 | grep "{" | head -1
done
