# L2 promotion of the run sets' maps on 2 GPUs (n = 31, fused split and fused in place)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for v in 256 128 256 128; do
  QSIM_L2PROMO=$v timeout 600 $TR --master-port 29561 tools/mgpu_prof.py --nlocal 30 --p 8 --tag oop$v 2>&1 | grep "{" | head -1
  QSIM_L2PROMO=$v QSIM_SWAP_INPLACE=1 timeout 600 $TR --master-port 29562 tools/mgpu_prof.py --nlocal 30 --p 8 --tag ip$v 2>&1 | grep "{" | head -1
done
