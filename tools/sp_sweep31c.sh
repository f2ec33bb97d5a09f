# m = 31 on 4 GPUs with 256-byte promotion: spatial split (forced share) vs the default (off)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for sp in 0.25 1 0.18 1; do
  QSIM_SP=$sp timeout 600 $TR --master-port 29571 tools/mgpu_prof.py --nlocal 31 --p 8 --tag m31sp$sp 2>&1 | grep "{" | head -1
done
