TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for sp in 0.12 0.18 0.35 0; do
  QSIM_SP=$sp timeout 600 $TR --master-port 29553 tools/mgpu_prof.py --nlocal 31 --p 8 --tag m31sp$sp 2>&1 | grep "{" | head -1
done
