# spatial split at n = 31 + log2 N (m = 31 per GPU: four tile sets), default share vs QSIM_SP=0
N=${1:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for sp in 1 0 1 0; do
  echo "== QSIM_SP=$sp"
  QSIM_SP=$sp timeout 600 $TR --master-port 29552 tools/mgpu_prof.py --nlocal ${NL:-31} --p 8 --tag m${NL:-31}sp$sp 2>&1 | grep "{" | head -1
done
