# split weights with the spatial split (n = 30 + log2 N on N GPUs): bash tools/sp_weights.sh N
N=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for w in 1,1,1 0.5,1,1 0,1,1 1,1.5,1 0.5,1.5,1 1,1,1; do
  echo "== QSIM_SPLIT_W=$w"
  QSIM_SPLIT_W=$w timeout 600 $TR --master-port 29541 tools/mgpu_prof.py --nlocal 30 --p 8 --tag w$w 2>&1 | grep "{" | head -1
done
