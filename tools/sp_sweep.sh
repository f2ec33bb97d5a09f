# spatial split of the whole-tile moving run passes: per-pass timing at n = 30 + log2 N on N GPUs,
# default share (the moving-tile fraction) against the group-bits-first order (QSIM_SP=0), twice
# each: bash tools/sp_sweep.sh N
N=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for sp in 1 0 1 0; do
  echo "== QSIM_SP=$sp"
  QSIM_SP=$sp timeout 600 $TR --master-port 29522 tools/mgpu_prof.py --nlocal 30 --p 8 --tag sp$sp 2>&1 | grep "{" | head -1
done
