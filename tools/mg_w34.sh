N=$1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in "0,0,1,1" "0,0.5,1,1" "0,1,1,1" "0,0.5,1,1.5"; do
QSIM_SPLIT_W=$W timeout 1200 $TR --master-port 2956$N tools/mgpu_prof.py --nlocal 33 --p 4 --tag ip33w 2>&1 | grep -E "{|rror" | head -1
done
