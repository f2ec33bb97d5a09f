TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in "0,1,1,1" "0.5,1,1,1" "0,1,1.5,1.5"; do
QSIM_SPLIT_W=$W timeout 1200 $TR --master-port 29531 tools/mgpu_prof.py --nlocal 33 --p 4 --tag ip33w 2>&1 | grep -E "{|rror" | head -1
done
for W in "0,1,1" "1,1,1"; do
QSIM_SWAP_INPLACE=1 QSIM_SPLIT_W=$W timeout 600 $TR --master-port 29532 tools/mgpu_prof.py --nlocal 30 --p 8 --tag ip30w 2>&1 | grep -E "{|rror" | head -1
done
