# spatial split on the in-place swap path: loopback parity (1 GPU), NCCL check, then n = 34 (137 GB
# shard per GPU, in place) per-pass timing on 2 GPUs, default share vs QSIM_SP=0
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -m gpu -x 2>&1 | tail -2
QSIM_SWAP_INPLACE=1 timeout 600 $TR --master-port 29531 tools/mgpu_check.py --qubits 21 24 2>&1 | grep -E "FAIL|PASS|rror" | head -5
for sp in 1 0; do
  echo "== QSIM_SP=$sp"
  QSIM_SP=$sp timeout 900 $TR --master-port 29532 tools/mgpu_prof.py --nlocal 33 --p 4 --tag ip34sp$sp 2>&1 | grep -E "\{|rror" | head -1
done
