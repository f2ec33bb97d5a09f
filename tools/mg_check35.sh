TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 2400 $TR --master-port 29581 tools/mgpu_check.py --qubits 35 --p 3 2>&1 | grep -E "PASS|FAIL|rror" | head -20
