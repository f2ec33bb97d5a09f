set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29501 tools/mgpu_check.py --qubits 20 24 31 2>&1 | grep -E "PASS|FAIL|Error|error" | head -60
QSIM_SWAP_INPLACE=1 timeout 900 $TR --master-port 29502 tools/mgpu_check.py --qubits 20 24 31 2>&1 | grep -E "PASS|FAIL|Error|error" | head -60
timeout 600 $TR --master-port 29503 tools/mgpu_prof.py --nlocal 30 --p 8 --tag oop 2>&1 | grep "{"
QSIM_SWAP_INPLACE=1 timeout 600 $TR --master-port 29504 tools/mgpu_prof.py --nlocal 30 --p 8 --tag ip 2>&1 | grep "{"
timeout 900 $TR --master-port 29505 tools/mgpu_prof.py --nlocal 33 --p 4 --tag ip34 2>&1 | grep -E "{|rror"
