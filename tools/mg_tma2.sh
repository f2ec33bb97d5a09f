timeout 1500 python -m pytest tests/test_gpu_loopback.py -x -q 2>&1 | tail -3
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29541 tools/mgpu_check.py --qubits 21 24 2>&1 | grep -E "FAIL|swap path|rror" | head
QSIM_SWAP_INPLACE=1 timeout 900 $TR --master-port 29542 tools/mgpu_check.py --qubits 21 24 2>&1 | grep -E "FAIL|swap path|rror" | head
timeout 600 $TR --master-port 29543 tools/mgpu_prof.py --nlocal 30 --p 8 --tag oop_tma 2>&1 | grep "{" | head -1
QSIM_TMA_MOVES=0 timeout 600 $TR --master-port 29544 tools/mgpu_prof.py --nlocal 30 --p 8 --tag oop_stg 2>&1 | grep "{" | head -1
QSIM_SWAP_INPLACE=1 timeout 600 $TR --master-port 29545 tools/mgpu_prof.py --nlocal 30 --p 8 --tag ip_tma 2>&1 | grep "{" | head -1
timeout 1200 $TR --master-port 29546 tools/mgpu_prof.py --nlocal 33 --p 4 --tag ip33_tma 2>&1 | grep -E "{|rror" | head -1
