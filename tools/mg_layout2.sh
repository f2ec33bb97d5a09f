TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29551 tools/mgpu_prof.py --nlocal 30 --p 8 --tag default 2>&1 | grep "{" | head -1
QSIM_SPLIT_W=1,0,1 timeout 600 $TR --master-port 29552 tools/mgpu_prof.py --nlocal 30 --p 8 --tag w101 2>&1 | grep "{" | head -1
QSIM_SPLIT_W=1,1,0 timeout 600 $TR --master-port 29553 tools/mgpu_prof.py --nlocal 30 --p 8 --tag w110 2>&1 | grep "{" | head -1
QSIM_RUNSPLIT=4 timeout 600 $TR --master-port 29554 tools/mgpu_prof.py --nlocal 30 --p 8 --tag runsplit4 2>&1 | grep "{" | head -1
QSIM_RUNSPLIT=4 QSIM_SPLIT_W=1,1,2 timeout 600 $TR --master-port 29555 tools/mgpu_prof.py --nlocal 30 --p 8 --tag runsplit4_w112 2>&1 | grep "{" | head -1
QSIM_RUNSPLIT=4 timeout 600 $TR --master-port 29556 tools/mgpu_check.py --qubits 31 2>&1 | grep -E "FAIL|swap path|rror" | head
