# multi-GPU measurements on N GPUs of one box: bash tools/mg_measure.sh N
N=$1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29511 tools/mgpu_check.py --qubits 21 24 2>&1 | grep -E "FAIL|swap path|rror" | head
QSIM_SWAP_INPLACE=1 timeout 900 $TR --master-port 29512 tools/mgpu_check.py --qubits 21 24 2>&1 | grep -E "FAIL|swap path|rror" | head
echo "== per-pass, fused split (out of place), n = 30 + log2 N"
timeout 600 $TR --master-port 29513 tools/mgpu_prof.py --nlocal 30 --p 8 --tag oop 2>&1 | grep "{"
echo "== per-pass, fused in place, n = 30 + log2 N"
QSIM_SWAP_INPLACE=1 timeout 600 $TR --master-port 29514 tools/mgpu_prof.py --nlocal 30 --p 8 --tag ip 2>&1 | grep "{"
echo "== per-pass, fused in place, n = 33 + log2 N (137 GB shard, the n = 36 / 8 GPU shape)"
timeout 1200 $TR --master-port 29515 tools/mgpu_prof.py --nlocal 33 --p 4 --tag ip33 2>&1 | grep -E "{|rror"
echo "== bench (weak scaling, n = 30 + log2 N)"
timeout 900 $TR --master-port 29516 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r2_bench_n$N.json 2> gpurun_out/r2_bench_n$N.err; tail -c 600 gpurun_out/r2_bench_n$N.json; tail -3 gpurun_out/r2_bench_n$N.err
