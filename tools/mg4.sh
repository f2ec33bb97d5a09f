T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 400 $T2 --master-port 29520 tools/mgpu_check.py --qubits 23 > gpurun_out/mg4_w2.log 2>&1
timeout 600 $T4 --master-port 29521 tools/mgpu_check.py --qubits 18 20 23 > gpurun_out/mg4_w4.log 2>&1
NG=4 WEIGHTS="0,1,1 0.5,1,1 1,1.2,1" bash tools/mg_prof.sh > gpurun_out/mg4_prof.jsonl 2> gpurun_out/mg4_prof.err
timeout 600 $T4 --master-port 29530 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/b4_mv.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fp32.py -x -q > gpurun_out/fp32_tests.log 2>&1
