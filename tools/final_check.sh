# one 2-GPU call: 1-GPU pytest + bench + smoke on GPU 0, then 2-GPU parity + bench
mkdir -p gpurun_out/fc
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fc/pytest.log 2>&1; echo pytest=$? >> gpurun_out/fc/pytest.log
CUDA_VISIBLE_DEVICES=0 python bench.py > gpurun_out/fc/bench_1.log 2>&1
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc/smoke.log 2>&1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29571 tools/mgpu_check.py --qubits 24 31 --p 3 > gpurun_out/fc/check_2.log 2>&1; echo check=$? >> gpurun_out/fc/check_2.log
timeout 400 $T --master-port 29572 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/fc/bench_2.log 2>&1
