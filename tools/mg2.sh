# 2-GPU checks: parity (mgpu_check) for the default (top-bit swap) and the opt-in low-bit swap
# schedule, then the bench line at N = 2
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
mkdir -p gpurun_out/mg2
timeout 900 $T --master-port 29521 tools/mgpu_check.py --qubits 18 24 31 --p 3 > gpurun_out/mg2/check_default.log 2>&1
echo check=$? >> gpurun_out/mg2/check_default.log
QSIM_LOWSWAP=1 timeout 900 $T --master-port 29522 tools/mgpu_check.py --qubits 23 31 --p 3 > gpurun_out/mg2/check_low.log 2>&1
echo check=$? >> gpurun_out/mg2/check_low.log
timeout 300 $T --master-port 29523 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/mg2/bench.log 2>&1
