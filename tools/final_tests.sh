# round-end parity evidence on a 2-B200 box: the whole GPU suite (single-GPU parity, loopback swap
# paths, debug build, determinism, and the torchrun NCCL tests that need >= 2 GPUs)
timeout 3000 python -m pytest tests -m gpu -q -rs 2>&1 | tail -15 | tee gpurun_out/r2_final_pytest_gpu.log
