python tools/passbench.py --n 30 --f32 > gpurun_out/pb_f32b.log 2>&1
timeout 600 python tools/fp32_check.py > gpurun_out/fp32_check_b.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_b.log 2>&1
python tools/passbench.py --n 31 32 33 > gpurun_out/pb_bal.log 2>&1
python bench.py --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f32.log 2>&1
