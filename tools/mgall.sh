# multi-GPU validation + bench lines: 4 GPUs then 2 GPUs (parity via mgpu_check, bench, per-pass)
mkdir -p gpurun_out/mga
for NG in 4 2; do
  if [ $NG = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; QB="24 31"; else QB="20 32"; fi
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
  timeout 900 $T --master-port 29561 tools/mgpu_check.py --qubits $QB --p 3 > gpurun_out/mga/check_$NG.log 2>&1
  echo check=$? >> gpurun_out/mga/check_$NG.log
  timeout 400 $T --master-port 29562 bench.py --gpus $NG --steps 3 --warmup 3 > gpurun_out/mga/bench_$NG.log 2>&1
  timeout 300 $T --master-port 29563 tools/mgpu_prof.py --tag final > gpurun_out/mga/prof_$NG.log 2>&1
done
