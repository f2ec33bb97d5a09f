N=$1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 $TR --master-port 2957$N bench.py --gpus $N --nlocal 33 --steps 3 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r2_bench33_n$N.json 2> gpurun_out/r2_bench33_n$N.err
grep "^{" gpurun_out/r2_bench33_n$N.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['config']['n'], d['n_gpus'], 'ms/layer', round(d['sec_per_layer']*1e3,2), 'value', d['value'], 'swap', d['nvlink']['swap_path'],
 {k:(round(v['avg_ms'],2),v['launches'],v['moving_launches']) for k,v in r['per_pass_program'].items()})"
tail -2 gpurun_out/r2_bench33_n$N.err
