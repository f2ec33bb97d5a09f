# final multi-GPU bench lines (weak scaling n = 30 + log2 N, plus the n = 33 strong-scaling extra):
# bash tools/mg_bench_final.sh N
N=$1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1800 $TR --master-port 2958$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r2_final_bench_n$N.json 2> gpurun_out/r2_final_bench_n$N.err
grep "^{" gpurun_out/r2_final_bench_n$N.json | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']
print(d['n_gpus'], 'ms/layer', round(d['sec_per_layer']*1e3,2), 'value', d['value'], 'clk', d['clocks'].get('sm_mhz'),
 {k:(round(v['avg_ms'],2),v['launches'],v['moving_launches']) for k,v in r['per_pass_program'].items()})
print(json.dumps(d.get('extra_configs', {}))[:600])"
tail -2 gpurun_out/r2_final_bench_n$N.err
