timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -x -q -k "not loopback" 2>&1 | tail -2
timeout 300 python tools/passbench.py --n 30 --reps 5 2>&1 | grep -E "phase=1 "
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r2_pw_bench.json 2>gpurun_out/r2_pw_bench.err; python -c "
import json; d=json.load(open('gpurun_out/r2_pw_bench.json')); r=d['roofline']
print(d['sec_per_layer'], d['value'], r['frac'], {k:(v['avg_ms'],round(v['frac_measured_peak'],3)) for k,v in r['per_pass_program'].items()}, d['clocks'])"
