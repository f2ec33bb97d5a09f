timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_loopback.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for pw in 1 0; do QSIM_TURN_PW=$pw timeout 900 python bench.py --nlocal 33 --p 8 --steps 3 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r2_pw5.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_pw5.json')); r=d['roofline']
print('TURN_PW=$pw n=33', round(d['sec_per_layer']*1e3,2), {k:(round(v['avg_ms'],2),round(v['frac_measured_peak'],3)) for k,v in r['per_pass_program'].items()}, d['clocks']['sm_mhz'])"; done
