QSIM_PW_STG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled_parity or all_set_layouts or full_size_p1 or full_size_product" 2>&1 | tail -2
for m in 0 1; do echo "QSIM_PW_STG=$m"; QSIM_PW_STG=$m timeout 300 python tools/passbench.py --n 30 --reps 5 2>&1 | grep -E "set=(1|2) phase=1 "; done
for m in 0 1; do QSIM_PW_STG=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r2_stg.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_stg.json')); r=d['roofline']
print('STG=$m', d['sec_per_layer'], r['frac'], {k:(round(v['avg_ms'],3),round(v['frac_measured_peak'],3)) for k,v in r['per_pass_program'].items()}, d['clocks']['sm_mhz'])"; done
