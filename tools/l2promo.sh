# L2 promotion of the run sets' tensor maps (default 256 B) vs 128 B: bench step A/B, twice
for v in 256 128 256 128; do
  QSIM_L2PROMO=$v timeout 200 python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/l2p_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/l2p_$v.json').read().strip().splitlines()[-1])
pp=d['roofline']['per_pass_program']
print('l2promo $v', round(d['ms_per_step'],2), {k:round(x['avg_ms'],3) for k,x in pp.items()}, d['clocks']['sm_mhz'], d['results']['expect_hc'])
"
done
