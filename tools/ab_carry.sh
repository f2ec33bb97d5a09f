mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4/pytest.log 2>&1; echo pytest=$? >> gpurun_out/s4/pytest.log
for c in 0 1 0 1; do
QSIM_CARRY=$c python bench.py --no-cpu-baseline > gpurun_out/s4/bench_$c.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/s4/bench_$c.log').read().strip().splitlines()[-1]); print('carry', $c, d['sec_per_layer'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['roofline']['avg_launch_ms'])" >> gpurun_out/s4/summary.txt
done
