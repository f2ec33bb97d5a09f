timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "qaoa_batch" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_batch_bench.json 2>gpurun_out/r2_batch_bench.err; python -c "
import json; d=json.load(open('gpurun_out/r2_batch_bench.json')); print(d['sec_per_layer'], d['extra_configs']['n12_2sat'])"
