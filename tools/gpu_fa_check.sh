set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k attention 2>&1 | tail -15
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_dist.py::test_two_rank_sharded_c5_merge_equals_single_gpu_and_oracle 2>&1 | tail -15
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c5 --no-serving 2>&1 | tail -1 > gpurun_out/fa_bench.json
python -c "
import json; d=json.load(open('gpurun_out/fa_bench.json')); r=d['roofline']
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'attn', r['attention'], r['per_class_ms'], d['clocks'])"
