#!/bin/bash
# LN-after epilogue check: gpu tests, then interleaved bench A/B (SRK_LN_AFTER=0/1).
timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_dist.py::test_two_rank_sharded_c5_merge_equals_single_gpu_and_oracle --deselect tests/test_gpu_headline.py::test_c5_8192_candidates_every_item 2>&1 | tail -6
for i in 1 2; do
  for v in 0 1; do
    val=$(SRK_LN_AFTER=$v timeout -s KILL 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c5 --no-serving ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],3), r['per_class_ms'])")
    echo "LN_AFTER=$v $val"
  done
done
