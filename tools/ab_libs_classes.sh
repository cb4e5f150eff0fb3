#!/bin/bash
# Interleaved A/B of lib/*.so build variants with per-class device times.
for i in $(seq ${ROUNDS:-2}); do
  for v in paper_2602_07309_b200/lib/*.so; do
    val=$(env ${AB_ENV} SEMRANK_LIB=$v timeout -s KILL 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c5 --no-serving ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],3), r['per_class_ms'])")
    echo "$(basename $v) $val"
  done
done
