#!/bin/bash
# Interleaved A/B of environment variants (AB_VARIANTS="A=1 A=0 ...", "-" = none)
# on the default build: bench value, ms per step and per-class device times.
for i in $(seq ${ROUNDS:-2}); do
  for v in ${AB_VARIANTS}; do
    e=""; [ "$v" != "-" ] && e="$v"
    val=$(env $e timeout -s KILL 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c5 --no-serving ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],3), 'attn', r['per_class_ms']['attention'])")
    echo "$v $val"
  done
done
