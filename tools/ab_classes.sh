#!/bin/bash
# Interleaved A/B of build variants: bench value + per-class ms (graph replay).
for i in $(seq ${ROUNDS:-3}); do
  for v in paper_2602_07309_b200/lib/*.so; do
    SEMRANK_LIB=$v timeout -s KILL 150 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['roofline']['per_class_ms']; print('$(basename $v)', round(d['value']), d['clocks']['sm_mhz'], ' '.join(f'{k}={v}' for k,v in c.items() if k.startswith('gemm') or k in ('attention','layernorm')))"
  done
done
