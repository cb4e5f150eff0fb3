#!/bin/bash
# Interleaved A/B of build variants on one box: bench value per run for each
# paper_2602_07309_b200/lib/*.so (default build included), ROUNDS rounds.
for i in $(seq ${ROUNDS:-3}); do
  for v in paper_2602_07309_b200/lib/*.so; do
    val=$(SEMRANK_LIB=$v timeout -s KILL 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3))")
    echo "$(basename $v) $val"
  done
done
