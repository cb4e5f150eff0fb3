#!/bin/bash
# Interleaved A/B of attention variants: bench value + attention class ms per
# lib/*.so build, plus the single-tile kernel (SRK_ATTN=tc) on the default build.
for i in $(seq ${ROUNDS:-2}); do
  for v in paper_2602_07309_b200/lib/*.so tc; do
    if [ "$v" = tc ]; then envs="SRK_ATTN=tc"; lib=paper_2602_07309_b200/lib/libsemrank_b200.so; else envs=""; lib=$v; fi
    val=$(env $envs SEMRANK_LIB=$lib timeout -s KILL 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c5 --no-serving ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), 'attn_ms', d['roofline']['per_class_ms']['attention'], 'frac', round(d['roofline']['attention']['frac'],3))")
    echo "$(basename $v) $val"
  done
done
