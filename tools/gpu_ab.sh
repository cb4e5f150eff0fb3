#!/bin/bash
# A/B: kernel tests, parity suite, bench with the default engine and with an env override.
# usage: AB_ENV="SRK_FOLD_LN=0" bash tools/gpu_ab.sh
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -4
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
summ() {
python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 1),
      "gemm_frac", round(r["frac"], 3), "clocks", d["clocks"])
print({k: round(v, 3) for k, v in r["per_class_ms"].items()})
PY
}
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab_a.json 2>gpurun_out/ab_a.err; summ gpurun_out/ab_a.json
timeout -s KILL 300 env ${AB_ENV:-SRK_FOLD_LN=0} python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab_b.json 2>gpurun_out/ab_b.err; summ gpurun_out/ab_b.json
