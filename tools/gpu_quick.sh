#!/bin/bash
# quick GPU loop: kernel tests, parity suite, one bench line summary
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider 2>&1 | grep -E "max dev|passed|failed|Error|assert" | head
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} 2>&1 | tail -1 > gpurun_out/quick_bench.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/quick_bench.json"))
r = d["roofline"]
print("value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 1),
      "gemm_frac", round(r["frac"], 3), "clocks", d["clocks"])
print(r["per_class_ms"])
PY
