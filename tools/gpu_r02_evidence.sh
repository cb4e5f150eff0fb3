#!/bin/bash
# Round-2 evidence on one box: headline parity report, every bench workload,
# the ncu launch list of the C2 step and ncu --set full of its top kernels
# (GEMMs, attention) and row kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
SR_PARITY_REPORT=gpurun_out/r02_parity.json timeout -s KILL 900 python -m pytest tests/test_gpu_headline.py -q -p no:cacheprovider 2>&1 | tail -2
for w in c1 c3 c3_rows c4 c5 c3_wire retrieval retrieval_xl; do
  timeout -s KILL 900 python bench.py --workload $w --no-serving > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 120 gpurun_out/bench_$w.json; echo
done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 --no-serving > /dev/null 2>&1
wc -l gpurun_out/launches.csv
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 4 -c 4 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c5 --no-serving > gpurun_out/ncu_gemm.log 2>&1; tail -1 gpurun_out/ncu_gemm.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c5 --no-serving > gpurun_out/ncu_attn.log 2>&1; tail -1 gpurun_out/ncu_attn.log
bash tools/gpu_rowops_profiles.sh
