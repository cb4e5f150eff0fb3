#!/bin/bash
# Round evidence: smoke, gpu tests, all-config bench lines, reference arm,
# ncu launch list, ncu --set full captures of the GEMM and attention kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout -s KILL 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 200 gpurun_out/bench_c2.json
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 200 gpurun_out/bench_ref.json
for w in c1 c3 c4 c3_wire retrieval retrieval_xl; do
  timeout -s KILL 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 150 gpurun_out/bench_$w.json; echo
done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
wc -l gpurun_out/launches.csv
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 4 -c 4 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; tail -1 gpurun_out/ncu_gemm.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1; tail -1 gpurun_out/ncu_attn.log
ls gpurun_out
