#!/bin/bash
# ncu --set full of the retrieval scan kernel on the 33.5M-doc corpus + launch list
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none -k regex:retrieval_scan -s 3 -c 1 -o gpurun_out/prof_retrieval python bench.py --workload retrieval_xl --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_retrieval.log 2>&1; tail -2 gpurun_out/ncu_retrieval.log
