# ncu --set full of the two-tile attention kernel (one C2 launch)
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 -o gpurun_out/prof_fa python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c5 --no-serving > gpurun_out/ncu_fa.log 2>&1; tail -3 gpurun_out/ncu_fa.log
