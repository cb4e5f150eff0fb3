mkdir -p gpurun_out
python bench.py --workload c3 --steps 20 --warmup 5 > gpurun_out/c3.json 2>gpurun_out/c3.err
tail -1 gpurun_out/c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks'])"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 2 -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c5 --no-serving > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
