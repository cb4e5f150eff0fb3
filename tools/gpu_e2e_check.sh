# GPU suite + the e2e (public API) legs of C1 / C2 / C3
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for wl in c1 c2 c3; do
  timeout -s KILL 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_$wl.json 2>/dev/null
  tail -1 gpurun_out/e2e_$wl.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl', round(d['value']), round(d['e2e']['value']), round(d['e2e']['value']/d['value'],3))"
done
