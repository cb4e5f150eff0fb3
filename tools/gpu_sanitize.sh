# compute-sanitizer memcheck / synccheck over small requests through every
# production kernel class (tools/sanitize_small.py), and memcheck over the
# wire / post-processing GPU tests
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 200 \
    python tools/sanitize_small.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -h "^ok\|ERROR SUMMARY" gpurun_out/san_$tool.log
  grep -h -A1 "error detected\|Invalid\|Race" gpurun_out/san_$tool.log | grep " at " | sort | uniq -c
done
timeout -s KILL 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 50 \
  python -m pytest tests/test_gpu_wire.py tests/test_gpu_postprocess.py -x -q -p no:cacheprovider \
  > gpurun_out/san_memcheck_tests.log 2>&1
echo "tests memcheck rc=$?"; grep -h "passed\|failed\|ERROR SUMMARY" gpurun_out/san_memcheck_tests.log | tail -3
