mkdir -p gpurun_out
for v in paper_2602_07309_b200/lib/libsemrank_b200_v1stg2.so paper_2602_07309_b200/lib/libsemrank_b200_v2stg3.so; do
  echo "== $v"; SEMRANK_LIB=$v timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
done
ROUNDS=3 bash tools/ab_libs.sh
