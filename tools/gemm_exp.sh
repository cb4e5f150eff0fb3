# GEMM tuning sweep: build variants with `make OUT=../lib/var_X.so BUILD=... EXTRA=-D...`
S="o2:1024:1024:2,o0:1024:1024:0,wi1:1536:1024:1,wi0:1536:1024:0,wo2:1024:1536:2,q0:3072:1024:0"
for v in paper_2602_07309_b200/lib/var_*.so; do
  echo "== $v"
  SEMRANK_LIB=$v GB_SHAPES=$S python tools/gemm_bench.py
  echo "-- flushed"
  GB_FLUSH=1 SEMRANK_LIB=$v GB_SHAPES=$S python tools/gemm_bench.py
done
