# ncu --set full of our pair GEMM and cuBLAS's nvjet kernel on one C2 shape.
mkdir -p gpurun_out
SH=${1:-q0:3072:1024:0}
GB_SHAPES=$SH timeout -s KILL 600 ncu --set full --clock-control none --import-source on \
  -k regex:"nvjet|pair_kernel" -c 2 -o gpurun_out/prof_cmp_${SH%%:*} python tools/gemm_bench.py > gpurun_out/ncu_cmp.log 2>&1
tail -3 gpurun_out/ncu_cmp.log
