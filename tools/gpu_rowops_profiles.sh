#!/bin/bash
# ncu --set full captures of the HBM-bound row kernels of the C2 step
# (LayerNorm, embed+LN1, fused final-LN score head, top-k), one launch each,
# plus a per-kernel SASS instruction census of the built library.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c5 --no-serving"
for k in layer_norm_kernel embed_ln_kernel score_head_kernel topk_scores_kernel; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
  tail -1 gpurun_out/ncu_$k.log
done
ls gpurun_out
