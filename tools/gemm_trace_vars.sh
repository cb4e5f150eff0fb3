#!/bin/bash
# GEMM timeline per build variant (paper_2602_07309_b200/lib/*.so): per-tile MMA interval + epilogue time.
export GT_BRIEF=1
S=${GT_SHAPES:-q0:3072:1024:0,o2:1024:1024:2,o4:1024:1024:4,wi1:1536:1024:1,q5:3072:1024:5,wi6:1536:1024:6,wo2:1024:1536:2,wo4:1024:1536:4}
for v in paper_2602_07309_b200/lib/*.so; do echo "=== $v"; SEMRANK_LIB=$v GT_SHAPES=$S python tools/gemm_trace.py 2>&1 | grep -v "entry spread\|exit:"; done
