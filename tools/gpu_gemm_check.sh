# GEMM correctness + timeline after a GEMM kernel change (each step bounded).
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm 2>&1 | tail -5
echo "== NP=2 (default)"; timeout -s KILL 120 python tools/gemm_trace.py 2>&1 | grep -v "cta "
echo "== NP=1"; SRK_GEMM_NP=1 timeout -s KILL 120 python tools/gemm_trace.py 2>&1 | grep -v "cta "
