"""Kernel-level numerics on the B200, through the C-ABI kernel entry points.

Floating-point kernels are compared against plain PyTorch fp32 references of
the same op on the same (bf16-exact) inputs; tolerances are written per test.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2602_07309_b200._capi import lib
    return lib


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _ok(st):
    from paper_2602_07309_b200._capi import lib
    assert st == 0, lib.sr_last_error().decode()


# N % 256 == 0 takes the CTA-pair path (SRK_GEMM_NP=2: 4-CTA clusters with A
# multicast when N % 512 == 0), other N the 1-CTA kernel.
GEMM_SHAPES = [(128, 256, 64), (300, 3072, 1024), (1000, 1536, 1024), (257, 1024, 1536),
               (77, 192, 64), (500, 64, 256), (4096, 1024, 1024), (129, 128, 2048),
               (6000, 3072, 1024), (2000, 512, 64), (700, 768, 512),
               # 80 pair tiles on 74 pairs: the 6 tail tiles run as 256 x 128 halves
               (5120, 1024, 1024), (5000, 1024, 1536)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_fp32_epilogue_matches_torch(cuda, M, N, K):
    import torch
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, generator=g).bfloat16().to(cuda)
    b = torch.randn(N, K, generator=g).bfloat16().to(cuda)
    c = torch.full((M, N), float("nan"), device=cuda)
    _ok(_lib().sr_kernel_gemm(_vp(a), _vp(b), M, N, K, _vp(c), N, 3, None))
    ref = a.float() @ b.float().T
    # bf16 inputs are exact in fp32; only the accumulation order differs.
    err = (c - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K", [(300, 3072, 1024), (77, 192, 64), (1000, 1536, 1024),
                                   (5120, 1024, 1024)])
def test_gemm_bf16_and_gelu_epilogues(cuda, M, N, K):
    import torch
    g = torch.Generator(device="cpu").manual_seed(5)
    a = (torch.randn(M, K, generator=g) / K ** 0.5).bfloat16().to(cuda)
    b = torch.randn(N, K, generator=g).bfloat16().to(cuda)
    ref = a.float() @ b.float().T
    c = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    _ok(_lib().sr_kernel_gemm(_vp(a), _vp(b), M, N, K, _vp(c), N, 0, None))
    # one bf16 rounding of the fp32 result: rel 2^-8
    assert torch.allclose(c.float(), ref, rtol=8e-3, atol=1e-3)
    _ok(_lib().sr_kernel_gemm(_vp(a), _vp(b), M, N, K, _vp(c), N, 1, None))
    gref = torch.nn.functional.gelu(ref)  # exact erf GELU
    assert torch.allclose(c.float(), gref, rtol=8e-3, atol=1e-3)


@pytest.mark.parametrize("M,N,K", [(300, 1024, 1024), (257, 1024, 1536), (64, 64, 256),
                                   (5000, 1024, 1536), (24832, 1024, 1024)])
def test_gemm_residual_epilogue(cuda, M, N, K):
    import torch
    g = torch.Generator(device="cpu").manual_seed(9)
    a = torch.randn(M, K, generator=g).bfloat16().to(cuda)
    b = torch.randn(N, K, generator=g).bfloat16().to(cuda)
    x0 = torch.randn(M, N, generator=g).to(cuda)
    x = x0.clone()
    _ok(_lib().sr_kernel_gemm(_vp(a), _vp(b), M, N, K, _vp(x), N, 2, None))
    ref = x0 + a.float() @ b.float().T
    err = (x - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K", [(300, 1024, 1024), (5000, 1024, 1536), (257, 2048, 1024),
                                   (100, 256, 512)])
def test_gemm_residual_ln_statistics_epilogue(cuda, M, N, K):
    """epi 4: x += A.B^T (fp32), xb = bf16(x) exactly, per-128-column (mean, M2)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    a = (torch.randn(M, K, generator=g) / K ** 0.5).bfloat16().to(cuda)
    b = torch.randn(N, K, generator=g).bfloat16().to(cuda)
    x0 = (torch.randn(M, N, generator=g) + torch.randn(M, 1, generator=g)).to(cuda)
    x = x0.clone()
    xb = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    ld = M + 7
    stats = torch.full((N // 128, ld, 2), float("nan"), device=cuda)
    _ok(_lib().sr_kernel_gemm_ln(_vp(a), _vp(b), M, N, K, _vp(x), N, 4, _vp(xb), _vp(stats), 0,
                                 None, ld, None))
    ref = x0 + a.float() @ b.float().T
    assert (x - ref).abs().max().item() <= 1e-3 * max(1.0, ref.abs().max().item())
    assert torch.equal(xb, x.bfloat16())
    parts = x.view(M, N // 128, 128)
    mean = parts.double().mean(-1)
    m2 = ((parts.double() - mean[..., None]) ** 2).sum(-1)
    got = stats[:, :M].permute(1, 0, 2).double()
    assert torch.allclose(got[..., 0], mean, rtol=1e-5, atol=1e-5)
    assert torch.allclose(got[..., 1], m2, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("M,N,K,P", [(300, 3072, 1024, 8), (1000, 1536, 1024, 1),
                                     (777, 6144, 2048, 16), (64, 256, 256, 2)])
def test_gemm_folded_layernorm_epilogues(cuda, M, N, K, P):
    """epi 5/6: bf16([gelu](LN(x)*gain . W)) from xb, partial stats and diag(gain) W."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(M * 3 + N + K)
    x = (torch.randn(M, K, generator=g) * 0.5 + 0.2 * torch.randn(M, 1, generator=g)).to(cuda)
    gain = (1 + 0.1 * torch.randn(K, generator=g)).to(cuda)
    w = (torch.randn(K, N, generator=g) / K ** 0.5).to(cuda)  # reference layout [d_in x d_out]
    bt = (gain[:, None] * w).T.contiguous().bfloat16()        # folded, K-major [N x K]
    colsum = bt.float().sum(1).contiguous()
    xb = x.bfloat16()
    ld = M + 3
    parts = x.view(M, P, K // P).double()
    pm = parts.mean(-1)
    stats = torch.zeros(P, ld, 2, device=cuda)
    stats[:, :M, 0] = pm.T.float()
    stats[:, :M, 1] = ((parts - pm[..., None]) ** 2).sum(-1).T.float()
    mean = x.double().mean(-1, keepdim=True)
    rstd = 1 / torch.sqrt(((x.double() - mean) ** 2).mean(-1, keepdim=True) + 1e-5)
    # Same algebra in fp64 on the same bf16 operands: only accumulation order differs.
    algebra = (rstd * (xb.double() @ bt.double().T - mean * colsum.double()[None])).float()
    ln_ref = (((x - mean.float()) * rstd.float() * gain) @ w)  # the reference's LN . W in fp32
    for epi, fn in ((5, lambda z: z), (6, torch.nn.functional.gelu)):
        c = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
        _ok(_lib().sr_kernel_gemm_ln(_vp(xb), _vp(bt), M, N, K, _vp(c), N, epi, None, _vp(stats),
                                     P, _vp(colsum), ld, None))
        assert torch.allclose(c.float(), fn(algebra), rtol=8e-3, atol=2e-3)
        # vs the unfused reference: bf16 operand rounding (x and gain*W) on top
        assert (c.float() - fn(ln_ref)).abs().max().item() < 6e-2


def _attention_ref(qkv, spans, H, hd):
    """fp32 reference of kernels.cpp:51-95 with explicit allowed sets."""
    import torch
    M = qkv.shape[0]
    d = H * hd
    q = qkv[:, :d].float().view(M, H, hd)
    k = qkv[:, d:2 * d].float().view(M, H, hd)
    v = qkv[:, 2 * d:].float().view(M, H, hd)
    keys = torch.arange(M, device=qkv.device)
    sp = torch.as_tensor(spans, device=qkv.device)
    rows = torch.arange(M, device=qkv.device)[:, None]
    allowed = ((keys[None, :] >= sp[:, 0:1]) & (keys[None, :] < sp[:, 1:2])) | \
              ((keys[None, :] >= sp[:, 2:3]) & (keys[None, :] <= rows))
    s = torch.einsum("qhd,khd->hqk", q, k) / hd ** 0.5
    s = s.masked_fill(~allowed[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqk,khd->qhd", p, v).reshape(M, d)


def _multi_item_spans(prefix, lens, base=0):
    spans = [[base, base, base, 0] for _ in range(prefix)]
    spans = [[base, base, base, 0] for _ in range(prefix)]
    cur = base + prefix
    for L in lens:
        for _ in range(L):
            spans.append([base, base + prefix, cur, 0])
        cur += L
    return spans


@pytest.mark.parametrize("H,hd,prefix,lens", [
    (2, 16, 4, [5, 3]),                       # test_kernels.cpp:83-137 layout (scaled up heads)
    (4, 16, 500, [50] * 12),                  # toy C1 shape
    (8, 128, 256, [96] * 6 + [7, 1, 130]),    # C2 shape, ragged tail
    (8, 128, 256, [8] * 40),                  # C3 soft-token items
    (4, 64, 33, [1, 2, 65, 64, 3]),
    (2, 32, 0, [17, 80]),                     # empty prefix
])
def test_attention_segment_mask_matches_torch(cuda, H, hd, prefix, lens):
    import torch
    spans = _multi_item_spans(prefix, lens)
    M = len(spans)
    d = H * hd
    g = torch.Generator(device="cpu").manual_seed(M + H)
    qkv = torch.randn(M, 3 * d, generator=g).bfloat16().to(cuda)
    out = torch.zeros(M, d, dtype=torch.bfloat16, device=cuda)
    sp = np.asarray(spans, np.int32).reshape(-1)
    _ok(_lib().sr_kernel_attention(_vp(qkv), sp.ctypes.data_as(C.POINTER(C.c_int32)), M, H, hd,
                                   _vp(out), None))
    ref = _attention_ref(qkv, spans, H, hd)
    # P is rounded to bf16 before the PV product and O is stored as bf16.
    err = (out.float() - ref).abs().max().item()
    assert err < 3e-2, err


def test_attention_reference_kernel_test_layout(cuda):
    """The exact span set of test_kernels.cpp:91-95 (prefix [0,4), items [4,9), [9,12))."""
    import torch
    H, hd = 2, 16
    spans = [[0, 0, 0, 0]] * 4 + [[0, 4, 4, 0]] * 5 + [[0, 4, 9, 0]] * 3
    M, d = 12, H * hd
    g = torch.Generator(device="cpu").manual_seed(17)
    qkv = torch.randn(M, 3 * d, generator=g).bfloat16().to(cuda)
    out = torch.zeros(M, d, dtype=torch.bfloat16, device=cuda)
    sp = np.asarray(spans, np.int32).reshape(-1)
    _ok(_lib().sr_kernel_attention(_vp(qkv), sp.ctypes.data_as(C.POINTER(C.c_int32)), M, H, hd,
                                   _vp(out), None))
    ref = _attention_ref(qkv, spans, H, hd)
    assert (out.float() - ref).abs().max().item() < 2e-2
    # single slot attending itself returns V exactly (test_kernels.cpp:69-81)
    assert torch.equal(out[0], qkv[0, 2 * d:])


@pytest.mark.parametrize("M,d", [(1, 64), (333, 1024), (50, 2048), (1000, 64)])
def test_layernorm_matches_torch(cuda, M, d):
    import torch
    g = torch.Generator(device="cpu").manual_seed(M)
    x = (torch.randn(M, d, generator=g) * 3 + 0.5).to(cuda)
    gain = torch.rand(d, generator=g).to(cuda) + 0.5
    out = torch.zeros(M, d, dtype=torch.bfloat16, device=cuda)
    _ok(_lib().sr_kernel_layernorm(_vp(x), _vp(gain), _vp(out), M, d, None))
    mean = x.mean(-1, keepdim=True)
    var = ((x - mean) ** 2).mean(-1, keepdim=True)
    ref = (x - mean) / torch.sqrt(var + 1e-5) * gain
    assert torch.allclose(out.float(), ref, rtol=8e-3, atol=8e-3)


@pytest.mark.parametrize("n,k,ties", [(256, 10, False), (8192, 100, False), (5000, 64, True),
                                      (3, 10, False), (20000, 10, True)])
def test_topk_matches_stable_sort(cuda, n, k, ties):
    import torch
    rng = np.random.default_rng(n)
    scores = rng.random(n)
    if ties:
        scores = np.round(scores * 20) / 20  # many exact ties -> id rule decides
    ids = rng.permutation(n * 3)[:n].astype(np.int64)
    ds = torch.as_tensor(scores, device=cuda)
    di = torch.as_tensor(ids, device=cuda)
    kk = min(k, n)
    oi = np.zeros(kk, np.int64)
    osc = np.zeros(kk)
    ox = np.zeros(kk, np.int32)
    _ok(_lib().sr_kernel_topk(_vp(ds), _vp(di), n, k, oi.ctypes.data_as(C.POINTER(C.c_int64)),
                              osc.ctypes.data_as(C.POINTER(C.c_double)),
                              ox.ctypes.data_as(C.POINTER(C.c_int32))))
    order = sorted(range(n), key=lambda i: (-scores[i], ids[i]))[:kk]
    assert list(oi) == [int(ids[i]) for i in order]
    assert list(ox) == order


def test_gemm_single_pair_path_matches_cluster_path(cuda):
    """SRK_GEMM_NP=2 (4-CTA clusters, A multicast to two pairs) gives the same
    bits as the default single-pair path: the K order per tile is identical."""
    import subprocess
    import sys
    code = (
        "import torch, ctypes as C\n"
        "from paper_2602_07309_b200._capi import lib\n"
        "g = torch.Generator().manual_seed(3)\n"
        "a = torch.randn(3000, 1024, generator=g).bfloat16().cuda()\n"
        "b = torch.randn(1536, 1024, generator=g).bfloat16().cuda()\n"
        "c = torch.zeros(3000, 1536, device='cuda')\n"
        "assert lib.sr_kernel_gemm(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), 3000, 1536,"
        " 1024, C.c_void_p(c.data_ptr()), 1536, 3, None) == 0\n"
        "import hashlib, sys; sys.stdout.write(hashlib.sha1(c.cpu().numpy().tobytes()).hexdigest())\n")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for np_ in ("1", "2"):
        env = dict(os.environ, SRK_GEMM_NP=np_, PYTHONPATH=root)
        out[np_] = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                  text=True, timeout=300, check=True).stdout
    assert out["1"] == out["2"] and len(out["1"]) == 40


def test_pingpong_attention_variant_matches_torch(cuda):
    """The opt-in two-slot attention kernel (SRK_ATTN=pp, read once per
    process) against the same fp32 references, in a child process."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, SRK_ATTN="pp")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.abspath(__file__), "-k", "attention_segment_mask"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_two_tile_attention_variant_matches_torch(cuda):
    """The opt-in two-tile ping-pong attention kernel (SRK_ATTN=fa,
    kernels/attention_fa.cu, head 128) against the same fp32 references, in a
    child process."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, SRK_ATTN="fa")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.abspath(__file__), "-k", "attention_segment_mask"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("M,N,K", [(300, 1024, 1024), (4096, 1024, 1536), (257, 2048, 512)])
def test_residual_gemm_with_overlapped_layernorm(cuda, M, N, K):
    """Opt-in LN-after path (SRK_LN_AFTER=1): epilogue 7 adds into x and counts
    finished 128-row blocks, a concurrent kernel normalises each block
    (kernels.cpp:31-45). x must equal the plain residual epilogue bit for bit,
    the LN output a torch fp32 LayerNorm of that x within bf16 rounding, and
    the counters must be back to zero."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    a = (torch.randn(M, K, generator=g) / K ** 0.5).bfloat16().to(cuda)
    b = torch.randn(N, K, generator=g).bfloat16().to(cuda)
    x0 = torch.randn(M, N, generator=g).to(cuda)
    gain = (torch.rand(N, generator=g) + 0.5).to(cuda)
    x_ref = x0.clone()
    _ok(_lib().sr_kernel_gemm(_vp(a), _vp(b), M, N, K, _vp(x_ref), N, 2, None))
    x = x0.clone()
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    cnt = torch.zeros((M + 127) // 128 + 1, dtype=torch.int32, device=cuda)
    for _ in range(2):  # counters are reusable
        x.copy_(x0)
        _ok(_lib().sr_kernel_gemm_resid_ln(_vp(a), _vp(b), M, N, K, _vp(x), _vp(gain), _vp(out),
                                           _vp(cnt), None))
        assert torch.equal(x, x_ref)
        ref = torch.nn.functional.layer_norm(x_ref, (N,), eps=1e-5) * gain
        assert (out.float() - ref).abs().max().item() <= 2e-2 * max(1.0, ref.abs().max().item())
        assert int(cnt.abs().sum().item()) == 0


def test_engine_ln_after_variant_matches_oracle(cuda):
    """The engine with SRK_LN_AFTER=1 (read once per process) through the
    headline parity suite, in a child process."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, SRK_LN_AFTER="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_headline.py"), "-k", "c2 or batch or c4"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_block_parity_attention_variant_matches_torch(cuda):
    """The opt-in attention kernel whose softmax warps own alternate key
    blocks (SRK_ATTN=eo, kernels/attention_eo.cu, head 128) against the same
    fp32 references, in a child process."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, SRK_ATTN="eo")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.abspath(__file__), "-k", "attention_segment_mask"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
