"""Deterministic inputs of the headline parity fixtures (tests/golden/
headline_*.npz, made by oracle/gen_golden_headline.py). The generators are
bench.py's request streams (numpy PCG64 seeds), so the GPU box rebuilds the
exact inputs; each fixture stores a sha256 of them and the tests check it."""
import hashlib

import numpy as np


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def tokens_request(seed, t_q, t_i, n):
    """bench.make_request (token workloads): prefix then [n x t_i] ids."""
    rng = np.random.default_rng(seed)
    prefix = rng.integers(0, 256, t_q).astype(np.int32)
    toks = rng.integers(0, 256, (n, t_i)).astype(np.int32)
    return prefix, toks


def soft_request(seed, t_q, n_soft, n, d):
    """bench.make_request (c3): prefix then N(0, 0.08^2) rows [n x n_soft x d]."""
    rng = np.random.default_rng(seed)
    prefix = rng.integers(0, 256, t_q).astype(np.int32)
    rows = rng.standard_normal((n, n_soft, d)).astype(np.float32) * np.float32(0.08)
    return prefix, rows


def emb_request(seed, t_q, n, d_emb):
    """Compact per-item embeddings (unit-variance components)."""
    rng = np.random.default_rng(seed)
    prefix = rng.integers(0, 256, t_q).astype(np.int32)
    emb = rng.standard_normal((n, d_emb)).astype(np.float32)
    return prefix, emb


def projection_matrix(seed, d_emb, n_soft, d):
    """Fixed projection [d_emb x n_soft*d] (reference weight layout [in x out]),
    std 0.08/sqrt(d_emb) so projected rows have the embedding scale."""
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((d_emb, n_soft * d)) * (0.08 / np.sqrt(d_emb))).astype(np.float32)


def bf16(a):
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def project_rows(emb, proj, n_soft, d):
    """The projection pre-step both sides share: bf16(e) . bf16(P), exact
    products summed in double, rounded once to fp32 (the device accumulates
    the same bf16 products in fp32)."""
    r = bf16(emb).astype(np.float64) @ bf16(proj).astype(np.float64)
    return r.astype(np.float32).reshape(len(emb), n_soft, d)


def pad_rows(emb, d):
    """service.cpp:208-217: one row, embedding copied in, zero-padded to d."""
    out = np.zeros((len(emb), 1, d), np.float32)
    n = min(emb.shape[1], d)
    out[:, 0, :n] = emb[:, :n]
    return out


def batch_requests():
    """Two ragged queries packed into one pass."""
    rng = np.random.default_rng(23)
    out = []
    for t_q, n in ((256, 64), (181, 48)):
        prefix = rng.integers(0, 256, t_q).astype(np.int32)
        lens = rng.integers(1, 97, n)
        items = [rng.integers(0, 256, int(L)).astype(np.int32) for L in lens]
        out.append((prefix, items))
    return out


def ragged_long_request():
    """One query whose items straddle the 128-row attention tiles: lengths 1, 2,
    127-129, 255-256, 300-400 and random ones, prefix not a multiple of 128."""
    rng = np.random.default_rng(31)
    prefix = rng.integers(0, 256, 100).astype(np.int32)
    lens = [1, 2, 127, 128, 129, 255, 256, 300, 400, 1, 64, 96, 97, 33]
    lens += [int(L) for L in rng.integers(1, 401, 18)]
    items = [rng.integers(0, 256, L).astype(np.int32) for L in lens]
    return prefix, items


def ragged_soft_request():
    """Mixed-mode query with 1 ... 20 soft rows per item (N(0, 0.08^2))."""
    rng = np.random.default_rng(37)
    prefix = rng.integers(0, 256, 64).astype(np.int32)
    counts = [1, 20, 2, 19, 8] + [int(c) for c in rng.integers(1, 21, 35)]
    rows = [rng.standard_normal((c, 1024)).astype(np.float32) * np.float32(0.08) for c in counts]
    return prefix, rows


C5_SUBSET_SEED = 5
