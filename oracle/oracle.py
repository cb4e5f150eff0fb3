"""ctypes bindings of the CPU oracles. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module; the product never does.

  Port  : build/liboracle.so   — C restatement (semrank_oracle.c), always buildable
  Ref   : _ref/libsemrank_ref.so — the reference's own sources compiled in place
          (present only where /root/reference existed at build time)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsemrank_ref.so")

i32p = C.POINTER(C.c_int32)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)


class OrConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int),
                ("d_ff", C.c_int), ("vocab_size", C.c_int), ("max_seq", C.c_int),
                ("yes_token_id", C.c_int), ("no_token_id", C.c_int), ("n_task_heads", C.c_int),
                ("head_arity", C.c_int * 16), ("head_names", (C.c_char * 32) * 16)]


_port = None
_ref = None


def build_port() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "build/liboracle.so"], check=True)


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            build_port()
        lib = C.CDLL(PORT_PATH)
        lib.or_init.restype = C.c_void_p
        lib.or_init.argtypes = [C.POINTER(OrConfig), C.c_uint64, C.c_int]
        lib.or_load.restype = C.c_void_p
        lib.or_load.argtypes = [C.c_char_p]
        lib.or_save.argtypes = [C.c_void_p, C.c_char_p]
        lib.or_free.argtypes = [C.c_void_p]
        lib.or_round_bf16.argtypes = [C.c_void_p]
        lib.or_tensor_count.argtypes = [C.c_void_p]
        lib.or_tensor.restype = f32p
        lib.or_tensor.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_size_t),
                                  C.POINTER(C.c_char_p)]
        lib.or_version.restype = C.c_char_p
        lib.or_version.argtypes = [C.c_void_p]
        lib.or_score.argtypes = [C.c_void_p, i32p, C.c_int, i32p, i32p, f32p, C.c_int, f64p, f32p,
                                 C.c_int]
        lib.or_prefill.argtypes = [C.c_void_p, i32p, C.c_int, f32p]
        lib.or_attention.argtypes = [f32p, f32p, f32p, f32p, C.c_int, C.c_int, C.c_int, i32p]
        lib.or_bench_tokens.argtypes = [C.c_uint64, C.c_char_p, C.c_int, C.c_int, C.c_int, i32p]
        lib.or_uniform_ints.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int, i64p]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_PATH)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_set_parallel.argtypes = [C.c_int]
        for fn in (lib.ref_init_save, lib.ref_init_fanin_save):
            fn.argtypes = [i32p, C.c_int32, C.POINTER(C.c_char_p), i32p, C.c_uint64, C.c_char_p]
        lib.ref_score.argtypes = [C.c_char_p, C.c_int32, i32p, C.c_int32, i32p, i32p, f32p,
                                  C.c_int32, f64p, f64p, f64p]
        lib.ref_prefill.argtypes = [C.c_char_p, i32p, C.c_int32, f32p]
        lib.ref_attention.argtypes = [f32p, f32p, f32p, f32p, C.c_int32, C.c_int32, C.c_int32,
                                      i32p]
        lib.ref_flops.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int64, f64p]
        lib.ref_plan_batches.argtypes = [C.c_int32, i32p, i32p, i32p, C.c_int64, i32p, C.c_int32,
                                         i32p, i64p]
        lib.ref_uniform_ints.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32, i64p]
        lib.ref_build_prompt.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int32, i32p, i32p,
                                         C.c_int32, i32p]
        lib.ref_score_result_json.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p),
                                              C.c_int32, C.POINTER(C.c_char_p), f64p, C.c_double,
                                              C.c_double, C.c_char_p, C.c_int64, i64p]
        _ref = lib
    return _ref


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def config_struct(cfg) -> OrConfig:
    """From a paper_2602_07309_b200.ModelConfig-like object (duck-typed)."""
    c = OrConfig()
    c.n_layers, c.d_model, c.n_heads, c.d_ff = cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.d_ff
    c.vocab_size, c.max_seq = cfg.vocab_size, cfg.max_seq
    c.yes_token_id, c.no_token_id = cfg.yes_token_id, cfg.no_token_id
    c.n_task_heads = len(cfg.head_specs)
    for i, h in enumerate(cfg.head_specs):
        c.head_arity[i] = h.arity
        c.head_names[i].value = h.name.encode()
    return c


class OracleWeights:
    """Weights held by the C restatement."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        if not self.h.value:
            raise RuntimeError("oracle: weight load/init failed")
        self.cfg = OrConfig()
        # config read back through the tensor table is enough for tests

    @staticmethod
    def init(cfg, seed: int, scheme: int = 0) -> "OracleWeights":
        c = config_struct(cfg)
        w = OracleWeights(port().or_init(C.byref(c), seed, scheme))
        w.cfg = c
        return w

    @staticmethod
    def load(path: str, cfg=None) -> "OracleWeights":
        w = OracleWeights(port().or_load(path.encode()))
        if cfg is not None:
            w.cfg = config_struct(cfg)
        return w

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            port().or_free(self.h)
            self.h = C.c_void_p()

    def save(self, path: str) -> None:
        if port().or_save(self.h, path.encode()) != 0:
            raise RuntimeError("oracle: save failed")

    def round_bf16(self) -> None:
        port().or_round_bf16(self.h)

    def tensors(self):
        lib = port()
        out = {}
        for i in range(lib.or_tensor_count(self.h)):
            n = C.c_size_t()
            name = C.c_char_p()
            ptr = lib.or_tensor(self.h, i, C.byref(n), C.byref(name))
            out[name.value.decode()] = np.ctypeslib.as_array(ptr, shape=(n.value,)).copy()
        return out

    @property
    def version(self) -> str:
        return port().or_version(self.h).decode()

    def score(self, prefix, items=None, rows=None, n_tasks=6, threads=0, hidden=False):
        """items: list of token lists, or rows: list of [n x d] arrays (mixed)."""
        prefix = np.ascontiguousarray(prefix, np.int32)
        seq = items if items is not None else rows
        lens = [len(x) if items is not None else np.asarray(x).shape[0] for x in seq]
        off = np.zeros(len(lens) + 1, np.int32)
        off[1:] = np.cumsum(lens)
        tok = np.ascontiguousarray(np.concatenate([np.asarray(x, np.int32) for x in items]), np.int32) \
            if items is not None else None
        rw = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float32).reshape(-1) for x in rows]),
                                  np.float32) if rows is not None else None
        scores = np.zeros((len(lens), n_tasks))
        d = int(self.cfg.d_model) if self.cfg.d_model else 0
        hid = np.zeros((len(lens), d), np.float32) if hidden else None
        st = port().or_score(self.h, _p(prefix, i32p), len(prefix), _p(off, i32p), _p(tok, i32p),
                             _p(rw, f32p), len(lens), _p(scores, f64p), _p(hid, f32p), threads)
        if st != 0:
            raise ValueError("oracle: request violates a reference precondition")
        return (scores, hid) if hidden else scores


def bench_tokens(seed: int, t_q: int, t_i: int, n_items: int, stream: str = "bench"):
    """cmd_bench token stream (semrank_main.cpp:602-616)."""
    out = np.zeros(t_q + t_i * n_items, np.int32)
    port().or_bench_tokens(seed, stream.encode(), t_q, t_i, n_items, _p(out, i32p))
    return out[:t_q], [out[t_q + i * t_i: t_q + (i + 1) * t_i] for i in range(n_items)]


def uniform_ints(seed: int, lo: int, hi: int, n: int):
    out = np.zeros(n, np.int64)
    port().or_uniform_ints(seed, lo, hi, n, _p(out, i64p))
    return out


def ref_score(weights_path: str, mode: int, prefix, items=None, rows=None, n_tasks=6):
    lib = ref()
    prefix = np.ascontiguousarray(prefix, np.int32)
    seq = items if items is not None else rows
    lens = [len(x) if items is not None else np.asarray(x).shape[0] for x in seq]
    off = np.zeros(len(lens) + 1, np.int32)
    off[1:] = np.cumsum(lens)
    tok = np.ascontiguousarray(np.concatenate([np.asarray(x, np.int32) for x in items]), np.int32) \
        if items is not None else None
    rw = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float32).reshape(-1) for x in rows]),
                              np.float32) if rows is not None else None
    scores = np.zeros((len(lens), n_tasks))
    fl = np.zeros(5)
    kv = np.zeros(1)
    st = lib.ref_score(weights_path.encode(), mode, _p(prefix, i32p), len(prefix), _p(off, i32p),
                       _p(tok, i32p), _p(rw, f32p), len(lens), _p(scores, f64p), _p(fl, f64p),
                       _p(kv, f64p))
    if st != 0:
        raise RuntimeError(f"reference error {st}: {lib.ref_last_error().decode()}")
    return scores, fl, float(kv[0])


def ref_init_save(cfg, seed: int, path: str, fan_in: bool = False) -> None:
    lib = ref()
    dims = np.array([cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.d_ff, cfg.vocab_size,
                     cfg.max_seq, cfg.yes_token_id, cfg.no_token_id], np.int32)
    names = (C.c_char_p * max(1, len(cfg.head_specs)))(*[h.name.encode() for h in cfg.head_specs])
    ar = np.array([h.arity for h in cfg.head_specs] or [1], np.int32)
    fn = lib.ref_init_fanin_save if fan_in else lib.ref_init_save
    st = fn(_p(dims, i32p), len(cfg.head_specs), names, _p(ar, i32p), seed, path.encode())
    if st != 0:
        raise RuntimeError(lib.ref_last_error().decode())


# ---------------------------------------------------------------- retrieval
class RetrievalError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # semrank ErrorCode value (3 SpecViolation, 6 Alignment, 9 Degenerate)


def oracle_topk(emb, feat, ids, keep, query, w0, w, k):
    """C restatement of exhaustive_topk (retrieval.cpp:134-173) -> (ids, scores)."""
    lib = port()
    emb = np.ascontiguousarray(emb, np.float32)
    n, d = emb.shape
    feat = np.ascontiguousarray(feat, np.float32).reshape(n, -1)
    ids = np.ascontiguousarray(ids, np.int64)
    q = np.ascontiguousarray(query, np.float32)
    wv = np.ascontiguousarray(w, np.float64)
    kp = None if keep is None else np.ascontiguousarray(keep, np.uint8)
    kk = max(int(k), 1)
    oi = np.zeros(kk, np.int64)
    os_ = np.zeros(kk, np.float64)
    fn = lib.or_exhaustive_topk
    fn.restype = C.c_int
    fn.argtypes = [f32p, f32p, i64p, C.POINTER(C.c_uint8), C.c_int64, C.c_int, C.c_int, f32p,
                   C.c_int, C.c_double, f64p, C.c_int, C.c_int, i64p, f64p]
    r = fn(_p(emb, f32p), _p(feat, f32p), _p(ids, i64p),
           kp.ctypes.data_as(C.POINTER(C.c_uint8)) if kp is not None else None, n, d,
           feat.shape[1], _p(q, f32p), q.shape[0], float(w0), _p(wv, f64p), wv.shape[0], int(k),
           _p(oi, i64p), _p(os_, f64p))
    if r < 0:
        raise RetrievalError(-r, "oracle error")
    return oi[:r], os_[:r]


def ref_topk(emb, feat, ids, color, query, w0, w, allowed, k, timing=None):
    """The reference's own exhaustive_topk through oracle/_ref (attribute
    "color" per doc from color codes; allowed=None -> no filter)."""
    lib = ref()
    emb = np.ascontiguousarray(emb, np.float32)
    n, d = emb.shape
    feat = np.ascontiguousarray(feat, np.float32).reshape(n, -1)
    ids = np.ascontiguousarray(ids, np.int64)
    col = None if color is None else np.ascontiguousarray(color, np.int32)
    q = np.ascontiguousarray(query, np.float32)
    wv = np.ascontiguousarray(w, np.float64)
    al = np.ascontiguousarray(allowed if allowed is not None else [0], np.int32)
    kk = max(int(k), 1)
    oi = np.zeros(kk, np.int64)
    os_ = np.zeros(kk, np.float64)
    cnt = np.zeros(1, np.int32)
    fn = lib.ref_exhaustive_topk
    fn.argtypes = [f32p, f32p, i64p, i32p, C.c_int64, C.c_int32, C.c_int32, f32p, C.c_int32,
                   C.c_double, f64p, C.c_int32, i32p, C.c_int32, C.c_int32, i64p, f64p, i32p,
                   f64p]
    st = fn(_p(emb, f32p), _p(feat, f32p), _p(ids, i64p), _p(col, i32p), n, d, feat.shape[1],
            _p(q, f32p), q.shape[0], float(w0), _p(wv, f64p), wv.shape[0], _p(al, i32p),
            -1 if allowed is None else len(allowed), int(k), _p(oi, i64p), _p(os_, f64p),
            _p(cnt, i32p), _p(timing, f64p))
    if st != 0:
        raise RetrievalError(st - 1, lib.ref_last_error().decode())
    return oi[:cnt[0]], os_[:cnt[0]]


# ------------------------------------------------------------- calibration
def oracle_final_scores(scores, lo, hi, val, blend_task=(), blend_w=()):
    """C restatement of calibrate + blend (calibration.cpp:65-88, service.cpp:250-266)."""
    lib = port()
    sc = np.ascontiguousarray(scores, np.float64)
    n, stride = sc.shape
    lo, hi, val = (np.ascontiguousarray(a, np.float64) for a in (lo, hi, val))
    bt = np.ascontiguousarray(list(blend_task) or [0], np.int32)
    bw = np.ascontiguousarray(list(blend_w) or [0.0], np.float64)
    out = np.zeros(n, np.float64)
    fn = lib.or_final_scores
    fn.argtypes = [f64p, C.c_int, C.c_int, f64p, f64p, f64p, C.c_int, i32p, f64p, C.c_int, f64p]
    fn(_p(sc, f64p), stride, n, _p(lo, f64p), _p(hi, f64p), _p(val, f64p), len(lo), _p(bt, i32p),
       _p(bw, f64p), len(list(blend_task)), _p(out, f64p))
    return out


def ref_fit_calibrate(raw, outcome, raws):
    """The reference's fit_isotonic + calibrate (oracle/_ref) -> (lo, hi, val, calibrated)."""
    lib = ref()
    raw = np.ascontiguousarray(raw, np.float64)
    oc = np.ascontiguousarray(outcome, np.int32)
    rs = np.ascontiguousarray(raws, np.float64)
    cap = len(raw) + 1
    lo, hi, val = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    nb = np.zeros(1, np.int32)
    out = np.zeros(len(rs))
    fn = lib.ref_fit_calibrate
    fn.argtypes = [f64p, i32p, C.c_int32, f64p, C.c_int32, f64p, f64p, f64p, C.c_int32, i32p, f64p]
    st = fn(_p(raw, f64p), _p(oc, i32p), len(raw), _p(rs, f64p), len(rs), _p(lo, f64p),
            _p(hi, f64p), _p(val, f64p), cap, _p(nb, i32p), _p(out, f64p))
    if st != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    n = int(nb[0])
    return lo[:n], hi[:n], val[:n], out


# ------------------------------------------------------------------ base64
def ref_decode_f32_base64(text: str):
    """The reference's decode_f32_base64 (oracle/_ref) -> (floats | None, status, message)."""
    lib = ref()
    b = text.encode("latin-1")
    cap = len(b) // 4 * 3 // 4 + 1
    out = np.zeros(cap, np.float32)
    n = np.zeros(1, np.int64)
    fn = lib.ref_decode_f32_base64
    fn.argtypes = [C.c_char_p, C.c_int64, f32p, C.c_int64, i64p]
    st = fn(b, len(b), _p(out, f32p), cap, _p(n, i64p))
    if st != 0:
        return None, st - 1, lib.ref_last_error().decode()
    return out[:int(n[0])], 0, ""


# ------------------------------------------------------------ score cache
def ref_canonical_query(text: str, filters):
    """canonical_query + fnv1a64 (midtier.cpp:14-53) via oracle/_ref.
    filters: list of (attr, value) pairs."""
    lib = ref()
    n = len(filters)
    A = (C.c_char_p * max(n, 1))(*[a.encode() for a, _ in filters])
    V = (C.c_char_p * max(n, 1))(*[v.encode() for _, v in filters])
    cap = 4 * (len(text.encode()) + sum(len(a) + len(v) + 2 for a, v in filters)) + 16
    out = C.create_string_buffer(cap)
    ln = C.c_int64(0)
    h = C.c_uint64(0)
    fn = lib.ref_canonical_query
    fn.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
                   C.c_char_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
    st = fn(text.encode(), n, A, V, out, cap, C.byref(ln), C.byref(h))
    if st != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return out.raw[:ln.value].decode(), int(h.value)


def ref_cache_trace(capacity: int, ops):
    """Run ops [(op, searcher, sig, entity, version, value)] on the
    reference's ScoreCache -> (status, [(hit_or_status, value, size)])."""
    lib = ref()
    n = len(ops)
    op = np.array([o[0] for o in ops] or [0], np.int32)
    S = (C.c_char_p * max(n, 1))(*[o[1].encode() for o in ops])
    sig = np.array([o[2] for o in ops] or [0], np.uint64)
    ent = np.array([o[3] for o in ops] or [0], np.int64)
    Vv = (C.c_char_p * max(n, 1))(*[o[4].encode() for o in ops])
    val = np.array([o[5] for o in ops] or [0], np.float64)
    hit = np.zeros(max(n, 1), np.int32)
    outv = np.zeros(max(n, 1), np.float64)
    size = np.zeros(max(n, 1), np.int64)
    fn = lib.ref_cache_trace
    fn.argtypes = [C.c_int64, C.c_int32, i32p, C.POINTER(C.c_char_p), C.POINTER(C.c_uint64), i64p,
                   C.POINTER(C.c_char_p), f64p, i32p, f64p, i64p]
    st = fn(capacity, n, _p(op, i32p), S, _p(sig, C.POINTER(C.c_uint64)), _p(ent, i64p), Vv,
            _p(val, f64p), _p(hit, i32p), _p(outv, f64p), _p(size, i64p))
    msg = lib.ref_last_error().decode() if st != 0 else ""
    return st, msg, [(int(hit[i]), float(outv[i]), int(size[i])) for i in range(n)]


# ------------------------------------------------------------- text API
def ref_build_prompt(system: bytes, query: bytes, document: bytes, max_seq: int):
    """(status, message, prefix_tokens, item_tokens) from prompt.cpp:14-38."""
    lib = ref()
    cap = len(system) + len(query) + len(document) + 64
    pre, item, n = (np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(2, np.int32))
    st = lib.ref_build_prompt(system, query, document, max_seq, _p(pre, i32p), _p(item, i32p), cap,
                              _p(n, i32p))
    msg = lib.ref_last_error().decode() if st else ""
    return st, msg, pre[:n[0]].tolist() if st == 0 else None, item[:n[1]].tolist() if st == 0 else None


def ref_score_result_json(request_id: bytes, ids, names, scores, attention: float, linear: float):
    """score_result_to_json (service.cpp:380-391) over the reference's nlohmann::json."""
    lib = ref()
    sc = np.ascontiguousarray(scores, np.float64).reshape(len(ids), len(names))
    cid = (C.c_char_p * max(1, len(ids)))(*ids)
    cnm = (C.c_char_p * max(1, len(names)))(*names)
    n = np.zeros(1, np.int64)
    st = lib.ref_score_result_json(request_id, len(ids), cid, len(names), cnm, _p(sc, f64p),
                                   attention, linear, None, 0, _p(n, i64p))
    if st != 0:
        return st, lib.ref_last_error().decode(), None
    buf = C.create_string_buffer(int(n[0]) + 1)
    lib.ref_score_result_json(request_id, len(ids), cid, len(names), cnm, _p(sc, f64p), attention,
                              linear, buf, int(n[0]), _p(n, i64p))
    return 0, "", buf.raw[:int(n[0])]
