"""Python mirror of the reference scorer API (semrank, include/semrank/*.hpp).

Same names, argument meaning and error behaviour as the reference C++ API so
parity tests read like the reference's own tests; every call goes through the
C-ABI (include/semrank_b200.h) into the B200 engine. Nothing here computes
scores on the host.

  reference                                   here
  ModelConfig / HeadSpec   (model.hpp:16-40)  ModelConfig / HeadSpec
  ModelWeights, init_model (model.hpp:56-70)  ModelWeights, init_model
  save/load_weights   (weights_io.hpp:16-17)  save_weights / load_weights
  ScoreMode/Item/Request/Result (engine.hpp)  same names
  flops, build_multi_item_mask, plan_batches  same names (host-side logic)
  ScoringEngine::score  (engine.hpp:109-119)  ScoringEngine.score (+ top-k)
  semrank::Error{ErrorCode} (error.hpp)       SemrankError(code)
"""
from __future__ import annotations

import ctypes as C
import sys as _sys
from itertools import accumulate as _accumulate
import enum
from dataclasses import dataclass, field
from typing import Dict, List, Mapping, Optional, Sequence

import numpy as np

from . import _capi as _c
from ._capi import lib as _lib


class ErrorCode(enum.IntEnum):
    """semrank::ErrorCode (error.hpp:13-29); values are the C-ABI statuses."""
    LengthOverflow = 1
    MaskInvalid = 2
    SpecViolation = 3
    PayloadInvalid = 4
    SchemaUnknown = 5
    Alignment = 6
    Divergence = 7
    Parameter = 8
    DegenerateInput = 9
    UndefinedMetric = 10
    StateInvalid = 11
    OversizeItem = 12
    Consistency = 13
    Reconciliation = 14
    Io = 15
    Cuda = 100
    Nccl = 101


class SemrankError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = ErrorCode(code)


def _check(status: int) -> None:
    if status != 0:
        msg = _lib.sr_last_error().decode(errors="replace")
        raise SemrankError(status, f"[{_lib.sr_status_name(status).decode()}] {msg}")


class ScoreMode(enum.IntEnum):
    Naive = 0
    Ibpc = 1
    MultiItem = 2
    Mixed = 3


_MODE_NAMES = {ScoreMode.Naive: "naive", ScoreMode.Ibpc: "ibpc",
               ScoreMode.MultiItem: "multi_item", ScoreMode.Mixed: "mixed"}


def score_mode_name(mode: ScoreMode) -> str:  # engine.cpp:12-20
    return _MODE_NAMES.get(ScoreMode(mode), "unknown")


def score_mode_from_name(name: str) -> ScoreMode:  # engine.cpp:22-29
    for m, n in _MODE_NAMES.items():
        if n == name:
            return m
    if name == "multi-item":
        return ScoreMode.MultiItem
    raise SemrankError(ErrorCode.Parameter, "unknown scoring mode: " + name)


kRelevanceTask = "relevance"


@dataclass
class HeadSpec:
    name: str
    arity: int = 1


@dataclass
class ModelConfig:
    n_layers: int = 2
    d_model: int = 64
    n_heads: int = 4
    d_ff: int = 256
    vocab_size: int = 300
    max_seq: int = 4096
    yes_token_id: int = 261
    no_token_id: int = 262
    head_specs: List[HeadSpec] = field(default_factory=list)

    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @staticmethod
    def default_toy() -> "ModelConfig":  # model.cpp:52-57
        return ModelConfig(head_specs=[HeadSpec(n) for n in
                                       ("click", "apply", "badfit", "shortlist", "dismiss")])

    def _to_c(self):
        names = (C.c_char_p * max(1, len(self.head_specs)))(
            *[h.name.encode() for h in self.head_specs])
        arity = (C.c_int32 * max(1, len(self.head_specs)))(*[h.arity for h in self.head_specs])
        c = _c.ModelConfigC(self.n_layers, self.d_model, self.n_heads, self.d_ff,
                            self.vocab_size, self.max_seq, self.yes_token_id, self.no_token_id,
                            len(self.head_specs), names, arity)
        c._keep = (names, arity)
        return c

    def validate(self) -> None:  # model.cpp:29-50
        c = self._to_c()
        _check(_lib.sr_config_validate(C.byref(c)))

    @staticmethod
    def _from_c(c) -> "ModelConfig":
        heads = [HeadSpec(c.head_names[i].decode(), c.head_arity[i]) for i in range(c.n_task_heads)]
        return ModelConfig(c.n_layers, c.d_model, c.n_heads, c.d_ff, c.vocab_size, c.max_seq,
                           c.yes_token_id, c.no_token_id, heads)


class _OwnedBuffer:
    """float32 array interface over library memory that pins its owner."""

    def __init__(self, owner, addr: int, n: int):
        self._owner = owner
        self.__array_interface__ = {"data": (addr, False), "shape": (n,), "typestr": "<f4",
                                    "version": 3}


class ModelWeights:
    """Host weights (model.hpp:56-67), owned by the C library."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        cfg = _c.ModelConfigC()
        _check(_lib.sr_weights_config(self._h, C.byref(cfg)))
        self.config = ModelConfig._from_c(cfg)
        self.version = _lib.sr_weights_version(self._h).decode()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and not _sys.is_finalizing():  # process exit frees it
            _lib.sr_weights_free(h)
            self._h = C.c_void_p()

    def tensors(self) -> Dict[str, np.ndarray]:
        """name -> zero-copy float32 view, in SRNKWTS1 canonical order.

        Each view keeps this ModelWeights alive (its base holds a reference),
        so views may outlive the Python handle they came from."""
        out = {}
        n = _lib.sr_weights_tensor_count(self._h)
        for i in range(n):
            name = C.c_char_p()
            data = C.POINTER(C.c_float)()
            numel = C.c_size_t()
            _check(_lib.sr_weights_tensor(self._h, i, C.byref(name), C.byref(data), C.byref(numel)))
            if numel.value:
                arr = np.asarray(_OwnedBuffer(self, C.cast(data, C.c_void_p).value, numel.value))
            else:
                arr = np.zeros(0, np.float32)
            out[name.value.decode()] = arr
        return out

    def save(self, path: str) -> None:
        _check(_lib.sr_weights_save(self._h, path.encode()))

    @staticmethod
    def from_tensors(cfg: ModelConfig, tensors: Sequence[np.ndarray], version: str = "") \
            -> "ModelWeights":
        arrs = [np.ascontiguousarray(t, dtype=np.float32).ravel() for t in tensors]
        ptrs = (C.POINTER(C.c_float) * len(arrs))(
            *[a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrs])
        c = cfg._to_c()
        h = C.c_void_p()
        _check(_lib.sr_weights_from_tensors(C.byref(c), version.encode(), ptrs, C.byref(h)))
        return ModelWeights(h)


def init_model(config: ModelConfig, seed: int, scheme: str = "reference") -> ModelWeights:
    """init_model (model.cpp:94-134). scheme "fan_in" = DESIGN.md §2 scaled init."""
    sch = {"reference": 0, "fan_in": 1}[scheme]
    c = config._to_c()
    h = C.c_void_p()
    _check(_lib.sr_weights_init(C.byref(c), C.c_uint64(seed), sch, C.byref(h)))
    return ModelWeights(h)


def load_weights(path: str) -> ModelWeights:
    h = C.c_void_p()
    _check(_lib.sr_weights_load(path.encode(), C.byref(h)))
    return ModelWeights(h)


def save_weights(w: ModelWeights, path: str) -> None:
    w.save(path)


# ------------------------------------------------------------------ engine
@dataclass
class FlopReport:
    attention_units: float = 0.0
    linear_units: float = 0.0
    t_q: float = 0.0
    t_i_mean: float = 0.0
    n_items: float = 0.0

    @staticmethod
    def _from_c(f) -> "FlopReport":
        return FlopReport(f.attention_units, f.linear_units, f.t_q, f.t_i_mean, f.n_items)


def flops(mode: ScoreMode, t_q: int, t_i: int, n_items: int) -> FlopReport:  # engine.cpp:30-47
    f = _c.FlopReportC()
    _check(_lib.sr_flops(int(mode), t_q, t_i, n_items, C.byref(f)))
    return FlopReport._from_c(f)


@dataclass
class ScoreItem:
    id: str = ""
    tokens: Sequence[int] = ()
    embedding: Optional[np.ndarray] = None  # mixed mode: [n_emb_tokens x d_model]
    n_emb_tokens: int = 0
    embedding_b64: Optional[str] = None  # wire form (decoded on the device)


@dataclass
class ScoreRequest:
    request_id: str = ""
    prefix_tokens: Sequence[int] = ()
    items: List[ScoreItem] = field(default_factory=list)
    mode: ScoreMode = ScoreMode.Ibpc
    latency_sensitive: bool = False


@dataclass
class ItemScores:
    item_id: str
    tasks: Dict[str, float]


@dataclass
class ScoreResult:
    request_id: str = ""
    items: List[ItemScores] = field(default_factory=list)
    mode: ScoreMode = ScoreMode.Naive
    flops: FlopReport = field(default_factory=FlopReport)
    kv_incremental_per_item: float = 0.0
    topk: List[tuple] = field(default_factory=list)  # (item_id, relevance or final score)
    scores: Optional[np.ndarray] = None  # [n_items x n_tasks], col 0 relevance
    final_scores: Optional[np.ndarray] = None  # [n_items] with post-processing on
    cache_hits: int = 0  # score_cached: items served from the ScoreCache


class MultiItemMask:  # engine.hpp:63-72
    def __init__(self, prefix_len: int, item_spans: List[tuple]):
        self.prefix_len = prefix_len
        self.item_spans = item_spans

    def allowed_pair_count(self) -> int:
        lens = np.array([e - s for s, e in self.item_spans], np.int32)
        out = C.c_int64()
        _check(_lib.sr_multi_item_pair_count(
            self.prefix_len, lens.ctypes.data_as(C.POINTER(C.c_int32)), len(lens), C.byref(out)))
        return out.value

    def to_attention_mask(self) -> List[tuple]:
        """[(prefix_end, span_start)] per packed item row."""
        lens = np.array([e - s for s, e in self.item_spans], np.int32)
        n_rows = int(lens.sum())
        buf = np.zeros(2 * max(n_rows, 1), np.int32)
        nr = C.c_int32()
        _check(_lib.sr_multi_item_mask(self.prefix_len, lens.ctypes.data_as(C.POINTER(C.c_int32)),
                                       len(lens), buf.ctypes.data_as(C.POINTER(C.c_int32)),
                                       n_rows, C.byref(nr)))
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(nr.value)]


def build_multi_item_mask(prefix_len: int, item_lengths: Sequence[int]) -> MultiItemMask:
    lens = np.asarray(list(item_lengths), np.int32)
    nr = C.c_int32()
    _check(_lib.sr_multi_item_mask(prefix_len, lens.ctypes.data_as(C.POINTER(C.c_int32)),
                                   len(lens), None, 0, C.byref(nr)))
    spans, cur = [], prefix_len
    for l in lens:
        spans.append((cur, cur + int(l)))
        cur += int(l)
    return MultiItemMask(prefix_len, spans)


@dataclass
class BatchEntry:
    request_index: int
    item_begin: int
    item_end: int


@dataclass
class Batch:
    entries: List[BatchEntry] = field(default_factory=list)
    token_count: int = 0


def _item_len(it: ScoreItem) -> int:
    return it.n_emb_tokens if it.n_emb_tokens > 0 else len(it.tokens)


def plan_batches(requests: Sequence[ScoreRequest], max_batch_tokens: int) -> List[Batch]:
    """plan_batches (engine.cpp:278-326), computed by the native planner."""
    pl = np.array([len(r.prefix_tokens) for r in requests], np.int32)
    off = np.zeros(len(requests) + 1, np.int32)
    lens = []
    for i, r in enumerate(requests):
        lens += [_item_len(it) for it in r.items]
        off[i + 1] = len(lens)
    il = np.array(lens if lens else [0], np.int32)
    cap_e, cap_b = max(1, len(lens)), max(1, len(lens))
    ent = np.zeros(4 * cap_e, np.int32)
    tok = np.zeros(cap_b, np.int64)
    ne, nb = C.c_int32(), C.c_int32()
    I = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    _check(_lib.sr_plan_batches(len(requests), I(pl), I(off), I(il), max_batch_tokens, I(ent), cap_e,
                                C.byref(ne), tok.ctypes.data_as(C.POINTER(C.c_int64)), cap_b,
                                C.byref(nb)))
    batches = [Batch(token_count=int(tok[b])) for b in range(nb.value)]
    for e in range(ne.value):
        b, r, lo, hi = (int(x) for x in ent[4 * e:4 * e + 4])
        batches[b].entries.append(BatchEntry(r, lo, hi))
    return batches


def request_report(config: ModelConfig, request: ScoreRequest):
    """Host-side validation + the reference FlopReport for the request's mode."""
    pr = _PackedRequest(request, config.d_model)
    c = config._to_c()
    f = _c.FlopReportC()
    kv = C.c_double()
    _check(_lib.sr_request_report(C.byref(c), C.byref(pr.c), C.byref(f), C.byref(kv)))
    return FlopReport._from_c(f), kv.value


def _item_doc_ids(items: Sequence[ScoreItem]) -> Optional[np.ndarray]:
    try:
        return np.fromiter(map(int, (it.id for it in items)), np.int64, len(items))
    except (TypeError, ValueError):
        return None


def _addresses(arrs) -> List[int]:
    try:  # ~3x cheaper per array than ndarray.ctypes.data
        return [C.addressof(C.c_char.from_buffer(a)) for a in arrs]
    except (TypeError, ValueError):  # read-only or empty buffers
        return [a.ctypes.data for a in arrs]


def _adjacent_rows(arrs) -> np.ndarray:
    """The items' embedding arrays as one contiguous float32 array. When they
    are already consecutive slices of one buffer (a [N x n x d] batch), that
    buffer is used in place — the engine then copies it straight to HBM —
    instead of being gathered into a new array."""
    a0 = arrs[0]
    if type(a0) is np.ndarray and a0.dtype == np.float32 and a0.flags.c_contiguous and a0.size:
        shp, st, dt = a0.shape, a0.strides, a0.dtype
        # same shape and strides as a C-contiguous a0 => each is C-contiguous
        if all(type(a) is np.ndarray and a.shape == shp and a.strides == st and a.dtype is dt
               for a in arrs):
            ptrs = _addresses(arrs)
            base, step = ptrs[0], a0.nbytes
            if all(p == base + i * step for i, p in enumerate(ptrs)):
                total = len(arrs) * a0.size
                root = a0
                while isinstance(root.base, np.ndarray):
                    root = root.base
                if root.dtype == np.float32 and root.flags.c_contiguous:
                    lo = (base - root.ctypes.data) // 4
                    flat = root.reshape(-1)
                    if 0 <= lo and lo + total <= flat.size:
                        return flat[lo:lo + total]
    return np.ascontiguousarray(np.concatenate(
        [np.asarray(a, np.float32).reshape(-1) for a in arrs]))


class _LazyIds(Sequence):
    """Item ids as strings for an int64 id array (or 0..n-1), converted on
    access."""

    def __init__(self, ids_or_n):
        self._ids = ids_or_n

    def __len__(self):
        return self._ids if isinstance(self._ids, int) else len(self._ids)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if isinstance(self._ids, int):
            if not -self._ids <= i < self._ids:
                raise IndexError(i)
            return str(i % self._ids)
        return str(int(self._ids[i]))


class _LazyItemScores(Sequence):
    """ScoreResult.items (engine.hpp:46-51): built on first access from the
    score matrix, so callers that only need the top-k or the matrix do not
    pay for n_items Python dicts per call."""

    def __init__(self, ids, scores, names):
        self._ids, self._scores, self._names, self._items = ids, scores, names, None

    def _build(self):
        if self._items is None:
            names = self._names
            self._items = [ItemScores(i, dict(zip(names, row)))
                           for i, row in zip(self._ids, self._scores.tolist())]
        return self._items

    def __len__(self):
        return len(self._ids)

    def __getitem__(self, i):
        return self._build()[i]

    def __iter__(self):
        return iter(self._build())

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self):
        return repr(self._build())


class _WireIds(Sequence):
    """Item ids of a parsed /score body, read from the native handle on
    demand (the handle and the body it points into live as long as this)."""

    def __init__(self, h, raw: bytes, n: int):
        self._h, self._raw, self._n, self._cache = h, raw, n, None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.sr_wire_destroy(h)
            self._h = C.c_void_p()

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if self._cache is None:
            if isinstance(i, slice):
                return [self[j] for j in range(*i.indices(self._n))]
            if not -self._n <= i < self._n:
                raise IndexError(i)
            return _lib.sr_wire_item_id(self._h, i % self._n).decode()
        return self._cache[i]

    def __iter__(self):
        if self._cache is None:
            self._cache = [_lib.sr_wire_item_id(self._h, i).decode() for i in range(self._n)]
        return iter(self._cache)


_PI32, _PI64, _PF32, _PF64 = (C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_float),
                              C.POINTER(C.c_double))
_SCALAR = {_PI32: C.c_int32, _PI64: C.c_int64, _PF32: C.c_float, _PF64: C.c_double}


def _ptr(a: np.ndarray, ptype):
    """Typed pointer to a contiguous array's data (~3x cheaper than
    ndarray.ctypes.data_as; read-only buffers take the slow path)."""
    try:
        return ptype(_SCALAR[ptype].from_buffer(a))
    except (TypeError, ValueError):
        return a.ctypes.data_as(ptype)


class _PackedRequest:
    """Flattened sr_request; keeps the numpy buffers alive. ``want_ids``
    False leaves sr_request.item_ids null (the result's top-k is then mapped
    back to the items by index)."""

    def __init__(self, req: ScoreRequest, d_model: int, item_ids: Optional[np.ndarray] = None,
                 want_ids: bool = True):
        self.prefix = np.ascontiguousarray(np.asarray(req.prefix_tokens, np.int32).reshape(-1))
        items = req.items
        n = len(items)
        mixed = ScoreMode(req.mode) == ScoreMode.Mixed
        if mixed:
            lens = [it.n_emb_tokens for it in items]
            arrs = [it.embedding for it in items]
            for i, (it, ln, e) in enumerate(zip(items, lens, arrs)):
                if type(e) is not np.ndarray:
                    e = arrs[i] = np.asarray(e if e is not None else [], np.float32)
                if ln < 1 or e.size != ln * d_model:
                    raise SemrankError(ErrorCode.PayloadInvalid,
                                       f"item {it.id} embedding payload is not [n x {d_model}]")
            self.rows = _adjacent_rows(arrs) if items else np.zeros(1, np.float32)
            self.tokens = np.zeros(1, np.int32)
        else:
            toks = [it.tokens for it in items]
            lens = [len(t) for t in toks]
            self.tokens = (np.ascontiguousarray(np.concatenate(toks).astype(np.int32, copy=False))
                           if toks and any(lens) else np.zeros(1, np.int32))
            self.rows = None
        self.offsets = np.fromiter(_accumulate(lens, initial=0), np.int32, n + 1)
        self.ids = (item_ids if item_ids is not None
                    else _item_doc_ids(items) if want_ids else None)
        self.c = _c.RequestC(
            _ptr(self.prefix, _PI32), len(self.prefix), n, _ptr(self.offsets, _PI32),
            _ptr(self.tokens, _PI32),
            _ptr(self.rows, _PF32) if self.rows is not None else None,
            _ptr(self.ids, _PI64) if self.ids is not None else None,
            int(req.mode))


class _ResultBuf:
    def __init__(self, n_items: int, n_tasks: int, k: int):
        # every field the caller reads is written by the library (scores for
        # n_items rows, the first k_returned top-k entries)
        self.scores = np.empty((max(n_items, 1), n_tasks), np.float64)
        self.kk = max(k, 1)
        self.ids = np.empty(self.kk, np.int64)
        self.top = np.empty(self.kk, np.float64)
        self.idx = np.empty(self.kk, np.int32)
        self.c = _c.ResultC(_ptr(self.scores, _PF64), k, _ptr(self.ids, _PI64),
                            _ptr(self.top, _PF64), _ptr(self.idx, _PI32),
                            _c.FlopReportC(), 0.0, 0)

    def topk(self, name) -> List[tuple]:
        """(item id, score) of the returned top-k; ``name(i)`` maps an item
        index to its id (a negative index, no local item: the global doc id)."""
        kr = self.c.k_returned
        return [(name(i) if i >= 0 else str(g), t) for i, g, t in
                zip(self.idx[:kr].tolist(), self.ids[:kr].tolist(), self.top[:kr].tolist())]


@dataclass
class CalibrationBlock:  # calibration.hpp:18-23
    lo: float = 0.0
    hi: float = 0.0
    value: float = 0.0
    count: int = 0


@dataclass
class CalibrationHead:  # calibration.hpp:17-27 (fitted offline by fit_isotonic)
    blocks: List[CalibrationBlock] = field(default_factory=list)

    def fitted(self) -> bool:
        return bool(self.blocks)


def _filter_arrays(filters: Optional[Mapping[str, Sequence[str]]]):
    pairs = [(a, v) for a, vs in (filters or {}).items() for v in vs]
    attrs = (C.c_char_p * max(len(pairs), 1))(*[a.encode() for a, _ in pairs])
    vals = (C.c_char_p * max(len(pairs), 1))(*[v.encode() for _, v in pairs])
    return len(pairs), attrs, vals


def canonical_query(query_text: str, filters: Optional[Mapping[str, Sequence[str]]] = None) -> str:
    """midtier.cpp:14-44 (native): lowercase, collapse and trim whitespace,
    then ``|attr=v1,v2`` per attribute in sorted order with sorted values."""
    n, attrs, vals = _filter_arrays(filters)
    text = query_text.encode()
    ln = C.c_int64(0)
    _check(_lib.sr_canonical_query(text, n, attrs, vals, None, 0, C.byref(ln)))
    buf = C.create_string_buffer(max(ln.value, 1))
    _check(_lib.sr_canonical_query(text, n, attrs, vals, buf, ln.value, C.byref(ln)))
    return buf.raw[:ln.value].decode()


def fnv1a64(text) -> int:  # midtier.cpp:46-53
    raw = text.encode() if isinstance(text, str) else bytes(text)
    return int(_lib.sr_fnv1a64(raw, len(raw)))


def query_signature(query_text: str, filters: Optional[Mapping[str, Sequence[str]]] = None) -> int:
    """fnv1a64(canonical_query(...)), the signature handle_search keys the cache with."""
    n, attrs, vals = _filter_arrays(filters)
    out = C.c_uint64(0)
    _check(_lib.sr_query_signature(query_text.encode(), n, attrs, vals, C.byref(out)))
    return int(out.value)


@dataclass(frozen=True)
class CacheKey:  # midtier.hpp:30-37
    searcher_id: str
    query_signature: int
    entity_id: int
    model_version: str


class ScoreCache:
    """ScoreCache (midtier.hpp:42-69) in native code: LRU over whole entries,
    get refreshes recency, a conflicting put raises Consistency. Rows are
    stored in ``task_names`` order (the engine's: relevance, then heads)."""

    def __init__(self, capacity: int, task_names: Optional[Sequence[str]] = None):
        if task_names is None:
            task_names = [kRelevanceTask] + [h.name for h in ModelConfig.default_toy().head_specs]
        self.task_names = list(task_names)
        h = C.c_void_p()
        _check(_lib.sr_score_cache_create(int(capacity), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and not _sys.is_finalizing():  # process exit frees it
            _lib.sr_score_cache_destroy(h)
            self._h = C.c_void_p()

    def get(self, key: CacheKey) -> Optional[Dict[str, float]]:
        row = np.zeros(len(self.task_names), np.float64)
        hit = C.c_int32(0)
        _check(_lib.sr_score_cache_get(self._h, key.searcher_id.encode(), key.query_signature,
                                       key.entity_id, key.model_version.encode(),
                                       row.ctypes.data_as(C.POINTER(C.c_double)), len(row),
                                       C.byref(hit)))
        return dict(zip(self.task_names, row.tolist())) if hit.value else None

    def put(self, key: CacheKey, scores: Mapping[str, float]) -> None:
        if set(scores) != set(self.task_names):
            raise SemrankError(ErrorCode.Alignment, "score map does not match the cache's tasks")
        row = np.array([scores[t] for t in self.task_names], np.float64)
        _check(_lib.sr_score_cache_put(self._h, key.searcher_id.encode(), key.query_signature,
                                       key.entity_id, key.model_version.encode(),
                                       row.ctypes.data_as(C.POINTER(C.c_double)), len(row)))

    def size(self) -> int:
        return int(_lib.sr_score_cache_size(self._h))

    def capacity(self) -> int:
        return int(_lib.sr_score_cache_capacity(self._h))


class ScoringEngine:
    """ScoringEngine (engine.hpp:109-119) bound to one B200; serialises callers."""

    _post = False

    def __init__(self, weights: ModelWeights, device: int = 0):
        self.weights = weights
        self.config = weights.config
        self.task_names = [kRelevanceTask] + [h.name for h in self.config.head_specs]
        h = C.c_void_p()
        _check(_lib.sr_engine_create(weights._h, device, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and not _sys.is_finalizing():  # process exit frees it
            _lib.sr_engine_destroy(h)
            self._h = C.c_void_p()

    def _to_result(self, req: ScoreRequest, rb: _ResultBuf) -> ScoreResult:
        n = len(req.items)
        res = ScoreResult(request_id=req.request_id, mode=ScoreMode(req.mode),
                          flops=FlopReport._from_c(rb.c.flops),
                          kv_incremental_per_item=rb.c.kv_incremental_per_item,
                          scores=rb.scores[:n].copy())
        items = req.items
        res.items = _LazyItemScores([it.id for it in items], res.scores, self.task_names)
        res.topk = rb.topk(lambda i: items[i].id)
        return res

    def score(self, request: ScoreRequest, k: int = 0) -> ScoreResult:
        rb = _ResultBuf(len(request.items), len(self.task_names), k)
        if (ScoreMode(request.mode) == ScoreMode.Mixed and request.items
                and all(it.embedding_b64 is not None for it in request.items)):
            self._score_b64(request, rb)
        else:
            pr = _PackedRequest(request, self.config.d_model)
            _check(_lib.sr_engine_score(self._h, C.byref(pr.c), C.byref(rb.c)))
        res = self._to_result(request, rb)
        if self._post:
            res.final_scores = self._final(len(request.items))
        return res

    def score_cached(self, request: ScoreRequest, cache: ScoreCache, searcher_id: str,
                     query_signature: int, k: int = 0, model_version: Optional[str] = None,
                     entity_ids: Optional[Sequence[int]] = None) -> ScoreResult:
        """handle_search's cache path (service.cpp:160-234): cached items are
        served from ``cache``, the misses are scored in one device pass and put
        back, then every row is ranked on the device. Item ids (or
        ``entity_ids``) are the cache keys' entity ids; ``model_version``
        defaults to the weights' version string."""
        if cache.task_names != self.task_names:
            raise SemrankError(ErrorCode.Alignment, "cache tasks differ from the engine's tasks")
        ids = (np.ascontiguousarray(np.asarray(entity_ids, np.int64)) if entity_ids is not None
               else _item_doc_ids(request.items))
        if ids is None:
            raise SemrankError(ErrorCode.SpecViolation,
                               "cached scoring needs integer entity ids (item ids or entity_ids)")
        pr = _PackedRequest(request, self.config.d_model, ids)
        rb = _ResultBuf(len(request.items), len(self.task_names), k)
        hits = C.c_int32(0)
        version = self.weights.version if model_version is None else model_version
        _check(_lib.sr_engine_score_cached(self._h, cache._h, searcher_id.encode(),
                                           int(query_signature), version.encode(),
                                           C.byref(pr.c), C.byref(rb.c), C.byref(hits)))
        res = self._to_result(request, rb)
        res.cache_hits = hits.value
        if self._post:
            res.final_scores = self._final(len(request.items))
        return res

    def score_json(self, body, k: int = 0, max_seq: Optional[int] = None) -> ScoreResult:
        """The /score wire path in native code: the body is parsed in one pass
        (sr_wire_parse) and embedding_b64 payloads go to the device as spans of
        the body, decoded in HBM (sr_engine_score_wire)."""
        raw = body.encode("utf-8") if isinstance(body, str) else bytes(body)
        h = C.c_void_p()
        _check(_lib.sr_wire_parse(raw, len(raw), max_seq or self.config.max_seq, C.byref(h)))
        n, mode, tq = C.c_int32(), C.c_int32(), C.c_int32()
        ids = None
        try:
            _check(_lib.sr_wire_info(h, C.byref(n), C.byref(mode), C.byref(tq)))
            ids = _WireIds(h, raw, n.value)  # owns the handle from here on
            rb = _ResultBuf(n.value, len(self.task_names), k)
            _check(_lib.sr_engine_score_wire(self._h, h, C.byref(rb.c)))
            rid = _lib.sr_wire_request_id(h).decode()
        finally:
            if ids is None:
                _lib.sr_wire_destroy(h)
        nv = n.value
        res = ScoreResult(request_id=rid, mode=ScoreMode(mode.value),
                          flops=FlopReport._from_c(rb.c.flops),
                          kv_incremental_per_item=rb.c.kv_incremental_per_item,
                          scores=rb.scores[:nv].copy())
        res.items = _LazyItemScores(ids, res.scores, self.task_names)
        res.topk = rb.topk(ids.__getitem__)
        if self._post:
            res.final_scores = self._final(nv)
        return res

    def _score_b64(self, request: ScoreRequest, rb: "_ResultBuf") -> None:
        """embedding_b64 items: the base64 text goes to the device as is."""
        parts = [it.embedding_b64.encode("ascii", "replace") for it in request.items]
        off = np.zeros(len(parts) + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in parts])
        text = b"".join(parts)
        prefix = np.ascontiguousarray(np.asarray(request.prefix_tokens, np.int32).reshape(-1))
        ids = _item_doc_ids(request.items)
        _check(_lib.sr_engine_score_b64(
            self._h, prefix.ctypes.data_as(C.POINTER(C.c_int32)), len(prefix), text,
            off.ctypes.data_as(C.POINTER(C.c_int64)), len(parts),
            ids.ctypes.data_as(C.POINTER(C.c_int64)) if ids is not None else None, C.byref(rb.c)))

    # ------------------------------------------------ compact embeddings
    EMB_PAD, EMB_PROJECT = 0, 1  # sr_emb_form

    def reserve(self, rows: int) -> None:
        """Workspace for passes of up to `rows` packed rows (sr_engine_reserve):
        call once with the largest pass before warming pass shapes, so no later
        growth invalidates their captured graphs."""
        _check(_lib.sr_engine_reserve(self._h, int(rows)))

    def set_projection(self, proj: Optional[np.ndarray], n_soft: int = 0) -> None:
        """Context compression (north_star (d)): P [d_emb x n_soft*d_model] in
        the reference's weight layout; each item's compact embedding becomes
        n_soft soft-token rows bf16(e).bf16(P) on the tensor cores. None removes it."""
        if proj is None:
            _check(_lib.sr_engine_set_projection(self._h, None, 0, 0))
            return
        P_ = np.ascontiguousarray(proj, np.float32)
        d = self.config.d_model
        if P_.ndim != 2 or (n_soft and P_.shape[1] != n_soft * d) or P_.shape[1] % d:
            raise SemrankError(ErrorCode.Alignment,
                               f"projection must be [d_emb x n_soft*{d}], got {P_.shape}")
        self._proj = P_.shape
        _check(_lib.sr_engine_set_projection(self._h, P_.ctypes.data_as(C.POINTER(C.c_float)),
                                             P_.shape[0], P_.shape[1] // d))

    @staticmethod
    def _emb_form(form) -> int:
        if form in ("pad", 0):
            return 0
        if form in ("project", 1):
            return 1
        raise SemrankError(ErrorCode.Parameter, f"unknown embedding form: {form}")

    def score_embeddings(self, prefix_tokens, embeddings: np.ndarray, form="project", k: int = 0,
                         item_ids=None, request_id: str = "") -> ScoreResult:
        """Mixed-mode scoring of items given as compact embeddings [n x d_emb]
        (sr_engine_score_emb): form "pad" = the service's one zero-padded row
        per item (service.cpp:208-217), "project" = n_soft projected rows."""
        prefix = np.ascontiguousarray(np.asarray(prefix_tokens, np.int32).reshape(-1))
        emb = np.ascontiguousarray(embeddings, np.float32)
        if emb.ndim != 2:
            raise SemrankError(ErrorCode.PayloadInvalid, "embeddings must be [n x d_emb]")
        n = emb.shape[0]
        ids = None if item_ids is None else np.ascontiguousarray(np.asarray(item_ids, np.int64))
        rb = _ResultBuf(n, len(self.task_names), k)
        _check(_lib.sr_engine_score_emb(
            self._h, prefix.ctypes.data_as(C.POINTER(C.c_int32)), len(prefix),
            emb.ctypes.data_as(C.POINTER(C.c_float)), emb.shape[1], n,
            ids.ctypes.data_as(C.POINTER(C.c_int64)) if ids is not None else None,
            self._emb_form(form), C.byref(rb.c)))
        # item ids as strings, made on access only (no per-item objects per call)
        names = _LazyIds(ids if ids is not None else n)
        res = ScoreResult(request_id=request_id, mode=ScoreMode.Mixed,
                          flops=FlopReport._from_c(rb.c.flops),
                          kv_incremental_per_item=rb.c.kv_incremental_per_item,
                          scores=rb.scores[:n].copy())
        res.items = _LazyItemScores(names, res.scores, self.task_names)
        res.topk = rb.topk(names.__getitem__)
        if self._post:
            res.final_scores = self._final(n)
        return res

    def plan_embeddings(self, prefix_tokens, embeddings: np.ndarray, form="project", k: int = 0,
                        item_ids=None) -> "Plan":
        """Resident variant of score_embeddings (the pad / projection step is
        inside the plan's CUDA graph)."""
        return EmbPlan(self, prefix_tokens, embeddings, form, k, item_ids)

    def set_postprocess(self, calibration: Optional["CalibrationHead"] = None,
                        score_blend: Optional[Dict[str, float]] = None) -> None:
        """The service's output side on the device (service.cpp:242-277):
        calibrated relevance (fitted isotonic head, calibration.cpp:65-88) and
        the optional ``score_blend`` (task -> weight, summed in task-name order
        like the reference's std::map); the top-k then ranks by the final score."""
        blocks = calibration.blocks if calibration is not None else []
        if score_blend and not blocks:  # calibration.cpp:65-68: calibrate() on an unfitted head
            raise SemrankError(ErrorCode.StateInvalid, "calibration head not fitted")
        lo = np.array([b.lo for b in blocks] or [0.0], np.float64)
        hi = np.array([b.hi for b in blocks] or [0.0], np.float64)
        val = np.array([b.value for b in blocks] or [0.0], np.float64)
        names = ["relevance"] + list(self.task_names[1:])
        tasks, ws = [], []
        for name, w in sorted((score_blend or {}).items()):
            if name not in names:
                raise SemrankError(ErrorCode.Alignment, f"blend references unknown task: {name}")
            tasks.append(names.index(name))
            ws.append(float(w))
        t = np.array(tasks or [0], np.int32)
        wv = np.array(ws or [0.0], np.float64)
        D = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        _check(_lib.sr_engine_set_postprocess(self._h, D(lo), D(hi), D(val), len(blocks),
                                              t.ctypes.data_as(C.POINTER(C.c_int32)), D(wv),
                                              len(tasks)))
        self._post = bool(blocks) or bool(tasks)

    def _final(self, n: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.float64)
        got = C.c_int32(0)
        _check(_lib.sr_engine_final_scores(self._h, out.ctypes.data_as(C.POINTER(C.c_double)),
                                           len(out), C.byref(got)))
        return out[:got.value]

    def score_batch(self, requests: Sequence[ScoreRequest], k: int = 0) -> List[ScoreResult]:
        prs = [_PackedRequest(r, self.config.d_model) for r in requests]
        rbs = [_ResultBuf(len(r.items), len(self.task_names), k) for r in requests]
        reqs = (_c.RequestC * len(prs))(*[p.c for p in prs])
        ress = (_c.ResultC * len(rbs))(*[r.c for r in rbs])
        _check(_lib.sr_engine_score_batch(self._h, reqs, len(prs), ress))
        out = []
        for r, rb, rc in zip(requests, rbs, ress):
            rb.c = rc
            out.append(self._to_result(r, rb))
        return out

    def plan(self, request: ScoreRequest, k: int = 0, item_ids=None) -> "Plan":
        return Plan(self, request, k, item_ids)

    def score_sharded(self, comm: "Comm", request: ScoreRequest, k: int,
                      item_ids: Optional[np.ndarray] = None) -> ScoreResult:
        """Score this rank's shard; top-k is merged across ranks (NCCL)."""
        pr = _PackedRequest(request, self.config.d_model, item_ids)
        rb = _ResultBuf(len(request.items), len(self.task_names), k)
        _check(_lib.sr_engine_score_sharded(self._h, comm._h, C.byref(pr.c), C.byref(rb.c)))
        return self._to_result(request, rb)

    @property
    def stream_ptr(self) -> int:
        return _lib.sr_engine_stream(self._h) or 0

    def item_hidden(self, request: ScoreRequest) -> np.ndarray:
        pr = _PackedRequest(request, self.config.d_model)
        out = np.zeros((len(request.items), self.config.d_model), np.float32)
        _check(_lib.sr_engine_item_hidden(self._h, C.byref(pr.c),
                                          out.ctypes.data_as(C.POINTER(C.c_float))))
        return out


PROF_CLASSES = ["embed_ln", "gemm_qkv", "attention", "gemm_o", "layernorm", "gemm_in",
                "gemm_out", "score_head", "topk"]


class Comm:
    """NCCL communicator for candidate-sharded scoring (one rank per GPU)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(_lib.sr_nccl_unique_id(buf))
        return bytes(buf)

    def __init__(self, nranks: int, rank: int, uid: bytes, device: int):
        buf = (C.c_uint8 * 128)(*uid)
        h = C.c_void_p()
        _check(_lib.sr_comm_create(nranks, rank, buf, device, C.byref(h)))
        self._h = h

    @classmethod
    def host(cls, nranks: int, rank: int, device: int, allgather) -> "Comm":
        """Top-k exchange over a caller transport (sr_comm_create_host):
        ``allgather(bytes) -> list of every rank's bytes in rank order`` (e.g.
        torch.distributed.all_gather_object under gloo)."""
        self = cls.__new__(cls)

        def fn(send, recv, nbytes, user):
            try:
                mine = C.string_at(send, nbytes)
                parts = allgather(mine)
                blob = b"".join(parts)
                if len(parts) != nranks or len(blob) != nbytes * nranks:
                    return 1
                C.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # reported as SR_NCCL by the library
                return 1

        self._fn = _c.ALLGATHER_FN(fn)  # kept alive with the communicator
        h = C.c_void_p()
        _check(_lib.sr_comm_create_host(nranks, rank, device, self._fn, None, C.byref(h)))
        self._h = h
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and not _sys.is_finalizing():  # process exit frees it
            _lib.sr_comm_destroy(h)
            self._h = C.c_void_p()


class Plan:
    """Resident request (packed inputs on the device + captured CUDA graph)."""

    def __init__(self, engine: "ScoringEngine", request: ScoreRequest, k: int = 0,
                 item_ids: Optional[np.ndarray] = None):
        self.engine = engine
        self.request = request
        self._pr = _PackedRequest(request, engine.config.d_model, item_ids)
        h = C.c_void_p()
        _check(_lib.sr_plan_create(engine._h, C.byref(self._pr.c), k, C.byref(h)))
        self._h = h
        self.k = k
        self._rb = _ResultBuf(len(request.items), len(engine.task_names), k)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and not _sys.is_finalizing():  # process exit frees it
            _lib.sr_plan_destroy(h)
            self._h = C.c_void_p()

    def run(self) -> None:
        _check(_lib.sr_plan_run(self._h))

    def run_sharded(self, comm: Comm) -> None:
        _check(_lib.sr_plan_run_sharded(self._h, comm._h))

    def sync(self) -> None:
        _check(_lib.sr_plan_sync(self._h))

    def fetch(self) -> ScoreResult:
        _check(_lib.sr_plan_fetch(self._h, C.byref(self._rb.c)))
        return self.engine._to_result(self.request, self._rb)

    def kernel_count(self) -> int:
        n = C.c_int32()
        _check(_lib.sr_plan_kernel_count(self._h, C.byref(n)))
        return n.value

    def shape(self) -> dict:
        o = np.zeros(8, np.int64)
        _check(_lib.sr_plan_shape(self._h, o.ctypes.data_as(C.POINTER(C.c_int64))))
        keys = ["rows", "items", "attn_tiles", "soft_rows", "h2d_bytes", "d2h_bytes", "k", "tasks"]
        return {k: int(v) for k, v in zip(keys, o)}

    def profile(self, reps: int = 3) -> dict:
        ms = np.zeros(len(PROF_CLASSES), np.float32)
        cnt = np.zeros(len(PROF_CLASSES), np.int32)
        _check(_lib.sr_plan_profile(self._h, reps, ms.ctypes.data_as(C.POINTER(C.c_float)),
                                    cnt.ctypes.data_as(C.POINTER(C.c_int32))))
        return {c: (float(m), int(n)) for c, m, n in zip(PROF_CLASSES, ms, cnt)}


class EmbPlan(Plan):
    """Resident compact-embedding request (sr_plan_create_emb)."""

    def __init__(self, engine: "ScoringEngine", prefix_tokens, embeddings, form, k: int = 0,
                 item_ids=None):
        self.engine = engine
        self._prefix = np.ascontiguousarray(np.asarray(prefix_tokens, np.int32).reshape(-1))
        self._emb = np.ascontiguousarray(embeddings, np.float32)
        n = self._emb.shape[0]
        self._ids = None if item_ids is None else np.ascontiguousarray(np.asarray(item_ids, np.int64))
        names = ([str(int(i)) for i in self._ids] if self._ids is not None
                 else [str(i) for i in range(n)])
        self.request = ScoreRequest(prefix_tokens=self._prefix, mode=ScoreMode.Mixed,
                                    items=[ScoreItem(id=x) for x in names])
        h = C.c_void_p()
        _check(_lib.sr_plan_create_emb(
            engine._h, self._prefix.ctypes.data_as(C.POINTER(C.c_int32)), len(self._prefix),
            self._emb.ctypes.data_as(C.POINTER(C.c_float)), self._emb.shape[1], n,
            self._ids.ctypes.data_as(C.POINTER(C.c_int64)) if self._ids is not None else None,
            ScoringEngine._emb_form(form), k, C.byref(h)))
        self._h = h
        self.k = k
        self._rb = _ResultBuf(n, len(engine.task_names), k)


class BatchPlan(Plan):
    """Several requests resident in one packed device pass (plan_batches
    consumer; BASELINE config C4 runs 32 queries per pass)."""

    def __init__(self, engine: "ScoringEngine", requests: Sequence[ScoreRequest], k: int = 0):
        self.engine = engine
        self.requests = list(requests)
        self.request = self.requests[0]
        self._prs = [_PackedRequest(r, engine.config.d_model) for r in self.requests]
        arr = (_c.RequestC * len(self._prs))(*[p.c for p in self._prs])
        h = C.c_void_p()
        _check(_lib.sr_plan_create_batch(engine._h, arr, len(self._prs), k, C.byref(h)))
        self._h = h
        self.k = k
        self._rbs = [_ResultBuf(len(r.items), len(engine.task_names), k) for r in self.requests]

    def fetch_all(self) -> List[ScoreResult]:
        ress = (_c.ResultC * len(self._rbs))(*[rb.c for rb in self._rbs])
        _check(_lib.sr_plan_fetch_batch(self._h, ress, len(self._rbs)))
        out = []
        for r, rb, rc in zip(self.requests, self._rbs, ress):
            rb.c = rc
            out.append(self.engine._to_result(r, rb))
        return out


class Scheduler:
    """Latency-bounded dynamic batching in front of one engine (SURVEY §8(f)
    row 1; include/semrank_b200.h sr_sched_*). ``submit`` deep-copies and
    queues a whole request and returns a ticket; the native dispatcher packs
    queued requests FIFO into device passes (plan_batches' greedy rule over
    whole requests, engine.cpp:278-326, under ``max_rows``; at most
    ``max_queries`` per pass; with ``budget_ms`` only while the oldest
    request's age plus the learned pass time fits the budget). ``wait``
    returns (ScoreResult, latency_ms, queries in its pass); latency is
    submit -> completion on the host clock. ``stats`` reports nearest-rank
    p50/p99 (service.cpp:28-34).

    ``executor`` (tests only) replaces the engine with a host function
    ``fn(requests: list[RequestC], results: list[ResultC]) -> None`` that fills
    the result buffers; ``config`` is then the model config to validate against."""

    def __init__(self, engine: Optional["ScoringEngine"] = None, *, max_queries: int = 8,
                 max_rows: int = 1 << 22, budget_ms: float = 0.0, max_wait_us: int = 0,
                 k: int = 10, borrow: bool = True, executor=None,
                 config: Optional[ModelConfig] = None, sat_rows: int = 0):
        self.engine = engine
        self.k = k
        self.config = engine.config if engine is not None else config
        self.task_names = [kRelevanceTask] + [h.name for h in self.config.head_specs]
        opt = _c.SchedOptionsC(max_queries, max_rows, float(budget_ms), max_wait_us, k,
                               int(bool(borrow)), int(sat_rows))
        self.borrow = bool(borrow)
        h = C.c_void_p()
        self._pending: Dict[int, tuple] = {}
        if executor is None:
            if engine is None:
                raise SemrankError(ErrorCode.SpecViolation, "scheduler needs an engine")
            _check(_lib.sr_sched_create(engine._h, C.byref(opt), C.byref(h)))
        else:
            def fn(reqs, n, ress, user):
                try:
                    executor([reqs[i] for i in range(n)], [ress[i] for i in range(n)])
                    return 0
                except SemrankError as e:
                    return int(e.code)
                except Exception:  # noqa: BLE001
                    return int(ErrorCode.StateInvalid)
            self._fn = _c.SCHED_EXEC_FN(fn)
            cfg = self._cfg_keep = self.config._to_c()
            _check(_lib.sr_sched_create_host(C.byref(cfg), C.byref(opt), self._fn, None,
                                             C.byref(h)))
        self._h = h

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and not _sys.is_finalizing():  # process exit frees it
            _lib.sr_sched_destroy(h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def pack(self, request: ScoreRequest) -> "_PackedRequest":
        """Flattened request for repeated submission (bench load generators)."""
        return _PackedRequest(request, self.config.d_model)

    def submit(self, request: ScoreRequest, packed: Optional["_PackedRequest"] = None) -> int:
        pr = packed if packed is not None else _PackedRequest(request, self.config.d_model)
        t = C.c_uint64(0)
        _check(_lib.sr_sched_submit(self._h, C.byref(pr.c), C.byref(t)))
        self._pending[t.value] = (request, pr)  # pr keeps borrowed arrays alive
        return t.value

    def wait(self, ticket: int):
        request, _pr = self._pending.pop(ticket)
        rb = _ResultBuf(len(request.items), len(self.task_names), self.k)
        lat, nb = C.c_double(0), C.c_int32(0)
        _check(_lib.sr_sched_wait(self._h, ticket, C.byref(rb.c), C.byref(lat), C.byref(nb)))
        if self.engine is not None:
            res = self.engine._to_result(request, rb)
        else:
            res = ScoreResult(request_id=request.request_id, mode=ScoreMode(request.mode),
                              scores=rb.scores[:len(request.items)].copy())
            res.topk = rb.topk(lambda i: request.items[i].id)
        return res, lat.value, nb.value

    def stats(self, reset: bool = False) -> dict:
        st = _c.SchedStatsC()
        _check(_lib.sr_sched_get_stats(self._h, int(reset), C.byref(st)))
        return {f: getattr(st, f) for f, _ in _c.SchedStatsC._fields_}


def score_by_mode(engine: ScoringEngine, request: ScoreRequest, k: int = 0) -> ScoreResult:
    """score_by_mode (engine.cpp:379-387): dispatch on request.mode."""
    return engine.score(request, k)


def tokenize(text: str, max_seq: int = 4096) -> List[int]:
    """Byte tokenizer (tokenizer.cpp:10-20)."""
    data = text.encode("utf-8")
    if len(data) > max_seq:
        raise SemrankError(ErrorCode.LengthOverflow,
                           f"text of {len(data)} bytes exceeds max_seq {max_seq}")
    return list(data)


@dataclass
class PromptParts:  # prompt.hpp:17-20
    prefix_tokens: List[int]
    item_tokens: List[int]


kPromptSuffix = "\nRelevant (Yes/No): "  # prompt.hpp:23


def _text_bytes(t) -> bytes:
    return t if isinstance(t, (bytes, bytearray)) else str(t).encode("utf-8")


def build_prompt(system, query_context, document, max_seq: int = 4096) -> PromptParts:
    """build_prompt (prompt.cpp:14-38) through the library (sr_build_prompt):
    prefix = system + query context, item = document + kPromptSuffix, byte
    tokens; LengthOverflow / SpecViolation as the reference."""
    s, q, d = _text_bytes(system), _text_bytes(query_context), _text_bytes(document)
    n_p, n_i = C.c_int32(0), C.c_int32(0)
    cap_p, cap_i = len(s) + len(q), len(d) + len(kPromptSuffix)
    pre = np.zeros(max(cap_p, 1), np.int32)
    item = np.zeros(max(cap_i, 1), np.int32)
    I = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    _check(_lib.sr_build_prompt(s, len(s), q, len(q), d, len(d), max_seq, I(pre), cap_p,
                                C.byref(n_p), I(item), cap_i, C.byref(n_i)))
    return PromptParts(pre[:n_p.value].tolist(), item[:n_i.value].tolist())


def score_result_to_json(result: "ScoreResult") -> str:
    """The /score response body (score_result_to_json, service.cpp:380-391),
    serialised by the library byte-identically to the reference's
    nlohmann::json dump()."""
    items = list(result.items)
    names = list(items[0].tasks.keys()) if items else []
    sc = np.ascontiguousarray([[it.tasks[n] for n in names] for it in items] or [[0.0]], np.float64)
    ids = (C.c_char_p * max(1, len(items)))(*[_text_bytes(it.item_id) for it in items])
    nm = (C.c_char_p * max(1, len(names)))(*[_text_bytes(n) for n in names])
    fl = _c.FlopReportC(result.flops.attention_units, result.flops.linear_units, result.flops.t_q,
                        result.flops.t_i_mean, result.flops.n_items)
    n = C.c_int64(0)
    rid = _text_bytes(result.request_id)
    args = (rid, len(items), ids, len(names), nm, sc.ctypes.data_as(C.POINTER(C.c_double)),
            C.byref(fl))
    _check(_lib.sr_score_result_to_json(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(_lib.sr_score_result_to_json(*args, buf, n.value, C.byref(n)))
    return buf.raw[:n.value].decode("utf-8")


def parse_score_request_json(body: str, d_model: int, max_seq: int = 4096) -> ScoreRequest:
    """The /score wire format (service.cpp:326-372); embedding_b64 items keep
    their base64 text, which ScoringEngine.score decodes on the device."""
    import json
    try:
        j = json.loads(body)
    except ValueError as e:
        raise SemrankError(ErrorCode.PayloadInvalid, f"request body is not JSON: {e}")
    req = ScoreRequest(request_id=j.get("request_id", ""))
    if "prefix_tokens" in j:
        req.prefix_tokens = [int(t) for t in j["prefix_tokens"]]
    elif "prefix_text" in j:
        req.prefix_tokens = tokenize(j["prefix_text"], max_seq)
    else:
        raise SemrankError(ErrorCode.PayloadInvalid, "request needs prefix_text or prefix_tokens")
    req.mode = score_mode_from_name(j.get("mode", "ibpc"))
    req.latency_sensitive = bool(j.get("latency_sensitive", False))
    items = j.get("items")
    if not isinstance(items, list) or not items:
        raise SemrankError(ErrorCode.PayloadInvalid, "request needs a non-empty items[]")
    for it in items:
        item = ScoreItem(id=it.get("id", ""))
        if "tokens" in it:
            item.tokens = [int(t) for t in it["tokens"]]
        elif "text" in it:
            item.tokens = tokenize(it["text"], max_seq)
        elif "embedding_b64" in it:
            item.embedding_b64 = it["embedding_b64"]
        else:
            raise SemrankError(ErrorCode.PayloadInvalid,
                               f"item needs text, tokens, or embedding_b64: {item.id}")
        req.items.append(item)
    return req


def topk_host(scores: np.ndarray, ids: Optional[np.ndarray], k: int):
    """Caller-side ordering (semrank_main.cpp:393-398) via the native comparator."""
    s = np.ascontiguousarray(scores, np.float64)
    n = len(s)
    kk = min(k, n)
    oi, os_, ox = np.zeros(max(kk, 1), np.int64), np.zeros(max(kk, 1)), np.zeros(max(kk, 1), np.int32)
    idp = None
    if ids is not None:
        ids = np.ascontiguousarray(ids, np.int64)
        idp = ids.ctypes.data_as(C.POINTER(C.c_int64))
    _check(_lib.sr_topk_host(s.ctypes.data_as(C.POINTER(C.c_double)), idp, n, k,
                             oi.ctypes.data_as(C.POINTER(C.c_int64)),
                             os_.ctypes.data_as(C.POINTER(C.c_double)),
                             ox.ctypes.data_as(C.POINTER(C.c_int32))))
    return oi[:kk], os_[:kk], ox[:kk]
