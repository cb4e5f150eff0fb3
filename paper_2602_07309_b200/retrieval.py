"""Python mirror of the reference retrieval API (include/semrank/retrieval.hpp)
on the B200 scan (C-ABI sr_corpus_*, kernels/retrieval.cu).

  reference                                     here
  DocumentRecord / Corpus (retrieval.hpp:16-33) DocumentRecord / Corpus
  QuerySpec, RARWeights, RankedDoc (:35-58)     same names
  filter_candidates (retrieval.cpp:79-97)       filter_candidates (host: string attributes)
  exhaustive_topk (retrieval.cpp:134-173)       exhaustive_topk (device scan, exact top-K)

Scores are the reference's doubles bit for bit (fp32 pre-pass + exact fp64
rescoring of the candidates); the order is (score desc, doc_id asc). There
is no host scoring path.
"""
from __future__ import annotations

import ctypes as C
import sys as _sys
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from ._capi import lib as _lib
from .semrank import Comm, ErrorCode, SemrankError, _check


@dataclass
class DocumentRecord:
    doc_id: int = 0
    attributes: Dict[str, str] = field(default_factory=dict)
    embedding: Sequence[float] = ()
    features: Sequence[float] = ()


@dataclass
class QuerySpec:
    query_id: int = 0
    text: str = ""
    embedding: Sequence[float] = ()
    filters: Dict[str, Sequence[str]] = field(default_factory=dict)
    k: int = 10


@dataclass
class RARWeights:  # S(q,d) = w0 * cos(e_q, e_d) + sum_i w_i f_i(d)
    w0: float = 1.0
    w: Sequence[float] = ()
    lambda_: float = 0.5


@dataclass
class RankedDoc:
    doc_id: int
    score: float


class Corpus:
    """Columnar corpus (embeddings [n x d], features [n x F], doc ids,
    per-doc attribute maps); uploaded to the device on first use."""

    def __init__(self, feature_names: Sequence[str] = (), docs: Sequence[DocumentRecord] = ()):
        self.feature_names = list(feature_names)
        self.docs = list(docs)
        self._arrays = None
        self._dev = {}

    @classmethod
    def from_arrays(cls, embeddings, features, doc_ids, attributes=None, feature_names=None):
        emb = np.ascontiguousarray(embeddings, dtype=np.float32)
        feat = np.ascontiguousarray(features, dtype=np.float32).reshape(emb.shape[0], -1)
        c = cls(feature_names if feature_names is not None
                else [f"f{i}" for i in range(feat.shape[1])])
        c._arrays = (emb, feat, np.ascontiguousarray(doc_ids, dtype=np.int64),
                     list(attributes) if attributes is not None else None)
        return c

    def arrays(self):
        if self._arrays is None:
            n = len(self.docs)
            d = len(self.docs[0].embedding) if n else 0
            F = len(self.feature_names)
            emb = np.zeros((n, d), np.float32)
            feat = np.zeros((n, F), np.float32)
            for i, doc in enumerate(self.docs):
                if len(doc.embedding) != d or len(doc.features) != F:
                    raise SemrankError(ErrorCode.Alignment,
                                       f"doc {doc.doc_id} does not match the corpus layout")
                emb[i] = doc.embedding
                feat[i] = doc.features
            ids = np.array([doc.doc_id for doc in self.docs], np.int64)
            self._arrays = (emb, feat, ids, [dict(doc.attributes) for doc in self.docs])
        return self._arrays

    def __len__(self):
        return self.arrays()[0].shape[0]

    def has_attribute(self, name: str) -> bool:  # retrieval.cpp:36-41
        attrs = self.arrays()[3]
        return attrs is not None and any(name in a for a in attrs)

    def device(self, device: int = 0) -> "DeviceCorpus":
        if device not in self._dev:
            emb, feat, ids, _ = self.arrays()
            self._dev[device] = DeviceCorpus(emb, feat, ids, device)
        return self._dev[device]


class DeviceCorpus:
    """sr_corpus: the corpus resident in one device's HBM."""

    def __init__(self, emb: np.ndarray, feat: np.ndarray, ids: np.ndarray, device: int = 0):
        self._emb, self._feat, self._ids = emb, feat, ids  # keep alive for the upload
        h = C.c_void_p()
        _check(_lib.sr_corpus_create(emb.ctypes.data, feat.ctypes.data if feat.size else None,
                                     ids.ctypes.data, emb.shape[0], emb.shape[1] if emb.ndim > 1 else 0,
                                     feat.shape[1], device, C.byref(h)))
        self._h = h
        self.n, self.d, self.f = emb.shape[0], emb.shape[1], feat.shape[1]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and not _sys.is_finalizing():  # process exit frees it
            _lib.sr_corpus_destroy(self._h)
            self._h = None

    def topk(self, query, w0: float, w, k: int, keep: Optional[np.ndarray] = None,
             comm: Optional[Comm] = None):
        q = np.ascontiguousarray(query, dtype=np.float32)
        wv = np.ascontiguousarray(w, dtype=np.float64)
        kp = None if keep is None else np.ascontiguousarray(keep, dtype=np.uint8)
        kk = max(int(k), 1)
        ids = np.zeros(kk, np.int64)
        sc = np.zeros(kk, np.float64)
        n = C.c_int32(0)
        args = (q.ctypes.data, q.shape[0], float(w0), wv.ctypes.data if wv.size else None,
                wv.shape[0], kp.ctypes.data if kp is not None else None, int(k),
                ids.ctypes.data_as(C.POINTER(C.c_int64)), sc.ctypes.data_as(C.POINTER(C.c_double)),
                C.byref(n))
        if comm is not None:
            _check(_lib.sr_corpus_topk_sharded(self._h, comm._h, *args))
        else:
            _check(_lib.sr_corpus_topk(self._h, *args))
        return ids[:n.value], sc[:n.value]

    def last_candidates(self) -> int:
        return int(_lib.sr_corpus_last_candidates(self._h))

    def last_scan_ms(self) -> float:
        """Device time of the last call's fp32 scan kernel (CUDA events)."""
        return float(_lib.sr_corpus_last_scan_ms(self._h))


def filter_candidates(corpus: Corpus, filters: Dict[str, Sequence[str]]) -> np.ndarray:
    """Boolean keep mask of docs satisfying every predicate (retrieval.cpp:79-97);
    an attribute no doc carries raises SchemaUnknown."""
    for attr in filters:
        if not corpus.has_attribute(attr):
            raise SemrankError(ErrorCode.SchemaUnknown, f"unknown attribute: {attr}")
    attrs = corpus.arrays()[3]
    n = len(corpus)
    keep = np.ones(n, np.uint8)
    if not filters:
        return keep
    for i in range(n):
        a = attrs[i]
        for attr, values in filters.items():
            v = a.get(attr)
            if v is None or v not in values:
                keep[i] = 0
                break
    return keep


def exhaustive_topk(corpus: Corpus, query: QuerySpec, weights: RARWeights,
                    device: int = 0, comm: Optional[Comm] = None) -> List[RankedDoc]:
    """Exact top-K by score (descending, doc_id ascending on ties) over the
    filtered candidates (retrieval.hpp:60-70)."""
    if query.k < 1:
        raise SemrankError(ErrorCode.SpecViolation, "top-K requires K >= 1")
    keep = filter_candidates(corpus, query.filters) if query.filters else None
    ids, sc = corpus.device(device).topk(query.embedding, weights.w0, weights.w, query.k, keep, comm)
    return [RankedDoc(int(i), float(s)) for i, s in zip(ids, sc)]
