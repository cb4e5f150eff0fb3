"""Exhaustive retrieval scan on the B200 vs the
reference's exhaustive_topk (retrieval.cpp:134-173): golden vectors from the
reference itself and the pinned C restatement (oracle/) on larger corpora.

The bar is exact: identical doc ids in identical order and bit-identical
double scores (the device rescoring follows the reference's operation order;
the fp32 pre-pass only selects candidates, with a proven error margin)."""
import numpy as np
import pytest

import paper_2602_07309_b200 as sr
from oracle import oracle as O
from tests.retrieval_cases import golden_cases, random_corpus

pytestmark = pytest.mark.gpu


def dev_topk(emb, feat, ids, keep, q, w0, w, k):
    c = sr.DeviceCorpus(np.ascontiguousarray(emb, np.float32),
                        np.ascontiguousarray(feat, np.float32).reshape(len(emb), -1),
                        np.ascontiguousarray(ids, np.int64))
    return c.topk(q, w0, w, k, keep), c


def test_golden_cases_bit_identical(cuda):
    for c in golden_cases():
        (ids, sc), _ = dev_topk(c["emb"], c["feat"], c["ids"], c["keep"], c["query"], c["w0"],
                                c["w"], c["k"])
        assert np.array_equal(ids, c["ref_ids"]), (ids, c["ref_ids"])
        assert np.array_equal(sc, c["ref_scores"])


@pytest.mark.parametrize("n,d,f,k,filt,unit", [
    (3000, 16, 2, 17, False, True),      # test_retrieval.cpp:170-188 shape
    (200_000, 32, 1, 100, False, True),  # bench_kernels.cpp:130-164 shape
    (100_003, 48, 3, 64, True, False),   # ragged tail, D > 32 chunks, non-unit vectors
    (5000, 7, 0, 512, True, True),       # D % 4 != 0, no features, k = max
    (10, 4, 1, 50, False, True),         # k above the corpus size
    (20_000, 16, 1, 1500, True, True),   # 512 < k <= 2048: every doc rescored + multi-level select
    (9_000, 16, 1, 3000, True, False),   # k > 2048: every doc rescored + full device sort
    (300_000, 32, 1, 256, True, True),   # largest k of the 3-CTA x 1024-candidate scan
    (60_000, 32, 2, 400, False, False),  # 257..512: the 2-CTA x 2048-candidate scan
])
def test_random_corpora_match_oracle(cuda, n, d, f, k, filt, unit):
    emb, feat, ids, color = random_corpus(n + d, n, d, f, unit=unit)
    rng = np.random.default_rng(n)
    q = rng.standard_normal(d).astype(np.float32)
    w = list(rng.standard_normal(f) * 0.3)
    keep = (color != 2).astype(np.uint8) if filt else None
    (ids_d, sc_d), c = dev_topk(emb, feat, ids, keep, q, 0.9, w, k)
    ids_o, sc_o = O.oracle_topk(emb, feat, ids, keep, q, 0.9, w, k)
    assert np.array_equal(ids_d, ids_o)
    assert np.array_equal(sc_d, sc_o)
    assert c.last_candidates() < max(4 * k * 600, 10 * n)  # the fp32 pass pruned


def test_adversarial_increasing_scores_and_ties(cuda):
    """Scores rising along the scan order (every doc beats the running
    threshold: compactions every tile) and exact duplicates (ties broken by
    ascending doc id, test_retrieval.cpp:223-240)."""
    n, d = 60_000, 8
    t = np.linspace(0.0, 1.0, n, dtype=np.float32)
    emb = np.stack([t, 1 - t] + [np.full(n, 0.1, np.float32)] * (d - 2), 1).astype(np.float32)
    emb[::7] = emb[3]  # duplicated rows -> tied scores
    ids = np.arange(n, dtype=np.int64)[::-1].copy()
    q = np.zeros(d, np.float32)
    q[0] = 1.0
    (ids_d, sc_d), _ = dev_topk(emb, np.zeros((n, 0), np.float32), ids, None, q, 1.0, [], 300)
    ids_o, sc_o = O.oracle_topk(emb, np.zeros((n, 0), np.float32), ids, None, q, 1.0, [], 300)
    assert np.array_equal(ids_d, ids_o) and np.array_equal(sc_d, sc_o)


def test_all_equal_scores_take_the_exact_fallback(cuda):
    """Every doc within the fp32 margin of the threshold: the candidate buffer
    overflows and the scan rescores every doc in double."""
    n = 20_000
    emb = np.tile(np.array([[0.6, 0.8]], np.float32), (n, 1))
    ids = np.random.default_rng(1).permutation(n).astype(np.int64)
    (ids_d, sc_d), c = dev_topk(emb, np.zeros((n, 0), np.float32), ids, None,
                                np.array([1, 0], np.float32), 1.0, [], 25)
    assert list(ids_d) == list(range(25))
    assert c.last_candidates() == n
    ids_o, sc_o = O.oracle_topk(emb, np.zeros((n, 0), np.float32), ids, None,
                                np.array([1, 0], np.float32), 1.0, [], 25)
    assert np.array_equal(sc_d, sc_o)


def test_reference_error_rules(cuda):
    emb, feat, ids, _ = random_corpus(5, 100, 8, 2)
    c = sr.DeviceCorpus(emb, feat, ids)
    with pytest.raises(sr.SemrankError) as e:
        c.topk(emb[0], 1.0, [0.1, 0.2], 0)
    assert e.value.code == sr.ErrorCode.SpecViolation
    with pytest.raises(sr.SemrankError) as e:
        c.topk(emb[0], 1.0, [0.1], 5)
    assert e.value.code == sr.ErrorCode.Alignment
    with pytest.raises(sr.SemrankError) as e:
        c.topk(emb[0][:4], 1.0, [0.1, 0.2], 5)
    assert e.value.code == sr.ErrorCode.Alignment
    with pytest.raises(sr.SemrankError) as e:
        c.topk(np.zeros(8, np.float32), 1.0, [0.1, 0.2], 5)
    assert e.value.code == sr.ErrorCode.DegenerateInput
    bad = emb.copy()
    bad[40] = 0
    with pytest.raises(sr.SemrankError) as e:
        sr.DeviceCorpus(bad, feat, ids).topk(emb[0], 1.0, [0.1, 0.2], 5)
    assert e.value.code == sr.ErrorCode.DegenerateInput
    # no candidates: empty result, no checks (retrieval.cpp:166-172)
    ids_d, _ = c.topk(np.zeros(8, np.float32), 1.0, [0.1], 5, keep=np.zeros(100, np.uint8))
    assert len(ids_d) == 0


def test_python_api_filters_like_the_reference(cuda):
    """Corpus / QuerySpec / RARWeights / exhaustive_topk with string attribute
    filters (filter_candidates, retrieval.cpp:79-97)."""
    emb, feat, ids, color = random_corpus(9, 2000, 8, 2)
    names = ["red", "blue", "green"]
    docs = [sr.DocumentRecord(int(ids[i]), {"color": names[color[i]]}, emb[i], feat[i])
            for i in range(2000)]
    corpus = sr.Corpus(["ctr", "age"], docs)
    q = sr.QuerySpec(embedding=emb[3], filters={"color": ["red", "blue"]}, k=30)
    w = sr.RARWeights(1.0, [0.4, -0.3])
    got = sr.exhaustive_topk(corpus, q, w)
    ids_o, sc_o = O.oracle_topk(emb, feat, ids, (color < 2).astype(np.uint8), emb[3], 1.0,
                                [0.4, -0.3], 30)
    assert [r.doc_id for r in got] == list(ids_o)
    assert [r.score for r in got] == list(sc_o)
    with pytest.raises(sr.SemrankError) as e:
        sr.exhaustive_topk(corpus, sr.QuerySpec(embedding=emb[3], filters={"size": ["x"]}), w)
    assert e.value.code == sr.ErrorCode.SchemaUnknown
    # filter-then-score == score-then-filter (test_retrieval.cpp:190-221)
    full = sr.exhaustive_topk(corpus, sr.QuerySpec(embedding=emb[3], k=2000), w)
    keep_ids = {int(ids[i]) for i in range(2000) if color[i] < 2}
    assert [r.doc_id for r in full if r.doc_id in keep_ids][:30] == [r.doc_id for r in got]


def test_single_rank_sharded_path(cuda):
    emb, feat, ids, _ = random_corpus(11, 30_000, 32, 1)
    c = sr.DeviceCorpus(emb, feat, ids)
    uid = sr.Comm.unique_id()
    comm = sr.Comm(1, 0, uid, 0)
    a = c.topk(emb[7], 1.0, [0.25], 100)
    b = c.topk(emb[7], 1.0, [0.25], 100, comm=comm)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
