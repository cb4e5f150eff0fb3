"""Multi-process (world_size 2, gloo on CPU) coverage of the candidate-sharded
path's host logic: contiguous shards with global ids, per-rank top-k with the
reference comparator, all-gather, merge. The merged list must equal the
single-process top-k exactly — the reference's own shard-merge invariant
(retrieval.cpp:144-165). On the GPU box the all-gather is one
ncclAllGather of TopkEntry structs and the merge is the same comparator on
the device (kernels/head_topk.cu topk_entries_kernel)."""
import json
import os
import socket

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard(n, world, rank):
    per = (n + world - 1) // world
    return rank * per, min(n, (rank + 1) * per)


def _worker(rank, world, port, scores, ids, k, out_path):
    import torch.distributed as dist

    import paper_2602_07309_b200 as sr
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    lo, hi = shard(len(scores), world, rank)
    li, ls, _ = sr.topk_host(scores[lo:hi], ids[lo:hi], k)
    gathered = [None] * world
    dist.all_gather_object(gathered, (list(map(int, li)), list(map(float, ls))))
    all_ids = np.array([i for g in gathered for i in g[0]], np.int64)
    all_sc = np.array([s for g in gathered for s in g[1]])
    mi, ms, _ = sr.topk_host(all_sc, all_ids, k)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump({"ids": list(map(int, mi)), "scores": list(map(float, ms))}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k,ties", [(10, False), (64, False), (7, True)])
def test_two_rank_topk_merge_equals_single(tmp_path, k, ties):
    import torch.multiprocessing as mp

    import paper_2602_07309_b200 as sr
    with open(os.path.join(GOLD, "toy_bench.json")) as f:
        g = json.load(f)
    scores = np.asarray(g["modes"]["multi_item"]["scores"])[:, 0]
    if ties:
        scores = np.round(scores, 2)  # exact ties: the doc-id rule decides
    ids = np.random.default_rng(1).permutation(10_000)[:len(scores)].astype(np.int64)
    out = str(tmp_path / "merged.json")
    mp.spawn(_worker, args=(2, _free_port(), scores, ids, k, out), nprocs=2, join=True)
    with open(out) as f:
        merged = json.load(f)
    want_ids, want_sc, _ = sr.topk_host(scores, ids, k)
    assert merged["ids"] == list(map(int, want_ids))
    assert merged["scores"] == list(map(float, want_sc))


def test_shards_cover_all_candidates_once():
    for n in (1, 7, 256, 8192, 8193):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard(n, world, r)
                seen += list(range(lo, hi))
            assert seen == list(range(n))


def _retrieval_worker(rank, world, port, seed, n, d, k, out_path):
    """Corpus shard per rank (contiguous, global doc ids), the shard's exact
    top-k by the C restatement of exhaustive_topk, all-gather, comparator
    merge (retrieval.cpp:144-165) — the host half of sr_corpus_topk_sharded."""
    import torch.distributed as dist

    from oracle import oracle as O
    from tests.retrieval_cases import random_corpus
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    emb, feat, ids, color = random_corpus(seed, n, d, 1)
    keep = (color != 1).astype(np.uint8)
    q = emb[11]
    lo, hi = shard(n, world, rank)
    li, ls = O.oracle_topk(emb[lo:hi], feat[lo:hi], ids[lo:hi], keep[lo:hi], q, 1.0, [0.25], k)
    gathered = [None] * world
    dist.all_gather_object(gathered, (list(map(int, li)), list(map(float, ls))))
    pool = sorted(((s, i) for g in gathered for i, s in zip(*g)), key=lambda e: (-e[0], e[1]))
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump({"ids": [i for _, i in pool[:k]], "scores": [s for s, _ in pool[:k]]}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 100), (2, 1), (2, 5000)])
def test_two_rank_retrieval_merge_equals_single(tmp_path, world, k):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from tests.retrieval_cases import random_corpus
    n, d, seed = 20_011, 16, 5
    out = str(tmp_path / "merged.json")
    mp.spawn(_retrieval_worker, args=(world, _free_port(), seed, n, d, k, out), nprocs=world,
             join=True)
    with open(out) as f:
        merged = json.load(f)
    emb, feat, ids, color = random_corpus(seed, n, d, 1)
    want_ids, want_sc = O.oracle_topk(emb, feat, ids, (color != 1).astype(np.uint8), emb[11], 1.0,
                                      [0.25], k)
    assert merged["ids"] == list(map(int, want_ids))
    assert merged["scores"] == list(map(float, want_sc))
