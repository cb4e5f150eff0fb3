"""Serving scheduler policy on the CPU: the native
dispatcher (host/scheduler.cpp) driven through sr_sched_create_host with a
host stand-in for the device pass. Checks FIFO batching, the request cap, the
row budget (plan_batches' greedy rule over whole requests, engine.cpp:278-326),
the latency rule, max_wait, error isolation, submit-time validation with the
scoring error categories, and nearest-rank percentiles (service.cpp:28-34)."""
import math
import threading
import time

import numpy as np
import pytest

import paper_2602_07309_b200 as sr

CFG = sr.ModelConfig.default_toy()


def req(rid, n_items=3, t_q=5, t_i=4, base=0):
    r = sr.ScoreRequest(request_id=rid, prefix_tokens=[1 + (base % 200)] * t_q,
                        mode=sr.ScoreMode.MultiItem)
    for i in range(n_items):
        r.items.append(sr.ScoreItem(id=f"{rid}-{i}", tokens=[(base + i) % 250] * t_i))
    return r


class FakeDevice:
    """Scores item i of a request as its first token / 1000 (column 0); top-k
    by that score; records every pass's composition."""

    def __init__(self, delay=0.0, fail_on=None):
        self.delay = delay
        self.passes = []
        self.fail_on = fail_on
        self.lock = threading.Lock()

    def __call__(self, reqs, ress):
        with self.lock:
            self.passes.append([r.prefix_tokens[0] for r in reqs])
        if self.delay:
            time.sleep(self.delay)
        for r, res in zip(reqs, ress):
            if self.fail_on is not None and r.prefix_tokens[0] == self.fail_on:
                raise sr.SemrankError(sr.ErrorCode.PayloadInvalid, "boom")
        T = 1 + len(CFG.head_specs)
        for r, res in zip(reqs, ress):
            sc = [r.item_tokens[r.item_offsets[i]] / 1000.0 for i in range(r.n_items)]
            for i, v in enumerate(sc):
                for t in range(T):
                    res.scores[i * T + t] = v if t == 0 else 0.5
            order = sorted(range(r.n_items), key=lambda i: (-sc[i], i))[:res.k]
            for j, i in enumerate(order):
                res.topk_ids[j] = i
                res.topk_scores[j] = sc[i]
                res.topk_index[j] = i
            res.k_returned = len(order)


def test_results_reach_their_own_tickets():
    dev = FakeDevice()
    with sr.Scheduler(executor=dev, config=CFG, k=2) as s:
        reqs = [req(f"q{j}", n_items=2 + j % 3, base=10 * j) for j in range(12)]
        tickets = [s.submit(r) for r in reqs]
        for r, t in zip(reqs, tickets):
            res, lat, nb = s.wait(t)
            want = [((10 * int(r.request_id[1:]) + i) % 250) / 1000.0 for i in range(len(r.items))]
            assert np.allclose(res.scores[:, 0], want)
            assert res.topk[0][0] == r.items[int(np.argmax(want))].id
            assert lat >= 0 and 1 <= nb <= 8
        st = s.stats()
        assert st["completed"] == 12 and st["failed"] == 0 and st["submitted"] == 12
        assert st["p50_ms"] <= st["p99_ms"] <= st["max_ms"]


def test_fifo_batches_respect_cap_and_rows():
    dev = FakeDevice(delay=0.05)
    # 9 rows per request (t_q 5 + 1 item of 4): max_rows 20 -> at most 2 per pass
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=8, max_rows=20) as s:
        ts = [s.submit(req(f"q{j}", n_items=1, base=j)) for j in range(7)]
        for t in ts:
            s.wait(t)
    flat = [p for ps in dev.passes for p in ps]
    assert flat == [1 + j for j in range(7)]  # FIFO
    assert all(len(ps) <= 2 for ps in dev.passes)
    assert len(dev.passes) >= 4
    dev = FakeDevice(delay=0.05)
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=3) as s:
        ts = [s.submit(req(f"q{j}", n_items=1, base=j)) for j in range(10)]
        for t in ts:
            s.wait(t)
    assert max(len(ps) for ps in dev.passes) == 3  # the backlog fills passes to the cap
    # sat_rows: requests of at least that many rows run alone (13 rows: 2
    # items), smaller ones (9 rows: 1 item) still batch from the backlog
    dev = FakeDevice(delay=0.05)
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=8, sat_rows=13) as s:
        ts = [s.submit(req(f"q{j}", n_items=2 if j in (3, 4) else 1, base=j)) for j in range(10)]
        for t in ts:
            s.wait(t)
    assert [p for ps in dev.passes for p in ps] == [1 + j for j in range(10)]  # FIFO
    for ps in dev.passes:
        if 4 in ps or 5 in ps:  # the two 13-row requests (base 3, 4)
            assert len(ps) == 1
    assert max(len(ps) for ps in dev.passes) > 1
    # a request larger than the row budget still runs (alone)
    dev = FakeDevice()
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_rows=4) as s:
        ts = [s.submit(req(f"q{j}", n_items=2, base=j)) for j in range(3)]
        for t in ts:
            s.wait(t)
    assert all(len(ps) == 1 for ps in dev.passes)


def test_latency_rule_shrinks_passes():
    # each pass costs ~2 ms per request (1 ms per 9 rows ~ 0.11 ms/row + sleep)
    class Timed(FakeDevice):
        def __call__(self, reqs, ress):
            time.sleep(0.01 * len(reqs))
            super().__call__(reqs, ress)

    dev = Timed()
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=64, budget_ms=35.0) as s:
        s.wait(s.submit(req("warm", n_items=1)))  # learns ms_per_row
        ts = [s.submit(req(f"q{j}", n_items=1, base=j)) for j in range(20)]
        for t in ts:
            s.wait(t)
        st = s.stats()
    # est(rows) = 10 ms per request: a pass never plans past the 35 ms budget
    assert max(len(ps) for ps in dev.passes) <= 3
    assert st["ms_per_row"] > 0


def test_max_wait_collects_late_arrivals():
    dev = FakeDevice()
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=2, max_wait_us=300_000) as s:
        t0 = s.submit(req("a", n_items=1, base=1))
        time.sleep(0.05)
        t1 = s.submit(req("b", n_items=1, base=2))
        (_, _, n0), (_, _, n1) = s.wait(t0), s.wait(t1)
    assert n0 == n1 == 2 and dev.passes == [[2, 3]]
    dev = FakeDevice()
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=2, max_wait_us=20_000) as s:
        t0 = s.submit(req("a", n_items=1, base=1))
        _, lat, n = s.wait(t0)
    assert n == 1 and lat >= 19.0  # waited out max_wait, then ran alone


def test_failures_stay_in_their_pass_and_validation_at_submit():
    dev = FakeDevice(delay=0.02, fail_on=1 + 5)
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=1) as s:
        ts = [s.submit(req(f"q{j}", n_items=1, base=j)) for j in range(8)]
        for j, t in enumerate(ts):
            if j == 5:
                with pytest.raises(sr.SemrankError) as e:
                    s.wait(t)
                assert e.value.code == sr.ErrorCode.PayloadInvalid
            else:
                s.wait(t)
        assert s.stats()["failed"] == 1
        # the scoring error categories, raised by submit
        bad = req("bad", n_items=1)
        bad.items[0].tokens = [CFG.vocab_size]
        with pytest.raises(sr.SemrankError) as e:
            s.submit(bad)
        want = None
        try:
            sr.request_report(CFG, bad)
        except sr.SemrankError as e2:
            want = e2.code
        assert want is not None and e.value.code == want
        empty = sr.ScoreRequest(request_id="e", prefix_tokens=[1], mode=sr.ScoreMode.MultiItem)
        with pytest.raises(sr.SemrankError):
            s.submit(empty)
    with pytest.raises(sr.SemrankError) as e:
        sr.Scheduler(executor=dev, config=CFG, max_queries=0)
    assert e.value.code == sr.ErrorCode.Parameter


def test_concurrent_submitters_and_percentiles():
    dev = FakeDevice(delay=0.002)
    lats = {}
    with sr.Scheduler(executor=dev, config=CFG, k=1, max_queries=4) as s:
        def client(c):
            for j in range(10):
                r = req(f"c{c}_{j}", n_items=2, base=c * 20 + j)
                res, lat, _ = s.wait(s.submit(r))
                lats[r.request_id] = lat
                assert res.request_id == r.request_id
        th = [threading.Thread(target=client, args=(c,)) for c in range(4)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        st = s.stats(reset=True)
        assert s.stats()["completed"] == 0  # reset
    v = sorted(lats.values())
    assert st["completed"] == 40
    # nearest rank: sorted[ceil(q n) - 1]
    assert st["p99_ms"] == pytest.approx(v[math.ceil(0.99 * 40) - 1], rel=1e-9)
    assert st["p50_ms"] == pytest.approx(v[math.ceil(0.50 * 40) - 1], rel=1e-9)
