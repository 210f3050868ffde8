"""Scheduler parity (CPU): the product's restated global scheduler vs the
reference's own known answers and the compiled reference itself.

Known answers restate /root/reference/proj/tests/test_scheduler.cpp (cited
per test); random conformance restates acceptance criterion C8
(/root/reference/proj/tests/acceptance.cpp:422-515) and adds a live
comparison against oracle/_ref on every trial."""

import random

import pytest

import paper_2602_21548_b200 as dp
from oracle import refpy

needs_ref = pytest.mark.skipif(not refpy.ref_available(), reason="oracle/_ref not built")


def pe(i, tok, rq, seq=0):
    return [i, 0, seq, tok, rq, 0]


def de(i, tok, hbm, seq=0):
    return [i, 1, seq, tok, 0, hbm]


def fetch(q, snaps, alpha=1000, beta=5000, z=1.05):
    return dp.schedule_pe_fetch(q, snaps, alpha, beta, z)


def place(q, snaps, alpha=1000, beta=5000, z=1.05):
    return dp.schedule_de_within_group(q, snaps, alpha, beta, z)


def test_pe_fetch_argmin_in_c2():  # test_scheduler.cpp:81-89
    assert fetch([(42, 50)], [pe(0, 200, 0), pe(1, 100, 0)]) == [(42, 1, 2)]


def test_pe_fetch_reclassifies_into_c1():  # test_scheduler.cpp:91-101
    a = fetch([(1, 50), (2, 50)], [pe(0, 290, 0), pe(1, 100, 2000)], 1000, 300)
    assert [x[1] for x in a] == [0, 1] and a[1][2] == 3


def test_pe_fetch_c3_then_stop():  # test_scheduler.cpp:103-113
    a = fetch([(1, 200), (2, 200), (3, 200)], [pe(0, 10, 2000)], 1000, 300)
    assert a == [(1, 0, 3), (2, 0, 3)]


def test_beta_boundary_is_not_overloaded():  # test_scheduler.cpp:44-56 (tok == beta -> C2)
    a = fetch([(1, 1)], [pe(0, 6000, 500), pe(3, 5000, 500)])
    assert a == [(1, 3, 2)]


def test_de_groups_min_sum_ties_low_id():  # test_scheduler.cpp:139-153
    assert dp.schedule_de_groups([(7, 100)], [(0, 1000), (1, 500)]) == [(7, 1)]
    out = dp.schedule_de_groups([(1, 100), (2, 100), (3, 100)], [(0, 0), (1, 0)])
    assert [g for _, g in out] == [0, 1, 0]


def test_de_phase2_z_threshold_kat():  # test_scheduler.cpp:155-167 (Z = 3150)
    a = place([(1, 500), (2, 1500)], [de(0, 1000, 100000, 5), de(1, 3000, 100000, 1)])
    assert a[0] == (1, 0, 2) and a[1][1] == 0


def test_de_phase2_fallback_min_tok():  # test_scheduler.cpp:169-177 (Z = 6825)
    assert place([(1, 4000)], [de(0, 5000, 100000), de(1, 4000, 100000)]) == [(1, 1, 1)]


def test_de_phase2_hbm_stop():  # test_scheduler.cpp:179-188
    # Z = 1.05 * 500 / 2 = 262.5 < 500: the fit-only fallback (category 1) picks DE0
    assert place([(1, 500), (2, 500), (3, 100)], [de(0, 0, 600), de(1, 0, 300)]) == [(1, 0, 1)]


def test_read_path_tie_goes_to_pe():  # test_scheduler.cpp:190-194
    assert dp.select_read_path(100, 500) == 0
    assert dp.select_read_path(500, 100) == 1
    assert dp.select_read_path(100, 100) == 0


def independent_alg1(q, snaps, alpha, beta):
    """Algorithm 1 re-derived per assignment (acceptance.cpp:454-481)."""
    tok = [s[3] for s in snaps]
    out = []
    for rid, t in q:
        best2 = best3 = -1
        for e, s in enumerate(snaps):
            if tok[e] > beta:
                continue
            if s[4] <= alpha:
                if best2 < 0 or tok[e] < tok[best2]:
                    best2 = e
            elif best3 < 0 or tok[e] < tok[best3]:
                best3 = e
        want = best2 if best2 >= 0 else best3
        if want < 0:
            break
        out.append((rid, snaps[want][0], 2 if best2 >= 0 else 3))
        tok[want] += t
    return out


@needs_ref
def test_alg1_conformance_10000_snapshots():
    rng = random.Random(4242)
    for _ in range(10_000):
        alpha, beta = 1 + rng.randrange(4000), 1 + rng.randrange(10000)
        n = 1 + rng.randrange(10)
        snaps = [pe(i, rng.randrange(12000), rng.randrange(6000)) for i in range(n)]
        q = [(i, 1 + rng.randrange(900)) for i in range(rng.randrange(8))]
        mine = fetch(q, snaps, alpha, beta)
        assert mine == independent_alg1(q, snaps, alpha, beta)
        assert mine == refpy.ref_schedule("ref_schedule_pe_fetch", q, snaps, alpha, beta)


@needs_ref
def test_de_phase2_random_vs_reference():
    rng = random.Random(99)
    for _ in range(3000):
        n = 1 + rng.randrange(6)
        snaps = [de(10 + i, rng.randrange(20000), rng.randrange(30000), rng.randrange(9))
                 for i in range(n)]
        q = [(i, 1 + rng.randrange(6000)) for i in range(rng.randrange(10))]
        z = 1.0 + rng.random()
        assert place(q, snaps, 1000, 5000, z) == refpy.ref_schedule(
            "ref_schedule_de_within_group", q, snaps, 1000, 5000, z)


@needs_ref
def test_de_groups_random_vs_reference():
    rng = random.Random(7)
    for _ in range(2000):
        groups = [(g, rng.randrange(5000)) for g in range(1 + rng.randrange(5))]
        q = [(i, 1 + rng.randrange(3000)) for i in range(rng.randrange(12))]
        assert dp.schedule_de_groups(q, groups) == refpy.ref_schedule_de_groups(q, groups)


@needs_ref
def test_select_read_path_vs_reference():
    rng = random.Random(5)
    for _ in range(1000):
        a, b = rng.randrange(100), rng.randrange(100)
        assert dp.select_read_path(a, b) == refpy.ref().ref_select_read_path(a, b)


# ---- intra-engine compute-quota batching ----------------
# proj/src/scheduler.cpp:163-219; KATs from proj/tests/test_scheduler.cpp:196-285.

def fwd(queue, quota, cost):
    return dp.build_forward_batch(queue, quota, cost)


def test_attention_time_closed_forms():  # test_scheduler.cpp:196-208
    assert dp.estimate_attention_time([], (0, 0, 0, 0.5)) == pytest.approx(0.5)
    assert dp.estimate_attention_time([(0, 0, 8)], (0, 2.0, 0, 0)) == pytest.approx(128.0)
    assert dp.estimate_attention_time([(0, 100, 1)], (3.0, 0, 0, 0)) == pytest.approx(300.0)


def test_forward_batch_whole_queue():  # :210-221
    items, chunked, _, _, whole, t = fwd([(0, 0, 30), (1, 0, 40)], 100, (0, 0, 1.0, 0))
    assert len(items) == 2 and not chunked and whole == 2 and t == pytest.approx(70.0)


def test_forward_batch_quadratic_chunk():  # :223-234
    _, chunked, rid, bsz, whole, _ = fwd([(0, 0, 50)], 100.0, (0, 1.0, 0, 0))
    assert chunked and rid == 0 and bsz == 10 and whole == 0


def test_forward_batch_second_request_chunked():  # :236-247
    _, chunked, _, bsz, whole, t = fwd([(0, 0, 80), (1, 0, 50)], 100.0, (0, 0, 1.0, 0))
    assert chunked and whole == 1 and bsz == 20 and t == pytest.approx(100.0)


def test_forward_batch_quota_infeasible():  # :249-256
    with pytest.raises(dp.QuotaInfeasibleError):
        fwd([(0, 0, 10)], 0.5, (0, 0, 1.0, 0))


def test_forward_batch_binary_search_equals_linear_scan():  # :258-285
    rng = random.Random(5)
    cost = (1e-7, 3e-6, 2e-4, 1e-3)
    for _ in range(150):
        bsz = 1 + rng.randrange(4096)
        cached = rng.randrange(100000)
        quota = 1e-3 + rng.randrange(1000) * 5e-3
        best = 0
        for b in range(1, bsz + 1):
            if dp.estimate_attention_time([(0, cached, b)], cost) <= quota:
                best = b
            else:
                break  # monotone in b
        if best == 0:
            with pytest.raises(dp.QuotaInfeasibleError):
                fwd([(0, cached, bsz)], quota, cost)
            continue
        _, chunked, _, cb, _, t = fwd([(0, cached, bsz)], quota, cost)
        assert (cb if chunked else bsz) == best and t <= quota


@needs_ref
def test_forward_batch_random_queues_vs_reference():
    rng = random.Random(11)
    for trial in range(400):
        n = rng.randrange(0, 12)
        q = [(i, rng.randrange(0, 200000), 1 + rng.randrange(6000)) for i in range(n)]
        cost = (rng.choice([0, 2e-10, 1e-9]), rng.choice([0, 1e-9, 3e-8]),
                rng.choice([0, 4e-7, 1e-6]), rng.choice([0, 1e-5, 2e-4]))
        quota = rng.choice([2e-4, 2e-3, 2e-2, 0.3])
        try:
            want = refpy.ref_build_forward_batch(q, quota, cost)
        except refpy.QuotaInfeasible:
            with pytest.raises(dp.QuotaInfeasibleError):
                fwd(q, quota, cost)
            continue
        got = fwd(q, quota, cost)
        assert list(got[0]) == want[0], trial
        assert tuple(got[1:5]) == tuple(want[1:5]), trial
        assert got[5] == want[5], trial  # bit-identical double


def test_forward_batch_balances_ranks_criterion_6():
    # proj/tests/acceptance.cpp:333-381: 8 ranks each pack their own FIFO;
    # per-forward attention-time max/avg <= 1.10 in >= 90% of loaded forwards
    cost = (2e-10, 1e-9, 4e-7, 1e-5)
    quota, layers, ranks = 2e-3, 4, 8
    rng = random.Random(77)
    queues = [[] for _ in range(ranks)]
    nid = [0]

    def refill(r, k):
        for _ in range(k):
            queues[r].append([nid[0], int(rng.lognormvariate(8.5, 1.0)),
                              max(1, int(rng.lognormvariate(5.5, 0.9)))])
            nid[0] += 1

    for r in range(ranks):
        refill(r, 60)
    loaded = balanced = 0
    for _ in range(400):
        all_loaded = all(len(q) >= 4 for q in queues)
        times = []
        for r in range(ranks):
            if not queues[r]:
                refill(r, 10)
            _, chunked, _, cb, whole, t = fwd([tuple(x) for x in queues[r]], quota, cost)
            times.append(layers * t)
            del queues[r][:whole]
            if chunked:
                queues[r][0][2] -= cb
            refill(r, 2 + rng.randrange(2))
        if all_loaded:
            loaded += 1
            if max(times) / (sum(times) / len(times)) <= 1.10:
                balanced += 1
    assert loaded >= 100 and balanced / loaded >= 0.90
