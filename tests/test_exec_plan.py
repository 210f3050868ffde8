"""Executor plan invariants (CPU): the decisions -> block tables / slots /
hazards translation that every engine derives identically."""

import pytest

import paper_2602_21548_b200 as dp

SB = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)


def cluster(P, D, L=8, b=576, T=64, cap=6.25e9):
    c = dp.ClusterConfig()
    c.prefill_nodes, c.decode_nodes, c.engines_per_node = P, D, 1
    c.n_layer, c.kv_bytes_per_token_per_layer, c.block_size_tokens = L, b, T
    c.cnic_bandwidth, c.storage_multiple, c.dram_bandwidth = 50e9, cap / 50e9, 500e9
    c.hbm_capacity_tokens, c.pe_buffer_bytes, c.de_buffer_bytes = 100_000_000, 1 << 42, 1 << 42
    return c


def build(P, D, policy="dual_path", pool_slots=0, count=10, turns=6, seed=8):
    cfg = cluster(P, D)
    trajs = dp.synthesize(max_len=20000, count=count, seed=seed, mean_turns=turns, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy=policy, **SB)
    opt = dp.ExecOptions()
    opt.pool_slots = pool_slots
    return cfg, trajs, planned, dp.build_exec_plan(cfg, trajs, planned, opt)


def replay(xp, planned):
    """Re-derive live slots in virtual time and check no two live jobs share one."""
    reqs = {r[0]: r for r in planned["requests"]}
    jobs = xp.jobs()
    evs = []
    for j in jobs:
        r = reqs[j[0]]
        evs.append((r[12], 1, j[0], j))
        if r[13] >= 0:
            evs.append((r[13], 0, j[0], j))
    evs.sort(key=lambda e: (e[0], e[1], e[2]))
    live = {}
    for t, kind, req, j in evs:
        for s in j[9]:
            key = (j[4], s)
            if kind == 1:
                assert key not in live, f"slot {key} double-booked"
                live[key] = req
            else:
                assert live.pop(key) == req


@pytest.mark.parametrize("P,D", [(1, 1), (2, 2), (1, 3), (3, 1)])
def test_decisions_become_jobs(P, D):
    cfg, trajs, planned, xp = build(P, D)
    dec = {d[1]: d for d in planned["decisions"]}
    jobs = xp.jobs()
    hit = 0
    for req, traj, rnd, reader, pe, de_path, cached, nblk, ticket, slots, fbs, preds, fence, *_ in jobs:
        d = dec[req]
        assert pe == d[2] and de_path == (d[4] == 1)
        assert reader == (d[3] if de_path else d[2])
        assert cached == dp.context_before(trajs[traj], rnd) > 0
        assert nblk == dp.blocks_for(cached, cfg) == len(slots) == len(fbs)
        assert all(0 <= f < xp.store_fb for f in fbs)
        assert fbs == [xp.fb_of(traj, k) for k in range(nblk)]
        hit += cached * cfg.kv_bytes_per_token()
    assert hit == xp.hit_bytes == sum(xp.reader_bytes)
    # every request with cached KV has exactly one job
    want = sorted(r[0] for r in planned["requests"] if r[3] > 0)
    assert sorted(j[0] for j in jobs) == want
    # tickets are dense per PE
    for pe in range(xp.n_pe):
        t = sorted(j[8] for j in jobs if j[4] == pe)
        assert t == list(range(len(t))) and len(t) == xp.n_tickets[pe]
    replay(xp, planned)


def test_pe_only_reads_only_on_prefill_engines():
    cfg, trajs, planned, xp = build(2, 2, policy="pe_only")
    assert xp.reader_bytes[2] == xp.reader_bytes[3] == 0
    assert all(not j[5] for j in xp.jobs())


def test_tight_pool_records_hazards():
    _, _, planned, probe = build(1, 1, count=12)
    _, _, planned, xp = build(1, 1, count=12, pool_slots=probe.peak_slots)
    jobs = xp.jobs()
    by_ticket = {j[8]: j for j in jobs}
    last_writer = {}
    for j in jobs:  # global (allocation) order
        preds, fence = set(), False
        for s in j[9]:
            if s in last_writer:
                w = last_writer[s]
                if w[3] == j[3]:
                    fence = True
                else:
                    preds.add(w[8])
            last_writer[s] = j
        assert set(j[11]) == preds and j[12] == fence
        for t in j[11]:
            assert by_ticket[t][3] != j[3]
    assert any(j[11] for j in jobs) and any(j[12] for j in jobs)
    replay(xp, planned)


def test_pool_below_peak_is_rejected():
    _, _, planned, probe = build(1, 1)
    with pytest.raises(ValueError, match="peak"):
        build(1, 1, pool_slots=max(1, probe.peak_slots - 1))


def test_store_mapping_and_size_cap():
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=20000, count=6, seed=1, mean_turns=4, sigma_turns=0)
    planned = dp.plan(cfg, trajs, **SB)
    opt = dp.ExecOptions()
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert xp.store_fb == xp.fb_stride * len(trajs)  # no aliasing when it fits
    opt.store_bytes_max = 3 * cfg.full_block_bytes()
    xp2 = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert xp2.store_fb == 3
    assert all(0 <= f < 3 for j in xp2.jobs() for f in j[10])


def build_handoff(P, D, policy="dual_path", tight=False, count=10, turns=6, seed=8):
    cfg = cluster(P, D)
    trajs = dp.synthesize(max_len=20000, count=count, seed=seed, mean_turns=turns, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy=policy, **SB)
    opt = dp.ExecOptions()
    opt.handoff = True
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots, opt.de_pool_slots = xp.peak_slots, xp.de_peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    return cfg, trajs, planned, xp


@pytest.mark.parametrize("P,D,tight", [(1, 1, False), (2, 2, False), (1, 1, True), (1, 3, True)])
def test_handoff_plan_invariants(P, D, tight):
    cfg, trajs, planned, xp = build_handoff(P, D, tight=tight)
    T = cfg.block_size_tokens
    reqs = {r[0]: r for r in planned["requests"]}
    jobs = xp.jobs()
    # every request that reached prefill has a job, cold ones included
    assert sorted(j[0] for j in jobs) == sorted(r[0] for r in planned["requests"] if r[6] >= 0)
    ho = 0
    for j in jobs:
        r = reqs[j[0]]
        cached, prompt = r[3], r[3] + r[4]
        assert j[6] == cached and j[14] == prompt and j[13] == r[7]
        assert j[15] == -(-prompt // T) == len(j[17]) == len(j[18])
        assert j[17][:j[7]] == j[9]  # the hit blocks are the first prompt blocks
        ho += (prompt - cached if j[5] else prompt) * cfg.kv_bytes_per_token()
    assert ho == xp.handoff_bytes
    pos = {j[0]: i for i, j in enumerate(jobs)}
    # live-slot exclusivity: PE slots [t_read_done, t_pe_release), DE slots [t_read_done, t_done)
    for which, free_col, slot_col, key_col in (("pe", 13, 17, 4), ("de", 14, 18, 13)):
        evs = []
        for j in jobs:
            r = reqs[j[0]]
            evs.append((r[12], 1, j[0], j))
            if r[free_col] >= 0:
                evs.append((r[free_col], 0, j[0], j))
        evs.sort(key=lambda e: (e[0], e[1], e[2]))
        live, last = {}, {}
        for t, kind, req, j in evs:
            for s in j[slot_col]:
                key = (j[key_col], s)
                if kind == 1:
                    assert key not in live, f"{which} slot {key} double-booked"
                    live[key] = req
                    if which == "de" and key in last:  # predecessor recorded, and earlier
                        prev = last[key]
                        assert prev[16] in j[19] and pos[prev[0]] < pos[j[0]]
                    last[key] = j
                else:
                    assert live.pop(key) == req
    # decode tickets dense per DE
    for d in range(xp.n_pe, xp.n_engines):
        t = sorted(j[16] for j in jobs if j[13] == d)
        assert t == list(range(len(t))) and len(t) == xp.n_de_tickets[d]
    if tight:
        assert any(j[19] for j in jobs)  # decode-slot reuse hazards exercised


def test_persist_chunks_match_the_reference_ledger():
    """PersistD2H ledger (proj/tests/test_desim.cpp:168-188): the executor's
    persist chunks equal, request by request, the planner's PersistD2H flows
    (bit-identical to the reference's)."""
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=20000, count=8, seed=3, mean_turns=5, sigma_turns=0)
    planned = dp.plan(cfg, trajs, flows=True, **SB)
    opt = dp.ExecOptions()
    opt.handoff = True
    opt.persist = True
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    per_tok = cfg.kv_bytes_per_token()
    flows = {}
    for req, stage, nbytes, t0, t1 in planned["flows"]:
        if stage == 8:  # PersistD2H
            flows.setdefault(req, []).append(nbytes)
    total = 0
    for i, j in enumerate(xp.jobs()):
        chunks = xp.persist_chunks(i)
        # flows are logged at completion, so concurrent chunks may finish out of order
        assert sorted((b - a) * per_tok for a, b in chunks) == sorted(flows[j[0]])
        assert chunks[0][0] == j[14] and chunks[-1][1] == j[14] + xp.job_gen(i)
        total += xp.job_gen(i) * per_tok
    assert total == xp.persist_bytes
    # the KATs of test_desim.cpp:168-188: gen 130 -> 64, 64, 2; gen 64 -> one block
    t = dp.Trajectory()
    t.id = "t"
    t.rounds = [dp.Round(32, 130)]
    u = dp.Trajectory()
    u.id = "u"
    u.rounds = [dp.Round(32, 64)]
    planned = dp.plan(cfg, [t, u], **SB)
    xp = dp.build_exec_plan(cfg, [t, u], planned, opt)
    sizes = sorted([b - a for a, b in xp.persist_chunks(i)] for i in range(2))
    assert sizes == [[64], [64, 64, 2]]


def test_persist_requires_handoff():
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=8000, count=2, seed=3, mean_turns=2, sigma_turns=0)
    planned = dp.plan(cfg, trajs, **SB)
    opt = dp.ExecOptions()
    opt.persist = True
    with pytest.raises(ValueError, match="handoff"):
        dp.build_exec_plan(cfg, trajs, planned, opt)


# ---- prefill forwards -----------------------------------
COST = (2e-10, 1e-9, 4e-7, 1e-5)


def build_prefill(P, D, quota=2e-3, tight=False, count=10, turns=6, seed=8, cost=COST):
    cfg = cluster(P, D)
    trajs = dp.synthesize(max_len=20000, count=count, seed=seed, mean_turns=turns, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.prefill = True
    opt.compute_quota = quota
    opt.prefill_cost = cost
    xp0 = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots = xp0.peak_slots
        xp0 = dp.build_exec_plan(cfg, trajs, planned, opt)
    return cfg, trajs, planned, xp0


@pytest.mark.parametrize("P,D,tight,quota", [(1, 1, False, 2e-3), (2, 2, True, 2e-3), (1, 3, True, 5e-4),
                                             (2, 2, False, 0.3)])
def test_prefill_forwards_cover_every_prompt(P, D, tight, quota):
    cfg, trajs, planned, xp = build_prefill(P, D, quota=quota, tight=tight)
    assert xp.prefill
    reqs = {r[0]: r for r in planned["requests"]}
    jobs = xp.jobs()
    job_of = {j[0]: i for i, j in enumerate(jobs)}
    for pe in range(xp.n_pe):
        rows = xp.fwd_rows(pe)
        # FIFO = the PE's requests in landing order (t_read_done, id)
        want = sorted((r for r in planned["requests"] if r[6] == pe and r[12] >= 0),
                      key=lambda r: (r[12], r[0]))
        assert rows == [r[0] for r in want]
        done = {rid: 0 for rid in rows}
        fwds = xp.forwards(pe)
        for fi, (est, items) in enumerate(fwds):
            assert items, "empty forward"
            rws = [it[5] for it in items]
            assert rws == list(range(rws[0], rws[0] + len(rws))), "a forward is a FIFO range"
            for req, job, cached, q0, bsz, row in items:
                r = reqs[req]
                assert rows[row] == req and cached == r[3]
                assert q0 == done[req], "chunks run in order, without gaps"
                done[req] += bsz
                assert job == job_of.get(req, -1)
            assert est <= quota or len(items) == 1
            # the estimate is the cost model of exactly these chunks
            assert est == dp.estimate_attention_time([(it[0], it[2], it[4]) for it in items], COST)
        for rid in rows:
            assert done[rid] == reqs[rid][4], "every append token runs exactly once"


@pytest.mark.parametrize("P,D", [(1, 1), (2, 2), (1, 3)])
def test_prefill_slot_reuse_waits_for_the_reader_forward(P, D):
    cfg, trajs, planned, xp = build_prefill(P, D, tight=True, count=12, turns=8)
    jobs = xp.jobs()
    first_fwd = {}
    for pe in range(xp.n_pe):
        for fi, (_, items) in enumerate(xp.forwards(pe)):
            for it in items:
                if it[1] >= 0:
                    first_fwd.setdefault(it[1], fi)
                    assert xp.last_fwd(it[1]) >= fi
    n_waits = 0
    for i, j in enumerate(jobs):
        for w in xp.consumer_waits(i):
            n_waits += 1
            assert w < i and jobs[w][4] == j[4]
            # the forward that reads w last runs before this job is first read
            assert xp.last_fwd(w) < first_fwd[i]
        # prefill mode replaces the same-reader fence; DE loads wait on the
        # PE's consumed rows (ticket + n_tickets, target 1)
        assert not j[12]
        if j[3] != j[4]:
            assert j[11] == [jobs[w][8] + xp.n_tickets[j[4]] for w in xp.consumer_waits(i)]
    assert n_waits > 0, "the tight pool should force slot reuse"


@pytest.mark.skipif(not __import__("oracle.refpy", fromlist=["x"]).ref_available(),
                    reason="oracle/_ref not built")
def test_prefill_forwards_are_reference_build_forward_batch():
    """Each forward is the reference's build_forward_batch over the FIFO
    window that starts at the head chunk and stops before the first request
    reusing a slot of a request in the window (restated here)."""
    from oracle import refpy
    cfg, trajs, planned, xp = build_prefill(2, 2, tight=True, count=12, turns=8, quota=1e-3)
    reqs = {r[0]: r for r in planned["requests"]}
    jobs = xp.jobs()
    for pe in range(xp.n_pe):
        rows = xp.fwd_rows(pe)
        job_of_row = {}
        for _, items in xp.forwards(pe):
            for it in items:
                job_of_row[it[5]] = it[1]
        row_of_job = {j: r for r, j in job_of_row.items() if j >= 0}
        pred_row = [max([row_of_job[w] for w in xp.consumer_waits(job_of_row[r])], default=-1)
                    if job_of_row.get(r, -1) >= 0 else -1 for r in range(len(rows))]
        head, done = 0, 0
        for est, items in xp.forwards(pe):
            assert items[0][5] == head and items[0][3] == done
            barrier = head + 1
            while barrier < len(rows) and pred_row[barrier] < head:
                barrier += 1
            window = [(rows[i], reqs[rows[i]][3], reqs[rows[i]][4] - (done if i == head else 0))
                      for i in range(head, barrier)]
            got_items, chunked, _, cb, whole, t = refpy.ref_build_forward_batch(window, 1e-3, COST)
            assert [(it[0], it[2], it[4]) for it in items] == got_items
            assert est == t
            if chunked:
                done = done + cb if whole == 0 else cb
            else:
                done = 0
            head += whole
        assert head == len(rows)


def test_prefill_rejects_bad_quota():
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=20000, count=4, seed=8, mean_turns=4, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.prefill, opt.compute_quota = True, 0.0
    with pytest.raises(ValueError):
        dp.build_exec_plan(cfg, trajs, planned, opt)


@pytest.mark.parametrize("P,D,tight", [(1, 1, True), (2, 2, True), (1, 3, False)])
def test_prefill_with_handoff_keeps_k3_after_forwards(P, D, tight):
    """Handoff + prefill: K3 of a request runs after its last forward, so a
    load that waits for an earlier request's K3 (PE slot reuse) must not share
    a forward with it; every request of the PE is prefilled exactly once."""
    cfg = cluster(P, D)
    trajs = dp.synthesize(max_len=20000, count=10, seed=8, mean_turns=6, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.handoff, opt.prefill, opt.compute_quota, opt.prefill_cost = True, True, 2e-3, COST
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots = xp.peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    jobs = xp.jobs()
    reqs = {r[0]: r for r in planned["requests"]}
    n_waits = 0
    for pe in range(xp.n_pe):
        first = {}
        done = {}
        for fi, (_, items) in enumerate(xp.forwards(pe)):
            for req, job, cached, q0, bsz, row in items:
                assert job >= 0, "with the handoff every prefilled request has a job"
                first.setdefault(job, fi)
                assert q0 == done.get(req, 0)
                done[req] = q0 + bsz
        for rid, n in done.items():
            assert n == reqs[rid][4]
        for i in xp.by_pe(pe):
            for w in xp.consumer_waits(i):
                n_waits += 1
                assert xp.last_fwd(w) < first[i]
            # the k3_waits / pe_done_preds hazards are all covered
            assert set(jobs[i][20]) <= set(xp.consumer_waits(i))
    if tight:
        assert n_waits > 0


def test_prefill_quota_infeasible_propagates():
    # a quota below a 1-token chunk of some request: the reference's
    # QuotaInfeasibleError (scheduler.cpp:203-206) reaches the caller
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=20000, count=4, seed=8, mean_turns=4, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.prefill, opt.compute_quota, opt.prefill_cost = True, 1e-6, (1e-9, 0.0, 0.0, 1e-5)
    with pytest.raises(dp.QuotaInfeasibleError):
        dp.build_exec_plan(cfg, trajs, planned, opt)


@pytest.mark.parametrize("P,D,persist,cap", [(2, 2, True, 6.25e9), (2, 2, False, 6.25e9), (1, 3, True, 0),
                                             (3, 1, True, 6.25e9)])
def test_handoff_prefill_de_orders_respect_every_wait(P, D, persist, cap):
    """Each DE's enqueue order puts every spin-wait after its producers on
    that DE: a decode after this DE's reads of every request its K3 follows,
    a read reusing decode slots after the previous occupant's decode (or, with
    no persistence, after the reads its K3 follows)."""
    cfg = cluster(P, D, cap=cap if cap else 6.25e9)
    trajs = dp.synthesize(max_len=20000, count=6 * (P + D), seed=8, mean_turns=6, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.handoff, opt.persist, opt.prefill = True, persist, True
    opt.compute_quota, opt.prefill_cost = 2e-3, COST
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots, opt.de_pool_slots = xp.peak_slots, xp.de_peak_slots  # tight: reuse everywhere
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    jobs = xp.jobs()
    # the loads each job's K3 follows: jobs of its PE up to the largest job of
    # its forwards 0..last
    upto = {}
    for pe in range(xp.n_pe):
        m = -1
        for fi, (_, items) in enumerate(xp.forwards(pe)):
            m = max([m] + [it[1] for it in items])
            upto[(pe, fi)] = m
    bound = lambda j: upto[(jobs[j][4], xp.last_fwd(j))]
    n_reuse = 0
    for d in range(xp.n_pe, xp.n_engines):
        order = xp.de_order(d)
        assert sorted(c for c in order if c >= 0) == sorted(xp.by_reader(d))
        assert [-1 - c for c in order if c < 0] == (xp.by_de(d) if persist else [])
        pos = {("r", c) if c >= 0 else ("d", -1 - c): i for i, c in enumerate(order)}
        reads = [c for c in order if c >= 0]
        for i, c in enumerate(order):
            if c < 0:  # decode of j
                j = -1 - c
                need = [y for y in reads if jobs[y][4] == jobs[j][4] and y <= bound(j)]
                assert all(pos[("r", y)] < i for y in need)
            else:
                for p in xp.de_pred_jobs(c):
                    n_reuse += 1
                    if persist:
                        assert pos[("d", p)] < i
                    else:
                        need = [y for y in reads if jobs[y][4] == jobs[p][4] and y <= bound(p)]
                        assert all(pos[("r", y)] < i for y in need)
    assert n_reuse > 0
