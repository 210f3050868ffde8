"""A model of the executor's enqueue order in handoff + prefill (+
persistence) mode, checked for deadlock under the worst case the runtime
guards against: every stream of a device multiplexed onto ONE hardware FIFO,
so an operation waits for everything enqueued before it on its device
(CPU).  It mirrors engine_handoff.cpp: a PE enqueues its loads in FIFO order,
draining forwards (and the K3s they finish) before a load that reuses slots;
a DE follows the plan's de_order."""

import pytest

import paper_2602_21548_b200 as dp

SB = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)
COST = (2e-10, 1e-9, 4e-7, 1e-5)


def cluster(P, D, cap):
    c = dp.ClusterConfig()
    c.prefill_nodes, c.decode_nodes, c.engines_per_node = P, D, 1
    c.n_layer, c.kv_bytes_per_token_per_layer, c.block_size_tokens = 8, 576, 64
    c.cnic_bandwidth, c.storage_multiple, c.dram_bandwidth = 50e9, cap / 50e9, 500e9
    c.hbm_capacity_tokens, c.pe_buffer_bytes, c.de_buffer_bytes = 100_000_000, 1 << 42, 1 << 42
    return c


def enqueue_model(xp, persist, gated=False):
    jobs = xp.jobs()
    n_pe = xp.n_pe
    fifo = {}   # device -> [(op, deps)]
    row, last_row = {}, {}
    for p in range(n_pe):
        for fi, (_, items) in enumerate(xp.forwards(p)):
            for it in items:
                if it[1] >= 0:
                    row[it[1]] = it[5]
            last_row[(p, fi)] = max(it[5] for it in items)

    def fetch(y):  # the op that lands y's hit KV in its PE pool
        return ("load", y) if jobs[y][3] == jobs[y][4] else ("read", y)

    def release(p):  # what a reuse of p's decode slots waits for
        return [("decode", p)] if persist else [("k3", p)] + ([("read", p)] if jobs[p][5] and jobs[p][7] else [])

    for p in range(n_pe):
        ops = fifo.setdefault(("pe", p), [])
        fwds = xp.forwards(p)
        mine = xp.by_pe(p)
        st = {"fi": 0, "ki": 0}

        def enqueue_k3(j):
            deps = [("fwd", p, xp.last_fwd(j))]
            for q in xp.de_pred_jobs(j):
                deps += release(q)
            ops.append((("k3", j), deps))

        def drain(r):
            while st["fi"] < len(fwds) and last_row[(p, st["fi"])] < r:
                fi = st["fi"]
                deps = [fetch(it[1]) for it in fwds[fi][1] if it[1] >= 0 and it[2] > 0]
                ops.append((("fwd", p, fi), deps))
                st["fi"] += 1
                while st["ki"] < len(mine) and xp.last_fwd(mine[st["ki"]]) < st["fi"]:
                    enqueue_k3(mine[st["ki"]])
                    st["ki"] += 1

        for j in mine:
            if jobs[j][20] or gated:  # slot reuse, or the storage gate before each load
                drain(row[j])
            if not jobs[j][5] and jobs[j][7] > 0:
                ops.append((("load", j), [("k3", w) for w in jobs[j][20]]))
        drain(float("inf"))
        while st["ki"] < len(mine):
            enqueue_k3(mine[st["ki"]])
            st["ki"] += 1
    for d in range(n_pe, xp.n_engines):
        ops = fifo.setdefault(("de", d), [])
        for code in xp.de_order(d):
            if code >= 0:
                deps = [("k3", q) for q in xp.consumer_waits(code)]
                for q in xp.de_pred_jobs(code):
                    deps += release(q)
                ops.append((("read", code), deps))
            else:
                j = -1 - code
                ops.append((("decode", j), [("k3", j)] + ([("read", j)] if jobs[j][5] and jobs[j][7] else [])))
    # run every device's FIFO; an op completes when all its dependencies have
    done, heads = set(), {k: 0 for k in fifo}
    progress = True
    while progress:
        progress = False
        for k, ops in fifo.items():
            while heads[k] < len(ops) and all(dep in done for dep in ops[heads[k]][1]):
                done.add(ops[heads[k]][0])
                heads[k] += 1
                progress = True
    stuck = {k: fifo[k][heads[k]] for k in fifo if heads[k] < len(fifo[k])}
    return stuck, sum(len(v) for v in fifo.values())


@pytest.mark.parametrize("P,D,sessions,cap,persist", [
    (1, 1, 8, 6.25e9, True), (2, 2, 24, 6.25e9, True), (2, 2, 24, 6.25e9, False),
    (1, 3, 16, 50e9, True), (3, 1, 16, 6.25e9, True), (2, 2, 12, 50e9, True)])
@pytest.mark.parametrize("tight", [False, True])
@pytest.mark.parametrize("gated", [False, True])
def test_handoff_prefill_enqueue_order_cannot_deadlock(P, D, sessions, cap, persist, tight, gated):
    cfg = cluster(P, D, cap)
    trajs = dp.synthesize(max_len=20000, count=sessions, seed=9, mean_turns=8, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.handoff, opt.persist, opt.prefill = True, persist, True
    opt.compute_quota, opt.prefill_cost = 5e-4, COST
    if gated:
        opt.storage_cap_Bps = cap
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots, opt.de_pool_slots = xp.peak_slots, xp.de_peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    stuck, n_ops = enqueue_model(xp, persist, gated)
    assert n_ops > 0
    assert not stuck, f"deadlock under one FIFO per device: {stuck}"


def handoff_model(xp, persist):
    """engine_handoff.cpp without the prefill: a PE enqueues per job its load
    then its K3; a DE interleaves reads and decodes in global order."""
    jobs = xp.jobs()
    by_ticket = {(j[4], j[8]): i for i, j in enumerate(jobs)}          # PE row -> job
    by_de_ticket = {(j[13], j[16]): i for i, j in enumerate(jobs)}     # decode row -> job
    fifo = {}

    def release(q):
        if persist:
            return [("decode", q)]
        return [("k3", q)] + ([("read", q)] if jobs[q][5] and jobs[q][7] else [])

    de_pred = {i: [by_de_ticket[(j[13], t)] for t in j[19]] for i, j in enumerate(jobs)}
    for p in range(xp.n_pe):
        ops = fifo.setdefault(("pe", p), [])
        for j in xp.by_pe(p):
            jj = jobs[j]
            if not jj[5] and jj[7] > 0:
                ops.append((("load", j), [("k3", w) for w in jj[20]]))
            deps = []
            if jj[7] > 0:
                deps.append(("read", j) if jj[5] else ("load", j))
            if not jj[5] and jj[7] == 0:
                deps += [("k3", w) for w in jj[20]]
            for q in de_pred[j]:
                deps += release(q)
            ops.append((("k3", j), deps))
    for d in range(xp.n_pe, xp.n_engines):
        ops = fifo.setdefault(("de", d), [])
        reads, decs = xp.by_reader(d), (xp.by_de(d) if persist else [])
        ri = di = 0
        while ri < len(reads) or di < len(decs):
            if ri < len(reads) and (di >= len(decs) or reads[ri] <= decs[di]):
                x = reads[ri]
                ri += 1
                deps = [("k3", by_ticket[(jobs[x][4], t)]) for t in jobs[x][21]]
                for q in de_pred[x]:
                    deps += release(q)
                ops.append((("read", x), deps))
            else:
                j = decs[di]
                di += 1
                ops.append((("decode", j), [("k3", j)] + ([("read", j)] if jobs[j][5] and jobs[j][7] else [])))
    done, heads = set(), {k: 0 for k in fifo}
    progress = True
    while progress:
        progress = False
        for k, ops in fifo.items():
            while heads[k] < len(ops) and all(dep in done for dep in ops[heads[k]][1]):
                done.add(ops[heads[k]][0])
                heads[k] += 1
                progress = True
    return {k: fifo[k][heads[k]] for k in fifo if heads[k] < len(fifo[k])}


@pytest.mark.parametrize("P,D,persist", [(1, 1, True), (2, 2, True), (2, 2, False), (1, 3, True), (3, 1, True)])
def test_handoff_enqueue_order_cannot_deadlock(P, D, persist):
    cfg = cluster(P, D, 6.25e9)
    trajs = dp.synthesize(max_len=20000, count=6 * (P + D), seed=9, mean_turns=8, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.handoff, opt.persist = True, persist
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots, opt.de_pool_slots = xp.peak_slots, xp.de_peak_slots
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    stuck = handoff_model(xp, persist)
    assert not stuck, f"deadlock under one FIFO per device: {stuck}"


def prefill_model(xp, gated):
    """engine_prefill.cpp (PE) + engine.cpp run_step (DE) in prefill mode."""
    jobs = xp.jobs()
    fifo = {}
    for p in range(xp.n_pe):
        ops = fifo.setdefault(("pe", p), [])
        fwds = xp.forwards(p)
        rows = xp.fwd_rows(p)
        job_of_row = {}
        for _, items in fwds:
            for it in items:
                job_of_row[it[5]] = it[1]
        last_row = [max(it[5] for it in items) for _, items in fwds]
        fi = 0

        def fetch(y):
            return ("load", y) if jobs[y][3] == jobs[y][4] else ("read", y)

        def forwards_before(r):
            nonlocal fi
            while fi < len(fwds) and last_row[fi] < r:
                ops.append((("fwd", p, fi), [fetch(it[1]) for it in fwds[fi][1] if it[1] >= 0 and it[2] > 0]))
                fi += 1

        for r in range(len(rows)):
            j = job_of_row.get(r, -1)
            if j < 0 or jobs[j][3] != p or jobs[j][7] == 0:
                continue
            waits = xp.consumer_waits(j)
            if gated or waits:
                forwards_before(r)
            ops.append((("load", j), [("fwd", p, xp.last_fwd(w)) for w in waits]))
        forwards_before(float("inf"))
    for d in range(xp.n_pe, xp.n_engines):
        ops = fifo.setdefault(("de", d), [])
        for x in xp.by_reader(d):
            ops.append((("read", x), [("fwd", jobs[x][4], xp.last_fwd(w)) for w in xp.consumer_waits(x)]))
    done, heads = set(), {k: 0 for k in fifo}
    progress = True
    while progress:
        progress = False
        for k, ops in fifo.items():
            while heads[k] < len(ops) and all(dep in done for dep in ops[heads[k]][1]):
                done.add(ops[heads[k]][0])
                heads[k] += 1
                progress = True
    return {k: fifo[k][heads[k]] for k in fifo if heads[k] < len(fifo[k])}


@pytest.mark.parametrize("P,D", [(1, 1), (2, 2), (1, 3), (3, 1)])
@pytest.mark.parametrize("gated", [False, True])
def test_prefill_enqueue_order_cannot_deadlock(P, D, gated):
    cfg = cluster(P, D, 6.25e9)
    trajs = dp.synthesize(max_len=20000, count=6 * (P + D), seed=9, mean_turns=8, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.prefill, opt.compute_quota, opt.prefill_cost = True, 5e-4, COST
    if gated:
        opt.storage_cap_Bps = 6.25e9
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots = xp.peak_slots
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert any(xp.consumer_waits(i) for i in range(len(xp.jobs())))
    stuck = prefill_model(xp, gated)
    assert not stuck, f"deadlock under one FIFO per device: {stuck}"


def plain_model(xp):
    """engine.cpp run_step: each reader's loads in its order, a load reusing a
    slot another engine wrote waits for that load; a PE ends with a wait on
    every push into its pool."""
    jobs = xp.jobs()
    by_ticket = {(j[4], j[8]): i for i, j in enumerate(jobs)}
    fifo = {}
    for e in range(xp.n_engines):
        ops = fifo.setdefault(e, [])
        for x in xp.by_reader(e):
            ops.append((("load", x), [("load", by_ticket[(jobs[x][4], t)]) for t in jobs[x][11]]))
        if e < xp.n_pe:
            ops.append((("end", e), [("load", i) for i in xp.by_pe(e) if jobs[i][3] != e]))
    done, heads = set(), {k: 0 for k in fifo}
    progress = True
    while progress:
        progress = False
        for k, ops in fifo.items():
            while heads[k] < len(ops) and all(dep in done for dep in ops[heads[k]][1]):
                done.add(ops[heads[k]][0])
                heads[k] += 1
                progress = True
    return {k: fifo[k][heads[k]] for k in fifo if heads[k] < len(fifo[k])}


@pytest.mark.parametrize("P,D", [(1, 1), (2, 2), (1, 3), (3, 1)])
def test_plain_enqueue_order_cannot_deadlock(P, D):
    cfg = cluster(P, D, 6.25e9)
    trajs = dp.synthesize(max_len=20000, count=6 * (P + D), seed=9, mean_turns=8, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots = xp.peak_slots
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert any(j[11] for j in xp.jobs())  # cross-reader reuse exists
    stuck = plain_model(xp)
    assert not stuck, f"deadlock under one FIFO per device: {stuck}"
