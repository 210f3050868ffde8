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
