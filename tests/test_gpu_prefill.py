"""GPU parity of K5 (dp_prefill_attend), the prefill stand-in that the
compute-quota batching drives.

K5 reads the KV the loader landed in the PE pool and accumulates, per
request and layer, sum_q sum_t dot_u8(Q[q], K[t]) mod 2^64.  The oracle
(oracle/kvref.c kvref_attend_digest) computes the same integer from column
sums; integer sums are exact, so the comparison is bit-for-bit."""

import numpy as np
import pytest

from oracle import refpy
from paper_2602_21548_b200 import abi

pytestmark = pytest.mark.gpu
SEED = 9


def dev(x, dtype):
    import torch
    return torch.tensor(np.asarray(x, dtype=dtype), device="cuda:0")


@pytest.mark.parametrize("L,T,b", [(4, 64, 576), (2, 64, 4096), (3, 16, 64), (2, 128, 208)])
def test_attend_digest_matches_oracle(gpus, L, T, b):
    import torch
    rng = np.random.default_rng(b + T)
    g = abi.geom(L, T, b)
    gr = refpy.geom(L, T, b)
    n_fb, n_slots = 24, 48
    st = abi.Store(0, g, n_fb, SEED)
    pool = abi.Pool(0, g, n_slots, 8)
    try:
        # requests: (cached, [(q_begin, bsz) chunks]) -- edge cases: no cache,
        # partial last block, a 1-token chunk, chunks split over launches
        reqs = [(0, [(0, 50)]), (T * 3 + 5, [(0, 64), (64, 1), (65, 70)]), (T, [(0, 0)]),
                (T * 2 - 1, [(3, 130)]), (T * 5, [(0, 1)])]
        free = list(rng.permutation(n_slots))
        keep, specs, meta = [], [], []
        for r, (C, _) in enumerate(reqs):
            nb = -(-C // T)
            fbs = rng.choice(n_fb, size=max(nb, 1), replace=False).astype(np.int64)[:nb]
            slots = np.array([free.pop() for _ in range(nb)], dtype=np.int32)
            meta.append((fbs, slots))
            if nb:
                tf, ts = dev(fbs, np.int64), dev(slots, np.int32)
                keep += [tf, ts]
                specs.append((tf.data_ptr(), ts.data_ptr(), C, nb, 0, L, r))
        abi.h2d_layer_gather(pool, st, abi.make_jobs(specs), len(specs))
        digest = torch.zeros((len(reqs), L), dtype=torch.int64, device="cuda:0")
        for layer in range(L):
            for pass_ in range(2):  # two launches per layer: chunks split between them
                items = []
                for r, (C, chunks) in enumerate(reqs):
                    ts = dev(meta[r][1] if len(meta[r][1]) else [0], np.int32)
                    keep.append(ts)
                    for ci, (q0, bsz) in enumerate(chunks):
                        if ci % 2 != pass_:
                            continue
                        items.append(abi.AttendItem(ts.data_ptr(), C, q0, bsz,
                                                    digest[r].data_ptr(), 1000 + r, 0))
                arr = (abi.AttendItem * max(1, len(items)))(*items)
                abi.prefill_attend(pool, layer, arr, len(items), SEED)
        torch.cuda.synchronize()
        got = digest.cpu().numpy().view(np.uint64)
        for r, (C, chunks) in enumerate(reqs):
            for layer in range(L):
                want = 0
                for q0, bsz in chunks:
                    want = (want + refpy.attend_digest(gr, SEED, list(map(int, meta[r][0])), C, 1000 + r,
                                                       layer, q0, bsz)) % (1 << 64)
                assert int(got[r, layer]) == want, (r, layer)
    finally:
        pool.close()
        st.close()


def test_attend_many_items_and_ctas(gpus):
    """More items than one launch carries (48) and a CTA cap of 1: the unit
    loop and the launch split give the same digests."""
    import torch
    L, T, b = 2, 64, 576
    g, gr = abi.geom(L, T, b), refpy.geom(L, T, b)
    st = abi.Store(0, g, 8, SEED)
    pool = abi.Pool(0, g, 8, 1)
    try:
        fbs = np.arange(8, dtype=np.int64)
        slots = np.arange(8, dtype=np.int32)[::-1].copy()
        tf, ts = dev(fbs, np.int64), dev(slots, np.int32)
        C = 8 * T - 7
        abi.h2d_layer_gather(pool, st, abi.make_jobs([(tf.data_ptr(), ts.data_ptr(), C, 8, 0, L, 0)]), 1)
        n = 100
        for cap in (0, 1):
            abi.set_attend_ctas(0, cap)
            digest = torch.zeros((n, L), dtype=torch.int64, device="cuda:0")
            items = (abi.AttendItem * n)(*[abi.AttendItem(ts.data_ptr(), C, i, 1 + i % 3,
                                                          digest[i].data_ptr(), 7, 0) for i in range(n)])
            for layer in range(L):
                abi.prefill_attend(pool, layer, items, n, SEED)
            torch.cuda.synchronize()
            got = digest.cpu().numpy().view(np.uint64)
            for i in (0, 1, 47, 48, 99):
                for layer in range(L):
                    assert int(got[i, layer]) == refpy.attend_digest(gr, SEED, list(map(int, fbs)), C, 7,
                                                                     layer, i, 1 + i % 3)
        abi.set_attend_ctas(0, 0)
    finally:
        pool.close()
        st.close()


def test_attend_rejects_bad_arguments(gpus):
    g = abi.geom(2, 64, 576)
    pool = abi.Pool(0, g, 4, 1)
    try:
        bad = (abi.AttendItem * 1)(abi.AttendItem(None, 64, 0, 4, None, 0, 0))
        with pytest.raises(abi.DualPathError):
            abi.prefill_attend(pool, 0, bad, 1, SEED)       # cached KV without slots
        ok = (abi.AttendItem * 1)(abi.AttendItem(None, 0, 0, 0, None, 0, 0))
        with pytest.raises(abi.DualPathError):
            abi.prefill_attend(pool, 2, ok, 1, SEED)        # layer out of range
        abi.prefill_attend(pool, 0, ok, 1, SEED)            # empty item: no launch
    finally:
        pool.close()


# ---- the executor's prefill mode: quota-batched forwards over landed KV ----
import paper_2602_21548_b200 as dp  # noqa: E402

STORAGE_BOUND = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)
COST = (2e-10, 1e-9, 4e-7, 1e-5)


def cluster(P, D, L=4, b=576, T=64):
    cfg = dp.ClusterConfig()
    cfg.prefill_nodes, cfg.decode_nodes, cfg.engines_per_node = P, D, 1
    cfg.n_layer, cfg.kv_bytes_per_token_per_layer, cfg.block_size_tokens = L, b, T
    cfg.cnic_bandwidth, cfg.storage_multiple, cfg.dram_bandwidth = 50e9, 0.125, 500e9
    cfg.hbm_capacity_tokens, cfg.pe_buffer_bytes, cfg.de_buffer_bytes = 100_000_000, 1 << 42, 1 << 42
    return cfg


def prefill_plan(cfg, policy, tight, quota=5e-4, count=6, turns=5, seed=4, k1_mode=0):
    trajs = dp.synthesize(max_len=12000, count=count, seed=seed, mean_turns=turns, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy=policy, **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.k1_mode = k1_mode
    opt.prefill = True
    opt.compute_quota = quota
    opt.prefill_cost = COST
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots = xp.peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    return trajs, planned, xp


def expected_digests(cfg, planned, xp, pe):
    g = refpy.geom(cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer)
    reqs = {r[0]: r for r in planned["requests"]}
    out = []
    for rid in xp.fwd_rows(pe):
        r = reqs[rid]
        C, A, traj = r[3], r[4], r[1]
        fbs = [xp.fb_of(traj, k) for k in range(-(-C // cfg.block_size_tokens))]
        out.append([refpy.attend_digest(g, SEED, fbs, C, rid, layer, 0, A) if C and A else 0
                    for layer in range(cfg.n_layer)])
    return out


def check_digests(eng, cfg, planned, xp, skip=()):
    got = np.asarray(eng.prefill_digests(), dtype=np.uint64).reshape(-1, cfg.n_layer)
    want = expected_digests(cfg, planned, xp, eng.engine)
    assert len(want) == got.shape[0] > 0
    for row, w in enumerate(want):
        if row not in skip:
            assert [int(v) for v in got[row]] == w, f"digest mismatch on row {row}"


@pytest.mark.parametrize("tight", [False, True])
def test_prefill_single_pe(gpus, tight):
    cfg = cluster(1, 1)
    trajs, planned, xp = prefill_plan(cfg, "pe_only", tight)
    n_fwd = len(xp.forwards(0))
    assert n_fwd > 1
    eng = dp.EngineRuntime(xp, 0, 0)
    for _ in range(2):
        eng.reset_counters()
        r = eng.run_step()
        assert r.forwards == n_fwd and r.bytes_read == xp.hit_bytes
        check_digests(eng, cfg, planned, xp)
    # the compute alone over the KV left in the pool: same digests for every
    # request whose slots no later request reused
    r = eng.run_forwards()
    assert r.forwards == n_fwd and r.bytes_read == 0
    reused = {w for i in range(len(xp.jobs())) for w in xp.consumer_waits(i)}
    rows = xp.fwd_rows(0)
    jobs = xp.jobs()
    skip = {rows.index(jobs[w][0]) for w in reused}
    assert len(skip) < len(rows)
    check_digests(eng, cfg, planned, xp, skip=skip)


@pytest.mark.parametrize("tight", [False, True])
def test_prefill_1p1d_dual_path(de_dev, tight):
    cfg = cluster(1, 1)
    trajs, planned, xp = prefill_plan(cfg, "dual_path", tight, count=8, turns=6, seed=8)
    assert xp.reader_bytes[1] > 0
    if tight:
        assert any(xp.consumer_waits(i) for i in range(len(xp.jobs())))
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    for _ in range(2):
        pe.reset_counters()
        res = dp.run_step_all([pe, de])
        assert res[0].bytes_read + res[1].bytes_read == xp.hit_bytes
        check_digests(pe, cfg, planned, xp)


@pytest.mark.parametrize("tight,persist,layerwise,k1,k3,k4", [
    (False, False, True, 0, 0, 0), (True, False, True, 0, 0, 0), (True, True, True, 0, 0, 0),
    (True, False, False, 0, 0, 0), (True, True, True, 3, 0, 0),
    # K3 on the copy engines (gated per layer / after the forward), staged K4
    (True, False, True, 3, 1, 0), (True, True, False, 3, 1, 1), (False, True, False, 0, 1, 1)])
def test_prefill_with_handoff_1p1d(de_dev, tight, persist, layerwise, k1, k3, k4):
    """The whole pipeline: loads on both paths, quota-batched K5 forwards on
    the PE, K3 handoff of each prompt -- layer by layer as its finishing
    forward computes each layer (layerwise), or after that forward -- (decode
    + K4 persistence).  Digests equal the oracle's and every prompt lands in
    its DE's decode pool."""
    from test_gpu_engine import handoff_engines, verify_prompt_pool
    cfg = cluster(1, 1, L=4)
    trajs = dp.synthesize(max_len=12000, count=8, seed=6, mean_turns=5, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.handoff = True
    opt.persist = persist
    opt.prefill = True
    opt.compute_quota = 5e-4
    opt.prefill_cost = COST
    opt.handoff_layerwise = layerwise
    opt.k1_mode = k1
    opt.k3_mode = k3
    opt.persist_mode = k4
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots, opt.de_pool_slots = xp.peak_slots, xp.de_peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    rts = handoff_engines(xp, 2, [0, de_dev])
    for _ in range(2):
        for rt in rts:
            rt.reset_counters()
        res = dp.run_step_all(rts)
        assert sum(r.bytes_read for r in res) == xp.hit_bytes
        assert res[0].forwards == len(xp.forwards(0)) > 1
        check_digests(rts[0], cfg, planned, xp)
        # every request's prompt is handed off, after (layerwise: as) its last forward computes
        assert len(res[0].ttft_ms) == len(res[0].handoff_lag_ms) == len(xp.jobs())
        assert min(res[0].handoff_lag_ms) > -1e-3 and max(res[0].ttft_ms) <= res[0].device_ms + 1e-3
    if not persist:  # (with persistence the decode pool's last occupants also hold generated tokens)
        assert verify_prompt_pool(rts[1], xp, cfg) > 0
    ctr = np.asarray(rts[1].counters(), dtype=np.int64).reshape(-1, cfg.n_layer + 1)
    for job in xp.jobs():
        blocks = (job[7] if job[5] else 0) + job[15]
        assert ctr[job[16], cfg.n_layer] == blocks * xp.items_per_block * cfg.n_layer


@pytest.mark.parametrize("L,T,b", [(3, 64, 4096), (4, 16, 1024), (2, 128, 208)])
def test_prefill_other_geometries(gpus, L, T, b):
    """Qwen-sized KV rows, small and large blocks: the executor's forwards
    and K5 digests stay exact."""
    cfg = cluster(1, 1, L=L, b=b, T=T)
    trajs, planned, xp = prefill_plan(cfg, "pe_only", tight=True, quota=2e-4, count=5, turns=4, seed=3)
    eng = dp.EngineRuntime(xp, 0, 0)
    eng.reset_counters()
    r = eng.run_step()
    assert r.forwards == len(xp.forwards(0)) > 1
    check_digests(eng, cfg, planned, xp)


@pytest.mark.parametrize("tight", [False, True])
def test_prefill_with_staged_loads(gpus, tight):
    """k1_mode 3 (copy engine into the HBM ring + scatter kernel) under the
    quota-batched prefill: every K5 digest equals the oracle's."""
    cfg = cluster(1, 1)
    trajs, planned, xp = prefill_plan(cfg, "pe_only", tight, k1_mode=3)
    eng = dp.EngineRuntime(xp, 0, 0)
    for _ in range(2):
        eng.reset_counters()
        r = eng.run_step()
        assert r.bytes_read == xp.hit_bytes
        check_digests(eng, cfg, planned, xp)


def test_attend_signal_sets_the_layer_flag(gpus):
    """dp_prefill_attend_signal: the layer's 'computed' flag is 1 after the
    call, released by K5's last CTA, or by a stream write when the call has
    nothing to compute (the layerwise handoff's gate)."""
    import ctypes
    import torch
    L, T, b = 2, 64, 576
    g = abi.geom(L, T, b)
    st = abi.Store(0, g, 4, SEED)
    pool = abi.Pool(0, g, 8, 1)
    try:
        slots = dev([0, 1], np.int32)
        fbs = dev([0, 1], np.int64)
        abi.h2d_layer_gather(pool, st, abi.make_jobs([(fbs.data_ptr(), slots.data_ptr(), 100, 2, 0, L, -1)]), 1)
        flags = torch.zeros(2, dtype=torch.int32, device="cuda:0")
        digest = torch.zeros(L, dtype=torch.int64, device="cuda:0")
        items = (abi.AttendItem * 1)()
        items[0] = abi.AttendItem(slots.data_ptr(), 100, 0, 40, digest.data_ptr(), 3, 0)
        abi.check(abi.lib().dp_prefill_attend_signal(pool.ptr, 0, items, 1, SEED, flags.data_ptr(), None))
        empty = (abi.AttendItem * 1)()
        empty[0] = abi.AttendItem(slots.data_ptr(), 0, 0, 40, digest.data_ptr(), 3, 0)  # no cached keys
        abi.check(abi.lib().dp_prefill_attend_signal(pool.ptr, 1, empty, 1, SEED,
                                                     flags.data_ptr() + 4, None))
        torch.cuda.synchronize()
        assert flags.tolist() == [1, 1]
        want = refpy.attend_digest(refpy.geom(L, T, b), SEED, [0, 1], 100, 3, 0, 0, 40)
        assert int(digest[0].item()) & (2 ** 64 - 1) == want
    finally:
        pool.close()
        st.close()
