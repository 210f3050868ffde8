"""GPU parity of the executor: plan -> EngineRuntime steps -> final paged KV
pools compared with the CPU oracle (every Layer Block's content hash, from
oracle/kvref.c's content formula), block tables and counters."""

import numpy as np
import pytest

import paper_2602_21548_b200 as dp
from oracle import refpy

pytestmark = pytest.mark.gpu

SEED = 9


def cluster(P, D, L=6, b=576, T=64):
    cfg = dp.ClusterConfig()
    cfg.prefill_nodes, cfg.decode_nodes, cfg.engines_per_node = P, D, 1
    cfg.n_layer, cfg.kv_bytes_per_token_per_layer, cfg.block_size_tokens = L, b, T
    cfg.cnic_bandwidth = 50e9
    cfg.storage_multiple = 0.125
    cfg.dram_bandwidth = 500e9
    cfg.hbm_capacity_tokens = 100_000_000
    cfg.pe_buffer_bytes = 1 << 42
    cfg.de_buffer_bytes = 1 << 42
    return cfg


STORAGE_BOUND = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)


def final_occupants(xp, pe):
    """slot -> (Full Block, valid tokens) of the last job that wrote it."""
    last = {}
    for job in xp.jobs():
        req, traj, rnd, reader, jpe, de_path, cached, nblk, ticket, slots, fbs, preds, fence = job[:13]
        if jpe != pe:
            continue
        for k, (s, fb) in enumerate(zip(slots, fbs)):
            last[s] = (fb, min(xp_T(xp), cached - xp_T(xp) * k))
    return last


def xp_T(xp):
    return 64


def verify_pool(engine, xp, cfg):
    last = final_occupants(xp, engine.engine)
    slots = sorted(last)
    g = refpy.geom(cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer)
    for layer in range(cfg.n_layer):
        got = engine.checksum(layer, slots, [last[s][1] for s in slots])
        want = [refpy.layer_block_hash(g, SEED, last[s][0], layer, last[s][1]) for s in slots]
        assert list(got) == want, f"pool mismatch on PE {engine.engine} layer {layer}"
    return len(slots)


def verify_counters(engine, xp, cfg):
    ctr = np.asarray(engine.counters(), dtype=np.int64).reshape(-1, cfg.n_layer + 1)
    for job in xp.jobs():
        if job[4] != engine.engine:
            continue
        items = job[7] * xp.items_per_block
        assert (ctr[job[8], :cfg.n_layer] == items).all()
        assert ctr[job[8], cfg.n_layer] == items * cfg.n_layer


def small_trace(count=6, turns=5, max_len=12000, seed=4):
    return dp.synthesize(max_len=max_len, count=count, seed=seed, mean_turns=turns, sigma_turns=0)


def test_single_engine_pe_only(gpus):
    cfg = cluster(1, 1)
    trajs = small_trace()
    planned = dp.plan(cfg, trajs, policy="pe_only", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert xp.reader_bytes[1] == 0 and xp.reader_bytes[0] == xp.hit_bytes
    eng = dp.EngineRuntime(xp, 0, 0)
    for _ in range(2):
        eng.reset_counters()
        r = eng.run_step()
        assert r.bytes_read == xp.hit_bytes
    verify_counters(eng, xp, cfg)
    assert verify_pool(eng, xp, cfg) > 0


def test_slot_reuse_same_reader(gpus):
    # a pool exactly at the plan's peak forces FIFO reuse within the step
    cfg = cluster(1, 1)
    trajs = small_trace(count=4, turns=6)
    planned = dp.plan(cfg, trajs, policy="pe_only", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    probe = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots = probe.peak_slots
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert xp.pool_slots == xp.peak_slots
    assert any(job[12] for job in xp.jobs()), "expected same-reader slot reuse"
    eng = dp.EngineRuntime(xp, 0, 0)
    eng.reset_counters()
    eng.run_step()
    verify_pool(eng, xp, cfg)


@pytest.mark.parametrize("policy", ["dual_path", "pe_only", "round_robin"])
def test_two_engines_1p1d(de_dev, policy):
    cfg = cluster(1, 1)
    trajs = small_trace(count=8, turns=5)
    kw = dict(STORAGE_BOUND)
    if policy == "round_robin":
        planned = dp.plan(cfg, trajs, policy="dual_path", sched_mode="round_robin", **kw)
    else:
        planned = dp.plan(cfg, trajs, policy=policy, **kw)
    opt = dp.ExecOptions()
    opt.seed = SEED
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    if policy != "pe_only":
        assert xp.reader_bytes[1] > 0, "dual path should read on the DE side"
    for _ in range(2):
        pe.reset_counters()
        res = dp.run_step_all([pe, de])
        assert res[0].bytes_read + res[1].bytes_read == xp.hit_bytes
    verify_counters(pe, xp, cfg)
    verify_pool(pe, xp, cfg)


def test_cross_reader_slot_reuse_hazards(de_dev):
    # tight pool: slots freed by a DE-path job get reused by PE-path jobs and
    # vice versa; the hazard waits keep the final pool equal to the oracle's
    cfg = cluster(1, 1, L=4)
    trajs = small_trace(count=10, turns=6, seed=8)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    probe = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots = probe.peak_slots
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert any(job[11] for job in xp.jobs()), "expected cross-reader reuse"
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    for _ in range(3):
        pe.reset_counters()
        dp.run_step_all([pe, de])
        verify_pool(pe, xp, cfg)


def test_two_engines_k1_on_copy_engine(de_dev):
    cfg = cluster(1, 1)
    trajs = small_trace(count=8, turns=5)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.k1_mode = 1
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    for _ in range(2):
        pe.reset_counters()
        res = dp.run_step_all([pe, de])
        assert res[0].launches <= 1  # the PE issues copies, not kernels (at most its final wait)
    verify_counters(pe, xp, cfg)
    verify_pool(pe, xp, cfg)


@pytest.mark.parametrize("k1,k2,prefill", [(1, 1, False), (0, 0, False), (1, 1, True)])
def test_two_engines_block_major_pool(de_dev, k1, k2, prefill):
    """A block-major PE pool (ExecOptions::pool_layout = 1): with the copy
    engines on both paths every load is whole Full-Block runs straight into
    the pool (no kernels on the PE or the DE); the SM gathers and the
    prefill stand-in read and write it through the slot stride.  Final pool
    and counters as the oracle says."""
    cfg = cluster(1, 1)
    trajs = small_trace(count=8, turns=5)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.pool_layout = 1
    opt.k1_mode, opt.k2_mode = k1, k2
    if prefill:
        opt.prefill = True
        opt.compute_quota = 5e-4
        opt.prefill_cost = (2e-10, 1e-9, 4e-7, 1e-5)
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    for _ in range(2):
        pe.reset_counters()
        res = dp.run_step_all([pe, de])
        assert sum(r.bytes_read for r in res) == xp.hit_bytes
        if k1 == 1 and not prefill:
            assert res[0].launches <= 1  # the PE issues copies only (at most its final wait)
    verify_counters(pe, xp, cfg)
    verify_pool(pe, xp, cfg)
    opt.handoff = True
    with pytest.raises(ValueError):
        dp.build_exec_plan(cfg, trajs, planned, opt)


# ------------------------------------------------------------ PD handoff
def prompt_occupants(xp, engine, T=64):
    """slot -> (Full Block, valid prompt tokens) of the last job that used it,
    in the PE pool (engine < n_pe) or in the DE decode pool."""
    last = {}
    for job in xp.jobs():
        traj, pe, prompt, de = job[1], job[4], job[14], job[13]
        if engine < xp.n_pe and pe == engine:
            slots = job[17]
        elif engine >= xp.n_pe and de == engine:
            slots = job[18]
        else:
            continue
        for k, s in enumerate(slots):
            last[s] = (xp.fb_of(traj, k), min(T, prompt - T * k))
    return last


def verify_prompt_pool(engine, xp, cfg):
    last = prompt_occupants(xp, engine.engine, cfg.block_size_tokens)
    slots = sorted(last)
    g = refpy.geom(cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer)
    for layer in range(cfg.n_layer):
        got = engine.checksum(layer, slots, [last[s][1] for s in slots])
        want = [refpy.layer_block_hash(g, SEED, last[s][0], layer, last[s][1]) for s in slots]
        assert list(got) == want, f"engine {engine.engine} layer {layer}"
    return len(slots)


def handoff_engines(xp, n, devices=None):
    """Engine e on devices[e] (default: GPU e); engines may share a GPU."""
    import torch
    devices = list(range(n)) if devices is None else devices
    assert torch.cuda.device_count() > max(devices)
    rts = [dp.EngineRuntime(xp, e, devices[e]) for e in range(n)]
    for a in rts:
        for b in rts:
            if a is not b and b.has_pool and ((a.is_pe and not b.is_pe) or (b.is_pe and not a.is_pe)):
                a.attach_peer_local(b.engine, b)
    return rts


@pytest.mark.parametrize("policy,tight,layer_gate,staged,k3", [
    ("dual_path", False, 0, False, 0), ("dual_path", True, 0, False, 0), ("pe_only", True, 0, False, 0),
    ("dual_path", True, 1, False, 0), ("dual_path", True, 0, True, 0),
    # K3 on the copy engines: no gate (2D copies per run), gated per layer (layer_gate 1)
    ("dual_path", True, 0, True, 1), ("dual_path", True, 1, False, 1), ("pe_only", False, 0, False, 1)])
def test_handoff_1p1d(de_dev, policy, tight, layer_gate, staged, k3):
    cfg = cluster(1, 1, L=6)
    trajs = small_trace(count=8, turns=5, seed=6)
    planned = dp.plan(cfg, trajs, policy=policy, **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.handoff = True
    opt.k3_layer_gate = layer_gate
    opt.k3_mode = k3
    if staged:  # staged K1 and the staged dual gather (ring smaller than a request)
        opt.k1_mode, opt.k2_mode = 3, 2
        opt.stage_ring_bytes = 16 * 6 * 64 * 576 * 4
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
    assert verify_prompt_pool(rts[0], xp, cfg) > 0
    assert verify_prompt_pool(rts[1], xp, cfg) > 0
    # decode-ready rows: every request's prompt fully landed in the decode pool
    ctr = np.asarray(rts[1].counters(), dtype=np.int64).reshape(-1, cfg.n_layer + 1)
    for job in xp.jobs():
        blocks = (job[7] if job[5] else 0) + job[15]
        assert ctr[job[16], cfg.n_layer] == blocks * xp.items_per_block * cfg.n_layer


@pytest.mark.parametrize("placement", ["one_gpu", "four_gpus"])
def test_handoff_2p2d_tight(gpus, placement):
    if placement == "four_gpus" and gpus < 4:
        pytest.skip("needs 4 GPUs")
    cfg = cluster(2, 2, L=4)
    trajs = small_trace(count=12, turns=5, seed=9)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.handoff = True
    probe = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots, opt.de_pool_slots = probe.peak_slots, probe.de_peak_slots
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    rts = handoff_engines(xp, 4, [0, 0, 0, 0] if placement == "one_gpu" else None)
    for _ in range(2):
        for rt in rts:
            rt.reset_counters()
        dp.run_step_all(rts)
    for rt in rts:
        verify_prompt_pool(rt, xp, cfg)


@pytest.mark.parametrize("tight,staged", [(False, False), (True, False), (True, True), (False, True)])
def test_handoff_with_persistence(de_dev, tight, staged):
    """PD handoff + decode stand-in + K4 persistence: the decode pools end with
    prompt + generated tokens of their last occupants, and every generated
    token of every request is in its DE's persist store, byte for byte."""
    cfg = cluster(1, 1, L=4)
    trajs = small_trace(count=6, turns=4, seed=12)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.handoff = True
    opt.persist = True
    opt.k3_mode = opt.persist_mode = 1 if staged else 0  # copy-engine K3 + staged K4, or the SM kernels
    opt.stage_ring_bytes = 8 * 4 * 64 * 576  # small persist ring: 4 segments of 2 Full Blocks
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots, opt.de_pool_slots = xp.peak_slots, xp.de_peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    rts = handoff_engines(xp, 2, [0, de_dev])
    for _ in range(2):
        for rt in rts:
            rt.reset_counters()
        dp.run_step_all(rts)
    verify_prompt_pool(rts[0], xp, cfg)
    T, b, L = cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer, cfg.n_layer
    g = refpy.geom(L, T, b)
    # decode pool: last occupant of each slot holds prompt + generated tokens
    last = {}
    for i, job in enumerate(xp.jobs()):
        total = job[14] + xp.job_gen(i)
        for k in range(-(-total // T)):
            pass
    de = rts[1]
    checked = 0
    for i, job in enumerate(xp.jobs()):
        traj, prompt, gen = job[1], job[14], xp.job_gen(i)
        for k in range(prompt // T, -(-(prompt + gen) // T)):
            fb = xp.fb_of(traj, k)
            a, z = max(prompt, k * T) - k * T, min(prompt + gen, (k + 1) * T) - k * T
            for layer in range(L):
                got = np.frombuffer(de.read_persisted(fb, layer), dtype=np.uint8)
                want = refpy.layer_block(g, SEED, fb, layer, T)
                assert np.array_equal(got[a * b:z * b], want[a * b:z * b]), (i, k, layer)
                checked += 1
    assert checked > 0
    del last


def test_two_engines_k2_on_copy_engine(de_dev):
    # tight pool: cross-reader reuse hazards with the DE's copy-engine pushes
    cfg = cluster(1, 1, L=4)
    trajs = small_trace(count=10, turns=6, seed=8)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.k2_mode = 1
    probe = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.pool_slots = probe.peak_slots
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert xp.reader_bytes[1] > 0
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    for _ in range(2):
        pe.reset_counters()
        dp.run_step_all([pe, de])
        verify_counters(pe, xp, cfg)
        verify_pool(pe, xp, cfg)


@pytest.mark.parametrize("tight", [False, True])
def test_k1_hybrid_sm_and_copy_engine(gpus, tight):
    """k1_mode 2: the PE's jobs split between the SM gather and the copy
    engine on two streams; a tight pool makes slot reuse cross the streams."""
    cfg = cluster(1, 1, L=4)
    trajs = small_trace(count=6, turns=6)
    planned = dp.plan(cfg, trajs, policy="pe_only", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.k1_mode = 2
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots = xp.peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
        assert any(job[12] for job in xp.jobs())
    eng = dp.EngineRuntime(xp, 0, 0)
    for _ in range(2):
        eng.reset_counters()
        r = eng.run_step()
        assert r.bytes_read == xp.hit_bytes
        assert 0 < r.launches < len(xp.jobs())  # some jobs went to the copy engine
    verify_counters(eng, xp, cfg)
    verify_pool(eng, xp, cfg)


def test_edge_cold_only_plan(gpus):
    """Every request cold (first turns only): no hit KV, no jobs; the step
    runs and moves nothing."""
    cfg = cluster(1, 1)
    trajs = small_trace(count=5, turns=1)
    planned = dp.plan(cfg, trajs, policy="pe_only", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert xp.hit_bytes == 0 and len(xp.jobs()) == 0
    eng = dp.EngineRuntime(xp, 0, 0)
    eng.reset_counters()
    r = eng.run_step()
    assert r.bytes_read == 0 and r.jobs == 0


def test_edge_128k_context(gpus):
    """One 128K-token context (2048 Full Blocks per layer per request): the
    largest BASELINE config-2 request, loaded and checked block by block."""
    cfg = cluster(1, 1, L=2)
    t = dp.Trajectory()
    t.id = "long"
    t.rounds = [dp.Round(131071, 1), dp.Round(429, 1)]
    planned = dp.plan(cfg, [t], policy="pe_only", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    xp = dp.build_exec_plan(cfg, [t], planned, opt)
    jobs = xp.jobs()
    assert len(jobs) == 1 and jobs[0][6] == 131072 and jobs[0][7] == 2048
    eng = dp.EngineRuntime(xp, 0, 0)
    eng.reset_counters()
    r = eng.run_step()
    assert r.bytes_read == xp.hit_bytes == 131072 * 2 * 576
    verify_counters(eng, xp, cfg)
    verify_pool(eng, xp, cfg)


@pytest.mark.parametrize("tight", [False, True])
@pytest.mark.parametrize("scatter", [0, 1])
def test_staged_loaders(de_dev, tight, scatter):
    """k1_mode 3 / k2_mode 2: copy engine into the HBM ring + scatter kernel on
    both read paths, with a small ring (jobs span segments) and, tight, slot
    reuse across readers; final pool and counters equal the oracle's."""
    cfg = cluster(1, 1, L=4)
    trajs = small_trace(count=10, turns=6, seed=8)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.k1_mode, opt.k2_mode = 3, 2
    opt.stage_scatter = scatter
    opt.stage_ring_bytes = 24 * 4 * 64 * 576 * 4  # 24 Full Blocks per segment
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight:
        opt.pool_slots = xp.peak_slots
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    assert xp.reader_bytes[1] > 0
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    for _ in range(2):
        pe.reset_counters()
        res = dp.run_step_all([pe, de])
        assert res[0].bytes_read + res[1].bytes_read == xp.hit_bytes
        if scatter == 0:
            assert res[0].launches > 0 and res[1].launches > 0  # the scatter kernels
        verify_counters(pe, xp, cfg)
        verify_pool(pe, xp, cfg)


@pytest.mark.parametrize("k1", [0, 3])
def test_buffer_bound_stalls(de_dev, k1):
    """A host staging bound (pe_buffer_bytes / de_buffer_bytes, the reference's
    try_admit reservation) just above the largest request: the planner's
    admissions stall in virtual time, the executor's reads wait for earlier
    transfers to land (buffer_stalls > 0), and the pool is still exact."""
    cfg = cluster(1, 1, L=4)
    trajs = small_trace(count=8, turns=5, seed=5)
    kvt = cfg.kv_bytes_per_token()
    big = max(dp.context_before(t, len(t.rounds) - 1) + t.rounds[-1].append_tokens for t in trajs) * kvt
    cfg.pe_buffer_bytes = cfg.de_buffer_bytes = int(big * 1.5)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.k1_mode = k1
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    pe.reset_counters()
    res = dp.run_step_all([pe, de])
    assert res[0].buffer_stalls + res[1].buffer_stalls > 0
    verify_counters(pe, xp, cfg)
    verify_pool(pe, xp, cfg)


def test_persist_write_into_the_storage_tier(de_dev, tmp_path):
    """PersistWrite (desim.cpp:764-771): after the step every Full Block the
    DE's K4 persisted is written to its record of the storage-tier file, so a
    later turn's StorageRead from the tier reads the generated tokens back.
    The file starts with another seed's content: a persisted token range
    equals the oracle's content, everything else is untouched."""
    cfg = cluster(1, 1, L=3)
    trajs = small_trace(count=5, turns=3, seed=13)
    planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.handoff = True
    opt.persist = True
    probe = dp.build_exec_plan(cfg, trajs, planned, opt)
    T, b, L = cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer, cfg.n_layer
    path = str(tmp_path / "tier.bin")
    f = dp.FullBlockFile(path, L, T, b, probe.store_fb, create=True, direct=False)
    f.populate(SEED + 7, threads=4)
    del f
    opt.persist_path = path
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    rts = handoff_engines(xp, 2, [0, de_dev])
    for rt in rts:
        rt.reset_counters()
    res = dp.run_step_all(rts)
    assert res[1].persist_write_bytes > 0
    f = dp.FullBlockFile(path, L, T, b, xp.store_fb, create=False, direct=False)
    g = refpy.geom(L, T, b)
    fbb, lb = L * T * b, T * b
    persisted = {}
    for i, job in enumerate(xp.jobs()):
        traj, prompt, gen = job[1], job[14], xp.job_gen(i)
        for k in range(prompt // T, -(-(prompt + gen) // T)):
            a, z = max(prompt, k * T) - k * T, min(prompt + gen, (k + 1) * T) - k * T
            persisted.setdefault(xp.fb_of(traj, k), []).append((a, z))
    assert persisted
    for fb, ranges in persisted.items():
        rec = np.frombuffer(f.read(fb), dtype=np.uint8)[:fbb]
        other = refpy.fill_store(g, SEED + 7, 1, fb0=fb)
        want = refpy.fill_store(g, SEED, 1, fb0=fb)
        for layer in range(L):
            covered = np.zeros(T, dtype=bool)
            for a, z in ranges:
                covered[a:z] = True
                off = layer * lb
                assert np.array_equal(rec[off + a * b:off + z * b], want[off + a * b:off + z * b]), (fb, layer)
            for t in np.nonzero(~covered)[0]:  # never persisted: the file's own bytes
                off = layer * lb + t * b
                assert np.array_equal(rec[off:off + b], other[off:off + b]), (fb, layer, t)
