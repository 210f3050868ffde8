"""Live-mode scheduling (include/dualpath/live.hpp): the
reference's scheduler glue driven by measured completions.  Every scheduler
invocation's inputs and outputs are logged; each is replayed through the
REFERENCE's own functions (oracle/_ref: schedule_de_groups,
schedule_de_within_group, schedule_pe_fetch, select_read_path) and must agree
bit for bit.  Host tests use the timed backend (transfers sleep bytes /
rate); the GPU tests move the bytes with K1 / K2 and check the final pools
against the content oracle."""

import numpy as np
import pytest

import paper_2602_21548_b200 as dp
from oracle import refpy

needs_ref = pytest.mark.skipif(not refpy.ref_available(), reason="oracle/_ref not built")


def cluster(P, D, L=4, b=576, T=64, hbm=100_000_000):
    cfg = dp.ClusterConfig()
    cfg.prefill_nodes, cfg.decode_nodes, cfg.engines_per_node = P, D, 1
    cfg.n_layer, cfg.kv_bytes_per_token_per_layer, cfg.block_size_tokens = L, b, T
    cfg.hbm_capacity_tokens = hbm
    return cfg


def replay(rep, alpha, beta, z=1.05):
    """Every logged invocation through the reference's function."""
    n = 0
    for inv in rep["invocations"]:
        fn = inv["fn"]
        q = [tuple(x) for x in inv["queue"]]
        snaps = [(s[0], s[1], s[3], s[4], s[5], s[6]) for s in inv["snapshots"]]
        got = [tuple(x) for x in inv["out"]]
        if fn == "schedule_de_groups":
            want = refpy.ref_schedule_de_groups(q, [tuple(g) for g in inv["groups"]])
            assert [(r, g) for r, g, _ in got] == want, inv
        elif fn == "schedule_de_within_group":
            assert got == refpy.ref_schedule("ref_schedule_de_within_group", q, snaps, alpha, beta, z), inv
        elif fn == "schedule_pe_fetch":
            assert got == refpy.ref_schedule("ref_schedule_pe_fetch", q, snaps, alpha, beta, z), inv
        elif fn == "select_read_path":
            assert inv["path"] == refpy.ref().ref_select_read_path(inv["pe_read_q"], inv["de_read_q"]), inv
        else:
            raise AssertionError(fn)
        n += 1
    return n


def check_lifecycle(rep, trajs, prefill=False, gpu=False):
    reqs = rep["requests"]
    assert len(reqs) == sum(len(t.rounds) for t in trajs)
    assert len(rep["decisions"]) == len(reqs)
    by_traj = {}
    for r in reqs:
        rid, traj, rnd, C, A, G, pe, de, path, reader, t_arr, t_sched, t_admit, t_read, t_land, t_done = r[:16]
        t_pref, n_fwd = r[16:18]
        assert 0 <= t_arr <= t_sched <= t_admit <= t_read <= t_land <= t_done
        if prefill:  # the PE release after its last forward, before the turn completes
            assert n_fwd >= 1 and t_admit <= t_pref <= t_done
            if not gpu:
                assert t_land <= t_pref
        else:
            assert t_pref == -1 and n_fwd == 0
        assert reader == (pe if path == 0 else de)
        by_traj.setdefault(traj, []).append((rnd, t_arr, t_done))
    for turns in by_traj.values():  # a session's next turn arrives after the previous completes
        turns.sort()
        for (r0, _, done), (r1, arr, _) in zip(turns, turns[1:]):
            assert r1 == r0 + 1 and arr >= done


@needs_ref
@pytest.mark.parametrize("P,D,policy,mode,cap,slots", [
    (1, 1, "dual_path", "adaptive", 2e9, 0),
    (2, 2, "dual_path", "adaptive", 1e9, 0),
    (1, 3, "dual_path", "adaptive", 4e9, 0),
    (2, 2, "pe_only", "adaptive", 1e9, 0),
    (2, 2, "dual_path", "round_robin", 1e9, 0),
    (2, 2, "dual_path", "adaptive", 1e9, "tight"),
])
def test_live_invocations_replay_through_the_reference(P, D, policy, mode, cap, slots):
    trajs = dp.synthesize(max_len=16000, count=4 * (P + D), seed=11, mean_turns=5, sigma_turns=0)
    cfg = cluster(P, D, hbm=60_000)  # DE HBM bound: phase 2 leaves requests queued
    ex = dp.ExecOptions()
    ex.storage_cap_Bps = cap
    big = max(-(-dp.context_before(t, len(t.rounds) - 1) // 64) for t in trajs)
    rep = dp.run_live(cfg, trajs, policy=policy, sched_mode=mode, alpha=20000, beta=60000, exec=ex,
                      gpu=False, link_Bps=8e9, decode_s_per_token=2e-6,
                      pe_pool_slots=big if slots == "tight" else 0)
    check_lifecycle(rep, trajs)
    n = replay(rep, 20000, 60000)
    assert n >= len(rep["decisions"]) if mode == "adaptive" else n == 0
    if policy == "pe_only":
        assert all(d[4] == 0 for d in rep["decisions"])
    if policy == "dual_path" and mode == "adaptive" and P == 2:
        assert any(d[4] == 1 for d in rep["decisions"])   # both read paths used
    if slots == "tight":
        assert rep["admission_stalls"] > 0                 # the bounded pool made requests wait
    assert sum(rep["reader_bytes"]) == sum(r[3] for r in rep["requests"]) * cfg.kv_bytes_per_token()


def test_live_rejects_a_pool_smaller_than_a_request():
    trajs = dp.synthesize(max_len=16000, count=2, seed=1, mean_turns=4, sigma_turns=0)
    with pytest.raises(dp.ConfigError):
        dp.run_live(cluster(1, 1), trajs, gpu=False, pe_pool_slots=1)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("k1,k2,tight", [(0, 0, False), (3, 2, True)])
def test_live_gpu_moves_the_bytes(de_dev, k1, k2, tight):
    """1P1D live on the GPU: K1 / K2 (or staged) move every request's hit KV
    into the PE pool; the final occupant of every slot matches the oracle's
    content and the invocations replay through the reference."""
    trajs = dp.synthesize(max_len=12000, count=6, seed=4, mean_turns=5, sigma_turns=0)
    cfg = cluster(1, 1)
    ex = dp.ExecOptions()
    ex.seed = 9
    ex.storage_cap_Bps = 4e9
    ex.k1_mode, ex.k2_mode = k1, k2
    big = max(-(-dp.context_before(t, len(t.rounds) - 1) // 64) for t in trajs)
    rep = dp.run_live(cfg, trajs, exec=ex, devices=[0, de_dev], pe_pool_slots=big + 4 if tight else 0,
                      alpha=20000, beta=60000)
    check_lifecycle(rep, trajs)
    replay(rep, 20000, 60000)
    assert rep["reader_bytes"][1] > 0
    g = refpy.geom(cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer)
    assert rep["final_slots"]
    for pe, slot, fb, ntok, h0, h1 in rep["final_slots"]:
        assert h0 == refpy.layer_block_hash(g, 9, fb, 0, ntok)
        assert h1 == refpy.layer_block_hash(g, 9, fb, cfg.n_layer - 1, ntok)


def test_live_online_slo_stop_and_arrivals():
    """Online: sessions arrive at given times (run_online's Poisson arrivals,
    desim.cpp:1036-1051); a turn's measured load TTFT over the SLO stops the
    run (desim.cpp:679-685), a generous SLO lets it finish."""
    trajs = dp.synthesize(max_len=16000, count=12, seed=3, mean_turns=4, sigma_turns=0)
    rng = np.random.default_rng(5)
    arrivals = list(np.cumsum(rng.exponential(1 / 400.0, len(trajs))))  # 400 sessions/s
    ex = dp.ExecOptions()
    ex.storage_cap_Bps = 1e9
    ok = dp.run_live(cluster(1, 1), trajs, exec=ex, gpu=False, link_Bps=8e9, arrival_times=arrivals,
                     slo_ttft=10.0)
    assert not ok["slo_violated"] and ok["completed_requests"] == ok["total_requests"]
    first = {}
    for r in ok["requests"]:
        if r[2] == 0:
            first[r[1]] = r[10]
    for t, a in enumerate(arrivals):
        assert first[t] >= a - 1e-4  # no session arrives before its time
    tight = dp.run_live(cluster(1, 1), trajs, exec=ex, gpu=False, link_Bps=8e9, arrival_times=arrivals,
                        slo_ttft=1e-4)
    assert tight["slo_violated"] and tight["completed_requests"] < tight["total_requests"]
    steady = dp.run_live(cluster(1, 1), trajs, exec=ex, gpu=False, link_Bps=8e9, arrival_times=arrivals,
                         steady_window=0.002, steady_lookback=0.01, steady_threshold=0.9)
    assert steady["steady_state"] or steady["completed_requests"] == steady["total_requests"]


def prefill_exec(quota_s=2e-4, tops=2e12):
    """exec options of the live prefill stand-in: forwards under a compute
    quota of quota_s per layer, cost model b / tops per (query, key) token."""
    ex = dp.ExecOptions()
    ex.prefill = True
    ex.compute_quota = quota_s
    ex.prefill_cost = (576 / tops, 0.0, 0.0, 2e-6)
    return ex


@needs_ref
@pytest.mark.parametrize("P,D,policy", [(1, 1, "dual_path"), (2, 2, "dual_path"), (2, 2, "pe_only")])
def test_live_prefill_timed(P, D, policy):
    """Live mode with the prefill stand-in (timed backend): each PE packs its
    landed requests into quota-bounded forwards, the PE is released after a
    request's last forward (so tok_e / seq_e cover prefill, as the
    reference's on_prefill_side_done), TTFT = arrival -> prefill done, and
    every scheduler invocation still replays through the reference."""
    trajs = dp.synthesize(max_len=16000, count=4 * (P + D), seed=12, mean_turns=4, sigma_turns=0)
    ex = prefill_exec()
    ex.storage_cap_Bps = 2e9
    rep = dp.run_live(cluster(P, D), trajs, policy=policy, alpha=20000, beta=60000, exec=ex, gpu=False,
                      link_Bps=8e9, decode_s_per_token=2e-6)
    check_lifecycle(rep, trajs, prefill=True)
    replay(rep, 20000, 60000)
    assert rep["forwards"] >= 1
    assert any(r[17] > 1 for r in rep["requests"]) or rep["forwards"] < len(rep["requests"])
    for (t, ttft), r in zip(sorted(rep["ttft_series"]), sorted(rep["requests"], key=lambda r: r[16])):
        assert abs(t - r[16]) < 1e-9 and abs(ttft - (r[16] - r[10])) < 1e-9


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("k1,k2", [(0, 0), (3, 2)])
def test_live_prefill_gpu_digests(de_dev, k1, k2):
    """Live prefill on the GPU: K5 forwards, gated per layer on the landed
    counters of the loads the scheduler launched, read every request's hit KV
    from the PE pool; each request's digest (layers 0 and L-1) equals the
    oracle's for its full query range, whatever the batching was."""
    trajs = dp.synthesize(max_len=12000, count=6, seed=4, mean_turns=4, sigma_turns=0)
    cfg = cluster(1, 1)
    ex = prefill_exec()
    ex.seed = 9
    ex.storage_cap_Bps = 4e9
    ex.k1_mode, ex.k2_mode = k1, k2
    rep = dp.run_live(cfg, trajs, exec=ex, devices=[0, de_dev], alpha=20000, beta=60000)
    check_lifecycle(rep, trajs, prefill=True, gpu=True)
    replay(rep, 20000, 60000)
    g = refpy.geom(cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer)
    reqs = {r[0]: r for r in rep["requests"]}
    assert len(rep["digests"]) == len(reqs)
    stride, n_fb, T, L = rep["fb_stride"], rep["store_fb"], cfg.block_size_tokens, cfg.n_layer
    for rid, d0, d1 in rep["digests"]:
        r = reqs[rid]
        traj, C, A = r[1], r[3], r[4]
        fbs = [(traj * stride + k) % n_fb for k in range(-(-C // T))]
        for layer, d in ((0, d0), (L - 1, d1)):
            assert d == (refpy.attend_digest(g, 9, fbs, C, rid, layer, 0, A) if C and A else 0), (rid, layer)


@needs_ref
@pytest.mark.parametrize("P,D", [(1, 1), (2, 2)])
def test_live_handoff_timed(P, D):
    """Live mode with prefill + PD handoff (timed backend): admission also
    reserves the prompt's decode-pool slots (a tight decode pool stalls it),
    the PE releases a request after its K3, and its TTFT includes one decode
    step after the prompt reached the decode pool."""
    trajs = dp.synthesize(max_len=16000, count=4 * (P + D), seed=13, mean_turns=4, sigma_turns=0)
    ex = prefill_exec()
    ex.handoff = True
    ex.storage_cap_Bps = 2e9
    big = max(-(-(dp.context_before(t, k) + t.rounds[k].append_tokens) // 64)
              for t in trajs for k in range(len(t.rounds)))
    rep = dp.run_live(cluster(P, D), trajs, alpha=20000, beta=60000, exec=ex, gpu=False, link_Bps=8e9,
                      decode_s_per_token=2e-6, de_pool_slots=big + 2)
    check_lifecycle(rep, trajs, prefill=True)
    replay(rep, 20000, 60000)
    assert rep["admission_stalls"] > 0  # the decode pool held requests back
    ttfts = sorted(x[1] for x in rep["ttft_series"])
    firsts = sorted(r[16] + 2e-6 - r[10] for r in rep["requests"])
    assert all(abs(a - b) < 1e-9 for a, b in zip(ttfts, firsts))


def test_live_handoff_needs_prefill():
    trajs = dp.synthesize(max_len=8000, count=2, seed=1, mean_turns=2, sigma_turns=0)
    ex = dp.ExecOptions()
    ex.handoff = True
    with pytest.raises(ValueError):
        dp.run_live(cluster(1, 1), trajs, exec=ex, gpu=False)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("k1,k2,k3", [(0, 0, 0), (3, 2, 1)])
def test_live_handoff_gpu(de_dev, k1, k2, k3):
    """Live prefill + handoff on the GPU: the DE read path is the dual gather,
    K3 (SM kernel or copy engines) moves each finished prompt into its DE's
    decode pool; the final occupant of every PE and decode-pool slot holds
    the whole prompt block the oracle says, and every digest matches."""
    trajs = dp.synthesize(max_len=12000, count=6, seed=4, mean_turns=4, sigma_turns=0)
    cfg = cluster(1, 1)
    ex = prefill_exec()
    ex.handoff = True
    ex.seed = 9
    ex.storage_cap_Bps = 4e9
    ex.k1_mode, ex.k2_mode, ex.k3_mode = k1, k2, k3
    rep = dp.run_live(cfg, trajs, exec=ex, devices=[0, de_dev], alpha=20000, beta=60000)
    check_lifecycle(rep, trajs, prefill=True, gpu=True)
    replay(rep, 20000, 60000)
    assert any(r[8] == 1 for r in rep["requests"]) or rep["reader_bytes"][1] == 0
    g = refpy.geom(cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer)
    assert rep["final_slots"] and rep["final_decode_slots"]
    for slots in (rep["final_slots"], rep["final_decode_slots"]):
        for eng, slot, fb, ntok, h0, h1 in slots:
            assert h0 == refpy.layer_block_hash(g, 9, fb, 0, ntok), (eng, slot)
            assert h1 == refpy.layer_block_hash(g, 9, fb, cfg.n_layer - 1, ntok), (eng, slot)
    reqs = {r[0]: r for r in rep["requests"]}
    stride, n_fb, T, L = rep["fb_stride"], rep["store_fb"], cfg.block_size_tokens, cfg.n_layer
    for rid, d0, d1 in rep["digests"]:
        r = reqs[rid]
        fbs = [(r[1] * stride + k) % n_fb for k in range(-(-r[3] // T))]
        for layer, d in ((0, d0), (L - 1, d1)):
            assert d == (refpy.attend_digest(g, 9, fbs, r[3], rid, layer, 0, r[4]) if r[3] and r[4] else 0)


def range_hash(words):
    """dp_pool_checksum's hash over a range of 64-bit words (restated)."""
    golden = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = words + np.arange(1, len(words) + 1, dtype=np.uint64) * golden + golden
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return int(z.sum(dtype=np.uint64))


@needs_ref
def test_live_persist_timed():
    """Live prefill + handoff + persistence (timed backend): every request
    completes, the decode pool holds prompt + generated blocks until the
    request is persisted, and the invocations replay through the reference."""
    trajs = dp.synthesize(max_len=16000, count=8, seed=14, mean_turns=4, sigma_turns=0)
    ex = prefill_exec()
    ex.handoff = ex.persist = True
    ex.storage_cap_Bps = 2e9
    rep = dp.run_live(cluster(1, 1), trajs, alpha=20000, beta=60000, exec=ex, gpu=False, link_Bps=8e9,
                      decode_s_per_token=2e-6)
    check_lifecycle(rep, trajs, prefill=True)
    replay(rep, 20000, 60000)
    assert rep["completed_requests"] == rep["total_requests"]


def test_live_persist_needs_handoff():
    trajs = dp.synthesize(max_len=8000, count=2, seed=1, mean_turns=2, sigma_turns=0)
    ex = prefill_exec()
    ex.persist = True
    with pytest.raises(ValueError):
        dp.run_live(cluster(1, 1), trajs, exec=ex, gpu=False)


@pytest.mark.gpu
@needs_ref
def test_live_persist_gpu(de_dev, tmp_path):
    """Live mode with persistence on the GPU: each request's generated tokens
    (decode stand-in) are persisted by staged K4 into its DE's persist store
    and written into the storage-tier file (PersistWrite); every persisted
    range of layers 0 and L-1 equals the content oracle (in the store and in
    the file), and the decode pools' last occupants hold prompt + generated
    tokens."""
    trajs = dp.synthesize(max_len=12000, count=5, seed=5, mean_turns=4, sigma_turns=0)
    cfg = cluster(1, 1)
    T, b, L = cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer, cfg.n_layer
    ex = prefill_exec()
    ex.handoff = ex.persist = True
    ex.seed = 9
    ex.storage_cap_Bps = 4e9
    ex.k1_mode, ex.k2_mode = 3, 2
    n_rec = max(-(-t.total_tokens() // T) for t in trajs) * len(trajs)  # = the live store's Full Blocks
    path = str(tmp_path / "tier.bin")
    f = dp.FullBlockFile(path, L, T, b, n_rec, create=True, direct=False)
    f.populate(9 + 7, threads=4)
    del f
    ex.persist_path = path
    rep = dp.run_live(cfg, trajs, exec=ex, devices=[0, de_dev], alpha=20000, beta=60000, decode_s_per_token=1e-5)
    assert rep["persist_write_bytes"] == sum(r[5] for r in rep["requests"]) * L * b
    f = dp.FullBlockFile(path, L, T, b, n_rec, create=False, direct=False)
    for rid, fb, layer, t0, t1, h in rep["persisted"]:
        rec = np.frombuffer(f.read(fb), dtype=np.uint8)
        assert h == range_hash(rec[layer * T * b + t0 * b:layer * T * b + t1 * b].copy().view(np.uint64)), (rid, fb)
    check_lifecycle(rep, trajs, prefill=True, gpu=True)
    replay(rep, 20000, 60000)
    T, b = cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer
    g = refpy.geom(cfg.n_layer, T, b)
    reqs = {r[0]: r for r in rep["requests"]}
    want_tokens = sum(2 * r[5] for r in rep["requests"])  # layers 0 and L-1
    assert sum(t1 - t0 for _, _, _, t0, t1, _ in rep["persisted"]) == want_tokens
    for rid, fb, layer, t0, t1, h in rep["persisted"]:
        full = refpy.layer_block(g, 9, fb, layer, T)
        assert h == range_hash(full[t0 * b:t1 * b].view(np.uint64)), (rid, fb, layer, t0, t1)
    for eng, slot, fb, ntok, h0, h1 in rep["final_decode_slots"]:
        assert h0 == refpy.layer_block_hash(g, 9, fb, 0, ntok), (eng, slot)
        assert h1 == refpy.layer_block_hash(g, 9, fb, cfg.n_layer - 1, ntok), (eng, slot)
    assert len(reqs) == rep["total_requests"]
