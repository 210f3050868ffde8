"""The storage tier: Full Block trie index, Full Block
file records, and the executor plan's staging ring (CPU).

Record contents are checked against the oracle's content formula
(oracle/kvref.c kvref_fill_store): record r of the file is page r."""

import os

import numpy as np
import pytest

import paper_2602_21548_b200 as dp
from oracle import refpy

SB = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)


def test_session_chain_is_a_prefix_key():
    a = dp.session_chain("s1", 6)
    assert a[:3] == dp.session_chain("s1", 3)
    assert len(set(a)) == 6
    assert dp.session_chain("s2", 6)[0] != a[0]
    assert dp.session_chain("s1", 0) == []


def test_trie_shares_prefixes_and_matches_longest():
    t = dp.FullBlockTrie()
    c1 = [11, 12, 13, 14]
    c2 = [11, 12, 99]
    assert t.insert(c1, [100, 101, 102, 103]) == [100, 101, 102, 103]
    # the shared prefix keeps its records; only the new node takes one
    assert t.insert(c2, [7, 7, 104]) == [100, 101, 104]
    assert t.nodes() == 5
    assert t.match([11, 12, 13]) == [100, 101, 102]
    assert t.match([11, 12, 99, 5]) == [100, 101, 104]
    assert t.match([12]) == []
    assert t.match([]) == []


def test_trie_save_load_round_trip(tmp_path):
    t = dp.FullBlockTrie()
    for s in range(5):
        ch = dp.session_chain(f"sess{s}", 3 + s)
        t.insert(ch, list(range(100 * s, 100 * s + len(ch))))
    p = str(tmp_path / "index.trie")
    t.save(p)
    u = dp.FullBlockTrie.load(p)
    assert u.nodes() == t.nodes()
    for s in range(5):
        ch = dp.session_chain(f"sess{s}", 3 + s)
        assert u.match(ch) == t.match(ch) == list(range(100 * s, 100 * s + len(ch)))
    bad = tmp_path / "bad.trie"
    bad.write_bytes(b"not a trie index at all")
    with pytest.raises(RuntimeError):
        dp.FullBlockTrie.load(str(bad))


@pytest.mark.parametrize("L,T,b", [(61, 64, 576), (3, 16, 64), (2, 64, 4096)])
def test_full_block_file_records_match_the_oracle(tmp_path, L, T, b):
    p = str(tmp_path / "fb.bin")
    n = 6
    f = dp.FullBlockFile(p, L, T, b, n, create=True)
    assert f.record_bytes() == L * T * b and f.stride() % 4096 == 0 and f.stride() >= f.record_bytes()
    f.populate(9, threads=3)
    g = refpy.geom(L, T, b)
    for r in (0, 3, n - 1):
        assert f.read(r) == refpy.fill_store(g, 9, 1, fb0=r).tobytes()
    assert os.path.getsize(p) == n * f.stride()
    with pytest.raises(IndexError):
        f.read(n)
    # runs of consecutive records: one read when records are packed
    assert f.read_run(1, 4) == b"".join(f.read(r) for r in range(1, 5))
    with pytest.raises(IndexError):
        f.read_run(n - 2, 3)
    # reopen read-only; asking for more records than the file holds fails
    assert dp.FullBlockFile(p, L, T, b, n).read(2) == f.read(2)
    with pytest.raises(RuntimeError):
        dp.FullBlockFile(p, L, T, b, n + 1)


def cluster(P, D, L=4, b=576, T=64):
    c = dp.ClusterConfig()
    c.prefill_nodes, c.decode_nodes, c.engines_per_node = P, D, 1
    c.n_layer, c.kv_bytes_per_token_per_layer, c.block_size_tokens = L, b, T
    c.cnic_bandwidth, c.storage_multiple, c.dram_bandwidth = 50e9, 0.125, 500e9
    c.hbm_capacity_tokens, c.pe_buffer_bytes, c.de_buffer_bytes = 100_000_000, 1 << 42, 1 << 42
    return c


def tier_plan(P, D, ring=0, path="/nonexistent/tier.bin", policy="dual_path"):
    cfg = cluster(P, D)
    trajs = dp.synthesize(max_len=12000, count=8, seed=4, mean_turns=5, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy=policy, **SB)
    opt = dp.ExecOptions()
    opt.tier_path = path
    opt.tier_ring_fb = ring
    return cfg, trajs, planned, dp.build_exec_plan(cfg, trajs, planned, opt)


@pytest.mark.parametrize("P,D,ring", [(1, 1, 0), (2, 2, 0), (1, 1, -1)])
def test_tier_plan_stages_through_a_ring(P, D, ring):
    if ring == -1:  # a ring just big enough for the largest job: reuse everywhere
        _, _, _, probe = tier_plan(P, D)
        ring = max(j[7] for j in probe.jobs())
    cfg, trajs, planned, xp = tier_plan(P, D, ring)
    assert xp.tier and xp.ring_fb >= max(j[7] for j in xp.jobs())
    jobs = xp.jobs()
    n_waits = 0
    for e in range(xp.n_engines):
        src, rec = xp.src_fb(e), xp.tier_rec(e)
        assert len(src) == len(rec)
        owner = {}
        for ji in xp.by_reader(e):
            j = jobs[ji]
            traj, nblk = j[1], j[7]
            # the job's records are what the trie holds for its session: the
            # procedural store's pages, so the bytes are the same
            k0 = sum(jobs[k][7] for k in xp.by_reader(e)[:xp.by_reader(e).index(ji)])
            assert rec[k0:k0 + nblk] == [xp.fb_of(traj, k) for k in range(nblk)]
            pos = src[k0:k0 + nblk]
            assert all(0 <= p < xp.ring_fb for p in pos) and len(set(pos)) == nblk
            want = sorted({owner[p] for p in pos if p in owner})
            assert sorted(xp.ring_waits(ji)) == want
            n_waits += len(want)
            for p in pos:
                owner[p] = ji
    trie_nodes = sum(dp.blocks_for(t.total_tokens(), cfg) for t in trajs)
    assert xp.trie_nodes == trie_nodes
    if ring and ring == max(j[7] for j in jobs):
        assert n_waits > 0


def test_tier_plan_rejects_bad_configs():
    with pytest.raises(ValueError):
        tier_plan(1, 1, ring=3)
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=12000, count=4, seed=4, mean_turns=4, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="dual_path", **SB)
    opt = dp.ExecOptions()
    opt.tier_path = "/x"
    opt.handoff = True
    with pytest.raises(ValueError):
        dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.handoff, opt.prefill = False, True  # the tier feeds the prefill path
    assert dp.build_exec_plan(cfg, trajs, planned, opt).tier
