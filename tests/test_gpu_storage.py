"""GPU parity of the storage tier: StorageRead as real
file reads (FullBlockFile, trie lookups, pinned staging ring) feeding K1/K2.
The final PE pools must equal the oracle's content, as with the procedural
store."""

import numpy as np
import pytest

import paper_2602_21548_b200 as dp
from oracle import refpy

pytestmark = pytest.mark.gpu
SEED = 9
SB = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)


def cluster(P, D, L=4, b=576, T=64):
    c = dp.ClusterConfig()
    c.prefill_nodes, c.decode_nodes, c.engines_per_node = P, D, 1
    c.n_layer, c.kv_bytes_per_token_per_layer, c.block_size_tokens = L, b, T
    c.cnic_bandwidth, c.storage_multiple, c.dram_bandwidth = 50e9, 0.125, 500e9
    c.hbm_capacity_tokens, c.pe_buffer_bytes, c.de_buffer_bytes = 100_000_000, 1 << 42, 1 << 42
    return c


def make(tmp_path, P, D, policy, tight_ring, direct=True, threads=4):
    cfg = cluster(P, D)
    trajs = dp.synthesize(max_len=12000, count=8, seed=4, mean_turns=5, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy=policy, **SB)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.tier_path = str(tmp_path / "tier.bin")
    opt.io_threads = threads
    opt.tier_direct = direct
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    if tight_ring:
        opt.tier_ring_fb = max(j[7] for j in xp.jobs())
        xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    f = dp.FullBlockFile(opt.tier_path, cfg.n_layer, cfg.block_size_tokens,
                         cfg.kv_bytes_per_token_per_layer, xp.store_fb, create=True)
    f.populate(SEED, threads=4)
    return cfg, xp


def verify_pool(engine, xp, cfg):
    last = {}
    T = cfg.block_size_tokens
    for job in xp.jobs():
        if job[4] != engine.engine:
            continue
        # job[10] is the staging-ring position here; the page is fb_of
        for k, s in enumerate(job[9]):
            last[s] = (xp.fb_of(job[1], k), min(T, job[6] - T * k))
    slots = sorted(last)
    g = refpy.geom(cfg.n_layer, T, cfg.kv_bytes_per_token_per_layer)
    for layer in range(cfg.n_layer):
        got = engine.checksum(layer, slots, [last[s][1] for s in slots])
        want = [refpy.layer_block_hash(g, SEED, last[s][0], layer, last[s][1]) for s in slots]
        assert list(got) == want, f"pool mismatch on PE {engine.engine} layer {layer}"


@pytest.mark.parametrize("tight_ring,direct", [(False, True), (True, True), (True, False)])
def test_tier_single_pe(gpus, tmp_path, tight_ring, direct):
    cfg, xp = make(tmp_path, 1, 1, "pe_only", tight_ring, direct)
    assert xp.tier
    eng = dp.EngineRuntime(xp, 0, 0)
    for _ in range(2):
        eng.reset_counters()
        r = eng.run_step()
        assert r.bytes_read == xp.hit_bytes
    verify_pool(eng, xp, cfg)


@pytest.mark.parametrize("tight_ring", [False, True])
def test_tier_1p1d_dual_path(de_dev, tmp_path, tight_ring):
    cfg, xp = make(tmp_path, 1, 1, "dual_path", tight_ring)
    assert xp.reader_bytes[1] > 0
    pe = dp.EngineRuntime(xp, 0, 0)
    de = dp.EngineRuntime(xp, 1, de_dev)
    de.attach_peer_local(0, pe)
    for _ in range(2):
        pe.reset_counters()
        res = dp.run_step_all([pe, de])
        assert res[0].bytes_read + res[1].bytes_read == xp.hit_bytes
    verify_pool(pe, xp, cfg)


def test_tier_missing_file_fails_loudly(gpus, tmp_path):
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=12000, count=2, seed=4, mean_turns=3, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="pe_only", **SB)
    opt = dp.ExecOptions()
    opt.tier_path = str(tmp_path / "absent.bin")
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    with pytest.raises(RuntimeError):
        dp.EngineRuntime(xp, 0, 0)


def test_tier_with_prefill(gpus, tmp_path):
    """StorageRead from the file feeding the quota-batched forwards: the K5
    digests equal the oracle's (a tight ring: reads wait on earlier loads)."""
    from test_gpu_prefill import check_digests, COST
    cfg = cluster(1, 1)
    trajs = dp.synthesize(max_len=12000, count=8, seed=4, mean_turns=5, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy="pe_only", **SB)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.tier_path = str(tmp_path / "tier.bin")
    opt.io_threads = 4
    opt.prefill, opt.compute_quota, opt.prefill_cost = True, 5e-4, COST
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    opt.tier_ring_fb = max(j[7] for j in xp.jobs())
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    f = dp.FullBlockFile(opt.tier_path, cfg.n_layer, cfg.block_size_tokens,
                         cfg.kv_bytes_per_token_per_layer, xp.store_fb, create=True)
    f.populate(SEED, threads=4)
    eng = dp.EngineRuntime(xp, 0, 0)
    for _ in range(2):
        eng.reset_counters()
        r = eng.run_step()
        assert r.forwards == len(xp.forwards(0)) and r.bytes_read == xp.hit_bytes
        check_digests(eng, cfg, planned, xp)
