"""N > 1 host logic on CPU with the gloo backend (world size 2): every rank
plans independently and agrees on the decisions, each rank's reader share
partitions the jobs, and the pool-handle exchange reaches every DE."""

import os
import socket

import pytest
import torch.multiprocessing as mp

import paper_2602_21548_b200 as dp
from paper_2602_21548_b200 import dist

SB = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class FakeRuntime:
    """Stands in for EngineRuntime: the handle protocol only (IPC needs GPUs)."""

    def __init__(self, engine):
        self.engine = engine
        self.attached = {}

    def export_pool(self):
        return bytes([self.engine]) * 128

    def attach_peer(self, pe, handle):
        self.attached[pe] = handle


def worker(rank, world, port, P, policy, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    g = dist.Group("gloo")
    try:
        cfg = dp.ClusterConfig()
        cfg.prefill_nodes, cfg.decode_nodes, cfg.engines_per_node = P, world - P, 1
        cfg.n_layer, cfg.kv_bytes_per_token_per_layer = 8, 576
        cfg.cnic_bandwidth, cfg.storage_multiple = 50e9, 0.125
        cfg.hbm_capacity_tokens, cfg.pe_buffer_bytes, cfg.de_buffer_bytes = 10**8, 1 << 42, 1 << 42
        trajs = dp.synthesize(max_len=20000, count=10, seed=5, mean_turns=5, sigma_turns=0)
        planned = dp.plan(cfg, trajs, policy=policy, **SB)
        xp = dp.build_exec_plan(cfg, trajs, planned, dp.ExecOptions())
        digests = g.allgather(dist.plan_digest(planned))
        # the full pipeline's plan (forwards, DE orders) is the same on every rank
        opt = dp.ExecOptions()
        opt.handoff = opt.persist = opt.prefill = True
        opt.compute_quota, opt.prefill_cost = 1e-3, (2e-10, 1e-9, 4e-7, 1e-5)
        full = dp.build_exec_plan(cfg, trajs, planned, opt)
        shape = repr([full.forwards(p) for p in range(P)] +
                     [full.de_order(d) for d in range(P, world)])
        pipeline = g.allgather(shape)
        mine = sorted(xp.jobs()[i][0] for i in xp.by_reader(rank))
        shares = g.allgather(mine)
        rt = {rank: FakeRuntime(rank)}
        table = dist.connect_pools(g, rt, P)
        t = g.max(float(rank))
        q.put((rank, digests, shares, sorted(j[0] for j in xp.jobs()), xp.reader_bytes,
               sorted(rt[rank].attached), sorted(table), t, len(set(pipeline))))
    finally:
        g.close()


@pytest.mark.parametrize("P,policy", [(1, "dual_path"), (1, "pe_only")])
def test_two_rank_plan_agreement_and_partition(P, policy):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, P, policy, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        r = q.get(timeout=120)
        out[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = out[0], out[1]
    assert len(set(r0[1])) == 1 and r0[1] == r1[1]          # same decisions on both ranks
    all_jobs = r0[3]
    shares = r0[2]
    assert sorted(shares[0] + shares[1]) == all_jobs         # readers partition the jobs
    if policy == "pe_only":
        assert shares[1] == []
    else:
        assert shares[1], "the DE rank should read its share"
    assert r1[5] == [0] and r0[5] == []                      # the DE attached the PE pool
    assert r0[6] == [0] and r0[7] == 1.0                     # handle table, max over ranks
    assert r0[8] == r1[8] == 1                               # same forwards and DE orders


def test_roles():
    assert dist.roles(8, 4) == ["pe"] * 4 + ["de"] * 4
    assert dist.roles(8, 1) == ["pe"] + ["de"] * 7
