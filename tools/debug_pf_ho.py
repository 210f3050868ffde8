#!/usr/bin/env python
"""Debug: handoff + prefill digests on 2 GPUs, per-row report."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2602_21548_b200 as dp  # noqa: E402
from oracle import refpy  # noqa: E402
from test_gpu_prefill import cluster, expected_digests, STORAGE_BOUND, COST, SEED  # noqa: E402
from test_gpu_engine import handoff_engines  # noqa: E402


def run(handoff, policy, steps=2):
    cfg = cluster(1, 1, L=4)
    trajs = dp.synthesize(max_len=12000, count=8, seed=6, mean_turns=5, sigma_turns=0)
    planned = dp.plan(cfg, trajs, policy=policy, **STORAGE_BOUND)
    opt = dp.ExecOptions()
    opt.seed = SEED
    opt.handoff = handoff
    opt.prefill = True
    opt.compute_quota = 5e-4
    opt.prefill_cost = COST
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    rts = handoff_engines(xp, 2) if handoff else [dp.EngineRuntime(xp, 0, 0), dp.EngineRuntime(xp, 1, 1)]
    if not handoff:
        rts[1].attach_peer_local(0, rts[0])
    want = expected_digests(cfg, planned, xp, 0)
    reqs = {r[0]: r for r in planned["requests"]}
    jobs = xp.jobs()
    fwd_of = {}
    for fi, (_, items) in enumerate(xp.forwards(0)):
        for it in items:
            fwd_of.setdefault(it[5], []).append(fi)
    for step in range(steps):
        for rt in rts:
            rt.reset_counters()
        dp.run_step_all(rts)
        got = np.asarray(rts[0].prefill_digests(), dtype=np.uint64).reshape(-1, cfg.n_layer)
        bad = [row for row in range(len(want)) if [int(v) for v in got[row]] != want[row]]
        print(f"handoff={handoff} policy={policy} step={step}: {len(bad)} bad rows of {len(want)}")
        for row in bad[:6]:
            rid = xp.fwd_rows(0)[row]
            r = reqs[rid]
            job = [i for i, j in enumerate(jobs) if j[0] == rid]
            j = jobs[job[0]] if job else None
            print(f"  row {row} req {rid} C={r[3]} A={r[4]} path={'DE' if j and j[5] else 'PE'} "
                  f"job={job} fwds={fwd_of.get(row)} last_fwd={xp.last_fwd(job[0]) if job else None}")
            print("    got ", [int(v) for v in got[row]])
            print("    want", want[row])
    # the compute alone afterwards, over the pool as the step left it
    rts[0].run_forwards()
    got = np.asarray(rts[0].prefill_digests(), dtype=np.uint64).reshape(-1, cfg.n_layer)
    bad = [row for row in range(len(want)) if [int(v) for v in got[row]] != want[row]]
    print(f"  run_forwards after the step: {len(bad)} bad rows {bad[:12]}")
    # pool content of the bad rows' hit blocks after the step
    g = refpy.geom(cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer)
    T = cfg.block_size_tokens
    for row in bad[:3]:
        rid = xp.fwd_rows(0)[row]
        j = [jj for jj in jobs if jj[0] == rid][0]
        slots = j[9]
        ntok = [min(T, j[6] - T * k) for k in range(len(slots))]
        for layer in range(cfg.n_layer):
            gotc = list(rts[0].checksum(layer, slots, ntok))
            wantc = [refpy.layer_block_hash(g, SEED, xp.fb_of(j[1], k), layer, ntok[k]) for k in range(len(slots))]
            print(f"    row {row} layer {layer}: {sum(a != b for a, b in zip(gotc, wantc))} of {len(slots)} blocks differ; slots {slots}")


if __name__ == "__main__":
    run(True, "pe_only", steps=1)
