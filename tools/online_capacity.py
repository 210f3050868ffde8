#!/usr/bin/env python
"""BASELINE config 5 / the paper's online metric on the GPU path: the APS
capacity (most sessions per second the system serves within the TTFT SLO)
of dual path vs 1-path, measured with live-mode scheduling
(dualpath::run_live: the reference's scheduler on measured completions, K1 /
K2 moving the bytes, every engine's storage NIC capped).

Sessions arrive as a Poisson process (run_online's arrivals,
/root/reference/proj/src/desim.cpp:1036-1051); a session's next turn arrives
when its previous turn completes (its KV landed, then gen x decode_s of
emulated decode).  A run stops on the first turn whose measured load TTFT
(arrival -> hit KV landed in the PE pool) exceeds the SLO (desim.cpp:679-685)
or when the TTFT series is steady (detect_steady_state, desim.cpp:942-953);
the capacity is the largest APS of a geometric bisection that never
violates.  Prints one JSON object.

    python tools/online_capacity.py [--pd 1:1] [--cap-gbps 6.25] [--slo 2.0] [--cpu]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2602_21548_b200 as dp  # noqa: E402


def pool_slots(a, L, b):
    """Paged-pool slots of --pool-gb HBM (a B200 holds 180 GB; the rest is the
    model): the PE pool and each DE's decode pool."""
    return int(a.pool_gb * 1e9 // (L * 64 * b))


def cluster(P, D, L, b, hbm_tokens=100_000_000):
    cfg = dp.ClusterConfig()
    cfg.prefill_nodes, cfg.decode_nodes, cfg.engines_per_node = P, D, 1
    cfg.n_layer, cfg.kv_bytes_per_token_per_layer, cfg.block_size_tokens = L, b, 64
    cfg.hbm_capacity_tokens = hbm_tokens
    cfg.pe_buffer_bytes = cfg.de_buffer_bytes = int(80e9 / 8)
    return cfg


def one(a, cfg, trajs, policy, aps, devices):
    rng = np.random.default_rng(a.seed)
    arrivals = list(np.cumsum(rng.exponential(1.0 / aps, len(trajs))))
    ex = dp.ExecOptions()
    ex.seed = 9
    ex.storage_cap_Bps = a.cap_gbps * 1e9
    if a.caps:  # config 5: asymmetric per-engine storage NICs
        ex.storage_cap_per_engine = [float(x) * 1e9 for x in a.caps.split(",")]
    ex.k1_mode, ex.k2_mode = 3, 2
    if a.prefill:  # the prefill stand-in (K5 forwards): TTFT = arrival -> prefill done
        ex.prefill = True
        ex.compute_quota = a.quota_ms * 1e-3
        ex.prefill_cost = (576 / (a.attend_tops * 1e12), 0.0, 0.0, 20e-6)
        ex.handoff = a.handoff  # + K3 into the DE decode pools: TTFT = first token, as the reference's
    t0 = time.time()
    slots = pool_slots(a, cfg.n_layer, cfg.kv_bytes_per_token_per_layer)
    rep = dp.run_live(cfg, trajs, policy=policy, exec=ex, arrival_times=arrivals, slo_ttft=a.slo,
                      pe_pool_slots=slots, de_pool_slots=slots if a.handoff else 0,
                      steady_window=a.steady_window, steady_lookback=a.steady_lookback, steady_threshold=0.1,
                      decode_s_per_token=a.decode_ms * 1e-3, gpu=not a.cpu, link_Bps=50e9, devices=devices,
                      alpha=a.alpha, beta=a.beta)
    ttft = [t for _, t in rep["ttft_series"]]
    return {"aps": round(aps, 4), "ok": not rep["slo_violated"], "slo_violated": rep["slo_violated"],
            "steady": rep["steady_state"], "completed": rep["completed_requests"],
            "total": rep["total_requests"], "wall_s": round(time.time() - t0, 2),
            "ttft_p50": round(float(np.percentile(ttft, 50)), 4) if ttft else None,
            "ttft_max": round(max(ttft), 4) if ttft else None,
            "de_path": sum(1 for d in rep["decisions"] if d[4] == 1), "decisions": len(rep["decisions"]),
            "read_gb": [round(x / 1e9, 2) for x in rep["reader_bytes"]], "forwards": rep["forwards"]}


def capacity(a, cfg, trajs, policy, devices):
    lo, hi, runs = None, a.aps_start, []
    while True:  # grow until the SLO breaks
        r = one(a, cfg, trajs, policy, hi, devices)
        runs.append(r)
        if not r["ok"]:
            break
        lo, hi = hi, hi * 2
        if hi > a.aps_max:
            return lo, runs
    if lo is None:
        lo = 0.0
    for _ in range(a.bisect):
        mid = (lo + hi) / 2 if lo == 0 else (lo * hi) ** 0.5
        r = one(a, cfg, trajs, policy, mid, devices)
        runs.append(r)
        lo, hi = (mid, hi) if r["ok"] else (lo, mid)
    return lo, runs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pd", default="1:1")
    ap.add_argument("--sessions", type=int, default=96)
    ap.add_argument("--turns", type=int, default=6)
    ap.add_argument("--cap-gbps", type=float, default=6.25)
    ap.add_argument("--caps", default="", help="config 5: per-engine storage caps, GB/s, comma list (one per engine)")
    ap.add_argument("--slo", type=float, default=0.3, help="load-TTFT SLO, seconds")
    ap.add_argument("--decode-ms", type=float, default=1.0, help="emulated decode per generated token")
    ap.add_argument("--steady-window", type=float, default=4.0)
    ap.add_argument("--steady-lookback", type=float, default=12.0)
    ap.add_argument("--aps-start", type=float, default=4.0)
    ap.add_argument("--aps-max", type=float, default=256.0)
    ap.add_argument("--bisect", type=int, default=3)
    ap.add_argument("--alpha", type=int, default=100000)
    ap.add_argument("--beta", type=int, default=500000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu", action="store_true", help="timed backend (no GPU): host check of the tool")
    ap.add_argument("--prefill", action="store_true",
                    help="run the prefill stand-in (K5 forwards under the compute quota) on the PEs; the PE "
                         "is released and the TTFT taken when a request's prefill is done")
    ap.add_argument("--quota-ms", type=float, default=0.5, help="--prefill: compute quota per layer")
    ap.add_argument("--pool-gb", type=float, default=100.0,
                    help="HBM of the PE pool and of each decode pool; with --handoff the DEs' HBM capacity "
                         "the scheduler balances (hbm_capacity_tokens) is the decode pool's")
    ap.add_argument("--handoff", action="store_true",
                    help="with --prefill: the PD handoff (dual gather on the DE path, K3 into decode pools); the "
                         "PE releases after K3 and the TTFT is the first token's")
    ap.add_argument("--attend-tops", type=float, default=40.0, help="--prefill: K5 speed of the cost model")
    a = ap.parse_args()
    if a.handoff and not a.prefill:
        ap.error("--handoff needs --prefill")
    if a.caps and len(a.caps.split(",")) != sum(int(x) for x in a.pd.split(":")):
        ap.error("--caps needs one cap per engine")
    P, D = (int(x) for x in a.pd.split(":"))
    L, b = 61, 576
    cfg = cluster(P, D, L, b, pool_slots(a, L, b) * 64 if a.handoff else 100_000_000)
    trajs = dp.synthesize(max_len=131072, count=a.sessions, seed=9, mean_turns=a.turns, sigma_turns=0.0,
                          mean_append=429, mean_gen=500)
    ndev = 0
    if not a.cpu:
        import torch
        ndev = torch.cuda.device_count()
    devices = [e % max(1, ndev) for e in range(P + D)] if ndev else []
    if ndev:  # engines sharing a GPU share its HBM
        a.pool_gb /= -(-(P + D) // ndev)
    out = {"what": "online APS capacity (sessions/s within the load-TTFT SLO), live-mode scheduling on "
                   "measured completions", "pd": a.pd, "sessions": a.sessions, "turns": a.turns,
           "cap_gbps_per_engine": [float(x) for x in a.caps.split(",")] if a.caps else a.cap_gbps,
           "slo_s": a.slo, "decode_ms_per_token": a.decode_ms,
           "devices": devices, "backend": "timed" if a.cpu else "gpu",
           "ttft": ("arrival -> first token (prefill, K3 handoff, one decode step)" if a.handoff else
                    "arrival -> prefill done (K5 forwards)") if a.prefill else "arrival -> hit KV landed",
           "prefill": {"quota_ms": a.quota_ms, "attend_tops": a.attend_tops} if a.prefill else None}
    for policy in ("dual_path", "pe_only"):
        cap, runs = capacity(a, cfg, trajs, policy, devices)
        out[policy] = {"capacity_aps": round(cap, 4), "runs": runs}
    pe = out["pe_only"]["capacity_aps"]
    out["dual_vs_one_path"] = round(out["dual_path"]["capacity_aps"] / pe, 3) if pe else None
    print(json.dumps(out))


if __name__ == "__main__":
    main()
