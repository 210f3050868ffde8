#!/usr/bin/env python
"""DualPath KV-Cache loading benchmark on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c1|c2|c3] [--cap-gbps X] [--sessions-per-gpu S]

N = 1: BASELINE config 1 (64 sessions x 20 turns, DeepSeek-V3 MLA KV) loaded
by the K1 loader alone (the PE of a 1P1D prefill-only plan; P/D needs two
engines, proj/src/types.cpp:11-12).  N > 1: one process per GPU (re-launched
under torch.distributed.run when WORLD_SIZE is unset), engines 0..N/2-1
prefill (PE), the rest decode (DE), dual-path plan over 16 sessions per GPU;
the same workload also runs prefill-only ("1-path", Policy::PEOnly,
proj/src/desim.cpp:826-827), and BASELINE config 2 (32K-128K contexts,
per-engine storage NIC capped at 6.25 GB/s, dual vs 1-path) runs in the same
line under "storage_capped".

A step = one offline pass of the synthetic agentic trace: every request's
hit KV (C*L*b bytes) moved from the emulated storage tier (pinned host DRAM
on each GPU's NUMA node, read over each engine's own PCIe link, optionally
rate-capped per engine) into the PE's paged HBM pool, by K1 (PE path) or K2
(DE path, NVLink push).  Inputs are larger than L2 (hundreds of GB per
step), so no flush is needed.

The scheduler decisions of every plan are digested into the line and, when
tests/golden/bench_*.json holds the reference's own decisions for the exact
configuration (tests/golden/make_golden.py, oracle/_ref), compared with them.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DSV3 = dict(L=61, b=576, T=64)          # DeepSeek-V3 MLA fp8 KV (BASELINE configs 1-2)
QWEN = dict(L=64, b=4096, T=64)         # Qwen2.5-32B GQA bf16 KV (config 3)
PCIE_ZC_BPS = 51.5e9                    # measured SM zero-copy H2D per GPU (profiles/r01_probe_links.txt)
NVLINK_BPS = 778e9                      # measured memcpyPeer per direction (same probe)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c1", choices=["c1", "c2", "c3"])
    ap.add_argument("--trace", default="",
                    help="sessions from a reference-format trace TSV instead of the generator "
                         "(first sessions-per-gpu x N lines; KV shape of --workload)")
    ap.add_argument("--cap-gbps", type=float, default=0.0,
                    help="per-engine storage-NIC cap (0 = uncapped: the PCIe link binds)")
    ap.add_argument("--sessions-per-gpu", type=int, default=0,
                    help="0 = default: config 1's 64 sessions at N = 1, 16 per GPU at N > 1")
    ap.add_argument("--link-model", default="fixed", choices=["fixed", "measured"],
                    help="per-engine storage-read rate the planner (the reference's model) uses when "
                         "uncapped: fixed = the SM zero-copy rate 51.5 GB/s (decisions pinned by "
                         "tests/golden/bench_*.json); measured = min(51.5, this box's concurrent "
                         "host-link ceiling / N)")
    ap.add_argument("--no-capped", action="store_true",
                    help="N > 1: skip the config-2 storage-capped dual vs 1-path sub-run")
    ap.add_argument("--capped-steps", type=int, default=2, help="timed steps of the storage-capped sub-run")
    ap.add_argument("--capped-sessions-per-gpu", type=int, default=6)
    ap.add_argument("--capped-gbps", type=float, default=6.25,
                    help="per-engine storage-NIC cap of the sub-run (400 Gbps SNIC per 8 GPUs, PAPER.md:496)")
    ap.add_argument("--store-gb", type=float, default=0.0,
                    help="host store per engine, GB (0 = the whole trace, within half the host RAM)")
    ap.add_argument("--no-one-path", action="store_true", help="skip the prefill-only comparison")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pd", default="", help="override P:D, e.g. 2:6")
    ap.add_argument("--online", type=float, default=0.0,
                    help="config 5: Poisson arrivals at this many sessions/s, replayed in real time")
    ap.add_argument("--caps", default="", help="config 5: per-engine storage caps, GB/s, comma list")
    ap.add_argument("--handoff", action="store_true",
                    help="also run the PD handoff: prefill stand-in + PeToDe/MissMerge per layer "
                         "into the DE decode pools, DE read path fused with DecodeH2D")
    ap.add_argument("--persist", action="store_true",
                    help="also persist generated tokens (decode stand-in + K4 D2H), implies --handoff")
    ap.add_argument("--handoff-ctas", type=int, default=0, help="K3 CTA cap on PEs (0 = default)")
    ap.add_argument("--k3-tma", action="store_true", help="K3's hit push through the TMA (bulk copies)")
    ap.add_argument("--persist-mode", default="staged", choices=["kernel", "staged"],
                    help="K4 (PersistD2H): SM zero-copy stores, or a gather into an HBM ring + copy engine")
    ap.add_argument("--k3", default="ce", choices=["kernel", "ce"],
                    help="K3 (PD handoff push): SM kernel, or copy engines + a small side kernel per layer")
    ap.add_argument("--layerwise", action="store_true",
                    help="handoff + prefill: K3 pushes layer l as soon as the finishing forward has computed it "
                         "(the reference's order), instead of after the forward (the default: measured faster)")
    ap.add_argument("--gather-ctas", type=int, default=-1, help="K1/K2 CTA cap (-1 = auto)")
    ap.add_argument("--prefill", action="store_true",
                    help="run the prefill stand-in on every PE: compute-quota batched forwards "
                         "(build_forward_batch) of K5 attention-score passes over the landed KV, "
                         "layer by layer, overlapped with the loads")
    ap.add_argument("--quota-ms", type=float, default=0.5,
                    help="prefill: compute quota per layer of a forward (ms of the cost model)")
    ap.add_argument("--attend-tops", type=float, default=40.0,
                    help="prefill: cost-model rate of K5 in tera multiply-adds/s (bilinear term)")
    ap.add_argument("--tier", default="",
                    help="storage tier: StorageRead reads every Full Block from this file (created "
                         "and populated once per box; O_DIRECT) through a pinned staging ring")
    ap.add_argument("--io-threads", type=int, default=8, help="storage tier: host IO threads per engine")
    ap.add_argument("--wait-timeout-ms", type=int, default=30000, help="watchdog of every cross-engine wait")
    ap.add_argument("--k2", default="staged", choices=["sm", "ce", "staged"],
                    help="DE-path loads: sm = K2 gather pushing over NVLink, ce = the DE's copy engine, "
                         "staged = copy engine into an HBM ring + NVLink scatter kernel")
    ap.add_argument("--k1", default="staged", choices=["sm", "ce", "hybrid", "staged"],
                    help="PE-path loads: sm = K1 gather kernel, ce = copy engine (no SMs), "
                         "hybrid = both at once, jobs split by bytes, staged = copy engine into an HBM "
                         "ring + scatter kernel")
    ap.add_argument("--stage-ctas", type=int, default=32, help="staged K1: scatter kernel CTAs")
    ap.add_argument("--stage-ring-mb", type=int, default=1024, help="staged loaders: HBM ring per engine, MiB")
    ap.add_argument("--pool-layout", default="layer", choices=["layer", "block"],
                    help="PE pool: per-layer planes, or whole Full Blocks per slot (with --k1 ce / --k2 ce the copy "
                         "engine lands Full-Block runs in one copy: no ring, no SM work)")
    ap.add_argument("--stage-push-ctas", type=int, default=148,
                    help="staged K2: CTAs of the scatter pushing over NVLink")
    ap.add_argument("--stage-scatter", default="kernel", choices=["kernel", "ce"],
                    help="staged modes: ring -> pool scatter by a kernel or by the copy engine (no SMs)")
    return ap.parse_args()


# ----------------------------------------------------------------- workload
GEN_C1 = dict(max_len=131072, seed=9, mean_turns=20, sigma_turns=0.0, mean_append=429, mean_gen=500)


def n_sessions(args, n_gpus):
    if args.sessions_per_gpu > 0:
        return args.sessions_per_gpu * max(1, n_gpus)
    return 64 if n_gpus <= 1 else 16 * n_gpus


def c2_rounds(i):
    """Config 2 session i: one cold prefill round {C-1, 1} that builds a
    32K / 64K / 128K context, then three warm rounds {429, 1} (a cold append
    instead of the reference tests' long generation round, whose 64-token
    persistence flows would dominate planning)."""
    c = (32768, 65536, 131072)[i % 3]
    return [(c - 1, 1)] + [(429, 1)] * 3


def workload(args, n_gpus, kind=None, sessions=None):
    """Trajectories + KV shape.  c1: BASELINE config 1 generator (20 turns,
    mean append 429, mean gen 500, ~95% hit); c2: 32K/64K/128K contexts
    (config 2); c3: c1 with the Qwen2.5-32B KV shape (config 3)."""
    import paper_2602_21548_b200 as dp
    kind = kind or args.workload
    sessions = sessions or n_sessions(args, n_gpus)
    if getattr(args, "trace", "") and kind == args.workload:
        trajs = dp.load_trace(args.trace)[:sessions]
        if not trajs:
            raise SystemExit(f"--trace {args.trace}: no sessions")
        return trajs, (QWEN if kind == "c3" else DSV3)
    if kind in ("c1", "c3"):
        trajs = dp.synthesize(count=sessions, **GEN_C1)
        return trajs, (DSV3 if kind == "c1" else QWEN)
    trajs = []
    for i in range(sessions):
        t = dp.Trajectory()
        t.id = f"ctx{i}"
        t.rounds = [dp.Round(a, g) for a, g in c2_rounds(i)]
        trajs.append(t)
    return trajs, DSV3


def trace_stats(rounds_per_session, shape):
    """requests, hit bytes (sum C*L*b) and prompt tokens (sum C+A) of a trace,
    from its rounds alone (context_before, proj/src/types.cpp:44-53)."""
    req = hit = prompt = 0
    for rounds in rounds_per_session:
        ctx = 0
        for a, g in rounds:
            req += 1
            hit += ctx * shape["L"] * shape["b"]
            prompt += ctx + a
            ctx += a + g
    return req, hit, prompt


def config_dict(kind, sessions, P, D, policy, shape, cap_gbps, stats, extra=None):
    """The `config` of a line: identical for both arms of the same run."""
    req, hit, prompt = stats
    cfg = {"workload": f"{kind}: {sessions} sessions, {P}P{D}D {policy}"
                       + (" (1 PE loader, K1)" if P + D == 2 and policy == "pe_only" else ""),
           "sessions": sessions, "kv": shape, "storage_cap_gbps_per_engine": cap_gbps or None,
           "host_buffer_bytes_per_engine": buffer_bytes(shape),
           "requests": req, "hit_bytes_per_step": hit, "prompt_tokens_per_step": prompt,
           "l2": "inputs >> L2 (hundreds of GB per step; no flush needed)"}
    if extra:
        cfg.update(extra)
    return cfg


def buffer_bytes(shape):
    """Host staging per engine (pe_buffer_bytes = de_buffer_bytes): the
    reference's own preset, 128 GiB per node (proj/src/config.cpp:57-58), one
    node per engine here (g = 1).  The planner's admissions and the executor's
    reads (BufferGate) both honour it."""
    return 1 << 37


def golden_key(kind, sessions, P, D, policy, cap_gbps, link_bps):
    link = "cap%g" % cap_gbps if cap_gbps else "link%g" % (link_bps / 1e9)
    return f"{kind}_{sessions}s_{P}p{D}d_{policy}_{link}_buf"


def golden_check(key, digest):
    """Compare a plan's decision digest with the reference's own decisions for
    the same configuration (tests/golden/bench_<key>.json), when recorded."""
    path = os.path.join(ROOT, "tests", "golden", f"bench_{key}.json")
    if not os.path.exists(path):
        return {"fixture": None, "match": None}
    with open(path) as f:
        want = json.load(f)["decisions_digest"]
    return {"fixture": os.path.relpath(path, ROOT), "match": want == digest}


def cluster(shape, P, D, cap_bps, caps=None, link_bps=PCIE_ZC_BPS):
    import paper_2602_21548_b200 as dp
    cfg = dp.ClusterConfig()
    if caps:
        cfg.storage_bandwidth_per_node = list(caps)  # g = 1: one node per engine
    cfg.prefill_nodes, cfg.decode_nodes, cfg.engines_per_node = P, D, 1
    cfg.n_layer, cfg.kv_bytes_per_token_per_layer, cfg.block_size_tokens = shape["L"], shape["b"], shape["T"]
    # compute network = NVLink (the DE->PE push), storage NIC = the engine's
    # PCIe read rate, or the emulated cap when one is set
    cfg.cnic_bandwidth = NVLINK_BPS
    cfg.storage_multiple = (cap_bps if cap_bps > 0 else link_bps) / NVLINK_BPS
    cfg.dram_bandwidth = 2e12
    cfg.hbm_capacity_tokens = 100_000_000
    cfg.pe_buffer_bytes = cfg.de_buffer_bytes = buffer_bytes(shape)
    return cfg


# storage-bound cost model (proj/tests/acceptance.cpp:62-72): the bench
# measures loading, compute is nearly free
PLAN_KW = dict(cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0.0, beta=1_000_000_000)


# ------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, devices):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if not self.proc or not os.path.exists(self.path):
            return out
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9 or not p[0].isdigit() or int(p[0]) not in devices:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if sm:
            out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                   "samples": len(sm)}
        return out


# ------------------------------------------------------------ distributed
def my_device(dist):
    """This rank's GPU: its local rank (one process per GPU).  More ranks than
    GPUs (a control-plane rehearsal of a larger N) wrap around."""
    import torch
    return (dist.local if dist.world > 1 else 0) % max(1, torch.cuda.device_count())


def make_group(n):
    from paper_2602_21548_b200 import dist as dpdist
    g = dpdist.Group("nccl")
    if g.world != n and n > 1:
        raise SystemExit(f"--gpus {n} needs torchrun with {n} ranks (WORLD_SIZE={g.world})")
    return g


# --------------------------------------------------------------- measuring
def measure_pcie_peak(device):
    """Copy-engine H2D of 1 GiB pinned, best of 5 (the PCIe link roofline)."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    s = torch.cuda.Stream(device=device)
    best = 1e9
    with torch.cuda.stream(s):
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            d.copy_(h, non_blocking=True)
            b.record(s)
            b.synchronize()
            best = min(best, a.elapsed_time(b))
    del h, d
    return n / (best * 1e-3)


def measure_concurrent_h2d(dist, device, reps=3):
    """Every rank at once: copy-engine H2D of 1 GiB pinned, after a barrier.
    The box's aggregate host-link ceiling for an N-GPU line (PCIe switches may
    be shared between GPUs, so N x the single-GPU peak can overstate it)."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    s = torch.cuda.Stream(device=device)
    best = 0.0
    for _ in range(reps):
        dist.barrier()
        with torch.cuda.stream(s):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(4):
                d.copy_(h, non_blocking=True)
            b.record(s)
            b.synchronize()
        ms = dist.max(a.elapsed_time(b))  # the slowest rank bounds the aggregate
        best = max(best, dist.world * 4 * n / (ms * 1e-3))
    del h, d
    return best


def measure_host_ceiling_local(n, reps=3):
    """One process driving GPUs 0..n-1 at once: copy-engine H2D of 1 GiB pinned
    x 4 per GPU on its own stream.  The same aggregate host-link ceiling as
    measure_concurrent_h2d, for the reference arm (rank 0 alone)."""
    import torch
    size = 1 << 30
    bufs = []
    n = min(n, torch.cuda.device_count())
    for d in range(n):
        with torch.cuda.device(d):
            bufs.append((torch.empty(size, dtype=torch.uint8, pin_memory=True),
                         torch.empty(size, dtype=torch.uint8, device=f"cuda:{d}"),
                         torch.cuda.Stream(device=d)))
    best = 0.0
    for _ in range(reps):
        for d in range(n):
            torch.cuda.synchronize(d)
        evs = []
        for d, (h, dv, st) in enumerate(bufs):
            with torch.cuda.device(d), torch.cuda.stream(st):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(4):
                    dv.copy_(h, non_blocking=True)
                b.record(st)
                evs.append((a, b))
        ms = 0.0
        for a, b in evs:
            b.synchronize()
            ms = max(ms, a.elapsed_time(b))
        best = max(best, n * 4 * size / (ms * 1e-3))
    del bufs
    return best


def link_per_engine(ceiling_bps, n):
    """The storage-read rate one engine can sustain on this box: the SM
    zero-copy rate, or its share of the box's concurrent host-link ceiling
    when all engines read at once (some boxes cap 4 GPUs at 116-152 GB/s)."""
    if not ceiling_bps or n <= 1:
        return PCIE_ZC_BPS
    return min(PCIE_ZC_BPS, ceiling_bps / n)


def measure_k1(device, shape, mode="staged", stage_ctas=32, target_bytes=18421383168):
    """The dominant transfer alone, live: one K1 call of 64 requests x 128
    random Full Blocks (DS-V3: 18.4 GB, the launch ncu profiled) through the
    C ABI -- the staged path (copy engine into the HBM ring + scatter kernel)
    or the SM gather kernel -- CUDA events on its stream, median of 3 after a
    warm-up."""
    import numpy as np
    import torch
    from paper_2602_21548_b200 import abi
    L, T, b = shape["L"], shape["T"], shape["b"]
    blocks = 128
    per_job = blocks * T * b * L
    jobs_n = max(1, min(64, target_bytes // per_job))
    g = abi.geom(L, T, b)
    n_fb = max(2 * blocks, (2 << 30) // (L * T * b))
    st = abi.Store(device, g, n_fb, 9)
    pool = abi.Pool(device, g, jobs_n * blocks, jobs_n)
    stager = abi.Stager(device, g) if mode == "staged" else None
    if stager:
        stager.set_ctas(stage_ctas)
    try:
        rng = np.random.default_rng(0)
        keep, specs = [], []
        perm = rng.permutation(jobs_n * blocks).astype(np.int32)
        for j in range(jobs_n):
            fbs = rng.integers(0, n_fb - blocks + 1) + np.arange(blocks)  # one session's consecutive Full Blocks
            f_host = np.ascontiguousarray(fbs, dtype=np.int64)
            f = torch.tensor(f_host, device=f"cuda:{device}")
            sl = torch.tensor(perm[j * blocks:(j + 1) * blocks], device=f"cuda:{device}")
            keep += [f_host, f, sl]
            src = f_host.ctypes.data if stager else f.data_ptr()
            specs.append((src, sl.data_ptr(), blocks * T, blocks, 0, L, j))
        jobs = abi.make_jobs(specs)
        s = torch.cuda.Stream(device=device)
        times = []
        for r in range(4):
            pool.reset_counters(s.cuda_stream)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(device):
                e0.record(s)
                if stager:
                    abi.h2d_layer_staged(pool, st, stager, jobs, len(specs), s.cuda_stream)
                else:
                    abi.h2d_layer_gather(pool, st, jobs, len(specs), s.cuda_stream)
                e1.record(s)
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        ms = sorted(times)[1]
        nbytes = jobs_n * per_job
        return nbytes / (ms * 1e-3) / 1e9, ms, nbytes
    finally:
        if stager:
            stager.close()
        pool.close()
        st.close()


def prefill_cost(args, shape):
    """Cost model of the prefill stand-in per layer (AttentionCostModel):
    K5 does bsz * cached * b multiply-adds per request chunk (bilinear), plus
    a fixed per-layer cost of the gate and the launch (constant)."""
    return (shape["b"] / (args.attend_tops * 1e12), 0.0, 0.0, 20e-6)


def store_budget(args, dist):
    """Host store per engine: the whole trace (no two sessions share a Full
    Block), within half of this host's RAM shared by its local engines."""
    if args.store_gb > 0:
        return int(args.store_gb * 1e9)
    try:
        mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        mem = 64 << 30
    local = int(os.environ.get("LOCAL_WORLD_SIZE", str(max(1, dist.world))))
    return max(8 << 30, mem // 2 // max(1, local))


def run_policy(args, dist, variant, trajs, shape, P, D, clocks=None, prefill=None, link_bps=PCIE_ZC_BPS):
    """Plan, build engines, run W + K steps; returns per-step max-over-ranks
    device and host times, plus per-rank info.  variant = (policy, sched_mode)."""
    import paper_2602_21548_b200 as dp
    policy, sched_mode = variant
    cap = args.cap_gbps * 1e9
    caps = [float(x) * 1e9 for x in args.caps.split(",")] if args.caps else None
    if caps and len(caps) != P + D:
        raise SystemExit(f"--caps needs {P + D} entries")
    cfg = cluster(shape, P, D, cap, caps, link_bps)
    kw = dict(PLAN_KW)
    if args.online > 0:
        # Poisson arrivals (desim.cpp:1036-1051); SLO / steady-state stops off
        kw.update(aps=args.online, seed=1, slo_ttft=1e9, steady_lookback=1e9)
    t0 = time.time()
    planned = dp.plan(cfg, trajs, policy=policy, sched_mode=sched_mode, **kw)
    plan_s = time.time() - t0
    opt = dp.ExecOptions()
    opt.storage_cap_Bps = cap
    if caps:
        opt.storage_cap_per_engine = caps
    if args.online > 0:
        opt.pace_scale = 1.0
    opt.k1_mode = {"sm": 0, "ce": 1, "hybrid": 2, "staged": 3}[args.k1]
    opt.stage_ring_bytes = args.stage_ring_mb << 20
    opt.pool_layout = 1 if args.pool_layout == "block" else 0
    opt.k2_mode = {"sm": 0, "ce": 1, "staged": 2}[args.k2]
    opt.stage_ctas = args.stage_ctas
    opt.stage_push_ctas = args.stage_push_ctas
    opt.stage_scatter = 1 if args.stage_scatter == "ce" else 0
    opt.wait_timeout_ms = args.wait_timeout_ms
    opt.handoff = bool(args.handoff or args.persist)
    opt.persist = bool(args.persist)
    opt.handoff_ctas = args.handoff_ctas
    opt.handoff_layerwise = args.layerwise
    opt.handoff_tma = args.k3_tma
    opt.k3_mode = 1 if args.k3 == "ce" else 0
    opt.persist_mode = 1 if args.persist_mode == "staged" else 0
    opt.gather_ctas = args.gather_ctas
    opt.seed = 9
    if args.tier:
        opt.tier_path = args.tier
        opt.io_threads = args.io_threads
    prefill = args.prefill if prefill is None else prefill
    if prefill:
        opt.prefill = True
        opt.compute_quota = args.quota_ms * 1e-3
        opt.prefill_cost = prefill_cost(args, shape)
    opt.store_bytes_max = store_budget(args, dist)
    xp = dp.build_exec_plan(cfg, trajs, planned, opt)
    tier = None
    if args.tier:
        # one file per box, written by local rank 0 (the same pages every
        # policy reads); the others wait at the barrier
        t0 = time.time()
        if dist.local == 0:
            need = xp.store_fb
            ok = False
            if os.path.exists(args.tier):
                try:
                    dp.FullBlockFile(args.tier, cfg.n_layer, cfg.block_size_tokens,
                                     cfg.kv_bytes_per_token_per_layer, need)
                    ok = True
                except RuntimeError:
                    ok = False
            if not ok:
                f = dp.FullBlockFile(args.tier, cfg.n_layer, cfg.block_size_tokens,
                                     cfg.kv_bytes_per_token_per_layer, need, create=True)
                f.populate(9, threads=os.cpu_count() or 8)
                del f
        dist.barrier()
        f = dp.FullBlockFile(args.tier, cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer,
                             xp.store_fb)
        tier = dict(path=args.tier, direct=f.direct(), records=f.records(),
                    file_gb=round(f.records() * f.stride() / 1e9, 2), ring_fb=xp.ring_fb,
                    trie_nodes=xp.trie_nodes, io_threads=args.io_threads,
                    open_or_populate_s=round(time.time() - t0, 2))
        del f
    from paper_2602_21548_b200 import dist as dpdist
    digest = dpdist.plan_digest(planned)
    digests = dist.allgather(digest)
    assert len(set(digests)) == 1, "ranks planned differently"
    if dist.world > 1:
        my = [dist.rank]
    else:
        my = [0]  # N=1: only the PE engine exists on this box
    engines = {}
    for e in my:
        dev = my_device(dist)
        engines[e] = dp.EngineRuntime(xp, e, dev)
    if dist.world > 1:
        dpdist.connect_pools(dist, engines, cfg.prefill_nodes)
    dev_ms, host_ms, launches, read_bytes, spans, per_engine = [], [], 0, 0, None, None
    r0_bytes, r0_ms = 0, 0.0  # rank 0's own engine over the timed steps (the roofline)
    ttft, lag = [], []
    stalls, bwait = 0, 0.0
    io_wait = 0.0
    d2h = 0
    for step in range(args.warmup + args.steps):
        for rt in engines.values():
            rt.reset_counters()
        dist.barrier()
        if clocks is not None and step == args.warmup:
            clocks.__enter__()  # sample clocks during the timed steps only
        res = [rt.run_step() for rt in engines.values()]
        d = dist.max(max(r.device_ms for r in res))
        h = dist.max(max(r.host_ms for r in res))
        if step >= args.warmup:
            dev_ms.append(d)
            host_ms.append(h)
            launches += sum(dist.allgather(sum(r.launches for r in res)))
            io_wait = max(io_wait, dist.max(max(r.io_wait_ms for r in res)))
            d2h = sum(dist.allgather(sum(r.d2h_bytes for r in res)))  # per step (the same each step)
            read_bytes += sum(dist.allgather(sum(r.bytes_read for r in res)))
            r0_bytes += res[0].bytes_read
            r0_ms += res[0].device_ms
            stalls += sum(dist.allgather(sum(r.buffer_stalls for r in res)))
            bwait = max(bwait, dist.max(max(r.buffer_wait_ms for r in res)))
            ttft, lag = list(res[0].ttft_ms), list(res[0].handoff_lag_ms)
            spans, per_engine = {}, {}
            for part in dist.allgather({e: (r.spans, r.device_ms) for e, r in zip(engines, res)}):
                for e, (sp, ms) in part.items():
                    spans[e] = sp
                    per_engine[e] = round(ms, 1)
    fwd = None
    if prefill:
        # the compute alone: the PEs' forwards again over the KV already landed
        pes = [rt for e, rt in engines.items() if e < P]
        dist.barrier()
        r = [rt.run_forwards() for rt in pes]
        alone = dist.max(max([x.device_ms for x in r], default=0.0))
        n_fwd = sum(dist.allgather(sum(x.forwards for x in r)))
        work = sum(it[2] * it[4] for pe in range(P) for _, items in xp.forwards(pe) for it in items)
        fwd = dict(forwards_per_step=n_fwd, compute_alone_ms=round(alone, 3),
                   macs_per_step=work * shape["b"] * shape["L"],
                   est_s_per_step=sum(est for pe in range(P) for est, _ in xp.forwards(pe)) * shape["L"])
    snic = sum(u["total_bytes"] for u in planned["usage"] if u["kind"] == "snic_read")
    info = dict(plan_s=plan_s, hit_bytes=xp.hit_bytes, prompt_tokens=xp.prompt_tokens, digest=digest,
                r0_bytes=r0_bytes, r0_ms=r0_ms, policy=policy, ttft_ms=ttft, lag_ms=lag,
                buffer_stalls=stalls, buffer_wait_ms=bwait,
                handoff_bytes=xp.handoff_bytes if (args.handoff or args.persist) else 0,
                persist_bytes=xp.persist_bytes if args.persist else 0,
                model_gbps=snic / planned["makespan"] / 1e9 if planned["makespan"] > 0 else None,
                requests=xp.requests, reader_bytes=list(xp.reader_bytes),
                de_path=sum(1 for d in planned["decisions"] if d[4] == 1),
                decisions=len(planned["decisions"]), pool_slots=xp.pool_slots, spans=spans,
                per_engine_ms=[per_engine[e] for e in sorted(per_engine)] if per_engine else None,
                caps=caps,
                store_fb=xp.store_fb, launches=launches, read_bytes=read_bytes, prefill=fwd, d2h=d2h,
                tier=dict(tier, io_wait_ms_max_step=round(io_wait, 1)) if tier else None)
    if clocks is not None:
        clocks.__exit__()
    engines.clear()  # frees pools, stores and peer mappings before the next policy
    dist.barrier()
    return dict(dev_ms=dev_ms, host_ms=host_ms, info=info, xp=xp, cfg=cfg)


def cpu_baseline(xp, shape, seconds=12.0):
    """oracle/kvref.c gather of the same Layer Blocks on all host cores
    (the CPU port of the path), on a bounded sample of the workload."""
    import ctypes
    import numpy as np
    from oracle import refpy
    g = refpy.geom(shape["L"], shape["T"], shape["b"])
    fb_bytes = shape["L"] * shape["T"] * shape["b"]
    n_fb = min(xp.store_fb, 256)
    store = np.empty(n_fb * fb_bytes, dtype=np.uint8)
    # content restated on the CPU (multi-threaded by Full Block range)
    threads = os.cpu_count() or 1
    chunks = np.array_split(np.arange(n_fb), threads)
    ths = []
    for c in chunks:
        if len(c) == 0:
            continue
        def work(c=c):
            refpy.kvref().kvref_fill_store(ctypes.byref(g), 9, int(c[0]), len(c),
                                           store[int(c[0]) * fb_bytes:].ctypes.data)
        th = threading.Thread(target=work)
        th.start()
        ths.append(th)
    for th in ths:
        th.join()
    jobs = xp.jobs()
    specs, moved = [], 0
    target = 8 << 30
    for j in jobs:
        fbs = [f % n_fb for f in j[10]]
        specs.append((fbs, j[9], j[6], 0, shape["L"]))
        moved += j[6] * shape["L"] * shape["b"]
        if moved >= target:
            break
    n_slots = xp.pool_slots
    lb = shape["T"] * shape["b"]
    pool = np.zeros(shape["L"] * n_slots * lb, dtype=np.uint8)
    arr, keep = refpy.make_jobs(specs)
    t0 = time.time()
    total = 0
    reps = 0
    while time.time() - t0 < seconds or reps == 0:
        total += refpy.kvref().kvref_gather_mt(ctypes.byref(g), store.ctypes.data, arr, len(specs),
                                               pool.ctypes.data, n_slots, threads)
        reps += 1
    dt = time.time() - t0
    return {"value": round(total / dt / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{len(specs)} requests ({moved / 1e9:.1f} GB of Layer Blocks) x {reps} reps, "
                      f"memcpy gather store->host pool, {threads} threads"}


# ---------------------------------------------------------------- reference
def reference_trace(args, kind, sessions, path):
    """The same trace, built by the REFERENCE (oracle/_ref = pdsim compiled
    from /root/reference sources: its synthesize, proj/src/workload.cpp) or,
    for config 2, written as a reference-format TSV -- no repo .so loaded."""
    from oracle import refpy
    if kind in ("c1", "c3"):
        if getattr(args, "trace", ""):
            with open(args.trace) as f, open(path, "w") as g:
                for i, line in enumerate(f):
                    if i >= sessions:
                        break
                    g.write(line)
        else:
            refpy.ref_synthesize(path, count=sessions, **GEN_C1)
    else:
        with open(path, "w") as f:
            for i in range(sessions):
                f.write(f"ctx{i}\t" + ",".join(f"{a}:{g}" for a, g in c2_rounds(i)) + "\n")
    rounds = []
    with open(path) as f:
        for line in f:
            _, r = line.rstrip("\n").split("\t")
            rounds.append([tuple(int(v) for v in x.split(":")) for x in r.split(",")])
    return rounds


def reference_arm(args):
    """The reference's CPU implementation of the path, timed on this box's
    host cores on the SAME workload and config as our arm.

    The reference (pdsim) moves no bytes: its KV loading is a byte count in a
    fluid flow.  Its CPU path is therefore the oracle port
    (oracle/kvref.c, kind "port"): the memcpy gather of every request's hit
    Layer Blocks C*L*b from the host store (Full Blocks [L][T][b]) into a host
    paged pool [L][slot][T][b], on all host threads, over the full job list
    of the trace (a bounded prefix when the list exceeds ~8 s of CPU per
    step).  The trace comes from the reference's own generator and the
    reference simulator desim::run_offline plans it once (its decisions'
    digest and wall time are reported beside the value).  Only oracle/
    libraries are loaded."""
    import ctypes
    import numpy as np
    from oracle import refpy
    n = args.gpus
    P, D = (1, 1) if n == 1 else (n // 2, n - n // 2)
    if args.pd:
        P, D = (int(x) for x in args.pd.split(":"))
    kind = args.workload
    shape = QWEN if kind == "c3" else DSV3
    sessions = n_sessions(args, n)
    policy = "pe_only" if n == 1 else "dual_path"
    cap = args.cap_gbps * 1e9
    path = f"/tmp/dp_ref_trace_{os.getpid()}.tsv"
    try:
        rounds = reference_trace(args, kind, sessions, path)
        stats = trace_stats(rounds, shape)
        # the reference simulator on (a sample of) the trace: decisions + wall time
        sim_sessions = min(sessions, 64 if n == 1 else 16)
        sim_path = path + ".sim"
        with open(path) as f, open(sim_path, "w") as g:
            for i, line in enumerate(f):
                if i < sim_sessions:
                    g.write(line)
        link_bps = PCIE_ZC_BPS
        kv = dict(P=P, D=D, g=1, L=shape["L"], b=shape["b"], T=shape["T"], B=NVLINK_BPS,
                  s=(cap if cap > 0 else link_bps) / NVLINK_BPS, M=2e12, hbm=100_000_000,
                  pe_buf=buffer_bytes(shape), de_buf=buffer_bytes(shape), policy=policy, **PLAN_KW)
        t0 = time.time()
        rep = refpy.ref_simulate(sim_path, **kv)
        sim_wall = time.time() - t0
        os.unlink(sim_path)
    finally:
        if os.path.exists(path):
            os.unlink(path)
    import hashlib
    h = hashlib.sha1()
    for d in rep["decisions"]:
        h.update(repr((d[1], d[2], d[3], d[4])).encode())

    # the CPU port over the job list: every warm request's hit blocks
    L, T, b = shape["L"], shape["T"], shape["b"]
    g = refpy.geom(L, T, b)
    fb_bytes, lb = L * T * b, T * b
    stride = max(-(-sum(a + gg for a, gg in r) // T) for r in rounds)
    n_fb = max(1, min(stride * sessions, (16 << 30) // fb_bytes))   # host store <= 16 GiB
    n_slots = max(64, min(stride * 4, (8 << 30) // (L * lb)))       # host pool <= 8 GiB
    threads = os.cpu_count() or 1
    store = np.empty(n_fb * fb_bytes, dtype=np.uint8)
    parts = [c for c in np.array_split(np.arange(n_fb), threads) if len(c)]
    ths = [threading.Thread(target=lambda c=c: refpy.kvref().kvref_fill_store(
        ctypes.byref(g), 9, int(c[0]), len(c), store[int(c[0]) * fb_bytes:].ctypes.data)) for c in parts]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    pool = np.zeros(L * n_slots * lb, dtype=np.uint8)
    specs, moved, slot = [], 0, 0
    budget = 8.0 * 45e9  # ~8 s of the r01 box's 16-thread rate
    for s, rr in enumerate(rounds):
        ctx = 0
        for a, gg in rr:
            if ctx > 0:
                nblk = -(-ctx // T)
                fbs = [(s * stride + k) % n_fb for k in range(nblk)]
                slots = [(slot + k) % n_slots for k in range(nblk)]
                slot = (slot + nblk) % n_slots
                specs.append((fbs, slots, ctx, 0, L))
                moved += ctx * L * b
            ctx += a + gg
    full = moved
    if moved > 1.5 * budget:  # a bounded prefix of the job list
        acc, keep = 0, []
        for sp in specs:
            if acc >= budget:
                break
            keep.append(sp)
            acc += sp[2] * L * b
        specs, moved = keep, acc
    arr, keepalive = refpy.make_jobs(specs)
    vals, total_bytes, total_s = [], 0, 0.0
    for step in range(args.warmup + args.steps):
        t0 = time.time()
        nbytes = refpy.kvref().kvref_gather_mt(ctypes.byref(g), store.ctypes.data, arr, len(specs),
                                               pool.ctypes.data, n_slots, threads)
        dt = time.time() - t0
        if step >= args.warmup:
            vals.append(nbytes / dt / 1e9)
            total_bytes += nbytes
            total_s += dt
    v = total_bytes / total_s / 1e9
    sample = (f"the full job list ({len(specs)} requests, {moved / 1e9:.1f} GB of Layer Blocks) per step"
              if moved == full else
              f"the first {len(specs)} requests of the job list ({moved / 1e9:.1f} of {full / 1e9:.1f} GB) per step")
    return {"metric": "aggregate KV-load GB/s", "value": round(v, 3), "unit": "GB/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_s * 1e3 / args.steps, 1),
            "higher_is_better": True, "impl": "reference", "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": config_dict(kind, sessions, P, D, policy, shape, args.cap_gbps, stats),
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"oracle/kvref.c memcpy gather (the reference moves no bytes: "
                                       f"SPEC.md:106), {threads} threads, {sample}"},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_sim": {"what": "desim::run_offline of the reference (oracle/_ref, 1 thread) on the "
                                      f"first {sim_sessions} sessions of the same trace and config",
                              "wall_s": round(sim_wall, 3), "decisions": len(rep["decisions"]),
                              "decisions_digest": h.hexdigest(),
                              "model_gbps": round(sum(u[4] for u in rep["usage"] if u[0] == "snic_read")
                                                  / rep["makespan"] / 1e9, 3) if rep["makespan"] > 0 else None},
            "same_config_as": "bench.py --impl ours with the same flags (config dict built identically)"}


def storage_balance(spans, caps, n_engines, width=0.05, window=4):
    """Windowed max/avg of per-engine storage-read traffic (the paper's SNIC
    balance metric, load_balance_ratio proj/src/metrics.cpp:9-42) from the
    executor's measured storage spans; with caps, also per-NIC utilisation."""
    import paper_2602_21548_b200 as dp
    if not spans or not any(spans.values()):
        return None
    end = max(t1 for ss in spans.values() for _, t1, _ in ss)
    nb = int(end / width) + 1

    def series(norm):
        out = []
        for e in range(n_engines):
            b = [0.0] * nb
            for t0, t1, nbytes in spans.get(e, []):
                rate = nbytes / max(t1 - t0, 1e-12) / (norm[e] if norm else 1.0)
                k0, k1 = int(t0 / width), int(t1 / width)
                for k in range(k0, min(k1, nb - 1) + 1):
                    lo, hi = max(t0, k * width), min(t1, (k + 1) * width)
                    if hi > lo:
                        b[k] += rate * (hi - lo)
            out.append(b)
        return out

    def mean_ratio(ser):
        pts = [m for _, m, ok in dp.load_balance_ratio(ser, width, window) if ok]
        return round(sum(pts) / len(pts), 4) if pts else None
    res = {"bytes_max_avg": mean_ratio(series(None)), "bucket_s": width, "window": window}
    if caps:
        res["utilisation_max_avg"] = mean_ratio(series(caps))
    return res


# --------------------------------------------------------------------- main
def relaunch_under_torchrun(n):
    """`python bench.py --gpus N` without an external launcher: re-run this
    script as N ranks under torch.distributed.run (one process per GPU)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def policy_rate(res, K):
    s = sum(res["dev_ms"]) / 1e3
    return res["info"]["hit_bytes"] * K / s / 1e9, res["info"]["prompt_tokens"] * K / s


def plan_block(info, kind, sessions, P, D, cap_gbps, link_bps):
    key = golden_key(kind, sessions, P, D, info["policy"], cap_gbps, link_bps)
    return dict({"decisions": info["decisions"], "decisions_digest": info["digest"], "golden_key": key},
                **golden_check(key, info["digest"]),
                de_path_requests=info["de_path"],
                read_gb_per_engine=[round(x / 1e9, 2) for x in info["reader_bytes"]],
                last_step_ms_per_engine=info["per_engine_ms"], pool_slots=info["pool_slots"],
                store_fb_per_engine=info["store_fb"], plan_s=round(info["plan_s"], 2))


def capped_subrun(args, dist, n, P, D):
    """BASELINE config 2 in the same line: 32K-128K contexts, every engine's
    storage NIC capped (6.25 GB/s = a 400 Gbps SNIC per 8 GPUs), dual path vs
    1-path -- the regime of the paper's headline (storage-bound prefill)."""
    import copy
    sub = copy.copy(args)
    sub.cap_gbps, sub.steps, sub.warmup = args.capped_gbps, args.capped_steps, 1
    sub.prefill = sub.handoff = sub.persist = False
    sub.tier, sub.online, sub.caps = "", 0.0, ""
    sessions = args.capped_sessions_per_gpu * n
    trajs, shape = workload(sub, n, kind="c2", sessions=sessions)
    out = {}
    for name in ("dual_path", "pe_only"):
        r = run_policy(sub, dist, (name, "adaptive"), trajs, shape, P, D, None)
        v, tok = policy_rate(r, sub.steps)
        out[name] = (v, tok, r["info"])
    if dist.rank != 0:
        return None
    (dv, dt, di), (pv, pt, pi) = out["dual_path"], out["pe_only"]
    stats = (di["requests"], di["hit_bytes"], di["prompt_tokens"])
    return {"config": config_dict("c2", sessions, P, D, "dual_path", shape, sub.cap_gbps, stats),
            "steps": sub.steps, "warmup": 1,
            "value": round(dv, 3), "unit": "GB/s", "tokens_per_s": round(dt, 1),
            "model_prediction_gbps": round(di["model_gbps"], 3) if di["model_gbps"] else None,
            "ceiling_gbps": round((P + D) * sub.cap_gbps, 3),
            "one_path": {"value": round(pv, 3), "tokens_per_s": round(pt, 1),
                         "ceiling_gbps": round(P * sub.cap_gbps, 3),
                         "plan": plan_block(pi, "c2", sessions, P, D, sub.cap_gbps, PCIE_ZC_BPS)},
            "dual_vs_one_path": round(dv / pv, 3), "tokens_dual_vs_one_path": round(dt / pt, 3),
            "plan": plan_block(di, "c2", sessions, P, D, sub.cap_gbps, PCIE_ZC_BPS)}


def traffic_for(launch_bytes, mode):
    """DRAM bytes of the K1 call measure_k1 runs, from the committed ncu
    --set full capture of that same call (profiles/k1_traffic*.json)."""
    path = os.path.join(ROOT, "profiles", "k1_traffic.json" if mode == "sm" else f"k1_traffic_{mode}.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        t = json.load(f)
    if t.get("launch_bytes") != launch_bytes:
        return None, None
    if t.get("scatter_kernel"):  # staged: the copy engine carries the bytes; the kernel only scatters
        return t["dram_bytes"], dict(t["scatter_kernel"], note=t["source"])
    return t["dram_bytes"], t["source"]


def main():
    args = parse()
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        print(json.dumps(reference_arm(args)))
        return
    n = args.gpus
    if n > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(n))
    import paper_2602_21548_b200 as dp  # noqa: F401  (fails loudly without the extension)
    from paper_2602_21548_b200 import abi
    dist = make_group(n)
    trajs, shape = workload(args, n)
    sessions = len(trajs)
    if args.pd:
        P, D = (int(x) for x in args.pd.split(":"))
    else:
        P, D = (1, 1) if n == 1 else (n // 2, n - n // 2)
    if args.online > 0:
        variants = [("dual_path", "adaptive"), ("dual_path", "round_robin")]
    elif n == 1:
        variants = [("pe_only", "adaptive")]
    else:
        variants = [("dual_path", "adaptive")] + ([] if args.no_one_path else [("pe_only", "adaptive")])
    policies = [v[0] if v[1] == "adaptive" else v[1] for v in variants]
    peak = None
    if dist.rank == 0:
        peak = measure_pcie_peak(my_device(dist))
    # the box's aggregate host-link ceiling (reported; the planner's link
    # model uses it only with --link-model measured)
    concurrent = measure_concurrent_h2d(dist, my_device(dist)) if dist.world > 1 else None
    link_bps = link_per_engine(concurrent, n) if args.link_model == "measured" else PCIE_ZC_BPS
    numa = dist.allgather(abi.device_numa_node(my_device(dist)))
    results = {}
    clocks = ClockSampler(os.path.join(ROOT, "gpurun_out", f"clocks_bench_{os.getpid()}.csv")
                          if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_{os.getpid()}.csv")
    for name, var in zip(policies, variants):
        results[name] = run_policy(args, dist, var, trajs, shape, P, D,
                                   clocks if (name == policies[0] and dist.local == 0) else None,
                                   link_bps=link_bps)
    if args.prefill:  # the same loads without the prefill: the overlap baseline
        results["load_only"] = run_policy(args, dist, variants[0], trajs, shape, P, D, None, prefill=False,
                                          link_bps=link_bps)
    capped = None
    if n > 1 and not args.no_capped and args.online == 0 and not args.caps:
        capped = capped_subrun(args, dist, n, P, D)
    head = results[policies[0]]
    info = head["info"]
    dev_s = sum(head["dev_ms"]) / 1e3
    host_s = sum(head["host_ms"]) / 1e3
    K = args.steps
    value = info["hit_bytes"] * K / dev_s / 1e9
    e2e = info["hit_bytes"] * K / host_s / 1e9
    tokens_s = info["prompt_tokens"] * K / dev_s
    cpu = None
    if dist.rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(head["xp"], shape)
        except Exception as exc:  # reported, never fatal to the GPU number
            cpu = {"error": str(exc)[:200]}
    clk = clocks.summary(set(range(n)))
    if dist.rank == 0:
        # the dominant kernel alone (K1, one launch of 64 requests), for the
        # ncu capture of the same launch
        k1_mode = "staged" if args.k1 == "staged" else "sm"
        k1_alone, k1_ms, k1_bytes = measure_k1(my_device(dist), shape, k1_mode, args.stage_ctas)
        # roofline: rank 0's engine over the timed steps -- the PE's loads
        # (K1 launches back to back on its load stream; at N > 1 also the
        # wait for the DE pushes landing in its pool): algorithmic bytes
        # C*L*b / CUDA-event time on that stream
        achieved = info["r0_bytes"] / (info["r0_ms"] * 1e-3) / 1e9 if info["r0_ms"] > 0 else None
        traffic, traffic_src = traffic_for(k1_bytes, k1_mode)
        stats = (info["requests"], info["hit_bytes"], info["prompt_tokens"])
        extra = {"pd": args.pd} if args.pd else None
        out = {
            "metric": "aggregate KV-load GB/s",
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": n,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": round(dev_s * 1e3 / K, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic",
            "config": config_dict(args.workload, sessions, P, D, info["policy"] if args.online == 0 else
                                  "dual_path", shape, args.cap_gbps, stats, extra),
            "plan": plan_block(info, args.workload, sessions, P, D, args.cap_gbps, link_bps),
            "loaders": {"k1": args.k1, "k2": args.k2, "stage_ctas": args.stage_ctas,
                        "stage_push_ctas": args.stage_push_ctas,
                        "stage_scatter": args.stage_scatter,
                        "handoff_ctas": args.handoff_ctas or None,
                        "k3": args.k3 if (args.handoff or args.persist) else None,
                        "k4": args.persist_mode if args.persist else None,
                        "pool_layout": args.pool_layout,
                        "buffer_stalls": info["buffer_stalls"],
                        "buffer_wait_ms": round(info["buffer_wait_ms"], 1)},
            "model_prediction_gbps": round(info["model_gbps"], 3) if info["model_gbps"] else None,
            "tokens_per_s": round(tokens_s, 1),
            "e2e": {"value": round(e2e, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": info["hit_bytes"],
                    "d2h_bytes_per_step": info["d2h"] + info["persist_bytes"],
                    "what": "host wall time of run_step: storage read (pinned host) -> HBM inside, "
                            "then the landed-counter column of every request read back and checked "
                            "(+ K4's persisted tokens with --persist)"},
            "gpu_launches": info["launches"],
            "roofline": {"bound": "pcie", "achieved": round(achieved, 2) if achieved else None,
                         "peak": round(peak / 1e9, 2) if peak else None, "unit": "GB/s",
                         "frac": round(achieved / (peak / 1e9), 4) if (peak and achieved) else None,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": {"sm": "kv_gather<false> (K1)",
                                    "staged": "K1 staged: copy-engine Full-Block runs into the HBM ring "
                                              "+ kv_gather<false> scatter (dp_h2d_layer_staged)"}.get(
                                        args.k1, f"K1 ({args.k1})"),
                         "achieved_what": "rank 0's PE: hit bytes it loaded / CUDA-event time of its "
                                          "load stream over the timed steps",
                         "kernel_alone": {"mode": k1_mode, "achieved": round(k1_alone, 2), "launch_bytes": k1_bytes,
                                          "launch_ms": round(k1_ms, 3),
                                          "frac": round(k1_alone / (peak / 1e9), 4) if peak else None},
                         "peak_source": "cudaMemcpyAsync H2D 1 GiB pinned (copy engine), best of 5, "
                                        "measured in this run (MEASURED_PEAKS.json has no PCIe entry)",
                         "frac_of_box_share": (round(achieved / (concurrent / 1e9 / n), 4)
                                               if (concurrent and achieved) else None),
                         "box_share_what": "achieved / (all GPUs' concurrent copy-engine H2D / N): on boxes "
                                           "whose GPUs share host links the per-GPU link peak is not "
                                           "reachable by all at once"},
            "cpu_baseline": cpu,
            "clocks": clk,
            "numa_node_per_rank": numa,
            "host_links": ({"concurrent_h2d_gbps": round(concurrent / 1e9, 2),
                            "value_frac": round(value / (concurrent / 1e9), 4),
                            "planner_link_gbps": round(link_bps / 1e9, 2), "link_model": args.link_model,
                            "what": "all ranks' copy-engine H2D at once: the box's aggregate host-link "
                                    "ceiling for this line"} if concurrent else None),
        }
        if args.online > 0:
            out["config"]["online_sessions_per_s"] = args.online
            out["config"]["caps_gbps"] = [float(x) for x in args.caps.split(",")] if args.caps else None
            out["balance"] = {"adaptive": storage_balance(info["spans"], info["caps"], P + D)}
            if "round_robin" in results:
                rr = results["round_robin"]
                rr_v, _ = policy_rate(rr, K)
                out["round_robin"] = {"value": round(rr_v, 3), "unit": "GB/s",
                                      "adaptive_vs_rr": round(value / rr_v, 3)}
                out["balance"]["round_robin"] = storage_balance(rr["info"]["spans"], rr["info"]["caps"], P + D)
        if args.persist:
            out["persist"] = {"bytes_per_step": info["persist_bytes"],
                              "gbps": round(info["persist_bytes"] * K / dev_s / 1e9, 3),
                              "what": "decode stand-in + K4 D2H Full-Block gather every 64 generated "
                                      "tokens + final partial (PersistD2H ledger of the reference)"}
        if args.handoff or args.persist:
            tt = sorted(info["ttft_ms"] or [0.0])
            lag = sorted(info["lag_ms"] or [0.0])
            out["handoff_latency_ms"] = {
                "what": "per request (rank 0's PE, last timed step): step start -> whole prompt KV in "
                        "its DE's decode pool (offline TTFT of the prefill path); lag = that minus the end "
                        "of the forward that finishes it",
                "layerwise": args.layerwise,
                "ttft_mean": round(sum(tt) / len(tt), 3), "ttft_p50": round(tt[len(tt) // 2], 3),
                "ttft_p99": round(tt[min(len(tt) - 1, int(len(tt) * 0.99))], 3),
                "lag_mean": round(sum(lag) / len(lag), 3), "lag_p99": round(lag[min(len(lag) - 1, int(len(lag) * 0.99))], 3)}
            out["handoff"] = {"bytes_per_step": info["handoff_bytes"],
                              "gbps": round(info["handoff_bytes"] * K / dev_s / 1e9, 3),
                              "what": "PeToDe/MissMerge per layer into DE decode pools (K3, NVLink) "
                                      "+ prefill stand-in; DE read path fused with DecodeH2D"}
        if args.tier:
            out["tier"] = dict(info["tier"], what="StorageRead = pread of Full Block records (trie lookup) "
                                                  "into a pinned staging ring, then K1/K2")
            out["config"]["storage"] = "file tier (" + ("O_DIRECT" if info["tier"]["direct"] else "buffered") + ")"
        if args.prefill:
            pf = info["prefill"]
            lo = results["load_only"]
            lo_ms = sum(lo["dev_ms"]) / K
            step_ms = dev_s * 1e3 / K
            both = pf["compute_alone_ms"]
            out["prefill"] = {
                "what": "quota-batched forwards (build_forward_batch) of K5 attention-score passes "
                        "over the landed KV, layer l gated on the batch's landed counters",
                "quota_ms_per_layer": args.quota_ms, "cost_model": prefill_cost(args, shape),
                "forwards_per_step": pf["forwards_per_step"],
                "prompt_tokens_per_s": round(tokens_s, 1),
                "step_ms": round(step_ms, 3), "load_only_ms": round(lo_ms, 3),
                "compute_alone_ms": both,
                "overlap": round((lo_ms + both - step_ms) / min(lo_ms, both), 3) if min(lo_ms, both) > 0 else None,
                "k5_tmacs": round(pf["macs_per_step"] / (both * 1e-3) / 1e12, 2) if both > 0 else None,
                "cost_model_s_per_step": round(pf["est_s_per_step"], 4)}
        if "pe_only" in results and n > 1:
            po = results["pe_only"]
            po_v, po_tok = policy_rate(po, K)
            out["one_path"] = {"value": round(po_v, 3), "unit": "GB/s", "tokens_per_s": round(po_tok, 1),
                               "dual_vs_one_path": round(value / po_v, 3),
                               "plan": plan_block(po["info"], args.workload, sessions, P, D, args.cap_gbps,
                                                  link_bps)}
        if capped:
            out["storage_capped"] = capped
        print(json.dumps(out))
    dist.barrier()
    dist.close()


if __name__ == "__main__":
    main()
