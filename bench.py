#!/usr/bin/env python
"""DualPath KV-Cache loading benchmark on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c1|c2] [--cap-gbps X] [--sessions-per-gpu S]

N = 1: the K1 loader alone (the PE of a 1P1D prefill-only plan; P/D needs
two engines, proj/src/types.cpp:11-12).  N > 1: one process per GPU under
torchrun, engines 0..N/2-1 prefill (PE), the rest decode (DE), dual-path
plan; the same workload is also run prefill-only ("1-path",
Policy::PEOnly, proj/src/desim.cpp:826-827) for the vs-1-path ratio.

A step = one offline pass of the synthetic agentic trace: every request's
hit KV (C*L*b bytes) moved from the emulated storage tier (pinned host DRAM,
read over each engine's own PCIe link, optionally rate-capped per engine)
into the PE's paged HBM pool, by K1 (PE path) or K2 (DE path, NVLink push).
Inputs are larger than L2 (hundreds of GB per step), so no flush is needed.
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
    ap.add_argument("--sessions-per-gpu", type=int, default=16)
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
    ap.add_argument("--k2", default="sm", choices=["sm", "ce"],
                    help="DE-path loads: sm = K2 gather pushing over NVLink, ce = the DE's copy engine")
    ap.add_argument("--k1", default="sm", choices=["sm", "ce", "hybrid"],
                    help="PE-path loads: sm = K1 gather kernel, ce = copy engine (no SMs), "
                         "hybrid = both at once, jobs split by bytes")
    return ap.parse_args()


# ----------------------------------------------------------------- workload
def workload(args, n_gpus):
    """Trajectories + KV shape.  c1: BASELINE config 1 generator (20 turns,
    mean append 429, mean gen 500, ~95% hit); c2: 32K/64K/128K contexts built
    by one cold prefill round {C, 1}, then warm {429, 1} rounds (config 2; a
    cold append instead of the reference tests' long generation round, whose
    64-token persistence flows would dominate planning); c3: c1 with the
    Qwen2.5-32B KV shape (config 3)."""
    import paper_2602_21548_b200 as dp
    sessions = max(1, args.sessions_per_gpu * max(1, n_gpus))
    if getattr(args, "trace", ""):
        trajs = dp.load_trace(args.trace)[:sessions]
        if not trajs:
            raise SystemExit(f"--trace {args.trace}: no sessions")
        return trajs, (QWEN if args.workload == "c3" else DSV3)
    if args.workload in ("c1", "c3"):
        trajs = dp.synthesize(max_len=131072, count=sessions, seed=9, mean_turns=20,
                              sigma_turns=0.0, mean_append=429, mean_gen=500)
        shape = DSV3 if args.workload == "c1" else QWEN
    else:
        trajs = []
        for i in range(sessions):
            t = dp.Trajectory()
            t.id = f"ctx{i}"
            c = (32768, 65536, 131072)[i % 3]
            t.rounds = [dp.Round(c - 1, 1)] + [dp.Round(429, 1) for _ in range(3)]
            trajs.append(t)
        shape = DSV3
    return trajs, shape


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
    cfg.pe_buffer_bytes = 1 << 42
    cfg.de_buffer_bytes = 1 << 42
    return cfg


# ncu --set full of the K1 launch (profiles/r01_k1_full.ncu-rep): dram read +
# write bytes per launch over the launch's algorithmic bytes (18.42 GB)
TRAFFIC = {"c1": 18454911288, "c2": 18454911288}  # 85.6 MB read + 18.37 GB write

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


def measure_k1(device, shape, target_bytes=18421383168):
    """The dominant kernel alone, live: one K1 launch (DS-V3 or Qwen Layer
    Blocks, 8K-token requests, random Full Blocks and slots) through the C
    ABI, CUDA events on its stream, median of 3 after a warm-up."""
    import numpy as np
    import torch
    from paper_2602_21548_b200 import abi
    L, T, b = shape["L"], shape["T"], shape["b"]
    blocks = 128
    per_job = blocks * T * b * L
    jobs_n = max(1, min(64, target_bytes // per_job))  # DS-V3: the 64-job launch ncu profiled
    g = abi.geom(L, T, b)
    n_fb = max(blocks, (2 << 30) // (L * T * b))
    st = abi.Store(device, g, n_fb, 9)
    pool = abi.Pool(device, g, jobs_n * blocks, jobs_n)
    try:
        rng = np.random.default_rng(0)
        keep, specs = [], []
        perm = rng.permutation(jobs_n * blocks).astype(np.int32)
        for j in range(jobs_n):
            f = torch.tensor(rng.integers(0, n_fb, blocks), dtype=torch.int64, device=f"cuda:{device}")
            sl = torch.tensor(perm[j * blocks:(j + 1) * blocks], device=f"cuda:{device}")
            keep += [f, sl]
            specs.append((f.data_ptr(), sl.data_ptr(), blocks * T, blocks, 0, L, j))
        jobs = abi.make_jobs(specs)
        s = torch.cuda.Stream(device=device)
        times = []
        for r in range(4):
            pool.reset_counters(s.cuda_stream)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(device):
                e0.record(s)
                abi.h2d_layer_gather(pool, st, jobs, len(specs), s.cuda_stream)
                e1.record(s)
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        ms = sorted(times)[1]
        nbytes = jobs_n * per_job
        return nbytes / (ms * 1e-3) / 1e9, ms, nbytes
    finally:
        pool.close()
        st.close()


def prefill_cost(args, shape):
    """Cost model of the prefill stand-in per layer (AttentionCostModel):
    K5 does bsz * cached * b multiply-adds per request chunk (bilinear), plus
    a fixed per-layer cost of the gate and the launch (constant)."""
    return (shape["b"] / (args.attend_tops * 1e12), 0.0, 0.0, 20e-6)


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
    opt.k1_mode = {"sm": 0, "ce": 1, "hybrid": 2}[args.k1]
    opt.k2_mode = 1 if args.k2 == "ce" else 0
    opt.wait_timeout_ms = args.wait_timeout_ms
    opt.handoff = bool(args.handoff or args.persist)
    opt.persist = bool(args.persist)
    opt.handoff_ctas = args.handoff_ctas
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
    digests = dist.allgather(dpdist.plan_digest(planned))
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
    info = dict(plan_s=plan_s, hit_bytes=xp.hit_bytes, prompt_tokens=xp.prompt_tokens,
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
def reference_arm(args):
    """The reference's own CPU implementation of the path: pdsim's
    desim::run_offline, compiled from /root/reference sources into
    oracle/_ref, run on this box's host (single-threaded by design,
    SPEC.md:403) on a session sample of the same workload and P:D config.
    The reference moves no bytes; its value of the metric is its own
    aggregate KV-load GB/s for the workload: storage-read bytes / makespan
    (the SnicRead ledger, desim.cpp:405-425, 956-987).  Wall time per run is
    reported beside it."""
    import paper_2602_21548_b200 as dp
    from oracle import refpy
    n = args.gpus
    trajs, shape = workload(args, n)
    P, D = (1, 1) if n == 1 else (n // 2, n - n // 2)
    if args.pd:
        P, D = (int(x) for x in args.pd.split(":"))
    cap = args.cap_gbps * 1e9
    # the same per-engine link rate our arm plans with on this box
    ceiling = measure_host_ceiling_local(n) if n > 1 else None
    link_bps = link_per_engine(ceiling, n)
    cfg = cluster(shape, P, D, cap, None, link_bps)
    sample = trajs[: max(2, min(len(trajs), 4 * n))]
    path = f"/tmp/dp_ref_sample_{os.getpid()}.tsv"
    dp.save_trace(path, sample)
    kv = dict(P=P, D=D, g=1, L=shape["L"], b=shape["b"], T=shape["T"], B=cfg.cnic_bandwidth,
              s=cfg.storage_multiple, M=cfg.dram_bandwidth, hbm=cfg.hbm_capacity_tokens,
              pe_buf=cfg.pe_buffer_bytes, de_buf=cfg.de_buffer_bytes,
              policy="pe_only" if n == 1 else "dual_path", **PLAN_KW)
    vals, walls = [], []
    try:
        for step in range(args.warmup + args.steps):
            t0 = time.time()
            rep = refpy.ref_simulate(path, **kv)
            wall = time.time() - t0
            snic = sum(u[4] for u in rep["usage"] if u[0] == "snic_read")
            if step >= args.warmup:
                vals.append(snic / rep["makespan"] / 1e9)
                walls.append(wall)
    finally:
        os.unlink(path)
    v = statistics.median(vals)
    return {"metric": "aggregate KV-load GB/s", "value": round(v, 3), "unit": "GB/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "impl": "reference",
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {len(sample)} sessions, "
                                   + ("1P loader (pe_only)" if n == 1 else f"{P}P{D}D dual_path"),
                       "kv": shape},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": 1, "kind": "reference",
                             "sample": f"desim::run_offline on {len(sample)} sessions of the workload "
                                       f"(the reference simulator, 1 thread); value = its storage-read "
                                       f"bytes / makespan; {statistics.median(walls):.2f} s wall per run"},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_wall_s_per_run": round(statistics.median(walls), 3),
            "link_model": {"per_engine_gbps": round(link_bps / 1e9, 2),
                           "concurrent_h2d_gbps": round(ceiling / 1e9, 2) if ceiling else None,
                           "what": "the reference simulator's storage rate per engine: the same "
                                   "min(51.5, box ceiling / N) our arm plans with"}}


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
def main():
    args = parse()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        print(json.dumps(reference_arm(args)))
        return
    import paper_2602_21548_b200 as dp  # noqa: F401  (fails loudly without the extension)
    n = args.gpus
    dist = make_group(n)
    trajs, shape = workload(args, n)
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
    # the box's aggregate host-link ceiling, measured before planning: the
    # planner (the reference's model) then uses the per-engine rate this box
    # actually sustains when every engine reads
    concurrent = measure_concurrent_h2d(dist, my_device(dist)) if dist.world > 1 else None
    link_bps = link_per_engine(concurrent, n)
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
    k1 = None
    if dist.rank == 0:
        k1 = measure_k1(my_device(dist), shape)
    if dist.rank == 0:
        # roofline of the dominant kernel, K1 (K2 is the same kernel body with
        # peer stores, 0.999x its rate, profiles/r01_k1_k2_events.json),
        # measured live on rank 0 after the timed steps: algorithmic bytes
        # (C*L*b of the launch) / CUDA-event time of the launch
        achieved, k1_ms, k1_bytes = k1
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
            "config": {"workload": f"{args.workload}: {len(trajs)} sessions, "
                                   + ("1 PE loader (K1)" if n == 1 else f"{P}P{D}D dual_path"),
                       "kv": shape, "storage_cap_gbps_per_engine": args.cap_gbps or None,
                       "k1": args.k1, "k2": args.k2, "handoff_ctas": args.handoff_ctas or None,
                       "requests": info["requests"], "hit_bytes_per_step": info["hit_bytes"],
                       "de_path_requests": info["de_path"],
                       "read_gb_per_engine": [round(x / 1e9, 2) for x in info["reader_bytes"]],
                       "last_step_ms_per_engine": info["per_engine_ms"],
                       "l2": "inputs >> L2 (no flush needed)"},
            "model_prediction_gbps": round(info["model_gbps"], 3) if info["model_gbps"] else None,
            "tokens_per_s": round(tokens_s, 1),
            "e2e": {"value": round(e2e, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": info["hit_bytes"],
                    "d2h_bytes_per_step": info["d2h"] + info["persist_bytes"],
                    "what": "host wall time of run_step: storage read (pinned host) -> HBM inside, "
                            "then the landed-counter column of every request read back and checked "
                            "(+ K4's persisted tokens with --persist)"},
            "gpu_launches": info["launches"],
            "roofline": {"bound": "pcie", "achieved": round(achieved, 2),
                         "peak": round(peak / 1e9, 2) if peak else None, "unit": "GB/s",
                         "frac": round(achieved / (peak / 1e9), 4) if peak else None,
                         "traffic": TRAFFIC.get(args.workload),
                         "kernel": "kv_gather<false> (K1)", "launch_bytes": k1_bytes,
                         "launch_ms": round(k1_ms, 3),
                         "peak_source": "cudaMemcpyAsync H2D 1 GiB pinned, best of 5, measured in this run",
                         "step_rate_per_engine": round(value / max(1, n), 2)},
            "cpu_baseline": cpu,
            "clocks": clk,
            "host_links": ({"concurrent_h2d_gbps": round(concurrent / 1e9, 2),
                            "value_frac": round(value / (concurrent / 1e9), 4),
                            "per_engine_model_gbps": round(link_bps / 1e9, 2),
                            "what": "all ranks' copy-engine H2D at once: the box's aggregate host-link "
                                    "ceiling for this line; the planner's per-engine storage rate is "
                                    "min(51.5, ceiling / N)"} if concurrent else None),
            "plan_s": round(info["plan_s"], 2),
        }
        if args.online > 0:
            out["config"]["online_sessions_per_s"] = args.online
            out["config"]["caps_gbps"] = [float(x) for x in args.caps.split(",")] if args.caps else None
            out["balance"] = {"adaptive": storage_balance(info["spans"], info["caps"], P + D)}
            if "round_robin" in results:
                rr = results["round_robin"]
                rr_s = sum(rr["dev_ms"]) / 1e3
                rr_v = rr["info"]["hit_bytes"] * K / rr_s / 1e9
                out["round_robin"] = {"value": round(rr_v, 3), "unit": "GB/s",
                                      "adaptive_vs_rr": round(value / rr_v, 3)}
                out["balance"]["round_robin"] = storage_balance(rr["info"]["spans"], rr["info"]["caps"], P + D)
        if args.persist:
            out["persist"] = {"bytes_per_step": info["persist_bytes"],
                              "gbps": round(info["persist_bytes"] * K / dev_s / 1e9, 3),
                              "what": "decode stand-in + K4 D2H Full-Block gather every 64 generated "
                                      "tokens + final partial (PersistD2H ledger of the reference)"}
        if args.handoff or args.persist:
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
            po_s = sum(po["dev_ms"]) / 1e3
            po_v = po["info"]["hit_bytes"] * K / po_s / 1e9
            out["one_path"] = {"value": round(po_v, 3), "unit": "GB/s",
                               "tokens_per_s": round(po["info"]["prompt_tokens"] * K / po_s, 1),
                               "dual_vs_one_path": round(value / po_v, 3)}
        print(json.dumps(out))
    dist.barrier()
    dist.close()


if __name__ == "__main__":
    main()
