#!/usr/bin/env python
"""Profiling driver: one K1 (and, with --k2 and 2 GPUs, one K2) launch of a
realistic size through the C ABI, timed with CUDA events on the launching
stream.  --ctas sweeps the gather CTA cap (dp_set_gather_ctas).  Used plain
and under ncu (profiles/)."""

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_21548_b200 import abi  # noqa: E402


def one(kind, a, g, L, T, b, n_fb, n_slots):
    src_dev = 1 if kind == "k2" else 0
    st = abi.Store(src_dev, g, n_fb, 9)
    pool = abi.Pool(0, g, n_slots, a.jobs)
    dst = pool.peer_view(1) if kind == "k2" else pool
    try:
        rng = np.random.default_rng(0)
        keep, specs = [], []
        perm = rng.permutation(n_slots)
        for j in range(a.jobs):
            fbs = torch.tensor(rng.integers(0, n_fb, a.blocks), dtype=torch.int64, device=f"cuda:{src_dev}")
            sl = torch.tensor(perm[(j * a.blocks) % n_slots:][:a.blocks].astype(np.int32),
                              device=f"cuda:{src_dev}")
            keep += [fbs, sl]
            specs.append((fbs.data_ptr(), sl.data_ptr(), a.blocks * T, a.blocks, 0, L, j))
        jobs = abi.make_jobs(specs)
        nbytes = a.jobs * a.blocks * T * b * L
        s = torch.cuda.Stream(device=src_dev)
        times = []
        for r in range(a.reps + 1):
            pool.reset_counters()
            torch.cuda.synchronize(0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(src_dev):
                e0.record(s)
                if kind == "k1":
                    abi.h2d_layer_gather(dst, st, jobs, len(specs), s.cuda_stream)
                else:
                    abi.h2d_push_p2p_layer(dst, st, jobs, len(specs), s.cuda_stream)
                e1.record(s)
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        ms = sorted(times)[len(times) // 2]
        return {"bytes": nbytes, "ms": ms, "GBps": nbytes / ms / 1e6}
    finally:
        if dst is not pool:
            dst.close()
        pool.close()
        st.close()


def k3(a, g, L, T, b, n_fb, n_slots, ce=False, contiguous=False):
    """K3 alone (PE path: push the whole prompt of each job, C = 7/8 of it).
    ce: dp_prefill_handoff_copy (copy engines + side kernel); contiguous: the
    jobs' slots are consecutive runs in both pools (the executor's FIFO
    allocation) instead of a random permutation."""
    st = abi.Store(0, g, n_fb, 9)
    pool = abi.Pool(0, g, n_slots, 2 * a.jobs)
    de_pool = abi.Pool(1, g, n_slots, a.jobs)
    de_view = de_pool.peer_view(0)
    try:
        rng = np.random.default_rng(0)
        keep, specs, ho = [], [], (abi.HandoffJob * a.jobs)()
        perm = rng.permutation(n_slots)
        for j in range(a.jobs):
            fbs = torch.tensor(rng.integers(0, n_fb, a.blocks), dtype=torch.int64, device="cuda:0")
            idx = (np.arange(j * a.blocks, (j + 1) * a.blocks) % n_slots) if contiguous else \
                perm[(j * a.blocks) % n_slots:][:a.blocks]
            sl_h = idx.astype(np.int32)
            fb_h = fbs.cpu().numpy()
            sl = torch.tensor(sl_h, device="cuda:0")
            keep += [fbs, sl, sl_h, fb_h]
            prompt = a.blocks * T
            cached = prompt * 7 // 8
            specs.append((fbs.data_ptr(), sl.data_ptr(), cached, -(-cached // T), 0, L, j))
            if ce:
                ho[j] = abi.HandoffJob(fb_h.ctypes.data, sl_h.ctypes.data, sl_h.ctypes.data, cached, prompt,
                                       a.blocks, 1, -1, 0, j, a.jobs + j)
            else:
                ho[j] = abi.HandoffJob(fbs.data_ptr(), sl.data_ptr(), sl.data_ptr(), cached, prompt, a.blocks,
                                       1, -1, 0, j, a.jobs + j)
        abi.h2d_layer_gather(pool, st, abi.make_jobs(specs), len(specs))
        torch.cuda.synchronize(0)
        nbytes = a.jobs * a.blocks * T * b * L
        times = []
        s = torch.cuda.Stream(device=0)
        for r in range(a.reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if ce:
                abi.prefill_handoff_copy(pool, de_view, ho, a.jobs, 9, 20000, s.cuda_stream)
            else:
                abi.prefill_handoff(pool, de_view, ho, a.jobs, 9, 20000, s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        ms = sorted(times)[len(times) // 2]
        return {"bytes": nbytes, "ms": ms, "GBps": nbytes / ms / 1e6}
    finally:
        de_view.close()
        de_pool.close()
        pool.close()
        st.close()


def k4(a, g, L, T, b, n_fb, n_slots, staged=False):
    """K4 alone (PersistD2H): every token of a.jobs requests of a.blocks blocks
    gathered from the decode pool into storage Full Blocks in pinned host
    memory (zero-copy stores over PCIe D2H; staged: gather into an HBM ring,
    copy engine to the host)."""
    pool = abi.Pool(0, g, n_slots, 1)
    target = abi.Store(0, g, n_fb, 10)
    stager = abi.Stager(0, g) if staged else None
    try:
        rng = np.random.default_rng(0)
        keep, spans, hspans = [], (abi.SpanJob * a.jobs)(), (abi.SpanJob * a.jobs)()
        perm = rng.permutation(n_slots)
        for j in range(a.jobs):
            if staged:  # a request persists into its session's consecutive Full Blocks (the executor's fb_of)
                fbs = torch.tensor(np.arange(j * a.blocks, (j + 1) * a.blocks) % n_fb, dtype=torch.int64,
                                   device="cuda:0")
            else:
                fbs = torch.tensor(rng.integers(0, n_fb, a.blocks), dtype=torch.int64, device="cuda:0")
            sl = torch.tensor(perm[(j * a.blocks) % n_slots:][:a.blocks].astype(np.int32), device="cuda:0")
            fbs_h = fbs.cpu().numpy()
            keep += [fbs, sl, fbs_h]
            spans[j] = abi.SpanJob(sl.data_ptr(), fbs.data_ptr(), 0, 0, a.blocks * T, a.blocks, 0)
            if staged:
                hspans[j] = abi.SpanJob(sl.data_ptr(), fbs_h.ctypes.data, 0, 0, a.blocks * T, a.blocks, 0)
        abi.decode_fill(pool, spans, a.jobs, 9)
        torch.cuda.synchronize(0)
        nbytes = a.jobs * a.blocks * T * b * L
        times = []
        s = torch.cuda.Stream(device=0)
        for r in range(a.reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if staged:
                abi.persist_staged(pool, target, stager, hspans, a.jobs, s.cuda_stream)
            else:
                abi.persist_d2h(pool, target, spans, a.jobs, s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        ms = sorted(times)[len(times) // 2]
        # the copy-engine D2H peak for comparison
        h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
        d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
        best = 1e9
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            with torch.cuda.stream(s):
                h.copy_(d, non_blocking=True)
            e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        # the same copy into the target store's own pages (NUMA-bound,
        # registered): the ceiling for K4, whose bytes land there
        rt = ctypes.CDLL("libcudart.so.12")
        rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        host, tbytes, _ = target.info()
        n = min(1 << 30, tbytes)
        best_st = 1e9
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            assert rt.cudaMemcpyAsync(host, d.data_ptr(), n, 2, s.cuda_stream) == 0  # cudaMemcpyDeviceToHost
            e1.record(s)
            e1.synchronize()
            best_st = min(best_st, e0.elapsed_time(e1))
        return {"bytes": nbytes, "ms": ms, "GBps": nbytes / ms / 1e6, "ce_d2h_GBps": (1 << 30) / best / 1e6,
                "ce_d2h_store_GBps": n / best_st / 1e6}
    finally:
        if stager:
            stager.close()
        pool.close()
        target.close()


def ce_peer():
    """cudaMemcpyPeerAsync of 1 GiB device 0 -> device 1, best of 5: the copy
    engine's NVLink rate, the practical ceiling K3 is compared with."""
    n = 1 << 30
    a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    s = torch.cuda.Stream(device=0)
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            b.copy_(a, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return {"bytes": n, "ms": best, "GBps": n / best / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k2", action="store_true")
    ap.add_argument("--k3", action="store_true")
    ap.add_argument("--k3-ctas", default="0")
    ap.add_argument("--k3-tma", default="off", choices=["off", "on", "both"])
    ap.add_argument("--peer", action="store_true", help="also the copy-engine peer copy of 1 GiB (0 -> 1)")
    ap.add_argument("--k4", action="store_true")
    ap.add_argument("--jobs", type=int, default=64)
    ap.add_argument("--blocks", type=int, default=128)  # 8K-token requests
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--shape", default="dsv3", choices=["dsv3", "qwen"])
    ap.add_argument("--ctas", default="0", help="comma list of gather CTA caps (0 = default)")
    a = ap.parse_args()
    L, T, b = (61, 64, 576) if a.shape == "dsv3" else (64, 64, 4096)
    g = abi.geom(L, T, b)
    n_fb = 2048 if a.shape == "dsv3" else 256
    n_slots = a.jobs * a.blocks if a.shape == "dsv3" else min(a.jobs * a.blocks, 4096)
    out = {}
    for ctas in [int(x) for x in a.ctas.split(",")]:
        for dev in range(torch.cuda.device_count()):
            abi.set_gather_ctas(dev, ctas)
        for kind in ["k1"] + (["k2"] if a.k2 else []):
            out[kind if ctas == 0 else f"{kind}@{ctas}"] = one(kind, a, g, L, T, b, n_fb, n_slots)
    for dev in range(torch.cuda.device_count()):
        abi.set_gather_ctas(dev, 0)
    if a.k3:
        for tma in ([False, True] if a.k3_tma == "both" else [a.k3_tma == "on"]):
            abi.set_handoff_tma(tma)
            for ctas in [int(x) for x in a.k3_ctas.split(",")]:
                abi.set_handoff_ctas(0, ctas)
                key = ("k3_tma" if tma else "k3") + ("" if ctas == 0 else f"@{ctas}")
                out[key] = k3(a, g, L, T, b, n_fb, n_slots)
        abi.set_handoff_ctas(0, 0)
        abi.set_handoff_tma(False)
        out["k3_contiguous"] = k3(a, g, L, T, b, n_fb, n_slots, contiguous=True)
        out["k3_ce_contiguous"] = k3(a, g, L, T, b, n_fb, n_slots, ce=True, contiguous=True)
        out["k3_ce_scattered"] = k3(a, g, L, T, b, n_fb, n_slots, ce=True)
    if a.peer:
        out["ce_peer_copy"] = ce_peer()
    if a.k4:
        out["k4"] = k4(a, g, L, T, b, n_fb, n_slots)
        out["k4_staged"] = k4(a, g, L, T, b, n_fb, n_slots, staged=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
