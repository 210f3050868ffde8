#!/usr/bin/env python
"""BASELINE config 4: a per-layer bf16 GEMM stand-in on the prefill GPU and
the interference of the KV loading path on it.

Single process, two GPUs (PE = cuda:0, DE = cuda:1):

1. isolation: mean GEMM time alone, then while (a) the DE pushes KV into the
   PE pool over NVLink (K2), (b) the PE loads its own KV over PCIe (K1) at
   several copy-CTA caps (dp_set_gather_ctas), (c) both.  The reference's
   isolation bar is <= 2 % slowdown (proj/tests/acceptance.cpp:383-420).
2. layerwise overlap: a 32K-token request's KV is pushed by the DE while the
   PE computes layer l as soon as layer l has landed (dp_wait_layer on the
   compute stream, the maybe_start_compute gate, proj/src/desim.cpp:623-628);
   compare with load-then-compute.

r02: the staged loaders (copy engine into an HBM ring + a scatter kernel of
8 / 32 CTAs) on both sides, and the DE's own compute (a GEMM on the DE)
while it pushes with K2 on SMs or staged.

Prints one JSON object.  GEMMs use torch.matmul (cuBLAS) — a stand-in for
the model's prefill compute, not part of the product path.
"""

import argparse
import json
import time
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_21548_b200 import abi  # noqa: E402

L, T, B = 61, 64, 576


def make_jobs(device, n_jobs, blocks, n_fb, n_slots, rng, layers=(0, L), ticket0=0):
    keep, specs = [], []
    perm = rng.permutation(n_slots)
    for j in range(n_jobs):
        fbs = torch.tensor(rng.integers(0, n_fb, blocks), dtype=torch.int64, device=f"cuda:{device}")
        sl = torch.tensor(perm[(j * blocks) % n_slots:][:blocks].astype(np.int32), device=f"cuda:{device}")
        keep += [fbs, sl]
        specs.append((fbs.data_ptr(), sl.data_ptr(), blocks * T, blocks, layers[0], layers[1], ticket0 + j))
    return abi.make_jobs(specs), keep


def gemm_times(a, b, n, stream, dev=0):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    with torch.cuda.stream(stream):
        for e0, e1 in ev:
            e0.record(stream)
            torch.matmul(a, b)
            e1.record(stream)
    torch.cuda.synchronize(dev)
    return [e0.elapsed_time(e1) for e0, e1 in ev]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--gemms", type=int, default=6000)
    ap.add_argument("--only-staged", action="store_true", help="only the staged-loader cases")
    ap.add_argument("--skip-layerwise", action="store_true")
    ap.add_argument("--ring-mb", default="", help="only K1 staged (scatter kernel) at these HBM ring sizes, MiB")
    ap.add_argument("--block-major", action="store_true",
                    help="only the copy-engine loaders into a block-major PE pool (whole Full-Block runs, no ring)")
    a = ap.parse_args()
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    g = abi.geom(L, T, B)
    n_fb, blocks, n_jobs = 2048, 128, 64
    n_slots = n_jobs * blocks
    st_pe = abi.Store(0, g, n_fb, 9)
    st_de = abi.Store(1, g, n_fb, 9)
    pool = abi.Pool(0, g, n_slots, 2 * n_jobs + 1)
    view = pool.peer_view(1)
    bpool = abi.Pool(0, g, n_slots, 2 * n_jobs + 1, layout=abi.POOL_BLOCK_MAJOR) if a.block_major else None
    bview = bpool.peer_view(1) if bpool else None
    rng = np.random.default_rng(0)
    jobs_k2, keep2 = make_jobs(1, n_jobs, blocks, n_fb, n_slots, rng)
    jobs_k1, keep1 = make_jobs(0, n_jobs, blocks, n_fb, n_slots, rng)
    # the same PE-path load for the copy engine: host block tables, contiguous runs
    ce_keep, ce_specs = [], []
    for j in range(n_jobs):
        fbs = np.arange(j * blocks, (j + 1) * blocks, dtype=np.int64) % n_fb
        sl = np.arange(j * blocks, (j + 1) * blocks, dtype=np.int32) % n_slots
        ce_keep += [fbs, sl]
        ce_specs.append((fbs.ctypes.data, sl.ctypes.data, blocks * T, blocks, 0, L, j))
    jobs_ce = abi.make_jobs(ce_specs)
    # staged (copy engine into an HBM ring + scatter kernel): host src_fb, device slots
    st_keep, st1, st2 = [], [], []
    for j in range(n_jobs):
        fbs = np.arange(j * blocks, (j + 1) * blocks, dtype=np.int64) % n_fb
        s0 = torch.tensor(np.arange(j * blocks, (j + 1) * blocks, dtype=np.int32) % n_slots, device="cuda:0")
        s1 = torch.tensor(np.arange(j * blocks, (j + 1) * blocks, dtype=np.int32) % n_slots, device="cuda:1")
        st_keep += [fbs, s0, s1]
        st1.append((fbs.ctypes.data, s0.data_ptr(), blocks * T, blocks, 0, L, j))
        st2.append((fbs.ctypes.data, s1.data_ptr(), blocks * T, blocks, 0, L, n_jobs + j))
    jobs_st1, jobs_st2 = abi.make_jobs(st1), abi.make_jobs(st2)
    ce1, ce2 = [], []  # the copy-engine scatter reads HOST slot tables
    for j in range(n_jobs):
        fbs = st_keep[3 * j]
        sl = np.arange(j * blocks, (j + 1) * blocks, dtype=np.int32) % n_slots
        st_keep.append(sl)
        ce1.append((fbs.ctypes.data, sl.ctypes.data, blocks * T, blocks, 0, L, j))
        ce2.append((fbs.ctypes.data, sl.ctypes.data, blocks * T, blocks, 0, L, n_jobs + j))
    jobs_ce1, jobs_ce2 = abi.make_jobs(ce1), abi.make_jobs(ce2)
    stager0, stager1 = abi.Stager(0, g), abi.Stager(1, g)
    ring_stagers = {int(r): abi.Stager(0, g, int(r) << 20) for r in a.ring_mb.split(",") if r}
    s_gemm = torch.cuda.Stream(device=0, priority=-1)  # high priority compute
    s_k1 = torch.cuda.Stream(device=0, priority=0)
    s_k2 = torch.cuda.Stream(device=1)
    x = torch.randn(a.m, a.k, device="cuda:0", dtype=torch.bfloat16)
    w = torch.randn(a.k, a.m, device="cuda:0", dtype=torch.bfloat16)
    s_gemm_de = torch.cuda.Stream(device=1, priority=-1)
    x1 = torch.randn(a.m, a.k, device="cuda:1", dtype=torch.bfloat16)
    w1 = torch.randn(a.k, a.m, device="cuda:1", dtype=torch.bfloat16)
    for _ in range(20):
        torch.matmul(x, w)
        torch.matmul(x1, w1)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    flops = 2.0 * a.m * a.m * a.k

    def run_with(k1=False, k2=False, ctas=0, ce=False, staged=False, stage_ctas=32, on_de=False, ce_scatter=False,
                 push_ctas=None, ring=None, block=False):
        for dev in (0, 1):
            abi.set_gather_ctas(dev, ctas)
        stager0.set_ctas(stage_ctas)
        stager1.set_ctas(push_ctas or stage_ctas)
        for sg in (stager0, stager1):
            sg.set_mode(abi.SCATTER_CE if ce_scatter else abi.SCATTER_KERNEL)
        stop = threading.Event()
        done = {"k1": [], "k2": []}  # completion wall times of each loader launch
        per_launch = n_jobs * blocks * T * B * L

        def loader(kind):
            dev, stream = (0, s_k1) if kind == "k1" else (1, s_k2)
            with torch.cuda.device(dev):
                while not stop.is_set():
                    if staged and kind == "k1":
                        abi.h2d_layer_staged(pool, st_pe, ring_stagers[ring] if ring else stager0,
                                             jobs_ce1 if ce_scatter else jobs_st1, n_jobs, stream.cuda_stream)
                    elif staged:
                        abi.h2d_push_staged(view, st_de, stager1, jobs_ce2 if ce_scatter else jobs_st2, n_jobs,
                                            stream.cuda_stream)
                    elif kind == "k1" and ce:
                        abi.h2d_layer_copy_job(bpool if block else pool, st_pe, jobs_ce1, n_jobs, stream.cuda_stream)
                    elif ce:
                        abi.h2d_push_copy_job(bview if block else view, st_de, jobs_ce2, n_jobs, stream.cuda_stream)
                    elif kind == "k1":
                        abi.h2d_layer_gather(pool, st_pe, jobs_k1, n_jobs, stream.cuda_stream)
                    else:
                        abi.h2d_push_p2p_layer(view, st_de, jobs_k2, n_jobs, stream.cuda_stream)
                    stream.synchronize()
                    done[kind].append(time.time())
        ths = [threading.Thread(target=loader, args=(kk,)) for kk, on in (("k1", k1), ("k2", k2)) if on]
        for t in ths:
            t.start()
        time.sleep(0.5)
        t0 = time.time()
        if on_de:  # the DE's own compute (its decode stand-in) while it pushes
            with torch.cuda.device(1):
                ts = gemm_times(x1, w1, a.gemms, s_gemm_de, dev=1)
        else:
            ts = gemm_times(x, w, a.gemms, s_gemm)
        t1 = time.time()
        stop.set()
        for t in ths:
            t.join()
        ts = sorted(ts)[len(ts) // 10: -len(ts) // 10]  # trimmed mean
        mean = sum(ts) / len(ts)
        rates = {}
        for k, ts_done in done.items():
            inside = [t for t in ts_done if t0 <= t <= t1]
            if len(inside) >= 2:  # whole launches completed inside the GEMM window
                rates[k] = round((len(inside) - 1) * per_launch / (inside[-1] - inside[0]) / 1e9, 1)
        return {"gemm_ms": round(mean, 4), "tflops": round(flops / mean / 1e9, 1),
                "window_s": round(t1 - t0, 2), "loader_gbps_during": rates}

    def bracketed(kw, on_de=False):
        """The case between two runs of the GEMM alone on the same GPU (A/B/A):
        the slowdown is against the mean of the two, and `noise_pct` (their
        difference) is the resolution of that number."""
        before = run_with(on_de=on_de)["gemm_ms"]
        r = run_with(on_de=on_de, **kw)
        after = run_with(on_de=on_de)["gemm_ms"]
        alone = 0.5 * (before + after)
        r["alone_ms"] = [before, after]
        r["noise_pct"] = round(100.0 * abs(after - before) / alone, 2)
        r["slowdown_pct"] = round(100.0 * (r["gemm_ms"] / alone - 1.0), 2)
        return r

    out = {"gemm": {"m": a.m, "n": a.m, "k": a.k, "dtype": "bf16"},
           "method": "each case bracketed by the GEMM alone before and after (A/B/A); trimmed mean of "
                     "per-GEMM CUDA-event times"}
    out["alone"] = run_with()
    base = out["alone"]["gemm_ms"]
    out["de_alone"] = run_with(on_de=True)
    base_de = out["de_alone"]["gemm_ms"]
    for name, kw in [("de_k2_sm", dict(k2=True)), ("de_k2_staged", dict(k2=True, staged=True)),
                     ("de_k2_staged_ce", dict(k2=True, staged=True, ce_scatter=True)),
                     ("de_k2_staged_148ctas", dict(k2=True, staged=True, push_ctas=148)),
                     ("de_k2_staged_8ctas", dict(k2=True, staged=True, stage_ctas=8)),
                     ("de_k2_copy_engine", dict(k2=True, ce=True))]:
        if a.block_major or a.ring_mb:
            break  # the focused sweeps below
        out[name] = bracketed(kw, on_de=True)
    ce_cases = [("k1_copy_engine_job", dict(k1=True, ce=True)), ("k2_copy_engine_job", dict(k2=True, ce=True)),
                ("k1_copy_engine_job+k2_copy_engine_job", dict(k1=True, k2=True, ce=True)),
                ("k2_staged_148ctas", dict(k2=True, staged=True, push_ctas=148)),
                ("k1_staged+k2_staged_148ctas", dict(k1=True, k2=True, staged=True, push_ctas=148)),
                ("k1_staged_ce", dict(k1=True, staged=True, ce_scatter=True)),
                ("k2_staged_ce", dict(k2=True, staged=True, ce_scatter=True)),
                ("k1_staged_ce+k2_staged_ce", dict(k1=True, k2=True, staged=True, ce_scatter=True))]
    if a.block_major:
        for name, kw, de in [("k1_ce_block_major", dict(k1=True, ce=True, block=True), False),
                             ("k2_ce_block_major", dict(k2=True, ce=True, block=True), False),
                             ("k1_ce_block_major+k2_ce_block_major", dict(k1=True, k2=True, ce=True, block=True), False),
                             ("de_k2_ce_block_major", dict(k2=True, ce=True, block=True), True)]:
            out[name] = bracketed(kw, on_de=de)
        print(json.dumps(out))
        return
    if a.ring_mb:
        cases = [(f"k1_staged_ring{r}MiB", dict(k1=True, staged=True, ring=r)) for r in ring_stagers]
        for name, kw in cases:
            out[name] = bracketed(kw)
        print(json.dumps(out))
        return
    if a.only_staged:
        cases = ce_cases + [("k1_staged", dict(k1=True, staged=True)), ("k1_staged_8ctas", dict(k1=True, staged=True, stage_ctas=8)),
                 ("k2_staged", dict(k2=True, staged=True)),
                 ("k1_staged+k2_staged", dict(k1=True, k2=True, staged=True)),
                 ("k1_staged_8ctas+k2_staged_8ctas", dict(k1=True, k2=True, staged=True, stage_ctas=8))]
    else:
        cases = [("k1_staged", dict(k1=True, staged=True)), ("k1_staged_8ctas", dict(k1=True, staged=True, stage_ctas=8)),
                 ("k2_staged", dict(k2=True, staged=True)),
                 ("k1_staged+k2_staged", dict(k1=True, k2=True, staged=True)),
                 ("k1_staged_8ctas+k2_staged_8ctas", dict(k1=True, k2=True, staged=True, stage_ctas=8))] + [("k2_push", dict(k2=True)), ("k1_default", dict(k1=True)),
             ("k1_148ctas", dict(k1=True, ctas=148)), ("k1_32ctas", dict(k1=True, ctas=32)),
             ("k1_8ctas", dict(k1=True, ctas=8)), ("k1_32ctas+k2", dict(k1=True, k2=True, ctas=32)),
             ("k1_default+k2", dict(k1=True, k2=True)),
             ("k1_copy_engine", dict(k1=True, ce=True)),
             ("k1_copy_engine+k2", dict(k1=True, k2=True, ce=True))]

    for name, kw in cases:
        out[name] = bracketed(kw)
    for dev in (0, 1):
        abi.set_gather_ctas(dev, 0)
    stager0.set_mode(abi.SCATTER_KERNEL)
    stager1.set_mode(abi.SCATTER_KERNEL)
    if a.skip_layerwise:
        print(json.dumps(out))
        return

    # layerwise overlap: push one 32K-token request (512 blocks) and compute
    # layer l once layer l has landed
    req_blocks = 512
    rng2 = np.random.default_rng(1)
    jobs_req, keep3 = make_jobs(1, 1, req_blocks, n_fb, n_slots, rng2, ticket0=2 * n_jobs)
    items = abi.layer_items(g, req_blocks)

    def pipeline(overlap):
        pool.reset_counters()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        t0 = time.time()
        with torch.cuda.device(1):
            abi.h2d_push_p2p_layer(view, st_de, jobs_req, 1, s_k2.cuda_stream)
        if not overlap:
            s_k2.synchronize()
        with torch.cuda.stream(s_gemm):
            for layer in range(L):
                abi.wait_layer(pool, 2 * n_jobs, layer, items, 20000, s_gemm.cuda_stream)
                torch.matmul(x, w)
        torch.cuda.synchronize(0)
        assert abi.wait_status(pool) == abi.DP_OK
        return (time.time() - t0) * 1e3
    pipeline(True)
    ser = min(pipeline(False) for _ in range(3))
    ovl = min(pipeline(True) for _ in range(3))
    out["layerwise_32k_request"] = {"serial_ms": round(ser, 2), "overlapped_ms": round(ovl, 2),
                                    "per_layer_load_ms": round(req_blocks * T * B / 51.5e9 * 1e3, 3),
                                    "per_layer_gemm_ms": base, "speedup": round(ser / ovl, 3)}
    view.close()
    pool.close()
    st_pe.close()
    st_de.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
