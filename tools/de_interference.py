#!/usr/bin/env python
"""The DE's own compute next to its K2 pushes: SM gather (dp_h2d_push_p2p_layer)
vs the DE's copy engine (dp_h2d_push_copy).  Two GPUs: cuda:1 is the DE,
cuda:0 the PE whose pool receives the KV.  The DE's compute stand-in is K5 on
its own pool.  Not product code.  Prints one JSON object."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_21548_b200 import abi  # noqa: E402

L, T, B = 61, 64, 576


def main():
    g = abi.geom(L, T, B)
    n_fb, blocks, n_jobs = 2048, 128, 32
    n_slots = n_jobs * blocks
    st = abi.Store(1, g, n_fb, 9)
    pe_pool = abi.Pool(0, g, n_slots, n_jobs + 1)
    view = pe_pool.peer_view(1)
    de_pool = abi.Pool(1, g, 512, 4)  # the DE's own pool for its compute stand-in
    keep, specs, ce_specs = [], [], []
    for j in range(n_jobs):
        fbs = np.arange(j * blocks, (j + 1) * blocks, dtype=np.int64) % n_fb
        sl = np.arange(j * blocks, (j + 1) * blocks, dtype=np.int32)  # fresh, contiguous slots
        tf = torch.tensor(fbs, device="cuda:1")
        ts = torch.tensor(sl, device="cuda:1")
        keep += [tf, ts, fbs, sl]
        specs.append((tf.data_ptr(), ts.data_ptr(), blocks * T, blocks, 0, L, j))
        ce_specs.append((fbs.ctypes.data, sl.ctypes.data, blocks * T, blocks, 0, L, j))
    jobs, ce_jobs = abi.make_jobs(specs), abi.make_jobs(ce_specs)
    k2_bytes = n_jobs * blocks * T * B * L
    # DE compute stand-in: K5 over its own pool (4 x 8192 cached tokens, 429 queries)
    fill = []
    for i in range(4):
        tf = torch.tensor(np.arange(i * 128, (i + 1) * 128, dtype=np.int64), device="cuda:1")
        ts = torch.tensor(np.arange(i * 128, (i + 1) * 128, dtype=np.int32), device="cuda:1")
        keep += [tf, ts]
        fill.append((tf.data_ptr(), ts.data_ptr(), 128 * T, 128, 0, L, i))
    abi.h2d_layer_gather(de_pool, st, abi.make_jobs(fill), 4)
    digest = torch.zeros((4, L), dtype=torch.int64, device="cuda:1")
    att = (abi.AttendItem * 4)(*[abi.AttendItem(keep[-1 - 2 * (3 - i)].data_ptr(), 128 * T, 0, 429,
                                                digest[i].data_ptr(), i, 0) for i in range(4)])
    macs = 4 * 128 * T * 429 * B * L
    torch.cuda.synchronize(1)

    def run(mode, k5_reps):
        s_load = torch.cuda.Stream(device=1)
        s_comp = torch.cuda.Stream(device=1)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        pe_pool.reset_counters()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        with torch.cuda.device(1):
            e[0].record(s_load)
            s_comp.wait_event(e[0])
            if mode == "sm":
                abi.h2d_push_p2p_layer(view, st, jobs, n_jobs, s_load.cuda_stream)
            elif mode == "ce":
                abi.h2d_push_copy(view, st, ce_jobs, n_jobs, s_load.cuda_stream)
            e[1].record(s_load)
            e[2].record(s_comp)
            for _ in range(k5_reps):
                for layer in range(L):
                    abi.prefill_attend(de_pool, layer, att, 4, 9, s_comp.cuda_stream)
            e[3].record(s_comp)
        torch.cuda.synchronize(1)
        torch.cuda.synchronize(0)
        return e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])

    out = {}
    run("sm", 0)
    for mode in ("sm", "ce"):
        t, _ = run(mode, 0)
        out[f"k2_{mode}_alone_gbps"] = round(k2_bytes / t / 1e6, 2)
    _, t5 = run("none", 3)
    out["de_k5_alone_tmacs"] = round(3 * macs / t5 / 1e9, 2)
    reps = max(1, int(round(k2_bytes / 51e9 / (t5 / 3e3) * 1.5)))
    for mode in ("sm", "ce"):
        tk, tc = run(mode, reps)
        out[f"both_{mode}"] = {"k2_gbps": round(k2_bytes / tk / 1e6, 2),
                               "de_k5_tmacs": round(reps * macs / tc / 1e9, 2)}
    print(json.dumps(out))
    for p in (view, pe_pool, de_pool):
        p.close()
    st.close()


if __name__ == "__main__":
    main()
