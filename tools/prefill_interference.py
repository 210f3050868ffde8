#!/usr/bin/env python
"""K1 (SM zero-copy gather) next to K5 (prefill stand-in) on one GPU: how
much does each slow the other?  Single GPU.  Not product code.

  K1 alone / K5 alone / both, at several K1 CTA caps and stream priorities,
  and K1 on the copy engine.  Prints one JSON object.
"""
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
    st = abi.Store(0, g, n_fb, 9)
    pool = abi.Pool(0, g, n_slots, n_jobs + 1)
    rng = np.random.default_rng(0)
    keep, specs, ce_specs = [], [], []
    perm = rng.permutation(n_slots).astype(np.int32)
    for j in range(n_jobs):
        fbs = np.arange(j * blocks, (j + 1) * blocks, dtype=np.int64) % n_fb
        sl = perm[j * blocks:(j + 1) * blocks]
        tf = torch.tensor(fbs, device="cuda:0")
        ts = torch.tensor(sl, device="cuda:0")
        keep += [tf, ts, fbs, sl]
        specs.append((tf.data_ptr(), ts.data_ptr(), blocks * T, blocks, 0, L, j))
        ce_specs.append((fbs.ctypes.data, sl.ctypes.data, blocks * T, blocks, 0, L, j))
    jobs = abi.make_jobs(specs)
    ce_jobs = abi.make_jobs(ce_specs)
    k1_bytes = n_jobs * blocks * T * B * L
    # K5 work: 4 requests of 8192 cached tokens, 429 queries, all layers, repeated
    digest = torch.zeros((64, L), dtype=torch.int64, device="cuda:0")
    items = []
    for i in range(4):
        ts = torch.tensor(perm[i * 128:(i + 1) * 128], device="cuda:0")
        keep.append(ts)
        items.append(abi.AttendItem(ts.data_ptr(), 128 * T, 0, 429, digest[i].data_ptr(), i, 0))
    att = (abi.AttendItem * 4)(*items)
    macs = 4 * 128 * T * 429 * B

    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)

    def run(k1=True, k5_reps=0, ctas=64, ce=False, prio=True):
        abi.set_gather_ctas(0, ctas)
        s_load = torch.cuda.Stream(device=0, priority=-1 if prio else 0)
        s_comp = torch.cuda.Stream(device=0, priority=0)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        pool.reset_counters()
        torch.cuda.synchronize()
        e[0].record(s_load)
        s_comp.wait_event(e[0])
        if k1:
            if ce:
                abi.h2d_layer_copy(pool, st, ce_jobs, n_jobs, s_load.cuda_stream)
            else:
                abi.h2d_layer_gather(pool, st, jobs, n_jobs, s_load.cuda_stream)
        e[1].record(s_load)
        e[2].record(s_comp)
        for _ in range(k5_reps):
            for layer in range(L):
                abi.prefill_attend(pool, layer, att, 4, 9, s_comp.cuda_stream)
        e[3].record(s_comp)
        torch.cuda.synchronize()
        return e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])

    out = {}
    run()  # warm
    t, _ = run()
    out["k1_alone_gbps"] = round(k1_bytes / t / 1e6, 2)
    _, t5 = run(k1=False, k5_reps=4)
    out["k5_alone_tmacs"] = round(4 * macs * L / t5 / 1e9, 2)
    reps = max(1, int(round(t / t5 * 4 * 1.5)))  # keep K5 busy past the end of K1
    for ctas in (32, 64, 148, 0):
        for prio in (True, False):
            tk, tc = run(k5_reps=reps, ctas=ctas, prio=prio)
            out[f"both_ctas{ctas}_prio{int(prio)}"] = {
                "k1_gbps": round(k1_bytes / tk / 1e6, 2),
                "k5_tmacs": round(reps * macs * L / tc / 1e9, 2)}
    tk, tc = run(k5_reps=reps, ce=True)
    out["both_ce"] = {"k1_gbps": round(k1_bytes / tk / 1e6, 2), "k5_tmacs": round(reps * macs * L / tc / 1e9, 2)}
    abi.set_gather_ctas(0, 0)
    print(json.dumps(out))
    pool.close()
    st.close()


if __name__ == "__main__":
    main()
