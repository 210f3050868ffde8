#!/usr/bin/env python
"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/libpdsim_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Fixtures:
  decisions_<name>.json  scheduler decisions + makespan + per-stage byte
                         ledger of desim::run_offline on a synthetic trace
  kvref_kat.json         known answers of the content / hash formulas
  bench_<key>.json       the reference's decisions (digest, makespan, ledger)
                         for the exact workloads bench.py measures
                         (`python tests/golden/make_golden.py --bench`; the
                         8-GPU ones take ~10 min of reference CPU each)
"""

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refpy  # noqa: E402

# name -> (synthesize kwargs, simulate kwargs)
CASES = {
    # reference tests' tiny_cluster + quick_options (proj/tests/test_desim.cpp:15-36)
    "tiny_2p2d": (dict(max_len=4096, count=24, seed=7),
                  dict(P=2, D=2, g=2, L=4, b=1024, T=64, cl=1e-6, dctx=1e-10, dstep=1e-4)),
    # storage-bound 1P1D, DS-V3 shape, BASELINE config 1 generator (5 sessions)
    "dsv3_1p1d": (dict(max_len=131072, count=5, seed=9, mean_turns=20, sigma_turns=0.0, mean_gen=500),
                  dict(P=1, D=1, g=1, L=61, b=576, T=64, B=50e9, s=0.125, M=500e9, hbm=100000000,
                       pe_buf=1 << 42, de_buf=1 << 42, cl=1e-12, dctx=1e-15, dstep=1e-9, sub=0,
                       beta=1000000000)),
    # 4P4D, Qwen shape, round-robin baseline
    "qwen_4p4d_rr": (dict(max_len=65536, count=12, seed=3, mean_turns=6, sigma_turns=0.3),
                     dict(P=4, D=4, g=1, L=64, b=4096, T=64, B=778e9, s=0.066, M=2e12,
                          hbm=100000000, pe_buf=1 << 42, de_buf=1 << 42, cl=1e-12, dctx=1e-15,
                          dstep=1e-9, sub=0, beta=1000000000, sched_mode="round_robin")),
}

STAGES = ["storage_read", "loopback_h2d", "pe_to_de", "de_to_pe", "miss_merge", "decode_h2d",
          "layer_compute", "decode", "persist_d2h", "persist_write", "burst"]


# bench.py's configurations: (workload, sessions, P, D, policy, cap GB/s)
BENCH = [("c1", 64, 1, 1, "pe_only", 0), ("c1", 16, 1, 1, "pe_only", 0)]
for _n in (2, 4, 8):
    for _pol in ("dual_path", "pe_only"):
        BENCH.append(("c1", 16 * _n, _n // 2, _n - _n // 2, _pol, 0))
        BENCH.append(("c2", 6 * _n, _n // 2, _n - _n // 2, _pol, 6.25))
for _pol in ("dual_path", "pe_only"):
    BENCH.append(("c1", 128, 2, 6, _pol, 0))
    BENCH.append(("c2", 24, 1, 3, _pol, 6.25))  # N = 4, P:D = 1:3


def bench_case(case):
    """One bench configuration through the reference simulator."""
    import bench
    wl, sessions, P, D, policy, cap = case
    shape = bench.QWEN if wl == "c3" else bench.DSV3
    key = bench.golden_key(wl, sessions, P, D, policy, cap, bench.PCIE_ZC_BPS)
    trace = f"/tmp/golden_bench_{key}.tsv"

    class A:
        workload, trace_path = wl, ""
    A.trace = ""
    rounds = bench.reference_trace(A, wl, sessions, trace)
    rate = cap * 1e9 if cap else bench.PCIE_ZC_BPS
    kv = dict(P=P, D=D, g=1, L=shape["L"], b=shape["b"], T=shape["T"], B=bench.NVLINK_BPS,
              s=rate / bench.NVLINK_BPS, M=2e12, hbm=100_000_000, pe_buf=bench.buffer_bytes(shape),
              de_buf=bench.buffer_bytes(shape),
              policy=policy, flows=1, **bench.PLAN_KW)
    t0 = __import__("time").time()
    rep = refpy.ref_simulate(trace, **kv)
    wall = __import__("time").time() - t0
    h = hashlib.sha1()
    for d in rep["decisions"]:
        h.update(repr((d[1], d[2], d[3], d[4])).encode())
    ledger = {}
    for req, stage, nbytes, a, b in rep["flows"]:
        ledger[STAGES[stage]] = ledger.get(STAGES[stage], 0.0) + nbytes
    out = {"key": key, "workload": wl, "sessions": sessions, "P": P, "D": D, "policy": policy,
           "cap_gbps": cap, "simulate": {k: v for k, v in kv.items() if k != "flows"},
           "trace_md5": hashlib.md5(open(trace, "rb").read()).hexdigest(),
           "requests": sum(len(r) for r in rounds), "decisions": len(rep["decisions"]),
           "de_path": sum(1 for d in rep["decisions"] if d[4] == 1),
           "decisions_digest": h.hexdigest(), "makespan": rep["makespan"], "ledger": ledger,
           "reference_wall_s": round(wall, 2)}
    os.unlink(trace)
    with open(os.path.join(HERE, f"bench_{key}.json"), "w") as f:
        json.dump(out, f, indent=1)
    return key, len(rep["decisions"]), round(wall, 1)


def main_bench(only=None):
    from multiprocessing import Pool
    sys.path.insert(0, ROOT)
    cases = [c for c in BENCH if not only or any(o in "_".join(map(str, c)) for o in only)]
    # longest first: the 8-GPU c1 cases dominate
    cases.sort(key=lambda c: -(c[1] * (3 if c[0] == "c1" else 1)))
    with Pool(min(len(cases), os.cpu_count() or 1)) as pool:
        for res in pool.imap_unordered(bench_case, cases):
            print(*res, flush=True)


def main():
    for name, (syn, sim) in CASES.items():
        trace = os.path.join(HERE, f"trace_{name}.tsv")
        refpy.ref_synthesize(trace, **syn)
        rep = refpy.ref_simulate(trace, flows=1, **sim)
        ledger = {}
        for req, stage, nbytes, t0, t1 in rep["flows"]:
            ledger[STAGES[stage]] = ledger.get(STAGES[stage], 0.0) + nbytes
        out = {"synthesize": syn, "simulate": sim, "makespan": rep["makespan"],
               "completed_requests": rep["completed_requests"], "decisions": rep["decisions"],
               "ledger": ledger,
               "trace_md5": hashlib.md5(open(trace, "rb").read()).hexdigest()}
        with open(os.path.join(HERE, f"decisions_{name}.json"), "w") as f:
            json.dump(out, f)
        os.unlink(trace)
        print(name, len(rep["decisions"]), rep["makespan"])

    # content / hash known answers (from the C oracle)
    g = refpy.geom(61, 64, 576)
    kat = {"splitmix64": {str(x): refpy.kvref().kvref_splitmix64(x) for x in (0, 1, 0xDEADBEEF)},
           "word": [[9, fb, w, refpy.kvref().kvref_word(9, fb, w)]
                    for fb, w in ((0, 0), (1, 1), (123, 4607), (4095, 281087))],
           "layer_block_hash": [[9, fb, layer, ntok, refpy.layer_block_hash(g, 9, fb, layer, ntok)]
                                for fb, layer, ntok in ((0, 0, 64), (7, 60, 17), (300, 31, 64))]}
    with open(os.path.join(HERE, "kvref_kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    print("kvref_kat.json")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--bench":
        main_bench(sys.argv[2:])
    else:
        main()
