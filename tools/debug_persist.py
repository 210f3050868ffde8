#!/usr/bin/env python
"""Diagnostic: one handoff+persist step with a short watchdog; on failure,
dump every counter row that did not reach its target (not product code)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2602_21548_b200 as dp  # noqa: E402
from test_gpu_engine import STORAGE_BOUND, cluster, handoff_engines, small_trace  # noqa: E402

persist = len(sys.argv) < 2 or sys.argv[1] != "nopersist"
cfg = cluster(1, 1, L=4)
trajs = small_trace(count=6, turns=4, seed=12)
planned = dp.plan(cfg, trajs, policy="dual_path", **STORAGE_BOUND)
opt = dp.ExecOptions()
opt.seed = 9
opt.handoff = True
opt.persist = persist
opt.wait_timeout_ms = int(os.environ.get("DBG_TIMEOUT", "3000"))
opt.k3_layer_gate = int(os.environ.get("DBG_GATE", "0"))
import time  # noqa: E402
opt.de_pool_slots = int(os.environ.get("DBG_DESLOTS", "0"))
opt.pool_slots = int(os.environ.get("DBG_PESLOTS", "0"))
xp = dp.build_exec_plan(cfg, trajs, planned, opt)
print("pe slots", xp.pool_slots, "peak", xp.peak_slots, "de slots", xp.de_pool_slots, "peak", xp.de_peak_slots)
rts = handoff_engines(xp, 2)
for rt in rts:
    rt.reset_counters()
import threading  # noqa: E402
snap = {}


def grab():
    time.sleep(float(os.environ.get("DBG_SNAP", "1.0")))
    snap["pe"] = np.asarray(rts[0].counters(), dtype=np.int64)
    snap["de"] = np.asarray(rts[1].counters(), dtype=np.int64)


th = threading.Thread(target=grab)
th.start()
t0 = time.time()
try:
    dp.run_step_all(rts)
    print("step ok", round(time.time() - t0, 3), "s")
except Exception as exc:
    print("step failed:", exc, round(time.time() - t0, 3), "s")
th.join()
L = cfg.n_layer
ipb = xp.items_per_block
pe = snap["pe"].reshape(-1, L + 1)
de = snap["de"].reshape(-1, L + 1)
print("(counters snapshot taken while the step runs)")
n_pe = xp.n_tickets[0]
n_de = xp.n_de_tickets[1]
print("rows pe", pe.shape, "de", de.shape, "n_pe", n_pe, "n_de", n_de)
for i, j in enumerate(xp.jobs()):
    req, traj, rnd, reader, jpe, de_path, cached, nblk, ticket = j[:9]
    npblk, de_ticket, de_preds, k3w, ped = j[15], j[16], j[19], j[20], j[21]
    load_t = nblk * ipb * L
    done_t = npblk * ipb * L
    de_t = ((nblk if de_path else 0) + npblk) * ipb * L
    bad = []
    if nblk and pe[ticket, L] != load_t:
        bad.append(f"load {pe[ticket, L]}/{load_t}")
    if pe[n_pe + ticket, L] != done_t:
        bad.append(f"k3done {pe[n_pe + ticket, L]}/{done_t}")
    if de[de_ticket, L] != de_t:
        bad.append(f"de {de[de_ticket, L]}/{de_t}")
    if persist and de[n_de + de_ticket, L] != 1:
        bad.append(f"persist {de[n_de + de_ticket, L]}")
    print(i, "req", req, "path", "DE" if de_path else "PE", "C", cached, "nblk", nblk, "npblk", npblk,
          "ticket", ticket, "de_ticket", de_ticket, "de_preds", de_preds, "k3w", k3w, "pe_done", ped,
          "BAD " + ", ".join(bad) if bad else "")
