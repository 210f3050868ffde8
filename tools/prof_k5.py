#!/usr/bin/env python
"""One K5 (dp_prefill_attend) launch for an ncu capture: 4 requests of 8192
cached DS-V3 tokens, 429 queries each, one layer.  Not product code."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_21548_b200 import abi  # noqa: E402

L, T, B = 61, 64, 576
N_SLOTS = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = abi.geom(L, T, B)
st = abi.Store(0, g, 1024, 9)
pool = abi.Pool(0, g, N_SLOTS, 4)
perm = np.random.default_rng(0).permutation(N_SLOTS).astype(np.int32)
keep, specs, items = [], [], []
digest = torch.zeros((4, L), dtype=torch.int64, device="cuda:0")
for i in range(4):
    tf = torch.tensor(np.arange(i * 128, (i + 1) * 128, dtype=np.int64), device="cuda:0")
    ts = torch.tensor(perm[i * 128:(i + 1) * 128], device="cuda:0")
    keep += [tf, ts]
    specs.append((tf.data_ptr(), ts.data_ptr(), 128 * T, 128, 0, L, i))
    items.append(abi.AttendItem(ts.data_ptr(), 128 * T, 0, 429, digest[i].data_ptr(), i, 0))
abi.h2d_layer_gather(pool, st, abi.make_jobs(specs), 4)
att = (abi.AttendItem * 4)(*items)
for layer in range(3):
    abi.prefill_attend(pool, layer, att, 4, 9)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for layer in range(L):
    abi.prefill_attend(pool, layer, att, 4, 9)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / L
macs = 4 * 128 * T * 429 * B
print(f"[{N_SLOTS} pool slots] K5 per layer: {ms:.3f} ms, {macs / ms / 1e9:.2f} TMAC/s "
      f"({4 * 128 * T * B * 7 / ms / 1e6:.1f} GB/s of key-tile reads incl. 7 query tiles)")
pool.close()
st.close()
