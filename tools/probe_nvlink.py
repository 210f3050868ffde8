#!/usr/bin/env python
"""NVLink probe (2 GPUs): what the copy engines deliver device 0 -> device 1,
the ceiling a copy-engine K3 (dp_prefill_handoff_copy) is compared with.

* 1D cudaMemcpyPeerAsync of 1 GiB on 1, 2, 4, 8 streams (the bytes split
  evenly; concurrent copies may run on different copy engines);
* 2D copies shaped like K3's: rows = layers (61), row width = a run of
  Layer Blocks (36 KB x blocks), pitches = the pools' layer planes;
* the same 2D copies on 1 / 2 / 4 streams.

Prints one JSON object (GB/s = payload bytes / CUDA-event time, best of 5).
"""

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def timed(fn, streams, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        main = streams[0]
        e0.record(main)
        for s in streams[1:]:
            s.wait_event(e0)
        fn()
        for s in streams[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        e1.record(main)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    assert torch.cuda.device_count() >= 2
    torch.cuda.set_device(0)
    n = 1 << 30
    a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    out = {}
    streams = [torch.cuda.Stream(device=0) for _ in range(8)]
    for k in (1, 2, 4, 8):
        part = n // k

        def go(k=k, part=part):
            for i in range(k):
                with torch.cuda.stream(streams[i]):
                    b[i * part:(i + 1) * part].copy_(a[i * part:(i + 1) * part], non_blocking=True)
        ms = timed(go, streams[:k])
        out[f"1d_1GiB_{k}streams"] = round(n / ms / 1e6, 1)
    # K3-shaped 2D copies: layer planes of n_slots Layer Blocks
    L, lb = 61, 64 * 576
    n_slots = n // (L * lb)
    plane = n_slots * lb
    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    for blocks in (8, 32, 128, 256):
        runs = n_slots // blocks
        for k in (1, 2, 4):
            def go(blocks=blocks, runs=runs, k=k):
                for r in range(runs):
                    off = r * blocks * lb
                    rc = rt.cudaMemcpy2DAsync(b.data_ptr() + off, plane, a.data_ptr() + off, plane, blocks * lb, L,
                                              3, streams[r % k].cuda_stream)  # cudaMemcpyDeviceToDevice
                    assert rc == 0, rc
            ms = timed(go, streams[:k])
            out[f"2d_L61_run{blocks}blk_{k}streams"] = round(runs * blocks * lb * L / ms / 1e6, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
