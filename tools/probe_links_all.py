#!/usr/bin/env python
"""Link peaks of every visible GPU (SURVEY.md §8(d) asks for them beside
MEASURED_PEAKS.json, which has none): copy-engine H2D of 1 GiB pinned per
GPU, alone and all at once, and cudaMemcpyPeerAsync of 1 GiB for every
ordered pair.  Best of 3, CUDA events.  Prints one JSON object."""

import json
import threading

import torch


def timed_copy(dst, src, stream, reps=3):
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            dst.copy_(src, non_blocking=True)
            e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return src.numel() / best / 1e6


def main():
    n = torch.cuda.device_count()
    size = 1 << 30
    host = [torch.empty(size, dtype=torch.uint8).pin_memory() for _ in range(n)]
    dev = [torch.empty(size, dtype=torch.uint8, device=f"cuda:{d}") for d in range(n)]
    streams = [torch.cuda.Stream(device=d) for d in range(n)]
    out = {"gpus": n, "h2d_alone_gbps": [], "d2d_peer_gbps": {}}
    for d in range(n):
        with torch.cuda.device(d):
            out["h2d_alone_gbps"].append(round(timed_copy(dev[d], host[d], streams[d]), 1))
    res = [0.0] * n

    def run(d):
        with torch.cuda.device(d):
            res[d] = timed_copy(dev[d], host[d], streams[d])
    ths = [threading.Thread(target=run, args=(d,)) for d in range(n)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    out["h2d_concurrent_gbps"] = [round(x, 1) for x in res]
    out["h2d_concurrent_sum_gbps"] = round(sum(res), 1)
    for a in range(n):
        for b in range(n):
            if a == b:
                continue
            with torch.cuda.device(a):
                out["d2d_peer_gbps"][f"{a}->{b}"] = round(timed_copy(dev[b], dev[a], streams[a]), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
