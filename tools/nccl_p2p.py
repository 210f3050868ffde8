#!/usr/bin/env python
"""NCCL as a measured comparison point (not on the data path): send/recv of
a 1 GiB buffer from rank 1 (the DE) to rank 0 (the PE), and the staged
alternative to K2 -- the DE's copy engine lands the KV in its own HBM, then
NCCL sends it -- against K2's direct PCIe-read + NVLink-store push.
Run: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_p2p.py"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
    n = 1 << 30
    buf = torch.empty(n, dtype=torch.uint8, device=f"cuda:{rank}")
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True) if rank == 1 else None
    out = {}
    for name, staged in (("nccl_send_recv", False), ("ce_h2d_then_nccl", True)):
        times = []
        for rep in range(4):
            dist.barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            if rank == 1:
                if staged:
                    buf.copy_(host, non_blocking=True)
                dist.send(buf, dst=0)
            else:
                dist.recv(buf, src=1)
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b)], device=f"cuda:{rank}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rep:
                times.append(t.item())
        out[name] = round(n / (min(times) * 1e-3) / 1e9, 1)
    if rank == 0:
        out["note"] = ("GB/s for 1 GiB, max over ranks; K2 pushes from host memory at 51.4 GB/s with "
                       "no staging copy and no NCCL")
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
