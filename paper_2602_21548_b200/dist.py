"""Multi-process (one process per GPU) plumbing of the DualPath executor.

torch.distributed is used only as the control plane: barriers, the max over
ranks of step times, and the one-time exchange of PE pool IPC handles.  No
KV byte crosses it; the DE -> PE transfer is the in-kernel NVLink push (K2).

Rank r runs engine r: ranks [0, P) are prefill engines (own a pool), ranks
[P, N) decode engines (open every PE pool through CUDA IPC)."""

import hashlib


def roles(world, n_pe):
    return ["pe" if r < n_pe else "de" for r in range(world)]


def plan_digest(planned):
    """Digest of the scheduler decisions (request, pe, de, path): every rank
    plans independently and must agree bit for bit."""
    h = hashlib.sha1()
    for d in planned["decisions"]:
        h.update(repr((d[1], d[2], d[3], d[4])).encode())
    return h.hexdigest()


class Group:
    """Thin wrapper over torch.distributed (or a single process)."""

    def __init__(self, backend=None, device=None):
        import os
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", str(self.rank)))
        self.td = None
        if self.world > 1:
            import torch
            import torch.distributed as td
            n_dev = torch.cuda.device_count() if backend == "nccl" else 0
            if backend == "nccl" and self.local < n_dev:
                torch.cuda.set_device(self.local)
                td.init_process_group("nccl", device_id=torch.device(f"cuda:{self.local}"))
            else:
                # more ranks than GPUs (a rehearsal of a larger N): NCCL
                # cannot put two ranks on one GPU; the control plane is gloo
                if backend == "nccl" and n_dev:
                    torch.cuda.set_device(self.local % n_dev)
                td.init_process_group("gloo")
            self.td = td

    def barrier(self):
        if self.td:
            self.td.barrier()

    def allgather(self, obj):
        if not self.td:
            return [obj]
        out = [None] * self.world
        self.td.all_gather_object(out, obj)
        return out

    def max(self, x):
        return max(self.allgather(x))

    def close(self):
        if self.td:
            self.td.destroy_process_group()
            self.td = None


def connect_pools(group, engines, n_pe):
    """Exchange pool handles: every DE attaches every PE pool (K2 pushes), and
    with the PD handoff every PE attaches every DE decode pool (K3 pushes).
    `engines` maps engine id -> EngineRuntime for the engines of this process."""
    mine = {e: rt.export_pool() for e, rt in engines.items()
            if e < n_pe or getattr(rt, "has_pool", False)}
    table = {}
    for part in group.allgather(mine):
        table.update(part)
    missing = [pe for pe in range(n_pe) if pe not in table]
    if missing:
        raise RuntimeError(f"no process exported PE pools {missing}")
    for e, rt in engines.items():
        if e >= n_pe:
            for pe in range(n_pe):
                rt.attach_peer(pe, table[pe])
        else:
            for de, h in sorted(table.items()):
                if de >= n_pe:
                    rt.attach_peer(de, h)
    return table
