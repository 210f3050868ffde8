"""ctypes binding of the C ABI (include/dualpath/kv_abi.h).

This is the binding a maintainer of the reference's Python shim would add
(INTEGRATION.md): plain pointers and sizes, no torch types.  Errors raise
``DualPathError`` carrying ``dp_last_error()``.  Streams are passed as raw
``cudaStream_t`` integers (0 = legacy default stream).
"""

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdualpath.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "dualpath", "kv_abi.h")

DP_OK, DP_EINVAL, DP_ECUDA, DP_ENOMEM, DP_ETIMEOUT = 0, -1, -2, -3, -4
MAX_JOBS_PER_LAUNCH = 64


class DualPathError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Geom(ctypes.Structure):
    _fields_ = [("n_layer", ctypes.c_int32), ("block_tokens", ctypes.c_int32),
                ("bytes_per_token_layer", ctypes.c_int64)]


class Job(ctypes.Structure):
    _fields_ = [("src_fb", ctypes.c_void_p), ("dst_slot", ctypes.c_void_p),
                ("n_tokens", ctypes.c_int64), ("n_blk", ctypes.c_int32),
                ("layer_begin", ctypes.c_int32), ("layer_end", ctypes.c_int32),
                ("ticket", ctypes.c_int32)]


class DualJob(ctypes.Structure):
    _fields_ = [("pe", Job), ("de_slot", ctypes.c_void_p), ("de_ticket", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class HandoffJob(ctypes.Structure):
    _fields_ = [("src_fb", ctypes.c_void_p), ("pe_slot", ctypes.c_void_p), ("de_slot", ctypes.c_void_p),
                ("n_cached", ctypes.c_int64), ("n_prompt", ctypes.c_int64), ("n_blk", ctypes.c_int32),
                ("push_hit", ctypes.c_int32), ("pe_ticket", ctypes.c_int32),
                ("pe_wait_items", ctypes.c_uint32), ("de_ticket", ctypes.c_int32),
                ("pe_done_ticket", ctypes.c_int32)]


class SpanJob(ctypes.Structure):
    _fields_ = [("slot", ctypes.c_void_p), ("fb", ctypes.c_void_p), ("blk0", ctypes.c_int64),
                ("tok_begin", ctypes.c_int64), ("tok_end", ctypes.c_int64), ("n_blk", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class AttendItem(ctypes.Structure):
    _fields_ = [("slot", ctypes.c_void_p), ("cached", ctypes.c_int64), ("q_begin", ctypes.c_int64),
                ("bsz", ctypes.c_int64), ("digest", ctypes.c_void_p), ("req", ctypes.c_uint32),
                ("reserved", ctypes.c_int32)]


class PoolHandle(ctypes.Structure):
    _fields_ = [("ipc", ctypes.c_ubyte * 64), ("geom", Geom), ("n_slots", ctypes.c_int32),
                ("n_tickets", ctypes.c_int32), ("device", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 9)]


_lib = None


def lib():
    """Load libdualpath.so (raises if the native build is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: the CUDA extension is not built")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "dp_abi_version": ([], ctypes.c_int),
        "dp_last_error": ([], ctypes.c_char_p),
        "dp_geom_check": ([ctypes.POINTER(Geom)], ctypes.c_int),
        "dp_store_create": ([ctypes.c_int, ctypes.POINTER(Geom), ctypes.c_int64, ctypes.c_uint64, PP],
                            ctypes.c_int),
        "dp_store_destroy": ([P], ctypes.c_int),
        "dp_store_info": ([P, PP, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)],
                          ctypes.c_int),
        "dp_pool_create": ([ctypes.c_int, ctypes.POINTER(Geom), ctypes.c_int32, ctypes.c_int32, PP],
                           ctypes.c_int),
        "dp_pool_destroy": ([P], ctypes.c_int),
        "dp_pool_info": ([P, PP, PP, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "dp_pool_reset_counters": ([P, P], ctypes.c_int),
        "dp_pool_export": ([P, ctypes.POINTER(PoolHandle)], ctypes.c_int),
        "dp_pool_import": ([ctypes.c_int, ctypes.POINTER(PoolHandle), PP], ctypes.c_int),
        "dp_pool_create_layout": ([ctypes.c_int, ctypes.POINTER(Geom), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                   PP], ctypes.c_int),
        "dp_pool_layout": ([P, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
        "dp_pool_peer_view": ([ctypes.c_int, P, PP], ctypes.c_int),
        "dp_h2d_layer_gather": ([P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_push_p2p_layer": ([P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_layer_copy": ([P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_push_copy": ([P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_layer_copy_job": ([P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_push_copy_job": ([P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_push_p2p_dual": ([P, P, P, ctypes.POINTER(DualJob), ctypes.c_int32, P], ctypes.c_int),
        "dp_prefill_handoff": ([P, P, ctypes.POINTER(HandoffJob), ctypes.c_int32, ctypes.c_uint64,
                                ctypes.c_int32, P], ctypes.c_int),
        "dp_prefill_handoff_copy": ([P, P, ctypes.POINTER(HandoffJob), ctypes.c_int32, ctypes.c_uint64,
                                     ctypes.c_int32, P], ctypes.c_int),
        "dp_handoff_copy_launches": ([ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "dp_set_handoff_gate_memop": ([ctypes.c_int32], ctypes.c_int),
        "dp_persist_staged": ([P, P, P, ctypes.POINTER(SpanJob), ctypes.c_int32, P], ctypes.c_int),
        "dp_layer_items": ([ctypes.POINTER(Geom), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)],
                           ctypes.c_int),
        "dp_wait_layer": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, ctypes.c_int32, P],
                          ctypes.c_int),
        "dp_wait_tickets": ([P, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P],
                            ctypes.c_int),
        "dp_wait_status": ([P], ctypes.c_int),
        "dp_wait_clear": ([P], ctypes.c_int),
        "dp_store_create_on_node": ([ctypes.c_int, ctypes.POINTER(Geom), ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_int32, PP], ctypes.c_int),
        "dp_store_numa_node": ([P, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
        "dp_device_numa_node": ([ctypes.c_int, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
        "dp_nic_create": ([ctypes.c_double, PP], ctypes.c_int),
        "dp_nic_destroy": ([P], ctypes.c_int),
        "dp_nic_start": ([P], ctypes.c_int),
        "dp_nic_read": ([P, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                         ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "dp_storage_read": ([P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, P], ctypes.c_int),
        "dp_stager_create": ([ctypes.c_int, ctypes.POINTER(Geom), ctypes.c_int64, PP], ctypes.c_int),
        "dp_stager_destroy": ([P], ctypes.c_int),
        "dp_stager_set_ctas": ([P, ctypes.c_int32], ctypes.c_int),
        "dp_stager_launches": ([P, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "dp_stager_set_mode": ([P, ctypes.c_int32], ctypes.c_int),
        "dp_h2d_layer_staged": ([P, P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_push_staged": ([P, P, P, ctypes.POINTER(Job), ctypes.c_int32, P], ctypes.c_int),
        "dp_h2d_push_dual_staged": ([P, P, P, P, ctypes.POINTER(DualJob), ctypes.c_int32, P], ctypes.c_int),
        "dp_stream_wait_counter": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, P], ctypes.c_int),
        "dp_stream_write_counter": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, P], ctypes.c_int),
        "dp_decode_fill": ([P, ctypes.POINTER(SpanJob), ctypes.c_int32, ctypes.c_uint64, P], ctypes.c_int),
        "dp_persist_d2h": ([P, P, ctypes.POINTER(SpanJob), ctypes.c_int32, P], ctypes.c_int),
        "dp_pool_checksum": ([P, ctypes.c_int32, P, P, ctypes.c_int32, P, P], ctypes.c_int),
        "dp_pool_copy_out": ([P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, P], ctypes.c_int),
        "dp_device_count": ([], ctypes.c_int),
        "dp_set_gather_ctas": ([ctypes.c_int, ctypes.c_int32], ctypes.c_int),
        "dp_set_handoff_ctas": ([ctypes.c_int, ctypes.c_int32], ctypes.c_int),
        "dp_set_handoff_tma": ([ctypes.c_int32], ctypes.c_int),
        "dp_prefill_attend": ([P, ctypes.c_int32, ctypes.POINTER(AttendItem), ctypes.c_int32,
                               ctypes.c_uint64, P], ctypes.c_int),
        "dp_set_attend_ctas": ([ctypes.c_int, ctypes.c_int32], ctypes.c_int),
        "dp_prefill_attend_signal": ([P, ctypes.c_int32, ctypes.POINTER(AttendItem), ctypes.c_int32,
                                      ctypes.c_uint64, P, P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def declared_symbols(header=HEADER):
    """Entry points declared in include/dualpath/kv_abi.h."""
    text = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dp_\w+)\s*\(", text, re.M)))


def check(rc):
    if rc != DP_OK:
        raise DualPathError(rc, lib().dp_last_error().decode())
    return rc


def geom(n_layer, block_tokens, b):
    return Geom(n_layer, block_tokens, b)


NUMA_DEVICE, NUMA_NONE = -1, -2
POOL_LAYER_MAJOR, POOL_BLOCK_MAJOR = 0, 1
SCATTER_KERNEL, SCATTER_CE = 0, 1


class Store:
    """Pinned+mapped host Full Blocks filled with the deterministic content
    (NUMA-bound to `numa_node`: NUMA_DEVICE = the GPU's own node)."""

    def __init__(self, device, g, n_fb, seed, numa_node=NUMA_DEVICE):
        self.ptr = ctypes.c_void_p()
        check(lib().dp_store_create_on_node(device, ctypes.byref(g), n_fb, seed, numa_node,
                                            ctypes.byref(self.ptr)))
        self.geom = g
        self.n_fb = n_fb

    def numa_node(self):
        n = ctypes.c_int32()
        check(lib().dp_store_numa_node(self.ptr, ctypes.byref(n)))
        return n.value

    def storage_read(self, dst_fb, src_fb, n_fb, nic=None):
        check(lib().dp_storage_read(self.ptr, dst_fb, src_fb, n_fb, nic.ptr if nic else None))

    def info(self):
        host = ctypes.c_void_p()
        nbytes = ctypes.c_int64()
        nfb = ctypes.c_int64()
        check(lib().dp_store_info(self.ptr, ctypes.byref(host), ctypes.byref(nbytes), ctypes.byref(nfb)))
        return host.value, nbytes.value, nfb.value

    def bytes(self):
        host, nbytes, _ = self.info()
        return ctypes.string_at(host, nbytes)

    def close(self):
        if self.ptr:
            check(lib().dp_store_destroy(self.ptr))
            self.ptr = ctypes.c_void_p()


class Pool:
    """Paged HBM pool [L][n_slots][T][b] + landed counters [n_tickets][L+1]."""

    def __init__(self, device=None, g=None, n_slots=0, n_tickets=0, _ptr=None, layout=0):
        self.geom = g
        self.n_slots = n_slots
        self.n_tickets = n_tickets
        if _ptr is not None:
            self.ptr = _ptr
            return
        self.ptr = ctypes.c_void_p()
        check(lib().dp_pool_create_layout(device, ctypes.byref(g), n_slots, n_tickets, layout,
                                          ctypes.byref(self.ptr)))

    def layout(self):
        out = ctypes.c_int32()
        check(lib().dp_pool_layout(self.ptr, ctypes.byref(out)))
        return out.value

    def info(self):
        base = ctypes.c_void_p()
        ctr = ctypes.c_void_p()
        nbytes = ctypes.c_int64()
        check(lib().dp_pool_info(self.ptr, ctypes.byref(base), ctypes.byref(ctr), ctypes.byref(nbytes)))
        return base.value, ctr.value, nbytes.value

    def peer_view(self, device):
        v = ctypes.c_void_p()
        check(lib().dp_pool_peer_view(device, self.ptr, ctypes.byref(v)))
        return Pool(g=self.geom, n_slots=self.n_slots, n_tickets=self.n_tickets, _ptr=v)

    def export(self):
        h = PoolHandle()
        check(lib().dp_pool_export(self.ptr, ctypes.byref(h)))
        return bytes(h)

    @staticmethod
    def open(device, handle_bytes):
        h = PoolHandle.from_buffer_copy(handle_bytes)
        v = ctypes.c_void_p()
        check(lib().dp_pool_import(device, ctypes.byref(h), ctypes.byref(v)))
        return Pool(g=h.geom, n_slots=h.n_slots, n_tickets=h.n_tickets, _ptr=v)

    def copy_out(self, layer, slot, nbytes):
        buf = ctypes.create_string_buffer(nbytes)
        check(lib().dp_pool_copy_out(self.ptr, layer, slot, nbytes, buf))
        return buf.raw

    def reset_counters(self, stream=0):
        check(lib().dp_pool_reset_counters(self.ptr, ctypes.c_void_p(stream)))

    def close(self):
        if self.ptr:
            check(lib().dp_pool_destroy(self.ptr))
            self.ptr = ctypes.c_void_p()


class Nic:
    """Emulated storage NIC: FIFO token bucket at rate_Bps (0 = unlimited)."""

    def __init__(self, rate_Bps):
        self.ptr = ctypes.c_void_p()
        check(lib().dp_nic_create(rate_Bps, ctypes.byref(self.ptr)))

    def start(self):
        check(lib().dp_nic_start(self.ptr))

    def read(self, nbytes, not_before_s=0.0):
        b, e = ctypes.c_double(), ctypes.c_double()
        check(lib().dp_nic_read(self.ptr, nbytes, not_before_s, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def close(self):
        if self.ptr:
            check(lib().dp_nic_destroy(self.ptr))
            self.ptr = ctypes.c_void_p()


class Stager:
    """HBM staging ring of the staged K1 / K2 (copy engine + scatter kernel)."""

    def __init__(self, device, g, ring_bytes=0):
        self.ptr = ctypes.c_void_p()
        check(lib().dp_stager_create(device, ctypes.byref(g), ring_bytes, ctypes.byref(self.ptr)))

    def set_ctas(self, n):
        check(lib().dp_stager_set_ctas(self.ptr, n))

    def set_mode(self, mode):
        """SCATTER_KERNEL (0) or SCATTER_CE (1: copy engines only; host slot tables)."""
        check(lib().dp_stager_set_mode(self.ptr, mode))

    def launches(self):
        n = ctypes.c_int64()
        check(lib().dp_stager_launches(self.ptr, ctypes.byref(n)))
        return n.value

    def close(self):
        if self.ptr:
            check(lib().dp_stager_destroy(self.ptr))
            self.ptr = ctypes.c_void_p()


def h2d_layer_staged(pool, store, stager, jobs, n, stream=0):
    return check(lib().dp_h2d_layer_staged(pool.ptr, store.ptr, stager.ptr, jobs, n, ctypes.c_void_p(stream)))


def h2d_push_staged(pool_view, store, stager, jobs, n, stream=0):
    return check(lib().dp_h2d_push_staged(pool_view.ptr, store.ptr, stager.ptr, jobs, n, ctypes.c_void_p(stream)))


def push_dual_staged(pe_view, de_pool, store, stager, jobs, n, stream=0):
    return check(lib().dp_h2d_push_dual_staged(pe_view.ptr, de_pool.ptr, store.ptr, stager.ptr, jobs, n,
                                               ctypes.c_void_p(stream)))


def device_numa_node(device):
    n = ctypes.c_int32()
    check(lib().dp_device_numa_node(device, ctypes.byref(n)))
    return n.value


def wait_clear(pool):
    return check(lib().dp_wait_clear(pool.ptr))


def make_jobs(specs):
    """specs: list of (src_fb_devptr, dst_slot_devptr, n_tokens, n_blk, l0, l1, ticket)."""
    arr = (Job * max(1, len(specs)))()
    for i, (fb, sl, ntok, nblk, l0, l1, tk) in enumerate(specs):
        arr[i] = Job(fb, sl, ntok, nblk, l0, l1, tk)
    return arr


def h2d_layer_gather(pool, store, jobs, n, stream=0):
    check(lib().dp_h2d_layer_gather(pool.ptr, store.ptr, jobs, n, ctypes.c_void_p(stream)))


def h2d_push_p2p_layer(pool_view, store, jobs, n, stream=0):
    check(lib().dp_h2d_push_p2p_layer(pool_view.ptr, store.ptr, jobs, n, ctypes.c_void_p(stream)))


def h2d_layer_copy(pool, store, jobs, n, stream=0):
    """K1 on the copy engine; jobs' block arrays must be host memory."""
    check(lib().dp_h2d_layer_copy(pool.ptr, store.ptr, jobs, n, ctypes.c_void_p(stream)))


def h2d_layer_copy_job(pool, store, jobs, n, stream=0):
    """K1 on the copy engine, counters released once per job."""
    check(lib().dp_h2d_layer_copy_job(pool.ptr, store.ptr, jobs, n, ctypes.c_void_p(stream)))


def h2d_push_copy_job(pool_view, store, jobs, n, stream=0):
    check(lib().dp_h2d_push_copy_job(pool_view.ptr, store.ptr, jobs, n, ctypes.c_void_p(stream)))


def h2d_push_copy(pool_view, store, jobs, n, stream=0):
    """K2 on the DE's copy engine; jobs' block arrays must be host memory."""
    check(lib().dp_h2d_push_copy(pool_view.ptr, store.ptr, jobs, n, ctypes.c_void_p(stream)))


def push_p2p_dual(pe_view, de_pool, store, jobs, n, stream=0):
    check(lib().dp_h2d_push_p2p_dual(pe_view.ptr, de_pool.ptr, store.ptr, jobs, n, ctypes.c_void_p(stream)))


def prefill_handoff(pe_pool, de_view, jobs, n, seed, timeout_ms=20000, stream=0):
    check(lib().dp_prefill_handoff(pe_pool.ptr, de_view.ptr, jobs, n, seed, timeout_ms,
                                   ctypes.c_void_p(stream)))


def prefill_handoff_copy(pe_pool, de_view, jobs, n, seed, timeout_ms=20000, stream=0):
    """K3 on the copy engines; the jobs' block arrays must be host memory."""
    check(lib().dp_prefill_handoff_copy(pe_pool.ptr, de_view.ptr, jobs, n, seed, timeout_ms,
                                        ctypes.c_void_p(stream)))


def set_handoff_gate_memop(on):
    check(lib().dp_set_handoff_gate_memop(1 if on else 0))


def handoff_copy_launches():
    out = ctypes.c_int64()
    check(lib().dp_handoff_copy_launches(ctypes.byref(out)))
    return out.value


def layer_items(g, n_blk):
    out = ctypes.c_int32()
    check(lib().dp_layer_items(ctypes.byref(g), n_blk, ctypes.byref(out)))
    return out.value


def wait_layer(pool, ticket, layer, target, timeout_ms=10000, stream=0):
    check(lib().dp_wait_layer(pool.ptr, ticket, layer, target, timeout_ms, ctypes.c_void_p(stream)))


def stream_wait_counter(pool, ticket, layer, target, stream=0):
    check(lib().dp_stream_wait_counter(pool.ptr, ticket, layer, target, ctypes.c_void_p(stream)))


def stream_write_counter(pool, ticket, layer, value, stream=0):
    check(lib().dp_stream_write_counter(pool.ptr, ticket, layer, value, ctypes.c_void_p(stream)))


def decode_fill(pool, jobs, n, seed, stream=0):
    check(lib().dp_decode_fill(pool.ptr, jobs, n, seed, ctypes.c_void_p(stream)))


def persist_d2h(pool, target, jobs, n, stream=0):
    check(lib().dp_persist_d2h(pool.ptr, target.ptr, jobs, n, ctypes.c_void_p(stream)))


def persist_staged(pool, target, stager, jobs, n, stream=0):
    """K4 staged; the jobs' fb arrays must be host memory, slot arrays device memory."""
    check(lib().dp_persist_staged(pool.ptr, target.ptr, stager.ptr, jobs, n, ctypes.c_void_p(stream)))


def wait_status(pool):
    return lib().dp_wait_status(pool.ptr)


def set_gather_ctas(device, ctas):
    check(lib().dp_set_gather_ctas(device, ctas))


def set_handoff_tma(on):
    check(lib().dp_set_handoff_tma(1 if on else 0))


def set_handoff_ctas(device, ctas):
    check(lib().dp_set_handoff_ctas(device, ctas))


def prefill_attend(pool, layer, items, n, seed, stream=0):
    """K5: attention-score pass of one prefill layer (items: AttendItem array)."""
    check(lib().dp_prefill_attend(pool.ptr, layer, items, n, seed, ctypes.c_void_p(stream)))


def set_attend_ctas(device, ctas):
    check(lib().dp_set_attend_ctas(device, ctas))


def device_count():
    return lib().dp_device_count()
