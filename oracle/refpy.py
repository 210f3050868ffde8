"""Python access to the oracles (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module, and only as the checker / CPU baseline.  Two libraries:

* ``oracle/_ref/libpdsim_ref.so`` -- the reference pdsim compiled from its own
  sources (oracle/Makefile) behind ``oracle/ref_shim.cpp``: scheduler
  decisions, byte ledgers, traces.
* ``oracle/lib/libkvref.so`` -- ``oracle/kvref.c``, the CPU restatement of the
  KV bytes the path moves (content generator, Layer Block hashes, memcpy
  gather).
"""

import ctypes
import json
import os
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpdsim_ref.so")
KVREF_SO = os.path.join(HERE, "lib", "libkvref.so")

GOLDEN = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


class KvGeom(ctypes.Structure):
    _fields_ = [("n_layer", ctypes.c_int32), ("block_tokens", ctypes.c_int32),
                ("bytes_per_token_layer", ctypes.c_int64)]


class KvJob(ctypes.Structure):
    _fields_ = [("src_fb", ctypes.POINTER(ctypes.c_int64)),
                ("dst_slot", ctypes.POINTER(ctypes.c_int32)),
                ("n_tokens", ctypes.c_int64), ("n_blk", ctypes.c_int32),
                ("layer_begin", ctypes.c_int32), ("layer_end", ctypes.c_int32),
                ("ticket", ctypes.c_int32)]


_kv = None
_ref = None


def kvref():
    global _kv
    if _kv is None:
        lib = ctypes.CDLL(KVREF_SO)
        lib.kvref_word.restype = ctypes.c_uint64
        lib.kvref_word.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
        lib.kvref_attend_digest.restype = ctypes.c_uint64
        lib.kvref_attend_digest.argtypes = [ctypes.POINTER(KvGeom), ctypes.c_uint64,
                                            ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                            ctypes.c_uint32, ctypes.c_int32, ctypes.c_int64,
                                            ctypes.c_int64]
        lib.kvref_query_word.restype = ctypes.c_uint64
        lib.kvref_query_word.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32,
                                         ctypes.c_int64, ctypes.c_int64]
        lib.kvref_splitmix64.restype = ctypes.c_uint64
        lib.kvref_splitmix64.argtypes = [ctypes.c_uint64]
        lib.kvref_fill_store.argtypes = [ctypes.POINTER(KvGeom), ctypes.c_uint64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_void_p]
        lib.kvref_layer_block.argtypes = [ctypes.POINTER(KvGeom), ctypes.c_uint64, ctypes.c_int64,
                                          ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p]
        lib.kvref_hash_words.restype = ctypes.c_uint64
        lib.kvref_hash_words.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.kvref_layer_block_hash.restype = ctypes.c_uint64
        lib.kvref_layer_block_hash.argtypes = [ctypes.POINTER(KvGeom), ctypes.c_uint64,
                                               ctypes.c_int64, ctypes.c_int32, ctypes.c_int64]
        lib.kvref_gather.restype = ctypes.c_int
        lib.kvref_gather.argtypes = [ctypes.POINTER(KvGeom), ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.POINTER(KvJob), ctypes.c_int32, ctypes.c_void_p,
                                     ctypes.c_int32]
        lib.kvref_gather_mt.restype = ctypes.c_int64
        lib.kvref_gather_mt.argtypes = [ctypes.POINTER(KvGeom), ctypes.c_void_p,
                                        ctypes.POINTER(KvJob), ctypes.c_int32, ctypes.c_void_p,
                                        ctypes.c_int32, ctypes.c_int]
        _kv = lib
    return _kv


def geom(n_layer, block_tokens, b):
    return KvGeom(n_layer, block_tokens, b)


def fill_store(g, seed, n_fb, fb0=0):
    fb_bytes = g.n_layer * g.block_tokens * g.bytes_per_token_layer
    out = np.empty(n_fb * fb_bytes, dtype=np.uint8)
    kvref().kvref_fill_store(ctypes.byref(g), seed, fb0, n_fb, out.ctypes.data)
    return out


def layer_block(g, seed, fb, layer, ntok):
    out = np.empty(ntok * g.bytes_per_token_layer, dtype=np.uint8)
    kvref().kvref_layer_block(ctypes.byref(g), seed, fb, layer, ntok, out.ctypes.data)
    return out


def attend_digest(g, seed, fbs, cached, req, layer, q_begin, bsz):
    """Oracle of K5 (dp_prefill_attend) for one request chunk at one layer."""
    arr = (ctypes.c_int64 * max(1, len(fbs)))(*fbs)
    return kvref().kvref_attend_digest(ctypes.byref(g), seed, arr, cached, req, layer, q_begin, bsz)


def attend_digest_bruteforce(g, seed, fbs, cached, req, layer, q_begin, bsz):
    """The literal double sum in numpy (small cases): pins the column-sum form."""
    b = g.bytes_per_token_layer
    keys = np.concatenate([layer_block(g, seed, fb, layer, g.block_tokens) for fb in fbs])[: cached * b]
    keys = keys.reshape(cached, b).astype(np.uint64)
    qw = np.array([[kvref().kvref_query_word(seed, req, layer, q, w) for w in range(b // 8)]
                   for q in range(q_begin, q_begin + bsz)], dtype=np.uint64)
    qs = qw.view(np.uint8).reshape(bsz, b).astype(np.uint64)
    return int((qs @ keys.T).sum(dtype=np.uint64))


def layer_block_hash(g, seed, fb, layer, ntok):
    return kvref().kvref_layer_block_hash(ctypes.byref(g), seed, fb, layer, ntok)


def hash_bytes(buf):
    buf = np.ascontiguousarray(buf)
    return kvref().kvref_hash_words(buf.ctypes.data, buf.nbytes // 8)


def make_jobs(job_specs):
    """job_specs: list of (src_fb list, slot list, n_tokens, layer_begin, layer_end).
    Returns (ctypes array, keepalive)."""
    keep = []
    arr = (KvJob * max(1, len(job_specs)))()
    for i, (fbs, slots, ntok, l0, l1) in enumerate(job_specs):
        a = np.ascontiguousarray(fbs, dtype=np.int64)
        s = np.ascontiguousarray(slots, dtype=np.int32)
        keep += [a, s]
        arr[i].src_fb = a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        arr[i].dst_slot = s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        arr[i].n_tokens = ntok
        arr[i].n_blk = len(fbs)
        arr[i].layer_begin = l0
        arr[i].layer_end = l1
        arr[i].ticket = -1
    return arr, keep


def gather(g, store, store_fb, job_specs, n_slots, pool=None):
    """CPU restatement of K1/K2: returns the pool image [L][n_slots][T][b] (uint8)."""
    lb = g.block_tokens * g.bytes_per_token_layer
    if pool is None:
        pool = np.zeros(g.n_layer * n_slots * lb, dtype=np.uint8)
    arr, keep = make_jobs(job_specs)
    rc = kvref().kvref_gather(ctypes.byref(g), store.ctypes.data, store_fb, arr, len(job_specs),
                              pool.ctypes.data, n_slots)
    if rc != 0:
        raise ValueError("kvref_gather: job out of range")
    return pool


# ---------------------------------------------------------------- reference
def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle)")
        lib = ctypes.CDLL(REF_SO)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_synthesize.restype = ctypes.c_int
        lib.ref_synthesize.argtypes = [ctypes.c_int64] + [ctypes.c_double] * 6 + [
            ctypes.c_int, ctypes.c_uint64, ctypes.c_char_p]
        lib.ref_simulate.restype = ctypes.c_int
        I64P = ctypes.POINTER(ctypes.c_int64)
        lib.ref_build_forward_batch.restype = ctypes.c_int
        lib.ref_build_forward_batch.argtypes = [ctypes.c_int, I64P, ctypes.c_double,
                                                ctypes.POINTER(ctypes.c_double), I64P, I64P,
                                                ctypes.POINTER(ctypes.c_double)]
        lib.ref_derive_variant.restype = ctypes.c_int
        lib.ref_derive_variant.argtypes = [ctypes.c_char_p, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_int64, ctypes.c_char_p]
        lib.ref_extend_trace.restype = ctypes.c_int
        lib.ref_extend_trace.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p]
        lib.ref_poisson.restype = ctypes.c_int64
        lib.ref_poisson.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                    ctypes.POINTER(ctypes.c_double), ctypes.c_int64]
        lib.ref_simulate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p]
        I64P = ctypes.POINTER(ctypes.c_int64)
        IP = ctypes.POINTER(ctypes.c_int)
        for name in ("ref_schedule_pe_fetch", "ref_schedule_de_within_group"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_int, IP, I64P, ctypes.c_int, I64P, ctypes.c_int64,
                          ctypes.c_int64, ctypes.c_double, IP]
        lib.ref_schedule_de_groups.restype = ctypes.c_int
        lib.ref_schedule_de_groups.argtypes = [ctypes.c_int, IP, I64P, ctypes.c_int, I64P, IP]
        lib.ref_select_read_path.restype = ctypes.c_int
        lib.ref_select_read_path.argtypes = [ctypes.c_int64, ctypes.c_int64]
        _ref = lib
    return _ref


def ref_available():
    return os.path.exists(REF_SO)


def ref_synthesize(path, max_len=65536, count=500, seed=1, mean_turns=157.0, mean_append=429.0,
                   mean_gen=176.0, sigma_turns=0.5, sigma_append=0.6, sigma_gen=0.6):
    n = ref().ref_synthesize(max_len, mean_turns, mean_append, mean_gen, sigma_turns,
                             sigma_append, sigma_gen, count, seed, path.encode())
    if n < 0:
        raise ValueError(ref().ref_last_error().decode())
    return n


def _check(rc):
    if rc < 0:
        raise ValueError(ref().ref_last_error().decode())
    return rc


class QuotaInfeasible(Exception):
    pass


def ref_build_forward_batch(items, quota, cost):
    """Reference build_forward_batch.  items: [(request_id, cached, bsz)],
    cost: (bilinear, quadratic, linear, constant).  Returns (items, chunked,
    chunked_request_id, chunk_bsz, consumed_whole, estimated_time)."""
    n = len(items)
    flat = (ctypes.c_int64 * max(1, 3 * n))(*[v for it in items for v in it])
    c = (ctypes.c_double * 4)(*cost)
    out = (ctypes.c_int64 * max(1, 3 * n))()
    meta = (ctypes.c_int64 * 4)()
    t = ctypes.c_double()
    k = ref().ref_build_forward_batch(n, flat, quota, c, out, meta, ctypes.byref(t))
    if k == -2:
        raise QuotaInfeasible(ref().ref_last_error().decode())
    _check(k)
    got = [tuple(out[3 * i:3 * i + 3]) for i in range(k)]
    return got, bool(meta[0]), meta[1], meta[2], meta[3], t.value


def ref_derive_variant(in_path, out_path, append_scale, gen_scale, max_len):
    _check(ref().ref_derive_variant(in_path.encode(), append_scale, gen_scale, max_len,
                                    out_path.encode()))


def ref_extend_trace(in_path, out_path, seed):
    _check(ref().ref_extend_trace(in_path.encode(), seed, out_path.encode()))


def ref_poisson(rate, horizon, seed):
    n = _check(ref().ref_poisson(rate, horizon, seed, None, 0))
    buf = (ctypes.c_double * max(n, 1))()
    _check(ref().ref_poisson(rate, horizon, seed, buf, n))
    return list(buf[:n])


class RefError(Exception):
    pass


def ref_simulate(trace_path, **kv):
    """Run the reference simulator; kv keys as in oracle/ref_shim.cpp."""
    spec = ";".join(f"{k}={v}" for k, v in kv.items())
    fd, out = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    try:
        rc = ref().ref_simulate(trace_path.encode(), spec.encode(), out.encode())
        if rc != 0:
            kind = {-2: "ConfigError", -3: "SimulationError"}.get(rc, "Error")
            raise RefError(f"{kind}: {ref().ref_last_error().decode()}")
        with open(out) as f:
            return json.load(f)
    finally:
        os.unlink(out)


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def ref_schedule(name, queue, snaps, alpha, beta, z=1.05):
    ids, pid = _i32([q[0] for q in queue] or [0])
    tok, ptok = _i64([q[1] for q in queue] or [0])
    sn, psn = _i64(np.asarray(snaps, dtype=np.int64).reshape(-1) if snaps else [0])
    out = np.zeros(3 * max(1, len(queue)), dtype=np.int32)
    n = getattr(ref(), name)(len(queue), pid, ptok, len(snaps), psn, alpha, beta, z,
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    if n < 0:
        raise ValueError(ref().ref_last_error().decode())
    return [tuple(int(v) for v in out[3 * i:3 * i + 3]) for i in range(n)]


def ref_schedule_de_groups(queue, groups):
    ids, pid = _i32([q[0] for q in queue] or [0])
    tok, ptok = _i64([q[1] for q in queue] or [0])
    gr, pgr = _i64(np.asarray(groups, dtype=np.int64).reshape(-1) if groups else [0])
    out = np.zeros(2 * max(1, len(queue)), dtype=np.int32)
    n = ref().ref_schedule_de_groups(len(queue), pid, ptok, len(groups), pgr,
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n)]
