"""GPU parity of the PD handoff kernels through the C ABI:
the DE read path fused with DecodeH2D (dp_h2d_push_p2p_dual) and K3
(dp_prefill_handoff: prefill stand-in + PeToDe / MissMerge per layer).

After a request's handoff, both the PE pool and the DE decode pool must hold
the whole prompt KV [0, C+A) of every prompt block, byte for byte the content
formula of oracle/kvref.c (the hit part comes from storage, the miss part is
what the prefill stand-in writes: the same formula, i.e. what storage will
hold once the turn is persisted)."""

import numpy as np
import pytest

from oracle import refpy
from paper_2602_21548_b200 import abi

pytestmark = pytest.mark.gpu
SEED = 9


def dev(x, device, dtype):
    import torch
    return torch.tensor(np.asarray(x, dtype=dtype), device=f"cuda:{device}")


_streams = {}


def de_stream(device):
    """A non-blocking stream of the DE device (kept alive for the session)."""
    import torch
    if device not in _streams:
        _streams[device] = torch.cuda.Stream(device=device)
    return _streams[device].cuda_stream


def sync_all():
    import torch
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)


def check_prompt(pool, g_ref, fbs, slots, n_prompt, T, b, L):
    for k, (f, s) in enumerate(zip(fbs, slots)):
        n = min(T, n_prompt - k * T)
        for layer in range(L):
            got = pool.copy_out(layer, int(s), n * b)
            want = refpy.layer_block(g_ref, SEED, int(f), layer, n).tobytes()
            assert got == want, (k, layer)


@pytest.mark.parametrize("L,T,b,C,A", [
    (L, T, b, C, A) for L, T, b in [(8, 64, 576), (4, 64, 4096)]
    for C, A in [(64 * 5 + 10, 300), (64 * 3, 64), (0, 200), (130, 0)]] + [
    (61, 64, 576, 64 * 9 + 17, 429),    # DeepSeek-V3 MLA fp8, all 61 layers
    (64, 64, 4096, 64 * 4 + 33, 100)])  # config 3: Qwen2.5-32B GQA bf16, all 64 layers
def test_de_path_dual_then_missmerge(de_dev, L, T, b, C, A):
    """DE read path: the DE reads the hit blocks once (dual: PE pool + its own
    decode pool), the PE gates each layer on them, writes the miss KV and
    pushes only the miss part (MissMerge)."""
    g = abi.geom(L, T, b)
    P = C + A
    n_hit, n_prompt = -(-C // T), -(-P // T)
    rng = np.random.default_rng(C * 7 + A)
    s_de = de_stream(de_dev)  # before K3 spins: stream creation may wait for the device
    st_de = abi.Store(de_dev, g, 40, SEED)
    pe_pool = abi.Pool(0, g, 32, 2)   # row 0: hit KV landed, row 1: handoff done
    de_pool = abi.Pool(de_dev, g, 32, 2)
    pe_view_on_de = pe_pool.peer_view(de_dev)
    de_view_on_pe = de_pool.peer_view(0)
    try:
        fbs = (rng.integers(0, 40 - n_prompt) + np.arange(n_prompt)).astype(np.int64)
        pe_slots = rng.permutation(32)[:n_prompt].astype(np.int32)
        de_slots = rng.permutation(32)[:n_prompt].astype(np.int32)
        keep = [dev(fbs if n_prompt else [0], de_dev, np.int64), dev(pe_slots if n_prompt else [0], de_dev, np.int32),
                dev(de_slots if n_prompt else [0], de_dev, np.int32)]
        dj = (abi.DualJob * 1)()
        dj[0].pe = abi.Job(keep[0].data_ptr(), keep[1].data_ptr(), C, n_hit, 0, L, 0)
        dj[0].de_slot = keep[2].data_ptr()
        dj[0].de_ticket = 0
        on_pe = [dev(fbs if n_prompt else [0], 0, np.int64), dev(pe_slots if n_prompt else [0], 0, np.int32),
                 dev(de_slots if n_prompt else [0], 0, np.int32)]
        items = abi.layer_items(g, n_hit)
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(on_pe[0].data_ptr(), on_pe[1].data_ptr(), on_pe[2].data_ptr(), C, P,
                               n_prompt, 0, 0 if C else -1, items, 0, 1)
        # K3 first: it must block on the dual gather's per-layer releases
        # (the DE's own stream: on a shared GPU the legacy stream would
        # queue the producer behind its waiter)
        abi.prefill_handoff(pe_pool, de_view_on_pe, hj, 1, SEED, timeout_ms=20000)
        abi.push_p2p_dual(pe_view_on_de, de_pool, st_de, dj, 1, s_de)
        sync_all()
        assert abi.wait_status(pe_pool) == abi.DP_OK
        gr = refpy.geom(L, T, b)
        check_prompt(pe_pool, gr, fbs, pe_slots, P, T, b, L)
        check_prompt(de_pool, gr, fbs, de_slots, P, T, b, L)
        per_block = abi.layer_items(g, 1)
        want_layer = (n_hit + n_prompt) * per_block
        abi.wait_layer(de_pool, 0, L, want_layer * L, timeout_ms=2000)
        abi.wait_layer(de_pool, 0, L - 1, want_layer, timeout_ms=2000)
        abi.wait_layer(pe_pool, 1, L, n_prompt * per_block * L, timeout_ms=2000)  # K3 done row
        sync_all()
        assert abi.wait_status(de_pool) == abi.DP_OK
        assert abi.wait_status(pe_pool) == abi.DP_OK
    finally:
        for x in (de_view_on_pe, pe_view_on_de, de_pool, pe_pool, st_de):
            x.close()


@pytest.mark.parametrize("L,T,b,C,A", [(8, 64, 576, 64 * 7 + 33, 429), (8, 64, 576, 64 * 2, 1),
                                       (8, 64, 576, 0, 64 * 3 + 5), (61, 64, 576, 64 * 6 + 1, 429),
                                       (64, 64, 4096, 64 * 3 + 40, 90)])
@pytest.mark.parametrize("tma", [False, True])
def test_pe_path_load_then_petode(de_dev, L, T, b, C, A, tma):
    """PE read path: K1 loads the hit KV into the PE pool; K3 (stream-ordered
    after it) writes the miss KV and pushes the whole prompt (PeToDe) --
    the hit part by 16-byte register copies or through the TMA."""
    abi.set_handoff_tma(tma)
    g = abi.geom(L, T, b)
    P = C + A
    n_hit, n_prompt = -(-C // T), -(-P // T)
    rng = np.random.default_rng(P)
    st_pe = abi.Store(0, g, 40, SEED)
    pe_pool = abi.Pool(0, g, 32, 1)
    de_pool = abi.Pool(de_dev, g, 32, 1)
    de_view = de_pool.peer_view(0)
    try:
        fbs = (rng.integers(0, 40 - n_prompt) + np.arange(n_prompt)).astype(np.int64)
        pe_slots = rng.permutation(32)[:n_prompt].astype(np.int32)
        de_slots = rng.permutation(32)[:n_prompt].astype(np.int32)
        t = [dev(fbs, 0, np.int64), dev(pe_slots, 0, np.int32), dev(de_slots, 0, np.int32)]
        if n_hit:
            abi.h2d_layer_gather(pe_pool, st_pe, abi.make_jobs(
                [(t[0].data_ptr(), t[1].data_ptr(), C, n_hit, 0, L, -1)]), 1)
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), C, P, n_prompt, 1, -1, 0, 0, -1)
        abi.prefill_handoff(pe_pool, de_view, hj, 1, SEED)  # same (legacy) stream: ordered after K1
        sync_all()
        gr = refpy.geom(L, T, b)
        check_prompt(pe_pool, gr, fbs, pe_slots, P, T, b, L)
        check_prompt(de_pool, gr, fbs, de_slots, P, T, b, L)
        abi.wait_layer(de_pool, 0, L, n_prompt * abi.layer_items(g, 1) * L, timeout_ms=2000)
        sync_all()
        assert abi.wait_status(de_pool) == abi.DP_OK
    finally:
        abi.set_handoff_tma(False)
        for x in (de_view, de_pool, pe_pool, st_pe):
            x.close()


def test_handoff_gate_watchdog(de_dev):
    """A layer whose hit KV never lands trips the watchdog instead of hanging."""
    L, T, b = 2, 64, 576
    g = abi.geom(L, T, b)
    pe_pool = abi.Pool(0, g, 4, 1)
    de_pool = abi.Pool(de_dev, g, 4, 1)
    de_view = de_pool.peer_view(0)
    try:
        t = [dev([0, 1], 0, np.int64), dev([0, 1], 0, np.int32), dev([0, 1], 0, np.int32)]
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), 64, 100, 2, 0, 0, 1, 0, -1)
        abi.prefill_handoff(pe_pool, de_view, hj, 1, SEED, timeout_ms=50)
        sync_all()
        assert abi.wait_status(pe_pool) == abi.DP_ETIMEOUT
    finally:
        for x in (de_view, de_pool, pe_pool):
            x.close()


def test_stream_wait_counter_orders_a_stream(de_dev):
    """dp_stream_wait_counter: the PE stream waits (no SMs) for a counter the
    DE's dual gather releases, then K3 runs without its in-kernel gate."""
    L, T, b = 4, 64, 576
    g = abi.geom(L, T, b)
    C, A = 64 * 3 + 5, 70
    P = C + A
    n_hit, n_prompt = -(-C // T), -(-P // T)
    s_de = de_stream(de_dev)
    st_de = abi.Store(de_dev, g, 16, SEED)
    pe_pool = abi.Pool(0, g, 16, 2)
    de_pool = abi.Pool(de_dev, g, 16, 1)
    pe_view = pe_pool.peer_view(de_dev)
    de_view = de_pool.peer_view(0)
    try:
        fbs = np.arange(3, 3 + n_prompt, dtype=np.int64)
        ps = np.arange(n_prompt, dtype=np.int32)
        dsl = np.arange(8, 8 + n_prompt, dtype=np.int32)
        on_de = [dev(fbs, de_dev, np.int64), dev(ps, de_dev, np.int32), dev(dsl, de_dev, np.int32)]
        on_pe = [dev(fbs, 0, np.int64), dev(ps, 0, np.int32), dev(dsl, 0, np.int32)]
        items = abi.layer_items(g, n_hit)
        abi.stream_wait_counter(pe_pool, 0, L, items * L)  # legacy stream of device 0
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(on_pe[0].data_ptr(), on_pe[1].data_ptr(), on_pe[2].data_ptr(), C, P,
                               n_prompt, 0, -1, 0, 0, 1)
        abi.prefill_handoff(pe_pool, de_view, hj, 1, SEED)
        dj = (abi.DualJob * 1)()
        dj[0].pe = abi.Job(on_de[0].data_ptr(), on_de[1].data_ptr(), C, n_hit, 0, L, 0)
        dj[0].de_slot = on_de[2].data_ptr()
        dj[0].de_ticket = 0
        abi.push_p2p_dual(pe_view, de_pool, st_de, dj, 1, s_de)
        sync_all()
        gr = refpy.geom(L, T, b)
        check_prompt(pe_pool, gr, fbs, ps, P, T, b, L)
        check_prompt(de_pool, gr, fbs, dsl, P, T, b, L)
    finally:
        for x in (de_view, pe_view, de_pool, pe_pool, st_de):
            x.close()


# ------------------------------------------------------------ persistence
@pytest.mark.parametrize("L,T,b", [(6, 64, 576), (3, 64, 4096)])
@pytest.mark.parametrize("P,gen", [(64 * 3 + 10, 130), (128, 64), (5, 1)])
def test_decode_fill_then_persist_d2h(gpus, L, T, b, P, gen):
    """Decode stand-in writes generated tokens [P, P+gen) into the decode pool;
    K4 gathers them, every layer, into host Full Blocks [L][T][b] in chunks of
    64 generated tokens plus the final partial (desim.cpp:666-672, :690-693)."""
    g = abi.geom(L, T, b)
    total = P + gen
    blk0, blk1 = P // T, -(-total // T)
    n = blk1 - blk0
    pool = abi.Pool(0, g, 16, 1)
    target = abi.Store(0, g, 24, SEED + 1)  # different content: proves the write
    try:
        slots = np.arange(3, 3 + n, dtype=np.int32)
        fbs = np.arange(10, 10 + n, dtype=np.int64)
        ds, df = dev(slots, 0, np.int32), dev(fbs, 0, np.int64)
        fill = (abi.SpanJob * 1)()
        fill[0] = abi.SpanJob(ds.data_ptr(), df.data_ptr(), blk0, P, total, n, 0)
        abi.decode_fill(pool, fill, 1, SEED)
        chunks, done = [], 0
        for k in list(range(T, gen, T)) + [gen]:  # persist_tokens milestones
            if k > done:
                chunks.append((P + done, P + k))
                done = k
        jobs = (abi.SpanJob * len(chunks))()
        for i, (t0, t1) in enumerate(chunks):
            jobs[i] = abi.SpanJob(ds.data_ptr(), df.data_ptr(), blk0, t0, t1, n, 0)
        abi.persist_d2h(pool, target, jobs, len(chunks))
        sync_all()
        img = np.frombuffer(target.bytes(), dtype=np.uint8)
        gr = refpy.geom(L, T, b)
        fb_bytes, lb = L * T * b, T * b
        for i in range(n):
            k = blk0 + i
            a, z = max(P, k * T) - k * T, min(total, (k + 1) * T) - k * T
            for layer in range(L):
                full = refpy.layer_block(gr, SEED, int(fbs[i]), layer, T)
                other = refpy.layer_block(gr, SEED + 1, int(fbs[i]), layer, T)
                off = int(fbs[i]) * fb_bytes + layer * lb
                got = img[off:off + lb]
                assert np.array_equal(got[a * b:z * b], full[a * b:z * b])      # persisted
                assert np.array_equal(got[:a * b], other[:a * b])               # untouched
                assert np.array_equal(got[z * b:], other[z * b:])
        assert sum(t1 - t0 for t0, t1 in chunks) == gen
    finally:
        target.close()
        pool.close()


@pytest.mark.parametrize("L,T,b", [(6, 64, 576), (3, 64, 4096), (61, 64, 576)])
@pytest.mark.parametrize("P,gen", [(64 * 3 + 10, 330), (128, 64 * 5), (5, 1), (64 * 2 + 63, 2)])
def test_persist_staged(gpus, L, T, b, P, gen):
    """K4 staged: the persist chunks of a request (64 generated tokens each +
    the final partial) gathered into the HBM ring and copied to the host
    Full Blocks by the copy engine (whole blocks 1D, partial ones 2D), with
    a ring of 2 Full Blocks per segment so the spans cross segments: the
    same bytes as dp_persist_d2h, nothing outside the spans touched."""
    g = abi.geom(L, T, b)
    total = P + gen
    blk0, blk1 = P // T, -(-total // T)
    n = blk1 - blk0
    pool = abi.Pool(0, g, 16, 1)
    target = abi.Store(0, g, 24, SEED + 1)
    stager = abi.Stager(0, g, 2 * L * T * b * 4)  # 4 segments of 2 Full Blocks
    try:
        slots = np.arange(3, 3 + n, dtype=np.int32)
        fbs = (np.arange(n) * 2 + 1).astype(np.int64)  # non-consecutive targets, plus a run below
        if n > 3:
            fbs[1:4] = [14, 15, 16]
        ds, df = dev(slots, 0, np.int32), dev(fbs, 0, np.int64)
        fill = (abi.SpanJob * 1)()
        fill[0] = abi.SpanJob(ds.data_ptr(), df.data_ptr(), blk0, P, total, n, 0)
        abi.decode_fill(pool, fill, 1, SEED)
        chunks, done = [], 0
        for k in list(range(T, gen, T)) + [gen]:
            if k > done:
                chunks.append((P + done, P + k))
                done = k
        jobs = (abi.SpanJob * len(chunks))()
        for i, (t0, t1) in enumerate(chunks):
            jobs[i] = abi.SpanJob(ds.data_ptr(), fbs.ctypes.data, blk0, t0, t1, n, 0)
        l0 = stager.launches()
        abi.persist_staged(pool, target, stager, jobs, len(chunks))
        sync_all()
        assert stager.launches() > l0
        img = np.frombuffer(target.bytes(), dtype=np.uint8)
        gr = refpy.geom(L, T, b)
        fb_bytes, lb = L * T * b, T * b
        for i in range(n):
            k = blk0 + i
            a, z = max(P, k * T) - k * T, min(total, (k + 1) * T) - k * T
            for layer in range(L):
                full = refpy.layer_block(gr, SEED, int(fbs[i]), layer, T)
                other = refpy.layer_block(gr, SEED + 1, int(fbs[i]), layer, T)
                off = int(fbs[i]) * fb_bytes + layer * lb
                got = img[off:off + lb]
                assert np.array_equal(got[a * b:z * b], full[a * b:z * b]), (i, layer)
                assert np.array_equal(got[:a * b], other[:a * b])
                assert np.array_equal(got[z * b:], other[z * b:])
        untouched = set(range(24)) - set(int(f) for f in fbs)
        for f in untouched:
            off = f * fb_bytes
            assert np.array_equal(img[off:off + lb], refpy.layer_block(gr, SEED + 1, f, 0, T))
    finally:
        for x in (stager, target, pool):
            x.close()


@pytest.mark.parametrize("L,T,b,C", [(8, 64, 576, 64 * 9 + 5), (4, 64, 4096, 64 * 5), (61, 64, 576, 64 * 3 + 1)])
def test_dual_staged(de_dev, L, T, b, C):
    """The DE read path fused with DecodeH2D, staged (copy engine into the
    ring, then the dual scatter): PE pool and decode pool both hold the hit
    KV, both rows released, with a ring smaller than the request."""
    import torch
    g = abi.geom(L, T, b)
    nh = -(-C // T)
    s_de = de_stream(de_dev)
    st_de = abi.Store(de_dev, g, 40, SEED)
    pe_pool = abi.Pool(0, g, 32, 1)
    de_pool = abi.Pool(de_dev, g, 32, 1)
    pe_view = pe_pool.peer_view(de_dev)
    stager = abi.Stager(de_dev, g, 3 * L * T * b * 4)  # 3 Full Blocks per segment
    try:
        fbs = (np.arange(nh) * 2 + 1).astype(np.int64)  # non-consecutive: one copy per block
        ps = np.arange(3, 3 + nh, dtype=np.int32)
        ds = np.arange(20, 20 + nh, dtype=np.int32)[::-1].copy()
        keep = [fbs, dev(ps, de_dev, np.int32), dev(ds, de_dev, np.int32)]
        dj = (abi.DualJob * 1)()
        dj[0].pe = abi.Job(fbs.ctypes.data, keep[1].data_ptr(), C, nh, 0, L, 0)
        dj[0].de_slot = keep[2].data_ptr()
        dj[0].de_ticket = 0
        abi.push_dual_staged(pe_view, de_pool, st_de, stager, dj, 1, s_de)
        sync_all()
        gr = refpy.geom(L, T, b)
        check_prompt(pe_pool, gr, fbs, ps, C, T, b, L)
        check_prompt(de_pool, gr, fbs, ds, C, T, b, L)
        items = abi.layer_items(g, nh)
        abi.wait_layer(pe_pool, 0, L, items * L, timeout_ms=2000)
        abi.wait_layer(de_pool, 0, L, items * L, timeout_ms=2000)
        sync_all()
        assert abi.wait_status(pe_pool) == abi.DP_OK and abi.wait_status(de_pool) == abi.DP_OK
        assert stager.launches() >= 2
    finally:
        for x in (stager, pe_view, de_pool, pe_pool, st_de):
            x.close()


# ------------------------------------------------- K3 on the copy engines
def _slots(rng, n, pool_slots, layout):
    """Block tables: 'runs' = two consecutive runs (the executor's usual
    FIFO allocation), 'scattered' = a permutation (one copy per block)."""
    if layout == "scattered":
        return rng.permutation(pool_slots)[:n].astype(np.int32)
    cut = n // 2
    return np.concatenate([np.arange(1, 1 + cut), np.arange(pool_slots - (n - cut), pool_slots)]).astype(np.int32)


@pytest.mark.parametrize("L,T,b,C,A", [(8, 64, 576, 64 * 7 + 33, 429), (8, 64, 576, 64 * 2, 1),
                                       (8, 64, 576, 0, 64 * 3 + 5), (8, 64, 576, 64 * 4, 0),
                                       (61, 64, 576, 64 * 6 + 1, 429), (64, 64, 4096, 64 * 3 + 40, 90)])
@pytest.mark.parametrize("layout", ["runs", "scattered"])
def test_pe_path_petode_copy_engine(de_dev, L, T, b, C, A, layout):
    """dp_prefill_handoff_copy, PE read path, no gate: one 2D copy per run of
    hit blocks (all layers), the side kernel writes the miss KV into both
    pools, then releases every layer -- pools and counters as K3's."""
    g = abi.geom(L, T, b)
    P = C + A
    n_hit, n_prompt = -(-C // T), -(-P // T)
    rng = np.random.default_rng(P + 1)
    st_pe = abi.Store(0, g, 40, SEED)
    pe_pool = abi.Pool(0, g, 32, 2)
    de_pool = abi.Pool(de_dev, g, 32, 1)
    de_view = de_pool.peer_view(0)
    try:
        fbs = (rng.integers(0, 40 - n_prompt) + np.arange(n_prompt)).astype(np.int64)
        pe_slots = _slots(rng, n_prompt, 32, layout)
        de_slots = _slots(rng, n_prompt, 32, layout)[::-1].copy() if layout == "scattered" else \
            _slots(rng, n_prompt, 32, layout)
        t = [dev(fbs, 0, np.int64), dev(pe_slots, 0, np.int32)]
        if n_hit:
            abi.h2d_layer_gather(pe_pool, st_pe, abi.make_jobs(
                [(t[0].data_ptr(), t[1].data_ptr(), C, n_hit, 0, L, -1)]), 1)
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(fbs.ctypes.data, pe_slots.ctypes.data, de_slots.ctypes.data, C, P, n_prompt, 1,
                               -1, 0, 0, 1)
        n0 = abi.handoff_copy_launches()
        abi.prefill_handoff_copy(pe_pool, de_view, hj, 1, SEED)  # legacy stream: ordered after K1
        sync_all()
        assert abi.handoff_copy_launches() - n0 <= 2
        gr = refpy.geom(L, T, b)
        check_prompt(pe_pool, gr, fbs, pe_slots, P, T, b, L)
        check_prompt(de_pool, gr, fbs, de_slots, P, T, b, L)
        per = n_prompt * abi.layer_items(g, 1)
        abi.wait_layer(de_pool, 0, L, per * L, timeout_ms=2000)
        abi.wait_layer(de_pool, 0, L - 1, per, timeout_ms=2000)
        abi.wait_layer(pe_pool, 1, L, per * L, timeout_ms=2000)  # K3 done row
        sync_all()
        assert abi.wait_status(de_pool) == abi.DP_OK and abi.wait_status(pe_pool) == abi.DP_OK
    finally:
        for x in (de_view, de_pool, pe_pool, st_pe):
            x.close()


@pytest.mark.parametrize("L,T,b,C,A", [(8, 64, 576, 64 * 5 + 10, 300), (8, 64, 576, 0, 200),
                                       (61, 64, 576, 64 * 9 + 17, 429), (64, 64, 4096, 64 * 4 + 33, 100)])
@pytest.mark.parametrize("memop", [False, True])
def test_de_path_missmerge_copy_engine(de_dev, L, T, b, C, A, memop):
    """dp_prefill_handoff_copy gated per layer on the DE's dual gather (the
    DE read path): the side kernel of layer l waits for l's hit KV (or, with
    dp_set_handoff_gate_memop, the stream waits for it), writes the miss KV
    into both pools and releases layer l - 1."""
    if memop and de_dev == 0:
        pytest.skip("a stream wait blocks its hardware queue: its producer on the same GPU must be "
                    "enqueued first (the executor's order), which this two-stream test does not do")
    abi.set_handoff_gate_memop(memop)
    g = abi.geom(L, T, b)
    P = C + A
    n_hit, n_prompt = -(-C // T), -(-P // T)
    rng = np.random.default_rng(C * 3 + A)
    s_de = de_stream(de_dev)
    st_de = abi.Store(de_dev, g, 40, SEED)
    pe_pool = abi.Pool(0, g, 32, 2)
    de_pool = abi.Pool(de_dev, g, 32, 2)
    pe_view_on_de = pe_pool.peer_view(de_dev)
    de_view_on_pe = de_pool.peer_view(0)
    try:
        fbs = (rng.integers(0, 40 - n_prompt) + np.arange(n_prompt)).astype(np.int64)
        pe_slots = rng.permutation(32)[:n_prompt].astype(np.int32)
        de_slots = rng.permutation(32)[:n_prompt].astype(np.int32)
        keep = [dev(fbs if n_prompt else [0], de_dev, np.int64), dev(pe_slots if n_prompt else [0], de_dev, np.int32),
                dev(de_slots if n_prompt else [0], de_dev, np.int32)]
        dj = (abi.DualJob * 1)()
        dj[0].pe = abi.Job(keep[0].data_ptr(), keep[1].data_ptr(), C, n_hit, 0, L, 0)
        dj[0].de_slot = keep[2].data_ptr()
        dj[0].de_ticket = 0
        items = abi.layer_items(g, n_hit)
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(fbs.ctypes.data, pe_slots.ctypes.data, de_slots.ctypes.data, C, P,
                               n_prompt, 0, 0 if C else -1, items, 0, 1)
        abi.prefill_handoff_copy(pe_pool, de_view_on_pe, hj, 1, SEED, timeout_ms=20000)
        abi.push_p2p_dual(pe_view_on_de, de_pool, st_de, dj, 1, s_de)
        sync_all()
        assert abi.wait_status(pe_pool) == abi.DP_OK
        gr = refpy.geom(L, T, b)
        check_prompt(pe_pool, gr, fbs, pe_slots, P, T, b, L)
        check_prompt(de_pool, gr, fbs, de_slots, P, T, b, L)
        per_block = abi.layer_items(g, 1)
        want_layer = (n_hit + n_prompt) * per_block
        abi.wait_layer(de_pool, 0, L, want_layer * L, timeout_ms=2000)
        abi.wait_layer(de_pool, 0, L - 1, want_layer, timeout_ms=2000)
        abi.wait_layer(pe_pool, 1, L, n_prompt * per_block * L, timeout_ms=2000)
        sync_all()
        assert abi.wait_status(de_pool) == abi.DP_OK and abi.wait_status(pe_pool) == abi.DP_OK
    finally:
        abi.set_handoff_gate_memop(False)
        for x in (de_view_on_pe, pe_view_on_de, de_pool, pe_pool, st_de):
            x.close()


def test_handoff_copy_gate_watchdog(de_dev):
    """The copy-engine K3's layer gate trips the watchdog instead of hanging."""
    L, T, b = 2, 64, 576
    g = abi.geom(L, T, b)
    pe_pool = abi.Pool(0, g, 4, 1)
    de_pool = abi.Pool(de_dev, g, 4, 1)
    de_view = de_pool.peer_view(0)
    try:
        fbs, sl = np.array([0, 1], dtype=np.int64), np.array([0, 1], dtype=np.int32)
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(fbs.ctypes.data, sl.ctypes.data, sl.ctypes.data, 64, 100, 2, 0, 0, 1, 0, -1)
        abi.prefill_handoff_copy(pe_pool, de_view, hj, 1, SEED, timeout_ms=50)
        sync_all()
        assert abi.wait_status(pe_pool) == abi.DP_ETIMEOUT
    finally:
        for x in (de_view, de_pool, pe_pool):
            x.close()


def test_handoff_copy_many_jobs(de_dev):
    """dp_prefill_handoff_copy with more jobs than one parameter block holds
    (50 > DP_MAX_HANDOFF_JOBS_PER_LAUNCH): handled in groups, every prompt in
    both pools, every DE row released once per layer and block."""
    L, T, b = 3, 64, 576
    g = abi.geom(L, T, b)
    n_jobs, per = 50, 2  # 2 prompt blocks per job: 1 hit block + a partial miss block
    st_pe = abi.Store(0, g, 2 * n_jobs + 4, SEED)
    pe_pool = abi.Pool(0, g, 2 * n_jobs, 1)
    de_pool = abi.Pool(de_dev, g, 2 * n_jobs, n_jobs)
    de_view = de_pool.peer_view(0)
    try:
        keep, jobs_k1 = [], []
        hj = (abi.HandoffJob * n_jobs)()
        C, P = T, T + 17
        for j in range(n_jobs):
            fbs = np.array([2 * j + 1, 2 * j + 2], dtype=np.int64)
            ps = np.array([2 * j, 2 * j + 1], dtype=np.int32)
            ds = np.array([2 * n_jobs - 1 - 2 * j, 2 * n_jobs - 2 - 2 * j], dtype=np.int32)  # reversed: runs of 1
            t = [dev(fbs, 0, np.int64), dev(ps, 0, np.int32)]
            keep += [fbs, ps, ds] + t
            jobs_k1.append((t[0].data_ptr(), t[1].data_ptr(), C, 1, 0, L, -1))
            hj[j] = abi.HandoffJob(fbs.ctypes.data, ps.ctypes.data, ds.ctypes.data, C, P, per, 1, -1, 0, j, -1)
        abi.h2d_layer_gather(pe_pool, st_pe, abi.make_jobs(jobs_k1), n_jobs)
        abi.prefill_handoff_copy(pe_pool, de_view, hj, n_jobs, SEED)
        sync_all()
        gr = refpy.geom(L, T, b)
        items = abi.layer_items(g, per)
        for j in range(n_jobs):
            fbs, ds = keep[5 * j], keep[5 * j + 2]
            check_prompt(de_pool, gr, fbs, ds, P, T, b, L)
            abi.wait_layer(de_pool, j, L, items * L, timeout_ms=2000)
        sync_all()
        assert abi.wait_status(de_pool) == abi.DP_OK
    finally:
        for x in (de_view, de_pool, pe_pool, st_pe):
            x.close()


def test_persist_staged_two_requests(gpus):
    """dp_persist_staged with the chunks of two requests interleaved in one
    call, an empty span among them, and a ring of one Full Block per segment:
    spans are merged only within a request; the bytes equal dp_persist_d2h's."""
    L, T, b = 4, 64, 576
    g = abi.geom(L, T, b)
    pool = abi.Pool(0, g, 32, 1)
    a_store = abi.Store(0, g, 24, SEED + 1)
    b_store = abi.Store(0, g, 24, SEED + 1)
    stager = abi.Stager(0, g, 1 * L * T * b * 4)
    try:
        reqs = [(64 * 2 + 5, 200, np.arange(0, 6, dtype=np.int32), np.arange(10, 16, dtype=np.int64)),
                (64 + 63, 70, np.arange(8, 12, dtype=np.int32), np.array([3, 5, 7, 9], dtype=np.int64))]
        keep, dev_jobs, host_jobs = [], [], []
        for P, gen, slots, fbs in reqs:
            blk0, n = P // T, -(-(P + gen) // T) - P // T
            ds, df = dev(slots[:n], 0, np.int32), dev(fbs[:n], 0, np.int64)
            fh = fbs[:n].copy()
            keep += [ds, df, fh]
            fill = (abi.SpanJob * 1)()
            fill[0] = abi.SpanJob(ds.data_ptr(), df.data_ptr(), blk0, P, P + gen, n, 0)
            abi.decode_fill(pool, fill, 1, SEED)
            done = 0
            for k in list(range(T, gen, T)) + [gen]:
                if k > done:
                    dev_jobs.append((ds.data_ptr(), df.data_ptr(), blk0, P + done, P + k, n))
                    host_jobs.append((ds.data_ptr(), fh.ctypes.data, blk0, P + done, P + k, n))
                    done = k
        order = [0, len(dev_jobs) - 1, 1] + list(range(2, len(dev_jobs) - 1))  # interleave the requests
        for jobs, fn, target in ((dev_jobs, abi.persist_d2h, a_store), (host_jobs, None, b_store)):
            arr = (abi.SpanJob * (len(order) + 1))()
            for i, o in enumerate(order):
                arr[i] = abi.SpanJob(*jobs[o], 0)
            arr[len(order)] = abi.SpanJob(jobs[0][0], jobs[0][1], jobs[0][2], jobs[0][3], jobs[0][3], jobs[0][5], 0)
            if fn:
                fn(pool, target, arr, len(order) + 1)
            else:
                abi.persist_staged(pool, target, stager, arr, len(order) + 1)
        sync_all()
        assert a_store.bytes() == b_store.bytes()
    finally:
        for x in (stager, b_store, a_store, pool):
            x.close()
