"""GPU parity of the sm_100a kernels, called through the C ABI
(include/dualpath/kv_abi.h), against the CPU oracle (oracle/kvref.c).

Bar: bit-exact bytes for every moved Layer Block (integer/byte work)."""

import ctypes

import numpy as np
import pytest

from oracle import refpy
from paper_2602_21548_b200 import abi

pytestmark = pytest.mark.gpu

SEED = 9
GEOMS = [(4, 64, 576), (61, 64, 576), (2, 64, 4096), (3, 16, 1024)]  # DS-V3, Qwen-like, tiny


def dev_i64(x, device=0):
    import torch
    return torch.tensor(np.asarray(x, dtype=np.int64), device=f"cuda:{device}")


def dev_i32(x, device=0):
    import torch
    return torch.tensor(np.asarray(x, dtype=np.int32), device=f"cuda:{device}")


def sync():
    import torch
    torch.cuda.synchronize()


@pytest.mark.parametrize("L,T,b", GEOMS)
def test_store_content_matches_oracle(gpus, L, T, b):
    g = abi.geom(L, T, b)
    st = abi.Store(0, g, 5, SEED)
    try:
        got = np.frombuffer(st.bytes(), dtype=np.uint8)
        want = refpy.fill_store(refpy.geom(L, T, b), SEED, 5)
        assert got.shape == want.shape
        assert np.array_equal(got, want)
    finally:
        st.close()


def random_jobs(rng, L, T, n_jobs, n_fb, n_slots, max_blk, device=0, layers=None):
    """Random jobs with partial last blocks and disjoint slots."""
    perm = rng.permutation(n_slots)
    used = 0
    specs, keep, plain = [], [], []
    for t in range(n_jobs):
        nblk = int(rng.integers(0, max_blk + 1))
        if used + nblk > n_slots:
            nblk = 0
        ntok = 0 if nblk == 0 else (nblk - 1) * T + int(rng.integers(1, T + 1))
        fbs = rng.integers(0, n_fb, nblk).astype(np.int64)
        slots = perm[used:used + nblk].astype(np.int32)
        used += nblk
        l0, l1 = layers if layers else (0, L)
        df, ds = dev_i64(fbs if nblk else [0], device), dev_i32(slots if nblk else [0], device)
        keep += [df, ds]
        specs.append((df.data_ptr(), ds.data_ptr(), ntok, nblk, l0, l1, t))
        plain.append((fbs, slots, ntok, l0, l1))
    return specs, keep, plain


def check_pool(pool, g_ref, plain, T, b, store_img, n_slots):
    want = refpy.gather(g_ref, store_img, store_img.nbytes // (g_ref.n_layer * T * b),
                        [(f, s, n, l0, l1) for f, s, n, l0, l1 in plain], n_slots)
    lb = T * b
    for fbs, slots, ntok, l0, l1 in plain:
        for k, s in enumerate(slots):
            n = min(T, ntok - k * T) * b
            for layer in range(l0, l1):
                got = pool.copy_out(layer, int(s), n)
                off = (layer * n_slots + int(s)) * lb
                assert got == want[off:off + n].tobytes(), (layer, s, k)


@pytest.mark.parametrize("L,T,b", GEOMS + [(64, 64, 4096)])  # + config 3's full Qwen shape
def test_k1_gather_parity(gpus, L, T, b):
    rng = np.random.default_rng(L * 1000 + b)
    g = abi.geom(L, T, b)
    n_fb, n_slots = 12, 64
    st = abi.Store(0, g, n_fb, SEED)
    pool = abi.Pool(0, g, n_slots, 80)
    try:
        # 70 jobs -> two launches (64 job headers per launch); some empty
        specs, keep, plain = random_jobs(rng, L, T, 70, n_fb, n_slots, 3)
        jobs = abi.make_jobs(specs)
        abi.h2d_layer_gather(pool, st, jobs, len(specs))
        sync()
        store_img = np.frombuffer(st.bytes(), dtype=np.uint8).copy()
        check_pool(pool, refpy.geom(L, T, b), plain, T, b, store_img, n_slots)
        # landed counters: the all-layer column reaches items * layers
        for t, (fbs, slots, ntok, l0, l1) in enumerate(plain):
            items = abi.layer_items(g, len(slots))
            abi.wait_layer(pool, t, L, items * (l1 - l0), timeout_ms=5000)
            if len(slots):
                abi.wait_layer(pool, t, l0, items, timeout_ms=5000)
        sync()
        assert abi.wait_status(pool) == abi.DP_OK
    finally:
        pool.close()
        st.close()


def test_k1_layer_subrange_and_chunks(gpus):
    # Qwen-like Layer Block (256 KiB) -> 4 chunk items per block; layers 3..5 only
    L, T, b = 8, 64, 4096
    rng = np.random.default_rng(5)
    g = abi.geom(L, T, b)
    st = abi.Store(0, g, 6, SEED)
    pool = abi.Pool(0, g, 16, 8)
    try:
        specs, keep, plain = random_jobs(rng, L, T, 6, 6, 16, 2, layers=(3, 6))
        assert abi.layer_items(g, 1) == 4
        abi.h2d_layer_gather(pool, st, abi.make_jobs(specs), len(specs))
        sync()
        store_img = np.frombuffer(st.bytes(), dtype=np.uint8).copy()
        check_pool(pool, refpy.geom(L, T, b), plain, T, b, store_img, 16)
    finally:
        pool.close()
        st.close()


def test_checksum_matches_oracle(gpus):
    L, T, b = 4, 64, 576
    g = abi.geom(L, T, b)
    st = abi.Store(0, g, 4, SEED)
    pool = abi.Pool(0, g, 8, 1)
    try:
        fbs, slots, ntok = [3, 1, 2], [5, 0, 7], 64 * 2 + 9
        df, ds = dev_i64(fbs), dev_i32(slots)
        abi.h2d_layer_gather(pool, st, abi.make_jobs([(df.data_ptr(), ds.data_ptr(), ntok, 3, 0, L, 0)]), 1)
        import torch
        ntoks = [64, 64, 9]
        out = torch.zeros(3, dtype=torch.int64, device="cuda:0")
        dn = dev_i32(ntoks)
        for layer in range(L):
            abi.check(abi.lib().dp_pool_checksum(pool.ptr, layer, ctypes.c_void_p(ds.data_ptr()),
                                                 ctypes.c_void_p(dn.data_ptr()), 3,
                                                 ctypes.c_void_p(out.data_ptr()), None))
            sync()
            got = [int(v) & refpy.MASK for v in out.cpu().tolist()]
            want = [refpy.layer_block_hash(refpy.geom(L, T, b), SEED, f, layer, n)
                    for f, n in zip(fbs, ntoks)]
            assert got == want
    finally:
        pool.close()
        st.close()


def test_wait_layer_watchdog(gpus):
    g = abi.geom(2, 64, 576)
    pool = abi.Pool(0, g, 2, 2)
    try:
        abi.wait_layer(pool, 0, 0, 0, timeout_ms=1000)  # already satisfied
        sync()
        assert abi.wait_status(pool) == abi.DP_OK
        abi.wait_layer(pool, 1, 2, 1, timeout_ms=50)  # never released -> watchdog
        sync()
        assert abi.wait_status(pool) == abi.DP_ETIMEOUT
        pool.reset_counters()
        sync()
        assert abi.wait_status(pool) == abi.DP_OK
    finally:
        pool.close()


def test_abi_rejects_bad_arguments(gpus):
    with pytest.raises(abi.DualPathError) as e:
        abi.Store(0, abi.geom(2, 64, 100), 1, SEED)  # b not a multiple of 16
    assert e.value.code == abi.DP_EINVAL
    g = abi.geom(2, 64, 576)
    st = abi.Store(0, g, 2, SEED)
    pool = abi.Pool(0, g, 4, 1)
    try:
        df, ds = dev_i64([0, 1]), dev_i32([0, 1])
        bad = abi.make_jobs([(df.data_ptr(), ds.data_ptr(), 64 * 3, 2, 0, 2, 0)])  # n_blk != ceil
        with pytest.raises(abi.DualPathError):
            abi.h2d_layer_gather(pool, st, bad, 1)
        ok = abi.make_jobs([(df.data_ptr(), ds.data_ptr(), 100, 2, 0, 2, 0)])
        with pytest.raises(abi.DualPathError):  # K2 needs a peer view, not the local pool
            abi.h2d_push_p2p_layer(pool, st, ok, 1)
        with pytest.raises(abi.DualPathError):
            abi.wait_layer(pool, 5, 0, 1)  # ticket out of range
    finally:
        pool.close()
        st.close()


@pytest.mark.parametrize("L,T,b", [(61, 64, 576), (4, 64, 4096), (64, 64, 4096)])
def test_k2_push_p2p_parity(de_dev, L, T, b):
    """The DE (device de_dev) reads its own host store and stores into the PE
    pool on device 0 (over NVLink when de_dev = 1); the PE's counters see the
    system-scope release.  (64, 64, 4096) is config 3's full Qwen2.5-32B shape."""
    rng = np.random.default_rng(11)
    g = abi.geom(L, T, b)
    st_de = abi.Store(de_dev, g, 10, SEED)
    pool = abi.Pool(0, g, 48, 40)
    view = pool.peer_view(de_dev)
    try:
        specs, keep, plain = random_jobs(rng, L, T, 36, 10, 48, 3, device=de_dev)
        abi.h2d_push_p2p_layer(view, st_de, abi.make_jobs(specs), len(specs))
        for t, (fbs, slots, ntok, l0, l1) in enumerate(plain):
            abi.wait_layer(pool, t, L, abi.layer_items(g, len(slots)) * (l1 - l0), timeout_ms=10000)
        sync()
        import torch
        torch.cuda.synchronize(de_dev)
        assert abi.wait_status(pool) == abi.DP_OK
        store_img = np.frombuffer(st_de.bytes(), dtype=np.uint8).copy()
        check_pool(pool, refpy.geom(L, T, b), plain, T, b, store_img, 48)
    finally:
        view.close()
        pool.close()
        st_de.close()


@pytest.mark.parametrize("L,T,b", [(61, 64, 576), (4, 64, 4096), (3, 16, 1024)])
@pytest.mark.parametrize("per_job", [False, True])
def test_k1_copy_engine_parity(gpus, L, T, b, per_job):
    """K1 on the copy engine (dp_h2d_layer_copy): strided 2D copies of block
    runs + fenced counter writes; same bytes and counters as the kernel."""
    rng = np.random.default_rng(21)
    g = abi.geom(L, T, b)
    n_fb, n_slots = 16, 64
    st = abi.Store(0, g, n_fb, SEED)
    pool = abi.Pool(0, g, n_slots, 12)
    try:
        plain, keep, specs, used = [], [], [], 0
        for t in range(12):
            nblk = int(rng.integers(0, 6))
            if used + nblk + 1 > n_slots:
                nblk = 0
            ntok = 0 if nblk == 0 else (nblk - 1) * T + int(rng.integers(1, T + 1))
            # contiguous runs with breaks: consecutive Full Blocks and slots, split once
            fb0 = int(rng.integers(0, n_fb - nblk)) if nblk else 0
            fbs = np.arange(fb0, fb0 + nblk, dtype=np.int64)
            slots = np.arange(used, used + nblk, dtype=np.int32)
            if nblk >= 3:
                slots[nblk // 2:] += 1  # a slot gap: two runs
            used += nblk + 1
            keep += [fbs, slots]
            specs.append((fbs.ctypes.data, slots.ctypes.data, ntok, nblk, 0, L, t))
            plain.append((fbs, slots, ntok, 0, L))
        (abi.h2d_layer_copy_job if per_job else abi.h2d_layer_copy)(pool, st, abi.make_jobs(specs), len(specs))
        for t, (fbs, slots, ntok, l0, l1) in enumerate(plain):
            items = abi.layer_items(g, len(slots))
            abi.wait_layer(pool, t, L, items * L, timeout_ms=5000)
            if len(slots):
                abi.wait_layer(pool, t, L - 1, items, timeout_ms=5000)
        sync()
        assert abi.wait_status(pool) == abi.DP_OK
        store_img = np.frombuffer(st.bytes(), dtype=np.uint8).copy()
        check_pool(pool, refpy.geom(L, T, b), plain, T, b, store_img, n_slots)
    finally:
        pool.close()
        st.close()


@pytest.mark.parametrize("L,T,b", [(61, 64, 576), (4, 64, 4096), (3, 16, 1024)])
@pytest.mark.parametrize("per_job", [False, True])
def test_k2_copy_engine_parity(de_dev, L, T, b, per_job):
    """K2 on the DE's copy engine (dp_h2d_push_copy): the DE's stream copies
    its host store into the PE pool through the peer view and writes the PE's
    counters; same bytes and counters as the kernel."""
    rng = np.random.default_rng(23)
    g = abi.geom(L, T, b)
    n_fb, n_slots = 16, 64
    st_de = abi.Store(de_dev, g, n_fb, SEED)
    pool = abi.Pool(0, g, n_slots, 12)
    view = pool.peer_view(de_dev)
    try:
        plain, keep, specs, used = [], [], [], 0
        for t in range(12):
            nblk = int(rng.integers(0, 6))
            if used + nblk + 1 > n_slots:
                nblk = 0
            ntok = 0 if nblk == 0 else (nblk - 1) * T + int(rng.integers(1, T + 1))
            fb0 = int(rng.integers(0, n_fb - nblk)) if nblk else 0
            fbs = np.arange(fb0, fb0 + nblk, dtype=np.int64)
            slots = np.arange(used, used + nblk, dtype=np.int32)
            if nblk >= 3:
                slots[nblk // 2:] += 1
            used += nblk + 1
            keep += [fbs, slots]
            specs.append((fbs.ctypes.data, slots.ctypes.data, ntok, nblk, 0, L, t))
            plain.append((fbs, slots, ntok, 0, L))
        import torch
        s_de = torch.cuda.Stream(device=de_dev)
        (abi.h2d_push_copy_job if per_job else abi.h2d_push_copy)(view, st_de, abi.make_jobs(specs), len(specs),
                                                                  s_de.cuda_stream)
        # the PE observes completion through its own counters only
        for t, (fbs, slots, ntok, l0, l1) in enumerate(plain):
            abi.wait_layer(pool, t, L, abi.layer_items(g, len(slots)) * L, timeout_ms=10000)
        sync()
        torch.cuda.synchronize(de_dev)
        assert abi.wait_status(pool) == abi.DP_OK
        store_img = np.frombuffer(st_de.bytes(), dtype=np.uint8).copy()
        check_pool(pool, refpy.geom(L, T, b), plain, T, b, store_img, n_slots)
        # a local pool is rejected (the copy targets a peer view)
        with pytest.raises(abi.DualPathError):
            abi.h2d_push_copy(pool, st_de, abi.make_jobs(specs), len(specs))
    finally:
        view.close()
        pool.close()
        st_de.close()


@pytest.mark.parametrize("placement", ["device", "none"])
def test_numa_store_and_storage_read(gpus, placement):
    """dp_store_create_on_node (NUMA-bound pinned staging) holds the oracle's
    content; dp_storage_read materialises other storage Full Blocks into
    staging positions (content keyed on the source block), paced by a NIC."""
    import time
    L, T, b = 4, 64, 576
    g = abi.geom(L, T, b)
    node = abi.NUMA_DEVICE if placement == "device" else abi.NUMA_NONE
    st = abi.Store(0, g, 8, SEED, numa_node=node)
    nic = abi.Nic(2e9)
    try:
        want_node = abi.device_numa_node(0)
        if placement == "device" and want_node >= 0:
            assert st.numa_node() == want_node
        gr = refpy.geom(L, T, b)
        assert np.array_equal(np.frombuffer(st.bytes(), dtype=np.uint8), refpy.fill_store(gr, SEED, 8))
        nic.start()
        t0 = time.monotonic()
        st.storage_read(2, 100, 3, nic)  # staging 2..4 <- storage Full Blocks 100..102
        fb = L * T * b
        assert time.monotonic() - t0 >= 3 * fb / 2e9 * 0.99
        img = np.frombuffer(st.bytes(), dtype=np.uint8)
        assert np.array_equal(img[2 * fb:5 * fb], refpy.fill_store(gr, SEED, 3, fb0=100))
        assert np.array_equal(img[:2 * fb], refpy.fill_store(gr, SEED, 2))   # untouched
        assert np.array_equal(img[5 * fb:], refpy.fill_store(gr, SEED, 3, fb0=5))
        with pytest.raises(abi.DualPathError):
            st.storage_read(7, 0, 2)  # past the staging
    finally:
        nic.close()
        st.close()


@pytest.mark.parametrize("L,T,b,ring", [(61, 64, 576, 40 << 20), (4, 64, 4096, 16 << 20), (3, 16, 1024, 0),
                                        (64, 64, 4096, 256 << 20)])
@pytest.mark.parametrize("side", ["pe", "de_same_gpu", "de_peer_gpu"])
@pytest.mark.parametrize("scatter", ["kernel", "ce"])
def test_staged_k1_k2_parity(gpus, L, T, b, ring, side, scatter):
    """Staged K1 / K2 (copy engine into an HBM ring + scatter kernel): same
    bytes and counters as the gather kernel, with runs broken by
    non-consecutive Full Blocks, partial last blocks, jobs larger than a ring
    segment (small rings) and more than one call reusing the ring."""
    import torch
    if side == "de_peer_gpu" and gpus < 2:
        pytest.skip("needs >= 2 GPUs")
    dev = {"pe": 0, "de_same_gpu": 0, "de_peer_gpu": 1}[side]
    rng = np.random.default_rng(L + b)
    g = abi.geom(L, T, b)
    n_fb, n_slots = 40, 192
    st = abi.Store(dev, g, n_fb, SEED)
    pool = abi.Pool(0, g, n_slots, 16)
    view = pool.peer_view(dev) if side != "pe" else None
    stager = abi.Stager(dev, g, ring)
    ce = scatter == "ce"
    if ce:
        stager.set_mode(abi.SCATTER_CE)
    s = torch.cuda.Stream(device=dev)
    try:
        plain, keep, specs, used = [], [], [], 0
        for t in range(16):
            nblk = int(rng.integers(0, 9))
            if used + nblk > n_slots:
                nblk = 0
            ntok = 0 if nblk == 0 else (nblk - 1) * T + int(rng.integers(1, T + 1))
            fb0 = int(rng.integers(0, n_fb - nblk)) if nblk else 0
            fbs = np.arange(fb0, fb0 + nblk, dtype=np.int64)
            if nblk >= 4:
                fbs[nblk // 2:] = rng.integers(0, n_fb, nblk - nblk // 2)  # break the run
            # runs of consecutive slots (the copy-engine scatter's 2D copies), broken once
            slots = (used + np.arange(nblk)).astype(np.int32)
            if nblk >= 4:
                slots[nblk // 2:] += 1
            used += nblk + 2
            ds = dev_i32(slots if nblk else [0], dev)
            keep += [fbs, ds, slots]
            specs.append((fbs.ctypes.data, slots.ctypes.data if ce else ds.data_ptr(), ntok, nblk, 0, L, t))
            plain.append((fbs, slots, ntok, 0, L))
        for half in (specs[:7], specs[7:]):  # two calls: the ring is reused across calls
            jobs = abi.make_jobs(half)
            if side == "pe":
                abi.h2d_layer_staged(pool, st, stager, jobs, len(half), s.cuda_stream)
            else:
                abi.h2d_push_staged(view, st, stager, jobs, len(half), s.cuda_stream)
        s.synchronize()
        for t, (fbs, slots, ntok, l0, l1) in enumerate(plain):
            items = abi.layer_items(g, len(slots))
            abi.wait_layer(pool, t, L, items * L, timeout_ms=10000)
            if len(slots):
                abi.wait_layer(pool, t, L - 1, items, timeout_ms=10000)
        sync()
        assert abi.wait_status(pool) == abi.DP_OK
        assert stager.launches() >= (0 if ce else 2)
        store_img = np.frombuffer(st.bytes(), dtype=np.uint8).copy()
        check_pool(pool, refpy.geom(L, T, b), plain, T, b, store_img, n_slots)
        bad = abi.make_jobs([(specs[1][0], specs[1][1], specs[1][2], specs[1][3], 1, L, 1)])  # layer subrange
        with pytest.raises(abi.DualPathError):
            abi.h2d_layer_staged(pool, st, stager, bad, 1) if side == "pe" else \
                abi.h2d_push_staged(view, st, stager, bad, 1)
    finally:
        stager.close()
        if view:
            view.close()
        pool.close()
        st.close()
