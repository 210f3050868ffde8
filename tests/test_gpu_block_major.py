"""Block-major PE pools (DP_POOL_BLOCK_MAJOR: [slots][L][T][b], a whole Full
Block per slot): the loading path's kernels and copy-engine paths land the
same bytes as into a layer-major pool -- checked against the oracle block by
block and layer by layer -- and a run of storage Full Blocks into
consecutive slots is one contiguous copy-engine copy (no ring, no SM work).
The handoff and persistence kernels refuse block-major pools."""

import numpy as np
import pytest

from oracle import refpy
from paper_2602_21548_b200 import abi

pytestmark = pytest.mark.gpu
SEED = 9


def dev(x, device, dtype):
    import torch
    return torch.tensor(np.asarray(x, dtype=dtype), device=f"cuda:{device}")


def sync_all():
    import torch
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)


def check_blocks(pool, gr, fbs, slots, n_tokens, T, b, L):
    for k, (f, s) in enumerate(zip(fbs, slots)):
        n = min(T, n_tokens - k * T)
        for layer in range(L):
            assert pool.copy_out(layer, int(s), n * b) == refpy.layer_block(gr, SEED, int(f), layer, n).tobytes(), \
                (k, layer)


def job(C, T, L, fb_arr, slot_arr, ticket, keep):
    """One all-layer job; fb_arr / slot_arr are numpy (host) or torch (device) arrays."""
    keep += [fb_arr, slot_arr]
    ptr = lambda a: a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()  # noqa: E731
    return abi.make_jobs([(ptr(fb_arr), ptr(slot_arr), C, -(-C // T), 0, L, ticket)])


@pytest.mark.parametrize("L,T,b", [(4, 64, 576), (61, 64, 576), (3, 64, 4096)])
@pytest.mark.parametrize("mode", ["gather", "copy_job", "staged", "staged_ce"])
def test_k1_into_block_major(gpus, L, T, b, mode):
    """K1 (SM gather, copy engine per job, staged with the scatter kernel or
    the copy-engine scatter) into a block-major pool: every Layer Block equals
    the oracle's; the landed counters reach their targets."""
    g = abi.geom(L, T, b)
    C = 64 * 7 + 21
    nb = -(-C // T)
    st = abi.Store(0, g, 24, SEED)
    pool = abi.Pool(0, g, 16, 2, layout=abi.POOL_BLOCK_MAJOR)
    stager = abi.Stager(0, g, 2 * L * T * b * 4) if mode.startswith("staged") else None
    try:
        assert pool.layout() == abi.POOL_BLOCK_MAJOR
        # two runs (consecutive storage blocks into consecutive slots), then a lone block
        fbs = [3, 4, 5, 6, 10, 11, 15, 2][:nb]
        slots = [1, 2, 3, 4, 9, 10, 0, 14][:nb]
        host_fb = mode != "gather"                      # copy-engine paths plan on the host
        host_slot = mode in ("copy_job", "staged_ce")   # the staged kernel scatter reads device slots
        keep = []
        jobs = job(C, T, L, np.asarray(fbs, dtype=np.int64) if host_fb else dev(fbs, 0, np.int64),
                   np.asarray(slots, dtype=np.int32) if host_slot else dev(slots, 0, np.int32), 0, keep)
        if mode == "gather":
            abi.h2d_layer_gather(pool, st, jobs, 1)
        elif mode == "copy_job":
            abi.lib().dp_h2d_layer_copy_job(pool.ptr, st.ptr, jobs, 1, None)
        else:
            stager.set_mode(abi.SCATTER_CE if mode == "staged_ce" else abi.SCATTER_KERNEL)
            abi.h2d_layer_staged(pool, st, stager, jobs, 1)
        sync_all()
        check_blocks(pool, refpy.geom(L, T, b), fbs, slots, C, T, b, L)
        items = abi.layer_items(g, nb)
        abi.wait_layer(pool, 0, L, items * L, timeout_ms=2000)
        abi.wait_layer(pool, 0, L - 1, items, timeout_ms=2000)
        sync_all()
        assert abi.wait_status(pool) == abi.DP_OK
    finally:
        if stager:
            stager.close()
        pool.close()
        st.close()


@pytest.mark.parametrize("mode", ["push", "copy_job"])
def test_k2_into_block_major_view(de_dev, mode):
    """K2 from the DE's store into a block-major PE pool through its view
    (NVLink peer stores, or the DE's copy engine: whole Full-Block runs)."""
    L, T, b = 8, 64, 576
    g = abi.geom(L, T, b)
    C = 64 * 5 + 3
    nb = -(-C // T)
    st = abi.Store(de_dev, g, 24, SEED)
    pool = abi.Pool(0, g, 16, 1, layout=abi.POOL_BLOCK_MAJOR)
    view = pool.peer_view(de_dev)
    try:
        assert view.layout() == abi.POOL_BLOCK_MAJOR
        fbs, slots = [7, 8, 9, 1, 2, 3], [5, 6, 7, 12, 13, 14]
        keep = []
        host = mode == "copy_job"
        jobs = job(C, T, L, np.asarray(fbs[:nb], dtype=np.int64) if host else dev(fbs[:nb], de_dev, np.int64),
                   np.asarray(slots[:nb], dtype=np.int32) if host else dev(slots[:nb], de_dev, np.int32), 0, keep)
        if mode == "push":
            abi.h2d_push_p2p_layer(view, st, jobs, 1)
        else:
            abi.lib().dp_h2d_push_copy_job(view.ptr, st.ptr, jobs, 1, None)
        sync_all()
        check_blocks(pool, refpy.geom(L, T, b), fbs[:nb], slots[:nb], C, T, b, L)
        abi.wait_layer(pool, 0, L, abi.layer_items(g, nb) * L, timeout_ms=2000)
        sync_all()
        assert abi.wait_status(pool) == abi.DP_OK
    finally:
        view.close()
        pool.close()
        st.close()


def test_attend_and_checksum_on_block_major(gpus):
    """K5 reads its keys and the checksum its blocks through the pool's slot
    stride: the same digests and hashes as the oracle's."""
    import torch
    L, T, b = 3, 64, 576
    g, gr = abi.geom(L, T, b), refpy.geom(L, T, b)
    C, A = 64 * 4 + 9, 100
    nb = -(-C // T)
    st = abi.Store(0, g, 12, SEED)
    pool = abi.Pool(0, g, 8, 1, layout=abi.POOL_BLOCK_MAJOR)
    try:
        fbs, slots = [4, 2, 9, 1, 6][:nb], [7, 0, 3, 5, 1][:nb]
        keep = []
        abi.h2d_layer_gather(pool, st, job(C, T, L, dev(fbs, 0, np.int64), dev(slots, 0, np.int32), 0, keep), 1)
        digest = torch.zeros(L, dtype=torch.int64, device="cuda:0")
        items = (abi.AttendItem * 1)()
        items[0] = abi.AttendItem(keep[1].data_ptr(), C, 0, A, digest.data_ptr(), 11, 0)
        for layer in range(L):
            abi.prefill_attend(pool, layer, items, 1, SEED)
        out = torch.zeros(nb, dtype=torch.int64, device="cuda:0")
        ntok = dev([min(T, C - k * T) for k in range(nb)], 0, np.int32)
        abi.lib().dp_pool_checksum(pool.ptr, L - 1, keep[1].data_ptr(), ntok.data_ptr(), nb, out.data_ptr(), None)
        sync_all()
        for layer in range(L):
            assert int(digest[layer].item()) & (2 ** 64 - 1) == refpy.attend_digest(gr, SEED, fbs, C, 11, layer, 0, A)
        for k in range(nb):
            assert int(out[k].item()) & (2 ** 64 - 1) == refpy.layer_block_hash(gr, SEED, fbs[k], L - 1,
                                                                                 min(T, C - k * T))
    finally:
        pool.close()
        st.close()


def test_handoff_refuses_block_major(gpus):
    g = abi.geom(2, 64, 576)
    pe = abi.Pool(0, g, 4, 1, layout=abi.POOL_BLOCK_MAJOR)
    de = abi.Pool(0, g, 4, 1)
    view = de.peer_view(0)
    try:
        fbs, sl = np.array([0], dtype=np.int64), np.array([0], dtype=np.int32)
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(fbs.ctypes.data, sl.ctypes.data, sl.ctypes.data, 10, 20, 1, 1, -1, 0, -1, -1)
        with pytest.raises(abi.DualPathError, match="layer-major"):
            abi.prefill_handoff_copy(pe, view, hj, 1, SEED)
    finally:
        view.close()
        de.close()
        pe.close()
