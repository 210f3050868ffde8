#!/usr/bin/env python
"""Small, stream-ordered invocations of every kernel of libdualpath.so for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck): K1 gather,
K2 push (a same-GPU pool view), staged K1 (copy engine + scatter), the dual
gather, K3 handoff (SM kernel and copy engines + kv_handoff_side), the
decode stand-in + K4 persistence (SM kernel and staged), K5 attend, the
checksum and the store fill.  No cross-kernel spin waits (the
sanitizers serialise kernels), every result checked against the oracle."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import refpy  # noqa: E402
from paper_2602_21548_b200 import abi  # noqa: E402

SEED = 9


def dev(x, dtype):
    return torch.tensor(np.asarray(x, dtype=dtype), device="cuda:0")


def main():
    L, T, b = 3, 64, 576
    g, gr = abi.geom(L, T, b), refpy.geom(L, T, b)
    st = abi.Store(0, g, 12, SEED)
    pe = abi.Pool(0, g, 16, 4)
    de = abi.Pool(0, g, 16, 4)
    pe_view, de_view = pe.peer_view(0), de.peer_view(0)
    stager = abi.Stager(0, g, 4 * L * T * b * 4)
    try:
        C, A = 64 * 2 + 17, 70
        P = C + A
        nh, npb = -(-C // T), -(-P // T)
        fbs = np.arange(2, 2 + npb, dtype=np.int64)
        ps, ds = np.arange(npb, dtype=np.int32), np.arange(5, 5 + npb, dtype=np.int32)
        t = [dev(fbs, np.int64), dev(ps, np.int32), dev(ds, np.int32)]
        # K1 (ticket 0) then K3 on the PE path (stream-ordered, push_hit)
        abi.h2d_layer_gather(pe, st, abi.make_jobs([(t[0].data_ptr(), t[1].data_ptr(), C, nh, 0, L, 0)]), 1)
        hj = (abi.HandoffJob * 1)()
        hj[0] = abi.HandoffJob(t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), C, P, npb, 1, -1, 0, 0, 2)
        abi.prefill_handoff(pe, de_view, hj, 1, SEED)
        # the same handoff on the copy engines into a second decode pool
        # (host block tables; kv_handoff_side + 2D copies)
        de2 = abi.Pool(0, g, 16, 4)
        de2_view = de2.peer_view(0)
        hc = (abi.HandoffJob * 1)()
        hc[0] = abi.HandoffJob(fbs.ctypes.data, ps.ctypes.data, ds.ctypes.data, C, P, npb, 1, -1, 0, 0, -1)
        abi.prefill_handoff_copy(pe, de2_view, hc, 1, SEED)
        torch.cuda.synchronize()
        for k in range(npb):
            n = min(T, P - k * T)
            for layer in range(L):
                want = refpy.layer_block(gr, SEED, int(fbs[k]), layer, n).tobytes()
                assert pe.copy_out(layer, int(ps[k]), n * b) == want
                assert de.copy_out(layer, int(ds[k]), n * b) == want
                assert de2.copy_out(layer, int(ds[k]), n * b) == want
        de2_view.close()
        de2.close()
        # K2 into the PE pool (view on the same GPU), ticket 1; the dual gather, ticket 3
        ps2 = np.arange(8, 8 + nh, dtype=np.int32)
        t2 = dev(ps2, np.int32)
        abi.h2d_push_p2p_layer(pe_view, st, abi.make_jobs([(t[0].data_ptr(), t2.data_ptr(), C, nh, 0, L, 1)]), 1)
        dj = (abi.DualJob * 1)()
        dj[0].pe = abi.Job(t[0].data_ptr(), t[1].data_ptr(), C, nh, 0, L, 3)
        dj[0].de_slot = t[2].data_ptr()
        dj[0].de_ticket = 1
        abi.push_p2p_dual(pe_view, de, st, dj, 1)
        # staged K1 (host src_fb), ticket 2
        ps3 = np.arange(12, 12 + nh, dtype=np.int32)
        t3 = dev(ps3, np.int32)
        abi.h2d_layer_staged(pe, st, stager, abi.make_jobs([(fbs.ctypes.data, t3.data_ptr(), C, nh, 0, L, 2)]), 1)
        torch.cuda.synchronize()
        for slots in (ps2, ps3):
            for k in range(nh):
                n = min(T, C - k * T)
                for layer in range(L):
                    assert pe.copy_out(layer, int(slots[k]), n * b) == \
                        refpy.layer_block(gr, SEED, int(fbs[k]), layer, n).tobytes()
        # decode stand-in + K4 persistence
        target = abi.Store(0, g, 12, SEED + 1)
        sp = (abi.SpanJob * 1)()
        sp[0] = abi.SpanJob(t[2].data_ptr(), t[0].data_ptr(), 0, P, npb * T, npb, 0)
        abi.decode_fill(de, sp, 1, SEED)
        abi.persist_d2h(de, target, sp, 1)
        # staged K4 (gather into an HBM ring + copy engine): the same bytes
        target2 = abi.Store(0, g, 12, SEED + 1)
        pstager = abi.Stager(0, g, 4 * L * T * b * 4)
        sph = (abi.SpanJob * 1)()
        sph[0] = abi.SpanJob(t[2].data_ptr(), fbs.ctypes.data, 0, P, npb * T, npb, 0)
        abi.persist_staged(de, target2, pstager, sph, 1)
        torch.cuda.synchronize()
        assert target2.bytes() == target.bytes()
        pstager.close()
        target2.close()
        img = np.frombuffer(target.bytes(), dtype=np.uint8)
        fbb = L * T * b
        k = npb - 1
        a0 = P - k * T
        for layer in range(L):
            off = int(fbs[k]) * fbb + layer * T * b
            assert np.array_equal(img[off + a0 * b:off + T * b],
                                  refpy.layer_block(gr, SEED, int(fbs[k]), layer, T)[a0 * b:])
        target.close()
        # K5 over the PE pool's first request
        digest = torch.zeros(L, dtype=torch.int64, device="cuda:0")
        items = (abi.AttendItem * 1)()
        items[0] = abi.AttendItem(t[1].data_ptr(), C, 0, A, digest.data_ptr(), 7, 0)
        for layer in range(L):
            abi.prefill_attend(pe, layer, items, 1, SEED)
        torch.cuda.synchronize()
        for layer in range(L):
            want = refpy.attend_digest(gr, SEED, [int(f) for f in fbs[:nh]], C, 7, layer, 0, A)
            assert int(digest[layer].item()) & (2 ** 64 - 1) == want
        # checksum
        out = torch.zeros(nh, dtype=torch.int64, device="cuda:0")
        ntok = dev([min(T, C - k * T) for k in range(nh)], np.int32)
        abi.lib().dp_pool_checksum(pe.ptr, 0, t[1].data_ptr(), ntok.data_ptr(), nh, out.data_ptr(), None)
        torch.cuda.synchronize()
        for k in range(nh):
            assert int(out[k].item()) & (2 ** 64 - 1) == refpy.layer_block_hash(gr, SEED, int(fbs[k]), 0,
                                                                                 min(T, C - k * T))
        print("kernels_small ok")
    finally:
        stager.close()
        de_view.close()
        pe_view.close()
        de.close()
        pe.close()
        st.close()


if __name__ == "__main__":
    main()
