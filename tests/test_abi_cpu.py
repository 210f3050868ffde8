"""The C ABI library loads and exports every entry point include/dualpath/kv_abi.h
declares; argument validation that needs no GPU (CPU only)."""

import ctypes

import pytest

from paper_2602_21548_b200 import abi


def test_header_declares_the_path_entry_points():
    syms = abi.declared_symbols()
    for need in ("dp_h2d_layer_gather", "dp_h2d_push_p2p_layer", "dp_wait_layer", "dp_store_create",
                 "dp_pool_create", "dp_pool_export", "dp_pool_import", "dp_pool_checksum",
                 "dp_last_error"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(abi.LIB_PATH)
    missing = [s for s in abi.declared_symbols() if not hasattr(lib, s)]
    assert missing == []


def test_abi_version_and_geometry_checks():
    L = abi.lib()
    assert L.dp_abi_version() == 1
    assert L.dp_geom_check(ctypes.byref(abi.geom(61, 64, 576))) == abi.DP_OK
    assert L.dp_geom_check(ctypes.byref(abi.geom(64, 64, 4096))) == abi.DP_OK
    for bad in (abi.geom(0, 64, 576), abi.geom(4, 0, 576), abi.geom(4, 64, 100), abi.geom(4, 64, 0)):
        assert L.dp_geom_check(ctypes.byref(bad)) == abi.DP_EINVAL
        assert L.dp_last_error()  # thread-local message set
    assert L.dp_geom_check(None) == abi.DP_EINVAL


def test_layer_items():
    # 64 KiB chunks: one item per DS-V3 Layer Block, four per Qwen Layer Block
    assert abi.layer_items(abi.geom(61, 64, 576), 10) == 10
    assert abi.layer_items(abi.geom(64, 64, 4096), 10) == 40
    with pytest.raises(abi.DualPathError):
        abi.layer_items(abi.geom(61, 64, 576), -1)


def test_null_arguments_fail_cleanly():
    L = abi.lib()
    assert L.dp_h2d_layer_gather(None, None, None, 0, None) == abi.DP_EINVAL
    assert L.dp_h2d_push_p2p_layer(None, None, None, 0, None) == abi.DP_EINVAL
    assert L.dp_wait_layer(None, 0, 0, 0, 1, None) == abi.DP_EINVAL
    assert L.dp_pool_checksum(None, 0, None, None, 0, None, None) == abi.DP_EINVAL
    assert L.dp_store_info(None, None, None, None) == abi.DP_EINVAL
    assert L.dp_store_destroy(None) == abi.DP_OK
    assert L.dp_pool_destroy(None) == abi.DP_OK
    out = ctypes.c_void_p()
    assert L.dp_pool_create(0, ctypes.byref(abi.geom(4, 64, 100)), 4, 1, ctypes.byref(out)) == abi.DP_EINVAL
    assert out.value is None


def test_pool_handle_layout_is_128_bytes():
    assert ctypes.sizeof(abi.PoolHandle) == 128
    assert ctypes.sizeof(abi.Job) == 40
    assert ctypes.sizeof(abi.Geom) == 16


def test_nic_is_a_fifo_token_bucket():
    """dp_nic (StorageRead's rate cap, desim.cpp:603-606): FIFO at the rate,
    not_before honoured, thread-safe; rate 0 = unlimited."""
    import threading
    import time
    nic = abi.Nic(1e9)  # 1 GB/s
    try:
        nic.start()
        t0 = time.monotonic()
        b, e = nic.read(50_000_000)
        assert 0.0 <= b < 0.005 and e == pytest.approx(b + 0.05)
        b2, e2 = nic.read(20_000_000, not_before_s=0.1)  # idle gap until 0.1 s
        assert round(b2, 6) == 0.1 and round(e2, 6) == 0.12
        assert time.monotonic() - t0 >= 0.119
        time.sleep(0.05)  # the NIC sits idle: the next read starts now, not at 0.12
        b3, e3 = nic.read(10_000_000)
        assert b3 >= 0.169 and e3 == pytest.approx(b3 + 0.01)
        spans = []
        ths = [threading.Thread(target=lambda: spans.append(nic.read(10_000_000))) for _ in range(4)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        spans.sort()
        starts = [s for s, _ in spans]
        assert all(abs((b - a) - 0.01) < 1e-9 for a, b in zip(starts, starts[1:]))  # served back to back
    finally:
        nic.close()
    free = abi.Nic(0.0)
    free.start()
    b, e = free.read(1 << 40)
    assert b == e and b < 0.01  # unlimited: no time
    free.close()
    with pytest.raises(abi.DualPathError):
        abi.Nic(-1.0)


def test_new_entry_points_reject_bad_arguments():
    L = abi.lib()
    assert L.dp_storage_read(None, 0, 0, 1, None) == abi.DP_EINVAL
    assert L.dp_store_numa_node(None, None) == abi.DP_EINVAL
    assert L.dp_wait_clear(None) == abi.DP_EINVAL
    assert L.dp_nic_read(None, 1, 0.0, None, None) == abi.DP_EINVAL
    assert L.dp_device_numa_node(0, None) == abi.DP_EINVAL
