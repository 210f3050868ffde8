"""The oracles are pinned before they are trusted (CPU only).

* oracle/kvref.c (the CPU restatement of the bytes) against published
  splitmix64 answers, an independent pure-Python restatement, and the
  committed known-answer fixture tests/golden/kvref_kat.json;
* the compiled reference (oracle/_ref) against the reference's own golden
  trace proj/data/trace_64k.tsv (md5 f066ac89...), and the
  product's synthesize() against the same md5.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2602_21548_b200 as dp
from oracle import refpy

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TRACE_64K_MD5 = "f066ac893c54f85c265bc48a41e2dec0"  # /root/reference/proj/data/trace_64k.tsv
MASK = (1 << 64) - 1


def py_splitmix64(x):
    z = (x + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def py_word(seed, fb, w):
    return py_splitmix64(((fb << 32) | w) ^ ((seed * 0xD1B54A32D192ED03) & MASK))


def test_splitmix64_published_answer():
    # first output of the splitmix64 generator seeded with 0 (Vigna)
    assert refpy.kvref().kvref_splitmix64(0) == 0xE220A8397B1DCDAF
    assert py_splitmix64(0) == 0xE220A8397B1DCDAF


def test_kvref_word_matches_python_restatement():
    rng = np.random.default_rng(1)
    for _ in range(500):
        seed = int(rng.integers(0, 1 << 62))
        fb = int(rng.integers(0, 1 << 20))
        w = int(rng.integers(0, 1 << 31))
        assert refpy.kvref().kvref_word(seed, fb, w) == py_word(seed, fb, w)


def test_kvref_known_answers_fixture():
    kat = json.load(open(os.path.join(GOLDEN, "kvref_kat.json")))
    for x, v in kat["splitmix64"].items():
        assert refpy.kvref().kvref_splitmix64(int(x)) == v
    for seed, fb, w, v in kat["word"]:
        assert refpy.kvref().kvref_word(seed, fb, w) == v == py_word(seed, fb, w)
    g = refpy.geom(61, 64, 576)
    for seed, fb, layer, ntok, v in kat["layer_block_hash"]:
        assert refpy.layer_block_hash(g, seed, fb, layer, ntok) == v


def test_store_layout_full_block_is_layer_blocks_concatenated():
    # Full Block [L][T][b] = L Layer Blocks back to back
    L, T, b = 5, 16, 64
    g = refpy.geom(L, T, b)
    store = refpy.fill_store(g, 9, 3)
    fb_bytes = L * T * b
    for fb in range(3):
        for layer in range(L):
            lb = refpy.layer_block(g, 9, fb, layer, T)
            off = fb * fb_bytes + layer * T * b
            assert np.array_equal(store[off:off + T * b], lb)
    words = store.view(np.uint64)
    for i in (0, 17, len(words) - 1):
        fb, w = divmod(i, fb_bytes // 8)
        assert int(words[i]) == py_word(9, fb, w)


def test_layer_block_hash_is_hash_of_bytes():
    g = refpy.geom(4, 64, 576)
    for fb, layer, ntok in ((0, 0, 64), (3, 2, 1), (9, 3, 40)):
        raw = refpy.layer_block(g, 9, fb, layer, ntok)
        assert refpy.hash_bytes(raw) == refpy.layer_block_hash(g, 9, fb, layer, ntok)
        words = raw.view(np.uint64)
        h = 0
        for i, x in enumerate(words.tolist()):
            h = (h + py_splitmix64((x + (i + 1) * 0x9E3779B97F4A7C15) & MASK)) & MASK
        assert h == refpy.hash_bytes(raw)


def test_kvref_gather_matches_numpy_restatement():
    rng = np.random.default_rng(3)
    L, T, b = 3, 16, 64
    g = refpy.geom(L, T, b)
    n_fb, n_slots = 6, 20
    store = refpy.fill_store(g, 5, n_fb)
    perm = rng.permutation(n_slots)
    specs, used = [], 0
    for _ in range(5):
        nblk = int(rng.integers(1, 4))
        ntok = (nblk - 1) * T + int(rng.integers(1, T + 1))
        fbs = rng.integers(0, n_fb, nblk).tolist()
        slots = perm[used:used + nblk].tolist()
        used += nblk
        specs.append((fbs, slots, ntok, 0, L))
    pool = refpy.gather(g, store, n_fb, specs, n_slots)
    want = np.zeros_like(pool)
    lb, fbb = T * b, L * T * b
    for fbs, slots, ntok, l0, l1 in specs:
        for k, (f, s) in enumerate(zip(fbs, slots)):
            n = min(T, ntok - k * T) * b
            for layer in range(l0, l1):
                dst = (layer * n_slots + s) * lb
                src = f * fbb + layer * lb
                want[dst:dst + n] = store[src:src + n]
    assert np.array_equal(pool, want)


def test_kvref_gather_rejects_out_of_range():
    g = refpy.geom(2, 16, 64)
    store = refpy.fill_store(g, 5, 2)
    with pytest.raises(ValueError):
        refpy.gather(g, store, 2, [([5], [0], 16, 0, 2)], 4)


@pytest.mark.skipif(not refpy.ref_available(), reason="oracle/_ref not built")
def test_reference_regenerates_its_golden_trace(tmp_path):
    p = str(tmp_path / "t.tsv")
    assert refpy.ref_synthesize(p, max_len=65536, count=500, seed=9) == 500
    assert hashlib.md5(open(p, "rb").read()).hexdigest() == TRACE_64K_MD5


def test_product_synthesize_regenerates_golden_trace(tmp_path):
    # the product's generator is draw-for-draw the reference's
    # (proj/src/workload.cpp:96-130): same bytes as proj/data/trace_64k.tsv
    p = str(tmp_path / "t.tsv")
    dp.save_trace(p, dp.synthesize(max_len=65536, count=500, seed=9))
    assert hashlib.md5(open(p, "rb").read()).hexdigest() == TRACE_64K_MD5
    back = dp.load_trace(p)
    mean_total = sum(t.total_tokens() for t in back) / len(back)
    # proj/tests/python/test_smoke.py:84-89
    assert abs(mean_total - 55958) / 55958 < 0.10


@pytest.mark.skipif(not refpy.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scales", [(1.0, 1.0, 65536), (2.0, 0.5, 200000), (0.37, 3.3, 9000),
                                    (1.5, 1.5, 1)])
def test_derive_variant_matches_reference(tmp_path, scales):
    # proj/src/workload.cpp:131-162: half-up rounding, gen >= 1, cap clamp
    a, g, cap = scales
    src = str(tmp_path / "src.tsv")
    dp.save_trace(src, dp.synthesize(max_len=65536, count=40, seed=3))
    want = str(tmp_path / "ref.tsv")
    refpy.ref_derive_variant(src, want, a, g, cap)
    got = str(tmp_path / "got.tsv")
    dp.save_trace(got, dp.derive_variant(dp.load_trace(src), a, g, cap))
    assert open(got).read() == open(want).read()


@pytest.mark.skipif(not refpy.ref_available(), reason="oracle/_ref not built")
def test_extend_and_poisson_match_reference(tmp_path):
    src = str(tmp_path / "src.tsv")
    dp.save_trace(src, dp.synthesize(max_len=20000, count=8, seed=5))
    want = str(tmp_path / "ref.tsv")
    refpy.ref_extend_trace(src, want, 77)
    got = str(tmp_path / "got.tsv")
    dp.save_trace(got, [dp.extend_with_synthetic_round(t, 77) for t in dp.load_trace(src)])
    assert open(got).read() == open(want).read()
    for rate, horizon, seed in [(0.1, 500.0, 1), (3.0, 100.0, 42)]:
        assert dp.poisson_arrivals(rate, horizon, seed) == refpy.ref_poisson(rate, horizon, seed)
    with pytest.raises(ValueError):
        dp.derive_variant(dp.load_trace(src), 0.0, 1.0, 100)


@pytest.mark.parametrize("L,T,b", [(2, 16, 64), (3, 64, 576), (1, 8, 208)])
def test_attend_digest_column_sum_form_is_exact(L, T, b):
    """The oracle of K5 computes sum_q sum_t dot(Q, K) as an inner product of
    column sums; pin it against the literal double sum on small cases,
    including partial blocks and a chunk starting mid-append."""
    g = refpy.geom(L, T, b)
    fbs = [5, 2, 9, 1]
    for C, q0, bsz in [(1, 0, 1), (T + 3, 2, 5), (3 * T, 0, 17), (4 * T - 1, 11, 3)]:
        for layer in range(L):
            assert refpy.attend_digest(g, 9, fbs, C, 123, layer, q0, bsz) == \
                refpy.attend_digest_bruteforce(g, 9, fbs, C, 123, layer, q0, bsz)
