"""S-digit cache of the int8 product (k2i_product.cu, sdig_item_bytes): the
solve's first product pass stores every (row block, k-step) item's digit
planes of D o D, the later passes stream them instead of D. The digits are
the same bytes the converters would produce, so a solve with the cache is
BIT-identical to one without it when every pass runs the same plan, and
equal to the fp64 summation-order level when the streaming passes run on
clusters (another stream-K split) — on every kernel variant the cache
feeds: the single-CTA NB = 32 / 64 groups and the CTA pair storing it, the
streaming clusters of 2, 3 and 4 CTAs (multicast items, one 32-column group
per CTA), the Hamming 3-byte slices, f32 D, two column groups in one storing
pass (the first group stores, the second streams), ragged n and the int32
chunk edge.
The oracle comparison (ref src/rsvd.cpp:81-145, mds.cpp:81-124) runs on the
cached path of each case as well.
"""
import os

import numpy as np
import pytest

from helpers import coords_match_up_to_sign

pytestmark = pytest.mark.gpu


def _solve(ds, g, k, p, q, seed, cache):
    ds.set_product_path(2)
    ds.set_sdig_cache(cache)
    try:
        e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
        st = ds.stats_get()
    finally:
        ds.set_product_path(0)
        ds.set_sdig_cache(1)
    return e, st


def _gram(ds, d, cache):
    """gram() with the cache policy `cache`: 0 keeps K1 from writing the
    digit planes (the solves then store them in their first pass)."""
    ds.set_sdig_cache(cache)
    try:
        return ds.gram(d)
    finally:
        ds.set_sdig_cache(1)


CASES = [
    # (kind, n, rank, over, expect pair, sdigits)
    ("f64", 4133, 20, 10, 0, 7),   # NB = 32, ragged n
    ("f64", 4500, 40, 10, 0, 7),   # NB = 64 hybrid (digits 5-7 via shared memory)
    ("f64", 4250, 50, 20, 1, 7),   # w = 70: CTA pair, multicast item halves
    ("f32", 4200, 100, 20, 0, 7),  # w = 120 on f32 D: two 64-column groups
    ("ham", 4300, 30, 20, 0, 3),   # Hamming slices, NB = 64
    ("ham", 4400, 10, 10, 0, 3),   # Hamming slices, NB = 32
    ("ham", 4100, 50, 20, 1, 3),   # Hamming slices on the CTA pair
]


def _matrix(ds, kind, n, seed):
    if kind == "ham":
        return ds.matrix_hamming(ds.synth_reads(n, 400, 20, 0.05, seed))
    return ds.matrix_euclidean(ds.synth_points(2, n, seed), store_f32=(kind == "f32"))


@pytest.mark.parametrize("kind,n,rank,over,pair,sdigits", CASES)
def test_sdig_cache_bit_identical(ds, oracle, kind, n, rank, over, pair, sdigits):
    d = _matrix(ds, kind, n, n % 11)
    g = _gram(ds, d, 0)  # the first product pass stores the cache
    off, st0 = _solve(ds, g, rank, over, 2, 3, 0)
    assert st0.last_product_kernel == 1 and st0.last_product_sdig == 0
    on, st1 = _solve(ds, g, rank, over, 2, 3, 2)
    assert st1.last_product_kernel == 1 and st1.last_product_sdig == 1
    assert (st1.last_product_pair, st1.last_product_sdigits) == (pair, sdigits)
    # the streaming passes run on the storing pass's plan (the pair for
    # 64 < WP <= 96), or with DSB_K2I_STREAM_CL=1 on clusters of
    # ceil(WP / 32) CTAs sharing each digit item (one 32-column group per CTA)
    wp = (rank + over + 7) // 8 * 8
    want_cl = min(4, (wp + 31) // 32) if os.environ.get("DSB_K2I_STREAM_CL") == "1" else \
        (2 if pair else 1)
    assert st1.last_product_stream_cl == want_cl
    if os.environ.get("DSB_K2I_STREAM_CL") != "1":
        # same plan for every pass: bit-identical
        assert np.array_equal(on.eigenvalues, off.eigenvalues)
        assert np.array_equal(on.coords, off.coords)
    else:
        # the streaming clusters split the rows' column range differently,
        # so the fp64 partial slots are summed in another order
        np.testing.assert_allclose(on.eigenvalues, off.eigenvalues, rtol=1e-10,
                                   atol=1e-13 * abs(off.eigenvalues[0]))
        assert coords_match_up_to_sign(on.coords, off.coords) < 1e-9 * np.sqrt(off.eigenvalues[0])
    # a second cached solve (graph replay) stores and streams again
    again, _ = _solve(ds, g, rank, over, 2, 3, 2)
    assert np.array_equal(again.coords, on.coords)
    if kind != "f32":
        dm = d.to_numpy()
        _, rm, grand = oracle.gram_stats(dm)
        want = oracle.embed(rank, over, 2, 3, d=dm, row_mean=rm, grand=grand)
        top = min(on.dims, 12)
        np.testing.assert_allclose(on.eigenvalues[:top], want["eigenvalues"][:top], rtol=1e-10)
        assert coords_match_up_to_sign(on.coords[:, :top], want["coords"][:, :top]) < \
            1e-7 * np.sqrt(want["eigenvalues"][0])


def test_sdig_cache_chunk_edge(ds, oracle):
    # n > 8192 columns: the int32 accumulation flushes mid-row (kChunk); the
    # streamed passes follow the same walk
    n = 8400
    d = ds.matrix_euclidean(ds.synth_points(1, n, 4))
    g = _gram(ds, d, 0)
    off, _ = _solve(ds, g, 40, 10, 1, 9, 0)
    on, st = _solve(ds, g, 40, 10, 1, 9, 2)
    assert st.last_product_sdig == 1
    if os.environ.get("DSB_K2I_STREAM_CL") != "1":
        assert np.array_equal(on.coords, off.coords)
    else:
        assert coords_match_up_to_sign(on.coords, off.coords) < 1e-9 * np.sqrt(off.eigenvalues[0])


def test_sdig_cache_auto_policy(ds):
    # auto: on whenever the int8 path runs and the cache fits; policy 0
    # disables it; the first-pass statistics count one storing pass per solve
    g = _gram(ds, ds.matrix_euclidean(ds.synth_points(2, 4200, 5)), 0)
    ds.set_product_path(2)
    try:
        ds.stats_reset()
        ds.embed(g, rank=40, oversampling=10, power_iters=1, seed=1)
        st = ds.stats_get()
        assert st.last_product_sdig == 1
        assert (st.product_launches, st.product_first_launches) == (4, 1)
        ds.embed(g, rank=20, oversampling=10, power_iters=1, seed=1)
        assert ds.stats_get().last_product_sdig == 1
        ds.set_sdig_cache(0)
        ds.embed(g, rank=40, oversampling=10, power_iters=1, seed=1)
        assert ds.stats_get().last_product_sdig == 0
    finally:
        ds.set_product_path(0)
        ds.set_sdig_cache(1)
    with pytest.raises(ds.DivscopeError):
        ds.set_sdig_cache(3)


K1_CASES = [
    # (kind, n, rank, over): K1 writes the planes while it reads D for the gram
    ("f64", 4133, 20, 10),   # NB = 32, ragged n (odd 64-row tile count)
    ("f64", 4300, 20, 10),   # the last 64-column tile ends past the last k-step
    ("f64", 4500, 40, 10),   # NB = 64 hybrid
    ("f64", 4250, 50, 20),   # the CTA pair
    ("ham", 4300, 30, 20),   # Hamming slices: no exponents needed
    ("ham", 4100, 50, 20),   # Hamming slices on the pair
]


@pytest.mark.parametrize("kind,n,rank,over", K1_CASES)
def test_k1_written_cache_matches_oracle(ds, oracle, kind, n, rank, over):
    # every product pass streams the planes K1 wrote (digits of d^2 scaled
    # by the row-0 triangle bound, within 3 bits of the true row exponent)
    d = _matrix(ds, kind, n, n % 7)
    g = _gram(ds, d, 1)
    off, _ = _solve(ds, g, rank, over, 2, 5, 0)
    on, st = _solve(ds, g, rank, over, 2, 5, 1)
    assert st.last_product_kernel == 1 and st.last_product_sdig == 2
    assert st.product_first_launches >= 1
    np.testing.assert_allclose(on.eigenvalues, off.eigenvalues, rtol=1e-10,
                               atol=1e-13 * abs(off.eigenvalues[0]))
    dm = d.to_numpy()
    _, rm, grand = oracle.gram_stats(dm)
    want = oracle.embed(rank, over, 2, 5, d=dm, row_mean=rm, grand=grand)
    top = min(on.dims, 12)
    np.testing.assert_allclose(on.eigenvalues[:top], want["eigenvalues"][:top], rtol=1e-10)
    assert coords_match_up_to_sign(on.coords[:, :top], want["coords"][:, :top]) < \
        1e-7 * np.sqrt(want["eigenvalues"][0])
    if kind == "ham":
        # exact slices: the same digits as the storing pass, bit-identical
        g0 = _gram(ds, d, 0)
        stored, st0 = _solve(ds, g0, rank, over, 2, 5, 1)
        assert st0.last_product_sdig == 1
        assert np.array_equal(stored.coords, on.coords)


def test_k1_cache_non_metric_falls_back(ds, oracle):
    # a point 1e-3 from every other one breaks the triangle inequality the
    # row-0 bound rests on: K1's check rejects its planes, the solve stores
    # its own
    n = 4200
    d = ds.matrix_euclidean(ds.synth_points(2, n, 3)).to_numpy()
    d[0, 1:] = 1e-3
    d[1:, 0] = 1e-3
    m = ds.matrix_from_host(d)
    g = _gram(ds, m, 1)
    on, st = _solve(ds, g, 20, 10, 1, 2, 1)
    assert st.last_product_kernel == 1 and st.last_product_sdig == 1
    off, _ = _solve(ds, g, 20, 10, 1, 2, 0)
    assert np.array_equal(on.coords, off.coords)


def test_k1_cache_generation(ds):
    # a later gram (or a storing solve) overwrites the slot: an older gram's
    # solves must not stream it
    a = _gram(ds, ds.matrix_euclidean(ds.synth_points(2, 4400, 1)), 1)
    ref_a, _ = _solve(ds, a, 20, 10, 1, 4, 0)
    b = _gram(ds, ds.matrix_euclidean(ds.synth_points(3, 4400, 2)), 1)
    got_a, st = _solve(ds, a, 20, 10, 1, 4, 1)
    assert st.last_product_sdig == 1  # a's planes are gone: stored again
    assert np.array_equal(got_a.coords, ref_a.coords)
    got_b, st = _solve(ds, b, 20, 10, 1, 4, 1)
    assert st.last_product_sdig == 1  # a's storing solve overwrote b's planes
    again_a, st = _solve(ds, a, 20, 10, 1, 4, 1)
    assert st.last_product_sdig == 1
    assert np.array_equal(again_a.coords, got_a.coords)


def test_evicted_cache_is_stored_again(ds):
    # a failed device allocation drops the slot (and the graphs that address
    # it): the gram's planes are gone, its next solve stores them again and
    # gets the same answer; with the slot back, later solves stream it
    import ctypes as C
    ev = ds.lib.divscope_debug_evict_workspace
    ev.restype = C.c_int
    g = _gram(ds, ds.matrix_euclidean(ds.synth_points(2, 4600, 6)), 1)
    first, st = _solve(ds, g, 20, 10, 1, 8, 1)
    assert st.last_product_sdig == 2
    assert ev() == 1
    again, st = _solve(ds, g, 20, 10, 1, 8, 1)
    assert st.last_product_sdig == 1
    np.testing.assert_allclose(again.eigenvalues, first.eigenvalues, rtol=1e-12)
    assert coords_match_up_to_sign(again.coords, first.coords) < 1e-9 * np.sqrt(first.eigenvalues[0])
    third, st = _solve(ds, g, 20, 10, 1, 8, 1)
    assert st.last_product_sdig == 1
    assert np.array_equal(third.coords, again.coords)
