"""GPU tests of the row-sharded (multi-GPU) path, run with one rank: the same
code as N ranks with every collective over a single-rank NCCL communicator.
(One GPU per box here; ranks that wait on each other must not share a GPU.)"""
import numpy as np
import pytest

from helpers import coords_match_up_to_sign, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm1(ds):
    uid = ds.comm_unique_id()
    ds.comm_init(1, 0, uid)
    yield
    ds.comm_destroy()



@pytest.fixture(autouse=True, params=["auto", "int8"])
def product_path(request, ds):
    """Sharded solves on both product kernels (fp64 DMMA at these n / forced int8)."""
    ds.set_product_path(2 if request.param == "int8" else 0)
    yield request.param
    ds.set_product_path(0)


def test_sharded_embed_matches_oracle(ds, oracle, comm1):
    pts = ds.synth_points(2, 1800, 4)
    n = pts.shape[0]
    b, e = ds.shard_range(n, 1, 0)
    assert (b, e) == (0, n)
    d_sh = ds.matrix_euclidean_rows(pts, b, e)
    g = ds.gram(d_sh)
    emb = ds.embed(g, rank=20, oversampling=10, power_iters=2, seed=9)
    d = oracle.euclidean_matrix(pts)
    st, rm, grand = oracle.gram_stats(d)
    ref = oracle.embed(20, 10, 2, 9, d=d, row_mean=rm, grand=grand)
    assert emb.dims == ref["r"]
    assert rel_err(emb.eigenvalues, ref["eigenvalues"]) < 1e-10
    assert coords_match_up_to_sign(emb.coords, ref["coords"]) < 1e-8 * np.sqrt(ref["eigenvalues"][0])
    vals, resid = ds.eigs(g, rank=20, oversampling=10, power_iters=2, seed=9)
    assert rel_err(vals, ref["eigenvalues"][: len(vals)]) < 1e-10


def test_sharded_matches_unsharded(ds, comm1):
    pts = ds.synth_points(1, 1000, 2)
    a = ds.embed(ds.gram(ds.matrix_euclidean(pts)), rank=10, oversampling=10, power_iters=1, seed=1)
    b = ds.embed(ds.gram(ds.matrix_euclidean_rows(pts, 0, 1000)), rank=10, oversampling=10,
                 power_iters=1, seed=1)
    assert rel_err(b.eigenvalues, a.eigenvalues) < 1e-12
    assert coords_match_up_to_sign(b.coords, a.coords) < 1e-9 * np.sqrt(a.eigenvalues[0])


def test_sharded_host_rows_and_validation(ds, oracle, comm1):
    pts = ds.synth_points(1, 300, 3)
    d = oracle.euclidean_matrix(pts)
    m = ds.matrix_from_host_rows(d, 300, 0, 300)
    assert (m.rows, m.cols) == (300, 300)
    emb = ds.embed(ds.gram(m), rank=5, oversampling=5, power_iters=1, seed=2)
    assert emb.dims == 5
    lie = d.copy()
    lie[3, 7] += 1e-6
    with pytest.raises(ds.DivscopeError) as ei:
        ds.gram(ds.matrix_from_host_rows(lie, 300, 0, 300))
    assert ei.value.status == ds.Status.ERR_NOT_SYMMETRIC
    with pytest.raises(ds.DivscopeError) as ei:
        ds.gram(ds.matrix_from_host_rows(d[:100], 300, 0, 100))  # not this rank's range
    assert ei.value.status == ds.Status.ERR_SHAPE_MISMATCH


def test_sharded_f32(ds, oracle, comm1):
    pts = ds.synth_points(4, 1200, 5)
    d32 = oracle.euclidean_matrix(pts).astype(np.float32)
    m = ds.matrix_from_host_rows_f32(d32, 1200, 0, 1200)
    emb = ds.embed(ds.gram(m), rank=30, oversampling=10, power_iters=2, seed=3)
    dw = d32.astype(np.float64)
    st, rm, grand = oracle.gram_stats(dw)
    ref = oracle.embed(30, 10, 2, 3, d=dw, row_mean=rm, grand=grand)
    assert rel_err(emb.eigenvalues[:30], ref["eigenvalues"][:30]) < 1e-4


def test_sharded_from_dvs_rows(ds, oracle, comm1, tmp_path):
    # each rank streams only its rows of the DVS file (divscope_matrix_read_rows)
    n, k, p, q, seed = 600, 8, 8, 1, 4
    pts = ds.synth_points(2, n, seed)
    d = oracle.euclidean_matrix(pts)
    f = tmp_path / "d.dvs"
    ds.matrix_from_host(d).write(f)
    rb, re_ = ds.shard_range(n, 1, 0)
    shard = ds.matrix_read_rows(f, rb, re_)
    e = ds.embed(ds.gram(shard), rank=k, oversampling=p, power_iters=q, seed=seed)
    ref = ds.embed(ds.gram(ds.matrix_from_host(d)), rank=k, oversampling=p, power_iters=q,
                   seed=seed)
    np.testing.assert_allclose(e.eigenvalues, ref.eigenvalues, rtol=1e-10)


def test_symmetry_fingerprint_matches_restatement(ds, oracle):
    # the sharded gram decides symmetry from one all-reduced pair of 32-bit
    # sums of per-shard antisymmetric fingerprints (k1_shard.cu, sharded.cpp)
    import ctypes as C
    from helpers import sym_fingerprint
    fn = ds.lib.divscope_debug_sym_fingerprint
    fn.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]

    def fp(m):
        out = (C.c_uint64 * 2)()
        assert fn(m.handle, out) == 0
        return (out[0], out[1])

    def total(*parts):
        return tuple(sum(p[k] for p in parts) % 2**32 for k in range(2))

    n = 700
    d = oracle.euclidean_matrix(ds.synth_points(2, n, 9))
    a = ds.matrix_from_host_rows(d[0:256], n, 0, 256)
    b = ds.matrix_from_host_rows(d[256:700], n, 256, 700)
    fa, fb = fp(a), fp(b)
    assert fa == sym_fingerprint(d[0:256], 0) and fb == sym_fingerprint(d[256:700], 256)
    assert total(fa, fb) == (0, 0) and fa != (0, 0)
    d2 = d.copy()
    d2[300, 10] = np.nextafter(d2[300, 10], 1e9)  # one ulp off its mirror
    b2 = ds.matrix_from_host_rows(d2[256:700], n, 256, 700)
    assert total(fa, fp(b2)) != (0, 0)
    # f32 storage hashes the widened values; an unsharded handle covers all rows
    af = ds.matrix_from_host_rows_f32(d[0:256].astype(np.float32), n, 0, 256)
    assert fp(af) == sym_fingerprint(d[0:256].astype(np.float32), 0)
    assert fp(ds.matrix_from_host(d)) == (0, 0)


def test_sharded_gram_tolerates_tiny_asymmetry(ds, oracle, comm1):
    # a nonzero fingerprint triggers the exact max |d_ij - d_ji| measurement;
    # the reference's 1e-12 * max(1, max|d|) tolerance decides (mds.cpp:23-27)
    n = 500
    d = oracle.euclidean_matrix(ds.synth_points(1, n, 4))
    near = d.copy()
    near[3, 7] = np.nextafter(near[3, 7], 1e9)
    g = ds.gram(ds.matrix_from_host_rows(near, n, 0, n))
    e = ds.embed(g, rank=5, oversampling=5, power_iters=1, seed=1)
    ref = ds.embed(ds.gram(ds.matrix_from_host(d)), rank=5, oversampling=5, power_iters=1, seed=1)
    np.testing.assert_allclose(e.eigenvalues, ref.eigenvalues, rtol=1e-10)
    far = d.copy()
    far[7, 3] += 1e-9 * d.max()
    with pytest.raises(ds.DivscopeError) as ei:
        ds.gram(ds.matrix_from_host_rows(far, n, 0, n))
    assert ei.value.status == ds.Status.ERR_NOT_SYMMETRIC


@pytest.mark.parametrize("rank,over,f32", [(60, 10, False), (100, 20, True)])
def test_sharded_wide_panel_matches_unsharded(ds, comm1, product_path, rank, over, f32):
    # w > 64: the int8 product runs in two column groups on each rank's rows
    # (forced int8) or the fp64 DMMA kernel at WP > 64 (auto at this n)
    pts = ds.synth_points(3, 1500, 6)
    n = pts.shape[0]
    a = ds.embed(ds.gram(ds.matrix_euclidean(pts, store_f32=f32)), rank=rank, oversampling=over,
                 power_iters=2, seed=3)
    b = ds.embed(ds.gram(ds.matrix_euclidean_rows(pts, 0, n, store_f32=f32)), rank=rank,
                 oversampling=over, power_iters=2, seed=3)
    st = ds.stats_get()
    if product_path == "int8":
        assert (st.last_product_kernel, st.last_product_groups) == (1, 2)
    assert b.dims == a.dims
    np.testing.assert_allclose(b.eigenvalues[:30], a.eigenvalues[:30], rtol=1e-10)
    np.testing.assert_allclose(b.eigenvalues, a.eigenvalues, rtol=1e-6)


def test_sharded_rank_deficient_panel_shifts(ds, oracle, comm1):
    # 3-D points, w = 24: the panel is numerically rank 3, CholeskyQR shifts
    # on its first pass and the shift-gated third pass runs (sharded.cpp
    # orth_local); the kept spectrum must match the unsharded solve
    rng = np.random.default_rng(11)
    pts = rng.standard_normal((900, 3)) * 5.0
    d = oracle.euclidean_matrix(pts)
    a = ds.embed(ds.gram(ds.matrix_from_host(d)), rank=12, oversampling=12, power_iters=2, seed=4)
    b = ds.embed(ds.gram(ds.matrix_from_host_rows(d, 900, 0, 900)), rank=12, oversampling=12,
                 power_iters=2, seed=4)
    assert ds.stats_get().last_orth_shifted == 1
    assert a.dims == b.dims == 3
    np.testing.assert_allclose(b.eigenvalues, a.eigenvalues, rtol=1e-10)
    assert coords_match_up_to_sign(b.coords, a.coords) < 1e-8 * np.sqrt(a.eigenvalues[0])


def test_hamming_rows_shard_matches_full(ds, comm1):
    # K7 row shards (divscope_matrix_hamming_rows) keep the Hamming tag, so the
    # sharded int8 product slices S in three bytes like the full matrix
    reads = ds.synth_reads(700, 400, 9, 0.05, 3)
    full = ds.matrix_hamming(reads)
    rows = ds.matrix_hamming_rows(np.frombuffer(b"".join(reads), np.uint8).reshape(700, 400),
                                  0, 700)
    assert np.array_equal(rows.to_numpy(), full.to_numpy())
    part = ds.matrix_hamming_rows(reads, 256, 700)
    assert np.array_equal(part.to_numpy(), full.to_numpy()[256:700])
    a = ds.embed(ds.gram(full), rank=8, oversampling=8, power_iters=2, seed=2)
    b = ds.embed(ds.gram(rows), rank=8, oversampling=8, power_iters=2, seed=2)
    np.testing.assert_allclose(b.eigenvalues, a.eigenvalues, rtol=1e-10)
    with pytest.raises(ds.DivscopeError) as ei:
        ds.matrix_hamming_rows([b"ACGT", b"ACGN"], 0, 2)
    assert ei.value.status == ds.Status.ERR_INVALID_CHARACTER
