"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle
and the reference's own known-answer tests.

Reference KATs ported from /root/reference/proj/tests/test_mds.cpp,
test_rsvd.cpp, test_capi.cpp and acceptance.cpp (cited per test).
Tolerances: eigenvalues relative 1e-10 (fp64 D) / 1e-4 (fp32 D) per
BASELINE.json north_star; coordinates per column up to sign; integer Hamming
counts and Euclidean distances bit-exact.
"""
import numpy as np
import pytest

from helpers import coords_match_up_to_sign, rel_err, sin_subspace, with_spectrum

pytestmark = pytest.mark.gpu


def err(ds, fn, *a, **k):
    with pytest.raises(ds.DivscopeError) as ei:
        fn(*a, **k)
    return ei.value.status


# ---------------------------------------------------------------- builders


@pytest.fixture(autouse=True, params=["auto", "int8"])
def product_path(request, ds):
    """Every parity test runs twice: with the automatic product-kernel choice
    (fp64 DMMA at these small n) and with the int8 slice product forced for
    every lazy gram it supports (k2i_product.cu)."""
    ds.set_product_path(2 if request.param == "int8" else 0)
    yield request.param
    ds.set_product_path(0)


def test_euclid_bit_exact_vs_oracle(ds, oracle):
    pts = ds.synth_points(1, 301, 11)
    d_gpu = ds.matrix_euclidean(pts).to_numpy()
    d_cpu = oracle.euclidean_matrix(pts)
    assert np.array_equal(d_gpu, d_cpu)
    d32 = ds.matrix_euclidean(pts, store_f32=True).to_numpy()
    assert np.array_equal(d32, d_cpu.astype(np.float32).astype(np.float64))


def test_euclid_matches_reference_fixture(ds, ref):
    # ref tests/testdata.cpp:157-184 compiled from the reference sources
    pts = ref.uniform_box(97, 5, 303)
    assert np.array_equal(ds.matrix_euclidean(pts).to_numpy(), ref.euclidean_matrix(pts))


def test_hamming_counts_bit_exact(ds, oracle):
    reads = ds.synth_reads(203, 400, 7, 0.05, 5)
    h = ds.hamming_counts(reads)
    st, h_cpu = oracle.hamming_counts(b"".join(reads), len(reads), 400)
    assert st == 0
    assert np.array_equal(h, h_cpu)
    d = ds.matrix_hamming(reads).to_numpy()
    assert np.array_equal(d, h_cpu.astype(np.float64) / 400.0)


def test_hamming_edge_cases(ds, oracle):
    # odd length (partial last word), identical reads, single read
    reads = [b"ACGTA", b"ACGTA", b"TTTTT"]
    h = ds.hamming_counts(reads)
    assert h.tolist() == [[0, 0, 4], [0, 0, 4], [4, 4, 0]]
    assert ds.hamming_counts([b"A" * 33]).tolist() == [[0]]
    assert err(ds, ds.hamming_counts, [b"ACGN"]) == ds.Status.ERR_INVALID_CHARACTER


@pytest.mark.parametrize("count,length", [(1, 1), (3, 5), (127, 10), (128, 11), (129, 33),
                                          (300, 400), (1000, 150), (257, 1000), (140, 4095)])
def test_hamming_tensor_core_builder_bit_exact(ds, count, length):
    # K7's D on the int8 tensor cores (hamming_tc.cu: +-1 encoding, one GEMM,
    # h = (3 L - acc) / 4) against plain character comparison, the POPC
    # counts kernel, and 128-aligned row bands (tensor cores) next to
    # unaligned ones (POPC kernel)
    rng = np.random.default_rng(count * 7919 + length)
    arr = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, (count, length))]
    if count > 2:
        arr[1] = arr[0]  # an identical pair
        arr[2, : length // 2] = arr[0, : length // 2]
    reads = [r.tobytes() for r in arr]
    h = (arr[:, None, :] != arr[None, :, :]).sum(-1) if count * count * length < 2e8 else None
    d = ds.matrix_hamming(reads).to_numpy()
    counts = ds.hamming_counts(reads)
    if h is not None:
        assert np.array_equal(counts, h)
    assert np.array_equal(d, counts.astype(np.float64) / length)
    for r0, r1 in [(128, count), (0, min(count, 200)), (5, min(count, 140))]:
        if r0 >= r1:
            continue
        band = ds.matrix_hamming_rows(reads, r0, r1).to_numpy()
        assert np.array_equal(band, d[r0:r1])


# ---------------------------------------------------------------- gram

def test_gram_two_point_exact(ds):
    # ref tests/test_mds.cpp:27-34
    g = ds.gram(ds.matrix_from_host(np.array([[0.0, 2.0], [2.0, 0.0]])))
    assert g.to_numpy().tolist() == [[1.0, -1.0], [-1.0, 1.0]]
    assert g.get(1, 0) == -1.0 and g.symmetric


def test_gram_zero(ds):
    # ref tests/test_mds.cpp:36-39
    g = ds.gram(ds.matrix_from_host(np.zeros((3, 3))))
    assert not np.any(g.to_numpy())


def test_gram_matches_oracle(ds, oracle):
    pts = ds.synth_points(2, 513, 3)
    d = oracle.euclidean_matrix(pts)
    st, g_cpu = oracle.gram(d)
    assert st == 0
    g_gpu = ds.gram(ds.matrix_from_host(d)).to_numpy()
    assert np.max(np.abs(g_gpu - g_cpu)) <= 1e-13 * np.max(np.abs(g_cpu))
    assert np.array_equal(g_gpu, g_gpu.T)
    # double-centering: rows sum to ~0 (ref tests/test_mds.cpp:41-55)
    assert np.max(np.abs(g_gpu.sum(1))) < 1e-9 * np.max(np.abs(g_gpu)) * 513


def test_gram_validation(ds):
    # ref tests/test_mds.cpp:76-101
    rect = ds.matrix_from_host(np.zeros((2, 3)), symmetric=False)
    assert err(ds, ds.gram, rect) == ds.Status.ERR_NOT_SYMMETRIC
    lie = ds.matrix_from_host(np.array([[0.0, 1.0], [2.0, 0.0]]))
    assert err(ds, ds.gram, lie) == ds.Status.ERR_NOT_SYMMETRIC
    empty = ds.matrix_from_host(np.zeros((0, 0)))
    assert err(ds, ds.gram, empty) == ds.Status.ERR_EMPTY_INPUT
    unflagged = ds.matrix_from_host(np.zeros((2, 2)), symmetric=False)
    assert err(ds, ds.gram, unflagged) == ds.Status.ERR_NOT_SYMMETRIC


def test_gram_tolerance_boundary(ds):
    # |d_ij - d_ji| <= 1e-12 max(1, max|d|) passes (ref mds.cpp:23-27)
    d = np.array([[0.0, 3.0], [3.0 + 2e-12, 0.0]])
    ds.gram(ds.matrix_from_host(d))
    d[1, 0] = 3.0 + 8e-12
    assert err(ds, ds.gram, ds.matrix_from_host(d)) == ds.Status.ERR_NOT_SYMMETRIC


@pytest.mark.parametrize("where", ["diag_tile", "off_tile", "tail_tile", "zero_vs_neg_zero"])
def test_gram_f32_symmetry_check(ds, oracle, where):
    # f32 tiles compare the mirrored pairs by their bits (k1_stats.cu) and
    # take the reference's f64 difference only for a differing pair: one
    # asymmetric pair anywhere (inside a diagonal 64 x 64 tile, an
    # off-diagonal one, the ragged last tile) is found; -0.0 against +0.0
    # differs in bits but not in value, as in the reference
    n = 200
    d = oracle.euclidean_matrix(ds.synth_points(1, n, 3)).astype(np.float32)
    ds.gram(ds.matrix_from_host_f32(d))
    i, j = {"diag_tile": (5, 40), "off_tile": (150, 20), "tail_tile": (199, 130),
            "zero_vs_neg_zero": (7, 7)}[where]
    bad = d.copy()
    if where == "zero_vs_neg_zero":
        bad[3, 9] = bad[9, 3] = 0.0
        bad[3, 9] = -0.0
        ds.gram(ds.matrix_from_host_f32(bad))  # |0 - (-0)| = 0: symmetric
        return
    bad[i, j] = np.nextafter(bad[i, j], np.float32(1e9))
    assert err(ds, ds.gram, ds.matrix_from_host_f32(bad)) == ds.Status.ERR_NOT_SYMMETRIC


# ---------------------------------------------------------------- eigs KATs

def test_eigs_signed_diagonal(ds):
    # ref tests/test_rsvd.cpp:103-118
    g = ds.matrix_from_host(np.diag([3.0, -2.0, 1.0]))
    vals, _ = ds.eigs(g, rank=2, oversampling=1, power_iters=2, seed=0)
    assert vals.shape == (2,)
    assert vals[0] == pytest.approx(3.0, rel=1e-12)
    assert vals[1] == pytest.approx(-2.0, rel=1e-12)


def test_eigs_magnitude_order_positive_first(ds):
    # ref tests/test_rsvd.cpp:120-130
    g = ds.matrix_from_host(np.diag([2.0, -2.0, 1.0]))
    vals, _ = ds.eigs(g, rank=3, oversampling=0, power_iters=2, seed=0)
    assert vals == pytest.approx([2.0, -2.0, 1.0], rel=1e-12)


def test_eigs_rank_one(ds, oracle):
    # ref tests/test_rsvd.cpp:132-156
    x = oracle.fill_gaussian(3, 40)
    x /= np.linalg.norm(x)
    vals, resid = ds.eigs(ds.matrix_from_host(np.outer(x, x)), rank=1, oversampling=10,
                          power_iters=2, seed=0)
    assert vals[0] == pytest.approx(1.0, rel=1e-10)
    assert resid < 1e-6


def test_eigs_vs_dense(ds, oracle):
    # ref tests/test_rsvd.cpp:158-183
    w = [100.0 * 0.7 ** i for i in range(20)] + [0.0] * 40
    g = with_spectrum(w, 12345, oracle)
    vals, _ = ds.eigs(ds.matrix_from_host(g), rank=10, oversampling=10, power_iters=3, seed=0)
    dense = np.sort(np.linalg.eigvalsh(g))[::-1][:10]
    assert rel_err(vals, dense) < 1e-6


def test_eigs_residual_tail(ds, oracle):
    # ref tests/test_rsvd.cpp:202-216
    g = ds.matrix_from_host(with_spectrum([6, 5, 4, 0, 0, 0, 0, 0], 8, oracle))
    _, r3 = ds.eigs(g, rank=3, oversampling=5, power_iters=2, seed=0)
    assert r3 < 1e-6
    _, r2 = ds.eigs(g, rank=2, oversampling=0, power_iters=6, seed=0)
    assert r2 == pytest.approx(4.0, rel=0.02)


def test_eigs_errors(ds):
    # ref tests/test_rsvd.cpp:218-250, test_capi.cpp:254-260
    g = ds.matrix_from_host(np.diag([1.0, 2.0, 3.0]))
    assert err(ds, ds.eigs, g, rank=3, oversampling=1) == ds.Status.ERR_RANK_TOO_LARGE
    assert err(ds, ds.eigs, g, rank=0, oversampling=1) == ds.Status.ERR_INVALID_ARGUMENT
    asym = ds.matrix_from_host(np.array([[0.0, 1.0], [2.0, 0.0]]))
    assert err(ds, ds.eigs, asym, rank=1, oversampling=0) == ds.Status.ERR_NOT_SYMMETRIC
    rect = ds.matrix_from_host(np.zeros((2, 3)), symmetric=False)
    assert err(ds, ds.eigs, rect, rank=1, oversampling=0) == ds.Status.ERR_NOT_SYMMETRIC
    empty = ds.matrix_from_host(np.zeros((0, 0)))
    assert err(ds, ds.eigs, empty, rank=1, oversampling=0) == ds.Status.ERR_INVALID_ARGUMENT


def test_eigs_matches_oracle_explicit(ds, oracle):
    w = [50, 20, 10, 5, 2, 1, 0.5, 0.1] + [0.0] * 52
    g = with_spectrum(w, 321, oracle)
    vals, resid = ds.eigs(ds.matrix_from_host(g), rank=5, oversampling=5, power_iters=2, seed=9)
    st, v_cpu, _, r_cpu = oracle.eigs(5, 5, 2, 9, g=g)
    assert st == 0
    assert rel_err(vals, v_cpu) < 1e-10
    fro2 = float(np.sum(g * g))
    assert abs(resid ** 2 - r_cpu ** 2) <= 1e-12 * fro2


# ---------------------------------------------------------------- range

def test_range_orthonormal(ds, oracle):
    # ref tests/test_rsvd.cpp:50-62
    g = ds.matrix_from_host(with_spectrum([9, 7, 5, 3, 1, 0.5, 0.1, 0.05], 4, oracle))
    q = ds.randomized_range(g, rank=3, oversampling=2, power_iters=2, seed=0)
    assert q.shape == (8, 5)
    assert np.max(np.abs(q.T @ q - np.eye(5))) < 1e-8


def test_range_captures_diagonal_subspace(ds):
    # ref tests/test_rsvd.cpp:64-79
    g = ds.matrix_from_host(np.diag([10.0, 5.0, 1.0] + [0.0] * 7))
    q = ds.randomized_range(g, rank=3, oversampling=5, power_iters=2, seed=0)
    for axis in range(3):
        e = np.zeros(10)
        e[axis] = 1.0
        assert np.linalg.norm(q @ (q.T @ e) - e) < 1e-10


# ---------------------------------------------------------------- embed KATs

def test_embed_two_points(ds):
    # ref tests/test_mds.cpp:103-114
    g = ds.gram(ds.matrix_from_host(np.array([[0.0, 2.0], [2.0, 0.0]])))
    e = ds.embed(g, rank=1, oversampling=10, power_iters=2, seed=0)
    assert (e.rows, e.dims) == (2, 1)
    assert e.eigenvalues[0] == pytest.approx(2.0, rel=1e-12)
    c = e.coords
    assert c[0, 0] == pytest.approx(1.0, rel=1e-10)
    assert c[1, 0] == pytest.approx(-1.0, rel=1e-10)
    assert e.dropped_negative_mass == 0.0 and not e.truncated


def test_embed_zero_gram(ds):
    # ref tests/test_mds.cpp:116-126
    e = ds.embed(ds.matrix_from_host(np.zeros((3, 3))), rank=2, oversampling=10, seed=0)
    assert e.rows == 3 and e.dims == 0 and e.truncated and e.dropped_negative_mass == 0.0


def test_embed_euclidean_round_trip(ds, oracle):
    # ref tests/test_mds.cpp:128-147 (and acceptance #3, acceptance.cpp:97-123)
    pts = oracle.fill_gaussian(21, 40 * 3).reshape(40, 3)
    d = oracle.euclidean_matrix(pts)
    g = ds.gram(ds.matrix_from_host(d))
    e = ds.embed(g, rank=3, oversampling=10, power_iters=2, seed=1)
    assert e.dims == 3
    x = e.coords
    dd = np.sqrt(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1))
    iu = np.triu_indices(40, 1)
    assert np.max(np.abs(dd[iu] - d[iu]) / d[iu]) < 1e-8


def test_embed_truncation(ds, oracle):
    # ref tests/test_mds.cpp:149-159
    pts = oracle.fill_gaussian(33, 20 * 3).reshape(20, 3)
    g = ds.gram(ds.matrix_from_host(oracle.euclidean_matrix(pts)))
    e = ds.embed(g, rank=5, oversampling=10, power_iters=2, seed=0)
    assert e.dims == 3 and e.truncated and len(e.eigenvalues) == 3


def test_embed_column_norms_and_sign(ds, oracle):
    # ref tests/test_mds.cpp:161-195
    pts = oracle.fill_gaussian(44, 30 * 4).reshape(30, 4)
    g = ds.gram(ds.matrix_from_host(oracle.euclidean_matrix(pts)))
    e = ds.embed(g, rank=4, oversampling=10, power_iters=2, seed=0)
    assert e.dims == 4
    ev, x = e.eigenvalues, e.coords
    assert np.all(ev > 0) and np.all(np.diff(ev) <= 0)
    assert np.allclose((x * x).sum(0), ev, rtol=1e-6)
    for c in range(4):
        assert x[np.argmax(np.abs(x[:, c])), c] > 0


def test_embed_negative_mass(ds):
    # ref tests/test_mds.cpp:197-214, acceptance.cpp:191-217
    d = np.ones((4, 4)) - np.eye(4)
    d[2, 3] = d[3, 2] = 2.0
    e = ds.embed(ds.gram(ds.matrix_from_host(d)), rank=4, oversampling=10, seed=5)
    assert e.dropped_negative_mass > 0.0 and e.truncated and e.dims >= 2
    assert np.all(e.eigenvalues > 0)


def test_embed_rank_bounds(ds):
    # ref tests/test_mds.cpp:216-225, test_capi.cpp:281-285
    g = ds.gram(ds.matrix_from_host(np.array([[0.0, 2.0], [2.0, 0.0]])))
    assert err(ds, ds.embed, g, rank=0) == ds.Status.ERR_RANK_TOO_LARGE
    assert err(ds, ds.embed, g, rank=3) == ds.Status.ERR_RANK_TOO_LARGE
    assert err(ds, ds.embed, g, rank=1, ids=["a", "b", "c"]) == ds.Status.ERR_SHAPE_MISMATCH


def test_embed_ids_and_files(ds, tmp_path):
    # ref tests/test_capi.cpp:255-278 (write / load round trip)
    g = ds.gram(ds.matrix_from_host(np.array([[0.0, 2.0], [2.0, 0.0]])))
    e = ds.embed(g, rank=1, ids=["a", "b"])
    assert e.id(0) == "a" and e.id(2) is None
    e.write(tmp_path / "e.tsv", tmp_path / "e.meta")
    back = ds.embedding_load(tmp_path / "e.tsv")
    assert back.rows == 2 and back.dims == 1 and back.get(1, 0) == e.get(1, 0)
    assert len(back.eigenvalues) == 0
    meta = (tmp_path / "e.meta").read_text().splitlines()
    assert meta[0] == "rank=1" and meta[1] == "truncated=0"


# ---------------------------------------------------------------- parity at scale

def _parity(ds, oracle, d, k, p, q, seed, eig_tol, d_host=None, f32=False):
    """embed through the GPU vs the oracle restatement on the same D and Omega."""
    dm = ds.matrix_from_host_f32(d) if f32 else ds.matrix_from_host(d)
    e = ds.embed(ds.gram(dm), rank=k, oversampling=p, power_iters=q, seed=seed)
    dh = d_host if d_host is not None else d
    st, rm, grand = oracle.gram_stats(dh)
    assert st == 0
    ref = oracle.embed(k, p, q, seed, d=dh, row_mean=rm, grand=grand)
    assert ref["status"] == 0
    return e, ref


def test_c1_parity(ds, oracle):
    # BASELINE config 1 at full size: n=2000, k=10, p=10, q=1
    pts = ds.synth_points(1, 2000, 1)
    d = oracle.euclidean_matrix(pts)
    e, ref = _parity(ds, oracle, d, 10, 10, 1, 1, 1e-10)
    assert e.dims == ref["r"] == 10 and e.truncated == ref["truncated"]
    assert rel_err(e.eigenvalues, ref["eigenvalues"]) < 1e-10
    lam = ref["eigenvalues"]
    # coordinates: per column up to sign, scaled by sqrt(lambda_k)
    assert coords_match_up_to_sign(e.coords, ref["coords"]) < 1e-8 * np.sqrt(lam[0])
    assert sin_subspace(e.coords, ref["coords"]) < 1e-9
    fro2 = float(np.sum(oracle.gram(d)[1] ** 2))
    assert abs(e.resid ** 2 - ref["resid"] ** 2) <= 1e-11 * fro2


def test_c5_like_hamming_parity(ds, oracle):
    reads = ds.synth_reads(1500, 400, 50, 0.05, 5)
    d = ds.matrix_hamming(reads).to_numpy()
    e, ref = _parity(ds, oracle, d, 30, 20, 2, 5, 1e-10)
    assert e.dims == ref["r"]
    assert rel_err(e.eigenvalues, ref["eigenvalues"]) < 1e-10
    assert abs(e.dropped_negative_mass - ref["dropped_negative_mass"]) <= 1e-10 * max(
        1.0, abs(ref["eigenvalues"][0]))


def test_c4_like_f32_parity(ds, oracle):
    # fp32-stored D, fp64 arithmetic; w = 70 > dim 64: rank-deficient panel
    pts = ds.synth_points(4, 1500, 7)
    d32 = oracle.euclidean_matrix(pts).astype(np.float32)
    d_wide = d32.astype(np.float64)
    e, ref = _parity(ds, oracle, d32, 50, 20, 3, 7, 1e-4, d_host=d_wide, f32=True)
    top = min(40, ref["r"])
    assert rel_err(e.eigenvalues[:top], ref["eigenvalues"][:top]) < 1e-4


def test_deterministic(ds):
    pts = ds.synth_points(2, 700, 2)
    g = ds.gram(ds.matrix_euclidean(pts))
    a = ds.embed(g, rank=20, oversampling=10, power_iters=2, seed=3)
    b = ds.embed(g, rank=20, oversampling=10, power_iters=2, seed=3)
    assert np.array_equal(a.coords, b.coords) and np.array_equal(a.eigenvalues, b.eigenvalues)


def test_graph_replay_follows_inputs(ds, oracle):
    # a solve is captured as a CUDA graph on the first call of its signature
    # and replayed afterwards (solver.cpp run): replays must follow a new seed
    # (Omega re-uploaded into the same workspace slot), a second matrix of the
    # same shape, and eigs / embed / eigs_vectors interleaved on one gram
    n, k, p, q = 900, 10, 8, 1
    d = oracle.euclidean_matrix(ds.synth_points(2, n, 4))
    d2 = oracle.euclidean_matrix(ds.synth_points(2, n, 9))
    g, g2 = ds.gram(ds.matrix_from_host(d)), ds.gram(ds.matrix_from_host(d2))
    refs = {}
    for dd, key in ((d, 1), (d2, 2)):
        st, rm, grand = oracle.gram_stats(dd)
        assert st == 0
        for seed in (5, 6):
            refs[key, seed] = oracle.embed(k, p, q, seed, d=dd, row_mean=rm, grand=grand)
    first = {}
    for key, gm, seed in [(1, g, 5), (1, g, 6), (2, g2, 5), (1, g, 5), (2, g2, 6), (1, g, 6)]:
        e = ds.embed(gm, rank=k, oversampling=p, power_iters=q, seed=seed)
        ref = refs[key, seed]
        assert e.dims == ref["r"]
        assert rel_err(e.eigenvalues, ref["eigenvalues"]) < 1e-10
        assert coords_match_up_to_sign(e.coords, ref["coords"]) < 1e-8 * np.sqrt(ref["eigenvalues"][0])
        if (key, seed) in first:  # a replay: bit-identical to the captured run
            assert np.array_equal(e.coords, first[key, seed])
        first[key, seed] = e.coords
        vals, _ = ds.eigs(gm, rank=k, oversampling=p, power_iters=q, seed=seed)
        vv, vecs, _ = ds.eigs_vectors(gm, rank=k, oversampling=p, power_iters=q, seed=seed)
        assert np.array_equal(vals, vv) and vecs.shape == (n, k)
    # the launch counter advances by the same count on every replay (the
    # first call re-lays out Omega for the new seed: one launch more)
    ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=5)
    l0 = ds.stats_get().kernel_launches
    ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=5)
    l1 = ds.stats_get().kernel_launches
    ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=5)
    l2 = ds.stats_get().kernel_launches
    assert l2 - l1 == l1 - l0 > 0


# ---------------------------------------------------------------- stable rank

def test_stable_rank(ds):
    # ref tests/test_rsvd.cpp:252-279, acceptance.cpp:219-238
    assert ds.stable_rank(ds.matrix_from_host(np.diag([10.0, 5.0, 1.0]))) == pytest.approx(
        1.26, rel=1e-11)
    x = np.array([0.5, -1.25, 2.0, 0.75])
    assert ds.stable_rank(ds.matrix_from_host(np.outer(x, x))) == pytest.approx(1.0, rel=1e-9)
    assert ds.stable_rank(ds.matrix_from_host(np.eye(7))) == pytest.approx(7.0, rel=1e-9)
    assert err(ds, ds.stable_rank, ds.matrix_from_host(np.zeros((3, 3)))) == \
        ds.Status.ERR_ZERO_MATRIX


def test_stable_rank_lazy_gram_matches_oracle(ds, oracle):
    # device-side power iteration (batched, convergence on the device) on a
    # lazy gram vs the reference loop over the materialized gram
    pts = ds.synth_points(1, 300, 11)
    d = oracle.euclidean_matrix(pts)
    st, g = oracle.gram(d)
    assert st == 0
    st, want = oracle.stable_rank(g)
    assert st == 0
    got = ds.stable_rank(ds.gram(ds.matrix_from_host(d)))
    assert got == pytest.approx(want, rel=1e-10)
    # explicit matrix with a slowly converging spectrum (many batches)
    lam = np.linspace(1.0, 0.9, 40)
    q, _ = np.linalg.qr(np.random.default_rng(5).standard_normal((40, 40)))
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    st, want = oracle.stable_rank(a)
    assert st == 0
    assert ds.stable_rank(ds.matrix_from_host(a)) == pytest.approx(want, rel=1e-8)


# ---------------------------------------------------------------- DVS

def test_dvs_round_trip(ds, tmp_path):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((5, 7))
    m = ds.matrix_from_host(a, symmetric=False)
    m.write(tmp_path / "a.dvs")
    b = ds.matrix_read(tmp_path / "a.dvs")
    assert (b.rows, b.cols, b.symmetric) == (5, 7, False)
    assert np.array_equal(b.to_numpy(), a)


def test_dvs_streaming_ingest_and_row_shards(ds, oracle, tmp_path):
    # ref src/distmat.cpp:189-222 (DVS1), streamed in 1 MB chunks (conftest):
    # a 700 x 700 f64 payload spans 4 double-buffered chunks
    pts = ds.synth_points(1, 700, 5)
    d = oracle.euclidean_matrix(pts)
    f = tmp_path / "d.dvs"
    ds.matrix_from_host(d).write(f)
    full = ds.matrix_read(f)
    assert (full.rows, full.cols, full.symmetric) == (700, 700, True)
    assert np.array_equal(full.to_numpy(), d)
    part = ds.matrix_read_rows(f, 256, 512)
    assert (part.rows, part.cols) == (256, 700)
    assert np.array_equal(part.to_numpy(), d[256:512])
    empty = ds.matrix_read_rows(f, 300, 300)
    assert empty.rows == 0
    assert err(ds, ds.matrix_read_rows, f, 512, 256) == ds.Status.ERR_INVALID_ARGUMENT
    assert err(ds, ds.matrix_read_rows, f, 0, 701) == ds.Status.ERR_INVALID_ARGUMENT
    # non-symmetric file: no row shards
    rect = tmp_path / "r.dvs"
    ds.matrix_from_host(np.ones((3, 4)), symmetric=False).write(rect)
    assert err(ds, ds.matrix_read_rows, rect, 0, 1) == ds.Status.ERR_NOT_SYMMETRIC
    # truncated payload / header, bad magic (same codes as the reference)
    raw = f.read_bytes()
    (tmp_path / "t.dvs").write_bytes(raw[:-8])
    assert err(ds, ds.matrix_read, tmp_path / "t.dvs") == ds.Status.ERR_TRUNCATED
    (tmp_path / "h.dvs").write_bytes(raw[:20])
    assert err(ds, ds.matrix_read, tmp_path / "h.dvs") == ds.Status.ERR_TRUNCATED
    (tmp_path / "m.dvs").write_bytes(b"XXXX" + raw[4:64])
    assert err(ds, ds.matrix_read, tmp_path / "m.dvs") == ds.Status.ERR_BAD_FORMAT
    assert err(ds, ds.matrix_read, tmp_path / "missing.dvs") == ds.Status.ERR_IO


def test_reconstruction_error_matches_oracle(ds, oracle):
    # ref src/mds.cpp:126-150 and tests/test_mds.cpp:128-147 (recon < 1e-8 ||G||_F
    # for an exact low-rank cloud); lazy gram (upper tiles only) and explicit
    for n, dim, seed in ((300, 3, 7), (517, 20, 8)):
        rng = np.random.default_rng(seed)
        pts = rng.standard_normal((n, dim))
        d = oracle.euclidean_matrix(pts)
        st, g = oracle.gram(d)
        g_lazy = ds.gram(ds.matrix_from_host(d))
        e = ds.embed(g_lazy, rank=min(dim, 10), oversampling=5, power_iters=2, seed=1)
        want = oracle.reconstruction_error(g, e.coords)
        fro = np.sqrt(np.sum(g * g))
        got = ds.reconstruction_error(g_lazy, e)
        assert abs(got - want) <= 1e-12 * fro
        got_x = ds.reconstruction_error(ds.matrix_from_host(g), e)
        assert abs(got_x - want) <= 1e-12 * fro
        if dim <= 10:
            assert got < 1e-8 * fro
    # truncated embedding of a higher-dimensional cloud: a large error, still exact
    pts = np.random.default_rng(3).standard_normal((400, 30))
    d = oracle.euclidean_matrix(pts)
    st, g = oracle.gram(d)
    gl = ds.gram(ds.matrix_from_host(d))
    e = ds.embed(gl, rank=4, oversampling=8, power_iters=2, seed=2)
    want = oracle.reconstruction_error(g, e.coords)
    assert ds.reconstruction_error(gl, e) == pytest.approx(want, rel=1e-12)
    # size mismatch (ref mds.cpp:128-129)
    other = ds.gram(ds.matrix_from_host(oracle.euclidean_matrix(pts[:100])))
    assert err(ds, ds.reconstruction_error, other, e) == ds.Status.ERR_SHAPE_MISMATCH


def test_workspace_reuse_large_then_small(ds, oracle):
    # panel rows past the last product row block must read as zero even when a
    # larger earlier solve left data in the reused workspace (BM = 128 for the
    # int8 kernel and for w > 64 in fp64)
    for w_rank, w_p in ((60, 10), (4, 4)):
        big = oracle.euclidean_matrix(ds.synth_points(2, 900, 1))
        ds.embed(ds.gram(ds.matrix_from_host(big)), rank=w_rank, oversampling=w_p, seed=3)
        n = 300  # 300 mod 256 = 44: one 128-row block short of the 256-row padding
        d = oracle.euclidean_matrix(ds.synth_points(2, n, 2))
        st, rm, grand = oracle.gram_stats(d)
        st, want, _, _ = oracle.eigs(w_rank, w_p, 2, 5, d=d, row_mean=rm, grand=grand,
                                     vectors=False)
        vals, _ = ds.eigs(ds.gram(ds.matrix_from_host(d)), rank=w_rank, oversampling=w_p,
                          power_iters=2, seed=5)
        np.testing.assert_allclose(vals[:8], want[:8], rtol=1e-9)


def test_int8_product_admission_and_f32(ds, oracle, product_path):
    # K2i admission (solver.cpp use_int8_product): finite data with a row
    # max/mean ratio <= 2^12 and w <= 128; otherwise the fp64 kernel runs
    if product_path != "int8":
        pytest.skip("int8-specific")
    n = 600
    pts = ds.synth_points(2, n, 4)
    d = oracle.euclidean_matrix(pts)
    k, p = 12, 8
    e8_d = ds.embed(ds.gram(ds.matrix_from_host(d)), rank=k, oversampling=p, seed=2)
    assert ds.stats_get().last_product_kernel == 1
    # f32 storage on the int8 path vs the fp64 kernel on the same f32 D
    d32 = d.astype(np.float32)
    e8 = ds.embed(ds.gram(ds.matrix_from_host_f32(d32)), rank=k, oversampling=p, seed=2)
    assert ds.stats_get().last_product_kernel == 1
    ds.set_product_path(1)
    e64 = ds.embed(ds.gram(ds.matrix_from_host_f32(d32)), rank=k, oversampling=p, seed=2)
    assert ds.stats_get().last_product_kernel == 0
    ds.set_product_path(2)
    np.testing.assert_allclose(e8.eigenvalues, e64.eigenvalues, rtol=1e-12)
    # the ratio bound 2^e_i / r_i is <= 2 n, so rejection needs n > 2048: a
    # tight cluster plus one far point gives rows with max d^2 ~ n * mean
    rng = np.random.default_rng(6)
    clu = rng.standard_normal((5000, 3)) * 1e-3
    clu[0] = (1e3, 0.0, 0.0)
    dfar = oracle.euclidean_matrix(clu)
    ds.embed(ds.gram(ds.matrix_from_host(dfar)), rank=k, oversampling=p, seed=2)
    assert ds.stats_get().last_product_kernel == 0
    # the same cluster without the outlier is admitted
    dclu = oracle.euclidean_matrix(clu[1:])
    ds.embed(ds.gram(ds.matrix_from_host(dclu)), rank=k, oversampling=p, seed=2)
    assert ds.stats_get().last_product_kernel == 1
    # non-finite data -> fp64 kernel; the NaN Ritz matrix fails the small
    # eigensolve like Eigen's (ref rsvd.cpp:113-114), without corrupting state
    dn = d.copy()
    dn[3, 5] = dn[5, 3] = np.inf
    assert err(ds, ds.embed, ds.gram(ds.matrix_from_host(dn)), rank=k, oversampling=p,
               seed=2) == ds.Status.ERR_INTERNAL
    assert ds.stats_get().last_product_kernel == 0
    again = ds.embed(ds.gram(ds.matrix_from_host(d)), rank=k, oversampling=p, seed=2)
    np.testing.assert_allclose(again.eigenvalues, e8_d.eigenvalues, rtol=1e-12)
    # 64 < w <= 128 (the GPU path's limit): int8 in two column groups
    ds.embed(ds.gram(ds.matrix_from_host(d)), rank=100, oversampling=20, seed=2)
    assert (ds.stats_get().last_product_kernel, ds.stats_get().last_product_groups) == (1, 2)


@pytest.mark.parametrize("rank,over", [(60, 10), (100, 20), (100, 28)])
def test_int8_column_groups_match_fp64(ds, oracle, rank, over):
    # w = 70 (wp 72): the CTA pair, 48 + 48 columns in ONE read of D;
    # w = 120, 128: two 64-column group passes
    n = 900
    d = oracle.euclidean_matrix(ds.synth_points(3, n, 7))
    g = ds.gram(ds.matrix_from_host(d))
    ds.set_product_path(2)
    try:
        e8 = ds.embed(g, rank=rank, oversampling=over, power_iters=2, seed=4)
        st = ds.stats_get()
        assert (st.last_product_kernel, st.last_product_groups) == (1, 2)
        assert st.last_product_pair == (1 if rank + over <= 96 else 0)
        ds.set_product_path(1)
        e64 = ds.embed(g, rank=rank, oversampling=over, power_iters=2, seed=4)
        assert ds.stats_get().last_product_kernel == 0
    finally:
        ds.set_product_path(0)
    assert e8.dims == e64.dims
    np.testing.assert_allclose(e8.eigenvalues[:40], e64.eigenvalues[:40], rtol=1e-10)
    np.testing.assert_allclose(e8.eigenvalues, e64.eigenvalues, rtol=1e-6)
    st_, rm, grand = oracle.gram_stats(d)
    want = oracle.embed(rank, over, 2, 4, d=d, row_mean=rm, grand=grand)
    np.testing.assert_allclose(e8.eigenvalues[:20], want["eigenvalues"][:20], rtol=1e-10)


def test_matrix_write_tsv_byte_identical(ds, oracle, ref, tmp_path):
    # ref src/distmat.cpp:224-244 through capi.cpp:270-282: index ids, the
    # shortest round-trip number format (textio.hpp:11-16)
    d = oracle.euclidean_matrix(ds.synth_points(1, 37, 3))
    ds.matrix_from_host(d).write_tsv(tmp_path / "ours.tsv")
    assert ref.write_matrix_tsv(tmp_path / "ref.tsv", d) == 0
    assert (tmp_path / "ours.tsv").read_bytes() == (tmp_path / "ref.tsv").read_bytes()
    # a gram handle writes G (as matrix_get / _write do)
    g = ds.gram(ds.matrix_from_host(d))
    g.write_tsv(tmp_path / "g.tsv", row_ids=[f"r{i}" for i in range(37)])
    lines = (tmp_path / "g.tsv").read_text().splitlines()
    assert lines[0].split("\t")[:3] == ["id", "0", "1"] and lines[1].startswith("r0\t")
    st, gref = oracle.gram(d)
    vals = np.array([[float(x) for x in ln.split("\t")[1:]] for ln in lines[1:]])
    assert np.max(np.abs(vals - gref)) <= 1e-13 * np.max(np.abs(gref))
    assert err(ds, g.write_tsv, tmp_path / "x.tsv", row_ids=["a"]) == ds.Status.ERR_SHAPE_MISMATCH


@pytest.mark.parametrize("n,rank,over", [(4095, 6, 2), (4096, 22, 10), (4097, 30, 3),
                                         (4225, 40, 25), (2049, 60, 5), (1153, 90, 38)])
def test_int8_tile_boundaries_match_fp64(ds, n, rank, over):
    # row counts around the 128-row block / 32-column k-step / 256-row padding
    # and panel widths around the 32 / 64 column-group edges (wp 8..128)
    d = ds.matrix_euclidean(ds.synth_points(2, n, n % 97))
    g = ds.gram(d)
    ds.set_product_path(2)
    try:
        e8 = ds.embed(g, rank=rank, oversampling=over, power_iters=1, seed=n)
        assert ds.stats_get().last_product_kernel == 1
        ds.set_product_path(1)
        e64 = ds.embed(g, rank=rank, oversampling=over, power_iters=1, seed=n)
    finally:
        ds.set_product_path(0)
    assert e8.dims == e64.dims
    top = min(e8.dims, 12)
    np.testing.assert_allclose(e8.eigenvalues[:top], e64.eigenvalues[:top], rtol=1e-10)
    from helpers import coords_match_up_to_sign
    assert coords_match_up_to_sign(e8.coords[:, :top], e64.coords[:, :top]) < \
        1e-7 * np.sqrt(e64.eigenvalues[0])


def test_handles_shared_across_threads(ds):
    # ref include/divscope.h:5-9: handles are immutable and shareable across
    # threads; the library serializes device work on its context and every
    # thread gets the same answer (ctypes drops the GIL inside the calls)
    import threading
    g = ds.gram(ds.matrix_euclidean(ds.synth_points(2, 3000, 8)))
    want = ds.embed(g, rank=8, oversampling=6, power_iters=2, seed=5)
    shared = ds.embed(g, rank=8, oversampling=6, power_iters=2, seed=5)
    out, errs = {}, []

    def work(t):
        try:
            e = ds.embed(g, rank=8, oversampling=6, power_iters=2, seed=5)
            out[t] = (e.eigenvalues.copy(), e.coords.copy(), shared.coords.copy())
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(repr(ex))

    th = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    for vals, coords, sh in out.values():
        assert np.array_equal(vals, want.eigenvalues)
        assert np.array_equal(coords, want.coords)
        assert np.array_equal(sh, want.coords)  # first-access download raced by 6 threads


@pytest.mark.parametrize("n,rank,over", [(1500, 10, 10), (2200, 30, 20)])
def test_int8_hamming_slices_match_fp64_and_oracle(ds, oracle, n, rank, over):
    # Hamming D (K7) on the int8 path slices the exact S = h^2 / L^2 into
    # three bytes (k2i_product.cu, SD = 3); NB = 32 and NB = 64 groups
    reads = ds.synth_reads(n, 400, 20, 0.05, n % 13)
    d = ds.matrix_hamming(reads)
    g = ds.gram(d)
    ds.set_product_path(2)
    try:
        e8 = ds.embed(g, rank=rank, oversampling=over, power_iters=2, seed=7)
        st = ds.stats_get()
        assert (st.last_product_kernel, st.last_product_sdigits) == (1, 3)
        ds.set_product_path(1)
        e64 = ds.embed(g, rank=rank, oversampling=over, power_iters=2, seed=7)
    finally:
        ds.set_product_path(0)
    assert e8.dims == e64.dims
    top = min(e8.dims, 15)
    np.testing.assert_allclose(e8.eigenvalues[:top], e64.eigenvalues[:top], rtol=1e-10)
    dm = d.to_numpy()
    st_, rm, grand = oracle.gram_stats(dm)
    want = oracle.embed(rank, over, 2, 7, d=dm, row_mean=rm, grand=grand)
    np.testing.assert_allclose(e8.eigenvalues[:top], want["eigenvalues"][:top], rtol=1e-10)
    assert coords_match_up_to_sign(e8.coords[:, :top], want["coords"][:, :top]) < \
        1e-7 * np.sqrt(want["eigenvalues"][0])


def test_hamming_builder_row_bands_and_errors(ds, oracle):
    # K7 full (upper-triangle tiles + mirror) and arbitrary row bands against
    # the oracle's popcount restatement; device-side validation reports the
    # first non-ACGT byte in read-major order
    reads = ds.synth_reads(333, 150, 7, 0.1, 9)
    st, want = oracle.hamming_counts(b"".join(reads), 333, 150)
    assert st == 0
    assert np.array_equal(ds.hamming_counts(reads), want)
    full = ds.matrix_hamming(reads).to_numpy()
    assert np.array_equal(full, want / 150.0)
    band = ds.matrix_hamming_rows(reads, 100, 301).to_numpy()
    assert np.array_equal(band, (want / 150.0)[100:301])
    bad = [bytearray(r) for r in reads]
    bad[200][17] = ord("N")
    bad[201][3] = ord("x")
    with pytest.raises(ds.DivscopeError) as ei:
        ds.matrix_hamming([bytes(r) for r in bad])
    assert ei.value.status == ds.Status.ERR_INVALID_CHARACTER
    assert "read 200" in ei.value.message and "base 18" in ei.value.message


def test_device_switch_refused_while_handles_live(ds, oracle, product_path):
    # one device per process: with handles holding device memory
    # a switch is refused, and the context keeps working on its device
    # (including the resident Omega panel, dropped with the workspace)
    d = oracle.euclidean_matrix(ds.synth_points(1, 300, 2))
    g = ds.gram(ds.matrix_from_host(d))
    a = ds.embed(g, rank=5, oversampling=5, power_iters=1, seed=3)
    with pytest.raises(ds.DivscopeError) as ei:
        ds.set_device(1)
    assert ei.value.status == ds.Status.ERR_INVALID_ARGUMENT
    ds.set_device(0)  # same device: a no-op
    b = ds.embed(g, rank=5, oversampling=5, power_iters=1, seed=3)
    assert np.array_equal(a.eigenvalues, b.eigenvalues)
    assert np.array_equal(a.coords, b.coords)
