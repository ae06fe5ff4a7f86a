"""CPU tests: the oracle restatement pinned against the reference's own outputs.

The golden fixtures in tests/golden/ were produced by the reference sources
(oracle/_ref, see tests/golden/make_golden.py). Integer / byte / RNG work and
the reference loops that the oracle restates verbatim (gram, multiply_sym) must
match bit-for-bit; results that go through the QR / small EVD (Eigen in the
reference, restated in the oracle) match to the north-star tolerance.
"""
from pathlib import Path

import numpy as np
import pytest

from helpers import coords_match_up_to_sign, rel_err

G = Path(__file__).resolve().parent / "golden"
GOLDEN = G


def test_fill_gaussian_bit_exact(oracle):
    rng = np.load(G / "rng.npz")
    assert np.array_equal(oracle.fill_gaussian(7, 1001), rng["gauss_7_1001"])  # odd tail
    assert np.array_equal(oracle.fill_gaussian(0, 4096), rng["gauss_0_4096"])
    assert np.array_equal(oracle.fill_gaussian(42, 600), rng["gauss_42_30x20"])


def test_mt19937_64_known_answer():
    # the C++ standard pins std::mt19937_64's 10000th output for the default seed
    rng = np.load(G / "rng.npz")
    assert int(rng["mt_5489"][-1]) == 9981545732273789042


def test_euclid_and_gram_bit_exact(oracle):
    e = np.load(G / "euclid.npz")
    assert np.array_equal(oracle.euclidean_matrix(e["pts"]), e["d"])
    g = np.load(G / "gram.npz")
    st, gg = oracle.gram(e["d"])
    assert st == 0 and np.array_equal(gg, g["g"])
    assert np.array_equal(oracle.multiply_sym(g["g"], g["omega"]), g["prod"])
    st, rm, grand = oracle.gram_stats(e["d"])
    assert np.array_equal(oracle.multiply_gram_otf(e["d"], rm, grand, g["omega"]), g["prod"])
    st_lie, _ = oracle.gram(np.array([[0.0, 1.0], [2.0, 0.0]]))
    assert st_lie == int(g["status_asym"]) == 9  # NOT_SYMMETRIC


@pytest.mark.parametrize("name", ["diag_3m21", "diag_2m21", "dense60", "rank5_10"])
def test_eigs_matches_reference(oracle, name):
    k = np.load(G / "kats.npz")
    rank, p, q, seed = (int(x) for x in k[f"{name}__opts"])
    st, vals, _, resid = oracle.eigs(rank, p, q, seed, g=np.ascontiguousarray(k[f"{name}__g"]))
    assert st == 0
    assert rel_err(vals, k[f"{name}__vals"]) < 1e-10
    gm = k[f"{name}__g"]
    fro2 = float(np.sum(gm * gm))
    assert abs(resid ** 2 - float(k[f"{name}__resid"][0]) ** 2) <= 1e-12 * max(fro2, 1.0)


@pytest.mark.parametrize("name", ["euclid64", "noneucl4"])
def test_embed_matches_reference(oracle, name):
    k = np.load(G / "kats.npz")
    rank, p, q, seed = (int(x) for x in k[f"{name}__opts"])
    d = np.ascontiguousarray(k[f"{name}__d"])
    st, rm, grand = oracle.gram_stats(d)
    e = oracle.embed(rank, min(p, d.shape[0] - rank), q, seed, d=d, row_mean=rm, grand=grand)
    assert e["status"] == 0
    assert e["r"] == k[f"{name}__coords"].shape[1]
    assert e["truncated"] == bool(k[f"{name}__truncated"][0])
    assert rel_err(e["eigenvalues"], k[f"{name}__evals"]) < 1e-10
    assert coords_match_up_to_sign(e["coords"], k[f"{name}__coords"]) < 1e-9
    assert abs(e["dropped_negative_mass"] - float(k[f"{name}__mass"][0])) < 1e-10


def test_stable_rank_reference(oracle):
    k = np.load(G / "kats.npz")
    st, sr = oracle.stable_rank(np.diag([10.0, 5.0, 1.0]))
    assert st == 0 and sr == pytest.approx(float(k["stable_rank_diag"][0]), rel=1e-12)
    assert sr == pytest.approx(1.26, rel=1e-11)  # ref tests/test_rsvd.cpp:254


def test_hamming_oracle_on_reference_reads(oracle):
    reads = np.load(G / "reads.npz")["reads"]
    st, h = oracle.hamming_counts(reads.tobytes(), reads.shape[0], reads.shape[1])
    assert st == 0
    direct = (reads[:, None, :] != reads[None, :, :]).sum(-1)
    assert np.array_equal(h, direct.astype(np.uint32))
    assert np.all(np.diag(h) == 0) and np.array_equal(h, h.T)


# ---- ported reference KATs on the oracle (ref tests/test_rsvd.cpp, test_mds.cpp)

def test_oracle_kat_gram_two_point(oracle):
    st, g = oracle.gram(np.array([[0.0, 2.0], [2.0, 0.0]]))
    assert st == 0 and g.tolist() == [[1.0, -1.0], [-1.0, 1.0]]


def test_oracle_kat_errors(oracle):
    g = np.diag([1.0, 2.0, 3.0])
    assert oracle.eigs(3, 1, 2, 0, g=g)[0] == 10       # RANK_TOO_LARGE
    assert oracle.eigs(0, 1, 2, 0, g=g)[0] == 17       # INVALID_ARGUMENT
    assert oracle.eigs(1, 0, 2, 0, g=np.array([[0.0, 1.0], [2.0, 0.0]]))[0] == 9
    assert oracle.embed(3, 10, 2, 0, g=np.array([[1.0, -1.0], [-1.0, 1.0]]))["status"] == 10
    st, _ = oracle.gram(np.zeros((0, 0)))
    assert st == 2  # EMPTY_INPUT


def test_oracle_kat_two_points_embed(oracle):
    st, g = oracle.gram(np.array([[0.0, 2.0], [2.0, 0.0]]))
    e = oracle.embed(1, 1, 2, 0, g=g)
    assert e["eigenvalues"][0] == pytest.approx(2.0, rel=1e-12)
    assert e["coords"][:, 0] == pytest.approx([1.0, -1.0], rel=1e-10)


def test_oracle_thin_qr_orthonormal(oracle):
    y = oracle.fill_gaussian(4, 50 * 7).reshape(50, 7)
    q = oracle.thin_orthonormal(y)
    assert np.max(np.abs(q.T @ q - np.eye(7))) < 1e-13
    # same span
    assert np.linalg.norm(y - q @ (q.T @ y)) < 1e-12 * np.linalg.norm(y)


def test_oracle_matches_ref_directly(oracle, ref):
    """When oracle/_ref is present: random cross-check of the whole path."""
    pts = ref.uniform_box(150, 6, 9)
    d = ref.euclidean_matrix(pts)
    st, g = ref.gram(d)
    e_ref = ref.embed(g, 6, 10, 2, 4)
    st, rm, grand = oracle.gram_stats(d)
    e = oracle.embed(6, 10, 2, 4, d=d, row_mean=rm, grand=grand)
    assert rel_err(e["eigenvalues"], e_ref["eigenvalues"]) < 1e-12
    assert coords_match_up_to_sign(e["coords"], e_ref["coords"]) < 1e-10


def test_sw_oracle_matches_reference_fixture(oracle):
    # tests/golden/sw.npz from the reference's sw_align / pairwise_self
    z = np.load(GOLDEN / "sw.npz")
    cat, lens = z["cat"].tobytes(), z["lens"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    seqs = [cat[offs[i]:offs[i + 1]] for i in range(len(lens))]
    for row in z["aln"]:
        m, mm, g, i, j = (int(x) for x in row[:5])
        st, r6 = oracle.sw_align(seqs[i], seqs[j], (m, mm, g))
        assert st == 0 and r6 == tuple(int(x) for x in row[5:])
    n = len(seqs)
    for i in range(n):
        for j in range(n):
            if i != j:
                st, dist = oracle.sw_distance(seqs[i], seqs[j])
                assert st == 0 and dist == z["dself"][i, j]
    # error precedence (ref align.cpp:33-35): scheme first, then empty operands
    assert oracle.sw_align(b"", b"A")[0] == 6          # EMPTY_SEQUENCE
    assert oracle.sw_align(b"AC", b"A", (0, -1, -1))[0] == 17  # INVALID_ARGUMENT


def test_oracle_synthesis_matches_product(oracle, ds):
    # the reference arm of bench.py synthesizes its inputs with the oracle
    # (it must not load the product): both generators, bit for bit
    import numpy as np
    for cfg, n, seed in [(1, 257, 1), (2, 1000, 2), (3, 700, 3), (4, 333, 4)]:
        assert np.array_equal(oracle.synth_points(cfg, n, seed), ds.synth_points(cfg, n, seed))
    assert oracle.synth_reads(300, 400, 50, 0.05, 5) == ds.synth_reads(300, 400, 50, 0.05, 5)
    assert oracle.synth_reads(17, 33, 3, 0.2, 9) == ds.synth_reads(17, 33, 3, 0.2, 9)


def test_oracle_fast_helpers_match_definitions(oracle):
    # the packed Hamming matrix equals the plain character-count definition;
    # a row-range product equals those rows of the full pass, bit for bit
    import numpy as np
    reads = oracle.synth_reads(120, 77, 4, 0.1, 3)
    st, h = oracle.hamming_counts(b"".join(reads), 120, 77)
    assert st == 0
    assert np.array_equal(oracle.hamming_matrix_mt(reads, 77), h.astype(np.float64) / 77.0)
    d = oracle.euclidean_matrix_mt(oracle.synth_points(1, 300, 2))
    st, rm, grand = oracle.gram_stats(d)
    m = oracle.fill_gaussian(4, 300 * 9).reshape(300, 9)
    full = oracle.multiply_gram_otf(d, rm, grand, m)
    assert np.array_equal(oracle.multiply_gram_otf_rows(d, rm, grand, m, 37, 211), full[37:211])
