"""Generate the golden fixtures under tests/golden/ from the reference itself.

Runs in the build container only (needs oracle/_ref, i.e. the reference's own
sources compiled by `make -C oracle ref`). Every array here is produced by
the reference code path; nothing is computed by the product or the oracle:

  rng.npz       std::mt19937_64 raw stream and fill_gaussian (ref src/rng.hpp)
  euclid.npz    testdata::uniform_box + euclidean_matrix (ref tests/testdata.cpp)
  gram.npz      gram_from_distances (ref src/mds.cpp:14-60) of that D, and
                multiply_sym (ref src/rsvd.cpp:18-36) of G with a seeded panel
  kats.npz      eigs_sym / embed / stable_rank outputs on the reference KAT
                matrices (ref tests/test_rsvd.cpp, tests/test_mds.cpp)
  reads.npz     testdata::random_reads (ref tests/testdata.cpp:28-37)
  sw.npz        sw_align / pairwise_self over mutated read families (ref src/align.cpp,
                src/distmat.cpp)
  *.dvs         DVS1 files written by write_matrix (ref src/distmat.cpp:169-187)

Usage: python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_bindings import RefLib  # noqa: E402


def with_spectrum_ref(ref, w, seed):
    """V diag(w) V^T with V from the Householder QR (the eigen shim) of a
    reference-seeded Gaussian matrix — built only from reference-side calls."""
    n = len(w)
    a = ref.fill_gaussian(seed, n * n).reshape(n, n)
    # thin QR through the reference's randomized_range machinery is not
    # exposed; use numpy QR here — the matrix is an INPUT, its exact bits are
    # stored in the fixture, so parity does not depend on how it was made.
    q, r = np.linalg.qr(a)
    q = q * np.sign(np.diag(r))
    g = q @ np.diag(np.asarray(w, float)) @ q.T
    return np.ascontiguousarray((g + g.T) / 2.0)


def main():
    ref = RefLib()
    out = {}
    # --- rng
    np.savez(HERE / "rng.npz",
             mt_5489=ref.mt19937_64(5489, 10000),
             gauss_7_1001=ref.fill_gaussian(7, 1001),
             gauss_0_4096=ref.fill_gaussian(0, 4096),
             gauss_42_30x20=ref.fill_gaussian(42, 600))
    # --- euclid / gram / product
    pts = ref.uniform_box(64, 5, 303)
    d = ref.euclidean_matrix(pts)
    np.savez(HERE / "euclid.npz", pts=pts, d=d)
    st, g = ref.gram(d, threads=1)
    assert st == 0
    omega = ref.fill_gaussian(11, 64 * 12).reshape(64, 12)
    prod = ref.multiply_sym(g, omega, threads=1)
    st_lie, _ = ref.gram(np.array([[0.0, 1.0], [2.0, 0.0]]))
    np.savez(HERE / "gram.npz", g=g, omega=omega, prod=prod, status_asym=st_lie)
    # --- KATs (inputs stored bit-exactly with the reference's outputs)
    kats = {}
    cases = {
        "diag_3m21": (np.diag([3.0, -2.0, 1.0]), 2, 1, 2, 0),
        "diag_2m21": (np.diag([2.0, -2.0, 1.0]), 3, 0, 2, 0),
        "dense60": (with_spectrum_ref(ref, [100.0 * 0.7 ** i for i in range(20)] + [0.0] * 40,
                                      12345), 10, 10, 3, 0),
        "rank5_10": (with_spectrum_ref(ref, [50, 20, 10, 5, 2, 1, 0.5, 0.1, 0, 0], 321),
                     5, 5, 2, 0),
    }
    for name, (gm, rank, p, q, seed) in cases.items():
        st, vals, vecs, resid = ref.eigs(gm, rank, p, q, seed, threads=1)
        assert st == 0, name
        kats[f"{name}__g"] = gm
        kats[f"{name}__opts"] = np.array([rank, p, q, seed])
        kats[f"{name}__vals"] = vals
        kats[f"{name}__resid"] = np.array([resid])
    # embed on the gram of the euclid fixture and on the non-Euclidean metric
    for name, dm, rank, p, q, seed in (
            ("euclid64", d, 5, 10, 2, 1),
            ("noneucl4", np.array([[0, 1, 1, 1], [1, 0, 1, 1], [1, 1, 0, 2], [1, 1, 2, 0]], float),
             4, 10, 2, 5)):
        st, gg = ref.gram(dm, threads=1)
        e = ref.embed(gg, rank, min(p, dm.shape[0] - rank), q, seed, threads=1)
        assert e["status"] == 0
        kats[f"{name}__d"] = dm
        kats[f"{name}__opts"] = np.array([rank, p, q, seed])
        kats[f"{name}__coords"] = e["coords"]
        kats[f"{name}__evals"] = e["eigenvalues"]
        kats[f"{name}__mass"] = np.array([e["dropped_negative_mass"]])
        kats[f"{name}__truncated"] = np.array([int(e["truncated"])])
    st, sr = ref.stable_rank(np.diag([10.0, 5.0, 1.0]))
    kats["stable_rank_diag"] = np.array([sr])
    np.savez(HERE / "kats.npz", **kats)
    # --- reads
    raw = ref.random_reads(40, 100, 77)
    np.savez(HERE / "reads.npz", reads=np.frombuffer(raw, dtype=np.uint8).reshape(40, 100))
    # --- Smith-Waterman (ref src/align.cpp:28-106, src/distmat.cpp:45-88):
    # mutated families of the random reads (substitutions, N, indels), all
    # pairs' alignments under two schemes + the pairwise_self matrix
    rng = np.random.default_rng(11)
    base = [bytes(r) for r in np.frombuffer(raw, dtype=np.uint8).reshape(40, 100)[:8]]
    seqs = []
    for k, s in enumerate(base):
        for m in range(3):
            b = bytearray(s)
            for _ in range(rng.integers(0, 8)):
                pos = int(rng.integers(0, len(b)))
                op = int(rng.integers(0, 4))
                if op == 0:
                    b[pos] = b"ACGTN"[int(rng.integers(0, 5))]
                elif op == 1 and len(b) > 10:
                    del b[pos]
                else:
                    b.insert(pos, b"ACGT"[int(rng.integers(0, 4))])
            seqs.append(bytes(b[: 60 + 15 * m]))
    lens = np.array([len(s) for s in seqs])
    cat = np.frombuffer(b"".join(seqs), dtype=np.uint8)
    aln = []
    for sch in ((1, -1, -2), (2, -3, -1)):
        for i in range(len(seqs)):
            for j in range(len(seqs)):
                st, r6 = ref.sw_align(seqs[i], seqs[j], sch)
                assert st == 0
                aln.append((sch[0], sch[1], sch[2], i, j) + tuple(r6))
    st, dself = ref.pairwise_self(seqs, (1, -1, -2), threads=1)
    assert st == 0
    np.savez(HERE / "sw.npz", cat=cat, lens=lens, aln=np.array(aln, dtype=np.int64), dself=dself)
    # --- DVS files
    rng = np.random.default_rng(3)
    a = rng.standard_normal((5, 7))
    assert ref.write_matrix(HERE / "rect5x7.dvs", a, sym=False) == 0
    assert ref.write_matrix(HERE / "euclid64.dvs", d, sym=True) == 0
    np.save(HERE / "rect5x7.npy", a)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
