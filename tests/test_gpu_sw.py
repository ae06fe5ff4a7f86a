"""GPU Smith-Waterman distances (sw.cu) against the reference's own
sw_align / pairwise_self / pairwise_cross (oracle/_ref) and the golden
fixtures: bit-exact integer distances, scores and spans."""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def _golden_seqs():
    z = np.load(GOLDEN / "sw.npz")
    cat, lens = z["cat"].tobytes(), z["lens"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    return [cat[offs[i]:offs[i + 1]] for i in range(len(lens))], z


def err(ds, fn, *a, **k):
    try:
        fn(*a, **k)
    except ds.DivscopeError as e:
        return e.status
    return ds.Status.OK


def test_align_matches_golden(ds):
    seqs, z = _golden_seqs()
    for row in z["aln"][::7]:
        m, mm, g, i, j = (int(x) for x in row[:5])
        r = ds.align(seqs[i], seqs[j], ds.Scoring(m, mm, g))
        got = (r.score, r.distance, r.a_begin, r.a_end, r.b_begin, r.b_end)
        assert got == tuple(int(x) for x in row[5:])


def test_pairwise_self_matches_golden(ds):
    seqs, z = _golden_seqs()
    d = ds.pairwise_self(seqs)
    assert d.symmetric and d.rows == len(seqs)
    assert np.array_equal(d.to_numpy(), z["dself"])


def test_pairwise_and_distance_vs_reference(ds, ref):
    # C5-like reads: ancestors with 5 % substitutions, plus N, indels and
    # length variation; reference pairwise_self / pairwise_cross on the CPU
    rng = np.random.default_rng(5)
    reads = ds.synth_reads(90, 400, 6, 0.05, 3)
    seqs = []
    for k, r in enumerate(reads):
        b = bytearray(r)
        if k % 5 == 0:
            b[int(rng.integers(0, 400))] = ord("N")
        if k % 7 == 0:
            del b[int(rng.integers(0, 300)):int(rng.integers(300, 400))]
        if k % 11 == 0:
            b[50:50] = b"ACGTTGCA"
        seqs.append(bytes(b))
    st, want = ref.pairwise_self(seqs)
    assert st == 0
    got = ds.pairwise_self(seqs).to_numpy()
    assert np.array_equal(got, want)
    st, wx = ref.pairwise_cross(seqs[:17], seqs[40:], (2, -3, -1))
    assert st == 0
    gx = ds.pairwise_cross(seqs[:17], seqs[40:], ds.Scoring(2, -3, -1))
    assert (gx.rows, gx.cols, gx.symmetric) == (17, 50, False)
    assert np.array_equal(gx.to_numpy(), wx)
    for i, j in ((0, 1), (3, 77), (14, 2), (21, 21)):
        st, dw = ref.sw_distance(seqs[i], seqs[j])
        assert st == 0 and ds.distance(seqs[i], seqs[j]) == dw


def test_sw_errors(ds):
    # ref align.cpp:12-15, :33-35; distmat.cpp:37-41, :47-52, :92-97
    assert err(ds, ds.align, b"AC", b"A", ds.Scoring(0, -1, -1)) == ds.Status.ERR_INVALID_ARGUMENT
    assert err(ds, ds.align, b"", b"A") == ds.Status.ERR_EMPTY_SEQUENCE
    assert err(ds, ds.pairwise_self, [b"ACGT"]) == ds.Status.ERR_INVALID_ARGUMENT
    assert err(ds, ds.pairwise_self, [b"ACGT", b""]) == ds.Status.ERR_EMPTY_SEQUENCE
    assert err(ds, ds.pairwise_cross, [], [b"A"]) == ds.Status.ERR_INVALID_ARGUMENT
    assert err(ds, ds.pairwise_self, [b"AC", b"AG"], ds.Scoring(1, 1, -1)) == \
        ds.Status.ERR_INVALID_ARGUMENT
    # two identical reads: distance 0; disjoint alphabets: no positive alignment
    assert ds.pairwise_self([b"ACGTACGT", b"ACGTACGT"]).to_numpy()[0, 1] == 0
    r = ds.align(b"AAAA", b"CCCC")
    assert (r.score, r.distance, r.a_begin, r.a_end) == (0, 0, 0, 0)
    # 'N' never matches, itself included
    assert ds.align(b"NNNN", b"NNNN").score == 0


@pytest.mark.parametrize("scheme", [(81, -90, -60),     # forward-only kernel, |H| near 2^15
                                    (100, -150, -120),  # scores past 2^15: traceback kernel
                                    (1, -1, -1)])
def test_both_sw_kernels_vs_reference(ds, ref, scheme):
    # sw_plan picks k_sw_e (events carried forward) while every key fits
    # 32 bits and k_sw (stored traceback codes) otherwise; both bit-exact
    reads = ds.synth_reads(40, 400, 3, 0.08, 11)
    seqs = [bytes(r) if k % 3 else bytes(r[: 150 + 5 * k]) for k, r in enumerate(reads)]
    st, want = ref.pairwise_self(seqs, scheme)
    assert st == 0
    assert np.array_equal(ds.pairwise_self(seqs, ds.Scoring(*scheme)).to_numpy(), want)
    st, wx = ref.pairwise_cross(seqs[:9], seqs[9:], scheme)
    assert st == 0
    assert np.array_equal(ds.pairwise_cross(seqs[:9], seqs[9:], ds.Scoring(*scheme)).to_numpy(), wx)
