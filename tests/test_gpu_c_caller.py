"""A plain C program compiled against include/divscope.h (tools/divscope_mds.c,
linked with libdivscope_b200.so) runs the reference CLI's `mds` and `spectrum`
flows (ref tools/divscope_main.cpp:267-304) on the GPU; its files and output
are compared with the reference's own flow (oracle/_ref: read_matrix,
gram_from_distances, embed, write_embedding_tsv / _meta compiled from the
reference sources) on the same DVS file. Coordinates are compared numerically
(the GPU's last bits differ), everything else exactly."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from helpers import coords_match_up_to_sign, rel_err

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
CALLER = ROOT / "tools" / "divscope_mds"
REF_MDS = ROOT / "oracle" / "_ref" / "ref_mds"  # the reference flow as an executable


@pytest.fixture(scope="module")
def caller():
    if not CALLER.exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_1803_02272_b200" / "csrc"), "caller"],
                       check=True)
    return str(CALLER)


def read_tsv(path):
    lines = Path(path).read_text().splitlines()
    header = lines[0].split("\t")
    ids, rows = [], []
    for ln in lines[1:]:
        f = ln.split("\t")
        ids.append(f[0])
        rows.append([float(x) for x in f[1:]])
    return header, ids, np.array(rows)


def read_meta(path):
    out = {}
    for ln in Path(path).read_text().splitlines():
        k, v = ln.split("=", 1)
        out[k] = v
    return out


def test_c_caller_mds_matches_reference_flow(caller, ds, ref, oracle, tmp_path):
    n, rank, p, q, seed = 600, 8, 10, 1, 7
    d = oracle.euclidean_matrix(ds.synth_points(1, n, 3))
    dvs = tmp_path / "d.dvs"
    assert ref.write_matrix(dvs, d) == 0  # the reference's DVS1 writer
    out = tmp_path / "gpu.tsv"
    r = subprocess.run([caller, "mds", str(dvs), str(out), str(rank), str(p), str(q), str(seed)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    if not REF_MDS.exists():
        pytest.skip("oracle/_ref/ref_mds not built (needs /root/reference at build time)")
    rtsv, rmeta = tmp_path / "ref.tsv", tmp_path / "ref.tsv.meta"
    r = subprocess.run([str(REF_MDS), str(dvs), str(rtsv), str(rank), str(p), str(q), str(seed)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    h1, ids1, x1 = read_tsv(out)
    h2, ids2, x2 = read_tsv(rtsv)
    assert h1 == h2 and ids1 == ids2 and x1.shape == x2.shape
    m1, m2 = read_meta(str(out) + ".meta"), read_meta(rmeta)
    assert m1.keys() == m2.keys()
    for k in m1:
        if k == "eigenvalues":
            e1 = np.array([float(v) for v in m1[k].split(",")])
            e2 = np.array([float(v) for v in m2[k].split(",")])
            assert rel_err(e1, e2) < 1e-10
        elif k == "dropped_negative_mass":
            assert float(m1[k]) == pytest.approx(float(m2[k]), abs=1e-9)
        else:
            assert m1[k] == m2[k], k
    lam1 = float(m2["eigenvalues"].split(",")[0])
    assert coords_match_up_to_sign(x1, x2) < 1e-8 * np.sqrt(lam1)
    # the library reads its own output back (divscope_embedding_load)
    e = ds.embedding_load(out)
    assert e.rows == n and e.dims == x1.shape[1]


def test_c_caller_spectrum_matches_reference(caller, ds, ref, oracle, tmp_path):
    n, rank, p, q, seed = 500, 12, 10, 2, 3
    d = oracle.euclidean_matrix(ds.synth_points(2, n, 5))
    dvs = tmp_path / "d.dvs"
    assert ref.write_matrix(dvs, d) == 0
    r = subprocess.run([caller, "spectrum", str(dvs), str(rank), str(p), str(q), str(seed)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    vals, resid, sr = [], None, None
    for ln in r.stdout.splitlines():
        f = ln.split("\t")
        if f[0] == "eigenvalue":
            vals.append(float(f[2]))
        elif f[0] == "resid":
            resid = float(f[1])
        elif f[0] == "stable_rank":
            sr = float(f[1])
    st, g = ref.gram(d)
    assert st == 0
    st, rvals, _, rresid = ref.eigs(g, rank, p, q, seed)
    assert st == 0 and len(vals) == len(rvals)
    assert rel_err(np.array(vals), rvals) < 1e-10
    fro2 = ref.frobenius_sq(g)
    assert abs(resid ** 2 - rresid ** 2) <= 1e-11 * fro2
    assert sr == pytest.approx(ref.stable_rank(g)[1], rel=1e-10)


def test_c_caller_reports_errors(caller, tmp_path):
    r = subprocess.run([caller, "mds", str(tmp_path / "missing.dvs"), str(tmp_path / "o.tsv")],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "io_error" in r.stderr
    bad = tmp_path / "bad.dvs"
    bad.write_bytes(b"NOPE" + bytes(28))
    r = subprocess.run([caller, "spectrum", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1 and "bad_format" in r.stderr
