"""The library's row-sharded path (sharded.cpp) run by 2, 3 and 4 real
processes (one rank each) on the test GPU, through the host-staged
collective transport (DSB_COMM_TRANSPORT=host, comm.cpp). This is the
device-count-invariance check that replaces the reference's thread-count
invariance (ref tests/test_rsvd.cpp:81-101): every rank's solve must match
the oracle and the one-process result.

Covered on real ranks: unequal shards (the last rank's padded panel chunk),
a rank with no rows at all, the panel all-gather (overlapped with the
product over each rank's own columns, and gather-first), the per-rank lift
partials and the coordinate all-gather, the ring-shift block exchange of
the symmetry check, both product kernels (fp64 DMMA and the int8 slice
product, two column groups), Hamming row shards, and errors: one rank
failing validation, ranks disagreeing on arguments, and an asymmetric D —
each returns an error on every rank instead of hanging."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import coords_match_up_to_sign, rel_err

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


def run_ranks(world, case, tmp_path, timeout=300, extra_env=None):
    uid = str(tmp_path / "uid.bin")
    env = dict(os.environ, DSB_COMM_TRANSPORT="host", **(extra_env or {}))
    procs, outs = [], []
    for r in range(world):
        out = str(tmp_path / f"rank{r}.npz")
        outs.append(out)
        procs.append(subprocess.Popen(
            [sys.executable, str(HERE / "mr_worker.py"), str(world), str(r), uid, out,
             json.dumps(case)], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    logs = []
    try:
        for pr in procs:
            o, _ = pr.communicate(timeout=timeout)
            logs.append(o.decode(errors="replace"))
    finally:
        for pr in procs:
            if pr.poll() is None:
                pr.kill()
    for r, pr in enumerate(procs):
        assert pr.returncode == 0, f"rank {r} exited {pr.returncode}:\n{logs[r][-3000:]}"
    return [dict(np.load(o)) for o in outs]


def one_process(ds, case):
    ds.set_product_path(case.get("product", 0))
    try:
        if case["kind"] == "hamming":
            reads = ds.synth_reads(case["n"], case["length"], case["ancestors"], 0.05,
                                   case["data_seed"])
            d = ds.matrix_hamming(reads)
        elif case["kind"] == "host_rows":
            d = ds.matrix_from_host(np.load(case["d_path"]))
        else:
            d = ds.matrix_euclidean(ds.synth_points(case["config"], case["n"], case["data_seed"]),
                                    store_f32=case.get("f32", False))
        return ds.embed(ds.gram(d), rank=case["k"], oversampling=case["p"],
                        power_iters=case["q"], seed=case["seed"])
    finally:
        ds.set_product_path(0)


def check_against(ds, oracle, case, res, tol_oracle=1e-10):
    ref1 = one_process(ds, case)
    sc = np.sqrt(ref1.eigenvalues[0])
    for r, out in enumerate(res):
        assert int(out["dims"]) == ref1.dims, r
        # identical across ranks (every rank solves the same EVD and gathers
        # the same coordinates)
        assert np.array_equal(out["eigenvalues"], res[0]["eigenvalues"])
        assert np.array_equal(out["coords"], res[0]["coords"])
        assert rel_err(out["eigenvalues"], ref1.eigenvalues) < 1e-12
        assert coords_match_up_to_sign(out["coords"], ref1.coords) < 1e-9 * sc
    if oracle is not None and case["kind"] in ("euclid", "host_rows") and not case.get("f32"):
        if case["kind"] == "host_rows":
            d = np.load(case["d_path"])
        else:
            d = oracle.euclidean_matrix(ds.synth_points(case["config"], case["n"],
                                                        case["data_seed"]))
        st, rm, grand = oracle.gram_stats(d)
        ref = oracle.embed(case["k"], case["p"], case["q"], case["seed"], d=d, row_mean=rm,
                           grand=grand)
        assert int(res[0]["dims"]) == ref["r"]
        assert rel_err(res[0]["eigenvalues"], ref["eigenvalues"]) < tol_oracle
        assert coords_match_up_to_sign(res[0]["coords"], ref["coords"]) < 1e-8 * sc
    return ref1


BASE = dict(kind="euclid", config=2, n=1300, data_seed=5, k=12, p=8, q=2, seed=7)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("product", [0, 2], ids=["auto", "int8"])
def test_ranks_match_oracle_and_one_process(ds, oracle, tmp_path, world, product):
    # n = 1300: 6 blocks of 256 -> shards 768 + 532 (world 2), 512 + 512 + 276
    # (world 3): unequal, the last chunk zero-padded in the panel
    case = dict(BASE, product=product)
    res = run_ranks(world, case, tmp_path)
    sizes = [int(o["re"]) - int(o["rb"]) for o in res]
    assert sum(sizes) == case["n"] and len(set(sizes)) > 1
    if product == 2:
        assert all(int(o["product_kernel"]) == 1 for o in res)
        # each rank stores its rows' S-digit planes in the first product pass
        # and streams them in the others (k-step ranges of the overlapped
        # gather index the items by global k-step)
        assert all(int(o["sdig"]) == 1 for o in res)
    check_against(ds, oracle, case, res)
    # eigs on the same sharded gram
    for o in res:
        assert rel_err(o["eig_vals"], res[0]["eigenvalues"][: len(o["eig_vals"])]) < 1e-12


@pytest.mark.parametrize("product", [0, 2], ids=["auto", "int8"])
def test_overlapped_gather_matches_gather_first(ds, oracle, tmp_path, product):
    # the panel all-gather overlapped with the product over each rank's own
    # columns (k-step ranges, one slot set each, colsums reduced from the
    # ranks' rows) against gather-then-product (DSB_SHARD_OVERLAP=0)
    case = dict(BASE, product=product)
    (tmp_path / "on").mkdir()
    (tmp_path / "off").mkdir()
    on = run_ranks(3, case, tmp_path / "on")
    off = run_ranks(3, case, tmp_path / "off", extra_env={"DSB_SHARD_OVERLAP": "0"})
    lam1 = on[0]["eigenvalues"][0]
    for a, b in zip(on, off):
        assert rel_err(a["eigenvalues"], b["eigenvalues"]) < 1e-12
        assert coords_match_up_to_sign(a["coords"], b["coords"]) < 1e-10 * np.sqrt(lam1)
    check_against(ds, oracle, case, on)


def test_rank_without_rows(ds, oracle, tmp_path):
    # n = 600 over 4 ranks: 256 + 256 + 88 + 0 rows
    case = dict(BASE, n=600, k=8, p=8, q=1)
    res = run_ranks(4, case, tmp_path)
    assert [int(o["re"]) - int(o["rb"]) for o in res] == [256, 256, 88, 0]
    check_against(ds, oracle, case, res)


def test_wide_panel_f32_two_column_groups(ds, tmp_path):
    # w = 70 > 64 on f32 storage: the int8 product in two column groups on
    # each rank's rows
    case = dict(BASE, n=1500, config=4, k=60, p=10, q=2, f32=True, product=2)
    res = run_ranks(2, case, tmp_path)
    assert all((int(o["product_kernel"]), int(o["groups"])) == (1, 2) for o in res)
    ref1 = one_process(ds, case)
    for o in res:
        np.testing.assert_allclose(o["eigenvalues"][:30], ref1.eigenvalues[:30], rtol=1e-10)
        np.testing.assert_allclose(o["eigenvalues"], ref1.eigenvalues, rtol=1e-6)


def test_hamming_row_shards(ds, tmp_path):
    case = dict(kind="hamming", n=900, length=400, ancestors=9, data_seed=3, k=8, p=8, q=2,
                seed=2, product=2)
    res = run_ranks(3, case, tmp_path)
    check_against(ds, None, case, res)


def test_tiny_asymmetry_takes_the_block_exchange(ds, oracle, tmp_path):
    # one mirrored pair one ulp apart: the fingerprint is nonzero, the ranks
    # ring-shift their off-diagonal blocks (sendrecv) and the reference's
    # 1e-12 tolerance accepts it
    n = 700
    d = oracle.euclidean_matrix(ds.synth_points(1, n, 4))
    near = d.copy()
    near[600, 10] = np.nextafter(near[600, 10], 1e9)  # rows of rank 2 vs rank 0
    path = tmp_path / "near.npy"
    np.save(path, near)
    case = dict(kind="host_rows", d_path=str(path), n=n, k=6, p=6, q=1, seed=1)
    res = run_ranks(3, case, tmp_path)
    clean = tmp_path / "clean.npy"
    np.save(clean, d)
    ref = one_process(ds, dict(case, d_path=str(clean)))
    for o in res:
        np.testing.assert_allclose(o["eigenvalues"], ref.eigenvalues, rtol=1e-10)


def test_asymmetry_fails_on_every_rank(ds, oracle, tmp_path):
    n = 700
    d = oracle.euclidean_matrix(ds.synth_points(1, n, 4))
    far = d.copy()
    far[650, 3] += 1e-9 * d.max()
    path = tmp_path / "far.npy"
    np.save(path, far)
    case = dict(kind="host_rows", d_path=str(path), n=n, k=6, p=6, q=1, seed=1,
                fail="not_symmetric")
    res = run_ranks(3, case, tmp_path)
    assert [int(o["status_gram"]) for o in res] == [int(ds.Status.ERR_NOT_SYMMETRIC)] * 3


@pytest.mark.parametrize("world", [2, 3])
def test_one_rank_fails_validation_all_return(ds, oracle, tmp_path, world):
    # rank 1 hands in the wrong rows: SHAPE_MISMATCH there, and the peers
    # return the same error instead of blocking in the first collective;
    # afterwards the communicator still runs a correct solve
    case = dict(BASE, fail="bad_rows")
    res = run_ranks(world, case, tmp_path)
    assert [int(o["status_gram"]) for o in res] == [int(ds.Status.ERR_SHAPE_MISMATCH)] * world
    check_against(ds, oracle, case, res)


def test_ranks_disagreeing_on_arguments_all_fail(ds, oracle, tmp_path):
    case = dict(BASE, fail="seed_mismatch")
    res = run_ranks(3, case, tmp_path)
    assert [int(o["status_embed"]) for o in res] == [int(ds.Status.ERR_INVALID_ARGUMENT)] * 3
    check_against(ds, oracle, case, res)
