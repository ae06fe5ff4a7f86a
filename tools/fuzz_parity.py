"""Randomized parity sweep (GPU vs the CPU oracle): random n, rank,
oversampling, storage dtype, product path and point configuration; eigenvalues
and coordinates compared at the north-star tolerances. Prints one line per
case and a summary; exits 1 on any mismatch."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import paper_1803_02272_b200 as ds
from helpers import coords_match_up_to_sign, rel_err
from oracle_bindings import Oracle

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
sharded = len(sys.argv) > 3 and sys.argv[3] == "sharded"  # single-rank NCCL, row-shard handles
orc = Oracle()
ds.set_device(0)
if sharded:
    ds.comm_init(1, 0, ds.comm_unique_id())
bad = 0
for c in range(cases):
    cfg = int(rng.integers(1, 5))
    n = int(rng.integers(300, 6000))
    rank = int(rng.integers(1, 60))
    over = int(rng.integers(0, min(128 - rank, 40) + 1))
    q = int(rng.integers(0, 3))
    f32 = bool(rng.integers(0, 2))
    path = int(rng.integers(0, 3))
    seed = int(rng.integers(0, 1000))
    pts = ds.synth_points(cfg, n, seed)
    d = orc.euclidean_matrix(pts)
    if f32:
        d = d.astype(np.float32).astype(np.float64)
    ds.set_product_path(path)
    try:
        if sharded:
            m = ds.matrix_from_host_rows_f32(d.astype(np.float32), n, 0, n) if f32 else \
                ds.matrix_from_host_rows(d, n, 0, n)
        else:
            m = ds.matrix_from_host_f32(d.astype(np.float32)) if f32 else ds.matrix_from_host(d)
        e = ds.embed(ds.gram(m), rank=rank, oversampling=over, power_iters=q, seed=seed)
        kern = ds.stats_get().last_product_kernel
    finally:
        ds.set_product_path(0)
    st, rm, grand = orc.gram_stats(d)
    want = orc.embed(rank, min(over, n - rank), q, seed, d=d, row_mean=rm, grand=grand)
    top = min(e.dims, want["r"], 10)
    ev = rel_err(e.eigenvalues[:top], want["eigenvalues"][:top]) if top else 0.0
    co = coords_match_up_to_sign(e.coords[:, :top], want["coords"][:, :top]) / \
        max(np.sqrt(abs(want["eigenvalues"][0])), 1e-300) if top else 0.0
    tol = 1e-4 if f32 else 1e-9
    ok = e.dims == want["r"] and ev < tol and co < (1e-3 if f32 else 1e-6)
    bad += not ok
    print(f"{'ok ' if ok else 'BAD'} cfg={cfg} n={n} rank={rank} p={over} q={q} f32={f32} "
          f"path={path} kernel={kern} dims={e.dims}/{want['r']} eig={ev:.1e} coords={co:.1e}",
          flush=True)
print(f"{cases - bad}/{cases} cases within tolerance{' (sharded path)' if sharded else ''}")
sys.exit(1 if bad else 0)
