"""Int8 slice product vs the fp64 DMMA product: eigenvalues, coordinates and
per-pass device time (run with DSB_K2_INT8=0/1 in two processes)."""
import os, subprocess, sys, json
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def one(wl, out):
    import bench, paper_1803_02272_b200 as ds
    ds.set_device(0)
    cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
    D = bench.make_distance(ds, wl)
    g = ds.gram(D)
    e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
    ds.stats_enable_timing(True)
    ds.stats_reset()
    for _ in range(3):
        e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
    s = ds.stats_get()
    np.savez(out, vals=e.eigenvalues, coords=e.coords, ms=s.product_ms / max(s.product_launches, 1),
             n=n)


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        one(sys.argv[2], sys.argv[3])
        sys.exit(0)
    for wl in sys.argv[1:] or ["C1", "C2", "C5"]:
        res = {}
        for mode in ("0", "2"):
            out = f"/tmp/i8_{wl}_{mode}.npz"
            env = dict(os.environ, DSB_K2_INT8=mode)
            subprocess.run([sys.executable, __file__, "--one", wl, out], check=True, env=env)
            res[mode] = np.load(out)
        a, b = res["0"], res["2"]
        rel = np.max(np.abs(a["vals"] - b["vals"]) / np.abs(a["vals"]))
        lam = a["vals"]
        cols = min(a["coords"].shape[1], b["coords"].shape[1])
        cd = np.max(np.abs(np.abs(a["coords"][:, :cols]) - np.abs(b["coords"][:, :cols])))
        n = int(a["n"])
        print(f"{wl}: eig rel diff {rel:.3e}; max |coord| diff {cd:.3e} (sqrt(l1) {np.sqrt(lam[0]):.3e}); "
              f"K2 fp64 {float(a['ms'])*1e3:.1f} us  int8 {float(b['ms'])*1e3:.1f} us/pass "
              f"({n*n*8/(float(b['ms'])*1e-3)/1e9:.0f} GB/s of D)")
