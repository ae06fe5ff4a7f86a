"""One device-resident MDS step (gram + embed) of a BASELINE workload, for
ncu launch lists / captures: warm-up steps first, then the profiled step."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import paper_1803_02272_b200 as ds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
wl = a.workload
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
ds.set_device(0)
D = bench.make_distance(ds, wl)
for _ in range(a.warmup + a.steps):
    e = ds.embed(ds.gram(D), rank=k, oversampling=p, power_iters=q, seed=seed)
st = ds.stats_get()
print("dims", e.dims, "lambda1", e.eigenvalues[0] if e.dims else None, "evd_sweeps", st.last_evd_sweeps, "shifted", st.last_orth_shifted)
