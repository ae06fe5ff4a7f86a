"""Device time per int8 K2 pass (k2i) on a workload, product path forced."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench, paper_1803_02272_b200 as ds
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
ds.set_device(0)
ds.set_product_path(2)
D = bench.make_distance(ds, wl)
g = ds.gram(D)
ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
ds.stats_enable_timing(True)
ds.stats_reset()
for _ in range(3):
    ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
s = ds.stats_get()
ms = s.product_ms / max(s.product_launches, 1)
print(f"{wl}: {ms*1e3:.1f} us/pass  {n*n*(4 if f32 else 8)/(ms*1e-3)/1e9:.0f} GB/s")
