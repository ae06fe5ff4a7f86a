"""stable_rank on the C2 gram: iterations, device ms per power-iteration pass,
and the GEMV pass's HBM rate (ref rsvd.cpp:147-178)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench, paper_1803_02272_b200 as ds
ds.set_device(0)
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
D = bench.make_distance(ds, sys.argv[1] if len(sys.argv) > 1 else "C2")
g = ds.gram(D)
ds.stable_rank(g)
ds.stats_enable_timing(True)
ds.stats_reset()
t = time.perf_counter()
sr = ds.stable_rank(g)
wall = time.perf_counter() - t
s = ds.stats_get()
iters = s.last_power_iters
ms = s.product_ms / max(iters, 1)
print(f"n={n} stable_rank={sr:.12g} passes={iters} wall={wall*1e3:.1f} ms "
      f"K2(wp=8) {ms*1e3:.1f} us/pass = {n*n*(4 if f32 else 8)/(ms*1e-3)/1e9:.0f} GB/s; "
      f"wall/pass {wall*1e3/max(iters,1)*1e3:.1f} us")
