"""Wall-clock breakdown of one e2e step (pinned host D -> coords) by phase."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench, paper_1803_02272_b200 as ds
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
torch.cuda.set_device(0)
ds.set_device(0)
D = bench.make_distance(ds, wl)
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
h.numpy()[...] = D.to_numpy()
del D
for mode in (0, 1):
    ds.set_product_path(mode)
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = ds.matrix_from_host(h.numpy())
        torch.cuda.synchronize(); t1 = time.perf_counter()
        g = ds.gram(m)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
        c = e.coords
        torch.cuda.synchronize(); t3 = time.perf_counter()
        del m, g, e
        torch.cuda.synchronize(); t4 = time.perf_counter()
        print(f"path={mode} it={it}: upload {1e3*(t1-t0):.1f} ms  gram {1e3*(t2-t1):.1f}  "
              f"embed+coords {1e3*(t3-t2):.1f}  free {1e3*(t4-t3):.1f}  total {1e3*(t4-t0):.1f}")
