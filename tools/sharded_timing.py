"""Host-side breakdown of one row-sharded MDS step on a single-rank NCCL
communicator (the N>1 code path, its fixed overheads measured on one GPU)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1803_02272_b200 as ds  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
ds.set_device(0)
ds.comm_init(1, 0, ds.comm_unique_id())
pts = ds.synth_points(cfg, n, seed)
D = ds.matrix_euclidean_rows(pts, 0, n, store_f32=f32)
for _ in range(3):
    e = ds.embed(ds.gram(D), rank=k, oversampling=p, power_iters=q, seed=seed)
for it in range(3):
    t0 = time.perf_counter()
    g = ds.gram(D)
    t1 = time.perf_counter()
    e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
    t2 = time.perf_counter()
    print(f"sharded gram {1e3*(t1-t0):.3f} ms  embed {1e3*(t2-t1):.3f} ms  total {1e3*(t2-t0):.3f} ms")
ds.comm_destroy()
