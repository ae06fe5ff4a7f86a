# Host vs device time of gram() and embed() per step (where the step's
# launch gaps come from): python tools/host_gaps.py [workload]
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench, paper_1803_02272_b200 as ds
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
ds.set_device(0)
D = bench.make_distance(ds, wl)
st = torch.cuda.ExternalStream(ds.stream_ptr())
for _ in range(3):
    ds.embed(ds.gram(D), rank=k, oversampling=p, power_iters=q, seed=seed)
torch.cuda.synchronize()
rows = []
for _ in range(10):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    h0 = time.perf_counter()
    e0.record(st)
    g = ds.gram(D)
    h1 = time.perf_counter()
    e1.record(st)
    e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
    e2.record(st)
    h2 = time.perf_counter()
    torch.cuda.synchronize()
    rows.append(((h1 - h0) * 1e3, (h2 - h1) * 1e3, e0.elapsed_time(e1), e1.elapsed_time(e2)))
import statistics as S
for name, i in (("gram host", 0), ("embed host", 1), ("gram device span", 2), ("embed device span", 3)):
    print(f"{name:20s} {S.median(r[i] for r in rows):.3f} ms")
