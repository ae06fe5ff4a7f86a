import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench, paper_1803_02272_b200 as ds
ds.set_device(0)
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]

D = bench.make_distance(ds, sys.argv[1] if len(sys.argv) > 1 else "C2")
for _ in range(3):
    e = ds.embed(ds.gram(D), rank=k, oversampling=p, power_iters=q, seed=seed)
buf = (C.c_longlong * 16)()
ds.lib.divscope_debug_evd_prof(buf)
print("total/phase1/phase2/conv/finish/sweeps", list(buf)[:6])
