import ctypes as C, sys, torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench, paper_1803_02272_b200 as ds
ds.set_device(0)
buf = torch.zeros(64, dtype=torch.int64, device="cuda")
ds.lib.divscope_debug_orth_prof.argtypes = [C.c_void_p]
ds.lib.divscope_debug_orth_prof(buf.data_ptr())
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
D = ds.matrix_euclidean(ds.synth_points(cfg, n, seed))
for _ in range(3):
    e = ds.embed(ds.gram(D), rank=k, oversampling=p, power_iters=q, seed=seed)
torch.cuda.synchronize()
print([int(x) for x in buf.cpu().tolist()[:24]])
