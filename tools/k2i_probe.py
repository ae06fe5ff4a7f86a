# K2i pass timing at an arbitrary (n, w): python tools/k2i_probe.py n k p [config] [f32]
import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_02272_b200 as ds
n, k, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = int(sys.argv[4]) if len(sys.argv) > 4 else 3
f32 = len(sys.argv) > 5 and sys.argv[5] == "f32"
ds.set_device(0); ds.set_product_path(2)
D = ds.matrix_euclidean(ds.synth_points(cfg, n, 3), store_f32=f32)
g = ds.gram(D)
ds.embed(g, rank=k, oversampling=p, power_iters=1, seed=1)
ds.stats_enable_timing(True); ds.stats_reset()
for _ in range(2):
    ds.embed(g, rank=k, oversampling=p, power_iters=1, seed=1)
s = ds.stats_get()
ms = s.product_ms / max(s.product_launches, 1)
print(f"n={n} w={k+p} groups={s.last_product_groups}: {ms*1e3:.1f} us/pass {n*n*(4 if f32 else 8)/(ms*1e-3)/1e9:.0f} GB/s")
