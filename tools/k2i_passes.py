# Store pass vs streaming pass of the int8 product with the S-digit cache:
# python tools/k2i_passes.py n k p [euclid|f32|ham]
# Solves with q = 1 (4 product passes) and q = 3 (8 passes), CUDA-event times
# summed by the library; the difference is 4 streaming passes, the rest of
# the q = 1 solve is the storing pass plus 3 streaming ones.
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_02272_b200 as ds

n, k, p = (int(x) for x in sys.argv[1:4])
kind = sys.argv[4] if len(sys.argv) > 4 else "euclid"
ds.set_device(0)
ds.set_product_path(2)
if kind == "ham":
    D = ds.matrix_hamming(ds.synth_reads(n, 400, 50, 0.05, 3))
else:
    D = ds.matrix_euclidean(ds.synth_points(3, n, 3), store_f32=(kind == "f32"))
g = ds.gram(D)


def summed(q, reps=2):
    ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=1)
    ds.stats_enable_timing(True)
    ds.stats_reset()
    for _ in range(reps):
        ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=1)
    s = ds.stats_get()
    ds.stats_enable_timing(False)
    return s.product_ms / reps, s.product_launches / reps, s.last_product_sdig


for cache in (0, 2):
    ds.set_sdig_cache(cache)
    t1, l1, sd = summed(1)
    t3, l3, _ = summed(3)
    stream = (t3 - t1) / 4
    first = t1 - 3 * stream
    elem = n * n
    print(f"n={n} w={k + p} {kind} cache={cache} (used {sd}): first pass {first:.3f} ms, "
          f"later passes {stream:.3f} ms ({elem / (stream * 1e-3) / 1e9:.0f} G entries/s)")
