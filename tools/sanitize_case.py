"""Small classical-MDS runs that exercise every hand-written kernel of the
product path (K1 tile pairs, K2 DMMA, K2i int8 single-CTA and CTA-pair,
CholeskyQR, EVD, lift, K7 Hamming, K9 Euclid) for compute-sanitizer:
    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_case.py
(one tool per run; profiles/r02_sanitizer_*.txt)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_02272_b200 as ds  # noqa: E402

ds.set_device(0)
pts = ds.synth_points(1, 600, 3)
for path, (k, p) in [(1, (10, 10)), (2, (10, 10)), (2, (40, 30))]:
    ds.set_product_path(path)  # 1 fp64 DMMA, 2 int8 (w = 20: one CTA; w = 70: CTA pair)
    d = ds.matrix_euclidean(pts)
    e = ds.embed(ds.gram(d), rank=k, oversampling=p, power_iters=1, seed=1)
    print(f"path {path} w {k + p}: dims {e.dims} lambda_1 {e.eigenvalues[0]:.6g} "
          f"kernel {ds.stats_get().last_product_kernel}")
ds.set_product_path(2)
reads = ds.synth_reads(300, 400, 5, 0.05, 2)
e = ds.embed(ds.gram(ds.matrix_hamming(reads)), rank=8, oversampling=8, power_iters=1, seed=2)
print(f"hamming: dims {e.dims} sdigits {ds.stats_get().last_product_sdigits}")
f32 = ds.matrix_euclidean(pts, store_f32=True)
e = ds.embed(ds.gram(f32), rank=10, oversampling=10, power_iters=1, seed=1)
print(f"f32: dims {e.dims}")
print("sanitize case done")
