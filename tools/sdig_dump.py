# debug: compare the S-digit cache written by K1 with the one a storing pass
# writes, item by item (Hamming D: the bytes must agree)
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1803_02272_b200 as ds
n, k, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kind = sys.argv[4] if len(sys.argv) > 4 else "ham"
ds.set_device(0); ds.set_product_path(2)
if kind == "ham":
    D = ds.matrix_hamming(ds.synth_reads(n, 400, 20, 0.05, 3)); sd = 3
else:
    D = ds.matrix_euclidean(ds.synth_points(2, n, 3)); sd = 7
nblk, nks = (n + 127) // 128, (n + 31) // 32
nbytes = nblk * nks * sd * 4096
f = ds.lib.divscope_debug_sdig_read
f.argtypes = [C.c_void_p, C.c_size_t]
ds.set_sdig_cache(1)
g1 = ds.gram(D)
a = np.zeros(nbytes, np.uint8); print("read", f(a.ctypes.data, nbytes))
ds.set_sdig_cache(0); g0 = ds.gram(D); ds.set_sdig_cache(2)
ds.embed(g0, rank=k, oversampling=p, power_iters=0, seed=1)
print("sdig", ds.stats_get().last_product_sdig)
b = np.zeros(nbytes, np.uint8); print("read", f(b.ctypes.data, nbytes))
A = a.reshape(nblk, nks, 2, sd, 4, 64, 8); B = b.reshape(nblk, nks, 2, sd, 4, 64, 8)
rows = np.arange(nblk)[:, None] * 128 + np.arange(2)[None, :] * 64
diff = (A != B)
print("differing bytes", diff.sum(), "of", diff.size)
if diff.any():
    idx = np.argwhere(diff)
    print("first", idx[:10])
    for ax, name in enumerate(["rb", "ks", "half", "plane", "part", "row", "byte"]):
        print(name, np.unique(idx[:, ax])[:20])
