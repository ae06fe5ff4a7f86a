"""K2 tuning sweep: device ms per launch for several n / panel widths."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_02272_b200 as ds

ds.set_device(0)
peak = ds.fp64_tensor_peak_tflops(20000)
print(f"fp64 DMMA peak {peak:.2f} TF/s")
for n, f32 in ((20000, False), (20000, True)):
    pts = ds.synth_points(2, n, 2)
    D = ds.matrix_euclidean(pts, store_f32=f32)
    for wp in (8, 16, 32, 56, 72, 120, 128):
        for mode in (1, 0):
            ms = ds.bench_product(D, wp, mode, 5)
            tf = 2.0 * n * n * wp / (ms * 1e-3) / 1e12
            gbs = n * n * (4 if f32 else 8) / (ms * 1e-3) / 1e9
            print(f"n={n} f32={f32} wp={wp:3d} mode={mode}: {ms*1e3:8.1f} us  {tf:6.2f} TF/s "
                  f"({100*tf/peak:5.1f}% DMMA)  {gbs:7.1f} GB/s")
