"""DVS1 ingest throughput: streaming divscope_matrix_read vs the host-decode
path (dvs_read_host + matrix_from_host, the reference's two-copy pattern)."""
import os, sys, time, tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench, paper_1803_02272_b200 as ds
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
ds.set_device(0)
D = bench.make_distance(ds, wl)
path = Path(tempfile.gettempdir()) / f"dsb_{wl}.dvs"
t = time.perf_counter(); D.write(path); tw = time.perf_counter() - t
gb = path.stat().st_size / 1e9
for it in range(3):
    t = time.perf_counter(); m = ds.matrix_read(path); ts = time.perf_counter() - t
    del m
    t = time.perf_counter(); a, sym = ds.dvs_read_host(path); m = ds.matrix_from_host(a); th = time.perf_counter() - t
    del m, a
    print(f"{wl}: {gb:.2f} GB  streaming read {ts*1e3:.0f} ms ({gb/ts:.1f} GB/s)   host decode + upload {th*1e3:.0f} ms ({gb/th:.1f} GB/s)   [write {tw*1e3:.0f} ms]")
path.unlink()
