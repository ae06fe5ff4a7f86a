import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_02272_b200 as ds
ds.set_device(0)
n = int(sys.argv[1]); f32 = len(sys.argv) > 2
D = ds.matrix_euclidean(ds.synth_points(2, n, 2), store_f32=f32)
for _ in range(3): ds.gram(D)
ds.stats_enable_timing(True); ds.stats_reset()
for _ in range(10): ds.gram(D)
st = ds.stats_get(); ms = st.stats_ms / st.stats_launches
print(f"K1 n={n} {'f32' if f32 else 'f64'}: {ms*1e3:.1f} us {n*n*(4 if f32 else 8)/(ms*1e-3)/1e9:.0f} GB/s")
