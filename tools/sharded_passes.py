"""Product-pass device time on the row-sharded code path (single-rank NCCL
communicator, one GPU) with the S-digit cache off and on: the first pass
stores each rank's planes, the later ones stream them.
python tools/sharded_passes.py [workload]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1803_02272_b200 as ds  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"  # Euclidean workloads
cfg, n, k, p, q, seed, f32 = bench.WORKLOADS[wl]
ds.set_device(0)
ds.comm_init(1, 0, ds.comm_unique_id())
D = ds.matrix_euclidean_rows(ds.synth_points(cfg, n, seed), 0, n, store_f32=f32)
g = ds.gram(D)
for cache in (0, 1):
    ds.set_sdig_cache(cache)
    ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
    ds.stats_enable_timing(True)
    ds.stats_reset()
    e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
    st = ds.stats_get()
    ds.stats_enable_timing(False)
    first = st.product_first_ms / max(st.product_first_launches, 1)
    later = (st.product_ms - st.product_first_ms) / max(st.product_launches - st.product_first_launches, 1)
    print(f"{wl} sharded (1 rank) cache={cache} sdig={st.last_product_sdig}: "
          f"first pass {first:.3f} ms, later passes {later:.3f} ms, "
          f"{st.product_launches} passes")
ds.comm_destroy()
