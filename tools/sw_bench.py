"""Smith-Waterman pairwise_self throughput: GPU (sw.cu) vs the reference's
pairwise_self (oracle/_ref, all host threads) on C5-like reads (L = 400)."""
import os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import paper_1803_02272_b200 as ds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
n_cpu = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ds.set_device(0)
reads = ds.synth_reads(n, 400, 50, 0.05, 5)
cells = lambda m: m * (m - 1) / 2 * 400 * 400
ds.pairwise_self(reads[:64])  # warm-up
t = time.perf_counter(); D = ds.pairwise_self(reads); tg = time.perf_counter() - t
print(f"GPU  pairwise_self n={n}: {tg:.3f} s  {cells(n)/tg/1e9:.1f} GCUPS  ({n*(n-1)//2/tg:.0f} pairs/s)")
try:
    from oracle_bindings import RefLib
    ref = RefLib()
    th = os.cpu_count()
    t = time.perf_counter(); st, want = ref.pairwise_self(reads[:n_cpu], threads=th); tc = time.perf_counter() - t
    ok = np.array_equal(D.to_numpy()[:n_cpu, :n_cpu], want)
    print(f"CPU reference pairwise_self n={n_cpu} ({th} threads): {tc:.3f} s  {cells(n_cpu)/tc/1e9:.2f} GCUPS; "
          f"GPU block bit-identical: {ok}")
except FileNotFoundError as e:
    print("reference not available:", e)
