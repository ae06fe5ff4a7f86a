"""Time the Hamming distance build (K7) for C5: reads (pinned host) ->
device packing -> D (f64, n x n) on the GPU, through the public API."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1803_02272_b200 as ds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
ds.set_device(0)
reads = ds.synth_reads(n, 400, 50, 0.05, 5)
rh = torch.empty((n, 400), dtype=torch.uint8, pin_memory=True)
rh.numpy()[...] = np.frombuffer(b"".join(reads), np.uint8).reshape(n, 400)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = ds.matrix_hamming(rh.numpy())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del d
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"n={n}: build {1e3*(t1-t0):.2f} ms ({n*n*8/(t1-t0)/1e9:.0f} GB/s of D written), free {1e3*(t2-t1):.2f} ms")
