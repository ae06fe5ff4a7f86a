# K7 A/B: matrix_hamming wall time at n = 50k, L = 400 (DSB_HAMMING_TC read
# once per process, so each arm is its own process)
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import numpy as np
    import torch
    import paper_1803_02272_b200 as ds
    n = int(sys.argv[1])
    reads = ds.synth_reads(n, 400, 50, 0.05, 5)
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        m = ds.matrix_hamming(reads)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
        del m
    print(f"TC={os.environ.get('DSB_HAMMING_TC','1')} n={n} matrix_hamming ms: "
          + " ".join(f"{x*1e3:.2f}" for x in ts))
    sys.exit(0)
for rep in range(2):
    for tc in ["0", "1"]:
        env = dict(os.environ, DSB_HAMMING_TC=tc, PYTHONPATH=os.getcwd())
        subprocess.run([sys.executable, __file__, "50000"], env=env, check=True)
