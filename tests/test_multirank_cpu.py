"""CPU tests of the multi-GPU decomposition with world_size 2 over gloo.

The product's N>1 path (paper_1803_02272_b200/csrc/sharded.cpp) row-shards D
with divscope_shard_range, replicates the panel, all-reduces the w x w Grams
and all-gathers the panel / row means. Here two CPU processes run exactly that
data flow (numpy stands in for the kernels, gloo for NCCL) on shards chosen by
the library's own divscope_shard_range, and the result must equal the
single-process oracle — i.e. the decomposition is exact up to rounding.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, k, p, q, seed, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import paper_1803_02272_b200 as ds
    from oracle_bindings import Oracle
    orc = Oracle()
    pts = ds.synth_points(1, n, seed)
    d_full = orc.euclidean_matrix(pts)
    rb, re = ds.shard_range(n, world, rank)
    d = d_full[rb:re]                               # this rank's rows only
    w = k + min(p, n - k)

    def allgather_rows(local):                      # grouped broadcasts (allgatherv)
        parts = []
        for r in range(world):
            b, e = ds.shard_range(n, world, r)
            t = torch.from_numpy(np.ascontiguousarray(local)) if r == rank else \
                torch.zeros((e - b,) + local.shape[1:], dtype=torch.float64)
            dist.broadcast(t, src=r)
            parts.append(t.numpy())
        return np.concatenate(parts, axis=0)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    # gram (pass 0): symmetry from the all-reduced antisymmetric fingerprint
    # of each rank's rows (k1_shard.cu), then local row sums, gathered row
    # means, grand mean in index order
    from helpers import sym_fingerprint

    def fp_total(rows):
        t = torch.tensor(sym_fingerprint(rows, rb), dtype=torch.int64)
        dist.all_reduce(t)                          # the two 32-bit halves, summed
        return tuple(int(x) % 2**32 for x in t)

    sym_ok = fp_total(d)
    bent = d.copy()
    if rank == 0:
        bent[3, n - 5] = np.nextafter(bent[3, n - 5], 1e9)  # mirror lives on rank 1
    sym_bent = fp_total(bent)
    r_full = allgather_rows((d * d).sum(1) / n)
    grand = r_full.sum() / n
    omega = orc.fill_gaussian(seed, n * w).reshape(n, w)  # replicated panel

    def product(x):                                 # K2 on the local rows
        s = x.sum(0)
        t = r_full @ x
        return -0.5 * ((d * d) @ x - np.outer(r_full[rb:re], s) - t + grand * s)

    def orth(y):                                    # CholeskyQR2 with all-reduced Grams
        for _ in range(2):
            wm = allreduce(y.T @ y)
            rr = np.linalg.cholesky(wm).T
            y = np.linalg.solve(rr.T, y.T).T
        return allgather_rows(y)

    x = orth(product(omega))
    for _ in range(q):
        x = orth(product(x))
        x = orth(product(x))
    z = product(x)
    b = allreduce(x[rb:re].T @ z)
    lam = np.linalg.eigvalsh(0.5 * (b + b.T))
    order = sorted(range(w), key=lambda a: (-abs(lam[a]), -lam[a]))
    vals = lam[order][:k]
    if rank == 0:
        out_q.put((vals.tolist(), sym_ok, sym_bent))
    dist.destroy_process_group()


def test_shard_ranges_partition(ds):
    for n in (1, 255, 256, 257, 2000, 20000, 100001):
        for world in (1, 2, 3, 4, 8):
            prev = 0
            chunk = -(-(-(-n // 256)) // world) * 256  # ceil(blocks / world) blocks
            for r in range(world):
                b, e = ds.shard_range(n, world, r)
                assert b == prev and e >= b
                assert b % 256 == 0 or b == e == n  # an empty tail rank starts at n
                # equal chunks (the panel all-gather moves one per rank);
                # only the tail is short, possibly empty
                assert e - b == chunk or e == n
                prev = e
            assert prev == n


@pytest.mark.timeout(300)
def test_two_rank_decomposition_matches_oracle(oracle, ds):
    n, k, p, q, seed = 700, 10, 10, 1, 3
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, k, p, q, seed, out_q))
             for r in range(2)]
    for pr in procs:
        pr.start()
    vals, sym_ok, sym_bent = out_q.get(timeout=240)
    assert sym_ok == (0, 0) and sym_bent != (0, 0)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    pts = ds.synth_points(1, n, seed)
    d = oracle.euclidean_matrix(pts)
    st, rm, grand = oracle.gram_stats(d)
    st, ref, _, _ = oracle.eigs(k, p, q, seed, d=d, row_mean=rm, grand=grand, vectors=False)
    assert st == 0
    np.testing.assert_allclose(vals, ref, rtol=1e-10)
