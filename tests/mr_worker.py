"""One rank of a multi-process run of the library's row-sharded path
(sharded.cpp) on ONE GPU, test infrastructure for tests/test_gpu_multirank.py.

The ranks talk through the host-staged transport (DSB_COMM_TRANSPORT=host,
comm.cpp): every collective synchronizes the stream, stages the buffer
through rank 0 over loopback sockets and copies the result back, so no
kernel ever waits on another process; only the collectives' transport
differs from NCCL, the sharded algorithm is the product code.

usage: python mr_worker.py WORLD RANK UID_FILE OUT.npz CASE_JSON
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1803_02272_b200 as ds  # noqa: E402


def share_uid(world, rank, path):
    if rank == 0:
        uid = ds.comm_unique_id()
        tmp = path + ".tmp"
        with open(tmp, "wb") as f:
            f.write(uid)
        os.replace(tmp, path)
        return uid
    t0 = time.time()
    while not os.path.exists(path):
        if time.time() - t0 > 120:
            raise SystemExit("rank %d: no uid from rank 0" % rank)
        time.sleep(0.02)
    return open(path, "rb").read()


def status_of(fn):
    try:
        fn()
        return 0
    except ds.DivscopeError as e:
        return int(e.status)


def main():
    world, rank = int(sys.argv[1]), int(sys.argv[2])
    uid_path, out = sys.argv[3], sys.argv[4]
    case = json.loads(sys.argv[5])
    ds.set_device(0)
    ds.set_product_path(case.get("product", 0))
    ds.comm_init(world, rank, share_uid(world, rank, uid_path))
    n, k, p, q, seed = case["n"], case["k"], case["p"], case["q"], case["seed"]
    rb, re_ = ds.shard_range(n, world, rank)
    res = {"rb": rb, "re": re_}
    kind = case["kind"]

    def shard():
        if kind == "hamming":
            reads = ds.synth_reads(n, case["length"], case["ancestors"], 0.05, case["data_seed"])
            return ds.matrix_hamming_rows(reads, rb, re_)
        if kind == "host_rows":
            d = np.load(case["d_path"])
            return ds.matrix_from_host_rows(np.ascontiguousarray(d[rb:re_]), n, rb, re_)
        pts = ds.synth_points(case["config"], n, case["data_seed"])
        return ds.matrix_euclidean_rows(pts, rb, re_, store_f32=case.get("f32", False))

    if case.get("fail") == "bad_rows" and rank == case.get("fail_rank", 1):
        # this rank hands in a shard that is not its range: it fails
        # validation; its peers must fail with it instead of hanging
        pts = ds.synth_points(case["config"], n, case["data_seed"])
        bad = ds.matrix_euclidean_rows(pts, 0, min(n, 100))
        res["status_gram"] = status_of(lambda: ds.gram(bad))
    elif case.get("fail") == "bad_rows":
        res["status_gram"] = status_of(lambda: ds.gram(shard()))
    if case.get("fail") == "seed_mismatch":
        g = ds.gram(shard())
        s = seed + (1 if rank == case.get("fail_rank", 1) else 0)
        res["status_embed"] = status_of(
            lambda: ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=s))
    if case.get("fail") == "not_symmetric":
        res["status_gram"] = status_of(lambda: ds.gram(shard()))
    else:
        # the communicator stays usable after a call failed on all ranks
        g = ds.gram(shard())
        e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
        res.update(eigenvalues=e.eigenvalues, coords=e.coords, dims=e.dims,
                   mass=e.dropped_negative_mass, truncated=int(e.truncated))
        vals, resid = ds.eigs(g, rank=k, oversampling=p, power_iters=q, seed=seed)
        res.update(eig_vals=vals, resid=resid)
        st = ds.stats_get()
        res.update(product_kernel=st.last_product_kernel, groups=st.last_product_groups,
                   sdig=st.last_product_sdig)
    ds.comm_destroy()
    np.savez(out, **{key: np.asarray(v) for key, v in res.items()})


if __name__ == "__main__":
    main()
