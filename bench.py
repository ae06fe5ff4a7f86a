#!/usr/bin/env python
"""bench.py — BASELINE.json metric "MDS distance entries/s per streaming pass;
achieved HBM GB/s as % of roofline" on the B200 path.

Workload: at N = 1 (default) C2 = BASELINE.json configs[1], the config quoted
for one GPU: n = 20,000 points from a seeded mixture of 20 Gaussian clusters
in R^50 (Dirichlet(1) weights), fp64 Euclidean D (3.2 GB), classical MDS with
k = 20, p = 10, q = 2. At N > 1 (torchrun) the default is C3 = configs[2]
(n = 100,000, 80 GB D, k 50, p 20, q 2) with n FIXED (strong scaling), D
row-sharded over the ranks. Inputs are seeded synthetic data generated with
the reference's RNG conventions.

One *step* = one full classical MDS of D through the public API:
  divscope_gram (pass 0: K1 reads D once) + divscope_embed (2q + 2 streaming
  product passes over D, CholeskyQR, Rayleigh-Ritz EVD, lift / sign / scale)
so a step makes 2q + 3 streaming passes over D, and
  value = n^2 * (2q + 3) * steps / time      [entries/s per streaming pass]
  e2e   = same metric through the C ABI from a pinned HOST copy of D: the
          host->device copy of D (the step's input) and the device->host read
          of the coordinates are inside the timed region. Omega is a pure
          function of (seed, n, w): the library generates it on the host once
          and keeps the device panel resident, so it is not re-uploaded.
D is larger than the 126 MB L2 at C2..C5, so every pass streams from HBM.
With the S-digit cache (default when it fits) the first
product pass of a solve also stores the exact digit planes of D o D and the
remaining 2q + 1 passes stream those (7 bytes per element, 3 for Hamming D)
instead of D; `roofline` then describes that streaming pass and carries the
storing pass as `store_pass`.

cpu_baseline (N = 1, rank 0) and --impl reference time the reference's own
CPU implementation of the path — gram_from_distances + embed (ref
src/mds.cpp:14-124, src/rsvd.cpp:18-145), compiled from the reference sources
into oracle/_ref — with every host thread. The reference arm synthesizes its
inputs with the oracle (never the product library). The N = 1 line also
carries `parity`: the timed GPU embedding against that reference embedding
(outside every timed region).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

WORKLOADS = {
    # name: (synth config, n, k, p, q, seed, fp32 storage)
    "C1": (1, 2000, 10, 10, 1, 1, False),
    "C2": (2, 20000, 20, 10, 2, 2, False),
    "C3": (3, 100000, 50, 20, 2, 3, False),
    "C4": (4, 200000, 100, 20, 3, 4, True),
    "C5": (5, 50000, 30, 20, 2, 5, False),   # Hamming D of 50k reads (L=400, 50 ancestors)
}
FP64_FALLBACK_TFLOPS = 37.1  # DMMA microbenchmark on this pool (profiles/fp64_peak_r01.txt)
INT8_PEAK_TOPS = 4533.5  # tcgen05 kind::i8, measured (profiles/r02_umma_seq.txt)


def make_distance(ds, wl: str):
    """Device-resident D of a workload (unsharded): Euclidean (K9) or Hamming (K7)."""
    cfg, n, k, p, q, seed, f32 = WORKLOADS[wl]
    if cfg == 5:
        return ds.matrix_hamming(ds.synth_reads(n, 400, 50, 0.05, seed))
    return ds.matrix_euclidean(ds.synth_points(cfg, n, seed), store_f32=f32)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML during the timed
    region, from a separate process (tools/nvml_sampler.py): NVML calls from
    a thread of this interpreter cost the timed region ~0.2 ms per step
    (measured), a sampler process nothing measurable."""

    def __init__(self, index: int, period_s: float = 0.02):
        self.index = index
        self.period = period_s
        self.samples: list = []
        self.error = None
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(
                [sys.executable, str(ROOT / "tools" / "nvml_sampler.py"), str(self.index),
                 str(self.period)], stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            if self._p.stdout.readline().strip() != "ready":
                raise RuntimeError("sampler did not start")
        except Exception as e:  # pragma: no cover - reported in the JSON
            self.error = repr(e)
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        try:
            out, _ = self._p.communicate("stop\n", timeout=30)
            got = json.loads(out.strip().splitlines()[-1])
            # drop the samples taken just before and just after the region
            self.samples = [tuple(x) for x in got[1:-1]] or [tuple(x) for x in got]
        except Exception as e:  # pragma: no cover
            self.error = repr(e)
            self._p.kill()

    def summary(self) -> dict:
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for name, b in bits.items() if s[2] & b})
        out = {"sm_mhz": float(np.median(sm)) if sm else None,
               "sm_max_mhz": max(s[1] for s in self.samples) if sm else None,
               "reasons": reasons, "samples": len(self.samples), "source": "nvml"}
        if self.error:
            out["error"] = self.error
        return out


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_ram_bytes() -> int:
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except Exception:  # pragma: no cover
        return 64 << 30


def host_distance(wl: str) -> np.ndarray:
    """D of a workload built on the host by the oracle (bit-identical to the
    device builders K9 / K7, pinned by the tests) — no product code."""
    from oracle_bindings import Oracle
    cfg, n, k, p, q, seed, f32 = WORKLOADS[wl]
    o = Oracle()
    if cfg == 5:
        return o.hamming_matrix_mt(o.synth_reads(n, 400, 50, 0.05, seed), 400)
    d = o.euclidean_matrix_mt(o.synth_points(cfg, n, seed))
    return d.astype(np.float32).astype(np.float64) if f32 else d


def reference_path(n: int):
    """The reference's own build when it is available and G fits next to D in
    host RAM (the reference materializes G), else the oracle port (G on the
    fly, same loops). Returns (lib, kind)."""
    from oracle_bindings import Oracle, RefLib, ref_available
    if ref_available() and 2 * n * n * 8 < 0.45 * host_ram_bytes():
        return RefLib(), "reference"
    return Oracle(), "port"


def reference_step(lib, kind, d, k, p, q, seed, cores):
    """One step of the reference CPU path: gram_from_distances + embed."""
    if kind == "reference":
        st, g = lib.gram(d, threads=cores)
        assert st == 0, "reference gram failed"
        e = lib.embed(g, k, p, q, seed, threads=cores)
        del g
    else:
        st, rm, grand = lib.gram_stats(d)
        assert st == 0
        e = lib.embed(k, p, q, seed, d=d, row_mean=rm, grand=grand)
    assert e["status"] == 0, "reference embed failed"
    return e


def parity_block(e, ref) -> dict:
    """The GPU embedding of the timed region against the reference's."""
    from helpers import coords_match_up_to_sign, rel_err, sin_subspace
    out = {"against": "reference gram_from_distances + embed (oracle/_ref)",
           "dims": [int(e.dims), int(ref["r"])]}
    if e.dims == ref["r"] and e.dims:
        lam1 = float(ref["eigenvalues"][0])
        out.update(eig_max_rel_err=float(rel_err(e.eigenvalues, ref["eigenvalues"])),
                   coord_max_err_over_sqrt_lambda1=float(
                       coords_match_up_to_sign(e.coords, ref["coords"]) / math.sqrt(lam1)),
                   sin_theta=float(sin_subspace(e.coords, ref["coords"])),
                   dropped_negative_mass=[float(e.dropped_negative_mass),
                                          float(ref["dropped_negative_mass"])])
        out["ok"] = bool(out["eig_max_rel_err"] < 1e-10 and
                         out["coord_max_err_over_sqrt_lambda1"] < 1e-8)
    else:
        out["ok"] = False
    return out


def cpu_sample(d, wl: str, budget_s: float = 20.0):
    """cpu_baseline on a bounded sample: the full reference step when it fits
    the budget (then also the reference embedding for the parity block),
    else one reference product pass over a block of rows (entries/s per
    pass over the block). Returns (baseline dict, reference embedding|None)."""
    cfg, n, k, p, q, seed, f32 = WORKLOADS[wl]
    cores = os.cpu_count() or 1
    passes = 2 * q + 3
    w = k + min(p, n - k)
    lib, kind = reference_path(n)
    if n <= 20000:
        t0 = time.perf_counter()
        ref = reference_step(lib, kind, d, k, p, q, seed, cores)
        t = time.perf_counter() - t0
        return ({"value": n * n * passes / t, "unit": "entries/s", "cores": cores, "kind": kind,
                 "sample": f"one full reference step at {wl}: gram_from_distances + embed "
                           f"(n={n}, k={k}, p={p}, q={q}; {passes} passes incl. the gram), "
                           f"{cores} threads, {t:.1f} s"}, ref)
    from oracle_bindings import Oracle
    o = Oracle()
    st, rm, grand = o.gram_stats(d)
    omega = o.fill_gaussian(seed, n * w).reshape(n, w)
    rows = 256
    t = 0.0
    while True:  # grow the row block until the sample takes ~2 s (capped)
        t0 = time.perf_counter()
        o.multiply_gram_otf_rows(d, rm, grand, omega, 0, rows, threads=cores)
        t = time.perf_counter() - t0
        if t > 2.0 or rows >= n or t * (n / rows) < budget_s:
            break
        rows = min(n, rows * 4)
    return ({"value": rows * n / t, "unit": "entries/s", "cores": cores, "kind": "port",
             "sample": f"reference product pass (multiply_sym over the on-the-fly gram, "
                       f"ref src/rsvd.cpp:18-36) over rows 0..{rows} of {wl} (n={n}, w={w}), "
                       f"{cores} threads, {t:.2f} s; gram stats untimed"}, None)


def reference_arm(args, wl):
    """--impl reference: the reference's own CPU path on the host cores (rank
    0 only under torchrun). Each step is one full gram_from_distances + embed;
    the number of timed steps is bounded so the run stays within minutes."""
    world, rank, _ = dist_init()
    cfg, n, k, p, q, seed, f32 = WORKLOADS[wl]
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    passes = 2 * q + 3
    d = host_distance(wl)
    if n <= 20000:
        lib, kind = reference_path(n)
        t0 = time.perf_counter()
        reference_step(lib, kind, d, k, p, q, seed, cores)  # warm-up (page cache, threads)
        t_w = time.perf_counter() - t0
        steps = max(1, min(args.steps, int(150.0 / max(t_w, 1e-3))))
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            reference_step(lib, kind, d, k, p, q, seed, cores)
            times.append(time.perf_counter() - t0)
        t = float(np.mean(times))
        value = n * n * passes / t
        sample = (f"{steps} x (gram_from_distances + embed) at {wl}, n={n}, k={k}, p={p}, "
                  f"q={q}, {cores} threads ("
                  f"{'oracle/_ref: the reference sources' if kind == 'reference' else 'oracle port, G on the fly'})")
    else:
        # a full reference step at this n takes minutes to hours (and G would
        # not fit next to D): each step is the reference product pass over a
        # block of rows, timed as entries/s per pass
        base, _ = cpu_sample(d, wl, budget_s=5.0)
        kind, steps = base["kind"], 1
        value = base["value"]
        t = passes * n * n / value  # a full step at the sampled rate (extrapolated)
        sample = base["sample"] + f"; ms_per_step extrapolated to {passes} full passes"
    line = {
        "impl": "reference", "metric": "MDS distance entries/s per streaming pass",
        "value": value, "unit": "entries/s", "n_gpus": args.gpus, "steps": steps,
        "steps_requested": args.steps, "warmup": 1, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, reference RNG conventions; built by the oracle on the host)",
        "config": {"workload": wl, "n": n, "k": k, "p": p, "q": q, "seed": seed,
                   "d_dtype": "f32" if f32 else "f64", "streaming_passes_per_step": passes,
                   "step": "reference gram_from_distances + embed on the host cores"},
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def b200_arm(args, wl):
    import torch
    world, rank, local = dist_init()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import paper_1803_02272_b200 as ds
    ds.set_device(torch.cuda.current_device())
    cfg, n, k, p, q, seed, f32 = WORKLOADS[wl]
    n1 = n
    sharded = world > 1 or args.force_sharded
    if sharded and args.weak:
        # weak scaling (opt-in): every GPU streams the same n1^2 entries of D
        # per pass, the matrix grows as n = n1 sqrt(N)
        n = int(round(n1 * math.sqrt(world)))
    w = k + min(p, n - k)
    passes = 2 * q + 3
    stream = torch.cuda.ExternalStream(ds.stream_ptr())
    if sharded:
        # one NCCL communicator over the box; D row-sharded
        obj = [ds.comm_unique_id() if rank == 0 else None]
        if world > 1:
            torch.distributed.broadcast_object_list(obj, src=0)
        ds.comm_init(world, rank, obj[0])

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # ---- inputs: D built on the device (K9), host copy for the e2e leg
    rb, re_ = ds.shard_range(n, world, rank) if sharded else (0, n)
    reads_host = None
    if cfg == 5:
        # C5's input is the reads: D is built on the GPU by K7 (a row shard
        # per rank); the e2e leg uploads the reads, not a 20 GB matrix
        reads = ds.synth_reads(n, 400, 50, 0.05, seed)
        reads_host = torch.empty((n, 400), dtype=torch.uint8, pin_memory=True)
        reads_host.numpy()[...] = np.frombuffer(b"".join(reads), np.uint8).reshape(n, 400)
        del reads
        D = ds.matrix_hamming_rows(reads_host.numpy(), rb, re_) if sharded else \
            ds.matrix_hamming(reads_host.numpy())
    else:
        pts = ds.synth_points(cfg, n, seed)
        D = ds.matrix_euclidean_rows(pts, rb, re_, store_f32=f32) if sharded else \
            ds.matrix_euclidean(pts, store_f32=f32)
    if not args.no_e2e and cfg != 5:
        d_host = torch.empty((re_ - rb, n), dtype=torch.float32 if f32 else torch.float64,
                             pin_memory=True)
        d_np = d_host.numpy()
        d_np[...] = D.to_numpy().astype(d_np.dtype)  # this rank's rows
    fp64_peak = ds.fp64_tensor_peak_tflops(20000)
    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))

    def step_device():
        g = ds.gram(D)
        e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
        return e

    def step_e2e():
        if cfg == 5:
            rh = reads_host.numpy()
            m = ds.matrix_hamming_rows(rh, rb, re_) if sharded else ds.matrix_hamming(rh)
            g = ds.gram(m)
            e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
            return e.coords
        if sharded:
            m = (ds.matrix_from_host_rows_f32 if f32 else ds.matrix_from_host_rows)(
                d_np, n, rb, re_)
        else:
            m = ds.matrix_from_host_f32(d_np) if f32 else ds.matrix_from_host(d_np)
        g = ds.gram(m)
        e = ds.embed(g, rank=k, oversampling=p, power_iters=q, seed=seed)
        c = e.coords  # result on the host
        return c

    # ---- device-resident leg
    for _ in range(max(3, args.warmup)):
        step_device()
    ds.stats_enable_timing(True)
    torch.cuda.synchronize()
    barrier()
    ds.stats_reset()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            e = step_device()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    t_ms = ev0.elapsed_time(ev1)
    st = ds.stats_get()
    ds.stats_enable_timing(False)
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = n * n * passes * args.steps / (t_ms * 1e-3)

    # ---- roofline of the dominant kernel (K2, the centered product pass)
    k2_ms = st.product_ms / max(st.product_launches, 1)
    m_rows = re_ - rb  # rows of D this rank streams per product pass
    bytes_per_launch = m_rows * n * (4 if f32 else 8) + n * w * 8 + m_rows * w * 8 + m_rows * 8
    # with the S-digit cache (k2i_product.cu) the solve's first pass reads D
    # and stores the digit planes of D o D (SD bytes per element of each
    # 128-row x 32-column item), the other 2q+1 passes — the dominant kernel —
    # stream those planes instead of D
    # (last_product_sdig 2: K1 — pass 0, the gram — wrote the planes while
    # reading D, and every product pass streams them)
    sdig_mode = int(st.last_product_sdig) if int(st.last_product_kernel) == 1 else 0
    sdig = sdig_mode >= 1
    store_pass = None
    item_bytes = ((m_rows + 127) // 128) * ((n + 31) // 32) * int(st.last_product_sdigits) * 4096
    if sdig_mode == 2:
        bytes_per_launch = item_bytes + n * w * 8 + m_rows * w * 8 + m_rows * 8
    if sdig_mode == 1:
        nfirst = max(int(st.product_first_launches), 1)
        first_ms = st.product_first_ms / nfirst
        k2_ms = (st.product_ms - st.product_first_ms) / max(int(st.product_launches) - nfirst, 1)
        d_bytes = m_rows * n * (4 if f32 else 8)
        bytes_per_launch = item_bytes + n * w * 8 + m_rows * w * 8 + m_rows * 8
        store_bytes = d_bytes + item_bytes + n * w * 8 + m_rows * w * 8 + m_rows * 8
        store_pass = {"launches_per_step": 1, "avg_ms": first_ms,
                      "bytes_per_launch": store_bytes,
                      "achieved_gbs": store_bytes / (first_ms * 1e-3) / 1e9,
                      "what": "reads D, stores the S digit planes (and runs the product)"}
    flops_per_launch = 2.0 * m_rows * n * w
    tflops = flops_per_launch / (k2_ms * 1e-3) / 1e12
    gbs = bytes_per_launch / (k2_ms * 1e-3) / 1e9
    int8_path = int(st.last_product_kernel) == 1
    kname = "k2i_product" if int8_path else "k2_product"
    traffic = None
    tp = ROOT / "profiles" / "k2_traffic.json"
    if tp.exists():
        try:
            tv = json.loads(tp.read_text()).get(wl)
            traffic = tv.get(kname) if isinstance(tv, dict) else (None if int8_path else tv)
            if store_pass is not None and isinstance(tv, dict):
                store_pass["traffic"] = tv.get("k2i_product_store")
        except Exception:
            traffic = None
    hbm = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
           "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
           else "fallback 6650 GB/s (B200_PROFILING.md)"}
    common = {"k2_avg_ms": k2_ms, "k2_launches": int(st.product_launches),
              "sdig_cache": ("written by K1 (pass 0)" if sdig_mode == 2 else
                             "stored by the first product pass" if sdig_mode == 1 else None),
              "store_pass": store_pass,
              "flops_per_launch": flops_per_launch, "bytes_per_launch": bytes_per_launch,
              "pass0": {"k1_avg_ms": st.stats_ms / max(st.stats_launches, 1),
                        "achieved_gbs": (m_rows * n * (4 if f32 else 8) +
                                         (item_bytes if sdig_mode == 2 else 0)) /
                        (st.stats_ms / max(st.stats_launches, 1) * 1e-3) / 1e9,
                        "writes_digit_planes_bytes": item_bytes if sdig_mode == 2 else 0}}
    if int8_path:
        # exact integer slice product on the int8 tensor cores: one read of D
        # per column group (w <= 64: one group), HBM-bound; `achieved` counts
        # the pass's algorithmic bytes (D once), `streamed_gbs` every read
        groups = max(int(st.last_product_groups), 1)
        # the int8 tensor roof of the same pass: digit products x MMA columns
        # (k2i_plan: WP <= 32 one 32-wide group, <= 64 one 64-wide, <= 96 a
        # CTA pair of 48 + 48, else 64 + 64), at the measured kind::i8 peak
        wpad = (w + 7) // 8 * 8
        mma_cols = 32 if wpad <= 32 else 64 if wpad <= 64 else 96 if wpad <= 96 else 128
        products = 18 if int(st.last_product_sdigits) == 3 else 28
        i8_ops = 2.0 * m_rows * n * mma_cols * products
        i8_ms = i8_ops / (INT8_PEAK_TOPS * 1e12) * 1e3
        hbm_ms = bytes_per_launch / (hbm_peak * 1e9) * 1e3 * (groups if wpad > 96 else 1)
        binding = "int8" if i8_ms > hbm_ms else "hbm"
        roofline = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": gbs / hbm_peak, "traffic": traffic,
                    "binding_roof": {"bound": binding, "roof_ms": max(i8_ms, hbm_ms),
                                     "frac": max(i8_ms, hbm_ms) / k2_ms,
                                     "hbm_ms": hbm_ms, "int8_ms": i8_ms,
                                     "int8_ops_per_launch": i8_ops,
                                     "int8_peak_tops": INT8_PEAK_TOPS,
                                     "int8_peak_source": "profiles/r02_umma_seq.txt (7 x N=256 kind::i8 MMAs, A in TMEM)"},
                    "kernel": ("k2i_product (3x7-digit int8 slice product of the exact Hamming "
                               "h^2, tcgen05 kind::i8)" if int(st.last_product_sdigits) == 3 else
                               "k2i_product (7x7-digit int8 slice product, tcgen05 kind::i8)") +
                              (", streaming the S-digit cache" if sdig else ""),
                    "peak_source": hbm["peak_source"],
                    **({"peak_note": "frac > 1: the peak is MEASURED_PEAKS.json's device copy "
                                     "(read + write traffic); this pass is a pure read stream of "
                                     "the S-digit planes, which HBM serves faster — ncu DRAM bytes "
                                     "for the same kernel: 2.818 GB read in 0.416 ms (profiles/"
                                     "r02_final_ncu_k2i_c2_stream.txt, k2_traffic.json)"}
                       if gbs > hbm_peak else {}),
                    "column_groups": groups,
                    "reads_of_D_per_pass": 1 if int(st.last_product_pair) else groups,
                    "cta_pair": bool(int(st.last_product_pair)),
                    "s_slices": int(st.last_product_sdigits),
                    "streamed_gbs": gbs * groups if groups > 1 else gbs,
                    "fp64_equiv": {"achieved": tflops, "unit": "TFLOP/s",
                                   "fp64_dmma_peak": fp64_peak}, **common}
    else:
        roofline = {"bound": "tensor", "achieved": tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": tflops / fp64_peak, "traffic": traffic,
                    "kernel": "k2_product (DMMA f64) — FP64-bound at this w; HBM shown alongside",
                    "peak_source": "live f64 DMMA microbenchmark (divscope_fp64_tensor_peak_tflops)",
                    "hbm": hbm, **common}

    # ---- e2e leg through the C ABI from pinned host memory
    e2e = None
    if not args.no_e2e:
        step_e2e()
        torch.cuda.synchronize()
        barrier()
        ds.stats_reset()
        ev2 = torch.cuda.Event(enable_timing=True)
        ev3 = torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        for _ in range(args.steps):
            step_e2e()
        ev3.record(stream)
        torch.cuda.synchronize()
        barrier()
        te_ms = ev2.elapsed_time(ev3)
        st2 = ds.stats_get()
        if world > 1:
            tt = torch.tensor([te_ms], device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te_ms = float(tt.item())
        e2e = {"value": n * n * passes * args.steps / (te_ms * 1e-3), "unit": "entries/s",
               "h2d_bytes_per_step": int(st2.h2d_bytes // max(args.steps, 1)),
               "d2h_bytes_per_step": int(st2.d2h_bytes // max(args.steps, 1))}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dd = D.to_numpy()  # the same D the GPU streamed (K9/K7 output)
        cpu, ref = cpu_sample(dd, wl)
        if ref is not None:
            parity = parity_block(e, ref)
        del dd

    if rank == 0:
        line = {
            "metric": "MDS distance entries/s per streaming pass", "value": value,
            "unit": "entries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if (world == 1 or args.weak) else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, reference RNG conventions; D built on the GPU)",
            "config": {"workload": wl, "n": n, "n_single_gpu": n1, "k": k, "p": p, "q": q,
                       "seed": seed,
                       "d_dtype": "f32" if f32 else "f64", "streaming_passes_per_step": passes,
                       "l2": "inputs larger than L2 (D = %.1f GB)" % (n * n * (4 if f32 else 8) / 1e9),
                       "parallelism": (f"dp{world} (D row-sharded, panel all-gather + Gram "
                                       "all-reduce over NCCL)") if sharded else "single"},
            "e2e": e2e,
            "gpu_launches": int(st.kernel_launches),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity": parity,
            "clocks": clk.summary(),
            "result_check": {"dims": int(e.dims), "lambda_1": float(e.eigenvalues[0])
                             if e.dims else None},
        }
        emit(line)
    if sharded:
        ds.comm_destroy()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


_JSON_OUT = None


def emit(line: dict) -> None:
    """The one JSON line, on the process's original stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # stdout carries exactly one JSON line: keep a handle on the original
    # stdout for it and send everything else written to fd 1 (NCCL's version
    # banner and debug lines, library prints) to stderr
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: C2 at N = 1, C3 (fixed n, strong scaling) at N > 1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (huge D)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the row-sharded path even on one GPU (testing)")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: grow n as n1 sqrt(N) so each GPU streams n1^2 entries per pass "
                         "(weak scaling); default keeps the workload's n (strong scaling)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    wl = args.workload or ("C3" if max(world, args.gpus) > 1 else "C2")
    if args.impl == "reference":
        return reference_arm(args, wl)
    return b200_arm(args, wl)


if __name__ == "__main__":
    sys.exit(main())
