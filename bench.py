#!/usr/bin/env python
"""bench.py — BASELINE.json metric "MDS distance entries/s per streaming pass;
achieved HBM GB/s as % of roofline" on the B200 path.

Workload (default C2 = BASELINE.json configs[1], the largest config quoted for
one GPU): n = 20,000 points from a seeded mixture of 20 Gaussian clusters in
R^50 (Dirichlet(1) weights), fp64 Euclidean D (3.2 GB), classical MDS with
k = 20, p = 10, q = 2. Inputs are seeded synthetic data generated with the
reference's RNG conventions.

One *step* = one full classical MDS of D through the public API:
  divscope_gram (pass 0: K1 reads D once) + divscope_embed (2q + 2 = 6 streaming
  product passes over D, CholeskyQR, Rayleigh-Ritz EVD, lift / sign / scale)
so a step makes 2q + 3 = 7 streaming passes over D, and
  value = n^2 * (2q + 3) * steps / time      [entries/s per streaming pass]
  e2e   = same metric through the C ABI from a pinned HOST copy of D, the
          host->device copy of D and Omega and the device->host read of the
          coordinates inside the timed region.
D (3.2 GB) is larger than the 126 MB L2, so every pass streams from HBM.

--impl reference times the reference's own CPU implementation of the
streaming pass (multiply_sym, ref src/rsvd.cpp:18-36, compiled from the
reference sources into oracle/_ref; the oracle port when _ref is absent) on
the same D, with all host threads: one step = one pass.
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


def cpu_reference_pass(d_host: np.ndarray, omega: np.ndarray, steps: int, warmup: int):
    """Time the reference streaming pass (multiply_sym) on the host cores.
    Returns (seconds per pass list, kind, cores)."""
    from oracle_bindings import Oracle, RefLib, ref_available
    cores = os.cpu_count() or 1
    if ref_available():
        lib, kind = RefLib(), "reference"
        st, g = lib.gram(d_host, threads=cores)
        assert st == 0, "reference gram failed"
        run = lambda: lib.multiply_sym(g, omega, threads=cores)  # noqa: E731
    else:
        lib, kind = Oracle(), "port"
        st, rm, grand = lib.gram_stats(d_host)
        assert st == 0
        run = lambda: lib.multiply_gram_otf(d_host, rm, grand, omega, threads=cores)  # noqa: E731
    for _ in range(warmup):
        run()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    return times, kind, cores


def reference_arm(args, wl):
    world, rank, _ = dist_init()
    cfg, n, k, p, q, seed, f32 = WORKLOADS[wl]
    metric = "MDS distance entries/s per streaming pass"
    if rank != 0:
        return 0
    import paper_1803_02272_b200 as ds  # host-only synthesis (no GPU work)
    from oracle_bindings import Oracle
    pts = ds.synth_points(cfg, n, seed)
    d = Oracle().euclidean_matrix_mt(pts)
    if f32:
        d = d.astype(np.float32).astype(np.float64)
    w = k + min(p, n - k)
    omega = Oracle().fill_gaussian(seed, n * w).reshape(n, w)
    steps = max(1, args.steps)
    times, kind, cores = cpu_reference_pass(d, omega, steps, max(0, min(args.warmup, 1)))
    t = float(np.mean(times))
    value = n * n / t
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": "entries/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, reference RNG conventions)",
        "config": {"workload": wl, "n": n, "k": k, "p": p, "q": q, "seed": seed,
                   "d_dtype": "f32" if f32 else "f64",
                   "step": "one reference multiply_sym pass over the materialized gram"},
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": cores, "kind": kind,
                         "sample": f"{steps} x multiply_sym(G[{n}x{n}], Omega[{n}x{w}]), "
                                   f"{cores} threads (ref src/rsvd.cpp:18-36)"},
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
    if sharded and not args.strong:
        # weak scaling: every GPU streams the same n1^2 entries of D per pass,
        # the matrix grows as n = n1 sqrt(N) (row-sharded over the N GPUs)
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
        except Exception:
            traffic = None
    hbm = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
           "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
           else "fallback 6650 GB/s (B200_PROFILING.md)"}
    common = {"k2_avg_ms": k2_ms, "k2_launches": int(st.product_launches),
              "flops_per_launch": flops_per_launch, "bytes_per_launch": bytes_per_launch,
              "pass0": {"k1_avg_ms": st.stats_ms / max(st.stats_launches, 1),
                        "achieved_gbs": m_rows * n * (4 if f32 else 8) /
                        (st.stats_ms / max(st.stats_launches, 1) * 1e-3) / 1e9}}
    if int8_path:
        # exact integer slice product on the int8 tensor cores: one read of D
        # per column group (w <= 64: one group), HBM-bound; `achieved` counts
        # the pass's algorithmic bytes (D once), `streamed_gbs` every read
        groups = max(int(st.last_product_groups), 1)
        roofline = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": gbs / hbm_peak, "traffic": traffic,
                    "kernel": ("k2i_product (3x7-digit int8 slice product of the exact Hamming "
                               "h^2, tcgen05 kind::i8)" if int(st.last_product_sdigits) == 3 else
                               "k2i_product (7x7-digit int8 slice product, tcgen05 kind::i8)"),
                    "peak_source": hbm["peak_source"],
                    "column_groups": groups,
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
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle_bindings import Oracle
        omega = Oracle().fill_gaussian(seed, n * w).reshape(n, w)
        dd = D.to_numpy()
        times, kind, cores = cpu_reference_pass(dd, omega, 1, 0)
        cpu = {"value": n * n / times[0], "unit": "entries/s", "cores": cores, "kind": kind,
               "sample": f"one multiply_sym pass (ref src/rsvd.cpp:18-36) over the materialized "
                         f"{wl} gram, n={n}, w={w}, {cores} threads; gram build untimed"}

    if rank == 0:
        line = {
            "metric": "MDS distance entries/s per streaming pass", "value": value,
            "unit": "entries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (sharded and args.strong) else "weak",
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
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (huge D)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the row-sharded path even on one GPU (testing)")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1: keep the workload's n (strong scaling); default grows n as "
                         "n1 sqrt(N) so each GPU streams n1^2 entries per pass (weak scaling)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args, args.workload)
    return b200_arm(args, args.workload)


if __name__ == "__main__":
    sys.exit(main())
