// FP64 tensor-core roof, measured live: a register-resident DMMA loop on every
// SM (the same mma.sync m8n8k4 f64 instruction K2 issues). bench.py uses it as
// the denominator of roofline.frac for the FP64-bound product pass; the
// MEASURED_PEAKS.json figures cover HBM and bf16 only.
#include "device_utils.cuh"
#include "host_core.hpp"

namespace dsb {
namespace {
__global__ void k_dmma_peak(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma884(c[i][0], c[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}
}  // namespace
}  // namespace dsb

extern "C" double divscope_fp64_tensor_peak_tflops(int iters) {
    try {
        dsb::Ctx& c = dsb::Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        dsb::DevBuf out(8);
        const int blocks = c.sms * 4, threads = 512;
        cudaEvent_t e0, e1;
        DSB_CUDA(cudaEventCreate(&e0));
        DSB_CUDA(cudaEventCreate(&e1));
        dsb::k_dmma_peak<<<blocks, threads, 0, c.stream>>>(out.as<double>(), 64);
        DSB_CUDA(cudaEventRecord(e0, c.stream));
        dsb::k_dmma_peak<<<blocks, threads, 0, c.stream>>>(out.as<double>(), iters);
        DSB_CUDA(cudaEventRecord(e1, c.stream));
        DSB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.0f;
        DSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        dsb::count_launch(2);
        const double flops = 2.0 * 8 * 8 * 4 * 8 * static_cast<double>(iters) * (threads / 32) * blocks;
        return flops / (ms * 1e-3) / 1e12;
    } catch (...) {
        return -1.0;
    }
}

// K2 alone, for kernel tuning: `iters` launches of the streaming product
// over matrix handle m with panel width wp (zero panel), mode 0/1. Returns
// the mean device time per launch in ms (< 0 on failure).
#include "solver.hpp"
struct divscope_matrix {
    dsb::Matrix m;
};
extern "C" double divscope_bench_product(const divscope_matrix* mh, int wp, int mode, int iters) {
    try {
        dsb::Ctx& c = dsb::Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        dsb::Store& s = *mh->m.store;
        const size_t n = s.rows;
        const size_t n_pad = dsb::round_up(n, dsb::kRowPad);
        if (!s.tmap_ok) {
            c.encode_tmap(&s.tmap128, s.buf->p, s.dt, s.rows, s.cols, s.ld, 128);
            c.encode_tmap(&s.tmap256, s.buf->p, s.dt, s.rows, s.cols, s.ld, 256);
            s.tmap_ok = true;
        }
        const dsb::K2Plan plan = dsb::k2_plan(n, wp, s.dt, c.sms);
        dsb::DevBuf x(n_pad * wp * 8), y(n_pad * wp * 8), part(plan.part_elems * 8 + 64),
            rm(n * 8 + 64), sc(dsb::S_COUNT * 8), cs(2 * wp * 8);
        DSB_CUDA(cudaMemsetAsync(x.p, 0, n_pad * wp * 8, c.stream));
        DSB_CUDA(cudaMemsetAsync(rm.p, 0, n * 8 + 64, c.stream));
        DSB_CUDA(cudaMemsetAsync(sc.p, 0, dsb::S_COUNT * 8, c.stream));
        DSB_CUDA(cudaMemsetAsync(cs.p, 0, 2 * wp * 8, c.stream));
        cudaEvent_t e0, e1;
        DSB_CUDA(cudaEventCreate(&e0));
        DSB_CUDA(cudaEventCreate(&e1));
        double total = 0.0;
        for (int it = 0; it < iters + 1; ++it) {
            dsb::launch_k2(s.tmap_for(plan.bm), s.dt, mode, plan, x.as<double>(), part.as<double>(),
                           rm.as<double>(), sc.as<double>(), cs.as<double>(), y.as<double>(),
                           n_pad, c.stream, e0, e1);
            DSB_CUDA(cudaEventSynchronize(e1));
            float ms = 0.0f;
            DSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (it > 0) total += ms;
        }
        c.sync();
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return total / iters;
    } catch (...) {
        return -1.0;
    }
}
