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
