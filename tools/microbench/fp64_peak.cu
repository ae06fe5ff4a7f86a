// Microbenchmark: FP64 throughput on B200 via DFMA (CUDA cores) and DMMA
// (mma.sync m8n8k4 f64). Used to pick the inner product engine of the
// centered skinny product (K2) and as the measured FP64 roof.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void dmma16_loop(double* out, int iters) {
    // m16n8k4 f64 (sm_90+ shape)
    double a0 = threadIdx.x * 1e-3, a1 = 0.5, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[0] = s;
}

// a launch that failed (e.g. too many registers for the block size) must not
// print a rate: the events around it measure nothing
static bool launch_ok(const char* what, int threads, int bps) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("%s threads=%d bps=%d: launch failed (%s), skipped\n", what, threads, bps,
               cudaGetErrorString(e));
        return false;
    }
    return true;
}

int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int threads : {256, 512, 1024}) {
        for (int bps : {1, 2, 4}) {
            if (threads * bps > 2048) continue;
            int iters = 4096;
            dim3 grid(sms * bps);
            dfma_loop<<<grid, threads>>>(d, 16, 1.0000001, 1e-9);
            cudaEventRecord(e0);
            dfma_loop<<<grid, threads>>>(d, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 16 * iters * (double)threads * grid.x;
            if (launch_ok("DFMA", threads, bps))
                printf("DFMA threads=%d bps=%d: %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
            dmma_loop<<<grid, threads>>>(d, 16);
            cudaEventRecord(e0);
            dmma_loop<<<grid, threads>>>(d, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = 2.0 * 8 * 8 * 4 * 8 * iters * (double)(threads / 32) * grid.x;
            if (launch_ok("DMMA884", threads, bps))
                printf("DMMA884 threads=%d bps=%d: %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
            dmma16_loop<<<grid, threads>>>(d, 16);
            cudaEventRecord(e0);
            dmma16_loop<<<grid, threads>>>(d, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = 2.0 * 16 * 8 * 4 * 8 * iters * (double)(threads / 32) * grid.x;
            if (launch_ok("DMMA1684", threads, bps))
                printf("DMMA1684 threads=%d bps=%d: %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
