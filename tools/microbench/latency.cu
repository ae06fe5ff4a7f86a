// Latency microbenchmarks (single warp / single CTA / cooperative grid) used
// to size the serial small-matrix kernels (Cholesky, Jacobi).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void dfma_chain(double* out, int n, double a) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, 1e-9);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / n; }
}
__global__ void ddiv_chain(double* out, int n, double a) {
    double x = threadIdx.x + 1.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = a / x + 1.0;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / n; }
}
__global__ void dsqrt_chain(double* out, int n) {
    double x = threadIdx.x + 2.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / n; }
}
__global__ void lds_chain(double* out, int n) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    int j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) j = idx[j];
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = j; out[1] = double(t1 - t0) / n; }
}
__global__ void sync_cost(double* out, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[1] = double(t1 - t0) / n; }
}
__global__ void grid_sync_cost(double* out, int n) {
    cg::grid_group g = cg::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) g.sync();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[1] = double(t1 - t0) / n; }
}

int main() {
    double* d; cudaMalloc(&d, 64);
    double h[2];
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    auto rep = [&](const char* name) { cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("%-28s %8.1f cycles\n", name, h[1]); };
    dfma_chain<<<1, 32>>>(d, 10000, 1.0000001); rep("DFMA dependent latency");
    ddiv_chain<<<1, 32>>>(d, 10000, 1.3); rep("DDIV dependent latency");
    dsqrt_chain<<<1, 32>>>(d, 10000); rep("DSQRT dependent latency");
    lds_chain<<<1, 32>>>(d, 10000); rep("LDS dependent latency");
    for (int t : {32, 128, 256, 512}) { sync_cost<<<1, t>>>(d, 10000); char b[64]; sprintf(b, "__syncthreads (%d thr)", t); rep(b); }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int blocks : {16, 74, 148}) {
        int n = 1000; void* args[] = {&d, &n};
        cudaLaunchCooperativeKernel((void*)grid_sync_cost, blocks, 256, args, 0, 0);
        cudaDeviceSynchronize();
        char b[64]; sprintf(b, "grid.sync (%d CTAs)", blocks); rep(b);
    }
    printf("clock %d kHz, status %s\n", clk, cudaGetErrorString(cudaGetLastError()));
}
