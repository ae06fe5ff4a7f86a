// Throughput of tcgen05 kind::i8 MMAs (M = 128, K = 32) from shared memory,
// one CTA per SM, operands resident: the K2 digit pattern (7 MMAs per k-step
// with N' = (8-t) NB, NB = 32/64) vs plain N = 256 MMAs, no-swizzle K-major.
// Prints achieved int8 TOPS (2 ops per MAC).
#include <cstdio>
#include <cstdlib>

#include "umma.cuh"

using namespace dsb;

__global__ void k_rate(int iters, int pattern, int nb, unsigned long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    unsigned char* sa = sm;                 // 7 x 4 KB
    unsigned char* sb = sm + 7 * 4096;      // 7 x nb x 32
    for (int i = threadIdx.x; i < 7 * 4096 + 7 * 64 * 32; i += blockDim.x) sm[i] = (i * 37) & 255;
    fence_proxy_async();
    if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const unsigned long long c0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (pattern == 2) {
                for (int t = 1; t <= 7; ++t)
                    umma_i8_ts(tmem + (t - 1) * nb, tmem + 256 + (t - 1) * 8,
                               umma_desc_k_interleave(smem_u32(sb)),
                               umma_idesc_i8((8 - t) * nb, false, true), 1);
            } else if (pattern == 3 || pattern == 4) {
                // NB = 64: digits 1..4 from TMEM (pattern 3: 5..7 from smem;
                // pattern 4: all from TMEM), N' split at 256
                for (int t = 1; t <= 7; ++t) {
                    const int per = 256 / nb, umax = 8 - t;
                    for (int u0 = 1; u0 <= umax; u0 += per) {
                        const int nu = (umax - u0 + 1 < per) ? (umax - u0 + 1) : per;
                        const uint64_t bd = umma_desc_k_interleave(smem_u32(sb + (u0 - 1) * nb * 32));
                        if (t <= 4 || pattern == 4)
                            umma_i8_ts(tmem + (t + u0 - 2) * nb, tmem + 448, bd,
                                       umma_idesc_i8(nu * nb, false, true), 1);
                        else
                            umma_i8(tmem + (t + u0 - 2) * nb,
                                    umma_desc_k_interleave(smem_u32(sa + (t - 1) * 4096)), bd,
                                    umma_idesc_i8(nu * nb, false, true), 1);
                    }
                }
            } else if (pattern == 5 || pattern == 7) {
                // NB = 64, all digits in TMEM, N' split at 128 (5) or the
                // digit loop order reversed, largest-N last (7)
                for (int tt = 1; tt <= 7; ++tt) {
                    const int t = pattern == 7 ? 8 - tt : tt;
                    const int per = (pattern == 5 ? 128 : 256) / nb, umax = 8 - t;
                    for (int u0 = 1; u0 <= umax; u0 += per) {
                        const int nu = (umax - u0 + 1 < per) ? (umax - u0 + 1) : per;
                        const uint64_t bd = umma_desc_k_interleave(smem_u32(sb + (u0 - 1) * nb * 32));
                        umma_i8_ts(tmem + (t + u0 - 2) * nb, tmem + 448, bd,
                                   umma_idesc_i8(nu * nb, false, true), 1);
                    }
                }
            } else if (pattern == 6) {
                // 7 x N = 256 from TMEM (same accumulator region, 1792 columns)
                for (int t = 0; t < 7; ++t)
                    umma_i8_ts(tmem + (t & 1) * 192, tmem + 448, umma_desc_k_interleave(smem_u32(sb)),
                               umma_idesc_i8(256, false, true), 1);
            } else if (pattern == 8) {
                // 14 x N = 128 from TMEM (1792 columns)
                for (int t = 0; t < 14; ++t)
                    umma_i8_ts(tmem + (t % 3) * 128, tmem + 448, umma_desc_k_interleave(smem_u32(sb)),
                               umma_idesc_i8(128, false, true), 1);
            } else if (pattern == 9) {
                // 28 x N = 64 from TMEM (1792 columns)
                for (int t = 0; t < 28; ++t)
                    umma_i8_ts(tmem + (t % 6) * 64, tmem + 448, umma_desc_k_interleave(smem_u32(sb)),
                               umma_idesc_i8(64, false, true), 1);
            } else if (pattern == 0) {
                for (int t = 1; t <= 7; ++t) {
                    const int per = 256 / nb, umax = 8 - t;
                    for (int u0 = 1; u0 <= umax; u0 += per) {
                        const int nu = (umax - u0 + 1 < per) ? (umax - u0 + 1) : per;
                        umma_i8(tmem + (t + u0 - 2) * nb,
                                umma_desc_k_interleave(smem_u32(sa + (t - 1) * 4096)),
                                umma_desc_k_interleave(smem_u32(sb + (u0 - 1) * nb * 32)),
                                umma_idesc_i8(nu * nb, false, true), 1);
                    }
                }
            } else {
                // 4 MMAs of N = 224 (same MAC count as pattern 0 at nb=32 would be 28*32 cols)
                for (int t = 0; t < 4; ++t)
                    umma_i8(tmem, umma_desc_k_interleave(smem_u32(sa + t * 4096)),
                            umma_desc_k_interleave(smem_u32(sb)), umma_idesc_i8(224, false, true), 1);
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        const unsigned long long c1 = clock64();
        if (blockIdx.x == 0) *cycles = c1 - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    const int smem = 7 * 4096 + 7 * 64 * 32;
    cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { int pattern, nb; double cols_per_iter; const char* name; };
    const Cfg cfgs[] = {{0, 32, 28 * 32, "digit pattern NB=32 (7 MMAs, N'=224..32)"},
                        {0, 64, 28 * 64, "digit pattern NB=64 (10 MMAs)"},
                        {1, 32, 4 * 224, "4 x N=224"},
                        {2, 32, 28 * 32, "digit pattern NB=32, A in TMEM"},
                        {3, 64, 28 * 64, "NB=64 hybrid (digits 1-4 TMEM, 5-7 smem)"},
                        {4, 64, 28 * 64, "NB=64 all digits in TMEM"},
                        {5, 64, 28 * 64, "NB=64 all TMEM, N split at 128"},
                        {7, 64, 28 * 64, "NB=64 all TMEM, t reversed"},
                        {6, 64, 28 * 64, "7 x N=256 TS"},
                        {8, 64, 28 * 64, "14 x N=128 TS"},
                        {9, 64, 28 * 64, "28 x N=64 TS"}};
    for (const Cfg& c : cfgs) {
        const int iters = 4000;
        k_rate<<<sms, 128, smem>>>(10, c.pattern, c.nb, dc);
        cudaEventRecord(e0);
        k_rate<<<sms, 128, smem>>>(iters, c.pattern, c.nb, dc);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(err));
            return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc;
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        const double macs = static_cast<double>(sms) * iters * 128.0 * 32.0 * c.cols_per_iter;
        printf("%-45s %8.3f ms  %7.1f TOPS  (%.1f cycles per iteration on SM0)\n", c.name, ms,
               2.0 * macs / (ms * 1e-3) / 1e12, static_cast<double>(cyc) / iters);
    }
    return 0;
}
