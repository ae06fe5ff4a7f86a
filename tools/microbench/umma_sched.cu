// NB = 64 digit-product MMA schedules (tcgen05 kind::i8, A in TMEM at column
// 448, B digits resident in shared memory): cycles per k-step for different
// orders / splits of the 28 (t, u) digit products into N <= 256 MMAs.
#include <cstdio>
#include <vector>

#include "umma.cuh"

using namespace dsb;

struct Mma { int acc, boff, n, ss; };
__constant__ Mma c_s[32];

__device__ volatile int g_stop;
__global__ void k_sched(int iters, int nm, unsigned long long* cycles, int noise) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 7 * 64 * 32 + 3 * 4096; i += blockDim.x) sm[i] = (i * 37) & 255;
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
    if (threadIdx.x >= 32 && threadIdx.x < 32 * (1 + noise)) {
        // shared-memory traffic beside the MMAs: 16-byte stores + loads
        // over a 16 KB region past the operands
        unsigned char* reg = sm + 7 * 64 * 32 + 3 * 4096;
        uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        const unsigned long long t0 = clock64();
        int it = 0;
        while (clock64() - t0 < 4000ull * iters / 10 * 10) {
            const int o = ((threadIdx.x + it * 128) * 16) & 16383;
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(reg + o)),
                         "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
            uint32_t a, b, c, d;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(smem_u32(reg + (o ^ 8192))) : "memory");
            v.x += a ^ b ^ c ^ d;
            if (++it % 64 == 0 && g_stop) break;
        }
        if (v.x == 12345) cycles[1] = v.y;
    }
    if (threadIdx.x == 0) {
        const unsigned long long c0 = clock64();
        for (int it = 0; it < iters; ++it)
            for (int m = 0; m < nm; ++m) {
                if (c_s[m].ss)  // A digit from shared memory (after the B digits)
                    umma_i8(tmem + c_s[m].acc,
                            umma_desc_k_interleave(smem_u32(sm + 7 * 64 * 32 + (c_s[m].ss - 1) * 4096)),
                            umma_desc_k_interleave(smem_u32(sm + c_s[m].boff)),
                            umma_idesc_i8(c_s[m].n, false, true), 1);
                else
                    umma_i8_ts(tmem + c_s[m].acc, tmem + 448,
                               umma_desc_k_interleave(smem_u32(sm + c_s[m].boff)),
                               umma_idesc_i8(c_s[m].n, false, true), 1);
            }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        if (blockIdx.x == 0) *cycles = clock64() - c0;
        g_stop = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// (t, u0, nu): A digit t times B digits u0..u0+nu-1 -> diagonals t+u0 .. t+u0+nu-1
struct P { int t, u0, nu; };
static bool g_hybrid = false;

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* dc;
    cudaMalloc(&dc, 16);
    const int smem = 7 * 64 * 32 + 3 * 4096 + 16384;
    cudaFuncSetAttribute(k_sched, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nb = 64;
    struct Named { const char* name; std::vector<P> s; };
    std::vector<Named> all = {
        {"t-major 4+rest (current)", {{1,1,4},{1,5,3},{2,1,4},{2,5,2},{3,1,4},{3,5,1},{4,1,4},{5,1,3},{6,1,2},{7,1,1}}},
        {"t reversed", {{7,1,1},{6,1,2},{5,1,3},{4,1,4},{3,1,4},{3,5,1},{2,1,4},{2,5,2},{1,1,4},{1,5,3}}},
        {"rest first then 4", {{1,5,3},{1,1,4},{2,5,2},{2,1,4},{3,5,1},{3,1,4},{4,1,4},{5,1,3},{6,1,2},{7,1,1}}},
        {"split 3+4 (suffix 4)", {{1,1,3},{1,4,4},{2,1,2},{2,3,4},{3,1,1},{3,2,4},{4,1,4},{5,1,3},{6,1,2},{7,1,1}}},
        {"split 3+4 prefix last", {{1,4,4},{1,1,3},{2,3,4},{2,1,2},{3,2,4},{3,1,1},{4,1,4},{5,1,3},{6,1,2},{7,1,1}}},
        {"interleave lo/hi", {{1,1,4},{2,5,2},{2,1,4},{1,5,3},{3,1,4},{4,1,4},{3,5,1},{5,1,3},{6,1,2},{7,1,1}}},
        {"suffix-aligned desc", {{1,4,4},{2,3,4},{3,2,4},{4,1,4},{1,1,3},{5,1,3},{2,1,2},{6,1,2},{3,1,1},{7,1,1}}},
        {"prefix blocks then suffix", {{1,1,3},{2,1,2},{3,1,1},{1,4,4},{2,3,4},{3,2,4},{4,1,4},{5,1,3},{6,1,2},{7,1,1}}},
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int noise = 0; noise < 4; noise += 1)
    for (int hy = 0; hy < 2; ++hy)
    for (auto& nmd : all) {
        g_hybrid = hy;
        if (&nmd != &all[0]) continue;
        int zero = 0;
        cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
        Mma h[32];
        int nm = 0, cols = 0;
        for (auto& p : nmd.s) {
            h[nm++] = Mma{(p.t + p.u0 - 2) * nb, (p.u0 - 1) * nb * 32, p.nu * nb,
                          (g_hybrid && p.t >= 5) ? p.t - 4 : 0};
            cols += p.nu * nb;
        }
        cudaMemcpyToSymbol(c_s, h, sizeof(h));
        const int iters = 4000;
        k_sched<<<sms, 128, smem>>>(10, nm, dc, 0);
        cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
        cudaEventRecord(e0);
        k_sched<<<sms, 128, smem>>>(iters, nm, dc, noise);
        cudaEventRecord(e1);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc;
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        printf("noise warps %d ", noise);
        printf("%s%-30s %2d MMAs %4d cols  %7.1f cycles/k-step (ideal %d)\n", hy ? "[hybrid SS t>=5] " : "", nmd.name, nm, cols,
               static_cast<double>(cyc) / iters, cols / 2);
    }
    return 0;
}
