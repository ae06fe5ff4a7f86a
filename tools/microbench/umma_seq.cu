// Cycle cost of sequences of tcgen05 kind::i8 MMAs (M = 128, K = 32, A from
// TMEM, B from shared memory), one CTA per SM, whole-warp issue with
// elect.sync as in k2i_product_ts. Each sequence is a list of
// (accumulator column, N, B byte offset); the kernel replays it `iters`
// times and reports cycles per replay. Used to choose the digit-MMA
// arrangement of the int8 slice product for column groups wider than 32.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1803_02272_b200/csrc \
//        -o tools/microbench/umma_seq tools/microbench/umma_seq.cu
#include <cstdio>
#include <string>
#include <vector>

#include "umma.cuh"

using namespace dsb;

struct Op {
    int acc, n, boff, acol;
};
__constant__ Op g_ops[64];

__global__ void k_seq(int nops, int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sm[i] = (i * 37) & 255;
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
    if (threadIdx.x < 32) {
        const unsigned long long c0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int o = 0; o < nops; ++o) {
                const Op op = g_ops[o];
                umma_i8_ts_w(tmem + op.acc, tmem + op.acol,
                             umma_desc_k_interleave(smem_u32(sm + op.boff)),
                             umma_idesc_i8(op.n, false, true), 1);
            }
        }
        umma_commit_w(&bar);
        mbar_wait(&bar, 0);
        const unsigned long long c1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = c1 - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// digit pattern: A digit t (1..7) against B digits u0.. (concatenated, nb
// columns each) into diagonal accumulators; `cap` = widest MMA, `order` 1 =
// t descending; `acol` = TMEM column of the A stage
static std::vector<Op> digits(int nb, int cap, bool rev, int acol, bool balanced = false) {
    std::vector<Op> v;
    for (int tt = 1; tt <= 7; ++tt) {
        const int t = rev ? 8 - tt : tt;
        const int umax = 8 - t;
        const int per = cap / nb;
        int parts = (umax + per - 1) / per;
        int u0 = 1;
        for (int pidx = 0; pidx < parts; ++pidx) {
            int nu = balanced ? (umax - u0 + 1 + (parts - pidx) - 1) / (parts - pidx)
                              : std::min(per, umax - u0 + 1);
            v.push_back({(t + u0 - 2) * nb, nu * nb, (u0 - 1) * nb * 32, acol});
            u0 += nu;
        }
    }
    return v;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    cudaFuncSetAttribute(k_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    struct Seq {
        std::string name;
        std::vector<Op> ops;
        double ideal;  // sum N / 2
    };
    std::vector<Seq> seqs;
    auto add = [&](const std::string& nm, std::vector<Op> ops) {
        double s = 0;
        for (auto& o : ops) s += o.n / 2.0;
        seqs.push_back({nm, ops, s});
    };
    add("NB=32 digits (7 MMAs)", digits(32, 256, false, 256));
    add("NB=32 digits, t reversed", digits(32, 256, true, 256));
    add("NB=64 digits, split at 256", digits(64, 256, false, 448));
    add("NB=64 digits, split at 256, t reversed", digits(64, 256, true, 448));
    add("NB=64 digits, balanced split", digits(64, 256, false, 448, true));
    add("NB=64 digits, balanced, t reversed", digits(64, 256, true, 448, true));
    add("NB=48 digits, split at 240", digits(48, 256, false, 448));
    add("NB=48 digits, balanced, t reversed", digits(48, 256, true, 448, true));
    add("NB=16 digits", digits(16, 256, false, 448));
    add("NB=40 digits (N = 40 u, steps of 8)", digits(40, 256, false, 448));
    add("NB=40 digits, balanced, t reversed", digits(40, 256, true, 448, true));
    add("NB=56 digits", digits(56, 256, false, 448));
    {
        std::vector<Op> v;
        for (int i = 0; i < 7; ++i) v.push_back({0, 256, 0, 448});
        add("7 x N=256 same accumulator", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 7; ++i) v.push_back({(i & 1) * 192, 256, 0, 448});
        add("7 x N=256 alternating 0/192", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 14; ++i) v.push_back({0, 128, 0, 448});
        add("14 x N=128 same accumulator", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 14; ++i) v.push_back({(i % 3) * 128, 128, 0, 448});
        add("14 x N=128 rotating", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 28; ++i) v.push_back({0, 64, 0, 448});
        add("28 x N=64 same accumulator", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 28; ++i) v.push_back({(i % 7) * 64, 64, 0, 448});
        add("28 x N=64 rotating", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 56; ++i) v.push_back({(i % 7) * 32, 32, 0, 448});
        add("56 x N=32 rotating", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 8; ++i) v.push_back({(i % 2) * 224, 224, 0, 448});
        add("8 x N=224 alternating", v);
    }
    {
        std::vector<Op> v;
        for (int i = 0; i < 12; ++i) v.push_back({(i % 3) * 160, 160, 0, 480});
        add("12 x N=160 rotating", v);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto& s : seqs) {
        if (s.ops.size() > 64) continue;
        cudaMemcpyToSymbol(g_ops, s.ops.data(), s.ops.size() * sizeof(Op));
        const int iters = 4000;
        k_seq<<<sms, 128, 32768>>>(static_cast<int>(s.ops.size()), 10, dc);
        cudaEventRecord(e0);
        k_seq<<<sms, 128, 32768>>>(static_cast<int>(s.ops.size()), iters, dc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) {
            printf("%-42s error %s\n", s.name.c_str(), cudaGetErrorString(err));
            return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc = 0;
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        const double per = static_cast<double>(cyc) / iters;
        double cols = 0;
        for (auto& o : s.ops) cols += o.n;
        const double tops = 2.0 * 128 * 32 * cols * iters * sms / (ms * 1e-3) / 1e12;
        printf("%-42s %3zu MMAs  %7.1f cycles/replay (ideal %6.1f, %5.1f%%)  %7.1f TOPS\n",
               s.name.c_str(), s.ops.size(), per, s.ideal, 100.0 * s.ideal / per, tops);
    }
    return 0;
}
