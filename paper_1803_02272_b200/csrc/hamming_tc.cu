// K7 on the int8 tensor cores: the Hamming distance matrix of 2-bit-coded
// reads as one exact integer GEMM (tcgen05 kind::i8), so the builder is
// bound by writing D instead of by POPC issue.
//
// Encoding: base code (A=00, C=01, G=10, T=11, bits lo / hi) -> three signs
// s1 = 1 - 2 lo, s2 = 1 - 2 hi, s12 = s1 s2 (int8 +-1). Two bases are equal
// iff both bits are, and [x == y] = (1 + s1 s1' + s2 s2' + s12 s12') / 4, so
// over a read pair  sum_t [x_t == y_t] = (L + acc) / 4  with
// acc = E_i . E_j (K = 3 L, zero-padded to a multiple of 32), and
//   h_ij = L - (L + acc) / 4 = (3 L - acc) / 4   (exact: acc is an int32 sum)
// D_ij = h_ij / L in fp64, the same IEEE operation as the reference formula.
//
// Layout: E is stored in UMMA tiles — for each 128-row block and each 32-byte
// k-step one contiguous 4 KB (128 rows x 32 bytes, K-major, core matrices of
// 8 rows x 16 bytes) — so every operand tile is one cp.async.bulk.
// Kernel: persistent, one CTA per SM over 128 x 128 output tiles (upper tiles
// I <= J of the full matrix in 32 x 32-tile super-tiles, or every tile of a
// 128-aligned row band). Warp 0 streams the A / B k-step tiles through a
// 3-stage mbarrier ring of 4 k-steps each (evict_last: E stays in L2); warp 1
// issues one M = N = 128, K = 32 MMA per k-step into one of four 128-column
// TMEM accumulators; warps 4..11 turn finished accumulators into D, stage
// each 32 x 32 chunk in shared memory as rows of the tile and, off the
// diagonal, transposed as rows of the mirror tile, and store both with TMA
// tensor stores. The D stream (8 n^2 bytes) is the roofline; measured at
// 0.80 of it at C5 (profiles/r02_k7_hamming.txt), the operand reads through
// L2 and the shared-memory staging sharing the rest.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "device_utils.cuh"
#include "host_core.hpp"
#include "kernels.cuh"
#include "umma.cuh"

namespace dsb {

namespace {

constexpr int kTT = 128;      // output tile edge (M = N)
constexpr int kTK = 32;       // K bytes per MMA
constexpr int kKPer = 4;                     // k-steps per ring stage
constexpr int kTStages = 3;
constexpr int kStageOps = 2 * kKPer * 4096;  // A | B, 32 KB
constexpr int kAccBufs = 4;                  // 4 x 128 TMEM columns
constexpr int kEpiWarps = 8;                 // warps 4..11
constexpr int kTThreads = 128 + 32 * kEpiWarps;
constexpr int kWarpStage = 2 * 2 * 32 * 16 * 8;      // per epilogue warp: main + mirror, 2 boxes each
constexpr int kStageBytes = kEpiWarps * kWarpStage;  // 128 KB
constexpr int kTileBytes = kTT * kTK;  // 4 KB operand tile

// E tiles from the bit planes (k_pack_reads): thread per (row, k-step, 4-byte
// group); rows >= count and positions >= length are zero
__global__ void __launch_bounds__(256) k_hamming_encode(const uint32_t* __restrict__ plo,
                                                        const uint32_t* __restrict__ phi,
                                                        int count, int words, int length,
                                                        int nblk, int nks,
                                                        int8_t* __restrict__ enc) {
    const long long total = static_cast<long long>(nblk) * kTT * nks * 8;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(e & 7);  // 4-byte group of the k-step
        const long long rk = e >> 3;
        const int ks = static_cast<int>(rk % nks);
        const int row = static_cast<int>(rk / nks);
        uint32_t word = 0;
        if (row < count) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int k = ks * kTK + g * 4 + b;  // K index: position k / 3, sign k % 3
                const int t = k / 3, which = k - 3 * (k / 3);
                int v = 0;
                if (t < length) {
                    const uint32_t lo = (plo[static_cast<size_t>(row) * words + (t >> 5)] >> (t & 31)) & 1u;
                    const uint32_t hi = (phi[static_cast<size_t>(row) * words + (t >> 5)] >> (t & 31)) & 1u;
                    const int s1 = 1 - 2 * static_cast<int>(lo), s2 = 1 - 2 * static_cast<int>(hi);
                    v = which == 0 ? s1 : (which == 1 ? s2 : s1 * s2);
                }
                word |= (static_cast<uint32_t>(v) & 0xffu) << (8 * b);
            }
        }
        const int rb = row / kTT, r = row % kTT;
        int8_t* tile = enc + (static_cast<size_t>(rb) * nks + ks) * kTileBytes;
        *reinterpret_cast<uint32_t*>(tile + umma_tile_off(static_cast<uint32_t>(r),
                                                          static_cast<uint32_t>(g * 4))) = word;
    }
}

// E stays in L2 (61 MB at C5) while 20 GB of D streams past it: operand
// loads carry an evict_last policy, D stores are evict-first (st.global.cs)
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes,
                                               uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
        "%2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// TMA tensor store of one box (shared -> global), its group commit and waits
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], "
        "%4;" ::"l"(reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Persistent: one CTA per SM walks tiles t = blockIdx.x, += gridDim.x. Warp 0
// streams operand k-steps through the ring across tile boundaries, warp 1
// rotates four TMEM accumulators (acc_full / acc_empty), so the MMAs of later
// tiles run while warps 4..11 convert and store earlier ones — the store
// stream, which bounds the kernel, never waits for operands.
template <bool SYM, bool FASTDIV>
__global__ void __launch_bounds__(kTThreads, 1)
    k_hamming_tc(const __grid_constant__ CUtensorMap dmap, const int8_t* __restrict__ enc,
                 int count, int length, int nblk, int nks,
                 const int2* __restrict__ order, long long tiles, double* __restrict__ out,
                 size_t ld, int row0, int nrows) {
    extern __shared__ __align__(1024) unsigned char smh[];
    unsigned char* sm = smh + ((1024u - (smem_u32(smh) & 1023u)) & 1023u);
    unsigned char* ring = sm;                            // [stages][A kKPer x 4 KB | B ...]
    unsigned char* stage = ring + kTStages * kStageOps;  // [warp][2 x 8 KB] staged D boxes
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + kStageBytes);
    uint64_t* empty = full + kTStages;
    uint64_t* acc_full = empty + kTStages;     // [kAccBufs]
    uint64_t* acc_empty = acc_full + kAccBufs;  // [kAccBufs]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + kAccBufs);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], kEpiWarps);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tslot, kAccBufs * kTT);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (warp == 0) {
        // a stage holds kKPer consecutive k-steps of A and of B: E keeps a
        // row block's k-steps contiguous, so that is one bulk copy each
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            long long it = 0;
            const uint64_t pol = policy_evict_last();
            for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int I = order[t].x, J = order[t].y;
                const int8_t* ablk = enc + static_cast<size_t>(I) * nks * kTileBytes;
                const int8_t* bblk = enc + static_cast<size_t>(J) * nks * kTileBytes;
                for (int ks = 0; ks < nks; ks += kKPer, ++it) {
                    if (it >= kTStages) mbar_wait(&empty[s], ph ^ 1);
                    const uint32_t bytes = static_cast<uint32_t>(min(kKPer, nks - ks)) * kTileBytes;
                    unsigned char* dst = ring + s * kStageOps;
                    mbar_arrive_expect_tx(&full[s], 2 * bytes);
                    bulk_load_hint(dst, ablk + static_cast<size_t>(ks) * kTileBytes, bytes, &full[s],
                                   pol);
                    bulk_load_hint(dst + kKPer * kTileBytes, bblk + static_cast<size_t>(ks) * kTileBytes,
                                   bytes, &full[s], pol);
                    if (++s == kTStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        int s = 0;
        uint32_t ph = 0;
        int u = 0;  // tiles issued
        const uint32_t idesc = umma_idesc_i8(kTT, true, true);  // s8 x s8 -> s32
        for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++u) {
            const int b = u % kAccBufs;
            if (u >= kAccBufs) mbar_wait(&acc_empty[b], ((u / kAccBufs) - 1) & 1);
            tc_fence_after();
            const uint32_t acc = tmem + static_cast<uint32_t>(b * kTT);
            for (int ks = 0; ks < nks; ks += kKPer) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t base = smem_u32(ring + s * kStageOps);
                const int cnt = min(kKPer, nks - ks);
                for (int kk = 0; kk < cnt; ++kk)
                    umma_i8_w(acc, umma_desc_k_interleave(base + kk * kTileBytes),
                              umma_desc_k_interleave(base + (kKPer + kk) * kTileBytes), idesc,
                              (ks + kk) > 0 ? 1 : 0);
                umma_commit_w(&empty[s]);
                if (++s == kTStages) {
                    s = 0;
                    ph ^= 1;
                }
            }
            umma_commit_w(&acc_full[b]);
        }
    } else if (warp >= 4) {
        // epilogue: warp ew = warp - 4 owns TMEM lanes 32 (warp & 3) .. + 31
        // (tile rows) and columns [64 (ew >> 2), + 64), read 32 columns at a
        // time (lane = row, 32 consecutive columns). Each 32 x 32 chunk is
        // staged twice in the TMA's 128-byte-swizzled box layout (boxes of 32
        // rows x 16 columns): as rows of the tile (16-byte writes) and, off
        // the diagonal, transposed as rows of the mirror tile (J, I) (8-byte
        // writes, a warp covering one 256-byte mirror row) — both
        // conflict-free — and one lane hands the boxes to the TMA (tensor
        // stores, evict-first, edge tiles clipped by the tensor map). The
        // mirror costs shared-memory bandwidth once, not a second product.
        // With an odd leading dimension (no tensor map) 8-byte stores go
        // straight from registers instead.
        const int ew = warp - 4, q = warp & 3, cw = (ew >> 2) * 64;
        unsigned char* wst = stage + ew * kWarpStage;  // [main 8 KB | mirror 8 KB]
        const int l3 = 3 * length;
        const double L = static_cast<double>(length), rinv = 1.0 / L;
        const bool vec = (ld & 1) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
        const uint64_t pol = policy_evict_first();
        bool pending = false;
        // D = h / L with x = 4 h = 3 L - acc: the reference's IEEE division,
        // or (FASTDIV, checked on the host for every h in [0, L]) q = h / L
        // from the reciprocal and one remainder step, bit-identical to it;
        // the factor 4 is folded into the constants (exact power-of-2 scaling)
        const double L4 = 4.0 * L, rinv4 = 0.25 * rinv;
        auto conv = [&](int32_t acc) -> double {
            const int x = l3 - acc;  // 0 <= x = 4 h <= 4 L
            const double xd = __hiloint2double(0x43300000, x) - 4503599627370496.0;  // exact
            if constexpr (!FASTDIV) {
                return (0.25 * xd) / L;
            } else {
                const double q0 = xd * rinv4;
                return fma(fma(-q0, L4, xd), rinv4, q0);
            }
        };
        int u = 0;
        for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++u) {
            const int I = order[t].x, J = order[t].y;
            const bool mirror = SYM && I != J;
            const int b = u % kAccBufs;
            mbar_wait(&acc_full[b], (u / kAccBufs) & 1);
            tc_fence_after();
            const int r0 = I * kTT + q * 32;  // this warp's first tile row
#pragma unroll 1
            for (int ch = 0; ch < 2; ++ch) {
                const int c0 = J * kTT + cw + ch * 32;  // first column of the chunk
                int32_t v[32];
                tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) +
                              static_cast<uint32_t>(b * kTT + cw + ch * 32),
                          v);
                tmem_ld_wait();
                if (ch == 1) {
                    // this warp's accumulator reads are done: the MMA warp
                    // may reuse buffer b
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&acc_empty[b]);
                }
                double dv[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) dv[j] = conv(v[j]);
                if (!vec) {
                    const int i = r0 + lane;
                    if (i < (SYM ? count : row0 + nrows))
                        for (int j = 0; j < 32; ++j)
                            if (c0 + j < count) out[static_cast<size_t>(i - (SYM ? 0 : row0)) * ld + c0 + j] = dv[j];
                    if (mirror)
                        for (int j = 0; j < 32; ++j)
                            if (c0 + j < count && r0 + lane < count)
                                out[static_cast<size_t>(c0 + j) * ld + r0 + lane] = dv[j];
                    continue;
                }
                // the staged boxes are free once the previous stores read them
                if (lane == 0 && pending) bulk_wait_read0();
                __syncwarp();
                // tile rows: box k = j / 16 (32 rows x 16 columns), row = lane,
                // 16-byte chunk (j % 16) / 2 swizzled with lane & 7
#pragma unroll
                for (int j = 0; j < 32; j += 2)
                    *reinterpret_cast<double2*>(wst + (j >> 4) * 4096 + lane * 128 +
                                                ((((j & 15) >> 1) ^ (lane & 7)) << 4)) =
                        make_double2(dv[j], dv[j + 1]);
                if (mirror) {
                    // mirror rows c0 + j, columns r0 + lane: box lane / 16,
                    // row j, chunk (lane % 16) / 2 swizzled with j & 7
                    unsigned char* mb = wst + 8192 + (lane >> 4) * 4096 + (lane & 1) * 8;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        *reinterpret_cast<double*>(mb + j * 128 + ((((lane & 15) >> 1) ^ (j & 7)) << 4)) =
                            dv[j];
                }
                fence_proxy_async();  // generic-proxy writes -> TMA reads
                __syncwarp();
                if (lane == 0) {
                    const int rr = r0 - (SYM ? 0 : row0);
#pragma unroll
                    for (int k = 0; k < 2; ++k) tma_store_2d(&dmap, wst + k * 4096, c0 + 16 * k, rr, pol);
                    if (mirror)
#pragma unroll
                        for (int k = 0; k < 2; ++k)
                            tma_store_2d(&dmap, wst + 8192 + k * 4096, r0 + 16 * k, c0, pol);
                    bulk_commit();
                    pending = true;
                }
            }
        }
        if (lane == 0 && pending) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, kAccBufs * kTT);
}

size_t hamming_tc_smem() {
    return 1024 + static_cast<size_t>(kTStages) * kStageOps +
           static_cast<size_t>(kStageBytes) + (2 * kTStages + 2 * kAccBufs) * 8 + 64;
}

// q = h (1 / L) corrected by one remainder step equals the IEEE quotient h / L
// for every count h in [0, L]?
// (the kernel's FASTDIV arithmetic, x = 4 h)
bool fast_div_exact(int length) {
    const double L = static_cast<double>(length), rinv = 1.0 / L;
    const double L4 = 4.0 * L, rinv4 = 0.25 * rinv;
    for (int h = 0; h <= length; ++h) {
        const double xd = 4.0 * h, q0 = xd * rinv4;
        if (std::fma(std::fma(-q0, L4, xd), rinv4, q0) != static_cast<double>(h) / L) return false;
    }
    return true;
}

}  // namespace

bool hamming_tc_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DSB_HAMMING_TC");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

bool launch_hamming_tc(const uint32_t* lo, const uint32_t* hi, size_t count, int words, int length,
                       double* d, size_t ld, cudaStream_t st, size_t row0, size_t nrows) {
    if (!hamming_tc_enabled() || count == 0 || length <= 0 || length > (1 << 20)) return false;
    if (row0 % kTT != 0) return false;  // row bands start on a 128-row block
    const int nblk = static_cast<int>((count + kTT - 1) / kTT);
    const int nks = static_cast<int>((3 * static_cast<size_t>(length) + kTK - 1) / kTK);
    // E is 3 bytes per base and read: beyond a few GB (very long reads at
    // large n) the POPC kernel, which needs no E, builds D instead
    const size_t enc_bytes = static_cast<size_t>(nblk) * nks * kTileBytes;
    if (enc_bytes > (static_cast<size_t>(4) << 30)) return false;
    DevBuf enc(enc_bytes);
    {
        const long long items = static_cast<long long>(nblk) * kTT * nks * 8;
        const int grid =
            static_cast<int>(std::min<long long>((items + 255) / 256, Ctx::get().sms * 16LL));
        k_hamming_encode<<<grid, 256, 0, st>>>(lo, hi, static_cast<int>(count), words, length,
                                               nblk, nks, enc.as<int8_t>());
    }
    // D's tensor map (box 16 columns x 32 rows, 128-byte swizzle): rows of
    // the band (or the whole matrix), 16-byte aligned rows only
    CUtensorMap dmap{};
    if ((ld & 1) == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0 &&
        !Ctx::get().encode_tmap(&dmap, d, DType::F64, nrows, count, ld, 32))
        throw Error(errc::internal, "cuTensorMapEncodeTiled failed (Hamming D)");
    const size_t smem = hamming_tc_smem();
    const bool fast_div = fast_div_exact(length);
    const bool sym = row0 == 0 && nrows == count;
    // tile order: S x S super-tiles, so the ~148 tiles in flight share 2 S
    // operand blocks (L2 reuse of E under the D store stream)
    constexpr int S = 32;
    std::vector<int2> order;
    const int ib0 = static_cast<int>(row0 / kTT);
    const int ib1 = sym ? nblk : static_cast<int>((row0 + nrows + kTT - 1) / kTT);
    for (int si = ib0; si < ib1; si += S)
        for (int sj = sym ? si : 0; sj < nblk; sj += S)
            for (int i = si; i < std::min(si + S, ib1); ++i)
                for (int j = std::max(sj, sym ? i : 0); j < std::min(sj + S, nblk); ++j)
                    order.push_back(make_int2(i, j));
    const long long tiles = static_cast<long long>(order.size());
    DevBuf dorder(order.size() * sizeof(int2));
    DSB_CUDA(cudaMemcpyAsync(dorder.p, order.data(), order.size() * sizeof(int2),
                             cudaMemcpyHostToDevice, st));
    const int grid = static_cast<int>(std::min<long long>(tiles, Ctx::get().sms));
    auto go = [&](auto sym_tag, auto fast_tag) {
        constexpr bool S_ = decltype(sym_tag)::value, F_ = decltype(fast_tag)::value;
        ensure_dyn_smem(reinterpret_cast<const void*>(k_hamming_tc<S_, F_>), smem);
        k_hamming_tc<S_, F_><<<grid, kTThreads, smem, st>>>(
            dmap, enc.as<int8_t>(), static_cast<int>(count), length, nblk, nks, dorder.as<int2>(), tiles,
            d, ld, static_cast<int>(row0), static_cast<int>(nrows));
    };
    if (sym) {
        if (fast_div) go(std::true_type{}, std::true_type{});
        else go(std::true_type{}, std::false_type{});
    } else {
        if (fast_div) go(std::false_type{}, std::true_type{});
        else go(std::false_type{}, std::false_type{});
    }
    DSB_CUDA(cudaGetLastError());
    count_launch(2);
    return true;
}

}  // namespace dsb
