// K2 — the centered tall-skinny product Y = G X that replaces multiply_sym
// over the materialized gram (ref src/rsvd.cpp:18-36, called 2q+2 times by
// randomized_range / eigs_sym, rsvd.cpp:94-98 and :108; G built by
// gram_from_distances, ref src/mds.cpp:43-58).
//
// G is never formed. With S = D o D, r the row means of S and g the grand
// mean,  G X = -1/2 [ S X - r (1^T X) - 1 (r^T X) + g 1 (1^T X) ],  so the
// streaming part is S X: D is read once per pass, squared in registers
// (fp32 D is widened first, so d^2 is exact), and multiplied into the panel
// on the FP64 tensor cores (mma.sync m8n8k4 f64 -> DMMA, measured 37.1 TF/s
// vs 33.6 for DFMA on this B200; see profiles/).
//
// Structure (one CTA per SM, persistent, stream-K):
//  * warp 8 = producer: one elected lane issues, per (row block, k tile)
//    iteration, a TMA 2D load of the 128 x 128-byte D tile (SWIZZLE_128B) and
//    a cp.async.bulk of the matching contiguous k4-interleaved panel chunk,
//    both completing on the stage's mbarrier; a ring of `stages` buffers.
//  * warps 0-7 = consumers: each owns 16 rows x WP columns of the 128-row
//    block; per k4 step it reads 2 A fragments (swizzled smem, squared) and
//    WP/8 B fragments (one contiguous 256-byte smem read each) and issues
//    2*WP/8 DMMAs into register accumulators.
//  * the flattened iteration space (row blocks x k tiles) is split evenly
//    over the grid with the reference's own chunk rule (parallel.hpp:33-34),
//    so every SM streams the same number of D bytes; a CTA flushes its
//    accumulators to a private partial slot whenever its range crosses a row
//    block. k2_reduce sums the slots of a block in CTA order (deterministic,
//    run-to-run bit-identical) and applies the rank-3 centering.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "device_utils.cuh"
#include "host_core.hpp"
#include "kernels.cuh"

namespace dsb {

namespace {

// CW consumer warps own 16 rows each: BM = 16 CW rows of D per tile.
template <int CW>
constexpr int bm_of() {
    return 16 * CW;
}
template <int CW>
constexpr int tile_bytes() {
    return bm_of<CW>() * 128;  // one D stage: BM rows x 128 bytes
}

template <typename TD>
constexpr int kt_cols() {
    return 128 / static_cast<int>(sizeof(TD));
}

// A stage holds KS boxes of D (BM rows x 128 bytes each, KS*kt columns) and
// the matching KS*kt-row panel chunk.
template <int WP, typename TD, int CW, int KS>
constexpr int stage_bytes() {
    // D boxes (1024-aligned for the 128B swizzle) + panel chunk, rounded to 1024
    return ((KS * tile_bytes<CW>() + KS * kt_cols<TD>() * WP * 8) + 1023) / 1024 * 1024;
}

__device__ __forceinline__ long long chunk_begin(long long total, long long c, long long P) {
    return total * c / P;
}

// A(row r, col k) inside a TMA SWIZZLE_128B tile with 128-byte rows
template <typename TD>
__device__ __forceinline__ double load_a(const unsigned char* tile, int r, int k) {
    if constexpr (sizeof(TD) == 8) {
        const int off = r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3);
        return *reinterpret_cast<const double*>(tile + off);
    } else {
        const int off = r * 128 + ((((k >> 2) ^ (r & 7))) << 4) + ((k & 3) << 2);
        return static_cast<double>(*reinterpret_cast<const float*>(tile + off));
    }
}

template <int WP, typename TD, bool SQUARE, int CW, int KS>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    k2_product(const __grid_constant__ CUtensorMap tmD, const double* __restrict__ X, int nk,
               long long total, double* __restrict__ part, int maxseg, int stages,
               const int* __restrict__ skip) {
    if (skip && *skip) return;  // power-iteration batches past convergence
    constexpr int KT = kt_cols<TD>();
    constexpr int K4 = KT / 4;
    constexpr int NF = WP / 8;
    constexpr int XB = KS * KT * WP * 8;
    constexpr int SB = stage_bytes<WP, TD, CW, KS>();
    constexpr int BM = bm_of<CW>();
    constexpr int kTileBytes = tile_bytes<CW>();

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B swizzle, by integer offset so the
    // compiler keeps the shared address space (LDS, not generic loads)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * SB);
    uint64_t* empty = full + stages;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long P = gridDim.x, c = blockIdx.x;
    const long long t0 = chunk_begin(total, c, P), t1 = chunk_begin(total, c + 1, P);

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == CW) {
        // ---------------- producer ----------------
        if (lane == 0) {
            prefetch_tmap(&tmD);
            int s = 0;
            uint32_t ph = 0;
            for (long long t = t0; t < t1; ++t) {
                if (t - t0 >= stages) mbar_wait(&empty[s], ph ^ 1);
                const int b = static_cast<int>(t / nk), kt = static_cast<int>(t % nk);
                unsigned char* st = smem + static_cast<size_t>(s) * SB;
                mbar_arrive_expect_tx(&full[s], KS * kTileBytes + XB);
#pragma unroll
                for (int kb = 0; kb < KS; ++kb)
                    tma_load_2d(st + kb * kTileBytes, &tmD, (kt * KS + kb) * KT, b * BM, &full[s]);
                bulk_load(st + KS * kTileBytes, X + static_cast<size_t>(kt) * KS * KT * WP, XB,
                          &full[s]);
                if (++s == stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    double acc[2][NF][2];
#pragma unroll
    for (int fm = 0; fm < 2; ++fm)
#pragma unroll
        for (int fn = 0; fn < NF; ++fn) acc[fm][fn][0] = acc[fm][fn][1] = 0.0;

    const int m0 = warp * 16;
    const int rq = lane >> 2, kq = lane & 3;
    auto flush = [&](int seg) {
        double* dst = part + (static_cast<size_t>(c) * maxseg + seg) * BM * WP;
#pragma unroll
        for (int fm = 0; fm < 2; ++fm) {
            const int row = m0 + 8 * fm + rq;
#pragma unroll
            for (int fn = 0; fn < NF; ++fn) {
                double2 v;
                v.x = acc[fm][fn][0];
                v.y = acc[fm][fn][1];
                *reinterpret_cast<double2*>(dst + row * WP + 8 * fn + 2 * kq) = v;
                acc[fm][fn][0] = acc[fm][fn][1] = 0.0;
            }
        }
    };

    if (t0 < t1) {
        int cur_b = static_cast<int>(t0 / nk);
        int seg = 0;
        int s = 0;
        uint32_t ph = 0;
        for (long long t = t0; t < t1; ++t) {
            const int b = static_cast<int>(t / nk);
            if (b != cur_b) {
                flush(seg);
                ++seg;
                cur_b = b;
            }
            mbar_wait(&full[s], ph);
            const unsigned char* tile = smem + static_cast<size_t>(s) * SB;
            const double* xs = reinterpret_cast<const double*>(tile + KS * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < KS * K4; ++kk) {
                double a[2];
#pragma unroll
                for (int fm = 0; fm < 2; ++fm) {
                    const double v = load_a<TD>(tile + (kk / K4) * kTileBytes, m0 + 8 * fm + rq,
                                                4 * (kk % K4) + kq);
                    a[fm] = SQUARE ? v * v : v;
                }
#pragma unroll
                for (int fn = 0; fn < NF; ++fn) {
                    const double bv = xs[(kk * WP + 8 * fn + rq) * 4 + kq];
                    dmma1684(acc[0][fn][0], acc[0][fn][1], acc[1][fn][0], acc[1][fn][1], a[0],
                             a[1], bv);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
        flush(seg);
    }
}

// Sum the partial slots of each row block in CTA order, then
//   mode 1: y = -1/2 (y - r_i s_c - t_c + g s_c)   (rank-3 centering)
//   mode 0: y as is.
// Rows >= n are written as zero. Output in the k4-interleaved panel layout,
// one element per thread in panel order (coalesced stores). `tab` is the
// split's slot table (k2_slot_table): tab[b] .. tab[b + 1] index the slots
// (cta * maxseg + segment) of row block b in tab[nb + 1 ..], in CTA order.
template <int WP, int BM, int RPT>
__global__ void __launch_bounds__(256)
    k2_reduce(const double* __restrict__ part, const int* __restrict__ tab, int nb, int n,
              int mode, const double* __restrict__ row_mean, const double* __restrict__ scalars,
              const double* __restrict__ colsums, double* __restrict__ y,
              const int* __restrict__ skip) {
    if (skip && *skip) return;
    // RPT = 4: thread = one 4-row group of one column, panel elements
    // 4 t .. 4 t + 3 (one 32-byte store); RPT = 1 (small n, few elements,
    // many slots): thread = one element. Every load is issued before any sum.
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    size_t i0;
    int col;
    if constexpr (RPT == 4) {
        i0 = static_cast<size_t>(t / WP) * 4;
        col = static_cast<int>(t % WP);
    } else {
        i0 = static_cast<size_t>((t / (4 * WP)) * 4 + (t & 3));
        col = static_cast<int>((t >> 2) % WP);
    }
    const int b = static_cast<int>(i0 / BM), r0 = static_cast<int>(i0 % BM);
    const int s_begin = tab[b], nslot = tab[b + 1] - s_begin;
    const int* slots = tab + nb + 1 + s_begin;
    double rm[RPT], cs = 0.0, ct = 0.0, gr = 0.0;
    if (mode) {
        cs = colsums[col];
        ct = colsums[WP + col];
        gr = scalars[S_GRAND];
#pragma unroll
        for (int j = 0; j < RPT; ++j) rm[j] = i0 + j < static_cast<size_t>(n) ? row_mean[i0 + j] : 0.0;
    }
    const double* pp = part + static_cast<long long>(r0) * WP + col;
    // slot loads issued in batches, summed in CTA order (deterministic); the
    // batch width follows the slot count (2-3 at large n, ~20 at small n)
    double v[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) v[j] = 0.0;
    auto sum_batches = [&](auto width) {
        constexpr int kB = decltype(width)::value;
        for (int s0 = 0; s0 < nslot; s0 += kB) {
            int si[kB];
#pragma unroll
            for (int sl = 0; sl < kB; ++sl) si[sl] = s0 + sl < nslot ? slots[s0 + sl] : 0;
            double pb[kB][RPT];
#pragma unroll
            for (int sl = 0; sl < kB; ++sl)
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    pb[sl][j] = s0 + sl < nslot
                                    ? pp[static_cast<long long>(si[sl]) * (BM * WP) + j * WP]
                                    : 0.0;
#pragma unroll
            for (int sl = 0; sl < kB; ++sl)
                if (s0 + sl < nslot)
#pragma unroll
                    for (int j = 0; j < RPT; ++j) v[j] += pb[sl][j];
        }
    };
    if (nslot <= 4)
        sum_batches(std::integral_constant<int, 4>{});
    else
        sum_batches(std::integral_constant<int, 32 / RPT>{});
    double o[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        if (i0 + j >= static_cast<size_t>(n)) o[j] = 0.0;
        else if (mode) o[j] = -0.5 * (v[j] - rm[j] * cs - ct + gr * cs);
        else o[j] = v[j];
    }
    if constexpr (RPT == 4)
        *reinterpret_cast<double4*>(y + pidx(i0, col, WP)) = make_double4(o[0], o[1], o[2], o[3]);
    else
        y[pidx(i0, col, WP)] = o[0];
}

// 4 rows per thread when that still fills the GPU (>= 4 CTAs per SM), else 1
template <int WP, int BM>
void reduce_launch(const double* part, const int* tab, int nb, int n, int mode,
                   const double* row_mean, const double* scalars, const double* colsums, double* y,
                   cudaStream_t st, const int* skip) {
    const long long elems = static_cast<long long>(nb) * BM * WP;
    if (elems / 4 >= 148LL * 4 * 256)
        k2_reduce<WP, BM, 4><<<static_cast<unsigned>(elems / 1024), 256, 0, st>>>(
            part, tab, nb, n, mode, row_mean, scalars, colsums, y, skip);
    else
        k2_reduce<WP, BM, 1><<<static_cast<unsigned>(elems / 256), 256, 0, st>>>(
            part, tab, nb, n, mode, row_mean, scalars, colsums, y, skip);
}

template <int WP, typename TD, bool SQ, int CW, int KS>
void run_product_ks(const CUtensorMap* tmap, const K2Plan& p, const double* x, double* part,
                    cudaStream_t st, const int* skip) {
    ensure_dyn_smem(reinterpret_cast<const void*>(k2_product<WP, TD, SQ, CW, KS>), p.smem);
    k2_product<WP, TD, SQ, CW, KS><<<p.grid, (CW + 1) * 32, p.smem, st>>>(
        *tmap, x, p.nk, p.total, part, p.maxseg, p.stages, skip);
}

template <int WP, typename TD, bool SQ, int CW>
void run_product(const CUtensorMap* tmap, const K2Plan& p, const double* x, double* part,
                 cudaStream_t st, const int* skip) {
    if (p.ks == 2)
        run_product_ks<WP, TD, SQ, CW, 2>(tmap, p, x, part, st, skip);
    else
        run_product_ks<WP, TD, SQ, CW, 1>(tmap, p, x, part, st, skip);
}

template <int WP, int CW>
void launch_wp(const CUtensorMap* tmap, DType dt, int mode, const K2Plan& p, const double* x,
               double* part, const double* row_mean, const double* scalars,
               const double* colsums, double* y, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1,
               const int* skip) {
    if (e0) record_timing_event(e0, st);
    if (dt == DType::F64) {
        if (mode)
            run_product<WP, double, true, CW>(tmap, p, x, part, st, skip);
        else
            run_product<WP, double, false, CW>(tmap, p, x, part, st, skip);
    } else {
        if (mode)
            run_product<WP, float, true, CW>(tmap, p, x, part, st, skip);
        else
            run_product<WP, float, false, CW>(tmap, p, x, part, st, skip);
    }
    if (e1) record_timing_event(e1, st);
    const int* tab = k2_slot_table(p.nb, p.nk, p.total, p.grid, p.maxseg);
    reduce_launch<WP, bm_of<CW>()>(part, tab, p.nb, p.n, mode, row_mean, scalars, colsums, y, st,
                                   skip);
}

}  // namespace

const int* k2_slot_table_multi(int nb, const std::vector<K2Split>& splits) {
    std::string name = "k2_slots_" + std::to_string(nb);
    for (const K2Split& sp : splits)
        name += "_" + std::to_string(sp.nk) + "_" + std::to_string(sp.total) + "_" +
                std::to_string(sp.P) + "_" + std::to_string(sp.maxseg) + "_" +
                std::to_string(sp.slot_base);
    std::vector<int> host;
    if (!Ctx::get().has_table(name)) {
        // row block -> the slots (slot_base + cta * maxseg + segment) of the
        // CTAs that touched it: split by split, each in CTA order
        std::vector<std::vector<int>> per(nb);
        for (const K2Split& sp : splits)
            for (long long c = 0; c < sp.P; ++c) {
                const long long t0 = sp.total * c / sp.P, t1 = sp.total * (c + 1) / sp.P;
                if (t1 <= t0) continue;
                const long long bf = t0 / sp.nk, bl = (t1 - 1) / sp.nk;
                for (long long b = bf; b <= bl && b < nb; ++b)
                    per[b].push_back(static_cast<int>(sp.slot_base + c * sp.maxseg + (b - bf)));
            }
        host.resize(nb + 1);
        host[0] = 0;
        for (int b = 0; b < nb; ++b) host[b + 1] = host[b] + static_cast<int>(per[b].size());
        for (int b = 0; b < nb; ++b) host.insert(host.end(), per[b].begin(), per[b].end());
    }
    return static_cast<const int*>(
        Ctx::get().const_table(name, host.data(), host.size() * sizeof(int)));
}

const int* k2_slot_table(int nb, int nk, long long total, int P, int maxseg) {
    return k2_slot_table_multi(nb, {K2Split{nk, total, P, maxseg, 0}});
}

void launch_k2_reduce_multi(int wp, int bm, const double* part, const std::vector<K2Split>& splits,
                            int n, int mode, const double* row_mean, const double* scalars,
                            const double* colsums, double* y, cudaStream_t st, const int* skip) {
    const int nb = (n + bm - 1) / bm;
    const int* tab = k2_slot_table_multi(nb, splits);
    switch (wp * 1000 + bm) {
#define DSB_RED(W, B)                                                                          \
    case W * 1000 + B:                                                                         \
        reduce_launch<W, B>(part, tab, nb, n, mode, row_mean, scalars, colsums, y, st, skip);  \
        break;
        DSB_RED(8, 128) DSB_RED(16, 128) DSB_RED(24, 128) DSB_RED(32, 128) DSB_RED(40, 128)
        DSB_RED(48, 128) DSB_RED(56, 128) DSB_RED(64, 128) DSB_RED(72, 128) DSB_RED(80, 128)
        DSB_RED(88, 128) DSB_RED(96, 128) DSB_RED(104, 128) DSB_RED(112, 128)
        DSB_RED(120, 128) DSB_RED(128, 128)
#undef DSB_RED
        default:
            throw std::invalid_argument("unsupported reduce shape");
    }
}

void launch_k2_reduce(int wp, int bm, const double* part, int maxseg, int nk, long long total,
                      int P, int n, int mode, const double* row_mean, const double* scalars,
                      const double* colsums, double* y, cudaStream_t st, const int* skip) {
    launch_k2_reduce_multi(wp, bm, part, {K2Split{nk, total, P, maxseg, 0}}, n, mode, row_mean,
                           scalars, colsums, y, st, skip);
}

int k2_warps(int wp) { return wp <= 64 ? 16 : 8; }

// 128-byte D boxes per pipeline stage (DSB_K2_KS overrides, for sweeps)
int k2_ks(int wp, DType dt) {
    (void)wp;
    (void)dt;
    static const int env = [] {
        const char* e = std::getenv("DSB_K2_KS");
        return e ? std::atoi(e) : 0;
    }();
    if (env == 1 || env == 2) return env;
    return 2;  // halves the per-stage barrier work; +1-4 % DMMA util (tools/k2_sweep.py)
}

K2Plan k2_plan(size_t n, int wp, DType dt, int sms) { return k2_plan_rect(n, n, wp, dt, sms); }

K2Plan k2_plan_rect(size_t n, size_t ncols, int wp, DType dt, int sms) {
    K2Plan p;
    p.wp = wp;
    p.cw = k2_warps(wp);
    p.bm = 16 * p.cw;
    p.n = static_cast<int>(n);
    p.nb = static_cast<int>((n + p.bm - 1) / p.bm);
    p.ks = k2_ks(wp, dt);
    const int kt = (dt == DType::F64 ? 16 : 32) * p.ks;  // columns per stage
    p.nk = static_cast<int>((ncols + kt - 1) / kt);
    p.total = static_cast<long long>(p.nb) * p.nk;
    p.grid = static_cast<int>(std::min<long long>(sms, p.total));
    const int sb = ((p.ks * p.bm * 128 + kt * wp * 8) + 1023) / 1024 * 1024;
    const size_t budget = 222 * 1024;
    int stages = static_cast<int>((budget - 1024 - 256) / sb);
    stages = std::max(2, std::min(stages, 8));
    p.stages = stages;
    p.smem = static_cast<size_t>(stages) * sb + 1024 + 2 * 8 * stages;
    // max row blocks a CTA range touches
    int maxseg = 1;
    for (long long c = 0; c < p.grid; ++c) {
        const long long a = p.total * c / p.grid, b = p.total * (c + 1) / p.grid;
        if (b > a) maxseg = std::max<int>(maxseg, static_cast<int>((b - 1) / p.nk - a / p.nk + 1));
    }
    p.maxseg = maxseg;
    p.part_elems = static_cast<size_t>(p.grid) * maxseg * p.bm * wp;
    return p;
}

void launch_k2(const CUtensorMap* tmap, DType dt, int mode, const K2Plan& p, const double* x,
               double* part, const double* row_mean, const double* scalars,
               const double* colsums, double* y, size_t n_pad, cudaStream_t st, cudaEvent_t e0,
               cudaEvent_t e1, const int* skip) {
    // rows beyond the last BM-row block up to the panel padding must read as
    // zero (BM = 128 for WP > 64 leaves up to 128 rows unwritten)
    const size_t r_done = static_cast<size_t>(p.nb) * p.bm;
    if (n_pad > r_done)
        cudaMemsetAsync(y + r_done * p.wp, 0, (n_pad - r_done) * p.wp * sizeof(double), st);
    switch (p.wp) {
#define DSB_WP(W)                                                                               \
    case W:                                                                                     \
        launch_wp<W, (W <= 64 ? 16 : 8)>(tmap, dt, mode, p, x, part, row_mean, scalars, colsums, \
                                         y, st, e0, e1, skip);                                   \
        break;
        DSB_WP(8)
        DSB_WP(16)
        DSB_WP(24)
        DSB_WP(32)
        DSB_WP(40)
        DSB_WP(48)
        DSB_WP(56)
        DSB_WP(64)
        DSB_WP(72)
        DSB_WP(80)
        DSB_WP(88)
        DSB_WP(96)
        DSB_WP(104)
        DSB_WP(112)
        DSB_WP(120)
        DSB_WP(128)
#undef DSB_WP
        default:
            throw std::invalid_argument("unsupported panel width");
    }
    count_launch(2);
}

}  // namespace dsb
