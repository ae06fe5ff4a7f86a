// K2 on the integer tensor cores — the centered product Y = G X of
// multiply_sym (ref src/rsvd.cpp:18-36 over the gram of mds.cpp:43-58) as an
// exact-integer slice product (Ozaki-style splitting) on tcgen05 kind::i8.
//
// Why: in fp64 the pass is bounded by the FP64 tensor rate (2 n^2 w flops at
// ~37 TF/s: 0.65 ms at C2), above the HBM time of reading D once (0.49 ms).
// Integer MMAs run ~60x faster, so the pass becomes HBM-bound again.
//
// Splitting (all scalings are exact powers of two):
//   S_ij = d_ij^2 = 2^e_i  * sum_{t=1..7} a_t 2^-8t,  a_t in [0,255]  (e_i: K1 row
//          exponent, d^2 < 2^e_i; the 56-bit fixed-point value is truncated)
//   X_jc = 2^f_c  * sum_{u=1..7} b_u 2^-8u,  b_u in [-128,127] (balanced digits
//          of round(X 2^(56-f_c)), |X| 2^-f_c < 1/4)
//   (S X)_ic = 2^(e_i+f_c) sum_{d=2..8} 2^-8d acc_d,  acc_d = sum_j sum_{t+u=d} a_t b_u
// The terms with t+u >= 9 (weight <= 2^-72) are dropped; each acc_d is an
// exact int32 sum over at most 8192 columns (7 * 255 * 128 * 8192 < 2^31;
// Hamming slices: 3 products per diagonal, 16384 columns), after which it is
// flushed to fp64. Digits of S are produced on the fly from
// the fp64 (or fp32) D tile, so HBM traffic is exactly one read of D per
// pass, as in the fp64 kernel.
//
// MMA structure (one CTA per SM, persistent, stream-K over (128-row block x
// 32-column k-step) like the fp64 kernel): for each A digit t one
// tcgen05.mma (M=128, K=32) against the CONCATENATION of B digits
// 1..8-t (N' = (8-t) NB <= 256, else split), writing TMEM columns
// (t-1) NB.. — so digit pair (t, u) lands on the accumulator of its
// diagonal d = t+u: 28 digit products per k-step.
//
// Warp roles: warp 0 TMA producer of D tiles (128 rows x 128 B boxes,
// SWIZZLE_128B) (and, with a single A stage, of the panel digits); warp 1
// TMEM owner + single-thread MMA issuer; warps 2-17 converters (d -> d^2 ->
// 56-bit fixed point -> byte planes, written into TMEM with tcgen05.st, see
// k2i_product_ts below), converters 0-3 double as the epilogue (tcgen05.ld
// of the 7 diagonals, fp64 combine, exact 2^(e+f) scaling, partial slot RMW).
// k2_reduce sums the partial slots in CTA order and applies the centering.
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "device_utils.cuh"
#include "host_core.hpp"
#include "kernels.cuh"
#include "sdig.cuh"
#include "umma.cuh"

namespace dsb {

namespace {

constexpr int kRowsI8 = 128;   // M
constexpr int kKStep = 32;     // int8 MMA K
constexpr int kDig = 7;        // digits of S and of X
constexpr int kChunk = 256;    // k-steps per int32 accumulation chunk (8192 columns)
// Hamming slices: a diagonal sums at most 3 digit products (t <= 3), so
// 3 * 255 * 128 * 16384 < 2^31: chunks twice as long, half the flushes
template <int SD>
constexpr int chunk_ks() {
    return SD == 3 ? 512 : kChunk;
}
constexpr int kConv = 16;      // converter warps (8 rows each)
constexpr int kThreadsI8 = (2 + kConv) * 32;
constexpr int kExpZeroI8 = -1100;  // matches K1's exponent of an all-zero row

template <int NB>
constexpr int b_bytes() {
    return kDig * NB * kKStep;
}
template <typename TD>
constexpr int d_bytes() {
    return kRowsI8 * kKStep * static_cast<int>(sizeof(TD));
}
// Walks a CTA's stream-K range [t0, t1) of (row block, k-step) items without
// divisions: row block, k-step, segment index and position in the int32
// accumulation chunk (chunks restart at every row block).
template <int CH = kChunk>
struct Walk {
    int it, t1, nks, rb, ks, seg, pos;
    bool seg_first;  // the current chunk is the first one of its segment
    __device__ Walk(int t0_, int t1_, int nks_)
        : it(t0_), t1(t1_), nks(nks_), rb(t0_ / nks_), ks(t0_ % nks_), seg(0), pos(0),
          seg_first(true) {}
    __device__ bool more() const { return it < t1; }
    __device__ bool first() const { return pos == 0; }
    __device__ bool last() const { return it + 1 == t1 || ks + 1 == nks || pos + 1 == CH; }
    __device__ void next() {
        ++it;
        ++ks;
        ++pos;
        if (ks == nks) {
            ks = 0;
            ++rb;
            ++seg;
            pos = 0;
            seg_first = true;
        } else if (pos == CH) {
            pos = 0;
            seg_first = false;
        }
    }
};

// ---- A digits in tensor memory ---------------------------------------------
// An MMA whose A operand comes from shared memory costs at least ~128 cycles
// (the 4 KB A tile is read at ~32 B/clk; tools/microbench/umma_i8_rate.cu),
// so the digit MMAs of a k-step (N' = 224..32) ran at half the tensor rate or
// worse. With A in TMEM (written by the converters with tcgen05.st) each MMA
// takes N'/2 cycles: 448 (NB = 32) / 896 (NB = 64) cycles per k-step, under
// the ~1400-cycle HBM time of the k-step's 32 KB of D.
// TMEM: columns [0, 7 NB) the diagonal accumulators, then NA stages of the
// 7 x 8-column A digit planes (row = lane, byte k at column k / 4): NA = 4
// for NB = 32, NA = 1 for NB = 64 (448 + 56 columns). With one A stage the
// converters overlap the next k-step's conversion (into registers) with the
// MMAs of the current one and only the TMEM stores wait for the stage.
// The panel digits stream through their own ring (the producer warp issues
// them next to the D tiles; the MMA commits free both).
// Converter warp w (2..17) handles tile rows 32 (w % 4) + lane (its TMEM lane
// quadrant) and columns 8 p .. 8 p + 7 of the k-step, p = (w - 2) / 4.
#ifndef DSB_TS_SMEM_KB
#define DSB_TS_SMEM_KB 208
#endif

constexpr int kBStagesTs = 4;
#ifndef DSB_K2I_WARP_ISSUE
#define DSB_K2I_WARP_ISSUE 1
#endif
constexpr bool kWarpIssue = DSB_K2I_WARP_ISSUE != 0;
// panel digits get their own producer-filled ring when the A ring is this
// shallow or shallower: the 2-deep NB = 64 A ring too (w = 120 on f32 D,
// n = 60k: 13.3 -> 12.7 ms per pass; NB = 64 f64 and the Hamming slices
// unchanged)
#ifndef DSB_TS_BPROD_NA
#define DSB_TS_BPROD_NA 2
#endif
template <int NB, int SD = kDig, int DM = 0>
constexpr bool bprod_ts();


#ifndef DSB_TS_NB64_HYBRID
#define DSB_TS_NB64_HYBRID 1
#endif
// NB = 64 hybrid: digits 1..4 of each A stage in TMEM (4 x 8 columns, two
// stages in the 64 columns left after the 448 accumulator columns), digits
// 5..7 — whose MMAs are narrow (N' <= 192) and so pay the shared-memory
// A floor anyway — from shared memory. Two stages let the conversion of the
// next k-step proceed while the MMAs of the current one run.
// SD: digits of S per element — 7 (56-bit fixed point of d^2 per row) or 3
// (Hamming distances: d = h / L with integer h, S = h^2 / L^2 exactly, h^2 <
// 2^24 in three bytes; see launch_k2i)
template <int NB, int SD = kDig>
constexpr bool hybrid_ts() {
    return NB > 48 && SD > 4 && DSB_TS_NB64_HYBRID;
}
template <int NB, int SD = kDig>
constexpr int tmem_digits_ts() {
    return hybrid_ts<NB, SD>() ? 4 : SD;
}
// NB = 32: four 64-column A stages after the 224 accumulator columns (a
// fifth 56-column stage fits — DSB_TS_NA32=5 DSB_TS_ACOLS32=56
// DSB_TS_ABASE32=224 — and measured no faster)
#ifndef DSB_TS_NA32
#define DSB_TS_NA32 4
#endif
template <int NB, int SD = kDig>
constexpr uint32_t a_stage_cols_ts();
template <int NB>
constexpr uint32_t a_base_ts();
template <int NB, int SD = kDig>
constexpr int a_stages_ts() {
    // NB = 32: four 64-column stages; NB = 48: the 3 x 56 columns after the
    // 336 accumulator columns; NB = 64: two (hybrid / 3-byte) or one stage
    return NB <= 32 ? DSB_TS_NA32
                    : (NB <= 48 ? static_cast<int>((512u - a_base_ts<NB>()) / a_stage_cols_ts<NB, SD>()) > 4
                                      ? 4
                                      : static_cast<int>((512u - a_base_ts<NB>()) /
                                                         a_stage_cols_ts<NB, SD>())
                                : ((hybrid_ts<NB, SD>() || 16 * SD <= 64) ? 2 : 1));
}
#ifndef DSB_TS_ACOLS32
#define DSB_TS_ACOLS32 64
#endif
#ifndef DSB_TS_ABASE32
#define DSB_TS_ABASE32 256
#endif
template <int NB, int SD>
constexpr uint32_t a_stage_cols_ts() {
    return SD != kDig ? 8u * SD
                      : (hybrid_ts<NB, SD>() ? 32u
                                             : (NB <= 32 ? DSB_TS_ACOLS32 : (NB <= 48 ? 56u : 64u)));
}
template <int NB>
constexpr uint32_t a_base_ts() {  // first TMEM column of the A stages
    return NB <= 32 ? DSB_TS_ABASE32 : static_cast<uint32_t>(7 * NB);
}
template <int NB, int SD = kDig>
constexpr int a_smem_stage_ts() {  // bytes of shared-memory A digits per stage
    return (SD - tmem_digits_ts<NB, SD>()) * kRowsI8 * kKStep;
}
template <int NB, int SD = kDig, int DM = 0>
constexpr int b_stages_ts() {
    return bprod_ts<NB, SD, DM>() ? kBStagesTs : a_stages_ts<NB, SD>();
}
// streaming the S-digit cache (DM = 2) an A stage turns over in ~the MMA
// time, too fast to hide a panel-digit load issued when the stage is claimed:
// the producer streams them ahead then too
template <int NB, int SD, int DM>
constexpr bool bprod_ts() {
    return DM == 2 || a_stages_ts<NB, SD>() <= DSB_TS_BPROD_NA;
}
// shared-memory budget of the rings: the CTA pair (NB = 48 and the pair's
// NB = 64 launches) feeds TWO SMs' bandwidth from one D ring, so it takes the
// maximum; the single-CTA kernel keeps the measured-best 208 KB
#ifndef DSB_TS_PAIR_SMEM_KB
#define DSB_TS_PAIR_SMEM_KB 224
#endif
// bytes of one ring slot: the D tile, or (DM = 2) an item's digit planes
template <typename TD, int SD, int DM>
constexpr int slot_bytes() {
    return DM == 2 ? sdig_item_bytes<SD>() : d_bytes<TD>();
}
// streaming the cache with 4 A stages, the converters work in 4 groups that
// take items round-robin (k2i_product_ts); each group must own its ring slots
// and A stage (an mbarrier wait tells phases apart by parity only, so a group
// running ahead on a slot another group still has to see would pass a wait it
// should block on): the D ring depth is then a multiple of 4
template <int NB, int SD, int DM>
constexpr int conv_groups_ts() {
    // one group of 4 converter warps per A stage (2, 3 or 4 stages)
    return (DM == 2 && a_stages_ts<NB, SD>() >= 2 && a_stages_ts<NB, SD>() <= 4)
               ? a_stages_ts<NB, SD>()
               : 1;
}
template <int NB, typename TD, int SD = kDig, int CL = 1, int DM = 0>
constexpr int d_stages_ts() {
    return std::min(8, ((CL > 1 ? DSB_TS_PAIR_SMEM_KB : DSB_TS_SMEM_KB) * 1024 -
                        b_stages_ts<NB, SD, DM>() * b_bytes<NB>() -
                        a_stages_ts<NB, SD>() * a_smem_stage_ts<NB, SD>()) /
                           slot_bytes<TD, SD, DM>()) /
           conv_groups_ts<NB, SD, DM>() * conv_groups_ts<NB, SD, DM>();
}
template <int NB, typename TD, int SD = kDig, int CL = 1, int DM = 0>
constexpr size_t ts_smem() {
    return 1024 +
           static_cast<size_t>(d_stages_ts<NB, TD, SD, CL, DM>()) * slot_bytes<TD, SD, DM>() +
           b_stages_ts<NB, SD, DM>() * b_bytes<NB>() +
           a_stages_ts<NB, SD>() * a_smem_stage_ts<NB, SD>() + 448 + NB * 8;
}

// 8 consecutive d values of row `row`, columns c0..c0+7 of the k-step tile
template <typename TD>
__device__ __forceinline__ void load8(const unsigned char* tile, int row, int c0, double (&d)[8]) {
    if constexpr (sizeof(TD) == 8) {
        const unsigned char* box = tile + (c0 >> 4) * (kRowsI8 * 128) + row * 128;
        const int c = (c0 & 15) >> 1;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const double2 v = *reinterpret_cast<const double2*>(box + (((c + h) ^ (row & 7)) << 4));
            d[2 * h] = v.x;
            d[2 * h + 1] = v.y;
        }
    } else {
        const unsigned char* rp = tile + row * 128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 v =
                *reinterpret_cast<const float4*>(rp + ((((c0 >> 2) + h) ^ (row & 7)) << 4));
            d[4 * h] = v.x;
            d[4 * h + 1] = v.y;
            d[4 * h + 2] = v.z;
            d[4 * h + 3] = v.w;
        }
    }
}

// an item's digit planes t = 1..SD of (row, converter part) from a ring
// slot / into the cache (sdig_off layout)
template <int SD>
__device__ __forceinline__ void sdig_read(const unsigned char* slot, int row, int part,
                                          uint32_t (&wd)[SD][2]) {
#pragma unroll
    for (int t = 1; t <= SD; ++t) {
        const uint2 v = *reinterpret_cast<const uint2*>(slot + sdig_off(row, part, t, SD));
        wd[t - 1][0] = v.x;
        wd[t - 1][1] = v.y;
    }
}
template <int SD>
__device__ __forceinline__ void sdig_write(unsigned char* item, int row, int part,
                                           const uint32_t (&wd)[SD][2]) {
#pragma unroll
    for (int t = 1; t <= SD; ++t)
        *reinterpret_cast<uint2*>(item + sdig_off(row, part, t, SD)) =
            make_uint2(wd[t - 1][0], wd[t - 1][1]);
}

// CL = 2: a cluster of two CTAs (on two SMs) shares every D tile — each
// CTA TMA-loads one 64-row half of the tile and multicasts it to both, so D
// is read from HBM once per pass — and each CTA multiplies it into its own
// column group (panel columns cg0 + rank NB ..): two 48- or 64-column groups
// cover w <= 128 in ONE pass, where one SM's TMEM holds at most 64 columns x
// 7 diagonal accumulators. Both CTAs convert the whole tile (their MMAs need
// every row's digits in their own TMEM); a slot of the D ring is refilled
// only after the consumers of BOTH CTAs released it (each consumer warp
// arrives on its own and on the peer's empty barrier). tmD then has 64-row
// boxes; bdig holds the groups' digit planes bdig_stride bytes apart.
// DM: S-digit cache mode (see sdig_item_bytes): 0 off, 1 convert and store
// the items' digit planes at sdig, 2 stream them from sdig (no D tile, no
// conversion). Items are indexed rb * nks_c + global k-step. Streaming, a
// cluster of up to 4 CTAs shares every item (each bulk-loads 1/CL of it,
// multicast to all) with one NB = 32 column group per CTA: with nothing to
// convert, the narrow groups' 4 A stages and short MMA sequence keep the
// tensor pipe fed where one CTA's 48/64-column group could not.
template <int NB, typename TD, int SD, int CL, int DM = 0>
__global__ void __launch_bounds__(kThreadsI8, 1)
    k2i_product_ts(const __grid_constant__ CUtensorMap tmD, const unsigned char* __restrict__ bdig,
                   const int* __restrict__ row_exp, const int* __restrict__ col_exp, int nrows,
                   int nks, int total, double* __restrict__ part, int maxseg, int wp, int cg0,
                   const int* __restrict__ skip, int dbg, double hlen, size_t bdig_stride,
                   int k_off, unsigned char* __restrict__ sdig, int nks_c) {
    // k_off: first global k-step of this launch (a column range of D and the
    // matching panel rows; the walk's k-steps are local to the range)
    if (skip && *skip) return;
    static_assert(CL == 1 || CL == 2 || (DM == 2 && CL <= 4),
                  "one CTA, a pair sharing the D tiles, or up to 4 CTAs sharing the digit items");
    const int crank = CL > 1 ? static_cast<int>(cluster_ctarank()) : 0;
    cg0 += crank * NB;
    bdig += static_cast<size_t>(crank) * bdig_stride;
    static_assert(SD == kDig || SD == 3, "S digit counts: 7 (general) or 3 (Hamming)");
    static_assert(DM >= 0 && DM <= 2, "S-digit cache mode");
    constexpr int ND = d_stages_ts<NB, TD, SD, CL, DM>();
    constexpr int NA = a_stages_ts<NB, SD>();
    // panel digits: with several A stages they ride with the A stage (loaded
    // by one converter lane when it claims the stage); with a single A stage
    // they get their own ring filled ahead by the producer
    constexpr bool kBProd = bprod_ts<NB, SD, DM>();
    constexpr int NBR = kBProd ? kBStagesTs : NA;
    constexpr int DB = slot_bytes<TD, SD, DM>();  // one slot of the D ring
    constexpr int IB = sdig_item_bytes<SD>();
    constexpr int BB = b_bytes<NB>();
    constexpr int TD_DIG = tmem_digits_ts<NB, SD>();  // digits 1..TD_DIG in TMEM
    constexpr int ASB = a_smem_stage_ts<NB, SD>();     // the rest in shared memory
    constexpr uint32_t ACOLS = a_stage_cols_ts<NB, SD>();
    // converter warps per item: all 16 (each 8 of the 32 columns), or, when
    // streaming the cache (nothing to convert), groups of 4 warps (one per
    // TMEM lane quadrant, all 32 columns) taking items round-robin, so that
    // four items' load -> tcgen05.st -> arrive chains overlap
    constexpr int kGrp = conv_groups_ts<NB, SD, DM>();
    static_assert(kGrp == 1 || (ND % kGrp == 0 && NA % kGrp == 0), "groups own their slots");
    constexpr int kCW = kGrp > 1 ? 4 : kConv;  // converter warps per item

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* dring = sm;
    unsigned char* bring = sm + ND * DB;
    unsigned char* aring = bring + NBR * BB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(aring + NA * ASB);
    uint64_t* full_d = bars;
    uint64_t* empty_d = full_d + ND;
    uint64_t* full_a = empty_d + ND;
    uint64_t* empty_a = full_a + NA;
    uint64_t* full_b = empty_a + NA;
    uint64_t* empty_b = full_b + NBR;
    uint64_t* acc_full = empty_b + NBR;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
    double* colscale = reinterpret_cast<double*>(bars + 56);  // <= 34 barriers + slot

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // work unit: the CTA, or the pair (both CTAs walk the same items)
    const int cta = blockIdx.x / CL;
    const int units = gridDim.x / CL;
    const int t0 = static_cast<int>(static_cast<long long>(total) * cta / units);
    const int t1 = static_cast<int>(static_cast<long long>(total) * (cta + 1) / units);

    if (threadIdx.x == 0) {
        for (int s = 0; s < ND; ++s) {
            mbar_init(&full_d[s], 1);
            mbar_init(&empty_d[s], kCW * CL);  // every CTA's converters of the item
        }
        for (int s = 0; s < NA; ++s) {
            // with the digits riding on the A stage, their expect_tx arrival
            // is the stage's 17th
            mbar_init(&full_a[s], kBProd ? kCW : kCW + 1);
            mbar_init(&empty_a[s], 1);
        }
        for (int s = 0; s < NBR; ++s) {
            mbar_init(&full_b[s], 1);
            mbar_init(&empty_b[s], 1);
        }
        static_assert(kBProd || NBR == NA, "B ring rides with the A ring");
        static_assert(kBProd || NA > 1, "a single A stage needs the producer's B ring");
        static_assert(a_base_ts<NB>() + NA * ACOLS <= 512 && a_base_ts<NB>() >= 7 * NB,
                      "A stages fit in TMEM after the accumulators");
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 4);
        fence_mbar_init();
    }
    // this launch's column group: panel columns cg0 .. cg0 + NB - 1
    for (int c = threadIdx.x; c < NB; c += blockDim.x) {
        const int f = cg0 + c < wp ? col_exp[cg0 + c] : kExpZeroI8;
        colscale[c] = f > kExpZeroI8 ? ldexp(1.0, f) : 0.0;
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    if constexpr (CL > 1)
        cluster_sync_all();  // the peer's barriers are initialized before any remote use
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tmem_a = tmem + a_base_ts<NB>();

    if (warp == 0) {
        // ---------------- TMA producer: D tiles and panel digits ----------------
        if (lane == 0) {
            if constexpr (DM != 2) prefetch_tmap(&tmD);
            // streaming: the items pass through L2 once (evict first), the
            // panel digits every row block re-reads stay (evict last)
            const uint64_t pol_item = l2_policy(true), pol_panel = l2_policy(false);
            (void)pol_item;
            (void)pol_panel;
            int sd = 0, sb = 0, k = 0;
            uint32_t pd = 0, pb = 0;
            for (Walk<chunk_ks<SD>()> w(t0, t1, nks); w.more(); w.next(), ++k) {
                if (k >= ND) mbar_wait(&empty_d[sd], pd ^ 1);
                unsigned char* dst = dring + sd * DB;
                mbar_arrive_expect_tx(&full_d[sd], DB);  // the whole tile / item
                if constexpr (DM == 2) {
                    // the item's digit planes (each CTA of a pair fetches one
                    // 64-row half into both)
                    const unsigned char* src =
                        sdig + (static_cast<size_t>(w.rb) * nks_c + k_off + w.ks) * IB;
                    if constexpr (CL > 1) {
                        // this CTA's 1/CL of the item, into every CTA of the cluster
                        constexpr int CH = (IB / CL + 15) / 16 * 16;
                        const int off = crank * CH;
                        bulk_load_mc_pol(dst + off, src + off,
                                         static_cast<uint32_t>(IB - off < CH ? IB - off : CH),
                                         &full_d[sd], static_cast<uint16_t>((1u << CL) - 1u),
                                         pol_item);
                    } else
                        bulk_load_pol(dst, src, IB, &full_d[sd], pol_item);
                } else if constexpr (CL > 1) {
                    // this CTA's 64-row half of the tile, into both CTAs
                    // (64 rows x 128 B keeps the SWIZZLE_128B phase)
                    const int r0 = w.rb * kRowsI8 + 64 * crank;
                    unsigned char* hd = dst + crank * (64 * 128);
                    tma_load_2d_mc(hd, &tmD, (k_off + w.ks) * kKStep, r0, &full_d[sd], 0x3);
                    if constexpr (sizeof(TD) == 8)
                        tma_load_2d_mc(hd + kRowsI8 * 128, &tmD, (k_off + w.ks) * kKStep + 16, r0,
                                       &full_d[sd], 0x3);
                } else if constexpr (sizeof(TD) == 8) {
                    tma_load_2d(dst, &tmD, (k_off + w.ks) * kKStep, w.rb * kRowsI8, &full_d[sd]);
                    tma_load_2d(dst + kRowsI8 * 128, &tmD, (k_off + w.ks) * kKStep + 16,
                                w.rb * kRowsI8, &full_d[sd]);
                } else {
                    tma_load_2d(dst, &tmD, (k_off + w.ks) * kKStep, w.rb * kRowsI8, &full_d[sd]);
                }
                if (++sd == ND) {
                    sd = 0;
                    pd ^= 1;
                }
                if constexpr (kBProd) {
                    if (k >= NBR) mbar_wait(&empty_b[sb], pb ^ 1);
                    mbar_arrive_expect_tx(&full_b[sb], BB);
                    if constexpr (DM == 2)
                        bulk_load_pol(bring + sb * BB,
                                      bdig + static_cast<size_t>(k_off + w.ks) * BB, BB,
                                      &full_b[sb], pol_panel);
                    else
                        bulk_load(bring + sb * BB, bdig + static_cast<size_t>(k_off + w.ks) * BB,
                                  BB, &full_b[sb]);
                    if (++sb == NBR) {
                        sb = 0;
                        pb ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // the whole warp runs the issuer loop (warp-uniform operands, one
        // elected lane issues); DSB_K2I_WARP_ISSUE=0 restores the lane-0 loop
        if (kWarpIssue || lane == 0) {
            int sa = 0, sb = 0, nflush = 0;
            uint32_t pa = 0, pb = 0;
            bool started = false;
            for (Walk<chunk_ks<SD>()> w(t0, t1, nks); w.more(); w.next()) {
                mbar_wait(&full_a[sa], pa);
                if constexpr (kBProd) mbar_wait(&full_b[sb], pb);
                tc_fence_after();
                const bool first = w.first();
                if (first && started) {
                    mbar_wait(acc_empty, static_cast<uint32_t>((nflush - 1) & 1));
                    tc_fence_after();
                }
                started = true;
                const uint32_t bbase = smem_u32(bring + sb * BB);
                const uint32_t ta = tmem_a + static_cast<uint32_t>(sa) * ACOLS;
                const uint32_t asm_base = smem_u32(aring + sa * ASB);
                if (dbg != 2) {
#pragma unroll
                    for (int t = 1; t <= SD; ++t) {
                        constexpr int per = 256 / NB;
                        const int umax = 8 - t;
#pragma unroll
                        for (int u0 = 1; u0 <= umax; u0 += per) {
                            const int nu = (umax - u0 + 1 < per) ? (umax - u0 + 1) : per;
                            const uint64_t bd =
                                umma_desc_k_interleave(bbase + (u0 - 1) * (NB * kKStep));
                            const uint32_t dcol = tmem + static_cast<uint32_t>((t + u0 - 2) * NB);
                            const uint32_t idesc = umma_idesc_i8(nu * NB, false, true);
                            const int acc = (first && t == 1) ? 0 : 1;
                            if (t <= TD_DIG) {
                                const uint32_t ta_t = ta + static_cast<uint32_t>((t - 1) * 8);
                                if constexpr (kWarpIssue)
                                    umma_i8_ts_w(dcol, ta_t, bd, idesc, acc);
                                else
                                    umma_i8_ts(dcol, ta_t, bd, idesc, acc);
                            } else {
                                const uint64_t ad = umma_desc_k_interleave(
                                    asm_base + (t - TD_DIG - 1) * (kRowsI8 * kKStep));
                                if constexpr (kWarpIssue)
                                    umma_i8_w(dcol, ad, bd, idesc, acc);
                                else
                                    umma_i8(dcol, ad, bd, idesc, acc);
                            }
                        }
                    }
                }
                if constexpr (kWarpIssue) {
                    umma_commit_w(&empty_a[sa]);
                    if constexpr (kBProd) umma_commit_w(&empty_b[sb]);
                } else {
                    umma_commit(&empty_a[sa]);
                    if constexpr (kBProd) umma_commit(&empty_b[sb]);
                }
                if (w.last()) {
                    if constexpr (kWarpIssue)
                        umma_commit_w(acc_full);
                    else
                        umma_commit(acc_full);
                    ++nflush;
                }
                if (++sa == NA) {
                    sa = 0;
                    pa ^= 1;
                }
                if (++sb == NBR) {
                    sb = 0;
                    pb ^= 1;
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- converters (+ epilogue on p == 0) ----------------
        const int q = warp & 3;
        const int part_k = (warp - 2) >> 2;
        const int row = q * 32 + lane;
        const int c0 = part_k * 8;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        // ---- epilogue of an accumulation chunk: this warp's 32 TMEM lanes ----
        auto epilogue = [&](const Walk<chunk_ks<SD>()>& w, int nfl) {
            mbar_wait(acc_full, static_cast<uint32_t>(nfl & 1));
            tc_fence_after();
            const int grow = w.rb * kRowsI8 + row;
            double rscale;
            if constexpr (SD == kDig) {
                const int e = grow < nrows ? row_exp[grow] : kExpZeroI8;
                rscale = e > kExpZeroI8 ? ldexp(1.0, e) : 0.0;
            } else {
                rscale = grow < nrows ? 0x1.0p24 / (hlen * hlen) : 0.0;  // S = S' 2^-24 * this
            }
            double* prow = part +
                           (static_cast<size_t>(cta) * maxseg + w.seg) * kRowsI8 * wp +
                           static_cast<size_t>(row) * wp;
#pragma unroll
            for (int cb = 0; cb < NB / 16; ++cb) {
                double v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = 0.0;
#pragma unroll
                for (int dd = 2; dd <= 8; ++dd) {
                    int32_t iv[16];
                    tmem_ld16(tmem + lane_off + static_cast<uint32_t>((dd - 2) * NB + cb * 16),
                              iv);
                    tmem_ld_wait();
                    const double wgt = ldexp(1.0, -8 * dd);
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] += static_cast<double>(iv[j]) * wgt;
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int col = cg0 + cb * 16 + j;
                    if (col < wp) {
                        const double val = v[j] * rscale * colscale[col - cg0];
                        prow[col] = w.seg_first ? val : prow[col] + val;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
        };
        if constexpr (kGrp > 1) {
            // streaming the cache: group part_k takes items k = part_k mod kGrp
            // (and so always the same ring slots and A stage); every group
            // walks every item to keep the ring indices
            int sd = 0, sa = 0, k = 0, nflush = 0;
            uint32_t pd = 0, pa = 0;
            for (Walk<chunk_ks<SD>()> w(t0, t1, nks); w.more(); w.next(), ++k) {
                if (k % kGrp == part_k) {
                    mbar_wait(&full_d[sd], pd);
                    if (k >= NA) {
                        mbar_wait(&empty_a[sa], pa ^ 1);
                        tc_fence_after();
                    }
                    if (dbg != 1) {
                        const unsigned char* slot = dring + sd * DB;
                        const uint32_t ta = tmem_a + static_cast<uint32_t>(sa) * ACOLS + lane_off;
#pragma unroll
                        for (int t = 1; t <= SD; ++t) {
                            uint32_t v[8];
#pragma unroll
                            for (int pp = 0; pp < 4; ++pp) {
                                const uint2 u = *reinterpret_cast<const uint2*>(
                                    slot + sdig_off(row, pp, t, SD));
                                v[2 * pp] = u.x;
                                v[2 * pp + 1] = u.y;
                            }
                            if (t <= TD_DIG) {
                                tmem_st8(ta + static_cast<uint32_t>((t - 1) * 8), v);
                            } else {
#pragma unroll
                                for (int pp = 0; pp < 4; ++pp)
                                    *reinterpret_cast<uint2*>(aring + sa * ASB +
                                                              umma_tile_off(row, pp * 8) +
                                                              (t - TD_DIG - 1) * (kRowsI8 * kKStep)) =
                                        make_uint2(v[2 * pp], v[2 * pp + 1]);
                            }
                        }
                        tmem_st_wait();
                        if constexpr (TD_DIG < SD) fence_proxy_async();
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&empty_d[sd]);
                        mbar_arrive(&full_a[sa]);
                    }
                    if constexpr (CL > 1)
                        if (lane >= 1 && lane < CL)
                            mbar_arrive_peer(&empty_d[sd],
                                             static_cast<uint32_t>((crank + lane) % CL));
                }
                if (++sd == ND) {
                    sd = 0;
                    pd ^= 1;
                }
                if (++sa == NA) {
                    sa = 0;
                    pa ^= 1;
                }
                if (w.last()) {
                    // the chunk epilogues stay on group 0: a partial slot's
                    // read-modify-writes of consecutive chunks of one row
                    // block are then ordered by program order
                    if (part_k == 0) epilogue(w, nflush);
                    ++nflush;
                }
            }
        } else {
        int cur_rb = -1;
        double sc = 0.0;
        int sd = 0, sa = 0, k = 0, nflush = 0;
        uint32_t pd = 0, pa = 0;
        for (Walk<chunk_ks<SD>()> w(t0, t1, nks); w.more(); w.next(), ++k) {
            if (SD == kDig && w.rb != cur_rb) {
                cur_rb = w.rb;
                const int grow = w.rb * kRowsI8 + row;
                const int e = grow < nrows ? row_exp[grow] : kExpZeroI8;
                sc = e > kExpZeroI8 ? ldexp(1.0, 56 - e) : 0.0;
            }
            mbar_wait(&full_d[sd], pd);
            if constexpr (NA > 1) {
                // several A stages: claim the stage (and load its panel
                // digits, unless the producer streams them) first, then
                // convert and store digit by digit
                if (k >= NA) {
                    mbar_wait(&empty_a[sa], pa ^ 1);
                    tc_fence_after();
                }
                if (!kBProd && warp == 2 && lane == 0) {
                    mbar_arrive_expect_tx(&full_a[sa], BB);
                    bulk_load(bring + sa * BB, bdig + static_cast<size_t>(k_off + w.ks) * BB, BB,
                              &full_a[sa]);
                }
                if (dbg != 1) {
                    const uint32_t ta = tmem_a + static_cast<uint32_t>(sa) * ACOLS + lane_off;
                    unsigned char* as = aring + sa * ASB + umma_tile_off(row, c0);
                    uint32_t wd[SD][2];
                    if constexpr (DM == 2) {
                        sdig_read<SD>(dring + sd * DB, row, part_k, wd);
                    } else {
                    double d[8];
                    load8<TD>(dring + sd * DB, row, c0, d);
                    if constexpr (SD == kDig) {
                        uint32_t lo[8], hi[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const unsigned long long m = __double2ull_rz((d[j] * d[j]) * sc);
                            lo[j] = static_cast<uint32_t>(m);
                            hi[j] = static_cast<uint32_t>(m >> 32);
                        }
                        pack_digits(lo, hi, wd);
                    } else {
                        // Hamming: h = L d exactly (d = fl(h / L), h <= L < 2^12),
                        // S' = h^2 < 2^24 in three bytes, high first
                        uint32_t s2[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const uint32_t h = static_cast<uint32_t>(__double2int_rn(d[j] * hlen));
                            s2[j] = h * h;
                        }
#pragma unroll
                        for (int g = 0; g < 2; ++g) {
                            const int e = 4 * g;
                            // plane t: byte j = byte (3 - t) of element 4 g + j
                            const uint32_t h01 = __byte_perm(s2[e], s2[e + 1], 0x0062);
                            const uint32_t h23 = __byte_perm(s2[e + 2], s2[e + 3], 0x0062);
                            const uint32_t m01 = __byte_perm(s2[e], s2[e + 1], 0x0051);
                            const uint32_t m23 = __byte_perm(s2[e + 2], s2[e + 3], 0x0051);
                            const uint32_t l01 = __byte_perm(s2[e], s2[e + 1], 0x0040);
                            const uint32_t l23 = __byte_perm(s2[e + 2], s2[e + 3], 0x0040);
                            wd[0][g] = __byte_perm(h01, h23, 0x5410);
                            wd[1][g] = __byte_perm(m01, m23, 0x5410);
                            wd[2][g] = __byte_perm(l01, l23, 0x5410);
                        }
                    }
                    if constexpr (DM == 1)
                        if (CL == 1 || (row >> 6) == crank)
                            sdig_write<SD>(
                                sdig + (static_cast<size_t>(w.rb) * nks_c + k_off + w.ks) * IB,
                                row, part_k, wd);
                    }
#pragma unroll
                    for (int t = 1; t <= SD; ++t) {
                        const uint32_t w0 = wd[t - 1][0], w1 = wd[t - 1][1];
                        if (t <= TD_DIG)
                            tmem_st2(ta + static_cast<uint32_t>((t - 1) * 8 + part_k * 2), w0, w1);
                        else
                            *reinterpret_cast<uint2*>(as + (t - TD_DIG - 1) * (kRowsI8 * kKStep)) =
                                make_uint2(w0, w1);
                    }
                    tmem_st_wait();
                    if constexpr (TD_DIG < SD) fence_proxy_async();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty_d[sd]);
                    mbar_arrive(&full_a[sa]);
                }
                if constexpr (CL > 1)
                    if (lane >= 1 && lane < CL)
                        mbar_arrive_peer(&empty_d[sd], static_cast<uint32_t>((crank + lane) % CL));
            } else {
                // single A stage: convert into registers while the MMAs of the
                // previous k-step still read the stage, then store
                uint32_t wd[kDig][2];
                static_assert(NA > 1 || SD == kDig, "one A stage: general slices only");
                if (dbg != 1) {
                    if constexpr (DM == 2) {
                        sdig_read<kDig>(dring + sd * DB, row, part_k, wd);
                    } else {
                        double d[8];
                        load8<TD>(dring + sd * DB, row, c0, d);
                        uint32_t lo[8], hi[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const unsigned long long m = __double2ull_rz((d[j] * d[j]) * sc);
                            lo[j] = static_cast<uint32_t>(m);
                            hi[j] = static_cast<uint32_t>(m >> 32);
                        }
                        pack_digits(lo, hi, wd);
                        if constexpr (DM == 1)
                            if (CL == 1 || (row >> 6) == crank)
                                sdig_write<kDig>(
                                    sdig + (static_cast<size_t>(w.rb) * nks_c + k_off + w.ks) * IB,
                                    row, part_k, wd);
                    }
                }
                if (k >= NA) {
                    mbar_wait(&empty_a[sa], pa ^ 1);
                    tc_fence_after();
                }
                if (dbg != 1) {
                    const uint32_t ta = tmem_a + static_cast<uint32_t>(sa) * ACOLS + lane_off;
#pragma unroll
                    for (int t = 1; t <= kDig; ++t)
                        tmem_st2(ta + static_cast<uint32_t>((t - 1) * 8 + part_k * 2),
                                 wd[t - 1][0], wd[t - 1][1]);
                    tmem_st_wait();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty_d[sd]);
                    mbar_arrive(&full_a[sa]);
                }
                if constexpr (CL > 1)
                    if (lane >= 1 && lane < CL)
                        mbar_arrive_peer(&empty_d[sd], static_cast<uint32_t>((crank + lane) % CL));
            }
            if (++sd == ND) {
                sd = 0;
                pd ^= 1;
            }
            if (++sa == NA) {
                sa = 0;
                pa ^= 1;
            }
            if (part_k == 0 && w.last()) {
                epilogue(w, nflush);
                ++nflush;
            }
        }
        }
    }
    tc_fence_before();
    if constexpr (CL > 1)
        cluster_sync_all();  // no CTA leaves while its peer may still signal or fill it
    else
        __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---- B digits of the panel (per pass) --------------------------------------
// one thread per (k-step, column, 4 rows): balanced base-256 digits of
// round(X 2^(56 - f_c)), written as 7 byte planes in the UMMA layout
__global__ void __launch_bounds__(256) k_panel_digits(const double* __restrict__ x, int ks0, int nks,
                                                      int wp, int nb, int cg0,
                                                      const int* __restrict__ col_exp,
                                                      unsigned char* __restrict__ bdig) {
    // k-steps ks0 .. ks0 + nks - 1
    const long long total = static_cast<long long>(nks) * nb * 8;
    const int bb = kDig * nb * kKStep;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int kq = static_cast<int>(e & 7);
        const int c = static_cast<int>((e >> 3) % nb);
        const long long ks = ks0 + (e >> 3) / nb;
        uint32_t word[kDig];
#pragma unroll
        for (int u = 0; u < kDig; ++u) word[u] = 0;
        const int gc = cg0 + c;
        const int f = gc < wp ? col_exp[gc] : kExpZeroI8;
        if (f > kExpZeroI8) {
            const double scale = ldexp(1.0, 56 - f);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const size_t j = static_cast<size_t>(ks) * kKStep + kq * 4 + jj;
                long long m = __double2ll_rn(x[pidx(j, gc, wp)] * scale);
                int dig[kDig];
#pragma unroll
                for (int u = kDig - 1; u >= 1; --u) {
                    const int b = static_cast<int>((m + 128) & 255) - 128;
                    dig[u] = b;
                    m = (m - b) >> 8;
                }
                dig[0] = static_cast<int>(m);
#pragma unroll
                for (int u = 0; u < kDig; ++u)
                    word[u] |= (static_cast<uint32_t>(dig[u]) & 0xffu) << (8 * jj);
            }
        }
        unsigned char* dst = bdig + static_cast<size_t>(ks) * bb;
        const uint32_t off = umma_tile_off(static_cast<uint32_t>(c), static_cast<uint32_t>(kq * 4));
#pragma unroll
        for (int u = 0; u < kDig; ++u)
            *reinterpret_cast<uint32_t*>(dst + u * (nb * kKStep) + off) = word[u];
    }
}

// DSB_K2I_PAIR=0: w > 64 in separate column-group passes (one read of D
// each) instead of the CTA-pair kernel (comparisons)
bool k2i_pair_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DSB_K2I_PAIR");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

// DSB_K2I_DEBUG: 1 = skip the digit conversion, 2 = skip the MMAs (timing
// experiments only; results are wrong)
int k2i_debug_mode() {
    static const int m = [] {
        const char* e = std::getenv("DSB_K2I_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    return m;
}

template <int NB, typename TD, int SD, int CL, int DM>
void run_i8_dm(const CUtensorMap* tmap, const K2iPlan& p, int wp, const unsigned char* bdig,
               size_t bdig_stride, const int* row_exp, const int* col_exp, double* part, int cg0,
               cudaStream_t st, const int* skip, double hlen, int k_off, unsigned char* sdig,
               int nks_c) {
    const void* fn = reinterpret_cast<const void*>(k2i_product_ts<NB, TD, SD, CL, DM>);
    constexpr size_t smem = ts_smem<NB, TD, SD, CL, DM>();
    ensure_dyn_smem(fn, smem);
    if constexpr (CL == 1) {
        k2i_product_ts<NB, TD, SD, 1, DM><<<p.grid, kThreadsI8, smem, st>>>(
            *tmap, bdig, row_exp, col_exp, p.nrows, p.nks, static_cast<int>(p.total), part,
            p.maxseg, wp, cg0, skip, k2i_debug_mode(), hlen, bdig_stride, k_off, sdig, nks_c);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(p.grid * CL));
        cfg.blockDim = dim3(kThreadsI8);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        DSB_CUDA(cudaLaunchKernelEx(&cfg, k2i_product_ts<NB, TD, SD, CL, DM>, *tmap, bdig,
                                    row_exp, col_exp, p.nrows, p.nks, static_cast<int>(p.total),
                                    part, p.maxseg, wp, cg0, skip, k2i_debug_mode(), hlen,
                                    bdig_stride, k_off, sdig, nks_c));
    }
}
// dm: S-digit cache mode of this launch (0 off, 1 store, 2 stream; sdig and
// nks_c as in k2i_product_ts)
template <int NB, typename TD, int SD = kDig, int CL = 1>
void run_i8(const CUtensorMap* tmap, const K2iPlan& p, int wp, const unsigned char* bdig,
            size_t bdig_stride, const int* row_exp, const int* col_exp, double* part, int cg0,
            cudaStream_t st, const int* skip, double hlen = 0.0, int k_off = 0, int dm = 0,
            unsigned char* sdig = nullptr, int nks_c = 0) {
    if constexpr (CL > 2) {  // clusters wider than a pair only stream the cache
        (void)dm;
        run_i8_dm<NB, TD, SD, CL, 2>(tmap, p, wp, bdig, bdig_stride, row_exp, col_exp, part, cg0,
                                     st, skip, hlen, k_off, sdig, nks_c);
    } else {
    if (dm == 1)
        run_i8_dm<NB, TD, SD, CL, 1>(tmap, p, wp, bdig, bdig_stride, row_exp, col_exp, part, cg0,
                                     st, skip, hlen, k_off, sdig, nks_c);
    else if (dm == 2)
        run_i8_dm<NB, TD, SD, CL, 2>(tmap, p, wp, bdig, bdig_stride, row_exp, col_exp, part, cg0,
                                     st, skip, hlen, k_off, sdig, nks_c);
    else
        run_i8_dm<NB, TD, SD, CL, 0>(tmap, p, wp, bdig, bdig_stride, row_exp, col_exp, part, cg0,
                                     st, skip, hlen, k_off, nullptr, 0);
    }
}

// Co-resident clusters of CL CTAs (one ~210 KB CTA per SM): at most sms / CL,
// fewer when some GPC's SM count leaves SMs without a full cluster. Queried
// once per device and kernel variant.
template <int NB, typename TD, int SD, int CL, int DM>
int cluster_units(int sms) {
    static std::mutex mu;
    static std::map<int, int> units;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = units.find(dev);
    if (it != units.end()) return it->second;
    const void* fn = reinterpret_cast<const void*>(k2i_product_ts<NB, TD, SD, CL, DM>);
    constexpr size_t smem = ts_smem<NB, TD, SD, CL, DM>();
    ensure_dyn_smem(fn, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(sms / CL * CL));
    cfg.blockDim = dim3(kThreadsI8);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = sms / CL;
    }
    n = std::min(n, sms / CL);
    if (const char* e = std::getenv("DSB_K2I_UNITS")) n = std::max(1, std::min(n, std::atoi(e)));
    if (std::getenv("DSB_TRACE"))
        std::fprintf(stderr, "[k2i] clusters of %d co-resident: %d\n", CL, n);
    units[dev] = n;
    return n;
}
int pair_units(int sms) { return cluster_units<48, double, kDig, 2, 0>(sms); }

}  // namespace

K2iPlan k2i_plan(size_t nrows, size_t ncols, int wp, int sms) {
    K2iPlan p;
    const size_t nks = (ncols + kKStep - 1) / kKStep;
    // the CTA pair only for 64 < WP <= 96 (two 48-column groups): at
    // WP > 96 each CTA's 64-column digit MMAs bind (C4-like w = 120: pair
    // 6.2 vs 5.7 ms per pass on f32 D, equal on f64), at WP <= 96 one read of
    // D beats two (w = 70, n = 40k: 4.61 vs 5.07 ms; C3: 32.4 vs 36.3 ms)
    if (wp <= 64 || wp > 96 || !k2i_pair_enabled()) {
        // column groups, one full pass over D each: NB = 64 groups while more
        // than 32 columns remain, then one NB = 32 or 64 group for the rest
        for (int c0 = 0; c0 < wp && p.ngroups < K2iPlan::kMaxGroups; ++p.ngroups) {
            const int rest = wp - c0;
            const int nb = rest <= 32 ? 32 : 64;
            p.gc0[p.ngroups] = c0;
            p.gnb[p.ngroups] = nb;
            p.bdig_bytes = std::max(p.bdig_bytes, nks * kDig * nb * kKStep);
            c0 += nb;
            p.nb = c0;
        }
    } else {
        // 64 < WP <= 96: one pass, a CTA pair sharing each D tile, one
        // 48-column group per CTA
        const int nb = 48;
        p.pair = true;
        p.ngroups = 2;
        p.gc0[0] = 0;
        p.gc0[1] = nb;
        p.gnb[0] = p.gnb[1] = nb;
        p.nb = 2 * nb;
        p.bdig_stride = nks * kDig * nb * kKStep;
        p.bdig_bytes = 2 * p.bdig_stride;
        sms = 2 * pair_units(sms);  // the work units below are pairs
    }
    p.nrows = static_cast<int>(nrows);
    p.nblk = static_cast<int>((nrows + kRowsI8 - 1) / kRowsI8);
    p.nks = static_cast<int>((ncols + kKStep - 1) / kKStep);
    p.total = static_cast<long long>(p.nblk) * p.nks;
    // work units (CTAs, or CTA pairs): one partial slot each
    p.grid = static_cast<int>(std::min<long long>(p.pair ? sms / 2 : sms, p.total));
    int maxseg = 1;
    for (long long c = 0; c < p.grid; ++c) {
        const long long a = p.total * c / p.grid, b = p.total * (c + 1) / p.grid;
        if (b > a) maxseg = std::max<int>(maxseg, static_cast<int>((b - 1) / p.nks - a / p.nks + 1));
    }
    p.maxseg = maxseg;
    p.part_elems = static_cast<size_t>(p.grid) * maxseg * kRowsI8 * wp;
    p.colmax_grid = sms;
    p.cl = p.pair ? 2 : 1;
    return p;
}

// DSB_K2I_STREAM_CL=1: the streaming passes of WP > 32 run on clusters of
// 32-column groups (k2i_stream_plan). Off by default: measured slower than
// the storing pass's own plan (C5 3.25 vs 2.37 ms, n = 40k w = 70 3.90 vs
// 3.46 ms, w = 50 3.04 vs 2.71 ms per pass) — multicast at cluster sizes
// <= 4 does not reduce the L2 -> SM traffic, and each CTA of a cluster still
// takes in every item plus its own panel digits, now for twice the items.
bool stream_clusters_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DSB_K2I_STREAM_CL");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

K2iPlan k2i_stream_plan(size_t nrows, size_t ncols, int wp, int sms, int sdigits) {
    const int cl = std::min(4, (wp + 31) / 32);
    if (cl <= 1 || !stream_clusters_enabled()) return k2i_plan(nrows, ncols, wp, sms);
    K2iPlan p;
    const size_t nks = (ncols + kKStep - 1) / kKStep;
    p.cl = cl;
    p.pair = true;
    p.ngroups = cl;
    for (int g = 0; g < cl; ++g) {
        p.gc0[g] = 32 * g;
        p.gnb[g] = 32;
    }
    p.nb = 32 * cl;
    p.bdig_stride = nks * kDig * 32 * kKStep;
    p.bdig_bytes = cl * p.bdig_stride;
    int units = 0;
    const bool ham = sdigits == 3;
    switch (cl) {
        case 2: units = ham ? cluster_units<32, double, 3, 2, 2>(sms)
                            : cluster_units<32, double, kDig, 2, 2>(sms); break;
        case 3: units = ham ? cluster_units<32, double, 3, 3, 2>(sms)
                            : cluster_units<32, double, kDig, 3, 2>(sms); break;
        default: units = ham ? cluster_units<32, double, 3, 4, 2>(sms)
                             : cluster_units<32, double, kDig, 4, 2>(sms); break;
    }
    p.nrows = static_cast<int>(nrows);
    p.nblk = static_cast<int>((nrows + kRowsI8 - 1) / kRowsI8);
    p.nks = static_cast<int>(nks);
    p.total = static_cast<long long>(p.nblk) * p.nks;
    p.grid = static_cast<int>(std::min<long long>(units, p.total));
    int maxseg = 1;
    for (long long c = 0; c < p.grid; ++c) {
        const long long a = p.total * c / p.grid, b = p.total * (c + 1) / p.grid;
        if (b > a) maxseg = std::max<int>(maxseg, static_cast<int>((b - 1) / p.nks - a / p.nks + 1));
    }
    p.maxseg = maxseg;
    p.part_elems = static_cast<size_t>(p.grid) * maxseg * kRowsI8 * wp;
    p.colmax_grid = sms;
    return p;
}

bool k2i_supported(int wp) { return wp >= 8 && wp <= 128; }

size_t k2i_sdig_bytes(const K2iPlan& p, int sdigits) {
    return static_cast<size_t>(p.nblk) * p.nks * (sdigits == 3 ? sdig_item_bytes<3>()
                                                               : sdig_item_bytes<kDig>());
}

namespace {
// a streaming pass on a cluster plan (k2i_stream_plan): CL CTAs share every
// digit item, CTA g computes panel columns 32 g .. 32 g + 31
void launch_k2i_stream(const K2iPlan& p, int wp, const double* x, const int* col_exp,
                       unsigned char* bdig, double* part, const double* row_mean,
                       const double* scalars, const double* colsums, double* y,
                       size_t y_rows_pad, const int* row_exp, cudaStream_t st, cudaEvent_t e0,
                       cudaEvent_t e1, const int* skip, int hamming_len, unsigned char* sdig,
                       int nks_c) {
    const size_t r_done = static_cast<size_t>(p.nblk) * kRowsI8;
    if (y_rows_pad > r_done)
        DSB_CUDA(cudaMemsetAsync(y + r_done * wp, 0, (y_rows_pad - r_done) * wp * sizeof(double),
                                 st));
    for (int g = 0; g < p.cl; ++g) {
        const long long items = static_cast<long long>(p.nks) * 32 * 8;
        const int grid = static_cast<int>(std::min<long long>((items + 255) / 256, 4 * 148));
        k_panel_digits<<<grid, 256, 0, st>>>(x, 0, p.nks, wp, 32, p.gc0[g], col_exp,
                                             bdig + g * p.bdig_stride);
    }
    if (e0) record_timing_event(e0, st);
    const double hl = static_cast<double>(hamming_len);
    const size_t bs = p.bdig_stride;
    // (the tensor map is unused when streaming)
    static const CUtensorMap no_map{};
    const CUtensorMap* tm = &no_map;
    const bool ham = hamming_len > 0;
    switch (p.cl) {
        case 2:
            if (ham)
                run_i8<32, double, 3, 2>(tm, p, wp, bdig, bs, row_exp, col_exp, part, 0, st, skip,
                                         hl, 0, 2, sdig, nks_c);
            else
                run_i8<32, double, kDig, 2>(tm, p, wp, bdig, bs, row_exp, col_exp, part, 0, st,
                                            skip, 0.0, 0, 2, sdig, nks_c);
            break;
        case 3:
            if (ham)
                run_i8<32, double, 3, 3>(tm, p, wp, bdig, bs, row_exp, col_exp, part, 0, st, skip,
                                         hl, 0, 2, sdig, nks_c);
            else
                run_i8<32, double, kDig, 3>(tm, p, wp, bdig, bs, row_exp, col_exp, part, 0, st,
                                            skip, 0.0, 0, 2, sdig, nks_c);
            break;
        default:
            if (ham)
                run_i8<32, double, 3, 4>(tm, p, wp, bdig, bs, row_exp, col_exp, part, 0, st, skip,
                                         hl, 0, 2, sdig, nks_c);
            else
                run_i8<32, double, kDig, 4>(tm, p, wp, bdig, bs, row_exp, col_exp, part, 0, st,
                                            skip, 0.0, 0, 2, sdig, nks_c);
            break;
    }
    count_launch(1 + p.cl);
    if (e1) record_timing_event(e1, st);
    launch_k2_reduce(wp, kRowsI8, part, p.maxseg, p.nks, p.total, p.grid, p.nrows, 1, row_mean,
                     scalars, colsums, y, st, skip);
    count_launch(1);
}
}  // namespace

void launch_k2i(const CUtensorMap* tmap128, const CUtensorMap* tmap64, DType dt, const K2iPlan& p,
                int wp, const double* x, size_t x_rows_pad, const int* row_exp, double* pmax,
                int* col_exp, unsigned char* bdig, double* part, const double* row_mean,
                const double* scalars, const double* colsums, double* y, size_t y_rows_pad,
                cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1, const int* skip, int hamming_len,
                unsigned char* sdig, int sdig_mode, const K2iPlan* stream_plan) {
    if (!sdig) sdig_mode = 0;
    const int nks_c = p.nks;
    if (sdig_mode == 2 && stream_plan && stream_plan->cl > 1 && stream_plan->gnb[0] == 32) {
        launch_k2i_stream(*stream_plan, wp, x, col_exp, bdig, part, row_mean, scalars, colsums, y,
                          y_rows_pad, row_exp, st, e0, e1, skip, hamming_len, sdig, nks_c);
        return;
    }
    // k2_reduce writes the 128-row blocks; the panel rows beyond them (up to
    // the 256-row padding) must read as zero, whatever an earlier, larger
    // solve left in this workspace
    const size_t r_done = static_cast<size_t>(p.nblk) * kRowsI8;
    if (y_rows_pad > r_done)
        DSB_CUDA(cudaMemsetAsync(y + r_done * wp, 0, (y_rows_pad - r_done) * wp * sizeof(double),
                                 st));
    (void)x_rows_pad;
    (void)pmax;  // column exponents come from launch_colsums (same pass over X)
    auto digits = [&](int nb, int cg0, unsigned char* dst) {
        const long long items = static_cast<long long>(p.nks) * nb * 8;
        const int grid = static_cast<int>(std::min<long long>((items + 255) / 256, 4 * 148));
        k_panel_digits<<<grid, 256, 0, st>>>(x, 0, p.nks, wp, nb, cg0, col_exp, dst);
    };
    const double hl = static_cast<double>(hamming_len);
    const bool ham = dt == DType::F64 && hamming_len > 0;
    if (p.pair) {
        // one launch: the CTA pair shares every D tile (64-row multicast
        // boxes), CTA r computes panel columns gc0[r] .. with its digits
        const int nb = p.gnb[0];
        digits(nb, p.gc0[0], bdig);
        digits(nb, p.gc0[1], bdig + p.bdig_stride);
        if (e0) record_timing_event(e0, st);
        const size_t bs = p.bdig_stride;
        (void)nb;  // 48 (k2i_plan)
        const int dm = sdig_mode;
        if (ham)
            run_i8<48, double, 3, 2>(tmap64, p, wp, bdig, bs, row_exp, col_exp, part, 0, st, skip,
                                     hl, 0, dm, sdig, nks_c);
        else if (dt == DType::F64)
            run_i8<48, double, kDig, 2>(tmap64, p, wp, bdig, bs, row_exp, col_exp, part, 0, st,
                                        skip, 0.0, 0, dm, sdig, nks_c);
        else
            run_i8<48, float, kDig, 2>(tmap64, p, wp, bdig, bs, row_exp, col_exp, part, 0, st,
                                       skip, 0.0, 0, dm, sdig, nks_c);
        count_launch(2);
    } else {
        for (int g = 0; g < p.ngroups; ++g) {
            const int nb = p.gnb[g], cg0 = p.gc0[g];
            digits(nb, cg0, bdig);
            if (g == 0 && e0) record_timing_event(e0, st);
            // the first group of a storing pass stores, the later ones stream
            const int dm = (sdig_mode == 1 && g > 0) ? 2 : sdig_mode;
            if (ham) {
                if (nb == 32)
                    run_i8<32, double, 3>(tmap128, p, wp, bdig, 0, row_exp, col_exp, part, cg0, st,
                                          skip, hl, 0, dm, sdig, nks_c);
                else
                    run_i8<64, double, 3>(tmap128, p, wp, bdig, 0, row_exp, col_exp, part, cg0, st,
                                          skip, hl, 0, dm, sdig, nks_c);
            } else if (dt == DType::F64) {
                if (nb == 32)
                    run_i8<32, double>(tmap128, p, wp, bdig, 0, row_exp, col_exp, part, cg0, st,
                                       skip, 0.0, 0, dm, sdig, nks_c);
                else
                    run_i8<64, double>(tmap128, p, wp, bdig, 0, row_exp, col_exp, part, cg0, st,
                                       skip, 0.0, 0, dm, sdig, nks_c);
            } else {
                if (nb == 32)
                    run_i8<32, float>(tmap128, p, wp, bdig, 0, row_exp, col_exp, part, cg0, st,
                                      skip, 0.0, 0, dm, sdig, nks_c);
                else
                    run_i8<64, float>(tmap128, p, wp, bdig, 0, row_exp, col_exp, part, cg0, st,
                                      skip, 0.0, 0, dm, sdig, nks_c);
            }
        }
        count_launch(2 * p.ngroups);
    }
    // (external records: real event nodes when the solve is captured as a graph)
    if (e1) record_timing_event(e1, st);
    launch_k2_reduce(wp, kRowsI8, part, p.maxseg, p.nks, p.total, p.grid, p.nrows, 1, row_mean,
                     scalars, colsums, y, st, skip);
    count_launch(1);
}

size_t k2i_ranges_part_elems(const K2iPlan& full, int wp,
                             const std::vector<std::pair<int, int>>& ranges, int sms) {
    size_t slots = 0;
    for (const auto& r : ranges) {
        const K2iPlan pr = k2i_plan(full.nrows, static_cast<size_t>(r.second - r.first) * kKStep,
                                    wp, sms);
        slots += static_cast<size_t>(pr.grid) * pr.maxseg;
    }
    return slots * kRowsI8 * wp;
}

void launch_k2i_ranges(const CUtensorMap* tmap128, const CUtensorMap* tmap64, DType dt,
                       const K2iPlan& full, int wp, const double* x, const int* row_exp,
                       const int* col_exp, unsigned char* bdig, double* part,
                       const double* row_mean, const double* scalars, const double* colsums,
                       double* y, size_t y_rows_pad, cudaStream_t st, cudaEvent_t gathered,
                       const std::vector<std::pair<int, int>>& ranges, int sms, cudaEvent_t e0,
                       cudaEvent_t e1, int hamming_len, unsigned char* sdig, int sdig_mode) {
    if (!sdig) sdig_mode = 0;
    const size_t r_done = static_cast<size_t>(full.nblk) * kRowsI8;
    if (y_rows_pad > r_done)
        DSB_CUDA(cudaMemsetAsync(y + r_done * wp, 0, (y_rows_pad - r_done) * wp * sizeof(double),
                                 st));
    const double hl = static_cast<double>(hamming_len);
    const bool ham = dt == DType::F64 && hamming_len > 0;
    std::vector<K2iPlan> plans;
    std::vector<K2Split> splits;
    long long slot = 0;
    for (size_t ri = 0; ri < ranges.size(); ++ri) {
        const auto& r = ranges[ri];
        // the range that runs next to the all-gather leaves a few SMs free:
        // the persistent product otherwise fills every SM and the collective's
        // kernel could only start after it
        const int sms_r = (ri == 0 && gathered) ? std::max(sms - 8, sms / 2) : sms;
        plans.push_back(k2i_plan(full.nrows, static_cast<size_t>(r.second - r.first) * kKStep, wp,
                                 sms_r));
        const K2iPlan& pr = plans.back();
        splits.push_back(K2Split{pr.nks, pr.total, pr.grid, pr.maxseg, slot});
        slot += static_cast<long long>(pr.grid) * pr.maxseg;
    }
    auto digits = [&](int ri, int nb, int cg0, unsigned char* dst) {
        const int k0 = ranges[ri].first, nk = ranges[ri].second - ranges[ri].first;
        const long long items = static_cast<long long>(nk) * nb * 8;
        const int grid = static_cast<int>(std::min<long long>((items + 255) / 256, 4 * 148));
        k_panel_digits<<<grid, 256, 0, st>>>(x, k0, nk, wp, nb, cg0, col_exp, dst);
        count_launch();
    };
    // cache items are indexed by global k-step (k_off) over the full plan's
    // k-steps; a storing pass's later column groups already find them
    auto run = [&](int ri, int g, unsigned char* bd, size_t bs) {
        const K2iPlan& pr = plans[ri];
        const int dm = (sdig_mode == 1 && g > 0) ? 2 : sdig_mode;
        const int nkc = full.nks;
        double* pp = part + static_cast<size_t>(splits[ri].slot_base) * kRowsI8 * wp;
        const int k0 = ranges[ri].first;
        if (full.pair) {
            if (ham)
                run_i8<48, double, 3, 2>(tmap64, pr, wp, bd, bs, row_exp, col_exp, pp, 0, st,
                                         nullptr, hl, k0, dm, sdig, nkc);
            else if (dt == DType::F64)
                run_i8<48, double, kDig, 2>(tmap64, pr, wp, bd, bs, row_exp, col_exp, pp, 0, st,
                                            nullptr, 0.0, k0, dm, sdig, nkc);
            else
                run_i8<48, float, kDig, 2>(tmap64, pr, wp, bd, bs, row_exp, col_exp, pp, 0, st,
                                           nullptr, 0.0, k0, dm, sdig, nkc);
        } else {
            const int nb = full.gnb[g], cg0 = full.gc0[g];
            if (ham) {
                if (nb == 32)
                    run_i8<32, double, 3>(tmap128, pr, wp, bd, 0, row_exp, col_exp, pp, cg0, st,
                                          nullptr, hl, k0, dm, sdig, nkc);
                else
                    run_i8<64, double, 3>(tmap128, pr, wp, bd, 0, row_exp, col_exp, pp, cg0, st,
                                          nullptr, hl, k0, dm, sdig, nkc);
            } else if (dt == DType::F64) {
                if (nb == 32)
                    run_i8<32, double>(tmap128, pr, wp, bd, 0, row_exp, col_exp, pp, cg0, st,
                                       nullptr, 0.0, k0, dm, sdig, nkc);
                else
                    run_i8<64, double>(tmap128, pr, wp, bd, 0, row_exp, col_exp, pp, cg0, st,
                                       nullptr, 0.0, k0, dm, sdig, nkc);
            } else {
                if (nb == 32)
                    run_i8<32, float>(tmap128, pr, wp, bd, 0, row_exp, col_exp, pp, cg0, st,
                                      nullptr, 0.0, k0, dm, sdig, nkc);
                else
                    run_i8<64, float>(tmap128, pr, wp, bd, 0, row_exp, col_exp, pp, cg0, st,
                                      nullptr, 0.0, k0, dm, sdig, nkc);
            }
        }
        count_launch();
    };
    bool waited = gathered == nullptr;
    auto wait_gathered = [&] {
        if (!waited) DSB_CUDA(cudaStreamWaitEvent(st, gathered, 0));
        waited = true;
    };
    if (e0) record_timing_event(e0, st);
    if (full.pair) {
        // one launch per range; the pair's two 48-column groups' digits sit
        // bdig_stride apart (the full plan's layout: global k-steps)
        for (size_t ri = 0; ri < ranges.size(); ++ri) {
            if (ri > 0) wait_gathered();
            digits(static_cast<int>(ri), full.gnb[0], full.gc0[0], bdig);
            digits(static_cast<int>(ri), full.gnb[1], full.gc0[1], bdig + full.bdig_stride);
            run(static_cast<int>(ri), 0, bdig, full.bdig_stride);
        }
    } else {
        // column groups share one digit buffer: group-major, every range of a
        // group before the next group's digits
        for (int g = 0; g < full.ngroups; ++g)
            for (size_t ri = 0; ri < ranges.size(); ++ri) {
                if (ri > 0) wait_gathered();
                digits(static_cast<int>(ri), full.gnb[g], full.gc0[g], bdig);
                run(static_cast<int>(ri), g, bdig, 0);
            }
    }
    if (e1) record_timing_event(e1, st);
    launch_k2_reduce_multi(wp, kRowsI8, part, splits, full.nrows, 1, row_mean, scalars, colsums,
                           y, st, nullptr);
    count_launch(1);
}

}  // namespace dsb
