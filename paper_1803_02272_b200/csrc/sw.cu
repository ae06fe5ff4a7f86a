// Smith-Waterman alignment distances on the GPU — the distance builder
// upstream of the MDS path: pairwise_self / pairwise_cross
// (ref src/distmat.cpp:45-128) over sw_distance / sw_align (ref
// src/align.cpp:28-106), bit-exact.
//
// One pair per thread (inter-task parallelism: the pairs are independent and
// of similar length). The distance modes run k_sw_e, which carries the
// traceback's event count forward in the cell keys and needs no traceback
// storage (see below); k_sw, described here, serves divscope_align (spans)
// and score ranges past the 32-bit key. The DP is strip-mined over 8-column strips: a strip's
// 8 cells of the previous row live in registers, the strip's left boundary
// column H[.][j0-1] lives in a per-thread global column (coalesced across
// threads: element (i, thread) at i * T + thread). Every cell also gets its
// traceback code — the FIRST predecessor, in the reference's preference
// order diagonal > up > left, whose value exactly accounts for the cell (0,
// 1, 2), else 3 (stop) — packed 2 bits per cell, 16 bits per strip row,
// stored [row][strip][thread] (coalesced). The first maximal cell in
// row-major order (the reference's strict-greater scan) is found from the
// strip visiting order: a tie can only improve on the current best from an
// earlier row of a later strip, so `v > best || (v == best && i < bi)`.
// The traceback then walks the codes from that cell exactly as
// align.cpp:70-92 (the diagonal step counts when the substitution is not a
// match; gap steps count), so distance, score and spans equal the
// reference's. Canonical operand order of sw_distance (b < a lexicographic
// -> swap, align.cpp:99-104) is applied per pair.
#include <algorithm>

#include "device_utils.cuh"
#include "kernels.cuh"

namespace dsb {

namespace {

constexpr int kSwStrip = 8;
constexpr int kSwThreads = 128;

__device__ __forceinline__ bool seq_less(const unsigned char* x, int lx, const unsigned char* y,
                                         int ly) {
    const int m = lx < ly ? lx : ly;
    for (int k = 0; k < m; ++k) {
        if (x[k] != y[k]) return x[k] < y[k];
    }
    return lx < ly;
}

// row-major upper-triangle pair index -> (i, j), i < j (ref distmat.cpp:17-35)
__device__ __forceinline__ void pair_of_index(long long k, long long n, long long& i,
                                              long long& j) {
    auto row_off = [&](long long r) { return r * (n - 1) - r * (r - 1) / 2; };
    const double nf = static_cast<double>(n);
    const double g = nf - 0.5 - sqrt((nf - 0.5) * (nf - 0.5) - 2.0 * static_cast<double>(k));
    long long gi = g <= 0.0 ? 0 : static_cast<long long>(g);
    if (gi >= n - 1) gi = n - 2;
    while (gi > 0 && row_off(gi) > k) --gi;
    while (row_off(gi + 1) <= k) ++gi;
    i = gi;
    j = gi + 1 + (k - row_off(gi));
}

// mode 0: all pairs i < j of the n_a reads (self); 1: n_a queries x n_b refs
// (refs stored after the queries); 2: the pairs (0, 1) as given, no operand
// swap (divscope_align). aux (mode 2): score, distance, a_begin, a_end,
// b_begin, b_end.
__global__ void __launch_bounds__(kSwThreads) k_sw(
    const unsigned char* __restrict__ seq, const long long* __restrict__ off,
    const int* __restrict__ len, int mode, long long n_a, long long n_b, long long npairs,
    int match, int mismatch, int gap, int nstr_max, unsigned short* __restrict__ dirs,
    int* __restrict__ hb, double* __restrict__ dout, size_t ld, long long* __restrict__ aux) {
    const long long T = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (long long p = tid; p < npairs; p += T) {
        long long ia, ib, ra, rbi;
        if (mode == 0) {
            pair_of_index(p, n_a, ia, ib);
            ra = ia;
            rbi = ib;
        } else if (mode == 1) {
            ia = p / n_b;
            ib = p % n_b;
            ra = ia;
            rbi = n_a + ib;
        } else {
            ia = 0;
            ib = 1;
            ra = 0;
            rbi = 1;
        }
        const unsigned char* A = seq + off[ra];
        const unsigned char* B = seq + off[rbi];
        int na = len[ra], nb = len[rbi];
        if (mode != 2 && seq_less(B, nb, A, na)) {
            const unsigned char* t = A;
            A = B;
            B = t;
            const int tl = na;
            na = nb;
            nb = tl;
        }
        // ---- forward fill
        for (int i = 0; i <= na; ++i) hb[i * T + tid] = 0;
        int best = 0, bi = 0, bj = 0;
        const int nstr = (nb + kSwStrip - 1) / kSwStrip;
        for (int s = 0; s < nstr; ++s) {
            const int j0 = s * kSwStrip + 1;
            unsigned int bc[kSwStrip];
#pragma unroll
            for (int c = 0; c < kSwStrip; ++c) bc[c] = (j0 + c <= nb) ? B[j0 - 1 + c] : 0x100u;
            int top[kSwStrip];
#pragma unroll
            for (int c = 0; c < kSwStrip; ++c) top[c] = 0;
            int diag_l = 0;  // H[i-1][j0-1]
            const int valid = nb - j0 + 1;  // cells of this strip inside the matrix (>= 1)
            for (int i = 1; i <= na; ++i) {
                const unsigned int ca = A[i - 1];
                const bool ca_n = (ca == 'N');
                const int left_l = hb[i * T + tid];  // H[i][j0-1]
                int cur[kSwStrip];
                unsigned int code = 0;
#pragma unroll
                for (int c = 0; c < kSwStrip; ++c) {
                    const int sub = (ca == bc[c] && !ca_n) ? match : mismatch;
                    const int d = (c == 0 ? diag_l : top[c - 1]) + sub;
                    const int u = top[c] + gap;
                    const int l = (c == 0 ? left_l : cur[c - 1]) + gap;
                    int v = max(max(d, u), max(l, 0));
                    // cells past column nb (last strip) are clamped to 0: they
                    // feed only other padded cells and never become the maximum
                    if (c >= valid) v = 0;
                    const unsigned int cd = (d == v) ? 0u : (u == v) ? 1u : (l == v) ? 2u : 3u;
                    code |= cd << (2 * c);
                    cur[c] = v;
                    // first maximum in row-major order: strips are visited left to
                    // right and rows top-down within a strip, so a tie replaces the
                    // current best only from an earlier row of a later strip
                    if (v > best || (v == best && i < bi)) {
                        best = v;
                        bi = i;
                        bj = j0 + c;
                    }
                }
                hb[i * T + tid] = cur[kSwStrip - 1];
                diag_l = left_l;
#pragma unroll
                for (int c = 0; c < kSwStrip; ++c) top[c] = cur[c];
                dirs[(static_cast<long long>(i) * nstr_max + s) * T + tid] =
                    static_cast<unsigned short>(code);
            }
        }
        // ---- traceback (ref align.cpp:70-92)
        int i = bi, j = bj, events = 0;
        while (i > 0 && j > 0) {
            const unsigned int cw =
                dirs[(static_cast<long long>(i) * nstr_max + (j - 1) / kSwStrip) * T + tid];
            const unsigned int cd = (cw >> (2 * ((j - 1) % kSwStrip))) & 3u;
            if (cd == 0u) {
                const unsigned int x = A[i - 1], y = B[j - 1];
                const int sub = (x == y && x != 'N') ? match : mismatch;
                if (sub != match) ++events;
                --i;
                --j;
            } else if (cd == 1u) {
                ++events;
                --i;
            } else if (cd == 2u) {
                ++events;
                --j;
            } else {
                break;
            }
        }
        if (mode == 2) {
            aux[0] = best;
            aux[1] = events;
            aux[2] = i;
            aux[3] = bi;
            aux[4] = j;
            aux[5] = bj;
        } else {
            const double v = static_cast<double>(events);
            dout[static_cast<size_t>(ia) * ld + ib] = v;
            if (mode == 0) dout[static_cast<size_t>(ib) * ld + ia] = v;
        }
    }
}

// Forward-only variant for the distance modes (0, 1). The traceback is a
// deterministic walk over the codes, so the event count it returns can be
// carried forward instead: E(i,j) = E(predecessor) + step cost, with the
// predecessor chosen by the same first-match rule and E = 0 at a stop (code
// 3) or on the matrix border. Each cell holds one key
//     key = H << 16 | E          (E < 2^14; bits 14-15 free)
// and a predecessor's candidate key adds its score delta in the high half, a
// preference tag in bits 14-15 (diagonal 2, up 1, left 0) and its step cost
// in the low bits, so ONE signed max-with-zero (__vimax3_s32_relu, a DPX
// instruction) picks the maximum score, breaks ties diagonal > up > left and
// yields the stop cell's key 0 — exactly the reference's code at every cell
// (align.cpp:70-92) with no traceback storage. The distance is E at the first
// maximal cell. Used when |H| stays below 2^15 and na + nb < 2^14 (sw_plan);
// otherwise k_sw above.
#ifndef DSB_SW_STRIP_E
#define DSB_SW_STRIP_E 16
#endif
constexpr int kStripE = DSB_SW_STRIP_E;  // strip width of the forward-only kernel
constexpr int kTie = 1 << 14;
constexpr unsigned int kTieMask = 3u << 14;
constexpr unsigned int kEMask = kTie - 1;

template <bool TAIL>
__device__ __forceinline__ void sw_e_rows(const unsigned char* __restrict__ A, int na,
                                          const unsigned int (&bc)[kStripE], int valid, int s,
                                          int* __restrict__ hb, long long T, long long tid,
                                          int sdm, int sdx, int cu, int cl, int& best_h,
                                          int& bi, int& best_e) {
    int top[kStripE];
#pragma unroll
    for (int c = 0; c < kStripE; ++c) top[c] = 0;
    int diag_l = 0;
    // the boundary column is read two rows ahead: one row of the strip is
    // ~75 instructions per thread, far short of a DRAM round trip
    int nxt1 = (s && na >= 1) ? hb[T + tid] : 0;
    int nxt2 = (s && na >= 2) ? hb[2 * T + tid] : 0;
    unsigned int ca_n = __ldg(A);
    for (int i = 1; i <= na; ++i) {
        unsigned int ca = ca_n;
        if (i < na) ca_n = __ldg(A + i);
        if (ca == 'N') ca = 0x1FFu;  // 'N' never matches (align.cpp:56)
        const int left_l = nxt1;
        nxt1 = nxt2;
        nxt2 = (s && i + 2 <= na) ? hb[(i + 2) * T + tid] : 0;
        int cur[kStripE];
#pragma unroll
        for (int c = 0; c < kStripE; ++c) {
            const int kd = (c == 0 ? diag_l : top[c - 1]) + (ca == bc[c] ? sdm : sdx);
            const int ku = top[c] + cu;
            const int kl = (c == 0 ? left_l : cur[c - 1]) + cl;
            int v = static_cast<int>(static_cast<unsigned int>(__vimax3_s32_relu(kd, ku, kl)) &
                                     ~kTieMask);
            if (TAIL && c >= valid) v = 0;
            cur[c] = v;
        }
        hb[i * T + tid] = cur[kStripE - 1];
        diag_l = left_l;
        int rmax = cur[0];
#pragma unroll
        for (int c = 1; c < kStripE; ++c) rmax = max(rmax, cur[c]);
        const int h = rmax >> 16;
        // first maximum in row-major order (see k_sw): a later strip replaces
        // an equal best only from an earlier row
        if (h > best_h || (h == best_h && i < bi)) {
            int e = 0;
#pragma unroll
            for (int c = kStripE - 1; c >= 0; --c)
                if ((cur[c] >> 16) == h) e = cur[c] & static_cast<int>(kEMask);
            best_h = h;
            bi = i;
            best_e = e;
        }
#pragma unroll
        for (int c = 0; c < kStripE; ++c) top[c] = cur[c];
    }
}

__global__ void __launch_bounds__(kSwThreads) k_sw_e(
    const unsigned char* __restrict__ seq, const long long* __restrict__ off,
    const int* __restrict__ len, int mode, long long n_a, long long n_b, long long npairs,
    int match, int mismatch, int gap, int* __restrict__ hb, double* __restrict__ dout,
    size_t ld) {
    const long long T = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    // the match key goes through shared memory so that it lands in a vector
    // register: SEL cannot take two uniform operands, and a uniform copy
    // would cost one extra instruction per cell
    __shared__ int s_sdm;
    if (threadIdx.x == 0) s_sdm = static_cast<int>(static_cast<unsigned int>(match) << 16) + 2 * kTie;
    __syncthreads();
    const int sdm = *static_cast<volatile int*>(&s_sdm);
    const int sdx = static_cast<int>(static_cast<unsigned int>(mismatch) << 16) + 2 * kTie + 1;
    const int cu = static_cast<int>(static_cast<unsigned int>(gap) << 16) + kTie + 1;
    const int cl = static_cast<int>(static_cast<unsigned int>(gap) << 16) + 1;
    for (long long p = tid; p < npairs; p += T) {
        long long ia, ib, ra, rbi;
        if (mode == 0) {
            pair_of_index(p, n_a, ia, ib);
            ra = ia;
            rbi = ib;
        } else {
            ia = p / n_b;
            ib = p % n_b;
            ra = ia;
            rbi = n_a + ib;
        }
        const unsigned char* A = seq + off[ra];
        const unsigned char* B = seq + off[rbi];
        int na = len[ra], nb = len[rbi];
        if (seq_less(B, nb, A, na)) {
            const unsigned char* t = A;
            A = B;
            B = t;
            const int tl = na;
            na = nb;
            nb = tl;
        }
        int best_h = 0, bi = 0, best_e = 0;
        const int nstr = (nb + kStripE - 1) / kStripE;
        for (int s = 0; s < nstr; ++s) {
            const int j0 = s * kStripE + 1;
            unsigned int bc[kStripE];
#pragma unroll
            for (int c = 0; c < kStripE; ++c) bc[c] = (j0 + c <= nb) ? B[j0 - 1 + c] : 0x100u;
            const int valid = nb - j0 + 1;
            if (valid >= kStripE)
                sw_e_rows<false>(A, na, bc, valid, s, hb, T, tid, sdm, sdx, cu, cl, best_h, bi,
                                 best_e);
            else
                sw_e_rows<true>(A, na, bc, valid, s, hb, T, tid, sdm, sdx, cu, cl, best_h, bi,
                                best_e);
        }
        const double v = static_cast<double>(best_e);
        dout[static_cast<size_t>(ia) * ld + ib] = v;
        if (mode == 0) dout[static_cast<size_t>(ib) * ld + ia] = v;
    }
}

}  // namespace

SwPlan sw_plan(int max_len, int sms, int mode, int match, int mismatch, int gap) {
    SwPlan p;
    p.nstr_max = (std::max(max_len, 1) + kSwStrip - 1) / kSwStrip;
    // forward-only kernel: scores and (score + penalty) fit the key's signed
    // high half, and the event count (<= na + nb) its 14 low bits
    const long long hmax = static_cast<long long>(match) * std::max(max_len, 1);
    p.forward_only = mode != 2 && 2LL * max_len + 1 < kTie &&
                     hmax + match - static_cast<long long>(std::min(mismatch, gap)) < 32767;
    const size_t per_thread =
        (static_cast<size_t>(max_len) + 1) *
        ((p.forward_only ? 0 : static_cast<size_t>(p.nstr_max) * sizeof(unsigned short)) +
         sizeof(int));
    const size_t budget = size_t(12) << 30;  // traceback codes + boundary columns
    // one wave of co-resident blocks: the kernels are persistent (pair p on
    // thread p mod T), so blocks past the resident set would run as a second,
    // thinner wave
    int per_sm = 0;
    if (p.forward_only)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sw_e, kSwThreads, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sw, kSwThreads, 0);
    per_sm = std::max(1, std::min(per_sm, 16));
    size_t threads = static_cast<size_t>(sms) * per_sm * kSwThreads;
    threads = std::min(threads, std::max<size_t>(kSwThreads, budget / std::max<size_t>(per_thread, 1)));
    threads = std::max<size_t>(kSwThreads, threads / kSwThreads * kSwThreads);
    p.threads = static_cast<long long>(threads);
    p.dirs_elems = p.forward_only ? 1 : (static_cast<size_t>(max_len) + 1) * p.nstr_max * threads;
    p.hb_elems = (static_cast<size_t>(max_len) + 1) * threads;
    return p;
}

void launch_sw(const unsigned char* seq, const long long* off, const int* len, int mode,
               long long n_a, long long n_b, long long npairs, int match, int mismatch, int gap,
               const SwPlan& p, unsigned short* dirs, int* hb, double* dout, size_t ld,
               long long* aux, cudaStream_t st) {
    if (npairs <= 0) return;
    const long long blocks_needed = (npairs + kSwThreads - 1) / kSwThreads;
    const int grid = static_cast<int>(std::min<long long>(p.threads / kSwThreads, blocks_needed));
    // the kernel indexes the per-thread columns with the FULL plan width T
    // (gridDim * blockDim); keep it equal to p.threads
    const int grid_full = static_cast<int>(p.threads / kSwThreads);
    (void)grid;
    if (p.forward_only) {
        k_sw_e<<<grid_full, kSwThreads, 0, st>>>(seq, off, len, mode, n_a, n_b, npairs, match,
                                                 mismatch, gap, hb, dout, ld);
        count_launch();
        return;
    }
    k_sw<<<grid_full, kSwThreads, 0, st>>>(seq, off, len, mode, n_a, n_b, npairs, match, mismatch,
                                           gap, p.nstr_max, dirs, hb, dout, ld, aux);
    count_launch();
}

}  // namespace dsb
