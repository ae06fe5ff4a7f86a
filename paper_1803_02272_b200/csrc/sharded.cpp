// Multi-GPU MDS path: D row-sharded over the ranks of one box
// (one process per GPU), NCCL over NVLink only for the exchange steps.
//
//   gram   : ONE pass over the local rows (row sums / sum d^4 / max |d| —
//            the reference's row means use full rows, mds.cpp:31-38, which a
//            row shard has — plus an antisymmetric fingerprint of the rows:
//            summed over all ranks it is zero iff D is exactly symmetric, so
//            one 64-bit all-reduce replaces a block exchange); only when it is
//            nonzero are the off-diagonal blocks exchanged pairwise (ring
//            shift) to measure max |d_ij - d_ji| against the reference's
//            tolerance; row means are all-gathered (every rank keeps the full
//            r) and the grand-mean sums run in one fixed order on the device,
//            so they do not depend on the rank count. One host sync.
//   solve  : the panel X (n x w) is replicated; each pass computes the local
//            rows Y_g = G[R_g, :] X with K2, CholeskyQR all-reduces the w x w
//            Gram, applies R^{-1} to the local rows and all-gathers the panel
//            (grouped broadcasts: shards differ by at most one block); the
//            Ritz Gram Q^T GQ is all-reduced and every rank solves the same
//            EVD; the sign rule gathers the per-CTA (max |u|, first index)
//            partials of all ranks; the coordinates are all-gathered.
// With one rank the same code runs with every collective a no-op.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>

#include "comm.hpp"
#include "solver.hpp"

namespace dsb {

namespace {

struct Layout {
    int world = 1, rank = 0;
    std::vector<size_t> rb, re;  // row ranges of every rank
};

Layout layout_of(size_t n) {
    Comm& cm = Comm::get();
    Layout L;
    L.world = cm.active() ? cm.world() : 1;
    L.rank = cm.active() ? cm.rank() : 0;
    L.rb.resize(L.world);
    L.re.resize(L.world);
    for (int r = 0; r < L.world; ++r) shard_rows(n, L.world, r, L.rb[r], L.re[r]);
    return L;
}

void check_shard(const Store& s) {
    Layout L = layout_of(s.n_global);
    if (s.row_begin != L.rb[L.rank] || s.row_begin + s.rows != L.re[L.rank])
        throw Error(errc::shape_mismatch,
                    "row shard does not match this rank's range (divscope_shard_range)");
}

// Cross-rank agreement before the first collective of a call: every rank
// runs its local validation, then one all-reduce of (error code, call
// signature, -signature) decides. A rank whose validation failed and its
// peers all return an error (the failing rank's own code; peers get the same
// code), and ranks that entered the call with different arguments (n, w, q,
// seed, mode) all fail with INVALID_ARGUMENT — instead of the peers blocking
// forever in a collective the failing rank never reaches.
template <typename F>
void agree_or_throw(uint64_t signature, F&& validate) {
    Ctx& c = Ctx::get();
    Comm& cm = Comm::get();
    int code = 0;
    std::string msg;
    try {
        validate();
    } catch (const Error& e) {
        code = static_cast<int>(e.code());
        msg = e.what();
    }
    if (!cm.active() || cm.world() == 1) {
        if (code) throw Error(static_cast<errc>(code), msg);
        return;
    }
    const double sig = static_cast<double>(signature & ((1ull << 52) - 1));
    double h[3] = {static_cast<double>(code), sig, -sig};
    double* d = static_cast<double*>(c.scratch("sh_agree", sizeof(h)));
    DSB_CUDA(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, c.stream));
    cm.allreduce_max(d, 3, c.stream);
    c.d2h_copy(h, d, sizeof(h));
    if (code) throw Error(static_cast<errc>(code), msg);
    if (h[0] != 0.0)
        throw Error(static_cast<errc>(static_cast<int>(h[0])),
                    "a peer rank failed this call's validation");
    if (h[1] != -h[2])
        throw Error(errc::invalid_argument, "ranks entered the call with different arguments");
}

uint64_t mix_sig(std::initializer_list<uint64_t> v) {
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (uint64_t x : v) {
        h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xBF58476D1CE4E5B9ull;
    }
    return h;
}

}  // namespace

Matrix matrix_from_host_rows(const void* rows, size_t n, size_t row_begin, size_t row_end,
                             bool symmetric, DType dt) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (row_end < row_begin || row_end > n) throw Error(errc::invalid_argument, "bad row range");
    Matrix m;
    m.store = make_store(row_end - row_begin, n, symmetric, dt);
    m.store->sharded = true;
    m.store->n_global = n;
    m.store->row_begin = row_begin;
    upload_rows(*m.store, rows, n);
    c.sync();
    return m;
}

Matrix matrix_euclidean_rows(const double* pts, size_t n, size_t dim, bool f32, size_t row_begin,
                             size_t row_end) {
    // K9 on this shard's row window only (every (i, j) is computed
    // independently, so the shard has exactly the bits of the full matrix)
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (row_end < row_begin || row_end > n) throw Error(errc::invalid_argument, "bad row range");
    if (n == 0 || dim == 0) throw Error(errc::empty_input, "no points");
    if (dim > 256) throw Error(errc::invalid_argument, "dimension > 256 not supported");
    Matrix m;
    m.store = make_store(row_end - row_begin, n, true, f32 ? DType::F32 : DType::F64);
    m.store->sharded = true;
    m.store->n_global = n;
    m.store->row_begin = row_begin;
    DevBuf dp(n * dim * sizeof(double));
    c.h2d_copy(dp.p, pts, n * dim * sizeof(double));
    launch_euclid_rows(dp.as<double>(), n, static_cast<int>(dim), m.store->buf->p, m.store->dt,
                       m.store->ld, row_begin, row_end - row_begin, c.stream);
    c.sync();
    return m;
}

Matrix gram_sharded(const Matrix& d) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    Comm& cm = Comm::get();
    const Store& s = *d.store;
    const size_t n = s.n_global;
    agree_or_throw(mix_sig({1, n}), [&] {
        if (!s.square() || !s.symmetric)
            throw Error(errc::not_symmetric, "gram matrix requires a symmetric distance matrix");
        if (n == 0) throw Error(errc::empty_input, "empty distance matrix");
        check_shard(s);
    });
    Layout L = layout_of(n);
    const size_t m = s.rows, rb = s.row_begin;
    const size_t esz = s.dt == DType::F64 ? 8 : 4;
    // ---- ONE pass over the local rows: row sums of d^2, row exponents, CTA
    // partials of sum d^4 / max |d|, and the antisymmetric fingerprint whose
    // sum over all ranks is zero iff D is exactly symmetric
    const int grid = k1_rows_grid(m, c.sms);
    auto row_mean = std::make_shared<DevBuf>(std::max<size_t>(n, 1) * 8);  // full r
    double* rowsum = static_cast<double*>(c.scratch("sh_rowsum", std::max<size_t>(m, 1) * 8));
    double* cta = static_cast<double*>(c.scratch("sh_cta", static_cast<size_t>(grid) * 3 * 8));
    auto row_exp = std::make_shared<DevBuf>(std::max<size_t>(m, 1) * sizeof(int));  // local rows
    // red: [0] sum d^4, [1] max |d|, [2] max asym (bits), [3] int8 ratio,
    //      [4] sum r, [5] sum r^2, [6..7] symmetry fingerprint halves (u64)
    double* red = static_cast<double*>(c.scratch("sh_red", 8 * 8));
    auto* fp = reinterpret_cast<unsigned long long*>(red + 6);
    DSB_CUDA(cudaMemsetAsync(red, 0, 8 * 8, c.stream));
    cudaEvent_t e0, e1;
    c.make_events(&e0, &e1);
    if (e0) DSB_CUDA(cudaEventRecord(e0, c.stream));
    if (m) {
        launch_k1_rows(s.buf->p, s.dt, s.ld, m, n, rb, rowsum, row_mean->as<double>() + rb, cta,
                       grid, c.stream, row_exp->as<int>(), fp);
        launch_shard_fold(cta, grid, red, c.stream);
    }
    cm.allreduce_sum(red, 1, c.stream);
    cm.allreduce_max(red + 1, 3, c.stream);
    cm.allreduce_sum_u64(fp, 2, c.stream);
    {
        // row means: every rank keeps the full r
        std::vector<size_t> cnt(L.world), off(L.world);
        for (int r = 0; r < L.world; ++r) {
            off[r] = L.rb[r];
            cnt[r] = L.re[r] - L.rb[r];
        }
        cm.allgatherv(row_mean->as<double>(), cnt.data(), off.data(), c.stream);
    }
    // grand-mean terms in one fixed order over the full r (rank-count independent)
    launch_rowmean_sums(row_mean->as<double>(), n, red + 4, c.stream);
    if (e1) DSB_CUDA(cudaEventRecord(e1, c.stream));
    c.add_timed(0, e0, e1);
    double hred[8];
    c.d2h_copy(hred, red, sizeof(hred));  // the one sync of the common case
    const double maxabs = hred[1];
    unsigned long long fp_sum[2];
    std::memcpy(fp_sum, &hred[6], 16);
    double maxasym = 0.0;
    if (((fp_sum[0] | fp_sum[1]) & 0xFFFFFFFFull) != 0) {
        // some mirrored pair differs: measure max |d_ij - d_ji| exactly (the
        // reference's tolerance decides, mds.cpp:23-27) — local diagonal block,
        // then a ring shift of the off-diagonal blocks
        double* asym = static_cast<double*>(c.scratch("sh_asym", 64));
        DSB_CUDA(cudaMemsetAsync(asym, 0, 64, c.stream));
        launch_asym_block(static_cast<const char*>(s.buf->p) + rb * esz, s.ld,
                          static_cast<const char*>(s.buf->p) + rb * esz, s.ld, s.dt, m, m, asym,
                          c.stream);
        size_t maxm = 0;
        for (int r = 0; r < L.world; ++r) maxm = std::max(maxm, L.re[r] - L.rb[r]);
        // staging in f64 element units (f32 blocks travel as raw bytes)
        const size_t stage_elems = (maxm * maxm * esz + 7) / 8;
        double* sbuf =
            L.world > 1 ? static_cast<double*>(c.scratch("sh_send", stage_elems * 8 + 64)) : nullptr;
        double* rbuf =
            L.world > 1 ? static_cast<double*>(c.scratch("sh_recv", stage_elems * 8 + 64)) : nullptr;
        for (int sft = 1; sft < L.world; ++sft) {
            const int ps = (L.rank + sft) % L.world, pr = (L.rank - sft + L.world) % L.world;
            const size_t ms = L.re[ps] - L.rb[ps], mr = L.re[pr] - L.rb[pr];
            // send D[R_g, C_ps] packed (m x ms)
            if (m && ms)
                DSB_CUDA(cudaMemcpy2DAsync(sbuf, ms * esz,
                                           static_cast<const char*>(s.buf->p) + L.rb[ps] * esz,
                                           s.ld * esz, ms * esz, m, cudaMemcpyDeviceToDevice,
                                           c.stream));
            cm.sendrecv(sbuf, (m * ms * esz + 7) / 8, ps, rbuf, (mr * m * esz + 7) / 8, pr,
                        c.stream);
            // received D[R_pr, C_g] (mr x m) vs local D[R_g, C_pr] (m x mr)
            launch_asym_block(static_cast<const char*>(s.buf->p) + L.rb[pr] * esz, s.ld, rbuf, m,
                              s.dt, m, mr, asym, c.stream);
        }
        cm.allreduce_max(asym, 1, c.stream);
        uint64_t bits = 0;
        c.d2h_copy(&bits, asym, 8);
        std::memcpy(&maxasym, &bits, 8);  // non-negative doubles order as integers
    }
    if (maxasym > 1e-12 * std::max(1.0, maxabs))  // ref mds.cpp:23-27
        throw Error(errc::not_symmetric, "distance matrix values are not symmetric");
    Matrix g;
    g.store = d.store;
    g.gram = std::make_shared<GramInfo>();
    GramInfo& gi = *g.gram;
    gi.n = n;
    gi.row_mean = row_mean;
    gi.row_exp = row_exp;  // this rank's rows
    // the host copy of r is fetched on first use (matrix_get / _write)
    const double nf = static_cast<double>(n);
    const double sr = hred[4], sr2 = hred[5];
    gi.sc[S_GRAND] = sr / nf;
    gi.sc[S_FRO2_LAZY] = 0.25 * (hred[0] - 2.0 * nf * sr2 + nf * nf * gi.sc[S_GRAND] * gi.sc[S_GRAND]);
    gi.sc[S_MAXABS] = maxabs;
    gi.sc[S_MAXASYM] = maxasym;
    gi.sc[S_SUM4] = hred[0];
    gi.sc[S_SUMR] = sr;
    gi.sc[S_SUMR2] = sr2;
    gi.sc[S_ROWRATIO] = hred[3];
    gi.scalars = std::make_shared<DevBuf>(S_COUNT * 8);
    // stream-ordered (the source, gi.sc, lives as long as the handle)
    DSB_CUDA(cudaMemcpyAsync(gi.scalars->p, gi.sc, S_COUNT * 8, cudaMemcpyHostToDevice, c.stream));
    return g;
}

namespace {

const double* omega_pinned(uint64_t seed, size_t n, size_t w) {
    static std::deque<std::tuple<uint64_t, size_t, size_t, PinnedVec>> cache;
    for (auto& e : cache)
        if (std::get<0>(e) == seed && std::get<1>(e) == n && std::get<2>(e) == w)
            return std::get<3>(e).data();
    PinnedVec v(std::max<size_t>(n * w, 1));
    std::mt19937_64 eng(seed);
    fill_gaussian(eng, v.data(), n * w);
    if (cache.size() >= 2) cache.pop_front();
    cache.emplace_back(seed, n, w, std::move(v));
    return std::get<3>(cache.back()).data();
}

struct ShardOut {
    std::vector<double> vals;
    size_t keep = 0;
    double resid = 0.0;
    Embedding emb;
};

ShardOut run_sharded(const Matrix& g, size_t rank, size_t p, size_t q, uint64_t seed,
                     bool embed_mode, size_t requested) {
    Ctx& c = Ctx::get();
    Comm& cm = Comm::get();
    Store& s = *g.store;
    const size_t n = s.n_global, m = s.rows, rb = s.row_begin;
    const size_t w = rank + p;
    agree_or_throw(mix_sig({2, n, rank, p, q, seed, embed_mode ? 1u : 0u, requested}), [&] {
        if (!g.gram) throw Error(errc::invalid_argument, "sharded solve needs a gram handle");
        check_shard(s);
        if (rank < 1) throw Error(errc::invalid_argument, "rank must be >= 1");
        if (w > n) throw Error(errc::rank_too_large, "rank + oversampling exceeds matrix order");
        if (w > static_cast<size_t>(kMaxWP))
            throw Error(errc::invalid_argument,
                        "rank + oversampling > 128 is not supported by the GPU path");
        std::lock_guard<std::mutex> lk(s.mu);
        if (!s.tmap_ok) {
            if (!c.encode_tmap(&s.tmap128, s.buf->p, s.dt, std::max<size_t>(m, 1), s.cols, s.ld,
                               128) ||
                !c.encode_tmap(&s.tmap256, s.buf->p, s.dt, std::max<size_t>(m, 1), s.cols, s.ld,
                               256) ||
                !c.encode_tmap(&s.tmap64, s.buf->p, s.dt, std::max<size_t>(m, 1), s.cols, s.ld,
                               64))
                throw Error(errc::internal, "cuTensorMapEncodeTiled failed");
            s.tmap64_ok = true;
            s.tmap_ok = true;
        }
    });
    Layout L = layout_of(n);
    const int wi = static_cast<int>(w), wp = static_cast<int>(round_up(w, 8));
    // every rank owns one equal panel chunk (its rows, zero-padded): the
    // panel is world * chunk rows and all-gathers with ncclAllGather
    const size_t m_pad = shard_chunk_rows(n, L.world);
    const size_t n_pad = m_pad * static_cast<size_t>(L.world);
    const double* r_full = g.gram->row_mean->as<double>();
    const double* scal = g.gram->scalars->as<double>();
    const K2Plan plan = k2_plan_rect(std::max<size_t>(m, 1), n, wp, s.dt, c.sms);
    // int8 slice product on this rank's rows (same admission rule as 1 GPU)
    const bool use_i8 = m > 0 && use_int8_product(*g.gram, wp);
    K2iPlan iplan;
    double* pmax = nullptr;
    int* col_exp = nullptr;
    unsigned char* bdig = nullptr;
    // the panel all-gather overlapped with the product over this rank's own
    // columns (DSB_SHARD_OVERLAP=0: gather, then product). The choice is the
    // same on every rank (the collective sequence must match); ranks without
    // the int8 product still run the same collectives
    static const bool overlap_env = [] {
        const char* e = std::getenv("DSB_SHARD_OVERLAP");
        return !(e && std::atoi(e) == 0);
    }();
    const bool overlap = L.world > 1 && overlap_env;
    if (use_i8) {
        iplan = k2i_plan(m, n, wp, c.sms);
        col_exp = static_cast<int*>(c.scratch("i8_colexp", 128 * sizeof(int)));
        bdig = static_cast<unsigned char*>(c.scratch("i8_bdig", iplan.bdig_bytes));
    }
    if (use_i8 || overlap)
        pmax = static_cast<double*>(c.scratch(
            "i8_pmax", static_cast<size_t>(panel_grid(n_pad, c.sms)) * wp * sizeof(double)));
    double* cmax = overlap ? static_cast<double*>(c.scratch("shard_cmax", wp * sizeof(double)))
                           : nullptr;
    // k-step ranges of this rank's product: its own panel rows' columns first
    std::vector<std::pair<int, int>> ranges;
    if (use_i8 && overlap) {
        const int nks = (static_cast<int>(n) + 31) / 32;
        const int k_lo = static_cast<int>(std::min(n, L.rank * m_pad) / 32);
        const int k_hi = static_cast<int>((std::min(n, (L.rank + 1) * m_pad) + 31) / 32);
        if (k_hi > k_lo) ranges.emplace_back(k_lo, k_hi);
        if (k_lo > 0) ranges.emplace_back(0, k_lo);
        if (nks > k_hi) ranges.emplace_back(k_hi, nks);
    }
    c.last_product_kernel = use_i8 ? 1 : 0;
    // Hamming shards (divscope_matrix_hamming_rows): three exact S bytes
    const int hamming_i8 = (use_i8 && s.dt == DType::F64 && s.hamming_len > 0 &&
                            s.hamming_len < 4096 && hamming_slices_enabled())
                               ? s.hamming_len
                               : 0;
    c.last_product_sdigits = use_i8 ? (hamming_i8 ? 3 : 7) : 0;
    c.last_product_pair = use_i8 && iplan.pair ? 1 : 0;
    c.last_product_stream_cl = 0;
    c.last_product_groups = use_i8 ? iplan.ngroups : 1;
    const size_t pbytes = n_pad * wp * 8;
    double* P0 = static_cast<double*>(c.scratch("panel0", pbytes));
    double* P1 = static_cast<double*>(c.scratch("panel1", pbytes));
    double* P2 = static_cast<double*>(c.scratch("panel2", pbytes));
    const size_t part_elems =
        std::max({plan.part_elems, use_i8 ? iplan.part_elems : size_t(0),
                  ranges.empty() ? size_t(0) : k2i_ranges_part_elems(iplan, wp, ranges, c.sms)});
    double* part = static_cast<double*>(c.scratch("k2_part", part_elems * 8 + 64));
    const int pg = panel_grid(std::max<size_t>(m_pad, 4), c.sms);
    const int pgf = panel_grid(n_pad, c.sms);
    double* psmall = static_cast<double*>(c.scratch(
        "panel_part", static_cast<size_t>(std::max(pg, pgf)) * std::max(wp * wp, 2 * wp) * 8));
    double* colsums = static_cast<double*>(c.scratch("colsums", 2 * wp * 8));
    double* wmat = static_cast<double*>(c.scratch("wmat", wp * wp * 8));
    double* rinv = static_cast<double*>(c.scratch("rinv", wp * wp * 8));
    int* flags = static_cast<int*>(c.scratch("flags", 64));
    // the rank's S-digit cache (k2i_product.cu): its rows x every k-step;
    // the first product pass stores it, the later ones stream it. Local to
    // the rank (no collective depends on it), claimed last (evictable)
    unsigned char* sdig = nullptr;
    if (use_i8 && sdig_policy() > 0 && m > 0)
        sdig = static_cast<unsigned char*>(
            c.try_scratch("i8_sdig", k2i_sdig_bytes(iplan, hamming_i8 ? 3 : 7)));
    if (sdig) ++c.sdig_gen;  // overwrites whatever the slot held
    c.last_product_sdig = sdig ? 1 : 0;
    int sdig_pass = 0;
    DSB_CUDA(cudaMemsetAsync(flags, 0, 64, c.stream));
    DSB_CUDA(cudaMemsetAsync(P1, 0, pbytes, c.stream));
    {
        const double* om = omega_pinned(seed, n, w);
        double* stage = static_cast<double*>(c.scratch("omega_rm", n * w * 8));
        c.h2d_copy(stage, om, n * w * 8);
        launch_panel_from_rowmajor(stage, n, wi, wp, n_pad, P0, c.stream);
    }
    const size_t lo = static_cast<size_t>(L.rank) * m_pad * wp;  // this rank's panel chunk
    // gather: the panel's other chunks must first be all-gathered (every
    // product after a CholeskyQR; the first one multiplies the replicated Omega)
    auto product = [&](double* x_full, double* y_full, bool gather) {
        cudaEvent_t e0, e1;
        const int timed_kind = sdig_pass == 0 ? 3 : 1;  // the first pass: kind 3
        const int sdm = sdig ? (sdig_pass == 0 ? 1 : 2) : 0;
        ++sdig_pass;
        if (gather && overlap) {
            // s = 1^T X, t = r^T X and the column maxima of this rank's rows,
            // reduced over the ranks; then the all-gather on the side stream
            // while the product runs over the locally-owned columns
            launch_colsums(x_full + lo, r_full + rb, m, m_pad, wp, psmall, colsums, c.sms,
                           c.stream, pmax, 0, nullptr);
            launch_colmax(pmax, panel_grid(m_pad, c.sms), wp, cmax, c.stream);
            cm.allreduce_sum(colsums, static_cast<size_t>(2) * wp, c.stream);
            cm.allreduce_max(cmax, static_cast<size_t>(wp), c.stream);
            if (use_i8) launch_colexp(cmax, wp, iplan.nb, col_exp, c.stream);
            DSB_CUDA(cudaEventRecord(c.side_ready, c.stream));
            DSB_CUDA(cudaStreamWaitEvent(c.side, c.side_ready, 0));
            cm.allgather(x_full, m_pad * wp, c.side);
            DSB_CUDA(cudaEventRecord(c.side_done, c.side));
            c.make_events(&e0, &e1);
            if (use_i8) {
                launch_k2i_ranges(s.tmap_for(128), &s.tmap64, s.dt, iplan, wp, x_full,
                                  g.gram->row_exp->as<int>(), col_exp, bdig, part, r_full + rb,
                                  scal, colsums, y_full + lo, m_pad, c.stream, c.side_done, ranges,
                                  c.sms, e0, e1, hamming_i8, sdig, sdm);
            } else {
                DSB_CUDA(cudaStreamWaitEvent(c.stream, c.side_done, 0));
                if (m)
                    launch_k2(s.tmap_for(plan.bm), s.dt, 1, plan, x_full, part, r_full + rb, scal,
                              colsums, y_full + lo, m_pad, c.stream, e0, e1);
            }
            // every later collective (and panel write) comes after the gather
            DSB_CUDA(cudaStreamWaitEvent(c.stream, c.side_done, 0));
            c.add_timed(timed_kind, e0, e1);
            return;
        }
        if (gather) cm.allgather(x_full, m_pad * wp, c.stream);
        // s = 1^T X, t = r^T X over the full replicated panel (+ the int8
        // column exponents: identical on every rank)
        if (use_i8)
            launch_colsums(x_full, r_full, n, n_pad, wp, psmall, colsums, c.sms, c.stream, pmax,
                           iplan.nb, col_exp);
        else
            launch_colsums(x_full, r_full, n, n_pad, wp, psmall, colsums, c.sms, c.stream);
        c.make_events(&e0, &e1);
        if (use_i8)
            launch_k2i(s.tmap_for(128), &s.tmap64, s.dt, iplan, wp, x_full, n_pad,
                       g.gram->row_exp->as<int>(),
                       pmax, col_exp, bdig, part, r_full + rb, scal, colsums, y_full + lo, m_pad,
                       c.stream, e0, e1, nullptr, hamming_i8, sdig, sdm);
        else if (m)
            launch_k2(s.tmap_for(plan.bm), s.dt, 1, plan, x_full, part, r_full + rb, scal, colsums,
                      y_full + lo, m_pad, c.stream, e0, e1);
        c.add_timed(timed_kind, e0, e1);
    };
    auto orth_local = [&](double* y_full, double* t_full, double* out_full) {
        double* y = y_full + lo;
        double* t = t_full + lo;
        double* o = out_full + lo;
        double* bufs[3][2] = {{y, t}, {t, y}, {y, o}};
        // CholQR2, or CholQR3 after a shifted first pass: the third pass's
        // kernels are gated on the device-side shift flag (no host sync); its
        // all-reduce runs either way so the ranks' collectives stay matched
        const bool elim = wp <= 64;
        DSB_CUDA(cudaMemsetAsync(flags + 1, 0, sizeof(int), c.stream));
        for (int ps = 0; ps < 3; ++ps) {
            const int* gate = (ps == 2 && elim) ? flags + 1 : nullptr;
            launch_panel_dot(bufs[ps][0], bufs[ps][0], m_pad, wp, psmall, wmat, c.sms, c.stream,
                             gate);
            cm.allreduce_sum(wmat, static_cast<size_t>(wp) * wp, c.stream);
            // factor + apply in one launch (every CTA factors W redundantly
            // while its panel rows stream into shared memory); else the two kernels
            if (!launch_chol_inv_elim(wmat, wp, wi, n, ps, nullptr, flags, c.stream, gate,
                                      bufs[ps][0], bufs[ps][1], m_pad, c.sms)) {
                if (!launch_chol_inv_elim(wmat, wp, wi, n, ps, rinv, flags, c.stream, gate))
                    launch_chol_inv(wmat, wp, wi, n, ps == 0 ? 1 : 0, rinv, flags, c.stream);
                launch_panel_apply(bufs[ps][0], rinv, m_pad, wp, bufs[ps][1], c.stream, gate);
            }
        }
        (void)out_full;  // its other chunks are all-gathered by the next product
    };
    product(P0, P1, false);
    orth_local(P1, P2, P0);
    for (size_t it = 0; it < q; ++it) {
        product(P0, P1, true);
        orth_local(P1, P2, P0);
        product(P0, P1, true);
        orth_local(P1, P2, P0);
    }
    product(P0, P1, true);
    launch_panel_dot(P0 + lo, P1 + lo, m_pad, wp, psmall, wmat, c.sms, c.stream);
    cm.allreduce_sum(wmat, static_cast<size_t>(wp) * wp, c.stream);
    const size_t req = embed_mode ? requested : std::min(rank, w);
    EvdOut eo;
    eo.vals = static_cast<double*>(c.scratch("evd_vals", kMaxWP * 8));
    eo.vkeep = static_cast<double*>(c.scratch("evd_vkeep", w * std::max<size_t>(req, 1) * 8));
    eo.kept_vals = static_cast<double*>(c.scratch("evd_kept", kMaxWP * 8));
    eo.dmeta = static_cast<double*>(c.scratch("evd_dmeta", 64));
    eo.imeta = static_cast<int*>(c.scratch("evd_imeta", 64));
    launch_evd(wmat, wp, wi, static_cast<int>(rank), static_cast<int>(req), scal, S_FRO2_LAZY, eo,
               c.stream);
    ShardOut out;
    double* coords = nullptr;
    std::shared_ptr<DevBuf> dcoords;  // owned by the returned embedding
    if (embed_mode) {
        const size_t rq = std::max<size_t>(req, 1);
        dcoords = std::make_shared<DevBuf>(n * rq * 8);
        coords = dcoords->as<double>();
        // the partial-table geometry must agree on every rank (it sizes the
        // gather): CTAs per rank from the largest shard, not the local one
        size_t maxm = 1;
        for (int k = 0; k < L.world; ++k) maxm = std::max(maxm, L.re[k] - L.rb[k]);
        const int P = lift_grid(maxm, c.sms);
        // all ranks' CTA partials side by side: [world][P][rmax][2]
        double* lp = static_cast<double*>(
            c.scratch("lift_part_all", (static_cast<size_t>(L.world) * P * 2 + 1) * rq * 8));
        DSB_CUDA(cudaMemsetAsync(lp, 0xff, static_cast<size_t>(L.world) * P * 2 * rq * 8,
                                 c.stream));  // -NaN index => ignored
        // local rows written at their global row positions (r-wide rows
        // once r is known on the device: the lift writes row-major n_local x r)
        double* my_coords = static_cast<double*>(c.scratch("coords_local", std::max<size_t>(m, 1) * rq * 8));
        if (m)
            launch_lift_partial(P0 + lo, m, wp, wi, eo.vkeep, eo.imeta, static_cast<int>(req),
                                my_coords, lp + static_cast<size_t>(L.rank) * P * 2 * rq,
                                static_cast<long long>(rb), P, c.stream);
        cm.allgather(lp, static_cast<size_t>(P) * 2 * rq, c.stream);
        double* scale = lp + static_cast<size_t>(L.world) * P * 2 * rq;
        launch_lift_finish(m, eo.imeta, L.world * P, static_cast<int>(req), eo.kept_vals, lp, scale,
                           my_coords, c.stream);
        DSB_CUDA(cudaGetLastError());
        int im[8];
        c.d2h_copy(im, eo.imeta, sizeof(im));
        const size_t r = static_cast<size_t>(im[1]);
        // gather n x r coordinates (row chunks are contiguous in row-major)
        if (r) {
            DSB_CUDA(cudaMemcpyAsync(coords + rb * r, my_coords, m * r * 8,
                                     cudaMemcpyDeviceToDevice, c.stream));
            std::vector<size_t> cc(L.world), co(L.world);
            for (int k = 0; k < L.world; ++k) {
                co[k] = L.rb[k] * r;
                cc[k] = (L.re[k] - L.rb[k]) * r;
            }
            cm.allgatherv(coords, cc.data(), co.data(), c.stream);
        }
    }
    DSB_CUDA(cudaGetLastError());
    double vals[kMaxWP], kept[kMaxWP], dmeta[8];
    int imeta[8];
    DSB_CUDA(cudaMemcpyAsync(vals, eo.vals, w * 8, cudaMemcpyDeviceToHost, c.stream));
    DSB_CUDA(cudaMemcpyAsync(kept, eo.kept_vals, w * 8, cudaMemcpyDeviceToHost, c.stream));
    DSB_CUDA(cudaMemcpyAsync(dmeta, eo.dmeta, 64, cudaMemcpyDeviceToHost, c.stream));
    c.d2h_copy(imeta, eo.imeta, sizeof(imeta));
    c.last_evd_sweeps = imeta[3];
    if (!imeta[4]) throw Error(errc::internal, "small eigensolve failed");
    out.vals.assign(vals, vals + w);
    out.keep = static_cast<size_t>(imeta[0]);
    out.resid = dmeta[0];
    if (embed_mode) {
        Embedding& e = out.emb;
        e.n = n;
        e.r = static_cast<size_t>(imeta[1]);
        e.truncated = imeta[2] != 0;
        e.dropped_negative_mass = dmeta[1];
        e.resid = dmeta[0];
        e.eigenvalues.assign(kept, kept + e.r);
        e.dcoords = std::move(dcoords);
    }
    return out;
}

}  // namespace

Embedding embed_sharded(const Matrix& g, size_t rank, SolverOptions opts) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const size_t n = g.n();
    if (rank < 1 || rank > n) throw Error(errc::rank_too_large, "rank must be in [1, n]");
    opts.rank = rank;
    opts.oversampling = std::min(opts.oversampling, n - rank);
    ShardOut r = run_sharded(g, opts.rank, opts.oversampling, opts.power_iters, opts.seed, true, rank);
    return std::move(r.emb);
}

Spectrum eigs_sharded(const Matrix& g, const SolverOptions& opts) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    ShardOut r = run_sharded(g, opts.rank, opts.oversampling, opts.power_iters, opts.seed, false,
                             opts.rank);
    Spectrum s;
    s.eigenvalues.assign(r.vals.begin(), r.vals.begin() + r.keep);
    s.resid = r.resid;
    return s;
}

}  // namespace dsb
