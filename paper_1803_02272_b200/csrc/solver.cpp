// Host orchestration of the B200 MDS path: K1 (pass 0) at gram time, then
// the randomized range finder, Rayleigh-Ritz and the embedding, all
// enqueued on the library stream with no host round trip until the final
// read-back (ref src/rsvd.cpp:81-145, src/mds.cpp:14-124).
#include "solver.hpp"
#include "device_utils.cuh"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <functional>
#include <thread>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <tuple>

namespace dsb {

namespace {

struct StatsOut {
    double sc[S_COUNT];
    std::shared_ptr<DevBuf> scalars;
    std::shared_ptr<DevBuf> row_mean;
    std::shared_ptr<DevBuf> row_exp;
};

// K1 over a store; returns scalars (host) plus device scalars/row means.
// claim_digits (lazy grams of f64 D): called after every other allocation of
// the pass (a failed one would evict the cache slot) to set up the S-digit
// cache K1 writes; returns nullptr when there is none
StatsOut run_k1(Store& s, const std::function<const K1Digits*()>& claim_digits = nullptr) {
    Ctx& c = Ctx::get();
    {
        std::lock_guard<std::mutex> lk(s.mu);
        if (!s.tmap64_ok) {
            if (!c.encode_tmap(&s.tmap64, s.buf->p, s.dt, s.rows, s.cols, s.ld, 64))
                throw Error(errc::internal, "cuTensorMapEncodeTiled failed");
            s.tmap64_ok = true;
        }
    }
    const size_t n = s.rows;
    K1Work w;
    w.grid = k1_grid(n, c.sms);
    w.part = static_cast<double*>(c.scratch("k1_part", k1_part_elems(n) * sizeof(double)));
    w.cta_stats = static_cast<double*>(c.scratch("k1_cta", static_cast<size_t>(w.grid) * 4 * 8));
    w.pexp = static_cast<int*>(c.scratch("k1_pexp", k1_part_elems(n) * sizeof(int)));
    w.blk_stats = static_cast<double*>(c.scratch("k1_blk", ((n + 31) / 32) * 4 * 8 + 64));
    w.blk_bad = static_cast<int*>(c.scratch("k1_blkbad", ((n + 31) / 32) * sizeof(int) + 64));
    StatsOut o;
    o.row_mean = std::make_shared<DevBuf>(std::max<size_t>(n, 1) * sizeof(double));
    o.row_exp = std::make_shared<DevBuf>(std::max<size_t>(n, 1) * sizeof(int));
    o.scalars = std::make_shared<DevBuf>(S_COUNT * sizeof(double));
    DSB_CUDA(cudaMemsetAsync(o.scalars->p, 0, S_COUNT * sizeof(double), c.stream));
    cudaEvent_t ev;
    c.begin_timed(0, &ev);
    const K1Digits* dig = claim_digits ? claim_digits() : nullptr;
    if (dig && dig->row_eb) launch_row0_bound(s.buf->as<double>(), n, dig->row_eb, c.stream);
    launch_k1(&s.tmap64, s.dt, n, w, o.row_mean->as<double>(), o.row_exp->as<int>(),
              o.scalars->as<double>(), c.sms, c.stream, dig);
    c.end_timed(0, ev);
    DSB_CUDA(cudaGetLastError());
    c.d2h_copy(o.sc, o.scalars->p, S_COUNT * sizeof(double));
    return o;
}

void ensure_tmap(Store& s) {
    std::lock_guard<std::mutex> lk(s.mu);
    if (s.tmap_ok) return;
    if (!Ctx::get().encode_tmap(&s.tmap128, s.buf->p, s.dt, s.rows, s.cols, s.ld, 128) ||
        !Ctx::get().encode_tmap(&s.tmap256, s.buf->p, s.dt, s.rows, s.cols, s.ld, 256))
        throw Error(errc::internal, "cuTensorMapEncodeTiled failed");
    if (!s.tmap64_ok) {  // K1's boxes, also the CTA-pair product's multicast halves
        if (!Ctx::get().encode_tmap(&s.tmap64, s.buf->p, s.dt, s.rows, s.cols, s.ld, 64))
            throw Error(errc::internal, "cuTensorMapEncodeTiled failed");
        s.tmap64_ok = true;
    }
    s.tmap_ok = true;
}

// check_symmetric (ref rsvd.cpp:46-60) for explicit matrices, cached
void ensure_explicit_stats(Store& s) {
    {
        std::lock_guard<std::mutex> lk(s.mu);
        if (s.stats_ok) return;
    }
    StatsOut o = run_k1(s);
    std::lock_guard<std::mutex> lk(s.mu);
    std::memcpy(s.stats, o.sc, sizeof(s.stats));
    s.stats_dev = o.scalars;
    s.stats_ok = true;
}

// Omega = fill_gaussian(mt19937_64(seed)) as n x w row-major (rsvd.cpp:90-92),
// generated on the host (bit-identical to the reference) into pinned memory
// and memoized for the most recent shapes (a pure function of (seed, n, w));
// it is copied to the device on every solve.
struct PinnedOmega {
    uint64_t seed = 0;
    size_t n = 0, w = 0;
    double* p = nullptr;
    ~PinnedOmega() {
        if (p) cudaFreeHost(p);
    }
};

const double* omega_host(uint64_t seed, size_t n, size_t w) {
    static std::deque<std::unique_ptr<PinnedOmega>> cache;
    for (auto& e : cache)
        if (e->seed == seed && e->n == n && e->w == w) return e->p;
    auto e = std::make_unique<PinnedOmega>();
    e->seed = seed;
    e->n = n;
    e->w = w;
    DSB_CUDA(cudaMallocHost(&e->p, std::max<size_t>(n * w, 1) * sizeof(double)));
    std::mt19937_64 eng(seed);
    fill_gaussian(eng, e->p, n * w);
    if (cache.size() >= 2) cache.pop_front();
    cache.push_back(std::move(e));
    return cache.back()->p;
}

// The int8 slice product keeps ~53 bits relative to the ROW maximum of d^2;
// accept it when every row's max / mean ratio is bounded (so the error stays
// at the fp64 level relative to the row's own magnitude) and the data are
// finite. DSB_K2_INT8=0 forces the fp64 kernel (parity comparisons).
std::atomic<int> g_product_path{-1};  // -1: not yet read from DSB_K2_INT8

int product_path() {
    int m = g_product_path.load();
    if (m < 0) {
        // DSB_K2_INT8: unset/1 -> auto, 0 -> fp64 only, 2 -> int8 whenever supported
        const char* e = std::getenv("DSB_K2_INT8");
        const int v = e ? std::atoi(e) : 1;
        m = v == 0 ? 1 : (v == 2 ? 2 : 0);
        g_product_path.store(m);
    }
    return m;  // 0 auto, 1 fp64 only, 2 int8 whenever supported
}

}  // namespace

// DSB_K2I_HAMMING=0 keeps Hamming matrices on the general 7-byte slices
// (parity comparisons)
bool hamming_slices_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DSB_K2I_HAMMING");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

void set_product_path(int mode) { g_product_path.store(mode); }

std::atomic<int> g_sdig_policy{-1};  // -1: not yet read from DSB_SDIG

int sdig_policy() {
    int m = g_sdig_policy.load();
    if (m < 0) {
        const char* e = std::getenv("DSB_SDIG");
        m = e ? std::min(2, std::max(0, std::atoi(e))) : 1;
        g_sdig_policy.store(m);
    }
    return m;
}

void set_sdig_policy(int mode) { g_sdig_policy.store(mode); }

bool use_int8_product(const GramInfo& gi, int wp) {
    const int mode = product_path();
    if (mode == 1 || !gi.row_exp || !k2i_supported(wp)) return false;
    // small (L2-resident) problems: the extra digit launches outweigh the gain
    if (gi.n < 4096 && mode != 2) return false;
    const double ratio = gi.sc[S_ROWRATIO], s4 = gi.sc[S_SUM4];
    return std::isfinite(s4) && std::isfinite(ratio) && ratio <= 4096.0;
}

namespace {

struct RunOut {
    std::vector<double> vals;  // w values, reference order
    size_t keep = 0;
    double resid = 0.0;
    Embedding emb;
    std::vector<double> vectors;  // EigsVectors: n x keep
};

enum class What { Eigs, Embed, Range, EigsVectors };

RunOut run(const Matrix& g, size_t rank, size_t p, size_t q, uint64_t seed, What what,
           size_t requested, double* range_out) {
    Ctx& c = Ctx::get();
    Store& s = *g.store;
    const size_t n = s.rows;
    const bool lazy = static_cast<bool>(g.gram);
    const double* scal_dev = nullptr;
    const double* row_mean = nullptr;
    int fro_index;
    if (lazy) {
        scal_dev = g.gram->scalars->as<double>();
        row_mean = g.gram->row_mean->as<double>();
        fro_index = S_FRO2_LAZY;
    } else {
        // ref rsvd.cpp:46-60: n == 0 -> invalid_argument; asymmetry -> not_symmetric
        if (n == 0) throw Error(errc::invalid_argument, "empty matrix");
        ensure_explicit_stats(s);
        if (s.stats[S_MAXASYM] > 1e-10 * std::max(1.0, s.stats[S_MAXABS_UP]))
            throw Error(errc::not_symmetric, "matrix is not symmetric");
        scal_dev = s.stats_dev->as<double>();
        fro_index = S_FRO2_EXPL;
    }
    // ref rsvd.cpp:83-88
    if (rank < 1) throw Error(errc::invalid_argument, "rank must be >= 1");
    const size_t w = rank + p;
    if (w > n) throw Error(errc::rank_too_large, "rank + oversampling exceeds matrix order");
    if (w > static_cast<size_t>(kMaxWP))
        throw Error(errc::invalid_argument,
                    "rank + oversampling > 128 is not supported by the GPU path");
    const int wi = static_cast<int>(w);
    const int wp = static_cast<int>(round_up(w, 8));
    const size_t n_pad = round_up(n, kRowPad);
    const int mode = lazy ? 1 : 0;

    ensure_tmap(s);
    const K2Plan plan = k2_plan(n, wp, s.dt, c.sms);
    // integer-tensor-core product (k2i_product.cu) for lazy grams of moderate
    // dynamic range; the fp64 DMMA kernel otherwise
    const bool use_i8 = lazy && use_int8_product(*g.gram, wp);
    c.last_product_kernel = use_i8 ? 1 : 0;
    K2iPlan iplan, splan;
    double* pmax = nullptr;
    int* col_exp = nullptr;
    unsigned char* bdig = nullptr;
    // Hamming distances (K7): three exact S bytes per element (h^2 < 2^24)
    const int hamming_i8 =
        (use_i8 && s.dt == DType::F64 && s.hamming_len > 0 && s.hamming_len < 4096 &&
         hamming_slices_enabled())
            ? s.hamming_len
            : 0;
    if (use_i8) {
        iplan = k2i_plan(n, n, wp, c.sms);
        // the plan of the passes that stream the S-digit cache (when it is on)
        splan = k2i_stream_plan(n, n, wp, c.sms, hamming_i8 ? 3 : 7);
        pmax = static_cast<double*>(c.scratch(
            "i8_pmax", static_cast<size_t>(panel_grid(n_pad, c.sms)) * wp * sizeof(double)));
        col_exp = static_cast<int*>(c.scratch("i8_colexp", 128 * sizeof(int)));
        bdig = static_cast<unsigned char*>(
            c.scratch("i8_bdig", std::max(iplan.bdig_bytes, splan.bdig_bytes)));
    }
    const int i8_nb = std::max(iplan.nb, splan.nb);  // panel columns with int8 exponents
    c.last_product_groups = use_i8 ? iplan.ngroups : 1;
    c.last_product_sdigits = use_i8 ? (hamming_i8 ? 3 : 7) : 0;
    c.last_product_pair = use_i8 && iplan.pair ? 1 : 0;
    const size_t pbytes = n_pad * wp * sizeof(double);
    double* P0 = static_cast<double*>(c.scratch("panel0", pbytes));
    double* P1 = static_cast<double*>(c.scratch("panel1", pbytes));
    double* P2 = static_cast<double*>(c.scratch("panel2", pbytes));
    double* part = static_cast<double*>(c.scratch(
        "k2_part",
        std::max({plan.part_elems, use_i8 ? iplan.part_elems : 0, use_i8 ? splan.part_elems : 0}) *
            sizeof(double)));
    const int pg = panel_grid(n_pad, c.sms);
    const size_t part_small =
        std::max<size_t>(static_cast<size_t>(pg) * wp * wp, static_cast<size_t>(pg) * 2 * wp);
    double* psmall = static_cast<double*>(c.scratch("panel_part", part_small * sizeof(double)));
    double* colsums = static_cast<double*>(c.scratch("colsums", 2 * wp * sizeof(double)));
    double* wmat = static_cast<double*>(c.scratch("wmat", wp * wp * sizeof(double)));
    double* rinv = static_cast<double*>(c.scratch("rinv", wp * wp * sizeof(double)));
    int* flags = static_cast<int*>(c.scratch("flags", 64));

    // Omega: host-generated (bit-identical to the reference), relayout on the
    // device once per (seed, n, w) and kept resident (a pure function of the
    // seed); every solve starts from a device copy of it
    double* omega_cached = static_cast<double*>(c.scratch("omega_panel", pbytes));
    {
        Ctx::OmegaKey& key = c.omega_key;
        if (!key.ok || key.seed != seed || key.n != n || key.w != w || key.n_pad != n_pad) {
            key.ok = false;  // the slot may have been reallocated by the scratch call above
            const double* om = omega_host(seed, n, w);
            double* stage = static_cast<double*>(c.scratch("omega_rm", n * w * sizeof(double)));
            c.h2d_copy(stage, om, n * w * sizeof(double));
            launch_panel_from_rowmajor(stage, n, wi, wp, n_pad, omega_cached, c.stream);
            key = Ctx::OmegaKey{true, seed, n, w, n_pad};
        }
    }

    // DSB_TRACE=1: device timestamps between the stages of this solve (stderr)
    static const bool trace = std::getenv("DSB_TRACE") != nullptr;
    const auto h0 = std::chrono::steady_clock::now();
    auto host_us = [&] {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0)
            .count();
    };
    std::vector<std::pair<const char*, cudaEvent_t>> marks;
    auto mark = [&](const char* what_) {
        if (!trace) return;
        std::fprintf(stderr, "[trace] host at %-10s %.1f us\n", what_, host_us());
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, c.stream);
        marks.emplace_back(what_, e);
    };
    // per-CTA column statistics left by the fused orth kernel for the next
    // product pass (saves its separate column-statistics pass)
    double* cstat = static_cast<double*>(c.scratch(
        "orth_cstat", static_cast<size_t>(orth_fused_grid(n_pad, c.sms)) * 3 * wp * sizeof(double)));
    // every workspace of the solve is claimed before any work is enqueued, so
    // the sequence below can be captured as a graph (no allocation inside)
    const size_t req = what == What::Embed ? requested : std::min(rank, w);
    // eigenvector mode: k_evd keeps the first `keep` vectors whatever their sign
    const int evd_req = what == What::EigsVectors ? -1 : static_cast<int>(req);
    EvdOut eo;
    eo.vals = static_cast<double*>(c.scratch("evd_vals", kMaxWP * sizeof(double)));
    eo.vkeep = static_cast<double*>(c.scratch("evd_vkeep", w * std::max<size_t>(req, 1) * 8));
    eo.kept_vals = static_cast<double*>(c.scratch("evd_kept", kMaxWP * sizeof(double)));
    eo.dmeta = static_cast<double*>(c.scratch("evd_dmeta", 8 * sizeof(double)));
    eo.imeta = static_cast<int*>(c.scratch("evd_imeta", 8 * sizeof(int)));
    const int lift_P = lift_grid(n, c.sms);
    double* lp = nullptr;
    double* res_out = nullptr;  // U (n x req): coordinates or Ritz vectors
    if (what == What::Embed || what == What::EigsVectors) {
        lp = static_cast<double*>(c.scratch(
            "lift_part", (static_cast<size_t>(lift_P) * 2 + 1) * std::max<size_t>(req, 1) * 8));
        res_out = static_cast<double*>(
            c.scratch("lift_out", n * std::max<size_t>(req, 1) * sizeof(double)));
    }
    // the solve's own copy of its result (the workspace is reused), allocated
    // here: an allocation that fails evicts the S-digit slot and the captured
    // graphs, so none may happen once the slot is claimed (below)
    std::shared_ptr<DevBuf> dres;
    if (res_out) dres = std::make_shared<DevBuf>(n * std::max<size_t>(req, 1) * 8);
    // read back into pinned memory, one sync for all of it
    struct Meta {
        double vals[kMaxWP];
        double kept[kMaxWP];
        double dmeta[8];
        int imeta[8];
        int flags;
    };
    Meta& meta = *static_cast<Meta*>(c.pinned_scratch("run_meta", sizeof(Meta)));

    // the reduce's slot table of this split (uploaded here, outside a capture)
    const int* slot_tab =
        use_i8 ? k2_slot_table((static_cast<int>(n) + 127) / 128, iplan.nks, iplan.total, iplan.grid,
                               iplan.maxseg)
               : k2_slot_table(plan.nb, plan.nk, plan.total, plan.grid, plan.maxseg);
    const int* slot_tab_s =
        use_i8 ? k2_slot_table((static_cast<int>(n) + 127) / 128, splan.nks, splan.total,
                               splan.grid, splan.maxseg)
               : nullptr;

    // S-digit cache (k2i_product.cu, sdig_item_bytes): the first product
    // pass stores every item's S digit planes, the later passes stream them
    // instead of D: no conversion (the bound of the CTA pair, the NB = 64
    // groups and the Hamming slices) and SD instead of 8 bytes per element
    // (measured per later pass: C5 4.3 -> 2.4 ms, n = 40k w = 70 5.0 -> 3.5
    // ms, w = 50 3.6 -> 2.7 ms; the HBM-bound C2 pass 0.556 -> 0.437 ms
    // against a storing pass of 1.07 ms: 3.34 -> 3.25 ms per solve).
    // Claimed last (evictable: a later failed allocation drops it); skipped
    // when it would leave less than max(1 GB, 2 %) of the device free.
    // DSB_SDIG / divscope_set_sdig_cache: 0 off, 1 auto (default: on when it
    // fits), 2 on.
    unsigned char* sdig = nullptr;
    // the gram's K1 pass already wrote the digits (and nothing has written
    // or evicted the slot since): every pass streams them
    const bool k1dig = use_i8 && sdig_policy() > 0 && g.gram->sdig_gen != 0 &&
                       g.gram->sdig_gen == c.sdig_gen &&
                       g.gram->sdig_sd == (hamming_i8 ? 3 : 7);
    if (use_i8) {
        const int pol = sdig_policy();
        if (pol > 0)
            sdig = static_cast<unsigned char*>(
                c.try_scratch("i8_sdig", k2i_sdig_bytes(iplan, hamming_i8 ? 3 : 7)));
    }
    const bool stores = sdig && !k1dig;
    if (stores) ++c.sdig_gen;  // this solve's first pass overwrites the slot
    // the row exponents the product scales by: the digits' own
    const int* prod_row_exp =
        !use_i8 ? nullptr
                : (k1dig && g.gram->sdig_sd == 7 ? g.gram->row_eb->as<int>()
                                                 : g.gram->row_exp->as<int>());
    c.last_product_sdig = sdig ? (k1dig ? 2 : 1) : 0;
    c.last_product_stream_cl = sdig ? splan.cl : 0;
    int sdig_pass = 0;

    // the solve as one stream sequence: eager, or captured once per signature
    // (shape, product kernel, workspace addresses) and replayed as a CUDA
    // graph — 25-40 dependent launches per solve, whose launch gaps are most
    // of a small solve's time
    bool stats_ready = false;
    int nprod = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* graph_timed = nullptr;
    auto product = [&](const double* x, double* y) {
        if (stats_ready) {
            // the orth kernel that produced x left its column statistics
            launch_colstats_final(cstat, orth_fused_grid(n_pad, c.sms), wp, use_i8 ? i8_nb : 0,
                                  colsums, use_i8 ? col_exp : nullptr, c.stream);
        } else if (use_i8) {
            launch_colsums(x, row_mean, n, n_pad, wp, psmall, colsums, c.sms, c.stream, pmax,
                           i8_nb, col_exp);
        } else if (mode) {
            launch_colsums(x, row_mean, n, n_pad, wp, psmall, colsums, c.sms, c.stream);
        }
        stats_ready = false;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (graph_timed) {
            // graph-owned timing events (read after every replay)
            if (c.timing) {
                DSB_CUDA(cudaEventCreate(&e0));
                DSB_CUDA(cudaEventCreate(&e1));
                graph_timed->emplace_back(e0, e1);
            }
        } else {
            c.make_events(&e0, &e1);
        }
        if (use_i8)
            launch_k2i(s.tmap_for(128), &s.tmap64, s.dt, iplan, wp, x, n_pad,
                       prod_row_exp, pmax,
                       col_exp, bdig, part, row_mean, scal_dev, colsums, y, n_pad, c.stream, e0,
                       e1, nullptr, hamming_i8, sdig,
                       sdig ? ((k1dig || sdig_pass++ > 0) ? 2 : 1) : 0,
                       &splan);
        else
            launch_k2(s.tmap_for(plan.bm), s.dt, mode, plan, x, part, row_mean, scal_dev, colsums,
                      y, n_pad, c.stream, e0, e1);
        if (!graph_timed) c.add_timed(nprod == 0 ? 3 : 1, e0, e1);
        ++nprod;
        mark("product");
    };
    // CholeskyQR3 with shift/drop handling: y -> t -> y -> out
    auto orth = [&](double* y, double* t, double* out) {
        if (wp <= 64 &&
            launch_orth_fused(y, t, out, n_pad, wp, wi, n, psmall, wmat, flags, c.sms, c.stream,
                              mode ? row_mean : nullptr, (mode || use_i8) ? cstat : nullptr)) {
            stats_ready = mode || use_i8;
            mark("orth");
            return;
        }
        stats_ready = false;
        launch_panel_dot(y, y, n_pad, wp, psmall, wmat, c.sms, c.stream);
        launch_chol_inv(wmat, wp, wi, n, 1, rinv, flags, c.stream);
        launch_panel_apply(y, rinv, n_pad, wp, t, c.stream);
        launch_panel_dot(t, t, n_pad, wp, psmall, wmat, c.sms, c.stream);
        launch_chol_inv(wmat, wp, wi, n, 0, rinv, flags, c.stream);
        launch_panel_apply(t, rinv, n_pad, wp, y, c.stream);
        launch_panel_dot(y, y, n_pad, wp, psmall, wmat, c.sms, c.stream);
        launch_chol_inv(wmat, wp, wi, n, 0, rinv, flags, c.stream);
        launch_panel_apply(y, rinv, n_pad, wp, out, c.stream);
    };
    // ref rsvd.cpp:94-98, then (not for the range) :108-145
    auto enqueue = [&] {
        stats_ready = false;
        nprod = 0;
        sdig_pass = 0;  // every solve stores the cache in its first pass
        DSB_CUDA(cudaMemsetAsync(flags, 0, 64, c.stream));
        DSB_CUDA(cudaMemcpyAsync(P0, omega_cached, pbytes, cudaMemcpyDeviceToDevice, c.stream));
        mark("start");
        product(P0, P1);
        orth(P1, P2, P0);
        for (size_t it = 0; it < q; ++it) {
            product(P0, P1);
            orth(P1, P2, P0);
            product(P0, P1);
            orth(P1, P2, P0);
        }
        if (what == What::Range) return;
        // ref rsvd.cpp:108-110: GQ, B = Q^T GQ (symmetrized inside K5)
        product(P0, P1);
        launch_panel_dot(P0, P1, n_pad, wp, psmall, wmat, c.sms, c.stream);
        mark("ritz_gram");
        launch_evd(wmat, wp, wi, static_cast<int>(rank), evd_req, scal_dev, fro_index, eo,
                   c.stream);
        mark("evd");
        if (what == What::Embed)
            launch_lift(P0, n, wp, wi, eo.vkeep, eo.kept_vals, eo.imeta, static_cast<int>(req),
                        res_out, lp, c.sms, c.stream);
        if (what == What::EigsVectors)  // U = Q V_keep (no sign rule, no scaling)
            launch_lift_partial(P0, n, wp, wi, eo.vkeep, eo.imeta, static_cast<int>(req), res_out,
                                lp, 0, lift_P, c.stream);
        DSB_CUDA(cudaGetLastError());
        DSB_CUDA(cudaMemcpyAsync(meta.vals, eo.vals, w * 8, cudaMemcpyDeviceToHost, c.stream));
        DSB_CUDA(cudaMemcpyAsync(meta.kept, eo.kept_vals, w * 8, cudaMemcpyDeviceToHost, c.stream));
        DSB_CUDA(cudaMemcpyAsync(meta.dmeta, eo.dmeta, 8 * 8, cudaMemcpyDeviceToHost, c.stream));
        DSB_CUDA(cudaMemcpyAsync(meta.imeta, eo.imeta, 8 * sizeof(int), cudaMemcpyDeviceToHost,
                                 c.stream));
        DSB_CUDA(cudaMemcpyAsync(&meta.flags, flags, sizeof(int), cudaMemcpyDeviceToHost,
                                 c.stream));
        mark("lift");
    };

    RunOut out;
    if (what == What::Range) {
        enqueue();
        double* rm = static_cast<double*>(c.scratch("range_rm", n * w * sizeof(double)));
        launch_panel_to_rowmajor(P0, n, wi, wp, rm, c.stream);
        DSB_CUDA(cudaGetLastError());
        c.d2h_copy(range_out, rm, n * w * sizeof(double));
        return out;
    }
    static const bool graphs_on = [] {
        const char* e = std::getenv("DSB_GRAPH");
        return !(e && std::atoi(e) == 0);
    }();
    Ctx::GraphEntry* ge = nullptr;
    if (graphs_on && !trace && !c.graphs_broken) {
        uint64_t h = 1469598103934665603ull;
        auto mix = [&](uint64_t v) {
            for (int i = 0; i < 8; ++i) {
                h ^= (v >> (8 * i)) & 0xff;
                h *= 1099511628211ull;
            }
        };
        auto mixp = [&](const void* ptr) { mix(reinterpret_cast<uintptr_t>(ptr)); };
        mix(n); mix(w); mix(wp); mix(q); mix(rank); mix(req); mix(static_cast<uint64_t>(evd_req));
        mix(static_cast<uint64_t>(what)); mix(use_i8); mix(static_cast<uint64_t>(hamming_i8));
        mix(mode); mix(static_cast<uint64_t>(s.dt)); mix(s.rows); mix(s.cols); mix(s.ld);
        mix(static_cast<uint64_t>(fro_index)); mix(c.timing); mix(static_cast<uint64_t>(c.sms));
        mix(static_cast<uint64_t>(product_path()));
        mixp(s.buf ? s.buf->p : nullptr); mixp(scal_dev); mixp(row_mean);
        mixp(use_i8 ? g.gram->row_exp->p : nullptr);
        mixp(prod_row_exp);
        mix(k1dig);
        for (const void* ptr : {static_cast<const void*>(P0), static_cast<const void*>(P1),
                                static_cast<const void*>(P2), static_cast<const void*>(part),
                                static_cast<const void*>(psmall),
                                static_cast<const void*>(colsums),
                                static_cast<const void*>(wmat), static_cast<const void*>(rinv),
                                static_cast<const void*>(flags), static_cast<const void*>(cstat),
                                static_cast<const void*>(pmax), static_cast<const void*>(col_exp),
                                static_cast<const void*>(bdig),
                                static_cast<const void*>(sdig),
                                static_cast<const void*>(omega_cached),
                                static_cast<const void*>(eo.vals),
                                static_cast<const void*>(eo.vkeep),
                                static_cast<const void*>(eo.kept_vals),
                                static_cast<const void*>(eo.dmeta),
                                static_cast<const void*>(eo.imeta), static_cast<const void*>(lp),
                                static_cast<const void*>(res_out),
                                static_cast<const void*>(&meta),
                                static_cast<const void*>(slot_tab),
                                static_cast<const void*>(slot_tab_s)})
            mixp(ptr);
        auto it = c.graphs.find(h);
        if (it != c.graphs.end()) {
            ge = &it->second;
            count_launch(static_cast<int>(ge->launches));
        } else {
            if (c.graphs.size() >= 16) c.clear_graphs();
            Ctx::GraphEntry e;
            graph_timed = &e.timed;
            const uint64_t l0 = kernel_launch_count();
            cudaGraph_t graph = nullptr;
            DSB_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
            try {
                enqueue();
            } catch (...) {
                cudaStreamEndCapture(c.stream, &graph);
                if (graph) cudaGraphDestroy(graph);
                graph_timed = nullptr;
                for (auto& ev : e.timed) {
                    cudaEventDestroy(ev.first);
                    cudaEventDestroy(ev.second);
                }
                throw;
            }
            graph_timed = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(c.stream, &graph);
            cudaGraphExec_t exec = nullptr;
            if (ce == cudaSuccess && graph &&
                cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
                e.exec = exec;
                e.launches = kernel_launch_count() - l0;
                e.products = nprod;
                ge = &(c.graphs[h] = std::move(e));
            } else {
                // this sequence does not capture here: eager from now on
                (void)cudaGetLastError();
                c.graphs_broken = true;
                for (auto& ev : e.timed) {
                    cudaEventDestroy(ev.first);
                    cudaEventDestroy(ev.second);
                }
            }
            if (graph) cudaGraphDestroy(graph);
        }
    }
    if (ge) {
        DSB_CUDA(cudaGraphLaunch(ge->exec, c.stream));
        c.k2_launches += static_cast<uint64_t>(ge->products);
        if (ge->products > 0) ++c.k2_first_launches;
    } else {
        enqueue();
    }
    if (res_out)
        DSB_CUDA(cudaMemcpyAsync(dres->p, res_out, n * std::max<size_t>(req, 1) * 8,
                                 cudaMemcpyDeviceToDevice, c.stream));
    if (trace) std::fprintf(stderr, "[trace] host enqueue done %.1f us\n", host_us());
    c.sync();
    if (ge && c.timing)
        for (size_t i = 0; i < ge->timed.size(); ++i) {
            float ms = 0.f;
            DSB_CUDA(cudaEventElapsedTime(&ms, ge->timed[i].first, ge->timed[i].second));
            c.k2_ms += ms;
            if (i == 0) c.k2_first_ms += ms;
        }
    if (trace) std::fprintf(stderr, "[trace] host meta synced %.1f us\n", host_us());
    if (trace) {
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
            std::fprintf(stderr, "[trace] %-10s %8.1f us\n", marks[i].first, ms * 1e3);
        }
        for (auto& m : marks) cudaEventDestroy(m.second);
    }
    c.d2h += w * 16 + 64 + 32 + 4;
    c.last_evd_sweeps = meta.imeta[3];
    c.last_orth_shifted = meta.flags & 1;
    if (!meta.imeta[4])
        throw Error(errc::internal, "small eigensolve failed");  // ref rsvd.cpp:113-114
    out.vals.assign(meta.vals, meta.vals + w);
    out.keep = static_cast<size_t>(meta.imeta[0]);
    out.resid = meta.dmeta[0];
    if (what == What::EigsVectors) {
        out.vectors.resize(n * out.keep);
        c.d2h_copy(out.vectors.data(), dres->p, out.vectors.size() * sizeof(double));
    }
    if (what == What::Embed) {
        Embedding& e = out.emb;
        e.n = n;
        e.r = static_cast<size_t>(meta.imeta[1]);
        e.truncated = meta.imeta[2] != 0;
        e.dropped_negative_mass = meta.dmeta[1];
        e.resid = meta.dmeta[0];
        e.eigenvalues.assign(meta.kept, meta.kept + e.r);
        // the lift wrote n x req with row stride r (= kept columns)
        e.dcoords = std::move(dres);
    }
    if (trace) std::fprintf(stderr, "[trace] host coords done %.1f us\n", host_us());
    return out;
}

}  // namespace

Matrix matrix_from_host(const void* values, size_t rows, size_t cols, bool symmetric, DType dt) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    Matrix m;
    m.store = make_store(rows, cols, symmetric, dt);
    upload_rows(*m.store, values, cols);
    c.sync();  // the caller may release its buffer on return
    return m;
}

Matrix gram_from_distances(const Matrix& d) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    Store& s = *d.store;
    // ref mds.cpp:15-20
    if (s.rows != s.cols || !s.symmetric)
        throw Error(errc::not_symmetric, "gram matrix requires a symmetric distance matrix");
    const size_t n = s.rows;
    if (n == 0) throw Error(errc::empty_input, "empty distance matrix");
    // K1 also writes the S-digit cache when the solves on this gram will run
    // the int8 product (f64 D, n >= 4096, unsharded) and the cache fits: the
    // row exponents of the digits are then a bound from row 0 (verified by
    // K1 against the true ones); Hamming slices need none
    K1Digits dig;
    std::shared_ptr<DevBuf> row_eb;
    const int ham_sd = (s.hamming_len > 0 && s.hamming_len < 4096 && hamming_slices_enabled());
    auto claim = [&]() -> const K1Digits* {
        if (!(s.dt == DType::F64 && !s.sharded && n >= 4096 && sdig_policy() > 0 &&
              product_path() != 1))
            return nullptr;
        const size_t nblk = (n + 127) / 128, nks = (n + 31) / 32;
        dig.sd = ham_sd ? 3 : 7;
        dig.nks = static_cast<int>(nks);
        dig.hlen = static_cast<double>(s.hamming_len);
        if (dig.sd == 7) {
            row_eb = std::make_shared<DevBuf>(n * sizeof(int));
            dig.row_eb = row_eb->as<int>();
        }
        dig.sdig = static_cast<unsigned char*>(
            c.try_scratch("i8_sdig", nblk * nks * static_cast<size_t>(dig.sd) * 4096));
        return dig.sdig ? &dig : nullptr;
    };
    StatsOut o = run_k1(s, claim);
    uint64_t gen = 0;
    if (dig.sdig) {
        gen = ++c.sdig_gen;  // whatever the slot held before is overwritten
        if (dig.sd == 7 && o.sc[S_SDIG_BAD] != 0.0) gen = 0;  // bound failed: unused
    }
    // ref mds.cpp:21-27
    if (o.sc[S_MAXASYM] > 1e-12 * std::max(1.0, o.sc[S_MAXABS]))
        throw Error(errc::not_symmetric, "distance matrix values are not symmetric");
    Matrix g;
    g.store = d.store;
    g.gram = std::make_shared<GramInfo>();
    g.gram->n = n;
    g.gram->row_mean = o.row_mean;
    g.gram->row_exp = o.row_exp;
    g.gram->scalars = o.scalars;
    std::memcpy(g.gram->sc, o.sc, sizeof(o.sc));
    g.gram->sdig_gen = gen;
    g.gram->sdig_sd = gen ? dig.sd : 0;
    g.gram->row_eb = gen ? row_eb : nullptr;
    return g;
}

Spectrum eigs_sym(const Matrix& g, const SolverOptions& opts) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    RunOut r = run(g, opts.rank, opts.oversampling, opts.power_iters, opts.seed, What::Eigs,
                   opts.rank, nullptr);
    Spectrum s;
    s.eigenvalues.assign(r.vals.begin(), r.vals.begin() + r.keep);
    s.resid = r.resid;
    return s;
}

Spectrum eigs_sym_vectors(const Matrix& g, const SolverOptions& opts) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (g.store->sharded)
        throw Error(errc::invalid_argument, "eigenvectors are not available on row shards");
    RunOut r = run(g, opts.rank, opts.oversampling, opts.power_iters, opts.seed,
                   What::EigsVectors, opts.rank, nullptr);
    Spectrum s;
    s.eigenvalues.assign(r.vals.begin(), r.vals.begin() + r.keep);
    s.resid = r.resid;
    s.vectors = std::move(r.vectors);
    return s;
}

const double* Embedding::host_coords() const {
    if (n * r == 0) return nullptr;
    std::call_once(*once_, [this] {
        if (!dcoords) return;
        Ctx& c = Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        PinnedVec h(n * r);
        c.d2h_copy(h.data(), dcoords->p, n * r * sizeof(double));
        coords_ = std::move(h);
    });
    return coords_.empty() ? nullptr : coords_.data();
}

void Embedding::set_host_coords(const std::vector<double>& v) {
    coords_.assign(v);
    dcoords.reset();
}

Embedding embed(const Matrix& g, size_t rank, SolverOptions opts) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const size_t n = g.n();
    // ref mds.cpp:118-121
    if (rank < 1 || rank > n) throw Error(errc::rank_too_large, "rank must be in [1, n]");
    opts.rank = rank;
    opts.oversampling = std::min(opts.oversampling, n - rank);
    RunOut r = run(g, opts.rank, opts.oversampling, opts.power_iters, opts.seed, What::Embed, rank,
                   nullptr);
    return std::move(r.emb);
}

// ref src/mds.cpp:126-150 (shape check, then sqrt of the summed squares)
double reconstruction_error(const Matrix& g, const Embedding& e) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    Store& s = *g.store;
    if (s.sharded)
        throw Error(errc::invalid_argument, "reconstruction_error on a row shard is not supported");
    const size_t n = g.n();
    if (e.n != n) throw Error(errc::shape_mismatch, "embedding/gram size mismatch");
    if (n == 0) return 0.0;
    const bool lazy = static_cast<bool>(g.gram);
    const size_t r = e.r;
    double* x = static_cast<double*>(c.scratch("recon_x", std::max<size_t>(n * r, 1) * 8));
    if (r && e.dcoords)
        DSB_CUDA(cudaMemcpyAsync(x, e.dcoords->p, n * r * sizeof(double), cudaMemcpyDeviceToDevice,
                                 c.stream));
    else if (r)
        c.h2d_copy(x, e.host_coords(), n * r * sizeof(double));
    double* part = static_cast<double*>(c.scratch("recon_part", recon_blocks(n, lazy) * 8));
    double* out = static_cast<double*>(c.scratch("recon_out", 64));
    launch_recon(s.buf->p, s.dt, s.ld, n, lazy, lazy ? g.gram->row_mean->as<double>() : nullptr,
                 lazy ? g.gram->scalars->as<double>() : nullptr, x, static_cast<int>(r), part,
                 out, c.stream);
    DSB_CUDA(cudaGetLastError());
    double total = 0.0;
    c.d2h_copy(&total, out, sizeof(double));
    return std::sqrt(total);
}

void randomized_range(const Matrix& g, const SolverOptions& opts, double* q_out) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    run(g, opts.rank, opts.oversampling, opts.power_iters, opts.seed, What::Range, opts.rank,
        q_out);
}

// host copy of the row means, fetched on first use (matrix_get / _write)
static const std::vector<double>& host_row_means(GramInfo& g) {
    std::lock_guard<std::mutex> lk(g.mu);
    if (g.row_mean_h.size() != g.n) {
        g.row_mean_h.resize(g.n);
        Ctx::get().d2h_copy(g.row_mean_h.data(), g.row_mean->p, g.n * sizeof(double));
    }
    return g.row_mean_h;
}

double matrix_get(const Matrix& m, size_t i, size_t j) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const Store& s = *m.store;
    const size_t esz = s.dt == DType::F64 ? 8 : 4;
    auto fetch = [&](size_t a, size_t b) {
        unsigned char buf[8];
        c.d2h_copy(buf, static_cast<const char*>(s.buf->p) + (a * s.ld + b) * esz, esz);
        if (esz == 8) {
            double v;
            std::memcpy(&v, buf, 8);
            return v;
        }
        float f;
        std::memcpy(&f, buf, 4);
        return static_cast<double>(f);
    };
    if (!m.gram) return fetch(i, j);
    // ref mds.cpp:50-51 (upper) and :57-58 (mirror)
    const auto& rm = host_row_means(*m.gram);
    const double grand = m.gram->sc[S_GRAND];
    if (i <= j) {
        const double dij = fetch(i, j);
        return -0.5 * (dij * dij - rm[i] - rm[j] + grand);
    }
    const double dji = fetch(j, i);
    return -0.5 * (dji * dji - rm[j] - rm[i] + grand);
}

void matrix_to_host(const Matrix& m, double* out) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const Store& s = *m.store;
    const size_t esz = s.dt == DType::F64 ? 8 : 4;
    std::vector<unsigned char> raw(s.rows * s.cols * esz);
    if (!raw.empty()) {
        DSB_CUDA(cudaMemcpy2DAsync(raw.data(), s.cols * esz, s.buf->p, s.ld * esz, s.cols * esz,
                                   s.rows, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        c.d2h += raw.size();
    }
    const size_t rows = s.rows, cols = s.cols;
    auto at = [&](size_t a, size_t b) {
        if (esz == 8) {
            double v;
            std::memcpy(&v, &raw[(a * cols + b) * 8], 8);
            return v;
        }
        float f;
        std::memcpy(&f, &raw[(a * cols + b) * 4], 4);
        return static_cast<double>(f);
    };
    if (!m.gram) {
        for (size_t a = 0; a < rows; ++a)
            for (size_t b = 0; b < cols; ++b) out[a * cols + b] = at(a, b);
        return;
    }
    const auto& rm = host_row_means(*m.gram);
    const double grand = m.gram->sc[S_GRAND];
    for (size_t a = 0; a < rows; ++a)
        for (size_t b = a; b < cols; ++b) {
            const double dab = at(a, b);
            const double v = -0.5 * (dab * dab - rm[a] - rm[b] + grand);
            out[a * cols + b] = v;
            out[b * cols + a] = v;
        }
}

constexpr int kSrMaxIters = 20000;  // ref rsvd.cpp:160

double stable_rank(const Matrix& g) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    Store& s = *g.store;
    const size_t n = s.rows;
    const bool lazy = static_cast<bool>(g.gram);
    double fro2;
    const double* scal_dev;
    const double* row_mean = nullptr;
    if (lazy) {
        fro2 = g.gram->sc[S_FRO2_LAZY];
        scal_dev = g.gram->scalars->as<double>();
        row_mean = g.gram->row_mean->as<double>();
    } else {
        if (n == 0) throw Error(errc::invalid_argument, "empty matrix");
        ensure_explicit_stats(s);
        if (s.stats[S_MAXASYM] > 1e-10 * std::max(1.0, s.stats[S_MAXABS_UP]))
            throw Error(errc::not_symmetric, "matrix is not symmetric");
        fro2 = s.stats[S_FRO2_EXPL];
        scal_dev = s.stats_dev->as<double>();
    }
    if (fro2 == 0.0) throw Error(errc::zero_matrix, "stable rank undefined for zero matrix");
    const int mode = lazy ? 1 : 0;
    const int wp = 8;
    const size_t n_pad = round_up(n, kRowPad);
    ensure_tmap(s);
    const K2Plan plan = k2_plan(n, wp, s.dt, c.sms);
    double* X = static_cast<double*>(c.scratch("sr_x", n_pad * wp * 8));
    double* Y = static_cast<double*>(c.scratch("sr_y", n_pad * wp * 8));
    double* part = static_cast<double*>(c.scratch("k2_part", plan.part_elems * 8));
    const int pg = panel_grid(n_pad, c.sms);
    double* psmall = static_cast<double*>(c.scratch("panel_part", static_cast<size_t>(pg) * wp * wp * 8 + 64));
    double* colsums = static_cast<double*>(c.scratch("colsums", 2 * wp * 8));
    double* stage = static_cast<double*>(c.scratch("sr_stage", n * 8));
    // ref rsvd.cpp:157-176: v ~ fill_gaussian(mt19937_64(0x5eed)), normalized
    std::mt19937_64 eng(0x5eedULL);
    std::vector<double> v(n);
    auto load_v = [&](bool from_engine) {
        if (from_engine) {
            fill_gaussian(eng, v.data(), n);
            double ss = 0.0;
            for (double a : v) ss += a * a;
            const double nrm = std::sqrt(ss);
            for (double& a : v) a /= nrm;
        }
        c.h2d_copy(stage, v.data(), n * 8);
        launch_panel_from_rowmajor(stage, n, 1, wp, n_pad, X, c.stream);
    };
    // The loop runs on the device in batches: K2 (skipped once converged),
    // then launch_sr_step (norm, restart flag, convergence test, v = w/norm).
    // The host reads the state once per batch.
    SrState* dstate = static_cast<SrState*>(c.scratch("sr_state", sizeof(SrState)));
    static SrState* hstate = nullptr;
    if (!hstate) DSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hstate), sizeof(SrState)));
    double* npart = static_cast<double*>(c.scratch("sr_part", static_cast<size_t>(c.sms) * 8));
    auto reset_state = [&](int iters) {
        *hstate = SrState{0.0, 0.0, 0, 0, iters, 0};
        DSB_CUDA(cudaMemcpyAsync(dstate, hstate, sizeof(SrState), cudaMemcpyHostToDevice, c.stream));
        DSB_CUDA(cudaStreamSynchronize(c.stream));
    };
    load_v(true);
    reset_state(0);
    double sigma = 0.0;
    int batch = 8;
    for (;;) {
        const int todo = std::min(batch, kSrMaxIters - hstate->iters);
        if (todo <= 0) break;
        for (int k = 0; k < todo; ++k) {
            if (mode) launch_colsums(X, row_mean, n, n_pad, wp, psmall, colsums, c.sms, c.stream);
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            c.make_events(&e0, &e1);
            launch_k2(s.tmap_for(plan.bm), s.dt, mode, plan, X, part, row_mean, scal_dev, colsums,
                      Y, n_pad, c.stream, e0, e1, &dstate->done);
            c.add_timed(1, e0, e1);
            launch_sr_step(Y, n, wp, npart, dstate, X, c.sms, c.stream);
        }
        DSB_CUDA(cudaMemcpyAsync(hstate, dstate, sizeof(SrState), cudaMemcpyDeviceToHost, c.stream));
        DSB_CUDA(cudaStreamSynchronize(c.stream));
        if (hstate->zero) {  // ref rsvd.cpp:163-168: redraw, sigma = 0, continue
            load_v(true);
            reset_state(hstate->iters);
            continue;
        }
        sigma = hstate->sigma;
        if (hstate->done) break;
        batch = 32;
    }
    c.last_power_iters = hstate->iters;
    c.sync();
    return fro2 / (sigma * sigma);
}

Matrix matrix_euclidean(const double* pts, size_t n, size_t dim, bool f32) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (n == 0 || dim == 0) throw Error(errc::empty_input, "no points");
    if (dim > 256) throw Error(errc::invalid_argument, "dimension > 256 not supported");
    Matrix m;
    m.store = make_store(n, n, true, f32 ? DType::F32 : DType::F64);
    DevBuf dp(n * dim * sizeof(double));
    c.h2d_copy(dp.p, pts, n * dim * sizeof(double));
    launch_euclid(dp.as<double>(), n, static_cast<int>(dim), m.store->buf->p, m.store->dt,
                  m.store->ld, c.stream);
    c.sync();
    return m;
}

namespace {
// Reads -> the two bit planes of K7 on the device: one host->device copy of
// the bytes (count x length), packing and validation in a kernel. Errors as
// a host scan would report them: the first non-A/C/G/T byte in read-major
// order. Returns lo planes at [0, count * words), hi planes after them.
std::shared_ptr<DevBuf> pack_reads_device(const char* reads, size_t count, size_t length,
                                          int& words) {
    Ctx& c = Ctx::get();
    if (count == 0 || length == 0) throw Error(errc::empty_input, "no reads");
    words = static_cast<int>((length + 31) / 32);
    DevBuf raw(count * length);
    c.h2d_copy(raw.p, reads, count * length);
    auto planes = std::make_shared<DevBuf>(2 * count * static_cast<size_t>(words) * 4);
    auto* bad = static_cast<unsigned long long*>(c.scratch("pack_bad", 8));
    DSB_CUDA(cudaMemsetAsync(bad, 0xff, 8, c.stream));
    uint32_t* lo = planes->as<uint32_t>();
    launch_pack_reads(raw.as<unsigned char>(), count, static_cast<int>(length), words, lo,
                      lo + count * static_cast<size_t>(words), bad, c.sms, c.stream);
    unsigned long long first = ~0ull;
    c.d2h_copy(&first, bad, 8);
    if (first != ~0ull) {
        const size_t i = static_cast<size_t>(first / length), t = static_cast<size_t>(first % length);
        throw Error(errc::invalid_character, "read " + std::to_string(i) + ": base " +
                                                 std::to_string(t + 1) + " is not A/C/G/T");
    }
    return planes;
}
}  // namespace

Matrix matrix_hamming(const char* reads, size_t count, size_t length) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    int words = 0;
    const auto packed = pack_reads_device(reads, count, length, words);
    Matrix m;
    m.store = make_store(count, count, true, DType::F64);
    m.store->hamming_len = static_cast<int>(length);
    launch_hamming(packed->as<uint32_t>(), packed->as<uint32_t>() + count * static_cast<size_t>(words),
                   count, words, static_cast<int>(length),
                   m.store->buf->as<double>(), m.store->ld, nullptr, c.stream);
    c.sync();
    return m;
}

// rows [row_begin, row_end) of the Hamming matrix as a row shard (K7 shards
// by output rows with no communication)
Matrix matrix_hamming_rows(const char* reads, size_t count, size_t length, size_t row_begin,
                           size_t row_end) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (row_end < row_begin || row_end > count)
        throw Error(errc::invalid_argument, "bad row range");
    int words = 0;
    const auto packed = pack_reads_device(reads, count, length, words);
    Matrix m;
    m.store = make_store(row_end - row_begin, count, true, DType::F64);
    m.store->sharded = true;
    m.store->n_global = count;
    m.store->row_begin = row_begin;
    m.store->hamming_len = static_cast<int>(length);
    launch_hamming(packed->as<uint32_t>(), packed->as<uint32_t>() + count * static_cast<size_t>(words),
                   count, words, static_cast<int>(length),
                   m.store->buf->as<double>(), m.store->ld, nullptr, c.stream, row_begin,
                   row_end - row_begin);
    c.sync();
    return m;
}

void hamming_counts(const char* reads, size_t count, size_t length, uint32_t* out) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    int words = 0;
    const auto packed = pack_reads_device(reads, count, length, words);
    DevBuf dc(count * count * sizeof(uint32_t));
    launch_hamming(packed->as<uint32_t>(), packed->as<uint32_t>() + count * static_cast<size_t>(words),
                   count, words, static_cast<int>(length),
                   nullptr, 0, dc.as<uint32_t>(), c.stream);
    c.d2h_copy(out, dc.p, count * count * sizeof(uint32_t));
}

// test hook (divscope_debug_omega_panel): the Omega panel exactly as a
// solve starts from it — host fill_gaussian into the pinned buffer, H2D,
// relayout into the k4-interleaved device panel — read back row-major
void debug_omega_panel(uint64_t seed, size_t n, size_t w, double* out) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (n == 0 || w == 0 || w > static_cast<size_t>(kMaxWP))
        throw Error(errc::invalid_argument, "bad Omega shape");
    const int wp = static_cast<int>(round_up(w, 8));
    const size_t n_pad = round_up(n, kRowPad);
    DevBuf panel(n_pad * wp * sizeof(double));
    DevBuf stage(n * w * sizeof(double));
    c.h2d_copy(stage.p, omega_host(seed, n, w), n * w * sizeof(double));
    launch_panel_from_rowmajor(stage.as<double>(), n, static_cast<int>(w), wp, n_pad,
                               panel.as<double>(), c.stream);
    std::vector<double> h(n_pad * wp);
    c.d2h_copy(h.data(), panel.p, h.size() * sizeof(double));
    for (size_t i = 0; i < n; ++i)
        for (size_t k = 0; k < w; ++k) out[i * w + k] = h[pidx(i, static_cast<int>(k), wp)];
    for (size_t i = n; i < n_pad; ++i)  // padding rows must be zero
        for (int k = 0; k < wp; ++k)
            if (h[pidx(i, k, wp)] != 0.0) throw Error(errc::internal, "nonzero Omega padding");
}

}  // namespace dsb
