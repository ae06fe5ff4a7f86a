// Seeded synthetic workloads of BASELINE.json (host side). All randomness
// follows the reference conventions: std::mt19937_64(seed) with
// fill_gaussian / uniform_* / bounded_uint64 (ref src/rng.hpp:16-48), and the
// DNA alphabet draw of ref tests/testdata.cpp:16-26.
#include <cmath>
#include <random>
#include <vector>

#include "divscope.h"
#include "host_core.hpp"

namespace {

using dsb::bounded_uint64;
using dsb::fill_gaussian;
using dsb::uniform_closed_open;
using dsb::uniform_open_closed;

struct ClusterSpec {
    size_t dim, clusters;
    double center_sd;
    bool dirichlet;      // cluster weights ~ Dirichlet(1) (else equal)
    size_t subcenters;   // > 0: hierarchical (config 3)
    double sub_sd;
};

ClusterSpec spec_of(int config) {
    switch (config) {
        case 1: return {20, 5, 10.0, false, 0, 0.0};
        case 2: return {50, 20, 5.0, true, 0, 0.0};
        case 3: return {100, 10, 20.0, false, 10, 3.0};
        case 4: return {64, 100, 8.0, false, 0, 0.0};
        default: throw dsb::Error(dsb::errc::invalid_argument, "config must be 1..4");
    }
}

void synth_points(int config, size_t n, uint64_t seed, double* out, size_t* dim_out) {
    const ClusterSpec sp = spec_of(config);
    std::mt19937_64 eng(seed);
    const size_t dim = sp.dim;
    // 1. top-level centers ~ N(0, center_sd^2 I)
    std::vector<double> centers(sp.clusters * dim);
    fill_gaussian(eng, centers.data(), centers.size());
    for (double& v : centers) v *= sp.center_sd;
    // 2. hierarchical: each top center gets `subcenters` offsets ~ N(0, sub_sd^2 I)
    size_t k_total = sp.clusters;
    if (sp.subcenters) {
        k_total = sp.clusters * sp.subcenters;
        std::vector<double> sub(k_total * dim);
        fill_gaussian(eng, sub.data(), sub.size());
        for (size_t k = 0; k < k_total; ++k)
            for (size_t c = 0; c < dim; ++c)
                sub[k * dim + c] = centers[(k / sp.subcenters) * dim + c] + sp.sub_sd * sub[k * dim + c];
        centers.swap(sub);
    }
    // 3. labels: equal weights -> bounded_uint64; Dirichlet(1) weights are
    //    normalized Exp(1) = -log(uniform_open_closed) draws, then each point
    //    picks the first k with u < cumulative weight (u = uniform_closed_open)
    std::vector<size_t> label(n);
    if (sp.dirichlet) {
        std::vector<double> wts(k_total);
        double tot = 0.0;
        for (double& g : wts) {
            g = -std::log(uniform_open_closed(eng));
            tot += g;
        }
        std::vector<double> cum(k_total);
        double acc = 0.0;
        for (size_t k = 0; k < k_total; ++k) {
            acc += wts[k] / tot;
            cum[k] = acc;
        }
        for (size_t i = 0; i < n; ++i) {
            const double u = uniform_closed_open(eng);
            size_t k = 0;
            while (k + 1 < k_total && !(u < cum[k])) ++k;
            label[i] = k;
        }
    } else {
        for (size_t i = 0; i < n; ++i) label[i] = bounded_uint64(eng, k_total);
    }
    // 4. within-cluster noise sigma = 1
    fill_gaussian(eng, out, n * dim);
    for (size_t i = 0; i < n; ++i)
        for (size_t c = 0; c < dim; ++c) out[i * dim + c] += centers[label[i] * dim + c];
    if (dim_out) *dim_out = dim;
}

void synth_reads(size_t count, size_t length, size_t ancestors, double sub_rate, uint64_t seed,
                 char* out) {
    static const char bases[4] = {'A', 'C', 'G', 'T'};
    std::mt19937_64 eng(seed);
    std::vector<int> anc(ancestors * length);
    for (int& b : anc) b = static_cast<int>(bounded_uint64(eng, 4));  // testdata.cpp:16-26
    for (size_t i = 0; i < count; ++i) {
        const size_t a = bounded_uint64(eng, ancestors);
        for (size_t t = 0; t < length; ++t) {
            int b = anc[a * length + t];
            if (uniform_closed_open(eng) < sub_rate)
                b = static_cast<int>((b + 1 + bounded_uint64(eng, 3)) % 4);  // a different base
            out[i * length + t] = bases[b];
        }
    }
}

template <typename F>
divscope_status guard(F&& f) noexcept {
    try {
        f();
        return DIVSCOPE_OK;
    } catch (const dsb::Error& e) {
        return static_cast<divscope_status>(static_cast<int>(e.code()));
    } catch (...) {
        return DIVSCOPE_ERR_INTERNAL;
    }
}

}  // namespace

extern "C" {

divscope_status divscope_synth_points(int config, size_t n, uint64_t seed, double* out,
                                      size_t* dim_out) {
    if (!out) return DIVSCOPE_ERR_INVALID_ARGUMENT;
    return guard([&] { synth_points(config, n, seed, out, dim_out); });
}

divscope_status divscope_synth_reads(size_t count, size_t length, size_t ancestors,
                                     double sub_rate, uint64_t seed, char* out) {
    if (!out || ancestors == 0) return DIVSCOPE_ERR_INVALID_ARGUMENT;
    return guard([&] { synth_reads(count, length, ancestors, sub_rate, seed, out); });
}

}  // extern "C"
