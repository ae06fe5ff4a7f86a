// C++ API of the B200 MDS path — the host-side mirror of the reference's
// C++ entry points (ref src/mds.hpp:34-59, src/rsvd.hpp:20-62) over
// device-resident handles. The C ABI (capi.cpp) is a thin wrapper.
#pragma once

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host_core.hpp"

namespace dsb {

// ref src/rsvd.hpp:20-25 (C++ defaults; the C API defaults differ)
struct SolverOptions {
    size_t rank = 1;
    size_t oversampling = 10;
    size_t power_iters = 2;
    uint64_t seed = 0;
};

// A matrix handle: device store + optional lazy-gram terms.
struct Matrix {
    std::shared_ptr<Store> store;
    std::shared_ptr<GramInfo> gram;  // non-null => this handle denotes G(store)
    size_t n() const { return store->order(); }
};

// ref src/rsvd.hpp:29-33 (vectors omitted: the C ABI never returns them)
struct Spectrum {
    std::vector<double> eigenvalues;  // keep = min(rank, w), reference order
    double resid = 0.0;
    // n x keep row-major Ritz vectors, column a pairs with eigenvalues[a]
    // (ref rsvd.hpp:29-33 Spectrum::vectors); filled by eigs_sym_vectors only
    std::vector<double> vectors;
};

// ref src/mds.hpp:21-28
struct Embedding {
    size_t n = 0, r = 0;
    // n x r row-major coordinates. The solver leaves them on the device
    // (dcoords); the host copy is made on first access, so an embed call
    // does not pay the download unless the caller reads them.
    std::shared_ptr<DevBuf> dcoords;
    const double* host_coords() const;  // nullptr when n * r == 0
    void set_host_coords(const std::vector<double>& v);
    std::vector<double> eigenvalues;  // retained, descending
    double dropped_negative_mass = 0.0;
    bool truncated = false;
    double resid = 0.0;

private:
    mutable PinnedVec coords_;
    mutable std::shared_ptr<std::once_flag> once_ = std::make_shared<std::once_flag>();
};

// ref src/mds.cpp:14-60 (validation + centering terms; G not materialized)
Matrix gram_from_distances(const Matrix& d);

// ref src/rsvd.cpp:102-145
Spectrum eigs_sym(const Matrix& g, const SolverOptions& opts);
// eigs_sym with the Ritz vectors Q V_keep (ref rsvd.cpp:129-138), unsharded
Spectrum eigs_sym_vectors(const Matrix& g, const SolverOptions& opts);

// ref src/mds.cpp:116-124 (rank overrides opts.rank, p clamped to n - rank)
Embedding embed(const Matrix& g, size_t rank, SolverOptions opts);

// ref src/rsvd.cpp:81-100 (basis written n x w row-major)
void randomized_range(const Matrix& g, const SolverOptions& opts, double* q_out);

// ref src/rsvd.cpp:147-178
double stable_rank(const Matrix& g);
// ref src/mds.cpp:126-150
double reconstruction_error(const Matrix& g, const Embedding& e);
// product kernel choice: 0 auto, 1 fp64 DMMA only, 2 int8 slice product
// whenever supported (lazy grams, w <= 64)
void set_product_path(int mode);
// S-digit cache policy (divscope_set_sdig_cache): 0 off, 1 auto, 2 on
void set_sdig_policy(int mode);
int sdig_policy();
// whether a product pass on this gram uses the int8 slice product
bool hamming_slices_enabled();  // DSB_K2I_HAMMING (default on)
bool use_int8_product(const GramInfo& gi, int wp);

// G_ij of a handle (lazy gram evaluated like ref mds.cpp:50-58)
double matrix_get(const Matrix& m, size_t i, size_t j);
void matrix_to_host(const Matrix& m, double* out);

Matrix matrix_from_host(const void* values, size_t rows, size_t cols, bool symmetric, DType dt);

// ---- multi-GPU (sharded.cpp): one process per GPU, NCCL ----------------
// rows [row_begin, row_end) of an n x n matrix, uploaded by this rank
// Smith-Waterman distances on the GPU (sw.cu, pairwise.cpp; ref src/align.cpp,
// src/distmat.cpp:45-128)
struct SwScheme {
    int match = 1, mismatch = -1, gap = -2;  // ref align.hpp:13-17
};
struct SwAlignment {
    int score = 0, distance = 0;
    size_t a_begin = 0, a_end = 0, b_begin = 0, b_end = 0;
};
SwAlignment sw_align(const std::string& a, const std::string& b, const SwScheme& s);
int sw_distance(const std::string& a, const std::string& b, const SwScheme& s);
Matrix pairwise_self(const std::vector<std::string>& ids, const std::vector<std::string>& seqs,
                     const SwScheme& s);
Matrix pairwise_cross(const std::vector<std::string>& qids, const std::vector<std::string>& q,
                      const std::vector<std::string>& rids, const std::vector<std::string>& r,
                      const SwScheme& s);

// DVS1 files (streaming ingest, dvs_stream.cpp)
struct DvsHeader {
    size_t rows = 0, cols = 0;
    bool symmetric = false;
};
DvsHeader read_dvs_header(const std::string& path);
// whole matrix, or (rows_only) rows [row_begin, row_end) as a row-shard handle
Matrix matrix_read_dvs(const std::string& path, bool rows_only, size_t row_begin, size_t row_end);

Matrix matrix_from_host_rows(const void* rows, size_t n, size_t row_begin, size_t row_end,
                             bool symmetric, DType dt);
Matrix matrix_euclidean_rows(const double* pts, size_t n, size_t dim, bool f32,
                             size_t row_begin, size_t row_end);
Matrix gram_sharded(const Matrix& d);
Embedding embed_sharded(const Matrix& g, size_t rank, SolverOptions opts);
Spectrum eigs_sharded(const Matrix& g, const SolverOptions& opts);
Matrix matrix_euclidean(const double* pts, size_t n, size_t dim, bool f32);
Matrix matrix_hamming(const char* reads, size_t count, size_t length);
Matrix matrix_hamming_rows(const char* reads, size_t count, size_t length, size_t row_begin,
                           size_t row_end);
void hamming_counts(const char* reads, size_t count, size_t length, uint32_t* out);

// test hook: the device-resident Omega panel of a solve, row-major n x w
void debug_omega_panel(uint64_t seed, size_t n, size_t w, double* out);

}  // namespace dsb
