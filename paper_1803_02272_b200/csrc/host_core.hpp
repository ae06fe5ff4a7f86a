// Host runtime of divscope-b200: error model, device context (stream,
// workspace arena, instrumentation), device-resident matrix handles.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace dsb {

// error codes: mirror of ref src/error.hpp:10-30 (and the C enum)
enum class errc {
    ok = 0,
    io_error,
    empty_input,
    invalid_character,
    duplicate_id,
    sample_too_large,
    empty_sequence,
    bad_format,
    truncated,
    not_symmetric,
    rank_too_large,
    zero_matrix,
    bad_gap,
    shape_mismatch,
    missing_label,
    join_error,
    bad_axis,
    invalid_argument,
    internal,
};

class Error : public std::runtime_error {
public:
    Error(errc code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    errc code() const noexcept { return code_; }

private:
    errc code_;
};

void cuda_check(cudaError_t e, const char* what);
#define DSB_CUDA(call) ::dsb::cuda_check((call), #call)

// Host array of doubles in pinned (page-locked) memory drawn from a recycling
// pool, so device->host result copies run at full PCIe / C2C speed without
// paying cudaMallocHost per call. Falls back to pageable memory when pinning
// is unavailable.
class PinnedVec {
public:
    PinnedVec() = default;
    explicit PinnedVec(size_t n) { resize(n); }
    PinnedVec(const PinnedVec&) = delete;
    PinnedVec& operator=(const PinnedVec&) = delete;
    PinnedVec(PinnedVec&& o) noexcept { swap(o); }
    PinnedVec& operator=(PinnedVec&& o) noexcept {
        swap(o);
        return *this;
    }
    ~PinnedVec() { release(); }
    void resize(size_t n);
    void assign(const std::vector<double>& v);
    double* data() { return p_; }
    const double* data() const { return p_; }
    size_t size() const { return n_; }
    bool empty() const { return n_ == 0; }
    double& operator[](size_t i) { return p_[i]; }
    double operator[](size_t i) const { return p_[i]; }

private:
    void release();
    void swap(PinnedVec& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        std::swap(cap_, o.cap_);
        std::swap(pinned_, o.pinned_);
    }
    double* p_ = nullptr;
    size_t n_ = 0, cap_ = 0;
    bool pinned_ = false;
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    explicit DevBuf(size_t b);
    ~DevBuf();
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct TimedPair {
    cudaEvent_t a, b;
    int kind;  // 0 = K1, 1 = K2
};

class Ctx {
public:
    static Ctx& get();
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    // a second stream (the sharded path's panel all-gather, overlapped with
    // the product over the locally-owned columns) and its two events
    cudaStream_t side = nullptr;
    cudaEvent_t side_ready = nullptr, side_done = nullptr;
    std::recursive_mutex mu;  // one solver at a time per process

    // grow-only workspace arena
    void* scratch(const std::string& slot, size_t bytes);
    // an evictable slot (the S-digit cache): nullptr instead of an error
    // when `bytes` plus `reserve` bytes are not available; a failed device
    // allocation elsewhere evicts these slots (evict_scratch) and retries
    // (reserve: max(1 GB, 2 % of the device))
    void* try_scratch(const std::string& slot, size_t bytes);
    bool evict_scratch();
    void* find_scratch(const std::string& slot) const;  // nullptr when absent
    // immutable device table named by its content key: uploaded on first
    // use (never inside a graph capture), then returned as is
    bool has_table(const std::string& name) const { return tables_.count(name) != 0; }
    const void* const_table(const std::string& name, const void* host, size_t bytes);

    // instrumentation
    bool timing = false;
    uint64_t launches_base = 0;
    uint64_t k2_launches = 0, k1_launches = 0, h2d = 0, d2h = 0;
    double k2_ms = 0.0, k1_ms = 0.0;
    // the first product pass of each solve (kind 3 below; also in k2_*):
    // the pass that stores the S-digit cache when it is on
    uint64_t k2_first_launches = 0;
    double k2_first_ms = 0.0;
    int last_evd_sweeps = 0, last_orth_shifted = 0, last_power_iters = 0;
    int last_product_kernel = 0;  // 0 fp64 DMMA, 1 int8 slice product
    int last_product_groups = 1;  // int8 column groups (reads of D per pass)
    int last_product_sdigits = 0;  // int8 S slices per element (7, or 3 for Hamming D)
    int last_product_sdig = 0;     // int8 S-digit cache: 1 stored by the first pass, 2 by K1
    // generation of the "i8_sdig" slot's contents: bumped whenever K1 or a
    // storing pass writes it and when it is evicted
    uint64_t sdig_gen = 0;
    int last_product_stream_cl = 0;  // CTAs per cluster of those streaming passes
    int last_product_pair = 0;     // int8: the CTA-pair kernel (one read of D for two groups)
    std::vector<TimedPair> pending;
    std::vector<cudaEvent_t> event_pool;
    void begin_timed(int kind, cudaEvent_t* a);
    void end_timed(int kind, cudaEvent_t a);
    // events created (when timing) for a caller that records them itself
    void make_events(cudaEvent_t* a, cudaEvent_t* b);
    void add_timed(int kind, cudaEvent_t a, cudaEvent_t b);
    void drain_timing();
    void set_timing(bool on);
    cudaEvent_t pooled_event();

    void h2d_copy(void* dst, const void* src, size_t bytes);
    void d2h_copy(void* dst, const void* src, size_t bytes);
    // named page-locked host buffer (grown on demand, never shrunk)
    void* pinned_scratch(const std::string& name, size_t bytes);
    void sync();

    bool encode_tmap(CUtensorMap* map, const void* base, DType dt, size_t rows, size_t cols,
                     size_t ld_elems, int box_rows);

    void set_device(int dev);

    // captured solve sequences (solver.cpp run): signature -> executable
    // graph, the kernel launches it contains, its product passes and, when
    // captured with timing on, the graph-owned event pair of each pass
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        uint64_t launches = 0;
        int products = 0;
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
    };
    std::map<uint64_t, GraphEntry> graphs;
    bool graphs_broken = false;  // a capture failed once: eager from then on
    void clear_graphs();

    // key of the device-resident Omega panel ("omega_panel" scratch slot)
    struct OmegaKey {
        bool ok = false;
        uint64_t seed = 0;
        size_t n = 0, w = 0, n_pad = 0;
    } omega_key;

private:
    Ctx();
    void init();
    bool inited_ = false;
    std::map<std::string, std::unique_ptr<DevBuf>> arena_;
    std::map<std::string, std::unique_ptr<DevBuf>> tables_;
    std::map<std::string, std::unique_ptr<PinnedVec>> pinned_arena_;
    void* encode_fn_ = nullptr;
};

// Device-resident dense matrix (row-major, leading dimension ld elements).
struct Store {
    size_t rows = 0, cols = 0, ld = 0;
    // row shard of a distributed matrix (multi-GPU): this store holds rows
    // [row_begin, row_begin + rows) of an n_global x cols matrix
    bool sharded = false;
    size_t n_global = 0, row_begin = 0;
    size_t order() const { return sharded ? n_global : rows; }
    bool square() const { return sharded ? n_global == cols : rows == cols; }
    bool symmetric = false;
    DType dt = DType::F64;
    std::shared_ptr<DevBuf> buf;
    // > 0: every value is fl(h / hamming_len) for an integer 0 <= h <=
    // hamming_len (the Hamming builder, K7); the int8 product then slices the
    // exact S = h^2 / L^2 into three bytes instead of seven
    int hamming_len = 0;
    // cached TMA descriptor for the K2 streaming read
    bool tmap_ok = false;
    CUtensorMap tmap128{}, tmap256{};  // box heights of the two K2 tile shapes
    bool tmap64_ok = false;
    CUtensorMap tmap64{};              // K1 tile-pair boxes
    const CUtensorMap* tmap_for(int bm) const { return bm == 256 ? &tmap256 : &tmap128; }
    // cached K1 results when used as an explicit symmetric matrix
    bool stats_ok = false;
    double stats[S_COUNT] = {};
    std::shared_ptr<DevBuf> stats_dev;
    std::mutex mu;
};

// Lazy gram: the distance store plus the centering terms of
// gram_from_distances (ref mds.cpp:29-41). G itself is never formed.
struct GramInfo {
    size_t n = 0;
    std::shared_ptr<DevBuf> row_mean;     // [n]
    std::shared_ptr<DevBuf> row_exp;      // [n] int, K1 (unsharded grams only; else null)
    std::vector<double> row_mean_h;       // host copy (for _get / _write)
    std::shared_ptr<DevBuf> scalars;      // [S_COUNT]
    double sc[S_COUNT] = {};
    // S-digit cache written by this gram's K1 pass: its generation (matches
    // Ctx::sdig_gen while the "i8_sdig" slot still holds it; 0 = none), the
    // digits per element (7 or 3) and, for 7, the bound row exponents the
    // digits are scaled by
    uint64_t sdig_gen = 0;
    int sdig_sd = 0;
    std::shared_ptr<DevBuf> row_eb;
    std::mutex mu;
};


size_t round_up(size_t x, size_t m);
std::shared_ptr<Store> make_store(size_t rows, size_t cols, bool symmetric, DType dt);
void upload_rows(Store& s, const void* host, size_t host_ld_elems);

// reference RNG conventions (ref src/rng.hpp:16-48)
double uniform_open_closed(std::mt19937_64& eng);
double uniform_closed_open(std::mt19937_64& eng);
uint64_t bounded_uint64(std::mt19937_64& eng, uint64_t bound);
void fill_gaussian(std::mt19937_64& eng, double* out, size_t n);

// DVS1 container (ref src/distmat.cpp:132-222)
void write_dvs(const std::string& path, size_t rows, size_t cols, bool symmetric,
               const double* values);
std::vector<double> read_dvs(const std::string& path, size_t& rows, size_t& cols,
                             bool& symmetric);

std::string format_double(double v);

}  // namespace dsb
