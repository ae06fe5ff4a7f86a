// Host runtime of divscope-b200 (see host_core.hpp).
#include "host_core.hpp"

#include <cudaTypedefs.h>

#include <atomic>
#include <charconv>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <fstream>
#include <map>
#include <mutex>

namespace dsb {

namespace {
std::atomic<uint64_t> g_launches{0};
}

namespace {
// kernel attributes are per device: remembered per (device, kernel)
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, size_t> g_attr_set;
std::atomic<long long> g_live_bufs{0};
int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
}  // namespace

void allow_dyn_smem(const void* kernel) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& set = g_attr_set[{current_device(), kernel}];
    if (set == ~size_t(0)) return;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kernel);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(227 * 1024 - fa.sharedSizeBytes));
    set = ~size_t(0);
}

void ensure_dyn_smem(const void* kernel, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& set = g_attr_set[{current_device(), kernel}];
    if (set >= bytes) return;
    DSB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
    set = bytes;
}

void count_launch(int k) { g_launches.fetch_add(static_cast<uint64_t>(k)); }
uint64_t kernel_launch_count() { return g_launches.load(); }

void record_timing_event(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else
        cudaEventRecord(e, st);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(errc::internal, std::string("CUDA error: ") + cudaGetErrorString(e) + " (" +
                                        what + ")");
}

// Device buffers come from the stream-ordered pool on the library stream
// (release threshold unlimited, see Ctx::init): a matrix handle created and
// freed per call (the e2e path) reuses its blocks instead of paying a
// synchronizing cudaMalloc/cudaFree of gigabytes every time.
DevBuf::DevBuf(size_t b) : bytes(b) {
    if (b == 0) return;
    cudaError_t e = cudaMallocAsync(&p, b, Ctx::get().stream);
    if (e != cudaSuccess) {
        // the evictable workspace (S-digit cache) yields to data and other
        // workspace: drop it and try once more
        cudaGetLastError();
        if (Ctx::get().evict_scratch()) e = cudaMallocAsync(&p, b, Ctx::get().stream);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        throw Error(errc::internal, "device out of memory allocating " + std::to_string(b) +
                                        " bytes: " + cudaGetErrorString(e));
    }
    g_live_bufs.fetch_add(1);
}

DevBuf::~DevBuf() {
    if (p) {
        cudaFreeAsync(p, Ctx::get().stream);
        g_live_bufs.fetch_sub(1);
    }
}

Ctx::Ctx() = default;

Ctx& Ctx::get() {
    static Ctx* c = new Ctx();  // never destroyed: avoids teardown-order issues with the driver
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (!c->inited_) c->init();
    return *c;
}

void Ctx::init() {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw Error(errc::internal,
                    "no usable CUDA device (divscope-b200 has no CPU fallback): " +
                        std::string(cudaGetErrorString(e)));
    int dev = 0;
    DSB_CUDA(cudaGetDevice(&dev));
    device = dev;
    DSB_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    DSB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        throw Error(errc::internal, std::string("divscope-b200 needs an sm_100 device, found ") +
                                        prop.name);
    sms = prop.multiProcessorCount;
    DSB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    DSB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    DSB_CUDA(cudaEventCreateWithFlags(&side_ready, cudaEventDisableTiming));
    DSB_CUDA(cudaEventCreateWithFlags(&side_done, cudaEventDisableTiming));
    {
        cudaMemPool_t pool;
        DSB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = ~0ull;
        DSB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    DSB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
        throw Error(errc::internal, "cuTensorMapEncodeTiled unavailable");
    encode_fn_ = fn;
    inited_ = true;
}

// One device per process (the multi-GPU path is one process per GPU). A
// switch is allowed only while no device memory is alive: the workspace, the
// resident Omega panel, pooled events and the stream all belong to the old
// device and are dropped here; kernel attributes are tracked per device.
void Ctx::set_device(int dev) {
    std::lock_guard<std::recursive_mutex> lk(mu);
    if (inited_ && dev == device) return;
    if (inited_) {
        DSB_CUDA(cudaStreamSynchronize(stream));
        clear_graphs();  // they address the arena
        arena_.clear();
        tables_.clear();
        omega_key = OmegaKey{};  // its panel lived in the arena
        if (g_live_bufs.load() != 0)
            throw Error(errc::invalid_argument,
                        "cannot change device while handles hold memory on device " +
                            std::to_string(device) + " (free them first)");
        for (cudaEvent_t e : event_pool) cudaEventDestroy(e);
        event_pool.clear();
        for (auto& t : pending) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        pending.clear();
        cudaStreamSynchronize(side);
        cudaEventDestroy(side_ready);
        cudaEventDestroy(side_done);
        cudaStreamDestroy(side);
        side = nullptr;
        cudaStreamDestroy(stream);
        stream = nullptr;
        inited_ = false;
    }
    DSB_CUDA(cudaSetDevice(dev));
    init();
}

const void* Ctx::const_table(const std::string& name, const void* host, size_t bytes) {
    auto it = tables_.find(name);
    if (it != tables_.end()) return it->second->p;
    if (tables_.size() >= 256) {
        // many distinct shapes: start over (graphs may address the tables)
        DSB_CUDA(cudaStreamSynchronize(stream));
        clear_graphs();
        tables_.clear();
    }
    auto buf = std::make_unique<DevBuf>(std::max<size_t>(bytes, 256));
    DSB_CUDA(cudaMemcpyAsync(buf->p, host, bytes, cudaMemcpyHostToDevice, stream));
    DSB_CUDA(cudaStreamSynchronize(stream));
    const void* p = buf->p;
    tables_[name] = std::move(buf);
    return p;
}

void Ctx::clear_graphs() {
    for (auto& kv : graphs) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        for (auto& e : kv.second.timed) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
    }
    graphs.clear();
}

void* Ctx::scratch(const std::string& slot, size_t bytes) {
    auto& b = arena_[slot];
    if (!b || b->bytes < bytes) {
        if (b) {
            DSB_CUDA(cudaStreamSynchronize(stream));
            b.reset();
        }
        b = std::make_unique<DevBuf>(std::max<size_t>(bytes, 256));
    }
    return b->p;
}

namespace {
bool evictable_slot(const std::string& slot) { return slot == "i8_sdig"; }
}  // namespace

void* Ctx::try_scratch(const std::string& slot, size_t bytes) {
    auto it = arena_.find(slot);
    if (it != arena_.end() && it->second && it->second->bytes >= bytes) return it->second->p;
    size_t fr = 0, tot = 0;
    DSB_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t reserve = std::max<size_t>(size_t(1) << 30, tot / 50);
    if (it != arena_.end()) {
        DSB_CUDA(cudaStreamSynchronize(stream));
        arena_.erase(it);
    }
    // probe for the slot plus the reserve, then keep only the slot (the
    // stream-ordered pool hands the probe's block back)
    void* probe = nullptr;
    if (cudaMallocAsync(&probe, bytes + reserve, stream) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    cudaFreeAsync(probe, stream);
    return scratch(slot, bytes);
}

void* Ctx::find_scratch(const std::string& slot) const {
    auto it = arena_.find(slot);
    return (it != arena_.end() && it->second) ? it->second->p : nullptr;
}

bool Ctx::evict_scratch() {
    bool any = false;
    for (auto it = arena_.begin(); it != arena_.end();) {
        if (evictable_slot(it->first)) {
            if (!any) DSB_CUDA(cudaStreamSynchronize(stream));
            clear_graphs();  // they address the slot
            ++sdig_gen;      // a gram's K1 digits are gone with it
            it = arena_.erase(it);
            any = true;
        } else {
            ++it;
        }
    }
    if (any) DSB_CUDA(cudaStreamSynchronize(stream));
    return any;
}

// debug / tests: what a failed device allocation does first — drop the
// evictable workspace (the S-digit cache) and the graphs that address it;
// returns 1 when something was evicted
extern "C" int divscope_debug_evict_workspace(void) {
    try {
        Ctx& c = Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        return c.evict_scratch() ? 1 : 0;
    } catch (...) {
        return -1;
    }
}

// debug: copy the first `bytes` of the S-digit cache slot to host memory
extern "C" int divscope_debug_sdig_read(void* host, size_t bytes) {
    try {
        Ctx& c = Ctx::get();
        void* p = c.find_scratch("i8_sdig");
        if (!p) return -1;
        DSB_CUDA(cudaStreamSynchronize(c.stream));
        DSB_CUDA(cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost));
        return 0;
    } catch (...) {
        return -2;
    }
}

void* Ctx::pinned_scratch(const std::string& name, size_t bytes) {
    auto& b = pinned_arena_[name];
    const size_t elems = (bytes + sizeof(double) - 1) / sizeof(double);
    if (!b || b->size() < elems) {
        if (b) DSB_CUDA(cudaStreamSynchronize(stream));  // an async copy may still target it
        b = std::make_unique<PinnedVec>(elems);
    }
    return b->data();
}

cudaEvent_t Ctx::pooled_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    DSB_CUDA(cudaEventCreate(&e));
    return e;
}

void Ctx::set_timing(bool on) {
    timing = on;
    // events come from a pool filled here, so a timed region creates none
    while (on && event_pool.size() < 1024) {
        cudaEvent_t e;
        DSB_CUDA(cudaEventCreate(&e));
        event_pool.push_back(e);
    }
}

void Ctx::begin_timed(int kind, cudaEvent_t* a) {
    (void)kind;
    *a = nullptr;
    if (!timing) return;
    *a = pooled_event();
    DSB_CUDA(cudaEventRecord(*a, stream));
}

void Ctx::end_timed(int kind, cudaEvent_t a) {
    if (kind == 1) ++k2_launches;
    else ++k1_launches;
    if (!timing || !a) return;
    cudaEvent_t b = pooled_event();
    DSB_CUDA(cudaEventRecord(b, stream));
    pending.push_back({a, b, kind});
}

void Ctx::make_events(cudaEvent_t* a, cudaEvent_t* b) {
    *a = *b = nullptr;
    if (!timing) return;
    *a = pooled_event();
    *b = pooled_event();
}

void Ctx::add_timed(int kind, cudaEvent_t a, cudaEvent_t b) {
    if (kind == 1 || kind == 3) ++k2_launches;
    else ++k1_launches;
    if (kind == 3) ++k2_first_launches;
    if (a && b) pending.push_back({a, b, kind});
}

void Ctx::drain_timing() {
    if (pending.empty()) return;
    DSB_CUDA(cudaStreamSynchronize(stream));
    for (auto& t : pending) {
        float ms = 0.0f;
        DSB_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
        (t.kind == 1 || t.kind == 3 ? k2_ms : k1_ms) += ms;
        if (t.kind == 3) k2_first_ms += ms;
        event_pool.push_back(t.a);
        event_pool.push_back(t.b);
    }
    pending.clear();
}

void Ctx::h2d_copy(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    DSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
    h2d += bytes;
}

void Ctx::d2h_copy(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    DSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
    DSB_CUDA(cudaStreamSynchronize(stream));
    d2h += bytes;
}

void Ctx::sync() {
    DSB_CUDA(cudaStreamSynchronize(stream));
    DSB_CUDA(cudaGetLastError());
}

bool Ctx::encode_tmap(CUtensorMap* map, const void* base, DType dt, size_t rows, size_t cols,
                      size_t ld_elems, int box_rows) {
    auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(encode_fn_);
    const size_t esz = dt == DType::F64 ? 8 : 4;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems * esz)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r =
        fn(map, dt == DType::F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
           2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }

namespace {
std::mutex g_pool_mu;
std::multimap<size_t, void*> g_pool;  // capacity (bytes) -> free pinned block
size_t g_pool_bytes = 0;
constexpr size_t kPoolCap = size_t(4) << 30;
}  // namespace

void PinnedVec::resize(size_t n) {
    if (n <= cap_) {
        n_ = n;
        return;
    }
    release();
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(double);
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        auto it = g_pool.lower_bound(bytes);
        if (it != g_pool.end() && it->first <= 2 * bytes) {
            p_ = static_cast<double*>(it->second);
            cap_ = it->first / sizeof(double);
            g_pool_bytes -= it->first;
            g_pool.erase(it);
            pinned_ = true;
            n_ = n;
            return;
        }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) == cudaSuccess) {
        pinned_ = true;
    } else {
        cudaGetLastError();
        p = std::malloc(bytes);
        if (!p) throw std::bad_alloc();
        pinned_ = false;
    }
    p_ = static_cast<double*>(p);
    cap_ = bytes / sizeof(double);
    n_ = n;
}

void PinnedVec::assign(const std::vector<double>& v) {
    resize(v.size());
    if (!v.empty()) std::memcpy(p_, v.data(), v.size() * sizeof(double));
}

void PinnedVec::release() {
    if (!p_) return;
    if (pinned_) {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        const size_t bytes = cap_ * sizeof(double);
        if (g_pool_bytes + bytes <= kPoolCap) {
            g_pool.emplace(bytes, p_);
            g_pool_bytes += bytes;
        } else {
            cudaFreeHost(p_);
        }
    } else {
        std::free(p_);
    }
    p_ = nullptr;
    n_ = cap_ = 0;
}

std::shared_ptr<Store> make_store(size_t rows, size_t cols, bool symmetric, DType dt) {
    auto s = std::make_shared<Store>();
    s->rows = rows;
    s->cols = cols;
    s->symmetric = symmetric;
    s->dt = dt;
    // TMA needs 16-byte row pitch; keep rows 256-byte aligned
    s->ld = round_up(std::max<size_t>(cols, 1), dt == DType::F64 ? 32 : 64);
    const size_t esz = dt == DType::F64 ? 8 : 4;
    s->buf = std::make_shared<DevBuf>(std::max<size_t>(rows, 1) * s->ld * esz);
    return s;
}

void upload_rows(Store& s, const void* host, size_t host_ld_elems) {
    Ctx& c = Ctx::get();
    const size_t esz = s.dt == DType::F64 ? 8 : 4;
    if (s.rows == 0 || s.cols == 0) return;
    // Large uploads are split into row chunks alternated over the library
    // stream and a side stream (two DMA engines in flight), then joined.
    const size_t bytes = s.rows * s.cols * esz;
    const size_t nchunk = bytes >= (size_t(64) << 20) ? 8 : 1;
    if (nchunk == 1) {
        DSB_CUDA(cudaMemcpy2DAsync(s.buf->p, s.ld * esz, host, host_ld_elems * esz, s.cols * esz,
                                   s.rows, cudaMemcpyHostToDevice, c.stream));
    } else {
        static cudaStream_t side = nullptr;
        static cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
        if (!side) {
            DSB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
            DSB_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
            DSB_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        }
        DSB_CUDA(cudaEventRecord(ev_fork, c.stream));
        DSB_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
        for (size_t k = 0; k < nchunk; ++k) {
            const size_t r0 = s.rows * k / nchunk, r1 = s.rows * (k + 1) / nchunk;
            if (r1 == r0) continue;
            cudaStream_t st = (k & 1) ? side : c.stream;
            DSB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(s.buf->p) + r0 * s.ld * esz, s.ld * esz,
                                       static_cast<const char*>(host) + r0 * host_ld_elems * esz,
                                       host_ld_elems * esz, s.cols * esz, r1 - r0,
                                       cudaMemcpyHostToDevice, st));
        }
        DSB_CUDA(cudaEventRecord(ev_join, side));
        DSB_CUDA(cudaStreamWaitEvent(c.stream, ev_join, 0));
    }
    c.h2d += bytes;
    if (s.ld > s.cols)  // zero the pitch padding so full-row reads stay clean
        DSB_CUDA(cudaMemset2DAsync(static_cast<char*>(s.buf->p) + s.cols * esz, s.ld * esz, 0,
                                   (s.ld - s.cols) * esz, s.rows, c.stream));
}

// ---- RNG: restatement of ref src/rng.hpp:16-48 ------------------------------
double uniform_open_closed(std::mt19937_64& eng) {
    return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53;
}
double uniform_closed_open(std::mt19937_64& eng) {
    return static_cast<double>(eng() >> 11) * 0x1.0p-53;
}
uint64_t bounded_uint64(std::mt19937_64& eng, uint64_t bound) {
    const uint64_t threshold = -bound % bound;
    for (;;) {
        const uint64_t x = eng();
        if (x >= threshold) return x % bound;
    }
}
void fill_gaussian(std::mt19937_64& eng, double* out, size_t n) {
    const double two_pi = 6.283185307179586476925286766559;
    size_t i = 0;
    while (i < n) {
        const double u1 = uniform_open_closed(eng);
        const double u2 = uniform_closed_open(eng);
        const double radius = std::sqrt(-2.0 * std::log(u1));
        out[i++] = radius * std::cos(two_pi * u2);
        if (i < n) out[i++] = radius * std::sin(two_pi * u2);
    }
}

// ---- DVS1 (ref src/distmat.cpp:132-222; format ref distmat.hpp:42-44) -----
namespace {
constexpr char kMagic[4] = {'D', 'V', 'S', '1'};
void put_le(std::string& b, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) b.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}
uint64_t get_le(const unsigned char* p, int bytes) {
    uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}
}  // namespace

void write_dvs(const std::string& path, size_t rows, size_t cols, bool symmetric,
               const double* values) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error(errc::io_error, "cannot open " + path + " for writing");
    std::string header(kMagic, 4);
    put_le(header, 1, 4);
    put_le(header, rows, 8);
    put_le(header, cols, 8);
    put_le(header, symmetric ? 1u : 0u, 8);
    out.write(header.data(), static_cast<std::streamsize>(header.size()));
    // x86-64 is little-endian: the payload is the raw IEEE bytes
    static_assert(sizeof(double) == 8, "");
    out.write(reinterpret_cast<const char*>(values),
              static_cast<std::streamsize>(rows * cols * sizeof(double)));
    out.flush();
    if (!out) throw Error(errc::io_error, "write failed for " + path);
}

std::vector<double> read_dvs(const std::string& path, size_t& rows, size_t& cols,
                             bool& symmetric) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(errc::io_error, "cannot open " + path);
    unsigned char header[32];
    in.read(reinterpret_cast<char*>(header), 32);
    if (in.gcount() != 32) throw Error(errc::truncated, path + ": header truncated");
    if (std::memcmp(header, kMagic, 4) != 0) throw Error(errc::bad_format, path + ": bad magic");
    const uint64_t version = get_le(header + 4, 4);
    if (version != 1)
        throw Error(errc::bad_format, path + ": unsupported version " + std::to_string(version));
    rows = get_le(header + 8, 8);
    cols = get_le(header + 16, 8);
    symmetric = (get_le(header + 24, 8) & 1) != 0;
    if (symmetric && rows != cols)
        throw Error(errc::bad_format, path + ": symmetric flag on non-square matrix");
    const uint64_t count = rows * cols;
    std::vector<double> v(count);
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(count * 8));
    if (static_cast<uint64_t>(in.gcount()) != count * 8)
        throw Error(errc::truncated, path + ": payload truncated");
    return v;
}

// ref src/textio.hpp:11-16 (shortest round-trip form)
std::string format_double(double v) {
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

}  // namespace dsb
