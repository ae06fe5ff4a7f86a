// divscope CPU oracle — TEST INFRASTRUCTURE ONLY.
//
// A CPU restatement of the reference's randomized classical-MDS path
// (/root/reference/proj/src/{mds,rsvd,rng,parallel}.hpp/.cpp), used as the
// parity checker for the B200 product library and as the "port" CPU baseline.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load it. The product (paper_1803_02272_b200/) never links or calls it.
//
// Parity pinning: the restatement is checked against oracle/_ref (the
// reference's own sources compiled against oracle/eigen_shim) through the
// committed fixtures in tests/golden/ (tests/golden/make_golden.py).
//
// Every function cites the reference lines it follows. Loop orders and
// floating-point expressions are kept identical to the reference so that
// gram, products and Omega are bit-identical; the QR and the small
// symmetric eigensolver (Eigen in the reference) are restated as Householder
// QR and cyclic Jacobi.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <atomic>
#include <string_view>
#include <vector>

namespace {

// error codes: src/error.hpp:10-30 (order mirrored)
enum Errc : int {
    OK = 0,
    EMPTY_INPUT = 2,
    EMPTY_SEQUENCE = 6,
    NOT_SYMMETRIC = 9,
    RANK_TOO_LARGE = 10,
    ZERO_MATRIX = 11,
    SHAPE_MISMATCH = 13,
    INVALID_ARGUMENT = 17,
    INTERNAL = 18,
};

// src/parallel.hpp:17-46: chunk w covers [total*w/W, total*(w+1)/W)
template <typename Fn>
void chunks(std::size_t total, unsigned threads, Fn&& fn) {
    if (threads == 0) threads = 1;
    const std::size_t workers = std::min<std::size_t>(threads, total == 0 ? 1 : total);
    if (workers <= 1) {
        fn(std::size_t{0}, total);
        return;
    }
    std::vector<std::thread> pool;
    for (std::size_t w = 0; w < workers; ++w) {
        const std::size_t b = total * w / workers, e = total * (w + 1) / workers;
        pool.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
}

// src/rng.hpp:26-33
inline double u_open_closed(std::mt19937_64& eng) {
    return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53;
}
inline double u_closed_open(std::mt19937_64& eng) {
    return static_cast<double>(eng() >> 11) * 0x1.0p-53;
}
// src/rng.hpp:16-22
inline std::uint64_t bounded(std::mt19937_64& eng, std::uint64_t bound) {
    const std::uint64_t threshold = -bound % bound;
    for (;;) {
        const std::uint64_t x = eng();
        if (x >= threshold) return x % bound;
    }
}
// src/rng.hpp:38-48
void gaussian(std::mt19937_64& eng, double* out, std::size_t n) {
    const double two_pi = 6.283185307179586476925286766559;
    std::size_t i = 0;
    while (i < n) {
        const double u1 = u_open_closed(eng);
        const double u2 = u_closed_open(eng);
        const double radius = std::sqrt(-2.0 * std::log(u1));
        out[i++] = radius * std::cos(two_pi * u2);
        if (i < n) out[i++] = radius * std::sin(two_pi * u2);
    }
}

// ---- Gram operator -------------------------------------------------------
// The reference materializes G (mds.cpp:43-58); the oracle can either
// materialize it the same way or evaluate the identical per-entry expression
// on the fly (same operands, same operation order => same bits), which lets
// it check n where n^2 doubles of G would not fit next to D.
struct GramOp {
    const double* g = nullptr;   // explicit symmetric matrix (n x n), or
    const double* d = nullptr;   // distance matrix + centering terms
    const double* row_mean = nullptr;
    double grand = 0.0;
    std::size_t n = 0;
    // d verified BIT-symmetric (exact_symmetric below): the mirrored entry
    // d_ji is then read from row i (same bits, cache-friendly); the
    // expression and its operand order stay the reference's
    bool row_sym = false;

    // mds.cpp:50-51 for i <= j; lower triangle mirrored (mds.cpp:57-58)
    double at(std::size_t i, std::size_t j) const {
        if (g) return g[i * n + j];
        if (i <= j) {
            const double dij = d[i * n + j];
            return -0.5 * (dij * dij - row_mean[i] - row_mean[j] + grand);
        }
        const double dji = row_sym ? d[i * n + j] : d[j * n + i];
        return -0.5 * (dji * dji - row_mean[j] - row_mean[i] + grand);
    }
};

// true iff d_ij and d_ji have identical bits for every pair (64 x 64 tiles,
// threaded over tile rows)
bool exact_symmetric(const double* d, std::size_t n, unsigned threads) {
    constexpr std::size_t T = 64;
    const std::size_t nt = (n + T - 1) / T;
    std::vector<char> bad(nt, 0);
    chunks(nt, threads, [&](std::size_t b0, std::size_t b1) {
        for (std::size_t bi = b0; bi < b1; ++bi)
            for (std::size_t bj = bi; bj < nt && !bad[bi]; ++bj)
                for (std::size_t i = bi * T; i < std::min(n, bi * T + T); ++i)
                    for (std::size_t j = std::max(i + 1, bj * T); j < std::min(n, bj * T + T); ++j)
                        if (std::memcmp(d + i * n + j, d + j * n + i, sizeof(double)) != 0)
                            bad[bi] = 1;
    });
    for (char b : bad)
        if (b) return false;
    return true;
}

// src/rsvd.cpp:18-36. Every output row is the reference's loop — zero-fill,
// then j ascending, skipping g_ij == 0, out_i[c] += g_ij * m_j[c] — so the
// result is bit-identical; rows are processed in blocks of kIB against
// column blocks of kJB only so that a block of m stays in cache while the
// rows of the block consume it (the per-row order of additions is unchanged).
void multiply(const GramOp& op, const double* m, std::size_t k, double* out, unsigned threads) {
    constexpr std::size_t kIB = 32, kJB = 512;
    const std::size_t n = op.n;
    chunks(n, threads, [&](std::size_t begin, std::size_t end) {
        std::vector<double> gblk(kIB * kJB);
        for (std::size_t i0 = begin; i0 < end; i0 += kIB) {
            const std::size_t i1 = std::min(end, i0 + kIB);
            for (std::size_t i = i0; i < i1; ++i) std::fill(out + i * k, out + i * k + k, 0.0);
            for (std::size_t j0 = 0; j0 < n; j0 += kJB) {
                const std::size_t j1 = std::min(n, j0 + kJB);
                for (std::size_t i = i0; i < i1; ++i) {
                    double* out_row = out + i * k;
                    const double* row;
                    if (op.g) {
                        row = op.g + i * n + j0;
                    } else {
                        double* gr = gblk.data() + (i - i0) * kJB;
                        for (std::size_t j = j0; j < j1; ++j) gr[j - j0] = op.at(i, j);
                        row = gr;
                    }
                    for (std::size_t j = j0; j < j1; ++j) {
                        const double gij = row[j - j0];
                        if (gij == 0.0) continue;
                        const double* mrow = m + j * k;
                        for (std::size_t c = 0; c < k; ++c) out_row[c] += gij * mrow[c];
                    }
                }
            }
        }
    });
}

// src/rsvd.cpp:64-79
double frobenius_sq(const GramOp& op, unsigned threads) {
    const std::size_t n = op.n;
    std::vector<double> row_sq(n, 0.0);
    chunks(n, threads, [&](std::size_t begin, std::size_t end) {
        for (std::size_t i = begin; i < end; ++i) {
            double s = 0.0;
            for (std::size_t j = 0; j < n; ++j) {
                const double v = op.at(i, j);
                s += v * v;
            }
            row_sq[i] = s;
        }
    });
    double total = 0.0;
    for (double s : row_sq) total += s;
    return total;
}

// Householder thin QR (substitute for Eigen::HouseholderQR, rsvd.cpp:38-44):
// y (n x k row-major) -> q (n x k) with orthonormal columns.
void thin_orthonormal(const double* y, std::size_t n, std::size_t k, double* q) {
    std::vector<double> r(y, y + n * k);
    std::vector<std::vector<double>> vs;
    std::vector<double> taus;
    for (std::size_t h = 0; h < k; ++h) {
        const double alpha = r[h * k + h];
        double sigma = 0.0;
        for (std::size_t i = h + 1; i < n; ++i) sigma += r[i * k + h] * r[i * k + h];
        std::vector<double> v(n - h, 0.0);
        v[0] = 1.0;
        double tau = 0.0;
        if (sigma != 0.0) {
            const double norm = std::sqrt(alpha * alpha + sigma);
            const double beta = alpha >= 0.0 ? -norm : norm;
            tau = (beta - alpha) / beta;
            const double scale = 1.0 / (alpha - beta);
            for (std::size_t i = h + 1; i < n; ++i) v[i - h] = r[i * k + h] * scale;
            for (std::size_t c = h; c < k; ++c) {
                double dot = 0.0;
                for (std::size_t i = h; i < n; ++i) dot += v[i - h] * r[i * k + c];
                dot *= tau;
                for (std::size_t i = h; i < n; ++i) r[i * k + c] -= dot * v[i - h];
            }
        }
        vs.push_back(std::move(v));
        taus.push_back(tau);
    }
    std::fill(q, q + n * k, 0.0);
    for (std::size_t c = 0; c < k; ++c) q[c * k + c] = 1.0;
    for (std::size_t hh = k; hh-- > 0;) {
        const auto& v = vs[hh];
        const double tau = taus[hh];
        if (tau == 0.0) continue;
        for (std::size_t c = 0; c < k; ++c) {
            double dot = 0.0;
            for (std::size_t i = hh; i < n; ++i) dot += v[i - hh] * q[i * k + c];
            dot *= tau;
            for (std::size_t i = hh; i < n; ++i) q[i * k + c] -= dot * v[i - hh];
        }
    }
}

// Cyclic Jacobi (substitute for Eigen::SelfAdjointEigenSolver,
// rsvd.cpp:112-116): vals ascending, vecs column c pairs with vals[c].
bool sym_evd(const double* a_in, std::size_t n, double* vals, double* vecs) {
    std::vector<double> a(a_in, a_in + n * n), v(n * n, 0.0);
    for (std::size_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
    bool ok = n == 0;
    for (int sweep = 0; sweep < 100 && !ok; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (std::size_t i = 0; i < n; ++i) {
            diag += a[i * n + i] * a[i * n + i];
            for (std::size_t j = i + 1; j < n; ++j) off += a[i * n + j] * a[i * n + j];
        }
        if (off == 0.0 || off <= 1e-34 * diag) {
            ok = true;
            break;
        }
        for (std::size_t p = 0; p + 1 < n; ++p)
            for (std::size_t q = p + 1; q < n; ++q) {
                const double apq = a[p * n + q];
                if (std::abs(apq) < 1e-300) continue;
                const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) /
                                 (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (std::size_t k = 0; k < n; ++k) {
                    const double akp = a[k * n + p], akq = a[k * n + q];
                    a[k * n + p] = c * akp - s * akq;
                    a[k * n + q] = s * akp + c * akq;
                }
                for (std::size_t k = 0; k < n; ++k) {
                    const double apk = a[p * n + k], aqk = a[q * n + k];
                    a[p * n + k] = c * apk - s * aqk;
                    a[q * n + k] = s * apk + c * aqk;
                }
                a[p * n + q] = a[q * n + p] = 0.0;
                for (std::size_t k = 0; k < n; ++k) {
                    const double vkp = v[k * n + p], vkq = v[k * n + q];
                    v[k * n + p] = c * vkp - s * vkq;
                    v[k * n + q] = s * vkp + c * vkq;
                }
            }
    }
    std::vector<std::size_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](std::size_t x, std::size_t y) { return a[x * n + x] < a[y * n + y]; });
    for (std::size_t c = 0; c < n; ++c) {
        vals[c] = a[order[c] * n + order[c]];
        for (std::size_t i = 0; i < n; ++i) vecs[i * n + c] = v[i * n + order[c]];
    }
    return ok;
}

// src/rsvd.cpp:46-60 (explicit matrices only; the lazy gram is mirrored)
int check_symmetric(const GramOp& op) {
    if (op.n == 0) return INVALID_ARGUMENT;
    if (!op.g) return OK;
    double maxabs = 0.0, maxasym = 0.0;
    for (std::size_t i = 0; i < op.n; ++i)
        for (std::size_t j = i; j < op.n; ++j) {
            const double a = op.g[i * op.n + j], b = op.g[j * op.n + i];
            maxabs = std::max(maxabs, std::abs(a));
            maxasym = std::max(maxasym, std::abs(a - b));
        }
    return maxasym > 1e-10 * std::max(1.0, maxabs) ? NOT_SYMMETRIC : OK;
}

struct Spectrum {
    std::vector<double> vals;
    std::vector<double> vecs;  // n x keep
    std::size_t keep = 0;
    double resid = 0.0;
};

// src/rsvd.cpp:81-100 + :102-145
int eigs(const GramOp& op, std::size_t rank, std::size_t p, std::size_t q, std::uint64_t seed,
         unsigned threads, Spectrum& out) {
    if (int e = check_symmetric(op)) return e;
    if (rank < 1) return INVALID_ARGUMENT;
    const std::size_t n = op.n, w = rank + p;
    if (w > n) return RANK_TOO_LARGE;
    std::vector<double> omega(n * w), y(n * w), qm(n * w);
    std::mt19937_64 eng(seed);
    gaussian(eng, omega.data(), n * w);
    multiply(op, omega.data(), w, y.data(), threads);
    thin_orthonormal(y.data(), n, w, qm.data());
    for (std::size_t t = 0; t < q; ++t) {
        multiply(op, qm.data(), w, y.data(), threads);
        thin_orthonormal(y.data(), n, w, qm.data());
        multiply(op, qm.data(), w, y.data(), threads);
        thin_orthonormal(y.data(), n, w, qm.data());
    }
    multiply(op, qm.data(), w, y.data(), threads);  // GQ
    std::vector<double> b(w * w, 0.0), bs(w * w);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t a = 0; a < w; ++a) {
            const double qa = qm[i * w + a];
            for (std::size_t c = 0; c < w; ++c) b[a * w + c] += qa * y[i * w + c];
        }
    for (std::size_t a = 0; a < w; ++a)
        for (std::size_t c = 0; c < w; ++c) bs[a * w + c] = 0.5 * (b[a * w + c] + b[c * w + a]);
    std::vector<double> vals(w), vecs(w * w);
    if (!sym_evd(bs.data(), w, vals.data(), vecs.data())) return INTERNAL;
    std::vector<std::size_t> order(w);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t c) {
        if (std::abs(vals[a]) != std::abs(vals[c])) return std::abs(vals[a]) > std::abs(vals[c]);
        return vals[a] > vals[c];
    });
    const std::size_t keep = std::min(rank, w);
    out.keep = keep;
    out.vals.assign(keep, 0.0);
    out.vecs.assign(n * keep, 0.0);
    for (std::size_t a = 0; a < keep; ++a) out.vals[a] = vals[order[a]];
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t a = 0; a < keep; ++a) {
            double s = 0.0;
            for (std::size_t c = 0; c < w; ++c) s += qm[i * w + c] * vecs[c * w + order[a]];
            out.vecs[i * keep + a] = s;
        }
    double sum_sq = 0.0;
    for (double lam : out.vals) sum_sq += lam * lam;
    out.resid = std::sqrt(std::max(0.0, frobenius_sq(op, threads) - sum_sq));
    return OK;
}

// src/mds.cpp:62-77
void sign_normalize(double* col, std::size_t n, std::size_t stride) {
    std::size_t best = 0;
    double best_abs = std::abs(col[0]);
    for (std::size_t i = 1; i < n; ++i) {
        const double a = std::abs(col[i * stride]);
        if (a > best_abs) {
            best_abs = a;
            best = i;
        }
    }
    if (col[best * stride] < 0.0)
        for (std::size_t i = 0; i < n; ++i) col[i * stride] = -col[i * stride];
}

}  // namespace

extern "C" {

// src/rng.hpp:38-48 driven by std::mt19937_64(seed) (rsvd.cpp:90-92)
void orc_fill_gaussian(std::uint64_t seed, double* out, std::size_t count) {
    std::mt19937_64 eng(seed);
    gaussian(eng, out, count);
}

// src/mds.cpp:14-41: validation, row means of d^2, grand mean.
// Returns an errc code. Also reports max|d| and the Frobenius norm of G via
// the exact definition when fro_out != NULL (rsvd.cpp:64-79 over the mirrored
// gram, evaluated on the fly).
int orc_gram_stats(const double* d, std::size_t rows, std::size_t cols, int sym,
                   unsigned threads, double* row_mean, double* grand_out) {
    if (rows != cols || !sym) return NOT_SYMMETRIC;
    const std::size_t n = rows;
    if (n == 0) return EMPTY_INPUT;
    // max |d| and the pairwise test of mds.cpp:21-27 (order-independent
    // decisions, so threaded and tiled; exact symmetry short-cuts the test)
    std::vector<double> part_max(std::max(threads, 1u), 0.0);
    {
        std::atomic<unsigned> slot{0};
        chunks(n, threads, [&](std::size_t b, std::size_t e) {
            double mx = 0.0;
            for (std::size_t k = b * n; k < e * n; ++k) mx = std::max(mx, std::abs(d[k]));
            part_max[slot.fetch_add(1)] = mx;
        });
    }
    double maxabs = 0.0;
    for (double v : part_max) maxabs = std::max(maxabs, v);
    if (!exact_symmetric(d, n, threads)) {
        const double tol = 1e-12 * std::max(1.0, maxabs);
        std::atomic<int> bad{0};
        chunks(n, threads, [&](std::size_t b, std::size_t e) {
            for (std::size_t i = b; i < e; ++i)
                for (std::size_t j = i + 1; j < n; ++j)
                    if (std::abs(d[i * n + j] - d[j * n + i]) > tol) bad = 1;
        });
        if (bad) return NOT_SYMMETRIC;
    }
    chunks(n, threads, [&](std::size_t begin, std::size_t end) {
        for (std::size_t i = begin; i < end; ++i) {
            const double* row = d + i * n;
            double s = 0.0;
            for (std::size_t j = 0; j < n; ++j) s += row[j] * row[j];
            row_mean[i] = s / static_cast<double>(n);
        }
    });
    double grand = 0.0;
    for (std::size_t i = 0; i < n; ++i) grand += row_mean[i];
    *grand_out = grand / static_cast<double>(n);
    return OK;
}

// src/mds.cpp:43-58: materialized, mirrored gram.
int orc_gram(const double* d, std::size_t rows, std::size_t cols, int sym, unsigned threads,
             double* g) {
    std::vector<double> rm(rows);
    double grand = 0.0;
    if (int e = orc_gram_stats(d, rows, cols, sym, threads, rm.data(), &grand)) return e;
    GramOp op{nullptr, d, rm.data(), grand, rows};
    const std::size_t n = rows;
    chunks(n, threads, [&](std::size_t begin, std::size_t end) {
        for (std::size_t i = begin; i < end; ++i)
            for (std::size_t j = 0; j < n; ++j) g[i * n + j] = op.at(i, j);
    });
    return OK;
}

// src/rsvd.cpp:18-36 over an explicit symmetric matrix
void orc_multiply_sym(const double* g, std::size_t n, const double* m, std::size_t k,
                      unsigned threads, double* out) {
    GramOp op{g, nullptr, nullptr, 0.0, n};
    multiply(op, m, k, out, threads);
}

// 2-bit code of A,C,G,T = 0,1,2,3; anything else -> -1.
static int base_code(char c) {
    switch (c) {
        case 'A': return 0;
        case 'C': return 1;
        case 'G': return 2;
        case 'T': return 3;
        default: return -1;
    }
}

// rows [row_begin, row_end) of the same pass (a bounded CPU-baseline sample:
// each output row is computed exactly as in the full pass)
void orc_multiply_gram_otf_rows(const double* d, std::size_t n, const double* row_mean,
                                double grand, const double* m, std::size_t k,
                                std::size_t row_begin, std::size_t row_end, unsigned threads,
                                double* out) {
    GramOp op{nullptr, d, row_mean, grand, n};
    op.row_sym = exact_symmetric(d, n, threads);
    const std::size_t rows = row_end - row_begin;
    chunks(rows, threads, [&](std::size_t b, std::size_t e) {
        std::vector<double> grow(n);
        for (std::size_t i = row_begin + b; i < row_begin + e; ++i) {
            double* out_row = out + (i - row_begin) * k;
            std::fill(out_row, out_row + k, 0.0);
            for (std::size_t j = 0; j < n; ++j) grow[j] = op.at(i, j);
            for (std::size_t j = 0; j < n; ++j) {
                const double gij = grow[j];
                if (gij == 0.0) continue;
                const double* mrow = m + j * k;
                for (std::size_t c = 0; c < k; ++c) out_row[c] += gij * mrow[c];
            }
        }
    });
}

// Hamming counts of 2-bit packed reads (the definition of orc_hamming_counts,
// evaluated 32 positions per 64-bit word pair: a position differs iff its
// two code bits differ in either plane), full n x n, threaded. Returns 3
// (INVALID_CHARACTER) on a non-ACGT byte.
int orc_hamming_matrix_mt(const char* reads, std::size_t count, std::size_t length,
                          unsigned threads, double* d_out) {
    const std::size_t words = (length + 63) / 64;
    std::vector<std::uint64_t> lo(count * words, 0), hi(count * words, 0);
    for (std::size_t i = 0; i < count; ++i)
        for (std::size_t t = 0; t < length; ++t) {
            const int c = base_code(reads[i * length + t]);
            if (c < 0) return 3;
            lo[i * words + t / 64] |= static_cast<std::uint64_t>(c & 1) << (t % 64);
            hi[i * words + t / 64] |= static_cast<std::uint64_t>(c >> 1) << (t % 64);
        }
    const double len = static_cast<double>(length);
    chunks(count, threads, [&](std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i)
            for (std::size_t j = 0; j < count; ++j) {
                std::uint64_t h = 0;
                for (std::size_t w = 0; w < words; ++w)
                    h += static_cast<std::uint64_t>(__builtin_popcountll(
                        (lo[i * words + w] ^ lo[j * words + w]) |
                        (hi[i * words + w] ^ hi[j * words + w])));
                d_out[i * count + j] = static_cast<double>(h) / len;
            }
    });
    return OK;
}

// rsvd.cpp:18-36 over the gram of D evaluated on the fly (bit-identical to
// multiply over orc_gram's output).
void orc_multiply_gram_otf(const double* d, std::size_t n, const double* row_mean, double grand,
                           const double* m, std::size_t k, unsigned threads, double* out) {
    GramOp op{nullptr, d, row_mean, grand, n};
    op.row_sym = exact_symmetric(d, n, threads);
    multiply(op, m, k, out, threads);
}

// src/rsvd.cpp:64-79
double orc_frobenius_sq(const double* g, std::size_t n, unsigned threads) {
    GramOp op{g, nullptr, nullptr, 0.0, n};
    return frobenius_sq(op, threads);
}

// Householder thin QR (rsvd.cpp:38-44 semantics)
void orc_thin_orthonormal(const double* y, std::size_t n, std::size_t k, double* q) {
    thin_orthonormal(y, n, k, q);
}

// dense symmetric EVD (ascending), for test-side dense references
int orc_sym_evd(const double* a, std::size_t n, double* vals, double* vecs) {
    return sym_evd(a, n, vals, vecs) ? OK : INTERNAL;
}

// src/rsvd.cpp:102-145. If d != NULL the operator is the gram of d (on the
// fly, row_mean/grand from orc_gram_stats); otherwise g is explicit.
int orc_eigs(const double* g, const double* d, const double* row_mean, double grand,
             std::size_t n, std::size_t rank, std::size_t p, std::size_t q, std::uint64_t seed,
             unsigned threads, double* vals_out, double* vecs_out, std::size_t* keep_out,
             double* resid_out) {
    GramOp op{g, d, row_mean, grand, n};
    if (d) op.row_sym = exact_symmetric(d, n, threads);
    Spectrum s;
    if (int e = eigs(op, rank, p, q, seed, threads, s)) return e;
    *keep_out = s.keep;
    std::copy(s.vals.begin(), s.vals.end(), vals_out);
    if (vecs_out) std::copy(s.vecs.begin(), s.vecs.end(), vecs_out);
    *resid_out = s.resid;
    return OK;
}

// src/mds.cpp:116-124 + embed_from_spectrum (mds.cpp:81-114). coords_out
// holds n*rank; returns r etc.
int orc_embed(const double* g, const double* d, const double* row_mean, double grand,
              std::size_t n, std::size_t rank, std::size_t p, std::size_t q, std::uint64_t seed,
              unsigned threads, double* coords_out, double* evals_out, std::size_t* r_out,
              double* mass_out, int* truncated_out, double* resid_out) {
    if (rank < 1 || rank > n) return RANK_TOO_LARGE;  // mds.cpp:118-119
    p = std::min(p, n - rank);                         // mds.cpp:121
    GramOp op{g, d, row_mean, grand, n};
    if (d) op.row_sym = exact_symmetric(d, n, threads);
    Spectrum s;
    if (int e = eigs(op, rank, p, q, seed, threads, s)) return e;
    double maxabs = 0.0;
    for (double lam : s.vals) maxabs = std::max(maxabs, std::abs(lam));
    const double eps = 1e-9 * maxabs;
    std::vector<std::size_t> keep;
    double mass = 0.0;
    for (std::size_t a = 0; a < s.vals.size(); ++a) {
        const double lam = s.vals[a];
        if (lam > eps && keep.size() < rank)
            keep.push_back(a);
        else if (lam < 0.0)
            mass += -lam;
    }
    const std::size_t r = keep.size();
    for (std::size_t c = 0; c < r; ++c) {
        const std::size_t a = keep[c];
        const double lam = s.vals[a];
        evals_out[c] = lam;
        for (std::size_t i = 0; i < n; ++i) coords_out[i * r + c] = s.vecs[i * s.keep + a];
        sign_normalize(coords_out + c, n, r);
        const double scale = std::sqrt(lam);
        for (std::size_t i = 0; i < n; ++i) coords_out[i * r + c] *= scale;
    }
    *r_out = r;
    *mass_out = mass;
    *truncated_out = r < rank ? 1 : 0;
    if (resid_out) *resid_out = s.resid;
    return OK;
}

// --- inputs without a reference implementation (C5 / Hamming, a14) -------


// h_ij = number of positions where reads i and j differ (plain character
// comparison: the definition, independent of any packing).
int orc_hamming_counts(const char* reads, std::size_t count, std::size_t length,
                       std::uint32_t* h_out) {
    for (std::size_t k = 0; k < count * length; ++k)
        if (base_code(reads[k]) < 0) return 3;  // INVALID_CHARACTER
    for (std::size_t i = 0; i < count; ++i)
        for (std::size_t j = 0; j < count; ++j) {
            std::uint32_t h = 0;
            for (std::size_t t = 0; t < length; ++t)
                h += reads[i * length + t] != reads[j * length + t] ? 1u : 0u;
            h_out[i * count + j] = h;
        }
    return OK;
}

// tests/testdata.cpp:165-184: exact, bit-symmetric Euclidean distances.
void orc_euclidean_matrix(const double* pts, std::size_t n, std::size_t dim, double* out) {
    std::fill(out, out + n * n, 0.0);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = i + 1; j < n; ++j) {
            double sq = 0.0;
            for (std::size_t c = 0; c < dim; ++c) {
                const double diff = pts[i * dim + c] - pts[j * dim + c];
                sq += diff * diff;
            }
            const double dist = std::sqrt(sq);
            out[i * n + j] = dist;
            out[j * n + i] = dist;
        }
}

// same, rows chunked over threads (parallel.hpp:17-46); each row's values do
// not depend on the chunking, so the output is identical
void orc_euclidean_matrix_mt(const double* pts, std::size_t n, std::size_t dim, unsigned threads,
                             double* out) {
    chunks(n, threads, [&](std::size_t begin, std::size_t end) {
        for (std::size_t i = begin; i < end; ++i)
            for (std::size_t j = 0; j < n; ++j) {
                if (i == j) {
                    out[i * n + j] = 0.0;
                    continue;
                }
                const std::size_t a = std::min(i, j), b = std::max(i, j);
                double sq = 0.0;
                for (std::size_t c = 0; c < dim; ++c) {
                    const double diff = pts[a * dim + c] - pts[b * dim + c];
                    sq += diff * diff;
                }
                out[i * n + j] = std::sqrt(sq);
            }
    });
}

// ---- BASELINE.json workload synthesis (test / reference-arm inputs) -------
// Restates the seeded generators of the configs so that bench.py's
// reference arm builds its inputs without loading the product library; a
// CPU test pins them bit-for-bit to divscope_synth_points / _reads. The RNG
// calls follow ref src/rng.hpp: fill_gaussian for normals,
// uniform_open_closed / uniform_closed_open for uniforms, bounded for
// categorical draws; DNA bases as ref tests/testdata.cpp:16-26.
//   config 1: 5 clusters in R^20, centers N(0, 10^2 I), equal weights
//   config 2: 20 clusters in R^50, centers N(0, 5^2 I), Dirichlet(1) weights
//   config 3: 10 centers N(0, 20^2 I) in R^100, each with 10 sub-centers
//             offset N(0, 3^2 I) (100 equal-weight clusters)
//   config 4: 100 clusters in R^64, centers N(0, 8^2 I), equal weights
// Order of draws: centers, sub-center offsets, weights (Dirichlet only),
// labels, then the unit within-cluster noise of all points.
int orc_synth_points(int config, std::size_t n, std::uint64_t seed, double* out,
                     std::size_t* dim_out) {
    std::size_t dim, top, sub = 0;
    double csd, ssd = 0.0;
    bool dir = false;
    switch (config) {
        case 1: dim = 20; top = 5; csd = 10.0; break;
        case 2: dim = 50; top = 20; csd = 5.0; dir = true; break;
        case 3: dim = 100; top = 10; csd = 20.0; sub = 10; ssd = 3.0; break;
        case 4: dim = 64; top = 100; csd = 8.0; break;
        default: return INVALID_ARGUMENT;
    }
    std::mt19937_64 eng(seed);
    std::vector<double> ctr(top * dim);
    gaussian(eng, ctr.data(), ctr.size());
    for (double& v : ctr) v *= csd;
    std::size_t nclu = top;
    if (sub) {
        nclu = top * sub;
        std::vector<double> off(nclu * dim);
        gaussian(eng, off.data(), off.size());
        for (std::size_t k = 0; k < nclu; ++k)
            for (std::size_t c = 0; c < dim; ++c)
                off[k * dim + c] = ctr[(k / sub) * dim + c] + ssd * off[k * dim + c];
        ctr.swap(off);
    }
    std::vector<std::size_t> lab(n);
    if (dir) {
        std::vector<double> e(nclu), cdf(nclu);
        double sum = 0.0;
        for (double& x : e) {
            x = -std::log(u_open_closed(eng));
            sum += x;
        }
        double run = 0.0;
        for (std::size_t k = 0; k < nclu; ++k) cdf[k] = (run += e[k] / sum);
        for (std::size_t i = 0; i < n; ++i) {
            const double u = u_closed_open(eng);
            std::size_t k = 0;
            while (k + 1 < nclu && !(u < cdf[k])) ++k;
            lab[i] = k;
        }
    } else {
        for (std::size_t i = 0; i < n; ++i) lab[i] = bounded(eng, nclu);
    }
    gaussian(eng, out, n * dim);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t c = 0; c < dim; ++c) out[i * dim + c] += ctr[lab[i] * dim + c];
    if (dim_out) *dim_out = dim;
    return OK;
}

// config 5 reads: `ancestors` uniform random sequences (a base per
// bounded(4) draw), each read copies a bounded(ancestors)-chosen ancestor and
// substitutes each base with probability sub_rate (uniform_closed_open <
// rate) by one of the three other bases, (b + 1 + bounded(3)) mod 4.
void orc_synth_reads(std::size_t count, std::size_t length, std::size_t ancestors,
                     double sub_rate, std::uint64_t seed, char* out) {
    const char acgt[4] = {'A', 'C', 'G', 'T'};
    std::mt19937_64 eng(seed);
    std::vector<unsigned char> anc(ancestors * length);
    for (auto& b : anc) b = static_cast<unsigned char>(bounded(eng, 4));
    for (std::size_t i = 0; i < count; ++i) {
        const std::size_t a = bounded(eng, ancestors);
        for (std::size_t t = 0; t < length; ++t) {
            std::size_t b = anc[a * length + t];
            if (u_closed_open(eng) < sub_rate) b = (b + 1 + bounded(eng, 3)) % 4;
            out[i * length + t] = acgt[b];
        }
    }
}

// sum_i sum_j of the explicit reconstruction error (mds.cpp:126-150)
double orc_reconstruction_error(const double* g, std::size_t n, const double* coords,
                                std::size_t r) {
    double total = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (std::size_t j = 0; j < n; ++j) {
            double dot = 0.0;
            for (std::size_t c = 0; c < r; ++c) dot += coords[i * r + c] * coords[j * r + c];
            const double diff = g[i * n + j] - dot;
            s += diff * diff;
        }
        total += s;
    }
    return std::sqrt(total);
}

// rsvd.cpp:147-178 (GEMV power iteration, seed 0x5eed)
int orc_stable_rank(const double* g, std::size_t n, unsigned threads, double* out) {
    GramOp op{g, nullptr, nullptr, 0.0, n};
    if (int e = check_symmetric(op)) return e;
    const double fro2 = frobenius_sq(op, threads);
    if (fro2 == 0.0) return ZERO_MATRIX;
    std::vector<double> v(n), w(n);
    std::mt19937_64 eng(0x5eedULL);
    auto normalize = [&](std::vector<double>& x) {
        double s = 0.0;
        for (double a : x) s += a * a;
        const double nrm = std::sqrt(s);
        for (double& a : x) a /= nrm;
    };
    gaussian(eng, v.data(), n);
    normalize(v);
    double sigma = 0.0;
    for (int it = 0; it < 20000; ++it) {
        multiply(op, v.data(), 1, w.data(), threads);
        double s = 0.0;
        for (double a : w) s += a * a;
        const double norm = std::sqrt(s);
        if (norm == 0.0) {
            gaussian(eng, v.data(), n);
            normalize(v);
            sigma = 0.0;
            continue;
        }
        for (std::size_t i = 0; i < n; ++i) v[i] = w[i] / norm;
        if (sigma != 0.0 && std::abs(norm - sigma) <= 1e-13 * norm) {
            sigma = norm;
            break;
        }
        sigma = norm;
    }
    *out = fro2 / (sigma * sigma);
    return OK;
}


// ---- Smith-Waterman alignment distance: CPU restatement of src/align.cpp:28-106
// (forward fill with the first maximal cell in row-major order, greedy
// traceback preferring diagonal > up > left among the predecessors that
// exactly account for the cell, zero cells walked through when accounted for;
// distance = mismatch + gap steps) and the canonical operand order of
// sw_distance (align.cpp:99-104: b < a lexicographically -> swap).
// out6 = score, distance, a_begin, a_end, b_begin, b_end
int orc_sw_align(const char* a, std::size_t na, const char* b, std::size_t nb, int match,
                 int mismatch, int gap, long long* out6) {
    if (!(match > 0 && mismatch < 0 && gap < 0)) return INVALID_ARGUMENT;
    if (na == 0 || nb == 0) return EMPTY_SEQUENCE;
    const std::size_t ld = nb + 1;
    std::vector<int> h((na + 1) * ld, 0);
    int best = 0;
    std::size_t bi = 0, bj = 0;
    auto sub = [&](std::size_t i, std::size_t j) {
        return (a[i - 1] == b[j - 1] && a[i - 1] != 'N') ? match : mismatch;
    };
    for (std::size_t i = 1; i <= na; ++i)
        for (std::size_t j = 1; j <= nb; ++j) {
            int v = h[(i - 1) * ld + j - 1] + sub(i, j);
            v = std::max(v, h[(i - 1) * ld + j] + gap);
            v = std::max(v, h[i * ld + j - 1] + gap);
            v = std::max(v, 0);
            h[i * ld + j] = v;
            if (v > best) {
                best = v;
                bi = i;
                bj = j;
            }
        }
    std::size_t i = bi, j = bj;
    long long events = 0;
    while (i > 0 && j > 0) {
        const int v = h[i * ld + j], s = sub(i, j);
        if (h[(i - 1) * ld + j - 1] + s == v) {
            if (s != match) ++events;
            --i;
            --j;
        } else if (h[(i - 1) * ld + j] + gap == v) {
            ++events;
            --i;
        } else if (h[i * ld + j - 1] + gap == v) {
            ++events;
            --j;
        } else {
            break;
        }
    }
    out6[0] = best;
    out6[1] = events;
    out6[2] = static_cast<long long>(i);
    out6[3] = static_cast<long long>(bi);
    out6[4] = static_cast<long long>(j);
    out6[5] = static_cast<long long>(bj);
    return 0;
}

int orc_sw_distance(const char* a, std::size_t na, const char* b, std::size_t nb, int match,
                    int mismatch, int gap, int* out) {
    const std::string_view va(a, na), vb(b, nb);
    long long r[6];
    const int st = (vb < va) ? orc_sw_align(b, nb, a, na, match, mismatch, gap, r)
                             : orc_sw_align(a, na, b, nb, match, mismatch, gap, r);
    if (st == 0) *out = static_cast<int>(r[1]);
    return st;
}

}  // extern "C"
