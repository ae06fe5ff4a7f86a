// C ABI of divscope-b200 (include/divscope.h). Mirrors the reference's MDS
// section of the C API (ref src/capi.cpp:37-103, :286-414): status mapping,
// thread-local last error, `wrap` semantics (nothing throws across the ABI),
// NULL checks, out-handles written only on success, option defaults and the
// clamp / error precedence of divscope_eigs / divscope_embed.
#include "divscope.h"

#include <charconv>
#include <cstring>
#include <fstream>
#include <new>
#include <sstream>
#include <mutex>
#include <string>
#include <vector>

#include "comm.hpp"
#include "kernels.cuh"
#include "solver.hpp"

using dsb::errc;
using dsb::Error;

struct divscope_readset {
    std::vector<std::string> ids;
    std::vector<std::string> seqs;  // empty for ids-only readsets
};
struct divscope_matrix {
    dsb::Matrix m;
};
static std::vector<std::string> index_ids(size_t n) {
    std::vector<std::string> ids;
    ids.reserve(n);
    for (size_t i = 0; i < n; ++i) ids.push_back(std::to_string(i));
    return ids;
}

struct divscope_embedding {
    // default ids "0".."n-1" (ref capi.cpp:345-348) are materialized on first
    // use: an embed call should not pay n string allocations it may not need
    std::vector<std::string> ids;
    bool default_ids = false;
    std::once_flag ids_once;
    dsb::Embedding emb;
    const std::vector<std::string>& id_list() {
        if (default_ids) std::call_once(ids_once, [this] { ids = index_ids(emb.n); });
        return ids;
    }
};

namespace {

thread_local std::string g_last_error;  // ref capi.cpp:39

divscope_status map_errc(errc c) { return static_cast<divscope_status>(static_cast<int>(c)); }

template <typename F>
divscope_status wrap(F&& f) noexcept {  // ref capi.cpp:66-82
    try {
        f();
        g_last_error.clear();
        return DIVSCOPE_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return map_errc(e.code());
    } catch (const std::bad_alloc&) {
        g_last_error = "out of memory";
        return DIVSCOPE_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return DIVSCOPE_ERR_INTERNAL;
    }
}

divscope_status fail_invalid(const char* msg) {  // ref capi.cpp:84-87
    g_last_error = msg;
    return DIVSCOPE_ERR_INVALID_ARGUMENT;
}

dsb::SolverOptions to_options(const divscope_solver_options* o) {  // ref capi.cpp:94-103
    dsb::SolverOptions opts;
    if (o) {
        opts.rank = o->rank;
        opts.oversampling = o->oversampling;
        opts.power_iters = o->power_iters;
        opts.seed = o->seed;
    }
    return opts;
}


// ref src/mds.cpp:152-188
void write_embedding_tsv(const dsb::Embedding& e, const std::vector<std::string>& ids,
                         const std::string& path) {
    if (ids.size() != e.n) throw Error(errc::shape_mismatch, "id count does not match embedding");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error(errc::io_error, "cannot open " + path + " for writing");
    out << "id";
    for (size_t c = 0; c < e.r; ++c) out << "\tdim" << (c + 1);
    out << '\n';
    const double* xy = e.host_coords();
    for (size_t i = 0; i < e.n; ++i) {
        out << ids[i];
        for (size_t c = 0; c < e.r; ++c) out << '\t' << dsb::format_double(xy[i * e.r + c]);
        out << '\n';
    }
    if (!out.flush()) throw Error(errc::io_error, "failed writing " + path);
}

void write_embedding_meta(const dsb::Embedding& e, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error(errc::io_error, "cannot open " + path + " for writing");
    out << "rank=" << e.r << '\n';
    out << "truncated=" << (e.truncated ? 1 : 0) << '\n';
    out << "eigenvalues=";
    for (size_t i = 0; i < e.eigenvalues.size(); ++i) {
        if (i) out << ',';
        out << dsb::format_double(e.eigenvalues[i]);
    }
    out << '\n';
    out << "dropped_negative_mass=" << dsb::format_double(e.dropped_negative_mass) << '\n';
    if (!out.flush()) throw Error(errc::io_error, "failed writing " + path);
}

// ref src/mds.cpp:190-238
void load_embedding_tsv(const std::string& path, std::vector<std::string>& ids, size_t& dims,
                        std::vector<double>& coords) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(errc::io_error, "cannot open " + path);
    std::string line;
    if (!std::getline(in, line)) throw Error(errc::bad_format, path + ": empty embedding table");
    if (!line.empty() && line.back() == '\r') line.pop_back();
    dims = 0;
    {
        std::istringstream header(line);
        std::string tok;
        if (!std::getline(header, tok, '\t') || tok != "id")
            throw Error(errc::bad_format, path + ": missing id header column");
        while (std::getline(header, tok, '\t')) ++dims;
        if (dims == 0) throw Error(errc::bad_format, path + ": no dimension columns");
    }
    size_t lineno = 1;
    while (std::getline(in, line)) {
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        std::istringstream row(line);
        std::string tok;
        if (!std::getline(row, tok, '\t') || tok.empty())
            throw Error(errc::bad_format, path + ": missing id on line " + std::to_string(lineno));
        ids.push_back(tok);
        size_t got = 0;
        while (std::getline(row, tok, '\t')) {
            char* endp = nullptr;
            const double v = std::strtod(tok.c_str(), &endp);
            if (endp == tok.c_str() || *endp != '\0')
                throw Error(errc::bad_format, path + ": bad number '" + tok + "' on line " +
                                                  std::to_string(lineno));
            coords.push_back(v);
            ++got;
        }
        if (got != dims)
            throw Error(errc::bad_format, path + ": expected " + std::to_string(dims) +
                                              " coordinates on line " + std::to_string(lineno));
    }
    if (ids.empty()) throw Error(errc::empty_input, path + ": no embedding rows");
}

}  // namespace

extern "C" {

const char* divscope_status_name(divscope_status s) {  // ref capi.cpp:116-139
    switch (s) {
        case DIVSCOPE_OK: return "ok";
        case DIVSCOPE_ERR_IO: return "io_error";
        case DIVSCOPE_ERR_EMPTY_INPUT: return "empty_input";
        case DIVSCOPE_ERR_INVALID_CHARACTER: return "invalid_character";
        case DIVSCOPE_ERR_DUPLICATE_ID: return "duplicate_id";
        case DIVSCOPE_ERR_SAMPLE_TOO_LARGE: return "sample_too_large";
        case DIVSCOPE_ERR_EMPTY_SEQUENCE: return "empty_sequence";
        case DIVSCOPE_ERR_BAD_FORMAT: return "bad_format";
        case DIVSCOPE_ERR_TRUNCATED: return "truncated";
        case DIVSCOPE_ERR_NOT_SYMMETRIC: return "not_symmetric";
        case DIVSCOPE_ERR_RANK_TOO_LARGE: return "rank_too_large";
        case DIVSCOPE_ERR_ZERO_MATRIX: return "zero_matrix";
        case DIVSCOPE_ERR_BAD_GAP: return "bad_gap";
        case DIVSCOPE_ERR_SHAPE_MISMATCH: return "shape_mismatch";
        case DIVSCOPE_ERR_MISSING_LABEL: return "missing_label";
        case DIVSCOPE_ERR_JOIN_ERROR: return "join_error";
        case DIVSCOPE_ERR_BAD_AXIS: return "bad_axis";
        case DIVSCOPE_ERR_INVALID_ARGUMENT: return "invalid_argument";
        case DIVSCOPE_ERR_INTERNAL: return "internal";
    }
    return "internal";
}

const char* divscope_last_error(void) { return g_last_error.c_str(); }

const char* divscope_version(void) { return "1.0.0-b200"; }

/* ---- readsets (ids only) ---- */

divscope_status divscope_readset_from_ids(const char* const* ids, size_t count,
                                          divscope_readset** out) {
    if ((!ids && count) || !out) return fail_invalid("null argument");
    return wrap([&] {
        auto* rs = new divscope_readset;
        for (size_t i = 0; i < count; ++i) {
            if (!ids[i]) {
                delete rs;
                throw Error(errc::invalid_argument, "null id");
            }
            rs->ids.emplace_back(ids[i]);
        }
        *out = rs;
    });
}

divscope_status divscope_readset_from_sequences(const char* const* ids,
                                                const char* const* sequences, size_t count,
                                                divscope_readset** out) {
    if ((!sequences && count) || !out) return fail_invalid("null argument");
    return wrap([&] {
        auto* rs = new divscope_readset;
        try {
            rs->ids.reserve(count);
            rs->seqs.reserve(count);
            for (size_t i = 0; i < count; ++i) {
                if (!sequences[i] || (ids && !ids[i])) throw Error(errc::invalid_argument, "null entry");
                rs->ids.emplace_back(ids ? std::string(ids[i]) : std::to_string(i));
                rs->seqs.emplace_back(sequences[i]);
            }
        } catch (...) {
            delete rs;
            throw;
        }
        *out = rs;
    });
}

const char* divscope_readset_sequence(const divscope_readset* rs, size_t i) {
    if (!rs || i >= rs->seqs.size()) return nullptr;
    return rs->seqs[i].c_str();
}

size_t divscope_readset_size(const divscope_readset* rs) { return rs ? rs->ids.size() : 0; }

const char* divscope_readset_id(const divscope_readset* rs, size_t i) {
    if (!rs || i >= rs->ids.size()) return nullptr;
    return rs->ids[i].c_str();
}

void divscope_readset_free(divscope_readset* rs) { delete rs; }

/* ---- matrices ---- */

divscope_status divscope_matrix_from_host(const double* values, size_t rows, size_t cols,
                                          int symmetric, divscope_matrix** out) {
    if ((!values && rows * cols != 0) || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_from_host(values, rows, cols, symmetric != 0, dsb::DType::F64);
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_matrix_from_host_f32(const float* values, size_t rows, size_t cols,
                                              int symmetric, divscope_matrix** out) {
    if ((!values && rows * cols != 0) || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_from_host(values, rows, cols, symmetric != 0, dsb::DType::F32);
        *out = new divscope_matrix{std::move(m)};
    });
}

size_t divscope_matrix_rows(const divscope_matrix* m) { return m ? m->m.store->rows : 0; }
size_t divscope_matrix_cols(const divscope_matrix* m) { return m ? m->m.store->cols : 0; }
int divscope_matrix_symmetric(const divscope_matrix* m) {
    return m && m->m.store->symmetric ? 1 : 0;
}

double divscope_matrix_get(const divscope_matrix* m, size_t i, size_t j) {
    if (!m || i >= m->m.store->rows || j >= m->m.store->cols) return 0.0;
    double v = 0.0;
    const divscope_status st = wrap([&] { v = dsb::matrix_get(m->m, i, j); });
    return st == DIVSCOPE_OK ? v : 0.0;
}

divscope_status divscope_matrix_copy_to_host(const divscope_matrix* m, double* out) {
    if (!m || (!out && m->m.store->rows * m->m.store->cols != 0)) return fail_invalid("null argument");
    return wrap([&] { dsb::matrix_to_host(m->m, out); });
}

divscope_status divscope_matrix_write(const divscope_matrix* m, const char* dvs_path) {
    if (!m || !dvs_path) return fail_invalid("null argument");
    return wrap([&] {
        const dsb::Store& s = *m->m.store;
        std::vector<double> host(s.rows * s.cols);
        dsb::matrix_to_host(m->m, host.data());
        dsb::write_dvs(dvs_path, s.rows, s.cols, m->m.gram ? true : s.symmetric, host.data());
    });
}

divscope_status divscope_matrix_write_tsv(const divscope_matrix* m, const divscope_readset* row_ids,
                                          const divscope_readset* col_ids,
                                          const char* tsv_path) {  // ref capi.cpp:270-282
    if (!m || !tsv_path) return fail_invalid("null argument");
    return wrap([&] {
        const dsb::Store& s = *m->m.store;
        const std::vector<std::string> rows = row_ids ? row_ids->ids : index_ids(s.rows);
        const std::vector<std::string> cols = col_ids ? col_ids->ids : index_ids(s.cols);
        // ref distmat.cpp:224-244
        if (rows.size() != s.rows || cols.size() != s.cols)
            throw Error(errc::shape_mismatch, "id lists do not match matrix shape");
        std::vector<double> host(s.rows * s.cols);
        dsb::matrix_to_host(m->m, host.data());
        std::ofstream out(tsv_path, std::ios::binary);
        if (!out) throw Error(errc::io_error, std::string("cannot open ") + tsv_path + " for writing");
        std::string line = "id";
        for (const std::string& id : cols) line += '\t' + id;
        line += '\n';
        out << line;
        for (size_t i = 0; i < s.rows; ++i) {
            line = rows[i];
            for (size_t j = 0; j < s.cols; ++j) {
                line += '\t';
                line += dsb::format_double(host[i * s.cols + j]);
            }
            line += '\n';
            out << line;
        }
        out.flush();
        if (!out) throw Error(errc::io_error, std::string("write failed for ") + tsv_path);
    });
}

divscope_status divscope_matrix_read(const char* dvs_path, divscope_matrix** out) {
    if (!dvs_path || !out) return fail_invalid("null argument");
    return wrap([&] {
        // streaming ingest: pinned double-buffered pread -> H2D (dvs_stream.cpp)
        dsb::Matrix m = dsb::matrix_read_dvs(dvs_path, false, 0, 0);
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_matrix_read_rows(const char* dvs_path, size_t row_begin,
                                          size_t row_end, divscope_matrix** out) {
    if (!dvs_path || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_read_dvs(dvs_path, true, row_begin, row_end);
        *out = new divscope_matrix{std::move(m)};
    });
}

void divscope_matrix_free(divscope_matrix* m) { delete m; }

divscope_status divscope_dvs_read_host(const char* dvs_path, size_t* rows, size_t* cols,
                                       int* symmetric, double* values) {
    if (!dvs_path || !rows || !cols || !symmetric) return fail_invalid("null argument");
    return wrap([&] {
        size_t r = 0, c = 0;
        bool sym = false;
        const std::vector<double> v = dsb::read_dvs(dvs_path, r, c, sym);
        *rows = r;
        *cols = c;
        *symmetric = sym ? 1 : 0;
        if (values && !v.empty()) std::memcpy(values, v.data(), v.size() * sizeof(double));
    });
}

divscope_status divscope_matrix_euclidean(const double* points, size_t n, size_t dim,
                                          int store_f32, divscope_matrix** out) {
    if (!points || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_euclidean(points, n, dim, store_f32 != 0);
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_matrix_hamming(const char* reads, size_t count, size_t length,
                                        divscope_matrix** out) {
    if (!reads || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_hamming(reads, count, length);
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_matrix_hamming_rows(const char* reads, size_t count, size_t length,
                                            size_t row_begin, size_t row_end,
                                            divscope_matrix** out) {
    if (!reads || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_hamming_rows(reads, count, length, row_begin, row_end);
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_hamming_counts(const char* reads, size_t count, size_t length,
                                        uint32_t* out) {
    if (!reads || !out) return fail_invalid("null argument");
    return wrap([&] { dsb::hamming_counts(reads, count, length, out); });
}

/* ---- Smith-Waterman distances on the GPU (ref capi.cpp:190-245) ---- */

void divscope_scoring_init(divscope_scoring* s) {
    if (!s) return;
    s->match = 1;
    s->mismatch = -1;
    s->gap = -2;
}

static dsb::SwScheme to_scheme(const divscope_scoring* s) {
    dsb::SwScheme x;
    if (s) {
        x.match = s->match;
        x.mismatch = s->mismatch;
        x.gap = s->gap;
    }
    return x;
}

divscope_status divscope_align(const char* a, const char* b, const divscope_scoring* scoring,
                               divscope_alignment* out) {
    if (!a || !b || !out) return fail_invalid("null argument");
    return wrap([&] {
        const dsb::SwAlignment r = dsb::sw_align(a, b, to_scheme(scoring));
        out->score = r.score;
        out->distance = r.distance;
        out->a_begin = r.a_begin;
        out->a_end = r.a_end;
        out->b_begin = r.b_begin;
        out->b_end = r.b_end;
    });
}

divscope_status divscope_distance(const char* a, const char* b, const divscope_scoring* scoring,
                                  int* out) {
    if (!a || !b || !out) return fail_invalid("null argument");
    return wrap([&] { *out = dsb::sw_distance(a, b, to_scheme(scoring)); });
}

static void need_sequences(const divscope_readset* rs) {
    if (rs->seqs.size() != rs->ids.size())
        throw Error(errc::invalid_argument, "readset has no sequences (ids-only)");
}

divscope_status divscope_pairwise_self(const divscope_readset* rs, const divscope_scoring* scoring,
                                       unsigned threads, divscope_matrix** out) {
    (void)threads;
    if (!rs || !out) return fail_invalid("null argument");
    return wrap([&] {
        need_sequences(rs);
        dsb::Matrix m = dsb::pairwise_self(rs->ids, rs->seqs, to_scheme(scoring));
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_pairwise_cross(const divscope_readset* queries,
                                        const divscope_readset* refs,
                                        const divscope_scoring* scoring, unsigned threads,
                                        divscope_matrix** out) {
    (void)threads;
    if (!queries || !refs || !out) return fail_invalid("null argument");
    return wrap([&] {
        need_sequences(queries);
        need_sequences(refs);
        dsb::Matrix m = dsb::pairwise_cross(queries->ids, queries->seqs, refs->ids, refs->seqs,
                                            to_scheme(scoring));
        *out = new divscope_matrix{std::move(m)};
    });
}

/* ---- spectra and embeddings ---- */

void divscope_solver_options_init(divscope_solver_options* o) {  // ref capi.cpp:288-294
    if (!o) return;
    o->rank = 50;
    o->oversampling = 10;
    o->power_iters = 2;
    o->seed = 0;
}

divscope_status divscope_gram(const divscope_matrix* dist, unsigned threads,
                              divscope_matrix** out) {  // ref capi.cpp:296-307
    (void)threads;
    if (!dist || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix g = dist->m.store->sharded ? dsb::gram_sharded(dist->m)
                                               : dsb::gram_from_distances(dist->m);
        *out = new divscope_matrix{std::move(g)};
    });
}

divscope_status divscope_eigs(const divscope_matrix* gram, const divscope_solver_options* opts,
                              unsigned threads, double* eigenvalues, size_t* count,
                              double* resid) {  // ref capi.cpp:309-325
    (void)threads;
    if (!gram || !opts || !eigenvalues) return fail_invalid("null argument");
    return wrap([&] {
        if (!gram->m.store->square())
            throw Error(errc::not_symmetric, "matrix is not square");
        const dsb::Spectrum s = gram->m.store->sharded ? dsb::eigs_sharded(gram->m, to_options(opts))
                                                       : dsb::eigs_sym(gram->m, to_options(opts));
        for (size_t i = 0; i < s.eigenvalues.size(); ++i) eigenvalues[i] = s.eigenvalues[i];
        if (count) *count = s.eigenvalues.size();
        if (resid) *resid = s.resid;
    });
}

divscope_status divscope_eigs_vectors(const divscope_matrix* gram,
                                      const divscope_solver_options* opts, unsigned threads,
                                      double* eigenvalues, double* vectors, size_t* count,
                                      double* resid) {  // ref rsvd.hpp:43-62 eigs_sym
    (void)threads;
    if (!gram || !opts || !eigenvalues || !vectors) return fail_invalid("null argument");
    return wrap([&] {
        if (!gram->m.store->square())
            throw Error(errc::not_symmetric, "matrix is not square");
        const dsb::Spectrum s = dsb::eigs_sym_vectors(gram->m, to_options(opts));
        for (size_t i = 0; i < s.eigenvalues.size(); ++i) eigenvalues[i] = s.eigenvalues[i];
        std::copy(s.vectors.begin(), s.vectors.end(), vectors);
        if (count) *count = s.eigenvalues.size();
        if (resid) *resid = s.resid;
    });
}

divscope_status divscope_stable_rank(const divscope_matrix* gram, unsigned threads,
                                     double* out) {  // ref capi.cpp:327-335
    (void)threads;
    if (!gram || !out) return fail_invalid("null argument");
    return wrap([&] {
        if (!gram->m.store->square())
            throw Error(errc::not_symmetric, "matrix is not square");
        *out = dsb::stable_rank(gram->m);
    });
}

divscope_status divscope_embed(const divscope_matrix* gram, const divscope_solver_options* opts,
                               unsigned threads, const divscope_readset* ids,
                               divscope_embedding** out) {  // ref capi.cpp:337-354
    (void)threads;
    if (!gram || !opts || !out) return fail_invalid("null argument");
    return wrap([&] {
        if (!gram->m.store->square())
            throw Error(errc::not_symmetric, "matrix is not square");
        if (ids && ids->ids.size() != gram->m.store->order())
            throw Error(errc::shape_mismatch, "id count does not match matrix");
        dsb::Embedding e = gram->m.store->sharded
                               ? dsb::embed_sharded(gram->m, opts->rank, to_options(opts))
                               : dsb::embed(gram->m, opts->rank, to_options(opts));
        auto* handle = new divscope_embedding;
        if (ids)
            handle->ids = ids->ids;
        else
            handle->default_ids = true;
        handle->emb = std::move(e);
        *out = handle;
    });
}

divscope_status divscope_reconstruction_error(const divscope_matrix* gram,
                                              const divscope_embedding* e, unsigned threads,
                                              double* out) {  // ref mds.hpp:54-58
    (void)threads;
    if (!gram || !e || !out) return fail_invalid("null argument");
    return wrap([&] { *out = dsb::reconstruction_error(gram->m, e->emb); });
}

divscope_status divscope_randomized_range(const divscope_matrix* gram,
                                          const divscope_solver_options* opts, double* q_out) {
    if (!gram || !opts || !q_out) return fail_invalid("null argument");
    return wrap([&] {
        if (!gram->m.store->square())
            throw Error(errc::not_symmetric, "matrix is not square");
        dsb::randomized_range(gram->m, to_options(opts), q_out);
    });
}

size_t divscope_embedding_rows(const divscope_embedding* e) { return e ? e->emb.n : 0; }
size_t divscope_embedding_dims(const divscope_embedding* e) { return e ? e->emb.r : 0; }

const char* divscope_embedding_id(const divscope_embedding* e, size_t i) {
    if (!e) return nullptr;
    const auto& v = const_cast<divscope_embedding*>(e)->id_list();
    if (i >= v.size()) return nullptr;
    return v[i].c_str();
}

double divscope_embedding_get(const divscope_embedding* e, size_t i, size_t c) {
    if (!e || i >= e->emb.n || c >= e->emb.r) return 0.0;
    return e->emb.host_coords()[i * e->emb.r + c];
}

size_t divscope_embedding_eigenvalues(const divscope_embedding* e, double* out, size_t cap) {
    if (!e) return 0;
    if (out)
        for (size_t i = 0; i < e->emb.eigenvalues.size() && i < cap; ++i)
            out[i] = e->emb.eigenvalues[i];
    return e->emb.eigenvalues.size();
}

double divscope_embedding_dropped_negative_mass(const divscope_embedding* e) {
    return e ? e->emb.dropped_negative_mass : 0.0;
}

int divscope_embedding_truncated(const divscope_embedding* e) {
    return e && e->emb.truncated ? 1 : 0;
}

const double* divscope_embedding_coords(const divscope_embedding* e) {
    if (!e) return nullptr;
    return e->emb.host_coords();
}

double divscope_embedding_resid(const divscope_embedding* e) { return e ? e->emb.resid : 0.0; }

divscope_status divscope_embedding_write(const divscope_embedding* e, const char* tsv_path,
                                         const char* meta_path) {
    if (!e || !tsv_path) return fail_invalid("null argument");
    return wrap([&] {
        write_embedding_tsv(e->emb, const_cast<divscope_embedding*>(e)->id_list(), tsv_path);
        if (meta_path) write_embedding_meta(e->emb, meta_path);
    });
}

divscope_status divscope_embedding_load(const char* tsv_path, divscope_embedding** out) {
    if (!tsv_path || !out) return fail_invalid("null argument");
    return wrap([&] {
        auto* handle = new divscope_embedding;
        try {
            size_t dims = 0;
            std::vector<double> coords;
            load_embedding_tsv(tsv_path, handle->ids, dims, coords);
            handle->emb.set_host_coords(coords);
            handle->emb.n = handle->ids.size();
            handle->emb.r = dims;
        } catch (...) {
            delete handle;
            throw;
        }
        *out = handle;
    });
}

void divscope_embedding_free(divscope_embedding* e) { delete e; }

/* ---- multi-GPU ---- */

divscope_status divscope_comm_unique_id(void* id128) {
    if (!id128) return fail_invalid("null argument");
    return wrap([&] { dsb::Comm::get().unique_id(id128); });
}

divscope_status divscope_comm_init(int world, int rank, const void* id128) {
    if (!id128) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Ctx& c = dsb::Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        dsb::Comm::get().init(world, rank, id128, c.stream);
    });
}

divscope_status divscope_comm_destroy(void) {
    return wrap([&] { dsb::Comm::get().destroy(); });
}

divscope_status divscope_shard_range(size_t n, int world, int rank, size_t* begin, size_t* end) {
    if (!begin || !end) return fail_invalid("null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail_invalid("bad world/rank");
    dsb::shard_rows(n, world, rank, *begin, *end);
    g_last_error.clear();
    return DIVSCOPE_OK;
}

divscope_status divscope_matrix_from_host_rows(const double* rows, size_t n, size_t row_begin,
                                               size_t row_end, int symmetric,
                                               divscope_matrix** out) {
    if ((!rows && row_end > row_begin) || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_from_host_rows(rows, n, row_begin, row_end, symmetric != 0,
                                                   dsb::DType::F64);
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_matrix_from_host_rows_f32(const float* rows, size_t n, size_t row_begin,
                                                   size_t row_end, int symmetric,
                                                   divscope_matrix** out) {
    if ((!rows && row_end > row_begin) || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m = dsb::matrix_from_host_rows(rows, n, row_begin, row_end, symmetric != 0,
                                                   dsb::DType::F32);
        *out = new divscope_matrix{std::move(m)};
    });
}

divscope_status divscope_matrix_euclidean_rows(const double* points, size_t n, size_t dim,
                                               int store_f32, size_t row_begin, size_t row_end,
                                               divscope_matrix** out) {
    if (!points || !out) return fail_invalid("null argument");
    return wrap([&] {
        dsb::Matrix m =
            dsb::matrix_euclidean_rows(points, n, dim, store_f32 != 0, row_begin, row_end);
        *out = new divscope_matrix{std::move(m)};
    });
}

/* ---- device / instrumentation ---- */

divscope_status divscope_set_product_path(int mode) {
    if (mode < 0 || mode > 2) return fail_invalid("mode must be 0, 1 or 2");
    dsb::set_product_path(mode);
    return DIVSCOPE_OK;
}

divscope_status divscope_set_sdig_cache(int mode) {
    if (mode < 0 || mode > 2) return fail_invalid("mode must be 0, 1 or 2");
    dsb::set_sdig_policy(mode);
    return DIVSCOPE_OK;
}

divscope_status divscope_set_device(int device) {
    return wrap([&] { dsb::Ctx::get().set_device(device); });
}

void divscope_stats_enable_timing(int on) {
    try {
        dsb::Ctx& c = dsb::Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        c.set_timing(on != 0);
    } catch (...) {
    }
}

void divscope_stats_reset(void) {
    try {
        dsb::Ctx& c = dsb::Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        c.drain_timing();
        c.k2_ms = c.k1_ms = c.k2_first_ms = 0.0;
        c.k2_launches = c.k1_launches = c.k2_first_launches = 0;
        c.h2d = c.d2h = 0;
        c.launches_base = dsb::kernel_launch_count();
    } catch (...) {
    }
}

void divscope_stats_get(divscope_stats* out) {
    if (!out) return;
    std::memset(out, 0, sizeof(*out));
    try {
        dsb::Ctx& c = dsb::Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        c.drain_timing();
        out->kernel_launches = dsb::kernel_launch_count() - c.launches_base;
        out->product_launches = c.k2_launches;
        out->product_ms = c.k2_ms;
        out->stats_launches = c.k1_launches;
        out->stats_ms = c.k1_ms;
        out->h2d_bytes = c.h2d;
        out->d2h_bytes = c.d2h;
        out->last_evd_sweeps = c.last_evd_sweeps;
        out->last_orth_shifted = c.last_orth_shifted;
        out->last_power_iters = c.last_power_iters;
        out->last_product_kernel = c.last_product_kernel;
        out->last_product_groups = c.last_product_groups;
        out->last_product_sdigits = c.last_product_sdigits;
        out->last_product_pair = c.last_product_pair;
        out->last_product_sdig = c.last_product_sdig;
        out->product_first_launches = c.k2_first_launches;
        out->product_first_ms = c.k2_first_ms;
        out->last_product_stream_cl = c.last_product_stream_cl;
    } catch (...) {
    }
}

void* divscope_stream(void) {
    try {
        return dsb::Ctx::get().stream;
    } catch (...) {
        return nullptr;
    }
}

}  // extern "C"

// test hook: the antisymmetric symmetry fingerprint of a matrix handle's rows
// (the sharded gram's one-pass symmetry check, k1_shard.cu / sharded.cpp):
// out[0], out[1] = its two 32-bit halves
extern "C" int divscope_debug_sym_fingerprint(const divscope_matrix* m, unsigned long long* out) {
    if (!m || !out) return DIVSCOPE_ERR_INVALID_ARGUMENT;
    return wrap([&] {
        dsb::Ctx& c = dsb::Ctx::get();
        std::lock_guard<std::recursive_mutex> lk(c.mu);
        const dsb::Store& st = *m->m.store;
        const size_t rows = st.rows;
        const int grid = dsb::k1_rows_grid(rows, c.sms);
        auto* d = static_cast<unsigned long long*>(c.scratch("dbg_fp", 16));
        double* rs = static_cast<double*>(c.scratch("dbg_fp_rs", std::max<size_t>(rows, 1) * 8));
        double* cta = static_cast<double*>(c.scratch("dbg_fp_cta", static_cast<size_t>(grid) * 24));
        int* ex = static_cast<int*>(c.scratch("dbg_fp_ex", std::max<size_t>(rows, 1) * 4));
        DSB_CUDA(cudaMemsetAsync(d, 0, 16, c.stream));
        if (rows)
            dsb::launch_k1_rows(st.buf->p, st.dt, st.ld, rows, st.cols,
                                st.sharded ? st.row_begin : 0, rs, nullptr, cta, grid, c.stream,
                                ex, d);
        c.d2h_copy(out, d, 16);
        out[0] &= 0xFFFFFFFFull;
        out[1] &= 0xFFFFFFFFull;
    });
}

// test hook: Omega of (seed, n, w) as the solver uploads it (rng.hpp
// fill_gaussian on the host, relayout on the device), read back row-major
extern "C" int divscope_debug_omega_panel(uint64_t seed, size_t n, size_t w, double* out) {
    if (!out) return DIVSCOPE_ERR_INVALID_ARGUMENT;
    return wrap([&] { dsb::debug_omega_panel(seed, n, w, out); });
}

// test hook, host only: the product's fill_gaussian (host_core.cpp) driven
// by std::mt19937_64(seed), as omega_host fills the pinned Omega buffer
extern "C" int divscope_debug_fill_gaussian(uint64_t seed, size_t count, double* out) {
    if (!out) return DIVSCOPE_ERR_INVALID_ARGUMENT;
    return wrap([&] {
        std::mt19937_64 eng(seed);
        dsb::fill_gaussian(eng, out, count);
    });
}
