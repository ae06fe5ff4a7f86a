// Host side of the GPU Smith-Waterman distance builder (sw.cu): validation
// with the reference's error codes and messages (ref src/align.cpp:12-15,
// src/distmat.cpp:37-41, :47-52, :92-97), read packing, result matrices.
#include <algorithm>
#include <string>
#include <vector>

#include "solver.hpp"

namespace dsb {

namespace {

void validate(const SwScheme& s) {  // ref align.cpp:12-15
    if (s.match <= 0 || s.mismatch >= 0 || s.gap >= 0)
        throw Error(errc::invalid_argument,
                    "scoring scheme requires match > 0, mismatch < 0, gap < 0");
}

void check_alignable(const std::vector<std::string>& ids, const std::vector<std::string>& seqs) {
    for (size_t i = 0; i < seqs.size(); ++i)  // ref distmat.cpp:37-41
        if (seqs[i].empty())
            throw Error(errc::empty_sequence,
                        "read '" + (i < ids.size() ? ids[i] : std::to_string(i)) + "' is empty");
}

struct Packed {
    std::shared_ptr<DevBuf> bytes, off, len;
    int max_len = 0;
};

Packed pack(const std::vector<const std::string*>& seqs) {
    Ctx& c = Ctx::get();
    Packed p;
    std::vector<long long> off(seqs.size());
    std::vector<int> len(seqs.size());
    size_t total = 0;
    for (size_t i = 0; i < seqs.size(); ++i) {
        off[i] = static_cast<long long>(total);
        len[i] = static_cast<int>(seqs[i]->size());
        total += seqs[i]->size();
        p.max_len = std::max(p.max_len, len[i]);
    }
    std::string cat;
    cat.reserve(total);
    for (const std::string* s : seqs) cat += *s;
    p.bytes = std::make_shared<DevBuf>(std::max<size_t>(total, 1));
    p.off = std::make_shared<DevBuf>(std::max<size_t>(off.size(), 1) * sizeof(long long));
    p.len = std::make_shared<DevBuf>(std::max<size_t>(len.size(), 1) * sizeof(int));
    if (total) c.h2d_copy(p.bytes->p, cat.data(), total);
    if (!off.empty()) {
        c.h2d_copy(p.off->p, off.data(), off.size() * sizeof(long long));
        c.h2d_copy(p.len->p, len.data(), len.size() * sizeof(int));
    }
    return p;
}

void run(const Packed& p, int mode, long long na, long long nb, long long npairs,
         const SwScheme& s, double* dout, size_t ld, long long* aux) {
    Ctx& c = Ctx::get();
    const SwPlan plan = sw_plan(p.max_len, c.sms, mode, s.match, s.mismatch, s.gap);
    auto* dirs = static_cast<unsigned short*>(c.scratch("sw_dirs", plan.dirs_elems * 2));
    int* hb = static_cast<int*>(c.scratch("sw_hb", plan.hb_elems * 4));
    launch_sw(p.bytes->as<unsigned char>(), p.off->as<long long>(), p.len->as<int>(), mode, na, nb,
              npairs, s.match, s.mismatch, s.gap, plan, dirs, hb, dout, ld, aux, c.stream);
    DSB_CUDA(cudaGetLastError());
}

}  // namespace

SwAlignment sw_align(const std::string& a, const std::string& b, const SwScheme& s) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    validate(s);
    if (a.empty() || b.empty())
        throw Error(errc::empty_sequence, "cannot align an empty sequence");
    const Packed p = pack({&a, &b});
    auto* aux = static_cast<long long*>(c.scratch("sw_aux", 8 * sizeof(long long)));
    run(p, 2, 1, 1, 1, s, nullptr, 0, aux);
    long long h[6];
    c.d2h_copy(h, aux, sizeof(h));
    SwAlignment r;
    r.score = static_cast<int>(h[0]);
    r.distance = static_cast<int>(h[1]);
    r.a_begin = static_cast<size_t>(h[2]);
    r.a_end = static_cast<size_t>(h[3]);
    r.b_begin = static_cast<size_t>(h[4]);
    r.b_end = static_cast<size_t>(h[5]);
    return r;
}

int sw_distance(const std::string& a, const std::string& b, const SwScheme& s) {
    // canonical operand order (ref align.cpp:99-104)
    return (b < a) ? sw_align(b, a, s).distance : sw_align(a, b, s).distance;
}

Matrix pairwise_self(const std::vector<std::string>& ids, const std::vector<std::string>& seqs,
                     const SwScheme& s) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const size_t n = seqs.size();
    if (n < 2)  // ref distmat.cpp:47-52
        throw Error(errc::invalid_argument,
                    "pairwise_self needs at least 2 reads, got " + std::to_string(n));
    validate(s);
    check_alignable(ids, seqs);
    std::vector<const std::string*> v;
    for (const auto& x : seqs) v.push_back(&x);
    const Packed p = pack(v);
    Matrix m;
    m.store = make_store(n, n, true, DType::F64);
    Store& st = *m.store;
    DSB_CUDA(cudaMemsetAsync(st.buf->p, 0, st.ld * n * sizeof(double), c.stream));
    const long long npairs = static_cast<long long>(n) * (static_cast<long long>(n) - 1) / 2;
    run(p, 0, static_cast<long long>(n), 0, npairs, s, st.buf->as<double>(), st.ld, nullptr);
    c.sync();
    return m;
}

Matrix pairwise_cross(const std::vector<std::string>& qids, const std::vector<std::string>& q,
                      const std::vector<std::string>& rids, const std::vector<std::string>& r,
                      const SwScheme& s) {
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (q.empty() || r.empty())  // ref distmat.cpp:92-97
        throw Error(errc::invalid_argument, "pairwise_cross needs nonempty sets");
    validate(s);
    check_alignable(qids, q);
    check_alignable(rids, r);
    std::vector<const std::string*> v;
    for (const auto& x : q) v.push_back(&x);
    for (const auto& x : r) v.push_back(&x);
    const Packed p = pack(v);
    Matrix m;
    m.store = make_store(q.size(), r.size(), false, DType::F64);
    Store& st = *m.store;
    const long long npairs = static_cast<long long>(q.size()) * static_cast<long long>(r.size());
    run(p, 1, static_cast<long long>(q.size()), static_cast<long long>(r.size()), npairs, s,
        st.buf->as<double>(), st.ld, nullptr);
    c.sync();
    return m;
}

}  // namespace dsb
