// oracle/_ref/ref_mds — TEST INFRASTRUCTURE ONLY: the reference CLI's `mds`
// flow (ref tools/divscope_main.cpp:267-282) as a standalone executable over
// the reference sources compiled into oracle/_ref (ref_harness.cpp
// ref_mds_files: read_matrix, gram_from_distances, embed,
// write_embedding_tsv / _meta). Run as a subprocess by the tests.
//   ref_mds <dist.dvs> <out.tsv> <rank> <oversampling> <power_iters> <seed>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>

extern "C" int ref_mds_files(const char*, std::size_t, std::size_t, std::size_t, std::uint64_t,
                             unsigned, const char*, const char*);
extern "C" const char* ref_last_error(void);

int main(int argc, char** argv) {
    if (argc != 7) {
        std::fprintf(stderr, "usage: ref_mds <dist.dvs> <out.tsv> <rank> <p> <q> <seed>\n");
        return 2;
    }
    const std::string meta = std::string(argv[2]) + ".meta";
    const unsigned threads = std::max(1u, std::thread::hardware_concurrency());
    const int rc = ref_mds_files(argv[1], std::strtoull(argv[3], nullptr, 10),
                                 std::strtoull(argv[4], nullptr, 10),
                                 std::strtoull(argv[5], nullptr, 10),
                                 std::strtoull(argv[6], nullptr, 10), threads, argv[2], meta.c_str());
    if (rc) std::fprintf(stderr, "ref_mds: status %d: %s\n", rc, ref_last_error());
    return rc ? 1 : 0;
}
