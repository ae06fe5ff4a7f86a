/* divscope_mds — a plain C caller of the drop-in boundary (include/divscope.h),
 * compiled with `-I include` and linked against libdivscope_b200.so. It
 * mirrors the two subcommands of the reference CLI that this library serves
 * (ref tools/divscope_main.cpp:267-282 `mds`, :284-304 `spectrum`):
 *
 *   divscope_mds mds      <dist.dvs> <out.tsv> [rank] [oversampling] [power_iters] [seed]
 *     read the DVS1 matrix, build the gram, clamp rank to n, embed with ids
 *     "0".."n-1", write <out.tsv> and <out.tsv>.meta
 *   divscope_mds spectrum <dist.dvs> [rank] [oversampling] [power_iters] [seed]
 *     eigenvalues, resid and stable rank, printed as the reference prints them
 *
 * Defaults come from divscope_solver_options_init (rank 50, p 10, q 2, seed 0,
 * ref src/capi.cpp:288-296). Every call's status is checked and reported with
 * divscope_status_name / divscope_last_error, as the reference CLI does.
 *
 * Build: make -C paper_1803_02272_b200/csrc caller   (tools/divscope_mds) */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "divscope.h"

static int check(divscope_status st, const char* what) {
    if (st == DIVSCOPE_OK) return 0;
    fprintf(stderr, "divscope_mds: %s: %s: %s\n", what, divscope_status_name(st),
            divscope_last_error());
    return 1;
}

static void options(int argc, char** argv, int first, divscope_solver_options* o) {
    divscope_solver_options_init(o);
    if (argc > first) o->rank = (size_t)strtoull(argv[first], NULL, 10);
    if (argc > first + 1) o->oversampling = (size_t)strtoull(argv[first + 1], NULL, 10);
    if (argc > first + 2) o->power_iters = (size_t)strtoull(argv[first + 2], NULL, 10);
    if (argc > first + 3) o->seed = (uint64_t)strtoull(argv[first + 3], NULL, 10);
}

static int load_gram(const char* path, const char* what, divscope_matrix** dist,
                     divscope_matrix** gram) {
    *dist = NULL;
    *gram = NULL;
    if (check(divscope_matrix_read(path, dist), what)) return 1;
    if (check(divscope_gram(*dist, 1, gram), what)) {
        divscope_matrix_free(*dist);
        *dist = NULL;
        return 1;
    }
    return 0;
}

static int cmd_mds(int argc, char** argv) {
    if (argc < 4) return 2;
    divscope_solver_options o;
    options(argc, argv, 4, &o);
    divscope_matrix *dist, *gram;
    if (load_gram(argv[2], "mds", &dist, &gram)) return 1;
    const size_t n = divscope_matrix_rows(gram);
    if (o.rank > n) o.rank = n; /* tools/divscope_main.cpp:271 */
    divscope_embedding* e = NULL;
    int rc = check(divscope_embed(gram, &o, 1, NULL, &e), "mds");
    if (!rc) {
        char* meta = (char*)malloc(strlen(argv[3]) + 6);
        sprintf(meta, "%s.meta", argv[3]);
        rc = check(divscope_embedding_write(e, argv[3], meta), "mds");
        free(meta);
        divscope_embedding_free(e);
    }
    divscope_matrix_free(gram);
    divscope_matrix_free(dist);
    return rc;
}

static int cmd_spectrum(int argc, char** argv) {
    if (argc < 3) return 2;
    divscope_solver_options o;
    options(argc, argv, 3, &o);
    divscope_matrix *dist, *gram;
    if (load_gram(argv[2], "spectrum", &dist, &gram)) return 1;
    const size_t n = divscope_matrix_rows(gram);
    if (o.rank > n) o.rank = n; /* tools/divscope_main.cpp:287-290 */
    if (o.oversampling > n - o.rank) o.oversampling = n - o.rank;
    double* ev = (double*)calloc(o.rank ? o.rank : 1, sizeof(double));
    size_t count = 0;
    double resid = 0.0, sr = 0.0;
    int rc = check(divscope_eigs(gram, &o, 1, ev, &count, &resid), "spectrum");
    if (!rc) rc = check(divscope_stable_rank(gram, 1, &sr), "spectrum");
    if (!rc) {
        for (size_t i = 0; i < count; ++i) printf("eigenvalue\t%zu\t%.17g\n", i + 1, ev[i]);
        printf("resid\t%.17g\n", resid);
        printf("stable_rank\t%.17g\n", sr);
    }
    free(ev);
    divscope_matrix_free(gram);
    divscope_matrix_free(dist);
    return rc;
}

int main(int argc, char** argv) {
    int rc = 2;
    if (argc >= 2 && strcmp(argv[1], "mds") == 0) rc = cmd_mds(argc, argv);
    if (argc >= 2 && strcmp(argv[1], "spectrum") == 0) rc = cmd_spectrum(argc, argv);
    if (rc == 2)
        fprintf(stderr,
                "usage: divscope_mds mds <dist.dvs> <out.tsv> [rank] [p] [q] [seed]\n"
                "       divscope_mds spectrum <dist.dvs> [rank] [p] [q] [seed]\n");
    return rc;
}
