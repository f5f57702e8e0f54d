/* examples/ks_example.c -- the C ABI without Python: one B200, G-DD(n, kd=16)
 * generated on the device, BiCGSTAB and CG (G-SPD needs a circulant table, so CG
 * runs on a small explicit SPD matrix loaded with ks_load_rows, then multi-RHS CG
 * with 3 right-hand sides on it).  Prints one JSON
 * line.  Build: see __graft_entry__.build(); run: ./examples/ks_example [n]       */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ks.h"

#define CHECK(call)                                                                 \
    do {                                                                            \
        ks_status s_ = (call);                                                      \
        if (s_ != KS_OK && s_ != KS_EMAXIT) {                                       \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, (int)s_, ks_last_error(ctx)); \
            return 1;                                                               \
        }                                                                           \
    } while (0)

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 4096;
    ks_ctx* ctx = NULL;
    if (ks_create(&ctx, n, KS_FLOAT64, 1) != KS_OK) {
        fprintf(stderr, "ks_create: %s\n", ks_last_error(NULL));
        return 1;
    }
    double* b = (double*)malloc((size_t)n * sizeof(double));
    double* x = (double*)malloc((size_t)n * sizeof(double));
    double* hist = (double*)malloc(1000 * sizeof(double));
    ks_gen_spec spec = {1, 151107174ULL, 0.0, 16, NULL};          /* G-DD, kd = 16 */
    CHECK(ks_generate(ctx, &spec, b));
    ks_report rb;
    CHECK(ks_bicgstab(ctx, b, NULL, 1e-10, 1000, x, hist, 1000, &rb));
    /* CG on a diagonally dominant SPD matrix: A_ij = 1/(1+|i-j|), A_ii = n */
    const int64_t m = 512;
    ks_ctx* c2 = NULL;
    if (ks_create(&c2, m, KS_FLOAT64, 1) != KS_OK) return 1;
    double* A = (double*)malloc((size_t)m * m * sizeof(double));
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < m; ++j) A[i * m + j] = i == j ? (double)m : 1.0 / (1.0 + fabs((double)(i - j)));
    ks_ctx* keep = ctx;
    ctx = c2;
    CHECK(ks_load_rows(c2, 0, m, A, m));
    ks_report rc;
    CHECK(ks_cg(c2, b, NULL, 1e-12, 1000, x, hist, 1000, &rc));
    /* multi-RHS CG: 3 right-hand sides (column-major m x 3) in one solve */
    double* B3 = (double*)malloc((size_t)m * 3 * sizeof(double));
    double* X3 = (double*)malloc((size_t)m * 3 * sizeof(double));
    for (int64_t i = 0; i < m; ++i) {
        B3[i] = b[i];
        B3[m + i] = 1.0;
        B3[2 * m + i] = (double)(i % 7) - 3.0;
    }
    ks_report r3[3];
    CHECK(ks_cg_multi(c2, 3, B3, NULL, 1e-12, 1000, X3, NULL, 0, r3));
    double worst = 0.0;                      /* max_k ||B_k - A X_k|| / ||B_k|| on the host */
    for (int k = 0; k < 3; ++k) {
        double rr = 0.0, bb = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            double y = 0.0;
            for (int64_t j = 0; j < m; ++j) y += A[i * m + j] * X3[k * m + j];
            rr += (B3[k * m + i] - y) * (B3[k * m + i] - y);
            bb += B3[k * m + i] * B3[k * m + i];
        }
        if (sqrt(rr / bb) > worst) worst = sqrt(rr / bb);
    }
    ctx = keep;
    printf("{\"version\": \"%s\", \"n\": %lld, \"bicgstab\": {\"iterations\": %lld, \"converged\": %d, "
           "\"true_relres\": %.3e, \"us_per_iter\": %.2f}, \"cg\": {\"iterations\": %lld, \"converged\": %d, "
           "\"true_relres\": %.3e}, \"cg_multi\": {\"nrhs\": 3, \"converged\": %d, \"max_true_relres\": %.3e}}\n",
           ks_version(), (long long)n, (long long)rb.iterations, rb.converged, rb.true_relres,
           1e6 * rb.seconds_loop / (rb.iterations ? rb.iterations : 1), (long long)rc.iterations,
           rc.converged, rc.true_relres, r3[0].converged && r3[1].converged && r3[2].converged, worst);
    ks_destroy(c2);
    ks_destroy(ctx);
    free(A); free(b); free(x); free(hist); free(B3); free(X3);
    return 0;
}
