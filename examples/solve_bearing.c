/*
 * solve_bearing.c -- the C ABI (include/gpcg.h) used from plain C, no Python: build the
 * journal-bearing QP of BASELINE.json configs[0] (50 x 50, eps = 0.1, l = 0, u = +inf;
 * PAPER.md P:742-786, reading R2 for the finite-difference operator) in host
 * arrays, solve it on the GPU, and print the result.
 *
 *   gcc -O2 -I include examples/solve_bearing.c -L paper_cs_0101018_b200 -lgpcg \
 *       -Wl,-rpath,paper_cs_0101018_b200 -lm -o solve_bearing
 *   ./solve_bearing [n]          (n x n grid, default 50)
 *
 * Prints one line: status, objective, ||grad_Omega q||, iteration counts, free count.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "gpcg.h"

int main(int argc, char **argv) {
    const int64_t n1 = argc > 1 ? atoll(argv[1]) : 50;
    const int64_t nx = n1, ny = n1, n = nx * ny;
    const double pi = 3.14159265358979323846, eps = 0.1;
    const double hx = 2.0 * pi / (double)(nx + 1), hy = 20.0 / (double)(ny + 1);
    double *wx = malloc((size_t)(nx + 1) * sizeof(double));     /* x faces, broadcast over rows */
    double *wy = malloc((size_t)nx * sizeof(double));           /* y faces, broadcast           */
    double *b = malloc((size_t)n * sizeof(double)), *l = malloc((size_t)n * sizeof(double));
    double *u = malloc((size_t)n * sizeof(double)), *x = malloc((size_t)n * sizeof(double));
    double *x0 = calloc((size_t)n, sizeof(double));
    /* w(xi) = (1 + eps cos xi)^3; x-face i between points i-1, i sits at xi = (i + 1/2) hx
       (1-based point i at i hx), y-faces at the point's xi = (i + 1) hx */
    for (int64_t i = 0; i <= nx; ++i) {
        const double w = 1.0 + eps * cos(((double)i + 0.5) * hx);
        wx[i] = (hy / hx) * w * w * w;
    }
    for (int64_t i = 0; i < nx; ++i) {
        const double w = 1.0 + eps * cos((double)(i + 1) * hx);
        wy[i] = (hx / hy) * w * w * w;
    }
    for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
            const int64_t v = i + nx * j;
            b[v] = eps * sin((double)(i + 1) * hx) * hx * hy;
            l[v] = 0.0;
            u[v] = INFINITY;
        }
    gpcg_problem *h = NULL;
    int rc = gpcg_create_stencil2d(&h, NULL, nx, ny, wx, 0, wy, 0, NULL, b, l, u, 0.0);
    if (rc != GPCG_OK) {
        fprintf(stderr, "create: %d %s\n", rc, gpcg_last_error());
        return 1;
    }
    gpcg_stats st;
    rc = gpcg_solve(h, x0, -1e-8, 500, x, &st);     /* tau = 1e-8 ||g(x0)|| (R5) */
    int64_t nfree = 0;
    for (int64_t v = 0; v < n; ++v) nfree += x[v] > 0.0;
    printf("status=%d q=%.15g pg=%.3e outer=%lld gp=%lld cg=%lld free=%lld n=%lld\n", rc, st.q, st.pg_norm,
           (long long)st.outer_iters, (long long)st.gp_iters, (long long)st.cg_iters, (long long)nfree,
           (long long)n);
    gpcg_destroy(h);
    free(wx); free(wy); free(b); free(l); free(u); free(x); free(x0);
    return rc == GPCG_OK ? 0 : 2;
}
