/*
 * ens_c_example.c -- the C ABI (include/ens.h) used from plain C, no Python, no torch.
 *
 * A thin cylinder (radius R, length L, ends fixed) under a uniform internal pressure p,
 * two wall realisations (E and 1.25 E), mass-proportional damping so that the explicit
 * central-difference run (Eq. 22) settles to the static state.  At
 * mid-length the radial displacement of a long thin cylinder is the Laplace-law value
 * u_r = (1 - nu^2) p R^2 / (E h) (with the end correction of SURVEY.md §8(c) C10,
 * ~1% here); realisation 1 must come out 1.25x stiffer.
 *
 *   gcc -O2 -Iinclude examples/ens_c_example.c -Lpaper_2101_09059_b200 -lens \
 *       -Wl,-rpath,$PWD/paper_2101_09059_b200 -lm -o ens_c_example && ./ens_c_example
 *
 * Exit codes: 0 ok, 1 wrong answer, 2 an ens_* call failed (e.g. ENS_E_CUDA: no GPU).
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ens.h"

#define NC 48           /* nodes per ring */
#define NA 121          /* rings */

static int die(const char* what, int rc) {
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, ens_last_error(NULL));
    return 2;
}

int main(void) {
    const double R = 2.0, L = 30.0, E0 = 7e6, h0 = 0.4, rho = 1.06, nu = 0.5, p = 13.0 * 1333.22;
    const int64_t V = (int64_t)NC * NA, F = 2 * (int64_t)NC * (NA - 1);
    const int32_t n_s = 2;
    double* xyz = malloc(sizeof(double) * 3 * V);
    int32_t* tris = malloc(sizeof(int32_t) * 3 * F);
    uint8_t* fixed = calloc((size_t)V, 1);
    double* E = malloc(sizeof(double) * n_s * V);
    double* h = malloc(sizeof(double) * n_s * V);
    double* force = calloc((size_t)(3 * V), sizeof(double));
    double* u = malloc(sizeof(double) * n_s * 3 * V);
    const double pi = 3.14159265358979323846;

    /* offset rings: node r * NC + i at angle 2 pi (i + r/2) / NC, height r L / (NA - 1) */
    for (int r = 0; r < NA; ++r)
        for (int i = 0; i < NC; ++i) {
            const double th = 2.0 * pi * (i + 0.5 * (r & 1)) / NC;
            double* x = xyz + 3 * ((int64_t)r * NC + i);
            x[0] = R * cos(th);
            x[1] = R * sin(th);
            x[2] = L * r / (NA - 1);
            if (r == 0 || r == NA - 1) fixed[(int64_t)r * NC + i] = ENS_FIX_X | ENS_FIX_Y | ENS_FIX_Z;
        }
    int64_t f = 0;
    for (int r = 0; r + 1 < NA; ++r)
        for (int i = 0; i < NC; ++i) {
            const int32_t a = r * NC + i, b = r * NC + (i + 1) % NC;
            const int32_t c = (r + 1) * NC + i, d = (r + 1) * NC + (i + 1) % NC;
            /* counter-clockwise about the outward normal */
            if (r & 1) {
                int32_t t0[3] = {a, b, d}, t1[3] = {a, d, c};
                for (int k = 0; k < 3; ++k) { tris[3 * f + k] = t0[k]; tris[3 * f + 3 + k] = t1[k]; }
            } else {
                int32_t t0[3] = {a, b, c}, t1[3] = {b, d, c};
                for (int k = 0; k < 3; ++k) { tris[3 * f + k] = t0[k]; tris[3 * f + 3 + k] = t1[k]; }
            }
            f += 2;
        }
    /* nodal forces of the uniform pressure: p A_e / 3 along the element normal */
    for (int64_t e = 0; e < F; ++e) {
        const double* X[3];
        for (int k = 0; k < 3; ++k) X[k] = xyz + 3 * (int64_t)tris[3 * e + k];
        const double a[3] = {X[1][0] - X[0][0], X[1][1] - X[0][1], X[1][2] - X[0][2]};
        const double b[3] = {X[2][0] - X[0][0], X[2][1] - X[0][1], X[2][2] - X[0][2]};
        const double n[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
        for (int k = 0; k < 3; ++k)
            for (int c = 0; c < 3; ++c) force[3 * (int64_t)tris[3 * e + k] + c] += p * n[c] / 6.0;   /* |n| = 2 A */
    }
    for (int s = 0; s < n_s; ++s)
        for (int64_t i = 0; i < V; ++i) {
            E[s * V + i] = E0 * (s == 0 ? 1.0 : 1.25);
            h[s * V + i] = h0;
        }

    ens_mesh mesh = {V, F, xyz, tris, fixed};
    ens_materials mat = {n_s, E, h, rho, nu, 5.0 / 6.0, 0};
    ens_options opt = {0};
    opt.damping = ENS_DAMP_MASS;
    opt.c_d = 250.0;
    opt.kernel = ENS_KERNEL_ASSEMBLED_SYM;
    opt.device = -1;
    ens_ctx* ctx = NULL;
    int rc = ens_create(&mesh, &mat, &opt, &ctx);
    if (rc) return die("ens_create", rc);
    if ((rc = ens_set_traction(ctx, 1, force, 0, NULL, NULL, 0.0, 0.0))) return die("ens_set_traction", rc);
    if ((rc = ens_prepare(ctx))) return die("ens_prepare", rc);   /* step-loop graphs, no step run */
    if ((rc = ens_step(ctx, 12000))) return die("ens_step", rc);
    double t = 0.0;
    int64_t step = 0;
    if ((rc = ens_get_state(ctx, u, NULL, &t, &step))) return die("ens_get_state", rc);
    ens_info info;
    ens_query(ctx, &info);

    const int rm = NA / 2;
    double ur[2] = {0.0, 0.0};
    for (int s = 0; s < n_s; ++s)
        for (int i = 0; i < NC; ++i) {
            const int64_t node = (int64_t)rm * NC + i;
            const double* x = xyz + 3 * node;
            const double* us = u + 3 * ((int64_t)s * V + node);
            ur[s] += (us[0] * x[0] + us[1] * x[1]) / R / NC;
        }
    const double ell = R * sqrt((5.0 / 6.0) / (2.0 * (1.0 + nu)));
    const double ref = (1.0 - nu * nu) * p * R * R / (E0 * h0) / (1.0 - 2.0 * nu * nu * ell / L);
    printf("steps %lld (t = %.4f s, dt = %.3e s), nnzb %lld, %.0f MB/step algorithmic\n", (long long)step, t,
           info.dt, (long long)info.nnzb, info.bytes_per_step / 1e6);
    printf("mid-length u_r: s=0 %.6e cm, s=1 %.6e cm; Laplace law %.6e cm (rel %.2e); ratio %.4f\n", ur[0], ur[1],
           ref, ur[0] / ref - 1.0, ur[0] / ur[1]);
    ens_destroy(ctx);
    const int ok = fabs(ur[0] / ref - 1.0) < 2e-2 && fabs(ur[0] / ur[1] - 1.25) < 1e-3;
    free(xyz); free(tris); free(fixed); free(E); free(h); free(force); free(u);
    return ok ? 0 : 1;
}
