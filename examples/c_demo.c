/*
 * c_demo.c -- the C ABI of libdeblur used from plain C (no Python, no torch): a small
 * synthetic problem (2x2 grid of Gaussian PSFs with bilinear interpolation weights, a
 * star field blurred by the library's own H plus noise), 2x2 overlapping facets, a few
 * full distributed iterations, the objective before and after, the blended image.
 *
 * Build (done by __graft_entry__.build()):
 *   gcc -O2 -std=c99 -I include -o examples/c_demo examples/c_demo.c \
 *       -L paper_1705_06603_b200 -ldeblur -Wl,-rpath,'$ORIGIN/../paper_1705_06603_b200' -lm
 * Run:    examples/c_demo [iterations]        (needs an sm_100 GPU; exit code 0 on success)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "deblur.h"

#define CHECK(h, call)                                                                   \
    do {                                                                                 \
        deblur_status s_ = (call);                                                       \
        if (s_ != DEBLUR_OK) {                                                           \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)s_, deblur_last_error(h)); \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

/* first-order interpolation hats for G grid points at cell centres, clamped (A14, A15) */
static void hats(float *w, int G, int64_t n) {
    const double L = (double)n / G;
    for (int g = 0; g < G; ++g)
        for (int64_t t = 0; t < n; ++t) {
            const double c = (g + 0.5) * L;
            double v = 1.0 - fabs((double)t - c) / L;
            if (v < 0) v = 0;
            if (g == 0 && t <= c) v = 1;
            if (g == G - 1 && t >= c) v = 1;
            w[(int64_t)g * n + t] = (float)v;
        }
}

static uint64_t rng = 88172645463325252ull;
static double urand(void) {              /* xorshift64 */
    rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
    return (double)(rng >> 11) / 9007199254740992.0;
}

int main(int argc, char **argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 10;
    const int64_t N = 512;
    const int P = 15, G = 2, c = (P - 1) / 2;
    const int64_t M = N - P + 1;
    float *psfs = malloc(sizeof(float) * G * G * P * P);
    for (int k = 0; k < G * G; ++k) {    /* Gaussian PSFs, sigma 1.2 .. 2.1, unit sum */
        const double sg = 1.2 + 0.3 * k;
        double sum = 0;
        for (int a = 0; a < P; ++a)
            for (int b = 0; b < P; ++b) sum += exp(-0.5 * ((a - c) * (a - c) + (b - c) * (b - c)) / (sg * sg));
        for (int a = 0; a < P; ++a)
            for (int b = 0; b < P; ++b)
                psfs[(k * P + a) * P + b] = (float)(exp(-0.5 * ((a - c) * (a - c) + (b - c) * (b - c)) / (sg * sg)) / sum);
    }
    float *wy = malloc(sizeof(float) * G * N), *wx = malloc(sizeof(float) * G * N);
    hats(wy, G, N);
    hats(wx, G, N);
    float *truth = calloc((size_t)(N * N), sizeof(float));
    for (int64_t i = 0; i < N * N; ++i) truth[i] = 0.05f;
    for (int s = 0; s < 300; ++s) truth[(int64_t)(urand() * N) * N + (int64_t)(urand() * N)] += (float)(0.2 + 0.8 * urand());
    float *y = calloc((size_t)(M * M), sizeof(float));

    deblur_params p;
    memset(&p, 0, sizeof p);
    p.abi_version = DEBLUR_ABI_VERSION;
    p.ny = N; p.nx = N; p.psf_gy = G; p.psf_gx = G; p.psf_size = P;
    p.psfs = psfs; p.interp_wy = wy; p.interp_wx = wx; p.y = y;
    p.noise_w = NULL; p.noise_w_scalar = 1e4f;
    p.lambda = 0.01f; p.eps = 1e-3f; p.gamma = 4000.f; p.rho = 1.f; p.tau = 0.0; p.inner_steps = 1;
    p.facet_gy = 2; p.facet_gx = 2; p.overlap = 32;
    p.world = 1;
    deblur_t h = NULL;
    CHECK(NULL, deblur_create(&p, &h));

    /* observation: y = H truth + noise (sigma 0.01), through the library's own H */
    CHECK(h, deblur_apply_H(h, truth, y));
    for (int64_t i = 0; i < M * M; ++i) {
        const double u1 = urand() + 1e-12, u2 = urand();
        y[i] += (float)(0.01 * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
    }
    CHECK(h, deblur_reset(h, y, NULL));
    double tau = 0, o0[4], o1[4];
    CHECK(h, deblur_get_step(h, &tau));
    CHECK(h, deblur_objective(h, o0));
    CHECK(h, deblur_iterate(h, iters));
    CHECK(h, deblur_objective(h, o1));
    float *img = malloc(sizeof(float) * N * N);
    CHECK(h, deblur_get_image(h, img));
    double err0 = 0, err1 = 0, ref = 0;
    for (int64_t r = c; r < N - c; ++r)          /* against the truth: observed vs estimate */
        for (int64_t q = c; q < N - c; ++q) {
            const double t = truth[r * N + q];
            err0 += (y[(r - c) * M + q - c] - t) * (y[(r - c) * M + q - c] - t);
            err1 += (img[r * N + q] - t) * (img[r * N + q] - t);
            ref += t * t;
        }
    printf("c_demo: %dx%d, P=%d, %dx%d PSFs, 2x2 facets, tau=%.6g, %d iterations\n", (int)N, (int)N, P, G, G, tau,
           iters);
    printf("objective %.6e -> %.6e (data %.6e, reg %.6e, consensus max-diff %.3e)\n", o0[0], o1[0], o1[1], o1[2],
           o1[3]);
    printf("SNR observed %.2f dB, estimate %.2f dB\n", 10 * log10(ref / err0), 10 * log10(ref / err1));
    const int ok = o1[0] < o0[0] && isfinite(o1[0]);
    CHECK(h, deblur_destroy(h));
    free(psfs); free(wy); free(wx); free(truth); free(y); free(img);
    return ok ? 0 : 2;
}
