/*
 * oracle.c -- fp64 direct-sum reference for the PSF-interpolation blur H and
 * its adjoint H^T.  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this.  It shares no code, header or
 * constant with the CUDA path (paper_1705_06603_b200/csrc).
 *
 * Operator (Sec. II-B):  y = R sum_k Z_k H_k W_k C_k x
 *   W_k = diag(omega_k), omega_k(r, c) = wy[p][r] * wx[q][c], k = p*Gx + q
 *   H_k = C_k' calH_k: convolution with h_k chopped to the valid region
 *         (PAPER.md:109), R restricts to the sensor, M = N - P + 1 (PAPER.md:61 fn).
 * Written out as the plain double sum (readings A16-A18):
 *   (Hx)(i,j) = sum_k sum_{a,b} h_k[a][b] * omega_k(i+2c-a, j+2c-b) * x(i+2c-a, j+2c-b)
 *   (H^T r)(p,q) = sum_k omega_k(p,q) * sum_{a,b} h_k[a][b] * r(p-2c+a, q-2c+b)
 * with c = (P-1)/2 and r = 0 outside the observed window.
 *
 * "Window" variants evaluate the facet-local operator H_f: the
 * global H restricted to the estimate window [e0y, e0y+ny) x [e0x, e0x+nx)
 * and the observed rows/cols whose footprint lies inside it.  omega_k is always
 * evaluated at GLOBAL coordinates.
 *
 * Loop order is row-axpy (SURVEY §8d "loop order matters"): the same sum,
 * terms skipped only where omega_k == 0 exactly (rows where wy_p = 0, and columns
 * outside the support [tlo, thi] of wx_q on the window: the skipped terms are exact
 * zeros, so every nonzero term is added in the same order).  OpenMP over output rows.
 */

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* [*lo, *hi] = first / last index of w[0..n) that is nonzero (lo > hi: none) */
static void nz_span(const double *w, int64_t n, int64_t *lo, int64_t *hi)
{
    *lo = 0; *hi = -1;
    while (*lo < n && w[*lo] == 0.0) ++*lo;
    if (*lo == n) return;
    *hi = n - 1;
    while (w[*hi] == 0.0) --*hi;
}

/* out[(ny-P+1) x (nx-P+1)] = H_f x_win.  x_win is [ny][nx] at global origin (e0y, e0x). */
void orc_H_window(int64_t Ny, int64_t Nx, int P, int Gy, int Gx,
                  const double *psfs, const double *wy, const double *wx,
                  int64_t e0y, int64_t e0x, int64_t ny, int64_t nx,
                  const double *x, double *out)
{
    const int64_t c2 = P - 1;               /* 2c */
    const int64_t my = ny - c2, mx = nx - c2;
    (void)Ny; (void)Nx;
    if (my <= 0 || mx <= 0) return;
    memset(out, 0, sizeof(double) * (size_t)(my * mx));
    double *xw = (double *)malloc(sizeof(double) * (size_t)(ny * nx));
    for (int p = 0; p < Gy; ++p) {
        for (int q = 0; q < Gx; ++q) {
            const double *wyp = wy + (int64_t)p * Ny + e0y;
            const double *wxq = wx + (int64_t)q * Nx + e0x;
            int any = 0;
            for (int64_t r = 0; r < ny && !any; ++r) any = (wyp[r] != 0.0);
            int anyx = 0;
            for (int64_t t = 0; t < nx && !anyx; ++t) anyx = (wxq[t] != 0.0);
            if (!any || !anyx) continue;
            int64_t tlo, thi;                     /* columns of the window where wx_q != 0 */
            nz_span(wxq, nx, &tlo, &thi);
            /* W_k C_k x : weighted copy of the window */
            #pragma omp parallel for schedule(static)
            for (int64_t r = 0; r < ny; ++r)
                for (int64_t t = 0; t < nx; ++t)
                    xw[r * nx + t] = wyp[r] * wxq[t] * x[r * nx + t];
            const double *h = psfs + (int64_t)(p * Gx + q) * P * P;
            /* H_k: valid convolution, accumulated into the shared output (Z_k, R) */
            #pragma omp parallel for schedule(dynamic, 4)
            for (int64_t i = 0; i < my; ++i) {
                double *o = out + i * mx;
                for (int a = 0; a < P; ++a) {
                    const int64_t li = i + c2 - a;
                    if (wyp[li] == 0.0) continue;
                    const double *row = xw + li * nx;
                    for (int b = 0; b < P; ++b) {
                        const double hv = h[a * P + b];
                        const double *src = row + (c2 - b);
                        /* src[j] = xw[li][j + c2 - b] is zero unless tlo <= j + c2 - b <= thi */
                        int64_t j0 = tlo - c2 + b, j1 = thi - c2 + b + 1;
                        if (j0 < 0) j0 = 0;
                        if (j1 > mx) j1 = mx;
                        for (int64_t j = j0; j < j1; ++j) o[j] += hv * src[j];
                    }
                }
            }
        }
    }
    free(xw);
}

/* g[ny x nx] = H_f^T r_win.  r_win is the observed window [ny-P+1][nx-P+1] whose
 * global observed origin is (e0y, e0x); r is zero outside it. */
void orc_HT_window(int64_t Ny, int64_t Nx, int P, int Gy, int Gx,
                   const double *psfs, const double *wy, const double *wx,
                   int64_t e0y, int64_t e0x, int64_t ny, int64_t nx,
                   const double *r, double *g)
{
    const int64_t c2 = P - 1;
    const int64_t my = ny - c2, mx = nx - c2;
    memset(g, 0, sizeof(double) * (size_t)(ny * nx));
    if (my <= 0 || mx <= 0) return;
    for (int p = 0; p < Gy; ++p) {
        for (int q = 0; q < Gx; ++q) {
            const double *wyp = wy + (int64_t)p * Ny + e0y;
            const double *wxq = wx + (int64_t)q * Nx + e0x;
            const double *h = psfs + (int64_t)(p * Gx + q) * P * P;
            int64_t tlo, thi;                     /* columns of the window where wx_q != 0 */
            nz_span(wxq, nx, &tlo, &thi);
            if (tlo > thi) continue;
            #pragma omp parallel
            {
                double *corr = (double *)malloc(sizeof(double) * (size_t)nx);
                #pragma omp for schedule(dynamic, 4)
                for (int64_t pr = 0; pr < ny; ++pr) {
                    if (wyp[pr] == 0.0) continue;
                    memset(corr, 0, sizeof(double) * (size_t)nx);
                    for (int a = 0; a < P; ++a) {
                        const int64_t ri = pr - c2 + a;          /* observed row */
                        if (ri < 0 || ri >= my) continue;
                        const double *rrow = r + ri * mx;
                        for (int b = 0; b < P; ++b) {
                            const double hv = h[a * P + b];
                            /* corr[q] += h[a][b] * r[ri][q - 2c + b] for valid columns */
                            int64_t q0 = c2 - b, q1 = mx + c2 - b; /* q in [q0, q1) */
                            if (q0 < tlo) q0 = tlo;           /* corr is used only where wx_q != 0 */
                            if (q1 > thi + 1) q1 = thi + 1;
                            const double *src = rrow + (b - c2);
                            for (int64_t qq = q0; qq < q1; ++qq) corr[qq] += hv * src[qq];
                        }
                    }
                    double *go = g + pr * nx;
                    for (int64_t qq = tlo; qq <= thi; ++qq) go[qq] += wyp[pr] * wxq[qq] * corr[qq];
                }
                free(corr);
            }
        }
    }
}

/* Point evaluation of the global H at observed pixels (oi[n], oj[n]) from the
 * full estimate x[Ny][Nx] (for sampled parity at full size). */
void orc_H_points(int64_t Ny, int64_t Nx, int P, int Gy, int Gx,
                  const double *psfs, const double *wy, const double *wx,
                  const double *x, int64_t n, const int64_t *oi, const int64_t *oj,
                  double *out)
{
    const int64_t c2 = P - 1;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < n; ++s) {
        double acc = 0.0;
        for (int p = 0; p < Gy; ++p)
            for (int q = 0; q < Gx; ++q) {
                const double *h = psfs + (int64_t)(p * Gx + q) * P * P;
                for (int a = 0; a < P; ++a) {
                    const int64_t E = oi[s] + c2 - a;
                    const double wyv = wy[(int64_t)p * Ny + E];
                    if (wyv == 0.0) continue;
                    for (int b = 0; b < P; ++b) {
                        const int64_t F = oj[s] + c2 - b;
                        acc += h[a * P + b] * wyv * wx[(int64_t)q * Nx + F] * x[E * Nx + F];
                    }
                }
            }
        out[s] = acc;
    }
}

/* Point evaluation of the global H^T at estimate pixels (ei[n], ej[n]) from the
 * full observed r[My][Mx]. */
void orc_HT_points(int64_t Ny, int64_t Nx, int P, int Gy, int Gx,
                   const double *psfs, const double *wy, const double *wx,
                   const double *r, int64_t n, const int64_t *ei, const int64_t *ej,
                   double *out)
{
    const int64_t c2 = P - 1;
    const int64_t My = Ny - c2, Mx = Nx - c2;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < n; ++s) {
        double acc = 0.0;
        for (int p = 0; p < Gy; ++p)
            for (int q = 0; q < Gx; ++q) {
                const double om = wy[(int64_t)p * Ny + ei[s]] * wx[(int64_t)q * Nx + ej[s]];
                if (om == 0.0) continue;
                const double *h = psfs + (int64_t)(p * Gx + q) * P * P;
                double corr = 0.0;
                for (int a = 0; a < P; ++a) {
                    const int64_t ri = ei[s] - c2 + a;
                    if (ri < 0 || ri >= My) continue;
                    for (int b = 0; b < P; ++b) {
                        const int64_t rj = ej[s] - c2 + b;
                        if (rj < 0 || rj >= Mx) continue;
                        corr += h[a * P + b] * r[ri * Mx + rj];
                    }
                }
                acc += om * corr;
            }
        out[s] = acc;
    }
}
