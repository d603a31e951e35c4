// k_fft.cu -- hand-written FFT overlap-save path for H and H^T.
//
// The paper evaluates each local blur in the Fourier domain as a circular
// convolution chopped to its valid region.  Here the facet is cut
// into S x S windows (S = 2^n) whose valid part is T = S - P + 1 per axis
// (overlap-save).  For an H tile (observed origin (i0, j0), window = estimate
// rows/cols [i0, i0+S)):
//     z = IDFT2( sum_{k=(p,q)} Hhat_k . DFT2(omega_k . x_win) ),  Hx = z[2c.., 2c..]
// and the separable hat omega_k = wy_p (x) wx_q is split across the two passes:
//   pass A (rows):    R2C DFT along x of x_win . wx_q       -- one per active q
//   pass B (columns): for each active (p, q): DFT along y of wy_p . A_q, times
//                     Hhat_k, accumulated; one inverse DFT along y
//   pass C (rows):    C2R inverse along x, crop, epilogue r = W (Hx - y)
// H^T mirrors it (correlation = conj(Hhat), omega_k applied after):
//   pass A' : R2C of the r window (observed rows/cols [p0-2c, p0-2c+S))
//   pass B' : DFT along y once; per (p, q): IDFT_y(conj(Hhat_k) . R), weighted by
//             wy_p and accumulated per q
//   pass C' : per q C2R along x, weighted by wx_q, summed -> g
// Every DFT is a radix-8/4/2 Stockham FFT in shared memory with twiddles from a
// table computed in fp64 on the host and rounded to fp32 (A24).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "epilogue.cuh"
#include "fft.hpp"

namespace deblur {

namespace {

constexpr int NT = 256;
constexpr int INV_HT = 3;   // k_rows_inv mode for H^T (H modes are FftMode values)

struct FftArgs {
    const FacetDev *facets;
    const TileDesc *tiles;
    int ntiles;
    const float2 *W;        // [S] exp(-2 pi i k / S)
    const float2 *Hhat;     // [nslots][S][LDF]
    const int *psf_slot;    // [K] -> slot
    const float *wy, *wx;   // [Gy][Ny], [Gx][Nx]
    int Ny, Nx, P, Gx;
    float2 *scratch;        // per tile: tile_rows x LDF
    int64_t tile_rows;      // rows of LDF complex per tile
    int NQ;                 // q slots per tile
    double *partials;
    float scale;            // 2 / S^2
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// multiply by -i*SIGN... : rot(v) = v * (SIGN < 0 ? -i : +i)
template <int SIGN>
__device__ __forceinline__ float2 rot90(float2 v) {
    return SIGN < 0 ? make_float2(v.y, -v.x) : make_float2(-v.y, v.x);
}

template <int SIGN>
__device__ __forceinline__ void dft2(float2 &a, float2 &b) {
    float2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <int SIGN>
__device__ __forceinline__ void dft4(float2 &a0, float2 &a1, float2 &a2, float2 &a3) {
    // X_k = sum_n a_n e^{SIGN 2 pi i n k / 4}
    float2 s0 = cadd(a0, a2), d0 = csub(a0, a2);
    float2 s1 = cadd(a1, a3), d1 = rot90<SIGN>(csub(a1, a3));
    a0 = cadd(s0, s1);
    a2 = csub(s0, s1);
    a1 = cadd(d0, d1);
    a3 = csub(d0, d1);
}

template <int SIGN>
__device__ __forceinline__ void dft8(float2 (&v)[8]) {
    const float r = 0.70710678118654752f;
    // even/odd split: X_k = E_k + w8^k O_k, X_{k+4} = E_k - w8^k O_k
    float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<SIGN>(e0, e1, e2, e3);
    dft4<SIGN>(o0, o1, o2, o3);
    // w8^1 = (r, SIGN r), w8^2 = SIGN i, w8^3 = (-r, SIGN r)
    const float2 t1 = make_float2(r * (o1.x - SIGN * o1.y), r * (o1.y + SIGN * o1.x));
    const float2 t2 = rot90<SIGN>(o2);
    const float2 t3 = make_float2(-r * (o3.x + SIGN * o3.y), r * (SIGN * o3.x - o3.y));
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, t1); v[5] = csub(e1, t1);
    v[2] = cadd(e2, t2); v[6] = csub(e2, t2);
    v[3] = cadd(e3, t3); v[7] = csub(e3, t3);
}

// One Stockham stage (Govindaraju et al. formulation) over nb transforms of length L
// stored at in[t*stride + n]; twiddles W[idx * wmul] with W the size-S table.
template <int R, int SIGN>
__device__ __forceinline__ void stage(const float2 *__restrict__ in, float2 *__restrict__ out, int L, int Ns, int nb,
                                      int stride, const float2 *__restrict__ W, int wmul, int S) {
    const int LR = L / R;
    const int total = nb * LR;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int t = idx / LR, j = idx - t * LR;
        const float2 *src = in + (int64_t)t * stride;
        float2 *dst = out + (int64_t)t * stride;
        float2 v[8];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[j + r * LR];
        const int k = j % Ns;
        if (Ns > 1) {
            const int base = k * (L / (Ns * R));
#pragma unroll
            for (int r = 1; r < R; ++r) {
                float2 w = __ldg(W + ((base * r * wmul) & (S - 1)));
                if (SIGN > 0) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        if (R == 8) {
            dft8<SIGN>(v);
        } else if (R == 4) {
            dft4<SIGN>(v[0], v[1], v[2], v[3]);
        } else {
            dft2<SIGN>(v[0], v[1]);
        }
        const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[idxD + r * Ns] = v[r];
    }
}

// In-smem FFT of nb transforms of length L (power of 2).  Data starts in a; the
// result pointer (a or b) is returned.  All threads of the CTA participate; ends
// with __syncthreads().  SIGN = -1 forward, +1 inverse (unnormalised).
template <int SIGN>
__device__ float2 *fft_smem(float2 *a, float2 *b, int L, int nb, int stride, const float2 *W, int S) {
    const int wmul = S / L;
    int Ns = 1;
    while (Ns < L) {
        const int R = (L / Ns >= 8) ? 8 : (L / Ns);
        if (R == 8) stage<8, SIGN>(a, b, L, Ns, nb, stride, W, wmul, S);
        else if (R == 4) stage<4, SIGN>(a, b, L, Ns, nb, stride, W, wmul, S);
        else stage<2, SIGN>(a, b, L, Ns, nb, stride, W, wmul, S);
        __syncthreads();
        float2 *t = a; a = b; b = t;
        Ns *= R;
    }
    return a;
}

template <int S>
struct Geo {
    static constexpr int SH = S / 2;
    static constexpr int NF = SH + 1;
    static constexpr int LDF = SH + 16;            // padded row length of spectra
    static constexpr int ROWS = (S >= 512) ? 8 : 16;  // rows per CTA in the row passes
    static constexpr int C = (S >= 1024) ? 4 : 8;   // columns per CTA in the column pass
    static constexpr int CS = S + 1;                // smem column stride (bank spread)
    static constexpr int RS = SH + 1;               // smem row stride in the row passes
};

// ------------------------------------------------------------------ pass A / A'
// mode 0: H (x window . wx_q, one R2C per active q); mode 1: H^T (r window); mode 2: PSF spectra
template <int S>
__global__ void __launch_bounds__(NT) k_rows_fwd(FftArgs A, int mode, int par, const float *psfs, int npsf,
                                                 float2 *hrows) {
    using G = Geo<S>;
    extern __shared__ __align__(16) float2 sm2[];
    float *xs = reinterpret_cast<float *>(sm2);                  // ROWS x S reals
    float2 *a = sm2 + G::ROWS * S / 2;                           // ROWS x RS
    float2 *b = a + G::ROWS * G::RS;
    const int nblk = S / G::ROWS;
    const int tile = blockIdx.x / nblk, r0 = (blockIdx.x % nblk) * G::ROWS;
    const int P = A.P, c2 = P - 1;
    int nq = 1, q0 = 0;
    TileDesc t{};
    const FacetDev *F = nullptr;
    if (mode == 2) {
        if (tile >= npsf) return;
    } else {
        t = A.tiles[tile];
        F = &A.facets[t.f];
        if (mode == 0) { q0 = t.q0; nq = t.q1 - t.q0 + 1; }
    }
    // load the real rows
    for (int idx = threadIdx.x; idx < G::ROWS * S; idx += NT) {
        const int rr = idx / S, cc = idx - rr * S;
        const int row = r0 + rr;
        float v = 0.f;
        if (mode == 0) {
            const int ly = t.y0 + row, lx = t.x0 + cc;
            if (ly < F->ny && lx < F->nx) v = F->x[par][(int64_t)ly * F->ep + lx];
        } else if (mode == 1) {
            const int ri = t.y0 - c2 + row, rj = t.x0 - c2 + cc;
            if (ri >= 0 && ri < F->my && rj >= 0 && rj < F->mx) v = F->r[(int64_t)ri * F->op + rj];
        } else {
            if (row < P && cc < P) v = psfs[(int64_t)tile * P * P + row * P + cc];
        }
        xs[idx] = v;
    }
    __syncthreads();
    for (int qi = 0; qi < nq; ++qi) {
        const float *wxq = (mode == 0) ? A.wx + (size_t)(q0 + qi) * A.Nx + F->ex0 + t.x0 : nullptr;
        for (int idx = threadIdx.x; idx < G::ROWS * G::SH; idx += NT) {
            const int rr = idx / G::SH, n = idx - rr * G::SH;
            float e = xs[rr * S + 2 * n], o = xs[rr * S + 2 * n + 1];
            if (mode == 0) {
                const int lx = t.x0 + 2 * n;
                e *= (lx < F->nx) ? __ldg(wxq + 2 * n) : 0.f;
                o *= (lx + 1 < F->nx) ? __ldg(wxq + 2 * n + 1) : 0.f;
            }
            a[rr * G::RS + n] = make_float2(e, o);
        }
        __syncthreads();
        float2 *Z = fft_smem<-1>(a, b, G::SH, G::ROWS, G::RS, A.W, S);
        // R2C post-processing: X[k] = (Zk + conj Z_{SH-k})/2 - i/2 W_S^k (Zk - conj Z_{SH-k})
        for (int idx = threadIdx.x; idx < G::ROWS * G::NF; idx += NT) {
            const int rr = idx / G::NF, k = idx - rr * G::NF;
            const float2 zk = Z[rr * G::RS + (k & (G::SH - 1))];
            const float2 zc = conjf2(Z[rr * G::RS + ((G::SH - k) & (G::SH - 1))]);
            const float2 s = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y + zc.y));
            const float2 d = make_float2(0.5f * (zk.x - zc.x), 0.5f * (zk.y - zc.y));
            const float2 w = __ldg(A.W + (k & (S - 1)));
            const float2 wd = cmul(w, d);                 // W^k d
            const float2 X = make_float2(s.x + wd.y, s.y - wd.x);   // s - i W^k d
            float2 *dst;
            if (mode == 2)
                dst = hrows + ((int64_t)tile * S + r0 + rr) * G::LDF;
            else
                dst = A.scratch + (int64_t)tile * A.tile_rows * G::LDF + ((int64_t)qi * S + r0 + rr) * G::LDF;
            dst[k] = X;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ pass B / B'
// mode 0: H; mode 1: H^T; mode 2: PSF spectra (forward column DFT of hrows -> Hhat)
template <int S>
__global__ void __launch_bounds__(NT) k_cols(FftArgs A, int mode, const float2 *hrows, float2 *hhat, int npsf) {
    using G = Geo<S>;
    extern __shared__ __align__(16) float2 sm2[];
    constexpr int C = G::C, CS = G::CS;
    float2 *colq = sm2;               // C x CS : A_q columns (H) / R-hat (H^T)
    float2 *w0 = colq + C * CS;       // work (ping)
    float2 *w1 = w0 + C * CS;         // work (pong)
    float2 *acc = w1 + C * CS;        // accumulator
    const int nchunk = (G::NF + C - 1) / C;
    const int tile = blockIdx.x / nchunk, f0 = (blockIdx.x % nchunk) * C;
    const int P = A.P, c2 = P - 1, T = S - P + 1;

    if (mode == 2) {
        if (tile >= npsf) return;
        for (int idx = threadIdx.x; idx < C * S; idx += NT) {
            const int c = idx % C, ky = idx / C;
            w0[c * CS + ky] = (f0 + c < G::NF) ? hrows[((int64_t)tile * S + ky) * G::LDF + f0 + c] : make_float2(0, 0);
        }
        __syncthreads();
        float2 *Z = fft_smem<-1>(w0, w1, S, C, CS, A.W, S);
        for (int idx = threadIdx.x; idx < C * S; idx += NT) {
            const int c = idx % C, ky = idx / C;
            if (f0 + c < G::NF) hhat[((int64_t)tile * S + ky) * G::LDF + f0 + c] = Z[c * CS + ky];
        }
        return;
    }

    const TileDesc t = A.tiles[tile];
    const FacetDev &F = A.facets[t.f];
    float2 *base = A.scratch + (int64_t)tile * A.tile_rows * G::LDF;

    if (mode == 0) {
        for (int idx = threadIdx.x; idx < C * S; idx += NT) acc[(idx % C) * CS + idx / C] = make_float2(0, 0);
        for (int q = t.q0; q <= t.q1; ++q) {
            __syncthreads();
            const float2 *Aq = base + (int64_t)(q - t.q0) * S * G::LDF;
            for (int idx = threadIdx.x; idx < C * S; idx += NT) {
                const int c = idx % C, row = idx / C;
                colq[c * CS + row] = Aq[(int64_t)row * G::LDF + f0 + c];
            }
            for (int p = t.p0; p <= t.p1; ++p) {
                __syncthreads();
                const float *wyp = A.wy + (size_t)p * A.Ny + F.ey0 + t.y0;
                for (int idx = threadIdx.x; idx < C * S; idx += NT) {
                    const int c = idx % C, row = idx / C;
                    const float wv = (t.y0 + row < F.ny) ? __ldg(wyp + row) : 0.f;
                    const float2 v = colq[c * CS + row];
                    w0[c * CS + row] = make_float2(wv * v.x, wv * v.y);
                }
                __syncthreads();
                float2 *Z = fft_smem<-1>(w0, w1, S, C, CS, A.W, S);
                const int slot = A.psf_slot[p * A.Gx + q];
                const float2 *Hk = A.Hhat + (int64_t)slot * S * G::LDF;
                for (int idx = threadIdx.x; idx < C * S; idx += NT) {
                    const int c = idx % C, ky = idx / C;
                    const float2 h = __ldg(Hk + (int64_t)ky * G::LDF + f0 + c);
                    float2 &o = acc[c * CS + ky];
                    o = cadd(o, cmul(Z[c * CS + ky], h));
                }
            }
        }
        __syncthreads();
        // inverse DFT along y of the accumulated spectrum (acc, w0 as pong)
        float2 *z = fft_smem<+1>(acc, w0, S, C, CS, A.W, S);
        float2 *O = base + (int64_t)A.NQ * S * G::LDF;
        for (int idx = threadIdx.x; idx < C * T; idx += NT) {
            const int c = idx % C, rr = idx / C;
            if (f0 + c < G::NF) O[(int64_t)rr * G::LDF + f0 + c] = z[c * CS + c2 + rr];
        }
        return;
    }

    // mode 1 (H^T)
    for (int idx = threadIdx.x; idx < C * S; idx += NT) {
        const int c = idx % C, row = idx / C;
        w0[c * CS + row] = base[(int64_t)row * G::LDF + f0 + c];
    }
    __syncthreads();
    {
        float2 *R = fft_smem<-1>(w0, w1, S, C, CS, A.W, S);
        if (R != colq)
            for (int idx = threadIdx.x; idx < C * CS; idx += NT) colq[idx] = R[idx];
    }
    float2 *Bbase = base + (int64_t)S * G::LDF;
    for (int q = t.q0; q <= t.q1; ++q) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < C * S; idx += NT) acc[(idx % C) * CS + idx / C] = make_float2(0, 0);
        for (int p = t.p0; p <= t.p1; ++p) {
            __syncthreads();
            const int slot = A.psf_slot[p * A.Gx + q];
            const float2 *Hk = A.Hhat + (int64_t)slot * S * G::LDF;
            for (int idx = threadIdx.x; idx < C * S; idx += NT) {
                const int c = idx % C, ky = idx / C;
                const float2 h = __ldg(Hk + (int64_t)ky * G::LDF + f0 + c);
                w0[c * CS + ky] = cmulc(colq[c * CS + ky], h);
            }
            __syncthreads();
            float2 *z = fft_smem<+1>(w0, w1, S, C, CS, A.W, S);
            const float *wyp = A.wy + (size_t)p * A.Ny + F.ey0 + t.y0;
            for (int idx = threadIdx.x; idx < C * T; idx += NT) {
                const int c = idx % C, rr = idx / C;
                const float wv = (t.y0 + rr < F.ny) ? __ldg(wyp + rr) : 0.f;
                const float2 v = z[c * CS + rr];
                float2 &o = acc[c * CS + rr];
                o = make_float2(o.x + wv * v.x, o.y + wv * v.y);
            }
        }
        __syncthreads();
        float2 *Bq = Bbase + (int64_t)(q - t.q0) * T * G::LDF;
        for (int idx = threadIdx.x; idx < C * T; idx += NT) {
            const int c = idx % C, rr = idx / C;
            if (f0 + c < G::NF) Bq[(int64_t)rr * G::LDF + f0 + c] = acc[c * CS + rr];
        }
    }
}

// ------------------------------------------------------------------ pass C / C'
// C2R of one spectrum row X[0..SH] (global) into smem reals out[0..S) (unscaled: SH x)
template <int S>
__device__ void c2r_rows(const float2 *__restrict__ src0, int64_t src_stride, int nrows, float2 *a, float2 *b,
                         float *outs, const float2 *W) {
    using G = Geo<S>;
    for (int idx = threadIdx.x; idx < nrows * G::SH; idx += NT) {
        const int rr = idx / G::SH, k = idx - rr * G::SH;
        const float2 *X = src0 + rr * src_stride;
        const float2 xk = X[k], xc = conjf2(X[G::SH - k]);
        const float2 e = make_float2(0.5f * (xk.x + xc.x), 0.5f * (xk.y + xc.y));
        const float2 d = make_float2(0.5f * (xk.x - xc.x), 0.5f * (xk.y - xc.y));
        const float2 w = conjf2(__ldg(W + k));
        const float2 o = cmul(d, w);                       // O_k
        a[rr * G::RS + k] = make_float2(e.x - o.y, e.y + o.x);   // E + i O
    }
    __syncthreads();
    float2 *z = fft_smem<+1>(a, b, G::SH, nrows, G::RS, W, S);
    for (int idx = threadIdx.x; idx < nrows * G::SH; idx += NT) {
        const int rr = idx / G::SH, n = idx - rr * G::SH;
        const float2 v = z[rr * G::RS + n];
        outs[rr * S + 2 * n] = v.x;
        outs[rr * S + 2 * n + 1] = v.y;
    }
    __syncthreads();
}

template <int S>
__global__ void __launch_bounds__(NT) k_rows_inv(FftArgs A, int mode) {
    using G = Geo<S>;
    extern __shared__ __align__(16) float2 sm2[];
    float *outs = reinterpret_cast<float *>(sm2);            // ROWS x S reals
    float2 *a = sm2 + G::ROWS * S / 2;
    float2 *b = a + G::ROWS * G::RS;
    float *gacc = reinterpret_cast<float *>(b + G::ROWS * G::RS);   // ROWS x T (H^T)
    __shared__ double red[NT / 32];
    const int P = A.P, c2 = P - 1, T = S - P + 1;
    const int nblk = (T + G::ROWS - 1) / G::ROWS;
    const int tile = blockIdx.x / nblk, r0 = (blockIdx.x % nblk) * G::ROWS;
    const int nrows = min(G::ROWS, T - r0);
    const TileDesc t = A.tiles[tile];
    const FacetDev &F = A.facets[t.f];
    const float2 *base = A.scratch + (int64_t)tile * A.tile_rows * G::LDF;
    const float scale = A.scale;

    if (mode != INV_HT) {
        const float2 *O = base + ((int64_t)A.NQ * S + r0) * G::LDF;
        c2r_rows<S>(O, G::LDF, nrows, a, b, outs, A.W);
        double dsum = 0.0;
        for (int idx = threadIdx.x; idx < nrows * T; idx += NT) {
            const int rr = idx / T, cc = idx - rr * T;
            const int oi = t.y0 + r0 + rr, oj = t.x0 + cc;
            if (oi >= F.my || oj >= F.mx) continue;
            const float hx = outs[rr * S + c2 + cc] * scale;
            const int64_t o = (int64_t)oi * F.op + oj;
            if (mode == FFT_PLAIN) {
                F.r[o] = hx;
            } else {
                const float wv = F.w ? F.w[o] : F.w_scalar;
                const float d = hx - F.y[o];
                if (mode == FFT_RESIDUAL) F.r[o] = wv * d;
                dsum += 0.5 * (double)wv * (double)d * (double)d;
            }
        }
        if (mode != FFT_PLAIN && A.partials) {
            const double s = block_sum(dsum, red);
            if (threadIdx.x == 0) A.partials[blockIdx.x] = s;
        }
        return;
    }
    // H^T: g = sum_q wx_q . C2R(B_q)
    for (int idx = threadIdx.x; idx < nrows * T; idx += NT) gacc[idx] = 0.f;
    const float2 *Bbase = base + (int64_t)S * G::LDF;
    for (int q = t.q0; q <= t.q1; ++q) {
        __syncthreads();
        const float2 *Bq = Bbase + ((int64_t)(q - t.q0) * T + r0) * G::LDF;
        c2r_rows<S>(Bq, G::LDF, nrows, a, b, outs, A.W);
        const float *wxq = A.wx + (size_t)q * A.Nx + F.ex0 + t.x0;
        for (int idx = threadIdx.x; idx < nrows * T; idx += NT) {
            const int rr = idx / T, cc = idx - rr * T;
            const float wv = (t.x0 + cc < F.nx) ? __ldg(wxq + cc) : 0.f;
            gacc[idx] += wv * (outs[rr * S + cc] * scale);
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nrows * T; idx += NT) {
        const int rr = idx / T, cc = idx - rr * T;
        const int fy = t.y0 + r0 + rr, fx = t.x0 + cc;
        if (fy < F.ny && fx < F.nx) F.g[(int64_t)fy * F.ep + fx] = gacc[idx];
    }
}

}  // namespace

struct FftPlan {
    int S = 0, T = 0, P = 0, NQ = 1;
    int K = 0, Gx = 1;
    std::vector<TileDesc> tH, tHT;
    TileDesc *d_tH = nullptr, *d_tHT = nullptr;
    std::vector<int> tile_facet_H;    // local facet index per H tile
    float2 *W = nullptr, *Hhat = nullptr, *scratch = nullptr;
    int *psf_slot = nullptr;
    int64_t tile_rows = 0;
    double *partials = nullptr;
    std::vector<double> h_part;
    int nblk_inv = 0;
    int nlocal = 0;
    const float *wy = nullptr, *wx = nullptr;
    int Ny = 0, Nx = 0;
    std::vector<void *> allocs;
    ~FftPlan() {
        for (void *p : allocs) cudaFree(p);
    }
    FftArgs args(const FacetDev *facets, bool ht) const {
        FftArgs a;
        a.facets = facets;
        a.tiles = ht ? d_tHT : d_tH;
        a.ntiles = (int)(ht ? tHT.size() : tH.size());
        a.W = W; a.Hhat = Hhat; a.psf_slot = psf_slot;
        a.wy = wy; a.wx = wx; a.Ny = Ny; a.Nx = Nx; a.P = P; a.Gx = Gx;
        a.scratch = scratch; a.tile_rows = tile_rows; a.NQ = NQ;
        a.partials = partials;
        a.scale = 2.0f / ((float)S * (float)S);
        return a;
    }
};

// FFT size per P: minimise S^2 log2(S) / T^2 (work per valid pixel), T = S - P + 1
static int choose_S(int P) {
    int best = 0;
    double bc = 1e300;
    for (int S = 64; S <= 1024; S *= 2) {
        const int T = S - P + 1;
        if (T < 8) continue;
        const double c = (double)S * S * std::log2((double)S) / ((double)T * T) * (1.0 + 0.02 * std::log2((double)S));
        if (c < bc) { bc = c; best = S; }
    }
    return best;
}

bool fft_prefer(int P) {
    // Crossover: measured on B200; direct below, FFT at and above.
    return P >= 31;
}

template <int S>
static size_t smem_rows_fwd() { using G = Geo<S>; return (size_t)G::ROWS * S * 4 + 2 * (size_t)G::ROWS * G::RS * 8; }
template <int S>
static size_t smem_cols() { using G = Geo<S>; return 4 * (size_t)G::C * G::CS * 8; }
template <int S>
static size_t smem_rows_inv(int T) { using G = Geo<S>; return (size_t)G::ROWS * S * 4 + 2 * (size_t)G::ROWS * G::RS * 8 + (size_t)G::ROWS * T * 4; }

template <int S>
static cudaError_t setup_attrs(int T) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_rows_fwd<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rows_fwd<S>())) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_cols<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cols<S>())) != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_rows_inv<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rows_inv<S>(T));
}

template <int S>
static cudaError_t run_rows_fwd(const FftArgs &a, int ntiles, int mode, int par, const float *psfs, int npsf,
                                float2 *hrows, cudaStream_t s) {
    if (ntiles == 0) return cudaSuccess;
    k_rows_fwd<S><<<ntiles * (S / Geo<S>::ROWS), NT, smem_rows_fwd<S>(), s>>>(a, mode, par, psfs, npsf, hrows);
    return cudaGetLastError();
}
template <int S>
static cudaError_t run_cols(const FftArgs &a, int ntiles, int mode, const float2 *hrows, float2 *hhat, int npsf,
                            cudaStream_t s) {
    if (ntiles == 0) return cudaSuccess;
    const int nchunk = (Geo<S>::NF + Geo<S>::C - 1) / Geo<S>::C;
    k_cols<S><<<ntiles * nchunk, NT, smem_cols<S>(), s>>>(a, mode, hrows, hhat, npsf);
    return cudaGetLastError();
}
template <int S>
static cudaError_t run_rows_inv(const FftArgs &a, int ntiles, int T, int mode, cudaStream_t s) {
    if (ntiles == 0) return cudaSuccess;
    const int nblk = (T + Geo<S>::ROWS - 1) / Geo<S>::ROWS;
    k_rows_inv<S><<<ntiles * nblk, NT, smem_rows_inv<S>(T), s>>>(a, mode);
    return cudaGetLastError();
}

#define FFT_DISPATCH(S_, CALL)                 \
    switch (S_) {                              \
    case 64: { constexpr int SS = 64; CALL; } break;   \
    case 128: { constexpr int SS = 128; CALL; } break; \
    case 256: { constexpr int SS = 256; CALL; } break; \
    case 512: { constexpr int SS = 512; CALL; } break; \
    case 1024: { constexpr int SS = 1024; CALL; } break; \
    default: return cudaErrorInvalidValue;     \
    }

static cudaError_t do_rows_fwd(int S, const FftArgs &a, int nt, int mode, int par, const float *psfs, int npsf,
                               float2 *hrows, cudaStream_t s) {
    FFT_DISPATCH(S, return run_rows_fwd<SS>(a, nt, mode, par, psfs, npsf, hrows, s));
    return cudaSuccess;
}
static cudaError_t do_cols(int S, const FftArgs &a, int nt, int mode, const float2 *hrows, float2 *hhat, int npsf,
                           cudaStream_t s) {
    FFT_DISPATCH(S, return run_cols<SS>(a, nt, mode, hrows, hhat, npsf, s));
    return cudaSuccess;
}
static cudaError_t do_rows_inv(int S, const FftArgs &a, int nt, int T, int mode, cudaStream_t s) {
    FFT_DISPATCH(S, return run_rows_inv<SS>(a, nt, T, mode, s));
    return cudaSuccess;
}
static cudaError_t do_attrs(int S, int T) {
    FFT_DISPATCH(S, return setup_attrs<SS>(T));
    return cudaSuccess;
}

FftPlan *fft_create(const Plan &pl, const std::vector<int> &local, const std::vector<FacetDev> &fh,
                    const float *d_psfs, const float *d_wy, const float *d_wx, int Gy, int Gx, const float *h_wy,
                    const float *h_wx, cudaStream_t s, std::string &err) {
    FftPlan *f = new FftPlan();
    auto fail = [&](const std::string &m) { err = m; delete f; return (FftPlan *)nullptr; };
#define FC(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) return fail(std::string(cudaGetErrorString(e_)) + " at " #call); \
    } while (0)
    f->P = pl.P;
    f->S = choose_S(pl.P);
    if (!f->S) return fail("no FFT size fits P");
    f->T = f->S - f->P + 1;
    f->Gx = Gx;
    f->K = Gy * Gx;
    f->wy = d_wy; f->wx = d_wx; f->Ny = (int)pl.ny; f->Nx = (int)pl.nx;
    f->nlocal = (int)local.size();
    const int S = f->S, T = f->T, P = f->P;
    const int LDF = S / 2 + 16;
    // active ranges
    auto range = [](const float *w, int G, int64_t n, int64_t a, int64_t b, int &lo, int &hi) {
        a = std::max<int64_t>(0, a); b = std::min<int64_t>(n, b);
        lo = G; hi = -1;
        for (int g = 0; g < G; ++g)
            for (int64_t i = a; i < b; ++i)
                if (w[(int64_t)g * n + i] != 0.f) { lo = std::min(lo, g); hi = std::max(hi, g); break; }
    };
    std::vector<char> used(f->K, 0);
    for (size_t li = 0; li < fh.size(); ++li) {
        const FacetDev &F = fh[li];
        for (int y0 = 0; y0 < F.my; y0 += T)
            for (int x0 = 0; x0 < F.mx; x0 += T) {
                TileDesc t{(int)li, y0, x0, 0, -1, 0, -1};
                range(h_wy, Gy, pl.ny, F.ey0 + y0, F.ey0 + std::min(y0 + S, F.ny), t.p0, t.p1);
                range(h_wx, Gx, pl.nx, F.ex0 + x0, F.ex0 + std::min(x0 + S, F.nx), t.q0, t.q1);
                if (t.q1 < t.q0) { t.q0 = 0; t.q1 = -1; }
                f->tH.push_back(t);
                f->tile_facet_H.push_back((int)li);
            }
        for (int y0 = 0; y0 < F.ny; y0 += T)
            for (int x0 = 0; x0 < F.nx; x0 += T) {
                TileDesc t{(int)li, y0, x0, 0, -1, 0, -1};
                range(h_wy, Gy, pl.ny, F.ey0 + y0, F.ey0 + std::min(y0 + T, F.ny), t.p0, t.p1);
                range(h_wx, Gx, pl.nx, F.ex0 + x0, F.ex0 + std::min(x0 + T, F.nx), t.q0, t.q1);
                if (t.q1 < t.q0) { t.q0 = 0; t.q1 = -1; }
                f->tHT.push_back(t);
            }
    }
    for (auto *lst : {&f->tH, &f->tHT})
        for (auto &t : *lst) {
            f->NQ = std::max(f->NQ, t.q1 - t.q0 + 1);
            for (int p = t.p0; p <= t.p1; ++p)
                for (int q = t.q0; q <= t.q1; ++q) used[p * Gx + q] = 1;
        }
    std::vector<int> slot(f->K, -1);
    std::vector<int> psf_ids;
    for (int k = 0; k < f->K; ++k)
        if (used[k]) { slot[k] = (int)psf_ids.size(); psf_ids.push_back(k); }
    const int nslots = std::max<int>(1, (int)psf_ids.size());
    f->tile_rows = std::max<int64_t>((int64_t)f->NQ * S + T, (int64_t)S + (int64_t)f->NQ * T);
    const size_t ntile_max = std::max(f->tH.size(), f->tHT.size());

    auto dalloc = [&](void **p, size_t bytes) {
        cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
        if (e == cudaSuccess) f->allocs.push_back(*p);
        return e;
    };
    FC(dalloc((void **)&f->W, sizeof(float2) * S));
    FC(dalloc((void **)&f->Hhat, sizeof(float2) * (size_t)nslots * S * LDF));
    FC(dalloc((void **)&f->scratch, sizeof(float2) * (size_t)ntile_max * f->tile_rows * LDF));
    FC(dalloc((void **)&f->psf_slot, sizeof(int) * f->K));
    FC(dalloc((void **)&f->d_tH, sizeof(TileDesc) * std::max<size_t>(1, f->tH.size())));
    FC(dalloc((void **)&f->d_tHT, sizeof(TileDesc) * std::max<size_t>(1, f->tHT.size())));
    f->nblk_inv = (T + (S >= 512 ? 8 : 16) - 1) / (S >= 512 ? 8 : 16);
    FC(dalloc((void **)&f->partials, sizeof(double) * std::max<size_t>(1, f->tH.size() * f->nblk_inv)));
    f->h_part.resize(std::max<size_t>(1, f->tH.size() * f->nblk_inv));
    // twiddles in fp64, rounded (A24)
    std::vector<float2> w(S);
    for (int k = 0; k < S; ++k) {
        const double ang = -2.0 * M_PI * (double)k / (double)S;
        w[k] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
    FC(cudaMemcpy(f->W, w.data(), sizeof(float2) * S, cudaMemcpyHostToDevice));
    FC(cudaMemcpy(f->psf_slot, slot.data(), sizeof(int) * f->K, cudaMemcpyHostToDevice));
    FC(cudaMemcpy(f->d_tH, f->tH.data(), sizeof(TileDesc) * f->tH.size(), cudaMemcpyHostToDevice));
    FC(cudaMemcpy(f->d_tHT, f->tHT.data(), sizeof(TileDesc) * f->tHT.size(), cudaMemcpyHostToDevice));
    FC(do_attrs(S, T));
    // PSF spectra Hhat_k = DFT2(h_k zero-padded to S x S), for every PSF a local tile touches
    if (!psf_ids.empty()) {
        float *d_sel = nullptr;
        float2 *hrows = nullptr;
        FC(cudaMalloc((void **)&d_sel, sizeof(float) * psf_ids.size() * P * P));
        FC(cudaMalloc((void **)&hrows, sizeof(float2) * psf_ids.size() * S * LDF));
        for (size_t i = 0; i < psf_ids.size(); ++i)
            FC(cudaMemcpyAsync(d_sel + i * P * P, d_psfs + (size_t)psf_ids[i] * P * P, sizeof(float) * P * P,
                               cudaMemcpyDeviceToDevice, s));
        FftArgs a = f->args(nullptr, false);
        const int n = (int)psf_ids.size();
        FC(do_rows_fwd(S, a, n, 2, 0, d_sel, n, hrows, s));
        FC(do_cols(S, a, n, 2, hrows, f->Hhat, n, s));
        FC(cudaStreamSynchronize(s));
        cudaFree(d_sel);
        cudaFree(hrows);
    }
#undef FC
    return f;
}

void fft_destroy(FftPlan *f) { delete f; }

cudaError_t fft_H(FftPlan &f, const FacetDev *d_facets, int par, int mode, cudaStream_t s) {
    FftArgs a = f.args(d_facets, false);
    const int n = (int)f.tH.size();
    cudaError_t e;
    if ((e = do_rows_fwd(f.S, a, n, 0, par, nullptr, 0, nullptr, s)) != cudaSuccess) return e;
    if ((e = do_cols(f.S, a, n, 0, nullptr, nullptr, 0, s)) != cudaSuccess) return e;
    return do_rows_inv(f.S, a, n, f.T, mode, s);
}

cudaError_t fft_HT(FftPlan &f, const FacetDev *d_facets, cudaStream_t s) {
    FftArgs a = f.args(d_facets, true);
    const int n = (int)f.tHT.size();
    cudaError_t e;
    if ((e = do_rows_fwd(f.S, a, n, 1, 0, nullptr, 0, nullptr, s)) != cudaSuccess) return e;
    if ((e = do_cols(f.S, a, n, 1, nullptr, nullptr, 0, s)) != cudaSuccess) return e;
    return do_rows_inv(f.S, a, n, f.T, INV_HT, s);
}

cudaError_t fft_data_partials(FftPlan &f, std::vector<double> &out) {
    out.assign(f.nlocal, 0.0);
    const size_t n = f.tH.size() * f.nblk_inv;
    cudaError_t e = cudaMemcpy(f.h_part.data(), f.partials, sizeof(double) * n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return e;
    for (size_t b = 0; b < n; ++b) out[f.tile_facet_H[b / f.nblk_inv]] += f.h_part[b];
    return cudaSuccess;
}

}  // namespace deblur
