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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include <cuda_pipeline.h>

#include "epilogue.cuh"
#include "fft.hpp"

// Tuning constants (each measured on c4, B200; alternatives in profiles/r1/SUMMARY.md and
// profiles/r2/SUMMARY.md).  The row passes keep S/2 + 2 twiddles (a length-S/2 plan over an
// S table uses W^k, k < S/2, and the R2C / C2R pre/post twiddles W^k, k <= S/2); the TMEM
// column pass keeps S/2 (a length-S plan uses W^k, k < S/2).
#define ROWS_TW(S) ((S) / 2 + 2)
#define COLS_TM_TW (S / 2)
constexpr int COLS_TM_NB = 8;      // columns per CTA of the TMEM column pass (256 threads, 16 elements each)
constexpr int COLS_TM_CPB = 4;     // column chunks per CTA (while the grid keeps >= 4 waves of 2 CTAs/SM)
constexpr int COLS_TM_MINB = 2;    // CTAs per SM (128 registers, ~80 KB smem)


namespace deblur {

namespace {

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
    int NP;                 // max active p per tile (wy rows staged per CTA)
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
// The R2C post step and the C2R pre step omit their factors 1/2: every spectrum between
// the passes (and the PSF spectra) is 2x the DFT, and the C2R output 8x the operator's
// value; the epilogue scale absorbs the 1/8 (FftArgs::scale).  Powers of two are exact,
// so the results are bit-identical to the textbook form.
// R2C post step for bin k from Z_k, Z_{SH-k} and W_S^k: 2 X_k = (Z_k + Z*_{SH-k}) - i W^k (Z_k - Z*_{SH-k})
__device__ __forceinline__ float2 r2c_post(float2 zk, float2 zp, float2 w) {
    const float2 sh = make_float2(zk.x + zp.x, zk.y - zp.y);
    const float2 d = make_float2(zk.x - zp.x, zk.y + zp.y);
    const float2 wd = cmul(w, d);
    return make_float2(sh.x + wd.y, sh.y - wd.x);
}
// C2R pre step for bin k from X_k, X_{SH-k} and W_S^k: 2 (E + i O) with 2 E = X_k + X*_{SH-k},
// 2 O = (X_k - X*_{SH-k}) conj(W^k)
__device__ __forceinline__ float2 c2r_pre(float2 xk, float2 xp, float2 w) {
    const float2 e = make_float2(xk.x + xp.x, xk.y - xp.y);
    const float2 d = make_float2(xk.x - xp.x, xk.y + xp.y);
    const float2 o = cmul(d, conjf2(w));
    return make_float2(e.x - o.y, e.y + o.x);
}
// Both bins of a C2R pre pair from one product: 2 (E + i O)_{SH-k} = conj(e) + i conj(o)
__device__ __forceinline__ void c2r_pre_pair(float2 xk, float2 xp, float2 w, float2 &zk, float2 &zp) {
    const float2 e = make_float2(xk.x + xp.x, xk.y - xp.y);
    const float2 d = make_float2(xk.x - xp.x, xk.y + xp.y);
    const float2 o = cmul(d, conjf2(w));
    zk = make_float2(e.x - o.y, e.y + o.x);
    zp = make_float2(e.x + o.y, o.x - e.y);
}
// Both bins of an R2C post pair from one product: with W^{SH-k} = -conj W^k the (SH - k)
// output's product is the conjugate of bin k's, so 2 X_{SH-k} = conj(sh) - i conj(W d)
// (12 instructions per pair instead of 20).
__device__ __forceinline__ void r2c_post_pair(float2 zk, float2 zp, float2 w, float2 &xk, float2 &xp) {
    const float2 sh = make_float2(zk.x + zp.x, zk.y - zp.y);
    const float2 d = make_float2(zk.x - zp.x, zk.y + zp.y);
    const float2 wd = cmul(w, d);
    xk = make_float2(sh.x + wd.y, sh.y - wd.x);
    xp = make_float2(sh.x - wd.y, -sh.y - wd.x);
}

// v * (SIGN < 0 ? -i : +i)
template <int SIGN>
__device__ __forceinline__ float2 rot90(float2 v) {
    return SIGN < 0 ? make_float2(v.y, -v.x) : make_float2(-v.y, v.x);
}

template <int SIGN>
__device__ __forceinline__ void dft2(float2 &a, float2 &b) {
    const float2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

// X_k = sum_n a_n e^{SIGN 2 pi i n k / 4}
template <int SIGN>
__device__ __forceinline__ void dft4(float2 &a0, float2 &a1, float2 &a2, float2 &a3) {
    const float2 s0 = cadd(a0, a2), d0 = csub(a0, a2);
    const float2 s1 = cadd(a1, a3), d1 = rot90<SIGN>(csub(a1, a3));
    a0 = cadd(s0, s1);
    a2 = csub(s0, s1);
    a1 = cadd(d0, d1);
    a3 = csub(d0, d1);
}

// Radix-8 DFT from its first-level pair sums / differences: s0, d0 = a0 +- a4 and
// s1, m1 = a2 +- a6 of the even inputs, S0, D0 = a1 +- a5 and S1, M1 = a3 +- a7 of the odd
// ones.  The w8^1, w8^3 products (r = sqrt(1/2)) are folded into the last additions as
// FMAs (6 instructions per product-and-butterfly instead of 8).
template <int SIGN>
__device__ __forceinline__ void dft8_tail(float2 &v0, float2 &v1, float2 &v2, float2 &v3, float2 &v4, float2 &v5,
                                          float2 &v6, float2 &v7, float2 s0, float2 d0, float2 s1, float2 m1,
                                          float2 S0, float2 D0, float2 S1, float2 M1) {
    const float r = 0.70710678118654752f;
    const float2 d1 = rot90<SIGN>(m1), D1 = rot90<SIGN>(M1);
    const float2 e0 = cadd(s0, s1), e2 = csub(s0, s1), e1 = cadd(d0, d1), e3 = csub(d0, d1);
    const float2 o0 = cadd(S0, S1), o2 = rot90<SIGN>(csub(S0, S1)), o1 = cadd(D0, D1), o3 = csub(D0, D1);
    v0 = cadd(e0, o0); v4 = csub(e0, o0);
    v2 = cadd(e2, o2); v6 = csub(e2, o2);
    // w8^1 o1 = r (o1.x - SIGN o1.y, o1.y + SIGN o1.x)
    const float p1 = o1.x - SIGN * o1.y, q1 = o1.y + SIGN * o1.x;
    v1 = make_float2(__fmaf_rn(r, p1, e1.x), __fmaf_rn(r, q1, e1.y));
    v5 = make_float2(__fmaf_rn(-r, p1, e1.x), __fmaf_rn(-r, q1, e1.y));
    // w8^3 o3 = (-r (o3.x + SIGN o3.y), r (SIGN o3.x - o3.y))
    const float p3 = o3.x + SIGN * o3.y, q3 = SIGN * o3.x - o3.y;
    v3 = make_float2(__fmaf_rn(-r, p3, e3.x), __fmaf_rn(r, q3, e3.y));
    v7 = make_float2(__fmaf_rn(r, p3, e3.x), __fmaf_rn(-r, q3, e3.y));
}

template <int SIGN>
__device__ __forceinline__ void dft8(float2 &v0, float2 &v1, float2 &v2, float2 &v3, float2 &v4, float2 &v5,
                                     float2 &v6, float2 &v7) {
    dft8_tail<SIGN>(v0, v1, v2, v3, v4, v5, v6, v7, cadd(v0, v4), csub(v0, v4), cadd(v2, v6), csub(v2, v6),
                    cadd(v1, v5), csub(v1, v5), cadd(v3, v7), csub(v3, v7));
}

// a_n * w_n (w real) followed by the radix-8 DFT, the weights folded into the first-level
// sums: w_a a + w_b b = fma(w_b, b, w_a a) (3 instructions per component pair instead of 4)
__device__ __forceinline__ void wpair(float2 a, float2 b, float wa, float wb, float2 &s, float2 &d) {
    const float2 t = make_float2(wa * a.x, wa * a.y);
    s = make_float2(__fmaf_rn(wb, b.x, t.x), __fmaf_rn(wb, b.y, t.y));
    d = make_float2(__fmaf_rn(-wb, b.x, t.x), __fmaf_rn(-wb, b.y, t.y));
}
template <int SIGN>
__device__ __forceinline__ void dft8w(float2 *v, const float (&w)[8]) {
    float2 s0, d0, s1, m1, S0, D0, S1, M1;
    wpair(v[0], v[4], w[0], w[4], s0, d0);
    wpair(v[2], v[6], w[2], w[6], s1, m1);
    wpair(v[1], v[5], w[1], w[5], S0, D0);
    wpair(v[3], v[7], w[3], w[7], S1, M1);
    dft8_tail<SIGN>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], s0, d0, s1, m1, S0, D0, S1, M1);
}

// Radix plans.  For L >= 64 the first and the last stage are radix 8, so the
// elements a thread produces in the last stage of one transform are exactly the
// ones it consumes in the first stage of the next (accumulators stay in registers).
// MAP = 2 (the forward row passes at L = 256): radix 16 x 16, one exchange per transform.
__host__ __device__ constexpr int fft_nst(int L, int MAP = 0) {
    return (MAP == 2 && (L == 256 || L == 128)) ? 2
         : L == 16 ? 2 : L == 32 ? 2 : L == 64 ? 2 : L == 128 ? 3 : L == 256 ? 3 : L == 512 ? 3 : L == 1024 ? 4 : 0;
}
__host__ __device__ constexpr int fft_rad(int L, int s, int MAP = 0) {
    return (MAP == 2 && L == 256) ? 16
         : (MAP == 2 && L == 128) ? (s == 0 ? 16 : 8)
         : L == 16 ? 4
         : L == 32 ? (s == 0 ? 8 : 4)
         : L == 64 ? 8
         : L == 128 ? (s == 1 ? 2 : 8)
         : L == 256 ? (s == 1 ? 4 : 8)
         : L == 512 ? 8
         : ((s == 1 || s == 2) ? 4 : 8);
}
__host__ __device__ constexpr int fft_ns(int L, int s, int MAP = 0) {
    return s == 0 ? 1 : fft_ns(L, s - 1, MAP) * fft_rad(L, s - 1, MAP);
}

// X_k = sum_n a_n e^{SIGN 2 pi i n k / 16}: two radix-8 halves (even / odd n) and one
// radix-2 combination with w16^k folded into FMAs
template <int SIGN>
__device__ __forceinline__ void dft16(float2 *v) {
    float2 e[8], o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { e[k] = v[2 * k]; o[k] = v[2 * k + 1]; }
    dft8<SIGN>(e[0], e[1], e[2], e[3], e[4], e[5], e[6], e[7]);
    dft8<SIGN>(o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
    const float c1 = 0.92387953251128676f, s1 = 0.38268343236508977f, r = 0.70710678118654752f;
    // w16^k = (cos 2 pi k / 16, SIGN sin 2 pi k / 16), k = 0..7
    const float wr[8] = {1.f, c1, r, s1, 0.f, -s1, -r, -c1};
    const float wi[8] = {0.f, SIGN * s1, SIGN * r, SIGN * c1, (float)SIGN, SIGN * c1, SIGN * r, SIGN * s1};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float2 a = o[k], ek = e[k];
        if (k == 0) {
            v[0] = cadd(ek, a);
            v[8] = csub(ek, a);
        } else if (k == 4) {
            const float2 t = rot90<SIGN>(a);
            v[4] = cadd(ek, t);
            v[12] = csub(ek, t);
        } else {
            v[k] = make_float2(__fmaf_rn(a.x, wr[k], __fmaf_rn(-a.y, wi[k], ek.x)),
                               __fmaf_rn(a.x, wi[k], __fmaf_rn(a.y, wr[k], ek.y)));
            v[k + 8] = make_float2(__fmaf_rn(-a.x, wr[k], __fmaf_rn(a.y, wi[k], ek.x)),
                                   __fmaf_rn(-a.x, wi[k], __fmaf_rn(-a.y, wr[k], ek.y)));
        }
    }
}

// Twiddle providers for the stages with Ns > 1: get<Ns, R>(i, j, w) fills w[1..R-1] =
// W_L^{r k}, k = j % Ns, for butterfly j (the thread's i-th of the stage).
// TwTable: w, w^2, w^4 from the fp64-built table in shared memory, the rest by at most
// two products (<= ~2 ulp), saving shared-memory loads.
struct TwTable {
    const float2 *W;
    int S;
    template <int Ns>
    __device__ __forceinline__ TwTable pre() const { return *this; }
    __device__ __forceinline__ void ready() const {}
    template <int Ns, int R>
    __device__ __forceinline__ void get(int, int j, float2 (&w)[8]) const {
        const int k = j % Ns;
        const int step = S / (Ns * R);
        w[1] = W[(k * step) & (S - 1)];
        if (R >= 4) {
            w[2] = W[(2 * k * step) & (S - 1)];
            w[3] = cmul(w[1], w[2]);
        }
        if (R == 8) {
            w[4] = W[(4 * k * step) & (S - 1)];
            w[5] = cmul(w[4], w[1]);
            w[6] = cmul(w[4], w[2]);
            w[7] = cmul(w[4], w[3]);
        }
    }
    // radix 16: w, w^2, w^4, w^8 from the table, the rest by at most three products
    template <int Ns>
    __device__ __forceinline__ void get16(int j, float2 (&w)[16]) const {
        const int k = j % Ns;
        const int step = S / (Ns * 16);
        w[1] = W[(k * step) & (S - 1)];
        w[2] = W[(2 * k * step) & (S - 1)];
        w[4] = W[(4 * k * step) & (S - 1)];
        w[8] = W[(8 * k * step) & (S - 1)];
        w[3] = cmul(w[1], w[2]);
#pragma unroll
        for (int q = 5; q < 8; ++q) w[q] = cmul(w[4], w[q - 4]);
#pragma unroll
        for (int q = 9; q < 16; ++q) w[q] = cmul(w[8], w[q - 8]);
    }
};

// One Stockham stage of NB batched length-L transforms at buf[t*STRIDE + n] executed
// by NTH threads.  Thread tid owns transform t = tid % NB (transform-fastest: a
// quarter-/half-warp touches 8/16 transforms at one position, which the padded
// STRIDE spreads over distinct banks) and the BPT consecutive butterflies
// j = (tid / NB) * BPT + i.  Consecutive butterflies read and write adjacent
// positions, so with an even STRIDE the exchanges move element pairs with 16-byte
// shared-memory accesses (VEC): half the LDS/STS instructions of 8-byte accesses.
//
// MAP = 2 (the row passes at L = 256: 16 rows x 16 threads of 16 elements): radix 16 x 16,
// one butterfly per thread per stage; t = (tid & 7) | (tid >> 7) << 3, j = (tid >> 3) & 15,
// so a half-warp is 8 rows x 2 consecutive butterflies and the 8-byte exchanges are
// conflict-free with the even row stride the paired 16-byte paths need.
template <int L, int NB, int STRIDE, int NTH, int s, int MAP = 0>
struct Stage {
    static constexpr bool MIR = MAP != 0;
    static constexpr int R = fft_rad(L, s, MAP), Ns = fft_ns(L, s, MAP), LR = L / R, NS = fft_nst(L, MAP);
    static constexpr int E = NB * L / NTH, BPT = E / R;
    static_assert(E % R == 0, "elements per thread must be a multiple of the radix");
    static_assert(NTH * BPT * R == NB * L, "thread/butterfly mapping");
    // MAP 2: 16 x L/16 (L = 256 or 128), L/16 threads per transform, 8 <= NB <= 16 transforms
    static constexpr int TPR = L / 16, JB = TPR == 16 ? 4 : 3;
    static_assert(!MIR || (MAP == 2 && (L == 256 || L == 128) && NTH == TPR * NB && NB >= 8 && NB <= 16), "radix 16 plans");
    static constexpr bool VEC = (STRIDE % 2 == 0) && (BPT % 2 == 0) && (LR % 2 == 0);
    // outputs r, r + 1 of one first-stage butterfly are adjacent for any butterfly mapping
    static constexpr bool VEC0 = (VEC || MIR) && Ns == 1 && STRIDE % 2 == 0 && R % 2 == 0;
    __device__ static __forceinline__ void bj(int i, int tid, int &t, int &j) {
        if constexpr (MIR) {
            t = (tid & 7) | ((tid >> (3 + JB)) << 3);
            j = ((tid >> 3) & (TPR - 1)) * BPT + i;
        } else {
            t = tid % NB;
            j = (tid / NB) * BPT + i;
        }
    }
    __device__ static __forceinline__ int in_n(int j, int r) { return j + r * LR; }
    __device__ static __forceinline__ int out_n(int j, int r) { return (j / Ns) * Ns * R + (j % Ns) + r * Ns; }
    template <int SIGN, class TW>
    __device__ static __forceinline__ void bfly_tw(float2 *v, int i, int j, const TW &tw) {
        if constexpr (R == 16) {
            if constexpr (Ns > 1) {
                float2 w[16];
                tw.template get16<Ns>(j, w);
#pragma unroll
                for (int r = 1; r < 16; ++r) {
                    float2 ww = w[r];
                    if (SIGN > 0) ww.y = -ww.y;
                    v[r] = cmul(v[r], ww);
                }
            }
            dft16<SIGN>(v);
            return;
        }
        if (Ns > 1) {
            float2 w[8];
            tw.template get<Ns, R>(i, j, w);
#pragma unroll
            for (int r = 1; r < R; ++r) {
                float2 ww = w[r];
                if (SIGN > 0) ww.y = -ww.y;
                v[r] = cmul(v[r], ww);
            }
        }
        if (R == 8) dft8<SIGN>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
        else if (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
        else dft2<SIGN>(v[0], v[1]);
    }
    template <int SIGN>
    __device__ static __forceinline__ void bfly(float2 *v, int j, const float2 *W, int S) {
        bfly_tw<SIGN>(v, 0, j, TwTable{W, S});
    }
    template <int SIGN, class TW>
    __device__ static __forceinline__ void load_bfly_tw(const float2 *buf, float2 (&v)[E], int tid, const TW &tw) {
        if constexpr (VEC) {
            // butterflies (i, i+1) read the adjacent positions (n, n+1)
#pragma unroll
            for (int i = 0; i < BPT; i += 2) {
                int t, j;
                bj(i, tid, t, j);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 q = *reinterpret_cast<const float4 *>(buf + t * STRIDE + in_n(j, r));
                    v[i * R + r] = make_float2(q.x, q.y);
                    v[(i + 1) * R + r] = make_float2(q.z, q.w);
                }
                bfly_tw<SIGN>(&v[i * R], i, j, tw);
                bfly_tw<SIGN>(&v[(i + 1) * R], i + 1, j + 1, tw);
            }
        } else {
#pragma unroll
            for (int i = 0; i < BPT; ++i) {
                int t, j;
                bj(i, tid, t, j);
#pragma unroll
                for (int r = 0; r < R; ++r) v[i * R + r] = buf[t * STRIDE + in_n(j, r)];
                bfly_tw<SIGN>(&v[i * R], i, j, tw);
            }
        }
    }
    template <int SIGN>
    __device__ static __forceinline__ void load_bfly(const float2 *buf, float2 (&v)[E], int tid, const float2 *W, int S) {
        load_bfly_tw<SIGN>(buf, v, tid, TwTable{W, S});
    }
    __device__ static __forceinline__ void store(float2 *buf, const float2 (&v)[E], int tid) {
        if constexpr (VEC0) {
            // first stage: outputs r, r+1 of one butterfly are adjacent
#pragma unroll
            for (int i = 0; i < BPT; ++i) {
                int t, j;
                bj(i, tid, t, j);
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const float2 a = v[i * R + r], b = v[i * R + r + 1];
                    *reinterpret_cast<float4 *>(buf + t * STRIDE + out_n(j, r)) = make_float4(a.x, a.y, b.x, b.y);
                }
            }
        } else if constexpr (VEC) {
            // later stages: output r of butterflies j, j+1 (j even) are adjacent
#pragma unroll
            for (int i = 0; i < BPT; i += 2) {
                int t, j;
                bj(i, tid, t, j);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float2 a = v[i * R + r], b = v[(i + 1) * R + r];
                    *reinterpret_cast<float4 *>(buf + t * STRIDE + out_n(j, r)) = make_float4(a.x, a.y, b.x, b.y);
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < BPT; ++i) {
                int t, j;
                bj(i, tid, t, j);
#pragma unroll
                for (int r = 0; r < R; ++r) buf[t * STRIDE + out_n(j, r)] = v[i * R + r];
            }
        }
    }
};

// stages 1 .. NS-1 with exchanges through `work`; v holds stage-0 outputs on entry
// and last-stage outputs on exit.  Contains the barriers it needs.
// TAIL = false drops the barrier after the last stage's loads, for callers whose next
// write to `work` comes after a barrier of their own.
template <int L, int NB, int STRIDE, int NTH, int SIGN, int s, int NS, bool TAIL = true, int MIR = 0>
struct Mid {
    static constexpr int E = NB * L / NTH;
    template <class TW>
    __device__ static __forceinline__ void run(float2 *work, float2 (&v)[E], int tid, const TW &tw) {
        Stage<L, NB, STRIDE, NTH, s - 1, MIR>::store(work, v, tid);
        // the stage's twiddles (a TMEM provider issues its loads here, under the barrier)
        auto tws = tw.template pre<Stage<L, NB, STRIDE, NTH, s, MIR>::Ns>();
        __syncthreads();
        tws.ready();
        Stage<L, NB, STRIDE, NTH, s, MIR>::template load_bfly_tw<SIGN>(work, v, tid, tws);
        if (TAIL || s + 1 < NS) __syncthreads();
        Mid<L, NB, STRIDE, NTH, SIGN, s + 1, NS, TAIL, MIR>::run(work, v, tid, tw);
    }
};
template <int L, int NB, int STRIDE, int NTH, int SIGN, int NS, bool TAIL, int MIR>
struct Mid<L, NB, STRIDE, NTH, SIGN, NS, NS, TAIL, MIR> {
    static constexpr int E = NB * L / NTH;
    template <class TW>
    __device__ static __forceinline__ void run(float2 *, float2 (&)[E], int, const TW &) {}
};

template <int L, int NB, int STRIDE, int NTH, int MIR = 0>
struct Fft {
    static constexpr int NS = fft_nst(L, MIR);
    static constexpr int E = NB * L / NTH;
    using First = Stage<L, NB, STRIDE, NTH, 0, MIR>;
    using Last = Stage<L, NB, STRIDE, NTH, NS - 1, MIR>;
    template <int SIGN>
    __device__ static __forceinline__ void middle(float2 *work, float2 (&v)[E], int tid, const float2 *W, int S) {
        Mid<L, NB, STRIDE, NTH, SIGN, 1, NS, true, MIR>::run(work, v, tid, TwTable{W, S});
    }
    template <int SIGN, class TW>
    __device__ static __forceinline__ void middle_tw(float2 *work, float2 (&v)[E], int tid, const TW &tw) {
        Mid<L, NB, STRIDE, NTH, SIGN, 1, NS, true, MIR>::run(work, v, tid, tw);
    }
    // without the trailing barrier (the caller's next write to `work` follows a barrier)
    template <int SIGN, class TW>
    __device__ static __forceinline__ void middle_open(float2 *work, float2 (&v)[E], int tid, const TW &tw) {
        Mid<L, NB, STRIDE, NTH, SIGN, 1, NS, false, MIR>::run(work, v, tid, tw);
    }
};

// geometry of the row passes (length SH complex transforms, NBR rows per CTA)
template <int S>
struct GR {
    static constexpr int SH = S / 2;
    // 128 threads at S = 256 (the strip plan): 16 elements per thread, paired 16-byte exchanges
    static constexpr int NTH = S == 256 ? 128 : 256;
    static constexpr int NB = (S <= 64) ? 64 : (S <= 128) ? 32 : 16;
    static constexpr int RS = SH + 2;    // smem row stride (float2): even (16-byte pair exchanges), conflict-free
    // smem real-row stride (floats): 4 banks per row for the row mapping's 8-byte accesses
    // radix 16 x SH/16 with the row mapping at S = 512 (256 threads) and S = 256 (128)
    static constexpr bool MIR = (SH == 256 || SH == 128) && NB == 16 && NTH == NB * SH / 16;
    static constexpr int XS = S + (MIR ? 4 : 2);
    using F = Fft<SH, NB, RS, NTH, MIR ? 2 : 0>;
    static constexpr int E = F::E;
};
// geometry of the column pass (length S complex transforms, NBC columns per CTA)
template <int S>
struct GC {
    // 8 columns per CTA from S = 256 up; at S = 256 (the strip plan) 128 threads of 16
    // elements (paired 16-byte exchanges, 4 CTAs/SM), at S = 512 256 threads
    static constexpr int NTH = (S <= 128) ? 512 : (S == 256) ? 128 : 256;
    static constexpr int MINB = (S == 256 && NTH == 128) ? 4 : 1;
    static constexpr int NB = (S <= 64) ? 64 : (S <= 128) ? 32 : (S == 512) ? COLS_TM_NB : 8;
    static constexpr int CS = S + ((NB >= 16) ? 1 : 16 / NB);
    // S = 256: radix 16 x 16 (one exchange per transform), the row passes' thread mapping
    using F = Fft<S, NB, CS, NTH, S == 256 ? 2 : 0>;
    static constexpr int E = F::E;
};
template <int S>
struct LD {
    static constexpr int LDF = S / 2 + GC<S>::NB;   // padded spectrum row length (float2)
};

// tensor-memory helpers (32x32b shape: each thread its own lane, consecutive columns)
__device__ __forceinline__ void tm_st32(uint32_t ta, const uint32_t (&r)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31};\n" :: "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(ta) : "memory");
}
__device__ __forceinline__ void tm_ld32(uint32_t ta, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(ta) : "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t ta, const uint32_t (&r)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15};\n" :: "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(ta) : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(ta) : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t ta, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%8], {%0, %1, %2, %3, %4, %5, %6, %7};\n" :: "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(ta) : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// E = 16 complex per thread <-> 32 TMEM columns
template <int E>
__device__ __forceinline__ void tm_put(uint32_t ta, const float2 (&v)[E]) {
    static_assert(E == 16, "TMEM column pass holds 16 complex per thread");
    uint32_t r[32];
#pragma unroll
    for (int e = 0; e < E; ++e) { r[2 * e] = __float_as_uint(v[e].x); r[2 * e + 1] = __float_as_uint(v[e].y); }
    tm_st32(ta, r);
}
template <int E>
__device__ __forceinline__ void tm_get(uint32_t ta, float2 (&v)[E]) {
    uint32_t r[32];
    tm_ld32(ta, r);
    tm_wait_ld();
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = make_float2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
}

// ------------------------------------------------------------------ pass A / A'
// mode 0: H (x window . wx_q, one R2C per active q); 1: H^T (r window); 2: PSF spectra rows
// TMX: the mode-0 instantiation with the TMEM stash (a kernel containing tcgen05 code ran
// the other modes 2x slower, so they use the TMX = false instantiation)
template <int S, bool TMX>
__global__ void __launch_bounds__(GR<S>::NTH, S == 512 ? 4 : S == 1024 ? 2 : GR<S>::NTH == 128 ? 6 : 5) k_rows_fwd(FftArgs A, int mode, int par, const float *psfs, int npsf,
                                                  float2 *hrows) {
    using G = GR<S>;
    using F = typename G::F;
    constexpr int NB = G::NB, SH = G::SH, RS = G::RS, XS = G::XS, LDF = LD<S>::LDF;
    extern __shared__ __align__(16) float2 sm2[];
    float2 *Wsm = sm2;                                      // ROWS_TW(S) twiddles
    float2 *work = Wsm + ROWS_TW(S);                        // NB x RS
    // NB x XS real rows; at S = 512 with a single transform per CTA (modes 1, 2) they live in the
    // exchange buffer (stage 0 reads them before the barrier that precedes the first exchange
    // write): 4 CTAs/SM with <= 64 registers (H^T R2C 0.74 -> 0.62 ms)
    static_assert(NB * XS <= 2 * NB * RS, "xs fits in work");
    // Mode 0 (one transform per active q) at S = 512: each thread's stage-0 inputs are
    // stashed in TMEM (32 columns) once, so xs can alias work there too (37 KB smem)
    constexpr bool TMX_S = TMX;
    const bool tmx = TMX;                 // launched for mode 0 only
    float *xs = reinterpret_cast<float *>((S == 512 && (mode != 0 || tmx)) ? work : work + NB * RS);
    float *wxs = tmx ? reinterpret_cast<float *>(work + NB * RS) : xs + NB * XS;   // S
    __shared__ uint32_t tm_slot_x;
    const int tid = threadIdx.x;
    const int nblk = S / NB;
    const int tile = blockIdx.x / nblk, r0 = (blockIdx.x % nblk) * NB;
    const int P = A.P, c2 = P - 1;
    int nq = 1, q0 = 0;
    TileDesc t{};
    const FacetDev *Fd = nullptr;
    if (mode == 2) {
        if (tile >= npsf) return;
    } else {
        t = A.tiles[tile];
        Fd = &A.facets[t.f];
        if (mode == 0) { q0 = t.q0; nq = t.q1 - t.q0 + 1; }
    }
    if (tmx && (tid >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&tm_slot_x)), "n"(64) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    for (int i = tid; i < ROWS_TW(S); i += G::NTH) Wsm[i] = A.W[i];
    {
        // batched loads (all in flight before the first use): real rows of the window;
        // thread -> (row offset rt, column ct), the row / column bounds tested once each
        constexpr int NTH = G::NTH, LPT = NB * S / NTH;
        constexpr int CPR = S >= NTH ? S / NTH : 1, RPI = S >= NTH ? 1 : NTH / S;
        const float *src;
        int pitch, gy0, gx0, limy, limx;
        if (mode == 0) {
            src = Fd->x[par]; pitch = Fd->ep; gy0 = t.y0 + r0; gx0 = t.x0; limy = Fd->ny; limx = Fd->nx;
        } else if (mode == 1) {
            src = Fd->r; pitch = Fd->op; gy0 = t.y0 - c2 + r0; gx0 = t.x0 - c2; limy = Fd->my; limx = Fd->mx;
        } else {
            src = psfs + (int64_t)tile * P * P; pitch = P; gy0 = r0; gx0 = 0; limy = P; limx = P;
        }
        if (((gx0 | pitch) & 1) == 0 && ((uintptr_t)src & 7) == 0) {
            // column pairs: 8-byte loads (a pair straddling the right edge is loaded per element)
            constexpr int SP = S / 2, LP = LPT / 2;
            constexpr int CP2 = SP >= NTH ? SP / NTH : 1, RP2 = SP >= NTH ? 1 : NTH / SP;
            const int ct = SP >= NTH ? tid : tid % SP, rt = SP >= NTH ? 0 : tid / SP;
            const float *bp = src + (int64_t)(gy0 + rt) * pitch + gx0 + 2 * ct;
            int okx[CP2];      // 2: both columns in range, 1: the first only, 0: none
#pragma unroll
            for (int c = 0; c < CP2; ++c) {
                const int gx = gx0 + 2 * (ct + c * NTH);
                okx[c] = (gx >= 0 && gx < limx) + (gx + 1 >= 0 && gx + 1 < limx);
            }
            float2 vals[LP];
#pragma unroll
            for (int it = 0; it < LP; ++it) {
                const int ro = (it / CP2) * RP2, c = it % CP2, gy = gy0 + rt + ro;
                const float *pp = bp + ro * pitch + 2 * c * NTH;
                vals[it] = make_float2(0.f, 0.f);
                if (gy >= 0 && gy < limy) {
                    if (okx[c] == 2) vals[it] = __ldg(reinterpret_cast<const float2 *>(pp));
                    else if (okx[c] == 1) vals[it].x = __ldg(pp);
                }
            }
#pragma unroll
            for (int it = 0; it < LP; ++it) {
                const int ro = (it / CP2) * RP2, c = it % CP2;
                *reinterpret_cast<float2 *>(xs + (rt + ro) * XS + 2 * (ct + c * NTH)) = vals[it];
            }
        } else {
            const int ct = S >= NTH ? tid : tid % S, rt = S >= NTH ? 0 : tid / S;
            const float *bp = src + (int64_t)(gy0 + rt) * pitch + gx0 + ct;
            bool okx[CPR];
#pragma unroll
            for (int c = 0; c < CPR; ++c) okx[c] = gx0 + ct + c * NTH >= 0 && gx0 + ct + c * NTH < limx;
            float vals[LPT];
#pragma unroll
            for (int it = 0; it < LPT; ++it) {
                const int ro = (it / CPR) * RPI, c = it % CPR, gy = gy0 + rt + ro;
                vals[it] = (okx[c] && gy >= 0 && gy < limy) ? __ldg(bp + ro * pitch + c * NTH) : 0.f;
            }
#pragma unroll
            for (int it = 0; it < LPT; ++it) {
                const int ro = (it / CPR) * RPI, c = it % CPR;
                xs[(rt + ro) * XS + ct + c * NTH] = vals[it];
            }
        }
    }
    using S0 = typename F::First;
    uint32_t t_x = 0;
    if constexpr (TMX_S) {
        if (tmx) {
            static_assert(G::E == 16, "32 TMEM columns per thread");
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncthreads();                      // xs and the TMEM address visible
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const int warp = tid >> 5;
            t_x = tm_slot_x + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 32);
            float2 z[G::E];
#pragma unroll
            for (int i = 0; i < S0::BPT; ++i) {
                int tt, j;
                S0::bj(i, tid, tt, j);
#pragma unroll
                for (int r = 0; r < S0::R; ++r) z[i * S0::R + r] = *reinterpret_cast<const float2 *>(xs + tt * XS + 2 * S0::in_n(j, r));
            }
            tm_put<G::E>(t_x, z);
            tm_wait_st();
            __syncthreads();                      // xs (= work) readers done
        }
    }
    // wx_q of the next active q in flight during this q's transform (mode 0)
    constexpr int WPT = (S + G::NTH - 1) / G::NTH;
    float wpre[WPT];
    auto load_w = [&](int q) {
        const float *wxq = A.wx + (size_t)q * A.Nx + Fd->ex0 + t.x0;
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int i = tid + k * G::NTH;
            wpre[k] = (i < S && t.x0 + i < Fd->nx) ? __ldg(wxq + i) : 0.f;
        }
    };
    if (mode == 0 && nq > 0) load_w(q0);
    for (int qi = 0; qi < nq; ++qi) {
        if (mode == 0) {
            // the previous q's stage-0 readers of wxs passed a barrier since
#pragma unroll
            for (int k = 0; k < WPT; ++k)
                if (tid + k * G::NTH < S) wxs[tid + k * G::NTH] = wpre[k];
            if (qi + 1 < nq) load_w(q0 + qi + 1);
        }
        __syncthreads();
        // stage 0 straight from the real rows: z[n] = (x[2n] w[2n], x[2n+1] w[2n+1])
        float2 v[G::E];
        if constexpr (TMX_S) {
            if (tmx) tm_get<G::E>(t_x, v);
        }
#pragma unroll
        for (int i = 0; i < S0::BPT; ++i) {
            int tt, j;
            S0::bj(i, tid, tt, j);
#pragma unroll
            for (int r = 0; r < S0::R; ++r) {
                const int n = S0::in_n(j, r);
                float2 z = tmx ? v[i * S0::R + r] : *reinterpret_cast<const float2 *>(xs + tt * XS + 2 * n);
                if (mode == 0) {
                    const float2 w = *reinterpret_cast<const float2 *>(wxs + 2 * n);
                    z.x *= w.x;
                    z.y *= w.y;
                }
                v[i * S0::R + r] = z;
            }
            S0::template bfly<-1>(&v[i * S0::R], j, Wsm, S);
        }
        // stage 0 read xs, which aliases work at S = 512 outside the TMEM-stash variant: its
        // readers finish before middle() writes work (elsewhere stage 0 reads TMEM / a disjoint xs)
        if (S == 512 && !tmx) __syncthreads();
        F::template middle<-1>(work, v, tid, Wsm, S);
        F::Last::store(work, v, tid);
        __syncthreads();
        // R2C post-processing, one (k, SH - k) pair per item (both outputs read the same two
        // values; W^{SH-k} = -conj W^k); the self-paired k = SH/2 is done by the k = 0 item
        // thread -> fixed k, rows rr0, rr0 + RPP, ... (twiddles and row pointer set once)
        constexpr int HP = SH / 2, RPP = G::NTH / HP;
        static_assert(G::NTH % HP == 0 && NB % RPP == 0, "post-processing split");
        const int k = tid % HP, rr0 = tid / HP;
        const float2 w = Wsm[k], wc = make_float2(-w.x, w.y), wm = Wsm[HP];
        float2 *dst = (mode == 2) ? hrows + ((int64_t)tile * S + r0 + rr0) * LDF
                                  : A.scratch + (int64_t)tile * A.tile_rows * LDF + ((int64_t)qi * S + r0 + rr0) * LDF;
#pragma unroll 4
        for (int rr = rr0; rr < NB; rr += RPP, dst += RPP * LDF) {
            const float2 *wr = work + rr * RS;
            const float2 a = wr[k], b = wr[(SH - k) & (SH - 1)];
            r2c_post_pair(a, b, w, dst[k], dst[SH - k]);
            if (k == 0) {
                const float2 m = wr[HP];
                dst[HP] = r2c_post(m, m, wm);
            }
        }
    }
    if constexpr (TMX_S) {
        if (tmx) {
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncthreads();
            if ((tid >> 5) == 0)
                asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tm_slot_x), "n"(64) : "memory");
        }
    }
}

// ------------------------------------------------------------------ pass B / B'
// PSF spectra are stored with row pairs interleaved, in global memory
// (element (n, f) at ((n >> 1) * LDF + f) * 2 + (n & 1)) and in the shared chunk
// (element (n, t) at ((n >> 1) * NB + t) * 2 + (n & 1)): the values at rows n, n+1
// of one column -- which the paired butterflies (j, j+1) of a thread need -- are
// one 16-byte access, and a pair-row of a chunk is one contiguous 16*NB-byte run.
__host__ __device__ __forceinline__ int64_t hg_idx(int n, int64_t f, int LDF) { return (((int64_t)(n >> 1) * LDF + f) << 1) + (n & 1); }
template <int NB>
__device__ __forceinline__ int hb_idx(int n, int t) { return (((n >> 1) * NB + t) << 1) + (n & 1); }

// mbarrier + TMA (cp.async.bulk.tensor) helpers: one elected thread arms the barrier with
// the byte count and issues the tensor copy; consumers wait on the barrier's phase parity.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(m)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}\n" :: "r"(smem_u32(m)), "r"(parity) : "memory");
}
// 2-D tiled tensor copy global -> shared, completion counted on mbarrier m (expect_tx armed
// here by the issuing thread); the generic-proxy reads of dst before it (ordered by the
// caller's barrier) are fenced against the async-proxy write
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *m,
                                            uint32_t bytes) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(smem_u32(m)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(m))
                 : "memory");
}

// Hhat chunk (S rows x NB columns starting at f0) of spectrum Hk -> smem hbuf with cp.async
template <int S, int NB, int NTH, int LDF>
__device__ __forceinline__ void prefetch_hhat(float2 *hbuf, const float2 *Hk, int f0, int tid) {
    constexpr int V = NB;                     // 16-byte vectors per pair-row
    constexpr int N = (S / 2) * V;
#pragma unroll
    for (int it = 0; it < (N + NTH - 1) / NTH; ++it) {
        const int idx = tid + it * NTH;
        if (idx < N) {
            const int m = idx / V, v = idx % V;
            __pipeline_memcpy_async(hbuf + m * 2 * NB + 2 * v, Hk + (((int64_t)m * LDF + f0) << 1) + 2 * v, 16);
        }
    }
    __pipeline_commit();
}
// column S/2 (Nyquist) of a pair-interleaved PSF spectrum -> hn[0, S) (not committed: the
// prefetch_hhat that follows commits it with the chunk)
template <int S, int NTH, int LDF>
__device__ __forceinline__ void prefetch_hnyq(float2 *hn, const float2 *Hk, int tid) {
    for (int m = tid; m < S / 2; m += NTH)
        __pipeline_memcpy_async(hn + 2 * m, Hk + (((int64_t)m * LDF + S / 2) << 1), 16);
}
__device__ __forceinline__ float4 ld4(const float2 *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ float2 lo2(float4 q) { return make_float2(q.x, q.y); }
__device__ __forceinline__ float2 hi2(float4 q) { return make_float2(q.z, q.w); }

// mode 0: H; 1: H^T; 2: PSF spectra (forward column DFT of hrows -> Hhat)
template <int S>
__global__ void __launch_bounds__(GC<S>::NTH, GC<S>::MINB) k_cols(FftArgs A, int mode, const float2 *hrows, float2 *hhat, int npsf) {
    using G = GC<S>;
    using F = typename G::F;
    constexpr int NB = G::NB, CS = G::CS, E = G::E, LDF = LD<S>::LDF, NF = S / 2 + 1, NTH = G::NTH;
    using S0 = typename F::First;
    using SL = typename F::Last;
    static_assert(S0::R == SL::R, "first/last radix must match");
    extern __shared__ __align__(16) float2 sm2[];
    float2 *Wsm = sm2;               // S
    float2 *hbuf = Wsm + S;          // S x NB (prefetched PSF spectrum chunk)
    float2 *colq = hbuf + S * NB;    // NB x CS
    float2 *work = colq + NB * CS;   // NB x CS
    float *wys_all = reinterpret_cast<float *>(work + NB * CS);   // NP x S: every active wy_p of the tile
    int *slot_s = reinterpret_cast<int *>(wys_all + (size_t)A.NP * S);   // NP x NQ PSF-spectrum slots
    const int tid = threadIdx.x;
    const int nchunk = (NF + NB - 1) / NB;
    const int tile = blockIdx.x / nchunk, f0 = (blockIdx.x % nchunk) * NB;
    const int P = A.P, c2 = P - 1, T = S - P + 1;
    for (int i = tid; i < S; i += NTH) Wsm[i] = A.W[i];
    float2 v[E];

    if (mode == 2) {
        __syncthreads();
        if (tile >= npsf) return;
        const float2 *src = hrows + (int64_t)tile * S * LDF + f0;
#pragma unroll
        for (int i = 0; i < S0::BPT; ++i) {
            int t, j;
            S0::bj(i, tid, t, j);
#pragma unroll
            for (int r = 0; r < S0::R; ++r) v[i * S0::R + r] = src[(int64_t)S0::in_n(j, r) * LDF + t];
            S0::template bfly<-1>(&v[i * S0::R], j, Wsm, S);
        }
        F::template middle<-1>(work, v, tid, Wsm, S);
        float2 *dst = hhat + (int64_t)tile * S * LDF;
#pragma unroll
        for (int i = 0; i < SL::BPT; ++i) {
            int t, j;
            SL::bj(i, tid, t, j);
#pragma unroll
            for (int r = 0; r < SL::R; ++r) dst[hg_idx(SL::out_n(j, r), f0 + t, LDF)] = v[i * SL::R + r];
        }
        return;
    }

    const TileDesc td = A.tiles[tile];
    const FacetDev &Fd = A.facets[td.f];
    float2 *base = A.scratch + (int64_t)tile * A.tile_rows * LDF;
    {
        // stage every active row weight wy_p and PSF slot once per CTA: no global
        // latency is exposed inside the (p, q) loops
        const int np = td.p1 - td.p0 + 1, nq = td.q1 - td.q0 + 1;
        for (int idx = tid; idx < np * S; idx += NTH) {
            const int pi = idx / S, i = idx - pi * S;
            // (H^T weights its outputs: rows >= T, which are dropped, get weight 0)
            wys_all[idx] = (td.y0 + i < Fd.ny && (mode == 0 || i < T))
                               ? __ldg(A.wy + (size_t)(td.p0 + pi) * A.Ny + Fd.ey0 + td.y0 + i) : 0.f;
        }
        for (int idx = tid; idx < np * nq; idx += NTH) {
            const int pi = idx / nq, qi = idx - pi * nq;
            slot_s[idx] = __ldg(A.psf_slot + (td.p0 + pi) * A.Gx + td.q0 + qi);
        }
    }
    __syncthreads();
    const int nqt = td.q1 - td.q0 + 1;
    auto hk = [&](int p, int q) { return A.Hhat + (int64_t)slot_s[(p - td.p0) * nqt + (q - td.q0)] * S * LDF; };
    constexpr bool VP = S0::VEC && SL::VEC;        // paired 16-byte accesses
    const float *wys = wys_all;
    auto fill_wys = [&](int p) { wys = wys_all + (size_t)(p - td.p0) * S; };

    if (mode == 0) {
        float2 acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = make_float2(0.f, 0.f);
        for (int q = td.q0; q <= td.q1; ++q) {
            // (colq is free: every stage-0 read of the previous q precedes a barrier in middle())
            {   // batched load of the row-spectrum chunk of A_q
                constexpr int LPT = NB * S / NTH;
                const float2 *Aq = base + (int64_t)(q - td.q0) * S * LDF + f0;
                float2 tmp[LPT];
#pragma unroll
                for (int it = 0; it < LPT; ++it) {
                    const int idx = tid + it * NTH;
                    tmp[it] = __ldg(Aq + (int64_t)(idx / NB) * LDF + (idx % NB));
                }
#pragma unroll
                for (int it = 0; it < LPT; ++it) {
                    const int idx = tid + it * NTH;
                    colq[(idx % NB) * CS + idx / NB] = tmp[it];
                }
            }
            for (int p = td.p0; p <= td.p1; ++p) {
                __syncthreads();
                prefetch_hhat<S, NB, NTH, LDF>(hbuf, hk(p, q), f0, tid);   // overlaps the FFT below
                fill_wys(p);
                // stage 0 from colq, weighted by the row weight wy_p (constant along the row)
                if constexpr (VP) {
#pragma unroll
                    for (int i = 0; i < S0::BPT; i += 2) {
                        int t, j;
                        S0::bj(i, tid, t, j);
#pragma unroll
                        for (int r = 0; r < S0::R; ++r) {
                            const int n = S0::in_n(j, r);
                            const float4 c = ld4(colq + t * CS + n);
                            const float2 wv = *reinterpret_cast<const float2 *>(wys + n);
                            v[i * S0::R + r] = make_float2(wv.x * c.x, wv.x * c.y);
                            v[(i + 1) * S0::R + r] = make_float2(wv.y * c.z, wv.y * c.w);
                        }
                        S0::template bfly<-1>(&v[i * S0::R], j, Wsm, S);
                        S0::template bfly<-1>(&v[(i + 1) * S0::R], j + 1, Wsm, S);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < S0::BPT; ++i) {
                        int t, j;
                        S0::bj(i, tid, t, j);
                        float wv[S0::R];
#pragma unroll
                        for (int r = 0; r < S0::R; ++r) {
                            const int n = S0::in_n(j, r);
                            v[i * S0::R + r] = colq[t * CS + n];
                            wv[r] = wys[n];
                        }
                        if constexpr (S0::R == 8 && S0::Ns == 1) {
                            const float (&w8)[8] = reinterpret_cast<const float (&)[8]>(wv);
                            dft8w<-1>(&v[i * S0::R], w8);              // weights folded into the first level
                        } else {
#pragma unroll
                            for (int r = 0; r < S0::R; ++r) {
                                v[i * S0::R + r].x *= wv[r];
                                v[i * S0::R + r].y *= wv[r];
                            }
                            S0::template bfly<-1>(&v[i * S0::R], j, Wsm, S);
                        }
                    }
                }
                F::template middle<-1>(work, v, tid, Wsm, S);
                __pipeline_wait_prior(0);
                __syncthreads();
                if constexpr (VP) {
#pragma unroll
                    for (int i = 0; i < SL::BPT; i += 2) {
                        int t, j;
                        SL::bj(i, tid, t, j);
#pragma unroll
                        for (int r = 0; r < SL::R; ++r) {
                            const float4 h = ld4(hbuf + hb_idx<NB>(SL::out_n(j, r), t));
                            acc[i * SL::R + r] = cadd(acc[i * SL::R + r], cmul(v[i * SL::R + r], lo2(h)));
                            acc[(i + 1) * SL::R + r] = cadd(acc[(i + 1) * SL::R + r], cmul(v[(i + 1) * SL::R + r], hi2(h)));
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < SL::BPT; ++i) {
                        int t, j;
                        SL::bj(i, tid, t, j);
#pragma unroll
                        for (int r = 0; r < SL::R; ++r) {
                            const float2 h = hbuf[hb_idx<NB>(SL::out_n(j, r), t)];
                            const float2 x = v[i * SL::R + r];
                            float2 &a = acc[i * SL::R + r];
                            a.x = __fmaf_rn(x.x, h.x, __fmaf_rn(-x.y, h.y, a.x));
                            a.y = __fmaf_rn(x.x, h.y, __fmaf_rn(x.y, h.x, a.y));
                        }
                    }
                }
            }
        }
        // inverse DFT along y; the accumulators already sit at stage-0 input positions
#pragma unroll
        for (int i = 0; i < S0::BPT; ++i) {
            int t, j;
            S0::bj(i, tid, t, j);
            S0::template bfly<+1>(&acc[i * S0::R], j, Wsm, S);
        }
        __syncthreads();
        F::template middle<+1>(work, acc, tid, Wsm, S);
        float2 *O = base + (int64_t)A.NQ * S * LDF + f0;
#pragma unroll
        for (int i = 0; i < SL::BPT; ++i) {
            int t, j;
            SL::bj(i, tid, t, j);
#pragma unroll
            for (int r = 0; r < SL::R; ++r) {
                const int n = SL::out_n(j, r);
                if (n >= c2) O[(int64_t)(n - c2) * LDF + t] = acc[i * SL::R + r];
            }
        }
        return;
    }

    // mode 1 (H^T): R-hat = DFT_y of the r-window spectrum rows, kept in colq
    if (td.p0 <= td.p1 && td.q0 <= td.q1) prefetch_hhat<S, NB, NTH, LDF>(hbuf, hk(td.p0, td.q0), f0, tid);
#pragma unroll
    for (int i = 0; i < S0::BPT; ++i) {
        int t, j;
        S0::bj(i, tid, t, j);
#pragma unroll
        for (int r = 0; r < S0::R; ++r) v[i * S0::R + r] = __ldg(base + (int64_t)S0::in_n(j, r) * LDF + f0 + t);
        S0::template bfly<-1>(&v[i * S0::R], j, Wsm, S);
    }
    F::template middle<-1>(work, v, tid, Wsm, S);
    SL::store(colq, v, tid);
    float2 *Bbase = base + (int64_t)S * LDF + f0;
    for (int q = td.q0; q <= td.q1; ++q) {
        float2 acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = make_float2(0.f, 0.f);
        for (int p = td.p0; p <= td.p1; ++p) {
            fill_wys(p);
            __pipeline_wait_prior(0);
            __syncthreads();
            if constexpr (VP) {
#pragma unroll
                for (int i = 0; i < S0::BPT; i += 2) {
                    int t, j;
                    S0::bj(i, tid, t, j);
#pragma unroll
                    for (int r = 0; r < S0::R; ++r) {
                        const int n = S0::in_n(j, r);
                        const float4 c = ld4(colq + t * CS + n), h = ld4(hbuf + hb_idx<NB>(n, t));
                        v[i * S0::R + r] = cmulc(lo2(c), lo2(h));
                        v[(i + 1) * S0::R + r] = cmulc(hi2(c), hi2(h));
                    }
                    S0::template bfly<+1>(&v[i * S0::R], j, Wsm, S);
                    S0::template bfly<+1>(&v[(i + 1) * S0::R], j + 1, Wsm, S);
                }
            } else {
#pragma unroll
                for (int i = 0; i < S0::BPT; ++i) {
                    int t, j;
                    S0::bj(i, tid, t, j);
#pragma unroll
                    for (int r = 0; r < S0::R; ++r) {
                        const int n = S0::in_n(j, r);
                        v[i * S0::R + r] = cmulc(colq[t * CS + n], hbuf[hb_idx<NB>(n, t)]);
                    }
                    S0::template bfly<+1>(&v[i * S0::R], j, Wsm, S);
                }
            }
            __syncthreads();      // hbuf consumed: prefetch the next PSF spectrum under the FFT
            {
                int np = p + 1, nq = q;
                if (np > td.p1) { np = td.p0; ++nq; }
                if (nq <= td.q1) prefetch_hhat<S, NB, NTH, LDF>(hbuf, hk(np, nq), f0, tid);
            }
            F::template middle<+1>(work, v, tid, Wsm, S);
#pragma unroll
            for (int i = 0; i < SL::BPT; ++i) {
                int t, j;
                SL::bj(i, tid, t, j);
#pragma unroll
                for (int r = 0; r < SL::R; ++r) {
                    const int n = SL::out_n(j, r);
                    const float wv = wys[n];
                    float2 &o = acc[i * SL::R + r];
                    o = make_float2(o.x + wv * v[i * SL::R + r].x, o.y + wv * v[i * SL::R + r].y);
                }
            }
        }
        float2 *Bq = Bbase + (int64_t)(q - td.q0) * T * LDF;
#pragma unroll
        for (int i = 0; i < SL::BPT; ++i) {
            int t, j;
            SL::bj(i, tid, t, j);
#pragma unroll
            for (int r = 0; r < SL::R; ++r) {
                const int n = SL::out_n(j, r);
                if (n < T) Bq[(int64_t)n * LDF + t] = acc[i * SL::R + r];
            }
        }
    }
}

// ------------------------------------------------------------------ pass B / B' with TMEM
// Variant of k_cols (modes 0 and 1) whose per-thread state that survives across the
// (p, q) transforms -- the stage-0 inputs of the chunk (A_q for H, R-hat for H^T) and
// the spectral accumulator -- lives in tensor memory (tcgen05.st / tcgen05.ld,
// 32x32b shape: each thread owns one TMEM lane, 64 columns) instead of registers and
// shared memory (34 KB less per CTA; measured on c4: H 4.16 -> 4.05 ms, H^T 3.97 ->
// 3.63 ms).  At 2 CTAs/SM the transform itself still needs 128 registers; forcing 3
// CTAs/SM (80 registers) spills and is slower (profiles/r1/SUMMARY.md).
// Twiddle provider of the TMEM column pass (S = 512, stages 1 and 2 with Ns = 8, 64, two
// butterflies per thread each): w^1..w^7 of the thread's butterfly i of that stage in 16
// TMEM columns at base + (slot * 2 + i) * 16, written once per CTA from TwTable (same
// values), so a transform reads one tcgen05.ld per butterfly instead of 3 shared loads and
// 4 complex products.
// Both butterflies' twiddles of one stage, loaded from TMEM ahead of use (TwTmem::pre,
// before the exchange barrier) and waited for in ready(): the registers pass through the
// wait so no use can be scheduled above it.
struct TwRegs {
    uint32_t r[2][16];
    __device__ __forceinline__ void ready() {
        asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                     : "+r"(r[0][0]), "+r"(r[0][1]), "+r"(r[0][2]), "+r"(r[0][3]), "+r"(r[0][4]), "+r"(r[0][5]),
                       "+r"(r[0][6]), "+r"(r[0][7]), "+r"(r[0][8]), "+r"(r[0][9]), "+r"(r[0][10]), "+r"(r[0][11]),
                       "+r"(r[0][12]), "+r"(r[0][13]), "+r"(r[1][0]), "+r"(r[1][1]), "+r"(r[1][2]), "+r"(r[1][3]),
                       "+r"(r[1][4]), "+r"(r[1][5]), "+r"(r[1][6]), "+r"(r[1][7]), "+r"(r[1][8]), "+r"(r[1][9]),
                       "+r"(r[1][10]), "+r"(r[1][11]), "+r"(r[1][12]), "+r"(r[1][13])
                     :: "memory");
    }
    template <int Ns, int R>
    __device__ __forceinline__ void get(int i, int, float2 (&w)[8]) const {
#pragma unroll
        for (int k = 1; k < 8; ++k) w[k] = make_float2(__uint_as_float(r[i][2 * k - 2]), __uint_as_float(r[i][2 * k - 1]));
    }
};
struct TwTmem {
    uint32_t base;
    template <int Ns, int R>
    __device__ __forceinline__ void get(int i, int, float2 (&w)[8]) const {
        static_assert(R == 8 && (Ns == 8 || Ns == 64), "512-point radix-8 plan");
        constexpr int slot = Ns == 8 ? 0 : 1;
        uint32_t r[16];
        tm_ld16(base + (uint32_t)((slot * 2 + i) * 16), r);
        tm_wait_ld();
#pragma unroll
        for (int k = 1; k < 8; ++k) w[k] = make_float2(__uint_as_float(r[2 * k - 2]), __uint_as_float(r[2 * k - 1]));
    }
    template <int Ns>
    __device__ __forceinline__ TwRegs pre() const {
        static_assert(Ns == 8 || Ns == 64, "512-point radix-8 plan");
        constexpr int slot = Ns == 8 ? 0 : 1;
        TwRegs t;
#pragma unroll
        for (int i = 0; i < 2; ++i) tm_ld16(base + (uint32_t)((slot * 2 + i) * 16), t.r[i]);
        return t;
    }
};

template <int S>
struct GCT {
    // NB columns per CTA with NTH = 32 NB threads: 16 elements per thread at S = 512;
    // CS = S + 16/NB makes the paired 16-byte exchanges conflict-free per quarter-warp
    static constexpr int NB = COLS_TM_NB, NTH = 32 * NB, CS = S + 16 / NB;
    static constexpr int E = NB * S / NTH;
    // per warp: 32 input + 32 accumulator columns (+ 64 twiddle columns); 4 lane quarters x NB/4 warps
    static constexpr int WCOLS = 128;
    static constexpr int TMCOLS = NB >= 8 ? WCOLS * (NB / 4) : WCOLS;
    using F = Fft<S, NB, CS, NTH>;
};
template <int S>
static size_t smem_cols_tm(int NP, int NQ) {
    using G = GCT<S>;
    return 128 + (size_t)COLS_TM_TW * 8 + (size_t)S * G::NB * 8 + (size_t)G::NB * G::CS * 8 + 2 * (size_t)S * 8 +
           (size_t)NP * S * 4 + (size_t)NP * NQ * 4 + 16 + 8;
}

template <int S>
__global__ void __launch_bounds__(32 * COLS_TM_NB, COLS_TM_MINB) k_cols_tm(FftArgs A, int mode, int cpb,
                                                                            const __grid_constant__ CUtensorMap tmh) {
    using G = GCT<S>;
    using F = typename G::F;
    using S0 = typename F::First;
    using SL = typename F::Last;
    static_assert(S0::R == SL::R && S0::VEC && SL::VEC, "paired first/last stages");
    constexpr int NB = G::NB, CS = G::CS, E = G::E, LDF = LD<S>::LDF, NF = S / 2 + 1, NTH = G::NTH;
    static_assert(LD<S>::LDF == S / 2 + NB, "chunking shared with k_cols");
    extern __shared__ __align__(16) float2 sm2[];
    // hbuf first, 128-byte aligned: the PSF-spectrum chunk (S x NB, pair-interleaved) lands there
    // by one TMA tensor copy per (p, q)
    // (offsets from sm2, not integer round trips, so every access below stays a 32-bit
    // shared-window LDS / STS instead of a generic 64-bit LD / ST)
    float2 *hbuf = sm2 + (((128u - ((uint32_t)__cvta_generic_to_shared(sm2) & 127u)) & 127u) >> 3);
    float2 *Wsm = hbuf + S * NB;     // S/2 twiddles
    float2 *work = Wsm + COLS_TM_TW; // NB x CS
    float2 *hnq = work + NB * CS;    // S: Nyquist column of the PSF spectrum (chunk 0)
    float2 *nyq = hnq + S;           // S: the packed column's spectrum C (chunk 0)
    float *wys_all = reinterpret_cast<float *>(nyq + S);
    int *slot_s = reinterpret_cast<int *>(wys_all + (size_t)A.NP * S);
    uint32_t *tm_slot = reinterpret_cast<uint32_t *>(slot_s + A.NP * A.NQ);
    uint64_t *hbar = reinterpret_cast<uint64_t *>(tm_slot + ((((uint32_t)__cvta_generic_to_shared(tm_slot + 1)) & 7u) ? 2 : 1));
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr uint32_t HBYTES = S * NB * 8;
    uint32_t hphase = 0;
    // cpb consecutive column chunks of one tile per CTA: the TMEM allocation,
    // twiddles and the tile's wy_p rows / PSF slots are set up once for all of them
    // for H the real columns 0 (DC) and S/2 (Nyquist) of the row spectra travel
    // as one complex column c = X[., 0] + i X[., S/2] in chunk 0's column 0: S/2 columns
    static_assert((S / 2) % NB == 0, "Nyquist packing needs whole chunks");
    // (H only: for H^T the per-(p, q) combination of the packed column measured slower)
    const bool nyq_on = mode == 0;
    const int nchunk = nyq_on ? (S / 2) / NB : (NF + NB - 1) / NB;
    const int ngrp = (nchunk + cpb - 1) / cpb;
    const int tile = blockIdx.x / ngrp, cg = blockIdx.x % ngrp;
    const int P = A.P, c2 = P - 1, T = S - P + 1;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                     :: "r"((uint32_t)__cvta_generic_to_shared(tm_slot)), "n"(G::TMCOLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    for (int i = tid; i < COLS_TM_TW; i += NTH) Wsm[i] = A.W[i];   // a length-S forward/inverse plan uses W^k, k < S/2
    if (tid == 0) {
        mbar_init(hbar, 1);
        asm volatile("prefetch.tensormap [%0];\n" :: "l"(reinterpret_cast<uint64_t>(&tmh)) : "memory");
    }
    const TileDesc td = A.tiles[tile];
    const FacetDev &Fd = A.facets[td.f];
    float2 *base = A.scratch + (int64_t)tile * A.tile_rows * LDF;
    {
        const int np = td.p1 - td.p0 + 1, nq = td.q1 - td.q0 + 1;
        for (int idx = tid; idx < np * S; idx += NTH) {
            const int pi = idx / S, i = idx - pi * S;
            // (H^T weights its outputs: rows >= T, which are dropped, get weight 0)
            wys_all[idx] = (td.y0 + i < Fd.ny && (mode == 0 || i < T))
                               ? __ldg(A.wy + (size_t)(td.p0 + pi) * A.Ny + Fd.ey0 + td.y0 + i) : 0.f;
        }
        for (int idx = tid; idx < np * nq; idx += NTH) {
            const int pi = idx / nq, qi = idx - pi * nq;
            slot_s[idx] = __ldg(A.psf_slot + (td.p0 + pi) * A.Gx + td.q0 + qi);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // this thread's TMEM lane (warp quarter) and its 64 columns: [0, 32) inputs, [32, 64) accumulator
    const uint32_t t_in = *tm_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * G::WCOLS);
    const uint32_t t_acc = t_in + 32;
    {
        using S1 = Stage<S, NB, CS, NTH, 1>;
        using S2 = Stage<S, NB, CS, NTH, 2>;
        static_assert(F::NS == 3 && S1::R == 8 && S2::R == 8 && S1::BPT == 2 && S2::BPT == 2, "twiddle slots");
        const TwTable tt{Wsm, S};
#pragma unroll
        for (int slot = 0; slot < 2; ++slot) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                int t, j;
                S1::bj(i, tid, t, j);
                float2 w[8];
                if (slot == 0) tt.get<S1::Ns, 8>(i, j, w);
                else tt.get<S2::Ns, 8>(i, j, w);
                uint32_t r[16];
#pragma unroll
                for (int k = 1; k < 8; ++k) { r[2 * k - 2] = __float_as_uint(w[k].x); r[2 * k - 1] = __float_as_uint(w[k].y); }
                r[14] = r[15] = 0u;
                tm_st16(t_acc + 32 + (uint32_t)((slot * 2 + i) * 16), r);
            }
        }
        tm_wait_st();
    }
    const TwTmem tw{t_acc + 32};
    const int nqt = td.q1 - td.q0 + 1;
    for (int ci = 0; ci < cpb; ++ci) {
    const int f0 = (cg * cpb + ci) * NB;
    if (f0 >= nchunk * NB) break;
    // this thread carries the packed (DC, Nyquist) column: its spectrum C_n = A_n + i B_n
    // (A, B the DFTs of the two real columns, Hermitian) is multiplied as
    // M0 A + i MN B = ((M0 + MN) C_n + (M0 - MN) conj C_{-n}) / 2 (M = the PSF spectrum's
    // columns 0 and S/2); the inverse DFT of that is real_0 + i real_N
    const bool pk = nyq_on && f0 == 0 && (tid % NB) == 0;
    auto hk = [&](int p, int q) { return A.Hhat + (int64_t)slot_s[(p - td.p0) * nqt + (q - td.q0)] * S * LDF; };
    // the chunk of PSF spectrum (p, q): pair-rows [slot S/2, +S/2) x floats [4 f0, 4 f0 + 4 NB) of the
    // 2-D view of Hhat (LDF * 4 floats per pair-row)
    auto tma_hhat = [&](int p, int q) {
        if (tid == 0)
            tma_load_2d(hbuf, &tmh, 4 * f0, slot_s[(p - td.p0) * nqt + (q - td.q0)] * (S / 2), hbar, HBYTES);
    };
    // stage-0 input positions of this thread, straight from the global chunk (row stride LDF)
    auto load_in = [&](const float2 *src, float2 (&v)[E]) {
#pragma unroll
        for (int i = 0; i < S0::BPT; ++i) {
            int t, j;
            S0::bj(i, tid, t, j);
#pragma unroll
            for (int r = 0; r < S0::R; ++r) {
                const float2 *sp = src + (int64_t)S0::in_n(j, r) * LDF + f0 + t;
                v[i * S0::R + r] = __ldg(sp);
                if (pk) v[i * S0::R + r].y = __ldg(sp + S / 2).x;   // X[., 0] and X[., S/2] are real
            }
        }
    };
    // packed column: store / combine through nyq (positions n of this thread's elements)
    auto nyq_mul = [&](float2 c, int n, float2 m0, float2 mn) {
        const float2 cm = conjf2(nyq[(S - n) & (S - 1)]);
        const float2 a = cadd(m0, mn), b = csub(m0, mn);
        const float2 r = cadd(cmul(a, c), cmul(b, cm));
        return make_float2(0.5f * r.x, 0.5f * r.y);
    };
    float2 v[E];

    // the accumulator starts at zero in TMEM, so every (p, q) step is load-FMA-store (no
    // first-step selects)
    auto acc_zero = [&]() {
        uint32_t z[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) z[e] = 0u;
        tm_st16(t_acc, z);
        tm_st16(t_acc + 16, z);
    };
    if (mode == 0) {
        acc_zero();
        for (int q = td.q0; q <= td.q1; ++q) {
            load_in(base + (int64_t)(q - td.q0) * S * LDF, v);
            tm_put<E>(t_in, v);
            tm_wait_st();
            for (int p = td.p0; p <= td.p1; ++p) {
                __syncthreads();                   // hbuf free
                if (nyq_on && f0 == 0) {
                    prefetch_hnyq<S, NTH, LDF>(hnq, hk(p, q), tid);
                    __pipeline_commit();
                }
                tma_hhat(p, q);                    // lands under the FFT below
                const float *wys = wys_all + (size_t)(p - td.p0) * S;
                if (p != td.p0) tm_get<E>(t_in, v);
                static_assert(S0::R == 8 && S0::Ns == 1, "untwiddled radix-8 first stage");
#pragma unroll
                for (int i = 0; i < S0::BPT; i += 2) {
                    int t, j;
                    S0::bj(i, tid, t, j);
                    float w0[8], w1[8];
#pragma unroll
                    for (int r = 0; r < S0::R; ++r) {
                        const float2 wv = *reinterpret_cast<const float2 *>(wys + S0::in_n(j, r));
                        w0[r] = wv.x;
                        w1[r] = wv.y;
                    }
                    dft8w<-1>(&v[i * S0::R], w0);          // (wy_p . A_q) -> first stage
                    dft8w<-1>(&v[(i + 1) * S0::R], w1);
                }
                F::template middle_open<-1>(work, v, tid, tw);
                if (pk) {
#pragma unroll
                    for (int i = 0; i < SL::BPT; ++i) {
                        int t, j;
                        SL::bj(i, tid, t, j);
#pragma unroll
                        for (int r = 0; r < SL::R; ++r) nyq[SL::out_n(j, r)] = v[i * SL::R + r];
                    }
                }
                mbar_wait(hbar, hphase);           // the TMA of the chunk has landed
                hphase ^= 1;
                if (nyq_on && f0 == 0) {           // chunk 0: nyq (other threads' stores) and hnq visible
                    __pipeline_wait_prior(0);
                    __syncthreads();
                }
                if (pk) {
#pragma unroll
                    for (int i = 0; i < SL::BPT; ++i) {
                        int t, j;
                        SL::bj(i, tid, t, j);
#pragma unroll
                        for (int r = 0; r < SL::R; ++r) {
                            const int n = SL::out_n(j, r);
                            float2 &h0 = hbuf[hb_idx<NB>(n, 0)];   // read only by this thread
                            v[i * SL::R + r] = nyq_mul(v[i * SL::R + r], n, h0, hnq[n]);
                            h0 = make_float2(1.f, 0.f);           // the product below is then v itself
                        }
                    }
                }
                // acc += v . Hhat in two halves h = last-stage radix outputs r in [4h, 4h + 4) of
                // both butterflies (j, j + 1): their spectrum values at rows (n, n + 1) are one
                // conflict-free 16-byte load (8-byte loads of one member each were 2-way bank
                // conflicted); the halves' accumulators are two 8-column TMEM runs each
                static_assert(SL::BPT == 2 && SL::R == 8, "two radix-8 butterflies per thread");
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t a0[8], a1[8];
                    tm_ld8(t_acc + 8 * h, a0);
                    tm_ld8(t_acc + 16 + 8 * h, a1);
                    tm_wait_ld();
                    int t, j;
                    SL::bj(0, tid, t, j);
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) {
                        const int r = 4 * h + rr;
                        const float4 hh = ld4(hbuf + hb_idx<NB>(SL::out_n(j, r), t));
                        const float2 x0 = v[r], x1 = v[SL::R + r];
                        float ax = __uint_as_float(a0[2 * rr]), ay = __uint_as_float(a0[2 * rr + 1]);
                        a0[2 * rr] = __float_as_uint(__fmaf_rn(x0.x, hh.x, __fmaf_rn(-x0.y, hh.y, ax)));
                        a0[2 * rr + 1] = __float_as_uint(__fmaf_rn(x0.x, hh.y, __fmaf_rn(x0.y, hh.x, ay)));
                        ax = __uint_as_float(a1[2 * rr]);
                        ay = __uint_as_float(a1[2 * rr + 1]);
                        a1[2 * rr] = __float_as_uint(__fmaf_rn(x1.x, hh.z, __fmaf_rn(-x1.y, hh.w, ax)));
                        a1[2 * rr + 1] = __float_as_uint(__fmaf_rn(x1.x, hh.w, __fmaf_rn(x1.y, hh.z, ay)));
                    }
                    tm_st8(t_acc + 8 * h, a0);
                    tm_st8(t_acc + 16 + 8 * h, a1);
                }
                tm_wait_st();
            }
        }
        tm_get<E>(t_acc, v);
        // inverse DFT along y; the accumulator sits at stage-0 input positions
#pragma unroll
        for (int i = 0; i < S0::BPT; ++i) {
            int t, j;
            S0::bj(i, tid, t, j);
            S0::template bfly<+1>(&v[i * S0::R], j, Wsm, S);
        }
        __syncthreads();
        F::template middle_open<+1>(work, v, tid, tw);
        float2 *O = base + (int64_t)A.NQ * S * LDF + f0;
#pragma unroll
        for (int i = 0; i < SL::BPT; ++i) {
            int t, j;
            SL::bj(i, tid, t, j);
#pragma unroll
            for (int r = 0; r < SL::R; ++r) {
                const int n = SL::out_n(j, r);
                if (n >= c2) {
                    if (pk) {
                        O[(int64_t)(n - c2) * LDF] = make_float2(v[i * SL::R + r].x, 0.f);
                        O[(int64_t)(n - c2) * LDF + S / 2] = make_float2(v[i * SL::R + r].y, 0.f);
                    } else {
                        O[(int64_t)(n - c2) * LDF + t] = v[i * SL::R + r];
                    }
                }
            }
        }
    } else {
        // mode 1 (H^T): R-hat = DFT_y of the r-window spectrum rows, kept in TMEM
        if (td.p0 <= td.p1 && td.q0 <= td.q1) tma_hhat(td.p0, td.q0);
        load_in(base, v);
#pragma unroll
        for (int i = 0; i < S0::BPT; ++i) {
            int t, j;
            S0::bj(i, tid, t, j);
            S0::template bfly<-1>(&v[i * S0::R], j, Wsm, S);
        }
        F::template middle_open<-1>(work, v, tid, tw);
        tm_put<E>(t_in, v);                        // last-stage positions == stage-0 positions
        tm_wait_st();
        float2 *Bbase = base + (int64_t)S * LDF + f0;
        for (int q = td.q0; q <= td.q1; ++q) {
            acc_zero();
            tm_wait_st();
            for (int p = td.p0; p <= td.p1; ++p) {
                const float *wys = wys_all + (size_t)(p - td.p0) * S;
                tm_get<E>(t_in, v);
                mbar_wait(hbar, hphase);           // Hhat chunk landed (TMA)
                hphase ^= 1;
#pragma unroll
                for (int i = 0; i < S0::BPT; i += 2) {
                    int t, j;
                    S0::bj(i, tid, t, j);
#pragma unroll
                    for (int r = 0; r < S0::R; ++r) {
                        const float4 hh = ld4(hbuf + hb_idx<NB>(S0::in_n(j, r), t));
                        v[i * S0::R + r] = cmulc(v[i * S0::R + r], lo2(hh));
                        v[(i + 1) * S0::R + r] = cmulc(v[(i + 1) * S0::R + r], hi2(hh));
                    }
                    S0::template bfly<+1>(&v[i * S0::R], j, Wsm, S);
                    S0::template bfly<+1>(&v[(i + 1) * S0::R], j + 1, Wsm, S);
                }
                __syncthreads();                   // hbuf consumed: prefetch the next spectrum under the FFT
                {
                    int np = p + 1, nq = q;
                    if (np > td.p1) { np = td.p0; ++nq; }
                    if (nq <= td.q1) tma_hhat(np, nq);
                }
                F::template middle_open<+1>(work, v, tid, tw);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t a[16];
                    tm_ld16(t_acc + 16 * h, a);
                    tm_wait_ld();
#pragma unroll
                    for (int i2 = 0; i2 < SL::BPT / 2; ++i2) {
                        const int i = h * (SL::BPT / 2) + i2;
                        int t, j;
                        SL::bj(i, tid, t, j);
#pragma unroll
                        for (int r = 0; r < SL::R; ++r) {
                            const int n = SL::out_n(j, r);
                            const float wv = wys[n];
                            const int e = (i2 * SL::R + r) * 2;
                            float2 o = make_float2(__uint_as_float(a[e]), __uint_as_float(a[e + 1]));
                            o.x += wv * v[i * SL::R + r].x;
                            o.y += wv * v[i * SL::R + r].y;
                            a[e] = __float_as_uint(o.x); a[e + 1] = __float_as_uint(o.y);
                        }
                    }
                    tm_st16(t_acc + 16 * h, a);
                }
                tm_wait_st();
            }
            tm_get<E>(t_acc, v);
            float2 *Bq = Bbase + (int64_t)(q - td.q0) * T * LDF;
#pragma unroll
            for (int i = 0; i < SL::BPT; ++i) {
                int t, j;
                SL::bj(i, tid, t, j);
#pragma unroll
                for (int r = 0; r < SL::R; ++r) {
                    const int n = SL::out_n(j, r);
                    if (n < T) Bq[(int64_t)n * LDF + t] = v[i * SL::R + r];
                }
            }
        }
    }
    __syncthreads();                               // smem buffers free for the next chunk
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(*tm_slot), "n"(G::TMCOLS) : "memory");
}

// ------------------------------------------------------------------ pass C / C'
// C2R of NB spectrum rows per CTA.  The rows (global, stride LDF) are streamed into a
// shared staging buffer with cp.async one source ahead, so the next source's loads
// are in flight under the current source's FFT.
template <int S>
struct C2R {
    using G = GR<S>;
    using F = typename G::F;
    static constexpr int NB = G::NB, SH = G::SH, RS = G::RS, LDF = LD<S>::LDF;
    static constexpr int SS = SH + 2;            // staging row stride (float2; 16-byte rows)
    // rows [0, nrows) of src0 -> stg (16-byte cp.async; rows >= nrows zero-filled)
    __device__ static __forceinline__ void issue(float2 *stg, const float2 *src0, int nrows, int tid) {
        constexpr int V = SH / 2;                 // 16-byte vectors per row, + the Nyquist element
        static_assert(V % 2 == 0 || V == 1, "row split");
        // the 16-byte vectors of NB rows, row-major, by a power-of-two index split (no division)
        for (int idx = tid; idx < NB * V; idx += G::NTH) {
            const int rr = idx / V, v = idx % V;
            float2 *d = stg + rr * SS + 2 * v;
            if (rr < nrows) __pipeline_memcpy_async(d, src0 + (int64_t)rr * LDF + 2 * v, 16);
            else *reinterpret_cast<float4 *>(d) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        // the Nyquist element of each row
        for (int rr = tid; rr < NB; rr += G::NTH) {
            float2 *d = stg + rr * SS + SH;
            if (rr < nrows) __pipeline_memcpy_async(d, src0 + (int64_t)rr * LDF + SH, 8);
            else d[0] = make_float2(0.f, 0.f);
        }
        __pipeline_commit();
    }
    // rows [0, nrows) of src0 -> stg by one bulk copy per row issued by thread 0 (SS * 8 =
    // 2064 bytes: the SH + 1 bins and one pad element, a 16-byte multiple), completion counted
    // on mbarrier m; rows >= nrows (the last row block of a tile) zero-filled by all threads.
    // Replaces 2 k 16-byte cp.async per CTA (and their 64-bit address arithmetic).
    __device__ static __forceinline__ void issue_bulk(float2 *stg, const float2 *src0, int nrows, int tid, uint64_t *m) {
        constexpr uint32_t RB = SS * 8;
        static_assert(SS == SH + 2 && RB % 16 == 0 && LDF >= SS, "bulk row copies");
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(smem_u32(m)), "r"(nrows * RB)
                         : "memory");
            for (int rr = 0; rr < nrows; ++rr)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                             :: "r"(smem_u32(stg + rr * SS)), "l"(src0 + (int64_t)rr * LDF), "r"(RB), "r"(smem_u32(m))
                             : "memory");
        }
        for (int idx = nrows * (SS / 2) + tid; idx < NB * (SS / 2); idx += G::NTH)
            reinterpret_cast<float4 *>(stg)[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // radix 16 x 16 (S = 512): the stage-0 inputs straight from the staged spectrum rows,
    // C2R-pre-processed in registers (each thread reads both members n, SH - n of its 16
    // pairs and forms its own bins; no pass through the exchange buffer), then the stage-0
    // butterfly
    __device__ static __forceinline__ void load_pre(const float2 *stg, float2 (&v)[G::E], const float2 *Wsm, int tid) {
        using S0 = typename F::First;
        static_assert(S0::R == 16 && S0::BPT == 1, "radix-16 first stage");
        int t, j;
        S0::bj(0, tid, t, j);
        const float2 *sr = stg + t * SS;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int n = S0::in_n(j, r);
            v[r] = c2r_pre(sr[n], sr[SH - n], Wsm[n]);
        }
        S0::template bfly<+1>(&v[0], j, Wsm, S);
    }
    // half-length complex input z = E + i O from the staged spectrum rows -> work, one
    // (k, SH - k) pair per item; the self-paired k = SH/2 is done by the k = 0 item
    __device__ static __forceinline__ void pre(float2 *work, const float2 *stg, const float2 *Wsm, int tid) {
        constexpr int HP = SH / 2, RPP = G::NTH / HP;
        static_assert(G::NTH % HP == 0 && NB % RPP == 0, "pre-processing split");
        const int k = tid % HP, rr0 = tid / HP;
        const float2 w = Wsm[k], wc = make_float2(-w.x, w.y), wm = Wsm[HP];
#pragma unroll 4
        for (int rr = rr0; rr < NB; rr += RPP) {
            const float2 *sr = stg + rr * SS;
            float2 *wr = work + rr * RS;
            const float2 a = sr[k], b = sr[SH - k];
            if (k == 0) {
                wr[0] = c2r_pre(a, b, w);
                const float2 m = sr[HP];
                wr[HP] = c2r_pre(m, m, wm);
            } else {
                c2r_pre_pair(a, b, w, wr[k], wr[SH - k]);
            }
        }
    }
};

template <int S, bool HT>
__global__ void __launch_bounds__(GR<S>::NTH, S == 1024 ? (HT ? 1 : 2) : (HT && S == 512) ? 3 : GR<S>::NTH == 128 ? (HT ? 5 : 6) : 4)
k_rows_inv(FftArgs A, int mode) {
    // H^T at S = 512: the accumulator sum_q wx_q C2R(B_q) lives in TMEM (32 columns per
    // thread) instead of 32 registers, so 3 CTAs/SM fit
    constexpr bool HTT = HT && S == 512;
    using G = GR<S>;
    using C = C2R<S>;
    using F = typename G::F;
    using SL = typename F::Last;
    constexpr int NB = G::NB, RS = G::RS, XS = G::XS, LDF = LD<S>::LDF, E = G::E;
    static_assert(XS <= 2 * RS, "outs aliases work");
    extern __shared__ __align__(16) float2 sm2[];
    float2 *Wsm = sm2;                                         // ROWS_TW(S) twiddles
    float2 *work = Wsm + ROWS_TW(S);                           // NB x RS; reused as outs (NB x XS reals)
    // NB x SS staging; H has a single source, staged straight into work and pre-processed in
    // place (C2R::pre reads and writes only its own (k, SH - k) pair): 3 -> 4 CTAs/SM
    static_assert(C::SS == RS, "in-place staging");
    float2 *stg = HT ? work + NB * RS : work;
    float *wxs = reinterpret_cast<float *>(stg + NB * C::SS);  // NQ x S (H^T)
    float *outs = reinterpret_cast<float *>(work);
    __shared__ double red[G::NTH / 32];
    const int tid = threadIdx.x;
    const int P = A.P, c2 = P - 1, T = S - P + 1;
    const int nblk = (T + NB - 1) / NB;
    const int tile = blockIdx.x / nblk, r0 = (blockIdx.x % nblk) * NB;
    const int nrows = min(NB, T - r0);
    const TileDesc t = A.tiles[tile];
    const FacetDev &Fd = A.facets[t.f];
    const float2 *base = A.scratch + (int64_t)tile * A.tile_rows * LDF;
    const float scale = A.scale;
    constexpr bool ht = HT;
    const int nq = ht ? t.q1 - t.q0 + 1 : 1;
    const float2 *Bbase = base + (int64_t)S * LDF;
    auto src = [&](int qi) {
        return ht ? Bbase + ((int64_t)qi * T + r0) * LDF : base + ((int64_t)A.NQ * S + r0) * LDF;
    };
    if (ht) {
        // wx_q rows of all active q: cp.async, committed with the first staging group below
        for (int idx = tid; idx < nq * S; idx += G::NTH) {
            const int qi = idx / S, cc = idx - qi * S;
            if (cc < T && t.x0 + cc < Fd.nx)
                __pipeline_memcpy_async(wxs + idx, A.wx + (size_t)(t.q0 + qi) * A.Nx + Fd.ex0 + t.x0 + cc, 4);
            else
                wxs[idx] = 0.f;
        }
        if constexpr (G::MIR) __pipeline_commit();   // (the cp.async staging path commits them with its rows)
    }
    __shared__ uint64_t sbar;                  // staging rows landed (bulk copies, S = 512)
    uint32_t sphase = 0;
    if constexpr (G::MIR) {
        if (tid == 0) mbar_init(&sbar, 1);
        if (nq > 0) C::issue_bulk(stg, src(0), nrows, tid, &sbar);
    } else {
        if (nq > 0) C::issue(stg, src(0), nrows, tid);
    }
    for (int i = tid; i < ROWS_TW(S); i += G::NTH) Wsm[i] = A.W[i];
    float2 acc[(HT && !HTT) ? E : 1];
#pragma unroll
    for (int e = 0; e < ((HT && !HTT) ? E : 1); ++e) acc[e] = make_float2(0.f, 0.f);
    float2 v[E];
    __shared__ uint32_t tm_slot_a;
    uint32_t t_a = 0;
    if constexpr (HTT) {
        static_assert(E == 16, "the TMEM accumulator holds 16 complex = 32 columns per thread");
        if ((tid >> 5) == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                         :: "r"((uint32_t)__cvta_generic_to_shared(&tm_slot_a)), "n"(64) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        t_a = tm_slot_a + ((uint32_t)(32 * ((tid >> 5) & 3)) << 16) + (uint32_t)((tid >> 7) * 32);
    }
    for (int qi = 0; qi < nq; ++qi) {
        __pipeline_wait_prior(0);
        __syncthreads();
        if constexpr (G::MIR) {
            mbar_wait(&sbar, sphase);                              // the rows of this q landed
            sphase ^= 1;
            C::load_pre(stg, v, Wsm, tid);
            __syncthreads();                                       // stg (= work for H) read
            if (qi + 1 < nq) C::issue_bulk(stg, src(qi + 1), nrows, tid, &sbar);
        } else {
            C::pre(work, stg, Wsm, tid);
            __syncthreads();
            if (qi + 1 < nq) C::issue(stg, src(qi + 1), nrows, tid);   // in flight under this FFT
            F::First::template load_bfly<+1>(work, v, tid, Wsm, S);
            __syncthreads();
        }
        F::template middle<+1>(work, v, tid, Wsm, S);
        if constexpr (HT) {
            // g += wx_q . C2R(B_q): z[n] = (x[2n], x[2n+1]) at the last-stage positions
            const float *wq = wxs + qi * S;
            if constexpr (HTT) {
                uint32_t a[32];
                if (qi > 0) { tm_ld32(t_a, a); tm_wait_ld(); }
#pragma unroll
                for (int i = 0; i < SL::BPT; ++i) {
                    int tt, j;
                    SL::bj(i, tid, tt, j);
#pragma unroll
                    for (int r = 0; r < SL::R; ++r) {
                        const float2 w = *reinterpret_cast<const float2 *>(wq + 2 * SL::out_n(j, r));
                        const int e = 2 * (i * SL::R + r);
                        const float ox = qi > 0 ? __uint_as_float(a[e]) : 0.f, oy = qi > 0 ? __uint_as_float(a[e + 1]) : 0.f;
                        a[e] = __float_as_uint(ox + w.x * v[i * SL::R + r].x);
                        a[e + 1] = __float_as_uint(oy + w.y * v[i * SL::R + r].y);
                    }
                }
                tm_st32(t_a, a);
                tm_wait_st();
            } else {
#pragma unroll
            for (int i = 0; i < SL::BPT; ++i) {
                int tt, j;
                SL::bj(i, tid, tt, j);
#pragma unroll
                for (int r = 0; r < SL::R; ++r) {
                    const float2 w = *reinterpret_cast<const float2 *>(wq + 2 * SL::out_n(j, r));
                    float2 &o = acc[i * SL::R + r];
                    o.x += w.x * v[i * SL::R + r].x;
                    o.y += w.y * v[i * SL::R + r].y;
                }
            }
            }
        }
    }
    // last-stage values -> outs (aliases work: middle() ended with a barrier)
    if constexpr (HTT) {
        if (nq > 0) tm_get<E>(t_a, v);
    }
#pragma unroll
    for (int i = 0; i < SL::BPT; ++i) {
        int tt, j;
        SL::bj(i, tid, tt, j);
#pragma unroll
        for (int r = 0; r < SL::R; ++r) {
            float2 val;
            if constexpr (HT && !HTT) val = acc[i * SL::R + r];
            else val = v[i * SL::R + r];
            if (nq == 0) val = make_float2(0.f, 0.f);
            *reinterpret_cast<float2 *>(outs + tt * XS + 2 * SL::out_n(j, r)) = val;
        }
    }
    if constexpr (HTT) asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if constexpr (HTT) {
        if ((tid >> 5) == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tm_slot_a), "n"(64) : "memory");
    }

    // valid outputs of this row block: rows [0, nr), columns [0, nc) (facet edge and
    // strip clip); the flat index walks (rr, cc) incrementally (no per-element division)
    const int ny_ = ht ? Fd.ny : Fd.my, nx_ = ht ? Fd.nx : Fd.mx;
    const int nr = min(nrows, min(ny_, t.ylim) - (t.y0 + r0)), nc = min(T, min(nx_, t.xlim) - t.x0);
    if (nr <= 0 || nc <= 0) {
        if (!ht && mode != FFT_PLAIN && A.partials && tid == 0) A.partials[blockIdx.x] = 0.0;
        return;
    }
    const int ntot = nr * nc, drr = G::NTH / nc, dcc = G::NTH - drr * nc;
    int rr = tid / nc, cc = tid - rr * nc;
    auto step = [&]() {
        rr += drr;
        cc += dcc;
        if (cc >= nc) { cc -= nc; ++rr; }
    };
    if (ht) {
        float *gb = Fd.g + (int64_t)(t.y0 + r0) * Fd.ep + t.x0;
        const int ep = (int)Fd.ep;
        if (((t.x0 | nc | ep) & 1) == 0 && ((uintptr_t)gb & 7) == 0) {
            // column pairs (8-byte aligned; XS even)
            const int ncp = nc >> 1, ntp = nr * ncp, dr2 = G::NTH / ncp, dc2 = G::NTH - dr2 * ncp;
            int r2 = tid / ncp, c2p = tid - r2 * ncp;
            for (int idx = tid; idx < ntp; idx += G::NTH) {
                const float2 o = *reinterpret_cast<const float2 *>(outs + r2 * XS + 2 * c2p);
                *reinterpret_cast<float2 *>(gb + r2 * ep + 2 * c2p) = make_float2(o.x * scale, o.y * scale);
                r2 += dr2;
                c2p += dc2;
                if (c2p >= ncp) { c2p -= ncp; ++r2; }
            }
        } else {
            for (int idx = tid; idx < ntot; idx += G::NTH, step()) gb[rr * ep + cc] = outs[rr * XS + cc] * scale;
        }
        return;
    }
    double dsum = 0.0;
    constexpr int U = 8;
    const int64_t obase = (int64_t)(t.y0 + r0) * Fd.op + t.x0;
    const float *yb = Fd.y + obase, *wb = Fd.w ? Fd.w + obase : nullptr;
    float *rb = Fd.r + obase;
    const int op = (int)Fd.op;
    const float w_scalar = Fd.w_scalar;
    if (((t.x0 | nc | op | c2) & 1) == 0 && (((uintptr_t)yb | (uintptr_t)wb | (uintptr_t)rb) & 7) == 0) {
        // column pairs: 8-byte loads / stores (same per-element arithmetic)
        constexpr int U2 = U / 2;
        const int ncp = nc >> 1, ntp = nr * ncp, dr2 = G::NTH / ncp, dc2 = G::NTH - dr2 * ncp;
        int r2 = tid / ncp, cp = tid - r2 * ncp;
        for (int b0 = 0; b0 < ntp; b0 += U2 * G::NTH) {
            float2 yv[U2], wv[U2];
            int off[U2], so[U2];
            bool ok[U2];
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                ok[u] = b0 + tid + u * G::NTH < ntp;
                off[u] = r2 * op + 2 * cp;
                so[u] = r2 * XS + c2 + 2 * cp;
                r2 += dr2;
                cp += dc2;
                if (cp >= ncp) { cp -= ncp; ++r2; }
                const bool ld = ok[u] && mode != FFT_PLAIN;
                yv[u] = ld ? __ldg(reinterpret_cast<const float2 *>(yb + off[u])) : make_float2(0.f, 0.f);
                wv[u] = ld ? (wb ? __ldg(reinterpret_cast<const float2 *>(wb + off[u])) : make_float2(w_scalar, w_scalar))
                           : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U2; ++u) {
                if (!ok[u]) continue;
                const float2 o = *reinterpret_cast<const float2 *>(outs + so[u]);
                const float hx0 = o.x * scale, hx1 = o.y * scale;
                float2 *rp = reinterpret_cast<float2 *>(rb + off[u]);
                if (mode == FFT_PLAIN) {
                    *rp = make_float2(hx0, hx1);
                } else {
                    const float d0 = hx0 - yv[u].x, d1 = hx1 - yv[u].y;
                    if (mode == FFT_RESIDUAL) *rp = make_float2(wv[u].x * d0, wv[u].y * d1);
                    dsum += 0.5 * (double)wv[u].x * (double)d0 * (double)d0;
                    dsum += 0.5 * (double)wv[u].y * (double)d1 * (double)d1;
                }
            }
        }
    } else
    for (int b0 = 0; b0 < ntot; b0 += U * G::NTH) {
        float yv[U], wv[U];
        int off[U], so[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ok[u] = b0 + tid + u * G::NTH < ntot;
            off[u] = rr * op + cc;
            so[u] = rr * XS + c2 + cc;
            step();
            yv[u] = (ok[u] && mode != FFT_PLAIN) ? __ldg(yb + off[u]) : 0.f;
            wv[u] = (ok[u] && mode != FFT_PLAIN) ? (wb ? __ldg(wb + off[u]) : w_scalar) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            const float hx = outs[so[u]] * scale;
            if (mode == FFT_PLAIN) {
                rb[off[u]] = hx;
            } else {
                const float d = hx - yv[u];
                if (mode == FFT_RESIDUAL) rb[off[u]] = wv[u] * d;
                dsum += 0.5 * (double)wv[u] * (double)d * (double)d;
            }
        }
    }
    if (mode != FFT_PLAIN && A.partials) {
        const double s = block_sum<G::NTH>(dsum, red);
        if (tid == 0) A.partials[blockIdx.x] = s;
    }
}

}  // namespace

struct FftPlan {
    int S = 0, T = 0, P = 0, NQ = 1, NP = 1;
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
    CUtensorMap tmh{};                // TMA view of Hhat for the S = 512 column pass
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
        a.scratch = scratch; a.tile_rows = tile_rows; a.NQ = NQ; a.NP = NP;
        a.partials = partials;
        a.scale = 0.25f / ((float)S * (float)S);   // 2 / S^2 (C2R) / 8 (the omitted 1/2 factors, r2c_post / c2r_pre)
        return a;
    }
};

// FFT size per P: minimise S^2 log2(S) / T^2 (work per valid pixel), T = S - P + 1,
// over S <= 512; S = 1024 only when P leaves fewer than 64 valid rows at 512.
// Measured at P = 63 (c4, B200): S = 256 / 512 / 1024 -> 9856 / 9880 / 5924 Mpix-it/s;
// the 1024 kernels run 1 CTA per SM (smem) and are latency-bound.
static int choose_S(int P) {
    int best = 0;
    double bc = 1e300;
    for (int S = 64; S <= 512; S *= 2) {
        const int T = S - P + 1;
        if (T < 8) continue;
        const double c = (double)S * S * std::log2((double)S) / ((double)T * T);
        if (c < bc) { bc = c; best = S; }
    }
    if (512 - P + 1 < 64 && 1024 - P + 1 >= 8) best = 1024;
    return best;
}

int fft_choose_size(int P) { return choose_S(P); }

bool fft_prefer(int P) {
    // Measured crossover (profiles/r1/crossover.jsonl; 4096^2, 8x8 PSFs, 1 facet, B200):
    // direct 1.24 ms vs FFT 1.17 ms per step already at P = 7, FFT 5-80x faster from P = 15.
    return P >= 7;
}

template <int S>
static size_t smem_rows_fwd(int mode, bool tmx) {
    using G = GR<S>;
    if (S == 512 && mode != 0) return (size_t)ROWS_TW(S) * 8 + (size_t)G::NB * G::RS * 8;
    if (tmx) return (size_t)ROWS_TW(S) * 8 + (size_t)G::NB * G::RS * 8 + (size_t)S * 4;
    return (size_t)ROWS_TW(S) * 8 + (size_t)G::NB * G::RS * 8 + (size_t)G::NB * G::XS * 4 + (size_t)S * 4;
}
template <int S>
static size_t smem_cols(int NP, int NQ) {
    using G = GC<S>;
    return (size_t)S * 8 + (size_t)S * G::NB * 8 + 2 * (size_t)G::NB * G::CS * 8 + (size_t)NP * S * 4 + (size_t)NP * NQ * 4;
}
template <int S>
static size_t smem_rows_inv(int NQ, bool ht = true) {
    using G = GR<S>;
    return (size_t)ROWS_TW(S) * 8 + (size_t)G::NB * G::RS * 8 + (ht ? (size_t)G::NB * C2R<S>::SS * 8 + (size_t)NQ * S * 4 : 0);
}

// The dynamic-shared-memory limit is a property of the kernel function, shared by
// every handle in the process: only ever raise it (handles of different geometry
// need different sizes; lowering it would break a live handle's launches).
static std::mutex g_attr_mu;
template <typename K>
static cudaError_t raise_smem(K kern, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    if ((size_t)fa.maxDynamicSharedSizeBytes >= bytes) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int S>
static cudaError_t setup_attrs(int T, int NP, int NQ) {
    cudaError_t e;
    (void)T;
    if ((e = raise_smem(k_rows_fwd<S, false>, smem_rows_fwd<S>(0, false))) != cudaSuccess) return e;
    if constexpr (S == 512)
        if ((e = raise_smem(k_rows_fwd<S, true>, smem_rows_fwd<S>(0, true))) != cudaSuccess) return e;
    if ((e = raise_smem(k_cols<S>, smem_cols<S>(NP, NQ))) != cudaSuccess) return e;
    if constexpr (S == 512)
        if ((e = raise_smem(k_cols_tm<S>, smem_cols_tm<S>(NP, NQ))) != cudaSuccess) return e;
    if ((e = raise_smem(k_rows_inv<S, false>, smem_rows_inv<S>(NQ, false))) != cudaSuccess) return e;
    return raise_smem(k_rows_inv<S, true>, smem_rows_inv<S>(NQ));
}

template <int S>
static cudaError_t run_rows_fwd(const FftArgs &a, int ntiles, int mode, int par, const float *psfs, int npsf,
                                float2 *hrows, cudaStream_t s) {
    if (ntiles == 0) return cudaSuccess;
    if constexpr (S == 512) {
        if (mode == 0) {
            k_rows_fwd<S, true><<<ntiles * (S / GR<S>::NB), GR<S>::NTH, smem_rows_fwd<S>(mode, true), s>>>(a, mode, par, psfs, npsf, hrows);
            return cudaGetLastError();
        }
    }
    k_rows_fwd<S, false><<<ntiles * (S / GR<S>::NB), GR<S>::NTH, smem_rows_fwd<S>(mode, false), s>>>(a, mode, par, psfs, npsf, hrows);
    return cudaGetLastError();
}
template <int S>
static cudaError_t run_cols(const FftArgs &a, int ntiles, int mode, const float2 *hrows, float2 *hhat, int npsf,
                            const CUtensorMap *tmh, cudaStream_t s) {
    if (ntiles == 0) return cudaSuccess;
    const int nchunk = (S / 2 + 1 + GC<S>::NB - 1) / GC<S>::NB;
    if constexpr (S == 512) {
        if (mode != 2) {
            const int nck = mode == 0 ? (S / 2) / GCT<S>::NB : nchunk;
            // several chunks per CTA only while the grid keeps >= 4 waves of 2 CTAs per SM
            static const int nsm = [] {       // thread-safe one-time init (one GPU per process)
                int dev = 0, n = 0;
                cudaGetDevice(&dev);
                if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
                return n;
            }();
            int cpb = COLS_TM_CPB;
            while (cpb > 1 && (int64_t)ntiles * ((nck + cpb - 1) / cpb) < 8LL * nsm) --cpb;
            k_cols_tm<S><<<ntiles * ((nck + cpb - 1) / cpb), GCT<S>::NTH, smem_cols_tm<S>(a.NP, a.NQ), s>>>(a, mode, cpb,
                                                                                                      *tmh);
            return cudaGetLastError();
        }
    }
    k_cols<S><<<ntiles * nchunk, GC<S>::NTH, smem_cols<S>(a.NP, a.NQ), s>>>(a, mode, hrows, hhat, npsf);
    return cudaGetLastError();
}
template <int S>
static cudaError_t run_rows_inv(const FftArgs &a, int ntiles, int T, int mode, cudaStream_t s) {
    if (ntiles == 0) return cudaSuccess;
    const int nblk = (T + GR<S>::NB - 1) / GR<S>::NB;
    if (mode == INV_HT)
        k_rows_inv<S, true><<<ntiles * nblk, GR<S>::NTH, smem_rows_inv<S>(a.NQ, true), s>>>(a, mode);
    else
        k_rows_inv<S, false><<<ntiles * nblk, GR<S>::NTH, smem_rows_inv<S>(a.NQ, false), s>>>(a, mode);
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
                           const CUtensorMap *tmh, cudaStream_t s) {
    FFT_DISPATCH(S, return run_cols<SS>(a, nt, mode, hrows, hhat, npsf, tmh, s));
    return cudaSuccess;
}
static cudaError_t do_rows_inv(int S, const FftArgs &a, int nt, int T, int mode, cudaStream_t s) {
    FFT_DISPATCH(S, return run_rows_inv<SS>(a, nt, T, mode, s));
    return cudaSuccess;
}
template <int S>
static cudaError_t geom(int &ldf, int &nb) {
    ldf = LD<S>::LDF;
    nb = GR<S>::NB;
    return cudaSuccess;
}
static cudaError_t do_geom(int S, int &ldf, int &nb) {
    FFT_DISPATCH(S, return geom<SS>(ldf, nb));
    return cudaSuccess;
}
static cudaError_t do_attrs(int S, int T, int NP, int NQ) {
    FFT_DISPATCH(S, return setup_attrs<SS>(T, NP, NQ));
    return cudaSuccess;
}

FftPlan *fft_create(const Plan &pl, const std::vector<int> &local, const std::vector<FacetDev> &fh,
                    const float *d_psfs, const float *d_wy, const float *d_wx, int Gy, int Gx, const float *h_wy,
                    const float *h_wx, bool per_node, cudaStream_t s, std::string &err, int S_force,
                    const FftRegions *regions) {
    FftPlan *f = new FftPlan();
    auto fail = [&](const std::string &m) { err = m; delete f; return (FftPlan *)nullptr; };
#define FC(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) return fail(std::string(cudaGetErrorString(e_)) + " at " #call); \
    } while (0)
    f->P = pl.P;
    f->S = S_force ? S_force : choose_S(pl.P);
    if (const char *ov = std::getenv("DEBLUR_FFT_SIZE")) {      // measurement override (crossover sweeps)
        const int v = std::atoi(ov);
        if (v >= 64 && v <= 1024 && (v & (v - 1)) == 0 && v - pl.P + 1 >= 8) f->S = v;
    }
    if (!f->S) return fail("no FFT size fits P");
    f->T = f->S - f->P + 1;
    f->Gx = Gx;
    f->K = Gy * Gx;
    f->wy = d_wy; f->wx = d_wx; f->Ny = (int)pl.ny; f->Nx = (int)pl.nx;
    f->nlocal = (int)local.size();
    const int S = f->S, T = f->T, P = f->P;
    int LDF = 0, rows_nb = 0;
    if (do_geom(S, LDF, rows_nb) != cudaSuccess) return fail("bad FFT size");
    // active ranges
    auto range_nz = [](const float *w, int G, int64_t n, int64_t a, int64_t b, int &lo, int &hi) {
        a = std::max<int64_t>(0, a); b = std::min<int64_t>(n, b);
        lo = G; hi = -1;
        for (int g = 0; g < G; ++g)
            for (int64_t i = a; i < b; ++i)
                if (w[(int64_t)g * n + i] != 0.f) { lo = std::min(lo, g); hi = std::max(hi, g); break; }
    };
    std::vector<char> used(f->K, 0);
    for (size_t li = 0; li < fh.size(); ++li) {
        const FacetDev &F = fh[li];
        // per-node operator mode: every tile of facet (a, b) uses PSF (a, b) alone
        auto range = [&](const float *w, int G, int64_t n, int64_t a, int64_t b, int &lo, int &hi) {
            if (per_node) {
                lo = hi = (w == h_wy) ? pl.facets[F.id].fy : pl.facets[F.id].fx;
                return;
            }
            range_nz(w, G, n, a, b, lo, hi);
        };
        const std::vector<FftRect> allH{{0, F.my, 0, F.mx}}, allHT{{0, F.ny, 0, F.nx}};
        const auto &rH = regions ? regions->H[li] : allH;
        const auto &rHT = regions ? regions->HT[li] : allHT;
        for (const FftRect &R : rH)
            for (int y0 = R.y0; y0 < R.y1; y0 += T)
                for (int x0 = R.x0; x0 < R.x1; x0 += T) {
                    TileDesc t{(int)li, y0, x0, 0, -1, 0, -1, R.y1, R.x1};
                    range(h_wy, Gy, pl.ny, F.ey0 + y0, F.ey0 + std::min(y0 + S, F.ny), t.p0, t.p1);
                    range(h_wx, Gx, pl.nx, F.ex0 + x0, F.ex0 + std::min(x0 + S, F.nx), t.q0, t.q1);
                    if (t.q1 < t.q0) { t.q0 = 0; t.q1 = -1; }
                    f->tH.push_back(t);
                    f->tile_facet_H.push_back((int)li);
                }
        for (const FftRect &R : rHT)
            for (int y0 = R.y0; y0 < R.y1; y0 += T)
                for (int x0 = R.x0; x0 < R.x1; x0 += T) {
                    TileDesc t{(int)li, y0, x0, 0, -1, 0, -1, R.y1, R.x1};
                    range(h_wy, Gy, pl.ny, F.ey0 + y0, F.ey0 + std::min(y0 + T, F.ny), t.p0, t.p1);
                    range(h_wx, Gx, pl.nx, F.ex0 + x0, F.ex0 + std::min(x0 + T, F.nx), t.q0, t.q1);
                    if (t.q1 < t.q0) { t.q0 = 0; t.q1 = -1; }
                    f->tHT.push_back(t);
                }
    }
    // PSF-cell-major tile order: tiles with the same active PSF range run back to back, so
    // the CTAs in flight share their PSF spectra in L2
    {
        std::vector<int> ord(f->tH.size());
        for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
        auto key = [](const TileDesc &t) { return std::make_tuple(t.p0, t.q0, t.p1, t.q1); };
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key(f->tH[a]) < key(f->tH[b]); });
        std::vector<TileDesc> th;
        std::vector<int> tf;
        for (int i : ord) { th.push_back(f->tH[i]); tf.push_back(f->tile_facet_H[i]); }
        f->tH.swap(th);
        f->tile_facet_H.swap(tf);
        std::stable_sort(f->tHT.begin(), f->tHT.end(), [&](const TileDesc &a, const TileDesc &b) { return key(a) < key(b); });
    }
    for (auto *lst : {&f->tH, &f->tHT})
        for (auto &t : *lst) {
            f->NQ = std::max(f->NQ, t.q1 - t.q0 + 1);
            f->NP = std::max(f->NP, t.p1 - t.p0 + 1);
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
    f->nblk_inv = (T + rows_nb - 1) / rows_nb;
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
    FC(do_attrs(S, T, f->NP, f->NQ));
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
        FC(do_cols(S, a, n, 2, hrows, f->Hhat, n, nullptr, s));
        FC(cudaStreamSynchronize(s));
        cudaFree(d_sel);
        cudaFree(hrows);
    }
    if (S == 512) {
        // 2-D view of Hhat for the TMEM column pass: rows = pair-rows (nslots * S/2), each
        // LDF * 4 floats (pair-interleaved complex); box = S/2 pair-rows x 4 NB floats = one
        // column chunk of one PSF spectrum (32 KB), copied by a single TMA instruction
        static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                fn = nullptr;
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }();
        if (!encode) return fail("cuTensorMapEncodeTiled not available from the driver");
        const cuuint64_t dims[2] = {(cuuint64_t)LDF * 4, (cuuint64_t)nslots * (S / 2)};
        const cuuint64_t strides[1] = {(cuuint64_t)LDF * 16};
        const cuuint32_t box[2] = {(cuuint32_t)(4 * GCT<512>::NB), (cuuint32_t)(S / 2)};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = encode(&f->tmh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)f->Hhat, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled failed for the PSF spectra");
    }
#undef FC
    return f;
}

void fft_destroy(FftPlan *f) { delete f; }

cudaError_t fft_H_pass(FftPlan &f, int pass, const FacetDev *d_facets, int par, int mode, cudaStream_t s) {
    FftArgs a = f.args(d_facets, false);
    const int n = (int)f.tH.size();
    if (pass == 0) return do_rows_fwd(f.S, a, n, 0, par, nullptr, 0, nullptr, s);
    if (pass == 1) return do_cols(f.S, a, n, 0, nullptr, nullptr, 0, &f.tmh, s);
    return do_rows_inv(f.S, a, n, f.T, mode, s);
}

cudaError_t fft_HT_pass(FftPlan &f, int pass, const FacetDev *d_facets, cudaStream_t s) {
    FftArgs a = f.args(d_facets, true);
    const int n = (int)f.tHT.size();
    if (pass == 0) return do_rows_fwd(f.S, a, n, 1, 0, nullptr, 0, nullptr, s);
    if (pass == 1) return do_cols(f.S, a, n, 1, nullptr, nullptr, 0, &f.tmh, s);
    return do_rows_inv(f.S, a, n, f.T, INV_HT, s);
}

double fft_pass_bytes(const FftPlan &f, bool ht, int pass) {
    const double S = f.S, T = f.T, NF = f.S / 2 + 1;
    const double spec = S * NF * 8.0;       // one S x (S/2+1) complex spectrum
    const double ospec = T * NF * 8.0;      // T valid rows of it
    double b = 0.0;
    for (const TileDesc &t : (ht ? f.tHT : f.tH)) {
        const double nq = std::max(0, t.q1 - t.q0 + 1);
        if (!ht) {
            if (pass == 0) b += S * S * 4.0 + nq * spec;          // x window in, A_q out
            else if (pass == 1) b += nq * spec + ospec;            // A_q in, O out
            else b += ospec + T * T * 12.0;                        // O in; y, W in; r out
        } else {
            if (pass == 0) b += S * S * 4.0 + spec;               // r window in, R out
            else if (pass == 1) b += spec + nq * ospec;            // R in, B_q out
            else b += nq * ospec + T * T * 4.0;                    // B_q in, g out
        }
    }
    return b;
}

double fft_pass_flops(const FftPlan &f, bool ht, int pass) {
    const double S = f.S, T = f.T, NF = f.S / 2 + 1, lg = std::log2((double)f.S);
    const double cdft = 5.0 * S * lg, rdft = 2.5 * S * lg;   // one length-S transform
    double fl = 0.0;
    for (const TileDesc &t : (ht ? f.tHT : f.tH)) {
        const double nq = std::max(0, t.q1 - t.q0 + 1), npq = nq * std::max(0, t.p1 - t.p0 + 1);
        if (!ht) {
            if (pass == 0) fl += nq * S * (S + rdft);                           // x . wx_q, R2C per row
            else if (pass == 1) fl += NF * (npq * (2.0 * S + cdft + 8.0 * S) + cdft);   // wy_p, DFT, Hhat MAC; inverse
            else fl += T * rdft + 3.0 * T * T;                                   // C2R rows, W (Hx - y)
        } else {
            if (pass == 0) fl += S * rdft;                                       // R2C of the r window rows
            else if (pass == 1) fl += NF * (cdft + npq * (6.0 * S + cdft + 4.0 * S));  // DFT; conj Hhat, IDFT, wy_p MAC
            else fl += nq * T * (rdft + 2.0 * S);                                // C2R per q, wx_q MAC
        }
    }
    return fl;
}

int fft_tiles(const FftPlan &f, bool ht) { return (int)(ht ? f.tHT.size() : f.tH.size()); }

cudaError_t fft_data_partials(FftPlan &f, std::vector<double> &out) {
    out.assign(f.nlocal, 0.0);
    const size_t n = f.tH.size() * f.nblk_inv;
    cudaError_t e = cudaMemcpy(f.h_part.data(), f.partials, sizeof(double) * n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return e;
    for (size_t b = 0; b < n; ++b) out[f.tile_facet_H[b / f.nblk_inv]] += f.h_part[b];
    return cudaSuccess;
}

}  // namespace deblur
