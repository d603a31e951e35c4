// k_direct.cu -- direct (FP32-FMA stencil) blur H / adjoint H^T with fused epilogues.
//
//  K1 k_H_direct: for an observed tile of facet f,
//      (H x)(i,j) = sum_k sum_{a,b} h_k[a][b] omega_k(i+2c-a, j+2c-b) x(i+2c-a, j+2c-b)
//      (PAPER.md:107 PSF interpolation, :109 valid region), epilogue
//      r = w (Hx - y) and the fp64 partial 1/2 sum w (Hx - y)^2 (Eq. (3)).
//  K2 k_HT_direct  (rows a2-a4): for an estimate tile,
//      g(p,q) = sum_k omega_k(p,q) sum_{a,b} h_k[a][b] r(p-2c+a, q-2c+b)   (r = 0 outside O_f)
//      epilogue: t = D^T psi(D x) (smoothed TV / Huber),
//      x+ = max(0, x - tau (g + lambda t + gamma omega^F (x - u)))  (Local-Solver step, R2;
//      alpha = gamma omega PAPER.md:206; iota_{>=0} PAPER.md:129), and on the last
//      inner step the single-owner dual update / band value v = 2x+ - u.
//
// Design: 256 threads = 16 (x) x 16 (y); each thread owns RY rows x
// 2 groups of 4 adjacent columns 64 apart (conflict-free LDS.128 of the input
// window), TX = 128 output columns per tile.  The omega_k-weighted input tile and
// the P x P taps of PSF k sit in shared memory; the inner loop is 8 taps x
// (RY x 8) outputs of FFMA per 6 LDS.128 of input and 2 broadcast LDS.128 of taps.
// Accumulation is blocked per tap row (A24: sequential fp32 accumulation fails the
// 1e-5 bar at P >= 63): a row partial over b is folded into the output with one
// FFMA by the row weight wy_p (H) or by omega_k (H^T).
#include <cstdio>

#include "epilogue.cuh"
#include "kernels.hpp"

namespace deblur {
namespace {

constexpr int BX = 16, BY = 16, NT = BX * BY;
constexpr int TX = 128;

__host__ __device__ constexpr int padP(int P) { return (P + 7) & ~7; }

// Accumulate one tap row-block: part[ry][*] += h[a][cb..cb+7] (.) window, for every
// ry whose tap row a = s - ry is valid.  xa/xb: 12-float windows of the two column groups.
template <int RY>
__device__ __forceinline__ void fma_block(float (&part)[RY][8], const float (&xa)[12], const float (&xb)[12],
                                          const float *__restrict__ hs, int Pp, int P, int s, int cb) {
#pragma unroll
    for (int ry = 0; ry < RY; ++ry) {
        const int a = s - ry;
        if (a >= 0 && a < P) {
            const float4 h0 = *reinterpret_cast<const float4 *>(hs + a * Pp + cb);
            const float4 h1 = *reinterpret_cast<const float4 *>(hs + a * Pp + cb + 4);
            const float hh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
            for (int bb = 0; bb < 8; ++bb) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    part[ry][j] = fmaf(hh[bb], xa[j + bb], part[ry][j]);
                    part[ry][4 + j] = fmaf(hh[bb], xb[j + bb], part[ry][4 + j]);
                }
            }
        }
    }
}

// Same as fma_block when every tap row a = s - ry (ry < RY) is valid: no branches, so
// all 2*RY tap loads and the window loads can be issued ahead of the FFMAs.
template <int RY>
__device__ __forceinline__ void fma_block_full(float (&part)[RY][8], const float (&xa)[12], const float (&xb)[12],
                                               const float *__restrict__ hs, int Pp, int s, int cb) {
    float hh[RY][8];
#pragma unroll
    for (int ry = 0; ry < RY; ++ry) {
        const float4 h0 = *reinterpret_cast<const float4 *>(hs + (s - ry) * Pp + cb);
        const float4 h1 = *reinterpret_cast<const float4 *>(hs + (s - ry) * Pp + cb + 4);
        hh[ry][0] = h0.x; hh[ry][1] = h0.y; hh[ry][2] = h0.z; hh[ry][3] = h0.w;
        hh[ry][4] = h1.x; hh[ry][5] = h1.y; hh[ry][6] = h1.z; hh[ry][7] = h1.w;
    }
#pragma unroll
    for (int ry = 0; ry < RY; ++ry)
#pragma unroll
        for (int bb = 0; bb < 8; ++bb)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                part[ry][j] = fmaf(hh[ry][bb], xa[j + bb], part[ry][j]);
                part[ry][4 + j] = fmaf(hh[ry][bb], xb[j + bb], part[ry][4 + j]);
            }
}

__device__ __forceinline__ void load12(float (&w)[12], const float *p) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    const float4 b = *reinterpret_cast<const float4 *>(p + 4);
    const float4 c = *reinterpret_cast<const float4 *>(p + 8);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    w[8] = c.x; w[9] = c.y; w[10] = c.z; w[11] = c.w;
}

// ---------------------------------------------------------------------------- K1
template <int RY>
__global__ void __launch_bounds__(NT) k_H_direct(ConvArgs A, int mode, int par) {
    extern __shared__ __align__(16) float sm[];
    constexpr int TY = RY * BY;
    const TileDesc t = A.tiles[blockIdx.x];
    const FacetDev &F = A.facets[t.f];
    const int P = A.P, Pp = padP(P), c2 = P - 1;
    const int XP = TX + Pp;
    const int rows = TY + c2;
    float *xs = sm;
    float *hs = sm + rows * XP;
    double *red = reinterpret_cast<double *>(hs + P * Pp);
    const int tid = threadIdx.x, tx = tid & (BX - 1), ty = tid / BX;
    const float *__restrict__ xin = F.x[par];
    const int fny = F.ny, fnx = F.nx;
    const int64_t ep = F.ep;

    float acc[RY][8];
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    for (int p = t.p0; p <= t.p1; ++p) {
        for (int q = t.q0; q <= t.q1; ++q) {
            __syncthreads();
            // W_k C_k x restricted to the tile footprint: x * wx_q (wy_p is folded per row below)
            const float *__restrict__ wxq = A.wx + (size_t)q * A.Nx + F.ex0;
            for (int rr = ty; rr < rows; rr += BY) {
                const int ly = t.y0 + rr;
                float *dst = xs + rr * XP;
                if (ly < fny) {
                    const float *src = xin + (size_t)ly * ep;
                    for (int cc = tx * 4; cc < XP; cc += 4 * BX) {
                        const int lx = t.x0 + cc;
                        float4 v;
                        if (lx + 3 < fnx) {
                            v = *reinterpret_cast<const float4 *>(src + lx);
                            v.x *= __ldg(wxq + lx); v.y *= __ldg(wxq + lx + 1);
                            v.z *= __ldg(wxq + lx + 2); v.w *= __ldg(wxq + lx + 3);
                        } else {
                            v.x = (lx < fnx) ? src[lx] * __ldg(wxq + lx) : 0.f;
                            v.y = (lx + 1 < fnx) ? src[lx + 1] * __ldg(wxq + lx + 1) : 0.f;
                            v.z = (lx + 2 < fnx) ? src[lx + 2] * __ldg(wxq + lx + 2) : 0.f;
                            v.w = 0.f;
                        }
                        *reinterpret_cast<float4 *>(dst + cc) = v;
                    }
                } else {
                    for (int cc = tx * 4; cc < XP; cc += 4 * BX)
                        *reinterpret_cast<float4 *>(dst + cc) = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            // taps of PSF k, flipped (true convolution, A17), zero-padded to Pp columns
            const float *__restrict__ h = A.psfs + (size_t)(p * A.Gx + q) * P * P;
            for (int i = tid; i < P * Pp; i += NT) {
                const int aa = i / Pp, bb = i - aa * Pp;
                hs[i] = (bb < P) ? h[(c2 - aa) * P + (c2 - bb)] : 0.f;
            }
            __syncthreads();

            const float *__restrict__ wyp = A.wy + (size_t)p * A.Ny + F.ey0 + t.y0 + ty * RY;
            const int rowlim = fny - t.y0 - ty * RY;
            for (int s = 0; s < RY + c2; ++s) {
                const float wys = (s < rowlim) ? __ldg(wyp + s) : 0.f;
                if (__all_sync(0xffffffffu, wys == 0.f)) continue;
                float part[RY][8];
#pragma unroll
                for (int i = 0; i < RY; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) part[i][j] = 0.f;
                const float *xr = xs + (ty * RY + s) * XP + tx * 4;
                if (s >= RY - 1 && s < P) {          // bulk: every tap row valid
                    for (int cb = 0; cb < Pp; cb += 8) {
                        float xa[12], xb[12];
                        load12(xa, xr + cb);
                        load12(xb, xr + 64 + cb);
                        fma_block_full<RY>(part, xa, xb, hs, Pp, s, cb);
                    }
                } else {
                    for (int cb = 0; cb < Pp; cb += 8) {
                        float xa[12], xb[12];
                        load12(xa, xr + cb);
                        load12(xb, xr + 64 + cb);
                        fma_block<RY>(part, xa, xb, hs, Pp, P, s, cb);
                    }
                }
#pragma unroll
                for (int ry = 0; ry < RY; ++ry) {
                    const int a = s - ry;
                    if (a >= 0 && a < P) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[ry][j] = fmaf(wys, part[ry][j], acc[ry][j]);
                    }
                }
            }
        }
    }

    // epilogue: r = w (Hx - y), fp64 data partial
    double dsum = 0.0;
#pragma unroll
    for (int ry = 0; ry < RY; ++ry) {
        const int oi = t.y0 + ty * RY + ry;
        if (oi >= F.my) continue;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int oj = t.x0 + g * 64 + tx * 4 + j;
                if (oj >= F.mx) continue;
                const int64_t o = (int64_t)oi * F.op + oj;
                const float hx = acc[ry][g * 4 + j];
                if (mode == H_PLAIN) {
                    F.r[o] = hx;
                } else {
                    const float wv = F.w ? F.w[o] : F.w_scalar;
                    const float d = hx - F.y[o];
                    if (mode == H_RESIDUAL) F.r[o] = wv * d;
                    dsum += 0.5 * (double)wv * (double)d * (double)d;
                }
            }
        }
    }
    if (A.partials && mode != H_PLAIN) {
        const double s = block_sum(dsum, red);
        if (tid == 0) A.partials[blockIdx.x] = s;
    }
}

}  // namespace

namespace {

// ---------------------------------------------------------------------------- K2
template <int RY>
__global__ void __launch_bounds__(NT) k_HT_direct(ConvArgs A, int mode, int par, int last, SolverConst sc) {
    extern __shared__ __align__(16) float sm[];
    constexpr int TY = RY * BY;
    const TileDesc t = A.tiles[blockIdx.x];
    const FacetDev &F = A.facets[t.f];
    const int P = A.P, Pp = padP(P), c2 = P - 1;
    const int XP = TX + Pp;
    const int rows = TY + c2;
    const int rbuf = max(rows * XP, (TY + 2) * (TX + 2));
    float *rs = sm;
    float *hs = sm + ((rbuf + 7) & ~7);
    double *red = reinterpret_cast<double *>(hs + P * Pp);
    const int tid = threadIdx.x, tx = tid & (BX - 1), ty = tid / BX;

    // r tile: observed rows y0-2c .. y0+TY-1, cols x0-2c .. ; r = 0 outside O_f
    for (int rr = ty; rr < rows; rr += BY) {
        const int ri = t.y0 - c2 + rr;
        float *dst = rs + rr * XP;
        const bool rowok = ri >= 0 && ri < F.my;
        const float *src = F.r + (int64_t)ri * F.op;
        for (int cc = tx; cc < XP; cc += BX) {
            const int rj = t.x0 - c2 + cc;
            dst[cc] = (rowok && rj >= 0 && rj < F.mx) ? src[rj] : 0.f;
        }
    }

    float gacc[RY][8];
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) gacc[i][j] = 0.f;

    const int oy = t.y0 + ty * RY;                  // first output row of this thread (facet-local)
    for (int p = t.p0; p <= t.p1; ++p) {
        for (int q = t.q0; q <= t.q1; ++q) {
            __syncthreads();
            const float *__restrict__ h = A.psfs + (size_t)(p * A.Gx + q) * P * P;
            for (int i = tid; i < P * Pp; i += NT) {
                const int aa = i / Pp, bb = i - aa * Pp;
                hs[i] = (bb < P) ? h[aa * P + bb] : 0.f;
            }
            __syncthreads();
            // omega_k at this thread's outputs (applied after the correlation, A16)
            float om[RY][8];
            unsigned rowmask = 0;
#pragma unroll
            for (int ry = 0; ry < RY; ++ry) {
                const int fy = oy + ry;
                const float wyv = (fy < F.ny) ? __ldg(A.wy + (size_t)p * A.Ny + F.ey0 + fy) : 0.f;
                if (__any_sync(0xffffffffu, wyv != 0.f)) rowmask |= 1u << ry;
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int fx = t.x0 + g * 64 + tx * 4 + j;
                        const float wxv = (fx < F.nx) ? __ldg(A.wx + (size_t)q * A.Nx + F.ex0 + fx) : 0.f;
                        om[ry][g * 4 + j] = wyv * wxv;
                    }
            }
            for (int s = 0; s < RY + c2; ++s) {
                unsigned need = 0;
#pragma unroll
                for (int ry = 0; ry < RY; ++ry)
                    if (s - ry >= 0 && s - ry < P) need |= rowmask & (1u << ry);
                if (!need) continue;
                float part[RY][8];
#pragma unroll
                for (int i = 0; i < RY; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) part[i][j] = 0.f;
                const float *xr = rs + (ty * RY + s) * XP + tx * 4;
                if (s >= RY - 1 && s < P) {
                    for (int cb = 0; cb < Pp; cb += 8) {
                        float xa[12], xb[12];
                        load12(xa, xr + cb);
                        load12(xb, xr + 64 + cb);
                        fma_block_full<RY>(part, xa, xb, hs, Pp, s, cb);
                    }
                } else {
                    for (int cb = 0; cb < Pp; cb += 8) {
                        float xa[12], xb[12];
                        load12(xa, xr + cb);
                        load12(xb, xr + 64 + cb);
                        fma_block<RY>(part, xa, xb, hs, Pp, P, s, cb);
                    }
                }
#pragma unroll
                for (int ry = 0; ry < RY; ++ry) {
                    const int a = s - ry;
                    if (a >= 0 && a < P) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) gacc[ry][j] = fmaf(om[ry][j], part[ry][j], gacc[ry][j]);
                    }
                }
            }
        }
    }

    if (mode == HT_PLAIN) {
#pragma unroll
        for (int ry = 0; ry < RY; ++ry) {
            const int fy = oy + ry;
            if (fy >= F.ny) continue;
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int fx = t.x0 + g * 64 + tx * 4 + j;
                    if (fx < F.nx) F.g[(int64_t)fy * F.ep + fx] = gacc[ry][g * 4 + j];
                }
        }
        return;
    }

    // fused update epilogue (a3 + a4)
    __syncthreads();
    constexpr int XH = TX + 2;
    stage_halo(F, rs, XH, TY + 2, t.y0, t.x0, par);
    __syncthreads();
    double rsum = 0.0;
#pragma unroll
    for (int ry = 0; ry < RY; ++ry) {
        const int fy = oy + ry;
        if (fy >= F.ny) continue;
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int lx = g * 64 + tx * 4 + j;
                const int fx = t.x0 + lx;
                if (fx >= F.nx) continue;
                rsum += (double)update_pixel(F, rs, XH, ty * RY + ry + 1, lx + 1, fy, fx, gacc[ry][g * 4 + j], par,
                                             last, sc);
            }
    }
    if (A.partials) {
        const double s = block_sum(rsum, red);
        if (tid == 0) A.partials[blockIdx.x] = s;
    }
}

constexpr int ry_H(int P) { return P <= 63 ? 4 : 2; }
constexpr int RY_HT = 2;

}  // namespace

bool direct_supported(int P) { return P >= 1 && direct_smem_H(P) <= 232448 && direct_smem_HT(P) <= 232448; }
int direct_ty_H(int P) { return ry_H(P) * BY; }
int direct_ty_HT(int) { return RY_HT * BY; }

size_t direct_smem_H(int P) {
    const int Pp = padP(P), TY = direct_ty_H(P);
    return ((size_t)(TY + P - 1) * (TX + Pp) + (size_t)P * Pp) * 4 + 64;
}

size_t direct_smem_HT(int P) {
    const int Pp = padP(P), TY = direct_ty_HT(P);
    size_t rbuf = std::max((size_t)(TY + P - 1) * (TX + Pp), (size_t)(TY + 2) * (TX + 2));
    rbuf = (rbuf + 7) & ~(size_t)7;
    return (rbuf + (size_t)P * Pp) * 4 + 64;
}

template <typename K>
static cudaError_t set_smem(K kern, size_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t launch_H_direct(const ConvArgs &a, int mode, int par, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    const size_t smem = direct_smem_H(a.P);
    cudaError_t e;
    if (ry_H(a.P) == 4) {
        if ((e = set_smem(k_H_direct<4>, smem)) != cudaSuccess) return e;
        k_H_direct<4><<<a.ntiles, NT, smem, s>>>(a, mode, par);
    } else {
        if ((e = set_smem(k_H_direct<2>, smem)) != cudaSuccess) return e;
        k_H_direct<2><<<a.ntiles, NT, smem, s>>>(a, mode, par);
    }
    return cudaGetLastError();
}

cudaError_t launch_HT_direct(const ConvArgs &a, int mode, int par, int last, const SolverConst &sc, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    const size_t smem = direct_smem_HT(a.P);
    cudaError_t e;
    if ((e = set_smem(k_HT_direct<RY_HT>, smem)) != cudaSuccess) return e;
    k_HT_direct<RY_HT><<<a.ntiles, NT, smem, s>>>(a, mode, par, last, sc);
    return cudaGetLastError();
}

}  // namespace deblur
