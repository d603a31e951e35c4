// k_update.cu -- elementwise and band kernels of the hot path.
//
//  K4 k_update_from_g (rows a3-a4 when H^T comes from the FFT path): the same
//      fused TV-gradient / prox / projection / dual epilogue as K2, with g read
//      from the facet's g array.
//  K5 k_consensus (row a6, Lemma 1, update PAPER.md:201-202):
//      on band pixels only, zbar = sum_{f' ascending id} omega^F_{f'} v_{f'} /
//      sum omega^F_{f'} (A8, A9), u_f += rho (zbar - x+_f).  Neighbour values are
//      read through View descriptors: the neighbour's v array when it lives on
//      this GPU, the received halo buffer otherwise.
//  K6 k_tv_value / k_maxdiff (row a7): fp64 per-block partials of
//      sum phi(D x) and max |x_f - x_f'| over shared pixels (A22).
#include <cuda_pipeline.h>

#include "epilogue.cuh"
#include "kernels.hpp"

namespace deblur {
namespace {

constexpr int K4_MINB = 3;              // CTAs per SM of K4 (85 registers: no spills; 4 CTAs at 64 spilled ~150 B, same speed)
constexpr int UT_TY = 32, UT_TX = 128;   // update tile (matches the H^T tile grid)

// K4: tile of UT_TY x UT_TX pixels; each thread owns a 4-pixel strip in 4 rows.
// x halo staged with 16-byte loads (interior tiles) or a wrapped scalar path
// (tiles touching the facet border: circular D within the facet, A2).
template <int REG, bool NEU>
__global__ void __launch_bounds__(EPI_NT, K4_MINB) k_update_from_g(const FacetDev *facets, const TileDesc *tiles, int par,
                                                           int last, SolverConst sc, double *partials) {
    constexpr int XH = UT_TX + 8;                    // smem col c <-> facet col x0 - 4 + c
    __shared__ __align__(16) float xh[(UT_TY + 2) * XH];
    __shared__ double red[EPI_NT / 32];
    __shared__ __align__(16) float om_c[UT_TX];
    __shared__ float om_r[UT_TY];
    __shared__ __align__(4) unsigned char sb_c[UT_TX];
    __shared__ unsigned char sb_r[UT_TY];
    const TileDesc t = tiles[blockIdx.x];
    const FacetDev &F = facets[t.f];
    const float *__restrict__ x = F.x[par];
    const int tid = threadIdx.x;
    const bool interior = t.y0 >= 1 && t.y0 + UT_TY + 1 <= F.ny && t.x0 >= 4 && t.x0 + UT_TX + 4 <= F.nx;
    // every load of the CTA is in flight before the first wait: the x halo streams into
    // shared memory with 16-byte cp.async (interior tiles), g and u into registers
    if (interior) {
        constexpr int NV = XH / 4;                   // float4 per smem row
        for (int idx = tid; idx < (UT_TY + 2) * NV; idx += EPI_NT) {
            const int i = idx / NV, v = idx - i * NV;
            __pipeline_memcpy_async(xh + i * XH + 4 * v, x + (int64_t)(t.y0 - 1 + i) * F.ep + t.x0 - 4 + 4 * v, 16);
        }
        __pipeline_commit();
    }
    const int tx = tid & 31, ty = tid >> 5;          // 32 strips of 4 columns x 8 row groups
    constexpr int KR = UT_TY / 8;
    const int lx0 = 4 * tx, fx0 = t.x0 + lx0;
    const bool full = fx0 + 3 < F.nx;
    const float *__restrict__ gp = F.g;
    float *__restrict__ up = F.u;
    float *__restrict__ vp = F.v;
    float *__restrict__ xo = F.x[par ^ 1];
    float gv[KR][4], uv[KR][4];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
        const int fy = t.y0 + ty + 8 * k;
        const int64_t o = (int64_t)fy * F.ep + fx0;
        if (fy < F.ny && full) {
            const float4 g4 = __ldg(reinterpret_cast<const float4 *>(gp + o));
            const float4 u4 = *reinterpret_cast<const float4 *>(up + o);
            gv[k][0] = g4.x; gv[k][1] = g4.y; gv[k][2] = g4.z; gv[k][3] = g4.w;
            uv[k][0] = u4.x; uv[k][1] = u4.y; uv[k][2] = u4.z; uv[k][3] = u4.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool ok = fy < F.ny && fx0 + j < F.nx;
                gv[k][j] = ok ? gp[o + j] : 0.f;
                uv[k][j] = ok ? up[o + j] : 0.f;
            }
        }
    }
    // band membership and omega^F (A13 ramps or per-node weights) once per tile column
    // and row, into shared memory (in registers they would spill at 4 CTAs / SM)
    if (tid < UT_TX) {
        const int fx = t.x0 + tid;
        om_c[tid] = fx < F.nx ? omega_axis(F.ax, fx) : 1.f;
        sb_c[tid] = fx < F.ax.b_prev || fx >= F.ax.b_next;
    } else if (tid < UT_TX + UT_TY) {
        const int fy = t.y0 + tid - UT_TX;
        om_r[tid - UT_TX] = fy < F.ny ? omega_axis(F.ay, fy) : 1.f;
        sb_r[tid - UT_TX] = fy < F.ay.b_prev || fy >= F.ay.b_next;
    }
    if (!interior) {
        for (int idx = tid; idx < (UT_TY + 2) * XH; idx += EPI_NT) {
            const int i = idx / XH, c = idx - i * XH;
            int fy = t.y0 - 1 + i, fx = t.x0 - 4 + c;
            fy = ((fy % F.ny) + F.ny) % F.ny;
            fx = ((fx % F.nx) + F.nx) % F.nx;
            xh[idx] = x[(int64_t)fy * F.ep + fx];
        }
    } else {
        __pipeline_wait_prior(0);
    }
    __syncthreads();
    double rsum = 0.0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
        const int ly = ty + 8 * k;
        const int fy = t.y0 + ly;
        if (fy >= F.ny || fx0 >= F.nx) continue;
        const int64_t o = (int64_t)fy * F.ep + fx0;
        const bool shy = sb_r[ly];
        const float omy = om_r[ly];
        const float4 omx = *reinterpret_cast<const float4 *>(om_c + lx0);
        const uchar4 shx = *reinterpret_cast<const uchar4 *>(sb_c + lx0);
        const float omxj[4] = {omx.x, omx.y, omx.z, omx.w};
        const bool shxj[4] = {shx.x != 0, shx.y != 0, shx.z != 0, shx.w != 0};
        float xn[4], nu[4], nv[4];
        bool sh[4];
        if constexpr (REG == 0 && !NEU) {
            // the strip's TV gradient with shared psi evaluations (tv_grad4)
            float td[4], ph[4];
            tv_grad4(xh, XH, ly + 1, lx0 + 4, sc, partials != nullptr, td, ph);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                sh[j] = shy || shxj[j];
                const float xc = xh[(ly + 1) * XH + lx0 + 4 + j];
                const float gt = gv[k][j] + sc.lambda * td[j] + sc.gamma * (omy * omxj[j]) * (xc - uv[k][j]);
                xn[j] = fmaxf(0.f, xc - sc.tau * gt);
                nu[j] = uv[k][j] + sc.rho * (xn[j] - uv[k][j]);
                nv[j] = 2.f * xn[j] - uv[k][j];
                if (fx0 + j < F.nx) rsum += (double)ph[j];
            }
        } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int fx = fx0 + j;
            float phi;
            sh[j] = shy || shxj[j];
            xn[j] = update_value_t<REG, NEU>(F.ny, F.nx, xh, XH, ly + 1, lx0 + j + 4, fy, fx, gv[k][j], uv[k][j],
                                             omy * omxj[j], sc, partials != nullptr, phi, nu[j], nv[j]);
            if (fx < F.nx) rsum += (double)phi;
        }
        }
        if (full) {
            *reinterpret_cast<float4 *>(xo + o) = make_float4(xn[0], xn[1], xn[2], xn[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (fx0 + j < F.nx) xo[o + j] = xn[j];
        }
        if (last) {
            if (full && !sh[0] && !sh[1] && !sh[2] && !sh[3]) {
                *reinterpret_cast<float4 *>(up + o) = make_float4(nu[0], nu[1], nu[2], nu[3]);
            } else if (full && sh[0] && sh[1] && sh[2] && sh[3]) {
                *reinterpret_cast<float4 *>(vp + o) = make_float4(nv[0], nv[1], nv[2], nv[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (fx0 + j >= F.nx) continue;
                    if (sh[j]) vp[o + j] = nv[j];
                    else up[o + j] = nu[j];
                }
            }
        }
    }
    if (partials) {
        const double s2 = block_sum(rsum, red);
        if (tid == 0) partials[blockIdx.x] = s2;
    }
}

__global__ void __launch_bounds__(EPI_NT) k_tv_value(const FacetDev *facets, const TileDesc *tiles, int par,
                                                      SolverConst sc, double *partials) {
    __shared__ double red[EPI_NT / 32];
    const TileDesc t = tiles[blockIdx.x];
    const FacetDev &F = facets[t.f];
    const float *__restrict__ x = F.x[par];
    const bool neu = sc.tv_boundary == 1;
    const float e2 = sc.eps * sc.eps;
    double rsum = 0.0;
    for (int idx = threadIdx.x; idx < UT_TY * UT_TX; idx += EPI_NT) {
        const int fy = t.y0 + idx / UT_TX, fx = t.x0 + idx % UT_TX;
        if (fy >= F.ny || fx >= F.nx) continue;
        const int fy1 = (fy + 1 == F.ny) ? 0 : fy + 1, fx1 = (fx + 1 == F.nx) ? 0 : fx + 1;
        const float xc = x[(int64_t)fy * F.ep + fx];
        const float dy = (neu && fy == F.ny - 1) ? 0.f : x[(int64_t)fy1 * F.ep + fx] - xc;
        const float dx = (neu && fx == F.nx - 1) ? 0.f : x[(int64_t)fy * F.ep + fx1] - xc;
        const float t2 = dy * dy + dx * dx;
        float phi;
        if (sc.reg_kind == 0) {
            phi = t2 / (sqrtf(t2 + e2) + sc.eps);
        } else {
            const float tt = sqrtf(t2);
            phi = (tt <= sc.eps) ? 0.5f * t2 : sc.eps * (tt - 0.5f * sc.eps);
        }
        rsum += (double)phi;
    }
    const double s = block_sum(rsum, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__device__ __forceinline__ float view_at(const View &v, int par, int gy, int gx) {
    return v.base[par][(int64_t)(gy - v.y0) * v.pitch + (gx - v.x0)];
}

// one CTA per RectTile (CT_ROWS rows x 256 columns of a band piece).  The contributing
// neighbour offsets are constant on the piece: their descriptors (v pointer at this
// column, pitch, omega along x) are resolved once per thread and the rows' omega along
// y once per CTA (shared memory), so the row loop is loads + arithmetic only.
// K5_GR rows per load batch, 4 CTAs/SM (61 registers): per-node c4, where almost every pixel
// is shared by 4 facets, 7.2 -> 5.8 ms against 8 rows at 2 CTAs/SM (profiles/r1/SUMMARY.md)
constexpr int K5_GR = 2;                // rows whose loads are in flight together
constexpr int K5_MINB = 4;
__global__ void __launch_bounds__(256, K5_MINB) k_consensus(const FacetDev *facets, const BandRect *rects,
                                                   const RectTile *tiles, int par, float rho) {
    __shared__ float omy_s[2][CT_ROWS];
    const RectTile T = tiles[blockIdx.x];
    const BandRect R = rects[T.rect];
    const FacetDev &F = facets[R.f];
    const int gy0 = F.ey0 + T.y0;
    const int nr = min(CT_ROWS, R.y1 - T.y0);
    if (threadIdx.x < 2 * CT_ROWS) {
        const int a = threadIdx.x / CT_ROWS, r = threadIdx.x % CT_ROWS;
        const int dy = R.dy0 + a;
        const Neighbour &nb = F.nb[min(dy, 1) + 1][R.dx0 + 1];
        omy_s[a][r] = (dy <= R.dy1 && r < nr) ? omega_axis(nb.ay, gy0 + r - nb.ay.e0) : 0.f;
    }
    __syncthreads();
    const int lx = T.x0 + (int)threadIdx.x;
    if (lx >= R.x1) return;
    const int gx = F.ex0 + lx;
    const int ndx = R.dx1 - R.dx0 + 1, nc = (R.dy1 - R.dy0 + 1) * ndx;
    const float *vp[4];
    int64_t vpitch[4];
    float omx[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        vp[c] = nullptr; vpitch[c] = 0; omx[c] = 0.f;
        if (c < nc) {
            const int dy = R.dy0 + c / ndx, dx = R.dx0 + c % ndx;     // ascending facet id (A9)
            const Neighbour &nb = F.nb[dy + 1][dx + 1];
            vpitch[c] = nb.v.pitch;
            vp[c] = nb.v.base[par] + (int64_t)(gy0 - nb.v.y0) * nb.v.pitch + (gx - nb.v.x0);
            omx[c] = omega_axis(nb.ax, gx - nb.ax.e0);
        }
    }
    const int64_t ep = F.ep;
    float *__restrict__ up = F.u + (int64_t)T.y0 * ep + lx;
    const float *__restrict__ xp = F.x[par] + (int64_t)T.y0 * ep + lx;
    for (int g = 0; g < nr; g += K5_GR) {
        // every load of K5_GR rows in flight before the first use (v / x through the
        // read-only path: the u stores cannot alias them); more rows hold more registers
        // than 4 CTAs/SM allow
        float vv[K5_GR][4], xv[K5_GR], uv[K5_GR];
#pragma unroll
        for (int r = 0; r < K5_GR; ++r) {
            const bool ok = g + r < nr;
            const int64_t rr = g + r;
#pragma unroll
            for (int c = 0; c < 4; ++c) vv[r][c] = (ok && c < nc) ? __ldg(vp[c] + rr * vpitch[c]) : 0.f;
            xv[r] = ok ? __ldg(xp + rr * ep) : 0.f;
            uv[r] = ok ? up[rr * ep] : 0.f;
        }
#pragma unroll
        for (int r = 0; r < K5_GR; ++r) {
            if (g + r >= nr) break;
            float num = 0.f, den = 0.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c < nc) {
                    const float om = omy_s[c / ndx][g + r] * omx[c];
                    num += om * vv[r][c];
                    den += om;
                }
            }
            const float zbar = num / den;
            up[(int64_t)(g + r) * ep] = uv[r] + rho * (zbar - xv[r]);
        }
    }
}

__global__ void __launch_bounds__(256) k_maxdiff(const FacetDev *facets, const BandRect *rects, int par,
                                                 double *partials) {
    __shared__ float red[8];
    const BandRect R = rects[blockIdx.x];
    const FacetDev &F = facets[R.f];
    const int w = R.x1 - R.x0;
    const int64_t n = (int64_t)(R.y1 - R.y0) * w;
    float m = 0.f;
    for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) {
        const int ly = R.y0 + (int)(idx / w), lx = R.x0 + (int)(idx % w);
        const int gy = F.ey0 + ly, gx = F.ex0 + lx;
        const int dy0 = (ly < F.ay.b_prev) ? -1 : 0, dy1 = (ly >= F.ay.b_next) ? 1 : 0;
        const int dx0 = (lx < F.ax.b_prev) ? -1 : 0, dx1 = (lx >= F.ax.b_next) ? 1 : 0;
        const float xs = F.x[par][(int64_t)ly * F.ep + lx];
        for (int dy = dy0; dy <= dy1; ++dy)
            for (int dx = dx0; dx <= dx1; ++dx) {
                if (dy == 0 && dx == 0) continue;
                m = fmaxf(m, fabsf(xs - view_at(F.nb[dy + 1][dx + 1].x, par, gy, gx)));
            }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int i = 0; i < 8; ++i) t = fmaxf(t, red[i]);
        partials[blockIdx.x] = (double)t;
    }
}

// A6 default start: x0 = u0 = max(0, y edge-replicated into the c-wide margin),
// from a device copy of the observed rows/cols the facet needs (origin (dy0, dx0)).
__global__ void k_x0_from_y(FacetDev F, const float *ydil, int64_t dpitch, int dy0, int dx0, int My, int Mx, int c) {
    const int64_t n = (int64_t)F.ny * F.nx;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(idx / F.nx), q = (int)(idx % F.nx);
        const int yr = min(max(F.ey0 + r - c, 0), My - 1), yq = min(max(F.ex0 + q - c, 0), Mx - 1);
        const float v = fmaxf(0.f, ydil[(int64_t)(yr - dy0) * dpitch + (yq - dx0)]);
        const int64_t o = (int64_t)r * F.ep + q;
        F.x[0][o] = v;
        F.u[o] = v;
    }
}

// image += omega^F_f . x_f over the facet's estimate block (A7); launched per facet in id order
// img += omega^F_f x_f (A7); wsum (per-node mode) += omega_f for the normalisation
__global__ void k_blend(FacetDev F, int par, float *img, float *wsum, int64_t Nx) {
    const int64_t n = (int64_t)F.ny * F.nx;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(idx / F.nx), q = (int)(idx % F.nx);
        const float om = omega_axis(F.ay, r) * omega_axis(F.ax, q);
        const int64_t o = (int64_t)(F.ey0 + r) * Nx + F.ex0 + q;
        img[o] += om * F.x[par][(int64_t)r * F.ep + q];
        if (wsum) wsum[o] += om;
    }
}

__global__ void k_normalize(float *img, const float *wsum, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        img[i] /= wsum[i];
}

}  // namespace

cudaError_t launch_x0_from_y(const FacetDev &F, const float *ydil, int64_t dpitch, int dy0, int dx0, int My, int Mx,
                             int c, cudaStream_t s) {
    k_x0_from_y<<<1184, 256, 0, s>>>(F, ydil, dpitch, dy0, dx0, My, Mx, c);
    return cudaGetLastError();
}

cudaError_t launch_blend(const FacetDev &F, int par, float *img, float *wsum, int64_t Nx, cudaStream_t s) {
    k_blend<<<1184, 256, 0, s>>>(F, par, img, wsum, Nx);
    return cudaGetLastError();
}

cudaError_t launch_normalize(float *img, const float *wsum, int64_t n, cudaStream_t s) {
    k_normalize<<<1184, 256, 0, s>>>(img, wsum, n);
    return cudaGetLastError();
}

cudaError_t launch_update_from_g(const FacetDev *facets, const TileDesc *tiles, int ntiles, int, int par, int last,
                                 const SolverConst &sc, double *partials, cudaStream_t s) {
    if (!ntiles) return cudaSuccess;
    if (sc.reg_kind == 0 && sc.tv_boundary == 0)
        k_update_from_g<0, false><<<ntiles, EPI_NT, 0, s>>>(facets, tiles, par, last, sc, partials);
    else if (sc.reg_kind == 0)
        k_update_from_g<0, true><<<ntiles, EPI_NT, 0, s>>>(facets, tiles, par, last, sc, partials);
    else if (sc.tv_boundary == 0)
        k_update_from_g<1, false><<<ntiles, EPI_NT, 0, s>>>(facets, tiles, par, last, sc, partials);
    else
        k_update_from_g<1, true><<<ntiles, EPI_NT, 0, s>>>(facets, tiles, par, last, sc, partials);
    return cudaGetLastError();
}

cudaError_t launch_tv_value(const FacetDev *facets, const TileDesc *tiles, int ntiles, int, int par,
                            const SolverConst &sc, double *partials, cudaStream_t s) {
    if (!ntiles) return cudaSuccess;
    k_tv_value<<<ntiles, EPI_NT, 0, s>>>(facets, tiles, par, sc, partials);
    return cudaGetLastError();
}

cudaError_t launch_consensus(const FacetDev *facets, const BandRect *rects, const RectTile *tiles, int ntiles,
                             int par, float rho, cudaStream_t s) {
    if (!ntiles) return cudaSuccess;
    k_consensus<<<ntiles, 256, 0, s>>>(facets, rects, tiles, par, rho);
    return cudaGetLastError();
}

cudaError_t launch_maxdiff(const FacetDev *facets, const BandRect *rects, int nrect, int par, double *partials,
                           cudaStream_t s) {
    if (!nrect) return cudaSuccess;
    k_maxdiff<<<nrect, 256, 0, s>>>(facets, rects, par, partials);
    return cudaGetLastError();
}

}  // namespace deblur
