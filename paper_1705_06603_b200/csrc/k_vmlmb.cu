// k_vmlmb.cu -- vector kernels of the VMLM-B Local-Solver (PAPER.md:287,
// :290; reading V1-V6 in DESIGN.md §2 / oracle/vmlmb.py).
//
// Every kernel runs over the H^T tile grid (32 x 128 estimate pixels per CTA, all
// local facets in one launch) and, where a scalar is needed, writes one fp64
// partial per tile; the host sums a facet's partials in tile order (deterministic,
// independent of the GPU count) and takes the line-search / memory decisions in
// fp64.  Per-facet vectors and coefficients arrive by value in VmArgs.
#include "epilogue.cuh"
#include "vmlmb.hpp"

namespace deblur {
namespace {

constexpr int VT_Y = 32, VT_X = 128, VNT = 256;

__device__ __forceinline__ double block_sum3(double v, double *red, int which) {
    // one of up to three independent block sums (red holds 3 x 8 doubles)
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[which * 8 + (threadIdx.x >> 5)] = v;
    return v;
}
__device__ __forceinline__ void block_finish(double *red, int nsum, double *out, int ntiles) {
    __syncthreads();
    if (threadIdx.x < nsum) {
        double t = 0.0;
        for (int i = 0; i < VNT / 32; ++i) t += red[threadIdx.x * 8 + i];
        out[(int64_t)threadIdx.x * ntiles + blockIdx.x] = t;
    }
}

// iterate the tile in groups of 4 consecutive pixels of a row (a warp covers one
// 128-pixel row: 512-byte coalesced accesses, 16-byte vectors when the group is
// whole): fn(offset o of the first pixel, facet row fy, facet col fx, count nv)
template <typename Fn>
__device__ __forceinline__ void for_tile4(const FacetDev &F, const TileDesc &t, Fn fn) {
#pragma unroll
    for (int i = 0; i < VT_Y * VT_X / 4 / VNT; ++i) {
        const int gi = threadIdx.x + VNT * i;
        const int fy = t.y0 + (gi >> 5), fx = t.x0 + 4 * (gi & 31);
        if (fy < F.ny && fx < F.nx) fn((int64_t)fy * F.ep + fx, fy, fx, min(4, F.nx - fx));
    }
}
__device__ __forceinline__ void ld4(const float *p, int nv, float (&v)[4]) {
    if (nv == 4) {
        const float4 q = *reinterpret_cast<const float4 *>(p);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = j < nv ? p[j] : 0.f;
    }
}
__device__ __forceinline__ void st4(float *p, int nv, const float (&v)[4]) {
    if (nv == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < nv) p[j] = v[j];
    }
}
__device__ __forceinline__ void ldm4(const uint8_t *p, int nv, bool (&m)[4]) {
    if (nv == 4) {
        const uchar4 q = *reinterpret_cast<const uchar4 *>(p);
        m[0] = q.x; m[1] = q.y; m[2] = q.z; m[3] = q.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = j < nv ? p[j] != 0 : false;
    }
}

// M = free set (x > 0 or g < 0) (V2);  A = M ? G : 0  (q of the two-loop)
__global__ void __launch_bounds__(VNT) k_mask_q(VmArgs a) {
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    const float *x = F.x[a.par];
    float *q = a.A[t.f];
    const float *g = a.B[t.f];
    uint8_t *m = a.Mo[t.f];
    for_tile4(F, t, [&](int64_t o, int, int, int nv) {
        float xv[4], gv[4], qv[4];
        ld4(x + o, nv, xv);
        ld4(g + o, nv, gv);
        uchar4 mv;
        bool fr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            fr[j] = xv[j] > 0.f || gv[j] < 0.f;
            qv[j] = fr[j] ? gv[j] : 0.f;
        }
        mv = make_uchar4(fr[0], fr[1], fr[2], fr[3]);
        if (nv == 4) *reinterpret_cast<uchar4 *>(m + o) = mv;
        else for (int j = 0; j < nv; ++j) m[o + j] = fr[j];
        st4(q + o, nv, qv);
    });
}

// partial <B, C> (and <B, B>, <C, C> when a.nsum == 3)
__global__ void __launch_bounds__(VNT) k_dot(VmArgs a) {
    __shared__ double red[3 * 8];
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    const float *b = a.B[t.f], *c = a.C[t.f];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for_tile4(F, t, [&](int64_t o, int, int, int nv) {
        float bv[4], cv[4];
        ld4(b + o, nv, bv);
        ld4(c + o, nv, cv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            s0 += (double)bv[j] * cv[j];
            s1 += (double)bv[j] * bv[j];
            s2 += (double)cv[j] * cv[j];
        }
    });
    block_sum3(s0, red, 0);
    if (a.nsum > 1) block_sum3(s1, red, 1);
    if (a.nsum > 2) block_sum3(s2, red, 2);
    block_finish(red, a.nsum, a.partials, a.ntiles);
}

// A = c1 * A + c0 * (M ? B : 0);  partial <C, A_new> if C != NULL
__global__ void __launch_bounds__(VNT) k_axpy_dot(VmArgs a) {
    __shared__ double red[3 * 8];
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    float *A = a.A[t.f];
    const float *B = a.B[t.f], *C = a.C[t.f];
    const uint8_t *M = a.M[t.f];
    const float c0 = (float)a.c0[t.f], c1 = (float)a.c1[t.f];
    double s = 0.0;
    for_tile4(F, t, [&](int64_t o, int, int, int nv) {
        float av[4], bv[4] = {0.f, 0.f, 0.f, 0.f}, cv[4];
        bool mv[4];
        ld4(A + o, nv, av);
        if (B) {
            ld4(B + o, nv, bv);
            ldm4(M + o, nv, mv);
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = mv[j] ? bv[j] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) av[j] = c1 * av[j] + c0 * bv[j];
        st4(A + o, nv, av);
        if (C) {
            ld4(C + o, nv, cv);
#pragma unroll
            for (int j = 0; j < 4; ++j) s += (double)cv[j] * (double)av[j];
        }
    });
    if (a.nsum) {
        block_sum3(s, red, 0);
        block_finish(red, 1, a.partials, a.ntiles);
    }
}

// direction D = -(M ? R : 0) where c0 == 0, else the reset D = -c0 (M ? G : 0);
// partial <G, D> (descent check, V3)
__global__ void __launch_bounds__(VNT) k_direction(VmArgs a) {
    __shared__ double red[3 * 8];
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    const float *R = a.B[t.f], *G = a.C[t.f];
    float *D = a.A[t.f];
    const uint8_t *M = a.M[t.f];
    const float h0 = (float)a.c0[t.f];
    const bool reset = a.c0[t.f] != 0.0;
    double s = 0.0;
    for_tile4(F, t, [&](int64_t o, int, int, int nv) {
        float rv[4], gv[4], dv[4];
        bool mv[4];
        ld4(R + o, nv, rv);
        ld4(G + o, nv, gv);
        ldm4(M + o, nv, mv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            dv[j] = mv[j] ? (reset ? -h0 * gv[j] : -rv[j]) : 0.f;
            s += (double)gv[j] * (double)dv[j];
        }
        st4(D + o, nv, dv);
    });
    block_sum3(s, red, 0);
    block_finish(red, 1, a.partials, a.ntiles);
}

// trial point x[par^1] = max(0, x[par] + t D) (V1, V4); partial <G, x_t - x>
__global__ void __launch_bounds__(VNT) k_trial(VmArgs a) {
    __shared__ double red[3 * 8];
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    const float *x = F.x[a.par];
    float *xn = F.x[a.par ^ 1];
    const float *D = a.B[t.f], *G = a.C[t.f];
    const float step = (float)a.c0[t.f];
    double s = 0.0;
    for_tile4(F, t, [&](int64_t o, int, int, int nv) {
        float xv[4], dv[4], gv[4], nvv[4];
        ld4(x + o, nv, xv);
        ld4(D + o, nv, dv);
        ld4(G + o, nv, gv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            nvv[j] = fmaxf(0.f, xv[j] + step * dv[j]);
            s += (double)gv[j] * ((double)nvv[j] - (double)xv[j]);
        }
        st4(xn + o, nv, nvv);
    });
    block_sum3(s, red, 0);
    block_finish(red, 1, a.partials, a.ntiles);
}

// memory pair S = x[par^1] - x[par], Y = Gn - G (V5); partials <s,y>, <s,s>, <y,y>
__global__ void __launch_bounds__(VNT) k_pair(VmArgs a) {
    __shared__ double red[3 * 8];
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    const float *x = F.x[a.par], *xn = F.x[a.par ^ 1];
    const float *G = a.B[t.f], *Gn = a.C[t.f];
    float *S = a.A[t.f], *Y = a.A2[t.f];
    double sy = 0.0, ss = 0.0, yy = 0.0;
    for_tile4(F, t, [&](int64_t o, int, int, int nv) {
        float xv[4], xnv[4], gv[4], gnv[4], sv[4], yv[4];
        ld4(x + o, nv, xv);
        ld4(xn + o, nv, xnv);
        ld4(G + o, nv, gv);
        ld4(Gn + o, nv, gnv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            sv[j] = xnv[j] - xv[j];
            yv[j] = gnv[j] - gv[j];
            sy += (double)sv[j] * yv[j];
            ss += (double)sv[j] * sv[j];
            yy += (double)yv[j] * yv[j];
        }
        st4(S + o, nv, sv);
        st4(Y + o, nv, yv);
    });
    block_sum3(sy, red, 0);
    block_sum3(ss, red, 1);
    block_sum3(yy, red, 2);
    block_finish(red, 3, a.partials, a.ntiles);
}

// full local gradient G = g_data + lambda D^T psi(D x) + gamma omega (x - u) at x[par]
// (g_data = H_f^T W (H_f x - y) already in F.g) and the partials lambda-free
// sum phi(D x) and 1/2 sum gamma omega (x - u)^2 of the local objective value
template <int REG, bool NEU>
__global__ void __launch_bounds__(VNT) k_grad(VmArgs a, SolverConst sc) {
    constexpr int XH = VT_X + 8;
    __shared__ __align__(16) float xh[(VT_Y + 2) * XH];
    __shared__ double red[3 * 8];
    __shared__ float om_c[VT_X], om_r[VT_Y];
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    const float *__restrict__ x = F.x[a.par];
    const bool interior = t.y0 >= 1 && t.y0 + VT_Y + 1 <= F.ny && t.x0 >= 4 && t.x0 + VT_X + 4 <= F.nx;
    if (interior) {            // 16-byte loads, all in flight (row starts x0 - 4: 16-byte aligned)
        constexpr int NV = XH / 4;
        constexpr int PER = ((VT_Y + 2) * NV + VNT - 1) / VNT;
        float4 tmp[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int idx = threadIdx.x + VNT * k;
            if (idx < (VT_Y + 2) * NV) {
                const int i = idx / NV, v = idx - i * NV;
                tmp[k] = __ldg(reinterpret_cast<const float4 *>(x + (int64_t)(t.y0 - 1 + i) * F.ep + t.x0 - 4) + v);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int idx = threadIdx.x + VNT * k;
            if (idx < (VT_Y + 2) * NV) *reinterpret_cast<float4 *>(xh + 4 * idx) = tmp[k];
        }
    } else {
        for (int idx = threadIdx.x; idx < (VT_Y + 2) * XH; idx += VNT) {
            const int i = idx / XH, c = idx - i * XH;
            int fy = t.y0 - 1 + i, fx = t.x0 - 4 + c;
            fy = ((fy % F.ny) + F.ny) % F.ny;
            fx = ((fx % F.nx) + F.nx) % F.nx;
            xh[idx] = x[(int64_t)fy * F.ep + fx];
        }
    }
    // omega^F once per tile column / row (A13 ramps are 1 off the bands, so the product is the
    // pixel's weight everywhere; per-node weight rows likewise)
    if (threadIdx.x < VT_X) {
        const int fx = t.x0 + threadIdx.x;
        om_c[threadIdx.x] = fx < F.nx ? omega_axis(F.ax, fx) : 1.f;
    } else if (threadIdx.x < VT_X + VT_Y) {
        const int fy = t.y0 + threadIdx.x - VT_X;
        om_r[threadIdx.x - VT_X] = fy < F.ny ? omega_axis(F.ay, fy) : 1.f;
    }
    __syncthreads();
    // facet fields in registers: the G stores could alias them for the compiler
    float *__restrict__ G = a.A[t.f];
    const float *__restrict__ up = F.u;
    const float *__restrict__ gp = F.g;
    const int ny = F.ny, nx = F.nx;
    const int64_t ep = F.ep;
    double reg = 0.0, prox = 0.0;
#pragma unroll
    for (int i = 0; i < VT_Y * VT_X / 4 / VNT; ++i) {
        const int gi = threadIdx.x + VNT * i;
        const int ly = gi >> 5, lx4 = 4 * (gi & 31);
        const int fy = t.y0 + ly, fx4 = t.x0 + lx4;
        if (fy >= ny || fx4 >= nx) continue;
        const int nv = min(4, nx - fx4);
        const int64_t o4 = (int64_t)fy * ep + fx4;
        float uv[4], gv[4], out[4];
        ld4(up + o4, nv, uv);
        ld4(gp + o4, nv, gv);
        const float omy = om_r[ly];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int fx = fx4 + jj;
            float phi;
            const float tdiv = tv_grad_t<REG, NEU>(ny, nx, xh, XH, ly + 1, lx4 + jj + 4, fy, fx, sc, true, phi);
            const float xc = xh[(ly + 1) * XH + lx4 + jj + 4], uc = uv[jj];
            const float om = omy * om_c[lx4 + jj];
            out[jj] = gv[jj] + sc.lambda * tdiv + sc.gamma * om * (xc - uc);
            if (jj < nv) {
                reg += (double)phi;
                prox += 0.5 * (double)sc.gamma * (double)om * ((double)xc - uc) * ((double)xc - uc);
            }
        }
        st4(G + o4, nv, out);
    }
    block_sum3(reg, red, 0);
    block_sum3(prox, red, 1);
    block_finish(red, 2, a.partials, a.ntiles);
}

// end of the Local-Solver at x[par]: single owners u += rho (x - u); band pixels
// v = 2x - u (what the last projected-gradient step's epilogue writes)
__global__ void __launch_bounds__(VNT) k_finalize(VmArgs a, float rho) {
    const TileDesc t = a.tiles[blockIdx.x];
    const FacetDev &F = a.facets[t.f];
    const float *x = F.x[a.par];
    for_tile4(F, t, [&](int64_t o4, int fy, int fx4, int nv) {
        for (int jj = 0; jj < nv; ++jj) {
            const int fx = fx4 + jj;
            const int64_t o = o4 + jj;
            const bool shared = fy < F.ay.b_prev || fy >= F.ay.b_next || fx < F.ax.b_prev || fx >= F.ax.b_next;
            const float uc = F.u[o];
            if (shared) F.v[o] = 2.f * x[o] - uc;
            else F.u[o] = uc + rho * (x[o] - uc);
        }
    });
}

}  // namespace

#define VM_LAUNCH(kern, ...)                                                     \
    do {                                                                         \
        if (a.ntiles == 0) return cudaSuccess;                                   \
        kern<<<a.ntiles, VNT, 0, s>>>(__VA_ARGS__);                              \
        return cudaGetLastError();                                               \
    } while (0)

cudaError_t vm_mask_q(const VmArgs &a, cudaStream_t s) { VM_LAUNCH(k_mask_q, a); }
cudaError_t vm_dot(const VmArgs &a, cudaStream_t s) { VM_LAUNCH(k_dot, a); }
cudaError_t vm_axpy_dot(const VmArgs &a, cudaStream_t s) { VM_LAUNCH(k_axpy_dot, a); }
cudaError_t vm_direction(const VmArgs &a, cudaStream_t s) { VM_LAUNCH(k_direction, a); }
cudaError_t vm_trial(const VmArgs &a, cudaStream_t s) { VM_LAUNCH(k_trial, a); }
cudaError_t vm_pair(const VmArgs &a, cudaStream_t s) { VM_LAUNCH(k_pair, a); }
cudaError_t vm_finalize(const VmArgs &a, float rho, cudaStream_t s) { VM_LAUNCH(k_finalize, a, rho); }
cudaError_t vm_grad(const VmArgs &a, const SolverConst &sc, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    if (sc.reg_kind == 0 && sc.tv_boundary == 0) k_grad<0, false><<<a.ntiles, VNT, 0, s>>>(a, sc);
    else if (sc.reg_kind == 0) k_grad<0, true><<<a.ntiles, VNT, 0, s>>>(a, sc);
    else if (sc.tv_boundary == 0) k_grad<1, false><<<a.ntiles, VNT, 0, s>>>(a, sc);
    else k_grad<1, true><<<a.ntiles, VNT, 0, s>>>(a, sc);
    return cudaGetLastError();
}

}  // namespace deblur
