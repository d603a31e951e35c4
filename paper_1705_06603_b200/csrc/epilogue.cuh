// epilogue.cuh -- device helpers shared by the direct and FFT paths (internal).
#pragma once
#include "device.cuh"

namespace deblur {

constexpr int EPI_NT = 256;

template <int NT = EPI_NT>
__device__ __forceinline__ double block_sum(double v, double *scratch) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; ++i) t += scratch[i];
    return t;
}

// ----------------------------------------------------------------- shared epilogue
// TV gradient + prox + projection + dual/band update for one output pixel, reading
// x from a (TYh+2) x (TXh+2) smem halo tile xh whose element (i, j) holds facet
// pixel (wrap(y0-1+i), wrap(x0-1+j)).  Returns phi(D x) at the pixel (reg partial).
__device__ __forceinline__ float update_pixel(const FacetDev &F, const float *xh, int XH, int i, int j, int fy, int fx, float g,
                              int par, int last, const SolverConst &sc) {
    const int ny = F.ny, nx = F.nx;
    const bool neu = sc.tv_boundary == 1;
    const float e2 = sc.eps * sc.eps;
    auto X = [&](int a, int b) { return xh[a * XH + b]; };
    const int fyu = (fy == 0) ? ny - 1 : fy - 1;
    const int fxl = (fx == 0) ? nx - 1 : fx - 1;
    // D x at (i,j), (i-1,j), (i,j-1): forward differences, circular or Neumann
    const float xc = X(i, j);
    const float dyc = (neu && fy == ny - 1) ? 0.f : X(i + 1, j) - xc;
    const float dxc = (neu && fx == nx - 1) ? 0.f : X(i, j + 1) - xc;
    const float dyu = (neu && fyu == ny - 1) ? 0.f : xc - X(i - 1, j);
    const float dxu = (neu && fx == nx - 1) ? 0.f : X(i - 1, j + 1) - X(i - 1, j);
    const float dyl = (neu && fy == ny - 1) ? 0.f : X(i + 1, j - 1) - X(i, j - 1);
    const float dxl = (neu && fxl == nx - 1) ? 0.f : xc - X(i, j - 1);
    float sc_c, sc_u, sc_l, phi;
    const float t2c = dyc * dyc + dxc * dxc;
    if (sc.reg_kind == 0) {
        const float rc = sqrtf(t2c + e2);
        sc_c = 1.f / rc;
        sc_u = 1.f / sqrtf(dyu * dyu + dxu * dxu + e2);
        sc_l = 1.f / sqrtf(dyl * dyl + dxl * dxl + e2);
        phi = t2c / (rc + sc.eps);                       // sqrt(t2+e2) - eps without cancellation
    } else {
        const float d = sc.eps;
        const float tc = sqrtf(t2c), tu = sqrtf(dyu * dyu + dxu * dxu), tl = sqrtf(dyl * dyl + dxl * dxl);
        sc_c = (tc <= d) ? 1.f : d / tc;
        sc_u = (tu <= d) ? 1.f : d / tu;
        sc_l = (tl <= d) ? 1.f : d / tl;
        phi = (tc <= d) ? 0.5f * t2c : d * (tc - 0.5f * d);
    }
    // D^T psi(D x): psi_y(p-1) - psi_y(p) + psi_x(q-1) - psi_x(q)
    const float tdiv = dyu * sc_u - dyc * sc_c + dxl * sc_l - dxc * sc_c;
    const int64_t o = (int64_t)fy * F.ep + fx;
    const float uc = F.u[o];
    const float om = omega_axis(F.ay, fy) * omega_axis(F.ax, fx);
    const float gt = g + sc.lambda * tdiv + sc.gamma * om * (xc - uc);
    const float xn = fmaxf(0.f, xc - sc.tau * gt);
    F.x[par ^ 1][o] = xn;
    if (last) {
        const bool shared = fy < F.ay.b_prev || fy >= F.ay.b_next || fx < F.ax.b_prev || fx >= F.ax.b_next;
        if (!shared)
            F.u[o] = uc + sc.rho * (xn - uc);      // single owner: zbar = 2x+ - u (Lemma 1 with one term)
        else
            F.v[o] = 2.f * xn - uc;                // band value sent to the consensus
    }
    return phi;
}

// TV gradient (D^T psi(D x))(i, j) from the smem halo tile (the divergence form
// psi_y(i-1,j) - psi_y(i,j) + psi_x(i,j-1) - psi_x(i,j)) and, if asked, phi(D x)(i, j).
// Compile-time regulariser / D boundary (REG: 0 smoothed TV, 1 Huber; NEU: Neumann).
template <int REG, bool NEU>
__device__ __forceinline__ float tv_grad_t(int ny, int nx, const float *xh, int XH, int i, int j, int fy, int fx,
                                           const SolverConst &sc, bool want_phi, float &phi) {
    const float e2 = sc.eps * sc.eps;
    auto X = [&](int a, int b) { return xh[a * XH + b]; };
    const float xc = X(i, j);
    float dyc = X(i + 1, j) - xc;
    float dxc = X(i, j + 1) - xc;
    float dyu = xc - X(i - 1, j);
    float dxu = X(i - 1, j + 1) - X(i - 1, j);
    float dyl = X(i + 1, j - 1) - X(i, j - 1);
    float dxl = xc - X(i, j - 1);
    if (NEU) {
        const int fyu = (fy == 0) ? ny - 1 : fy - 1;
        const int fxl = (fx == 0) ? nx - 1 : fx - 1;
        if (fy == ny - 1) { dyc = 0.f; dyl = 0.f; }
        if (fx == nx - 1) { dxc = 0.f; dxu = 0.f; }
        if (fyu == ny - 1) dyu = 0.f;
        if (fxl == nx - 1) dxl = 0.f;
    }
    float sc_c, sc_u, sc_l;
    const float t2c = dyc * dyc + dxc * dxc;
    phi = 0.f;
    if (REG == 0) {
        sc_c = rsqrtf(t2c + e2);
        sc_u = rsqrtf(dyu * dyu + dxu * dxu + e2);
        sc_l = rsqrtf(dyl * dyl + dxl * dxl + e2);
        if (want_phi) phi = t2c / (sqrtf(t2c + e2) + sc.eps);
    } else {
        const float d = sc.eps;
        const float tc = sqrtf(t2c), tu = sqrtf(dyu * dyu + dxu * dxu), tl = sqrtf(dyl * dyl + dxl * dxl);
        sc_c = (tc <= d) ? 1.f : d / tc;
        sc_u = (tu <= d) ? 1.f : d / tu;
        sc_l = (tl <= d) ? 1.f : d / tl;
        if (want_phi) phi = (tc <= d) ? 0.5f * t2c : d * (tc - 0.5f * d);
    }
    return dyu * sc_u - dyc * sc_c + dxl * sc_l - dxc * sc_c;
}

// Same arithmetic as update_pixel, returning x+ and the dual/band values instead of
// storing them (the caller vectorises the stores and supplies omega^F at the pixel,
// computed once per row and column); phi is computed only when asked.
template <int REG, bool NEU>
__device__ __forceinline__ float update_value_t(int ny, int nx, const float *xh, int XH, int i, int j, int fy, int fx,
                                                float g, float uc, float om, const SolverConst &sc, bool want_phi,
                                                float &phi, float &u_new, float &v_new) {
    const float xc = xh[i * XH + j];
    const float tdiv = tv_grad_t<REG, NEU>(ny, nx, xh, XH, i, j, fy, fx, sc, want_phi, phi);
    const float gt = g + sc.lambda * tdiv + sc.gamma * om * (xc - uc);
    const float xn = fmaxf(0.f, xc - sc.tau * gt);
    u_new = uc + sc.rho * (xn - uc);
    v_new = 2.f * xn - uc;
    return xn;
}

// TV gradient of 4 adjacent pixels (i, j .. j+3) of one row, smoothed TV with the circular D
// (the path of the north-star step): psi_x(q - 1) of pixel q is psi(q - 1) of its left
// neighbour in the strip, so the strip needs psi at (i, j-1 .. j+3) and (i-1, j .. j+3):
// 9 reciprocal square roots instead of 12, each with the same operands as tv_grad_t's.
__device__ __forceinline__ void tv_grad4(const float *xh, int XH, int i, int j, const SolverConst &sc,
                                         bool want_phi, float (&td)[4], float (&phi)[4]) {
    const float e2 = sc.eps * sc.eps;
    const float *r0 = xh + (i - 1) * XH + j, *r1 = xh + i * XH + j, *r2 = xh + (i + 1) * XH + j;
    float a[5], b[6], c[5];                        // rows i-1 (j..j+4), i (j-1..j+4), i+1 (j-1..j+3)
#pragma unroll
    for (int k = 0; k < 5; ++k) { a[k] = r0[k]; c[k] = r2[k - 1]; }
#pragma unroll
    for (int k = 0; k < 6; ++k) b[k] = r1[k - 1];
    float dy[5], dx[5], s[5];                      // psi at (i, j-1+k): D and 1/sqrt(|D|^2 + eps^2)
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        dy[k] = c[k] - b[k];
        dx[k] = b[k + 1] - b[k];
        s[k] = rsqrtf(dy[k] * dy[k] + dx[k] * dx[k] + e2);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float xc = b[q + 1];
        const float dyu = xc - a[q], dxu = a[q + 1] - a[q];      // psi at (i-1, j+q)
        const float su = rsqrtf(dyu * dyu + dxu * dxu + e2);
        // psi_y(p-1) - psi_y(p) + psi_x(q-1) - psi_x(q)
        td[q] = dyu * su - dy[q + 1] * s[q + 1] + dx[q] * s[q] - dx[q + 1] * s[q + 1];
        phi[q] = 0.f;
        if (want_phi) {
            const float t2c = dy[q + 1] * dy[q + 1] + dx[q + 1] * dx[q + 1];
            phi[q] = t2c / (sqrtf(t2c + e2) + sc.eps);
        }
    }
}

// stage the (TYh+2) x (TXh+2) circular halo of x[par] for a tile at (y0, x0)
__device__ __forceinline__ void stage_halo(const FacetDev &F, float *xh, int XH, int YH, int y0, int x0, int par) {
    const float *__restrict__ x = F.x[par];
    for (int idx = threadIdx.x; idx < YH * XH; idx += blockDim.x) {
        const int i = idx / XH, j = idx - i * XH;
        int fy = y0 - 1 + i, fx = x0 - 1 + j;
        fy = ((fy % F.ny) + F.ny) % F.ny;
        fx = ((fx % F.nx) + F.nx) % F.nx;
        xh[idx] = x[(int64_t)fy * F.ep + fx];
    }
}


}  // namespace deblur
