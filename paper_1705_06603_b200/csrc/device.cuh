// device.cuh -- device-side descriptors shared by libdeblur's kernels and host code.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace deblur {

// Consensus weight omega^F along one axis (A13, Fig. 1 ramp PAPER.md:239).
// Local index t of a facet whose estimate block starts at global e0:
//   t < b_prev : omega = (e0 + t - s_prev + 0.5) / (e_prev - s_prev)   (ramp up)
//   t >= b_next: omega = 1 - (e0 + t - s_next + 0.5) / (e_next - s_next)  (ramp down)
//   else       : 1 (single owner along this axis)
struct AxisW {
    int e0;              // global origin of the facet along this axis
    int n;               // facet extent along this axis
    int b_prev;          // local rows [0, b_prev) are shared with the previous facet (0 = none)
    int b_next;          // local rows [b_next, n) are shared with the next facet (n = none)
    int s_prev, e_prev;  // global band with previous facet [s_prev, e_prev)
    int s_next, e_next;  // global band with next facet [s_next, e_next)
    // per-node operator mode (alpha_i = gamma omega_i): omega along this
    // axis is the facet's own interpolation weight row, indexed by the global
    // coordinate (device pointer); NULL -> the A13 ramps above
    const float *w;
};

__host__ __device__ inline float omega_axis(const AxisW &a, int t) {
    if (a.w) return a.w[a.e0 + t];
    if (t < a.b_prev) return ((float)(a.e0 + t - a.s_prev) + 0.5f) / (float)(a.e_prev - a.s_prev);
    if (t >= a.b_next) return 1.0f - ((float)(a.e0 + t - a.s_next) + 0.5f) / (float)(a.e_next - a.s_next);
    return 1.0f;
}

// A view mapping global estimate coordinates to an address: base[par] +
// (gy - y0) * pitch + (gx - x0).  par selects the x ping/pong buffer for
// facet-local views; remote (received) bands set base[0] == base[1].
struct View {
    const float *base[2];
    int64_t pitch;
    int y0, x0;
    int valid;
};

struct Neighbour {        // facet at grid offset (dy, dx) in {-1,0,1}^2
    int id;               // global facet id (-1 if none)
    AxisW ay, ax;         // its consensus-weight axes
    View v;               // its v = 2x - u values (band region)
    View x;               // its x values (for the objective's consensus residual)
};

struct FacetDev {
    int id;
    int ny, nx;           // estimate block extent
    int my, mx;           // observed block extent
    int ey0, ex0;         // global estimate (= observed) origin
    int64_t ep;           // pitch (floats) of estimate arrays (multiple of 32)
    int64_t op;           // pitch of observed arrays
    float *x[2];          // estimate ping / pong
    float *u;             // dual variable u_f
    float *v;             // 2 x+ - u on band pixels
    float *g;             // scratch estimate array (H^T r for apply_HT / FFT path)
    const float *y;       // observed slice
    const float *w;       // observed weights slice (NULL -> w_scalar)
    float w_scalar;
    float *r;             // observed scratch: residual w (H x - y) or H x
    AxisW ay, ax;         // own consensus-weight axes
    Neighbour nb[3][3];   // [dy+1][dx+1]
};

struct TileDesc {         // one CTA's tile
    int f;                // local facet index
    int y0, x0;           // tile origin (facet-local; observed coords for H, estimate coords for H^T)
    int p0, p1, q0, q1;   // active PSF grid rows/cols (inclusive); p1 < p0 -> none
    int ylim = 1 << 30;   // FFT tiles: outputs only in rows < ylim, cols < xlim (the tile's region)
    int xlim = 1 << 30;
};

struct BandRect {         // consensus work item: facet-local rectangle of band pixels
    int f;
    int y0, y1, x0, x1;
    int dy0, dy1, dx0, dx1;   // the neighbour offsets contributing on the whole rectangle
};

constexpr int CT_ROWS = 32;   // rows of a consensus launch unit
struct RectTile {         // consensus launch unit: CT_ROWS rows x 256 columns of one BandRect
    int rect, y0, x0;
};

struct SolverConst {
    float lambda, eps, gamma, rho, tau;
    int reg_kind, tv_boundary;
};

}  // namespace deblur
