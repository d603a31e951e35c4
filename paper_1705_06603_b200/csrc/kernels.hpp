// kernels.hpp -- launch wrappers of libdeblur's CUDA kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"

namespace deblur {

// Direct-path tile shapes (see k_direct.cu): BX=16 threads x 2 groups x 4 cols.
constexpr int DIRECT_TX = 128;
int direct_ty_H(int P);    // output rows per H tile
int direct_ty_HT(int P);   // output rows per H^T tile
size_t direct_smem_H(int P);
size_t direct_smem_HT(int P);
bool direct_supported(int P);

struct ConvArgs {
    const FacetDev *facets;   // device array of local facets
    const TileDesc *tiles;    // device tile list
    int ntiles;
    const float *psfs;        // [K][P][P]
    const float *wy, *wx;     // [Gy][Ny], [Gx][Nx]
    int P, Gx;
    int Ny, Nx;
    double *partials;         // [ntiles] fp64 partial sums (or NULL)
};

enum HMode { H_RESIDUAL = 0, H_PLAIN = 1, H_OBJECTIVE = 2 };
enum HTMode { HT_UPDATE = 0, HT_PLAIN = 1 };

cudaError_t launch_H_direct(const ConvArgs &a, int mode, int par, cudaStream_t s);
cudaError_t launch_HT_direct(const ConvArgs &a, int mode, int par, int last_step, const SolverConst &sc,
                             cudaStream_t s);

// k_update.cu: elementwise / band kernels
cudaError_t launch_update_from_g(const FacetDev *facets, const TileDesc *tiles, int ntiles, int P, int par,
                                 int last_step, const SolverConst &sc, double *partials, cudaStream_t s);
cudaError_t launch_consensus(const FacetDev *facets, const BandRect *rects, const RectTile *tiles, int ntiles,
                             int par, float rho, cudaStream_t s);
cudaError_t launch_tv_value(const FacetDev *facets, const TileDesc *tiles, int ntiles, int P, int par,
                            const SolverConst &sc, double *partials, cudaStream_t s);
cudaError_t launch_maxdiff(const FacetDev *facets, const BandRect *rects, int nrect, int par, double *partials,
                           cudaStream_t s);

cudaError_t launch_x0_from_y(const FacetDev &F, const float *ydil, int64_t dpitch, int dy0, int dx0, int My, int Mx,
                             int c, cudaStream_t s);
cudaError_t launch_blend(const FacetDev &F, int par, float *img, float *wsum, int64_t Nx, cudaStream_t s);
cudaError_t launch_normalize(float *img, const float *wsum, int64_t n, cudaStream_t s);

}  // namespace deblur
