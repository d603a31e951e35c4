// vmlmb.hpp -- VMLM-B Local-Solver vector kernels (internal; see k_vmlmb.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace deblur {

constexpr int VM_MAXF = 64;     // local facets per rank in VMLM-B mode (kernel-argument arrays)

// Kernel arguments: per-local-facet vector pointers in roles A/A2 (written), B/C
// (read), M (free mask read) / Mo (written), per-facet coefficients c0/c1, and
// the per-tile fp64 partials [nsum][ntiles].
struct VmArgs {
    const FacetDev *facets;
    const TileDesc *tiles;       // the H^T tile grid (32 x 128)
    int ntiles;
    int par;                     // x = F.x[par]; trial point F.x[par ^ 1]
    int nsum;                    // partial sums written per tile (k_dot: 1..3)
    double *partials;
    float *A[VM_MAXF];
    float *A2[VM_MAXF];
    const float *B[VM_MAXF];
    const float *C[VM_MAXF];
    const uint8_t *M[VM_MAXF];
    uint8_t *Mo[VM_MAXF];
    double c0[VM_MAXF], c1[VM_MAXF];
};

cudaError_t vm_mask_q(const VmArgs &a, cudaStream_t s);          // Mo = free set; A = Mo ? B : 0
cudaError_t vm_dot(const VmArgs &a, cudaStream_t s);             // partials <B,C> (, <B,B>, <C,C>)
cudaError_t vm_axpy_dot(const VmArgs &a, cudaStream_t s);        // A = c1 A + c0 M.B; partial <C, A>
cudaError_t vm_direction(const VmArgs &a, cudaStream_t s);       // A = -M.B or -c0 M.C; partial <C, A>
cudaError_t vm_trial(const VmArgs &a, cudaStream_t s);           // x[par^1] = max(0, x + c0 B); partial <C, dx>
cudaError_t vm_pair(const VmArgs &a, cudaStream_t s);            // A = dx, A2 = C - B; partials sy, ss, yy
cudaError_t vm_grad(const VmArgs &a, const SolverConst &sc, cudaStream_t s);   // A = full gradient; reg, prox
cudaError_t vm_finalize(const VmArgs &a, float rho, cudaStream_t s);           // u (single owner) / v (band)

}  // namespace deblur
