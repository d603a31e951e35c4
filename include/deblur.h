/*
 * deblur.h -- C ABI of libdeblur: one full distributed iteration of the
 * facet-consensus deblurring method of Mourya et al., "Distributed Deblurring
 * of Large Images of Wide Field-Of-View" (arXiv 1705.06603), on B200 GPUs.
 *
 * Citations "P:n" are lines of the paper text, "§8x"/"Ann" are
 * sections / readings of SURVEY.md and DESIGN.md.
 *
 * Problem (Eq. (3)/(4)):
 *   y = H x + noise, H = R sum_k Z_k H_k W_k C_k (PSF interpolation)
 *   minimise sum_f f_f(x_f) s.t. overlapping facets agree, with
 *   f_f(x) = 1/2 |y_f - H_f x|^2_{W_f} + lambda phi(D x) + iota_{x >= 0}
 * solved by Douglas-Rachford splitting with consensus (Algorithm 1, P:208-233,
 * Lemma 1).
 *
 * Conventions
 *   - Images are row-major fp32 ("lexicographically ordering"; A23).
 *   - Estimate/scene domain N_y x N_x; observed domain M = N - P + 1 per axis
 *     (valid region, P:61 footnote; A18).  Observed pixel (i, j) sees
 *     estimate pixels (i .. i+P-1, j .. j+P-1) (A17: true convolution,
 *     PSF centre at ((P-1)/2, (P-1)/2)).
 *   - PSF k = p*G_x + q is the PSF of grid point (p, q); its interpolation
 *     weight is omega_k(r, c) = interp_wy[p][r] * interp_wx[q][c] (A16:
 *     the weight multiplies x BEFORE blurring; H^T multiplies after).
 *
 * Ownership and threading
 *   - Every input pointer is a HOST pointer borrowed for the duration of the
 *     call and copied (except the *_device entry points, which take device
 *     pointers on the handle's device).  Outputs are caller-allocated.
 *   - The handle owns every device buffer, stream and NCCL communicator.  No
 *     global state: a process may hold several handles.  Calls on one handle
 *     are blocking (they return after the device work completes) and not
 *     thread-safe.
 *
 * Errors
 *   - Every call returns a deblur_status; no exception or abort crosses the
 *     ABI.  deblur_last_error(h) names the offending argument / facet / peer.
 *   - deblur_create never returns a half-built handle (*out = NULL on error).
 *   - After DEBLUR_ECUDA or DEBLUR_ENCCL the handle is poisoned: every call
 *     but deblur_destroy / deblur_last_error returns DEBLUR_ESTATE.
 *   - There is no CPU fallback: without a usable sm_100 device deblur_create
 *     returns DEBLUR_ECUDA.
 *
 * Multi-GPU (SPMD, one process per GPU, §8e)
 *   - Every rank passes identical global params (same host arrays); each rank
 *     uploads only the slices of its own facets.  Facets map to ranks as
 *     contiguous rectangles of a g_y x g_x GPU grid (g_y | F_y, g_x | F_x,
 *     minimum cut).  Results are bitwise independent of the GPU count.
 *   - Collective calls (marked) must be made by all ranks in the same order.
 *   - Full-image outputs (apply_H, apply_HT, get_image) are written on rank 0
 *     only; other ranks may pass NULL.
 */
#ifndef DEBLUR_H_
#define DEBLUR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DEBLUR_API __attribute__((visibility("default")))
#else
#define DEBLUR_API
#endif

#define DEBLUR_ABI_VERSION 3

typedef struct deblur_ctx *deblur_t;

typedef enum {
    DEBLUR_OK = 0,
    DEBLUR_EINVAL = -1,   /* invalid scalar argument (names it) */
    DEBLUR_ESHAPE = -2,   /* inconsistent sizes / geometry */
    DEBLUR_ENOMEM = -3,   /* device or host allocation failed */
    DEBLUR_ECUDA = -4,    /* CUDA error or no sm_100 device (poisons the handle) */
    DEBLUR_ENCCL = -5,    /* NCCL error (poisons the handle; names peer and phase) */
    DEBLUR_ENUMERIC = -6, /* non-finite objective partial (names facet) */
    DEBLUR_ESTATE = -7    /* handle poisoned, or call not valid in this state */
} deblur_status;

/* Facet-local operator model.
 *   DEBLUR_OP_INTERP: H_f = the global PSF-interpolation operator H
 *     restricted to the facet's observed rows O_f and estimate columns P_f (R1);
 *     consensus weights omega^F = the A13 ramps on the shared bands.
 *   DEBLUR_OP_PER_NODE: the paper's node model: facet
 *     (a, b) of an F_y x F_x grid with F = G owns PSF k = a*G_x + b and its local
 *     operator is the valid convolution with that single PSF, H_f = C_f calH_f (no
 *     interpolation weights inside H_f); alpha_f = gamma * omega_f with omega_f =
 *     interp_wy[a] (x) interp_wx[b] (the interpolation weights of its PSF), so the
 *     consensus z = sum_f omega_f v_f / sum_f omega_f and the prox term
 *     gamma omega_f (x - u) act with the interpolation weights; get_image returns
 *     sum_f omega_f x_f / sum_f omega_f.  Requires psf_gy == facet_gy,
 *     psf_gx == facet_gx and sum_{f containing l} omega_f(l) > 0 at every
 *     estimate pixel (else DEBLUR_EINVAL naming the axis and pixel). */
typedef enum {
    DEBLUR_OP_INTERP = 0,
    DEBLUR_OP_PER_NODE = 1
} deblur_operator_mode;

/* Blur-operator implementation for H / H^T (a1, a2 of §8a). */
typedef enum {
    DEBLUR_CONV_AUTO = 0,   /* library choice by the measured crossover in P */
    DEBLUR_CONV_DIRECT = 1, /* FP32-FMA direct stencil */
    DEBLUR_CONV_FFT = 2     /* hand-written FFT overlap-save path */
} deblur_conv_path;

typedef struct {
    int32_t abi_version;          /* must equal DEBLUR_ABI_VERSION */
    /* geometry of the scene / estimate (A19) */
    int64_t ny, nx;               /* N_y, N_x; observed is (ny-P+1) x (nx-P+1) */
    int32_t psf_gy, psf_gx;       /* PSF grid G_y x G_x */
    int32_t psf_size;             /* P, odd, 1 <= P <= min(ny, nx) */
    const float *psfs;            /* [G_y*G_x][P][P], used verbatim (no renormalisation) */
    const float *interp_wy;       /* [G_y][N_y] first-order interpolation weights */
    const float *interp_wx;       /* [G_x][N_x] */
    /* data (Eq. (3)) */
    const float *y;               /* [M_y][M_x] observed image */
    const float *noise_w;         /* [M_y][M_x] W = 1/sigma^2 (0 = unmeasured), or NULL */
    float noise_w_scalar;         /* used when noise_w == NULL; must be >= 0 */
    /* regulariser (A1, A2) */
    float lambda;                 /* >= 0 */
    float eps;                    /* > 0: smoothing eps (reg_kind 0) or Huber delta (reg_kind 1) */
    int32_t reg_kind;             /* 0: sqrt(|Dx|^2+eps^2)-eps (default)  1: Huber (paper) */
    int32_t tv_boundary;          /* 0: circular per facet (paper)  1: Neumann */
    /* Douglas-Rachford (A3, A4, A10, A11) */
    float gamma;                  /* >= 0: alpha_f = gamma * omega^F_f */
    float rho;                    /* relaxation, 0 < rho < 2 */
    double tau;                   /* Local-Solver step; <= 0 -> library default (A4') */
    int32_t inner_steps;          /* K_in >= 1 projected-gradient steps per outer iteration (R2) */
    /* facets (A12, A13) */
    int32_t facet_gy, facet_gx;   /* F_y x F_x */
    int32_t overlap;              /* O >= 0, even: overlap between OBSERVED blocks */
    const float *x0;              /* [N_y][N_x] initial estimate, or NULL -> A6 default; u0 = x0 */
    /* execution */
    int32_t conv_path;            /* deblur_conv_path */
    int32_t rank, world, device;  /* SPMD rank / world size; CUDA device ordinal */
    const void *nccl_id;          /* 128-byte ncclUniqueId identical on all ranks; NULL if world == 1 */
    int32_t operator_mode;        /* deblur_operator_mode (default DEBLUR_OP_INTERP) */
    int32_t independent;          /* 1: the paper's "independent" baseline (NEXT-3): every
                                     facet solves its own problem, no consensus, no halo exchange,
                                     alpha = 0 (gamma is ignored, also in the default tau);
                                     get_image blends with omega^F.  0: Algorithm 1 (default) */
    int32_t local_solver;         /* 0: inner_steps projected-gradient steps (R2, default);
                                     1: VMLM-B (reading V1-V6): projected L-BFGS, m = 5, Armijo
                                     backtracking, warm start at x_f, budget inner_steps +
                                     k * inner_increment inner iterations at outer iteration k (P:290:
                                     10 + 10k); eager launches (host-side line-search decisions); at most
                                     64 facets per rank */
    int32_t inner_increment;      /* >= 0, VMLM-B budget increment per outer iteration */
    int32_t loopback_world;       /* world == 1 only; 0 or 1: off.  V > 1: the facets are assigned to V
                                     VIRTUAL ranks by the same GPU-grid planner as a world-V run, and
                                     every band shared by facets of different virtual ranks takes the
                                     multi-rank path of a5/a6 (Fig. 2): packed
                                     into per-message send buffers, moved into the matching receive
                                     buffers (a device copy stands in for ncclSend/ncclRecv) and read
                                     by the consensus kernel from there.  Results are bitwise equal
                                     to V = 1 (ascending facet id, A9).  V must factor
                                     into a GPU grid dividing the facet grid (else DEBLUR_ESHAPE). */
} deblur_params;

/* 128-byte NCCL unique id for a world > 1 run: call on rank 0, broadcast
 * (e.g. through a torch.distributed process group), pass as params.nccl_id. */
DEBLUR_API deblur_status deblur_nccl_id(void *out128);

/* Validate params (§8b), plan facets/bands/GPU grid, allocate device state,
 * upload this rank's slices, compute tau if tau <= 0.  COLLECTIVE. */
DEBLUR_API deblur_status deblur_create(const deblur_params *p, deblur_t *out);
DEBLUR_API deblur_status deblur_destroy(deblur_t h);

/* hx = H x on the whole image.  x: host [N_y][N_x]; hx: host
 * [M_y][M_x], written on rank 0.  Facet-wise, owner computes (§8b).  In the
 * per-node operator mode each observed pixel takes the local operator H_f of the
 * facet owning it (the piecewise shift-invariant model of P:109).  COLLECTIVE. */
DEBLUR_API deblur_status deblur_apply_H(deblur_t h, const float *x, float *hx);
/* g = H^T r (adjoint).  r: host [M_y][M_x]; g: host [N_y][N_x] on rank 0.
 * Requires overlap >= P-1 when there is more than one facet (else EINVAL).  COLLECTIVE. */
DEBLUR_API deblur_status deblur_apply_HT(deblur_t h, const float *r, float *g);
/* Same on device pointers of the handle's device (world == 1 only). */
DEBLUR_API deblur_status deblur_apply_H_device(deblur_t h, const float *d_x, float *d_hx);
DEBLUR_API deblur_status deblur_apply_HT_device(deblur_t h, const float *d_r, float *d_g);

/* n full distributed iterations (Algorithm 1): per facet K_in projected
 * gradient steps on f_f + 1/2|. - u_f|^2_alpha (a1-a4), halo exchange of
 * v = 2x - u (a5), consensus and dual update (a6).  COLLECTIVE. */
DEBLUR_API deblur_status deblur_iterate(deblur_t h, int32_t n);

/* n iterations with the objective traced: trace[4k .. 4k+3] = deblur_objective at
 * the state x^(k) before iteration k+1 (k = 0 .. n-1), i.e. the convergence
 * history of Eq. (4) and of the consensus residual.  trace is a
 * caller-allocated host array of 4n doubles.  Each entry costs one extra H
 * evaluation (the objective's data term) and eager (non-graph) launches.
 * COLLECTIVE; identical values on every rank. */
DEBLUR_API deblur_status deblur_iterate_traced(deblur_t h, int32_t n, double *trace);

/* out = {total, data, reg, consensus_maxdiff} at the current state (A22):
 * sum_f [1/2 sum_{O_f} w (H_f x_f - y)^2 + lambda sum_{P_f} phi(D x_f)] and
 * max |x_f(l) - x_g(l)| over shared pixels.  Identical on all ranks.  COLLECTIVE. */
DEBLUR_API deblur_status deblur_objective(deblur_t h, double out[4]);

/* x_hat = sum_f omega^F_f x_f (A7); host [N_y][N_x] on rank 0.  COLLECTIVE. */
DEBLUR_API deblur_status deblur_get_image(deblur_t h, float *x);

/* Per-facet state (x_f, u_f) of ALL facets concatenated in facet-id order
 * (row-major within each facet), host.  get: written on rank 0.  set: every
 * rank passes the full arrays and uploads its own facets.  COLLECTIVE. */
DEBLUR_API deblur_status deblur_state_size(deblur_t h, int64_t *n_floats);
DEBLUR_API deblur_status deblur_get_state(deblur_t h, float *x_facets, float *u_facets);
DEBLUR_API deblur_status deblur_set_state(deblur_t h, const float *x_facets, const float *u_facets);
/* Outer-iteration counter k of the run (Algorithm 1's loop index), which sets the
 * VMLM-B inner budget inner_steps + k * inner_increment.  A checkpoint stores it
 * next to (x_f, u_f); set restores it (k >= 0, else DEBLUR_EINVAL).  deblur_reset sets 0. */
DEBLUR_API deblur_status deblur_get_outer_iteration(deblur_t h, int32_t *k);
DEBLUR_API deblur_status deblur_set_outer_iteration(deblur_t h, int32_t k);

/* New observation with the same geometry and PSFs (e.g. the next exposure):
 * upload y (host [M_y][M_x]) and restart from x0 (host [N_y][N_x] or NULL ->
 * A6 default).  noise weights are kept.  COLLECTIVE. */
DEBLUR_API deblur_status deblur_reset(deblur_t h, const float *y, const float *x0);

/* Pipelined jobs (a stream of observations of the same geometry, e.g. successive exposures):
 * the next observation's upload and the previous image's download overlap the current
 * job's iterations.
 *   deblur_stage_y(h, y): start copying y (host [M_y][M_x]; page-locked for the copy to be
 *     asynchronous) into the handle's second staging buffer on an upload stream; y must stay
 *     valid until the next deblur_reset_staged / deblur_sync returns.
 *   deblur_reset_staged(h, x0): restart from the staged observation (x0 host or NULL -> the
 *     A6 default) -- the same state as deblur_reset(h, y, x0); returns without waiting for
 *     the device (the next call on the handle is ordered after it).  DEBLUR_ESTATE if nothing
 *     was staged.
 *   deblur_get_image_async(h, x): the blended image (as deblur_get_image) into host x
 *     (page-locked, [N_y][N_x]) on a download stream; x is complete when deblur_sync returns.
 *     world == 1 only (else DEBLUR_ESTATE).
 *   deblur_sync(h): wait for every outstanding upload, download and kernel of the handle. */
DEBLUR_API deblur_status deblur_stage_y(deblur_t h, const float *y);
DEBLUR_API deblur_status deblur_reset_staged(deblur_t h, const float *x0);
DEBLUR_API deblur_status deblur_get_image_async(deblur_t h, float *x);
DEBLUR_API deblur_status deblur_sync(deblur_t h);

/* The Local-Solver step actually used (fp64 value from which the fp32 device
 * copy was rounded). */
DEBLUR_API deblur_status deblur_get_step(deblur_t h, double *tau_used);

/* Instrumentation (bench.py): when enabled, every kernel launch is bracketed
 * by CUDA events on the launching stream.  deblur_kernel_stats returns, per
 * kernel class (names via deblur_kernel_name), the number of launches and the
 * summed event time in ms since the last reset; n_classes in/out. */
DEBLUR_API deblur_status deblur_set_profiling(deblur_t h, int32_t enable);
DEBLUR_API deblur_status deblur_kernel_stats(deblur_t h, int32_t *n_classes, int64_t *launches, double *ms);
DEBLUR_API const char *deblur_kernel_name(int32_t cls);
DEBLUR_API deblur_status deblur_reset_stats(deblur_t h);
/* Algorithmic work of ONE launch of kernel class `cls` on this rank (DESIGN.md
 * §5-6): flops = 2 a P^2 per output pixel for the direct stencils (a = number of
 * PSFs with nonzero weight at the pixel) and the FFT-convention count of the FFT
 * passes (5 L log2 L per complex length-L DFT, half that per real one, plus the
 * spectral products and weights); bytes = the compulsory HBM traffic of the pass
 * (FFT passes, elementwise kernels).  0 where not applicable. */
DEBLUR_API deblur_status deblur_kernel_work(deblur_t h, int32_t cls, double *flops, double *bytes);

/* The cudaStream_t (as void*) every kernel of this handle is launched on, so a
 * caller can bracket calls with CUDA events on the launching stream. */
DEBLUR_API deblur_status deblur_get_stream(deblur_t h, void **stream);

/* Conv path actually used (deblur_conv_path, never AUTO). */
DEBLUR_API deblur_status deblur_get_conv_path(deblur_t h, int32_t *path);

/* Host-only planning queries (no GPU needed; used by the multi-rank tests).
 * deblur_plan_facets: F = F_y*F_x; boxes[F][8] = {oy0, oy1, ox0, ox1, ey0, ey1,
 * ex0, ex1} (observed / estimate blocks, A12), owner[F] = rank.
 * deblur_plan_messages: for `rank`, the halo messages it SENDS per iteration:
 * msgs[n][8] = {peer_rank, src_facet, dst_facet, y0, y1, x0, x1, bytes}
 * (rectangle in global estimate coordinates); pass msgs = NULL to get n. */
DEBLUR_API deblur_status deblur_plan_facets(const deblur_params *p, int32_t *n_facets, int64_t *boxes, int32_t *owner);
DEBLUR_API deblur_status deblur_plan_messages(const deblur_params *p, int32_t rank, int32_t *n, int64_t *msgs);

/* NULL-safe; per handle; valid until the next call on the handle.
 * deblur_last_error(NULL) returns the error of the last failed create/plan in this thread. */
DEBLUR_API const char *deblur_last_error(deblur_t h);

#ifdef __cplusplus
}
#endif
#endif /* DEBLUR_H_ */
