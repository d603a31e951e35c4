// deblur.cu -- libdeblur: C ABI (include/deblur.h), device state, orchestration.
//
// One handle = one rank = one GPU.  It owns the device copies of this rank's
// facets (x ping/pong, u, v, y, w, r, g), the PSF taps and interpolation
// weights, the tile / band work lists, the stream and (world > 1) the NCCL
// communicator.  deblur_iterate runs Algorithm 1:
//   per inner step: K1 (H + residual) -> K2 (H^T + TV + prox + projection)
//   then: halo exchange of v = 2x+ - u over NCCL (world > 1)  -> K5 consensus.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/deblur.h"
#include "fft.hpp"
#include "kernels.hpp"
#include "plan.hpp"
#include "vmlmb.hpp"

using namespace deblur;

namespace {

thread_local std::string g_last_error;

enum KClass {
    KC_H = 0, KC_HT_UPDATE, KC_CONSENSUS, KC_H_OBJ, KC_TV, KC_MAXDIFF, KC_XCHG, KC_HT_PLAIN, KC_H_PLAIN,
    KC_FFT_H0, KC_FFT_H1, KC_FFT_H2, KC_FFT_HT0, KC_FFT_HT1, KC_FFT_HT2, KC_UPDATE_G, KC_VM_VEC, KC_VM_GRAD,
    KC_FFT2_H0, KC_FFT2_H1, KC_FFT2_H2, KC_FFT2_HT0, KC_FFT2_HT1, KC_FFT2_HT2, KC_COUNT
};
const char *k_names[KC_COUNT] = {"H_direct_residual", "HT_direct_update", "consensus", "H_direct_objective",
                                 "tv_value", "maxdiff", "halo_exchange", "HT_direct_plain", "H_direct_plain",
                                 "H_fft_rows", "H_fft_cols", "H_fft_rows_inv", "HT_fft_rows", "HT_fft_cols",
                                 "HT_fft_rows_inv", "update_from_g", "vmlmb_vector", "vmlmb_grad",
                                 "H_fft2_rows", "H_fft2_cols", "H_fft2_rows_inv", "HT_fft2_rows", "HT_fft2_cols",
                                 "HT_fft2_rows_inv"};

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

struct SendRecv {
    Message m;
    float *vbuf = nullptr;   // device buffer for v band
    float *xbuf = nullptr;   // device buffer for x band (objective)
    int peer_index = -1;     // loopback transport: index of the matching receive (sends only)
};

}  // namespace

struct deblur_ctx {
    deblur_params prm{};
    Plan plan;
    int rank = 0, world = 1, device = 0;
    cudaStream_t stream = nullptr;
    // consensus stream (§8e): the halo exchange and K5 of iteration k run here, under
    // the H / H^T passes of iteration k+1 (which read only x); the first kernel of
    // iteration k+1 that reads u waits for ev_cons
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_upd = nullptr, ev_cons = nullptr;
    bool cons_pending = false;
    // loopback transport (params.loopback_world = V > 1, world == 1): virtual owner of
    // every facet under a world-V plan; bands between virtual ranks use send / recv buffers
    int vworld = 1;
    std::vector<int> vowner;
    std::vector<int> local;               // facet ids owned by this rank (ascending)
    std::vector<int> local_index;         // facet id -> local index or -1
    std::vector<FacetDev> fh;             // host copies of the descriptors
    FacetDev *d_facets = nullptr;
    FacetDev *d_facets_alt = nullptr;     // x[] -> g (apply_H input)
    std::vector<void *> allocs;
    float *d_psfs = nullptr, *d_wy = nullptr, *d_wx = nullptr;
    // weights the operator kernels apply inside H_f: the interpolation weights (mode
    // INTERP) or all-ones rows with one PSF per facet (mode PER_NODE)
    float *d_owy = nullptr, *d_owx = nullptr;
    bool per_node = false;
    float *d_wsum = nullptr;          // per-node get_image normalisation
    std::vector<TileDesc> tilesH, tilesHT;
    TileDesc *d_tilesH = nullptr, *d_tilesHT = nullptr;
    std::vector<BandRect> rects;
    BandRect *d_rects = nullptr;
    std::vector<RectTile> rect_tiles;
    RectTile *d_rect_tiles = nullptr;
    double *d_partials = nullptr;
    std::vector<double> h_partials;
    SolverConst sc{};
    double tau = 0.0;
    int par = 0;
    int conv_path = DEBLUR_CONV_DIRECT;
    FftPlan *fft = nullptr;
    FftPlan *fft2 = nullptr;              // S/2 plan for the ragged bottom / right strips of each facet
    // host copies needed after create
    std::vector<float> h_wy, h_wx;
    // communication
    ncclComm_t comm = nullptr;
    std::vector<SendRecv> sends, recvs;
    // instrumentation
    bool prof = false;
    struct Pending { int cls; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> ev_pool;
    int64_t stat_n[KC_COUNT] = {0};
    double stat_ms[KC_COUNT] = {0};
    // persistent staging buffers for reset / get_image (allocated on first use)
    float *d_ystage = nullptr;            // staged observed image (bounding box of this rank's needs)
    int64_t ys_y0 = 0, ys_x0 = 0, ys_pitch = 1;
    // pipelined jobs (deblur_stage_y / deblur_reset_staged / deblur_get_image_async): a second
    // staging buffer filled on the upload stream while the current job iterates, and two image
    // buffers downloaded on the download stream while the next job runs
    float *d_ystage2 = nullptr;
    cudaStream_t up_stream = nullptr, down_stream = nullptr;
    cudaEvent_t ev_staged = nullptr, ev_yfree = nullptr, ev_blend = nullptr, ev_down[2] = {nullptr, nullptr};
    bool staged = false;
    float *d_image2[2] = {nullptr, nullptr};
    int img_slot = 0;
    float *d_image = nullptr;
    // CUDA graphs of two full iterations (parity returns to its start), one per start parity
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int64_t graph_counts[2][KC_COUNT] = {{0}};
    bool use_graphs = true;
    // VMLM-B Local-Solver state (local_solver == 1): per local facet gradient pair,
    // direction, two-loop work vector, free mask and m = 5 memory pairs
    struct Vm {
        bool on = false;
        static constexpr int m = 5;
        std::vector<float *> G, Gn, D, Q;
        std::vector<uint8_t *> M;
        std::vector<std::array<float *, 5>> S, Y;
        std::vector<std::array<double, 5>> sy, yy;   // <s,y>, <y,y> of each memory slot
        double *d_part = nullptr;            // [3][ntilesHT]
        std::vector<double> h_part;
        int k_outer = 0;                     // outer iteration counter (budget schedule)
        int64_t evaluations = 0, iterations = 0;
    } vm;
    // errors
    std::string err;
    bool poisoned = false;

    deblur_status fail(deblur_status s, const std::string &m) {
        err = m;
        if (s == DEBLUR_ECUDA || s == DEBLUR_ENCCL) poisoned = true;
        return s;
    }
    deblur_status cuda_fail(cudaError_t e, const char *what) {
        std::ostringstream o;
        o << "CUDA error " << cudaGetErrorName(e) << " (" << cudaGetErrorString(e) << ") in " << what;
        return fail(DEBLUR_ECUDA, o.str());
    }
    deblur_status nccl_fail(ncclResult_t r, const char *phase, int peer) {
        std::ostringstream o;
        o << "NCCL error " << ncclGetErrorString(r) << " in " << phase;
        if (peer >= 0) o << " (peer rank " << peer << ")";
        return fail(DEBLUR_ENCCL, o.str());
    }
    template <typename T>
    cudaError_t dalloc(T **p, size_t n) {
        void *q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
        if (e == cudaSuccess) { allocs.push_back(q); *p = (T *)q; }
        return e;
    }
    cudaEvent_t get_event() {
        if (!ev_pool.empty()) { cudaEvent_t e = ev_pool.back(); ev_pool.pop_back(); return e; }
        cudaEvent_t e; cudaEventCreate(&e); return e;
    }
    void prof_begin(int cls, cudaEvent_t *a, cudaStream_t st = nullptr) {
        if (!prof) return;
        *a = get_event();
        cudaEventRecord(*a, st ? st : stream);
        (void)cls;
    }
    void prof_end(int cls, cudaEvent_t a, cudaStream_t st = nullptr) {
        stat_n[cls] += 1;
        if (!prof) return;
        cudaEvent_t b = get_event();
        cudaEventRecord(b, st ? st : stream);
        pending.push_back({cls, a, b});
    }
    double *d_objbuf = nullptr;           // world > 1: objective all-reduce buffer (2F + 1 doubles)
    void prof_collect() {
        for (auto &p : pending) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) stat_ms[p.cls] += ms;
            ev_pool.push_back(p.a);
            ev_pool.push_back(p.b);
        }
        pending.clear();
    }
    ConvArgs conv_args(const FacetDev *facets, bool ht) const {
        ConvArgs a;
        a.facets = facets;
        a.tiles = ht ? d_tilesHT : d_tilesH;
        a.ntiles = (int)(ht ? tilesHT.size() : tilesH.size());
        a.psfs = d_psfs; a.wy = d_owy; a.wx = d_owx;
        a.P = plan.P; a.Gx = prm.psf_gx; a.Ny = (int)plan.ny; a.Nx = (int)plan.nx;
        a.partials = d_partials;
        return a;
    }
};

#define CU(call)                                                      \
    do {                                                              \
        cudaError_t e_ = (call);                                      \
        if (e_ != cudaSuccess) return h->cuda_fail(e_, #call);        \
    } while (0)
#define NC(call, phase, peer)                                         \
    do {                                                              \
        ncclResult_t r_ = (call);                                     \
        if (r_ != ncclSuccess) return h->nccl_fail(r_, phase, peer);  \
    } while (0)

namespace {

deblur_status validate(const deblur_params *p, std::string &err) {
    std::ostringstream o;
    if (!p) { err = "params is NULL"; return DEBLUR_EINVAL; }
    if (p->abi_version != DEBLUR_ABI_VERSION) { o << "abi_version " << p->abi_version << " != " << DEBLUR_ABI_VERSION; err = o.str(); return DEBLUR_EINVAL; }
    if (p->ny < 1 || p->nx < 1 || p->ny > (1 << 30) || p->nx > (1 << 30)) { err = "ny/nx out of range"; return DEBLUR_ESHAPE; }
    if (p->psf_size < 1 || p->psf_size % 2 == 0) { err = "psf_size must be odd and >= 1"; return DEBLUR_EINVAL; }
    if (p->psf_size > p->ny || p->psf_size > p->nx) { err = "psf_size larger than the image"; return DEBLUR_ESHAPE; }
    if (p->psf_gy < 1 || p->psf_gx < 1) { err = "psf_gy/psf_gx must be >= 1"; return DEBLUR_EINVAL; }
    if (!p->psfs) { err = "psfs is NULL"; return DEBLUR_EINVAL; }
    if (!p->interp_wy || !p->interp_wx) { err = "interp_wy/interp_wx is NULL"; return DEBLUR_EINVAL; }
    if (!p->y) { err = "y is NULL"; return DEBLUR_EINVAL; }
    if (!p->noise_w && !(p->noise_w_scalar >= 0.f)) { err = "noise_w_scalar must be >= 0"; return DEBLUR_EINVAL; }
    if (!(p->lambda >= 0.f)) { err = "lambda must be >= 0"; return DEBLUR_EINVAL; }
    if (!(p->eps > 0.f)) { err = "eps must be > 0"; return DEBLUR_EINVAL; }
    if (p->reg_kind != 0 && p->reg_kind != 1) { err = "reg_kind must be 0 or 1"; return DEBLUR_EINVAL; }
    if (p->tv_boundary != 0 && p->tv_boundary != 1) { err = "tv_boundary must be 0 or 1"; return DEBLUR_EINVAL; }
    if (!(p->gamma >= 0.f)) { err = "gamma must be >= 0"; return DEBLUR_EINVAL; }
    if (!(p->rho > 0.f && p->rho < 2.f)) { err = "rho must be in (0, 2) (PAPER.md:147)"; return DEBLUR_EINVAL; }
    if (p->inner_steps < 1) { err = "inner_steps must be >= 1"; return DEBLUR_EINVAL; }
    if (p->facet_gy < 1 || p->facet_gx < 1) { err = "facet_gy/facet_gx must be >= 1"; return DEBLUR_EINVAL; }
    if (p->overlap < 0 || p->overlap % 2) { err = "overlap must be even and >= 0"; return DEBLUR_EINVAL; }
    if (p->conv_path < 0 || p->conv_path > 2) { err = "conv_path must be 0, 1 or 2"; return DEBLUR_EINVAL; }
    if (p->world < 1 || p->rank < 0 || p->rank >= p->world) { err = "rank/world out of range"; return DEBLUR_EINVAL; }
    if (p->world > 1 && !p->nccl_id) { err = "nccl_id is NULL with world > 1"; return DEBLUR_EINVAL; }
    if (!(std::isfinite(p->tau))) { err = "tau must be finite"; return DEBLUR_EINVAL; }
    if (p->independent != 0 && p->independent != 1) { err = "independent must be 0 or 1"; return DEBLUR_EINVAL; }
    if (p->local_solver != 0 && p->local_solver != 1) { err = "local_solver must be 0 (projected gradient) or 1 (VMLM-B)"; return DEBLUR_EINVAL; }
    if (p->inner_increment < 0) { err = "inner_increment must be >= 0"; return DEBLUR_EINVAL; }
    if (p->loopback_world < 0) { err = "loopback_world must be >= 0"; return DEBLUR_EINVAL; }
    if (p->loopback_world > 1 && p->world > 1) { err = "loopback_world needs world == 1"; return DEBLUR_EINVAL; }
    if (p->operator_mode != DEBLUR_OP_INTERP && p->operator_mode != DEBLUR_OP_PER_NODE) {
        err = "operator_mode must be 0 (interpolated H) or 1 (per-node PSFs)";
        return DEBLUR_EINVAL;
    }
    if (p->operator_mode == DEBLUR_OP_PER_NODE && (p->psf_gy != p->facet_gy || p->psf_gx != p->facet_gx)) {
        o << "per-node operator mode needs the facet grid to equal the PSF grid (facets " << p->facet_gy << "x"
          << p->facet_gx << ", PSFs " << p->psf_gy << "x" << p->psf_gx << ")";
        err = o.str();
        return DEBLUR_EINVAL;
    }
    return DEBLUR_OK;
}

// Per-node mode: every estimate pixel needs a positive consensus weight sum over the
// facets containing it (P:201 divides by it).  Separable: checked per axis.
static std::string check_node_weights(const Plan &pl, const float *wy, const float *wx) {
    for (int axis = 0; axis < 2; ++axis) {
        const int F = axis == 0 ? pl.Fy : pl.Fx;
        const int64_t n = axis == 0 ? pl.ny : pl.nx;
        const std::vector<AxisFacet> &af = axis == 0 ? pl.ay : pl.ax;
        const float *w = axis == 0 ? wy : wx;
        std::vector<double> sum(n, 0.0);
        for (int k = 0; k < F; ++k)
            for (int64_t i = af[k].e_lo; i < af[k].e_hi; ++i) {
                const double v = w[(int64_t)k * n + i];
                if (!(v >= 0.0)) {
                    std::ostringstream o;
                    o << (axis == 0 ? "interp_wy" : "interp_wx") << "[" << k << "][" << i << "] is negative or NaN";
                    return o.str();
                }
                sum[i] += v;
            }
        for (int64_t i = 0; i < n; ++i)
            if (!(sum[i] > 0.0)) {
                std::ostringstream o;
                o << "per-node mode: the consensus weights of the facets containing " << (axis == 0 ? "row " : "column ")
                  << i << " sum to 0";
                return o.str();
            }
    }
    return "";
}

// A4': tau = 1/L, L = max(w) S^2 a_row a_col + lambda * 8 * Lip(psi) + gamma
double default_tau(const deblur_params *p) {
    const int P = p->psf_size, K = p->psf_gy * p->psf_gx;
    const int64_t my = p->ny - P + 1, mx = p->nx - P + 1;
    double sy = 0, sx = 0;
    for (int64_t r = 0; r < p->ny; ++r) {
        double s = 0;
        for (int k = 0; k < p->psf_gy; ++k) s += std::fabs((double)p->interp_wy[(int64_t)k * p->ny + r]);
        sy = std::max(sy, s);
    }
    for (int64_t c = 0; c < p->nx; ++c) {
        double s = 0;
        for (int k = 0; k < p->psf_gx; ++k) s += std::fabs((double)p->interp_wx[(int64_t)k * p->nx + c]);
        sx = std::max(sx, s);
    }
    const double S = sy * sx;
    double a_row = 0, a_col = 0;
    for (int i = 0; i < P * P; ++i) {
        double m = 0;
        for (int k = 0; k < K; ++k) m = std::max(m, std::fabs((double)p->psfs[(int64_t)k * P * P + i]));
        a_row += m;
    }
    for (int k = 0; k < K; ++k) {
        double s = 0;
        for (int i = 0; i < P * P; ++i) s += std::fabs((double)p->psfs[(int64_t)k * P * P + i]);
        a_col = std::max(a_col, s);
    }
    double wmax = 0;
    if (p->noise_w) {
        for (int64_t i = 0; i < my * mx; ++i) wmax = std::max(wmax, (double)p->noise_w[i]);
    } else {
        wmax = (double)p->noise_w_scalar;
    }
    const double lip = (p->reg_kind == 0) ? 1.0 / (double)p->eps : 1.0;
    const double gamma = p->independent ? 0.0 : (double)p->gamma;     // independent: alpha = 0
    const double L = wmax * S * S * a_row * a_col + (double)p->lambda * 8.0 * lip + gamma;
    return L > 0 ? 1.0 / L : 1.0;
}

// Active PSF index range [lo, hi] whose weight row is nonzero somewhere on [a, b).
struct NzIndex {
    int G = 0; int64_t n = 0;
    std::vector<int64_t> pre;   // [G][n+1] prefix counts of nonzeros
    void build(const float *w, int G_, int64_t n_) {
        G = G_; n = n_;
        pre.assign((size_t)G * (n + 1), 0);
        for (int g = 0; g < G; ++g)
            for (int64_t i = 0; i < n; ++i)
                pre[(size_t)g * (n + 1) + i + 1] = pre[(size_t)g * (n + 1) + i] + (w[(size_t)g * n + i] != 0.f);
    }
    void range(int64_t a, int64_t b, int &lo, int &hi) const {
        a = std::max<int64_t>(0, a); b = std::min<int64_t>(n, b);
        lo = G; hi = -1;
        if (a >= b) return;
        for (int g = 0; g < G; ++g) {
            if (pre[(size_t)g * (n + 1) + b] - pre[(size_t)g * (n + 1) + a] > 0) { lo = std::min(lo, g); hi = std::max(hi, g); }
        }
    }
};

}  // namespace

// ----------------------------------------------------------------------------- helpers
static deblur_status upload_slice(deblur_t h, float *dst, int64_t dpitch, const float *src, int64_t spitch,
                                  int64_t y0, int64_t x0, int64_t rows, int64_t cols) {
    CU(cudaMemcpy2DAsync(dst, dpitch * 4, src + y0 * spitch + x0, spitch * 4, cols * 4, rows,
                         cudaMemcpyHostToDevice, h->stream));
    return DEBLUR_OK;
}

// The observed image crosses PCIe once: the bounding box of what this rank's facets need
// (their observed blocks O_f for y, and O_f dilated by c -- clipped -- for the A6 start)
// is uploaded into a staging buffer; F.y and the A6 start are formed from it on the device.
static void ystage_box(deblur_t h, int64_t &y0, int64_t &y1, int64_t &x0, int64_t &x1) {
    const Plan &pl = h->plan;
    const int c = (pl.P - 1) / 2;
    y0 = pl.my; y1 = 0; x0 = pl.mx; x1 = 0;
    for (int id : h->local) {
        const FacetPlan &fp = pl.facets[id];
        y0 = std::min(y0, std::max<int64_t>(0, fp.ey0 - c)); y1 = std::max(y1, std::min<int64_t>(pl.my, fp.ey1 - c));
        x0 = std::min(x0, std::max<int64_t>(0, fp.ex0 - c)); x1 = std::max(x1, std::min<int64_t>(pl.mx, fp.ex1 - c));
    }
}

static deblur_status stage_y(deblur_t h, const float *y) {
    const Plan &pl = h->plan;
    int64_t y0, y1, x0, x1;
    ystage_box(h, y0, y1, x0, x1);
    if (!h->d_ystage) CU(h->dalloc(&h->d_ystage, (size_t)pl.my * pl.mx));
    h->ys_y0 = y0; h->ys_x0 = x0; h->ys_pitch = std::max<int64_t>(1, x1 - x0);
    if (y1 > y0 && x1 > x0)
        CU(cudaMemcpy2DAsync(h->d_ystage, h->ys_pitch * 4, y + y0 * pl.mx + x0, pl.mx * 4, (x1 - x0) * 4, y1 - y0,
                             cudaMemcpyHostToDevice, h->stream));
    return DEBLUR_OK;
}

// F.y of every local facet from the staged y (device copies)
static deblur_status upload_y(deblur_t h) {
    for (size_t li = 0; li < h->local.size(); ++li) {
        const FacetPlan &fp = h->plan.facets[h->local[li]];
        FacetDev &F = h->fh[li];
        const float *src = h->d_ystage + (fp.oy0 - h->ys_y0) * h->ys_pitch + (fp.ox0 - h->ys_x0);
        CU(cudaMemcpy2DAsync((float *)F.y, F.op * 4, src, h->ys_pitch * 4, F.mx * 4, F.my, cudaMemcpyDeviceToDevice,
                             h->stream));
    }
    return DEBLUR_OK;
}

// x0 given: upload its facet slices to x[0] and copy to u.  x0 == NULL: the A6
// default computed on the device from the staged y.
static deblur_status upload_state_x0(deblur_t h, const float *x0, bool sync = true) {
    const Plan &pl = h->plan;
    const int c = (pl.P - 1) / 2;
    for (size_t li = 0; li < h->local.size(); ++li) {
        const FacetPlan &fp = pl.facets[h->local[li]];
        FacetDev &F = h->fh[li];
        if (x0) {
            deblur_status s = upload_slice(h, F.x[0], F.ep, x0, pl.nx, fp.ey0, fp.ex0, F.ny, F.nx);
            if (s != DEBLUR_OK) return s;
            CU(cudaMemcpy2DAsync(F.u, F.ep * 4, F.x[0], F.ep * 4, F.nx * 4, F.ny, cudaMemcpyDeviceToDevice, h->stream));
        } else {
            CU(launch_x0_from_y(F, h->d_ystage, h->ys_pitch, (int)h->ys_y0, (int)h->ys_x0, (int)pl.my, (int)pl.mx, c,
                                h->stream));
        }
    }
    h->par = 0;
    if (sync) CU(cudaStreamSynchronize(h->stream));
    return DEBLUR_OK;
}

static deblur_status check_state(deblur_t h) {
    if (!h) return DEBLUR_EINVAL;
    if (h->poisoned) { return DEBLUR_ESTATE; }
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return h->cuda_fail(e, "cudaSetDevice");
    return DEBLUR_OK;
}

// halo exchange (a5): v bands (which == 0) or x[par] bands (which == 1)
// of every band shared with a facet of another rank, on stream `st`: pack each
// message's rectangle into its contiguous send buffer, then one grouped NCCL
// send/recv round (world > 1) or, for the loopback transport (one process, virtual
// ranks), a device copy of each send buffer into the matching receive buffer.
static deblur_status exchange(deblur_t h, int which, cudaStream_t st) {
    if (h->sends.empty() && h->recvs.empty()) return DEBLUR_OK;
    cudaEvent_t ev = nullptr;
    h->prof_begin(KC_XCHG, &ev, st);
    for (auto &s : h->sends) {
        const FacetDev &F = h->fh[h->local_index[s.m.src_facet]];
        const float *src = which == 0 ? F.v : F.x[h->par];
        const int64_t w = s.m.rect.x1 - s.m.rect.x0, hh = s.m.rect.y1 - s.m.rect.y0;
        const float *p = src + (s.m.rect.y0 - F.ey0) * F.ep + (s.m.rect.x0 - F.ex0);
        CU(cudaMemcpy2DAsync(which == 0 ? s.vbuf : s.xbuf, w * 4, p, F.ep * 4, w * 4, hh, cudaMemcpyDeviceToDevice,
                             st));
    }
    if (h->world > 1) {
        NC(ncclGroupStart(), "halo group start", -1);
        for (auto &s : h->sends)
            NC(ncclSend(which == 0 ? s.vbuf : s.xbuf, (size_t)s.m.rect.area(), ncclFloat, s.m.peer, h->comm, st),
               "halo send", s.m.peer);
        for (auto &r : h->recvs)
            NC(ncclRecv(which == 0 ? r.vbuf : r.xbuf, (size_t)r.m.rect.area(), ncclFloat, r.m.peer, h->comm, st),
               "halo recv", r.m.peer);
        NC(ncclGroupEnd(), "halo group end", -1);
    } else {
        for (auto &s : h->sends) {
            const SendRecv &r = h->recvs[s.peer_index];
            CU(cudaMemcpyAsync(which == 0 ? r.vbuf : r.xbuf, which == 0 ? s.vbuf : s.xbuf,
                               (size_t)s.m.rect.area() * 4, cudaMemcpyDeviceToDevice, st));
        }
    }
    h->prof_end(KC_XCHG, ev, st);
    return DEBLUR_OK;
}

// the stream waits for the consensus (K5) of the previous iteration, if one is pending
static deblur_status join_consensus(deblur_t h) {
    if (!h->cons_pending) return DEBLUR_OK;
    CU(cudaStreamWaitEvent(h->stream, h->ev_cons, 0));
    h->cons_pending = false;
    return DEBLUR_OK;
}

static deblur_status finish(deblur_t h) {
    deblur_status js = join_consensus(h);
    if (js != DEBLUR_OK) return js;
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    if (h->comm) {
        ncclResult_t ar;
        if (ncclCommGetAsyncError(h->comm, &ar) == ncclSuccess && ar != ncclSuccess)
            return h->nccl_fail(ar, "async", -1);
    }
    h->prof_collect();
    return DEBLUR_OK;
}

static deblur_status run_fft_H(deblur_t h, const FacetDev *facets, int par, int mode) {
    for (FftPlan *fp : {h->fft, h->fft2}) {
        if (!fp || !fft_tiles(*fp, false)) continue;
        const int c0 = fp == h->fft ? KC_FFT_H0 : KC_FFT2_H0;
        for (int pass = 0; pass < 3; ++pass) {
            cudaEvent_t ev = nullptr;
            h->prof_begin(c0 + pass, &ev);
            CU(fft_H_pass(*fp, pass, facets, par, mode, h->stream));
            h->prof_end(c0 + pass, ev);
        }
    }
    return DEBLUR_OK;
}

// per-local-facet data partial sums of the last run_fft_H (both plans)
static cudaError_t fft_partials_all(deblur_t h, std::vector<double> &out) {
    cudaError_t e = fft_data_partials(*h->fft, out);
    if (e != cudaSuccess || !h->fft2) return e;
    std::vector<double> o2;
    if ((e = fft_data_partials(*h->fft2, o2)) != cudaSuccess) return e;
    for (size_t i = 0; i < out.size(); ++i) out[i] += o2[i];
    return cudaSuccess;
}

static deblur_status run_fft_HT(deblur_t h, const FacetDev *facets) {
    for (FftPlan *fp : {h->fft, h->fft2}) {
        if (!fp || !fft_tiles(*fp, true)) continue;
        const int c0 = fp == h->fft ? KC_FFT_HT0 : KC_FFT2_HT0;
        for (int pass = 0; pass < 3; ++pass) {
            cudaEvent_t ev = nullptr;
            h->prof_begin(c0 + pass, &ev);
            CU(fft_HT_pass(*fp, pass, facets, h->stream));
            h->prof_end(c0 + pass, ev);
        }
    }
    return DEBLUR_OK;
}

// One Local-Solver step on every local facet (K1 + K2, or the FFT path + K4).
static deblur_status local_step(deblur_t h, int last) {
    cudaEvent_t ev = nullptr;
    if (h->conv_path == DEBLUR_CONV_FFT) {
        deblur_status st;
        if ((st = run_fft_H(h, h->d_facets, h->par, FFT_RESIDUAL)) != DEBLUR_OK) return st;
        if ((st = run_fft_HT(h, h->d_facets)) != DEBLUR_OK) return st;
        if ((st = join_consensus(h)) != DEBLUR_OK) return st;          // K4 reads u
        h->prof_begin(KC_UPDATE_G, &ev);
        CU(launch_update_from_g(h->d_facets, h->d_tilesHT, (int)h->tilesHT.size(), h->plan.P, h->par, last, h->sc,
                                nullptr, h->stream));
        h->prof_end(KC_UPDATE_G, ev);
    } else {
        h->prof_begin(KC_H, &ev);
        CU(launch_H_direct(h->conv_args(h->d_facets, false), H_RESIDUAL, h->par, h->stream));
        h->prof_end(KC_H, ev);
        deblur_status st = join_consensus(h);                          // K2's epilogue reads u
        if (st != DEBLUR_OK) return st;
        h->prof_begin(KC_HT_UPDATE, &ev);
        CU(launch_HT_direct(h->conv_args(h->d_facets, true), HT_UPDATE, h->par, last, h->sc, h->stream));
        h->prof_end(KC_HT_UPDATE, ev);
    }
    h->par ^= 1;
    return DEBLUR_OK;
}

// ----------------------------------------------------------------------------- C ABI
extern "C" {

deblur_status deblur_nccl_id(void *out128) {
    if (!out128) return DEBLUR_EINVAL;
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) { g_last_error = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r); return DEBLUR_ENCCL; }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
    return DEBLUR_OK;
}

const char *deblur_last_error(deblur_t h) { return h ? h->err.c_str() : g_last_error.c_str(); }

const char *deblur_kernel_name(int32_t cls) { return (cls >= 0 && cls < KC_COUNT) ? k_names[cls] : ""; }

deblur_status deblur_plan_facets(const deblur_params *p, int32_t *n_facets, int64_t *boxes, int32_t *owner) {
    std::string err;
    deblur_status s = validate(p, err);
    if (s != DEBLUR_OK) { g_last_error = err; return s; }
    Plan pl;
    err = make_plan(p->ny, p->nx, p->psf_size, p->facet_gy, p->facet_gx, p->overlap, p->world, pl);
    if (!err.empty()) { g_last_error = err; return DEBLUR_ESHAPE; }
    if (n_facets) *n_facets = (int32_t)pl.facets.size();
    for (size_t i = 0; i < pl.facets.size(); ++i) {
        const FacetPlan &f = pl.facets[i];
        if (boxes) {
            const int64_t b[8] = {f.oy0, f.oy1, f.ox0, f.ox1, f.ey0, f.ey1, f.ex0, f.ex1};
            std::memcpy(boxes + 8 * i, b, sizeof b);
        }
        if (owner) owner[i] = f.owner;
    }
    return DEBLUR_OK;
}

deblur_status deblur_plan_messages(const deblur_params *p, int32_t rank, int32_t *n, int64_t *msgs) {
    std::string err;
    deblur_status s = validate(p, err);
    if (s != DEBLUR_OK) { g_last_error = err; return s; }
    if (!n) { g_last_error = "n is NULL"; return DEBLUR_EINVAL; }
    Plan pl;
    err = make_plan(p->ny, p->nx, p->psf_size, p->facet_gy, p->facet_gx, p->overlap, p->world, pl);
    if (!err.empty()) { g_last_error = err; return DEBLUR_ESHAPE; }
    if (rank < 0 || rank >= p->world) { g_last_error = "rank out of range"; return DEBLUR_EINVAL; }
    auto m = messages_from(pl, rank);
    *n = (int32_t)m.size();
    if (msgs)
        for (size_t i = 0; i < m.size(); ++i) {
            const int64_t r[8] = {m[i].peer, m[i].src_facet, m[i].dst_facet, m[i].rect.y0, m[i].rect.y1,
                                  m[i].rect.x0, m[i].rect.x1, m[i].bytes()};
            std::memcpy(msgs + 8 * i, r, sizeof r);
        }
    return DEBLUR_OK;
}

deblur_status deblur_destroy(deblur_t h) {
    if (!h) return DEBLUR_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->cstream) cudaStreamSynchronize(h->cstream);
    if (h->up_stream) cudaStreamSynchronize(h->up_stream);
    if (h->down_stream) cudaStreamSynchronize(h->down_stream);
    for (auto &g : h->gexec)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    if (h->fft) { fft_destroy(h->fft); h->fft = nullptr; }
    if (h->fft2) { fft_destroy(h->fft2); h->fft2 = nullptr; }
    if (h->comm) { ncclCommDestroy(h->comm); h->comm = nullptr; }
    for (auto &p : h->pending) { h->ev_pool.push_back(p.a); h->ev_pool.push_back(p.b); }
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    for (void *p : h->allocs) cudaFree(p);
    for (cudaEvent_t e : {h->ev_staged, h->ev_yfree, h->ev_blend, h->ev_down[0], h->ev_down[1]})
        if (e) cudaEventDestroy(e);
    if (h->up_stream) cudaStreamDestroy(h->up_stream);
    if (h->down_stream) cudaStreamDestroy(h->down_stream);
    if (h->ev_upd) cudaEventDestroy(h->ev_upd);
    if (h->ev_cons) cudaEventDestroy(h->ev_cons);
    if (h->cstream) cudaStreamDestroy(h->cstream);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return DEBLUR_OK;
}

deblur_status deblur_create(const deblur_params *p, deblur_t *out) {
    if (!out) { g_last_error = "out is NULL"; return DEBLUR_EINVAL; }
    *out = nullptr;
    std::string err;
    deblur_status st = validate(p, err);
    if (st != DEBLUR_OK) { g_last_error = err; return st; }
    std::unique_ptr<deblur_ctx> hp(new (std::nothrow) deblur_ctx());
    if (!hp) { g_last_error = "host allocation failed"; return DEBLUR_ENOMEM; }
    deblur_t h = hp.get();
    h->prm = *p;
    h->rank = p->rank; h->world = p->world; h->device = p->device;
    if (const char *ng = std::getenv("DEBLUR_NO_GRAPHS")) h->use_graphs = (ng[0] == '0');
    err = make_plan(p->ny, p->nx, p->psf_size, p->facet_gy, p->facet_gx, p->overlap, p->world, h->plan);
    if (!err.empty()) { g_last_error = err; return DEBLUR_ESHAPE; }
    const Plan &pl = h->plan;
    const int P = pl.P;
    Plan vplan;                           // loopback transport: the world-V plan of the virtual ranks
    h->vowner.assign(pl.facets.size(), h->rank);
    if (p->world == 1 && p->loopback_world > 1) {
        err = make_plan(p->ny, p->nx, p->psf_size, p->facet_gy, p->facet_gx, p->overlap, p->loopback_world, vplan);
        if (!err.empty()) { g_last_error = "loopback_world: " + err; return DEBLUR_ESHAPE; }
        h->vworld = p->loopback_world;
        for (const auto &f : vplan.facets) h->vowner[f.id] = f.owner;
    }
    h->per_node = p->operator_mode == DEBLUR_OP_PER_NODE;
    if (h->per_node) {
        err = check_node_weights(pl, p->interp_wy, p->interp_wx);
        if (!err.empty()) { g_last_error = err; return DEBLUR_EINVAL; }
    }

    // device
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0) {
        g_last_error = std::string("no CUDA device: ") + (ce != cudaSuccess ? cudaGetErrorString(ce) : "count 0");
        return DEBLUR_ECUDA;
    }
    if (p->device < 0 || p->device >= ndev) { g_last_error = "device ordinal out of range"; return DEBLUR_EINVAL; }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, p->device) != cudaSuccess || prop.major != 10) {
        g_last_error = "device is not sm_100 (this library is built for sm_100a only; no fallback)";
        return DEBLUR_ECUDA;
    }
#define CUC(call)                                                                             \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            g_last_error = std::string("CUDA error in create: ") + cudaGetErrorString(e_) + " at " #call; \
            return e_ == cudaErrorMemoryAllocation ? DEBLUR_ENOMEM : DEBLUR_ECUDA;             \
        }                                                                                     \
    } while (0)
    CUC(cudaSetDevice(p->device));
    CUC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    {
        // the exchange + consensus stream at the greatest priority: its few CTAs are
        // dispatched ahead of the next iteration's H passes instead of trickling in beside
        // them (c4: K5 0.144 ms instead of 1.13 ms spread over the H R2C pass; step time
        // unchanged, 10.80 ms) -- the band values reach the neighbours as early as possible
        int lo = 0, hi = 0;
        CUC(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUC(cudaStreamCreateWithPriority(&h->cstream, cudaStreamNonBlocking, hi));
    }
    CUC(cudaEventCreateWithFlags(&h->ev_upd, cudaEventDisableTiming));
    CUC(cudaEventCreateWithFlags(&h->ev_cons, cudaEventDisableTiming));
    CUC(cudaStreamCreateWithFlags(&h->up_stream, cudaStreamNonBlocking));
    CUC(cudaStreamCreateWithFlags(&h->down_stream, cudaStreamNonBlocking));
    for (cudaEvent_t *e : {&h->ev_staged, &h->ev_yfree, &h->ev_blend, &h->ev_down[0], &h->ev_down[1]})
        CUC(cudaEventCreateWithFlags(e, cudaEventDisableTiming));

    // conv path (A: measured crossover)
    int path = p->conv_path;
    if (path == DEBLUR_CONV_AUTO) path = fft_prefer(P) ? DEBLUR_CONV_FFT : DEBLUR_CONV_DIRECT;
    if (path == DEBLUR_CONV_DIRECT && !direct_supported(P)) {
        g_last_error = "psf_size too large for the direct path; use conv_path FFT";
        return DEBLUR_EINVAL;
    }
    h->conv_path = path;

    // global read-only inputs
    const int K = p->psf_gy * p->psf_gx;
    CUC(h->dalloc(&h->d_psfs, (size_t)K * P * P));
    CUC(h->dalloc(&h->d_wy, (size_t)p->psf_gy * p->ny));
    CUC(h->dalloc(&h->d_wx, (size_t)p->psf_gx * p->nx));
    CUC(cudaMemcpy(h->d_psfs, p->psfs, sizeof(float) * K * P * P, cudaMemcpyHostToDevice));
    CUC(cudaMemcpy(h->d_wy, p->interp_wy, sizeof(float) * p->psf_gy * p->ny, cudaMemcpyHostToDevice));
    CUC(cudaMemcpy(h->d_wx, p->interp_wx, sizeof(float) * p->psf_gx * p->nx, cudaMemcpyHostToDevice));
    h->h_wy.assign(p->interp_wy, p->interp_wy + (size_t)p->psf_gy * p->ny);
    h->h_wx.assign(p->interp_wx, p->interp_wx + (size_t)p->psf_gx * p->nx);
    h->d_owy = h->d_wy;
    h->d_owx = h->d_wx;
    if (h->per_node) {
        const std::vector<float> oy((size_t)p->psf_gy * p->ny, 1.f), ox((size_t)p->psf_gx * p->nx, 1.f);
        CUC(h->dalloc(&h->d_owy, oy.size()));
        CUC(h->dalloc(&h->d_owx, ox.size()));
        CUC(cudaMemcpy(h->d_owy, oy.data(), sizeof(float) * oy.size(), cudaMemcpyHostToDevice));
        CUC(cudaMemcpy(h->d_owx, ox.data(), sizeof(float) * ox.size(), cudaMemcpyHostToDevice));
    }

    // local facets
    h->local_index.assign(pl.facets.size(), -1);
    for (const auto &f : pl.facets)
        if (f.owner == h->rank) { h->local_index[f.id] = (int)h->local.size(); h->local.push_back(f.id); }
    auto axisw = [](int64_t e0, int64_t e1, int64_t pe, int64_t ns, const float *w) {
        AxisW a;
        a.e0 = (int)e0; a.n = (int)(e1 - e0);
        a.b_prev = (int)(pe - e0); a.b_next = (int)(ns - e0);
        a.s_prev = (int)e0; a.e_prev = (int)pe;
        a.s_next = (int)ns; a.e_next = (int)e1;
        a.w = w;
        return a;
    };
    // per-node consensus weights: facet (a, b) uses interp_wy[a], interp_wx[b]
    auto node_wy = [&](const FacetPlan &f) { return h->per_node ? h->d_wy + (size_t)f.fy * p->ny : nullptr; };
    auto node_wx = [&](const FacetPlan &f) { return h->per_node ? h->d_wx + (size_t)f.fx * p->nx : nullptr; };
    for (int id : h->local) {
        const FacetPlan &fp = pl.facets[id];
        FacetDev F{};
        F.id = id;
        F.ny = (int)(fp.ey1 - fp.ey0); F.nx = (int)(fp.ex1 - fp.ex0);
        F.my = (int)(fp.oy1 - fp.oy0); F.mx = (int)(fp.ox1 - fp.ox0);
        F.ey0 = (int)fp.ey0; F.ex0 = (int)fp.ex0;
        F.ep = round_up(F.nx, 32); F.op = round_up(F.mx, 32);
        const size_t ne = (size_t)F.ny * F.ep, no = (size_t)F.my * F.op;
        float *y_ = nullptr, *w_ = nullptr;
        CUC(h->dalloc(&F.x[0], ne)); CUC(h->dalloc(&F.x[1], ne));
        CUC(h->dalloc(&F.u, ne)); CUC(h->dalloc(&F.v, ne)); CUC(h->dalloc(&F.g, ne));
        CUC(h->dalloc(&y_, no)); CUC(h->dalloc(&F.r, no));
        for (float *b : {F.x[0], F.x[1], F.u, F.v, F.g}) CUC(cudaMemsetAsync(b, 0, ne * 4, h->stream));
        CUC(cudaMemsetAsync(y_, 0, no * 4, h->stream)); CUC(cudaMemsetAsync(F.r, 0, no * 4, h->stream));
        if (p->noise_w) {
            CUC(h->dalloc(&w_, no));
            CUC(cudaMemsetAsync(w_, 0, no * 4, h->stream));
            CUC(cudaMemcpy2DAsync(w_, F.op * 4, p->noise_w + fp.oy0 * pl.mx + fp.ox0, pl.mx * 4, F.mx * 4, F.my,
                                  cudaMemcpyHostToDevice, h->stream));
        }
        F.y = y_; F.w = w_; F.w_scalar = p->noise_w_scalar;
        F.ay = axisw(fp.ey0, fp.ey1, fp.py_e, fp.ny_s, node_wy(fp));
        F.ax = axisw(fp.ex0, fp.ex1, fp.px_e, fp.nx_s, node_wx(fp));
        for (int dy = 0; dy < 3; ++dy)
            for (int dx = 0; dx < 3; ++dx) F.nb[dy][dx].id = -1;
        h->fh.push_back(F);
    }

    // halo messages (world > 1) and neighbour views
    h->sends.clear(); h->recvs.clear();
    if (h->world > 1) {
        for (auto &m : messages_from(pl, h->rank)) { SendRecv s; s.m = m; h->sends.push_back(s); }
        for (auto &m : messages_to(pl, h->rank)) { SendRecv s; s.m = m; h->recvs.push_back(s); }
    } else if (h->vworld > 1) {
        for (int vr = 0; vr < h->vworld; ++vr) {
            for (auto &m : messages_from(vplan, vr)) { SendRecv s; s.m = m; h->sends.push_back(s); }
            for (auto &m : messages_to(vplan, vr)) { SendRecv s; s.m = m; h->recvs.push_back(s); }
        }
        for (auto &s : h->sends)
            for (size_t i = 0; i < h->recvs.size(); ++i)
                if (h->recvs[i].m.src_facet == s.m.src_facet && h->recvs[i].m.dst_facet == s.m.dst_facet)
                    s.peer_index = (int)i;
        for (auto &s : h->sends)
            if (s.peer_index < 0) { g_last_error = "loopback: unmatched halo message"; return DEBLUR_ESHAPE; }
    }
    {
        for (auto *lst : {&h->sends, &h->recvs})
            for (auto &s : *lst) {
                CUC(h->dalloc(&s.vbuf, (size_t)s.m.rect.area()));
                CUC(h->dalloc(&s.xbuf, (size_t)s.m.rect.area()));
            }
    }
    for (size_t li = 0; li < h->local.size(); ++li) {
        FacetDev &F = h->fh[li];
        const FacetPlan &fp = pl.facets[F.id];
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int gy = fp.fy + dy, gx = fp.fx + dx;
                if (gy < 0 || gy >= pl.Fy || gx < 0 || gx >= pl.Fx) continue;
                const FacetPlan &np = pl.facets[gy * pl.Fx + gx];
                Neighbour &nb = F.nb[dy + 1][dx + 1];
                nb.id = np.id;
                nb.ay = axisw(np.ey0, np.ey1, np.py_e, np.ny_s, node_wy(np));
                nb.ax = axisw(np.ex0, np.ex1, np.px_e, np.nx_s, node_wx(np));
                const int nli = h->local_index[np.id];
                if (nli >= 0 && h->vowner[np.id] == h->vowner[F.id]) {     // same (virtual) rank: direct read
                    const FacetDev &N = (nli == (int)li) ? F : h->fh[nli];
                    nb.v.base[0] = nb.v.base[1] = N.v;
                    nb.v.pitch = N.ep; nb.v.y0 = N.ey0; nb.v.x0 = N.ex0; nb.v.valid = 1;
                    nb.x.base[0] = N.x[0]; nb.x.base[1] = N.x[1];
                    nb.x.pitch = N.ep; nb.x.y0 = N.ey0; nb.x.x0 = N.ex0; nb.x.valid = 1;
                } else {
                    for (auto &r : h->recvs)
                        if (r.m.src_facet == np.id && r.m.dst_facet == F.id) {
                            const int64_t w = r.m.rect.x1 - r.m.rect.x0;
                            nb.v.base[0] = nb.v.base[1] = r.vbuf;
                            nb.v.pitch = w; nb.v.y0 = (int)r.m.rect.y0; nb.v.x0 = (int)r.m.rect.x0; nb.v.valid = 1;
                            nb.x.base[0] = nb.x.base[1] = r.xbuf;
                            nb.x.pitch = w; nb.x.y0 = (int)r.m.rect.y0; nb.x.x0 = (int)r.m.rect.x0; nb.x.valid = 1;
                        }
                }
            }
        // band rectangles (facet-local): pixels in >= 2 facets, split into the 8 pieces
        // of the 3 x 3 (previous band | core | next band) grid around the core, so the
        // set of contributing neighbours is constant on each piece
        const int rb[4] = {0, F.ay.b_prev, F.ay.b_next, F.ny}, cb[4] = {0, F.ax.b_prev, F.ax.b_next, F.nx};
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                if (a == 1 && b == 1) continue;                    // single-owner core
                if (rb[a + 1] <= rb[a] || cb[b + 1] <= cb[b]) continue;
                const BandRect R{(int)li, rb[a], rb[a + 1], cb[b], cb[b + 1],
                                 a == 0 ? -1 : 0, a == 2 ? 1 : 0, b == 0 ? -1 : 0, b == 2 ? 1 : 0};
                const int ri = (int)h->rects.size();
                h->rects.push_back(R);
                for (int y = R.y0; y < R.y1; y += CT_ROWS)
                    for (int x = R.x0; x < R.x1; x += 256) h->rect_tiles.push_back({ri, y, x});
            }
    }

    // tiles with active PSF ranges
    NzIndex nzy, nzx;
    nzy.build(p->interp_wy, p->psf_gy, p->ny);
    nzx.build(p->interp_wx, p->psf_gx, p->nx);
    const int tyH = direct_ty_H(P), tyHT = direct_ty_HT(P), TXd = DIRECT_TX;
    auto node_range = [](TileDesc &t, const FacetPlan &f) {   // the facet's own PSF only
        t.p0 = t.p1 = f.fy;
        t.q0 = t.q1 = f.fx;
    };
    for (size_t li = 0; li < h->local.size(); ++li) {
        const FacetDev &F = h->fh[li];
        for (int y0 = 0; y0 < F.my; y0 += tyH)
            for (int x0 = 0; x0 < F.mx; x0 += TXd) {
                TileDesc t{(int)li, y0, x0, 0, -1, 0, -1};
                nzy.range(F.ey0 + y0, F.ey0 + std::min(y0 + tyH + P - 1, F.ny), t.p0, t.p1);
                nzx.range(F.ex0 + x0, F.ex0 + std::min(x0 + TXd + P - 1, F.nx), t.q0, t.q1);
                if (h->per_node) node_range(t, pl.facets[F.id]);
                h->tilesH.push_back(t);
            }
        for (int y0 = 0; y0 < F.ny; y0 += tyHT)
            for (int x0 = 0; x0 < F.nx; x0 += TXd) {
                TileDesc t{(int)li, y0, x0, 0, -1, 0, -1};
                nzy.range(F.ey0 + y0, F.ey0 + std::min(y0 + tyHT, F.ny), t.p0, t.p1);
                nzx.range(F.ex0 + x0, F.ex0 + std::min(x0 + TXd, F.nx), t.q0, t.q1);
                if (h->per_node) node_range(t, pl.facets[F.id]);
                h->tilesHT.push_back(t);
            }
    }
    CUC(h->dalloc(&h->d_tilesH, h->tilesH.size()));
    CUC(h->dalloc(&h->d_tilesHT, h->tilesHT.size()));
    CUC(h->dalloc(&h->d_rects, h->rects.size()));
    CUC(cudaMemcpy(h->d_tilesH, h->tilesH.data(), sizeof(TileDesc) * h->tilesH.size(), cudaMemcpyHostToDevice));
    CUC(cudaMemcpy(h->d_tilesHT, h->tilesHT.data(), sizeof(TileDesc) * h->tilesHT.size(), cudaMemcpyHostToDevice));
    CUC(cudaMemcpy(h->d_rects, h->rects.data(), sizeof(BandRect) * h->rects.size(), cudaMemcpyHostToDevice));
    CUC(h->dalloc(&h->d_rect_tiles, std::max<size_t>(1, h->rect_tiles.size())));
    if (!h->rect_tiles.empty())
        CUC(cudaMemcpy(h->d_rect_tiles, h->rect_tiles.data(), sizeof(RectTile) * h->rect_tiles.size(),
                       cudaMemcpyHostToDevice));
    const size_t npart = std::max({h->tilesH.size(), h->tilesHT.size(), h->rects.size(), (size_t)1});
    CUC(h->dalloc(&h->d_partials, npart));
    h->h_partials.resize(npart);

    CUC(h->dalloc(&h->d_facets, h->fh.size()));
    CUC(h->dalloc(&h->d_facets_alt, h->fh.size()));
    CUC(cudaMemcpy(h->d_facets, h->fh.data(), sizeof(FacetDev) * h->fh.size(), cudaMemcpyHostToDevice));
    {
        std::vector<FacetDev> alt = h->fh;
        for (auto &F : alt) { F.x[0] = F.x[1] = F.g; }
        CUC(cudaMemcpy(h->d_facets_alt, alt.data(), sizeof(FacetDev) * alt.size(), cudaMemcpyHostToDevice));
    }

    // VMLM-B Local-Solver state
    if (p->local_solver == 1) {
        if (h->local.size() > (size_t)VM_MAXF) {
            g_last_error = "VMLM-B Local-Solver: more than 64 facets on one rank";
            return DEBLUR_EINVAL;
        }
        auto &V = h->vm;
        V.on = true;
        const size_t nl = h->local.size();
        V.G.resize(nl); V.Gn.resize(nl); V.D.resize(nl); V.Q.resize(nl); V.M.resize(nl);
        V.S.resize(nl); V.Y.resize(nl); V.sy.resize(nl); V.yy.resize(nl);
        for (size_t li = 0; li < nl; ++li) {
            const size_t ne = (size_t)h->fh[li].ny * h->fh[li].ep;
            for (float **b : {&V.G[li], &V.Gn[li], &V.D[li], &V.Q[li]}) {
                CUC(h->dalloc(b, ne));
                CUC(cudaMemsetAsync(*b, 0, ne * 4, h->stream));
            }
            CUC(h->dalloc(&V.M[li], ne));
            for (int k = 0; k < deblur_ctx::Vm::m; ++k) {
                CUC(h->dalloc(&V.S[li][k], ne));
                CUC(h->dalloc(&V.Y[li][k], ne));
            }
        }
        CUC(h->dalloc(&V.d_part, std::max<size_t>(1, 3 * h->tilesHT.size())));
        V.h_part.resize(3 * h->tilesHT.size() + 1);
    }

    // solver constants
    h->tau = (p->tau > 0) ? p->tau : default_tau(p);
    h->sc.lambda = p->lambda; h->sc.eps = p->eps; h->sc.gamma = p->independent ? 0.f : p->gamma; h->sc.rho = p->rho;
    h->sc.tau = (float)h->tau; h->sc.reg_kind = p->reg_kind; h->sc.tv_boundary = p->tv_boundary;

    // data + initial state
    st = stage_y(h, p->y);
    if (st == DEBLUR_OK) st = upload_y(h);
    if (st != DEBLUR_OK) { g_last_error = h->err; return st; }
    st = upload_state_x0(h, p->x0);
    if (st != DEBLUR_OK) { g_last_error = h->err; return st; }

    // FFT path plan
    if (h->conv_path == DEBLUR_CONV_FFT) {
        std::string ferr;
        // ragged strips: where the last row / column of S-tiles would hold at most T2 valid
        // outputs, a plan of size S2 = S/2 covers that strip (about half the work per
        // output column); the S plan covers the rest
        const int S1 = fft_choose_size(P), S2 = S1 / 2, T1 = S1 - P + 1, T2 = S2 - P + 1;
        FftRegions r1, r2;
        bool strips = false;
        const bool want = T2 >= 64 && !std::getenv("DEBLUR_FFT_NO_STRIPS") && !std::getenv("DEBLUR_FFT_SIZE");
        auto bulk = [&](int m) {
            const int t = (m + T1 - 1) / T1, rem = m - (t - 1) * T1;
            return (want && t > 1 && rem <= T2) ? (t - 1) * T1 : m;
        };
        auto split = [&](int my, int mx, std::vector<FftRect> &a, std::vector<FftRect> &b) {
            const int yb = bulk(my), xb = bulk(mx);
            a.push_back({0, yb, 0, xb});
            if (yb < my) b.push_back({yb, my, 0, mx});
            if (xb < mx) b.push_back({0, yb, xb, mx});
            strips |= (yb < my || xb < mx);
        };
        for (const FacetDev &F : h->fh) {
            r1.H.emplace_back(); r1.HT.emplace_back(); r2.H.emplace_back(); r2.HT.emplace_back();
            split(F.my, F.mx, r1.H.back(), r2.H.back());
            split(F.ny, F.nx, r1.HT.back(), r2.HT.back());
        }
        h->fft = fft_create(pl, h->local, h->fh, h->d_psfs, h->d_owy, h->d_owx, p->psf_gy, p->psf_gx, h->h_wy.data(),
                            h->h_wx.data(), h->per_node, h->stream, ferr, 0, strips ? &r1 : nullptr);
        if (!h->fft) { g_last_error = "FFT path: " + ferr; return DEBLUR_ECUDA; }
        if (strips) {
            h->fft2 = fft_create(pl, h->local, h->fh, h->d_psfs, h->d_owy, h->d_owx, p->psf_gy, p->psf_gx,
                                 h->h_wy.data(), h->h_wx.data(), h->per_node, h->stream, ferr, S2, &r2);
            if (!h->fft2) { g_last_error = "FFT path (strips): " + ferr; return DEBLUR_ECUDA; }
        }
    }

    // NCCL
    if (h->world > 1) {
        CUC(h->dalloc(&h->d_objbuf, 2 * pl.facets.size() + 1));
        ncclUniqueId id;
        std::memcpy(&id, p->nccl_id, sizeof id);
        ncclResult_t r = ncclCommInitRank(&h->comm, h->world, id, h->rank);
        if (r != ncclSuccess) { g_last_error = std::string("ncclCommInitRank: ") + ncclGetErrorString(r); return DEBLUR_ENCCL; }
    }
    CUC(cudaStreamSynchronize(h->stream));
    h->prm.psfs = nullptr; h->prm.interp_wy = h->prm.interp_wx = nullptr;
    h->prm.y = h->prm.noise_w = h->prm.x0 = nullptr; h->prm.nccl_id = nullptr;
    *out = hp.release();
#undef CUC
    return DEBLUR_OK;
}

// ----------------------------------------------------------------- VMLM-B Local-Solver
// Reading V1-V6 (oracle/vmlmb.py): projected L-BFGS with the free set
// x > 0 or g < 0, two-loop recursion over the last m = 5 pairs restricted to it,
// H0 = <s,y>/<y,y> or tau, projected backtracking (Armijo c1 = 1e-4, <= 10 halvings;
// a facet without an acceptable step stops), pairs kept iff <s,y> > 1e-12 |s||y|.
// The vector work runs on the device for all local facets at once; the per-facet
// scalars come back as fp64 partial sums and every decision is taken on the host.
#define VMK(cls, call)                          \
    do {                                        \
        cudaEvent_t ev_ = nullptr;              \
        h->prof_begin(cls, &ev_);               \
        CU(call);                               \
        h->prof_end(cls, ev_);                  \
    } while (0)

static VmArgs vm_base(deblur_t h, int nsum) {
    VmArgs a;
    std::memset(&a, 0, sizeof a);
    a.facets = h->d_facets;
    a.tiles = h->d_tilesHT;
    a.ntiles = (int)h->tilesHT.size();
    a.par = h->par;
    a.nsum = nsum;
    a.partials = h->vm.d_part;
    return a;
}

// per-local-facet sums of the nsum partial rows (tile order; after a stream sync)
static deblur_status vm_sums(deblur_t h, int nsum, std::vector<std::array<double, 3>> &out) {
    const size_t nt = h->tilesHT.size();
    CU(cudaMemcpyAsync(h->vm.h_part.data(), h->vm.d_part, sizeof(double) * 3 * nt, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    out.assign(h->local.size(), {0.0, 0.0, 0.0});
    for (int k = 0; k < nsum; ++k)
        for (size_t t = 0; t < nt; ++t) out[h->tilesHT[t].f][k] += h->vm.h_part[k * nt + t];
    return DEBLUR_OK;
}

// f_f(w) + 1/2 |w - u_f|^2_alpha at w = x[par_w] (without the indicator) and its
// gradient into Gd, for every local facet
static deblur_status vm_eval(deblur_t h, int par_w, std::vector<float *> &Gd, std::vector<double> &f) {
    deblur_status s;
    const size_t nl = h->local.size();
    std::vector<double> data(nl, 0.0);
    if (h->conv_path == DEBLUR_CONV_FFT) {
        if ((s = run_fft_H(h, h->d_facets, par_w, FFT_RESIDUAL)) != DEBLUR_OK) return s;
        CU(cudaStreamSynchronize(h->stream));
        CU(fft_partials_all(h, data));
        if ((s = run_fft_HT(h, h->d_facets)) != DEBLUR_OK) return s;
    } else {
        cudaEvent_t ev = nullptr;
        h->prof_begin(KC_H, &ev);
        CU(launch_H_direct(h->conv_args(h->d_facets, false), H_RESIDUAL, par_w, h->stream));
        h->prof_end(KC_H, ev);
        CU(cudaMemcpyAsync(h->h_partials.data(), h->d_partials, sizeof(double) * h->tilesH.size(),
                           cudaMemcpyDeviceToHost, h->stream));
        CU(cudaStreamSynchronize(h->stream));
        for (size_t t = 0; t < h->tilesH.size(); ++t) data[h->tilesH[t].f] += h->h_partials[t];
        ConvArgs ca = h->conv_args(h->d_facets, true);
        ca.partials = nullptr;
        h->prof_begin(KC_HT_PLAIN, &ev);
        CU(launch_HT_direct(ca, HT_PLAIN, par_w, 0, h->sc, h->stream));
        h->prof_end(KC_HT_PLAIN, ev);
    }
    VmArgs a = vm_base(h, 2);
    a.par = par_w;
    for (size_t li = 0; li < nl; ++li) a.A[li] = Gd[li];
    VMK(KC_VM_GRAD, vm_grad(a, h->sc, h->stream));
    std::vector<std::array<double, 3>> rp;
    if ((s = vm_sums(h, 2, rp)) != DEBLUR_OK) return s;
    f.assign(nl, 0.0);
    for (size_t li = 0; li < nl; ++li) {
        f[li] = data[li] + (double)h->sc.lambda * rp[li][0] + rp[li][1];
        if (!std::isfinite(f[li])) {
            std::ostringstream o;
            o << "non-finite local objective on facet " << h->local[li] << " (VMLM-B)";
            return h->fail(DEBLUR_ENUMERIC, o.str());
        }
    }
    ++h->vm.evaluations;
    return DEBLUR_OK;
}

static deblur_status vm_local_solve(deblur_t h) {
    auto &V = h->vm;
    constexpr int m = deblur_ctx::Vm::m;
    const size_t nl = h->local.size();
    const int budget = h->prm.inner_steps + V.k_outer * h->prm.inner_increment;
    const double h0 = h->tau, c1 = 1e-4;
    deblur_status s;
    std::vector<double> f, fn;
    if ((s = vm_eval(h, h->par, V.G, f)) != DEBLUR_OK) return s;
    std::vector<int> head(nl, 0), np(nl, 0);
    std::vector<std::array<double, m>> rho(nl), alpha(nl);
    std::vector<char> done(nl, 0);
    std::vector<std::array<double, 3>> sm;
    for (int it = 0; it < budget; ++it) {
        if (std::all_of(done.begin(), done.end(), [](char d) { return d != 0; })) break;
        ++V.iterations;
        // V2 free set, q = g on it
        VmArgs a = vm_base(h, 0);
        for (size_t li = 0; li < nl; ++li) { a.A[li] = V.Q[li]; a.B[li] = V.G[li]; a.Mo[li] = V.M[li]; }
        VMK(KC_VM_VEC, vm_mask_q(a, h->stream));
        // V3 two-loop: newest -> oldest (pair j of facet li: slot (head - 1 - j) mod m)
        int maxp = 0;
        for (size_t li = 0; li < nl; ++li) maxp = std::max(maxp, np[li]);
        auto slot = [&](size_t li, int j) { return ((head[li] - 1 - j) % m + m) % m; };
        std::vector<std::array<double, 3>> dots;
        if (maxp > 0) {       // <s_newest, q>
            VmArgs d = vm_base(h, 1);
            for (size_t li = 0; li < nl; ++li) { d.B[li] = V.Q[li]; d.C[li] = np[li] > 0 ? V.S[li][slot(li, 0)] : V.Q[li]; }
            VMK(KC_VM_VEC, vm_dot(d, h->stream));
            if ((s = vm_sums(h, 1, dots)) != DEBLUR_OK) return s;
        }
        for (int j = 0; j < maxp; ++j) {
            VmArgs x = vm_base(h, j + 1 < maxp ? 1 : 0);
            for (size_t li = 0; li < nl; ++li) {
                const bool has = j < np[li];
                alpha[li][j] = has ? rho[li][slot(li, j)] * dots[li][0] : 0.0;
                x.A[li] = V.Q[li];
                x.B[li] = has ? V.Y[li][slot(li, j)] : nullptr;
                x.M[li] = V.M[li];
                x.c0[li] = -alpha[li][j];
                x.c1[li] = 1.0;
                x.C[li] = (j + 1 < maxp) ? (j + 1 < np[li] ? V.S[li][slot(li, j + 1)] : V.Q[li]) : nullptr;
            }
            VMK(KC_VM_VEC, vm_axpy_dot(x, h->stream));
            if (j + 1 < maxp && (s = vm_sums(h, 1, dots)) != DEBLUR_OK) return s;
        }
        // r = H0 q (in place in Q), and <y_oldest, r> for the forward loop
        {
            VmArgs x = vm_base(h, maxp > 0 ? 1 : 0);
            for (size_t li = 0; li < nl; ++li) {
                double H0 = h0;
                if (np[li] > 0) H0 = V.sy[li][slot(li, 0)] / V.yy[li][slot(li, 0)];
                x.A[li] = V.Q[li];
                x.B[li] = nullptr;
                x.M[li] = V.M[li];
                x.c0[li] = 0.0;
                x.c1[li] = H0;
                x.C[li] = maxp > 0 ? (np[li] > 0 ? V.Y[li][slot(li, np[li] - 1)] : V.Q[li]) : nullptr;
            }
            VMK(KC_VM_VEC, vm_axpy_dot(x, h->stream));
            if (maxp > 0 && (s = vm_sums(h, 1, dots)) != DEBLUR_OK) return s;
        }
        // forward loop oldest -> newest: b = rho <y, r>; r += (alpha - b) s
        for (int j = maxp - 1; j >= 0; --j) {
            VmArgs x = vm_base(h, j > 0 ? 1 : 0);
            for (size_t li = 0; li < nl; ++li) {
                const bool has = j < np[li];
                const int jj = has ? j : 0;
                // the facet's own order: its oldest pair is j = np - 1
                const bool act = has && j <= np[li] - 1;
                const double b = act ? rho[li][slot(li, jj)] * dots[li][0] : 0.0;
                x.A[li] = V.Q[li];
                x.B[li] = act ? V.S[li][slot(li, jj)] : nullptr;
                x.M[li] = V.M[li];
                x.c0[li] = act ? alpha[li][jj] - b : 0.0;
                x.c1[li] = 1.0;
                x.C[li] = (j > 0) ? (j - 1 < np[li] ? V.Y[li][slot(li, j - 1)] : V.Q[li]) : nullptr;
            }
            VMK(KC_VM_VEC, vm_axpy_dot(x, h->stream));
            if (j > 0 && (s = vm_sums(h, 1, dots)) != DEBLUR_OK) return s;
        }
        // d = -r on the free set; descent check, else reset (memory dropped, d = -h0 g_F)
        {
            VmArgs x = vm_base(h, 1);
            for (size_t li = 0; li < nl; ++li) {
                x.A[li] = V.D[li]; x.B[li] = V.Q[li]; x.C[li] = V.G[li]; x.M[li] = V.M[li]; x.c0[li] = 0.0;
            }
            VMK(KC_VM_VEC, vm_direction(x, h->stream));
            if ((s = vm_sums(h, 1, dots)) != DEBLUR_OK) return s;
            bool any = false;
            for (size_t li = 0; li < nl; ++li)
                if (!(dots[li][0] < 0.0) && !done[li]) { x.c0[li] = h0; np[li] = 0; head[li] = 0; any = true; }
            if (any) VMK(KC_VM_VEC, vm_direction(x, h->stream));
        }
        // V4 projected backtracking
        std::vector<double> t(nl, 1.0), gdx(nl, 0.0);
        std::vector<char> acc(nl, 0);
        for (size_t li = 0; li < nl; ++li)
            if (done[li]) { t[li] = 0.0; acc[li] = 1; }
        bool stalled = false;
        for (int ls = 0; ls < 10; ++ls) {
            VmArgs x = vm_base(h, 1);
            for (size_t li = 0; li < nl; ++li) { x.B[li] = V.D[li]; x.C[li] = V.G[li]; x.c0[li] = t[li]; }
            VMK(KC_VM_VEC, vm_trial(x, h->stream));
            std::vector<std::array<double, 3>> gd;
            if ((s = vm_sums(h, 1, gd)) != DEBLUR_OK) return s;
            if ((s = vm_eval(h, h->par ^ 1, V.Gn, fn)) != DEBLUR_OK) return s;
            bool all = true;
            for (size_t li = 0; li < nl; ++li) {
                if (acc[li]) continue;
                if (fn[li] <= f[li] + c1 * gd[li][0]) acc[li] = 1;
                else { t[li] *= 0.5; all = false; }
            }
            if (all) break;
            if (ls == 9) stalled = true;
        }
        if (stalled) {        // no acceptable step: the facet stops at x (trial with t = 0)
            for (size_t li = 0; li < nl; ++li)
                if (!acc[li]) { done[li] = 1; t[li] = 0.0; }
            VmArgs x = vm_base(h, 1);
            for (size_t li = 0; li < nl; ++li) { x.B[li] = V.D[li]; x.C[li] = V.G[li]; x.c0[li] = t[li]; }
            VMK(KC_VM_VEC, vm_trial(x, h->stream));
            if ((s = vm_eval(h, h->par ^ 1, V.Gn, fn)) != DEBLUR_OK) return s;
        }
        // V5 memory pair
        {
            VmArgs x = vm_base(h, 3);
            for (size_t li = 0; li < nl; ++li) {
                x.A[li] = V.S[li][head[li]]; x.A2[li] = V.Y[li][head[li]]; x.B[li] = V.G[li]; x.C[li] = V.Gn[li];
            }
            VMK(KC_VM_VEC, vm_pair(x, h->stream));
            if ((s = vm_sums(h, 3, sm)) != DEBLUR_OK) return s;
            for (size_t li = 0; li < nl; ++li) {
                const double sy = sm[li][0], ss = sm[li][1], yy = sm[li][2];
                if (!done[li] && sy > 1e-12 * std::sqrt(ss) * std::sqrt(yy)) {
                    rho[li][head[li]] = 1.0 / sy;
                    V.sy[li][head[li]] = sy;
                    V.yy[li][head[li]] = yy;
                    head[li] = (head[li] + 1) % m;
                    np[li] = std::min(np[li] + 1, m);
                }
            }
        }
        std::swap(V.G, V.Gn);
        h->par ^= 1;
        f = fn;
    }
    return DEBLUR_OK;
}

static deblur_status one_iteration(deblur_t h) {
    deblur_status s;
    if (h->vm.on) {
        if ((s = join_consensus(h)) != DEBLUR_OK) return s;

        if ((s = vm_local_solve(h)) != DEBLUR_OK) return s;
        ++h->vm.k_outer;
        if (!h->prm.independent) {     // what the last projected-gradient step's epilogue writes
            VmArgs a = vm_base(h, 0);
            VMK(KC_VM_VEC, vm_finalize(a, h->sc.rho, h->stream));
        }
    } else {
        for (int k = 0; k < h->prm.inner_steps; ++k)
            // independent baseline: no dual / band values either (u stays u0, v unused)
            if ((s = local_step(h, k == h->prm.inner_steps - 1 && !h->prm.independent)) != DEBLUR_OK) return s;
    }
    if (h->prm.independent) return DEBLUR_OK;        // baseline: no exchange, no consensus
    // a5 + a6 on the consensus stream: they need x+ and v of this iteration; the next
    // iteration's H / H^T passes (x only) run under them (§8e)
    CU(cudaEventRecord(h->ev_upd, h->stream));
    CU(cudaStreamWaitEvent(h->cstream, h->ev_upd, 0));
    if ((s = exchange(h, 0, h->cstream)) != DEBLUR_OK) return s;
    cudaEvent_t ev = nullptr;
    h->prof_begin(KC_CONSENSUS, &ev, h->cstream);
    CU(launch_consensus(h->d_facets, h->d_rects, h->d_rect_tiles, (int)h->rect_tiles.size(), h->par, h->sc.rho,
                        h->cstream));
    h->prof_end(KC_CONSENSUS, ev, h->cstream);
    CU(cudaEventRecord(h->ev_cons, h->cstream));
    h->cons_pending = true;
    return DEBLUR_OK;
}

// Capture two iterations starting at the current parity into a CUDA graph (the
// launch-bound small configs spend most of a step in launch latency otherwise).
static deblur_status capture_pair(deblur_t h) {
    const int p0 = h->par;
    int64_t before[KC_COUNT];
    std::copy(h->stat_n, h->stat_n + KC_COUNT, before);
    CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
    deblur_status s = one_iteration(h);
    if (s == DEBLUR_OK) s = one_iteration(h);
    if (s == DEBLUR_OK) s = join_consensus(h);            // the forked consensus stream rejoins
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (s != DEBLUR_OK) { if (g) cudaGraphDestroy(g); return s; }
    if (e != cudaSuccess) return h->cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&h->gexec[p0], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return h->cuda_fail(e, "cudaGraphInstantiate");
    for (int i = 0; i < KC_COUNT; ++i) { h->graph_counts[p0][i] = h->stat_n[i] - before[i]; h->stat_n[i] = before[i]; }
    h->par = p0;     // 2 iterations flip the parity an even number of times
    return DEBLUR_OK;
}

deblur_status deblur_iterate(deblur_t h, int32_t n) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (n < 0) return h->fail(DEBLUR_EINVAL, "n must be >= 0");
    int done = 0;
    if (!h->prof && h->use_graphs && n >= 2 && !h->vm.on) {
        const int p0 = h->par;
        if (!h->gexec[p0] && (s = capture_pair(h)) != DEBLUR_OK) return s;
        for (; done + 2 <= n; done += 2) {
            CU(cudaGraphLaunch(h->gexec[p0], h->stream));
            for (int i = 0; i < KC_COUNT; ++i) h->stat_n[i] += h->graph_counts[p0][i];
        }
    }
    for (; done < n; ++done)
        if ((s = one_iteration(h)) != DEBLUR_OK) return s;
    if ((s = join_consensus(h)) != DEBLUR_OK) return s;    // callers time on h->stream
    return finish(h);
}

deblur_status deblur_iterate_traced(deblur_t h, int32_t n, double *trace) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (n < 0) return h->fail(DEBLUR_EINVAL, "n must be >= 0");
    if (!trace && n > 0) return h->fail(DEBLUR_EINVAL, "trace is NULL");
    for (int32_t k = 0; k < n; ++k) {
        double o[4];
        if ((s = deblur_objective(h, o)) != DEBLUR_OK) return s;
        trace[4 * k + 0] = o[0];
        trace[4 * k + 1] = o[1];
        trace[4 * k + 2] = o[2];
        trace[4 * k + 3] = o[3];
        if ((s = deblur_iterate(h, 1)) != DEBLUR_OK) return s;
    }
    return DEBLUR_OK;
}

deblur_status deblur_objective(deblur_t h, double out[4]) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (!out) return h->fail(DEBLUR_EINVAL, "out is NULL");
    const int F = (int)h->plan.facets.size();
    std::vector<double> data(F, 0.0), reg(F, 0.0);
    double md = 0.0;
    cudaEvent_t ev = nullptr;
    // data term at the current x (A22)
    if (h->conv_path == DEBLUR_CONV_FFT) {
        if ((s = run_fft_H(h, h->d_facets, h->par, FFT_OBJECTIVE)) != DEBLUR_OK) return s;
        CU(cudaStreamSynchronize(h->stream));
        std::vector<double> fd;
        CU(fft_partials_all(h, fd));
        for (size_t li = 0; li < h->local.size(); ++li) data[h->local[li]] = fd[li];
    } else {
        h->prof_begin(KC_H_OBJ, &ev);
        CU(launch_H_direct(h->conv_args(h->d_facets, false), H_OBJECTIVE, h->par, h->stream));
        h->prof_end(KC_H_OBJ, ev);
        CU(cudaMemcpyAsync(h->h_partials.data(), h->d_partials, sizeof(double) * h->tilesH.size(),
                           cudaMemcpyDeviceToHost, h->stream));
        CU(cudaStreamSynchronize(h->stream));
        for (size_t t = 0; t < h->tilesH.size(); ++t) data[h->local[h->tilesH[t].f]] += h->h_partials[t];
    }
    h->prof_begin(KC_TV, &ev);
    CU(launch_tv_value(h->d_facets, h->d_tilesHT, (int)h->tilesHT.size(), h->plan.P, h->par, h->sc, h->d_partials,
                       h->stream));
    h->prof_end(KC_TV, ev);
    CU(cudaMemcpyAsync(h->h_partials.data(), h->d_partials, sizeof(double) * h->tilesHT.size(), cudaMemcpyDeviceToHost,
                       h->stream));
    CU(cudaStreamSynchronize(h->stream));
    for (size_t t = 0; t < h->tilesHT.size(); ++t) reg[h->local[h->tilesHT[t].f]] += h->h_partials[t];
    if ((s = join_consensus(h)) != DEBLUR_OK) return s;
    if ((s = exchange(h, 1, h->stream)) != DEBLUR_OK) return s;
    h->prof_begin(KC_MAXDIFF, &ev);
    CU(launch_maxdiff(h->d_facets, h->d_rects, (int)h->rects.size(), h->par, h->d_partials, h->stream));
    h->prof_end(KC_MAXDIFF, ev);
    CU(cudaMemcpyAsync(h->h_partials.data(), h->d_partials, sizeof(double) * h->rects.size(), cudaMemcpyDeviceToHost,
                       h->stream));
    if ((s = finish(h)) != DEBLUR_OK) return s;
    for (size_t r = 0; r < h->rects.size(); ++r) md = std::max(md, h->h_partials[r]);
    if (h->world > 1) {
        // per-facet values are nonzero only on their owner: a sum all-reduce is exact
        double *d = h->d_objbuf;              // allocated once in deblur_create
        std::vector<double> buf(2 * F + 1);
        for (int f = 0; f < F; ++f) { buf[f] = data[f]; buf[F + f] = reg[f]; }
        buf[2 * F] = md;
        CU(cudaMemcpyAsync(d, buf.data(), sizeof(double) * (2 * F + 1), cudaMemcpyHostToDevice, h->stream));
        NC(ncclAllReduce(d, d, 2 * F, ncclDouble, ncclSum, h->comm, h->stream), "objective allreduce", -1);
        NC(ncclAllReduce(d + 2 * F, d + 2 * F, 1, ncclDouble, ncclMax, h->comm, h->stream), "objective allreduce", -1);
        CU(cudaMemcpyAsync(buf.data(), d, sizeof(double) * (2 * F + 1), cudaMemcpyDeviceToHost, h->stream));
        CU(cudaStreamSynchronize(h->stream));
        for (int f = 0; f < F; ++f) { data[f] = buf[f]; reg[f] = buf[F + f]; }
        md = buf[2 * F];
    }
    double dt = 0, rt = 0;
    for (int f = 0; f < F; ++f) {      // facet-id order
        if (!std::isfinite(data[f]) || !std::isfinite(reg[f])) {
            std::ostringstream o;
            o << "non-finite objective partial on facet " << f;
            return h->fail(DEBLUR_ENUMERIC, o.str());
        }
        dt += data[f];
        rt += (double)h->prm.lambda * reg[f];
    }
    out[0] = dt + rt; out[1] = dt; out[2] = rt; out[3] = md;
    return DEBLUR_OK;
}

}  // extern "C"

// gather facet-local rectangles to rank 0's host buffer.  For each local facet
// li, rect (local coords [y0,y1) x [x0,x1) of array `which`) goes to host dst at
// (gy0, gx0) with pitch dpitch.  `pick` selects the device array of a facet.
struct Piece { int facet; int64_t y0, y1, x0, x1; int64_t gy0, gx0; };
template <typename Pick>
static deblur_status gather_pieces(deblur_t h, const std::vector<Piece> &all, Pick pick, float *dst, int64_t dpitch) {
    // all: pieces of ALL facets (every rank computes the same list)
    for (const Piece &pc : all) {
        const int owner = h->plan.facets[pc.facet].owner;
        const int64_t w = pc.x1 - pc.x0, hh = pc.y1 - pc.y0;
        if (w <= 0 || hh <= 0) continue;
        if (owner == h->rank) {
            const FacetDev &F = h->fh[h->local_index[pc.facet]];
            int64_t pitch; const float *src = pick(F, pitch);
            if (h->rank == 0) {
                if (dst)
                    CU(cudaMemcpy2DAsync(dst + pc.gy0 * dpitch + pc.gx0, dpitch * 4, src + pc.y0 * pitch + pc.x0,
                                         pitch * 4, w * 4, hh, cudaMemcpyDeviceToHost, h->stream));
            } else {
                float *tmp = nullptr;
                CU(cudaMallocAsync((void **)&tmp, w * hh * 4, h->stream));
                CU(cudaMemcpy2DAsync(tmp, w * 4, src + pc.y0 * pitch + pc.x0, pitch * 4, w * 4, hh,
                                     cudaMemcpyDeviceToDevice, h->stream));
                NC(ncclSend(tmp, (size_t)(w * hh), ncclFloat, 0, h->comm, h->stream), "gather send", 0);
                CU(cudaFreeAsync(tmp, h->stream));
            }
        } else if (h->rank == 0) {
            float *tmp = nullptr;
            CU(cudaMallocAsync((void **)&tmp, w * hh * 4, h->stream));
            NC(ncclRecv(tmp, (size_t)(w * hh), ncclFloat, owner, h->comm, h->stream), "gather recv", owner);
            if (dst)
                CU(cudaMemcpy2DAsync(dst + pc.gy0 * dpitch + pc.gx0, dpitch * 4, tmp, w * 4, w * 4, hh,
                                     cudaMemcpyDeviceToHost, h->stream));
            CU(cudaFreeAsync(tmp, h->stream));
        }
    }
    return finish(h);
}

// owner-computes regions (§8b): observed core [b_k, b_{k+1}); estimate [b_k + c, b_{k+1} + c) with the ends extended
static void core_range(const Plan &pl, bool rows, int k, bool estimate, int64_t &lo, int64_t &hi) {
    const int64_t M = rows ? pl.my : pl.mx;
    const int F = rows ? pl.Fy : pl.Fx;
    const int64_t c = (pl.P - 1) / 2;
    lo = (int64_t)k * M / F; hi = (int64_t)(k + 1) * M / F;
    if (estimate) {
        lo = (k == 0) ? 0 : lo + c;
        hi = (k == F - 1) ? (rows ? pl.ny : pl.nx) : hi + c;
    }
}

static deblur_status apply_common(deblur_t h, bool adjoint, const float *in, bool in_dev, float *out, bool out_dev) {
    const Plan &pl = h->plan;
    if (adjoint && (pl.Fy > 1 || pl.Fx > 1) && pl.O < pl.P - 1)
        return h->fail(DEBLUR_EINVAL, "apply_HT with several facets needs overlap >= P - 1 (SURVEY §8b)");
    const cudaMemcpyKind kin = in_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (size_t li = 0; li < h->local.size(); ++li) {
        const FacetPlan &fp = pl.facets[h->local[li]];
        const FacetDev &F = h->fh[li];
        if (!adjoint)
            CU(cudaMemcpy2DAsync(F.g, F.ep * 4, in + fp.ey0 * pl.nx + fp.ex0, pl.nx * 4, F.nx * 4, F.ny, kin, h->stream));
        else
            CU(cudaMemcpy2DAsync(F.r, F.op * 4, in + fp.oy0 * pl.mx + fp.ox0, pl.mx * 4, F.mx * 4, F.my, kin, h->stream));
    }
    cudaEvent_t ev = nullptr;
    if (h->conv_path == DEBLUR_CONV_FFT) {
        if (!adjoint) {
            deblur_status st = run_fft_H(h, h->d_facets_alt, 0, FFT_PLAIN);
            if (st != DEBLUR_OK) return st;
        } else {
            deblur_status st = run_fft_HT(h, h->d_facets);
            if (st != DEBLUR_OK) return st;
        }
    } else if (!adjoint) {
        h->prof_begin(KC_H_PLAIN, &ev);
        CU(launch_H_direct(h->conv_args(h->d_facets_alt, false), H_PLAIN, 0, h->stream));
        h->prof_end(KC_H_PLAIN, ev);
    } else {
        h->prof_begin(KC_HT_PLAIN, &ev);
        CU(launch_HT_direct(h->conv_args(h->d_facets, true), HT_PLAIN, h->par, 0, h->sc, h->stream));
        h->prof_end(KC_HT_PLAIN, ev);
    }
    std::vector<Piece> pieces;
    for (const auto &fp : pl.facets) {
        int64_t y0, y1, x0, x1;
        core_range(pl, true, fp.fy, adjoint, y0, y1);
        core_range(pl, false, fp.fx, adjoint, x0, x1);
        const int64_t oy = adjoint ? fp.ey0 : fp.oy0, ox = adjoint ? fp.ex0 : fp.ox0;
        pieces.push_back({fp.id, y0 - oy, y1 - oy, x0 - ox, x1 - ox, y0, x0});
    }
    const int64_t dp = adjoint ? pl.nx : pl.mx;
    if (out_dev) {
        for (const Piece &pc : pieces) {
            const FacetDev &F = h->fh[h->local_index[pc.facet]];
            const float *src = adjoint ? F.g : F.r;
            const int64_t pitch = adjoint ? F.ep : F.op;
            CU(cudaMemcpy2DAsync(out + pc.gy0 * dp + pc.gx0, dp * 4, src + pc.y0 * pitch + pc.x0, pitch * 4,
                                 (pc.x1 - pc.x0) * 4, pc.y1 - pc.y0, cudaMemcpyDeviceToDevice, h->stream));
        }
        return finish(h);
    }
    return gather_pieces(
        h, pieces,
        [adjoint](const FacetDev &F, int64_t &pitch) -> const float * {
            pitch = adjoint ? F.ep : F.op;
            return adjoint ? F.g : F.r;
        },
        out, dp);
}

extern "C" {

deblur_status deblur_apply_H(deblur_t h, const float *x, float *hx) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (!x) return h->fail(DEBLUR_EINVAL, "x is NULL");
    if (h->rank == 0 && !hx) return h->fail(DEBLUR_EINVAL, "hx is NULL on rank 0");
    return apply_common(h, false, x, false, hx, false);
}

deblur_status deblur_apply_HT(deblur_t h, const float *r, float *g) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (!r) return h->fail(DEBLUR_EINVAL, "r is NULL");
    if (h->rank == 0 && !g) return h->fail(DEBLUR_EINVAL, "g is NULL on rank 0");
    return apply_common(h, true, r, false, g, false);
}

deblur_status deblur_apply_H_device(deblur_t h, const float *d_x, float *d_hx) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (h->world != 1) return h->fail(DEBLUR_ESTATE, "device apply needs world == 1");
    if (!d_x || !d_hx) return h->fail(DEBLUR_EINVAL, "NULL device pointer");
    return apply_common(h, false, d_x, true, d_hx, true);
}

deblur_status deblur_apply_HT_device(deblur_t h, const float *d_r, float *d_g) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (h->world != 1) return h->fail(DEBLUR_ESTATE, "device apply needs world == 1");
    if (!d_r || !d_g) return h->fail(DEBLUR_EINVAL, "NULL device pointer");
    return apply_common(h, true, d_r, true, d_g, true);
}

deblur_status deblur_state_size(deblur_t h, int64_t *n) {
    if (!h || !n) return DEBLUR_EINVAL;
    int64_t t = 0;
    for (const auto &f : h->plan.facets) t += (f.ey1 - f.ey0) * (f.ex1 - f.ex0);
    *n = t;
    return DEBLUR_OK;
}

static std::vector<int64_t> facet_offsets(const Plan &pl) {
    std::vector<int64_t> off(pl.facets.size() + 1, 0);
    for (size_t i = 0; i < pl.facets.size(); ++i)
        off[i + 1] = off[i] + (pl.facets[i].ey1 - pl.facets[i].ey0) * (pl.facets[i].ex1 - pl.facets[i].ex0);
    return off;
}

deblur_status deblur_get_state(deblur_t h, float *xf, float *uf) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    const Plan &pl = h->plan;
    auto off = facet_offsets(pl);
    for (int which = 0; which < 2; ++which) {
        float *dst = which == 0 ? xf : uf;
        if (h->rank == 0 && !dst) return h->fail(DEBLUR_EINVAL, "NULL output on rank 0");
        // each facet is its own "image" with pitch = its width: use per-facet pieces
        for (const auto &fp : pl.facets) {
            const int64_t w = fp.ex1 - fp.ex0, hh = fp.ey1 - fp.ey0;
            std::vector<Piece> one{{fp.id, 0, hh, 0, w, 0, 0}};
            const int par = h->par;
            s = gather_pieces(
                h, one,
                [which, par](const FacetDev &F, int64_t &pitch) -> const float * {
                    pitch = F.ep;
                    return which == 0 ? F.x[par] : F.u;
                },
                dst ? dst + off[fp.id] : nullptr, w);
            if (s != DEBLUR_OK) return s;
        }
    }
    return DEBLUR_OK;
}

deblur_status deblur_set_state(deblur_t h, const float *xf, const float *uf) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (!xf || !uf) return h->fail(DEBLUR_EINVAL, "NULL state array");
    auto off = facet_offsets(h->plan);
    for (size_t li = 0; li < h->local.size(); ++li) {
        const FacetDev &F = h->fh[li];
        const int64_t o = off[F.id];
        CU(cudaMemcpy2DAsync(F.x[h->par], F.ep * 4, xf + o, F.nx * 4, F.nx * 4, F.ny, cudaMemcpyHostToDevice, h->stream));
        CU(cudaMemcpy2DAsync(F.u, F.ep * 4, uf + o, F.nx * 4, F.nx * 4, F.ny, cudaMemcpyHostToDevice, h->stream));
    }
    return finish(h);
}

deblur_status deblur_get_image(deblur_t h, float *x) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    const Plan &pl = h->plan;
    if (h->rank == 0 && !x) return h->fail(DEBLUR_EINVAL, "x is NULL on rank 0");
    if (h->world == 1) {       // blend on the device in facet order, one D2H copy
        if (!h->d_image) CU(h->dalloc(&h->d_image, (size_t)pl.ny * pl.nx));
        float *img = h->d_image;
        CU(cudaMemsetAsync(img, 0, (size_t)pl.ny * pl.nx * 4, h->stream));
        float *wsum = nullptr;
        if (h->per_node) {      // per-node weights need not sum to 1 on every facet union
            if (!h->d_wsum) CU(h->dalloc(&h->d_wsum, (size_t)pl.ny * pl.nx));
            wsum = h->d_wsum;
            CU(cudaMemsetAsync(wsum, 0, (size_t)pl.ny * pl.nx * 4, h->stream));
        }
        for (size_t li = 0; li < h->local.size(); ++li) CU(launch_blend(h->fh[li], h->par, img, wsum, pl.nx, h->stream));
        if (wsum) CU(launch_normalize(img, wsum, (int64_t)pl.ny * pl.nx, h->stream));
        CU(cudaMemcpyAsync(x, img, (size_t)pl.ny * pl.nx * 4, cudaMemcpyDeviceToHost, h->stream));
        return finish(h);
    }
    // gather every facet's x to rank 0, then x_hat = sum_f omega^F_f x_f in facet order (A7)
    int64_t n = 0;
    deblur_state_size(h, &n);
    std::vector<float> xs(h->rank == 0 ? (size_t)n : 0);
    auto off = facet_offsets(pl);
    for (const auto &fp : pl.facets) {
        const int64_t w = fp.ex1 - fp.ex0, hh = fp.ey1 - fp.ey0;
        std::vector<Piece> one{{fp.id, 0, hh, 0, w, 0, 0}};
        const int par = h->par;
        s = gather_pieces(
            h, one,
            [par](const FacetDev &F, int64_t &pitch) -> const float * {
                pitch = F.ep;
                return F.x[par];
            },
            h->rank == 0 ? xs.data() + off[fp.id] : nullptr, w);
        if (s != DEBLUR_OK) return s;
    }
    if (h->rank != 0) return DEBLUR_OK;
    std::fill(x, x + pl.ny * pl.nx, 0.f);
    std::vector<float> wsum(h->per_node ? (size_t)pl.ny * pl.nx : 0, 0.f);
    for (const auto &fp : pl.facets) {
        // host copies of the device AxisW (per-node: host weight rows)
        const AxisW ay = {(int)fp.ey0, (int)(fp.ey1 - fp.ey0), (int)(fp.py_e - fp.ey0), (int)(fp.ny_s - fp.ey0),
                          (int)fp.ey0, (int)fp.py_e, (int)fp.ny_s, (int)fp.ey1,
                          h->per_node ? h->h_wy.data() + (size_t)fp.fy * pl.ny : nullptr};
        const AxisW ax = {(int)fp.ex0, (int)(fp.ex1 - fp.ex0), (int)(fp.px_e - fp.ex0), (int)(fp.nx_s - fp.ex0),
                          (int)fp.ex0, (int)fp.px_e, (int)fp.nx_s, (int)fp.ex1,
                          h->per_node ? h->h_wx.data() + (size_t)fp.fx * pl.nx : nullptr};
        const int64_t w = fp.ex1 - fp.ex0;
        for (int64_t r = 0; r < fp.ey1 - fp.ey0; ++r) {
            const float oy = omega_axis(ay, (int)r);
            for (int64_t q = 0; q < w; ++q) {
                const float om = oy * omega_axis(ax, (int)q);
                const int64_t o = (fp.ey0 + r) * pl.nx + fp.ex0 + q;
                x[o] += om * xs[off[fp.id] + r * w + q];
                if (h->per_node) wsum[o] += om;
            }
        }
    }
    if (h->per_node)
        for (size_t i = 0; i < wsum.size(); ++i) x[i] /= wsum[i];
    return DEBLUR_OK;
}

deblur_status deblur_reset(deblur_t h, const float *y, const float *x0) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (!y) return h->fail(DEBLUR_EINVAL, "y is NULL");
    if ((s = stage_y(h, y)) != DEBLUR_OK) return s;
    if ((s = upload_y(h)) != DEBLUR_OK) return s;
    h->vm.k_outer = 0;                                // a fresh solve: VMLM-B budget schedule restarts
    return upload_state_x0(h, x0);
}

// ---------------------------------------------------------------- pipelined jobs
deblur_status deblur_stage_y(deblur_t h, const float *y) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (!y) return h->fail(DEBLUR_EINVAL, "y is NULL");
    const Plan &pl = h->plan;
    if (!h->d_ystage2) CU(h->dalloc(&h->d_ystage2, (size_t)pl.my * pl.mx));
    int64_t y0, y1, x0, x1;
    ystage_box(h, y0, y1, x0, x1);
    // the buffer may still feed the previous reset_staged's device copies
    CU(cudaStreamWaitEvent(h->up_stream, h->ev_yfree, 0));
    if (y1 > y0 && x1 > x0)
        CU(cudaMemcpy2DAsync(h->d_ystage2, std::max<int64_t>(1, x1 - x0) * 4, y + y0 * pl.mx + x0, pl.mx * 4,
                             (x1 - x0) * 4, y1 - y0, cudaMemcpyHostToDevice, h->up_stream));
    CU(cudaEventRecord(h->ev_staged, h->up_stream));
    h->staged = true;
    return DEBLUR_OK;
}

deblur_status deblur_reset_staged(deblur_t h, const float *x0) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (!h->staged) return h->fail(DEBLUR_ESTATE, "no observation staged (deblur_stage_y)");
    int64_t y0, y1, xa, x1;
    ystage_box(h, y0, y1, xa, x1);
    CU(cudaStreamWaitEvent(h->stream, h->ev_staged, 0));
    if (!h->d_ystage) CU(h->dalloc(&h->d_ystage, (size_t)h->plan.my * h->plan.mx));
    std::swap(h->d_ystage, h->d_ystage2);
    h->ys_y0 = y0; h->ys_x0 = xa; h->ys_pitch = std::max<int64_t>(1, x1 - xa);
    h->staged = false;
    if ((s = upload_y(h)) != DEBLUR_OK) return s;
    h->vm.k_outer = 0;
    if ((s = upload_state_x0(h, x0, false)) != DEBLUR_OK) return s;
    CU(cudaEventRecord(h->ev_yfree, h->stream));       // the other buffer may be refilled after this
    return DEBLUR_OK;
}

deblur_status deblur_get_image_async(deblur_t h, float *x) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    if (h->world != 1) return h->fail(DEBLUR_ESTATE, "get_image_async needs world == 1 (use deblur_get_image)");
    if (!x) return h->fail(DEBLUR_EINVAL, "x is NULL");
    const Plan &pl = h->plan;
    const int b = h->img_slot;
    h->img_slot ^= 1;
    if (!h->d_image2[b]) CU(h->dalloc(&h->d_image2[b], (size_t)pl.ny * pl.nx));
    float *img = h->d_image2[b];
    CU(cudaStreamWaitEvent(h->stream, h->ev_down[b], 0));   // its previous download is done
    CU(cudaMemsetAsync(img, 0, (size_t)pl.ny * pl.nx * 4, h->stream));
    float *wsum = nullptr;
    if (h->per_node) {
        if (!h->d_wsum) CU(h->dalloc(&h->d_wsum, (size_t)pl.ny * pl.nx));
        wsum = h->d_wsum;
        CU(cudaMemsetAsync(wsum, 0, (size_t)pl.ny * pl.nx * 4, h->stream));
    }
    for (size_t li = 0; li < h->local.size(); ++li) CU(launch_blend(h->fh[li], h->par, img, wsum, pl.nx, h->stream));
    if (wsum) CU(launch_normalize(img, wsum, (int64_t)pl.ny * pl.nx, h->stream));
    CU(cudaEventRecord(h->ev_blend, h->stream));
    CU(cudaStreamWaitEvent(h->down_stream, h->ev_blend, 0));
    CU(cudaMemcpyAsync(x, img, (size_t)pl.ny * pl.nx * 4, cudaMemcpyDeviceToHost, h->down_stream));
    CU(cudaEventRecord(h->ev_down[b], h->down_stream));
    return DEBLUR_OK;
}

deblur_status deblur_sync(deblur_t h) {
    deblur_status s = check_state(h);
    if (s != DEBLUR_OK) return s;
    CU(cudaStreamSynchronize(h->up_stream));
    CU(cudaStreamSynchronize(h->down_stream));
    return finish(h);
}

deblur_status deblur_get_outer_iteration(deblur_t h, int32_t *k) {
    if (!h || !k) return DEBLUR_EINVAL;
    *k = h->vm.k_outer;
    return DEBLUR_OK;
}

deblur_status deblur_set_outer_iteration(deblur_t h, int32_t k) {
    if (!h) return DEBLUR_EINVAL;
    if (k < 0) return h->fail(DEBLUR_EINVAL, "outer iteration must be >= 0");
    h->vm.k_outer = k;
    return DEBLUR_OK;
}

deblur_status deblur_get_step(deblur_t h, double *tau) {
    if (!h || !tau) return DEBLUR_EINVAL;
    *tau = h->tau;
    return DEBLUR_OK;
}

deblur_status deblur_get_stream(deblur_t h, void **stream) {
    if (!h || !stream) return DEBLUR_EINVAL;
    *stream = (void *)h->stream;
    return DEBLUR_OK;
}

deblur_status deblur_get_conv_path(deblur_t h, int32_t *path) {
    if (!h || !path) return DEBLUR_EINVAL;
    *path = h->conv_path;
    return DEBLUR_OK;
}

deblur_status deblur_set_profiling(deblur_t h, int32_t enable) {
    if (!h) return DEBLUR_EINVAL;
    h->prof = enable != 0;
    return DEBLUR_OK;
}

deblur_status deblur_kernel_stats(deblur_t h, int32_t *n_classes, int64_t *launches, double *ms) {
    if (!h || !n_classes) return DEBLUR_EINVAL;
    const int n = std::min<int>(*n_classes, KC_COUNT);
    for (int i = 0; i < n; ++i) {
        if (launches) launches[i] = h->stat_n[i];
        if (ms) ms[i] = h->stat_ms[i];
    }
    *n_classes = KC_COUNT;
    return DEBLUR_OK;
}

deblur_status deblur_kernel_work(deblur_t h, int32_t cls, double *flops, double *bytes) {
    if (!h || !flops || !bytes || cls < 0 || cls >= KC_COUNT) return DEBLUR_EINVAL;
    *flops = 0.0;
    *bytes = 0.0;
    const Plan &pl = h->plan;
    const double P2 = (double)pl.P * pl.P;
    // a(pixel) = #{k : omega_k(pixel) != 0} = nzy(row) * nzx(col) (separable hats)
    auto nz_sum = [&](const std::vector<float> &w, int G, int64_t n, int64_t a, int64_t b) {
        double t = 0;
        for (int64_t i = a; i < b; ++i) {
            int c = 0;
            for (int g = 0; g < G; ++g) c += w[(size_t)g * n + i] != 0.f;
            t += c;
        }
        return t;
    };
    const int c = (pl.P - 1) / 2;
    double est_px = 0, obs_px = 0;
    for (int id : h->local) {
        const FacetPlan &f = pl.facets[id];
        est_px += (double)(f.ey1 - f.ey0) * (f.ex1 - f.ex0);
        obs_px += (double)(f.oy1 - f.oy0) * (f.ox1 - f.ox0);
        if (h->per_node) {     // one PSF per pixel: a = 1
            if (cls == KC_H || cls == KC_H_OBJ || cls == KC_H_PLAIN)
                *flops += 2.0 * P2 * (double)(f.oy1 - f.oy0) * (f.ox1 - f.ox0);
            if (cls == KC_HT_UPDATE || cls == KC_HT_PLAIN)
                *flops += 2.0 * P2 * (double)(f.ey1 - f.ey0) * (f.ex1 - f.ex0);
            continue;
        }
        if (cls == KC_H || cls == KC_H_OBJ || cls == KC_H_PLAIN)
            *flops += 2.0 * P2 * nz_sum(h->h_wy, h->prm.psf_gy, pl.ny, f.oy0 + c, f.oy1 + c) *
                      nz_sum(h->h_wx, h->prm.psf_gx, pl.nx, f.ox0 + c, f.ox1 + c);
        if (cls == KC_HT_UPDATE || cls == KC_HT_PLAIN)
            *flops += 2.0 * P2 * nz_sum(h->h_wy, h->prm.psf_gy, pl.ny, f.ey0, f.ey1) *
                      nz_sum(h->h_wx, h->prm.psf_gx, pl.nx, f.ex0, f.ex1);
    }
    if (cls >= KC_FFT_H0 && cls <= KC_FFT_HT2 && h->fft) {
        *bytes = fft_pass_bytes(*h->fft, cls >= KC_FFT_HT0, (cls - KC_FFT_H0) % 3);
        *flops = fft_pass_flops(*h->fft, cls >= KC_FFT_HT0, (cls - KC_FFT_H0) % 3);
    }
    if (cls >= KC_FFT2_H0 && cls <= KC_FFT2_HT2 && h->fft2) {
        *bytes = fft_pass_bytes(*h->fft2, cls >= KC_FFT2_HT0, (cls - KC_FFT2_H0) % 3);
        *flops = fft_pass_flops(*h->fft2, cls >= KC_FFT2_HT0, (cls - KC_FFT2_H0) % 3);
    }
    if (cls == KC_UPDATE_G) *bytes = 20.0 * est_px;            // g, u, x in; x+, u|v out
    if (cls == KC_HT_UPDATE) *bytes = 24.0 * est_px;           // r (~obs), x, u in; x+, u|v out
    if (cls == KC_H) *bytes = 4.0 * est_px + 12.0 * obs_px;    // x, y, W in; r out
    if (cls == KC_CONSENSUS) {
        double b = 0;
        for (const BandRect &r : h->rects) {
            const FacetDev &F = h->fh[r.f];
            for (int yy = r.y0; yy < r.y1; ++yy) {
                const int cy = 1 + (yy < F.ay.b_prev || yy >= F.ay.b_next);
                for (int xx = r.x0; xx < r.x1; ++xx) {
                    const int cx = 1 + (xx < F.ax.b_prev || xx >= F.ax.b_next);
                    b += 4.0 * cy * cx + 12.0;                     // v of each contributor; x+ in, u in/out
                }
            }
        }
        *bytes = b;
    }
    return DEBLUR_OK;
}

deblur_status deblur_reset_stats(deblur_t h) {
    if (!h) return DEBLUR_EINVAL;
    for (int i = 0; i < KC_COUNT; ++i) { h->stat_n[i] = 0; h->stat_ms[i] = 0; }
    return DEBLUR_OK;
}

}  // extern "C"
