// fft.hpp -- hand-written FFT overlap-save path for H / H^T (internal).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "device.cuh"
#include "plan.hpp"

namespace deblur {

enum FftMode { FFT_RESIDUAL = 0, FFT_PLAIN = 1, FFT_OBJECTIVE = 2 };

struct FftPlan;

// Measured crossover: true when the FFT path beats the direct stencil for P.
bool fft_prefer(int P);
// A facet-local rectangle [y0, y1) x [x0, x1) of outputs a plan covers (observed
// coordinates for H, estimate coordinates for H^T); tiles start at (y0, x0) and step
// by T.  Empty lists mean the whole facet.
struct FftRect {
    int y0, y1, x0, x1;
};
struct FftRegions {
    std::vector<std::vector<FftRect>> H, HT;   // per local facet
};
// FFT size for P (the plan's S) and its valid extent T = S - P + 1.
int fft_choose_size(int P);

// d_wy/d_wx: the weights applied inside H_f (all ones in per-node mode, where every
// tile of facet (a, b) uses PSF (a, b) only); h_wy/h_wx: the interpolation weights.
FftPlan *fft_create(const Plan &pl, const std::vector<int> &local, const std::vector<FacetDev> &fh,
                    const float *d_psfs, const float *d_wy, const float *d_wx, int Gy, int Gx, const float *h_wy,
                    const float *h_wx, bool per_node, cudaStream_t s, std::string &err, int S_force = 0,
                    const FftRegions *regions = nullptr);
void fft_destroy(FftPlan *f);
// H / H^T on every local facet, one pass at a time (0 rows forward, 1 columns, 2 rows
// inverse): H mode RESIDUAL writes r = w (Hx - y) and data partials, PLAIN r = Hx,
// OBJECTIVE only the partials; H^T writes g = H^T r into FacetDev::g
cudaError_t fft_H_pass(FftPlan &f, int pass, const FacetDev *d_facets, int par, int mode, cudaStream_t s);
cudaError_t fft_HT_pass(FftPlan &f, int pass, const FacetDev *d_facets, cudaStream_t s);
// algorithmic HBM bytes moved by one launch of a pass: the pass's
// compulsory reads/writes of x / r / y / W and of the inter-pass spectra.  The PSF
// spectra are not counted: each Hhat_k (S x (S/2+1) complex, 1.1 MB at S = 512) is shared
// by the tiles of its PSF cell and re-read per tile; at c4 the 256 spectra (277 MB) do
// not fit the 126 MB L2, so part of the re-reads reach DRAM (ncu: profiles/).
double fft_pass_bytes(const FftPlan &f, bool ht, int pass);
// algorithmic flops of one launch of a pass in the FFT convention:
// 5 L log2 L per complex length-L DFT, 2.5 L log2 L per real one (R2C / C2R), 6 per
// complex product, 2 per complex add, 1 per real weight multiply / add.
double fft_pass_flops(const FftPlan &f, bool ht, int pass);
int fft_tiles(const FftPlan &f, bool ht);      // tiles of the H (ht = false) or H^T tile list

// per-local-facet data partial sums of the last H pass 2 (after a stream sync).
cudaError_t fft_data_partials(FftPlan &f, std::vector<double> &out);

}  // namespace deblur
