// k_fft.cu -- FFT overlap-save path (placeholder until the hand-written path lands).
#include "fft.hpp"

namespace deblur {

struct FftPlan {};

bool fft_prefer(int) { return false; }

FftPlan *fft_create(const Plan &, const std::vector<int> &, const std::vector<FacetDev> &, const float *,
                    const float *, const float *, int, int, const float *, const float *, cudaStream_t,
                    std::string &err) {
    err = "FFT path not built yet";
    return nullptr;
}

void fft_destroy(FftPlan *f) { delete f; }
cudaError_t fft_H(FftPlan &, const FacetDev *, int, int, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fft_HT(FftPlan &, const FacetDev *, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fft_data_partials(FftPlan &, std::vector<double> &) { return cudaErrorNotSupported; }

}  // namespace deblur
