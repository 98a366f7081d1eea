// Missing-wedge filter and power kernel (see wedge.cu).
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <complex>
#include <map>
#include <utility>
#include <vector>

#include "basis_host.hpp"
#include "context.hpp"

namespace bmb {

constexpr double kPiH = 3.14159265358979323846;
constexpr double kWedgeTaperDeg = 6.0;  // xcorr.hpp:114

double keep_profile(double theta_deg, double nx, double ny, double nz, double taper_deg);

// Tapered (or binary, taper 0) wedge filter for batches of n^3 float volumes.
struct WedgeFilter {
    int n;
    double theta_deg, taper_deg;
    DevBuf profile;    // n*n*(n/2+1) keep profile / n^3 (float)
    DevBuf profile_d;  // same, double
    DevBuf spec;
    std::map<int, std::pair<cufftHandle, cufftHandle>> plans;
    WedgeFilter(int n, double theta_deg, double taper_deg);
    ~WedgeFilter();
    void apply(const float* in, float* out, int count, cudaStream_t s);
};

void apply_wedge_d(const double* in, double* out, int n, const double* profile_d, cudaStream_t s);

struct WedgePowerFactors {
    std::vector<std::complex<double>> chi_hat, q_hat;  // packed (l, m >= 0)
    double total = 0.0;
};
WedgePowerFactors wedge_power_factors(const float* tmpl_dev, int n, int l_max, double theta_deg,
                                      double taper_deg, cudaStream_t s);

}  // namespace bmb
