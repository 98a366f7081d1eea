// Host builders for the device evaluation tables (per band L) and the seed grid.
#pragma once

#include <complex>
#include <vector>

#include "basis_host.hpp"
#include "kernels.cuh"

namespace bmb {

struct BandTablesHost {
    int L = 0;
    int n_items = 0, n_groups = 0, rows = 0;
    std::vector<int> row_off;
    std::vector<char2> item_mm;
    std::vector<int> item_len;
    std::vector<float> bfac;
    std::vector<int> bexp;
    std::vector<float> P, Q, R;
    std::vector<int16_t> item_of;
};
BandTablesHost build_band_tables(int L);

// wedge-power kernel entries in the band layout:
// W_l[m,m'] = conj(chi_hat_lm) q_hat_lm' / total  (src/xcorr.cpp:344-355)
std::vector<float2> wedge_band_entries(const BandTablesHost& t,
                                       const std::vector<std::complex<double>>& chi_hat,
                                       const std::vector<std::complex<double>>& q_hat,
                                       double total);

// little-d^l_{m,m'}(beta) for all l <= L (reference recursion, FP64), packed
// (2l+1)^2 row-major blocks l = 0..L.
std::vector<double> little_d_full(int L, double beta);

}  // namespace bmb
