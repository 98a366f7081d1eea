// Host builders for the device evaluation tables (per band L) and the seed grid.
#pragma once

#include <complex>
#include <vector>

#include "basis_host.hpp"
#include "kernels.cuh"

namespace bmb {

// Recursion items (m, m') with m >= |m'| (the (m,m') <-> (m',m) and
// (m,m') <-> (-m',-m) symmetries of d^l): one chain serves the half-plane entry
// A = (m, m') and its partner B = (m', m) (sign (-1)^(m-m')) or (-m', -m) (sign +1);
// items with m' = +-m are their own partner (B weight 0).  Kernel entries per
// (row, lane) are float4 (A.re, A.im, B.re, B.im).
struct BandTablesHost {
    int L = 0;
    int n_items = 0, n_groups = 0, rows = 0;
    std::vector<int> row_off;
    std::vector<char2> item_mm;   // (m, m')
    std::vector<char2> item_pm;   // partner (pa, pb) in the half plane
    std::vector<float2> item_w;   // (weight of A, sign * weight of B)
    std::vector<int> item_len;
    std::vector<float> bfac;
    std::vector<int> bexp;
    std::vector<float> P, Q, R;
    std::vector<int> item_of;     // [(m+L)(2L+1) + m'+L]: 2 item + slot of half-plane entries, else -1
    std::vector<int2> at_desc;    // [rows*32] per layout position: x = valid | hasB << 1 | l << 2 | (mA+64) << 8 | (m'A+64) << 16,
                                  //                               y = (mB+64) | (m'B+64) << 8
    std::vector<int> out_pos;     // [(m+L)(2L+1) + m'+L]: 2 ((row_off[g] - m_item) 32 + lane) + slot; +64 l gives 2 at + slot
};
BandTablesHost build_band_tables(int L);

// wedge-power kernel entries in the band layout:
// W_l[m,m'] = conj(chi_hat_lm) q_hat_lm' / total  (src/xcorr.cpp:344-355)
std::vector<float4> wedge_band_entries(const BandTablesHost& t,
                                       const std::vector<std::complex<double>>& chi_hat,
                                       const std::vector<std::complex<double>>& q_hat,
                                       double total);

// little-d^l_{m,m'}(beta) for all l <= L (reference recursion, FP64), packed
// (2l+1)^2 row-major blocks l = 0..L.
std::vector<double> little_d_full(int L, double beta);

// Side kernels of the anchored-candidate evaluation (refine.cu chart_transform):
// xi' = xi D(b)^T with b = K^-1 is xi_coefficients(f, D(b) t), so the side
// kernels only need the rotated template (rotate_expansion, src/steer.cpp:208-223)
// and, for the wedge-power kernel conj(chi) q^T / total, the rotated q.
// Wigner D^l_{m,m'}(b) = e^{-i m a} d^l_{m,m'}(beta) e^{-i m' g} (steer.cpp:158-178),
// packed (2l+1)^2 row-major blocks l = 0..L.
std::vector<std::complex<double>> wigner_D_blocks(int L, double alpha, double beta, double gamma);
// f' = D f per (l, k) row of a real-packed FP32 coefficient set (real-volume
// symmetric in and out), FP64 arithmetic
std::vector<float> rotate_real_packed(const std::vector<float>& f, const host::Basis& b,
                                      const std::vector<std::complex<double>>& D);
// q'_l = D^l q_l for packed m >= 0 factors (tri(l, m)) of a real function
std::vector<std::complex<double>> rotate_tri(const std::vector<std::complex<double>>& q, int L,
                                             const std::vector<std::complex<double>>& D);

}  // namespace bmb
