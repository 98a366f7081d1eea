// Host-side (FP64) basis setup of the B200 path: built once per context, then
// resident in HBM.  Mirrors BasisSpec / ExpandPlan of the reference
// (include/ballmatch/basis.hpp:31-58, src/basis.cpp:88-115, 174-219) and adds
// the pulled-back expansion operator E = R.Theta.Phi.T.
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace bmb {
namespace host {

constexpr double kPi = 3.14159265358979323846;

// spherical Bessel j_l (upward recurrence above l, Miller downward below)
double sph_jl(int l, double x);
// Bessel root table: rows[l] = roots of j_l up to lambda_cut (src/detail/bessel.cpp:150-178)
std::vector<std::vector<double>> bessel_roots(int l_max, double lambda_cut);
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w);
// fully normalized Condon-Shortley Pbar_l^m(u), packed (l,m>=0) triangle
void legendre(int l_max, double u, double* out);
inline size_t tri(int l, int m) { return (size_t)l * (l + 1) / 2 + m; }
inline size_t tri_count(int l_max) { return (size_t)(l_max + 1) * (l_max + 2) / 2; }
double default_lambda_cut(int n, int l_max);

// Basis index set + quadrature plan.
struct Basis {
    int l_max = 0;
    double lambda_cut = 0;
    std::vector<std::vector<double>> roots, norms;  // [l][k-1]
    std::vector<int> block_off;                     // real-packed row offset per degree
    int coeffs = 0;                                 // C = sum_l k_l (2l+1) real rows
    int n_r = 0, n_theta = 0, n_phi = 0;
    std::vector<double> r, wr, u, wu;               // radial / polar GL nodes & weights
    int radial_count(int l) const { return (int)roots[l].size(); }
    // real-packed row of (l, k, m>=0, part): part 0 = Re, 1 = Im (m > 0 only)
    int row(int l, int k, int m, int part) const {
        return block_off[l] + (k - 1) * (2 * l + 1) + (m == 0 ? 0 : 2 * m - 1 + part);
    }
};
Basis make_basis(int l_max, double lambda_cut);

// Dense pulled-back operator on the support voxels of an n^3 grid, stored as
// the FP16 three-pass split: E[r][v] ~= row_scale[r] * (hi[r][v] + lo[r][v]),
// row_scale a power of two with |E[r][:]| / row_scale <= 1, hi = RNE half,
// lo = RNE half of the residual (FP16 subnormals kept).  Padded to
// m_pad x k_pad (multiples of 128 rows / 64 voxels) with zeros.
struct Operator {
    int n = 0;
    int rows = 0;                  // C
    int support = 0;               // V
    int m_pad = 0, k_pad = 0;
    std::vector<int32_t> voxels;   // raster index (z*n+y)*n+x of each support voxel, ascending
    std::vector<float> row_scale;  // m_pad
    std::vector<uint16_t> hi, lo;  // m_pad x k_pad, __half bit patterns
};
Operator build_operator(const Basis& b, int n);

// Separable factors of expand() stages 2-4 (src/basis.cpp:254-328), FP64:
//   radial[(pair_off[l] + k-1) * n_r + i] = c_lk j_l(lambda_lk r_i) r_i^2 w_i 2pi/n_phi
//   ptab[tri(l,m) * n_theta + t]        = Pbar_l^m(u_t) w_t
//   cs/sn[m * n_phi + p]                 = cos / -sin(2 pi (m p mod n_phi) / n_phi)
struct FactorTables {
    std::vector<double> radial, ptab, cs, sn;
    std::vector<int> pair_off;  // [l_max + 1]
    int pairs = 0;
};
FactorTables build_factor_tables(const Basis& b);
// voxels whose trilinear footprint reaches a quadrature sample (the support V)
int support_count(const Basis& b, int n);
uint16_t half_bits(double x);      // round-to-nearest-even, subnormals kept
double half_value(uint16_t h);

}  // namespace host
}  // namespace bmb
