// Device vs host check of the register-only 3x3 FullPivLU (rotation.cuh).
#include <cstdio>
#include <random>
#include <cmath>
#include "rotation.cuh"
using namespace bmb;
__global__ void k(const double* m, const double* b, double* x, int* inv, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    LU3 lu; lu.factor(m + 9 * i);
    inv[i] = lu.invertible();
    double xx[3] = {0, 0, 0};
    if (inv[i]) lu.solve(b + 3 * i, xx);
    for (int j = 0; j < 3; ++j) x[3 * i + j] = xx[j];
}
int main() {
    const int n = 4096;
    std::mt19937 rng(3); std::normal_distribution<double> N(0, 1);
    std::vector<double> m(9 * n), b(3 * n), x(3 * n), xh(3 * n);
    std::vector<int> inv(n);
    for (int i = 0; i < n; ++i) { for (int j = 0; j < 9; ++j) m[9*i+j] = N(rng); for (int j=0;j<3;++j) b[3*i+j]=N(rng); }
    double *dm, *db, *dx; int* di;
    cudaMalloc(&dm, 8*m.size()); cudaMalloc(&db, 8*b.size()); cudaMalloc(&dx, 8*x.size()); cudaMalloc(&di, 4*n);
    cudaMemcpy(dm, m.data(), 8*m.size(), cudaMemcpyHostToDevice); cudaMemcpy(db, b.data(), 8*b.size(), cudaMemcpyHostToDevice);
    k<<<(n+127)/128,128>>>(dm, db, dx, di, n);
    cudaMemcpy(x.data(), dx, 8*x.size(), cudaMemcpyDeviceToHost); cudaMemcpy(inv.data(), di, 4*n, cudaMemcpyDeviceToHost);
    double worst = 0; int bad_inv = 0;
    for (int i = 0; i < n; ++i) {
        LU3 lu; lu.factor(&m[9*i]); double h[3] = {0,0,0};
        if (lu.invertible() != (bool)inv[i]) ++bad_inv;
        if (lu.invertible()) lu.solve(&b[3*i], h);
        double d = 0;
        for (int j = 0; j < 3; ++j) d = std::max(d, std::fabs(h[j] - x[3*i+j]) / (1 + std::fabs(h[j])));
        if (d > 1e-9 && d > worst) {
            printf("case %d: m=", i); for (int j=0;j<9;++j) printf("%.3f ", m[9*i+j]);
            printf("\n host x = %.6f %.6f %.6f  dev x = %.6f %.6f %.6f\n", h[0],h[1],h[2], x[3*i],x[3*i+1],x[3*i+2]);
        }
        worst = std::max(worst, d);
    }
    printf("device vs host LU: worst rel diff %g, invertibility mismatches %d\n", worst, bad_inv);
    return worst > 1e-9 || bad_inv;
}
