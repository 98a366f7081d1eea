#include <cstdio>
#include "rotation.cuh"
using namespace bmb;
__global__ void k(const double* m, double* out) {
    LU3 lu; lu.factor(m);
    for (int i = 0; i < 9; ++i) out[i] = lu.a[i];
    for (int i = 0; i < 3; ++i) { out[9 + i] = lu.rp[i]; out[12 + i] = lu.cp[i]; }
    out[15] = lu.nz; out[16] = lu.maxpiv;
}
int main() {
    double m[9] = {-0.473, 0.104, 0.229, -0.481, -0.659, 1.075, 1.724, -1.577, -0.386};
    double *dm, *dout, out[17];
    cudaMalloc(&dm, 72); cudaMalloc(&dout, 17 * 8);
    cudaMemcpy(dm, m, 72, cudaMemcpyHostToDevice);
    k<<<1, 1>>>(dm, dout);
    cudaMemcpy(out, dout, 17 * 8, cudaMemcpyDeviceToHost);
    LU3 h; h.factor(m);
    printf("dev : "); for (int i = 0; i < 17; ++i) printf("%.4f ", out[i]); printf("\n");
    printf("host: "); for (int i = 0; i < 9; ++i) printf("%.4f ", h.a[i]);
    for (int i = 0; i < 3; ++i) printf("%d ", h.rp[i]); for (int i = 0; i < 3; ++i) printf("%d ", h.cp[i]);
    printf("%d %.4f\n", h.nz, h.maxpiv);
}
