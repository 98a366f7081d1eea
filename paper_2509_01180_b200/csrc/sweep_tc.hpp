// Rotate-score-gradient sweep on the tensor cores (sweep_tc.cu).
#pragma once

#include <cuda_runtime.h>

namespace bmb {

struct SweepTcTimes {
    float tables_ms = 0, gemm_ms = 0, gather_ms = 0;
    double gemm_flops = 0;  // tensor-pipe FLOPs of the two GEMMs (three FP16 passes)
};
// K of the real half-plane rows at band L
long long sweep_tc_k(int L);
// xi: P XiBlocks kernels of degree L (device complex128, full plane), euler: G
// triples (device double); out (device double, P x G x 4): value, dC/dalpha,
// dC/dbeta, dC/dgamma.  times (optional) synchronizes and reports the phases.
int sweep_tc(const double* xi, int P, int L, const double* euler, int G, double* out, void* scratch, cudaStream_t s,
             SweepTcTimes* times = nullptr);
size_t sweep_tc_bytes(int P, int L, int G);  // scratch the call needs (context-owned, grow-only)

}  // namespace bmb
