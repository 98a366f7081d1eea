// Seeded synthetic inputs on the device (kernel K10), see generate.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bmb {

void make_template(int n, int blobs, uint64_t seed, float* out, cudaStream_t s);
// particles p = 0..count-1 use seed base_seed + p; quats (4 per particle, host)
// and shifts (3 per particle, host) receive the ground truth.
void make_particles(const float* tmpl, int n, int count, uint64_t base_seed, int shift_max, double snr,
                    double wedge_deg, float* out, double* quats, int* shifts, cudaStream_t s);

}  // namespace bmb
