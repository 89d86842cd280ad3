// kernels.cuh -- launch parameters shared by the kernels and the device plan.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_smem.cuh"

namespace pftdev {

constexpr int K1_THREADS = 256;  // 8 warps
constexpr int K1_GROUP = 8;      // lanes per row: one 128-byte line per load instruction per group
constexpr int K1_ROWS_PER_PASS = K1_THREADS / K1_GROUP;
constexpr int K1_UNROLL = 4;     // independent 16-byte loads in flight per lane
constexpr int K2_THREADS = 256;

struct K1Params {
    const double2* a;       // signal 0, element 0 of the local buffer
    uint64_t batch_stride;  // elements between signals
    uint64_t row_stride;    // elements between consecutive rows k (q, or the local width)
    uint64_t lq;            // columns of each row processed by this launch
    uint64_t l0;            // global column index of local column 0 (table offset)
    const double2* phase;   // [q]  e^{-2 pi i mu (l - q/2) / N}
    const double* tvals;    // [q]  1 - 2l/q
    const double2* w;       // [r]  w_{eps, r-1, j}
    const double2* omega;   // [p]  e^{-2 pi i t / p}
    uint32_t P1, P2;        // p = P1 * P2
    FftRadices fft;         // radices of P1
    double2* Y;             // [batch][P1][P2][r]
};

struct K2Params {
    const double2* Y;           // [batch][P1][P2][r]
    const double* post_powers;  // [W][r]
    const double2* post_twiddles;  // [W]
    const double2* omega;       // [p]
    uint64_t p;
    uint32_t P1, P2;
    uint64_t W;                 // 2M + 1
    uint64_t first_mod_p;       // (mu - M) mod p
    uint32_t first_mod_p1;      // (mu - M) mod P1
    double2* out;               // [batch][W]
    int* status;
};

struct GenParams {
    int kind;
    uint64_t seed, N, index_offset, count;
    int n_tones;
    const int64_t* freqs;   // device
    const double2* amps;    // device
    double sigma;
    double2* out;
};

inline size_t k1_smem_bytes(int r, uint32_t P1) {
    return P1 > 1 ? 2 * sizeof(double2) * (size_t)r * P1 : sizeof(double2) * (size_t)r;
}

cudaError_t configure_k1(int r, uint32_t P1, bool mu0);
cudaError_t launch_k1(const K1Params& P, int r, uint32_t batch, bool mu0, cudaStream_t st);
cudaError_t launch_k2(const K2Params& P, int r, uint32_t batch, cudaStream_t st);
cudaError_t launch_k0(const GenParams& G, cudaStream_t st);

}  // namespace pftdev
