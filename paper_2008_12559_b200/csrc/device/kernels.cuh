// kernels.cuh -- launch parameters shared by the kernels and the device plan.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_smem.cuh"

namespace pftdev {

// K1: 8 consumer warps + 1 TMA producer warp; a stage is a 32-row x 32-column box of A
// (16 KiB of complex128); 4 stages in flight per CTA, 2 CTAs per SM.
constexpr int K1_CONSUMER_WARPS = 8;
constexpr int K1_THREADS = 32 * (K1_CONSUMER_WARPS + 1);
constexpr int K1_GROUP = 8;       // lanes per row
constexpr int K1_BOX_ROWS = 32;   // = K1_CONSUMER_WARPS * (32 / K1_GROUP)
constexpr int K1_CH = 32;         // columns per stage
constexpr int K1_STAGES = 4;
constexpr int K1_STAGE_ELEMS = K1_BOX_ROWS * K1_CH;
constexpr uint32_t K1_STAGE_BYTES = K1_STAGE_ELEMS * 16;
constexpr size_t K1_RING_BYTES = (size_t)K1_STAGES * K1_STAGE_BYTES;
static_assert(K1_BOX_ROWS == K1_CONSUMER_WARPS * (32 / K1_GROUP), "one row per lane group");

constexpr int K2_THREADS = 256;

struct K1Params {
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
    const double2* Y;              // [batch][P1][P2][r]
    const double* post_powers;     // [W][r]
    const double2* post_twiddles;  // [W]
    const double2* omega;          // [p]
    uint64_t p;
    uint32_t P1, P2;
    uint64_t W;                    // 2M + 1
    uint64_t first_mod_p;          // (mu - M) mod p
    uint32_t first_mod_p1;         // (mu - M) mod P1
    int use_fft;                   // k2_fft_post (1) or k2_direct_post (0)
    FftRadices fft2;               // radices of P2
    double2* out;                  // [batch][W]
    int* status;
};

struct GenParams {
    int kind;
    uint64_t seed, N, index_offset, count;
    int n_tones;
    const int64_t* freqs;  // device
    const double2* amps;   // device
    double sigma;
    double2* out;
};

// ring + C slab + 2*S mbarriers; the ring doubles as the FFT scratch (needs r*P1*16 <= ring)
inline size_t k1_smem_bytes(int r, uint32_t P1) {
    return K1_RING_BYTES + sizeof(double2) * (size_t)r * (P1 ? P1 : 1) + 2 * K1_STAGES * sizeof(uint64_t);
}
inline size_t k2_smem_bytes(int r, uint32_t P2) { return 2 * sizeof(double2) * (size_t)r * P2; }

cudaError_t configure_k1(int r, uint32_t P1, bool mu0);
cudaError_t configure_k2(int r, uint32_t P2);
cudaError_t launch_k1(const CUtensorMap& map, const K1Params& P, int r, uint32_t batch, bool mu0, cudaStream_t st);
cudaError_t launch_k2(const K2Params& P, int r, uint32_t batch, cudaStream_t st);
cudaError_t launch_k0(const GenParams& G, cudaStream_t st);

}  // namespace pftdev
