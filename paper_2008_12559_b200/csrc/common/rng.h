/* rng.h -- counter-based generators for the seeded synthetic inputs of BASELINE.json.
 * Shared verbatim by the host library and the device generator kernel so that the
 * uniform kind is bit-identical on CPU and GPU (integer mixing + exact scaling). */
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PFT_HD __host__ __device__ __forceinline__
#else
#define PFT_HD inline
#endif

/* SplitMix64 finaliser (Steele, Lea & Flood 2014). */
PFT_HD uint64_t pft_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* 64 random bits for (seed, stream, global element index). */
PFT_HD uint64_t pft_bits(uint64_t seed, uint32_t stream, uint64_t index) {
    return pft_mix64(pft_mix64(seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(stream + 1))) ^ index);
}

/* Uniform on [-1, 1): k * 2^-52 - 1 with k uniform in [0, 2^53); exact in binary64. */
PFT_HD double pft_uniform_pm1(uint64_t bits) {
    return (double)(bits >> 11) * 0x1.0p-52 - 1.0;
}

/* Uniform on (0, 1]. */
PFT_HD double pft_uniform_open0(uint64_t bits) {
    return ((double)(bits >> 11) + 1.0) * 0x1.0p-53;
}

/* Streams used by the generators (stable numbering: changing them changes every fixture). */
enum { PFT_STREAM_RE = 0, PFT_STREAM_IM = 1, PFT_STREAM_G1 = 2, PFT_STREAM_G2 = 3,
       PFT_STREAM_TONE_F = 4, PFT_STREAM_TONE_A1 = 5, PFT_STREAM_TONE_A2 = 6 };
