// pft_kernels.cu -- sm_100a kernels of transform.execute (Algorithm 2
// PAPER.md:379-395) and the seeded input generator.
//
//  K1  k1_contract_fft<R, MU0>   one CTA per (residue class c mod P2, signal).  Streams
//      the P1 rows k = c + P2*k1 of A (A[k][l] = a[q k + l]) straight from
//      HBM with 128-bit coalesced loads, contracts each row against the plan in the
//      structured form B[l][j] = phase_l * w_j * t_l^j -- 3r+3 FP64 ops per
//      element instead of 4r -- reduces over the 8 lanes that share a row by shuffles,
//      keeps the P1 x r slab C_c in shared memory and runs the first FFT pass there:
//      Y_c[m1][j] = sum_k1 C[c + P2 k1][j] e^{-2 pi i m1 k1 / P1}.
//  K2  k2_combine_post<R>        one CTA per m1 in [P1].  Finishes the length-p FFT only
//      at the 2M+1 bins that Eq. (7) reads (m' = m mod p, m1 = m' mod P1):
//      Chat[m'][j] = sum_c e^{-2 pi i m' c / p} Y_c[m1][j], fused with the post-process
//      out[m] = e^{-pi i m/p} sum_j Chat[m'][j] ((m - mu)/p)^j.
//  K0  k0_generate               BASELINE.json synthetic inputs (bench only).
//
// Summation orders are fixed (lane-strided partial sums + xor-butterfly), so results
// are deterministic run to run.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../common/rng.h"
#include "fft_smem.cuh"
#include "kernels.cuh"

namespace pftdev {

// ----------------------------------------------------------------------------- K1

__device__ __forceinline__ double2 ld_stream(const double2* p) {
    // read-once input: do not allocate in L1
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}

template <int R, bool MU0>
__global__ void __launch_bounds__(K1_THREADS) k1_contract_fft(K1Params P) {
    extern __shared__ double2 smem[];
    double2* Cs = smem;                        // [R][P1]
    double2* scratch = smem + (size_t)R * P.P1;  // [R][P1]

    const uint32_t c = blockIdx.x;      // residue class
    const uint32_t b = blockIdx.y;      // signal in the batch
    const int gl = threadIdx.x & (K1_GROUP - 1);  // lane within the row group
    const int grp = threadIdx.x / K1_GROUP;       // row group
    const double2* __restrict__ sig = P.a + (size_t)b * P.batch_stride;
    const double2* __restrict__ phase = P.phase + P.l0;
    const double* __restrict__ tv = P.tvals + P.l0;
    const uint64_t lq = P.lq;

    // Warp-uniform trip count: the shuffles below need all 32 lanes.
    for (uint32_t k1base = 0; k1base < P.P1; k1base += K1_ROWS_PER_PASS) {
        const uint32_t k1 = k1base + grp;
        const bool active = k1 < P.P1;
        const uint64_t k = (uint64_t)c + (uint64_t)P.P2 * (active ? k1 : 0);
        const double2* __restrict__ row = sig + k * P.row_stride;
        const uint64_t my_lq = active ? lq : 0;
        double are[R], aim[R];
#pragma unroll
        for (int j = 0; j < R; ++j) are[j] = aim[j] = 0.0;

        for (uint64_t s0 = gl; s0 < my_lq; s0 += (uint64_t)K1_GROUP * K1_UNROLL) {
            double2 v[K1_UNROLL];
            double2 ph[K1_UNROLL];
            double t[K1_UNROLL];
#pragma unroll
            for (int u = 0; u < K1_UNROLL; ++u) {
                const uint64_t l = s0 + (uint64_t)u * K1_GROUP;
                if (l < lq) {
                    v[u] = ld_stream(row + l);
                    if constexpr (!MU0) ph[u] = __ldg(phase + l);
                    t[u] = __ldg(tv + l);
                } else {
                    v[u] = make_double2(0.0, 0.0);
                    if constexpr (!MU0) ph[u] = make_double2(0.0, 0.0);
                    t[u] = 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < K1_UNROLL; ++u) {
                double2 x = v[u];
                if constexpr (!MU0) x = cmul(x, ph[u]);  // a_{qk+l} * e^{-2 pi i mu (l - q/2)/N}
                are[0] += x.x;
                aim[0] += x.y;
                double tp = t[u];
#pragma unroll
                for (int j = 1; j < R; ++j) {
                    are[j] = fma(x.x, tp, are[j]);
                    aim[j] = fma(x.y, tp, aim[j]);
                    if (j + 1 < R) tp *= t[u];
                }
            }
        }
        // reduce over the K1_GROUP lanes of this row (fixed xor-butterfly order)
#pragma unroll
        for (int j = 0; j < R; ++j) {
#pragma unroll
            for (int off = K1_GROUP / 2; off >= 1; off >>= 1) {
                are[j] += __shfl_xor_sync(0xffffffffu, are[j], off);
                aim[j] += __shfl_xor_sync(0xffffffffu, aim[j], off);
            }
        }
        // C[k][j] = w_j * acc_j ; lane gl stores the columns j == gl (mod K1_GROUP)
#pragma unroll
        for (int j = 0; j < R; ++j) {
            if (active && (j % K1_GROUP) == gl) {
                const double2 wj = __ldg(P.w + j);
                Cs[(size_t)j * P.P1 + k1] = cmul(make_double2(are[j], aim[j]), wj);
            }
        }
    }
    __syncthreads();

    // First FFT pass over k1 (length P1) for every column j, in shared memory.
    const double2* res = Cs;
    if (P.P1 > 1) {
        Twiddles tw{P.omega, P.P2};  // omega_P1^t = omega_p^{t P2}
        res = fft_columns(Cs, scratch, R, P.fft, tw);
    }
    // Y[b][m1][c][j]: the slab for one m1 is contiguous over (c, j) for K2.
    double2* __restrict__ Y = P.Y + (size_t)b * P.P1 * P.P2 * R;
    for (uint32_t idx = threadIdx.x; idx < (uint32_t)R * P.P1; idx += blockDim.x) {
        const uint32_t m1 = idx / R, j = idx - m1 * R;
        Y[((size_t)m1 * P.P2 + c) * R + j] = res[(size_t)j * P.P1 + m1];
    }
}

// ----------------------------------------------------------------------------- K2

template <int R>
__global__ void __launch_bounds__(K2_THREADS) k2_combine_post(K2Params P) {
    const uint32_t m1 = blockIdx.x;
    const uint32_t b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    constexpr int NW = K2_THREADS / 32;
    // slots s whose bin m' = (first + s) mod p satisfies m' mod P1 == m1
    const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
    const double2* __restrict__ Y = P.Y + ((size_t)b * P.P1 + m1) * (size_t)P.P2 * R;
    double2* __restrict__ out = P.out + (size_t)b * P.W;

    for (uint64_t s = s0 + (uint64_t)P.P1 * warp; s < P.W; s += (uint64_t)P.P1 * NW) {
        // m' = (first + s) mod p, computed without overflow from first mod p
        uint64_t mp = P.first_mod_p + s % P.p;
        if (mp >= P.p) mp -= P.p;
        double pw[R];
#pragma unroll
        for (int j = 0; j < R; ++j) pw[j] = __ldg(P.post_powers + s * R + j);
        double2 acc = make_double2(0.0, 0.0);
        for (uint32_t c = lane; c < P.P2; c += 32) {
            const double2* yc = Y + (size_t)c * R;
            double2 S = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < R; ++j) {  // ascending j
                const double2 y = __ldg(yc + j);
                S.x = fma(y.x, pw[j], S.x);
                S.y = fma(y.y, pw[j], S.y);
            }
            const uint64_t e = (mp * (uint64_t)c) % P.p;
            const double2 tw = __ldg(P.omega + e);  // e^{-2 pi i m' c / p}
            acc = cadd(acc, cmul(S, tw));
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
        }
        if (lane == 0) {
            const double2 v = cmul(acc, __ldg(P.post_twiddles + s));  // e^{-pi i m / p}
            out[s] = v;
            if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
        }
    }
}

// ----------------------------------------------------------------------------- K0

__global__ void k0_generate(GenParams G) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G.count; i += stride) {
        const uint64_t g = G.index_offset + i;
        double2 v;
        if (G.kind == 0) {
            v.x = pft_uniform_pm1(pft_bits(G.seed, PFT_STREAM_RE, g));
            v.y = pft_uniform_pm1(pft_bits(G.seed, PFT_STREAM_IM, g));
        } else {
            const double u1 = pft_uniform_open0(pft_bits(G.seed, PFT_STREAM_G1, g));
            const uint64_t b2 = pft_bits(G.seed, PFT_STREAM_G2, g) >> 11;
            const double rad = sqrt(-log(u1));
            double sn, cs;
            sincospi((double)b2 * 0x1.0p-52, &sn, &cs);
            v = make_double2(rad * cs, rad * sn);
            if (G.kind == 2) {
                const uint64_t n = g % G.N;
                double2 acc = make_double2(0.0, 0.0);
                for (int t = 0; t < G.n_tones; ++t) {
                    // e^{2 pi i f n / N} with (f n) mod N reduced exactly
                    const int64_t f = G.freqs[t];
                    const uint64_t fm = (uint64_t)(((f % (int64_t)G.N) + (int64_t)G.N) % (int64_t)G.N);
                    const unsigned __int128 prod = (unsigned __int128)fm * n;
                    const uint64_t red = (uint64_t)(prod % G.N);
                    double s2, c2;
                    sincospi(2.0 * ((double)red / (double)G.N), &s2, &c2);
                    acc = cadd(acc, cmul(G.amps[t], make_double2(c2, s2)));
                }
                v = make_double2(acc.x + G.sigma * v.x, acc.y + G.sigma * v.y);
            }
        }
        G.out[i] = v;
    }
}

// ----------------------------------------------------------------------------- dispatch

template <int R>
static cudaError_t launch_k1_r(const K1Params& P, dim3 grid, size_t smem, cudaStream_t st, bool mu0) {
    if (mu0)
        k1_contract_fft<R, true><<<grid, K1_THREADS, smem, st>>>(P);
    else
        k1_contract_fft<R, false><<<grid, K1_THREADS, smem, st>>>(P);
    return cudaGetLastError();
}

template <int R>
static cudaError_t configure_k1_r(size_t smem, bool mu0) {
    if (mu0)
        return cudaFuncSetAttribute(k1_contract_fft<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return cudaFuncSetAttribute(k1_contract_fft<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int R>
static cudaError_t launch_k2_r(const K2Params& P, dim3 grid, cudaStream_t st) {
    k2_combine_post<R><<<grid, K2_THREADS, 0, st>>>(P);
    return cudaGetLastError();
}

#define PFT_R_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) \
    X(14) X(15) X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25)

cudaError_t launch_k1(const K1Params& P, int r, uint32_t batch, bool mu0, cudaStream_t st) {
    const dim3 grid(P.P2, batch);
    const size_t smem = k1_smem_bytes(r, P.P1);
    switch (r) {
#define X(n) case n: return launch_k1_r<n>(P, grid, smem, st, mu0);
        PFT_R_CASES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t configure_k1(int r, uint32_t P1, bool mu0) {
    const size_t smem = k1_smem_bytes(r, P1);
    switch (r) {
#define X(n) case n: return configure_k1_r<n>(smem, mu0);
        PFT_R_CASES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_k2(const K2Params& P, int r, uint32_t batch, cudaStream_t st) {
    const dim3 grid(P.P1, batch);
    switch (r) {
#define X(n) case n: return launch_k2_r<n>(P, grid, st);
        PFT_R_CASES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_k0(const GenParams& G, cudaStream_t st) {
    const int threads = 256;
    uint64_t blocks = (G.count + threads - 1) / threads;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (blocks == 0) return cudaSuccess;
    k0_generate<<<(unsigned)blocks, threads, 0, st>>>(G);
    return cudaGetLastError();
}

}  // namespace pftdev
