// pft_kernels.cu -- sm_100a kernels of transform.execute (Algorithm 2
// PAPER.md:379-395) and the seeded input generator.
//
//  K1  k1_contract_fft<R, MU0>  one CTA per (residue class c mod P2, signal).  A producer
//      warp streams the P1 rows k = c + P2*k1 of A (A[k][l] = a[q k + l])
//      from HBM into a 4-stage shared-memory ring with 4-D bulk tensor copies (TMA,
//      cp.async.bulk.tensor + mbarrier complete_tx), 32 rows x 32 columns per stage.
//      Eight consumer warps contract each row against the plan in the structured form
//      B[l][j] = phase_l * w_j * t_l^j: 3r+3 FP64 ops per element instead of
//      the dense 4r, 8 lanes per row, xor-shuffle reduction per row.  The P1 x r slab C_c
//      stays in shared memory and gets the first FFT pass there:
//      Y_c[m1][j] = sum_k1 C[c + P2 k1][j] e^{-2 pi i m1 k1 / P1}.
//  K2  k2_fft_post<R>           one CTA per m1 in [P1].  Applies the four-step twiddle
//      e^{-2 pi i m1 c / p}, runs the length-P2 FFT over c in shared memory, and evaluates
//      Eq. (7) only at the 2M+1 requested bins (m' = m mod p, m' = m1 + P1 m2):
//      out[m] = e^{-pi i m/p} sum_j Chat[m'][j] ((m - mu)/p)^j.
//      k2_direct_post<R> is the any-P2 fallback (direct sum over c).
//  K0  k0_generate              BASELINE.json synthetic inputs (bench only).
//
// Summation orders are fixed (lane-strided partial sums + xor-butterfly), so results
// are deterministic run to run.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../common/rng.h"
#include "fft_smem.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace pftdev {

// ----------------------------------------------------------------------------- K1

template <int R, bool MU0>
__global__ void __launch_bounds__(K1_THREADS, 2) k1_contract_fft(const __grid_constant__ CUtensorMap tmap,
                                                                  const K1Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2* ring = reinterpret_cast<double2*>(smem_raw);    // [S][32 rows][CH]
    double2* Cs = ring + (size_t)K1_STAGES * K1_STAGE_ELEMS;  // [R][P1]
    uint64_t* full = reinterpret_cast<uint64_t*>(Cs + (size_t)R * P.P1);
    uint64_t* empty = full + K1_STAGES;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < K1_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], K1_CONSUMER_WARPS);
        }
        fence_barrier_init();
    }
    __syncthreads();

    const uint32_t c = blockIdx.x;  // residue class k = c (mod P2)
    const uint32_t b = blockIdx.y;  // signal
    const uint32_t nch = (uint32_t)((P.lq + K1_CH - 1) / K1_CH);
    const uint32_t nrb = (P.P1 + K1_BOX_ROWS - 1) / K1_BOX_ROWS;
    const uint32_t total = nch * nrb;

    if (warp == K1_CONSUMER_WARPS) {
        // ---- producer: one elected lane streams 32-row x CH-column boxes of A into the ring
        if (lane == 0) {
            prefetch_tensormap(&tmap);
            for (uint32_t it = 0; it < total; ++it) {
                const uint32_t s = it % K1_STAGES, n = it / K1_STAGES;
                if (n > 0) mbar_wait(&empty[s], (n - 1) & 1);
                const uint32_t rb = it / nch, ch = it - rb * nch;
                mbar_arrive_expect_tx(&full[s], K1_STAGE_BYTES);
                tma_load_4d(ring + (size_t)s * K1_STAGE_ELEMS, &tmap, (int)(2 * ch * K1_CH), (int)c,
                            (int)(rb * K1_BOX_ROWS), (int)b, &full[s]);
            }
        }
    } else {
        // ---- consumers: 8 lanes per row, 4 rows per warp, 32 rows per box
        const int gl = lane & (K1_GROUP - 1);
        const int grp = warp * (32 / K1_GROUP) + lane / K1_GROUP;
        const uint64_t lmax = P.l0 + P.lq - 1;  // last valid global column (clamp for zero-filled lanes)
        for (uint32_t rb = 0; rb < nrb; ++rb) {
            double are[R], aim[R];
#pragma unroll
            for (int j = 0; j < R; ++j) are[j] = aim[j] = 0.0;
            for (uint32_t ch = 0; ch < nch; ++ch) {
                const uint32_t it = rb * nch + ch;
                const uint32_t s = it % K1_STAGES, n = it / K1_STAGES;
                mbar_wait(&full[s], n & 1);
                // Reconverge before touching the stage: lane 0's `empty` arrive below leaves
                // the warp diverged, and reading a stage from a diverged warp was observed to
                // return corrupt rows on B200 when two K1 CTAs share an SM.
                __syncwarp();
                const double2* row = ring + (size_t)s * K1_STAGE_ELEMS + (size_t)grp * K1_CH;
#pragma unroll
                for (int u = 0; u < K1_CH / K1_GROUP; ++u) {
                    const int col = gl + u * K1_GROUP;
                    // out-of-range columns/rows arrive as TMA zero fill and contribute 0
                    uint64_t l = P.l0 + (uint64_t)ch * K1_CH + col;
                    l = l > lmax ? lmax : l;
                    double2 x = row[col];
                    if constexpr (!MU0) x = cmul(x, __ldg(P.phase + l));  // a * e^{-2 pi i mu (l - q/2)/N}
                    const double t = __ldg(P.tvals + l);                   // 1 - 2l/q
                    are[0] += x.x;
                    aim[0] += x.y;
                    double tp = t;
#pragma unroll
                    for (int j = 1; j < R; ++j) {
                        are[j] = fma(x.x, tp, are[j]);
                        aim[j] = fma(x.y, tp, aim[j]);
                        if (j + 1 < R) tp *= t;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);  // stage s may be refilled
            }
            // reduce over the 8 lanes of the row (fixed xor-butterfly order)
#pragma unroll
            for (int j = 0; j < R; ++j) {
#pragma unroll
                for (int off = K1_GROUP / 2; off >= 1; off >>= 1) {
                    are[j] += __shfl_xor_sync(0xffffffffu, are[j], off);
                    aim[j] += __shfl_xor_sync(0xffffffffu, aim[j], off);
                }
            }
            const uint32_t k1 = rb * K1_BOX_ROWS + grp;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (k1 < P.P1 && (j % K1_GROUP) == gl)
                    Cs[(size_t)j * P.P1 + k1] = cmul(make_double2(are[j], aim[j]), __ldg(P.w + j));  // C = w_j acc_j
            }
        }
    }
    __syncthreads();

    // First FFT pass over k1 (length P1) for every column j, in shared memory; the ring is
    // idle now and serves as the Stockham scratch buffer.
    const double2* res = Cs;
    if (P.P1 > 1) {
        Twiddles tw{P.omega, P.P2};  // omega_P1^t = omega_p^{t P2}
        res = fft_columns(Cs, ring, R, P.fft, tw);
    }
    // Y[b][m1][c][j]: the slab for one m1 is contiguous over (c, j) for K2.
    double2* __restrict__ Y = P.Y + (size_t)b * P.P1 * P.P2 * R;
    for (uint32_t idx = tid; idx < (uint32_t)R * P.P1; idx += blockDim.x) {
        const uint32_t m1 = idx / R, j = idx - m1 * R;
        Y[((size_t)m1 * P.P2 + c) * R + j] = res[(size_t)j * P.P1 + m1];
    }
}

// ----------------------------------------------------------------------------- K2

template <int R>
__global__ void __launch_bounds__(K2_THREADS) k2_fft_post(K2Params P) {
    extern __shared__ __align__(16) double2 zs[];
    double2* Z = zs;  // [R][P2]
    double2* scratch = zs + (size_t)R * P.P2;
    const uint32_t m1 = blockIdx.x, b = blockIdx.y;
    const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
    if (s0 >= P.W) return;  // no output slot maps to this m1 (block-uniform)
    const double2* __restrict__ Y = P.Y + ((size_t)b * P.P1 + m1) * (size_t)P.P2 * R;
    for (uint32_t idx = threadIdx.x; idx < P.P2 * (uint32_t)R; idx += blockDim.x) {
        const uint32_t c = idx / R, j = idx - c * R;
        const double2 y = Y[idx];
        // four-step twiddle e^{-2 pi i m1 c / p}; m1 c < P1 P2 = p needs no reduction
        Z[(size_t)j * P.P2 + c] = (m1 == 0 || c == 0) ? y : cmul(y, __ldg(P.omega + (size_t)m1 * c));
    }
    __syncthreads();
    const double2* res = Z;
    if (P.P2 > 1) {
        Twiddles tw{P.omega, P.P1};  // omega_P2^t = omega_p^{t P1}
        res = fft_columns(Z, scratch, R, P.fft2, tw);
    }
    double2* __restrict__ out = P.out + (size_t)b * P.W;
    for (uint64_t s = s0 + (uint64_t)P.P1 * threadIdx.x; s < P.W; s += (uint64_t)P.P1 * blockDim.x) {
        uint64_t mp = P.first_mod_p + s % P.p;
        if (mp >= P.p) mp -= P.p;
        const uint32_t m2 = (uint32_t)(mp / P.P1);
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < R; ++j) {  // ascending j
            const double pw = __ldg(P.post_powers + s * R + j);
            const double2 v = res[(size_t)j * P.P2 + m2];
            acc.x = fma(v.x, pw, acc.x);
            acc.y = fma(v.y, pw, acc.y);
        }
        const double2 v = cmul(acc, __ldg(P.post_twiddles + s));  // e^{-pi i m / p}
        out[s] = v;
        if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
    }
}

// Direct form for any P2 (P2 with a prime factor > 64, or too large for shared memory):
// Chat[m'][j] = sum_c e^{-2 pi i m' c / p} Y[m1][c][j], one warp per output slot.
template <int R>
__global__ void __launch_bounds__(K2_THREADS) k2_direct_post(K2Params P) {
    const uint32_t m1 = blockIdx.x;
    const uint32_t b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    constexpr int NW = K2_THREADS / 32;
    const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
    const double2* __restrict__ Y = P.Y + ((size_t)b * P.P1 + m1) * (size_t)P.P2 * R;
    double2* __restrict__ out = P.out + (size_t)b * P.W;

    for (uint64_t s = s0 + (uint64_t)P.P1 * warp; s < P.W; s += (uint64_t)P.P1 * NW) {
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
            acc = cadd(acc, cmul(S, __ldg(P.omega + e)));  // e^{-2 pi i m' c / p}
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

#define PFT_R_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) \
    X(14) X(15) X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25)

template <int R>
static cudaError_t launch_k1_r(const CUtensorMap& map, const K1Params& P, dim3 grid, size_t smem, cudaStream_t st,
                               bool mu0) {
    if (mu0)
        k1_contract_fft<R, true><<<grid, K1_THREADS, smem, st>>>(map, P);
    else
        k1_contract_fft<R, false><<<grid, K1_THREADS, smem, st>>>(map, P);
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
    if (P.use_fft)
        k2_fft_post<R><<<grid, K2_THREADS, k2_smem_bytes(R, P.P2), st>>>(P);
    else
        k2_direct_post<R><<<grid, K2_THREADS, 0, st>>>(P);
    return cudaGetLastError();
}

template <int R>
static cudaError_t configure_k2_r(size_t smem) {
    return cudaFuncSetAttribute(k2_fft_post<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// The attribute is only a cap (the launch's dynamic size decides occupancy), so set it to
// the device maximum once instead of per plan: plans with different P1 share a kernel.
constexpr size_t kMaxDynSmem = 227 * 1024;

cudaError_t configure_k1(int r, uint32_t P1, bool mu0) {
    (void)P1;
    const size_t smem = kMaxDynSmem;
    switch (r) {
#define X(n) case n: return configure_k1_r<n>(smem, mu0);
        PFT_R_CASES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t configure_k2(int r, uint32_t P2) {
    (void)P2;
    const size_t smem = kMaxDynSmem;
    switch (r) {
#define X(n) case n: return configure_k2_r<n>(smem);
        PFT_R_CASES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_k1(const CUtensorMap& map, const K1Params& P, int r, uint32_t batch, bool mu0, cudaStream_t st) {
    const dim3 grid(P.P2, batch);
    const size_t smem = k1_smem_bytes(r, P.P1);
    switch (r) {
#define X(n) case n: return launch_k1_r<n>(map, P, grid, smem, st, mu0);
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
