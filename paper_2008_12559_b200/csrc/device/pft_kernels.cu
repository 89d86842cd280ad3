// pft_kernels.cu -- dispatch of the sm_100a kernels on r, the 2-D transpose and the seeded input
// generator.  The kernel templates live in kernel_templates.cuh; their per-r instantiations are
// compiled by kinst_*.cu in parallel (declared extern here).
#include "kernel_templates.cuh"

namespace pftdev {

#define PFT_EXTERN_INSTANCES(R) PFT_INSTANCES(R, extern)
PFT_R_CASES(PFT_EXTERN_INSTANCES)
#undef PFT_EXTERN_INSTANCES

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

int k1_max_active_per_sm(int r, uint32_t P1, uint32_t stages, bool mu0) {
    const size_t smem = k1_smem_bytes(r, P1, stages);
    switch (r) {
#define X(n) case n: return k1_active_r<n>(smem, mu0);
        PFT_R_CASES(X)
#undef X
    }
    return 0;
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
    const dim3 grid(P.P2 * (P.split > 1 ? P.split : 1) + P.workers, batch);
    const size_t smem = k1_smem_bytes(r, P.rows ? P.rows : P.P1, P.stages);
    switch (r) {
#define X(n) case n: return launch_k1_r<n>(map, P, grid, smem, st, mu0);
        PFT_R_CASES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_k2(const K2Params& P, int r, uint32_t batch, cudaStream_t st) {
    const uint32_t gx = P.mode == K2_L2 ? (P.k2_ctas ? P.k2_ctas : 148u)
                        : (P.mode == K2_FFT && P.ring && P.k2_ctas > 0) ? (P.k2_ctas < P.P1 ? P.k2_ctas : P.P1)
                                                               : P.P1;
    const dim3 grid(gx, batch);
    switch (r) {
#define X(n) case n: return launch_k2_r<n>(P, grid, st);
        PFT_R_CASES(X)
#undef X
    }
    return cudaErrorInvalidValue;
}


// 2-D PFT glue: out[c][r] = in[r][c] for an rows x cols complex128 matrix, through a 32 x 33
// shared tile (coalesced on both sides).
__global__ void k_transpose(const double2* __restrict__ in, double2* __restrict__ out, uint64_t rows,
                            uint64_t cols) {
    __shared__ double2 tile[32][33];
    const uint64_t c0 = (uint64_t)blockIdx.x * 32, r0 = (uint64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
    }
}

cudaError_t launch_transpose(const double2* in, double2* out, uint64_t rows, uint64_t cols, cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    k_transpose<<<grid, dim3(32, 8), 0, st>>>(in, out, rows, cols);
    return cudaGetLastError();
}

// Exact-angle direct DFT (naive_dft; Eq. (1)): out[s] = sum_n a[n] e^{-2 pi i m n / N}
// for m = first + s, with (m n) mod N carried exactly in integers (k_{n+T} = k_n + (m T mod N) mod N)
// and one sincospi per term on the exactly reduced angle (no angle recurrence).
// One CTA per bin; lane-strided partial sums then a fixed shuffle / shared-memory tree:
// deterministic.  O(N (2M+1)) work: the CLI's --verify, the anomaly pipeline's "fft" source and
// the bench's naive column run it at desk scale.
constexpr int kNaiveThreads = 256;
__global__ void __launch_bounds__(kNaiveThreads) k_naive_dft(const double2* __restrict__ a, uint64_t N,
                                                            int64_t first, double2* __restrict__ out) {
    __shared__ double2 part[kNaiveThreads / 32];
    const int64_t m = first + (int64_t)blockIdx.x;
    const uint64_t mm = (uint64_t)(((m % (int64_t)N) + (int64_t)N) % (int64_t)N);  // m mod N
    const uint64_t t = threadIdx.x;
    uint64_t k = (uint64_t)(((unsigned __int128)mm * t) % N);                       // (m t) mod N
    const uint64_t step = (uint64_t)(((unsigned __int128)mm * kNaiveThreads) % N);  // (m T) mod N
    const double invN2 = 2.0 / (double)N;
    double2 acc = make_double2(0.0, 0.0);
    for (uint64_t n = t; n < N; n += kNaiveThreads) {
        double sn, cs;
        sincospi(-(double)k * invN2, &sn, &cs);  // e^{-2 pi i k / N}
        const double2 x = __ldg(a + n);
        acc.x = fma(x.x, cs, fma(-x.y, sn, acc.x));
        acc.y = fma(x.x, sn, fma(x.y, cs, acc.y));
        k += step;
        if (k >= N) k -= N;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if ((t & 31) == 0) part[t >> 5] = acc;
    __syncthreads();
    if (t == 0) {
        double2 tot = part[0];
        for (int w = 1; w < kNaiveThreads / 32; ++w) tot = cadd(tot, part[w]);
        out[blockIdx.x] = tot;
    }
}

cudaError_t launch_naive_dft(const double2* a, uint64_t N, int64_t first, uint64_t count, double2* out,
                             cudaStream_t st) {
    for (uint64_t done = 0; done < count;) {  // grid.x <= 2^31 - 1 bins per launch
        const uint64_t n = count - done < (1ull << 30) ? count - done : (1ull << 30);
        k_naive_dft<<<(unsigned)n, kNaiveThreads, 0, st>>>(a, N, first + (int64_t)done, out + done);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        done += n;
    }
    return cudaSuccess;
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
