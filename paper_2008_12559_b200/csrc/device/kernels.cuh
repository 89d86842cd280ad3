// kernels.cuh -- launch parameters shared by the kernels and the device plan.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_smem.cuh"

namespace pftdev {

// Checked builds (build.py --checked, -DPFT_CHECKED): every workspace / output / input access the
// kernels compute an index for is bounds-checked against the extents the host passes, and a
// violation traps the kernel (the launch then fails with a CUDA error).  Product builds compile
// the checks away.  (compute-sanitizer is closed on this GPU pool: profiles/r02/sanitizer_attempt.txt.)
#ifdef PFT_CHECKED
#define PFT_BOUND(idx, n)                                                      \
    do {                                                                       \
        if (!(static_cast<uint64_t>(idx) < static_cast<uint64_t>(n))) __trap(); \
    } while (0)
#else
#define PFT_BOUND(idx, n) \
    do {                  \
    } while (0)
#endif

// K1: 8 consumer warps + 1 TMA producer warp.  A stage holds, for 16 rows of A, a chunk of
// 32 column pairs (l, q-l): the "front" box (columns l ascending) and the "mirror" box
// (columns q-l), 16 x 32 complex128 each, plus the 32-entry pair table slice
// {Re phase_l, Im phase_l, t_l, 0}.  Two K1 CTAs share an SM.
constexpr int K1_CONSUMER_WARPS = 8;
constexpr int K1_THREADS = 32 * (K1_CONSUMER_WARPS + 1);
#ifndef PFT_K1_BR
#define PFT_K1_BR 32
#endif
#ifndef PFT_K1_CP
#define PFT_K1_CP 16
#endif
constexpr int K1_BR = PFT_K1_BR;   // rows per box
constexpr int K1_CP = PFT_K1_CP;   // column pairs per chunk
constexpr int K1_LANES_PER_ROW = 32 * K1_CONSUMER_WARPS / K1_BR;  // consumer lanes sharing a row
constexpr uint32_t K1_BOX_BYTES = K1_BR * K1_CP * 16;
constexpr uint32_t K1_TAB_BYTES = K1_CP * 32;
constexpr uint32_t K1_STAGE_BYTES = 2 * K1_BOX_BYTES + K1_TAB_BYTES;
#ifndef PFT_K1_MIN_STAGES
#define PFT_K1_MIN_STAGES 4
#endif
constexpr int K1_MIN_STAGES = PFT_K1_MIN_STAGES, K1_MAX_STAGES = 8;

// FP64 tensor-core contraction (mma.sync m8n8k4 f64, DMMA) for r in [PFT_K1_TC_MIN_R, 18]: per
// pair the even moments j = 2, 4, .., 16 and the odd moments j = 1, 3, .., 15 are two 8-column
// tiles, B fragments t_l^j come with each stage ([pair][g]{even, odd}, host-built), j = 0 and
// (r = 18) j = 17 stay on the FP64 pipe.  A DMMA does 256 FMAs per issue: the contraction
// sheds the power chain and most of its instruction overhead.  Stages carry the fragment
// slice, so the ring may be 3 stages deep to keep two CTAs per SM.
// Measured (same box, swizzled 4-stage layout): C3 p = 256, r = 18: 1017 vs 1276 us per batch
// (split vector path); C3 p = 512, r = 14: 1180 vs 1400 us; C2c p = 2^15, r = 14 with phases:
// 71.6 vs 79.6 us; C2c p = 2^16, r = 12: 83.8 vs 110.5 us.  An earlier unswizzled layout was
// slower than the vector path at r <= 9 (C2b r = 8: 56.8 vs 41.5 us), so from r = 12.
#ifndef PFT_K1_TC_MIN_R
#define PFT_K1_TC_MIN_R 12
#endif
__host__ __device__ constexpr bool k1_tc(int r) { return r >= PFT_K1_TC_MIN_R && r <= 18; }
constexpr uint32_t K1_TC_BYTES = K1_CP * 16 * 8;  // 16 pairs x 8 columns x {even, odd} doubles
// Tensor-core stages: each box arrives as two 8-pair halves (128-byte rows) with the TMA
// 128-byte swizzle (16-byte chunk c of row y at c ^ (y & 7)), so the four rows a warp reads
// together ({0, 1, 4, 5} + offset) hit eight distinct chunks: 2 wavefronts per operand load
// instead of 4.  Swizzled destinations need 1024-byte alignment (the 18 KB stage is a multiple).
constexpr uint32_t K1_TC_DATA_BYTES = 2 * K1_BOX_BYTES + K1_TC_BYTES;             // bytes landed per stage
constexpr uint32_t K1_TC_STAGE_BYTES = (K1_TC_DATA_BYTES + 1023) / 1024 * 1024;    // stage stride
static_assert(K1_CP == 16 && K1_BR == 32, "tensor-core stage layout assumes 32 rows x 16 pairs");
__host__ __device__ constexpr uint32_t k1_stage_bytes(int r) { return k1_tc(r) ? K1_TC_STAGE_BYTES : K1_STAGE_BYTES; }
__host__ __device__ constexpr uint32_t k1_stage_data_bytes(int r) { return k1_tc(r) ? K1_TC_DATA_BYTES : K1_STAGE_BYTES; }
__host__ __device__ constexpr uint32_t k1_ring_align_slack(int r) { return k1_tc(r) ? 1024 : 0; }
__host__ __device__ constexpr int k1_min_stages(int r) { return k1_tc(r) ? 3 : K1_MIN_STAGES; }
inline size_t k1_min_ring_bytes(int r) { return (size_t)k1_min_stages(r) * k1_stage_bytes(r); }
static_assert(K1_TC_BYTES % 128 == 0, "TMA destinations stay 128-byte aligned");
static_assert(K1_LANES_PER_ROW >= 1 && K1_LANES_PER_ROW <= 32 && K1_CP % K1_LANES_PER_ROW == 0, "row mapping");
static_assert(K1_STAGE_BYTES % 128 == 0, "TMA destinations stay 128-byte aligned");

constexpr int K2_THREADS = 256;
constexpr int K2L_THREADS = 128;
enum K2Mode { K2_DIRECT = 0, K2_FFT = 1, K2_DOT = 2, K2_L2 = 3, K2_BLUESTEIN = 4 };
// Bluestein (chirp-z) K2: the length-P2 DFT of any P2 (a prime factor > 64 included) as a
// convolution with a power-of-two length L >= 2 P2 - 1, columns in groups of K2B_GROUP.
constexpr uint32_t K2B_MAX_L = 4096;
inline uint32_t k2_bluestein_group(uint32_t L) { return L <= 2048 ? 2u : 1u; }  // columns per pass
inline size_t k2_bluestein_smem_bytes(uint32_t L) { return sizeof(double2) * 2 * (size_t)k2_bluestein_group(L) * L; }


struct K2Params {
    const double2* Y;              // signal b's slab [P1][P2][r] at Y + b * y_stride
    uint64_t y_stride;             // elements between consecutive signals' slabs
    const double* post_powers;     // [W][r]
    const double2* post_twiddles;  // [W]
    const double2* omega;          // [p]
    uint64_t p;
    uint32_t P1, P2;
    uint64_t W;                    // 2M + 1
    uint64_t first_mod_p;          // (mu - M) mod p
    double inv_p;                  // 1 / p
    uint32_t first_mod_p1;         // (mu - M) mod P1
    int mode;                      // K2_DIRECT / K2_FFT / K2_DOT
    uint32_t k2_ctas;              // K2_L2 grid width (0 = 148); K2_FFT with `ring`: grid width of k2_ring
    int release_next;              // trigger the next launch at K2 start (1) / end (2) (PDL chaining)
    int ring;                      // K2_FFT on k2_ctas CTAs as a bulk-copy ring over m1 (k2_ring)
    FftRadices fft2;               // radices of P2 (K2_FFT) or of L (K2_BLUESTEIN)
    const double2* chirp;          // K2_BLUESTEIN: [P2] e^{-pi i c^2 / P2}
    const double2* chirp_hat;      // K2_BLUESTEIN: [L] FFT_L of the conjugate chirp kernel / L
    const double2* omega_L;        // K2_BLUESTEIN: [L] e^{-2 pi i t / L}
    uint32_t L;                    // K2_BLUESTEIN: convolution length (power of two)
    uint32_t bl_group;             // K2_BLUESTEIN: columns per transform pass (smem: 2 x group x L)
    double2* out;                  // [batch][W]
    int* status;                   // non-finite flag word of the workspace (bit 0)
    uint64_t y_elems;              // checked builds: elements addressable from Y
    uint64_t out_elems;            // checked builds: elements of out
};

// Pair-table entry (host-built): phase_l = e^{-2 pi i mu (l - q/2)/N}, t_l = 1 - 2l/q and
// t_l^h, h = ceil(r/2) (start of the upper j half under the two-lane j split, k1_js).
// The mirror column q-l uses conj(phase_l) and -t_l (exact identities of SPEC.md:126).
struct PairEntry {
    double c, s, t, th;
};

// K1 splits the r moments of a row over JS lanes (JS = 2 from r >= PFT_K1_JS_MIN_R without
// phase factors (mu = 0), from r >= PFT_K1_JS_MIN_R_PHASE with them; vector path only): each
// lane keeps ceil(r/2) accumulator pairs instead of r (no spills with two CTAs per SM), takes
// twice the pairs of a chunk (more independent power chains) and the row reduction shuffles
// half the values over one level fewer.  With phases both lanes repeat the phase multiply, so
// the split pays later (measured C3 p = 256, r = 18, mu = 0: 1535 -> 1267 us per batch;
// C2c r = 14 with phases: 79.8 unsplit vs 84.2 us split; C4 r = 9: 21.0 vs 25.1 us).
#ifndef PFT_K1_JS_MIN_R
#define PFT_K1_JS_MIN_R 12
#endif
#ifndef PFT_K1_JS_MIN_R_PHASE
#define PFT_K1_JS_MIN_R_PHASE 19
#endif
__host__ __device__ constexpr int k1_js(int r, bool mu0) {
    return !k1_tc(r) && r >= (mu0 ? PFT_K1_JS_MIN_R : PFT_K1_JS_MIN_R_PHASE) ? 2 : 1;
}


struct K1Params {
    // local view of A (rows k = c + P2 k1 at a + k * row_stride, signal b at + b * batch_stride)
    const double2* a;
    uint64_t row_stride, batch_stride;
    // column pairs handled by this launch: global pair indices [gp0, gp_end), gp0 >= 1;
    // pair gp0 + t sits at local column fcol0 + t (front) and mcol0 - t (mirror)
    uint32_t gp0, gp_end;
    int32_t fcol0, mcol0;
    // unpaired columns: l = 0 (t = 1) and, for even q, l = q/2 (t = 0); -1 = not in this view
    int32_t single0_col, singleh_col;
    double2 phase0, phaseh;     // phase_0, phase_{q/2}
    const PairEntry* pairtab;   // [>= gp_end + K1_CP]
    const double2* tcfrag;      // [>= gp_end + K1_CP][8] {t^(2+2g), t^(1+2g)} (k1_tc(r) plans)
    const double2* w;           // [r]  w_{eps, r-1, j}
    const double2* omega;       // [p]  e^{-2 pi i t / p}
    uint32_t P1, P2;            // p = P1 * P2
    uint32_t rows;              // rows a CTA contracts: P1, or gsig * P1 when it holds gsig signals
    uint32_t gsig;              // signals per CTA (1; > 1 only for P2 = 1 sum-tail plans on contiguous batches:
                                // signal b * gsig + g's rows are rows g * P1 .. of the CTA's row block)
    FftRadices fft;             // radices of P1
    uint32_t stages;            // ring depth (K1_MIN_STAGES..K1_MAX_STAGES)
    int pdl;                    // launched with programmatic stream serialization
    uint32_t split;             // CTAs (a cluster) per residue class sharing its column chunks (1 or 2)
    double2* Y;                 // signal b's [P1][P2][r] slab, or [P2][W] residue rows (sum_tail),
                                // at Y + b * y_stride
    uint64_t y_stride;          // elements between consecutive signals' data
    int sum_tail;               // sum tail: no slab, no K2 (see k1_sum_tail)
    uint32_t reducers;          // sum tail: the last `reducers` CTAs of a signal reduce its rows
    unsigned* arrivals;         // signal b's control words at arrivals + b * ctl_stride (zeroed once):
                                // sum tail {tickets, done, ready[P2]}, K2 tail {tickets, done}
    uint64_t ctl_stride;        // words between consecutive signals' control words
    uint64_t in_elems;          // checked builds: elements addressable from a
    uint64_t y_elems;           // checked builds: elements addressable from Y
    uint64_t ctl_words;         // checked builds: words addressable from arrivals
    int k2_tail;                // K2 work done by the last `reducers` CTAs of a signal to write
                                // their slab (last-arrival, no grid-wide wait; see k1_k2_tail)
    uint32_t k2_group;          // k2_tail: columns j per FFT group (the group's Z + scratch fit the ring)
    uint32_t workers;           // K2 worker CTAs per signal riding after the P2 streamers (k1_k2_worker);
                                // the slab then has the two-column-group layout [m1][group][c][j']
    int fused;                  // run K2 in K1's tail behind a grid barrier (cooperative launch)
    unsigned* bar;              // grid-barrier state {count, generation} (workspace header, zeroed once)
    K2Params k2;                // K2 parameters for the fused tail
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

// ring + C slab + P1 twiddles + w (r) + 2*S mbarriers; the ring doubles as the FFT scratch
// (needs r*P1*16 <= the smallest ring)
inline size_t k1_smem_bytes(int r, uint32_t P1, uint32_t stages) {
    const size_t p1 = P1 ? P1 : 1;
    return k1_ring_align_slack(r) + (size_t)stages * k1_stage_bytes(r) + sizeof(double2) * ((size_t)r * p1 + p1 + r) +
           2 * stages * sizeof(uint64_t);
}
// K1 ring depth: as deep as possible while two CTAs still share an SM.
inline uint32_t k1_pick_stages(int r, uint32_t P1) {
    const size_t per_cta = (228 * 1024) / 2 - 1024;
    uint32_t s = K1_MAX_STAGES;
    while (s > (uint32_t)k1_min_stages(r) && k1_smem_bytes(r, P1, s) > per_cta) --s;
    return s;
}
// Z + scratch (r x P2 each) + omega_P2 + four-step twiddles (P2 each)
inline size_t k2_smem_bytes(int r, uint32_t P2) { return sizeof(double2) * (2 * (size_t)r * P2 + 2 * (size_t)P2); }
// ring K2 (k2_ring): three slab buffers (r x P2 each) + omega_P2 + four-step twiddles + 4 mbarriers
inline size_t k2_ring_smem_bytes(int r, uint32_t P2) {
    return sizeof(double2) * (3 * (size_t)r * P2 + 2 * (size_t)P2) + 4 * sizeof(uint64_t);
}
// Z (r x P2) + omega_P2 + four-step twiddles
inline size_t k2_dot_smem_bytes(int r, uint32_t P2) { return sizeof(double2) * ((size_t)r * P2 + 2 * (size_t)P2); }

cudaError_t configure_k1(int r, uint32_t P1, bool mu0);

int k1_max_active_per_sm(int r, uint32_t P1, uint32_t stages, bool mu0);
// Workspace layout (zeroed once by the caller; every kernel leaves it re-armed):
//   [header, 256 B: grid-barrier {count, generation}, status word, unused]
//   per signal b: [control words, padded to 256 B][data: slab or residue rows, padded to 256 B]
// A signal's control words and data sit at the same offsets whatever the batch of the call, so a
// workspace sized for batch B serves any batch <= B (remainder batches).
constexpr size_t kWsHeaderBytes = 256;
constexpr size_t kWsStatusOffset = 8;  // bytes into the header
inline size_t ws_align(size_t b) { return (b + 255) & ~size_t(255); }
// sum-tail scratch in the (idle) ring after the FFT scratch: twiddle tables, per-warp
// reducer partials, ticket
inline size_t k1_sum_scratch_bytes(uint32_t P1, uint32_t P2) {
    return 16 * ((size_t)P1 + P2) + (size_t)K1_THREADS / 32 * 64 * 16 + 16;
}
// r values with a K2-tail K1 instantiation: the long single transforms it pays for (C5: r = 6
// at p = 2^18-2^19; SPEC's pick for N = 2^30 has r = 4).  Other r run the K2 grid.
__host__ __device__ constexpr bool k1_k2_tail_instantiated(int r) { return r >= 4 && r <= 7; }
// r values with a K2-worker K1 instantiation (many-bin single transforms: C2c has r = 14)
__host__ __device__ constexpr bool k1_k2_workers_instantiated(int r) { return r >= 8 && r <= 18; }
// K2 workers: three buffers of one column group (P2 x ceil(r/2)) + omega_P2 + 4 mbarriers
// (+ alignment slack); must fit K1's shared memory
inline size_t k1_k2_worker_bytes(int r, uint32_t P2) {
    return sizeof(double2) * (3 * (size_t)((r + 1) / 2) * P2 + (size_t)P2) + 4 * sizeof(uint64_t) + 128;
}
// K1's last-arrival K2 tail: Z + scratch for `group` columns, omega_P2 + four-step twiddles,
// ticket word
inline size_t k1_k2_tail_bytes(uint32_t group, uint32_t P2) {
    return sizeof(double2) * (2 * (size_t)group * P2 + 2 * (size_t)P2) + 16;
}
cudaError_t configure_k2(int r, uint32_t P2);
cudaError_t launch_k1(const CUtensorMap& map, const K1Params& P, int r, uint32_t batch, bool mu0, cudaStream_t st);
cudaError_t launch_k2(const K2Params& P, int r, uint32_t batch, cudaStream_t st);
cudaError_t launch_k0(const GenParams& G, cudaStream_t st);
cudaError_t launch_naive_dft(const double2* a, uint64_t N, int64_t first, uint64_t count, double2* out,
                             cudaStream_t st);
cudaError_t launch_transpose(const double2* in, double2* out, uint64_t rows, uint64_t cols, cudaStream_t st);

}  // namespace pftdev
