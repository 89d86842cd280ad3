#pragma once
// kernel_templates.cuh -- the sm_100a kernels of transform.execute (Algorithm 2
// PAPER.md:379-395) and the seeded input generator.
//
//  K1  k1_contract_fft<R, MU0>  one CTA per (residue class c mod P2, signal).  A producer
//      warp streams the P1 rows k = c + P2*k1 of A (A[k][l] = a[q k + l])
//      from HBM into a shared-memory ring with 4-D bulk tensor copies (TMA,
//      cp.async.bulk.tensor + mbarrier complete_tx).  Columns are processed in mirror
//      pairs (l, q-l): with B[l][j] = phase_l w_j t_l^j, t_{q-l} = -t_l and
//      phase_{q-l} = conj(phase_l), so a pair contributes t_l^j (b_l + (-1)^j b_{q-l}),
//      b = a * phase -- (3r+10)/2 FP64 ops per element instead of the dense 4r.  A stage
//      is 16 rows x 32 pairs (front box, mirror box) plus the pair-table slice.  Eight
//      consumer warps (16 lanes per row) accumulate, reduce per row by shuffles, and keep
//      the P1 x r slab C_c in shared memory for the first FFT pass:
//      Y_c[m1][j] = sum_k1 C[c + P2 k1][j] e^{-2 pi i m1 k1 / P1}.
//  K2  k2_fft_post<R>           one CTA per m1 in [P1].  Applies the four-step twiddle
//      e^{-2 pi i m1 c / p}, runs the length-P2 FFT over c in shared memory, and evaluates
//      Eq. (7) only at the 2M+1 requested bins (m' = m mod p, m' = m1 + P1 m2):
//      out[m] = e^{-pi i m/p} sum_j Chat[m'][j] ((m - mu)/p)^j.
//      k2_direct_post<R> is the any-P2 fallback (direct sum over c); k2_ring<R> the same pass as
//      a bulk-copy ring on the slab's own layout (isolated single executes, power-of-two p).
//  Inside K1, after the first pass: the sum tail (few bins: K1 finishes the transform itself),
//      the K2 tail (K2's work by the last-arriving CTAs, r = 4..7), or -- k1_contract_fft<R, MU0, 2>,
//      r = 8..18, chained executes -- K2 worker CTAs riding at the end of the grid
//      (k1_k2_worker: the second pass of transform i under the stream of transform i + 1).
//      Short batched signals with one residue class each share a CTA (K1Params.gsig).
//  K0  k0_generate              BASELINE.json synthetic inputs (bench only).
//
// Summation orders are fixed (lane-strided partial sums + xor-butterfly), so results
// are deterministic run to run.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../common/rng.h"
#include "fft_smem.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace pftdev {
namespace cg = cooperative_groups;

// Grid-wide barrier for K1's fused K2 tail (all CTAs are co-resident: cooperative launch).
// Self-resetting: the last arriver zeroes the count and bumps the generation, so the state
// (two words at the end of the workspace, zeroed once) is reusable by the next launch.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_u32(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            atomicExch(count, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (ld_acquire_u32(gen) == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// ----------------------------------------------------------------------------- K1

template <int R>
__device__ __forceinline__ void k2_fft_block(const K2Params& P, uint32_t m1, uint32_t b, double2* zs);

// One TMA stage (a box of K1_BR rows x K1_CP mirror column pairs + the pair table slice)
// into the row accumulators of this lane.  The K1_LANES_PER_ROW lanes of row `rin` are
// li = pl * JS + jh: pair lane pl takes pairs pl, pl + LANES_PER_ROW / JS, ... and j half jh
// accumulates j = jh * H + jj (H = ceil(R / JS), jj < H) with powers t^j formed by
// ascending repeated multiplication from t^{jh H} (the pair table's t^h for jh = 1).
template <int R, int JS, bool MU0, bool FULL>
__device__ __forceinline__ void k1_accumulate_stage(const unsigned char* st, int rin, int li, uint32_t valid,
                                                    double (&are)[(R + JS - 1) / JS],
                                                    double (&aim)[(R + JS - 1) / JS]) {
    constexpr int H = (R + JS - 1) / JS;
    constexpr int PL = K1_LANES_PER_ROW / JS;  // pair lanes per row
    const double2* front = reinterpret_cast<const double2*>(st) + rin * K1_CP;
    const double2* mirror = reinterpret_cast<const double2*>(st + K1_BOX_BYTES) + rin * K1_CP;
    const PairEntry* tab = reinterpret_cast<const PairEntry*>(st + 2 * K1_BOX_BYTES);
    const int pl = li / JS, jh = li % JS;
    // the j parity of jj = 0 is that of jh * H: swap the (sum, difference) roles when odd
    const bool swap = ((jh * H) & 1) != 0;
#pragma unroll
    for (int u = 0; u < K1_CP / PL; ++u) {
        const int i = pl + u * PL;
        // branch-free masking of pairs past the end of the view (keeps the
        // independent pairs in one basic block so their chains interleave)
        const bool ok = FULL || (uint32_t)i < valid;  // FULL: every pair of the chunk is in the view
        const double2 z = make_double2(0.0, 0.0);
        const double2 x1 = ok ? front[i] : z;               // column l
        const double2 x2 = ok ? mirror[K1_CP - 1 - i] : z;  // column q - l
        const double2 cs = *reinterpret_cast<const double2*>(&tab[i].c);
        const double t = tab[i].t;
        const double2 su = make_double2(x1.x + x2.x, x1.y + x2.y);
        const double2 di = make_double2(x1.x - x2.x, x1.y - x2.y);
        double2 Sv, Dv;  // phase_l x1 +/- conj(phase_l) x2
        if constexpr (MU0) {
            Sv = su;
            Dv = di;
        } else {
            Sv = make_double2(fma(cs.x, su.x, -cs.y * di.y), fma(cs.x, su.y, cs.y * di.x));
            Dv = make_double2(fma(cs.x, di.x, -cs.y * su.y), fma(cs.x, di.y, cs.y * su.x));
        }
        if constexpr (JS == 1) {
            are[0] += Sv.x;
            aim[0] += Sv.y;
            double tp = t;
#pragma unroll
            for (int j = 1; j < R; ++j) {
                const double2 v = (j & 1) ? Dv : Sv;  // t^j (b + (-1)^j b')
                are[j] = fma(v.x, tp, are[j]);
                aim[j] = fma(v.y, tp, aim[j]);
                if (j + 1 < R) tp *= t;
            }
        } else {
            const double2 E = swap ? Dv : Sv, O = swap ? Sv : Dv;  // jj even / odd
            double tp = jh ? tab[i].th : 1.0;
#pragma unroll
            for (int jj = 0; jj < H; ++jj) {
                const double2 v = (jj & 1) ? O : E;
                are[jj] = fma(v.x, tp, are[jj]);
                aim[jj] = fma(v.y, tp, aim[jj]);
                if (jj + 1 < H) tp *= t;
            }
        }
    }
}

// End of a row batch: add the row's unpaired columns (l = 0 with t = 1 feeds every j: pair
// lane 0, both j halves; l = q/2 with t = 0 only j = 0: lane li = JS), reduce over the pair
// lanes of the row (fixed xor-butterfly order) and store C[k1][j] = w_j acc_j into Cs[j][k1].
template <int R, int JS, bool MU0>
__device__ __forceinline__ void k1_finish_row(const K1Params& P, double2 xs, int scol, int li, uint32_t k1,
                                              double (&are)[(R + JS - 1) / JS],
                                              double (&aim)[(R + JS - 1) / JS], double2* Cs) {
    constexpr int H = (R + JS - 1) / JS;
    constexpr int PL = K1_LANES_PER_ROW / JS;
    if (scol >= 0) {
        double2 x = xs;
        const bool zero_col = li < JS;  // l = 0; else l = q/2
        if constexpr (!MU0) x = cmul(x, zero_col ? P.phase0 : P.phaseh);
        are[0] += x.x;
        aim[0] += x.y;
        if (zero_col) {
#pragma unroll
            for (int j = 1; j < H; ++j) {
                are[j] += x.x;
                aim[j] += x.y;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
#pragma unroll
        for (int off = K1_LANES_PER_ROW / 2; off >= JS; off >>= 1) {
            are[j] += __shfl_xor_sync(0xffffffffu, are[j], off);
            aim[j] += __shfl_xor_sync(0xffffffffu, aim[j], off);
        }
    }
    const int pl = li / JS, jh = li % JS;
#pragma unroll
    for (int jj = 0; jj < H; ++jj) {
        const int j = jh * H + jj;
        if (k1 < P.rows && j < R && (jj % PL) == pl)
            Cs[(size_t)j * P.rows + k1] = cmul(make_double2(are[jj], aim[jj]), __ldg(P.w + j));  // C = w_j acc_j
    }
}

// ---- tensor-core contraction (k1_tc(R)): one warp = 4 rows of the box ({0, 1, 4, 5} + 8 (w / 2)
// + 2 (w % 2): distinct swizzle chunks) as the 8 m-rows of a DMMA tile (m = 2 * row index +
// part, part 0/1 = re/im); per k-step the 4 k-columns are pairs
// ks * 4 + t4.  A = (b_l + b_{q-l}) parts against the even-moment tile, (b_l - b_{q-l}) parts
// against the odd-moment tile; the MMA sums over the pairs, so only the FP64-pipe moments
// (j = 0, and j = 17 for R = 18) need a cross-lane reduction at the end of the row batch.
__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// Element (row y, pair column j) of a swizzled tensor-core box (two 8-pair halves of
// [32 rows][128 B], 16-byte chunk c of row y stored at chunk c ^ (y & 7)).
__device__ __forceinline__ const double2* tc_box_elt(const unsigned char* box, int y, int j) {
    return reinterpret_cast<const double2*>(box + (j >> 3) * (K1_BR * 128) + y * 128 + (((j & 7) ^ (y & 7)) << 4));
}

// gs: this lane's fragment column g stored at g ^ 2 (pair & 3) (global pair index): the eight
// lanes of a 128-bit load phase (g = 2h, 2h + 1; t4 = 0..3) then read eight distinct chunks.
// The stage holds the two boxes and the fragment slice only (18 KB: four stages fit beside the
// C slab at two CTAs per SM); phases (mu != 0) come from the L1-resident pair table `ptab`
// (this chunk's entries), and t^17 (R = 18) = t^16 t from the pair's own fragment record.
template <int R, bool MU0, bool FULL>
__device__ __forceinline__ void k1_tc_stage(const unsigned char* st, const PairEntry* __restrict__ ptab, int rin,
                                            int part, int t4, int gs, int fsw, uint32_t valid, double (&de)[2],
                                            double (&dd)[2], double& v0, double& vl) {
    const double2* frag = reinterpret_cast<const double2*>(st + 2 * K1_BOX_BYTES);  // [pair][g ^ fsw]
#pragma unroll
    for (int ks = 0; ks < K1_CP / 4; ++ks) {
        const int i = ks * 4 + t4;
        const bool ok = FULL || (uint32_t)i < valid;
        double ae, ao;  // this lane's part of phase_l x1 + conj(phase_l) x2 and of the difference
        const double2* p1 = tc_box_elt(st, rin, i);                                // column l
        const double2* p2 = tc_box_elt(st + K1_BOX_BYTES, rin, K1_CP - 1 - i);     // column q - l
        if constexpr (MU0) {
            const double x1 = ok ? reinterpret_cast<const double*>(p1)[part] : 0.0;
            const double x2 = ok ? reinterpret_cast<const double*>(p2)[part] : 0.0;
            ae = x1 + x2;
            ao = x1 - x2;
        } else {
            const double2 z = make_double2(0.0, 0.0);
            const double2 x1 = ok ? *p1 : z;
            const double2 x2 = ok ? *p2 : z;
            const double2 cs = __ldg(reinterpret_cast<const double2*>(&ptab[i].c));
            const double2 su = make_double2(x1.x + x2.x, x1.y + x2.y);
            const double2 di = make_double2(x1.x - x2.x, x1.y - x2.y);
            ae = part ? fma(cs.x, su.y, cs.y * di.x) : fma(cs.x, su.x, -cs.y * di.y);
            ao = part ? fma(cs.x, di.y, cs.y * su.x) : fma(cs.x, di.x, -cs.y * su.y);
        }
        const double2 b = frag[i * 8 + gs];  // {t^(2+2g), t^(1+2g)}
        dmma_m8n8k4(de, ae, b.x);
        dmma_m8n8k4(dd, ao, b.y);
        v0 += ae;
        if constexpr (R == 18) {  // t^17 = t^16 (g = 7, even) * t (g = 0, odd)
            const double t16 = frag[i * 8 + (7 ^ fsw)].x, t1 = frag[i * 8 + fsw].y;
            vl = fma(ao, t16 * t1, vl);
        }
    }
}

// End of a tensor-core row batch: the unpaired columns (l = 0, t = 1: every j, so every tile
// column of every lane plus the FP64 moments once on t4 = 0; l = q/2, t = 0: j = 0 only, on
// t4 = 1), the 4-lane reduction of the FP64 moments, and the raw moment parts into Cs (the w_j
// factor is applied in one pass after the loop).  Tile column n = 2 t4 + e holds j = 2 + 2n
// (even tile) and j = 1 + 2n (odd tile).
template <int R, bool MU0>
__device__ __forceinline__ void k1_tc_finish_row(const K1Params& P, double2 x0, double2 xh, int part, int t4,
                                                 uint32_t k1, double (&de)[2], double (&dd)[2], double v0,
                                                 double vl, double2* Cs) {
    if constexpr (!MU0) {
        x0 = cmul(x0, P.phase0);
        xh = cmul(xh, P.phaseh);
    }
    const double x0p = part ? x0.y : x0.x, xhp = part ? xh.y : xh.x;  // zero when not in the view
    de[0] += x0p;
    de[1] += x0p;
    dd[0] += x0p;
    dd[1] += x0p;
    if (t4 == 0) {
        v0 += x0p;
        vl += x0p;
    }
    if (t4 == 1) v0 += xhp;
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, off);
        vl += __shfl_xor_sync(0xffffffffu, vl, off);
    }
    if (k1 >= P.rows) return;
    double* cs = reinterpret_cast<double*>(Cs);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int n = 2 * t4 + e, je = 2 + 2 * n, jo = 1 + 2 * n;
        if (je < R) cs[2 * ((size_t)je * P.rows + k1) + part] = de[e];
        if (jo < R) cs[2 * ((size_t)jo * P.rows + k1) + part] = dd[e];
    }
    if (t4 == 0) cs[2 * (size_t)k1 + part] = v0;
    if (R == 18 && t4 == 1) cs[2 * ((size_t)17 * P.rows + k1) + part] = vl;
}

// Sum tail (few output bins, W <= p/4), which replaces K2.  CTA (c, b) writes its residue row
//   S[b][c][s] = e^{-2 pi i (m mod p) c / p} sum_j Y_c[m1][j] x_s^j     (s in [W], x_s = (m - mu)/p,
// m1 = (m mod p) mod P1, powers by repeated multiplication in ascending j as the planner forms
// post_powers), raises the row's ready flag and takes a ticket; the last `reducers` CTAs of
// signal b each sum the P2 rows for a slice of the outputs in a fixed order (bitwise
// deterministic), times e^{-pi i m / p}.  The transform is one kernel: under PDL the next
// transform's K1 streams while these few CTAs finish, which a separate K2 (waiting for all of
// K1) could not allow.
// One entry of CTA c's residue row: e^{-2 pi i (m mod p) c / p} sum_j Y_c[m1][j] x^j at slot so.
template <int R>
__device__ __forceinline__ double2 k1_row_value(const K1Params& P, const double2* res, const double2* twc,
                                                const double2* tw2, uint32_t c, uint64_t so, int64_t Mh,
                                                bool p1_pow2, bool p2_pow2, int lg_p1, bool unit_tw = false) {
    // res: column j of this signal at res + j * P.rows (P.rows = P1 unless the CTA holds several signals)
    // unit_tw: one residue class per signal (c = 0): both twiddles are exactly 1, the tables are not read
    const K2Params& Q = P.k2;
    const uint64_t sr = so < Q.p ? so : (Q.W >> 32) ? so % Q.p : (uint64_t)((uint32_t)so % (uint32_t)Q.p);
    uint32_t mp = (uint32_t)(Q.first_mod_p + sr);
    if (mp >= Q.p) mp -= (uint32_t)Q.p;
    const uint32_t m1 = p1_pow2 ? mp & (P.P1 - 1) : mp % P.P1;
    const uint32_t m2 = p1_pow2 ? mp >> lg_p1 : mp / P.P1;
    const uint32_t e2 = p2_pow2 ? (m2 * c) & (P.P2 - 1) : (m2 * c) % P.P2;  // m2 c < p
    // x = (m - mu)/p; 1/p is exact for power-of-two p (then x^j is bit-identical to the
    // planner's post_powers), else within an ulp
    const double x = (double)((int64_t)so - Mh) * Q.inv_p;
    double2 acc = res[m1];
    double tp = x;
#pragma unroll
    for (int j = 1; j < R; ++j) {  // ascending j, powers by repeated multiplication
        const double2 v = res[(size_t)j * P.rows + m1];
        acc.x = fma(v.x, tp, acc.x);
        acc.y = fma(v.y, tp, acc.y);
        if (j + 1 < R) tp *= x;
    }
    if (unit_tw) return acc;  // cmul(., (1, 0)) is the identity on finite values
    return cmul(cmul(acc, twc[m1]), tw2[e2]);
}

// The small-P2 last-arrival reduction (see `fast` in k1_sum_tail).  Compiled only into the
// tensor-core K1 instantiations (r = 12..18: C3, the 2-D passes): present in the vector-path
// kernels it cost C1 9% and C4 4% though they never take it (same box A/B); out of line
// (__noinline__) the call's stack traffic cost every config 8-35%.
template <int R>
__device__ __forceinline__ void k1_sum_tail_fast(const K1Params& P, const double2* res, uint32_t c, uint32_t b,
                                              const double2* twc, double2* tw2, int64_t Mh, bool p1_pow2,
                                              bool p2_pow2, int lg_p1) {
    constexpr int FAST_OUT = 4, FAST_P2 = 8;
    const K2Params& Q = P.k2;
    const int tid = threadIdx.x, nt = blockDim.x;
    double2* __restrict__ rowc = P.Y + (size_t)b * P.y_stride + (size_t)c * Q.W;
    double2 keep[FAST_OUT];
#pragma unroll
    for (int i = 0; i < FAST_OUT; ++i) {
        const uint64_t so = (uint64_t)tid + (uint64_t)i * nt;
        if (so < Q.W) {
            keep[i] = k1_row_value<R>(P, res, twc, tw2, c, so, Mh, p1_pow2, p2_pow2, lg_p1);
            PFT_BOUND((size_t)b * P.y_stride + (size_t)c * Q.W + so, P.y_elems);
            rowc[so] = keep[i];
        }
    }
    unsigned* ctl = P.arrivals + (size_t)b * P.ctl_stride;  // {tickets, ...}
    PFT_BOUND((size_t)b * P.ctl_stride, P.ctl_words);
    unsigned* s_last = reinterpret_cast<unsigned*>(tw2 + P.P2);
    __syncthreads();  // every row store precedes thread 0's fence and ticket
    if (tid == 0) {
        __threadfence();
        *s_last = atomicAdd(ctl, 1u) == P.P2 - 1;
    }
    __syncthreads();
    if (!*s_last) {
        return;
    }
    __threadfence();  // the other rows were fenced before their tickets (threadFenceReduction)
    const double2* __restrict__ rows = P.Y + (size_t)b * P.y_stride;
#pragma unroll
    for (int i = 0; i < FAST_OUT; ++i) {
        const uint64_t so = (uint64_t)tid + (uint64_t)i * nt;
        if (so < Q.W) {
            double2 v[FAST_P2];
            PFT_BOUND((size_t)b * P.y_stride + (size_t)(P.P2 - 1) * Q.W + so, P.y_elems);
#pragma unroll
            for (int r = 0; r < FAST_P2; ++r)
                v[r] = (uint32_t)r >= P.P2 ? make_double2(0.0, 0.0)
                       : (uint32_t)r == c  ? keep[i]
                                           : __ldcg(rows + (size_t)r * Q.W + so);
            double2 tot = v[0];
#pragma unroll
            for (int r = 1; r < FAST_P2; ++r)
                if ((uint32_t)r < P.P2) tot = cadd(tot, v[r]);  // fixed order c = 0, 1, ...
            const double2 o = cmul(tot, __ldg(Q.post_twiddles + so));  // e^{-pi i m / p}
            PFT_BOUND((size_t)b * Q.W + so, Q.out_elems);
            Q.out[(size_t)b * Q.W + so] = o;
            if (!isfinite(o.x) || !isfinite(o.y)) atomicOr(Q.status, 1);
        }
    }
    if (tid == 0) ctl[0] = 0;  // every CTA of the signal has taken its ticket: re-arm
}

template <int R>
__device__ __forceinline__ void k1_sum_tail(const K1Params& P, const double2* res, uint32_t c, uint32_t b,
                                         unsigned char* scratch, double2 tail_tw) {
    const K2Params& Q = P.k2;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int64_t Mh = (int64_t)((Q.W - 1) / 2);
    const bool p1_pow2 = (P.P1 & (P.P1 - 1)) == 0, p2_pow2 = (P.P2 & (P.P2 - 1)) == 0;
    const int lg_p1 = 31 - __clz(P.P1);
    // omega_p^{(m mod p) c} = omega_p^{m1 c} omega_P2^{m2 c}: both factors from tables in the idle ring
    double2* twc = reinterpret_cast<double2*>(scratch);  // [P1] omega_p^{m1 c}
    double2* tw2 = twc + P.P1;                            // [P2] omega_P2^t
    // One residue class per signal (P2 = 1: short batched signals, e.g. the 2-D passes): the
    // row is the output; no row store, ready flag, ticket or read-back (same arithmetic as a
    // one-row reduction: cadd(0, v) = v), and no twiddle tables (c = 0: every entry is 1).
    const bool direct = P.P2 == 1;
    // entries t < blockDim.x were prefetched during the stream (tail_tw); the rest load now
    if (!direct) {
        for (uint32_t t = tid; t < P.P1 + P.P2; t += nt) {
            double2 v = tail_tw;
            if (t >= (uint32_t)nt) v = __ldg(P.omega + (t < P.P1 ? (size_t)t * c : (size_t)(t - P.P1) * P.P1));  // m1 c < p
            twc[t] = v;  // twc[P1 + t'] is tw2[t']
        }
        __syncthreads();
    }
    // Few residue classes and few outputs (batched short signals, e.g. C3: P2 = 2, W = 513):
    // only the last CTA of the signal to arrive reduces, each thread summing the P2 rows of its
    // own outputs with all loads in flight at once and its own row's values from registers;
    // the others exit at their ticket.  (The general reducers loop over 64-output groups with a
    // block barrier each: at C3 fence + wait + reduce took 10.5 of a CTA's 35.6 us.)
    constexpr int FAST_OUT = 4, FAST_P2 = 8;
    const bool fast = k1_tc(R) && !direct && P.P2 <= FAST_P2 && Q.W <= (uint64_t)FAST_OUT * nt;
    double2* __restrict__ rowc = P.Y + (size_t)b * P.y_stride + (size_t)c * Q.W;
    if constexpr (k1_tc(R)) {
        if (fast) {
            k1_sum_tail_fast<R>(P, res, c, b, twc, tw2, Mh, p1_pow2, p2_pow2, lg_p1);
            return;
        }
    }
    if (direct && P.gsig > 1) {
        // several signals per CTA (P2 = 1, short batched signals): signal g's column j is the
        // g-th length-P1 piece of row-block column j (res + j * rows + g * P1)
        for (uint64_t t = tid; t < Q.W * P.gsig; t += nt) {
            const uint32_t g = (uint32_t)(t / Q.W);
            const uint64_t so = t - (uint64_t)g * Q.W;
            const double2 v = k1_row_value<R>(P, res + (size_t)g * P.P1, twc, tw2, c, so, Mh, p1_pow2, p2_pow2, lg_p1, true);
            const double2 o = cmul(v, __ldg(Q.post_twiddles + so));  // e^{-pi i m / p}
            const size_t at = ((size_t)b * P.gsig + g) * Q.W + so;
            PFT_BOUND(at, Q.out_elems);
            Q.out[at] = o;
            if (!isfinite(o.x) || !isfinite(o.y)) atomicOr(Q.status, 1);
        }
        return;
    }
    for (uint64_t so = tid; so < Q.W; so += nt) {
        const double2 v = k1_row_value<R>(P, res, twc, tw2, c, so, Mh, p1_pow2, p2_pow2, lg_p1, direct);
        if (direct) {
            const double2 o = cmul(v, __ldg(Q.post_twiddles + so));  // e^{-pi i m / p}
            PFT_BOUND((size_t)b * Q.W + so, Q.out_elems);
            Q.out[(size_t)b * Q.W + so] = o;
            if (!isfinite(o.x) || !isfinite(o.y)) atomicOr(Q.status, 1);
        } else {
            PFT_BOUND((size_t)b * P.y_stride + (size_t)c * Q.W + so, P.y_elems);
            rowc[so] = v;
        }
    }
    if (direct) return;
    // publish the row, then take a ticket: the last `reducers` arrivals of signal b reduce
    unsigned* ctl = P.arrivals + (size_t)b * P.ctl_stride;  // {tickets, done, ready[P2]}
    PFT_BOUND((size_t)b * P.ctl_stride + P.P2 + 1, P.ctl_words);
    unsigned* ready = ctl + 2;
    double2* part = tw2 + P.P2;                           // [nw][64] reducer partials
    unsigned* s_ticket = reinterpret_cast<unsigned*>(part + (size_t)nw * 64);
    // the block barrier orders every thread's row stores before thread 0's gpu-scope fence and
    // release (the cooperative-groups grid-sync pattern); one fence instead of one per thread
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        st_release_u32(ready + c, 1u);
        *s_ticket = atomicAdd(ctl, 1u);
    }
    __syncthreads();
    const uint32_t t = *s_ticket, K = P.reducers;
    if (t + K < P.P2) {
        return;
    }
    // Reducer k sums rows c = 0..P2-1 (fixed order per warp: c = warp, warp + nw, ...) for
    // its slice of outputs once the warp's rows are flagged ready (most are by now).
    const uint32_t k = t + K - P.P2;
    const uint64_t s0 = (uint64_t)k * Q.W / K, s1 = (uint64_t)(k + 1) * Q.W / K;
    const double2* __restrict__ rows = P.Y + (size_t)b * P.y_stride;
    // this warp's rows c = warp, warp + nw, ...: all flags checked at once (one lane per row)
    for (uint32_t r = warp + (uint32_t)lane * nw; r < P.P2; r += 32u * nw)
        while (ld_acquire_u32(ready + r) == 0) __nanosleep(32);
    __syncwarp();
    for (uint64_t g0 = s0; g0 < s1; g0 += 64) {  // two 32-output groups per pass
        const uint64_t sa = g0 + lane, sb = g0 + 32 + lane;
        const bool oka = sa < s1, okb = sb < s1;
        double2 acca = make_double2(0.0, 0.0), accb = make_double2(0.0, 0.0);
        for (uint32_t r0 = warp; r0 < P.P2; r0 += 8 * nw) {
            double2 va[8], vb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t r = r0 + u * nw;
                const bool in = r < P.P2;
                if (in && oka) PFT_BOUND((size_t)b * P.y_stride + (size_t)r * Q.W + sa, P.y_elems);
                if (in && okb) PFT_BOUND((size_t)b * P.y_stride + (size_t)r * Q.W + sb, P.y_elems);
                va[u] = (in && oka) ? __ldcg(rows + (size_t)r * Q.W + sa) : make_double2(0.0, 0.0);
                vb[u] = (in && okb) ? __ldcg(rows + (size_t)r * Q.W + sb) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                acca = cadd(acca, va[u]);
                accb = cadd(accb, vb[u]);
            }
        }
        part[warp * 64 + lane] = acca;
        part[warp * 64 + 32 + lane] = accb;
        __syncthreads();
        if (warp < 2) {
            const uint64_t so = g0 + warp * 32 + lane;
            if (so < s1) {
                double2 tot = part[warp * 32 + lane];
                for (int w = 1; w < nw; ++w) tot = cadd(tot, part[w * 64 + warp * 32 + lane]);
                const double2 v = cmul(tot, __ldg(Q.post_twiddles + so));  // e^{-pi i m / p}
                PFT_BOUND((size_t)b * Q.W + so, Q.out_elems);
                Q.out[(size_t)b * Q.W + so] = v;
                if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(Q.status, 1);
            }
        }
        __syncthreads();
    }
    // the last reducer to finish re-arms the signal's counters and flags
    if (tid == 0) *s_ticket = atomicAdd(ctl + 1, 1u) == K - 1;
    __syncthreads();
    if (*s_ticket) {
        for (uint32_t i = tid; i < P.P2; i += nt) ready[i] = 0;
        if (tid == 0) {
            ctl[0] = 0;
            ctl[1] = 0;
        }
        __threadfence();
    }
}

// Last-arrival K2 tail (many output bins, e.g. C2c): K2's work -- the length-P2 pass for one
// m1 pruned to the bins Eq. (7) reads, fused with the post-process -- is done inside K1 by the
// last `reducers` CTAs of signal b to write their slab, not by a separate K2 grid that waits
// for all of K1 (and whose 123 KB CTAs cannot sit beside the next transform's K1 CTAs).  Each
// CTA publishes its slab and takes a ticket; the last L arrivals wait for the ticket count to
// reach P2 (they are the stragglers, so this wait is short), then worker k handles m1 = k,
// k + L, ...  The columns j go through the FFT in groups of `k2_group` so Z + scratch fit the
// idle ring beside two K1 CTAs per SM; a bin's partial sum over j is kept in `out` between
// groups (same thread, same ascending-j fma chain as k2_fft_block: results are bitwise those
// of the standalone K2).  Under PDL the next transform's K1 streams on the other slots.
template <int R>
__device__ __forceinline__ void k1_k2_tail(const K1Params& P, uint32_t c, uint32_t b, double2* zs) {
    const K2Params& Q = P.k2;
    const int tid = threadIdx.x, nt = blockDim.x;
    const uint32_t G = P.k2_group;
    double2* Z = zs;                              // [G][P2]
    double2* scratch = zs + (size_t)G * P.P2;     // [G][P2]
    double2* tw2 = scratch + (size_t)G * P.P2;    // omega_P2^t
    double2* pre = tw2 + P.P2;                    // omega_p^{m1 c}
    unsigned* s_t = reinterpret_cast<unsigned*>(pre + P.P2);
    unsigned* ctl = P.arrivals + (size_t)b * P.ctl_stride;   // {tickets, done}
    PFT_BOUND((size_t)b * P.ctl_stride + 1, P.ctl_words);
    __syncthreads();  // the CTA's slab stores precede thread 0's fence and ticket
    if (tid == 0) {
        __threadfence();
        *s_t = atomicAdd(ctl, 1u);
    }
    __syncthreads();
    const uint32_t t = *s_t, L = P.reducers;
    if (t + L < P.P2) return;
    const uint32_t k = t + L - P.P2;
    double2* __restrict__ out = Q.out + (size_t)b * Q.W;
    // Per m1, a thread's first bin s = s0 + P1 tid takes its r post powers and post twiddle from
    // registers loaded before the slab (these tables come from DRAM: the next transform's
    // stream has evicted them; a dependent load per j serialised ~r DRAM latencies).  The
    // first m1's tables load before the wait for the stragglers.
    double pw0[R];
    double2 ptw0 = make_double2(0.0, 0.0);
    auto prefetch = [&](uint32_t m1) {
        const uint64_t s0 = (uint64_t)((m1 + P.P1 - Q.first_mod_p1) % P.P1);
        for (uint32_t c2 = tid; c2 < P.P2; c2 += nt) pre[c2] = __ldg(P.omega + (size_t)m1 * c2);  // m1 c < p
        const uint64_t sf = s0 + (uint64_t)P.P1 * tid;
        if (sf < Q.W) {
#pragma unroll
            for (int j = 0; j < R; ++j) pw0[j] = __ldg(Q.post_powers + sf * R + j);
            ptw0 = __ldg(Q.post_twiddles + sf);
        }
    };
    for (uint32_t c2 = tid; c2 < P.P2; c2 += nt) tw2[c2] = __ldg(P.omega + (size_t)c2 * P.P1);  // omega_P2^c
    if (k < P.P1) prefetch(k);
    if (tid == 0) {
        while (ld_acquire_u32(ctl) < P.P2) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
    for (uint32_t m1 = k; m1 < P.P1; m1 += L) {
        const uint64_t s0 = (uint64_t)((m1 + P.P1 - Q.first_mod_p1) % P.P1);
        if (s0 >= Q.W) continue;  // no output slot maps to this m1 (block-uniform)
        if (m1 != k) {
            prefetch(m1);
            __syncthreads();
        }
        const double2* __restrict__ Ym = P.Y + (size_t)b * P.y_stride + (size_t)m1 * P.P2 * R;
        for (uint32_t j0 = 0; j0 < (uint32_t)R; j0 += G) {
            const uint32_t g = min(G, (uint32_t)R - j0), n = P.P2 * g;
            // Z[jj][c] = omega_p^{m1 c} Y[c][j0 + jj]; all of a thread's L2 loads in flight first
            constexpr int U = 8;
            for (uint32_t base = tid; base < n; base += U * nt) {
                double2 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t idx = base + u * nt;
                    const uint32_t cc = idx / g, jj = idx - cc * g;
                    if (idx < n) PFT_BOUND((size_t)b * P.y_stride + (size_t)m1 * P.P2 * R + (size_t)cc * R + j0 + jj, P.y_elems);
                    v[u] = idx < n ? __ldcg(Ym + (size_t)cc * R + j0 + jj) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t idx = base + u * nt;
                    if (idx < n) {
                        const uint32_t cc = idx / g, jj = idx - cc * g;
                        Z[(size_t)jj * P.P2 + cc] = (m1 == 0 || cc == 0) ? v[u] : cmul(v[u], pre[cc]);
                    }
                }
            }
            __syncthreads();
            const double2* res = Z;
            if (P.P2 > 1) res = fft_columns(Z, scratch, (int)g, Q.fft2, SmemTwiddles{tw2});
            const bool last = j0 + g == (uint32_t)R;
            const uint64_t sf = s0 + (uint64_t)P.P1 * tid;
            for (uint64_t s = sf; s < Q.W; s += (uint64_t)P.P1 * nt) {
                uint64_t mp = Q.first_mod_p + s % Q.p;
                if (mp >= Q.p) mp -= Q.p;
                const uint32_t m2 = (uint32_t)(mp / P.P1);
                const bool first = s == sf;
                double2 acc = j0 == 0 ? make_double2(0.0, 0.0) : out[s];  // this thread's partial
#pragma unroll
                for (int j = 0; j < R; ++j) {  // ascending j, this group's columns
                    if ((uint32_t)j < j0 || (uint32_t)j >= j0 + g) continue;
                    const double pw = first ? pw0[j] : __ldg(Q.post_powers + s * R + j);
                    const double2 v = res[(size_t)(j - j0) * P.P2 + m2];
                    acc.x = fma(v.x, pw, acc.x);
                    acc.y = fma(v.y, pw, acc.y);
                }
                if (last) {
                    acc = cmul(acc, first ? ptw0 : __ldg(Q.post_twiddles + s));  // e^{-pi i m / p}
                    if (!isfinite(acc.x) || !isfinite(acc.y)) atomicOr(Q.status, 1);
                }
                PFT_BOUND((size_t)b * Q.W + s, Q.out_elems);
                out[s] = acc;
            }
            __syncthreads();  // Z / scratch reuse by the next group or m1
        }
    }
    // the last worker to finish re-arms the signal's counters
    if (tid == 0 && atomicAdd(ctl + 1, 1u) == L - 1) {
        ctl[0] = 0;
        ctl[1] = 0;
        __threadfence();
    }
}

// One Stockham stage of the ring K2 on the slab's own layout: element (c, j) at c * R + j, the
// R columns of a point travelling together.  Work item idx = jj * R + j (j fastest): its RAD
// loads src[idx + r * nb * R] are contiguous across a warp; the stores are contiguous in runs of
// Ns * R elements (the first stage's, Ns = 1, in runs of R).  Same butterflies, twiddles and
// order as stockham_stage_fixed, so a column's result is bitwise the one the K2 grid computes.
// pre: four-step twiddles omega_p^{m1 c} folded into the first stage's loads (null = none).
template <int RAD, int R>
__device__ __forceinline__ void k2_ring_stage(const double2* __restrict__ src, double2* __restrict__ dst, int n, int Ns,
                                              int lg_ns, const double2* __restrict__ tw, const double2* __restrict__ pre,
                                              int t0, int nt) {
    const int nb = n / RAD;
    const uint32_t tstride = (uint32_t)(n / (Ns * RAD));
    for (int idx = t0; idx < nb * R; idx += nt) {
        const int jj = idx / R, j = idx - jj * R;
        const int k = jj & (Ns - 1);
        const int base = ((jj >> lg_ns) << lg_ns) * RAD + k;
        double2 v[RAD];
#pragma unroll
        for (int r = 0; r < RAD; ++r) v[r] = src[idx + r * nb * R];
        if (pre) {
#pragma unroll
            for (int r = 0; r < RAD; ++r) {
                const int c = jj + r * nb;
                if (c != 0) v[r] = cmul(v[r], pre[c]);
            }
        }
        if (k != 0) {
#pragma unroll
            for (int r = 1; r < RAD; ++r) v[r] = cmul(v[r], tw[(uint32_t)(k * r) * tstride]);
        }
        if constexpr (RAD == 2) dft2(v[0], v[1]);
        if constexpr (RAD == 4) dft4(v[0], v[1], v[2], v[3]);
        if constexpr (RAD == 8) dft8(v);
        if constexpr (RAD == 16) dft16(v);
#pragma unroll
        for (int r = 0; r < RAD; ++r) dst[(base + r * Ns) * R + j] = v[r];
    }
}

// K2 worker CTAs inside K1's grid (chained executes of one long transform with many bins: C2c).
// The grid carries `workers` extra CTAs after the P2 streaming CTAs.  They are dispatched last, so
// they land in the SM slots the streamers leave free (C2c: 256 streamers + 40 workers = the 296
// slots), release the next launch at once, and wait for the slab counter to reach P2 (each
// streamer bumps it after its slab store).  Then worker w runs K2 for m1 = w, w + workers, ...
// as a bulk-copy ring: the slab is stored in two column groups per m1 ([m1][group][c][j'],
// already multiplied by the four-step twiddles omega_p^{m1 c}) so a group (P2 x ceil(R/2) complex128) is one contiguous cp.async.bulk,
// issued by the CTA's ninth warp (K1's producer/consumer pattern: full/empty mbarriers) into one of
// two load buffers while the eight consumer warps work on the other; the length-P2 stages (radix
// 8/4/2: the CTA keeps K1's register budget) ping-pong between the load buffer and a scratch
// buffer on the group's own (c, j') layout, and a bin's Eq. (7) sum continues in registers from the first group into the
// second (one ascending-j fma chain).  With one kernel per execute the next transform's K1 is a
// direct programmatic dependent of this one: its streamers take the streamers' slots as they exit
// and stream while these workers finish -- a separate K2 kernel between two K1s cost the chain
// ~7 us even when empty (profiles/r02/ab_ring_k2.jsonl).  The next K1 writes the slab only after
// its griddepcontrol.wait, i.e. after every worker here has exited.
template <int R>
__device__ __forceinline__ void k1_k2_worker(const K1Params& P, uint32_t w, uint32_t b, unsigned char* smem) {
    const K2Params& Q = P.k2;
    constexpr int G0 = (R + 1) / 2, G1 = R - G0, NG = G1 > 0 ? 2 : 1;
    constexpr int NOUT = 2;   // bins per consumer thread and m1 (host: ceil(W / P1) <= NOUT * NT)
    constexpr int NT = 32 * K1_CONSUMER_WARPS;  // consumer threads (warps 0..7); warp 8 loads
    constexpr uint32_t kSpinLimit = 1u << 22;   // bounded waits: a lost signal becomes status bit 2, not a hang
    const int tid = threadIdx.x;
    const uint32_t n = P.P2, cap = n * (uint32_t)G0;
    double2* bufs = reinterpret_cast<double2*>(smem);     // [3][cap]: load buffers 0 and 1, FFT scratch 2
    double2* tw2 = bufs + 3 * (size_t)cap;                // omega_P2^t
    uint64_t* full = reinterpret_cast<uint64_t*>(tw2 + n);  // [2] slab group landed
    uint64_t* empty = full + 2;                              // [2] load buffer consumed
    unsigned* ctl = P.arrivals + (size_t)b * P.ctl_stride;  // {slabs stored, workers done}
    PFT_BOUND((size_t)b * P.ctl_stride + 1, P.ctl_words);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t NW = P.workers;
    const uint32_t nk = w < P.P1 ? (P.P1 - w + NW - 1) / NW : 0;
    const uint32_t nq = nk * NG;  // (m1, group) steps, in order
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    if (tid < NT && nk > 0)
        for (uint32_t c = tid; c < n; c += NT) tw2[c] = __ldg(P.omega + (size_t)c * P.P1);
    // the previous grid (the workers of the previous transform re-arm this signal's counters as
    // they finish, and read the slab this transform's streamers rewrite) must be complete first
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();  // barriers and tables ready; the two roles part here
    if (tid >= NT) {
        // ---- loader warp: one lane waits for the slab, then keeps two groups in flight
        if (tid == NT && nq > 0) {
            uint32_t spins = 0;
            while (ld_acquire_u32(ctl) < P.P2) {
                __nanosleep(256);
                if (++spins > kSpinLimit) {
                    atomicOr(Q.status, 2);
                    break;
                }
            }
            __threadfence();
            asm volatile("fence.proxy.async;" ::: "memory");  // the streamers' slab stores before the bulk reads
            const double2* __restrict__ Yb = P.Y + (size_t)b * P.y_stride;
            for (uint32_t q = 0; q < nq; ++q) {
                const uint32_t lb = q & 1u;
                if (q >= 2) {  // the consumers have finished with this buffer's previous group
                    const uint32_t par = ((q >> 1) - 1u) & 1u;
                    spins = 0;
                    while (!mbar_try_wait(&empty[lb], par))
                        if (++spins > kSpinLimit) {
                            atomicOr(Q.status, 2);
                            break;
                        }
                }
                const uint32_t m1 = w + (q / NG) * NW, g = q % NG;
                const uint32_t bytes = n * (uint32_t)(g ? G1 : G0) * (uint32_t)sizeof(double2);
                const size_t off = (size_t)m1 * n * R + (g ? (size_t)n * G0 : 0);
                PFT_BOUND((size_t)b * P.y_stride + off + bytes / sizeof(double2) - 1, P.y_elems);
                mbar_arrive_expect_tx(&full[lb], bytes);
                bulk_load(bufs + (size_t)lb * cap, Yb + off, bytes, &full[lb]);
            }
        }
    } else if (nq > 0) {
        // ---- consumers (named barrier 1 over the NT consumer threads)
        auto team_sync = [] { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); };
        const int lg_n = 31 - __clz((int)n);  // radix schedule of the power-of-two P2: 8s, then one 4 or 2
        const int64_t Mh = (int64_t)((Q.W - 1) / 2);
        double2* __restrict__ out = Q.out + (size_t)b * Q.W;
        double2 acc[NOUT];
        double tp[NOUT];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
            acc[o] = make_double2(0.0, 0.0);
            tp[o] = 0.0;
        }
        for (uint32_t q = 0; q < nq; ++q) {
            const uint32_t m1 = w + (q / NG) * NW, g = q % NG, lb = q & 1u;
            const uint64_t s0 = (uint64_t)((m1 + P.P1 - Q.first_mod_p1) % P.P1);
            {
                uint32_t spins = 0;
                while (!mbar_try_wait(&full[lb], (q >> 1) & 1u))
                    if (++spins > kSpinLimit) {
                        atomicOr(Q.status, 2);
                        break;
                    }
            }
            double2* src = bufs + (size_t)lb * cap;
            double2* dst = bufs + 2 * (size_t)cap;
            int Ns = 1, lg_ns = 0;
            while (lg_ns < lg_n) {
                const int lgr = lg_n - lg_ns >= 3 ? 3 : lg_n - lg_ns, RAD = 1 << lgr;
                const double2* pr = nullptr;  // the streamers stored the slab with its four-step twiddles
                if (g == 0) {
                    if (RAD == 8) k2_ring_stage<8, G0>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT);
                    else if (RAD == 4) k2_ring_stage<4, G0>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT);
                    else k2_ring_stage<2, G0>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT);
                } else if constexpr (G1 > 0) {
                    if (RAD == 8) k2_ring_stage<8, G1>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT);
                    else if (RAD == 4) k2_ring_stage<4, G1>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT);
                    else k2_ring_stage<2, G1>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT);
                }
                lg_ns += lgr;
                Ns *= RAD;
                team_sync();
                double2* t = src;
                src = dst;
                dst = t;
            }
            const int gw = g ? G1 : G0, j0 = g ? G0 : 0;
#pragma unroll
            for (int o = 0; o < NOUT; ++o) {
                const uint64_t s = s0 + (uint64_t)P.P1 * (tid + o * NT);
                if (s >= Q.W) continue;
                uint64_t mp = Q.first_mod_p + s % Q.p;
                if (mp >= Q.p) mp -= Q.p;
                const uint32_t m2 = (uint32_t)(mp / P.P1);
                const double x = (double)((int64_t)s - Mh) * Q.inv_p;
                const double2* rv = src + (size_t)m2 * gw;
                double2 a = acc[o];
                double t = tp[o];
#pragma unroll
                for (int jj = 0; jj < G0; ++jj) {  // ascending j, this group's columns
                    if (jj >= gw) break;
                    const double2 v = rv[jj];
                    if (j0 + jj == 0) {
                        a = v;
                        t = x;
                    } else {
                        a.x = fma(v.x, t, a.x);
                        a.y = fma(v.y, t, a.y);
                        if (j0 + jj + 1 < R) t *= x;
                    }
                }
                acc[o] = a;
                tp[o] = t;
                if (g == NG - 1) {
                    const double2 v = cmul(a, __ldg(Q.post_twiddles + s));  // e^{-pi i m / p}
                    PFT_BOUND((size_t)b * Q.W + s, Q.out_elems);
                    out[s] = v;
                    if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(Q.status, 1);
                }
            }
            // this step's reads and writes of the load buffer precede its asynchronous refill
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            team_sync();  // also: the scratch is free for the next step
            if (tid == 0) mbar_arrive(&empty[lb]);
        }
    }
    __syncthreads();
    // the last worker to finish re-arms the signal's counters
    if (tid == 0 && atomicAdd(ctl + 1, 1u) == NW - 1) {
        ctl[0] = 0;
        ctl[1] = 0;
        __threadfence();
    }
}

template <int R, bool MU0, int TK = 0>
__global__ void __launch_bounds__(K1_THREADS, 2) k1_contract_fft(const __grid_constant__ CUtensorMap tmap,
                                                                  const K1Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t S = P.stages;
    unsigned char* ring = smem_raw;                                                     // [S] stages
    constexpr uint32_t STAGE = k1_stage_bytes(R);
    if constexpr (k1_ring_align_slack(R) > 0)  // swizzled TMA destinations: 1024-byte aligned ring
        ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    double2* Cs = reinterpret_cast<double2*>(smem_raw + k1_ring_align_slack(R) + (size_t)S * STAGE);  // [R][P1]
    double2* tw1 = Cs + (size_t)R * P.rows;                                              // omega_P1^t
    double2* wsm = tw1 + P.rows;                                                         // w_j (tensor-core path)
    uint64_t* full = reinterpret_cast<uint64_t*>(wsm + R);
    uint64_t* empty = full + S;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if constexpr (TK == 2) {  // K2 worker CTAs ride at the end of the grid (see k1_k2_worker)
        const uint32_t streamers = P.P2 * (P.split > 1 ? P.split : 1);
        if (P.workers && blockIdx.x >= streamers) {
            unsigned char* wbase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
            k1_k2_worker<R>(P, blockIdx.x - streamers, blockIdx.y, wbase);
            return;
        }
    }
    if (tid == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], K1_CONSUMER_WARPS);
        }
        fence_barrier_init();
    }
    __syncthreads();  // barriers initialised: the producer starts streaming immediately
    // sum tail: this thread's entry of the tail's twiddle tables, fetched now so its latency
    // hides behind the stream (entry t < P1: omega_p^{t c}; P1 <= t < P1 + P2: omega_P2^{t - P1})
    // split > 1 (an isolated transform): a cluster of `split` CTAs per residue class, CTA `rank`
    // streaming its share of the column chunks; the shares' C slabs are summed over DSMEM below
    const uint32_t split = P.split > 1 ? P.split : 1;
    const uint32_t rank = blockIdx.x % split;
    const uint32_t c = blockIdx.x / split;  // residue class k = c (mod P2)
    const uint32_t b = blockIdx.y;          // signal
    double2 tail_tw = make_double2(0.0, 0.0);
    if constexpr (TK == 2) {  // K2 workers: the four-step twiddle omega_p^{m1 c} of this class, applied at the slab store
        if (P.workers && (uint32_t)tid < P.P1) tail_tw = __ldg(P.omega + (size_t)tid * (blockIdx.x / (P.split > 1 ? P.split : 1)));
    }
    if (P.sum_tail && (uint32_t)tid < P.P1 + P.P2) {
        const uint32_t t = tid;
        tail_tw = __ldg(P.omega + (t < P.P1 ? (size_t)t * c : (size_t)(t - P.P1) * P.P1));
    }
    const uint32_t npairs = P.gp_end > P.gp0 ? P.gp_end - P.gp0 : 0;
    const uint32_t nch_all = (npairs + K1_CP - 1) / K1_CP;
    const uint32_t ch_lo = (uint32_t)((uint64_t)nch_all * rank / split), ch_hi = (uint32_t)((uint64_t)nch_all * (rank + 1) / split);
    const uint32_t nch = ch_hi - ch_lo;  // this CTA's chunks [ch_lo, ch_hi) of every row
    const uint32_t nrb = (P.rows + K1_BR - 1) / K1_BR;
    const uint32_t total = nch * nrb;

    if (warp == K1_CONSUMER_WARPS) {
        // ---- producer: one elected lane streams front/mirror boxes + table slices
        if (lane == 0 && total > 0) {
            prefetch_tensormap(&tmap);
            uint32_t s = 0, ph = 0, rb = 0, ch = ch_lo;  // slot, its phase; row batch, chunk
            for (uint32_t it = 0; it < total; ++it) {
                if (it >= S) mbar_wait(&empty[s], ph ^ 1u);
                unsigned char* st = ring + (size_t)s * STAGE;
                mbar_arrive_expect_tx(&full[s], k1_stage_data_bytes(R));
                const int row0 = (int)(rb * K1_BR);
                const int f0 = P.fcol0 + (int)(ch * K1_CP);
                const int m0 = P.mcol0 - (int)(ch * K1_CP) - (K1_CP - 1);  // may be < 0: zero fill
                if constexpr (k1_tc(R)) {  // 8-pair swizzled halves
                    constexpr int HB = K1_BR * 128;
                    tma_load_4d(st, &tmap, 2 * f0, (int)c, row0, (int)b, &full[s]);
                    tma_load_4d(st + HB, &tmap, 2 * (f0 + 8), (int)c, row0, (int)b, &full[s]);
                    tma_load_4d(st + K1_BOX_BYTES, &tmap, 2 * m0, (int)c, row0, (int)b, &full[s]);
                    tma_load_4d(st + K1_BOX_BYTES + HB, &tmap, 2 * (m0 + 8), (int)c, row0, (int)b, &full[s]);
                } else {
                    tma_load_4d(st, &tmap, 2 * f0, (int)c, row0, (int)b, &full[s]);
                    tma_load_4d(st + K1_BOX_BYTES, &tmap, 2 * m0, (int)c, row0, (int)b, &full[s]);
                }
                if constexpr (k1_tc(R))
                    bulk_load(st + 2 * K1_BOX_BYTES, P.tcfrag + (size_t)(P.gp0 + ch * K1_CP) * 8, K1_TC_BYTES, &full[s]);
                else
                    bulk_load(st + 2 * K1_BOX_BYTES, P.pairtab + P.gp0 + ch * K1_CP, K1_TAB_BYTES, &full[s]);
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
                if (++ch == ch_hi) {
                    ch = ch_lo;
                    ++rb;
                }
            }
        }
    } else {
        // ---- consumers: K1_LANES_PER_ROW lanes per row, each taking pairs li + k*LANES_PER_ROW
        // FFT twiddles omega_P1^t = omega_p^{t P2} for the tail, staged while the first
        // TMA boxes are in flight (read after the __syncthreads that ends the main loop)
        for (uint32_t t = tid; t < P.P1; t += K1_CONSUMER_WARPS * 32) tw1[t] = __ldg(P.omega + (size_t)t * P.P2);
        if constexpr (k1_tc(R))
            for (uint32_t t = tid; t < (uint32_t)R; t += K1_CONSUMER_WARPS * 32) wsm[t] = __ldg(P.w + t);
        if constexpr (k1_tc(R)) {
            const int g = lane >> 2, t4 = lane & 3, part = g & 1, rr = g >> 1;
            // row within the box: the 16 lanes of a 64-bit load phase (rr = 0, 1) take rows y and
            // y + 4, whose swizzled chunks differ in bit 2 (conflict-free operand loads)
            const int rin = 8 * (warp >> 1) + 2 * (warp & 1) + 4 * (rr & 1) + (rr >> 1);
            const int fsw = 2 * (int)((P.gp0 + (uint32_t)t4) & 3u);  // fragment-table swizzle of this lane's pairs
            uint32_t s = 0, ph = 0;
            for (uint32_t rb = 0; rb < nrb; ++rb) {
                double de[2] = {0.0, 0.0}, dd[2] = {0.0, 0.0}, v0 = 0.0, vl = 0.0;
                const uint32_t k1 = rb * K1_BR + rin;
                // unpaired columns l = 0 (all lanes) and l = q/2 (t4 = 1): loads issued now,
                // consumed after the chunk loop
                double2 x0 = make_double2(0.0, 0.0), xh = make_double2(0.0, 0.0);
                if (k1 < P.rows && rank == 0) {
                    const double2* row = P.a + (size_t)b * P.batch_stride + ((size_t)c + (size_t)P.P2 * k1) * P.row_stride;
                    PFT_BOUND((size_t)b * P.batch_stride + ((size_t)c + (size_t)P.P2 * k1) * P.row_stride +
                                  (size_t)max(P.single0_col, P.singleh_col), P.in_elems);
                    if (P.single0_col >= 0) x0 = __ldg(row + P.single0_col);
                    if (t4 == 1 && P.singleh_col >= 0) xh = __ldg(row + P.singleh_col);
                }
                for (uint32_t ch = ch_lo; ch < ch_hi; ++ch) {
                    mbar_wait(&full[s], ph);
                    __syncwarp();
                    const uint32_t valid = min((uint32_t)K1_CP, npairs - ch * K1_CP);
                    const unsigned char* stage = ring + (size_t)s * STAGE;
                    const PairEntry* ptab = P.pairtab + P.gp0 + ch * K1_CP;
                    if (valid == (uint32_t)K1_CP)
                        k1_tc_stage<R, MU0, true>(stage, ptab, rin, part, t4, g ^ fsw, fsw, valid, de, dd, v0, vl);
                    else
                        k1_tc_stage<R, MU0, false>(stage, ptab, rin, part, t4, g ^ fsw, fsw, valid, de, dd, v0, vl);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                k1_tc_finish_row<R, MU0>(P, x0, xh, part, t4, k1, de, dd, v0, vl, Cs);
            }
        } else {
        constexpr int JS = k1_js(R, MU0), H = (R + JS - 1) / JS;
        const int li = lane & (K1_LANES_PER_ROW - 1);
        const int rin = (warp * 32 + lane) / K1_LANES_PER_ROW;  // row within the box
        uint32_t s = 0, ph = 0;                                  // ring slot and its phase
        for (uint32_t rb = 0; rb < nrb; ++rb) {
            double are[H], aim[H];
#pragma unroll
            for (int j = 0; j < H; ++j) are[j] = aim[j] = 0.0;
            const uint32_t k1 = rb * K1_BR + rin;
            // unpaired columns (l = 0 on the lanes li < JS, l = q/2 on li = JS): issue the load
            // now, consume it after the chunk loop so its DRAM latency is hidden
            const int scol = rank != 0 ? -1 : li < JS ? P.single0_col : (li == JS ? P.singleh_col : -1);
            double2 xs = make_double2(0.0, 0.0);
            if (k1 < P.rows && scol >= 0) {
                PFT_BOUND((size_t)b * P.batch_stride + ((size_t)c + (size_t)P.P2 * k1) * P.row_stride + scol, P.in_elems);
                xs = __ldg(P.a + (size_t)b * P.batch_stride + ((size_t)c + (size_t)P.P2 * k1) * P.row_stride + scol);
            }
            for (uint32_t ch = ch_lo; ch < ch_hi; ++ch) {
                mbar_wait(&full[s], ph);
                // Reconverge before touching the stage: lane 0's `empty` arrive below leaves
                // the warp diverged, and reading a stage from a diverged warp was observed to
                // return corrupt rows on B200 when two K1 CTAs share an SM.
                __syncwarp();
                // full chunks skip the per-pair masking (selects and zero moves were about as
                // many instructions as the FP64 work); only a row's last chunk can be partial
                const uint32_t valid = min((uint32_t)K1_CP, npairs - ch * K1_CP);
                const unsigned char* stage = ring + (size_t)s * STAGE;
                if (valid == (uint32_t)K1_CP)
                    k1_accumulate_stage<R, JS, MU0, true>(stage, rin, li, valid, are, aim);
                else
                    k1_accumulate_stage<R, JS, MU0, false>(stage, rin, li, valid, are, aim);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);  // stage s may be refilled
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            k1_finish_row<R, JS, MU0>(P, xs, scol, li, k1, are, aim, Cs);
        }
        }  // vector path
    }
    // All of A has been read: let K2 (launched with programmatic stream serialization)
    // get scheduled and run its prologue while this grid finishes its FFT tail.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __syncthreads();
    if (split > 1) {
        // the cluster's shares of C_c: rank 0 adds rank 1's slab from distributed shared memory
        // (fixed order: own + remote), then rank 1 leaves; rank 0 runs the FFT pass and the tail
        cg::cluster_group cluster = cg::this_cluster();
        cluster.sync();
        if (rank == 0) {
            const double2* remote = cluster.map_shared_rank(Cs, 1u);
            for (uint32_t idx = tid; idx < (uint32_t)R * P.rows; idx += blockDim.x) Cs[idx] = cadd(Cs[idx], remote[idx]);
        }
        cluster.sync();  // rank 1's shared memory stays alive until rank 0 has read it
        if (rank != 0) return;
    }
    // C = w_j acc_j: the vector path applies w_j at the row store; the tensor-core path folds
    // it into the first FFT stage's loads (or one pass when there is no FFT)
    if (k1_tc(R) && P.P1 <= 1) {
        for (uint32_t idx = tid; idx < (uint32_t)R * P.rows; idx += blockDim.x) Cs[idx] = cmul(Cs[idx], wsm[idx / P.rows]);
        __syncthreads();
    }

    // First FFT pass over k1 (length P1) for every column j, in shared memory; the ring is
    // idle now and serves as the Stockham scratch buffer.
    const double2* res = Cs;
    // (several signals per CTA: the row block's column j is gsig columns of length P1, one per signal)
    if (P.P1 > 1)
        res = fft_columns(Cs, reinterpret_cast<double2*>(ring), R * (int)P.gsig, P.fft, SmemTwiddles{tw1}, BlockTeam{},
                          k1_tc(R) ? static_cast<const double2*>(wsm) : nullptr, (int)P.gsig);
    // K1 is launched with programmatic stream serialization, so it may run while the previous
    // kernel of the stream (K2 of the previous transform, which may still read this
    // workspace) drains: wait for it only here, right before overwriting the slab.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (P.sum_tail) {
        k1_sum_tail<R>(P, res, c, b, ring + (size_t)R * P.rows * sizeof(double2), tail_tw);
        return;
    }
    // Y[b][m1][c][j]: the slab for one m1 is contiguous over (c, j) for K2.
    double2* __restrict__ Y = P.Y + (size_t)b * P.y_stride;
    if constexpr (TK == 2) {
        if (P.workers) {
            // two column groups per m1, each contiguous over (c, j') for the workers' bulk copies
            // and already carrying the four-step twiddle omega_p^{m1 c} (host: P1 <= K1_THREADS)
            constexpr uint32_t G0 = (R + 1) / 2, G1 = R - G0;
            if ((uint32_t)tid < P.P1) tw1[tid] = tail_tw;  // the first pass no longer needs omega_P1
            __syncthreads();
            for (uint32_t idx = tid; idx < (uint32_t)R * P.P1; idx += blockDim.x) {
                const uint32_t m1 = idx / R, j = idx - m1 * R;
                const size_t at = (size_t)m1 * P.P2 * R +
                                  (j < G0 ? (size_t)c * G0 + j : (size_t)P.P2 * G0 + (size_t)c * G1 + (j - G0));
                PFT_BOUND((size_t)b * P.y_stride + at, P.y_elems);
                const double2 v = res[(size_t)j * P.P1 + m1];
                Y[at] = (m1 == 0 || c == 0) ? v : cmul(v, tw1[m1]);
            }
            __syncthreads();  // the CTA's slab stores precede thread 0's fence and count
            if (tid == 0) {
                __threadfence();
                PFT_BOUND((size_t)b * P.ctl_stride, P.ctl_words);
                atomicAdd(P.arrivals + (size_t)b * P.ctl_stride, 1u);
            }
            return;
        }
    }
    for (uint32_t idx = tid; idx < (uint32_t)R * P.P1; idx += blockDim.x) {
        const uint32_t m1 = idx / R, j = idx - m1 * R;
        PFT_BOUND((size_t)b * P.y_stride + ((size_t)m1 * P.P2 + c) * R + j, P.y_elems);
        Y[((size_t)m1 * P.P2 + c) * R + j] = res[(size_t)j * P.P1 + m1];
    }
    // the K2 tail lives in its own instantiations (K2T, k1_k2_tail_instantiated(R)): its code in
    // every K1 cost C2b 2% (same-box A/B: 43.0 vs 42.2 us) though C2b never takes it
    if constexpr (TK == 1) {
        if (P.k2_tail) {
            k1_k2_tail<R>(P, c, b, reinterpret_cast<double2*>(ring));
            return;
        }
    }
    if (P.fused) {
        // Fused K2: once every residue's slab is in L2, CTA (c, b) finishes bins m1 = c,
        // c + P2, ... of signal b; the other CTAs exit and free their SM slots for the next
        // transform's K1 (already launched under PDL).
        grid_barrier(P.bar, P.bar + 1, gridDim.x * gridDim.y);
        for (uint32_t m1 = c; m1 < P.P1; m1 += P.P2)
            k2_fft_block<R>(P.k2, m1, b, reinterpret_cast<double2*>(ring));
    }
}

// ----------------------------------------------------------------------------- K2

// Z[j][c] = omega_p^{m1 c} Y[c][j] for the CTA's m1 slab: all of a thread's loads are
// issued before any is consumed (the slab comes from L2 right after K1; a dependent
// load per iteration made K2's time grow with r).
template <int R>
__device__ __forceinline__ void load_twiddled_slab(const double2* __restrict__ Y, uint32_t P2, uint32_t m1,
                                                   const double2* pre, double2* Z) {
    constexpr int U = 8;
    const uint32_t n = P2 * (uint32_t)R;
    for (uint32_t base = threadIdx.x; base < n; base += U * blockDim.x) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t idx = base + u * blockDim.x;
            v[u] = idx < n ? Y[idx] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t idx = base + u * blockDim.x;
            if (idx < n) {
                const uint32_t c = idx / R, j = idx - c * R;
                Z[(size_t)j * P2 + c] = (m1 == 0 || c == 0) ? v[u] : cmul(v[u], pre[c]);
            }
        }
    }
}

// K2 body for one (m1, signal): four-step twiddle, length-P2 FFT over c in shared memory,
// Eq. (7) at the output slots owned by m1.  smem: Z, scratch (r x P2 each), tw2, pre (P2).
// `prologue_done`: tw2/pre already staged.  Shared by the standalone K2 and K1's fused tail.
template <int R>
__device__ __forceinline__ void k2_fft_block(const K2Params& P, uint32_t m1, uint32_t b, double2* zs) {
    double2* Z = zs;                              // [R][P2]
    double2* scratch = zs + (size_t)R * P.P2;     // [R][P2]
    double2* tw2 = scratch + (size_t)R * P.P2;    // omega_P2^t
    double2* pre = tw2 + P.P2;                    // omega_p^{m1 c}
    const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
    if (s0 >= P.W) return;  // no output slot maps to this m1 (block-uniform)
    for (uint32_t c = threadIdx.x; c < P.P2; c += blockDim.x) {
        tw2[c] = __ldg(P.omega + (size_t)c * P.P1);  // omega_P2^c = omega_p^{c P1}
        pre[c] = __ldg(P.omega + (size_t)m1 * c);    // four-step twiddle; m1 c < p
    }
    __syncthreads();
    const double2* __restrict__ Y = P.Y + (size_t)b * P.y_stride + (size_t)m1 * P.P2 * R;
    PFT_BOUND((size_t)b * P.y_stride + ((size_t)m1 + 1) * P.P2 * R - 1, P.y_elems);
    load_twiddled_slab<R>(Y, P.P2, m1, pre, Z);
    __syncthreads();
    const double2* res = Z;
    if (P.P2 > 1) res = fft_columns(Z, scratch, R, P.fft2, SmemTwiddles{tw2});
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
        PFT_BOUND((size_t)b * P.W + s, P.out_elems);
        out[s] = v;
        if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
    }
    __syncthreads();  // smem reuse by a following m1
}

template <int R>
__global__ void __launch_bounds__(K2_THREADS) k2_fft_post(K2Params P) {
    extern __shared__ __align__(16) double2 zs[];
    double2* Z = zs;                              // [R][P2]
    double2* scratch = zs + (size_t)R * P.P2;     // [R][P2]
    double2* tw2 = scratch + (size_t)R * P.P2;    // omega_P2^t
    double2* pre = tw2 + P.P2;                    // omega_p^{m1 c}
    const uint32_t m1 = blockIdx.x, b = blockIdx.y;
    // the next transform's K1 may launch now: it only touches this workspace after its own
    // griddepcontrol.wait (which waits for this grid to complete)
    if (P.release_next) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
    if (s0 >= P.W) return;  // no output slot maps to this m1 (block-uniform)

    // ---- prologue (overlaps K1's tail under programmatic dependent launch): tables only
    for (uint32_t c = threadIdx.x; c < P.P2; c += blockDim.x) {
        tw2[c] = __ldg(P.omega + (size_t)c * P.P1);  // omega_P2^c = omega_p^{c P1}
        pre[c] = __ldg(P.omega + (size_t)m1 * c);    // four-step twiddle; m1 c < p
    }
    const uint64_t s_first = s0 + (uint64_t)P.P1 * threadIdx.x;
    double pw0[R];
    double2 ptw0 = make_double2(0.0, 0.0);
    if (s_first < P.W) {
#pragma unroll
        for (int j = 0; j < R; ++j) pw0[j] = __ldg(P.post_powers + s_first * R + j);
        ptw0 = __ldg(P.post_twiddles + s_first);
    }
    // ---- wait for K1's slab Y to be complete and visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    const double2* __restrict__ Y = P.Y + (size_t)b * P.y_stride + (size_t)m1 * P.P2 * R;
    PFT_BOUND((size_t)b * P.y_stride + ((size_t)m1 + 1) * P.P2 * R - 1, P.y_elems);
    load_twiddled_slab<R>(Y, P.P2, m1, pre, Z);
    __syncthreads();
    const double2* res = Z;
    if (P.P2 > 1) res = fft_columns(Z, scratch, R, P.fft2, SmemTwiddles{tw2});
    double2* __restrict__ out = P.out + (size_t)b * P.W;
    for (uint64_t s = s_first; s < P.W; s += (uint64_t)P.P1 * blockDim.x) {
        uint64_t mp = P.first_mod_p + s % P.p;
        if (mp >= P.p) mp -= P.p;
        const uint32_t m2 = (uint32_t)(mp / P.P1);
        const bool first = s == s_first;
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < R; ++j) {  // ascending j
            const double pw = first ? pw0[j] : __ldg(P.post_powers + s * R + j);
            const double2 v = res[(size_t)j * P.P2 + m2];
            acc.x = fma(v.x, pw, acc.x);
            acc.y = fma(v.y, pw, acc.y);
        }
        const double2 v = cmul(acc, first ? ptw0 : __ldg(P.post_twiddles + s));  // e^{-pi i m / p}
        PFT_BOUND((size_t)b * P.W + s, P.out_elems);
        out[s] = v;
        if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
    }
}

// K2 FFT form as a bulk-copy ring on a grid of K2Params.k2_ctas CTAs per signal that loops over m1
// (opt-in: pft_dplan_opts.k2_grid_ctas).  Each CTA runs m1 = blockIdx.x, + gridDim.x, ...: the m1
// slab Y[m1][c][j] (contiguous P2 * R complex128) arrives by one cp.async.bulk per slab, issued
// by the CTA's ninth warp into one of two load buffers (full/empty mbarriers, K1's
// producer/consumer pattern) while the eight consumer warps run the previous one: the length-P2
// Stockham stages on the slab's own (c, j) layout between the load buffer and a scratch buffer,
// then Eq. (7) where the result lies.  Power-of-two P2 with radices 2/4/8/16; the post powers
// ((m - mu)/p)^j are formed in registers by ascending repeated multiplication, as the planner
// forms post_powers (x = (m - mu) * (1/p): exact for power-of-two p, within an ulp otherwise).
// Measured at C2c (profiles/r02/c2c_k2_workers.md): 128 CTAs 64.0 us chained / 65.5 isolated vs
// 67.6 / 70.9 for k2_fft_post; on the 20 SMs K1 leaves free (12-20 CTAs) 54.6-55.8 us chained --
// but any kernel between two K1s costs the chain ~7 us, so the default for chains is the K2
// workers inside K1's grid (k1_k2_worker).
constexpr int K2R_THREADS = K2_THREADS + 32;  // 8 consumer warps + the loader warp
template <int R>
__global__ void __launch_bounds__(K2R_THREADS, 1) k2_ring(K2Params P) {
    extern __shared__ __align__(128) unsigned char k2r_raw[];
    constexpr int NT = K2_THREADS;
    constexpr uint32_t kSpinLimit = 1u << 22;  // bounded waits: a lost signal becomes status bit 1, not a hang
    const uint32_t n = P.P2, slab = n * (uint32_t)R;
    double2* bufs = reinterpret_cast<double2*>(k2r_raw);  // [3][slab]: load buffers 0 and 1, FFT scratch 2
    double2* tw2 = bufs + 3 * (size_t)slab;               // omega_P2^t
    double2* pre = tw2 + n;                               // omega_p^{m1 c}
    uint64_t* full = reinterpret_cast<uint64_t*>(pre + n);  // [2] slab landed
    uint64_t* empty = full + 2;                              // [2] load buffer consumed
    const int tid = threadIdx.x;
    const uint32_t b = blockIdx.y, G = gridDim.x;
    if (P.release_next) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    const uint32_t m1_first = blockIdx.x;
    const uint32_t nk = m1_first < P.P1 ? (P.P1 - m1_first + G - 1) / G : 0;
    if (tid < NT) {
        for (uint32_t c = tid; c < n; c += NT) tw2[c] = __ldg(P.omega + (size_t)c * P.P1);
        if (nk > 0)
            for (uint32_t c = tid; c < n; c += NT) pre[c] = __ldg(P.omega + (size_t)m1_first * c);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's slab complete and visible
    __syncthreads();  // barriers and tables ready; the two roles part here
    if (tid >= NT) {
        if (tid == NT) {  // ---- loader: keeps two slabs in flight
            const double2* __restrict__ Yb = P.Y + (size_t)b * P.y_stride;
            const uint32_t bytes = slab * (uint32_t)sizeof(double2);
            for (uint32_t k = 0; k < nk; ++k) {
                const uint32_t lb = k & 1u;
                if (k >= 2) {  // the consumers have finished with this buffer's previous slab
                    uint32_t spins = 0;
                    while (!mbar_try_wait(&empty[lb], ((k >> 1) - 1u) & 1u))
                        if (++spins > kSpinLimit) {
                            atomicOr(P.status, 2);
                            break;
                        }
                }
                const uint32_t m1 = m1_first + k * G;
                PFT_BOUND((size_t)b * P.y_stride + ((size_t)m1 + 1) * slab - 1, P.y_elems);
                mbar_arrive_expect_tx(&full[lb], bytes);
                bulk_load(bufs + (size_t)lb * slab, Yb + (size_t)m1 * slab, bytes, &full[lb]);
            }
        }
        return;
    }
    // ---- consumers (named barrier 1 over the NT consumer threads)
    auto team_sync = [] { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); };
    const int64_t Mh = (int64_t)((P.W - 1) / 2);
    double2* __restrict__ out = P.out + (size_t)b * P.W;
    constexpr int PRE_PER = 4;  // host: P2 <= PRE_PER * K2_THREADS
    double2 pre_next[PRE_PER];
    for (uint32_t k = 0; k < nk; ++k) {
        const uint32_t m1 = m1_first + k * G, lb = k & 1u;
        if (k + 1 < nk) {  // the next m1's four-step twiddles, stored after the first stage
#pragma unroll
            for (int i = 0; i < PRE_PER; ++i) {
                const uint32_t c = tid + i * NT;
                if (c < n) pre_next[i] = __ldg(P.omega + (size_t)(m1 + G) * c);  // (m1 + G) c < p
            }
        }
        // this thread's first output slot of m1 and its post twiddle (latency hidden by the FFT)
        const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
        const uint64_t s_first = s0 + (uint64_t)P.P1 * tid;
        double2 ptw0 = make_double2(0.0, 0.0);
        if (s_first < P.W) ptw0 = __ldg(P.post_twiddles + s_first);
        {
            uint32_t spins = 0;
            while (!mbar_try_wait(&full[lb], (k >> 1) & 1u))
                if (++spins > kSpinLimit) {
                    atomicOr(P.status, 2);
                    break;
                }
        }
        double2* src = bufs + (size_t)lb * slab;
        double2* dst = bufs + 2 * (size_t)slab;
        int Ns = 1, lg_ns = 0;
        for (int st = 0; st < P.fft2.count; ++st) {
            const int RAD = P.fft2.radix[st];
            const double2* pr = (st == 0 && m1 != 0) ? pre : nullptr;
            switch (RAD) {
                case 2: k2_ring_stage<2, R>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT); lg_ns += 1; break;
                case 4: k2_ring_stage<4, R>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT); lg_ns += 2; break;
                case 8: k2_ring_stage<8, R>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT); lg_ns += 3; break;
                default: k2_ring_stage<16, R>(src, dst, (int)n, Ns, lg_ns, tw2, pr, tid, NT); lg_ns += 4; break;
            }
            Ns *= RAD;
            team_sync();
            double2* t = src;
            src = dst;
            dst = t;
            if (st == 0 && k + 1 < nk) {  // pre[] was last read in the first stage
#pragma unroll
                for (int i = 0; i < PRE_PER; ++i) {
                    const uint32_t c = tid + i * NT;
                    if (c < n) pre[c] = pre_next[i];
                }
            }
        }
        const double2* res = src;
        for (uint64_t s = s_first; s < P.W; s += (uint64_t)P.P1 * NT) {
            uint64_t mp = P.first_mod_p + s % P.p;
            if (mp >= P.p) mp -= P.p;
            const uint32_t m2 = (uint32_t)(mp / P.P1);
            const double x = (double)((int64_t)s - Mh) * P.inv_p;
            const double2* rv = res + (size_t)m2 * R;
            double2 acc = rv[0];
            double tp = x;
#pragma unroll
            for (int j = 1; j < R; ++j) {  // ascending j
                const double2 v = rv[j];
                acc.x = fma(v.x, tp, acc.x);
                acc.y = fma(v.y, tp, acc.y);
                if (j + 1 < R) tp *= x;
            }
            const double2 v = cmul(acc, s == s_first ? ptw0 : __ldg(P.post_twiddles + s));  // e^{-pi i m / p}
            PFT_BOUND((size_t)b * P.W + s, P.out_elems);
            out[s] = v;
            if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
        }
        // this slab's reads and writes of the load buffer precede its asynchronous refill
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        team_sync();  // also: the scratch and pre[] are free for the next m1
        if (tid == 0) mbar_arrive(&empty[lb]);
    }
}

// K2, Bluestein (chirp-z) form, for P2 with prime factors the in-smem Stockham radices do not
// cover ("Bluestein for prime factors > 61").  With
// h_c = e^{-pi i c^2/P2} and m2 c = (m2^2 + c^2 - (m2 - c)^2) / 2,
//   X[m2] = sum_c x_c e^{-2 pi i m2 c / P2} = h_m2 * sum_c (x_c h_c) conj(h_{m2 - c}),
// a linear convolution evaluated as a length-L cyclic one (L >= 2 P2 - 1, a power of two, <= 4096):
// A = FFT_L(x h, zero-padded); A *= FFT_L(conj h wrapped)/L (host table chirp_hat); X = h * IFFT_L(A)
// (IFFT as conj(FFT(conj(.)))).  One CTA per m1: columns j in groups of K2B_GROUP through the
// two transforms in shared memory (2 columns per pass for L <= 2048, 1 for L = 4096: P2 <= 2048),
// each output's Eq. (7) sum accumulated in registers in
// ascending j as the columns complete (<= 4 outputs per thread).
template <int R>
__global__ void __launch_bounds__(K2_THREADS) k2_bluestein_post(K2Params P) {
    extern __shared__ __align__(16) double2 zs[];
    constexpr int NOUT = 4;
    const int G = (int)P.bl_group;
    const uint32_t L = P.L;
    double2* A = zs;                        // [G][L]
    double2* B = zs + (size_t)G * L;        // [G][L] Stockham scratch
    const uint32_t m1 = blockIdx.x, b = blockIdx.y;
    const int tid = threadIdx.x, nt = blockDim.x;
    if (P.release_next) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
    if (s0 >= P.W) return;  // block-uniform
    const int64_t Mh = (int64_t)((P.W - 1) / 2);
    // this thread's outputs s = s0 + P1 (tid + i nt) and their m2
    double2 acc[NOUT];
    uint32_t m2s[NOUT];
    double xs[NOUT], pws[NOUT];
#pragma unroll
    for (int i = 0; i < NOUT; ++i) {
        acc[i] = make_double2(0.0, 0.0);
        const uint64_t s = s0 + (uint64_t)P.P1 * (tid + (uint64_t)i * nt);
        m2s[i] = 0xffffffffu;
        if (s < P.W) {
            uint64_t mp = P.first_mod_p + s % P.p;
            if (mp >= P.p) mp -= P.p;
            m2s[i] = (uint32_t)(mp / P.P1);
            xs[i] = (double)((int64_t)s - Mh) * P.inv_p;  // (m - mu)/p
            pws[i] = 1.0;
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's slab complete and visible
    const double2* __restrict__ Y = P.Y + (size_t)b * P.y_stride + (size_t)m1 * P.P2 * R;
    PFT_BOUND((size_t)b * P.y_stride + ((size_t)m1 + 1) * P.P2 * R - 1, P.y_elems);
    const Twiddles twL{P.omega_L, 1u};
    for (int j0 = 0; j0 < R; j0 += G) {
        const int g = R - j0 < G ? R - j0 : G;
        // x_c h_c (x_c = omega_p^{m1 c} Y[c][j]), zero-padded to L
        for (uint32_t idx = tid; idx < (uint32_t)g * L; idx += nt) {
            const uint32_t jj = idx / L, c = idx - jj * L;
            double2 v = make_double2(0.0, 0.0);
            if (c < P.P2) {
                v = __ldcg(Y + (size_t)c * R + j0 + jj);
                if (m1 != 0 && c != 0) v = cmul(v, __ldg(P.omega + (size_t)m1 * c));  // m1 c < p
                v = cmul(v, __ldg(P.chirp + c));
            }
            A[idx] = v;
        }
        __syncthreads();
        double2* r1 = fft_columns(A, B, g, P.fft2, twL);
        double2* o1 = r1 == A ? B : A;
        // times the kernel's transform, conjugated for the inverse transform
        for (uint32_t idx = tid; idx < (uint32_t)g * L; idx += nt) {
            const double2 v = cmul(r1[idx], __ldg(P.chirp_hat + (idx % L)));
            o1[idx] = make_double2(v.x, -v.y);
        }
        __syncthreads();
        double2* r2 = fft_columns(o1, r1, g, P.fft2, twL);
        // X[m2] = h_m2 conj(r2[m2]) (chirp_hat carries the 1/L); Eq. (7) terms of these columns
        for (int jj = 0; jj < g; ++jj) {
#pragma unroll
            for (int i = 0; i < NOUT; ++i) {
                if (m2s[i] == 0xffffffffu) continue;
                const double2 t = r2[(size_t)jj * L + m2s[i]];
                const double2 X = cmul(make_double2(t.x, -t.y), __ldg(P.chirp + m2s[i]));
                acc[i].x = fma(X.x, pws[i], acc[i].x);  // ascending j
                acc[i].y = fma(X.y, pws[i], acc[i].y);
                pws[i] *= xs[i];
            }
        }
        __syncthreads();  // A / B reuse by the next group
    }
    double2* __restrict__ out = P.out + (size_t)b * P.W;
#pragma unroll
    for (int i = 0; i < NOUT; ++i) {
        if (m2s[i] == 0xffffffffu) continue;
        const uint64_t s = s0 + (uint64_t)P.P1 * (tid + (uint64_t)i * nt);
        const double2 v = cmul(acc[i], __ldg(P.post_twiddles + s));  // e^{-pi i m / p}
        PFT_BOUND((size_t)b * P.W + s, P.out_elems);
        out[s] = v;
        if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
    }
}

// K2 (dot form, few outputs per m1): only the ~W/P1 bins this CTA owns are needed, so
// instead of the full length-P2 FFT each warp evaluates
//   out[s] = e^{-pi i m/p} sum_c omega_P2^{m2 c} (sum_j Z[j][c] ((m - mu)/p)^j)
// directly from the twiddled slab Z in shared memory: one barrier instead of one per FFT
// stage.  Lane-strided partial sums + xor-butterfly keep the order fixed.
template <int R>
__global__ void __launch_bounds__(K2_THREADS) k2_dot_post(K2Params P) {
    extern __shared__ __align__(16) double2 zs[];
    double2* Z = zs;                           // [R][P2]
    double2* tw2 = zs + (size_t)R * P.P2;      // omega_P2^t
    double2* pre = tw2 + P.P2;                 // omega_p^{m1 c}
    const uint32_t m1 = blockIdx.x, b = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = K2_THREADS / 32;
    if (P.release_next) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t s0 = (uint64_t)((m1 + P.P1 - P.first_mod_p1) % P.P1);
    if (s0 >= P.W) return;  // block-uniform
    // ---- prologue (overlaps K1's tail under PDL): twiddle tables and this warp's first powers
    for (uint32_t c = threadIdx.x; c < P.P2; c += blockDim.x) {
        tw2[c] = __ldg(P.omega + (size_t)c * P.P1);
        pre[c] = __ldg(P.omega + (size_t)m1 * c);
    }
    const uint64_t s_first = s0 + (uint64_t)P.P1 * warp;
    double pw0[R];
    if (s_first < P.W) {
#pragma unroll
        for (int j = 0; j < R; ++j) pw0[j] = __ldg(P.post_powers + s_first * R + j);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    const double2* __restrict__ Y = P.Y + (size_t)b * P.y_stride + (size_t)m1 * P.P2 * R;
    PFT_BOUND((size_t)b * P.y_stride + ((size_t)m1 + 1) * P.P2 * R - 1, P.y_elems);
    load_twiddled_slab<R>(Y, P.P2, m1, pre, Z);
    __syncthreads();
    const bool p2_pow2 = (P.P2 & (P.P2 - 1)) == 0;
    double2* __restrict__ out = P.out + (size_t)b * P.W;
    for (uint64_t s = s_first; s < P.W; s += (uint64_t)P.P1 * NW) {
        uint64_t mp = P.first_mod_p + s % P.p;
        if (mp >= P.p) mp -= P.p;
        const uint32_t m2 = (uint32_t)(mp / P.P1);
        double pw[R];
#pragma unroll
        for (int j = 0; j < R; ++j) pw[j] = (s == s_first) ? pw0[j] : __ldg(P.post_powers + s * R + j);
        double2 acc = make_double2(0.0, 0.0);
        for (uint32_t c = lane; c < P.P2; c += 32) {
            double2 S = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < R; ++j) {  // ascending j
                const double2 z = Z[(size_t)j * P.P2 + c];
                S.x = fma(z.x, pw[j], S.x);
                S.y = fma(z.y, pw[j], S.y);
            }
            const uint32_t e = p2_pow2 ? ((m2 * c) & (P.P2 - 1)) : (uint32_t)(((uint64_t)m2 * c) % P.P2);
            acc = cadd(acc, cmul(S, tw2[e]));  // omega_P2^{m2 c}
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
        }
        if (lane == 0) {
            const double2 v = cmul(acc, __ldg(P.post_twiddles + s));  // e^{-pi i m / p}
            PFT_BOUND((size_t)b * P.W + s, P.out_elems);
            out[s] = v;
            if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
        }
    }
}

// K2 (L2 form, default): no shared memory and a small register footprint, so its CTAs
// can park beside two K1 CTAs on every SM while K1 streams (programmatic dependent launch).
// One warp per output slot reads the m1 slice of the L2-resident slab directly:
//   out[s] = e^{-pi i m/p} sum_c e^{-2 pi i m' c / p} (sum_j Y[m1][c][j] ((m - mu)/p)^j)
// (m' = m mod p, m1 = m' mod P1).  Lane-strided partial sums + xor-butterfly: fixed order.
template <int R>
__global__ void __launch_bounds__(K2L_THREADS) k2_l2_post(K2Params P) {
    // the next transform's K1 may launch now (it waits for this grid before touching Y)
    if (P.release_next) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const bool p_pow2 = (P.p & (P.p - 1)) == 0;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's slab complete and visible
    const double2* __restrict__ Yb = P.Y + (size_t)b * P.y_stride;
    double2* __restrict__ out = P.out + (size_t)b * P.W;
    for (uint64_t s = gwarp; s < P.W; s += nwarps) {
        uint64_t mp = P.first_mod_p + s % P.p;
        if (mp >= P.p) mp -= P.p;
        const uint32_t m1 = (uint32_t)(mp % P.P1);
        const double2* __restrict__ Y = Yb + (size_t)m1 * P.P2 * R;
        double pw[R];
#pragma unroll
        for (int j = 0; j < R; ++j) pw[j] = __ldg(P.post_powers + s * R + j);
        double2 acc = make_double2(0.0, 0.0);
        for (uint32_t c = lane; c < P.P2; c += 32) {
            const double2* yc = Y + (size_t)c * R;
            const uint64_t e = p_pow2 ? ((mp * c) & (P.p - 1)) : ((mp * c) % P.p);
            const double2 tw = __ldg(P.omega + e);  // e^{-2 pi i m' c / p}
            double2 S = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < R; ++j) {  // ascending j
                const double2 y = yc[j];
                S.x = fma(y.x, pw[j], S.x);
                S.y = fma(y.y, pw[j], S.y);
            }
            acc = cadd(acc, cmul(S, tw));
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
        }
        if (lane == 0) {
            const double2 v = cmul(acc, __ldg(P.post_twiddles + s));  // e^{-pi i m / p}
            PFT_BOUND((size_t)b * P.W + s, P.out_elems);
            out[s] = v;
            if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
        }
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
    const double2* __restrict__ Y = P.Y + (size_t)b * P.y_stride + (size_t)m1 * P.P2 * R;
    PFT_BOUND((size_t)b * P.y_stride + ((size_t)m1 + 1) * P.P2 * R - 1, P.y_elems);
    double2* __restrict__ out = P.out + (size_t)b * P.W;
    if (P.release_next) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

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
            PFT_BOUND((size_t)b * P.W + s, P.out_elems);
            out[s] = v;
            if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(P.status, 1);
        }
    }
}

// ----------------------------------------------------------------------------- launchers
// Defined here, instantiated per r in the kinst_*.cu translation units (compiled in parallel);
// pft_kernels.cu dispatches on r through the extern instantiations.

#define PFT_R_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) \
    X(14) X(15) X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25)

// The attribute is only a cap (the launch's dynamic size decides occupancy), so set it to
// the device maximum once instead of per plan: plans with different P1 share a kernel.
constexpr size_t kMaxDynSmem = 227 * 1024;

template <int R>
cudaError_t launch_k1_r(const CUtensorMap& map, const K1Params& P, dim3 grid, size_t smem, cudaStream_t st,
                               bool mu0) {
    // Programmatic dependent launch: when the previous kernel in the stream is a K2 (which
    // triggers at its start), this K1 starts streaming its input while that K2 finishes;
    // any other predecessor does not trigger, so ordinary stream order applies.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(K1_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    unsigned n = 0;
    if (P.pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (P.fused) {  // the grid barrier needs every CTA resident
        attr[n].id = cudaLaunchAttributeCooperative;
        attr[n].val.cooperative = 1;
        ++n;
    }
    if (P.split > 1) {  // clusters of `split` CTAs per residue class
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = P.split;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    if constexpr (k1_k2_tail_instantiated(R)) {
        if (P.k2_tail) {
            if (mu0) return cudaLaunchKernelEx(&cfg, k1_contract_fft<R, true, 1>, map, P);
            return cudaLaunchKernelEx(&cfg, k1_contract_fft<R, false, 1>, map, P);
        }
    }
    if (P.k2_tail) return cudaErrorInvalidValue;  // no K2-tail instantiation for this r
    if constexpr (k1_k2_workers_instantiated(R)) {
        if (P.workers) {
            if (mu0) return cudaLaunchKernelEx(&cfg, k1_contract_fft<R, true, 2>, map, P);
            return cudaLaunchKernelEx(&cfg, k1_contract_fft<R, false, 2>, map, P);
        }
    }
    if (P.workers) return cudaErrorInvalidValue;  // no worker instantiation for this r
    if (mu0) return cudaLaunchKernelEx(&cfg, k1_contract_fft<R, true>, map, P);
    return cudaLaunchKernelEx(&cfg, k1_contract_fft<R, false>, map, P);
}

template <int R>
cudaError_t configure_k1_r(size_t smem, bool mu0) {
    const auto a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = mu0 ? cudaFuncSetAttribute(k1_contract_fft<R, true>, a, (int)smem)
                        : cudaFuncSetAttribute(k1_contract_fft<R, false>, a, (int)smem);
    if constexpr (k1_k2_tail_instantiated(R)) {
        if (e == cudaSuccess)
            e = mu0 ? cudaFuncSetAttribute(k1_contract_fft<R, true, 1>, a, (int)smem)
                    : cudaFuncSetAttribute(k1_contract_fft<R, false, 1>, a, (int)smem);
    }
    if constexpr (k1_k2_workers_instantiated(R)) {
        if (e == cudaSuccess)
            e = mu0 ? cudaFuncSetAttribute(k1_contract_fft<R, true, 2>, a, (int)smem)
                    : cudaFuncSetAttribute(k1_contract_fft<R, false, 2>, a, (int)smem);
    }
    return e;
}


template <int R>
cudaError_t launch_k2_r(const K2Params& P, dim3 grid, cudaStream_t st) {
    // Programmatic dependent launch: K2 may start its table prologue while K1 drains;
    // griddepcontrol.wait in K2 orders its reads of Y after K1's completion.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(K2_THREADS);
    cfg.dynamicSmemBytes = P.mode == K2_FFT ? k2_smem_bytes(R, P.P2) : P.mode == K2_DOT ? k2_dot_smem_bytes(R, P.P2) : 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (P.mode == K2_L2) {
        cfg.blockDim = dim3(K2L_THREADS);
        return cudaLaunchKernelEx(&cfg, k2_l2_post<R>, P);
    }
    if (P.mode == K2_BLUESTEIN) {
        cfg.dynamicSmemBytes = k2_bluestein_smem_bytes(P.L);
        return cudaLaunchKernelEx(&cfg, k2_bluestein_post<R>, P);
    }
    if (P.mode == K2_FFT && P.ring) {
        cfg.blockDim = dim3(K2R_THREADS);
        cfg.dynamicSmemBytes = k2_ring_smem_bytes(R, P.P2);
        return cudaLaunchKernelEx(&cfg, k2_ring<R>, P);
    }
    if (P.mode == K2_FFT) return cudaLaunchKernelEx(&cfg, k2_fft_post<R>, P);
    if (P.mode == K2_DOT) return cudaLaunchKernelEx(&cfg, k2_dot_post<R>, P);
    return cudaLaunchKernelEx(&cfg, k2_direct_post<R>, P);
}

template <int R>
cudaError_t configure_k2_r(size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k2_fft_post<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k2_ring<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k2_bluestein_post<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k2_dot_post<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// The attribute is only a cap (the launch's dynamic size decides occupancy), so set it to
// the device maximum once instead of per plan: plans with different P1 share a kernel.

template <int R>
int k1_active_r(size_t smem, bool mu0) {
    int n = 0;
    if (mu0)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k1_contract_fft<R, true>, K1_THREADS, smem);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k1_contract_fft<R, false>, K1_THREADS, smem);
    return n;
}


#define PFT_INSTANCES(R, EXT)                                                                                   \
    EXT template cudaError_t launch_k1_r<R>(const CUtensorMap&, const K1Params&, dim3, size_t, cudaStream_t, bool); \
    EXT template cudaError_t configure_k1_r<R>(size_t, bool);                                                  \
    EXT template int k1_active_r<R>(size_t, bool);                                                             \
    EXT template cudaError_t launch_k2_r<R>(const K2Params&, dim3, cudaStream_t);                              \
    EXT template cudaError_t configure_k2_r<R>(size_t);

}  // namespace pftdev
