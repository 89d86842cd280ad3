// fft_smem.cuh -- batched mixed-radix Stockham FFT on shared memory (complex128).
//
// Realises batch_fft_columns for the per-CTA FFT pass of K1: `ncols`
// columns of length n, column c at x + c*n.  Autosort Stockham formulation: stage s with
// radix R and span Ns reads x[j + r*n/R] and writes y[(j/Ns)*Ns*R + j%Ns + r*Ns] after
// the twiddle e^{-2 pi i (j mod Ns) r / (Ns R)}; output is in natural order.  Every
// twiddle is a lookup in an exactly-reduced table of omega_n^t (host-computed,
// SPEC.md:261,377), never a recurrence.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pftdev {

struct FftRadices {
    int n;          // transform length (product of radices)
    int count;      // number of stages
    int radix[24];  // stage radices in order
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }

// Twiddle table accessor: omega_n^t for t in [n], stored as tab[t * stride] (the same
// table serves several lengths that divide the table length).
struct Twiddles {
    const double2* tab;
    uint32_t stride;
    __device__ __forceinline__ double2 operator()(uint32_t t) const { return __ldg(tab + (size_t)t * stride); }
};

// Same, for a dense omega_n table staged in shared memory (no global round trip per stage).
struct SmemTwiddles {
    const double2* tab;
    __device__ __forceinline__ double2 operator()(uint32_t t) const { return tab[t]; }
};

__device__ __forceinline__ void dft2(double2& a, double2& b) {
    const double2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
    const double2 a = cadd(v0, v2), b = csub(v0, v2);
    const double2 c = cadd(v1, v3), d = cmul_mi(csub(v1, v3));
    v0 = cadd(a, c);
    v2 = csub(a, c);
    v1 = cadd(b, d);
    v3 = csub(b, d);
}

__device__ __forceinline__ void dft8(double2 (&v)[8]) {
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4(e0, e1, e2, e3);
    dft4(o0, o1, o2, o3);
    const double s = 0.70710678118654752440;  // sqrt(1/2)
    const double2 t1 = make_double2((o1.x + o1.y) * s, (o1.y - o1.x) * s);  // o1 * e^{-i pi/4}
    const double2 t2 = cmul_mi(o2);                                          // o2 * e^{-i pi/2}
    const double2 t3 = make_double2((o3.y - o3.x) * s, -(o3.x + o3.y) * s);  // o3 * e^{-3 i pi/4}
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, t1);
    v[5] = csub(e1, t1);
    v[2] = cadd(e2, t2);
    v[6] = csub(e2, t2);
    v[3] = cadd(e3, t3);
    v[7] = csub(e3, t3);
}

// 16-point DFT as 4 x 4: DFT-4 over n1 (stride 4) for each n2, twiddles W16^{n2 k1}, DFT-4
// over n2; X[k1 + 4 k2] lands at v[4 k1 + k2] and is transposed back to v[k].
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[n2 + 4], v[n2 + 8], v[n2 + 12]);
    const double c = 0.92387953251128675613, s = 0.38268343236508977173, h = 0.70710678118654752440;
    // v[n2 + 4 k1] *= W16^{n2 k1}, W16^m = cos(2 pi m/16) - i sin(2 pi m/16)
    v[5] = cmul(v[5], make_double2(c, -s));     // m = 1
    v[9] = cmul(v[9], make_double2(h, -h));     // m = 2
    v[13] = cmul(v[13], make_double2(s, -c));   // m = 3
    v[6] = cmul(v[6], make_double2(h, -h));     // m = 2
    v[10] = cmul_mi(v[10]);                     // m = 4
    v[14] = cmul(v[14], make_double2(-h, -h));  // m = 6
    v[7] = cmul(v[7], make_double2(s, -c));     // m = 3
    v[11] = cmul(v[11], make_double2(-h, -h));  // m = 6
    v[15] = cmul(v[15], make_double2(-c, s));   // m = 9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    // transpose the 4 x 4 block: X[k1 + 4 k2] = v[4 k1 + k2]
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a + 1; b < 4; ++b) {
            const double2 t = v[4 * a + b];
            v[4 * a + b] = v[4 * b + a];
            v[4 * b + a] = t;
        }
}

__device__ __forceinline__ void dft3(double2& v0, double2& v1, double2& v2) {
    const double h = 0.86602540378443864676;  // sqrt(3)/2
    const double2 t = cadd(v1, v2);
    const double2 d = csub(v1, v2);
    const double2 m = make_double2(v0.x - 0.5 * t.x, v0.y - 0.5 * t.y);
    v0 = cadd(v0, t);
    // -i h d
    const double2 r = make_double2(h * d.y, -h * d.x);
    v1 = cadd(m, r);
    v2 = csub(m, r);
}

// The threads that run an FFT pass: the whole CTA (__syncthreads), or K1's consumer warps
// alone (named barrier 1) while the producer warp keeps streaming.
struct BlockTeam {
    __device__ __forceinline__ int tid() const { return threadIdx.x; }
    __device__ __forceinline__ int size() const { return blockDim.x; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
};
template <int NT>
struct WarpsTeam {
    int t;
    __device__ __forceinline__ int tid() const { return t; }
    __device__ __forceinline__ int size() const { return NT; }
    __device__ __forceinline__ void sync() const { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }
};

// Bank swizzle of the buffer between the first two stages of a power-of-two transform: the
// first stage (Ns = 1) writes y[R j + r], 8 lanes of a 128-bit store phase R * 16 bytes apart
// (8-way conflicts); XOR-ing the 16-byte slot within each 128-byte block with the block index
// spreads them, and the second stage's contiguous reads stay conflict-free.
__device__ __forceinline__ int fft_swz(int i) { return i ^ ((i >> 3) & 7); }

// One Stockham stage with a radix known at compile time (2, 3, 4, 8, 16).  When n is a power
// of two (POW2) the index arithmetic uses shifts/masks (lg_nb = log2(n/R), lg_ns =
// log2(Ns)); otherwise integer division.  sw: 1 = swizzled destination, 2 = swizzled source
// (POW2 only).  colw: per-column factor applied to the inputs (first stage), or null.
template <int R, bool POW2, class TW>
__device__ __forceinline__ void stockham_stage_fixed(const double2* __restrict__ src, double2* __restrict__ dst,
                                                     int ncols, int n, int Ns, int lg_nb, int lg_ns, const TW& tw,
                                                     int t0, int nt, int sw = 0, const double2* colw = nullptr,
                                                     int colw_div = 1) {
    const int nb = n / R;
    const uint32_t tstride = (uint32_t)(n / (Ns * R));
    for (int idx = t0; idx < ncols * nb; idx += nt) {
        int col, j, k, base;
        if constexpr (POW2) {
            col = idx >> lg_nb;
            j = idx & (nb - 1);
            k = j & (Ns - 1);
            base = ((j >> lg_ns) << lg_ns) * R + k;
        } else {
            col = idx / nb;
            j = idx - col * nb;
            k = j % Ns;
            base = (j / Ns) * Ns * R + k;
        }
        double2 v[R];
        if (POW2 && (sw & 2)) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = src[fft_swz(col * n + j + r * nb)];
        } else {
            const double2* s = src + (size_t)col * n;
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = s[j + r * nb];
        }
        if (colw) {
            const double2 wc = colw[colw_div == 1 ? col : col / colw_div];
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = cmul(v[r], wc);
        }
        if (k != 0) {
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw((uint32_t)(k * r) * tstride));
        }
        if constexpr (R == 2) dft2(v[0], v[1]);
        if constexpr (R == 3) dft3(v[0], v[1], v[2]);
        if constexpr (R == 4) dft4(v[0], v[1], v[2], v[3]);
        if constexpr (R == 8) dft8(v);
        if constexpr (R == 16) dft16(v);
        if (POW2 && (sw & 1)) {
#pragma unroll
            for (int r = 0; r < R; ++r) dst[fft_swz(col * n + base + r * Ns)] = v[r];
        } else {
            double2* d = dst + (size_t)col * n;
#pragma unroll
            for (int r = 0; r < R; ++r) d[base + r * Ns] = v[r];
        }
    }
}

// Generic radix (any R): O(R^2) per butterfly, twiddles omega_R^{rs} = omega_n^{rs n/R}.
template <class TW>
__device__ __forceinline__ void stockham_stage_generic(const double2* __restrict__ src, double2* __restrict__ dst,
                                                       int ncols, int n, int Ns, int R, const TW& tw, int t0, int nt) {
    const int nb = n / R;
    const uint32_t tstride = (uint32_t)(n / (Ns * R));
    const uint32_t rstride = (uint32_t)(n / R);
    for (int idx = t0; idx < ncols * nb * R; idx += nt) {
        const int col = idx / (nb * R);
        const int rem = idx - col * nb * R;
        const int j = rem / R, out_r = rem - j * R;
        const double2* s = src + (size_t)col * n;
        const int k = j % Ns;
        double2 acc = make_double2(0.0, 0.0);
        for (int r = 0; r < R; ++r) {
            double2 v = s[j + r * nb];
            if (k != 0 && r != 0) v = cmul(v, tw((uint32_t)(k * r) * tstride));
            const uint32_t e = (uint32_t)((out_r * r) % R);
            acc = cadd(acc, e ? cmul(v, tw(e * rstride)) : v);
        }
        dst[(size_t)col * n + (j / Ns) * Ns * R + k + out_r * Ns] = acc;
    }
}

// Full transform of ncols columns; returns the buffer holding the result (x or y).
// Caller must team.sync() before (inputs written); the last stage ends with a team.sync().
// colw: optional per-column factor folded into the first stage's loads (null = none); column
// col takes colw[col / colw_div] (several columns per factor: several signals per CTA).
template <class TW, class Team = BlockTeam>
__device__ __forceinline__ double2* fft_columns(double2* x, double2* y, int ncols, const FftRadices& plan,
                                                const TW& tw, const Team team = Team{},
                                                const double2* colw = nullptr, int colw_div = 1) {
    const int t0 = team.tid(), nt = team.size();
    double2* src = x;
    double2* dst = y;
    int Ns = 1, lg_ns = 0;
    const int n = plan.n;
    const bool pow2 = (n & (n - 1)) == 0;
    const int lg_n = 31 - __clz(n);
    for (int st = 0; st < plan.count; ++st) {
        const int R = plan.radix[st];
        const int lg_r = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4;
        const int lg_nb = lg_n - lg_r;
        const double2* cw = st == 0 ? colw : nullptr;
        if (pow2) {
            // swizzle the buffer between stages 0 and 1 (n >= 64 keeps every 8-block in a column)
            const int sw = (n >= 64 && plan.count >= 2) ? (st == 0 ? 1 : st == 1 ? 2 : 0) : 0;
            switch (R) {
                case 2: stockham_stage_fixed<2, true>(src, dst, ncols, n, Ns, lg_nb, lg_ns, tw, t0, nt, sw, cw, colw_div); break;
                case 4: stockham_stage_fixed<4, true>(src, dst, ncols, n, Ns, lg_nb, lg_ns, tw, t0, nt, sw, cw, colw_div); break;
                case 8: stockham_stage_fixed<8, true>(src, dst, ncols, n, Ns, lg_nb, lg_ns, tw, t0, nt, sw, cw, colw_div); break;
                default: stockham_stage_fixed<16, true>(src, dst, ncols, n, Ns, lg_nb, lg_ns, tw, t0, nt, sw, cw, colw_div); break;
            }
            lg_ns += lg_r;
        } else {
            switch (R) {
                case 2: stockham_stage_fixed<2, false>(src, dst, ncols, n, Ns, 0, 0, tw, t0, nt, 0, cw, colw_div); break;
                case 3: stockham_stage_fixed<3, false>(src, dst, ncols, n, Ns, 0, 0, tw, t0, nt, 0, cw, colw_div); break;
                case 4: stockham_stage_fixed<4, false>(src, dst, ncols, n, Ns, 0, 0, tw, t0, nt, 0, cw, colw_div); break;
                case 8: stockham_stage_fixed<8, false>(src, dst, ncols, n, Ns, 0, 0, tw, t0, nt, 0, cw, colw_div); break;
                case 16: stockham_stage_fixed<16, false>(src, dst, ncols, n, Ns, 0, 0, tw, t0, nt, 0, cw, colw_div); break;
                default:
                    if (cw) {  // generic radix: apply the column factor in place first
                        for (int i = t0; i < ncols * n; i += nt) src[i] = cmul(src[i], cw[i / n / colw_div]);
                        team.sync();
                    }
                    stockham_stage_generic(src, dst, ncols, n, Ns, R, tw, t0, nt);
                    break;
            }
        }
        team.sync();
        double2* t = src;
        src = dst;
        dst = t;
        Ns *= R;
    }
    return src;
}

}  // namespace pftdev
