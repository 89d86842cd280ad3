// pft_device.cu -- device plans and the extern "C" device entry points of pft_capi.h.
//
// A device plan is the immutable upload of a host PftPlan plus the
// decomposition p = P1 * P2 used by the kernels:
//   phase[q], tvals[q], w[r], omega[p] (e^{-2 pi i t/p}), post_powers[W][r],
//   post_twiddles[W], and a default workspace Y[P1][P2][r] for batch 1.
// There is no host compute path: if the device is missing every call fails.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../host/api_guard.hpp"
#include "../host/internal.hpp"
#include "kernels.cuh"

#ifndef PFT_BUILD_DESC
#define PFT_BUILD_DESC "dev"
#endif

using namespace pft;
using namespace pft::detail;

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear sticky-free errors
        fail(PFT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

int usable_device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Radix schedule for the per-CTA FFT (largest supported radices first).
bool factor_radices(uint32_t n, pftdev::FftRadices& out) {
    out.n = (int)n;
    out.count = 0;
    uint32_t m = n;
    auto push = [&](int r) {
        if (out.count >= 24) return false;
        out.radix[out.count++] = r;
        return true;
    };
    // powers of two: radix 16 first (P1 = 128: 16 x 8, two block barriers instead of three
    // for 8 x 8 x 2), then one 8, 4 or 2 for the rest (capping the radix at 8 / 4 measured C3
    // 765 -> 781 / 812 us per batch, C2b and C4 unchanged: profiles/r02/ab_fft_radix_cap.log)
    // (n = 64 as 8 x 8: twice the butterflies of 16 x 4's first stage at a third of its dependent chain --
    // the 2-D rows pass, 36 columns of 64 per CTA: 84.3 -> 79.8 us)
    if (m == 64) { push(8); push(8); m = 1; }
    while (m % 16 == 0) { if (!push(16)) return false; m /= 16; }
    while (m % 8 == 0) { if (!push(8)) return false; m /= 8; }
    while (m % 4 == 0) { if (!push(4)) return false; m /= 4; }
    while (m % 2 == 0) { if (!push(2)) return false; m /= 2; }
    while (m % 3 == 0) { if (!push(3)) return false; m /= 3; }
    for (uint32_t f = 5; m > 1 && f <= 64; f += 2) {
        while (m % f == 0) { if (!push((int)f)) return false; m /= f; }
    }
    return m == 1;
}

constexpr uint64_t kTargetCtas = 256;        // >= 1.7 CTAs per SM on 148 SMs
constexpr size_t kK2SmemLimit = 220 * 1024;

bool k1_feasible(uint64_t P1, int r) {
    pftdev::FftRadices fr;
    if (P1 > 1 && !factor_radices((uint32_t)P1, fr)) return false;
    return sizeof(double2) * (size_t)r * P1 <= pftdev::k1_min_ring_bytes(r);  // FFT scratch = the ring
}

bool k2_fft_feasible(uint64_t P2, int r) {
    pftdev::FftRadices fr;
    if (P2 > 1 && !factor_radices((uint32_t)P2, fr)) return false;
    return pftdev::k2_smem_bytes(r, (uint32_t)P2) <= kK2SmemLimit;
}

// P2 for the sum tail: at most one K1 CTA per SM per transform, so under PDL two transforms
// stream side by side (measured C2b p = 2^14: P2 = 128 42.5 us vs P2 = 256 46.5 us; C4
// p = 27648: 128 21.7 us, 144 22.9 us, 256 27.7 us).  Among divisors P2 <= n_sms whose
// P1 = p / P2 keeps two K1 CTAs per SM and fits the tail scratch: prefer a power-of-two
// P1 >= K1_BR, then P1 >= K1_BR (a box's 32 rows all belong to the CTA; P1 = 16 measured
// 62 vs 38 us at C2a), then the largest P2, taking a power of two if within 15% of it.
// 0 = none.
bool sum_p1_ok(uint64_t P1, int r, uint64_t P2) {
    if (!k1_feasible(P1, r)) return false;
    if (pftdev::k1_smem_bytes(r, (uint32_t)P1, pftdev::k1_min_stages(r)) > (228 * 1024) / 2 - 1024) return false;
    return sizeof(double2) * r * P1 + pftdev::k1_sum_scratch_bytes((uint32_t)P1, (uint32_t)P2) <=
           pftdev::k1_min_ring_bytes(r);
}

// The sum tail pays, per CTA, W outputs of r-term sums plus a W-long row written and reduced
// through L2.  It is used when that stays small against the CTA's streaming work: the rows'
// traffic 2 P2 W complex <= 1/8 of the input and the tail's ~(r + 20) W ops <= 10% of the
// contraction's (3r + 10)/2 per element (C2b: 3% / 3%; C3 at p = 512: 3% / 2%).
bool sum_tail_pays(uint64_t N, uint64_t W, uint64_t P2, int r) {
    const double n = static_cast<double>(N), w = static_cast<double>(W), p2 = static_cast<double>(P2);
    return 16.0 * p2 * w <= n && 10.0 * w * (r + 20) <= n / p2 * (3.0 * r + 10.0) / 2.0;
}

uint64_t choose_p2_sum(uint64_t p, int r, int n_sms, size_t batch) {
    if (batch > 1) {
        // batched signals supply the CTAs: give each CTA as many rows as fit (the smallest P2),
        // keeping >= 1 CTA per SM over the batch (the 2-D column pass, 129 signals of 4096 at
        // p = 128: P2 = 2 7.2 us vs P2 = 4 11.3 us, profiles/r02/p2d)
        for (uint64_t d : divisors(p))
            if (d * batch >= (uint64_t)n_sms && sum_p1_ok(p / d, r, d)) return d;
    }
    // pass 0: P1 a power of two >= K1_BR (full 32-row boxes, radix-16/8 FFT: C4 p = 11520
    // measured 17.6 us with P1 = 128, P2 = 90 vs 20.2 us with P1 = 90, P2 = 128);
    // pass 1: P1 >= K1_BR; pass 2: any.  Within a pass the largest P2, taking a power of two
    // if within 15% of it.
    for (int pass = 0; pass < 3; ++pass) {
        uint64_t any = 0, pow2 = 0;
        for (uint64_t d : divisors(p)) {
            if (d > (uint64_t)n_sms) break;
            const uint64_t P1 = p / d;
            if (pass < 2 && P1 < (uint64_t)pftdev::K1_BR) continue;
            if (pass == 0 && (P1 & (P1 - 1)) != 0) continue;
            if (!sum_p1_ok(P1, r, d)) continue;
            any = d;
            if ((d & (d - 1)) == 0) pow2 = d;
        }
        if (any) return (pow2 && 100 * pow2 >= 85 * any) ? pow2 : any;
    }
    return 0;
}

// Choose P2 | p (K1 grid = P2 x batch CTAs; P1 = p / P2 is K1's in-CTA FFT length, P2 is
// K2's).  Prefer decompositions where both FFT passes fit shared memory, then the
// smallest P2 that still gives >= kTargetCtas CTAs (fewer residue classes = less K2 work).
uint64_t choose_p2(uint64_t p, int r, size_t batch) {
    const auto divs = divisors(p);
    const size_t nb = std::max<size_t>(batch, 1);
    for (int pass = 0; pass < 2; ++pass) {
        uint64_t best = 0;
        for (uint64_t d : divs) {
            if (!k1_feasible(p / d, r)) continue;
            if (pass == 0 && !k2_fft_feasible(d, r)) continue;
            best = d;
            if (d * nb >= kTargetCtas) return d;
        }
        if (best) return best;
    }
    return p;
}

// Device-aware choice of p (not in the reference).  SPEC's cost
// r (N + p log p + M) models a CPU; here the transform is one streaming pass whose time is set
// by HBM and by the FP64 issue rate of the paired contraction, with the decomposition the
// device plan would pick for that p:
//   t_mem  = 16 N / bw * pad(q) * (1 + 48 / q) / rows(P1)   pad: TMA chunks of 16 column pairs;
//                                                           bw = min(BW, 55 GB/s per K1 CTA)
//   t_fp   = N (3r + 10) / 2 / F / rows(P1)                 rows: P1 / (32 ceil(P1 / 32)), the
//                                                           used share of a box's 32 rows
//   t_tail = 32 W P2 / BW                if W <= p/4 (sum tail: rows written + reduced in L2)
//          = 8 us + 32 p r / BW          otherwise (slab + K2)
//   t      = 2 us + max(t_mem, t_fp) + t_tail          (per batch of signals: t_mem, t_fp, t_tail
//                                                     scale with the batch, CTAs come from it)
// BW = F = 6.6e12 (bytes/s, element-ops/s), calibrated on one B200 at N = 2^24, M = 2^10 where
// p = 2^13 (r = 10) is FP64-bound and p = 2^14..2^16 follow the row term (measured 51.8, 42.5,
// 45.1, 48.4 us; model 51.6, 44.6, 46.3, 51.0).
std::vector<DivisorChoice> rank_divisors_device(const Table& t, uint64_t N, uint64_t M, double eps, int n_sms,
                                                size_t batch = 1) {
    batch = std::max<size_t>(batch, 1);
    if (N <= 1) fail(PFT_ERR_INVALID_ARGUMENT, "select_divisor_device: N = 1 has no non-trivial split");
    if (M > N) fail(PFT_ERR_INVALID_ARGUMENT, "select_divisor_device: M > N");
    if (!t.has_eps(eps)) fail(PFT_ERR_EPSILON_NOT_IN_TABLE, "select_divisor_device: table has no entries for epsilon");
    constexpr double BW = 6.6e12, F = 6.6e12;
    const uint64_t W = 2 * M + 1;
    const double n = static_cast<double>(N);
    std::vector<DivisorChoice> all;
    for (uint64_t p : divisors(N)) {
        if (p <= 1) continue;
        int r;
        try {
            r = min_terms(t, eps, M, p);
        } catch (const Error& e) {
            if (e.status == PFT_ERR_RATIO_OUT_OF_RANGE) continue;
            throw;
        }
        const uint64_t q = N / p;
        if (q < 2) continue;
        uint64_t P2 = choose_p2_sum(p, r, n_sms, batch);
        const bool sum = P2 && sum_tail_pays(N, W, P2, r);
        if (!sum) P2 = choose_p2(p, r, batch);
        const uint64_t P1 = p / P2;
        if (!k1_feasible(P1, r)) continue;
        const double rows = static_cast<double>(P1) / (32.0 * static_cast<double>((P1 + 31) / 32));
        const uint64_t pairs = q / 2, chunks = (pairs + 15) / 16;
        const double pad = pairs ? 16.0 * static_cast<double>(chunks) / static_cast<double>(pairs) : 1.0;
        // a K1 CTA streams at most ~55 GB/s (ring depth / latency); with the sum tail two
        // transforms' grids are in flight under PDL
        const double ctas = static_cast<double>(sum ? 2 * P2 * batch : std::min<uint64_t>(P2 * batch, 2ull * n_sms));
        const double bw = std::min(BW, 55e9 * ctas);
        const double t_mem = 16.0 * n / bw * pad * (1.0 + 48.0 / static_cast<double>(q)) / rows;
        const double t_fp = n * (3.0 * r + 10.0) / 2.0 / F / rows;
        const double nb = static_cast<double>(batch);
        const double t_tail = sum ? 32.0 * static_cast<double>(W * P2) * nb / BW
                                  : (batch > 1 ? 0.0 : 8e-6) + 32.0 * static_cast<double>(p) * r * nb / BW;
        const double cost = 2e-6 + nb * std::max(t_mem, t_fp) + t_tail;
        DivisorChoice c;
        c.p = p;
        c.r = r;
        c.cost = cost * 1e6;  // microseconds
        all.push_back(c);
    }
    if (all.empty()) fail(PFT_ERR_RATIO_OUT_OF_RANGE, "select_divisor_device: no feasible divisor p");
    std::stable_sort(all.begin(), all.end(),
                     [](const DivisorChoice& a, const DivisorChoice& b) { return a.cost < b.cost; });
    return all;
}

// The sharded transform over `world` GPUs (pft_execute_sharded): each rank streams its slice of
// ceil(pairs / world) column pairs per row (rank 0 also the unpaired columns), the p x r slab
// (16 p r bytes) is reduced onto the root, and the root runs K2.  Per p:
//   t = 2 us + max(t_mem, t_fp) over the slice      (the single-GPU K1 terms on q_local columns)
//     + t_reduce = 15 us + 16 p r (world - 1) / world / 400 GB/s      (NCCL reduce over NVLink)
//     + t_k2     = 8 us + 32 p r / BW                                  (root: slab read + FFT)
// Large p shortens the rows each rank streams less than it grows the slab every rank reduces, so
// the pick is a smaller p than the SPEC cost model's (avoid p = 2^22's 268 MB
// slab).  world = 1 is the unsharded K1 + K2 pair.
std::vector<DivisorChoice> rank_divisors_sharded(const Table& t, uint64_t N, uint64_t M, double eps, int n_sms,
                                                 int world) {
    if (N <= 1) fail(PFT_ERR_INVALID_ARGUMENT, "select_divisor_sharded: N = 1 has no non-trivial split");
    if (M > N) fail(PFT_ERR_INVALID_ARGUMENT, "select_divisor_sharded: M > N");
    if (world < 1) fail(PFT_ERR_INVALID_ARGUMENT, "select_divisor_sharded: world < 1");
    if (!t.has_eps(eps)) fail(PFT_ERR_EPSILON_NOT_IN_TABLE, "select_divisor_sharded: table has no entries for epsilon");
    constexpr double BW = 6.6e12, F = 6.6e12, LINK = 400e9;
    std::vector<DivisorChoice> all;
    for (uint64_t p : divisors(N)) {
        if (p <= 1) continue;
        int r;
        try {
            r = min_terms(t, eps, M, p);
        } catch (const Error& e) {
            if (e.status == PFT_ERR_RATIO_OUT_OF_RANGE) continue;
            throw;
        }
        const uint64_t q = N / p;
        if (q < 2) continue;
        const uint64_t P2 = choose_p2(p, r, 1), P1 = p / P2;
        if (!k1_feasible(P1, r)) continue;
        const uint64_t pairs = (q - 1) / 2, lpairs = std::max<uint64_t>(1, (pairs + world - 1) / world);
        const double ql = 2.0 * static_cast<double>(lpairs) + 2.0;
        const double rows = static_cast<double>(P1) / (32.0 * static_cast<double>((P1 + 31) / 32));
        const double pad = 16.0 * static_cast<double>((lpairs + 15) / 16) / static_cast<double>(lpairs);
        const double bw = std::min(BW, 55e9 * static_cast<double>(std::min<uint64_t>(P2, 2ull * n_sms)));
        const double elems = static_cast<double>(p) * ql;
        const double t_mem = 16.0 * elems / bw * pad * (1.0 + 48.0 / ql) / rows;
        const double t_fp = elems * (3.0 * r + 10.0) / 2.0 / F / rows;
        const double slab = 16.0 * static_cast<double>(p) * r;
        const double t_red = world > 1 ? 15e-6 + slab * (world - 1) / world / LINK : 0.0;
        const double t_k2 = 8e-6 + 2.0 * slab / BW;
        DivisorChoice c;
        c.p = p;
        c.r = r;
        c.cost = (2e-6 + std::max(t_mem, t_fp) + t_red + t_k2) * 1e6;
        all.push_back(c);
    }
    if (all.empty()) fail(PFT_ERR_RATIO_OUT_OF_RANGE, "select_divisor_sharded: no feasible divisor p");
    std::stable_sort(all.begin(), all.end(),
                     [](const DivisorChoice& a, const DivisorChoice& b) { return a.cost < b.cost; });
    return all;
}

DivisorChoice select_divisor_device(const Table& t, uint64_t N, uint64_t M, double eps, int n_sms) {
    return rank_divisors_device(t, N, M, eps, n_sms).front();
}

}  // namespace

struct pft_dplan_s {
    int device = 0;
    HostPlan host;  // parameters (tables are on the device)
    uint64_t P1 = 0, P2 = 0;
    pftdev::FftRadices fft{};   // radices of P1 (K1)
    pftdev::FftRadices fft2{};  // radices of P2 (K2)
    uint32_t k1_stages = pftdev::K1_MIN_STAGES;
    int k2_mode = pftdev::K2_DIRECT;
    uint32_t k2_ctas = 0;
    uint32_t gsig_max = 1;   // P2 = 1 sum-tail plans: most signals a K1 CTA can hold as one row block (1, 2 or 4)
    uint32_t k2_workers = 0; // chained single executes: K2 worker CTAs riding in K1's grid (k1_k2_worker); 0 = off
    bool ring_ok = false;    // single executes whose K2 is its own grid run the bulk-copy ring kernel (k2_ring)
    uint32_t ring_ctas = 0;  // its grid width when the caller chose one (k2_grid_ctas); 0 = one CTA per m1
    bool allow_fuse = false; // K2 fused into K1's tail (opt-in; measured slower at C2b/C4)
    bool allow_split = true; // isolated executes: two CTAs (a cluster) per residue class
    bool sum_tail = false;   // unsharded execute: K1 sum tail, no K2 (few output bins)
    bool k2_tail = false;    // unsharded execute: K2's work by K1's last arrivals (many bins)
    uint32_t k2_group = 0;   // k2_tail: columns j per FFT group
    uint32_t reducers = 0;   // sum tail: CTAs per signal that reduce the residue rows
    uint64_t k1_capacity = 0;  // co-resident K1 CTAs on the device
    bool mu0 = false;
    uint64_t W = 0;
    // device allocations
    void* tables = nullptr;
    pftdev::PairEntry* d_pairtab = nullptr;
    double2* d_tcfrag = nullptr;  // k1_tc plans: [pairs][8] B fragments
    double2* d_w = nullptr;
    double2 phase0{1.0, 0.0}, phaseh{1.0, 0.0};
    double2* d_omega = nullptr;
    // Bluestein K2 (K2_BLUESTEIN): chirp h_c, FFT_L of the conjugate chirp kernel / L, omega_L
    uint32_t bl_L = 0;
    void* bl_tables = nullptr;
    double2 *d_chirp = nullptr, *d_chirp_hat = nullptr, *d_omega_L = nullptr;
    double* d_post_powers = nullptr;
    double2* d_post_twiddles = nullptr;
    void* d_ws = nullptr;  // the plan's own batch-1 workspace (executes with d_ws == NULL, finalize)

    // Staging sets of pft_execute_host: device input/output buffers, a workspace and a stream,
    // allocated on first use and reused; one set per concurrent caller (SPEC.md:263-265:
    // concurrent executes on one plan), so no call allocates in the steady state.
    struct Staging {
        size_t batch = 0;
        double2 *din = nullptr, *dout = nullptr;
        void* ws = nullptr;
        cudaStream_t st = nullptr;
    };
    std::mutex staging_mu;
    std::vector<Staging*> staging_free;
    std::vector<Staging*> staging_all;

    ~pft_dplan_s() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (Staging* s : staging_all) {
            cudaFree(s->din);
            cudaFree(s->dout);
            cudaFree(s->ws);
            if (s->st) cudaStreamDestroy(s->st);
            delete s;
        }
        if (tables) cudaFree(tables);
        if (bl_tables) cudaFree(bl_tables);
        if (d_ws) cudaFree(d_ws);
        cudaSetDevice(prev);
    }

    size_t slab_elems() const { return (size_t)host.p * host.r; }
    size_t counters_per_signal() const { return sum_tail ? P2 + 2 : (k2_tail || k2_workers) ? 2 : 0; }
    size_t data_elems() const { return sum_tail ? std::max<size_t>(slab_elems(), (size_t)P2 * W) : slab_elems(); }
    // workspace layout (kernels.cuh): header, then per signal {control words, data}
    size_t ctl_bytes() const { return pftdev::ws_align(4 * counters_per_signal()); }
    size_t signal_bytes() const { return ctl_bytes() + pftdev::ws_align(data_elems() * sizeof(double2)); }
    size_t workspace_bytes(size_t batch) const {
        return pftdev::kWsHeaderBytes + std::max<size_t>(batch, 1) * signal_bytes();
    }
    struct WsView {
        unsigned* bar;       // grid barrier {count, generation}
        int* status;         // non-finite flag word
        unsigned* arrivals;  // signal 0's control words
        double2* Y;          // signal 0's data
        uint64_t y_stride;   // elements per signal block
        uint64_t ctl_stride; // words per signal block
    };
    WsView ws_view(void* base) const {
        char* b = static_cast<char*>(base);
        WsView v;
        v.bar = reinterpret_cast<unsigned*>(b);
        v.status = reinterpret_cast<int*>(b + pftdev::kWsStatusOffset);
        v.arrivals = reinterpret_cast<unsigned*>(b + pftdev::kWsHeaderBytes);
        v.Y = reinterpret_cast<double2*>(b + pftdev::kWsHeaderBytes + ctl_bytes());
        v.y_stride = signal_bytes() / sizeof(double2);
        v.ctl_stride = signal_bytes() / sizeof(unsigned);
        return v;
    }
    int* own_status() const { return ws_view(d_ws).status; }
    // signals a K1 CTA holds for a contiguous batch of this size (see run_execute)
    uint32_t signals_per_cta(size_t batch) const {
        if (!sum_tail || P2 != 1 || gsig_max <= 1 || batch < 2) return 1;
        uint32_t G = gsig_max;
        while (G > 1 && batch / G < 2 * k1_capacity) G >>= 1;
        return G;
    }
    bool fused(size_t batch) const {
        return allow_fuse && !sum_tail && k2_mode == pftdev::K2_FFT &&
               pftdev::k2_smem_bytes(host.r, (uint32_t)P2) <= (size_t)k1_stages * pftdev::k1_stage_bytes(host.r) &&
               P2 * batch <= k1_capacity;
    }

    pftdev::K1Params k1_params(const ShardLayout& v, const double2* a, uint64_t row_stride, size_t batch_stride,
                               double2* Y, uint64_t y_stride, bool pdl) const {
        pftdev::K1Params P{};
        P.a = a;
        P.row_stride = row_stride;
        P.batch_stride = batch_stride;
        P.gp0 = (uint32_t)v.pair_begin;
        P.gp_end = (uint32_t)v.pair_end;
        P.fcol0 = (int32_t)v.front_col;
        P.mcol0 = (int32_t)v.mirror_col;
        P.single0_col = (int32_t)v.single0_col;
        P.singleh_col = (int32_t)v.singleh_col;
        P.phase0 = phase0;
        P.phaseh = phaseh;
        P.pairtab = d_pairtab;
        P.tcfrag = d_tcfrag;
        P.w = d_w;
        P.omega = d_omega;
        P.P1 = (uint32_t)P1;
        P.P2 = (uint32_t)P2;
        P.rows = (uint32_t)P1;
        P.gsig = 1;
        P.fft = fft;
        P.stages = k1_stages;
        P.pdl = pdl ? 1 : 0;
        P.split = 1;
        P.Y = Y;
        P.y_stride = y_stride;
        return P;
    }

    pftdev::K2Params k2_params(const double2* Y, uint64_t y_stride, double2* out, int* status) const {
        pftdev::K2Params P{};
        P.Y = Y;
        P.y_stride = y_stride;
        P.post_powers = d_post_powers;
        P.post_twiddles = d_post_twiddles;
        P.omega = d_omega;
        P.p = host.p;
        P.P1 = (uint32_t)P1;
        P.P2 = (uint32_t)P2;
        P.W = W;
        const int64_t first = host.mu - (int64_t)host.M;
        P.first_mod_p = mod_index(first, host.p);
        P.first_mod_p1 = (uint32_t)mod_index(first, P1);
        P.inv_p = 1.0 / (double)host.p;
        P.mode = k2_mode;
        P.k2_ctas = k2_ctas;
        P.release_next = 1;  // a following K1 only streams early when its execute asked for it
        P.fft2 = fft2;
        P.chirp = d_chirp;
        P.chirp_hat = d_chirp_hat;
        P.omega_L = d_omega_L;
        P.L = bl_L;
        P.bl_group = bl_L ? pftdev::k2_bluestein_group(bl_L) : 1;
        P.out = out;
        P.status = status;
        return P;
    }
};

namespace {

pft_dplan_s* dp(pft_dplan_t d) {
    PFT_REQUIRE(d != nullptr, "null device plan");
    return d;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    if (!fn) fail(PFT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    return fn;
}

// 4-D view of the input for K1's bulk tensor copies: (2*row_len doubles of a row, residue
// c, k1, signal) with row k = c + P2 k1 at base + k * row_stride elements.  Boxes of
// 16 rows x 32 columns; out-of-range coordinates (including negative) are zero-filled.
// rows: rows per CTA in the k1 dimension (P1; gsig * P1 when a CTA holds gsig consecutive signals of a
// contiguous batch -- P2 = 1 plans only -- and `batch` then counts the groups, `batch_stride` a group).
CUtensorMap make_input_map(const pft_dplan_s* d, const void* base, uint64_t row_len, uint64_t row_stride,
                           size_t batch, size_t batch_stride, uint64_t rows = 0) {
    PFT_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, "input must be 16-byte aligned");
    CUtensorMap map;
    if (!rows) rows = d->P1;
    const cuuint64_t dims[4] = {2 * std::max<uint64_t>(row_len, 1), d->P2, rows, std::max<size_t>(batch, 1)};
    const cuuint64_t row_bytes = row_stride * 16;
    const cuuint64_t strides[3] = {row_bytes, row_bytes * d->P2,
                                   (batch > 1 ? batch_stride : rows * d->P2 * row_stride) * 16};
    // tensor-core plans: 8-pair half boxes (128-byte rows) with the 128-byte swizzle
    const bool tc = pftdev::k1_tc(d->host.r);
    const cuuint32_t box[4] = {(cuuint32_t)(tc ? pftdev::K1_CP : 2 * pftdev::K1_CP), 1, (cuuint32_t)pftdev::K1_BR, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims,
                                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            tc ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(PFT_ERR_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
    return map;
}

// ws: a workspace of workspace_bytes(>= batch) bytes (header + per-signal blocks, zeroed once).
// pdl: K1 may start streaming before the preceding kernel on `st` completes
// (PFT_EXEC_OVERLAP_PREVIOUS: the caller guarantees `in` is not that kernel's output).
void run_execute(pft_dplan_s* d, const double2* in, size_t batch, size_t in_stride, double2* out, void* ws,
                 cudaStream_t st, bool pdl) {
    const ShardLayout v = shard_layout(d->host.q, 1, 0);
    const CUtensorMap map = make_input_map(d, in, v.row_len, d->host.q, batch, in_stride);
    const pft_dplan_s::WsView w = d->ws_view(ws);
    auto P1 = d->k1_params(v, in, d->host.q, in_stride, w.Y, w.y_stride, pdl);
    auto P2 = d->k2_params(w.Y, w.y_stride, out, w.status);
    P1.arrivals = w.arrivals;
    P1.ctl_stride = w.ctl_stride;
    // extents for checked builds (PFT_BOUND): what this call may address
    P1.in_elems = (uint64_t)(batch - 1) * in_stride + d->host.N;
    P1.y_elems = (uint64_t)(batch - 1) * w.y_stride + d->data_elems();
    P1.ctl_words = (uint64_t)(batch - 1) * w.ctl_stride + d->counters_per_signal();
    P2.y_elems = P1.y_elems;
    P2.out_elems = (uint64_t)batch * d->W;
    // An isolated transform (no overlap with a neighbour) whose grid leaves half the CTA slots
    // idle runs two CTAs (a cluster) per residue class, each streaming half of the column chunks:
    // one transform then fills both slots of every SM (C2b: 128 -> 256 CTAs).
    if (!pdl && d->allow_split && !d->fused(batch) && 2 * d->P2 * batch <= d->k1_capacity && d->host.q >= 4 * pftdev::K1_CP)
        P1.split = 2;
    if (d->sum_tail) {
        P1.sum_tail = 1;
        P1.reducers = d->reducers;
        P1.k2 = P2;
        // Short batched signals with one residue class each (P2 = 1: the 2-D passes): a CTA holds
        // gsig consecutive signals of a contiguous batch as one row block of gsig * P1 rows -- the
        // contraction is per row, the first FFT pass runs gsig * r columns of length P1, the
        // direct tail gsig * W outputs -- so launch, prologue, FFT-stage and tail latencies are
        // paid once per gsig signals (2-D rows pass 4096 x 4096: 104 -> 7x us).  Taken when the
        // row block still fits two CTAs per SM and the groups still fill the device twice over.
        if (P1.split <= 1 && in_stride == d->host.N) {
            const uint32_t G = d->signals_per_cta(batch);
            if (G > 1) {
                const size_t groups = batch / G, rem = batch % G;
                auto Pg = P1;
                Pg.rows = G * (uint32_t)d->P1;
                Pg.gsig = G;
                Pg.stages = pftdev::k1_pick_stages(d->host.r, Pg.rows);
                Pg.batch_stride = (uint64_t)G * in_stride;
                const CUtensorMap mg = make_input_map(d, in, v.row_len, d->host.q, groups, (size_t)G * in_stride, Pg.rows);
                cuda_check(pftdev::launch_k1(mg, Pg, d->host.r, (uint32_t)groups, d->mu0, st), "K1 (signal groups) launch");
                if (rem) {  // the last batch % gsig signals, one per CTA
                    const size_t off = groups * G;
                    auto Pr = P1;
                    Pr.a = in + off * in_stride;
                    Pr.k2.out = out + off * d->W;
                    Pr.in_elems = (uint64_t)(rem - 1) * in_stride + d->host.N;
                    Pr.k2.out_elems = (uint64_t)rem * d->W;
                    const CUtensorMap mr = make_input_map(d, in + off * in_stride, v.row_len, d->host.q, rem, in_stride);
                    cuda_check(pftdev::launch_k1(mr, Pr, d->host.r, (uint32_t)rem, d->mu0, st), "K1 (remainder) launch");
                }
                return;
            }
        }
        cuda_check(pftdev::launch_k1(map, P1, d->host.r, (uint32_t)batch, d->mu0, st), "K1 launch");
        return;
    }
    if (d->k2_tail) {
        P1.k2_tail = 1;
        P1.k2_group = d->k2_group;
        P1.reducers = d->reducers;
        P1.k2 = P2;
        cuda_check(pftdev::launch_k1(map, P1, d->host.r, (uint32_t)batch, d->mu0, st), "K1 (K2 tail) launch");
        return;
    }
    if (d->fused(batch)) {
        P1.fused = 1;
        P1.bar = w.bar;
        P1.k2 = P2;
        cuda_check(pftdev::launch_k1(map, P1, d->host.r, (uint32_t)batch, d->mu0, st), "K1 (fused) launch");
        return;
    }
    if (d->k2_workers && batch == 1 && pdl) {  // one kernel: streamers + K2 workers in the slots they leave free
        P1.workers = d->k2_workers;
        P1.k2 = P2;
        cuda_check(pftdev::launch_k1(map, P1, d->host.r, (uint32_t)batch, d->mu0, st), "K1 (K2 workers) launch");
        return;
    }
    if (d->ring_ok && batch == 1) {  // slab by bulk copy, stages on its own layout (C2c isolated 70.9 -> 65.4 us)
        P2.ring = 1;
        P2.k2_ctas = d->ring_ctas ? d->ring_ctas : (uint32_t)d->P1;
    }
    cuda_check(pftdev::launch_k1(map, P1, d->host.r, (uint32_t)batch, d->mu0, st), "K1 launch");
    cuda_check(pftdev::launch_k2(P2, d->host.r, (uint32_t)batch, st), "K2 launch");
}

}  // namespace

extern "C" {

const char* pft_version(void) { return "pft-b200 " PFT_BUILD_DESC " sm_100a"; }

pft_status pft_select_divisor_device(pft_table_t t, uint64_t N, uint64_t M, double eps, int n_sms, uint64_t* p,
                                     int* r, double* est_us) {
    PFT_API_BEGIN
    PFT_REQUIRE(t != nullptr, "null table handle");
    PFT_REQUIRE(n_sms > 0, "n_sms must be positive");
    const DivisorChoice c = select_divisor_device(t->table, N, M, eps, n_sms);
    if (p) *p = c.p;
    if (r) *r = c.r;
    if (est_us) *est_us = c.cost;
    PFT_API_END
}

pft_status pft_select_divisor_sharded(pft_table_t t, uint64_t N, uint64_t M, double eps, int n_sms, int world,
                                      uint64_t* p, int* r, double* est_us) {
    PFT_API_BEGIN
    PFT_REQUIRE(t != nullptr, "null table handle");
    PFT_REQUIRE(n_sms > 0, "n_sms must be positive");
    const DivisorChoice c = rank_divisors_sharded(t->table, N, M, eps, n_sms, world).front();
    if (p) *p = c.p;
    if (r) *r = c.r;
    if (est_us) *est_us = c.cost;
    PFT_API_END
}

pft_status pft_dplan_device(pft_dplan_t d, int* device) {
    PFT_API_BEGIN
    PFT_REQUIRE(d != nullptr && device != nullptr, "dplan_device: bad arguments");
    *device = d->device;
    PFT_API_END
}

// Measured choice among the model's best candidates ("measured rather
// than modelled"): each candidate p is planned, uploaded and timed over `reps` back-to-back
// executes of the caller's device input on a private stream (after 3 warm-up executes).
pft_status pft_autotune_divisor(pft_table_t t, uint64_t N, uint64_t M, int64_t mu, double eps, int device,
                                const pft_c128* d_in, size_t batch, int n_candidates, uint64_t* p, double* us) {
    PFT_API_BEGIN
    PFT_REQUIRE(t != nullptr && d_in != nullptr && p != nullptr, "autotune_divisor: bad arguments");
    PFT_REQUIRE(n_candidates >= 1, "autotune_divisor: n_candidates < 1");
    const int ndev = usable_device_count();
    if (ndev == 0) fail(PFT_ERR_NO_DEVICE, "no CUDA device visible (this library has no CPU fallback)");
    PFT_REQUIRE(device >= 0 && device < ndev, "autotune_divisor: device ordinal out of range");
    DeviceGuard guard(device);
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    batch = std::max<size_t>(batch, 1);
    PFT_REQUIRE(batch <= 65535, "autotune_divisor: batch > 65535");
    const auto ranked = rank_divisors_device(t->table, N, M, eps, prop.multiProcessorCount, batch);
    struct Res {
        cudaStream_t st = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        double2* out = nullptr;
        void* ws = nullptr;
        ~Res() {
            if (ws) cudaFree(ws);
            if (out) cudaFree(out);
            if (e0) cudaEventDestroy(e0);
            if (e1) cudaEventDestroy(e1);
            if (st) cudaStreamDestroy(st);
        }
    } res;
    cuda_check(cudaStreamCreateWithFlags(&res.st, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreate(&res.e0), "cudaEventCreate");
    cuda_check(cudaEventCreate(&res.e1), "cudaEventCreate");
    cuda_check(cudaMalloc(&res.out, (2 * M + 1) * batch * sizeof(double2)), "cudaMalloc(out)");
    const int reps = batch > 1 ? 3 : 20;
    double best_us = 0.0;
    uint64_t best_p = 0;
    const size_t n = std::min<size_t>((size_t)n_candidates, ranked.size());
    for (size_t i = 0; i < n; ++i) {
        pft_hplan_s hp{build_plan(t->table, N, M, mu, ranked[i].p, eps)};
        pft_dplan_opts o{};
        o.device = device;
        o.batch_hint = batch;
        pft_dplan_t dpl = nullptr;
        if (pft_dplan_create(&hp, &o, &dpl) != PFT_OK) continue;  // infeasible decomposition
        std::unique_ptr<pft_dplan_s> guard_plan(dpl);
        const auto* in = reinterpret_cast<const double2*>(d_in);
        void* ws = dpl->d_ws;
        if (batch > 1) {
            if (res.ws) cudaFree(res.ws);
            res.ws = nullptr;
            const size_t wb = dpl->workspace_bytes(batch);
            cuda_check(cudaMalloc(&res.ws, wb), "cudaMalloc(workspace)");
            cuda_check(cudaMemset(res.ws, 0, wb), "cudaMemset(workspace)");
            ws = res.ws;
        }
        // the same input every time (never written by the previous execute): PDL overlap on,
        // as in a stream of independent transforms
        for (int w = 0; w < 3; ++w) run_execute(dpl, in, batch, N, res.out, ws, res.st, true);
        cuda_check(cudaEventRecord(res.e0, res.st), "cudaEventRecord");
        for (int k = 0; k < reps; ++k) run_execute(dpl, in, batch, N, res.out, ws, res.st, true);
        cuda_check(cudaEventRecord(res.e1, res.st), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(res.e1), "cudaEventSynchronize");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, res.e0, res.e1), "cudaEventElapsedTime");
        const double per = 1e3 * ms / reps;
        if (best_p == 0 || per < best_us) {
            best_us = per;
            best_p = ranked[i].p;
        }
    }
    if (best_p == 0) fail(PFT_ERR_UNSUPPORTED, "autotune_divisor: no candidate could be planned on the device");
    *p = best_p;
    if (us) *us = best_us;
    PFT_API_END
}

pft_status pft_device_count(int* n) {
    PFT_API_BEGIN
    PFT_REQUIRE(n != nullptr, "n is null");
    *n = usable_device_count();
    PFT_API_END
}

pft_status pft_dplan_create(pft_hplan_t plan, const pft_dplan_opts* opts, pft_dplan_t* out) {
    PFT_API_BEGIN
    PFT_REQUIRE(plan && out, "dplan_create: bad arguments");
    *out = nullptr;
    const HostPlan& H = plan->plan;
    const int device = opts ? opts->device : 0;
    const int ndev = usable_device_count();
    if (ndev == 0) fail(PFT_ERR_NO_DEVICE, "no CUDA device visible (this library has no CPU fallback)");
    PFT_REQUIRE(device >= 0 && device < ndev, "dplan_create: device ordinal out of range");
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        fail(PFT_ERR_NO_DEVICE, "device " + std::to_string(device) + " is sm_" + std::to_string(prop.major) +
                                    std::to_string(prop.minor) + "; this build targets sm_100a only");
    if (H.p >= (1ull << 32)) fail(PFT_ERR_UNSUPPORTED, "p >= 2^32");
    DeviceGuard guard(device);

    auto d = std::make_unique<pft_dplan_s>();
    d->device = device;
    d->host.N = H.N;
    d->host.M = H.M;
    d->host.mu = H.mu;
    d->host.p = H.p;
    d->host.q = H.q;
    d->host.r = H.r;
    d->host.epsilon = H.epsilon;
    d->host.achieved_epsilon = H.achieved_epsilon;
    d->host.plan_id = H.plan_id;
    d->W = 2 * H.M + 1;
    d->allow_split = !(opts && opts->k1_split == 1);
    PFT_REQUIRE(!opts || opts->reserved == 0, "dplan_create: reserved options must be 0");
    PFT_REQUIRE(!opts || (opts->k1_split >= 0 && opts->k1_split <= 1), "dplan_create: k1_split must be 0 or 1");
    const int pass2 = opts ? opts->second_pass : PFT_PASS2_AUTO;
    const int k2_at = opts ? opts->k2_at : PFT_K2_AT_AUTO;
    PFT_REQUIRE(pass2 >= PFT_PASS2_AUTO && pass2 <= PFT_PASS2_K2_BLUESTEIN, "dplan_create: unknown second_pass");
    PFT_REQUIRE(k2_at >= PFT_K2_AT_AUTO && k2_at <= PFT_K2_AT_FUSED, "dplan_create: unknown k2_at");
    PFT_REQUIRE(!opts || (opts->tail_ctas >= 0 && opts->k2_grid_ctas >= 0), "dplan_create: negative CTA count");
    const int tail_ctas = opts ? opts->tail_ctas : 0;
    uint64_t p2 = opts && opts->p2 ? opts->p2 : 0;
    const size_t batch_hint = opts && opts->batch_hint > 1 ? (size_t)opts->batch_hint : 1;
    if (!p2 && (pass2 == PFT_PASS2_AUTO || pass2 == PFT_PASS2_SUM_TAIL)) {  // sum tail, when it pays (or forced)
        p2 = choose_p2_sum(H.p, H.r, prop.multiProcessorCount, batch_hint);
        // batched plans (batch_hint > 1) always take the sum tail when it fits: a K2 grid of
        // P1 x batch CTAs was 2.5-16x slower at every batched shape measured
        // (tools/probe_cols.py: 129 x 4096, M = 64: 31 vs 12 us; 513 x 1024, M = 32: 92 vs 11 us)
        if (p2 && pass2 == PFT_PASS2_AUTO && batch_hint <= 1 && !sum_tail_pays(H.N, d->W, p2, H.r)) p2 = 0;
    }
    if (!p2) p2 = choose_p2(H.p, H.r, batch_hint);
    if (p2 == 0 || H.p % p2 != 0) fail(PFT_ERR_INVALID_ARGUMENT, "dplan_create: p2 must divide p");
    d->P2 = p2;
    d->P1 = H.p / p2;
    if (d->P1 > 1 && !factor_radices((uint32_t)d->P1, d->fft))
        fail(PFT_ERR_UNSUPPORTED, "dplan_create: P1 = p/P2 has a prime factor > 64");
    if (d->P1 <= 1) d->fft.n = 1;
    if (!k1_feasible(d->P1, H.r))
        fail(PFT_ERR_UNSUPPORTED, "dplan_create: P1 * r too large for K1 shared memory; choose a larger p2");
    d->k1_stages = (opts && opts->k1_stages) ? (uint32_t)opts->k1_stages : pftdev::k1_pick_stages(H.r, (uint32_t)d->P1);
    PFT_REQUIRE(d->k1_stages >= (uint32_t)pftdev::k1_min_stages(H.r) && d->k1_stages <= (uint32_t)pftdev::K1_MAX_STAGES,
                "dplan_create: k1_stages out of [min stages (3 or 4), 8]");
    // K2 form: length-P2 FFT when it fits shared memory (fastest measured), else the dot form,
    // else the direct global form.
    {
        const bool fft_ok = k2_fft_feasible(d->P2, H.r);
        const bool dot_ok = pftdev::k2_dot_smem_bytes(H.r, (uint32_t)d->P2) <= kK2SmemLimit;
        // L2 form when there are few output bins per m1 (W <= 2 P1, e.g. C1); it needs no shared
        // memory and parks beside K1 under PDL.  Otherwise the FFT form (the L2 form is
        // latency-bound at C2b/C4's 2049 / 2001 bins) -- unless the sum tail below applies
        // (measured C2b 49 vs 54 us, C4 35 vs 45 us per transform).
        const bool l2_ok = d->P2 <= 1024 && double(d->W) * d->P2 <= 64.0 * 1024 * 1024;
        uint32_t bl_L = 1;
        while (bl_L < 2 * d->P2 - 1) bl_L <<= 1;
        const bool bl_ok = d->P2 > 1 && bl_L <= pftdev::K2B_MAX_L && d->W <= 4ull * pftdev::K2_THREADS * d->P1;
        if (pass2 == PFT_PASS2_K2_FFT && fft_ok) d->k2_mode = pftdev::K2_FFT;
        else if (pass2 == PFT_PASS2_K2_DOT && dot_ok) d->k2_mode = pftdev::K2_DOT;
        else if (pass2 == PFT_PASS2_K2_DIRECT) d->k2_mode = pftdev::K2_DIRECT;
        else if (pass2 == PFT_PASS2_K2_L2) d->k2_mode = pftdev::K2_L2;
        else if (pass2 == PFT_PASS2_SUM_TAIL) d->k2_mode = pftdev::K2_FFT;  // with the sum tail below
        else if (l2_ok && d->W <= 2 * d->P1) d->k2_mode = pftdev::K2_L2;  // few bins per m1 (C1)
        else if (pass2 == PFT_PASS2_K2_BLUESTEIN && bl_ok) d->k2_mode = pftdev::K2_BLUESTEIN;
        else if (fft_ok) d->k2_mode = pftdev::K2_FFT;
        // P2 with a prime factor > 64 (no Stockham radix schedule) and many bins per m1: chirp-z
        // (two length-L FFTs per column) beats the dot / direct forms' O(bins x P2) per column
        else if (bl_ok && d->W >= 32 * d->P1) d->k2_mode = pftdev::K2_BLUESTEIN;
        else if (dot_ok) d->k2_mode = pftdev::K2_DOT;
        else d->k2_mode = pftdev::K2_DIRECT;
        if (d->k2_mode == pftdev::K2_FFT) {
            if (d->P2 > 1) factor_radices((uint32_t)d->P2, d->fft2);
            else d->fft2.n = 1;
        }
        if (d->k2_mode == pftdev::K2_BLUESTEIN) {
            d->bl_L = bl_L;
            factor_radices(bl_L, d->fft2);
        }
        // K2 CTAs (each loops over m1): few enough to all be resident beside K1 (opts override)
        d->k2_ctas = opts && opts->k2_grid_ctas > 0 ? (uint32_t)opts->k2_grid_ctas : 0;
        d->allow_fuse = k2_at == PFT_K2_AT_FUSED;
        // Sum tail when it pays (sum_tail_pays): K1 finishes the transform itself (see
        // k1_sum_tail).  Needs the ring to hold the FFT scratch and the tail scratch.  Forced
        // off by the K2 forms, forced on (if feasible) by PFT_PASS2_SUM_TAIL.
        const bool fits = sizeof(double2) * H.r * d->P1 +
                              pftdev::k1_sum_scratch_bytes((uint32_t)d->P1, (uint32_t)d->P2) <=
                          pftdev::k1_min_ring_bytes(H.r);
        d->sum_tail = fits && (pass2 == PFT_PASS2_SUM_TAIL ||
                               (pass2 == PFT_PASS2_AUTO && (batch_hint > 1 || sum_tail_pays(H.N, d->W, d->P2, H.r))));
        // reducing CTAs per signal: one per 64 outputs (measured best at C2b/C4: 32; more
        // reducers hold more SM slots from the next transform), opts override
        d->reducers = (uint32_t)std::min<uint64_t>(d->P2, std::max<uint64_t>(1, (d->W + 63) / 64));
        if (tail_ctas > 0) d->reducers = (uint32_t)std::min<uint64_t>(d->P2, (uint64_t)tail_ctas);
        // Last-arrival K2 tail (k1_k2_tail) when K2 takes the FFT form and the tail is short
        // against the stream: the columns go through the FFT in groups whose Z + scratch fit
        // the ring.  Workers hold their SM slots, and a K1 CTA of the next transform that starts
        // late finishes late (each CTA streams a fixed 1/P2 of the input), so the tail's m1
        // rounds (~15 us each beside a streaming CTA, per-CTA timestamps at C2c) must stay <= 10% of
        // the stream: C5 (2^30) gains 6% (3099 -> 2907 us), C2c (2^24, 2 rounds) loses (67 -> 77
        // us at 1 round).  k2_at: PFT_K2_AT_TAIL forces it on (if feasible), _GRID off.
        if (!d->sum_tail && d->k2_mode == pftdev::K2_FFT && !d->allow_fuse && k2_at != PFT_K2_AT_GRID &&
            pftdev::k1_k2_tail_instantiated(H.r)) {
            const size_t ring = (size_t)d->k1_stages * pftdev::k1_stage_bytes(H.r);
            const size_t fixed = pftdev::k1_k2_tail_bytes(0, (uint32_t)d->P2);
            const size_t per_col = 2 * sizeof(double2) * d->P2;
            const uint64_t gmax = ring > fixed ? (ring - fixed) / per_col : 0;
            if (gmax >= 1) {
                const uint64_t groups = ((uint64_t)H.r + gmax - 1) / gmax;
                d->k2_group = (uint32_t)(((uint64_t)H.r + groups - 1) / groups);
                d->k2_tail = true;
                // workers per signal: all m1 in one round when P1 is small, else 64 (opts override)
                d->reducers = (uint32_t)std::min<uint64_t>(d->P1, std::min<uint64_t>(d->P2, 64));
                if (tail_ctas > 0)
                    d->reducers = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(d->P1, d->P2), (uint64_t)tail_ctas);
                const double rounds = (double)((d->P1 + d->reducers - 1) / d->reducers);
                const double stream_us = 16.0 * (double)H.N * (double)batch_hint / 6.5e6;
                if (k2_at != PFT_K2_AT_TAIL && rounds * 15.0 > 0.10 * stream_us) d->k2_tail = false;
            }
        }
    }
    d->mu0 = std::all_of(H.phase.begin(), H.phase.end(), [](const cplx& z) { return z == cplx(1.0, 0.0); });

    // omega_p^t = e^{-2 pi i t / p}, exactly reduced
    std::vector<cplx> omega(H.p);
#pragma omp parallel for schedule(static)
    for (long long t = 0; t < (long long)H.p; ++t) omega[t] = cispi_frac(-2 * (__int128)t, H.p);

    // pair table {Re phase_l, Im phase_l, t_l, t_l^h} for l in [0, L), h = ceil(r/2) (the first
    // power of the upper j half when K1 splits j over two lanes; formed by the same ascending
    // repeated multiplication as the kernel's power chain, so both splits see identical powers),
    // zero-padded so a chunk read past the last pair stays in bounds
    const uint64_t L = (H.q + 1) / 2;
    const uint64_t n_pt = L + 2 * pftdev::K1_CP;
    // (tensor-core plans, k1_tc: t_l^17 for r = 18, the moment outside the two DMMA tiles).
    // Tensor-core plans also get the B-fragment table {t_l^(2+2g), t_l^(1+2g)}, g in [8]
    // (zero where j >= r), same ascending powers.
    const bool tc = pftdev::k1_tc(H.r);
    const int h_split = tc ? H.r - 1 : (H.r + 1) / 2;  // t^h serves the two-lane j split
    std::vector<pftdev::PairEntry> pairtab(n_pt, pftdev::PairEntry{0.0, 0.0, 0.0, 0.0});
    std::vector<double> tcfrag(tc ? n_pt * 16 : 0, 0.0);
    for (uint64_t l = 0; l < L; ++l) {
        const double t = H.tvals[l];
        double pw[32];  // r <= 25
        pw[0] = 1.0;
        for (int j = 1; j < 32; ++j) pw[j] = pw[j - 1] * t;  // pw[1] = 1 * t = t exactly
        pairtab[l] = {H.phase[l].real(), H.phase[l].imag(), t, pw[h_split]};
        if (tc) {
            for (int g = 0; g < 8; ++g) {  // column g stored at g ^ 2 (l & 3) (bank spread, k1_tc_stage)
                const int je = 2 + 2 * g, jo = 1 + 2 * g, gs = g ^ (2 * (int)(l & 3));
                tcfrag[l * 16 + 2 * gs] = je < H.r ? pw[je] : 0.0;
                tcfrag[l * 16 + 2 * gs + 1] = jo < H.r ? pw[jo] : 0.0;
            }
        }
    }
    d->phase0 = make_double2(H.phase[0].real(), H.phase[0].imag());
    if (H.q % 2 == 0) d->phaseh = make_double2(H.phase[H.q / 2].real(), H.phase[H.q / 2].imag());

    // one allocation for all tables, 256-byte aligned pieces
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t b_pt0 = al(n_pt * sizeof(pftdev::PairEntry)), b_w = al(H.r * sizeof(double2)),
                 b_om = al(H.p * sizeof(double2)), b_pp = al(d->W * H.r * sizeof(double)),
                 b_pt = al(d->W * sizeof(double2)), b_tc = al(tcfrag.size() * sizeof(double));
    const size_t total = b_pt0 + b_w + b_om + b_pp + b_pt + b_tc;
    cuda_check(cudaMalloc(&d->tables, total), "cudaMalloc(tables)");
    char* base = static_cast<char*>(d->tables);
    d->d_pairtab = reinterpret_cast<pftdev::PairEntry*>(base);
    d->d_w = reinterpret_cast<double2*>(base + b_pt0);
    d->d_omega = reinterpret_cast<double2*>(base + b_pt0 + b_w);
    d->d_post_powers = reinterpret_cast<double*>(base + b_pt0 + b_w + b_om);
    d->d_post_twiddles = reinterpret_cast<double2*>(base + b_pt0 + b_w + b_om + b_pp);
    if (tc) {
        d->d_tcfrag = reinterpret_cast<double2*>(base + b_pt0 + b_w + b_om + b_pp + b_pt);
        cuda_check(cudaMemcpy(d->d_tcfrag, tcfrag.data(), tcfrag.size() * sizeof(double), cudaMemcpyHostToDevice),
                   "upload tensor-core fragment table");
    }
    cuda_check(cudaMemcpy(d->d_pairtab, pairtab.data(), n_pt * sizeof(pftdev::PairEntry), cudaMemcpyHostToDevice),
               "upload pair table");
    cuda_check(cudaMemcpy(d->d_w, H.w.data(), H.r * sizeof(double2), cudaMemcpyHostToDevice), "upload w");
    cuda_check(cudaMemcpy(d->d_omega, omega.data(), H.p * sizeof(double2), cudaMemcpyHostToDevice), "upload omega");
    cuda_check(cudaMemcpy(d->d_post_powers, H.post_powers.data(), d->W * H.r * sizeof(double), cudaMemcpyHostToDevice),
               "upload post_powers");
    cuda_check(cudaMemcpy(d->d_post_twiddles, H.post_twiddles.data(), d->W * sizeof(double2), cudaMemcpyHostToDevice),
               "upload post_twiddles");
    if (d->k2_mode == pftdev::K2_BLUESTEIN) {
        // h_c = e^{-pi i c^2 / P2} (exact: c^2 mod 2 P2); kernel b_k = conj(h_k) for |k| < P2 wrapped
        // into length L; its FFT_L / L in long double; omega_L.
        const uint64_t P2 = d->P2, L = d->bl_L;
        std::vector<cplx> chirp(P2), hat(L), omL(L);
        for (uint64_t c = 0; c < P2; ++c) chirp[c] = cispi_frac(-(__int128)((c * c) % (2 * P2)), (__int128)P2);
        std::vector<std::complex<long double>> bk(L, 0.0L);
        for (uint64_t k = 0; k < P2; ++k) {
            const cplx v = std::conj(chirp[k]);
            bk[k] = {v.real(), v.imag()};
            if (k) bk[L - k] = bk[k];
        }
        const long double tau = 6.283185307179586476925286766559005768L;
#pragma omp parallel for schedule(static)
        for (long long t = 0; t < (long long)L; ++t) {
            std::complex<long double> acc = 0.0L;
            for (uint64_t k = 0; k < L; ++k) {
                if (bk[k] == std::complex<long double>(0.0L)) continue;
                const uint64_t e = ((uint64_t)t * k) % L;
                acc += bk[k] * std::polar(1.0L, -tau * (long double)e / (long double)L);
            }
            acc /= (long double)L;
            hat[t] = cplx((double)acc.real(), (double)acc.imag());
        }
        for (uint64_t t = 0; t < L; ++t) omL[t] = cispi_frac(-2 * (__int128)t, (__int128)L);
        cuda_check(cudaMalloc(&d->bl_tables, (P2 + 2 * L) * sizeof(double2)), "cudaMalloc(bluestein tables)");
        d->d_chirp = static_cast<double2*>(d->bl_tables);
        d->d_chirp_hat = d->d_chirp + P2;
        d->d_omega_L = d->d_chirp_hat + L;
        cuda_check(cudaMemcpy(d->d_chirp, chirp.data(), P2 * sizeof(double2), cudaMemcpyHostToDevice), "upload chirp");
        cuda_check(cudaMemcpy(d->d_chirp_hat, hat.data(), L * sizeof(double2), cudaMemcpyHostToDevice), "upload chirp_hat");
        cuda_check(cudaMemcpy(d->d_omega_L, omL.data(), L * sizeof(double2), cudaMemcpyHostToDevice), "upload omega_L");
    }
    cuda_check(pftdev::configure_k1(H.r, (uint32_t)d->P1, d->mu0), "configure K1 (early)");
    cuda_check(pftdev::configure_k1(H.r, (uint32_t)d->P1, d->mu0), "configure K1");
    cuda_check(pftdev::configure_k2(H.r, (uint32_t)d->P2), "configure K2");
    d->k1_capacity = (uint64_t)pftdev::k1_max_active_per_sm(H.r, (uint32_t)d->P1, d->k1_stages, d->mu0) *
                     (uint64_t)prop.multiProcessorCount;
    // Reducers (sum tail) and K2-tail workers hold their SM slots while they wait for the rest
    // of their signal's CTAs.  Forward progress needs a free slot for those CTAs: with CTAs
    // dispatched in launch order only the highest signal in flight can have undispatched CTAs,
    // and its waiting CTAs number at most `reducers`, so reducers < capacity suffices (a PDL
    // dependent grid gets slots only after every CTA of this grid has been dispatched).  The
    // sum tail also keeps them within the slots a transform leaves free (capacity - P2):
    // measured 40 reducers 46.4 us, 48 reducers 53.9 us per transform at C2b.  Caller overrides
    // (tail_ctas) are capped the same way.
    if (d->k1_capacity > 1) {
        const uint64_t cap = d->sum_tail && d->k1_capacity > d->P2 ? d->k1_capacity - d->P2 : d->k1_capacity - 1;
        d->reducers = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(d->reducers, cap));
    }
    // Signals per CTA for P2 = 1 sum-tail plans (see run_execute): the row block gsig * P1 must keep
    // two CTAs per SM, hold its FFT scratch and the tail scratch in the ring
    if (d->sum_tail && d->P2 == 1 && d->P1 > 1 && batch_hint > 1) {
        for (uint32_t G = 4; G > 1; G >>= 1) {
            const uint32_t rows = G * (uint32_t)d->P1;
            const uint32_t stg = pftdev::k1_pick_stages(H.r, rows);
            const size_t ring = (size_t)stg * pftdev::k1_stage_bytes(H.r);
            if (pftdev::k1_smem_bytes(H.r, rows, stg) <= (228 * 1024) / 2 - 1024 &&
                sizeof(double2) * H.r * rows + pftdev::k1_sum_scratch_bytes((uint32_t)d->P1, 1) <= ring) {
                d->gsig_max = G;
                break;
            }
        }
    }
    // Second pass of chained single executes whose K2 is its own grid (many bins: C2c).  A K2 kernel
    // between two K1s keeps the next K1 from starting until this K1 has completed (measured: an
    // empty K2 still costs the chain ~7 us), so the K2 work rides inside K1's grid instead:
    // K2 worker CTAs (k1_k2_worker) in the slots the P2 streamers leave free, taken when their m1
    // rounds (~8 us per m1 beside a streaming K1, measured at C2c) fit within the stream.
    // tail_ctas overrides the count; k2_at = GRID or a caller-chosen k2_grid_ctas turns them off.
    // Executes that do not take the workers (isolated ones, or k2_grid_ctas > 0) run the ring K2
    // kernel (k2_ring) when P2 is a power of two and three slabs fit shared memory: one CTA per
    // m1, or k2_grid_ctas CTAs looping over m1.
    {
        // power-of-two p: the ring forms build ((m - mu)/p)^j in registers, exact only then (the
        // post_powers table's values bit for bit: the ring K2 equals the K2 grid bitwise)
        const bool pow2 = d->P2 >= 4 && (d->P2 & (d->P2 - 1)) == 0 && (H.p & (H.p - 1)) == 0;
        const bool eligible = !d->sum_tail && !d->k2_tail && !d->allow_fuse && d->k2_mode == pftdev::K2_FFT && pow2 &&
                              batch_hint <= 1;
        const uint64_t free_slots = d->k1_capacity > d->P2 ? d->k1_capacity - d->P2 : 0;
        if (eligible && d->k2_ctas == 0 && k2_at != PFT_K2_AT_GRID && pftdev::k1_k2_workers_instantiated(H.r) &&
            pftdev::k1_k2_worker_bytes(H.r, (uint32_t)d->P2) <= pftdev::k1_smem_bytes(H.r, (uint32_t)d->P1, d->k1_stages) &&
            (d->W + d->P1 - 1) / d->P1 <= 2ull * 32 * pftdev::K1_CONSUMER_WARPS && d->P1 <= (uint64_t)pftdev::K1_THREADS &&
            free_slots >= 8) {
            // the fewest workers that keep the fewest m1 rounds: every slot not held by a worker
            // lets a streamer of the next transform start early and stream through the gap in
            // which this transform's streamers run their FFT pass and store the slab (C2c: 32
            // workers 55.9 us, 40 workers 56.8 us, workers that exit at once 48.5 us)
            uint64_t nw = std::min<uint64_t>(free_slots, d->P1);
            const uint64_t min_rounds = (d->P1 + nw - 1) / nw;
            nw = (d->P1 + min_rounds - 1) / min_rounds;
            if (tail_ctas > 0) nw = std::min<uint64_t>(std::min<uint64_t>(free_slots, d->P1), (uint64_t)tail_ctas);
            const double rounds = (double)((d->P1 + nw - 1) / nw);
            const double stream_us = 16.0 * (double)H.N / 6.5e6;
            if (k2_at == PFT_K2_AT_TAIL || rounds * 8.0 <= stream_us) d->k2_workers = (uint32_t)nw;
        }
        if (eligible && d->P2 <= 4ull * pftdev::K2_THREADS &&
            pftdev::k2_ring_smem_bytes(H.r, (uint32_t)d->P2) <= (size_t)227 * 1024) {
            d->ring_ok = true;
            d->ring_ctas = d->k2_ctas;
        }
    }
    // the plan's own batch-1 workspace (after every choice that sizes the control words)
    cuda_check(cudaMalloc(&d->d_ws, d->workspace_bytes(1)), "cudaMalloc(workspace)");
    cuda_check(cudaMemset(d->d_ws, 0, d->workspace_bytes(1)), "cudaMemset(workspace)");
    *out = d.release();
    PFT_API_END
}

void pft_dplan_destroy(pft_dplan_t d) { delete d; }

pft_status pft_dplan_shape(pft_dplan_t d, uint64_t* N, uint64_t* M, int64_t* mu) {
    PFT_API_BEGIN
    const pft_dplan_s* x = dp(d);
    if (N) *N = x->host.N;
    if (M) *M = x->host.M;
    if (mu) *mu = x->host.mu;
    PFT_API_END
}

pft_status pft_dplan_layout(pft_dplan_t d, uint64_t* p1, uint64_t* p2) {
    PFT_API_BEGIN
    if (p1) *p1 = dp(d)->P1;
    if (p2) *p2 = dp(d)->P2;
    PFT_API_END
}

pft_status pft_workspace_bytes(pft_dplan_t d, size_t batch, size_t* bytes) {
    PFT_API_BEGIN
    PFT_REQUIRE(bytes != nullptr, "bytes is null");
    *bytes = dp(d)->workspace_bytes(batch);
    PFT_API_END
}

pft_status pft_partial_bytes(pft_dplan_t d, size_t batch, size_t* bytes) {
    PFT_API_BEGIN
    PFT_REQUIRE(bytes != nullptr, "bytes is null");
    *bytes = dp(d)->slab_elems() * sizeof(double2) * batch;
    PFT_API_END
}

pft_status pft_dplan_signals_per_cta(pft_dplan_t d, size_t batch, int* signals) {
    PFT_API_BEGIN
    PFT_REQUIRE(signals != nullptr, "signals is null");
    *signals = (int)dp(d)->signals_per_cta(batch);
    PFT_API_END
}

pft_status pft_launches_per_execute(pft_dplan_t d, int* launches) {
    PFT_API_BEGIN
    dp(d);
    PFT_REQUIRE(launches != nullptr, "launches is null");
    *launches = (dp(d)->fused(1) || dp(d)->sum_tail || dp(d)->k2_tail) ? 1 : 2;
    PFT_API_END
}

pft_status pft_dplan_second_pass(pft_dplan_t d, int* form) {
    PFT_API_BEGIN
    const pft_dplan_s* x = dp(d);
    PFT_REQUIRE(form != nullptr, "form is null");
    if (x->sum_tail) *form = PFT_PASS2_SUM_TAIL;
    else
        switch (x->k2_mode) {
            case pftdev::K2_FFT: *form = PFT_PASS2_K2_FFT; break;
            case pftdev::K2_DOT: *form = PFT_PASS2_K2_DOT; break;
            case pftdev::K2_L2: *form = PFT_PASS2_K2_L2; break;
            case pftdev::K2_BLUESTEIN: *form = PFT_PASS2_K2_BLUESTEIN; break;
            default: *form = PFT_PASS2_K2_DIRECT; break;
        }
    PFT_API_END
}

pft_status pft_dplan_tail_kind(pft_dplan_t d, int* kind) {
    PFT_API_BEGIN
    const pft_dplan_s* x = dp(d);
    PFT_REQUIRE(kind != nullptr, "kind is null");
    *kind = x->sum_tail ? 1 : x->k2_tail ? 2 : x->fused(1) ? 3 : x->k2_workers ? 4 : 0;
    PFT_API_END
}

pft_status pft_execute_ex(pft_dplan_t dh, const pft_c128* d_in, size_t batch, size_t in_stride, pft_c128* d_out,
                          void* d_ws, void* stream, unsigned flags) {
    PFT_API_BEGIN
    pft_dplan_s* d = dp(dh);
    if (batch == 0) return PFT_OK;
    PFT_REQUIRE(d_in && d_out, "execute: null buffer");
    PFT_REQUIRE(batch <= 65535, "execute: batch > 65535 per call");
    PFT_REQUIRE((flags & ~PFT_EXEC_OVERLAP_PREVIOUS) == 0, "execute: unknown flags");
    if (in_stride == 0) in_stride = d->host.N;
    PFT_REQUIRE(in_stride >= d->host.N || batch == 1, "execute: in_stride < N");
    void* ws = d_ws;
    if (!ws) {
        PFT_REQUIRE(batch == 1, "execute: batch > 1 needs a caller workspace (pft_workspace_bytes)");
        ws = d->d_ws;
    }
    DeviceGuard guard(d->device);
    run_execute(d, reinterpret_cast<const double2*>(d_in), batch, in_stride, reinterpret_cast<double2*>(d_out), ws,
                static_cast<cudaStream_t>(stream), (flags & PFT_EXEC_OVERLAP_PREVIOUS) != 0);
    PFT_API_END
}

pft_status pft_execute(pft_dplan_t dh, const pft_c128* d_in, size_t batch, size_t in_stride, pft_c128* d_out,
                       void* d_ws, void* stream) {
    return pft_execute_ex(dh, d_in, batch, in_stride, d_out, d_ws, stream, PFT_EXEC_DEFAULT);
}

// ------------------------------------------------------------------ 2-D PFT
// Algorithm 4 as two batched 1-D passes: C^{(k1,k2)} = B1^T A B2 followed by the p1 x p2 FFT and
// the Eq. (14) product of per-dimension post factors is, by linearity, the 1-D PFT along axis 2
// of every row followed by the 1-D PFT along axis 1 of every resulting column (identical in
// exact arithmetic; SPEC.md:323 asks only 1e-10 between parenthesizations).  `rows` is the
// plan of axis 2 (length N2, applied to the N1 rows), `cols` the plan of axis 1 (length N1).
// Workspace: [rows ws (batch N1)] [cols ws (batch W2)] [X: N1 x W2] [X^T: W2 x N1] [Z: W2 x W1].
namespace {
size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
struct Ws2d {
    size_t rows_ws, cols_ws, x, xt, z, total;
};
Ws2d ws2d(const pft_dplan_s* rows, const pft_dplan_s* cols) {
    const size_t N1 = cols->host.N, W1 = cols->W, W2 = rows->W;
    Ws2d w{};
    w.rows_ws = al256(rows->workspace_bytes(N1));
    w.cols_ws = al256(cols->workspace_bytes(W2));
    w.x = al256(N1 * W2 * sizeof(double2));
    w.xt = w.x;
    w.z = al256(W2 * W1 * sizeof(double2));
    w.total = w.rows_ws + w.cols_ws + w.x + w.xt + w.z;
    return w;
}

int read_status(const int* d_status, bool reset, cudaStream_t st) {
    int f = 0;
    cuda_check(cudaMemcpyAsync(&f, d_status, sizeof(int), cudaMemcpyDeviceToHost, st), "read status");
    cuda_check(cudaStreamSynchronize(st), "stream synchronize");
    if (reset && f) {
        cuda_check(cudaMemsetAsync(const_cast<int*>(d_status), 0, sizeof(int), st), "reset status");
        cuda_check(cudaStreamSynchronize(st), "stream synchronize");
    }
    return f;
}
}  // namespace

pft_status pft_workspace_bytes_2d(pft_dplan_t rows, pft_dplan_t cols, size_t* bytes) {
    PFT_API_BEGIN
    PFT_REQUIRE(bytes != nullptr, "bytes is null");
    *bytes = ws2d(dp(rows), dp(cols)).total;
    PFT_API_END
}

pft_status pft_execute_2d(pft_dplan_t rows_h, pft_dplan_t cols_h, const pft_c128* d_in, pft_c128* d_out, void* d_ws,
                          void* stream) {
    PFT_API_BEGIN
    pft_dplan_s* rows = dp(rows_h);
    pft_dplan_s* cols = dp(cols_h);
    PFT_REQUIRE(d_in && d_out && d_ws, "execute_2d: null buffer (the workspace is required)");
    PFT_REQUIRE(rows->device == cols->device, "execute_2d: plans on different devices");
    const size_t N1 = cols->host.N, N2 = rows->host.N, W1 = cols->W, W2 = rows->W;
    PFT_REQUIRE(N1 <= 65535 && W2 <= 65535, "execute_2d: N1 and 2*M2+1 must be <= 65535 (batched passes)");
    DeviceGuard guard(rows->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Ws2d w = ws2d(rows, cols);
    char* base = static_cast<char*>(d_ws);
    void* ws_rows = base;
    void* ws_cols = base + w.rows_ws;
    double2* X = reinterpret_cast<double2*>(base + w.rows_ws + w.cols_ws);
    double2* XT = reinterpret_cast<double2*>(base + w.rows_ws + w.cols_ws + w.x);
    double2* Z = reinterpret_cast<double2*>(base + w.rows_ws + w.cols_ws + w.x + w.xt);
    // axis 2: every row (contiguous, length N2) -> X[n1][m2]
    run_execute(rows, reinterpret_cast<const double2*>(d_in), N1, N2, X, ws_rows, st, false);
    cuda_check(pftdev::launch_transpose(X, XT, N1, W2, st), "transpose");
    // axis 1: every column of X (now a contiguous row of X^T, length N1) -> Z[m2][m1]
    run_execute(cols, XT, W2, N1, Z, ws_cols, st, false);
    cuda_check(pftdev::launch_transpose(Z, reinterpret_cast<double2*>(d_out), W2, W1, st), "transpose");
    PFT_API_END
}

pft_status pft_execute_2d_host(pft_dplan_t rows_h, pft_dplan_t cols_h, const pft_c128* h_in, pft_c128* h_out) {
    PFT_API_BEGIN
    pft_dplan_s* rows = dp(rows_h);
    pft_dplan_s* cols = dp(cols_h);
    PFT_REQUIRE(h_in && h_out, "execute_2d_host: null host buffer");
    DeviceGuard guard(rows->device);
    const size_t n_in = cols->host.N * rows->host.N, n_out = cols->W * rows->W;
    const Ws2d w2 = ws2d(rows, cols);
    struct Bufs {
        void *in = nullptr, *out = nullptr, *ws = nullptr;
        cudaStream_t st = nullptr;
        ~Bufs() {
            if (st) cudaStreamDestroy(st);
            cudaFree(in);
            cudaFree(out);
            cudaFree(ws);
        }
    } b;
    cuda_check(cudaStreamCreateWithFlags(&b.st, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaMalloc(&b.in, n_in * sizeof(pft_c128)), "cudaMalloc(input)");
    cuda_check(cudaMalloc(&b.out, n_out * sizeof(pft_c128)), "cudaMalloc(output)");
    cuda_check(cudaMalloc(&b.ws, w2.total), "cudaMalloc(workspace)");
    cuda_check(cudaMemsetAsync(b.ws, 0, w2.total, b.st), "cudaMemset(workspace)");
    cuda_check(cudaMemcpyAsync(b.in, h_in, n_in * sizeof(pft_c128), cudaMemcpyHostToDevice, b.st), "H2D input");
    const pft_status s = pft_execute_2d(rows_h, cols_h, static_cast<const pft_c128*>(b.in),
                                        static_cast<pft_c128*>(b.out), b.ws, b.st);
    if (s != PFT_OK) return s;
    cuda_check(cudaMemcpyAsync(h_out, b.out, n_out * sizeof(pft_c128), cudaMemcpyDeviceToHost, b.st), "D2H output");
    const int f1 = read_status(rows->ws_view(b.ws).status, false, b.st);
    const int f2 = read_status(cols->ws_view(static_cast<char*>(b.ws) + w2.rows_ws).status, false, b.st);
    if (f1 || f2) fail(PFT_ERR_NON_FINITE, "execute_2d: non-finite input entries (non-finite output detected)");
    PFT_API_END
}

pft_status pft_execute_partial(pft_dplan_t dh, const pft_c128* d_in_local, int world, int rank,
                               uint64_t row_stride, pft_c128* d_partial, void* stream) {
    PFT_API_BEGIN
    pft_dplan_s* d = dp(dh);
    PFT_REQUIRE(d_in_local && d_partial, "execute_partial: null buffer");
    const ShardLayout v = shard_layout(d->host.q, world, rank);
    if (row_stride == 0) row_stride = v.row_len;
    PFT_REQUIRE(row_stride >= v.row_len, "execute_partial: row_stride < local row length");
    DeviceGuard guard(d->device);
    const CUtensorMap map = make_input_map(d, d_in_local, v.row_len, row_stride, 1, 0);
    auto P = d->k1_params(v, reinterpret_cast<const double2*>(d_in_local), row_stride, 0,
                          reinterpret_cast<double2*>(d_partial), d->slab_elems(), false);
    P.in_elems = d->host.p * row_stride;
    P.y_elems = d->slab_elems();
    cuda_check(pftdev::launch_k1(map, P, d->host.r, 1, d->mu0, static_cast<cudaStream_t>(stream)), "K1 launch");
    PFT_API_END
}

pft_status pft_finalize(pft_dplan_t dh, const pft_c128* d_partial, size_t batch, pft_c128* d_out, void* stream) {
    PFT_API_BEGIN
    pft_dplan_s* d = dp(dh);
    if (batch == 0) return PFT_OK;
    PFT_REQUIRE(d_partial && d_out, "finalize: null buffer");
    DeviceGuard guard(d->device);
    auto P = d->k2_params(reinterpret_cast<const double2*>(d_partial), d->slab_elems(),
                          reinterpret_cast<double2*>(d_out), d->own_status());
    P.y_elems = batch * d->slab_elems();
    P.out_elems = batch * d->W;
    cuda_check(pftdev::launch_k2(P, d->host.r, (uint32_t)batch, static_cast<cudaStream_t>(stream)), "K2 launch");
    PFT_API_END
}

pft_status pft_workspace_status(pft_dplan_t dh, void* d_ws, void* stream, int* flags, int reset) {
    PFT_API_BEGIN
    pft_dplan_s* d = dp(dh);
    PFT_REQUIRE(flags != nullptr, "flags is null");
    DeviceGuard guard(d->device);
    *flags = read_status(d->ws_view(d_ws ? d_ws : d->d_ws).status, reset != 0, static_cast<cudaStream_t>(stream));
    PFT_API_END
}

pft_status pft_status_query(pft_dplan_t dh, void* stream, int* flags, int reset) {
    return pft_workspace_status(dh, nullptr, stream, flags, reset);
}

pft_status pft_execute_host(pft_dplan_t dh, const pft_c128* h_in, size_t batch, pft_c128* h_out, pft_c128* d_in,
                            pft_c128* d_out, void* stream) {
    PFT_API_BEGIN
    pft_dplan_s* d = dp(dh);
    if (batch == 0) return PFT_OK;
    PFT_REQUIRE(h_in && h_out, "execute_host: null host buffer");
    PFT_REQUIRE(batch <= 65535, "execute_host: batch > 65535 per call");
    DeviceGuard guard(d->device);
    const size_t n_in = d->host.N * batch, n_out = d->W * batch;
    // check a staging set out of the plan's pool (or allocate one): its workspace and status
    // word are this call's alone
    pft_dplan_s::Staging* sg = nullptr;
    {
        std::lock_guard<std::mutex> lk(d->staging_mu);
        for (size_t i = 0; i < d->staging_free.size(); ++i)
            if (d->staging_free[i]->batch >= batch) {
                sg = d->staging_free[i];
                d->staging_free.erase(d->staging_free.begin() + (std::ptrdiff_t)i);
                break;
            }
    }
    if (!sg) {
        auto fresh = std::make_unique<pft_dplan_s::Staging>();
        fresh->batch = batch;
        cuda_check(cudaStreamCreateWithFlags(&fresh->st, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaMalloc(&fresh->ws, d->workspace_bytes(batch)), "cudaMalloc(workspace)");
        cuda_check(cudaMemsetAsync(fresh->ws, 0, d->workspace_bytes(batch), fresh->st), "cudaMemset(workspace)");
        cuda_check(cudaMalloc(&fresh->din, n_in * sizeof(double2)), "cudaMalloc(input)");
        cuda_check(cudaMalloc(&fresh->dout, n_out * sizeof(double2)), "cudaMalloc(output)");
        cuda_check(cudaStreamSynchronize(fresh->st), "stream synchronize");
        std::lock_guard<std::mutex> lk(d->staging_mu);
        d->staging_all.push_back(fresh.get());
        sg = fresh.release();
    }
    struct Return {
        pft_dplan_s* d;
        pft_dplan_s::Staging* s;
        ~Return() {
            std::lock_guard<std::mutex> lk(d->staging_mu);
            d->staging_free.push_back(s);
        }
    } give_back{d, sg};
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : sg->st;
    double2* din = d_in ? reinterpret_cast<double2*>(d_in) : sg->din;
    double2* dout = d_out ? reinterpret_cast<double2*>(d_out) : sg->dout;
    cuda_check(cudaMemcpyAsync(din, h_in, n_in * sizeof(pft_c128), cudaMemcpyHostToDevice, st), "H2D input");
    run_execute(d, din, batch, d->host.N, dout, sg->ws, st, false);
    cuda_check(cudaMemcpyAsync(h_out, dout, n_out * sizeof(pft_c128), cudaMemcpyDeviceToHost, st), "D2H output");
    if (const int f = read_status(d->ws_view(sg->ws).status, true, st)) {
        if (f & 2) fail(PFT_ERR_INTERNAL, "execute: a device-side wait of the second pass reached its bound");
        fail(PFT_ERR_NON_FINITE, "execute: non-finite input entries (non-finite output detected)");
    }
    PFT_API_END
}

pft_status pft_naive_dft_device(const pft_c128* d_in, uint64_t N, int64_t first_m, uint64_t count, pft_c128* d_out,
                                void* stream) {
    PFT_API_BEGIN
    PFT_REQUIRE(N >= 1 && d_in && (d_out || count == 0), "naive_dft: bad arguments");
    if (count == 0) return PFT_OK;
    if (usable_device_count() == 0) fail(PFT_ERR_NO_DEVICE, "no CUDA device visible (this library has no CPU fallback)");
    cuda_check(pftdev::launch_naive_dft(reinterpret_cast<const double2*>(d_in), N, first_m, count,
                                        reinterpret_cast<double2*>(d_out), static_cast<cudaStream_t>(stream)),
               "naive DFT launch");
    PFT_API_END
}

pft_status pft_naive_dft_host(const pft_c128* h_in, uint64_t N, int64_t first_m, uint64_t count, pft_c128* h_out) {
    PFT_API_BEGIN
    PFT_REQUIRE(N >= 1 && h_in && (h_out || count == 0), "naive_dft_host: bad arguments");
    if (count == 0) return PFT_OK;
    if (usable_device_count() == 0) fail(PFT_ERR_NO_DEVICE, "no CUDA device visible (this library has no CPU fallback)");
    struct Bufs {
        void *in = nullptr, *out = nullptr;
        cudaStream_t st = nullptr;
        ~Bufs() {
            if (st) cudaStreamDestroy(st);
            cudaFree(in);
            cudaFree(out);
        }
    } b;
    cuda_check(cudaStreamCreateWithFlags(&b.st, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaMalloc(&b.in, N * sizeof(pft_c128)), "cudaMalloc(input)");
    cuda_check(cudaMalloc(&b.out, count * sizeof(pft_c128)), "cudaMalloc(output)");
    cuda_check(cudaMemcpyAsync(b.in, h_in, N * sizeof(pft_c128), cudaMemcpyHostToDevice, b.st), "H2D input");
    cuda_check(pftdev::launch_naive_dft(static_cast<const double2*>(b.in), N, first_m, count,
                                        static_cast<double2*>(b.out), b.st),
               "naive DFT launch");
    cuda_check(cudaMemcpyAsync(h_out, b.out, count * sizeof(pft_c128), cudaMemcpyDeviceToHost, b.st), "D2H output");
    cuda_check(cudaStreamSynchronize(b.st), "stream synchronize");
    PFT_API_END
}

pft_status pft_generate_device(const pft_signal_desc* desc, pft_c128* d_out, uint64_t count, void* stream) {
    PFT_API_BEGIN
    PFT_REQUIRE(desc && (d_out || count == 0), "generate_device: bad arguments");
    PFT_REQUIRE(desc->kind >= 0 && desc->kind <= 2, "generate_device: unknown kind");
    PFT_REQUIRE(desc->kind != 2 || desc->N >= 1, "generate_device: sparse kind needs N");
    if (usable_device_count() == 0) fail(PFT_ERR_NO_DEVICE, "no CUDA device visible");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    pftdev::GenParams G{};
    G.kind = desc->kind;
    G.seed = desc->seed;
    G.N = desc->N ? desc->N : 1;
    G.index_offset = desc->index_offset;
    G.count = count;
    G.sigma = desc->sigma;
    G.out = reinterpret_cast<double2*>(d_out);
    void* tones = nullptr;
    if (desc->kind == 2 && desc->n_tones > 0) {
        PFT_REQUIRE(desc->freqs && desc->amps, "generate_device: tones missing");
        const size_t nt = desc->n_tones;
        cuda_check(cudaMalloc(&tones, nt * (sizeof(int64_t) + sizeof(double2))), "cudaMalloc(tones)");
        cuda_check(cudaMemcpy(tones, desc->freqs, nt * sizeof(int64_t), cudaMemcpyHostToDevice), "upload freqs");
        cuda_check(cudaMemcpy(static_cast<char*>(tones) + nt * sizeof(int64_t), desc->amps, nt * sizeof(double2),
                              cudaMemcpyHostToDevice),
                   "upload amps");
        G.n_tones = desc->n_tones;
        G.freqs = static_cast<const int64_t*>(tones);
        G.amps = reinterpret_cast<const double2*>(static_cast<char*>(tones) + nt * sizeof(int64_t));
    }
    cudaError_t e = pftdev::launch_k0(G, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (tones) cudaFree(tones);
    cuda_check(e, "K0 generate");
    PFT_API_END
}

}  // extern "C"
