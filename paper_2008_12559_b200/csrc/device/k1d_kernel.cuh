// k1d_kernel.cuh -- K1 with dynamic work distribution (included by kernel_templates.cuh).
//
// The static K1 gives each CTA one residue class: a CTA that starts late (its SM slot still
// held by the previous transform's tail, or by a K2) finishes late, and one transform alone
// cannot fill both CTA slots of every SM.  Here the grid is persistent (co-resident CTAs) and
// the unit of streaming is a work ITEM: 32 rows of one residue class c (rows c + P2 k1,
// k1 in [32 rb, 32 rb + 32)) times one segment g of the column pairs -- 64-256 KB of input.
//   * the producer warp claims items from a counter in the workspace header (atomicAdd) and
//     streams their TMA stages into the ring, tagging each stage with its item id; after the
//     first failed claim it triggers the dependent launch (PDL) -- every claim of this grid is
//     made by then, and the claim that is the grid's last re-arms the counter for the next launch;
//   * the consumer warps contract each item exactly as K1 does (vector FP64 or DMMA paths) and
//     store its 32 x r partial moments to Cpart[b][c][g] (L2);
//   * the CTA that completes a class's last item (class counter) sums the class's partials in
//     a fixed segment order, runs the length-P1 FFT pass in shared memory and its tail: the sum
//     tail's residue row (few bins; summed by the signal's last finisher when P2 <= 8, else by
//     k_sum_rows) or the K2 slab (many bins; K2 follows).  The producer keeps streaming the
//     next item meanwhile: finisher work overlaps the stream instead of idling it.
// Items are numbered class-fastest (c, then segment g, then row block rb): the CTAs streaming at
// any moment cover contiguous rows c + P2 k1 of A, spread over all HBM channels.  (Class-major
// numbering -- rows P2 apart, 1 MB strides at C2b -- measured 25% of DRAM peak: channel
// camping.)  So classes complete at the end of the stream, their finishers in parallel.
// Results are deterministic (fixed summation orders), not bitwise equal to the static K1 (the
// segment partials are summed separately).
#pragma once

namespace pftdev {

// Acquire-release atomic add (gpu scope): the CTA's prior writes, ordered before it by a named
// barrier, become visible to whoever observes the new count, and the last arriver acquires every
// earlier arriver's -- without the sequentially consistent fence (MEMBAR.SC) of
// __threadfence() + atomicAdd.
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void k1d_decode(const K1Params& P, uint32_t v, uint32_t& b, uint32_t& c, uint32_t& rb,
                                           uint32_t& g) {
    b = v / P.items_per_signal;
    uint32_t rem = v - b * P.items_per_signal;
    if (P.dev_flags & 16) {  // dev: segment fastest
        g = rem % P.nseg;
        rem /= P.nseg;
        c = rem % P.P2;
        rb = rem / P.P2;
    } else if (P.dev_flags & 32) {  // dev: row block fastest
        rb = rem % P.nrb;
        rem /= P.nrb;
        c = rem % P.P2;
        g = rem / P.P2;
    } else {
    c = rem % P.P2;  // class fastest: concurrent items cover contiguous rows (DRAM channel spread)
    rem /= P.P2;
    g = rem % P.nseg;
    rb = rem / P.nseg;
    }
}

// The class finisher (consumer warps only; the producer keeps streaming): C_c = w_j * (sum over
// segments of the partial moments), the length-P1 FFT over k1 in column groups, then the tail.
template <int R>
__device__ __noinline__ void k1d_finish_class(const K1Params& P, uint32_t b, uint32_t c, double2* Cs, double2* scr,
                                              const double2* tw1, const double2* wsm, int ctid, unsigned* sflag) {
    constexpr int NT = K1_CONSUMER_WARPS * 32;
    const WarpsTeam<NT> team{ctid};
    const K2Params& Q = P.k2;
    fence_acquire_gpu();  // the other items' partials were released with their class tickets
    const uint32_t n = (uint32_t)R * P.P1;
    const double2* __restrict__ Cp = P.Cpart + (size_t)b * P.y_stride + (size_t)c * P.nseg * n;
    // Cs = sum over segments (ascending g) with 8 L2 loads in flight per thread: the finisher's
    // read of its class's partials is latency-bound otherwise
    constexpr int U = 4;
    for (uint32_t i0 = ctid; i0 < n; i0 += U * NT) {
        double2 acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = make_double2(0.0, 0.0);
        for (uint32_t g0 = 0; g0 < P.nseg; g0 += 2) {
            double2 v[U][2];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t idx = i0 + u * NT;
                    v[u][e] = (idx < n && g0 + e < P.nseg) ? __ldcg(Cp + (size_t)(g0 + e) * n + idx)
                                                            : make_double2(0.0, 0.0);
                }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc[u] = g0 == 0 ? v[u][0] : cadd(acc[u], v[u][0]);
                if (g0 + 1 < P.nseg) acc[u] = cadd(acc[u], v[u][1]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * NT < n) Cs[i0 + u * NT] = acc[u];
    }
    team.sync();
    // the vector path stored w_j acc_j; the tensor-core path raw moments: w_j in the FFT's loads
    const double2* colw = k1_tc(R) ? wsm : nullptr;
    if (P.P1 > 1) {
        for (uint32_t j0 = 0; j0 < (uint32_t)R; j0 += P.fft_group) {
            const int ng = (int)min(P.fft_group, (uint32_t)R - j0);
            double2* x = Cs + (size_t)j0 * P.P1;
            const double2* res = fft_columns(x, scr, ng, P.fft, SmemTwiddles{tw1}, team, colw ? colw + j0 : nullptr);
            if (res != x) {
                for (uint32_t i = ctid; i < (uint32_t)ng * P.P1; i += NT) x[i] = res[i];
                team.sync();
            }
        }
    } else if (colw) {
        for (uint32_t j = ctid; j < (uint32_t)R; j += NT) Cs[j] = cmul(Cs[j], colw[j]);
        team.sync();
    }
    const double2* res = Cs;  // Y_c[m1][j] at res[j * P1 + m1]
    unsigned* ctl = P.cls + (size_t)b * P.ctl_stride;
    if (!P.sum_tail) {
        // K2 slab Y[b][m1][c][j] (K2 reads one m1's (c, j) block contiguously)
        double2* __restrict__ Y = P.rows + (size_t)b * P.y_stride;
        for (uint32_t idx = ctid; idx < n; idx += NT) {
            const uint32_t m1 = idx / R, j = idx - m1 * R;
            Y[((size_t)m1 * P.P2 + c) * R + j] = res[(size_t)j * P.P1 + m1];
        }
    } else {
        // residue row S_c[s] = omega_p^{(m mod p) c} sum_j Y_c[m1][j] x_s^j from smem tables
        double2* twc = scr;          // [P1] omega_p^{m1 c}
        double2* tw2 = scr + P.P1;   // [P2] omega_P2^t
        for (uint32_t t = ctid; t < P.P1 + P.P2; t += NT)
            twc[t] = __ldg(P.omega + (t < P.P1 ? (size_t)t * c : (size_t)(t - P.P1) * P.P1));  // m1 c < p
        team.sync();
        const int64_t Mh = (int64_t)((Q.W - 1) / 2);
        const bool p1_pow2 = (P.P1 & (P.P1 - 1)) == 0, p2_pow2 = (P.P2 & (P.P2 - 1)) == 0;
        const int lg_p1 = 31 - __clz(P.P1);
        double2* __restrict__ out = Q.out + (size_t)b * Q.W;
        if (P.P2 == 1) {  // one class per signal: the row is the output
            for (uint64_t so = ctid; so < Q.W; so += NT) {
                const double2 o =
                    cmul(k1_row_value<R>(P, res, twc, tw2, c, so, Mh, p1_pow2, p2_pow2, lg_p1), __ldg(Q.post_twiddles + so));
                out[so] = o;
                if (!isfinite(o.x) || !isfinite(o.y)) atomicOr(Q.status, 1);
            }
        } else {
            double2* __restrict__ rows = P.rows + (size_t)b * P.y_stride;
            constexpr int FAST_OUT = 4;
            double2 keep[FAST_OUT];
            for (uint64_t so = ctid, i = 0; so < Q.W; so += NT, ++i) {
                const double2 v = k1_row_value<R>(P, res, twc, tw2, c, so, Mh, p1_pow2, p2_pow2, lg_p1);
                rows[(size_t)c * Q.W + so] = v;
                if (i < FAST_OUT) keep[i] = v;
            }
            if (P.fast_reduce) {  // P2 <= 8, W <= 4 NT: the signal's last finisher sums the rows
                team.sync();  // every row store precedes thread 0's fence and ticket
                if (ctid == 0) {
                    __threadfence();
                    sflag[2] = atomicAdd(ctl + P.P2, 1u) == P.P2 - 1;
                }
                team.sync();
                if (sflag[2]) {
                    __threadfence();
#pragma unroll
                    for (int i = 0; i < FAST_OUT; ++i) {
                        const uint64_t so = (uint64_t)ctid + (uint64_t)i * NT;
                        if (so < Q.W) {
                            double2 v[8];
#pragma unroll
                            for (int r = 0; r < 8; ++r)
                                v[r] = (uint32_t)r >= P.P2 ? make_double2(0.0, 0.0)
                                       : (uint32_t)r == c  ? keep[i]
                                                           : __ldcg(rows + (size_t)r * Q.W + so);
                            double2 tot = v[0];
#pragma unroll
                            for (int r = 1; r < 8; ++r)
                                if ((uint32_t)r < P.P2) tot = cadd(tot, v[r]);  // fixed order c = 0, 1, ...
                            const double2 o = cmul(tot, __ldg(Q.post_twiddles + so));  // e^{-pi i m / p}
                            out[so] = o;
                            if (!isfinite(o.x) || !isfinite(o.y)) atomicOr(Q.status, 1);
                        }
                    }
                    if (ctid == 0) ctl[P.P2] = 0;  // every class of the signal has finished: re-arm
                }
            }
        }
    }
    if (ctid == 0) ctl[c] = 0;  // every item of the class has been counted: re-arm
    team.sync();                // smem (Cs, scr) reuse by the next finisher
}

// One work item on the consumer warps: the stages of its column segment (the first one already
// waited for by the caller), the row reduction and its partial moments into Cpart.  Out of line
// so the stage loop keeps the ring slot and phase in registers (with the class finisher inlined
// in the same loop they lived in local memory: a local load per stage on the barrier's path).
// sph = ring slot | phase << 31, returned advanced past the item.
template <int R, bool MU0>
__device__ __noinline__ uint32_t k1d_consume_item(const K1Params& P, const unsigned char* ring, uint64_t* full,
                                                 uint64_t* empty, uint32_t sph, uint32_t v, bool first) {
    constexpr uint32_t STAGE = k1_stage_bytes(R);
    const uint32_t S = P.stages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t npairs = P.gp_end > P.gp0 ? P.gp_end - P.gp0 : 0;
    uint32_t s = sph & 0x7fffffffu, ph = sph >> 31;
        uint32_t b, c, rb, g;
    k1d_decode(P, v, b, c, rb, g);
    const uint32_t ch0 = g * P.nch / P.nseg, ch1 = (g + 1) * P.nch / P.nseg;
    double2* Cg = P.Cpart + (size_t)b * P.y_stride + ((size_t)c * P.nseg + g) * (size_t)R * P.P1;
    if constexpr (k1_tc(R)) {
        const int gq = lane >> 2, t4 = lane & 3, part = gq & 1, rr = gq >> 1;
        const int rin = 8 * (warp >> 1) + 2 * (warp & 1) + 4 * (rr & 1) + (rr >> 1);
        const int fsw = 2 * (int)((P.gp0 + (uint32_t)t4) & 3u);
        double de[2] = {0.0, 0.0}, dd[2] = {0.0, 0.0}, v0 = 0.0, vl = 0.0;
        const uint32_t k1 = rb * K1_BR + rin;
        double2 x0 = make_double2(0.0, 0.0), xh = make_double2(0.0, 0.0);
        if (g == 0 && k1 < P.P1) {
            const double2* row = P.a + (size_t)b * P.batch_stride + ((size_t)c + (size_t)P.P2 * k1) * P.row_stride;
            if (P.single0_col >= 0) x0 = __ldg(row + P.single0_col);
            if (t4 == 1 && P.singleh_col >= 0) xh = __ldg(row + P.singleh_col);
        }
        for (uint32_t ch = ch0; ch < ch1; ++ch) {
            if (ch != ch0) {
                mbar_wait(&full[s], ph);
                __syncwarp();
            }
            const uint32_t valid = min((uint32_t)K1_CP, npairs - ch * K1_CP);
            const unsigned char* stage = ring + (size_t)s * STAGE;
            const PairEntry* ptab = P.pairtab + P.gp0 + ch * K1_CP;
            if (valid == (uint32_t)K1_CP)
                k1_tc_stage<R, MU0, true>(stage, ptab, rin, part, t4, gq ^ fsw, fsw, valid, de, dd, v0, vl);
            else
                k1_tc_stage<R, MU0, false>(stage, ptab, rin, part, t4, gq ^ fsw, fsw, valid, de, dd, v0, vl);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                ph ^= 1u;
            }
        }
        if (first)  // the previous launch completed before this grid writes the workspace
            asm volatile("griddepcontrol.wait;" ::: "memory");
        if (!(P.dev_flags & 4)) k1_tc_finish_row<R, MU0>(P, x0, xh, part, t4, k1, de, dd, v0, vl, Cg);
    } else {
        constexpr int JS = k1_js(R, MU0), H = (R + JS - 1) / JS;
        const int li = lane & (K1_LANES_PER_ROW - 1);
        const int rin = (warp * 32 + lane) / K1_LANES_PER_ROW;
        double are[H], aim[H];
#pragma unroll
        for (int j = 0; j < H; ++j) are[j] = aim[j] = 0.0;
        const uint32_t k1 = rb * K1_BR + rin;
        const int scol = g != 0 ? -1 : li < JS ? P.single0_col : (li == JS ? P.singleh_col : -1);
        double2 xs = make_double2(0.0, 0.0);
        if (k1 < P.P1 && scol >= 0)
            xs = __ldg(P.a + (size_t)b * P.batch_stride + ((size_t)c + (size_t)P.P2 * k1) * P.row_stride + scol);
        for (uint32_t ch = ch0; ch < ch1; ++ch) {
            if (ch != ch0) {
                mbar_wait(&full[s], ph);
                __syncwarp();
            }
            const uint32_t valid = min((uint32_t)K1_CP, npairs - ch * K1_CP);
            const unsigned char* stage = ring + (size_t)s * STAGE;
            if (valid == (uint32_t)K1_CP)
                k1_accumulate_stage<R, JS, MU0, true>(stage, rin, li, valid, are, aim);
            else
                k1_accumulate_stage<R, JS, MU0, false>(stage, rin, li, valid, are, aim);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                ph ^= 1u;
            }
        }
        if (first) asm volatile("griddepcontrol.wait;" ::: "memory");
        if (!(P.dev_flags & 4)) k1_finish_row<R, JS, MU0>(P, xs, scol, li, k1, are, aim, Cg);
    }
    return s | (ph << 31);
}

template <int R, bool MU0>
__global__ void __launch_bounds__(K1D_THREADS, 2) k1d_contract(const __grid_constant__ CUtensorMap tmap,
                                                                const __grid_constant__ K1Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t S = P.stages;
    constexpr uint32_t STAGE = k1_stage_bytes(R);
    unsigned char* ring = smem_raw;
    if constexpr (k1_ring_align_slack(R) > 0)  // swizzled TMA destinations: 1024-byte aligned ring
        ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    double2* Cs = reinterpret_cast<double2*>(smem_raw + k1_ring_align_slack(R) + (size_t)S * STAGE);  // [R][P1]
    double2* scr = Cs + (size_t)R * P.P1;                      // [fft_group][P1]
    double2* tw1 = scr + (size_t)P.fft_group * P.P1;           // omega_P1^t
    double2* wsm = tw1 + P.P1;                                 // w_j
    uint64_t* full = reinterpret_cast<uint64_t*>(wsm + R);
    uint64_t* empty = full + S;
    // item hand-off ring consumers -> ticket lane (mbarrier pairs, 8-byte aligned: right after the
    // ring barriers), finisher-job queue ticket lane -> consumers (polled at item boundaries)
    uint64_t* hfull = empty + S;                                                       // [K1D_HR]
    uint64_t* hempty = hfull + K1D_HR;                                                 // [K1D_HR]
    volatile uint32_t* qitem = reinterpret_cast<volatile uint32_t*>(hempty + K1D_HR);  // item id per stage
    unsigned* sflag = reinterpret_cast<unsigned*>(const_cast<uint32_t*>(qitem) + S);  // [4]: fast-reduce flag
    volatile uint32_t* hand = reinterpret_cast<volatile uint32_t*>(sflag + 4);         // [K1D_HR]
    volatile uint32_t* jq = hand + K1D_HR;                                             // [K1D_JQ]
    volatile uint32_t* jctl = jq + K1D_JQ;  // {tail (jobs posted), done, head (jobs taken), seen}

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], K1_CONSUMER_WARPS);
        }
        for (int s = 0; s < K1D_HR; ++s) {
            mbar_init(&hfull[s], 1);
            mbar_init(&hempty[s], 1);
        }
        jctl[0] = jctl[1] = jctl[2] = jctl[3] = 0;
        fence_barrier_init();
    }
    __syncthreads();
    const uint32_t npairs = P.gp_end > P.gp0 ? P.gp_end - P.gp0 : 0;
    constexpr uint32_t kDone = 0xffffffffu;

    if (warp == K1_CONSUMER_WARPS) {
        // ---- producer: claim items, stream their stages
        if (lane == 0) {
            prefetch_tensormap(&tmap);
            const uint32_t nclaims = P.total_items + gridDim.x;  // every CTA's last claim fails
            uint32_t s = 0, ph = 0, issued = 0;
            uint32_t next = atomicAdd(P.item_ctr, 1u);
            while (true) {
                const uint32_t v = next;
                if (v >= P.total_items) {
                    if (v == nclaims - 1) {  // the grid's last claim: re-arm for the next launch
                        atomicExch(P.item_ctr, 0u);
                        __threadfence();
                    }
                    if (issued >= S) mbar_wait(&empty[s], ph ^ 1u);
                    qitem[s] = kDone;
                    mbar_arrive(&full[s]);  // no bytes: completes the phase at once
                    // every claim of this CTA is made: the next launch (PDL) may start claiming
                    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
                    break;
                }
                next = atomicAdd(P.item_ctr, 1u);  // the following claim, in flight while v streams
                uint32_t b, c, rb, g;
                k1d_decode(P, v, b, c, rb, g);
                const uint32_t ch0 = g * P.nch / P.nseg, ch1 = (g + 1) * P.nch / P.nseg;
                const int row0 = (int)(rb * K1_BR);
                for (uint32_t ch = ch0; ch < ch1; ++ch) {
                    if (issued >= S) mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char* st = ring + (size_t)s * STAGE;
                    qitem[s] = v;
                    mbar_arrive_expect_tx(&full[s], k1_stage_data_bytes(R));
                    const int f0 = P.fcol0 + (int)(ch * K1_CP);
                    const int m0 = P.mcol0 - (int)(ch * K1_CP) - (K1_CP - 1);  // may be < 0: zero fill
                    if constexpr (k1_tc(R)) {  // 8-pair swizzled halves
                        constexpr int HB = K1_BR * 128;
                        tma_load_4d(st, &tmap, 2 * f0, (int)c, row0, (int)b, &full[s]);
                        tma_load_4d(st + HB, &tmap, 2 * (f0 + 8), (int)c, row0, (int)b, &full[s]);
                        tma_load_4d(st + K1_BOX_BYTES, &tmap, 2 * m0, (int)c, row0, (int)b, &full[s]);
                        tma_load_4d(st + K1_BOX_BYTES + HB, &tmap, 2 * (m0 + 8), (int)c, row0, (int)b, &full[s]);
                        bulk_load(st + 2 * K1_BOX_BYTES, P.tcfrag + (size_t)(P.gp0 + ch * K1_CP) * 8, K1_TC_BYTES,
                                  &full[s]);
                    } else {
                        tma_load_4d(st, &tmap, 2 * f0, (int)c, row0, (int)b, &full[s]);
                        tma_load_4d(st + K1_BOX_BYTES, &tmap, 2 * m0, (int)c, row0, (int)b, &full[s]);
                        bulk_load(st + 2 * K1_BOX_BYTES, P.pairtab + P.gp0 + ch * K1_CP, K1_TAB_BYTES, &full[s]);
                    }
                    ++issued;
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }
    constexpr int NC = K1_CONSUMER_WARPS * 32;
    if (warp == K1_CONSUMER_WARPS + 1) {
        // ---- ticket lane: per finished item, the class ticket (an acq_rel atomic: the consumers'
        // partial stores, ordered before the hand-off's mbarrier arrive, are released with it), and
        // a finisher job when the item completed its class.  The consumers never wait for it.
        if (lane == 0) {
            for (uint32_t k = 0;; ++k) {
                const uint32_t slot = k % K1D_HR, par = (k / K1D_HR) & 1u;
                mbar_wait(&hfull[slot], par);
                const uint32_t h = hand[slot];
                mbar_arrive(&hempty[slot]);
                if (h == kDone) break;
                const uint32_t b = h / P.P2, c = h - b * P.P2;
                if (atom_add_acq_rel_gpu(P.cls + (size_t)b * P.ctl_stride + c, 1u) == P.nrb * P.nseg - 1) {
                    while (jctl[0] - jctl[2] >= (uint32_t)K1D_JQ) __nanosleep(64);  // queue full (rare)
                    jq[jctl[0] % K1D_JQ] = h;
                    __threadfence_block();
                    jctl[0] = jctl[0] + 1;
                }
            }
            __threadfence_block();
            jctl[1] = 1;  // every job is posted
        }
        return;
    }

    // ---- consumers (256 threads)
    for (uint32_t t = tid; t < P.P1; t += K1_CONSUMER_WARPS * 32) tw1[t] = __ldg(P.omega + (size_t)t * P.P2);
    if constexpr (k1_tc(R))
        for (uint32_t t = tid; t < (uint32_t)R; t += K1_CONSUMER_WARPS * 32) wsm[t] = __ldg(P.w + t);
    asm volatile("bar.sync 1, %0;" ::"n"(K1_CONSUMER_WARPS * 32) : "memory");
    uint32_t s = 0, ph = 0;
    uint32_t nitem = 0, head = 0;  // items done, finisher jobs taken
    while (true) {
        mbar_wait(&full[s], ph);
        // reconverge before touching the stage (see k1_contract_fft)
        __syncwarp();
        const uint32_t v = qitem[s];
        if (v == kDone) break;
        const uint32_t sph = k1d_consume_item<R, MU0>(P, ring, full, empty, s | (ph << 31), v, nitem == 0);
        s = sph & 0x7fffffffu;
        ph = sph >> 31;
        uint32_t b, c, rb, g;
        k1d_decode(P, v, b, c, rb, g);
        // Item done.  Snapshot the job queue, then (after the barrier that orders every consumer's
        // partial stores) hand the item to the ticket lane; finish any classes completed so far.
        if (P.dev_flags & 2) { ++nitem; continue; }
        if (tid == 0) {
            jctl[3] = jctl[0];
            __threadfence_block();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
        const uint32_t seen = jctl[3];
        if (tid == 0) {
            const uint32_t slot = nitem % K1D_HR;
            if (nitem >= (uint32_t)K1D_HR) mbar_wait(&hempty[slot], ((nitem / K1D_HR) - 1) & 1u);
            hand[slot] = b * P.P2 + c;
            mbar_arrive(&hfull[slot]);
        }
        for (; head < seen; ++head) {
            const uint32_t h = jq[head % K1D_JQ];
            if (!(P.dev_flags & 1)) k1d_finish_class<R>(P, h / P.P2, h - (h / P.P2) * P.P2, Cs, scr, tw1, wsm, tid, sflag);
            if (tid == 0) jctl[2] = head + 1;
        }
        ++nitem;
    }
    // drain: hand over the end marker, then finish the classes still to come
    if (tid == 0) {
        const uint32_t slot = nitem % K1D_HR;
        if (!(P.dev_flags & 2)) {
            if (nitem >= (uint32_t)K1D_HR) mbar_wait(&hempty[slot], ((nitem / K1D_HR) - 1) & 1u);
            hand[slot] = kDone;
            mbar_arrive(&hfull[slot]);
        } else {
            hand[0] = kDone;
            mbar_arrive(&hfull[0]);
        }
    }
    while (true) {
        if (tid == 0) {
            const uint32_t done = jctl[1];
            __threadfence_block();  // the final tail is visible once `done` is
            jctl[3] = jctl[0] | (done ? 0x80000000u : 0u);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
        const uint32_t snap = jctl[3], seen = snap & 0x7fffffffu;
        asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");  // snapshot read before it is rewritten
        for (; head < seen; ++head) {
            const uint32_t h = jq[head % K1D_JQ];
            if (!(P.dev_flags & 1)) k1d_finish_class<R>(P, h / P.P2, h - (h / P.P2) * P.P2, Cs, scr, tw1, wsm, tid, sflag);
            if (tid == 0) jctl[2] = head + 1;
        }
        if (snap & 0x80000000u) break;
        __nanosleep(256);
    }
    if (nitem == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace pftdev
