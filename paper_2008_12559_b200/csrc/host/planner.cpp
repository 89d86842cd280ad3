// planner.cpp -- configuration phase of the PFT (Algorithm 1, PAPER.md:360-375;
// SPEC.md:116-195): divisor enumeration, the SPEC cost model, minimal-r lookup and the
// data-independent tables of the plan (B, phase, tvals, post_powers, post_twiddles).
//
// The plan is the single source of truth shared by the GPU path and the CPU oracle:
// both consume exactly these arrays, so the two agree on (p, q, r, w) bit-for-bit
// (SURVEY.md §0.2 finding 4).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

#include "internal.hpp"

namespace pft::detail {

std::vector<uint64_t> divisors(uint64_t N) {
    if (N == 0) fail(PFT_ERR_INVALID_ARGUMENT, "divisors: N must be >= 1");
    std::vector<uint64_t> lo, hi;
    for (uint64_t d = 1; d <= N / d; ++d) {
        if (N % d == 0) {
            lo.push_back(d);
            if (d != N / d) hi.push_back(N / d);
        }
    }
    lo.insert(lo.end(), hi.rbegin(), hi.rend());
    return lo;
}

int min_terms(const Table& t, double eps, uint64_t M, uint64_t p) {
    if (p == 0) fail(PFT_ERR_INVALID_ARGUMENT, "min_terms: p must be >= 1");
    if (!t.has_eps(eps)) fail(PFT_ERR_EPSILON_NOT_IN_TABLE, "min_terms: table has no entries for epsilon");
    if (M == 0) return 1;  // xi(eps, 1) >= 0 always
    const double ratio = static_cast<double>(M) / static_cast<double>(p);
    const int rmax = t.r_max_for(eps);
    for (int r = 1; r <= rmax; ++r) {
        const TableEntry* e = t.find(eps, r);
        if (e && e->xi >= ratio) return r;
    }
    fail(PFT_ERR_RATIO_OUT_OF_RANGE, "min_terms: ratio out of range (M/p exceeds every tabulated scope)");
}

double spec_cost(uint64_t N, uint64_t M, uint64_t p, int r) {
    // CostEstimate.cost = r (N + p log2(max(p, 2)) + M)
    const double pp = static_cast<double>(std::max<uint64_t>(p, 2));
    return static_cast<double>(r) *
           (static_cast<double>(N) + static_cast<double>(p) * std::log2(pp) + static_cast<double>(M));
}

namespace {
bool is_smooth(uint64_t N, uint64_t b) {
    for (uint64_t f = 2; f <= b && N > 1; ++f)
        while (N % f == 0) N /= f;
    return N == 1;
}
}  // namespace

DivisorChoice select_divisor(const Table& t, uint64_t N, uint64_t M, double eps) {
    if (N <= 1) fail(PFT_ERR_INVALID_ARGUMENT, "select_divisor: N = 1 has no non-trivial split");
    if (M > N) fail(PFT_ERR_INVALID_ARGUMENT, "select_divisor: M > N");
    if (!t.has_eps(eps)) fail(PFT_ERR_EPSILON_NOT_IN_TABLE, "select_divisor: table has no entries for epsilon");
    const auto divs = divisors(N);
    if (M == 0) {  // smallest divisor > 1 (N itself when prime), r = 1
        DivisorChoice c;
        c.p = divs[1];
        c.r = 1;
        c.cost = spec_cost(N, M, c.p, 1);
        return c;
    }
    // Lemma 2: for b-smooth N some divisor lies in [M/sqrt b, sqrt(b) M).
    for (uint64_t b : {2ull, 3ull, 5ull, 7ull}) {
        if (!is_smooth(N, b)) continue;
        const double lo = static_cast<double>(M) / std::sqrt(static_cast<double>(b));
        const double hi = static_cast<double>(M) * std::sqrt(static_cast<double>(b));
        bool found = false;
        for (uint64_t d : divs)
            if (static_cast<double>(d) >= lo && static_cast<double>(d) < hi) found = true;
        if (!found) fail(PFT_ERR_INTERNAL, "select_divisor: Lemma 2 window empty (cannot happen)");
        break;
    }
    DivisorChoice best;
    bool have = false;
    for (uint64_t p : divs) {
        if (p <= 1) continue;
        int r;
        try {
            r = min_terms(t, eps, M, p);
        } catch (const Error& e) {
            if (e.status == PFT_ERR_RATIO_OUT_OF_RANGE) continue;
            throw;
        }
        const double cost = spec_cost(N, M, p, r);
        if (!have || cost < best.cost) {  // ascending p: strict '<' breaks ties toward smaller p
            best = {p, r, cost};
            have = true;
        }
    }
    if (!have) fail(PFT_ERR_RATIO_OUT_OF_RANGE, "select_divisor: no divisor p with M/p inside the table's scope");
    return best;
}

namespace {
uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
template <class T>
uint64_t fnv(uint64_t h, const T& v) { return fnv1a(h, &v, sizeof(T)); }
}  // namespace

HostPlan build_plan(const Table& t, uint64_t N, uint64_t M, int64_t mu, uint64_t p_in, double eps) {
    if (N == 0) fail(PFT_ERR_INVALID_ARGUMENT, "build_plan: N must be >= 1");
    if (M > N / 2) fail(PFT_ERR_M_TOO_LARGE, "build_plan: M > N/2");
    if (!t.has_eps(eps)) fail(PFT_ERR_EPSILON_NOT_IN_TABLE, "build_plan: table missing epsilon");
    if (N > (1ull << 40)) fail(PFT_ERR_UNSUPPORTED, "build_plan: N > 2^40");
    HostPlan P;
    P.N = N;
    P.M = M;
    P.mu = mu;
    P.epsilon = eps;
    if (p_in == 0) {
        P.p = select_divisor(t, N, M, eps).p;
    } else {
        if (N % p_in != 0) fail(PFT_ERR_P_NOT_DIVISOR, "build_plan: p does not divide N");
        P.p = p_in;
    }
    P.q = N / P.p;
    P.r = min_terms(t, eps, M, P.p);
    const TableEntry* e = t.find(eps, P.r);
    if (!e) fail(PFT_ERR_INTERNAL, "build_plan: table entry vanished");
    P.w = e->coeffs;
    P.xi = e->xi;
    P.achieved_epsilon = e->achieved;
    P.cost = spec_cost(N, M, P.p, P.r);

    const uint64_t q = P.q;
    const int r = P.r;
    // mu enters the B phase as e^{-i pi mu (2l - q) / N}; reduce mu mod 2N exactly
    // (SURVEY.md Hard part 4: for odd q the phase is 2N-periodic, not N-periodic).
    const __int128 twoN = static_cast<__int128>(2) * N;
    __int128 mu_red = static_cast<__int128>(mu) % twoN;
    if (mu_red < 0) mu_red += twoN;
    P.phase.resize(q);
    P.tvals.resize(q);
    P.B = ComplexMatrix(q, r);
    for (uint64_t l = 0; l < q; ++l) {
        const __int128 num = -mu_red * (static_cast<__int128>(2) * l - static_cast<__int128>(q));
        P.phase[l] = cispi_frac(num, N);
        // (1 - 2l/q) with q/2 as an exact real
        P.tvals[l] = 1.0 - (2.0 * static_cast<double>(l)) / static_cast<double>(q);
        double tp = 1.0;
        for (int j = 0; j < r; ++j) {
            P.B.at(l, j) = (P.phase[l] * P.w[j]) * tp;  // Algorithm 1 line 4 / SPEC.md:126
            tp *= P.tvals[l];
        }
    }
    const uint64_t W = 2 * M + 1;
    P.post_powers.resize(W * r);
    P.post_twiddles.resize(W);
    for (uint64_t s = 0; s < W; ++s) {
        const int64_t m = mu - static_cast<int64_t>(M) + static_cast<int64_t>(s);
        const double x = static_cast<double>(static_cast<int64_t>(s) - static_cast<int64_t>(M)) /
                         static_cast<double>(P.p);  // (m - mu)/p
        double pw = 1.0;
        for (int j = 0; j < r; ++j) {
            P.post_powers[s * r + j] = pw;  // precomputed powers, ascending j
            pw *= x;
        }
        P.post_twiddles[s] = cispi_frac(-static_cast<__int128>(m), P.p);  // e^{-pi i m / p}
    }
    // Deterministic plan id: hash of the defining parameters and w bits.
    uint64_t h = 0xcbf29ce484222325ull;
    h = fnv(h, P.N);
    h = fnv(h, P.M);
    h = fnv(h, P.mu);
    h = fnv(h, P.p);
    h = fnv(h, P.r);
    h = fnv(h, P.epsilon);
    h = fnv(h, t.version);
    for (const auto& c : P.w) h = fnv(h, c);
    P.plan_id = h;
    return P;
}

ShardLayout shard_layout(uint64_t q, int world, int rank) {
    if (q == 0) fail(PFT_ERR_INVALID_ARGUMENT, "shard_layout: q must be >= 1");
    if (world < 1 || rank < 0 || rank >= world) fail(PFT_ERR_INVALID_ARGUMENT, "shard_layout: bad world/rank");
    const uint64_t L = (q + 1) / 2;  // pairs (l, q-l) for l in [1, L)
    const uint64_t npairs = L - 1;
    ShardLayout v;
    if (world == 1) {
        v.pair_begin = 1;
        v.pair_end = L;
        v.row_len = q;
        v.front_col = 1;
        v.mirror_col = static_cast<int64_t>(q) - 1;
        v.single0_col = 0;
        v.singleh_col = (q % 2 == 0) ? static_cast<int64_t>(q / 2) : -1;
        return v;
    }
    const uint64_t base = npairs / world, extra = npairs % world, r = static_cast<uint64_t>(rank);
    v.pair_begin = 1 + r * base + std::min<uint64_t>(r, extra);
    v.pair_end = v.pair_begin + base + (r < extra ? 1 : 0);
    const uint64_t n = v.pair_end - v.pair_begin;
    // local row: [front: l ascending | mirror: q-l ascending in global order | singles (rank 0)]
    v.front_col = 0;
    v.mirror_col = static_cast<int64_t>(2 * n) - 1;  // mirror of pair_begin is the last mirror column
    v.row_len = 2 * n;
    if (rank == 0) {
        v.single0_col = static_cast<int64_t>(v.row_len++);
        if (q % 2 == 0) v.singleh_col = static_cast<int64_t>(v.row_len++);
    }
    return v;
}

uint64_t ShardLayout::global_col(uint64_t q, uint64_t c) const {
    const int64_t ci = static_cast<int64_t>(c);
    if (ci == single0_col) return 0;
    if (ci == singleh_col) return q / 2;
    const uint64_t n = pair_end - pair_begin;
    if (front_col == 1 && row_len == q) return c;  // natural layout
    if (c < n) return pair_begin + c;              // front
    if (c < 2 * n) return q - (pair_begin + static_cast<uint64_t>(mirror_col - ci));  // mirror
    fail(PFT_ERR_INVALID_ARGUMENT, "shard layout: local column out of range");
}

std::string plan_json(const HostPlan& P) {
    char buf[512];
    std::snprintf(buf, sizeof buf,
                  "{\"N\": %llu, \"M\": %llu, \"mu\": %lld, \"p\": %llu, \"q\": %llu, \"r\": %d, "
                  "\"epsilon\": %.17g, \"achieved_epsilon\": %.17g, \"xi\": %.17g, "
                  "\"estimated_cost\": %.17g, \"plan_id\": \"%016llx\"}",
                  (unsigned long long)P.N, (unsigned long long)P.M, (long long)P.mu,
                  (unsigned long long)P.p, (unsigned long long)P.q, P.r, P.epsilon,
                  P.achieved_epsilon, P.xi, P.cost, (unsigned long long)P.plan_id);
    return buf;
}

}  // namespace pft::detail
