// capi_host.cpp -- extern "C" entry points for the host-side modules (minimax, table,
// planner, synthetic inputs).  Exceptions never cross the boundary: each entry point
// maps pft::detail::Error to its pft_status and records the message for pft_last_error.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <numbers>
#include <unordered_set>

#include "../common/rng.h"
#include "api_guard.hpp"
#include "internal.hpp"

namespace pft::detail {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }
}  // namespace pft::detail

using namespace pft;
using namespace pft::detail;

static_assert(sizeof(pft_c128) == sizeof(cplx), "pft_c128 must match std::complex<double>");

namespace {
void to_c(const std::vector<cplx>& v, pft_c128* out) {
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(cplx));
}
std::vector<cplx> from_c(const pft_c128* in, size_t n) {
    std::vector<cplx> v(n);
    if (n) std::memcpy(static_cast<void*>(v.data()), in, n * sizeof(cplx));
    return v;
}
const Table& tab(pft_table_t t) {
    PFT_REQUIRE(t != nullptr, "null table handle");
    return t->table;
}
const HostPlan& plan_of(pft_hplan_t p) {
    PFT_REQUIRE(p != nullptr, "null plan handle");
    return p->plan;
}
}  // namespace

extern "C" {

const char* pft_status_string(pft_status s) {
    switch (s) {
        case PFT_OK: return "ok";
        case PFT_ERR_INVALID_ARGUMENT: return "invalid argument";
        case PFT_ERR_P_NOT_DIVISOR: return "p does not divide N";
        case PFT_ERR_M_TOO_LARGE: return "M > N/2";
        case PFT_ERR_EPSILON_NOT_IN_TABLE: return "table missing epsilon";
        case PFT_ERR_RATIO_OUT_OF_RANGE: return "ratio out of range";
        case PFT_ERR_LENGTH_MISMATCH: return "length mismatch";
        case PFT_ERR_NON_FINITE: return "non-finite input entries";
        case PFT_ERR_IO: return "I/O error or corrupted file";
        case PFT_ERR_VERSION_MISMATCH: return "table version mismatch";
        case PFT_ERR_NO_DEVICE: return "no usable CUDA device";
        case PFT_ERR_CUDA: return "CUDA error";
        case PFT_ERR_UNSUPPORTED: return "unsupported shape";
        case PFT_ERR_INTERNAL: return "internal error";
        case PFT_ERR_BUFFER_TOO_SMALL: return "buffer too small";
    }
    return "unknown status";
}

const char* pft_last_error(void) { return last_error_cstr(); }

// ------------------------------------------------------------------ minimax

pft_status pft_best_approx(int r, double xi, double u, pft_c128* coeffs, double* achieved) {
    PFT_API_BEGIN
    PFT_REQUIRE(coeffs != nullptr, "coeffs is null");
    Poly P = best_approx(r, xi, u);
    to_c(P.coeffs, coeffs);
    if (achieved) *achieved = P.achieved_error;
    PFT_API_END
}

pft_status pft_scope_xi(double eps, int r, double* xi, pft_c128* coeffs, double* achieved) {
    PFT_API_BEGIN
    Poly P = scope_xi(eps, r);
    if (xi) *xi = P.scope;
    if (coeffs) to_c(P.coeffs, coeffs);
    if (achieved) *achieved = P.achieved_error;
    PFT_API_END
}

pft_status pft_translate_poly(const pft_c128* coeffs, int r, double u, double mu, pft_c128* out) {
    PFT_API_BEGIN
    PFT_REQUIRE(coeffs && out && r >= 1 && r <= PFT_MAX_TERMS, "translate_poly: bad arguments");
    PFT_REQUIRE(std::isfinite(u) && std::isfinite(mu), "translate_poly: non-finite u/mu");
    to_c(translate_poly(from_c(coeffs, r), u, mu), out);
    PFT_API_END
}

// ------------------------------------------------------------------ table

pft_status pft_table_default(pft_table_t* out) {
    PFT_API_BEGIN
    PFT_REQUIRE(out != nullptr, "out is null");
    static pft_table_s handle{default_table(), true};
    *out = &handle;
    PFT_API_END
}

pft_status pft_table_generate(const double* eps, int n_eps, int r_max, pft_table_t* out) {
    PFT_API_BEGIN
    PFT_REQUIRE(out && n_eps >= 0 && (eps || n_eps == 0), "table_generate: bad arguments");
    std::vector<double> grid = n_eps ? std::vector<double>(eps, eps + n_eps) : default_eps_grid();
    for (double e : grid) PFT_REQUIRE(e > 0 && std::isfinite(e), "table_generate: eps must be > 0");
    *out = new pft_table_s{generate_table(grid, r_max), false};
    PFT_API_END
}

pft_status pft_table_save(pft_table_t t, const char* path) {
    PFT_API_BEGIN
    PFT_REQUIRE(path != nullptr, "path is null");
    save_table(tab(t), path);
    PFT_API_END
}

pft_status pft_table_load(const char* path, pft_table_t* out) {
    PFT_API_BEGIN
    PFT_REQUIRE(path && out, "table_load: bad arguments");
    *out = new pft_table_s{load_table(path), false};
    PFT_API_END
}

pft_status pft_table_save_csv(pft_table_t t, const char* path) {
    PFT_API_BEGIN
    PFT_REQUIRE(path != nullptr, "path is null");
    save_table_csv(tab(t), path);
    PFT_API_END
}

void pft_table_destroy(pft_table_t t) {
    if (t && !t->owned_by_library) delete t;
}

pft_status pft_table_size(pft_table_t t, size_t* n) {
    PFT_API_BEGIN
    PFT_REQUIRE(n != nullptr, "n is null");
    *n = tab(t).entries.size();
    PFT_API_END
}

pft_status pft_table_entry(pft_table_t t, size_t i, double* eps, int* r, double* xi, pft_c128* coeffs,
                           double* achieved) {
    PFT_API_BEGIN
    const Table& T = tab(t);
    PFT_REQUIRE(i < T.entries.size(), "table_entry: index out of range");
    const TableEntry& e = T.entries[i];
    if (eps) *eps = e.eps;
    if (r) *r = e.r;
    if (xi) *xi = e.xi;
    if (coeffs) to_c(e.coeffs, coeffs);
    if (achieved) *achieved = e.achieved;
    PFT_API_END
}

pft_status pft_table_lookup(pft_table_t t, double eps, int r, double* xi, pft_c128* coeffs, double* achieved) {
    PFT_API_BEGIN
    const Table& T = tab(t);
    if (!T.has_eps(eps)) fail(PFT_ERR_EPSILON_NOT_IN_TABLE, "table_lookup: epsilon not in table");
    const TableEntry* e = T.find(eps, r);
    if (!e) fail(PFT_ERR_INVALID_ARGUMENT, "table_lookup: r not in table");
    if (xi) *xi = e->xi;
    if (coeffs) to_c(e->coeffs, coeffs);
    if (achieved) *achieved = e->achieved;
    PFT_API_END
}

// ------------------------------------------------------------------ planner

pft_status pft_divisors(uint64_t N, uint64_t* out, size_t cap, size_t* count) {
    PFT_API_BEGIN
    PFT_REQUIRE(count != nullptr, "count is null");
    const auto d = divisors(N);
    *count = d.size();
    if (cap < d.size()) fail(PFT_ERR_BUFFER_TOO_SMALL, "divisors: capacity too small");
    if (!d.empty()) std::memcpy(out, d.data(), d.size() * sizeof(uint64_t));
    PFT_API_END
}

pft_status pft_min_terms(pft_table_t t, double eps, uint64_t M, uint64_t p, int* r) {
    PFT_API_BEGIN
    PFT_REQUIRE(r != nullptr, "r is null");
    *r = min_terms(tab(t), eps, M, p);
    PFT_API_END
}

pft_status pft_select_divisor(pft_table_t t, uint64_t N, uint64_t M, double eps, uint64_t* p, int* r,
                              double* cost) {
    PFT_API_BEGIN
    const DivisorChoice c = select_divisor(tab(t), N, M, eps);
    if (p) *p = c.p;
    if (r) *r = c.r;
    if (cost) *cost = c.cost;
    PFT_API_END
}

pft_status pft_plan_build(pft_table_t t, uint64_t N, uint64_t M, int64_t mu, uint64_t p, double eps,
                          pft_hplan_t* out) {
    PFT_API_BEGIN
    PFT_REQUIRE(out != nullptr, "out is null");
    *out = new pft_hplan_s{build_plan(tab(t), N, M, mu, p, eps)};
    PFT_API_END
}

void pft_plan_destroy(pft_hplan_t plan) { delete plan; }

pft_status pft_plan_info_get(pft_hplan_t plan, pft_plan_info* info) {
    PFT_API_BEGIN
    PFT_REQUIRE(info != nullptr, "info is null");
    const HostPlan& P = plan_of(plan);
    std::memset(info, 0, sizeof *info);
    info->N = P.N;
    info->M = P.M;
    info->mu = P.mu;
    info->p = P.p;
    info->q = P.q;
    info->r = P.r;
    info->epsilon = P.epsilon;
    info->achieved_epsilon = P.achieved_epsilon;
    info->xi = P.xi;
    info->estimated_cost = P.cost;
    info->plan_id = P.plan_id;
    PFT_API_END
}

#define PFT_COPY_FN(name, field, ctype)                                    \
    pft_status name(pft_hplan_t plan, ctype* out) {                        \
        PFT_API_BEGIN                                                      \
        PFT_REQUIRE(out != nullptr, "out is null");                        \
        const auto& v = plan_of(plan).field;                               \
        if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(v[0])); \
        PFT_API_END                                                        \
    }

PFT_COPY_FN(pft_plan_copy_w, w, pft_c128)
PFT_COPY_FN(pft_plan_copy_phase, phase, pft_c128)
PFT_COPY_FN(pft_plan_copy_tvals, tvals, double)
PFT_COPY_FN(pft_plan_copy_post_powers, post_powers, double)
PFT_COPY_FN(pft_plan_copy_post_twiddles, post_twiddles, pft_c128)
PFT_COPY_FN(pft_plan_copy_B, B.data, pft_c128)

pft_status pft_plan_json(pft_hplan_t plan, char* buf, size_t cap, size_t* needed) {
    PFT_API_BEGIN
    const std::string s = plan_json(plan_of(plan));
    if (needed) *needed = s.size() + 1;
    if (!buf || cap < s.size() + 1) fail(PFT_ERR_BUFFER_TOO_SMALL, "plan_json: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    PFT_API_END
}

pft_status pft_shard_layout(uint64_t q, int world, int rank, pft_shard_info* info) {
    PFT_API_BEGIN
    PFT_REQUIRE(info != nullptr, "info is null");
    const ShardLayout v = shard_layout(q, world, rank);
    info->pair_begin = v.pair_begin;
    info->pair_end = v.pair_end;
    info->row_len = v.row_len;
    info->front_col = v.front_col;
    info->mirror_col = v.mirror_col;
    info->single0_col = v.single0_col;
    info->singleh_col = v.singleh_col;
    PFT_API_END
}

pft_status pft_shard_gather_host(uint64_t p, uint64_t q, int world, int rank, const pft_c128* a, pft_c128* local,
                                 uint64_t row_stride) {
    PFT_API_BEGIN
    PFT_REQUIRE(a && local && p >= 1, "shard_gather_host: bad arguments");
    const ShardLayout v = shard_layout(q, world, rank);
    if (row_stride == 0) row_stride = v.row_len;
    PFT_REQUIRE(row_stride >= v.row_len, "shard_gather_host: row_stride < row_len");
    std::vector<uint64_t> g(v.row_len);
    for (uint64_t c = 0; c < v.row_len; ++c) g[c] = v.global_col(q, c);
#pragma omp parallel for schedule(static)
    for (long long k = 0; k < static_cast<long long>(p); ++k)
        for (uint64_t c = 0; c < v.row_len; ++c) local[k * row_stride + c] = a[k * q + g[c]];
    PFT_API_END
}

// ------------------------------------------------------------------ synthetic inputs

pft_status pft_sparse_tones(uint64_t seed, int n, int64_t lo, int64_t hi, int64_t* freqs, pft_c128* amps) {
    PFT_API_BEGIN
    PFT_REQUIRE(n >= 0 && lo <= hi && (n == 0 || (freqs && amps)), "sparse_tones: bad arguments");
    const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
    PFT_REQUIRE(static_cast<uint64_t>(n) <= span, "sparse_tones: more tones than distinct frequencies");
    std::unordered_set<int64_t> seen;
    uint64_t draw = 0;
    for (int t = 0; t < n; ++t) {
        int64_t f;
        do {  // distinct frequencies: redraw on collision
            f = lo + static_cast<int64_t>(pft_bits(seed, PFT_STREAM_TONE_F, draw++) % span);
        } while (!seen.insert(f).second);
        freqs[t] = f;
        const double u1 = pft_uniform_open0(pft_bits(seed, PFT_STREAM_TONE_A1, t));
        const double u2 = pft_uniform_open0(pft_bits(seed, PFT_STREAM_TONE_A2, t));
        const double rad = std::sqrt(-std::log(u1));  // CN(0,1): re, im ~ N(0, 1/2)
        const cplx z = rad * cispi_frac(static_cast<__int128>(std::ldexp(u2, 53)) * 2, (__int128)1 << 53);
        amps[t] = {z.real(), z.imag()};
    }
    PFT_API_END
}

pft_status pft_generate_host(const pft_signal_desc* d, pft_c128* out, uint64_t count) {
    PFT_API_BEGIN
    PFT_REQUIRE(d && (out || count == 0), "generate_host: bad arguments");
    PFT_REQUIRE(d->kind >= 0 && d->kind <= 2, "generate_host: unknown kind");
    PFT_REQUIRE(d->kind != 2 || d->N >= 1, "generate_host: sparse kind needs N");
    PFT_REQUIRE(d->kind != 2 || d->n_tones == 0 || (d->freqs && d->amps), "generate_host: tones missing");
    const int kind = d->kind;
    const uint64_t seed = d->seed, off = d->index_offset;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < static_cast<long long>(count); ++i) {
        const uint64_t g = off + static_cast<uint64_t>(i);
        cplx v;
        if (kind == 0) {
            v = cplx(pft_uniform_pm1(pft_bits(seed, PFT_STREAM_RE, g)),
                     pft_uniform_pm1(pft_bits(seed, PFT_STREAM_IM, g)));
        } else {
            const double u1 = pft_uniform_open0(pft_bits(seed, PFT_STREAM_G1, g));
            const uint64_t b2 = pft_bits(seed, PFT_STREAM_G2, g) >> 11;  // 53-bit integer
            const double rad = std::sqrt(-std::log(u1));
            // e^{2 pi i b2 / 2^53} with exact angle reduction
            const cplx noise = rad * cispi_frac(static_cast<__int128>(b2) * 2, (__int128)1 << 53);
            if (kind == 1) {
                v = noise;
            } else {
                cplx acc(0.0, 0.0);
                const uint64_t n = g % d->N;
                for (int t = 0; t < d->n_tones; ++t) {
                    // e^{2 pi i f n / N}, (f n) mod N reduced exactly
                    const __int128 fn = static_cast<__int128>(d->freqs[t]) * n;
                    acc += cplx(d->amps[t].re, d->amps[t].im) * cispi_frac(2 * fn, d->N);
                }
                v = acc + d->sigma * noise;
            }
        }
        out[i] = {v.real(), v.imag()};
    }
    PFT_API_END
}

pft_status pft_l1_norm(const pft_c128* a, uint64_t n, double* l1) {
    PFT_API_BEGIN
    PFT_REQUIRE(l1 != nullptr && (a != nullptr || n == 0), "l1_norm: bad arguments");
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += std::hypot(a[i].re, a[i].im);  // ascending i
    *l1 = s;
    PFT_API_END
}

// SPEC.md:361-369 (compare -> ErrorReport), with its zero-denominator convention (:364, :376).
pft_status pft_compare(const pft_c128* actual, const pft_c128* estimate, uint64_t n, double l1_input, double epsilon,
                       int two_d_bound, pft_error_report* report) {
    PFT_API_BEGIN
    PFT_REQUIRE(report != nullptr && ((actual && estimate) || n == 0), "compare: bad arguments");
    double num = 0.0, den = 0.0, mx = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double dr = estimate[i].re - actual[i].re, di = estimate[i].im - actual[i].im;
        num += dr * dr + di * di;
        den += actual[i].re * actual[i].re + actual[i].im * actual[i].im;
        mx = std::max(mx, std::hypot(dr, di));
    }
    report->relative_l2 = den > 0.0 ? std::sqrt(num / den) : (num > 0.0 ? INFINITY : 0.0);
    report->max_abs = mx;
    report->l1_input = l1_input;
    report->bound = l1_input * (two_d_bound ? epsilon * epsilon + 2.0 * epsilon : epsilon);
    report->bound_satisfied = mx <= report->bound ? 1 : 0;
    PFT_API_END
}

}  // extern "C"
