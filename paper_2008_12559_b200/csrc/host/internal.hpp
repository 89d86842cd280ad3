// internal.hpp -- shared host-side declarations of libpft_b200 (not installed).
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pft/types.hpp"
#include "pft_capi.h"

namespace pft::detail {

// A C++ exception carrying a pft_status; converted to a return code at the C ABI.
struct Error : std::runtime_error {
    pft_status status;
    Error(pft_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(pft_status s, const std::string& msg) { throw Error(s, msg); }

void set_last_error(const std::string& msg);

// e^{i pi num / den} with the angle reduced exactly in integers (num mod 2*den) and the
// trigonometric evaluation done in 80-bit long double on an octant-reduced argument.
// This is the "exact angle" rule of SPEC.md:377 used for every twiddle/phase table.
cplx cispi_frac(__int128 num, __int128 den);

// ------------------------------------------------------------------ minimax
struct Poly {
    std::vector<cplx> coeffs;  // w_0..w_{r-1}
    double scope = 0.0;        // xi
    double base_frequency = 0.0;
    double achieved_error = 0.0;
};

Poly best_approx(int r, double xi, double u);
// max |P(x) - e^{iux}| over the certification grid of SPEC.md:102.
double certify(const std::vector<cplx>& coeffs, double xi, double u);
Poly scope_xi(double eps, int r);
std::vector<cplx> translate_poly(const std::vector<cplx>& coeffs, double u, double mu);

struct TableEntry {
    double eps = 0.0;
    int r = 0;
    double xi = 0.0;
    std::vector<cplx> coeffs;
    double achieved = 0.0;  // recomputed on load (not part of PFTT v1)
};

struct Table {
    uint32_t version = PFT_TABLE_VERSION;
    std::vector<TableEntry> entries;  // sorted by (eps descending, r ascending)

    const TableEntry* find(double eps, int r) const;
    bool has_eps(double eps) const;
    int r_max_for(double eps) const;
};

Table generate_table(const std::vector<double>& eps_grid, int r_max);
void save_table(const Table& t, const std::string& path);
Table load_table(const std::string& path);
Table parse_table(const unsigned char* data, size_t n, const std::string& what);
void save_table_csv(const Table& t, const std::string& path);
const Table& default_table();
std::vector<double> default_eps_grid();

// ------------------------------------------------------------------ planner
std::vector<uint64_t> divisors(uint64_t N);
int min_terms(const Table& t, double eps, uint64_t M, uint64_t p);
double spec_cost(uint64_t N, uint64_t M, uint64_t p, int r);
struct DivisorChoice {
    uint64_t p = 0;
    int r = 0;
    double cost = 0.0;
};
DivisorChoice select_divisor(const Table& t, uint64_t N, uint64_t M, double eps);

struct HostPlan {
    uint64_t N = 0, M = 0;
    int64_t mu = 0;
    uint64_t p = 0, q = 0;
    int r = 0;
    double epsilon = 0.0, achieved_epsilon = 0.0, xi = 0.0, cost = 0.0;
    uint64_t plan_id = 0;
    std::vector<cplx> w;             // r
    std::vector<cplx> phase;         // q : e^{-2 pi i mu (l - q/2) / N}
    std::vector<double> tvals;       // q : 1 - 2l/q
    ComplexMatrix B;                 // q x r
    std::vector<double> post_powers; // (2M+1) x r : ((m - mu)/p)^j
    std::vector<cplx> post_twiddles; // 2M+1 : e^{-pi i m / p}
};

HostPlan build_plan(const Table& t, uint64_t N, uint64_t M, int64_t mu, uint64_t p, double eps);
std::string plan_json(const HostPlan& plan);

// Contraction-axis layout of one rank's slice of A (see pft_shard_info in pft_capi.h).
// Columns are owned in mirror pairs (l, q-l), l in [1, L), L = ceil(q/2); the unpaired
// columns l = 0 and (even q) l = q/2 belong to rank 0.  world == 1 is the natural
// layout (local column == global column).
struct ShardLayout {
    uint64_t pair_begin = 1, pair_end = 1;
    uint64_t row_len = 0;
    int64_t front_col = 0, mirror_col = 0, single0_col = -1, singleh_col = -1;
    // global column of local column c (c < row_len)
    uint64_t global_col(uint64_t q, uint64_t c) const;
};
ShardLayout shard_layout(uint64_t q, int world, int rank);

}  // namespace pft::detail

struct pft_table_s {
    pft::detail::Table table;
    bool owned_by_library = false;
};

struct pft_hplan_s {
    pft::detail::HostPlan plan;
};
