// pft/pft.hpp -- C++ interface of the B200-native PFT, mirroring the reference's SPEC
// operations (plan from N, M, mu and the accuracy parameter, then execute) over the C ABI
// of libpft_b200.so (pft_capi.h).  Header-only: link with -lpft_b200.
//
//   pft::ScopeTable table = pft::ScopeTable::builtin();
//   pft::PftPlan plan = pft::build_plan(N, M, mu, std::nullopt, 1e-12, table);  // :166-174
//   pft::PartialSpectrum out = pft::execute(plan, a);            // :233-241 (on the GPU)
//
// Errors follow the reference's conventions: precondition violations throw
// std::invalid_argument, I/O problems std::runtime_error, index errors std::out_of_range
// (TargetRange::slot, types.hpp:34-40); device problems (no sm_100 GPU, CUDA failure)
// throw pft::DeviceError -- there is no CPU fallback.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pft/types.hpp"
#include "pft_capi.h"

namespace pft {

static_assert(sizeof(cplx) == sizeof(pft_c128), "std::complex<double> must match pft_c128");

struct DeviceError : std::runtime_error {
    pft_status status;
    DeviceError(pft_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

namespace detail_api {
[[noreturn]] inline void raise(pft_status s) {
    std::string msg = std::string(pft_status_string(s)) + ": " + pft_last_error();
    switch (s) {
        case PFT_ERR_IO:
        case PFT_ERR_VERSION_MISMATCH: throw std::runtime_error(msg);
        case PFT_ERR_NO_DEVICE:
        case PFT_ERR_CUDA:
        case PFT_ERR_INTERNAL: throw DeviceError(s, msg);
        default: throw std::invalid_argument(msg);
    }
}
inline void check(pft_status s) {
    if (s != PFT_OK) raise(s);
}
inline pft_c128* c(cplx* p) { return reinterpret_cast<pft_c128*>(p); }
inline const pft_c128* c(const cplx* p) { return reinterpret_cast<const pft_c128*>(p); }
}  // namespace detail_api

// ---------------------------------------------------------------- minimax

struct ApproxPoly {
    std::size_t degree = 0;
    std::vector<cplx> coeffs;
    double base_frequency = 0.0;
    double scope = 0.0;
    double achieved_error = 0.0;
};

inline ApproxPoly best_approx(int r, double xi, double u) {
    ApproxPoly P;
    P.coeffs.resize(r > 0 ? r : 1);
    detail_api::check(pft_best_approx(r, xi, u, detail_api::c(P.coeffs.data()), &P.achieved_error));
    P.degree = static_cast<std::size_t>(r - 1);
    P.base_frequency = u;
    P.scope = xi < 0 ? -xi : xi;
    return P;
}

inline std::pair<double, ApproxPoly> scope_xi(double epsilon, int r) {
    ApproxPoly P;
    P.coeffs.resize(r > 0 ? r : 1);
    double xi = 0.0;
    detail_api::check(pft_scope_xi(epsilon, r, &xi, detail_api::c(P.coeffs.data()), &P.achieved_error));
    P.degree = static_cast<std::size_t>(r - 1);
    P.base_frequency = 3.14159265358979323846;
    P.scope = xi;
    return {xi, P};
}

inline ApproxPoly translate_poly(const ApproxPoly& P, double u, double mu) {
    ApproxPoly Q = P;
    detail_api::check(pft_translate_poly(detail_api::c(P.coeffs.data()), static_cast<int>(P.coeffs.size()), u, mu,
                                         detail_api::c(Q.coeffs.data())));
    Q.base_frequency = u;
    return Q;
}

class ScopeTable {  // SPEC.md:43-49, PFTT v1 file format SPEC.md:108
public:
    static ScopeTable builtin() {
        pft_table_t t = nullptr;
        detail_api::check(pft_table_default(&t));
        return ScopeTable(t, false);
    }
    static ScopeTable generate(const std::vector<double>& epsilons, int r_max) {  // cmd_gen_table
        pft_table_t t = nullptr;
        detail_api::check(pft_table_generate(epsilons.data(), static_cast<int>(epsilons.size()), r_max, &t));
        return ScopeTable(t, true);
    }
    static ScopeTable load(const std::string& path) {  // load_table
        pft_table_t t = nullptr;
        detail_api::check(pft_table_load(path.c_str(), &t));
        return ScopeTable(t, true);
    }
    void save(const std::string& path) const { detail_api::check(pft_table_save(h_.get(), path.c_str())); }
    std::size_t size() const {
        std::size_t n = 0;
        detail_api::check(pft_table_size(h_.get(), &n));
        return n;
    }
    pft_table_t handle() const { return h_.get(); }

private:
    static void destroy(pft_table_s* p) { pft_table_destroy(p); }
    static void keep(pft_table_s*) {}  // the builtin table is owned by the library
    ScopeTable(pft_table_t t, bool owned) : h_(t, owned ? &ScopeTable::destroy : &ScopeTable::keep) {}
    std::shared_ptr<pft_table_s> h_;
};

// ---------------------------------------------------------------- planner

struct CostEstimate {
    std::size_t p = 0;
    std::size_t r = 0;
    double cost = 0.0;
};

inline std::vector<std::size_t> divisors(std::size_t N) {
    std::size_t n = 0;
    pft_status s = pft_divisors(N, nullptr, 0, &n);
    if (s != PFT_OK && s != PFT_ERR_BUFFER_TOO_SMALL) detail_api::raise(s);
    std::vector<uint64_t> d(n);
    detail_api::check(pft_divisors(N, d.data(), d.size(), &n));
    return std::vector<std::size_t>(d.begin(), d.end());
}

inline std::size_t min_terms(double epsilon, std::size_t M, std::size_t p, const ScopeTable& t) {  // :156-164
    int r = 0;
    detail_api::check(pft_min_terms(t.handle(), epsilon, M, p, &r));
    return static_cast<std::size_t>(r);
}

inline std::pair<std::size_t, CostEstimate> select_divisor(std::size_t N, std::size_t M, const ScopeTable& t,
                                                           double epsilon) {
    uint64_t p = 0;
    int r = 0;
    double cost = 0.0;
    detail_api::check(pft_select_divisor(t.handle(), N, M, epsilon, &p, &r, &cost));
    return {static_cast<std::size_t>(p), CostEstimate{static_cast<std::size_t>(p), static_cast<std::size_t>(r), cost}};
}

// Device-aware choice of p for the B200 path (not in the reference):
// the calibrated time model (cost = modelled microseconds per transform) ...
inline CostEstimate select_divisor_device(std::size_t N, std::size_t M, const ScopeTable& t, double epsilon,
                                          int n_sms = 148) {
    uint64_t p = 0;
    int r = 0;
    double us = 0.0;
    detail_api::check(pft_select_divisor_device(t.handle(), N, M, epsilon, n_sms, &p, &r, &us));
    return CostEstimate{static_cast<std::size_t>(p), static_cast<std::size_t>(r), us};
}

// ... or measured: the model's best `candidates` timed on `device` with the caller's device
// input (batch x N complex128).  Returns {p, microseconds per execute}.
inline std::pair<std::size_t, double> autotune_divisor(std::size_t N, std::size_t M, std::int64_t mu,
                                                       const ScopeTable& t, double epsilon, const cplx* d_in,
                                                       std::size_t batch = 1, int candidates = 4, int device = 0) {
    uint64_t p = 0;
    double us = 0.0;
    detail_api::check(pft_autotune_divisor(t.handle(), N, M, mu, epsilon, device, detail_api::c(d_in), batch,
                                           candidates, &p, &us));
    return {static_cast<std::size_t>(p), us};
}

// Frozen configuration.  Tables are host copies; the device upload is
// made on first use per device and cached in the plan.  A plan is shareable across threads
// (SPEC.md:188, 263-265): the cache is guarded by a mutex and shared by copies of the plan, and
// device plans are never replaced once created (a call on another device adds its own).
struct PftPlan {
    std::size_t N = 0, M = 0;
    std::int64_t mu = 0;
    std::size_t p = 0, q = 0, r = 0;
    double epsilon = 0.0, achieved_epsilon = 0.0;
    ComplexMatrix B;                  // q x r
    std::vector<double> post_powers;  // (2M+1) x r
    ComplexVec post_twiddles;         // 2M+1
    std::uint64_t plan_id = 0;

    TargetRange range() const { return TargetRange{mu, M}; }
    pft_hplan_t handle() const { return host_.get(); }
    pft_dplan_t device_plan(int device = 0) const {
        std::lock_guard<std::mutex> lk(devices_->mu);
        auto it = devices_->plans.find(device);
        if (it != devices_->plans.end()) return it->second.get();
        pft_dplan_opts o{};
        o.device = device;
        pft_dplan_t d = nullptr;
        detail_api::check(pft_dplan_create(host_.get(), &o, &d));
        auto& slot = devices_->plans[device];
        slot = std::shared_ptr<pft_dplan_s>(d, [](pft_dplan_s* x) { pft_dplan_destroy(x); });
        return slot.get();
    }

    struct DeviceCache {
        std::mutex mu;
        std::map<int, std::shared_ptr<pft_dplan_s>> plans;
    };
    std::shared_ptr<pft_hplan_s> host_;
    std::shared_ptr<DeviceCache> devices_ = std::make_shared<DeviceCache>();
};

inline PftPlan build_plan(std::size_t N, std::size_t M, std::int64_t mu, std::optional<std::size_t> p,
                          double epsilon, const ScopeTable& table) {  // Algorithm 1
    pft_hplan_t h = nullptr;
    detail_api::check(pft_plan_build(table.handle(), N, M, mu, p.value_or(0), epsilon, &h));
    PftPlan P;
    P.host_ = std::shared_ptr<pft_hplan_s>(h, [](pft_hplan_s* x) { pft_plan_destroy(x); });
    pft_plan_info info{};
    detail_api::check(pft_plan_info_get(h, &info));
    P.N = info.N;
    P.M = info.M;
    P.mu = info.mu;
    P.p = info.p;
    P.q = info.q;
    P.r = static_cast<std::size_t>(info.r);
    P.epsilon = info.epsilon;
    P.achieved_epsilon = info.achieved_epsilon;
    P.plan_id = info.plan_id;
    P.B = ComplexMatrix(P.q, P.r);
    detail_api::check(pft_plan_copy_B(h, detail_api::c(P.B.data.data())));
    P.post_powers.resize((2 * P.M + 1) * P.r);
    detail_api::check(pft_plan_copy_post_powers(h, P.post_powers.data()));
    P.post_twiddles.resize(2 * P.M + 1);
    detail_api::check(pft_plan_copy_post_twiddles(h, detail_api::c(P.post_twiddles.data())));
    return P;
}

inline std::string plan_json(const PftPlan& P) {
    std::size_t need = 0;
    pft_plan_json(P.handle(), nullptr, 0, &need);
    std::string s(need, '\0');
    detail_api::check(pft_plan_json(P.handle(), s.data(), s.size(), &need));
    s.resize(need ? need - 1 : 0);
    return s;
}

// ---------------------------------------------------------------- transform

// execute(plan, a) -> PartialSpectrum: host vector in, host spectrum out;
// the transform runs on the GPU (H2D, kernels, D2H through a staging set the device plan keeps,
// so repeated calls do not allocate).  Re-entrant: concurrent calls on one plan use distinct
// staging sets and status words.  Throws std::invalid_argument on a length mismatch or
// non-finite input, pft::DeviceError without a usable sm_100 GPU.
inline PartialSpectrum execute(const PftPlan& plan, const ComplexVec& a, int device = 0) {
    if (a.size() != plan.N)
        throw std::invalid_argument("execute: length mismatch (a.len=" + std::to_string(a.size()) +
                                    ", plan.N=" + std::to_string(plan.N) + ")");
    PartialSpectrum out;
    out.range = plan.range();
    out.values.resize(out.range.count());
    out.plan_id = plan.plan_id;
    detail_api::check(pft_execute_host(plan.device_plan(device), detail_api::c(a.data()), 1,
                                       detail_api::c(out.values.data()), nullptr, nullptr, nullptr));
    return out;
}

// Device-pointer form: asynchronous on `stream`, no allocation when `workspace` is given
// (pft_workspace_bytes), graph-capturable.  flags: PFT_EXEC_OVERLAP_PREVIOUS lets K1 stream
// while the preceding kernel on the stream finishes (d_in must not be that kernel's output).
inline void execute_device(const PftPlan& plan, const cplx* d_in, cplx* d_out, void* stream = nullptr,
                           void* workspace = nullptr, std::size_t batch = 1, std::size_t in_stride = 0,
                           int device = 0, unsigned flags = PFT_EXEC_DEFAULT) {
    detail_api::check(pft_execute_ex(plan.device_plan(device), detail_api::c(d_in), batch, in_stride,
                                     detail_api::c(d_out), workspace, stream, flags));
}

// ---------------------------------------------------------------- sharded transform

// A NCCL communicator made by the library (pft_nccl_comm_init); any ncclComm_t the application
// created with its own NCCL can be passed to execute_sharded instead.
class NcclComm {
public:
    static std::vector<unsigned char> unique_id() {  // on one rank; share it with the others
        std::vector<unsigned char> id(PFT_NCCL_UNIQUE_ID_BYTES);
        detail_api::check(pft_nccl_get_unique_id(id.data()));
        return id;
    }
    NcclComm(int world, int rank, const std::vector<unsigned char>& id, int device) {
        if (id.size() != PFT_NCCL_UNIQUE_ID_BYTES) throw std::invalid_argument("NCCL unique id must be 128 bytes");
        detail_api::check(pft_nccl_comm_init(world, rank, id.data(), device, &comm_));
    }
    NcclComm(const NcclComm&) = delete;
    NcclComm& operator=(const NcclComm&) = delete;
    ~NcclComm() { pft_nccl_comm_destroy(comm_); }
    struct ncclComm* get() const { return comm_; }

private:
    struct ncclComm* comm_ = nullptr;
};

// Device-aware p for the transform sharded over `world` GPUs (the collective included).
inline CostEstimate select_divisor_sharded(std::size_t N, std::size_t M, const ScopeTable& t, double epsilon,
                                           int world, int n_sms = 148) {
    uint64_t p = 0;
    int r = 0;
    double us = 0.0;
    detail_api::check(pft_select_divisor_sharded(t.handle(), N, M, epsilon, n_sms, world, &p, &r, &us));
    return CostEstimate{static_cast<std::size_t>(p), static_cast<std::size_t>(r), us};
}

// One rank's step of the contraction-axis sharded transform: K1 on this rank's slice
// (pft_shard_layout row layout, row_stride elements per row), ncclReduce of the p x r partial
// slab onto `root` over NVLink, K2 on the root into d_out (2M+1 values; unused elsewhere).
// d_slab: pft_partial_bytes(plan, 1) bytes of device memory on every rank.  Asynchronous on
// `stream`, graph-capturable.  The plan's device upload must be the communicator's device.
inline void execute_sharded(const PftPlan& plan, const cplx* d_in_local, std::uint64_t row_stride,
                            struct ncclComm* comm, int root, cplx* d_slab, cplx* d_out, void* stream = nullptr,
                            int device = 0) {
    detail_api::check(pft_execute_sharded(plan.device_plan(device), detail_api::c(d_in_local), row_stride, comm, root,
                                          detail_api::c(d_slab), detail_api::c(d_out), stream));
}

}  // namespace pft
