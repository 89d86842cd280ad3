// cpp_api_demo.cpp -- the reference's plan-then-execute interface, used from C++ exactly as
// code written against proj/include/pft/types.hpp + SPEC.md would use it.
//
//   g++ -std=c++20 -I include -I /usr/local/cuda/include examples/cpp_api_demo.cpp
//       -L paper_2008_12559_b200 -lpft_b200 -L /usr/local/cuda/lib64 -lcudart
//       -Wl,-rpath,$PWD/paper_2008_12559_b200 -pthread -o /tmp/pft_demo && /tmp/pft_demo [--require-gpu]
//
// Without a GPU the execute part reports pft::DeviceError and the demo still exits 0 (the
// library fails loudly, no CPU fallback); with --require-gpu a DeviceError is a failure (exit 6),
// and the execute part also runs 4 threads x 3 executes on ONE shared plan.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "pft/pft.hpp"

// DFT of a unit impulse at n0: X_m = e^{-2 pi i m n0 / N}; the worst deviation of a spectrum.
static double impulse_error(const pft::PartialSpectrum& s, std::size_t N, std::size_t n0) {
    double worst = 0.0;
    for (std::int64_t m = s.range.first(); m <= s.range.last(); ++m) {
        const long double ang = -2.0L * 3.14159265358979323846264338327950288L *
                                (long double)pft::mod_index(m * (std::int64_t)n0, (std::int64_t)N) / (long double)N;
        worst = std::max(worst, std::abs(s.at(m) - pft::cplx((double)std::cos(ang), (double)std::sin(ang))));
    }
    return worst;
}

int main(int argc, char** argv) {
    const bool require_gpu = argc > 1 && std::strcmp(argv[1], "--require-gpu") == 0;
    const pft::ScopeTable table = pft::ScopeTable::builtin();
    // N=16, M=2, p=4 -> q=4 and B row l=2 vanishes for j >= 1
    const pft::PftPlan small = pft::build_plan(16, 2, 0, 4, 1e-6, table);
    if (small.q != 4 || std::abs(small.B.at(2, 1)) != 0.0) return 2;
    // errors keep the reference's exception types
    try {
        pft::build_plan(16, 2, 0, 5, 1e-6, table);
        return 3;
    } catch (const std::invalid_argument&) {
    }
    try {
        (void)pft::TargetRange{0, 2}.slot(3);
        return 4;
    } catch (const std::out_of_range&) {
    }
    // BASELINE configs[1] (C2b) plan
    const pft::PftPlan plan = pft::build_plan(1u << 24, 1u << 10, 1 << 22, 1u << 15, 1e-12, table);
    std::printf("%s\n", pft::plan_json(plan).c_str());
    // the device-aware planner's choice for the same transform (model only; no GPU needed)
    const pft::CostEstimate dev = pft::select_divisor_device(1u << 24, 1u << 10, table, 1e-12);
    std::printf("device p = %zu, r = %zu, modelled %.1f us/transform\n", dev.p, dev.r, dev.cost);
    // execute an impulse: the DFT of delta is all ones
    const pft::PftPlan p2 = pft::build_plan(1u << 16, 64, 0, std::nullopt, 1e-12, table);
    pft::ComplexVec a(p2.N, pft::cplx(0.0, 0.0));
    a[0] = 1.0;
    try {
        const pft::PartialSpectrum s = pft::execute(p2, a);
        const double worst = impulse_error(s, p2.N, 0);
        std::printf("execute(impulse): max |X_m - 1| = %.3e (bound eps = %.1e)\n", worst, p2.achieved_epsilon);
        // Theorem 2: |error| <= ||a||_1 eps = eps, plus binary64 roundoff
        const double bound = p2.achieved_epsilon * 1.01 + 1e-14;
        if (!(worst <= bound)) return 5;
        // concurrent executes on one shared plan: distinct staging sets and status words
        std::vector<double> errs(12, 1.0);
        std::vector<std::thread> th;
        for (int t = 0; t < 4; ++t)
            th.emplace_back([&, t] {
                for (int k = 0; k < 3; ++k) {
                    const std::size_t n0 = 1 + 977 * (std::size_t)(3 * t + k);
                    pft::ComplexVec x(p2.N, pft::cplx(0.0, 0.0));
                    x[n0] = 1.0;
                    errs[3 * t + k] = impulse_error(pft::execute(p2, x), p2.N, n0);
                }
            });
        for (auto& x : th) x.join();
        double worst_mt = 0.0;
        for (double e : errs) worst_mt = std::max(worst_mt, e);
        std::printf("4 threads x 3 executes on one plan: max error %.3e\n", worst_mt);
        if (!(worst_mt <= bound)) return 7;
        // non-finite input maps to std::invalid_argument; the plan stays usable
        pft::ComplexVec bad(p2.N, pft::cplx(0.0, 0.0));
        bad[5] = pft::cplx(std::nan(""), 0.0);
        try {
            (void)pft::execute(p2, bad);
            return 8;
        } catch (const std::invalid_argument&) {
        }
        if (!(impulse_error(pft::execute(p2, a), p2.N, 0) <= bound)) return 9;
        // the sharded step through the C++ API on a 1-rank communicator: K1 | ncclReduce | K2
        int have_nccl = 0;
        pft_nccl_available(&have_nccl);
        if (have_nccl) {
            pft::NcclComm comm(1, 0, pft::NcclComm::unique_id(), 0);
            size_t slab_bytes = 0;
            pft_partial_bytes(p2.device_plan(), 1, &slab_bytes);
            pft::cplx *d_in = nullptr, *d_slab = nullptr, *d_out = nullptr;
            cudaMalloc(&d_in, p2.N * sizeof(pft::cplx));
            cudaMalloc(&d_slab, slab_bytes);
            cudaMalloc(&d_out, (2 * p2.M + 1) * sizeof(pft::cplx));
            cudaMemcpy(d_in, a.data(), p2.N * sizeof(pft::cplx), cudaMemcpyHostToDevice);
            pft::execute_sharded(p2, d_in, p2.q, comm.get(), 0, d_slab, d_out);
            std::vector<pft::cplx> got(2 * p2.M + 1);
            cudaMemcpy(got.data(), d_out, got.size() * sizeof(pft::cplx), cudaMemcpyDeviceToHost);
            cudaFree(d_in);
            cudaFree(d_slab);
            cudaFree(d_out);
            pft::PartialSpectrum sh;
            sh.range = p2.range();
            sh.values = got;
            const double e = impulse_error(sh, p2.N, 0);
            std::printf("execute_sharded (1 rank): max error %.3e\n", e);
            if (!(e <= bound)) return 10;
        }
        return 0;
    } catch (const pft::DeviceError& e) {
        std::printf("execute: %s\n", e.what());  // no GPU here: fails loudly, no CPU fallback
        return require_gpu ? 6 : 0;
    }
}
