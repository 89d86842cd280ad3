// cpp_api_demo.cpp -- the reference's plan-then-execute interface, used from C++ exactly as
// code written against proj/include/pft/types.hpp + SPEC.md would use it.
//
//   g++ -std=c++20 -I include examples/cpp_api_demo.cpp -L paper_2008_12559_b200 -lpft_b200
//       -Wl,-rpath,$PWD/paper_2008_12559_b200 -o /tmp/pft_demo && /tmp/pft_demo
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "pft/pft.hpp"

int main() {
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
        double worst = 0.0;
        for (std::int64_t m = s.range.first(); m <= s.range.last(); ++m)
            worst = std::max(worst, std::abs(s.at(m) - pft::cplx(1.0, 0.0)));
        std::printf("execute(impulse): max |X_m - 1| = %.3e (bound eps = %.1e)\n", worst, p2.achieved_epsilon);
        return worst <= p2.achieved_epsilon ? 0 : 5;
    } catch (const pft::DeviceError& e) {
        std::printf("execute: %s\n", e.what());  // no GPU here: fails loudly, no CPU fallback
        return 0;
    }
}
