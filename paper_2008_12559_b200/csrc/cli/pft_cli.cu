// pft_cli.cu -- the command-line surface of the reference (cli module) over the
// C ABI of libpft_b200.so: gen-table, plan, transform, transform2d, bench, anomaly.
//
//   pft gen-table  [--epsilons 1e-1,...] [--r-max 25] --out PATH [--csv PATH]
//   pft plan       --N n --M m [--mu u] [--p p] [--epsilon e] [--table PATH] [--device] [--world G]
//   pft transform  --input PATH [--N n] --M m [--mu u] [--p p] [--epsilon e] [--table PATH]
//                  --output CSV [--verify] [--device-p]
//   pft transform2d --input PATH --N1 a --N2 b --M1 c --M2 d [--mu1 x] [--mu2 y] [--p1 .] [--p2 .]
//                  --output CSV [--verify]
//   pft bench      --mode vary-n|vary-m|vary-ratio [--reps 100] [--warmup 5] --out CSV [--force]
//                  [--epsilon 1e-6] [--oracle-max-n 65536] [--max-n N]
//   pft anomaly    --input PATH --M m --k k [--source pft|fft] [--out PATH]
//
// Exit codes: 0 ok, 1 I/O or parse error, 2 invalid parameters, 3 verification
// failure (relative l2 >= 1e-6); and 4 when no usable sm_100 GPU / CUDA failure (this build has no
// CPU fallback; the reference's CLI has no such case).  Common flags: --table, --epsilon, --p, --json.
// Compiled by nvcc as host code (the bench times with CUDA events); the transform itself runs in the
// library.  The bench's full-FFT baseline is cuFFT, loaded at run time when present ("external
// baselines are report-only via a documented hook", SPEC.md cli DESIGN DECISIONS).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "pft_capi.h"

namespace {

constexpr int kExitIo = 1, kExitParam = 2, kExitVerify = 3, kExitDevice = 4;

struct CliError : std::runtime_error {
    int code;
    CliError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

int exit_code_for(pft_status s) {
    switch (s) {
        case PFT_ERR_IO:
        case PFT_ERR_VERSION_MISMATCH: return kExitIo;
        case PFT_ERR_NO_DEVICE:
        case PFT_ERR_CUDA:
        case PFT_ERR_INTERNAL: return kExitDevice;
        default: return kExitParam;
    }
}

void check(pft_status s, const char* what) {
    if (s != PFT_OK) {
        const std::string detail = pft_last_error();
        throw CliError(exit_code_for(s), std::string(what) + ": " + (detail.empty() ? pft_status_string(s) : detail));
    }
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CliError(kExitDevice, std::string(what) + ": " + cudaGetErrorString(e));
}

// --name value / --flag arguments
struct Args {
    std::map<std::string, std::string> kv;
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    std::string need(const std::string& k) const {
        if (!has(k)) throw CliError(kExitParam, "missing --" + k);
        return str(k);
    }
    long long integer(const std::string& k, long long def) const {
        if (!has(k)) return def;
        char* end = nullptr;
        const std::string v = str(k);
        const long long x = std::strtoll(v.c_str(), &end, 0);
        if (v.empty() || *end) throw CliError(kExitParam, "--" + k + ": not an integer: " + v);
        return x;
    }
    long long need_int(const std::string& k) const {
        need(k);
        return integer(k, 0);
    }
    double real(const std::string& k, double def) const {
        if (!has(k)) return def;
        char* end = nullptr;
        const std::string v = str(k);
        const double x = std::strtod(v.c_str(), &end);
        if (v.empty() || *end) throw CliError(kExitParam, "--" + k + ": not a number: " + v);
        return x;
    }
};

Args parse(int argc, char** argv, int from) {
    Args a;
    for (int i = from; i < argc; ++i) {
        std::string t = argv[i];
        if (t.rfind("--", 0) != 0) throw CliError(kExitParam, "unexpected argument: " + t);
        t = t.substr(2);
        const auto eq = t.find('=');
        if (eq != std::string::npos) {
            a.kv[t.substr(0, eq)] = t.substr(eq + 1);
        } else if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) {
            a.kv[t] = argv[++i];
        } else {
            a.kv[t] = "1";
        }
    }
    return a;
}

pft_table_t table_for(const Args& a) {
    pft_table_t t = nullptr;
    if (a.has("table")) check(pft_table_load(a.str("table").c_str(), &t), "load_table");
    else check(pft_table_default(&t), "default table");
    return t;
}
void release_table(const Args& a, pft_table_t t) {
    if (a.has("table")) pft_table_destroy(t);
}

std::string plan_json(pft_hplan_t h) {
    size_t need = 0;
    pft_plan_json(h, nullptr, 0, &need);
    std::string s(need, '\0');
    check(pft_plan_json(h, s.data(), s.size(), &need), "plan_json");
    s.resize(need ? need - 1 : 0);
    return s;
}

struct Signal {
    std::vector<pft_c128> v;
    bool is_complex = false;
};

Signal read_signal(const std::string& path, const Args& a) {
    const std::string fmt = a.str("format", path.size() > 4 && path.substr(path.size() - 4) == ".csv" ? "csv" : "f64le");
    const int f = fmt == "csv" ? PFT_SIGNAL_CSV : fmt == "f64le" ? PFT_SIGNAL_F64LE : -1;
    if (f < 0) throw CliError(kExitParam, "--format must be csv or f64le");
    uint64_t n = 0;
    int cx = 0;
    check(pft_signal_read(path.c_str(), f, nullptr, 0, &n, &cx), "read signal");
    Signal s;
    s.v.resize(n);
    check(pft_signal_read(path.c_str(), f, s.v.data(), n, &n, &cx), "read signal");
    s.is_complex = cx != 0;
    return s;
}

void print_report(const pft_error_report& r) {
    std::printf("{\"relative_l2\": %.17g, \"max_abs\": %.17g, \"l1_input\": %.17g, \"bound\": %.17g, "
                "\"bound_satisfied\": %s}\n",
                r.relative_l2, r.max_abs, r.l1_input, r.bound, r.bound_satisfied ? "true" : "false");
}

// ------------------------------------------------------------------ gen-table
int cmd_gen_table(const Args& a) {
    std::vector<double> eps;
    if (a.has("epsilons")) {
        std::string s = a.str("epsilons");
        size_t i = 0;
        while (i <= s.size()) {
            const size_t j = std::min(s.find(',', i), s.size());
            const std::string tok = s.substr(i, j - i);
            char* end = nullptr;
            const double e = std::strtod(tok.c_str(), &end);
            if (tok.empty() || *end) throw CliError(kExitParam, "--epsilons: bad value " + tok);
            eps.push_back(e);
            i = j + 1;
        }
    }
    const int r_max = (int)a.integer("r-max", 25);
    pft_table_t t = nullptr;
    check(pft_table_generate(eps.empty() ? nullptr : eps.data(), (int)eps.size(), r_max, &t), "gen_table");
    const pft_status s = pft_table_save(t, a.need("out").c_str());
    if (s == PFT_OK && a.has("csv")) check(pft_table_save_csv(t, a.str("csv").c_str()), "save_table_csv");
    size_t n = 0;
    pft_table_size(t, &n);
    pft_table_destroy(t);
    check(s, "save_table");
    std::printf("{\"entries\": %zu, \"r_max\": %d, \"out\": \"%s\"}\n", n, r_max, a.str("out").c_str());
    return 0;
}

// ------------------------------------------------------------------ plan
int cmd_plan(const Args& a) {
    pft_table_t t = table_for(a);
    const uint64_t N = (uint64_t)a.need_int("N"), M = (uint64_t)a.need_int("M");
    const int64_t mu = a.integer("mu", 0);
    const double eps = a.real("epsilon", 1e-12);
    pft_hplan_t h = nullptr;
    check(pft_plan_build(t, N, M, mu, (uint64_t)a.integer("p", 0), eps, &h), "build_plan");
    std::printf("%s\n", plan_json(h).c_str());
    if (a.has("device")) {  // the B200 planner's choices (not in the reference)
        uint64_t p = 0;
        int r = 0;
        double us = 0.0;
        check(pft_select_divisor_device(t, N, M, eps, 148, &p, &r, &us), "select_divisor_device");
        std::printf("{\"device_p\": %llu, \"device_r\": %d, \"modelled_us\": %.3f}\n", (unsigned long long)p, r, us);
        const int G = (int)a.integer("world", 0);
        if (G > 0) {
            check(pft_select_divisor_sharded(t, N, M, eps, 148, G, &p, &r, &us), "select_divisor_sharded");
            std::printf("{\"world\": %d, \"sharded_p\": %llu, \"sharded_r\": %d, \"modelled_us\": %.3f}\n", G,
                        (unsigned long long)p, r, us);
        }
    }
    pft_plan_destroy(h);
    release_table(a, t);
    return 0;
}

// ------------------------------------------------------------------ transform
int cmd_transform(const Args& a) {
    Signal sig = read_signal(a.need("input"), a);
    uint64_t N = (uint64_t)a.integer("N", (long long)sig.v.size());
    if (N == 0 || N > sig.v.size()) throw CliError(kExitParam, "--N must be in [1, signal length]");
    sig.v.resize(N);
    const uint64_t M = (uint64_t)a.need_int("M");
    const int64_t mu = a.integer("mu", 0);
    const double eps = a.real("epsilon", 1e-12);
    const std::string out_path = a.need("output");
    pft_table_t t = table_for(a);
    uint64_t p = (uint64_t)a.integer("p", 0);
    if (!p && a.has("device-p")) {
        int r = 0;
        double us = 0.0;
        check(pft_select_divisor_device(t, N, M, eps, 148, &p, &r, &us), "select_divisor_device");
    }
    pft_hplan_t h = nullptr;
    check(pft_plan_build(t, N, M, mu, p, eps, &h), "build_plan");
    pft_plan_info info{};
    check(pft_plan_info_get(h, &info), "plan_info");
    pft_dplan_t d = nullptr;
    check(pft_dplan_create(h, nullptr, &d), "device plan");
    std::vector<pft_c128> out(2 * M + 1);
    const pft_status st = pft_execute_host(d, sig.v.data(), 1, out.data(), nullptr, nullptr, nullptr);
    pft_dplan_destroy(d);
    check(st, "execute");
    check(pft_spectrum_write_csv(out_path.c_str(), mu, M, out.data()), "write spectrum");
    int code = 0;
    if (a.has("verify")) {  // naive DFT on the GPU (exact angles) + ErrorReport
        std::vector<pft_c128> exact(2 * M + 1);
        check(pft_naive_dft_host(sig.v.data(), N, mu - (int64_t)M, 2 * M + 1, exact.data()), "naive_dft");
        double l1 = 0.0;
        check(pft_l1_norm(sig.v.data(), N, &l1), "l1_norm");
        pft_error_report rep{};
        check(pft_compare(exact.data(), out.data(), 2 * M + 1, l1, info.achieved_epsilon, 0, &rep), "compare");
        print_report(rep);
        if (!(rep.relative_l2 < 1e-6)) code = kExitVerify;
    }
    pft_plan_destroy(h);
    release_table(a, t);
    return code;
}

// ------------------------------------------------------------------ transform2d
int cmd_transform2d(const Args& a) {
    Signal sig = read_signal(a.need("input"), a);
    const uint64_t N1 = (uint64_t)a.need_int("N1"), N2 = (uint64_t)a.need_int("N2");
    if (N1 * N2 != sig.v.size()) throw CliError(kExitParam, "N1 * N2 != signal length");
    const uint64_t M1 = (uint64_t)a.need_int("M1"), M2 = (uint64_t)a.need_int("M2");
    const int64_t mu1 = a.integer("mu1", 0), mu2 = a.integer("mu2", 0);
    const double eps = a.real("epsilon", 1e-12);
    if (2 * M1 > N1 || 2 * M2 > N2) throw CliError(kExitParam, "M_d > N_d / 2");
    pft_table_t t = table_for(a);
    pft_hplan_t h1 = nullptr, h2 = nullptr;
    check(pft_plan_build(t, N1, M1, mu1, (uint64_t)a.integer("p1", 0), eps, &h1), "build_plan (axis 1)");
    check(pft_plan_build(t, N2, M2, mu2, (uint64_t)a.integer("p2", 0), eps, &h2), "build_plan (axis 2)");
    pft_dplan_opts ro{}, co{};
    ro.batch_hint = N1;
    co.batch_hint = 2 * M2 + 1;
    pft_dplan_t rows = nullptr, cols = nullptr;
    check(pft_dplan_create(h2, &ro, &rows), "device plan (rows)");
    check(pft_dplan_create(h1, &co, &cols), "device plan (columns)");
    const uint64_t W1 = 2 * M1 + 1, W2 = 2 * M2 + 1;
    std::vector<pft_c128> out(W1 * W2);
    const pft_status st = pft_execute_2d_host(rows, cols, sig.v.data(), out.data());
    pft_dplan_destroy(rows);
    pft_dplan_destroy(cols);
    check(st, "execute_2d");
    std::FILE* f = std::fopen(a.need("output").c_str(), "w");
    if (!f) throw CliError(kExitIo, "cannot write " + a.str("output"));
    std::fprintf(f, "m1,m2,re,im\n");
    for (uint64_t i = 0; i < W1; ++i)
        for (uint64_t j = 0; j < W2; ++j)
            std::fprintf(f, "%lld,%lld,%.17g,%.17g\n", (long long)(mu1 - (int64_t)M1 + (int64_t)i),
                         (long long)(mu2 - (int64_t)M2 + (int64_t)j), out[i * W2 + j].re, out[i * W2 + j].im);
    if (std::fclose(f) != 0) throw CliError(kExitIo, "cannot write " + a.str("output"));
    int code = 0;
    if (a.has("verify")) {  // separable naive 2-D DFT (Eq. (10)): rows, then columns, on the GPU
        std::vector<pft_c128> X(N1 * W2), XT(W2 * N1), Z(W2 * W1), exact(W1 * W2);
        for (uint64_t r = 0; r < N1; ++r)
            check(pft_naive_dft_host(sig.v.data() + r * N2, N2, mu2 - (int64_t)M2, W2, X.data() + r * W2), "naive_dft");
        for (uint64_t r = 0; r < N1; ++r)
            for (uint64_t c = 0; c < W2; ++c) XT[c * N1 + r] = X[r * W2 + c];
        for (uint64_t c = 0; c < W2; ++c)
            check(pft_naive_dft_host(XT.data() + c * N1, N1, mu1 - (int64_t)M1, W1, Z.data() + c * W1), "naive_dft");
        for (uint64_t i = 0; i < W1; ++i)
            for (uint64_t j = 0; j < W2; ++j) exact[i * W2 + j] = Z[j * W1 + i];
        pft_plan_info i1{}, i2{};
        pft_plan_info_get(h1, &i1);
        pft_plan_info_get(h2, &i2);
        double l1 = 0.0;
        check(pft_l1_norm(sig.v.data(), sig.v.size(), &l1), "l1_norm");
        pft_error_report rep{};
        check(pft_compare(exact.data(), out.data(), W1 * W2, l1, std::max(i1.achieved_epsilon, i2.achieved_epsilon), 1,
                          &rep),
              "compare");
        print_report(rep);
        if (!(rep.relative_l2 < 1e-6)) code = kExitVerify;
    }
    pft_plan_destroy(h1);
    pft_plan_destroy(h2);
    release_table(a, t);
    return code;
}

// ------------------------------------------------------------------ bench
// cuFFT full-size transform as the "full_fft" baseline (report-only hook; absent -> skipped).
struct CuFft {
    void* h = nullptr;
    int (*plan1d)(int*, int, int, int) = nullptr;
    int (*exec)(int, void*, void*, int) = nullptr;
    int (*destroy)(int) = nullptr;
    CuFft() {
        for (const char* n : {"libcufft.so.11", "libcufft.so"})
            if ((h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) return;
        plan1d = reinterpret_cast<int (*)(int*, int, int, int)>(dlsym(h, "cufftPlan1d"));
        exec = reinterpret_cast<int (*)(int, void*, void*, int)>(dlsym(h, "cufftExecZ2Z"));
        destroy = reinterpret_cast<int (*)(int)>(dlsym(h, "cufftDestroy"));
        if (!plan1d || !exec || !destroy) h = nullptr;
    }
};

struct Stats {
    double mean = 0.0, sd = 0.0;
};
template <class F>
Stats time_reps(int warmup, int reps, F&& fn) {
    for (int i = 0; i < warmup; ++i) fn();
    cuda(cudaDeviceSynchronize(), "synchronize");
    cudaEvent_t e0, e1;
    cuda(cudaEventCreate(&e0), "event");
    cuda(cudaEventCreate(&e1), "event");
    std::vector<double> ms(reps);
    for (int i = 0; i < reps; ++i) {
        cuda(cudaEventRecord(e0, nullptr), "event record");
        fn();
        cuda(cudaEventRecord(e1, nullptr), "event record");
        cuda(cudaEventSynchronize(e1), "event synchronize");
        float f = 0.f;
        cuda(cudaEventElapsedTime(&f, e0, e1), "elapsed");
        ms[i] = f;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    Stats s;
    for (double x : ms) s.mean += x;
    s.mean /= reps;
    for (double x : ms) s.sd += (x - s.mean) * (x - s.mean);
    s.sd = reps > 1 ? std::sqrt(s.sd / (reps - 1)) : 0.0;
    return s;
}

double rel_l2(const std::vector<pft_c128>& exact, const std::vector<pft_c128>& est) {
    pft_error_report r{};
    check(pft_compare(exact.data(), est.data(), exact.size(), 0.0, 0.0, 0, &r), "compare");
    return r.relative_l2;
}

int cmd_bench(const Args& a) {
    const std::string mode = a.need("mode");
    const int reps = (int)a.integer("reps", 100), warmup = (int)a.integer("warmup", 5);
    if (reps < 1 || warmup < 0) throw CliError(kExitParam, "--reps >= 1, --warmup >= 0");
    const double eps = a.real("epsilon", 1e-6);
    const uint64_t oracle_max = (uint64_t)a.integer("oracle-max-n", 1 << 16);
    struct Cell {
        uint64_t N, M;
        uint64_t p;  // 0 = the planner's
    };
    std::vector<Cell> cells;
    if (mode == "vary-n") {
        for (int e = 12; e <= 22; ++e) cells.push_back({1ull << e, 1ull << 9, 0});
    } else if (mode == "vary-m") {
        for (int e = 9; e <= 18; ++e) cells.push_back({1ull << 22, 1ull << e, 0});
    } else if (mode == "vary-ratio") {  // Table 3: M/p in {1/32, 1/8, 1/2, 1, 2, 4}
        for (uint64_t M : {1ull << 9, 1ull << 12, 1ull << 15})
            for (double ratio : {1.0 / 32, 1.0 / 8, 0.5, 1.0, 2.0, 4.0}) {
                const uint64_t p = (uint64_t)std::llround((double)M / ratio);
                if (p > 1 && (1ull << 22) % p == 0) cells.push_back({1ull << 22, M, p});
            }
    } else {
        throw CliError(kExitParam, "--mode must be vary-n, vary-m or vary-ratio");
    }
    for (const Cell& c : cells)
        if (c.N > (1ull << 24) && !a.has("force")) throw CliError(kExitParam, "N > 2^24 needs --force");
    const uint64_t max_n = (uint64_t)a.integer("max-n", 0);  // skip larger cells (quick runs)
    std::FILE* f = std::fopen(a.need("out").c_str(), "w");
    if (!f) throw CliError(kExitIo, "cannot write " + a.str("out"));
    std::fprintf(f, "algo,N,M,mu,p,r,reps,mean_ms,stddev_ms,rel_l2\n");
    pft_table_t t = table_for(a);
    CuFft fft;
    for (const Cell& c : cells) {
        if (max_n && c.N > max_n) continue;
        const int64_t mu = 0;
        const uint64_t W = 2 * c.M + 1;
        pft_hplan_t h = nullptr;
        const pft_status bs = pft_plan_build(t, c.N, c.M, mu, c.p, eps, &h);
        if (bs == PFT_ERR_RATIO_OUT_OF_RANGE) continue;  // no table entry reaches this M/p
        check(bs, "build_plan");
        pft_plan_info info{};
        pft_plan_info_get(h, &info);
        void *in = nullptr, *out = nullptr, *full = nullptr, *ex = nullptr;
        cuda(cudaMalloc(&in, c.N * 16), "cudaMalloc");
        cuda(cudaMalloc(&out, W * 16), "cudaMalloc");
        pft_signal_desc sd{};
        sd.kind = 0;
        sd.seed = 12;
        sd.N = c.N;
        check(pft_generate_device(&sd, static_cast<pft_c128*>(in), c.N, nullptr), "generate");
        std::vector<pft_c128> exact, got(W);
        const bool run_oracle = c.N <= oracle_max;
        if (run_oracle) {
            cuda(cudaMalloc(&ex, W * 16), "cudaMalloc");
            exact.resize(W);
        }
        auto oracle_rel = [&](void* d_est) -> double {
            if (!run_oracle) return NAN;
            cuda(cudaMemcpy(got.data(), d_est, W * 16, cudaMemcpyDeviceToHost), "D2H");
            return rel_l2(exact, got);
        };
        if (run_oracle) {
            const Stats s = time_reps(0, std::min(reps, 3), [&] {
                check(pft_naive_dft_device(static_cast<const pft_c128*>(in), c.N, mu - (int64_t)c.M, W,
                                           static_cast<pft_c128*>(ex), nullptr),
                      "naive_dft");
            });
            cuda(cudaMemcpy(exact.data(), ex, W * 16, cudaMemcpyDeviceToHost), "D2H");
            std::fprintf(f, "naive,%llu,%llu,%lld,%llu,%d,%d,%.6f,%.6f,%.3g\n", (unsigned long long)c.N,
                         (unsigned long long)c.M, (long long)mu, (unsigned long long)info.p, info.r, std::min(reps, 3),
                         s.mean, s.sd, 0.0);
        }
        pft_dplan_t d = nullptr;
        check(pft_dplan_create(h, nullptr, &d), "device plan");
        const Stats sp = time_reps(warmup, reps, [&] {
            check(pft_execute(d, static_cast<const pft_c128*>(in), 1, 0, static_cast<pft_c128*>(out), nullptr, nullptr),
                  "execute");
        });
        std::fprintf(f, "pft,%llu,%llu,%lld,%llu,%d,%d,%.6f,%.6f,%.3g\n", (unsigned long long)c.N,
                     (unsigned long long)c.M, (long long)mu, (unsigned long long)info.p, info.r, reps, sp.mean, sp.sd,
                     oracle_rel(out));
        pft_dplan_destroy(d);
        if (fft.h && c.N <= (1ull << 30)) {  // full FFT of size N, then the 2M+1 bins sliced out
            int plan = 0;
            cuda(cudaMalloc(&full, c.N * 16), "cudaMalloc");
            if (fft.plan1d(&plan, (int)c.N, 0x69 /* CUFFT_Z2Z */, 1) == 0) {
                const uint64_t lo = (uint64_t)(((mu - (int64_t)c.M) % (int64_t)c.N + (int64_t)c.N) % (int64_t)c.N);
                const uint64_t first = std::min<uint64_t>(W, c.N - lo);
                const Stats sf = time_reps(warmup, reps, [&] {
                    fft.exec(plan, in, full, -1 /* CUFFT_FORWARD */);
                    cudaMemcpyAsync(out, static_cast<char*>(full) + lo * 16, first * 16, cudaMemcpyDeviceToDevice);
                    if (first < W)
                        cudaMemcpyAsync(static_cast<char*>(out) + first * 16, full, (W - first) * 16,
                                        cudaMemcpyDeviceToDevice);
                });
                std::fprintf(f, "full_fft,%llu,%llu,%lld,%llu,%d,%d,%.6f,%.6f,%.3g\n", (unsigned long long)c.N,
                             (unsigned long long)c.M, (long long)mu, 0ull, 0, reps, sf.mean, sf.sd, oracle_rel(out));
                fft.destroy(plan);
            }
            cudaFree(full);
        }
        cudaFree(in);
        cudaFree(out);
        if (ex) cudaFree(ex);
        pft_plan_destroy(h);
        std::fflush(f);
    }
    release_table(a, t);
    if (std::fclose(f) != 0) throw CliError(kExitIo, "cannot write " + a.str("out"));
    return 0;
}

// ------------------------------------------------------------------ anomaly
int cmd_anomaly(const Args& a) {
    Signal sig = read_signal(a.need("input"), a);
    const uint64_t N = sig.v.size(), M = (uint64_t)a.need_int("M"), k = (uint64_t)a.need_int("k");
    if (k < 1 || k > N) throw CliError(kExitParam, "--k must be in [1, N]");
    if (2 * M > N) throw CliError(kExitParam, "M > N / 2");
    const std::string source = a.str("source", "pft");
    std::vector<double> x(N);
    for (uint64_t i = 0; i < N; ++i) x[i] = sig.v[i].re;
    std::vector<uint64_t> idx(k);
    std::vector<double> score(k);
    if (source == "pft") {
        pft_table_t t = table_for(a);
        pft_hplan_t h = nullptr;
        check(pft_plan_build(t, N, M, 0, (uint64_t)a.integer("p", 0), a.real("epsilon", 1e-12), &h), "build_plan");
        pft_dplan_t d = nullptr;
        check(pft_dplan_create(h, nullptr, &d), "device plan");
        const pft_status st = pft_anomaly(d, x.data(), k, idx.data(), score.data(), nullptr);
        pft_dplan_destroy(d);
        pft_plan_destroy(h);
        release_table(a, t);
        check(st, "anomaly");
    } else if (source == "fft") {  // exact coefficients on R_{0,M} (naive DFT on the GPU)
        std::vector<pft_c128> xc(N), coeffs(2 * M + 1);
        for (uint64_t i = 0; i < N; ++i) xc[i] = {x[i], 0.0};
        check(pft_naive_dft_host(xc.data(), N, -(int64_t)M, 2 * M + 1, coeffs.data()), "naive_dft");
        check(pft_anomaly_from_coeffs(x.data(), N, coeffs.data(), M, k, idx.data(), score.data(), nullptr), "anomaly");
    } else {
        throw CliError(kExitParam, "--source must be pft or fft");
    }
    std::string js = "{\"k\": " + std::to_string(k) + ", \"fitted_curve_source\": \"" + source + "\", \"indices\": [";
    for (uint64_t i = 0; i < k; ++i) js += (i ? ", " : "") + std::to_string(idx[i]);
    js += "], \"scores\": [";
    char buf[64];
    for (uint64_t i = 0; i < k; ++i) {
        std::snprintf(buf, sizeof buf, "%s%.17g", i ? ", " : "", score[i]);
        js += buf;
    }
    js += "]}\n";
    if (a.has("out")) {
        std::FILE* f = std::fopen(a.str("out").c_str(), "w");
        if (!f || std::fputs(js.c_str(), f) < 0 || std::fclose(f) != 0) throw CliError(kExitIo, "cannot write " + a.str("out"));
    } else {
        std::fputs(js.c_str(), stdout);
    }
    return 0;
}

int usage() {
    std::fprintf(stderr,
                 "usage: pft <gen-table|plan|transform|transform2d|bench|anomaly> [--flag value ...]\n"
                 "exit codes: 0 ok, 1 I/O or parse, 2 invalid parameters, 3 verification failure, 4 no GPU\n");
    return kExitParam;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string verb = argv[1];
    try {
        const Args a = parse(argc, argv, 2);
        if (verb == "gen-table") return cmd_gen_table(a);
        if (verb == "plan") return cmd_plan(a);
        if (verb == "transform") return cmd_transform(a);
        if (verb == "transform2d") return cmd_transform2d(a);
        if (verb == "bench") return cmd_bench(a);
        if (verb == "anomaly") return cmd_anomaly(a);
        if (verb == "--version" || verb == "version") {
            std::printf("%s\n", pft_version());
            return 0;
        }
        return usage();
    } catch (const CliError& e) {
        std::fprintf(stderr, "pft %s: %s\n", verb.c_str(), e.what());
        return e.code;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "pft %s: %s\n", verb.c_str(), e.what());
        return kExitIo;
    }
}
