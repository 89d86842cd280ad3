// signal_io.cpp -- the data formats either side of transform.execute
// and the anomaly pipeline that calls it (SPEC.md cli module: SignalFile, cmd_transform's
// "m,re,im" output, cmd_anomaly; §4.4).
//
//   SignalFile (SPEC.md, cli "SignalFile"): csv rows "re" or "re,im"; f64le = 16-byte header
//   {magic "PFTS", u32 1 if complex else 0, u32 length} then little-endian doubles (re, or
//   interleaved re, im).  The named fields fill 12 of the 16 header bytes; bytes 12-15 are
//   reserved (written as zero, ignored on read).  Spectrum CSV: header "m,re,im", one row per m = mu - M .. mu + M,
//   values printed with 17 significant digits so re-parsing is bit-exact (SPEC.md cli
//   "File round-trip ... bit-exactly").
//
//   Anomaly scores (SPEC.md cli cmd_anomaly): fitted curve from the coefficients on R_{0,M},
//   x~_n = (1/N)(a_0 + 2 Re sum_{m=1..M} a_m e^{2 pi i m n / N}) (conjugate symmetry of real
//   input), score_n = |x_n - x~_n|, top k by descending score, ties by ascending index.  The
//   reconstruction is the direct O(N M) evaluation SPEC's design decision names, with the
//   angle (m n) mod N reduced exactly.  The coefficients come from the GPU execute
//   (pft_anomaly) or from the caller (pft_anomaly_from_coeffs).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "api_guard.hpp"
#include "internal.hpp"

using namespace pft;
using namespace pft::detail;

namespace {

struct FileCloser {
    FILE* f;
    ~FileCloser() {
        if (f) std::fclose(f);
    }
};

std::string trim(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
    while (b > a && std::isspace(static_cast<unsigned char>(s[b - 1]))) --b;
    return s.substr(a, b - a);
}

double parse_double(const std::string& tok, const char* path, size_t line) {
    const std::string t = trim(tok);
    char* end = nullptr;
    errno = 0;
    const double v = std::strtod(t.c_str(), &end);
    if (t.empty() || end != t.c_str() + t.size())
        fail(PFT_ERR_IO, std::string(path) + ":" + std::to_string(line) + ": not a number: '" + t + "'");
    return v;
}

std::vector<std::string> split_commas(const std::string& s) {
    std::vector<std::string> out;
    size_t a = 0;
    while (true) {
        const size_t b = s.find(',', a);
        out.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
        if (b == std::string::npos) break;
        a = b + 1;
    }
    return out;
}

// Signal in memory: values + channel flag.
struct Signal {
    std::vector<cplx> v;
    bool complex = false;
};

Signal read_csv_signal(const char* path) {
    std::ifstream in(path);
    if (!in) fail(PFT_ERR_IO, std::string("cannot open ") + path);
    Signal s;
    std::string line;
    size_t ln = 0;
    int fields = 0;
    while (std::getline(in, line)) {
        ++ln;
        const std::string t = trim(line);
        if (t.empty()) continue;
        const auto f = split_commas(t);
        if (f.size() > 2) fail(PFT_ERR_IO, std::string(path) + ":" + std::to_string(ln) + ": expected 're' or 're,im'");
        if (fields == 0) fields = (int)f.size();
        if ((int)f.size() != fields)
            fail(PFT_ERR_IO, std::string(path) + ":" + std::to_string(ln) + ": mixed real and complex rows");
        const double re = parse_double(f[0], path, ln);
        const double im = f.size() == 2 ? parse_double(f[1], path, ln) : 0.0;
        s.v.emplace_back(re, im);
    }
    s.complex = fields == 2;
    return s;
}

Signal read_f64le_signal(const char* path) {
    FileCloser fc{std::fopen(path, "rb")};
    if (!fc.f) fail(PFT_ERR_IO, std::string("cannot open ") + path);
    unsigned char hdr[16];
    if (std::fread(hdr, 1, 16, fc.f) != 16) fail(PFT_ERR_IO, std::string(path) + ": truncated PFTS header");
    if (std::memcmp(hdr, "PFTS", 4) != 0) fail(PFT_ERR_IO, std::string(path) + ": bad magic (expected PFTS)");
    auto u32 = [&](int o) {
        return (uint32_t)hdr[o] | ((uint32_t)hdr[o + 1] << 8) | ((uint32_t)hdr[o + 2] << 16) | ((uint32_t)hdr[o + 3] << 24);
    };
    const uint32_t cflag = u32(4), n = u32(8);
    if (cflag > 1) fail(PFT_ERR_IO, std::string(path) + ": channel flag must be 0 or 1");
    Signal s;
    s.complex = cflag == 1;
    const size_t per = s.complex ? 2 : 1;
    std::vector<double> raw((size_t)n * per);
    if (!raw.empty() && std::fread(raw.data(), sizeof(double), raw.size(), fc.f) != raw.size())
        fail(PFT_ERR_IO, std::string(path) + ": truncated PFTS payload (header length " + std::to_string(n) + ")");
    unsigned char extra;
    if (std::fread(&extra, 1, 1, fc.f) == 1) fail(PFT_ERR_IO, std::string(path) + ": trailing bytes after PFTS payload");
    s.v.resize(n);
    for (size_t i = 0; i < n; ++i) s.v[i] = cplx(raw[i * per], s.complex ? raw[i * per + 1] : 0.0);
    return s;
}

// "%.17g" round-trips every finite double exactly through strtod
std::string fmt17(double x) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", x);
    return buf;
}

void write_signal(const char* path, int fmt, const pft_c128* v, uint64_t n, bool complex) {
    if (fmt == PFT_SIGNAL_CSV) {
        FileCloser fc{std::fopen(path, "w")};
        if (!fc.f) fail(PFT_ERR_IO, std::string("cannot write ") + path);
        for (uint64_t i = 0; i < n; ++i) {
            const std::string row = complex ? fmt17(v[i].re) + "," + fmt17(v[i].im) : fmt17(v[i].re);
            std::fputs(row.c_str(), fc.f);
            std::fputc('\n', fc.f);
        }
        if (std::ferror(fc.f)) fail(PFT_ERR_IO, std::string("write error on ") + path);
        return;
    }
    PFT_REQUIRE(fmt == PFT_SIGNAL_F64LE, "signal_write: unknown format");
    PFT_REQUIRE(n <= 0xffffffffull, "signal_write: PFTS length field is u32");
    FileCloser fc{std::fopen(path, "wb")};
    if (!fc.f) fail(PFT_ERR_IO, std::string("cannot write ") + path);
    unsigned char hdr[16] = {'P', 'F', 'T', 'S'};
    const uint32_t cflag = complex ? 1u : 0u, len = (uint32_t)n;
    for (int b = 0; b < 4; ++b) {
        hdr[4 + b] = (unsigned char)(cflag >> (8 * b));
        hdr[8 + b] = (unsigned char)(len >> (8 * b));
    }
    std::fwrite(hdr, 1, 16, fc.f);
    std::vector<double> raw;
    raw.reserve((size_t)n * (complex ? 2 : 1));
    for (uint64_t i = 0; i < n; ++i) {
        raw.push_back(v[i].re);
        if (complex) raw.push_back(v[i].im);
    }
    if (!raw.empty()) std::fwrite(raw.data(), sizeof(double), raw.size(), fc.f);  // host is little-endian (x86-64)
    if (std::ferror(fc.f)) fail(PFT_ERR_IO, std::string("write error on ") + path);
}

}  // namespace

extern "C" {

pft_status pft_signal_read(const char* path, int fmt, pft_c128* out, uint64_t cap, uint64_t* n, int* is_complex) {
    PFT_API_BEGIN
    PFT_REQUIRE(path && n, "signal_read: null argument");
    PFT_REQUIRE(fmt == PFT_SIGNAL_CSV || fmt == PFT_SIGNAL_F64LE, "signal_read: unknown format");
    const Signal s = fmt == PFT_SIGNAL_CSV ? read_csv_signal(path) : read_f64le_signal(path);
    *n = s.v.size();
    if (is_complex) *is_complex = s.complex ? 1 : 0;
    if (out) {
        if (cap < s.v.size()) fail(PFT_ERR_BUFFER_TOO_SMALL, "signal_read: output capacity below the signal length");
        if (!s.v.empty()) std::memcpy(static_cast<void*>(out), s.v.data(), s.v.size() * sizeof(cplx));
    }
    PFT_API_END
}

pft_status pft_signal_write(const char* path, int fmt, const pft_c128* v, uint64_t n, int is_complex) {
    PFT_API_BEGIN
    PFT_REQUIRE(path && (v || n == 0), "signal_write: null argument");
    write_signal(path, fmt, v, n, is_complex != 0);
    PFT_API_END
}

pft_status pft_spectrum_write_csv(const char* path, int64_t mu, uint64_t M, const pft_c128* values) {
    PFT_API_BEGIN
    PFT_REQUIRE(path && values, "spectrum_write_csv: null argument");
    FileCloser fc{std::fopen(path, "w")};
    if (!fc.f) fail(PFT_ERR_IO, std::string("cannot write ") + path);
    std::fputs("m,re,im\n", fc.f);
    const int64_t first = mu - (int64_t)M;
    for (uint64_t s = 0; s < 2 * M + 1; ++s) {
        const std::string row =
            std::to_string(first + (int64_t)s) + "," + fmt17(values[s].re) + "," + fmt17(values[s].im);
        std::fputs(row.c_str(), fc.f);
        std::fputc('\n', fc.f);
    }
    if (std::ferror(fc.f)) fail(PFT_ERR_IO, std::string("write error on ") + path);
    PFT_API_END
}

pft_status pft_spectrum_read_csv(const char* path, int64_t* first_m, pft_c128* out, uint64_t cap, uint64_t* n) {
    PFT_API_BEGIN
    PFT_REQUIRE(path && n, "spectrum_read_csv: null argument");
    std::ifstream in(path);
    if (!in) fail(PFT_ERR_IO, std::string("cannot open ") + path);
    std::string line;
    size_t ln = 0;
    std::vector<cplx> vals;
    int64_t m0 = 0, prev = 0;
    while (std::getline(in, line)) {
        ++ln;
        const std::string t = trim(line);
        if (t.empty() || (ln == 1 && t == "m,re,im")) continue;
        const auto f = split_commas(t);
        if (f.size() != 3) fail(PFT_ERR_IO, std::string(path) + ":" + std::to_string(ln) + ": expected 'm,re,im'");
        char* end = nullptr;
        const std::string ms = trim(f[0]);
        const long long m = std::strtoll(ms.c_str(), &end, 10);
        if (ms.empty() || end != ms.c_str() + ms.size())
            fail(PFT_ERR_IO, std::string(path) + ":" + std::to_string(ln) + ": bad index '" + ms + "'");
        if (vals.empty()) m0 = m;
        else if (m != prev + 1) fail(PFT_ERR_IO, std::string(path) + ":" + std::to_string(ln) + ": indices not consecutive");
        prev = m;
        vals.emplace_back(parse_double(f[1], path, ln), parse_double(f[2], path, ln));
    }
    *n = vals.size();
    if (first_m) *first_m = m0;
    if (out) {
        if (cap < vals.size()) fail(PFT_ERR_BUFFER_TOO_SMALL, "spectrum_read_csv: output capacity too small");
        if (!vals.empty()) std::memcpy(static_cast<void*>(out), vals.data(), vals.size() * sizeof(cplx));
    }
    PFT_API_END
}

pft_status pft_anomaly_from_coeffs(const double* x, uint64_t N, const pft_c128* coeffs, uint64_t M, uint64_t k,
                                   uint64_t* idx_out, double* score_out, double* fitted_out) {
    PFT_API_BEGIN
    PFT_REQUIRE(x && coeffs && idx_out && score_out, "anomaly: null argument");
    PFT_REQUIRE(N >= 1, "anomaly: N must be positive");
    PFT_REQUIRE(k >= 1 && k <= N, "anomaly: need 1 <= k <= N");
    PFT_REQUIRE(2 * M <= N, "anomaly: M > N/2");
    // coeffs[s] = a_{s - M}, s in [0, 2M]; a_0 = coeffs[M]
    std::vector<double> score(N), fit(N);
    // e^{2 pi i t / N} for every residue t, each evaluated once with the exact-angle rule
    // (SPEC.md:377); term (m, n) then reads t = (m n) mod N, stepped by n without a 128-bit
    // modulo -- the same values as evaluating cispi per term (N + N M work instead of N M
    // angle evaluations)
    std::vector<cplx> tab(N);
#pragma omp parallel for schedule(static)
    for (long long t = 0; t < (long long)N; ++t) tab[t] = cispi_frac(2 * (__int128)t, N);
#pragma omp parallel for schedule(static)
    for (long long n = 0; n < (long long)N; ++n) {
        double acc = coeffs[M].re;
        uint64_t red = 0;  // (m n) mod N
        for (uint64_t m = 1; m <= M; ++m) {
            red += (uint64_t)n;
            if (red >= N) red -= N;
            const cplx& e = tab[red];
            acc += 2.0 * (coeffs[M + m].re * e.real() - coeffs[M + m].im * e.imag());
        }
        fit[n] = acc / (double)N;
        score[n] = std::fabs(x[n] - fit[n]);
    }
    std::vector<uint64_t> order(N);
    std::iota(order.begin(), order.end(), 0);
    auto by_score = [&](uint64_t a, uint64_t b) { return score[a] != score[b] ? score[a] > score[b] : a < b; };
    std::partial_sort(order.begin(), order.begin() + (ptrdiff_t)k, order.end(), by_score);
    for (uint64_t i = 0; i < k; ++i) {
        idx_out[i] = order[i];
        score_out[i] = score[order[i]];
    }
    if (fitted_out) std::memcpy(fitted_out, fit.data(), N * sizeof(double));
    PFT_API_END
}

pft_status pft_anomaly(pft_dplan_t d, const double* x, uint64_t k, uint64_t* idx_out, double* score_out,
                       double* fitted_out) {
    PFT_API_BEGIN
    PFT_REQUIRE(d && x && idx_out && score_out, "anomaly: null argument");
    uint64_t N = 0, M = 0;
    int64_t mu = 0;
    pft_status st = pft_dplan_shape(d, &N, &M, &mu);
    if (st != PFT_OK) return st;
    PFT_REQUIRE(mu == 0, "anomaly: the device plan must target R_{0,M} (mu = 0)");
    std::vector<cplx> a(N), coeffs(2 * M + 1);
    for (uint64_t n = 0; n < N; ++n) a[n] = cplx(x[n], 0.0);
    st = pft_execute_host(d, reinterpret_cast<const pft_c128*>(a.data()), 1, reinterpret_cast<pft_c128*>(coeffs.data()),
                          nullptr, nullptr, nullptr);
    if (st != PFT_OK) return st;
    return pft_anomaly_from_coeffs(x, N, reinterpret_cast<const pft_c128*>(coeffs.data()), M, k, idx_out, score_out,
                                   fitted_out);
    PFT_API_END
}

}  // extern "C"
