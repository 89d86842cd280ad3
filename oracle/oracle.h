/* oracle.h -- C ABI of the CPU oracle (TEST INFRASTRUCTURE ONLY; see oracle.cpp). */
#ifndef PFT_ORACLE_H
#define PFT_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_c128 { double re, im; } oracle_c128;

typedef struct oracle_error_report {
    double relative_l2;
    double max_abs;
    double l1_input;
    double bound;
    int bound_satisfied;
} oracle_error_report;

int oracle_fft(size_t n, const oracle_c128* in, oracle_c128* out);
int oracle_ifft(size_t n, const oracle_c128* in, oracle_c128* out);
int oracle_batch_fft_columns(size_t p, size_t r, const oracle_c128* C, oracle_c128* Chat);
int oracle_matmul(size_t p, size_t q, size_t r, const oracle_c128* A, size_t row_stride, const oracle_c128* B,
                  oracle_c128* C);
int oracle_build_B(uint64_t N, uint64_t q, int r, int64_t mu, const oracle_c128* w, oracle_c128* B,
                   double* tvals_out);
int oracle_post(uint64_t p, uint64_t M, int64_t mu, int r, const oracle_c128* Chat, const double* post_powers,
                const oracle_c128* post_twiddles, oracle_c128* out);
int oracle_execute(uint64_t N, uint64_t M, int64_t mu, uint64_t p, int r, const oracle_c128* B,
                   const double* post_powers, const oracle_c128* post_twiddles, const oracle_c128* a,
                   oracle_c128* out);
int oracle_contract_slice(uint64_t p, uint64_t q, int r, uint64_t l0, uint64_t lq, const oracle_c128* B,
                          const oracle_c128* a, oracle_c128* Cpart);
int oracle_naive_dft(uint64_t N, const oracle_c128* a, int64_t mu, uint64_t M, oracle_c128* out);
double oracle_l1(const oracle_c128* a, uint64_t n);
int oracle_compare(const oracle_c128* actual, const oracle_c128* estimate, uint64_t n, double l1_input,
                   double epsilon, int two_d, oracle_error_report* rep);
double oracle_certify(const oracle_c128* w, int r, double xi, double u);

#ifdef __cplusplus
}
#endif
#endif
