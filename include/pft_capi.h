/* pft_capi.h -- C ABI of the B200-native Partial Fourier Transform (arXiv 2008.12559).
 *
 * The reference (/root/reference) defines the PFT as SPEC modules with a C++ type
 * header (proj/include/pft/types.hpp) and no compiled entry points.  Every function
 * below replaces one SPEC operation; the citation after each declaration names it.
 * The C++ API in <pft/pft.hpp> (namespace pft, SPEC names, exceptions) is a thin
 * header-only layer over these symbols, and INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - No C++ types and no exceptions cross this boundary; every call returns pft_status.
 *   - Complex numbers are pft_c128 = {re, im} doubles, layout-identical to
 *     std::complex<double> / cuDoubleComplex / numpy complex128.
 *   - Host planning objects (pft_table_t, pft_hplan_t) are immutable once built and
 *     may be shared across threads.
 *   - Device plans (pft_dplan_t) are read-only after creation.  pft_execute is
 *     asynchronous on the given cudaStream_t, does not allocate, is capturable in a
 *     CUDA graph, and is re-entrant on distinct (stream, workspace) pairs
 *     (SPEC.md:263-265).  There is no CPU fallback: device calls fail with
 *     PFT_ERR_NO_DEVICE / PFT_ERR_CUDA when no sm_100 device is usable.
 */
#ifndef PFT_CAPI_H
#define PFT_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFT_TABLE_VERSION 1u
#define PFT_MAX_TERMS 25 /* r <= 25, "typically 1 <= r <= 25" */

typedef struct pft_c128 { double re, im; } pft_c128;

typedef enum pft_status {
    PFT_OK = 0,
    PFT_ERR_INVALID_ARGUMENT = 1,     /* generic precondition failure                       */
    PFT_ERR_P_NOT_DIVISOR = 2,        /* build_plan: p does not divide N       */
    PFT_ERR_M_TOO_LARGE = 3,          /* build_plan: M > N/2               */
    PFT_ERR_EPSILON_NOT_IN_TABLE = 4, /* build_plan/min_terms: table missing eps*/
    PFT_ERR_RATIO_OUT_OF_RANGE = 5,   /* min_terms: M/p above every tabulated scope (:160)   */
    PFT_ERR_LENGTH_MISMATCH = 6,      /* execute: a.len != plan.N              */
    PFT_ERR_NON_FINITE = 7,           /* execute: non-finite input entries     */
    PFT_ERR_IO = 8,                   /* table file unreadable / corrupted      */
    PFT_ERR_VERSION_MISMATCH = 9,     /* table file version != 1             */
    PFT_ERR_NO_DEVICE = 10,           /* no usable CUDA device                               */
    PFT_ERR_CUDA = 11,                /* CUDA runtime error                                  */
    PFT_ERR_UNSUPPORTED = 12,         /* shape this build does not handle                    */
    PFT_ERR_INTERNAL = 13,
    PFT_ERR_BUFFER_TOO_SMALL = 14
} pft_status;

const char* pft_status_string(pft_status s);
/* Last detailed error message of the calling thread ("" if none). */
const char* pft_last_error(void);
/* Build identification: "pft-b200 <git/desc> sm_100a". */
const char* pft_version(void);

/* ------------------------------------------------------------------ minimax
 * SPEC.md:30-114.  Near-minimax polynomial P(x)=sum_j w_j x^j for e^{iux} on |x|<=xi:
 * Chebyshev (first-kind) interpolation, monomial expansion, certification on a grid
 * of 4096*r equispaced points plus 8r Chebyshev nodes.          */

/* best_approx(r, xi, u) -> coeffs[r], achieved_error */
pft_status pft_best_approx(int r, double xi, double u, pft_c128* coeffs, double* achieved_error);
/* scope_xi(eps, r) -> xi, coeffs[r], achieved */
pft_status pft_scope_xi(double epsilon, int r, double* xi, pft_c128* coeffs, double* achieved_error);
/* translate_poly(P, u, mu): Q(x) = e^{iu mu} P(x - mu) */
pft_status pft_translate_poly(const pft_c128* coeffs, int r, double u, double mu, pft_c128* out);

typedef struct pft_table_s* pft_table_t;

/* The table shipped with the library: eps in {1e-1..1e-13} x r in 1..25 (SPEC.md:103,
 * extended to BASELINE's eps=1e-12).  Owned by the library; do not destroy. */
pft_status pft_table_default(pft_table_t* out);
/* cmd_gen_table core: deterministic, byte-identical on regeneration. */
pft_status pft_table_generate(const double* epsilons, int n_eps, int r_max, pft_table_t* out);
/* save_table / load_table, PFTT v1 little-endian format. */
pft_status pft_table_save(pft_table_t t, const char* path);
pft_status pft_table_load(const char* path, pft_table_t* out);
pft_status pft_table_save_csv(pft_table_t t, const char* path);
void pft_table_destroy(pft_table_t t);
/* Entry access.  n_entries counts (eps, r) cells; entry i has r_i coefficients. */
pft_status pft_table_size(pft_table_t t, size_t* n_entries);
pft_status pft_table_entry(pft_table_t t, size_t i, double* eps, int* r, double* xi,
                           pft_c128* coeffs /* >= PFT_MAX_TERMS */, double* achieved_error);
pft_status pft_table_lookup(pft_table_t t, double eps, int r, double* xi, pft_c128* coeffs,
                            double* achieved_error);

/* ------------------------------------------------------------------ planner
 * SPEC.md:116-195, Algorithm 1.                                */

/* divisors(N) ascending; *count is set even when cap is too small. */
pft_status pft_divisors(uint64_t N, uint64_t* out, size_t cap, size_t* count);
/* min_terms(eps, M, p) */
pft_status pft_min_terms(pft_table_t t, double epsilon, uint64_t M, uint64_t p, int* r);
/* select_divisor(N, M, table, eps): argmin_p r(N + p log2 max(p,2) + M), ties -> smaller p
 *                                                                   */
pft_status pft_select_divisor(pft_table_t t, uint64_t N, uint64_t M, double epsilon,
                              uint64_t* p, int* r, double* cost);
/* Device-aware choice of p for the B200 path (not in the reference):
 * argmin_p of a calibrated HBM / FP64 / row-length / tail time model, n_sms = SM count (148).
 * est_us = modelled microseconds per transform.  Pass the result to pft_plan_build.       */
pft_status pft_select_divisor_device(pft_table_t t, uint64_t N, uint64_t M, double epsilon, int n_sms,
                                     uint64_t* p, int* r, double* est_us);
/* Measured choice: times the n_candidates best modelled p on `device` with the caller's input
 * d_in (batch x N complex128 on that device, signals contiguous); returns the fastest p and its
 * microseconds per execute of the batch.                                                  */
pft_status pft_autotune_divisor(pft_table_t t, uint64_t N, uint64_t M, int64_t mu, double epsilon, int device,
                                const pft_c128* d_in, size_t batch, int n_candidates, uint64_t* p, double* us);

typedef struct pft_hplan_s* pft_hplan_t;

typedef struct pft_plan_info {
    uint64_t N, M;
    int64_t mu;
    uint64_t p, q;
    int32_t r;
    int32_t reserved;
    double epsilon;
    double achieved_epsilon;
    double xi;
    double estimated_cost; /* SPEC cost model value for this (p, r) */
    uint64_t plan_id;
} pft_plan_info;

/* build_plan(N, M, mu, p (0 = auto via select_divisor), eps, table) */
pft_status pft_plan_build(pft_table_t t, uint64_t N, uint64_t M, int64_t mu, uint64_t p,
                          double epsilon, pft_hplan_t* out);
void pft_plan_destroy(pft_hplan_t plan);
pft_status pft_plan_info_get(pft_hplan_t plan, pft_plan_info* info);
/* Plan tables (host copies).  B: q*r row-major; w: r; phase: q (e^{-2 pi i mu (l-q/2)/N});
 * tvals: q (1-2l/q); post_powers: (2M+1)*r row-major by slot; post_twiddles: 2M+1. */
pft_status pft_plan_copy_B(pft_hplan_t plan, pft_c128* out);
pft_status pft_plan_copy_w(pft_hplan_t plan, pft_c128* out);
pft_status pft_plan_copy_phase(pft_hplan_t plan, pft_c128* out);
pft_status pft_plan_copy_tvals(pft_hplan_t plan, double* out);
pft_status pft_plan_copy_post_powers(pft_hplan_t plan, double* out);
pft_status pft_plan_copy_post_twiddles(pft_hplan_t plan, pft_c128* out);
/* Plan summary JSON into buf; *needed includes the terminating NUL. */
pft_status pft_plan_json(pft_hplan_t plan, char* buf, size_t cap, size_t* needed);

/* ------------------------------------------------------------------ device (sm_100a)
 * transform.execute (Algorithm 2) as two kernels:
 *   K1  contraction C = A x B fused with the first (row-residue) pass of the r length-p
 *       FFTs, one CTA per residue class k = c (mod P2);
 *   K2  remaining FFT pass, pruned to the 2M+1 needed bins, fused with the Eq. (7)
 *       post-process.
 * See DESIGN.md for the data layout.                                                */

typedef struct pft_dplan_s* pft_dplan_t;

/* Second pass (the length-P2 FFT over the residue classes, pruned to the 2M+1 bins, fused with
 * the Eq. (7) post-process).  AUTO picks by the shape. */
#define PFT_PASS2_AUTO 0
#define PFT_PASS2_SUM_TAIL 1   /* inside K1: residue rows summed by K1's last arrivals (few bins) */
#define PFT_PASS2_K2_FFT 2     /* K2: length-P2 Stockham FFT in shared memory                  */
#define PFT_PASS2_K2_DOT 3     /* K2: direct dot over P2 from shared memory (few bins per m1)  */
#define PFT_PASS2_K2_DIRECT 4  /* K2: direct sum over P2 from global memory (any P2)           */
#define PFT_PASS2_K2_L2 5      /* K2: one warp per bin over the L2-resident slab, no smem       */
#define PFT_PASS2_K2_BLUESTEIN 6 /* K2: chirp-z length-P2 DFT via two power-of-two FFTs of L >=
                                    2 P2 - 1 (any P2 <= 2048, prime factors > 64 included)       */
/* Where the K2 work of the PFT_PASS2_K2_FFT form runs. */
#define PFT_K2_AT_AUTO 0
#define PFT_K2_AT_GRID 1       /* a separate K2 launch after K1                                 */
#define PFT_K2_AT_TAIL 2       /* by K1's last-arriving CTAs (r = 4..7)                         */
#define PFT_K2_AT_FUSED 3      /* in K1 behind a grid-wide barrier (cooperative launch)         */

typedef struct pft_dplan_opts {
    int device;          /* CUDA ordinal                                                      */
    uint64_t p2;         /* residue classes for K1 (0 = auto); must divide p                  */
    int k1_stages;       /* K1 TMA ring depth, 3..8 (0 = deepest that keeps 2 CTAs/SM)         */
    int second_pass;     /* PFT_PASS2_*                                                        */
    int k2_at;           /* PFT_K2_AT_*                                                        */
    int tail_ctas;       /* sum-tail reducers / K2-tail workers per signal (0 = plan); always
                            capped below the co-resident K1 capacity (forward progress)       */
    int k2_grid_ctas;    /* K2 grid width: the PFT_PASS2_K2_L2 form (0 = SM count); the
                            PFT_PASS2_K2_FFT form on its own grid with a power-of-two P2: > 0 =
                            the bulk-copy ring kernel on that many CTAs looping over m1
                            (0 = the plan's choice: one CTA per m1, or for chained executes K2
                            worker CTAs inside K1's grid, see pft_dplan_tail_kind)            */
    int k1_split;        /* 0: an isolated execute (no PFT_EXEC_OVERLAP_PREVIOUS) whose K1 grid
                            fills at most half of the SM slots runs two CTAs (a thread-block
                            cluster) per residue class, each streaming half of the columns and
                            summing their C slabs over distributed shared memory; 1: never    */
    int reserved;        /* must be 0                                                          */
    uint64_t batch_hint; /* typical batch per execute (0/1 = single signal): sizes the K1 grid */
} pft_dplan_opts;

/* Upload a host plan to the device.  opts may be NULL (defaults). */
pft_status pft_dplan_create(pft_hplan_t plan, const pft_dplan_opts* opts, pft_dplan_t* out);
void pft_dplan_destroy(pft_dplan_t d);
/* Chosen decomposition p = P1 * P2 (P1 = local FFT length per residue class). */
pft_status pft_dplan_layout(pft_dplan_t d, uint64_t* p1, uint64_t* p2);
/* Device workspace bytes for up to `batch` independent transforms per call.  Zero it once
 * before first use; every execute leaves it re-armed.  Layout: a 256-byte header (grid-barrier
 * words, the non-finite status word) then one block per signal (control words, data), so a
 * workspace sized for batch B serves every call with batch <= B. */
pft_status pft_workspace_bytes(pft_dplan_t d, size_t batch, size_t* bytes);
/* Bytes of one partial slab (the reducible intermediate, p*r complex128 per transform). */
pft_status pft_partial_bytes(pft_dplan_t d, size_t batch, size_t* bytes);

/* execute flags */
#define PFT_EXEC_DEFAULT 0u
/* Programmatic dependent launch (PDL): K1 may start streaming its input while the preceding
 * kernel on `stream` is still finishing -- the throughput mode for a stream of independent
 * transforms (execute i+1 streams while execute i reduces its last bins).  The caller
 * guarantees that d_in is NOT written by the preceding kernel on the stream (for example the
 * previous execute's d_out, or a kernel that triggers its dependents early, such as a PDL-enabled
 * GEMM).  Executes that share a workspace must still complete in order: the preceding kernel on
 * the stream has to be one that completes only after ITS predecessor completed -- another execute
 * of this library (every K1 waits for its predecessor before it writes its workspace) or any
 * kernel launched without programmatic stream serialization.  Without the flag K1 starts only
 * after the preceding work on the stream completed. */
#define PFT_EXEC_OVERLAP_PREVIOUS 1u

/* execute: d_in holds `batch` signals of N complex128, signal b at d_in + b*in_stride;
 * d_out receives batch x (2M+1) values, signal b at d_out + b*(2M+1).
 * d_ws: pft_workspace_bytes(>= batch) bytes of device memory, or NULL to use the plan's
 * own batch-1 workspace (then calls on the plan must be serialised).  stream: cudaStream_t.
 * Asynchronous, allocation-free, graph-capturable.  Non-finite input sets bit 0 of the
 * workspace's status word (pft_workspace_status / pft_status_query). */
pft_status pft_execute(pft_dplan_t d, const pft_c128* d_in, size_t batch, size_t in_stride,
                       pft_c128* d_out, void* d_ws, void* stream);
pft_status pft_execute_ex(pft_dplan_t d, const pft_c128* d_in, size_t batch, size_t in_stride,
                          pft_c128* d_out, void* d_ws, void* stream, unsigned flags);

/* Sharded single transform (contraction-axis split, BASELINE.json configs[4]).
 * Columns of A are owned in mirror pairs (l, q-l), l in [1, ceil(q/2)), split contiguously
 * over ranks; the unpaired columns l = 0 and (even q) l = q/2 belong to rank 0.  Each rank's
 * local buffer holds p rows of `row_stride` elements laid out as pft_shard_layout says.
 * execute_partial contracts the local slice and applies K1's FFT pass, writing a reducible
 * partial slab of pft_partial_bytes (the sum over ranks == the unsharded slab, e.g. via
 * ncclReduce/ncclAllReduce with ncclDouble/ncclSum); finalize turns the reduced slab into
 * the 2M+1 outputs.  world == 1 is the natural (unsharded) layout.  pft_execute_sharded
 * below does all three steps with the NCCL reduce inside the library. */
typedef struct pft_shard_info {
    uint64_t pair_begin, pair_end; /* global pair indices [pair_begin, pair_end)            */
    uint64_t row_len;              /* local columns per row                                 */
    int64_t front_col;             /* local column of l = pair_begin (l ascending)          */
    int64_t mirror_col;            /* local column of q - pair_begin (descending with l)    */
    int64_t single0_col;           /* local column of l = 0, or -1                          */
    int64_t singleh_col;           /* local column of l = q/2 (even q), or -1               */
} pft_shard_info;

pft_status pft_shard_layout(uint64_t q, int world, int rank, pft_shard_info* info);
/* Host helper: scatter the global signal a (p rows of q) into rank's local layout. */
pft_status pft_shard_gather_host(uint64_t p, uint64_t q, int world, int rank, const pft_c128* a,
                                 pft_c128* local, uint64_t row_stride);
pft_status pft_execute_partial(pft_dplan_t d, const pft_c128* d_in_local, int world, int rank,
                               uint64_t row_stride, pft_c128* d_partial, void* stream);
pft_status pft_finalize(pft_dplan_t d, const pft_c128* d_partial, size_t batch, pft_c128* d_out,
                        void* stream);

/* The sharded transform with its collective inside the library (SURVEY.md §8(b),(e)): on
 * every rank of `comm`, K1 on the local slice (pft_execute_partial) -> ncclReduce(sum, ncclDouble)
 * of the partial slab onto `root` over NVLink/NVSwitch -> on the root, K2 (pft_finalize) into
 * d_out.  One asynchronous call per rank on `stream` (graph-capturable).  d_slab:
 * pft_partial_bytes(d, 1) bytes on every rank (reduced in place); d_out (2M+1 values) is only
 * written on the root (may be NULL elsewhere).  The device plan must live on the
 * communicator's device.  World size and rank are the communicator's.  NCCL is loaded at run
 * time (libnccl.so.2; the copy already in the process when there is one), so `comm` may come
 * from the caller's own NCCL or from pft_nccl_comm_init.                                       */
struct ncclComm; /* NCCL's communicator: ncclComm_t == struct ncclComm* */
#define PFT_NCCL_UNIQUE_ID_BYTES 128
pft_status pft_nccl_available(int* available);
pft_status pft_nccl_get_unique_id(unsigned char* id /* [PFT_NCCL_UNIQUE_ID_BYTES] */);
pft_status pft_nccl_comm_init(int world, int rank, const unsigned char* id, int device, struct ncclComm** comm);
pft_status pft_nccl_comm_destroy(struct ncclComm* comm);
pft_status pft_execute_sharded(pft_dplan_t d, const pft_c128* d_in_local, uint64_t row_stride,
                               struct ncclComm* comm, int root, pft_c128* d_slab, pft_c128* d_out,
                               void* stream);
/* Device-aware p for the sharded transform over `world` GPUs: the single-GPU time model on the
 * per-rank slice (q/world columns per row) plus the collective (reduce of the 16 p r-byte slab:
 * latency + bytes over NVLink) and the root's K2 -- large p shrinks the contraction's row
 * overhead but grows the slab every rank must reduce. */
pft_status pft_select_divisor_sharded(pft_table_t t, uint64_t N, uint64_t M, double epsilon, int n_sms,
                                      int world, uint64_t* p, int* r, double* est_us);
/* CUDA ordinal a device plan lives on. */
pft_status pft_dplan_device(pft_dplan_t d, int* device);

/* Status word of a workspace (bit 0 = non-finite output, i.e. non-finite input, since the last
 * reset; bit 1 = a device-side wait of the K2 worker / ring forms ran into its bound -- an
 * internal error, the outputs of that execute are invalid).  Synchronises `stream`.  pft_status_query reads the plan's own workspace (executes
 * with d_ws == NULL, and pft_finalize). */
pft_status pft_workspace_status(pft_dplan_t d, void* d_ws, void* stream, int* flags, int reset);
pft_status pft_status_query(pft_dplan_t d, void* stream, int* flags, int reset);

/* End-to-end convenience used by the C++ API and the e2e benchmark: copies h_in
 * (pinned or pageable) H2D, executes, copies the result D2H, synchronises and maps
 * a non-finite flag to PFT_ERR_NON_FINITE.  d_in/d_out are device staging buffers of
 * batch*N and batch*(2M+1) elements, or NULL: then staging comes from the plan's pool
 * (allocated on first use, reused, one set per concurrent caller).  Thread-safe: concurrent
 * calls on one plan use distinct workspaces and status words.  stream NULL = the staging
 * set's own stream. */
pft_status pft_execute_host(pft_dplan_t d, const pft_c128* h_in, size_t batch, pft_c128* h_out,
                            pft_c128* d_in, pft_c128* d_out, void* stream);

/* ---- 2-D PFT (Algorithms 3-4).  `rows`: device plan of axis 2 (length N2,
 * applied to each of the N1 rows of the row-major N1 x N2 input); `cols`: device plan of axis 1
 * (length N1).  Output: (2M1+1) x (2M2+1) row-major, out[m1 - mu1 + M1][m2 - mu2 + M2].
 * Executed as the two batched 1-D passes the block contraction B1^T A B2 factors into.  The
 * workspace (pft_workspace_bytes_2d) is required; zero it once.                             */
pft_status pft_workspace_bytes_2d(pft_dplan_t rows, pft_dplan_t cols, size_t* bytes);
pft_status pft_execute_2d(pft_dplan_t rows, pft_dplan_t cols, const pft_c128* d_in, pft_c128* d_out,
                          void* d_ws, void* stream);
/* host convenience: H2D, execute_2d, D2H, synchronous; PFT_ERR_NON_FINITE on non-finite input */
pft_status pft_execute_2d_host(pft_dplan_t rows, pft_dplan_t cols, const pft_c128* h_in, pft_c128* h_out);

/* ------------------------------------------------------------------ synthetic inputs
 * Seeded counter-based generators (BASELINE.json configs), identical bit-for-bit on
 * host and device for the uniform kind.  kind: 0 = uniform[-1,1] re/im,
 * 1 = complex normal CN(0,1) (re,im ~ N(0,1/2)), 2 = sparse spectrum (n_tones tones at
 * integer frequencies freqs[] with amplitudes amps[] plus CN(0, sigma^2) noise). */
typedef struct pft_signal_desc {
    int kind;
    uint64_t seed;
    uint64_t N;
    uint64_t index_offset; /* global element index of element 0 (batched signals)  */
    int n_tones;
    const int64_t* freqs;  /* host pointer, n_tones                                  */
    const pft_c128* amps;  /* host pointer, n_tones                                  */
    double sigma;
} pft_signal_desc;

pft_status pft_generate_host(const pft_signal_desc* desc, pft_c128* out, uint64_t count);
pft_status pft_generate_device(const pft_signal_desc* desc, pft_c128* d_out, uint64_t count,
                               void* stream);
/* The tone set of BASELINE configs[1]: n distinct integer frequencies uniform in
 * [lo, hi] and CN(0,1) amplitudes, drawn from `seed`. */
pft_status pft_sparse_tones(uint64_t seed, int n, int64_t lo, int64_t hi, int64_t* freqs,
                            pft_c128* amps);

/* ------------------------------------------------------------------ device introspection */
/* Number of kernel launches one pft_execute issues (for launch accounting). */
pft_status pft_launches_per_execute(pft_dplan_t d, int* launches);
/* How an unsharded execute finishes after the contraction + first FFT pass (K1):
 * 0 separate K2 grid, 1 sum tail in K1 (few bins), 2 K2 work by K1's last arrivals (many
 * bins), 3 K2 in K1 behind a grid barrier (opt-in), 4 K2 worker CTAs riding in K1's grid when
 * the execute overlaps its predecessor (PFT_EXEC_OVERLAP_PREVIOUS), a separate K2 grid otherwise. */
pft_status pft_dplan_tail_kind(pft_dplan_t d, int* kind);
/* Signals one K1 CTA holds when `batch` contiguous signals (in_stride == N) are executed: short
 * batched signals with one residue class each (the 2-D passes) are contracted several per CTA as
 * one row block (1 = one signal per CTA).  For launch accounting and tests. */
pft_status pft_dplan_signals_per_cta(pft_dplan_t d, size_t batch, int* signals);
/* The second-pass form a device plan runs (PFT_PASS2_*, never _AUTO). */
pft_status pft_dplan_second_pass(pft_dplan_t d, int* form);

/* ------------------------------------------------------------------ data formats and callers
 * The formats either side of execute and the pipeline that calls it (
 * SPEC.md cli module: SignalFile, cmd_transform output, cmd_anomaly, §4.4).      */
#define PFT_SIGNAL_CSV 0   /* rows "re" or "re,im"                                             */
#define PFT_SIGNAL_F64LE 1 /* header {"PFTS", u32 complex flag, u32 length} + LE doubles        */
/* SignalFile read: *n = length (always set); values copied to out when out != NULL (cap >= n,
 * else PFT_ERR_BUFFER_TOO_SMALL); *is_complex = channel flag.  Parse errors: PFT_ERR_IO.    */
pft_status pft_signal_read(const char* path, int fmt, pft_c128* out, uint64_t cap, uint64_t* n, int* is_complex);
pft_status pft_signal_write(const char* path, int fmt, const pft_c128* v, uint64_t n, int is_complex);
/* cmd_transform output: CSV "m,re,im", m = mu - M .. mu + M, 17 significant digits (re-parsing
 * is bit-exact, SPEC.md cli "File round-trip").                                             */
pft_status pft_spectrum_write_csv(const char* path, int64_t mu, uint64_t M, const pft_c128* values);
pft_status pft_spectrum_read_csv(const char* path, int64_t* first_m, pft_c128* out, uint64_t cap, uint64_t* n);
/* cmd_anomaly core: fitted curve from coeffs[s] = a_{s-M} on R_{0,M} (conjugate symmetry of
 * real x), scores |x_n - fit_n|, top k by descending score, ties by ascending index.  fitted
 * (N doubles) may be NULL.                                                                  */
pft_status pft_anomaly_from_coeffs(const double* x, uint64_t N, const pft_c128* coeffs, uint64_t M, uint64_t k,
                                   uint64_t* idx, double* score, double* fitted);
/* cmd_anomaly with source = pft: the coefficients from one execute of a device plan built for
 * (N, M, mu = 0) on the real series x (host memory, N doubles), then the scoring above.      */
pft_status pft_anomaly(pft_dplan_t d, const double* x, uint64_t k, uint64_t* idx, double* score, double* fitted);
/* (N, M, mu) of a device plan. */
pft_status pft_dplan_shape(pft_dplan_t d, uint64_t* N, uint64_t* M, int64_t* mu);

/* ------------------------------------------------------------------ verification (SPEC.md oracle module)
 * naive_dft on the GPU: out[s] = sum_n a[n] e^{-2 pi i (first_m + s) n / N}, s in [count), every angle
 * reduced exactly in integers ((m n) mod N) before one sincospi per term.
 * O(N count); used by the CLI's --verify, the anomaly pipeline's "fft" source and bench's naive
 * column -- desk-scale ground truth on the device, not a CPU path. */
pft_status pft_naive_dft_device(const pft_c128* d_in, uint64_t N, int64_t first_m, uint64_t count, pft_c128* d_out,
                                void* stream);
pft_status pft_naive_dft_host(const pft_c128* h_in, uint64_t N, int64_t first_m, uint64_t count, pft_c128* h_out);
/* compare(actual, estimate, l1_input, epsilon, two_d_bound) -> ErrorReport: relative_l2 =
 * ||estimate - actual|| / ||actual|| (0 if both are zero, +inf if only actual is), max_abs, bound =
 * l1_input * eps (1-D, Theorem 2) or l1_input * (eps^2 + 2 eps) (2-D, Theorem 4). */
typedef struct pft_error_report {
    double relative_l2, max_abs, l1_input, bound;
    int bound_satisfied;
} pft_error_report;
pft_status pft_compare(const pft_c128* actual, const pft_c128* estimate, uint64_t n, double l1_input, double epsilon,
                       int two_d_bound, pft_error_report* report);
/* sum |a_i| (types.hpp:92-96) */
pft_status pft_l1_norm(const pft_c128* a, uint64_t n, double* l1);

pft_status pft_device_count(int* n);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* PFT_CAPI_H */
