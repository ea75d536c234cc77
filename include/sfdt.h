/*
 * sfdt.h -- C ABI of the B200-native sFFT-DT hot path (libsfdt_b200.so).
 *
 * Drop-in boundary for the reference package `sfft-dt`
 * (/root/reference/pkg/src/sfft_dt).  Two layers:
 *
 *  1. Kernel-level mirrors of the reference's backend seam
 *     (_kernels/__init__.py:19-24), batched on the device:
 *       sfdt_fft_radix2            <- _core.pyx:35-77    fft_radix2
 *       sfdt_hankel_solve          <- _core.pyx:127-162  hankel_solve
 *       sfdt_poly_roots            <- _core.pyx:238-266  poly_roots
 *       sfdt_vandermonde_solve     <- _core.pyx:273-312  vandermonde_solve
 *       sfdt_prune_eval            <- _core.pyx:319-346  prune_eval
 *       sfdt_hankel_singular_values<- _core.pyx:409-433  hankel_singular_values
 *  2. Solver-level entry points (one call per batch of signals) behind the
 *     reference's public solvers:
 *       sfdt_exact_solve   <- exact.py:161-200 solve_noniterative
 *                             exact.py:203-292 solve_iterative
 *       sfdt_general_solve <- general.py:272-372 solve_general
 *
 * Conventions
 *  - Complex numbers are interleaved (re, im) doubles (complex128); signals
 *    may also be complex64 storage (SFDT_C64), upconverted to FP64 at load.
 *  - Every pointer argument except the host twiddle buffer is a DEVICE
 *    pointer.  The library never allocates: callers pass workspaces sized by
 *    the *_workspace_bytes queries.  Work is asynchronous on `stream`.
 *  - Return 0 on success, a negative SFDT_E* code otherwise (argument
 *    errors mirror the reference's ValueErrors; numerical singularity is data,
 *    never an error, as in the reference).
 *  - Reentrant for distinct workspaces; no global mutable state (no
 *    environment reads, no library-owned streams: A/B switches arrive in an
 *    sfdt_tuning, a second stream in the args).
 */
#ifndef SFDT_H
#define SFDT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *sfdt_stream_t; /* a cudaStream_t */

enum {
    SFDT_OK = 0,
    SFDT_EINVAL = -1,     /* bad argument (reference: ValueError) */
    SFDT_ECUDA = -2,      /* CUDA launch / runtime failure */
    SFDT_EWORKSPACE = -3, /* workspace too small */
    SFDT_ECAPACITY = -4   /* output capacity too small */
};

enum { SFDT_C128 = 0, SFDT_C64 = 1 };

/* per-signal statistics block of sfdt_exact_solve (int64 each) */
enum {
    SFDT_ST_NITER = 0,        /* iterations recorded (1 non-iterative, a_max iterative) */
    SFDT_ST_FULL_SUCCESS = 1, /* trace.full_success */
    SFDT_ST_NENTRIES = 2,     /* entries written (duplicates counted once) */
    SFDT_ST_NUNRESOLVED = 3,  /* len(trace.unresolved_bins) */
    SFDT_ST_NDUP = 4,         /* duplicate-location overwrites (trace.warnings) */
    SFDT_ST_SYNDROMES = 5,    /* trace.syndromes_computed */
    SFDT_ST_FFT_SAMPLES = 6,  /* trace.fft_samples */
    SFDT_ST_ITER0 = 8,        /* per iteration: d, attempted, solved, deferred,
                                 syndromes, fft_samples (6 each, up to 4) */
    SFDT_ST_PER_SIGNAL = 32
};

const char *sfdt_strerror(int code);
const char *sfdt_last_cuda_error(void); /* cudaGetErrorString of the sticky/last CUDA error */
int sfdt_version(void);

/* Host helper: the twiddle table the reference's radix-2 recurrence produces
 * (_core.pyx:61-76: w *= wlen per butterfly, re-seeded by cexp every 256).
 * Stage m (2 <= m <= n_max) occupies entries [m/2 - 1, m - 1); n_max - 1
 * complex entries in total.  host_out holds 2*(n_max-1) doubles. */
int sfdt_fft_twiddles(int64_t n_max, int inverse, double *host_out);

/* ---------------------------------------------------------- kernel level */
int sfdt_fft_radix2(const double *x, double *out, int64_t batch, int64_t n, int inverse,
                    const double *twiddles, sfdt_stream_t stream);
int sfdt_hankel_solve(const double *m, int64_t nb, int64_t ld, int a, double *c, double *cd,
                      sfdt_stream_t stream);
int sfdt_poly_roots(const double *c, int64_t nb, int a, double *z, sfdt_stream_t stream);
int sfdt_vandermonde_solve(const double *z, const double *m, int64_t nb, int a, int64_t ld,
                           double *p, double *pd, sfdt_stream_t stream);
int sfdt_prune_eval(const double *c, const int64_t *k, int64_t nb, int a, int64_t n, int64_t d,
                    double *out, sfdt_stream_t stream);
int sfdt_hankel_singular_values(const double *m, int64_t nb, int64_t ld, int a_max, double *out,
                                sfdt_stream_t stream);

/* A/B switches of measured design decisions (experiment scripts and tests
 * select the alternatives); NULL = the measured-best defaults of
 * sfdt_default_tuning.  Only the solve that receives the struct reads it:
 * the library keeps no global state. */
typedef struct {
    int32_t fft_split;       /* bit 0 -- large views L = 2^17..2^19: 0 register-blocked pass A + one pass B,
                                1 the stage-split register passes (round-1 plan); bit 1 -- 4096-point
                                views: 0 the register-blocked radix-16 kernel, 2 k_fft_views (radix-8
                                shared-memory passes) */
    int32_t gen_dedup;       /* 1: a random shift equal to a consecutive one shares that view */
    int32_t gen_svd_closed;  /* 1: closed-form 3x3 singular values where accurate, Jacobi for the
                                rest; 0: Jacobi for every bin */
    int32_t gen_mf_small;    /* 1: lane groups per bin in the matched filter when d <= 32 */
    int32_t gen_mf_list;     /* matched-filter bins per CTA: 0 auto, else 32..4096 */
    int32_t gen_warp;        /* all-column pursuit: -1 auto, 0 thread per bin, 1 warp per bin */
    int32_t gen_split_a;     /* heavy bins with a >= gen_split_a dealt first (0: list order) */
    int32_t gen_prune_lanes; /* lanes per pruned bin: 0 auto, 1 or 4 */
    int32_t gen_deal;        /* heavy bins dealt lane-major while <= gen_deal per warp (0: take counter) */
    int32_t decode_coop;     /* non-iterative multi-collision decode: 0 one thread per bin for every a;
                                1 eight lanes per bin, the a = 2 and a = 3 trials side by side in two
                                warps (a = 4 afterwards where needed); 2 thread per bin for a = 2,
                                cooperative for a = 3 then 4; 3 cooperative, every a side by side;
                                -1 auto (1 for small batches, else 2) */
    int32_t latency_path;    /* non-iterative solves of <= 8 short signals (L <= 8192, n <= 2^20): -1 the
                                fused five-kernel chain; 0 the general ten-kernel chain; 1 the fused chain
                                for up to 64 signals */
    int32_t gen_window;      /* general path, 4096-point views: -1 auto (16 for host-mapped signals, else 0;
                                -2 / -3: auto with / without the 64-B fetch hint, -4: auto without the ring
                                (host-mapped 4096-point views take the gather kernel too) -- for A/B runs;
                                host-mapped signals of other view lengths: a window gather kernel into a
                                device buffer, then the ordinary view FFT);
                                0 each view's CTA gathers its own samples;
                                n > 0 window ring -- every CTA first gathers a piece of the d-block rows
                                (all views of a d-block in one warp instruction) of the signal n ahead,
                                then transforms its view from the ring of 2n signals (k_fft_win16) */
} sfdt_tuning;

void sfdt_default_tuning(sfdt_tuning *out);

/* ---------------------------------------------------------- exact solver */
typedef struct {
    /* input: batch x n signals, row-major, complex128 or complex64 */
    const void *x;
    int32_t x_dtype;
    int64_t batch;
    int64_t n;
    /* ExactConfig (exact.py:31-71): resolved initial d, a_max, zero_threshold */
    int64_t d;
    int32_t a_max;
    int32_t iterative; /* 0: solve_noniterative, 1: solve_iterative */
    double zero_threshold;
    const double *twiddles; /* device copy of sfdt_fft_twiddles(n_max >= n/d, inverse=0) */
    /* outputs (device) */
    int64_t *entry_offsets; /* batch + 1 : entries of signal b are [off[b], off[b+1]) */
    int64_t *locs;          /* entry_cap */
    double *vals;           /* 2 * entry_cap */
    int64_t entry_cap;
    int64_t *unres_offsets; /* batch + 1 */
    int32_t *unres_bins;    /* unres_cap, ascending per signal */
    int64_t unres_cap;
    int64_t *dup_locs;      /* optional (iterative): duplicate locations in write order */
    int64_t *dup_offsets;   /* batch + 1 */
    int64_t dup_cap;
    int64_t *stats;         /* batch * SFDT_ST_PER_SIGNAL */
    double *rms;            /* batch: rms(x) (spectral.py:215-218) */
    /* optional pipelining: with a second stream, the HBM stream kernel of
     * signal chunk c+1 (this stream) overlaps the FFT + decode of chunk c
     * (aux_stream).  chunk_signals <= 0 picks ~16 chunks. */
    void *aux_stream;
    int64_t chunk_signals;
    /* optional: rms(x) per signal already known (device, batch doubles) --
     * e.g. from an earlier stage of estimate_sparsity_and_solve; the HBM
     * stream pass is skipped and `rms` receives a copy */
    const double *rms_in;
    /* optional instrumentation (host side) */
    void *ev_stream_begin;  /* cudaEvent_t recorded right before / after the */
    void *ev_stream_end;    /* HBM stream kernel (roofline timing), or NULL  */
    const sfdt_tuning *tuning; /* optional A/B switches (NULL: defaults) */
    int32_t kernel_launches; /* out: kernels launched by the last solve */
} sfdt_exact_args;

/* capacities that can never overflow for these arguments */
int sfdt_exact_caps(const sfdt_exact_args *args, int64_t *entry_cap, int64_t *unres_cap,
                    int64_t *dup_cap);
size_t sfdt_exact_workspace_bytes(const sfdt_exact_args *args);
int sfdt_exact_solve(sfdt_exact_args *args, void *workspace, size_t workspace_bytes,
                     sfdt_stream_t stream);

/* -------------------------------------------------------- general solver */
/* per-signal statistics of sfdt_general_solve (int64 each) */
enum {
    SFDT_GS_NENTRIES = 0,  /* entries written */
    SFDT_GS_HIST0 = 1,     /* collision_histogram[a], a = 0..4 (5 slots) */
    SFDT_GS_NVOTED = 6,    /* bins with votes >= 1 */
    SFDT_GS_RANKDEF = 7,   /* rank-deficient least-squares calls (logged) */
    SFDT_GS_CLASS0 = 8,    /* entries per vote class a = 1..4 (4 slots) */
    SFDT_GS_PER_SIGNAL = 16
};

typedef struct {
    /* input: batch x n signals (complex128 or complex64 storage) */
    const void *x;
    int32_t x_dtype;
    int64_t batch;
    int64_t n;
    /* GeneralConfig (general.py:28-70), resolved */
    int64_t k;
    int64_t d;
    int32_t a_max;
    int32_t r_eff;            /* min(3*a_max, d) */
    int32_t keep_per_collision;
    int32_t prune;
    double zero_vote_rtol;
    /* draw_shifts (general.py:101-106), drawn on the host (numpy Generator):
     * shifts[b*shift_stride + j], j < r_eff (device, int64); shift_stride 0 =
     * one draw for the whole batch */
    const int64_t *shifts;
    int64_t shift_stride;
    /* base_phi[b*phi_stride + j*d + t] = exp(2 pi i shifts_j t / d)
     * (general.py:309), complex128 on the device, built by the host exactly
     * as numpy builds it */
    const double *base_phi;
    int64_t phi_stride;
    const double *twiddles;  /* sfdt_fft_twiddles(n_max >= n/d) on the device */
    /* outputs (device) */
    int64_t *entry_offsets;  /* batch + 1 */
    int64_t *locs;
    double *vals;
    int64_t entry_cap;
    int64_t *stats;          /* batch * SFDT_GS_PER_SIGNAL */
    int32_t *votes;          /* optional: batch * (n/d) estimated collision counts */
    double *singular_values; /* optional: batch * (n/d) * a_max */
    void *ev_fft_begin;      /* cudaEvent_t recorded right before / after the */
    void *ev_fft_end;        /* view gather + FFT kernels (optional, roofline timing) */
    /* optional phase events (GeneralTrace.timings, general.py:295-371): after
     * the collision vote, after pruning + matched filter, after the pursuit */
    void *ev_vote_end;
    void *ev_prune_end;
    void *ev_pursuit_end;
    /* optional second stream (cudaStream_t): the multi-collision pursuit
     * (a tail of a few long chains) forks onto it beside the single-collision
     * pursuit; NULL keeps everything on `stream`.  Forked and joined with
     * events, so a solve captured into a CUDA graph captures both branches. */
    void *aux_stream;
    const sfdt_tuning *tuning; /* optional A/B switches (NULL: defaults) */
    int32_t kernel_launches; /* out */
} sfdt_general_args;

/* estimate_collisions (general.py:131-155) on given consecutive syndromes
 * syn (nb, ld) row-major: singular values sv (nb, a_max) and votes (nb). */
size_t sfdt_estimate_collisions_workspace_bytes(int64_t nb);
int sfdt_estimate_collisions(const double *syn, int64_t nb, int64_t ld, int64_t k, int a_max, int64_t d,
                             double zero_vote_rtol, int32_t *votes, double *sv, void *workspace,
                             size_t workspace_bytes, sfdt_stream_t stream);

int sfdt_general_caps(const sfdt_general_args *args, int64_t *entry_cap);
/* args->x and args->tuning must already be the ones of the solve: host-mapped
 * signals (zero-copy) take a window buffer in the workspace (tuning.gen_window). */
size_t sfdt_general_workspace_bytes(const sfdt_general_args *args);
int sfdt_general_solve(sfdt_general_args *args, void *workspace, size_t workspace_bytes,
                       sfdt_stream_t stream);

/* ------------------------------------------------- library functions */
/* Device forms of the reference's per-view / per-bin library functions
 * (the drop-in surface around the solvers).  Batched: one call covers many
 * signals, views or bins.  Complex arrays are interleaved complex128. */

/* spectral.py:151-160 downsample: out[b, v, j] = x[b, (d*j + shifts[v]) mod n],
 * j < n/d, any n divisible by d (x complex128 or complex64 storage; out
 * complex128) */
int sfdt_downsample(const void *x, int32_t x_dtype, int64_t batch, int64_t n, int64_t d,
                    const int64_t *shifts, int32_t nshift, double *out, sfdt_stream_t stream);
/* spectral.py:163-172 transform_view / aliased_values:
 * out[b, v, :] = fft_radix2(view_v(x_b)) / (n/d), bit-identical to the
 * reference (the solvers' fused gather + FFT) */
size_t sfdt_aliased_values_workspace_bytes(int64_t batch, int64_t n, int64_t d, int32_t nshift);
int sfdt_aliased_values(const void *x, int32_t x_dtype, int64_t batch, int64_t n, int64_t d,
                        const int64_t *shifts, int32_t nshift, const double *twiddles, double *out,
                        void *workspace, size_t workspace_bytes, sfdt_stream_t stream);
/* spectral.py:110-125 forward_dft_oracle: O(n^2) direct DFT / n; roots_ws
 * holds n complex (the e^{-2 pi i q/n} table) */
int sfdt_direct_dft(const double *x, int64_t batch, int64_t n, double *roots_ws, double *out,
                    sfdt_stream_t stream);
/* spectral.py:215-218 rms(x) per signal (the solvers' own HBM pass) */
size_t sfdt_rms_workspace_bytes(int64_t batch, int64_t n);
int sfdt_rms(const void *x, int32_t x_dtype, int64_t batch, int64_t n, double *out, void *workspace,
             size_t workspace_bytes, sfdt_stream_t stream);

/* syndrome.py:69-175 (solve_coefficients, roots_closed_form, solve_values,
 * root_to_location, decode_bin) for nb bins: syndromes m (nb, ld), model a.
 * upto: 1 coefficients, 2 + roots, 3 + values, 4 + locations / snap /
 * membership against bins[] (mod n/d).  status[b]: 0 ok, 1 near-singular
 * (Hankel / m_0), 2 degenerate root branch, 3 ill-conditioned Vandermonde,
 * 4 zero root -- the reference's exceptions, as data; diag (nb, 2), optional:
 * the failing test's statistic and its bound (the exception messages).
 * upto >= 2 with a = 1 is decode_bin's ratio model (z = m1/m0, p = m0). */
enum { SFDT_DB_OK = 0, SFDT_DB_NEAR_SINGULAR = 1, SFDT_DB_DEGENERATE = 2, SFDT_DB_ILL_CONDITIONED = 3,
       SFDT_DB_ZERO_ROOT = 4 };
int sfdt_decode_bins(const double *m, int64_t nb, int64_t ld, int a, int64_t n, int64_t d,
                     const int64_t *bins, int upto, int32_t *status, double *c, double *roots,
                     double *vals, int64_t *locs, double *snap, int32_t *member, double *diag,
                     sfdt_stream_t stream);
/* syndrome.py:101-106: |P(z)| for c, z (nb, a) */
int sfdt_poly_residuals(const double *c, const double *z, int64_t nb, int a, double *out,
                        sfdt_stream_t stream);
/* syndrome.py:136-144: m_l = sum_j p_j z_j^l, l < count -> out (nb, count) */
int sfdt_reconstruct_syndromes(const double *roots, const double *vals, int64_t nb, int a, int count,
                               double *out, sfdt_stream_t stream);

/* general.py:109-121 sensing_matrix: out (r, ncols) with
 * Phi[j, t] = exp(2 pi i loc_t shifts_j / n), loc_t = (k + col_t n/d) mod n;
 * columns NULL = 0..ncols-1 */
int sfdt_sensing_matrix(int64_t n, int64_t d, int64_t k, const int64_t *shifts, int r,
                        const int64_t *columns, int64_t ncols, double *out, sfdt_stream_t stream);
/* general.py:184-221 prune_columns for nb bins (bin k[b], syndromes m (nb,
 * ld >= 2 a_max)): kept[b, :nkept[b]] sorted; nkept[b] = -1 means all d
 * columns.  y (nb, ldy) + shifts (r): the correlation fallback /
 * augmentation (NULL: none).  keep_per_collision * a <= 64; cap >= keep*a + a. */
int sfdt_prune_columns(const double *m, int64_t nb, int64_t ld, const int64_t *k, int a, int a_max,
                       int64_t n, int64_t d, int keep_per_collision, const double *y, int64_t ldy,
                       const int64_t *shifts, int r, int augment, int64_t *kept, int32_t *nkept,
                       int64_t cap, sfdt_stream_t stream);
/* general.py:224-269 subspace_pursuit on explicit problems: y (nb, rows),
 * phi (nb, rows, cols) -> coef (nb, cols) dense; rankdef[b] counts the
 * rank-deficient least-squares calls (the reference logs each).
 * rows <= 12, 2 * min(a, cols) <= 8 (the solver's shapes). */
int sfdt_subspace_pursuit(const double *y, const double *phi, int64_t nb, int rows, int cols, int a,
                          int max_iter, double *coef, int32_t *rankdef, sfdt_stream_t stream);

/* ------------------------------------------------------ latency path */
/* One small solve of SolvePipeline (graph.py): H2D of `bytes` from pinned
 * host memory into the captured graph's input buffer, event ev_h2d_done
 * (the host may then reuse host_src), replay of the instantiated graph
 * (a cudaGraphExec_t holding one complete solve + the D2H of its results),
 * event ev_done -- all on `stream`.  Events may be NULL. */
int sfdt_graph_submit(const void *host_src, void *dev_dst, size_t bytes, void *graph_exec,
                      sfdt_stream_t stream, void *ev_h2d_done, void *ev_done);

#ifdef __cplusplus
}
#endif
#endif /* SFDT_H */
