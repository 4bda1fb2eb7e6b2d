/*
 * cjt.h - C ABI of the B200 Chebyshev-Jacobi transform library (libcjt_b200.so).
 *
 * Plain C types only: pointers, sizes, int status codes.  Every entry point
 * returns 0 on success and a nonzero CJT_E* code on failure; the message of
 * the last failure on the calling thread is returned by cjt_last_error().
 *
 * Which reference interface each entry point replaces (reference package
 * `chebjac`, /root/reference/pkg/src/chebjac):
 *
 *   cjt_plan_create / cjt_plan_destroy   engine.plan (engine.py:96-130): the
 *        host builds the reference plan (partition, tables, weights) and
 *        hands the arrays over; the library uploads them once and derives the
 *        device work lists (recurrence checkpoints, chirp-z tables).
 *   cjt_execute          engine.forward (engine.py:153-186) / engine.inverse
 *        (engine.py:189-227), batched: device pointers in and out.
 *   cjt_execute_host     the same, host buffers in and out (H2D + execute +
 *        D2H on the given stream), i.e. what a drop-in caller of
 *        forward()/inverse() with NumPy arrays sees.
 *   cjt_clenshaw_points        backend plugin `clenshaw_points`
 *        (_kernels_cy.pyx:83-122, _kernels_np.py:22-57), same 12 arrays,
 *        host pointers, overwrites out.
 *   cjt_transpose_accumulate   backend plugin `transpose_accumulate`
 *        (_kernels_cy.pyx:201-237, _kernels_np.py:60-97), same 12 arrays,
 *        host pointers, accumulates into out.
 *   cjt_kernel_plan_create / _execute / _destroy   the same two plugin
 *        kernels with their per-plan device state kept across calls
 *        (backend.py caches one per reference plan).
 *   cjt_host_half_exact  alpha = beta = 1/2 exact-expansion tables
 *        (k_n, the reference's evaluation angles), host binary128.
 *   cjt_host_angles      the libm cos / half-angle evaluation the reference
 *        kernel performs per point (_kernels_cy.pyx:27,58-64), exposed so
 *        plans carry bit-identical x and x -+ 1 values.
 *   cjt_jacobi_shift     engine.increment_beta / decrement_beta /
 *        increment_alpha / decrement_alpha (engine.py:239-288), batched.
 *   cjt_clenshaw_points_dev / cjt_clenshaw_smith_points / cjt_jacobi_values
 *        recurrences.evaluate_expansion (batched), clenshaw_smith[_reinsch],
 *        jacobi_forward[_reinsch] (recurrences.py:74-171).
 *   cjt_chirpz_create / _execute / _destroy   trig.TrigPlanWorkspace.dct1 /
 *        dst1_bordered / chebyshev_synthesis / chebyshev_analysis
 *        (trig.py:35-63), batched.
 */
#ifndef CJT_B200_H
#define CJT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CJT_OK 0
#define CJT_EINVAL 1   /* bad argument (maps to ValueError) */
#define CJT_ECUDA 2    /* CUDA runtime failure */
#define CJT_ENOMEM 3   /* device allocation failed */
#define CJT_ENODEV 4   /* no CUDA device */

#define CJT_FORWARD 0
#define CJT_INVERSE 1

/* One batched chirp-z product with fused diagonals (see planner.py ChirpZ):
 *   out[b, q0-out_shift+s] (+)= sum_m Re(post[m, s] * z_{b,m}[s]),
 *   z_{b,m}[s] = sum_t exp(i pi (p0+t)(q0+s)/G) pre[m, t] x[b, p0+t].
 * Complex arrays are interleaved (re, im) float64. */
typedef struct {
    int64_t p0, width;      /* input index range */
    int64_t q0, count;      /* output index range */
    int64_t length;         /* power-of-two Bluestein length of one tile */
    int32_t m_count;        /* number of summed terms */
    int32_t accumulate;     /* 1: out +=, 0: out = */
    const double* pre;      /* [m_count][width] complex */
    const double* post;     /* [m_count][count] complex */
    /* tiling of the (width x count) index rectangle: tile (j, i) convolves
     * input tile i with output tile j; tiles_in[i] = (offset, width_i),
     * tiles_out[j] = (offset, count_j) relative to p0 / q0, and
     * width_i + count_j - 1 <= length.  Untiled: n_tiles_in = n_tiles_out = 1. */
    int32_t n_tiles_in, n_tiles_out;
    const int64_t* tiles_in;   /* [n_tiles_in][2] */
    const int64_t* tiles_out;  /* [n_tiles_out][2] */
    const double* kernel_hat;  /* [n_tiles_out][n_tiles_in][length] complex, 1/length folded in */
    int64_t out_shift;         /* results for q land at out[q - out_shift] (0: at out[q]) */
    /* device-side planning (device_tables = 1): pre / post are the bare
     * diagonals (no chirp), kernel_hat is ignored, and the library builds the
     * chirps, the folded tables and every tile's spectrum on the GPU for the
     * grid parameter grid_g.  A diagonal of kind CJT_DIAG_MODULATION is not
     * passed at all: it is u_m - i v_m (asymptotics.py:36-75) of the plan's
     * grid rows pre_row0 + t / post_row0 + s (plan create only). */
    int32_t device_tables;
    int32_t pre_kind, post_kind;   /* CJT_DIAG_ARRAY or CJT_DIAG_MODULATION */
    int64_t grid_g;
    int64_t pre_row0, post_row0;
} cjt_chirpz_desc;

#define CJT_DIAG_ARRAY 0
#define CJT_DIAG_MODULATION 1

typedef struct {
    int32_t direction;      /* CJT_FORWARD or CJT_INVERSE */
    int32_t m_terms;
    int64_t n;              /* degree N of the coefficient vectors */
    int64_t grid_n;         /* G = N (forward) or 2N (inverse) */
    /* recurrence region, one entry per grid row 0..G */
    const double* x;        /* cos(theta_i) (libm) */
    const double* xm;       /* x - x0 via half angles for regions +-1, unused for 0 */
    const int8_t* regions;  /* 0 interior, 1 near +1, -1 near -1 */
    const int64_t* cuts;    /* recurrence degrees at row i are 0..cuts[i]-1 (already capped) */
    /* recurrence tables, length table_len (>= max cut + 1) */
    int64_t table_len;
    const double* A;
    const double* B;
    const double* C;
    const double* rf_plus;
    const double* rf_minus;
    const double* rf_plus_inv;
    const double* rf_minus_inv;
    /* asymptotic blocks */
    int32_t n_blocks;
    const cjt_chirpz_desc* blocks;
    /* forward: Chebyshev analysis; inverse: weighted Chebyshev synthesis */
    cjt_chirpz_desc edge;
    /* inverse: 1/A_n for n = 0..N (NULL for forward) */
    const double* scalings;
    /* forward, alpha = beta = 1/2 only (else NULL): k_n = P_n(1) / (n+1),
     * n = 0..N, so P_n = k_n U_n; the forward then is the exact
     * U -> T conversion (cheb_j = e_j sum_{n >= j, n = j mod 2} k_n c_n) and
     * needs no recurrence rows, blocks or edge (edge.length may be 0) */
    const double* half_k;
    /* grid angles theta_i (i = 0..G) and (alpha, beta): needed when a block
     * diagonal is of kind CJT_DIAG_MODULATION (else may be NULL / unused) */
    const double* thetas;
    double alpha, beta;
    /* inverse exact-expansion plans only: 1 = run as the exact conversion plus
     * a bf16 tensor-core correction (blocks[0] is then the CORRECTION chirp-z;
     * the library applies edge + blocks[0] to the identity once to build the
     * (N+1) x (N+1) correction matrix) */
    int32_t half_gemm;
} cjt_plan_desc;

typedef struct cjt_plan cjt_plan;

typedef struct {
    int64_t launches_per_execute;   /* kernels one cjt_execute launches (batch-independent) */
    int64_t rec_steps;              /* sum over rows of recurrence degrees */
    int64_t checkpoint_bytes;
    int64_t workspace_bytes;
    int64_t reserved_batch;
    double rec_flops_per_vector;    /* 2 flop per (row, degree) contraction */
    double fft_points_per_vector;   /* sum over executed FFTs of length x log2(length) */
    int64_t rec_steps_executed;     /* (row, degree) pairs the contractions execute: rec_steps,
                                       or the rows i <= G/2 only for parity-folded plans */
} cjt_plan_stats;

int cjt_version(void);
const char* cjt_last_error(void);
int cjt_device_count(int* count);

int cjt_plan_create(const cjt_plan_desc* desc, cjt_plan** out);
int cjt_plan_destroy(cjt_plan* plan);
int cjt_plan_reserve(cjt_plan* plan, int64_t max_batch);
int cjt_plan_stats_get(const cjt_plan* plan, cjt_plan_stats* stats);

/* in: [batch][N+1] float64, out: [batch][N+1] float64, device pointers.
 * stream: a cudaStream_t (NULL = legacy default stream). */
int cjt_execute(cjt_plan* plan, const double* in, double* out, int64_t batch, void* stream);
/* Same with host buffers; copies happen on `stream`, returns after D2H completes. */
int cjt_execute_host(cjt_plan* plan, const double* in_host, double* out_host,
                     int64_t batch, void* stream);

/* Timing aid: run only some stages of one execution (results are not a
 * transform unless stages == CJT_STAGE_ALL).  batch <= reserved batch. */
#define CJT_STAGE_REC 1
#define CJT_STAGE_BLOCKS 2
#define CJT_STAGE_EDGE 4
#define CJT_STAGE_ALL 7
int cjt_execute_stage(cjt_plan* plan, const double* in, double* out, int64_t batch,
                      int32_t stages, void* stream);
/* Measured fp64 FMA throughput of the current device (TFLOP/s, best of 5). */
int cjt_probe_fp64_peak(double* tflops, void* stream);

/* Standalone batched chirp-z products: the trigonometric transforms of
 * trig.py (TrigPlanWorkspace.dct1 / dst1_bordered / chebyshev_synthesis /
 * chebyshev_analysis, trig.py:35-63), each one cjt_chirpz_desc with M = 1
 * (the Python layer builds pre / post / spectra).  Device pointers,
 * in: [batch][ldi] (reads p0 .. p0+width), out: [batch][ldo] (writes q0 ..
 * q0+count, overwritten or accumulated per desc.accumulate); stream ordered,
 * per-stream workspaces (allocated on a stream's first use, outside capture). */
typedef struct cjt_chirpz_plan cjt_chirpz_plan;
int cjt_chirpz_create(const cjt_chirpz_desc* desc, cjt_chirpz_plan** out);
int cjt_chirpz_execute(cjt_chirpz_plan* plan, const double* in, int64_t ldi, double* out,
                       int64_t ldo, int64_t batch, void* stream);
int cjt_chirpz_destroy(cjt_chirpz_plan* plan);

/* Reference backend-plugin signatures, host arrays (see header comment). */
int cjt_clenshaw_points(const double* A, const double* B, const double* C,
                        const double* rb_plus, const double* rb_minus,
                        const double* rb_plus_inv, const double* rb_minus_inv,
                        const double* coeffs, int64_t n_coeffs,
                        const double* thetas, const int64_t* cuts,
                        const int8_t* regions, double* out, int64_t n_points);
int cjt_transpose_accumulate(const double* A, const double* B, const double* C,
                             const double* rf_plus, const double* rf_minus,
                             const double* rf_plus_inv, const double* rf_minus_inv,
                             const double* wv, const double* thetas,
                             const int64_t* cuts, const int8_t* regions,
                             double* out, int64_t n_out, int64_t n_points,
                             int64_t table_len);

/* Reusable device state of one backend-plugin call site (the reference
 * engine passes the same plan arrays on every call, engine.py:177-183,
 * 220-225): tables, libm angles and row layout are uploaded once by
 * cjt_kernel_plan_create; each cjt_kernel_plan_execute moves one vector.
 *   CJT_KERNEL_CLENSHAW   clenshaw_points: r_* = rb+-, 1/rb+-; n_len = number
 *                         of coefficients; execute(in = coeffs, out = values
 *                         at the n_points rows, overwritten)
 *   CJT_KERNEL_TRANSPOSE  transpose_accumulate: r_* = rf+-, 1/rf+-; n_len =
 *                         length of out; execute(in = wv at the rows, out +=)
 * cjt_clenshaw_points / cjt_transpose_accumulate are create + execute +
 * destroy in one call.  Thread-safe (one call at a time per plan). */
#define CJT_KERNEL_CLENSHAW 0
#define CJT_KERNEL_TRANSPOSE 1
typedef struct cjt_kernel_plan cjt_kernel_plan;
int cjt_kernel_plan_create(int32_t kind, const double* A, const double* B, const double* C,
                           const double* r_plus, const double* r_minus,
                           const double* r_plus_inv, const double* r_minus_inv,
                           int64_t table_len, const double* thetas, const int64_t* cuts,
                           const int8_t* regions, int64_t n_points, int64_t n_len,
                           cjt_kernel_plan** out);
int cjt_kernel_plan_execute(cjt_kernel_plan* plan, const double* in, double* out);
int cjt_kernel_plan_destroy(cjt_kernel_plan* plan);

/* alpha = beta = 1/2 exact-expansion tables (planner.half_exact_tables):
 * k[m] = P_m(1)/(m+1), m = 0..n; for every row p of the inverse grid G the
 * angle phi_p of the point the reference's recurrence evaluates (interior:
 * acos(x_p); near +-1: from the half-angle x-+1 value xm_p), computed in
 * binary128, as inv_sin[p] = 1/sin(phi_p) and delta_over_sin[p] =
 * (phi_p - pi p/G)/sin(phi_p) (endpoint rows p = 0, G: 0).  With inv_sin ==
 * delta_over_sin == NULL only k is computed (forward plans).  Host only. */
int cjt_host_half_exact(const double* x, const double* xm, const int8_t* regions, int64_t G, int64_t n,
                        double* k, double* inv_sin, double* delta_over_sin);

int cjt_host_angles(const double* thetas, const int8_t* regions, int64_t n,
                    double* x, double* xm);

/* Batched reference-signature Clenshaw-Smith / Reinsch evaluation with DEVICE
 * pointers (recurrences.py:150-171 evaluate_expansion, over a batch):
 * out[b*ldo + i] = sum_{n < cuts[i]} coeffs[b*ldc + n] P_n(x_i), plain
 * Clenshaw-Smith where regions[i] == 0, Reinsch anchored at +-1 otherwise,
 * x / xm as cjt_host_angles returns them; tables hold >= max(cuts)+1
 * entries (table_len).  batch <= 65535.  Bit-identical to the reference
 * kernel per vector.  Stream ordered, no allocation. */
int cjt_clenshaw_points_dev(const double* A, const double* B, const double* C,
                            const double* rb_plus, const double* rb_minus,
                            const double* rb_plus_inv, const double* rb_minus_inv,
                            int64_t table_len, const double* coeffs, int64_t ldc,
                            const double* x, const double* xm, const int64_t* cuts,
                            const int8_t* regions, double* out, int64_t ldo,
                            int64_t n_points, int64_t batch, void* stream);

/* The scalar reference helpers clenshaw_smith (modes[i] = 0) and
 * clenshaw_smith_reinsch (modes[i] = end = +1 / -1) (recurrences.py:115-152),
 * host pointers: out[i] = sum_{n < n_coeffs} coeffs[n] P_n(cos theta_i) with
 * the Python helpers' operation order (the Reinsch step DIVIDES by rb[n]
 * where the Cython plugin multiplies by 1/rb[n]), bit-identical to them.
 * Tables hold >= n_coeffs + 1 entries. */
int cjt_clenshaw_smith_points(const double* A, const double* B, const double* C,
                              const double* rb_plus, const double* rb_minus,
                              const double* coeffs, int64_t n_coeffs,
                              const double* thetas, const int8_t* modes,
                              int64_t n_points, double* out);

/* P_0..P_{n_max} at each angle (recurrences.py:74-112 jacobi_forward /
 * jacobi_forward_reinsch), host pointers: modes[i] = 0 plain forward
 * recurrence at cos(theta_i); +1 / -1 Reinsch's modified recurrence anchored
 * at x0 = +1 / -1 (rf_plus / rf_minus).  out: [n_points][n_max+1], the
 * reference's operation order (bit-identical).  Tables hold >= n_max entries. */
int cjt_jacobi_values(const double* A, const double* B, const double* C,
                      const double* rf_plus, const double* rf_minus, int64_t table_len,
                      int64_t n_max, const double* thetas, const int8_t* modes,
                      int64_t n_points, double* out);

/* Integer parameter shifts of Jacobi coefficient vectors (engine.py:232-292),
 * device pointers, in/out: [batch][n+1] float64 (may not alias), (alpha,
 * beta) = the SOURCE parameters; the result is in the shifted basis
 * (beta+1, beta-1, alpha+1, alpha-1).  Increments are bit-identical to the
 * reference; decrements are its back-substitution run as a chunked
 * first-order recurrence (rounding differs at chunk boundaries only).
 * Target parameters must stay > -1 (CJT_EINVAL otherwise). */
#define CJT_SHIFT_INC_BETA 0
#define CJT_SHIFT_DEC_BETA 1
#define CJT_SHIFT_INC_ALPHA 2
#define CJT_SHIFT_DEC_ALPHA 3
int cjt_jacobi_shift(int32_t op, double alpha, double beta, const double* in, double* out,
                     int64_t n, int64_t batch, void* stream);

/* Plan-time host helper: Jacobi moments mu_0..mu_g by the reference's
 * three-term recurrence (quadrature.py:35-53), same operation order, given
 * mu_0 (the Gamma-function ratio, computed by the caller). */
int cjt_host_moments(double alpha, double beta, double mu0, int64_t g, double* mu);

#ifdef __cplusplus
}
#endif
#endif /* CJT_B200_H */
