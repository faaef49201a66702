/*
 * asyflexa.h -- C ABI of the B200 (sm_100a) AsyFLEXA hot path.
 *
 * Method: Cannelli, Facchinei, Kungurtsev, Scutari, "Asynchronous Parallel
 * Algorithms for Nonconvex Big-Data Optimization, Part II: Complexity and
 * Numerical Results" (arXiv:1701.04900).  Line numbers below are PAPER.md's.
 *
 *   problem (1) [PAPER.md:58-68]:  min_x F(x) = f(x) + G(x),
 *        x = (x_1..x_N) in blocks, x_i in X_i = [lo, hi]^{n_i},
 *        G(x) = lambda * sum_j h(x_j)  (h = |.| or the DC penalties of Eq. 12),
 *        f(x) = s*||Ax - b||^2 - c*||x||^2                      (ASY_LOSS_LS)
 *        f(x) = (1/m) sum_j log(1 + exp(-y_j (Ax)_j)) - c*||x||^2 (ASY_LOSS_LOGISTIC)
 *   block update, Algorithm 1 (S.2)-(S.4) [PAPER.md:246-260]:
 *        hat x_i = argmin_{x_i in X_i} grad_i f(tilde x)^T (x_i - tilde x_i)
 *                    + 1/2 sum_{j in i} tau_j (x_j - tilde x_j)^2 + g_i(x_i)   (Eq. 2)
 *        x_i <- x_i + gamma (hat x_i - x_i)                                    (S.4)
 *   with grad_i f read through the shared residual r (LS: r = Ax - b;
 *   logistic: r = Ax), and A_i * dx_i pushed back into r.
 *
 * Conventions for every entry point:
 *   - all floating point is IEEE binary64; A is dense column-major (element
 *     (i, j) at A[j*lda + i]) or CSC (colptr int64[n+1], rowidx int32[nnz],
 *     vals double[nnz], rows strictly increasing inside a column);
 *   - a `mem` field says whether the pointers of that call are host
 *     (ASY_MEM_HOST: the library copies them) or device (ASY_MEM_DEVICE);
 *     device A / CSC arrays are BORROWED (caller keeps them alive and
 *     unchanged until the next asy_set_problem or asy_destroy); all other
 *     inputs are copied;
 *   - every call returns ASY_OK (0) or an error code; the message of the last
 *     error is returned by asy_last_error(h).  No call aborts the process.
 *   - calls are synchronous with respect to the host: when they return, the
 *     device work they issued on the handle's stream has completed.
 */
#ifndef ASYFLEXA_H
#define ASYFLEXA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASY_API __attribute__((visibility("default")))

/* status codes */
#define ASY_OK 0
#define ASY_ERR_INVALID 1     /* bad argument (null pointer, size, enum, tau <= 0, lo > hi, ...) */
#define ASY_ERR_CUDA 2        /* CUDA runtime error (no device, launch failure, ...) */
#define ASY_ERR_NOMEM 3       /* device allocation failed */
#define ASY_ERR_STATE 4       /* call out of order (e.g. solve before set_problem) */
#define ASY_ERR_UNSUPPORTED 5 /* valid but unsupported combination */

/* memory kinds */
#define ASY_MEM_HOST 0
#define ASY_MEM_DEVICE 1

/* matrix formats */
#define ASY_DENSE_COLMAJOR 0
#define ASY_CSC 1

/* smooth part f */
#define ASY_LOSS_LS 0        /* s*||Ax-b||^2          (LASSO: s = 1/2 [PAPER.md:433]; Eq. 11: s = 1 [PAPER.md:523]) */
#define ASY_LOSS_LOGISTIC 1  /* (1/m) sum log(1+exp(-y_j (Ax)_j)), b holds y in {-1,+1} */

/* separable regularizer h in G = lambda sum_j h(x_j) */
#define ASY_REG_L1 0   /* |t| */
#define ASY_REG_EXP 1  /* 1 - exp(-theta|t|),            DC split of Eq. (12)-(13) [PAPER.md:526-541] */
#define ASY_REG_LOG 2  /* log(1+theta|t|)/log(1+theta),   DC split of Eq. (12)-(13) */

/* solver modes */
#define ASY_MODE_ASYNC 0        /* persistent fused kernel, Algorithm 1 with bounded delay (max_delay);
                                   max_delay == 0 gives the sequential d^k = 0 scheme of the
                                   Corollary [PAPER.md:346-357], bit-reproducible */
#define ASY_MODE_SYNC_JACOBI 1  /* deterministic synchronous Jacobi sweep x+ = x + gamma(hat x(x) - x)
                                   from two GEMVs (A^T w, then A dx) */

/* update kernels (asy_solve_stats.kernel) */
#define ASY_KERNEL_JACOBI 0      /* two GEMVs per sweep */
#define ASY_KERNEL_DENSE_PANEL 1 /* dense_async.cuh: G row panels of a block on G SMs, TMEM parking */
#define ASY_KERNEL_DENSE_SLAB 2  /* dense_slab.cuh: every SM owns a row slab, per-update all-reduce */
#define ASY_KERNEL_SPARSE 3      /* sparse_async.cuh: CSC column updates */
#define ASY_KERNEL_DENSE_SLAB_TMEM 4 /* dense_slabt.cuh: row slabs, the tile parked in TMEM between dot and axpy */

/* block schedules (S.1) [PAPER.md:253] */
#define ASY_SCHED_CYCLIC 0  /* sequence k updates block k mod N */
#define ASY_SCHED_RANDOM 1  /* sequence k updates block pi_e(k mod N), e = epoch, pi_e a
                               Philox4x32-10-keyed random permutation of the N blocks */

typedef struct asy_handle asy_handle;

/* Problem statement, problem (1) [PAPER.md:58-68]. */
typedef struct {
    int32_t kind;          /* ASY_DENSE_COLMAJOR | ASY_CSC */
    int32_t mem;           /* memory kind of every pointer below */
    int64_t m, n;          /* A is m x n, m >= 1, n >= 1 */
    /* dense */
    const double* A;       /* column-major, leading dimension lda >= m */
    int64_t lda;
    /* CSC */
    const int64_t* colptr; /* n+1 entries, colptr[0] = 0, colptr[n] = nnz */
    const int32_t* rowidx; /* nnz entries in [0, m) */
    const double* vals;    /* nnz entries */
    int64_t nnz;
    /* f */
    int32_t loss;          /* ASY_LOSS_* */
    int32_t reg;           /* ASY_REG_* */
    double loss_scale;     /* s (LS only), > 0 */
    double c_nonconvex;    /* c >= 0: f -= c||x||^2 */
    double lambda;         /* >= 0 */
    double theta;          /* > 0 for ASY_REG_EXP / ASY_REG_LOG */
    const double* b;       /* m entries: LS target b, or logistic labels y */
    /* surrogate: proximal weights tau_j > 0 (length n) -- Assumption B1 [PAPER.md:169] */
    const double* tau;
    /* box X_i: per-coordinate arrays (length n) or NULL to use lo_all / hi_all (may be +-inf) */
    const double* lo;
    const double* hi;
    double lo_all, hi_all;
    /* blocks: x_i = x[i*block_size, min(n,(i+1)*block_size)), 1 <= block_size <= 128 */
    int64_t block_size;
} asy_problem;

/* Kernel choice and geometry overrides of the dense asynchronous kernels, for tests and
 * measurements (every field 0 = automatic; NULL pointer = all automatic).  None changes the
 * arithmetic: every variant computes the same Algorithm 1 updates (Kernels). */
typedef struct {
    int32_t dense_kernel;    /* 0 auto | ASY_KERNEL_DENSE_PANEL | ASY_KERNEL_DENSE_SLAB_TMEM (row-slab family:
                                the TMEM form when its park ring fits, else the smem/L2 form) |
                                ASY_KERNEL_DENSE_SLAB (the smem/L2 row-slab form) */
    int32_t panel_park;      /* panel kernel: 0 park panels in TMEM, 2 never (re-read them from L2) */
    int32_t slab_hold;       /* smem/L2 slab form: 0 auto, 1 hold the chunks in smem, 2 re-load them from L2 */
    int32_t slab_chunk_rows; /* smem/L2 slab form: rows per chunk (even, <= 256; 0 auto) */
    int32_t slab_ring;       /* TMEM slab form: load-ring stages per dot warp (1..16; 0 auto) */
    int32_t measure_delay;   /* 1: the panel and CSC kernels sample the observed delay
                                (asy_solve_stats.delay_observed) -- a measurement mode: its polls of
                                counters under heavy atomic traffic slow the kernels (~9%) */
    int32_t reserved[2];
} asy_tuning;

typedef struct {
    int32_t mode;          /* ASY_MODE_* */
    int32_t schedule;      /* ASY_SCHED_* (async mode) */
    uint64_t seed;         /* Philox key for ASY_SCHED_RANDOM */
    double gamma;          /* fixed stepsize, 0 < gamma <= 1  [PAPER.md:154] */
    int64_t sweeps;        /* passes: async = sweeps*N block updates; Jacobi = sweeps iterations */
    int64_t max_delay;     /* async: max block updates in flight besides the one being read
                              (Assumption D1's delta [PAPER.md:224]); -1 = auto (N/8; N/4 for CSC problems), 0 = sequential */
    int32_t reset;         /* 1: start from x0 (NULL: zeros), residual recomputed; 0: continue */
    int32_t x_mem;         /* memory kind of x0 / x_out */
    const double* x0;      /* n entries or NULL */
    double* x_out;         /* n entries or NULL: final x copied here */
    double* f_hist;        /* HOST array of `sweeps` entries or NULL: F(x) after every sweep */
    int32_t workers;       /* async: CTAs (0 = all resident) */
    int32_t panel_rows;    /* panel kernel: rows per panel (0 = auto; multiple of 32, <= 256) */
    int32_t stages;        /* panel kernel: smem stages (0 = auto, else 4 or 8).  A (panel_rows, stages)
                              pair with no compiled kernel for the block width -> ASY_ERR_UNSUPPORTED */
    const asy_tuning* tuning; /* NULL or overrides (see asy_tuning) */
} asy_solve_params;

typedef struct {
    int64_t block_updates;   /* block updates performed by this call */
    int64_t launches;        /* kernels launched by this call */
    double kernel_ms;        /* device time of the update kernels (CUDA events, handle stream) */
    double total_ms;         /* device time of the whole call */
    double objective;        /* F(x) at return, from the maintained residual */
    int64_t epochs;          /* cumulative sweeps since the last reset */
    int32_t kernel;          /* update kernel of the last launch: ASY_KERNEL_* */
    int32_t delay;           /* async: bounded delay actually enforced (<= max_delay; capped by the
                                kernel's buffering), -1 for Jacobi */
    int32_t delay_observed;  /* async: the largest number of earlier block updates missing from the
                                residual a gradient was read from (observed delay d^k, Assumption D1
                                [PAPER.md:224]; <= delay).  Always measured by the TMEM row-slab kernel;
                                by the panel and CSC kernels only with asy_tuning.measure_delay = 1
                                (sampled, an upper bound); -1 when not measured */
} asy_solve_stats;

typedef struct {
    double objective;   /* F(x) with a freshly computed residual */
    double smooth;      /* f(x) */
    double mf_norm2;    /* ||M_F(x)||_2, Eq. (5) [PAPER.md:287-290] */
    double mf_norminf;  /* ||M_F(x)||_inf */
    double merit_inf;   /* ||hat x(x) - x||_inf, Sec. 4.3 [PAPER.md:549] (tau metric) */
} asy_stationarity_out;

/* Create a handle on CUDA device `device`.  `stream` is a cudaStream_t to use
 * (NULL: the library creates its own non-blocking stream).  On error *out is
 * NULL and the message is available from asy_last_error(NULL). */
ASY_API int asy_create(int device, void* stream, asy_handle** out);

/* Release every device buffer the handle owns.  NULL is a no-op. */
ASY_API int asy_destroy(asy_handle* h);

/* Install problem (1).  Validates sizes/enums, copies host data (dense A is
 * re-laid out with an even leading dimension), borrows device A/CSC, builds
 * the CSR transpose for sparse problems, and resets x = 0, r = A*0 - b. */
ASY_API int asy_set_problem(asy_handle* h, const asy_problem* p);

/* Run the solver (see asy_solve_params).  `st` may be NULL. */
ASY_API int asy_solve(asy_handle* h, const asy_solve_params* sp, asy_solve_stats* st);

/* Stationarity of x (NULL: the current iterate): recomputes r = Ax - b and
 * grad f(x) from scratch and reduces M_F (Eq. 5) and the Sec. 4.3 merit. */
ASY_API int asy_stationarity(asy_handle* h, const double* x, int32_t x_mem,
                             asy_stationarity_out* out);

/* Copy the current iterate (n entries) to x. */
ASY_API int asy_get_x(asy_handle* h, double* x, int32_t x_mem);

/* Copy the maintained residual (m entries: LS r = Ax - b, logistic r = Ax, as updated
 * in place by the block updates -- A_i dx_i pushed into r [PAPER.md:246-260]) to r.  Lets a
 * caller check it against a fresh Ax - b (rounding drift of the in-place updates). */
ASY_API int asy_get_residual(asy_handle* h, double* r, int32_t r_mem);

/* F at the current iterate from the maintained residual (no recomputation). */
ASY_API int asy_objective(asy_handle* h, double* F);

/* Message of the last failed call on h (h == NULL: last asy_create failure). */
ASY_API const char* asy_last_error(const asy_handle* h);

ASY_API const char* asy_version(void);

/* ---- host-side helpers: the same __host__ __device__ code the kernels run ---- */

/* Philox4x32-10 (Salmon et al., SC'11) block function. */
ASY_API void asy_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Block updated by sequence number k (0-based, counted from epoch 0) under
 * `schedule` for N = nblocks blocks.  Returns ASY_ERR_INVALID on bad input. */
ASY_API int asy_schedule_block(int32_t schedule, uint64_t seed, int64_t nblocks, int64_t k,
                               int64_t* out);

/* Global index of the previous update of the block that sequence k updates
 * (every epoch visits each block once, so it lies in epoch k/N - 1), or -1 in
 * epoch 0.  The dense async kernel uses it for Assumption D4 [PAPER.md:233]:
 * a block is not read again before its previous update is applied. */
ASY_API int asy_schedule_prev(int32_t schedule, uint64_t seed, int64_t nblocks, int64_t k, int64_t* out);

/* Device evaluation of the same schedule for k = k0..k0+count-1 (written to the
 * HOST array out); lets tests check host == device bit for bit. */
ASY_API int asy_schedule_device(asy_handle* h, int32_t schedule, uint64_t seed, int64_t nblocks,
                                int64_t k0, int64_t count, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* ASYFLEXA_H */
