/*
 * mpk_b200.h — C ABI of libmpkb200.so, the sm_100a implementation of the
 * multiprecision GMRES solve path of arXiv 2105.07544 (reference package
 * `mpkrylov`, /root/reference/pkg/src/mpkrylov).
 *
 * Conventions
 *   - Plain C types only: device pointers are `void*`/typed pointers, sizes
 *     are int64_t, streams are `void*` (a cudaStream_t; NULL = legacy stream).
 *   - Every entry point is stream-ordered and asynchronous; none allocates
 *     device memory (the caller owns all buffers, sized by the *_bytes
 *     queries) and none synchronises unless its name says so.
 *   - Return value: 0 on success, a negative MPK_E* code on a launch or
 *     argument error (message via mpk_last_error()).  Numerical outcomes
 *     (breakdowns, triangular breakdown, convergence) are reported through
 *     device-resident control words, never through the return value — the
 *     reference reports non-convergence as a flag, not an exception
 *     (SPEC.md:239), and raises typed errors the host layer re-creates.
 *   - No fast-math anywhere: IEEE division/sqrt, no FTZ.
 *
 * Each entry point names the reference interface (file:line under
 * /root/reference/pkg/src/mpkrylov/) whose arithmetic it replaces.
 */
#ifndef MPK_B200_H
#define MPK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPK_ABI_VERSION 2   /* 2: mpk_matrix.band */

/* storage precision (precision.py:14-71: binary32 / binary64) */
enum { MPK_F32 = 0, MPK_F64 = 1 };

/* operator kinds */
enum { MPK_CSR = 0, MPK_STENCIL = 1 };

/* stencil presets (stencils.py:22, builders 78-170) */
enum {
    MPK_LAPLACE2D = 0, MPK_LAPLACE3D = 1, MPK_UNIFLOW2D = 2,
    MPK_BENTPIPE2D = 3, MPK_STRETCHED2D = 4
};

/* preconditioner kinds (preconditioners.py:70-317) */
enum { MPK_PC_NONE = 0, MPK_PC_JACOBI = 1, MPK_PC_POLY = 2 };

/* breakdown rule of the CGS2 append test (kernels.py:122-123) */
enum { MPK_RULE_NU = 0 /* beta <= n*u*||w||, reference */, MPK_RULE_U = 1 /* beta <= u*||w|| */ };

/* error codes */
enum {
    MPK_OK = 0, MPK_EARG = -1, MPK_ELAUNCH = -2, MPK_EUNSUPPORTED = -3, MPK_EWORKSPACE = -4
};

/*
 * A square operator (or a row block of one).  CSR: row_ptr[n+1], col_idx[nnz]
 * (int32, columns index the x buffer), values[nnz] in `dtype`.  STENCIL: the
 * preset's coefficients are generated on the fly from (preset, nx, params)
 * with the reference's operation order, so the product is bit-identical to
 * the CSR product of generate_stencil's matrix (stencils.py:192-207).
 * `row0` is the first global row of a row block; x is addressed as
 * x[global_col - row0] (x points at local row 0; halo rows precede/follow).
 */
typedef struct mpk_matrix {
    int32_t kind;
    int32_t dtype;
    int64_t n;          /* local rows */
    int64_t nnz;        /* CSR only */
    const int32_t *row_ptr;
    const int32_t *col_idx;
    const void *values;
    int32_t preset;     /* STENCIL only */
    int32_t nx;
    int64_t row0;
    double diffusion, velocity, convection, stretch;
    int64_t band;       /* CSR only: x-window half-width for banded rows (0 = off);
                           the caller sets it from row statistics (sparse.py) */
} mpk_matrix;

/*
 * A preconditioner handle in the operator's precision.
 * JACOBI: k-by-k LU factors, block b at lu + b*k*k (row-major, LAPACK getrf
 * layout transposed: lu[b][i][j] = factor(i, j)), pivots piv[b*k + i]
 * (0-based row swapped with i), last block of size n - (nblocks-1)*k.
 * POLY: `degree` roots (Leja order, conjugate pairs adjacent), their matrix
 * is `poly_A`; work buffers of 3*n elements supplied by the caller.
 */
typedef struct mpk_precond {
    int32_t kind;
    int32_t dtype;
    int64_t n;
    int32_t block;             /* JACOBI */
    const void *lu;            /* JACOBI */
    const int32_t *piv;        /* JACOBI */
    int32_t degree;            /* POLY */
    const double *roots_re;    /* POLY (host or device-visible pinned pointer not needed: copied) */
    const double *roots_im;
    const mpk_matrix *poly_A;
    void *work;                /* POLY: 3*n elements of dtype */
} mpk_precond;

/* ------------------------------------------------------------------ */
/* library                                                             */
/* ------------------------------------------------------------------ */
int mpk_abi_version(void);
const char *mpk_last_error(void);
/* number of SMs of the current device (grids are sized in multiples of it) */
int mpk_sm_count(void);
/* Return the L2 lines the persistent cycle kernels marked persisting (their
 * access-policy window over the cycle's work vectors) to normal status; the
 * solve drivers call it once at the end of a solve (no reference
 * counterpart: B200 L2 residency control).  MPK_L2_PERSIST=0
 * turns the window off. */
int mpk_l2_release(void);

/* ------------------------------------------------------------------ */
/* sparse product and casts                                            */
/* ------------------------------------------------------------------ */
/* y = A x, rows summed sequentially with round-to-nearest multiply and add
 * (no FMA): bit-identical to scipy csr_matvec behind mpkrylov.spmv
 * (sparse.py:190-206). */
int mpk_spmv(const mpk_matrix *A, const void *x, void *y, void *stream);

/* dst = (dst_dtype) src, round to nearest (sparse.py:222-226, convert_vector;
 * also convert_matrix's values cast, sparse.py:209-219). */
int mpk_convert(int32_t src_dtype, int32_t dst_dtype, int64_t n, const void *src, void *dst,
                void *stream);

/* ------------------------------------------------------------------ */
/* dense vector kernels (kernels.py:31-52)                             */
/* ------------------------------------------------------------------ */
/* bytes of reduction workspace any reduction entry point may use */
int64_t mpk_reduce_ws_bytes(int64_t n, int32_t max_cols);
/* result[0] = x . y accumulated in dtype (deterministic two-stage tree) */
int mpk_dot(int32_t dtype, int64_t n, const void *x, const void *y, void *result, void *ws,
            void *stream);
/* result[0] = sqrt(x . x) in dtype */
int mpk_norm2(int32_t dtype, int64_t n, const void *x, void *result, void *ws, void *stream);
/* out = y + (dtype)alpha * x */
int mpk_axpy(int32_t dtype, int64_t n, double alpha, const void *x, const void *y, void *out,
             void *stream);
/* out = x / d[0] with d a device scalar in dtype (kernels.py:125 `w / beta`) */
int mpk_vdiv(int32_t dtype, int64_t n, const void *x, const void *d, void *out, void *stream);
/* out = (dtype)alpha * x */
int mpk_scale(int32_t dtype, int64_t n, double alpha, const void *x, void *out, void *stream);

/* ------------------------------------------------------------------ */
/* CGS2 append (kernels.py:98-126)                                     */
/* ------------------------------------------------------------------ */
/* Orthogonalise w against V[:, :count] (column-major, leading dim ld) with
 * two classical Gram-Schmidt passes.  Writes coeffs[count] = c1 + c2,
 * out[0] = beta, out[1] = ||w||, appended_dev[0] = beta > thresh (rule),
 * and, when appended, V[:, count] = w'' / beta.  w is not modified
 * (scratch: 2*n elements in `tmp`). */
int mpk_cgs2_append(int32_t dtype, int64_t n, int64_t ld, int32_t count, void *V, const void *w,
                    int32_t rule, void *coeffs, void *out, int32_t *appended_dev, void *tmp,
                    void *ws, void *stream);

/* ------------------------------------------------------------------ */
/* row-partitioned multi-GPU cycle                       */
/* ------------------------------------------------------------------ */
/* One rank per GPU owns the contiguous global rows [row0, row0 + n).  The
 * persistent cycle kernel of every rank writes its per-CTA dot-product
 * partials straight into every rank's partial buffer and its boundary rows
 * of w'' straight into the neighbours' global-length x buffers (P2P stores
 * over NVLink through CUDA-IPC-mapped pointers), then meets the other ranks
 * at a system-scope counter barrier; every rank reduces all ranks' partials
 * in the same fixed order and runs the same Givens update, so the cycle
 * needs no NCCL call and no host round trip.  Pointers below are indexed by
 * rank; the local rank's entries are its own buffers. */
#define MPK_MAX_RANKS 8
typedef struct mpk_comm {
    int32_t rank;
    int32_t nranks;
    int32_t ctas;                    /* CTAs of each rank's cycle kernel (0 = one per SM) */
    int32_t pad_;
    int64_t row0;                    /* first global row of this rank */
    void *part[MPK_MAX_RANKS];       /* mpk_comm_part_bytes(dtype) each */
    void *xbar[MPK_MAX_RANKS];       /* uint64 arrival counter each (zero-initialised) */
    void *epoch;                     /* uint64, this rank's barriers so far (zero-initialised) */
    void *xg[MPK_MAX_RANKS];         /* global-length vector (cycle dtype, global row 0) each */
    int64_t mir_lo[MPK_MAX_RANKS];   /* local rows [mir_lo[q], mir_hi[q]) of w'' are mirrored */
    int64_t mir_hi[MPK_MAX_RANKS];   /*   into rank q's xg (q != rank; empty: lo >= hi) */
} mpk_comm;

/* bytes of one rank's partial buffer (3 phases x 65 slots x 8 ranks x 320 CTAs) */
int64_t mpk_comm_part_bytes(int32_t dtype);
/* cudaMalloc'd (not pool) memory, so that CUDA IPC handles cover it exactly */
int mpk_dev_alloc(int64_t bytes, void **ptr);
int mpk_dev_free(void *ptr);
/* 64-byte cudaIpcMemHandle_t of an mpk_dev_alloc pointer, and its mapping in
 * another process (cudaIpcMemLazyEnablePeerAccess) */
int mpk_ipc_get(const void *ptr, void *handle64);
int mpk_ipc_open(const void *handle64, void **ptr);
int mpk_ipc_close(void *ptr);
/* 1 when device `dev` can map `peer`'s memory (cudaDeviceCanAccessPeer; 1
 * for dev == peer), 0 when it cannot; the communicator refuses to build on 0 */
int mpk_can_access_peer(int32_t dev, int32_t peer);
/* Per-restart collectives of the row-partitioned solve (gmres.py:290-291,
 * multiprecision.py:216-217 across ranks), device-side over the same peer
 * buffers and arrival counters as the cycle kernel; `dtype` names the
 * communicator's precision set.
 * push_rows: x (n local rows) -> own xg at row0, mirror rows -> the peers'
 *   xg, then a cross-rank barrier; the residual then reads xg's halo.
 * reduce_ctl: the 32-byte slot {r.r (dtype rn2_dtype), r_low.r_low (f32),
 *   moved (i32), timeout (i32, out), b.b (dtype bn2_dtype)} summed over the
 *   ranks in rank order, in place. */
int mpk_comm_push_rows(const mpk_comm *c, int32_t dtype, int64_t n, const void *x, void *stream);
int mpk_comm_reduce_ctl(const mpk_comm *c, int32_t dtype, void *slot32, int32_t rn2_dtype, int32_t bn2_dtype,
                        void *stream);

/* ------------------------------------------------------------------ */
/* restarted GMRES cycle (gmres.py:134-205)                            */
/* ------------------------------------------------------------------ */
/* Device control block of one cycle (read back once per cycle). */
#define MPK_MAX_STEPS 512
typedef struct mpk_cycle_ctl {
    int32_t done;           /* cycle finished */
    int32_t steps;          /* Arnoldi steps taken (k) */
    int32_t breakdown;      /* last step not appended (kernels.py:122-126) */
    int32_t tri_err;        /* TriangularBreakdownError (kernels.py:210-215) */
    int32_t tri_index;
    int32_t pad_;
    double tri_entry;
    double tri_threshold;
    double gamma;           /* ||r0|| (as double) */
    double scale;           /* norm_scale */
    double implicit_relres[MPK_MAX_STEPS];
} mpk_cycle_ctl;

typedef struct mpk_cycle_desc {
    const mpk_matrix *A;
    const mpk_precond *M;   /* NULL or kind NONE: identity */
    int32_t dtype;
    int32_t m;              /* restart length (columns), <= MPK_MAX_STEPS */
    int32_t steps_cap;      /* max steps this cycle (gmres.py:168) */
    int32_t rule;           /* MPK_RULE_* */
    double exit_tol;        /* implicit tolerance (gmres.py:169) */
    double norm_scale;      /* <= 0: use gamma (gmres.py:167) */
    int64_t n;
    int64_t ld;             /* leading dimension of V (>= n, multiple of 64) */
    void *V;                /* ld * (m + 1) */
    const void *r0;         /* initial residual (n) */
    const void *rnorm2;     /* device scalar: r0 . r0 in dtype (gamma = sqrt) */
    const void *x0;         /* iterate the correction is added to (n) */
    void *x_out;            /* x0 + M(V_k d) (n); may alias x0 */
    void *work;             /* 4 * ld elements */
    void *hess;             /* mpk_cycle_hess_bytes(m, dtype) */
    void *ws;               /* mpk_reduce_ws_bytes(n, m + 2) */
    mpk_cycle_ctl *ctl;     /* device */
    int32_t nranks;         /* 1, or > 1 with `comm` (row-partitioned; identity preconditioner) */
    int32_t flags;          /* bit0: per-kernel event timing; bit1: write the last basis column;
                               bit2: force the multi-kernel cycle (no persistent kernel);
                               bit3: phase profiler of the persistent kernel;
                               bit4: lagged one-reduction CGS2 (identity preconditioner, m <= 51);
                               bit5: basis stored in binary16 (scaled by a power of two; binary32
                                     cycles, one GPU, m <= 51, CGS2, identity or Jacobi(1)); V then
                                     holds ld * (m + 1) binary16 values;
                               bit6: the same with bfloat16 basis storage */
    const mpk_comm *comm;   /* nranks > 1: this rank's view of the communicator */
} mpk_cycle_desc;

int64_t mpk_cycle_hess_bytes(int32_t m, int32_t dtype);
/* Launch one whole cycle: begin, steps_cap x {normalise, M, SpMV+dot,
 * update+dot, update+norm+Givens}, back-substitution, correction.  Kernels
 * after an early exit (implicit <= exit_tol, or breakdown) are no-ops read
 * from ctl->done; the host reads ctl once per cycle. */
int mpk_cycle_run(const mpk_cycle_desc *d, void *stream);

/* Standalone rotated least-squares state (HessenbergSystem,
 * kernels.py:139-216) in `hess` (mpk_cycle_hess_bytes) + `ctl`.
 * init: g[0] = gamma, scale = norm_scale (kernels.py:152-165).
 * update: fold column j (1-based) = (coeffs[0..j), beta) in; the relative
 *   residual |g_j|/scale lands in ctl->implicit_relres[j-1] (kernels.py:166-196).
 * solve: d = R[:k,:k] \ g[:k] into the `d` slot, or ctl->tri_err/tri_* set
 *   (kernels.py:202-216). */
int mpk_lsq_init(int32_t dtype, int32_t m, double gamma, double norm_scale, void *hess,
                 mpk_cycle_ctl *ctl, void *stream);
int mpk_lsq_update(int32_t dtype, int32_t m, int32_t j, const void *coeffs, const void *beta,
                   void *hess, mpk_cycle_ctl *ctl, void *ws, void *stream);
int mpk_lsq_solve(int32_t dtype, int32_t m, int32_t k, void *hess, mpk_cycle_ctl *ctl,
                  void *stream);

/* ------------------------------------------------------------------ */
/* explicit residual and refinement passes (gmres.py:247,290-291;      */
/* multiprecision.py:180-181,207-217)                                  */
/* ------------------------------------------------------------------ */
/* r = b - A x (bit-identical to the reference's `b - spmv(A, x)`),
 * sums[0] = r . r in A's dtype.  If r_low != NULL (A fp64 only): also
 * r_low = (float) r and sums_low[0] = r_low . r_low in fp32. */
int mpk_residual(const mpk_matrix *A, const void *b, const void *x, void *r, void *sums,
                 float *r_low, float *sums_low, void *ws, void *stream);
/* x_next = x + (double) u; changed[0] |= any(x_next != x)  (multiprecision.py:207-214). */
int mpk_ir_update(int64_t n, double *x, const float *u, int32_t *changed, void *stream);

/* ------------------------------------------------------------------ */
/* preconditioner application (preconditioners.py:133-139, 276-305)    */
/* ------------------------------------------------------------------ */
int mpk_precond_apply(const mpk_precond *M, const void *v, void *out, void *stream);

/*
 * Block-Jacobi setup on the device (replaces build_block_jacobi's per-block
 * scipy.linalg.lu_factor loop, pkg/src/mpkrylov/preconditioners.py:96-130):
 * dense k-by-k diagonal blocks of the CSR matrix A (its dtype), LU with
 * partial pivoting, factors in mpk_precond's JACOBI layout (lu: nblocks*k*k,
 * piv: nblocks*k).  minpiv[b] = min|u_ii| (A's dtype), thr[b] = (kb*u)*max
 * row sum |a| (double); *bad (initialise to INT32_MAX) = the lowest block with
 * minpiv <= thr (the reference's SingularBlockError).  1 <= k <= 64.
 */
int mpk_block_lu(const mpk_matrix *A, int32_t k, void *lu, int32_t *piv, void *minpiv, double *thr, int32_t *bad,
                 void *stream);

/*
 * Stencil assembly on the device (replaces generate_stencil's numpy
 * assembly, pkg/src/mpkrylov/stencils.py:192-207): the binary64 CSR arrays
 * of the STENCIL operator S (whole matrix, row0 = 0), bit-identical to the
 * reference's (column order = displacement order, Dirichlet truncation).
 * row_ptr: n + 1 int64; col_idx: nnz int32; values: nnz doubles; work:
 * mpk_stencil_assemble_ws_bytes(n) bytes.
 */
int mpk_stencil_assemble(const mpk_matrix *S, int64_t *row_ptr, int32_t *col_idx, double *values, void *work,
                         void *stream);
int64_t mpk_stencil_assemble_ws_bytes(int64_t n);

/* ------------------------------------------------------------------ */
/* host-side setup                                                     */
/* ------------------------------------------------------------------ */
/* Reverse Cuthill-McKee permutation of a symmetrized off-diagonal pattern
 * (row-sorted CSR indptr[n+1] / indices, host memory) into perm[n]; the
 * permutation of mpkrylov's rcm_ordering (reorder.py:22-63).  Host code, no
 * device work. */
int mpk_rcm_host(int64_t n, const int64_t *indptr, const int64_t *indices, int64_t *perm);

/* ------------------------------------------------------------------ */
/* profiling hooks: per-kernel-class event timing inside mpk_cycle_run */
/* ------------------------------------------------------------------ */
/* classes: 0 SpMV+dot1, 1 update1+dot2, 2 update2+norm, 3 normalise, 4 precond,
 * 5 correction, 6 residual, 7 other */
int mpk_prof_reset(void);
/* number of kernels this library has enqueued so far (monotonic) */
int64_t mpk_launch_count(void);
/* kernel family the calling thread's last mpk_cycle_run launched
 * ("k_cycle_reg", "k_cycle_reg/big", "k_cycle_reg/multi", "k_cycle_dcgs2",
 * "k_cycle_dcgs2/multi", "k_cycle_fused", "multi-kernel"); diagnostics/tests */
const char *mpk_last_cycle_kernel(void);
/* totals[c] = summed milliseconds, counts[c] = launches, bytes[c] = algorithmic bytes */
int mpk_prof_read(double *ms, int64_t *counts, double *bytes, int32_t nclasses);
/* per-CTA clock64 totals of the persistent cycle's sections (16 slots per
 * CTA) from the last cycle run with flag bit3 */
int mpk_fused_prof_read(uint64_t *out, int32_t nctas);

#ifdef __cplusplus
}
#endif
#endif /* MPK_B200_H */
