// Device kernels of the GMRES solve path (sm_100a, HBM-bound; no tensor
// cores: SpMV is ~0.17 flop/B and the CGS2 skinny GEMVs ~0.25 flop/B).
//
// Per Arnoldi step the reference does (gmres.py:180-193, kernels.py:114-126):
//   z = M v_k; w = A z; ||w||; c1 = V^T w; w -= V c1; c2 = V^T w; w -= V c2;
//   beta = ||w||; append w/beta; Givens update.
// Here that is three streaming passes over the basis, each ending in a
// deterministic grid reduction finished by the last CTA:
//   P1 k_spmv_dot     v_k = w''/beta (fused normalise), w = A v_k, ||w||^2, V^T w
//   P2 k_update_dot   w' = w - V c1, V^T w'
//   P3 k_update_norm  w'' = w' - V c2, ||w''||^2, then (last CTA) beta, the
//                     append test and the Givens update of the Hessenberg column
// The basis V is column-major with leading dimension ld (multiple of 64), so
// every column read by a warp is one contiguous, aligned 128/256-byte line.
#pragma once

#include "ops.cuh"

namespace mpk {

constexpr int kStride = kMaxCols + 2;   // partial-row stride (columns + extra)

// sums[] layout (elements of T)
enum : int {
    S_C1 = 0,
    S_C2 = MPK_MAX_STEPS + 8,
    S_WN2 = 2 * (MPK_MAX_STEPS + 8),
    S_BN2,
    S_BETA,
    S_GAMMA,
    S_RN2,
    S_APP,
    S_TMP,
    S_TOTAL = S_TMP + 2 * kStride
};

template <typename T> struct Hess {
    T *h;    // (m+1) x m, column-major
    T *cs;   // m
    T *sn;   // m
    T *g;    // m+1
    T *d;    // m   (back-substitution result)
    T *raw;  // (m+1) x m unrotated columns (coeffs, beta) for diagnostics
    int m;
};

__device__ __forceinline__ bool skip(const int32_t *done) {
    return done != nullptr && *(volatile const int32_t *)done != 0;
}

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

// Row loop of an SpMV-carrying kernel.  Stencils: 16-byte row groups per
// thread (GROUPS) or thread per row, grid-strided.  CSR: 32-row groups per warp, grid-strided over groups, each
// evaluated by CsrOp::warp_rows (coalesced entry loads, bit-identical sums);
// fn(r, y_r) runs on the lane owning row r.  `sb` is the warp's staging.
template <typename T, class Op, class X, class F, bool GROUPS = true>
__device__ __forceinline__ void for_rows(const Op &A, X x, T *sb, F &&fn) {
    if constexpr (Op::kStencil) {
        constexpr int R = 16 / (int)sizeof(T);
        if (GROUPS && A.group_ok() && ((uintptr_t)x.p % 16) == 0) {
            // 16-byte row groups (vector reads of the group and its N/S/B/U
            // neighbours), bit-identical to row(); scalar tail past n - n % R
            const int64_t ng = A.n / R;
            auto xv = [&](int64_t c) { return x.vec(c); };
            // one group per thread per trip: two in flight raised the
            // standalone kernel to 114 registers (BentPipe's double
            // coefficient arithmetic) and halved its occupancy
            const int64_t st = gstride();
            int64_t gi = gtid();
            for (; gi < ng; gi += st) {
                T o[R];
                A.row_group(gi * R, xv, x, o);
#pragma unroll
                for (int e = 0; e < R; ++e) fn(gi * R + e, o[e]);
            }
            for (int64_t r = ng * R + gtid(); r < A.n; r += gstride()) fn(r, A.row(r, x));
        } else {
            for (int64_t r = gtid(); r < A.n; r += gstride()) fn(r, A.row(r, x));
        }
    } else {
        const int lane = threadIdx.x & 31;
        const int64_t gw = gtid() >> 5, nw = gstride() >> 5;
        for (int64_t r0 = gw * 32; r0 < A.n; r0 += nw * 32) {
            const T y = A.warp_rows(r0, A.n, x, sb);
            if (r0 + lane < A.n) fn(r0 + lane, y);
        }
    }
}

// ---------------------------------------------------------------------------
// P1: (normalise) + SpMV + ||w||^2 + first projection V^T w
// ---------------------------------------------------------------------------
template <typename T, int NC, class Op, bool NORM>
__global__ void __launch_bounds__(kBlock) k_spmv_dot(Op A, const T *__restrict__ src,
                                                     const T *__restrict__ divp, T *__restrict__ vcol,
                                                     const T *__restrict__ V, int64_t ld, int ndot,
                                                     T *__restrict__ w, T *partials, unsigned *counter,
                                                     T *out, T *out_wn2, const int32_t *done) {
    __shared__ T sm[(kBlock / 32) * (NC + 1)];
    if (skip(done)) return;
    const T dv = NORM ? *divp : T(1);
    T acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = T(0);
    T an = T(0);
    __shared__ T sbuf[Op::kStencil ? 1 : (kBlock / 32) * kCsrWarpBuf];
    T *sb = sbuf + (Op::kStencil ? 0 : (threadIdx.x >> 5) * kCsrWarpBuf);
    auto body = [&](int64_t r, T wr) {
        T own = T(0);
        if constexpr (NORM) {
            own = RN<T>::div(src[r], dv);
            vcol[r] = own;
        }
        w[r] = wr;
        an += wr * wr;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (c < ndot) {
                const T v = (NORM && c == ndot - 1) ? own : V[(int64_t)c * ld + r];
                acc[c] += v * wr;
            }
        }
    };
    if constexpr (NORM) {
        for_rows<T>(A, XScaled<T>{src, dv}, sb, body);
    } else {
        for_rows<T>(A, XPlain<T>{src}, sb, body);
    }
    block_reduce_cols<T, NC>(acc, ndot, an, sm, partials + (int64_t)blockIdx.x * kStride);
    if (last_cta(counter)) {
        reduce_partials<T, NC>(partials, gridDim.x, kStride, ndot, sm, out);
        if (threadIdx.x == 0) {
            *out_wn2 = out[ndot];
            *counter = 0u;
        }
    }
}

// ---------------------------------------------------------------------------
// P2: w' = w - V c ; V^T w'   (row of V staged in shared memory, reused)
// ---------------------------------------------------------------------------
template <typename T, int NC>
__global__ void __launch_bounds__(kBlock) k_update_dot(int64_t n, const T *__restrict__ V, int64_t ld,
                                                       int ncols, const T *__restrict__ coef,
                                                       const T *__restrict__ w, T *__restrict__ wout,
                                                       T *partials, unsigned *counter, T *out,
                                                       const int32_t *done) {
    extern __shared__ unsigned char dsm_raw[];
    T *stage = reinterpret_cast<T *>(dsm_raw);
    __shared__ T sm[(kBlock / 32) * (NC + 1)];
    __shared__ T sc[NC];
    if (skip(done)) return;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) sc[c] = coef[c];
    __syncthreads();
    T acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = T(0);
    const int t = threadIdx.x;
    for (int64_t r = gtid(); r < n; r += gstride()) {
        T s = T(0);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (c < ncols) {
                const T v = V[(int64_t)c * ld + r];
                stage[c * kBlock + t] = v;
                s += v * sc[c];
            }
        }
        const T wr = RN<T>::sub(w[r], s);
        wout[r] = wr;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c < ncols) acc[c] += stage[c * kBlock + t] * wr;
    }
    block_reduce_cols<T, NC>(acc, ncols, T(0), sm, partials + (int64_t)blockIdx.x * kStride);
    if (last_cta(counter)) {
        reduce_partials<T, NC>(partials, gridDim.x, kStride, ncols, sm, out);
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// Plain multi-dot out[c] = V[:, c0+c]^T w for a chunk of <= NC columns
// (used past kMaxCols columns and by the standalone cgs2 entry point).
template <typename T, int NC>
__global__ void __launch_bounds__(kBlock) k_multidot(int64_t n, const T *__restrict__ V, int64_t ld,
                                                     int ncols, const T *__restrict__ w, T *partials,
                                                     unsigned *counter, T *out, const int32_t *done) {
    __shared__ T sm[(kBlock / 32) * (NC + 1)];
    if (skip(done)) return;
    T acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = T(0);
    T an = T(0);
    for (int64_t r = gtid(); r < n; r += gstride()) {
        const T wr = w[r];
        an += wr * wr;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c < ncols) acc[c] += V[(int64_t)c * ld + r] * wr;
    }
    block_reduce_cols<T, NC>(acc, ncols, an, sm, partials + (int64_t)blockIdx.x * kStride);
    if (last_cta(counter)) {
        reduce_partials<T, NC>(partials, gridDim.x, kStride, ncols, sm, out);
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// ---------------------------------------------------------------------------
// Hessenberg / Givens (kernels.py:129-196) on one CTA
// ---------------------------------------------------------------------------
struct StepParams {
    int k;              // 0-based step index; column j = k + 1
    int steps_cap;
    double thresh_factor;   // n*u (rule n_u) or u (rule u)
    double exit_tol;
    int test_append;        // 0: standalone update (no append test, no exit)
};

// Executed by a whole CTA.  Reads c1, c2, beta (sums[S_BETA]) and ||w||^2,
// writes the rotated column to H and the step outcome to ctl.  Thread 0 runs
// the serial rotation chain with the column in shared memory.
template <typename T>
__device__ void hessenberg_step(T *sums, Hess<T> H, mpk_cycle_ctl *ctl, const StepParams p) {
    extern __shared__ unsigned char dsm_raw[];
    T *col = reinterpret_cast<T *>(dsm_raw);     // m+1
    T *scs = col + (H.m + 1);                    // m
    T *ssn = scs + H.m;                          // m
    __shared__ int s_app;
    const int j = p.k + 1;
    const T beta = sums[S_BETA];
    for (int i = threadIdx.x; i < j; i += blockDim.x) {
        col[i] = RN<T>::add(sums[S_C1 + i], sums[S_C2 + i]);
        if (i < j - 1) {
            scs[i] = H.cs[i];
            ssn[i] = H.sn[i];
        }
    }
    T *rc = H.raw + (int64_t)(j - 1) * (H.m + 1);
    for (int i = threadIdx.x; i < j; i += blockDim.x) rc[i] = col[i];
    if (threadIdx.x == 0) {
        rc[j] = beta;
        col[j] = beta;
        if (p.test_append) {
            const T wnorm = RN<T>::sqrt_(sums[S_WN2]);
            const double thr = p.thresh_factor * (double)wnorm;   // kernels.py:122-123
            s_app = ((double)beta > thr) ? 1 : 0;
        } else {
            s_app = 1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        T carry = col[0];
        for (int i = 0; i < j - 1; ++i) {
            const T a = carry, b = col[i + 1];
            const T c = scs[i], s = ssn[i];
            col[i] = RN<T>::add(RN<T>::mul(c, a), RN<T>::mul(s, b));
            carry = RN<T>::add(RN<T>::mul(-s, a), RN<T>::mul(c, b));
        }
        const T a = carry, b = col[j];
        T c, s, r;
        if (b == T(0)) {
            c = T(1); s = T(0); r = a;
        } else {
            r = RN<T>::hypot_(a, b);
            c = RN<T>::div(a, r);
            s = RN<T>::div(b, r);
        }
        H.cs[j - 1] = c;
        H.sn[j - 1] = s;
        col[j - 1] = r;
        col[j] = T(0);
        const T gprev = H.g[j - 1];
        const T gj = RN<T>::mul(-s, gprev);
        H.g[j] = gj;
        H.g[j - 1] = RN<T>::mul(c, gprev);
        const double rel = fabs((double)gj) / ctl->scale;
        ctl->implicit_relres[p.k] = rel;
        ctl->steps = j;
        if (p.test_append) {
            if (!s_app) {
                ctl->breakdown = 1;
                ctl->done = 1;
            } else if (rel <= p.exit_tol || j >= p.steps_cap) {
                ctl->done = 1;
            }
        }
    }
    __syncthreads();
    T *hc = H.h + (int64_t)(j - 1) * (H.m + 1);
    for (int i = threadIdx.x; i <= j; i += blockDim.x) hc[i] = col[i];
}

// ---------------------------------------------------------------------------
// P3: w'' = w' - V c ; ||w''||^2 ; last CTA: beta, append test, Givens
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kBlock) k_update_norm(int64_t n, const T *__restrict__ V, int64_t ld,
                                                        int ncols, const T *__restrict__ coef,
                                                        const T *__restrict__ w, T *__restrict__ wout,
                                                        T *partials, unsigned *counter, T *sums,
                                                        Hess<T> H, mpk_cycle_ctl *ctl, StepParams p,
                                                        int do_givens, const int32_t *done) {
    extern __shared__ unsigned char dsm_raw[];
    T *sc = reinterpret_cast<T *>(dsm_raw);      // ncols (reused by the Givens step)
    __shared__ T sm[(kBlock / 32) * 2];
    if (skip(done)) return;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) sc[c] = coef[c];
    __syncthreads();
    T an = T(0);
    for (int64_t r = gtid(); r < n; r += gstride()) {
        T s = T(0);
        int c = 0;
        for (; c + 8 <= ncols; c += 8) {
            T v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = V[(int64_t)(c + q) * ld + r];
#pragma unroll
            for (int q = 0; q < 8; ++q) s += v[q] * sc[c + q];
        }
        for (; c < ncols; ++c) s += V[(int64_t)c * ld + r] * sc[c];
        const T wr = RN<T>::sub(w[r], s);
        wout[r] = wr;
        an += wr * wr;
    }
    T dummy[1] = {T(0)};
    block_reduce_cols<T, 1>(dummy, 0, an, sm, partials + (int64_t)blockIdx.x * kStride);
    if (last_cta(counter)) {
        reduce_partials<T, 1>(partials, gridDim.x, kStride, 0, sm, sums + S_BN2);
        if (threadIdx.x == 0) {
            *counter = 0u;
            sums[S_BETA] = RN<T>::sqrt_(sums[S_BN2]);   // beta = norm2(w'') in T
        }
        __syncthreads();
        if (do_givens) hessenberg_step<T>(sums, H, ctl, p);
    }
}

// ---------------------------------------------------------------------------
// cycle prologue / epilogue
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_cycle_begin(const T *rnorm2, T *sums, Hess<T> H, mpk_cycle_ctl *ctl,
                              double norm_scale) {
    if (threadIdx.x != 0) return;
    const T gamma = RN<T>::sqrt_(*rnorm2);
    sums[S_GAMMA] = gamma;
    H.g[0] = gamma;
    ctl->gamma = (double)gamma;
    double scale = norm_scale > 0.0 ? norm_scale : (double)gamma;
    ctl->steps = 0;
    ctl->breakdown = 0;
    ctl->tri_err = 0;
    ctl->done = (gamma == T(0)) ? 1 : 0;
    if (gamma == T(0) && !(scale > 0.0)) scale = 1.0;   // gmres.py:170-172
    ctl->scale = scale;
}

// normalise: vcol = src / d (kernels.py:125 / gmres.py:174)
template <typename T>
__global__ void k_normalize(int64_t n, const T *__restrict__ src, const T *divp, T *__restrict__ vcol,
                            const int32_t *done) {
    if (skip(done)) return;
    const T d = *divp;
    for (int64_t r = gtid(); r < n; r += gstride()) vcol[r] = RN<T>::div(src[r], d);
}

// Back-substitution R d = g with the k*u*max|diag| guard (kernels.py:202-216).
// One warp.  k = ctl->steps.
template <typename T>
__global__ void k_lsq_solve(Hess<T> H, mpk_cycle_ctl *ctl, double u, int kfixed) {
    extern __shared__ unsigned char dsm_raw[];
    T *rhs = reinterpret_cast<T *>(dsm_raw);
    __shared__ T s_d;
    const int k = kfixed > 0 ? kfixed : ctl->steps;
    if (k <= 0 || ctl->tri_err) return;
    const int ldh = H.m + 1;
    if (threadIdx.x == 0) {
        T dmax = fabs(H.h[0]), dmin = dmax;
        int imin = 0;
        for (int i = 1; i < k; ++i) {
            const T a = fabs(H.h[(int64_t)i * ldh + i]);
            if (a > dmax) dmax = a;
            if (a < dmin) { dmin = a; imin = i; }     // np.argmin: first minimum
        }
        const double thr = (double)k * u * (double)dmax;
        if ((double)dmin <= thr) {
            ctl->tri_err = 1;
            ctl->tri_index = imin;
            ctl->tri_entry = (double)dmin;
            ctl->tri_threshold = thr;
        }
    }
    __syncwarp();
    if (*(volatile int32_t *)&ctl->tri_err) return;
    for (int i = threadIdx.x; i < k; i += 32) rhs[i] = H.g[i];
    __syncwarp();
    for (int i = k - 1; i >= 0; --i) {
        if (threadIdx.x == 0) {
            s_d = RN<T>::div(rhs[i], H.h[(int64_t)i * ldh + i]);
            H.d[i] = s_d;
        }
        __syncwarp();
        const T di = s_d;
        for (int q = threadIdx.x; q < i; q += 32) rhs[q] = rhs[q] - H.h[(int64_t)i * ldh + q] * di;
        __syncwarp();
    }
}

// x_out = x0 + V[:, :k] d   (mode 0)      or   y = V[:, :k] d   (mode 1)
// gmres.py:195-196.  k = ctl->steps; k == 0 copies x0.
template <typename T>
__global__ void __launch_bounds__(kBlock) k_correct(int64_t n, const T *__restrict__ V, int64_t ld,
                                                    const T *__restrict__ dvec, const T *__restrict__ x0,
                                                    T *__restrict__ out, const mpk_cycle_ctl *ctl,
                                                    int mode) {
    extern __shared__ unsigned char dsm_raw[];
    T *sd = reinterpret_cast<T *>(dsm_raw);
    if (ctl->tri_err) return;
    const int k = ctl->steps;
    for (int c = threadIdx.x; c < k; c += blockDim.x) sd[c] = dvec[c];
    __syncthreads();
    for (int64_t r = gtid(); r < n; r += gstride()) {
        T s = T(0);
        int c = 0;
        for (; c + 8 <= k; c += 8) {
            T v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = V[(int64_t)(c + q) * ld + r];
#pragma unroll
            for (int q = 0; q < 8; ++q) s += v[q] * sd[c + q];
        }
        for (; c < k; ++c) s += V[(int64_t)c * ld + r] * sd[c];
        if (mode == 0)
            out[r] = (k == 0) ? x0[r] : RN<T>::add(x0[r], s);
        else
            out[r] = s;
    }
}

// Diagnostics (collect_basis): write the last appended column
// V[:, steps] = w'' / beta, which the fused cycle otherwise leaves to the
// next step's P1 (gmres.py:198-199 returns basis.count columns).
template <typename T>
__global__ void k_final_column(int64_t n, const T *__restrict__ wpp, const T *betap, T *V, int64_t ld,
                               const mpk_cycle_ctl *ctl) {
    if (ctl->breakdown || ctl->steps <= 0) return;
    T *col = V + (int64_t)ctl->steps * ld;
    const T b = *betap;
    for (int64_t r = gtid(); r < n; r += gstride()) col[r] = RN<T>::div(wpp[r], b);
}

// out = x0 + z  (the preconditioned correction, gmres.py:196); ctl gates it
template <typename T>
__global__ void k_add_gated(int64_t n, const T *__restrict__ x0, const T *__restrict__ z,
                            T *__restrict__ out, const mpk_cycle_ctl *ctl) {
    if (ctl->tri_err) return;
    const int k = ctl->steps;
    for (int64_t r = gtid(); r < n; r += gstride()) out[r] = (k == 0) ? x0[r] : RN<T>::add(x0[r], z[r]);
}

// ---------------------------------------------------------------------------
// explicit residual r = b - A x (+ fp32 copy for refinement)
// ---------------------------------------------------------------------------
template <typename T, class Op, bool LOW>
__global__ void __launch_bounds__(kBlock) k_residual(Op A, const T *__restrict__ b, const T *__restrict__ x,
                                                     T *__restrict__ r, float *__restrict__ rlow,
                                                     T *partials, float *partials_low, unsigned *counter,
                                                     T *out, float *out_low) {
    __shared__ T sm[(kBlock / 32) * 2];
    __shared__ float smf[(kBlock / 32) * 2];
    T an = T(0);
    float al = 0.f;
    __shared__ T sbuf[Op::kStencil ? 1 : (kBlock / 32) * kCsrWarpBuf];
    T *sb = sbuf + (Op::kStencil ? 0 : (threadIdx.x >> 5) * kCsrWarpBuf);
    // thread per row: the order of the r.r partial sums fixes the refinement
    // trajectory of GMRES-IR (kept as measured against the reference counts)
    auto body = [&](int64_t i, T ax) {
        const T ri = RN<T>::sub(b[i], ax);
        if (r) r[i] = ri;
        an += ri * ri;
        if constexpr (LOW) {
            const float li = __double2float_rn((double)ri);
            rlow[i] = li;
            al += li * li;
        }
    };
    for_rows<T, Op, XPlain<T>, decltype(body) &, false>(A, XPlain<T>{x}, sb, body);
    T d1[1] = {T(0)};
    block_reduce_cols<T, 1>(d1, 0, an, sm, partials + (int64_t)blockIdx.x * kStride);
    if constexpr (LOW) {
        float d2[1] = {0.f};
        block_reduce_cols<float, 1>(d2, 0, al, smf, partials_low + (int64_t)blockIdx.x * 2);
    }
    if (last_cta(counter)) {
        reduce_partials<T, 1>(partials, gridDim.x, kStride, 0, sm, out);
        if constexpr (LOW) reduce_partials<float, 1>(partials_low, gridDim.x, 2, 0, smf, out_low);
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// x_next = x + (double) u ; changed |= (x_next != x)   (multiprecision.py:207-214)
__global__ void k_ir_update(int64_t n, double *__restrict__ x, const float *__restrict__ u,
                            int32_t *changed) {
    bool any = false;
    for (int64_t i = gtid(); i < n; i += gstride()) {
        const double xo = x[i];
        const double xn = __dadd_rn(xo, (double)u[i]);
        any |= !(xn == xo);
        x[i] = xn;
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(changed, 1);
}

// ---------------------------------------------------------------------------
// standalone vector kernels (kernels.py:31-52, sparse.py:190-226)
// ---------------------------------------------------------------------------
template <typename T, class Op>
__global__ void __launch_bounds__(kBlock) k_spmv(Op A, const T *__restrict__ x, T *__restrict__ y) {
    __shared__ T sbuf[Op::kStencil ? 1 : (kBlock / 32) * kCsrWarpBuf];
    T *sb = sbuf + (Op::kStencil ? 0 : (threadIdx.x >> 5) * kCsrWarpBuf);
    for_rows<T>(A, XPlain<T>{x}, sb, [&](int64_t r, T yr) { y[r] = yr; });
}

// Stencil presets in 16-byte row groups with the preset fixed at compile
// time: PRESET is written into a local copy of the operator, so the other
// presets' branches fold away (BentPipe's double coefficient arithmetic sets
// k_spmv's register count for every preset), and UG groups per thread per
// trip with every group's loads issued before any is evaluated.  Same
// per-row sums as row() (group_eval == row()).  Needs group_ok() and 16-byte
// aligned x / y; the host checks both.
template <typename T, int PRESET, int UG>
__global__ void __launch_bounds__(kBlock) k_spmv_pre(StencilOp<T> A, const T *__restrict__ x, T *__restrict__ y) {
    constexpr int R = 16 / (int)sizeof(T);
    StencilOp<T> B = A;
    B.k.preset = PRESET;
    const XPlain<T> xs{x};
    auto xv = [&](int64_t c) { return xs.vec(c); };
    const int64_t ng = B.n / R, st = gstride();
    int64_t gi = gtid();
    for (; gi + (UG - 1) * st < ng; gi += UG * st) {
        typename StencilOp<T>::GroupIn in[UG];
#pragma unroll
        for (int u = 0; u < UG; ++u) B.group_load((gi + u * st) * R, xv, xs, in[u]);
#pragma unroll
        for (int u = 0; u < UG; ++u) {
            Pack<T> o;
            B.group_eval((gi + u * st) * R, in[u], o.v);
            *reinterpret_cast<Pack<T> *>(y + (gi + u * st) * R) = o;
        }
    }
    for (; gi < ng; gi += st) {
        Pack<T> o;
        B.row_group(gi * R, xv, xs, o.v);
        *reinterpret_cast<Pack<T> *>(y + gi * R) = o;
    }
    for (int64_t r = ng * R + gtid(); r < B.n; r += st) y[r] = B.row(r, xs);
}

// Short CSR rows (<= 8 stored entries on average, e.g. the stencils in CSR
// form): thread per row.  A warp's 32 rows cover one contiguous run of
// entries, so each of a row's entry loads is coalesced across the warp and
// its x gathers hit L1; no shared-memory staging.  Two rows per thread
// keep two rows' loads in flight.  Same row sums as row() (csr_matvec).
template <typename T>
__global__ void __launch_bounds__(kBlock) k_spmv_rows(CsrOp<T> A, const T *__restrict__ x, T *__restrict__ y) {
    const XPlain<T> xs{x};
    const int64_t st = gstride();
    int64_t r = gtid();
    for (; r + st < A.n; r += 2 * st) {
        const T y0 = A.row(r, xs), y1 = A.row(r + st, xs);
        y[r] = y0;
        y[r + st] = y1;
    }
    for (; r < A.n; r += st) y[r] = A.row(r, xs);
}

// Banded CSR (A.band > 0): chunks of kSpmvChunk rows per CTA, x staged in a
// shared-memory window per chunk (csr_chunk), K entries per lane in flight.
constexpr int kSpmvChunk = 1024;
// (ncu, config 5: K = 16 took 97 / 164 registers and capped occupancy at
// 25% / 12.5%; the bounds below keep 4 / 3 CTAs per SM)
template <typename T, int K>
__global__ void __launch_bounds__(kBlock, sizeof(T) == 4 ? 4 : 3)
    k_spmv_win(CsrOp<T> A, const T *__restrict__ x, T *__restrict__ y) {
    extern __shared__ __align__(16) unsigned char dsm_win[];
    __shared__ T sbuf[(kBlock / 32) * kCsrWarpBuf];
    T *sx = reinterpret_cast<T *>(dsm_win);
    T *sb = sbuf + (threadIdx.x >> 5) * kCsrWarpBuf;
    for (int64_t R = (int64_t)blockIdx.x * kSpmvChunk; R < A.n; R += (int64_t)gridDim.x * kSpmvChunk) {
        const int64_t Re = R + kSpmvChunk < A.n ? R + kSpmvChunk : A.n;
        csr_chunk<K>(A, XPlain<T>{x}, R, Re, sx, sb, [&](int64_t r, T yr) { y[r] = yr; });
    }
}

template <typename S, typename D>
__global__ void k_convert(int64_t n, const S *__restrict__ s, D *__restrict__ d) {
    for (int64_t i = gtid(); i < n; i += gstride()) {
        if constexpr (sizeof(D) == 4 && sizeof(S) == 8)
            d[i] = __double2float_rn(s[i]);
        else
            d[i] = (D)s[i];
    }
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_dot(int64_t n, const T *__restrict__ x, const T *__restrict__ y,
                                                T *partials, unsigned *counter, T *out, int take_sqrt) {
    __shared__ T sm[(kBlock / 32) * 2];
    T a = T(0);
    for (int64_t i = gtid(); i < n; i += gstride()) a += x[i] * y[i];
    T d1[1] = {T(0)};
    block_reduce_cols<T, 1>(d1, 0, a, sm, partials + (int64_t)blockIdx.x * kStride);
    if (last_cta(counter)) {
        reduce_partials<T, 1>(partials, gridDim.x, kStride, 0, sm, out);
        if (threadIdx.x == 0) {
            if (take_sqrt) out[0] = RN<T>::sqrt_(out[0]);
            *counter = 0u;
        }
    }
}

template <typename T>
__global__ void k_axpy(int64_t n, T a, const T *__restrict__ x, const T *__restrict__ y, T *__restrict__ out) {
    for (int64_t i = gtid(); i < n; i += gstride())
        out[i] = y ? RN<T>::add(y[i], RN<T>::mul(a, x[i])) : RN<T>::mul(a, x[i]);
}

// standalone cgs2_append epilogue: coeffs = c1 + c2, beta, append test and
// the new column w''/beta when appended (kernels.py:121-126)
template <typename T>
__global__ void k_cgs2_finish(int64_t n, const T *sums, int count, double thresh_factor,
                              const T *__restrict__ wpp, T *__restrict__ vnew, T *coeffs, T *out,
                              int32_t *appended) {
    const T beta = RN<T>::sqrt_(sums[S_BN2]);
    const T wnorm = RN<T>::sqrt_(sums[S_WN2]);
    const bool app = (double)beta > thresh_factor * (double)wnorm;
    if (blockIdx.x == 0) {
        for (int c = threadIdx.x; c < count; c += blockDim.x)
            coeffs[c] = RN<T>::add(sums[S_C1 + c], sums[S_C2 + c]);
        if (threadIdx.x == 0) {
            out[0] = beta;
            out[1] = wnorm;
            *appended = app ? 1 : 0;
        }
    }
    if (!app) return;
    for (int64_t r = gtid(); r < n; r += gstride()) vnew[r] = RN<T>::div(wpp[r], beta);
}

// ---------------------------------------------------------------------------
// preconditioners (preconditioners.py:133-139, 276-305)
// ---------------------------------------------------------------------------
// Block Jacobi: one thread per k-by-k block; getrs order: row swaps (piv,
// sequential as dlaswp), unit-lower forward, upper backward.
template <typename T, int KMAX>
__global__ void k_jacobi(int64_t n, int k, const T *__restrict__ lu, const int32_t *__restrict__ piv,
                         const T *__restrict__ v, T *__restrict__ out, const int32_t *done) {
    if (skip(done)) return;
    const int64_t nb = (n + k - 1) / k;
    for (int64_t b = gtid(); b < nb; b += gstride()) {
        const int64_t s = b * k;
        const int kb = (int)((s + k <= n) ? k : (n - s));
        if (k == 1) {
            out[s] = RN<T>::div(v[s], lu[b]);
            continue;
        }
        const T *L = lu + b * (int64_t)k * k;   // row-major kb x kb (leading dim k)
        const int32_t *P = piv + b * (int64_t)k;
        T xb[KMAX];
        for (int i = 0; i < kb; ++i) xb[i] = v[s + i];
        for (int i = 0; i < kb; ++i) {
            const int p = P[i];
            if (p != i) { const T t = xb[i]; xb[i] = xb[p]; xb[p] = t; }
        }
        for (int i = 1; i < kb; ++i) {
            T a = xb[i];
            for (int j = 0; j < i; ++j) a -= L[i * k + j] * xb[j];
            xb[i] = a;
        }
        for (int i = kb - 1; i >= 0; --i) {
            T a = xb[i];
            for (int j = i + 1; j < kb; ++j) a -= L[i * k + j] * xb[j];
            xb[i] = RN<T>::div(a, L[i * k + i]);
        }
        for (int i = 0; i < kb; ++i) out[s + i] = xb[i];
    }
}

// ---------------------------------------------------------------------------
// Block-Jacobi setup on the device (preconditioners.py:96-130): dense k x k
// diagonal blocks of a CSR matrix, LU with partial pivoting, pivot test.
// ---------------------------------------------------------------------------
// numpy's pairwise sum of n contiguous |a_i| (np.abs(block).sum(axis=1) of
// the reference's threshold, preconditioners.py:120): 8 strided
// accumulators for n >= 8, combined ((0+1)+(2+3))+((4+5)+(6+7)), then the
// remainder; sequential from -0.0 below 8 (checked bit-exact against numpy).
template <typename T> __device__ T np_abs_pairwise(const T *a, int n) {
    if (n < 8) {
        T r = T(-0.0);
        for (int i = 0; i < n; ++i) r = RN<T>::add(r, fabs(a[i]));
        return r;
    }
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = fabs(a[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = RN<T>::add(r[j], fabs(a[i + j]));
    T res = RN<T>::add(RN<T>::add(RN<T>::add(r[0], r[1]), RN<T>::add(r[2], r[3])),
                       RN<T>::add(RN<T>::add(r[4], r[5]), RN<T>::add(r[6], r[7])));
    for (; i < n; ++i) res = RN<T>::add(res, fabs(a[i]));
    return res;
}

// One warp per block b (rows/columns [b*k, b*k + kb)), the block in shared
// memory (kb x kb, row-major).  Right-looking LU with partial pivoting in T:
// pivot = first row of maximal |a_ij| (LAPACK i?amax), full-row swap, the
// column below scaled by the reciprocal pivot (getf2 for |pivot| >= the
// smallest normal, division otherwise), rank-1 update of the trailing block.
// Output in the apply kernel's layout: lu[b][i][j] (stride k), piv[b*k + i]
// 0-based (scipy lu_factor).  minpiv[b] = min |u_ii|, thr[b] =
// (kb*u)*max row sum (double, as the reference's Python arithmetic);
// *bad = lowest failing block (atomicMin; the caller initialises INT32_MAX).
// The factors agree with LAPACK's to rounding, not bit for bit (OpenBLAS
// getrf is left-looking/recursive with FMA kernels).
constexpr int kLuWarps = 4;
template <typename T>
__global__ void __launch_bounds__(kLuWarps * 32) k_block_lu(CsrOp<T> A, int k, double u, T *__restrict__ lu,
                                                           int32_t *__restrict__ piv, T *__restrict__ minpiv,
                                                           double *__restrict__ thr, int32_t *bad) {
    extern __shared__ __align__(16) unsigned char dsm_lu[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    T *S = reinterpret_cast<T *>(dsm_lu) + (size_t)wib * k * k;
    const int64_t nb = (A.n + k - 1) / k;
    const T tiny = sizeof(T) == 8 ? T(2.2250738585072014e-308) : T(1.17549435e-38f);
    for (int64_t b = (int64_t)blockIdx.x * kLuWarps + wib; b < nb; b += (int64_t)gridDim.x * kLuWarps) {
        const int64_t s = b * k;
        const int kb = (int)(A.n - s < k ? A.n - s : k);
        for (int i = lane; i < kb * kb; i += 32) S[i] = T(0);
        __syncwarp();
        for (int i = lane; i < kb; i += 32) {
            const int32_t p0 = A.rp[s + i], p1 = A.rp[s + i + 1];
            for (int32_t p = p0; p < p1; ++p) {
                const int64_t c = A.ci[p];
                if (c >= s && c < s + kb) S[i * kb + (int)(c - s)] = A.v[p];
            }
        }
        __syncwarp();
        T rmax = T(0);
        for (int i = lane; i < kb; i += 32) rmax = fmax(rmax, np_abs_pairwise(S + i * kb, kb));
        for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        const double th = __dmul_rn(__dmul_rn((double)kb, u), (double)rmax);
        for (int j = 0; j < kb; ++j) {
            T best = T(-1);
            int bi = kb;
            for (int i = j + lane; i < kb; i += 32) {
                const T a = fabs(S[i * kb + j]);
                if (a > best) {
                    best = a;
                    bi = i;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const T ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            const int p = bi < kb ? bi : j;
            if (lane == 0) piv[b * k + j] = p;
            if (p != j)
                for (int l = lane; l < kb; l += 32) {
                    const T t = S[j * kb + l];
                    S[j * kb + l] = S[p * kb + l];
                    S[p * kb + l] = t;
                }
            __syncwarp();
            const T d = S[j * kb + j];
            if (d != T(0)) {
                const bool recip = fabs(d) >= tiny;
                const T r = RN<T>::div(T(1), d);
                for (int i = j + 1 + lane; i < kb; i += 32)
                    S[i * kb + j] = recip ? RN<T>::mul(S[i * kb + j], r) : RN<T>::div(S[i * kb + j], d);
            }
            __syncwarp();
            for (int i = j + 1 + lane; i < kb; i += 32) {
                const T lij = S[i * kb + j];
                for (int l = j + 1; l < kb; ++l) S[i * kb + l] = fma(-lij, S[j * kb + l], S[i * kb + l]);
            }
            __syncwarp();
        }
        T mp = T(INFINITY);
        for (int i = lane; i < kb; i += 32) mp = fmin(mp, fabs(S[i * kb + i]));
        for (int o = 16; o; o >>= 1) mp = fmin(mp, __shfl_xor_sync(0xffffffffu, mp, o));
        T *L = lu + (size_t)b * k * k;
        for (int e = lane; e < k * k; e += 32) {
            const int i = e / k, l = e % k;
            L[e] = (i < kb && l < kb) ? S[i * kb + l] : T(0);
        }
        for (int i = kb + lane; i < k; i += 32) piv[b * k + i] = i;
        if (lane == 0) {
            minpiv[b] = mp;
            thr[b] = th;
            if (!((double)mp > th)) atomicMin(bad, (int32_t)b);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Stencil assembly on the device (generate_stencil, stencils.py:192-207):
// per-row entry counts, an exclusive scan to row_ptr (int64), then each row's
// (column, value) pairs in the reference's order -- bit-identical arrays.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kBlock) k_stencil_count(StencilOp<T> A, int32_t *__restrict__ cnt) {
    for (int64_t r = gtid(); r < A.n; r += gstride()) cnt[r] = A.row_entries(r, [](int64_t, T) {});
}

constexpr int kScanThreads = 1024, kScanPer = 8, kScanChunk = kScanThreads * kScanPer;
// rp[i + 1] = cnt[0] + ... + cnt[i] within each kScanChunk block; bsum[b] = block total
__global__ void __launch_bounds__(kScanThreads) k_scan_local(const int32_t *__restrict__ cnt, int64_t n,
                                                             int64_t *__restrict__ rp, int64_t *__restrict__ bsum) {
    __shared__ int64_t sw[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kScanPer;
    int64_t v[kScanPer];
    int64_t run = 0;
#pragma unroll
    for (int e = 0; e < kScanPer; ++e) {
        run += (base + e < n) ? cnt[base + e] : 0;
        v[e] = run;
    }
    // exclusive scan of the per-thread totals over the block
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = run;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = sw[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sw[lane] = w;
    }
    __syncthreads();
    const int64_t off = (x - run) + (warp ? sw[warp - 1] : 0);
#pragma unroll
    for (int e = 0; e < kScanPer; ++e)
        if (base + e < n) rp[base + e + 1] = v[e] + off;
    if (threadIdx.x == kScanThreads - 1) bsum[blockIdx.x] = off + run;
}

// one block: exclusive prefix of the block totals (sequential per thread
// over a strided slice, then a block scan), then the offsets are added
__global__ void __launch_bounds__(kScanThreads) k_scan_blocks(int64_t *bsum, int64_t nb) {
    __shared__ int64_t sw[kScanThreads / 32];
    const int64_t per = (nb + kScanThreads - 1) / kScanThreads;
    const int64_t b0 = (int64_t)threadIdx.x * per;
    int64_t run = 0;
    for (int64_t b = b0; b < b0 + per && b < nb; ++b) run += bsum[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = run;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = sw[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sw[lane] = w;
    }
    __syncthreads();
    int64_t acc = (x - run) + (warp ? sw[warp - 1] : 0);
    for (int64_t b = b0; b < b0 + per && b < nb; ++b) {
        const int64_t t = bsum[b];
        bsum[b] = acc;   // exclusive offset of block b
        acc += t;
    }
}

__global__ void k_scan_add(int64_t *__restrict__ rp, int64_t n, const int64_t *__restrict__ boff) {
    for (int64_t i = gtid(); i < n; i += gstride()) rp[i + 1] += boff[i / kScanChunk];
    if (gtid() == 0) rp[0] = 0;
}

template <typename T>
__global__ void __launch_bounds__(kBlock) k_stencil_fill(StencilOp<T> A, const int64_t *__restrict__ rp,
                                                         int32_t *__restrict__ ci, T *__restrict__ val) {
    for (int64_t r = gtid(); r < A.n; r += gstride()) {
        int64_t p = rp[r];
        A.row_entries(r, [&](int64_t c, T v) {
            ci[p] = (int32_t)c;
            val[p] = v;
            ++p;
        });
    }
}

// GMRES polynomial, real root: acc += inv*work ; work_next = work - inv*(A work)
template <typename T, class Op>
__global__ void __launch_bounds__(kBlock) k_poly_real(Op A, const T *__restrict__ work, T *__restrict__ wnext,
                                                      T *__restrict__ acc, T inv, int first,
                                                      const int32_t *done) {
    if (skip(done)) return;
    for (int64_t r = gtid(); r < A.n; r += gstride()) {
        const T wr = work[r];
        const T p = RN<T>::mul(inv, wr);
        acc[r] = RN<T>::add(first ? T(0) : acc[r], p);
        if (wnext) {
            const T y = A.row(r, XPlain<T>{work});
            wnext[r] = RN<T>::sub(wr, RN<T>::mul(inv, y));
        }
    }
}

// conjugate pair, part 1: t = A work ; acc += (tr*work - t)/m2
template <typename T, class Op>
__global__ void __launch_bounds__(kBlock) k_poly_pair1(Op A, const T *__restrict__ work, T *__restrict__ t,
                                                       T *__restrict__ acc, T tr, T m2, int first,
                                                       const int32_t *done) {
    if (skip(done)) return;
    for (int64_t r = gtid(); r < A.n; r += gstride()) {
        const T tv = A.row(r, XPlain<T>{work});
        t[r] = tv;
        const T q = RN<T>::div(RN<T>::sub(RN<T>::mul(tr, work[r]), tv), m2);
        acc[r] = RN<T>::add(first ? T(0) : acc[r], q);
    }
}

// conjugate pair, part 2: work_next = work - (tr*t - A t)/m2
template <typename T, class Op>
__global__ void __launch_bounds__(kBlock) k_poly_pair2(Op A, const T *__restrict__ work, const T *__restrict__ t,
                                                       T *__restrict__ wnext, T tr, T m2, const int32_t *done) {
    if (skip(done)) return;
    for (int64_t r = gtid(); r < A.n; r += gstride()) {
        const T s = A.row(r, XPlain<T>{t});
        wnext[r] = RN<T>::sub(work[r], RN<T>::div(RN<T>::sub(RN<T>::mul(tr, t[r]), s), m2));
    }
}

template <typename S, typename D>
__global__ void k_convert_gated(int64_t n, const S *__restrict__ s, D *__restrict__ d, const int32_t *done) {
    if (skip(done)) return;
    for (int64_t i = gtid(); i < n; i += gstride()) {
        if constexpr (sizeof(D) == 4 && sizeof(S) == 8)
            d[i] = __double2float_rn(s[i]);
        else
            d[i] = (D)s[i];
    }
}

// Standalone HessenbergSystem (kernels.py:139-216) on device state.
template <typename T>
__global__ void k_lsq_init(Hess<T> H, mpk_cycle_ctl *ctl, double gamma, double norm_scale) {
    if (threadIdx.x != 0) return;
    H.g[0] = RN<T>::from_double(gamma);
    ctl->gamma = gamma;
    ctl->scale = norm_scale;
    ctl->steps = 0;
    ctl->done = 0;
    ctl->breakdown = 0;
    ctl->tri_err = 0;
}

template <typename T>
__global__ void k_lsq_update(const T *coeffs, const T *beta, T *sums, Hess<T> H, mpk_cycle_ctl *ctl,
                             StepParams p) {
    const int j = p.k + 1;
    for (int i = threadIdx.x; i < j; i += blockDim.x) {
        sums[S_C1 + i] = coeffs[i];
        sums[S_C2 + i] = T(0);    // c1 + 0 == c1 exactly
    }
    if (threadIdx.x == 0) sums[S_BETA] = *beta;
    __syncthreads();
    hessenberg_step<T>(sums, H, ctl, p);
}

}  // namespace mpk
