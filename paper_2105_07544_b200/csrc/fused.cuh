// Persistent, cooperative kernel for one whole restarted-GMRES cycle
// (gmres.py:134-205 with kernels.py:98-216), identity preconditioner,
// restart length m <= 63.
//
// Launch: one CTA of kFB threads per SM (cooperative, all co-resident).  CTA b
// owns the contiguous rows [b*rpc, (b+1)*rpc) for the whole cycle.  Each
// Arnoldi step is three streaming phases over the CTA's rows, separated by
// grid barriers; after each barrier every CTA reduces the per-CTA partials
// itself, in the same fixed order, so all CTAs hold bit-identical
// coefficients and run the (serial, O(j)) Givens update redundantly — no
// extra broadcast barrier, no kernel launches inside the cycle:
//
//   A  v_k = w''/beta (own rows -> V[:,k]), w = A v_k (neighbours read w''
//      through L2), ||w||^2, c1 = V[:,0..k]^T w            -> barrier, reduce
//   B  w' = w - V c1 (row-wise), c2 = V^T w' (column-wise; the chunk of V is
//      re-read from L1/L2, HBM sees it once)               -> barrier, reduce
//   C  w'' = w' - V c2, ||w''||^2                          -> barrier, reduce
//      beta, append test (kernels.py:122), Givens (kernels.py:183-196), exit
//
// Epilogue: each CTA back-substitutes R d = g (kernels.py:202-216) from its
// shared-memory copy of R and forms x_out = x0 + V_k d for its own rows.
// Dot products: row-wise -> thread accumulators; column-wise -> one warp per
// column (16 warps x 4 columns), lanes striding the chunk's rows.
#pragma once

#include "kernels.cuh"

namespace mpk {

constexpr int kFB = 512;                // threads per CTA
constexpr int kFW = kFB / 32;           // warps per CTA
constexpr int kFMaxCols = 64;           // m + 1 <= 64
constexpr int kFQ = kFMaxCols / kFW;    // columns owned per warp
constexpr int kFExtra = kFMaxCols;      // partial slot of the extra scalar
constexpr int kFSlots = kFMaxCols + 1;
constexpr int kFMaxCtas = 320;          // per-slot stride of the partials
constexpr int kCombineBatch = 8;        // 16-byte column loads in flight per row group
constexpr int kDotBatch = 8;            // 16-byte loads in flight per lane per column

template <typename T> struct FusedArgs {
    int64_t n, ld;
    int m, cap;
    T *V;
    const T *r0;
    const T *rnorm2;
    const T *x0;
    T *x_out;
    T *w, *wp, *wpp;
    T *part;          // 3 phases x kFSlots x kFMaxCtas
    unsigned *bar;    // [0] arrival count, [1] generation
    Hess<T> H;        // global mirrors (rotated R, raw columns, g, d) for diagnostics
    mpk_cycle_ctl *ctl;
    double tf, exit_tol, norm_scale, u;
    int final_col;    // collect_basis: also write V[:, steps] = w''/beta
};

// Sense-free grid barrier (all CTAs co-resident by cooperative launch).
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *vgen = bar + 1;
        const unsigned g0 = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nb - 1) {
            bar[0] = 0u;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == g0) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// out[s] = sum over CTAs b (fixed order) of part[idx(s)][b], for slots
// s < nslots, idx(s) = s for s < ncols else kFExtra.  One warp per slot,
// lanes stride the CTAs, then a fixed butterfly: identical in every CTA.
template <typename T>
__device__ __forceinline__ void cross_reduce(const T *part, unsigned nb, int ncols, int nslots, T *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < (kFSlots + kFW - 1) / kFW; ++q) {
        const int s = warp + kFW * q;
        if (s < nslots) {
            const int idx = (s < ncols) ? s : kFExtra;
            const T *p = part + (int64_t)idx * kFMaxCtas;
            T v[kFMaxCtas / 32];
#pragma unroll
            for (int i = 0; i < kFMaxCtas / 32; ++i) {
                const unsigned b = lane + 32 * i;
                v[i] = (b < nb) ? __ldcg(p + b) : T(0);
            }
            T acc = T(0);
#pragma unroll
            for (int i = 0; i < kFMaxCtas / 32; ++i) acc += v[i];
            acc = warp_sum(acc);
            if (lane == 0) out[s] = acc;
        }
    }
}

// Per-CTA partials: warp-owned column accumulators + one extra scalar.
template <typename T>
__device__ __forceinline__ void write_partials(T (&acc)[kFQ], int ncols, T extra, T *sred, T *part) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kFQ; ++q) {
        const int c = warp + kFW * q;
        const T v = warp_sum(acc[q]);
        if (lane == 0 && c < ncols) part[(int64_t)c * kFMaxCtas + blockIdx.x] = v;
    }
    const T e = warp_sum(extra);
    if (lane == 0) sred[warp] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        T s = sred[0];
        for (int w = 1; w < kFW; ++w) s += sred[w];
        part[(int64_t)kFExtra * kFMaxCtas + blockIdx.x] = s;
    }
}

// 16-byte row groups: RPT consecutive rows per thread (4 fp32 / 2 fp64),
// loaded from the column-major basis with one 16-byte load per column.
template <typename T> struct Vec16;
template <> struct Vec16<float> {
    using type = float4;
    static constexpr int R = 4;
    static __device__ __forceinline__ float get(const float4 &v, int i) {
        return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
    }
};
template <> struct Vec16<double> {
    using type = double2;
    static constexpr int R = 2;
    static __device__ __forceinline__ double get(const double2 &v, int i) { return i == 0 ? v.x : v.y; }
};

// s[e] = sum_{c < nc} V[c, r + e] * coef[c], e < RPT; 16 columns in flight.
template <typename T>
__device__ __forceinline__ void group_combine(const T *V, int64_t ld, int64_t r, int nc, const T *coef,
                                              T (&s)[Vec16<T>::R]) {
    using VT = typename Vec16<T>::type;
    constexpr int R = Vec16<T>::R;
#pragma unroll
    for (int e = 0; e < R; ++e) s[e] = T(0);
    constexpr int G = kCombineBatch;
    for (int c = 0; c < nc; c += G) {
        VT v[G];
#pragma unroll
        for (int q = 0; q < G; ++q)
            if (c + q < nc) v[q] = *reinterpret_cast<const VT *>(V + (int64_t)(c + q) * ld + r);
#pragma unroll
        for (int q = 0; q < G; ++q)
            if (c + q < nc) {
                const T cf = coef[c + q];
#pragma unroll
                for (int e = 0; e < R; ++e) s[e] += Vec16<T>::get(v[q], e) * cf;
            }
    }
}

// Row-wise s = sum_c V[c, r] * coef[c] for c < nc (coef in shared memory);
// loads issued in groups of 16 independent columns.
template <typename T>
__device__ __forceinline__ T row_combine(const T *V, int64_t ld, int64_t r, int nc, const T *coef) {
    T s = T(0);
    int c = 0;
    for (; c + 16 <= nc; c += 16) {
        T v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = V[(int64_t)(c + q) * ld + r];
#pragma unroll
        for (int q = 0; q < 16; ++q) s += v[q] * coef[c + q];
    }
    if (c < nc) {
        T v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = (c + q < nc) ? V[(int64_t)(c + q) * ld + r] : T(0);
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (c + q < nc) s += v[q] * coef[c + q];
    }
    return s;
}

// Column-wise acc[q] += sum_{rows of chunk} V[c, row] * x[row] for the
// warp's columns c = warp + kFW*q < nc.  The chunk is kFB*RPT rows; lane l
// reads 16-byte groups l, l+32, ... of the column; x (and, for column
// own_c, the column itself) come from shared memory as 16-byte groups.
template <typename T>
__device__ __forceinline__ void col_dots(const T *V, int64_t ld, int64_t c0, int nc, const T *x,
                                         int own_c, const T *own, T (&acc)[kFQ]) {
    using VT = typename Vec16<T>::type;
    constexpr int R = Vec16<T>::R;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const VT *xv = reinterpret_cast<const VT *>(x);
#pragma unroll
    for (int q = 0; q < kFQ; ++q) {
        const int c = warp + kFW * q;
        if (c < nc) {
            const VT *col = reinterpret_cast<const VT *>(c == own_c ? own : V + (int64_t)c * ld + c0);
            T s = T(0);
#pragma unroll
            for (int h = 0; h < kFB / 32; h += kDotBatch) {
                VT v[kDotBatch];
#pragma unroll
                for (int i = 0; i < kDotBatch; ++i) v[i] = col[lane + 32 * (h + i)];
#pragma unroll
                for (int i = 0; i < kDotBatch; ++i) {
                    const VT xx = xv[lane + 32 * (h + i)];
#pragma unroll
                    for (int e = 0; e < R; ++e) s += Vec16<T>::get(v[i], e) * Vec16<T>::get(xx, e);
                }
            }
            acc[q] += s;
        }
    }
}

template <typename T, class Op>
__global__ void __launch_bounds__(kFB, 1) k_cycle_fused(Op A, FusedArgs<T> a) {
    extern __shared__ unsigned char dsm_raw[];
    const int m = a.m, ldr = m + 1;
    T *sR = reinterpret_cast<T *>(dsm_raw);   // (m+1) x m rotated columns
    T *scs = sR + (int64_t)ldr * m;
    T *ssn = scs + m;
    T *sg = ssn + m;                           // m + 1
    T *sc1 = sg + (m + 1);                     // kFSlots
    T *sc2 = sc1 + kFSlots;                    // kFSlots
    constexpr int R = Vec16<T>::R;
    constexpr int CH = kFB * R;                // rows per chunk
    T *sx = reinterpret_cast<T *>(reinterpret_cast<uintptr_t>(sc2 + kFSlots + 1) & ~uintptr_t(15)) + 4;
    T *sv = sx + CH;                           // chunk of v_k (16-byte aligned)
    T *sred = sv + CH;                         // kFW
    __shared__ T s_gamma, s_beta, s_bn2;
    __shared__ int s_done, s_steps, s_break, s_app;
    __shared__ double s_scale;

    const int tid = threadIdx.x;
    const unsigned nb = gridDim.x;
    const int64_t rpc = ((a.n + nb - 1) / nb + 63) / 64 * 64;   // rows per CTA, 64-aligned
    const int64_t rb = (int64_t)blockIdx.x * rpc;
    const int64_t re = (rb + rpc < a.n) ? rb + rpc : a.n;
    T *partA = a.part, *partB = partA + (int64_t)kFSlots * kFMaxCtas,
      *partC = partB + (int64_t)kFSlots * kFMaxCtas;
    const bool lead = (blockIdx.x == 0);

    if (tid == 0) {
        const T gamma = RN<T>::sqrt_(__ldcg(a.rnorm2));
        s_gamma = gamma;
        double scale = a.norm_scale > 0.0 ? a.norm_scale : (double)gamma;
        if (gamma == T(0) && !(scale > 0.0)) scale = 1.0;   // gmres.py:170-172
        s_scale = scale;
        s_done = (gamma == T(0)) ? 1 : 0;
        s_steps = 0;
        s_break = 0;
        sg[0] = gamma;
        if (lead) {
            a.ctl->gamma = (double)gamma;
            a.ctl->scale = scale;
            a.ctl->steps = 0;
            a.ctl->breakdown = 0;
            a.ctl->tri_err = 0;
            a.ctl->done = s_done;
            a.H.g[0] = gamma;
        }
    }
    __syncthreads();

    for (int k = 0; k < a.cap && !s_done; ++k) {
        const int nc = k + 1;
        const T *src = (k == 0) ? a.r0 : a.wpp;
        const T dv = (k == 0) ? s_gamma : s_beta;
        T *vk = a.V + (int64_t)k * a.ld;
        T acc[kFQ];
        // ---------------- phase A: normalise, SpMV, ||w||^2, V^T w
#pragma unroll
        for (int q = 0; q < kFQ; ++q) acc[q] = T(0);
        T an = T(0);
        for (int64_t c0 = rb; c0 < re; c0 += CH) {
#pragma unroll
            for (int e = 0; e < R; ++e) {
                const int lr = tid * R + e;
                const int64_t r = c0 + lr;
                T own = T(0), wr = T(0);
                if (r < re) {
                    own = RN<T>::div(__ldcg(src + r), dv);
                    vk[r] = own;
                    wr = A.row(r, XScaledCG<T>{src, dv});
                    a.w[r] = wr;
                    an += wr * wr;
                }
                sv[lr] = own;
                sx[lr] = wr;
            }
            __syncthreads();
            col_dots<T>(a.V, a.ld, c0, nc, sx, k, sv, acc);
            __syncthreads();
        }
        write_partials<T>(acc, nc, an, sred, partA);
        grid_sync(a.bar, nb);
        cross_reduce<T>(partA, nb, nc, nc + 1, sc1);   // sc1[0..k], sc1[nc] = ||w||^2
        __syncthreads();
        // ---------------- phase B: w' = w - V c1 ; V^T w'
#pragma unroll
        for (int q = 0; q < kFQ; ++q) acc[q] = T(0);
        for (int64_t c0 = rb; c0 < re; c0 += CH) {
            const int64_t r = c0 + tid * R;
            T sl[R];
            if (r < re) group_combine<T>(a.V, a.ld, r, nc, sc1, sl);
#pragma unroll
            for (int e = 0; e < R; ++e) {
                T wr = T(0);
                if (r + e < re) {
                    wr = RN<T>::sub(a.w[r + e], sl[e]);
                    a.wp[r + e] = wr;
                }
                sx[tid * R + e] = wr;
            }
            __syncthreads();
            col_dots<T>(a.V, a.ld, c0, nc, sx, -1, sv, acc);
            __syncthreads();
        }
        write_partials<T>(acc, nc, T(0), sred, partB);
        grid_sync(a.bar, nb);
        cross_reduce<T>(partB, nb, nc, nc, sc2);
        __syncthreads();
        // ---------------- phase C: w'' = w' - V c2 ; ||w''||^2
        T bn = T(0);
        for (int64_t r = rb + tid * R; r < re; r += CH) {
            T sl[R];
            group_combine<T>(a.V, a.ld, r, nc, sc2, sl);
#pragma unroll
            for (int e = 0; e < R; ++e) {
                if (r + e < re) {
                    const T wr = RN<T>::sub(a.wp[r + e], sl[e]);
                    a.wpp[r + e] = wr;
                    bn += wr * wr;
                }
            }
        }
        {
            T dummy[kFQ];
#pragma unroll
            for (int q = 0; q < kFQ; ++q) dummy[q] = T(0);
            write_partials<T>(dummy, 0, bn, sred, partC);
        }
        grid_sync(a.bar, nb);
        cross_reduce<T>(partC, nb, 0, 1, &s_bn2);
        __syncthreads();
        // ---------------- beta, append test, Givens (every CTA, identical)
        T *col = sR + (int64_t)k * ldr;
        for (int i = tid; i < nc; i += kFB) col[i] = RN<T>::add(sc1[i], sc2[i]);
        __syncthreads();
        if (tid == 0) {
            const T beta = RN<T>::sqrt_(s_bn2);
            s_beta = beta;
            col[nc] = beta;
            const T wnorm = RN<T>::sqrt_(sc1[nc]);
            const int app = ((double)beta > a.tf * (double)wnorm) ? 1 : 0;   // kernels.py:122
            if (lead) {
                T *raw = a.H.raw + (int64_t)k * ldr;
                for (int i = 0; i <= nc; ++i) raw[i] = col[i];
            }
            T carry = col[0];
            for (int i = 0; i < nc - 1; ++i) {
                const T x0 = carry, x1 = col[i + 1], c = scs[i], s = ssn[i];
                col[i] = RN<T>::add(RN<T>::mul(c, x0), RN<T>::mul(s, x1));
                carry = RN<T>::add(RN<T>::mul(-s, x0), RN<T>::mul(c, x1));
            }
            const T x0 = carry, x1 = col[nc];
            T c, s, rr;
            if (x1 == T(0)) {
                c = T(1); s = T(0); rr = x0;
            } else {
                rr = RN<T>::hypot_(x0, x1);
                c = RN<T>::div(x0, rr);
                s = RN<T>::div(x1, rr);
            }
            scs[k] = c;
            ssn[k] = s;
            col[k] = rr;
            col[nc] = T(0);
            const T gprev = sg[k];
            const T gk = RN<T>::mul(-s, gprev);
            sg[nc] = gk;
            sg[k] = RN<T>::mul(c, gprev);
            const double rel = fabs((double)gk) / s_scale;
            int done = 0, brk = 0;
            if (!app) {
                brk = 1;
                done = 1;
            } else if (rel <= a.exit_tol || nc >= a.cap) {
                done = 1;
            }
            s_steps = nc;
            s_done = done;
            s_break = brk;
            if (lead) {
                a.ctl->implicit_relres[k] = rel;
                a.ctl->steps = nc;
                a.ctl->breakdown = brk;
                a.ctl->done = done;
                a.H.cs[k] = c;
                a.H.sn[k] = s;
            }
        }
        __syncthreads();
    }

    // ---------------- epilogue: d = R \ g, x_out = x0 + V_k d
    const int k = s_steps;
    T *sd = sc1;
    if (k > 0 && tid < 32) {
        if (tid == 0) {
            T dmax = fabs(sR[0]), dmin = dmax;
            int imin = 0;
            for (int i = 1; i < k; ++i) {
                const T v = fabs(sR[(int64_t)i * ldr + i]);
                if (v > dmax) dmax = v;
                if (v < dmin) { dmin = v; imin = i; }
            }
            const double thr = (double)k * a.u * (double)dmax;
            s_app = ((double)dmin <= thr) ? 1 : 0;
            if (s_app && lead) {
                a.ctl->tri_err = 1;
                a.ctl->tri_index = imin;
                a.ctl->tri_entry = (double)dmin;
                a.ctl->tri_threshold = thr;
            }
        }
        __syncwarp();
        if (!s_app) {
            T *rhs = sc2;
            for (int i = tid; i < k; i += 32) rhs[i] = sg[i];
            __syncwarp();
            for (int i = k - 1; i >= 0; --i) {
                if (tid == 0) sd[i] = RN<T>::div(rhs[i], sR[(int64_t)i * ldr + i]);
                __syncwarp();
                const T di = sd[i];
                for (int q = tid; q < i; q += 32) rhs[q] = rhs[q] - sR[(int64_t)i * ldr + q] * di;
                __syncwarp();
            }
        }
    }
    __syncthreads();
    if (k > 0 && s_app) return;   // TriangularBreakdownError: x_out untouched
    if (a.final_col && k > 0 && !s_break) {
        T *vn = a.V + (int64_t)k * a.ld;
        for (int64_t r = rb + tid; r < re; r += kFB) vn[r] = RN<T>::div(a.wpp[r], s_beta);
    }
    for (int64_t r = rb + tid * R; r < re; r += CH) {
        T sl[R];
        if (k > 0) group_combine<T>(a.V, a.ld, r, k, sd, sl);
#pragma unroll
        for (int e = 0; e < R; ++e)
            if (r + e < re) a.x_out[r + e] = (k == 0) ? a.x0[r + e] : RN<T>::add(a.x0[r + e], sl[e]);
    }
}

}  // namespace mpk
