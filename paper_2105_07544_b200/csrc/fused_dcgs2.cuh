// Persistent cycle kernel with the lagged one-reduction CGS2 ("DCGS2"):
// mathematically the reference's CGS2 Arnoldi (kernels.py:98-126), reordered
// so each step needs ONE global reduction and TWO passes over the basis
// (the reference's form needs 4 passes; k_cycle_reg needs 3 and 3 grid
// barriers).  Opt-in (SolverConfig.orthogonalization = "dcgs2"); identity or
// diagonal (block Jacobi k = 1, one GPU) right preconditioner, m <= 51.
//
// State entering step j (1..m): Q_j = [q_0..q_{j-1}] (final), u = w_{j-1} -
// Q_j c (w_{j-1} = A q_{j-1} after its first CGS pass c, neither
// re-orthogonalised nor normalised).  Step j:
//   z = A u                                           (SpMV, own rows)
//   [X0, X1, a, b] = [Q_j^T u, Q_j^T z, u.u, u.z]     (ONE reduction)
//   rho = sqrt(a - X0.X0)                             (norm of the re-orthogonalised u)
//   H[:, j-1] = [c + X0; rho]   (= CGS2's c1 + c2 and beta: column j-1 final)
//   Givens on column j-1, implicit residual of step j, exit test
//   t = (b - X0.X1)/rho,  tau = t/rho
//   c' = ([X1; t] - H[:j+1, :j] X0)/rho             (first-pass coefficients of A q_j)
//   q_j = (u - Q_j X0)/rho,  u' = (z - Q_j (X1 - X0 tau) - u tau)/rho     (ONE update pass)
// The identities used: A Q_j = Q_{j+1} H (Arnoldi), so A q_j = (z - Q_{j+1} H X0)/rho,
// and ||w_{j-1}||^2 = ||u||^2 + ||c||^2 for the reference's append test.
#pragma once

#include "fused_reg.cuh"

namespace mpk {

enum { kDcDots2 = 0, kDcUpdate2 = 1 };

// x accessor of the unnormalised candidate u (complete before the SpMV: every
// CTA wrote its rows before the last grid barrier)
template <typename T> struct XCg {
    const T *p;
    __device__ __forceinline__ T operator()(int64_t c) const { return __ldcg(p + c); }
    __device__ __forceinline__ Pack<T> vec(int64_t c) const { return ldcg16(p + c); }
};

// kDcDots2:   a0[i] += V[:, c].u, a1[i] += V[:, c].z, e0 += u.u, e1 += u.z
// kDcUpdate2: q = (u - V X0)/rho -> qout ; u' = (z - V Y - u tau)/rho -> u (in place)
// TV: basis storage (T, or binary16 holding q * vs; the scale is folded
// into the coefficients and the dot partials as in reg_phase_u)
template <typename T, int MODE, int U, int KU, typename TV = T>
__device__ __forceinline__ void dc_phase_u(const TV *V, int64_t ld, int nc, int64_t rb, int64_t re, T *u, const T *z,
                                           TV *qout, const T *X0, const T *Y, T rho, T tau,
                                           T (&a0)[RegCfg<T>::KP], T (&a1)[RegCfg<T>::KP], T &e0, T &e1, bool rev,
                                           const CommArgs<T> *cm, T vs = T(1), T vsi = T(1)) {
    using C = RegCfg<T, TV>;
    constexpr int R = C::R;
    constexpr bool half = sizeof(TV) != sizeof(T);
    // q and u' scale by 1/rho: one multiply per row instead of an IEEE
    // division (~10 instructions, executed by the part-0 lanes only, which
    // cost the 16-bit-basis stream as many issue slots as its FMAs).  The
    // lagged CGS2 is this repo's reformulation, not the reference's
    // operation order; oracle.dcgs2_cycle rounds the same way.
    const T rinv = MODE == kDcUpdate2 ? RN<T>::div(T(1), rho) : T(0);
    static_assert(KU <= C::KP, "columns per part");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane % C::G, p = lane / C::G;
    constexpr int64_t TRIP = (int64_t)C::WR * U;
    const int64_t b0 = rb + (int64_t)warp * TRIP, step = (int64_t)kFW * TRIP;
    const int64_t ntrip = (b0 < re) ? (re - b0 + step - 1) / step : 0;
    for (int64_t t = 0; t < ntrip; ++t) {
        const int64_t b = b0 + (rev ? ntrip - 1 - t : t) * step;
        Pack<TV> vv[U][KU];
        T uv[U][R], zv[U][R];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const int64_t r = b + (int64_t)(uu * C::G + g) * R;
            const bool live = r < re;
#pragma unroll
            for (int i = 0; i < KU; ++i) {
                const int c = p + C::P * i;
                if (c < nc && live) vv[uu][i] = ldcg16(V + (int64_t)c * ld + r);
                else {
#pragma unroll
                    for (int e = 0; e < R; ++e) vv[uu][i].v[e] = TV(0.0f);
                }
            }
            // kDcUpdate2 writes u in place from part 0: only part 0 reads it there
            const bool need = live && (MODE == kDcDots2 || p == 0);
            if (need) {
                ldrows<T, R>(u + r, uv[uu]);
                ldrows<T, R>(z + r, zv[uu]);
            } else {
#pragma unroll
                for (int e = 0; e < R; ++e) uv[uu][e] = zv[uu][e] = T(0);
            }
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const int64_t r = b + (int64_t)(uu * C::G + g) * R;
            const bool live = r < re;
            if (MODE == kDcDots2) {
#pragma unroll
                for (int i = 0; i < KU; ++i) {
                    if (p + C::P * i < nc) {
                        T vr[R];
                        raw_vals<T, TV>(vv[uu][i], vr);
#pragma unroll
                        for (int e = 0; e < R; ++e) {
                            a0[i] += vr[e] * uv[uu][e];
                            a1[i] += vr[e] * zv[uu][e];
                        }
                    }
                }
                if (p == 0) {
#pragma unroll
                    for (int e = 0; e < R; ++e) {
                        e0 += uv[uu][e] * uv[uu][e];
                        e1 += uv[uu][e] * zv[uu][e];
                    }
                }
                continue;
            }
            T s1[R], s2[R];
#pragma unroll
            for (int e = 0; e < R; ++e) s1[e] = s2[e] = T(0);
#pragma unroll
            for (int i = 0; i < KU; ++i) {
                const int c = p + C::P * i;
                if (c < nc) {
                    const T c1 = half ? X0[c] * vsi : X0[c], c2 = half ? Y[c] * vsi : Y[c];
                    T vr[R];
                    raw_vals<T, TV>(vv[uu][i], vr);
#pragma unroll
                    for (int e = 0; e < R; ++e) {
                        s1[e] += vr[e] * c1;
                        s2[e] += vr[e] * c2;
                    }
                }
            }
#pragma unroll
            for (int o = C::G; o < 32; o <<= 1) {
#pragma unroll
                for (int e = 0; e < R; ++e) {
                    s1[e] += __shfl_xor_sync(0xffffffffu, s1[e], o);
                    s2[e] += __shfl_xor_sync(0xffffffffu, s2[e], o);
                }
            }
            if (p == 0 && live) {
                T qv[R], un[R];
#pragma unroll
                for (int e = 0; e < R; ++e) {
                    qv[e] = RN<T>::mul(RN<T>::sub(uv[uu][e], s1[e]), rinv);
                    un[e] = RN<T>::mul(RN<T>::sub(RN<T>::sub(zv[uu][e], s2[e]), RN<T>::mul(uv[uu][e], tau)), rinv);
                }
                stvrows<T, TV, R>(qout + r, qv, vs);
                strows<T, R>(u + r, un);
                if (cm != nullptr) {   // halo rows of the candidate for the other ranks' SpMV (P2P)
                    for (int q = 0; q < cm->nranks; ++q)
                        if (q != cm->rank && r >= cm->mir_lo[q] && r < cm->mir_hi[q])
                            strows<T, R>(cm->xg[q] + cm->row0 + r, un);
                }
            }
        }
    }
    if constexpr (half) {
        if (MODE == kDcDots2) {
#pragma unroll
            for (int i = 0; i < KU; ++i) {
                a0[i] *= vsi;
                a1[i] *= vsi;
            }
        }
    }
}

template <typename T, int MODE, typename TV = T>
__device__ __forceinline__ void dc_phase(const TV *V, int64_t ld, int nc, int64_t rb, int64_t re, T *u, const T *z,
                                         TV *qout, const T *X0, const T *Y, T rho, T tau, T (&a0)[RegCfg<T>::KP],
                                         T (&a1)[RegCfg<T>::KP], T &e0, T &e1, bool rev, const CommArgs<T> *cm,
                                         T vs = T(1), T vsi = T(1)) {
    using C = RegCfg<T>;
    const int ncp = (nc + C::P - 1) / C::P;
#define MPK_DC_U(UU, KK) \
    dc_phase_u<T, MODE, UU, KK, TV>(V, ld, nc, rb, re, u, z, qout, X0, Y, rho, tau, a0, a1, e0, e1, rev, cm, vs, vsi)
    if constexpr (sizeof(TV) != sizeof(T)) {
        // 8 rows per 16-byte basis group: u and z take 16 registers per
        // group, so at most two groups per thread and trip
        if (ncp <= 6) MPK_DC_U(2, 6);
        else MPK_DC_U(1, 13);
        return;
    }
    switch (ncp) {
        case 1: case 2: case 3: MPK_DC_U(4, 3); break;
        case 4: MPK_DC_U(3, 4); break;
        case 5: case 6: MPK_DC_U(2, 6); break;
        case 7: MPK_DC_U(2, 7); break;
        case 8: MPK_DC_U(2, 8); break;
        default: MPK_DC_U(1, 13); break;
    }
#undef MPK_DC_U
}

// ... scaled by a diagonal right preconditioner: x = M u = u / a_ii
// (block Jacobi k = 1, preconditioners.py:133-139: one IEEE division)
template <typename T> struct XCgDiag {
    const T *p;
    const T *diag;
    __device__ __forceinline__ T operator()(int64_t c) const { return RN<T>::div(__ldcg(p + c), __ldg(diag + c)); }
    __device__ __forceinline__ Pack<T> vec(int64_t c) const {
        Pack<T> q = ldcg16(p + c);
#pragma unroll
        for (int e = 0; e < (int)(16 / sizeof(T)); ++e) q.v[e] = RN<T>::div(q.v[e], __ldg(diag + c + e));
        return q;
    }
};

// SpMV of the candidate: y = A x over the CTA's rows, x read through L2.
template <typename T, class Op, class X>
__device__ __noinline__ void dc_spmv_x(const Op &A, const X xs, T *y, int64_t rb, int64_t re, T *sstage) {
    if constexpr (!Op::kStencil) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        T *sb = sstage + warp * kCsrWarpBuf;
        const bool wide = sizeof(T) == 4 && A.rp[A.n] > 16 * (int64_t)A.n;   // long rows: 16 entries per lane
        for (int64_t r0 = rb + (int64_t)warp * 32; r0 < re; r0 += (int64_t)kFW * 32) {
            const T yr = wide ? A.template warp_rows<16>(r0, re, xs, sb) : A.template warp_rows<8>(r0, re, xs, sb);
            if (r0 + lane < re) y[r0 + lane] = yr;
        }
    } else if (A.group_ok()) {
        constexpr int R = RegCfg<T>::R;
        auto xv = [&](int64_t c) { return xs.vec(c); };
        for (int64_t r = rb + (int64_t)threadIdx.x * R; r < re; r += (int64_t)kFB * R) {
            Pack<T> o;
            A.row_group(r, xv, xs, o.v);
            stcg16(y + r, o);
        }
    } else {
        for (int64_t r = rb + threadIdx.x; r < re; r += kFB) y[r] = A.row(r, xs);
    }
}

template <typename T, class Op>
__device__ __forceinline__ void dc_spmv(const Op &A, const T *x, const T *diag, T *y, int64_t rb, int64_t re,
                                        T *sstage) {
    if (diag) dc_spmv_x<T>(A, XCgDiag<T>{x, diag}, y, rb, re, sstage);
    else dc_spmv_x<T>(A, XCg<T>{x}, y, rb, re, sstage);
}

template <typename T, class Op, bool MULTI, typename TV = T>
__global__ void __launch_bounds__(kFB, 1) k_cycle_dcgs2(Op A, FusedArgs<T> a) {
    static_assert(sizeof(TV) == sizeof(T) || !MULTI, "16-bit basis: one GPU");
    using C = RegCfg<T>;
    using IO = VIO<T, TV>;
    // basis storage: T, or binary16 holding q * vs (SolverConfig.basis_precision)
    TV *const Vb = reinterpret_cast<TV *>(a.V);
    const T vs = a.vs, vsi = a.vsi;
    extern __shared__ __align__(16) unsigned char dsm_dc[];
    const int m = a.m, ldr = m + 1;
    T *sR = reinterpret_cast<T *>(dsm_dc);     // (m+1) x m rotated columns
    T *sH = sR + (int64_t)ldr * m;             // (m+1) x m raw columns (c + X0, rho)
    T *scs = sH + (int64_t)ldr * m;
    T *ssn = scs + m;
    T *sg = ssn + m;                           // m + 1
    T *sX0 = sg + (m + 1);                     // 64 (+ a at [63])
    T *sX1 = sX0 + 64;                         // 64 (+ b at [63])
    T *sc = sX1 + 64;                          // 64: first-pass coefficients of the candidate
    T *sY = sc + 64;                           // 64
    T *scol = sY + 64;                         // 64: column being rotated
    T *sred = scol + 64;                       // kFW * kFSlots
    T *sstage = sred + kFW * kFSlots;          // kFW * kCsrWarpBuf
    __shared__ T s_gamma, s_rho, s_tau, s_beta;
    __shared__ int s_done, s_steps, s_break, s_app, s_trunc;
    __shared__ double s_scale;

    const int tid = threadIdx.x;
    const unsigned nb = gridDim.x;
    const int64_t rpc = ((a.n + nb - 1) / nb + 63) / 64 * 64;
    const int64_t rb = (int64_t)blockIdx.x * rpc;
    const int64_t re = (rb + rpc < a.n) ? rb + rpc : a.n;
    const bool lead = (blockIdx.x == 0);
    // partial slots: X0 -> [0, 52), a -> 104, X1 -> [52, 104), b -> 105.
    // Row-partitioned (nranks > 1): every rank's buffer, columns rank * nb + cta,
    // the candidate u lives in the rank's global-length x buffer (halo rows
    // mirrored P2P by the neighbours), barriers span all ranks.
    constexpr int kSlotB = 52, kXa = 104, kXb = 105;
    constexpr bool multi = MULTI;   // separate instantiations: the one-GPU kernel carries no comm code
    const CommArgs<T> *cmp = MULTI ? &a.cm : nullptr;
    const int pstride = multi ? kXStride : kFMaxCtas;
    const unsigned ncol = multi ? nb * (unsigned)a.cm.nranks : nb;
    T *part = multi ? a.cm.part[a.cm.rank] : a.part;
    T *u = multi ? a.wpp : a.w, *z = a.wp;
    unsigned long long ep = multi ? __ldcg(a.cm.epoch) : 0ull;
    auto sync_all = [&]() -> bool {
        if (!multi) {
            grid_sync(a.bar, nb);
            return false;
        }
        ++ep;
        return grid_sync_x<T>(a.bar, nb, a.cm, ep);
    };
    auto finish = [&]() {
        if (multi && lead && tid == 0) *a.cm.epoch = ep;
    };
#define MPK_DC_SYNC()                              \
    if (sync_all()) {                              \
        if (lead && tid == 0) a.ctl->pad_ = 1;     \
        finish();                                  \
        return;                                    \
    }

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
            a.ctl->pad_ = 0;
            a.ctl->done = s_done;
            a.H.g[0] = gamma;
        }
    }
    __syncthreads();
    T a0[C::KP], a1[C::KP];
    if (!s_done) {
        // ---- prologue: q_0 = r0/gamma ; w = A q_0 ; c = q_0.w ; u = w - q_0 c
        const T gm = s_gamma;
        TV *q0 = Vb;
        const T *src = a.r0;
        if (multi) {
            // q_0's SpMV reads halo rows of r0: stage r0 in the x buffer, mirror
            for (int64_t r = rb + tid; r < re; r += kFB) {
                const T v = a.r0[r];
                u[r] = v;
                for (int q = 0; q < a.cm.nranks; ++q)
                    if (q != a.cm.rank && r >= a.cm.mir_lo[q] && r < a.cm.mir_hi[q]) a.cm.xg[q][a.cm.row0 + r] = v;
            }
            src = u;
            MPK_DC_SYNC();
        }
        for (int64_t r = rb + tid; r < re; r += kFB) {
            const TV hv = IO::put(RN<T>::div(__ldcg(src + r), gm), vs);
            q0[r] = hv;
            const T v = IO::get(hv, vsi);   // as stored: the SpMV input is the stored q_0
            if (a.diag) a.z[r] = RN<T>::div(v, __ldg(a.diag + r));   // M q_0 on the own rows
        }
        __syncthreads();
        phase_a_spmv<T>(A, XSlab<T, TV>{src, q0, gm, rb, re, a.diag, a.z, vs, vsi}, z, rb, re, sstage);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < C::KP; ++i) a0[i] = T(0);
        T ext = T(0);
        reg_phase<T, kRegDots, TV>(Vb, a.ld, 1, rb, re, a.n, z, nullptr, nullptr, a0, ext, nullptr, nullptr, false, vsi);
        reg_write_partials<T>(a0, 1, T(0), sred, part, cmp, 0, 0, false, kXa);
        MPK_DC_SYNC();
        cross_reduce<T>(part, ncol, 1, 1, sc, pstride, kXa);   // sc[0] = c
        __syncthreads();
        reg_phase<T, kRegUpdateNorm, TV>(Vb, a.ld, 1, rb, re, a.n, z, u, sc, a0, ext, cmp, nullptr, false, vsi);   // u = w - q_0 c
        MPK_DC_SYNC();
    }
    // ---- steps j = 1..cap: finalise column j-1, build q_j and the next candidate
    for (int j = 1; j <= a.cap && !s_done; ++j) {
        dc_spmv<T>(A, u, a.diag, z, rb, re, sstage);   // z = A M u
        __syncthreads();
        T e0 = T(0), e1 = T(0);
#pragma unroll
        for (int i = 0; i < C::KP; ++i) a0[i] = a1[i] = T(0);
        dc_phase<T, kDcDots2, TV>(Vb, a.ld, j, rb, re, u, z, nullptr, nullptr, nullptr, T(0), T(0), a0, a1, e0, e1,
                                  j & 1, nullptr, vs, vsi);
        reg_write_partials<T>(a0, j, e0, sred, part, cmp, 0, 0, true, kXa);
        reg_write_partials<T>(a1, j, e1, sred, part, cmp, 0, kSlotB, true, kXb);
        MPK_DC_SYNC();
        cross_reduce<T>(part, ncol, j, j + 1, sX0, pstride, kXa);                                   // X0, a
        cross_reduce<T>(part + (int64_t)kSlotB * pstride, ncol, j, j + 1, sX1, pstride, kXb - kSlotB);   // X1, b
        __syncthreads();
        if (tid == 0) {
            sX0[63] = sX0[j];
            sX1[63] = sX1[j];
        }
        __syncthreads();
        // ---- column j-1 (every CTA, identical): H[:, j-1] = [c + X0; rho]
        const int k = j - 1, nc = j;
        if (tid == 0) {
            T x0x0 = T(0), cc = T(0), x0x1 = T(0);
            for (int i = 0; i < j; ++i) {
                x0x0 += sX0[i] * sX0[i];
                cc += sc[i] * sc[i];
                x0x1 += sX0[i] * sX1[i];
            }
            const T av = sX0[63], bv = sX1[63];
            T rho2 = RN<T>::sub(av, x0x0);
            // the Pythagorean norm is only trusted while it keeps ~2 digits
            // (rho^2 >= eta * ||u||^2, eta ~ 100 u / 1e-2); below that u is
            // (numerically) inside span(Q_j): treated as the reference's
            // lucky breakdown (beta = 0, kernels.py:122-126), which ends the
            // cycle with column j-1 included
            // Below the guard the step is NOT declared a lucky breakdown
            // (that would zero the implicit residual and can raise a false
            // loss of accuracy): rho is clamped to the guard and the cycle
            // ends after this column as if it had reached its cap, so the
            // restart recomputes the explicit residual from scratch.
            const T eta = sizeof(T) == 4 ? T(1e-3) : T(1e-11);
            s_trunc = 0;
            if (!(rho2 > eta * av)) {
                rho2 = eta * av;
                s_trunc = 1;
            }
            const T rho = RN<T>::sqrt_(rho2);
            s_rho = rho;
            const T t = RN<T>::div(RN<T>::sub(bv, x0x1), rho);
            s_tau = RN<T>::div(t, rho);
            sX1[j] = t;   // [X1; t]
            // the reference's append test uses ||w_{j-1}||^2 = ||u||^2 + ||c||^2
            sY[63] = RN<T>::add(av, cc);
            sY[62] = rho2;
        }
        __syncthreads();
        for (int i = tid; i < nc; i += kFB) {
            const T hv = RN<T>::add(sc[i], sX0[i]);
            sH[(int64_t)k * ldr + i] = hv;
            scol[i] = hv;
        }
        if (tid == 0) {
            sH[(int64_t)k * ldr + nc] = s_rho;
        }
        __syncthreads();
        if (tid == 0)
            givens_step<T>(a, k, nc, ldr, scol, sY[62], sY[63], s_scale, lead, scs, ssn, sg, s_beta, s_steps,
                           s_done, s_break);
        __syncthreads();
        if (tid == 0 && s_trunc && !s_done) {
            s_done = 1;
            if (lead) a.ctl->done = 1;
        }
        for (int i = tid; i <= nc; i += kFB) sR[(int64_t)k * ldr + i] = scol[i];
        __syncthreads();   // column k of R (all warps) before back_substitute (warp 0) or the next step
        if (s_done) break;
        // ---- next candidate: c' = ([X1; t] - H[:j+1, :j] X0)/rho ; Y = X1 - X0 tau
        const T rho = s_rho, tau = s_tau;
        for (int i = tid; i <= j; i += kFB) {
            T hs = T(0);
            // Hessenberg: H[i, l] = 0 below the subdiagonal (l < i - 1; never stored)
            for (int l = (i > 0 ? i - 1 : 0); l < j; ++l) hs += sH[(int64_t)l * ldr + i] * sX0[l];
            sc[i] = RN<T>::div(RN<T>::sub(sX1[i], hs), rho);
        }
        for (int i = tid; i < j; i += kFB) sY[i] = RN<T>::sub(sX1[i], RN<T>::mul(sX0[i], tau));
        __syncthreads();
        // ---- one update pass: q_j -> V[:, j], candidate u' in place
        T e0d = T(0), e1d = T(0);
        dc_phase<T, kDcUpdate2, TV>(Vb, a.ld, j, rb, re, u, z, Vb + (int64_t)j * a.ld, sX0, sY, rho, tau, a0, a1,
                                    e0d, e1d, (j + 1) & 1, cmp, vs, vsi);
        MPK_DC_SYNC();
    }

    // ---------------- epilogue: d = R \ g, x_out = x0 + V_k d
    const int k = s_steps;
    T *sd = sc;
    if (k > 0 && tid < 32) back_substitute<T>(a, k, ldr, sR, sg, sY, sd, lead, s_app);
    __syncthreads();
    finish();
    if (k > 0 && s_app) return;   // TriangularBreakdownError: x_out untouched
    if (lead) {
        for (int i = tid; i < k; i += kFB) a.H.d[i] = sd[i];
        for (int i = tid; i < k * ldr; i += kFB) a.H.h[i] = sR[i];
        for (int i = tid; i <= k; i += kFB) a.H.g[i] = sg[i];
    }
    if (k == 0) {
        for (int64_t r = rb + tid; r < re; r += kFB) a.x_out[r] = a.x0[r];
        return;
    }
    T ext = T(0);
    reg_phase<T, kRegCorrect, TV>(Vb, a.ld, k, rb, re, a.n, a.x0, a.x_out, sd, a0, ext, nullptr, a.diag, false, vsi);   // x0 + M V_k d
#undef MPK_DC_SYNC
}

}  // namespace mpk
