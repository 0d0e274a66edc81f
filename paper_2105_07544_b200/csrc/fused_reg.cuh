// Persistent cooperative cycle kernel, register-streaming variant
// (gmres.py:134-205 with kernels.py:98-216; identity or diagonal preconditioner;
// any m: beyond 51 the basis is streamed in 52-column blocks, BIG instantiation).
//
// Same phase structure, grid barriers, fixed-order cross-CTA reductions and
// redundant per-CTA Givens as k_cycle_fused (fused.cuh), but the basis is
// streamed HBM -> registers with 16-byte loads and no shared-memory staging
// or per-tile CTA barriers:
//
//   lane = p * G + g: g picks a 16-byte row group (R = 4 fp32 / 2 fp64 rows),
//   p one of P column parts (columns c = p, p + P, ...).  A warp covers G*R
//   rows per trip and every thread keeps its <= KP columns of the trip in
//   registers, so phase B's update w' = w - V c1 and dot c2 = V^T w' use one
//   HBM read of V: the P parts' partial row sums are combined with xor
//   shuffles (identical result in every part), then each thread folds
//   V[:, c] . w' into its per-column accumulators from the same registers.
//   Column accumulators are reduced over g lanes (shuffles), then over warps
//   in warp order, then over CTAs in CTA order: deterministic.
//
// Loads in flight: every thread issues its KP 16-byte column loads at once
// (16 warps x 32 lanes x 13 x 16 B ~ 100 KB per SM at m = 50).
#pragma once

#include "fused.cuh"

namespace mpk {

constexpr int kRegMaxCols = 52;          // columns per streaming block (one pass per phase when m <= 51)

template <typename T, typename TV = T> struct RegCfg {
    static constexpr int R = 16 / (int)sizeof(TV);     // rows per 16-byte basis group (4 fp32 / 2 fp64 / 8 fp16)
    static constexpr int G = 8;                        // row groups per warp (128-byte fp32 / 2 x 64-byte fp64 runs)
    static constexpr int P = 32 / G;                   // column parts per warp
    static constexpr int KP = kRegMaxCols / P;         // columns per part (13)
    static constexpr int WR = G * R;                   // rows per warp trip
};

enum { kRegDots = 0, kRegUpdateDots = 1, kRegUpdateNorm = 2, kRegCorrect = 3 };

// One streaming pass over the CTA's rows [rb, re) (n = global length for the
// masked tail of user buffers).  MODE
//   kRegDots        acc[i] += V[:, c] . x                      (phase A)
//   kRegUpdateDots  y = x - V coef; acc[i] += V[:, c] . y       (phase B)
//   kRegUpdateNorm  y = x - V coef; ext += y . y                (phase C)
//   kRegCorrect     y = x + V coef (x, y user buffers, masked)  (epilogue)
// U row groups per thread per trip (U * ceil(nc/P) <= KP): early in a cycle,
// when the basis is narrow, every thread still keeps ~KP 16-byte loads in
// flight instead of paying one memory latency per 32 rows.
template <typename T, typename TV, int MODE, int U, int KU>
__device__ __forceinline__ void reg_phase_u(const TV *V, int64_t ld, int nc, int64_t rb, int64_t re, int64_t n,
                                            const T *x, T *y, const T *coef, T (&acc)[RegCfg<T>::KP], T &ext,
                                            const CommArgs<T> *cm, const T *diag, bool rev, T vsi) {
    using C = RegCfg<T, TV>;
    constexpr int R = C::R;
    constexpr bool half = sizeof(TV) != sizeof(T);
    static_assert(KU <= C::KP, "columns per part");   // KU: columns per part held per row group
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane % C::G, p = lane / C::G;
    constexpr int64_t TRIP = (int64_t)C::WR * U;
    // rev: walk the rows last to first.  Consecutive phases alternate, so each
    // phase starts on the rows whose basis lines the previous phase touched
    // last and still finds them in L2 (up to its ~126 MB).
    const int64_t b0 = rb + (int64_t)warp * TRIP, step = (int64_t)kFW * TRIP;
    const int64_t ntrip = (b0 < re) ? (re - b0 + step - 1) / step : 0;
    for (int64_t t = 0; t < ntrip; ++t) {
        const int64_t b = b0 + (rev ? ntrip - 1 - t : t) * step;
        Pack<TV> vv[U][KU];
        T xv[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = b + (int64_t)(u * C::G + g) * R;
            const bool live = r < re;
#pragma unroll
            for (int i = 0; i < KU; ++i) {
                const int c = p + C::P * i;
                if (c < nc && live) vv[u][i] = ldcg16(V + (int64_t)c * ld + r);
                else {
#pragma unroll
                    for (int e = 0; e < R; ++e) vv[u][i].v[e] = TV(0.0f);
                }
            }
            if (MODE == kRegCorrect) {
#pragma unroll
                for (int e = 0; e < R; ++e)
                    xv[u][e] = (x != nullptr && p == 0 && live && r + e < n) ? x[r + e] : T(0);   // x may alias y; null: 0
            } else if (MODE == kRegUpdateNorm && p != 0) {
#pragma unroll
                for (int e = 0; e < R; ++e) xv[u][e] = T(0);   // only part 0 uses x (x may alias y)
            } else if (live) {
                ldrows<T, R>(x + r, xv[u]);
            } else {
#pragma unroll
                for (int e = 0; e < R; ++e) xv[u][e] = T(0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = b + (int64_t)(u * C::G + g) * R;
            const bool live = r < re;
            if (MODE == kRegDots) {
#pragma unroll
                for (int i = 0; i < KU; ++i) {
                    if (p + C::P * i < nc) {
                        T vr[R];
                        raw_vals<T, TV>(vv[u][i], vr);
#pragma unroll
                        for (int e = 0; e < R; ++e) acc[i] += vr[e] * xv[u][e];
                    }
                }
                continue;
            }
            T s[R];
#pragma unroll
            for (int e = 0; e < R; ++e) s[e] = T(0);
#pragma unroll
            for (int i = 0; i < KU; ++i) {
                const int c = p + C::P * i;
                if (c < nc) {
                    // binary16: the stored values carry the scale vs, folded
                    // into the coefficient (vsi is a power of two: exact)
                    const T cf = half ? coef[c] * vsi : coef[c];
                    T vr[R];
                    raw_vals<T, TV>(vv[u][i], vr);
#pragma unroll
                    for (int e = 0; e < R; ++e) s[e] += vr[e] * cf;
                }
            }
#pragma unroll
            for (int o = C::G; o < 32; o <<= 1) {
#pragma unroll
                for (int e = 0; e < R; ++e) s[e] += __shfl_xor_sync(0xffffffffu, s[e], o);
            }
            if (MODE == kRegCorrect && diag != nullptr && p == 0 && live) {
                // x + M (V_k d) with M = diag^-1 (gmres.py:195-196)
#pragma unroll
                for (int e = 0; e < R; ++e)
                    if (r + e < n) s[e] = RN<T>::div(s[e], __ldg(diag + r + e));
            }
            T yv[R];
#pragma unroll
            for (int e = 0; e < R; ++e)
                yv[e] = (MODE == kRegCorrect) ? RN<T>::add(xv[u][e], s[e]) : RN<T>::sub(xv[u][e], s[e]);
            if (p == 0 && live) {
                if (MODE == kRegCorrect && r + R > n) {
#pragma unroll
                    for (int e = 0; e < R; ++e)
                        if (r + e < n) y[r + e] = yv[e];
                } else {
                    strows<T, R>(y + r, yv);
                }
                if (MODE == kRegUpdateNorm && cm != nullptr) {
                    // halo rows of w'' for the other ranks' next SpMV (P2P)
                    for (int q = 0; q < cm->nranks; ++q)
                        if (q != cm->rank && r >= cm->mir_lo[q] && r < cm->mir_hi[q])
                            strows<T, R>(cm->xg[q] + cm->row0 + r, yv);
                }
            }
            if (MODE == kRegUpdateDots) {
#pragma unroll
                for (int i = 0; i < KU; ++i) {
                    if (p + C::P * i < nc) {
                        T vr[R];
                        raw_vals<T, TV>(vv[u][i], vr);
#pragma unroll
                        for (int e = 0; e < R; ++e) acc[i] += vr[e] * yv[e];
                    }
                }
            }
            if (MODE == kRegUpdateNorm && p == 0) {
#pragma unroll
                for (int e = 0; e < R; ++e) ext += yv[e] * yv[e];
            }
        }
    }
    if constexpr (half) {
        // dots against the stored (scaled) basis: undo the scale once
#pragma unroll
        for (int i = 0; i < KU; ++i) acc[i] *= vsi;
    }
}

template <typename T, int MODE, typename TV = T>
__device__ __forceinline__ void reg_phase(const TV *V, int64_t ld, int nc, int64_t rb, int64_t re, int64_t n,
                                          const T *x, T *y, const T *coef, T (&acc)[RegCfg<T>::KP], T &ext,
                                          const CommArgs<T> *cm = nullptr, const T *diag = nullptr, bool rev = false,
                                          T vsi = T(1)) {
    using C = RegCfg<T, TV>;
    const int ncp = (nc + C::P - 1) / C::P;   // columns per part
    // (U row groups, KU columns) per thread and trip: 12-18 sixteen-byte
    // loads in flight at every basis width.  Measured on B200 (phase-B pass,
    // tools/micro/stream_b_sweep.cu): the exact-width (2, 7..9) and (3, 4)
    // shapes stream 6.4-7.1 TB/s where (1, 13) with 7-9 live columns gave
    // 5.2-5.9 and (2, 6) with 4 gave 6.1-6.6; (2, 10..11) spill.
#define MPK_REG_U(UU, KK) \
    reg_phase_u<T, TV, MODE, UU, KK>(V, ld, nc, rb, re, n, x, y, coef, acc, ext, cm, diag, rev, vsi)
    static_assert(C::KP == 13, "shape table below assumes 13 columns per part");
    if constexpr (MODE == kRegUpdateNorm || MODE == kRegCorrect) {
        // update-only passes keep the round-1 shapes: with the exact-width
        // shapes stream C measured 19% slower (C2 phase profile, 2136 vs
        // 1795 us per cycle) while streams A and B gained 5-9%
        if (ncp * 8 <= C::KP) MPK_REG_U(8, 1);
        else if (ncp * 4 <= C::KP) MPK_REG_U(4, 3);
        else if (ncp * 2 <= C::KP) MPK_REG_U(2, 6);
        else MPK_REG_U(1, 13);
        return;
    }
    switch (ncp) {
        case 1: MPK_REG_U(8, 1); break;
        case 2:
        case 3: MPK_REG_U(4, 3); break;
        case 4: MPK_REG_U(3, 4); break;
        case 5:
        case 6: MPK_REG_U(2, 6); break;
        case 7: MPK_REG_U(2, 7); break;
        case 8: MPK_REG_U(2, 8); break;
        case 9: MPK_REG_U(2, 9); break;
        default: MPK_REG_U(1, 13); break;
    }
#undef MPK_REG_U
}

// CTA partials of the register layout: column c lives in part p = c % P,
// slot i = c / P of the G lanes with that p in every warp.
// `part` is this CTA's column of the local buffer (single GPU); with a comm,
// the CTA's column rank * nb + cta of the phase's block in EVERY rank's
// buffer is written (P2P stores; `off` = the phase block's element offset).
// Column block form (m > 51): the block's columns land at c0 + c and the
// extra scalar, if has_extra, at slot xslot.
template <typename T>
__device__ __forceinline__ void reg_write_partials(T (&acc)[RegCfg<T>::KP], int nc, T extra, T *sm, T *part,
                                                   const CommArgs<T> *cm = nullptr, int64_t off = 0, int c0 = 0,
                                                   bool has_extra = true, int xslot = kFExtra) {
    using C = RegCfg<T>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane % C::G, p = lane / C::G;
    if (c0 != 0 || !has_extra) __syncthreads();   // block form: sm reused by consecutive calls
#pragma unroll
    for (int i = 0; i < C::KP; ++i) {
        T v = acc[i];
#pragma unroll
        for (int o = 1; o < C::G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int c = p + C::P * i;
        if (g == 0 && c < nc) sm[warp * kFSlots + c] = v;
    }
    const T e = warp_sum(extra);
    if (lane == 0) sm[warp * kFSlots + kFExtra] = e;
    __syncthreads();
    for (int c = threadIdx.x; c < kFSlots; c += kFB) {
        if (c < nc || (c == kFExtra && has_extra)) {
            T s = sm[c];
            for (int w = 1; w < kFW; ++w) s += sm[w * kFSlots + c];
            if (cm == nullptr) {
                const int slot = (c == kFExtra) ? xslot : c0 + c;
                part[(int64_t)slot * kFMaxCtas + blockIdx.x] = s;
            } else {
                const int64_t col = (int64_t)cm->rank * gridDim.x + blockIdx.x;
                const int slot = (c == kFExtra) ? xslot : c0 + c;
                for (int q = 0; q < cm->nranks; ++q) cm->part[q][off + (int64_t)slot * kXStride + col] = s;
            }
        }
    }
}

// Phase A's SpMV w = A v_k over the CTA's rows, returns the thread's part of
// ||w||^2.  Out of line (noinline) so its register needs (BentPipe
// coefficient arithmetic, the CSR staging) do not raise register pressure in
// the streaming phases, which are kept spill-free.
template <typename T, class Op, class XS>
__device__ __noinline__ T phase_a_spmv(const Op &A, const XS xs, T *w, int64_t rb, int64_t re, T *sstage) {
    T an = T(0);
    if constexpr (!Op::kStencil) {
        // CSR: warp-cooperative 32-row groups (coalesced entries, row-sequential sums)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        T *sb = sstage + warp * kCsrWarpBuf;
        // long rows (config 5: ~49 entries): 16 entries per lane in flight (fp32)
        const bool wide = sizeof(T) == 4 && A.rp[A.n] > 16 * (int64_t)A.n;
        for (int64_t r0 = rb + (int64_t)warp * 32; r0 < re; r0 += (int64_t)kFW * 32) {
            const T wr = wide ? A.template warp_rows<16>(r0, re, xs, sb) : A.template warp_rows<8>(r0, re, xs, sb);
            if (r0 + lane < re) {
                w[r0 + lane] = wr;
                an += wr * wr;
            }
        }
    } else if (A.group_ok()) {
        // 16-byte row groups: vector reads of the group and its S/N (B/U)
        // neighbours; UG groups per thread per trip with every group's loads
        // issued before any is evaluated (||w||^2 summed in row order as
        // with one group per trip).  UG = 4 spilled (Laplace3D: 5 packs per
        // group) and cost 18% of the C4 cycle; 2 keeps the loads in registers
        constexpr int R = RegCfg<T>::R;
#ifndef MPK_PHASEA_UG
#define MPK_PHASEA_UG 1   // 2 measured 1% slower on C2/C4 (one group's loads suffice with 16 warps)
#endif
        constexpr int UG = MPK_PHASEA_UG;
        auto xv = [&](int64_t c) { return xs.vec(c); };
        constexpr int64_t S = (int64_t)kFB * R;
        int64_t r = rb + (int64_t)threadIdx.x * R;
        for (; r + (UG - 1) * S < re; r += UG * S) {
            typename Op::GroupIn in[UG];
#pragma unroll
            for (int u = 0; u < UG; ++u) A.group_load(r + u * S, xv, xs, in[u]);
#pragma unroll
            for (int u = 0; u < UG; ++u) {
                Pack<T> o;
                A.group_eval(r + u * S, in[u], o.v);
                stcg16(w + r + u * S, o);
#pragma unroll
                for (int e = 0; e < R; ++e) an += o.v[e] * o.v[e];
            }
        }
        for (; r < re; r += S) {
            Pack<T> o;
            A.row_group(r, xv, xs, o.v);
            stcg16(w + r, o);
#pragma unroll
            for (int e = 0; e < R; ++e) an += o.v[e] * o.v[e];
        }
    } else {
        // eight rows per thread per trip
        constexpr int UR = 8;
        int64_t r = rb + threadIdx.x;
        for (; r + (UR - 1) * kFB < re; r += UR * kFB) {
            T wv[UR];
#pragma unroll
            for (int u = 0; u < UR; ++u) wv[u] = A.row(r + u * kFB, xs);
#pragma unroll
            for (int u = 0; u < UR; ++u) {
                w[r + u * kFB] = wv[u];
                an += wv[u] * wv[u];
            }
        }
        for (; r < re; r += kFB) {
            const T wr = A.row(r, xs);
            w[r] = wr;
            an += wr * wr;
        }
    }
    return an;
}

// y = A x over the CTA's rows [rb, re) (x read through L2 from a vector the
// whole grid wrote before the last barrier); fn(r, y_r) on the thread that
// evaluated row r.  The row -> thread map is the same on every call, so fn
// may read-modify-write per-row state without a barrier.  Same row sums as
// the standalone SpMV (row_group == row(); CSR warp_rows == row()).
template <typename T, class Op, class F>
__device__ __forceinline__ void cta_rows(const Op &A, const T *x, int64_t rb, int64_t re, T *sstage, F &&fn) {
    const XCG<T> xs{x};
    if constexpr (!Op::kStencil) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        T *sb = sstage + warp * kCsrWarpBuf;
        for (int64_t r0 = rb + (int64_t)warp * 32; r0 < re; r0 += (int64_t)kFW * 32) {
            const T y = A.template warp_rows<8>(r0, re, xs, sb);
            if (r0 + lane < re) fn(r0 + lane, y);
        }
    } else if (A.group_ok()) {
        constexpr int R = RegCfg<T>::R;
        auto xv = [&](int64_t c) { return xs.vec(c); };
        const int64_t rv = rb + (re - rb) / R * R;
        for (int64_t r = rb + (int64_t)threadIdx.x * R; r < rv; r += (int64_t)kFB * R) {
            T o[R];
            A.row_group(r, xv, xs, o);
#pragma unroll
            for (int e = 0; e < R; ++e) fn(r + e, o[e]);
        }
        for (int64_t r = rv + threadIdx.x; r < re; r += kFB) fn(r, A.row(r, xs));
    } else {
        for (int64_t r = rb + threadIdx.x; r < re; r += kFB) fn(r, A.row(r, xs));
    }
}

// Buffers of the in-kernel GMRES polynomial (single GPU): units in shared
// memory, vectors in global memory.
template <typename T> struct PolyBufs {
    const PolyUnit<T> *unit;   // shared memory copy of FusedArgs::poly
    int npoly;
    T *w0, *w1, *t, *acc;
    unsigned *bar;
};

// z = p(A) v for the CTA's rows into pb.acc: apply_gmres_poly's product form
// (preconditioners.py:283-305) with the same per-row roundings as
// k_poly_real / k_poly_pair1 / k_poly_pair2 and one grid barrier before
// every SpMV after the first (`v` must be complete on every CTA).  Out of
// line so its register needs stay out of the streaming phases.
template <typename T, class Op>
__device__ __noinline__ void poly_apply_dev(const Op &A, PolyBufs<T> pb, const T *v, int64_t rb, int64_t re,
                                            T *sstage) {
    const T *work = v;
    T *const wbuf[2] = {pb.w0, pb.w1};
    int wi = 0;
    const unsigned nb = gridDim.x;
    for (int u = 0; u < pb.npoly; ++u) {
        const PolyUnit<T> pu = pb.unit[u];
        const bool first = (u == 0), last = (u + 1 == pb.npoly);
        T *wnext = wbuf[wi];
        T *acc = pb.acc;
        if (!pu.pair) {
            const T inv = pu.a;
            if (last) {
                for (int64_t r = rb + threadIdx.x; r < re; r += kFB)
                    acc[r] = RN<T>::add(first ? T(0) : acc[r], RN<T>::mul(inv, __ldcg(work + r)));
            } else {
                cta_rows<T>(A, work, rb, re, sstage, [&](int64_t r, T y) {
                    const T wr = __ldcg(work + r);
                    acc[r] = RN<T>::add(first ? T(0) : acc[r], RN<T>::mul(inv, wr));
                    wnext[r] = RN<T>::sub(wr, RN<T>::mul(inv, y));
                });
            }
        } else {
            const T tr = pu.a, m2 = pu.b;
            T *t = pb.t;
            cta_rows<T>(A, work, rb, re, sstage, [&](int64_t r, T tv) {
                t[r] = tv;
                const T q = RN<T>::div(RN<T>::sub(RN<T>::mul(tr, __ldcg(work + r)), tv), m2);
                acc[r] = RN<T>::add(first ? T(0) : acc[r], q);
            });
            if (!last) {
                __syncthreads();
                grid_sync(pb.bar, nb);
                cta_rows<T>(A, t, rb, re, sstage, [&](int64_t r, T sv) {
                    const T q = RN<T>::div(RN<T>::sub(RN<T>::mul(tr, __ldcg(t + r)), sv), m2);
                    wnext[r] = RN<T>::sub(__ldcg(work + r), q);
                });
            }
        }
        if (!last) {
            __syncthreads();
            grid_sync(pb.bar, nb);
            work = wnext;
            wi ^= 1;
        }
    }
}

// w = A z over the CTA's rows (z = the polynomial's accumulator, complete on
// every CTA); returns the thread's part of ||w||^2
template <typename T, class Op>
__device__ __noinline__ T poly_spmv_dev(const Op &A, const T *z, T *w, int64_t rb, int64_t re, T *sstage) {
    T an = T(0);
    cta_rows<T>(A, z, rb, re, sstage, [&](int64_t r, T y) {
        w[r] = y;
        an += y * y;
    });
    return an;
}

template <typename T, class Op, bool BIG, bool MULTI, typename TV = T, bool POLY = false>
__global__ void __launch_bounds__(kFB, 1) k_cycle_reg(Op A, FusedArgs<T> a) {
    // POLY: GMRES-polynomial instantiation (one GPU, m <= 51, TV == T); the
    // others carry no polynomial code (its call sites cost the streaming
    // phases registers even when not taken)
    static_assert(!POLY || (!BIG && !MULTI && sizeof(TV) == sizeof(T)), "polynomial cycle: one GPU, m <= 51");
    using C = RegCfg<T>;
    using IO = VIO<T, TV>;
    // basis storage: T, or binary16 holding v * vs (fp32 cycles, one GPU, m <= 51)
    TV *const Vb = reinterpret_cast<TV *>(a.V);
    const T vs = a.vs, vsi = a.vsi;
    extern __shared__ __align__(16) unsigned char dsm_reg[];
    const int m = a.m, ldr = m + 1;
    // big (m + 1 > 52 columns): the basis is streamed in blocks of 52 columns
    // (phase B as an update pass plus a dot pass), the rotated Hessenberg R
    // lives in global memory (a.H.h, identical copies written by every CTA),
    // the per-step vectors stay in shared memory
    constexpr bool big = BIG;   // instantiated separately: m + 1 > 52
    const int nslot = big ? m + 2 : kFSlots;   // c1 / c2 vector length
    T *sR = big ? a.H.h : reinterpret_cast<T *>(dsm_reg);    // (m+1) x m rotated columns
    T *scs = big ? reinterpret_cast<T *>(dsm_reg) : sR + (int64_t)ldr * m;
    T *ssn = scs + m;
    T *sg = ssn + m;                           // m + 1
    T *sc1 = sg + (m + 1);                     // nslot
    T *sc2 = sc1 + nslot;                      // nslot
    T *sred = sc2 + nslot;                     // kFW * kFSlots
    T *sctmp = sred + kFW * kFSlots;           // big: nslot (the column being rotated)
    T *sstage = sctmp + (big ? nslot : 0);     // kFW * kCsrWarpBuf (CSR SpMV staging)
    const int xslot = big ? m + 1 : kFExtra;   // partial slot of the extra scalar
    __shared__ T s_gamma, s_beta, s_bn2;
    __shared__ PolyUnit<T> s_poly[kMaxPolyUnits];
    __shared__ int s_done, s_steps, s_break, s_app;
    __shared__ double s_scale;

    const int tid = threadIdx.x;
    const unsigned nb = gridDim.x;
    __shared__ unsigned long long s_prof[kProfSlots];
    unsigned long long t_last = 0;
    if (a.prof && tid < kProfSlots) s_prof[tid] = 0;
    if (a.prof) t_last = clock64();
#define MPK_MARK(i)                                   \
    if (a.prof) {                                     \
        __syncthreads();                              \
        if (tid == 0) {                               \
            const unsigned long long t_ = clock64();  \
            s_prof[i] += t_ - t_last;                 \
            t_last = t_;                              \
        }                                             \
    }
    const int64_t rpc = ((a.n + nb - 1) / nb + 63) / 64 * 64;   // rows per CTA, 64-aligned
    const int64_t rb = (int64_t)blockIdx.x * rpc;
    const int64_t re = (rb + rpc < a.n) ? rb + rpc : a.n;
    constexpr bool multi = MULTI;   // separate instantiations: the one-GPU kernel carries no comm code
    const CommArgs<T> *cmp = MULTI ? &a.cm : nullptr;
    // partials: single GPU -> local [slot][cta]; multi -> every rank's
    // [phase][slot][rank * nb + cta], reduced over nranks * nb columns
    const int64_t pblk = multi ? (int64_t)kFSlots * kXStride : (int64_t)nslot * kFMaxCtas;
    T *pbase = multi ? a.cm.part[a.cm.rank] : a.part;
    T *partA = pbase, *partB = pbase + pblk, *partC = pbase + 2 * pblk;
    const unsigned ncol = multi ? nb * (unsigned)a.cm.nranks : nb;
    const int pstride = multi ? kXStride : kFMaxCtas;
    unsigned long long ep = multi ? __ldcg(a.cm.epoch) : 0ull;
    const bool lead = (blockIdx.x == 0);
    // one grid barrier (all ranks when multi); true = a rank timed out
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
#define MPK_SYNC_OR_ABORT()                        \
    if (sync_all()) {                              \
        if (lead && tid == 0) a.ctl->pad_ = 1;     \
        finish();                                  \
        return;                                    \
    }

    if (POLY && tid < a.npoly) s_poly[tid] = a.poly[tid];
    // built at the (rare) use sites from the kernel parameters: a struct
    // live across the cycle would cost the streaming phases registers
#define MPK_POLY_BUFS PolyBufs<T>{s_poly, a.npoly, a.pw0, a.pw1, a.pt, a.pacc, a.bar}
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
    if (multi) {
        // v_0 = r0 / gamma reads halo rows of r0: stage r0 in the rank's
        // global-length vector (the w'' slot) and mirror the boundary rows
        for (int64_t r = rb + tid; r < re; r += kFB) {
            const T v = a.r0[r];
            a.wpp[r] = v;
            for (int q = 0; q < a.cm.nranks; ++q)
                if (q != a.cm.rank && r >= a.cm.mir_lo[q] && r < a.cm.mir_hi[q]) a.cm.xg[q][a.cm.row0 + r] = v;
        }
        MPK_SYNC_OR_ABORT();
    }

    for (int k = 0; k < a.cap && !s_done; ++k) {
        const int nc = k + 1;
        MPK_MARK(12);
        const T *src = (k == 0 && !multi) ? a.r0 : a.wpp;
        const T dv = (k == 0) ? s_gamma : s_beta;
        TV *vk = Vb + (int64_t)k * a.ld;
        T acc[C::KP];
        T ext = T(0);
        // ---------------- phase A: v_k = src/dv, w = A v_k, ||w||^2 ; c1 = V^T w
        T an = T(0);
        {
            // own rows of v_k in 16-byte groups (rb is 64-aligned), scalar tail
            constexpr int R = C::R;
            const int64_t rv = rb + (re - rb) / R * R;
            int64_t r = rb + (int64_t)tid * R;
            constexpr int64_t S = (int64_t)kFB * R;
            for (; r + 3 * S < rv; r += 4 * S) {
                Pack<T> q[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) q[u] = ldcg16(src + r + u * S);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
#pragma unroll
                    for (int e = 0; e < R; ++e) q[u].v[e] = RN<T>::div(q[u].v[e], dv);
                    stv<T, TV>(vk + r + u * S, q[u], vs);
#pragma unroll
                    for (int e = 0; e < R; ++e) q[u].v[e] = IO::get(IO::put(q[u].v[e], vs), vsi);   // as stored
                    if (a.diag) {
#pragma unroll
                        for (int e = 0; e < R; ++e) q[u].v[e] = RN<T>::div(q[u].v[e], __ldg(a.diag + r + u * S + e));
                        stcg16(a.z + r + u * S, q[u]);
                    }
                }
            }
            for (; r < rv; r += S) {
                Pack<T> q = ldcg16(src + r);
#pragma unroll
                for (int e = 0; e < R; ++e) q.v[e] = RN<T>::div(q.v[e], dv);
                stv<T, TV>(vk + r, q, vs);
#pragma unroll
                for (int e = 0; e < R; ++e) q.v[e] = IO::get(IO::put(q.v[e], vs), vsi);
                if (a.diag) {
#pragma unroll
                    for (int e = 0; e < R; ++e) q.v[e] = RN<T>::div(q.v[e], __ldg(a.diag + r + e));
                    stcg16(a.z + r, q);
                }
            }
            for (int64_t t = rv + tid; t < re; t += kFB) {
                const TV hv = IO::put(RN<T>::div(__ldcg(src + t), dv), vs);
                vk[t] = hv;
                const T v = IO::get(hv, vsi);
                if (a.diag) a.z[t] = RN<T>::div(v, __ldg(a.diag + t));
            }
        }
        MPK_MARK(0);
        __syncthreads();
        if (POLY) {
            // right preconditioning by the GMRES polynomial: z = p(A) v_k,
            // then w = A z (gmres.py:181-182)
            MPK_SYNC_OR_ABORT();   // v_k complete on every CTA
            poly_apply_dev<T>(A, MPK_POLY_BUFS, reinterpret_cast<const T *>(vk), rb, re, sstage);
            MPK_SYNC_OR_ABORT();   // z complete
            an = poly_spmv_dev<T>(A, a.pacc, a.w, rb, re, sstage);
        } else if (!MULTI && a.vk_sync) {
            // wide halo (3-D stencils: +-nx^2 rows, about a CTA's slab):
            // make v_k (and z) complete on every CTA, then read every SpMV
            // input from the stored column instead of re-forming the halo
            // as w''/beta -- the same values, without a division each
            MPK_SYNC_OR_ABORT();
            an = phase_a_spmv<T>(A, XSlab<T, TV>{src, vk, dv, 0, a.n, a.diag, a.z, vs, vsi}, a.w, rb, re, sstage);
        } else {
            an = phase_a_spmv<T>(A, XSlab<T, TV>{src, vk, dv, rb, re, a.diag, a.z, vs, vsi}, a.w, rb, re, sstage);
        }
        MPK_MARK(1);
        __syncthreads();   // w rows of this CTA visible to the other lanes' 16-byte loads
        const int nbk = BIG ? (nc + kRegMaxCols - 1) / kRegMaxCols : 1;   // column blocks
        auto blk = [&](int bi, int total, int &c0, int &cn) {
            c0 = bi * kRegMaxCols;
            cn = (total - c0 < kRegMaxCols) ? total - c0 : kRegMaxCols;
        };
        if (!BIG) {
#pragma unroll
            for (int i = 0; i < C::KP; ++i) acc[i] = T(0);
            reg_phase<T, kRegDots, TV>(Vb, a.ld, nc, rb, re, a.n, a.w, nullptr, nullptr, acc, ext, nullptr, nullptr,
                                   (3 * k) & 1, vsi);
            MPK_MARK(2);
            reg_write_partials<T>(acc, nc, an, sred, partA, cmp, 0, 0, true, xslot);
        } else {
            for (int bi = 0; bi < nbk; ++bi) {
                int c0, cn;
                blk(bi, nc, c0, cn);
#pragma unroll
                for (int i = 0; i < C::KP; ++i) acc[i] = T(0);
                reg_phase<T, kRegDots, TV>(Vb + (int64_t)c0 * a.ld, a.ld, cn, rb, re, a.n, a.w, nullptr, nullptr, acc,
                                       ext);
                reg_write_partials<T>(acc, cn, an, sred, partA, nullptr, 0, c0, bi == nbk - 1, xslot);
            }
            MPK_MARK(2);
        }
        MPK_SYNC_OR_ABORT();
        MPK_MARK(3);
        cross_reduce<T>(partA, ncol, nc, nc + 1, sc1, pstride, xslot);   // sc1[0..k], sc1[nc] = ||w||^2
        __syncthreads();
        MPK_MARK(4);
        // ---------------- phase B: w' = w - V c1 ; c2 = V^T w'
        if (!BIG) {
#pragma unroll
            for (int i = 0; i < C::KP; ++i) acc[i] = T(0);
            reg_phase<T, kRegUpdateDots, TV>(Vb, a.ld, nc, rb, re, a.n, a.w, a.wp, sc1, acc, ext, nullptr, nullptr,
                                         (3 * k + 1) & 1, vsi);
            MPK_MARK(5);
            reg_write_partials<T>(acc, nc, T(0), sred, partB, cmp, pblk, 0, true, xslot);
        } else {
            // w' accumulated block by block in place (an update pass), then the
            // dot pass V^T w' (the basis is read twice in this phase)
            for (int bi = 0; bi < nbk; ++bi) {
                int c0, cn;
                blk(bi, nc, c0, cn);
                T dummy = T(0);
                reg_phase<T, kRegUpdateNorm, TV>(Vb + (int64_t)c0 * a.ld, a.ld, cn, rb, re, a.n, bi ? a.wp : a.w, a.wp,
                                             sc1 + c0, acc, dummy);
                __syncthreads();
            }
            for (int bi = 0; bi < nbk; ++bi) {
                int c0, cn;
                blk(bi, nc, c0, cn);
#pragma unroll
                for (int i = 0; i < C::KP; ++i) acc[i] = T(0);
                reg_phase<T, kRegDots, TV>(Vb + (int64_t)c0 * a.ld, a.ld, cn, rb, re, a.n, a.wp, nullptr, nullptr, acc,
                                       ext);
                reg_write_partials<T>(acc, cn, T(0), sred, partB, nullptr, pblk, c0, false, xslot);
            }
            MPK_MARK(5);
        }
        MPK_SYNC_OR_ABORT();
        MPK_MARK(6);
        cross_reduce<T>(partB, ncol, nc, nc, sc2, pstride, xslot);
        __syncthreads();
        MPK_MARK(7);
        // ---------------- phase C: w'' = w' - V c2 ; ||w''||^2
        T bn = T(0);
        if (!BIG) {
            reg_phase<T, kRegUpdateNorm, TV>(Vb, a.ld, nc, rb, re, a.n, a.wp, a.wpp, sc2, acc, bn, cmp, nullptr,
                                         (3 * k + 2) & 1, vsi);
        } else {
            for (int bi = 0; bi < nbk; ++bi) {
                int c0, cn;
                blk(bi, nc, c0, cn);
                T dummy = T(0);
                reg_phase<T, kRegUpdateNorm, TV>(Vb + (int64_t)c0 * a.ld, a.ld, cn, rb, re, a.n, bi ? a.wpp : a.wp,
                                             a.wpp, sc2 + c0, acc, bi == nbk - 1 ? bn : dummy);
                __syncthreads();
            }
        }
        MPK_MARK(8);
        reg_write_partials<T>(acc, 0, bn, sred, partC, cmp, 2 * pblk, 0, true, xslot);
        MPK_SYNC_OR_ABORT();
        MPK_MARK(9);
        cross_reduce<T>(partC, ncol, 0, 1, &s_bn2, pstride, xslot);
        __syncthreads();
        MPK_MARK(10);
        // ---------------- beta, append test, Givens (every CTA, identical)
        T *col = big ? sctmp : sR + (int64_t)k * ldr;
        for (int i = tid; i < nc; i += kFB) col[i] = RN<T>::add(sc1[i], sc2[i]);
        __syncthreads();
        if (tid == 0)
            givens_step<T>(a, k, nc, ldr, col, s_bn2, sc1[nc], s_scale, lead, scs, ssn, sg, s_beta, s_steps, s_done,
                           s_break);
        __syncthreads();
        if (big)   // every CTA keeps its own (identical) copy of R in global memory
            for (int i = tid; i <= nc; i += kFB) sR[(int64_t)k * ldr + i] = col[i];
    }
    // R's last column was stored by several warps (global memory when big):
    // visible to back_substitute's warp 0 regardless of profiling
    __threadfence_block();
    __syncthreads();

    MPK_MARK(11);
    // ---------------- epilogue: d = R \ g, x_out = x0 + V_k d
    const int k = s_steps;
    T *sd = sc1;
    if (k > 0 && tid < 32) back_substitute<T>(a, k, ldr, sR, sg, sc2, sd, lead, s_app);
    __syncthreads();
    finish();
    if (k > 0 && s_app) return;   // TriangularBreakdownError: x_out untouched
    if (lead) {
        for (int i = tid; i < k; i += kFB) a.H.d[i] = sd[i];
        if (!big)
            for (int i = tid; i < k * ldr; i += kFB) a.H.h[i] = sR[i];
        for (int i = tid; i <= k; i += kFB) a.H.g[i] = sg[i];
    }
    if (a.final_col && k > 0 && !s_break) {
        TV *vn = Vb + (int64_t)k * a.ld;
        for (int64_t r = rb + tid; r < re; r += kFB) vn[r] = IO::put(RN<T>::div(a.wpp[r], s_beta), vs);
    }
    if (k == 0) {
        for (int64_t r = rb + tid; r < re; r += kFB) a.x_out[r] = a.x0[r];
        return;
    }
    {
        T acc[C::KP];
        T ext = T(0);
        if (POLY) {
            // x = x0 + p(A) (V_k d) (gmres.py:194-196): V_k d into the free
            // w' slot, then the polynomial, then the update
            reg_phase<T, kRegCorrect, TV>(Vb, a.ld, k, rb, re, a.n, nullptr, a.wp, sd, acc, ext, nullptr, nullptr,
                                          (3 * k) & 1, vsi);
            MPK_SYNC_OR_ABORT();
            poly_apply_dev<T>(A, MPK_POLY_BUFS, a.wp, rb, re, sstage);
            for (int64_t r = rb + tid; r < re; r += kFB) a.x_out[r] = RN<T>::add(a.x0[r], a.pacc[r]);
        } else if (!BIG) {
            reg_phase<T, kRegCorrect, TV>(Vb, a.ld, k, rb, re, a.n, a.x0, a.x_out, sd, acc, ext, nullptr, a.diag,
                                      (3 * k) & 1, vsi);   // after step k-1's phase C (index 3k-1)
        } else {   // big: x += V_b d_b block by block (no diagonal preconditioner here)
            for (int c0 = 0; c0 < k; c0 += kRegMaxCols) {
                const int cn = (k - c0 < kRegMaxCols) ? k - c0 : kRegMaxCols;
                reg_phase<T, kRegCorrect, TV>(Vb + (int64_t)c0 * a.ld, a.ld, cn, rb, re, a.n, c0 ? a.x_out : a.x0,
                                          a.x_out, sd + c0, acc, ext);
                __syncthreads();
            }
        }
    }
    MPK_MARK(13);
    if (a.prof && tid < kProfSlots) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        // slot 15: the SM this CTA ran on (tools/cta_balance.py)
        g_fused_prof[blockIdx.x * kProfSlots + tid] = (tid == kProfSlots - 1) ? (unsigned long long)smid : s_prof[tid];
    }
#undef MPK_MARK
#undef MPK_SYNC_OR_ABORT
#undef MPK_POLY_BUFS
}

}  // namespace mpk
