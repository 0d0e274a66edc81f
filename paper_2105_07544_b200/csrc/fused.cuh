// Shared machinery of the persistent cooperative cycle kernels
// (k_cycle_reg in fused_reg.cuh, k_cycle_dcgs2 in fused_dcgs2.cuh):
// one CTA of kFB threads per SM, CTA b owning the rows [b*rpc, (b+1)*rpc) of
// the whole cycle (gmres.py:134-205 with kernels.py:98-216); grid barriers
// (cross-GPU when row-partitioned), fixed-order cross-CTA reductions after
// each barrier so every CTA holds bit-identical coefficients, the redundant
// per-CTA Givens update (kernels.py:166-196) and the back-substitution
// (kernels.py:202-216).
//
// A TMA-ring variant of the cycle (basis tiles HBM -> shared memory by
// cp.async.bulk.tensor, mbarrier ring) lived here in round 1; it measured
// 256 vs 178 us/iteration on C2 and a round-2 probe of warp-specialised
// bulk-copy rings (tools/micro/stream_b.cu) streamed at 1.4-3.7 TB/s against
// 5.3-7.5 TB/s for the register streams, so it was removed.
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

// Row-partitioned multi-GPU cycle (one process per GPU, or virtual ranks
// sharing one GPU in tests): peer pointers to every rank's partial buffer,
// arrival counter and global-length x buffer (all P2P-mapped; for the local
// rank they are its own).  See k_cycle_reg.
constexpr int kMaxRanks = MPK_MAX_RANKS;
constexpr int kXStride = kMaxRanks * kFMaxCtas;   // partial columns: rank * nb + cta
template <typename T> struct CommArgs {
    int rank, nranks;
    T *part[kMaxRanks];                      // 3 phases x kFSlots x kXStride
    unsigned long long *xbar[kMaxRanks];     // arrival counters (monotonic)
    unsigned long long *epoch;               // own barriers completed (persists across launches)
    T *xg[kMaxRanks];                        // global-length vectors, global row 0
    int64_t row0;                            // first global row of this rank
    int64_t mir_lo[kMaxRanks], mir_hi[kMaxRanks];   // own local rows mirrored into rank q's xg
};

// GMRES-polynomial preconditioner inside the persistent cycle
// (apply_gmres_poly, preconditioners.py:276-305): one unit per real root
// (a = 1/theta) or conjugate pair (a = 2 Re theta, b = |theta|^2), Leja order.
constexpr int kMaxPolyUnits = 32;
template <typename T> struct PolyUnit {
    int pair;
    T a, b;
};

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
    int prof;         // phase profiler on
    CommArgs<T> cm;   // nranks > 1: row-partitioned cycle
    const T *diag;    // k_cycle_reg: diagonal right preconditioner a_ii (block Jacobi k = 1), or nullptr
    T *z;             // k_cycle_reg: z = v_k / a_ii for the CTA's own rows
    T vs = T(1), vsi = T(1);   // k_cycle_reg, binary16 basis: stored = v * vs (power of two), vsi = 1 / vs
    int vk_sync = 0;           // k_cycle_reg: grid barrier after v_k, all SpMV inputs from the stored column
    // k_cycle_reg with a GMRES-polynomial right preconditioner (npoly > 0):
    // z = p(A) v_k and the correction's p(A) (V_k d) evaluated in-kernel,
    // one grid barrier per SpMV; pw0/pw1 ping-pong the product-form work
    // vector, pt the pair temporary, pacc the accumulator (z)
    int npoly = 0;
    PolyUnit<T> poly[kMaxPolyUnits];
    T *pw0 = nullptr, *pw1 = nullptr, *pt = nullptr, *pacc = nullptr;
};

// x accessor over a global vector written by other CTAs of this persistent
// kernel (after a grid barrier): L2 loads, never a stale L1 line
template <typename T> struct XCG {
    const T *p;
    __device__ __forceinline__ T operator()(int64_t c) const { return __ldcg(p + c); }
    __device__ __forceinline__ Pack<T> vec(int64_t c) const { return ldcg16(p + c); }
};

// Phase profiler (desc flag bit 3): per-CTA clock64 totals of each section,
// read back with mpk_fused_prof_read.  Sections: 0 v_k, 1 SpMV, 2 stream A,
// 3 barrier A, 4 reduce A, 5 stream B, 6 barrier B, 7 reduce B, 8 stream C,
// 9 barrier C, 10 reduce C, 11 Givens, 12 epilogue.
constexpr int kProfSlots = 16;
__device__ unsigned long long g_fused_prof[kFMaxCtas * kProfSlots];

// Sense-free grid barrier (all CTAs co-resident by cooperative launch).
// Release/acquire at GPU scope instead of two full fences: the arrival is an
// acq_rel atomic (publishes this CTA's partials, which __syncthreads ordered
// before thread 0's arrival), the last arrival releases the generation word,
// waiters acquire it.  bar[0] (count) and bar[1] (generation) are the
// caller's words (bar[0] count, bar[32] generation: the caller's 256-byte
// counter block).
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned *p, unsigned v) {
    asm volatile("st.relaxed.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned nb) {
    unsigned *gen = bar + 32;   // own 128-byte line: polls do not queue behind the arrivals
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = ld_acquire_gpu(gen);
        if (atom_add_acq_rel_gpu(bar, 1u) == nb - 1) {
            st_relaxed_gpu(bar, 0u);
            st_release_gpu(gen, g0 + 1u);
        } else {
            while (ld_acquire_gpu(gen) == g0) __nanosleep(20);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Grid barrier spanning all ranks: local arrival as in grid_sync; the last
// local CTA publishes the rank's arrival to every rank's counter (system-
// scope atomics through the P2P mapping) and waits until its own counter
// shows all ranks' arrivals for barrier number `target`, then releases the
// local CTAs.  The fences order every CTA's P2P partial/halo stores before
// the arrival.  A rank that never arrives (crashed peer, or virtual ranks
// not co-resident) trips a 20 s timeout instead of hanging the GPU: bar[2]
// is set and every CTA returns true (abort).
template <typename T>
__device__ __forceinline__ bool grid_sync_x(unsigned *bar, unsigned nb, const CommArgs<T> &cm,
                                            unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *vgen = bar + 1;
        const unsigned g0 = *vgen;
        __threadfence_system();
        if (atomicAdd(bar, 1u) == nb - 1) {
            bar[0] = 0u;
            __threadfence_system();
            for (int q = 0; q < cm.nranks; ++q) atomicAdd_system(cm.xbar[q], 1ull);
            volatile unsigned long long *mine = cm.xbar[cm.rank];
            const unsigned long long need = (unsigned long long)cm.nranks * target;
            const unsigned long long t0 = globaltimer_ns();
            while (*mine < need) {
                __nanosleep(64);
                if (globaltimer_ns() - t0 > 20000000000ull) {
                    atomicExch(bar + 2, 1u);
                    break;
                }
            }
            __threadfence_system();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == g0) __nanosleep(32);
        }
        __threadfence_system();
    }
    __syncthreads();
    return *(volatile unsigned *)(bar + 2) != 0u;
}

// out[s] = sum over CTAs b (fixed order) of part[idx(s)][b], for slots
// s < nslots, idx(s) = s for s < ncols else kFExtra.  One warp per slot,
// lanes stride the CTAs, then a fixed butterfly: identical in every CTA.
template <typename T>
__device__ __forceinline__ void cross_reduce(const T *part, unsigned nb, int ncols, int nslots, T *out,
                                             int stride = kFMaxCtas, int xslot = kFExtra) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NQ = (kFSlots + kFW - 1) / kFW;   // slots per warp
    if (nb <= 160u) {
      // one CTA per SM (148 on B200): every slot's loads of this warp are
      // issued before any is reduced (one L2 round trip, not one per slot);
      // more than NQ * kFW slots (m > 78) go in rounds
      for (int s0 = 0; s0 < nslots; s0 += NQ * kFW) {
        constexpr int NI = 5;
        T v[NQ][NI];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int s = s0 + warp + kFW * q;
            const T *p = part + (int64_t)((s < ncols) ? s : xslot) * stride;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const unsigned b = lane + 32 * i;
                v[q][i] = (s < nslots && b < nb) ? __ldcg(p + b) : T(0);
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int s = s0 + warp + kFW * q;
            T acc = T(0);
#pragma unroll
            for (int i = 0; i < NI; ++i) acc += v[q][i];
            acc = warp_sum(acc);
            if (lane == 0 && s < nslots) out[s] = acc;
        }
      }
      return;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int s = warp + kFW * q;
        if (s < nslots) {
            const int idx = (s < ncols) ? s : xslot;
            const T *p = part + (int64_t)idx * stride;
            T acc = T(0);
            // nb columns (multi-rank: nranks * CTAs per rank), same fixed order;
            // unrolled so the loads of a slot are in flight together
#pragma unroll 8
            for (unsigned b = lane; b < nb; b += 32) acc += __ldcg(p + b);
            acc = warp_sum(acc);
            if (lane == 0) out[s] = acc;
        }
    }
}

// beta, the append test (kernels.py:122-123) and the Givens update of column
// k (kernels.py:166-196) on one thread; every CTA runs it on identical inputs.
template <typename T, class Args>
__device__ __forceinline__ void givens_step(const Args &a, int k, int nc, int ldr, T *col, T bn2, T wn2, double scale,
                                            bool lead, T *scs, T *ssn, T *sg, T &s_beta, int &s_steps, int &s_done,
                                            int &s_break) {
    const T beta = RN<T>::sqrt_(bn2);
    s_beta = beta;
    col[nc] = beta;
    const T wnorm = RN<T>::sqrt_(wn2);
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
    const double rel = fabs((double)gk) / scale;
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

// d = R[:k,:k] \ g[:k] on one warp (kernels.py:202-216), with the
// TriangularBreakdownError guard min|diag| <= k*u*max|diag| (s_app = 1).
template <typename T, class Args>
__device__ __forceinline__ void back_substitute(const Args &a, int k, int ldr, const T *sR, const T *sg, T *rhs, T *sd,
                                                bool lead, int &s_app) {
    const int tid = threadIdx.x;
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

// x accessor of phase A: v_k = src / dv, read back from V[:, k] for the
// CTA's own rows (written just before, one division per row) and divided on
// the fly for halo rows owned by other CTAs (not yet written by them).  Own
// rows go through L1 (this SM wrote them; neighbouring rows share lines).
//
// With a diagonal (block-Jacobi k = 1) right preconditioner the SpMV input is
// z = M v_k = v_k / a_ii (lu_solve of a 1x1 block, preconditioners.py:133-139,
// one IEEE division): own rows from the z slab, halo rows recomputed with the
// same two roundings.
// Basis column v_k stored in TV (T, or binary16 scaled by vs): 4 or 2
// elements of T from 16 or 8 bytes of TV
template <typename T, typename TV> __device__ __forceinline__ Pack<T> ldv(const TV *p, T vsi) {
    if constexpr (sizeof(TV) == sizeof(T)) {
        return ldcg16(p);
    } else {
        static_assert(sizeof(T) == 4 && sizeof(TV) == 2, "16-bit basis with fp32 arithmetic");
        const uint2 w = __ldcg(reinterpret_cast<const uint2 *>(p));
        TV h[4];
        memcpy(h, &w, 8);
        Pack<T> q;
#pragma unroll
        for (int e = 0; e < 4; ++e) q.v[e] = VIO<T, TV>::get(h[e], vsi);
        return q;
    }
}
template <typename T, typename TV> __device__ __forceinline__ void stv(TV *p, const Pack<T> &q, T vs) {
    if constexpr (sizeof(TV) == sizeof(T)) {
        stcg16(p, q);
    } else {
        TV h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = VIO<T, TV>::put(q.v[e], vs);
        uint2 w;
        memcpy(&w, h, 8);
        __stcg(reinterpret_cast<uint2 *>(p), w);
    }
}

// SpMV input of phase A: x = v_k.  Own rows [rb, re) read the stored basis
// column vk (written by this CTA just before); halo rows are formed on the
// fly as src / d (the reference's w / beta, kernels.py:125) and rounded to
// the basis storage exactly as the owner stored them, so every row of the
// product sees the same v_k.  With a diagonal right preconditioner the input
// is z = v_k / a_ii instead.
template <typename T, typename TV = T> struct XSlab {
    const T *src;
    const TV *vk;
    T d;
    int64_t rb, re;
    const T *diag = nullptr;   // a_ii (device), or identity
    const T *z = nullptr;      // own rows of z = v_k / a_ii
    T vs = T(1), vsi = T(1);   // binary16 basis scaling
    __device__ __forceinline__ T rnd(T v) const { return VIO<T, TV>::get(VIO<T, TV>::put(v, vs), vsi); }
    __device__ __forceinline__ T operator()(int64_t c) const {
        if (c >= rb && c < re) return diag ? z[c] : VIO<T, TV>::get(vk[c], vsi);
        const T v = rnd(RN<T>::div(__ldcg(src + c), d));
        return diag ? RN<T>::div(v, __ldg(diag + c)) : v;
    }
    // 16-byte group of T starting at c (c and the CTA bounds are group-aligned,
    // so the whole group is own or halo)
    __device__ __forceinline__ Pack<T> vec(int64_t c) const {
        const bool own = c >= rb && c < re;
        if (own) return diag ? ldcg16(z + c) : ldv<T, TV>(vk + c, vsi);
        Pack<T> q = ldcg16(src + c);
#pragma unroll
        for (int e = 0; e < (int)(16 / sizeof(T)); ++e) {
            q.v[e] = rnd(RN<T>::div(q.v[e], d));
            if (diag) q.v[e] = RN<T>::div(q.v[e], __ldg(diag + c + e));
        }
        return q;
    }
};

}  // namespace mpk
