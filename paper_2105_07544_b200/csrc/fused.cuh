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
//      through L2), ||w||^2; then c1 = V[:,0..k]^T w       -> barrier, reduce
//   B  w' = w - V c1 (row-wise), c2 = V^T w' (column-wise) -> barrier, reduce
//   C  w'' = w' - V c2, ||w''||^2                          -> barrier, reduce
//      beta, append test (kernels.py:122), Givens (kernels.py:183-196), exit
//
// Streaming: the basis and the work vector of a phase are moved HBM ->
// shared memory by the TMA engine (cp.async.bulk, one bulk copy per column
// of a TR-row tile, completion on an mbarrier) through a 4-stage, 32 KB/stage
// ring, so bytes in flight are bounded by shared memory, not registers.  Each
// tile is consumed from shared memory: row-wise combinations (thread per row,
// P = 512/TR column parts summed in fixed order) and column-wise dots (one
// warp per column).  HBM sees every basis column exactly once per phase.
//
// Epilogue: each CTA back-substitutes R d = g (kernels.py:202-216) from its
// shared-memory copy of R and forms x_out = x0 + V_k d for its own rows.
#pragma once

#include "kernels.cuh"
#include "tma.cuh"

namespace mpk {

constexpr int kFB = 512;                // threads per CTA
constexpr int kFW = kFB / 32;           // warps per CTA
constexpr int kFMaxCols = 64;           // m + 1 <= 64
constexpr int kFQ = kFMaxCols / kFW;    // columns owned per warp
constexpr int kFExtra = kFMaxCols;      // partial slot of the extra scalar
constexpr int kFSlots = kFMaxCols + 1;
constexpr int kFMaxCtas = 320;          // per-slot stride of the partials
constexpr int kMaxStages = 8;           // TMA ring depth (upper bound)
constexpr int kRingBytes = 176 * 1024;  // shared memory of the ring
constexpr int kCB = 16;                 // basis columns per tensor-map box
constexpr int kMaxTR = 256;             // rows per tile, upper bound (TR is a template parameter)

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


// Shared-memory ring of TMA stages.  A stage holds a TR-row tile of the
// basis columns [0, nv) (ceil(nv/kCB) tensor-map boxes of TR x kCB, column
// c at offset c*TR) followed by the tile of one work vector (1-D bulk copy).
// The number of stages adapts to the tile size; `phase` holds the next wait
// parity of each mbarrier (identical in every thread).
struct Ring {
    unsigned char *base;
    uint64_t *full;
    uint32_t phase;
};

template <typename T>
__device__ __forceinline__ void ring_issue(Ring &R, int slot, size_t sbytes, int TR, const CUtensorMap *tmV, int nv,
                                           const T *vec, int64_t t0) {
    T *stage = reinterpret_cast<T *>(R.base + (size_t)slot * sbytes);
    const int nbox = (nv + kCB - 1) / kCB;
    const uint32_t boxb = (uint32_t)(TR * kCB * sizeof(T));
    const uint32_t vb = (uint32_t)(TR * sizeof(T));
    mbar_arrive_expect_tx(&R.full[slot], boxb * nbox + (vec ? vb : 0u));
    for (int b = 0; b < nbox; ++b)
        tma_load_2d(stage + (int64_t)b * kCB * TR, tmV, (int)t0, b * kCB, &R.full[slot]);
    if (vec) bulk_g2s(stage + (int64_t)nbox * kCB * TR, vec + t0, vb, &R.full[slot]);
}

// Stream the CTA's rows [rb, re) in TR-row tiles of (V[:, 0..nv) | vec) and
// call consume(stage, vec_tile, t0, rows) on each; all threads participate,
// thread 0 issues the copies.
template <typename T, int TR, class F>
__device__ __forceinline__ void stream_phase(Ring &R, int64_t rb, int64_t re, const CUtensorMap *tmV, int nv,
                                             const T *vec, F &&consume) {
    const int nbox = (nv + kCB - 1) / kCB;
    const size_t sbytes = ((size_t)(nbox * kCB + 1) * TR * sizeof(T) + 127) / 128 * 128;
    int S = (int)(kRingBytes / sbytes);
    if (S > kMaxStages) S = kMaxStages;
    const int ntiles = (re > rb) ? (int)((re - rb + TR - 1) / TR) : 0;
    fence_proxy_async_global();   // generic writes (own rows of V, w, w') before TMA reads
    __syncthreads();
    if (threadIdx.x == 0) {
        const int pre = ntiles < S ? ntiles : S;
        for (int i = 0; i < pre; ++i) ring_issue<T>(R, i, sbytes, TR, tmV, nv, vec, rb + (int64_t)i * TR);
    }
    for (int i = 0; i < ntiles; ++i) {
        const int slot = i % S;
        mbar_wait(&R.full[slot], (R.phase >> slot) & 1u);
        R.phase ^= 1u << slot;
        const int64_t t0 = rb + (int64_t)i * TR;
        const int rows = (int)((re - t0) < TR ? (re - t0) : TR);
        const T *st = reinterpret_cast<const T *>(R.base + (size_t)slot * sbytes);
        consume(st, st + (int64_t)nbox * kCB * TR, t0, rows);
        __syncthreads();          // every thread is done with the stage before it is refilled
        if (threadIdx.x == 0 && i + S < ntiles)
            ring_issue<T>(R, slot, sbytes, TR, tmV, nv, vec, rb + (int64_t)(i + S) * TR);
    }
}

// Strided dot over columns c = c0, c0+P, ... < nc of stage[c][rr] * coef[c]
// with four independent accumulators (combined in a fixed order).
template <typename T>
__device__ __forceinline__ T strided_combine(const T *stage, int TR, int rr, int c0, int P, int nc, const T *coef) {
    T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
    int c = c0;
    for (; c + 3 * P < nc; c += 4 * P) {
        s0 += stage[(int64_t)c * TR + rr] * coef[c];
        s1 += stage[(int64_t)(c + P) * TR + rr] * coef[c + P];
        s2 += stage[(int64_t)(c + 2 * P) * TR + rr] * coef[c + 2 * P];
        s3 += stage[(int64_t)(c + 3 * P) * TR + rr] * coef[c + 3 * P];
    }
    for (; c < nc; c += P) s0 += stage[(int64_t)c * TR + rr] * coef[c];
    return (s0 + s1) + (s2 + s3);
}

// Row-wise s[rr] = sum_{c < nc} stage[c][rr] * coef[c] for rr < rows; calls
// fin(rr, s).  TR >= kFB: each thread owns rows tid, tid+kFB, ...; TR < kFB:
// P = kFB/TR threads share a row (columns strided by P), partial sums
// combined in part order through `spart` (P*TR elements).
template <typename T, class Fin>
__device__ __forceinline__ void tile_rowcombine(const T *stage, int TR, int rows, int nc, const T *coef, T *spart,
                                                Fin &&fin) {
    const int tid = threadIdx.x;
    if (TR >= kFB) {
        for (int rr = tid; rr < rows; rr += kFB) fin(rr, strided_combine<T>(stage, TR, rr, 0, 1, nc, coef));
        return;
    }
    const int P = kFB / TR, rr = tid % TR, p = tid / TR;
    spart[p * TR + rr] = strided_combine<T>(stage, TR, rr, p, P, nc, coef);
    __syncthreads();
    if (p == 0 && rr < rows) {
        T t = spart[rr];
        for (int q = 1; q < P; ++q) t += spart[q * TR + rr];
        fin(rr, t);
    }
}

// Column-wise acc[q] += sum_{rr < rows} stage[c][rr] * x[rr] for the warp's
// columns c = warp + kFW*q < nc (rows past `rows` are masked by x == 0).
template <typename T>
__device__ __forceinline__ void tile_coldots(const T *stage, int TR, int rows, int nc, const T *x, T (&acc)[kFQ]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kFQ; ++q) {
        const int c = warp + kFW * q;
        if (c < nc) {
            const T *col = stage + (int64_t)c * TR;
            T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
            int rr = lane;
            for (; rr + 96 < rows; rr += 128) {
                s0 += col[rr] * x[rr];
                s1 += col[rr + 32] * x[rr + 32];
                s2 += col[rr + 64] * x[rr + 64];
                s3 += col[rr + 96] * x[rr + 96];
            }
            for (; rr < rows; rr += 32) s0 += col[rr] * x[rr];
            acc[q] += (s0 + s1) + (s2 + s3);
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
template <typename T> struct XSlab {
    const T *src;
    const T *vk;
    T d;
    int64_t rb, re;
    const T *diag = nullptr;   // a_ii (device), or identity
    const T *z = nullptr;      // own rows of z = v_k / a_ii
    __device__ __forceinline__ T operator()(int64_t c) const {
        if (c >= rb && c < re) return diag ? z[c] : vk[c];
        const T v = RN<T>::div(__ldcg(src + c), d);
        return diag ? RN<T>::div(v, __ldg(diag + c)) : v;
    }
    // 16-byte group starting at c (c and the CTA bounds are group-aligned,
    // so the whole group is own or halo)
    __device__ __forceinline__ Pack<T> vec(int64_t c) const {
        const bool own = c >= rb && c < re;
        Pack<T> q = ldcg16((own ? (diag ? z : vk) : src) + c);
        if (!own) {
#pragma unroll
            for (int e = 0; e < (int)(16 / sizeof(T)); ++e) {
                q.v[e] = RN<T>::div(q.v[e], d);
                if (diag) q.v[e] = RN<T>::div(q.v[e], __ldg(diag + c + e));
            }
        }
        return q;
    }
};

template <typename T, class Op, int TR>
__global__ void __launch_bounds__(kFB, 1) k_cycle_fused(Op A, FusedArgs<T> a, const __grid_constant__ CUtensorMap tmV) {
    extern __shared__ __align__(128) unsigned char dsm_raw[];
    const int m = a.m, ldr = m + 1;
    Ring R;
    R.base = dsm_raw;                                                    // kRingBytes
    R.full = reinterpret_cast<uint64_t *>(dsm_raw + kRingBytes);
    R.phase = 0;
    T *sR = reinterpret_cast<T *>(dsm_raw + kRingBytes + 8 * kMaxStages);   // (m+1) x m rotated columns
    T *scs = sR + (int64_t)ldr * m;
    T *ssn = scs + m;
    T *sg = ssn + m;                           // m + 1
    T *sc1 = sg + (m + 1);                     // kFSlots
    T *sc2 = sc1 + kFSlots;                    // kFSlots
    T *spart = sc2 + kFSlots;                  // kFB
    T *sx = spart + kFB;                       // TR (w' of the tile)
    T *sred = sx + kMaxTR;                     // kFW
    __shared__ T s_gamma, s_beta, s_bn2;
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
    T *partA = a.part, *partB = partA + (int64_t)kFSlots * kFMaxCtas,
      *partC = partB + (int64_t)kFSlots * kFMaxCtas;
    const bool lead = (blockIdx.x == 0);

    if (tid == 0) {
        for (int i = 0; i < kMaxStages; ++i) mbar_init(&R.full[i], 1);
        fence_mbar_init();
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
        MPK_MARK(12);
        const T *src = (k == 0) ? a.r0 : a.wpp;
        const T dv = (k == 0) ? s_gamma : s_beta;
        T *vk = a.V + (int64_t)k * a.ld;
        T acc[kFQ];
        // ---------------- phase A: v_k = src/dv, w = A v_k, ||w||^2 ; c1 = V^T w
        T an = T(0);
        {
            // own rows of v_k (4 independent loads in flight per thread)
            int64_t r = rb + tid;
            for (; r + 3 * kFB < re; r += 4 * kFB) {
                const T s0 = __ldcg(src + r), s1 = __ldcg(src + r + kFB), s2 = __ldcg(src + r + 2 * kFB),
                        s3 = __ldcg(src + r + 3 * kFB);
                vk[r] = RN<T>::div(s0, dv);
                vk[r + kFB] = RN<T>::div(s1, dv);
                vk[r + 2 * kFB] = RN<T>::div(s2, dv);
                vk[r + 3 * kFB] = RN<T>::div(s3, dv);
            }
            for (; r < re; r += kFB) vk[r] = RN<T>::div(__ldcg(src + r), dv);
        }
        MPK_MARK(0);
        __syncthreads();
        {
            // w = A v_k, four rows per thread per trip
            const XSlab<T> xs{src, vk, dv, rb, re};
            int64_t r = rb + tid;
            for (; r + 3 * kFB < re; r += 4 * kFB) {
                const T w0 = A.row(r, xs), w1 = A.row(r + kFB, xs), w2 = A.row(r + 2 * kFB, xs),
                        w3 = A.row(r + 3 * kFB, xs);
                a.w[r] = w0;
                a.w[r + kFB] = w1;
                a.w[r + 2 * kFB] = w2;
                a.w[r + 3 * kFB] = w3;
                an += w0 * w0;
                an += w1 * w1;
                an += w2 * w2;
                an += w3 * w3;
            }
            for (; r < re; r += kFB) {
                const T wr = A.row(r, xs);
                a.w[r] = wr;
                an += wr * wr;
            }
        }
        MPK_MARK(1);
#pragma unroll
        for (int q = 0; q < kFQ; ++q) acc[q] = T(0);
        stream_phase<T, TR>(R, rb, re, &tmV, nc, a.w, [&](const T *st, const T *wv, int64_t, int rows) {
            tile_coldots<T>(st, TR, rows, nc, wv, acc);
        });
        MPK_MARK(2);
        write_partials<T>(acc, nc, an, sred, partA);
        grid_sync(a.bar, nb);
        MPK_MARK(3);
        cross_reduce<T>(partA, nb, nc, nc + 1, sc1);   // sc1[0..k], sc1[nc] = ||w||^2
        __syncthreads();
        MPK_MARK(4);
        // ---------------- phase B: w' = w - V c1 ; c2 = V^T w'
#pragma unroll
        for (int q = 0; q < kFQ; ++q) acc[q] = T(0);
        stream_phase<T, TR>(R, rb, re, &tmV, nc, a.w, [&](const T *st, const T *wv, int64_t t0, int rows) {
            tile_rowcombine<T>(st, TR, rows, nc, sc1, spart, [&](int rr, T s) {
                const T wr = RN<T>::sub(wv[rr], s);
                a.wp[t0 + rr] = wr;
                sx[rr] = wr;
            });
            __syncthreads();
            tile_coldots<T>(st, TR, rows, nc, sx, acc);
        });
        MPK_MARK(5);
        write_partials<T>(acc, nc, T(0), sred, partB);
        grid_sync(a.bar, nb);
        MPK_MARK(6);
        cross_reduce<T>(partB, nb, nc, nc, sc2);
        __syncthreads();
        MPK_MARK(7);
        // ---------------- phase C: w'' = w' - V c2 ; ||w''||^2
        T bn = T(0);
        stream_phase<T, TR>(R, rb, re, &tmV, nc, a.wp, [&](const T *st, const T *wv, int64_t t0, int rows) {
            tile_rowcombine<T>(st, TR, rows, nc, sc2, spart, [&](int rr, T s) {
                const T wr = RN<T>::sub(wv[rr], s);
                a.wpp[t0 + rr] = wr;
                bn += wr * wr;
            });
        });
        MPK_MARK(8);
        {
            T dummy[kFQ];
#pragma unroll
            for (int q = 0; q < kFQ; ++q) dummy[q] = T(0);
            write_partials<T>(dummy, 0, bn, sred, partC);
        }
        grid_sync(a.bar, nb);
        MPK_MARK(9);
        cross_reduce<T>(partC, nb, 0, 1, &s_bn2);
        __syncthreads();
        MPK_MARK(10);
        // ---------------- beta, append test, Givens (every CTA, identical)
        T *col = sR + (int64_t)k * ldr;
        for (int i = tid; i < nc; i += kFB) col[i] = RN<T>::add(sc1[i], sc2[i]);
        __syncthreads();
        if (tid == 0)
            givens_step<T>(a, k, nc, ldr, col, s_bn2, sc1[nc], s_scale, lead, scs, ssn, sg, s_beta, s_steps, s_done,
                           s_break);
        __syncthreads();
    }

    MPK_MARK(11);
    // ---------------- epilogue: d = R \ g, x_out = x0 + V_k d
    const int k = s_steps;
    T *sd = sc1;
    if (k > 0 && tid < 32) back_substitute<T>(a, k, ldr, sR, sg, sc2, sd, lead, s_app);
    __syncthreads();
    if (k > 0 && s_app) return;   // TriangularBreakdownError: x_out untouched
    if (lead) {
        for (int i = tid; i < k; i += kFB) a.H.d[i] = sd[i];
        for (int i = tid; i < k * ldr; i += kFB) a.H.h[i] = sR[i];
        for (int i = tid; i <= k; i += kFB) a.H.g[i] = sg[i];
    }
    if (a.final_col && k > 0 && !s_break) {
        T *vn = a.V + (int64_t)k * a.ld;
        for (int64_t r = rb + tid; r < re; r += kFB) vn[r] = RN<T>::div(a.wpp[r], s_beta);
    }
    if (k == 0) {
        for (int64_t r = rb + tid; r < re; r += kFB) a.x_out[r] = a.x0[r];
        return;
    }
    stream_phase<T, TR>(R, rb, re, &tmV, k, (const T *)nullptr, [&](const T *st, const T *, int64_t t0, int rows) {
        tile_rowcombine<T>(st, TR, rows, k, sd, spart, [&](int rr, T s) {
            a.x_out[t0 + rr] = RN<T>::add(a.x0[t0 + rr], s);
        });
    });
    MPK_MARK(13);
    if (a.prof && tid < kProfSlots) g_fused_prof[blockIdx.x * kProfSlots + tid] = s_prof[tid];
#undef MPK_MARK
}

}  // namespace mpk
