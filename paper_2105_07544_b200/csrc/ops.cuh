// Row operators: CSR and matrix-free stencil rows with the reference's exact
// summation order.
//
// mpkrylov.spmv (sparse.py:190-206) is SciPy csr_matvec: per row, a running
// sum starting at 0 adds value*x[col] over the stored entries in storage
// order, rounding after each multiply and add.  Both operators below do the
// same with explicit _rn intrinsics, so they are bit-identical to the
// reference.  The stencil operator regenerates generate_stencil's values
// (stencils.py:78-207) on the fly, in the reference's operation order, so it
// is bit-identical to the CSR product of the assembled matrix while reading
// only x and writing y.
#pragma once

#include "common.cuh"

namespace mpk {

// Products staged per warp for the warp-cooperative CSR rows (elements of T):
// K entries per lane per chunk, 8 by default (16 is ~10% faster on the
// ~50-entry rows of config 5 in fp32 but 25-35% slower on 5-7-entry stencil
// rows; callers with long rows pick 16).
constexpr int kCsrWarpBuf = 512;               // staging elements per warp (K <= 16)

template <typename T> struct CsrOp {
    int64_t n;
    const int32_t *__restrict__ rp;
    const int32_t *__restrict__ ci;
    const T *__restrict__ v;
    // x-window half-width (0: off).  Banded matrices (90-99%
    // of the columns within +-2000 of the row) gather x from a shared-memory
    // copy of x[R - band, R + T + band) for a chunk of T rows (csr_chunk);
    // the global gathers of irregular rows otherwise saturate L1 (one
    // wavefront per entry: C5 ran at 90% L1/TEX throughput, 28% DRAM).
    int64_t band = 0;
    int64_t nnz_ = 0;    // stored entries (row statistics for the window choice)

    template <class X> __device__ __forceinline__ T row(int64_t r, X x) const {
        const int32_t p0 = __ldg(rp + r), p1 = __ldg(rp + r + 1);
        T acc = T(0);
        for (int32_t p = p0; p < p1; ++p)
            acc = RN<T>::add(acc, RN<T>::mul(__ldg(v + p), x((int64_t)__ldg(ci + p))));
        return acc;
    }

    // Rows [r0, min(r0 + 32, rend)) by one full warp, lane i owning row
    // r0 + i: the warp walks the rows' contiguous entry range in chunks of
    // 32 x kCsrStage, every lane loading consecutive entries (coalesced
    // values / column indices) and staging the rounded products value*x[col]
    // in shared memory in storage order; each lane then adds its own row's
    // products left to right.  Same roundings in the same order as
    // csr_matvec (sparse.py:190-206), so bit-identical to row(), at
    // coalesced-load speed for long, irregular rows.  `sb`: kCsrWarpBuf
    // elements of this warp.  Returns the lane's row value (0 past rend).
    template <int K = 8, class X> __device__ __forceinline__ T warp_rows(int64_t r0, int64_t rend, X x, T *sb) const {
        constexpr int kCsrStage = K;
        constexpr int kChunk = 32 * kCsrStage;
        const int lane = threadIdx.x & 31;
        const int64_t last = (r0 + 32 < rend ? r0 + 32 : rend) - 1;
        const bool mine = r0 + lane <= last;
        int32_t ps = 0, pe = 0;
        if (mine) {
            ps = __ldg(rp + r0 + lane);
            pe = __ldg(rp + r0 + lane + 1);
        }
        const int32_t base = __ldg(rp + r0), end = __ldg(rp + last + 1);
        T acc = T(0);
        int32_t p = ps;
        // software pipeline: the next chunk's values / column indices are in
        // flight while this chunk's x entries are gathered
        T va[kCsrStage];
        int32_t ca[kCsrStage];
#pragma unroll
        for (int j = 0; j < kCsrStage; ++j) {
            const int32_t e = base + j * 32 + lane;
            va[j] = (e < end) ? __ldg(v + e) : T(0);
            ca[j] = (e < end) ? __ldg(ci + e) : 0;
        }
        for (int32_t cb = base; cb < end; cb += kChunk) {
            T xs[kCsrStage];
#pragma unroll
            for (int j = 0; j < kCsrStage; ++j)   // columns may be negative (row blocks): mask by position
                xs[j] = (cb + j * 32 + lane < end) ? x((int64_t)ca[j]) : T(0);
            T vn[kCsrStage];
            int32_t cn[kCsrStage];
#pragma unroll
            for (int j = 0; j < kCsrStage; ++j) {
                const int32_t e = cb + kChunk + j * 32 + lane;
                vn[j] = (e < end) ? __ldg(v + e) : T(0);
                cn[j] = (e < end) ? __ldg(ci + e) : 0;
            }
#pragma unroll
            for (int j = 0; j < kCsrStage; ++j) sb[j * 32 + lane] = RN<T>::mul(va[j], xs[j]);
            __syncwarp();
            const int32_t ce = (cb + kChunk < pe) ? cb + kChunk : pe;
            for (; p < ce; ++p) acc = RN<T>::add(acc, sb[p - cb]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < kCsrStage; ++j) {
                va[j] = vn[j];
                ca[j] = cn[j];
            }
        }
        return acc;
    }
    static constexpr bool kStencil = false;
};

// x accessor of a chunk: columns inside [lo, hi) from the shared-memory
// window, the rest (far columns) through the wrapped accessor.  Same values,
// so the row sums stay bit-identical.
template <typename T, class X> struct XWin {
    X x;
    const T *sx;
    int64_t lo, hi;
    __device__ __forceinline__ T operator()(int64_t c) const { return (c >= lo && c < hi) ? sx[c - lo] : x(c); }
};

// Rows [R, Re) of a CSR operator by the whole CTA: x[lo, hi) (lo = R - band,
// hi = Re + band, clipped to [0, n)) is staged in `sx` (coalesced), then the
// warps evaluate 32-row groups with warp_rows<K> reading x through the
// window; fn(r, y_r) runs on the lane owning row r.  All threads of the CTA
// must call it (two __syncthreads).
template <int K, typename T, class X, class F>
__device__ __forceinline__ void csr_chunk(const CsrOp<T> &A, X x, int64_t R, int64_t Re, T *sx, T *sb, F &&fn) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t lo = R - A.band > 0 ? R - A.band : 0;
    const int64_t hi = Re + A.band < A.n ? Re + A.band : A.n;
    __syncthreads();   // the previous chunk's readers are done with sx
    for (int64_t c = lo + threadIdx.x; c < hi; c += blockDim.x) sx[c - lo] = x(c);
    __syncthreads();
    const XWin<T, X> xw{x, sx, lo, hi};
    for (int64_t r0 = R + (int64_t)warp * 32; r0 < Re; r0 += (int64_t)nw * 32) {
        const T y = A.template warp_rows<K>(r0, Re, xw, sb);
        if (r0 + lane < Re) fn(r0 + lane, y);
    }
}

// Division by a grid-invariant divisor (nx, nx^2) without the integer
// divider: q = (umulhi(x, mul) + x) >> shift, exact for x < 2^31.
struct FastDiv {
    uint32_t d, mul, shift;
    __host__ void init(uint32_t dv) {
        d = dv;
        shift = 0;
        while ((1ull << shift) < dv) ++shift;
        mul = (uint32_t)(((1ull << 32) * ((1ull << shift) - dv)) / dv + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t x) const {
        return (__umulhi(x, mul) + x) >> shift;
    }
};

// Host-computed constants of a stencil preset (double, reference formulas).
struct StencilConsts {
    int preset;
    int nx;
    int64_t row0;        // first global row of this block
    int64_t nglob;       // nx^2 or nx^3
    double c[9];         // constant coefficients (displacement order)
    double h, hh;        // h = 1/(nx+1), hh = 0.5*h      (BentPipe)
    double cc2, ncc2;    // c*2.0 and (-c)*2.0            (BentPipe)
    FastDiv dnx, dnxy;   // division by nx and nx^2 (n < 2^31)
};

template <typename T> struct StencilOp {
    int64_t n;
    StencilConsts k;
    T cT[9];

    template <class X> __device__ __forceinline__ T row(int64_t r, X x) const {
        const uint32_t g = (uint32_t)(k.row0 + r);
        const int nx = k.nx;
        T acc = T(0);
        const uint32_t q1 = k.dnx.div(g);
        const int ix = (int)(g - q1 * (uint32_t)nx);
        if (k.preset == MPK_LAPLACE3D) {
            const int64_t nxy = (int64_t)nx * nx;
            const uint32_t iz_ = k.dnxy.div(g);
            const int iy = (int)(q1 - iz_ * (uint32_t)nx), iz = (int)iz_;
            if (iz > 0) acc = RN<T>::add(acc, RN<T>::mul(cT[0], x(r - nxy)));
            if (iy > 0) acc = RN<T>::add(acc, RN<T>::mul(cT[1], x(r - nx)));
            if (ix > 0) acc = RN<T>::add(acc, RN<T>::mul(cT[2], x(r - 1)));
            acc = RN<T>::add(acc, RN<T>::mul(cT[3], x(r)));
            if (ix < nx - 1) acc = RN<T>::add(acc, RN<T>::mul(cT[4], x(r + 1)));
            if (iy < nx - 1) acc = RN<T>::add(acc, RN<T>::mul(cT[5], x(r + nx)));
            if (iz < nx - 1) acc = RN<T>::add(acc, RN<T>::mul(cT[6], x(r + nxy)));
            return acc;
        }
        const int iy = (int)q1;
        if (k.preset == MPK_STRETCHED2D) {
            const bool W = ix > 0, E = ix < nx - 1, S = iy > 0, N = iy < nx - 1;
            if (W && S) acc = RN<T>::add(acc, RN<T>::mul(cT[0], x(r - nx - 1)));
            if (S) acc = RN<T>::add(acc, RN<T>::mul(cT[1], x(r - nx)));
            if (E && S) acc = RN<T>::add(acc, RN<T>::mul(cT[2], x(r - nx + 1)));
            if (W) acc = RN<T>::add(acc, RN<T>::mul(cT[3], x(r - 1)));
            acc = RN<T>::add(acc, RN<T>::mul(cT[4], x(r)));
            if (E) acc = RN<T>::add(acc, RN<T>::mul(cT[5], x(r + 1)));
            if (W && N) acc = RN<T>::add(acc, RN<T>::mul(cT[6], x(r + nx - 1)));
            if (N) acc = RN<T>::add(acc, RN<T>::mul(cT[7], x(r + nx)));
            if (E && N) acc = RN<T>::add(acc, RN<T>::mul(cT[8], x(r + nx + 1)));
            return acc;
        }
        T c0 = cT[0], c1 = cT[1], c2 = cT[2], c3 = cT[3], c4 = cT[4];
        if (k.preset == MPK_BENTPIPE2D) {
            // stencils.py:104-115, evaluated left to right as numpy does
            const double px = __dmul_rn((double)(ix + 1), k.h);
            const double py = __dmul_rn((double)(iy + 1), k.h);
            const double ux = __dmul_rn(__dmul_rn(k.cc2, py), __dsub_rn(1.0, __dmul_rn(px, px)));
            const double uy = __dmul_rn(__dmul_rn(k.ncc2, px), __dsub_rn(1.0, __dmul_rn(py, py)));
            c0 = RN<T>::from_double(__dsub_rn(-1.0, __dmul_rn(k.hh, uy)));
            c1 = RN<T>::from_double(__dsub_rn(-1.0, __dmul_rn(k.hh, ux)));
            c3 = RN<T>::from_double(__dadd_rn(-1.0, __dmul_rn(k.hh, ux)));
            c4 = RN<T>::from_double(__dadd_rn(-1.0, __dmul_rn(k.hh, uy)));
        }
        if (iy > 0) acc = RN<T>::add(acc, RN<T>::mul(c0, x(r - nx)));
        if (ix > 0) acc = RN<T>::add(acc, RN<T>::mul(c1, x(r - 1)));
        acc = RN<T>::add(acc, RN<T>::mul(c2, x(r)));
        if (ix < nx - 1) acc = RN<T>::add(acc, RN<T>::mul(c3, x(r + 1)));
        if (iy < nx - 1) acc = RN<T>::add(acc, RN<T>::mul(c4, x(r + nx)));
        return acc;
    }
    // Rows [r, r + R) of one grid line (R = 16 / sizeof(T); needs r % R == 0
    // and group_ok()): the S/N (and B/U) neighbours and the rows themselves
    // are R-wide vector reads (xv), the W of the first and the E of the last
    // row two scalar reads (xs); every row's products are added in the
    // reference's displacement order, so out[] equals row(r + e).
    static constexpr int R = 16 / (int)sizeof(T);
    __device__ __forceinline__ bool group_ok() const {
        return k.preset != MPK_STRETCHED2D && k.nx % R == 0 && k.row0 % R == 0;
    }
    // Inputs of one row group (group_load), so callers can issue several
    // groups' loads before evaluating any (group_eval): the neighbour packs
    // a group needs (pb/pu: Laplace3D only) and the W/E end values.
    struct GroupIn {
        Pack<T> c, pb, ps, pn, pu;
        T xw, xe;
    };
    template <class XV, class XS>
    __device__ __forceinline__ void group_load(int64_t r, XV xv, XS xs, GroupIn &in) const {
        const uint32_t g = (uint32_t)(k.row0 + r);
        const int nx = k.nx;
        const uint32_t q1 = k.dnx.div(g);
        const int ix0 = (int)(g - q1 * (uint32_t)nx);
        in.c = xv(r);
        in.xw = (ix0 > 0) ? xs(r - 1) : T(0);
        in.xe = (ix0 + R - 1 < nx - 1) ? xs(r + R) : T(0);
        if (k.preset == MPK_LAPLACE3D) {
            const int64_t nxy = (int64_t)nx * nx;
            const uint32_t iz_ = k.dnxy.div(g);
            const int iy = (int)(q1 - iz_ * (uint32_t)nx), iz = (int)iz_;
            if (iz > 0) in.pb = xv(r - nxy);
            if (iy > 0) in.ps = xv(r - nx);
            if (iy < nx - 1) in.pn = xv(r + nx);
            if (iz < nx - 1) in.pu = xv(r + nxy);
            return;
        }
        const int iy = (int)q1;
        if (iy > 0) in.ps = xv(r - nx);
        if (iy < nx - 1) in.pn = xv(r + nx);
    }
    __device__ __forceinline__ void group_eval(int64_t r, const GroupIn &in, T (&out)[R]) const {
        const uint32_t g = (uint32_t)(k.row0 + r);
        const int nx = k.nx;
        const uint32_t q1 = k.dnx.div(g);
        const int ix0 = (int)(g - q1 * (uint32_t)nx);
        const Pack<T> &c = in.c;
        const T xw = in.xw, xe = in.xe;
        if (k.preset == MPK_LAPLACE3D) {
            const uint32_t iz_ = k.dnxy.div(g);
            const int iy = (int)(q1 - iz_ * (uint32_t)nx), iz = (int)iz_;
            const bool B = iz > 0, S = iy > 0, N = iy < nx - 1, U = iz < nx - 1;
#pragma unroll
            for (int e = 0; e < R; ++e) {
                const int ix = ix0 + e;
                T acc = T(0);
                if (B) acc = RN<T>::add(acc, RN<T>::mul(cT[0], in.pb.v[e]));
                if (S) acc = RN<T>::add(acc, RN<T>::mul(cT[1], in.ps.v[e]));
                if (ix > 0) acc = RN<T>::add(acc, RN<T>::mul(cT[2], e ? c.v[e ? e - 1 : 0] : xw));
                acc = RN<T>::add(acc, RN<T>::mul(cT[3], c.v[e]));
                if (ix < nx - 1) acc = RN<T>::add(acc, RN<T>::mul(cT[4], e < R - 1 ? c.v[e < R - 1 ? e + 1 : 0] : xe));
                if (N) acc = RN<T>::add(acc, RN<T>::mul(cT[5], in.pn.v[e]));
                if (U) acc = RN<T>::add(acc, RN<T>::mul(cT[6], in.pu.v[e]));
                out[e] = acc;
            }
            return;
        }
        const int iy = (int)q1;
        const bool S = iy > 0, N = iy < nx - 1;
        double pyc = 0.0, py1 = 0.0;
        if (k.preset == MPK_BENTPIPE2D) {
            const double py = __dmul_rn((double)(iy + 1), k.h);
            pyc = __dmul_rn(k.cc2, py);                      // (c*2.0)*py
            py1 = __dsub_rn(1.0, __dmul_rn(py, py));         // 1 - py*py
        }
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int ix = ix0 + e;
            T c0 = cT[0], c1 = cT[1], c2 = cT[2], c3 = cT[3], c4 = cT[4];
            if (k.preset == MPK_BENTPIPE2D) {
                // stencils.py:104-115, same operations and order as row()
                const double px = __dmul_rn((double)(ix + 1), k.h);
                const double ux = __dmul_rn(pyc, __dsub_rn(1.0, __dmul_rn(px, px)));
                const double uy = __dmul_rn(__dmul_rn(k.ncc2, px), py1);
                c0 = RN<T>::from_double(__dsub_rn(-1.0, __dmul_rn(k.hh, uy)));
                c1 = RN<T>::from_double(__dsub_rn(-1.0, __dmul_rn(k.hh, ux)));
                c3 = RN<T>::from_double(__dadd_rn(-1.0, __dmul_rn(k.hh, ux)));
                c4 = RN<T>::from_double(__dadd_rn(-1.0, __dmul_rn(k.hh, uy)));
            }
            T acc = T(0);
            if (S) acc = RN<T>::add(acc, RN<T>::mul(c0, in.ps.v[e]));
            if (ix > 0) acc = RN<T>::add(acc, RN<T>::mul(c1, e ? c.v[e ? e - 1 : 0] : xw));
            acc = RN<T>::add(acc, RN<T>::mul(c2, c.v[e]));
            if (ix < nx - 1) acc = RN<T>::add(acc, RN<T>::mul(c3, e < R - 1 ? c.v[e < R - 1 ? e + 1 : 0] : xe));
            if (N) acc = RN<T>::add(acc, RN<T>::mul(c4, in.pn.v[e]));
            out[e] = acc;
        }
    }
    template <class XV, class XS>
    __device__ __forceinline__ void row_group(int64_t r, XV xv, XS xs, T (&out)[R]) const {
        GroupIn in;
        group_load(r, xv, xs, in);
        group_eval(r, in, out);
    }
    // Stored entries of row r in the reference's column order
    // (generate_stencil, stencils.py:192-207: displacement order, Dirichlet
    // truncation): emit(col, value) with the coefficients row() multiplies
    // by (double for the binary64 assembly).  Returns the entry count.
    template <class F> __device__ __forceinline__ int row_entries(int64_t r, F &&emit) const {
        const uint32_t g = (uint32_t)(k.row0 + r);
        const int nx = k.nx;
        const uint32_t q1 = k.dnx.div(g);
        const int ix = (int)(g - q1 * (uint32_t)nx);
        int cnt = 0;
        auto put = [&](bool ok, int64_t c, T v) {
            if (ok) {
                emit(c, v);
                ++cnt;
            }
        };
        if (k.preset == MPK_LAPLACE3D) {
            const int64_t nxy = (int64_t)nx * nx;
            const uint32_t iz_ = k.dnxy.div(g);
            const int iy = (int)(q1 - iz_ * (uint32_t)nx), iz = (int)iz_;
            put(iz > 0, r - nxy, cT[0]);
            put(iy > 0, r - nx, cT[1]);
            put(ix > 0, r - 1, cT[2]);
            put(true, r, cT[3]);
            put(ix < nx - 1, r + 1, cT[4]);
            put(iy < nx - 1, r + nx, cT[5]);
            put(iz < nx - 1, r + nxy, cT[6]);
            return cnt;
        }
        const int iy = (int)q1;
        if (k.preset == MPK_STRETCHED2D) {
            const bool W = ix > 0, E = ix < nx - 1, S = iy > 0, N = iy < nx - 1;
            put(W && S, r - nx - 1, cT[0]);
            put(S, r - nx, cT[1]);
            put(E && S, r - nx + 1, cT[2]);
            put(W, r - 1, cT[3]);
            put(true, r, cT[4]);
            put(E, r + 1, cT[5]);
            put(W && N, r + nx - 1, cT[6]);
            put(N, r + nx, cT[7]);
            put(E && N, r + nx + 1, cT[8]);
            return cnt;
        }
        T c0 = cT[0], c1 = cT[1], c2 = cT[2], c3 = cT[3], c4 = cT[4];
        if (k.preset == MPK_BENTPIPE2D) {
            const double px = __dmul_rn((double)(ix + 1), k.h);
            const double py = __dmul_rn((double)(iy + 1), k.h);
            const double ux = __dmul_rn(__dmul_rn(k.cc2, py), __dsub_rn(1.0, __dmul_rn(px, px)));
            const double uy = __dmul_rn(__dmul_rn(k.ncc2, px), __dsub_rn(1.0, __dmul_rn(py, py)));
            c0 = RN<T>::from_double(__dsub_rn(-1.0, __dmul_rn(k.hh, uy)));
            c1 = RN<T>::from_double(__dsub_rn(-1.0, __dmul_rn(k.hh, ux)));
            c3 = RN<T>::from_double(__dadd_rn(-1.0, __dmul_rn(k.hh, ux)));
            c4 = RN<T>::from_double(__dadd_rn(-1.0, __dmul_rn(k.hh, uy)));
        }
        put(iy > 0, r - nx, c0);
        put(ix > 0, r - 1, c1);
        put(true, r, c2);
        put(ix < nx - 1, r + 1, c3);
        put(iy < nx - 1, r + nx, c4);
        return cnt;
    }
    // lane-per-row over [r0, r0 + 32) (interface of CsrOp::warp_rows)
    template <class X> __device__ __forceinline__ T warp_rows(int64_t r0, int64_t rend, X x, T *) const {
        const int64_t r = r0 + (threadIdx.x & 31);
        return r < rend ? row(r, x) : T(0);
    }
    static constexpr bool kStencil = true;
};

// x accessors
template <typename T> struct XPlain {
    const T *__restrict__ p;
    __device__ __forceinline__ T operator()(int64_t c) const { return p[c]; }
    __device__ __forceinline__ Pack<T> vec(int64_t c) const { return *reinterpret_cast<const Pack<T> *>(p + c); }
};
// x = src / d, exactly the reference's basis column w / beta (kernels.py:125)
template <typename T> struct XScaled {
    const T *__restrict__ p;
    T d;
    __device__ __forceinline__ T operator()(int64_t c) const { return RN<T>::div(p[c], d); }
    __device__ __forceinline__ Pack<T> vec(int64_t c) const {
        Pack<T> q = *reinterpret_cast<const Pack<T> *>(p + c);
#pragma unroll
        for (int e = 0; e < (int)(16 / sizeof(T)); ++e) q.v[e] = RN<T>::div(q.v[e], d);
        return q;
    }
};
// same, reading through L2 (data written by other CTAs of a persistent kernel)
template <typename T> struct XScaledCG {
    const T *p;
    T d;
    __device__ __forceinline__ T operator()(int64_t c) const { return RN<T>::div(__ldcg(p + c), d); }
};

}  // namespace mpk
