// Shared device helpers for libmpkb200 (sm_100a).
//
// Arithmetic rules: everything that must reproduce the
// reference bit-for-bit uses the explicit round-to-nearest intrinsics
// (__fmul_rn/__fadd_rn/__dmul_rn/__dadd_rn) so nvcc never contracts a
// multiply-add into an FMA; the library is built without fast-math, so `/`
// and sqrt are IEEE round-to-nearest and fp32 subnormals are preserved.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <type_traits>

#include "../../include/mpk_b200.h"

namespace mpk {

constexpr int kBlock = 256;          // threads per CTA for streaming kernels
constexpr int kMaxCols = 64;         // columns handled in registers per pass

template <typename T> struct RN;
template <> struct RN<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
    static __device__ __forceinline__ double hypot_(double a, double b) { return hypot(a, b); }
    static __device__ __forceinline__ double from_double(double a) { return a; }
};
template <> struct RN<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
    static __device__ __forceinline__ float hypot_(float a, float b) { return hypotf(a, b); }
    static __device__ __forceinline__ float from_double(double a) { return __double2float_rn(a); }
};

template <typename T> __device__ __forceinline__ T ldcg(const T *p) { return __ldcg(p); }

// 16-byte row groups (4 fp32 / 2 fp64 consecutive rows)
template <typename T> struct alignas(16) Pack {
    T v[16 / sizeof(T)];
};

// L2-cached 16-byte loads with a 256-byte L2 sector prefetch hint: a warp's
// 128-byte column segment also pulls in the neighbouring warp's segment
__device__ __forceinline__ Pack<float> ldcg16(const float *p) {
    Pack<float> r;
    asm volatile("ld.global.cg.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ Pack<double> ldcg16(const double *p) {
    Pack<double> r;
    asm volatile("ld.global.cg.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
    return r;
}
__device__ __forceinline__ void stcg16(float *p, const Pack<float> &v) {
    __stcg(reinterpret_cast<float4 *>(p), make_float4(v.v[0], v.v[1], v.v[2], v.v[3]));
}
__device__ __forceinline__ void stcg16(double *p, const Pack<double> &v) {
    __stcg(reinterpret_cast<double2 *>(p), make_double2(v.v[0], v.v[1]));
}

// binary16 basis storage (SolverConfig.basis_precision = "binary16", fp32
// cycles): 16-byte groups of 8 halves
__device__ __forceinline__ Pack<__half> ldcg16(const __half *p) {
    Pack<__half> r;
    uint32_t w[4];
    asm volatile("ld.global.cg.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p));
    memcpy(&r, w, 16);
    return r;
}

__device__ __forceinline__ Pack<__nv_bfloat16> ldcg16(const __nv_bfloat16 *p) {
    Pack<__nv_bfloat16> r;
    uint32_t w[4];
    asm volatile("ld.global.cg.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p));
    memcpy(&r, w, 16);
    return r;
}

// Basis element I/O: V stored in TV, arithmetic in T.  For TV == T the
// value itself; binary16 stores v*s and reads back h*(1/s) with s a power of
// two (exact scaling: it only moves the normalised basis entries, ~1/sqrt(n),
// into binary16's normal range).
template <typename T, typename TV> struct VIO {
    static __device__ __forceinline__ T get(TV v, T) { return v; }
    static __device__ __forceinline__ TV put(T v, T) { return v; }
};
template <> struct VIO<float, __half> {
    static __device__ __forceinline__ float get(__half v, float si) { return __fmul_rn(__half2float(v), si); }
    static __device__ __forceinline__ __half put(float v, float s) { return __float2half_rn(__fmul_rn(v, s)); }
};
// bfloat16 (8-bit significand, fp32's exponent range): the same power-of-two
// scaling is kept for uniformity (exact, and harmless to the range)
template <> struct VIO<float, __nv_bfloat16> {
    static __device__ __forceinline__ float get(__nv_bfloat16 v, float si) { return __fmul_rn(__bfloat162float(v), si); }
    static __device__ __forceinline__ __nv_bfloat16 put(float v, float s) { return __float2bfloat16_rn(__fmul_rn(v, s)); }
};

// Raw (unscaled) values of a 16-byte basis group as T: the binary16 stream
// kernels fold the power-of-two scale into their coefficients / partial sums
// instead of multiplying every element (exact either way).
template <typename T, typename TV>
__device__ __forceinline__ void raw_vals(const Pack<TV> &p, T (&o)[16 / sizeof(TV)]) {
    if constexpr (sizeof(TV) == sizeof(T)) {
#pragma unroll
        for (int e = 0; e < (int)(16 / sizeof(TV)); ++e) o[e] = p.v[e];
    } else if constexpr (std::is_same<TV, __half>::value) {
        const __half2 *h = reinterpret_cast<const __half2 *>(p.v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 f = __half22float2(h[q]);
            o[2 * q] = f.x;
            o[2 * q + 1] = f.y;
        }
    } else {
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(p.v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(h[q]);
            o[2 * q] = f.x;
            o[2 * q + 1] = f.y;
        }
    }
}

// R consecutive elements of T (16 or 32 bytes) through L2
template <typename T, int R> __device__ __forceinline__ void ldrows(const T *p, T (&o)[R]) {
    constexpr int E = 16 / (int)sizeof(T);
    static_assert(R % E == 0, "whole 16-byte groups");
#pragma unroll
    for (int q = 0; q < R / E; ++q) {
        const Pack<T> v = ldcg16(p + q * E);
#pragma unroll
        for (int e = 0; e < E; ++e) o[q * E + e] = v.v[e];
    }
}
template <typename T, int R> __device__ __forceinline__ void strows(T *p, const T (&o)[R]) {
    constexpr int E = 16 / (int)sizeof(T);
#pragma unroll
    for (int q = 0; q < R / E; ++q) {
        Pack<T> v;
#pragma unroll
        for (int e = 0; e < E; ++e) v.v[e] = o[q * E + e];
        stcg16(p + q * E, v);
    }
}

// R consecutive elements of T stored as TV (T, or a 16-bit basis holding
// v * vs): one 16-byte store of 8 halves, or strows
template <typename T, typename TV, int R> __device__ __forceinline__ void stvrows(TV *p, const T (&o)[R], T vs) {
    if constexpr (sizeof(TV) == sizeof(T)) {
        strows<T, R>(p, o);
    } else {
        static_assert(R * sizeof(TV) == 16, "one 16-byte group of the 16-bit basis");
        Pack<TV> h;
#pragma unroll
        for (int e = 0; e < R; ++e) h.v[e] = VIO<T, TV>::put(o[e], vs);
        uint4 w;
        memcpy(&w, &h, 16);
        __stcg(reinterpret_cast<uint4 *>(p), w);
    }
}

// Warp-level sum (fixed butterfly order -> deterministic).
template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Reduce NC per-thread accumulators plus one extra scalar across the CTA:
// out[c] = CTA total of column c (c < ncols), out[ncols] = CTA total of
// `extra`.  `sm` needs (blockDim/32) * (NC+1) elements.  Deterministic:
// fixed shuffle tree, then warps summed in index order.
template <typename T, int NC>
__device__ __forceinline__ void block_reduce_cols(T (&acc)[NC], int ncols, T extra, T *sm, T *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    constexpr int S = NC + 1;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c < ncols) {
            T v = warp_sum(acc[c]);
            if (lane == 0) sm[warp * S + c] = v;
        }
    }
    {
        T v = warp_sum(extra);
        if (lane == 0) sm[warp * S + NC] = v;
    }
    __syncthreads();
    for (int c = threadIdx.x; c <= ncols; c += blockDim.x) {
        const int cc = (c == ncols) ? NC : c;
        T s = sm[cc];
        for (int w = 1; w < nw; ++w) s += sm[w * S + cc];
        out[c] = s;
    }
    __syncthreads();
}

// Grid-wide "last CTA finishes the reduction" protocol.  Every CTA writes its
// partial row, then takes a ticket; the CTA drawing the last ticket sees all
// partials (after the fence) and resets the counter for the next launch.
__device__ __forceinline__ bool last_cta(unsigned *counter) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// Second stage: the last CTA sums partials[nblk][stride] (ncols columns
// plus the extra at index ncols) in a fixed order: thread t folds partial
// rows t, t+B, ... into registers (independent loads), then one CTA column
// reduction.  Results: out[0..ncols].
template <typename T, int NC>
__device__ __forceinline__ void reduce_partials(const T *partials, int nblk, int stride, int ncols,
                                                T *sm, T *out) {
    T acc[NC];
    T extra = T(0);
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = T(0);
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
        const T *row = partials + (int64_t)b * stride;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c < ncols) acc[c] += ldcg(row + c);
        extra += ldcg(row + ncols);
    }
    block_reduce_cols<T, NC>(acc, ncols, extra, sm, out);
}

// Workspace carved out of the caller's reduction buffer.
struct RedWs {
    unsigned *counters;   // 16 ticket counters (zero-initialised by the caller)
    void *partials;       // max_blocks * stride elements
    void *sums;           // 256 elements: reduced results
};

__host__ __device__ inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

}  // namespace mpk
