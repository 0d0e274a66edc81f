// Phase-B stream probe (w' = w - V c ; c2 = V^T w' over a CTA's row slab),
// the dominant pass of the persistent Arnoldi cycle: register streaming
// (k_cycle_reg's reg_phase_u) vs a TMA bulk-copy ring through shared memory
// with per-stage mbarriers and "last warp out refills the stage" hand-off
// (no producer warp, no CTA-wide barrier per tile).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2105_07544_b200/csrc \
//        -o stream_b stream_b.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "common.cuh"
#include "tma.cuh"  // tools/micro/tma.cuh

using namespace mpk;

constexpr int NT = 512, NW = 16;
constexpr int G = 8, P = 4, KP = 13;   // 8 rows x 4 column parts per warp; 13 columns per part

// ---------------- register streaming (as k_cycle_reg), U row groups of 4 rows
__device__ __forceinline__ void pf_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int U, int PF = 0, int KUX = 0, int PFD = 0>
__global__ void __launch_bounds__(NT, 1) k_reg(const float *V, int64_t ld, int nc, int64_t n, const float *x,
                                               float *y, const float *coef, float *part, int rev) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane % G, p = lane / G;
    const int64_t rpc = ((n + gridDim.x - 1) / gridDim.x + 63) / 64 * 64;
    const int64_t rb = blockIdx.x * rpc, re = rb + rpc < n ? rb + rpc : n;
    constexpr int KU = KUX ? KUX : KP / U;
    constexpr int64_t TRIP = 32 * U;
    float acc[KU > KP ? KU : KP];
#pragma unroll
    for (int i = 0; i < KP; ++i) acc[i] = 0.f;
    float cf[KU];
#pragma unroll
    for (int i = 0; i < KU; ++i) cf[i] = (p + P * i < nc) ? coef[p + P * i] : 0.f;
    const int64_t b0 = rb + (int64_t)warp * TRIP, step = (int64_t)NW * TRIP;
    const int64_t ntrip = (b0 < re) ? (re - b0 + step - 1) / step : 0;
    // L2 prefetch (PF rows per chunk per column, one chunk ahead): warp 0,
    // lane c < nc prefetches column c, lane 31 the x rows
    const int64_t rows_per_round = (int64_t)NW * TRIP;
    int64_t next_pf = 0;   // rows (from the walk's start) already prefetched
    if (PF && warp == 0) {
        for (int64_t o = 0; o < 2 * PF && o < re - rb; o += PF) {
            const int64_t len = (re - rb - o < PF) ? re - rb - o : PF;
            const int64_t r0 = rev ? re - o - len : rb + o;
            const uint32_t by = (uint32_t)((len + 3) / 4 * 16);
            if (lane < nc) pf_l2(V + (int64_t)lane * ld + r0, by);
            if (lane == 31) pf_l2(x + r0, by);
        }
        next_pf = 2 * PF;
    }
    for (int64_t t = 0; t < ntrip; ++t) {
        const int64_t b = b0 + (rev ? ntrip - 1 - t : t) * step;
        if (PF && warp == 0) {
            const int64_t done = (t + 1) * rows_per_round;     // rows of the walk consumed after this round
            if (done + PF > next_pf && next_pf < re - rb) {
                const int64_t o = next_pf;
                const int64_t len = (re - rb - o < PF) ? re - rb - o : PF;
                const int64_t r0 = rev ? re - o - len : rb + o;
                const uint32_t by = (uint32_t)((len + 3) / 4 * 16);
                if (lane < nc) pf_l2(V + (int64_t)lane * ld + r0, by);
                if (lane == 31) pf_l2(x + r0, by);
                next_pf += PF;
            }
        }
        if (PFD > 0 && t + PFD < ntrip) {
            // software prefetch into L2 of the trip PFD ahead (no registers)
            const int64_t bp = b0 + (rev ? ntrip - 1 - (t + PFD) : t + PFD) * step;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t r = bp + (int64_t)(u * G + g) * 4;
                if (r < re) {
#pragma unroll
                    for (int i = 0; i < KU; ++i) {
                        const int c = p + P * i;
                        if (c < nc) asm volatile("prefetch.global.L2 [%0];" ::"l"(V + (int64_t)c * ld + r));
                    }
                }
            }
        }
        Pack<float> vv[U][KU], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = b + (int64_t)(u * G + g) * 4;
            const bool live = r < re;
#pragma unroll
            for (int i = 0; i < KU; ++i) {
                const int c = p + P * i;
                if (c < nc && live) vv[u][i] = ldcg16(V + (int64_t)c * ld + r);
                else for (int e = 0; e < 4; ++e) vv[u][i].v[e] = 0.f;
            }
            if (live) xv[u] = ldcg16(x + r);
            else for (int e = 0; e < 4; ++e) xv[u].v[e] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = b + (int64_t)(u * G + g) * 4;
            float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < KU; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[e] += vv[u][i].v[e] * cf[i];
#pragma unroll
            for (int o = G; o < 32; o <<= 1)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[e] += __shfl_xor_sync(0xffffffffu, s[e], o);
            Pack<float> yv;
#pragma unroll
            for (int e = 0; e < 4; ++e) yv.v[e] = __fsub_rn(xv[u].v[e], s[e]);
            if (p == 0 && r < re) stcg16(y + r, yv);
#pragma unroll
            for (int i = 0; i < KU; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[i] += vv[u][i].v[e] * yv.v[e];
        }
    }
    __shared__ float sm[NW * 64];
#pragma unroll
    for (int i = 0; i < KP; ++i) {
        float v = acc[i];
        for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (g == 0 && p + P * i < 64) sm[warp * 64 + p + P * i] = v;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += NT) {
        float s = 0.f;
        for (int w = 0; w < NW; ++w) s += sm[w * 64 + c];
        part[(int64_t)c * gridDim.x + blockIdx.x] = s;
    }
}

// ---------------- TMA ring: stage = [nc columns][TRP floats] + [x rows]
// tile = 128*U rows of the CTA's slab; lane (warp w, g, p) owns rows
// w*8 + g + 128*u of the tile and columns p + 4i.  Columns are padded to
// TRP = TR + 8 floats so the 4 parts hit different banks.
constexpr int kRing = 160 * 1024;
constexpr int kMaxStages = 8;

template <int U>
__global__ void __launch_bounds__(NT, 1) k_tma(const float *V, int64_t ld, int nc, int64_t n, const float *x,
                                               float *y, const float *coef, float *part, int rev) {
    extern __shared__ __align__(128) float ring[];
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ unsigned cnt[kMaxStages];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane % G, p = lane / G;
    const int64_t rpc = ((n + gridDim.x - 1) / gridDim.x + 63) / 64 * 64;
    const int64_t rb = blockIdx.x * rpc, re = rb + rpc < n ? rb + rpc : n;
    constexpr int TR = 128 * U, TRP = TR + 8;
    const int stage_f = (nc + 1) * TRP;                       // floats per stage
    int S = kRing / (stage_f * 4);
    if (S > kMaxStages) S = kMaxStages;
    const int64_t ntile = (re > rb) ? (re - rb + TR - 1) / TR : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            cnt[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t t) {   // one lane: tile t into stage t % S
        const int s = (int)(t % S);
        const int64_t tt = rev ? ntile - 1 - t : t;
        const int64_t r0 = rb + tt * TR;
        int64_t rows = re - r0 < TR ? re - r0 : TR;
        rows = (rows + 3) / 4 * 4;                           // buffers padded to 64 rows
        const uint32_t bytes = (uint32_t)rows * 4;
        float *st = ring + (size_t)s * stage_f;
        mbar_arrive_expect_tx(&full[s], bytes * (nc + 1));
        for (int c = 0; c < nc; ++c) bulk_g2s(st + c * TRP, V + (int64_t)c * ld + r0, bytes, &full[s]);
        bulk_g2s(st + nc * TRP, x + r0, bytes, &full[s]);
    };
    if (threadIdx.x == 0)
        for (int64_t t = 0; t < S && t < ntile; ++t) issue(t);
    constexpr int KU = KP;
    float acc[KP];
#pragma unroll
    for (int i = 0; i < KP; ++i) acc[i] = 0.f;
    float cf[KU];
#pragma unroll
    for (int i = 0; i < KU; ++i) cf[i] = (p + P * i < nc) ? coef[p + P * i] : 0.f;
    for (int64_t t = 0; t < ntile; ++t) {
        const int s = (int)(t % S);
        mbar_wait(&full[s], (uint32_t)((t / S) & 1));
        const float *st = ring + (size_t)s * stage_f;
        const int64_t tt = rev ? ntile - 1 - t : t;
        const int64_t r0 = rb + tt * TR;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int lr = warp * G + g + 128 * u;
            float vv[KU];
#pragma unroll
            for (int i = 0; i < KU; ++i) vv[i] = (p + P * i < nc) ? st[(p + P * i) * TRP + lr] : 0.f;
            float sum = 0.f;
#pragma unroll
            for (int i = 0; i < KU; ++i) sum += vv[i] * cf[i];
            sum += __shfl_xor_sync(0xffffffffu, sum, 8);
            sum += __shfl_xor_sync(0xffffffffu, sum, 16);
            const float yv = __fsub_rn(st[nc * TRP + lr], sum);
            if (p == 0 && r0 + lr < re) __stcg(y + r0 + lr, yv);
#pragma unroll
            for (int i = 0; i < KU; ++i) acc[i] += vv[i] * yv;
        }
        __syncwarp();
        if (lane == 0) {
            const unsigned old = atomicAdd(&cnt[s], 1u);
            if (old == NW - 1) {
                cnt[s] = 0;
                if (t + S < ntile) issue(t + S);
            }
        }
    }
    __shared__ float sm[NW * 64];
#pragma unroll
    for (int i = 0; i < KP; ++i) {
        float v = acc[i];
        for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (g == 0 && p + P * i < 64) sm[warp * 64 + p + P * i] = v;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += NT) {
        float s = 0.f;
        for (int w = 0; w < NW; ++w) s += sm[w * 64 + c];
        part[(int64_t)c * gridDim.x + blockIdx.x] = s;
    }
}

// ---------------- 2-D TMA ring: one tensor-map box (TR rows x nc columns,
// OOB columns zero-filled and not fetched) + one 1-D bulk copy of x per
// tile; lane = row, the thread holds all nc columns of its row.  Warp group
// q (4 warps) consumes tiles t = q mod 4, warp (w % 4) its 32-row slice.
// The last warp of a group to finish a stage refills it.
template <int TR>
__global__ void __launch_bounds__(NT, 1) k_tma2d(const __grid_constant__ CUtensorMap tmap, const float *V, int64_t ld,
                                                 int nc, int64_t n, const float *x, float *y, const float *coef,
                                                 float *part, int rev) {
    extern __shared__ __align__(128) float ring[];
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ unsigned cnt[kMaxStages];
    constexpr int WPT = TR / 32;            // warps per tile
    constexpr int NG = NW / WPT;            // tiles consumed concurrently
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = warp / WPT, sl = warp % WPT;
    const int64_t rpc = ((n + gridDim.x - 1) / gridDim.x + 63) / 64 * 64;
    const int64_t rb = blockIdx.x * rpc, re = rb + rpc < n ? rb + rpc : n;
    const int stage_f = (nc + 1) * TR;
    int S = kRing / (stage_f * 4);
    if (S > kMaxStages) S = kMaxStages;
    const int64_t ntile = (re > rb) ? (re - rb + TR - 1) / TR : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            cnt[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t t) {
        const int s = (int)(t % S);
        const int64_t tt = rev ? ntile - 1 - t : t;
        const int64_t r0 = rb + tt * TR;
        float *st = ring + (size_t)s * stage_f;
        mbar_arrive_expect_tx(&full[s], (uint32_t)(nc + 1) * TR * 4);
        tma_load_2d(st, &tmap, (int)r0, 0, &full[s]);
        bulk_g2s(st + nc * TR, x + r0, TR * 4, &full[s]);
    };
    if (threadIdx.x == 0)
        for (int64_t t = 0; t < S && t < ntile; ++t) issue(t);
    float acc[52];
#pragma unroll
    for (int c = 0; c < 52; ++c) acc[c] = 0.f;
    for (int64_t t = grp; t < ntile; t += NG) {
        const int s = (int)(t % S);
        mbar_wait(&full[s], (uint32_t)((t / S) & 1));
        const float *st = ring + (size_t)s * stage_f;
        const int64_t tt = rev ? ntile - 1 - t : t;
        const int lr = sl * 32 + lane;
        const int64_t r = rb + tt * TR + lr;
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < 52; ++c)
            if (c < nc) sum += st[c * TR + lr] * coef[c];
        const float yv = __fsub_rn(st[nc * TR + lr], sum);
        if (r < re) __stcg(y + r, yv);
#pragma unroll
        for (int c = 0; c < 52; ++c)
            if (c < nc) acc[c] += st[c * TR + lr] * yv;
        __syncwarp();
        if (lane == 0) {
            const unsigned old = atomicAdd(&cnt[s], 1u);
            if (old == WPT - 1) {
                cnt[s] = 0;
                if (t + S < ntile) issue(t + S);
            }
        }
    }
    __shared__ float sm[NW * 64];
#pragma unroll
    for (int c = 0; c < 52; ++c) {
        const float v = warp_sum(acc[c]);
        if (lane == 0 && c < nc) sm[warp * 64 + c] = v;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += NT) {
        float s = 0.f;
        for (int w = 0; w < NW; ++w) s += sm[w * 64 + c];
        part[(int64_t)c * gridDim.x + blockIdx.x] = s;
    }
}

#include <cudaTypedefs.h>
static CUtensorMap make_map(const float *V, int64_t ld, int nc, int TR) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)nc};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)TR, (cuuint32_t)nc};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(V), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

static int g_pfd = 0;
template <int U, int KU> void launch_reg(int sms, const float *V, int64_t ld, int nc, int64_t n, const float *x,
                                         float *y, const float *coef, float *part, int rev) {
    if (g_pfd == 0) k_reg<U, 0, KU, 0><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
    else if (g_pfd == 1) k_reg<U, 0, KU, 1><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
    else if (g_pfd == 2) k_reg<U, 0, KU, 2><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
    else k_reg<U, 0, KU, 4><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int64_t n : {2250000LL, 8000000LL}) {
        const int64_t ld = (n + 63) / 64 * 64;
        float *V, *x, *y, *coef, *part;
        cudaMalloc(&V, ld * 52 * 4);
        cudaMalloc(&x, ld * 4 + 4096);
        cudaMalloc(&y, ld * 4 + 4096);
        cudaMalloc(&coef, 64 * 4);
        cudaMalloc(&part, 64 * 4 * 320);
        cudaMemset(V, 0, ld * 52 * 4);
        cudaMemset(x, 0, ld * 4);
        cudaMemset(coef, 0, 64 * 4);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int nc : {8, 16, 26, 32, 40, 51}) {
            const int ncp = (nc + 3) / 4;
            auto cur = [&](int rev) {
                if (ncp * 8 <= 13) launch_reg<8, 1>(sms, V, ld, nc, n, x, y, coef, part, rev);
                else if (ncp * 4 <= 13) launch_reg<4, 3>(sms, V, ld, nc, n, x, y, coef, part, rev);
                else if (ncp * 2 <= 13) launch_reg<2, 6>(sms, V, ld, nc, n, x, y, coef, part, rev);
                else launch_reg<1, 13>(sms, V, ld, nc, n, x, y, coef, part, rev);
            };
            auto best = [&](int rev) {
                switch (ncp) {
                    case 1: launch_reg<12, 1>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 2: launch_reg<6, 2>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 3: launch_reg<4, 3>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 4: launch_reg<3, 4>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 5: launch_reg<3, 5>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 6: launch_reg<2, 6>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 7: launch_reg<2, 7>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 8: launch_reg<2, 8>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 9: launch_reg<2, 9>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 10: launch_reg<1, 10>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 11: launch_reg<1, 11>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 12: launch_reg<1, 12>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    default: launch_reg<1, 13>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                }
            };
            const double bytes = (double)n * 4 * (nc + 2);
            double gbs[4];
            for (int impl = 0; impl < 4; ++impl) {
                g_pfd = impl == 3 ? 4 : impl;
                auto run = [&](int i) { best(i & 1); };
                for (int i = 0; i < 3; ++i) run(i);
                cudaEventRecord(a);
                const int R = 20;
                for (int i = 0; i < R; ++i) run(i);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                gbs[impl] = bytes * R / ms / 1e6;
            }
            printf("n=%8lld nc=%2d pf0 %7.1f  pf1 %7.1f  pf2 %7.1f  pf4 %7.1f GB/s (%s)\n", (long long)n, nc, gbs[0],
                   gbs[1], gbs[2], gbs[3], cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(V); cudaFree(x); cudaFree(y); cudaFree(coef); cudaFree(part);
    }
    return 0;
}
