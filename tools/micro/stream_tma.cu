// Phase-B stream probe, round 2b: warp-specialised 2-D TMA pipeline.
//   warps 0..15  consumers: lane = row of a 256-row tile half (two 8-warp
//                groups take alternate tiles), every column of the row
//   warp 16      producer: one elected lane issues one cp.async.bulk.tensor
//                box (256 rows x nc columns, OOB columns not fetched) + one
//                bulk copy of x per tile into an S-stage ring, waiting on the
//                stage's "empty" mbarrier (8 consumer-warp arrivals)
// vs the register streams (k_reg, round-1/2 shapes).  y = x - V c ; acc = V^T y.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2105_07544_b200/csrc -o stream_tma stream_tma.cu -lcuda
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "common.cuh"
#include "tma.cuh"

using namespace mpk;

constexpr int NW = 16, NT = NW * 32;
constexpr int G = 8, P = 4, KP = 13;

template <int U, int KU>
__global__ void __launch_bounds__(NT, 1) k_reg(const float *V, int64_t ld, int nc, int64_t n, const float *x,
                                               float *y, const float *coef, float *part, int rev) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane % G, p = lane / G;
    const int64_t rpc = ((n + gridDim.x - 1) / gridDim.x + 63) / 64 * 64;
    const int64_t rb = blockIdx.x * rpc, re = rb + rpc < n ? rb + rpc : n;
    constexpr int64_t TRIP = 32 * U;
    float acc[KP];
#pragma unroll
    for (int i = 0; i < KP; ++i) acc[i] = 0.f;
    float cf[KU];
#pragma unroll
    for (int i = 0; i < KU; ++i) cf[i] = (p + P * i < nc) ? coef[p + P * i] : 0.f;
    const int64_t b0 = rb + (int64_t)warp * TRIP, step = (int64_t)NW * TRIP;
    const int64_t ntrip = (b0 < re) ? (re - b0 + step - 1) / step : 0;
    for (int64_t t = 0; t < ntrip; ++t) {
        const int64_t b = b0 + (rev ? ntrip - 1 - t : t) * step;
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

// ---------------- warp-specialised TMA: per-consumer-warp double buffers
// tile t (32*U rows x nc columns, one 2-D box + one bulk copy of x) goes to
// consumer warp t % 16, buffer (t / 16) & 1; lane = row (U rows per lane).
// The producer warp issues tiles in order, waiting on the target buffer's
// empty barrier (1 arrival: the consumer warp's lane 0).
constexpr int kTileB = 6656;            // bytes per buffer (2 per warp: 208 KB)
template <int U, int NCMAX>
__global__ void __launch_bounds__(NT + 32, 1) k_tma(const __grid_constant__ CUtensorMap tmap, int64_t ld, int nc,
                                                     int64_t n, const float *x, float *y, const float *coef,
                                                     float *part, int rev) {
    extern __shared__ __align__(128) float ring[];
    __shared__ __align__(8) uint64_t full[NW][2], empty[NW][2];
    constexpr int TRW = 32 * U;                      // rows per tile
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t rpc = ((n + gridDim.x - 1) / gridDim.x + 63) / 64 * 64;
    const int64_t rb = blockIdx.x * rpc, re = rb + rpc < n ? rb + rpc : n;
    const int buf_f = kTileB / 4;                    // floats per buffer
    const int64_t ntile = (re > rb) ? (re - rb + TRW - 1) / TRW : 0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < NW; ++w)
            for (int s = 0; s < 2; ++s) {
                mbar_init(&full[w][s], 1);
                mbar_init(&empty[w][s], 1);
            }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NW) {   // producer
        if (lane == 0) {
            for (int64_t t = 0; t < ntile; ++t) {
                const int w = (int)(t % NW), s = (int)((t / NW) & 1);
                const int64_t j = t / NW;                // this warp's tile index
                if (j >= 2) mbar_wait(&empty[w][s], (uint32_t)(((j - 2) / 2) & 1));
                const int64_t tt = rev ? ntile - 1 - t : t;
                const int64_t r0 = rb + tt * TRW;
                float *st = ring + (size_t)(w * 2 + s) * buf_f;
                mbar_arrive_expect_tx(&full[w][s], (uint32_t)(nc + 1) * TRW * 4);
                tma_load_2d(st, &tmap, (int)r0, 0, &full[w][s]);
                bulk_g2s(st + nc * TRW, x + r0, TRW * 4, &full[w][s]);
            }
        }
        return;
    }
    float acc[NCMAX];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) acc[c] = 0.f;
    int64_t j = 0;
    for (int64_t t = warp; t < ntile; t += NW, ++j) {
        const int s = (int)(j & 1);
        mbar_wait(&full[warp][s], (uint32_t)((j >> 1) & 1));
        const float *st = ring + (size_t)(warp * 2 + s) * buf_f;
        const int64_t tt = rev ? ntile - 1 - t : t;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int lr = u * 32 + lane;
            const int64_t r = rb + tt * TRW + lr;
            float sum = 0.f;
#pragma unroll
            for (int c = 0; c < NCMAX; ++c)
                if (c < nc) sum += st[c * TRW + lr] * coef[c];
            const float yv = __fsub_rn(st[nc * TRW + lr], sum);
            if (r < re) __stcg(y + r, yv);
#pragma unroll
            for (int c = 0; c < NCMAX; ++c)
                if (c < nc) acc[c] += st[c * TRW + lr] * yv;
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[warp][s])) : "memory");
    }
    __shared__ float sm[NW * 64];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
        const float v = warp_sum(acc[c]);
        if (lane == 0 && c < nc) sm[warp * 64 + c] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NT));   // consumers only
    for (int c = threadIdx.x; c < nc; c += NT) {
        float sacc = 0.f;
        for (int w = 0; w < NW; ++w) sacc += sm[w * 64 + c];
        part[(int64_t)c * gridDim.x + blockIdx.x] = sacc;
    }
}

static CUtensorMap make_map(const float *V, int64_t ld, int nc, int TRW) {
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
    cuuint32_t box[2] = {(cuuint32_t)TRW, (cuuint32_t)nc};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(V), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

template <int U, int KU> void launch_reg(int sms, const float *V, int64_t ld, int nc, int64_t n, const float *x,
                                         float *y, const float *coef, float *part, int rev) {
    k_reg<U, KU><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int kRing = NW * 2 * kTileB;
    cudaFuncSetAttribute(k_tma<8, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing);
    cudaFuncSetAttribute(k_tma<4, 13>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing);
    cudaFuncSetAttribute(k_tma<2, 27>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing);
    cudaFuncSetAttribute(k_tma<1, 52>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing);
    for (int64_t n : {2250000LL, 8000000LL}) {
        const int64_t ld = (n + 255) / 256 * 256;   // tiles of <= 256 rows stay inside ld
        float *V, *x, *y, *coef, *part;
        cudaMalloc(&V, ld * 52 * 4);
        cudaMalloc(&x, ld * 4 + 8192);
        cudaMalloc(&y, ld * 4 + 8192);
        cudaMalloc(&coef, 64 * 4);
        cudaMalloc(&part, 64 * 4 * 320);
        cudaMemset(V, 0, ld * 52 * 4);
        cudaMemset(x, 0, ld * 4 + 8192);
        cudaMemset(coef, 0, 64 * 4);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int nc : {4, 8, 13, 16, 20, 26, 32, 40, 51}) {
            const int ncp = (nc + 3) / 4;
            // rows per tile: the largest 32*U with (nc + 1) * 32U * 4 <= 6.5 KB
            const int U = (nc + 1) * 32 * 8 * 4 <= kTileB ? 8 : (nc + 1) * 32 * 4 * 4 <= kTileB ? 4
                        : (nc + 1) * 32 * 2 * 4 <= kTileB ? 2 : 1;
            const CUtensorMap tm = make_map(V, ld, nc, 32 * U);
            auto reg = [&](int rev) {
                switch (ncp) {
                    case 1: launch_reg<8, 1>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 2: case 3: launch_reg<4, 3>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 4: launch_reg<3, 4>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 5: case 6: launch_reg<2, 6>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 7: launch_reg<2, 7>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 8: launch_reg<2, 8>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    case 9: launch_reg<2, 9>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                    default: launch_reg<1, 13>(sms, V, ld, nc, n, x, y, coef, part, rev); break;
                }
            };
            auto tma = [&](int rev) {
                if (U == 8) k_tma<8, 6><<<sms, NT + 32, kRing>>>(tm, ld, nc, n, x, y, coef, part, rev);
                else if (U == 4) k_tma<4, 13><<<sms, NT + 32, kRing>>>(tm, ld, nc, n, x, y, coef, part, rev);
                else if (U == 2) k_tma<2, 27><<<sms, NT + 32, kRing>>>(tm, ld, nc, n, x, y, coef, part, rev);
                else k_tma<1, 52><<<sms, NT + 32, kRing>>>(tm, ld, nc, n, x, y, coef, part, rev);
            };
            const double bytes = (double)n * 4 * (nc + 2);
            double gbs[2];
            for (int impl = 0; impl < 2; ++impl) {
                auto run = [&](int i) { impl ? tma(i & 1) : reg(i & 1); };
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
            printf("n=%8lld nc=%2d reg %7.1f GB/s  tma-ws %7.1f GB/s  (%s)\n", (long long)n, nc, gbs[0], gbs[1],
                   cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(V); cudaFree(x); cudaFree(y); cudaFree(coef); cudaFree(part);
    }
    return 0;
}
