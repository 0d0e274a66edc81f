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
#include "tma.cuh"

using namespace mpk;

constexpr int NT = 512, NW = 16;
constexpr int G = 8, P = 4, KP = 13;   // 8 rows x 4 column parts per warp; 13 columns per part

// ---------------- register streaming (as k_cycle_reg), U row groups of 4 rows
template <int U>
__global__ void __launch_bounds__(NT, 1) k_reg(const float *V, int64_t ld, int nc, int64_t n, const float *x,
                                               float *y, const float *coef, float *part, int rev) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane % G, p = lane / G;
    const int64_t rpc = ((n + gridDim.x - 1) / gridDim.x + 63) / 64 * 64;
    const int64_t rb = blockIdx.x * rpc, re = rb + rpc < n ? rb + rpc : n;
    constexpr int KU = KP / U;
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
        std::vector<float> h(ld);
        for (int64_t i = 0; i < ld; ++i) h[i] = (float)((i * 2654435761u) % 1000) * 1e-3f;
        for (int c = 0; c < 52; ++c) cudaMemcpy(V + c * ld, h.data(), ld * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(x, h.data(), ld * 4, cudaMemcpyHostToDevice);
        std::vector<float> hc(64, 0.01f);
        cudaMemcpy(coef, hc.data(), 64 * 4, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing);
        cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing);
        cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRing);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        std::vector<float> pr(64 * sms), pt(64 * sms);
        for (int nc : {4, 12, 26, 40, 51}) {
            auto reg = [&](int rev) {
                if (nc * 4 <= 13 * 4 && (nc + 3) / 4 * 4 <= 13) k_reg<4><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
                else if ((nc + 3) / 4 * 2 <= 13) k_reg<2><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
                else k_reg<1><<<sms, NT>>>(V, ld, nc, n, x, y, coef, part, rev);
            };
            auto tma = [&](int rev) {
                if (nc <= 12) k_tma<4><<<sms, NT, kRing>>>(V, ld, nc, n, x, y, coef, part, rev);
                else if (nc <= 26) k_tma<2><<<sms, NT, kRing>>>(V, ld, nc, n, x, y, coef, part, rev);
                else k_tma<1><<<sms, NT, kRing>>>(V, ld, nc, n, x, y, coef, part, rev);
            };
            const double bytes = (double)n * 4 * (nc + 2);
            for (int impl = 0; impl < 2; ++impl) {
                for (int serp = 0; serp < 2; ++serp) {
                    auto run = [&](int i) { impl ? tma(serp ? (i & 1) : 0) : reg(serp ? (i & 1) : 0); };
                    for (int i = 0; i < 3; ++i) run(i);
                    cudaEventRecord(a);
                    const int R = 20;
                    for (int i = 0; i < R; ++i) run(i);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    printf("n=%8lld nc=%2d %s serp=%d : %7.2f us  %7.1f GB/s  (%s)\n", (long long)n, nc,
                           impl ? "tma" : "reg", serp, ms * 1e3 / R, bytes * R / ms / 1e6,
                           cudaGetErrorString(cudaGetLastError()));
                }
                cudaMemcpy(impl ? pt.data() : pr.data(), part, 64 * 4 * sms, cudaMemcpyDeviceToHost);
            }
            double md = 0;
            for (int c = 0; c < nc; ++c) {
                double sa = 0, sb = 0;
                for (int k = 0; k < sms; ++k) sa += pr[c * sms + k], sb += pt[c * sms + k];
                md = fmax(md, fabs(sa - sb) / (fabs(sa) + 1e-30));
            }
            printf("   dots reg vs tma max rel diff %.3e\n", md);
        }
        cudaFree(V); cudaFree(x); cudaFree(y); cudaFree(coef); cudaFree(part);
    }
    return 0;
}
