// Read-throughput probe: is the basis stream bound by HBM or by L2 (LTS)
// request throughput?  Streams a buffer of S bytes R times with 16-byte
// ld.global.cg loads (U loads in flight per thread) and with 1-D bulk copies
// (cp.async.bulk, TMA engine) into a shared-memory ring, and prints GB/s.
// Buffers <= ~100 MB stay L2-resident across repeats; 4 GB comes from HBM.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o l2bw l2bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

__device__ float g_sink;

template <int U>
__global__ void __launch_bounds__(512) k_ldg(const float4 *p, int64_t n16, int reps) {
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride * U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j = i + u * stride;
                if (j < n16) {
                    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                                 : "l"(p + j));
                } else {
                    v[u] = make_float4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    }
    if (acc == 123.456f) g_sink = acc;
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one producer thread issues bulk copies of CH bytes into an NS-stage ring;
// the other warps consume (sum) each stage and release it
template <int CH, int NS>
__global__ void __launch_bounds__(256) k_bulk(const char *p, int64_t bytes, int reps) {
    extern __shared__ __align__(128) char ring[];
    __shared__ __align__(8) uint64_t full[NS], empty[NS];
    const int tid = threadIdx.x, nw = blockDim.x / 32 - 1;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(nw));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t nch = bytes / CH;
    const int64_t total = nch * reps;
    float acc = 0.f;
    if (tid / 32 == nw) {   // producer warp
        if (tid % 32 == 0) {
            int64_t it = 0;
            for (int64_t c = blockIdx.x; c < total; c += gridDim.x, ++it) {
                const int s = it % NS;
                const uint32_t ph = (it / NS) & 1;
                if (it >= NS) {
                    uint32_t ok = 0;
                    while (!ok)
                        asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}"
                                     : "=r"(ok) : "r"(su32(&empty[s])), "r"(ph ^ 1) : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(CH)
                             : "memory");
                const char *src = p + (c % nch) * CH;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        su32(ring + s * CH)),
                    "l"(src), "r"(CH), "r"(su32(&full[s]))
                    : "memory");
            }
        }
    } else {
        int64_t it = 0;
        for (int64_t c = blockIdx.x; c < total; c += gridDim.x, ++it) {
            const int s = it % NS;
            const uint32_t ph = (it / NS) & 1;
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}"
                             : "=r"(ok) : "r"(su32(&full[s])), "r"(ph) : "memory");
            const float4 *q = reinterpret_cast<const float4 *>(ring + s * CH);
            for (int i = tid; i < CH / 16; i += nw * 32) {
                float4 v = q[i];
                acc += v.x + v.y + v.z + v.w;
            }
            __syncwarp();
            if (tid % 32 == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
    }
    if (acc == 123.456f) g_sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t big = 4LL << 30;
    char *buf;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 0, big);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int64_t sizes[] = {16LL << 20, 48LL << 20, 96LL << 20, 256LL << 20, 4LL << 30};
    for (int64_t S : sizes) {
        const int reps = (int)((8LL << 30) / S) < 1 ? 1 : (int)((8LL << 30) / S);
        for (int bps : {1, 2, 4}) {
            for (int U : {4, 8, 16}) {
                auto run = [&]() {
                    if (U == 4) k_ldg<4><<<sms * bps, 512>>>((const float4 *)buf, S / 16, reps);
                    if (U == 8) k_ldg<8><<<sms * bps, 512>>>((const float4 *)buf, S / 16, reps);
                    if (U == 16) k_ldg<16><<<sms * bps, 512>>>((const float4 *)buf, S / 16, reps);
                };
                run();
                cudaEventRecord(a);
                run();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("ldg   S=%6lld MB ctas/sm=%d U=%2d : %8.1f GB/s\n", (long long)(S >> 20), bps, U,
                       (double)S * reps / ms / 1e6);
            }
        }
        // bulk ring: 16 KB chunks x 8 stages (128 KB) and 32 KB x 6, 1 or 2 CTAs/SM
        {
            constexpr int CH = 16384, NS = 8;
            cudaFuncSetAttribute(k_bulk<CH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * NS);
            for (int bps : {1}) {
                auto run = [&]() { k_bulk<CH, NS><<<sms * bps, 256, CH * NS>>>(buf, S, reps); };
                run();
                cudaEventRecord(a);
                run();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("bulk  S=%6lld MB 16KBx8 ctas/sm=%d : %8.1f GB/s  (%s)\n", (long long)(S >> 20), bps,
                       (double)S * reps / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
        {
            constexpr int CH = 32768, NS = 6;
            cudaFuncSetAttribute(k_bulk<CH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * NS);
            auto run = [&]() { k_bulk<CH, NS><<<sms, 256, CH * NS>>>(buf, S, reps); };
            run();
            cudaEventRecord(a);
            run();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("bulk  S=%6lld MB 32KBx6 ctas/sm=1 : %8.1f GB/s  (%s)\n", (long long)(S >> 20),
                   (double)S * reps / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
