// Per-restart collectives of the row-partitioned solve, on the device.
//
// Between two cycles a rank needs (gmres.py:290-291, multiprecision.py:216-217)
//   * the halo rows of x for its explicit residual r = b - A x, and
//   * the global sums of r.r, r_low.r_low, b.b and the "x moved" flag.
// Both go through the same peer memory the cycle kernel uses (CUDA-IPC
// mapped pointers, NVLink P2P stores) and the same monotonic system-scope
// arrival counter / epoch pair, so there is no host pickling, no NCCL call
// and no host round trip beyond the one control-block read per restart:
//   k_comm_push    own x rows -> own global-length buffer xg, mirror rows ->
//                  the neighbours' xg; last CTA: cross-rank barrier
//   k_comm_reduce  32-byte scalar slot -> every rank's slot table; barrier;
//                  sum the table in rank order (each value in its own type)
#pragma once

#include "fused.cuh"

namespace mpk {

constexpr int kCommScalBytes = 32;   // r.r | r_low.r_low (f32) | moved (i32) | timeout (i32) | b.b

struct CommView {
    int rank, nranks;
    int64_t row0;
    char *xg[kMaxRanks];
    unsigned long long *xbar[kMaxRanks];   // [0] arrivals (u64); +8 u32 last-CTA count; +12 u32 timeout
    unsigned long long *epoch;
    int64_t mir_lo[kMaxRanks], mir_hi[kMaxRanks];
    char *scal[kMaxRanks];                 // kMaxRanks x kCommScalBytes slot table per rank
};

// One cross-rank barrier step (the same epoch arithmetic as grid_sync_x):
// arrive on every rank's counter, wait for nranks * epoch arrivals on our own.
__device__ __forceinline__ void comm_barrier_x(const CommView &c) {
    const unsigned long long ep = *(volatile unsigned long long *)c.epoch + 1ull;
    __threadfence_system();
    for (int q = 0; q < c.nranks; ++q) atomicAdd_system(c.xbar[q], 1ull);
    volatile unsigned long long *mine = c.xbar[c.rank];
    const unsigned long long need = (unsigned long long)c.nranks * ep;
    const unsigned long long t0 = globaltimer_ns();
    while (*mine < need) {
        __nanosleep(64);
        if (globaltimer_ns() - t0 > 20000000000ull) {   // a peer is gone: flag, do not hang the GPU
            atomicExch(reinterpret_cast<unsigned *>(c.xbar[c.rank]) + 3, 1u);
            break;
        }
    }
    *c.epoch = ep;
    __threadfence_system();
}

template <typename T>
__global__ void __launch_bounds__(256) k_comm_push(CommView c, int64_t n, const T *x) {
    T *own = reinterpret_cast<T *>(c.xg[c.rank]) + c.row0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const T v = x[r];
        own[r] = v;
        for (int q = 0; q < c.nranks; ++q)
            if (q != c.rank && r >= c.mir_lo[q] && r < c.mir_hi[q])
                reinterpret_cast<T *>(c.xg[q])[c.row0 + r] = v;
    }
    // last CTA out: every CTA's stores are fenced before it arrives
    __threadfence_system();
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
        unsigned *cnt = reinterpret_cast<unsigned *>(c.xbar[c.rank]) + 2;
        last = atomicAdd(cnt, 1u) == gridDim.x - 1;
        if (last) {
            *cnt = 0u;
            comm_barrier_x(c);
        }
    }
}

// peers wrote these rows with P2P stores before arriving: read them uncached
template <typename T> __device__ __forceinline__ T slot_val(const char *p) {
    return *reinterpret_cast<const volatile T *>(p);
}

__global__ void k_comm_reduce(CommView c, char *slot, int rn2_f64, int bn2_f64) {
    if (threadIdx.x != 0) return;
    // publish this rank's 32 bytes into every rank's table row `rank`
    const uint4 *src = reinterpret_cast<const uint4 *>(slot);
    const uint4 a0 = src[0], a1 = src[1];
    for (int q = 0; q < c.nranks; ++q) {
        uint4 *dst = reinterpret_cast<uint4 *>(c.scal[q] + (int64_t)c.rank * kCommScalBytes);
        dst[0] = a0;
        dst[1] = a1;
    }
    comm_barrier_x(c);
    double rn2d = 0.0, bn2d = 0.0;
    float rn2f = 0.f, bn2f = 0.f, lowf = 0.f;
    int moved = 0;
    for (int q = 0; q < c.nranks; ++q) {   // rank order, each value in its own type
        const char *row = c.scal[c.rank] + (int64_t)q * kCommScalBytes;
        if (rn2_f64) rn2d = __dadd_rn(rn2d, slot_val<double>(row));
        else rn2f = __fadd_rn(rn2f, slot_val<float>(row));
        lowf = __fadd_rn(lowf, slot_val<float>(row + 8));
        moved |= slot_val<int>(row + 16);
        if (bn2_f64) bn2d = __dadd_rn(bn2d, slot_val<double>(row + 24));
        else bn2f = __fadd_rn(bn2f, slot_val<float>(row + 24));
    }
    if (rn2_f64) *reinterpret_cast<double *>(slot) = rn2d;
    else *reinterpret_cast<float *>(slot) = rn2f;
    *reinterpret_cast<float *>(slot + 8) = lowf;
    *reinterpret_cast<int *>(slot + 16) = moved;
    // barrier timeouts of this kernel or an earlier k_comm_push
    *reinterpret_cast<int *>(slot + 20) = (int)*(volatile unsigned *)(reinterpret_cast<unsigned *>(c.xbar[c.rank]) + 3);
    if (bn2_f64) *reinterpret_cast<double *>(slot + 24) = bn2d;
    else *reinterpret_cast<float *>(slot + 24) = bn2f;
}

}  // namespace mpk
