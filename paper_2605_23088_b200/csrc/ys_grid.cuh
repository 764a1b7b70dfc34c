// ys_grid.cuh — grid-wide synchronisation of the persistent cooperative PCG
// kernels (ys_solver.cu): counter barriers, fixed-order reductions
// of the per-CTA partials (every CTA sums them in the same order, so alpha /
// beta / status are bit-identical everywhere without a last-CTA round trip),
// and the %globaltimer phase clock.
#pragma once

#include "ys_spmv.cuh"

namespace ys {

struct GridBar {
  unsigned int count;  // generation barrier
  unsigned int gen;
  unsigned long long arrivals;  // counter barrier: only grows within a launch
};

__device__ __forceinline__ void grid_sync(GridBar* gb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = &gb->gen;
    const unsigned int g = *vgen;
    __threadfence();
    if (atomicAdd(&gb->count, 1u) == gridDim.x - 1) {
      gb->count = 0;
      __threadfence();
      atomicAdd(&gb->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// Counter barrier: one red.release (no return value) per CTA on a counter
// that only grows, then acquire-polling until it reaches G * epoch.  The
// release orders this CTA's writes before its arrival; the acquire load orders
// the poller's later reads after every arrival (and invalidates L1).  No
// returning atomic is serialised at one address and no generation word is
// needed; the counter is zeroed before each launch.
__device__ __forceinline__ void grid_sync_counter(unsigned long long* count, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(count) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// The counter barrier split in two: arrive (every thread's prior writes
// ordered before the CTA's release-add) and wait (acquire poll), so a CTA can
// issue loads that do not depend on other CTAs' writes in between.
__device__ __forceinline__ void grid_arrive(unsigned long long* count) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
}

__device__ __forceinline__ void grid_wait(unsigned long long* count, unsigned long long target) {
  if (threadIdx.x == 0) {
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(count) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// Fixed-order sum of n partials (stride between the K arrays = n) inside every CTA.
template <int K>
__device__ __forceinline__ void reduce_partials_all(const double* part, int n, double (&out)[K]) {
  __shared__ double res[K];
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = 0.0;
  for (int q = threadIdx.x; q < n; q += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] += __ldcg(part + k * n + q);
  block_reduce<K>(out);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) res[k] = out[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = res[k];
  __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace ys
