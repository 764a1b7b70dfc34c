// ys_spmv.cuh — device helpers shared by the single-GPU PCG (ys_solver.cu)
// and the row-partitioned multi-GPU PCG (ys_dist.cu): the 3x3 SpMV row
// accumulation, deterministic block reductions, 16-byte window loads.
#pragma once

#include "ys_device.cuh"

namespace ys {

namespace {
constexpr int kTB = 256;
}  // namespace

struct SpmvDev {
  const int32_t* rowptr;  // NB + 1
  const int32_t* ent;     // uid | transposed << 31, row-sorted
  const int32_t* oth;     // first DoF of the other block side per entry
  const int8_t* br;
  const int8_t* bc;
  const int64_t* voff;
  const double* values;   // reference layout (upper blocks, u sorted by (row, col))
  const int32_t* col;     // per uid
  const int32_t* nrow;    // 3x3 plan: NB + 1
  const int32_t* trow;    // 3x3 plan: NB + 1
  const int2* tlist;      // 3x3 plan: (u, row DoF) per transposed entry
};

static SpmvDev spmv_dev(Structure& st) {
  return SpmvDev{st.sp_rowptr.p, st.sp_ent.p, st.sp_oth.p, st.br.p, st.bc.p, st.voff.p, st.values.p,
                 st.col.p, st.nrow.p, st.trow.p, st.tlist.p};
}

// Block-level deterministic reduction of up to 3 doubles; result valid in thread 0.
template <int K>
__device__ __forceinline__ void block_reduce(double (&v)[K]) {
  __shared__ double sm[K][32];  // up to 1024 threads
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sm[k][w] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double a = 0.0;
      for (int q = 0; q < int(blockDim.x >> 5); ++q) a += sm[k][q];
      v[k] = a;
    }
  }
}

// Last-CTA election after every CTA stored its partials.
__device__ __forceinline__ bool last_cta(unsigned int* counter) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  return last;
}

// Sums `n` partials (stride `stride`, K of them) in a fixed order inside the last CTA.
template <int K>
__device__ __forceinline__ void sum_partials(const double* part, int n, int stride, double (&out)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = 0.0;
  for (int q = threadIdx.x; q < n; q += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] += ((volatile const double*)part)[k * stride + q];
  block_reduce<K>(out);
}

// --- SpMV row kernels -------------------------------------------------------

// Block row R of a 3x3 upper-storage structure: its own blocks (R, c) are the
// contiguous u range [nrow[R], nrow[R+1]) (y_R += B x_c); the blocks (r, R),
// r < R, come from tlist (y_R += B^T x_r) and are mostly L2 hits — row r
// streamed them moments earlier.
// 16-byte-aligned window loads: a 3x3 block (72 B at 8-byte alignment) is
// read as five 16 B loads of the enclosing 80 B window, a 3-vector (24 B) as
// two 16 B loads — fewer L1 wavefronts than nine / three 8 B loads.  The
// buffers carry 16 B of tail padding so the windows never leave the allocation.
__device__ __forceinline__ void load_block9(const double* __restrict__ p, double (&v)[9]) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const double2* w = reinterpret_cast<const double2*>(a & ~uintptr_t(15));
  const double2 w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2), w3 = __ldg(w + 3), w4 = __ldg(w + 4);
  if (a & 8) {
    v[0] = w0.y; v[1] = w1.x; v[2] = w1.y; v[3] = w2.x; v[4] = w2.y;
    v[5] = w3.x; v[6] = w3.y; v[7] = w4.x; v[8] = w4.y;
  } else {
    v[0] = w0.x; v[1] = w0.y; v[2] = w1.x; v[3] = w1.y; v[4] = w2.x;
    v[5] = w2.y; v[6] = w3.x; v[7] = w3.y; v[8] = w4.x;
  }
}

// L2-coherent variant (data written earlier in the same persistent kernel).
__device__ __forceinline__ void load_vec3_cg(const double* p, double& x0, double& x1, double& x2) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const double2* w = reinterpret_cast<const double2*>(a & ~uintptr_t(15));
  const double2 w0 = __ldcg(w), w1 = __ldcg(w + 1);
  if (a & 8) {
    x0 = w0.y; x1 = w1.x; x2 = w1.y;
  } else {
    x0 = w0.x; x1 = w0.y; x2 = w1.x;
  }
}

__device__ __forceinline__ void load_vec3(const double* __restrict__ p, double& x0, double& x1, double& x2) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const double2* w = reinterpret_cast<const double2*>(a & ~uintptr_t(15));
  const double2 w0 = w[0], w1 = w[1];
  if (a & 8) {
    x0 = w0.y; x1 = w1.x; x2 = w1.y;
  } else {
    x0 = w0.x; x1 = w0.y; x2 = w1.x;
  }
}

// Block row R of a 3x3 upper-storage structure: its own blocks (R, c) are the
// contiguous u range [nrow[R], nrow[R+1]) (y_R += B x_c, no index); the blocks
// (r, R), r < R, come from tlist (y_R += B^T x_r) and are mostly L2 hits — row
// r streamed them moments earlier.  The kernel is latency-bound on these
// dependent gathers, so it is shaped for rows in flight: 4 lanes per row,
// <= 64 registers (4 CTAs of 256 per SM), one resident wave.
struct RowPtrs {
  int32_t n0, n1, t0, t1;
};

__device__ __forceinline__ RowPtrs load_rowptrs(const SpmvDev& S, int64_t R) {
  return RowPtrs{S.nrow[R], S.nrow[R + 1], S.trow[R], S.trow[R + 1]};
}

template <int SW>
__device__ __forceinline__ void acc33(const SpmvDev& S, const RowPtrs& rp, int lane, const double* __restrict__ x,
                                      double& a0, double& a1, double& a2) {
  for (int32_t u = rp.n0 + lane; u < rp.n1; u += SW) {
    double v[9];
    load_block9(S.values + 9 * int64_t(u), v);
    double x0, x1, x2;
    load_vec3(x + S.col[u], x0, x1, x2);
    a0 += v[0] * x0 + v[1] * x1 + v[2] * x2;
    a1 += v[3] * x0 + v[4] * x1 + v[5] * x2;
    a2 += v[6] * x0 + v[7] * x1 + v[8] * x2;
  }
  for (int32_t j = rp.t0 + lane; j < rp.t1; j += SW) {
    const int2 t = S.tlist[j];
    double v[9];
    load_block9(S.values + 9 * int64_t(t.x), v);
    double x0, x1, x2;
    load_vec3(x + t.y, x0, x1, x2);
    a0 += v[0] * x0 + v[3] * x1 + v[6] * x2;
    a1 += v[1] * x0 + v[4] * x1 + v[7] * x2;
    a2 += v[2] * x0 + v[5] * x1 + v[8] * x2;
  }
}

constexpr int kSpmvSW = 4;

// The production row gather: two entries per lane per trip, both entries'
// index and data loads issued before any FMA (the second index is clamped so
// the loads stay unconditional) — twice the loads in flight per lane at
// <= 80 registers, 3 CTAs of 256 per SM (C5: 57.6 us vs 61.5 us one entry
// per trip at 4 CTAs).
template <int SW>
__device__ __forceinline__ void acc33_u2(const SpmvDev& S, const RowPtrs& rp, int lane, const double* __restrict__ x,
                                         double& a0, double& a1, double& a2) {
  for (int32_t u = rp.n0 + lane; u < rp.n1; u += 2 * SW) {
    const bool two = u + SW < rp.n1;
    const int32_t u2 = two ? u + SW : u;
    const int32_t c1 = S.col[u], c2 = S.col[u2];
    double v[9], w[9], x0, x1, x2, y0, y1, y2;
    load_block9(S.values + 9 * int64_t(u), v);
    load_block9(S.values + 9 * int64_t(u2), w);
    load_vec3(x + c1, x0, x1, x2);
    load_vec3(x + c2, y0, y1, y2);
    const double f = two ? 1.0 : 0.0;
    a0 += v[0] * x0 + v[1] * x1 + v[2] * x2;
    a1 += v[3] * x0 + v[4] * x1 + v[5] * x2;
    a2 += v[6] * x0 + v[7] * x1 + v[8] * x2;
    a0 += f * (w[0] * y0 + w[1] * y1 + w[2] * y2);
    a1 += f * (w[3] * y0 + w[4] * y1 + w[5] * y2);
    a2 += f * (w[6] * y0 + w[7] * y1 + w[8] * y2);
  }
  for (int32_t j = rp.t0 + lane; j < rp.t1; j += 2 * SW) {
    const bool two = j + SW < rp.t1;
    const int2 t = S.tlist[j];
    const int2 q = S.tlist[two ? j + SW : j];
    double v[9], w[9], x0, x1, x2, y0, y1, y2;
    load_block9(S.values + 9 * int64_t(t.x), v);
    load_block9(S.values + 9 * int64_t(q.x), w);
    load_vec3(x + t.y, x0, x1, x2);
    load_vec3(x + q.y, y0, y1, y2);
    const double f = two ? 1.0 : 0.0;
    a0 += v[0] * x0 + v[3] * x1 + v[6] * x2;
    a1 += v[1] * x0 + v[4] * x1 + v[7] * x2;
    a2 += v[2] * x0 + v[5] * x1 + v[8] * x2;
    a0 += f * (w[0] * y0 + w[3] * y1 + w[6] * y2);
    a1 += f * (w[1] * y0 + w[4] * y1 + w[7] * y2);
    a2 += f * (w[2] * y0 + w[5] * y1 + w[8] * y2);
  }
}

constexpr int kSpmvMinB = 3;  // CTAs per SM of the row-gather kernels

template <int N>
__device__ __forceinline__ void precond_apply(const double* __restrict__ M, const double* r, double* z) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) a += M[i * N + k] * r[k];
    z[i] = a;
  }
}


}  // namespace ys
