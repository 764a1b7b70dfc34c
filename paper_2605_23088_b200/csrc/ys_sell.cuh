// ys_sell.cuh — the PCG's streaming copy of H for uniform 3x3 systems.
//
// The reference multiplies from upper storage (spmv_add, solver.cpp:10-82):
// every off-diagonal block (r, c) contributes B x_c to row r and B^T x_r to
// row c.  Gathering both products per row from upper storage reads every
// off-diagonal block twice through L1 and the transposed half through a
// dependent index (tlist -> block), which bounds the row gather at ~0.37 of
// HBM peak (profiles/r01_spmv_breakdown_c5.md).
//
// Here H = H_static + H_dynamic is repacked ONCE per Newton iteration (its
// values change every iteration, the PCG then runs hundreds of SpMVs) into a
// full (both-triangle) sliced-ELL layout:
//   * rows are placed at positions q (row perm[q]): inside each window of
//     kSellSigma positions they are sorted by entry count (descending, stable),
//     so the long contact rows share slices instead of widening many
//     (C5: mean slice width 5.1 -> ~4.4 entry rows);
//   * a slice is 32 lanes = 32/H positions, H lanes per row; entry k of the
//     row at position q goes to lane (q mod 32/H)*H + k mod H, entry row k / H;
//   * an entry row of a slice is 32 int32 column DoFs and 32 x 72 B of values
//     as [4][32] double2 + [32] double, so every load instruction of a warp is
//     one contiguous 512 B (or 256 B) run: fully coalesced, no index chains;
//   * transposed blocks are stored transposed: all entries are y += B x.
// Entries of a row: static own blocks (the dynamic group's diagonal block is
// added into the static diagonal block: one entry, B_s + B_d), static
// transposed, dynamic own, dynamic transposed (the reference's
// static-then-dynamic order, summed per lane then by a fixed xor butterfly:
// deterministic, bitwise reproducible).
// Padding slots (k >= the lane's count) are never read.
#pragma once

#include "ys_spmv.cuh"

namespace ys {

struct SellDev {
  const int32_t* len;   // NB: entries of each block row
  const int64_t* soff;  // nslices + 1: first entry row of each slice
  const int32_t* col;   // entry rows x 32: column DoF
  const double* val;    // entry rows x 288
  int64_t nb;       // end of the row range (exclusive)
  int64_t nslices;
  int64_t r0;       // first row of the range (0; the owned rows' start in the distributed solve)
  const int32_t* perm;  // position q -> block row: rows sorted by entry count inside windows of
                        // kSellSigma positions (long contact rows share slices); len is by position
};

// 63 slices of 8 rows: nearly coprime with the warp counts of the grid-stride
// slice loops (multiples of 32), so the window position of a warp's slices
// rotates and the long slices spread over the warps (a 256-row window sent
// every window's longest slice to the same warps: phase A 43 -> 80 us).
// C5 phase A by window: 120 rows 43.2, 248 40.9, 504 40.0, 760 41.5, 1016 45.3 us.
constexpr int kSellSigma = 504;

// Block row at position q of the copy (q < nb - r0).
__device__ __forceinline__ int64_t sell_row(const SellDev& S, int64_t q) { return S.perm[q]; }

SellDev sell_dev(Context& c);  // ys_sell.cu

// Accumulates lane `lane`'s share of its row (lanes of a row: H consecutive).
template <int H>
__device__ __forceinline__ void sell_acc(const SellDev& S, int64_t slice, int lane, const double* x, double& a0,
                                         double& a1, double& a2, int64_t& R) {
  constexpr int RPS = 32 / H;
  const int64_t q = slice * RPS + lane / H;
  const bool live = q < S.nb - S.r0;
  R = live ? sell_row(S, q) : S.nb;
  const int h = lane % H;
  const int L = live ? S.len[q] : 0;
  const int Lh = L > h ? (L - h + H - 1) / H : 0;
  const int64_t e0 = S.soff[slice];
  for (int k = 0; k < Lh; k += 2) {
    const bool two = k + 1 < Lh;
    const int64_t e1 = e0 + k, e2 = e0 + (two ? k + 1 : k);
    const int32_t c1 = __ldcs(S.col + e1 * 32 + lane), c2 = __ldcs(S.col + e2 * 32 + lane);
    const double2* v1 = reinterpret_cast<const double2*>(S.val + e1 * 288) + lane;
    const double2* v2 = reinterpret_cast<const double2*>(S.val + e2 * 288) + lane;
    const double2 p0 = __ldcs(v1), p1 = __ldcs(v1 + 32), p2 = __ldcs(v1 + 64), p3 = __ldcs(v1 + 96);
    const double p4 = __ldcs(S.val + e1 * 288 + 256 + lane);
    const double2 q0 = __ldcs(v2), q1 = __ldcs(v2 + 32), q2 = __ldcs(v2 + 64), q3 = __ldcs(v2 + 96);
    const double q4 = __ldcs(S.val + e2 * 288 + 256 + lane);
    double x0, x1, x2, y0, y1, y2;
    load_vec3(x + c1, x0, x1, x2);
    load_vec3(x + c2, y0, y1, y2);
    a0 += p0.x * x0 + p0.y * x1 + p1.x * x2;
    a1 += p1.y * x0 + p2.x * x1 + p2.y * x2;
    a2 += p3.x * x0 + p3.y * x1 + p4 * x2;
    const double f = two ? 1.0 : 0.0;
    a0 += f * (q0.x * y0 + q0.y * y1 + q1.x * y2);
    a1 += f * (q1.y * y0 + q2.x * y1 + q2.y * y2);
    a2 += f * (q3.x * y0 + q3.y * y1 + q4 * y2);
  }
  if (H > 1) {
    const unsigned mask = 0xffffffffu;
#pragma unroll
    for (int off = H / 2; off > 0; off >>= 1) {
      a0 += __shfl_xor_sync(mask, a0, off, H);
      a1 += __shfl_xor_sync(mask, a1, off, H);
      a2 += __shfl_xor_sync(mask, a2, off, H);
    }
  }
}

// PCG vectors kept in L2 across the solve's phases: loads / stores carrying an
// L2::evict_last policy (the matrix copy streams with evict-first loads).
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_keep2(const double2* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void load_vec3_keep(const double* p, double& x0, double& x1, double& x2, uint64_t pol) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const double2* w = reinterpret_cast<const double2*>(a & ~uintptr_t(15));
  const double2 w0 = ld_keep2(w, pol), w1 = ld_keep2(w + 1, pol);
  if (a & 8) {
    x0 = w0.y; x1 = w1.x; x2 = w1.y;
  } else {
    x0 = w0.x; x1 = w0.y; x2 = w1.x;
  }
}

__device__ __forceinline__ void load_block9_keep(const double* p, double (&v)[9], uint64_t pol) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const double2* w = reinterpret_cast<const double2*>(a & ~uintptr_t(15));
  const double2 w0 = ld_keep2(w, pol), w1 = ld_keep2(w + 1, pol), w2 = ld_keep2(w + 2, pol),
                w3 = ld_keep2(w + 3, pol), w4 = ld_keep2(w + 4, pol);
  if (a & 8) {
    v[0] = w0.y; v[1] = w1.x; v[2] = w1.y; v[3] = w2.x; v[4] = w2.y;
    v[5] = w3.x; v[6] = w3.y; v[7] = w4.x; v[8] = w4.y;
  } else {
    v[0] = w0.x; v[1] = w0.y; v[2] = w1.x; v[3] = w1.y; v[4] = w2.x;
    v[5] = w2.y; v[6] = w3.x; v[7] = w3.y; v[8] = w4.x;
  }
}

// Same accumulation with the lane's column DoFs already in shared memory
// (cols[j * 32 + lane], j < Lh) and its first entry row e0: the x gathers and
// the value loads issue together.
template <int H>
__device__ __forceinline__ void sell_acc_cached(const SellDev& S, int64_t e0, const int32_t* cols, int Lh, int lane,
                                                const double* x, double& a0, double& a1, double& a2, uint64_t pol) {
  for (int k = 0; k < Lh; k += 2) {
    const bool two = k + 1 < Lh;
    const int k2 = two ? k + 1 : k;
    const int64_t e1 = e0 + k, e2 = e0 + k2;
    const int32_t c1 = cols[k * 32 + lane], c2 = cols[k2 * 32 + lane];
    double x0, x1, x2, y0, y1, y2;
    load_vec3_keep(x + c1, x0, x1, x2, pol);
    load_vec3_keep(x + c2, y0, y1, y2, pol);
    const double2* v1 = reinterpret_cast<const double2*>(S.val + e1 * 288) + lane;
    const double2* v2 = reinterpret_cast<const double2*>(S.val + e2 * 288) + lane;
    const double2 p0 = __ldcs(v1), p1 = __ldcs(v1 + 32), p2 = __ldcs(v1 + 64), p3 = __ldcs(v1 + 96);
    const double p4 = __ldcs(S.val + e1 * 288 + 256 + lane);
    const double2 q0 = __ldcs(v2), q1 = __ldcs(v2 + 32), q2 = __ldcs(v2 + 64), q3 = __ldcs(v2 + 96);
    const double q4 = __ldcs(S.val + e2 * 288 + 256 + lane);
    a0 += p0.x * x0 + p0.y * x1 + p1.x * x2;
    a1 += p1.y * x0 + p2.x * x1 + p2.y * x2;
    a2 += p3.x * x0 + p3.y * x1 + p4 * x2;
    const double f = two ? 1.0 : 0.0;
    a0 += f * (q0.x * y0 + q0.y * y1 + q1.x * y2);
    a1 += f * (q1.y * y0 + q2.x * y1 + q2.y * y2);
    a2 += f * (q3.x * y0 + q3.y * y1 + q4 * y2);
  }
  if (H > 1) {
#pragma unroll
    for (int off = H / 2; off > 0; off >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, off, H);
      a1 += __shfl_xor_sync(0xffffffffu, a1, off, H);
      a2 += __shfl_xor_sync(0xffffffffu, a2, off, H);
    }
  }
}

}  // namespace ys
