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
//   * a slice is 32 lanes = 32/H block rows, H lanes per row; entry k of row R
//     goes to lane (R mod 32/H)*H + k mod H, entry row k / H of the slice;
//   * an entry row of a slice is 32 int32 column DoFs and 32 x 72 B of values
//     as [4][32] double2 + [32] double, so every load instruction of a warp is
//     one contiguous 512 B (or 256 B) run: fully coalesced, no index chains;
//   * transposed blocks are stored transposed: all entries are y += B x.
// Entries of a row: static own blocks, static transposed, dynamic own,
// dynamic transposed (the reference's static-then-dynamic order, summed per
// lane then by a fixed xor butterfly: deterministic, bitwise reproducible).
// Padding slots (k >= the lane's count) are never read.
#pragma once

#include "ys_spmv.cuh"

namespace ys {

struct SellDev {
  const int32_t* len;   // NB: entries of each block row
  const int64_t* soff;  // nslices + 1: first entry row of each slice
  const int32_t* col;   // entry rows x 32: column DoF
  const double* val;    // entry rows x 288
  int64_t nb;
  int64_t nslices;
  // symmetric (upper-only) mode, null in full mode:
  const int32_t* tpos;    // entry rows x 32: transposed-product slot of an off-diagonal entry, -1 on the diagonal
  const int32_t* tstart;  // NB + 1: first slot of each block row's transposed products
  double* slots;          // 3 doubles per slot
};

SellDev sell_dev(Context& c);  // ys_sell.cu

// Accumulates lane `lane`'s share of its row (lanes of a row: H consecutive).
template <class T>
__device__ __forceinline__ T sell_ld(const T* p, bool stream) {
  return stream ? __ldcs(p) : __ldg(p);
}

// ST: streaming (evict-first) loads of the matrix copy; false: default policy
// (lets an L2 persisting window keep part of it resident).
template <int H, bool ST = true>
__device__ __forceinline__ void sell_acc(const SellDev& S, int64_t slice, int lane, const double* x, double& a0,
                                         double& a1, double& a2, int64_t& R) {
  constexpr int RPS = 32 / H;
  R = slice * RPS + lane / H;
  const int h = lane % H;
  const int L = R < S.nb ? S.len[R] : 0;
  const int Lh = L > h ? (L - h + H - 1) / H : 0;
  const int64_t e0 = S.soff[slice];
  for (int k = 0; k < Lh; k += 2) {
    const bool two = k + 1 < Lh;
    const int64_t e1 = e0 + k, e2 = e0 + (two ? k + 1 : k);
    const int32_t c1 = sell_ld(S.col + e1 * 32 + lane, ST), c2 = sell_ld(S.col + e2 * 32 + lane, ST);
    const double2* v1 = reinterpret_cast<const double2*>(S.val + e1 * 288) + lane;
    const double2* v2 = reinterpret_cast<const double2*>(S.val + e2 * 288) + lane;
    const double2 p0 = sell_ld(v1, ST), p1 = sell_ld(v1 + 32, ST), p2 = sell_ld(v1 + 64, ST), p3 = sell_ld(v1 + 96, ST);
    const double p4 = sell_ld(S.val + e1 * 288 + 256 + lane, ST);
    const double2 q0 = sell_ld(v2, ST), q1 = sell_ld(v2 + 32, ST), q2 = sell_ld(v2 + 64, ST), q3 = sell_ld(v2 + 96, ST);
    const double q4 = sell_ld(S.val + e2 * 288 + 256 + lane, ST);
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

// Same accumulation with the lane's column DoFs already in shared memory
// (cols[j * 32 + lane], j < Lh) and its first entry row e0: the x gathers and
// the value loads issue together.
template <int H>
__device__ __forceinline__ void sell_acc_cached(const SellDev& S, int64_t e0, const int32_t* cols, int Lh, int lane,
                                                const double* x, double& a0, double& a1, double& a2) {
  for (int k = 0; k < Lh; k += 2) {
    const bool two = k + 1 < Lh;
    const int k2 = two ? k + 1 : k;
    const int64_t e1 = e0 + k, e2 = e0 + k2;
    const int32_t c1 = cols[k * 32 + lane], c2 = cols[k2 * 32 + lane];
    double x0, x1, x2, y0, y1, y2;
    load_vec3(x + c1, x0, x1, x2);
    load_vec3(x + c2, y0, y1, y2);
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

// Symmetric mode, pass 1 (one read of every upper block): lane `lane`'s share
// of its row's own product a = sum_c B_Rc x_c (dg: the diagonal block's part),
// and for every off-diagonal block the transposed product B^T x_R stored to
// its slot in the column row's slot run (pass 2 adds the runs, ys_solver.cu).
template <int H>
__device__ __forceinline__ void usell_acc(const SellDev& S, int64_t slice, int lane, const double* x, double (&a)[3],
                                          double (&dg)[3], int64_t& R) {
  constexpr int RPS = 32 / H;
  R = slice * RPS + lane / H;
  const int h = lane % H;
  const bool live = R < S.nb;
  const int L = live ? S.len[R] : 0;
  const int Lh = L > h ? (L - h + H - 1) / H : 0;
  const int64_t e0 = S.soff[slice];
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
  if (Lh > 0) load_vec3(x + 3 * R, r0, r1, r2);
  for (int k = 0; k < Lh; k += 2) {
    const bool two = k + 1 < Lh;
    const int64_t e1 = e0 + k, e2 = e0 + (two ? k + 1 : k);
    const int32_t c1 = __ldcs(S.col + e1 * 32 + lane), c2 = __ldcs(S.col + e2 * 32 + lane);
    const int32_t t1 = __ldcs(S.tpos + e1 * 32 + lane), t2 = __ldcs(S.tpos + e2 * 32 + lane);
    const double2* v1 = reinterpret_cast<const double2*>(S.val + e1 * 288) + lane;
    const double2* v2 = reinterpret_cast<const double2*>(S.val + e2 * 288) + lane;
    const double2 p0 = __ldcs(v1), p1 = __ldcs(v1 + 32), p2 = __ldcs(v1 + 64), p3 = __ldcs(v1 + 96);
    const double p4 = __ldcs(S.val + e1 * 288 + 256 + lane);
    const double2 q0 = __ldcs(v2), q1 = __ldcs(v2 + 32), q2 = __ldcs(v2 + 64), q3 = __ldcs(v2 + 96);
    const double q4 = __ldcs(S.val + e2 * 288 + 256 + lane);
    double x0, x1, x2, y0, y1, y2;
    load_vec3(x + c1, x0, x1, x2);
    load_vec3(x + c2, y0, y1, y2);
    {
      const double b0 = p0.x * x0 + p0.y * x1 + p1.x * x2;
      const double b1 = p1.y * x0 + p2.x * x1 + p2.y * x2;
      const double b2 = p3.x * x0 + p3.y * x1 + p4 * x2;
      a[0] += b0;
      a[1] += b1;
      a[2] += b2;
      if (t1 < 0) {
        dg[0] += b0;
        dg[1] += b1;
        dg[2] += b2;
      } else {
        double2* o = reinterpret_cast<double2*>(S.slots + 4 * int64_t(t1));
        o[0] = make_double2(p0.x * r0 + p1.y * r1 + p3.x * r2, p0.y * r0 + p2.x * r1 + p3.y * r2);
        o[1] = make_double2(p1.x * r0 + p2.y * r1 + p4 * r2, 0.0);
      }
    }
    if (two) {
      const double b0 = q0.x * y0 + q0.y * y1 + q1.x * y2;
      const double b1 = q1.y * y0 + q2.x * y1 + q2.y * y2;
      const double b2 = q3.x * y0 + q3.y * y1 + q4 * y2;
      a[0] += b0;
      a[1] += b1;
      a[2] += b2;
      if (t2 < 0) {
        dg[0] += b0;
        dg[1] += b1;
        dg[2] += b2;
      } else {
        double2* o = reinterpret_cast<double2*>(S.slots + 4 * int64_t(t2));
        o[0] = make_double2(q0.x * r0 + q1.y * r1 + q3.x * r2, q0.y * r0 + q2.x * r1 + q3.y * r2);
        o[1] = make_double2(q1.x * r0 + q2.y * r1 + q4 * r2, 0.0);
      }
    }
  }
  if (H > 1) {
#pragma unroll
    for (int off = H / 2; off > 0; off >>= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        a[i] += __shfl_xor_sync(0xffffffffu, a[i], off, H);
        dg[i] += __shfl_xor_sync(0xffffffffu, dg[i], off, H);
      }
  }
}

// Symmetric mode, pass 2 for block row R, SW lanes per row: the sum of its
// slot run (lane l takes slots l, l + SW, ..., then a fixed xor butterfly),
// valid in every lane of the group.  One 32 B sector per slot, L2-coherent
// loads (the slots were written by other CTAs).
template <int SW>
__device__ __forceinline__ void usell_tsum(const SellDev& S, int64_t R, int lane, unsigned mask, double (&t)[3]) {
  t[0] = t[1] = t[2] = 0.0;
  const int32_t j0 = S.tstart[R], j1 = S.tstart[R + 1];
  for (int32_t j = j0 + lane; j < j1; j += SW) {
    const double2* o = reinterpret_cast<const double2*>(S.slots + 4 * int64_t(j));
    const double2 a = __ldcg(o), b = __ldcg(o + 1);
    t[0] += a.x;
    t[1] += a.y;
    t[2] += b.x;
  }
#pragma unroll
  for (int off = SW / 2; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) t[i] += __shfl_xor_sync(mask, t[i], off, SW);
}

}  // namespace ys
