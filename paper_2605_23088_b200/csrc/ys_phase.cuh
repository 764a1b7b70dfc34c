// ys_phase.cuh — the phases of the persistent uniform-3x3 PCG shared by the
// single-GPU solve (k_pcg33_stream, ys_solver.cu) and the peer-memory
// row-partitioned solve (k_dpcg_p2p, ys_dist.cu): phase A over the sliced-ELL
// copy with a per-warp plan cache, and the phase-B row update.
#pragma once

#include "ys_grid.cuh"
#include "ys_sell.cuh"

namespace ys {

__device__ __forceinline__ void prefetch_l2(const void* q) { asm volatile("prefetch.global.L2 [%0];" ::"l"(q)); }

struct SellPhaseA {
  SellDev SL;
  int64_t nb;
  int K, TW;
  int2* meta;
  int32_t* lhs;
  int32_t* cols;
  int kn, wl, grp, h, warp;
  int64_t gw, NW;
  uint64_t pol;  // L2 evict_last for the vectors

  // cb / G: this CTA's index and the CTA count of the rank (the whole grid
  // for the single-GPU solve; one rank's share of an emulated multi-rank grid)
  __device__ void prologue(double* smem) { prologue(smem, int(blockIdx.x), int(gridDim.x)); }
  __device__ void prologue(double* smem, int cb, int G) {
    constexpr int H = 4, RPS = 32 / H, WPB = kTB / 32;
    warp = threadIdx.x >> 5;
    wl = threadIdx.x & 31;
    grp = wl / H;
    h = wl % H;
    gw = int64_t(cb) * WPB + warp;
    NW = int64_t(G) * WPB;
    pol = l2_keep_policy();
    // per warp K int2 {first entry row, local entry-row offset}, K x 32 lane
    // counts, TW x 32 column DoFs
    meta = reinterpret_cast<int2*>(smem) + warp * K;
    lhs = reinterpret_cast<int32_t*>(reinterpret_cast<int2*>(smem) + WPB * K) + warp * K * 32;
    cols = lhs + (WPB - warp) * K * 32 + warp * TW * 32;
    kn = gw < SL.nslices ? int(min(int64_t(K), (SL.nslices - gw + NW - 1) / NW)) : 0;
    int off = 0;
    for (int k = 0; k < kn; ++k) {
      const int64_t sl = gw + k * NW;
      const int64_t e0 = SL.soff[sl], e1 = SL.soff[sl + 1];
      const int64_t q = sl * RPS + grp;
      const int L = q < SL.nb - SL.r0 ? SL.len[q] : 0;
      const int Lh = L > h ? (L - h + H - 1) / H : 0;
      if (wl == 0) meta[k] = make_int2(int(e0), off);
      lhs[k * 32 + wl] = Lh;
      for (int j = 0; j < Lh; ++j) cols[(off + j) * 32 + wl] = SL.col[(e0 + j) * 32 + wl];
      off += int(e1 - e0);
    }
    __syncwarp();
  }

  // hp = H p for the warp's rows; returns this thread's pHp partial
  __device__ double run(const double* __restrict__ p, double* __restrict__ hp) {
    constexpr int H = 4, RPS = 32 / H;
    double dot = 0.0;
    for (int k = 0; k < kn; ++k) {
      const int2 m = meta[k];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      sell_acc_cached<H>(SL, m.x, cols + m.y * 32, lhs[k * 32 + wl], wl, p, a0, a1, a2, pol);
      const int64_t q = (gw + k * NW) * RPS + grp;
      if (h == 0 && q < SL.nb - SL.r0) {
        const int64_t R = sell_row(SL, q);
        double* yo = hp + 3 * R;
        st_keep(yo, a0, pol);
        st_keep(yo + 1, a1, pol);
        st_keep(yo + 2, a2, pol);
        dot += p[3 * R] * a0 + p[3 * R + 1] * a1 + p[3 * R + 2] * a2;
      }
    }
    return dot;
  }
};

// Phase-B rows of one thread: b0 = global thread id, b0 + threads, ...  The
// operands of the first row (p, r, x, M^-1 — none written in phase A) are
// prefetched into L2 between the barrier's arrive and wait.

struct RowRegs {
  double p[3], r[3], x[3], M[9], z[3];
};

__device__ __forceinline__ void rowregs_load(RowRegs& q, int64_t b, const double* __restrict__ p,
                                             const double* __restrict__ r, const double* __restrict__ x,
                                             const double* __restrict__ minv, uint64_t pol) {
  load_vec3_keep(p + 3 * b, q.p[0], q.p[1], q.p[2], pol);
  load_vec3_keep(r + 3 * b, q.r[0], q.r[1], q.r[2], pol);
  load_vec3_keep(x + 3 * b, q.x[0], q.x[1], q.x[2], pol);
  load_block9_keep(minv + 9 * b, q.M, pol);
}

// x += a p, r -= a hp, z = M^-1 r (stores x, r; z stays in q), r.r / r.z partials
__device__ __forceinline__ void rowregs_update(RowRegs& q, int64_t b, double alpha, const double* hp, double* x,
                                               double* r, double (&v)[2], uint64_t pol) {
  double hh[3];
  load_vec3_keep(hp + 3 * b, hh[0], hh[1], hh[2], pol);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    q.x[i] += alpha * q.p[i];
    q.r[i] -= alpha * hh[i];
  }
  precond_apply<3>(q.M, q.r, q.z);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    st_keep(x + 3 * b + i, q.x[i], pol);
    st_keep(r + 3 * b + i, q.r[i], pol);
    v[0] += q.r[i] * q.r[i];
    v[1] += q.r[i] * q.z[i];
  }
}


}  // namespace ys
