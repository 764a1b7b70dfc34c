// ys_sell.cu — builds the PCG's sliced-ELL full copy of H (ys_sell.cuh) from
// the static and dynamic upper-storage structures, once per solve.
//
// Cost at C5 (3.0 M full entries): one pass reading the upper blocks twice
// (own + transposed) and writing the ~230 MB copy — a few hundred
// microseconds against the ~420 SpMVs of the solve that then stream it.
//
// Measured and rejected (C5, B200, profiles/r01_pcg_sell_c5.md):
//  * a symmetric copy — upper blocks streamed once, B^T x_R stored to a
//    per-column-row slot (32 B, sector aligned), slot runs summed after the
//    barrier: 137 MB instead of ~260 MB per SpMV, but the scattered slot
//    stores and the slot gathers made phases A + B 140 us vs 56 us;
//  * an L2 persisting window over the copy (83 MB set-aside): 49 -> 51-56 us;
//  * bulk L2 prefetch (cp.async.bulk.prefetch) of each warp's next slice:
//    49 -> 58 us.
#include <cub/cub.cuh>

#include <algorithm>

#include "ys_sell.cuh"

namespace ys {

namespace {

__device__ __forceinline__ int row_entries(const SpmvDev& S, int64_t R) {
  return (S.nrow[R + 1] - S.nrow[R]) + (S.trow[R + 1] - S.trow[R]);
}

// Row R's own blocks are sorted by column, so its diagonal block (if any) is
// the first one of each group.
__device__ __forceinline__ bool has_diag(const SpmvDev& S, int64_t R) {
  return S.nrow[R + 1] > S.nrow[R] && S.col[S.nrow[R]] == 3 * int32_t(R);
}

// The dynamic group's diagonal block of a row is merged into the static one
// (one entry, B_s + B_d): the contact rows lose one entry each.
__global__ void k_sell_len(SpmvDev S0, SpmvDev S1, int has1, int64_t r0, int64_t r1, int32_t* len) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t R = r0 + q;
  if (R >= r1) return;
  int n = row_entries(S0, R);
  if (has1) n += row_entries(S1, R) - ((has_diag(S0, R) && has_diag(S1, R)) ? 1 : 0);
  len[q] = n;
}

// perm / lenq: inside each window of kSellSigma positions the rows sorted by
// entry count, descending (stable: ties keep the row order).
__global__ void __launch_bounds__(kSellSigma) k_sell_sort_windows(const int32_t* len, int64_t r0, int64_t nb,
                                                                  int32_t* perm, int32_t* lenq) {
  using Sort = cub::BlockRadixSort<uint32_t, kSellSigma, 1, int32_t>;
  __shared__ typename Sort::TempStorage tmp;
  const int64_t q = int64_t(blockIdx.x) * kSellSigma + threadIdx.x;
  const bool live = q < nb;
  const int L = live ? len[q] : 0;
  // key: 0..1023 = 1023 - len for live rows (longest first), 1024 for padding
  uint32_t key[1] = {live ? uint32_t(1023 - min(L, 1023)) : 1024u};
  int32_t val[1] = {int32_t(q)};
  Sort(tmp).Sort(key, val, 0, 11);
  if (live) {
    perm[q] = int32_t(r0) + val[0];
    lenq[q] = len[val[0]];
  }
}

// width of slice s (in entry rows) = max over its rows of ceil(len / H); len and
// nb relative to the range
__global__ void k_sell_width(const int32_t* len, int64_t nb, int H, int64_t nslices, int64_t* width) {
  const int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  const int rps = 32 / H;
  int w = 0;
  for (int i = 0; i < rps; ++i) {
    const int64_t R = s * rps + i;
    if (R < nb) w = max(w, (len[R] + H - 1) / H);
  }
  width[s + 1] = w;
  if (s == 0) width[0] = 0;
}

struct SellOut {
  const int64_t* soff;
  int32_t* col;
  double* val;
  int H;
  int64_t r0;
};

// One lane per (row, k mod H) of a slice: lane l fills the entries k = l mod H,
// l mod H + H, ... of row l / H, i.e. exactly its own lane column of every
// entry row of the slice — each store instruction of the warp covers whole
// contiguous runs.  Entries of a row: static own (the dynamic diagonal block merged
// into the static one), static transposed, dynamic own, dynamic transposed.
__global__ void k_sell_fill_lanes(SpmvDev S0, SpmvDev S1, int has1, int64_t r0, int64_t r1, int H,
                                  const int32_t* __restrict__ perm, SellOut o) {
  const int64_t gt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t sl = gt >> 5;
  const int lane = int(gt & 31);
  const int rps = 32 / H;
  const int64_t q = sl * rps + lane / H;
  if (r0 + q >= r1) return;
  const int64_t R = perm[q];
  const int j = lane % H;
  const bool merge = has1 && has_diag(S0, R) && has_diag(S1, R);
  // segments: S0 own, S0 transposed, S1 own (minus a merged diagonal), S1 transposed
  const int32_t n0 = S0.nrow[R + 1] - S0.nrow[R], t0 = S0.trow[R + 1] - S0.trow[R];
  const int32_t u1 = has1 ? S1.nrow[R] + (merge ? 1 : 0) : 0;
  const int32_t n1 = has1 ? S1.nrow[R + 1] - u1 : 0, t1 = has1 ? S1.trow[R + 1] - S1.trow[R] : 0;
  const int L = n0 + t0 + n1 + t1;
  const int64_t e0 = o.soff[sl];
  for (int k = j; k < L; k += H) {
    int32_t xcol;
    const double* b;
    bool tr = false;
    const double* b2 = nullptr;
    if (k < n0) {
      const int32_t u = S0.nrow[R] + k;
      xcol = S0.col[u];
      b = S0.values + 9 * int64_t(u);
      if (k == 0 && merge) b2 = S1.values + 9 * int64_t(S1.nrow[R]);
    } else if (k < n0 + t0) {
      const int2 t = S0.tlist[S0.trow[R] + (k - n0)];
      xcol = t.y;
      b = S0.values + 9 * int64_t(t.x);
      tr = true;
    } else if (k < n0 + t0 + n1) {
      const int32_t u = u1 + (k - n0 - t0);
      xcol = S1.col[u];
      b = S1.values + 9 * int64_t(u);
    } else {
      const int2 t = S1.tlist[S1.trow[R] + (k - n0 - t0 - n1)];
      xcol = t.y;
      b = S1.values + 9 * int64_t(t.x);
      tr = true;
    }
    const int64_t e = e0 + k / H;
    o.col[e * 32 + lane] = xcol;
    double v[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int jj = 0; jj < 3; ++jj) v[3 * i + jj] = tr ? b[3 * jj + i] : b[3 * i + jj];
    if (b2)
#pragma unroll
      for (int i = 0; i < 9; ++i) v[i] += b2[i];
    double* base = o.val + e * 288;
#pragma unroll
    for (int q = 0; q < 4; ++q) reinterpret_cast<double2*>(base)[q * 32 + lane] = make_double2(v[2 * q], v[2 * q + 1]);
    base[256 + lane] = v[8];
  }
}

// Standalone y = H x through the sliced-ELL copy (ys_time_kernel and
// YS_APPLY_VARIANT diagnostics): one slice per warp, grid-stride.
template <int H>
__global__ void __launch_bounds__(kTB, kSpmvMinB) k_spmv_sell(SellDev S, const double* __restrict__ x,
                                                              double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t sl = w0; sl < S.nslices; sl += nw) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int64_t R;
    sell_acc<H>(S, sl, lane, x, a0, a1, a2, R);
    if (lane % H == 0 && R < S.nb) {
      y[3 * R] = a0;
      y[3 * R + 1] = a1;
      y[3 * R + 2] = a2;
    }
  }
}

// Entry rows of the slices gw + k NW (k < K) of every warp gw: the maximum
// sizes the persistent PCG's shared column cache.
__global__ void k_warp_rows(const int64_t* soff, int64_t nslices, int64_t NW, int K, int* out) {
  const int64_t gw = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gw >= NW) return;
  int64_t t = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t sl = gw + k * NW;
    if (sl >= nslices) break;
    t += soff[sl + 1] - soff[sl];
  }
  atomicMax(out, int(t));
}

}  // namespace

int sell_max_warp_rows(Context& c, int64_t NW, int K) {
  if (NW == c.sell_tw_nw && K == int(ceil_div(c.sell_slices, NW))) return c.sell_tw_host;  // from sell_build
  cudaStream_t s = c.stream;
  c.sell_tw.resize(1);
  YS_CUDA(cudaMemsetAsync(c.sell_tw.p, 0, sizeof(int), s));
  k_warp_rows<<<int(ceil_div(NW, kTB)), kTB, 0, s>>>(c.sell_soff.p, c.sell_slices, NW, K, c.sell_tw.p);
  YS_LAUNCH_CHECK();
  int v = 0;
  YS_CUDA(cudaMemcpyAsync(&v, c.sell_tw.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  return v;
}

SellDev sell_dev(Context& c) {
  return SellDev{c.sell_lenq.p, c.sell_soff.p, c.sell_col.p, c.sell_val.p, c.sell_r1, c.sell_slices, c.sell_r0,
                 c.sell_perm.p};
}

// Builds the sliced-ELL copy of S[0] + S[1] (uniform 3x3 systems only) with H
// lanes per block row, over the block rows [r0, r1) (r1 < 0: all rows).  One host synchronisation (the entry-row count sizes
// the buffers).
// The copy's layout (entry counts, window sort, slice widths, offsets) depends
// on the block structure only; sell_prepare builds it ahead of the values —
// Newton steps call it right after the dynamic rebuild, while the static
// evaluation still runs on the side streams — and the next sell_build with the
// same (H, r0, r1) only fills the values.
static void sell_layout(Context& c, int H, int64_t r0, int64_t r1);

void sell_prepare(Context& c, int H, int64_t r0, int64_t r1) {
  if (r1 < 0) r1 = c.NB;
  sell_layout(c, H, r0, r1);
  c.sell_prepared = true;
}

// The values of the prepared single-GPU copy, filled on stream s (the side
// stream, beside the preconditioner build): the next sell_build(c, 4) finds
// them ready.
void sell_fill_early(Context& c, cudaStream_t s) {
  if (!(c.sell_prepared && c.sell_h == 4 && c.sell_r0 == 0 && c.sell_r1 == c.NB) || c.NB == 0) return;
  c.sell_prepared = false;
  const bool has1 = c.S[1].n_blocks > 0;
  SpmvDev d0 = spmv_dev(c.S[0]);
  SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
  k_sell_fill_lanes<<<int(ceil_div(c.sell_slices * 32, kTB)), kTB, 0, s>>>(
      d0, d1, has1 ? 1 : 0, 0, c.NB, 4, c.sell_perm.p, SellOut{c.sell_soff.p, c.sell_col.p, c.sell_val.p, 4, 0});
  YS_LAUNCH_CHECK();
  c.sell_filled = true;
}

void sell_build(Context& c, int H, int64_t r0, int64_t r1) {
  if (r1 < 0) r1 = c.NB;
  if (c.sell_filled) {
    c.sell_filled = false;
    if (c.sell_h == H && c.sell_r0 == r0 && c.sell_r1 == r1) return;  // filled by sell_fill_early
  }
  const bool ready = c.sell_prepared && c.sell_h == H && c.sell_r0 == r0 && c.sell_r1 == r1;
  c.sell_prepared = false;
  if (!ready) sell_layout(c, H, r0, r1);
  if (r1 - r0 == 0) return;
  const bool has1 = c.S[1].n_blocks > 0;
  SpmvDev d0 = spmv_dev(c.S[0]);
  SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
  k_sell_fill_lanes<<<int(ceil_div(c.sell_slices * 32, kTB)), kTB, 0, c.stream>>>(
      d0, d1, has1 ? 1 : 0, r0, r1, H, c.sell_perm.p, SellOut{c.sell_soff.p, c.sell_col.p, c.sell_val.p, H, r0});
  YS_LAUNCH_CHECK();
}

static void sell_layout(Context& c, int H, int64_t r0, int64_t r1) {
  cudaStream_t s = c.stream;
  const bool has1 = c.S[1].n_blocks > 0;
  SpmvDev d0 = spmv_dev(c.S[0]);
  SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
  const int64_t nb = r1 - r0;
  const int rps = 32 / H;
  const int64_t nsl = ceil_div(nb, rps);
  c.sell_h = H;
  c.sell_r0 = r0;
  c.sell_r1 = r1;
  c.sell_slices = nsl;
  c.sell_len.resize(size_t(std::max<int64_t>(nb, 1)));
  c.sell_lenq.resize(size_t(std::max<int64_t>(nb, 1)));
  c.sell_perm.resize(size_t(std::max<int64_t>(nb, 1)));
  c.sell_soff.resize(size_t(nsl + 1));
  if (nb == 0) {
    c.sell_rows = 0;
    return;
  }
  k_sell_len<<<int(ceil_div(nb, kTB)), kTB, 0, s>>>(d0, d1, has1 ? 1 : 0, r0, r1, c.sell_len.p);
  k_sell_sort_windows<<<int(ceil_div(nb, kSellSigma)), kSellSigma, 0, s>>>(c.sell_len.p, r0, nb, c.sell_perm.p,
                                                                           c.sell_lenq.p);
  k_sell_width<<<int(ceil_div(nsl, kTB)), kTB, 0, s>>>(c.sell_lenq.p, nb, H, nsl, c.sell_soff.p);
  YS_LAUNCH_CHECK();
  int64_t* so = c.sell_soff.p;
  const int n = int(nsl + 1);
  size_t bytes = 0;
  YS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, so, so, n, s));
  c.cubtmp.resize(std::max<size_t>(bytes, 1));
  YS_CUDA(cub::DeviceScan::InclusiveSum(c.cubtmp.p, bytes, so, so, n, s));
  // the persistent PCG's plan-cache size for its grid (3 CTAs of 8 warps per
  // SM) comes back with the same synchronisation
  const int64_t nw = int64_t(kSpmvMinB) * sm_count() * (kTB / 32);
  const int kw = int(ceil_div(nsl, nw));
  c.sell_tw.resize(1);
  YS_CUDA(cudaMemsetAsync(c.sell_tw.p, 0, sizeof(int), s));
  k_warp_rows<<<int(ceil_div(nw, kTB)), kTB, 0, s>>>(so, nsl, nw, kw, c.sell_tw.p);
  YS_LAUNCH_CHECK();
  int64_t rows = 0;
  int tw = 0;
  YS_CUDA(cudaMemcpyAsync(&rows, so + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaMemcpyAsync(&tw, c.sell_tw.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  c.sell_rows = rows;
  c.sell_tw_nw = nw;
  c.sell_tw_host = tw;
  c.sell_col.resize(size_t(rows * 32 + 4));
  c.sell_val.resize(size_t(rows * 288 + 4));
}

template <int H>
static void launch_sell(Context& c, const double* x, double* y) {
  int occ = 0;
  YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv_sell<H>, kTB, 0));
  const int64_t warps = c.sell_slices;
  const int g = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(std::max(occ, 1)) * sm_count(),
                                                           ceil_div(warps * 32, kTB))));
  k_spmv_sell<H><<<g, kTB, 0, c.stream>>>(sell_dev(c), x, y);
  YS_LAUNCH_CHECK();
}

void spmv_sell(Context& c, const double* x, double* y) {
  switch (c.sell_h) {
    case 1: launch_sell<1>(c, x, y); break;
    case 2: launch_sell<2>(c, x, y); break;
    case 4: launch_sell<4>(c, x, y); break;
    case 8: launch_sell<8>(c, x, y); break;
    default: fail(YS_ERR_INTERNAL, "sliced-ELL SpMV: unsupported lanes per row");
  }
}

}  // namespace ys
