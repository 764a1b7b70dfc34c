// ys_sell.cu — builds the PCG's sliced-ELL full copy of H (ys_sell.cuh) from
// the static and dynamic upper-storage structures, once per solve.
//
// Cost at C5 (3.0 M full entries): one pass reading the 117 MB of upper
// blocks twice (own + transposed) and writing ~230 MB — a few tens of
// microseconds against the ~420 SpMVs of the solve that then stream it.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "ys_sell.cuh"

namespace ys {

namespace {

__device__ __forceinline__ int row_entries(const SpmvDev& S, int64_t R) {
  return (S.nrow[R + 1] - S.nrow[R]) + (S.trow[R + 1] - S.trow[R]);
}

__global__ void k_sell_len(SpmvDev S0, SpmvDev S1, int has1, int64_t nb, int sym, int32_t* len, int32_t* tcnt) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R >= nb) return;
  if (!sym) {
    len[R] = row_entries(S0, R) + (has1 ? row_entries(S1, R) : 0);
    return;
  }
  len[R] = (S0.nrow[R + 1] - S0.nrow[R]) + (has1 ? S1.nrow[R + 1] - S1.nrow[R] : 0);
  tcnt[R] = (S0.trow[R + 1] - S0.trow[R]) + (has1 ? S1.trow[R + 1] - S1.trow[R] : 0);
}

// Symmetric mode: slot of every off-diagonal upper block u = first slot of its
// column row + static transposed entries before it (dynamic after static).
__global__ void k_sell_utpos(SpmvDev S, int64_t nb, const int32_t* tstart, SpmvDev S0, int is_dyn, int32_t* utpos) {
  const int64_t C = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (C >= nb) return;
  const int32_t base = tstart[C] + (is_dyn ? S0.trow[C + 1] - S0.trow[C] : 0);
  const int32_t j0 = S.trow[C], j1 = S.trow[C + 1];
  for (int32_t j = j0; j < j1; ++j) utpos[S.tlist[j].x] = base + (j - j0);
}

// width of slice s (in entry rows) = max over its rows of ceil(len / H)
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
  int32_t* tpos;  // symmetric mode
};

__device__ __forceinline__ void put_entry(const SellOut& o, int64_t R, int k, int32_t xcol, const double* __restrict__ b,
                                          bool transpose, int32_t tp = -1) {
  const int rps = 32 / o.H;
  const int64_t slice = R / rps;
  const int lane = int(R % rps) * o.H + k % o.H;
  const int64_t e = o.soff[slice] + k / o.H;
  o.col[e * 32 + lane] = xcol;
  if (o.tpos) o.tpos[e * 32 + lane] = tp;
  double v[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) v[3 * i + j] = transpose ? b[3 * j + i] : b[3 * i + j];
  double* base = o.val + e * 288;
#pragma unroll
  for (int q = 0; q < 4; ++q) reinterpret_cast<double2*>(base)[q * 32 + lane] = make_double2(v[2 * q], v[2 * q + 1]);
  base[256 + lane] = v[8];
}

__device__ __forceinline__ int fill_from(const SpmvDev& S, const SellOut& o, int64_t R, int k) {
  for (int32_t u = S.nrow[R]; u < S.nrow[R + 1]; ++u) put_entry(o, R, k++, S.col[u], S.values + 9 * int64_t(u), false);
  for (int32_t j = S.trow[R]; j < S.trow[R + 1]; ++j) {
    const int2 t = S.tlist[j];
    put_entry(o, R, k++, t.y, S.values + 9 * int64_t(t.x), true);
  }
  return k;
}

__device__ __forceinline__ int fill_upper(const SpmvDev& S, const SellOut& o, int64_t R, int k, const int32_t* utpos) {
  for (int32_t u = S.nrow[R]; u < S.nrow[R + 1]; ++u) {
    const int32_t c = S.col[u];
    put_entry(o, R, k++, c, S.values + 9 * int64_t(u), false, c == 3 * int32_t(R) ? -1 : utpos[u]);
  }
  return k;
}

// One thread per block row; the threads of a slice write the same entry row
// together (coalesced stores).
__global__ void k_sell_fill(SpmvDev S0, SpmvDev S1, int has1, int64_t nb, SellOut o, const int32_t* utpos0,
                            const int32_t* utpos1) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R >= nb) return;
  if (o.tpos) {
    const int k = fill_upper(S0, o, R, 0, utpos0);
    if (has1) fill_upper(S1, o, R, k, utpos1);
    return;
  }
  int k = fill_from(S0, o, R, 0);
  if (has1) fill_from(S1, o, R, k);
}

// Symmetric mode, standalone: pass 1 (own products + transposed slots) and
// pass 2 (add the slot runs).
template <int H, int MINB>
__global__ void __launch_bounds__(kTB, MINB) k_spmv_usell1(SellDev S, const double* __restrict__ x,
                                                                double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t sl = w0; sl < S.nslices; sl += nw) {
    double a[3] = {0.0, 0.0, 0.0}, dg[3] = {0.0, 0.0, 0.0};
    int64_t R;
    usell_acc<H>(S, sl, lane, x, a, dg, R);
    if (lane % H == 0 && R < S.nb) {
      y[3 * R] = a[0];
      y[3 * R + 1] = a[1];
      y[3 * R + 2] = a[2];
    }
  }
}

__global__ void k_spmv_usell2(SellDev S, double* __restrict__ y) {
  constexpr int SW = 4;
  const int lane = threadIdx.x % SW;
  const unsigned mask = ((1u << SW) - 1u) << ((threadIdx.x & 31) & ~(SW - 1));
  const int64_t g0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / SW;
  const int64_t ng = int64_t(gridDim.x) * blockDim.x / SW;
  for (int64_t R = g0; R < S.nb; R += ng) {
    double t[3];
    usell_tsum<SW>(S, R, lane, mask, t);
    if (lane == 0) {
      y[3 * R] += t[0];
      y[3 * R + 1] += t[1];
      y[3 * R + 2] += t[2];
    }
  }
}

// Standalone y = H x through the sliced-ELL copy (timing diagnostics and the
// non-persistent path): one slice per warp, grid-stride.
template <int H, bool ST>
__global__ void __launch_bounds__(kTB, kSpmvMinB) k_spmv_sell(SellDev S, const double* __restrict__ x,
                                                              double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t sl = w0; sl < S.nslices; sl += nw) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int64_t R;
    sell_acc<H, ST>(S, sl, lane, x, a0, a1, a2, R);
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
  return SellDev{c.sell_len.p,  c.sell_soff.p,
                 c.sell_col.p,  c.sell_val.p,
                 c.NB,          c.sell_slices,
                 c.sell_sym ? c.sell_tpos.p : nullptr,
                 c.sell_sym ? c.sell_tstart.p : nullptr,
                 c.sell_sym ? c.sell_slots.p : nullptr};
}

// Builds the sliced-ELL copy of S[0] + S[1] (uniform 3x3 systems only) with H
// lanes per block row.  One host synchronisation (the entry-row count sizes
// the buffers).
void sell_build(Context& c, int H, bool sym) {
  cudaStream_t s = c.stream;
  const bool has1 = c.S[1].n_blocks > 0;
  SpmvDev d0 = spmv_dev(c.S[0]);
  SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
  const int64_t nb = c.NB;
  const int rps = 32 / H;
  const int64_t nsl = ceil_div(nb, rps);
  c.sell_h = H;
  c.sell_sym = sym;
  c.sell_slices = nsl;
  c.sell_len.resize(size_t(std::max<int64_t>(nb, 1)));
  c.sell_soff.resize(size_t(nsl + 1));
  if (nb == 0) {
    c.sell_rows = 0;
    return;
  }
  if (sym) c.sell_tstart.resize(size_t(nb + 1));
  k_sell_len<<<int(ceil_div(nb, kTB)), kTB, 0, s>>>(d0, d1, has1 ? 1 : 0, nb, sym ? 1 : 0, c.sell_len.p,
                                                    sym ? c.sell_tstart.p + 1 : nullptr);
  k_sell_width<<<int(ceil_div(nsl, kTB)), kTB, 0, s>>>(c.sell_len.p, nb, H, nsl, c.sell_soff.p);
  YS_LAUNCH_CHECK();
  int64_t* so = c.sell_soff.p;
  const int n = int(nsl + 1);
  size_t bytes = 0;
  YS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, so, so, n, s));
  c.cubtmp.resize(std::max<size_t>(bytes, 1));
  YS_CUDA(cub::DeviceScan::InclusiveSum(c.cubtmp.p, bytes, so, so, n, s));
  int64_t rows[2] = {0, 0};
  YS_CUDA(cudaMemcpyAsync(&rows[0], so + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (sym) {
    int32_t* ts = c.sell_tstart.p;
    YS_CUDA(cudaMemsetAsync(ts, 0, sizeof(int32_t), s));
    const int nt = int(nb + 1);
    YS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, ts, ts, nt, s));
    c.cubtmp.resize(std::max<size_t>(bytes, 1));
    YS_CUDA(cub::DeviceScan::InclusiveSum(c.cubtmp.p, bytes, ts, ts, nt, s));
    c.sell_utpos0.resize(size_t(std::max<int64_t>(c.S[0].n_blocks, 1)));
    c.sell_utpos1.resize(size_t(std::max<int64_t>(c.S[1].n_blocks, 1)));
    k_sell_utpos<<<int(ceil_div(nb, kTB)), kTB, 0, s>>>(d0, nb, ts, d0, 0, c.sell_utpos0.p);
    if (has1) k_sell_utpos<<<int(ceil_div(nb, kTB)), kTB, 0, s>>>(d1, nb, ts, d0, 1, c.sell_utpos1.p);
    YS_LAUNCH_CHECK();
    int32_t nslot = 0;
    YS_CUDA(cudaMemcpyAsync(&nslot, ts + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaStreamSynchronize(s));
    rows[1] = nslot;
    c.sell_slots.resize(size_t(4 * rows[1] + 4));
  }
  YS_CUDA(cudaStreamSynchronize(s));
  c.sell_rows = rows[0];
  c.sell_col.resize(size_t(rows[0] * 32 + 4));
  c.sell_val.resize(size_t(rows[0] * 288 + 4));
  if (sym) c.sell_tpos.resize(size_t(rows[0] * 32 + 4));
  k_sell_fill<<<int(ceil_div(nb, kTB)), kTB, 0, s>>>(
      d0, d1, has1 ? 1 : 0, nb, SellOut{c.sell_soff.p, c.sell_col.p, c.sell_val.p, H, sym ? c.sell_tpos.p : nullptr},
      c.sell_utpos0.p, c.sell_utpos1.p);
  YS_LAUNCH_CHECK();
}

// L2 residency of a streamed buffer: persisting-lines window over [base,
// base + bytes) on the context stream; frac scales the device's maximum
// persisting set-aside (0 clears the window).  Returns the bytes marked.
size_t l2_persist(Context& c, const void* base, size_t bytes, double frac) {
  static int max_persist = -1, max_window = 0;
  if (max_persist < 0) {
    YS_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c.device));
    YS_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c.device));
  }
  cudaStreamAttrValue a = {};
  if (frac <= 0.0 || bytes == 0 || max_persist <= 0) {
    a.accessPolicyWindow.num_bytes = 0;
    YS_CUDA(cudaStreamSetAttribute(c.stream, cudaStreamAttributeAccessPolicyWindow, &a));
    return 0;
  }
  const size_t set_aside = size_t(double(max_persist) * std::min(frac, 1.0));
  YS_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside));
  const size_t win = std::min(bytes, size_t(max_window));
  a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  a.accessPolicyWindow.num_bytes = win;
  a.accessPolicyWindow.hitRatio = float(std::min(1.0, double(set_aside) / double(win)));
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  YS_CUDA(cudaStreamSetAttribute(c.stream, cudaStreamAttributeAccessPolicyWindow, &a));
  fprintf(stderr, "[ys] L2 persist: max set-aside %d B, max window %d B, window %zu B, hitRatio %.3f\n", max_persist,
          max_window, win, double(a.accessPolicyWindow.hitRatio));
  return size_t(double(win) * a.accessPolicyWindow.hitRatio);
}

template <int H, bool ST = true>
static void launch_sell(Context& c, const double* x, double* y) {
  int occ = 0;
  YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv_sell<H, ST>, kTB, 0));
  const int64_t warps = c.sell_slices;
  const int g = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(std::max(occ, 1)) * sm_count(),
                                                           ceil_div(warps * 32, kTB))));
  k_spmv_sell<H, ST><<<g, kTB, 0, c.stream>>>(sell_dev(c), x, y);
  YS_LAUNCH_CHECK();
}

template <int H, int MINB = kSpmvMinB>
static void launch_usell(Context& c, const double* x, double* y) {
  int occ = 0;
  YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv_usell1<H, MINB>, kTB, 0));
  const int g = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(std::max(occ, 1)) * sm_count(),
                                                           ceil_div(c.sell_slices * 32, kTB))));
  static const int pass = getenv("YS_USELL_PASS") ? atoi(getenv("YS_USELL_PASS")) : 3;  // diagnostic: 1, 2 or both
  if (pass & 1) k_spmv_usell1<H, MINB><<<g, kTB, 0, c.stream>>>(sell_dev(c), x, y);
  if (pass & 2)
    k_spmv_usell2<<<int(std::min<int64_t>(ceil_div(c.NB * 4, kTB), 8 * sm_count())), kTB, 0, c.stream>>>(sell_dev(c),
                                                                                                     y);
  YS_LAUNCH_CHECK();
}

void spmv_sell(Context& c, const double* x, double* y, bool streaming) {
  if (c.sell_sym && !streaming) {  // diagnostic: 2 CTAs per SM (no spills)
    if (c.sell_h == 2) return launch_usell<2, 2>(c, x, y);
    if (c.sell_h == 4) return launch_usell<4, 2>(c, x, y);
  }
  if (c.sell_sym) {
    switch (c.sell_h) {
      case 1: return launch_usell<1>(c, x, y);
      case 2: return launch_usell<2>(c, x, y);
      case 4: return launch_usell<4>(c, x, y);
      case 8: return launch_usell<8>(c, x, y);
      default: fail(YS_ERR_INTERNAL, "sliced-ELL SpMV: unsupported lanes per row");
    }
  }
  if (!streaming) {  // diagnostic: default-policy loads
    if (c.sell_h == 4) return launch_sell<4, false>(c, x, y);
    if (c.sell_h == 8) return launch_sell<8, false>(c, x, y);
  }
  switch (c.sell_h) {
    case 1: launch_sell<1>(c, x, y); break;
    case 2: launch_sell<2>(c, x, y); break;
    case 4: launch_sell<4>(c, x, y); break;
    case 8: launch_sell<8>(c, x, y); break;
    default: fail(YS_ERR_INTERNAL, "sliced-ELL SpMV: unsupported lanes per row");
  }
}

}  // namespace ys
