// ys_dist.cu — row-partitioned multi-GPU PCG.
//
// One process per GPU.  Every rank holds the replicated scene, structures and
// assembled values; the solve splits the block rows into contiguous ranges
// balanced by stored entries (own + transposed, static + dynamic, + 1 per row
// for the vector work).  Per iteration (same recurrence as pcg,
// solver.cpp:151-200):
//
//   SpMV     hp = H p on owned rows (sliced-ELL copy of the owned rows);
//            pHp rank partial                      -> allgather -> alpha
//   update   x, r, z on owned rows; r.r, r.z partials plus z and the
//            pre-update p of the export rows       -> allgather -> rel, beta
//   p        p = z + beta p on owned rows, and on the halo rows from the
//            received z and p (the owner's formula: bitwise the owner's p)
// (the initial p halo is exchanged once before the loop).
//
// Every rank sums the gathered partials in rank order, so alpha / beta /
// status are bit-identical on all ranks and the loop ends on the same
// iteration everywhere; results are deterministic for a fixed rank count.
// Export rows are the rows referenced by a block whose other side is owned
// by a different rank (a block (R, C) makes row R need p_C and row C need
// p_R).  The transport of this loop is a single allgather primitive:
// ncclAllGather on the context stream (libnccl.so.2 dlopen-ed), or a host
// callback (tests).
//
// Transport kind 3 (peer memory, k_dpcg_p2p below) keeps the single-GPU
// structure per rank instead: one persistent cooperative kernel per rank for
// the whole solve, exchanging through NVLink peer memory with device-side
// flags — no host round trip and no collective launch per iteration.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <string>

#include <cub/cub.cuh>

#include "ys_phase.cuh"

namespace ys {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the library itself has no NCCL link dependency)
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = e ? e : "libnccl.so.2 not found";
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  if (!api.ok) fail(YS_ERR_CUDA, "NCCL unavailable: " + api.why);
  return api;
}

#define YS_NCCL(x)                                                                        \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess) ::ys::fail(YS_ERR_CUDA, std::string("NCCL: ") + nccl().GetErrorString(r_)); \
  } while (0)

constexpr int kMaxRanks = 64;

// ---------------------------------------------------------------------------
// Plan kernels

// Largest k with bounds[k] <= v (bounds nondecreasing, bounds[0] == 0).
__device__ __forceinline__ int owner_of(const int64_t* bounds, int n, int64_t v) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (bounds[mid] <= v) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Work prefix W(R) = entries of rows < R (own + transposed, both structures)
// + R; bounds[k] = first R with W(R) >= k W(NB) / n.  The four prefix arrays
// already are per-row entry offsets, so no scan is needed.
__global__ void k_partition(const int32_t* n0, const int32_t* t0, const int32_t* n1, const int32_t* t1, int64_t nb,
                            int n, int64_t* bounds) {
  const int k = threadIdx.x;
  if (k > n) return;
  auto W = [&](int64_t R) {
    return int64_t(n0[R]) + t0[R] + (n1 ? int64_t(n1[R]) + t1[R] : int64_t(0)) + R;
  };
  if (k == 0) {
    bounds[0] = 0;
    return;
  }
  if (k == n) {
    bounds[n] = nb;
    return;
  }
  const int64_t target = W(nb) * k / n;
  int64_t lo = 0, hi = nb;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (W(mid) < target) lo = mid + 1;
    else hi = mid;
  }
  bounds[k] = lo;
}

// Uniform 3x3 structures: block (R, C) across a rank boundary -> both rows exported.
__global__ void k_mark_need(const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t nblocks,
                            const int64_t* __restrict__ bounds, int n, uint8_t* need) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nblocks) return;
  const int64_t R = row[u] / 3, C = col[u] / 3;
  if (R == C || owner_of(bounds, n, R) == owner_of(bounds, n, C)) return;
  need[R] = 1;
  need[C] = 1;
}

// exp_off[k] = first export row >= bounds[k] (exp sorted).
__global__ void k_exp_offsets(const int32_t* exp, const int32_t* nsel, const int64_t* bounds, int n,
                              int64_t* exp_off) {
  const int k = threadIdx.x;
  if (k > n) return;
  int64_t lo = 0, hi = *nsel;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (exp[mid] < bounds[k]) lo = mid + 1;
    else hi = mid;
  }
  exp_off[k] = lo;
}

// ---------------------------------------------------------------------------
// Exchange kernels

__global__ void k_pack(const double* __restrict__ p, const int32_t* __restrict__ exp, int64_t cnt,
                       double* __restrict__ send, const PcgState* st) {
  if (st && st->status) return;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 3 * cnt) return;
  send[i] = p[3 * int64_t(exp[i / 3]) + i % 3];
}

__global__ void k_unpack(const double* __restrict__ recv, const int32_t* __restrict__ exp,
                         const int64_t* __restrict__ exp_off, int n, int me, int64_t maxc, int64_t total,
                         double* __restrict__ p, const PcgState* st) {
  if (st && st->status) return;
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= 3 * total) return;
  const int64_t e = j / 3;
  const int k = owner_of(exp_off, n, e);
  if (k == me) return;
  p[3 * int64_t(exp[e]) + j % 3] = recv[(int64_t(k) * maxc + (e - exp_off[k])) * 3 + j % 3];
}

// Fused exchange: after the update phase each rank sends, in one allgather,
// its r.r / r.z partials, z and the pre-update p of its export rows; every
// receiver forms the halo p = z + beta p itself (the owner's formula and
// operands: bitwise the owner's value), so the p halo needs no exchange of
// its own.  Send layout: [2 partials][3 max_exp z][3 max_exp p].
__global__ void k_pack_zp(const double* __restrict__ z, const double* __restrict__ p,
                          const int32_t* __restrict__ exp, int64_t cnt, int64_t maxc, double* __restrict__ send,
                          const PcgState* st) {
  if (st->status) return;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 3 * cnt) return;
  const int64_t g = 3 * int64_t(exp[i / 3]) + i % 3;
  send[2 + i] = z[g];
  send[2 + 3 * maxc + i] = p[g];
}

__global__ void k_unpack_zp(const double* __restrict__ recv, const int32_t* __restrict__ exp,
                            const int64_t* __restrict__ exp_off, int n, int me, int64_t maxc, int64_t total,
                            double* __restrict__ p, const PcgState* st) {
  if (st->status) return;
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= 3 * total) return;
  const int64_t e = j / 3;
  const int k = owner_of(exp_off, n, e);
  if (k == me) return;
  const double* rk = recv + int64_t(k) * (2 + 6 * maxc);
  const int64_t q = (e - exp_off[k]) * 3 + j % 3;
  const double b = st->beta;
  const double zz = rk[2 + q], pp = rk[2 + 3 * maxc + q];
  p[3 * int64_t(exp[e]) + j % 3] = zz + b * pp;
}

// x slices of every rank -> the full vector (rank k's rows at slot k).
__global__ void k_gather_rows(const double* __restrict__ recv, const int64_t* __restrict__ bounds, int n,
                              int64_t maxr, int64_t nb, double* __restrict__ x) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= 3 * nb) return;
  const int64_t R = j / 3;
  const int k = owner_of(bounds, n, R);
  x[j] = recv[(int64_t(k) * maxr + (R - bounds[k])) * 3 + j % 3];
}

__global__ void k_copy_rows(const double* __restrict__ x, int64_t r0, int64_t r1, double* __restrict__ send) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 3 * (r1 - r0)) return;
  send[i] = x[3 * r0 + i];
}

// ---------------------------------------------------------------------------
// Solver kernels over the owned rows [r0, r1); rank partials -> out.


// The same over the sliced-ELL copy of the owned rows (sell_build(c, 4, r0,
// r1): every block touching an owned row, stored for that row): coalesced
// value stream, one slice of 8 rows per warp, grid-stride.
__global__ void __launch_bounds__(kTB, kSpmvMinB) k_dspmv_sell(SellDev SL, const double* __restrict__ x,
                                                               double* __restrict__ y, PcgState* st, double* part,
                                                               double* out) {
  if (st->status) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  double dot[1] = {0.0};
  for (int64_t sl = w0; sl < SL.nslices; sl += nw) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int64_t R;
    sell_acc<4>(SL, sl, lane, x, a0, a1, a2, R);
    if ((lane & 3) == 0 && R < SL.nb) {
      double* yo = y + 3 * R;
      yo[0] = a0;
      yo[1] = a1;
      yo[2] = a2;
      dot[0] += x[3 * R] * a0 + x[3 * R + 1] * a1 + x[3 * R + 2] * a2;
    }
  }
  block_reduce<1>(dot);
  if (threadIdx.x == 0) part[blockIdx.x] = dot[0];
  if (!last_cta(&st->counter1)) return;
  double tot[1];
  sum_partials<1>(part, gridDim.x, 0, tot);
  if (threadIdx.x == 0) {
    st->counter1 = 0;
    out[0] = tot[0];
  }
}

// r = g; z = M^-1 r; p = z; x = 0 on owned rows; rank partials of g.g, r.z.
__global__ void k_dinit(const double* __restrict__ g, const double* __restrict__ minv, double* r, double* z,
                        double* p, double* x, int64_t r0, int64_t r1, PcgState* st, double* part, double* out) {
  double v[2] = {0.0, 0.0};
  for (int64_t b = r0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < r1;
       b += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s0 = 3 * b;
    double rr[3], zz[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rr[i] = g[s0 + i];
      r[s0 + i] = rr[i];
      x[s0 + i] = 0.0;
    }
    precond_apply<3>(minv + 9 * b, rr, zz);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      z[s0 + i] = zz[i];
      p[s0 + i] = zz[i];
      v[0] += rr[i] * rr[i];
      v[1] += rr[i] * zz[i];
    }
  }
  block_reduce<2>(v);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = v[0];
    part[gridDim.x + blockIdx.x] = v[1];
  }
  if (!last_cta(&st->counter2)) return;
  double tot[2];
  sum_partials<2>(part, gridDim.x, gridDim.x, tot);
  if (threadIdx.x == 0) {
    st->counter2 = 0;
    out[0] = tot[0];
    out[1] = tot[1];
  }
}

// Rank-ordered sums of the gathered partials (identical on every rank).
template <int K>
__device__ __forceinline__ void rank_sums(const double* all, int n, double (&t)[K], int64_t stride = K) {
#pragma unroll
  for (int k = 0; k < K; ++k) t[k] = 0.0;
  for (int q = 0; q < n; ++q)
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] += all[q * stride + k];
}

__global__ void k_dinit_fin(PcgState* st, const double* all, int n, double* hist) {
  double t[2];
  rank_sums<2>(all, n, t);
  st->gnorm = sqrt(t[0]);
  st->rz = t[1];
  st->it = 0;
  st->rel = 0.0;
  st->fail_it = -1;
  if (st->gnorm == 0.0) {
    st->status = 1;  // converged with x = 0 (solver.cpp:156-159)
  } else {
    st->status = st->max_iter > 0 ? 0 : 5;
    st->rel = 1.0;
    hist[0] = 1.0;
  }
}

__global__ void k_dalpha(PcgState* st, const double* all, int n) {
  if (st->status) return;
  double t[1];
  rank_sums<1>(all, n, t);
  const double php = t[0];
  st->php = php;
  if (!isfinite(php) || php <= 0.0) {
    if (php == 0.0) {
      st->status = 2;
    } else {
      st->status = 3;
      st->fail_it = int(st->it);
    }
  } else {
    st->alpha = st->rz / php;
  }
}

__global__ void __launch_bounds__(kTB) k_dupdate(const double* __restrict__ minv, double* __restrict__ x,
                                                 double* __restrict__ r, double* __restrict__ z,
                                                 const double* __restrict__ p, const double* __restrict__ hp,
                                                 int64_t r0, int64_t r1, PcgState* st, double* part, double* out) {
  if (st->status) return;
  const double a = st->alpha;
  double v[2] = {0.0, 0.0};
  for (int64_t b = r0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < r1;
       b += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s0 = 3 * b;
    double rr[3], zz[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      x[s0 + i] += a * p[s0 + i];
      rr[i] = r[s0 + i] - a * hp[s0 + i];
      r[s0 + i] = rr[i];
    }
    precond_apply<3>(minv + 9 * b, rr, zz);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      z[s0 + i] = zz[i];
      v[0] += rr[i] * rr[i];
      v[1] += rr[i] * zz[i];
    }
  }
  block_reduce<2>(v);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = v[0];
    part[gridDim.x + blockIdx.x] = v[1];
  }
  if (!last_cta(&st->counter2)) return;
  double tot[2];
  sum_partials<2>(part, gridDim.x, gridDim.x, tot);
  if (threadIdx.x == 0) {
    st->counter2 = 0;
    out[0] = tot[0];
    out[1] = tot[1];
  }
}

// rel, history, convergence test, beta (solver.cpp:183-197).
__global__ void k_dbeta(PcgState* st, const double* all, int n, double* hist, int64_t stride) {
  if (st->status) return;
  double t[2];
  rank_sums<2>(all, n, t, stride);
  const long long it = st->it;
  const double rel = sqrt(t[0]) / st->gnorm;
  st->it = it + 1;
  st->rel = rel;
  if (it + 1 < st->hist_cap) hist[it + 1] = rel;
  if (!isfinite(rel)) {
    st->status = 4;
    st->fail_it = int(it);
  } else if (rel <= st->tol) {
    st->status = 1;
  } else if (it + 1 >= st->max_iter) {
    st->status = 5;
  } else {
    st->beta = t[1] / st->rz;
    st->rz = t[1];
  }
}

__global__ void k_dpupdate(const double* __restrict__ z, double* __restrict__ p, int64_t r0, int64_t r1,
                           const PcgState* st) {
  if (st->status) return;
  const double b = st->beta;
  for (int64_t i = 3 * r0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < 3 * r1;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = z[i] + b * p[i];
}

unsigned blocks_for(int64_t n) { return unsigned(std::max<int64_t>(1, ceil_div(n, kTB))); }

int vgrid(int64_t rows) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, kTB), int64_t(sm_count()) * 8)));
}

// One allgather of `count` doubles per rank (rank-major result).
void allgather(Context& c, const double* send, double* recv, int64_t count) {
  DistState& d = c.dist;
  if (d.kind == 2) {
    YS_NCCL(nccl().AllGather(send, recv, size_t(count), ncclDouble, reinterpret_cast<ncclComm_t>(d.nccl), c.stream));
    return;
  }
  d.hsend.resize(size_t(count));
  d.hrecv.resize(size_t(count) * d.nranks);
  YS_CUDA(cudaMemcpyAsync(d.hsend.data(), send, size_t(count) * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  YS_CUDA(cudaStreamSynchronize(c.stream));
  if (d.fn(d.user, d.hsend.data(), d.hrecv.data(), count) != 0)
    fail(YS_ERR_CUDA, "distributed solve: the host allgather callback failed");
  YS_CUDA(cudaMemcpyAsync(recv, d.hrecv.data(), size_t(count) * d.nranks * sizeof(double), cudaMemcpyHostToDevice,
                          c.stream));
}

// Partition + halo plan of the current structures (identical on every rank).
void build_plan(Context& c) {
  DistState& d = c.dist;
  const int n = d.nranks;
  cudaStream_t s = c.stream;
  const bool has1 = c.S[1].n_blocks > 0;
  d.dbounds.resize(size_t(n + 1));
  d.dexp_off.resize(size_t(n + 1));
  // the partition is the static one (ctx_dist_static_plan), fixed across
  // Newton iterations
  ctx_dist_static_plan(c);
  YS_CUDA(cudaMemcpyAsync(d.dbounds.p, d.sbounds.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  d.need.resize(size_t(c.NB));
  YS_CUDA(cudaMemsetAsync(d.need.p, 0, size_t(c.NB), s));
  for (int w = 0; w < (has1 ? 2 : 1); ++w) {
    const Structure& st = c.S[w];
    if (st.n_blocks == 0) continue;
    k_mark_need<<<blocks_for(st.n_blocks), kTB, 0, s>>>(st.row.p, st.col.p, st.n_blocks, d.dbounds.p, n, d.need.p);
    YS_LAUNCH_CHECK();
  }
  d.exp.resize(size_t(c.NB) + 1);
  d.nsel.resize(1);
  size_t tmp = 0;
  cub::CountingInputIterator<int32_t> it(0);
  YS_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, d.need.p, d.exp.p, d.nsel.p, int(c.NB), s));
  c.cubtmp.resize(std::max(c.cubtmp.n, tmp + 1));
  YS_CUDA(cub::DeviceSelect::Flagged(c.cubtmp.p, tmp, it, d.need.p, d.exp.p, d.nsel.p, int(c.NB), s));
  k_exp_offsets<<<1, kMaxRanks + 1, 0, s>>>(d.exp.p, d.nsel.p, d.dbounds.p, n, d.dexp_off.p);
  YS_LAUNCH_CHECK();
  d.bounds.assign(size_t(n + 1), 0);
  d.exp_off.assign(size_t(n + 1), 0);
  YS_CUDA(cudaMemcpyAsync(d.bounds.data(), d.dbounds.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaMemcpyAsync(d.exp_off.data(), d.dexp_off.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  d.max_exp = d.max_rows = 0;
  for (int k = 0; k < n; ++k) {
    d.max_exp = std::max(d.max_exp, d.exp_off[k + 1] - d.exp_off[k]);
    d.max_rows = std::max(d.max_rows, d.bounds[k + 1] - d.bounds[k]);
  }
}

// Unique block u (DoF coordinates row/col) touches rows [r0, r1).
__global__ void k_flag_owned_blocks(const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t u0,
                                    int64_t n, int64_t r0, int64_t r1, uint8_t* __restrict__ flag) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t R = row[u0 + t] / 3, C = col[u0 + t] / 3;
  flag[t] = ((R >= r0 && R < r1) || (C >= r0 && C < r1)) ? 1 : 0;
}

// Sort key of selected block k: (window of 4096 positions, run length).
__global__ void k_sel_run_keys(const int64_t* __restrict__ seg, const int32_t* __restrict__ sel, int64_t n,
                               uint32_t* __restrict__ key) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t u = sel[k];
  const int64_t len = seg[u + 1] - seg[u];
  key[k] = (uint32_t(k >> 12) << 10) | uint32_t(len < 1023 ? len : 1023);
}

// Instance i of a 4-vertex stencil energy touches rows [r0, r1) (uniform 3x3).
__global__ void k_flag_owned(const int4* __restrict__ conn, int64_t n, int32_t startP, int64_t r0, int64_t r1,
                             uint8_t* __restrict__ flag) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 v = conn[i];
  const int vv[4] = {v.x, v.y, v.z, v.w};
  bool t = false;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int64_t R = (int64_t(startP) + 3 * int64_t(vv[l])) / 3;
    t = t || (R >= r0 && R < r1);
  }
  flag[i] = t ? 1 : 0;
}
}  // namespace

// Partition from the static structure's entry counts (the same weights as the
// per-solve plan: entries per block row + 1), and per static SNH / bending
// energy the instances touching this rank's rows.  Computed once per context.
void ctx_dist_static_plan(Context& c) {
  DistState& d = c.dist;
  if (d.have_static) return;
  const int n = d.nranks;
  cudaStream_t s = c.stream;
  if (!(c.uniform3 && c.S[0].all33)) fail(YS_ERR_VALIDATION, "distributed PCG supports uniform 3x3 block systems only");
  d.dbounds.resize(size_t(n + 1));
  k_partition<<<1, kMaxRanks + 1, 0, s>>>(c.S[0].nrow.p, c.S[0].trow.p, nullptr, nullptr, c.NB, n, d.dbounds.p);
  YS_LAUNCH_CHECK();
  d.sbounds.assign(size_t(n + 1), 0);
  YS_CUDA(cudaMemcpyAsync(d.sbounds.data(), d.dbounds.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  const int64_t r0 = d.sbounds[d.rank], r1 = d.sbounds[d.rank + 1];
  d.sel.clear();
  d.sel.resize(c.energies.size());
  d.nsel_e.assign(c.energies.size(), -1);
  d.eval_owned = d.eval_total = 0;
  DevBuf<uint8_t> flag;
  DevBuf<int32_t> cnt;
  cnt.resize(1);
  for (size_t id = 0; id < c.energies.size(); ++id) {
    const Energy& e = c.energies[id];
    if (e.dynamic || !(e.kind == K_SNH || e.kind == K_BENDING) || e.n == 0) continue;
    flag.resize(size_t(e.n));
    const int32_t startP = e.target >= 0 ? int32_t(c.targets[e.target].start) : 0;
    k_flag_owned<<<blocks_for(e.n), kTB, 0, s>>>(reinterpret_cast<const int4*>(e.conn.p), e.n, startP, r0, r1, flag.p);
    YS_LAUNCH_CHECK();
    d.sel[id].resize(size_t(e.n) + 1);
    size_t tmp = 0;
    cub::CountingInputIterator<int32_t> it(0);
    YS_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag.p, d.sel[id].p, cnt.p, int(e.n), s));
    c.cubtmp.resize(std::max(c.cubtmp.n, tmp + 1));
    YS_CUDA(cub::DeviceSelect::Flagged(c.cubtmp.p, tmp, it, flag.p, d.sel[id].p, cnt.p, int(e.n), s));
    int32_t h = 0;
    YS_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaStreamSynchronize(s));
    d.nsel_e[id] = h;
    d.eval_owned += h;
    d.eval_total += e.n;
  }
  // the static group's unique blocks touching owned rows (the assembly gather
  // of this rank)
  const Structure& st0 = c.S[0];
  d.gsel.clear();
  d.gsel.resize(st0.groups.size());
  d.ngsel.assign(st0.groups.size(), 0);
  for (size_t gi = 0; gi < st0.groups.size(); ++gi) {
    const auto& g = st0.groups[gi];
    const int64_t u0 = g[2], gcnt = g[3];
    if (gcnt == 0) continue;
    flag.resize(size_t(gcnt));
    k_flag_owned_blocks<<<blocks_for(gcnt), kTB, 0, s>>>(st0.row.p, st0.col.p, u0, gcnt, r0, r1, flag.p);
    YS_LAUNCH_CHECK();
    d.gsel[gi].resize(size_t(gcnt) + 1);
    size_t tmp = 0;
    cub::CountingInputIterator<int32_t> it(static_cast<int32_t>(u0));
    YS_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag.p, d.gsel[gi].p, cnt.p, int(gcnt), s));
    c.cubtmp.resize(std::max(c.cubtmp.n, tmp + 1));
    YS_CUDA(cub::DeviceSelect::Flagged(c.cubtmp.p, tmp, it, flag.p, d.gsel[gi].p, cnt.p, int(gcnt), s));
    int32_t h = 0;
    YS_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaStreamSynchronize(s));
    d.ngsel[gi] = h;
    // the gather order of the single-GPU static gather: run length sorted inside
    // windows of 4096 selected blocks (bit-identical sums, warps of similar runs)
    if (h > 1) {
      DevBuf<uint32_t> kin, kout;
      DevBuf<int32_t> vout;
      kin.resize(size_t(h));
      kout.resize(size_t(h));
      vout.resize(size_t(h) + 1);
      k_sel_run_keys<<<blocks_for(h), kTB, 0, s>>>(st0.seg.p, d.gsel[gi].p, h, kin.p);
      YS_LAUNCH_CHECK();
      size_t bytes = 0;
      YS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin.p, kout.p, d.gsel[gi].p, vout.p, h, 0, 32, s));
      c.cubtmp.resize(std::max(c.cubtmp.n, bytes + 1));
      YS_CUDA(cub::DeviceRadixSort::SortPairs(c.cubtmp.p, bytes, kin.p, kout.p, d.gsel[gi].p, vout.p, h, 0, 32, s));
      YS_CUDA(cudaStreamSynchronize(s));
      std::swap(d.gsel[gi], vout);
    }
  }
  // instances outside the subset are never evaluated while the partition is
  // active: their contributions read as zero (non-owned rows are neither
  // solved nor checked)
  c.S[0].hcontrib.zero(s);
  c.S[0].gcontrib.zero(s);
  d.have_static = true;
}

void ctx_dist_unique_id(unsigned char* id) {
  ncclUniqueId u;
  YS_NCCL(nccl().GetUniqueId(&u));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, sizeof(u));
}

void ctx_dist_init_nccl(Context& c, int rank, int nranks, const unsigned char* id) {
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t comm = nullptr;
  YS_CUDA(cudaSetDevice(c.device));
  YS_NCCL(nccl().CommInitRank(&comm, nranks, u, rank));
  c.dist.nccl = comm;
  c.dist.kind = 2;
}

namespace {
void p2p_release(Context& c);
}

void ctx_dist_finalize(Context& c) {
  if (c.dist.kind == 2 && c.dist.nccl) nccl().CommDestroy(reinterpret_cast<ncclComm_t>(c.dist.nccl));
  p2p_release(c);
  c.dist.nccl = nullptr;
  c.dist.kind = 0;
  c.dist.have_static = false;  // a new rank count recomputes the partition
}

void ctx_dist_pcg(Context& c, double tol, int64_t max_iter, ys_step_stats* stats) {
  DistState& d = c.dist;
  if (d.kind == 3) {
    if (!d.p2p.group.empty())
      fail(YS_ERR_VALIDATION, "P2P group: step the emulated ranks together (ys_dist_p2p_group_step)");
    ctx_dist_p2p_solve({&c}, tol, max_iter, stats);
    return;
  }
  const int n = d.nranks, me = d.rank;
  if (n < 1 || n > kMaxRanks || me < 0 || me >= n) fail(YS_ERR_VALIDATION, "distributed solve: bad rank / size");
  const bool has1 = c.S[1].n_blocks > 0;
  if (!(c.uniform3 && c.S[0].all33 && (!has1 || c.S[1].all33)))
    fail(YS_ERR_VALIDATION, "distributed PCG supports uniform 3x3 block systems only");
  cudaStream_t s = c.stream;
  build_plan(c);
  const int64_t r0 = d.bounds[me], r1 = d.bounds[me + 1];
  const int64_t my_exp = d.exp_off[me + 1] - d.exp_off[me];
  const int64_t total_exp = d.exp_off[n];

  c.r.resize(c.s + 2);
  c.z.resize(c.s + 2);
  c.p.resize(c.s + 2);
  c.hp.resize(c.s + 2);
  c.pcg.resize(1);
  const int grid = std::max(1, sm_count() * 8);
  c.partials.resize(std::max<size_t>(c.partials.n, size_t(2 * grid)));
  const int64_t hist_cap = std::min<int64_t>(max_iter, int64_t(1) << 22) + 2;
  c.hist.resize(std::max<size_t>(c.hist.n, size_t(hist_cap)));
  const int64_t zp = 2 + 6 * d.max_exp;  // fused exchange record per rank
  d.send.resize(size_t(std::max(3 * std::max(d.max_exp, d.max_rows), zp) + 1));
  d.recv.resize(size_t(std::max(3 * std::max(d.max_exp, d.max_rows), zp) * n + 1));
  d.dsend.resize(2);
  d.dall.resize(size_t(2 * n));

  PcgState init{};
  init.tol = tol;
  init.max_iter = max_iter;
  init.hist_cap = int64_t(c.hist.n);
  YS_CUDA(cudaMemcpyAsync(c.pcg.p, &init, sizeof(PcgState), cudaMemcpyHostToDevice, s));
  PcgState* st = c.pcg.p;
  double* part = c.partials.p;
  const int vg = vgrid(r1 - r0);
  k_dinit<<<vg, kTB, 0, s>>>(c.G.p, c.minv.p, c.r.p, c.z.p, c.p.p, c.DX.p, r0, r1, st, part, d.dsend.p);
  YS_LAUNCH_CHECK();
  allgather(c, d.dsend.p, d.dall.p, 2);
  k_dinit_fin<<<1, 1, 0, s>>>(st, d.dall.p, n, c.hist.p);
  YS_LAUNCH_CHECK();

  // the owned rows' sliced-ELL copy
  sell_build(c, 4, r0, r1);
  SellDev sl = sell_dev(c);
  static int occ_sell = 0;
  if (!occ_sell) {
    YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sell, k_dspmv_sell, kTB, 0));
    occ_sell = std::max(occ_sell, 1);
  }
  const int sg = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(32 * sl.nslices, kTB),
                                                            int64_t(occ_sell) * sm_count())));
  // the initial p (= z) halo; afterwards it travels with the update's partials
  if (d.max_exp > 0) {
    k_pack<<<blocks_for(3 * my_exp), kTB, 0, s>>>(c.p.p, d.exp.p + d.exp_off[me], my_exp, d.send.p, st);
    allgather(c, d.send.p, d.recv.p, 3 * d.max_exp);
    k_unpack<<<blocks_for(3 * total_exp), kTB, 0, s>>>(d.recv.p, d.exp.p, d.dexp_off.p, n, me, d.max_exp, total_exp,
                                                       c.p.p, st);
    YS_LAUNCH_CHECK();
  }
  // Two allgathers per iteration: pHp partials; then the r.r / r.z partials
  // together with z and the pre-update p of the export rows (k_pack_zp /
  // k_unpack_zp: the receivers update their halo p themselves).
  auto iteration = [&] {
    k_dspmv_sell<<<sg, kTB, 0, s>>>(sl, c.p.p, c.hp.p, st, part, d.dsend.p);
    allgather(c, d.dsend.p, d.dall.p, 1);
    k_dalpha<<<1, 1, 0, s>>>(st, d.dall.p, n);
    k_dupdate<<<vg, kTB, 0, s>>>(c.minv.p, c.DX.p, c.r.p, c.z.p, c.p.p, c.hp.p, r0, r1, st, part, d.send.p);
    if (d.max_exp > 0)
      k_pack_zp<<<blocks_for(3 * my_exp), kTB, 0, s>>>(c.z.p, c.p.p, d.exp.p + d.exp_off[me], my_exp, d.max_exp,
                                                        d.send.p, st);
    allgather(c, d.send.p, d.recv.p, zp);
    k_dbeta<<<1, 1, 0, s>>>(st, d.recv.p, n, c.hist.p, zp);
    k_dpupdate<<<vg, kTB, 0, s>>>(c.z.p, c.p.p, r0, r1, st);
    if (d.max_exp > 0)
      k_unpack_zp<<<blocks_for(3 * total_exp), kTB, 0, s>>>(d.recv.p, d.exp.p, d.dexp_off.p, n, me, d.max_exp,
                                                             total_exp, c.p.p, st);
    YS_LAUNCH_CHECK();
    c.launches += 6 + (d.max_exp > 0 ? 2 : 0);
  };
  // Status is identical on every rank, so every rank leaves after the same chunk.
  const int chunk = d.kind == 2 ? 8 : 1;
  PcgState fin{};
  for (;;) {
    YS_CUDA(cudaMemcpyAsync(&fin, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaStreamSynchronize(s));
    if (fin.status) break;
    for (int k = 0; k < chunk; ++k) iteration();
  }
  // every rank returns the full step
  if (n > 1) {
    k_copy_rows<<<blocks_for(3 * (r1 - r0)), kTB, 0, s>>>(c.DX.p, r0, r1, d.send.p);
    allgather(c, d.send.p, d.recv.p, 3 * d.max_rows);
    k_gather_rows<<<blocks_for(3 * c.NB), kTB, 0, s>>>(d.recv.p, d.dbounds.p, n, d.max_rows, c.NB, c.DX.p);
    YS_LAUNCH_CHECK();
  }
  c.hist_count = fin.status == 1 && fin.it == 0 && fin.gnorm == 0.0 ? 0 : fin.it + 1;
  if (fin.status == 3)
    fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) +
                               " (non-finite or negative curvature)");
  if (fin.status == 4)
    fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) + " (non-finite residual)");
  if (stats) {
    stats->pcg_iterations = fin.it;
    stats->pcg_converged = fin.status == 1 ? 1 : 0;
    stats->pcg_residual = (fin.gnorm == 0.0) ? 0.0 : fin.rel;
  }
}

// ---------------------------------------------------------------------------
// Peer-memory row-partitioned PCG (transport kind 3).
//
// One persistent cooperative kernel per rank runs the whole solve, the same
// recurrence and phases as k_pcg33_stream over the sliced-ELL copy of the
// owned rows.  Nothing is gathered: a rank only STORES into its peers'
// windows (NVLink P2P through cudaIpc-mapped pointers) —
//   * in the update phase, the z of every owned row that a peer needs (bit k
//     of mask[R]: a block couples row R with a row of rank k) straight into
//     that peer's z; the peer forms its halo p = z + beta p itself (the
//     owner's formula and operands, so bitwise the owner's p: p needs no
//     exchange of its own);
//   * after each rank-local reduction, the rank's partial sums (pHp; r.r and
//     r.z) into every peer's value slots, then a release store of the
//     exchange's sequence number into the peer's flag (`st.release.sys`);
//   * at the end, the owned rows of the step into every peer's step buffer.
// Every CTA acquire-polls the N flags in its own window and sums the N rank
// values in rank order, so alpha / beta / status are identical on every rank
// and every rank leaves the loop on the same iteration.  Per iteration: two
// cross-rank exchanges (~1-2 us of NVLink latency each) plus the rank-local
// grid barriers — instead of two NCCL allgathers with host-side chunking.
//
// A slot is reused by the next exchange of its kind only after every rank
// has consumed it: a rank sends exchange e+1 of a kind only after receiving
// the other kind's exchange from all ranks, which each of them sends after
// its CTAs read exchange e.
//
// One GPU cannot run several such kernels as separate processes (they spin
// on each other's flags and are not guaranteed to be co-resident), so the
// same kernel also runs N ranks' views as ONE cooperative launch on one
// device (ys_dist_p2p_group: every rank's data in its own context, the peers'
// windows are plain device pointers) — the test and profiling path here.

struct P2PHead {
  unsigned long long flag[3][kMaxP2P];  // [exchange kind: A pHp | B r.r, r.z | X step rows][sender]
  double val[2][kMaxP2P][2];            // [A | B][sender][value]
  unsigned long long probe[kMaxP2P];
};
constexpr size_t kP2PHead = 1024;  // window bytes ahead of z
static_assert(sizeof(P2PHead) <= kP2PHead, "P2P window head");

struct P2PView {
  SellPhaseA A;
  int64_t r0, r1;
  const double* g;
  const double* minv;
  double *r, *p, *hp;  // rank-local vectors (global DoF indexing)
  double *z, *x;       // in this rank's window
  P2PHead* head;
  P2PHead* phead[kMaxP2P];
  double* pz[kMaxP2P];
  double* px[kMaxP2P];
  const uint32_t* mask;
  const int32_t* halo;
  int64_t nhalo;
  double* part;
  unsigned long long* bar;
  PcgState* st;
  double* hist;
  int rank, n;
  unsigned long long seq0;
};

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* a) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(a) : "memory");
  return v;
}

// A peer that never answers (a dead rank) must not hang the device forever.
__device__ __forceinline__ void p2p_wait_flag(const unsigned long long* f, unsigned long long seq, int from) {
  const unsigned long long t0 = gtimer();
  while (ld_acquire_sys(f) < seq) {
    __nanosleep(32);
    if (gtimer() - t0 > 60ull * 1000000000ull) {
      printf("yasps_b200: P2P solve: no exchange %llu from rank %d within 60 s\n", seq, from);
      __trap();
    }
  }
}

// The rank's K partial sums (identical in every CTA) -> every peer; the
// rank-ordered sum of all ranks' values.  Thread j of a CTA serves peer j, so
// the release stores (CTA 0 only) and the acquire polls of the n - 1 peers
// overlap instead of paying n - 1 system-scope round trips in a row.
template <int K>
__device__ __forceinline__ void p2p_exchange(const P2PView& V, int kind, int cb, const double (&mine)[K],
                                             unsigned long long seq, double (&tot)[K]) {
  __shared__ double sv[kMaxP2P][2];
  const int j = threadIdx.x;
  if (j < V.n) {
    if (j == V.rank) {
#pragma unroll
      for (int k = 0; k < K; ++k) sv[j][k] = mine[k];
    } else {
      if (cb == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) V.phead[j]->val[kind][V.rank][k] = mine[k];
        st_release_sys(&V.phead[j]->flag[kind][V.rank], seq);
      }
      p2p_wait_flag(&V.head->flag[kind][j], seq, j);
#pragma unroll
      for (int k = 0; k < K; ++k) sv[j][k] = ld_relaxed_sys(&V.head->val[kind][j][k]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    tot[k] = 0.0;
    for (int q = 0; q < V.n; ++q) tot[k] += sv[q][k];
  }
  __syncthreads();
}

// Flag-only exchange (the step rows are in place).
__device__ __forceinline__ void p2p_signal(const P2PView& V, int kind, int cb, unsigned long long seq) {
  const int j = threadIdx.x;
  if (j < V.n && j != V.rank) {
    if (cb == 0) st_release_sys(&V.phead[j]->flag[kind][V.rank], seq);
    p2p_wait_flag(&V.head->flag[kind][j], seq, j);
  }
  __syncthreads();
}

// z of owned row b -> every peer that needs it.
__device__ __forceinline__ bool p2p_send_z(const P2PView& V, int64_t b, const double* zz) {
  uint32_t m = V.mask[b] & ~(1u << V.rank);
  if (!m) return false;
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    double* d = V.pz[j] + 3 * b;
    d[0] = zz[0];
    d[1] = zz[1];
    d[2] = zz[2];
  }
  return true;
}

__device__ __forceinline__ void rank_barrier(const P2PView& V, int G, unsigned long long& epoch) {
  grid_arrive(V.bar);
  grid_wait(V.bar, (unsigned long long)G * ++epoch);
}

}  // namespace

// Grid = (views) x G CTAs; CTA b runs rank view b / G as its CTA b % G.
__global__ void __launch_bounds__(kTB, kSpmvMinB) k_dpcg_p2p(const P2PView* __restrict__ views, int G) {
  extern __shared__ double smem[];
  const int cb = int(blockIdx.x) % G;
  const P2PView& V = views[blockIdx.x / G];
  SellPhaseA A = V.A;
  A.prologue(smem, cb, G);
  const uint64_t kpol = l2_keep_policy();
  const int64_t nth = int64_t(G) * blockDim.x;
  const int64_t t0 = int64_t(cb) * blockDim.x + threadIdx.x;
  PcgState* st = V.st;
  const double tol = st->tol;
  const long long max_iter = st->max_iter;
  const long long hist_cap = st->hist_cap;
  unsigned long long epoch = 0, seq = V.seq0;
  // ---- r = g, z = M^-1 r, p = z, x = 0 on the owned rows (pcg, solver.cpp:151-162)
  double v2[2] = {0.0, 0.0};
  bool remote = false;
  for (int64_t b = V.r0 + t0; b < V.r1; b += nth) {
    double rr[3], zz[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rr[i] = V.g[3 * b + i];
      V.r[3 * b + i] = rr[i];
      V.x[3 * b + i] = 0.0;
    }
    precond_apply<3>(V.minv + 9 * b, rr, zz);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      V.z[3 * b + i] = zz[i];
      V.p[3 * b + i] = zz[i];
      v2[0] += rr[i] * rr[i];
      v2[1] += rr[i] * zz[i];
    }
    remote |= p2p_send_z(V, b, zz);
  }
  if (remote) __threadfence_system();
  block_reduce<2>(v2);
  if (threadIdx.x == 0) {
    V.part[G + cb] = v2[0];
    V.part[2 * G + cb] = v2[1];
  }
  rank_barrier(V, G, epoch);
  double mine2[2], tot2[2];
  reduce_partials_all<2>(V.part + G, G, mine2);
  p2p_exchange<2>(V, 1, cb, mine2, ++seq, tot2);
  const double gnorm = sqrt(tot2[0]);
  double rz = tot2[1], rel = 0.0, php = 0.0, alpha = 0.0;
  int status;
  if (gnorm == 0.0) {
    status = 1;  // converged with x = 0 (solver.cpp:156-159)
  } else {
    status = max_iter > 0 ? 0 : 5;
    rel = 1.0;
    if (cb == 0 && threadIdx.x == 0) V.hist[0] = 1.0;
  }
  for (int64_t h = t0; h < V.nhalo; h += nth) {
    const int64_t b = V.halo[h];
#pragma unroll
    for (int i = 0; i < 3; ++i) V.p[3 * b + i] = __ldcg(V.z + 3 * b + i);
  }
  rank_barrier(V, G, epoch);
  long long it = 0;
  unsigned long long ph[4] = {0, 0, 0, 0};  // A + exchange, B + exchange, (unused), C + barrier
  unsigned long long tc = gtimer();
  while (status == 0) {
    // ---- hp = H p on the owned rows, pHp
    double dot[1] = {A.run(V.p, V.hp)};
    block_reduce<1>(dot);
    if (threadIdx.x == 0) V.part[cb] = dot[0];
    rank_barrier(V, G, epoch);
    double m1[1], t1[1];
    reduce_partials_all<1>(V.part, G, m1);
    p2p_exchange<1>(V, 0, cb, m1, ++seq, t1);
    unsigned long long tn = gtimer();
    ph[0] += tn - tc;
    tc = tn;
    php = t1[0];
    if (!isfinite(php) || php <= 0.0) {
      status = php == 0.0 ? 2 : 3;
      break;
    }
    alpha = rz / php;
    // ---- x += a p, r -= a hp, z = M^-1 r; the peers' z rows; r.r, r.z
    double v[2] = {0.0, 0.0};
    remote = false;
    for (int64_t b = V.r0 + t0; b < V.r1; b += nth) {
      RowRegs q;
      rowregs_load(q, b, V.p, V.r, V.x, V.minv, kpol);
      rowregs_update(q, b, alpha, V.hp, V.x, V.r, v, kpol);
#pragma unroll
      for (int i = 0; i < 3; ++i) st_keep(V.z + 3 * b + i, q.z[i], kpol);
      remote |= p2p_send_z(V, b, q.z);
    }
    if (remote) __threadfence_system();
    block_reduce<2>(v);
    if (threadIdx.x == 0) {
      V.part[G + cb] = v[0];
      V.part[2 * G + cb] = v[1];
    }
    rank_barrier(V, G, epoch);
    reduce_partials_all<2>(V.part + G, G, mine2);
    p2p_exchange<2>(V, 1, cb, mine2, ++seq, tot2);
    tn = gtimer();
    ph[1] += tn - tc;
    tc = tn;
    rel = sqrt(tot2[0]) / gnorm;
    if (cb == 0 && threadIdx.x == 0 && it + 1 < hist_cap) V.hist[it + 1] = rel;
    ++it;
    if (!isfinite(rel)) {
      status = 4;
      break;
    }
    if (rel <= tol) {
      status = 1;
      break;
    }
    if (it >= max_iter) {
      status = 5;
      break;
    }
    const double beta = tot2[1] / rz;
    rz = tot2[1];
    // ---- p = z + beta p on the owned rows and the halo rows
    for (int64_t b = V.r0 + t0; b < V.r1; b += nth) {
      double zz[3], pp[3];
      load_vec3_keep(V.z + 3 * b, zz[0], zz[1], zz[2], kpol);
      load_vec3_keep(V.p + 3 * b, pp[0], pp[1], pp[2], kpol);
#pragma unroll
      for (int i = 0; i < 3; ++i) st_keep(V.p + 3 * b + i, zz[i] + beta * pp[i], kpol);
    }
    for (int64_t h = t0; h < V.nhalo; h += nth) {
      const int64_t b = V.halo[h];
      double zz[3], pp[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        zz[i] = __ldcg(V.z + 3 * b + i);
        pp[i] = V.p[3 * b + i];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) V.p[3 * b + i] = zz[i] + beta * pp[i];
    }
    rank_barrier(V, G, epoch);
    tn = gtimer();
    ph[3] += tn - tc;
    tc = tn;
  }
  // ---- every rank returns the full step: owned rows -> every peer
  if (V.n > 1) {
    for (int64_t b = V.r0 + t0; b < V.r1; b += nth)
      for (int j = 0; j < V.n; ++j) {
        if (j == V.rank) continue;
#pragma unroll
        for (int i = 0; i < 3; ++i) V.px[j][3 * b + i] = V.x[3 * b + i];
      }
    __threadfence_system();
    rank_barrier(V, G, epoch);
    p2p_signal(V, 2, cb, ++seq);
  }
  if (cb == 0 && threadIdx.x == 0) {
    st->gnorm = gnorm;
    st->it = it;
    st->rel = rel;
    st->rz = rz;
    st->php = php;
    st->alpha = alpha;
    st->status = status;
    if (status == 3 || status == 4) st->fail_it = int(it - (status == 4 ? 1 : 0));
    for (int k = 0; k < 4; ++k) st->phase_ns[k] = ph[k];
  }
}

__global__ void k_p2p_probe(P2PHead* mine, P2PView V, int phase, long long* seen) {
  if (phase == 0) {
    for (int j = 0; j < V.n; ++j)
      if (j != V.rank) st_release_sys(&V.phead[j]->probe[V.rank], (unsigned long long)(V.rank + 1));
  } else {
    for (int j = 0; j < V.n; ++j) seen[j] = (long long)ld_acquire_sys(&mine->probe[j]);
  }
}

namespace {

// Block (R, C) across ranks: row R's z goes to owner(C), row C's to owner(R).
__global__ void k_p2p_mask(const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t nblocks,
                           const int64_t* __restrict__ bounds, int n, uint32_t* mask) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nblocks) return;
  const int64_t R = row[u] / 3, C = col[u] / 3;
  if (R == C) return;
  const int oR = owner_of(bounds, n, R), oC = owner_of(bounds, n, C);
  if (oR == oC) return;
  atomicOr(mask + R, 1u << oC);
  atomicOr(mask + C, 1u << oR);
}

__global__ void k_p2p_halo_flag(const uint32_t* __restrict__ mask, int64_t nb, int64_t r0, int64_t r1, int me,
                                uint8_t* flag) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R >= nb) return;
  flag[R] = (R < r0 || R >= r1) && ((mask[R] >> me) & 1u) ? 1 : 0;
}

size_t p2p_window_bytes(int64_t s) {
  const size_t vec = (size_t(s + 2) * sizeof(double) + 255) / 256 * 256;
  return kP2PHead + 2 * vec;
}
double* p2p_z(void* w) { return reinterpret_cast<double*>(static_cast<char*>(w) + kP2PHead); }
double* p2p_x(void* w, int64_t s) {
  return reinterpret_cast<double*>(static_cast<char*>(w) + kP2PHead + (size_t(s + 2) * sizeof(double) + 255) / 256 * 256);
}

void p2p_release(Context& c) {
  P2PState& q = c.dist.p2p;
  for (int j = 0; j < kMaxP2P; ++j) {
    if (q.ipc[j] && q.peer[j]) cudaIpcCloseMemHandle(q.peer[j]);
    q.peer[j] = nullptr;
    q.ipc[j] = false;
  }
  if (q.win) cudaFree(q.win);
  q.win = nullptr;
  q.win_bytes = 0;
  q.group.clear();
}

// Destination masks and this rank's halo list for the current structures.
void p2p_plan(Context& c) {
  DistState& d = c.dist;
  P2PState& q = d.p2p;
  cudaStream_t s = c.stream;
  build_plan(c);  // bounds (+ the export lists dist_info reports)
  q.mask.resize(size_t(c.NB) + 1);
  YS_CUDA(cudaMemsetAsync(q.mask.p, 0, sizeof(uint32_t) * size_t(c.NB), s));
  for (int w = 0; w < 2; ++w) {
    const Structure& st = c.S[w];
    if (st.n_blocks == 0) continue;
    k_p2p_mask<<<blocks_for(st.n_blocks), kTB, 0, s>>>(st.row.p, st.col.p, st.n_blocks, d.dbounds.p, d.nranks,
                                                       q.mask.p);
    YS_LAUNCH_CHECK();
  }
  const int64_t r0 = d.bounds[d.rank], r1 = d.bounds[d.rank + 1];
  q.hflag.resize(size_t(c.NB) + 1);
  k_p2p_halo_flag<<<blocks_for(c.NB), kTB, 0, s>>>(q.mask.p, c.NB, r0, r1, d.rank, q.hflag.p);
  YS_LAUNCH_CHECK();
  q.halo.resize(size_t(c.NB) + 1);
  q.nhalo.resize(1);
  size_t tmp = 0;
  cub::CountingInputIterator<int32_t> it(0);
  YS_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, q.hflag.p, q.halo.p, q.nhalo.p, int(c.NB), s));
  c.cubtmp.resize(std::max(c.cubtmp.n, tmp + 1));
  YS_CUDA(cub::DeviceSelect::Flagged(c.cubtmp.p, tmp, it, q.hflag.p, q.halo.p, q.nhalo.p, int(c.NB), s));
  int32_t h = 0;
  YS_CUDA(cudaMemcpyAsync(&h, q.nhalo.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  q.nhalo_host = h;
}

P2PView p2p_view(Context& c) {
  DistState& d = c.dist;
  P2PState& q = d.p2p;
  P2PView V{};
  V.r0 = d.bounds[d.rank];
  V.r1 = d.bounds[d.rank + 1];
  V.g = c.G.p;
  V.minv = c.minv.p;
  V.r = c.r.p;
  V.p = c.p.p;
  V.hp = c.hp.p;
  V.z = p2p_z(q.win);
  V.x = p2p_x(q.win, c.s);
  V.head = reinterpret_cast<P2PHead*>(q.win);
  for (int j = 0; j < d.nranks; ++j) {
    if (j == d.rank) continue;
    V.phead[j] = reinterpret_cast<P2PHead*>(q.peer[j]);
    V.pz[j] = p2p_z(q.peer[j]);
    V.px[j] = p2p_x(q.peer[j], c.s);
  }
  V.mask = q.mask.p;
  V.halo = q.halo.p;
  V.nhalo = q.nhalo_host;
  V.bar = q.bar.p;
  V.st = c.pcg.p;
  V.hist = c.hist.p;
  V.rank = d.rank;
  V.n = d.nranks;
  V.seq0 = q.solve_id << 32;
  return V;
}

}  // namespace

void ctx_dist_p2p_open(Context& c, int rank, int nranks, unsigned char* handle) {
  if (nranks < 1 || nranks > kMaxP2P || rank < 0 || rank >= nranks)
    fail(YS_ERR_VALIDATION, "P2P solve: rank " + std::to_string(rank) + " of " + std::to_string(nranks) +
                                " is out of range (1.." + std::to_string(kMaxP2P) + " ranks)");
  if (!c.finalized) fail(YS_ERR_VALIDATION, "P2P solve: finalize the scene before opening the window");
  ctx_dist_finalize(c);
  DistState& d = c.dist;
  P2PState& q = d.p2p;
  YS_CUDA(cudaSetDevice(c.device));
  q.win_bytes = p2p_window_bytes(c.s);
  q.win_s = c.s;
  void* w = nullptr;
  YS_CUDA(cudaMalloc(&w, q.win_bytes));
  q.win = static_cast<char*>(w);
  YS_CUDA(cudaMemset(q.win, 0, q.win_bytes));
  q.peer[rank] = q.win;
  if (handle) {
    cudaIpcMemHandle_t h;
    YS_CUDA(cudaIpcGetMemHandle(&h, q.win));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, sizeof(h));
  }
  d.rank = rank;
  d.nranks = nranks;
  d.kind = 3;
}

void ctx_dist_p2p_connect(Context& c, const unsigned char* handles) {
  DistState& d = c.dist;
  P2PState& q = d.p2p;
  if (d.kind != 3 || !q.win) fail(YS_ERR_VALIDATION, "P2P solve: open the window before connecting");
  for (int j = 0; j < d.nranks; ++j) {
    if (j == d.rank || q.peer[j]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * size_t(j), sizeof(h));
    void* ptr = nullptr;
    YS_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    q.peer[j] = ptr;
    q.ipc[j] = true;
  }
}

void ctx_dist_p2p_group(const std::vector<Context*>& cs) {
  const int n = int(cs.size());
  for (int k = 0; k < n; ++k) {
    if (cs[k]->device != cs[0]->device) fail(YS_ERR_VALIDATION, "P2P group: every rank must be on one device");
    if (cs[k]->s != cs[0]->s) fail(YS_ERR_VALIDATION, "P2P group: ranks hold different scenes");
    ctx_dist_p2p_open(*cs[k], k, n, nullptr);
  }
  for (int k = 0; k < n; ++k) {
    for (int j = 0; j < n; ++j) cs[k]->dist.p2p.peer[j] = cs[j]->dist.p2p.win;
    cs[k]->dist.p2p.group = cs;
  }
}

void ctx_dist_p2p_probe(Context& c, int64_t* seen) {
  DistState& d = c.dist;
  if (d.kind != 3) fail(YS_ERR_VALIDATION, "P2P probe: no window");
  P2PView V{};
  V.rank = d.rank;
  V.n = d.nranks;
  for (int j = 0; j < d.nranks; ++j) V.phead[j] = reinterpret_cast<P2PHead*>(d.p2p.peer[j]);
  P2PHead* mine = reinterpret_cast<P2PHead*>(d.p2p.win);
  if (!seen) {
    k_p2p_probe<<<1, 1, 0, c.stream>>>(mine, V, 0, nullptr);
    YS_LAUNCH_CHECK();
    YS_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  DevBuf<long long> dv;
  dv.resize(kMaxP2P);
  k_p2p_probe<<<1, 1, 0, c.stream>>>(mine, V, 1, dv.p);
  YS_LAUNCH_CHECK();
  std::vector<long long> h(kMaxP2P);
  YS_CUDA(cudaMemcpyAsync(h.data(), dv.p, sizeof(long long) * kMaxP2P, cudaMemcpyDeviceToHost, c.stream));
  YS_CUDA(cudaStreamSynchronize(c.stream));
  for (int j = 0; j < d.nranks; ++j) seen[j] = h[size_t(j)];
}

// One cooperative launch over the views of cs (one context per rank in this
// process: the whole job of an emulated group, or this rank alone).
void ctx_dist_p2p_solve(const std::vector<Context*>& cs, double tol, int64_t max_iter, ys_step_stats* stats) {
  const int nv = int(cs.size());
  Context& c0 = *cs[0];
  std::vector<P2PView> views(static_cast<size_t>(nv));
  for (int v = 0; v < nv; ++v) {
    Context& c = *cs[v];
    DistState& d = c.dist;
    if (d.kind != 3 || !d.p2p.win) fail(YS_ERR_VALIDATION, "P2P solve: no window");
    for (int j = 0; j < d.nranks; ++j)
      if (!d.p2p.peer[j]) fail(YS_ERR_VALIDATION, "P2P solve: rank " + std::to_string(j) + " is not connected");
    if (c.s != d.p2p.win_s) fail(YS_ERR_VALIDATION, "P2P solve: the window was sized for another scene");
    const bool has1 = c.S[1].n_blocks > 0;
    if (!(c.uniform3 && c.S[0].all33 && (!has1 || c.S[1].all33)))
      fail(YS_ERR_VALIDATION, "distributed PCG supports uniform 3x3 block systems only");
    p2p_plan(c);
    c.r.resize(c.s + 2);
    c.p.resize(c.s + 2);
    c.hp.resize(c.s + 2);
    c.pcg.resize(1);
    const int64_t hist_cap = std::min<int64_t>(max_iter, int64_t(1) << 22) + 2;
    c.hist.resize(std::max<size_t>(c.hist.n, size_t(hist_cap)));
    PcgState init{};
    init.tol = tol;
    init.max_iter = max_iter;
    init.hist_cap = int64_t(c.hist.n);
    YS_CUDA(cudaMemcpyAsync(c.pcg.p, &init, sizeof(PcgState), cudaMemcpyHostToDevice, c.stream));
    sell_build(c, 4, d.bounds[d.rank], d.bounds[d.rank + 1]);
    d.p2p.bar.resize(1);
    YS_CUDA(cudaMemsetAsync(d.p2p.bar.p, 0, sizeof(unsigned long long), c.stream));
    ++d.p2p.solve_id;
    YS_CUDA(cudaStreamSynchronize(c.stream));
  }
  // CTAs per rank: the single-GPU solve's occupancy, shared by the views
  void* kern = reinterpret_cast<void*>(k_dpcg_p2p);
  const int wpb = kTB / 32;
  int G = 0;
  size_t smem = 0;
  for (int per = kSpmvMinB; per >= 1 && !G; --per) {
    const int g = std::max(1, per * sm_count() / nv);
    size_t need = 0;
    for (int v = 0; v < nv; ++v) {
      Context& c = *cs[v];
      const int K = int(ceil_div(std::max<int64_t>(c.sell_slices, 1), int64_t(g) * wpb));
      const int TW = c.sell_slices ? sell_max_warp_rows(c, int64_t(g) * wpb, K) : 0;
      need = std::max(need, size_t(wpb) * K * 8 + size_t(wpb) * K * 32 * 4 + size_t(wpb) * TW * 32 * 4);
      views[size_t(v)] = p2p_view(c);
      views[size_t(v)].A.SL = sell_dev(c);
      views[size_t(v)].A.nb = c.NB;
      views[size_t(v)].A.K = K;
      views[size_t(v)].A.TW = TW;
    }
    if (need > size_t(220 * 1024) / per) continue;
    YS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(need)));
    int occ = 0;
    YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTB, need));
    if (int64_t(occ) * sm_count() < int64_t(g) * nv) continue;
    G = g;
    smem = need;
  }
  if (!G) fail(YS_ERR_VALIDATION, "P2P solve: the per-warp SpMV plan does not fit in shared memory");
  for (int v = 0; v < nv; ++v) {
    Context& c = *cs[v];
    c.partials.resize(std::max<size_t>(c.partials.n, size_t(3 * G)));
    views[size_t(v)].part = c.partials.p;
    c.dist.p2p.sm_share = G;
  }
  DevBuf<P2PView> dviews;
  dviews.resize(size_t(nv));
  YS_CUDA(cudaMemcpyAsync(dviews.p, views.data(), sizeof(P2PView) * size_t(nv), cudaMemcpyHostToDevice, c0.stream));
  const P2PView* vp = dviews.p;
  void* args[] = {&vp, &G};
  if (c0.profiling) YS_CUDA(cudaEventRecord(c0.ev[7], c0.stream));
  YS_CUDA(cudaLaunchCooperativeKernel(kern, dim3(unsigned(G) * unsigned(nv)), dim3(kTB), args, smem, c0.stream));
  if (c0.profiling) YS_CUDA(cudaEventRecord(c0.ev[8], c0.stream));
  YS_CUDA(cudaStreamSynchronize(c0.stream));
  float kms = 0.f;
  if (c0.profiling) YS_CUDA(cudaEventElapsedTime(&kms, c0.ev[7], c0.ev[8]));
  for (int v = 0; v < nv; ++v) {
    Context& c = *cs[v];
    PcgState fin{};
    YS_CUDA(cudaMemcpyAsync(&fin, c.pcg.p, sizeof(PcgState), cudaMemcpyDeviceToHost, c.stream));
    YS_CUDA(cudaMemcpyAsync(c.DX.p, p2p_x(c.dist.p2p.win, c.s), sizeof(double) * size_t(c.s),
                            cudaMemcpyDeviceToDevice, c.stream));
    YS_CUDA(cudaStreamSynchronize(c.stream));
    c.launches += 2;
    c.pcg_path = 3;
    c.stage_ms[7] = kms;
    for (int k = 0; k < 4; ++k) c.pcg_phase_ms[k] = double(fin.phase_ns[k]) * 1e-6;
    c.hist_count = fin.status == 1 && fin.it == 0 && fin.gnorm == 0.0 ? 0 : fin.it + 1;
    if (fin.status == 3)
      fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) +
                                 " (non-finite or negative curvature)");
    if (fin.status == 4)
      fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) + " (non-finite residual)");
    if (stats) {
      stats[v].pcg_iterations = fin.it;
      stats[v].pcg_converged = fin.status == 1 ? 1 : 0;
      stats[v].pcg_residual = (fin.gnorm == 0.0) ? 0.0 : fin.rel;
    }
  }
}

}  // namespace ys
