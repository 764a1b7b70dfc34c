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
// p_R).  The transport is a single allgather primitive: ncclAllGather on the
// context stream (libnccl.so.2 dlopen-ed), or a host callback (tests).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <string>

#include <cub/cub.cuh>

#include "ys_sell.cuh"

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

void ctx_dist_finalize(Context& c) {
  if (c.dist.kind == 2 && c.dist.nccl) nccl().CommDestroy(reinterpret_cast<ncclComm_t>(c.dist.nccl));
  c.dist.nccl = nullptr;
  c.dist.kind = 0;
  c.dist.have_static = false;  // a new rank count recomputes the partition
}

void ctx_dist_pcg(Context& c, double tol, int64_t max_iter, ys_step_stats* stats) {
  DistState& d = c.dist;
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

}  // namespace ys
