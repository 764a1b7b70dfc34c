// ys_stencil.cu — contact candidates of the point-triangle, edge-edge and
// point-edge barriers (NOT IN THE REFERENCE; its candidates are point-point
// only, sim.cpp:456-484), including self-contact.
//
// Specification (restated by the oracle's all-pairs loop, oracle/yo_oracle.c
// yo_refresh_stencils, and identical bit for bit):
//   PT: points a x triangles b;  PE: points a x edges b;  EE: edges a x edges
//   b > a (one list: self-contact).  A candidate is kept when no point is
//   shared (incident primitives), not every point is fixed, and the squared
//   distance of its IPC distance type (ys_contact4.cuh, explicitly rounded) is
//   strictly below dhat.  Stencils are emitted in (a, b) order as union
//   indices: (p, t0, t1, t2), (a0, a1, b0, b1), (p, e0, e1).
//
// Device algorithm: a uniform grid with cell edge h = max(sqrt(dhat), largest
// B extent) (each B primitive overlaps at most 2 cells per axis); every
// (B primitive, overlapped cell) entry sorted by cell key (stable: b ascending
// inside a cell); each A primitive scans the cells of its box grown by
// sqrt(dhat) and takes a candidate only in the first cell common to both
// boxes (no duplicates), then the exact test; its hits are sorted by b.  The
// candidate set is a superset of the qualifying pairs and the test is the
// oracle's, so the lists are identical.
#include <algorithm>
#include <cmath>
#include <string>

#include <cub/cub.cuh>

#include "ys_contact4.cuh"

namespace ys {

void ctx_domain_points(Context& c, int domain, double* out);

namespace {
constexpr int kTB = 256;
inline unsigned grid_for(int64_t n, int tb = kTB) { return unsigned(std::max<int64_t>(1, ceil_div(n, tb))); }

struct Prims {
  const int32_t* a;  // n_a x arity_a union indices
  const int32_t* b;  // n_b x arity_b
  int64_t na, nb;
  int aa, ab;
  int kind;  // K_PT, K_EE, K_PE
  bool self;
};

__device__ __forceinline__ void prim_box(const double* pos, const int32_t* p, int ar, double lo[3], double hi[3]) {
  for (int k = 0; k < 3; ++k) {
    lo[k] = INFINITY;
    hi[k] = -INFINITY;
  }
  for (int l = 0; l < ar; ++l)
    for (int k = 0; k < 3; ++k) {
      const double v = pos[3 * int64_t(p[l]) + k];
      lo[k] = fmin(lo[k], v);
      hi[k] = fmax(hi[k], v);
    }
}

// largest B extent (max over primitives and axes) and the scene box
__global__ void k_prim_extent(const double* pos, Prims P, double* out /* 7: extent, lo[3], hi[3] */) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= P.nb) return;
  double lo[3], hi[3];
  prim_box(pos, P.b + P.ab * j, P.ab, lo, hi);
  double e = 0.0;
  for (int k = 0; k < 3; ++k) e = fmax(e, hi[k] - lo[k]);
  // doubles >= 0 order like their bit patterns: integer atomics
  atomicMax(reinterpret_cast<unsigned long long*>(out), __double_as_longlong(e));
}

struct Grid {
  double inv_h, o[3];  // cell(x) = floor((x - o) / h)
  int64_t dim[3];
};

__device__ __forceinline__ int64_t cellc(const Grid& g, int k, double x) {
  int64_t c = int64_t(floor((x - g.o[k]) * g.inv_h));
  return c < 0 ? 0 : (c >= g.dim[k] ? g.dim[k] - 1 : c);
}
__device__ __forceinline__ uint64_t ckey(const Grid& g, int64_t x, int64_t y, int64_t z) {
  return (uint64_t(x) * uint64_t(g.dim[1]) + uint64_t(y)) * uint64_t(g.dim[2]) + uint64_t(z);
}

__global__ void k_b_count(const double* pos, Prims P, Grid g, int32_t* cnt) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j > P.nb) return;
  if (j == P.nb) {
    cnt[j] = 0;
    return;
  }
  double lo[3], hi[3];
  prim_box(pos, P.b + P.ab * j, P.ab, lo, hi);
  int64_t n = 1;
  for (int k = 0; k < 3; ++k) n *= cellc(g, k, hi[k]) - cellc(g, k, lo[k]) + 1;
  cnt[j] = int32_t(n);
}

__global__ void k_b_emit(const double* pos, Prims P, Grid g, const int32_t* off, uint64_t* keys, int32_t* vals) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= P.nb) return;
  double lo[3], hi[3];
  prim_box(pos, P.b + P.ab * j, P.ab, lo, hi);
  int64_t c0[3], c1[3];
  for (int k = 0; k < 3; ++k) {
    c0[k] = cellc(g, k, lo[k]);
    c1[k] = cellc(g, k, hi[k]);
  }
  int64_t o = off[j];
  for (int64_t x = c0[0]; x <= c1[0]; ++x)
    for (int64_t y = c0[1]; y <= c1[1]; ++y)
      for (int64_t z = c0[2]; z <= c1[2]; ++z) {
        keys[o] = ckey(g, x, y, z);
        vals[o] = int32_t(j);
        ++o;
      }
}

__device__ __forceinline__ int64_t lbound(const uint64_t* k, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (k[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool is_fixed(const UnionDev& u, int64_t g) {
  int64_t loc;
  return u.child[union_decode(u, g, &loc)].kind == YS_POINTS_FIXED;
}

// Exact test of candidate (a, b): incident / all-fixed exclusions, then the
// distance type's squared distance < dhat.  Fills the stencil's points.
__device__ __forceinline__ bool stencil_test(const double* pos, const Prims& P, const UnionDev& u, int64_t a,
                                             int64_t b, double dhat, int32_t* st) {
  const int32_t* pa = P.a + P.aa * a;
  const int32_t* pb = P.b + P.ab * b;
  for (int i = 0; i < P.aa; ++i)
    for (int j = 0; j < P.ab; ++j)
      if (pa[i] == pb[j]) return false;
  const int ar = P.aa + P.ab;
  for (int i = 0; i < P.aa; ++i) st[i] = pa[i];
  for (int j = 0; j < P.ab; ++j) st[P.aa + j] = pb[j];
  bool all_fixed = true;
  for (int l = 0; l < ar; ++l) all_fixed = all_fixed && is_fixed(u, st[l]);
  if (all_fixed) return false;
  double x[4][3];
  for (int l = 0; l < ar; ++l)
    for (int k = 0; k < 3; ++k) x[l][k] = pos[3 * int64_t(st[l]) + k];
  const ContactSel s = classify_contact(P.kind, x);
  return contact_dist2_value(s, x) < dhat;
}

// Pass over the candidates of A primitive a: counts (out == nullptr) or
// writes the b of every hit (then sorted ascending).
__device__ int64_t scan_a(const double* pos, const Prims& P, const UnionDev& u, const Grid& g, const uint64_t* keys,
                          const int32_t* vals, int64_t nent, int64_t a, double dhat, double r, int32_t* out) {
  double lo[3], hi[3];
  prim_box(pos, P.a + P.aa * a, P.aa, lo, hi);
  int64_t q0[3], q1[3];
  for (int k = 0; k < 3; ++k) {
    q0[k] = cellc(g, k, lo[k] - r);
    q1[k] = cellc(g, k, hi[k] + r);
  }
  int64_t n = 0;
  int32_t st[4];
  for (int64_t x = q0[0]; x <= q1[0]; ++x)
    for (int64_t y = q0[1]; y <= q1[1]; ++y)
      for (int64_t z = q0[2]; z <= q1[2]; ++z) {
        const uint64_t key = ckey(g, x, y, z);
        for (int64_t e = lbound(keys, nent, key); e < nent && keys[e] == key; ++e) {
          const int64_t b = vals[e];
          if (P.self && b <= a) continue;
          // the first cell common to the query range and b's cells owns the pair
          double bl[3], bh[3];
          prim_box(pos, P.b + P.ab * b, P.ab, bl, bh);
          const int64_t ox = max(q0[0], cellc(g, 0, bl[0])), oy = max(q0[1], cellc(g, 1, bl[1])),
                        oz = max(q0[2], cellc(g, 2, bl[2]));
          if (ox != x || oy != y || oz != z) continue;
          if (!stencil_test(pos, P, u, a, b, dhat, st)) continue;
          if (out) out[n] = int32_t(b);
          ++n;
        }
      }
  if (out)  // insertion sort by b (a primitive has few hits)
    for (int64_t i = 1; i < n; ++i) {
      const int32_t v = out[i];
      int64_t j = i - 1;
      while (j >= 0 && out[j] > v) {
        out[j + 1] = out[j];
        --j;
      }
      out[j + 1] = v;
    }
  return n;
}

__global__ void k_a_count(const double* pos, Prims P, UnionDev u, Grid g, const uint64_t* keys, const int32_t* vals,
                          int64_t nent, double dhat, double r, int32_t* cnt) {
  const int64_t a = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a > P.na) return;
  cnt[a] = a == P.na ? 0 : int32_t(scan_a(pos, P, u, g, keys, vals, nent, a, dhat, r, nullptr));
}

__global__ void k_a_emit(const double* pos, Prims P, UnionDev u, Grid g, const uint64_t* keys, const int32_t* vals,
                         int64_t nent, double dhat, double r, const int32_t* off, int32_t* hits_b) {
  const int64_t a = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= P.na) return;
  scan_a(pos, P, u, g, keys, vals, nent, a, dhat, r, hits_b + off[a]);
}

// stencil k = (A primitive a, B primitive hits_b[k]) as union indices
__global__ void k_write_stencils(Prims P, const int32_t* off, const int32_t* hits_b, int64_t total, int32_t* out) {
  const int64_t a = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= P.na) return;
  const int ar = P.aa + P.ab;
  for (int64_t k = off[a]; k < off[a + 1]; ++k) {
    const int64_t b = hits_b[k];
    for (int i = 0; i < P.aa; ++i) out[ar * k + i] = P.a[P.aa * a + i];
    for (int j = 0; j < P.ab; ++j) out[ar * k + P.aa + j] = P.b[P.ab * b + j];
  }
  (void)total;
}

template <class T>
void exclusive_sum(Context& c, T* a, int64_t n) {
  size_t bytes = 0;
  YS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, a, a, int(n), c.stream));
  c.cubtmp.resize(std::max<size_t>(bytes, 1));
  YS_CUDA(cub::DeviceScan::ExclusiveSum(c.cubtmp.p, bytes, a, a, int(n), c.stream));
}

}  // namespace

void ctx_refresh_stencils(Context& c, int set, double dhat, int64_t* n_out) {
  PairSet& ps = c.pairsets[set];
  StencilPrims& sp = ps.prims;
  if (!sp.kind) fail(YS_ERR_VALIDATION, "stencil set has no primitives (ys_set_stencil_primitives)");
  cudaStream_t s = c.stream;
  const Union& un = c.unions[ps.uni];
  const int nc = int(un.children.size());
  std::vector<int64_t> base(size_t(nc + 1), 0);
  for (int k = 0; k < nc; ++k) base[size_t(k + 1)] = base[size_t(k)] + c.domains[un.children[size_t(k)]].n;
  ContactScratch& X = c.contact;
  X.pos.resize(size_t(3 * std::max<int64_t>(base[size_t(nc)], 1)));
  for (int k = 0; k < nc; ++k) ctx_domain_points(c, un.children[size_t(k)], X.pos.p + 3 * base[size_t(k)]);
  Prims P{sp.a.p, sp.self ? sp.a.p : sp.b.p, sp.na, sp.self ? sp.na : sp.nb, sp.aa, sp.self ? sp.aa : sp.ab,
          sp.kind, sp.self};
  UnionDev u{};
  u.nchild = nc;
  u.kappa_u = un.kappa_u;
  u.width = un.width;
  u.child = un.d_child.p;
  u.offsets = un.d_offsets.p;
  // grid: h = max(sqrt(dhat), largest B extent), over the union's box
  X.part.resize(8);
  YS_CUDA(cudaMemsetAsync(X.part.p, 0, 8 * sizeof(double), s));
  if (P.nb > 0) k_prim_extent<<<grid_for(P.nb), kTB, 0, s>>>(X.pos.p, P, X.part.p);
  YS_LAUNCH_CHECK();
  double ext = 0.0;
  YS_CUDA(cudaMemcpyAsync(&ext, X.part.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  std::vector<double> hp(size_t(3 * base[size_t(nc)]));
  if (!hp.empty()) YS_CUDA(cudaMemcpyAsync(hp.data(), X.pos.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (size_t i = 0; i < hp.size(); ++i) {
    const double v = hp[i];
    if (v == v) {
      lo[i % 3] = std::min(lo[i % 3], v);
      hi[i % 3] = std::max(hi[i % 3], v);
    }
  }
  const double r = std::sqrt(dhat) * (1.0 + 1e-6);
  double h = std::max(r, ext * (1.0 + 1e-6));
  Grid g{};
  for (int k = 0; k < 3; ++k) {
    if (!(lo[k] <= hi[k])) lo[k] = hi[k] = 0.0;
    g.o[k] = lo[k] - 2.0 * r;
  }
  for (;;) {  // at most 2^20 cells per axis
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
      g.dim[k] = int64_t(std::floor((hi[k] - lo[k] + 4.0 * r) / h)) + 1;
      ok = ok && g.dim[k] <= (int64_t(1) << 20);
    }
    if (ok) break;
    h *= 2.0;
  }
  g.inv_h = 1.0 / h;
  // B entries sorted by cell
  X.cnt.resize(size_t(P.nb + 1));
  k_b_count<<<grid_for(P.nb + 1), kTB, 0, s>>>(X.pos.p, P, g, X.cnt.p);
  YS_LAUNCH_CHECK();
  exclusive_sum(c, X.cnt.p, P.nb + 1);
  int32_t nent = 0;
  YS_CUDA(cudaMemcpyAsync(&nent, X.cnt.p + P.nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  X.keys.resize(size_t(std::max(nent, 1)));
  X.keys_out.resize(size_t(std::max(nent, 1)));
  X.idx.resize(size_t(std::max(nent, 1)));
  X.idx_out.resize(size_t(std::max(nent, 1)));
  if (P.nb > 0) k_b_emit<<<grid_for(P.nb), kTB, 0, s>>>(X.pos.p, P, g, X.cnt.p, X.keys.p, X.idx.p);
  YS_LAUNCH_CHECK();
  if (nent > 0) {
    size_t bytes = 0;
    YS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, X.keys.p, X.keys_out.p, X.idx.p, X.idx_out.p, nent, 0,
                                            64, s));
    c.cubtmp.resize(std::max<size_t>(bytes, 1));
    YS_CUDA(cub::DeviceRadixSort::SortPairs(c.cubtmp.p, bytes, X.keys.p, X.keys_out.p, X.idx.p, X.idx_out.p, nent,
                                            0, 64, s));
  }
  // A queries: count, scan, emit (sorted by b), stencils
  X.off.resize(size_t(P.na + 1));
  k_a_count<<<grid_for(P.na + 1), kTB, 0, s>>>(X.pos.p, P, u, g, X.keys_out.p, X.idx_out.p, nent, dhat, r, X.off.p);
  YS_LAUNCH_CHECK();
  exclusive_sum(c, X.off.p, P.na + 1);
  int32_t total = 0;
  YS_CUDA(cudaMemcpyAsync(&total, X.off.p + P.na, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  X.scratch.resize(size_t(std::max(total, 1)));
  if (P.na > 0)
    k_a_emit<<<grid_for(P.na), kTB, 0, s>>>(X.pos.p, P, u, g, X.keys_out.p, X.idx_out.p, nent, dhat, r, X.off.p,
                                           X.scratch.p);
  const int ar = P.aa + P.ab;
  ps.pairs.resize(size_t(std::max<int64_t>(int64_t(ar) * total, 1)));
  if (P.na > 0 && total > 0)
    k_write_stencils<<<grid_for(P.na), kTB, 0, s>>>(P, X.off.p, X.scratch.p, total, ps.pairs.p);
  YS_LAUNCH_CHECK();
  c.launches += 8;
  ps.n = total;
  ps.h_pairs.clear();
  ps.host_stale = total > 0;
  ++c.epoch;  // resize_dynamic bumps the scene's dynamic epoch (scene.cpp:198)
  if (n_out) *n_out = total;
}

}  // namespace ys
