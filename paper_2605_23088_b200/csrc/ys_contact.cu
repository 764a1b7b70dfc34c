// ys_contact.cu — contact candidates of Simulation::refresh_dynamic_pairs
// (sim.cpp:456-484) on the device, bit-exact, with a uniform grid instead of
// the reference's all-pairs loop.
//
// Reference semantics: children of the contact union in union order; for
// every child pair ca < cb that is not fixed-fixed, every (i in ca, j in cb)
// with squaredNorm(p_i - q_j) < dhat (strict), emitted in (ca, cb, i, j)
// order as union indices (child offset + local index).
//
// Grid: cell edge h >= sqrt(dhat) (slightly enlarged so floating rounding in
// floor(x / h) can never separate a qualifying pair by two cells, and grown
// further if a child's box would need more than 2^20 cells per axis), so a
// qualifying pair always lies in the same or an adjacent cell.  The points of
// the B child are sorted by 63-bit cell key (radix sort is stable: j stays
// ascending inside a cell); an A point scans its 27 neighbour cells with the
// exact distance test the reference uses, and sorts its few hits by j.  The
// candidate set is a superset and the test is identical, so the pair list is
// identical.  Child pairs whose boxes (grown by h) are disjoint are skipped.
#include <algorithm>
#include <cmath>
#include <string>

#include <cub/cub.cuh>

#include "ys_device.cuh"

namespace ys {

void ctx_domain_points(Context& c, int domain, double* out);

namespace {
constexpr int kTB = 256;
constexpr int kBits = 21;  // bits per axis in a cell key
inline unsigned grid_for(int64_t n, int tb = kTB) { return unsigned(std::max<int64_t>(1, ceil_div(n, tb))); }

// d2 = ((dx*dx + dy*dy) + dz*dz) with explicit rounding (no FMA), Eigen's
// squaredNorm order for a 3-vector; strict d2 < dhat (sim.cpp:471-472).
__device__ __forceinline__ bool close_pair(const double* a, const double* b, double dhat) {
  const double dx = __dsub_rn(a[0], b[0]);
  const double dy = __dsub_rn(a[1], b[1]);
  const double dz = __dsub_rn(a[2], b[2]);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return d2 < dhat;
}

struct GridDev {
  const uint64_t* keys;  // sorted cell keys of the B points
  const int32_t* idx;    // B point of each sorted key
  int64_t n;
  double inv_h;
  int64_t lo[3];         // cell coordinate of key 0 along each axis
};

__device__ __forceinline__ uint64_t cell_key(int64_t cx, int64_t cy, int64_t cz) {
  return (uint64_t(cx) << (2 * kBits)) | (uint64_t(cy) << kBits) | uint64_t(cz);
}

__device__ __forceinline__ bool cell_of(const GridDev& g, const double* p, int64_t (&c)[3]) {
  for (int a = 0; a < 3; ++a) {
    const double q = floor(p[a] * g.inv_h);
    if (!(q > -4.0e15 && q < 4.0e15)) return false;  // NaN / inf positions never pair
    c[a] = int64_t(q) - g.lo[a];
  }
  return true;
}

__global__ void k_bbox_partial(const double* __restrict__ p, int64_t n, double* part) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    for (int a = 0; a < 3; ++a) {
      const double v = p[3 * i + a];
      if (v == v) {  // NaN coordinates are ignored (they can never pass the distance test)
        mn[a] = fmin(mn[a], v);
        mx[a] = fmax(mx[a], v);
      }
    }
  __shared__ double sm[6][kTB];
  for (int a = 0; a < 3; ++a) {
    sm[a][threadIdx.x] = mn[a];
    sm[3 + a][threadIdx.x] = mx[a];
  }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int a = 0; a < 3; ++a) {
        sm[a][threadIdx.x] = fmin(sm[a][threadIdx.x], sm[a][threadIdx.x + w]);
        sm[3 + a][threadIdx.x] = fmax(sm[3 + a][threadIdx.x], sm[3 + a][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) part[6 * blockIdx.x + k] = sm[k][0];
}

__global__ void k_bbox_final(const double* part, int nparts, double* out) {
  if (threadIdx.x != 0) return;
  double b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int q = 0; q < nparts; ++q)
    for (int a = 0; a < 3; ++a) {
      b[a] = fmin(b[a], part[6 * q + a]);
      b[3 + a] = fmax(b[3 + a], part[6 * q + 3 + a]);
    }
  for (int k = 0; k < 6; ++k) out[k] = b[k];
}

__global__ void k_cell_keys(const double* __restrict__ p, int64_t n, GridDev g, uint64_t* keys, int32_t* idx) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c[3];
  const bool ok = cell_of(g, p + 3 * i, c);
  keys[i] = ok ? cell_key(c[0], c[1], c[2]) : ~uint64_t(0);  // outside: sorts last, never looked up
  idx[i] = int32_t(i);
}

__device__ __forceinline__ int64_t lower_bound_key(const uint64_t* k, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (k[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Visits every B point in the 27 cells around p (cells outside the key range hold no points).
template <class F>
__device__ __forceinline__ void for_neighbours(const GridDev& g, const double* p, F&& f) {
  int64_t c[3];
  if (!cell_of(g, p, c)) return;
  const int64_t top = (int64_t(1) << kBits) - 1;
  for (int dx = -1; dx <= 1; ++dx) {
    const int64_t x = c[0] + dx;
    if (x < 0 || x > top) continue;
    for (int dy = -1; dy <= 1; ++dy) {
      const int64_t y = c[1] + dy;
      if (y < 0 || y > top) continue;
      for (int dz = -1; dz <= 1; ++dz) {
        const int64_t z = c[2] + dz;
        if (z < 0 || z > top) continue;
        const uint64_t key = cell_key(x, y, z);
        for (int64_t k = lower_bound_key(g.keys, g.n, key); k < g.n && g.keys[k] == key; ++k) f(g.idx[k]);
      }
    }
  }
}

__global__ void k_grid_count(const double* __restrict__ pa, int64_t na, const double* __restrict__ pb, GridDev g,
                             double dhat, int32_t* cnt) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= na) return;
  const double p[3] = {pa[3 * i], pa[3 * i + 1], pa[3 * i + 2]};
  int32_t n = 0;
  for_neighbours(g, p, [&](int32_t j) { n += close_pair(p, pb + 3 * int64_t(j), dhat) ? 1 : 0; });
  cnt[i] = n;
}

__global__ void k_grid_emit(const double* __restrict__ pa, int64_t na, const double* __restrict__ pb, GridDev g,
                            double dhat, const int32_t* __restrict__ off, int32_t* scratch, int64_t base_a,
                            int64_t base_b, int32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= na) return;
  const double p[3] = {pa[3 * i], pa[3 * i + 1], pa[3 * i + 2]};
  const int64_t w0 = off[i];
  int64_t w = w0;
  for_neighbours(g, p, [&](int32_t j) {
    if (close_pair(p, pb + 3 * int64_t(j), dhat)) scratch[w++] = j;
  });
  // the reference's inner loop runs j ascending
  for (int64_t a = w0 + 1; a < w; ++a) {
    const int32_t v = scratch[a];
    int64_t b = a - 1;
    while (b >= w0 && scratch[b] > v) {
      scratch[b + 1] = scratch[b];
      --b;
    }
    scratch[b + 1] = v;
  }
  for (int64_t k = w0; k < w; ++k) {
    out[2 * k] = int32_t(base_a + i);
    out[2 * k + 1] = int32_t(base_b + scratch[k]);
  }
}

struct ActivePair {
  int ca, cb;
  int64_t row0;  // first row of this pair in the concatenated count array
};
}  // namespace

void ctx_refresh_pairs(Context& c, int pairset, double dhat, const int32_t* child_fixed, int64_t* n_pairs) {
  PairSet& ps = c.pairsets[pairset];
  Union& u = c.unions[ps.uni];
  ContactScratch& X = c.contact;
  cudaStream_t s = c.stream;
  const int nc = int(u.children.size());
  std::vector<int64_t> base(nc + 1, 0);
  for (int k = 0; k < nc; ++k) base[k + 1] = base[k] + c.domains[u.children[k]].n;
  const int64_t nu = base[nc];
  X.pos.resize(size_t(3 * std::max<int64_t>(nu, 1)));
  for (int k = 0; k < nc; ++k) ctx_domain_points(c, u.children[k], X.pos.p + 3 * base[k]);
  auto fixed = [&](int k) {
    return child_fixed ? child_fixed[k] != 0 : c.domains[u.children[k]].kind == YS_POINTS_FIXED;
  };
  auto P = [&](int k) { return X.pos.p + 3 * base[k]; };
  int64_t total = 0;
  if (dhat > 0.0 && nc > 1) {
    // 1. boxes of every child (one sync)
    const int nparts = 64;
    X.part.resize(size_t(6 * nparts * nc));
    X.boxes.resize(size_t(6 * nc));
    for (int k = 0; k < nc; ++k) {
      const int64_t n = base[k + 1] - base[k];
      if (n == 0) continue;
      k_bbox_partial<<<nparts, kTB, 0, s>>>(P(k), n, X.part.p + 6 * nparts * k);
      k_bbox_final<<<1, 32, 0, s>>>(X.part.p + 6 * nparts * k, nparts, X.boxes.p + 6 * k);
      YS_LAUNCH_CHECK();
    }
    std::vector<double> box = X.boxes.to_host(s);
    // 2. active child pairs in the reference's (ca, cb) order
    const double h0 = std::sqrt(dhat) * (1.0 + 1e-6);
    std::vector<ActivePair> act;
    std::vector<char> need_grid(nc, 0);
    int64_t rows = 0;
    for (int ca = 0; ca < nc; ++ca)
      for (int cb = ca + 1; cb < nc; ++cb) {
        if (fixed(ca) && fixed(cb)) continue;
        const int64_t na = base[ca + 1] - base[ca], nbb = base[cb + 1] - base[cb];
        if (na == 0 || nbb == 0) continue;
        const double* A = &box[6 * ca];
        const double* B = &box[6 * cb];
        if (!(A[0] <= A[3]) || !(B[0] <= B[3])) continue;  // all-NaN child: no pair can pass
        bool apart = false;
        for (int a = 0; a < 3; ++a) apart = apart || A[a] - h0 > B[3 + a] || B[a] - h0 > A[3 + a];
        if (apart) continue;
        act.push_back({ca, cb, rows});
        rows += na;
        need_grid[cb] = 1;
      }
    if (!act.empty()) {
      // 3. grids of the B children (per-child slices, stable radix sort by cell key)
      std::vector<GridDev> grid(nc);
      X.keys.resize(size_t(nu));
      X.keys_out.resize(size_t(nu));
      X.idx.resize(size_t(nu));
      X.idx_out.resize(size_t(nu));
      for (int k = 0; k < nc; ++k) {
        if (!need_grid[k]) continue;
        const int64_t n = base[k + 1] - base[k];
        const double* B = &box[6 * k];
        double h = h0;
        for (int a = 0; a < 3; ++a) h = std::max(h, (B[3 + a] - B[a]) / double(1 << (kBits - 1)));
        GridDev g{X.keys_out.p + base[k], X.idx_out.p + base[k], n, 1.0 / h, {0, 0, 0}};
        for (int a = 0; a < 3; ++a) g.lo[a] = int64_t(std::floor(B[a] / h)) - 2;
        k_cell_keys<<<grid_for(n), kTB, 0, s>>>(P(k), n, g, X.keys.p + base[k], X.idx.p + base[k]);
        YS_LAUNCH_CHECK();
        size_t bytes = 0;
        YS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, X.keys.p + base[k], X.keys_out.p + base[k],
                                                X.idx.p + base[k], X.idx_out.p + base[k], int(n), 0, 64, s));
        c.cubtmp.resize(std::max(c.cubtmp.n, bytes + 1));
        YS_CUDA(cub::DeviceRadixSort::SortPairs(c.cubtmp.p, bytes, X.keys.p + base[k], X.keys_out.p + base[k],
                                                X.idx.p + base[k], X.idx_out.p + base[k], int(n), 0, 64, s));
        grid[k] = g;
      }
      // 4. counts of every (pair, i) row, one scan: the prefix is the output
      //    position in the reference's (ca, cb, i, j) order
      X.cnt.resize(size_t(rows) + 1);
      X.off.resize(size_t(rows) + 1);
      YS_CUDA(cudaMemsetAsync(X.cnt.p + rows, 0, sizeof(int32_t), s));
      for (const ActivePair& ap : act) {
        const int64_t na = base[ap.ca + 1] - base[ap.ca];
        k_grid_count<<<grid_for(na, 128), 128, 0, s>>>(P(ap.ca), na, P(ap.cb), grid[ap.cb], dhat, X.cnt.p + ap.row0);
        YS_LAUNCH_CHECK();
      }
      size_t bytes = 0;
      YS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, X.cnt.p, X.off.p, int(rows) + 1, s));
      c.cubtmp.resize(std::max(c.cubtmp.n, bytes + 1));
      YS_CUDA(cub::DeviceScan::ExclusiveSum(c.cubtmp.p, bytes, X.cnt.p, X.off.p, int(rows) + 1, s));
      int32_t tot = 0;
      YS_CUDA(cudaMemcpyAsync(&tot, X.off.p + rows, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      YS_CUDA(cudaStreamSynchronize(s));
      total = tot;
      // 5. emit straight into the pair set
      if (total > 0) {
        X.scratch.resize(size_t(total));
        ps.pairs.resize(size_t(2 * total));
        for (const ActivePair& ap : act) {
          const int64_t na = base[ap.ca + 1] - base[ap.ca];
          k_grid_emit<<<grid_for(na, 128), 128, 0, s>>>(P(ap.ca), na, P(ap.cb), grid[ap.cb], dhat, X.off.p + ap.row0,
                                                        X.scratch.p, base[ap.ca], base[ap.cb], ps.pairs.p);
          YS_LAUNCH_CHECK();
        }
      }
    }
  }
  if (total == 0) ps.pairs.resize(0);
  ps.n = total;
  ps.h_pairs.clear();
  ps.host_stale = total > 0;
  ++c.epoch;
  if (n_pairs) *n_pairs = ps.n;
}

}  // namespace ys
