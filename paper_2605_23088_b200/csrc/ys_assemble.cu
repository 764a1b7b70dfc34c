// ys_assemble.cu — local evaluation, deterministic assembly and the block
// Jacobi build.
//
// Reference: Engine::assemble (engine.cpp:47-60) -> assemble_group
// (assembly.cpp:323-374) -> assemble_local (284-321) -> serial scatter
// (346-372); DiagAccumulator (158-180); BlockJacobiPreconditioner::build
// (solver.cpp:93-122); Engine::total_energy (engine.cpp:64-68).
//
// Flow per Newton iteration:
//   1. one eval kernel per energy writes every instance's raw-slot gradient
//      and its oriented ublock-pair Hessian blocks into the group buffers
//      (contiguous per instance: coalesced stores);
//   2. k_gather_h sums the k-th sorted run of block contributions into
//      unique block k in (energy, instance) order — bit-identical to the
//      reference's serial `+=` for identical local blocks;
//   3. k_block_rows (one thread per target instance) gathers the gradient
//      (static runs then dynamic runs, the reference's order), forms the
//      DiagAccumulator block (static H block + dynamic contributions one by
//      one) and inverts it for the preconditioner.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "ys_contact4.cuh"
#include "ys_device.cuh"

namespace ys {

namespace {
constexpr int kTB = 256;
inline unsigned grid_for(int64_t n, int tb = kTB) { return unsigned(std::max<int64_t>(1, ceil_div(n, tb))); }
}  // namespace

// error flag bits (NumericalError sources in eval.cpp)
constexpr int kErrLog = 1;  // "log of non-positive value" (eval.cpp:296-301)
constexpr int kErrDiv = 2;  // "division by zero" (eval.cpp:226-237)

EnergyDev energy_dev(Context& c, Energy& e) {
  EnergyDev E{};
  E.kind = e.kind;
  E.kappa = e.kappa;
  E.width = e.width;
  E.mode = e.mode;
  E.n = e.n;
  E.conn = e.conn.p;
  E.cdata = e.cdata.p;
  E.anchor = e.anchor.p;
  E.startP = e.target >= 0 ? int32_t(c.targets[e.target].start) : 0;
  if (e.domain >= 0) {
    const Domain& d = c.domains[e.domain];
    E.dom.kind = d.kind;
    E.dom.n = d.n;
    E.dom.startA = d.ta >= 0 ? int32_t(c.targets[d.ta].start) : 0;
    E.dom.startB = d.tb >= 0 ? int32_t(c.targets[d.tb].start) : 0;
    E.dom.v2b = d.v2b.p;
    E.dom.rest = d.rest.p;
    E.dom.fixed = d.rest.p;
  }
  if (e.pairset >= 0) {
    const PairSet& ps = c.pairsets[e.pairset];
    const Union& u = c.unions[ps.uni];
    E.uni.nchild = int32_t(u.children.size());
    E.uni.kappa_u = u.kappa_u;
    E.uni.width = u.width;
    E.uni.child = u.d_child.p;
    E.uni.offsets = u.d_offsets.p;
    E.pairs = ps.pairs.p;
    E.arity = ps.arity;
  }
  for (int k = 0; k < 6; ++k) E.prm[k] = e.prm[k];
  E.slots = e.slots.p;
  E.m = e.m.p;
  E.hoff = e.uniform ? nullptr : e.hoff.p;
  E.goff = e.uniform ? nullptr : e.goff.p;
  E.doff = e.uniform ? nullptr : e.doff.p;
  E.soff = e.uniform ? nullptr : e.soff.p;
  E.hstride = e.hstride;
  E.gstride = e.gstride;
  E.dstride = e.dstride;
  E.sstride = e.sstride;
  E.hbase = e.hbase;
  E.gbase = e.gbase;
  E.dbase = e.dbase;
  E.sbase = e.sbase;
  return E;
}

// ---------------------------------------------------------------------------
// Evaluation kernels

struct VertexBlockWriter {
  double* h;
  uint32_t swap;  // bit p: store pair p transposed (gstart(a) > gstart(b))
  __device__ __forceinline__ void operator()(int pair, int k, int kk, double v) const {
    h[pair * 9 + (((swap >> pair) & 1u) ? kk * 3 + k : k * 3 + kk)] = v;
  }
  // a whole 3x3 block (row-major v): four 16-byte stores and one 8-byte store
  // (the block's 72 bytes start 16-byte aligned for every other pair)
  __device__ __forceinline__ void block(int pair, const double (&v)[9]) const {
    const bool sw = (swap >> pair) & 1u;
    double o[9];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) o[k * 3 + kk] = sw ? v[kk * 3 + k] : v[k * 3 + kk];
    double* d = h + pair * 9;
    if ((reinterpret_cast<uintptr_t>(d) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 8; q += 2) *reinterpret_cast<double2*>(d + q) = make_double2(o[q], o[q + 1]);
      d[8] = o[8];
    } else {
      d[0] = o[0];
#pragma unroll
      for (int q = 1; q < 9; q += 2) *reinterpret_cast<double2*>(d + q) = make_double2(o[q], o[q + 1]);
    }
  }
};

__device__ __forceinline__ uint32_t vertex_pair_swaps(const int32_t gs[4]) {
  uint32_t sw = 0;
  int pair = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = a; b < 4; ++b, ++pair)
      if (gs[a] > gs[b]) sw |= 1u << pair;
  return sw;
}

__device__ __forceinline__ void load_stencil(const EnergyDev& E, const double* __restrict__ X, int64_t i,
                                             double x[12], int32_t gs[4]) {
  const int4 v = reinterpret_cast<const int4*>(E.conn)[i];
  const int vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    gs[l] = E.startP + 3 * vv[l];
    const double* q = X + gs[l];
    x[3 * l + 0] = q[0];
    x[3 * l + 1] = q[1];
    x[3 * l + 2] = q[2];
  }
}

// Pass A of the 9x9-projected stencil terms (SNH: KIND 0, bending: KIND 1):
// gradient, edge-space Hessian, and — when the projection matrix M is positive
// definite (Cholesky succeeds) — the vertex blocks of M directly.  Indefinite
// elements are compacted into (list, M) for pass B.
template <int KIND>
__global__ void __launch_bounds__(128) k_eval_stencil_a(EnergyDev E, const double* __restrict__ X, int project,
                                                        int want_h, double* __restrict__ hc,
                                                        double* __restrict__ gc, int* err,
                                                        unsigned int* __restrict__ count,
                                                        int32_t* __restrict__ list, double* __restrict__ mbuf,
                                                        const int32_t* __restrict__ sel, int64_t nsel) {
  // sel: the instances to evaluate (the distributed solve's owned-row subset), else all
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= (sel ? nsel : E.n)) return;
  const int64_t i = sel ? int64_t(sel[t]) : t;
  double x[12];
  int32_t gs[4];
  load_stencil(E, X, i, x, gs);
  double g[12];
  double hd[45];
  if (KIND == 0) {
    double binv[9];
    const double* cd = E.cdata + 10 * i;
#pragma unroll
    for (int k = 0; k < 9; ++k) binv[k] = cd[k];
    const SnhParams P{E.prm[0], E.prm[1], E.prm[2], E.prm[3]};
    snh_local(x, binv, cd[9], P, want_h != 0, g, hd);
  } else {
    if (bending_local(x, E.cdata[i], want_h != 0, g, hd)) atomicOr(err, kErrDiv);
  }
  double* go = gc + inst_goff(E, i);
#pragma unroll
  for (int k = 0; k < 12; ++k) go[k] = g[k];
  if (!want_h) return;
  const VertexBlockWriter wr{hc + inst_hoff(E, i), vertex_pair_swaps(gs)};
  if (!project) {
    expand_vertex_blocks(hd, false, wr);
    return;
  }
  const bool full = KIND == 1 || E.mode != YS_PROJECT_REDUCED;
  if (full) edge_to_projection_space(hd);
  // M goes to the element's slot first; the positive-definiteness test then
  // factors the registers in place (no second 45-register copy)
  double* m = mbuf + kMStride * i;
  store_m(m, hd);
  if (cholesky_pd9_inplace(hd)) {
    // M is PD: the projection is M itself (reloaded from its slot)
    reload_m(m, hd);
    expand_vertex_blocks(hd, full, wr);
    return;
  }
  // indefinite: pass B projects M and writes the vertex blocks
  const unsigned k = atomicAdd(count, 1u);
  list[k] = int32_t(i);
}

// Pass B: Jacobi EVD + clamp + reconstruction for the compacted indefinite
// elements only (fully populated warps), then the vertex blocks.
//
// Pass B batched over up to kStencilBatch energies of one kind (C5: the 8 soft
// bodies): one launch whose grid-stride loop spans every energy's compacted
// list, so the ~9 EVDs per thread leave no per-energy tail (8 launches of
// ~1.2 EVDs per resident thread lost about half the SMs to the tail).
constexpr int kStencilBatch = 8;
struct StencilBatch {
  int n;
  EnergyDev e[kStencilBatch];
  double* hc[kStencilBatch];
  const unsigned int* count[kStencilBatch];
  int64_t base[kStencilBatch];  // first list / M slot of each energy
  unsigned int* fbcount[kStencilBatch];  // elements handed to the Jacobi path, per energy
  int32_t* fblist[kStencilBatch];        // their local list positions (k - first of the energy)
};

// Pass B, main path: the clamped-eigenpair projection (psd_project9_tri,
// ~5k FP64 operations, registers + 552 B of shared memory per thread); an
// element whose verification fails goes to its energy's fallback list.
template <int KIND>
__global__ void __launch_bounds__(kProjStride, 3) k_eval_stencil_b_tri(const __grid_constant__ StencilBatch B,
                                                                       const int32_t* __restrict__ list,
                                                                       const double* __restrict__ mbuf,
                                                                       double* __restrict__ scratch,
                                                                       int force_fallback) {
  extern __shared__ double sm_proj[];
  const int64_t gstride = int64_t(gridDim.x) * blockDim.x;
  double* gsc = scratch + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned pre[kStencilBatch + 1];
  pre[0] = 0;
#pragma unroll
  for (int j = 0; j < kStencilBatch; ++j) pre[j + 1] = pre[j] + (j < B.n ? *B.count[j] : 0u);
  const unsigned total = pre[kStencilBatch];
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    int j = 0;
    unsigned prej = 0;  // pre[j] by a static select (no local-memory array)
#pragma unroll
    for (int q = 1; q < kStencilBatch; ++q)
      if (k >= pre[q]) {
        j = q;
        prej = pre[q];
      }
    const EnergyDev& E = B.e[j];
    const int64_t slot = B.base[j] + (k - prej);
    const int64_t i = list[slot];
    double m[45];
    if (force_fallback || !psd_project9_tri(mbuf + kMStride * (B.base[j] + i), m, sm_proj + threadIdx.x, gsc, gstride)) {
      const unsigned f = atomicAdd(B.fbcount[j], 1u);
      B.fblist[j][f] = int32_t(i);
      continue;
    }
    const int4 v = reinterpret_cast<const int4*>(E.conn)[i];
    const int32_t gs[4] = {E.startP + 3 * v.x, E.startP + 3 * v.y, E.startP + 3 * v.z, E.startP + 3 * v.w};
    const bool full = KIND == 1 || E.mode != YS_PROJECT_REDUCED;
    const VertexBlockWriter wr{B.hc[j] + inst_hoff(E, i), vertex_pair_swaps(gs)};
    expand_vertex_blocks(m, full, wr);
  }
}

// Pass B, fallback: the cyclic Jacobi EVD (psd_project9) for the elements the
// main path handed over (all of them with ys_set_option("eval_evd", 0)).
template <int KIND>
__global__ void __launch_bounds__(128) k_eval_stencil_b_fallback(const __grid_constant__ StencilBatch B,
                                                                 const int32_t* __restrict__ list,
                                                                 const double* __restrict__ mbuf) {
  unsigned pre[kStencilBatch + 1];
  pre[0] = 0;
#pragma unroll
  for (int j = 0; j < kStencilBatch; ++j) pre[j + 1] = pre[j] + (j < B.n ? *B.fbcount[j] : 0u);
  const unsigned total = pre[kStencilBatch];
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    int j = 0;
#pragma unroll
    for (int q = 1; q < kStencilBatch; ++q) j += k >= pre[q] ? 1 : 0;
    const EnergyDev& E = B.e[j];
    const int64_t i = B.fblist[j][k - pre[j]];  // element id
    double m[45];
    const double* src = mbuf + kMStride * (B.base[j] + i);
#pragma unroll
    for (int q = 0; q < 45; ++q) m[q] = src[q];  // (fallback paths: scalar loads)
    psd_project9(m);
    const int4 v = reinterpret_cast<const int4*>(E.conn)[i];
    const int32_t gs[4] = {E.startP + 3 * v.x, E.startP + 3 * v.y, E.startP + 3 * v.z, E.startP + 3 * v.w};
    const bool full = KIND == 1 || E.mode != YS_PROJECT_REDUCED;
    const VertexBlockWriter wr{B.hc[j] + inst_hoff(E, i), vertex_pair_swaps(gs)};
    expand_vertex_blocks(m, full, wr);
  }
}

template <int KIND>
__global__ void __launch_bounds__(128) k_eval_stencil_b_batch(const __grid_constant__ StencilBatch B,
                                                              const int32_t* __restrict__ list,
                                                              const double* __restrict__ mbuf) {
  unsigned pre[kStencilBatch + 1];
  pre[0] = 0;
#pragma unroll
  for (int j = 0; j < kStencilBatch; ++j) pre[j + 1] = pre[j] + (j < B.n ? *B.count[j] : 0u);
  const unsigned total = pre[kStencilBatch];
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    int j = 0;
#pragma unroll
    for (int q = 1; q < kStencilBatch; ++q) j += k >= pre[q] ? 1 : 0;
    const EnergyDev& E = B.e[j];
    const int64_t slot = B.base[j] + (k - pre[j]);
    const int64_t i = list[slot];
    double m[45];
    const double* src = mbuf + kMStride * (B.base[j] + i);
#pragma unroll
    for (int q = 0; q < 45; ++q) m[q] = src[q];  // (fallback paths: scalar loads)
    psd_project9(m);
    const int4 v = reinterpret_cast<const int4*>(E.conn)[i];
    const int32_t gs[4] = {E.startP + 3 * v.x, E.startP + 3 * v.y, E.startP + 3 * v.z, E.startP + 3 * v.w};
    const bool full = KIND == 1 || E.mode != YS_PROJECT_REDUCED;
    const VertexBlockWriter wr{B.hc[j] + inst_hoff(E, i), vertex_pair_swaps(gs)};
    expand_vertex_blocks(m, full, wr);
  }
}

__device__ __forceinline__ void ortho_instance(const EnergyDev& E, int64_t i, const double* __restrict__ X,
                                               int project, int want_h, double* __restrict__ hc,
                                               double* __restrict__ gc) {
  double A[9];
  const double* q = X + E.startP + 9 * i;
#pragma unroll
  for (int k = 0; k < 9; ++k) A[k] = q[k];
  double g[9];
  ortho_local(A, E.prm[0], want_h != 0, project != 0, g, hc + inst_hoff(E, i));
  double* go = gc + inst_goff(E, i);
#pragma unroll
  for (int k = 0; k < 9; ++k) go[k] = g[k];
}

__global__ void __launch_bounds__(128) k_eval_ortho(EnergyDev E, const double* __restrict__ X, int project,
                                                    int want_h, double* __restrict__ hc, double* __restrict__ gc) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  ortho_instance(E, i, X, project, want_h, hc, gc);
}

// Inertia of free points: one 3x3 block m I (projection: max(m, 0) I).
__global__ void k_eval_inertia_free(EnergyDev E, const double* __restrict__ X, int project, int want_h,
                                    double* __restrict__ hc, double* __restrict__ gc) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  const double* q = X + E.dom.startA + 3 * i;
  const double* xt = E.anchor + 3 * i;
  const double m = E.cdata[i];
  double* go = gc + E.gbase + 3 * i;
#pragma unroll
  for (int k = 0; k < 3; ++k) go[k] = m * (q[k] - xt[k]);
  if (!want_h) return;
  const double d = (project && !(m > 0.0)) ? 0.0 : m;
  double* h = hc + E.hbase + 9 * i;
#pragma unroll
  for (int k = 0; k < 9; ++k) h[k] = (k % 4 == 0) ? d : 0.0;
}

// Pair energies over unions of free / fixed points (kappa_u == 1).
__global__ void k_eval_pair_free(EnergyDev E, const double* __restrict__ X, int project, int want_h,
                                 double* __restrict__ hc, double* __restrict__ gc, int* err) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  double p[2][3];
  int32_t gs[2];
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    int64_t loc;
    const int br = union_decode(E.uni, E.pairs[2 * i + l], &loc);
    const DomainDev& d = E.uni.child[br];
    if (d.kind == YS_POINTS_FREE) {
      gs[l] = int32_t(d.startA + 3 * loc);
      const double* q = X + gs[l];
      p[l][0] = q[0]; p[l][1] = q[1]; p[l][2] = q[2];
    } else {
      gs[l] = -1;
      const double* q = d.fixed + 3 * loc;
      p[l][0] = q[0]; p[l][1] = q[1]; p[l][2] = q[2];
    }
  }
  double dl[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) dl[k] = p[1][k] - p[0][k];
  const double d = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
  const PairParams PP{E.prm[0], E.prm[1], E.prm[2], E.kind == K_REPULSIVE};
  double b, b1, b2;
  const int st = pair_b(d, PP, &b, &b1, &b2);
  if (st) atomicOr(err, st == 1 ? kErrLog : kErrDiv);
  double* go = gc + inst_goff(E, i);
  int o = 0;
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    if (gs[l] < 0) continue;
    const double sg = l == 0 ? -2.0 * b1 : 2.0 * b1;
#pragma unroll
    for (int k = 0; k < 3; ++k) go[o + k] = sg * dl[k];
    o += 3;
  }
  if (!want_h) return;
  double P[9];
  proj_rank1_3(2.0 * b1, 4.0 * b2, dl, d, project != 0, P);
  double* h = hc + inst_hoff(E, i);
  const int nfree = (gs[0] >= 0) + (gs[1] >= 0);
  if (nfree == 2 && gs[0] == gs[1]) {  // both ends on one vertex: merged, rho = 0
#pragma unroll
    for (int k = 0; k < 9; ++k) h[k] = 0.0;
  } else if (nfree == 2) {  // (0,0) = P, (0,1) = -P (symmetric, orientation-free), (1,1) = P
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      h[k] = P[k];
      h[9 + k] = -P[k];
      h[18 + k] = P[k];
    }
  } else if (nfree == 1) {
#pragma unroll
    for (int k = 0; k < 9; ++k) h[k] = P[k];
  }
}

// Inertia over affine points and pair energies over unions with affine
// bodies: one 3-vector delta, linear in the compressed DoFs.
__device__ __forceinline__ void point_instance(const EnergyDev& E, int64_t i, const double* __restrict__ X,
                                               int project, int want_h, double* __restrict__ hc,
                                               double* __restrict__ gc, int* err) {
  PSlot s[kMaxKappa];
  energy_slots(E, i, s);
  double dl[3], gd[3], P[9];
  if (E.kind == K_INERTIA) {
    double p[3];
    point_position(E.dom, i, X, p);
    const double* xt = E.anchor + 3 * i;
    const double m = E.cdata[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      dl[k] = p[k] - xt[k];
      gd[k] = m * dl[k];
    }
    proj_rank1_3(m, 0.0, dl, 1.0, project != 0, P);
  } else {
    double p0[3], p1[3];
    int64_t l0, l1;
    const int c0 = union_decode(E.uni, E.pairs[2 * i], &l0);
    const int c1 = union_decode(E.uni, E.pairs[2 * i + 1], &l1);
    point_position(E.uni.child[c0], l0, X, p0);
    point_position(E.uni.child[c1], l1, X, p1);
#pragma unroll
    for (int k = 0; k < 3; ++k) dl[k] = p1[k] - p0[k];
    const double d = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
    const PairParams PP{E.prm[0], E.prm[1], E.prm[2], E.kind == K_REPULSIVE};
    double b, b1, b2;
    const int st = pair_b(d, PP, &b, &b1, &b2);
    if (st) atomicOr(err, st == 1 ? kErrLog : kErrDiv);
#pragma unroll
    for (int k = 0; k < 3; ++k) gd[k] = 2.0 * b1 * dl[k];
    proj_rank1_3(2.0 * b1, 4.0 * b2, dl, d, project != 0, P);
  }
  write_point_gradient(s, E.kappa, gd, gc + inst_goff(E, i));
  if (want_h) {
    UBlocks u;
    make_ublocks(s, E.kappa, u);
    write_point_blocks(u, P, hc + inst_hoff(E, i));
  }
}

__global__ void k_eval_point(EnergyDev E, const double* __restrict__ X, int project, int want_h,
                             double* __restrict__ hc, double* __restrict__ gc, int* err) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  point_instance(E, i, X, project, want_h, hc, gc, err);
}

// Point-triangle / edge-edge / point-edge barriers over a union of free and
// fixed points (ys_contact4.cuh): distance type on the current positions, the
// type's squared distance as a jet over the 3 A stencil coordinates, the
// point-point barrier's b(d) composed on it, then exactly the reference's
// assemble_local FullProject route (assembly.cpp:284-321): raw-slot gradient,
// local_compress, symmetrise, psd_project of the m x m block.
__device__ __forceinline__ void stencil_points(const EnergyDev& E, int64_t i, const double* __restrict__ X,
                                               double (*x)[3]) {
  for (int l = 0; l < E.arity; ++l) {
    int64_t loc;
    const int br = union_decode(E.uni, E.pairs[int64_t(E.arity) * i + l], &loc);
    point_position(E.uni.child[br], loc, X, x[l]);
  }
}

template <int A>
__global__ void __launch_bounds__(128) k_eval_contact(EnergyDev E, const double* __restrict__ X, int project,
                                                      int want_h, double* __restrict__ hc, double* __restrict__ gc,
                                                      int* err) {
  constexpr int N = 3 * A;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  double x[4][3];
  stencil_points(E, i, X, x);
  const ContactSel sel = classify_contact(E.kind, x);
  Jet<N> d;
  contact_dist2<N>(sel, x, d);
  const PairParams PP{E.prm[0], E.prm[1], E.prm[2], 0};
  double b, b1, b2;
  const int st = pair_b(d.v, PP, &b, &b1, &b2);
  if (st) atomicOr(err, st == 1 ? kErrLog : kErrDiv);
  PSlot s[kMaxKappa];
  energy_slots(E, i, s);
  // raw-slot gradient: g = b'(d) grad d
  double* go = gc + inst_goff(E, i);
  int o = 0;
  for (int l = 0; l < A; ++l) {
    if (s[l].gstart < 0) continue;
    for (int k = 0; k < 3; ++k) go[o + k] = b1 * d.g[3 * l + k];
    o += 3;
  }
  if (!want_h) return;
  UBlocks u;
  make_ublocks(s, A, u);
  int ub_of[4];
  for (int l = 0; l < A; ++l) {
    ub_of[l] = -1;
    for (int q = 0; q < u.nu; ++q)
      if (s[l].gstart >= 0 && u.gstart[q] == s[l].gstart) ub_of[l] = q;
  }
  const int m = 3 * u.nu;
  double Hc[144];
  for (int k = 0; k < m * m; ++k) Hc[k] = 0.0;
  // local_compress of H = b'(d) hess d + b''(d) grad d grad d^T (symmetric)
  for (int l = 0; l < A; ++l) {
    if (ub_of[l] < 0) continue;
    for (int lp = 0; lp < A; ++lp) {
      if (ub_of[lp] < 0) continue;
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q) {
          const int ir = 3 * l + r, iq = 3 * lp + q;
          Hc[(3 * ub_of[l] + r) * m + 3 * ub_of[lp] + q] += b1 * d.h[jh<N>(ir, iq)] + b2 * d.g[ir] * d.g[iq];
        }
    }
  }
  if (project) psd_project_dense(Hc, m);
  // ublock-pair blocks (a <= b), oriented so gstart(lo) <= gstart(hi)
  double* h = hc + inst_hoff(E, i);
  int64_t off = 0;
  for (int a = 0; a < u.nu; ++a)
    for (int bb = a; bb < u.nu; ++bb) {
      const bool sw = u.gstart[a] > u.gstart[bb];
      const int lo = sw ? bb : a, hi = sw ? a : bb;
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q) h[off + 3 * r + q] = Hc[(3 * lo + r) * m + 3 * hi + q];
      off += 9;
    }
}

__device__ __forceinline__ double contact_energy(const EnergyDev& E, int64_t i, const double* __restrict__ X,
                                                 int* err) {
  double x[4][3];
  stencil_points(E, i, X, x);
  const ContactSel sel = classify_contact(E.kind, x);
  const double d = contact_dist2_value(sel, x);
  const PairParams PP{E.prm[0], E.prm[1], E.prm[2], 0};
  double b, b1, b2;
  const int st = pair_b(d, PP, &b, &b1, &b2);
  if (st) atomicOr(err, st == 1 ? kErrLog : kErrDiv);
  return b;
}

// Many small energies of one kind (C3: 64 affine bodies, each with its own
// orthogonality and inertia energy of one / 27 instances) in one launch:
// thread t -> energy j (prefix[j] <= t < prefix[j + 1]), instance t - prefix[j].
// Each instance is computed exactly as by the per-energy kernels.
template <int KIND>  // 0: orthogonality, 1: point terms (k_eval_point)
__global__ void __launch_bounds__(128) k_eval_multi(const EnergyDev* __restrict__ Es, const int64_t* __restrict__ prefix,
                                                    int ne, const double* __restrict__ X, int project, int want_h,
                                                    double* __restrict__ hc, double* __restrict__ gc, int* err) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= prefix[ne]) return;
  int lo = 0, hi = ne - 1;  // last j with prefix[j] <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const EnergyDev& E = Es[lo];
  const int64_t i = t - prefix[lo];
  if (KIND == 0) ortho_instance(E, i, X, project, want_h, hc, gc);
  else point_instance(E, i, X, project, want_h, hc, gc, err);
}

// ---------------------------------------------------------------------------
// Energy-only kernels (line search): per-instance energy into out[i].

__global__ void k_energy(EnergyDev E, const double* __restrict__ X, double* __restrict__ out, int* err) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  double e = 0.0;
  switch (E.kind) {
    case K_SNH: {
      double x[12];
      int32_t gs[4];
      load_stencil(E, X, i, x, gs);
      const double* cd = E.cdata + 10 * i;
      double binv[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) binv[k] = cd[k];
      const SnhParams P{E.prm[0], E.prm[1], E.prm[2], E.prm[3]};
      if (!snh_energy(x, binv, cd[9], P, &e)) atomicOr(err, kErrLog);
      break;
    }
    case K_BENDING: {
      double x[12];
      int32_t gs[4];
      load_stencil(E, X, i, x, gs);
      if (bending_energy(x, E.cdata[i], &e)) atomicOr(err, kErrDiv);
      break;
    }
    case K_ORTHO: {
      double A[9];
      const double* q = X + E.startP + 9 * i;
#pragma unroll
      for (int k = 0; k < 9; ++k) A[k] = q[k];
      e = ortho_energy(A, E.prm[0]);
      break;
    }
    case K_INERTIA: {
      double p[3];
      point_position(E.dom, i, X, p);
      const double* xt = E.anchor + 3 * i;
      double d2 = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) d2 += (p[k] - xt[k]) * (p[k] - xt[k]);
      e = 0.5 * E.cdata[i] * d2;
      break;
    }
    case K_PT:
    case K_EE:
    case K_PE:
      e = contact_energy(E, i, X, err);
      break;
    default: {
      double p0[3], p1[3];
      int64_t l0, l1;
      const int c0 = union_decode(E.uni, E.pairs[2 * i], &l0);
      const int c1 = union_decode(E.uni, E.pairs[2 * i + 1], &l1);
      point_position(E.uni.child[c0], l0, X, p0);
      point_position(E.uni.child[c1], l1, X, p1);
      double d = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) d += (p1[k] - p0[k]) * (p1[k] - p0[k]);
      const PairParams PP{E.prm[0], E.prm[1], E.prm[2], E.kind == K_REPULSIVE};
      double b1, b2;
      const int st = pair_b(d, PP, &e, &b1, &b2);
      if (st) atomicOr(err, st == 1 ? kErrLog : kErrDiv);
      break;
    }
  }
  out[i] = e;
}

// Deterministic sum: fixed grid of partials, then one block sums them in order.
__global__ void k_sum_partials(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
  __shared__ double sm[kTB];
  double acc = 0.0;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
    acc += v[j];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w /= 2) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// ---------------------------------------------------------------------------
// FP64 FMA peak probe (the denominator of the local evaluation's roofline):
// 8 independent DFMA chains per thread, 8 resident CTAs of 256 per SM.
__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = double(threadIdx.x + k) * 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) t += x[k];
  if (t == 12345.0) out[0] = t;  // never true: keeps the chains alive
}

double fp64_probe(Context& c) {
  const int grid = sm_count() * 8, iters = 4096;
  c.scratch.resize(std::max<size_t>(c.scratch.n, 16));
  k_dfma_probe<<<grid, 256, 0, c.stream>>>(c.scratch.p, iters, 0.9999999, 1e-7);
  YS_LAUNCH_CHECK();
  return 2.0 * 8.0 * double(iters) * double(grid) * 256.0;  // flops per launch
}

// ---------------------------------------------------------------------------
// Assembly gather: unique block u = sum of its sorted contribution run.
__global__ void k_gather_h(const int64_t* __restrict__ seg, const uint32_t* __restrict__ perm,
                           const double* __restrict__ hc, int64_t u0, int64_t cnt, int rc,
                           const int64_t* __restrict__ voff, double* __restrict__ values) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= cnt * rc) return;
  const int64_t u = u0 + t / rc;
  const int e = int(t % rc);
  const int64_t j0 = seg[u], j1 = seg[u + 1];
  double acc = 0.0;
  for (int64_t j = j0; j < j1; ++j) acc += hc[perm[j] + e];
  values[voff[u] + e] = acc;
}

// The same with the blocks taken in a given order (k-th slot -> order[k]):
// the static group's blocks sorted by run length, so the lanes of a warp sum
// runs of similar length (in the structure's own (row, col) order every few
// blocks a ~24-long vertex run sits next to ~5-long edge runs and the warp
// waits for the longest).  Each block's sum keeps its left-to-right order:
// bit-identical values.  RC is a compile-time constant (no 64-bit division).
template <int RC>
__global__ void k_gather_h_ord(const int64_t* __restrict__ seg, const uint32_t* __restrict__ perm,
                               const double* __restrict__ hc, const int32_t* __restrict__ order, int nsel,
                               const int64_t* __restrict__ voff, double* __restrict__ values) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nsel * RC) return;
  const int k = t / RC, e = t - k * RC;
  const int64_t u = order[k];
  const int64_t j0 = seg[u], j1 = seg[u + 1];
  double acc = 0.0;
  // chunks of 8: the offsets, then the values, all in flight together; the
  // sum stays left to right
  for (int64_t j = j0; j < j1; j += 8) {
    uint32_t off[8];
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) off[q] = j + q < j1 ? perm[j + q] : 0u;
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = j + q < j1 ? hc[off[q] + e] : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (j + q < j1) acc += v[q];
  }
  values[voff[u] + e] = acc;
}

__global__ void k_run_keys(const int64_t* __restrict__ seg, int64_t u0, int64_t n, int wshift,
                           uint32_t* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  // sorted inside windows of 2^wshift consecutive blocks: similar lengths per warp,
  // while the window keeps the element contributions its blocks share close
  // (a global sort by length scattered them: 0.31 -> 0.41 ms at C5)
  const int64_t len = seg[u0 + k + 1] - seg[u0 + k];
  key[k] = (uint32_t(k >> wshift) << 10) | uint32_t(len < 1023 ? len : 1023);
  val[k] = int32_t(u0 + k);
}

// The same over a selection of unique blocks (the distributed solve's owned
// rows).
__global__ void k_gather_h_sel(const int64_t* __restrict__ seg, const uint32_t* __restrict__ perm,
                               const double* __restrict__ hc, const int32_t* __restrict__ sel, int64_t nsel, int rc,
                               const int64_t* __restrict__ voff, double* __restrict__ values) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nsel * rc) return;
  const int64_t u = sel[t / rc];
  const int e = int(t % rc);
  const int64_t j0 = seg[u], j1 = seg[u + 1];
  double acc = 0.0;
  for (int64_t j = j0; j < j1; ++j) acc += hc[perm[j] + e];
  values[voff[u] + e] = acc;
}

struct GroupView {
  const int32_t* gseg;
  const uint32_t* gperm;
  const double* gcontrib;
  const int32_t* diag_uid;
  const int64_t* seg;
  const uint32_t* perm;
  const double* hcontrib;
  const double* values;
  const int64_t* voff;
};

// Inverse by Gaussian elimination with partial pivoting (PartialPivLU, the
// algorithm behind Eigen's dynamic-size inverse(), solver.cpp:107).
template <int N>
__device__ __forceinline__ void lu_inverse(const double* B, double* inv) {
  double a[N * N];
  int piv[N];
#pragma unroll
  for (int k = 0; k < N * N; ++k) a[k] = B[k];
#pragma unroll
  for (int k = 0; k < N; ++k) piv[k] = k;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int p = k;
    double best = fabs(a[k * N + k]);
#pragma unroll
    for (int r = k + 1; r < N; ++r)
      if (fabs(a[r * N + k]) > best) {
        best = fabs(a[r * N + k]);
        p = r;
      }
    // swap rows k and p by static selects (a runtime row index would move a
    // and piv to local memory)
#pragma unroll
    for (int r = k + 1; r < N; ++r) {
      if (r == p) {
#pragma unroll
        for (int c = 0; c < N; ++c) {
          const double t = a[k * N + c];
          a[k * N + c] = a[r * N + c];
          a[r * N + c] = t;
        }
        const int t = piv[k];
        piv[k] = piv[r];
        piv[r] = t;
      }
    }
    const double d = a[k * N + k];
#pragma unroll
    for (int r = k + 1; r < N; ++r) {
      const double f = a[r * N + k] / d;
      a[r * N + k] = f;
#pragma unroll
      for (int c = k + 1; c < N; ++c) a[r * N + c] -= f * a[k * N + c];
    }
  }
  // solve L U X = P I column by column
#pragma unroll
  for (int col = 0; col < N; ++col) {
    double y[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double v = (piv[r] == col) ? 1.0 : 0.0;
#pragma unroll
      for (int c = 0; c < r; ++c) v -= a[r * N + c] * y[c];
      y[r] = v;
    }
#pragma unroll
    for (int r = N - 1; r >= 0; --r) {
      double v = y[r];
#pragma unroll
      for (int c = r + 1; c < N; ++c) v -= a[r * N + c] * y[c];
      y[r] = v / a[r * N + r];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) inv[r * N + col] = y[r];
  }
}

// BlockJacobiPreconditioner::build for one block (solver.cpp:98-120).
// Returns 0 ok, 1 identity fallback, 2 regularized, 3 singular.
template <int N>
__device__ __forceinline__ int jacobi_block_inverse(const double* B, double* inv) {
  bool zero = true;
  double nb = 0.0, tr = 0.0;
#pragma unroll
  for (int k = 0; k < N * N; ++k) {
    zero = zero && (fabs(B[k]) <= 0.0);
    nb += B[k] * B[k];
  }
#pragma unroll
  for (int k = 0; k < N; ++k) tr += B[k * N + k];
  if (zero) {
#pragma unroll
    for (int k = 0; k < N * N; ++k) inv[k] = (k % (N + 1) == 0) ? 1.0 : 0.0;
    return 1;
  }
  auto residual = [&](const double* M, const double* I) {
    double r = 0.0;
    bool finite = true;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) acc += M[i * N + k] * I[k * N + j];
        acc -= (i == j) ? 1.0 : 0.0;
        r += acc * acc;
        finite = finite && isfinite(I[i * N + j]);
      }
    return finite ? sqrt(r) : INFINITY;
  };
  lu_inverse<N>(B, inv);
  if (residual(B, inv) <= 1e-6 * (1.0 + sqrt(nb))) return 0;
  double eps = 1e-12 * tr / N;
  if (!(eps > 0.0)) eps = 1e-12;
  double reg[N * N];
  double nr = 0.0;
#pragma unroll
  for (int k = 0; k < N * N; ++k) {
    reg[k] = B[k] + ((k % (N + 1) == 0) ? eps : 0.0);
    nr += reg[k] * reg[k];
  }
  lu_inverse<N>(reg, inv);
  if (!(residual(reg, inv) <= 1e-3 * (1.0 + sqrt(nr)))) return 3;
  return 2;
}

template <int N, bool WITH_G = true>
__device__ __forceinline__ void block_row_work(int64_t b, const BlocksDev& B, const GroupView& S0,
                                               const GroupView& S1, double* G, double* diag, double* minv,
                                               int32_t* bflag, int want_h) {
  const int32_t st = B.start[b];
  if (WITH_G) {
  double acc[N];
#pragma unroll
  for (int k = 0; k < N; ++k) acc[k] = 0.0;
#pragma unroll
  for (int gi = 0; gi < 2; ++gi) {
    const GroupView& S = gi == 0 ? S0 : S1;
    if (!S.gseg) continue;
    const int32_t j0 = S.gseg[b], j1 = S.gseg[b + 1];
    for (int32_t j = j0; j < j1; ++j) {
      const double* src = S.gcontrib + (S.gperm[j] & 0x0FFFFFFFu);
#pragma unroll
      for (int k = 0; k < N; ++k) acc[k] += src[k];
    }
  }
#pragma unroll
  for (int k = 0; k < N; ++k) G[st + k] = acc[k];
  }
  if (!want_h) return;
  double blk[N * N];
#pragma unroll
  for (int k = 0; k < N * N; ++k) blk[k] = 0.0;
  if (S0.diag_uid) {
    const int32_t u = S0.diag_uid[b];
    if (u >= 0) {
      const double* v = S0.values + S0.voff[u];
#pragma unroll
      for (int k = 0; k < N * N; ++k) blk[k] = 0.0 + v[k];
    }
  }
  if (S1.diag_uid) {
    const int32_t u = S1.diag_uid[b];
    if (u >= 0) {
      const int64_t j0 = S1.seg[u], j1 = S1.seg[u + 1];
      for (int64_t j = j0; j < j1; ++j) {
        const double* src = S1.hcontrib + S1.perm[j];
#pragma unroll
        for (int k = 0; k < N * N; ++k) blk[k] += src[k];
      }
    }
  }
  double* dd = diag + B.voff[b];
#pragma unroll
  for (int k = 0; k < N * N; ++k) dd[k] = blk[k];
  bflag[b] = jacobi_block_inverse<N>(blk, minv + B.voff[b]);
}

// One launch per block-size class (block ids from the class list, or all
// blocks of a uniform layout).
template <int N>
__global__ void k_block_rows(BlocksDev B, const int32_t* __restrict__ list, int64_t nb, GroupView S0, GroupView S1,
                             double* G, double* diag, double* minv, int32_t* bflag, int want_h, int64_t b0 = 0) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nb) return;
  const int64_t b = list ? list[q] : b0 + q;
  block_row_work<N>(b, B, S0, S1, G, diag, minv, bflag, want_h);
}

// Uniform small blocks: the gradient gather with one thread per DoF (the
// row's N sums in parallel, each in block_row_work's order: bit-identical),
// then k_block_rows<N, false> for the diagonal block and its inverse.
template <int N>
__global__ void k_grad_rows(BlocksDev B, int64_t nb, GroupView S0, GroupView S1, double* G, int64_t b0) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nb * N) return;
  const int64_t b = b0 + t / N;
  const int k = int(t % N);
  double acc = 0.0;
#pragma unroll
  for (int gi = 0; gi < 2; ++gi) {
    const GroupView& S = gi == 0 ? S0 : S1;
    if (!S.gseg) continue;
    const int32_t j0 = S.gseg[b], j1 = S.gseg[b + 1];
    for (int32_t j = j0; j < j1; ++j) acc += S.gcontrib[(S.gperm[j] & 0x0FFFFFFFu) + k];
  }
  G[B.start[b] + k] = acc;
}

template <int N>
__global__ void k_block_rows_h(BlocksDev B, int64_t nb, GroupView S0, GroupView S1, double* diag, double* minv,
                               int32_t* bflag, int64_t b0) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nb) return;
  block_row_work<N, false>(b0 + q, B, S0, S1, nullptr, diag, minv, bflag, 1);
}

// Large blocks (affine bodies' 9x9 A block, 12x12): a warp per block row.
// Lane l accumulates entries l, l + 32, ... over the contributions in the same
// order as block_row_work (per entry the same sums, bit for bit); the row's
// whole diagonal block then goes through one lane's inverse.  (C3: 64 bodies
// each collecting ~100 contact blocks serially took 260 us in one thread.)
template <int N>
__global__ void k_block_rows_warp(BlocksDev B, const int32_t* __restrict__ list, int64_t nb, GroupView S0,
                                  GroupView S1, double* G, double* diag, double* minv, int32_t* bflag, int want_h) {
  const int64_t q = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nb) return;
  const int64_t b = list ? list[q] : q;
  const int32_t st = B.start[b];
  for (int k = lane; k < N; k += 32) {
    double acc = 0.0;
    for (int gi = 0; gi < 2; ++gi) {
      const GroupView& S = gi == 0 ? S0 : S1;
      if (!S.gseg) continue;
      const int32_t j0 = S.gseg[b], j1 = S.gseg[b + 1];
      for (int32_t j = j0; j < j1; ++j) acc += S.gcontrib[(S.gperm[j] & 0x0FFFFFFFu) + k];
    }
    G[st + k] = acc;
  }
  if (!want_h) return;
  double* dd = diag + B.voff[b];
  const int32_t u0 = S0.diag_uid ? S0.diag_uid[b] : -1;
  const int32_t u1 = S1.diag_uid ? S1.diag_uid[b] : -1;
  for (int k = lane; k < N * N; k += 32) {
    double v = 0.0;
    if (u0 >= 0) v = 0.0 + S0.values[S0.voff[u0] + k];
    if (u1 >= 0) {
      const int64_t j0 = S1.seg[u1], j1 = S1.seg[u1 + 1];
      for (int64_t j = j0; j < j1; ++j) v += S1.hcontrib[S1.perm[j] + k];
    }
    dd[k] = v;
  }
  __syncwarp();
  if (lane == 0) {
    double blk[N * N];
#pragma unroll
    for (int k = 0; k < N * N; ++k) blk[k] = dd[k];
    bflag[b] = jacobi_block_inverse<N>(blk, minv + B.voff[b]);
  }
}

// ---------------------------------------------------------------------------
// Host orchestration

static void check_err(Context& c) {
  int h = 0;
  YS_CUDA(cudaMemcpyAsync(&h, c.errflag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  YS_CUDA(cudaStreamSynchronize(c.stream));
  if (h) {
    c.errflag.zero(c.stream);
    if (h & kErrLog) fail(YS_ERR_NUMERICAL, "log of non-positive value");
    fail(YS_ERR_NUMERICAL, "division by zero");
  }
}

static GroupView group_view(Structure& st, bool present) {
  GroupView v{};
  if (!present) return v;
  v.gseg = st.gseg.p;
  v.gperm = st.gperm.p;
  v.gcontrib = st.gcontrib.p;
  v.diag_uid = st.diag_uid.p;
  v.seg = st.seg.p;
  v.perm = st.perm.p;
  v.hcontrib = st.hcontrib.p;
  v.values = st.values.p;
  v.voff = st.voff.p;
  return v;
}

void ctx_block_rows(Context& c, bool want_h);

static void record(Context& c, int idx) {
  if (c.profiling) YS_CUDA(cudaEventRecord(c.ev[idx], c.stream));
}

// only: -1 every energy, 0 the static group's, 1 the dynamic group's; s: the
// stream to launch on (default: the context stream).  The pass-B counters are
// zeroed by the call that evaluates the static group (the stencil energies).
// part: -1 every selected energy, 0 / 1 only those with an even / odd index
// (two streams share the static energies; the caller zeroes the counters).
void ctx_eval_all(Context& c, bool project, bool with_hessian, int only, cudaStream_t s, int part, bool zero_counts) {
  if (!s) s = c.stream;
  // evd_count: [0, n) indefinite elements per energy, [n, 2n) of those the
  // Jacobi fallback projects
  c.evd_count.resize(std::max(c.evd_count.n, 2 * c.energies.size()));
  if (only != 1 && zero_counts) c.evd_count.zero(s);
  // every stencil energy gets its own compacted-list / M range, so pass B can
  // run once for all energies of a kind after their pass A
  int64_t evd_total = 0;
  std::vector<int64_t> evd_base(c.energies.size(), 0);
  for (size_t id = 0; id < c.energies.size(); ++id) {
    const Energy& e = c.energies[id];
    if ((e.kind == K_SNH || e.kind == K_BENDING) && e.n > 0) {
      evd_base[id] = evd_total;
      evd_total += e.n;
    }
  }
  c.evd_m.resize(std::max(c.evd_m.n, size_t(kMStride * evd_total)));
  c.evd_list.resize(std::max(c.evd_list.n, size_t(evd_total)));
  c.evd_fblist.resize(std::max(c.evd_fblist.n, size_t(evd_total)));
  const bool pass_b = with_hessian && project;
  // pass B runs once per batch of up to kStencilBatch energies of one kind
  // after their pass A (one grid-stride launch, no per-energy tails): with the
  // clamped-eigenpair projection batching all C5 bodies is faster (eval 1.89
  // -> 1.72 ms); round 1's Jacobi pass B lost L2 residency of M when batched.
  constexpr int64_t kBatchElems = int64_t(1) << 40;
  const unsigned gb = unsigned(sm_count() * 4);
  std::vector<size_t> pending;
  int pending_kind = -1;
  int64_t pending_n = 0;
  auto flush = [&]() {
    if (pending.empty()) return;
    StencilBatch B{};
    B.n = int(pending.size());
    for (int j = 0; j < B.n; ++j) {
      Energy& e = c.energies[pending[j]];
      B.e[j] = energy_dev(c, e);
      B.hc[j] = c.S[e.dynamic ? 1 : 0].hcontrib.p;
      B.count[j] = c.evd_count.p + pending[j];
      B.base[j] = evd_base[pending[j]];
      B.fbcount[j] = c.evd_count.p + c.energies.size() + pending[j];
      B.fblist[j] = c.evd_fblist.p + evd_base[pending[j]];
    }
    if (c.evd_mode == 0) {
      // every indefinite element through the Jacobi EVD
      if (pending_kind == 0)
        k_eval_stencil_b_batch<0><<<gb, 128, 0, s>>>(B, c.evd_list.p, c.evd_m.p);
      else
        k_eval_stencil_b_batch<1><<<gb, 128, 0, s>>>(B, c.evd_list.p, c.evd_m.p);
      YS_LAUNCH_CHECK();
      ++c.launches;
    } else {
      // the dynamic shared-memory opt-in is per device (a process may hold
      // contexts on several devices)
      static std::atomic<uint64_t> attr_devices{0};
      const size_t smem = size_t(kProjSlots) * kProjStride * sizeof(double);
      const uint64_t bit = uint64_t(1) << (c.device & 63);
      if (!(attr_devices.load() & bit)) {
        YS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_eval_stencil_b_tri<0>),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        YS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_eval_stencil_b_tri<1>),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_devices.fetch_or(bit);
      }
      const unsigned gt = unsigned(sm_count() * 3);
      // per-thread reflector scratch; the two static-evaluation streams get
      // separate halves
      const size_t per = size_t(kProjScratch) * gt * kProjStride;
      c.evd_scratch.resize(std::max(c.evd_scratch.n, 2 * per));
      double* scr = c.evd_scratch.p + (part == 1 ? per : 0);
      if (pending_kind == 0) {
        k_eval_stencil_b_tri<0><<<gt, kProjStride, smem, s>>>(B, c.evd_list.p, c.evd_m.p, scr, c.evd_mode == 2);
        k_eval_stencil_b_fallback<0><<<sm_count(), 128, 0, s>>>(B, c.evd_list.p, c.evd_m.p);
      } else {
        k_eval_stencil_b_tri<1><<<gt, kProjStride, smem, s>>>(B, c.evd_list.p, c.evd_m.p, scr, c.evd_mode == 2);
        k_eval_stencil_b_fallback<1><<<sm_count(), 128, 0, s>>>(B, c.evd_list.p, c.evd_m.p);
      }
      YS_LAUNCH_CHECK();
      c.launches += 2;
    }
    pending.clear();
    pending_n = 0;
  };
  std::vector<size_t> multi[2][2];  // [group][0: orthogonality, 1: point-term inertia]
  for (size_t id = 0; id < c.energies.size(); ++id) {
    Energy& e = c.energies[id];
    if (e.n == 0 || e.kappa == 0) continue;
    if ((only == 0 && e.dynamic) || (only == 1 && !e.dynamic)) continue;
    if (part >= 0 && int(id % 2) != part) continue;
    Structure& st = c.S[e.dynamic ? 1 : 0];
    EnergyDev E = energy_dev(c, e);
    const int proj = project ? 1 : 0, wh = with_hessian ? 1 : 0;
    switch (e.kind) {
      case K_SNH:
      case K_BENDING: {
        unsigned int* cnt = c.evd_count.p + id;
        const unsigned ga = grid_for(e.n, 128);
        int32_t* lst = c.evd_list.p + evd_base[id];
        double* mb = c.evd_m.p + kMStride * evd_base[id];
        const int kind = e.kind == K_SNH ? 0 : 1;
        // distributed solve: only the instances touching this rank's rows
        const bool part_sel = c.dist.kind && c.dist.nranks > 1 && c.dist.have_static &&
                              id < c.dist.nsel_e.size() && c.dist.nsel_e[id] >= 0;
        const int32_t* sel = part_sel ? c.dist.sel[id].p : nullptr;
        const int64_t nsel = part_sel ? c.dist.nsel_e[id] : e.n;
        const unsigned gsel = grid_for(nsel, 128);
        if (kind == 0)
          k_eval_stencil_a<0><<<gsel, 128, 0, s>>>(E, c.X.p, proj, wh, st.hcontrib.p, st.gcontrib.p, c.errflag.p, cnt,
                                                   lst, mb, sel, nsel);
        else
          k_eval_stencil_a<1><<<gsel, 128, 0, s>>>(E, c.X.p, proj, wh, st.hcontrib.p, st.gcontrib.p, c.errflag.p, cnt,
                                                   lst, mb, sel, nsel);
        (void)ga;
        YS_LAUNCH_CHECK();
        if (pass_b) {
          if (pending_kind != kind || int(pending.size()) == kStencilBatch) flush();
          pending_kind = kind;
          pending.push_back(id);
          pending_n += e.n;
          if (pending_n >= kBatchElems) flush();
        }
        break;
      }
      case K_ORTHO:
        multi[e.dynamic ? 1 : 0][0].push_back(id);  // launched batched below
        continue;
      case K_INERTIA:
        if (c.domains[e.domain].kind == YS_POINTS_FREE) {
          k_eval_inertia_free<<<grid_for(e.n, 128), 128, 0, s>>>(E, c.X.p, proj, wh, st.hcontrib.p, st.gcontrib.p);
        } else {
          multi[e.dynamic ? 1 : 0][1].push_back(id);
          continue;
        }
        break;
      case K_PT:
      case K_EE:
        k_eval_contact<4><<<grid_for(e.n, 128), 128, 0, s>>>(E, c.X.p, proj, wh, st.hcontrib.p, st.gcontrib.p,
                                                              c.errflag.p);
        break;
      case K_PE:
        k_eval_contact<3><<<grid_for(e.n, 128), 128, 0, s>>>(E, c.X.p, proj, wh, st.hcontrib.p, st.gcontrib.p,
                                                              c.errflag.p);
        break;
      default:
        if (E.uni.kappa_u == 1)
          k_eval_pair_free<<<grid_for(e.n, 128), 128, 0, s>>>(E, c.X.p, proj, wh, st.hcontrib.p, st.gcontrib.p,
                                                              c.errflag.p);
        else
          k_eval_point<<<grid_for(e.n, 128), 128, 0, s>>>(E, c.X.p, proj, wh, st.hcontrib.p, st.gcontrib.p,
                                                          c.errflag.p);
    }
    YS_LAUNCH_CHECK();
    ++c.launches;
  }
  flush();
  // many small energies of one kind and group: one launch (k_eval_multi)
  {
    const int proj = project ? 1 : 0, wh = with_hessian ? 1 : 0;
    std::vector<EnergyDev> es;
    std::vector<int64_t> pre;
    struct Launch {
      int kind, group;
      size_t e0, ne, p0;
    };
    std::vector<Launch> ls;
    for (int g = 0; g < 2; ++g)
      for (int kind = 0; kind < 2; ++kind) {
        if (multi[g][kind].empty()) continue;
        Launch l{kind, g, es.size(), multi[g][kind].size(), pre.size()};
        int64_t acc = 0;
        for (size_t id : multi[g][kind]) {
          es.push_back(energy_dev(c, c.energies[id]));
          pre.push_back(acc);
          acc += c.energies[id].n;
        }
        pre.push_back(acc);
        ls.push_back(l);
      }
    if (!ls.empty()) {
      const int slot = only == 1 ? 1 : part == 1 ? 2 : 0;
      DevBuf<unsigned char>& me = c.multi_e[slot];
      DevBuf<int64_t>& mp = c.multi_pre[slot];
      me.resize(es.size() * sizeof(EnergyDev));
      mp.resize(pre.size());
      YS_CUDA(cudaMemcpyAsync(me.p, es.data(), es.size() * sizeof(EnergyDev), cudaMemcpyHostToDevice, s));
      YS_CUDA(cudaMemcpyAsync(mp.p, pre.data(), pre.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      const EnergyDev* de = reinterpret_cast<const EnergyDev*>(me.p);
      for (const Launch& l : ls) {
        Structure& st = c.S[l.group];
        const int64_t total = pre[l.p0 + l.ne];
        if (total == 0) continue;
        const unsigned grid = grid_for(total, 128);
        if (l.kind == 0)
          k_eval_multi<0><<<grid, 128, 0, s>>>(de + l.e0, mp.p + l.p0, int(l.ne), c.X.p, proj, wh,
                                               st.hcontrib.p, st.gcontrib.p, c.errflag.p);
        else
          k_eval_multi<1><<<grid, 128, 0, s>>>(de + l.e0, mp.p + l.p0, int(l.ne), c.X.p, proj, wh,
                                               st.hcontrib.p, st.gcontrib.p, c.errflag.p);
        YS_LAUNCH_CHECK();
        ++c.launches;
      }
    }
  }
}

// Run-length order of the static structure's blocks (once per structure; own
// temporaries: this runs on the side stream next to the dynamic rebuild).
static void build_gather_order(Structure& st, int wshift, cudaStream_t s) {
  st.gorder.clear();
  st.gorder.resize(st.groups.size());
  for (size_t gi = 0; gi < st.groups.size(); ++gi) {
    const auto& g = st.groups[gi];
    const int64_t cnt = g[3];
    if (cnt == 0) continue;
    DevBuf<uint32_t> kin, kout;
    DevBuf<int32_t> vin;
    DevBuf<char> tmp;
    kin.resize(size_t(cnt));
    kout.resize(size_t(cnt));
    vin.resize(size_t(cnt));
    st.gorder[gi].resize(size_t(cnt));
    k_run_keys<<<grid_for(cnt), kTB, 0, s>>>(st.seg.p, g[2], cnt, wshift, kin.p, vin.p);
    YS_LAUNCH_CHECK();
    size_t bytes = 0;
    YS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin.p, kout.p, vin.p, st.gorder[gi].p, int(cnt), 0, 32, s));
    tmp.resize(std::max<size_t>(bytes, 1));
    YS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, kin.p, kout.p, vin.p, st.gorder[gi].p, int(cnt), 0, 32, s));
    YS_CUDA(cudaStreamSynchronize(s));
  }
  st.gorder_valid = true;
}

void ctx_gather_all(Context& c, int only, cudaStream_t s) {
  if (!s) s = c.stream;
  for (int w = 0; w < 2; ++w) {
    if (only >= 0 && w != only) continue;
    Structure& st = c.S[w];
    const bool dsel = w == 0 && c.dist.kind && c.dist.nranks > 1 && c.dist.have_static &&
                      c.dist.ngsel.size() == st.groups.size();
    for (size_t gi = 0; gi < st.groups.size(); ++gi) {
      const auto& g = st.groups[gi];
      const int rc = int(g[0] * g[1]);
      const int64_t cnt = g[3];
      if (cnt == 0) continue;
      if (dsel) {  // only the blocks touching this rank's rows
        const int64_t ns = c.dist.ngsel[gi];
        if (ns > 0)
          k_gather_h_sel<<<grid_for(ns * rc), kTB, 0, s>>>(st.seg.p, st.perm.p, st.hcontrib.p, c.dist.gsel[gi].p, ns,
                                                           rc, st.voff.p, st.values.p);
        YS_LAUNCH_CHECK();
        ++c.launches;
        continue;
      }
      if (w == 0 && rc == 9 && cnt * 9 < (int64_t(1) << 31)) {
        if (!st.gorder_valid) build_gather_order(st, c.gather_wshift, s);
        k_gather_h_ord<9><<<grid_for(cnt * 9), kTB, 0, s>>>(st.seg.p, st.perm.p, st.hcontrib.p, st.gorder[gi].p,
                                                           int(cnt), st.voff.p, st.values.p);
      } else {
        k_gather_h<<<grid_for(cnt * rc), kTB, 0, s>>>(st.seg.p, st.perm.p, st.hcontrib.p, g[2], cnt, rc, st.voff.p,
                                                      st.values.p);
      }
      YS_LAUNCH_CHECK();
      ++c.launches;
    }
  }
}

// only / join: the static energies were already launched on the second
// stream (ys_minimize_step); evaluate the dynamic ones here, then wait for
// the join event before the gather.
void ctx_assemble(Context& c, bool project, bool with_hessian, int only, cudaEvent_t join, bool check) {
  if (c.seen_epoch != c.epoch)
    fail(YS_ERR_VALIDATION, "dynamic structures are stale after resize_dynamic; call refresh_dynamic()");
  record(c, 1);
  ctx_eval_all(c, project, with_hessian, only);
  record(c, 2);
  if (with_hessian) {
    ctx_gather_all(c, only);  // (only == 1: the static group was gathered on the second stream)
    if (join) YS_CUDA(cudaStreamWaitEvent(c.stream, join, 0));
  } else {
    if (join) YS_CUDA(cudaStreamWaitEvent(c.stream, join, 0));  // Engine::assemble zeroes both stores and the diagonal (engine.cpp:50-53)
    for (int w = 0; w < 2; ++w) c.S[w].values.zero(c.stream);
    c.diag.zero(c.stream);
  }
  record(c, 3);
  ctx_block_rows(c, with_hessian);
  record(c, 4);
  if (check) check_err(c);
  c.assembled = true;
  c.assembled_h = with_hessian;
}

void ctx_block_rows(Context& c, bool want_h) {
  const BlocksDev B = blocks_view(c);
  const GroupView S0 = group_view(c.S[0], true), S1 = group_view(c.S[1], true);
  const int wh = want_h ? 1 : 0;
  // distributed solve (uniform 3x3 only): the rank's rows [b0, b0 + nb)
  const bool own = c.dist.kind && c.dist.nranks > 1 && c.dist.have_static && c.rc_classes.size() == 1;
  const int64_t b0 = own ? c.dist.sbounds[size_t(c.dist.rank)] : 0;
  for (size_t k = 0; k < c.rc_classes.size(); ++k) {
    const int32_t* list = c.rc_classes.size() == 1 ? nullptr : c.rc_lists[k].p;
    const int64_t nb = own ? c.dist.sbounds[size_t(c.dist.rank) + 1] - b0
                           : (c.rc_classes.size() == 1 ? c.NB : int64_t(c.rc_lists[k].n));
    if (nb == 0) continue;
    const unsigned g = grid_for(nb, 128);
    if (c.rc_classes[k] == 9 || c.rc_classes[k] == 12) {
      const unsigned gw = grid_for(nb * 32, 128);
      if (c.rc_classes[k] == 9)
        k_block_rows_warp<9><<<gw, 128, 0, c.stream>>>(B, list, nb, S0, S1, c.G.p, c.diag.p, c.minv.p, c.bflag.p, wh);
      else
        k_block_rows_warp<12><<<gw, 128, 0, c.stream>>>(B, list, nb, S0, S1, c.G.p, c.diag.p, c.minv.p, c.bflag.p, wh);
      YS_LAUNCH_CHECK();
      ++c.launches;
      continue;
    }
    if (c.rc_classes[k] == 3 && !list) {
      k_grad_rows<3><<<grid_for(nb * 3, 128), 128, 0, c.stream>>>(B, nb, S0, S1, c.G.p, b0);
      YS_LAUNCH_CHECK();
      ++c.launches;
      if (want_h) {
        k_block_rows_h<3><<<g, 128, 0, c.stream>>>(B, nb, S0, S1, c.diag.p, c.minv.p, c.bflag.p, b0);
        YS_LAUNCH_CHECK();
        ++c.launches;
      }
      continue;
    }
#define YS_ROWS(N)                                                                                            \
  case N:                                                                                                     \
    k_block_rows<N><<<g, 128, 0, c.stream>>>(B, list, nb, S0, S1, c.G.p, c.diag.p, c.minv.p, c.bflag.p, wh, b0); \
    break;
    switch (c.rc_classes[k]) {
      YS_ROWS(1)
      YS_ROWS(2)
      YS_ROWS(3)
      YS_ROWS(4)
      YS_ROWS(6)
      YS_ROWS(9)
      YS_ROWS(12)
      default:
        fail(YS_ERR_INTERNAL, "unsupported target block size");
    }
#undef YS_ROWS
    YS_LAUNCH_CHECK();
    ++c.launches;
  }
}

// Flags of the last preconditioner build -> regularized count / singular error.
// Preconditioner flags summarised on the device (regularised count, first
// singular block) and read back together with the evaluation error flag: one
// 12-byte copy and one synchronisation instead of downloading NB flags.
__global__ void k_flag_summary(const int32_t* __restrict__ fl, int64_t nb, int* out) {
  int reg = 0, first = INT_MAX;
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nb; b += int64_t(gridDim.x) * blockDim.x) {
    const int f = fl[b];
    reg += (f == 1 || f == 2);
    if ((f == 3 || f == 4) && b < first) first = int(b);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    reg += __shfl_xor_sync(0xffffffffu, reg, off);
    first = min(first, __shfl_xor_sync(0xffffffffu, first, off));
  }
  if ((threadIdx.x & 31) == 0) {
    if (reg) atomicAdd(out, reg);
    if (first != INT_MAX) atomicMin(out + 1, first);
  }
}

static void* pinned_buf(Context& c) {
  if (!c.pinned) YS_CUDA(cudaMallocHost(&c.pinned, 65536));
  return c.pinned;
}

__global__ void k_flag_init(int* out) {
  out[0] = 0;
  out[1] = INT_MAX;
}

void ctx_build_preconditioner(Context& c) {
  cudaStream_t s = c.stream;
  c.flagsum.resize(4);
  k_flag_init<<<1, 1, 0, s>>>(c.flagsum.p + 1);
  // distributed solve: only this rank's rows are assembled (and solved)
  int64_t f0 = 0, f1 = c.NB;
  if (c.dist.kind && c.dist.nranks > 1 && c.dist.have_static) {
    f0 = c.dist.sbounds[size_t(c.dist.rank)];
    f1 = c.dist.sbounds[size_t(c.dist.rank) + 1];
  }
  k_flag_summary<<<int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(f1 - f0, kTB), 4 * sm_count()))), kTB, 0, s>>>(
      c.bflag.p + f0, f1 - f0, c.flagsum.p + 1);
  YS_LAUNCH_CHECK();
  YS_CUDA(cudaMemcpyAsync(c.flagsum.p, c.errflag.p, sizeof(int), cudaMemcpyDeviceToDevice, s));
  int* h = reinterpret_cast<int*>(pinned_buf(c));
  YS_CUDA(cudaMemcpyAsync(h, c.flagsum.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  if (h[0]) {  // evaluation error of the assembly (check_err, deferred to here by ys_minimize_step)
    c.errflag.zero(s);
    if (h[0] & kErrLog) fail(YS_ERR_NUMERICAL, "log of non-positive value");
    fail(YS_ERR_NUMERICAL, "division by zero");
  }
  if (h[2] != INT_MAX) {
    const int64_t b = f0 + h[2];
    int32_t st = 0, rc = 0;
    YS_CUDA(cudaMemcpyAsync(&st, c.bstart.p + b, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaMemcpyAsync(&rc, c.brc.p + b, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaStreamSynchronize(s));
    fail(YS_ERR_NUMERICAL, "diagonal block at DoF range [" + std::to_string(st) + ", " + std::to_string(st + rc) +
                               ") is singular");
  }
  c.regularized = h[1];
}

double ctx_total_energy(Context& c, double* per_energy) {
  cudaStream_t s = c.stream;
  const int nparts = 256;
  c.partials.resize(std::max<size_t>(c.partials.n, size_t(nparts) * (c.energies.size() + 1)));
  std::vector<double> parts(size_t(nparts) * c.energies.size(), 0.0);
  for (size_t id = 0; id < c.energies.size(); ++id) {
    Energy& e = c.energies[id];
    const int64_t n = e.pairset >= 0 ? c.pairsets[e.pairset].n : e.n;
    if (n == 0) continue;
    c.scratch.resize(std::max<size_t>(c.scratch.n, size_t(n)));
    EnergyDev E = energy_dev(c, e);
    E.n = n;  // Evaluator::total reads the current instance count (eval.cpp:394-401)
    k_energy<<<grid_for(n, 128), 128, 0, s>>>(E, c.X.p, c.scratch.p, c.errflag.p);
    YS_LAUNCH_CHECK();
    k_sum_partials<<<nparts, kTB, 0, s>>>(c.scratch.p, n, c.partials.p + id * nparts);
    YS_LAUNCH_CHECK();
  }
  if (!c.energies.empty())
    YS_CUDA(cudaMemcpyAsync(parts.data(), c.partials.p, parts.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  check_err(c);
  double sum = 0.0;
  for (size_t id = 0; id < c.energies.size(); ++id) {
    const int64_t n = c.energies[id].pairset >= 0 ? c.pairsets[c.energies[id].pairset].n : c.energies[id].n;
    double t = 0.0;
    if (n > 0)
      for (int k = 0; k < nparts; ++k) t += parts[id * nparts + k];
    if (per_energy) per_energy[id] = t;
    sum += t;
  }
  return sum;
}

}  // namespace ys
