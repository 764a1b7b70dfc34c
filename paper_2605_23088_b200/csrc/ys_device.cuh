// ys_device.cuh — per-instance placement logic shared by the structure build
// and the evaluation kernels.
//
// Reference: the placement walk (index_gen.cpp:77-122) over the layout the
// differentiator derives (diff.cpp:549-630), then make_pattern
// (assembly.cpp:201-219) and the ublock pair enumeration of
// build_global_structure / build_instance_plans (assembly.cpp:223-264).
#pragma once

#include "ys_context.cuh"
#include "ys_terms.cuh"

namespace ys {

constexpr int kMaxKappa = 4;

// Everything a kernel needs to know about one energy group.
struct EnergyDev {
  int32_t kind, kappa, width, mode;
  int64_t n;
  const int32_t* conn;   // SNH / bending
  const double* cdata;   // SNH: Binv+vol (10/inst); bending: c=k*w*l0 (1/inst); inertia: mass
  const double* anchor;  // inertia x_tilde
  int32_t startP;        // SNH/bending position target start; ortho amat target start
  int32_t arity;         // stencil energies over a union: points per instance
  DomainDev dom;         // inertia domain
  UnionDev uni;          // pair energies
  const int32_t* pairs;  // pair energies: 2n union-global ids
  double prm[6];
  // structure / outputs
  DSlot* slots;
  int32_t* m;
  const uint32_t* hoff;
  const uint32_t* goff;
  const uint32_t* doff;
  const uint32_t* soff;
  uint32_t hstride, gstride, dstride, sstride;
  int64_t hbase, gbase, dbase, sbase;
};

// Position of point `i` of a domain (sim.cpp:245-247 for affine bodies:
// position = affine.matmul(rest) + trans).  Products and sums are rounded
// explicitly (no FMA contraction) in the reference's evaluation order so the
// proximity test of refresh_dynamic_pairs reproduces the CPU bit for bit.
__device__ __forceinline__ void point_position(const DomainDev& d, int64_t i, const double* X, double p[3]) {
  if (d.kind == YS_POINTS_FREE) {
    const double* q = X + d.startA + 3 * i;
    p[0] = q[0]; p[1] = q[1]; p[2] = q[2];
  } else if (d.kind == YS_POINTS_AFFINE) {
    const int64_t b = d.v2b[i];
    const double* A = X + d.startA + 9 * b;
    const double* t = X + d.startB + 3 * b;
    const double* r = d.rest + 3 * i;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double acc = __dmul_rn(A[3 * k + 0], r[0]);
      acc = __dadd_rn(acc, __dmul_rn(A[3 * k + 1], r[1]));
      acc = __dadd_rn(acc, __dmul_rn(A[3 * k + 2], r[2]));
      p[k] = __dadd_rn(acc, t[k]);
    }
  } else {
    const double* q = d.fixed + 3 * i;
    p[0] = q[0]; p[1] = q[1]; p[2] = q[2];
  }
}

// One placement slot plus the linear map from the slot's DoFs to the point:
// p_c = sum_j rho[j] * dof[c * (len/3) + j]   (len 3: rho[0]; len 9: rho[0..2]).
struct PSlot {
  int32_t gstart;  // -1 = pad
  int32_t len;
  int32_t col;
  double rho[3];
};

// Slots of point `local` of domain d at column base `col` with sign `sg`
// (index_gen.cpp:77-122 walk of DataSlot / Seq[JoinRep(A), JoinRep(t)]).
__device__ __forceinline__ int point_slots(const DomainDev& d, int64_t local, int col, double sg, PSlot* out) {
  if (d.kind == YS_POINTS_FREE) {
    out[0] = PSlot{int32_t(d.startA + 3 * local), 3, col, {sg, 0.0, 0.0}};
    return 1;
  }
  if (d.kind == YS_POINTS_AFFINE) {
    const int64_t b = d.v2b[local];
    const double* r = d.rest + 3 * local;
    out[0] = PSlot{int32_t(d.startA + 9 * b), 9, col, {sg * r[0], sg * r[1], sg * r[2]}};
    out[1] = PSlot{int32_t(d.startB + 3 * b), 3, col + 9, {sg, 0.0, 0.0}};
    return 2;
  }
  return 0;
}

// PrimitiveUnion::decode (scene.cpp:227-237): last child whose offset <= g,
// skipping empty children that share an offset.
__device__ __forceinline__ int union_decode(const UnionDev& u, int64_t g, int64_t* local) {
  int br = 0;
  for (int c = 1; c < u.nchild; ++c)
    if (u.offsets[c] <= g) br = c;  // std::upper_bound(...) - 1
  while (u.child[br].n == 0 && br + 1 < u.nchild) ++br;
  *local = g - u.offsets[br];
  return br;
}

// All kappa slots of instance i (pads have gstart -1).
__device__ __forceinline__ void energy_slots(const EnergyDev& E, int64_t i, PSlot* s) {
#pragma unroll
  for (int k = 0; k < kMaxKappa; ++k) s[k] = PSlot{-1, 0, 0, {0.0, 0.0, 0.0}};
  switch (E.kind) {
    case K_SNH:
    case K_BENDING: {
#pragma unroll
      for (int l = 0; l < 4; ++l)
        s[l] = PSlot{int32_t(E.startP + 3 * E.conn[4 * i + l]), 3, 3 * l, {1.0, 0.0, 0.0}};
      break;
    }
    case K_ORTHO:
      s[0] = PSlot{int32_t(E.startP + 9 * i), 9, 0, {1.0, 0.0, 0.0}};
      break;
    case K_INERTIA:
      point_slots(E.dom, i, 0, 1.0, s);
      break;
    case K_PT:
    case K_EE:
    case K_PE: {  // stencil energies over a union of free / fixed points (kappa_u = 1)
      for (int l = 0; l < E.arity && l < kMaxKappa; ++l) {
        int64_t local;
        const int br = union_decode(E.uni, E.pairs[int64_t(E.arity) * i + l], &local);
        point_slots(E.uni.child[br], local, 3 * l, 1.0, s + l);
      }
      break;
    }
    default: {  // pair energies: JoinRep(pp2v, UnionSel)
      const int ku = E.uni.kappa_u;
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        int64_t local;
        const int br = union_decode(E.uni, E.pairs[2 * i + l], &local);
        point_slots(E.uni.child[br], local, l * E.uni.width, l == 0 ? -1.0 : 1.0, s + l * ku);
      }
      break;
    }
  }
}

// make_pattern (assembly.cpp:201-219): unique gstarts in slot order; rho of
// merged slots is summed (local_compress sums their blocks).
struct UBlocks {
  int nu;
  int m;
  int32_t gstart[kMaxKappa];
  int32_t len[kMaxKappa];
  double rho[kMaxKappa][3];
};

__device__ __forceinline__ void make_ublocks(const PSlot* s, int kappa, UBlocks& u) {
  u.nu = 0;
  u.m = 0;
#pragma unroll
  for (int k = 0; k < kMaxKappa; ++k) {
    if (k >= kappa || s[k].gstart < 0) continue;
    int found = -1;
#pragma unroll
    for (int q = 0; q < kMaxKappa; ++q)
      if (q < u.nu && u.gstart[q] == s[k].gstart) found = q;
    if (found < 0) {
      found = u.nu++;
      u.gstart[found] = s[k].gstart;
      u.len[found] = s[k].len;
      u.rho[found][0] = u.rho[found][1] = u.rho[found][2] = 0.0;
      u.m += s[k].len;
    }
    u.rho[found][0] += s[k].rho[0];
    u.rho[found][1] += s[k].rho[1];
    u.rho[found][2] += s[k].rho[2];
  }
}

// BlockSparseHessian::BlockCoord ordering key (assembly.hpp:21-25):
// (rows, cols, row, col) lexicographic == numeric order of this packing.
__host__ __device__ __forceinline__ uint64_t block_key(int rows, int cols, int64_t row, int64_t col) {
  return (uint64_t(rows) << 60) | (uint64_t(cols) << 56) | (uint64_t(row) << 28) | uint64_t(col);
}
__host__ __device__ __forceinline__ int key_rows(uint64_t k) { return int(k >> 60); }
__host__ __device__ __forceinline__ int key_cols(uint64_t k) { return int((k >> 56) & 0xF); }
__host__ __device__ __forceinline__ int64_t key_row(uint64_t k) { return int64_t((k >> 28) & 0xFFFFFFF); }
__host__ __device__ __forceinline__ int64_t key_col(uint64_t k) { return int64_t(k & 0xFFFFFFF); }

// Per-instance offsets into the group buffers.
__device__ __forceinline__ int64_t inst_hoff(const EnergyDev& E, int64_t i) {
  return E.hbase + (E.hoff ? int64_t(E.hoff[i]) : int64_t(E.hstride) * i);
}
__device__ __forceinline__ int64_t inst_goff(const EnergyDev& E, int64_t i) {
  return E.gbase + (E.goff ? int64_t(E.goff[i]) : int64_t(E.gstride) * i);
}

// Writes the local blocks of a point-parameterised term (inertia, pair
// energies): block(lo, hi)[a][b] = P[c_a][c_b] rho_lo[j_a] rho_hi[j_b], dests in
// ublock-pair order (a <= b), oriented so gstart(lo) <= gstart(hi).
__device__ __forceinline__ void write_point_blocks(const UBlocks& u, const double P[9], double* h) {
  int64_t off = 0;
  for (int a = 0; a < u.nu; ++a)
    for (int b = a; b < u.nu; ++b) {
      const bool sw = u.gstart[a] > u.gstart[b];
      const int lo = sw ? b : a, hi = sw ? a : b;
      const int ll = u.len[lo], lh = u.len[hi];
      const int sl = ll / 3, sh = lh / 3;  // sub-dimension per component
      for (int r = 0; r < ll; ++r) {
        const int cr = r / sl, jr = r % sl;
        const double fr = u.rho[lo][jr];
        for (int q = 0; q < lh; ++q) {
          const int cq = q / sh, jq = q % sh;
          h[off + r * lh + q] = P[3 * cr + cq] * fr * u.rho[hi][jq];
        }
      }
      off += ll * lh;
    }
}

// Gradient per raw slot: g_slot[r] = rho_slot[j_r] * gdelta[c_r].
__device__ __forceinline__ void write_point_gradient(const PSlot* s, int kappa, const double gd[3], double* g) {
  int64_t off = 0;
  for (int k = 0; k < kappa; ++k) {
    if (s[k].gstart < 0) continue;
    const int len = s[k].len, sub = len / 3;
    for (int r = 0; r < len; ++r) g[off + r] = s[k].rho[r % sub] * gd[r / sub];
    off += len;
  }
}

}  // namespace ys
