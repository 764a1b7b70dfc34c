// ys_structure.cu — device structure build of one energy group.
//
// Reference: compute_energy_tables (assembly.cpp:185-196) ->
// build_global_structure (223-246) -> BlockSparseHessian::build (22-61) ->
// build_instance_plans / value_offset (248-264, 63-81).  The reference sorts
// BlockCoord structs with std::sort and binary-searches every destination.
// Here each (instance, ublock pair) emits one 64-bit key whose numeric order
// is the BlockCoord order, a stable radix sort carries the contribution's
// buffer offset along, and run boundaries give (a) the unique coordinates,
// shape groups and value offsets and (b) the assembly plan: the contributions
// of unique block k are the k-th run, already in (energy, instance) order —
// exactly the order of the reference's serial scatter (assembly.cpp:346-372).
//
// The build runs on the device end to end and synchronises with the host
// twice: once for the buffer sizes of non-uniform (pair) energies and once
// for the small structure summary (unique count, shape groups).  The dynamic
// group is rebuilt every Newton iteration, so nothing here allocates once the
// capacities have grown.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "ys_device.cuh"

namespace ys {

namespace {

constexpr int kTB = 256;
constexpr int kMaxGroups = 64;

struct Cnt4 {
  uint32_t h, g, d, s;
};
struct Cnt4Sum {
  __host__ __device__ Cnt4 operator()(const Cnt4& a, const Cnt4& b) const {
    return {a.h + b.h, a.g + b.g, a.d + b.d, a.s + b.s};
  }
};

// Device-side summary of one structure build (read back once).
struct Summary {
  int64_t nu;            // unique blocks
  int64_t ng;            // shape groups
  int64_t n_values;
  int64_t groups[kMaxGroups][5];  // rows, cols, coord_start, count, value_start
};

inline unsigned grid_for(int64_t n, int tb = kTB) { return unsigned(std::max<int64_t>(1, ceil_div(n, tb))); }

// Pass 1: slot table, compressed size and buffer counts per instance.
__global__ void k_slots_count(EnergyDev E, Cnt4* cnt) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  PSlot s[kMaxKappa];
  energy_slots(E, i, s);
  UBlocks u;
  make_ublocks(s, E.kappa, u);
  Cnt4 c{0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < kMaxKappa; ++k) {
    if (k >= E.kappa) break;
    const bool pad = s[k].gstart < 0;
    E.slots[i * E.kappa + k] =
        DSlot{pad ? 0 : s[k].gstart + 1, int16_t(pad ? 0 : s[k].len), int16_t(pad ? 0 : s[k].col)};
    if (!pad) {
      c.g += s[k].len;
      c.s += 1;
    }
  }
  for (int a = 0; a < u.nu; ++a)
    for (int b = a; b < u.nu; ++b) {
      c.h += u.len[a] * u.len[b];
      c.d += 1;
    }
  E.m[i] = u.m;
  if (cnt) cnt[i] = c;
}

__global__ void k_split_offsets(const Cnt4* ex, int64_t n, uint32_t* h, uint32_t* g, uint32_t* d, uint32_t* s) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  h[i] = ex[i].h;
  g[i] = ex[i].g;
  d[i] = ex[i].d;
  s[i] = ex[i].s;
}

__global__ void k_total4(const Cnt4* ex, const Cnt4* cnt, int64_t last, Cnt4* out) {
  *out = Cnt4{ex[last].h + cnt[last].h, ex[last].g + cnt[last].g, ex[last].d + cnt[last].d, ex[last].s + cnt[last].s};
}

// Pass 2: sort keys with the contribution offsets as payload.
__global__ void k_fill_keys(EnergyDev E, uint64_t* keys, uint32_t* pay, uint32_t* gkeys, uint32_t* gpay) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  PSlot s[kMaxKappa];
  energy_slots(E, i, s);
  UBlocks u;
  make_ublocks(s, E.kappa, u);
  int64_t hoff = inst_hoff(E, i);
  int64_t doff = E.dbase + (E.doff ? int64_t(E.doff[i]) : int64_t(E.dstride) * i);
  for (int a = 0; a < u.nu; ++a)
    for (int b = a; b < u.nu; ++b) {
      const bool sw = u.gstart[a] > u.gstart[b];
      const int lo = sw ? b : a, hi = sw ? a : b;
      keys[doff] = block_key(u.len[lo], u.len[hi], u.gstart[lo], u.gstart[hi]);
      pay[doff] = uint32_t(hoff);
      ++doff;
      hoff += u.len[lo] * u.len[hi];
    }
  int64_t goff = inst_goff(E, i);
  int64_t soff = E.sbase + (E.soff ? int64_t(E.soff[i]) : int64_t(E.sstride) * i);
#pragma unroll
  for (int k = 0; k < kMaxKappa; ++k) {
    if (k >= E.kappa) break;
    if (s[k].gstart < 0) continue;
    gkeys[soff] = uint32_t(s[k].gstart);
    gpay[soff] = uint32_t(goff) | (uint32_t(s[k].len) << 28);
    ++soff;
    goff += s[k].len;
  }
}

__global__ void k_run_flags(const uint64_t* k, int64_t n, int32_t* flag) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  flag[j] = (j == 0 || k[j] != k[j - 1]) ? 1 : 0;
}

// Run heads -> unique key, segment start, shape-group head flag.
__global__ void k_emit_unique(const uint64_t* k, const int32_t* flag, const int32_t* incl, int64_t n,
                              uint64_t* ukey, int64_t* seg, int32_t* ghead) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (j == n - 1) seg[incl[j]] = n;  // terminal
  if (!flag[j]) return;
  const int32_t u = incl[j] - 1;
  ukey[u] = k[j];
  seg[u] = j;
  ghead[u] = (j == 0 || (k[j] >> 56) != (k[j - 1] >> 56)) ? 1 : 0;
}

// Group heads (at most kMaxGroups) collected in parallel, then one thread
// orders them and writes the group table.
__global__ void k_collect_heads(const int32_t* ghead, const int32_t* incl, int64_t n, int32_t* heads,
                                unsigned int* nheads) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= incl[n - 1] || !ghead[u]) return;
  const unsigned k = atomicAdd(nheads, 1u);
  if (k < kMaxGroups) heads[k] = int32_t(u);
}

__global__ void k_summarise(const uint64_t* ukey, const int32_t* incl, int64_t n, int32_t* heads,
                            const unsigned int* nheads, Summary* out) {
  const int64_t nu = incl[n - 1];
  const int64_t ng = *nheads;
  out->nu = nu;
  out->ng = ng;
  if (ng > kMaxGroups) return;
  for (int64_t a = 1; a < ng; ++a)  // insertion sort of <= 64 heads
    for (int64_t b = a; b > 0 && heads[b - 1] > heads[b]; --b) {
      const int32_t t = heads[b];
      heads[b] = heads[b - 1];
      heads[b - 1] = t;
    }
  int64_t acc = 0;
  for (int64_t g = 0; g < ng; ++g) {
    const int64_t start = heads[g], end = g + 1 < ng ? heads[g + 1] : nu;
    out->groups[g][0] = key_rows(ukey[start]);
    out->groups[g][1] = key_cols(ukey[start]);
    out->groups[g][2] = start;
    out->groups[g][3] = end - start;
    out->groups[g][4] = acc;
    acc += (end - start) * out->groups[g][0] * out->groups[g][1];
  }
  out->n_values = acc;
}

__global__ void k_block_attrs(const uint64_t* ukey, const Summary* sm, int32_t* row, int32_t* col, int8_t* br,
                              int8_t* bc, int64_t* voff, const int32_t* dof2block, int32_t* diag_uid) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= sm->nu || sm->ng > kMaxGroups) return;
  int g = 0;
  for (int q = 1; q < int(sm->ng); ++q)
    if (sm->groups[q][2] <= u) g = q;
  const int64_t rows = sm->groups[g][0], cols = sm->groups[g][1];
  const uint64_t k = ukey[u];
  const int32_t r = int32_t(key_row(k)), c = int32_t(key_col(k));
  row[u] = r;
  col[u] = c;
  br[u] = int8_t(rows);
  bc[u] = int8_t(cols);
  voff[u] = sm->groups[g][4] + (u - sm->groups[g][2]) * rows * cols;
  if (diag_uid && r == c) diag_uid[dof2block[r]] = int32_t(u);
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n) p[j] = v;
}

// seg[b] = lower_bound(keys, starts[b]) (starts == nullptr: search b itself,
// which also makes seg[nb] exclude the sentinel keys); seg[nb] = n otherwise.
__global__ void k_lower_bound_blocks(const uint32_t* keys, int64_t n, const int32_t* bstart, int64_t nb,
                                     int32_t* seg) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb && bstart) {
    seg[b] = int32_t(n);
    return;
  }
  const uint32_t v = bstart ? uint32_t(bstart[b]) : uint32_t(b);
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (keys[mid] < v) lo = mid + 1; else hi = mid;
  }
  seg[b] = int32_t(lo);
}

// SpMV plan entries: block u contributes to block-row(row) and, if off-diagonal,
// transposed to block-row(col).  Unused halves of diagonal blocks sort last.
__global__ void k_spmv_entries(const int32_t* row, const int32_t* col, int64_t nu, const int32_t* dof2block,
                               uint32_t* key, uint32_t* ent) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  key[2 * u] = uint32_t(dof2block[row[u]]);
  ent[2 * u] = uint32_t(u);
  if (row[u] != col[u]) {
    key[2 * u + 1] = uint32_t(dof2block[col[u]]);
    ent[2 * u + 1] = uint32_t(u) | 0x80000000u;
  } else {
    key[2 * u + 1] = 0xFFFFFFFFu;
    ent[2 * u + 1] = 0xFFFFFFFFu;
  }
}

// Per entry: DoF of the other side; per block: positions of its two entries.
__global__ void k_spmv_post(const int32_t* ent, const int32_t* rowptr, int64_t nb, const int32_t* row,
                            const int32_t* col, int32_t* oth, int32_t* pos_n, int32_t* pos_t) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= rowptr[nb]) return;
  const uint32_t e = uint32_t(ent[j]);
  const uint32_t u = e & 0x7fffffffu;
  if (e >> 31) {
    oth[j] = row[u];
    pos_t[u] = int32_t(j);
  } else {
    oth[j] = col[u];
    pos_n[u] = int32_t(j);
    if (row[u] == col[u]) pos_t[u] = -1;
  }
}

// Off-diagonal blocks keyed by their column block (transposed row plan).
__global__ void k_tlist_keys(const int32_t* row, const int32_t* col, int64_t nu, const int32_t* dof2block,
                             uint32_t* key, uint32_t* val) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  key[u] = row[u] != col[u] ? uint32_t(dof2block[col[u]]) : 0xFFFFFFFFu;
  val[u] = uint32_t(u);
}

__global__ void k_tlist_fill(const uint32_t* sorted_u, const int32_t* trow, int64_t nb, const int32_t* row,
                             int2* tlist) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= trow[nb]) return;
  const int32_t u = int32_t(sorted_u[j]);
  tlist[j] = make_int2(u, row[u]);
}

template <class F>
void cub_run(Context& c, F f) {
  size_t bytes = 0;
  YS_CUDA(f(nullptr, bytes));
  c.cubtmp.resize(std::max<size_t>(bytes, 1));
  YS_CUDA(f(c.cubtmp.p, bytes));
}

void* pinned(Context& c) {
  if (!c.pinned) YS_CUDA(cudaMallocHost(&c.pinned, 65536));
  return c.pinned;
}

}  // namespace

EnergyDev energy_dev(Context& c, Energy& e);  // ys_assemble.cu

static void set_uniform_strides(Context& c, Energy& e) {
  e.uniform = true;
  switch (e.kind) {
    case K_SNH:
    case K_BENDING:
      e.hstride = 90; e.gstride = 12; e.dstride = 10; e.sstride = 4;
      break;
    case K_ORTHO:
      e.hstride = 81; e.gstride = 9; e.dstride = 1; e.sstride = 1;
      break;
    case K_INERTIA: {
      const Domain& d = c.domains[e.domain];
      if (d.kind == YS_POINTS_FREE) {
        e.hstride = 9; e.gstride = 3; e.dstride = 1; e.sstride = 1;
      } else if (d.kind == YS_POINTS_AFFINE) {
        e.hstride = 117; e.gstride = 12; e.dstride = 3; e.sstride = 2;
      } else {
        e.hstride = e.gstride = e.dstride = e.sstride = 0;
      }
      break;
    }
    default:
      e.uniform = false;
      e.hstride = e.gstride = e.dstride = e.sstride = 0;
  }
}

BlocksDev blocks_view(Context& c) {
  return BlocksDev{c.NB, c.bstart.p, c.brc.p, c.bvoff.p, c.dof2block.p};
}

// Sort + unique + shape groups + value offsets, all on the device; one
// small D2H summary at the end.
void build_structure_from_keys(Context& c, Structure& st, DevBuf<uint64_t>& keys, DevBuf<uint32_t>& payload,
                               int64_t n, int64_t total_dofs, const BlocksDev& blocks, bool plan) {
  (void)total_dofs;
  (void)plan;
  cudaStream_t s = c.stream;
  st.n_contrib = n;
  st.checksum_valid = false;
  st.gorder_valid = false;
  st.diag_uid.resize(size_t(blocks.nb));
  if (blocks.nb) k_fill_i32<<<grid_for(blocks.nb), kTB, 0, s>>>(st.diag_uid.p, blocks.nb, -1);
  if (n == 0) {
    st.groups.clear();
    st.n_blocks = st.n_values = 0;
    st.all33 = true;
    st.seg.resize(1);
    YS_CUDA(cudaMemsetAsync(st.seg.p, 0, sizeof(int64_t), s));
    st.values.resize(0);
    st.perm.resize(0);
    return;
  }
  if (n >= (int64_t(1) << 31)) fail(YS_ERR_INTERNAL, "structure build: too many block contributions");
  const int ni = int(n);
  c.k_out.resize(n);
  st.perm.resize(n);
  uint64_t* kin = keys.p;
  uint64_t* kout = c.k_out.p;
  uint32_t* pin = payload.p;
  uint32_t* pout = st.perm.p;
  cub_run(c, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, pin, pout, ni, 0, 64, s);
  });
  c.flags.resize(n);
  c.incl.resize(n);
  k_run_flags<<<grid_for(n), kTB, 0, s>>>(kout, n, c.flags.p);
  int32_t* fl = c.flags.p;
  int32_t* inc = c.incl.p;
  cub_run(c, [&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, fl, inc, ni, s); });
  // capacities: nu <= n
  c.ukey.resize(n);
  st.seg.resize(n + 1);
  c.ghead.resize(n);
  k_emit_unique<<<grid_for(n), kTB, 0, s>>>(kout, fl, inc, n, c.ukey.p, st.seg.p, c.ghead.p);
  c.summary.resize(std::max(c.summary.n, sizeof(Summary)));
  Summary* dsum = reinterpret_cast<Summary*>(c.summary.p);
  c.heads.resize(kMaxGroups + 1);
  unsigned int* nheads = reinterpret_cast<unsigned int*>(c.heads.p + kMaxGroups);
  YS_CUDA(cudaMemsetAsync(nheads, 0, sizeof(unsigned int), s));
  k_collect_heads<<<grid_for(n), kTB, 0, s>>>(c.ghead.p, inc, n, c.heads.p, nheads);
  k_summarise<<<1, 1, 0, s>>>(c.ukey.p, inc, n, c.heads.p, nheads, dsum);
  st.row.resize(n);
  st.col.resize(n);
  st.br.resize(n);
  st.bc.resize(n);
  st.voff.resize(n);
  k_block_attrs<<<grid_for(n), kTB, 0, s>>>(c.ukey.p, dsum, st.row.p, st.col.p, st.br.p, st.bc.p, st.voff.p,
                                            blocks.dof2block, st.diag_uid.p);
  YS_LAUNCH_CHECK();
  Summary* hsum = reinterpret_cast<Summary*>(pinned(c));
  YS_CUDA(cudaMemcpyAsync(hsum, dsum, sizeof(Summary), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  if (hsum->ng > kMaxGroups) fail(YS_ERR_INTERNAL, "too many block shapes in one structure");
  st.groups.clear();
  st.all33 = true;
  for (int64_t g = 0; g < hsum->ng; ++g) {
    st.groups.push_back({hsum->groups[g][0], hsum->groups[g][1], hsum->groups[g][2], hsum->groups[g][3],
                         hsum->groups[g][4]});
    if (hsum->groups[g][0] != 3 || hsum->groups[g][1] != 3) st.all33 = false;
  }
  st.n_blocks = hsum->nu;
  st.n_values = hsum->n_values;
  st.values.resize(size_t(st.n_values) + 4);  // +32 B: aligned-window loads of the last block
  st.values.n = size_t(st.n_values);
}

void build_spmv_plan(Context& c, Structure& st, const BlocksDev& blocks) {
  cudaStream_t s = c.stream;
  const int64_t nu = st.n_blocks;
  if (st.all33) {
    // Upper storage, u sorted by (row, col): block row R owns u in
    // [nrow[R], nrow[R+1]); its transposed contributions are tlist[trow[R] ..].
    st.nrow.resize(size_t(blocks.nb + 1));
    st.trow.resize(size_t(blocks.nb + 1));
    if (nu == 0) {
      k_fill_i32<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(st.nrow.p, blocks.nb + 1, 0);
      k_fill_i32<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(st.trow.p, blocks.nb + 1, 0);
      return;
    }
    k_lower_bound_blocks<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(reinterpret_cast<const uint32_t*>(st.row.p), nu,
                                                                 blocks.start, blocks.nb, st.nrow.p);
    c.gk_in.resize(nu);
    c.gp_in.resize(nu);
    c.gk_out.resize(nu);
    c.p_in.resize(std::max(c.p_in.n, size_t(nu)));
    k_tlist_keys<<<grid_for(nu), kTB, 0, s>>>(st.row.p, st.col.p, nu, blocks.dof2block, c.gk_in.p, c.gp_in.p);
    uint32_t* ki = c.gk_in.p;
    uint32_t* ko = c.gk_out.p;
    uint32_t* vi = c.gp_in.p;
    uint32_t* vo = c.p_in.p;
    const int nui = int(nu);
    cub_run(c, [&](void* t, size_t& b) { return cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, nui, 0, 32, s); });
    k_lower_bound_blocks<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(ko, nu, nullptr, blocks.nb, st.trow.p);
    st.tlist.resize(size_t(nu));
    k_tlist_fill<<<grid_for(nu), kTB, 0, s>>>(vo, st.trow.p, blocks.nb, st.row.p, st.tlist.p);
    YS_LAUNCH_CHECK();
    return;
  }
  st.sp_rowptr.resize(size_t(blocks.nb + 1));
  if (nu == 0) {
    st.sp_ent.resize(0);
    k_fill_i32<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(st.sp_rowptr.p, blocks.nb + 1, 0);
    return;
  }
  const int64_t ne = 2 * nu;
  c.gk_in.resize(ne);
  c.gp_in.resize(ne);
  c.gk_out.resize(ne);
  st.sp_ent.resize(ne);
  k_spmv_entries<<<grid_for(nu), kTB, 0, s>>>(st.row.p, st.col.p, nu, blocks.dof2block, c.gk_in.p, c.gp_in.p);
  uint32_t* ki = c.gk_in.p;
  uint32_t* ko = c.gk_out.p;
  uint32_t* vi = c.gp_in.p;
  uint32_t* vo = reinterpret_cast<uint32_t*>(st.sp_ent.p);
  const int nei = int(ne);
  cub_run(c, [&](void* t, size_t& b) { return cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, nei, 0, 32, s); });
  k_lower_bound_blocks<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(ko, ne, nullptr, blocks.nb, st.sp_rowptr.p);
  st.sp_oth.resize(ne);
  st.sp_pos_n.resize(nu);
  st.sp_pos_t.resize(nu);
  k_spmv_post<<<grid_for(ne), kTB, 0, s>>>(st.sp_ent.p, st.sp_rowptr.p, blocks.nb, st.row.p, st.col.p, st.sp_oth.p,
                                          st.sp_pos_n.p, st.sp_pos_t.p);
  YS_LAUNCH_CHECK();
}

void ctx_build_group(Context& c, int which) {
  cudaStream_t s = c.stream;
  Structure& st = c.S[which];
  const BlocksDev blocks = blocks_view(c);
  std::vector<int> ids;
  for (size_t i = 0; i < c.energies.size(); ++i)
    if (c.energies[i].dynamic == (which == 1)) ids.push_back(int(i));

  // ---- pass 1: slot tables and per-instance counts
  int64_t n_nonuni = 0;
  for (int id : ids) {
    Energy& e = c.energies[id];
    if (e.pairset >= 0) e.n = c.pairsets[e.pairset].n;
    set_uniform_strides(c, e);
    if (!e.uniform && e.kappa > 0) n_nonuni += e.n;
  }
  c.cnt4.resize(size_t(std::max<int64_t>(n_nonuni, 1)) * sizeof(Cnt4));
  c.ex4.resize(size_t(std::max<int64_t>(n_nonuni, 1)) * sizeof(Cnt4));
  c.summary.resize(std::max(c.summary.n, std::max(sizeof(Summary), (ids.size() + 1) * sizeof(Cnt4))));
  Cnt4* cnt = reinterpret_cast<Cnt4*>(c.cnt4.p);
  Cnt4* ex = reinterpret_cast<Cnt4*>(c.ex4.p);
  Cnt4* htot = reinterpret_cast<Cnt4*>(pinned(c));
  Cnt4* dtot = reinterpret_cast<Cnt4*>(c.summary.p);
  if ((ids.size() + 1) * sizeof(Cnt4) > 65536) fail(YS_ERR_INTERNAL, "too many energies in one group");
  int64_t nonuni_off = 0;
  bool need_sync = false;
  for (size_t q = 0; q < ids.size(); ++q) {
    Energy& e = c.energies[ids[q]];
    e.slots.resize(size_t(e.n * e.kappa));
    e.m.resize(size_t(e.n));
    e.built = true;
    if (e.n == 0 || e.kappa == 0) {
      if (e.n) YS_CUDA(cudaMemsetAsync(e.m.p, 0, e.n * sizeof(int32_t), s));
      continue;
    }
    if (e.uniform) {
      EnergyDev E = energy_dev(c, e);
      k_slots_count<<<grid_for(e.n, 128), 128, 0, s>>>(E, nullptr);
      YS_LAUNCH_CHECK();
    } else {
      e.hoff.resize(e.n); e.goff.resize(e.n); e.doff.resize(e.n); e.soff.resize(e.n);
      EnergyDev E = energy_dev(c, e);
      E.hoff = E.goff = E.doff = E.soff = nullptr;
      Cnt4* ci = cnt + nonuni_off;
      Cnt4* co = ex + nonuni_off;
      k_slots_count<<<grid_for(e.n, 128), 128, 0, s>>>(E, ci);
      YS_LAUNCH_CHECK();
      const int ni = int(e.n);
      cub_run(c, [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveScan(t, b, ci, co, Cnt4Sum{}, Cnt4{0, 0, 0, 0}, ni, s);
      });
      k_split_offsets<<<grid_for(e.n), kTB, 0, s>>>(co, e.n, e.hoff.p, e.goff.p, e.doff.p, e.soff.p);
      k_total4<<<1, 1, 0, s>>>(co, ci, e.n - 1, dtot + q);
      nonuni_off += e.n;
      need_sync = true;
    }
  }
  if (need_sync) {
    YS_CUDA(cudaMemcpyAsync(htot, dtot, ids.size() * sizeof(Cnt4), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaStreamSynchronize(s));
  }
  int64_t H = 0, G = 0, D = 0, S = 0;
  for (size_t q = 0; q < ids.size(); ++q) {
    Energy& e = c.energies[ids[q]];
    e.hbase = H; e.gbase = G; e.dbase = D; e.sbase = S;
    if (e.n == 0 || e.kappa == 0) {
      e.hsize = e.gsize = e.ndest = e.nslot = 0;
      continue;
    }
    if (e.uniform) {
      e.hsize = e.n * e.hstride; e.gsize = e.n * e.gstride;
      e.ndest = e.n * e.dstride; e.nslot = e.n * e.sstride;
    } else {
      e.hsize = htot[q].h; e.gsize = htot[q].g; e.ndest = htot[q].d; e.nslot = htot[q].s;
    }
    H += e.hsize; G += e.gsize; D += e.ndest; S += e.nslot;
  }
  if (H >= (int64_t(1) << 32)) fail(YS_ERR_INTERNAL, "local Hessian buffer exceeds 2^32 doubles");
  if (G >= (int64_t(1) << 28)) fail(YS_ERR_INTERNAL, "local gradient buffer exceeds 2^28 doubles");

  // ---- pass 2: keys
  st.hcontrib.resize(size_t(H));
  st.gcontrib.resize(size_t(G));
  st.n_gcontrib = S;
  c.k_in.resize(size_t(D));
  c.p_in.resize(size_t(D));
  c.gk_in.resize(size_t(S));
  c.gp_in.resize(size_t(S));
  for (int id : ids) {
    Energy& e = c.energies[id];
    if (e.n == 0 || e.kappa == 0) continue;
    EnergyDev E = energy_dev(c, e);
    k_fill_keys<<<grid_for(e.n, 128), 128, 0, s>>>(E, c.k_in.p, c.p_in.p, c.gk_in.p, c.gp_in.p);
    YS_LAUNCH_CHECK();
  }
  // gradient plan first (it owns gk_in/gp_in until sorted)
  st.gseg.resize(size_t(c.NB + 1));
  st.gperm.resize(size_t(S));
  c.gk_out.resize(size_t(S));
  if (S > 0) {
    uint32_t* ki = c.gk_in.p;
    uint32_t* ko = c.gk_out.p;
    uint32_t* vi = c.gp_in.p;
    uint32_t* vo = st.gperm.p;
    const int si = int(S);
    cub_run(c, [&](void* t, size_t& b) { return cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, si, 0, 32, s); });
  }
  k_lower_bound_blocks<<<grid_for(c.NB + 1), kTB, 0, s>>>(c.gk_out.p, S, c.bstart.p, c.NB, st.gseg.p);
  YS_LAUNCH_CHECK();
  // ---- pass 3: BSR structure + assembly plan + SpMV plan
  build_structure_from_keys(c, st, c.k_in, c.p_in, D, c.s, blocks, true);
  build_spmv_plan(c, st, blocks);
}

uint64_t structure_checksum(Context& c, Structure& st, int64_t total_dofs) {
  if (st.checksum_valid) return st.checksum;
  std::vector<int32_t> row(size_t(st.n_blocks)), col(size_t(st.n_blocks));
  st.row.download(row.data(), row.size(), c.stream);
  st.col.download(col.data(), col.size(), c.stream);
  YS_CUDA(cudaStreamSynchronize(c.stream));
  // FNV-1a exactly as BlockSparseHessian::structure_checksum (assembly.cpp:136-153)
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    h ^= v;
    h *= 1099511628211ull;
  };
  mix(uint64_t(total_dofs));
  for (auto& g : st.groups) {
    mix(uint64_t(g[0]));
    mix(uint64_t(g[1]));
    mix(uint64_t(g[3]));
  }
  for (int64_t i = 0; i < st.n_blocks; ++i) {
    mix(uint64_t(int64_t(row[i])));
    mix(uint64_t(int64_t(col[i])));
  }
  st.checksum = h;
  st.checksum_valid = true;
  return h;
}

}  // namespace ys
