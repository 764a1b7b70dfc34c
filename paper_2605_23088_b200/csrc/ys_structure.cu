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
#include <cub/cub.cuh>

#include <algorithm>

#include "ys_device.cuh"

namespace ys {

namespace {

constexpr int kTB = 256;

struct Cnt4 {
  uint32_t h, g, d, s;
};
struct Cnt4Sum {
  __host__ __device__ Cnt4 operator()(const Cnt4& a, const Cnt4& b) const {
    return {a.h + b.h, a.g + b.g, a.d + b.d, a.s + b.s};
  }
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
  for (int k = 0; k < E.kappa; ++k) {
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
  for (int k = 0; k < E.kappa; ++k) {
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
  if (!flag[j]) return;
  const int32_t u = incl[j] - 1;
  ukey[u] = k[j];
  if (seg) seg[u] = j;
  ghead[u] = (j == 0 || (k[j] >> 56) != (k[j - 1] >> 56)) ? 1 : 0;
}

__global__ void k_set_i64(int64_t* p, int64_t idx, int64_t v) { p[idx] = v; }

struct GroupDev {
  int32_t head;  // first unique block
  int32_t rows, cols, pad;
  int64_t value_start;
};

__global__ void k_block_attrs(const uint64_t* ukey, int64_t nu, const GroupDev* grp, int ng, int32_t* row,
                              int32_t* col, int8_t* br, int8_t* bc, int64_t* voff, const int32_t* dof2block,
                              int32_t* diag_uid) {
  const int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  int lo = 0, hi = ng;  // last group with head <= u
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (grp[mid].head <= u) lo = mid; else hi = mid;
  }
  const GroupDev g = grp[lo];
  const uint64_t k = ukey[u];
  const int32_t r = int32_t(key_row(k)), c = int32_t(key_col(k));
  row[u] = r;
  col[u] = c;
  br[u] = int8_t(g.rows);
  bc[u] = int8_t(g.cols);
  voff[u] = g.value_start + (u - g.head) * int64_t(g.rows) * g.cols;
  if (diag_uid && r == c) diag_uid[dof2block[r]] = int32_t(u);
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n) p[j] = v;
}

// seg[b] = lower_bound(keys, starts[b]) (starts == nullptr: search b itself); seg[nb] = n.
__global__ void k_lower_bound_blocks(const uint32_t* keys, int64_t n, const int32_t* bstart, int64_t nb,
                                     int32_t* seg) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb && bstart) {
    seg[b] = int32_t(n);
    return;
  }
  // block-id keys: rowptr[nb] = first sentinel (diagonal blocks emit one entry)
  const uint32_t v = bstart ? uint32_t(bstart[b]) : uint32_t(b);
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (keys[mid] < v) lo = mid + 1; else hi = mid;
  }
  seg[b] = int32_t(lo);
}

// SpMV plan entries: block u contributes to block-row(row) and, if off-diagonal,
// transposed to block-row(col).
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
    key[2 * u + 1] = 0xFFFFFFFFu;  // sorts past every block row
    ent[2 * u + 1] = 0xFFFFFFFFu;
  }
}

__global__ void k_max_row(const int32_t* rowptr, int64_t nb, int32_t* out) {
  __shared__ int32_t sm[kTB];
  int32_t m = 0;
  for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) m = max(m, rowptr[b + 1] - rowptr[b]);
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w /= 2) {
    if (threadIdx.x < w) sm[threadIdx.x] = max(sm[threadIdx.x], sm[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

template <class F>
void cub_run(Context& c, F f) {
  size_t bytes = 0;
  YS_CUDA(f(nullptr, bytes));
  c.cubtmp.resize(std::max<size_t>(bytes, 1));
  YS_CUDA(f(c.cubtmp.p, bytes));
}

}  // namespace

EnergyDev energy_dev(Context& c, Energy& e);  // ys_capi.cu

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

void build_structure_from_keys(Context& c, Structure& st, DevBuf<uint64_t>& keys, DevBuf<uint32_t>& payload,
                               int64_t n, int64_t total_dofs, const BlocksDev& blocks, bool plan) {
  cudaStream_t s = c.stream;
  st.n_contrib = n;
  st.groups.clear();
  st.n_blocks = st.n_values = 0;
  st.all33 = true;
  st.checksum_valid = false;
  st.diag_uid.resize(size_t(blocks.nb));
  if (blocks.nb) k_fill_i32<<<grid_for(blocks.nb), kTB, 0, s>>>(st.diag_uid.p, blocks.nb, -1);
  if (n == 0) {
    st.seg.resize(1);
    k_set_i64<<<1, 1, 0, s>>>(st.seg.p, 0, 0);
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
  int32_t nu32 = 0;
  YS_CUDA(cudaMemcpyAsync(&nu32, inc + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  const int64_t nu = nu32;
  c.ukey.resize(nu);
  st.seg.resize(nu + 1);
  c.ghead.resize(nu);
  k_emit_unique<<<grid_for(n), kTB, 0, s>>>(kout, fl, inc, n, c.ukey.p, st.seg.p, c.ghead.p);
  k_set_i64<<<1, 1, 0, s>>>(st.seg.p, nu, n);
  // shape-group heads -> host
  std::vector<int32_t> gh = c.ghead.to_host(s);
  std::vector<int32_t> heads;
  for (int64_t u = 0; u < nu; ++u)
    if (gh[u]) heads.push_back(int32_t(u));
  std::vector<uint64_t> hkeys(heads.size());
  for (size_t g = 0; g < heads.size(); ++g)
    YS_CUDA(cudaMemcpyAsync(&hkeys[g], c.ukey.p + heads[g], sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  std::vector<GroupDev> gd(heads.size());
  int64_t value_acc = 0;
  for (size_t g = 0; g < heads.size(); ++g) {
    const int64_t start = heads[g];
    const int64_t end = g + 1 < heads.size() ? heads[g + 1] : nu;
    const int rows = key_rows(hkeys[g]), cols = key_cols(hkeys[g]);
    st.groups.push_back({rows, cols, start, end - start, value_acc});
    gd[g] = GroupDev{int32_t(start), rows, cols, 0, value_acc};
    if (rows != 3 || cols != 3) st.all33 = false;
    value_acc += (end - start) * rows * cols;
  }
  st.n_blocks = nu;
  st.n_values = value_acc;
  c.grpbuf.upload(reinterpret_cast<const unsigned char*>(gd.data()), gd.size() * sizeof(GroupDev), s);
  const GroupDev* dgrp = reinterpret_cast<const GroupDev*>(c.grpbuf.p);
  st.row.resize(nu);
  st.col.resize(nu);
  st.br.resize(nu);
  st.bc.resize(nu);
  st.voff.resize(nu);
  k_block_attrs<<<grid_for(nu), kTB, 0, s>>>(c.ukey.p, nu, dgrp, int(gd.size()), st.row.p, st.col.p, st.br.p,
                                             st.bc.p, st.voff.p, blocks.dof2block, st.diag_uid.p);
  YS_LAUNCH_CHECK();
  st.values.resize(size_t(value_acc));
  st.values.zero(s);
  (void)total_dofs;
  (void)plan;
}

void build_spmv_plan(Context& c, Structure& st, const BlocksDev& blocks) {
  cudaStream_t s = c.stream;
  const int64_t nu = st.n_blocks;
  st.sp_rowptr.resize(size_t(blocks.nb + 1));
  if (nu == 0) {
    st.sp_ent.resize(0);
    k_fill_i32<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(st.sp_rowptr.p, blocks.nb + 1, 0);
    st.max_row_len = 0;
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
  // row pointers over block-row ids 0..nb (keys are block ids, not DoFs)
  k_lower_bound_blocks<<<grid_for(blocks.nb + 1), kTB, 0, s>>>(ko, ne, nullptr, blocks.nb, st.sp_rowptr.p);
  YS_LAUNCH_CHECK();
  // the valid entries are the prefix [0, rowptr[nb])
  c.heads.resize(1);
  k_max_row<<<1, kTB, 0, s>>>(st.sp_rowptr.p, blocks.nb, c.heads.p);
  YS_CUDA(cudaMemcpyAsync(&st.max_row_len, c.heads.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
}

void ctx_build_group(Context& c, int which) {
  cudaStream_t s = c.stream;
  Structure& st = c.S[which];
  const BlocksDev blocks = blocks_view(c);
  int64_t H = 0, G = 0, D = 0, S = 0;
  std::vector<int> ids;
  for (size_t i = 0; i < c.energies.size(); ++i)
    if (c.energies[i].dynamic == (which == 1)) ids.push_back(int(i));

  DevBuf<Cnt4> cnt, ex;
  for (int id : ids) {
    Energy& e = c.energies[id];
    if (e.pairset >= 0) e.n = c.pairsets[e.pairset].n;
    set_uniform_strides(c, e);
    e.hbase = H; e.gbase = G; e.dbase = D; e.sbase = S;
    e.slots.resize(size_t(e.n * e.kappa));
    e.m.resize(size_t(e.n));
    e.hsize = e.gsize = e.ndest = e.nslot = 0;
    e.built = true;
    if (e.n == 0 || e.kappa == 0) {
      if (e.n) YS_CUDA(cudaMemsetAsync(e.m.p, 0, e.n * sizeof(int32_t), s));
      continue;
    }
    if (e.uniform) {
      e.hoff.release(); e.goff.release(); e.doff.release(); e.soff.release();
      EnergyDev E = energy_dev(c, e);
      k_slots_count<<<grid_for(e.n, 128), 128, 0, s>>>(E, nullptr);
      YS_LAUNCH_CHECK();
      e.hsize = e.n * e.hstride; e.gsize = e.n * e.gstride;
      e.ndest = e.n * e.dstride; e.nslot = e.n * e.sstride;
    } else {
      cnt.resize(e.n);
      ex.resize(e.n);
      e.hoff.resize(e.n); e.goff.resize(e.n); e.doff.resize(e.n); e.soff.resize(e.n);
      EnergyDev E = energy_dev(c, e);
      E.hoff = E.goff = E.doff = E.soff = nullptr;
      k_slots_count<<<grid_for(e.n, 128), 128, 0, s>>>(E, cnt.p);
      YS_LAUNCH_CHECK();
      Cnt4* ci = cnt.p;
      Cnt4* co = ex.p;
      const int ni = int(e.n);
      cub_run(c, [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveScan(t, b, ci, co, Cnt4Sum{}, Cnt4{0, 0, 0, 0}, ni, s);
      });
      Cnt4 last_ex, last_c;
      YS_CUDA(cudaMemcpyAsync(&last_ex, co + e.n - 1, sizeof(Cnt4), cudaMemcpyDeviceToHost, s));
      YS_CUDA(cudaMemcpyAsync(&last_c, ci + e.n - 1, sizeof(Cnt4), cudaMemcpyDeviceToHost, s));
      k_split_offsets<<<grid_for(e.n), kTB, 0, s>>>(co, e.n, e.hoff.p, e.goff.p, e.doff.p, e.soff.p);
      YS_CUDA(cudaStreamSynchronize(s));
      e.hsize = int64_t(last_ex.h) + last_c.h;
      e.gsize = int64_t(last_ex.g) + last_c.g;
      e.ndest = int64_t(last_ex.d) + last_c.d;
      e.nslot = int64_t(last_ex.s) + last_c.s;
    }
    H += e.hsize; G += e.gsize; D += e.ndest; S += e.nslot;
  }
  if (H >= (int64_t(1) << 32)) fail(YS_ERR_INTERNAL, "local Hessian buffer exceeds 2^32 doubles");
  if (G >= (int64_t(1) << 28)) fail(YS_ERR_INTERNAL, "local gradient buffer exceeds 2^28 doubles");
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
  build_structure_from_keys(c, st, c.k_in, c.p_in, D, c.s, blocks, true);

  // gradient plan: stable sort of slot contributions by gstart
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
  build_spmv_plan(c, st, blocks);
  YS_CUDA(cudaStreamSynchronize(s));
}

uint64_t structure_checksum(Context& c, Structure& st, int64_t total_dofs) {
  if (st.checksum_valid) return st.checksum;
  std::vector<int32_t> row = st.row.to_host(c.stream);
  std::vector<int32_t> col = st.col.to_host(c.stream);
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
