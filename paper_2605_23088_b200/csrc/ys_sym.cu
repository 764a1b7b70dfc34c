// ys_sym.cu — the uniform-3x3 PCG over a symmetric band copy of H.
//
// The reference multiplies from upper storage (spmv_add, solver.cpp:10-82):
// each off-diagonal block (r, c) contributes B x_c to row r and B^T x_r to row
// c.  The sliced-ELL copy (ys_sell.cuh) streams every off-diagonal block twice
// (once per row it touches); here every static block is streamed ONCE per
// SpMV and both of its products are formed from the same on-chip copy.
//
// Layout (rebuilt per solve — the dynamic structure changes every Newton
// iteration: the layout right after the dynamic rebuild, the values in the
// solve):
//  * the block rows are split into G contiguous ranges, one CTA per SM,
//    balanced by static block count;  CTA b keeps p of the window
//    [R_b, R_b + W) — its own rows plus the band that follows (C5: 871 block
//    rows) — in shared memory, and an accumulator for its own rows;
//  * "near" blocks — the static own blocks of a row (the dynamic diagonal
//    block added into the static one) whose column lies in the window — go to
//    tiles of <= 64 rows / ~36 KB: an image of the blocks (SoA: 9 arrays of E
//    doubles), their column block ids, and the tile's transposed-product plan
//    (the off-diagonal blocks grouped by column block — "targets" — in entry
//    order);
//  * every other block (the contact blocks of the dynamic group, static blocks
//    beyond the window) is split into two half-entries — (target r, source c,
//    B) and (target c, source r, B^T) — sorted by target and cut into G equal
//    chunks: CTA b forms the products of its chunk and sums each run of equal
//    target (a contact face row collects ~20 pairs) into one slot;
//  * transposed products whose target lies beyond the CTA's own rows (the
//    band's tail) go to a slot per (tile, target); every row adds its slots —
//    numbered in row order — in phase B.
//
// Per iteration, phase A of CTA b:
//  1. its half-entries, chunk by chunk with every load in flight: products
//     into shared memory, then one thread per run sums it in order into its
//     slot (p_t . sum to the pHp partial — no extra barrier);
//  2. its tiles, through a 3-stage shared-memory ring filled by cp.async.bulk
//     (mbarrier complete_tx).  The images do not change during the solve, so
//     the ring keeps cycling over the CTA's tiles across iterations (a CTA
//     whose tiles fit the ring loads them once).  Per tile: 4 lanes per row
//     form B p_c for the row's blocks (registers) and store B^T p_r of the
//     off-diagonal ones to shared memory | barrier | one thread per target
//     sums its products in order into the accumulator or a slot | barrier |
//     rows finalise y = accumulator + own sum (fixed butterfly), pHp partial.
// Every row's sum has a fixed order (transposed products in tile order, its
// own blocks, then its slots in slot order): deterministic and bitwise
// reproducible.  Phase B keeps hp and z on chip; phase C writes p to shared
// memory and to global memory (the other CTAs' windows and half-entries).
// Three grid barriers per iteration, as the reference's recurrence
// (solver.cpp:151-200) needs: pHp, (r.r, r.z), and the p exchange.
#include <cub/cub.cuh>

#include <algorithm>

#include "ys_grid.cuh"

namespace ys {

namespace {

constexpr int kSymTB = 256;        // threads of every kernel here
constexpr int kSymRows = 64;       // block rows per tile (4 lanes each)
constexpr int kSymBudget = 36864;  // tile image budget (bound: 256 + 96 per block)
constexpr int kSymCap = 2048;      // blocks per tile (transposed-plan sort capacity)
constexpr int kSymHdr = 32;
constexpr int kSymVals = kSymHdr + 144;  // rowptr: 65 x uint16, padded
constexpr int kSymChunk = 1024;    // half-entries / slots per shared-memory chunk

__host__ __device__ __forceinline__ int al16(int x) { return (x + 15) & ~15; }
__host__ __device__ __forceinline__ int sym_off_cols(int E) { return kSymVals + al16(72 * E); }
__host__ __device__ __forceinline__ int sym_off_tg(int E) { return sym_off_cols(E) + al16(4 * E); }
__host__ __device__ __forceinline__ int sym_off_list(int E, int NT) { return sym_off_tg(E) + 8 * NT; }
__host__ __device__ __forceinline__ int sym_off_slot(int E, int NT, int NL) { return al16(sym_off_list(E, NT) + 2 * NL); }
__host__ __device__ __forceinline__ int sym_size(int E, int NT, int NL, int NS) {
  return al16(sym_off_slot(E, NT, NL) + 4 * NS);
}
// image offsets: the size bound 256 + 96 E per tile keeps them 16-byte aligned
__host__ __device__ __forceinline__ int64_t sym_toff(int64_t t, int64_t e0) { return 256 * t + 96 * e0; }

struct TileHdr {
  int32_t E, NT, NL, NS;  // blocks, targets, transposed entries, spill targets (a suffix of the targets)
  int32_t row0, nr;       // first block row, rows
  int32_t pad0, pad1;
};

// summary slots (int64, device side, read back by the host)
enum { SM_MAXROW = 0, SM_BAND, SM_MAXRANGE, SM_MAXTILE, SM_MAXE, SM_ERR, SM_N };

// Block row R: static own blocks [u0, u0 + n0) sorted by column; the dynamic
// diagonal block ud is merged into the static diagonal block (entry 0) when
// both exist; dynamic own blocks [u1, u1 + n1) (after a merged diagonal).
struct RowSrc {
  int32_t u0, n0, u1, n1, ud;
};

__device__ __forceinline__ bool has_diag3(const SpmvDev& S, int64_t R) {
  return S.nrow[R + 1] > S.nrow[R] && S.col[S.nrow[R]] == 3 * int32_t(R);
}

__device__ __forceinline__ RowSrc row_src(const SpmvDev& S0, const SpmvDev& S1, int has1, int64_t R) {
  RowSrc s;
  s.u0 = S0.nrow[R];
  s.n0 = S0.nrow[R + 1] - s.u0;
  const bool merge = has1 && has_diag3(S0, R) && has_diag3(S1, R);
  s.ud = merge ? S1.nrow[R] : -1;
  s.u1 = has1 ? S1.nrow[R] + (merge ? 1 : 0) : 0;
  s.n1 = has1 ? S1.nrow[R + 1] - s.u1 : 0;
  return s;
}

__device__ __forceinline__ void atomic_max64(int64_t* a, int64_t v) {
  atomicMax(reinterpret_cast<unsigned long long*>(a), static_cast<unsigned long long>(v));
}

// Static work per row (1 + static blocks) for the CTA partition; the longest
// static row and the static band (max c - r) into the summary.
__global__ void k_sym_count(SpmvDev S0, int64_t nb, int32_t* work, int64_t* summary) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int n = 0, band = 0;
  if (R < nb) {
    const int32_t u0 = S0.nrow[R];
    n = S0.nrow[R + 1] - u0;
    if (n > 0) band = S0.col[u0 + n - 1] / 3 - int(R);
    work[R] = 1 + n;
  } else if (R == nb) {
    work[R] = 0;
  }
  n = __reduce_max_sync(0xffffffffu, n);
  band = __reduce_max_sync(0xffffffffu, band);
  if ((threadIdx.x & 31) == 0) {
    atomic_max64(summary + SM_MAXROW, n);
    atomic_max64(summary + SM_BAND, band);
  }
}

// CTA ranges: bound b = first row R with wpre[R] >= b wpre[nb] / G (wpre: the
// exclusive prefix of the work per row).
__global__ void k_sym_ranges(const int32_t* wpre, int64_t nb, int G, int32_t* range, int64_t* summary) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > G) return;
  const int64_t tot = int64_t(wpre[nb]);
  auto bound = [&](int q) -> int64_t {
    if (q >= G) return nb;
    const int64_t target = tot * q / G;
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (int64_t(wpre[mid]) >= target) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  };
  const int64_t r0 = bound(b);
  range[b] = int32_t(r0);
  if (b < G) atomic_max64(summary + SM_MAXRANGE, bound(b + 1) - r0);
}

__device__ __forceinline__ int cta_of(const int32_t* range, int G, int64_t R) {
  int lo = 0, hi = G - 1;  // the CTA b with range[b] <= R < range[b + 1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (range[mid] <= R) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Per row: near blocks (the static own blocks inside the window: a prefix,
// columns are sorted) and half-entries (2 per other off-diagonal block, 1 per
// other diagonal block).
__global__ void k_sym_classify(SpmvDev S0, SpmvDev S1, int has1, int64_t nb, const int32_t* range, int G, int W,
                               int32_t* cn, int32_t* ch) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R > nb) return;
  if (R == nb) {
    cn[R] = 0;
    ch[R] = 0;
    return;
  }
  const int32_t lim = range[cta_of(range, G, R)] + W;
  const RowSrc s = row_src(S0, S1, has1, R);
  int near = 0, half = 0;
  for (int k = 0; k < s.n0; ++k) {
    const int32_t c = S0.col[s.u0 + k] / 3;
    if (c < lim) ++near;
    else half += 2;
  }
  for (int k = 0; k < s.n1; ++k) half += S1.col[s.u1 + k] / 3 == R ? 1 : 2;
  cn[R] = near;
  ch[R] = half;
}

// Greedy tiling of each CTA range (<= kSymRows rows, image bound <= kSymBudget):
// one CTA per range stages the near counts in shared memory, thread 0 walks them.
__global__ void __launch_bounds__(kSymTB) k_sym_walk(const int32_t* enoff, const int32_t* range, int32_t* tflag) {
  __shared__ int32_t cnt[4096];
  const int b = blockIdx.x;
  const int r0 = range[b], r1 = range[b + 1];
  int rows = 0, est = 0;
  for (int c0 = r0; c0 < r1; c0 += 4096) {
    const int n = min(4096, r1 - c0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) cnt[i] = enoff[c0 + i + 1] - enoff[c0 + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < n; ++i) {
        const int e = 96 * cnt[i];
        const bool start = (c0 + i == r0) || rows == kSymRows || est + e > kSymBudget - 256;
        if (start) {
          rows = 0;
          est = 0;
        }
        tflag[c0 + i] = start ? 1 : 0;
        ++rows;
        est += e;
      }
    }
    __syncthreads();
  }
}

// tid = exclusive scan of the tile-start flags: trow0 / tcta per tile, ctile per CTA.
__global__ void k_sym_tiles(const int32_t* tid, const int32_t* range, int G, int64_t nb, int32_t* trow0,
                            int32_t* tcta, int32_t* ctile) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R <= G) ctile[R] = tid[range[R]];
  if (R > nb) return;
  if (R == nb) {
    trow0[tid[nb]] = int32_t(nb);
    return;
  }
  if (tid[R + 1] == tid[R]) return;
  trow0[tid[R]] = int32_t(R);
  tcta[tid[R]] = cta_of(range, G, R);
}

// One CTA per tile: header, row offsets, column block ids and the
// transposed-product plan (off-diagonal blocks sorted by (column block, entry)).
__global__ void __launch_bounds__(kSymTB) k_sym_layout(SpmvDev S0, const int32_t* enoff, const int32_t* trow0,
                                                       const int32_t* tcta, const int32_t* range,
                                                       unsigned char* blob, int64_t* toff, int32_t* tsize,
                                                       int32_t* tns, int64_t* summary) {
  using Sort = cub::BlockRadixSort<unsigned long long, kSymTB, kSymCap / kSymTB>;
  using Scan = cub::BlockScan<int, kSymTB>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ unsigned long long keys[kSymCap];
  __shared__ int32_t hs[kSymCap];
  __shared__ int32_t s_nt, s_nl, s_first_spill;
  const int t = blockIdx.x;
  const int row0 = trow0[t], nr = trow0[t + 1] - row0;
  const int re = range[tcta[t] + 1];
  const int e0 = enoff[row0];
  const int E = enoff[row0 + nr] - e0;
  if (E > kSymCap) {
    if (threadIdx.x == 0) atomic_max64(summary + SM_ERR, 1);
    return;
  }
  const int64_t off = sym_toff(t, e0);
  unsigned char* base = blob + off;
  uint16_t* rp = reinterpret_cast<uint16_t*>(base + kSymHdr);
  int32_t* cols = reinterpret_cast<int32_t*>(base + sym_off_cols(E));
  for (int i = threadIdx.x; i <= nr; i += blockDim.x) rp[i] = uint16_t(enoff[row0 + i] - e0);
  for (int i = threadIdx.x; i < kSymCap; i += blockDim.x) keys[i] = ~0ull;
  __syncthreads();
  if (threadIdx.x < nr) {
    const int64_t R = row0 + threadIdx.x;
    const int32_t u0 = S0.nrow[R];
    const int le0 = enoff[R] - e0, n = enoff[R + 1] - enoff[R];
    for (int k = 0; k < n; ++k) {
      const int32_t c = S0.col[u0 + k] / 3;
      const int le = le0 + k;
      cols[le] = c;
      if (c != R) keys[le] = (static_cast<unsigned long long>(c) << 11) | unsigned(le);
    }
  }
  __syncthreads();
  constexpr int IPT = kSymCap / kSymTB;
  unsigned long long k8[IPT];
#pragma unroll
  for (int j = 0; j < IPT; ++j) k8[j] = keys[threadIdx.x * IPT + j];
  __syncthreads();
  Sort(tmp.sort).Sort(k8);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < IPT; ++j) keys[threadIdx.x * IPT + j] = k8[j];
  __syncthreads();
  // run heads (targets) among the NL sorted off-diagonal blocks (a prefix)
  int hf[IPT], hsum = 0, nl_local = 0;
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int q = threadIdx.x * IPT + j;
    const unsigned long long k = keys[q];
    hf[j] = (k != ~0ull && (q == 0 || (keys[q - 1] >> 11) != (k >> 11))) ? 1 : 0;
    hsum += hf[j];
    nl_local += k != ~0ull ? 1 : 0;
  }
  int hex = 0, htot = 0;
  Scan(tmp.scan).ExclusiveSum(hsum, hex, htot);
  if (threadIdx.x == 0) {
    s_nt = htot;
    s_first_spill = htot;
  }
  __syncthreads();
  {
    int h = hex;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int q = threadIdx.x * IPT + j;
      if (hf[j]) {
        hs[h] = q;
        if (int(keys[q] >> 11) >= re) atomicMin(&s_first_spill, h);
        ++h;
      }
    }
  }
  __syncthreads();
  {
    int nl_ex = 0, nl_tot = 0;
    Scan(tmp.scan).ExclusiveSum(nl_local, nl_ex, nl_tot);
    if (threadIdx.x == 0) s_nl = nl_tot;
  }
  __syncthreads();
  const int NT = s_nt, NL = s_nl, NS = NT - s_first_spill;
  int2* tg = reinterpret_cast<int2*>(base + sym_off_tg(E));
  uint16_t* list = reinterpret_cast<uint16_t*>(base + sym_off_list(E, NT));
  for (int q = threadIdx.x; q < NL; q += blockDim.x) list[q] = uint16_t(keys[q] & 2047u);
  for (int h = threadIdx.x; h < NT; h += blockDim.x) {
    const int st = hs[h], en = h + 1 < NT ? hs[h + 1] : NL;
    tg[h] = make_int2(int(keys[st] >> 11), st | ((en - st) << 16));
  }
  if (threadIdx.x == 0) {
    TileHdr* hd = reinterpret_cast<TileHdr*>(base);
    *hd = TileHdr{E, NT, NL, NS, row0, nr, 0, 0};
    const int sz = sym_size(E, NT, NL, NS);
    tsize[t] = sz;
    toff[t] = off;
    tns[t] = NS;
    atomic_max64(summary + SM_MAXTILE, sz);
    atomic_max64(summary + SM_MAXE, E);
  }
}

// Half-entry records in any fixed order (key = target << 32 | position,
// payload = block | group << 30 | transposed << 31), sorted by key afterwards.
__global__ void k_sym_half_rec(SpmvDev S0, SpmvDev S1, int has1, int64_t nb, const int32_t* enoff,
                               const int32_t* hoff, unsigned long long* key, uint32_t* pay) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R >= nb || hoff[R + 1] == hoff[R]) return;
  const RowSrc s = row_src(S0, S1, has1, R);
  int h = hoff[R];
  auto put = [&](uint32_t tgt, uint32_t p) {
    key[h] = (static_cast<unsigned long long>(tgt) << 32) | unsigned(h);
    pay[h] = p;
    ++h;
  };
  const int near = enoff[R + 1] - enoff[R];
  for (int k = near; k < s.n0; ++k) {  // static blocks beyond the window (off-diagonal)
    const uint32_t u = uint32_t(s.u0 + k), c = uint32_t(S0.col[u] / 3);
    put(uint32_t(R), u);
    put(c, u | 0x80000000u);
  }
  for (int k = 0; k < s.n1; ++k) {
    const uint32_t u = uint32_t(s.u1 + k), c = uint32_t(S1.col[u] / 3);
    put(uint32_t(R), u | 0x40000000u);
    if (c != uint32_t(R)) put(c, u | 0xC0000000u);
  }
}

__device__ __forceinline__ int64_t half_bound(int64_t H, int G, int b) { return H * b / G; }

// Sorted half-entries: target, source block row, run heads (a run = equal
// targets inside one CTA's chunk [H b / G, H (b + 1) / G)).
__global__ void k_sym_half_info(const unsigned long long* key, const uint32_t* pay, int64_t H, int G,
                                const int32_t* row0, const int32_t* col0, const int32_t* row1,
                                const int32_t* col1, int32_t* tgt, int32_t* src, int32_t* head) {
  const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h > H) return;
  if (h == H) {
    head[h] = 0;
    return;
  }
  const int32_t t = int32_t(key[h] >> 32);
  const uint32_t p = pay[h];
  const int32_t u = int32_t(p & 0x3fffffffu);
  const bool dyn = p & 0x40000000u, tr = p & 0x80000000u;
  const int32_t rr = (dyn ? row1[u] : row0[u]) / 3, cc = (dyn ? col1[u] : col0[u]) / 3;
  tgt[h] = t;
  src[h] = tr ? rr : cc;
  int b = int(h * G / H);  // the CTA whose chunk holds h
  while (b > 0 && half_bound(H, G, b) > h) --b;
  while (b + 1 < G && half_bound(H, G, b + 1) <= h) ++b;
  head[h] = (h == half_bound(H, G, b) || int32_t(key[h - 1] >> 32) != t) ? 1 : 0;
}

// Run lists of the half-entry chunks (chunk q of CTA b covers
// [h0 + q K, min(h0 + (q + 1) K, h1)), K = kSymChunk): one CTA per chunk.
// Entry j of chunk c (at c K + j): start | length << 11 | starts-before << 22 |
// continues << 23, and the run's slot.  rid: exclusive scan of the run heads.
__global__ void __launch_bounds__(kSymTB) k_sym_runs(const int32_t* rid, const int32_t* hslot, int64_t H, int G,
                                                     const int32_t* cbase, uint32_t* runs, int32_t* rslot,
                                                     int32_t* nruns) {
  using Scan = cub::BlockScan<int, kSymTB>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int32_t pos[kSymChunk + 1];
  const int c = blockIdx.x;
  int b = 0;
  while (b + 1 < G && cbase[b + 1] <= c) ++b;
  const int64_t h0 = H * b / G, h1 = H * (b + 1) / G;
  const int64_t cb = h0 + int64_t(c - cbase[b]) * kSymChunk;
  const int n = int(min(int64_t(kSymChunk), h1 - cb));
  constexpr int IPT = kSymChunk / kSymTB;
  int f[IPT], cnt = 0;
#pragma unroll
  for (int m = 0; m < IPT; ++m) {
    const int k = threadIdx.x * IPT + m;
    f[m] = k < n && (k == 0 || rid[cb + k + 1] != rid[cb + k]) ? 1 : 0;
    cnt += f[m];
  }
  int ex = 0, tot = 0;
  Scan(tmp).ExclusiveSum(cnt, ex, tot);
#pragma unroll
  for (int m = 0; m < IPT; ++m)
    if (f[m]) pos[ex++] = threadIdx.x * IPT + m;
  if (threadIdx.x == 0) {
    pos[tot] = n;
    nruns[c] = tot;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < tot; j += blockDim.x) {
    const int k = pos[j], len = pos[j + 1] - k;
    const bool before = k == 0 && rid[cb + 1] == rid[cb];  // position 0 is not a run head
    const bool cont = k + len == n && cb + n < h1 && rid[cb + n + 1] == rid[cb + n];
    runs[int64_t(c) * kSymChunk + j] = uint32_t(k) | (uint32_t(len) << 11) | (before ? 1u << 22 : 0u) |
                                       (cont ? 1u << 23 : 0u);
    rslot[int64_t(c) * kSymChunk + j] = hslot[cb + k];
  }
}

// Spill records: target column block and producer index (tiles' spill targets
// in tile order, then half-entry runs).
__global__ void __launch_bounds__(kSymTB) k_sym_spill_rec(const unsigned char* blob, const int64_t* toff,
                                                          const int32_t* tsb, int32_t* spill_c, int32_t* spill_o) {
  const int t = blockIdx.x;
  const TileHdr* hd = reinterpret_cast<const TileHdr*>(blob + toff[t]);
  const int E = hd->E, NT = hd->NT, NS = hd->NS;
  const int2* tg = reinterpret_cast<const int2*>(blob + toff[t] + sym_off_tg(E));
  for (int q = threadIdx.x; q < NS; q += blockDim.x) {
    spill_c[tsb[t] + q] = tg[NT - NS + q].x;
    spill_o[tsb[t] + q] = tsb[t] + q;
  }
}

// runs: rid = exclusive scan of the heads
__global__ void k_sym_spill_rec_half(const int32_t* tgt, const int32_t* rid, int64_t H, int64_t nst,
                                     int32_t* spill_c, int32_t* spill_o) {
  const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= H || rid[h + 1] == rid[h]) return;
  spill_c[nst + rid[h]] = tgt[h];
  spill_o[nst + rid[h]] = int32_t(nst + rid[h]);
}

// pos[producer] = its slot (sorted position)
__global__ void k_sym_spill_pos(const int32_t* sorted_o, int64_t n, int32_t* pos) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) pos[sorted_o[k]] = int32_t(k);
}

__global__ void __launch_bounds__(kSymTB) k_sym_spill_tiles(unsigned char* blob, const int64_t* toff,
                                                            const int32_t* tsb, const int32_t* pos) {
  const int t = blockIdx.x;
  const TileHdr* hd = reinterpret_cast<const TileHdr*>(blob + toff[t]);
  const int E = hd->E, NT = hd->NT, NL = hd->NL, NS = hd->NS;
  int32_t* sl = reinterpret_cast<int32_t*>(blob + toff[t] + sym_off_slot(E, NT, NL));
  for (int q = threadIdx.x; q < NS; q += blockDim.x) sl[q] = pos[tsb[t] + q];
}

// slot of the run of every half-entry (rid: exclusive scan of the heads)
__global__ void k_sym_spill_half(const int32_t* pos, const int32_t* rid, int64_t H, int64_t nst, int32_t* hslot) {
  const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h < H) hslot[h] = pos[nst + rid[h + 1] - 1];
}

__global__ void k_sym_spill_ptr(const int32_t* cs, int64_t n, int64_t nb, int32_t* ptr) {
  const int64_t R = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R > nb) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cs[mid] >= R) hi = mid;
    else lo = mid + 1;
  }
  ptr[R] = int32_t(lo);
}

// Block values of one tile (every Newton iteration): SoA, value q of block e at
// q E + e; coalesced stores.  The dynamic diagonal block is added into the
// static one (s + d).
__global__ void __launch_bounds__(kSymTB) k_sym_values(SpmvDev S0, SpmvDev S1, int has1, unsigned char* blob,
                                                       const int64_t* toff) {
  __shared__ int32_t u0r[kSymRows], udr[kSymRows];
  __shared__ uint16_t rp[kSymRows + 1];
  const int t = blockIdx.x;
  unsigned char* base = blob + toff[t];
  const TileHdr hd = *reinterpret_cast<const TileHdr*>(base);
  if (threadIdx.x < hd.nr) {
    const RowSrc s = row_src(S0, S1, has1, hd.row0 + threadIdx.x);
    u0r[threadIdx.x] = s.u0;
    udr[threadIdx.x] = s.ud;
  }
  const uint16_t* grp = reinterpret_cast<const uint16_t*>(base + kSymHdr);
  if (threadIdx.x <= hd.nr) rp[threadIdx.x] = grp[threadIdx.x];
  __syncthreads();
  double* v = reinterpret_cast<double*>(base + kSymVals);
  const int E = hd.E;
  for (int i = threadIdx.x; i < 9 * E; i += blockDim.x) {
    const int q = i / E, e = i - q * E;
    int lo = 0, hi = hd.nr - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const int k = e - rp[lo];
    double x = S0.values[9 * int64_t(u0r[lo] + k) + q];
    if (k == 0 && udr[lo] >= 0) x += S1.values[9 * int64_t(udr[lo]) + q];
    v[i] = x;
  }
}

// Half-entry values, oriented (B or B^T), SoA: value q of half-entry h at q H + h.
__global__ void k_sym_half_values(SpmvDev S0, SpmvDev S1, const uint32_t* pay, int64_t H, double* hval) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 9 * H) return;
  const int q = int(i / H);
  const int64_t h = i - int64_t(q) * H;
  const uint32_t p = pay[h];
  const int64_t u = int64_t(p & 0x3fffffffu);
  const int qq = (p & 0x80000000u) ? (q % 3) * 3 + q / 3 : q;
  hval[i] = ((p & 0x40000000u) ? S1.values : S0.values)[9 * u + qq];
}

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy primitives (SASS UBLKCP / SYNCS)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct SymDev {
  const unsigned char* blob;
  const int64_t* toff;
  const int32_t* tsize;
  const int32_t* ctile;
  const int32_t* range;
  double* spill_val;
  const int32_t* spill_ptr;
  const int32_t* htgt;   // half-entries (sorted by target)
  const int32_t* hsrc;
  const int32_t* hslot;
  const int32_t* cbase;   // G + 1: first half-entry chunk of each CTA
  const uint32_t* runs;   // per chunk (capacity kSymChunk): run start | length | flags (k_sym_runs)
  const int32_t* rslot;
  const int32_t* nruns;
  const double* hval;
  int64_t* clocks;  // G x 8 per-CTA clocks (diagnostics)
  int64_t nb, H;
  int W, max_range, stage_bytes, nstages, em;
};

struct SymSmem {
  size_t stages, pw, acc, work, wi, total;
};

__host__ __device__ inline SymSmem sym_smem_layout(int nstages, int stage_bytes, int W, int max_range, int em) {
  SymSmem L;
  L.stages = 128;
  L.pw = L.stages + size_t(nstages) * size_t(stage_bytes);
  L.acc = L.pw + 24 * size_t(W);
  L.work = L.acc + 24 * size_t(max_range);                          // 3 x max(em, chunk) doubles
  L.wi = L.work + 24 * size_t(em > kSymChunk ? em : kSymChunk);     // chunk ints
  L.total = L.wi + 4 * size_t(kSymChunk) + 128;                     // + next target, carry
  return L;
}

__device__ __forceinline__ void vec3_ldcg(const double* p, double& a, double& b, double& c) {
  a = __ldcg(p);
  b = __ldcg(p + 1);
  c = __ldcg(p + 2);
}

// The whole solve: one cooperative launch, one CTA of 256 threads per SM.
__global__ void __launch_bounds__(kSymTB, 1) k_pcg33_sym(SymDev S, const double* __restrict__ minv,
                                                         double* __restrict__ x, double* __restrict__ r,
                                                         double* __restrict__ p, PcgState* st, double* part,
                                                         double* hist, GridBar* gb) {
  extern __shared__ __align__(128) unsigned char smem[];
  const SymSmem L = sym_smem_layout(S.nstages, S.stage_bytes, S.W, S.max_range, S.em);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  unsigned char* stage0 = smem + L.stages;
  double* pw = reinterpret_cast<double*>(smem + L.pw);
  double* acc = reinterpret_cast<double*>(smem + L.acc);
  double* Wk = reinterpret_cast<double*>(smem + L.work);  // T of a tile (3 x em) / a chunk (3 x kSymChunk)
  int32_t* Wi = reinterpret_cast<int32_t*>(smem + L.wi);
  double* carry = reinterpret_cast<double*>(smem + L.wi + 4 * kSymChunk + 16);  // 3 doubles + target

  const int ws = S.em > kSymChunk ? S.em : kSymChunk;  // stride of the 3 work arrays
  const int G = gridDim.x;
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  const int Rb = S.range[b], nrows = S.range[b + 1] - Rb;
  const int t0 = S.ctile[b], nt = S.ctile[b + 1] - t0;
  const int64_t h0 = S.H * b / G, h1 = S.H * (b + 1) / G;
  const int64_t cbase0 = S.cbase[b];
  const int wl = int(min(int64_t(S.W), S.nb - Rb));
  const int NSt = S.nstages;
  const bool resident = nt <= NSt;
  if (tid == 0) {
    for (int s = 0; s < NSt; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long gis = NSt < nt ? NSt : nt, gco = 0;  // tile copies issued / consumed (running)
  if (tid == 0) {
    for (int g = 0; g < gis; ++g) {
      const int tt = t0 + g;
      mbar_expect_tx(&mbar[g], unsigned(S.tsize[tt]));
      bulk_g2s(stage0 + size_t(g) * S.stage_bytes, S.blob + S.toff[tt], unsigned(S.tsize[tt]), &mbar[g]);
    }
  }
  for (int i = tid; i < wl; i += kSymTB) vec3_ldcg(p + 3 * int64_t(Rb + i), pw[3 * i], pw[3 * i + 1], pw[3 * i + 2]);

  const double gnorm = st->gnorm;
  const double tol = st->tol;
  const long long max_iter = st->max_iter;
  const long long hist_cap = st->hist_cap;
  double rz = st->rz;
  int status = st->status;
  long long it = 0;
  double rel = st->rel, php = 0.0, alpha = 0.0;
  unsigned long long ph[4] = {0, 0, 0, 0};
  unsigned long long aux[5] = {0, 0, 0, 0, 0};
  unsigned long long epoch = 0;
  unsigned long long* cnt = &gb->arrivals;
  unsigned long long t_0 = gtimer();
  const int lr = tid >> 2, h4 = tid & 3;
  // slot ranges of this thread's rows (tid + 256 m), loaded once per solve
  constexpr int kRowsPer = 12;  // rows per thread: CTAs up to 3072 rows (checked by the layout)
  int spr[kRowsPer];
#pragma unroll
  for (int m = 0; m < kRowsPer; ++m) {
    const int i = tid + m * kSymTB;
    spr[m] = i < nrows ? S.spill_ptr[Rb + i] : 0;
  }
  int spr_end[kRowsPer];
#pragma unroll
  for (int m = 0; m < kRowsPer; ++m) {
    const int i = tid + m * kSymTB;
    spr_end[m] = i < nrows ? S.spill_ptr[Rb + i + 1] : 0;
  }
  while (status == 0) {
    // ---- phase A: hp = H p (on chip except the slots), pHp partials
    for (int i = tid; i < 3 * nrows; i += kSymTB) acc[i] = 0.0;
    __syncthreads();
    double dot = 0.0;
    long long ck0 = (long long)gtimer();
    // half-entries: a chunk's products with every load in flight, then one
    // thread per run sums it in order (a run continuing into the next chunk
    // hands its partial sum over through `carry`)
    for (int64_t cb = h0; cb < h1; cb += kSymChunk) {
      const int n = int(min(int64_t(kSymChunk), h1 - cb));
      const int cpar = int(((cb - h0) / kSymChunk) & 1);
      const int64_t qc = cbase0 + (cb - h0) / kSymChunk;  // global chunk index
      const int nrun = __ldcs(S.nruns + qc);
      const uint32_t run0 = __ldcs(S.runs + qc * kSymChunk + tid);
      const int32_t slot0 = __ldcs(S.rslot + qc * kSymChunk + tid);
      const double* cin = carry + 3 * (cpar ^ 1);  // written by the previous chunk
      double* cout = carry + 3 * cpar;
      // kHalfPer half-entries per thread, every load issued before any use
      constexpr int kHalfPer = kSymChunk / kSymTB;
      int32_t sv[kHalfPer], tv[kHalfPer];
      double B[kHalfPer][9];
#pragma unroll
      for (int m = 0; m < kHalfPer; ++m) {
        const int k = tid + m * kSymTB;
        const int64_t h = cb + min(k, n - 1);
        sv[m] = __ldcs(S.hsrc + h);
        tv[m] = __ldcs(S.htgt + h);
#pragma unroll
        for (int q = 0; q < 9; ++q) B[m][q] = __ldcs(S.hval + q * S.H + h);
      }
      double ps[kHalfPer][3], pt[kHalfPer][3];
#pragma unroll
      for (int m = 0; m < kHalfPer; ++m) {
        const int si = sv[m] - Rb, ti = tv[m] - Rb;
        if (si >= 0 && si < wl) {
          ps[m][0] = pw[3 * si];
          ps[m][1] = pw[3 * si + 1];
          ps[m][2] = pw[3 * si + 2];
        } else {
          vec3_ldcg(p + 3 * int64_t(sv[m]), ps[m][0], ps[m][1], ps[m][2]);
        }
        if (ti >= 0 && ti < wl) {
          pt[m][0] = pw[3 * ti];
          pt[m][1] = pw[3 * ti + 1];
          pt[m][2] = pw[3 * ti + 2];
        } else {
          vec3_ldcg(p + 3 * int64_t(tv[m]), pt[m][0], pt[m][1], pt[m][2]);
        }
      }
#pragma unroll
      for (int m = 0; m < kHalfPer; ++m) {
        const int k = tid + m * kSymTB;
        if (k >= n) break;
        const double u0 = B[m][0] * ps[m][0] + B[m][1] * ps[m][1] + B[m][2] * ps[m][2];
        const double u1 = B[m][3] * ps[m][0] + B[m][4] * ps[m][1] + B[m][5] * ps[m][2];
        const double u2 = B[m][6] * ps[m][0] + B[m][7] * ps[m][1] + B[m][8] * ps[m][2];
        Wk[k] = u0;
        Wk[ws + k] = u1;
        Wk[2 * ws + k] = u2;
        dot += pt[m][0] * u0 + pt[m][1] * u1 + pt[m][2] * u2;  // pHp: p_t . (B p_s)
      }
      __syncthreads();
      // one thread per run: its products in order; a run continuing into the
      // next chunk hands its partial sum over through `carry`
      for (int j = tid; j < nrun; j += kSymTB) {
        const uint32_t ru = j < kSymTB ? run0 : __ldcs(S.runs + qc * kSymChunk + j);
        const int32_t sl = j < kSymTB ? slot0 : __ldcs(S.rslot + qc * kSymChunk + j);
        const int rs = int(ru & 2047u), re = rs + int((ru >> 11) & 2047u);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if (ru & (1u << 22)) {  // the run started in the previous chunk
          a0 = cin[0];
          a1 = cin[1];
          a2 = cin[2];
        }
        for (int q = rs; q < re; ++q) {
          a0 += Wk[q];
          a1 += Wk[ws + q];
          a2 += Wk[2 * ws + q];
        }
        if (ru & (1u << 23)) {
          cout[0] = a0;
          cout[1] = a1;
          cout[2] = a2;
        } else {
          double* o = S.spill_val + 3 * int64_t(sl);
          __stcg(o, a0);
          __stcg(o + 1, a1);
          __stcg(o + 2, a2);
        }
      }
      __syncthreads();
    }
    long long ck1 = (long long)gtimer();
    aux[0] += ck1 - ck0;
    for (int k = 0; k < nt; ++k, ++gco) {
      const int s = resident ? k : int(gco % NSt);
      long long cw = (long long)gtimer();
      if (!resident || it == 0) mbar_wait(&mbar[s], unsigned((gco / NSt) & 1));
      long long cx = (long long)gtimer();
      aux[1] += cx - cw;
      const unsigned char* base = stage0 + size_t(s) * S.stage_bytes;
      const TileHdr hd = *reinterpret_cast<const TileHdr*>(base);
      const int E = hd.E;
      const double* V = reinterpret_cast<const double*>(base + kSymVals);
      const int32_t* C = reinterpret_cast<const int32_t*>(base + sym_off_cols(E));
      const int lt = hd.row0 - Rb;
      // 4 lanes per row: own products in registers, transposed products to Wk
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      if (lr < hd.nr) {
        const uint16_t* RP = reinterpret_cast<const uint16_t*>(base + kSymHdr);
        const int ir = lt + lr;
        const double r0 = pw[3 * ir], r1 = pw[3 * ir + 1], r2 = pw[3 * ir + 2];
        const int e1 = RP[lr + 1];
        for (int e = RP[lr] + h4; e < e1; e += 4) {
          const int ic = C[e] - Rb;
          double B[9];
#pragma unroll
          for (int q = 0; q < 9; ++q) B[q] = V[q * E + e];
          const double c0 = pw[3 * ic], c1 = pw[3 * ic + 1], c2 = pw[3 * ic + 2];
          a0 += B[0] * c0 + B[1] * c1 + B[2] * c2;
          a1 += B[3] * c0 + B[4] * c1 + B[5] * c2;
          a2 += B[6] * c0 + B[7] * c1 + B[8] * c2;
          if (ic != ir) {
            Wk[e] = B[0] * r0 + B[3] * r1 + B[6] * r2;
            Wk[ws + e] = B[1] * r0 + B[4] * r1 + B[7] * r2;
            Wk[2 * ws + e] = B[2] * r0 + B[5] * r1 + B[8] * r2;
          }
        }
      }
#pragma unroll
      for (int off = 1; off < 4; off <<= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, off);
        a1 += __shfl_xor_sync(0xffffffffu, a1, off);
        a2 += __shfl_xor_sync(0xffffffffu, a2, off);
      }
      __syncthreads();
      // targets: transposed products in entry order -> accumulator or slot
      {
        const int2* TG = reinterpret_cast<const int2*>(base + sym_off_tg(E));
        const uint16_t* LI = reinterpret_cast<const uint16_t*>(base + sym_off_list(E, hd.NT));
        const int32_t* SL = reinterpret_cast<const int32_t*>(base + sym_off_slot(E, hd.NT, hd.NL));
        const int fs = hd.NT - hd.NS;
        for (int j = tid; j < hd.NT; j += kSymTB) {
          const int2 tg = TG[j];
          const int q0 = tg.y & 0xffff, n = tg.y >> 16;
          double v0 = 0.0, v1 = 0.0, v2 = 0.0;
          for (int q = q0; q < q0 + n; ++q) {
            const int e = LI[q];
            v0 += Wk[e];
            v1 += Wk[ws + e];
            v2 += Wk[2 * ws + e];
          }
          const int ci = tg.x - Rb;
          if (j < fs) {
            acc[3 * ci] += v0;
            acc[3 * ci + 1] += v1;
            acc[3 * ci + 2] += v2;
          } else {
            double* o = S.spill_val + 3 * int64_t(SL[j - fs]);
            __stcg(o, v0);
            __stcg(o + 1, v1);
            __stcg(o + 2, v2);
            dot += pw[3 * ci] * v0 + pw[3 * ci + 1] * v1 + pw[3 * ci + 2] * v2;
          }
        }
      }
      __syncthreads();
      long long cy = (long long)gtimer();
      aux[2] += cy - cx;
      // rows: y = accumulator (transposed products) + own products
      if (h4 == 0 && lr < hd.nr) {
        const int i = lt + lr;
        const double y0 = acc[3 * i] + a0, y1 = acc[3 * i + 1] + a1, y2 = acc[3 * i + 2] + a2;
        acc[3 * i] = y0;
        acc[3 * i + 1] = y1;
        acc[3 * i + 2] = y2;
        dot += pw[3 * i] * y0 + pw[3 * i + 1] * y1 + pw[3 * i + 2] * y2;
      }
      if (!resident) {
        if (tid == 0) {
          // the stage is free: refill it with the tile NSt copies ahead (cycling)
          const int tt = t0 + int(gis % nt);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&mbar[s], unsigned(S.tsize[tt]));
          bulk_g2s(stage0 + size_t(s) * S.stage_bytes, S.blob + S.toff[tt], unsigned(S.tsize[tt]), &mbar[s]);
        }
        ++gis;
      }
    }
    double d1[1] = {dot};
    block_reduce<1>(d1);
    if (tid == 0) part[b] = d1[0];
    grid_arrive(cnt);
    grid_wait(cnt, (unsigned long long)G * ++epoch);
    unsigned long long t1 = gtimer();
    ph[0] += t1 - t_0;
    t_0 = t1;
    double tot1[1];
    reduce_partials_all<1>(part, G, tot1);
    php = tot1[0];
    if (!isfinite(php) || php <= 0.0) {
      status = php == 0.0 ? 2 : 3;
      break;
    }
    alpha = rz / php;
    // ---- phase B: hp = on-chip part + slots (slot order); x += a p, r -= a hp,
    // z = M^-1 r (z kept in the accumulator)
    long long ck4 = (long long)gtimer();
    {
      // the CTA's slots are contiguous (numbered in row order): chunks loaded
      // with every load in flight, then each row adds its slots in order
      const int k0 = S.spill_ptr[Rb], k1 = S.spill_ptr[Rb + nrows];
      for (int cb = k0; cb < k1; cb += kSymChunk) {
        const int n = min(kSymChunk, k1 - cb);
        for (int i = tid; i < 3 * n; i += kSymTB) Wk[i] = __ldcg(S.spill_val + 3 * int64_t(cb) + i);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < kRowsPer; ++m) {
          const int i = tid + m * kSymTB;
          if (i >= nrows) break;
          const int a = max(spr[m], cb), e = min(spr_end[m], cb + n);
          for (int k = a; k < e; ++k) {
            acc[3 * i] += Wk[3 * (k - cb)];
            acc[3 * i + 1] += Wk[3 * (k - cb) + 1];
            acc[3 * i + 2] += Wk[3 * (k - cb) + 2];
          }
        }
        __syncthreads();
      }
    }
    const long long ck5 = (long long)gtimer();
    aux[3] += ck5 - ck4;
    double v[2] = {0.0, 0.0};
    for (int i = tid; i < nrows; i += kSymTB) {
      const int64_t R = Rb + i;
      const double hh[3] = {acc[3 * i], acc[3 * i + 1], acc[3 * i + 2]};
      double rr[3], xx[3], zz[3], M[9];
      load_vec3(r + 3 * R, rr[0], rr[1], rr[2]);
      load_vec3(x + 3 * R, xx[0], xx[1], xx[2]);
      load_block9(minv + 9 * R, M);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        xx[q] += alpha * pw[3 * i + q];
        rr[q] -= alpha * hh[q];
      }
      precond_apply<3>(M, rr, zz);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        x[3 * R + q] = xx[q];
        r[3 * R + q] = rr[q];
        acc[3 * i + q] = zz[q];
        v[0] += rr[q] * rr[q];
        v[1] += rr[q] * zz[q];
      }
    }
    aux[4] += (long long)gtimer() - ck5;
    block_reduce<2>(v);
    if (tid == 0) {
      part[G + b] = v[0];
      part[2 * G + b] = v[1];
    }
    grid_arrive(cnt);
    grid_wait(cnt, (unsigned long long)G * ++epoch);
    t1 = gtimer();
    ph[1] += t1 - t_0;
    t_0 = t1;
    double tot2[2];
    reduce_partials_all<2>(part + G, G, tot2);
    t1 = gtimer();
    ph[2] += t1 - t_0;
    t_0 = t1;
    rel = sqrt(tot2[0]) / gnorm;
    if (b == 0 && tid == 0 && it + 1 < hist_cap) hist[it + 1] = rel;
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
    // ---- phase C: p = z + beta p (own rows: shared and global)
    for (int i = tid; i < 3 * nrows; i += kSymTB) {
      const double pn = acc[i] + beta * pw[i];
      pw[i] = pn;
      p[3 * int64_t(Rb) + i] = pn;
    }
    grid_arrive(cnt);
    grid_wait(cnt, (unsigned long long)G * ++epoch);
    // the window beyond the own rows: other CTAs' new p
    for (int i = nrows + tid; i < wl; i += kSymTB)
      vec3_ldcg(p + 3 * int64_t(Rb + i), pw[3 * i], pw[3 * i + 1], pw[3 * i + 2]);
    t1 = gtimer();
    ph[3] += t1 - t_0;
    t_0 = t1;
  }
  // drain the copies still in flight before the CTA exits
  for (; gco < gis; ++gco) mbar_wait(&mbar[gco % NSt], unsigned((gco / NSt) & 1));
  if (b == 0 && tid == 0) {
    st->it += it;
    st->rel = rel;
    st->rz = rz;
    st->php = php;
    st->alpha = alpha;
    st->status = status;
    if (status == 3 || status == 4) st->fail_it = int(it - (status == 4 ? 1 : 0));
    for (int k = 0; k < 4; ++k) st->phase_ns[k] = ph[k];
    for (int k = 0; k < 4; ++k) st->aux_ns[k] = aux[k];
  }
  if (tid == 0) {
    int64_t* o = S.clocks + 8 * b;
    for (int k = 0; k < 5; ++k) o[k] = int64_t(aux[k]);
    o[5] = nrows;
    o[6] = h1 - h0;
    o[7] = S.spill_ptr[Rb + nrows] - S.spill_ptr[Rb];
  }
}

template <class T>
void cub_exclusive_sum(Context& c, T* a, int64_t n) {
  size_t bytes = 0;
  YS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, a, a, int(n), c.stream));
  c.cubtmp.resize(std::max<size_t>(bytes, 1));
  YS_CUDA(cub::DeviceScan::ExclusiveSum(c.cubtmp.p, bytes, a, a, int(n), c.stream));
}

int grid_for(int64_t n) { return int(std::max<int64_t>(1, ceil_div(n, kSymTB))); }

}  // namespace

// Layout of the symmetric band copy for the current static + dynamic
// structures (values are filled by sym_pcg).  Three host synchronisations
// (sizes); Newton steps run it while the static evaluation runs on the side
// streams.
void sym_prepare(Context& c) {
  auto& y = c.sym;
  y.prepared = false;
  y.usable = false;
  cudaStream_t s = c.stream;
  const int64_t nb = c.NB;
  if (nb == 0) return;
  const bool has1 = c.S[1].n_blocks > 0;
  const int h1 = has1 ? 1 : 0;
  SpmvDev d0 = spmv_dev(c.S[0]);
  SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
  const int32_t* row1 = has1 ? c.S[1].row.p : c.S[0].row.p;
  const int32_t* col1 = has1 ? c.S[1].col.p : c.S[0].col.p;
  const int G = int(std::max<int64_t>(1, std::min<int64_t>(sm_count(), nb / 64)));
  y.G = G;
  y.summary.resize(SM_N);
  YS_CUDA(cudaMemsetAsync(y.summary.p, 0, SM_N * sizeof(int64_t), s));
  y.eoff.resize(size_t(nb + 1));
  k_sym_count<<<grid_for(nb + 1), kSymTB, 0, s>>>(d0, nb, y.eoff.p, y.summary.p);
  YS_LAUNCH_CHECK();
  cub_exclusive_sum(c, y.eoff.p, nb + 1);
  y.range.resize(size_t(G + 1));
  k_sym_ranges<<<grid_for(G + 1), kSymTB, 0, s>>>(y.eoff.p, nb, G, y.range.p, y.summary.p);
  YS_LAUNCH_CHECK();
  int64_t sm[SM_N];
  YS_CUDA(cudaMemcpyAsync(sm, y.summary.p, SM_N * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  c.launches += 4;
  y.max_range = int(sm[SM_MAXRANGE]);
  // shared-memory plan: a ring of 3 (else 2) stages, the accumulator, the work
  // buffers, and the window W >= own rows (up to own rows + the static band)
  const int maxrow = int(sm[SM_MAXROW]);
  y.stage_bytes = (std::max(kSymBudget, 256 + 96 * maxrow) + 127) & ~127;
  y.em = std::max((kSymBudget - 256) / 96, maxrow);
  int dev = 0, optin = 0;
  YS_CUDA(cudaGetDevice(&dev));
  YS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t budget = size_t(optin) - 2048;  // static shared memory of the reductions
  const int64_t want = std::min<int64_t>(nb, int64_t(y.max_range) + sm[SM_BAND] + 1);
  y.W = 0;
  for (int ns = 3; ns >= 2 && !y.W; --ns) {
    const size_t fixed = sym_smem_layout(ns, y.stage_bytes, 0, y.max_range, y.em).total;
    if (fixed > budget) continue;
    const int64_t wmax = int64_t((budget - fixed) / 24);
    if (wmax < y.max_range) continue;
    y.nstages = ns;
    y.W = int(std::min<int64_t>(wmax, std::max<int64_t>(want, y.max_range)));
  }
  if (!y.W || maxrow > kSymCap || y.max_range > 12 * kSymTB) {
    y.prepared = true;  // does not fit: the caller takes the sliced-ELL copy
    return;
  }
  y.smem = sym_smem_layout(y.nstages, y.stage_bytes, y.W, y.max_range, y.em).total;
  // near blocks / half-entries per row, tiles
  y.enoff.resize(size_t(nb + 1));
  y.hoff.resize(size_t(nb + 1));
  k_sym_classify<<<grid_for(nb + 1), kSymTB, 0, s>>>(d0, d1, h1, nb, y.range.p, G, y.W, y.enoff.p, y.hoff.p);
  YS_LAUNCH_CHECK();
  cub_exclusive_sum(c, y.enoff.p, nb + 1);
  cub_exclusive_sum(c, y.hoff.p, nb + 1);
  y.tflag.resize(size_t(nb + 1));
  YS_CUDA(cudaMemsetAsync(y.tflag.p, 0, size_t(nb + 1) * sizeof(int32_t), s));
  k_sym_walk<<<G, kSymTB, 0, s>>>(y.enoff.p, y.range.p, y.tflag.p);
  YS_LAUNCH_CHECK();
  cub_exclusive_sum(c, y.tflag.p, nb + 1);
  int32_t h3[3] = {0, 0, 0};  // tiles, near blocks, half-entries
  YS_CUDA(cudaMemcpyAsync(&h3[0], y.tflag.p + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaMemcpyAsync(&h3[1], y.enoff.p + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaMemcpyAsync(&h3[2], y.hoff.p + nb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  c.launches += 4;
  const int nt = h3[0];
  y.ntiles = nt;
  y.nnear = h3[1];
  y.H = h3[2];
  y.trow0.resize(size_t(nt + 1));
  y.tcta.resize(size_t(std::max(nt, 1)));
  y.ctile.resize(size_t(G + 1));
  k_sym_tiles<<<grid_for(std::max<int64_t>(nb + 1, G + 1)), kSymTB, 0, s>>>(y.tflag.p, y.range.p, G, nb, y.trow0.p,
                                                                            y.tcta.p, y.ctile.p);
  YS_LAUNCH_CHECK();
  y.blob.resize(size_t(sym_toff(nt, y.nnear) + 256));
  y.toff.resize(size_t(std::max(nt, 1)));
  y.tsize.resize(size_t(std::max(nt, 1)));
  y.tns.resize(size_t(nt + 1));
  YS_CUDA(cudaMemsetAsync(y.tns.p + nt, 0, sizeof(int32_t), s));
  if (nt > 0)
    k_sym_layout<<<nt, kSymTB, 0, s>>>(d0, y.enoff.p, y.trow0.p, y.tcta.p, y.range.p, y.blob.p, y.toff.p,
                                         y.tsize.p, y.tns.p, y.summary.p);
  YS_LAUNCH_CHECK();
  // half-entries: records, sort by target, runs per CTA chunk
  const int64_t H = y.H;
  const size_t H1 = size_t(std::max<int64_t>(H, 1));
  y.hkey.resize(H1);
  y.hkey_s.resize(H1);
  y.hpay.resize(H1);
  y.hpay_s.resize(H1);
  y.htgt.resize(H1);
  y.hsrc.resize(H1);
  y.hslot.resize(H1);
  y.hrid.resize(H1 + 1);
  y.hval.resize(9 * H1);
  if (H > 0) {
    k_sym_half_rec<<<grid_for(nb), kSymTB, 0, s>>>(d0, d1, h1, nb, y.enoff.p, y.hoff.p, y.hkey.p, y.hpay.p);
    YS_LAUNCH_CHECK();
    size_t bytes = 0;
    YS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, y.hkey.p, y.hkey_s.p, y.hpay.p, y.hpay_s.p, int(H), 0,
                                            64, s));
    c.cubtmp.resize(std::max<size_t>(bytes, 1));
    YS_CUDA(cub::DeviceRadixSort::SortPairs(c.cubtmp.p, bytes, y.hkey.p, y.hkey_s.p, y.hpay.p, y.hpay_s.p, int(H),
                                            0, 64, s));
    k_sym_half_info<<<grid_for(H + 1), kSymTB, 0, s>>>(y.hkey_s.p, y.hpay_s.p, H, G, c.S[0].row.p, c.S[0].col.p,
                                                       row1, col1, y.htgt.p, y.hsrc.p, y.hrid.p);
    YS_LAUNCH_CHECK();
    cub_exclusive_sum(c, y.hrid.p, H + 1);
    c.launches += 5;
  }
  cub_exclusive_sum(c, y.tns.p, nt + 1);
  int32_t h2[2] = {0, 0};  // tile spill producers, half-entry runs
  YS_CUDA(cudaMemcpyAsync(sm, y.summary.p, SM_N * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaMemcpyAsync(&h2[0], y.tns.p + nt, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  if (H > 0) YS_CUDA(cudaMemcpyAsync(&h2[1], y.hrid.p + H, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  YS_CUDA(cudaStreamSynchronize(s));
  c.launches += 3;
  if (sm[SM_ERR] || sm[SM_MAXTILE] > y.stage_bytes || sm[SM_MAXE] > y.em) {
    y.prepared = true;  // a tile beyond the plan's capacity: not usable
    return;
  }
  // slots: one per tile spill target and per half-entry run, numbered in
  // target-row order (producers in order for equal targets: stable sort)
  const int64_t nst = h2[0], nruns = h2[1];
  const int64_t nsp = nst + nruns;
  y.nspill = nsp;
  const size_t nsp1 = size_t(std::max<int64_t>(nsp, 1));
  y.spill_c.resize(nsp1);
  y.spill_cs.resize(nsp1);
  y.spill_o.resize(nsp1);
  y.spill_os.resize(nsp1);
  y.spill_val.resize(3 * nsp1);
  y.spill_ptr.resize(size_t(nb + 1));
  if (nst > 0) k_sym_spill_rec<<<nt, kSymTB, 0, s>>>(y.blob.p, y.toff.p, y.tns.p, y.spill_c.p, y.spill_o.p);
  if (nruns > 0)
    k_sym_spill_rec_half<<<grid_for(H), kSymTB, 0, s>>>(y.htgt.p, y.hrid.p, H, nst, y.spill_c.p, y.spill_o.p);
  YS_LAUNCH_CHECK();
  if (nsp > 0) {
    int bits = 1;
    while ((int64_t(1) << bits) <= nb) ++bits;
    size_t bytes = 0;
    YS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, y.spill_c.p, y.spill_cs.p, y.spill_o.p, y.spill_os.p,
                                            int(nsp), 0, bits, s));
    c.cubtmp.resize(std::max<size_t>(bytes, 1));
    YS_CUDA(cub::DeviceRadixSort::SortPairs(c.cubtmp.p, bytes, y.spill_c.p, y.spill_cs.p, y.spill_o.p,
                                            y.spill_os.p, int(nsp), 0, bits, s));
    // spill_o <- slot of each producer
    k_sym_spill_pos<<<grid_for(nsp), kSymTB, 0, s>>>(y.spill_os.p, nsp, y.spill_o.p);
    if (nst > 0) k_sym_spill_tiles<<<nt, kSymTB, 0, s>>>(y.blob.p, y.toff.p, y.tns.p, y.spill_o.p);
    if (H > 0) k_sym_spill_half<<<grid_for(H), kSymTB, 0, s>>>(y.spill_o.p, y.hrid.p, H, nst, y.hslot.p);
    {
      // chunks per CTA: ceil(|chunk of b| / K), prefix on the host (G values)
      std::vector<int32_t> cb(size_t(G + 1), 0);
      for (int b = 0; b < G; ++b)
        cb[size_t(b + 1)] = cb[size_t(b)] + int32_t(ceil_div(H * (b + 1) / G - H * b / G, kSymChunk));
      const int nch = cb[size_t(G)];
      y.cbase.upload(cb, s);
      y.runs.resize(size_t(std::max(nch, 1)) * kSymChunk);
      y.rslot.resize(size_t(std::max(nch, 1)) * kSymChunk);
      y.nruns.resize(size_t(std::max(nch, 1)));
      if (nch > 0)
        k_sym_runs<<<nch, kSymTB, 0, s>>>(y.hrid.p, y.hslot.p, H, G, y.cbase.p, y.runs.p, y.rslot.p, y.nruns.p);
      YS_LAUNCH_CHECK();
    }
    YS_LAUNCH_CHECK();
    c.launches += 5;
  }
  if (H == 0) y.cbase.upload(std::vector<int32_t>(size_t(G + 1), 0), s);  // no half-entry chunks
  k_sym_spill_ptr<<<grid_for(nb + 1), kSymTB, 0, s>>>(y.spill_cs.p, nsp, nb, y.spill_ptr.p);
  YS_LAUNCH_CHECK();
  c.launches += 4;
  y.usable = true;
  y.prepared = true;
}

// The solve over the symmetric band copy (layout from sym_prepare, values
// filled here).  Returns false when the layout does not fit (the caller then
// runs the sliced-ELL copy and reports that path).
bool sym_pcg(Context& c, ys_step_stats* stats) {
  auto& y = c.sym;
  if (!y.prepared) sym_prepare(c);
  y.prepared = false;  // consumed: the next solve rebuilds (structures change every Newton iteration)
  if (!y.usable) return false;
  cudaStream_t s = c.stream;
  const bool has1 = c.S[1].n_blocks > 0;
  SpmvDev d0 = spmv_dev(c.S[0]);
  SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
  void* kern = reinterpret_cast<void*>(k_pcg33_sym);
  YS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(y.smem)));
  int occ = 0;
  YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kSymTB, y.smem));
  if (occ < 1) return false;
  if (y.ntiles > 0) k_sym_values<<<y.ntiles, kSymTB, 0, s>>>(d0, d1, has1 ? 1 : 0, y.blob.p, y.toff.p);
  if (y.H > 0) k_sym_half_values<<<grid_for(9 * y.H), kSymTB, 0, s>>>(d0, d1, y.hpay_s.p, y.H, y.hval.p);
  YS_LAUNCH_CHECK();
  y.clocks.resize(size_t(8 * y.G));
  SymDev S{y.blob.p,  y.toff.p,  y.tsize.p,  y.ctile.p, y.range.p, y.spill_val.p, y.spill_ptr.p, y.htgt.p,
           y.hsrc.p,  y.hslot.p, y.cbase.p,  y.runs.p,  y.rslot.p, y.nruns.p,     y.hval.p,      y.clocks.p,
           c.NB,      y.H,       y.W,        y.max_range, y.stage_bytes, y.nstages, y.em};
  const int G = y.G;
  c.partials.resize(std::max<size_t>(c.partials.n, size_t(3 * G)));
  c.gridbar.resize(sizeof(GridBar));
  YS_CUDA(cudaMemsetAsync(c.gridbar.p, 0, sizeof(GridBar), s));
  const double* minv = c.minv.p;
  double *xp = c.DX.p, *rp = c.r.p, *pp = c.p.p, *part = c.partials.p, *hist = c.hist.p;
  PcgState* stp = c.pcg.p;
  GridBar* gbp = reinterpret_cast<GridBar*>(c.gridbar.p);
  void* args[] = {&S, &minv, &xp, &rp, &pp, &stp, &part, &hist, &gbp};
  YS_CUDA(cudaLaunchCooperativeKernel(kern, dim3(G), dim3(kSymTB), args, y.smem, s));
  c.launches += 3;
  (void)stats;
  return true;
}

void sym_info(Context& c, int64_t* info, int64_t* cta) {
  const auto& y = c.sym;
  const int64_t v[12] = {y.G, y.ntiles, y.max_range, y.W, y.nstages, y.stage_bytes, y.em, y.nnear, y.H, y.nspill,
                         int64_t(y.smem), y.usable ? 1 : 0};
  for (int k = 0; k < 12; ++k) info[k] = v[k];
  if (cta && y.clocks.n) {
    std::vector<int64_t> h = y.clocks.to_host(c.stream);
    std::copy(h.begin(), h.end(), cta);
  }
}

}  // namespace ys
