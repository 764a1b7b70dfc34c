// ys_solver.cu — BSR SpMV and block-Jacobi PCG on the device.
//
// Reference: spmv_add / spmv_group_fixed (solver.cpp:10-82),
// BlockJacobiPreconditioner::apply (138-146), pcg (151-200),
// Engine::apply_hessian (engine.cpp:70-73), Engine::minimize_step (75-101).
//
// Layout: the upper-triangular blocks stay in the reference's storage
// (shape groups, row-major values).  Each block row gathers every block that
// touches it — (r, c) directly and (c, r) transposed — so y is produced row by
// row with no atomics: deterministic, one write per row; the second read of an
// off-diagonal block is an L2 hit.  Uniform 3x3 systems: 4 lanes per block row
// (ys_spmv.cuh); mixed shapes: a warp per row, launched per block-size class.
//
// Solve drivers:
//  * uniform 3x3: k_pcg33_persistent, one cooperative launch for the whole
//    solve; phases split by a grid barrier, every CTA reduces the same
//    partials in the same order (deterministic alpha / beta / status);
//  * otherwise 3 kernels per iteration (SpMV + pHp, update + precondition,
//    p update) captured into a CUDA graph with a conditional WHILE node that
//    loops on the device until the status word leaves 0.
#include <algorithm>
#include <cstdio>
#include <string>
#include <cstdlib>
#include <chrono>

#include "ys_grid.cuh"
#include "ys_phase.cuh"

namespace ys {

// y(+)= (S0 + S1) x over uniform 3-DoF block rows; optional p.y partials
// reduced to pHp and alpha by the last CTA.
__global__ void __launch_bounds__(kTB, kSpmvMinB) k_spmv33(SpmvDev S0, SpmvDev S1, int has1, int64_t nb,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   int accumulate, PcgState* st, double* part) {
  constexpr int SW = kSpmvSW;
  if (st && st->status) return;
  const int lane = threadIdx.x % SW;
  const int64_t sw0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / SW;
  const int64_t nsw = int64_t(gridDim.x) * blockDim.x / SW;
  const unsigned mask = ((1u << SW) - 1u) << ((threadIdx.x & 31) & ~(SW - 1));
  double dot[1] = {0.0};
  for (int64_t R = sw0; R < nb; R += nsw) {
    // both groups' row pointers issue together (one latency round, not two)
    const RowPtrs p0 = load_rowptrs(S0, R);
    RowPtrs p1{0, 0, 0, 0};
    if (has1) p1 = load_rowptrs(S1, R);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    acc33_u2<SW>(S0, p0, lane, x, a0, a1, a2);
    if (has1) acc33_u2<SW>(S1, p1, lane, x, a0, a1, a2);
#pragma unroll
    for (int off = SW / 2; off > 0; off >>= 1) {
      a0 += __shfl_xor_sync(mask, a0, off, SW);
      a1 += __shfl_xor_sync(mask, a1, off, SW);
      a2 += __shfl_xor_sync(mask, a2, off, SW);
    }
    if (lane == 0) {
      double* yo = y + 3 * R;
      if (accumulate) {
        a0 += yo[0];
        a1 += yo[1];
        a2 += yo[2];
      }
      yo[0] = a0;
      yo[1] = a1;
      yo[2] = a2;
      if (part) dot[0] += x[3 * R] * a0 + x[3 * R + 1] * a1 + x[3 * R + 2] * a2;
    }
  }
  if (!part) return;
  block_reduce<1>(dot);
  if (threadIdx.x == 0) part[blockIdx.x] = dot[0];
  if (!last_cta(&st->counter1)) return;
  double tot[1];
  sum_partials<1>(part, gridDim.x, 0, tot);
  if (threadIdx.x == 0) {
    st->counter1 = 0;
    const double php = tot[0];
    st->php = php;
    if (!isfinite(php) || php <= 0.0) {
      if (php == 0.0) {
        st->status = 2;  // stagnation on a semidefinite direction: break
      } else {
        st->status = 3;
        st->fail_it = int(st->it);
      }
    } else {
      st->alpha = st->rz / php;
    }
  }
}


// Generic shapes: one warp per block row of size RC (launched per block-size
// class), lanes over the row's entries, fixed xor-butterfly reduction.
// One block of row R's list: y_R += B^T x_other (TR, B is OT x RC) or
// B x_other (B is RC x OT), OT the other side's block size (compile time).
template <int RC, int OT, bool TR>
__device__ __forceinline__ void acc_block(const double* __restrict__ v, const double* __restrict__ xo,
                                          double (&acc)[RC]) {
  double xk[OT];
#pragma unroll
  for (int k = 0; k < OT; ++k) xk[k] = xo[k];
#pragma unroll
  for (int k = 0; k < OT; ++k)
#pragma unroll
    for (int i = 0; i < RC; ++i) acc[i] += (TR ? v[k * RC + i] : v[i * OT + k]) * xk[k];
}

template <int RC>
__device__ __forceinline__ void acc_gen(const SpmvDev& S, int64_t R, int lane, const double* __restrict__ x,
                                        double (&acc)[RC]) {
  const int32_t j0 = S.rowptr[R], j1 = S.rowptr[R + 1];
  for (int32_t j = j0 + lane; j < j1; j += 32) {
    const uint32_t e = uint32_t(S.ent[j]);
    const uint32_t u = e & 0x7fffffffu;
    const int r = S.br[u], c = S.bc[u];
    const double* v = S.values + S.voff[u];
    const double* xo = x + S.oth[j];
    const bool tr = (e >> 31) != 0;  // block (other, R): B is r x RC; else block (R, other): B is RC x c
    const int ot = tr ? r : c;
    if (ot == 3) {  // the common shapes unrolled (loads issued together)
      if (tr) acc_block<RC, 3, true>(v, xo, acc);
      else acc_block<RC, 3, false>(v, xo, acc);
    } else if (ot == 9) {
      if (tr) acc_block<RC, 9, true>(v, xo, acc);
      else acc_block<RC, 9, false>(v, xo, acc);
    } else if (tr) {
      for (int k = 0; k < r; ++k) {
        const double xk = xo[k];
#pragma unroll
        for (int i = 0; i < RC; ++i) acc[i] += v[k * RC + i] * xk;
      }
    } else {
      for (int k = 0; k < c; ++k) {
        const double xk = xo[k];
#pragma unroll
        for (int i = 0; i < RC; ++i) acc[i] += v[i * c + k] * xk;
      }
    }
  }
}

template <int RC>
__global__ void __launch_bounds__(kTB) k_spmv_gen(SpmvDev S0, SpmvDev S1, int has1, BlocksDev B,
                                                  const int32_t* __restrict__ rows, int64_t nrows,
                                                  const double* __restrict__ x, double* __restrict__ y,
                                                  int accumulate, const PcgState* st) {
  if (st && st->status) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = w0; q < nrows; q += nw) {
    const int64_t R = rows ? rows[q] : q;
    double acc[RC];
#pragma unroll
    for (int i = 0; i < RC; ++i) acc[i] = 0.0;
    acc_gen<RC>(S0, R, lane, x, acc);
    if (has1) acc_gen<RC>(S1, R, lane, x, acc);
#pragma unroll
    for (int i = 0; i < RC; ++i)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
    if (lane == 0) {
      double* yo = y + B.start[R];
#pragma unroll
      for (int i = 0; i < RC; ++i) yo[i] = accumulate ? yo[i] + acc[i] : acc[i];
    }
  }
}

// pHp over all rows, last CTA -> alpha / status (generic path).
__global__ void __launch_bounds__(kTB) k_dot_alpha(int64_t s, const double* __restrict__ p,
                                                   const double* __restrict__ hp, PcgState* st, double* part) {
  if (st->status) return;
  double dot[1] = {0.0};
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s; i += int64_t(gridDim.x) * blockDim.x)
    dot[0] += p[i] * hp[i];
  block_reduce<1>(dot);
  if (threadIdx.x == 0) part[blockIdx.x] = dot[0];
  if (!last_cta(&st->counter1)) return;
  double tot[1];
  sum_partials<1>(part, gridDim.x, 0, tot);
  if (threadIdx.x == 0) {
    st->counter1 = 0;
    const double php = tot[0];
    st->php = php;
    if (!isfinite(php) || php <= 0.0) {
      if (php == 0.0) st->status = 2;
      else {
        st->status = 3;
        st->fail_it = int(st->it);
      }
    } else {
      st->alpha = st->rz / php;
    }
  }
}

// --- PCG vector kernels -----------------------------------------------------

__device__ __forceinline__ void precond_apply_any(int rc, const double* M, const double* r, double* z) {
  if (rc == 3) precond_apply<3>(M, r, z);
  else if (rc == 9) precond_apply<9>(M, r, z);
  else
    for (int i = 0; i < rc; ++i) {
      double a = 0.0;
      for (int k = 0; k < rc; ++k) a += M[i * rc + k] * r[k];
      z[i] = a;
    }
}

// r = g; z = M^-1 r; p = z; x = 0; partials of g.g and r.z; last CTA -> gnorm, rz.
__global__ void k_pcg_init(BlocksDev B, int uniform3, const double* __restrict__ g, const double* __restrict__ minv,
                           double* r, double* z, double* p, double* x, PcgState* st, double* part, double* hist) {
  double v[2] = {0.0, 0.0};
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < B.nb; b += int64_t(gridDim.x) * blockDim.x) {
    const int rc = uniform3 ? 3 : B.rc[b];
    const int64_t s0 = uniform3 ? 3 * b : B.start[b];
    const double* M = minv + (uniform3 ? 9 * b : B.voff[b]);
    double rr[16], zz[16];
    for (int i = 0; i < rc; ++i) {
      rr[i] = g[s0 + i];
      r[s0 + i] = rr[i];
      x[s0 + i] = 0.0;
    }
    precond_apply_any(rc, M, rr, zz);
    for (int i = 0; i < rc; ++i) {
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
    st->gnorm = sqrt(tot[0]);
    st->rz = tot[1];
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
}

// x += a p; r -= a hp; z = M^-1 r; partials of r.r and r.z; last CTA -> rel,
// history, convergence test, beta (solver.cpp:170-197).
__global__ void __launch_bounds__(kTB) k_update(BlocksDev B, int uniform3, const double* __restrict__ minv,
                                                double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                                const double* __restrict__ p, const double* __restrict__ hp,
                                                PcgState* st, double* part, double* hist) {
  if (st->status) return;
  const double a = st->alpha;
  double v[2] = {0.0, 0.0};
  for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < B.nb; b += int64_t(gridDim.x) * blockDim.x) {
    if (uniform3) {
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
    } else {
      const int rc = B.rc[b];
      const int64_t s0 = B.start[b];
      double rr[16], zz[16];
      for (int i = 0; i < rc; ++i) {
        x[s0 + i] += a * p[s0 + i];
        rr[i] = r[s0 + i] - a * hp[s0 + i];
        r[s0 + i] = rr[i];
      }
      precond_apply_any(rc, minv + B.voff[b], rr, zz);
      for (int i = 0; i < rc; ++i) {
        z[s0 + i] = zz[i];
        v[0] += rr[i] * rr[i];
        v[1] += rr[i] * zz[i];
      }
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
    const long long it = st->it;
    const double rel = sqrt(tot[0]) / st->gnorm;
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
      st->beta = tot[1] / st->rz;
      st->rz = tot[1];
    }
  }
}

__global__ void k_pupdate(int64_t s, const double* __restrict__ z, double* __restrict__ p, PcgState* st,
                          cudaGraphConditionalHandle h, int use_cond) {
  const int status = st->status;
  if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, status == 0 ? 1u : 0u);
  if (status) return;
  const double b = st->beta;
  // 16-byte vectors (the PCG vectors are 16-byte aligned, s may be odd)
  const int64_t n2 = s >> 1;
  const double2* z2 = reinterpret_cast<const double2*>(z);
  double2* p2 = reinterpret_cast<double2*>(p);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += int64_t(gridDim.x) * blockDim.x) {
    const double2 zz = z2[i];
    double2 pp = p2[i];
    pp.x = zz.x + b * pp.x;
    pp.y = zz.y + b * pp.y;
    p2[i] = pp;
  }
  if ((s & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[s - 1] = z[s - 1] + b * p[s - 1];
}

// ---------------------------------------------------------------------------
// Persistent PCG for uniform 3x3 systems: the whole solve is one cooperative
// launch.  Phases (SpMV + pHp, update + precondition + dots, p update) are
// separated by a grid barrier; after each barrier every CTA reduces the same
// per-CTA partials in the same fixed order, so all CTAs hold bit-identical
// alpha / beta / status without a last-CTA round trip (deterministic).

// SH = 0: row gather from upper storage (ys_spmv.cuh); SH > 0: the sliced-ELL
// full copy with SH lanes per block row (ys_sell.cuh).
template <int TB, int MINB, int SH>
__global__ void __launch_bounds__(TB, MINB) k_pcg33_persistent(SpmvDev S0, SpmvDev S1, SellDev SL, int has1, int64_t nb,
                                                             const double* __restrict__ minv, double* __restrict__ x,
                                                             double* __restrict__ r, double* __restrict__ z,
                                                             double* __restrict__ p, double* __restrict__ hp,
                                                             PcgState* st, double* part, double* hist, GridBar* gb) {
  constexpr int SW = kSpmvSW;
  const int G = gridDim.x;
  const int lane = threadIdx.x % SW;
  const int64_t sw0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / SW;
  const int64_t nsw = int64_t(G) * blockDim.x / SW;
  const unsigned mask = ((1u << SW) - 1u) << ((threadIdx.x & 31) & ~(SW - 1));
  const double gnorm = st->gnorm;
  const double tol = st->tol;
  const long long max_iter = st->max_iter;
  const long long hist_cap = st->hist_cap;
  double rz = st->rz;
  int status = st->status;
  long long it = 0;
  double rel = st->rel, php = 0.0, alpha = 0.0;
  unsigned long long ph[4] = {0, 0, 0, 0};
  unsigned long long epoch = 0;  // grid barriers passed (the counter is zeroed before the launch)
  unsigned long long t0 = gtimer();
  while (status == 0) {
    // ---- phase A: hp = H p, pHp partials
    double dot[1] = {0.0};
    if constexpr (SH > 0) {
      const int wl = threadIdx.x & 31;
      const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
      const int64_t nw = (int64_t(G) * blockDim.x) >> 5;
      for (int64_t sl = w0; sl < SL.nslices; sl += nw) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        int64_t R;
        sell_acc<SH>(SL, sl, wl, p, a0, a1, a2, R);
        if (wl % SH == 0 && R < nb) {
          double* yo = hp + 3 * R;
          yo[0] = a0;
          yo[1] = a1;
          yo[2] = a2;
          dot[0] += p[3 * R] * a0 + p[3 * R + 1] * a1 + p[3 * R + 2] * a2;
        }
      }
    }
    for (int64_t R = SH > 0 ? nb : sw0; R < nb; R += nsw) {
      const RowPtrs p0 = load_rowptrs(S0, R);
      RowPtrs p1{0, 0, 0, 0};
      if (has1) p1 = load_rowptrs(S1, R);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      acc33_u2<SW>(S0, p0, lane, p, a0, a1, a2);
      if (has1) acc33_u2<SW>(S1, p1, lane, p, a0, a1, a2);
#pragma unroll
      for (int off = SW / 2; off > 0; off >>= 1) {
        a0 += __shfl_xor_sync(mask, a0, off, SW);
        a1 += __shfl_xor_sync(mask, a1, off, SW);
        a2 += __shfl_xor_sync(mask, a2, off, SW);
      }
      if (lane == 0) {
        double* yo = hp + 3 * R;
        yo[0] = a0;
        yo[1] = a1;
        yo[2] = a2;
        dot[0] += p[3 * R] * a0 + p[3 * R + 1] * a1 + p[3 * R + 2] * a2;
      }
    }
    block_reduce<1>(dot);
    if (threadIdx.x == 0) part[blockIdx.x] = dot[0];
    grid_sync_counter(&gb->arrivals, (unsigned long long)G * ++epoch);
    unsigned long long t1 = gtimer();
    ph[0] += t1 - t0;
    t0 = t1;
    double tot1[1];
    reduce_partials_all<1>(part, G, tot1);
    php = tot1[0];
    if (!isfinite(php) || php <= 0.0) {
      status = php == 0.0 ? 2 : 3;
      break;
    }
    alpha = rz / php;
    // ---- phase B: x += a p, r -= a hp, z = M^-1 r, partials of r.r and r.z
    double v[2] = {0.0, 0.0};
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nb; b += int64_t(G) * blockDim.x) {
      const int64_t s0 = 3 * b;
      double pp[3], hh[3], rr[3], xx[3], zz[3], M[9];
      load_vec3(p + s0, pp[0], pp[1], pp[2]);
      load_vec3_cg(hp + s0, hh[0], hh[1], hh[2]);
      load_vec3(r + s0, rr[0], rr[1], rr[2]);
      load_vec3(x + s0, xx[0], xx[1], xx[2]);
      load_block9(minv + 9 * b, M);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        xx[i] += alpha * pp[i];
        rr[i] -= alpha * hh[i];
      }
      precond_apply<3>(M, rr, zz);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        x[s0 + i] = xx[i];
        r[s0 + i] = rr[i];
        z[s0 + i] = zz[i];
        v[0] += rr[i] * rr[i];
        v[1] += rr[i] * zz[i];
      }
    }
    block_reduce<2>(v);
    if (threadIdx.x == 0) {
      part[G + blockIdx.x] = v[0];
      part[2 * G + blockIdx.x] = v[1];
    }
    grid_sync_counter(&gb->arrivals, (unsigned long long)G * ++epoch);
    t1 = gtimer();
    ph[1] += t1 - t0;
    t0 = t1;
    double tot2[2];
    reduce_partials_all<2>(part + G, G, tot2);
    t1 = gtimer();
    ph[2] += t1 - t0;
    t0 = t1;
    rel = sqrt(tot2[0]) / gnorm;
    if (blockIdx.x == 0 && threadIdx.x == 0 && it + 1 < hist_cap) hist[it + 1] = rel;
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
    // ---- phase C: p = z + beta p
    {
      const int64_t n2 = (3 * nb) >> 1;
      const double2* z2 = reinterpret_cast<const double2*>(z);
      double2* p2 = reinterpret_cast<double2*>(p);
      for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += int64_t(G) * blockDim.x) {
        const double2 zz = __ldcg(z2 + i);
        double2 q = p2[i];
        q.x = zz.x + beta * q.x;
        q.y = zz.y + beta * q.y;
        p2[i] = q;
      }
      if (((3 * nb) & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[3 * nb - 1] = z[3 * nb - 1] + beta * p[3 * nb - 1];
    }
    grid_sync_counter(&gb->arrivals, (unsigned long long)G * ++epoch);
    t1 = gtimer();
    ph[3] += t1 - t0;
    t0 = t1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->it += it;
    st->rel = rel;
    st->rz = rz;
    st->php = php;
    st->alpha = alpha;
    st->status = status;
    if (status == 3 || status == 4) st->fail_it = int(it - (status == 4 ? 1 : 0));
    for (int k = 0; k < 4; ++k) st->phase_ns[k] = ph[k];
  }
}

// ---------------------------------------------------------------------------
// Persistent PCG over a streamed copy of H (ys_sell.cuh): one cooperative
// launch per solve.  Phase A (SpMV + pHp partials) is a policy:
//  * SellPhaseA — the sliced-ELL full copy: warp w of CTA b owns the slices
//    gw + k NW (gw = b * 8 + w, k < K).  Its SpMV plan (each slice's first
//    entry row, each lane's entry count, the column DoFs of all its entries)
//    is loaded into shared memory once, so every SpMV issues the x gathers
//    together with the value stream (C5 phase A 51 -> 45 us);
//  (a warp-range symmetric copy — Morton-ordered row ranges per warp, blocks
//   inside a range stored once with their transposed products through
//   shared-memory slots — cut the entries by ~20% but not the time: phase A
//   45.1 vs 44.7 us at C5, 26.2 vs 17.6 us at C4; profiles/r01_pcg_sell_c5.md)
// Phases B and C keep one thread per block row over global vectors
// (independent loads; a shared-memory row state with the slice mapping was
// measured slower: its per-row chains are latency-bound).  Fixed-order
// reductions (deterministic).
template <class PA>
__global__ void __launch_bounds__(kTB, kSpmvMinB) k_pcg33_stream(PA A, int64_t nb, const double* __restrict__ minv,
                                                               double* __restrict__ x, double* __restrict__ r,
                                                               double* __restrict__ z, double* __restrict__ p,
                                                               double* __restrict__ hp, PcgState* st, double* part,
                                                               double* hist, GridBar* gb) {
  extern __shared__ double smem[];
  const int G = gridDim.x;
  A.prologue(smem);
  const uint64_t kpol = l2_keep_policy();
  const int64_t nth = int64_t(G) * blockDim.x;
  const int64_t b0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool has0 = b0 < nb;
  const double gnorm = st->gnorm;
  const double tol = st->tol;
  const long long max_iter = st->max_iter;
  const long long hist_cap = st->hist_cap;
  double rz = st->rz;
  int status = st->status;
  long long it = 0;
  double rel = st->rel, php = 0.0, alpha = 0.0;
  unsigned long long ph[4] = {0, 0, 0, 0};
  unsigned long long aux[2] = {0, 0};
  unsigned long long epoch = 0;
  unsigned long long* cnt = &gb->arrivals;
  unsigned long long t0 = gtimer();
  while (status == 0) {
    // ---- phase A: hp = H p, pHp partials
    double dot[1] = {A.run(p, hp)};
    block_reduce<1>(dot);
    if (threadIdx.x == 0) part[blockIdx.x] = dot[0];
    grid_arrive(cnt);
    // phase B operands that no CTA writes in phase A: pulled into L2 under the barrier
    if (has0) {
      prefetch_l2(p + 3 * b0);
      prefetch_l2(r + 3 * b0);
      prefetch_l2(x + 3 * b0);
      prefetch_l2(minv + 9 * b0);
      prefetch_l2(minv + 9 * b0 + 8);
    }
    grid_wait(cnt, (unsigned long long)G * ++epoch);
    unsigned long long t1 = gtimer();
    ph[0] += t1 - t0;
    t0 = t1;
    double tot1[1];
    reduce_partials_all<1>(part, G, tot1);
    php = tot1[0];
    if (!isfinite(php) || php <= 0.0) {
      status = php == 0.0 ? 2 : 3;
      break;
    }
    alpha = rz / php;
    // ---- phase B: x += a p, r -= a hp, z = M^-1 r, partials of r.r and r.z
    double v[2] = {0.0, 0.0};
    for (int64_t b = b0; b < nb; b += nth) {
      RowRegs q;
      rowregs_load(q, b, p, r, x, minv, kpol);
      rowregs_update(q, b, alpha, hp, x, r, v, kpol);
#pragma unroll
      for (int i = 0; i < 3; ++i) st_keep(z + 3 * b + i, q.z[i], kpol);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) aux[0] += gtimer() - t0;  // sub-phase: rows done (CTA 0 thread 0)
    block_reduce<2>(v);
    if (threadIdx.x == 0) {
      part[G + blockIdx.x] = v[0];
      part[2 * G + blockIdx.x] = v[1];
    }
    grid_arrive(cnt);
    if (blockIdx.x == 0 && threadIdx.x == 0) aux[1] += gtimer() - t0;  // arrived
    grid_wait(cnt, (unsigned long long)G * ++epoch);
    t1 = gtimer();
    ph[1] += t1 - t0;
    t0 = t1;
    double tot2[2];
    reduce_partials_all<2>(part + G, G, tot2);
    t1 = gtimer();
    ph[2] += t1 - t0;
    t0 = t1;
    rel = sqrt(tot2[0]) / gnorm;
    if (blockIdx.x == 0 && threadIdx.x == 0 && it + 1 < hist_cap) hist[it + 1] = rel;
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
    // ---- phase C: p = z + beta p (this thread's own rows: z is its own write)
    for (int64_t b = b0; b < nb; b += nth) {
      double zz[3], pp[3];
      load_vec3_keep(z + 3 * b, zz[0], zz[1], zz[2], kpol);
      load_vec3_keep(p + 3 * b, pp[0], pp[1], pp[2], kpol);
#pragma unroll
      for (int i = 0; i < 3; ++i) st_keep(p + 3 * b + i, zz[i] + beta * pp[i], kpol);
    }
    grid_arrive(cnt);
    grid_wait(cnt, (unsigned long long)G * ++epoch);
    t1 = gtimer();
    ph[3] += t1 - t0;
    t0 = t1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->it += it;
    st->rel = rel;
    st->rz = rz;
    st->php = php;
    st->alpha = alpha;
    st->status = status;
    if (status == 3 || status == 4) st->fail_it = int(it - (status == 4 ? 1 : 0));
    for (int k = 0; k < 4; ++k) st->phase_ns[k] = ph[k];
    st->aux_ns[0] = aux[0];
    st->aux_ns[1] = aux[1];
  }
}

// ---------------------------------------------------------------------------
// Persistent PCG for mixed block sizes (affine bodies: 9 + 3 DoF rows next to
// 3-DoF vertices; C3): the graph-looped kernels cost ~47 us per iteration in
// launch latency on small systems.  Same phases and fixed-order reductions as
// k_pcg33_stream; phase A is a warp per block row of each block-size class
// (acc_gen), phases B / C one thread per block row / DoF.
struct GenClasses {
  int n;
  int rc[8];
  const int32_t* rows[8];  // null: all block rows (single class)
  int64_t nrows[8];
};

template <int RC>
__device__ __forceinline__ double gen_row(const SpmvDev& S0, const SpmvDev& S1, int has1, const BlocksDev& B,
                                          int64_t R, int lane, const double* __restrict__ p, double* __restrict__ hp) {
  double acc[RC];
#pragma unroll
  for (int i = 0; i < RC; ++i) acc[i] = 0.0;
  acc_gen<RC>(S0, R, lane, p, acc);
  if (has1) acc_gen<RC>(S1, R, lane, p, acc);
#pragma unroll
  for (int i = 0; i < RC; ++i)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
  double dot = 0.0;
  if (lane == 0) {
    const int64_t s0 = B.start[R];
#pragma unroll
    for (int i = 0; i < RC; ++i) {
      hp[s0 + i] = acc[i];
      dot += p[s0 + i] * acc[i];
    }
  }
  return dot;
}

template <int N>
__device__ __forceinline__ void gen_update(const BlocksDev& B, int64_t b, double alpha, const double* __restrict__ minv,
                                           double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                           const double* __restrict__ p, const double* __restrict__ hp,
                                           double (&v)[2]) {
  const int64_t s0 = B.start[b];
  double rr[N], zz[N], pp[N], xx[N], hh[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    pp[i] = p[s0 + i];
    xx[i] = x[s0 + i];
    rr[i] = r[s0 + i];
    hh[i] = __ldcg(hp + s0 + i);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    x[s0 + i] = xx[i] + alpha * pp[i];
    rr[i] = rr[i] - alpha * hh[i];
    r[s0 + i] = rr[i];
  }
  precond_apply<N>(minv + B.voff[b], rr, zz);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    z[s0 + i] = zz[i];
    v[0] += rr[i] * rr[i];
    v[1] += rr[i] * zz[i];
  }
}

__global__ void __launch_bounds__(kTB) k_pcg_gen_persistent(SpmvDev S0, SpmvDev S1, int has1, BlocksDev B,
                                                            GenClasses cls, int64_t s, const double* __restrict__ minv,
                                                            double* __restrict__ x, double* __restrict__ r,
                                                            double* __restrict__ z, double* __restrict__ p,
                                                            double* __restrict__ hp, PcgState* st, double* part,
                                                            double* hist, GridBar* gb) {
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(G) * blockDim.x) >> 5;
  const int64_t t0i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = int64_t(G) * blockDim.x;
  const double gnorm = st->gnorm;
  const double tol = st->tol;
  const long long max_iter = st->max_iter;
  const long long hist_cap = st->hist_cap;
  double rz = st->rz;
  int status = st->status;
  long long it = 0;
  double rel = st->rel, php = 0.0, alpha = 0.0;
  unsigned long long epoch = 0;
  unsigned long long ph[4] = {0, 0, 0, 0};
  unsigned long long t0 = gtimer();
  while (status == 0) {
    // ---- phase A: hp = H p per block-size class, pHp partials
    double dot[1] = {0.0};
    for (int k = 0; k < cls.n; ++k) {
      const int rc = cls.rc[k];
      for (int64_t q = w0; q < cls.nrows[k]; q += nw) {
        const int64_t R = cls.rows[k] ? cls.rows[k][q] : q;
        switch (rc) {
          case 1: dot[0] += gen_row<1>(S0, S1, has1, B, R, lane, p, hp); break;
          case 2: dot[0] += gen_row<2>(S0, S1, has1, B, R, lane, p, hp); break;
          case 3: dot[0] += gen_row<3>(S0, S1, has1, B, R, lane, p, hp); break;
          case 4: dot[0] += gen_row<4>(S0, S1, has1, B, R, lane, p, hp); break;
          case 6: dot[0] += gen_row<6>(S0, S1, has1, B, R, lane, p, hp); break;
          case 9: dot[0] += gen_row<9>(S0, S1, has1, B, R, lane, p, hp); break;
          default: dot[0] += gen_row<12>(S0, S1, has1, B, R, lane, p, hp); break;
        }
      }
    }
    block_reduce<1>(dot);
    if (threadIdx.x == 0) part[blockIdx.x] = dot[0];
    grid_sync_counter(&gb->arrivals, (unsigned long long)G * ++epoch);
    unsigned long long t1 = gtimer();
    ph[0] += t1 - t0;
    t0 = t1;
    double tot1[1];
    reduce_partials_all<1>(part, G, tot1);
    php = tot1[0];
    if (!isfinite(php) || php <= 0.0) {
      status = php == 0.0 ? 2 : 3;
      break;
    }
    alpha = rz / php;
    // ---- phase B: x += a p, r -= a hp, z = M^-1 r per block row, partials of r.r and r.z
    double v[2] = {0.0, 0.0};
    for (int64_t b = t0i; b < B.nb; b += nth) {
      const int rc = B.rc[b];
      switch (rc) {  // unrolled (independent loads) for the common sizes
        case 3: gen_update<3>(B, b, alpha, minv, x, r, z, p, hp, v); break;
        case 9: gen_update<9>(B, b, alpha, minv, x, r, z, p, hp, v); break;
        case 12: gen_update<12>(B, b, alpha, minv, x, r, z, p, hp, v); break;
        default: {
          const int64_t s0 = B.start[b];
          double rr[16], zz[16];
          for (int i = 0; i < rc; ++i) {
            x[s0 + i] += alpha * p[s0 + i];
            rr[i] = r[s0 + i] - alpha * __ldcg(hp + s0 + i);
            r[s0 + i] = rr[i];
          }
          precond_apply_any(rc, minv + B.voff[b], rr, zz);
          for (int i = 0; i < rc; ++i) {
            z[s0 + i] = zz[i];
            v[0] += rr[i] * rr[i];
            v[1] += rr[i] * zz[i];
          }
        }
      }
    }
    block_reduce<2>(v);
    if (threadIdx.x == 0) {
      part[G + blockIdx.x] = v[0];
      part[2 * G + blockIdx.x] = v[1];
    }
    grid_sync_counter(&gb->arrivals, (unsigned long long)G * ++epoch);
    t1 = gtimer();
    ph[1] += t1 - t0;
    t0 = t1;
    double tot2[2];
    reduce_partials_all<2>(part + G, G, tot2);
    t1 = gtimer();
    ph[2] += t1 - t0;
    t0 = t1;
    rel = sqrt(tot2[0]) / gnorm;
    if (blockIdx.x == 0 && threadIdx.x == 0 && it + 1 < hist_cap) hist[it + 1] = rel;
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
    // ---- phase C: p = z + beta p
    for (int64_t i = t0i; i < s; i += nth) p[i] = __ldcg(z + i) + beta * p[i];
    grid_sync_counter(&gb->arrivals, (unsigned long long)G * ++epoch);
    t1 = gtimer();
    ph[3] += t1 - t0;
    t0 = t1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->it += it;
    st->rel = rel;
    st->rz = rz;
    st->php = php;
    st->alpha = alpha;
    st->status = status;
    if (status == 3 || status == 4) st->fail_it = int(it - (status == 4 ? 1 : 0));
    for (int k = 0; k < 4; ++k) st->phase_ns[k] = ph[k];
  }
}

// ---------------------------------------------------------------------------
// Host side

void spmv_launch(Context& c, Structure& s0, Structure* s1, const double* x, double* y, bool accumulate,
                 PcgState* st, double* part, int grid) {
  const bool has1 = s1 && s1->n_blocks > 0;
  const bool fast = c.uniform3 && s0.all33 && (!has1 || s1->all33);
  SpmvDev d0 = spmv_dev(s0);
  SpmvDev d1 = has1 ? spmv_dev(*s1) : d0;
  if (fast) {
    static int occ = 0;
    if (!occ) {
      YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv33, kTB, 0));
      if (occ < 1) occ = 1;
    }
    const int g = std::max(1, std::min(grid, occ * sm_count()));
    k_spmv33<<<g, kTB, 0, c.stream>>>(d0, d1, has1 ? 1 : 0, c.NB, x, y, accumulate ? 1 : 0, st, part);
    YS_LAUNCH_CHECK();
    return;
  }
  const BlocksDev B = blocks_view(c);
  for (size_t k = 0; k < c.rc_classes.size(); ++k) {
    const int rc = c.rc_classes[k];
    const int32_t* rows = c.rc_classes.size() == 1 ? nullptr : c.rc_lists[k].p;
    const int64_t nrows = c.rc_classes.size() == 1 ? c.NB : int64_t(c.rc_lists[k].n);
    if (nrows == 0) continue;
    const int g = int(std::min<int64_t>(grid, ceil_div(nrows * 32, kTB)));
#define YS_GEN(RC)                                                                                         \
  case RC:                                                                                                 \
    k_spmv_gen<RC><<<g, kTB, 0, c.stream>>>(d0, d1, has1 ? 1 : 0, B, rows, nrows, x, y, accumulate ? 1 : 0, st); \
    break;
    switch (rc) {
      YS_GEN(1)
      YS_GEN(2)
      YS_GEN(3)
      YS_GEN(4)
      YS_GEN(6)
      YS_GEN(9)
      YS_GEN(12)
      default:
        fail(YS_ERR_INTERNAL, "unsupported block size in SpMV");
    }
#undef YS_GEN
    YS_LAUNCH_CHECK();
  }
  if (part) {
    k_dot_alpha<<<grid, kTB, 0, c.stream>>>(c.s, x, y, st, part);
    YS_LAUNCH_CHECK();
  }
}

// Diagnostic: n grid barriers (and n fixed-order partial reductions) at the
// persistent PCG's grid, to price the per-iteration synchronisation.  Bit 1:
// counter barrier (production) instead of the generation barrier; bit 0: +
// reduce_partials_all.  Measured on B200 at 444 CTAs: generation barrier
// 3.1 us, counter barrier 2.2 us, + reduction ~1.1 us.  Also measured and
// dropped: 32 striped counters 3.5 us, relaxed polling 2.3 us, 256 ns backoff
// 2.6 us, master release through per-CTA flag lines 4.3 us.

void ctx_apply_hessian_dev(Context& c, const double* x, double* y) {
  spmv_launch(c, c.S[0], &c.S[1], x, y, true, nullptr, nullptr, std::max(1, sm_count() * 8));
}

// Grids of the vector kernels: one thread per block row (update) or per
// 16-byte pair (p-update), capped at one resident wave.
static int vec_grid(Context& c, int64_t work) {
  static int occ = 0;
  if (!occ) {
    YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update, kTB, 0));
    if (occ < 1) occ = 1;
  }
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, kTB), int64_t(occ) * sm_count())));
}

static void launch_iteration(Context& c, int grid, cudaGraphConditionalHandle h, bool use_cond) {
  PcgState* st = c.pcg.p;
  spmv_launch(c, c.S[0], &c.S[1], c.p.p, c.hp.p, false, st, c.partials.p, grid);
  k_update<<<vec_grid(c, c.NB), kTB, 0, c.stream>>>(blocks_view(c), c.uniform3 ? 1 : 0, c.minv.p, c.DX.p, c.r.p,
                                                     c.z.p, c.p.p, c.hp.p, st, c.partials.p, c.hist.p);
  YS_LAUNCH_CHECK();
  k_pupdate<<<vec_grid(c, (c.s + 1) / 2), kTB, 0, c.stream>>>(c.s, c.z.p, c.p.p, st, h, use_cond ? 1 : 0);
  YS_LAUNCH_CHECK();
}

static bool build_conditional_graph(Context& c, int grid) {
  cudaGraph_t g = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return false;
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) {
    cudaGraphDestroy(g);
    cudaGetLastError();
    return false;
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) {
    cudaGraphDestroy(g);
    cudaGetLastError();
    return false;
  }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess) {
    cudaGraphDestroy(g);
    cudaGetLastError();
    return false;
  }
  launch_iteration(c, grid, h, true);
  cudaGraph_t out = nullptr;
  if (cudaStreamEndCapture(c.stream, &out) != cudaSuccess) {
    cudaGraphDestroy(g);
    cudaGetLastError();
    return false;
  }
  cudaGraphExec_t exec = nullptr;
  if (cudaGraphInstantiate(&exec, g, 0) != cudaSuccess) {
    cudaGraphDestroy(g);
    cudaGetLastError();
    return false;
  }
  c.pcg_graph = g;
  c.pcg_exec = exec;
  c.pcg_cond = true;
  return true;
}

static void build_chunk_graph(Context& c, int grid, int chunk) {
  cudaGraph_t g = nullptr;
  YS_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < chunk; ++k) launch_iteration(c, grid, cudaGraphConditionalHandle{}, false);
  YS_CUDA(cudaStreamEndCapture(c.stream, &g));
  YS_CUDA(cudaGraphInstantiate(&c.pcg_exec, g, 0));
  c.pcg_graph = g;
  c.pcg_cond = false;
}

void drop_pcg_graph(Context& c) {
  if (c.pcg_exec) cudaGraphExecDestroy(c.pcg_exec);
  if (c.pcg_graph) cudaGraphDestroy(c.pcg_graph);
  c.pcg_exec = nullptr;
  c.pcg_graph = nullptr;
}

int pcg_grid(Context& c) { return std::max(1, sm_count() * 8); }

// The layout half of the uniform-3x3 solve's sliced-ELL copy (sell_prepare):
// built right after the dynamic rebuild, while the static evaluation still runs
// on the side streams.
void pcg_prepare(Context& c) {
  const bool has1 = c.S[1].n_blocks > 0;
  const bool fast = c.uniform3 && c.S[0].all33 && (!has1 || c.S[1].all33);
  if (fast) sell_prepare(c, 4);
}

void ctx_pcg(Context& c, double tol, int64_t max_iter, const double* g_dev, double* x_dev, ys_step_stats* stats) {
  cudaStream_t s = c.stream;
  const int grid = pcg_grid(c);
  c.r.resize(c.s + 2);
  c.z.resize(c.s + 2);
  c.p.resize(c.s + 2);
  c.hp.resize(c.s + 2);
  c.pcg.resize(1);
  c.partials.resize(std::max<size_t>(c.partials.n, size_t(2 * grid)));
  const int64_t hist_cap = std::min<int64_t>(max_iter, int64_t(1) << 22) + 2;
  c.hist.resize(std::max<size_t>(c.hist.n, size_t(hist_cap)));
  if (x_dev != c.DX.p) fail(YS_ERR_INTERNAL, "pcg: solution must live in the step buffer");
  (void)g_dev;
  PcgState init{};
  init.tol = tol;
  init.max_iter = max_iter;
  init.hist_cap = int64_t(c.hist.n);
  YS_CUDA(cudaMemcpyAsync(c.pcg.p, &init, sizeof(PcgState), cudaMemcpyHostToDevice, s));
  k_pcg_init<<<grid, kTB, 0, s>>>(blocks_view(c), c.uniform3 ? 1 : 0, c.G.p, c.minv.p, c.r.p, c.z.p, c.p.p, c.DX.p,
                                  c.pcg.p, c.partials.p, c.hist.p);
  YS_LAUNCH_CHECK();

  // Uniform 3x3 systems: one persistent cooperative kernel runs the whole solve
  // over the sliced-ELL full copy; when its per-warp plan does not fit the
  // shared memory (systems several times C5 per GPU), over the row gather from
  // upper storage.  The path taken is reported (ys_stage_times counts[2]).
  {
    const bool has1 = c.S[1].n_blocks > 0;
    const bool fast = c.uniform3 && c.S[0].all33 && (!has1 || c.S[1].all33);
    if (fast) {
      int64_t nb = c.NB;
      const double* minv = c.minv.p;
      double *xp = c.DX.p, *rp = c.r.p, *zp = c.z.p, *pp = c.p.p, *hpp = c.hp.p, *hist = c.hist.p;
      PcgState* stp = c.pcg.p;
      bool launched = false;
      c.gridbar.resize(sizeof(GridBar));
      GridBar* gbp = reinterpret_cast<GridBar*>(c.gridbar.p);
      YS_CUDA(cudaMemsetAsync(c.gridbar.p, 0, sizeof(GridBar), s));
      if (!launched && c.pcg_copy) {
        // full sliced-ELL copy, per-warp plan cache in shared memory
        sell_build(c, 4);
        SellDev sl = sell_dev(c);
        void* kern = (void*)k_pcg33_stream<SellPhaseA>;
        const int wpb = kTB / 32;
        for (int per = c.pcg_ctas > 0 ? std::min(c.pcg_ctas, kSpmvMinB) : kSpmvMinB; per >= 1 && !launched; --per) {
          // small systems: no more CTAs than give every warp two slices (at
          // least one per SM) — the grid barriers get cheaper with fewer CTAs
          int gsz = int(std::min<int64_t>(int64_t(per) * sm_count(),
                                          std::max<int64_t>(sm_count(), ceil_div(c.sell_slices, int64_t(wpb) * 2))));
          int K = int(ceil_div(c.sell_slices, int64_t(gsz) * wpb));
          int TW = sell_max_warp_rows(c, int64_t(gsz) * wpb, K);
          const size_t smem = size_t(wpb) * K * 8 + size_t(wpb) * K * 32 * 4 + size_t(wpb) * TW * 32 * 4;
          if (smem > size_t(220 * 1024) / per) continue;
          YS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
          int occ = 0;
          YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTB, smem));
          if (occ < per) continue;
          c.partials.resize(std::max<size_t>(c.partials.n, size_t(3 * gsz)));
          double* part = c.partials.p;
          SellPhaseA A{};
          A.SL = sl;
          A.nb = nb;
          A.K = K;
          A.TW = TW;
          void* args[] = {&A, &nb, &minv, &xp, &rp, &zp, &pp, &hpp, &stp, &part, &hist, &gbp};
          YS_CUDA(cudaLaunchCooperativeKernel(kern, dim3(gsz), dim3(kTB), args, smem, s));
          launched = true;
          c.pcg_path = 1;
        }
      }
      if (!launched) {
        // row gather from upper storage (no copy, no shared-memory plan):
        // ~0.36 of HBM against the copy's ~0.54 — said once per context, and
        // reported by ys_stage_times (counts[2] = 2)
        if (c.pcg_copy && !c.warned_pcg_fallback) {
          std::fprintf(stderr,
                       "yasps_b200: the sliced-ELL PCG plan (%lld slices) does not fit in shared memory; "
                       "solving over the slower row gather from upper storage\n",
                       (long long)c.sell_slices);
          c.warned_pcg_fallback = true;
        }
        void* kern = reinterpret_cast<void*>(k_pcg33_persistent<kTB, kSpmvMinB, 0>);
        int occ = 0;
        YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTB, 0));
        if (occ < 1) occ = 1;
        int gsz = occ * sm_count();
        c.partials.resize(std::max<size_t>(c.partials.n, size_t(3 * gsz)));
        SpmvDev d0 = spmv_dev(c.S[0]);
        SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
        SellDev sl{};
        int h1 = has1 ? 1 : 0;
        double* part = c.partials.p;
        void* args[] = {&d0, &d1, &sl, &h1, &nb, &minv, &xp, &rp, &zp, &pp, &hpp, &stp, &part, &hist, &gbp};
        YS_CUDA(cudaLaunchCooperativeKernel(kern, dim3(gsz), dim3(kTB), args, 0, s));
        c.pcg_path = 2;
      }
      PcgState fin{};
      YS_CUDA(cudaMemcpyAsync(&fin, c.pcg.p, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      YS_CUDA(cudaStreamSynchronize(s));
      c.launches += 2;
      for (int k = 0; k < 4; ++k) c.pcg_phase_ms[k] = double(fin.phase_ns[k]) * 1e-6;
      for (int k = 0; k < 4; ++k) c.pcg_phase_ms[4 + k] = double(fin.aux_ns[k]) * 1e-6;
      c.hist_count = fin.status == 1 && fin.it == 0 && fin.gnorm == 0.0 ? 0 : fin.it + 1;
      if (fin.status == 3)
        fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) +
                                   " (non-finite or negative curvature)");
      if (fin.status == 4)
        fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) +
                                   " (non-finite residual)");
      if (stats) {
        stats->pcg_iterations = fin.it;
        stats->pcg_converged = fin.status == 1 ? 1 : 0;
        stats->pcg_residual = (fin.gnorm == 0.0) ? 0.0 : fin.rel;
      }
      return;
    }
  }
  // Mixed block sizes: one persistent cooperative kernel (YS_PCG_GEN=graph keeps
  // the graph-looped kernels).
  if (c.rc_classes.size() <= 8) {
    GenClasses cls{};
    cls.n = int(c.rc_classes.size());
    for (int k = 0; k < cls.n; ++k) {
      cls.rc[k] = c.rc_classes[size_t(k)];
      cls.rows[k] = c.rc_classes.size() == 1 ? nullptr : c.rc_lists[size_t(k)].p;
      cls.nrows[k] = c.rc_classes.size() == 1 ? c.NB : int64_t(c.rc_lists[size_t(k)].n);
    }
    bool ok = true;
    for (int k = 0; k < cls.n; ++k) {
      const int rc = cls.rc[k];
      ok = ok && (rc == 1 || rc == 2 || rc == 3 || rc == 4 || rc == 6 || rc == 9 || rc == 12);
    }
    if (ok) {
      void* kern = reinterpret_cast<void*>(k_pcg_gen_persistent);
      int occ = 0;
      YS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTB, 0));
      occ = std::max(occ, 1);
      // small systems: fewer CTAs (cheaper barriers); at least one warp per 4 block rows
      const int64_t want = std::max<int64_t>(1, ceil_div(c.NB * 8, kTB));
      int gsz = int(std::min<int64_t>(int64_t(occ) * sm_count(), std::max<int64_t>(want, sm_count())));
      c.partials.resize(std::max<size_t>(c.partials.n, size_t(3 * gsz)));
      c.gridbar.resize(sizeof(GridBar));
      YS_CUDA(cudaMemsetAsync(c.gridbar.p, 0, sizeof(GridBar), s));
      const bool has1 = c.S[1].n_blocks > 0;
      SpmvDev d0 = spmv_dev(c.S[0]);
      SpmvDev d1 = has1 ? spmv_dev(c.S[1]) : d0;
      int h1 = has1 ? 1 : 0;
      BlocksDev B = blocks_view(c);
      int64_t sdofs = c.s;
      const double* minv = c.minv.p;
      double *xp = c.DX.p, *rp = c.r.p, *zp = c.z.p, *pp = c.p.p, *hpp = c.hp.p, *part = c.partials.p,
             *hist = c.hist.p;
      PcgState* stp = c.pcg.p;
      GridBar* gbp = reinterpret_cast<GridBar*>(c.gridbar.p);
      void* args[] = {&d0, &d1, &h1, &B, &cls, &sdofs, &minv, &xp, &rp, &zp, &pp, &hpp, &stp, &part, &hist, &gbp};
      YS_CUDA(cudaLaunchCooperativeKernel(kern, dim3(gsz), dim3(kTB), args, 0, s));
      PcgState fin{};
      YS_CUDA(cudaMemcpyAsync(&fin, c.pcg.p, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      YS_CUDA(cudaStreamSynchronize(s));
      c.launches += 2;
      for (int k = 0; k < 4; ++k) c.pcg_phase_ms[k] = double(fin.phase_ns[k]) * 1e-6;
      for (int k = 0; k < 4; ++k) c.pcg_phase_ms[4 + k] = double(fin.aux_ns[k]) * 1e-6;
      c.hist_count = fin.status == 1 && fin.it == 0 && fin.gnorm == 0.0 ? 0 : fin.it + 1;
      if (fin.status == 3)
        fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) +
                                   " (non-finite or negative curvature)");
      if (fin.status == 4)
        fail(YS_ERR_NUMERICAL, "PCG diverged at iteration " + std::to_string(fin.fail_it) +
                                   " (non-finite residual)");
      if (stats) {
        stats->pcg_iterations = fin.it;
        stats->pcg_converged = fin.status == 1 ? 1 : 0;
        stats->pcg_residual = (fin.gnorm == 0.0) ? 0.0 : fin.rel;
      }
      return;
    }
  }
  // graph cache key: every pointer / flag the captured launches bake in
  Structure& s0 = c.S[0];
  Structure& s1 = c.S[1];
  auto P = [](const void* q) { return uint64_t(uintptr_t(q)); };
  std::vector<uint64_t> key = {P(s0.sp_rowptr.p), P(s0.sp_ent.p), P(s0.values.p), P(s0.sp_oth.p), P(s0.nrow.p), P(s0.trow.p), P(s0.tlist.p), P(s0.col.p),
                               P(s0.br.p), P(s0.bc.p), P(s0.voff.p), P(s1.sp_rowptr.p), P(s1.sp_ent.p),
                               P(s1.values.p), P(s1.sp_oth.p), P(s1.nrow.p), P(s1.trow.p), P(s1.tlist.p), P(s1.col.p), P(s1.br.p), P(s1.bc.p), P(s1.voff.p),
                               P(c.DX.p), P(c.r.p), P(c.z.p), P(c.p.p), P(c.hp.p), P(c.minv.p), P(c.pcg.p),
                               P(c.partials.p), P(c.hist.p),
                               uint64_t(s1.n_blocks > 0) | (uint64_t(s0.all33) << 1) | (uint64_t(s1.all33) << 2),
                               uint64_t(grid), uint64_t(c.s)};
  PcgState fin{};
  // a device-side WHILE loop (conditional graph node); when the driver cannot
  // build one, graphs of 8 iterations with a status read per graph
  if (!c.pcg_exec || c.pcg_key != key) {
    drop_pcg_graph(c);
    if (!build_conditional_graph(c, grid)) build_chunk_graph(c, grid, 8);
    c.pcg_key = key;
  }
  if (c.pcg_cond) {
    YS_CUDA(cudaGraphLaunch(c.pcg_exec, s));
    YS_CUDA(cudaMemcpyAsync(&fin, c.pcg.p, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    YS_CUDA(cudaStreamSynchronize(s));
  } else {
    for (;;) {
      YS_CUDA(cudaMemcpyAsync(&fin, c.pcg.p, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      YS_CUDA(cudaStreamSynchronize(s));
      if (fin.status) break;
      YS_CUDA(cudaGraphLaunch(c.pcg_exec, s));
    }
  }
  c.launches += 2 + 3 * fin.it;
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

bool pcg_uses_conditional_graph(Context& c) { return c.pcg_cond; }

}  // namespace ys
