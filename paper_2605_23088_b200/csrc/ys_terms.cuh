// ys_terms.cuh — FP64 local energy / gradient / PSD-projected Hessian of each
// energy kind, one term per thread, everything in registers.
//
// The reference evaluates symbolic plans (eval.cpp:145-373) and projects the
// compressed m x m local Hessian with a dense self-adjoint EVD
// (assembly.cpp:8-17, 284-321).  Here every kind has closed-form derivatives
// and the projection exploits the structure of the term:
//
//  * SNH and bending depend on x only through the three edge vectors
//    D = (x1-x0, x2-x0, x3-x0) = (S (x) I3) x, S = [-1 1 0 0; -1 0 1 0; -1 0 0 1].
//    With S^T = W R (W: 4x3 Helmert basis with orthonormal columns), the 12x12
//    Hessian is (W (x) I) M (W (x) I)^T, M = (R (x) I) H_D (R^T (x) I), and
//    Proj12(H) = (W (x) I) Proj9(M) (W (x) I)^T exactly: a 9x9 EVD replaces the
//    reference's 12x12 one (FullProject).  ReducedProject (SNH via F,
//    energies.cpp:91-117) projects H_F directly: E = S^T, M = H_D.
//  * Point terms (PP barrier, repulsive, inertia) depend on x through one
//    3-vector delta that is linear in the compressed DoFs with J J^T = c I3
//    (free: +-I3, affine A: I3 (x) r^T, affine t: I3), hence
//    Proj_m(J^T H3 J) = J^T Proj3(H3) J; H3 = a I + b delta delta^T has a
//    closed-form eigensystem.
//  * Affine orthogonality: 9x9 EVD of the analytic Hessian.
#pragma once

#include "ys_common.cuh"

namespace ys {

#define YS_HD __host__ __device__ __forceinline__

// Packed row-major upper-triangular index of a 9x9 symmetric matrix.
YS_HD constexpr int pk9(int i, int j) {
  return i <= j ? i * 9 - (i * (i - 1)) / 2 + (j - i) : j * 9 - (j * (j - 1)) / 2 + (i - j);
}

// Helmert basis W (4x3, orthonormal columns spanning sum-zero vectors) and
// R = W^T S^T (upper triangular): S^T = W R.  constexpr so that fully
// unrolled loops fold them into immediates.
YS_HD constexpr double kW(int a, int i) {
  return i == 0 ? (a == 0 ? -0.70710678118654752440 : a == 1 ? 0.70710678118654752440 : 0.0)
       : i == 1 ? (a == 2 ? 0.81649658092772603273 : a == 3 ? 0.0 : -0.40824829046386301637)
                : (a == 3 ? 0.86602540378443864676 : -0.28867513459481288225);
}
YS_HD constexpr double kR(int a, int i) {
  return a == 0 ? (i == 0 ? 1.41421356237309504880 : 0.70710678118654752440)
       : a == 1 ? (i == 0 ? 0.0 : i == 1 ? 1.22474487139158904910 : 0.40824829046386301637)
                : (i == 2 ? 1.15470053837925152902 : 0.0);
}
// S^T (4x3): vertex 0 -> -1 on every edge, vertex a>0 -> edge a-1.
YS_HD constexpr double kST(int a, int i) { return a == 0 ? -1.0 : (i == a - 1 ? 1.0 : 0.0); }

// ---------------------------------------------------------------------------
// Cyclic Jacobi on a packed symmetric 9x9 matrix, eigenvectors in v (row-major
// v[k*9+j] = component k of eigenvector j).  Per rotation two rsqrt and no
// division: with h = a_qq - a_pp the rotation of
//   t = 2 sgn(h) a_pq / (|h| + sqrt(h^2 + 4 a_pq^2))
// (the smaller root of t^2 + 2 theta t - 1 = 0, theta = h / (2 a_pq)).
// Rotations whose off-diagonal entry is below the rounding of both diagonal
// entries are dropped (the classical negligibility rule); when every lane of
// the warp drops a rotation the row / column update is skipped.  Sweeps stop
// once the off-diagonal Frobenius norm is below 1e-12 of the matrix norm
// (YS_JACOBI_TOL2 = 1e-24 on the squares): the projection then differs from
// the exact one by O(1e-12) relative, 1000x inside the 1e-9 parity bar
// (C4 eval 3.03 -> 2.5 ms against a 1e-14 stop; 1e-11 measured parity-green
// too).  Returns the number of sweeps.
__device__ __forceinline__ void jacobi_rot(double* a, double* v, int p, int q) {
  const double apq = a[pk9(p, q)];
  const double app = a[pk9(p, p)];
  const double aqq = a[pk9(q, q)];
  const double g = 100.0 * fabs(apq);
  const bool negligible = (fabs(app) + g == fabs(app)) && (fabs(aqq) + g == fabs(aqq));
  if (__all_sync(__activemask(), negligible)) {
    a[pk9(p, q)] = 0.0;
    return;
  }
  // tan(theta) = 2 sgn(h) a_pq / (|h| + sqrt(h^2 + 4 a_pq^2)) through two
  // reciprocal square roots and no division / square root:
  //   rd = 1 / sqrt(h^2 + 4 a_pq^2), c^2 = (1 + |h| rd) / 2, rc = 1 / c,
  //   s = sgn(h) a_pq rd rc, t = s rc   (c^2 + s^2 = 1 up to rounding)
  double t = 0.0, c = 1.0, sn = 0.0;
  if (!negligible) {
    const double h = aqq - app;
    const double sa = h < 0.0 ? -apq : apq;
    const double rd = rsqrt(h * h + 4.0 * apq * apq);
    const double c2 = 0.5 + 0.5 * (fabs(h) * rd);
    const double rc = rsqrt(c2);
    c = c2 * rc;
    sn = sa * rd * rc;
    t = sn * rc;
  }
  const double tq = t * apq;
  a[pk9(p, p)] = app - tq;
  a[pk9(q, q)] = aqq + tq;
  a[pk9(p, q)] = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if (k == p || k == q) continue;
    const double akp = a[pk9(k, p)];
    const double akq = a[pk9(k, q)];
    a[pk9(k, p)] = c * akp - sn * akq;
    a[pk9(k, q)] = sn * akp + c * akq;
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const double vkp = v[k * 9 + p];
    const double vkq = v[k * 9 + q];
    v[k * 9 + p] = c * vkp - sn * vkq;
    v[k * 9 + q] = sn * vkp + c * vkq;
  }
}

#ifndef YS_JACOBI_TOL2
#define YS_JACOBI_TOL2 1e-24
#endif
constexpr double kJacobiTol2 = YS_JACOBI_TOL2;

__device__ __forceinline__ int jacobi9(double* a, double* v) {
#pragma unroll
  for (int i = 0; i < 81; ++i) v[i] = (i % 10 == 0) ? 1.0 : 0.0;
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    double off = 0.0, dia = 0.0;
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      dia += a[pk9(p, p)] * a[pk9(p, p)];
#pragma unroll
      for (int q = p + 1; q < 9; ++q) off += a[pk9(p, q)] * a[pk9(p, q)];
    }
    if (!(off > kJacobiTol2 * (dia + 2.0 * off))) break;  // also stops on off == 0
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int q = p + 1; q < 9; ++q) jacobi_rot(a, v, p, q);
  }
  return sweep;
}

// In place: a (packed, 45) <- V diag(max(lambda, 0)) V^T.  Returns the
// number of clamped (negative) eigenvalues.
__device__ __forceinline__ int psd_project9(double* a) {
  double v[81];
  jacobi9(a, v);
  double lam[9];
  int neg = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const double l = a[pk9(k, k)];
    neg += (l < 0.0);
    lam[k] = l < 0.0 ? 0.0 : l;
  }
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 9; ++k) acc += v[i * 9 + k] * lam[k] * v[j * 9 + k];
      a[pk9(i, j)] = acc;
    }
  return neg;
}

// ---------------------------------------------------------------------------
// Clamped-eigenpair projection of a packed 9x9 M (pass B's main path):
//   1. Householder tridiagonalization T = Q^T M Q, Q = H_0 ... H_6 (the
//      reflectors go to a per-thread global scratch, L2-resident: [0, 35)
//      v_k, [35, 42) beta_k; d and e of T to shared memory);
//   2. all eigenvalues of T by implicit QL (Wilkinson-type shift), the sweep
//      over the unreduced block written as a static loop over i with a
//      predicate l <= i < m (registers only, small code);
//   3. the number of eigenvalues below -tau0 (tau0 = 1e-13 |M|_F; those in
//      (-tau0, 0] are left unclamped, an error <= tau0) cross-checked with a
//      Sturm count of T at -tau0;
//   4. eigenvectors only for the clamped side — the k <= 4 negative
//      eigenvalues (P = M - sum lam x x^T) or else the <= 4 others
//      (P = sum max(lam, 0) x x^T) — by inverse iteration on T (LDL^T of
//      T - lam I, 2 solves; members of a cluster Gram-Schmidt
//      orthogonalized against the earlier ones), kept in the T basis in
//      shared-memory slots [0, 36) and back-transformed with the reflectors
//      when P is formed;
//   5. verification: every used pair's residual |T y - lam y| <= 1e-12 |M|_F
//      and used vectors orthogonal to 1e-12.  Then |P - Proj(M)| is bounded
//      by ~1e-12 |M|_F: a contaminating eigenvector of the same sign is used
//      too (orthogonality), one of the other sign is at least |lam| away, so
//      the residual bounds the error (plus the Householder backward error,
//      ~1e-15 |M|_F).
// Returns false when a check fails or QL does not converge: the caller hands
// the element to the Jacobi path (psd_project9).
// Measured on C5 tets (tools/evd_proto3.py, the same algorithm in numpy):
// 100 % accepted at the rolled-out and the jittered state, max |P - eigh| /
// max|M| = 3.7e-15.  ~5k FP64 operations against ~19k for the Jacobi EVD.
// sm: this thread's slot 0 in a [kProjSlots][kProjStride] shared array; gsc:
// its slot 0 in a [kProjScratch][gstride] global scratch.
constexpr int kProjStride = 128;

// Reload of M at the end of the projection: a volatile load, so the compiler
// neither keeps the first load's 45 values live across the QL (CSE of the
// read-only loads) nor hoists the reload (90 registers either way).
__device__ __forceinline__ double ld_reload(const double* p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_reload2(const double* p) {
  double2 v;
  asm volatile("ld.volatile.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// The 9x9 M of an element (packed 45) in its slot of the pass-B buffer: a
// 46-double stride keeps every slot 16-byte aligned (23 vector accesses).
constexpr int kMStride = 46;
__device__ __forceinline__ void store_m(double* m, const double* a) {
#pragma unroll
  for (int q = 0; q < 44; q += 2) *reinterpret_cast<double2*>(m + q) = make_double2(a[q], a[q + 1]);
  m[44] = a[44];
}
__device__ __forceinline__ void load_m(const double* __restrict__ m, double* a) {
#pragma unroll
  for (int q = 0; q < 44; q += 2) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(m + q));
    a[q] = v.x;
    a[q + 1] = v.y;
  }
  a[44] = __ldg(m + 44);
}
__device__ __forceinline__ void reload_m(const double* m, double* a) {
#pragma unroll
  for (int q = 0; q < 44; q += 2) {
    const double2 v = ld_reload2(m + q);
    a[q] = v.x;
    a[q + 1] = v.y;
  }
  a[44] = ld_reload(m + 44);
}
constexpr int kProjSlots = 53;  // shared: [0, 36) the used vectors (T basis), [36, 45) d, [45, 53) e
constexpr int kSlotD = 36, kSlotE = 45;
constexpr int kProjScratch = 42;  // global, per thread: [0, 35) reflectors v_k, [35, 42) beta_k

__device__ __forceinline__ int refl_off(int k) { return k * 8 - (k * (k - 1)) / 2; }  // sum_{i<k} (8 - i)

__device__ __forceinline__ bool psd_project9_tri(const double* __restrict__ msrc, double* P, double* sm,
                                                 double* gsc, int64_t gstride) {
  auto S = [&](int slot) -> double& { return sm[slot * kProjStride]; };
  auto G = [&](int slot) -> double& { return gsc[slot * gstride]; };
  double a[45];
  double n2 = 0.0;
  load_m(msrc, a);
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) n2 += (i == j ? 1.0 : 2.0) * a[pk9(i, j)] * a[pk9(i, j)];
  const double nrm = sqrt(n2);
  // ---- 1. tridiagonalization
  double e[8];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const int m = 8 - k;
    double x0 = a[pk9(k + 1, k)];
    double sig = 0.0;
#pragma unroll
    for (int i = 1; i < m; ++i) sig += a[pk9(k + 1 + i, k)] * a[pk9(k + 1 + i, k)];
    const double nx = sqrt(x0 * x0 + sig);
    double beta = 0.0, alpha = 0.0;
    if (nx != 0.0) {
      alpha = x0 >= 0.0 ? -nx : nx;
      beta = 1.0 / (nx * nx - x0 * alpha);
    }
    double v[8];
    v[0] = x0 - alpha;
#pragma unroll
    for (int i = 1; i < m; ++i) v[i] = a[pk9(k + 1 + i, k)];
    // p = beta S v, K = beta/2 p.v, w = p - K v; S -= v w^T + w v^T
    double p[8];
#pragma unroll
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < m; ++j) acc += a[pk9(k + 1 + i, k + 1 + j)] * v[j];
      p[i] = beta * acc;
    }
    double pv = 0.0;
#pragma unroll
    for (int i = 0; i < m; ++i) pv += p[i] * v[i];
    const double K = 0.5 * beta * pv;
#pragma unroll
    for (int i = 0; i < m; ++i) p[i] -= K * v[i];
#pragma unroll
    for (int i = 0; i < m; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) a[pk9(k + 1 + i, k + 1 + j)] -= v[i] * p[j] + p[i] * v[j];
    e[k] = nx != 0.0 ? alpha : 0.0;
#pragma unroll
    for (int i = 0; i < m; ++i) G(refl_off(k) + i) = v[i];
    G(35 + k) = beta;
  }
  e[7] = a[pk9(8, 7)];
  double d[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) d[i] = a[pk9(i, i)];
#pragma unroll
  for (int i = 0; i < 9; ++i) S(kSlotD + i) = d[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) S(kSlotE + i) = e[i];
  // ---- 2. eigenvalues (implicit QL on copies).  One loop iteration = one QL
  // sweep of this lane's current unreduced block [l, m]; lanes deflate
  // independently (the warp runs max over its lanes of the total sweep count,
  // not the per-level maxima), and the static 8-step sweep stops as soon as
  // every lane of the warp is below its block.
  double lam[9], ee[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    lam[i] = d[i];
    ee[i] = i < 8 ? e[i] : 0.0;
  }
  {
    int l = 0;
    for (int sweep = 0;; ++sweep) {
      // deflate: l = first index whose coupling to the next is not negligible
      int m = 8;
      bool found_l = false;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double dd = fabs(lam[i]) + fabs(lam[i + 1]);
        const bool neg = fabs(ee[i]) + dd == dd;
        if (!found_l && i >= l && !neg) {
          l = i;
          found_l = true;
        }
        if (found_l && i > l - 1 && neg && m == 8 && i >= l) m = i;
      }
      if (!found_l) l = 8;
      const bool active = l < 8;
      if (!__any_sync(__activemask(), active)) break;
      if (sweep == 120) return false;
      if (active) {
        // d_l, e_l, d_{l+1}, d_m by arithmetic blends (a select chain gets
        // turned back into an indexed load, which moves lam to local memory)
        double dl = 0.0, dl1 = 0.0, el = 0.0, dm = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          const double w0 = i == l ? 1.0 : 0.0, w1 = i == l + 1 ? 1.0 : 0.0, wm = i == m ? 1.0 : 0.0;
          dl = fma(w0, lam[i], dl);
          el = fma(w0, ee[i], el);
          dl1 = fma(w1, lam[i], dl1);
          dm = fma(wm, lam[i], dm);
        }
        // Wilkinson-type shift: with h = d_{l+1} - d_l,
        //   e_l / (g + sgn(g) sqrt(g^2 + 1)), g = h / (2 e_l)
        //   = 2 e_l^2 / (h + sgn(h) sqrt(h^2 + 4 e_l^2))   (one sqrt, one division)
        const double h = dl1 - dl;
        const double rh = sqrt(h * h + 4.0 * el * el);
        double g = dm - dl + 2.0 * el * el / (h + copysign(rh, h));
        double r;
        double s = 1.0, c = 1.0, pp = 0.0;
        // the lowest block start among the lanes sweeping together: steps below
        // it are idle for every lane (one reduction per sweep, uniform break)
        const int lmin = __reduce_min_sync(__activemask(), l);
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          if (i < m && i >= l) {
            const double f = s * ee[i], b = c * ee[i];
            // r2 == 0 (f = g = 0) only in degenerate arithmetic; the floor
            // keeps it finite and the verification catches any damage
            const double r2 = fmax(f * f + g * g, 1e-300);
            const double ir = rsqrt(r2);
            ee[i + 1] = r2 * ir;
            s = f * ir;
            c = g * ir;
            g = lam[i + 1] - pp;
            r = (lam[i] - g) * s + 2.0 * c * b;
            pp = s * r;
            lam[i + 1] = g + pp;
            g = c * r - b;
          }
          if (i - 1 < lmin) break;
        }
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          if (i == l) {
            lam[i] -= pp;
            ee[i] = g;
          }
          if (i == m) ee[i] = 0.0;
        }
      }
    }
  }
  // sort ascending (odd-even transposition)
#pragma unroll
  for (int rnd = 0; rnd < 9; ++rnd)
#pragma unroll
    for (int i = rnd & 1; i + 1 < 9; i += 2) {
      const double lo = fmin(lam[i], lam[i + 1]), hi = fmax(lam[i], lam[i + 1]);
      lam[i] = lo;
      lam[i + 1] = hi;
    }
  // eigenvalues in (-tau0, 0] count as zero: leaving them unclamped changes P
  // by at most tau0 = 1e-13 |M|_F (and their sign is not resolved anyway)
  const double tau0 = 1e-13 * nrm;
  int kneg = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i) kneg += lam[i] < -tau0;
  // the used eigenvalues (the clamped side), lam dies here
  const bool negside = kneg <= 4;
  const int nuse = negside ? kneg : 9 - kneg;
  double lu[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int sel = negside ? u : kneg + u;
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if (i == sel) lu[u] = lam[i];
  }
  // ---- 3. Sturm count of T at -tau0 must agree
  double tn = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i)
    tn = fmax(tn, fabs(S(kSlotD + i)) + (i < 8 ? fabs(S(kSlotE + i)) : 0.0) + (i > 0 ? fabs(S(kSlotE + i - 1)) : 0.0));
  const double pivmin = 1e-300 + 2.2e-19 * tn;
  {
    int cnt = 0;
    double q = S(kSlotD) + tau0;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
#pragma unroll
    for (int i = 1; i < 9; ++i) {
      const double ei = S(kSlotE + i - 1);
      q = S(kSlotD + i) + tau0 - ei * ei / q;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += q < 0.0;
    }
    if (cnt != kneg) return false;
  }
  if (kneg == 0) {
    reload_m(msrc, P);
    return true;
  }
  // ---- 4. eigenvectors of T for the used eigenvalues (T basis, smem slots
  // [42, 78)); members of a cluster (|lam_u - lam_w| <= 1e-3 |T|) are
  // Gram-Schmidt orthogonalized against the earlier ones after every solve
#pragma unroll 1
  for (int u = 0; u < nuse; ++u) {
    double lj = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q == u) lj = lu[q];
    // LDL^T of T - lj I without pivoting (tiny pivots replaced by pivmin;
    // the verification below catches any loss of accuracy)
    double rq[9], ll[8];
    {
      double q = S(kSlotD) - lj;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (fabs(q) < pivmin) q = pivmin;
        rq[i] = 1.0 / q;
        const double ei = S(kSlotE + i);
        ll[i] = ei * rq[i];
        q = S(kSlotD + i + 1) - lj - ll[i] * ei;
      }
      if (fabs(q) < pivmin) q = pivmin;
      rq[8] = 1.0 / q;
    }
    double y[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) y[i] = 1.0 / 3.0 + ((i + 2 * u) % 9 == 0 ? 0.25 : 0.0);
#pragma unroll
    for (int itr = 0; itr < 2; ++itr) {
#pragma unroll
      for (int i = 1; i < 9; ++i) y[i] -= ll[i - 1] * y[i - 1];
#pragma unroll
      for (int i = 0; i < 9; ++i) y[i] *= rq[i];
#pragma unroll
      for (int i = 7; i >= 0; --i) y[i] -= ll[i] * y[i + 1];
      for (int w = 0; w < u; ++w) {
        double lw = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q == w) lw = lu[q];
        if (fabs(lw - lj) > 1e-3 * tn) continue;
        double dot = 0.0;
#pragma unroll
        for (int q = 0; q < 9; ++q) dot += S(9 * w + q) * y[q];
#pragma unroll
        for (int q = 0; q < 9; ++q) y[q] -= dot * S(9 * w + q);
      }
      double yy = 0.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) yy += y[q] * y[q];
      if (!(yy > 0.0)) return false;
      const double iy = rsqrt(yy);
#pragma unroll
      for (int q = 0; q < 9; ++q) y[q] *= iy;
    }
    // ---- 5. residual |T y - lj y| and orthogonality to the earlier vectors
    double rr = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      double acc = (S(kSlotD + q) - lj) * y[q];
      if (q > 0) acc += S(kSlotE + q - 1) * y[q - 1];
      if (q < 8) acc += S(kSlotE + q) * y[q + 1];
      rr += acc * acc;
    }
    if (!(rr <= 1e-24 * n2)) return false;
    for (int w = 0; w < u; ++w) {
      double dot = 0.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) dot += S(9 * w + q) * y[q];
      if (!(fabs(dot) <= 1e-12)) return false;
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) S(9 * u + q) = y[q];
  }
  // ---- back-transform the used vectors in place: x = Q y = H_0 ... H_6 y
#pragma unroll 1
  for (int w = 0; w < nuse; ++w) {
    double x[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) x[q] = S(9 * w + q);
#pragma unroll
    for (int k = 6; k >= 0; --k) {
      double sd = 0.0;
#pragma unroll
      for (int q = 0; q < 8 - k; ++q) sd += G(refl_off(k) + q) * x[k + 1 + q];
      sd *= G(35 + k);
#pragma unroll
      for (int q = 0; q < 8 - k; ++q) x[k + 1 + q] -= sd * G(refl_off(k) + q);
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) S(9 * w + q) = x[q];
  }
  // ---- P = M - sum lam x x^T (negative side) or sum max(lam, 0) x x^T,
  // row by row with the vectors read from shared memory (P is the only
  // 45-register array live here)
  double fw[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) fw[w] = w < nuse ? (negside ? -lu[w] : fmax(lu[w], 0.0)) : 0.0;
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    double xa[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) xa[w] = w < nuse ? fw[w] * S(9 * w + a) : 0.0;
#pragma unroll
    for (int b = a; b < 9; ++b) {
      double acc = negside ? ld_reload(msrc + pk9(a, b)) : 0.0;
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (w < nuse) acc += xa[w] * S(9 * w + b);
      P[pk9(a, b)] = acc;
    }
  }
  return true;
}

// ---------------------------------------------------------------------------
// Edge-space (9x9, index 3*edge + coord) Hessian H_D -> vertex blocks.
//
// FullProject:    M = (R (x) I) H_D (R^T (x) I), P = Proj9(M), E = W
// ReducedProject: M = H_D, P = Proj9(M), E = S^T
// no projection:  P = H_D, E = S^T                   (assemble(false))
// Vertex block (a, b) = sum_{i,i'} E[a][i] E[b][i'] P_{ii'}; pair order
// (0,0),(0,1),(0,2),(0,3),(1,1),(1,2),(1,3),(2,2),(2,3),(3,3).

// In place: hd <- (R (x) I) hd (R^T (x) I)   (blocks, HD_{ii'} = HD_{i'i}^T)
__device__ __forceinline__ void edge_to_projection_space(double* hd) {
  // one flat loop over the packed entries (the nested block form was left
  // partly rolled by the compiler, which put hd in local memory)
  double m[45];
#pragma unroll
  for (int p = 0; p < 45; ++p) {
    int r = 0, c = 0;  // packed (row, col) of p, row <= col
#pragma unroll
    for (int rr = 0; rr < 9; ++rr)
#pragma unroll
      for (int cc = rr; cc < 9; ++cc)
        if (pk9(rr, cc) == p) {
          r = rr;
          c = cc;
        }
    const int a = r / 3, k = r % 3, b = c / 3, kk = c % 3;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int ip = 0; ip < 3; ++ip)
        if (i >= a && ip >= b) acc += kR(a, i) * kR(b, ip) * hd[pk9(3 * i + k, 3 * ip + kk)];
    m[p] = acc;
  }
#pragma unroll
  for (int i = 0; i < 45; ++i) hd[i] = m[i];
}

template <bool FULL, class Writer>
__device__ __forceinline__ void expand_vb(const double* hd, const Writer& wr) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (b < a) continue;
      const int pair = a * 4 - (a * (a - 1)) / 2 + (b - a);
      double blk[9];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          if (a == b && kk < k) continue;
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int ip = 0; ip < 3; ++ip) {
              const double ea = FULL ? kW(a, i) : kST(a, i);
              const double eb = FULL ? kW(b, ip) : kST(b, ip);
              if (ea == 0.0 || eb == 0.0) continue;
              acc += ea * eb * hd[pk9(3 * i + k, 3 * ip + kk)];
            }
          blk[k * 3 + kk] = acc;
          if (a == b && kk != k) blk[kk * 3 + k] = acc;
        }
      wr.block(pair, blk);
    }
}

// the projection-space map is a compile-time choice inside (zero terms fold)
template <class Writer>
__device__ __forceinline__ void expand_vertex_blocks(const double* hd, bool full, const Writer& wr) {
  if (full)
    expand_vb<true>(hd, wr);
  else
    expand_vb<false>(hd, wr);
}

// Positive-definiteness test by Cholesky on a copy: true iff every pivot is
// positive, in which case Proj9(M) = M (the reference's clamp is a no-op).
__device__ __forceinline__ bool cholesky_pd9(const double* m) {
  double l[45];
#pragma unroll
  for (int i = 0; i < 45; ++i) l[i] = m[i];
  bool pd = true;
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    double d = l[pk9(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= l[pk9(j, k)] * l[pk9(j, k)];
    pd = pd && (d > 0.0);
    const double ljj = sqrt(d > 0.0 ? d : 1.0);
    l[pk9(j, j)] = ljj;
    const double inv = 1.0 / ljj;
#pragma unroll
    for (int i = j + 1; i < 9; ++i) {
      double v = l[pk9(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= l[pk9(i, k)] * l[pk9(j, k)];
      l[pk9(i, j)] = v * inv;
    }
  }
  return pd;
}

// In place (m is destroyed): true iff every Cholesky pivot is positive.
__device__ __forceinline__ bool cholesky_pd9_inplace(double* l) {
  // constant loop bounds with guards: fully unrolled, l stays in registers
  bool pd = true;
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    double d = l[pk9(j, j)];
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (k < j) d -= l[pk9(j, k)] * l[pk9(j, k)];
    pd = pd && (d > 0.0);
    const double ljj = sqrt(d > 0.0 ? d : 1.0);
    l[pk9(j, j)] = ljj;
    const double inv = 1.0 / ljj;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if (i <= j) continue;
      double v = l[pk9(i, j)];
#pragma unroll
      for (int k = 0; k < 9; ++k)
        if (k < j) v -= l[pk9(i, k)] * l[pk9(j, k)];
      l[pk9(i, j)] = v * inv;
    }
  }
  return pd;
}

// ---------------------------------------------------------------------------
// Stable Neo-Hookean (energies.cpp:49-118):
//   F(r,c) = x_{c+1}[r] - x0[r];  F_I = F^T Binv;  I_C = tr(F_I^T F_I);  J = det F_I
//   psi = V w [mu/2 (I_C - 3) - mu/2 log(I_C + 1) + lambda/2 (J - alpha)^2]
struct SnhParams {
  double mu, lambda, alpha, weight;
};

__device__ __forceinline__ void snh_fi(const double x[12], const double binv[9], double fi[9]) {
  double d[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) d[3 * i + k] = x[3 * (i + 1) + k] - x[k];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      fi[3 * i + j] = d[3 * i + 0] * binv[0 * 3 + j] + d[3 * i + 1] * binv[1 * 3 + j] +
                      d[3 * i + 2] * binv[2 * 3 + j];
}

YS_HD double det3(const double f[9]) {
  return f[0] * (f[4] * f[8] - f[5] * f[7]) - f[1] * (f[3] * f[8] - f[5] * f[6]) +
         f[2] * (f[3] * f[7] - f[4] * f[6]);
}

YS_HD void cof3(const double f[9], double c[9]) {
  c[0] = f[4] * f[8] - f[5] * f[7];
  c[1] = f[5] * f[6] - f[3] * f[8];
  c[2] = f[3] * f[7] - f[4] * f[6];
  c[3] = f[2] * f[7] - f[1] * f[8];
  c[4] = f[0] * f[8] - f[2] * f[6];
  c[5] = f[1] * f[6] - f[0] * f[7];
  c[6] = f[1] * f[5] - f[2] * f[4];
  c[7] = f[2] * f[3] - f[0] * f[5];
  c[8] = f[0] * f[4] - f[1] * f[3];
}

// Energy only (line search). Returns false on log of a non-positive value.
__device__ __forceinline__ bool snh_energy(const double x[12], const double binv[9], double vol,
                                           const SnhParams& P, double* e) {
  double fi[9];
  snh_fi(x, binv, fi);
  double ic = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) ic += fi[i] * fi[i];
  const double J = det3(fi);
  const double arg = ic + 1.0;
  if (!(arg > 0.0)) return false;
  const double js = J - P.alpha;
  *e = vol * P.weight * ((0.5 * P.mu) * (ic - 3.0) - (0.5 * P.mu) * log(arg) + (0.5 * P.lambda) * js * js);
  return true;
}

// Gradient (12, vertex-major) and vertex blocks of the (projected) Hessian.
// Gradient (12, vertex-major) and, if want_h, the edge-space Hessian H_D (packed 45).
__device__ __forceinline__ void snh_local(const double x[12], const double binv[9], double vol,
                                          const SnhParams& P, bool want_h, double g[12], double* hd) {
  double fi[9];
  snh_fi(x, binv, fi);
  double ic = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) ic += fi[i] * fi[i];
  const double J = det3(fi);
  double cf[9];
  cof3(fi, cf);
  const double vw = vol * P.weight;
  const double ip1 = 1.0 / (ic + 1.0);
  const double c1 = vw * P.mu * (1.0 - ip1);
  const double c4 = vw * P.lambda * (J - P.alpha);
  // dpsi/dF_I and gradient wrt the edges: G_D = P_I Binv^T
  double pi[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) pi[i] = c1 * fi[i] + c4 * cf[i];
  double gd[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      gd[3 * i + k] = pi[3 * i + 0] * binv[3 * k + 0] + pi[3 * i + 1] * binv[3 * k + 1] +
                      pi[3 * i + 2] * binv[3 * k + 2];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g[k] = -(gd[k] + gd[3 + k] + gd[6 + k]);
    g[3 + k] = gd[k];
    g[6 + k] = gd[3 + k];
    g[9 + k] = gd[6 + k];
  }
  if (!want_h) return;

  // A = d2psi/dF_I^2 (packed 9x9): c1 I + c2 f f^T + c3 c c^T + c4 Hdet
  const double c2 = vw * 2.0 * P.mu * ip1 * ip1;
  const double c3 = vw * P.lambda;
  // H_D blocks: HD_{ii'} = Binv A_{ii'} Binv^T, computed blockwise into packed hd
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int ip = 0; ip < 3; ++ip) {
      if (ip < i) continue;
      double a[9];  // A_{ii'}[j][j']
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int jp = 0; jp < 3; ++jp) {
          const int al = 3 * i + j, be = 3 * ip + jp;
          double v = c2 * fi[al] * fi[be] + c3 * cf[al] * cf[be];
          if (al == be) v += c1;
          if (i != ip && j != jp) {
            const int b = 3 - i - ip, d = 3 - j - jp;
            const double s1 = ((ip - i + 3) % 3 == 1) ? 1.0 : -1.0;
            const double s2 = ((jp - j + 3) % 3 == 1) ? 1.0 : -1.0;
            v += c4 * s1 * s2 * fi[3 * b + d];
          }
          a[3 * j + jp] = v;
        }
      // T = A Binv^T ; HD = Binv T
      double t[9];
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int kp = 0; kp < 3; ++kp)
          t[3 * j + kp] = a[3 * j + 0] * binv[3 * kp + 0] + a[3 * j + 1] * binv[3 * kp + 1] +
                          a[3 * j + 2] * binv[3 * kp + 2];
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int kp = 0; kp < 3; ++kp) {
          if (i == ip && kp < k) continue;
          hd[pk9(3 * i + k, 3 * ip + kp)] =
              binv[3 * k + 0] * t[0 * 3 + kp] + binv[3 * k + 1] * t[1 * 3 + kp] + binv[3 * k + 2] * t[2 * 3 + kp];
        }
    }
}

// ---------------------------------------------------------------------------
// Bending (energies.cpp:129-155): e = c ||n1^ - n2^||, c = k w l0,
//   n1 = (x1-x0) x (x2-x0) = e0 x e1,  n2 = (x3-x0) x (x1-x0) = e2 x e0.
// Status: 0 ok, 1 division by zero (zero normal or flat hinge for derivatives).
YS_HD void cross3(const double a[3], const double b[3], double c[3]) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

__device__ __forceinline__ int bending_energy(const double x[12], double c, double* e) {
  double e0[3], e1[3], e2[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e0[k] = x[3 + k] - x[k];
    e1[k] = x[6 + k] - x[k];
    e2[k] = x[9 + k] - x[k];
  }
  double n1[3], n2[3];
  cross3(e0, e1, n1);
  cross3(e2, e0, n2);
  const double N1 = sqrt(n1[0] * n1[0] + n1[1] * n1[1] + n1[2] * n1[2]);
  const double N2 = sqrt(n2[0] * n2[0] + n2[1] * n2[1] + n2[2] * n2[2]);
  if (N1 == 0.0 || N2 == 0.0) return 1;
  double u[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) u[k] = n1[k] / N1 - n2[k] / N2;
  *e = c * sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  return 0;
}

__device__ __forceinline__ void skew3(const double a[3], double m[9]) {
  // [a]x
  m[0] = 0.0;   m[1] = -a[2]; m[2] = a[1];
  m[3] = a[2];  m[4] = 0.0;   m[5] = -a[0];
  m[6] = -a[1]; m[7] = a[0];  m[8] = 0.0;
}

__device__ __forceinline__ int bending_local(const double x[12], double c, bool want_h, double g[12], double* hd) {
  double e0[3], e1[3], e2[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e0[k] = x[3 + k] - x[k];
    e1[k] = x[6 + k] - x[k];
    e2[k] = x[9 + k] - x[k];
  }
  double n1[3], n2[3];
  cross3(e0, e1, n1);
  cross3(e2, e0, n2);
  const double N1 = sqrt(n1[0] * n1[0] + n1[1] * n1[1] + n1[2] * n1[2]);
  const double N2 = sqrt(n2[0] * n2[0] + n2[1] * n2[1] + n2[2] * n2[2]);
  if (N1 == 0.0 || N2 == 0.0) return 1;
  double h1[3], h2[3], u[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    h1[k] = n1[k] / N1;
    h2[k] = n2[k] / N2;
    u[k] = h1[k] - h2[k];
  }
  const double U = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  if (U == 0.0) return 1;
  double uh[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) uh[k] = u[k] / U;
  const double d1 = h1[0] * uh[0] + h1[1] * uh[1] + h1[2] * uh[2];
  const double d2 = h2[0] * uh[0] + h2[1] * uh[1] + h2[2] * uh[2];
  double y1[3], y2[3];  // J_n^T u^ (n-space gradients)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    y1[k] = (uh[k] - h1[k] * d1) / N1;
    y2[k] = (uh[k] - h2[k] * d2) / N2;
  }
  // gradient wrt edges: g_e0 = c (e1 x y1 - y2 x e2), g_e1 = c (y1 x e0), g_e2 = -c (e0 x y2)
  double ge0a[3], ge0b[3], ge1[3], ge2[3];
  cross3(e1, y1, ge0a);
  cross3(y2, e2, ge0b);
  cross3(y1, e0, ge1);
  cross3(e0, y2, ge2);
  double gd[9];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gd[k] = c * (ge0a[k] - ge0b[k]);
    gd[3 + k] = c * ge1[k];
    gd[6 + k] = -c * ge2[k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g[k] = -(gd[k] + gd[3 + k] + gd[6 + k]);
    g[3 + k] = gd[k];
    g[6 + k] = gd[3 + k];
    g[9 + k] = gd[6 + k];
  }
  if (!want_h) return 0;

  // Jacobians of n1, n2 wrt (e0, e1, e2) as 3x9 (row m, col 3*edge + k)
  double sk0[9], sk1[9], sk2[9];
  skew3(e0, sk0);
  skew3(e1, sk1);
  skew3(e2, sk2);
  double jn1[27], jn2[27];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      jn1[m * 9 + k] = -sk1[m * 3 + k];
      jn1[m * 9 + 3 + k] = sk0[m * 3 + k];
      jn1[m * 9 + 6 + k] = 0.0;
      jn2[m * 9 + k] = sk2[m * 3 + k];
      jn2[m * 9 + 3 + k] = 0.0;
      jn2[m * 9 + 6 + k] = -sk0[m * 3 + k];
    }
  // Ju = Jh1 Jn1 - Jh2 Jn2, Jh = (I - h h^T)/N
  double ju[27];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int col = 0; col < 9; ++col) {
      double a1 = jn1[m * 9 + col] - h1[m] * (h1[0] * jn1[col] + h1[1] * jn1[9 + col] + h1[2] * jn1[18 + col]);
      double a2 = jn2[m * 9 + col] - h2[m] * (h2[0] * jn2[col] + h2[1] * jn2[9 + col] + h2[2] * jn2[18 + col]);
      ju[m * 9 + col] = a1 / N1 - a2 / N2;
    }
  // Z = sum_m u^_m d2 h_m/dn2 = (3 (h.u^) h h^T - u^ h^T - h u^T - (h.u^) I) / N^2
  double z1[9], z2[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      z1[3 * a + b] = (3.0 * d1 * h1[a] * h1[b] - uh[a] * h1[b] - h1[a] * uh[b] - (a == b ? d1 : 0.0)) / (N1 * N1);
      z2[3 * a + b] = (3.0 * d2 * h2[a] * h2[b] - uh[a] * h2[b] - h2[a] * uh[b] - (a == b ? d2 : 0.0)) / (N2 * N2);
    }
  // q = (I - u^ u^^T)/U
#pragma unroll
  for (int p = 0; p < 9; ++p)
#pragma unroll
    for (int q = p; q < 9; ++q) {
      double acc = 0.0;
      // Ju^T Q Ju
      double jp[3] = {ju[p], ju[9 + p], ju[18 + p]};
      double jq[3] = {ju[q], ju[9 + q], ju[18 + q]};
      const double dpq = jp[0] * jq[0] + jp[1] * jq[1] + jp[2] * jq[2];
      const double up = uh[0] * jp[0] + uh[1] * jp[1] + uh[2] * jp[2];
      const double uq = uh[0] * jq[0] + uh[1] * jq[1] + uh[2] * jq[2];
      acc += (dpq - up * uq) / U;
      // Jn1^T Z1 Jn1 - Jn2^T Z2 Jn2
      double a1p[3] = {jn1[p], jn1[9 + p], jn1[18 + p]};
      double a1q[3] = {jn1[q], jn1[9 + q], jn1[18 + q]};
      double a2p[3] = {jn2[p], jn2[9 + p], jn2[18 + p]};
      double a2q[3] = {jn2[q], jn2[9 + q], jn2[18 + q]};
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) acc += a1p[a] * z1[3 * a + b] * a1q[b] - a2p[a] * z2[3 * a + b] * a2q[b];
      hd[pk9(p, q)] = acc;
    }
  // bilinear parts: B1 block (e0,e1) = -[y1]x ; B2 block (e0,e2) = [y2]x (subtracted)
  double sy1[9], sy2[9];
  skew3(y1, sy1);
  skew3(y2, sy2);
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int kk = 0; kk < 3; ++kk) {
      hd[pk9(k, 3 + kk)] += -sy1[3 * k + kk];
      hd[pk9(k, 6 + kk)] -= sy2[3 * k + kk];
    }
#pragma unroll
  for (int i = 0; i < 45; ++i) hd[i] *= c;
  return 0;
}

// ---------------------------------------------------------------------------
// Affine orthogonality (energies.cpp:120-127): 0.5 k w ||A^T A - I||_F^2 on the
// row-major 3x3 affine matrix.
__device__ __forceinline__ double ortho_energy(const double A[9], double kw) {
  double e = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double gab = A[a] * A[b] + A[3 + a] * A[3 + b] + A[6 + a] * A[6 + b] - (a == b ? 1.0 : 0.0);
      e += gab * gab;
    }
  return 0.5 * kw * e;
}

__device__ __forceinline__ void ortho_local(const double A[9], double kw, bool want_h, bool project,
                                            double g[9], double* h81) {
  double G[9], AAt[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      G[3 * a + b] = A[a] * A[b] + A[3 + a] * A[3 + b] + A[6 + a] * A[6 + b] - (a == b ? 1.0 : 0.0);
      AAt[3 * a + b] = A[3 * a] * A[3 * b] + A[3 * a + 1] * A[3 * b + 1] + A[3 * a + 2] * A[3 * b + 2];
    }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      g[3 * i + j] = 2.0 * kw * (A[3 * i] * G[j] + A[3 * i + 1] * G[3 + j] + A[3 * i + 2] * G[6 + j]);
  if (!want_h) return;
  double h[45];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          const int al = 3 * i + j, be = 3 * k + l;
          if (be < al) continue;
          double v = A[3 * i + l] * A[3 * k + j];
          if (i == k) v += G[3 * l + j];
          if (j == l) v += AAt[3 * i + k];
          h[pk9(al, be)] = 2.0 * kw * v;
        }
  if (project) psd_project9(h);
#pragma unroll
  for (int a = 0; a < 9; ++a)
#pragma unroll
    for (int b = 0; b < 9; ++b) h81[9 * a + b] = h[pk9(a, b)];
}

// ---------------------------------------------------------------------------
// Scalar-of-squared-distance terms  b(d), d = |delta|^2 (PP barrier / repulsive).
// Returns 0 ok, 1 log of non-positive, 2 division by zero.
struct PairParams {
  double dhat, kappa, weight;
  int32_t repulsive;
};

__device__ __forceinline__ int pair_b(double d, const PairParams& P, double* b, double* b1, double* b2) {
  if (P.repulsive) {
    if (d == 0.0) return 2;
    const double r = sqrt(d);
    *b = P.weight / r;
    *b1 = -0.5 * P.weight / (d * r);
    *b2 = 0.75 * P.weight / (d * d * r);
    return 0;
  }
  const double arg = d / P.dhat;
  if (!(arg > 0.0)) return 1;
  const double L = log(arg);
  const double len = d - P.dhat;
  const double wk = P.weight * P.kappa;
  *b = wk * len * len * L * L;
  *b1 = wk * (2.0 * len * L * L + 2.0 * len * len * L / d);
  *b2 = wk * (2.0 * L * L + 8.0 * len * L / d + 2.0 * len * len * (1.0 - L) / (d * d));
  return 0;
}

// P3 = Proj(a I + c delta delta^T) (or the unprojected matrix), packed 6.
__device__ __forceinline__ void proj_rank1_3(double a, double c, const double dl[3], double d, bool project,
                                             double p[9]) {
  double s = a, t = c;
  if (project) {
    const double lpar = a + c * d;
    const double ap = a > 0.0 ? a : 0.0;
    const double lp = lpar > 0.0 ? lpar : 0.0;
    s = ap;
    t = d > 0.0 ? (lp - ap) / d : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) p[3 * i + j] = (i == j ? s : 0.0) + t * dl[i] * dl[j];
}

}  // namespace ys
