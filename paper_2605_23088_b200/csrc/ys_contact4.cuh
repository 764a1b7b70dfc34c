// ys_contact4.cuh — point-triangle, edge-edge and point-edge barrier terms.
//
// NOT IN THE REFERENCE (relsim has point-point contact only,
// proj/README.md:110-111): these terms complete north_star part (1) and
// SURVEY §8 rows A10 / (f)3.  They follow the reference's pattern for the
// point-point term (energies.cpp:30-47) — a stencil primitive joined to a
// UNION of point domains, E = w kappa (d - dhat)^2 log(d / dhat)^2 with d the
// SQUARED distance, FullProject — with d the squared distance between the
// stencil's primitives (IPC's distance types, Li et al. 2020):
//   PT (p, t0, t1, t2): point-plane, point-edge or point-point by the region
//       of p's closest point on the triangle (Ericson, Real-Time Collision
//       Detection 5.1.5);
//   EE (a0, a1, b0, b1): line-line, point-edge or point-point by the clamped
//       closest-point parameters of the two segments (Ericson 5.1.9); nearly
//       parallel edges (|ea x eb|^2 <= 1e-20 |ea|^2 |eb|^2) take the s = 0 branch;
//   PE (p, e0, e1): point-line or point-point by the closest-point parameter.
// The distance type is decided on the current positions (IPC's piecewise
// formulation); d, its gradient and its Hessian come from second-order
// forward-mode jets of the type's formula over the stencil's 3 arity
// coordinates, exactly as the oracle does it (oracle/yo_oracle.c).  The
// classification is computed with explicitly rounded operations (no FMA
// contraction) so the GPU and the oracle pick the same type.
// Unions of free and fixed points only (kappa_u = 1): a fixed point's slot is
// a pad, exactly as in the point-point term.
#pragma once

#include "ys_device.cuh"

namespace ys {

enum ContactType : int {
  CT_PP = 0,  // point-point: a = stencil slot of the first point, b = second
  CT_PE = 1,  // point-edge: point a, edge (b, c)
  CT_PT = 2,  // point-plane: point a, triangle (b, c, e)
  CT_EE = 3   // line-line: edge (a, b), edge (c, e)
};
struct ContactSel {
  int type;
  int a, b, c, e;  // stencil slot indices (0..arity-1)
};

// ---- explicitly rounded 3-vector helpers (classification) -----------------
__host__ __device__ __forceinline__ double rn_dot(const double* x, const double* y) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(__dadd_rn(__dmul_rn(x[0], y[0]), __dmul_rn(x[1], y[1])), __dmul_rn(x[2], y[2]));
#else
  return x[0] * y[0] + x[1] * y[1] + x[2] * y[2];
#endif
}
__host__ __device__ __forceinline__ void rn_sub(const double* x, const double* y, double* o) {
#ifdef __CUDA_ARCH__
  o[0] = __dsub_rn(x[0], y[0]);
  o[1] = __dsub_rn(x[1], y[1]);
  o[2] = __dsub_rn(x[2], y[2]);
#else
  o[0] = x[0] - y[0];
  o[1] = x[1] - y[1];
  o[2] = x[2] - y[2];
#endif
}
__host__ __device__ __forceinline__ double rn_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ __forceinline__ double rn_msub(double a, double b, double c, double d) {  // a b - c d
#ifdef __CUDA_ARCH__
  return __dsub_rn(__dmul_rn(a, b), __dmul_rn(c, d));
#else
  return a * b - c * d;
#endif
}

// Point-triangle region (Ericson 5.1.5).  pts: p, t0, t1, t2 (slots 0..3).
__host__ __device__ inline ContactSel classify_pt(const double (*x)[3]) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  rn_sub(x[2], x[1], ab);
  rn_sub(x[3], x[1], ac);
  rn_sub(x[0], x[1], ap);
  const double d1 = rn_dot(ab, ap), d2 = rn_dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return {CT_PP, 0, 1, 0, 0};
  rn_sub(x[0], x[2], bp);
  const double d3 = rn_dot(ab, bp), d4 = rn_dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return {CT_PP, 0, 2, 0, 0};
  const double vc = rn_msub(d1, d4, d3, d2);
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return {CT_PE, 0, 1, 2, 0};
  rn_sub(x[0], x[3], cp);
  const double d5 = rn_dot(ab, cp), d6 = rn_dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return {CT_PP, 0, 3, 0, 0};
  const double vb = rn_msub(d5, d2, d1, d6);
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return {CT_PE, 0, 1, 3, 0};
  const double va = rn_msub(d3, d6, d5, d4);
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) return {CT_PE, 0, 2, 3, 0};
  return {CT_PT, 0, 1, 2, 3};
}

// Point-edge (slots p = 0, e0 = 1, e1 = 2).
__host__ __device__ inline ContactSel classify_pe(const double (*x)[3]) {
  double e[3], ap[3];
  rn_sub(x[2], x[1], e);
  rn_sub(x[0], x[1], ap);
  const double t = rn_dot(ap, e), ee = rn_dot(e, e);
  if (t <= 0.0) return {CT_PP, 0, 1, 0, 0};
  if (t >= ee) return {CT_PP, 0, 2, 0, 0};
  return {CT_PE, 0, 1, 2, 0};
}

// Segment-segment (Ericson 5.1.9), slots a0 = 0, a1 = 1, b0 = 2, b1 = 3.
__host__ __device__ inline ContactSel classify_ee(const double (*x)[3]) {
  double d1[3], d2[3], r[3];
  rn_sub(x[1], x[0], d1);
  rn_sub(x[3], x[2], d2);
  rn_sub(x[0], x[2], r);
  const double a = rn_dot(d1, d1), e = rn_dot(d2, d2), f = rn_dot(d2, r);
  const double c = rn_dot(d1, r), b = rn_dot(d1, d2);
  const double denom = rn_msub(a, e, b, b);
  // nearly parallel edges: the s = 0 branch (Ericson) instead of line-line
  double s;
  bool s_clamped;
  if (denom > 1e-20 * rn_mul(a, e)) {
    s = rn_msub(b, f, c, e) / denom;
    s_clamped = s <= 0.0 || s >= 1.0;
    s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
  } else {
    s = 0.0;
    s_clamped = true;
  }
  // t = (b s + f) / e
#ifdef __CUDA_ARCH__
  const double tn = __dadd_rn(__dmul_rn(b, s), f);
#else
  const double tn = b * s + f;
#endif
  bool t_clamped = false;
  if (tn <= 0.0) {  // t = 0, s = clamp(-c / a)
    t_clamped = true;
    const double sn = -c;
    s_clamped = sn <= 0.0 || sn >= a;
    s = sn <= 0.0 ? 0.0 : (sn >= a ? 1.0 : sn / a);
    const int ta = 2;  // b0
    if (s_clamped) return {CT_PP, s == 0.0 ? 0 : 1, ta, 0, 0};
    return {CT_PE, ta, 0, 1, 0};
  }
  if (tn >= e) {  // t = 1, s = clamp((b - c) / a)
    t_clamped = true;
    const double sn = b - c;
    s_clamped = sn <= 0.0 || sn >= a;
    s = sn <= 0.0 ? 0.0 : (sn >= a ? 1.0 : sn / a);
    const int tb = 3;  // b1
    if (s_clamped) return {CT_PP, s == 0.0 ? 0 : 1, tb, 0, 0};
    return {CT_PE, tb, 0, 1, 0};
  }
  (void)t_clamped;
  if (s_clamped) return {CT_PE, s == 0.0 ? 0 : 1, 2, 3, 0};  // endpoint of a against edge b
  return {CT_EE, 0, 1, 2, 3};
}

__host__ __device__ inline ContactSel classify_contact(int kind, const double (*x)[3]) {
  return kind == K_PT ? classify_pt(x) : kind == K_EE ? classify_ee(x) : classify_pe(x);
}

// ---- second-order forward-mode jets over N stencil coordinates ------------
template <int N>
struct Jet {
  static constexpr int M = N * (N + 1) / 2;
  double v;
  double g[N];
  double h[M];  // packed upper: (i, j), i <= j
};

template <int N>
__device__ __forceinline__ constexpr int jh(int i, int j) {
  return i <= j ? i * N - i * (i - 1) / 2 + (j - i) : j * N - j * (j - 1) / 2 + (i - j);
}

template <int N>
__device__ __forceinline__ void jz(Jet<N>& o, double v) {
  o.v = v;
  for (int i = 0; i < N; ++i) o.g[i] = 0.0;
  for (int i = 0; i < Jet<N>::M; ++i) o.h[i] = 0.0;
}

template <int N>
__device__ __forceinline__ void jsub(Jet<N>& o, const Jet<N>& a, const Jet<N>& b) {
  o.v = a.v - b.v;
  for (int i = 0; i < N; ++i) o.g[i] = a.g[i] - b.g[i];
  for (int i = 0; i < Jet<N>::M; ++i) o.h[i] = a.h[i] - b.h[i];
}

template <int N>
__device__ __forceinline__ void jadd(Jet<N>& o, const Jet<N>& a, const Jet<N>& b) {
  o.v = a.v + b.v;
  for (int i = 0; i < N; ++i) o.g[i] = a.g[i] + b.g[i];
  for (int i = 0; i < Jet<N>::M; ++i) o.h[i] = a.h[i] + b.h[i];
}

template <int N>
__device__ __forceinline__ void jmul(Jet<N>& o, const Jet<N>& a, const Jet<N>& b) {
  Jet<N> t;
  t.v = a.v * b.v;
  for (int i = 0; i < N; ++i) t.g[i] = a.g[i] * b.v + a.v * b.g[i];
  for (int i = 0; i < N; ++i)
    for (int j = i; j < N; ++j)
      t.h[jh<N>(i, j)] = a.h[jh<N>(i, j)] * b.v + a.v * b.h[jh<N>(i, j)] + a.g[i] * b.g[j] + b.g[i] * a.g[j];
  o = t;
}

// f(a) with derivatives f1, f2
template <int N>
__device__ __forceinline__ void junary(Jet<N>& o, const Jet<N>& a, double f, double f1, double f2) {
  Jet<N> t;
  t.v = f;
  for (int i = 0; i < N; ++i) t.g[i] = f1 * a.g[i];
  for (int i = 0; i < N; ++i)
    for (int j = i; j < N; ++j) t.h[jh<N>(i, j)] = f1 * a.h[jh<N>(i, j)] + f2 * a.g[i] * a.g[j];
  o = t;
}

template <int N>
__device__ __forceinline__ void jdiv(Jet<N>& o, const Jet<N>& a, const Jet<N>& b) {
  Jet<N> inv;
  const double r = 1.0 / b.v;
  junary(inv, b, r, -r * r, 2.0 * r * r * r);
  jmul(o, a, inv);
}

template <int N>
__device__ __forceinline__ void jdot3(Jet<N>& o, const Jet<N>* a, const Jet<N>* b) {
  Jet<N> q;
  jmul(o, a[0], b[0]);
  jmul(q, a[1], b[1]);
  jadd(o, o, q);
  jmul(q, a[2], b[2]);
  jadd(o, o, q);
}

template <int N>
__device__ __forceinline__ void jcross3(Jet<N>* o, const Jet<N>* a, const Jet<N>* b) {
  Jet<N> t1, t2, r[3];
  for (int k = 0; k < 3; ++k) {
    const int i1 = (k + 1) % 3, i2 = (k + 2) % 3;
    jmul(t1, a[i1], b[i2]);
    jmul(t2, a[i2], b[i1]);
    jsub(r[k], t1, t2);
  }
  o[0] = r[0];
  o[1] = r[1];
  o[2] = r[2];
}

// Squared distance of the selected type as a jet over the N = 3 arity stencil
// coordinates (slot l -> variables 3 l .. 3 l + 2).
template <int N>
__device__ inline void contact_dist2(const ContactSel& s, const double (*x)[3], Jet<N>& d) {
  auto pt = [&](int l, Jet<N>* p) {
    for (int k = 0; k < 3; ++k) {
      jz(p[k], x[l][k]);
      p[k].g[3 * l + k] = 1.0;
    }
  };
  Jet<N> A[3], B[3], Cc[3], D[3], u[3], v[3], w[3];
  if (s.type == CT_PP) {
    pt(s.a, A);
    pt(s.b, B);
    for (int k = 0; k < 3; ++k) jsub(u[k], B[k], A[k]);
    jdot3(d, u, u);
  } else if (s.type == CT_PE) {
    // |(e0 - p) x (e1 - p)|^2 / |e1 - e0|^2
    pt(s.a, A);
    pt(s.b, B);
    pt(s.c, Cc);
    for (int k = 0; k < 3; ++k) {
      jsub(u[k], B[k], A[k]);
      jsub(v[k], Cc[k], A[k]);
      jsub(w[k], Cc[k], B[k]);
    }
    Jet<N> cr[3], num, den;
    jcross3(cr, u, v);
    jdot3(num, cr, cr);
    jdot3(den, w, w);
    jdiv(d, num, den);
  } else if (s.type == CT_PT) {
    // ((p - t0) . n)^2 / |n|^2, n = (t1 - t0) x (t2 - t0)
    pt(s.a, A);
    pt(s.b, B);
    pt(s.c, Cc);
    pt(s.e, D);
    for (int k = 0; k < 3; ++k) {
      jsub(u[k], A[k], B[k]);
      jsub(v[k], Cc[k], B[k]);
      jsub(w[k], D[k], B[k]);
    }
    Jet<N> n[3], sp, num, den;
    jcross3(n, v, w);
    jdot3(sp, u, n);
    jmul(num, sp, sp);
    jdot3(den, n, n);
    jdiv(d, num, den);
  } else {
    // ((b0 - a0) . (ea x eb))^2 / |ea x eb|^2
    pt(s.a, A);
    pt(s.b, B);
    pt(s.c, Cc);
    pt(s.e, D);
    for (int k = 0; k < 3; ++k) {
      jsub(u[k], B[k], A[k]);
      jsub(v[k], D[k], Cc[k]);
      jsub(w[k], Cc[k], A[k]);
    }
    Jet<N> n[3], sp, num, den;
    jcross3(n, u, v);
    jdot3(sp, w, n);
    jmul(num, sp, sp);
    jdot3(den, n, n);
    jdiv(d, num, den);
  }
}

// Value-only squared distance (energy evaluation, line search, the candidate
// test): the same formulas as contact_dist2, explicitly rounded (no FMA
// contraction), so the candidate test agrees bit for bit with the oracle's.
__host__ __device__ inline void rn_cross(const double* a, const double* b, double* o) {
  o[0] = rn_msub(a[1], b[2], a[2], b[1]);
  o[1] = rn_msub(a[2], b[0], a[0], b[2]);
  o[2] = rn_msub(a[0], b[1], a[1], b[0]);
}

__host__ __device__ inline double contact_dist2_value(const ContactSel& s, const double (*x)[3]) {
  double u[3], v[3], w[3], n[3];
  if (s.type == CT_PP) {
    rn_sub(x[s.b], x[s.a], u);
    return rn_dot(u, u);
  }
  if (s.type == CT_PE) {
    rn_sub(x[s.b], x[s.a], u);
    rn_sub(x[s.c], x[s.a], v);
    rn_sub(x[s.c], x[s.b], w);
    rn_cross(u, v, n);
    return rn_dot(n, n) / rn_dot(w, w);
  }
  if (s.type == CT_PT) {
    rn_sub(x[s.a], x[s.b], u);
    rn_sub(x[s.c], x[s.b], v);
    rn_sub(x[s.e], x[s.b], w);
    rn_cross(v, w, n);
    const double sp = rn_dot(u, n);
    return rn_mul(sp, sp) / rn_dot(n, n);
  }
  rn_sub(x[s.b], x[s.a], u);
  rn_sub(x[s.e], x[s.c], v);
  rn_sub(x[s.c], x[s.a], w);
  rn_cross(u, v, n);
  const double sp = rn_dot(w, n);
  return rn_mul(sp, sp) / rn_dot(n, n);
}

// Dense symmetric m x m (m <= 12, row-major, full storage) <- V max(L, 0) V^T:
// cyclic Jacobi with jacobi_rot's rotation formula and stopping test.
__device__ inline void psd_project_dense(double* A, int m) {
  double V[144];
  for (int i = 0; i < m * m; ++i) V[i] = (i % (m + 1) == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int p = 0; p < m; ++p) {
      dia += A[p * m + p] * A[p * m + p];
      for (int q = p + 1; q < m; ++q) off += A[p * m + q] * A[p * m + q];
    }
    if (!(off > kJacobiTol2 * (dia + 2.0 * off))) break;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = A[p * m + q], app = A[p * m + p], aqq = A[q * m + q];
        const double g = 100.0 * fabs(apq);
        if ((fabs(app) + g == fabs(app)) && (fabs(aqq) + g == fabs(aqq))) {
          A[p * m + q] = A[q * m + p] = 0.0;
          continue;
        }
        const double h = aqq - app;
        const double sa = h < 0.0 ? -apq : apq;
        const double rd = rsqrt(h * h + 4.0 * apq * apq);
        const double c2 = 0.5 + 0.5 * (fabs(h) * rd);
        const double rc = rsqrt(c2);
        const double c = c2 * rc, sn = sa * rd * rc, t = sn * rc;
        const double tq = t * apq;
        A[p * m + p] = app - tq;
        A[q * m + q] = aqq + tq;
        A[p * m + q] = A[q * m + p] = 0.0;
        for (int k = 0; k < m; ++k) {
          if (k == p || k == q) continue;
          const double akp = A[k * m + p], akq = A[k * m + q];
          A[k * m + p] = A[p * m + k] = c * akp - sn * akq;
          A[k * m + q] = A[q * m + k] = sn * akp + c * akq;
        }
        for (int k = 0; k < m; ++k) {
          const double vkp = V[k * m + p], vkq = V[k * m + q];
          V[k * m + p] = c * vkp - sn * vkq;
          V[k * m + q] = sn * vkp + c * vkq;
        }
      }
  }
  double lam[12];
  for (int k = 0; k < m; ++k) lam[k] = A[k * m + k] < 0.0 ? 0.0 : A[k * m + k];
  for (int i = 0; i < m; ++i)
    for (int j = i; j < m; ++j) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc += V[i * m + k] * lam[k] * V[j * m + k];
      A[i * m + j] = A[j * m + i] = acc;
    }
}

}  // namespace ys
