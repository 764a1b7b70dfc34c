// ys_capi.cu — the extern "C" boundary (include/yasps_b200.h) and the host
// orchestration behind it: registration of targets / point domains / unions /
// pair primitives / energies (the scene side the reference's energy builders
// record, energies.cpp), Engine construction and refresh (engine.cpp:7-45),
// minimize_step (engine.cpp:75-101), gather/scatter (103-120), the device
// proximity filter (sim.cpp:456-484) and the free-standing BSR solver.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>

#include "ys_device.cuh"

namespace ys {

int64_t& device_bytes_counter() {
  static int64_t bytes = 0;
  return bytes;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

const char* kind_name(int k) {
  switch (k) {
    case K_SNH: return "stable_neo_hookean";
    case K_BENDING: return "bending";
    case K_INERTIA: return "inertia";
    case K_ORTHO: return "affine_orthogonality";
    case K_PP: return "point_point";
    case K_REPULSIVE: return "repulsive";
    case K_PT: return "point_triangle";
    case K_EE: return "edge_edge";
    case K_PE: return "point_edge";
  }
  return "?";
}

std::vector<int64_t> Union::offsets() const { return {}; }

EnergyDev energy_dev(Context& c, Energy& e);
void spmv_launch(Context& c, Structure& s0, Structure* s1, const double* x, double* y, bool accumulate,
                 PcgState* st, double* part, int grid);
int pcg_grid(Context& c);
void ctx_block_rows(Context& c, bool want_h);
double fp64_probe(Context& c);


namespace {

constexpr int kTB = 256;
inline unsigned grid_for(int64_t n, int tb = kTB) { return unsigned(std::max<int64_t>(1, ceil_div(n, tb))); }

__global__ void k_points(DomainDev d, const double* X, double* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  point_position(d, i, X, out + 3 * i);
}

// X = X0 - alpha * DX and block maxima of |alpha * DX| (sim.cpp:546, 562).
__global__ void k_step(int64_t s, const double* X0, const double* DX, double alpha, double* X, double* part) {
  __shared__ double sm[kTB];
  double m = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s; i += int64_t(gridDim.x) * blockDim.x) {
    const double ad = __dmul_rn(alpha, DX[i]);  // x0 - alpha * d, no FMA contraction
    X[i] = __dsub_rn(X0[i], ad);
    m = fmax(m, fabs(ad));
  }
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w /= 2) {
    if (threadIdx.x < w) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

__global__ void k_identity_minv(int64_t nb, int bs, double* minv, int32_t* flag) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  for (int k = 0; k < bs * bs; ++k) minv[b * bs * bs + k] = (k % (bs + 1) == 0) ? 1.0 : 0.0;
  flag[b] = 0;
}

DomainDev domain_dev(Context& c, const Domain& d) {
  DomainDev D{};
  D.kind = d.kind;
  D.n = d.n;
  D.startA = d.ta >= 0 ? int32_t(c.targets[d.ta].start) : 0;
  D.startB = d.tb >= 0 ? int32_t(c.targets[d.tb].start) : 0;
  D.v2b = d.v2b.p;
  D.rest = d.rest.p;
  D.fixed = d.rest.p;
  return D;
}

void require_not_finalized(Context& c, const char* what) {
  if (c.finalized) fail(YS_ERR_DECL, std::string(what) + ": the engine is already built (ys_finalize)");
}
void require_finalized(Context& c) {
  if (!c.finalized) fail(YS_ERR_VALIDATION, "engine not built: call ys_finalize first");
}

void check_target(Context& c, int32_t t, int rc, const char* what) {
  if (t < 0 || t >= int32_t(c.targets.size())) fail(YS_ERR_DECL, std::string(what) + ": unknown target");
  if (rc > 0 && c.targets[t].rc != rc)
    fail(YS_ERR_DECL, std::string(what) + ": target must have " + std::to_string(rc) + " values per instance");
}

int32_t add_energy(Context& c, Energy&& e) {
  require_not_finalized(c, "add energy");
  e.name = std::string(kind_name(e.kind));
  int k = 0;
  for (auto& o : c.energies)
    if (o.kind == e.kind) ++k;
  if (k) e.name += "_" + std::to_string(k);
  c.energies.push_back(std::move(e));
  return int32_t(c.energies.size() - 1);
}

}  // namespace

void ctx_upload_domains(Context& c) {
  for (Union& u : c.unions) {
    std::vector<DomainDev> ch;
    std::vector<int64_t> off;
    int64_t acc = 0;
    for (int32_t d : u.children) {
      ch.push_back(domain_dev(c, c.domains[d]));
      off.push_back(acc);
      acc += c.domains[d].n;
    }
    u.d_child.upload(ch, c.stream);
    u.d_offsets.upload(off, c.stream);
  }
}

void ctx_refresh_dynamic(Context& c, bool force) {
  if (!force && c.seen_epoch == c.epoch) return;
  ctx_build_group(c, 1);
  c.seen_epoch = c.epoch;
}

void ctx_finalize(Context& c) {
  require_not_finalized(c, "ys_finalize");
  if (c.targets.empty()) fail(YS_ERR_DECL, "no minimize targets registered");
  cudaStream_t s = c.stream;
  int64_t acc = 0, nb = 0, dv = 0;
  c.uniform3 = true;
  for (Target& t : c.targets) {
    t.start = acc;
    t.block0 = nb;
    acc += t.n * t.rc;
    nb += t.n;
    dv += t.n * t.rc * t.rc;
    if (t.rc != 3) c.uniform3 = false;
  }
  c.s = acc;
  c.NB = nb;
  c.diag_vals = dv;
  if (c.s >= (int64_t(1) << 28)) fail(YS_ERR_VALIDATION, "system too large: more than 2^28 degrees of freedom");
  std::vector<int32_t> bstart(nb), brc(nb), d2b(acc);
  std::vector<int64_t> bvoff(nb);
  int64_t b = 0, vo = 0;
  for (const Target& t : c.targets)
    for (int64_t i = 0; i < t.n; ++i, ++b) {
      bstart[b] = int32_t(t.start + i * t.rc);
      brc[b] = t.rc;
      bvoff[b] = vo;
      vo += int64_t(t.rc) * t.rc;
      for (int k = 0; k < t.rc; ++k) d2b[t.start + i * t.rc + k] = int32_t(b);
    }
  c.rc_classes.clear();
  c.rc_lists.clear();
  for (int32_t r : brc)
    if (std::find(c.rc_classes.begin(), c.rc_classes.end(), r) == c.rc_classes.end()) c.rc_classes.push_back(r);
  std::sort(c.rc_classes.begin(), c.rc_classes.end());
  for (int32_t r : c.rc_classes) {
    std::vector<int32_t> lst;
    for (int64_t q = 0; q < nb; ++q)
      if (brc[q] == r) lst.push_back(int32_t(q));
    c.rc_lists.emplace_back();
    c.rc_lists.back().upload(lst, s);
  }
  c.bstart.upload(bstart, s);
  c.brc.upload(brc, s);
  c.bvoff.upload(bvoff, s);
  c.dof2block.upload(d2b, s);
  std::vector<double> x(acc, 0.0);
  for (size_t t = 0; t < c.targets.size(); ++t)
    if (!c.h_target_init[t].empty())
      std::copy(c.h_target_init[t].begin(), c.h_target_init[t].end(), x.begin() + c.targets[t].start);
  c.X.upload(x, s);
  c.X0.upload(x, s);
  c.G.resize(acc);
  c.G.zero(s);
  c.DX.resize(acc);
  c.DX.zero(s);
  c.diag.resize(dv);
  c.diag.zero(s);
  c.minv.resize(dv);
  c.minv.zero(s);
  c.bflag.resize(nb);
  c.errflag.resize(1);
  c.errflag.zero(s);
  ctx_upload_domains(c);
  for (PairSet& p : c.pairsets) {
    std::vector<int32_t> q(p.h_pairs.begin(), p.h_pairs.end());
    p.pairs.upload(q, s);
  }
  c.finalized = true;
  ctx_build_group(c, 0);
  ctx_build_group(c, 1);
  c.seen_epoch = c.epoch;
  YS_CUDA(cudaStreamSynchronize(s));
}

void ctx_get_points(Context& c, int domain, double* out) {
  Domain& d = c.domains[domain];
  if (d.n == 0) return;
  DevBuf<double> buf;
  buf.resize(size_t(3 * d.n));
  k_points<<<grid_for(d.n), kTB, 0, c.stream>>>(domain_dev(c, d), c.X.p, buf.p);
  YS_LAUNCH_CHECK();
  buf.download(out, size_t(3 * d.n), c.stream);
  YS_CUDA(cudaStreamSynchronize(c.stream));
}

void ctx_domain_points(Context& c, int domain, double* out) {
  const Domain& d = c.domains[domain];
  if (d.n == 0) return;
  k_points<<<grid_for(d.n), kTB, 0, c.stream>>>(domain_dev(c, d), c.X.p, out);
  YS_LAUNCH_CHECK();
}

}  // namespace ys

// ===========================================================================
// extern "C"

using namespace ys;

struct ys_context : ys::Context {
  std::vector<std::unique_ptr<ys_context>> subs;  // free-standing BSR systems
  int32_t bsr_bs = 0;
};

namespace {

int set_error(ys_context* c, int cls, const std::string& msg) {
  if (c) {
    c->err = msg;
    c->err_cls = cls;
  }
  return cls;
}

template <class F>
int guarded(ys_context* c, F f) {
  if (!c) return YS_ERR_VALIDATION;
  try {
    if (c->device >= 0) cudaSetDevice(c->device);
    f();
    return YS_OK;
  } catch (const ys::Error& e) {
    return set_error(c, e.cls, e.what());
  } catch (const std::bad_alloc&) {
    return set_error(c, YS_ERR_CUDA, "out of memory");
  } catch (const std::exception& e) {
    return set_error(c, YS_ERR_INTERNAL, e.what());
  }
}

double elapsed(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void check_pairs_in_range(Context& c, PairSet& ps, int64_t n, const int64_t* pairs) {
  int64_t total = 0;
  for (int32_t d : c.unions[ps.uni].children) total += c.domains[d].n;
  for (int64_t k = 0; k < int64_t(ps.arity) * n; ++k)
    if (pairs[k] < 0 || pairs[k] >= total)
      fail(YS_ERR_VALIDATION, "connectivity 'pp2v': index " + std::to_string(pairs[k]) + " at position " +
                                  std::to_string(k) + " out of range [0, " + std::to_string(total) + ")");
}

}  // namespace

extern "C" {

const char* ys_version(void) {
  return "yasps_b200 0.1 (sm_100a, FP64, CUDA 12.9)";
}

int ys_create(ys_context** out, int32_t device) {
  if (!out) return YS_ERR_VALIDATION;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return YS_ERR_CUDA;
  if (device < 0 || device >= ndev) return YS_ERR_VALIDATION;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return YS_ERR_CUDA;
  if (prop.major != 10) return YS_ERR_CUDA;  // built for sm_100a only; no fallback
  auto* c = new ys_context();
  c->device = device;
  // the context stream at the highest priority: while the static evaluation
  // fills the device from the low-priority side stream, the dynamic rebuild's
  // short kernels are dispatched first as SMs free up
  int prio_lo = 0, prio_hi = 0;
  if (cudaSetDevice(device) != cudaSuccess || cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
    delete c;
    return YS_ERR_CUDA;
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  *out = c;
  return YS_OK;
}

void ys_destroy(ys_context* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  drop_pcg_graph(*c);
  try {
    ctx_dist_finalize(*c);
  } catch (...) {
  }
  for (auto& sub : c->subs) drop_pcg_graph(*sub);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (auto& sub : c->subs)
    if (sub->pinned) cudaFreeHost(sub->pinned);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream2) {
    cudaStreamSynchronize(c->stream2);
    cudaStreamDestroy(c->stream2);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
  }
  c->subs.clear();
  cudaStream_t s = c->stream;
  delete c;
  cudaStreamDestroy(s);
}

const char* ys_last_error(const ys_context* c) { return c ? c->err.c_str() : "null context"; }
int ys_last_error_class(const ys_context* c) { return c ? c->err_cls : YS_ERR_VALIDATION; }

int ys_add_target(ys_context* c, int64_t instances, int32_t rc, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "ys_add_target");
    if (instances < 0) fail(YS_ERR_DECL, "negative instance count");
    if (!(rc == 1 || rc == 2 || rc == 3 || rc == 4 || rc == 6 || rc == 9 || rc == 12))
      fail(YS_ERR_DECL, "minimize target block size " + std::to_string(rc) + " is not supported");
    Target t;
    t.n = instances;
    t.rc = rc;
    c->targets.push_back(t);
    c->h_target_init.emplace_back();
    if (id) *id = int32_t(c->targets.size() - 1);
  });
}

int ys_set_target_values(ys_context* c, int32_t target, const double* v) {
  return guarded(c, [&] {
    check_target(*c, target, 0, "ys_set_target_values");
    const Target& t = c->targets[target];
    const int64_t n = t.n * t.rc;
    if (!c->finalized) {
      c->h_target_init[target].assign(v, v + n);
    } else {
      YS_CUDA(cudaMemcpyAsync(c->X.p + t.start, v, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      YS_CUDA(cudaStreamSynchronize(c->stream));
    }
  });
}

int ys_get_target_values(ys_context* c, int32_t target, double* v) {
  return guarded(c, [&] {
    check_target(*c, target, 0, "ys_get_target_values");
    const Target& t = c->targets[target];
    const int64_t n = t.n * t.rc;
    if (!c->finalized) {
      if (c->h_target_init[target].empty()) std::fill(v, v + n, 0.0);
      else std::copy(c->h_target_init[target].begin(), c->h_target_init[target].end(), v);
    } else {
      YS_CUDA(cudaMemcpyAsync(v, c->X.p + t.start, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      YS_CUDA(cudaStreamSynchronize(c->stream));
    }
  });
}

int ys_total_dofs(ys_context* c, int64_t* s) {
  return guarded(c, [&] {
    int64_t acc = 0;
    for (auto& t : c->targets) acc += t.n * t.rc;
    *s = acc;
  });
}

int ys_add_points(ys_context* c, int32_t kind, int64_t n, int32_t ta, int32_t tb, const int64_t* v2b,
                  const double* rest, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "ys_add_points");
    Domain d;
    d.kind = kind;
    d.n = n;
    if (kind == YS_POINTS_FREE) {
      check_target(*c, ta, 3, "free points");
      if (c->targets[ta].n != n) fail(YS_ERR_DECL, "free points: count differs from the position target");
      d.ta = ta;
    } else if (kind == YS_POINTS_AFFINE) {
      check_target(*c, ta, 9, "affine points (affine matrix)");
      check_target(*c, tb, 3, "affine points (translation)");
      if (c->targets[ta].n != c->targets[tb].n) fail(YS_ERR_DECL, "affine points: body counts differ");
      d.ta = ta;
      d.tb = tb;
      d.h_v2b.assign(v2b, v2b + n);
      for (int64_t i = 0; i < n; ++i)
        if (v2b[i] < 0 || v2b[i] >= c->targets[ta].n)
          fail(YS_ERR_VALIDATION, "connectivity 'v2b': index " + std::to_string(v2b[i]) + " at position " +
                                      std::to_string(i) + " out of range [0, " + std::to_string(c->targets[ta].n) +
                                      ")");
      d.h_rest.assign(rest, rest + 3 * n);
      std::vector<int32_t> vb(v2b, v2b + n);
      d.v2b.upload(vb, c->stream);
      d.rest.upload(d.h_rest, c->stream);
    } else if (kind == YS_POINTS_FIXED) {
      d.h_rest.assign(rest, rest + 3 * n);
      d.rest.upload(d.h_rest, c->stream);
    } else {
      fail(YS_ERR_DECL, "unknown point-domain kind");
    }
    YS_CUDA(cudaStreamSynchronize(c->stream));
    c->domains.push_back(std::move(d));
    *id = int32_t(c->domains.size() - 1);
  });
}

int ys_get_points(ys_context* c, int32_t domain, double* out) {
  return guarded(c, [&] {
    require_finalized(*c);
    if (domain < 0 || domain >= int32_t(c->domains.size())) fail(YS_ERR_DECL, "unknown point domain");
    ctx_get_points(*c, domain, out);
  });
}

int ys_add_point_union(ys_context* c, int32_t n, const int32_t* doms, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "ys_add_point_union");
    if (n < 1) fail(YS_ERR_DECL, "primitive union needs at least one child");
    if (n > kMaxUnionChildren) fail(YS_ERR_DECL, "primitive union has too many children");
    Union u;
    for (int k = 0; k < n; ++k) {
      if (doms[k] < 0 || doms[k] >= int32_t(c->domains.size())) fail(YS_ERR_DECL, "unknown point domain");
      u.children.push_back(doms[k]);
      u.kappa_u = std::max(u.kappa_u, c->domains[doms[k]].kappa());
      u.width = std::max(u.width, c->domains[doms[k]].width());
    }
    c->unions.push_back(std::move(u));
    *id = int32_t(c->unions.size() - 1);
  });
}

int ys_add_stencil_set(ys_context* c, int32_t uni, int32_t arity, int32_t dynamic, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "ys_add_stencil_set");
    if (uni < 0 || uni >= int32_t(c->unions.size())) fail(YS_ERR_DECL, "unknown primitive union");
    if (arity < 2 || arity > 4) fail(YS_ERR_DECL, "stencil arity must be 2, 3 or 4");
    PairSet p;
    p.uni = uni;
    p.arity = arity;
    p.dynamic = dynamic != 0;
    c->pairsets.push_back(std::move(p));
    *id = int32_t(c->pairsets.size() - 1);
  });
}

int ys_set_stencil_primitives(ys_context* c, int32_t set, int32_t kind, int64_t n_a, const int64_t* prims_a,
                              int64_t n_b, const int64_t* prims_b) {
  return guarded(c, [&] {
    if (set < 0 || set >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown stencil set");
    PairSet& p = c->pairsets[set];
    if (kind < 1 || kind > 3) fail(YS_ERR_VALIDATION, "stencil kind must be 1 (PT), 2 (EE) or 3 (PE)");
    StencilPrims& sp = p.prims;
    sp.kind = kind == 1 ? K_PT : kind == 2 ? K_EE : K_PE;
    sp.self = kind == 2;
    sp.aa = kind == 2 ? 2 : 1;
    sp.ab = kind == 1 ? 3 : 2;
    if (sp.aa + sp.ab != p.arity) fail(YS_ERR_DECL, "stencil kind does not match the set's arity");
    if (n_a < 0 || n_b < 0) fail(YS_ERR_VALIDATION, "negative primitive count");
    if (sp.self) n_b = 0;
    int64_t total = 0;
    for (int32_t d : c->unions[p.uni].children) total += c->domains[d].n;
    std::vector<int32_t> a(size_t(n_a * sp.aa)), b(size_t(n_b * sp.ab));
    for (size_t k = 0; k < a.size(); ++k) {
      if (prims_a[k] < 0 || prims_a[k] >= total) fail(YS_ERR_VALIDATION, "primitive index out of the union");
      a[k] = int32_t(prims_a[k]);
    }
    for (size_t k = 0; k < b.size(); ++k) {
      if (prims_b[k] < 0 || prims_b[k] >= total) fail(YS_ERR_VALIDATION, "primitive index out of the union");
      b[k] = int32_t(prims_b[k]);
    }
    sp.na = n_a;
    sp.nb = n_b;
    sp.a.upload(a, c->stream);
    sp.b.upload(b, c->stream);
  });
}

int ys_refresh_stencils(ys_context* c, int32_t set, double dhat, int64_t* n) {
  return guarded(c, [&] {
    require_finalized(*c);
    if (set < 0 || set >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown stencil set");
    if (!c->pairsets[set].dynamic) fail(YS_ERR_VALIDATION, "resize_dynamic on a static stencil set");
    if (!(dhat > 0.0)) fail(YS_ERR_VALIDATION, "dhat must be positive");
    ctx_refresh_stencils(*c, set, dhat, n);
  });
}

int ys_add_pair_set(ys_context* c, int32_t uni, int32_t dynamic, int32_t* id) {
  return ys_add_stencil_set(c, uni, 2, dynamic, id);
}

int ys_set_pairs(ys_context* c, int32_t ps, int64_t n, const int64_t* pairs) {
  return guarded(c, [&] {
    if (ps < 0 || ps >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown pair set");
    PairSet& p = c->pairsets[ps];
    if (!p.dynamic && c->finalized) fail(YS_ERR_VALIDATION, "resize_dynamic on static primitive contact.pp");
    if (n < 0) fail(YS_ERR_VALIDATION, "negative instance count");
    check_pairs_in_range(*c, p, n, pairs);
    p.n = n;
    if (c->finalized) {
      // the device copy is authoritative; ys_get_pairs downloads it lazily.  The
      // pageable upload has staged q before returning, so no synchronisation.
      std::vector<int32_t> q(pairs, pairs + int64_t(p.arity) * n);
      p.pairs.upload(q, c->stream);
      p.h_pairs.clear();
      p.host_stale = n > 0;
    } else {
      p.h_pairs.assign(pairs, pairs + int64_t(p.arity) * n);
      p.host_stale = false;
    }
    ++c->epoch;  // Scene::bump_dynamic_epoch (scene.cpp:198)
  });
}

int ys_pair_count(ys_context* c, int32_t ps, int64_t* n) {
  return guarded(c, [&] {
    if (ps < 0 || ps >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown pair set");
    *n = c->pairsets[ps].n;
  });
}

int ys_get_pairs(ys_context* c, int32_t ps, int64_t* out) {
  return guarded(c, [&] {
    if (ps < 0 || ps >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown pair set");
    PairSet& p = c->pairsets[ps];
    if (p.host_stale) {
      std::vector<int32_t> h = p.pairs.to_host(c->stream);
      p.h_pairs.assign(h.begin(), h.begin() + int64_t(p.arity) * p.n);
      p.host_stale = false;
    }
    std::copy(p.h_pairs.begin(), p.h_pairs.end(), out);
  });
}

int ys_refresh_pairs(ys_context* c, int32_t ps, double dhat, const int32_t* child_is_fixed, int64_t* n) {
  return guarded(c, [&] {
    require_finalized(*c);
    if (ps < 0 || ps >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown pair set");
    if (!c->pairsets[ps].dynamic) fail(YS_ERR_VALIDATION, "resize_dynamic on static primitive contact.pp");
    if (c->pairsets[ps].arity != 2) fail(YS_ERR_DECL, "ys_refresh_pairs: point-point pair sets only");
    ctx_refresh_pairs(*c, ps, dhat, child_is_fixed, n);
  });
}

int ys_add_stable_neo_hookean(ys_context* c, int32_t pos, int64_t nt, const int64_t* t2v, const double* rest,
                              double E, double nu, double weight, int32_t via_f, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "add_stable_neo_hookean");
    check_target(*c, pos, 3, "stable Neo-Hookean positions");
    const int64_t nv = c->targets[pos].n;
    std::vector<int32_t> conn(4 * nt);
    std::vector<double> cd(10 * nt);
    for (int64_t t = 0; t < nt; ++t) {
      for (int l = 0; l < 4; ++l) {
        const int64_t v = t2v[4 * t + l];
        if (v < 0 || v >= nv)
          fail(YS_ERR_VALIDATION, "connectivity 'tet2v': index " + std::to_string(v) + " at position " +
                                      std::to_string(4 * t + l) + " out of range [0, " + std::to_string(nv) + ")");
        conn[4 * t + l] = int32_t(v);
      }
      // rest shape: fr(r, c) = X_{c+1}[r] - X_0[r]; B = fr^T; Binv = B^-1 (energies.cpp:59-74)
      double fr[9];
      const int64_t i0 = t2v[4 * t];
      for (int col = 0; col < 3; ++col) {
        const int64_t ic = t2v[4 * t + col + 1];
        for (int r = 0; r < 3; ++r) fr[3 * r + col] = rest[ic * 3 + r] - rest[i0 * 3 + r];
      }
      const double det = det3(fr);
      if (std::abs(det) < 1e-14) fail(YS_ERR_VALIDATION, "degenerate rest tetrahedron " + std::to_string(t));
      double b[9], cf[9];
      for (int r = 0; r < 3; ++r)
        for (int col = 0; col < 3; ++col) b[3 * r + col] = fr[3 * col + r];
      cof3(b, cf);
      const double db = det3(b);
      for (int r = 0; r < 3; ++r)
        for (int col = 0; col < 3; ++col) cd[10 * t + 3 * r + col] = cf[3 * col + r] / db;
      cd[10 * t + 9] = std::abs(det) / 6.0;
      bool distinct = true;
      for (int a = 0; a < 4; ++a)
        for (int q = a + 1; q < 4; ++q) distinct = distinct && t2v[4 * t + a] != t2v[4 * t + q];
      if (!distinct) fail(YS_ERR_VALIDATION, "degenerate rest tetrahedron " + std::to_string(t));
    }
    Energy e;
    e.kind = K_SNH;
    e.n = nt;
    e.kappa = 4;
    e.width = 12;
    e.target = pos;
    e.mode = via_f ? YS_PROJECT_REDUCED : YS_PROJECT_FULL;
    const double mu = E / (2.0 * (1.0 + nu));
    const double lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    e.prm[0] = mu;
    e.prm[1] = lambda;
    e.prm[2] = 1.0 + 3.0 * mu / (4.0 * lambda);
    e.prm[3] = weight;
    e.conn.upload(conn, c->stream);
    e.cdata.upload(cd, c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
    *id = add_energy(*c, std::move(e));
  });
}

int ys_add_bending(ys_context* c, int32_t pos, int64_t nh, const int64_t* h2v, const double* rest, double k,
                   double weight, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "add_bending");
    check_target(*c, pos, 3, "bending positions");
    const int64_t nv = c->targets[pos].n;
    std::vector<int32_t> conn(4 * nh);
    std::vector<double> cd(nh);
    for (int64_t h = 0; h < nh; ++h) {
      for (int l = 0; l < 4; ++l) {
        const int64_t v = h2v[4 * h + l];
        if (v < 0 || v >= nv)
          fail(YS_ERR_VALIDATION, "connectivity 'hinge2v': index " + std::to_string(v) + " at position " +
                                      std::to_string(4 * h + l) + " out of range [0, " + std::to_string(nv) + ")");
        conn[4 * h + l] = int32_t(v);
      }
      for (int a = 0; a < 4; ++a)
        for (int q = a + 1; q < 4; ++q)
          if (h2v[4 * h + a] == h2v[4 * h + q])
            fail(YS_ERR_VALIDATION, "hinge " + std::to_string(h) + " repeats a vertex");
      const int64_t a = h2v[4 * h], b = h2v[4 * h + 1];
      double acc = 0;
      for (int d = 0; d < 3; ++d) {
        const double diff = rest[a * 3 + d] - rest[b * 3 + d];
        acc += diff * diff;
      }
      cd[h] = (k * weight) * std::sqrt(acc);  // stiffness * weight * l_init (energies.cpp:152)
    }
    Energy e;
    e.kind = K_BENDING;
    e.n = nh;
    e.kappa = 4;
    e.width = 12;
    e.target = pos;
    e.prm[0] = k;
    e.prm[1] = weight;
    e.conn.upload(conn, c->stream);
    e.cdata.upload(cd, c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
    *id = add_energy(*c, std::move(e));
  });
}

int ys_add_inertia(ys_context* c, int32_t domain, const double* mass, const double* xt, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "add_inertia");
    if (domain < 0 || domain >= int32_t(c->domains.size())) fail(YS_ERR_DECL, "unknown point domain");
    const Domain& d = c->domains[domain];
    Energy e;
    e.kind = K_INERTIA;
    e.n = d.n;
    e.kappa = d.kappa();
    e.width = d.width();
    e.domain = domain;
    e.h_mass.assign(mass, mass + d.n);
    e.cdata.upload(e.h_mass, c->stream);
    std::vector<double> a(xt, xt + 3 * d.n);
    e.anchor.upload(a, c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
    *id = add_energy(*c, std::move(e));
  });
}

int ys_set_inertia_anchor(ys_context* c, int32_t id, const double* xt) {
  return guarded(c, [&] {
    if (id < 0 || id >= int32_t(c->energies.size()) || c->energies[id].kind != K_INERTIA)
      fail(YS_ERR_DECL, "ys_set_inertia_anchor: not an inertia energy");
    Energy& e = c->energies[id];
    YS_CUDA(cudaMemcpyAsync(e.anchor.p, xt, 3 * e.n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    YS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int ys_add_affine_orthogonality(ys_context* c, int32_t amat, double k, double weight, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, "add_affine_orthogonality");
    check_target(*c, amat, 9, "affine orthogonality");
    Energy e;
    e.kind = K_ORTHO;
    e.n = c->targets[amat].n;
    e.kappa = 1;
    e.width = 9;
    e.target = amat;
    e.prm[0] = k * weight;
    *id = add_energy(*c, std::move(e));
  });
}

static int add_pair_energy(ys_context* c, int kind, int32_t ps, double dhat, double kappa, double weight,
                           int32_t mode, int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, kind == K_PP ? "add_point_point_barrier" : "add_repulsive_energy");
    if (ps < 0 || ps >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown pair set");
    if (mode != YS_PROJECT_FULL && mode != YS_PROJECT_REDUCED)
      fail(YS_ERR_DECL, "projection mode is not supported by the B200 pair kernels");
    const PairSet& p = c->pairsets[ps];
    const Union& u = c->unions[p.uni];
    Energy e;
    e.kind = kind;
    e.dynamic = p.dynamic;
    e.mode = mode;
    e.pairset = ps;
    e.n = p.n;
    e.kappa = 2 * u.kappa_u;
    e.width = 2 * u.width;
    e.prm[0] = dhat;
    e.prm[1] = kappa;
    e.prm[2] = weight;
    *id = add_energy(*c, std::move(e));
  });
}

// Point-triangle / edge-edge / point-edge barriers (ys_contact4.cuh; not in
// the reference): a stencil set of arity 4 / 4 / 3 over a union of free and
// fixed points, the point-point barrier's b(d) on the squared distance,
// FullProject.
static int add_contact_energy(ys_context* c, int kind, int32_t ps, double dhat, double kappa, double weight,
                              int32_t* id) {
  return guarded(c, [&] {
    require_not_finalized(*c, kind_name(kind));
    if (ps < 0 || ps >= int32_t(c->pairsets.size())) fail(YS_ERR_DECL, "unknown stencil set");
    const PairSet& p = c->pairsets[ps];
    const int want = kind == K_PE ? 3 : 4;
    if (p.arity != want)
      fail(YS_ERR_DECL, std::string(kind_name(kind)) + " needs a stencil set of arity " + std::to_string(want));
    const Union& u = c->unions[p.uni];
    if (u.kappa_u != 1) fail(YS_ERR_DECL, std::string(kind_name(kind)) + ": unions of free and fixed points only");
    if (!(dhat > 0.0)) fail(YS_ERR_VALIDATION, "dhat must be positive");
    Energy e;
    e.kind = kind;
    e.dynamic = p.dynamic;
    e.mode = YS_PROJECT_FULL;
    e.pairset = ps;
    e.n = p.n;
    e.kappa = p.arity;
    e.width = 3 * p.arity;
    e.prm[0] = dhat;
    e.prm[1] = kappa;
    e.prm[2] = weight;
    *id = add_energy(*c, std::move(e));
  });
}

int ys_add_point_triangle_barrier(ys_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t* id) {
  return add_contact_energy(c, K_PT, ps, dhat, kappa, weight, id);
}
int ys_add_edge_edge_barrier(ys_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t* id) {
  return add_contact_energy(c, K_EE, ps, dhat, kappa, weight, id);
}
int ys_add_point_edge_barrier(ys_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t* id) {
  return add_contact_energy(c, K_PE, ps, dhat, kappa, weight, id);
}

int ys_add_point_point_barrier(ys_context* c, int32_t ps, double dhat, double kappa, double weight, int32_t mode,
                               int32_t* id) {
  return add_pair_energy(c, K_PP, ps, dhat, kappa, weight, mode, id);
}

int ys_add_repulsive(ys_context* c, int32_t ps, double weight, int32_t mode, int32_t* id) {
  return add_pair_energy(c, K_REPULSIVE, ps, 0.0, 0.0, weight, mode, id);
}

int ys_finalize(ys_context* c) { return guarded(c, [&] { ctx_finalize(*c); }); }

int ys_refresh_dynamic(ys_context* c) {
  return guarded(c, [&] {
    require_finalized(*c);
    ctx_refresh_dynamic(*c, false);
  });
}

int ys_dynamic_stale(ys_context* c, int32_t* stale) {
  return guarded(c, [&] { *stale = c->seen_epoch != c->epoch ? 1 : 0; });
}

int ys_assemble(ys_context* c, int32_t project, int32_t with_hessian) {
  return guarded(c, [&] {
    require_finalized(*c);
    ctx_assemble(*c, project != 0, with_hessian != 0);
  });
}

int ys_get_gradient(ys_context* c, double* g) {
  return guarded(c, [&] {
    require_finalized(*c);
    c->G.download(g, size_t(c->s), c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int ys_total_energy(ys_context* c, double* e) {
  return guarded(c, [&] {
    require_finalized(*c);
    *e = ctx_total_energy(*c, nullptr);
  });
}

int ys_energy_totals(ys_context* c, double* t) {
  return guarded(c, [&] {
    require_finalized(*c);
    ctx_total_energy(*c, t);
  });
}

int ys_apply_hessian(ys_context* c, const double* x, double* y) {
  return guarded(c, [&] {
    require_finalized(*c);
    c->r.resize(c->s + 2);
    c->hp.resize(c->s + 2);
    YS_CUDA(cudaMemcpyAsync(c->r.p, x, c->s * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    YS_CUDA(cudaMemcpyAsync(c->hp.p, y, c->s * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    ctx_apply_hessian_dev(*c, c->r.p, c->hp.p);
    YS_CUDA(cudaMemcpyAsync(y, c->hp.p, c->s * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    YS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// Everything of a Newton iteration before the solve: dynamic rebuild, local
// evaluation, assembly, block-Jacobi preconditioner (engine.cpp:75-95).
static void step_prepare(Context* c) {
  c->launches = 0;
  c->sell_prepared = false;
  c->sell_filled = false;
  if (c->profiling) YS_CUDA(cudaEventRecord(c->ev[0], c->stream));
  // The static energies' evaluation (SNH, inertia: nearly all of the local
  // work) does not depend on the dynamic structure: it runs on a second
  // stream while the dynamic group is rebuilt (whose host synchronisations
  // would otherwise leave the device idle); ys_set_option("overlap", 0):
  // sequential (bitwise the same step, tested).
  if (c->dist.kind && c->dist.nranks > 1) ctx_dist_static_plan(*c);  // owned-row instance lists (once)
  const bool overlap = c->overlap;
  bool dyn_stencil = false;
  for (auto& e : c->energies) dyn_stencil |= e.dynamic && (e.kind == K_SNH || e.kind == K_BENDING);
  if (overlap && !dyn_stencil) {
    if (!c->stream2) {
      int lo = 0, hi = 0;
      YS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      YS_CUDA(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, c->eval_low_priority ? lo : hi));
      YS_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      YS_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    // the static energies on one side stream (pass B batched over all of
    // them; two streams splitting even / odd energies measured slower once
    // pass B was batched: C5 step 5.02 vs 4.97 ms)
    c->evd_count.resize(std::max(c->evd_count.n, 2 * c->energies.size()));
    c->evd_count.zero(c->stream);
    YS_CUDA(cudaEventRecord(c->ev_fork, c->stream));
    YS_CUDA(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
    ctx_eval_all(*c, true, true, 0, c->stream2, -1, false);
    ctx_gather_all(*c, 0, c->stream2);
    YS_CUDA(cudaEventRecord(c->ev_join, c->stream2));
    try {
      ctx_refresh_dynamic(*c, false);
      // the solve's copy layout needs the structure only: built while the
      // static evaluation still runs on the side stream
      if (!c->dist.kind) pcg_prepare(*c);
      ctx_assemble(*c, true, true, 1, c->ev_join, false);  // errors checked by ctx_build_preconditioner
      // the copy's values (assembled H only) on the side stream, beside the
      // gradient / preconditioner pass on the context stream
      if (!c->dist.kind && c->sell_prepared) {
        YS_CUDA(cudaEventRecord(c->ev_fork, c->stream));
        YS_CUDA(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
        sell_fill_early(*c, c->stream2);
        YS_CUDA(cudaEventRecord(c->ev_join, c->stream2));
      }
    } catch (...) {
      c->sell_prepared = false;
      c->sell_filled = false;
      cudaStreamSynchronize(c->stream2);
      throw;
    }
  } else {
    ctx_refresh_dynamic(*c, false);
    ctx_assemble(*c, true, true, -1, nullptr, false);
  }
  try {
    ctx_build_preconditioner(*c);
    if (c->sell_filled) YS_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  } catch (...) {
    c->sell_prepared = false;  // the prepared layout is consumed by this step's solve only
    c->sell_filled = false;
    if (c->stream2) cudaStreamSynchronize(c->stream2);
    throw;
  }
  if (c->profiling) YS_CUDA(cudaEventRecord(c->ev[5], c->stream));
}

// After the solve: X0 <- X, the step to the host, stage clocks.
static void step_finish(Context* c, double* dx) {
  if (c->profiling) YS_CUDA(cudaEventRecord(c->ev[6], c->stream));
  YS_CUDA(cudaMemcpyAsync(c->X0.p, c->X.p, c->s * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if (dx) c->DX.download(dx, size_t(c->s), c->stream);
  YS_CUDA(cudaStreamSynchronize(c->stream));
  if (c->profiling) {
    float ms = 0.f;
    // [0] refresh [1] eval [2] gather [3] precond [4] pcg [6] total
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    c->stage_ms[0] = ms;
    cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]);
    c->stage_ms[1] = ms;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
    c->stage_ms[2] = ms;
    cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]);
    c->stage_ms[3] = ms;
    cudaEventElapsedTime(&ms, c->ev[5], c->ev[6]);
    c->stage_ms[4] = ms;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[6]);
    c->stage_ms[6] = ms;
  }
}

int ys_minimize_step(ys_context* c, double tol, int64_t max_iter, double* dx, ys_step_stats* stats) {
  return guarded(c, [&] {
    require_finalized(*c);
    auto t0 = std::chrono::steady_clock::now();
    step_prepare(c);
    const double t_asm = elapsed(t0);
    if (max_iter < 0) max_iter = std::max<int64_t>(2 * c->s, 64);
    ys_step_stats local{};
    if (c->dist.kind) ctx_dist_pcg(*c, tol, max_iter, &local);
    else ctx_pcg(*c, tol, max_iter, c->G.p, c->DX.p, &local);
    step_finish(c, dx);
    local.assemble_seconds = t_asm;
    local.solve_seconds = elapsed(t0) - t_asm;
    local.regularized_blocks = c->regularized;
    if (stats) *stats = local;
  });
}

int ys_pcg_history(ys_context* c, int64_t cap, double* h, int64_t* count) {
  return guarded(c, [&] {
    const int64_t n = std::min<int64_t>(cap, std::min<int64_t>(c->hist_count, int64_t(c->hist.n)));
    if (n > 0) c->hist.download(h, size_t(n), c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
    *count = c->hist_count;
  });
}

int ys_gather_targets(ys_context* c, double* x) {
  return guarded(c, [&] {
    require_finalized(*c);
    c->X.download(x, size_t(c->s), c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int ys_scatter_targets(ys_context* c, const double* x) {
  return guarded(c, [&] {
    require_finalized(*c);
    YS_CUDA(cudaMemcpyAsync(c->X.p, x, c->s * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    YS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int ys_step_targets(ys_context* c, double alpha, double* max_abs) {
  return guarded(c, [&] {
    require_finalized(*c);
    const int grid = 256;
    c->scratch.resize(std::max<size_t>(c->scratch.n, grid));
    k_step<<<grid, kTB, 0, c->stream>>>(c->s, c->X0.p, c->DX.p, alpha, c->X.p, c->scratch.p);
    YS_LAUNCH_CHECK();
    std::vector<double> part(grid);
    c->scratch.download(part.data(), grid, c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
    double m = 0.0;
    for (double v : part) m = std::max(m, v);
    if (max_abs) *max_abs = m;
  });
}

int ys_hessian_info(ys_context* c, int32_t which, int64_t* ng, int64_t* nb, int64_t* nv, uint64_t* cs) {
  return guarded(c, [&] {
    require_finalized(*c);
    Structure& st = c->S[which ? 1 : 0];
    if (ng) *ng = int64_t(st.groups.size());
    if (nb) *nb = st.n_blocks;
    if (nv) *nv = st.n_values;
    if (cs) *cs = structure_checksum(*c, st, c->s);
  });
}

int ys_hessian_groups(ys_context* c, int32_t which, int64_t* g) {
  return guarded(c, [&] {
    require_finalized(*c);
    Structure& st = c->S[which ? 1 : 0];
    for (size_t k = 0; k < st.groups.size(); ++k)
      for (int q = 0; q < 5; ++q) g[5 * k + q] = st.groups[k][q];
  });
}

int ys_hessian_coords(ys_context* c, int32_t which, int64_t* row, int64_t* col) {
  return guarded(c, [&] {
    require_finalized(*c);
    Structure& st = c->S[which ? 1 : 0];
    std::vector<int32_t> r = st.row.to_host(c->stream), q = st.col.to_host(c->stream);
    for (int64_t k = 0; k < st.n_blocks; ++k) {
      row[k] = r[k];
      col[k] = q[k];
    }
  });
}

int ys_hessian_values(ys_context* c, int32_t which, double* v) {
  return guarded(c, [&] {
    require_finalized(*c);
    Structure& st = c->S[which ? 1 : 0];
    st.values.download(v, size_t(st.n_values), c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int ys_energy_info(ys_context* c, int32_t id, int64_t* n, int32_t* kappa, int32_t* width, int32_t* dyn) {
  return guarded(c, [&] {
    if (id < 0 || id >= int32_t(c->energies.size())) fail(YS_ERR_DECL, "unknown energy");
    Energy& e = c->energies[id];
    if (n) *n = e.pairset >= 0 ? c->pairsets[e.pairset].n : e.n;
    if (kappa) *kappa = e.kappa;
    if (width) *width = e.width;
    if (dyn) *dyn = e.dynamic ? 1 : 0;
  });
}

int ys_energy_slots(ys_context* c, int32_t id, int64_t* index, int32_t* len, int32_t* col) {
  return guarded(c, [&] {
    require_finalized(*c);
    if (id < 0 || id >= int32_t(c->energies.size())) fail(YS_ERR_DECL, "unknown energy");
    Energy& e = c->energies[id];
    std::vector<DSlot> s = e.slots.to_host(c->stream);
    for (size_t k = 0; k < s.size(); ++k) {
      index[k] = s[k].idx;
      len[k] = s[k].len;
      col[k] = s[k].col;
    }
  });
}

int ys_energy_compressed_sizes(ys_context* c, int32_t id, int32_t* m) {
  return guarded(c, [&] {
    require_finalized(*c);
    if (id < 0 || id >= int32_t(c->energies.size())) fail(YS_ERR_DECL, "unknown energy");
    Energy& e = c->energies[id];
    std::vector<int32_t> h = e.m.to_host(c->stream);
    std::copy(h.begin(), h.end(), m);
  });
}

int ys_diag_blocks(ys_context* c, double* out) {
  return guarded(c, [&] {
    require_finalized(*c);
    c->diag.download(out, size_t(c->diag_vals), c->stream);
    YS_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int ys_device_bytes(ys_context* c, int64_t* bytes) {
  return guarded(c, [&] { *bytes = device_bytes_counter(); });
}

int ys_set_profiling(ys_context* c, int32_t on) {
  return guarded(c, [&] { c->profiling = on != 0; });
}

int ys_stage_times(ys_context* c, double* ms, int64_t* counts) {
  return guarded(c, [&] {
    for (int k = 0; k < 8; ++k) ms[k] = c->stage_ms[k];
    for (int k = 0; k < 8; ++k) ms[8 + k] = c->pcg_phase_ms[k];
    if (counts) {
      counts[0] = c->launches;
      int64_t evd = 0, fb = 0;
      if (c->evd_count.n) {
        std::vector<unsigned int> h = c->evd_count.to_host(c->stream);
        const size_t ne = c->energies.size();
        for (size_t k = 0; k < h.size(); ++k) (k < ne ? evd : fb) += k < 2 * ne ? h[k] : 0;
      }
      counts[1] = evd;  // indefinite 9x9 projections (pass B) in the last assembly
      counts[2] = c->pcg_path;
      counts[3] = fb;   // of those, projected by the Jacobi fallback
    }
  });
}

// --- free-standing BSR (BlockSparseHessian::build + spmv_add + pcg) -------------

int ys_bsr_build(ys_context* c, int64_t s, int64_t n, const int64_t* coords, int32_t* id) {
  return guarded(c, [&] {
    int bs = 0;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t r = coords[4 * k], q = coords[4 * k + 1], row = coords[4 * k + 2], col = coords[4 * k + 3];
      if (row < 0 || col < 0 || row + r > s || col + q > s)
        fail(YS_ERR_VALIDATION, "block coordinate outside the global system");
      if (row > col) fail(YS_ERR_INTERNAL, "block coordinate not upper-triangular");
      if (bs == 0) bs = int(r);
      if (r != bs || q != bs || row % bs || col % bs)
        fail(YS_ERR_VALIDATION, "free-standing BSR systems need uniform square blocks");
    }
    if (bs == 0) bs = 3;
    if (s % bs) fail(YS_ERR_VALIDATION, "system size is not a multiple of the block size");
    auto sub = std::make_unique<ys_context>();
    sub->device = c->device;
    sub->stream = c->stream;
    Target t;
    t.n = s / bs;
    t.rc = bs;
    sub->targets.push_back(t);
    sub->h_target_init.emplace_back();
    ctx_finalize(*sub);  // empty energy groups
    std::vector<uint64_t> keys(n);
    std::vector<uint32_t> pay(n, 0);
    for (int64_t k = 0; k < n; ++k) keys[k] = block_key(bs, bs, coords[4 * k + 2], coords[4 * k + 3]);
    sub->k_in.upload(keys, c->stream);
    sub->p_in.upload(pay, c->stream);
    build_structure_from_keys(*sub, sub->S[0], sub->k_in, sub->p_in, n, s, blocks_view(*sub), false);
    build_spmv_plan(*sub, sub->S[0], blocks_view(*sub));
    sub->bsr_bs = bs;
    c->subs.push_back(std::move(sub));
    *id = int32_t(c->subs.size() - 1);
  });
}

static ys_context& bsr_of(ys_context* c, int32_t id) {
  if (id < 0 || id >= int32_t(c->subs.size())) fail(YS_ERR_DECL, "unknown BSR system");
  return *c->subs[id];
}

int ys_bsr_info(ys_context* c, int32_t id, int64_t* ng, int64_t* nb, int64_t* nv, uint64_t* cs) {
  return guarded(c, [&] {
    ys_context& b = bsr_of(c, id);
    Structure& st = b.S[0];
    if (ng) *ng = int64_t(st.groups.size());
    if (nb) *nb = st.n_blocks;
    if (nv) *nv = st.n_values;
    if (cs) *cs = structure_checksum(b, st, b.s);
  });
}

int ys_bsr_groups(ys_context* c, int32_t id, int64_t* g) {
  return guarded(c, [&] {
    Structure& st = bsr_of(c, id).S[0];
    for (size_t k = 0; k < st.groups.size(); ++k)
      for (int q = 0; q < 5; ++q) g[5 * k + q] = st.groups[k][q];
  });
}

int ys_bsr_coords(ys_context* c, int32_t id, int64_t* row, int64_t* col) {
  return guarded(c, [&] {
    ys_context& b = bsr_of(c, id);
    Structure& st = b.S[0];
    std::vector<int32_t> r = st.row.to_host(b.stream), q = st.col.to_host(b.stream);
    for (int64_t k = 0; k < st.n_blocks; ++k) {
      row[k] = r[k];
      col[k] = q[k];
    }
  });
}

int ys_bsr_set_values(ys_context* c, int32_t id, const double* v) {
  return guarded(c, [&] {
    ys_context& b = bsr_of(c, id);
    Structure& st = b.S[0];
    YS_CUDA(cudaMemcpyAsync(st.values.p, v, st.n_values * sizeof(double), cudaMemcpyHostToDevice, b.stream));
    YS_CUDA(cudaStreamSynchronize(b.stream));
  });
}

int ys_bsr_spmv(ys_context* c, int32_t id, const double* x, double* y) {
  return guarded(c, [&] {
    ys_context& b = bsr_of(c, id);
    b.r.resize(b.s + 2);
    b.hp.resize(b.s + 2);
    YS_CUDA(cudaMemcpyAsync(b.r.p, x, b.s * sizeof(double), cudaMemcpyHostToDevice, b.stream));
    YS_CUDA(cudaMemcpyAsync(b.hp.p, y, b.s * sizeof(double), cudaMemcpyHostToDevice, b.stream));
    spmv_launch(b, b.S[0], nullptr, b.r.p, b.hp.p, true, nullptr, nullptr, pcg_grid(b));
    YS_CUDA(cudaMemcpyAsync(y, b.hp.p, b.s * sizeof(double), cudaMemcpyDeviceToHost, b.stream));
    YS_CUDA(cudaStreamSynchronize(b.stream));
  });
}

int ys_bsr_pcg(ys_context* c, int32_t id, int32_t bs, const double* g, double tol, int64_t max_iter, double* x,
               int64_t* iters, double* rel, int32_t* conv) {
  return guarded(c, [&] {
    ys_context& b = bsr_of(c, id);
    if (bs != 0 && bs != b.bsr_bs) fail(YS_ERR_VALIDATION, "preconditioner block size differs from the system's");
    if (bs == 0) {
      k_identity_minv<<<grid_for(b.NB), kTB, 0, b.stream>>>(b.NB, b.bsr_bs, b.minv.p, b.bflag.p);
      YS_LAUNCH_CHECK();
    } else {
      // diagonal blocks of the system itself (the tests' jacobi_of shim)
      ctx_block_rows(b, true);
      ctx_build_preconditioner(b);
    }
    YS_CUDA(cudaMemcpyAsync(b.G.p, g, b.s * sizeof(double), cudaMemcpyHostToDevice, b.stream));
    ys_step_stats st{};
    ctx_pcg(b, tol, max_iter, b.G.p, b.DX.p, &st);
    b.DX.download(x, size_t(b.s), b.stream);
    YS_CUDA(cudaStreamSynchronize(b.stream));
    if (iters) *iters = st.pcg_iterations;
    if (rel) *rel = st.pcg_residual;
    if (conv) *conv = st.pcg_converged;
  });
}

int ys_bump_dynamic_epoch(ys_context* c) {
  return guarded(c, [&] { ++c->epoch; });
}

int ys_dist_unique_id(unsigned char id[128]) {
  try {
    ctx_dist_unique_id(id);
    return YS_OK;
  } catch (const ys::Error& e) {
    return e.cls;
  }
}

static void check_ranks(int32_t rank, int32_t nranks) {
  if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks)
    fail(YS_ERR_VALIDATION, "distributed solve: rank " + std::to_string(rank) + " of " + std::to_string(nranks) +
                                " is out of range (1..64 ranks)");
}

int ys_dist_init_nccl(ys_context* c, int32_t rank, int32_t nranks, const unsigned char id[128]) {
  return guarded(c, [&] {
    check_ranks(rank, nranks);
    ctx_dist_finalize(*c);
    c->dist.rank = rank;
    c->dist.nranks = nranks;
    ctx_dist_init_nccl(*c, rank, nranks, id);
  });
}

int ys_dist_init_host(ys_context* c, int32_t rank, int32_t nranks, ys_allgather_fn fn, void* user) {
  return guarded(c, [&] {
    check_ranks(rank, nranks);
    if (!fn) fail(YS_ERR_VALIDATION, "distributed solve: null allgather callback");
    ctx_dist_finalize(*c);
    c->dist.rank = rank;
    c->dist.nranks = nranks;
    c->dist.fn = fn;
    c->dist.user = user;
    c->dist.kind = 1;
  });
}

int ys_dist_finalize(ys_context* c) {
  return guarded(c, [&] { ctx_dist_finalize(*c); });
}

int ys_dist_info(ys_context* c, int32_t* rank, int32_t* nranks, int64_t* bounds, int64_t* halo_rows,
                 int64_t* export_rows) {
  return guarded(c, [&] {
    const DistState& d = c->dist;
    if (rank) *rank = d.kind ? d.rank : 0;
    if (nranks) *nranks = d.kind ? d.nranks : 1;
    const bool have = d.kind && int(d.bounds.size()) == d.nranks + 1;
    if (bounds) {
      if (have) std::copy(d.bounds.begin(), d.bounds.end(), bounds);
      else {
        bounds[0] = 0;
        bounds[1] = c->NB;
      }
    }
    const int64_t mine = have ? d.exp_off[d.rank + 1] - d.exp_off[d.rank] : 0;
    if (halo_rows) *halo_rows = have ? d.exp_off[d.nranks] - mine : 0;
    if (export_rows) *export_rows = mine;
  });
}

int ys_dist_eval_counts(ys_context* c, int64_t* evaluated, int64_t* total) {
  return guarded(c, [&] {
    const DistState& d = c->dist;
    const bool part = d.kind && d.nranks > 1 && d.have_static;
    int64_t all = 0;
    for (auto& e : c->energies)
      if (!e.dynamic && (e.kind == K_SNH || e.kind == K_BENDING)) all += e.n;
    if (evaluated) *evaluated = part ? d.eval_owned : all;
    if (total) *total = all;
  });
}

int ys_dist_p2p_open(ys_context* c, int32_t rank, int32_t nranks, unsigned char handle[64]) {
  return guarded(c, [&] {
    require_finalized(*c);
    ctx_dist_p2p_open(*c, rank, nranks, handle);
  });
}

int ys_dist_p2p_connect(ys_context* c, const unsigned char* handles) {
  return guarded(c, [&] {
    if (!handles) fail(YS_ERR_VALIDATION, "P2P solve: null handle table");
    ctx_dist_p2p_connect(*c, handles);
  });
}

int ys_dist_p2p_probe(ys_context* c, int64_t* seen) {
  return guarded(c, [&] { ctx_dist_p2p_probe(*c, seen); });
}

static std::vector<Context*> group_of(ys_context** cs, int32_t n) {
  if (!cs || n < 1 || n > kMaxP2P) fail(YS_ERR_VALIDATION, "P2P group: 1.." + std::to_string(kMaxP2P) + " contexts");
  std::vector<Context*> v;
  for (int k = 0; k < n; ++k) {
    if (!cs[k]) fail(YS_ERR_VALIDATION, "P2P group: null context");
    require_finalized(*cs[k]);
    v.push_back(cs[k]);
  }
  return v;
}

int ys_dist_p2p_group(ys_context** cs, int32_t n) {
  if (!cs || n < 1 || !cs[0]) return YS_ERR_VALIDATION;
  return guarded(cs[0], [&] { ctx_dist_p2p_group(group_of(cs, n)); });
}

int ys_dist_p2p_group_step(ys_context** cs, int32_t n, double tol, int64_t max_iter, double** dx,
                           ys_step_stats* stats) {
  if (!cs || n < 1 || !cs[0]) return YS_ERR_VALIDATION;
  return guarded(cs[0], [&] {
    std::vector<Context*> g = group_of(cs, n);
    for (int k = 0; k < n; ++k)
      if (g[size_t(k)]->dist.kind != 3 || g[size_t(k)]->dist.p2p.group.size() != size_t(n) ||
          g[size_t(k)]->dist.p2p.group[size_t(k)] != g[size_t(k)])
        fail(YS_ERR_VALIDATION, "P2P group: the contexts were not grouped by ys_dist_p2p_group in this order");
    auto t0 = std::chrono::steady_clock::now();
    for (Context* c : g) {
      YS_CUDA(cudaSetDevice(c->device));
      step_prepare(c);
    }
    const double t_asm = elapsed(t0);
    if (max_iter < 0) max_iter = std::max<int64_t>(2 * g[0]->s, 64);
    std::vector<ys_step_stats> local(static_cast<size_t>(n));
    ctx_dist_p2p_solve(g, tol, max_iter, local.data());
    for (int k = 0; k < n; ++k) {
      step_finish(g[size_t(k)], dx ? dx[k] : nullptr);
      local[size_t(k)].assemble_seconds = t_asm;
      local[size_t(k)].solve_seconds = elapsed(t0) - t_asm;
      local[size_t(k)].regularized_blocks = g[size_t(k)]->regularized;
      if (stats) stats[k] = local[size_t(k)];
    }
  });
}

int ys_set_option(ys_context* c, const char* name, int64_t value) {
  return guarded(c, [&] {
    const std::string n = name ? name : "";
    if (n == "overlap") c->overlap = value != 0;
    else if (n == "pcg_copy") c->pcg_copy = value != 0;
    else if (n == "eval_low_priority") c->eval_low_priority = value != 0;  // before the first overlapped step
    else if (n == "pcg_ctas") {
      if (value < 0 || value > 3) fail(YS_ERR_VALIDATION, "pcg_ctas must be 0 (auto) .. 3 (CTAs per SM)");
      c->pcg_ctas = int(value);
    }
    else if (n == "gather_window") {
      if (value < 0 || value > 20) fail(YS_ERR_VALIDATION, "gather_window must be 0..20 (log2 of the window)");
      c->gather_wshift = int(value);
      c->S[0].gorder_valid = false;
    }
    else if (n == "eval_evd") {
      if (value < 0 || value > 2)
        fail(YS_ERR_VALIDATION, "eval_evd must be 0 (Jacobi), 1 (clamped eigenpairs) or 2 (every element through the fallback)");
      c->evd_mode = int(value);
    } else fail(YS_ERR_VALIDATION, "unknown option '" + n + "'");
  });
}

int ys_stream(ys_context* c, void** stream) {
  return guarded(c, [&] { *stream = reinterpret_cast<void*>(c->stream); });
}

int ys_time_kernel(ys_context* c, int32_t which, int32_t reps, double* avg_ms, double* bytes) {
  return guarded(c, [&] {
    require_finalized(*c);
    if (reps < 1) reps = 1;
    cudaStream_t s = c->stream;
    double alg = 0.0;
    auto launch = [&]() {
      if (which == 3) {
        spmv_sell(*c, c->p.p, c->hp.p);  // the PCG's SpMV: the sliced-ELL copy, 4 lanes per row
      } else if (which == 0) {
        spmv_launch(*c, c->S[0], &c->S[1], c->p.p, c->hp.p, false, nullptr, nullptr, pcg_grid(*c));
      } else if (which == 1) {
        ctx_gather_all(*c);
        ctx_block_rows(*c, true);
      } else if (which == 2) {
        ctx_eval_all(*c, true, true);
      } else if (which == 4) {
        alg = fp64_probe(*c);
      } else {
        fail(YS_ERR_VALIDATION, "ys_time_kernel: unknown kernel class");
      }
    };
    if (which == 3) {
      if (!c->uniform3) fail(YS_ERR_VALIDATION, "ys_time_kernel(3): the sliced-ELL copy needs uniform 3x3 blocks");
      sell_build(*c, 4);
    }
    if (which == 0 || which == 3) {
      c->p.resize(c->s + 2);
      c->hp.resize(c->s + 2);
      YS_CUDA(cudaMemcpyAsync(c->p.p, c->G.p, c->s * sizeof(double), cudaMemcpyDeviceToDevice, s));
      // 8 r c (values) + 8 (two int32 coords) per upper block, 16 s per SpMV
      for (int w = 0; w < 2; ++w)
        for (auto& g : c->S[w].groups) alg += double(g[3]) * (8.0 * g[0] * g[1] + 8.0);
      alg += 16.0 * double(c->s);
    } else if (which == 1) {
      // per instance 8 sum(r c) + 4 #dest + 8 width + 4 kappa; once 8 nvalues + 8 s + 8 diag
      for (auto& e : c->energies) {
        if (e.n == 0 || e.kappa == 0) continue;
        alg += 8.0 * double(e.hsize) + 4.0 * double(e.ndest) + 8.0 * double(e.n) * e.width + 4.0 * double(e.n) * e.kappa;
      }
      alg += 8.0 * double(c->S[0].n_values + c->S[1].n_values) + 8.0 * double(c->s) + 8.0 * double(c->diag_vals);
    }
    launch();  // warm
    YS_CUDA(cudaEventRecord(c->ev[7], s));
    for (int k = 0; k < reps; ++k) launch();
    YS_CUDA(cudaEventRecord(c->ev[8], s));
    YS_CUDA(cudaEventSynchronize(c->ev[8]));
    float ms = 0.f;
    YS_CUDA(cudaEventElapsedTime(&ms, c->ev[7], c->ev[8]));
    *avg_ms = double(ms) / reps;
    if (bytes) *bytes = alg;
  });
}

}  // extern "C"
