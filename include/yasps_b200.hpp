// yasps_b200.hpp — header-only C++17 facade over the C-ABI with the public
// shape of relsim::Engine (engine.hpp:27-80) and relsim's exception classes
// (core.hpp:33-71).  C++ hosts use this; the reference-side adapter that maps
// a relsim::Scene onto it is shown in INTEGRATION.md.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <array>
#include <string>
#include <vector>

#include "yasps_b200.h"

namespace yasps {

// relsim's error families (UserError -> exit 2, NumericalError -> exit 3)
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct UserError : Error { using Error::Error; };
struct ValidationError : UserError { using UserError::UserError; };
struct DeclError : UserError { using UserError::UserError; };
struct NumericalError : Error { using Error::Error; };
struct InternalError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

enum class ProjectionMode { FullProject = YS_PROJECT_FULL, ReducedProject = YS_PROJECT_REDUCED };

struct StepStats {  // engine.hpp:15-21
  int64_t pcg_iterations = 0;
  double pcg_residual = 0.0;
  bool pcg_converged = false;
  double assemble_seconds = 0.0;
  std::vector<double> residual_history;
};

class Engine {
 public:
  explicit Engine(int device = 0) {
    if (ys_create(&ctx_, device) != YS_OK)
      throw DeviceError("yasps_b200: no sm_100 device " + std::to_string(device) + " (no CPU fallback)");
  }
  ~Engine() { ys_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // ---- scene registration (Scene / energies.hpp builders) -----------------
  int32_t add_target(int64_t instances, int32_t rc, const std::vector<double>& values = {}) {
    int32_t id = -1;
    check(ys_add_target(ctx_, instances, rc, &id));
    targets_.push_back({instances, rc});
    if (!values.empty()) check(ys_set_target_values(ctx_, id, values.data()));
    return id;
  }
  int32_t add_free_points(int32_t position_target) {
    int32_t id = -1;
    check(ys_add_points(ctx_, YS_POINTS_FREE, targets_.at(position_target).first, position_target, -1, nullptr,
                        nullptr, &id));
    return id;
  }
  int32_t add_affine_points(int32_t amat, int32_t trans, const std::vector<int64_t>& v2b,
                            const std::vector<double>& rest) {
    int32_t id = -1;
    check(ys_add_points(ctx_, YS_POINTS_AFFINE, int64_t(v2b.size()), amat, trans, v2b.data(), rest.data(), &id));
    return id;
  }
  int32_t add_fixed_points(const std::vector<double>& positions) {
    int32_t id = -1;
    check(ys_add_points(ctx_, YS_POINTS_FIXED, int64_t(positions.size() / 3), -1, -1, nullptr, positions.data(), &id));
    return id;
  }
  int32_t add_point_union(const std::vector<int32_t>& domains) {
    int32_t id = -1;
    check(ys_add_point_union(ctx_, int32_t(domains.size()), domains.data(), &id));
    return id;
  }
  int32_t add_pair_set(int32_t uni, bool dynamic) {
    int32_t id = -1;
    check(ys_add_pair_set(ctx_, uni, dynamic ? 1 : 0, &id));
    return id;
  }
  void resize_dynamic(int32_t pairset, const std::vector<int64_t>& pairs) {
    check(ys_set_pairs(ctx_, pairset, int64_t(pairs.size() / 2), pairs.data()));
  }
  int32_t add_stable_neo_hookean(int32_t pos, const std::vector<int64_t>& t2v, const std::vector<double>& rest,
                                 double youngs, double poisson, double weight, bool via_deformation_gradient) {
    int32_t id = -1;
    check(ys_add_stable_neo_hookean(ctx_, pos, int64_t(t2v.size() / 4), t2v.data(), rest.data(), youngs, poisson,
                                    weight, via_deformation_gradient ? 1 : 0, &id));
    return id;
  }
  int32_t add_point_point_barrier(int32_t pairset, double dhat, double kappa, double weight,
                                  ProjectionMode mode = ProjectionMode::FullProject) {
    int32_t id = -1;
    check(ys_add_point_point_barrier(ctx_, pairset, dhat, kappa, weight, int32_t(mode), &id));
    return id;
  }
  int32_t add_repulsive_energy(int32_t pairset, double weight, ProjectionMode mode = ProjectionMode::FullProject) {
    int32_t id = -1;
    check(ys_add_repulsive(ctx_, pairset, weight, int32_t(mode), &id));
    return id;
  }
  int32_t add_inertia(int32_t domain, const std::vector<double>& mass, const std::vector<double>& x_tilde) {
    int32_t id = -1;
    check(ys_add_inertia(ctx_, domain, mass.data(), x_tilde.data(), &id));
    return id;
  }
  void set_inertia_anchor(int32_t energy, const std::vector<double>& x_tilde) {
    check(ys_set_inertia_anchor(ctx_, energy, x_tilde.data()));
  }
  int32_t add_affine_orthogonality(int32_t amat, double stiffness, double weight) {
    int32_t id = -1;
    check(ys_add_affine_orthogonality(ctx_, amat, stiffness, weight, &id));
    return id;
  }
  int32_t add_bending(int32_t pos, const std::vector<int64_t>& h2v, const std::vector<double>& rest, double stiffness,
                      double weight) {
    int32_t id = -1;
    check(ys_add_bending(ctx_, pos, int64_t(h2v.size() / 4), h2v.data(), rest.data(), stiffness, weight, &id));
    return id;
  }

  // ---- contact beyond point-point (not in the reference) --------------------
  int32_t add_stencil_set(int32_t union_id, int32_t arity, bool dynamic) {
    int32_t id = -1;
    check(ys_add_stencil_set(ctx_, union_id, arity, dynamic ? 1 : 0, &id));
    return id;
  }
  // kind 1 PT (points, triangles), 2 EE (edges), 3 PE (points, edges); union-local point indices
  void set_stencil_primitives(int32_t set, int32_t kind, const std::vector<int64_t>& a, int64_t arity_a,
                              const std::vector<int64_t>& b = {}, int64_t arity_b = 1) {
    check(ys_set_stencil_primitives(ctx_, set, kind, int64_t(a.size()) / arity_a, a.data(),
                                    int64_t(b.size()) / arity_b, b.empty() ? nullptr : b.data()));
  }
  int64_t refresh_stencils(int32_t set, double dhat) {
    int64_t n = 0;
    check(ys_refresh_stencils(ctx_, set, dhat, &n));
    return n;
  }
  int32_t add_point_triangle_barrier(int32_t set, double dhat, double kappa, double weight) {
    int32_t id = -1;
    check(ys_add_point_triangle_barrier(ctx_, set, dhat, kappa, weight, &id));
    return id;
  }
  int32_t add_edge_edge_barrier(int32_t set, double dhat, double kappa, double weight) {
    int32_t id = -1;
    check(ys_add_edge_edge_barrier(ctx_, set, dhat, kappa, weight, &id));
    return id;
  }
  int32_t add_point_edge_barrier(int32_t set, double dhat, double kappa, double weight) {
    int32_t id = -1;
    check(ys_add_point_edge_barrier(ctx_, set, dhat, kappa, weight, &id));
    return id;
  }

  // ---- Simulation helpers on the device -------------------------------------
  // refresh_dynamic_pairs (sim.cpp:456-484): the reference's pair list and order
  int64_t refresh_pairs(int32_t pairset, double dhat, const std::vector<int32_t>& child_is_fixed = {}) {
    int64_t n = 0;
    check(ys_refresh_pairs(ctx_, pairset, dhat, child_is_fixed.empty() ? nullptr : child_is_fixed.data(), &n));
    return n;
  }
  // X = X0 - alpha dx of the last minimize_step; returns |alpha dx|_inf (sim.cpp:545-562)
  double step_targets(double alpha) {
    double m = 0.0;
    check(ys_step_targets(ctx_, alpha, &m));
    return m;
  }
  void set_option(const char* name, int64_t value) { check(ys_set_option(ctx_, name, value)); }

  // ---- relsim::Engine members ---------------------------------------------
  void build() {  // Engine::Engine (engine.cpp:7-20)
    check(ys_finalize(ctx_));
    check(ys_total_dofs(ctx_, &s_));
  }
  void refresh_dynamic() { check(ys_refresh_dynamic(ctx_)); }
  bool dynamic_stale() const {
    int32_t st = 0;
    check(ys_dynamic_stale(ctx_, &st));
    return st != 0;
  }
  void assemble(bool project = true, bool with_hessian = true) {
    check(ys_assemble(ctx_, project ? 1 : 0, with_hessian ? 1 : 0));
  }
  std::vector<double> gradient() const {
    std::vector<double> g(static_cast<size_t>(s_));
    check(ys_get_gradient(ctx_, g.data()));
    return g;
  }
  double total_energy() {
    double e = 0.0;
    check(ys_total_energy(ctx_, &e));
    return e;
  }
  void apply_hessian(const std::vector<double>& x, std::vector<double>& y) const {
    check(ys_apply_hessian(ctx_, x.data(), y.data()));
  }
  // Solves H dx = g; returns dx sliced per target in registration order, unnegated.
  std::vector<std::vector<double>> minimize_step(double tol = 1e-6, int64_t max_iter = -1,
                                                 StepStats* stats = nullptr) {
    std::vector<double> dx(static_cast<size_t>(s_));
    ys_step_stats st{};
    check(ys_minimize_step(ctx_, tol, max_iter, dx.data(), &st));
    if (stats) {
      stats->pcg_iterations = st.pcg_iterations;
      stats->pcg_residual = st.pcg_residual;
      stats->pcg_converged = st.pcg_converged != 0;
      stats->assemble_seconds = st.assemble_seconds;
      std::vector<double> h(size_t(st.pcg_iterations + 1));
      int64_t n = 0;
      check(ys_pcg_history(ctx_, int64_t(h.size()), h.data(), &n));
      h.resize(size_t(std::min<int64_t>(n, int64_t(h.size()))));
      stats->residual_history = std::move(h);
    }
    std::vector<std::vector<double>> out;
    size_t off = 0;
    for (auto& t : targets_) {
      const size_t n = size_t(t.first * t.second);
      out.emplace_back(dx.begin() + off, dx.begin() + off + n);
      off += n;
    }
    return out;
  }
  std::vector<double> gather_targets() const {
    std::vector<double> x(static_cast<size_t>(s_));
    check(ys_gather_targets(ctx_, x.data()));
    return x;
  }
  void scatter_targets(const std::vector<double>& x) {
    if (int64_t(x.size()) != s_) throw ValidationError("scatter_targets: length mismatch");
    check(ys_scatter_targets(ctx_, x.data()));
  }
  int64_t total_dofs() const { return s_; }
  ys_context* raw() { return ctx_; }

  // ---- several GPUs of one node: peer-memory row-partitioned solve.  open()
  // returns this rank's 64-byte window handle; the caller all-gathers the
  // handles (MPI, torch.distributed, ...) in rank order and connects.
  std::array<unsigned char, 64> p2p_open(int32_t rank, int32_t nranks) {
    std::array<unsigned char, 64> h{};
    check(ys_dist_p2p_open(ctx_, rank, nranks, h.data()));
    return h;
  }
  void p2p_connect(const std::vector<std::array<unsigned char, 64>>& handles) {
    std::vector<unsigned char> table;
    for (const auto& h : handles) table.insert(table.end(), h.begin(), h.end());
    check(ys_dist_p2p_connect(ctx_, table.data()));
  }
  void dist_finalize() { check(ys_dist_finalize(ctx_)); }

 private:
  void check(int status) const {
    if (status == YS_OK) return;
    const std::string msg = ys_last_error(ctx_);
    switch (status) {
      case YS_ERR_VALIDATION: throw ValidationError(msg);
      case YS_ERR_DECL: throw DeclError(msg);
      case YS_ERR_NUMERICAL: throw NumericalError(msg);
      case YS_ERR_INTERNAL: throw InternalError(msg);
      default: throw DeviceError(msg);
    }
  }
  ys_context* ctx_ = nullptr;
  int64_t s_ = 0;
  std::vector<std::pair<int64_t, int32_t>> targets_;
};

}  // namespace yasps
