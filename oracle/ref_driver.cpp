// ref_driver — TEST INFRASTRUCTURE ONLY.  Links the reference (relsim) compiled
// from its unmodified sources (oracle/ref_build.sh) and records one prepared
// Newton step through the reference's own public API, for the parity tests
// (tests/test_reference.py) and the golden fixtures (tools/make_golden.py):
//
//   ref_driver <config.json> <out_prefix> [--x X.bin] [--threads N] [--no-step]
//
//  1. Simulation(config)                                  (sim.cpp:190-201)
//  2. optional: Engine::scatter_targets(X)  (the prepared, jittered state)
//  3. begin_frame's x_tilde update for every inertial body (sim.cpp:488-500),
//     through the public Evaluator and Attr::update_value
//  4. Simulation::refresh_dynamic_pairs()                 (sim.cpp:456-484)
//  5. Engine::minimize_step(pcg_tol, -1, &stats)          (engine.cpp:75-101)
//  6. Engine::assemble(true, true)                        (engine.cpp:47-60)
//  7. writes <out_prefix>.<name>.bin (raw little-endian arrays) and
//     <out_prefix>.json (scalars): structure checksums, groups, coordinates and
//     values of both BlockSparseHessians, the contact pair table, gradient,
//     diagonal blocks, the step dx (targets in registration order), PCG
//     iterations / residual / history, total energy.
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include <json.hpp>

#include "relsim/sim.hpp"

using namespace relsim;

namespace {

template <class T>
void dump(const std::string& path, const T* p, size_t n) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(p), std::streamsize(n * sizeof(T)));
}

void dump_hessian(const std::string& pre, const std::string& tag, const BlockSparseHessian& h, nlohmann::json& meta) {
  std::vector<int64_t> groups;
  for (const auto& g : h.groups()) {
    groups.push_back(g.rows);
    groups.push_back(g.cols);
    groups.push_back(g.coord_start);
    groups.push_back(g.count);
    groups.push_back(g.value_start);
  }
  dump(pre + "." + tag + "_groups.bin", groups.data(), groups.size());
  dump(pre + "." + tag + "_row.bin", h.row_coordinate().data(), h.row_coordinate().size());
  dump(pre + "." + tag + "_col.bin", h.col_coordinate().data(), h.col_coordinate().size());
  dump(pre + "." + tag + "_values.bin", h.values().data(), h.values().size());
  meta[tag + "_checksum"] = std::to_string(h.structure_checksum());
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: ref_driver <config.json> <out_prefix> [--x X.bin] [--threads N] [--no-step]\n";
    return 2;
  }
  const std::string cfg_path = argv[1], pre = argv[2];
  std::string xpath;
  int threads = 0;
  bool do_step = true;
  for (int i = 3; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--x" && i + 1 < argc) xpath = argv[++i];
    else if (a == "--threads" && i + 1 < argc) threads = std::stoi(argv[++i]);
    else if (a == "--no-step") do_step = false;
  }
  try {
    SimConfig config = SimConfig::load(cfg_path);
    if (threads > 0) config.threads = threads;
    Simulation sim(config);
    Engine& eng = sim.engine();
    const Index s = eng.layout().total_dofs;
    if (!xpath.empty()) {
      std::ifstream f(xpath, std::ios::binary);
      std::vector<double> x(static_cast<size_t>(s));
      f.read(reinterpret_cast<char*>(x.data()), std::streamsize(x.size() * sizeof(double)));
      if (!f) throw ValidationError("cannot read " + std::to_string(s) + " doubles from " + xpath);
      eng.scatter_targets(Eigen::Map<const VectorXd>(x.data(), s));
    }
    // begin_frame (sim.cpp:488-500) with the bodies' initial (zero) velocities
    for (const Body& b : sim.bodies()) {
      if (!b.inertial) continue;
      InstanceTensor t = eng.evaluator().evaluate(b.position);
      std::vector<double> xt;
      for (Index i = 0; i < t.count(); ++i) {
        VectorXd v = vec_rm(t.instance(i));
        for (Index d = 0; d < v.size(); ++d) xt.push_back(v[d]);
      }
      for (size_t k = 0; k < xt.size(); ++k) {
        const double vel = b.velocity.size() == Index(xt.size()) ? b.velocity[Index(k)] : 0.0;
        xt[k] += config.dt * vel;
      }
      for (size_t i = 0; i * size_t(b.dim) < xt.size(); ++i)
        for (int d = 0; d < b.dim; ++d) xt[i * size_t(b.dim) + size_t(d)] += config.dt * config.dt * config.gravity[size_t(d)];
      b.x_tilde.update_value(xt);
    }
    const Index npairs = sim.refresh_dynamic_pairs();
    nlohmann::json meta;
    meta["total_dofs"] = s;
    meta["pairs"] = npairs;
    if (Mesh* cm = sim.scene().find_mesh("contact")) {
      if (Domain* pp = cm->find_domain("pp")) {
        const auto& idx = pp->connectivity("pp2v").indices;
        dump(pre + ".pairs.bin", idx.data(), idx.size());
      }
    }
    if (do_step) {
      StepStats st;
      std::vector<VectorXd> dx = eng.minimize_step(config.pcg_tol, -1, &st);
      std::vector<double> flat;
      for (const VectorXd& part : dx)
        for (Index i = 0; i < part.size(); ++i) flat.push_back(part[i]);
      dump(pre + ".dx.bin", flat.data(), flat.size());
      dump(pre + ".pcg_history.bin", st.residual_history.data(), st.residual_history.size());
      meta["pcg_iterations"] = st.pcg_iterations;
      meta["pcg_residual"] = st.pcg_residual;
      meta["pcg_converged"] = st.pcg_converged;
    }
    eng.assemble(true, true);
    dump_hessian(pre, "static", eng.static_hessian(), meta);
    dump_hessian(pre, "dynamic", eng.dynamic_hessian(), meta);
    const VectorXd& g = eng.gradient();
    dump(pre + ".gradient.bin", g.data(), size_t(g.size()));
    std::vector<double> diag;
    for (const MatrixXd& blk : eng.diag().blocks)
      for (Index i = 0; i < blk.rows(); ++i)
        for (Index j = 0; j < blk.cols(); ++j) diag.push_back(blk(i, j));
    dump(pre + ".diag.bin", diag.data(), diag.size());
    meta["energy"] = eng.total_energy();
    std::ofstream(pre + ".json") << meta.dump(1) << "\n";
  } catch (const UserError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
  return 0;
}
