// C++ host through the facade: a stiff two-cluster contact scene (free +
// affine points, PP barrier), one Newton step; prints iterations and |dx|.
#include <cmath>
#include <cstdio>

#include "yasps_b200.hpp"

int main() {
  try {
    yasps::Engine eng(0);
    const std::vector<double> pa = {-0.12, 0, 0, -0.18, 0.05, 0.02, -0.18, -0.05, -0.02, -0.24, 0, 0.04};
    const std::vector<double> pb = {0.005, 0, 0, 0.06, 0.06, 0, 0.06, -0.06, 0.02, 0.12, 0, -0.03};
    const int32_t tf = eng.add_target(4, 3, pa);
    const int32_t ta = eng.add_target(1, 9, {1, 0, 0, 0, 1, 0, 0, 0, 1});
    const int32_t tt = eng.add_target(1, 3, {0, 0, 0});
    const int32_t df = eng.add_free_points(tf);
    const int32_t da = eng.add_affine_points(ta, tt, {0, 0, 0, 0}, pb);
    eng.add_affine_orthogonality(ta, 1e4, 2.5e-5);
    eng.add_inertia(df, {0.8, 0.8, 0.8, 0.8}, pa);
    eng.add_inertia(da, {1.2, 1.2, 1.2, 1.2}, pb);
    const int32_t u = eng.add_point_union({df, da});
    const int32_t ps = eng.add_pair_set(u, true);
    eng.add_point_point_barrier(ps, 0.02, 1e8, 2.5e-5);
    eng.resize_dynamic(ps, {0, 4});
    eng.build();
    yasps::StepStats st;
    auto dx = eng.minimize_step(1e-8, -1, &st);
    double m = 0;
    for (auto& part : dx)
      for (double v : part) m = std::fmax(m, std::fabs(v));
    std::printf("cpp facade ok: dofs=%lld pcg_iterations=%lld converged=%d max|dx|=%.6e history=%zu\n",
                (long long)eng.total_dofs(), (long long)st.pcg_iterations, int(st.pcg_converged), m,
                st.residual_history.size());
    bool threw = false;
    try {
      eng.resize_dynamic(ps, {0, 99});
    } catch (const yasps::ValidationError&) {
      threw = true;
    }
    return (st.pcg_converged && threw) ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
