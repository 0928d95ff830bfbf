// C++ drop-in check: the reference's cfd::simulation usage pattern, verbatim
// except for the include and the namespace alias (see include/sforge_b200.hpp).
#include <cstdio>
#include <cstring>

#include "sforge_b200.hpp"

namespace sforge = sforge_b200;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 64;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 1;
  const int workers = argc > 3 ? std::atoi(argv[3]) : 1;
  try {
    sforge::cfd::solver_config cfg;
    cfg.dom = sforge::cfd::unit_box(n, n, n);
    cfg.reynolds = 100.0;
    cfg.symmetry_z = false;
    sforge::cfd::simulation sim(cfg, sforge::cfd::cavity_fluid(cfg), workers);
    sim.init_cavity();
    sforge::cfd::step_stats st;
    for (int i = 0; i < steps; ++i) st = sim.step();
    std::printf("dt=%.17g sweeps=%d residual=%.17g checksum=%016llx\n", st.dt, st.sweeps, st.residual,
                (unsigned long long)sim.checksum());
    // reference error texts come through as the reference exception types
    try {
      sim.run_kernel("PRESSURE_SWEEP", {{"color", 0.0}});
    } catch (const sforge::exec::exec_error& e) {
      std::printf("exec_error: %s\n", e.what());
    }
    return 0;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
}
