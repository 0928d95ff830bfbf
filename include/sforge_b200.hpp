// sforge_b200.hpp -- header-only C++ face of the C ABI (sforge_b200.h) with the
// reference's names, so code written against stencilforge's cfd::simulation
// (proj/include/stencilforge/cfd.hpp:173-766), grid::gather/scatter
// (io.hpp:25-65) and cli::field_checksum (bench.hpp:24-39) switches by
// changing the include and namespace:
//
//   #include "sforge_b200.hpp"
//   namespace sforge = sforge_b200;          // was: stencilforge headers
//   sforge::cfd::solver_config cfg; cfg.dom = sforge::cfd::unit_box(64, 64, 64);
//   sforge::cfd::simulation sim(cfg, sforge::cfd::cavity_fluid(cfg), /*workers=*/1);
//   sim.init_cavity(); auto st = sim.step();
//
// Errors surface as the reference's exception types (cfd_error, grid_error,
// exec_error) carrying the reference's message texts.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sforge_b200.h"

namespace sforge_b200 {

namespace grid {
using index_t = std::int64_t;
struct grid_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct domain {  // grid.hpp:25-31
  std::array<index_t, 3> extents{};
  std::array<double, 3> spacing{};
  std::array<double, 3> origin{};
  index_t cells() const { return extents[0] * extents[1] * extents[2]; }
};
enum class reduce_op { max_abs = SF_MAX_ABS, sum = SF_SUM, sum_sq = SF_SUM_SQ, max_abs_diff = SF_MAX_ABS_DIFF };
}  // namespace grid

namespace exec {
struct exec_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
enum class region { all = SF_REGION_ALL, interior = SF_REGION_INTERIOR, boundary = SF_REGION_BOUNDARY };
enum class run_mode { plain = 0, overlap = 1 };
}  // namespace exec

namespace cfd {
struct cfd_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == SF_OK) return;
  const std::string m = sf_last_error();
  switch (rc) {
    case SF_ERR_GRID: throw grid::grid_error(m);
    case SF_ERR_EXEC: throw exec::exec_error(m);
    case SF_ERR_CONFIG:
    case SF_ERR_CFD: throw cfd_error(m);
    default: throw std::runtime_error(m);
  }
}

struct fluid_params {  // cfd.hpp:29-41
  double viscosity = 0.01;
  double density = 1.0;
  std::array<double, 3> body_force{0.0, 0.0, 0.0};
  double lid_speed = 1.0;
  double blend = 0.0;
};

struct solver_config {  // cfd.hpp:43-67
  grid::domain dom;
  std::array<bool, 3> periodic{false, false, false};
  double reynolds = 100.0;
  double sigma = 0.5;
  double tolerance = 1e-6;
  double omega = 1.7;
  int max_sweeps = 500;
  bool symmetry_z = true;
  int output_cadence = 0;
};

inline grid::domain unit_box(grid::index_t nx, grid::index_t ny, grid::index_t nz) {  // cfd.hpp:69-74
  return {{nx, ny, nz}, {1.0 / double(nx), 1.0 / double(ny), 1.0 / double(nz)}, {0.0, 0.0, 0.0}};
}

inline fluid_params cavity_fluid(const solver_config& cfg, double alpha = 0.0) {  // cfd.hpp:78-84
  fluid_params p;
  p.lid_speed = 1.0;
  p.viscosity = p.lid_speed * 1.0 / cfg.reynolds;
  p.blend = alpha;
  return p;
}

struct step_stats {  // cfd.hpp:86-90
  double dt = 0.0;
  int sweeps = 0;
  double residual = 0.0;
};

enum class kernel_form { rows, points };

// Device-resident cfd::simulation (cfd.hpp:173-766).
class simulation {
 public:
  simulation(const solver_config& cfg, const fluid_params& par, int workers = 1,
             exec::run_mode mode = exec::run_mode::plain, std::array<int, 3> tile_override = {0, 0, 0},
             int ghost = 1, kernel_form form = kernel_form::rows, int device = 0)
      : cfg_(cfg), par_(par) {
    sf_solver_config c{};
    for (int a = 0; a < 3; ++a) {
      c.extents[a] = cfg.dom.extents[a];
      c.spacing[a] = cfg.dom.spacing[a];
      c.origin[a] = cfg.dom.origin[a];
      c.periodic[a] = cfg.periodic[a] ? 1 : 0;
    }
    c.reynolds = cfg.reynolds;
    c.sigma = cfg.sigma;
    c.tolerance = cfg.tolerance;
    c.omega = cfg.omega;
    c.max_sweeps = cfg.max_sweeps;
    c.symmetry_z = cfg.symmetry_z ? 1 : 0;
    c.output_cadence = cfg.output_cadence;
    sf_fluid_params p{};
    p.viscosity = par.viscosity;
    p.density = par.density;
    for (int a = 0; a < 3; ++a) p.body_force[a] = par.body_force[a];
    p.lid_speed = par.lid_speed;
    p.blend = par.blend;
    sf_sim_options o;
    sf_sim_options_default(&o);
    o.workers = workers;
    o.mode = mode == exec::run_mode::overlap ? 1 : 0;
    for (int a = 0; a < 3; ++a) o.tile[a] = tile_override[a];
    o.ghost = ghost;
    o.form = form == kernel_form::points ? 1 : 0;
    o.device = device;
    sf_sim* h = nullptr;
    check(sf_sim_create(&c, &p, &o, &h));
    h_.reset(h);
  }

  void init_cavity() { check(sf_sim_init_cavity(h_.get())); }
  void init_uniform(std::array<double, 3> c) { check(sf_sim_init_uniform(h_.get(), c[0], c[1], c[2])); }
  void init_taylor_green() { check(sf_sim_init_taylor_green(h_.get())); }

  double compute_dt() {
    double dt = 0.0;
    check(sf_sim_compute_dt(h_.get(), &dt));
    return dt;
  }
  void provisional(double dt) { check(sf_sim_provisional(h_.get(), dt)); }
  std::pair<int, double> pressure_iteration(double dt) {
    int s = 0;
    double r = 0.0;
    check(sf_sim_pressure_iteration(h_.get(), dt, &s, &r));
    return {s, r};
  }
  step_stats step() {
    sf_step_stats st{};
    check(sf_sim_step(h_.get(), &st));
    return {st.dt, st.sweeps, st.residual};
  }
  step_stats advance(int n) {
    sf_step_stats st{};
    check(sf_sim_advance(h_.get(), n, &st));
    return {st.dt, st.sweeps, st.residual};
  }

  double max_divergence() {
    double v = 0.0;
    check(sf_sim_max_divergence(h_.get(), &v));
    return v;
  }
  double steady_delta() {
    double v = 0.0;
    check(sf_sim_steady_delta(h_.get(), &v));
    return v;
  }
  double kinetic_energy() {
    double v = 0.0;
    check(sf_sim_kinetic_energy(h_.get(), &v));
    return v;
  }
  double taylor_green_error(double t) {
    double v = 0.0;
    check(sf_sim_taylor_green_error(h_.get(), t, &v));
    return v;
  }

  double time() const { return sf_sim_time(h_.get()); }
  long step_count() const { return sf_sim_step_count(h_.get()); }
  int pending_color() { return sf_sim_pending_color(h_.get()); }
  const solver_config& config() const { return cfg_; }
  const fluid_params& params() const { return par_; }

  // executor operations on the simulation's fields (executor.hpp:500-527)
  void refresh(const std::vector<std::string>& fields) {
    std::vector<const char*> f;
    for (auto& s : fields) f.push_back(s.c_str());
    check(sf_sim_refresh(h_.get(), f.data(), (int)f.size()));
  }
  void run_kernel(const std::string& name, const std::map<std::string, double>& params,
                  exec::region reg = exec::region::all) {
    std::vector<const char*> n;
    std::vector<double> v;
    for (auto& kv : params) {
      n.push_back(kv.first.c_str());
      v.push_back(kv.second);
    }
    check(sf_sim_run_kernel(h_.get(), name.c_str(), n.data(), v.data(), (int)n.size(), (int)reg));
  }
  double reduce(const std::string& field, grid::reduce_op op) {
    double v = 0.0;
    check(sf_sim_reduce(h_.get(), field.c_str(), (int)op, &v));
    return v;
  }

  // grid::gather / grid::scatter (io.hpp:25-65) and cli::field_checksum (bench.hpp:24-39)
  std::vector<double> gather(const std::string& field) {
    std::vector<double> g((size_t)cfg_.dom.cells());
    check(sf_sim_gather(h_.get(), field.c_str(), g.data(), (int64_t)g.size()));
    return g;
  }
  void scatter(const std::string& field, const std::vector<double>& g) {
    check(sf_sim_scatter(h_.get(), field.c_str(), g.data(), (int64_t)g.size()));
  }
  std::uint64_t checksum() {
    std::uint64_t h = 0;
    check(sf_sim_checksum(h_.get(), &h));
    return h;
  }
  // one grid component's owned block as a dense x-fastest host array
  // (sf_sim_*_block*): synchronous, asynchronous (pinned host memory, valid
  // until synchronize()), and the staged upload (stage now, install in stream
  // order before the step that consumes it)
  void gather_block(const std::string& field, int worker, double* host, int64_t n) {
    check(sf_sim_gather_block(h_.get(), field.c_str(), worker, host, n));
  }
  void scatter_block(const std::string& field, int worker, const double* host, int64_t n) {
    check(sf_sim_scatter_block(h_.get(), field.c_str(), worker, host, n));
  }
  void gather_block_async(const std::string& field, int worker, double* host, int64_t n) {
    check(sf_sim_gather_block_async(h_.get(), field.c_str(), worker, host, n));
  }
  void scatter_block_async(const std::string& field, int worker, const double* host, int64_t n) {
    check(sf_sim_scatter_block_async(h_.get(), field.c_str(), worker, host, n));
  }
  void stage_block_async(const std::string& field, int worker, const double* host, int64_t n) {
    check(sf_sim_stage_block_async(h_.get(), field.c_str(), worker, host, n));
  }
  void install_staged(const std::string& field, int worker) {
    check(sf_sim_install_staged(h_.get(), field.c_str(), worker));
  }
  void synchronize() { check(sf_sim_synchronize(h_.get())); }
  sf_sim* handle() { return h_.get(); }

 private:
  struct del {
    void operator()(sf_sim* s) const { sf_sim_destroy(s); }
  };
  solver_config cfg_;
  fluid_params par_;
  std::unique_ptr<sf_sim, del> h_;
};

}  // namespace cfd
}  // namespace sforge_b200
