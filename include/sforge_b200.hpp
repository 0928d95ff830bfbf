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
enum class stagger : int { none = -1, x = 0, y = 1, z = 2 };  // field.hpp:23

struct face_bc {  // exchange.hpp:18-26
  enum class kind { unset = SF_BC_UNSET, wall = SF_BC_WALL, symmetry = SF_BC_SYMMETRY, outflow = SF_BC_OUTFLOW };
  kind k = kind::unset;
  std::array<double, 3> velocity{};
  static face_bc wall(std::array<double, 3> v = {0, 0, 0}) { return {kind::wall, v}; }
  static face_bc symmetry() { return {kind::symmetry, {}}; }
  static face_bc outflow() { return {kind::outflow, {}}; }
};
struct boundary_spec {  // exchange.hpp:30-42
  std::array<face_bc, 6> faces{};
  face_bc& at(int axis, int side) { return faces[static_cast<std::size_t>(2 * axis + side)]; }
  const face_bc& at(int axis, int side) const { return faces[static_cast<std::size_t>(2 * axis + side)]; }
  static boundary_spec uniform(face_bc fb) {
    boundary_spec b;
    b.faces.fill(fb);
    return b;
  }
};
}  // namespace grid

namespace ccl {
enum class intent { in = 0, out = 1, inout = 2, separate_inout = 3 };  // descriptor.hpp:216
}  // namespace ccl

namespace codegen {  // codegen.hpp:30-57
enum class template_id { threedblock };
struct binding {
  std::string field;
  ccl::intent io = ccl::intent::in;
  bool cached = false;
};
struct execution_plan {
  std::string kernel;
  template_id tmpl = template_id::threedblock;
  std::array<int, 3> tile{};
  std::array<int, 6> halo{};
  std::vector<binding> bindings;
  std::vector<std::string> parameters;
  int halo_lo(int axis) const { return halo[static_cast<std::size_t>(2 * axis)]; }
  int halo_hi(int axis) const { return halo[static_cast<std::size_t>(2 * axis + 1)]; }
  int max_halo() const {
    int m = 0;
    for (int h : halo) m = m < h ? h : m;
    return m;
  }
};
}  // namespace codegen

namespace exec {
struct exec_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
enum class region { all = SF_REGION_ALL, interior = SF_REGION_INTERIOR, boundary = SF_REGION_BOUNDARY };
enum class run_mode { plain = 0, overlap = 1 };
struct kernel_signature {  // executor.hpp:46-49
  std::vector<std::string> fields;
  std::vector<std::string> params;
};
// A point function for the device, given as the CUDA C++ text of the body of
// the reference's F(const point_ctx& c) (executor.hpp:130-184): c.field(s)(di,
// dj, dk), c.field(s).load(), c.field(s).store(v), c.param(s), c.i / c.j /
// c.k.  register_kernel JIT-compiles it for sm_100a (--fmad=false).
struct device_function {
  std::string body;
};
}  // namespace exec

// A point function usable by BOTH executors: SF_POINT_FUNCTION(NAME, body)
// defines a functor type whose templated operator() is the body (the
// reference's executor::register_kernel calls it with its point_ctx) and
// whose source() is the body's text (this executor::register_kernel compiles
// it for the device).  The body must be plain C++ over `c` without
// preprocessor directives or line comments.
#define SF_POINT_FUNCTION(NAME, ...)                                \
  struct NAME {                                                     \
    template <class Ctx>                                            \
    void operator()(const Ctx& c) const {                           \
      __VA_ARGS__                                                   \
    }                                                               \
    static const char* source() { return #__VA_ARGS__; }            \
  }

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

namespace exec {
struct schedule_step {  // executor.hpp:422-466
  enum class kind { run = 0, exchange = 1, physical_bc = 2, refresh = 3, reduce = 4 };
  kind what = kind::run;
  std::string kernel;
  region reg = region::all;
  std::vector<std::string> fields;
  grid::reduce_op op = grid::reduce_op::max_abs;
  std::string source;
  std::string target;
  static schedule_step run(std::string kernel, region r = region::all) {
    schedule_step s;
    s.what = kind::run;
    s.kernel = std::move(kernel);
    s.reg = r;
    return s;
  }
  static schedule_step exchange(std::vector<std::string> fields) {
    schedule_step s;
    s.what = kind::exchange;
    s.fields = std::move(fields);
    return s;
  }
  static schedule_step physical_bc(std::vector<std::string> fields) {
    schedule_step s;
    s.what = kind::physical_bc;
    s.fields = std::move(fields);
    return s;
  }
  static schedule_step refresh(std::vector<std::string> fields) {
    schedule_step s;
    s.what = kind::refresh;
    s.fields = std::move(fields);
    return s;
  }
  static schedule_step reduce(std::string source, grid::reduce_op op, std::string target) {
    schedule_step s;
    s.what = kind::reduce;
    s.source = std::move(source);
    s.op = op;
    s.target = std::move(target);
    return s;
  }
};
struct schedule {
  std::vector<schedule_step> steps;
};

// exec::executor (executor.hpp:477-862) over device-resident distributed
// fields: the grid components of grid::decompose(dom, workers, ghost,
// periodic) live on one device; fields, exchanges, physical boundary
// conditions, kernels, reductions, schedules and ghost validity keep the
// reference's semantics and error texts.  The reference builds the executor
// over its worker_group and field_store; here the constructor takes the
// decomposition's inputs and owns the store.
class executor {
 public:
  executor(const grid::domain& dom, int workers, int ghost, std::array<bool, 3> periodic,
           grid::boundary_spec bc = {}, int device = 0) {
    sf_solver_config c{};
    for (int a = 0; a < 3; ++a) {
      c.extents[a] = dom.extents[a];
      c.spacing[a] = dom.spacing[a];
      c.origin[a] = dom.origin[a];
      c.periodic[a] = periodic[a] ? 1 : 0;
    }
    c.reynolds = 100.0;
    c.sigma = 0.5;
    c.tolerance = 1e-6;
    c.omega = 1.7;
    c.max_sweeps = 1;
    c.symmetry_z = 0;
    sf_fluid_params p{};
    p.viscosity = 0.01;
    p.density = 1.0;
    sf_sim_options o;
    sf_sim_options_default(&o);
    o.workers = workers;
    o.ghost = ghost < 1 ? 1 : ghost;  // the device store always carries the CFD kernels' one layer
    o.device = device;
    sf_sim* h = nullptr;
    cfd::check(sf_sim_create(&c, &p, &o, &h));
    h_.reset(h);
    set_boundary(bc);
  }

  // executor::boundary() (executor.hpp:482): replace the face conditions
  void set_boundary(const grid::boundary_spec& bc) {
    bc_ = bc;
    for (int axis = 0; axis < 3; ++axis)
      for (int side = 0; side < 2; ++side) {
        const grid::face_bc& f = bc.at(axis, side);
        cfd::check(sf_sim_set_face_bc(h_.get(), axis, side, (int)f.k, f.velocity.data()));
      }
  }
  const grid::boundary_spec& boundary() const { return bc_; }

  // field_store::create (field.hpp:108-112); fp32 = false keeps fp64 storage
  void create_field(const std::string& name, grid::stagger st, bool fp32 = false) {
    cfd::check(sf_sim_create_field_typed(h_.get(), name.c_str(), (int)st, fp32 ? 4 : 8));
  }

  // executor::register_kernel (executor.hpp:484-488) with a device function
  void register_kernel(const codegen::execution_plan& plan, const kernel_signature& sig, const device_function& fn) {
    std::vector<sf_binding> b;
    for (const auto& x : plan.bindings) b.push_back({x.field.c_str(), (int)x.io, x.cached ? 1 : 0});
    std::vector<const char*> pn, sf, sp;
    for (const auto& x : plan.parameters) pn.push_back(x.c_str());
    for (const auto& x : sig.fields) sf.push_back(x.c_str());
    for (const auto& x : sig.params) sp.push_back(x.c_str());
    sf_plan cp{};
    cp.kernel = plan.kernel.c_str();
    for (int a = 0; a < 3; ++a) cp.tile[a] = plan.tile[a];
    for (int a = 0; a < 6; ++a) cp.halo[a] = plan.halo[a];
    cp.bindings = b.data();
    cp.n_bindings = (int)b.size();
    cp.params = pn.data();
    cp.n_params = (int)pn.size();
    cfd::check(sf_sim_register_kernel(h_.get(), &cp, sf.data(), (int)sf.size(), sp.data(), (int)sp.size(),
                                      fn.body.c_str()));
  }
  // ... or with an SF_POINT_FUNCTION functor (the reference's F: void(const point_ctx&))
  template <class F, class = decltype(F::source())>
  void register_kernel(const codegen::execution_plan& plan, const kernel_signature& sig, F) {
    register_kernel(plan, sig, device_function{F::source()});
  }

  void run_kernel(const std::string& name, const std::map<std::string, double>& params, region reg = region::all) {
    std::vector<const char*> n;
    std::vector<double> v;
    for (auto& kv : params) {
      n.push_back(kv.first.c_str());
      v.push_back(kv.second);
    }
    cfd::check(sf_sim_run_kernel(h_.get(), name.c_str(), n.data(), v.data(), (int)n.size(), (int)reg));
  }
  void exchange(const std::vector<std::string>& fields) { fields_call(sf_sim_exchange, fields); }
  void physical_bc(const std::vector<std::string>& fields) { fields_call(sf_sim_physical_bc, fields); }
  void refresh(const std::vector<std::string>& fields) { fields_call(sf_sim_refresh, fields); }
  double reduce(const std::string& field, grid::reduce_op op) {
    double v = 0.0;
    cfd::check(sf_sim_reduce(h_.get(), field.c_str(), (int)op, &v));
    return v;
  }

  // executor::run_schedule (executor.hpp:533-553): dry run, then `steps` passes
  void run_schedule(const schedule& s, const std::map<std::string, double>& params, int steps,
                    run_mode mode = run_mode::plain, std::map<std::string, double>* results = nullptr) {
    std::vector<sf_schedule_step> cs;
    std::vector<std::vector<const char*>> keep;
    keep.reserve(s.steps.size());
    for (const auto& st : s.steps) {
      keep.emplace_back();
      for (const auto& f : st.fields) keep.back().push_back(f.c_str());
      sf_schedule_step c{};
      c.kind = (int)st.what;
      c.kernel = st.kernel.c_str();
      c.region = (int)st.reg;
      c.fields = keep.back().data();
      c.n_fields = (int)keep.back().size();
      c.source = st.source.c_str();
      c.op = (int)st.op;
      c.target = st.target.c_str();
      cs.push_back(c);
    }
    std::vector<const char*> n;
    std::vector<double> v;
    for (auto& kv : params) {
      n.push_back(kv.first.c_str());
      v.push_back(kv.second);
    }
    cfd::check(sf_sim_run_schedule(h_.get(), cs.data(), (int)cs.size(), n.data(), v.data(), (int)n.size(), steps,
                                   (int)mode));
    if (results)
      for (const auto& st : s.steps)
        if (st.what == schedule_step::kind::reduce) {
          double r = 0.0;
          cfd::check(sf_sim_result(h_.get(), st.target.c_str(), &r));
          (*results)[st.target] = r;
        }
  }

  // ghost validity (executor.hpp:610-613)
  bool ghosts_valid(const std::string& field) const { return sf_sim_ghosts_valid(h_.get(), field.c_str()) == 1; }
  void invalidate_ghosts(const std::string& field) { cfd::check(sf_sim_invalidate_ghosts(h_.get(), field.c_str())); }
  void invalidate_all_ghosts() { cfd::check(sf_sim_invalidate_all_ghosts(h_.get())); }

  // grid::gather / grid::scatter (io.hpp:25-65) of a field of this store
  std::vector<double> gather(const std::string& field, grid::index_t cells) {
    std::vector<double> g((size_t)cells);
    cfd::check(sf_sim_gather(h_.get(), field.c_str(), g.data(), (int64_t)g.size()));
    return g;
  }
  void scatter(const std::string& field, const std::vector<double>& g) {
    cfd::check(sf_sim_scatter(h_.get(), field.c_str(), g.data(), (int64_t)g.size()));
  }
  sf_sim* handle() { return h_.get(); }

 private:
  template <class Fn>
  void fields_call(Fn fn, const std::vector<std::string>& fields) {
    std::vector<const char*> f;
    for (auto& x : fields) f.push_back(x.c_str());
    cfd::check(fn(h_.get(), f.data(), (int)f.size()));
  }
  struct del {
    void operator()(sf_sim* s) const { sf_sim_destroy(s); }
  };
  grid::boundary_spec bc_;
  std::unique_ptr<sf_sim, del> h_;
};
}  // namespace exec
}  // namespace sforge_b200
