// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A C-ABI shim over the UNMODIFIED reference implementation (stencilforge,
// header-only C++20 under /root/reference/proj/include), compiled in place by
// oracle/Makefile into oracle/_ref/libsfref.so.  Only tests/, the
// __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
// legs load it.  Nothing here is copied from the reference: every call below
// goes straight into the reference's own public API:
//   cfd::simulation            proj/include/stencilforge/cfd.hpp:173-766
//   grid::scatter / gather     proj/include/stencilforge/io.hpp:25-65
//   cli::field_checksum        proj/include/stencilforge/bench.hpp:24-39
//   exec::executor             proj/include/stencilforge/executor.hpp:477-862
//   grid::reduce               proj/include/stencilforge/reductions.hpp:28-90
//   ccl::parse_descriptors / render / validate_all   descriptor.hpp:148-381
//   codegen::render_header / write_generated         codegen.hpp:86-163
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "stencilforge/bench.hpp"
#include "stencilforge/cfd.hpp"
#include "stencilforge/codegen.hpp"
#include "stencilforge/config.hpp"
#include "stencilforge/descriptor.hpp"
#include "stencilforge/io.hpp"

using namespace sforge;

namespace {

thread_local std::string g_err;

struct handle {
  std::unique_ptr<cfd::simulation> sim;
};

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

std::vector<std::string> split_csv(const char* s) {
  std::vector<std::string> out;
  std::string cur;
  for (const char* p = s; *p; ++p) {
    if (*p == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += *p;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

}  // namespace

extern "C" {

// Mirrors the flat parameter set of cfd::solver_config + cfd::fluid_params
// (cfd.hpp:29-67).
struct sfref_params {
  int64_t extents[3];
  double spacing[3];
  int periodic[3];
  double reynolds, sigma, tolerance, omega;
  int max_sweeps;
  int symmetry_z;
  double viscosity, density;
  double body_force[3];
  double lid_speed, blend;
  int workers, mode;  // mode: 0 plain, 1 overlap
  int tile[3];
  int ghost;
  int form;  // 0 rows, 1 points
};

const char* sfref_last_error(void) { return g_err.c_str(); }

void* sfref_create(const sfref_params* p) {
  try {
    cfd::solver_config cfg;
    for (int a = 0; a < 3; ++a) {
      cfg.dom.extents[a] = p->extents[a];
      cfg.dom.spacing[a] = p->spacing[a];
      cfg.periodic[a] = p->periodic[a] != 0;
    }
    cfg.reynolds = p->reynolds;
    cfg.sigma = p->sigma;
    cfg.tolerance = p->tolerance;
    cfg.omega = p->omega;
    cfg.max_sweeps = p->max_sweeps;
    cfg.symmetry_z = p->symmetry_z != 0;
    cfd::fluid_params par;
    par.viscosity = p->viscosity;
    par.density = p->density;
    par.body_force = {p->body_force[0], p->body_force[1], p->body_force[2]};
    par.lid_speed = p->lid_speed;
    par.blend = p->blend;
    auto h = std::make_unique<handle>();
    h->sim = std::make_unique<cfd::simulation>(
        cfg, par, p->workers, p->mode ? exec::run_mode::overlap : exec::run_mode::plain,
        std::array<int, 3>{p->tile[0], p->tile[1], p->tile[2]}, p->ghost,
        p->form ? cfd::kernel_form::points : cfd::kernel_form::rows);
    return h.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void sfref_destroy(void* h) { delete static_cast<handle*>(h); }

static cfd::simulation& S(void* h) { return *static_cast<handle*>(h)->sim; }

int sfref_init_cavity(void* h) {
  try { S(h).init_cavity(); return 0; } catch (const std::exception& e) { return fail(e); }
}
int sfref_init_uniform(void* h, double cx, double cy, double cz) {
  try { S(h).init_uniform({cx, cy, cz}); return 0; } catch (const std::exception& e) { return fail(e); }
}
int sfref_init_taylor_green(void* h) {
  try { S(h).init_taylor_green(); return 0; } catch (const std::exception& e) { return fail(e); }
}

int sfref_scatter(void* h, const char* field, const double* global, int64_t n) {
  try {
    std::vector<double> g(global, global + n);
    grid::scatter(S(h).group(), S(h).store().at(field), g);
    S(h).engine().invalidate_ghosts(field);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int sfref_gather(void* h, const char* field, double* out) {
  try {
    auto g = grid::gather(S(h).group(), S(h).store().at(field));
    std::memcpy(out, g.data(), g.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Copies worker w's whole padded front array (ghosts included), x fastest,
// extents ld = dims + 2g (field.hpp:31-52).
int sfref_local_front(void* h, const char* field, int w, double* out, int64_t* dims, int64_t* lo) {
  try {
    const auto& lb = S(h).store().at(field).local(w);
    for (int a = 0; a < 3; ++a) {
      dims[a] = lb.dims[a];
      lo[a] = lb.lo[a];
    }
    std::memcpy(out, lb.front, static_cast<std::size_t>(lb.padded_cells()) * sizeof(double));
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int sfref_compute_dt(void* h, double* dt) {
  try { *dt = S(h).compute_dt(); return 0; } catch (const std::exception& e) { return fail(e); }
}
int sfref_provisional(void* h, double dt) {
  try { S(h).provisional(dt); return 0; } catch (const std::exception& e) { return fail(e); }
}
int sfref_pressure_iteration(void* h, double dt, int* sweeps, double* residual) {
  try {
    auto r = S(h).pressure_iteration(dt);
    *sweeps = r.first;
    *residual = r.second;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
int sfref_step(void* h, double* dt, int* sweeps, double* residual) {
  try {
    auto st = S(h).step();
    *dt = st.dt;
    *sweeps = st.sweeps;
    *residual = st.residual;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
// Runs n steps, writing per-step stats when the arrays are non-null.
int sfref_advance(void* h, int n, double* dts, int* sweeps, double* residuals) {
  try {
    for (int i = 0; i < n; ++i) {
      auto st = S(h).step();
      if (dts) dts[i] = st.dt;
      if (sweeps) sweeps[i] = st.sweeps;
      if (residuals) residuals[i] = st.residual;
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

uint64_t sfref_checksum(void* h) { return cli::field_checksum(S(h)); }

double sfref_time(void* h) { return S(h).time(); }
long sfref_step_count(void* h) { return S(h).step_count(); }
int sfref_pending_color(void* h) { return S(h).pending_color(); }

int sfref_reduce(void* h, const char* field, int op, double* out) {
  try {
    *out = S(h).engine().reduce(field, static_cast<grid::reduce_op>(op));
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int sfref_refresh(void* h, const char* fields_csv) {
  try { S(h).engine().refresh(split_csv(fields_csv)); return 0; } catch (const std::exception& e) { return fail(e); }
}
int sfref_exchange(void* h, const char* fields_csv) {
  try { S(h).engine().exchange(split_csv(fields_csv)); return 0; } catch (const std::exception& e) { return fail(e); }
}

// params: "name=value" pairs, comma separated, e.g. "beta=0.1,color=0"
int sfref_run_kernel(void* h, const char* name, const char* params_csv, int region) {
  try {
    std::map<std::string, double> pm;
    for (const auto& kv : split_csv(params_csv)) {
      auto eq = kv.find('=');
      pm[kv.substr(0, eq)] = std::stod(kv.substr(eq + 1));
    }
    S(h).engine().run_kernel(name, pm, static_cast<exec::region>(region));
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

void sfref_invalidate_all_ghosts(void* h) { S(h).engine().invalidate_all_ghosts(); }

int sfref_diag(void* h, double* max_div, double* steady_delta, double* kinetic) {
  try {
    if (steady_delta) *steady_delta = S(h).steady_delta();
    if (kinetic) *kinetic = S(h).kinetic_energy();
    if (max_div) *max_div = S(h).max_divergence();
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int sfref_taylor_green_error(void* h, double t, double* out) {
  try { *out = S(h).taylor_green_error(t); return 0; } catch (const std::exception& e) { return fail(e); }
}

// Descriptor front end. Results are text written to out (cap bytes); the
// return code says which stage failed: 0 ok, 1 parse_error, 2
// descriptor_error, 3 other, 4 buffer too small; g_err holds the message.
static int put(const std::string& r, char* out, size_t cap) {
  if (r.size() + 1 > cap) return 4;
  std::memcpy(out, r.c_str(), r.size() + 1);
  return 0;
}
int sfref_ccl_render(const char* text, char* out, size_t cap) {
  try {
    return put(ccl::render(ccl::parse_descriptors(text)), out, cap);
  } catch (const ccl::parse_error& e) { g_err = e.what(); return 1;
  } catch (const std::exception& e) { g_err = e.what(); return 3; }
}
// headers of every kernel (concatenated) followed by the plans.txt manifest
int sfref_ccl_generate(const char* text, const char* fields_csv, const char* dir, char* out, size_t cap) {
  try {
    const auto v = split_csv(fields_csv);
    const auto ks = ccl::validate_all(ccl::parse_descriptors(text), std::set<std::string>(v.begin(), v.end()));
    std::string r;
    for (const auto& k : ks) r += codegen::render_header(k, codegen::build_plan(k).tmpl).text;
    codegen::write_generated(ks, dir);
    return put(r, out, cap);
  } catch (const ccl::parse_error& e) { g_err = e.what(); return 1;
  } catch (const ccl::descriptor_error& e) { g_err = e.what(); return 2;
  } catch (const std::exception& e) { g_err = e.what(); return 3; }
}

// cli::parse_run_config on text: every field as key=value lines (%.17g for
// reals); 1 config_error, 2 cfd_error (the cross-field validate), 3 other.
int sfref_parse_config(const char* text, char* out, size_t cap) {
  try {
    std::istringstream in(text);
    const cli::run_config rc = cli::parse_run_config(in);
    char b[2048];
    std::snprintf(b, sizeof b,
                  "nx=%ld\nny=%ld\nnz=%ld\nre=%.17g\nsigma=%.17g\nomega=%.17g\ntolerance=%.17g\nmax_sweeps=%ld\n"
                  "alpha=%.17g\ndensity=%.17g\nlid_speed=%.17g\nsymmetry_z=%d\nsteady_tol=%.17g\nmax_steps=%ld\n"
                  "output_cadence=%ld\nworkers=%d\nmode=%s\ntile=%d,%d,%d\nghost=%d\n",
                  rc.nx, rc.ny, rc.nz, rc.re, rc.sigma, rc.omega, rc.tolerance, rc.max_sweeps, rc.alpha, rc.density,
                  rc.lid_speed, rc.symmetry_z ? 1 : 0, rc.steady_tol, rc.max_steps, rc.output_cadence, rc.workers,
                  rc.mode == exec::run_mode::plain ? "plain" : "overlap", rc.tile[0], rc.tile[1], rc.tile[2],
                  rc.ghost);
    return put(std::string(b) + "profiles_out=" + rc.profiles_out + "\nresiduals_out=" + rc.residuals_out +
                   "\nfields_out=" + rc.fields_out + "\n",
               out, cap);
  } catch (const cli::config_error& e) { g_err = e.what(); return 1;
  } catch (const cfd::cfd_error& e) { g_err = e.what(); return 2;
  } catch (const std::exception& e) { g_err = e.what(); return 3; }
}

// Bounded-sample timing probe for the CPU baseline:
// wall seconds of compute_dt+provisional and of one pressure_iteration with
// the configured max_sweeps, on this simulation's worker team.
int sfref_time_phases(void* h, double* t_prov, double* t_iter, int* sweeps) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    const double dt = S(h).compute_dt();
    S(h).provisional(dt);
    auto t1 = std::chrono::steady_clock::now();
    auto r = S(h).pressure_iteration(dt);
    auto t2 = std::chrono::steady_clock::now();
    *t_prov = std::chrono::duration<double>(t1 - t0).count();
    *t_iter = std::chrono::duration<double>(t2 - t1).count();
    *sweeps = r.first;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// One half-sweep of pressure_iteration's loop body (cfd.hpp:295-303) through
// the reference's own executor API, k times: refresh(divu), PRESSURE_SWEEP,
// refresh(vx,vy,vz), DIVERGENCE, reduce(divu, max_abs).  Wall seconds.
int sfref_time_half_sweeps(void* h, int k, double beta, double* seconds) {
  try {
    auto& e = S(h).engine();
    auto t0 = std::chrono::steady_clock::now();
    int color = 0;
    for (int q = 0; q < k; ++q) {
      e.refresh({"divu"});
      e.run_kernel("PRESSURE_SWEEP", {{"beta", beta}, {"color", static_cast<double>(color)}});
      color ^= 1;
      e.refresh({"vx", "vy", "vz"});
      e.run_kernel("DIVERGENCE", {});
      (void)e.reduce("divu", grid::reduce_op::max_abs);
    }
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// compute_dt + provisional (cfd.hpp:264-282) through the reference, wall seconds.
int sfref_time_provisional(void* h, double* seconds, double* dt_out) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    const double dt = S(h).compute_dt();
    S(h).provisional(dt);
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    *dt_out = dt;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

}  // extern "C"
