// executor_functors.cpp -- the same point functors through two executors.
//
// Built twice from this one file:
//   -DSF_REF   against the reference headers (proj/include/stencilforge), by
//              oracle/Makefile into oracle/_ref/executor_functors_ref: the
//              reference's exec::executor on its CPU worker threads is the
//              oracle ("the same functor can run through the
//              reference executor as its own oracle");
//   (default)  against include/sforge_b200.hpp + libsfb200.so: the device
//              executor, each functor JIT-compiled from its own source text.
// Each case mirrors a case of the reference's tests/test_executor.cpp; both
// programs write every gathered field and every reduce result to a binary
// file that tests/test_gpu_executor_cpp.py compares (fp64 bitwise; sums to
// rounding, as the reduction order differs).
#include <array>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "sforge_b200.hpp"  // SF_POINT_FUNCTION (and, without SF_REF, the device executor)

#ifdef SF_REF
#include "stencilforge/executor.hpp"
#include "stencilforge/io.hpp"
namespace S = sforge;
#else
namespace S = sforge_b200;
#endif

using idx = std::int64_t;

// ---- the point functions (plain C++ over `c`, valid for both executors) -------
SF_POINT_FUNCTION(Ident, c.field(1).store(c.field(0).load()););
SF_POINT_FUNCTION(Smooth, const auto& f = c.field(0);
                  c.field(1).store(((f(-1, 0, 0) + f(1, 0, 0)) + (f(0, -1, 0) + f(0, 1, 0))) +
                                   ((f(0, 0, -1) + f(0, 0, 1)) - 6.0 * f.load())););
SF_POINT_FUNCTION(Asym, const auto& f = c.field(0);
                  c.field(0).store(f(-2, 0, 0) + f(1, 0, 0) + f(0, 2, 0) + f(0, 0, -1) + f(0, 0, 1)););
SF_POINT_FUNCTION(ScaleShift, c.field(0).store(c.field(0).load() * c.param(0) + c.param(1)););
SF_POINT_FUNCTION(GlobalIndex, c.field(0).store(double(c.i) + 1000.0 * double(c.j) + 1000000.0 * double(c.k)););
SF_POINT_FUNCTION(Blend, const auto& u = c.field(0); const auto& v = c.field(1);
                  c.field(2).store(c.param(0) * (u(1, 0, 0) - u(-1, 0, 0)) + (1.0 - c.param(0)) * (v(0, 1, 0) - v(0, -1, 0))););

// ---- a rig per executor ----------------------------------------------------------
S::grid::domain unit_domain(idx nx, idx ny, idx nz) {
  return {{nx, ny, nz}, {1.0 / double(nx), 1.0 / double(ny), 1.0 / double(nz)}, {0.0, 0.0, 0.0}};
}

S::codegen::execution_plan make_plan(std::string name, std::array<int, 3> tile, std::array<int, 6> halo,
                                     std::vector<S::codegen::binding> binds, std::vector<std::string> params = {}) {
  S::codegen::execution_plan p;
  p.kernel = std::move(name);
  p.tile = tile;
  p.halo = halo;
  p.bindings = std::move(binds);
  p.parameters = std::move(params);
  return p;
}

#ifdef SF_REF
struct rig {
  S::grid::decomposition d;
  S::grid::worker_group g;
  S::grid::field_store store;
  S::exec::executor ex;
  rig(S::grid::domain dom, int workers, int ghost, std::array<bool, 3> periodic, S::grid::boundary_spec bc)
      : d(S::grid::decompose(dom, workers, ghost, periodic)), g(workers), store(d), ex(g, store, bc) {}
  void create(const std::string& n, S::grid::stagger s) { store.create(n, s); }
  void scatter(const std::string& n, const std::vector<double>& v) { S::grid::scatter(g, store.at(n), v); }
  std::vector<double> gather(const std::string& n) { return S::grid::gather(g, store.at(n)); }
};
#else
struct rig {
  idx cells;
  S::exec::executor ex;
  rig(S::grid::domain dom, int workers, int ghost, std::array<bool, 3> periodic, S::grid::boundary_spec bc)
      : cells(dom.cells()), ex(dom, workers, ghost, periodic, bc) {}
  void create(const std::string& n, S::grid::stagger s) { ex.create_field(n, s); }
  void scatter(const std::string& n, const std::vector<double>& v) { ex.scatter(n, v); }
  std::vector<double> gather(const std::string& n) { return ex.gather(n, cells); }
};
#endif

std::vector<double> random_global(const S::grid::domain& dom, unsigned seed) {
  std::vector<double> v((size_t)dom.cells());
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (auto& x : v) x = u(rng);
  return v;
}

// ---- output: records of (name, n doubles) -----------------------------------------
FILE* out_file = nullptr;
void emit(const std::string& name, const std::vector<double>& v) {
  const int nl = (int)name.size();
  const long long n = (long long)v.size();
  std::fwrite(&nl, sizeof nl, 1, out_file);
  std::fwrite(name.data(), 1, name.size(), out_file);
  std::fwrite(&n, sizeof n, 1, out_file);
  std::fwrite(v.data(), sizeof(double), v.size(), out_file);
}

using S::ccl::intent;
using S::grid::stagger;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s out.bin\n", argv[0]);
    return 2;
  }
  out_file = std::fopen(argv[1], "wb");
  // test_executor.cpp:68-81 identity
  {
    rig r(unit_domain(8, 6, 5), 2, 1, {false, false, false}, {});
    r.create("in", stagger::none);
    r.create("out", stagger::none);
    r.scatter("in", random_global(unit_domain(8, 6, 5), 1));
    r.ex.register_kernel(make_plan("IDENT", {4, 4, 4}, {0, 0, 0, 0, 0, 0},
                                   {{"in", intent::in, false}, {"out", intent::out, false}}),
                         {{"in", "out"}, {}}, Ident{});
    r.ex.run_kernel("IDENT", {});
    emit("ident", r.gather("out"));
  }
  // test_executor.cpp:150-194 tiling, caching and worker count (periodic)
  {
    struct variant {
      std::array<int, 3> tile;
      bool cached;
      int workers;
    };
    int q = 0;
    for (const variant& v : {variant{{16, 16, 16}, true, 1}, variant{{4, 4, 4}, true, 1}, variant{{5, 3, 7}, true, 4},
                             variant{{1, 1, 1}, false, 2}, variant{{16, 16, 16}, false, 4},
                             variant{{12, 12, 12}, true, 8}, variant{{32, 8, 4}, true, 2}}) {
      auto dom = unit_domain(12, 12, 12);
      rig r(dom, v.workers, 1, {true, true, true}, {});
      r.create("src", stagger::none);
      r.create("dst", stagger::none);
      r.scatter("src", random_global(dom, 2));
      r.ex.register_kernel(make_plan("SMOOTH", v.tile, {1, 1, 1, 1, 1, 1},
                                     {{"src", intent::in, v.cached}, {"dst", intent::out, v.cached}}),
                           {{"src", "dst"}, {}}, Smooth{});
      r.ex.exchange({"src"});
      r.ex.run_kernel("SMOOTH", {});
      emit("smooth" + std::to_string(q++), r.gather("dst"));
    }
  }
  // test_executor.cpp:682-695 asymmetric halo, separate in/out, 2-deep ghosts
  for (int workers : {1, 2}) {
    auto dom = unit_domain(8, 6, 6);
    rig r(dom, workers, 2, {true, true, true}, {});
    r.create("v", stagger::none);
    r.scatter("v", random_global(dom, 9));
    r.ex.register_kernel(make_plan("ASYM", {4, 4, 4}, {2, 1, 0, 2, 1, 1}, {{"v", intent::separate_inout, true}}),
                         {{"v"}, {}}, Asym{});
    for (int pass = 0; pass < 2; ++pass) {
      r.ex.exchange({"v"});
      r.ex.run_kernel("ASYM", {});
    }
    emit("asym_w" + std::to_string(workers), r.gather("v"));
  }
  // parameters by slot on an in-place binding, regions interior then boundary
  {
    auto dom = unit_domain(9, 7, 5);
    rig r(dom, 2, 1, {false, false, false}, S::grid::boundary_spec::uniform(S::grid::face_bc::outflow()));
    r.create("a", stagger::none);
    r.scatter("a", random_global(dom, 4));
    r.ex.register_kernel(make_plan("SCALE", {4, 4, 4}, {0, 0, 0, 0, 0, 0}, {{"a", intent::inout, false}},
                                   {"k", "b"}),
                         {{"a"}, {"k", "b"}}, ScaleShift{});
    r.ex.run_kernel("SCALE", {{"k", 2.5}, {"b", -0.75}}, S::exec::region::interior);
    r.ex.run_kernel("SCALE", {{"k", -1.25}, {"b", 0.5}}, S::exec::region::boundary);
    emit("scale", r.gather("a"));
    r.create("gi", stagger::none);
    r.ex.register_kernel(make_plan("GIDX", {3, 2, 5}, {0, 0, 0, 0, 0, 0}, {{"gi", intent::out, false}}), {{"gi"}, {}},
                         GlobalIndex{});
    r.ex.run_kernel("GIDX", {});
    emit("gidx", r.gather("gi"));
  }
  // physical boundary conditions (moving wall, symmetry, outflow) under
  // staggered fields, read through a halo kernel after refresh; then a
  // schedule with reductions, plain and overlap
  for (int mode = 0; mode < 2; ++mode)
    for (int workers : {1, 3}) {
      auto dom = unit_domain(11, 9, 7);
      S::grid::boundary_spec bc;
      bc.at(0, 0) = S::grid::face_bc::wall();
      bc.at(0, 1) = S::grid::face_bc::outflow();
      bc.at(1, 0) = S::grid::face_bc::symmetry();
      bc.at(1, 1) = S::grid::face_bc::wall({0.7, -0.2, 0.3});
      rig r(dom, workers, 1, {false, false, true}, bc);
      r.create("u", stagger::x);
      r.create("v", stagger::y);
      r.create("w", stagger::none);
      r.scatter("u", random_global(dom, 5));
      r.scatter("v", random_global(dom, 6));
      r.ex.register_kernel(make_plan("BLEND", {8, 4, 2}, {1, 1, 1, 1, 0, 0},
                                     {{"u", intent::in, true}, {"v", intent::in, false}, {"w", intent::out, false}},
                                     {"t"}),
                           {{"u", "v", "w"}, {"t"}}, Blend{});
      S::exec::schedule s;
      s.steps.push_back(S::exec::schedule_step::refresh({"u", "v"}));
      s.steps.push_back(S::exec::schedule_step::run("BLEND"));
      s.steps.push_back(S::exec::schedule_step::reduce("w", S::grid::reduce_op::max_abs, "wmax"));
      s.steps.push_back(S::exec::schedule_step::reduce("w", S::grid::reduce_op::sum, "wsum"));
      std::map<std::string, double> res;
      r.ex.run_schedule(s, {{"t", 0.375}}, 2, mode ? S::exec::run_mode::overlap : S::exec::run_mode::plain, &res);
      const std::string tag = "_m" + std::to_string(mode) + "_w" + std::to_string(workers);
      emit("blend" + tag, r.gather("w"));
      emit("wmax" + tag, {res["wmax"]});
      emit("wsum~" + tag, {res["wsum"]});
    }
  std::fclose(out_file);
  return 0;
}
