// sf_driver.cu -- C++ host driver + C ABI (include/sforge_b200.h).
//
// Mirrors the reference's host side on the hot path:
//   grid::decompose / decomposition        grid.hpp:44-163
//   grid::boundary_spec / face_bc          exchange.hpp:18-42
//   exchanger::refresh (3 axis phases)     exchange.hpp:98-119, 165-480
//   exec::executor run_kernel / refresh /  executor.hpp:477-862
//     reduce / ghost validity
//   cfd::simulation step loop              cfd.hpp:173-766
// One simulation owns every grid component ("worker") of its decomposition on
// one CUDA device; all work is ordered on one stream.  The pressure loop is
// device-driven: half-sweeps are predicated on a device flag and enqueued in
// batches, and the host only polls a host-mapped word.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <unistd.h>

#include "sf_kernels.cuh"
#include "sf_plan.hpp"
#include "sf_jit.hpp"

namespace sfb {

using i64 = long long;

struct error : std::runtime_error {
  int code;
  error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SF_CK(x)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw ::sfb::error(SF_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

static thread_local std::string g_last_error;

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (the libnccl.so.2 torch already mapped into the
// process when there is one).  Types restated from nccl.h (stable ABI).
// ---------------------------------------------------------------------------
struct nccl_uid {
  char internal[128];
};
typedef struct ncclComm* nccl_comm_t;
enum { kNcclUint64 = 5, kNcclFloat64 = 8, kNcclMax = 2 };
struct nccl_api {
  int (*GetUniqueId)(nccl_uid*) = nullptr;
  int (*CommInitRank)(nccl_comm_t*, int, nccl_uid, int) = nullptr;
  int (*CommDestroy)(nccl_comm_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

static nccl_api* nccl() {
  static nccl_api api;
  static bool tried = false;
  if (tried) return api.Send ? &api : nullptr;
  tried = true;
  void* h = nullptr;
  if (const char* e = getenv("SF_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  auto sym = [&](const char* n) { return dlsym(h, n); };
  api.GetUniqueId = (int (*)(nccl_uid*))sym("ncclGetUniqueId");
  api.CommInitRank = (int (*)(nccl_comm_t*, int, nccl_uid, int))sym("ncclCommInitRank");
  api.CommDestroy = (int (*)(nccl_comm_t))sym("ncclCommDestroy");
  api.GroupStart = (int (*)())sym("ncclGroupStart");
  api.GroupEnd = (int (*)())sym("ncclGroupEnd");
  api.Send = (int (*)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclSend");
  api.Recv = (int (*)(void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclRecv");
  api.AllReduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclAllReduce");
  api.AllGather = (int (*)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t))sym("ncclAllGather");
  api.GetErrorString = (const char* (*)(int))sym("ncclGetErrorString");
  if (!api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllReduce ||
      !api.AllGather || !api.GroupStart || !api.GroupEnd) {
    api.Send = nullptr;
    return nullptr;
  }
  return &api;
}

#define SF_NC(x)                                                                              \
  do {                                                                                        \
    const int r_ = (x);                                                                       \
    if (r_ != 0)                                                                              \
      throw ::sfb::error(SF_ERR_CUDA, std::string("NCCL: ") + #x + ": " +                     \
                                          (::sfb::nccl()->GetErrorString ? ::sfb::nccl()->GetErrorString(r_) : "?")); \
  } while (0)

// ---------------------------------------------------------------------------
// decomposition (grid.hpp:44-163), same choices and error texts
// ---------------------------------------------------------------------------
struct decomposition {
  i64 ext[3]{};
  int workers = 1, ghost = 0;
  int pg[3]{1, 1, 1};
  bool periodic[3]{false, false, false};
  std::vector<std::array<i64, 3>> lo, hi;

  std::array<int, 3> coords_of(int w) const {
    const int pz = pg[2], py = pg[1];
    return {w / (py * pz), (w / pz) % py, w % pz};
  }
  int id_of(const std::array<int, 3>& c) const { return (c[0] * pg[1] + c[1]) * pg[2] + c[2]; }
  int neighbor(int w, int axis, int side) const {
    auto c = coords_of(w);
    int& ca = c[axis];
    ca += side == 0 ? -1 : 1;
    const int p = pg[axis];
    if (ca < 0 || ca >= p) {
      if (!periodic[axis]) return -1;
      ca = (ca + p) % p;
    }
    return id_of(c);
  }
  std::array<i64, 3> dims(int w) const {
    return {hi[w][0] - lo[w][0], hi[w][1] - lo[w][1], hi[w][2] - lo[w][2]};
  }
};

static std::vector<i64> split_axis(i64 n, int p) {
  std::vector<i64> s(p);
  const i64 base = n / p, rem = n % p;
  for (int i = 0; i < p; ++i) s[i] = base + (i < rem ? 1 : 0);
  return s;
}

decomposition decompose(const i64 ext[3], const double spacing[3], int workers, int ghost,
                        const bool periodic[3]) {
  if (workers < 1) throw error(SF_ERR_GRID, "worker count must be >= 1");
  if (ghost < 0) throw error(SF_ERR_GRID, "ghost width must be >= 0");
  for (int a = 0; a < 3; ++a) {
    if (ext[a] < 1) throw error(SF_ERR_GRID, "domain extents must be >= 1");
    if (!(spacing[a] > 0.0)) throw error(SF_ERR_GRID, "grid spacing must be positive");
  }
  auto feasible = [&](int p, i64 n) { return p <= n && n / p > ghost; };
  bool found = false;
  int best[3] = {1, 1, 1};
  i64 best_area = 0;
  for (int px = 1; px <= workers; ++px) {
    if (workers % px) continue;
    const int rest = workers / px;
    for (int py = 1; py <= rest; ++py) {
      if (rest % py) continue;
      const int pz = rest / py;
      if (!feasible(px, ext[0]) || !feasible(py, ext[1]) || !feasible(pz, ext[2])) continue;
      const i64 area = (i64)(px - 1) * ext[1] * ext[2] + (i64)(py - 1) * ext[0] * ext[2] +
                       (i64)(pz - 1) * ext[0] * ext[1];
      const bool better = !found || area < best_area ||
                          (area == best_area && (px > best[0] || (px == best[0] && py > best[1])));
      if (better) {
        found = true;
        best[0] = px;
        best[1] = py;
        best[2] = pz;
        best_area = area;
      }
    }
  }
  if (!found)
    throw error(SF_ERR_GRID, "no feasible decomposition: " + std::to_string(workers) +
                                 " workers on " + std::to_string(ext[0]) + "x" +
                                 std::to_string(ext[1]) + "x" + std::to_string(ext[2]) +
                                 " cells with ghost width " + std::to_string(ghost) +
                                 " (blocks must exceed the ghost width)");
  decomposition d;
  for (int a = 0; a < 3; ++a) {
    d.ext[a] = ext[a];
    d.pg[a] = best[a];
    d.periodic[a] = periodic[a];
  }
  d.workers = workers;
  d.ghost = ghost;
  std::array<std::vector<i64>, 3> sizes;
  for (int a = 0; a < 3; ++a) sizes[a] = split_axis(ext[a], best[a]);
  d.lo.resize(workers);
  d.hi.resize(workers);
  for (int w = 0; w < workers; ++w) {
    const auto c = d.coords_of(w);
    for (int a = 0; a < 3; ++a) {
      i64 l = 0;
      for (int i = 0; i < c[a]; ++i) l += sizes[a][i];
      d.lo[w][a] = l;
      d.hi[w][a] = l + sizes[a][c[a]];
    }
  }
  return d;
}

// executor.hpp:81-109
static std::vector<std::array<i64, 6>> region_boxes(const std::array<i64, 3>& dims,
                                                    const std::array<int, 6>& halo, int reg) {
  using box = std::array<i64, 6>;  // lo0 lo1 lo2 hi0 hi1 hi2
  const box all = {0, 0, 0, dims[0], dims[1], dims[2]};
  if (reg == SF_REGION_ALL) return {all};
  i64 il[3], ih[3];
  bool have = true;
  for (int a = 0; a < 3; ++a) {
    il[a] = std::min<i64>(halo[2 * a], dims[a]);
    ih[a] = std::max<i64>(il[a], dims[a] - halo[2 * a + 1]);
    if (il[a] >= ih[a]) have = false;
  }
  if (reg == SF_REGION_INTERIOR) {
    if (!have) return {};
    return {box{il[0], il[1], il[2], ih[0], ih[1], ih[2]}};
  }
  if (!have) return {all};
  std::vector<box> out = {
      {0, 0, 0, dims[0], dims[1], il[2]},
      {0, 0, ih[2], dims[0], dims[1], dims[2]},
      {0, 0, il[2], dims[0], il[1], ih[2]},
      {0, ih[1], il[2], dims[0], dims[1], ih[2]},
      {0, il[1], il[2], il[0], ih[1], ih[2]},
      {ih[0], il[1], il[2], dims[0], ih[1], ih[2]},
  };
  std::vector<box> kept;
  for (auto& b : out)
    if (!(b[3] <= b[0] || b[4] <= b[1] || b[5] <= b[2])) kept.push_back(b);
  return kept;
}

// Padded layout with 128-byte aligned rows at local i = 0.
static sf_layout make_layout(const i64 dims[3], const i64 lo[3], int g) {
  sf_layout l{};
  for (int a = 0; a < 3; ++a) {
    l.dims[a] = dims[a];
    l.lo[a] = lo[a];
  }
  l.ghost = g;
  const i64 xo = ((i64)g + 15) / 16 * 16;
  l.sx = (xo + dims[0] + g + 15) / 16 * 16;
  l.sy = dims[1] + 2 * g;
  l.sz = dims[2] + 2 * g;
  l.base = ((i64)g * l.sy + g) * l.sx + xo;
  return l;
}

// ---------------------------------------------------------------------------
// the simulation
// ---------------------------------------------------------------------------

struct kernel_plan {  // codegen::execution_plan of the three CFD kernels (cfd.hpp:111-162)
  std::string name;
  std::array<int, 6> halo;
  std::vector<std::string> bindings;
  std::vector<bool> writable, to_back;
  std::vector<std::string> params;
};

static const std::vector<kernel_plan>& cfd_plans() {
  static const std::vector<kernel_plan> plans = {
      {"UPDATE_VELOCITY", {1, 1, 1, 1, 1, 1}, {"vx", "vy", "vz", "p"},
       {true, true, true, false}, {true, true, true, false}, {"density"}},
      {"DIVERGENCE", {1, 0, 1, 0, 1, 0}, {"vx", "vy", "vz", "divu"},
       {false, false, false, true}, {false, false, false, false}, {}},
      {"PRESSURE_SWEEP", {0, 1, 0, 1, 0, 1}, {"divu", "p", "vx", "vy", "vz"},
       {false, true, true, true, true}, {false, false, false, false, false}, {"beta", "color"}},
  };
  return plans;
}

class simulation {
 public:
  struct user_kernel {
    std::string name;
    std::array<int, 3> tile{};
    std::array<int, 6> halo{};
    std::vector<int> fid, intent;
    std::vector<std::string> params;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k = nullptr;
    int tx = 32, ty = 8, zc = 16;
    int rpt = 1;  // rows per thread (TMA template): the CTA tile is tx x (ty * rpt) cells
    bool debug = false;
    // TMA-staged template (CACHED readable bindings)
    bool tma = false;
    std::vector<int> cslot;  // binding index of each cached binding
    int xl = 0, bw = 0, bh = 0, ring = 0;
    size_t smem = 0;
    void* maps = nullptr;
    long long maps_gen = -1;
  };
  // world > 1: one process per GPU; this rank owns grid component `rank` of
  // grid::decompose(dom, world, ghost, periodic) and talks to the others over
  // NCCL (communicator from `uid`, created collectively here).
  // htr != nullptr: the same, with the CUDA-IPC transport (peers' device
  // buffers mapped into this process; host callbacks for handles, scalars
  // and barriers) instead of NCCL.
  simulation(const sf_solver_config& cfg, const sf_fluid_params& par, const sf_sim_options& opt,
             int rank = 0, int world = 1, const void* uid = nullptr, const sf_host_transport* htr = nullptr)
      : cfg_(cfg), par_(par), opt_(opt), rank_(rank), world_(world) {
    validate();
    const bool per[3] = {cfg.periodic[0] != 0, cfg.periodic[1] != 0, cfg.periodic[2] != 0};
    const i64 ext[3] = {cfg.extents[0], cfg.extents[1], cfg.extents[2]};
    dist_ = uid != nullptr || htr != nullptr;
    tr_ = htr ? TR_IPC : (uid ? TR_NCCL : TR_NONE);
    // the fp32 variant of the CFD fields: storage and arithmetic in fp32 on the
    // fused TMA path (the temporal pass, the plain-load kernels and the
    // single CFD kernels stay fp64)
    if (opt.precision != 0 && opt.precision != 8 && opt.precision != 4)
      throw error(SF_ERR_ARG, "precision must be 8 (fp64) or 4 (fp32) bytes per value");
    cfd_es_ = opt.precision == 4 ? 4 : 8;
    if (cfd_es_ == 4) {
      if (opt.fused != 1 && opt.fused != 3)
        throw error(SF_ERR_ARG, "fp32 CFD fields run the fused TMA half-sweep (fused = 1 or 3)");
      for (int f = 0; f < SF_NFIELDS; ++f) fes_[f] = 4;
    }
    if (htr) {
      if (!htr->allgather || !htr->barrier) throw error(SF_ERR_ARG, "host transport needs allgather and barrier");
      htr_ = *htr;
    }
    if (dist_) {
      if (opt.workers != 1)
        throw error(SF_ERR_ARG, "distributed mode owns one grid component per rank (workers must be 1)");
      if (rank_ < 0 || rank_ >= world_) throw error(SF_ERR_ARG, "rank out of range");
      dec_ = decompose(ext, cfg.spacing, world_, opt.ghost, per);
      gid_ = {rank_};
      owner_.resize(world_);
      for (int w = 0; w < world_; ++w) owner_[w] = w;
    } else {
      dec_ = decompose(ext, cfg.spacing, opt.workers, opt.ghost, per);
      for (int w = 0; w < dec_.workers; ++w) gid_.push_back(w);
      owner_.assign(dec_.workers, 0);
    }
    nloc_ = (int)gid_.size();
    lid_.assign(dec_.workers, -1);
    for (int b = 0; b < nloc_; ++b) lid_[gid_[b]] = b;
    if (nloc_ > kMaxBlocks)
      throw error(SF_ERR_ARG, "at most " + std::to_string(kMaxBlocks) + " workers per device");
    make_bc();
    make_consts();
    SF_CK(cudaSetDevice(opt.device));
    SF_CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    if (tr_ == TR_NCCL) {
      if (!nccl()) throw error(SF_ERR_CUDA, "NCCL library not found (set SF_NCCL_LIB)");
      nccl_uid id;
      std::memcpy(&id, uid, sizeof id);
      SF_NC(nccl()->CommInitRank(&comm_, world_, id, rank_));
    }
    allocate();
    if (cfd_es_ == 4 && (!maps_ || !uvmaps_))
      throw error(SF_ERR_CUDA, "fp32 CFD fields need the TMA kernels (cuTensorMapEncodeTiled unavailable)");
    SF_CK(cudaEventCreateWithFlags(&ev_[0], cudaEventDisableTiming));
    SF_CK(cudaEventCreateWithFlags(&ev_[1], cudaEventDisableTiming));
    SF_CK(cudaEventCreate(&t0_));
    SF_CK(cudaEventCreate(&t1_));
    launch_ctl(dtab_, dctl_, dflag_, CTL_CLEAR_ACC, 0, 0, 0, 0, consts_, 0, st_);
    launch_ctl(dtab_, dctl_, dflag_, CTL_RESET_CLOCK, 0, 0, 0, 0, consts_, 0, st_);
    launches_ += 2;
    sync();
  }

  ~simulation() {
    cudaSetDevice(opt_.device);
    cudaStreamSynchronize(st_);
    for (auto& kv : ukernels_)
      if (kv.second.lib) cudaLibraryUnload(kv.second.lib);
    for (void* p : dev_allocs_) cudaFree(p);
    if (hflag_) cudaFreeHost(hflag_);
    cudaEventDestroy(ev_[0]);
    cudaEventDestroy(ev_[1]);
    cudaEventDestroy(t0_);
    cudaEventDestroy(t1_);
    for (auto e : timers_) cudaEventDestroy(e);
    drop_loop_graph();
    if (xs_) {
      cudaStreamSynchronize(xs_);
      cudaStreamDestroy(xs_);
      cudaEventDestroy(ev_fork_);
      cudaEventDestroy(ev_join_);
    }
    if (io_[0]) {
      for (int k = 0; k < 2; ++k) {
        cudaStreamSynchronize(io_[k]);
        cudaStreamDestroy(io_[k]);
      }
      for (auto e : io_ev_) cudaEventDestroy(e);
      for (auto e : io_up_) cudaEventDestroy(e);
      for (auto e : io_snap_) cudaEventDestroy(e);
      for (auto e : io_snapdn_) cudaEventDestroy(e);
      for (auto e : io_inst_) cudaEventDestroy(e);
    }
    for (auto& kv : ipc_open_) cudaIpcCloseMemHandle(kv.second);
    if (comm_ && nccl() && nccl()->CommDestroy) nccl()->CommDestroy(comm_);
    cudaStreamDestroy(st_);
  }

  // ---- helpers ------------------------------------------------------------
  void sync() {
    flush_io();
    SF_CK(cudaStreamSynchronize(st_));
  }
  void check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw error(SF_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  }

  int field_id(const std::string& name) const {
    for (int f = 0; f < (int)fname_.size(); ++f)
      if (name == fname_[f]) return f;
    throw error(SF_ERR_GRID, "no field named '" + name + "'");
  }
  int nfields() const { return (int)fname_.size(); }
  const std::string& field_name(int f) const { return fname_[f]; }

  // field_store::create (field.hpp:108-112): a zero-filled front buffer on
  // every local component; stagger -1 none, 0/1/2 = x/y/z (field.hpp:23)
  int create_field(const std::string& name, int stagger, int esize = 8) {
    if (esize != 8 && esize != 4) throw error(SF_ERR_ARG, "fields hold fp64 (8) or fp32 (4) values");
    for (const auto& n : fname_)
      if (n == name) throw error(SF_ERR_GRID, "field '" + name + "' already exists");
    if ((int)fname_.size() >= kMaxFields)
      throw error(SF_ERR_ARG, "at most " + std::to_string(kMaxFields) + " fields");
    if (stagger < -1 || stagger > 2) throw error(SF_ERR_ARG, "stagger must be -1, 0, 1 or 2");
    download_table();
    const int f = (int)fname_.size();
    fname_.push_back(name);
    fstag_.push_back(stagger);
    fes_.push_back(esize);
    htab_->esize[f] = (unsigned char)esize;
    for (int b = 0; b < nloc_; ++b) alloc_slot(b, f, FRONT);
    upload_table();
    return f;
  }
  // distributed_field::ensure_back (field.hpp:80-87)
  void ensure_back(int f) {
    download_table();
    bool any = false;
    for (int b = 0; b < nloc_; ++b)
      if (!htab_->ptr[b][f][BACK]) {
        alloc_slot(b, f, BACK);
        any = true;
      }
    if (any) upload_table();
  }
  bool has_back(int f) const { return htab_->ptr[0][f][BACK] != nullptr; }

  // ---- initial states (cfd.hpp:229-257) -------------------------------------
  void reset_clock() {
    time_ = 0.0;
    steps_ = 0;
    last_ = {0.0, 0, 0.0};
    ctl(CTL_RESET_CLOCK);
  }
  void fill_const(int f, double v) {
    download_table();
    for (int b = 0; b < nloc_; ++b) {
      const auto& L = lay_[b];
      const i64 lo[3] = {0, 0, 0};
      const i64 dims[3] = {L.dims[0], L.dims[1], L.dims[2]};
      launch_fill_box(htab_->ptr[b][f][FRONT], L.base, L.sx, L.sy, lo, dims, v, st_, fes_[f]);
      ++launches_;
    }
    check_launch();
    ghosts_ok_[fname_[f]] = false;
  }
  void init_cavity() {
    for (int f = 0; f < SF_NFIELDS; ++f) fill_const(f, 0.0);
    reset_clock();
  }
  void init_uniform(double cx, double cy, double cz) {
    fill_const(SF_VX, cx);
    fill_const(SF_VY, cy);
    fill_const(SF_VZ, cz);
    fill_const(SF_P, 0.0);
    fill_const(SF_DIVU, 0.0);
    reset_clock();
  }
  void init_taylor_green() {
    // host-side sampling with the C library's sin/cos, exactly as cfd.hpp:246-257
    const double tau = 2.0 * 3.14159265358979323846;
    const double dx = cfg_.spacing[0], dy = cfg_.spacing[1];
    const i64 nx = cfg_.extents[0], ny = cfg_.extents[1], nz = cfg_.extents[2];
    std::vector<double> u(nx * ny * nz), v(u.size()), q(u.size());
    for (i64 k = 0; k < nz; ++k)
      for (i64 j = 0; j < ny; ++j)
        for (i64 i = 0; i < nx; ++i) {
          const double xc = ((double)i + 0.5) * dx, yc = ((double)j + 0.5) * dy;
          const double xf = xc + 0.5 * dx, yf = yc + 0.5 * dy;
          const i64 o = (k * ny + j) * nx + i;
          u[o] = std::sin(tau * xf) * std::cos(tau * yc);
          v[o] = -std::cos(tau * xc) * std::sin(tau * yf);
          q[o] = 0.25 * (std::cos(2.0 * tau * xc) + std::cos(2.0 * tau * yc));
        }
    scatter(SF_VX, u.data(), false);
    scatter(SF_VY, v.data(), false);
    fill_const(SF_VZ, 0.0);
    scatter(SF_P, q.data(), false);
    fill_const(SF_DIVU, 0.0);
    reset_clock();
  }

  // ---- data movement (io.hpp:25-65) ----------------------------------------
  i64 cells() const { return cfg_.extents[0] * cfg_.extents[1] * cfg_.extents[2]; }
  double* staging() {
    if (!staging_) staging_ = (double*)dalloc(sizeof(double) * (size_t)cells());
    return staging_;
  }
  void gather_to_device(int f, double* dglobal) {
    download_table();
    flush_io();  // bumps the compute epoch: a later block_io must wait for this launch
    const i64 N[3] = {cfg_.extents[0], cfg_.extents[1], cfg_.extents[2]};
    for (int b = 0; b < nloc_; ++b) {
      const auto& L = lay_[b];
      const i64 n[3] = {L.dims[0], L.dims[1], L.dims[2]};
      const i64 lo[3] = {L.lo[0], L.lo[1], L.lo[2]};
      launch_gather_owned(htab_->ptr[b][f][FRONT], L.base, L.sx, L.sy, n, lo, N, dglobal, 0, st_, fes_[f]);
      ++launches_;
    }
    check_launch();
  }
  void scatter_from_device(int f, const double* dglobal) {
    download_table();
    flush_io();  // bumps the compute epoch: a later block_io must wait for this launch
    const i64 N[3] = {cfg_.extents[0], cfg_.extents[1], cfg_.extents[2]};
    for (int b = 0; b < nloc_; ++b) {
      const auto& L = lay_[b];
      const i64 n[3] = {L.dims[0], L.dims[1], L.dims[2]};
      const i64 lo[3] = {L.lo[0], L.lo[1], L.lo[2]};
      launch_gather_owned(htab_->ptr[b][f][FRONT], L.base, L.sx, L.sy, n, lo, N,
                          const_cast<double*>(dglobal), 1, st_, fes_[f]);
      ++launches_;
    }
    check_launch();
    ghosts_ok_[fname_[f]] = false;
  }
  // grid::gather across ranks: every rank packs its owned block, one
  // all-gather, every rank places all blocks (bitwise, no arithmetic)
  void gather_global(int f, double* host) {
    download_table();
    i64 maxc = 0;
    for (int w = 0; w < dec_.workers; ++w) {
      const auto d = dec_.dims(w);
      maxc = std::max(maxc, d[0] * d[1] * d[2]);
    }
    double* snd = (double*)dalloc_tmp(sizeof(double) * (size_t)maxc);
    double* all = (double*)dalloc_tmp(sizeof(double) * (size_t)(maxc * world_));
    const auto& L = lay_[0];
    const i64 n[3] = {L.dims[0], L.dims[1], L.dims[2]};
    const i64 z[3] = {0, 0, 0};
    launch_copy_box_es(htab_->ptr[0][f][FRONT], fes_[f], L.base, L.sx, L.sy, snd, 8, 0, n[0], n[1], z, n, z, st_);
    ++launches_;
    dev_allgather(snd, all, (size_t)maxc);
    std::vector<double> h((size_t)(maxc * world_));
    SF_CK(cudaMemcpyAsync(h.data(), all, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st_));
    sync();
    SF_CK(cudaFree(snd));
    SF_CK(cudaFree(all));
    const i64 N0 = cfg_.extents[0], N1 = cfg_.extents[1];
    for (int w = 0; w < dec_.workers; ++w) {
      const auto d = dec_.dims(w);
      const double* src = h.data() + (size_t)(maxc * w);
      for (i64 k = 0; k < d[2]; ++k)
        for (i64 j = 0; j < d[1]; ++j)
          std::memcpy(host + ((dec_.lo[w][2] + k) * N1 + dec_.lo[w][1] + j) * N0 + dec_.lo[w][0],
                      src + (k * d[1] + j) * d[0], sizeof(double) * (size_t)d[0]);
    }
  }
  // Owned block of local component w (global worker id) <-> dense x-fastest
  // host array: one 3-D copy-engine transfer straight between the host array
  // and the padded device block (row pitch sx, slice pitch sx*sy), on a
  // dedicated stream per direction. Ordering, all on the device:
  //  - a gather waits for the compute stream (the table download syncs it);
  //  - a scatter of field f waits for the last gather of f;
  //  - later compute waits for both.
  // Async mode returns at once: host memory must be pinned and stay untouched
  // until sf_sim_synchronize. Uploads then overlap downloads of other fields
  // (PCIe is full duplex).
  // The two halves of an asynchronous upload. stage: H2D into the field's
  // dense upload buffer on the upload stream, once the last install out of
  // that buffer ran; install: a kernel on the compute stream, after the
  // upload, copies the buffer into FRONT. Staging the next step's inputs
  // before stepping overlaps their transfer with the step.
  void ensure_io() {
    if (io_[0]) return;
    for (int k = 0; k < 2; ++k) SF_CK(cudaStreamCreateWithFlags(&io_[k], cudaStreamNonBlocking));
    for (int k = 0; k < kMaxFields; ++k) {
      SF_CK(cudaEventCreateWithFlags(&io_ev_[k], cudaEventDisableTiming));
      SF_CK(cudaEventCreateWithFlags(&io_up_[k], cudaEventDisableTiming));
      SF_CK(cudaEventCreateWithFlags(&io_snap_[k], cudaEventDisableTiming));
      SF_CK(cudaEventCreateWithFlags(&io_snapdn_[k], cudaEventDisableTiming));
      SF_CK(cudaEventCreateWithFlags(&io_inst_[k], cudaEventDisableTiming));
    }
  }
  int owned_block(int w, i64 n) const {
    if (w < 0 || w >= dec_.workers || lid_[w] < 0)
      throw error(SF_ERR_ARG, "worker " + std::to_string(w) + " is not owned by this process");
    const auto& L = lay_[lid_[w]];
    if (n >= 0 && n < L.dims[0] * L.dims[1] * L.dims[2]) throw error(SF_ERR_ARG, "block buffer too small");
    return lid_[w];
  }
  void stage_upload(int f, int b, const double* host, size_t cnt) {
    ensure_io();
    if (!upb_[b][f]) upb_[b][f] = (double*)dalloc(sizeof(double) * cnt);
    SF_CK(cudaStreamWaitEvent(io_[0], io_inst_[f], 0));  // the last install out of this buffer
    SF_CK(cudaMemcpyAsync(upb_[b][f], host, sizeof(double) * cnt, cudaMemcpyHostToDevice, io_[0]));
    SF_CK(cudaEventRecord(io_up_[f], io_[0]));
    staged_[b][f] = true;
  }
  void install_staged(int f, int b) {
    if (!staged_[b][f]) throw error(SF_ERR_ARG, "no staged upload of field '" + fname_[f] + "'");
    const auto& L = lay_[b];
    flush_io();
    SF_CK(cudaStreamWaitEvent(st_, io_up_[f], 0));
    launch_install(dtab_, b, f, upb_[b][f], L.dims[1] * L.dims[2], st_);
    ++launches_;
    SF_CK(cudaEventRecord(io_inst_[f], st_));
    staged_[b][f] = false;
    ghosts_ok_[fname_[f]] = false;
    check_launch();
  }
  void stage_block(int f, int w, const double* host, i64 n) {
    const int b = owned_block(w, n);
    const auto& L = lay_[b];
    stage_upload(f, b, host, (size_t)(L.dims[0] * L.dims[1] * L.dims[2]));
  }
  void install_block(int f, int w) { install_staged(f, owned_block(w, -1)); }

  void block_io(int f, int w, double* host, i64 n, bool to_device, bool async = false) {
    if (w < 0 || w >= dec_.workers || lid_[w] < 0)
      throw error(SF_ERR_ARG, "worker " + std::to_string(w) + " is not owned by this process");
    const int b = lid_[w];
    const auto& L = lay_[b];
    const i64 d[3] = {L.dims[0], L.dims[1], L.dims[2]};
    if (n < d[0] * d[1] * d[2]) throw error(SF_ERR_ARG, "block buffer too small");
    ensure_io();
    if (!to_device && async) {
      // Snapshot, then download in the background: a pack task on the compute
      // stream copies the owned block into a dense device buffer (FRONT is
      // resolved on the device, so no host synchronisation), and the copy
      // engine moves that buffer while later compute proceeds.
      const size_t cnt = (size_t)(d[0] * d[1] * d[2]);
      if (!snap_[b][f]) snap_[b][f] = (double*)dalloc(sizeof(double) * cnt);
      SF_CK(cudaStreamWaitEvent(st_, io_snapdn_[f], 0));  // the last download out of this buffer
      flush_io();
      launch_snapshot(dtab_, b, f, snap_[b][f], d[1] * d[2], st_);
      ++launches_;
      SF_CK(cudaEventRecord(io_snap_[f], st_));
      SF_CK(cudaStreamWaitEvent(io_[1], io_snap_[f], 0));
      SF_CK(cudaMemcpyAsync(host, snap_[b][f], sizeof(double) * cnt, cudaMemcpyDeviceToHost, io_[1]));
      SF_CK(cudaEventRecord(io_snapdn_[f], io_[1]));
      check_launch();
      return;
    }
    if (to_device && async) {
      // Upload into a dense device buffer on the upload stream, then install
      // it into FRONT with a kernel on the compute stream (FRONT resolved on
      // the device): no host synchronisation, and compute enqueued later sees
      // the new values.
      stage_upload(f, b, host, (size_t)(d[0] * d[1] * d[2]));
      install_staged(f, b);
      return;
    }
    if (fes_[f] != 8) {  // fp32 field: host values are fp64, converted through the staging buffer
      download_table();
      double* sg = staging();
      const i64 z[3] = {0, 0, 0};
      const size_t bytes = sizeof(double) * (size_t)(d[0] * d[1] * d[2]);
      if (to_device) {
        SF_CK(cudaMemcpyAsync(sg, host, bytes, cudaMemcpyHostToDevice, st_));
        launch_copy_box_es(sg, 8, 0, d[0], d[1], htab_->ptr[b][f][FRONT], fes_[f], L.base, L.sx, L.sy, z, d, z,
                           st_);
        ghosts_ok_[fname_[f]] = false;
      } else {
        launch_copy_box_es(htab_->ptr[b][f][FRONT], fes_[f], L.base, L.sx, L.sy, sg, 8, 0, d[0], d[1], z, d, z,
                           st_);
        SF_CK(cudaMemcpyAsync(host, sg, bytes, cudaMemcpyDeviceToHost, st_));
      }
      ++launches_;
      sync();
      return;
    }
    download_table(false);
    cudaMemcpy3DParms prm = {};
    double* dev = htab_->ptr[b][f][FRONT] + L.base;
    cudaPitchedPtr dp = make_cudaPitchedPtr(dev, (size_t)L.sx * sizeof(double), (size_t)d[0] * sizeof(double),
                                            (size_t)L.sy);
    cudaPitchedPtr hp = make_cudaPitchedPtr(host, (size_t)d[0] * sizeof(double), (size_t)d[0] * sizeof(double),
                                            (size_t)d[1]);
    prm.extent = make_cudaExtent((size_t)d[0] * sizeof(double), (size_t)d[1], (size_t)d[2]);
    if (to_device) {
      prm.srcPtr = hp;
      prm.dstPtr = dp;
      prm.kind = cudaMemcpyHostToDevice;
      SF_CK(cudaStreamWaitEvent(io_[0], io_ev_[f], 0));    // the last direct download of f
      SF_CK(cudaStreamWaitEvent(io_[0], io_snap_[f], 0));  // the last snapshot of f
      SF_CK(cudaMemcpy3DAsync(&prm, io_[0]));
      SF_CK(cudaEventRecord(io_up_[f], io_[0]));
      io_pending_.push_back(io_up_[f]);
      ghosts_ok_[fname_[f]] = false;
    } else {
      prm.srcPtr = dp;
      prm.dstPtr = hp;
      prm.kind = cudaMemcpyDeviceToHost;
      SF_CK(cudaStreamWaitEvent(io_[1], io_up_[f], 0));  // after the last upload of f
      SF_CK(cudaMemcpy3DAsync(&prm, io_[1]));
      SF_CK(cudaEventRecord(io_ev_[f], io_[1]));
      io_pending_.push_back(io_ev_[f]);  // compute may not overwrite f before it is read
    }
    if (!async) SF_CK(cudaStreamSynchronize(io_[to_device ? 0 : 1]));
  }
  void io_sync() {
    for (int k = 0; k < 2; ++k)
      if (io_[k]) SF_CK(cudaStreamSynchronize(io_[k]));
  }
  int rank() const { return rank_; }
  int world() const { return world_; }

  void gather(int f, double* host) {
    if (dist_) {
      gather_global(f, host);
      return;
    }
    double* sg = staging();
    gather_to_device(f, sg);
    SF_CK(cudaMemcpyAsync(host, sg, sizeof(double) * (size_t)cells(), cudaMemcpyDeviceToHost, st_));
    sync();
  }
  void scatter(int f, const double* host, bool do_sync = true) {
    double* sg = staging();
    SF_CK(cudaMemcpyAsync(sg, host, sizeof(double) * (size_t)cells(), cudaMemcpyHostToDevice, st_));
    scatter_from_device(f, sg);
    if (do_sync) sync();
  }
  void local_front(int f, int w, double* host, i64 host_elems, i64 dims[3], i64 lo[3]) {
    if (w < 0 || w >= dec_.workers || lid_[w] < 0)
      throw error(SF_ERR_ARG, "worker " + std::to_string(w) + " is not owned by this process");
    w = lid_[w];
    const auto& L = lay_[w];
    const int g = L.ghost;
    const i64 ld[3] = {L.dims[0] + 2 * g, L.dims[1] + 2 * g, L.dims[2] + 2 * g};
    if (host_elems < ld[0] * ld[1] * ld[2]) throw error(SF_ERR_ARG, "host buffer too small");
    for (int a = 0; a < 3; ++a) {
      dims[a] = L.dims[a];
      lo[a] = L.lo[a];
    }
    download_table();
    double* sg = (double*)dalloc_tmp(sizeof(double) * (size_t)(ld[0] * ld[1] * ld[2]));
    const i64 slo[3] = {-g, -g, -g};
    const i64 zero[3] = {0, 0, 0};
    launch_copy_box_es(htab_->ptr[w][f][FRONT], fes_[f], L.base, L.sx, L.sy, sg, 8, 0, ld[0], ld[1], slo, ld,
                       zero, st_);
    ++launches_;
    check_launch();
    SF_CK(cudaMemcpyAsync(host, sg, sizeof(double) * (size_t)(ld[0] * ld[1] * ld[2]),
                          cudaMemcpyDeviceToHost, st_));
    sync();
    SF_CK(cudaFree(sg));
  }
  uint64_t checksum() {  // bench.hpp:24-39
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* data, size_t n) {
      const unsigned char* p = static_cast<const unsigned char*>(data);
      for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
      }
    };
    std::vector<double> g((size_t)cells());
    for (int f : {SF_VX, SF_VY, SF_VZ, SF_P}) {
      mix(fname_[f].data(), fname_[f].size());
      gather(f, g.data());
      mix(g.data(), g.size() * sizeof(double));
    }
    return h;
  }

  // ---- executor operations (executor.hpp:500-527) ---------------------------
  void refresh(const std::vector<int>& fields, bool predicated = false) {
    if (fields.empty()) return;
    validate_bc(fields);
    unsigned mask = 0;
    for (int f : fields) mask |= 1u << f;
    for (int axis = 0; axis < 3; ++axis) run_phase(phase_for(mask, axis, SF_SCOPE_ALL, false), predicated);
    check_launch();
    for (int f : fields) ghosts_ok_[fname_[f]] = true;
  }
  void exchange_only(const std::vector<int>& fields) {
    unsigned mask = 0;
    for (int f : fields) mask |= 1u << f;
    for (int axis = 0; axis < 3; ++axis) run_phase(phase_for(mask, axis, SF_SCOPE_ALL, true), false);
    check_launch();
    for (int f : fields) ghosts_ok_[fname_[f]] = true;
  }

  void run_kernel(const std::string& name, const std::map<std::string, double>& params, int reg) {
    if (is_user_kernel(name)) {
      run_user_kernel(name, params, reg);
      check_launch();
      return;
    }
    const kernel_plan* kp = nullptr;
    for (const auto& p : cfd_plans())
      if (p.name == name) kp = &p;
    if (!kp) throw error(SF_ERR_EXEC, "unknown kernel '" + name + "'");
    if (cfd_es_ != 8)
      throw error(SF_ERR_ARG, "kernel '" + name + "': the single CFD kernels are fp64; an fp32 simulation runs them "
                              "fused inside step() / provisional() / pressure_iteration()");
    std::vector<double> pv;
    for (const auto& pn : kp->params) {
      auto it = params.find(pn);
      if (it == params.end())
        throw error(SF_ERR_EXEC, "kernel '" + name + "': parameter '" + pn + "' not supplied");
      pv.push_back(it->second);
    }
    if (reg < 0 || reg > 2) throw error(SF_ERR_ARG, "bad region");
    const work_set& ws = items_for(reg, kp->halo, zc_plain_);
    if (name == "UPDATE_VELOCITY") {
      launch_update_velocity(tview(ws), ws.nctas, zc_plain_, consts_, dctl_, 0.0, st_);
      ++launches_;
    } else if (name == "DIVERGENCE") {
      launch_divergence(tview(ws), ws.nctas, zc_plain_, consts_, dctl_, -1, 0, st_);
      ++launches_;
    } else {
      // beta and colour come from the call, dt from the simulation (cfd.hpp:630-697)
      const double bcd[3] = {pv[0], pv[1], 0.0};
      launch_pressure_sweep(tview(ws), ws.nctas, zc_plain_, consts_, dctl_, 0, bcd, st_);
      ++launches_;
    }
    check_launch();
    // finish_run (executor.hpp:769-779)
    for (size_t b = 0; b < kp->bindings.size(); ++b) {
      if (reg != SF_REGION_INTERIOR) {
        if (kp->writable[b]) ghosts_ok_[kp->bindings[b]] = false;
      } else if (kp->writable[b] && !kp->to_back[b]) {
        ghosts_ok_[kp->bindings[b]] = false;
      }
    }
    if (reg != SF_REGION_INTERIOR && name == "UPDATE_VELOCITY") swap_front_back();
  }

  // ---- descriptor-declared kernels (executor.hpp:484-498, 650-692) ---------
  void register_kernel(const std::string& name, const std::array<int, 3>& tile,
                       const std::array<int, 6>& halo, const std::vector<std::string>& bfields,
                       const std::vector<int>& intents, const std::vector<int>& cached,
                       const std::vector<std::string>& params,
                       const std::vector<std::string>& sig_fields,
                       const std::vector<std::string>& sig_params, const std::string& body) {
    const std::string head = "kernel '" + name + "': ";
    for (const auto& p : cfd_plans())
      if (p.name == name) throw error(SF_ERR_EXEC, "kernel '" + name + "' is already registered");
    if (ukernels_.count(name)) throw error(SF_ERR_EXEC, "kernel '" + name + "' is already registered");
    if (bfields.empty()) throw error(SF_ERR_EXEC, "kernel '" + name + "' has no field bindings");
    for (int a = 0; a < 3; ++a)
      if (tile[a] < 1) throw error(SF_ERR_EXEC, head + "tile extents must be positive");
    // check_signature (executor.hpp:715-737)
    for (size_t i = 0; i < std::max(bfields.size(), sig_fields.size()); ++i) {
      if (i >= sig_fields.size()) throw error(SF_ERR_EXEC, head + "function is missing binding '" + bfields[i] + "'");
      if (i >= bfields.size())
        throw error(SF_ERR_EXEC, head + "function declares unknown binding '" + sig_fields[i] + "'");
      if (bfields[i] != sig_fields[i])
        throw error(SF_ERR_EXEC, head + "slot " + std::to_string(i) + " binds '" + bfields[i] +
                                     "' but the function declares '" + sig_fields[i] + "'");
    }
    for (size_t i = 0; i < std::max(params.size(), sig_params.size()); ++i) {
      if (i >= sig_params.size()) throw error(SF_ERR_EXEC, head + "function is missing parameter '" + params[i] + "'");
      if (i >= params.size())
        throw error(SF_ERR_EXEC, head + "function declares unknown parameter '" + sig_params[i] + "'");
      if (params[i] != sig_params[i])
        throw error(SF_ERR_EXEC, head + "parameter slot " + std::to_string(i) + " is '" + params[i] +
                                     "' but the function declares '" + sig_params[i] + "'");
    }
    int mh = 0;
    for (int h : halo) mh = std::max(mh, h);
    if (mh > dec_.ghost)
      throw error(SF_ERR_EXEC, head + "stencil needs " + std::to_string(mh) + " ghost layers but fields carry " +
                                   std::to_string(dec_.ghost));
    user_kernel uk;
    uk.name = name;
    uk.tile = tile;
    uk.halo = halo;
    uk.params = params;
    for (size_t i = 0; i < bfields.size(); ++i) {
      int f = -1;
      for (int q = 0; q < (int)fname_.size(); ++q)
        if (fname_[q] == bfields[i]) f = q;
      if (f < 0) throw error(SF_ERR_EXEC, "kernel '" + name + "' binds unknown field '" + bfields[i] + "'");
      if (intents[i] < 0 || intents[i] > 3) throw error(SF_ERR_ARG, "bad intent");
      uk.fid.push_back(f);
      uk.intent.push_back(intents[i]);
    }
    for (size_t i = 0; i < uk.fid.size(); ++i)
      if (uk.intent[i] == 3) ensure_back(uk.fid[i]);
    // CTA tile = the descriptor's TILE (x, y threads), z chunk = TILE z
    uk.tx = std::min(tile[0], 1024);
    uk.ty = std::max(1, std::min(tile[1], 1024 / uk.tx));
    uk.zc = tile[2];
    // Each thread sweeps SF_JIT_ROWS (1 or 2; default 2) adjacent rows of the
    // tile with its stores deferred to the end of the pair, so the
    // shared-memory reads that coincide between the rows fold into one load
    // (768^3 fp64: radius 2 1.43 -> 1.34 ms, radius 3 1.84 -> 1.64 ms;
    // DESIGN.md §9).  Needs an even tile height and no INOUT binding (a
    // deferred INOUT store would be invisible to a later read of the same
    // cell).  Four rows measured slower (register pressure; the compiler
    // stops folding loads that far apart).
    static const int rows_env = getenv("SF_JIT_ROWS") ? atoi(getenv("SF_JIT_ROWS")) : 2;
    bool inout = false;
    for (int in : uk.intent) inout = inout || in == 2;
    const int trows = uk.ty;  // cell rows per CTA tile
    const int rpt = rows_env == 2 && trows % 2 == 0 && !inout ? 2 : 1;
    // CACHED readable bindings -> TMA plane ring (needs an even TX for the
    // 16-byte aligned box start, boxes <= 256 per dimension, fitting smem)
    std::vector<int> cs;
    for (size_t i = 0; i < bfields.size(); ++i)
      if (i < cached.size() && cached[i] && uk.intent[i] != 1) cs.push_back((int)i);
    // TMA box x start and row bytes must be 16-byte multiples: 2 fp64 or 4 fp32
    int xa = 2;
    for (int c : cs)
      if (fes_[uk.fid[c]] == 4) xa = 4;
    if (!cs.empty() && uk.tx % xa == 0 && !getenv("SF_JIT_NO_TMA")) {
      const int xl = (halo[0] + xa - 1) / xa * xa;
      const int bw = (xl + uk.tx + halo[1] + xa - 1) / xa * xa;
      const int bh = halo[2] + trows + halo[3];
      // window + the two planes of a round + one plane of look-ahead (2 extra
      // planes measured 20-50 % slower, 4 within noise)
      const int ring = halo[4] + halo[5] + 1 + 3;
      const size_t smem = (size_t)cs.size() * ring * ((bw * bh + 15) / 16 * 16) * 8;
      bool fits = true;  // a box larger than the padded array is pointless (and rejected)
      for (const auto& L : lay_) fits = fits && bw <= L.sx && bh <= L.sy;
      if (bw <= 256 && bh <= 256 && smem <= 200 * 1024 && fits) {
        uk.tma = true;
        uk.cslot = cs;
        uk.xl = xl;
        uk.bw = bw;
        uk.bh = bh;
        uk.ring = ring;
        uk.smem = smem;
        uk.rpt = rpt;
        uk.ty = trows / rpt;
      }
    }
    compile_user(uk, body);
    ukernels_.emplace(name, uk);
  }

  void compile_user(user_kernel& uk, const std::string& body) {
    nvrtc_api* rt = getenv("SF_JIT_DUMP_ONLY") ? nullptr : nvrtc();
    if (!rt && !getenv("SF_JIT_DUMP_ONLY")) throw error(SF_ERR_CUDA, "NVRTC not found (set SF_NVRTC_LIB)");
    std::string src;
    src += "#define SF_NB " + std::to_string(uk.fid.size()) + "\n";
    src += "#define SF_NP " + std::to_string(uk.params.size()) + "\n";
    src += "#define SF_TX " + std::to_string(uk.tx) + "\n#define SF_TY " + std::to_string(uk.ty) + "\n";
    src += "#define SF_RPT " + std::to_string(uk.rpt) + "\n";
    // no minimum of resident CTAs per SM: every explicit minimum measured
    // slower or equal
    src += "#define SF_LAUNCH_BOUNDS __launch_bounds__(SF_TX * SF_TY)\n";
    src += "#define SF_MAXF " + std::to_string(kMaxFields) + "\n#define SF_SLOTS " + std::to_string(kSlots) + "\n";
    std::string fids, wsl;
    for (size_t i = 0; i < uk.fid.size(); ++i) {
      fids += (i ? "," : "") + std::to_string(uk.fid[i]);
      wsl += (i ? "," : "") + std::string(uk.intent[i] == 3 ? "1" : "0");
    }
    std::string rdb, wrb, cen;
    for (size_t i = 0; i < uk.fid.size(); ++i) {
      const int in = uk.intent[i];
      rdb += (i ? "," : "") + std::string(in != 1 ? "1" : "0");
      wrb += (i ? "," : "") + std::string(in != 0 ? "1" : "0");
      cen += (i ? "," : "") + std::string(in == 2 ? "1" : "0");
    }
    src += "__device__ constexpr int SF_FID[] = {" + fids + "};\n";
    src += "__device__ constexpr int SF_WSLOT[] = {" + wsl + "};\n";
    src += "__device__ constexpr int SF_READABLE[] = {" + rdb + "};\n";
    src += "__device__ constexpr int SF_WRITABLE[] = {" + wrb + "};\n";
    src += "__device__ constexpr int SF_CENTER_ONLY[] = {" + cen + "};\n";
    std::string f32;
    for (size_t i = 0; i < uk.fid.size(); ++i) f32 += (i ? "," : "") + std::string(fes_[uk.fid[i]] == 4 ? "1" : "0");
    src += "__device__ constexpr int SF_F32[] = {" + f32 + "};\n";
    // a kernel whose bindings are all fp32 computes in fp32: accessors return
    // sf_real = float (bodies written with sf_real run in either precision)
    bool all32 = !uk.fid.empty();
    for (int f : uk.fid) all32 = all32 && fes_[f] == 4;
    src += std::string("typedef ") + (all32 ? "float" : "double") + " sf_real;\n";
    src += "__device__ constexpr int SF_HALO[] = {";
    for (int a = 0; a < 6; ++a) src += (a ? "," : "") + std::to_string(uk.halo[a]);
    src += "};\n#define SF_DEBUG " + std::string(debug_bounds() ? "1" : "0") + "\n";
    uk.debug = debug_bounds();
    if (uk.tma) {
      std::string csl;
      for (size_t i = 0; i < uk.cslot.size(); ++i) csl += (i ? "," : "") + std::to_string(uk.cslot[i]);
      std::string cached_flags, cidx;
      for (size_t b = 0; b < uk.fid.size(); ++b) {
        int ci = -1;
        for (size_t q = 0; q < uk.cslot.size(); ++q)
          if (uk.cslot[q] == (int)b) ci = (int)q;
        cached_flags += (b ? "," : "") + std::string(ci >= 0 ? "1" : "0");
        cidx += (b ? "," : "") + std::to_string(ci >= 0 ? ci : 0);
      }
      src += "__device__ constexpr int SF_CACHED[] = {" + cached_flags + "};\n";
      src += "__device__ constexpr int SF_CIDX[] = {" + cidx + "};\n";
      src += "#define SF_NC " + std::to_string(uk.cslot.size()) + "\n__device__ constexpr int SF_CSLOT[] = {" + csl +
             "};\n#define SF_XL " + std::to_string(uk.xl) + "\n#define SF_BW " + std::to_string(uk.bw) +
             "\n#define SF_BH " + std::to_string(uk.bh) + "\n#define SF_R " + std::to_string(uk.ring) + "\n";
      // one unrolled two-plane body per z-queue phase (sf_jit.hpp)
      src += "#define SF_PLANE_CASES";
      for (int p = 0; p < uk.halo[4] + uk.halo[5] + 1; ++p) src += " SF_PLANES(" + std::to_string(p) + ")";
      src += "\n";
      size_t txb = 0;  // bytes one plane of every cached binding brings in
      for (int c : uk.cslot) txb += (size_t)uk.bw * uk.bh * fes_[uk.fid[c]];
      src += "#define SF_TXB " + std::to_string(txb) + "\n";
    }
    std::string tmpl = uk.tma ? jit_template_tma() : jit_template();
    const size_t at = tmpl.find("SF_BODY");
    tmpl.replace(at, 7, "#line 1 \"" + uk.name + "\"\n" + body + "\n");
    src += tmpl;
    if (const char* dump = getenv("SF_JIT_DUMP")) {  // inspect the generated tile kernel
      std::string fn = std::string(dump) + "/" + uk.name + ".cu";
      if (FILE* fp = std::fopen(fn.c_str(), "w")) {
        std::fputs(src.c_str(), fp);
        std::fclose(fp);
      }
    }
    if (!rt) throw error(SF_ERR_EXEC, "SF_JIT_DUMP_ONLY: source written, not compiled");
    void* prog = nullptr;
    if (rt->create(&prog, src.c_str(), (uk.name + ".cu").c_str(), 0, nullptr, nullptr) != 0)
      throw error(SF_ERR_CUDA, "nvrtcCreateProgram failed");
    const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17", "-lineinfo",
                          "-default-device"};
    const int rc = rt->compile(prog, 5, opts);
    std::string log;
    size_t ls = 0;
    if (rt->log_size && rt->log_size(prog, &ls) == 0 && ls > 1) {
      log.resize(ls);
      rt->log(prog, &log[0]);
    }
    if (rc != 0) {
      rt->destroy(&prog);
      throw error(SF_ERR_EXEC, "kernel '" + uk.name + "': device compilation failed:\n" + log);
    }
    size_t cs = 0;
    rt->cubin_size(prog, &cs);
    std::string cubin(cs, '\0');
    rt->cubin(prog, &cubin[0]);
    rt->destroy(&prog);
    SF_CK(cudaLibraryLoadData(&uk.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    SF_CK(cudaLibraryGetKernel(&uk.k, uk.lib, "sf_user_kernel"));
    if (uk.tma)
      SF_CK(cudaFuncSetAttribute((const void*)uk.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)uk.smem));
    if (uk.debug) {  // point the module's error word at a device buffer
      if (!dbg_word_) {
        dbg_word_ = (int*)dalloc(8 * sizeof(int));
        SF_CK(cudaMemset(dbg_word_, 0, 8 * sizeof(int)));
      }
      void* sym = nullptr;
      size_t bytes = 0;
      SF_CK(cudaLibraryGetGlobal(&sym, &bytes, uk.lib, "sf_err_word"));
      SF_CK(cudaMemcpy(sym, &dbg_word_, sizeof(int*), cudaMemcpyHostToDevice));
    }
  }

  bool is_user_kernel(const std::string& name) const { return ukernels_.count(name) > 0; }

  // executor::boundary() (executor.hpp:482): replace one face condition
  void set_face_bc(int axis, int side, int kind, const double vel[3]) {
    if (axis < 0 || axis > 2 || side < 0 || side > 1 || kind < 0 || kind > 3)
      throw error(SF_ERR_ARG, "bad face condition");
    bc_[2 * axis + side] = {kind, {vel ? vel[0] : 0.0, vel ? vel[1] : 0.0, vel ? vel[2] : 0.0}};
    // refresh the block face kinds the fused kernels read and drop cached phases
    download_table();
    for (int b = 0; b < nloc_; ++b) {
      const int fi = 2 * axis + side;
      if (dec_.neighbor(gid_[b], axis, side) < 0) {
        htab_->blk[b].face[fi] = kind == SF_BC_WALL ? FACE_WALL : kind == SF_BC_SYMMETRY ? FACE_SYM
                                 : kind == SF_BC_OUTFLOW ? FACE_OUT : FACE_WALL;
        for (int c = 0; c < 3; ++c) htab_->blk[b].fvel[fi][c] = bc_[fi].velocity[c];
      }
    }
    SF_CK(cudaMemcpy(dtab_->blk, htab_->blk, sizeof(htab_->blk), cudaMemcpyHostToDevice));
    phases_.clear();
    drop_loop_graph();
  }

  // executor::physical_bc (executor.hpp:516-518): bc fills only, x then y then z
  void physical_bc(const std::vector<int>& fields) {
    if (fields.empty()) return;
    validate_bc(fields);
    unsigned mask = 0;
    for (int f : fields) mask |= 1u << f;
    for (int axis = 0; axis < 3; ++axis) run_phase(phase_for(mask, axis, SF_SCOPE_ALL, false, true), false);
    check_launch();
  }

  // ---- schedules (executor.hpp:420-470, 533-601) ---------------------------
  struct sched_step {
    int kind;  // 0 run, 1 exchange, 2 physical_bc, 3 refresh, 4 reduce (schedule_step::kind)
    std::string kernel;
    int reg = 0;
    std::vector<std::string> fields;
    std::string source, target;
    int op = 0;
  };
  std::map<std::string, double> results_;

  void kernel_io(const std::string& name, std::vector<std::string>& reads, std::vector<std::string>& writes,
                 int& max_halo) {
    reads.clear();
    writes.clear();
    max_halo = 0;
    if (is_user_kernel(name)) {
      const auto& k = ukernels_.at(name);
      for (int h : k.halo) max_halo = std::max(max_halo, h);
      for (size_t b = 0; b < k.fid.size(); ++b) {
        if (k.intent[b] != 1) reads.push_back(fname_[k.fid[b]]);
        if (k.intent[b] != 0) writes.push_back(fname_[k.fid[b]]);
      }
      return;
    }
    for (const auto& p : cfd_plans())
      if (p.name == name) {
        for (int h : p.halo) max_halo = std::max(max_halo, h);
        for (size_t b = 0; b < p.bindings.size(); ++b) {
          const bool w = p.writable[b];
          // every CFD binding is readable except DIVERGENCE's OUT divu (cfd.hpp:139-142)
          if (!(p.name == "DIVERGENCE" && p.bindings[b] == "divu")) reads.push_back(p.bindings[b]);
          if (w) writes.push_back(p.bindings[b]);
        }
        return;
      }
    throw error(SF_ERR_EXEC, "unknown kernel '" + name + "'");
  }

  void dry_run(const std::vector<sched_step>& s, int steps) {  // executor.hpp:559-601
    auto ok = ghosts_ok_;
    const int passes = std::min(steps, 4);
    for (int pass = 0; pass < passes; ++pass) {
      const auto before = ok;
      for (size_t i = 0; i < s.size(); ++i) {
        const auto& st = s[i];
        const std::string where = "schedule step " + std::to_string(i + 1);
        auto require = [&](const std::string& f) {
          bool found = false;
          for (const auto& n : fname_) found = found || n == f;
          if (!found) throw error(SF_ERR_EXEC, where + ": unknown field '" + f + "'");
        };
        switch (st.kind) {
          case 1:
          case 3:
            for (const auto& f : st.fields) {
              require(f);
              ok[f] = true;
            }
            break;
          case 2:
            for (const auto& f : st.fields) require(f);
            break;
          case 4:
            require(st.source);
            break;
          case 0: {
            std::vector<std::string> rd, wr;
            int mh = 0;
            try {
              kernel_io(st.kernel, rd, wr, mh);
            } catch (const error&) {
              throw error(SF_ERR_EXEC, where + ": unknown kernel '" + st.kernel + "'");
            }
            if (mh > 0 && st.reg != SF_REGION_INTERIOR)
              for (const auto& f : rd) {
                auto it = ok.find(f);
                if (it == ok.end() || !it->second)
                  throw error(SF_ERR_EXEC, where + ": kernel '" + st.kernel + "' reads ghosts of '" + f +
                                               "' that were never exchanged");
              }
            for (const auto& f : wr) ok[f] = false;
            break;
          }
        }
      }
      if (ok == before) break;
    }
  }

  void run_schedule(const std::vector<sched_step>& s, const std::map<std::string, double>& params, int steps) {
    dry_run(s, steps);
    for (int pass = 0; pass < steps; ++pass)
      for (const auto& st : s) {
        std::vector<int> fl;
        for (const auto& f : st.fields) fl.push_back(field_id(f));
        switch (st.kind) {
          case 0: run_kernel(st.kernel, params, st.reg); break;
          case 1: exchange_only(fl); break;
          case 2: physical_bc(fl); break;
          case 3: refresh(fl); break;
          case 4: results_[st.target] = reduce(field_id(st.source), st.op); break;
        }
      }
  }
  bool result(const std::string& name, double* v) const {
    auto it = results_.find(name);
    if (it == results_.end()) return false;
    *v = it->second;
    return true;
  }

  void run_user_kernel(const std::string& name, const std::map<std::string, double>& params, int reg) {
    user_kernel& uk = ukernels_.at(name);
    struct { double v[32]; } prm{};
    if (uk.params.size() > 32) throw error(SF_ERR_ARG, "at most 32 parameters");
    for (size_t i = 0; i < uk.params.size(); ++i) {
      auto it = params.find(uk.params[i]);
      if (it == params.end())
        throw error(SF_ERR_EXEC, "kernel '" + name + "': parameter '" + uk.params[i] + "' not supplied");
      prm.v[i] = it->second;
    }
    if (reg < 0 || reg > 2) throw error(SF_ERR_ARG, "bad region");
    if (debug_bounds()) check_ghosts(uk, reg);
    const work_set& ws = items_for(reg, uk.halo, uk.zc, uk.tx, uk.ty * uk.rpt);
    if (ws.nctas > 0) {
      flush_io();
      double* const* ptrs = &dtab_->ptr[0][0][0];
      const void* geo = geo_;
      const sf_work* items = ws.d;
      int nitems = ws.n, zc = uk.zc;
      if (uk.tma) {
        if (uk.maps_gen != alloc_gen_) build_user_maps(uk);
        const unsigned char* bidx = &dtab_->bidx[0][0][0];
        const void* maps = uk.maps;
        void* args[] = {(void*)&ptrs, (void*)&geo, (void*)&items, (void*)&nitems, (void*)&zc,
                        (void*)&prm,  (void*)&bidx, (void*)&maps};
        SF_CK(cudaLaunchKernel((const void*)uk.k, dim3(ws.nctas), dim3(uk.tx, uk.ty), args, uk.smem, st_));
      } else {
        void* args[] = {(void*)&ptrs, (void*)&geo, (void*)&items, (void*)&nitems, (void*)&zc, (void*)&prm};
        SF_CK(cudaLaunchKernel((const void*)uk.k, dim3(ws.nctas), dim3(uk.tx, uk.ty), args, 0, st_));
      }
      ++launches_;
      if (uk.debug) {
        int w[5] = {0, 0, 0, 0, 0};
        sync();
        SF_CK(cudaMemcpy(w, dbg_word_, sizeof w, cudaMemcpyDeviceToHost));
        if (w[0]) {
          SF_CK(cudaMemset(dbg_word_, 0, 8 * sizeof(int)));
          const std::string f = fname_[uk.fid[w[1]]];
          const std::string k = "kernel '" + name + "': ";
          switch (w[0]) {  // executor.hpp:153-172
            case 1: throw error(SF_ERR_EXEC, k + "read of write-only binding '" + f + "'");
            case 2: throw error(SF_ERR_EXEC, k + "non-center read of in-place binding '" + f + "'");
            case 3:
              throw error(SF_ERR_EXEC, k + "read offset (" + std::to_string(w[2]) + "," + std::to_string(w[3]) + "," +
                                           std::to_string(w[4]) + ") outside the declared stencil of '" + f + "'");
            default: throw error(SF_ERR_EXEC, k + "store to read-only binding '" + f + "'");
          }
        }
      }
    }
    // finish_run (executor.hpp:769-779)
    for (size_t b = 0; b < uk.fid.size(); ++b) {
      const bool writable = uk.intent[b] != 0;
      const bool to_back = uk.intent[b] == 3;
      if (reg != SF_REGION_INTERIOR) {
        if (to_back) ctl(CTL_SWAP, 0.0, uk.fid[b], FRONT, BACK);
        if (writable) ghosts_ok_[fname_[uk.fid[b]]] = false;
      } else if (writable && !to_back) {
        ghosts_ok_[fname_[uk.fid[b]]] = false;
      }
    }
  }

  // tensor maps [block][cached binding][physical buffer] for the TMA template
  void build_user_maps(user_kernel& uk) {
    download_table();
    const size_t n = (size_t)nloc_ * uk.cslot.size() * kSlots;
    std::vector<unsigned char> hm(n * 128, 0);
    for (int b = 0; b < nloc_; ++b)
      for (size_t c = 0; c < uk.cslot.size(); ++c) {
        const int f = uk.fid[uk.cslot[c]];
        for (int sl = 0; sl < kSlots; ++sl) {
          // the buffer whose physical index is sl (slots permute on swaps)
          double* p = nullptr;
          for (int q = 0; q < kSlots; ++q)
            if (htab_->ptr[b][f][q] && htab_->bidx[b][f][q] == sl) p = htab_->ptr[b][f][q];
          if (!p) continue;
          const sf_layout& L = lay_[b];
          if (encode_box_map(hm.data() + 128 * ((b * uk.cslot.size() + c) * kSlots + sl), p, L.sx, L.sy, L.sz,
                             uk.bw, uk.bh, fes_[f]))
            throw error(SF_ERR_CUDA, "cuTensorMapEncodeTiled failed for kernel '" + uk.name + "'");
        }
      }
    if (!uk.maps) uk.maps = dalloc(std::max<size_t>(hm.size(), 128) + 64 * n);
    SF_CK(cudaMemcpy(uk.maps, hm.data(), hm.size(), cudaMemcpyHostToDevice));
    uk.maps_gen = alloc_gen_;
  }

  static bool debug_bounds() {  // executor.hpp:645-648
    const char* e = getenv("SF_DEBUG_BOUNDS");
    return e && *e && std::string(e) != "0";
  }
  void check_ghosts(const user_kernel& k, int reg) const {  // executor.hpp:751-757
    int mh = 0;
    for (int h : k.halo) mh = std::max(mh, h);
    if (mh == 0 || reg == SF_REGION_INTERIOR) return;
    for (size_t b = 0; b < k.fid.size(); ++b)
      if (k.intent[b] != 1 && !ghosts_valid(fname_[k.fid[b]]))
        throw error(SF_ERR_EXEC, "kernel '" + k.name + "' reads ghosts of '" + fname_[k.fid[b]] +
                                     "' that were never exchanged");
  }

  double reduce(int f, int op) {
    if (op == SF_MAX_ABS || op == SF_MAX_ABS_DIFF) {
      if (op == SF_MAX_ABS_DIFF && !has_back(f))
        throw error(SF_ERR_GRID,
                    std::string("field '") + fname_[f] + "' has no back buffer to diff against");
      ctl(CTL_CLEAR_ACC);
      const work_set& ws = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_plain_);
      const int fl[1] = {f};
      launch_reduce_max(tview(ws), ws.nctas, zc_plain_, fl, 1, op == SF_MAX_ABS_DIFF ? 1 : 0,
                        &dctl_->acc[7], st_);
      ++launches_;
      check_launch();
      allreduce_max(&dctl_->acc[7], 1);
      return read_acc(7);
    }
    const work_set& ws = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_plain_);
    double* parts = (double*)dalloc_tmp(sizeof(double) * (size_t)ws.nctas);
    launch_reduce_sum(tview(ws), ws.nctas, zc_plain_, f, op == SF_SUM_SQ ? 1 : 0, parts, st_);
    ++launches_;
    check_launch();
    std::vector<double> hp(ws.nctas);
    SF_CK(cudaMemcpyAsync(hp.data(), parts, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, st_));
    sync();
    SF_CK(cudaFree(parts));
    double acc = 0.0;
    for (double x : hp) acc += x;
    if (dist_) {  // partials combined in rank order, as reductions.hpp:75-88 does
      double* d = (double*)dalloc_tmp(sizeof(double) * (size_t)(world_ + 1));
      SF_CK(cudaMemcpyAsync(d, &acc, sizeof(double), cudaMemcpyHostToDevice, st_));
      dev_allgather(d, d + 1, 1);
      std::vector<double> all(world_);
      SF_CK(cudaMemcpyAsync(all.data(), d + 1, sizeof(double) * world_, cudaMemcpyDeviceToHost, st_));
      sync();
      SF_CK(cudaFree(d));
      acc = all[0];
      for (int r = 1; r < world_; ++r) acc += all[r];
    }
    return acc;
  }

  // ---- the time step (cfd.hpp:264-316) --------------------------------------
  void compute_dt_device() {
    const work_set& ws = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_plain_);
    const int fl[3] = {SF_VX, SF_VY, SF_VZ};
    ctl(CTL_CLEAR_ACC);
    launch_reduce_max(tview(ws), ws.nctas, zc_plain_, fl, 3, 0, &dctl_->acc[0], st_);
    ++launches_;
    allreduce_max(&dctl_->acc[0], 3);
    ctl(CTL_DT_FROM_ACC);
    check_launch();
  }
  double compute_dt() {
    compute_dt_device();
    sync();
    return hflag_->dt;
  }

  void provisional_device() {
    refresh({SF_VX, SF_VY, SF_VZ, SF_P});
    if (cfd_es_ != 8 && !(uvmaps_ && uv_tma_env_)) throw error(SF_ERR_ARG, "fp32 CFD fields need the TMA UPDATE_VELOCITY");
    if (uvmaps_ && uv_tma_env_) {
      const work_set& ws = items_for(SF_REGION_ALL, {1, 1, 1, 1, 1, 1}, zc_fused_, kTX, kTY);
      launch_update_velocity_tma(tview(ws), ws.nctas, zc_fused_, consts_, dctl_, uvmaps_, st_, cfd_es_);
    } else {
      const work_set& ws = items_for(SF_REGION_ALL, {1, 1, 1, 1, 1, 1}, zc_uv_);
      launch_update_velocity(tview(ws), ws.nctas, zc_uv_, consts_, dctl_, 0.0, st_);
    }
    ++launches_;
    check_launch();
    swap_front_back();
    for (int f : {SF_VX, SF_VY, SF_VZ}) ghosts_ok_[fname_[f]] = false;
    allreduce_max(&dctl_->acc[1], 3);
    ctl(CTL_CHECK_FINITE);
  }
  void check_finite_or_throw() {
    sync();
    const int a = hflag_->abort_field;
    if (a >= 0) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%f", time_);  // std::to_string(double)
      throw error(SF_ERR_CFD, std::string("non-finite ") + fname_[a] +
                                  " after the velocity update at step " + std::to_string(steps_) +
                                  ", t = " + buf);
    }
  }
  void provisional(double dt) {
    ctl(CTL_SET_DT, dt);
    provisional_device();
    check_finite_or_throw();
  }

  // Also re-arms one batched call, which builds any work sets and exchange
  // phases the capture will need (they allocate, which a capture may not).
  void drop_loop_graph() {
    if (loop_exec_) cudaGraphExecDestroy(loop_exec_);
    loop_exec_ = nullptr;
    loop_mode_ = -1;
    pressure_calls_ = 0;
  }
  // The whole pressure loop without the host: a conditional WHILE node runs
  // the body (kUnits units of the device-predicated loop) until the last
  // unit's finalize sets ctl->done. The body is captured from the same
  // enqueue code as the batched path, so both issue identical kernels.
  void build_loop_graph(int mode) {
    constexpr int kUnits = 2;
    drop_loop_graph();
    flush_io();  // no pending transfer events may be waited on inside the capture
    cudaGraph_t g = nullptr;
    SF_CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    SF_CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    SF_CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    SF_CK(cudaStreamBeginCaptureToGraph(st_, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const i64 l0 = launches_;
    capturing_ = true;
    for (int q = 0; q < kUnits; ++q) enqueue_sweep_unit();
    launch_loop_cond(h, dctl_, st_);
    capturing_ = false;
    cudaGraph_t cap = nullptr;
    SF_CK(cudaStreamEndCapture(st_, &cap));
    SF_CK(cudaGraphInstantiate(&loop_exec_, g, 0));
    SF_CK(cudaGraphDestroy(g));
    loop_units_launches_ = launches_ - l0;
    launches_ = l0;
    loop_mode_ = mode;
  }
  i64 loop_units_launches_ = 0;
  // Inside the captured loop no kernel writes the host-mapped flag (a
  // system-scope fence per sweep); CTL_PUBLISH writes it once afterwards.
  bool capturing_ = false;
  sf_host_flag* loop_flag() const { return capturing_ ? nullptr : dflag_; }

  std::pair<int, double> pressure_iteration_device() {
    refresh({SF_VX, SF_VY, SF_VZ});
    const work_set& wd = items_for(SF_REGION_ALL, {1, 0, 1, 0, 1, 0}, zc_plain_);
    launch_divergence(tview(wd), wd.nctas, zc_plain_, consts_, dctl_, -1, 0, st_, cfd_es_);
    ++launches_;
    check_launch();
    if (opt_.fused) refresh({SF_DIVU});
    ctl(CTL_BEGIN_ITERATION);
    if (persistent()) {
      const int zc = zc_persist();
      const work_set& ws = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc);
      SF_CK(launch_pressure_loop(tview(ws), ws.nctas, zc, consts_, dctl_, st_));
      ++launches_;
      ctl(CTL_PUBLISH);
      sync();
      if (hflag_->sweeps > 0) est_sweeps_ = hflag_->sweeps;
      return finish_pressure_iteration();
    }
    const int maxs = std::max(1, cfg_.max_sweeps);
    const bool graph = graph_env_ && !dist_ && !timing_ && pressure_calls_++ > 0;
    if (graph) {
      const int mode = opt_.fused | (temporal() ? 16 : 0);
      if (!loop_exec_ || loop_mode_ != mode) build_loop_graph(mode);
      SF_CK(cudaGraphLaunch(loop_exec_, st_));
      enqueue_redo_after_loop();
      ctl(CTL_PUBLISH);
      sync();
      const int sweeps = hflag_->sweeps;
      // launches the graph ran: bodies of kUnits units, one per 2*kUnits (or kUnits) sweeps
      const int per_body = temporal() ? 4 : 2;
      launches_ += (i64)((sweeps + per_body - 1) / per_body) * (loop_units_launches_ + 1);
      if (sweeps > 0) est_sweeps_ = sweeps;
      return finish_pressure_iteration();
    }
    int issued = 0;
    int batch = std::max(1, std::min(maxs, est_sweeps_));
    const bool two = temporal();
    auto enqueue = [&](int n, cudaEvent_t ev) {
      int c = 0;
      while (c < n) c += enqueue_sweep_unit();
      issued += c;
      SF_CK(cudaEventRecord(ev, st_));
    };
    iter_launch_ = 0;
    enqueue(batch, ev_[0]);
    int cur = 0;
    while (true) {
      bool more = false;
      if (issued < maxs) {
        const int nb = std::min(maxs - issued, batch);
        enqueue(nb, ev_[cur ^ 1]);
        more = true;
        batch = std::min(batch * 2, 4096);
      }
      SF_CK(cudaEventSynchronize(ev_[cur]));
      if (hflag_->done) break;
      if (!more) break;
      cur ^= 1;
    }
    enqueue_redo_after_loop();
    sync();
    const int sweeps = hflag_->sweeps;
    const double residual = hflag_->residual;
    if (sweeps > 0) est_sweeps_ = sweeps;
    if (timing_ && opt_.fused) {
      // the first units ran (a temporal pass covers two half-sweeps, the last
      // one possibly only its first); the rest were predicated off
      const int ran = two ? (sweeps + 1) / 2 : sweeps;
      for (int q = 0; q < ran && q < iter_launch_; ++q) {
        float ms = 0.f;
        SF_CK(cudaEventElapsedTime(&ms, timer(q, 0), timer(q, 1)));
        (two ? pass_ms_ : sweep_ms_) += ms;
        ++(two ? pass_launches_ : sweep_launches_);
        if (two && q < (int)unit_form_.size() && unit_form_[q]) ++interior_passes_;
      }
    }
    (void)residual;
    return finish_pressure_iteration();
  }
  std::pair<int, double> finish_pressure_iteration() {
    const int sweeps = hflag_->sweeps;
    const double residual = hflag_->residual;
    if (opt_.fused) refresh({SF_VX, SF_VY, SF_VZ});
    // ghost state as the reference leaves it (executor.hpp:769-779)
    ghosts_ok_["p"] = false;
    ghosts_ok_["divu"] = false;
    for (int f : {SF_VX, SF_VY, SF_VZ}) ghosts_ok_[fname_[f]] = true;
    return {sweeps, residual};
  }
  std::pair<int, double> pressure_iteration(double dt) {
    ctl(CTL_SET_DT, dt);
    return pressure_iteration_device();
  }

  // The NaN guard after UPDATE_VELOCITY (cfd.hpp:278-281) is read once the
  // pressure loop has synchronised: the loop is predicated off on the device
  // after a non-finite velocity, so no host round trip sits between the two.
  sf_step_stats step() {
    compute_dt_device();
    provisional_device();
    auto r = pressure_iteration_device();
    check_finite_or_throw();
    const double dt = hflag_->dt;
    refresh({SF_P});
    time_ += dt;
    ++steps_;
    last_ = {dt, r.first, r.second};
    return last_;
  }
  sf_step_stats advance(int n) {
    for (int i = 0; i < n; ++i) step();
    return last_;
  }

  // ---- diagnostics (cfd.hpp:342-363) -----------------------------------------
  double max_divergence() {
    refresh({SF_VX, SF_VY, SF_VZ});
    ctl(CTL_CLEAR_ACC);
    const work_set& wd = items_for(SF_REGION_ALL, {1, 0, 1, 0, 1, 0}, zc_plain_);
    launch_divergence(tview(wd), wd.nctas, zc_plain_, consts_, dctl_, 7, 0, st_, cfd_es_);
    ++launches_;
    check_launch();
    allreduce_max(&dctl_->acc[7], 1);
    ghosts_ok_["divu"] = false;
    return read_acc(7);
  }
  // cfd.hpp:347-355: max over vx, vy, vz of max|front - back|. One launch
  // reduces all three into acc[4..6] (exact bit-pattern maxima), combined on
  // the host in the reference's order.
  double steady_delta() {
    for (int f : {SF_VX, SF_VY, SF_VZ})
      if (!has_back(f))
        throw error(SF_ERR_GRID, std::string("field '") + fname_[f] + "' has no back buffer to diff against");
    ctl(CTL_CLEAR_ACC);
    const work_set& ws = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_plain_);
    const int fl[3] = {SF_VX, SF_VY, SF_VZ};
    launch_reduce_max(tview(ws), ws.nctas, zc_plain_, fl, 3, 1, &dctl_->acc[4], st_);
    ++launches_;
    check_launch();
    allreduce_max(&dctl_->acc[4], 3);
    double m[3];
    read_accs(4, 3, m);
    double d = m[0];
    d = d < m[1] ? m[1] : d;  // std::max
    d = d < m[2] ? m[2] : d;
    return d;
  }
  // RMS distance to the decayed analytic vortex (cfd.hpp:367-401). The
  // analytic factors use the host's sin/cos/exp as the reference does; the
  // device evaluates each cell's term with the reference's operations; the
  // host sums them in the reference's order (x-fastest within a worker,
  // workers in order), so the result is bitwise the reference's.
  double taylor_green_error(double t) {
    if (cfd_es_ != 8) throw error(SF_ERR_ARG, "taylor_green_error needs fp64 CFD fields");
    const double tau = 2.0 * 3.14159265358979323846;
    const double decay = std::exp(-2.0 * par_.viscosity * tau * tau * t);
    const double dx = cfg_.spacing[0], dy = cfg_.spacing[1];
    download_table();
    std::vector<std::pair<int, double>> part;  // (worker, partial)
    for (int b = 0; b < nloc_; ++b) {
      const auto& L = lay_[b];
      const sf_dev_block& B = htab_->blk[b];
      const i64 nx = L.dims[0], ny = L.dims[1], nz = L.dims[2];
      std::vector<double> tab(2 * (size_t)(nx * ny));
      for (i64 j = 0; j < ny; ++j)
        for (i64 i = 0; i < nx; ++i) {
          const double xc = (static_cast<double>(B.lo[0] + i) + 0.5) * dx;
          const double yc = (static_cast<double>(B.lo[1] + j) + 0.5) * dy;
          const double xf = static_cast<double>(B.lo[0] + i + 1) * dx;
          const double yf = static_cast<double>(B.lo[1] + j + 1) * dy;
          tab[j * nx + i] = std::sin(tau * xf) * std::cos(tau * yc);
          tab[nx * ny + j * nx + i] = std::cos(tau * xc) * std::sin(tau * yf);
        }
      double* dtabv = (double*)dalloc_tmp(sizeof(double) * tab.size());
      SF_CK(cudaMemcpyAsync(dtabv, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice, st_));
      const i64 dims[3] = {nx, ny, nz};
      double* out = staging();
      launch_tg_cells(htab_->ptr[b][SF_VX][FRONT], htab_->ptr[b][SF_VY][FRONT], htab_->ptr[b][SF_VZ][FRONT],
                      L.base, L.sx, L.sy, dims, dtabv, dtabv + nx * ny, decay, out, st_);
      ++launches_;
      check_launch();
      std::vector<double> cellv((size_t)(nx * ny * nz));
      SF_CK(cudaMemcpyAsync(cellv.data(), out, sizeof(double) * cellv.size(), cudaMemcpyDeviceToHost, st_));
      sync();
      SF_CK(cudaFree(dtabv));
      double sum = 0.0;
      for (double x : cellv) sum += x;
      part.push_back({gid_[b], sum});
    }
    std::vector<double> all;
    if (dist_) {  // one block per rank: gather the partials, combine in rank (= worker) order
      double* d = (double*)dalloc_tmp(sizeof(double) * (size_t)(world_ + 1));
      SF_CK(cudaMemcpyAsync(d, &part[0].second, sizeof(double), cudaMemcpyHostToDevice, st_));
      dev_allgather(d, d + 1, 1);
      all.resize(world_);
      SF_CK(cudaMemcpyAsync(all.data(), d + 1, sizeof(double) * world_, cudaMemcpyDeviceToHost, st_));
      sync();
      SF_CK(cudaFree(d));
    } else {
      std::sort(part.begin(), part.end());
      for (const auto& p : part) all.push_back(p.second);
    }
    double total = 0.0;
    for (double x : all) total += x;
    const double n = static_cast<double>(cells());
    return std::sqrt(total / (3.0 * n));
  }
  double kinetic_energy() {
    const double s = reduce(SF_VX, SF_SUM_SQ) + reduce(SF_VY, SF_SUM_SQ) + reduce(SF_VZ, SF_SUM_SQ);
    const double cell = cfg_.spacing[0] * cfg_.spacing[1] * cfg_.spacing[2];
    return 0.5 * par_.density * s * cell;
  }

  double time() const { return time_; }
  long steps() const { return steps_; }
  int pending_color() {
    sync();
    return hflag_->color;
  }
  bool ghosts_valid(const std::string& f) const {
    auto it = ghosts_ok_.find(f);
    return it != ghosts_ok_.end() && it->second;
  }
  void invalidate(const std::string& f) { ghosts_ok_[f] = false; }
  void invalidate_all() { ghosts_ok_.clear(); }
  cudaStream_t stream() const { return st_; }
  i64 launch_count(bool reset) {
    const i64 n = launches_;
    if (reset) launches_ = 0;
    return n;
  }
  void set_timing(bool on) {
    timing_ = on;
    sweep_ms_ = pass_ms_ = 0.0;
    sweep_launches_ = pass_launches_ = interior_passes_ = 0;
  }
  // which = 0: single half-sweep kernel; 1: temporal pass (two half-sweeps)
  // which: 0 single half-sweeps, 1 temporal passes, 2 the passes among them
  // that ran on the interior form (k_sweep2i beside the slabs; count only)
  void timing(int which, double* ms, i64* n) const {
    *ms = which == 1 ? pass_ms_ : which == 0 ? sweep_ms_ : 0.0;
    *n = which == 1 ? pass_launches_ : which == 0 ? sweep_launches_ : interior_passes_;
  }

 private:
  struct work_set {
    sf_work* d = nullptr;
    int n = 0;
    int nctas = 0;
  };
  struct task_set {
    sf_task* d = nullptr;
    int n = 0;
    i64 max_count = 0;
  };

  sf_solver_config cfg_;
  sf_fluid_params par_;
  sf_sim_options opt_;
  std::map<std::string, user_kernel> ukernels_;
  long long alloc_gen_ = 0;  // bumps on every buffer allocation (TMA maps go stale)
  int* dbg_word_ = nullptr;  // debug policing: {code, slot, di, dj, dk}
  void* geo_ = nullptr;  // per local block: n[3], lo[3], sx, sy, base (sf_jit.hpp sf_geo)
  std::vector<std::string> fname_ = {"vx", "vy", "vz", "p", "divu"};
  std::vector<int> fstag_ = {0, 1, 2, -1, -1};  // stagger per field (field.hpp:23)
  std::vector<int> fes_ = {8, 8, 8, 8, 8};       // bytes per value per field (user fields: 8 or 4)
  int rank_ = 0, world_ = 1;
  int cfd_es_ = 8;     // bytes per value of the five CFD fields (4: the fp32 variant)
  bool dist_ = false;  // NCCL transport (one grid component per rank)
  decomposition dec_;
  int nloc_ = 0;
  std::vector<int> gid_;    // local block -> global worker id
  std::vector<int> lid_;    // global worker id -> local block, or -1
  std::vector<int> owner_;  // global worker id -> rank
  nccl_comm_t comm_ = nullptr;
  enum { TR_NONE = 0, TR_NCCL = 1, TR_IPC = 2 };
  int tr_ = TR_NONE;         // how ranks talk: NCCL, or CUDA IPC + host callbacks
  sf_host_transport htr_{};
  std::map<std::string, void*> ipc_open_;  // peer allocations mapped here, by handle
  // the temporal pass's exchange as direct stores into the peers' arrays
  // sf_sim_set_direct_exchange: 1 = fused into the pass (default), 2 = one
  // separate launch of direct stores after it, 0 = exchange phases
  int direct_mode_ = 1;
  sweep2_remote* remote_ = nullptr;  // device table of the fused exchange
  int direct_state_ = 0;    // 0 not set up, 1 active, -1 unavailable (a peer is not mappable)
  struct task_set_ref {
    sf_task* d = nullptr;
    int n = 0;
    i64 max_count = 0;
  } direct_tasks_;
  sf_face_bc bc_[6]{};
  sf_consts consts_{};
  std::vector<sf_layout> lay_;
  cudaStream_t st_ = nullptr;
  cudaEvent_t ev_[2]{}, t0_{}, t1_{};
  std::unique_ptr<sf_dev_table> htab_;
  sf_dev_table* dtab_ = nullptr;
  sf_dev_ctl* dctl_ = nullptr;
  sf_host_flag* hflag_ = nullptr;
  sf_host_flag* dflag_ = nullptr;
  double* staging_ = nullptr;
  void* maps_ = nullptr;  // TMA descriptors (null: no driver entry point -> LDG kernel)
  cudaStream_t io_[2]{};    // host transfers: 0 uploads, 1 downloads
  cudaEvent_t io_ev_[kMaxFields]{};  // last download of each field
  cudaEvent_t io_up_[kMaxFields]{};  // last upload of each field
  cudaEvent_t io_snap_[kMaxFields]{};    // last snapshot (pack) of each field for a background download
  cudaEvent_t io_snapdn_[kMaxFields]{};  // last background download out of each snapshot buffer
  double* snap_[kMaxBlocks][kMaxFields]{};
  double* upb_[kMaxBlocks][kMaxFields]{};   // dense upload buffers of the asynchronous scatter
  cudaEvent_t io_inst_[kMaxFields]{};
  bool staged_[kMaxBlocks][kMaxFields]{};  // an upload is staged, not yet installed       // last install out of each upload buffer
  mutable std::vector<cudaEvent_t> io_pending_;  // not yet ordered before compute
  // compute enqueues so far / at the last table download: block_io skips the
  // download (a copy that would queue behind large transfers) when equal
  mutable unsigned long long compute_epoch_ = 1;
  unsigned long long table_epoch_ = 0;
  void* maps2_ = nullptr;  // temporal-pass descriptors (null: pass unavailable)
  void* maps3_ = nullptr;  // descriptors of the interior form of the pass (sweep2i_box shapes)
  void* maps4_ = nullptr;  // descriptors of the pass's x-slab form (sweep2_box shape 1)
  int ibzc_ = 32;          // z chunk of the boundary slabs beside the interior form
  const bool interior_env_ = getenv("SF_NO_INTERIOR_PASS") == nullptr;
  void* uvmaps_ = nullptr;  // TMA UPDATE_VELOCITY descriptors (null: plain-load kernel)
  cudaStream_t xs_ = nullptr;  // halo exchange overlapped with the temporal pass
  const bool overlap_env_ = getenv("SF_NO_OVERLAP") == nullptr;
  const bool force_overlap_ = getenv("SF_OVERLAP") != nullptr;  // also on one device (tests)
  work_set empty_ws_{};
  cudaEvent_t ev_fork_{}, ev_join_{};
  const bool uv_tma_env_ = getenv("SF_NO_UV_TMA") == nullptr;
  const bool temporal_env_ = getenv("SF_NO_TEMPORAL") == nullptr;
  const int persist_env_ = getenv("SF_PERSIST") ? atoi(getenv("SF_PERSIST")) : -1;
  const double persist_cells_ = getenv("SF_PERSIST_CELLS") ? atof(getenv("SF_PERSIST_CELLS")) : 4.0e5;
  const int zc_persist_env_ = getenv("SF_PZC") ? atoi(getenv("SF_PZC")) : 0;
  // z chunk of the persistent loop: about one tile per co-resident CTA
  int zc_persist() const {
    if (zc_persist_env_ > 0) return zc_persist_env_;
    const sf_dev_block& B = htab_->blk[0];
    const i64 cols = ((B.n[0] + kTX - 1) / kTX) * ((B.n[1] + kTY - 1) / kTY);
    const i64 ctas = pressure_loop_ctas();
    return (int)std::max<i64>(1, (B.n[2] * cols + ctas - 1) / ctas);
  }
  std::vector<void*> dev_allocs_;
  std::map<std::string, work_set> items_;
  std::map<std::string, task_set> tasks_;
  task_set divu_faces_;
  bool divu_faces_built_ = false;
  std::map<std::string, bool> ghosts_ok_;
  double time_ = 0.0;
  long steps_ = 0;
  sf_step_stats last_{0.0, 0, 0.0};
  int est_sweeps_ = 8;
  // pressure loop as one CUDA graph: a while node whose body is kUnits sweep
  // units and the condition kernel (single process, no per-launch timing)
  cudaGraphExec_t loop_exec_ = nullptr;
  int loop_mode_ = -1;  // fused mode | temporal << 4 the graph was built for
  long pressure_calls_ = 0;
  const bool graph_env_ = getenv("SF_NO_GRAPH") == nullptr;
  i64 launches_ = 0;
  bool timing_ = false;
  double sweep_ms_ = 0.0, pass_ms_ = 0.0;
  i64 sweep_launches_ = 0, pass_launches_ = 0, interior_passes_ = 0;
  std::vector<char> unit_form_;  // (timing) per timed unit: 1 = the interior form ran
  void mark_form(int q, char f) {
    if (!timing_) return;
    if ((int)unit_form_.size() <= q) unit_form_.resize((size_t)q + 1, 0);
    unit_form_[(size_t)q] = f;
  }
  std::vector<cudaEvent_t> timers_;
  int iter_launch_ = 0;
  cudaEvent_t timer(int q, int which) {
    while ((int)timers_.size() < 2 * (q + 1)) {
      cudaEvent_t e;
      SF_CK(cudaEventCreate(&e));
      timers_.push_back(e);
    }
    return timers_[2 * q + which];
  }
  const int zc_plain_ = 16;
  const int zc_uv_ = 8;
  const int zc_fused_ = getenv("SF_ZC") ? atoi(getenv("SF_ZC")) : 64;
  // z chunk of the temporal pass: longer chunks amortise its 3 prologue planes
  // (512^3: 2.64 ms at 64, 2.59 ms at 128, 2.61 ms at 256)
  const int zc_pass_env_ = getenv("SF_ZC2") ? atoi(getenv("SF_ZC2")) : 0;
  int zc_pass_cache_ = 0;
  int sms_ = 0;
  // z chunk of the temporal pass: 128 planes (fewer pipeline prologues) unless
  // that leaves fewer than about two waves of CTAs (2 per SM), then halved
  // down to 16 (a 128^3 grid has only 64 column tiles)
  int zc_pass() {
    if (zc_pass_env_ > 0) return zc_pass_env_;
    if (zc_pass_cache_) return zc_pass_cache_;
    if (!sms_) SF_CK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, opt_.device));
    const int ty = sweep2_tile_y();
    i64 cols = 0, nz = 1;
    for (int b = 0; b < nloc_; ++b) {
      const sf_dev_block& B = htab_->blk[b];
      cols += ((B.n[0] + kTX - 1) / kTX) * ((B.n[1] + ty - 1) / ty);
      nz = std::max<i64>(nz, B.n[2]);
    }
    int zc = 128;
    while (zc > 16 && cols * ((nz + zc - 1) / zc) < (i64)4 * sms_) zc /= 2;
    return zc_pass_cache_ = zc;
  }

  void validate() {
    // solver_config::validate / fluid_params::validate (cfd.hpp:36-66)
    for (int a = 0; a < 3; ++a) {
      if (cfg_.extents[a] < 1) throw error(SF_ERR_CONFIG, "domain extents must be positive");
      if (!(cfg_.spacing[a] > 0.0)) throw error(SF_ERR_CONFIG, "grid spacing must be positive");
    }
    if (!(cfg_.reynolds > 0.0)) throw error(SF_ERR_CONFIG, "Reynolds number must be positive");
    if (!(cfg_.sigma > 0.0 && cfg_.sigma < 1.0)) throw error(SF_ERR_CONFIG, "sigma must lie in (0,1)");
    if (!(cfg_.tolerance > 0.0)) throw error(SF_ERR_CONFIG, "pressure tolerance must be positive");
    if (!(cfg_.omega >= 1.0 && cfg_.omega < 2.0)) throw error(SF_ERR_CONFIG, "omega must lie in [1,2)");
    if (cfg_.max_sweeps < 1) throw error(SF_ERR_CONFIG, "max_sweeps must be at least 1");
    if (!(par_.viscosity > 0.0)) throw error(SF_ERR_CONFIG, "viscosity must be positive");
    if (!(par_.density > 0.0)) throw error(SF_ERR_CONFIG, "density must be positive");
    if (!(par_.blend >= 0.0 && par_.blend <= 1.0)) throw error(SF_ERR_CONFIG, "blend must lie in [0,1]");
    if (opt_.ghost < 1)
      throw error(SF_ERR_EXEC, "kernel 'UPDATE_VELOCITY': stencil needs 1 ghost layers but fields carry " +
                                   std::to_string(opt_.ghost));
  }

  void make_bc() {  // cfd.hpp:500-512
    for (int axis = 0; axis < 3; ++axis) {
      if (cfg_.periodic[axis]) continue;
      for (int side = 0; side < 2; ++side) bc_[2 * axis + side] = {SF_BC_WALL, {0, 0, 0}};
    }
    if (!cfg_.periodic[1]) bc_[3] = {SF_BC_WALL, {par_.lid_speed, 0.0, 0.0}};
    if (!cfg_.periodic[2] && cfg_.symmetry_z) {
      bc_[4] = {SF_BC_SYMMETRY, {0, 0, 0}};
      bc_[5] = {SF_BC_SYMMETRY, {0, 0, 0}};
    }
  }

  void make_consts() {  // cfd.hpp:192-217
    sf_consts& s = consts_;
    s.nu = par_.viscosity;
    s.alpha = par_.blend;
    s.fx = par_.body_force[0];
    s.fy = par_.body_force[1];
    s.fz = par_.body_force[2];
    s.ix = 1.0 / cfg_.spacing[0];
    s.iy = 1.0 / cfg_.spacing[1];
    s.iz = 1.0 / cfg_.spacing[2];
    s.ix2 = s.ix * s.ix;
    s.iy2 = s.iy * s.iy;
    s.iz2 = s.iz * s.iz;
    for (int a = 0; a < 3; ++a) {
      s.nm1[a] = cfg_.extents[a] - 1;
      s.N[a] = cfg_.extents[a];
      s.per[a] = cfg_.periodic[a] ? 1 : 0;
      s.spacing[a] = cfg_.spacing[a];
    }
    auto act = [&](double ax, double ay, double az) { return ax * s.ix2 + ay * s.iy2 + az * s.iz2; };
    for (int bx = 0; bx < 2; ++bx)
      for (int by = 0; by < 2; ++by)
        for (int bz = 0; bz < 2; ++bz)
          s.bscale[bx][by][bz] = act(2.0, 2.0, 2.0) / act(bx ? 2.0 : 1.0, by ? 2.0 : 1.0, bz ? 2.0 : 1.0);
    s.sigma = cfg_.sigma;
    s.omega = cfg_.omega;
    s.tolerance = cfg_.tolerance;
    s.max_sweeps = cfg_.max_sweeps;
  }

  void* dalloc(size_t bytes) {
    void* p = nullptr;
    SF_CK(cudaMalloc(&p, bytes));
    dev_allocs_.push_back(p);
    return p;
  }
  void* dalloc_tmp(size_t bytes) {
    void* p = nullptr;
    SF_CK(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
    return p;
  }

  void allocate() {
    htab_ = std::make_unique<sf_dev_table>();
    for (int f = 0; f < kMaxFields; ++f) htab_->esize[f] = 8;
    std::memset(htab_.get(), 0, sizeof(sf_dev_table));
    htab_->nblocks = nloc_;
    for (int f = 0; f < SF_NFIELDS; ++f) htab_->esize[f] = (unsigned char)cfd_es_;
    lay_.resize(nloc_);
    for (int b = 0; b < nloc_; ++b) {
      const int gw = gid_[b];
      const auto dims = dec_.dims(gw);
      const i64 lo[3] = {dec_.lo[gw][0], dec_.lo[gw][1], dec_.lo[gw][2]};
      const i64 dd[3] = {dims[0], dims[1], dims[2]};
      lay_[b] = make_layout(dd, lo, dec_.ghost);
      const sf_layout& L = lay_[b];
      sf_dev_block& B = htab_->blk[b];
      for (int a = 0; a < 3; ++a) {
        B.n[a] = L.dims[a];
        B.lo[a] = L.lo[a];
      }
      B.sx = L.sx;
      B.sy = L.sy;
      B.sz = L.sz;
      B.base = L.base;
      B.g = L.ghost;
      for (int a = 0; a < 3; ++a)
        for (int side = 0; side < 2; ++side) {
          const int fi = 2 * a + side;
          const int nb = dec_.neighbor(gw, a, side);
          if (nb < 0) {
            const int k = bc_[fi].kind;
            B.face[fi] = k == SF_BC_WALL ? FACE_WALL
                         : k == SF_BC_SYMMETRY ? FACE_SYM
                         : k == SF_BC_OUTFLOW ? FACE_OUT : FACE_WALL;
          } else {
            B.face[fi] = nb == gw ? FACE_SELF : FACE_PROC;
          }
          for (int c = 0; c < 3; ++c) B.fvel[fi][c] = bc_[fi].velocity[c];
          const i64 N = cfg_.extents[a];
          B.nb_ghost_gidx[fi] = side == 0 ? (L.lo[a] - 1 + N) % N : (L.lo[a] + L.dims[a]) % N;
        }
      for (int f = 0; f < SF_NFIELDS; ++f) {
        const bool velocity = f <= SF_VZ;
        for (int s = 0; s < kSlots; ++s) {
          // p gets an ALT buffer for the temporal pass (sf_sweep2.cu)
          const bool need = s == FRONT || (velocity && (s == BACK || s == ALT)) ||
                            (f == SF_DIVU && s == ALT) || (f == SF_P && s == ALT);
          if (need) alloc_slot(b, f, s);
        }
      }
    }
    // TMA descriptors of every physical buffer the fused half-sweep reads
    {
      std::vector<unsigned char> hm(sweep_maps_bytes(), 0);
      bool ok = true;
      for (int b = 0; b < nloc_ && ok; ++b)
        for (int f = 0; f < SF_NFIELDS && ok; ++f)
          for (int s = 0; s < kSlots && ok; ++s) {
            double* p = htab_->ptr[b][f][s];
            if (!p) continue;
            const sf_layout& L = lay_[b];
            ok = encode_sweep_map(hm.data() + sweep_map_offset(b, f, s), p, L.sx, L.sy, L.sz, f, fes_[f]) == 0;
          }
      if (ok) {
        maps_ = dalloc(hm.size());
        SF_CK(cudaMemcpy(maps_, hm.data(), hm.size(), cudaMemcpyHostToDevice));
      }
    }
    // descriptors of the TMA-staged UPDATE_VELOCITY
    if (maps_) {
      std::vector<unsigned char> hm(uv_maps_bytes(), 0);
      bool ok = true;
      const int uvf[4] = {SF_VX, SF_VY, SF_VZ, SF_P};
      for (int b = 0; b < nloc_ && ok; ++b)
        for (int k = 0; k < 4 && ok; ++k)
          for (int s = 0; s < kSlots && ok; ++s) {
            double* p = htab_->ptr[b][uvf[k]][s];
            if (!p) continue;
            const sf_layout& L = lay_[b];
            int bw, bh;
            uv_box(uvf[k], &bw, &bh, fes_[uvf[k]]);
            ok = bw <= L.sx && bh <= L.sy &&
                 encode_box_map(hm.data() + uv_map_offset(b, k, s), p, L.sx, L.sy, L.sz, bw, bh, fes_[uvf[k]]) == 0;
          }
      if (ok) {
        uvmaps_ = dalloc(hm.size());
        SF_CK(cudaMemcpy(uvmaps_, hm.data(), hm.size(), cudaMemcpyHostToDevice));
      }
    }
    // descriptors of the temporal pass (halo'd boxes)
    if (maps_) {
      std::vector<unsigned char> hm(sweep2_maps_bytes(), 0);
      bool ok = true;
      for (int b = 0; b < nloc_ && ok; ++b)
        for (int f : {SF_VX, SF_VY, SF_VZ, SF_P, SF_DIVU})
          for (int s = 0; s < kSlots && ok; ++s) {
            double* p = htab_->ptr[b][f][s];
            if (!p) continue;
            const sf_layout& L = lay_[b];
            int bw, bh;
            sweep2_box(f, &bw, &bh, fes_[f]);
            ok = bw <= L.sx && bh <= L.sy &&
                 encode_box_map(hm.data() + sweep2_map_offset(b, f, s), p, L.sx, L.sy, L.sz, bw, bh, fes_[f]) == 0;
          }
      if (ok) {
        maps2_ = dalloc(hm.size());
        SF_CK(cudaMemcpy(maps2_, hm.data(), hm.size(), cudaMemcpyHostToDevice));
      }
    }
    // descriptors of the interior form of the pass (one component)
    if (maps2_ && nloc_ == 1) {
      std::vector<unsigned char> hm(sweep2_maps_bytes(), 0);
      bool ok = true;
      for (int f : {SF_VX, SF_VY, SF_VZ, SF_P, SF_DIVU})
        for (int s = 0; s < kSlots && ok; ++s) {
          double* p = htab_->ptr[0][f][s];
          if (!p) continue;
          const sf_layout& L = lay_[0];
          int bw, bh;
          sweep2i_box(f, &bw, &bh, cfd_es_);
          ok = bw <= L.sx && bh <= L.sy &&
               encode_box_map(hm.data() + sweep2_map_offset(0, f, s), p, L.sx, L.sy, L.sz, bw, bh, cfd_es_) == 0;
        }
      if (ok) {
        maps3_ = dalloc(hm.size());
        SF_CK(cudaMemcpy(maps3_, hm.data(), hm.size(), cudaMemcpyHostToDevice));
      }
      hm.assign(sweep2_maps_bytes(), 0);
      for (int f : {SF_VX, SF_VY, SF_VZ, SF_P, SF_DIVU})
        for (int s = 0; s < kSlots && ok; ++s) {
          double* p = htab_->ptr[0][f][s];
          if (!p) continue;
          const sf_layout& L = lay_[0];
          int bw, bh;
          sweep2_box(f, &bw, &bh, cfd_es_, 1);
          ok = bw <= L.sx && bh <= L.sy &&
               encode_box_map(hm.data() + sweep2_map_offset(0, f, s), p, L.sx, L.sy, L.sz, bw, bh, cfd_es_) == 0;
        }
      if (ok) {
        maps4_ = dalloc(hm.size());
        SF_CK(cudaMemcpy(maps4_, hm.data(), hm.size(), cudaMemcpyHostToDevice));
      }
    }
    {
      std::vector<long long> geo;
      for (int b = 0; b < nloc_; ++b) {
        const sf_layout& L = lay_[b];
        for (int a = 0; a < 3; ++a) geo.push_back(L.dims[a]);
        for (int a = 0; a < 3; ++a) geo.push_back(L.lo[a]);
        geo.push_back(L.sx);
        geo.push_back(L.sy);
        geo.push_back(L.base);
      }
      geo_ = dalloc(sizeof(long long) * geo.size());
      SF_CK(cudaMemcpy(geo_, geo.data(), sizeof(long long) * geo.size(), cudaMemcpyHostToDevice));
    }
    dtab_ = (sf_dev_table*)dalloc(sizeof(sf_dev_table));
    SF_CK(cudaMemcpyAsync(dtab_, htab_.get(), sizeof(sf_dev_table), cudaMemcpyHostToDevice, st_));
    dctl_ = (sf_dev_ctl*)dalloc(sizeof(sf_dev_ctl));
    SF_CK(cudaMemsetAsync(dctl_, 0, sizeof(sf_dev_ctl), st_));
    SF_CK(cudaHostAlloc((void**)&hflag_, sizeof(sf_host_flag), cudaHostAllocMapped));
    std::memset((void*)hflag_, 0, sizeof(sf_host_flag));
    SF_CK(cudaHostGetDevicePointer((void**)&dflag_, (void*)hflag_, 0));
    sync();
  }

  // flush = false: wait for enqueued compute only, without first ordering the
  // compute stream after pending host transfers (block_io)
  void download_table(bool flush = true) {
    if (!flush && table_epoch_ == compute_epoch_) return;  // nothing enqueued since the last download
    if (flush)
      sync();
    else
      SF_CK(cudaStreamSynchronize(st_));
    SF_CK(cudaMemcpy(htab_->ptr, dtab_->ptr, sizeof(htab_->ptr), cudaMemcpyDeviceToHost));
    SF_CK(cudaMemcpy(htab_->bidx, dtab_->bidx, sizeof(htab_->bidx), cudaMemcpyDeviceToHost));
    table_epoch_ = compute_epoch_;
  }
  void upload_table() {
    SF_CK(cudaMemcpy(dtab_->ptr, htab_->ptr, sizeof(htab_->ptr), cudaMemcpyHostToDevice));
    SF_CK(cudaMemcpy(dtab_->bidx, htab_->bidx, sizeof(htab_->bidx), cudaMemcpyHostToDevice));
    SF_CK(cudaMemcpy(dtab_->esize, htab_->esize, sizeof(htab_->esize), cudaMemcpyHostToDevice));
  }
  int field_esize(int f) const { return fes_[f]; }
  void alloc_slot(int b, int f, int s) {
    const sf_layout& L = lay_[b];
    const size_t bytes = (size_t)fes_[f] * (size_t)(L.sx * L.sy * L.sz);
    double* p = (double*)dalloc(bytes);
    SF_CK(cudaMemsetAsync(p, 0, bytes, st_));
    htab_->ptr[b][f][s] = p;
    htab_->bidx[b][f][s] = (unsigned char)s;
    ++alloc_gen_;
  }

  table_view tview() const {
    flush_io();
    return table_view{dtab_, nullptr, 0};
  }
  table_view tview(const work_set& w) const {
    flush_io();
    return table_view{dtab_, w.d, w.n};
  }
  // Compute enqueued from here on waits for the pending host transfers
  // (uploads it must read, downloads of fields it may overwrite).
  void flush_io() const {
    ++compute_epoch_;  // called before every compute enqueue: the table may change
    for (cudaEvent_t e : io_pending_) SF_CK(cudaStreamWaitEvent(st_, e, 0));
    io_pending_.clear();
  }

  void ctl(int op, double arg = 0.0, int f = 0, int a = 0, int b = 0, int predicated = 0) {
    flush_io();
    launch_ctl(dtab_, dctl_, loop_flag(), op, arg, f, a, b, consts_, predicated, st_);
    ++launches_;
  }

  void swap_front_back() {
    for (int f : {SF_VX, SF_VY, SF_VZ}) ctl(CTL_SWAP, 0.0, f, FRONT, BACK);
  }

  void read_accs(int slot, int n, double* out) {
    sync();
    unsigned long long bits[8];
    SF_CK(cudaMemcpy(bits, &dctl_->acc[slot], sizeof(bits[0]) * (size_t)n, cudaMemcpyDeviceToHost));
    for (int q = 0; q < n; ++q) {
      if (bits[q] > 0x7ff0000000000000ull) {
        out[q] = std::nan("");
      } else {
        std::memcpy(&out[q], &bits[q], sizeof(double));
      }
    }
  }
  double read_acc(int slot) {
    sync();
    unsigned long long bits = 0;
    SF_CK(cudaMemcpy(&bits, &dctl_->acc[slot], sizeof(bits), cudaMemcpyDeviceToHost));
    if (bits > 0x7ff0000000000000ull) return std::nan("");
    double v;
    std::memcpy(&v, &bits, sizeof v);
    return v;
  }

  const work_set& items_for(int reg, const std::array<int, 6>& halo, int zc, int tx = kTX,
                            int ty = kTY) {
    char key[160];
    std::snprintf(key, sizeof key, "%d:%d,%d,%d,%d,%d,%d:%d:%d:%d", reg, halo[0], halo[1], halo[2],
                  halo[3], halo[4], halo[5], zc, tx, ty);
    auto it = items_.find(key);
    if (it != items_.end()) return it->second;
    std::vector<sf_work> v;
    int cta = 0;
    for (int b = 0; b < nloc_; ++b) {
      const auto dims = dec_.dims(gid_[b]);
      for (const auto& bx : region_boxes(dims, halo, reg)) {
        sf_work w{};
        w.blk = b;
        w.cta_begin = cta;
        for (int a = 0; a < 3; ++a) {
          w.lo[a] = bx[a];
          w.hi[a] = bx[3 + a];
        }
        w.tiles[0] = (int)((w.hi[0] - w.lo[0] + tx - 1) / tx);
        w.tiles[1] = (int)((w.hi[1] - w.lo[1] + ty - 1) / ty);
        w.tiles[2] = (int)((w.hi[2] - w.lo[2] + zc - 1) / zc);
        cta += w.tiles[0] * w.tiles[1] * w.tiles[2];
        v.push_back(w);
      }
    }
    work_set ws;
    ws.n = (int)v.size();
    ws.nctas = cta;
    if (!v.empty()) {
      ws.d = (sf_work*)dalloc(sizeof(sf_work) * v.size());
      SF_CK(cudaMemcpy(ws.d, v.data(), sizeof(sf_work) * v.size(), cudaMemcpyHostToDevice));
    }
    return items_.emplace(key, ws).first->second;
  }

  void validate_bc(const std::vector<int>& fields) const {  // exchange.hpp:86-95
    for (int axis = 0; axis < 3; ++axis) {
      if (cfg_.periodic[axis]) continue;
      for (int side = 0; side < 2; ++side)
        if (bc_[2 * axis + side].kind == SF_BC_UNSET && !fields.empty())
          throw error(SF_ERR_GRID, std::string("field '") + fname_[fields.front()] +
                                       "': no boundary condition on axis " + std::to_string(axis) +
                                       (side == 0 ? " low" : " high") + " face");
    }
  }

  // One phase of exchanger::refresh_worker (exchange.hpp:107-119) on device:
  // launch 1 = copies between local blocks + bc_face fills + packs of the
  // messages to other ranks; then one NCCL group of per-peer send/recv; then
  // launch 2 = unpacks.  All work of launch 1 is independent (disjoint writes;
  // reads of owned cells and of ghosts filled by earlier phases).
  struct phase {
    task_set first;   // copies + bcs + packs
    task_set unpack;
    struct msg {
      int peer;
      long long off, count;
    };
    std::vector<msg> sends, recvs;
    double* sbuf = nullptr;
    double* rbuf = nullptr;
    // CUDA-IPC transport: the peer's send buffer (mapped) at the offset of the
    // message for this rank, per receive; set up collectively on first use
    mutable bool x_ready = false, x_any = false;
    mutable std::vector<const double*> x_src;
  };
  std::map<std::string, phase> phases_;

  task_set upload_tasks(const std::vector<sf_task>& v) {
    task_set ts;
    ts.n = (int)v.size();
    for (const auto& t : v) ts.max_count = std::max(ts.max_count, t.count);
    if (!v.empty()) {
      ts.d = (sf_task*)dalloc(sizeof(sf_task) * v.size());
      SF_CK(cudaMemcpy(ts.d, v.data(), sizeof(sf_task) * v.size(), cudaMemcpyHostToDevice));
    }
    return ts;
  }

  static sf_task task_of(const plan_box& p, int type) {
    sf_task t{};
    t.type = type;
    t.field = p.field;
    t.axis = p.axis;
    t.side = p.side;
    t.src_blk = p.blk;
    t.dst_blk = type == 0 ? p.dst_blk : p.blk;
    for (int a = 0; a < 3; ++a) {
      t.lo[a] = p.lo[a];
      t.dims[a] = p.dims[a];
      t.dlo[a] = p.dlo[a];
    }
    t.count = p.count;
    return t;
  }

  // axis >= 0: refresh/exchange phase of that axis (slabs widened over earlier
  // axes).  axis < 0: the fused loop's divu faces, all axes, owned tangential
  // ranges, no physical fills (the half-sweep writes those itself).
  const phase& phase_for(unsigned mask, int axis, int scope, bool exchange_only, bool bc_only = false) {
    char key[64];
    std::snprintf(key, sizeof key, "%u:%d:%d:%d:%d", mask, axis, scope, exchange_only ? 1 : 0, bc_only ? 1 : 0);
    auto it = phases_.find(key);
    if (it != phases_.end()) return it->second;
    const bool faces = axis < 0;
    const std::vector<int> axes = faces ? std::vector<int>{0, 1, 2} : std::vector<int>{axis};
    phase_plan P = build_phase_plan(dec_, gid_, lid_, owner_, mask, axes, !faces, exchange_only, faces);
    if (bc_only) {  // executor::physical_bc: no exchange at all
      P.copies.clear();
      P.sends.clear();
      P.recvs.clear();
    }
    phase ph;
    std::vector<sf_task> first, unpack;
    for (const auto& c : P.copies) first.push_back(task_of(c, 0));
    for (const auto& b : P.bcs) {
      sf_task t = task_of(b, 1);
      const sf_face_bc& fb = bc_[2 * b.axis + b.side];
      t.kind = fb.kind;
      t.scope = scope;
      t.normal = fstag_[b.field] == b.axis;
      t.velocity = fstag_[b.field] >= 0;
      const double vwall = t.velocity ? fb.velocity[fstag_[b.field]] : 0.0;
      t.v = (t.normal && fb.kind == SF_BC_SYMMETRY) ? 0.0 : vwall;
      first.push_back(t);
    }
    long long soff = 0, roff = 0;
    for (const auto& kv : P.sends) {
      long long n = 0;
      for (const auto& b : kv.second) n += b.count;
      ph.sends.push_back({kv.first, soff, n});
      soff += n;
    }
    for (const auto& kv : P.recvs) {
      long long n = 0;
      for (const auto& b : kv.second) n += b.count;
      ph.recvs.push_back({kv.first, roff, n});
      roff += n;
    }
    if (soff) ph.sbuf = (double*)dalloc(sizeof(double) * soff);
    if (roff) ph.rbuf = (double*)dalloc(sizeof(double) * roff);
    soff = roff = 0;
    for (const auto& kv : P.sends)
      for (const auto& b : kv.second) {
        sf_task t = task_of(b, 2);
        t.buf = ph.sbuf + soff;
        soff += b.count;
        first.push_back(t);
      }
    for (const auto& kv : P.recvs)
      for (const auto& b : kv.second) {
        sf_task t = task_of(b, 3);
        t.buf = ph.rbuf + roff;
        roff += b.count;
        unpack.push_back(t);
      }
    ph.first = upload_tasks(first);
    ph.unpack = upload_tasks(unpack);
    return phases_.emplace(key, ph).first->second;
  }

  void run_phase(const phase& ph, bool predicated, cudaStream_t on = nullptr) {
    const sf_dev_ctl* pred = predicated ? dctl_ : nullptr;
    cudaStream_t s = on ? on : st_;
    if (ph.first.n) {
      launch_tasks(tview(), ph.first.d, ph.first.n, ph.first.max_count, pred, s);
      ++launches_;
    }
    sendrecv(ph, s);
    if (ph.unpack.n) {
      launch_tasks(tview(), ph.unpack.d, ph.unpack.n, ph.unpack.max_count, pred, s);
      ++launches_;
    }
  }

  // The temporal pass with processor faces, split so the halo exchange
  // overlaps compute. Interior tiles read no ghost cell: their S0 boxes
  // (x in [i0-2, i0+33], y in [j0-2, j0+9], z in [k0-2, k1+1]) stay inside
  // the owned block. Boundary tiles are the rest, covered by up to six slabs.
  // All tile origins are even in x (the TMA start rule).
  std::pair<const work_set*, const work_set*> pass_split() {
    const int ty = sweep2_tile_y(), zc = zc_pass();
    char key[64];
    std::snprintf(key, sizeof key, "split:%d:%d", zc, ty);
    auto ii = items_.find(std::string(key) + ":i");
    if (ii != items_.end()) return {&ii->second, &items_.find(std::string(key) + ":b")->second};
    std::vector<sf_work> vi, vb;
    int ci = 0, cb = 0;
    auto add = [&](std::vector<sf_work>& v, int& cta, int b, const i64 lo[3], const i64 hi[3]) {
      if (lo[0] >= hi[0] || lo[1] >= hi[1] || lo[2] >= hi[2]) return;
      sf_work w{};
      w.blk = b;
      w.cta_begin = cta;
      for (int a = 0; a < 3; ++a) {
        w.lo[a] = lo[a];
        w.hi[a] = hi[a];
      }
      w.tiles[0] = (int)((hi[0] - lo[0] + kTX - 1) / kTX);
      w.tiles[1] = (int)((hi[1] - lo[1] + ty - 1) / ty);
      w.tiles[2] = (int)((hi[2] - lo[2] + zc - 1) / zc);
      cta += w.tiles[0] * w.tiles[1] * w.tiles[2];
      v.push_back(w);
    };
    for (int b = 0; b < nloc_; ++b) {
      const auto n = dec_.dims(gid_[b]);
      // interior: x tiles from 32 with i0 + 33 <= n0 - 1, y tiles from ty
      // with j0 + ty + 1 <= n1 - 1, z in [2, n2 - 2)
      const i64 qx = n[0] >= 66 ? (n[0] - 66) / kTX + 1 : 0;
      const i64 qy = n[1] >= 2 * ty + 2 ? (n[1] - 2 * ty - 2) / ty + 1 : 0;
      const i64 ilo[3] = {kTX, ty, 2}, ihi[3] = {kTX + kTX * qx, ty + ty * qy, n[2] - 2};
      const bool has_int = qx > 0 && qy > 0 && ihi[2] > ilo[2];
      if (!has_int) {
        const i64 lo[3] = {0, 0, 0}, hi[3] = {n[0], n[1], n[2]};
        add(vb, cb, b, lo, hi);
        continue;
      }
      add(vi, ci, b, ilo, ihi);
      const i64 z0[3] = {0, 0, 0}, zl[3] = {n[0], n[1], ilo[2]};
      const i64 z1[3] = {0, 0, ihi[2]}, zh[3] = {n[0], n[1], n[2]};
      add(vb, cb, b, z0, zl);  // z slabs: whole x-y planes
      add(vb, cb, b, z1, zh);
      const i64 y0[3] = {0, 0, ilo[2]}, yl[3] = {n[0], ilo[1], ihi[2]};
      const i64 y1[3] = {0, ihi[1], ilo[2]}, yh[3] = {n[0], n[1], ihi[2]};
      add(vb, cb, b, y0, yl);  // y slabs: full x rows
      add(vb, cb, b, y1, yh);
      const i64 x0[3] = {0, ilo[1], ilo[2]}, xl[3] = {ilo[0], ihi[1], ihi[2]};
      const i64 x1[3] = {ihi[0], ilo[1], ilo[2]}, xh[3] = {n[0], ihi[1], ihi[2]};
      add(vb, cb, b, x0, xl);  // x slabs
      add(vb, cb, b, x1, xh);
    }
    auto mk = [&](std::vector<sf_work>& v, int nctas) {
      work_set ws;
      ws.n = (int)v.size();
      ws.nctas = nctas;
      if (!v.empty()) {
        ws.d = (sf_work*)dalloc(sizeof(sf_work) * v.size());
        SF_CK(cudaMemcpy(ws.d, v.data(), sizeof(sf_work) * v.size(), cudaMemcpyHostToDevice));
      }
      return ws;
    };
    items_.emplace(std::string(key) + ":i", mk(vi, ci));
    items_.emplace(std::string(key) + ":b", mk(vb, cb));
    return {&items_.find(std::string(key) + ":i")->second, &items_.find(std::string(key) + ":b")->second};
  }

  // The temporal pass over one walled component as two work sets: the interior
  // tiles, where k_sweep2 takes its fast path everywhere (every widened cell
  // inside [1, N-3] on x and y: i0 in [3, N-35], j0 in [3, N-11]; S0 planes
  // k0-2 .. k1+1 inside [1, N-2] on z: planes [3, N-3)), for k_sweep2i, and
  // the six boundary slabs around them for k_sweep2. {null, null} when it
  // does not apply (fp32, several components, periodic axes, small grids).
  struct isplit {
    const work_set* in = nullptr;    // interior tiles (k_sweep2i)
    const work_set* slab = nullptr;  // z and y slabs (k_sweep2, 32 x sweep2_tile_y tiles)
    const work_set* xs = nullptr;    // x slabs (k_sweep2, x-slab form)
  };
  // proc: the caller stores the slabs' processor-face layers into the peers
  // (the fused exchange, k_sweep2's REMOTE instantiation)
  isplit interior_split(bool proc = false) {
    if (!maps3_ || !maps4_ || !interior_env_ || nloc_ != 1 || !temporal()) return {};
    if ((dist_ || has_proc_faces()) && !proc) return {};
    if (cfg_.periodic[0] || cfg_.periodic[1] || cfg_.periodic[2]) return {};
    if (!xs_) {
      SF_CK(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking));
      SF_CK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
      SF_CK(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    int stx, sty;
    sweep2_tile(1, &stx, &sty);
    const int ty = sweep2_tile_y(), tyi = sweep2i_tile_y(cfd_es_), zc = zc_pass();
    // the slabs: 32-plane chunks, more CTAs to fill in beside the interior
    // (measured per pass with 32x20 interior tiles: 16 / 32 / 64 planes
    // 2.31 / 2.27 / 2.27 ms)
    const int bzc = std::min(zc, 32);
    ibzc_ = bzc;
    char key[64];
    std::snprintf(key, sizeof key, "isplit:%d:%d:%d:%d", zc, ty, tyi, bzc);
    auto ii = items_.find(std::string(key) + ":i");
    if (ii != items_.end()) {
      if (!ii->second.nctas) return {};
      return {&ii->second, &items_.find(std::string(key) + ":b")->second,
              &items_.find(std::string(key) + ":x")->second};
    }
    const auto n = dec_.dims(gid_[0]);
    // interior tiles: i0 = ox + 32 a <= N - 35, j0 = oy + tyi b <= N - tyi - 3.
    // ox = 16 keeps the tiles' rows 128-byte aligned and leaves x slabs one
    // 16-wide tile column each side (x-slab form); oy = 8: one 32 x 8 tile row
    const i64 ox = stx, oy = ty;
    const i64 qx = n[0] >= ox + kTX + 3 ? (n[0] - 3 - kTX - ox) / kTX + 1 : 0;
    const i64 qy = n[1] >= oy + tyi + 3 ? (n[1] - 3 - tyi - oy) / tyi + 1 : 0;
    const i64 ilo[3] = {ox, oy, 3}, ihi[3] = {ox + kTX * qx, oy + tyi * qy, n[2] - 3};
    std::vector<sf_work> vi, vb, vx;
    int ci = 0, cb = 0, cx = 0;
    auto add = [&](std::vector<sf_work>& v, int& cta, const i64 lo[3], const i64 hi[3], int zcb, int txb, int tyb) {
      if (lo[0] >= hi[0] || lo[1] >= hi[1] || lo[2] >= hi[2]) return;
      sf_work w{};
      w.blk = 0;
      w.cta_begin = cta;
      for (int a = 0; a < 3; ++a) {
        w.lo[a] = lo[a];
        w.hi[a] = hi[a];
      }
      w.tiles[0] = (int)((hi[0] - lo[0] + txb - 1) / txb);
      w.tiles[1] = (int)((hi[1] - lo[1] + tyb - 1) / tyb);
      w.tiles[2] = (int)((hi[2] - lo[2] + zcb - 1) / zcb);
      cta += w.tiles[0] * w.tiles[1] * w.tiles[2];
      v.push_back(w);
    };
    if (qx > 0 && qy > 0 && ihi[2] > ilo[2]) {
      add(vi, ci, ilo, ihi, zc, kTX, tyi);
      const i64 z0[3] = {0, 0, 0}, zl[3] = {n[0], n[1], ilo[2]};
      const i64 z1[3] = {0, 0, ihi[2]}, zh[3] = {n[0], n[1], n[2]};
      add(vb, cb, z0, zl, bzc, kTX, ty);
      add(vb, cb, z1, zh, bzc, kTX, ty);
      const i64 y0[3] = {0, 0, ilo[2]}, yl[3] = {n[0], ilo[1], ihi[2]};
      const i64 y1[3] = {0, ihi[1], ilo[2]}, yh[3] = {n[0], n[1], ihi[2]};
      add(vb, cb, y0, yl, bzc, kTX, ty);
      add(vb, cb, y1, yh, bzc, kTX, ty);
      const i64 x0[3] = {0, ilo[1], ilo[2]}, xl[3] = {ilo[0], ihi[1], ihi[2]};
      const i64 x1[3] = {ihi[0], ilo[1], ilo[2]}, xh[3] = {n[0], ihi[1], ihi[2]};
      add(vx, cx, x0, xl, bzc, stx, sty);
      add(vx, cx, x1, xh, bzc, stx, sty);
    }
    auto mk = [&](std::vector<sf_work>& v, int nctas) {
      work_set ws;
      ws.n = (int)v.size();
      ws.nctas = nctas;
      if (!v.empty()) {
        ws.d = (sf_work*)dalloc(sizeof(sf_work) * v.size());
        SF_CK(cudaMemcpy(ws.d, v.data(), sizeof(sf_work) * v.size(), cudaMemcpyHostToDevice));
      }
      return ws;
    };
    items_.emplace(std::string(key) + ":i", mk(vi, ci));
    items_.emplace(std::string(key) + ":b", mk(vb, cb));
    items_.emplace(std::string(key) + ":x", mk(vx, cx));
    return interior_split(proc);
  }

  // max over ranks of n accumulators (IEEE bit patterns of |x|): order-free,
  // NaN-sticky, so bitwise the reference's worker-order combine
  // (reductions.hpp:75-88)
  void allreduce_max(unsigned long long* dev, int n) {
    if (!dist_) return;
    if (tr_ == TR_NCCL) {
      SF_NC(nccl()->AllReduce(dev, dev, (size_t)n, kNcclUint64, kNcclMax, comm_, st_));
      return;
    }
    unsigned long long mine[8];
    std::vector<unsigned long long> all((size_t)(8 * world_));
    SF_CK(cudaMemcpyAsync(mine, dev, sizeof(mine[0]) * (size_t)n, cudaMemcpyDeviceToHost, st_));
    SF_CK(cudaStreamSynchronize(st_));
    host_allgather(mine, all.data(), sizeof(mine[0]) * (size_t)n);
    for (int r = 0; r < world_; ++r)
      for (int q = 0; q < n; ++q) mine[q] = std::max(mine[q], all[(size_t)(r * n + q)]);
    SF_CK(cudaMemcpyAsync(dev, mine, sizeof(mine[0]) * (size_t)n, cudaMemcpyHostToDevice, st_));
    SF_CK(cudaStreamSynchronize(st_));
  }

  // ---- transports -------------------------------------------------------------
  // NCCL (one rank per GPU; the production path) or CUDA IPC: every rank maps
  // its peers' device buffers (cudaIpcOpenMemHandle) and moves messages with
  // device copies or direct stores; the caller's host callbacks carry the
  // 64-byte handles, the residual maxima and barriers. The IPC transport also
  // runs several ranks on ONE device (each a separate process), which is how
  // the cross-process data plane is tested on a one-GPU box: no kernel ever
  // waits on another rank's kernel, the host orders them.
  void host_allgather(const void* send, void* recv, size_t bytes) {
    if (tr_ == TR_IPC) {
      if (htr_.allgather(htr_.ctx, send, recv, (int64_t)bytes) != 0)
        throw error(SF_ERR_CUDA, "host transport: allgather failed");
      return;
    }
    const size_t w = (bytes + 7) / 8;  // NCCL: through device memory
    double* d = (double*)dalloc_tmp(8 * w * (size_t)(world_ + 1));
    std::vector<double> h(w * (size_t)(world_ + 1), 0.0);
    std::memcpy(h.data(), send, bytes);
    SF_CK(cudaMemcpyAsync(d, h.data(), 8 * w, cudaMemcpyHostToDevice, st_));
    SF_NC(nccl()->AllGather(d, d + w, w, kNcclFloat64, comm_, st_));
    SF_CK(cudaMemcpyAsync(h.data() + w, d + w, 8 * w * (size_t)world_, cudaMemcpyDeviceToHost, st_));
    SF_CK(cudaStreamSynchronize(st_));
    SF_CK(cudaFree(d));
    for (int r = 0; r < world_; ++r) std::memcpy((char*)recv + r * bytes, h.data() + w * (size_t)(r + 1), bytes);
  }
  void host_barrier() {
    if (tr_ == TR_IPC) {
      if (htr_.barrier(htr_.ctx) != 0) throw error(SF_ERR_CUDA, "host transport: barrier failed");
      return;
    }
    int x = 0;
    std::vector<int> all((size_t)world_);
    host_allgather(&x, all.data(), sizeof x);
  }
  // count doubles per rank from device buffer snd into all (rank order), on st_
  void dev_allgather(const double* snd, double* all, size_t count) {
    if (tr_ == TR_NCCL) {
      SF_NC(nccl()->AllGather(snd, all, count, kNcclFloat64, comm_, st_));
      return;
    }
    std::vector<double> mine(count), h(count * (size_t)world_);
    SF_CK(cudaMemcpyAsync(mine.data(), snd, 8 * count, cudaMemcpyDeviceToHost, st_));
    SF_CK(cudaStreamSynchronize(st_));
    host_allgather(mine.data(), h.data(), 8 * count);
    SF_CK(cudaMemcpyAsync(all, h.data(), 8 * h.size(), cudaMemcpyHostToDevice, st_));
    SF_CK(cudaStreamSynchronize(st_));
  }
  // open_ipc without throwing: false (and the CUDA error cleared) on failure
  bool try_open_ipc(const cudaIpcMemHandle_t& h) {
    const std::string key(reinterpret_cast<const char*>(&h), sizeof h);
    if (ipc_open_.count(key)) return true;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    ipc_open_[key] = p;
    return true;
  }
  void* open_ipc(const cudaIpcMemHandle_t& h) {
    const std::string key(reinterpret_cast<const char*>(&h), sizeof h);
    auto it = ipc_open_.find(key);
    if (it != ipc_open_.end()) return it->second;
    void* p = nullptr;
    SF_CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ipc_open_[key] = p;
    return p;
  }
  // One phase's messages. NCCL: one group of per-peer send/recv. IPC: every
  // rank pulls its messages out of the senders' buffers with device copies,
  // between two host barriers (all packed / all pulled).
  void sendrecv(const phase& ph, cudaStream_t s) {
    if (tr_ == TR_NCCL) {
      if (ph.sends.empty() && ph.recvs.empty()) return;
      SF_NC(nccl()->GroupStart());
      for (const auto& m : ph.sends)
        SF_NC(nccl()->Send(ph.sbuf + m.off, (size_t)m.count, kNcclFloat64, m.peer, comm_, s));
      for (const auto& m : ph.recvs)
        SF_NC(nccl()->Recv(ph.rbuf + m.off, (size_t)m.count, kNcclFloat64, m.peer, comm_, s));
      SF_NC(nccl()->GroupEnd());
      return;
    }
    if (tr_ != TR_IPC) return;
    if (!ph.x_ready) setup_phase_ipc(ph);
    if (!ph.x_any) return;
    SF_CK(cudaStreamSynchronize(s));  // this rank's packs are in its send buffer
    host_barrier();
    for (size_t q = 0; q < ph.recvs.size(); ++q)
      SF_CK(cudaMemcpyAsync(ph.rbuf + ph.recvs[q].off, ph.x_src[q], sizeof(double) * (size_t)ph.recvs[q].count,
                            cudaMemcpyDeviceToDevice, s));
    SF_CK(cudaStreamSynchronize(s));
    host_barrier();  // every rank pulled: the send buffers may be refilled
  }
  static constexpr int kMaxMsgs = 32;
  struct ipc_phase_rec {
    cudaIpcMemHandle_t h;
    int has, n;
    int peer[kMaxMsgs];
    long long off[kMaxMsgs], cnt[kMaxMsgs];
  };
  // Collective (every rank runs the same phases in the same order): publish
  // this rank's send buffer and the offset of each peer's message in it.
  void setup_phase_ipc(const phase& ph) {
    ipc_phase_rec me;
    std::memset(&me, 0, sizeof me);
    if ((int)ph.sends.size() > kMaxMsgs) throw error(SF_ERR_ARG, "too many messages in one exchange phase");
    me.has = ph.sbuf != nullptr;
    if (me.has) SF_CK(cudaIpcGetMemHandle(&me.h, ph.sbuf));
    me.n = (int)ph.sends.size();
    for (int q = 0; q < me.n; ++q) {
      me.peer[q] = ph.sends[q].peer;
      me.off[q] = ph.sends[q].off;
      me.cnt[q] = ph.sends[q].count;
    }
    std::vector<ipc_phase_rec> all((size_t)world_);
    host_allgather(&me, all.data(), sizeof me);
    ph.x_src.clear();
    for (const auto& m : ph.recvs) {
      const ipc_phase_rec& r = all[(size_t)m.peer];
      int at = -1;
      for (int q = 0; q < r.n; ++q)
        if (r.peer[q] == rank_) at = q;
      if (at < 0 || r.cnt[at] != m.count || !r.has)
        throw error(SF_ERR_CUDA, "IPC transport: send and receive plans disagree with rank " + std::to_string(m.peer));
      ph.x_src.push_back(static_cast<const double*>(open_ipc(r.h)) + r.off[at]);
    }
    ph.x_any = false;
    for (const auto& r : all) ph.x_any = ph.x_any || r.n > 0;
    ph.x_ready = true;
  }

  // ---- direct exchange of the temporal pass ------------------------------------
  // After each pass, the pass's outputs in the g owned layers next to every
  // processor face, edge and corner are stored straight into the ghost shell
  // of the neighbour across it (26 directions, diagonal neighbours included):
  // pack + send + unpack of exchange.hpp:165-224 become one launch of direct
  // peer stores. It runs before the pass's max-allreduce, which every rank
  // waits for before its next pass, so the stores have landed when they are
  // read (and the ghosts they overwrite are in the buffer the peers' current
  // pass does not read: outputs ping-pong). Ghost cells beside a physical face
  // are left as the 3-phase exchange-only refresh leaves them: the pass never
  // reads their values (sf_sweep2.cu takes pins there).
  struct ipc_field_rec {
    unsigned long long host;
    char pci[32];
    int has[4][kSlots];
    cudaIpcMemHandle_t h[4][kSlots];
    long long sx, sy, base, n[3];
  };
  // blocks of at least 2g cells per axis: a cell lies in at most one layer
  // band per axis (the fused epilogue's assumption)
  bool thick_blocks() const {
    for (const auto& L : lay_)
      for (int a = 0; a < 3; ++a)
        if (L.dims[a] < 2 * dec_.ghost) return false;
    return true;
  }
  // The fused-exchange table of local block b: one entry per direction of
  // the direct-store plan; ptr_of(peer, field k, physical buffer) and
  // layout_of(peer, {sx, sy, base}) resolve the neighbour's arrays.
  template <class P, class Lay>
  sweep2_remote build_remote(int b, P ptr_of, Lay layout_of) {
    static const int F4[4] = {SF_VX, SF_VY, SF_VZ, SF_DIVU};
    (void)F4;
    sweep2_remote h{};
    h.g = dec_.ghost;
    for (int q = 0; q < 27; ++q) h.idx[q] = -1;
    int np = 0;
    for (const auto& dr : build_direct_plan(dec_, gid_[b])) {
      sweep2_peer& Pe = h.peer[np];
      for (int k = 0; k < 4; ++k)
        for (int q = 0; q < kSlots; ++q) Pe.ptr[k][q] = ptr_of(dr.peer, k, q);
      long long l[3];
      layout_of(dr.peer, l);
      Pe.rsx = l[0];
      Pe.rsy = l[1];
      Pe.rbase = l[2];
      for (int a = 0; a < 3; ++a) Pe.shift[a] = dr.dlo[a] - dr.lo[a];
      h.idx[(dr.d[0] + 1) + 3 * (dr.d[1] + 1) + 9 * (dr.d[2] + 1)] = np++;
    }
    return h;
  }
  sweep2_remote* upload_remote(const std::vector<sweep2_remote>& v) {
    auto* d = (sweep2_remote*)dalloc(sizeof(sweep2_remote) * v.size());
    SF_CK(cudaMemcpy(d, v.data(), sizeof(sweep2_remote) * v.size(), cudaMemcpyHostToDevice));
    return d;
  }
  // One process, several grid components on the device: the temporal pass
  // stores its boundary outputs straight into the neighbouring components'
  // ghost shells (pointers by physical buffer; every component swaps alike),
  // so no exchange runs between passes. SF_OVERLAP (tests) keeps the phases.
  int local_fused_ = 0;  // 0 not set up, 1 active, -1 unavailable
  bool local_fused() {
    if (dist_ || force_overlap_ || !direct_mode_) return false;
    if (local_fused_ == 0) {
      local_fused_ = -1;
      if (thick_blocks()) {
        static const int F4[4] = {SF_VX, SF_VY, SF_VZ, SF_DIVU};
        download_table();
        std::vector<sweep2_remote> v;
        for (int b = 0; b < nloc_; ++b)
          v.push_back(build_remote(b, [&](int peer, int k, int phys) -> double* {
            const int lb = lid_[peer];
            for (int q = 0; q < kSlots; ++q)
              if (htab_->ptr[lb][F4[k]][q] && htab_->bidx[lb][F4[k]][q] == phys) return htab_->ptr[lb][F4[k]][q];
            return nullptr;
          }, [&](int peer, long long* l) {
            const sf_layout& L = lay_[lid_[peer]];
            l[0] = L.sx;
            l[1] = L.sy;
            l[2] = L.base;
          }));
        remote_ = upload_remote(v);
        local_fused_ = 1;
      }
    }
    return local_fused_ > 0;
  }
  bool direct_active() {
    // the separate direct-store launch (mode 2) moves fp64 values; an fp32
    // simulation uses the fused stores or the phases
    if (!dist_ || !direct_mode_ || (direct_mode_ == 2 && cfd_es_ != 8)) return false;
    if (direct_state_ == 0) setup_direct();
    return direct_state_ > 0;
  }
  void setup_direct() {
    static const int F4[4] = {SF_VX, SF_VY, SF_VZ, SF_DIVU};
    download_table();
    ipc_field_rec me;
    std::memset(&me, 0, sizeof me);
    int me_ok = 1;
    char hn[256] = {0};
    gethostname(hn, sizeof hn - 1);
    me.host = std::hash<std::string>()(std::string(hn));
    SF_CK(cudaDeviceGetPCIBusId(me.pci, (int)sizeof me.pci, opt_.device));
    const sf_layout& L = lay_[0];
    me.sx = L.sx;
    me.sy = L.sy;
    me.base = L.base;
    for (int a = 0; a < 3; ++a) me.n[a] = L.dims[a];
    for (int k = 0; k < 4; ++k)
      for (int q = 0; q < kSlots; ++q) {
        double* p = htab_->ptr[0][F4[k]][q];
        if (!p) continue;
        const int phys = htab_->bidx[0][F4[k]][q];
        if (cudaIpcGetMemHandle(&me.h[k][phys], p) == cudaSuccess) {
          me.has[k][phys] = 1;
        } else {  // not exportable: the collective decision falls back to the phases
          cudaGetLastError();
          me_ok = 0;
        }
      }
    std::vector<ipc_field_rec> all((size_t)world_);
    host_allgather(&me, all.data(), sizeof me);
    const auto dirs = build_direct_plan(dec_, rank_);
    // every peer must be mappable here (same node, device visible and
    // peer-accessible, or the same device); the decision is collective
    int ok = me_ok;
    for (const auto& dr : dirs) {
      const ipc_field_rec& r = all[(size_t)dr.peer];
      int dev = -1;
      if (r.host != me.host || cudaDeviceGetByPCIBusId(&dev, r.pci) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        continue;
      }
      int can = dev == opt_.device;
      if (!can) cudaDeviceCanAccessPeer(&can, opt_.device, dev);
      for (int k = 0; k < 4; ++k)
        for (int q = 0; q < kSlots; ++q)
          if (me.has[k][q] != r.has[k][q]) can = 0;
      // map every buffer now: a failure (driver, permissions) turns the
      // collective decision below into the exchange phases on every rank
      for (int k = 0; k < 4 && can; ++k)
        for (int q = 0; q < kSlots && can; ++q)
          if (r.has[k][q] && !try_open_ipc(r.h[k][q])) can = 0;
      ok = ok && can;
    }
    std::vector<int> oks((size_t)world_);
    host_allgather(&ok, oks.data(), sizeof ok);
    for (int v : oks) ok = ok && v;
    if (!ok) {
      direct_state_ = -1;
      return;
    }
    std::vector<sf_task> tasks;
    for (const auto& dr : dirs) {
      const ipc_field_rec& r = all[(size_t)dr.peer];
      sf_task t{};
      t.type = 4;
      t.src_blk = 0;
      t.slot = ALT;
      t.rsx = r.sx;
      t.rsy = r.sy;
      t.rbase = r.base;
      for (int a = 0; a < 3; ++a) {
        t.lo[a] = dr.lo[a];
        t.dims[a] = dr.dims[a];
        t.dlo[a] = dr.dlo[a];
      }
      t.count = dr.count;
      for (int k = 0; k < 4; ++k) {
        t.field = F4[k];
        for (int q = 0; q < kSlots; ++q) t.rptr[q] = r.has[k][q] ? static_cast<double*>(open_ipc(r.h[k][q])) : nullptr;
        tasks.push_back(t);
      }
    }
    task_set ts = upload_tasks(tasks);
    direct_tasks_.d = ts.d;
    direct_tasks_.n = ts.n;
    direct_tasks_.max_count = ts.max_count;
    // the same plan as the pass's fused epilogue table
    if (thick_blocks())
      remote_ = upload_remote({build_remote(0, [&](int peer, int k, int phys) {
                                 const ipc_field_rec& r = all[(size_t)peer];
                                 return r.has[k][phys] ? static_cast<double*>(open_ipc(r.h[k][phys])) : nullptr;
                               }, [&](int peer, long long* sxsybase) {
                                 const ipc_field_rec& r = all[(size_t)peer];
                                 sxsybase[0] = r.sx;
                                 sxsybase[1] = r.sy;
                                 sxsybase[2] = r.base;
                               })});
    direct_state_ = 1;
  }
 public:
  void set_direct(int mode) {
    if (mode < 0 || mode > 2) throw error(SF_ERR_ARG, "direct exchange mode must be 0, 1 or 2");
    direct_mode_ = mode;
  }
  int direct_enabled() { return direct_active() ? (direct_mode_ == 1 && remote_ ? 1 : 2) : 0; }
 private:

  // The temporal pass (two half-sweeps per launch, sf_sweep2.cu) applies with
  // fused = 1 when every face of every local grid component is a wall, a
  // symmetry plane or a processor face, and the ghost shell is 2 deep where
  // there are processor faces (the pass reads 2-deep halos of the old state).
  // A periodic axis split over grid components wraps through processor faces:
  // the pass gives ghost cells across the wrap their wrapped parity
  // (sf_sweep2.cu; scripts/probes/parity_stress.py found the unwrapped
  // version wrong on 39x43x13, periodic y, two components, ghost 2).
  bool temporal() const {
    if (!maps2_ || !temporal_env_ || opt_.fused != 1) return false;
    for (int b = 0; b < nloc_; ++b)  // the pass addresses its arrays with 32-bit element offsets
      if ((unsigned long long)(lay_[b].sx * lay_[b].sy * lay_[b].sz) >= (1ull << 32)) return false;
    bool proc = false;
    for (int b = 0; b < nloc_; ++b)
      for (int fi = 0; fi < 6; ++fi) {
        const int k = htab_->blk[b].face[fi];
        if (k == FACE_PROC)
          proc = true;
        else if (k != FACE_WALL && k != FACE_SYM)
          return false;
      }
    return !proc || opt_.ghost >= 2;
  }
  bool has_proc_faces() const {
    for (int b = 0; b < nloc_; ++b)
      for (int fi = 0; fi < 6; ++fi)
        if (htab_->blk[b].face[fi] == FACE_PROC) return true;
    return false;
  }
  // wall-normal velocities pinned on the domain's faces (exchange.hpp:288-316)
  sweep2_pins wall_pins() const {
    sweep2_pins p{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (bc_[1].kind == SF_BC_WALL) p.u = bc_[1].velocity[0];
    if (bc_[3].kind == SF_BC_WALL) p.v = bc_[3].velocity[1];
    if (bc_[5].kind == SF_BC_WALL) p.w = bc_[5].velocity[2];
    if (bc_[0].kind == SF_BC_WALL) p.ul = bc_[0].velocity[0];
    if (bc_[2].kind == SF_BC_WALL) p.vl = bc_[2].velocity[1];
    if (bc_[4].kind == SF_BC_WALL) p.wl = bc_[4].velocity[2];
    return p;
  }
  // The persistent pressure loop (k_pressure_loop) applies to a single grid
  // component in a single process whose fused half-sweep writes every divu
  // ghost itself, when the grid is small enough that launches dominate
  // (SF_PERSIST=0 off, =1 whenever it applies).
  bool persistent() {
    if (persist_env_ == 0 || dist_ || timing_ || !opt_.fused || nloc_ != 1 || has_proc_faces() || cfd_es_ != 8)
      return false;
    if (pressure_loop_ctas() < 1) return false;  // no co-resident CTA (occupancy query failed)
    const phase& ph = phase_for(1u << SF_DIVU, -1, SF_SCOPE_ALL, true);
    if (ph.first.n || ph.unpack.n || !ph.sends.empty() || !ph.recvs.empty()) return false;
    if (persist_env_ == 1) return true;
    const sf_dev_block& B = htab_->blk[0];
    return (double)B.n[0] * B.n[1] * B.n[2] <= persist_cells_;
  }
  bool tma_sweep() const { return maps_ && (opt_.fused == 1 || opt_.fused == 3); }

  // Enqueues one unit of the pressure loop; returns the half-sweeps it covers.
  int enqueue_sweep_unit() {
    if (!temporal()) {
      enqueue_half_sweep();
      return 1;
    }
    const int fin = dist_ ? 0 : 1;
    const auto split = interior_split();
    if (!has_proc_faces() && split.in) {
      // the interior tiles on the interior form (sweep2i_tile_y rows), the
      // slabs on k_sweep2 (x slabs on its x-slab form) on the second stream
      // at the same time; one last-CTA count spans the launches
      const work_set& wi = *split.in;
      const work_set& wb = *split.slab;
      const work_set& wx = *split.xs;
      const unsigned total = (unsigned)(wi.nctas + wb.nctas + wx.nctas);
      mark_form(iter_launch_, 1);
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 0), st_));
      // boundary slabs first on the second stream, the interior beside them
      // (measured with 32x20 interior tiles: concurrent 2.27 ms, interior
      // launched first 2.27, either order on one stream 2.33; slab chunks of
      // 16 / 32 / 64 planes 2.31 / 2.27 / 2.27)
      SF_CK(cudaEventRecord(ev_fork_, st_));
      SF_CK(cudaStreamWaitEvent(xs_, ev_fork_, 0));
      launch_sweep2(tview(wb), wb.nctas, ibzc_, consts_, dctl_, loop_flag(), maps2_, fin, wall_pins(), xs_, total,
                    nullptr, cfd_es_);
      launch_sweep2(tview(wx), wx.nctas, ibzc_, consts_, dctl_, loop_flag(), maps4_, fin, wall_pins(), xs_, total,
                    nullptr, cfd_es_, 1);
      launch_sweep2i(tview(wi), wi.nctas, zc_pass(), consts_, dctl_, loop_flag(), maps3_, fin, st_, total, cfd_es_);
      SF_CK(cudaEventRecord(ev_join_, xs_));
      SF_CK(cudaStreamWaitEvent(st_, ev_join_, 0));
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 1), st_));
      launches_ += (wi.nctas > 0) + (wb.nctas > 0) + (wx.nctas > 0);
    } else if (!has_proc_faces()) {
      const work_set& ws = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_pass(), kTX, sweep2_tile_y());
      mark_form(iter_launch_, 0);
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 0), st_));
      launch_sweep2(tview(ws), ws.nctas, zc_pass(), consts_, dctl_, loop_flag(), maps2_, fin, wall_pins(), st_, 0,
                    nullptr, cfd_es_);
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 1), st_));
      ++launches_;
    } else {
      // Processor faces: the pass reads 2-deep halos of vx, vy, vz, divu (p
      // only on owned cells). The exchange of the state the previous unit
      // left (redundant for the first unit, skipped once the loop is done)
      // runs on the exchange stream while the interior tiles compute; the
      // boundary tiles follow it. Both launches share one last-CTA count.
      const unsigned mask = (1u << SF_VX) | (1u << SF_VY) | (1u << SF_VZ) | (1u << SF_DIVU);
      if (!xs_) {
        SF_CK(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking));
        SF_CK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        SF_CK(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
      }
      // The split costs 2-5 % (boundary slabs run with little work per CTA):
      // measured on one device, where the exchange is a few device copies,
      // serialising is faster. Across ranks the exchange goes through NCCL and
      // is hidden behind the interior (SF_NO_OVERLAP serialises there too).
      if (local_fused()) {
        // components on this device: one launch, the exchange fused into it
        const work_set& wa = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_pass(), kTX, sweep2_tile_y());
        if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 0), st_));
        launch_sweep2(tview(wa), wa.nctas, zc_pass(), consts_, dctl_, loop_flag(), maps2_, fin, wall_pins(), st_, 0,
                      remote_, cfd_es_);
        if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 1), st_));
        ++launches_;
        ++iter_launch_;
        int ftx, fty;
        sweep_tile_shape(&ftx, &fty);
        const work_set& wr = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_fused_, ftx, fty);
        launch_sweep_div_tma(tview(wr), wr.nctas, zc_fused_, consts_, dctl_, loop_flag(), maps_, 2, st_, cfd_es_);
        launches_ += 2;
        check_launch();
        return 2;
      }
      if (direct_active()) {
        // one launch over all tiles, then the direct stores into the peers
        // (predicated like the pass), then the max-allreduce below
        const work_set& wa = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_pass(), kTX, sweep2_tile_y());
        const bool fused_x = direct_mode_ == 1 && remote_;
        const auto ps = fused_x ? interior_split(true) : isplit{};
        mark_form(iter_launch_, ps.in ? 1 : 0);
        if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 0), st_));
        if (ps.in) {
          // the interior tiles on the interior form; the slabs (which hold
          // every layer next to a processor face) on k_sweep2's REMOTE
          // instantiation on the second stream, storing into the peers
          const work_set& wi = *ps.in;
          const work_set& wb = *ps.slab;
          const work_set& wx = *ps.xs;
          const unsigned total = (unsigned)(wi.nctas + wb.nctas + wx.nctas);
          SF_CK(cudaEventRecord(ev_fork_, st_));
          SF_CK(cudaStreamWaitEvent(xs_, ev_fork_, 0));
          launch_sweep2(tview(wb), wb.nctas, ibzc_, consts_, dctl_, loop_flag(), maps2_, fin, wall_pins(), xs_, total,
                        remote_, cfd_es_);
          launch_sweep2(tview(wx), wx.nctas, ibzc_, consts_, dctl_, loop_flag(), maps4_, fin, wall_pins(), xs_, total,
                        remote_, cfd_es_, 1);
          launch_sweep2i(tview(wi), wi.nctas, zc_pass(), consts_, dctl_, loop_flag(), maps3_, fin, st_, total,
                         cfd_es_);
          SF_CK(cudaEventRecord(ev_join_, xs_));
          SF_CK(cudaStreamWaitEvent(st_, ev_join_, 0));
          launches_ += (wi.nctas > 0) + (wb.nctas > 0) + (wx.nctas > 0) - 1;
        } else {
          launch_sweep2(tview(wa), wa.nctas, zc_pass(), consts_, dctl_, loop_flag(), maps2_, fin, wall_pins(), st_, 0,
                        fused_x ? remote_ : nullptr, cfd_es_);
        }
        if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 1), st_));
        if (!fused_x) {
          launch_tasks(tview(), direct_tasks_.d, direct_tasks_.n, direct_tasks_.max_count, dctl_, st_, 296);
          ++launches_;
        }
        ++launches_;
        ++iter_launch_;
        allreduce_max(&dctl_->acc[0], 2);
        ctl(CTL_FINISH_PASS, 0.0, 0, 0, 0, 1);
        int ftx, fty;
        sweep_tile_shape(&ftx, &fty);
        const work_set& wr = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_fused_, ftx, fty);
        launch_sweep_div_tma(tview(wr), wr.nctas, zc_fused_, consts_, dctl_, loop_flag(), maps_, 2, st_, cfd_es_);
        launches_ += 2;
        check_launch();
        return 2;
      }
      const bool overlap = (dist_ || force_overlap_) && overlap_env_;
      const auto split = pass_split();
      const work_set& wi = overlap ? *split.first : empty_ws_;
      const work_set& wb =
          overlap ? *split.second : items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_pass(), kTX, sweep2_tile_y());
      const unsigned total = (unsigned)(wi.nctas + wb.nctas);
      SF_CK(cudaEventRecord(ev_fork_, st_));
      SF_CK(cudaStreamWaitEvent(xs_, ev_fork_, 0));
      for (int axis = 0; axis < 3; ++axis) run_phase(phase_for(mask, axis, SF_SCOPE_ALL, true), true, xs_);
      SF_CK(cudaEventRecord(ev_join_, xs_));
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 0), st_));
      if (wi.nctas)
        launch_sweep2(tview(wi), wi.nctas, zc_pass(), consts_, dctl_, loop_flag(), maps2_, fin, wall_pins(), st_,
                      total, nullptr, cfd_es_);
      SF_CK(cudaStreamWaitEvent(st_, ev_join_, 0));
      launch_sweep2(tview(wb), wb.nctas, zc_pass(), consts_, dctl_, loop_flag(), maps2_, fin, wall_pins(), st_,
                    total, nullptr, cfd_es_);
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 1), st_));
      ++launches_;
    }
    ++iter_launch_;
    if (!fin) {
      allreduce_max(&dctl_->acc[0], 2);
      ctl(CTL_FINISH_PASS, 0.0, 0, 0, 0, 1);
      enqueue_redo();
    }
    // (one process: the redo, if any, runs once after the loop -- a pass that
    // stops after its first sweep also ends the loop, and every later unit is
    // predicated off without touching the fields or ctl->redo)
    check_launch();
    return 2;
  }
  // predicated redo of a temporal pass's first sweep when the pass stopped
  // after it (ctl->redo): k_sweep_div_tma on the pass's input
  void enqueue_redo() {
    int ftx, fty;
    sweep_tile_shape(&ftx, &fty);
    const work_set& wr = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_fused_, ftx, fty);
    launch_sweep_div_tma(tview(wr), wr.nctas, zc_fused_, consts_, dctl_, loop_flag(), maps_, 2, st_, cfd_es_);
    ++launches_;
  }
  void enqueue_redo_after_loop() {
    if (temporal() && !dist_) enqueue_redo();
  }

  void enqueue_half_sweep() {
    if (opt_.fused) {
      int ftx = kTX, fty = kTY;
      if (tma_sweep()) sweep_tile_shape(&ftx, &fty);
      const work_set& ws = items_for(SF_REGION_ALL, {0, 0, 0, 0, 0, 0}, zc_fused_, ftx, fty);
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 0), st_));
      // single process: the kernel's last CTA finalises the sweep; across
      // ranks the residual first needs the max over ranks
      const int fin = dist_ ? 0 : 1;
      if (tma_sweep())
        launch_sweep_div_tma(tview(ws), ws.nctas, zc_fused_, consts_, dctl_, loop_flag(), maps_, fin, st_, cfd_es_);
      else
        launch_sweep_div(tview(ws), ws.nctas, zc_fused_, consts_, dctl_, loop_flag(), fin, st_);
      ++launches_;
      if (timing_) SF_CK(cudaEventRecord(timer(iter_launch_, 1), st_));
      ++iter_launch_;
      if (!fin) {
        allreduce_max(&dctl_->acc[0], 1);
        ctl(CTL_FINISH_FUSED, 0.0, 0, 0, 0, 1);
      }
      run_phase(phase_for(1u << SF_DIVU, -1, SF_SCOPE_ALL, true), true);
    } else {
      // the reference's dataflow, predicated step by step (cfd.hpp:295-303)
      refresh({SF_DIVU}, true);
      const work_set& ws = items_for(SF_REGION_ALL, {0, 1, 0, 1, 0, 1}, zc_plain_);
      launch_pressure_sweep(tview(ws), ws.nctas, zc_plain_, consts_, dctl_, 1, nullptr, st_);
      ++launches_;
      ctl(CTL_AFTER_SWEEP, 0.0, 0, 0, 0, 1);
      refresh({SF_VX, SF_VY, SF_VZ}, true);
      const work_set& wd = items_for(SF_REGION_ALL, {1, 0, 1, 0, 1, 0}, zc_plain_);
      launch_divergence(tview(wd), wd.nctas, zc_plain_, consts_, dctl_, 0, 1, st_);
      ++launches_;
      allreduce_max(&dctl_->acc[0], 1);
      ctl(CTL_FINISH_SWEEP, 0.0, 0, 0, 0, 1);
    }
    check_launch();
  }
};

}  // namespace sfb

// ===========================================================================
// C ABI (include/sforge_b200.h)
// ===========================================================================
struct sf_sim {
  std::unique_ptr<sfb::simulation> s;
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SF_OK;
  } catch (const sfb::error& e) {
    sfb::g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    sfb::g_last_error = e.what();
    return SF_ERR_ARG;
  }
}

int need(const void* p, const char* what) {
  if (!p) throw sfb::error(SF_ERR_ARG, std::string(what) + " is null");
  return 0;
}

std::vector<int> field_list(const sfb::simulation& S, const char* const* fields, int n) {
  std::vector<int> out;
  for (int i = 0; i < n; ++i) out.push_back(S.field_id(fields[i]));
  return out;
}

// direct-view helpers for level-2 launches
sfb::direct_view make_view(const sf_layout* l, const sf_box* boxes, int nbox, int zc) {
  sfb::direct_view v;
  std::memset(&v, 0, sizeof v);
  for (int a = 0; a < 3; ++a) {
    v.b0.n[a] = l->dims[a];
    v.b0.lo[a] = l->lo[a];
  }
  v.b0.sx = l->sx;
  v.b0.sy = l->sy;
  v.b0.sz = l->sz;
  v.b0.base = l->base;
  v.b0.g = l->ghost;
  if (nbox < 1 || nbox > sfb::kDirectItems)
    throw sfb::error(SF_ERR_ARG, "nbox must lie in [1, 8]");
  int cta = 0;
  v.nitems = 0;
  for (int q = 0; q < nbox; ++q) {
    sfb::sf_work& w = v.it[v.nitems];
    w.blk = 0;
    w.cta_begin = cta;
    bool empty = false;
    for (int a = 0; a < 3; ++a) {
      w.lo[a] = boxes[q].lo[a];
      w.hi[a] = boxes[q].hi[a];
      if (w.hi[a] <= w.lo[a]) empty = true;
      if (w.lo[a] < 0 || w.hi[a] > l->dims[a]) throw sfb::error(SF_ERR_ARG, "box outside the block");
    }
    if (empty) continue;
    w.tiles[0] = (int)((w.hi[0] - w.lo[0] + sfb::kTX - 1) / sfb::kTX);
    w.tiles[1] = (int)((w.hi[1] - w.lo[1] + sfb::kTY - 1) / sfb::kTY);
    w.tiles[2] = (int)((w.hi[2] - w.lo[2] + zc - 1) / zc);
    cta += w.tiles[0] * w.tiles[1] * w.tiles[2];
    ++v.nitems;
  }
  v.b0.face[0] = cta;  // scratch: total CTAs (read back by the caller, faces unused here)
  return v;
}

sfb::sf_consts to_consts(const sf_cfd_consts* c) {
  sfb::sf_consts s{};
  s.nu = c->nu;
  s.alpha = c->alpha;
  s.fx = c->fx;
  s.fy = c->fy;
  s.fz = c->fz;
  s.ix = c->ix;
  s.iy = c->iy;
  s.iz = c->iz;
  s.ix2 = c->ix2;
  s.iy2 = c->iy2;
  s.iz2 = c->iz2;
  std::memcpy(s.bscale, c->bscale, sizeof s.bscale);
  s.nm1[0] = c->nxm1;
  s.nm1[1] = c->nym1;
  s.nm1[2] = c->nzm1;
  s.per[0] = c->px;
  s.per[1] = c->py;
  s.per[2] = c->pz;
  return s;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

void check_last() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw sfb::error(SF_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace

extern "C" {

int sf_abi_version(void) { return SF_ABI_VERSION; }
const char* sf_last_error(void) { return sfb::g_last_error.c_str(); }
int sf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int sf_decompose(const int64_t extents[3], const double spacing[3], int workers, int ghost,
                 const int periodic[3], int proc_grid[3], int64_t* lo, int64_t* hi) {
  return guarded([&] {
    need(extents, "extents");
    need(spacing, "spacing");
    const long long ext[3] = {extents[0], extents[1], extents[2]};
    const bool per[3] = {periodic && periodic[0] != 0, periodic && periodic[1] != 0,
                         periodic && periodic[2] != 0};
    const auto d = sfb::decompose(ext, spacing, workers, ghost, per);
    for (int a = 0; a < 3; ++a)
      if (proc_grid) proc_grid[a] = d.pg[a];
    for (int w = 0; w < d.workers; ++w)
      for (int a = 0; a < 3; ++a) {
        if (lo) lo[3 * w + a] = d.lo[w][a];
        if (hi) hi[3 * w + a] = d.hi[w][a];
      }
  });
}

int sf_decomp_neighbor(const int proc_grid[3], const int periodic[3], int w, int axis, int side) {
  sfb::decomposition d;
  for (int a = 0; a < 3; ++a) {
    d.pg[a] = proc_grid[a];
    d.periodic[a] = periodic[a] != 0;
  }
  return d.neighbor(w, axis, side);
}

int sf_nccl_unique_id(void* out128) {
  return guarded([&] {
    need(out128, "out");
    if (!sfb::nccl()) throw sfb::error(SF_ERR_CUDA, "NCCL library not found (set SF_NCCL_LIB)");
    sfb::nccl_uid id;
    SF_NC(sfb::nccl()->GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof id);
  });
}

int sf_exchange_plan(const int64_t extents[3], int world, int ghost, const int periodic[3], int rank,
                     unsigned field_mask, int axis, int max_msgs, int64_t* out, int* n_out) {
  return guarded([&] {
    need(extents, "extents");
    need(n_out, "n_out");
    const long long ext[3] = {extents[0], extents[1], extents[2]};
    const double sp[3] = {1.0, 1.0, 1.0};
    const bool per[3] = {periodic && periodic[0] != 0, periodic && periodic[1] != 0,
                         periodic && periodic[2] != 0};
    const auto d = sfb::decompose(ext, sp, world, ghost, per);
    if (rank < 0 || rank >= world) throw sfb::error(SF_ERR_ARG, "rank out of range");
    std::vector<int> gid = {rank}, lid(world, -1), owner(world);
    lid[rank] = 0;
    for (int w = 0; w < world; ++w) owner[w] = w;
    const bool faces = axis < 0;
    const std::vector<int> axes = faces ? std::vector<int>{0, 1, 2} : std::vector<int>{axis};
    const auto P = sfb::build_phase_plan(d, gid, lid, owner, field_mask, axes, !faces, true, faces);
    // rows: kind (0 send, 1 recv, 2 local copy), peer, field, axis, side, lo[3], dims[3], dlo[3]
    int n = 0;
    auto emit = [&](int kind, int peer, const sfb::plan_box& b) {
      if (out && n < max_msgs) {
        int64_t* r = out + 15 * n;
        r[0] = kind;
        r[1] = peer;
        r[2] = b.field;
        r[3] = b.axis;
        r[4] = b.side;
        for (int a = 0; a < 3; ++a) {
          r[5 + a] = b.lo[a];
          r[8 + a] = b.dims[a];
          r[11 + a] = b.dlo[a];
        }
        r[14] = b.count;
      }
      ++n;
    };
    for (const auto& kv : P.sends)
      for (const auto& b : kv.second) emit(0, kv.first, b);
    for (const auto& kv : P.recvs)
      for (const auto& b : kv.second) emit(1, kv.first, b);
    for (const auto& b : P.copies) emit(2, rank, b);
    *n_out = n;
  });
}

int sf_sim_create_distributed(const sf_solver_config* cfg, const sf_fluid_params* par,
                              const sf_sim_options* opt, int rank, int world, const void* nccl_id,
                              sf_sim** out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(par, "par");
    need(out, "out");
    *out = nullptr;
    sf_sim_options o;
    if (opt) o = *opt; else sf_sim_options_default(&o);
    auto h = std::make_unique<sf_sim>();
    h->s = std::make_unique<sfb::simulation>(*cfg, *par, o, rank, world, nccl_id);
    *out = h.release();
  });
}

int sf_direct_plan(const int64_t extents[3], int world, int ghost, const int periodic[3], int rank, int max_boxes,
                   int64_t* out, int* n_out) {
  return guarded([&] {
    need(extents, "extents");
    need(n_out, "n_out");
    const long long ext[3] = {extents[0], extents[1], extents[2]};
    const double sp[3] = {1.0, 1.0, 1.0};
    const bool per[3] = {periodic && periodic[0] != 0, periodic && periodic[1] != 0,
                         periodic && periodic[2] != 0};
    const auto d = sfb::decompose(ext, sp, world, ghost, per);
    if (rank < 0 || rank >= world) throw sfb::error(SF_ERR_ARG, "rank out of range");
    const auto P = sfb::build_direct_plan(d, rank);
    // rows: peer, d[3], lo[3], dims[3], dlo[3], count
    int n = 0;
    for (const auto& b : P) {
      if (out && n < max_boxes) {
        int64_t* r = out + 14 * n;
        r[0] = b.peer;
        for (int a = 0; a < 3; ++a) {
          r[1 + a] = b.d[a];
          r[4 + a] = b.lo[a];
          r[7 + a] = b.dims[a];
          r[10 + a] = b.dlo[a];
        }
        r[13] = b.count;
      }
      ++n;
    }
    *n_out = n;
  });
}
int sf_sim_create_ipc(const sf_solver_config* cfg, const sf_fluid_params* par, const sf_sim_options* opt,
                      int rank, int world, const sf_host_transport* tr, sf_sim** out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(par, "par");
    need(tr, "transport");
    need(out, "out");
    *out = nullptr;
    sf_sim_options o;
    if (opt) o = *opt; else sf_sim_options_default(&o);
    auto h = std::make_unique<sf_sim>();
    h->s = std::make_unique<sfb::simulation>(*cfg, *par, o, rank, world, nullptr, tr);
    *out = h.release();
  });
}
int sf_sim_set_direct_exchange(sf_sim* s, int on) {
  return guarded([&] {
    need(s, "sim");
    s->s->set_direct(on);
  });
}
int sf_sim_direct_exchange(sf_sim* s) { return s ? s->s->direct_enabled() : 0; }
int sf_sim_rank(const sf_sim* s) { return s ? s->s->rank() : -1; }
int sf_sim_gather_block(sf_sim* s, const char* field, int worker, double* host, int64_t n) {
  return guarded([&] {
    need(s, "sim");
    s->s->block_io(s->s->field_id(field), worker, host, n, false);
  });
}
int sf_sim_scatter_block(sf_sim* s, const char* field, int worker, const double* host, int64_t n) {
  return guarded([&] {
    need(s, "sim");
    s->s->block_io(s->s->field_id(field), worker, const_cast<double*>(host), n, true);
  });
}
int sf_sim_gather_block_async(sf_sim* s, const char* field, int worker, double* host, int64_t n) {
  return guarded([&] {
    need(s, "sim");
    s->s->block_io(s->s->field_id(field), worker, host, n, false, true);
  });
}
int sf_sim_scatter_block_async(sf_sim* s, const char* field, int worker, const double* host, int64_t n) {
  return guarded([&] {
    need(s, "sim");
    s->s->block_io(s->s->field_id(field), worker, const_cast<double*>(host), n, true, true);
  });
}
int sf_sim_stage_block_async(sf_sim* s, const char* field, int worker, const double* host, int64_t n) {
  return guarded([&] {
    need(s, "sim");
    s->s->stage_block(s->s->field_id(field), worker, host, n);
  });
}
int sf_sim_install_staged(sf_sim* s, const char* field, int worker) {
  return guarded([&] {
    need(s, "sim");
    s->s->install_block(s->s->field_id(field), worker);
  });
}
int sf_sim_world(const sf_sim* s) { return s ? s->s->world() : 0; }

void sf_sim_options_default(sf_sim_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->workers = 1;
  o->mode = 0;
  o->ghost = 1;
  o->form = 0;
  o->device = 0;
  o->fused = 1;
  o->precision = 8;
}

int sf_sim_create(const sf_solver_config* cfg, const sf_fluid_params* par,
                  const sf_sim_options* opt, sf_sim** out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(par, "par");
    need(out, "out");
    *out = nullptr;
    sf_sim_options o;
    if (opt) o = *opt; else sf_sim_options_default(&o);
    auto h = std::make_unique<sf_sim>();
    h->s = std::make_unique<sfb::simulation>(*cfg, *par, o);
    *out = h.release();
  });
}

void sf_sim_destroy(sf_sim* s) { delete s; }

#define SIM(s) (need((s), "sim"), *(s)->s)

int sf_sim_init_cavity(sf_sim* s) { return guarded([&] { SIM(s).init_cavity(); }); }
int sf_sim_init_uniform(sf_sim* s, double cx, double cy, double cz) {
  return guarded([&] { SIM(s).init_uniform(cx, cy, cz); });
}
int sf_sim_init_taylor_green(sf_sim* s) { return guarded([&] { SIM(s).init_taylor_green(); }); }

int sf_sim_compute_dt(sf_sim* s, double* dt) {
  return guarded([&] {
    need(dt, "dt");
    *dt = SIM(s).compute_dt();
  });
}
int sf_sim_provisional(sf_sim* s, double dt) { return guarded([&] { SIM(s).provisional(dt); }); }
int sf_sim_pressure_iteration(sf_sim* s, double dt, int* sweeps, double* residual) {
  return guarded([&] {
    auto r = SIM(s).pressure_iteration(dt);
    if (sweeps) *sweeps = r.first;
    if (residual) *residual = r.second;
  });
}
int sf_sim_step(sf_sim* s, sf_step_stats* out) {
  return guarded([&] {
    auto r = SIM(s).step();
    if (out) *out = r;
  });
}
int sf_sim_advance(sf_sim* s, int n, sf_step_stats* last) {
  return guarded([&] {
    auto r = SIM(s).advance(n);
    if (last) *last = r;
  });
}
double sf_sim_time(const sf_sim* s) { return s ? s->s->time() : 0.0; }
long sf_sim_step_count(const sf_sim* s) { return s ? s->s->steps() : 0; }
int sf_sim_pending_color(sf_sim* s) {
  int c = -1;
  guarded([&] { c = SIM(s).pending_color(); });
  return c;
}
int sf_sim_max_divergence(sf_sim* s, double* out) {
  return guarded([&] { *out = SIM(s).max_divergence(); });
}
int sf_sim_steady_delta(sf_sim* s, double* out) {
  return guarded([&] { *out = SIM(s).steady_delta(); });
}
int sf_sim_taylor_green_error(sf_sim* s, double t, double* out) {
  return guarded([&] { *out = SIM(s).taylor_green_error(t); });
}
int sf_sim_kinetic_energy(sf_sim* s, double* out) {
  return guarded([&] { *out = SIM(s).kinetic_energy(); });
}

static void check_n(const sf_sim* s, int64_t n) {
  (void)s;
  if (n < 0) throw sfb::error(SF_ERR_ARG, "negative element count");
}

int sf_sim_scatter(sf_sim* s, const char* field, const double* host, int64_t n) {
  return guarded([&] {
    auto& S = SIM(s);
    need(host, "host");
    check_n(s, n);
    if (n != S.cells())
      throw sfb::error(SF_ERR_GRID, "scatter: global array has " + std::to_string(n) +
                                        " values, domain has " + std::to_string(S.cells()) + " cells");
    S.scatter(S.field_id(field), host);
  });
}
int sf_sim_gather(sf_sim* s, const char* field, double* host, int64_t n) {
  return guarded([&] {
    auto& S = SIM(s);
    need(host, "host");
    if (n < S.cells()) throw sfb::error(SF_ERR_ARG, "gather: host buffer too small");
    S.gather(S.field_id(field), host);
  });
}
int sf_sim_scatter_device(sf_sim* s, const char* field, const double* dev, int64_t n) {
  return guarded([&] {
    auto& S = SIM(s);
    need(dev, "dev");
    if (n != S.cells()) throw sfb::error(SF_ERR_GRID, "scatter: size mismatch");
    S.scatter_from_device(S.field_id(field), dev);
  });
}
int sf_sim_gather_device(sf_sim* s, const char* field, double* dev, int64_t n) {
  return guarded([&] {
    auto& S = SIM(s);
    need(dev, "dev");
    if (n < S.cells()) throw sfb::error(SF_ERR_ARG, "gather: device buffer too small");
    S.gather_to_device(S.field_id(field), dev);
  });
}
int sf_sim_checksum(sf_sim* s, uint64_t* out) {
  return guarded([&] {
    need(out, "out");
    *out = SIM(s).checksum();
  });
}
int sf_sim_local_front(sf_sim* s, const char* field, int worker, double* host, int64_t host_elems,
                       int64_t dims[3], int64_t lo[3]) {
  return guarded([&] {
    need(host, "host");
    long long d[3], l[3];
    SIM(s).local_front(SIM(s).field_id(field), worker, host, host_elems, d, l);
    for (int a = 0; a < 3; ++a) {
      dims[a] = d[a];
      lo[a] = l[a];
    }
  });
}
int sf_sim_refresh(sf_sim* s, const char* const* fields, int n) {
  return guarded([&] {
    auto& S = SIM(s);
    S.refresh(field_list(S, fields, n));
  });
}
int sf_sim_exchange(sf_sim* s, const char* const* fields, int n) {
  return guarded([&] {
    auto& S = SIM(s);
    S.exchange_only(field_list(S, fields, n));
  });
}
int sf_sim_run_kernel(sf_sim* s, const char* name, const char* const* param_names,
                      const double* param_values, int n_params, int region) {
  return guarded([&] {
    auto& S = SIM(s);
    std::map<std::string, double> pm;
    for (int i = 0; i < n_params; ++i) pm[param_names[i]] = param_values[i];
    S.run_kernel(name, pm, region);
  });
}
int sf_sim_reduce(sf_sim* s, const char* field, int op, double* out) {
  return guarded([&] {
    need(out, "out");
    if (op < 0 || op > 3) throw sfb::error(SF_ERR_ARG, "bad reduce op");
    *out = SIM(s).reduce(SIM(s).field_id(field), op);
  });
}
int sf_sim_create_field_typed(sf_sim* s, const char* name, int stagger, int value_bytes) {
  return guarded([&] {
    need(name, "name");
    SIM(s).create_field(name, stagger, value_bytes);
  });
}
int sf_sim_create_field(sf_sim* s, const char* name, int stagger) {
  return guarded([&] {
    need(name, "name");
    SIM(s).create_field(name, stagger);
  });
}

int sf_sim_register_kernel(sf_sim* s, const sf_plan* plan, const char* const* sig_fields, int n_sig_fields,
                           const char* const* sig_params, int n_sig_params, const char* point_body) {
  return guarded([&] {
    need(plan, "plan");
    need(plan->kernel, "plan->kernel");
    need(point_body, "point_body");
    std::array<int, 3> tile{plan->tile[0], plan->tile[1], plan->tile[2]};
    std::array<int, 6> halo{};
    for (int a = 0; a < 6; ++a) halo[a] = plan->halo[a];
    std::vector<std::string> bf, pr, sf, sp;
    std::vector<int> in, ca;
    for (int i = 0; i < plan->n_bindings; ++i) {
      bf.push_back(plan->bindings[i].field);
      in.push_back(plan->bindings[i].intent);
      ca.push_back(plan->bindings[i].cached);
    }
    for (int i = 0; i < plan->n_params; ++i) pr.push_back(plan->params[i]);
    for (int i = 0; i < n_sig_fields; ++i) sf.push_back(sig_fields[i]);
    for (int i = 0; i < n_sig_params; ++i) sp.push_back(sig_params[i]);
    SIM(s).register_kernel(plan->kernel, tile, halo, bf, in, ca, pr, sf, sp, point_body);
  });
}

int sf_sim_set_face_bc(sf_sim* s, int axis, int side, int kind, const double velocity[3]) {
  return guarded([&] { SIM(s).set_face_bc(axis, side, kind, velocity); });
}

int sf_sim_physical_bc(sf_sim* s, const char* const* fields, int n) {
  return guarded([&] {
    auto& S = SIM(s);
    S.physical_bc(field_list(S, fields, n));
  });
}

int sf_sim_run_schedule(sf_sim* s, const sf_schedule_step* steps, int n_steps, const char* const* param_names,
                        const double* param_values, int n_params, int passes, int mode) {
  return guarded([&] {
    (void)mode;  // overlap and plain give identical results (executor.hpp:812-861); one stream here
    auto& S = SIM(s);
    std::vector<sfb::simulation::sched_step> v;
    for (int i = 0; i < n_steps; ++i) {
      sfb::simulation::sched_step st;
      st.kind = steps[i].kind;
      if (steps[i].kernel) st.kernel = steps[i].kernel;
      st.reg = steps[i].region;
      for (int q = 0; q < steps[i].n_fields; ++q) st.fields.push_back(steps[i].fields[q]);
      if (steps[i].source) st.source = steps[i].source;
      if (steps[i].target) st.target = steps[i].target;
      st.op = steps[i].op;
      v.push_back(st);
    }
    std::map<std::string, double> pm;
    for (int i = 0; i < n_params; ++i) pm[param_names[i]] = param_values[i];
    S.run_schedule(v, pm, passes);
  });
}

int sf_sim_result(sf_sim* s, const char* name, double* value) {
  return guarded([&] {
    need(value, "value");
    if (!SIM(s).result(name, value)) throw sfb::error(SF_ERR_EXEC, std::string("no result named '") + name + "'");
  });
}

int sf_sim_invalidate_ghosts(sf_sim* s, const char* field) {
  return guarded([&] { SIM(s).invalidate(field); });
}
int sf_sim_invalidate_all_ghosts(sf_sim* s) { return guarded([&] { SIM(s).invalidate_all(); }); }
int sf_sim_ghosts_valid(sf_sim* s, const char* field) {
  int v = 0;
  guarded([&] { v = SIM(s).ghosts_valid(field) ? 1 : 0; });
  return v;
}
int sf_sim_synchronize(sf_sim* s) {
  return guarded([&] {
    SIM(s).sync();
    SIM(s).io_sync();
  });
}
void* sf_sim_stream(sf_sim* s) { return s ? (void*)s->s->stream() : nullptr; }
int64_t sf_sim_launch_count(sf_sim* s, int reset) { return s ? s->s->launch_count(reset != 0) : 0; }
int sf_sim_set_kernel_timing(sf_sim* s, int enable) {
  return guarded([&] { SIM(s).set_timing(enable != 0); });
}
int sf_sim_kernel_timing(sf_sim* s, const char* kernel, double* total_ms, int64_t* launches) {
  return guarded([&] {
    const std::string k = kernel ? kernel : "";
    if (k != "sweep_div" && k != "sweep2" && k != "sweep2i")
      throw sfb::error(SF_ERR_ARG, "timed kernels: sweep_div, sweep2, sweep2i");
    double ms = 0.0;
    long long n = 0;
    SIM(s).timing(k == "sweep2" ? 1 : k == "sweep2i" ? 2 : 0, &ms, &n);
    *total_ms = ms;
    *launches = n;
  });
}

// ---- level 2 -----------------------------------------------------------------
int sf_make_layout(const int64_t dims[3], const int64_t lo[3], int ghost, sf_layout* out) {
  return guarded([&] {
    need(out, "out");
    if (ghost < 0) throw sfb::error(SF_ERR_ARG, "ghost width must be >= 0");
    long long d[3] = {dims[0], dims[1], dims[2]}, l[3] = {lo[0], lo[1], lo[2]};
    *out = sfb::make_layout(d, l, ghost);
  });
}
int64_t sf_layout_elems(const sf_layout* l) { return l ? l->sx * l->sy * l->sz : 0; }

int sf_make_cfd_consts(const sf_solver_config* cfg, const sf_fluid_params* par, sf_cfd_consts* out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(par, "par");
    need(out, "out");
    sf_cfd_consts& s = *out;
    std::memset(&s, 0, sizeof s);
    s.nu = par->viscosity;
    s.alpha = par->blend;
    s.fx = par->body_force[0];
    s.fy = par->body_force[1];
    s.fz = par->body_force[2];
    s.ix = 1.0 / cfg->spacing[0];
    s.iy = 1.0 / cfg->spacing[1];
    s.iz = 1.0 / cfg->spacing[2];
    s.ix2 = s.ix * s.ix;
    s.iy2 = s.iy * s.iy;
    s.iz2 = s.iz * s.iz;
    s.nxm1 = cfg->extents[0] - 1;
    s.nym1 = cfg->extents[1] - 1;
    s.nzm1 = cfg->extents[2] - 1;
    s.px = cfg->periodic[0] ? 1 : 0;
    s.py = cfg->periodic[1] ? 1 : 0;
    s.pz = cfg->periodic[2] ? 1 : 0;
    auto act = [&](double ax, double ay, double az) { return ax * s.ix2 + ay * s.iy2 + az * s.iz2; };
    for (int bx = 0; bx < 2; ++bx)
      for (int by = 0; by < 2; ++by)
        for (int bz = 0; bz < 2; ++bz)
          s.bscale[bx][by][bz] = act(2.0, 2.0, 2.0) / act(bx ? 2.0 : 1.0, by ? 2.0 : 1.0, bz ? 2.0 : 1.0);
  });
}

int sf_launch_update_velocity(const sf_layout* l, const double* vx, const double* vy,
                              const double* vz, const double* p, double* vx_out, double* vy_out,
                              double* vz_out, const sf_cfd_consts* c, const sf_box* boxes, int nbox,
                              void* stream) {
  return guarded([&] {
    need(l, "layout");
    need(c, "consts");
    const int zc = 8;
    auto v = make_view(l, boxes, nbox, zc);
    const int nctas = v.b0.face[0];
    v.p[SF_VX][sfb::FRONT] = const_cast<double*>(vx);
    v.p[SF_VY][sfb::FRONT] = const_cast<double*>(vy);
    v.p[SF_VZ][sfb::FRONT] = const_cast<double*>(vz);
    v.p[SF_P][sfb::FRONT] = const_cast<double*>(p);
    v.p[SF_VX][sfb::BACK] = vx_out;
    v.p[SF_VY][sfb::BACK] = vy_out;
    v.p[SF_VZ][sfb::BACK] = vz_out;
    sfb::launch_update_velocity(v, nctas, zc, to_consts(c), nullptr, c->dt, as_stream(stream));
    check_last();
  });
}

int sf_launch_divergence(const sf_layout* l, const double* vx, const double* vy, const double* vz,
                         double* divu, const sf_cfd_consts* c, const sf_box* boxes, int nbox,
                         void* stream) {
  return guarded([&] {
    need(l, "layout");
    need(c, "consts");
    const int zc = 16;
    auto v = make_view(l, boxes, nbox, zc);
    const int nctas = v.b0.face[0];
    v.p[SF_VX][sfb::FRONT] = const_cast<double*>(vx);
    v.p[SF_VY][sfb::FRONT] = const_cast<double*>(vy);
    v.p[SF_VZ][sfb::FRONT] = const_cast<double*>(vz);
    v.p[SF_DIVU][sfb::FRONT] = divu;
    sfb::launch_divergence(v, nctas, zc, to_consts(c), nullptr, -1, 0, as_stream(stream));
    check_last();
  });
}

int sf_launch_pressure_sweep(const sf_layout* l, const double* divu, double* p, double* vx,
                             double* vy, double* vz, const sf_cfd_consts* c, double beta, int color,
                             const sf_box* boxes, int nbox, void* stream) {
  return guarded([&] {
    need(l, "layout");
    need(c, "consts");
    const int zc = 16;
    auto v = make_view(l, boxes, nbox, zc);
    const int nctas = v.b0.face[0];
    v.p[SF_DIVU][sfb::FRONT] = const_cast<double*>(divu);
    v.p[SF_P][sfb::FRONT] = p;
    v.p[SF_VX][sfb::FRONT] = vx;
    v.p[SF_VY][sfb::FRONT] = vy;
    v.p[SF_VZ][sfb::FRONT] = vz;
    const double bcd[3] = {beta, (double)color, c->dt};
    sfb::launch_pressure_sweep(v, nctas, zc, to_consts(c), nullptr, 0, bcd, as_stream(stream));
    check_last();
  });
}

int sf_launch_bc_face(const sf_layout* l, double* front, int stagger, int axis, int side,
                      const sf_face_bc* bc, int scope, void* stream) {
  return guarded([&] {
    need(l, "layout");
    need(bc, "bc");
    if (axis < 0 || axis > 2 || side < 0 || side > 1) throw sfb::error(SF_ERR_ARG, "bad face");
    if (bc->kind == SF_BC_UNSET)
      throw sfb::error(SF_ERR_GRID, std::string("no boundary condition on axis ") +
                                        std::to_string(axis) + (side == 0 ? " low" : " high") + " face");
    if (l->ghost == 0) return;
    const sf_box whole = {{0, 0, 0}, {l->dims[0], l->dims[1], l->dims[2]}};
    auto v = make_view(l, &whole, 1, 1);
    v.p[0][sfb::FRONT] = front;
    sfb::sf_task t{};
    t.type = 1;
    t.field = 0;
    t.axis = axis;
    t.side = side;
    t.kind = bc->kind;
    t.scope = scope;
    t.normal = stagger == axis;
    t.velocity = stagger >= 0;
    const double vwall = t.velocity ? bc->velocity[stagger] : 0.0;
    t.v = (t.normal && bc->kind == SF_BC_SYMMETRY) ? 0.0 : vwall;
    const long long g = l->ghost;
    for (int a = 0; a < 3; ++a) {
      if (a == axis) {
        t.lo[a] = 0;
        t.dims[a] = 1;
      } else if (a < axis) {
        t.lo[a] = -g;
        t.dims[a] = l->dims[a] + 2 * g;
      } else {
        t.lo[a] = 0;
        t.dims[a] = l->dims[a];
      }
    }
    t.count = t.dims[0] * t.dims[1] * t.dims[2];
    sfb::launch_task_one(v, t, as_stream(stream));
    check_last();
  });
}

int sf_launch_copy_box(const sf_layout* sl, const double* src, const sf_layout* dl, double* dst,
                       const int64_t src_lo[3], const int64_t dims[3], const int64_t dst_lo[3],
                       void* stream) {
  return guarded([&] {
    need(sl, "src layout");
    need(dl, "dst layout");
    const long long lo[3] = {src_lo[0], src_lo[1], src_lo[2]};
    const long long d[3] = {dims[0], dims[1], dims[2]};
    const long long m[3] = {dst_lo[0], dst_lo[1], dst_lo[2]};
    sfb::launch_copy_box(src, sl->base, sl->sx, sl->sy, dst, dl->base, dl->sx, dl->sy, lo, d, m,
                         as_stream(stream));
    check_last();
  });
}

int sf_launch_pack_box(const sf_layout* l, const double* src, const int64_t lo[3],
                       const int64_t dims[3], double* buf, void* stream) {
  return guarded([&] {
    need(l, "layout");
    const long long s[3] = {lo[0], lo[1], lo[2]};
    const long long d[3] = {dims[0], dims[1], dims[2]};
    const long long z[3] = {0, 0, 0};
    sfb::launch_copy_box(src, l->base, l->sx, l->sy, buf, 0, d[0], d[1], s, d, z, as_stream(stream));
    check_last();
  });
}

int sf_launch_unpack_box(const sf_layout* l, double* dst, const int64_t lo[3],
                         const int64_t dims[3], const double* buf, void* stream) {
  return guarded([&] {
    need(l, "layout");
    const long long s[3] = {lo[0], lo[1], lo[2]};
    const long long d[3] = {dims[0], dims[1], dims[2]};
    const long long z[3] = {0, 0, 0};
    sfb::launch_copy_box(buf, 0, d[0], d[1], dst, l->base, l->sx, l->sy, z, d, s, as_stream(stream));
    check_last();
  });
}

int sf_launch_reduce_max(const sf_layout* l, const double* front, const double* back, int op,
                         double* dev_out, void* stream) {
  return guarded([&] {
    need(l, "layout");
    need(dev_out, "dev_out");
    if (op != SF_MAX_ABS && op != SF_MAX_ABS_DIFF) throw sfb::error(SF_ERR_ARG, "op must be a max op");
    if (op == SF_MAX_ABS_DIFF && !back) throw sfb::error(SF_ERR_GRID, "no back buffer to diff against");
    const sf_box whole = {{0, 0, 0}, {l->dims[0], l->dims[1], l->dims[2]}};
    const int zc = 16;
    auto v = make_view(l, &whole, 1, zc);
    const int nctas = v.b0.face[0];
    v.p[0][sfb::FRONT] = const_cast<double*>(front);
    v.p[0][sfb::BACK] = const_cast<double*>(back);
    const int fl[1] = {0};
    sfb::launch_reduce_max(v, nctas, zc, fl, 1, op == SF_MAX_ABS_DIFF ? 1 : 0,
                           reinterpret_cast<unsigned long long*>(dev_out), as_stream(stream));
    check_last();
  });
}

}  // extern "C"
