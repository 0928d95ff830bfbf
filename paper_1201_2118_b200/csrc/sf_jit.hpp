// sf_jit.hpp -- descriptor-declared stencil kernels, generated and compiled on
// the fly for sm_100a (the B200 form of CaCUDA's "kernel descriptor ->
// generated CUDA tile template"; reference API
// exec::executor::register_kernel, executor.hpp:484-488, 650-692).
//
// The user supplies the BODY of a point function written against the
// reference's point_ctx / cell_view API (executor.hpp:130-184):
//     c.field(s)(di, dj, dk)   read at an offset inside the declared halo
//     c.field(s).load()        read the centre
//     c.field(s).store(v)      write the centre (OUT, INOUT, SEPARATEINOUT)
//     c.param(s)               parameter value in plan order
//     c.i, c.j, c.k            global cell index
// The body is pasted into a tile template (one 2-D column tile per CTA from
// the plan's TILE, marching z, reads through the read-only path) and compiled
// with NVRTC.  SEPARATEINOUT bindings read the front buffer and write the
// back buffer; the executor swaps after the run (executor.hpp:769-779).
#pragma once

#include <dlfcn.h>

#include <string>

namespace sfb {

struct nvrtc_api {
  typedef int (*create_t)(void**, const char*, const char*, int, const char* const*, const char* const*);
  typedef int (*compile_t)(void*, int, const char* const*);
  typedef int (*size_t_fn)(void*, size_t*);
  typedef int (*get_t)(void*, char*);
  typedef int (*destroy_t)(void**);
  typedef const char* (*err_t)(int);
  create_t create = nullptr;
  compile_t compile = nullptr;
  size_t_fn log_size = nullptr;
  get_t log = nullptr;
  size_t_fn cubin_size = nullptr;
  get_t cubin = nullptr;
  destroy_t destroy = nullptr;
  err_t err = nullptr;
};

inline nvrtc_api* nvrtc() {
  static nvrtc_api api;
  static bool tried = false;
  if (tried) return api.create ? &api : nullptr;
  tried = true;
  const char* names[] = {getenv("SF_NVRTC_LIB"), "libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12",
                         "libnvrtc.so"};
  void* h = nullptr;
  for (const char* n : names)
    if (n && (h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return nullptr;
  api.create = (nvrtc_api::create_t)dlsym(h, "nvrtcCreateProgram");
  api.compile = (nvrtc_api::compile_t)dlsym(h, "nvrtcCompileProgram");
  api.log_size = (nvrtc_api::size_t_fn)dlsym(h, "nvrtcGetProgramLogSize");
  api.log = (nvrtc_api::get_t)dlsym(h, "nvrtcGetProgramLog");
  api.cubin_size = (nvrtc_api::size_t_fn)dlsym(h, "nvrtcGetCUBINSize");
  api.cubin = (nvrtc_api::get_t)dlsym(h, "nvrtcGetCUBIN");
  api.destroy = (nvrtc_api::destroy_t)dlsym(h, "nvrtcDestroyProgram");
  api.err = (nvrtc_api::err_t)dlsym(h, "nvrtcGetErrorString");
  if (!api.create || !api.compile || !api.cubin || !api.cubin_size) api.create = nullptr;
  return api.create ? &api : nullptr;
}

// The tile template.  SF_NB bindings, SF_NP parameters, SF_TX x SF_TY threads,
// SF_MAXF fields / SF_SLOTS slots per block in the device pointer table.
inline const char* jit_template() {
  return R"JIT(
struct sf_work { int blk; int cta_begin; int tiles[3]; long long lo[3], hi[3]; };
struct sf_params { double v[SF_NP > 0 ? SF_NP : 1]; };
struct sf_geo { long long n[3], lo[3], sx, sy, base; };

// Debug policing (SF_DEBUG_BOUNDS, executor.hpp:153-172): the first
// violation is recorded as {code, slot, di, dj, dk} and the access skipped;
// the host raises exec_error with the reference's text after the launch.
__device__ int* sf_err_word;
__device__ __forceinline__ void sf_violation(int code, int slot, int di, int dj, int dk) {
  if (atomicCAS(sf_err_word, 0, code) == 0) {
    sf_err_word[1] = slot;
    sf_err_word[2] = di;
    sf_err_word[3] = dj;
    sf_err_word[4] = dk;
  }
}

struct cell_view {
  const double* rd;
  double* wr;
  long long o, sx, sxy;
  int slot;
  __device__ __forceinline__ sf_real operator()(int di, int dj, int dk) const {
#if SF_DEBUG
    if (!SF_READABLE[slot]) { sf_violation(1, slot, di, dj, dk); return 0.0; }
    if (SF_CENTER_ONLY[slot] && (di != 0 || dj != 0 || dk != 0)) { sf_violation(2, slot, di, dj, dk); return 0.0; }
    if (di < -SF_HALO[0] || di > SF_HALO[1] || dj < -SF_HALO[2] || dj > SF_HALO[3] || dk < -SF_HALO[4] ||
        dk > SF_HALO[5]) { sf_violation(3, slot, di, dj, dk); return 0.0; }
#endif
    const long long q = o + di + dj * sx + dk * sxy;
    // fp32 fields widen to fp64 unless the whole kernel runs in fp32 (sf_real)
    return SF_F32[slot] ? (sf_real)reinterpret_cast<const float*>(rd)[q] : (sf_real)rd[q];
  }
  __device__ __forceinline__ sf_real load() const { return (*this)(0, 0, 0); }
  __device__ __forceinline__ void store(sf_real v) const {
#if SF_DEBUG
    if (!SF_WRITABLE[slot]) { sf_violation(4, slot, 0, 0, 0); return; }
#endif
    if (SF_F32[slot])
      reinterpret_cast<float*>(wr)[o] = (float)v;  // fp32 fields round to nearest
    else
      __stwb(wr + o, (double)v);
  }
};

struct point_ctx {
  cell_view f_[SF_NB];
  const double* p_;
  long long i, j, k;
  __device__ __forceinline__ const cell_view& field(int s) const { return f_[s]; }
  __device__ __forceinline__ double param(int s) const { return p_[s]; }
};

__device__ __forceinline__ void sf_user_point(const point_ctx& c) {
SF_BODY
}

extern "C" __global__ void __launch_bounds__(SF_TX * SF_TY)
sf_user_kernel(double* const* __restrict__ ptrs, const sf_geo* __restrict__ geo,
               const sf_work* __restrict__ items, int nitems, int zc, sf_params prm) {
  const int cta = blockIdx.x;
  int lo_i = 0, hi_i = nitems - 1;
  while (lo_i < hi_i) {
    const int mid = (lo_i + hi_i + 1) >> 1;
    if (items[mid].cta_begin <= cta) lo_i = mid; else hi_i = mid - 1;
  }
  const sf_work& w = items[lo_i];
  const int local = cta - w.cta_begin;
  const int tx = local % w.tiles[0];
  const int ty = (local / w.tiles[0]) % w.tiles[1];
  const int tz = local / (w.tiles[0] * w.tiles[1]);
  const long long i = w.lo[0] + (long long)tx * SF_TX + threadIdx.x;
  const long long j = w.lo[1] + (long long)ty * SF_TY + threadIdx.y;
  if (i >= w.hi[0] || j >= w.hi[1]) return;
  const long long k0 = w.lo[2] + (long long)tz * zc;
  const long long k1 = k0 + zc < w.hi[2] ? k0 + zc : w.hi[2];
  const sf_geo& G = geo[w.blk];
  const long long sx = G.sx, sxy = G.sx * G.sy;
  __shared__ double sp[SF_NP > 0 ? SF_NP : 1];
  point_ctx c;
  c.p_ = prm.v;
  (void)sp;
#pragma unroll
  for (int s = 0; s < SF_NB; ++s) {
    c.f_[s].rd = ptrs[(w.blk * SF_MAXF + SF_FID[s]) * SF_SLOTS + 0];
    c.f_[s].wr = ptrs[(w.blk * SF_MAXF + SF_FID[s]) * SF_SLOTS + SF_WSLOT[s]];
    c.f_[s].sx = sx;
    c.f_[s].sxy = sxy;
    c.f_[s].slot = s;
  }
  c.i = G.lo[0] + i;
  c.j = G.lo[1] + j;
  for (long long k = k0; k < k1; ++k) {
    const long long o = G.base + (k * G.sy + j) * sx + i;
#pragma unroll
    for (int s = 0; s < SF_NB; ++s) c.f_[s].o = o;
    c.k = G.lo[2] + k;
    sf_user_point(c);
  }
}
)JIT";
}

// The TMA-staged variant for plans with CACHED readable bindings (the CaCUDA
// template: "shared arrays with appropriate stencil sizes ... streamed in while
// calculations proceed").  Each cached binding gets a ring
// of SF_R z planes in shared memory, one (SF_BW x SF_BH) halo box per plane,
// filled by cp.async.bulk.tensor and guarded by one mbarrier per ring slot;
// the CTA marches its z chunk and refills the slot of the plane that left the
// stencil window.  Uncached bindings read global memory directly.
inline const char* jit_template_tma() {
  return R"JIT(
struct sf_work { int blk; int cta_begin; int tiles[3]; long long lo[3], hi[3]; };
struct sf_params { double v[SF_NP > 0 ? SF_NP : 1]; };
struct sf_geo { long long n[3], lo[3], sx, sy, base; };
struct __align__(64) sf_tmap { unsigned long long opaque[16]; };

__device__ int* sf_err_word;
__device__ __forceinline__ void sf_violation(int code, int slot, int di, int dj, int dk) {
  if (atomicCAS(sf_err_word, 0, code) == 0) {
    sf_err_word[1] = slot; sf_err_word[2] = di; sf_err_word[3] = dj; sf_err_word[4] = dk;
  }
}
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

constexpr int SF_PLANE = (SF_BW * SF_BH + 15) / 16 * 16;  // 128-byte aligned ring planes

constexpr int SF_ZW = SF_HALO[4] + SF_HALO[5] + 1;  // z window of the stencil
template <int N> struct sf_ic { static constexpr int value = N; };

struct cell_view {
  const double* rd;
  double* wr;
  long long o, sx, sxy;
  int slot;
  const double* rb;  // cached: ring base of this binding (fp32 planes hold floats)
  int e0;            // cached: this cell's in-plane element (shared index arithmetic lets two rows' loads fold)
  int zoff[SF_ZW];   // cached: ring-plane offset for dk = t - halo_lo_z (updated per plane)
  // cached: this column's values of the z window, plane z in slot z % SF_ZW
  // (a circular register queue: nothing shifts; ph = this plane's slot is a
  // compile-time constant in every unrolled plane body)
  sf_real zq[SF_ZW];
  int ph;
  mutable sf_real dv;  // SF_RPT > 1: the deferred store of this cell
  mutable bool dw;
  __device__ __forceinline__ sf_real operator()(int di, int dj, int dk) const {
#if SF_DEBUG
    if (!SF_READABLE[slot]) { sf_violation(1, slot, di, dj, dk); return 0.0; }
    if (SF_CENTER_ONLY[slot] && (di != 0 || dj != 0 || dk != 0)) { sf_violation(2, slot, di, dj, dk); return 0.0; }
    if (di < -SF_HALO[0] || di > SF_HALO[1] || dj < -SF_HALO[2] || dj > SF_HALO[3] || dk < -SF_HALO[4] ||
        dk > SF_HALO[5]) { sf_violation(3, slot, di, dj, dk); return 0.0; }
#endif
    // the column itself comes from the register queue: one shared-memory load
    // per plane instead of one per z offset (offsets fold to constants)
    if (SF_CACHED[slot] && di == 0 && dj == 0) return zq[(ph + dk + SF_ZW) % SF_ZW];
    if (SF_CACHED[slot]) return ring(zoff[dk + SF_HALO[4]], dj * SF_BW + di);
    const long long q = o + di + dj * sx + dk * sxy;
    if (SF_F32[slot]) {  // fp32 fields widen exactly (to sf_real)
      const float* f = reinterpret_cast<const float*>(rd);
      return (sf_real)(SF_CENTER_ONLY[slot] ? __ldcg(f + q) : __ldg(f + q));
    }
    return (sf_real)(SF_CENTER_ONLY[slot] ? __ldcg(rd + q) : __ldg(rd + q));
  }
  // ring plane at offset zo (in fp64 slots; an fp32 plane uses the first half),
  // element e of the box relative to this cell
  __device__ __forceinline__ sf_real ring(int zo, int e) const {
    if (SF_F32[slot]) return (sf_real)reinterpret_cast<const float*>(rb)[2 * zo + e0 + e];
    return (sf_real)rb[zo + e0 + e];
  }
  __device__ __forceinline__ sf_real load() const { return (*this)(0, 0, 0); }
  __device__ __forceinline__ void store(sf_real v) const {
#if SF_DEBUG
    if (!SF_WRITABLE[slot]) { sf_violation(4, slot, 0, 0, 0); return; }
#endif
#if SF_RPT > 1
    dv = v;  // written after both rows' bodies (the last store of a body wins)
    dw = true;
#else
    put(v);
#endif
  }
  __device__ __forceinline__ void put(sf_real v) const {
    if (SF_F32[slot])
      reinterpret_cast<float*>(wr)[o] = (float)v;  // fp32 fields round to nearest
    else
      __stwb(wr + o, (double)v);
  }
};

struct point_ctx {
  cell_view f_[SF_NB];
  const double* p_;
  long long i, j, k;
  __device__ __forceinline__ const cell_view& field(int s) const { return f_[s]; }
  __device__ __forceinline__ double param(int s) const { return p_[s]; }
};

__device__ __forceinline__ void sf_user_point(const point_ctx& c) {
SF_BODY
}

// SF_ROWS(stmt): stmt once per row r = 0 .. SF_RPT - 1 of the thread, with r
// a compile-time constant and crow that row's context (the locals c0 .. c3,
// picked by name so they stay in registers)
#define SF_ROW_DO(R, ...) if constexpr ((R) < SF_RPT) { constexpr int r = (R); point_ctx& crow = c##R; (void)r; (void)crow; __VA_ARGS__ }
#define SF_ROWS(...) SF_ROW_DO(0, __VA_ARGS__) SF_ROW_DO(1, __VA_ARGS__) SF_ROW_DO(2, __VA_ARGS__) SF_ROW_DO(3, __VA_ARGS__)

extern "C" __global__ void SF_LAUNCH_BOUNDS
sf_user_kernel(double* const* __restrict__ ptrs, const sf_geo* __restrict__ geo,
               const sf_work* __restrict__ items, int nitems, int zc, sf_params prm,
               const unsigned char* __restrict__ bidx, const sf_tmap* __restrict__ maps) {
  extern __shared__ __align__(128) double sring[];
  __shared__ __align__(8) unsigned long long bars[SF_R];
  const int cta = blockIdx.x;
  int lo_i = 0, hi_i = nitems - 1;
  while (lo_i < hi_i) {
    const int mid = (lo_i + hi_i + 1) >> 1;
    if (items[mid].cta_begin <= cta) lo_i = mid; else hi_i = mid - 1;
  }
  const sf_work& w = items[lo_i];
  const int local = cta - w.cta_begin;
  const int tix = local % w.tiles[0];
  const int tiy = (local / w.tiles[0]) % w.tiles[1];
  const int tiz = local / (w.tiles[0] * w.tiles[1]);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * SF_TX + tx;
  const long long i0 = w.lo[0] + (long long)tix * SF_TX, j0 = w.lo[1] + (long long)tiy * (SF_TY * SF_RPT);
  const long long i = i0 + tx, j = j0 + SF_RPT * ty;  // rows j .. j + SF_RPT - 1
  const long long k0 = w.lo[2] + (long long)tiz * zc;
  const long long k1 = k0 + zc < w.hi[2] ? k0 + zc : w.hi[2];
  const int nplanes = (int)(k1 - k0);
  const int nload = nplanes + SF_HALO[4] + SF_HALO[5];  // planes k0-hzl .. k1-1+hzh
  const sf_geo& G = geo[w.blk];
  const long long sx = G.sx, sxy = G.sx * G.sy;
  const int g = (int)(G.base / sxy);  // ghost width: base = (g*sy + g)*sx + xo
  const int xo = (int)(G.base % G.sx);
  const int xcs = xo + (int)i0 - SF_XL, ycs = g + (int)j0 - SF_HALO[2], zcs = g + (int)k0 - SF_HALO[4];

  if (tid == 0) {
    for (int q = 0; q < SF_R; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {  // load plane q (z = k0 - hzl + q) of every cached binding
    const int slot = q % SF_R;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[slot])),
                 "r"((unsigned)(SF_TXB)) : "memory");
    for (int c = 0; c < SF_NC; ++c) {
      const int b = SF_CSLOT[c];
      const int phys = bidx[(w.blk * SF_MAXF + SF_FID[b]) * SF_SLOTS + 0];
      const sf_tmap* m = &maps[((w.blk * SF_NC) + c) * SF_SLOTS + phys];
      double* dst = sring + (c * SF_R + slot) * SF_PLANE;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sa(dst)), "l"((unsigned long long)m),
          "r"(sa(&bars[slot])), "r"(xcs), "r"(ycs), "r"(zcs + q) : "memory");
    }
  };
  auto wait = [&](int q) {
    const unsigned par = (unsigned)((q / SF_R) & 1);
    asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 " @!P1 bra W_%=;\n}" ::"r"(sa(&bars[q % SF_R])), "r"(par) : "memory");
  };
  if (tid == 0)
    for (int q = 0; q < SF_R && q < nload; ++q) issue(q);

  const bool act = i < w.hi[0] && j < w.hi[1];
  point_ctx c0, c1, c2, c3;  // rows j .. j + SF_RPT - 1 of this thread (SF_ROWS)
  const long long jleft = w.hi[1] - j;  // row r is active when act && r < jleft
  SF_ROWS({
    point_ctx& c = crow;
    c.p_ = prm.v;
#pragma unroll
    for (int s = 0; s < SF_NB; ++s) {
      c.f_[s].rd = ptrs[(w.blk * SF_MAXF + SF_FID[s]) * SF_SLOTS + 0];
      c.f_[s].wr = ptrs[(w.blk * SF_MAXF + SF_FID[s]) * SF_SLOTS + SF_WSLOT[s]];
      c.f_[s].sx = sx;
      c.f_[s].sxy = sxy;
      c.f_[s].slot = s;
      c.f_[s].rb = sring + SF_CIDX[s] * SF_R * SF_PLANE;  // ring base of this binding
      c.f_[s].e0 = ((int)(j - j0) + r + SF_HALO[2]) * SF_BW + tx + SF_XL;  // this cell's in-plane element
    }
    c.i = G.lo[0] + i;
    c.j = G.lo[1] + j + r;
  })
  for (int q = 0; q < SF_HALO[4] + SF_HALO[5] && q < nload; ++q) wait(q);
  long long o = G.base + (k0 * G.sy + j) * sx + i;
  int zr[SF_ZW];  // rolling ring-plane offsets of the z window
#pragma unroll
  for (int t = 0; t < SF_ZW; ++t) zr[t] = (t % SF_R) * SF_PLANE;
  // two planes per barrier round: the fixed per-round work (waits, barrier,
  // refills, ring offsets) is shared by two cells per thread
  for (int kk = 0; kk < nplanes; kk += 2) {
    const bool two = kk + 1 < nplanes;
    const int qn = kk + SF_HALO[4] + SF_HALO[5];
    if (qn < nload) wait(qn);
    if (two && qn + 1 < nload) wait(qn + 1);
    if (act) {
      // plane kq's body with its queue slot PH = kq % SF_ZW known at compile time
      auto plane = [&](auto phc, int kq) {
        constexpr int PH = decltype(phc)::value;
        auto setup = [&](point_ctx& cc, long long oc) {
#pragma unroll
          for (int s = 0; s < SF_NB; ++s) {
            cc.f_[s].o = oc;
            cc.f_[s].ph = PH;
            cc.f_[s].dw = false;
#pragma unroll
            for (int t = 0; t < SF_ZW; ++t) cc.f_[s].zoff[t] = zr[t];
            if (SF_CACHED[s]) {  // column queue: load the plane that entered the window
              if (kq == 0) {
#pragma unroll
                for (int t = 0; t < SF_ZW; ++t)
                  cc.f_[s].zq[(PH + t - SF_HALO[4] + SF_ZW) % SF_ZW] = cc.f_[s].ring(zr[t], 0);
              } else {
                cc.f_[s].zq[(PH + SF_HALO[5]) % SF_ZW] = cc.f_[s].ring(zr[SF_ZW - 1], 0);
              }
            }
          }
          cc.k = G.lo[2] + k0 + kq;
        };
        SF_ROWS(setup(crow, o + r * sx);)
#if SF_RPT > 1
        SF_ROWS(if (r < jleft) sf_user_point(crow);)
        SF_ROWS({  // the rows' deferred stores
          const point_ctx& c = crow;
          if (r < jleft) {
#pragma unroll
            for (int s = 0; s < SF_NB; ++s)
              if (SF_WRITABLE[s] && c.f_[s].dw) c.f_[s].put(c.f_[s].dv);
          }
        })
#else
        sf_user_point(c0);
#endif
        o += sxy;
#pragma unroll
        for (int t = 0; t < SF_ZW - 1; ++t) zr[t] = zr[t + 1];
        zr[SF_ZW - 1] = ((kq + SF_ZW) % SF_R) * SF_PLANE;
      };
#define SF_PLANES(P)                                              \
  case P:                                                         \
    plane(sf_ic<(P) % SF_ZW>{}, kk);                              \
    if (two) plane(sf_ic<((P) + 1) % SF_ZW>{}, kk + 1);           \
    break;
      switch (kk % SF_ZW) {
        SF_PLANE_CASES
      }
#undef SF_PLANES
    }
    __syncthreads();  // planes kk, kk+1 (ring q = kk, kk+1) left every window
    if (tid == 0) {
      if (kk + SF_R < nload) issue(kk + SF_R);
      if (two && kk + 1 + SF_R < nload) issue(kk + 1 + SF_R);
    }
  }
}
)JIT";
}

}  // namespace sfb
