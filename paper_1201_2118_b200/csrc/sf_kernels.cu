// sf_kernels.cu -- sm_100a kernels of the staggered-grid stencil hot path.
//
// Every arithmetic expression keeps the association order of the reference
// (cfd.hpp:524-720) and the library is compiled with --fmad=false, so each
// cell is bitwise identical to the reference CPU implementation.
//
// Kernels (reference function each replaces):
//   k_tasks        ghost refresh phase: exchange copies + bc_face (exchange.hpp:98-480)
//   k_update_vel   UPDATE_VELOCITY point kernel (cfd.hpp:524-589) + NaN-guard maxima
//   k_divergence   DIVERGENCE (cfd.hpp:595-618) + max|divu| epilogue (reductions.hpp:28-90)
//   k_sweep        PRESSURE_SWEEP (cfd.hpp:630-720), in place
//   k_sweep_div    fused half-sweep: PRESSURE_SWEEP + velocity refresh + DIVERGENCE +
//                  max|divu| + the loop test of pressure_iteration (cfd.hpp:295-303)
//   k_reduce_*     grid::reduce (reductions.hpp:28-90)
//   k_ctl          compute_dt / beta / loop bookkeeping (cfd.hpp:264-305)
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <set>
#include <utility>

#include "sf_kernels.cuh"
#include "sf_uv.cuh"

namespace sfb {

// ---------------------------------------------------------------------------
// tile location
// ---------------------------------------------------------------------------
struct tile_loc {
  int item;
  int blk;
  long long i, j, k0, k1;
  bool act;
};

__device__ __forceinline__ tile_loc locate_at(const sf_work* __restrict__ items, int nitems, int zc, int cta) {
  tile_loc t;
  t.item = nitems > 1 ? find_item(items, nitems, cta) : 0;
  const sf_work& w = items[t.item];
  t.blk = w.blk;
  const int local = cta - w.cta_begin;
  const int tx = local % w.tiles[0];
  const int ty = (local / w.tiles[0]) % w.tiles[1];
  const int tz = local / (w.tiles[0] * w.tiles[1]);
  t.i = w.lo[0] + (long long)tx * kTX + threadIdx.x;
  t.j = w.lo[1] + (long long)ty * kTY + threadIdx.y;
  t.k0 = w.lo[2] + (long long)tz * zc;
  t.k1 = min(t.k0 + zc, w.hi[2]);
  t.act = t.i < w.hi[0] && t.j < w.hi[1];
  return t;
}
__device__ __forceinline__ tile_loc locate(const sf_work* __restrict__ items, int nitems, int zc) {
  return locate_at(items, nitems, zc, blockIdx.x);
}

__device__ __forceinline__ bool pred_done(const sf_dev_ctl* ctl) {
  return *reinterpret_cast<const volatile int*>(&ctl->done) != 0;
}

// ---------------------------------------------------------------------------
// ghost refresh tasks
// ---------------------------------------------------------------------------
// bc_face (exchange.hpp:231-480) on element type E: one thread per
// tangential line. For fp64 the arithmetic is the reference's (2.0 * v - src).
template <class E>
__device__ __forceinline__ void bc_task(const sf_task& T, const sf_dev_block& B, E* f, long long stride) {
  const int a = T.axis;
  const int t1 = a == 0 ? 1 : 0;
  const int t2 = a == 2 ? 1 : 2;
  const long long g = B.g, b = B.n[a];
  const long long n1 = T.dims[t1];
  const long long astr = a == 0 ? 1 : (a == 1 ? B.sx : B.sx * B.sy);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < T.count; e += stride) {
    long long c[3];
    c[t1] = T.lo[t1] + e % n1;
    c[t2] = T.lo[t2] + e / n1;
    c[a] = 0;
    const long long o0 = off(B, c[0], c[1], c[2]);  // position 0 along the axis
#define LINE(pos) f[o0 + (long long)(pos) * astr]
    const E v = (E)T.v;
    if (T.normal) {
      if (T.kind == SF_BC_WALL || T.kind == SF_BC_SYMMETRY) {
        if (T.side == 0) {
          if (T.scope != SF_SCOPE_OWNED_ONLY) {
            LINE(-1) = v;
            for (long long m = 2; m <= g; ++m) {
              const E src = LINE(m - 2);
              LINE(-m) = (E)2 * v - src;
            }
          }
        } else {
          bool tang_owned = true;
          for (int t = 0; t < 3; ++t)
            if (t != a && (c[t] < 0 || c[t] >= B.n[t])) tang_owned = false;
          if (T.scope == SF_SCOPE_ALL || (T.scope == SF_SCOPE_OWNED_ONLY && tang_owned) ||
              (T.scope == SF_SCOPE_GHOSTS_ONLY && !tang_owned))
            LINE(b - 1) = v;
          if (T.scope != SF_SCOPE_OWNED_ONLY)
            for (long long m = 1; m <= g; ++m) {
              const E src = LINE(b - 1 - m);
              LINE(b - 1 + m) = (E)2 * v - src;
            }
        }
      } else if (T.kind == SF_BC_OUTFLOW && T.scope != SF_SCOPE_OWNED_ONLY) {
        if (T.side == 0) {
          const E v0 = LINE(0);
          for (long long m = 1; m <= g; ++m) LINE(-m) = v0;
        } else {
          const E v0 = LINE(b - 1);
          for (long long m = 1; m <= g; ++m) LINE(b - 1 + m) = v0;
        }
      }
    } else if (T.scope != SF_SCOPE_OWNED_ONLY) {
      if (T.kind == SF_BC_WALL && T.velocity) {
        if (T.side == 0)
          for (long long m = 1; m <= g; ++m) {
            const E src = LINE(m - 1);
            LINE(-m) = (E)2 * v - src;
          }
        else
          for (long long m = 1; m <= g; ++m) {
            const E src = LINE(b - m);
            LINE(b - 1 + m) = (E)2 * v - src;
          }
      } else if (T.kind == SF_BC_WALL || T.kind == SF_BC_SYMMETRY) {
        if (T.side == 0)
          for (long long m = 1; m <= g; ++m) LINE(-m) = LINE(m - 1);
        else
          for (long long m = 1; m <= g; ++m) LINE(b - 1 + m) = LINE(b - m);
      } else if (T.kind == SF_BC_OUTFLOW) {
        if (T.side == 0) {
          const E v0 = LINE(0);
          for (long long m = 1; m <= g; ++m) LINE(-m) = v0;
        } else {
          const E v0 = LINE(b - 1);
          for (long long m = 1; m <= g; ++m) LINE(b - 1 + m) = v0;
        }
      }
    }
#undef LINE
  }
}

// One refresh task. Box copies of rows at least a warp wide go warp per
// row (one 64-bit div/mod per row, not per element; each warp moves a
// contiguous run); narrow boxes (the x faces, 1-3 cells wide) go element per
// thread.
template <class View, class F>
__device__ __forceinline__ void for_box_elems(const sf_task& T, F&& body) {
  const long long nx = T.dims[0], ny = T.dims[1], rows = T.dims[1] * T.dims[2];
  if (nx >= 32) {
    const int lane = threadIdx.x & 31;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long ws = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w0; r < rows; r += ws) {
      const long long kk = r / ny, jj = r - kk * ny;
      for (long long ii = lane; ii < nx; ii += 32) body(r * nx + ii, ii, jj, kk);
    }
  } else {
    const long long nxy = nx * ny, stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < T.count; e += stride) {
      const long long kk = e / nxy, rem = e - kk * nxy, jj = rem / nx, ii = rem - jj * nx;
      body(e, ii, jj, kk);
    }
  }
}

template <class View>
__device__ __forceinline__ void run_task(const View& vw, const sf_task& T) {
  const bool f32 = vw.esize(T.field) == 4;
  if (T.type == 2 || T.type == 3) {  // message pack / unpack (exchange.hpp:165-224)
    // fp32 values travel as exact fp64 conversions (message sizes stay fp64)
    const sf_dev_block& Bk = vw.blk(T.dst_blk);
    double* f = vw.ptr(T.dst_blk, T.field, FRONT);
    float* ff = reinterpret_cast<float*>(f);
    double* buf = T.buf;
    const bool pack = T.type == 2;
    for_box_elems<View>(T, [&](long long e, long long ii, long long jj, long long kk) {
      const long long o = off(Bk, T.lo[0] + ii, T.lo[1] + jj, T.lo[2] + kk);
      if (pack)
        buf[e] = f32 ? (double)ff[o] : f[o];
      else if (f32)
        ff[o] = (float)buf[e];
      else
        f[o] = buf[e];
    });
    return;
  }
  if (T.type == 4) {  // direct store into a peer's ghost region (fp64 CFD fields)
    const sf_dev_block& S = vw.blk(T.src_blk);
    const double* src = vw.ptr(T.src_blk, T.field, T.slot);
    double* dst = T.rptr[vw.phys(T.src_blk, T.field, T.slot)];
    for_box_elems<View>(T, [&](long long, long long ii, long long jj, long long kk) {
      dst[T.rbase + ((T.dlo[2] + kk) * T.rsy + T.dlo[1] + jj) * T.rsx + T.dlo[0] + ii] =
          src[off(S, T.lo[0] + ii, T.lo[1] + jj, T.lo[2] + kk)];
    });
    // the stores cross to another device or process: make them visible
    // system-wide before this kernel completes (the max-allreduce that
    // follows on this stream is what the peer waits for)
    __threadfence_system();
    return;
  }
  if (T.type == 0) {  // box copy between blocks of this process
    const sf_dev_block& S = vw.blk(T.src_blk);
    const sf_dev_block& D = vw.blk(T.dst_blk);
    const double* src = vw.ptr(T.src_blk, T.field, FRONT);
    double* dst = vw.ptr(T.dst_blk, T.field, FRONT);
    for_box_elems<View>(T, [&](long long, long long ii, long long jj, long long kk) {
      const long long od = off(D, T.dlo[0] + ii, T.dlo[1] + jj, T.dlo[2] + kk);
      const long long os = off(S, T.lo[0] + ii, T.lo[1] + jj, T.lo[2] + kk);
      if (f32)
        reinterpret_cast<float*>(dst)[od] = reinterpret_cast<const float*>(src)[os];
      else
        dst[od] = src[os];
    });
    return;
  }
  const long long stride = (long long)gridDim.x * blockDim.x;
  const sf_dev_block& B = vw.blk(T.dst_blk);
  double* f = vw.ptr(T.dst_blk, T.field, FRONT);
  if (f32)
    bc_task<float>(T, B, reinterpret_cast<float*>(f), stride);
  else
    bc_task<double>(T, B, f, stride);
}

template <class View>
__global__ void k_tasks(View vw, const sf_task* __restrict__ tasks, const sf_dev_ctl* pred) {
  if (pred && pred_done(pred)) return;
  run_task(vw, tasks[blockIdx.y]);
}
// a single task passed by value (level-2 sf_launch_bc_face: no device allocation per call)
template <class View>
__global__ void k_task_one(View vw, sf_task task) {
  run_task(vw, task);
}

// CTAs per task: one thread per element or tangential line, at most 1184 (8 per SM)
static unsigned task_ctas(const sf_task& t) {
  return (unsigned)std::max(1ll, std::min((t.count + 255) / 256, 1184ll));
}

template <class View>
void launch_tasks(const View& vw, const sf_task* tasks, int ntasks, long long max_count,
                  const sf_dev_ctl* pred, cudaStream_t st, int max_ctas) {
  if (ntasks <= 0) return;
  long long bx = (max_count + 255) / 256;
  if (bx > max_ctas) bx = max_ctas;
  if (bx < 1) bx = 1;
  dim3 grid((unsigned)bx, (unsigned)ntasks);
  k_tasks<View><<<grid, 256, 0, st>>>(vw, tasks, pred);
}
void launch_task_one(const direct_view& vw, const sf_task& t, cudaStream_t st) {
  k_task_one<direct_view><<<task_ctas(t), 256, 0, st>>>(vw, t);
}
template void launch_tasks<table_view>(const table_view&, const sf_task*, int, long long,
                                       const sf_dev_ctl*, cudaStream_t, int);
template void launch_tasks<direct_view>(const direct_view&, const sf_task*, int, long long,
                                        const sf_dev_ctl*, cudaStream_t, int);

// ---------------------------------------------------------------------------
// UPDATE_VELOCITY (cfd.hpp:524-589): reads front, writes back (SEPARATEINOUT)
// ---------------------------------------------------------------------------
template <class View, bool BLEND>
__global__ void __launch_bounds__(kTX* kTY) k_update_vel(View vw, int zc, sf_consts s,
                                                         sf_dev_ctl* ctl, double dt_arg) {
  const tile_loc t = locate(vw.work(), vw.nitems, zc);
  const sf_dev_block& B = vw.blk(t.blk);
  const double* __restrict__ U = vw.ptr(t.blk, SF_VX, FRONT);
  const double* __restrict__ V = vw.ptr(t.blk, SF_VY, FRONT);
  const double* __restrict__ W = vw.ptr(t.blk, SF_VZ, FRONT);
  const double* __restrict__ Q = vw.ptr(t.blk, SF_P, FRONT);
  double* __restrict__ Uo = vw.ptr(t.blk, SF_VX, BACK);
  double* __restrict__ Vo = vw.ptr(t.blk, SF_VY, BACK);
  double* __restrict__ Wo = vw.ptr(t.blk, SF_VZ, BACK);
  const double dt = ctl ? ctl->dt : dt_arg;
  const long long sx = B.sx, sxy = B.sx * B.sy;
  unsigned long long mx[3] = {0ull, 0ull, 0ull};
  if (t.act) {
    for (long long k = t.k0; k < t.k1; ++k) {
      const long long o = off(B, t.i, t.j, k);
      struct ldg_acc {
        const double *U, *V, *W, *Q;
        long long o, sx, sxy;
        __device__ __forceinline__ double u(int a, int b, int c) const { return __ldg(U + o + a + b * sx + c * sxy); }
        __device__ __forceinline__ double v(int a, int b, int c) const { return __ldg(V + o + a + b * sx + c * sxy); }
        __device__ __forceinline__ double w(int a, int b, int c) const { return __ldg(W + o + a + b * sx + c * sxy); }
        __device__ __forceinline__ double q(int a, int b, int c) const { return __ldg(Q + o + a + b * sx + c * sxy); }
      };
      const ldg_acc A{U, V, W, Q, o, sx, sxy};
      double r[3];
      uv_point<ldg_acc, BLEND>(A, uv_consts<double>(s), dt, r);
      Uo[o] = r[0];
      Vo[o] = r[1];
      Wo[o] = r[2];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const unsigned long long bb = abs_bits(r[a]);
        mx[a] = bb > mx[a] ? bb : mx[a];
      }
    }
  }
  if (ctl) block_max_atomic<3>(mx, &ctl->acc[1]);
}

template <class View>
void launch_update_velocity(const View& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                            double dt, cudaStream_t st) {
  if (nctas <= 0) return;
  // alpha == 0 (either sign): the blend terms are only evaluated on zero fluxes (sf_uv.cuh)
  if (c.alpha == 0.0)
    k_update_vel<View, false><<<nctas, dim3(kTX, kTY), 0, st>>>(vw, zc, c, ctl, dt);
  else
    k_update_vel<View, true><<<nctas, dim3(kTX, kTY), 0, st>>>(vw, zc, c, ctl, dt);
}
template void launch_update_velocity<table_view>(const table_view&, int, int, const sf_consts&,
                                                 sf_dev_ctl*, double, cudaStream_t);
template void launch_update_velocity<direct_view>(const direct_view&, int, int, const sf_consts&,
                                                  sf_dev_ctl*, double, cudaStream_t);

// ---------------------------------------------------------------------------
// DIVERGENCE (cfd.hpp:595-618) with max|divu| into acc[acc_slot]
// ---------------------------------------------------------------------------
// T = float: the fp32 variant of the CFD fields
template <class View, class T>
__global__ void __launch_bounds__(kTX* kTY) k_divergence(View vw, int zc, sf_consts s,
                                                         sf_dev_ctl* ctl, int acc_slot,
                                                         int predicated) {
  if (predicated && pred_done(ctl)) return;
  const tile_loc t = locate(vw.work(), vw.nitems, zc);
  const sf_dev_block& B = vw.blk(t.blk);
  const T* __restrict__ U = reinterpret_cast<const T*>(vw.ptr(t.blk, SF_VX, FRONT));
  const T* __restrict__ V = reinterpret_cast<const T*>(vw.ptr(t.blk, SF_VY, FRONT));
  const T* __restrict__ W = reinterpret_cast<const T*>(vw.ptr(t.blk, SF_VZ, FRONT));
  T* __restrict__ D = reinterpret_cast<T*>(vw.ptr(t.blk, SF_DIVU, FRONT));
  const T ix = (T)s.ix, iy = (T)s.iy, iz = (T)s.iz;
  const long long sx = B.sx, sxy = B.sx * B.sy;
  unsigned long long mx[1] = {0ull};
  if (t.act) {
    for (long long k = t.k0; k < t.k1; ++k) {
      const long long o = off(B, t.i, t.j, k);
      T d = (__ldg(U + o) - __ldg(U + o - 1)) * ix;
      d += (__ldg(V + o) - __ldg(V + o - sx)) * iy;
      d += (__ldg(W + o) - __ldg(W + o - sxy)) * iz;
      D[o] = d;
      const unsigned long long bb = abs_bits((double)d);
      mx[0] = bb > mx[0] ? bb : mx[0];
    }
  }
  if (acc_slot >= 0) block_max_atomic<1>(mx, &ctl->acc[acc_slot]);
}

template <class View>
void launch_divergence(const View& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                       int acc_slot, int predicated, cudaStream_t st, int es) {
  if (nctas <= 0) return;
  if (es == 4)
    k_divergence<View, float><<<nctas, dim3(kTX, kTY), 0, st>>>(vw, zc, c, ctl, acc_slot, predicated);
  else
    k_divergence<View, double><<<nctas, dim3(kTX, kTY), 0, st>>>(vw, zc, c, ctl, acc_slot, predicated);
}
template void launch_divergence<table_view>(const table_view&, int, int, const sf_consts&,
                                            sf_dev_ctl*, int, int, cudaStream_t, int);
template void launch_divergence<direct_view>(const direct_view&, int, int, const sf_consts&,
                                             sf_dev_ctl*, int, int, cudaStream_t, int);

// ---------------------------------------------------------------------------
// PRESSURE_SWEEP (cfd.hpp:699-720), in place on p, vx, vy, vz
// ---------------------------------------------------------------------------
template <class View>
__global__ void __launch_bounds__(kTX* kTY) k_sweep(View vw,
                                                    int zc, sf_consts s, sf_dev_ctl* ctl,
                                                    int predicated, int explicit_bc,
                                                    double beta_arg, int color_arg,
                                                    double dt_arg) {
  if (predicated && pred_done(ctl)) return;
  const tile_loc t = locate(vw.work(), vw.nitems, zc);
  if (!t.act) return;
  const sf_dev_block& B = vw.blk(t.blk);
  const double* __restrict__ Dv = vw.ptr(t.blk, SF_DIVU, FRONT);
  double* __restrict__ P = vw.ptr(t.blk, SF_P, FRONT);
  double* __restrict__ U = vw.ptr(t.blk, SF_VX, FRONT);
  double* __restrict__ V = vw.ptr(t.blk, SF_VY, FRONT);
  double* __restrict__ W = vw.ptr(t.blk, SF_VZ, FRONT);
  const double beta = explicit_bc ? beta_arg : ctl->beta;
  const int color = explicit_bc ? color_arg : ctl->color;
  const double dt = ctl ? ctl->dt : dt_arg;
  const long long sx = B.sx, sxy = B.sx * B.sy;
  const long long gi = B.lo[0] + t.i, gj = B.lo[1] + t.j;
  const int bx = s.per[0] | ((gi > 0) & (gi < s.nm1[0]));
  const int by = s.per[1] | ((gj > 0) & (gj < s.nm1[1]));
  const int bxp = s.per[0] | (gi + 1 < s.nm1[0]);
  const int byp = s.per[1] | (gj + 1 < s.nm1[1]);
  for (long long k = t.k0; k < t.k1; ++k) {
    const long long gk = B.lo[2] + k;
    const long long o = off(B, t.i, t.j, k);
    const int bz = s.per[2] | ((gk > 0) & (gk < s.nm1[2]));
    const int bzp = s.per[2] | (gk + 1 < s.nm1[2]);
    const double a0 = ((gi + gj + gk) & 1) == color ? 1.0 : 0.0;
    const double a1 = ((gi + gj + gk + 1) & 1) == color ? 1.0 : 0.0;
    const double d0 = -(beta * s.bscale[bx][by][bz]) * Dv[o] * a0;
    const double ex = -(beta * s.bscale[bxp][by][bz]) * Dv[o + 1] * a1;
    const double ey = -(beta * s.bscale[bx][byp][bz]) * Dv[o + sx] * a1;
    const double ez = -(beta * s.bscale[bx][by][bzp]) * Dv[o + sxy] * a1;
    P[o] = P[o] + d0;
    U[o] = U[o] + dt * s.ix * (d0 - ex);
    V[o] = V[o] + dt * s.iy * (d0 - ey);
    W[o] = W[o] + dt * s.iz * (d0 - ez);
  }
}

template <class View>
void launch_pressure_sweep(const View& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                           int predicated, const double* beta_color_dt, cudaStream_t st) {
  if (nctas <= 0) return;
  const int ex = beta_color_dt != nullptr;
  k_sweep<View><<<nctas, dim3(kTX, kTY), 0, st>>>(
      vw, zc, c, ctl, predicated, ex, ex ? beta_color_dt[0] : 0.0,
      ex ? (int)beta_color_dt[1] : 0, ex ? beta_color_dt[2] : 0.0);
}
template void launch_pressure_sweep<table_view>(const table_view&, int, int, const sf_consts&,
                                                sf_dev_ctl*, int, const double*, cudaStream_t);
template void launch_pressure_sweep<direct_view>(const direct_view&, int, int, const sf_consts&,
                                                 sf_dev_ctl*, int, const double*, cudaStream_t);

// ---------------------------------------------------------------------------
// Fused half-sweep (the inner loop of pressure_iteration, cfd.hpp:295-303):
//   refresh(divu) [done by the previous half-sweep] ; PRESSURE_SWEEP ;
//   color ^= 1 ; ++sweeps ; refresh(vx,vy,vz) ; DIVERGENCE ; r = max|divu| ;
//   loop test.
// One pass reads divu, p, vx, vy, vz and writes p, vx', vy', vz', divu' (80 B
// per cell).  The velocity refresh is replaced by computing, per cell, the
// swept values of its -x/-y/-z neighbours (for a ghost neighbour: the value
// the refresh would deliver -- the neighbour block's swept cell, the pinned
// wall value, or the outflow copy), so the new divergence needs no grid-wide
// barrier.  Wall-normal planes are stored pinned, as the refresh leaves them
// (exchange.hpp:288-316).  Velocities and divu ping-pong FRONT <-> ALT; the
// last CTA swaps the table, flips the colour, counts the sweep and evaluates
// `residual > tolerance && sweeps < max_sweeps`.
// ---------------------------------------------------------------------------
struct sweep_ctx {
  double mb[2][2][2];  // -(beta * bscale[..]) exactly as cfd.hpp:712-715 forms it
  int color;
  long long nm1[3];
  int per[3];
  // selects instead of a dynamically indexed array (which lives in local memory)
  __device__ __forceinline__ double m(int a, int b, int c) const {
    const double x0 = c ? mb[0][0][1] : mb[0][0][0], x1 = c ? mb[0][1][1] : mb[0][1][0];
    const double x2 = c ? mb[1][0][1] : mb[1][0][0], x3 = c ? mb[1][1][1] : mb[1][1][0];
    return a ? (b ? x3 : x2) : (b ? x1 : x0);
  }
};

__device__ __forceinline__ int bit_in(const sweep_ctx& x, int a, long long g) {
  return x.per[a] | ((g > 0) & (g < x.nm1[a]));
}
__device__ __forceinline__ int bit_next(const sweep_ctx& x, int a, long long g) {
  return x.per[a] | (g + 1 < x.nm1[a]);
}
__device__ __forceinline__ double act0(const sweep_ctx& x, long long gsum) {
  return ((gsum & 1) == x.color) ? 1.0 : 0.0;
}

// One tile of the fused half-sweep; returns the tile's max |divu'| bits for
// this thread. CG = the persistent loop (k_pressure_loop): the tile reads
// state other SMs wrote since the kernel started, so data loads bypass L1
// (ld.global.cg).
template <bool CG>
__device__ __forceinline__ double ldd(const double* p) {
  if constexpr (CG) return __ldcg(p); else return *p;
}

// the buffers of one half-sweep: read divu, vx, vy, vz; write their next
// versions; p in place
struct sd_bufs {
  double *D, *U, *V, *W;  // read
  double *Dn, *Un, *Vn, *Wn, *P;
  __device__ __forceinline__ void flip() {  // the next half-sweep reads what this one wrote
    double* t;
    t = D; D = Dn; Dn = t;
    t = U; U = Un; Un = t;
    t = V; V = Vn; Vn = t;
    t = W; W = Wn; Wn = t;
  }
};
__device__ __forceinline__ sd_bufs table_bufs(const sf_dev_table* __restrict__ tab, int b, int cur) {
  const int nxt = cur == FRONT ? ALT : FRONT;
  return {tab->ptr[b][SF_DIVU][cur], tab->ptr[b][SF_VX][cur], tab->ptr[b][SF_VY][cur], tab->ptr[b][SF_VZ][cur],
          tab->ptr[b][SF_DIVU][nxt], tab->ptr[b][SF_VX][nxt], tab->ptr[b][SF_VY][nxt], tab->ptr[b][SF_VZ][nxt],
          tab->ptr[b][SF_P][FRONT]};
}

template <bool CG>
__device__ __forceinline__ unsigned long long sweep_div_tile(const sf_dev_block& B, const sd_bufs& bf,
                                                             const tile_loc& t, const sf_consts& s, double beta,
                                                             double dt, int color) {
  const double* __restrict__ D = bf.D;
  double* __restrict__ Dn = bf.Dn;
  double* __restrict__ P = bf.P;
  const double* __restrict__ U = bf.U;
  const double* __restrict__ V = bf.V;
  const double* __restrict__ W = bf.W;
  double* __restrict__ Un = bf.Un;
  double* __restrict__ Vn = bf.Vn;
  double* __restrict__ Wn = bf.Wn;
  sweep_ctx x;
  x.color = color;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) x.mb[a][b][c] = -(beta * s.bscale[a][b][c]);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    x.nm1[a] = s.nm1[a];
    x.per[a] = s.per[a];
  }
  // (dt * ix) exactly as s.dt * s.ix in cfd.hpp:717-719
  const double cu = dt * s.ix, cv = dt * s.iy, cw = dt * s.iz;
  unsigned long long rmax[1] = {0ull};

  if (t.act) {
    const long long n0 = B.n[0], n1 = B.n[1], n2 = B.n[2];
    const long long sx = B.sx, sxy = B.sx * B.sy;
    const long long i = t.i, j = t.j;
    const long long gi = B.lo[0] + i, gj = B.lo[1] + j;
    const int bx = bit_in(x, 0, gi), bxp = bit_next(x, 0, gi);
    const int by = bit_in(x, 1, gj), byp = bit_next(x, 1, gj);
    // the -x neighbour column (owned, or the cell behind the ghost)
    const long long gim = i > 0 ? gi - 1 : B.nb_ghost_gidx[0];
    const int bxm = bit_in(x, 0, gim), bxpm = bit_next(x, 0, gim);
    const long long gjm = j > 0 ? gj - 1 : B.nb_ghost_gidx[2];
    const int bym = bit_in(x, 1, gjm), bypm = bit_next(x, 1, gjm);
    const int fxl = B.face[0], fxh = B.face[1], fyl = B.face[2], fyh = B.face[3];
    const int fzl = B.face[4], fzh = B.face[5];
    // pinned high wall planes (exchange.hpp:296-315)
    const bool pin_u = (fxh == FACE_WALL || fxh == FACE_SYM) && i == n0 - 1;
    const bool pin_v = (fyh == FACE_WALL || fyh == FACE_SYM) && j == n1 - 1;
    const double pv_u = fxh == FACE_WALL ? B.fvel[1][0] : 0.0;
    const double pv_v = fyh == FACE_WALL ? B.fvel[3][1] : 0.0;
    const double pv_w = fzh == FACE_WALL ? B.fvel[5][2] : 0.0;
    const bool pinz_face = (fzh == FACE_WALL || fzh == FACE_SYM);

    long long o = off(B, i, j, t.k0);
    double wm_new;  // swept w of the -z neighbour
    double dC = ldd<CG>(D + o);
    {
      const long long k = t.k0;
      const long long gk = B.lo[2] + k;
      const int bz = bit_in(x, 2, gk);
      (void)bz;
      if (k > 0) {
        const long long gkm = gk - 1;
        const int bzm = bit_in(x, 2, gkm), bzpm = bit_next(x, 2, gkm);
        const double a0m = act0(x, gi + gj + gkm), a1m = 1.0 - a0m;
        const double d0m = x.m(bx, by, bzm) * ldd<CG>(D + o - sxy) * a0m;
        const double ezm = x.m(bx, by, bzpm) * dC * a1m;
        wm_new = ldd<CG>(W + o - sxy) + cw * (d0m - ezm);
      } else if (fzl == FACE_PROC || fzl == FACE_SELF) {
        const long long gkm = B.nb_ghost_gidx[4];
        const int bzm = bit_in(x, 2, gkm), bzpm = bit_next(x, 2, gkm);
        const double a0m = act0(x, gi + gj + gkm), a1m = 1.0 - a0m;
        const double d0m = x.m(bx, by, bzm) * ldd<CG>(D + o - sxy) * a0m;
        const double ezm = x.m(bx, by, bzpm) * dC * a1m;
        wm_new = ldd<CG>(W + o - sxy) + cw * (d0m - ezm);
      } else {
        wm_new = ldd<CG>(W + o - sxy);  // wall / symmetry pin; outflow fixed up below
      }
    }
    for (long long k = t.k0; k < t.k1; ++k, o += sxy) {
      const long long gk = B.lo[2] + k;
      const int bz = bit_in(x, 2, gk), bzp = bit_next(x, 2, gk);
      const double dXp = ldd<CG>(D + o + 1), dYp = ldd<CG>(D + o + sx), dZp = ldd<CG>(D + o + sxy);
      const double dXm = ldd<CG>(D + o - 1), dYm = ldd<CG>(D + o - sx);
      const double p0 = ldd<CG>(P + o), u0 = ldd<CG>(U + o), v0 = ldd<CG>(V + o), w0 = ldd<CG>(W + o);
      const double a0 = act0(x, gi + gj + gk), a1 = 1.0 - a0;
      // this cell's sweep (cfd.hpp:712-719)
      const double d0 = x.m(bx, by, bz) * dC * a0;
      const double ex = x.m(bxp, by, bz) * dXp * a1;
      const double ey = x.m(bx, byp, bz) * dYp * a1;
      const double ez = x.m(bx, by, bzp) * dZp * a1;
      P[o] = p0 + d0;
      double un = u0 + cu * (d0 - ex);
      double vn = v0 + cv * (d0 - ey);
      double wn = w0 + cw * (d0 - ez);
      if (pin_u) un = pv_u;
      if (pin_v) vn = pv_v;
      if (pinz_face && k == n2 - 1) wn = pv_w;
      // swept -x neighbour of u
      double umn;
      if (i > 0 || fxl == FACE_PROC || fxl == FACE_SELF) {
        const double a0m = i > 0 ? a1 : act0(x, gim + gj + gk);
        const double a1m = 1.0 - a0m;
        const double d0m = x.m(bxm, by, bz) * dXm * a0m;
        const double exm = x.m(bxpm, by, bz) * dC * a1m;
        umn = ldd<CG>(U + o - 1) + cu * (d0m - exm);
      } else if (fxl == FACE_OUT) {
        umn = un;
      } else {
        umn = ldd<CG>(U + o - 1);
      }
      // swept -y neighbour of v
      double vmn;
      if (j > 0 || fyl == FACE_PROC || fyl == FACE_SELF) {
        const double a0m = j > 0 ? a1 : act0(x, gi + gjm + gk);
        const double a1m = 1.0 - a0m;
        const double d0m = x.m(bx, bym, bz) * dYm * a0m;
        const double eym = x.m(bx, bypm, bz) * dC * a1m;
        vmn = ldd<CG>(V + o - sx) + cv * (d0m - eym);
      } else if (fyl == FACE_OUT) {
        vmn = vn;
      } else {
        vmn = ldd<CG>(V + o - sx);
      }
      if (k == 0 && fzl == FACE_OUT) wm_new = wn;
      // DIVERGENCE on the refreshed velocities (cfd.hpp:605-608)
      double dd = (un - umn) * s.ix;
      dd += (vn - vmn) * s.iy;
      dd += (wn - wm_new) * s.iz;
      Un[o] = un;
      Vn[o] = vn;
      Wn[o] = wn;
      Dn[o] = dd;
      // ghost values the next half-sweep reads (depth 1)
      if (i == 0) Un[o - 1] = umn;
      if (j == 0) Vn[o - sx] = vmn;
      if (k == 0) Wn[o - sxy] = wm_new;
      if (i == 0) {
        if (fxl == FACE_WALL || fxl == FACE_SYM || fxl == FACE_OUT) Dn[o - 1] = dd;
        if (fxh == FACE_SELF) Dn[o + n0] = dd;
      }
      if (i == n0 - 1) {
        if (fxh == FACE_WALL || fxh == FACE_SYM || fxh == FACE_OUT) Dn[o + 1] = dd;
        if (fxl == FACE_SELF) Dn[o - n0] = dd;
      }
      if (j == 0) {
        if (fyl == FACE_WALL || fyl == FACE_SYM || fyl == FACE_OUT) Dn[o - sx] = dd;
        if (fyh == FACE_SELF) Dn[o + n1 * sx] = dd;
      }
      if (j == n1 - 1) {
        if (fyh == FACE_WALL || fyh == FACE_SYM || fyh == FACE_OUT) Dn[o + sx] = dd;
        if (fyl == FACE_SELF) Dn[o - n1 * sx] = dd;
      }
      if (k == 0) {
        if (fzl == FACE_WALL || fzl == FACE_SYM || fzl == FACE_OUT) Dn[o - sxy] = dd;
        if (fzh == FACE_SELF) Dn[o + n2 * sxy] = dd;
      }
      if (k == n2 - 1) {
        if (fzh == FACE_WALL || fzh == FACE_SYM || fzh == FACE_OUT) Dn[o + sxy] = dd;
        if (fzl == FACE_SELF) Dn[o - n2 * sxy] = dd;
      }
      const unsigned long long bb = abs_bits(dd);
      rmax[0] = bb > rmax[0] ? bb : rmax[0];
      // march: this plane's swept w is the next plane's -z neighbour
      wm_new = wn;
      dC = dZp;
    }
  }
  return rmax[0];
}

// The last CTA's bookkeeping after a half-sweep (cfd.hpp:295-303): residual,
// colour flip, sweep count, loop test, FRONT <-> ALT swap of the velocities
// and divu of every block, and (hflag) the host-visible copy.
__device__ __forceinline__ void finish_half_sweep(sf_dev_table* __restrict__ tab, sf_dev_ctl* ctl,
                                                  sf_host_flag* hflag) {
  __threadfence();
  const unsigned long long rb = *reinterpret_cast<volatile unsigned long long*>(&ctl->acc[0]);
  const double residual = bits_to_max(rb);
  ctl->acc[0] = 0ull;
  ctl->ctas_done = 0u;
  ctl->residual = residual;
  ctl->color ^= 1;
  const int sweeps = ctl->sweeps + 1;
  ctl->sweeps = sweeps;
  const int more = (residual > ctl->tolerance) && (sweeps < ctl->max_sweeps);
  ctl->done = more ? 0 : 1;
  for (int b = 0; b < tab->nblocks; ++b) {
    for (int f = 0; f < 5; ++f) {
      if (f == SF_P) continue;
      double* tmp = tab->ptr[b][f][FRONT];
      tab->ptr[b][f][FRONT] = tab->ptr[b][f][ALT];
      tab->ptr[b][f][ALT] = tmp;
      const unsigned char ti = tab->bidx[b][f][FRONT];
      tab->bidx[b][f][FRONT] = tab->bidx[b][f][ALT];
      tab->bidx[b][f][ALT] = ti;
    }
  }
  if (hflag) {
    hflag->sweeps = sweeps;
    hflag->residual = residual;
    hflag->done = more ? 0 : 1;
    hflag->color = ctl->color;
    __threadfence_system();
  }
}

__global__ void __launch_bounds__(kTX* kTY) k_sweep_div(sf_dev_table* __restrict__ tab,
                                                        const sf_work* __restrict__ items,
                                                        int nitems, int zc, sf_consts s,
                                                        sf_dev_ctl* ctl, sf_host_flag* hflag,
                                                        unsigned int total_ctas, int finalize) {
  if (pred_done(ctl)) return;
  const tile_loc t = locate(items, nitems, zc);
  unsigned long long rmax[1] = {
      sweep_div_tile<false>(tab->blk[t.blk], table_bufs(tab, t.blk, FRONT), t, s, ctl->beta, ctl->dt, ctl->color)};
  block_max_atomic<1>(rmax, &ctl->acc[0]);
  if (!finalize) return;  // across ranks: allreduce, then CTL_FINISH_FUSED
  if (last_cta(&ctl->ctas_done, total_ctas))
    if (threadIdx.x == 0 && threadIdx.y == 0) finish_half_sweep(tab, ctl, hflag);
}

void launch_sweep_div(const table_view& vw, int nctas, int zc, const sf_consts& c,
                      sf_dev_ctl* ctl, sf_host_flag* hflag, int fin, cudaStream_t st) {
  if (nctas <= 0) return;
  k_sweep_div<<<nctas, dim3(kTX, kTY), 0, st>>>(vw.tab, vw.items, vw.nitems, zc, c, ctl, hflag,
                                                 (unsigned)nctas, fin);
}

// Persistent pressure loop (cooperative launch) for grids smaller than about
// one wave of CTAs, where a launch per half-sweep costs more than the sweep.
// Every CTA strides over the tiles; one grid barrier per half-sweep replaces
// the kernel boundary. After it every CTA reads the half-sweep's residual and
// takes the loop decision itself (the same test as finish_half_sweep), so no
// second barrier is needed: the residual maxima rotate over three slots
// (half-sweep m accumulates into racc[m % 3]; CTA 0 clears racc[(m + 1) % 3],
// whose readers all passed barrier m - 1), and the FRONT/ALT parity is kept
// in registers. CTA 0 writes the loop state and the table swap once at the
// end. The cells are the same sweep_div_tile as k_sweep_div: bitwise equal.
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kTX* kTY, 2) k_pressure_loop(sf_dev_table* __restrict__ tab,
                                                            const sf_work* __restrict__ items, int nitems,
                                                            int zc, sf_consts s, sf_dev_ctl* ctl, int ntiles) {
  __shared__ unsigned long long s_res;
  if (pred_done(ctl)) return;
  const int tid = threadIdx.y * kTX + threadIdx.x;
  const int b = items[0].blk;  // one grid component
  const sf_dev_block& B = tab->blk[b];
  sd_bufs bf = table_bufs(tab, b, FRONT);
  const double beta = ctl->beta, dt = ctl->dt, tol = ctl->tolerance;
  const int sweeps0 = ctl->sweeps, max_sweeps = ctl->max_sweeps, color0 = ctl->color;
  const unsigned int nctas = gridDim.x;
  int m = 0;
  double residual = 0.0;
  bool more = true;
  while (more) {
    if (blockIdx.x == 0 && tid == 0) ctl->racc[(m + 1) % 3] = 0ull;
    unsigned long long rmax[1] = {0ull};
    for (int c = blockIdx.x; c < ntiles; c += gridDim.x) {
      const unsigned long long r = sweep_div_tile<true>(B, bf, locate_at(items, nitems, zc, c), s, beta, dt,
                                                        color0 ^ (m & 1));
      rmax[0] = r > rmax[0] ? r : rmax[0];
    }
    block_max_atomic<1>(rmax, &ctl->racc[m % 3]);  // ends with thread 0's atomic
    __syncthreads();
    if (tid == 0) {  // arrive (release: this CTA's stores and atomics), wait (acquire)
      const unsigned int target = nctas * (unsigned)(m + 1);
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&ctl->bar) : "memory");
      while (ld_acquire(&ctl->bar) < target) {
      }
      s_res = ld_acquire64(&ctl->racc[m % 3]);
    }
    __syncthreads();
    residual = bits_to_max(s_res);
    const int sweeps = sweeps0 + m + 1;
    more = (residual > tol) && (sweeps < max_sweeps);
    bf.flip();
    ++m;
  }
  if (blockIdx.x == 0 && tid == 0) {
    ctl->residual = residual;
    ctl->sweeps = sweeps0 + m;
    ctl->color = color0 ^ (m & 1);
    ctl->done = 1;
    if (m & 1) {
      for (int f = 0; f < 5; ++f) {
        if (f == SF_P) continue;
        double* tmp = tab->ptr[b][f][FRONT];
        tab->ptr[b][f][FRONT] = tab->ptr[b][f][ALT];
        tab->ptr[b][f][ALT] = tmp;
        const unsigned char ti = tab->bidx[b][f][FRONT];
        tab->bidx[b][f][FRONT] = tab->bidx[b][f][ALT];
        tab->bidx[b][f][ALT] = ti;
      }
    }
  }
}

int pressure_loop_ctas() {
  static std::mutex mu;
  static std::map<int, int> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it != per_dev.end()) return it->second;
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pressure_loop, kTX * kTY, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_dev[dev] = per_sm * sms;
}

cudaError_t launch_pressure_loop(const table_view& vw, int ntiles, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                                 cudaStream_t st) {
  if (ntiles <= 0) return cudaSuccess;
  const int grid = std::min(ntiles, pressure_loop_ctas());
  sf_dev_table* tab = vw.tab;
  const sf_work* items = vw.items;
  int nitems = vw.nitems;
  sf_consts cc = c;
  void* args[] = {&tab, &items, &nitems, &zc, &cc, &ctl, &ntiles};
  return cudaLaunchCooperativeKernel((const void*)k_pressure_loop, dim3(grid), dim3(kTX, kTY), args, 0, st);
}

// taylor_green_error per cell (cfd.hpp:388-393): eu = u - (sin*cos)*decay,
// ev = v + (cos*sin)*decay, ew = w; the host sums the terms in the
// reference's order (x-fastest per worker, workers in order).
__global__ void k_tg_cells(const double* __restrict__ U, const double* __restrict__ V,
                           const double* __restrict__ W, long long base, long long sx, long long sy, int nx,
                           int ny, int nz, const double* __restrict__ su, const double* __restrict__ sv,
                           double decay, double* __restrict__ out) {
  const long long n = (long long)nx * ny * nz;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx), j = (int)((e / nx) % ny), k = (int)(e / ((long long)nx * ny));
    const long long o = base + ((long long)k * sy + j) * sx + i;
    const double eu = U[o] - su[(long long)j * nx + i] * decay;
    const double ev = V[o] + sv[(long long)j * nx + i] * decay;
    const double ew = W[o];
    out[e] = eu * eu + ev * ev + ew * ew;
  }
}

void launch_tg_cells(const double* U, const double* V, const double* W, long long base, long long sx, long long sy,
                     const long long dims[3], const double* su, const double* sv, double decay, double* out,
                     cudaStream_t st) {
  const long long n = dims[0] * dims[1] * dims[2];
  if (n <= 0) return;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  k_tg_cells<<<blocks, 256, 0, st>>>(U, V, W, base, sx, sy, (int)dims[0], (int)dims[1], (int)dims[2], su, sv, decay,
                                     out);
}

// ---------------------------------------------------------------------------
// reductions (reductions.hpp:28-90)
// ---------------------------------------------------------------------------
template <class View>
__global__ void __launch_bounds__(kTX* kTY) k_reduce_max(View vw, int zc, int f0, int f1,
                                                         int f2, int nfields, int diff,
                                                         unsigned long long* acc) {
  const tile_loc t = locate(vw.work(), vw.nitems, zc);
  const sf_dev_block& B = vw.blk(t.blk);
  unsigned long long mx[3] = {0ull, 0ull, 0ull};
  const int fl[3] = {f0, f1, f2};
  if (t.act && nfields == 3 && !diff && vw.esize(f0) == 8 && vw.esize(f1) == 8 && vw.esize(f2) == 8) {
    // compute_dt's three maxima (cfd.hpp:264-273): the three fields in one
    // z loop, four planes per iteration -- 12 independent loads in flight
    const double* __restrict__ F0 = vw.ptr(t.blk, f0, FRONT);
    const double* __restrict__ F1 = vw.ptr(t.blk, f1, FRONT);
    const double* __restrict__ F2 = vw.ptr(t.blk, f2, FRONT);
    const long long sxy = B.sx * B.sy;
    long long o = off(B, t.i, t.j, t.k0);
#pragma unroll 4
    for (long long k = t.k0; k < t.k1; ++k, o += sxy) {
      const unsigned long long b0 = abs_bits(fabs(__ldg(F0 + o)));
      const unsigned long long b1 = abs_bits(fabs(__ldg(F1 + o)));
      const unsigned long long b2 = abs_bits(fabs(__ldg(F2 + o)));
      mx[0] = b0 > mx[0] ? b0 : mx[0];
      mx[1] = b1 > mx[1] ? b1 : mx[1];
      mx[2] = b2 > mx[2] ? b2 : mx[2];
    }
  } else if (t.act) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q >= nfields) break;
      const double* __restrict__ F = vw.ptr(t.blk, fl[q], FRONT);
      const double* __restrict__ Bk = vw.ptr(t.blk, fl[q], BACK);
      const bool f32 = vw.esize(fl[q]) == 4;  // fp32 values widen exactly
      for (long long k = t.k0; k < t.k1; ++k) {
        const long long o = off(B, t.i, t.j, k);
        const double x = f32 ? (double)__ldg(reinterpret_cast<const float*>(F) + o) : __ldg(F + o);
        const double a = diff ? fabs(x - (f32 ? (double)__ldg(reinterpret_cast<const float*>(Bk) + o) : __ldg(Bk + o)))
                              : fabs(x);
        const unsigned long long bb = abs_bits(a);
        mx[q] = bb > mx[q] ? bb : mx[q];
      }
    }
  }
  if (nfields == 1) {
    unsigned long long m1[1] = {mx[0]};
    block_max_atomic<1>(m1, acc);
  } else {
    block_max_atomic<3>(mx, acc);
  }
}

template <class View>
void launch_reduce_max(const View& vw, int nctas, int zc, const int* fields, int nfields, int diff,
                       unsigned long long* acc, cudaStream_t st) {
  if (nctas <= 0) return;
  k_reduce_max<View><<<nctas, dim3(kTX, kTY), 0, st>>>(
      vw, zc, fields[0], nfields > 1 ? fields[1] : 0, nfields > 2 ? fields[2] : 0, nfields, diff,
      acc);
}
template void launch_reduce_max<table_view>(const table_view&, int, int, const int*, int, int,
                                            unsigned long long*, cudaStream_t);
template void launch_reduce_max<direct_view>(const direct_view&, int, int, const int*, int, int,
                                             unsigned long long*, cudaStream_t);

// Deterministic sums: one partial per CTA (x-fastest within the tile), the
// host folds partials in CTA order.  Not the reference's serial order, so
// sums agree to rounding, not bitwise (they are off the hot path:
// kinetic_energy / taylor_green_error, cfd.hpp:357-401).
template <class View>
__global__ void __launch_bounds__(kTX* kTY) k_reduce_sum(View vw, int zc, int field, int square,
                                                         double* partials) {
  const tile_loc t = locate(vw.work(), vw.nitems, zc);
  const sf_dev_block& B = vw.blk(t.blk);
  const double* __restrict__ F = vw.ptr(t.blk, field, FRONT);
  const bool f32 = vw.esize(field) == 4;
  double acc = 0.0;
  if (t.act)
    for (long long k = t.k0; k < t.k1; ++k) {
      const long long o = off(B, t.i, t.j, k);
      const double x = f32 ? (double)__ldg(reinterpret_cast<const float*>(F) + o) : __ldg(F + o);
      acc += square ? x * x : x;
    }
  __shared__ double red[kTX * kTY];
  const int tid = threadIdx.y * kTX + threadIdx.x;
  red[tid] = acc;
  __syncthreads();
  for (int w = kTX * kTY / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  if (tid == 0) partials[blockIdx.x] = red[0];
}

void launch_reduce_sum(const table_view& vw, int nctas, int zc, int field, int square,
                       double* partials, cudaStream_t st) {
  if (nctas <= 0) return;
  k_reduce_sum<table_view><<<nctas, dim3(kTX, kTY), 0, st>>>(vw, zc, field, square, partials);
}

// ---------------------------------------------------------------------------
// control
// ---------------------------------------------------------------------------
__device__ void set_beta(sf_dev_ctl* ctl, const sf_consts& s) {
  // beta = omega / (2 dt (ix2 + iy2 + iz2))   (cfd.hpp:291)
  ctl->beta = s.omega / (2.0 * ctl->dt * (s.ix2 + s.iy2 + s.iz2));
}

__global__ void k_ctl(sf_dev_table* tab, sf_dev_ctl* ctl, sf_host_flag* hflag, int op, double arg,
                      int f, int sa, int sb, sf_consts s, int predicated) {
  if (predicated && pred_done(ctl)) return;
  switch (op) {
    case CTL_DT_FROM_ACC: {  // compute_dt (cfd.hpp:264-273)
      double dt = 1.0 / (2.0 * s.nu * (s.ix2 + s.iy2 + s.iz2));
      const double m[3] = {bits_to_max(ctl->acc[0]), bits_to_max(ctl->acc[1]),
                           bits_to_max(ctl->acc[2])};
      for (int a = 0; a < 3; ++a) {
        ctl->vmax[a] = m[a];
        if (m[a] > 0.0) {
          const double c = s.spacing[a] / m[a];
          dt = c < dt ? c : dt;  // std::min(dt, c)
        }
        ctl->acc[a] = 0ull;
      }
      ctl->dt = s.sigma * dt;
      set_beta(ctl, s);
      if (hflag) {
        hflag->dt = ctl->dt;
        __threadfence_system();
      }
      break;
    }
    case CTL_SET_DT:
      ctl->dt = arg;
      set_beta(ctl, s);
      if (hflag) {
        hflag->dt = ctl->dt;
        __threadfence_system();
      }
      break;
    case CTL_RESET_CLOCK:
      ctl->color = 0;
      ctl->abort_field = -1;
      if (hflag) {
        hflag->color = 0;
        hflag->abort_field = -1;
        __threadfence_system();
      }
      break;
    case CTL_BEGIN_ITERATION:
      ctl->sweeps = 0;
      ctl->residual = 0.0;
      ctl->acc[0] = 0ull;
      ctl->acc[1] = 0ull;
      ctl->ctas_done = 0u;
      ctl->redo = 0;
      ctl->racc[0] = ctl->racc[1] = ctl->racc[2] = 0ull;
      ctl->bar = 0u;
      ctl->done = ctl->abort_field >= 0 ? 1 : 0;
      ctl->max_sweeps = s.max_sweeps;
      ctl->tolerance = s.tolerance;
      if (hflag) {
        hflag->done = ctl->done;
        hflag->sweeps = 0;
        hflag->residual = 0.0;
        __threadfence_system();
      }
      break;
    case CTL_AFTER_SWEEP:
      ctl->color ^= 1;
      ctl->sweeps += 1;
      if (hflag) {
        hflag->color = ctl->color;
        __threadfence_system();
      }
      break;
    case CTL_FINISH_SWEEP: {
      const double r = bits_to_max(ctl->acc[0]);
      ctl->acc[0] = 0ull;
      ctl->residual = r;
      const int more = (r > ctl->tolerance) && (ctl->sweeps < ctl->max_sweeps);
      ctl->done = more ? 0 : 1;
      if (hflag) {
        hflag->sweeps = ctl->sweeps;
        hflag->residual = r;
        hflag->done = ctl->done;
        __threadfence_system();
      }
      break;
    }
    case CTL_CHECK_FINITE: {
      ctl->abort_field = -1;
      for (int a = 0; a < 3; ++a) {
        const double m = bits_to_max(ctl->acc[1 + a]);
        ctl->acc[1 + a] = 0ull;
        ctl->vmax[a] = m;
        if (ctl->abort_field < 0 && !isfinite(m)) ctl->abort_field = a;
      }
      if (hflag) {
        hflag->abort_field = ctl->abort_field;
        __threadfence_system();
      }
      break;
    }
    case CTL_FINISH_FUSED: {  // the fused kernel's finalize, after the residual allreduce
      const double r = bits_to_max(ctl->acc[0]);
      ctl->acc[0] = 0ull;
      ctl->residual = r;
      ctl->color ^= 1;
      ctl->sweeps += 1;
      const int more = (r > ctl->tolerance) && (ctl->sweeps < ctl->max_sweeps);
      ctl->done = more ? 0 : 1;
      for (int b = 0; b < tab->nblocks; ++b)
        for (int q = 0; q < 5; ++q) {
          if (q == SF_P) continue;
          double* tmp = tab->ptr[b][q][FRONT];
          tab->ptr[b][q][FRONT] = tab->ptr[b][q][ALT];
          tab->ptr[b][q][ALT] = tmp;
          const unsigned char ti = tab->bidx[b][q][FRONT];
          tab->bidx[b][q][FRONT] = tab->bidx[b][q][ALT];
          tab->bidx[b][q][ALT] = ti;
        }
      if (hflag) {
        hflag->sweeps = ctl->sweeps;
        hflag->residual = r;
        hflag->done = ctl->done;
        hflag->color = ctl->color;
        __threadfence_system();
      }
      break;
    }
    case CTL_FINISH_PASS: {  // the temporal pass's in-kernel finalize (sf_sweep2.cu), across ranks
      const double r1 = bits_to_max(ctl->acc[0]), r2 = bits_to_max(ctl->acc[1]);
      ctl->acc[0] = 0ull;
      ctl->acc[1] = 0ull;
      const int sw = ctl->sweeps;
      if (!((r1 > ctl->tolerance) && (sw + 1 < ctl->max_sweeps))) {
        ctl->sweeps = sw + 1;
        ctl->residual = r1;
        ctl->color ^= 1;
        ctl->done = 1;
        ctl->redo = 1;
      } else {
        ctl->sweeps = sw + 2;
        ctl->residual = r2;
        ctl->done = ((r2 > ctl->tolerance) && (sw + 2 < ctl->max_sweeps)) ? 0 : 1;
        for (int b = 0; b < tab->nblocks; ++b)
          for (int q = 0; q < 5; ++q) {
            double* tmp = tab->ptr[b][q][FRONT];
            tab->ptr[b][q][FRONT] = tab->ptr[b][q][ALT];
            tab->ptr[b][q][ALT] = tmp;
            const unsigned char ti = tab->bidx[b][q][FRONT];
            tab->bidx[b][q][FRONT] = tab->bidx[b][q][ALT];
            tab->bidx[b][q][ALT] = ti;
          }
      }
      if (hflag) {
        hflag->sweeps = ctl->sweeps;
        hflag->residual = ctl->residual;
        hflag->done = ctl->done;
        hflag->color = ctl->color;
        __threadfence_system();
      }
      break;
    }
    case CTL_PUBLISH:
      if (hflag) {
        hflag->sweeps = ctl->sweeps;
        hflag->residual = ctl->residual;
        hflag->done = ctl->done;
        hflag->color = ctl->color;
        __threadfence_system();
      }
      break;
    case CTL_CLEAR_ACC:
      for (int a = 0; a < 8; ++a) ctl->acc[a] = 0ull;
      ctl->ctas_done = 0u;
      break;
    case CTL_SWAP:
      for (int b = 0; b < tab->nblocks; ++b) {
        double* tmp = tab->ptr[b][f][sa];
        tab->ptr[b][f][sa] = tab->ptr[b][f][sb];
        tab->ptr[b][f][sb] = tmp;
        const unsigned char ti = tab->bidx[b][f][sa];
        tab->bidx[b][f][sa] = tab->bidx[b][f][sb];
        tab->bidx[b][f][sb] = ti;
      }
      break;
  }
}

void ensure_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({kernel, dev}).second)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// Condition of the pressure loop's CUDA-graph while node: run another body
// iteration while the device predicate says the loop goes on.
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const sf_dev_ctl* ctl) {
  cudaGraphSetConditional(h, *reinterpret_cast<const volatile int*>(&ctl->done) ? 0u : 1u);
}
void launch_loop_cond(cudaGraphConditionalHandle h, const sf_dev_ctl* ctl, cudaStream_t st) {
  k_loop_cond<<<1, 1, 0, st>>>(h, ctl);
}

// Owned block of (b, f) FRONT -> dense x-fastest fp64 buffer, FRONT resolved
// on the device (a snapshot that needs no host synchronisation). One warp
// group per row, rows strided over the grid; fp32 fields widen.
__global__ void k_snapshot(const sf_dev_table* __restrict__ tab, int b, int f, double* __restrict__ buf) {
  const sf_dev_block& B = tab->blk[b];
  const double* src = tab->ptr[b][f][FRONT];
  const bool f32 = tab->esize[f] == 4;
  const long long n0 = B.n[0], n1 = B.n[1], rows = B.n[1] * B.n[2];
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long k = r / n1, j = r - k * n1;
    const long long o = off(B, 0, j, k);
    double* dst = buf + r * n0;
    for (long long i = threadIdx.x; i < n0; i += blockDim.x)
      dst[i] = f32 ? (double)reinterpret_cast<const float*>(src)[o + i] : src[o + i];
  }
}
void launch_snapshot(const sf_dev_table* tab, int b, int f, double* buf, long long rows, cudaStream_t st) {
  const long long nb = rows < 148 * 32 ? rows : 148 * 32;
  if (nb > 0) k_snapshot<<<(unsigned)nb, 256, 0, st>>>(tab, b, f, buf);
}
// the reverse: dense fp64 buffer -> owned block of (b, f) FRONT (fp32 fields round)
__global__ void k_install(const sf_dev_table* __restrict__ tab, int b, int f, const double* __restrict__ buf) {
  const sf_dev_block& B = tab->blk[b];
  double* dst = tab->ptr[b][f][FRONT];
  const bool f32 = tab->esize[f] == 4;
  const long long n0 = B.n[0], n1 = B.n[1], rows = B.n[1] * B.n[2];
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long k = r / n1, j = r - k * n1;
    const long long o = off(B, 0, j, k);
    const double* src = buf + r * n0;
    for (long long i = threadIdx.x; i < n0; i += blockDim.x) {
      if (f32)
        reinterpret_cast<float*>(dst)[o + i] = (float)src[i];
      else
        dst[o + i] = src[i];
    }
  }
}
void launch_install(const sf_dev_table* tab, int b, int f, const double* buf, long long rows, cudaStream_t st) {
  const long long nb = rows < 148 * 32 ? rows : 148 * 32;
  if (nb > 0) k_install<<<(unsigned)nb, 256, 0, st>>>(tab, b, f, buf);
}

void launch_ctl(sf_dev_table* tab, sf_dev_ctl* ctl, sf_host_flag* hflag, int op, double arg,
                int f, int a, int b, const sf_consts& c, int predicated, cudaStream_t st) {
  k_ctl<<<1, 1, 0, st>>>(tab, ctl, hflag, op, arg, f, a, b, c, predicated);
}

// ---------------------------------------------------------------------------
// raw box copies (level-2 ABI, gather / scatter)
// ---------------------------------------------------------------------------
// element types S -> D (fp32 <-> fp64 conversions are exact widenings, or
// round-to-nearest narrowings on the way into an fp32 field)
template <class TS, class TD>
__global__ void k_copy_box(const TS* __restrict__ src, long long s_base, long long s_sx,
                           long long s_sy, TD* __restrict__ dst, long long d_base,
                           long long d_sx, long long d_sy, long long l0, long long l1,
                           long long l2, long long n0, long long n1, long long n2, long long m0,
                           long long m1, long long m2) {
  const long long total = n0 * n1 * n2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const long long k = e / (n0 * n1), r = e - k * n0 * n1, j = r / n0, i = r - j * n0;
    dst[d_base + ((m2 + k) * d_sy + (m1 + j)) * d_sx + (m0 + i)] =
        (TD)src[s_base + ((l2 + k) * s_sy + (l1 + j)) * s_sx + (l0 + i)];
  }
}

void launch_copy_box_es(const void* src, int s_es, long long s_base, long long s_sx, long long s_sy, void* dst,
                        int d_es, long long d_base, long long d_sx, long long d_sy, const long long lo[3],
                        const long long dims[3], const long long dlo[3], cudaStream_t st) {
  const long long total = dims[0] * dims[1] * dims[2];
  if (total <= 0) return;
  long long nb = (total + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
#define SF_COPY(TS, TD)                                                                                  \
  k_copy_box<TS, TD><<<(unsigned)nb, 256, 0, st>>>(static_cast<const TS*>(src), s_base, s_sx, s_sy,    \
                                                    static_cast<TD*>(dst), d_base, d_sx, d_sy, lo[0], lo[1], \
                                                    lo[2], dims[0], dims[1], dims[2], dlo[0], dlo[1], dlo[2])
  if (s_es == 4 && d_es == 4)
    SF_COPY(float, float);
  else if (s_es == 4)
    SF_COPY(float, double);
  else if (d_es == 4)
    SF_COPY(double, float);
  else
    SF_COPY(double, double);
#undef SF_COPY
}

void launch_copy_box(const double* src, long long s_base, long long s_sx, long long s_sy,
                     double* dst, long long d_base, long long d_sx, long long d_sy,
                     const long long lo[3], const long long dims[3], const long long dlo[3],
                     cudaStream_t st) {
  launch_copy_box_es(src, 8, s_base, s_sx, s_sy, dst, 8, d_base, d_sx, d_sy, lo, dims, dlo, st);
}

template <class T>
__global__ void k_fill_box(T* __restrict__ dst, long long base, long long sx, long long sy,
                           long long l0, long long l1, long long l2, long long n0, long long n1,
                           long long n2, T v) {
  const long long total = n0 * n1 * n2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const long long k = e / (n0 * n1), r = e - k * n0 * n1, j = r / n0, i = r - j * n0;
    dst[base + ((l2 + k) * sy + (l1 + j)) * sx + (l0 + i)] = v;
  }
}

void launch_fill_box(void* dst, long long base, long long sx, long long sy, const long long lo[3],
                     const long long dims[3], double v, cudaStream_t st, int es) {
  const long long total = dims[0] * dims[1] * dims[2];
  if (total <= 0) return;
  long long nb = (total + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  if (es == 4)
    k_fill_box<float><<<(unsigned)nb, 256, 0, st>>>(static_cast<float*>(dst), base, sx, sy, lo[0], lo[1], lo[2],
                                                    dims[0], dims[1], dims[2], (float)v);
  else
    k_fill_box<double><<<(unsigned)nb, 256, 0, st>>>(static_cast<double*>(dst), base, sx, sy, lo[0], lo[1], lo[2],
                                                     dims[0], dims[1], dims[2], v);
}

// owned cells <-> a global x-fastest array (grid::gather / scatter, io.hpp:25-65)
void launch_gather_owned(const double* src, long long base, long long sx, long long sy,
                         const long long n[3], const long long lo[3], const long long N[3],
                         double* dst_global, int to_field, cudaStream_t st, int field_es) {
  const long long zero[3] = {0, 0, 0};
  if (!to_field)
    launch_copy_box_es(src, field_es, base, sx, sy, dst_global, 8, 0, N[0], N[1], zero, n, lo, st);
  else
    launch_copy_box_es(dst_global, 8, 0, N[0], N[1], const_cast<double*>(src), field_es, base, sx, sy, lo, n,
                       zero, st);
}

}  // namespace sfb
