// sf_uv.cuh -- the UPDATE_VELOCITY point update (cfd.hpp:524-589), written
// once against an accessor so the plain-load and the TMA-staged kernels
// evaluate the identical IEEE operations in the identical order.
//   A.u(a, b, c), A.v(..), A.w(..), A.q(..): vx, vy, vz, p at offset (a, b, c)
// out[0..2]: the provisional vx, vy, vz of the cell.
//
// BLEND = false is the specialisation for a zero upwind blend (alpha = +-0,
// the reference's default, cfd.hpp:40): each flux then equals
// f + alpha * X with alpha * X = +-0, which leaves f unchanged unless f is a
// zero (a signed zero can flip: -0 + +0 = +0).  So the blend term X is only
// evaluated, and added as in the reference, when f == 0 -- bitwise the
// reference's result with 126 instead of 189 DP add/sub/mul per cell (plus
// one compare per flux).  Inputs large enough to overflow a blend product
// (|v| > 1e154) make the state non-finite on both paths; the NaN guard then
// raises the same error.
#pragma once

#include "sf_device.cuh"

namespace sfb {

// T = float is the fp32 variant of the CFD fields (storage and arithmetic in
// fp32; constants rounded from the host's fp64 step constants).  For T =
// double every expression is the reference's, operation for operation.
template <class T>
struct uv_consts {
  T alpha, ix, iy, iz, ix2, iy2, iz2, nu, fx, fy, fz;
  __device__ __forceinline__ explicit uv_consts(const sf_consts& c)
      : alpha((T)c.alpha), ix((T)c.ix), iy((T)c.iy), iz((T)c.iz), ix2((T)c.ix2), iy2((T)c.iy2), iz2((T)c.iz2),
        nu((T)c.nu), fx((T)c.fx), fy((T)c.fy), fz((T)c.fz) {}
};

// flux + alpha * X, X evaluated lazily (see above)
#define SF_BLEND(f, X)                            \
  do {                                            \
    if (BLEND || f == (T)0) f += s.alpha * (X);   \
  } while (0)

template <class Acc, bool BLEND = true, class T = double>
__device__ __forceinline__ void uv_point(const Acc& A, const uv_consts<T>& s, T dt, T out[3]) {
  const T u0 = A.u(0, 0, 0), v0 = A.v(0, 0, 0), w0 = A.w(0, 0, 0);
  {  // x momentum, at this cell's high x face
    const T ue = A.u(1, 0, 0), uw = A.u(-1, 0, 0);
    const T un = A.u(0, 1, 0), us = A.u(0, -1, 0);
    const T ut = A.u(0, 0, 1), ub = A.u(0, 0, -1);
    const T vn = A.v(0, 0, 0) + A.v(1, 0, 0), vs = A.v(0, -1, 0) + A.v(1, -1, 0);
    const T wt = A.w(0, 0, 0) + A.w(1, 0, 0), wb = A.w(0, 0, -1) + A.w(1, 0, -1);
    T fux = (u0 + ue) * (u0 + ue) - (uw + u0) * (uw + u0);
    SF_BLEND(fux, (fabs(u0 + ue) * (u0 - ue) - fabs(uw + u0) * (uw - u0)));
    T fuy = vn * (u0 + un) - vs * (us + u0);
    SF_BLEND(fuy, (fabs(vn) * (u0 - un) - fabs(vs) * (us - u0)));
    T fuz = wt * (u0 + ut) - wb * (ub + u0);
    SF_BLEND(fuz, (fabs(wt) * (u0 - ut) - fabs(wb) * (ub - u0)));
    const T lapu = (ue - (T)2 * u0 + uw) * s.ix2 + (un - (T)2 * u0 + us) * s.iy2 +
                        (ut - (T)2 * u0 + ub) * s.iz2;
    const T rhsu = (A.q(0, 0, 0) - A.q(1, 0, 0)) * s.ix -
                        (T)0.25 * (fux * s.ix + fuy * s.iy + fuz * s.iz) + s.nu * lapu + s.fx;
    const T r = u0 + dt * rhsu;
    out[0] = r;
  }
  {  // y momentum, at the high y face
    const T ve = A.v(1, 0, 0), vw = A.v(-1, 0, 0);
    const T vnn = A.v(0, 1, 0), vss = A.v(0, -1, 0);
    const T vt = A.v(0, 0, 1), vb = A.v(0, 0, -1);
    const T ue2 = A.u(0, 0, 0) + A.u(0, 1, 0), uw2 = A.u(-1, 0, 0) + A.u(-1, 1, 0);
    const T wt2 = A.w(0, 0, 0) + A.w(0, 1, 0), wb2 = A.w(0, 0, -1) + A.w(0, 1, -1);
    T fvx = ue2 * (v0 + ve) - uw2 * (vw + v0);
    SF_BLEND(fvx, (fabs(ue2) * (v0 - ve) - fabs(uw2) * (vw - v0)));
    T fvy = (v0 + vnn) * (v0 + vnn) - (vss + v0) * (vss + v0);
    SF_BLEND(fvy, (fabs(v0 + vnn) * (v0 - vnn) - fabs(vss + v0) * (vss - v0)));
    T fvz = wt2 * (v0 + vt) - wb2 * (vb + v0);
    SF_BLEND(fvz, (fabs(wt2) * (v0 - vt) - fabs(wb2) * (vb - v0)));
    const T lapv = (ve - (T)2 * v0 + vw) * s.ix2 + (vnn - (T)2 * v0 + vss) * s.iy2 +
                        (vt - (T)2 * v0 + vb) * s.iz2;
    const T rhsv = (A.q(0, 0, 0) - A.q(0, 1, 0)) * s.iy -
                        (T)0.25 * (fvx * s.ix + fvy * s.iy + fvz * s.iz) + s.nu * lapv + s.fy;
    const T r = v0 + dt * rhsv;
    out[1] = r;
  }
  {  // z momentum, at the high z face
    const T we = A.w(1, 0, 0), ww = A.w(-1, 0, 0);
    const T wn = A.w(0, 1, 0), ws = A.w(0, -1, 0);
    const T wtt = A.w(0, 0, 1), wbb = A.w(0, 0, -1);
    const T ue3 = A.u(0, 0, 0) + A.u(0, 0, 1), uw3 = A.u(-1, 0, 0) + A.u(-1, 0, 1);
    const T vn3 = A.v(0, 0, 0) + A.v(0, 0, 1), vs3 = A.v(0, -1, 0) + A.v(0, -1, 1);
    T fwx = ue3 * (w0 + we) - uw3 * (ww + w0);
    SF_BLEND(fwx, (fabs(ue3) * (w0 - we) - fabs(uw3) * (ww - w0)));
    T fwy = vn3 * (w0 + wn) - vs3 * (ws + w0);
    SF_BLEND(fwy, (fabs(vn3) * (w0 - wn) - fabs(vs3) * (ws - w0)));
    T fwz = (w0 + wtt) * (w0 + wtt) - (wbb + w0) * (wbb + w0);
    SF_BLEND(fwz, (fabs(w0 + wtt) * (w0 - wtt) - fabs(wbb + w0) * (wbb - w0)));
    const T lapw = (we - (T)2 * w0 + ww) * s.ix2 + (wn - (T)2 * w0 + ws) * s.iy2 +
                        (wtt - (T)2 * w0 + wbb) * s.iz2;
    const T rhsw = (A.q(0, 0, 0) - A.q(0, 0, 1)) * s.iz -
                        (T)0.25 * (fwx * s.ix + fwy * s.iy + fwz * s.iz) + s.nu * lapw + s.fz;
    const T r = w0 + dt * rhsw;
    out[2] = r;
  }
}

#undef SF_BLEND

}  // namespace sfb
