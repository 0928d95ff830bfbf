// sf_sweep_tma.cu -- the fused red-black half-sweep, TMA-pipelined for sm_100a.
//
// Same arithmetic and boundary semantics as k_sweep_div in sf_kernels.cu (see
// the comment there and cfd.hpp:289-305, 595-720, exchange.hpp:231-480), but
// the loads are 3-D TMA boxes (cp.async.bulk.tensor) into a kStages-deep ring
// of shared-memory plane tiles, each stage guarded by an mbarrier with
// expect_tx.  Per stage and CTA (tile 32 x 8 cells of one z plane):
//     divu  36 x 10  (x and y halo: the sweep reads +x/+y, the -x/-y swept
//                    neighbours need -x/-y; x starts at i0-2, see kXL)
//     vx    34 x 8   (columns i0-2, i0-1 for the -x neighbour)
//     vy    32 x 9   (row j0-1 for the -y neighbour)
//     p, vz 32 x 8
// The +z neighbour of divu is the next stage's centre; the -z swept neighbour
// of vz is carried in a register while marching z.  One elected thread
// refills the stage just consumed after a CTA barrier, keeping kStages-1
// planes (~34 KB) in flight per CTA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "sf_kernels.cuh"

namespace sfb {

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// ---------------------------------------------------------------------------
// stage layout (every TMA destination 128-byte aligned)
// ---------------------------------------------------------------------------
// On B200 a TMA tile load must START on a 16-byte aligned inner coordinate
// (an odd fp64 x start raises "illegal instruction"; measured with
// scripts/probes/tma_probe2.cu), so the x halo boxes begin kXL = 16 / sizeof(T)
// cells left of the tile (2 fp64, 4 fp32): for fp64 divu covers x in
// [i0-2, i0+34), vx covers [i0-2, i0+32).
//
// Shared-memory stage of one z plane for a TX x TY tile (every TMA
// destination 128-byte aligned), element type T (fp64, or fp32 for the fp32
// variant of the CFD fields):
//   divu (TX+2kXL) x (TY+2), vx (TX+kXL) x TY, vy TX x (TY+1), p and vz TX x TY
template <int TX, int TY, class T = double>
struct tile {
  static constexpr int ES = (int)sizeof(T), kXL = 16 / ES;
  static constexpr int DW = TX + 2 * kXL, DH = TY + 2, UW = TX + kXL, VH = TY + 1;
  static constexpr int r128(int b) { return (b + 127) / 128 * 128; }
  static constexpr int OFF_D = 0;
  static constexpr int OFF_U = r128(ES * DH * DW);
  static constexpr int OFF_V = OFF_U + r128(ES * TY * UW);
  static constexpr int OFF_P = OFF_V + r128(ES * VH * TX);
  static constexpr int OFF_W = OFF_P + r128(ES * TY * TX);
  static constexpr int BYTES = OFF_W + r128(ES * TY * TX);
  static constexpr uint32_t TXB = (uint32_t)ES * (DH * DW + TY * UW + VH * TX + 2 * TY * TX);
  static_assert((UW * ES) % 16 == 0 && (DW * ES) % 16 == 0 && (TX * ES) % 16 == 0,
                "TMA rows must be 16-byte multiples");
};

struct sweep_maps {  // per block: [field][physical buffer]
  CUtensorMap m[kMaxBlocks][SF_NFIELDS][kSlots];
};

// STAGES: ring depth.  MINB: CTAs per SM the register budget targets.
// (Measured alternatives -- a warp-specialised TMA producer, 2-8 stages,
// 64x4 / 128x2 tiles, streaming stores, evict-first loads -- were all slower;
// DESIGN.md §4.)
template <int STAGES, int MINB, int TX, int TY, class T>
__global__ void __launch_bounds__(TX* TY, MINB)
    k_sweep_div_tma(sf_dev_table* __restrict__ tab, const sf_work* __restrict__ items, int nitems,
                    int zc, sf_consts s, sf_dev_ctl* ctl, sf_host_flag* hflag,
                    unsigned int total_ctas, const sweep_maps* __restrict__ maps, int finalize) {
  constexpr int kStages = STAGES;
  using TL = tile<TX, TY, T>;
  constexpr int kXL = TL::kXL;
  // finalize 2: redo of a temporal pass's first sweep (sf_sweep2.cu), runs
  // only when that pass flagged it
  if (finalize == 2) {
    if (!*reinterpret_cast<const volatile int*>(&ctl->redo)) return;
  } else if (*reinterpret_cast<const volatile int*>(&ctl->done)) {
    return;
  }
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto sptr = [&](int st, int off) { return reinterpret_cast<T*>(smem_raw + st * TL::BYTES + off); };
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ T smb[8];

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX + tx;
  // tile location
  const int cta = blockIdx.x;
  const int it = nitems > 1 ? find_item(items, nitems, cta) : 0;
  const sf_work& wk = items[it];
  const int b = wk.blk;
  const int local = cta - wk.cta_begin;
  const int tix = local % wk.tiles[0];
  const int tiy = (local / wk.tiles[0]) % wk.tiles[1];
  const int tiz = local / (wk.tiles[0] * wk.tiles[1]);
  const long long i0 = wk.lo[0] + (long long)tix * TX;
  const long long j0 = wk.lo[1] + (long long)tiy * TY;
  const long long k0 = wk.lo[2] + (long long)tiz * zc;
  const long long k1 = min(k0 + zc, wk.hi[2]);
  const int nplanes = (int)(k1 - k0);
  const sf_dev_block& B = tab->blk[b];

  const double beta = ctl->beta, dt = ctl->dt;
  const T Tix = (T)s.ix, Tiy = (T)s.iy, Tiz = (T)s.iz;
  const int color = finalize == 2 ? (ctl->color ^ 1) : ctl->color;
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < kStages; ++q) {
      mbar_init(&bars[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 8) {
    // -(beta * bscale[bx][by][bz]) exactly as cfd.hpp:712-715 forms it
    double sc = 1.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q == tid) sc = s.bscale[q >> 2][(q >> 1) & 1][q & 1];
    smb[tid] = (T)(-(beta * sc));
  }
  __syncthreads();

  // TMA box origins (tensor coordinates: x = xo + i, y = g + j, z = g + k)
  const long long xo = B.base % B.sx;
  const int g = B.g;
  const CUtensorMap* mD = &maps->m[b][SF_DIVU][tab->bidx[b][SF_DIVU][FRONT]];
  const CUtensorMap* mU = &maps->m[b][SF_VX][tab->bidx[b][SF_VX][FRONT]];
  const CUtensorMap* mV = &maps->m[b][SF_VY][tab->bidx[b][SF_VY][FRONT]];
  const CUtensorMap* mW = &maps->m[b][SF_VZ][tab->bidx[b][SF_VZ][FRONT]];
  const CUtensorMap* mP = &maps->m[b][SF_P][tab->bidx[b][SF_P][FRONT]];
  const int xc = (int)(xo + i0), yc = (int)(g + j0), zc0 = (int)(g + k0);
  auto issue = [&](int stage, int plane) {
    mbar_expect_tx(&bars[stage], TL::TXB);
    tma_load_3d(sptr(stage, TL::OFF_D), mD, &bars[stage], xc - kXL, yc - 1, zc0 + plane);
    tma_load_3d(sptr(stage, TL::OFF_U), mU, &bars[stage], xc - kXL, yc, zc0 + plane);
    tma_load_3d(sptr(stage, TL::OFF_V), mV, &bars[stage], xc, yc - 1, zc0 + plane);
    tma_load_3d(sptr(stage, TL::OFF_P), mP, &bars[stage], xc, yc, zc0 + plane);
    tma_load_3d(sptr(stage, TL::OFF_W), mW, &bars[stage], xc, yc, zc0 + plane);
  };
  if (tid == 0) {
    const int npro = nplanes < kStages ? nplanes : kStages;
    for (int q = 0; q < npro; ++q) issue(q, q);
  }

  T* __restrict__ Dn = reinterpret_cast<T*>(tab->ptr[b][SF_DIVU][ALT]);
  T* __restrict__ P = reinterpret_cast<T*>(tab->ptr[b][SF_P][FRONT]);
  T* __restrict__ Un = reinterpret_cast<T*>(tab->ptr[b][SF_VX][ALT]);
  T* __restrict__ Vn = reinterpret_cast<T*>(tab->ptr[b][SF_VY][ALT]);
  T* __restrict__ Wn = reinterpret_cast<T*>(tab->ptr[b][SF_VZ][ALT]);
  const T* __restrict__ D = reinterpret_cast<T*>(tab->ptr[b][SF_DIVU][FRONT]);
  const T* __restrict__ W = reinterpret_cast<T*>(tab->ptr[b][SF_VZ][FRONT]);
  const T cu = (T)(dt * Tix), cv = (T)(dt * Tiy), cw = (T)(dt * Tiz);

  const long long i = i0 + tx, j = j0 + ty;
  const bool act = i < wk.hi[0] && j < wk.hi[1];
  const long long n0 = B.n[0], n1 = B.n[1], n2 = B.n[2];
  const long long sx = B.sx, sxy = B.sx * B.sy;
  const long long gi = B.lo[0] + i, gj = B.lo[1] + j;
  const int per0 = s.per[0], per1 = s.per[1], per2 = s.per[2];
  auto bin = [](int per, long long gg, long long nm1) { return per | ((gg > 0) & (gg < nm1)); };
  auto bnx = [](int per, long long gg, long long nm1) { return per | (gg + 1 < nm1); };
  const long long gim = i > 0 ? gi - 1 : B.nb_ghost_gidx[0];
  const long long gjm = j > 0 ? gj - 1 : B.nb_ghost_gidx[2];
  const int bx = bin(per0, gi, s.nm1[0]), bxp = bnx(per0, gi, s.nm1[0]);
  const int by = bin(per1, gj, s.nm1[1]), byp = bnx(per1, gj, s.nm1[1]);
  const int bxm = bin(per0, gim, s.nm1[0]), bxpm = bnx(per0, gim, s.nm1[0]);
  const int bym = bin(per1, gjm, s.nm1[1]), bypm = bnx(per1, gjm, s.nm1[1]);
  // scale-table row indices per use (the z bit is or-ed in per plane)
  const int ic = (bx << 2) | (by << 1), iex = (bxp << 2) | (by << 1), iey = (bx << 2) | (byp << 1);
  const int ixm = (bxm << 2) | (by << 1), ixpm = (bxpm << 2) | (by << 1);
  const int iym = (bx << 2) | (bym << 1), iypm = (bx << 2) | (bypm << 1);
  const int fxl = B.face[0], fxh = B.face[1], fyl = B.face[2], fyh = B.face[3];
  const int fzl = B.face[4], fzh = B.face[5];
  const bool pin_u = (fxh == FACE_WALL || fxh == FACE_SYM) && i == n0 - 1;
  const bool pin_v = (fyh == FACE_WALL || fyh == FACE_SYM) && j == n1 - 1;
  const bool pin_w = (fzh == FACE_WALL || fzh == FACE_SYM);
  const T pv_u = fxh == FACE_WALL ? B.fvel[1][0] : 0.0;
  const T pv_v = fyh == FACE_WALL ? B.fvel[3][1] : 0.0;
  const T pv_w = fzh == FACE_WALL ? B.fvel[5][2] : 0.0;
  const bool xm_swept = i > 0 || fxl == FACE_PROC || fxl == FACE_SELF;
  const bool ym_swept = j > 0 || fyl == FACE_PROC || fyl == FACE_SELF;
  // Interior column: every x/y scale bit of the cell and of its -x/-y
  // neighbours is 1 (so each -(beta*bscale) is -(beta*1.0)), the -x/-y
  // neighbours are owned cells of opposite parity, and no pin or ghost write
  // applies.  The z part is checked per plane.  The fast path evaluates the
  // identical IEEE operations in the identical order, so it is bitwise the
  // general path restricted to such cells.
  const bool col_fast = i >= 1 && i <= n0 - 2 && j >= 1 && j <= n1 - 2 && bx && bxp && bxm &&
                        bxpm && by && byp && bym && bypm;
  const T mbI = smb[7];  // -(beta * bscale[1][1][1])
  const int zlo_fast = (int)max(1ll, (per2 ? 0ll : 1ll) - B.lo[2]);  // local k range of the fast path
  const int zhi_fast = (int)min(n2 - 2, (per2 ? n2 - 2 : s.nm1[2] - 2 - B.lo[2]));
  const int par_col = (int)((gi + gj) & 1);

  long long o = off(B, i, j, k0);
  unsigned long long rmax = 0ull;
  T wm_new = 0.0;
  if (act) {  // swept w of the cell below the chunk (carried while marching)
    const long long gk = B.lo[2] + k0;
    const T dC0 = D[o];
    if (k0 > 0 || fzl == FACE_PROC || fzl == FACE_SELF) {
      const long long gkm = k0 > 0 ? gk - 1 : B.nb_ghost_gidx[4];
      const int bzm = bin(per2, gkm, s.nm1[2]), bzpm = bnx(per2, gkm, s.nm1[2]);
      const T a0m = (((gi + gj + gkm) & 1) == color) ? 1.0 : 0.0, a1m = 1.0 - a0m;
      const T d0m = smb[ic | bzm] * D[o - sxy] * a0m;
      const T ezm = smb[ic | bzpm] * dC0 * a1m;
      wm_new = W[o - sxy] + cw * (d0m - ezm);
    } else {
      wm_new = W[o - sxy];
    }
  }

  for (int kk = 0; kk < nplanes; ++kk, o += sxy) {
    const int st = kk % kStages;
    mbar_wait(&bars[st], (uint32_t)((kk / kStages) & 1));
    const bool has_next = kk + 1 < nplanes;
    const int st1 = (kk + 1) % kStages;
    if (has_next) mbar_wait(&bars[st1], (uint32_t)(((kk + 1) / kStages) & 1));
    const int kl = (int)(k0 + kk);
    if (act && col_fast && kl >= zlo_fast && kl <= zhi_fast) {
      const T* Td = sptr(st, TL::OFF_D);
      const T* Tu = sptr(st, TL::OFF_U);
      const T* Tv = sptr(st, TL::OFF_V);
      const T* Tp = sptr(st, TL::OFF_P);
      const T* Tw = sptr(st, TL::OFF_W);
      const T dC = Td[(ty + 1) * TL::DW + (tx + kXL)];
      const T dXp = Td[(ty + 1) * TL::DW + (tx + kXL + 1)], dXm = Td[(ty + 1) * TL::DW + (tx + kXL - 1)];
      const T dYp = Td[(ty + 2) * TL::DW + (tx + kXL)], dYm = Td[(ty) * TL::DW + (tx + kXL)];
      const T dZp = has_next ? sptr(st1, TL::OFF_D)[(ty + 1) * TL::DW + (tx + kXL)] : D[o + sxy];
      const T p0 = Tp[(ty) * TX + (tx)], u0 = Tu[(ty) * TL::UW + (tx + kXL)], uml = Tu[(ty) * TL::UW + (tx + kXL - 1)];
      const T v0 = Tv[(ty + 1) * TX + (tx)], vml = Tv[(ty) * TX + (tx)], w0 = Tw[(ty) * TX + (tx)];
      const int par = par_col ^ ((int)(B.lo[2] + kl) & 1);
      const T a0 = (par == color) ? 1.0 : 0.0, a1 = 1.0 - a0;
      const T d0 = mbI * dC * a0;
      const T ex = mbI * dXp * a1;
      const T ey = mbI * dYp * a1;
      const T ez = mbI * dZp * a1;
      const T pn = p0 + d0;
      const T un = u0 + cu * (d0 - ex);
      const T vn = v0 + cv * (d0 - ey);
      const T wn = w0 + cw * (d0 - ez);
      // -x / -y neighbours: parity a1, their +x/+y term is mbI*dC*a0 == d0
      const T umn = uml + cu * (mbI * dXm * a1 - d0);
      const T vmn = vml + cv * (mbI * dYm * a1 - d0);
      T dd = (un - umn) * Tix;
      dd += (vn - vmn) * Tiy;
      dd += (wn - wm_new) * Tiz;
      P[o] = pn;
      Un[o] = un;
      Vn[o] = vn;
      Wn[o] = wn;
      Dn[o] = dd;
      const unsigned long long bb = abs_bits((double)dd);
      rmax = bb > rmax ? bb : rmax;
      wm_new = wn;
    } else if (act) {
      const T* Td = sptr(st, TL::OFF_D);
      const T* Tu = sptr(st, TL::OFF_U);
      const T* Tv = sptr(st, TL::OFF_V);
      const T* Tp = sptr(st, TL::OFF_P);
      const T* Tw = sptr(st, TL::OFF_W);
      const long long k = k0 + kk;
      const long long gk = B.lo[2] + k;
      const int bz = bin(per2, gk, s.nm1[2]), bzp = bnx(per2, gk, s.nm1[2]);
      const T dC = Td[(ty + 1) * TL::DW + (tx + kXL)];
      const T dXp = Td[(ty + 1) * TL::DW + (tx + kXL + 1)], dXm = Td[(ty + 1) * TL::DW + (tx + kXL - 1)];
      const T dYp = Td[(ty + 2) * TL::DW + (tx + kXL)], dYm = Td[(ty) * TL::DW + (tx + kXL)];
      const T dZp = has_next ? sptr(st1, TL::OFF_D)[(ty + 1) * TL::DW + (tx + kXL)] : D[o + sxy];
      const T p0 = Tp[(ty) * TX + (tx)], u0 = Tu[(ty) * TL::UW + (tx + kXL)], uml = Tu[(ty) * TL::UW + (tx + kXL - 1)];
      const T v0 = Tv[(ty + 1) * TX + (tx)], vml = Tv[(ty) * TX + (tx)], w0 = Tw[(ty) * TX + (tx)];
      const T a0 = (((gi + gj + gk) & 1) == color) ? 1.0 : 0.0, a1 = 1.0 - a0;
      // this cell's sweep (cfd.hpp:712-719)
      const T d0 = smb[ic | bz] * dC * a0;
      const T ex = smb[iex | bz] * dXp * a1;
      const T ey = smb[iey | bz] * dYp * a1;
      const T ez = smb[ic | bzp] * dZp * a1;
      P[o] = p0 + d0;
      T un = u0 + cu * (d0 - ex);
      T vn = v0 + cv * (d0 - ey);
      T wn = w0 + cw * (d0 - ez);
      if (pin_u) un = pv_u;
      if (pin_v) vn = pv_v;
      if (pin_w && k == n2 - 1) wn = pv_w;
      // swept -x / -y neighbours (the refreshed values DIVERGENCE reads)
      T umn, vmn;
      if (xm_swept) {
        const T a0m = i > 0 ? a1 : ((((gim + gj + gk) & 1) == color) ? 1.0 : 0.0);
        const T a1m = 1.0 - a0m;
        const T d0m = smb[ixm | bz] * dXm * a0m;
        const T exm = smb[ixpm | bz] * dC * a1m;
        umn = uml + cu * (d0m - exm);
      } else {
        umn = fxl == FACE_OUT ? un : uml;
      }
      if (ym_swept) {
        const T a0m = j > 0 ? a1 : ((((gi + gjm + gk) & 1) == color) ? 1.0 : 0.0);
        const T a1m = 1.0 - a0m;
        const T d0m = smb[iym | bz] * dYm * a0m;
        const T eym = smb[iypm | bz] * dC * a1m;
        vmn = vml + cv * (d0m - eym);
      } else {
        vmn = fyl == FACE_OUT ? vn : vml;
      }
      if (k == 0 && fzl == FACE_OUT) wm_new = wn;
      // DIVERGENCE (cfd.hpp:605-608)
      T dd = (un - umn) * Tix;
      dd += (vn - vmn) * Tiy;
      dd += (wn - wm_new) * Tiz;
      Un[o] = un;
      Vn[o] = vn;
      Wn[o] = wn;
      Dn[o] = dd;
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
      const unsigned long long bb = abs_bits((double)dd);
      rmax = bb > rmax ? bb : rmax;
      wm_new = wn;
    }
    __syncthreads();  // every thread is done with stage st
    if (tid == 0 && kk + kStages < nplanes) issue(st, kk + kStages);
  }

  if (finalize == 2) {  // counters and residual were set by the temporal pass
    if (last_cta(&ctl->ctas_done, total_ctas) && tid == 0) {
      __threadfence();
      ctl->ctas_done = 0u;
      ctl->redo = 0;
      for (int q = 0; q < tab->nblocks; ++q)
        for (int f = 0; f < 5; ++f) {
          if (f == SF_P) continue;
          double* tmp = tab->ptr[q][f][FRONT];
          tab->ptr[q][f][FRONT] = tab->ptr[q][f][ALT];
          tab->ptr[q][f][ALT] = tmp;
          const unsigned char ti = tab->bidx[q][f][FRONT];
          tab->bidx[q][f][FRONT] = tab->bidx[q][f][ALT];
          tab->bidx[q][f][ALT] = ti;
        }
    }
    return;
  }
  unsigned long long rm[1] = {rmax};
  block_max_atomic<1>(rm, &ctl->acc[0]);
  if (!finalize) return;  // across ranks: allreduce, then CTL_FINISH_FUSED
  if (last_cta(&ctl->ctas_done, total_ctas)) {
    if (tid == 0) {
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
      for (int q = 0; q < tab->nblocks; ++q)
        for (int f = 0; f < SF_NFIELDS; ++f) {
          if (f == SF_P) continue;
          double* tmp = tab->ptr[q][f][FRONT];
          tab->ptr[q][f][FRONT] = tab->ptr[q][f][ALT];
          tab->ptr[q][f][ALT] = tmp;
          const unsigned char ti = tab->bidx[q][f][FRONT];
          tab->bidx[q][f][FRONT] = tab->bidx[q][f][ALT];
          tab->bidx[q][f][ALT] = ti;
        }
      if (hflag) {
        hflag->sweeps = sweeps;
        hflag->residual = residual;
        hflag->done = more ? 0 : 1;
        hflag->color = ctl->color;
        __threadfence_system();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps + launch
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

constexpr int kSweepTX = 32, kSweepTY = 8, kSweepStages = 4, kSweepMinB = 2;
// tile shape of the single half-sweep kernel
void sweep_tile_shape(int* tx, int* ty) {
  *tx = kSweepTX;
  *ty = kSweepTY;
}

// Box shape per field role (see tile<>); es = bytes per value.
static void box_for(int field, cuuint32_t box[3], int es) {
  const int tx = kSweepTX, ty = kSweepTY, xl = 16 / es;
  box[2] = 1;
  switch (field) {
    case SF_DIVU: box[0] = tx + 2 * xl; box[1] = ty + 2; break;
    case SF_VX: box[0] = tx + xl; box[1] = ty; break;
    case SF_VY: box[0] = tx; box[1] = ty + 1; break;
    default: box[0] = tx; box[1] = ty; break;
  }
}

int encode_sweep_map(void* map_out, double* base, long long sx, long long sy, long long sz, int field, int es) {
  auto fn = encode_fn();
  if (!fn) return 1;
  cuuint64_t gdim[3] = {(cuuint64_t)sx, (cuuint64_t)sy, (cuuint64_t)sz};
  cuuint64_t gstride[2] = {(cuuint64_t)(sx * es), (cuuint64_t)(sx * sy * es)};
  cuuint32_t box[3];
  box_for(field, box, es);
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(map_out),
                  es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, gdim,
                  gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 2;
}

// a 3-D tensor map over one padded array with a (bw, bh, 1) box; es = bytes
// per value (8: FLOAT64, 4: FLOAT32 with the same layout in elements)
int encode_box_map(void* map_out, double* base, long long sx, long long sy, long long sz, int bw, int bh, int es) {
  auto fn = encode_fn();
  if (!fn) return 1;
  cuuint64_t gdim[3] = {(cuuint64_t)sx, (cuuint64_t)sy, (cuuint64_t)sz};
  cuuint64_t gstride[2] = {(cuuint64_t)(sx * es), (cuuint64_t)(sx * sy * es)};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(map_out),
                  es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, gdim,
                  gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 2;
}

size_t sweep_maps_bytes() { return sizeof(sweep_maps); }
size_t sweep_map_offset(int b, int f, int s) {
  return offsetof(sweep_maps, m) + sizeof(CUtensorMap) * ((size_t)(b * SF_NFIELDS + f) * kSlots + s);
}

template <class T>
static void launch_sweep_tma_t(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                               sf_host_flag* hflag, const void* maps, int fin, cudaStream_t st) {
  constexpr int S = kSweepStages, M = kSweepMinB, TX = kSweepTX, TY = kSweepTY;
  const size_t smem = (size_t)tile<TX, TY, T>::BYTES * S;
  auto k = k_sweep_div_tma<S, M, TX, TY, T>;
  ensure_smem_attr((const void*)k, (int)smem);
  k<<<nctas, dim3(TX, TY), smem, st>>>(vw.tab, vw.items, vw.nitems, zc, c, ctl, hflag, (unsigned)nctas,
                                       static_cast<const sweep_maps*>(maps), fin);
}
void launch_sweep_div_tma(const table_view& vw, int nctas, int zc, const sf_consts& c,
                          sf_dev_ctl* ctl, sf_host_flag* hflag, const void* maps, int fin,
                          cudaStream_t st, int es) {
  if (nctas <= 0) return;
  if (es == 4)
    launch_sweep_tma_t<float>(vw, nctas, zc, c, ctl, hflag, maps, fin, st);
  else
    launch_sweep_tma_t<double>(vw, nctas, zc, c, ctl, hflag, maps, fin, st);
}

}  // namespace sfb
