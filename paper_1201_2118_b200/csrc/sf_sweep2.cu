// sf_sweep2.cu -- two red-black half-sweeps per pass (temporal blocking).
//
// pressure_iteration (cfd.hpp:289-305) runs sweep A (colour c) and then sweep B
// (colour c^1). Each sweep is followed by the velocity refresh, DIVERGENCE and
// the loop test. This kernel keeps the intermediate state S1 = (p1, u1, v1,
// w1, divu1) on chip. For each z plane it first computes S1 over the tile
// widened by the halo sweep B reads, x in [i0-2, i0+TX] and y in
// [j0-2, j0+TY], into a 2-plane shared-memory ring. It then runs sweep B on
// the tile. A pass therefore reads S0 (divu, p, vx, vy, vz) and writes S2
// once: 80 bytes per cell for TWO half-sweeps instead of 160.
//
// Every value is produced by the same IEEE operations in the same order as
// the single-sweep kernel (sf_sweep_tma.cu). Updates of neighbouring cells
// are recomputed, never approximated, so S2 and both residuals are bitwise
// those of two single sweeps.
//
// S2 goes to the ALT buffers and S0 stays intact. If the loop test after
// sweep A says stop, the last CTA sets ctl->redo. The predicated single-sweep
// kernel then recomputes S1 from S0 (launch_sweep_div_tma, fin = 2).
//
// Scope: one grid component per device whose six faces are all physical
// walls or symmetry planes (the cavity of the benchmark). The driver checks
// this; every other configuration keeps the single-sweep kernel.
//
// Wall/symmetry ghost rules used on chip (exchange.hpp:231-480, as the
// single kernel applies them):
//  - the pinned wall-normal ghosts u(-1), v(-1), w(-1) keep their S0 value;
//  - the last owned wall-normal velocities are pinned to the wall value;
//  - divu ghosts mirror the adjacent owned cell.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "sf_kernels.cuh"

namespace sfb {

namespace {

__device__ __forceinline__ uint32_t smem32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem32(bar)));
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

constexpr int r128(int b) { return (b + 127) / 128 * 128; }

// Tile geometry: TX x TY cells per CTA (one thread each), the S1 tile widened
// to EW x EH, and the S0 stage layout (every TMA destination 128-byte aligned)
// for element type T (fp64; fp32 for the fp32 variant of the CFD fields). A
// TMA box starts on a 16-byte aligned x: XA = 16 / sizeof(T) cells left of the
// tile (2 fp64, 4 fp32), so the widened S1 region (from i0-2) sits XSH = XA-2
// cells into each S0 row.
template <int TXV, int TYV, class T = double>
struct geom {
  static constexpr int ES = (int)sizeof(T), XA = 16 / ES, XSH = XA - 2;
  static constexpr int TX = TXV, TY = TYV, NT = TX * TY;
  static constexpr int EW = TX + 3, EH = TY + 3, EN = EW * EH;  // widened S1 tile
  static constexpr int NE = (EN + NT - 1) / NT;                  // widened cells per thread
  static constexpr int R2 = EN - 1 - NT;                         // second-round cells
  static constexpr int IW = (TX + 2 + XA + XA - 1) / XA * XA;    // S0 box width (x from i0-XA): 36 / 40
  static constexpr int IDH = TY + 4, IFH = TY + 3;               // divu / other S0 box heights
  static constexpr int IN_D = 0;
  static constexpr int IN_U = r128(ES * IW * IDH);
  static constexpr int IN_V = IN_U + r128(ES * IW * IFH);
  static constexpr int IN_W = IN_V + r128(ES * IW * IFH);
  static constexpr int IN_P = IN_W + r128(ES * IW * IFH);
  static constexpr int IN_BYTES = IN_P + r128(ES * IW * IFH);
  static constexpr uint32_t IN_TX = (uint32_t)ES * (IW * IDH + 4 * IW * IFH);
  static constexpr int smem_bytes(int nin) { return nin * IN_BYTES + (4 * 4 + 3) * EN * ES; }
  static_assert(NE == 2 && R2 > 0 && R2 <= NT, "two rounds of widened cells per thread");
  static_assert(IN_BYTES % ES == 0 && (IW * ES) % 16 == 0, "TMA rows");
};

enum { U1 = 0, V1 = 1, W1 = 2, P1 = 3, D1 = 4 };

struct maps2_t {  // [block][field][physical buffer]
  CUtensorMap m[kMaxBlocks][SF_NFIELDS][kSlots];
};

}  // namespace

size_t sweep2_maps_bytes() { return sizeof(maps2_t); }
size_t sweep2_map_offset(int b, int f, int s) {
  return sizeof(CUtensorMap) * (((size_t)b * SF_NFIELDS + f) * kSlots + s);
}
// 32 x 8 tiles, 3 S0 stages, 2 CTAs per SM. (Measured alternatives: 32 x 16
// tiles, 6 stages at 1 CTA/SM, L2 prefetch of later planes -- all slower;
// DESIGN.md §10.)
constexpr int kPassTY = 8, kPassStages = 3, kPassMinB = 2, kPassMinB32 = 3;
// the x-slab form: 16 x 16 tiles for the slabs beside the interior tiles
// along x (16 cells wide: one tile column where 32-wide tiles would take two
// half-empty ones)
constexpr int kSlabTX = 16, kSlabTY = 16;
int sweep2_tile_y() { return kPassTY; }
void sweep2_tile(int shape, int* tx, int* ty) {
  *tx = shape ? kSlabTX : kTX;
  *ty = shape ? kSlabTY : kPassTY;
}
void sweep2_box(int field, int* bw, int* bh, int es, int shape) {
  if (shape) {
    *bw = es == 4 ? geom<kSlabTX, kSlabTY, float>::IW : geom<kSlabTX, kSlabTY, double>::IW;
    *bh = field == SF_DIVU ? kSlabTY + 4 : kSlabTY + 3;
    return;
  }
  *bw = es == 4 ? geom<kTX, kPassTY, float>::IW : geom<kTX, kPassTY, double>::IW;
  *bh = field == SF_DIVU ? kPassTY + 4 : kPassTY + 3;
}

// Schedule (S0 plane q and S1 plane m both mean z = k0 - 2 + q / m). One CTA
// barrier per plane; iteration u runs
//     phase u:  s1_fields(m = u+2)  and  s1_div(m = u+1)     (independent)
//     barrier
//     sweep B on plane m = u (u >= 2), overlapping phase u+1 of other warps
// The first threads take the second round of s1_fields, the last ones that of
// s1_div (R2 cells each), so the phases are balanced across warps; with 32x8
// every warp does three cell updates per phase. Rings: S0 planes in q % NIN
// (NIN >= 3), S1 fields (u1 v1 w1 p1) in m % 4, divu1 in m % 3 -- the slot a
// phase overwrites was last read before the previous barrier.
// The end of a temporal pass (every CTA of every launch of the pass): fold
// both sweeps' residual maxima; with finalize, the last CTA evaluates both loop
// tests (cfd.hpp:295-303): stop after sweep A (S0 intact: the single kernel
// redoes it, ctl->redo), or count both sweeps and swap FRONT/ALT. Across ranks
// (finalize 0) the caller allreduces acc[0..1] and runs CTL_FINISH_PASS.
__device__ __forceinline__ void pass_finalize(unsigned long long (&rr)[2], sf_dev_table* tab, sf_dev_ctl* ctl,
                                              sf_host_flag* hflag, unsigned total_ctas, int finalize) {
  block_max_atomic<2>(rr, &ctl->acc[0]);
  if (!finalize) return;
  if (last_cta(&ctl->ctas_done, total_ctas)) {
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      __threadfence();
      const double res1 = bits_to_max(*reinterpret_cast<volatile unsigned long long*>(&ctl->acc[0]));
      const double res2 = bits_to_max(*reinterpret_cast<volatile unsigned long long*>(&ctl->acc[1]));
      ctl->acc[0] = 0ull;
      ctl->acc[1] = 0ull;
      ctl->ctas_done = 0u;
      const int sw = ctl->sweeps;
      if (!((res1 > ctl->tolerance) && (sw + 1 < ctl->max_sweeps))) {
        ctl->sweeps = sw + 1;
        ctl->residual = res1;
        ctl->color ^= 1;
        ctl->done = 1;
        ctl->redo = 1;
      } else {
        ctl->sweeps = sw + 2;
        ctl->residual = res2;
        const int more = (res2 > ctl->tolerance) && (sw + 2 < ctl->max_sweeps);
        ctl->done = more ? 0 : 1;
        for (int q = 0; q < tab->nblocks; ++q)
          for (int f = 0; f < 5; ++f) {
            double* tmp = tab->ptr[q][f][FRONT];
            tab->ptr[q][f][FRONT] = tab->ptr[q][f][ALT];
            tab->ptr[q][f][ALT] = tmp;
            const unsigned char ti = tab->bidx[q][f][FRONT];
            tab->bidx[q][f][FRONT] = tab->bidx[q][f][ALT];
            tab->bidx[q][f][ALT] = ti;
          }
      }
      if (hflag) {
        hflag->sweeps = ctl->sweeps;
        hflag->residual = ctl->residual;
        hflag->done = ctl->done;
        hflag->color = ctl->color;
        __threadfence_system();
      }
    }
  }
}

// REMOTE: the outputs of cells within g of a processor face also go straight
// into the neighbours' ghost shells (sweep2_remote), up to 7 directions per
// cell (face, edges, corner): the ghost exchange of the next pass fused into
// this one.
template <int TXV, int TYV, int NIN, int MINB, bool PER, bool REMOTE, class T>
__global__ void __launch_bounds__(TXV * TYV, MINB)
    k_sweep2(sf_dev_table* __restrict__ tab, const sf_work* __restrict__ items, int nitems, int zc,
             sf_consts s, sf_dev_ctl* ctl, sf_host_flag* hflag, unsigned int total_ctas,
             const maps2_t* __restrict__ maps, int finalize, sweep2_pins pins,
             const sweep2_remote* __restrict__ rem) {
  static_assert(NIN >= 3, "three S0 planes are read or in flight per phase");
  using G = geom<TXV, TYV, T>;
  constexpr int ES = G::ES, XSH = G::XSH;
  constexpr int TX = G::TX, TY = G::TY, NT = G::NT, EW = G::EW, EN = G::EN, NE = G::NE, R2 = G::R2;
  constexpr int IW = G::IW, IN_D = G::IN_D, IN_U = G::IN_U, IN_V = G::IN_V, IN_W = G::IN_W, IN_P = G::IN_P;
  constexpr int IN_BYTES = G::IN_BYTES;
  constexpr uint32_t IN_TX = G::IN_TX;
  if (*reinterpret_cast<const volatile int*>(&ctl->done)) return;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[NIN];
  __shared__ T smb[8];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int cta = blockIdx.x;
  const sf_work& wk = items[nitems > 1 ? find_item(items, nitems, cta) : 0];
  const int local = cta - wk.cta_begin;
  const int tix = local % wk.tiles[0], tiy = (local / wk.tiles[0]) % wk.tiles[1];
  const int tiz = local / (wk.tiles[0] * wk.tiles[1]);
  const int i0 = (int)wk.lo[0] + tix * TX, j0 = (int)wk.lo[1] + tiy * TY;
  const int k0 = (int)wk.lo[2] + tiz * zc;
  const int k1 = (int)min((long long)k0 + zc, wk.hi[2]);
  const int nplanes = k1 - k0;
  const int b = wk.blk;
  const sf_dev_block& B = tab->blk[b];
  const int n0 = (int)B.n[0], n1 = (int)B.n[1], n2 = (int)B.n[2];
  // global extents and this block's origin: cells across a processor face
  // (another block's, valid in the ghost shell, g >= 2) are computed like
  // owned ones; cells outside the domain are physical ghosts
  const int N0 = (int)s.N[0], N1 = (int)s.N[1], N2 = (int)s.N[2];
  // periodic axes (split over components: processor faces through the
  // wrap): cells beyond the domain are the wrapped cells, with the wrapped
  // parity, owned, never pinned
  // (PER = false: no periodic axis; the wrap logic folds away at compile time)
  const int per0 = PER ? s.per[0] : 0, per1 = PER ? s.per[1] : 0, per2 = PER ? s.per[2] : 0;
  auto wrp = [](int g, int n, int per) { return per ? ((g % n) + n) % n : g; };
  const int lo0 = (int)B.lo[0], lo1 = (int)B.lo[1], lo2 = (int)B.lo[2];
  // element offsets fit 32 bits (the driver checks sx * sy * sz < 2^32):
  // one IMAD.WIDE per store address instead of a 64-bit add pair
  const unsigned sx = (unsigned)B.sx, sxy = (unsigned)(B.sx * B.sy);
  const double beta = ctl->beta, dt = ctl->dt;
  const T Tix = (T)s.ix, Tiy = (T)s.iy, Tiz = (T)s.iz;
  const int colA = ctl->color, colB = colA ^ 1;
  const T cu = (T)(dt * s.ix), cv = (T)(dt * s.iy), cw = (T)(dt * s.iz);
  const T pin_u = (T)pins.u, pin_v = (T)pins.v, pin_w = (T)pins.w;  // global high-wall normals
  const long long nm0 = s.nm1[0], nm1 = s.nm1[1], nm2 = s.nm1[2];
  auto bin = [](int per, long long gg, long long nm) { return per | ((gg > 0) & (gg < nm)); };
  auto bnx = [](int per, long long gg, long long nm) { return per | (gg + 1 < nm); };

  if (tid == 0) {
    for (int q = 0; q < NIN; ++q) bar_init(&bars[q]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 8) {
    double sc = 1.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q == tid) sc = s.bscale[q >> 2][(q >> 1) & 1][q & 1];
    smb[tid] = (T)(-(beta * sc));  // -(beta * bscale[..]) as cfd.hpp:712-715 forms it
  }
  __syncthreads();

  // ---- S0 input ring ---------------------------------------------------------
  // The x-slab form next to a physical x face: the S0 boxes start (end) on
  // the face's cache line instead of XA cells beyond it. The ghost columns
  // there never reach a result: the -x ghost's normal u is the pin and its
  // divergence only feeds the -x term a low-wall cell discards; the +x ghost's
  // divergence is the mirror of N-1 and the high-wall cell's u the pin. So
  // their box elements are clamped into the row (any value), and a 16-wide
  // slab row touches 2 lines of 128 B instead of 3 (fp32: 1 instead of 2).
  const int xsh = (TXV != kSlabTX || PER) ? 0
                  : (i0 == 0 && B.face[0] != FACE_PROC) ? G::XA
                  : (i0 + TX >= n0 && B.face[1] != FACE_PROC) ? -G::XA
                  : 0;
  const int xo = (int)(B.base % B.sx), g = B.g;
  const int xs = xo + i0 - 2 - XSH + xsh, ys = g + j0 - 2, zs = g + k0 - 2;
  const CUtensorMap* mD = &maps->m[b][SF_DIVU][tab->bidx[b][SF_DIVU][FRONT]];
  const CUtensorMap* mU = &maps->m[b][SF_VX][tab->bidx[b][SF_VX][FRONT]];
  const CUtensorMap* mV = &maps->m[b][SF_VY][tab->bidx[b][SF_VY][FRONT]];
  const CUtensorMap* mW = &maps->m[b][SF_VZ][tab->bidx[b][SF_VZ][FRONT]];
  const CUtensorMap* mP = &maps->m[b][SF_P][tab->bidx[b][SF_P][FRONT]];
  const int nin = nplanes + 4;  // S0 planes k0-2 .. k1+1
  auto issue = [&](int q) {
    if (q >= nin) return;
    unsigned char* st = sm + (q % NIN) * IN_BYTES;
    uint64_t* bar = &bars[q % NIN];
    bar_expect(bar, IN_TX);
    tma3(st + IN_D, mD, bar, xs, ys, zs + q);
    tma3(st + IN_U, mU, bar, xs, ys, zs + q);
    tma3(st + IN_V, mV, bar, xs, ys, zs + q);
    tma3(st + IN_W, mW, bar, xs, ys, zs + q);
    tma3(st + IN_P, mP, bar, xs, ys, zs + q);
  };
  const uint32_t bar0 = smem32(&bars[0]);
  auto wait_in = [&](int q) {
    if (q < nin) {
      const uint32_t a = bar0 + 8u * (uint32_t)(q % NIN), par = (uint32_t)((q / NIN) & 1);
      asm volatile(
          "{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          " @!P1 bra W_%=;\n}\n" ::"r"(a),
          "r"(par)
          : "memory");
    }
  };
  if (tid == 0)
    for (int q = 0; q < NIN; ++q) issue(q);

  // All shared-memory accesses below index one array with 32-bit offsets.
  T* const S = reinterpret_cast<T*>(sm);
  constexpr int FRING = NIN * IN_BYTES / ES, DRING = FRING + 4 * 4 * EN;
  auto so = [&](int q) { return (q % NIN) * (IN_BYTES / ES); };  // S0 stage offset

  // ---- per-thread widened cells ---------------------------------------------
  // s1_fields: thread t owns e = t + 1 and, for t < R2, e = t + 1 + NT.
  // s1_div: e = EN - 1 - t and, for t >= NT - R2, e = NT - t. (32x8: R2 = 128,
  // warps 0-3 / 4-7.) The corner e = 0 (x = i0-2, y = j0-2) is never read.
  // f_ia: index into the S0 boxes; f_bt: scale-table rows rc | rx << 3 |
  // ry << 6 (x/y bits), parity << 9, owned << 10, x pin << 11, y pin << 12.
  // d_q: DIVERGENCE operand cell (wall mirror applied), d_ok: bit r set when
  // div cell r is a source (x >= i0-1, y >= j0-1).
  const bool has2f = tid < R2, has2d = tid >= NT - R2;
  int f_e[NE], f_ia[NE], f_bt[NE], d_e[NE], d_q[NE], d_ok = 0;
#pragma unroll
  for (int r = 0; r < NE; ++r) {
    {
      const int e = r == 0 ? tid + 1 : (has2f ? tid + 1 + NT : EN - 1);
      const int ex = e % EW, ey = e / EW;
      const int x = i0 - 2 + ex, y = j0 - 2 + ey;
      const long long gi = B.lo[0] + x, gj = B.lo[1] + y;
      const int bx = bin(s.per[0], gi, nm0), bxp = bnx(s.per[0], gi, nm0);
      const int by = bin(s.per[1], gj, nm1), byp = bnx(s.per[1], gj, nm1);
      f_e[r] = e;
      const int ix = ex + XSH - xsh;
      f_ia[r] = ey * IW + (ix < 0 ? 0 : ix > IW - 1 ? IW - 1 : ix);
      f_bt[r] = ((bx << 2) | (by << 1)) | (((bxp << 2) | (by << 1)) << 3) | (((bx << 2) | (byp << 1)) << 6) |
                ((int)((wrp((int)gi, N0, per0) + wrp((int)gj, N1, per1)) & 1) << 9) |
                (((per0 || (gi >= 0 && gi < N0)) && (per1 || (gj >= 0 && gj < N1))) << 10) |
                ((!per0 && gi == N0 - 1) << 11) | ((!per1 && gj == N1 - 1) << 12) | ((!per0 && gi == -1) << 13) |
                ((!per1 && gj == -1) << 14);
    }
    {
      const int e = r == 0 ? EN - 1 - tid : (has2d ? NT - tid : EN - 1);
      const int ex = e % EW, ey = e / EW;
      const int x = i0 - 2 + ex, y = j0 - 2 + ey;
      // the +x / +y ghost (x = n0, y = n1) takes the wall mirror of the last
      // owned cell (exchange.hpp:438-449), evaluated with that cell's operands
      int dx = ex, dy = ey;
      if (!per0 && lo0 + x >= N0) dx -= lo0 + x - (N0 - 1);
      if (!per1 && lo1 + y >= N1) dy -= lo1 + y - (N1 - 1);
      d_e[r] = e;
      d_q[r] = dy * EW + dx;
      if (ex >= 1 && ey >= 1 && (r == 0 || has2d)) d_ok |= 1 << r;
    }
  }
  // Interior tile: every widened cell has all x/y scale bits 1 (so each
  // -(beta*bscale) is -(beta*1.0) = smb[7]), is owned and unpinned, and needs
  // no divu mirror; planes with z in [zf_lo, zf_hi] add the same for z. The
  // fast paths evaluate the identical IEEE operations in the identical order,
  // so they are bitwise the general paths restricted to such cells.
  // (the tile must also lie wholly inside the block: the fast path has no
  // per-thread guard)
  const bool fast_xy = B.lo[0] + i0 - 2 >= 1 && B.lo[0] + i0 + TX <= nm0 - 2 && B.lo[1] + j0 - 2 >= 1 &&
                       B.lo[1] + j0 + TY <= nm1 - 2 && !s.per[0] && !s.per[1] && i0 + TX <= (int)wk.hi[0] &&
                       j0 + TY <= (int)wk.hi[1];
  const int zf_lo = s.per[2] ? 1 << 30 : (int)max(1ll, 1ll - B.lo[2]);
  const int zf_hi = (int)(nm2 - 2 - B.lo[2]);
  const T mbI = smb[7];

  // S1 fields of plane z from its S0 stage (st) and divu0 of plane z+1 (stn):
  // sweep A's cell update (cfd.hpp:699-719) with the wall pins, into field
  // slot fo. Cells outside the domain carry S0; their wall-normal values are
  // the constant pins.
  auto s1_fields = [&](int z, int st, int stn, int fo) {
    const int Di = st + IN_D / ES, Ui = st + IN_U / ES, Vi = st + IN_V / ES, Wi = st + IN_W / ES,
              Pi = st + IN_P / ES, Dz = stn + IN_D / ES;
    const int u1 = fo + U1 * EN, v1 = fo + V1 * EN, w1 = fo + W1 * EN, p1 = fo + P1 * EN;
    const int gk = lo2 + z;
    const int zpar = wrp(gk, N2, per2) & 1;
    if (fast_xy && z >= zf_lo && z <= zf_hi) {
      // both rounds' loads are issued before either round's stores (the
      // compiler cannot reorder them itself: one shared array), doubling the
      // independent work in flight for the warps that own two cells (warps
      // 0-3; the branch is warp-uniform)
      struct ld8 {
        T dc, dx, dy, dz, uu, vv, ww, pp;
      };
      auto load = [&](int r) {
        const int ia = f_ia[r];
        return ld8{S[Di + ia], S[Di + ia + 1], S[Di + ia + IW], S[Dz + ia],
                   S[Ui + ia], S[Vi + ia],     S[Wi + ia],      S[Pi + ia]};
      };
      auto update = [&](int r, const ld8& L) {
        const int e = f_e[r];
        const T a0 = ((((f_bt[r] >> 9) & 1) ^ zpar) == colA) ? 1.0 : 0.0, a1 = 1.0 - a0;
        const T d0 = mbI * L.dc * a0;
        const T exv = mbI * L.dx * a1;
        const T eyv = mbI * L.dy * a1;
        const T ezv = mbI * L.dz * a1;
        S[p1 + e] = L.pp + d0;
        S[u1 + e] = L.uu + cu * (d0 - exv);
        S[v1 + e] = L.vv + cv * (d0 - eyv);
        S[w1 + e] = L.ww + cw * (d0 - ezv);
      };
      if (has2f) {
        const ld8 L0 = load(0), L1 = load(1);
        update(0, L0);
        update(1, L1);
      } else {
        update(0, load(0));
      }
      return;
    }
    if (z >= zf_lo && z <= zf_hi) {
      // boundary tile, interior plane (bz = bzp = 1): every cell evaluates the
      // update and selects apply the wall cases, so no warp runs both sides of
      // a branch (owned cells: bitwise the general path below)
#pragma unroll
      for (int r = 0; r < NE; ++r) {
        if (r > 0 && !has2f) break;
        const int ia = f_ia[r], e = f_e[r], bt = f_bt[r];
        const T dc = S[Di + ia], dx = S[Di + ia + 1], dy = S[Di + ia + IW], dz = S[Dz + ia];
        const T uu = S[Ui + ia], vv = S[Vi + ia], ww = S[Wi + ia], pp = S[Pi + ia];
        const int rc = (bt & 7) | 1, rx = ((bt >> 3) & 7) | 1, ry = ((bt >> 6) & 7) | 1;
        const T a0 = ((((bt >> 9) & 1) ^ zpar) == colA) ? 1.0 : 0.0, a1 = 1.0 - a0;
        const T d0 = smb[rc] * dc * a0;
        const T exv = smb[rx] * dx * a1;
        const T eyv = smb[ry] * dy * a1;
        const T ezv = smb[rc] * dz * a1;
        const bool own = (bt >> 10) & 1;
        const T un = ((bt >> 11) & 1) ? pin_u : uu + cu * (d0 - exv);
        const T vn = ((bt >> 12) & 1) ? pin_v : vv + cv * (d0 - eyv);
        S[p1 + e] = own ? pp + d0 : pp;
        S[u1 + e] = own ? un : (((bt >> 13) & 1) ? pins.ul : uu);
        S[v1 + e] = own ? vn : (((bt >> 14) & 1) ? pins.vl : vv);
        S[w1 + e] = own ? ww + cw * (d0 - ezv) : ww;
      }
      return;
    }
    const bool zin = per2 || (gk >= 0 && gk < N2);
    const int bz = s.per[2] | ((gk > 0) & (gk < (int)nm2)), bzp = s.per[2] | (gk + 1 < (int)nm2);
    const bool pz = !per2 && lo2 + z == N2 - 1, zlow = !per2 && lo2 + z == -1;
#pragma unroll
    for (int r = 0; r < NE; ++r) {
      if (r > 0 && !has2f) break;
      const int e = f_e[r], ia = f_ia[r], bt = f_bt[r];
      if (!(zin && ((bt >> 10) & 1))) {
        // outside the domain: the low-wall normals are the pins (a ghost
        // corner next to a processor face may hold an older copy); the rest
        // is carried over and never read
        S[u1 + e] = ((bt >> 13) & 1) ? pins.ul : S[Ui + ia];
        S[v1 + e] = ((bt >> 14) & 1) ? pins.vl : S[Vi + ia];
        S[w1 + e] = zlow ? pins.wl : S[Wi + ia];
        S[p1 + e] = S[Pi + ia];
        continue;
      }
      const int rc = bt & 7, rx = (bt >> 3) & 7, ry = (bt >> 6) & 7;
      const T a0 = ((((bt >> 9) & 1) ^ zpar) == colA) ? 1.0 : 0.0, a1 = 1.0 - a0;
      const T d0 = smb[rc | bz] * S[Di + ia] * a0;
      const T exv = smb[rx | bz] * S[Di + ia + 1] * a1;
      const T eyv = smb[ry | bz] * S[Di + ia + IW] * a1;
      const T ezv = smb[rc | bzp] * S[Dz + ia] * a1;
      S[p1 + e] = S[Pi + ia] + d0;
      S[u1 + e] = ((bt >> 11) & 1) ? pin_u : S[Ui + ia] + cu * (d0 - exv);
      S[v1 + e] = ((bt >> 12) & 1) ? pin_v : S[Vi + ia] + cv * (d0 - eyv);
      S[w1 + e] = pz ? pin_w : S[Wi + ia] + cw * (d0 - ezv);
    }
  };
  // DIVERGENCE of S1 on plane z (cfd.hpp:605-608) from field slots fo (z) and
  // fom (z-1) into divu1 slot d1; the ghost plane above a top wall mirrors
  // plane N2-1 (dm).
  auto s1_div = [&](int z, int fo, int fom, int d1, int dm) {
    if (!per2 && lo2 + z >= N2) {
#pragma unroll
      for (int r = 0; r < NE; ++r) {
        if (r > 0 && !has2d) break;
        S[d1 + d_e[r]] = S[dm + d_e[r]];
      }
      return;
    }
    const int u1 = fo + U1 * EN, v1 = fo + V1 * EN, w1 = fo + W1 * EN, w1m = fom + W1 * EN;
    // non-source cells compute on in-bounds operands and skip the store; both
    // rounds' loads precede the stores (see s1_fields)
    struct ld6 {
      T u, um, v, vm, w, wm;
    };
    auto load = [&](int r) {
      const int q = d_q[r];
      return ld6{S[u1 + q], S[u1 + q - 1], S[v1 + q], S[v1 + q - EW], S[w1 + q], S[w1m + q]};
    };
    auto div = [&](int r, const ld6& L) {
      const T du = L.u - L.um;
      const T dv = L.v - L.vm;
      const T dw = L.w - L.wm;
      T dd = du * Tix;
      dd += dv * Tiy;
      dd += dw * Tiz;
      if ((d_ok >> r) & 1) S[d1 + d_e[r]] = dd;
    };
    if (has2d) {
      const ld6 L0 = load(0), L1 = load(1);
      div(0, L0);
      div(1, L1);
    } else {
      div(0, load(0));
    }
  };
  auto F = [&](int slot) { return FRING + slot * 4 * EN; };  // field slot offset
  auto Dr = [&](int slot) { return DRING + slot * EN; };     // divu1 slot offset

  // ---- this thread's tile cell ----------------------------------------------
  const int i = i0 + tx, j = j0 + ty;
  const bool act = i < (int)wk.hi[0] && j < (int)wk.hi[1];
  const int gi = lo0 + i, gj = lo1 + j;  // global indices fit in int
  const int bx = bin(s.per[0], gi, nm0), bxp = bnx(s.per[0], gi, nm0);
  const int by = bin(s.per[1], gj, nm1), byp = bnx(s.per[1], gj, nm1);
  const int bxm = bin(s.per[0], gi - 1, nm0), bxpm = bnx(s.per[0], gi - 1, nm0);
  const int bym = bin(s.per[1], gj - 1, nm1), bypm = bnx(s.per[1], gj - 1, nm1);
  const int ic = (bx << 2) | (by << 1), iex = (bxp << 2) | (by << 1), iey = (bx << 2) | (byp << 1);
  const int ixm = (bxm << 2) | (by << 1), ixpm = (bxpm << 2) | (by << 1);
  const int iym = (bx << 2) | (bym << 1), iypm = (bx << 2) | (bypm << 1);
  const int par_col = (gi + gj) & 1;
  const int N2m1 = per2 ? -1 : N2 - 1, nm2i = (int)nm2;  // no pinned top plane on a periodic z
  // Boundary tiles on interior planes (bz = bzp = 1): this cell's scale
  // factors and wall flags are per-thread constants, so sweep B runs the fast
  // path's operations with them instead of the general path's lookups and
  // branches (bitwise the same values).
  const T sc_ = smb[ic | 1], sex_ = smb[iex | 1], sey_ = smb[iey | 1];
  const T sxm_ = smb[ixm | 1], sxpm_ = smb[ixpm | 1], sym_ = smb[iym | 1], sypm_ = smb[iypm | 1];
  const bool xlo = !per0 && gi == 0, ylo = !per1 && gj == 0, xhi = !per0 && gi == N0 - 1, yhi = !per1 && gj == N1 - 1;
  // -x / -y neighbour parities (the complement of this cell's, except across
  // an odd periodic wrap)
  const bool xm_same = per0 && gi == 0 && (N0 & 1), ym_same = per1 && gj == 0 && (N1 & 1);
  const int q0 = (ty + 2) * EW + (tx + 2);

  T* __restrict__ Dn = reinterpret_cast<T*>(tab->ptr[b][SF_DIVU][ALT]);
  T* __restrict__ Pn = reinterpret_cast<T*>(tab->ptr[b][SF_P][ALT]);
  T* __restrict__ Un = reinterpret_cast<T*>(tab->ptr[b][SF_VX][ALT]);
  T* __restrict__ Vn = reinterpret_cast<T*>(tab->ptr[b][SF_VY][ALT]);
  T* __restrict__ Wn = reinterpret_cast<T*>(tab->ptr[b][SF_VZ][ALT]);
  // fused exchange: this cell's class along x / y (-1 low layers, +1 high
  // layers, 0 neither) and the physical buffers the outputs land in
  int rcx = 0, rcy = 0, rg = 0, rphys = 0;
  const sweep2_remote* __restrict__ R = REMOTE ? rem + b : nullptr;  // this component's table
  if (REMOTE) {
    rg = R->g;
    rcx = i < rg ? -1 : (i >= n0 - rg ? 1 : 0);
    rcy = j < rg ? -1 : (j >= n1 - rg ? 1 : 0);
    rphys = tab->bidx[b][SF_VX][ALT] | (tab->bidx[b][SF_VY][ALT] << 2) | (tab->bidx[b][SF_VZ][ALT] << 4) |
            (tab->bidx[b][SF_DIVU][ALT] << 6);
  }
  auto remote_store = [&](int z, T un, T vn, T wn, T dd) {
    const int rcz = z < rg ? -1 : (z >= n2 - rg ? 1 : 0);
    if (!(rcx | rcy | rcz)) return;
    for (int ez = 0; ez < 2; ++ez)
      for (int ey = 0; ey < 2; ++ey)
        for (int ex = 0; ex < 2; ++ex) {
          const int dx = ex ? rcx : 0, dy = ey ? rcy : 0, dz = ez ? rcz : 0;
          if ((ex && !rcx) || (ey && !rcy) || (ez && !rcz) || !(dx | dy | dz)) continue;
          const int q = R->idx[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)];
          if (q < 0) continue;
          const sweep2_peer& P = R->peer[q];
          const long long ro =
              P.rbase + ((z + P.shift[2]) * P.rsy + (j + P.shift[1])) * P.rsx + (i + P.shift[0]);
          __stwb(reinterpret_cast<T*>(P.ptr[0][rphys & 3]) + ro, un);
          __stwb(reinterpret_cast<T*>(P.ptr[1][(rphys >> 2) & 3]) + ro, vn);
          __stwb(reinterpret_cast<T*>(P.ptr[2][(rphys >> 4) & 3]) + ro, wn);
          __stwb(reinterpret_cast<T*>(P.ptr[3][(rphys >> 6) & 3]) + ro, dd);
        }
  };
  unsigned long long r1 = 0ull, r2 = 0ull;
  T wm2 = 0.0;  // swept w2 of the -z neighbour (marching register)
  unsigned o = (unsigned)(B.base + ((long long)k0 * B.sy + j) * B.sx + i);

  // pre-phase: S1 fields of planes 0 and 1 (S0 planes 0..2)
  wait_in(0);
  wait_in(1);
  wait_in(2);
  s1_fields(k0 - 2, so(0), so(1), F(0));
  s1_fields(k0 - 1, so(1), so(2), F(1));
  __syncthreads();
  if (tid == 0) {  // S0 planes 0 and 1 are consumed
    issue(NIN);
    issue(NIN + 1);
  }

  // S1 plane m: fields in slot m & 3, divu1 in slot m % 3 (dsu = u % 3).
  // S0 planes u+2 and u+3 sit in stages st2 and st3 (carried, not divided:
  // the ring indices are uniform per CTA and cost nothing per cell)
  int dsu = 0, st2 = 2 % NIN, st3 = 3 % NIN;
  uint32_t ph3 = (uint32_t)((3 / NIN) & 1);
  for (int u = 0; u <= nplanes + 1; ++u) {
    const int dsu1 = dsu == 2 ? 0 : dsu + 1;
    if (u + 3 < nin) {
      const uint32_t a = bar0 + 8u * (uint32_t)st3;
      asm volatile(
          "{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          " @!P1 bra W_%=;\n}\n" ::"r"(a),
          "r"(ph3)
          : "memory");
    }
    if (u <= nplanes) s1_fields(k0 + u, st2 * (IN_BYTES / ES), st3 * (IN_BYTES / ES), F((u + 2) & 3));
    s1_div(k0 + u - 1, F((u + 1) & 3), F(u & 3), Dr(dsu1), Dr(dsu));
    __syncthreads();
    if (tid == 0) issue(u + 2 + NIN);  // S0 plane u+2 is consumed
    st2 = st3;
    st3 = st3 + 1 == NIN ? 0 : st3 + 1;
    ph3 ^= st3 == 0 ? 1u : 0u;
    if (u == 1 && act) {
      // swept w2 of the plane below the chunk: sweep B's -z neighbour at k0
      const T w1_below = S[F(1) + W1 * EN + q0];
      if (lo2 + k0 > 0 || per2) {
        const long long gkm = B.lo[2] + k0 - 1;
        const int bzm = bin(s.per[2], gkm, nm2), bzpm = bnx(s.per[2], gkm, nm2);
        const T a0m = (((gi + gj + wrp((int)gkm, N2, per2)) & 1) == colB) ? 1.0 : 0.0, a1m = 1.0 - a0m;
        const T d0m = smb[ic | bzm] * S[Dr(1) + q0] * a0m;
        const T ezm = smb[ic | bzpm] * S[Dr(2) + q0] * a1m;
        wm2 = w1_below + cw * (d0m - ezm);
      } else {
        wm2 = w1_below;  // pinned ghost plane
      }
    }
    if (u >= 2) {
      // sweep B on plane m = u, z = k0 + u - 2
      const int z = k0 + u - 2;
      const T* u1 = S + F(u & 3) + U1 * EN;
      const T* v1 = S + F(u & 3) + V1 * EN;
      const T* w1 = S + F(u & 3) + W1 * EN;
      const T* p1 = S + F(u & 3) + P1 * EN;
      const T* d1 = S + Dr(dsu);
      const T* d1p = S + Dr(dsu1);
      if (fast_xy && z >= zf_lo && z <= zf_hi) {
        // interior plane (see fast_xy): bitwise the general path below
        const T dC = d1[q0], dXp = d1[q0 + 1], dYp = d1[q0 + EW];
        const T dXm = d1[q0 - 1], dYm = d1[q0 - EW], dZp = d1p[q0];
        const T p0 = p1[q0], u0 = u1[q0], uml = u1[q0 - 1], v0 = v1[q0], vml = v1[q0 - EW], w0 = w1[q0];
        const int par = par_col ^ (int)((B.lo[2] + z) & 1);
        const T a0 = (par == colB) ? 1.0 : 0.0, a1 = 1.0 - a0;
        const T d0 = mbI * dC * a0;
        const T exv = mbI * dXp * a1;
        const T eyv = mbI * dYp * a1;
        const T ezv = mbI * dZp * a1;
        const T pn = p0 + d0;
        const T un = u0 + cu * (d0 - exv);
        const T vn = v0 + cv * (d0 - eyv);
        const T wn = w0 + cw * (d0 - ezv);
        // -x / -y neighbours: parity a1, their +x / +y term is mbI*dC*a0 == d0
        const T umn = uml + cu * (mbI * dXm * a1 - d0);
        const T vmn = vml + cv * (mbI * dYm * a1 - d0);
        T dd = (un - umn) * Tix;
        dd += (vn - vmn) * Tiy;
        dd += (wn - wm2) * Tiz;
        __stwb(Pn + o, pn);
        __stwb(Un + o, un);
        __stwb(Vn + o, vn);
        __stwb(Wn + o, wn);
        __stwb(Dn + o, dd);
        if (REMOTE) remote_store(z, un, vn, wn, dd);
        const unsigned long long b1 = abs_bits((double)dC), b2 = abs_bits((double)dd);
        r1 = b1 > r1 ? b1 : r1;
        r2 = b2 > r2 ? b2 : r2;
        wm2 = wn;
      } else if (act && z >= zf_lo && z <= zf_hi && !(per0 | per1)) {
        // boundary tile, interior plane: the general path's arithmetic with
        // per-thread scales, selects for the wall cases (see sc_ above)
        const T dC = d1[q0], dXp = d1[q0 + 1], dYp = d1[q0 + EW];
        const T dXm = d1[q0 - 1], dYm = d1[q0 - EW], dZp = d1p[q0];
        const T p0 = p1[q0], u0 = u1[q0], uml = u1[q0 - 1], v0 = v1[q0], vml = v1[q0 - EW], w0 = w1[q0];
        const int par = par_col ^ ((lo2 + z) & 1);
        const T a0 = (par == colB) ? 1.0 : 0.0, a1 = 1.0 - a0;
        const T d0 = sc_ * dC * a0;
        const T exv = sex_ * dXp * a1;
        const T eyv = sey_ * dYp * a1;
        const T ezv = sc_ * dZp * a1;
        const T pn = p0 + d0;
        T un = u0 + cu * (d0 - exv);
        T vn = v0 + cv * (d0 - eyv);
        const T wn = w0 + cw * (d0 - ezv);
        un = xhi ? pin_u : un;
        vn = yhi ? pin_v : vn;
        // swept -x / -y neighbours (parity a1; 1 - a1 == a0 exactly); at a low
        // wall the pinned ghost
        const T a1m = 1.0 - a1;
        const T umr = uml + cu * (sxm_ * dXm * a1 - sxpm_ * dC * a1m);
        const T vmr = vml + cv * (sym_ * dYm * a1 - sypm_ * dC * a1m);
        const T umn = xlo ? uml : umr, vmn = ylo ? vml : vmr;
        T dd = (un - umn) * Tix;
        dd += (vn - vmn) * Tiy;
        dd += (wn - wm2) * Tiz;
        __stwb(Pn + o, pn);
        __stwb(Un + o, un);
        __stwb(Vn + o, vn);
        __stwb(Wn + o, wn);
        __stwb(Dn + o, dd);
        if (REMOTE) remote_store(z, un, vn, wn, dd);
        if (xlo) {
          Un[o - 1] = umn;
          Dn[o - 1] = dd;
        }
        if (ylo) {
          Vn[o - sx] = vmn;
          Dn[o - sx] = dd;
        }
        if (xhi) Dn[o + 1] = dd;
        if (yhi) Dn[o + sx] = dd;
        const unsigned long long b1 = abs_bits((double)dC), b2 = abs_bits((double)dd);
        r1 = b1 > r1 ? b1 : r1;
        r2 = b2 > r2 ? b2 : r2;
        wm2 = wn;
      } else if (act) {
        const T dZp = d1p[q0];
        const int gk = lo2 + z;
        const int bz = per2 | ((gk > 0) & (gk < nm2i)), bzp = per2 | (gk + 1 < nm2i);
        const T dC = d1[q0], dXp = d1[q0 + 1], dYp = d1[q0 + EW];
        const T dXm = d1[q0 - 1], dYm = d1[q0 - EW];
        const int par = par_col ^ (int)(gk & 1);
        const T a0 = (par == colB) ? 1.0 : 0.0, a1 = 1.0 - a0;
        const T d0 = smb[ic | bz] * dC * a0;
        const T exv = smb[iex | bz] * dXp * a1;
        const T eyv = smb[iey | bz] * dYp * a1;
        const T ezv = smb[ic | bzp] * dZp * a1;
        const T pn = p1[q0] + d0;
        T un = u1[q0] + cu * (d0 - exv);
        T vn = v1[q0] + cv * (d0 - eyv);
        T wn = w1[q0] + cw * (d0 - ezv);
        if (xhi) un = pin_u;
        if (yhi) vn = pin_v;
        if (gk == N2m1) wn = pin_w;
        // swept -x / -y neighbours; at the low wall the pinned ghost (in S1)
        T umn, vmn;
        if (gi > 0 || per0) {
          const T a0m = xm_same ? a0 : a1, a1m = 1.0 - a0m;
          const T d0m = smb[ixm | bz] * dXm * a0m;
          const T exm = smb[ixpm | bz] * dC * a1m;
          umn = u1[q0 - 1] + cu * (d0m - exm);
        } else {
          umn = u1[q0 - 1];
        }
        if (gj > 0 || per1) {
          const T a0m = ym_same ? a0 : a1, a1m = 1.0 - a0m;
          const T d0m = smb[iym | bz] * dYm * a0m;
          const T eym = smb[iypm | bz] * dC * a1m;
          vmn = v1[q0 - EW] + cv * (d0m - eym);
        } else {
          vmn = v1[q0 - EW];
        }
        T dd = (un - umn) * Tix;
        dd += (vn - vmn) * Tiy;
        dd += (wn - wm2) * Tiz;
        __stwb(Pn + o, pn);
        __stwb(Un + o, un);
        __stwb(Vn + o, vn);
        __stwb(Wn + o, wn);
        __stwb(Dn + o, dd);
        if (REMOTE) remote_store(z, un, vn, wn, dd);
        // ghosts the next pass reads: pinned low-face velocities, mirrored divu
        if (xlo) {
          Un[o - 1] = umn;
          Dn[o - 1] = dd;
        }
        if (ylo) {
          Vn[o - sx] = vmn;
          Dn[o - sx] = dd;
        }
        if (!per2 && gk == 0) {
          Wn[o - sxy] = wm2;
          Dn[o - sxy] = dd;
        }
        if (xhi) Dn[o + 1] = dd;
        if (yhi) Dn[o + sx] = dd;
        if (gk == N2m1) Dn[o + sxy] = dd;
        const unsigned long long b1 = abs_bits((double)dC), b2 = abs_bits((double)dd);
        r1 = b1 > r1 ? b1 : r1;
        r2 = b2 > r2 ? b2 : r2;
        wm2 = wn;
      }
      o += sxy;
    }
    dsu = dsu1;
  }

  // stores into peers (other devices or processes) are visible system-wide
  // before this kernel completes; the max-allreduce after it is what the
  // peers wait for
  if (REMOTE) __threadfence_system();
  unsigned long long rr[2] = {r1, r2};
  pass_finalize(rr, tab, ctl, hflag, total_ctas, finalize);
}

// ---------------------------------------------------------------------------
// The interior form of the temporal pass (fp64). Tiles whose widened region
// lies inside the domain on x and y and whose S0 planes k0-2 .. k1+1 are
// interior in z take k_sweep2's fast path everywhere; for them this kernel
// drops the S1 field ring. Each thread keeps its own tile cell's sweep-A
// values (p1, u1, v1, w1 and the -x / -y neighbours' u1, v1) in registers from
// the plane it computes them to the plane sweep B consumes them, and computes
// the neighbours' values it needs from S0 with the same IEEE operations as the
// fast path (the -x neighbour's +x term IS this cell's d0). Shared memory holds
// a 4-stage S0 ring (p only over the tile, u and w one row shorter) and a
// 3-slot divu1 ring over the tile and its 1-cell ring: 65 KB, so 3 CTAs (24
// warps) per SM instead of 2 (16). Bitwise the fast path of k_sweep2.
// Geometry for element type T: the boxes start XA = 16 / sizeof(T) cells
// left of the tile's x (a 16-byte aligned TMA start; 2 fp64, 4 fp32), i.e. the
// cells of a row sit XSH = XA - 2 further in than for fp64.
#ifndef SF_ITY
#define SF_ITY 20
#endif
#ifndef SF_ITY32
#define SF_ITY32 16
#endif
#ifndef SF_ININ
#define SF_ININ 4
#endif
#ifndef SF_ININ32
#define SF_ININ32 6
#endif
// tile height and S0 stages of the interior form per element type. Measured
// at 512^3 (ms per pass, same box): fp64 32x8 (3 CTAs/SM) 2.48, 32x12 (2)
// 2.41, 32x16 (1) 2.31, 32x20 (1) 2.28, 32x24 2.32 (a 24-row slab), 32x32
// (3 stages, spills) 2.49; 32x20 with 3 / 5 stages 2.46 / 2.28. fp32 32x8
// 1.398, 32x12 1.411, 32x16 1.389, 32x8 6 stages 1.378, 32x16 6 stages 1.371.
// Taller tiles re-read fewer halo rows: DRAM reads per interior cell 53.7 B
// at 32x8, 45.5 B at 32x20 (40 B without halos).
template <class T>
constexpr int kInteriorTY = sizeof(T) == 8 ? SF_ITY : SF_ITY32;
int sweep2i_tile_y(int es) { return es == 4 ? kInteriorTY<float> : kInteriorTY<double>; }

template <class T, int TYV = kInteriorTY<T>>
struct ig {
  static constexpr int ES = (int)sizeof(T), XA = 16 / ES, XSH = XA - 2;
  static constexpr int TX = 32, TY = TYV, NT = TX * TY;
  static constexpr int RW = TX + 2, RH = TY + 2, RN = RW * RH;  // divu1 region: x from i0-1, y from j0-1
  static constexpr int R2N = RN - NT;                            // its ring cells (84), one more per thread 0..83
  static constexpr int BW = (TX + 4 + XSH + XA - 1) / XA * XA;   // S0 box width, x from i0-2-XSH: 36 / 40
  static constexpr int DH = TY + 4, UH = TY + 2, VH = TY + 3, WH = TY + 2;  // divu, vx, vy, vz box heights
  static constexpr int O_D = 0, O_U = r128(ES * BW * DH), O_V = O_U + r128(ES * BW * UH);
  static constexpr int O_W = O_V + r128(ES * BW * VH), O_P = O_W + r128(ES * BW * WH);
  static constexpr int ST_BYTES = O_P + r128(ES * TX * TY);
  static constexpr uint32_t ST_TX = (uint32_t)ES * (BW * DH + BW * UH + BW * VH + BW * WH + TX * TY);
  static constexpr int D1_BYTES = r128(ES * RN);
  static constexpr int NIN = ES == 8 ? SF_ININ : SF_ININ32;
  static constexpr int SMEM = NIN * ST_BYTES + 3 * D1_BYTES;
  // CTAs per SM the registers are budgeted for: 768 fp64 threads (<= 85
  // registers each), 1024 fp32 threads (<= 64)
  static constexpr int MINB = (ES == 8 ? 768 : 1024) / NT > 0 ? (ES == 8 ? 768 : 1024) / NT : 1;
};

template <class T>
__global__ void __launch_bounds__(ig<T>::NT, ig<T>::MINB)
    k_sweep2i(sf_dev_table* __restrict__ tab, const sf_work* __restrict__ items, int nitems, int zc, sf_consts s,
              sf_dev_ctl* ctl, sf_host_flag* hflag, unsigned int total_ctas, const maps2_t* __restrict__ maps,
              int finalize) {
  using G = ig<T>;
  constexpr int TX = G::TX, TY = G::TY, RW = G::RW, RH = G::RH, R2N = G::R2N, BW = G::BW, XSH = G::XSH;
  constexpr int O_D = G::O_D, O_U = G::O_U, O_V = G::O_V, O_W = G::O_W, O_P = G::O_P, ES = G::ES;
  constexpr int ST_BYTES = G::ST_BYTES, D1_BYTES = G::D1_BYTES, NIN = G::NIN;
  constexpr uint32_t ST_TX = G::ST_TX;
  if (*reinterpret_cast<const volatile int*>(&ctl->done)) return;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[NIN];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const sf_work& wk = items[nitems > 1 ? find_item(items, nitems, blockIdx.x) : 0];
  const int local = blockIdx.x - wk.cta_begin;
  const int tix = local % wk.tiles[0], tiy = (local / wk.tiles[0]) % wk.tiles[1];
  const int tiz = local / (wk.tiles[0] * wk.tiles[1]);
  const int i0 = (int)wk.lo[0] + tix * TX, j0 = (int)wk.lo[1] + tiy * TY;
  const int k0 = (int)wk.lo[2] + tiz * zc;
  const int k1 = (int)min((long long)k0 + zc, wk.hi[2]);
  const int nplanes = k1 - k0;
  const int b = wk.blk;
  const sf_dev_block& B = tab->blk[b];
  const double beta = ctl->beta, dt = ctl->dt;
  const T Tix = (T)s.ix, Tiy = (T)s.iy, Tiz = (T)s.iz;
  const int colA = ctl->color, colB = colA ^ 1;
  const T cu = (T)(dt * s.ix), cv = (T)(dt * s.iy), cw = (T)(dt * s.iz);
  const T mbI = (T)(-(beta * s.bscale[1][1][1]));  // every scale of an interior cell (cfd.hpp:712-715)
  if (tid == 0) {
    for (int q = 0; q < NIN; ++q) bar_init(&bars[q]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // S0 plane q holds z = k0 - 2 + q (q = 0 .. nplanes + 3)
  const int xo = (int)(B.base % B.sx), g = B.g;
  const int xs = xo + i0 - 2 - XSH, ys = g + j0 - 2, zs = g + k0 - 2;
  const CUtensorMap* mD = &maps->m[b][SF_DIVU][tab->bidx[b][SF_DIVU][FRONT]];
  const CUtensorMap* mU = &maps->m[b][SF_VX][tab->bidx[b][SF_VX][FRONT]];
  const CUtensorMap* mV = &maps->m[b][SF_VY][tab->bidx[b][SF_VY][FRONT]];
  const CUtensorMap* mW = &maps->m[b][SF_VZ][tab->bidx[b][SF_VZ][FRONT]];
  const CUtensorMap* mP = &maps->m[b][SF_P][tab->bidx[b][SF_P][FRONT]];
  const int nin = nplanes + 4;
  auto issue = [&](int q) {
    if (q >= nin) return;
    unsigned char* st = sm + (q % NIN) * ST_BYTES;
    uint64_t* bar = &bars[q % NIN];
    bar_expect(bar, ST_TX);
    tma3(st + O_D, mD, bar, xs, ys, zs + q);
    tma3(st + O_U, mU, bar, xs, ys + 1, zs + q);
    tma3(st + O_V, mV, bar, xs, ys, zs + q);
    tma3(st + O_W, mW, bar, xs, ys + 1, zs + q);
    tma3(st + O_P, mP, bar, xs + 2 + XSH, ys + 2, zs + q);
  };
  const uint32_t bar0 = smem32(&bars[0]);
  auto wait_in = [&](int q) {
    if (q < nin) {
      const uint32_t a = bar0 + 8u * (uint32_t)(q % NIN), par = (uint32_t)((q / NIN) & 1);
      asm volatile(
          "{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          " @!P1 bra W_%=;\n}\n" ::"r"(a),
          "r"(par)
          : "memory");
    }
  };
  if (tid == 0)
    for (int q = 0; q < NIN; ++q) issue(q);

  const T* const S = reinterpret_cast<const T*>(sm);
  T* const D1 = reinterpret_cast<T*>(sm + NIN * ST_BYTES);
  constexpr int SST = ST_BYTES / ES, SD1 = D1_BYTES / ES;

  // the two divu1-region cells of this thread: its tile cell (A) and, for
  // tid < 84, one cell of the region's 1-cell ring (R)
  const int rA = (ty + 1) * RW + (tx + 1);
  const int rR = tid < RW ? tid
                 : tid < 2 * RW ? (RH - 1) * RW + (tid - RW)
                 : tid < 2 * RW + (RH - 2) ? (tid - 2 * RW + 1) * RW
                 : (tid - 2 * RW - (RH - 2) + 1) * RW + (RW - 1);
  const bool hasR = tid < R2N;
  auto dv = [](int r) { return (r / RW + 1) * BW + (r % RW) + 1 + XSH; };  // divu / vy box element (rows from j0-2)
  auto uw = [](int r) { return (r / RW) * BW + (r % RW) + 1 + XSH; };      // vx / vz box element (rows from j0-1)
  const int dA = dv(rA), uA = uw(rA), pA = ty * TX + tx;
  const int dR = dv(rR), uR = uw(rR);
  const int gi = (int)B.lo[0] + i0 + tx, gj = (int)B.lo[1] + j0 + ty;
  const int parA = (gi + gj) & 1;
  const int parR = ((int)B.lo[0] + i0 - 1 + rR % RW + (int)B.lo[1] + j0 - 1 + rR / RW) & 1;
  const int gk0 = (int)B.lo[2] + k0;  // global z of local plane k0

  // sweep A (colour colA, cfd.hpp:699-719) at a region cell on S0 stage st
  // (plane z) with stn (plane z+1): its u1, v1, w1 and the swept -x / -y
  // neighbours' u1, v1 (their parity is the complement; their +x / +y term is
  // this cell's d0, the identical product)
  auto sweepA = [&](int st, int stn, int d, int uo, int par, int zpar, T& u, T& v, T& w,
                    T& um, T& vm, T& d0) {
    const T dc = S[st + O_D / ES + d], dxp = S[st + O_D / ES + d + 1], dyp = S[st + O_D / ES + d + BW];
    const T dzp = S[stn + O_D / ES + d], dxm = S[st + O_D / ES + d - 1], dym = S[st + O_D / ES + d - BW];
    const T uu = S[st + O_U / ES + uo], uum = S[st + O_U / ES + uo - 1];
    const T vv = S[st + O_V / ES + d], vvm = S[st + O_V / ES + d - BW], ww = S[st + O_W / ES + uo];
    const T a0 = ((par ^ zpar) == colA) ? 1.0 : 0.0, a1 = 1.0 - a0;
    d0 = mbI * dc * a0;
    const T exv = mbI * dxp * a1;
    const T eyv = mbI * dyp * a1;
    const T ezv = mbI * dzp * a1;
    u = uu + cu * (d0 - exv);
    v = vv + cv * (d0 - eyv);
    w = ww + cw * (d0 - ezv);
    um = uum + cu * (mbI * dxm * a1 - d0);
    vm = vvm + cv * (mbI * dym * a1 - d0);
  };
  // DIVERGENCE of S1 (cfd.hpp:605-608)
  auto div1 = [&](T u, T um, T v, T vm, T w, T wbelow) {
    T dd = (u - um) * Tix;
    dd += (v - vm) * Tiy;
    dd += (w - wbelow) * Tiz;
    return dd;
  };

  // prologue: w1 of plane k0-2 (for the divergence at k0-1), then plane k0-1
  wait_in(0);
  wait_in(1);
  wait_in(2);
  T cp, cu1, cv1, cw1, cum, cvm;  // this cell's S1 at the plane sweep B handles next
  T wA, wR = 0.0;                 // w1 one plane below (tile cell, ring cell)
  {
    T u, v, um, vm, d0;
    sweepA(0, SST, dA, uA, parA, (gk0 - 2) & 1, u, v, wA, um, vm, d0);
    if (hasR) sweepA(0, SST, dR, uR, parR, (gk0 - 2) & 1, u, v, wR, um, vm, d0);
    T d0A;
    sweepA(SST, 2 * SST, dA, uA, parA, (gk0 - 1) & 1, cu1, cv1, cw1, cum, cvm, d0A);
    cp = S[SST + O_P / ES + pA] + d0A;
    D1[rA] = div1(cu1, cum, cv1, cvm, cw1, wA);
    wA = cw1;
    if (hasR) {
      T w;
      sweepA(SST, 2 * SST, dR, uR, parR, (gk0 - 1) & 1, u, v, w, um, vm, d0);
      D1[rR] = div1(u, um, v, vm, w, wR);
      wR = w;
    }
  }
  __syncthreads();
  if (tid == 0) {  // S0 planes 0 and 1 are consumed
    issue(NIN);
    issue(NIN + 1);
  }

  const int i = i0 + tx, j = j0 + ty;
  T* __restrict__ Dn = reinterpret_cast<T*>(tab->ptr[b][SF_DIVU][ALT]);
  T* __restrict__ Pn = reinterpret_cast<T*>(tab->ptr[b][SF_P][ALT]);
  T* __restrict__ Un = reinterpret_cast<T*>(tab->ptr[b][SF_VX][ALT]);
  T* __restrict__ Vn = reinterpret_cast<T*>(tab->ptr[b][SF_VY][ALT]);
  T* __restrict__ Wn = reinterpret_cast<T*>(tab->ptr[b][SF_VZ][ALT]);
  const unsigned sxy = (unsigned)(B.sx * B.sy);
  unsigned o = (unsigned)(B.base + ((long long)k0 * B.sy + j) * B.sx + i);
  unsigned long long r1 = 0ull, r2 = 0ull;
  T wm2 = 0.0;  // swept w2 of the -z neighbour
  // iteration t: sweep A on plane m+1 = k0+t (S0 planes t+2, t+3) and its
  // divergence into divu1 slot (t+1) % 3; barrier; sweep B on plane m = k0-1+t
  // (divu1 slots t % 3, (t+1) % 3), or at t = 0 the -z neighbour's swept w
  int s0 = 2 % NIN, s1 = 3 % NIN;  // stages of S0 planes t+2, t+3
  int dcur = 0, dnxt = 1;          // divu1 slots of planes m, m+1
  for (int t = 0; t <= nplanes; ++t) {
    wait_in(t + 3);
    const int zp = (gk0 + t) & 1;
    T np, nu1, nv1, nw1, num, nvm;
    {
      T d0A;
      sweepA(s0 * SST, s1 * SST, dA, uA, parA, zp, nu1, nv1, nw1, num, nvm, d0A);
      np = S[s0 * SST + O_P / ES + pA] + d0A;
      D1[dnxt * SD1 + rA] = div1(nu1, num, nv1, nvm, nw1, wA);
      wA = nw1;
      if (hasR) {
        T u, v, w, um, vm, d0;
        sweepA(s0 * SST, s1 * SST, dR, uR, parR, zp, u, v, w, um, vm, d0);
        D1[dnxt * SD1 + rR] = div1(u, um, v, vm, w, wR);
        wR = w;
      }
    }
    __syncthreads();
    if (tid == 0) issue(t + 2 + NIN);  // S0 plane t+2 is consumed
    const T* d1 = D1 + dcur * SD1;
    const T* d1p = D1 + dnxt * SD1;
    if (t == 0) {
      // swept w2 of the plane below the chunk: sweep B's -z neighbour at k0
      const T a0m = (((gi + gj + gk0 - 1) & 1) == colB) ? 1.0 : 0.0, a1m = 1.0 - a0m;
      const T d0m = mbI * d1[rA] * a0m;
      const T ezm = mbI * d1p[rA] * a1m;
      wm2 = cw1 + cw * (d0m - ezm);
    } else {
      // sweep B on plane m = k0 + t - 1 (k_sweep2's interior fast path)
      const T dC = d1[rA], dXp = d1[rA + 1], dYp = d1[rA + RW];
      const T dXm = d1[rA - 1], dYm = d1[rA - RW], dZp = d1p[rA];
      const int par = (parA ^ ((gk0 + t - 1) & 1));
      const T a0 = (par == colB) ? 1.0 : 0.0, a1 = 1.0 - a0;
      const T d0 = mbI * dC * a0;
      const T exv = mbI * dXp * a1;
      const T eyv = mbI * dYp * a1;
      const T ezv = mbI * dZp * a1;
      const T pn = cp + d0;
      const T un = cu1 + cu * (d0 - exv);
      const T vn = cv1 + cv * (d0 - eyv);
      const T wn = cw1 + cw * (d0 - ezv);
      const T umn = cum + cu * (mbI * dXm * a1 - d0);
      const T vmn = cvm + cv * (mbI * dYm * a1 - d0);
      T dd = (un - umn) * Tix;
      dd += (vn - vmn) * Tiy;
      dd += (wn - wm2) * Tiz;
      __stwb(Pn + o, pn);
      __stwb(Un + o, un);
      __stwb(Vn + o, vn);
      __stwb(Wn + o, wn);
      __stwb(Dn + o, dd);
      const unsigned long long b1 = abs_bits((double)dC), b2 = abs_bits((double)dd);
      r1 = b1 > r1 ? b1 : r1;
      r2 = b2 > r2 ? b2 : r2;
      wm2 = wn;
      o += sxy;
    }
    cp = np;
    cu1 = nu1;
    cv1 = nv1;
    cw1 = nw1;
    cum = num;
    cvm = nvm;
    s0 = s1;
    s1 = s1 + 1 == NIN ? 0 : s1 + 1;
    dcur = dnxt;
    dnxt = dnxt == 2 ? 0 : dnxt + 1;
  }
  unsigned long long rr[2] = {r1, r2};
  pass_finalize(rr, tab, ctl, hflag, total_ctas, finalize);
}

template <class T, int MINB, int TXV = kTX, int TYV = kPassTY>
static void launch2(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                    sf_host_flag* hflag, const void* maps, int fin, const sweep2_pins& pins, cudaStream_t st,
                    unsigned total, const sweep2_remote* remote) {
  constexpr int NIN = kPassStages;
  using G = geom<TXV, TYV, T>;
  const bool per = c.per[0] || c.per[1] || c.per[2];
  auto k = remote ? (per ? k_sweep2<TXV, TYV, NIN, MINB, true, true, T> : k_sweep2<TXV, TYV, NIN, MINB, false, true, T>)
                  : (per ? k_sweep2<TXV, TYV, NIN, MINB, true, false, T>
                         : k_sweep2<TXV, TYV, NIN, MINB, false, false, T>);
  ensure_smem_attr((const void*)k, G::smem_bytes(NIN));
  k<<<nctas, dim3(G::TX, G::TY), G::smem_bytes(NIN), st>>>(vw.tab, vw.items, vw.nitems, zc, c, ctl, hflag,
                                                           total ? total : (unsigned)nctas,
                                                           static_cast<const maps2_t*>(maps), fin, pins, remote);
}

template <class G>
static void box2i(int field, int* bw, int* bh) {
  switch (field) {
    case SF_DIVU: *bw = G::BW; *bh = G::DH; break;
    case SF_VX: *bw = G::BW; *bh = G::UH; break;
    case SF_VY: *bw = G::BW; *bh = G::VH; break;
    case SF_VZ: *bw = G::BW; *bh = G::WH; break;
    default: *bw = G::TX; *bh = G::TY; break;
  }
}
void sweep2i_box(int field, int* bw, int* bh, int es) {
  if (es == 4)
    box2i<ig<float>>(field, bw, bh);
  else
    box2i<ig<double>>(field, bw, bh);
}

template <class T>
static void launch2i(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                     sf_host_flag* hflag, const void* maps, int fin, cudaStream_t st, unsigned total) {
  using G = ig<T>;
  ensure_smem_attr((const void*)k_sweep2i<T>, G::SMEM);
  k_sweep2i<T><<<nctas, dim3(G::TX, G::TY), G::SMEM, st>>>(vw.tab, vw.items, vw.nitems, zc, c, ctl, hflag,
                                                           total ? total : (unsigned)nctas,
                                                           static_cast<const maps2_t*>(maps), fin);
}
void launch_sweep2i(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                    sf_host_flag* hflag, const void* maps, int fin, cudaStream_t st, unsigned total, int es) {
  if (nctas <= 0) return;
  if (es == 4)
    launch2i<float>(vw, nctas, zc, c, ctl, hflag, maps, fin, st, total);
  else
    launch2i<double>(vw, nctas, zc, c, ctl, hflag, maps, fin, st, total);
}

void launch_sweep2(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                   sf_host_flag* hflag, const void* maps, int fin, const sweep2_pins& pins, cudaStream_t st,
                   unsigned total, const sweep2_remote* remote, int es, int shape) {
  if (nctas <= 0) return;
  if (shape) {  // the x-slab form (the interior split: no periodic axis)
    if (es == 4)
      launch2<float, kPassMinB32, kSlabTX, kSlabTY>(vw, nctas, zc, c, ctl, hflag, maps, fin, pins, st, total, remote);
    else
      launch2<double, kPassMinB, kSlabTX, kSlabTY>(vw, nctas, zc, c, ctl, hflag, maps, fin, pins, st, total, remote);
    return;
  }
  if (es == 4)  // fp32: half the shared memory per CTA (56 KB), up to 3 CTAs per SM
    launch2<float, kPassMinB32>(vw, nctas, zc, c, ctl, hflag, maps, fin, pins, st, total, remote);
  else
    launch2<double, kPassMinB>(vw, nctas, zc, c, ctl, hflag, maps, fin, pins, st, total, remote);
}

}  // namespace sfb
