// sf_uv_tma.cu -- UPDATE_VELOCITY (cfd.hpp:524-589), TMA-staged for sm_100a.
//
// The plain-load kernel (k_update_vel) reads each velocity value up to 13
// times through L1. Here each CTA (32 x 8 column tile, marching a z chunk)
// streams halo'd z planes into a shared-memory ring with cp.async.bulk.tensor:
//     vx, vy, vz  36 x 10  (x from i0-2: TMA needs an even fp64 x start;
//                           y from j0-1), planes z-1 .. z+1 of each cell
//     p           34 x 9   (x from i0, y from j0), planes z .. z+1
// Every cell is the same uv_point() as the plain kernel (sf_uv.cuh), so the
// result is bitwise identical. SEPARATEINOUT: read FRONT, write BACK; the
// NaN-guard maxima of the new velocities go to ctl->acc[1..3].
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sf_kernels.cuh"
#include "sf_uv.cuh"

namespace sfb {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int rnd128(int b) { return (b + 127) / 128 * 128; }
constexpr int NST = 4;  // ring: planes z-1, z, z+1 in use, one in flight
// Stage layout for element type T (8: fp64, 4: fp32). A TMA box starts on a
// 16-byte aligned x and spans a 16-byte multiple: the velocity boxes start
// XL = 16 / sizeof(T) cells left of the tile (2 fp64, 4 fp32).
template <class T>
struct uvg {
  static constexpr int ES = (int)sizeof(T), XL = 16 / ES;
  static constexpr int VW = TX + 2 * XL, VH = TY + 2;            // velocity boxes
  static constexpr int PW = (TX + 1 + XL - 1) / XL * XL, PH = TY + 1;  // pressure box (x from i0)
  static constexpr int ST_U = 0;
  static constexpr int ST_V = rnd128(ES * VW * VH);
  static constexpr int ST_W = ST_V + rnd128(ES * VW * VH);
  static constexpr int ST_P = ST_W + rnd128(ES * VW * VH);
  static constexpr int ST_BYTES = ST_P + rnd128(ES * PW * PH);
  static constexpr uint32_t ST_TX = (uint32_t)ES * (3 * VW * VH + PW * PH);
};

struct uvmaps_t {  // [block][field vx vy vz p][physical buffer]
  CUtensorMap m[kMaxBlocks][4][kSlots];
};

}  // namespace

size_t uv_maps_bytes() { return sizeof(uvmaps_t); }
size_t uv_map_offset(int b, int f, int s) { return sizeof(CUtensorMap) * (((size_t)b * 4 + f) * kSlots + s); }
void uv_box(int field, int* bw, int* bh, int es) {
  if (es == 4) {
    *bw = field == SF_P ? uvg<float>::PW : uvg<float>::VW;
    *bh = field == SF_P ? uvg<float>::PH : uvg<float>::VH;
  } else {
    *bw = field == SF_P ? uvg<double>::PW : uvg<double>::VW;
    *bh = field == SF_P ? uvg<double>::PH : uvg<double>::VH;
  }
}

template <class T, bool BLEND>
__global__ void __launch_bounds__(NT, 2)
    k_update_vel_tma(sf_dev_table* __restrict__ tab, const sf_work* __restrict__ items, int nitems, int zc,
                     sf_consts s, sf_dev_ctl* ctl, const uvmaps_t* __restrict__ maps) {
  using G = uvg<T>;
  constexpr int VW = G::VW, PW = G::PW, ST_U = G::ST_U, ST_V = G::ST_V, ST_W = G::ST_W, ST_P = G::ST_P;
  constexpr int ST_BYTES = G::ST_BYTES, XL = G::XL;
  constexpr uint32_t ST_TX = G::ST_TX;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[NST];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int cta = blockIdx.x;
  const sf_work& wk = items[nitems > 1 ? find_item(items, nitems, cta) : 0];
  const int b = wk.blk;
  const int local = cta - wk.cta_begin;
  const int tix = local % wk.tiles[0], tiy = (local / wk.tiles[0]) % wk.tiles[1];
  const int tiz = local / (wk.tiles[0] * wk.tiles[1]);
  const int i0 = (int)wk.lo[0] + tix * TX, j0 = (int)wk.lo[1] + tiy * TY;
  const int k0 = (int)wk.lo[2] + tiz * zc;
  const int k1 = (int)min((long long)k0 + zc, wk.hi[2]);
  const int nplanes = k1 - k0;
  const sf_dev_block& B = tab->blk[b];
  const T dt = (T)ctl->dt;
  const uv_consts<T> uc(s);

  if (tid == 0) {
    for (int q = 0; q < NST; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // planes q = 0 .. nplanes+1 hold z = k0-1+q
  const int xo = (int)(B.base % B.sx), g = B.g;
  const int zs = g + k0 - 1;
  const CUtensorMap* mU = &maps->m[b][0][tab->bidx[b][SF_VX][FRONT]];
  const CUtensorMap* mV = &maps->m[b][1][tab->bidx[b][SF_VY][FRONT]];
  const CUtensorMap* mW = &maps->m[b][2][tab->bidx[b][SF_VZ][FRONT]];
  const CUtensorMap* mP = &maps->m[b][3][tab->bidx[b][SF_P][FRONT]];
  const int nq = nplanes + 2;
  auto tma = [&](unsigned char* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_addr(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
  };
  auto issue = [&](int q) {
    if (q >= nq) return;
    unsigned char* st = sm + (q % NST) * ST_BYTES;
    uint64_t* bar = &bars[q % NST];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(ST_TX)
                 : "memory");
    tma(st + ST_U, mU, bar, xo + i0 - XL, g + j0 - 1, zs + q);
    tma(st + ST_V, mV, bar, xo + i0 - XL, g + j0 - 1, zs + q);
    tma(st + ST_W, mW, bar, xo + i0 - XL, g + j0 - 1, zs + q);
    tma(st + ST_P, mP, bar, xo + i0, g + j0, zs + q);
  };
  auto wait = [&](int q) {
    if (q >= nq) return;
    asm volatile(
        "{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra W_%=;\n}\n" ::"r"(smem_addr(&bars[q % NST])),
        "r"((uint32_t)((q / NST) & 1))
        : "memory");
  };
  if (tid == 0)
    for (int q = 0; q < NST; ++q) issue(q);

  const int i = i0 + tx, j = j0 + ty;
  const bool act = i < (int)wk.hi[0] && j < (int)wk.hi[1];
  T* __restrict__ Uo = reinterpret_cast<T*>(tab->ptr[b][SF_VX][BACK]);
  T* __restrict__ Vo = reinterpret_cast<T*>(tab->ptr[b][SF_VY][BACK]);
  T* __restrict__ Wo = reinterpret_cast<T*>(tab->ptr[b][SF_VZ][BACK]);
  long long o = B.base + ((long long)k0 * B.sy + j) * B.sx + i;
  unsigned long long mx[3] = {0ull, 0ull, 0ull};
  const int cv = (ty + 1) * VW + (tx + XL), cp = ty * PW + tx;  // this cell in the boxes

  // smem accessor over the three planes around z (stage of plane q = kk + 1 + c)
  struct acc {
    const T* vel[3][3];  // [field][dz + 1]
    const T* pr[2];      // [dz]
    int cv, cp;
    __device__ __forceinline__ T u(int a, int b, int c) const { return vel[0][c + 1][cv + b * VW + a]; }
    __device__ __forceinline__ T v(int a, int b, int c) const { return vel[1][c + 1][cv + b * VW + a]; }
    __device__ __forceinline__ T w(int a, int b, int c) const { return vel[2][c + 1][cv + b * VW + a]; }
    __device__ __forceinline__ T q(int a, int b, int c) const { return pr[c][cp + b * PW + a]; }
  };

  wait(0);
  for (int kk = 0; kk < nplanes; ++kk, o += B.sx * B.sy) {
    wait(kk + 1);
    wait(kk + 2);
    if (act) {
      acc A;
      A.cv = cv;
      A.cp = cp;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned char* st = sm + ((kk + c) % NST) * ST_BYTES;
        A.vel[0][c] = reinterpret_cast<const T*>(st + ST_U);
        A.vel[1][c] = reinterpret_cast<const T*>(st + ST_V);
        A.vel[2][c] = reinterpret_cast<const T*>(st + ST_W);
        if (c > 0) A.pr[c - 1] = reinterpret_cast<const T*>(st + ST_P);
      }
      T r[3];
      uv_point<acc, BLEND, T>(A, uc, dt, r);
      Uo[o] = r[0];
      Vo[o] = r[1];
      Wo[o] = r[2];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const unsigned long long bb = abs_bits((double)r[a]);  // fp32 widens exactly
        mx[a] = bb > mx[a] ? bb : mx[a];
      }
    }
    __syncthreads();  // plane kk (z-1 of this cell) left every window
    if (tid == 0) issue(kk + NST);
  }
  block_max_atomic<3>(mx, &ctl->acc[1]);
}

template <class T>
static void launch_uv_tma(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                          const void* maps, cudaStream_t st) {
  // alpha == 0 (either sign): the blend terms are only evaluated on zero fluxes (sf_uv.cuh)
  auto k = c.alpha == 0.0 ? k_update_vel_tma<T, false> : k_update_vel_tma<T, true>;
  const int smem = NST * uvg<T>::ST_BYTES;
  ensure_smem_attr((const void*)k, smem);
  k<<<nctas, dim3(TX, TY), smem, st>>>(vw.tab, vw.items, vw.nitems, zc, c, ctl, static_cast<const uvmaps_t*>(maps));
}
void launch_update_velocity_tma(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                                const void* maps, cudaStream_t st, int es) {
  if (nctas <= 0) return;
  if (es == 4)
    launch_uv_tma<float>(vw, nctas, zc, c, ctl, maps, st);
  else
    launch_uv_tma<double>(vw, nctas, zc, c, ctl, maps, st);
}

}  // namespace sfb
