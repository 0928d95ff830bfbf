// sf_device.cuh -- device-side data model of the B200 stencil path.
//
// Field storage mirrors distributed_field::local_block (field.hpp:31-52):
// one padded array per (worker block, field), x fastest, ghost shell of width
// g, but with an explicit 128-byte-aligned row pitch:
//     offset(i,j,k) = base + (k*sy + j)*sx + i,   i,j,k in [-g, dims+g)
// (sf_layout in include/sforge_b200.h).  Every kernel that runs inside the
// device-driven pressure loop resolves its arrays through a device-resident
// pointer table (sf_dev_table) so buffer swaps -- SEPARATEINOUT front/back
// (executor.hpp:772-773) and the half-sweep ping-pong -- happen on the device
// without the host knowing how many sweeps ran.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sforge_b200.h"

namespace sfb {

constexpr int kMaxBlocks = 64;   // grid components per device
constexpr int kMaxFields = 16;   // vx, vy, vz, p, divu + user fields
constexpr int kSlots = 3;        // front, back, alt

enum slot { FRONT = 0, BACK = 1, ALT = 2 };

// What lies across one face of a block (2*axis + side).
enum face_kind : int {
  FACE_PROC = 0,   // another block (or this block through a periodic wrap)
  FACE_WALL = 1,   // physical, face_bc::wall
  FACE_SYM = 2,    // physical, face_bc::symmetry
  FACE_OUT = 3,    // physical, face_bc::outflow
  FACE_SELF = 4,   // periodic wrap onto this same block (grid.hpp:76-79)
};

struct sf_dev_block {
  long long n[3];    // owned dims
  long long lo[3];   // global coordinates of local (0,0,0)
  long long sx, sy, sz, base;
  int g;
  int face[6];       // face_kind per face
  double fvel[6][3]; // wall velocity per face (exchange.hpp:21)
  long long nb_ghost_gidx[6];  // global index (along the face axis) of the cell behind ghost -1 / n
};

struct sf_dev_table {
  int nblocks;
  sf_dev_block blk[kMaxBlocks];
  double* ptr[kMaxBlocks][kMaxFields][kSlots];
  // physical buffer (0..2) occupying each slot: selects the TMA descriptor
  unsigned char bidx[kMaxBlocks][kMaxFields][kSlots];
  // bytes per value of each field: 8 (fp64; every CFD field) or 4 (fp32 user
  // fields). An fp32 field uses the block's padded layout in elements.
  unsigned char esize[kMaxFields];
};

// Device control block of the pressure loop.  acc[] are max accumulators on
// the IEEE bit patterns of |x| (non-negative doubles order like their bits;
// NaN > inf keeps NaN sticky, reductions.hpp:39-71).
struct sf_dev_ctl {
  unsigned long long acc[8];
  unsigned int ctas_done;
  int done;          // pressure-loop predicate: 1 = stop
  int sweeps;
  int max_sweeps;
  int color;         // red-black colour carried across sweeps and steps (cfd.hpp:299)
  int abort_field;   // -1, or first non-finite velocity after UPDATE_VELOCITY
  int redo;          // temporal pass stopped after its first sweep: redo it single
  double dt, beta, tolerance, residual;
  double vmax[3];
  unsigned long long racc[3];  // persistent loop: residual maxima, rotating per half-sweep
  unsigned int bar;            // persistent loop: grid barrier arrivals
};

// Host-mapped mirror the finalising CTA writes for the polling host.
struct sf_host_flag {
  volatile int done;
  volatile int sweeps;
  volatile double residual;
  volatile double dt;
  volatile int abort_field;
  volatile int color;
};

// One unit of kernel work: a box of one block, tiled by the launching kernel.
struct sf_work {
  int blk;
  int cta_begin;        // first flattened CTA index of this item
  int tiles[3];
  long long lo[3], hi[3];
};

// Kernel-side access to blocks, arrays and work items.  table_view resolves
// through the device table (driver path, swaps happen on the device);
// direct_view carries one block's pointers by value (level-2 C ABI launches).
struct table_view {
  sf_dev_table* tab;
  const sf_work* items;
  int nitems;
  __device__ __forceinline__ const sf_dev_block& blk(int b) const { return tab->blk[b]; }
  __device__ __forceinline__ double* ptr(int b, int f, int s) const { return tab->ptr[b][f][s]; }
  __device__ __forceinline__ const sf_work* work() const { return items; }
  __device__ __forceinline__ int esize(int f) const { return tab->esize[f]; }
  __device__ __forceinline__ int phys(int b, int f, int s) const { return tab->bidx[b][f][s]; }
};

constexpr int kDirectItems = 8;
struct direct_view {
  sf_dev_block b0;
  double* p[kMaxFields][kSlots];
  sf_work it[kDirectItems];
  int nitems;
  __device__ __forceinline__ const sf_dev_block& blk(int) const { return b0; }
  __device__ __forceinline__ double* ptr(int, int f, int s) const { return p[f][s]; }
  __device__ __forceinline__ const sf_work* work() const { return it; }
  __device__ __forceinline__ int esize(int) const { return 8; }
  __device__ __forceinline__ int phys(int, int, int s) const { return s; }
};

// Global (all-block) constants of the CFD kernels: step_constants
// (cfd.hpp:473-487) minus dt, which lives in sf_dev_ctl.
struct sf_consts {
  double nu, alpha, fx, fy, fz, ix, iy, iz, ix2, iy2, iz2;
  double bscale[2][2][2];
  long long nm1[3];
  long long N[3];
  int per[3];
  double spacing[3];
  double sigma, omega, tolerance;
  int max_sweeps;
};

__device__ __forceinline__ long long off(const sf_dev_block& b, long long i, long long j, long long k) {
  return b.base + (k * b.sy + j) * b.sx + i;
}

__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7fffffffffffffffull;
}

__device__ __forceinline__ double bits_to_max(unsigned long long b) {
  // canonical quiet NaN like std::numeric_limits<double>::quiet_NaN()
  if (b > 0x7ff0000000000000ull) return __longlong_as_double(0x7ff8000000000000ll);
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Block-wide max of up to 4 accumulators; thread 0 does the atomics.
template <int N>
__device__ __forceinline__ void block_max_atomic(unsigned long long (&v)[N], unsigned long long* dst) {
  __shared__ unsigned long long red[N][32];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nwarps = (blockDim.x * blockDim.y + 31) >> 5;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    v[q] = warp_max_u64(v[q]);
    if (lane == 0) red[q][warp] = v[q];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      unsigned long long x = lane < nwarps ? red[q][lane] : 0ull;
      x = warp_max_u64(x);
      if (lane == 0 && x) atomicMax(dst + q, x);
    }
  }
}

// Binary search of the work item that owns flattened CTA `cta`.
__device__ __forceinline__ int find_item(const sf_work* __restrict__ items, int n, int cta) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (items[mid].cta_begin <= cta) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Last-CTA election after a grid-wide accumulation (threadfence reduction).
__device__ __forceinline__ bool last_cta(unsigned int* counter, unsigned int total) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(counter, 1u);
    is_last = (t == total - 1);
  }
  __syncthreads();
  return is_last;
}

}  // namespace sfb
