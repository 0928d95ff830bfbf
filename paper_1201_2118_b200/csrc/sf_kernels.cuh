// sf_kernels.cuh -- launch interface between the host driver and the kernels.
#pragma once

#include "sf_device.cuh"

namespace sfb {

// One ghost-refresh task: a copy between blocks (one message of
// exchange.hpp:165-224) or one physical face fill (bc_face, :231-480).
struct sf_task {
  int type;  // 0 copy, 1 bc, 2 pack (box -> buf), 3 unpack (buf -> box),
             // 4 direct store into a peer process's array (pack + send + unpack in one)
  int field;
  int src_blk, dst_blk;
  long long lo[3];    // copy: source box (src-local); bc: tangential box (axis entry unused)
  long long dims[3];  // copy: box extents; bc: tangential extents (axis entry 1)
  long long dlo[3];   // copy: destination lo (dst-local)
  long long count;    // elements (copy) or lines (bc)
  int axis, side, normal, velocity, kind, scope;
  double v;           // wall velocity component (normal pin / tangential reflection)
  double* buf;        // pack / unpack: contiguous x-fastest message buffer
  // direct store (type 4): the source is slot `slot` of (src_blk, field); the
  // destination is the peer's array of the same physical buffer index (every
  // rank swaps identically), mapped into this process (CUDA IPC), with the
  // peer's padded layout; dlo is in the peer's local coordinates
  int slot;
  double* rptr[kSlots];
  long long rsx, rsy, rbase;
};

// Tile shapes (threads = TX x TY; each thread marches z over a chunk).
constexpr int kTX = 32;
constexpr int kTY = 8;

// max_ctas: CTAs per task (grid x); 1184 = 8 per SM
template <class View>
void launch_tasks(const View& vw, const sf_task* tasks, int ntasks, long long max_count,
                  const sf_dev_ctl* pred, cudaStream_t st, int max_ctas = 1184);
// one task passed by value (no device task list)
void launch_task_one(const direct_view& vw, const sf_task& t, cudaStream_t st);
template <class View>
void launch_update_velocity(const View& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                            double dt, cudaStream_t st);
// TMA-staged UPDATE_VELOCITY (sf_uv_tma.cu): table view, 32 x 8 tiles;
// maps = device table of uv descriptors (uv_box shapes).
void launch_update_velocity_tma(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                                const void* maps, cudaStream_t st, int es = 8);
size_t uv_maps_bytes();
size_t uv_map_offset(int b, int f, int s);  // f: 0 vx, 1 vy, 2 vz, 3 p
void uv_box(int field, int* bw, int* bh, int es = 8);
template <class View>
void launch_divergence(const View& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                       int acc_slot, int predicated, cudaStream_t st, int es = 8);
// beta_color_dt: null = beta, colour and dt from ctl; else {beta, colour, dt}
template <class View>
void launch_pressure_sweep(const View& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                           int predicated, const double* beta_color_dt, cudaStream_t st);
// fin = 1: the last CTA finalises the sweep; 0: the caller allreduces acc[0]
// across ranks and runs CTL_FINISH_FUSED; 2 (TMA kernel only): the predicated
// redo of a temporal pass's first sweep (see launch_sweep2)
void launch_sweep_div(const table_view& vw, int nctas, int zc, const sf_consts& c,
                      sf_dev_ctl* ctl, sf_host_flag* hflag, int fin, cudaStream_t st);
// The whole pressure loop in one cooperative launch (single process, no
// processor faces): min(ntiles, co-resident CTAs) CTAs stride over the tiles.
cudaError_t launch_pressure_loop(const table_view& vw, int ntiles, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                                 cudaStream_t st);
int pressure_loop_ctas();
// TMA-pipelined fused half-sweep (sf_sweep_tma.cu); maps = device sweep_maps.
// es = 4: the fp32 variant of the CFD fields (storage and arithmetic in fp32).
void launch_sweep_div_tma(const table_view& vw, int nctas, int zc, const sf_consts& c,
                          sf_dev_ctl* ctl, sf_host_flag* hflag, const void* maps, int fin,
                          cudaStream_t st, int es = 8);
// Temporal pass: two half-sweeps per launch (sf_sweep2.cu). Blocks whose
// faces are walls, symmetry planes or processor faces (ghost width >= 2 when
// there are processor faces); maps = device table of sweep2 descriptors.
// fin = 1: the last CTA finalises; 0: the caller allreduces acc[0..1] across
// ranks and runs CTL_FINISH_PASS. pins: wall-normal velocities of the
// domain's high walls (u, v, w) and low walls (ul, vl, wl); 0 for symmetry.
struct sweep2_pins {
  double u, v, w, ul, vl, wl;
};
// Across ranks, the pass can store its outputs in the g owned layers next to
// every processor face, edge and corner straight into the neighbour's ghost
// shell (the ghost exchange fused into the update): one entry per direction
// of the direct-store plan (sf_plan.hpp build_direct_plan), the peer's arrays
// mapped into this process.
struct sweep2_peer {
  double* ptr[4][kSlots];  // vx, vy, vz, divu of the peer, by physical buffer index
  long long rsx, rsy, rbase;
  long long shift[3];      // peer-local index = this block's local index + shift
};
struct sweep2_remote {
  int g;
  int idx[27];  // direction (dx+1) + 3 (dy+1) + 9 (dz+1) -> peer entry, or -1
  sweep2_peer peer[26];
};
// total_ctas: CTAs of the whole pass when it is split over several launches
// (the last one to finish finalises); 0 = this launch alone.
// remote: device array of sweep2_remote (one per local block) for the fused
// exchange, or null
void launch_sweep2(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                   sf_host_flag* hflag, const void* maps, int fin, const sweep2_pins& pins, cudaStream_t st,
                   unsigned total_ctas = 0, const sweep2_remote* remote = nullptr, int es = 8, int shape = 0);
// The interior form of the temporal pass (fp64; tiles where k_sweep2 takes its
// fast path everywhere): no S1 field ring, 3 CTAs per SM. maps: a maps table
// with sweep2i_box shapes; total: CTAs of the whole pass (with the k_sweep2
// launch over the boundary slabs).
void launch_sweep2i(const table_view& vw, int nctas, int zc, const sf_consts& c, sf_dev_ctl* ctl,
                    sf_host_flag* hflag, const void* maps, int fin, cudaStream_t st, unsigned total, int es = 8);
void sweep2i_box(int field, int* bw, int* bh, int es = 8);
size_t sweep2_maps_bytes();
size_t sweep2_map_offset(int b, int f, int s);
// shape 0: the pass's tiles (32 x sweep2_tile_y()); 1: the x-slab form
void sweep2_box(int field, int* bw, int* bh, int es = 8, int shape = 0);
void sweep2_tile(int shape, int* tx, int* ty);
int sweep2_tile_y();  // tile height of the selected temporal-pass variant (tile width 32)
int sweep2i_tile_y(int es = 8);  // tile height of the interior form (k_sweep2i; width 32)
int encode_sweep_map(void* map_out, double* base, long long sx, long long sy, long long sz, int field, int es = 8);
size_t sweep_maps_bytes();
int encode_box_map(void* map_out, double* base, long long sx, long long sy, long long sz, int bw, int bh,
                   int es = 8);
void sweep_tile_shape(int* tx, int* ty);  // tile of the selected TMA pipeline variant
size_t sweep_map_offset(int b, int f, int s);
template <class View>
void launch_reduce_max(const View& vw, int nctas, int zc, const int* fields, int nfields, int diff,
                       unsigned long long* acc, cudaStream_t st);
void launch_reduce_sum(const table_view& vw, int nctas, int zc, int field, int square,
                       double* partials, cudaStream_t st);
// Single-thread control updates.
enum ctl_op {
  CTL_DT_FROM_ACC = 0,       // compute_dt from acc[0..2] (cfd.hpp:264-273), beta (cfd.hpp:291)
  CTL_SET_DT = 1,            // dt = arg, beta from dt
  CTL_BEGIN_ITERATION = 2,   // sweeps = 0, done = abort, residual = 0, acc[0] = 0
  CTL_AFTER_SWEEP = 3,       // unfused loop: color ^= 1, ++sweeps (cfd.hpp:299-300)
  CTL_FINISH_SWEEP = 4,      // unfused loop: residual from acc[0], done test (cfd.hpp:302-303)
  CTL_CHECK_FINITE = 5,      // NaN guard after UPDATE_VELOCITY from acc[1..3] (cfd.hpp:278-281)
  CTL_CLEAR_ACC = 6,
  CTL_SWAP = 7,              // swap slots (a, b) of field f in every block
  CTL_RESET_CLOCK = 8,       // colour = 0, abort cleared (cfd.hpp:733-738)
  CTL_FINISH_FUSED = 9,      // fused half-sweep finalise after a cross-rank residual allreduce
  CTL_PUBLISH = 10,          // loop state -> host-mapped flag (after the graph-captured loop)
  CTL_FINISH_PASS = 11,      // temporal pass finalise after the cross-rank allreduce of acc[0..1]
};
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
void ensure_smem_attr(const void* kernel, int bytes);
// owned block of (b, f) FRONT -> dense fp64 buffer, FRONT read from the device table
void launch_snapshot(const sf_dev_table* tab, int b, int f, double* buf, long long rows, cudaStream_t st);
// dense fp64 buffer -> owned block of (b, f) FRONT, FRONT read from the device table
void launch_install(const sf_dev_table* tab, int b, int f, const double* buf, long long rows, cudaStream_t st);
// sets the pressure-loop graph's while condition to !ctl->done
void launch_loop_cond(cudaGraphConditionalHandle h, const sf_dev_ctl* ctl, cudaStream_t st);
void launch_ctl(sf_dev_table* tab, sf_dev_ctl* ctl, sf_host_flag* hflag, int op, double arg,
                int f, int a, int b, const sf_consts& c, int predicated, cudaStream_t st);
void launch_copy_box(const double* src, long long s_base, long long s_sx, long long s_sy,
                     double* dst, long long d_base, long long d_sx, long long d_sy,
                     const long long lo[3], const long long dims[3], const long long dlo[3],
                     cudaStream_t st);
void launch_fill_box(void* dst, long long base, long long sx, long long sy, const long long lo[3],
                     const long long dims[3], double v, cudaStream_t st, int es = 8);
// taylor_green_error's per-cell term (cfd.hpp:388-393) of one block into a
// dense x-fastest buffer; su / sv: the analytic sin*cos factors per (i, j)
void launch_tg_cells(const double* U, const double* V, const double* W, long long base, long long sx, long long sy,
                     const long long dims[3], const double* su, const double* sv, double decay, double* out,
                     cudaStream_t st);
// element sizes 8 (double) or 4 (float); values convert on the way
void launch_copy_box_es(const void* src, int s_es, long long s_base, long long s_sx, long long s_sy, void* dst,
                        int d_es, long long d_base, long long d_sx, long long d_sy, const long long lo[3],
                        const long long dims[3], const long long dlo[3], cudaStream_t st);
// field_es: bytes per value of the field (the global array is always fp64)
void launch_gather_owned(const double* src, long long base, long long sx, long long sy,
                         const long long n[3], const long long lo[3], const long long N[3],
                         double* dst_global, int to_field /* 1 = scatter */, cudaStream_t st,
                         int field_es = 8);

}  // namespace sfb
