/* sforge_b200.h -- C ABI of the B200-native stencil hot path.
 *
 * Drop-in boundary for the reference's (stencilforge, /root/reference/proj)
 * plugin/operator API on the data-parallel hot path: the staggered-grid
 * incompressible step (UPDATE_VELOCITY, PRESSURE_SWEEP, DIVERGENCE), the
 * ghost refresh between grid components and the max reductions.
 *
 * Two levels, both plain C (pointers, sizes, status codes; no torch types):
 *
 *  1. sf_sim_*   -- one simulation owning its fields on one CUDA device.  Each
 *                   entry point replaces one public member of
 *                   sforge::cfd::simulation / exec::executor (cited per call).
 *                   A simulation may hold several grid components ("workers")
 *                   of one decomposition on the same device; their ghost
 *                   exchange runs as device copies.
 *  2. sf_launch_* -- single-kernel launches on caller-owned device memory for
 *                   an external executor: one call per (kernel, region box
 *                   list, stream), exactly the granularity of
 *                   exec::executor::run_region_worker (executor.hpp:759-767).
 *
 * Error behaviour: every int-returning call returns SF_OK (0) or an sf_status
 * code; sf_last_error() gives the message.  Messages reuse the reference's
 * texts where the reference throws (e.g. "non-finite vx after the velocity
 * update at step N, t = ..." from cfd.hpp:278-281, the grid_error texts of
 * grid.hpp:94-137, the exec_error texts of executor.hpp:500-757).
 *
 * Numerics: fp64, IEEE round-to-nearest, no FMA contraction, the reference's
 * association order everywhere: results are bitwise identical to the
 * reference CPU implementation.
 */
#ifndef SFORGE_B200_H
#define SFORGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_ABI_VERSION 2

enum sf_status {
  SF_OK = 0,
  SF_ERR_CONFIG = 1, /* cfd_error from validate() (cfd.hpp:36-66) */
  SF_ERR_GRID = 2,   /* grid_error (grid.hpp:18-21) */
  SF_ERR_EXEC = 3,   /* exec_error (executor.hpp:32-35) */
  SF_ERR_CFD = 4,    /* cfd_error at run time, e.g. the NaN guard (cfd.hpp:278-281) */
  SF_ERR_CUDA = 5,   /* CUDA runtime failure (no reference analogue) */
  SF_ERR_ARG = 6     /* bad argument to the C ABI itself */
};

enum sf_field_id { SF_VX = 0, SF_VY = 1, SF_VZ = 2, SF_P = 3, SF_DIVU = 4, SF_NFIELDS = 5 };
enum sf_region { SF_REGION_ALL = 0, SF_REGION_INTERIOR = 1, SF_REGION_BOUNDARY = 2 }; /* executor.hpp:40 */
enum sf_reduce_op { SF_MAX_ABS = 0, SF_SUM = 1, SF_SUM_SQ = 2, SF_MAX_ABS_DIFF = 3 }; /* reductions.hpp:17-22 */
enum sf_bc_kind { SF_BC_UNSET = 0, SF_BC_WALL = 1, SF_BC_SYMMETRY = 2, SF_BC_OUTFLOW = 3 }; /* exchange.hpp:18-26 */
enum sf_bc_scope { SF_SCOPE_ALL = 0, SF_SCOPE_GHOSTS_ONLY = 1, SF_SCOPE_OWNED_ONLY = 2 };    /* exchange.hpp:49 */

/* Returns the library's SF_ABI_VERSION. */
int sf_abi_version(void);
/* Message of the last failing call on this thread (never NULL). */
const char* sf_last_error(void);
/* Number of CUDA devices visible (0 without a GPU); never fails. */
int sf_device_count(void);

/* grid::decompose (grid.hpp:92-163) without a device: proc_grid[3] and, per
 * worker w, lo[3w..3w+2] / hi[3w..3w+2] (arrays of 3*workers).  Same process
 * grid choice, balanced split and error texts as the reference. */
int sf_decompose(const int64_t extents[3], const double spacing[3], int workers, int ghost,
                 const int periodic[3], int proc_grid[3], int64_t* lo, int64_t* hi);
/* decomposition::neighbor (grid.hpp:69-81): worker across (axis, side) or -1. */
int sf_decomp_neighbor(const int proc_grid[3], const int periodic[3], int w, int axis, int side);

/* ------------------------------------------------------------------------
 * Level 1: simulation (replaces sforge::cfd::simulation, cfd.hpp:173-766)
 * ---------------------------------------------------------------------- */

/* cfd::solver_config (cfd.hpp:43-67) */
typedef struct sf_solver_config {
  int64_t extents[3];
  double spacing[3];
  double origin[3];
  int periodic[3];
  double reynolds, sigma, tolerance, omega;
  int max_sweeps;
  int symmetry_z;
  int output_cadence;
} sf_solver_config;

/* cfd::fluid_params (cfd.hpp:29-41) */
typedef struct sf_fluid_params {
  double viscosity, density;
  double body_force[3];
  double lid_speed, blend;
} sf_fluid_params;

/* Constructor arguments of cfd::simulation (cfd.hpp:175-178) plus device
 * placement.  workers = grid components of grid::decompose() on `device`. */
typedef struct sf_sim_options {
  int workers;
  int mode;    /* 0 plain, 1 overlap (exec::run_mode, executor.hpp:42) */
  int tile[3]; /* tile override, 0,0,0 = descriptor default (cfd.hpp:520) */
  int ghost;
  int form;    /* 0 rows, 1 points (cfd.hpp:169): one device form serves both */
  int device;
  int fused;   /* 1 = fused half-sweep, TMA-pipelined (default), with the
                  temporal pass (two half-sweeps per launch) where it applies:
                  one grid component per device, wall / symmetry faces;
                  3 = TMA half-sweep only; 2 = fused, plain loads (A/B
                  baseline); 0 = the reference's unfused dataflow */
  int precision; /* bytes per value of the CFD fields: 8 = fp64 (default; bitwise
                    the reference), 4 = fp32 storage and arithmetic on the fused
                    TMA half-sweep (fused 1 or 3; compared with the reference
                    under stated per-field tolerances) */
} sf_sim_options;

/* cfd::step_stats (cfd.hpp:86-90) */
typedef struct sf_step_stats {
  double dt;
  int sweeps;
  double residual;
} sf_step_stats;

typedef struct sf_sim sf_sim;

void sf_sim_options_default(sf_sim_options* o);
/* simulation::simulation (cfd.hpp:175-222).  Validates like cfd.hpp:36-66 and
 * decomposes like grid::decompose (grid.hpp:92-163). */
int sf_sim_create(const sf_solver_config* cfg, const sf_fluid_params* par,
                  const sf_sim_options* opt, sf_sim** out);
void sf_sim_destroy(sf_sim* s);

int sf_sim_init_cavity(sf_sim* s);                                   /* cfd.hpp:229-232 */
int sf_sim_init_uniform(sf_sim* s, double cx, double cy, double cz); /* cfd.hpp:234-241 */
int sf_sim_init_taylor_green(sf_sim* s);                             /* cfd.hpp:246-257 */

int sf_sim_compute_dt(sf_sim* s, double* dt);                        /* cfd.hpp:264-273 */
int sf_sim_provisional(sf_sim* s, double dt);                        /* cfd.hpp:275-282 */
int sf_sim_pressure_iteration(sf_sim* s, double dt, int* sweeps, double* residual); /* cfd.hpp:289-305 */
int sf_sim_step(sf_sim* s, sf_step_stats* out);                      /* cfd.hpp:307-316 */
int sf_sim_advance(sf_sim* s, int n, sf_step_stats* last);           /* cfd.hpp:318-321 */

double sf_sim_time(const sf_sim* s);          /* cfd.hpp:461 */
long sf_sim_step_count(const sf_sim* s);      /* cfd.hpp:462 */
int sf_sim_pending_color(sf_sim* s);          /* cfd.hpp:470 */

int sf_sim_max_divergence(sf_sim* s, double* out);  /* cfd.hpp:342-345 */
int sf_sim_steady_delta(sf_sim* s, double* out);    /* cfd.hpp:350-355 */
int sf_sim_kinetic_energy(sf_sim* s, double* out);  /* cfd.hpp:357-363 */
/* RMS distance of vx, vy, vz to the decayed Taylor-Green vortex at time t,
 * bitwise the reference's (host sin/cos/exp, reference summation order). */
int sf_sim_taylor_green_error(sf_sim* s, double t, double* out); /* cfd.hpp:367-401 */

/* grid::scatter / grid::gather on one field (io.hpp:25-65): global x-fastest
 * float64 arrays of extents[0]*extents[1]*extents[2] values in HOST memory. */
int sf_sim_scatter(sf_sim* s, const char* field, const double* host, int64_t n);
int sf_sim_gather(sf_sim* s, const char* field, double* host, int64_t n);
/* Same, from/to a DEVICE buffer on the simulation's device (no host trip). */
int sf_sim_scatter_device(sf_sim* s, const char* field, const double* dev, int64_t n);
int sf_sim_gather_device(sf_sim* s, const char* field, double* dev, int64_t n);
/* cli::field_checksum (bench.hpp:24-39): FNV-1a of the gathered vx,vy,vz,p. */
int sf_sim_checksum(sf_sim* s, uint64_t* out);
/* One worker's padded front array, ghosts included, x fastest with extents
 * dims+2g (the reference layout local_block::offset, field.hpp:39-44). */
int sf_sim_local_front(sf_sim* s, const char* field, int worker, double* host,
                       int64_t host_elems, int64_t dims[3], int64_t lo[3]);

/* exec::executor operations on this simulation's fields (executor.hpp:500-527).
 * fields: array of n field names.  params: n_params (name, value) pairs. */
int sf_sim_refresh(sf_sim* s, const char* const* fields, int n);  /* :520-523 */
int sf_sim_exchange(sf_sim* s, const char* const* fields, int n); /* :511-514 */
int sf_sim_run_kernel(sf_sim* s, const char* name, const char* const* param_names,
                      const double* param_values, int n_params, int region); /* :500-509 */
int sf_sim_reduce(sf_sim* s, const char* field, int op, double* out);        /* :525-527 */
int sf_sim_invalidate_ghosts(sf_sim* s, const char* field);                  /* :612 */
int sf_sim_invalidate_all_ghosts(sf_sim* s);                                 /* :613 */
int sf_sim_ghosts_valid(sf_sim* s, const char* field);                       /* :610 */

/* ---- one process per GPU ---------------------------
 * Rank r of `world` owns grid component r of grid::decompose(dom, world, g,
 * periodic); ghost faces between ranks move over NCCL (send/recv per peer and
 * refresh phase), the per-sweep residual, dt maxima and NaN guard over
 * ncclAllReduce(max).  Rank 0 creates the NCCL unique id (128 bytes), the
 * caller broadcasts it (e.g. torch.distributed) and every rank calls
 * sf_sim_create_distributed collectively.  opt->workers must be 1. */
int sf_nccl_unique_id(void* out128);
int sf_sim_create_distributed(const sf_solver_config* cfg, const sf_fluid_params* par,
                              const sf_sim_options* opt, int rank, int world, const void* nccl_id,
                              sf_sim** out);
/* The same decomposition with the CUDA-IPC transport instead of NCCL: every
 * rank maps its peers' device buffers into its own address space
 * (cudaIpcGetMemHandle / cudaIpcOpenMemHandle) and moves ghost messages with
 * device-to-device copies or direct stores; the host callbacks below carry
 * only the 64-byte handles, residual maxima and barriers.  All ranks call
 * every function of a simulation in the same order (as with NCCL).  The ranks
 * may share one device (separate processes; the host orders them, no kernel
 * waits on another rank) or sit on peer-accessible devices of one node.
 * Callbacks return 0 on success. */
typedef struct sf_host_transport {
  void* ctx;
  /* recv (world * bytes) = every rank's `bytes` of send, in rank order */
  int (*allgather)(void* ctx, const void* send, void* recv, int64_t bytes);
  int (*barrier)(void* ctx);
} sf_host_transport;
/* Host-only: the direct-store plan of the temporal pass's exchange for one
 * rank (no device needed): up to 26 rows of 14 int64 each -- peer, direction
 * d[3], source box lo[3] and dims[3] (this rank's local coordinates),
 * destination dlo[3] (the peer's local coordinates), count. */
int sf_direct_plan(const int64_t extents[3], int world, int ghost, const int periodic[3], int rank, int max_boxes,
                   int64_t* out, int* n_out);
int sf_sim_create_ipc(const sf_solver_config* cfg, const sf_fluid_params* par, const sf_sim_options* opt,
                      int rank, int world, const sf_host_transport* transport, sf_sim** out);
/* Exchange of the temporal pass across ranks (exchange.hpp:165-224), where
 * every peer's buffers map into this process: 1 (default) = fused into the
 * pass -- its cells within g of a processor face also store their outputs
 * straight into the neighbours' ghost shells (26 directions: faces, edges,
 * corners); 2 = one separate launch of the same direct stores after each
 * pass; 0 = pack, send/recv, unpack in three axis phases, overlapped with the
 * interior tiles.  sf_sim_direct_exchange returns the mode in use (0 when the
 * peers do not map; a collective call the first time). */
int sf_sim_set_direct_exchange(sf_sim* s, int on);
int sf_sim_direct_exchange(sf_sim* s);
int sf_sim_rank(const sf_sim* s);
int sf_sim_world(const sf_sim* s);
/* Owned cells of one grid component (global worker id) as a dense x-fastest
 * host array of dims[0]*dims[1]*dims[2] values: the per-rank slice of
 * grid::gather / grid::scatter (io.hpp:25-65). */
int sf_sim_gather_block(sf_sim* s, const char* field, int worker, double* host, int64_t n);
int sf_sim_scatter_block(sf_sim* s, const char* field, int worker, const double* host, int64_t n);
/* Asynchronous forms; the call returns at once and `host` must be
 * page-locked and left untouched until sf_sim_synchronize.
 *  - gather_block_async snapshots the block on the device, in order with the
 *    compute already enqueued, and downloads the snapshot in the background:
 *    later compute overlaps the transfer.
 *  - scatter_block_async queues the upload on the library's upload stream;
 *    later compute waits for it.
 * Uploads and downloads of different fields overlap (PCIe is full duplex). */
int sf_sim_gather_block_async(sf_sim* s, const char* field, int worker, double* host, int64_t n);
int sf_sim_scatter_block_async(sf_sim* s, const char* field, int worker, const double* host, int64_t n);
/* scatter_block_async in two halves, so the next step's inputs cross PCIe
 * while the current step computes: stage queues the upload into the field's
 * device buffer (after the last install out of it); install_staged queues the
 * copy into the field, in order with compute enqueued before and after it.
 * install_staged without a staged upload fails (SF_ERR_ARG). */
int sf_sim_stage_block_async(sf_sim* s, const char* field, int worker, const double* host, int64_t n);
int sf_sim_install_staged(sf_sim* s, const char* field, int worker);
/* The exchange plan of one refresh phase (axis 0..2, slabs widened as in
 * exchange.hpp:165-206) or of the fused loop's face exchange (axis = -1) for
 * rank `rank` of a `world`-rank decomposition -- host logic, no device.  Rows
 * of 15 int64: kind (0 send, 1 recv, 2 local copy), peer, field, axis, side,
 * lo[3], dims[3], dlo[3], count; sends and receives per peer in posting order
 * (sender: sides 0,1; receiver: sides 1,0). */
int sf_exchange_plan(const int64_t extents[3], int world, int ghost, const int periodic[3], int rank,
                     unsigned field_mask, int axis, int max_msgs, int64_t* out, int* n_out);

/* ---- descriptor-declared kernels (the plugin path, executor.hpp:484-498) -----
 * codegen::execution_plan (codegen.hpp:41-57): tile, halo (-x,+x,-y,+y,-z,+z),
 * bindings (field, intent, cached) in declaration order, parameter names.
 * intent: 0 IN, 1 OUT, 2 INOUT, 3 SEPARATEINOUT (descriptor.hpp:216). */
typedef struct sf_binding {
  const char* field;
  int intent;
  int cached;
} sf_binding;
typedef struct sf_plan {
  const char* kernel;
  int tile[3];
  int halo[6];
  const sf_binding* bindings;
  int n_bindings;
  const char* const* params;
  int n_params;
} sf_plan;
/* field_store::create (field.hpp:108-112); stagger -1 none, 0/1/2 = x/y/z. */
int sf_sim_create_field(sf_sim* s, const char* name, int stagger);
/* The same with fp32 storage (value_bytes 4) or fp64 (8). An fp32 field is
 * exchanged, reduced and read by descriptor kernels like any field; its
 * values cross this interface as fp64 (gather widens exactly, scatter rounds
 * to nearest), and kernels compute on them in fp64 and store rounded. */
int sf_sim_create_field_typed(sf_sim* s, const char* name, int stagger, int value_bytes);
/* executor::register_kernel with the point function given as the CUDA C++
 * BODY of `void f(const point_ctx& c)` against the reference's accessors
 * (c.field(s)(di,dj,dk), .load(), .store(v), c.param(s), c.i/c.j/c.k;
 * executor.hpp:130-184).  The body is JIT-compiled for sm_100a (NVRTC,
 * --fmad=false) into a tile kernel whose CTA is the plan's TILE.  Same checks
 * and error texts as register_common (executor.hpp:650-692); a compile error
 * returns SF_ERR_EXEC with the compiler log.  Run with sf_sim_run_kernel. */
int sf_sim_register_kernel(sf_sim* s, const sf_plan* plan, const char* const* sig_fields, int n_sig_fields,
                           const char* const* sig_params, int n_sig_params, const char* point_body);

/* executor::boundary() (executor.hpp:482): one physical face condition
 * (kind sf_bc_kind, velocity used by walls); faces indexed (axis, side). */
int sf_sim_set_face_bc(sf_sim* s, int axis, int side, int kind, const double velocity[3]);
/* executor::physical_bc (executor.hpp:516-518) */
int sf_sim_physical_bc(sf_sim* s, const char* const* fields, int n);

/* exec::schedule_step (executor.hpp:422-466): kind 0 run, 1 exchange,
 * 2 physical_bc, 3 refresh, 4 reduce. */
typedef struct sf_schedule_step {
  int kind;
  const char* kernel;
  int region;
  const char* const* fields;
  int n_fields;
  const char* source;
  int op;
  const char* target;
} sf_schedule_step;
/* executor::run_schedule (executor.hpp:533-553) incl. the dry run's
 * ghost-validity check and its error texts; reduce steps store results. */
int sf_sim_run_schedule(sf_sim* s, const sf_schedule_step* steps, int n_steps, const char* const* param_names,
                        const double* param_values, int n_params, int passes, int mode);
/* executor::results() (executor.hpp:615) */
int sf_sim_result(sf_sim* s, const char* name, double* value);

/* Device plumbing for benches and transports. */
int sf_sim_synchronize(sf_sim* s);        /* waits for compute and host transfers */
void* sf_sim_stream(sf_sim* s);            /* the cudaStream_t all work is ordered on */
/* Kernel launches issued by this simulation since creation (or the last reset). */
int64_t sf_sim_launch_count(sf_sim* s, int reset);
/* Per-kernel CUDA-event timing of the pressure loop: when enabled, the driver
 * records events around every executed launch of the fused half-sweep
 * (kernel "sweep_div") or of the temporal pass (kernel "sweep2", two
 * half-sweeps per launch); read back the summed milliseconds and launches.
 * "sweep2i" counts the passes among them that ran on the interior form
 * (k_sweep2i beside the slab launches; milliseconds 0). */
int sf_sim_set_kernel_timing(sf_sim* s, int enable);
int sf_sim_kernel_timing(sf_sim* s, const char* kernel, double* total_ms, int64_t* launches);

/* ------------------------------------------------------------------------
 * Level 2: single-kernel launches for an external executor
 * ---------------------------------------------------------------------- */

/* Device geometry of one local block (local_block, field.hpp:31-52) with an
 * explicit, aligned pitch:  offset(i,j,k) = base + (k*sy + j)*sx + i  for
 * local i,j,k in [-ghost, dims+ghost).  Rows are 128-byte aligned at i = 0. */
typedef struct sf_layout {
  int64_t dims[3];
  int64_t lo[3];
  int ghost;
  int64_t sx, sy, sz;
  int64_t base;
} sf_layout;

/* executor.hpp:73-79, local owned coordinates, hi exclusive */
typedef struct sf_box {
  int64_t lo[3];
  int64_t hi[3];
} sf_box;

/* One physical face condition (exchange.hpp:18-26) */
typedef struct sf_face_bc {
  int kind;
  double velocity[3];
} sf_face_bc;

/* step_constants (cfd.hpp:473-487), computed on the host exactly as
 * cfd.hpp:192-217 does; global extents and periodic bits included. */
typedef struct sf_cfd_consts {
  double dt, nu, alpha, fx, fy, fz, ix, iy, iz, ix2, iy2, iz2;
  double bscale[2][2][2];
  int64_t nxm1, nym1, nzm1;
  int px, py, pz;
} sf_cfd_consts;

int sf_make_layout(const int64_t dims[3], const int64_t lo[3], int ghost, sf_layout* out);
int64_t sf_layout_elems(const sf_layout* l);
int sf_make_cfd_consts(const sf_solver_config* cfg, const sf_fluid_params* par, sf_cfd_consts* out);

/* UPDATE_VELOCITY (cfd.hpp:524-589) over the boxes: reads front vx,vy,vz,p
 * (ghosts valid), writes back vx,vy,vz.  The caller swaps (executor.hpp:772-773). */
int sf_launch_update_velocity(const sf_layout* l, const double* vx, const double* vy,
                              const double* vz, const double* p, double* vx_out,
                              double* vy_out, double* vz_out, const sf_cfd_consts* c,
                              const sf_box* boxes, int nbox, void* stream);
/* DIVERGENCE (cfd.hpp:595-618) */
int sf_launch_divergence(const sf_layout* l, const double* vx, const double* vy,
                         const double* vz, double* divu, const sf_cfd_consts* c,
                         const sf_box* boxes, int nbox, void* stream);
/* PRESSURE_SWEEP (cfd.hpp:630-720), in place on p,vx,vy,vz */
int sf_launch_pressure_sweep(const sf_layout* l, const double* divu, double* p, double* vx,
                             double* vy, double* vz, const sf_cfd_consts* c, double beta,
                             int color, const sf_box* boxes, int nbox, void* stream);
/* bc_face (exchange.hpp:231-480) of one field on one face of one block.
 * stagger: -1 none, 0/1/2 = x/y/z.  Tangential ranges follow the axis phase. */
int sf_launch_bc_face(const sf_layout* l, double* front, int stagger, int axis, int side,
                      const sf_face_bc* bc, int scope, void* stream);
/* Box copy between two blocks' arrays (one pack+unpack of exchange.hpp:165-224):
 * copies src box (src-local coords) to dst box starting at dst_lo. */
int sf_launch_copy_box(const sf_layout* src_l, const double* src, const sf_layout* dst_l,
                       double* dst, const int64_t src_lo[3], const int64_t dims[3],
                       const int64_t dst_lo[3], void* stream);
/* Pack / unpack a box to / from a contiguous x-fastest buffer (for NCCL /
 * peer transports between processes). */
int sf_launch_pack_box(const sf_layout* l, const double* src, const int64_t lo[3],
                       const int64_t dims[3], double* buf, void* stream);
int sf_launch_unpack_box(const sf_layout* l, double* dst, const int64_t lo[3],
                         const int64_t dims[3], const double* buf, void* stream);
/* max_abs / max_abs_diff over owned cells (reductions.hpp:39-71), folded
 * into *dev_out, a device double the caller initialises (0.0 to start a
 * reduction; calls on further blocks or fields accumulate into it).  The
 * kernel combines with an integer atomicMax on the IEEE bit pattern of |x|,
 * which orders non-negative doubles exactly, so the result is bitwise the
 * reference's max for any evaluation order; a NaN anywhere wins (its |x|
 * pattern exceeds +inf's, 0x7ff0000000000000) and reads back as a NaN. */
int sf_launch_reduce_max(const sf_layout* l, const double* front, const double* back, int op,
                         double* dev_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SFORGE_B200_H */
