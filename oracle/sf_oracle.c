/* oracle/sf_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's hot path: the staggered-grid
 * incompressible step of stencilforge (/root/reference/proj/include/stencilforge)
 * for ONE worker (the whole domain in one padded block).  Results of the
 * reference are decomposition-invariant (tests/test_cfd.cpp:231-273, 436-461),
 * so a single-block restatement is a full oracle for the field values.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against the golden
 * checksums of SURVEY.md Appendix A (64^3 cavity: 1 step 1b07d1f577d4bad0,
 * 10 steps 32b900f8b9e72ed2) and bitwise against oracle/_ref/libsfref.so (the
 * reference compiled in place) on random fields, every BC kind and periodic
 * axes.
 *
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off, as proj/CMakeLists.txt:26-33).
 * Every expression keeps the reference's association order; -ffp-contract=off
 * keeps a*b+c from fusing.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- parameters: flat mirror of cfd::solver_config + cfd::fluid_params
 *      (cfd.hpp:29-67); same struct as oracle/ref_shim.cpp ------------------ */
typedef struct sfo_params {
  int64_t extents[3];
  double spacing[3];
  int periodic[3];
  double reynolds, sigma, tolerance, omega;
  int max_sweeps;
  int symmetry_z;
  double viscosity, density;
  double body_force[3];
  double lid_speed, blend;
  int workers, mode;
  int tile[3];
  int ghost;
  int form;
} sfo_params;

enum { BC_UNSET = 0, BC_WALL = 1, BC_SYM = 2, BC_OUT = 3 };
enum { ST_NONE = -1, ST_X = 0, ST_Y = 1, ST_Z = 2 };
enum { F_VX = 0, F_VY, F_VZ, F_P, F_DIVU, NF };
static const char* const fnames[NF] = {"vx", "vy", "vz", "p", "divu"};
static const int fstag[NF] = {ST_X, ST_Y, ST_Z, ST_NONE, ST_NONE};

typedef struct { int kind; double vel[3]; } facebc; /* exchange.hpp:18-26 */

typedef struct {
  int64_t n[3], ld[3];
  int g;
  double *front, *back;
  int stag;
} fld; /* field.hpp:31-52 (x fastest, ld = dims + 2g) */

typedef struct sfo_sim {
  sfo_params P;
  fld f[NF];
  facebc bc[6];
  /* step_constants (cfd.hpp:473-487) */
  double dt, nu, alpha, fx, fy, fz, ix, iy, iz, ix2, iy2, iz2;
  double bscale[2][2][2];
  int64_t nxm1, nym1, nzm1;
  int px, py, pz;
  double time;
  long steps;
  int color;
  char err[256];
} sfo_sim;

static char g_err[512];
const char* sfo_last_error(void) { return g_err; }

static inline int64_t off(const fld* F, int64_t i, int64_t j, int64_t k) {
  /* field.hpp:39-44 */
  return ((k + F->g) * F->ld[1] + (j + F->g)) * F->ld[0] + (i + F->g);
}
#define AT(F, i, j, k) ((F)->front[off((F), (i), (j), (k))])

static int field_id(const char* name) {
  for (int i = 0; i < NF; ++i)
    if (strcmp(name, fnames[i]) == 0) return i;
  return -1;
}

/* ---- construction ------------------------------------------------------ */
void sfo_destroy(sfo_sim* s);

sfo_sim* sfo_create(const sfo_params* p) {
  /* validation as solver_config::validate / fluid_params::validate (cfd.hpp:36-66) */
  for (int a = 0; a < 3; ++a) {
    if (p->extents[a] < 1) { snprintf(g_err, sizeof g_err, "domain extents must be positive"); return NULL; }
    if (!(p->spacing[a] > 0.0)) { snprintf(g_err, sizeof g_err, "grid spacing must be positive"); return NULL; }
  }
  if (!(p->sigma > 0.0 && p->sigma < 1.0)) { snprintf(g_err, sizeof g_err, "sigma must lie in (0,1)"); return NULL; }
  if (!(p->tolerance > 0.0)) { snprintf(g_err, sizeof g_err, "pressure tolerance must be positive"); return NULL; }
  if (!(p->omega >= 1.0 && p->omega < 2.0)) { snprintf(g_err, sizeof g_err, "omega must lie in [1,2)"); return NULL; }
  if (p->max_sweeps < 1) { snprintf(g_err, sizeof g_err, "max_sweeps must be at least 1"); return NULL; }
  if (!(p->viscosity > 0.0)) { snprintf(g_err, sizeof g_err, "viscosity must be positive"); return NULL; }
  if (p->workers != 1) { snprintf(g_err, sizeof g_err, "the C restatement runs one worker"); return NULL; }
  const int g = p->ghost;
  if (g < 1) { snprintf(g_err, sizeof g_err, "ghost width must be >= 1"); return NULL; }
  for (int a = 0; a < 3; ++a)
    if (!(p->extents[a] > g)) { /* grid.hpp:103-105 */
      snprintf(g_err, sizeof g_err, "no feasible decomposition"); return NULL;
    }

  sfo_sim* s = (sfo_sim*)calloc(1, sizeof(sfo_sim));
  s->P = *p;
  for (int fi = 0; fi < NF; ++fi) {
    fld* F = &s->f[fi];
    F->g = g;
    F->stag = fstag[fi];
    for (int a = 0; a < 3; ++a) { F->n[a] = p->extents[a]; F->ld[a] = p->extents[a] + 2 * g; }
    size_t cells = (size_t)(F->ld[0] * F->ld[1] * F->ld[2]);
    F->front = (double*)calloc(cells, sizeof(double));
    /* SEPARATEINOUT bindings get a zero-filled back buffer (executor.hpp:680-683) */
    if (fi <= F_VZ) F->back = (double*)calloc(cells, sizeof(double));
  }
  /* make_bc (cfd.hpp:500-512) */
  for (int axis = 0; axis < 3; ++axis) {
    if (p->periodic[axis]) continue;
    for (int side = 0; side < 2; ++side) { s->bc[2 * axis + side].kind = BC_WALL; }
  }
  if (!p->periodic[1]) { s->bc[3].kind = BC_WALL; s->bc[3].vel[0] = p->lid_speed; }
  if (!p->periodic[2] && p->symmetry_z) { s->bc[4].kind = BC_SYM; s->bc[5].kind = BC_SYM; }

  /* step constants (cfd.hpp:192-217) */
  s->nu = p->viscosity;
  s->alpha = p->blend;
  s->fx = p->body_force[0]; s->fy = p->body_force[1]; s->fz = p->body_force[2];
  s->ix = 1.0 / p->spacing[0]; s->iy = 1.0 / p->spacing[1]; s->iz = 1.0 / p->spacing[2];
  s->ix2 = s->ix * s->ix; s->iy2 = s->iy * s->iy; s->iz2 = s->iz * s->iz;
  s->nxm1 = p->extents[0] - 1; s->nym1 = p->extents[1] - 1; s->nzm1 = p->extents[2] - 1;
  s->px = p->periodic[0] ? 1 : 0; s->py = p->periodic[1] ? 1 : 0; s->pz = p->periodic[2] ? 1 : 0;
  for (int bx = 0; bx < 2; ++bx)
    for (int by = 0; by < 2; ++by)
      for (int bz = 0; bz < 2; ++bz) {
        const double num = 2.0 * s->ix2 + 2.0 * s->iy2 + 2.0 * s->iz2;
        const double den = (bx ? 2.0 : 1.0) * s->ix2 + (by ? 2.0 : 1.0) * s->iy2 + (bz ? 2.0 : 1.0) * s->iz2;
        s->bscale[bx][by][bz] = num / den;
      }
  return s;
}

void sfo_destroy(sfo_sim* s) {
  if (!s) return;
  for (int fi = 0; fi < NF; ++fi) { free(s->f[fi].front); free(s->f[fi].back); }
  free(s);
}

static int fail(sfo_sim* s, const char* msg) {
  (void)s;
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

/* ---- ghost refresh: exchange.hpp:107-119 for one worker --------------
 * Per axis: the periodic self-exchange (grid.hpp:71-81 wraps the neighbour
 * onto the worker itself), then the physical BC of that axis (bc_face,
 * exchange.hpp:231-480).  Tangential ranges widen over earlier axes. */
static void wrap_axis(fld* F, int axis) {
  const int64_t g = F->g, b = F->n[axis];
  int64_t lo[3], hi[3];
  for (int t = 0; t < 3; ++t) {
    if (t < axis) { lo[t] = -g; hi[t] = F->n[t] + g; }
    else { lo[t] = 0; hi[t] = F->n[t]; }
  }
  /* pack_axis :165-206 then unpack :208-224; source (owned layers) and
   * destination (ghost layers) are disjoint, so copy directly. */
  for (int side = 0; side < 2; ++side) {
    const int64_t src0 = side == 0 ? 0 : b - g;
    const int64_t dst0 = side == 0 ? b : -g;
    for (int64_t l = 0; l < g; ++l) {
      int64_t a0 = axis == 0 ? src0 + l : lo[0], a1 = axis == 0 ? src0 + l + 1 : hi[0];
      int64_t b0 = axis == 1 ? src0 + l : lo[1], b1 = axis == 1 ? src0 + l + 1 : hi[1];
      int64_t e0 = axis == 2 ? src0 + l : lo[2], e1 = axis == 2 ? src0 + l + 1 : hi[2];
      for (int64_t k = e0; k < e1; ++k)
        for (int64_t j = b0; j < b1; ++j)
          for (int64_t i = a0; i < a1; ++i) {
            int64_t di = i, dj = j, dk = k;
            if (axis == 0) di = dst0 + l;
            if (axis == 1) dj = dst0 + l;
            if (axis == 2) dk = dst0 + l;
            AT(F, di, dj, dk) = AT(F, i, j, k);
          }
    }
  }
}

static inline double* line_at(fld* F, int64_t* c, int axis, int64_t pos) {
  c[axis] = pos;
  return &F->front[off(F, c[0], c[1], c[2])];
}

static void bc_face(sfo_sim* s, fld* F, int axis, int side) {
  const facebc fb = s->bc[2 * axis + side];
  const int64_t g = F->g, b = F->n[axis];
  const int normal = F->stag == axis;
  const int velocity = F->stag != ST_NONE;
  const double vwall = velocity ? fb.vel[F->stag] : 0.0;
  int64_t tlo[3] = {0, 0, 0}, thi[3] = {0, 0, 0};
  for (int t = 0; t < 3; ++t) {
    if (t == axis) continue;
    if (t < axis) { tlo[t] = -g; thi[t] = F->n[t] + g; }
    else { tlo[t] = 0; thi[t] = F->n[t]; }
  }
  const int t1 = axis == 0 ? 1 : 0;
  const int t2 = axis == 2 ? 1 : 2;
  int64_t c[3];
#define LINE(pos) (*line_at(F, c, axis, (pos)))
  for (c[t2] = tlo[t2]; c[t2] < thi[t2]; ++c[t2]) {
    for (c[t1] = tlo[t1]; c[t1] < thi[t1]; ++c[t1]) {
      if (normal) {
        if (fb.kind == BC_WALL || fb.kind == BC_SYM) {
          const double v = fb.kind == BC_WALL ? vwall : 0.0;
          if (side == 0) {
            LINE(-1) = v;
            for (int64_t m = 2; m <= g; ++m) { const double src = LINE(m - 2); LINE(-m) = 2.0 * v - src; }
          } else {
            LINE(b - 1) = v; /* bc_scope::all */
            for (int64_t m = 1; m <= g; ++m) { const double src = LINE(b - 1 - m); LINE(b - 1 + m) = 2.0 * v - src; }
          }
        } else if (fb.kind == BC_OUT) {
          if (side == 0) { const double v0 = LINE(0); for (int64_t m = 1; m <= g; ++m) LINE(-m) = v0; }
          else { const double v0 = LINE(b - 1); for (int64_t m = 1; m <= g; ++m) LINE(b - 1 + m) = v0; }
        }
      } else {
        if (fb.kind == BC_WALL && velocity) {
          if (side == 0) for (int64_t m = 1; m <= g; ++m) { const double src = LINE(m - 1); LINE(-m) = 2.0 * vwall - src; }
          else for (int64_t m = 1; m <= g; ++m) { const double src = LINE(b - m); LINE(b - 1 + m) = 2.0 * vwall - src; }
        } else if (fb.kind == BC_WALL || fb.kind == BC_SYM) {
          if (side == 0) for (int64_t m = 1; m <= g; ++m) { const double src = LINE(m - 1); LINE(-m) = src; }
          else for (int64_t m = 1; m <= g; ++m) { const double src = LINE(b - m); LINE(b - 1 + m) = src; }
        } else if (fb.kind == BC_OUT) {
          if (side == 0) { const double v0 = LINE(0); for (int64_t m = 1; m <= g; ++m) LINE(-m) = v0; }
          else { const double v0 = LINE(b - 1); for (int64_t m = 1; m <= g; ++m) LINE(b - 1 + m) = v0; }
        }
      }
    }
  }
#undef LINE
}

static int refresh_ids(sfo_sim* s, const int* ids, int n) {
  for (int axis = 0; axis < 3; ++axis)
    if (!s->P.periodic[axis])
      for (int side = 0; side < 2; ++side)
        if (s->bc[2 * axis + side].kind == BC_UNSET) return fail(s, "no boundary condition");
  for (int axis = 0; axis < 3; ++axis) {
    if (s->P.periodic[axis])
      for (int q = 0; q < n; ++q) wrap_axis(&s->f[ids[q]], axis);
    else
      for (int q = 0; q < n; ++q)
        for (int side = 0; side < 2; ++side) bc_face(s, &s->f[ids[q]], axis, side);
  }
  return 0;
}

/* ---- kernels (cfd.hpp:524-720) ------------------------------------------ */
static void update_velocity(sfo_sim* s) {
  fld *U = &s->f[F_VX], *V = &s->f[F_VY], *W = &s->f[F_VZ], *Q = &s->f[F_P];
  const int64_t nx = U->n[0], ny = U->n[1], nz = U->n[2];
#define u(a, b, c) U->front[off(U, i + (a), j + (b), k + (c))]
#define v(a, b, c) V->front[off(V, i + (a), j + (b), k + (c))]
#define w(a, b, c) W->front[off(W, i + (a), j + (b), k + (c))]
#define q(a, b, c) Q->front[off(Q, i + (a), j + (b), k + (c))]
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const double u0 = u(0, 0, 0), v0 = v(0, 0, 0), w0 = w(0, 0, 0);
        /* x momentum :537-552 */
        const double ue = u(1, 0, 0), uw = u(-1, 0, 0);
        const double un = u(0, 1, 0), us = u(0, -1, 0);
        const double ut = u(0, 0, 1), ub = u(0, 0, -1);
        const double vn = v(0, 0, 0) + v(1, 0, 0), vs = v(0, -1, 0) + v(1, -1, 0);
        const double wt = w(0, 0, 0) + w(1, 0, 0), wb = w(0, 0, -1) + w(1, 0, -1);
        double fux = (u0 + ue) * (u0 + ue) - (uw + u0) * (uw + u0);
        fux += s->alpha * (fabs(u0 + ue) * (u0 - ue) - fabs(uw + u0) * (uw - u0));
        double fuy = vn * (u0 + un) - vs * (us + u0);
        fuy += s->alpha * (fabs(vn) * (u0 - un) - fabs(vs) * (us - u0));
        double fuz = wt * (u0 + ut) - wb * (ub + u0);
        fuz += s->alpha * (fabs(wt) * (u0 - ut) - fabs(wb) * (ub - u0));
        const double lapu = (ue - 2.0 * u0 + uw) * s->ix2 + (un - 2.0 * u0 + us) * s->iy2 +
                            (ut - 2.0 * u0 + ub) * s->iz2;
        const double rhsu = (q(0, 0, 0) - q(1, 0, 0)) * s->ix -
                            0.25 * (fux * s->ix + fuy * s->iy + fuz * s->iz) + s->nu * lapu + s->fx;
        U->back[off(U, i, j, k)] = u0 + s->dt * rhsu;
        /* y momentum :554-570 */
        const double ve = v(1, 0, 0), vw = v(-1, 0, 0);
        const double vnn = v(0, 1, 0), vss = v(0, -1, 0);
        const double vt = v(0, 0, 1), vb = v(0, 0, -1);
        const double ue2 = u(0, 0, 0) + u(0, 1, 0), uw2 = u(-1, 0, 0) + u(-1, 1, 0);
        const double wt2 = w(0, 0, 0) + w(0, 1, 0), wb2 = w(0, 0, -1) + w(0, 1, -1);
        double fvx = ue2 * (v0 + ve) - uw2 * (vw + v0);
        fvx += s->alpha * (fabs(ue2) * (v0 - ve) - fabs(uw2) * (vw - v0));
        double fvy = (v0 + vnn) * (v0 + vnn) - (vss + v0) * (vss + v0);
        fvy += s->alpha * (fabs(v0 + vnn) * (v0 - vnn) - fabs(vss + v0) * (vss - v0));
        double fvz = wt2 * (v0 + vt) - wb2 * (vb + v0);
        fvz += s->alpha * (fabs(wt2) * (v0 - vt) - fabs(wb2) * (vb - v0));
        const double lapv = (ve - 2.0 * v0 + vw) * s->ix2 + (vnn - 2.0 * v0 + vss) * s->iy2 +
                            (vt - 2.0 * v0 + vb) * s->iz2;
        const double rhsv = (q(0, 0, 0) - q(0, 1, 0)) * s->iy -
                            0.25 * (fvx * s->ix + fvy * s->iy + fvz * s->iz) + s->nu * lapv + s->fy;
        V->back[off(V, i, j, k)] = v0 + s->dt * rhsv;
        /* z momentum :572-588 */
        const double we = w(1, 0, 0), ww = w(-1, 0, 0);
        const double wn = w(0, 1, 0), ws = w(0, -1, 0);
        const double wtt = w(0, 0, 1), wbb = w(0, 0, -1);
        const double ue3 = u(0, 0, 0) + u(0, 0, 1), uw3 = u(-1, 0, 0) + u(-1, 0, 1);
        const double vn3 = v(0, 0, 0) + v(0, 0, 1), vs3 = v(0, -1, 0) + v(0, -1, 1);
        double fwx = ue3 * (w0 + we) - uw3 * (ww + w0);
        fwx += s->alpha * (fabs(ue3) * (w0 - we) - fabs(uw3) * (ww - w0));
        double fwy = vn3 * (w0 + wn) - vs3 * (ws + w0);
        fwy += s->alpha * (fabs(vn3) * (w0 - wn) - fabs(vs3) * (ws - w0));
        double fwz = (w0 + wtt) * (w0 + wtt) - (wbb + w0) * (wbb + w0);
        fwz += s->alpha * (fabs(w0 + wtt) * (w0 - wtt) - fabs(wbb + w0) * (wbb - w0));
        const double lapw = (we - 2.0 * w0 + ww) * s->ix2 + (wn - 2.0 * w0 + ws) * s->iy2 +
                            (wtt - 2.0 * w0 + wbb) * s->iz2;
        const double rhsw = (q(0, 0, 0) - q(0, 0, 1)) * s->iz -
                            0.25 * (fwx * s->ix + fwy * s->iy + fwz * s->iz) + s->nu * lapw + s->fz;
        W->back[off(W, i, j, k)] = w0 + s->dt * rhsw;
      }
#undef u
#undef v
#undef w
#undef q
  /* finish_run: SEPARATEINOUT swap (executor.hpp:769-779, field.hpp:89-93) */
  for (int fi = F_VX; fi <= F_VZ; ++fi) {
    double* t = s->f[fi].front; s->f[fi].front = s->f[fi].back; s->f[fi].back = t;
  }
}

static void divergence(sfo_sim* s) { /* cfd.hpp:612-618 */
  fld *U = &s->f[F_VX], *V = &s->f[F_VY], *W = &s->f[F_VZ], *D = &s->f[F_DIVU];
  for (int64_t k = 0; k < D->n[2]; ++k)
    for (int64_t j = 0; j < D->n[1]; ++j)
      for (int64_t i = 0; i < D->n[0]; ++i) {
        double d = (AT(U, i, j, k) - AT(U, i - 1, j, k)) * s->ix;
        d += (AT(V, i, j, k) - AT(V, i, j - 1, k)) * s->iy;
        d += (AT(W, i, j, k) - AT(W, i, j, k - 1)) * s->iz;
        AT(D, i, j, k) = d;
      }
}

static void pressure_sweep(sfo_sim* s, double beta, int color) { /* cfd.hpp:699-720 */
  fld *D = &s->f[F_DIVU], *Pf = &s->f[F_P], *U = &s->f[F_VX], *V = &s->f[F_VY], *W = &s->f[F_VZ];
  for (int64_t k = 0; k < D->n[2]; ++k)
    for (int64_t j = 0; j < D->n[1]; ++j)
      for (int64_t i = 0; i < D->n[0]; ++i) {
        const double a0 = ((i + j + k) & 1) == color ? 1.0 : 0.0;
        const double a1 = ((i + j + k + 1) & 1) == color ? 1.0 : 0.0;
        const int bx = s->px | ((i > 0) & (i < s->nxm1));
        const int by = s->py | ((j > 0) & (j < s->nym1));
        const int bz = s->pz | ((k > 0) & (k < s->nzm1));
        const int bxp = s->px | (i + 1 < s->nxm1);
        const int byp = s->py | (j + 1 < s->nym1);
        const int bzp = s->pz | (k + 1 < s->nzm1);
        const double d0 = -(beta * s->bscale[bx][by][bz]) * AT(D, i, j, k) * a0;
        const double ex = -(beta * s->bscale[bxp][by][bz]) * AT(D, i + 1, j, k) * a1;
        const double ey = -(beta * s->bscale[bx][byp][bz]) * AT(D, i, j + 1, k) * a1;
        const double ez = -(beta * s->bscale[bx][by][bzp]) * AT(D, i, j, k + 1) * a1;
        AT(Pf, i, j, k) = AT(Pf, i, j, k) + d0;
        AT(U, i, j, k) = AT(U, i, j, k) + s->dt * s->ix * (d0 - ex);
        AT(V, i, j, k) = AT(V, i, j, k) + s->dt * s->iy * (d0 - ey);
        AT(W, i, j, k) = AT(W, i, j, k) + s->dt * s->iz * (d0 - ez);
      }
}

/* ---- reductions (reductions.hpp:28-90, one worker) ----------------------- */
static double reduce_f(const fld* F, int op) {
  double acc = 0.0;
  int nanhit = 0;
  for (int64_t k = 0; k < F->n[2]; ++k)
    for (int64_t j = 0; j < F->n[1]; ++j)
      for (int64_t i = 0; i < F->n[0]; ++i) {
        const int64_t o = off(F, i, j, k);
        const double x = F->front[o];
        switch (op) {
          case 0: { const double a = fabs(x); acc = a > acc ? a : acc; nanhit |= a != a; break; }
          case 1: acc += x; break;
          case 2: acc += x * x; break;
          case 3: { const double a = fabs(x - F->back[o]); acc = a > acc ? a : acc; nanhit |= a != a; break; }
        }
      }
  if (nanhit) acc = NAN;
  return acc;
}

int sfo_reduce(sfo_sim* s, const char* name, int op, double* out) {
  const int id = field_id(name);
  if (id < 0) return fail(s, "no field named");
  if (op == 3 && !s->f[id].back) return fail(s, "field has no back buffer to diff against");
  *out = reduce_f(&s->f[id], op);
  return 0;
}

/* ---- the time step (cfd.hpp:264-316) ------------------------------------ */
int sfo_compute_dt(sfo_sim* s, double* out) {
  double dt = 1.0 / (2.0 * s->nu * (s->ix2 + s->iy2 + s->iz2));
  const double mx = reduce_f(&s->f[F_VX], 0);
  const double my = reduce_f(&s->f[F_VY], 0);
  const double mz = reduce_f(&s->f[F_VZ], 0);
  /* std::min(a, b) == (b < a) ? b : a */
  if (mx > 0.0) { const double c = s->P.spacing[0] / mx; dt = c < dt ? c : dt; }
  if (my > 0.0) { const double c = s->P.spacing[1] / my; dt = c < dt ? c : dt; }
  if (mz > 0.0) { const double c = s->P.spacing[2] / mz; dt = c < dt ? c : dt; }
  *out = s->P.sigma * dt;
  return 0;
}

int sfo_provisional(sfo_sim* s, double dt) {
  s->dt = dt;
  static const int ids[4] = {F_VX, F_VY, F_VZ, F_P};
  if (refresh_ids(s, ids, 4)) return 1;
  update_velocity(s);
  for (int fi = F_VX; fi <= F_VZ; ++fi)
    if (!isfinite(reduce_f(&s->f[fi], 0))) {
      snprintf(g_err, sizeof g_err, "non-finite %s after the velocity update at step %ld, t = %f",
               fnames[fi], s->steps, s->time);
      return 1;
    }
  return 0;
}

static void refresh_divergence(sfo_sim* s) { /* cfd.hpp:723-726 */
  static const int ids[3] = {F_VX, F_VY, F_VZ};
  refresh_ids(s, ids, 3);
  divergence(s);
}

int sfo_pressure_iteration(sfo_sim* s, double dt, int* sweeps_out, double* residual_out) {
  s->dt = dt;
  const double beta = s->P.omega / (2.0 * dt * (s->ix2 + s->iy2 + s->iz2));
  refresh_divergence(s);
  int sweeps = 0;
  double residual = 0.0;
  static const int dv[1] = {F_DIVU};
  do {
    refresh_ids(s, dv, 1);
    pressure_sweep(s, beta, s->color);
    s->color ^= 1;
    ++sweeps;
    refresh_divergence(s);
    residual = reduce_f(&s->f[F_DIVU], 0);
  } while (residual > s->P.tolerance && sweeps < s->P.max_sweeps);
  *sweeps_out = sweeps;
  *residual_out = residual;
  return 0;
}

int sfo_step(sfo_sim* s, double* dt_out, int* sweeps, double* residual) {
  double dt;
  sfo_compute_dt(s, &dt);
  if (sfo_provisional(s, dt)) return 1;
  sfo_pressure_iteration(s, dt, sweeps, residual);
  static const int pp[1] = {F_P};
  refresh_ids(s, pp, 1);
  s->time += dt;
  ++s->steps;
  *dt_out = dt;
  return 0;
}

int sfo_advance(sfo_sim* s, int n, double* dts, int* sweeps, double* residuals) {
  for (int i = 0; i < n; ++i) {
    double dt, r;
    int sw;
    if (sfo_step(s, &dt, &sw, &r)) return 1;
    if (dts) dts[i] = dt;
    if (sweeps) sweeps[i] = sw;
    if (residuals) residuals[i] = r;
  }
  return 0;
}

/* ---- initial states (cfd.hpp:229-257, 444-459) -------------------------- */
static void reset_clock(sfo_sim* s) { s->time = 0.0; s->steps = 0; s->color = 0; }

static void fill_const(sfo_sim* s, int id, double c) {
  fld* F = &s->f[id];
  for (int64_t k = 0; k < F->n[2]; ++k)
    for (int64_t j = 0; j < F->n[1]; ++j)
      for (int64_t i = 0; i < F->n[0]; ++i) AT(F, i, j, k) = c;
}

int sfo_init_cavity(sfo_sim* s) {
  for (int fi = 0; fi < NF; ++fi) fill_const(s, fi, 0.0);
  reset_clock(s);
  return 0;
}

int sfo_init_uniform(sfo_sim* s, double cx, double cy, double cz) {
  fill_const(s, F_VX, cx); fill_const(s, F_VY, cy); fill_const(s, F_VZ, cz);
  fill_const(s, F_P, 0.0); fill_const(s, F_DIVU, 0.0);
  reset_clock(s);
  return 0;
}

int sfo_init_taylor_green(sfo_sim* s) {
  const double tau = 2.0 * 3.14159265358979323846;
  const double dx = s->P.spacing[0], dy = s->P.spacing[1];
  fld *U = &s->f[F_VX], *V = &s->f[F_VY], *Q = &s->f[F_P];
  for (int64_t k = 0; k < U->n[2]; ++k)
    for (int64_t j = 0; j < U->n[1]; ++j)
      for (int64_t i = 0; i < U->n[0]; ++i) {
        const double xc = ((double)i + 0.5) * dx, yc = ((double)j + 0.5) * dy;
        const double xf = xc + 0.5 * dx, yf = yc + 0.5 * dy;
        AT(U, i, j, k) = sin(tau * xf) * cos(tau * yc);
        AT(V, i, j, k) = -cos(tau * xc) * sin(tau * yf);
        AT(Q, i, j, k) = 0.25 * (cos(2.0 * tau * xc) + cos(2.0 * tau * yc));
      }
  fill_const(s, F_VZ, 0.0);
  fill_const(s, F_DIVU, 0.0);
  reset_clock(s);
  return 0;
}

/* cfd.hpp:367-401: RMS distance to the decayed analytic vortex, x-fastest
 * over the owned cells (one worker, so one partial). */
int sfo_taylor_green_error(sfo_sim* s, double t, double* out) {
  const double tau = 2.0 * 3.14159265358979323846;
  const double decay = exp(-2.0 * s->P.viscosity * tau * tau * t);
  const double dx = s->P.spacing[0], dy = s->P.spacing[1];
  fld *U = &s->f[F_VX], *V = &s->f[F_VY], *W = &s->f[F_VZ];
  double sum = 0.0;
  for (int64_t k = 0; k < U->n[2]; ++k)
    for (int64_t j = 0; j < U->n[1]; ++j)
      for (int64_t i = 0; i < U->n[0]; ++i) {
        const double xc = ((double)i + 0.5) * dx, yc = ((double)j + 0.5) * dy;
        const double xf = (double)(i + 1) * dx, yf = (double)(j + 1) * dy;
        const double eu = AT(U, i, j, k) - sin(tau * xf) * cos(tau * yc) * decay;
        const double ev = AT(V, i, j, k) + cos(tau * xc) * sin(tau * yf) * decay;
        const double ew = AT(W, i, j, k);
        sum += eu * eu + ev * ev + ew * ew;
      }
  const double n = (double)(U->n[0] * U->n[1] * U->n[2]);
  *out = sqrt(sum / (3.0 * n));
  return 0;
}

/* ---- data movement (io.hpp:25-65) ---------------------------------------- */
int sfo_scatter(sfo_sim* s, const char* name, const double* global, int64_t n) {
  const int id = field_id(name);
  if (id < 0) return fail(s, "no field named");
  fld* F = &s->f[id];
  if (n != F->n[0] * F->n[1] * F->n[2]) return fail(s, "scatter: size mismatch");
  for (int64_t k = 0; k < F->n[2]; ++k)
    for (int64_t j = 0; j < F->n[1]; ++j)
      memcpy(&AT(F, 0, j, k), global + (k * F->n[1] + j) * F->n[0], (size_t)F->n[0] * sizeof(double));
  return 0;
}

int sfo_gather(sfo_sim* s, const char* name, double* out) {
  const int id = field_id(name);
  if (id < 0) return fail(s, "no field named");
  fld* F = &s->f[id];
  for (int64_t k = 0; k < F->n[2]; ++k)
    for (int64_t j = 0; j < F->n[1]; ++j)
      memcpy(out + (k * F->n[1] + j) * F->n[0], &AT(F, 0, j, k), (size_t)F->n[0] * sizeof(double));
  return 0;
}

int sfo_local_front(sfo_sim* s, const char* name, int w, double* out, int64_t* dims, int64_t* lo) {
  const int id = field_id(name);
  if (id < 0 || w != 0) return fail(s, "no such field/worker");
  fld* F = &s->f[id];
  for (int a = 0; a < 3; ++a) { dims[a] = F->n[a]; lo[a] = 0; }
  memcpy(out, F->front, (size_t)(F->ld[0] * F->ld[1] * F->ld[2]) * sizeof(double));
  return 0;
}

int sfo_refresh(sfo_sim* s, const char* csv) {
  int ids[NF], n = 0;
  char buf[128];
  snprintf(buf, sizeof buf, "%s", csv);
  for (char* tok = strtok(buf, ","); tok; tok = strtok(NULL, ",")) {
    const int id = field_id(tok);
    if (id < 0) return fail(s, "no field named");
    ids[n++] = id;
  }
  return refresh_ids(s, ids, n);
}

int sfo_run_kernel(sfo_sim* s, const char* name, const char* params, int region) {
  if (region != 0) return fail(s, "the C restatement runs region::all only");
  if (strcmp(name, "DIVERGENCE") == 0) { divergence(s); return 0; }
  if (strcmp(name, "UPDATE_VELOCITY") == 0) { update_velocity(s); return 0; }
  if (strcmp(name, "PRESSURE_SWEEP") == 0) {
    double beta = 0.0, color = 0.0;
    const char* b = strstr(params, "beta=");
    const char* c = strstr(params, "color=");
    if (!b || !c) return fail(s, "parameter not supplied");
    beta = strtod(b + 5, NULL);
    color = strtod(c + 6, NULL);
    pressure_sweep(s, beta, (int)color);
    return 0;
  }
  return fail(s, "unknown kernel");
}

uint64_t sfo_fnv1a(uint64_t h, const unsigned char* p, int64_t n) {
  for (int64_t i = 0; i < n; ++i) { h ^= p[i]; h *= 1099511628211ull; }
  return h;
}

uint64_t sfo_checksum(sfo_sim* s) { /* bench.hpp:24-39 */
  uint64_t h = 1469598103934665603ull;
  static const int ids[4] = {F_VX, F_VY, F_VZ, F_P};
  for (int q = 0; q < 4; ++q) {
    const fld* F = &s->f[ids[q]];
    h = sfo_fnv1a(h, (const unsigned char*)fnames[ids[q]], (int64_t)strlen(fnames[ids[q]]));
    for (int64_t k = 0; k < F->n[2]; ++k)
      for (int64_t j = 0; j < F->n[1]; ++j)
        h = sfo_fnv1a(h, (const unsigned char*)&F->front[off(F, 0, j, k)], F->n[0] * 8);
  }
  return h;
}

double sfo_time(sfo_sim* s) { return s->time; }
long sfo_step_count(sfo_sim* s) { return s->steps; }
int sfo_pending_color(sfo_sim* s) { return s->color; }
void sfo_invalidate_all_ghosts(sfo_sim* s) { (void)s; }

int sfo_diag(sfo_sim* s, double* max_div, double* steady_delta, double* kinetic) {
  if (steady_delta) { /* cfd.hpp:350-355 */
    double d = reduce_f(&s->f[F_VX], 3);
    const double dy = reduce_f(&s->f[F_VY], 3);
    d = d < dy ? dy : d;
    const double dz = reduce_f(&s->f[F_VZ], 3);
    d = d < dz ? dz : d;
    *steady_delta = d;
  }
  if (kinetic) { /* cfd.hpp:357-363 */
    const double sum = reduce_f(&s->f[F_VX], 2) + reduce_f(&s->f[F_VY], 2) + reduce_f(&s->f[F_VZ], 2);
    const double cell = s->P.spacing[0] * s->P.spacing[1] * s->P.spacing[2];
    *kinetic = 0.5 * s->P.density * sum * cell;
  }
  if (max_div) { refresh_divergence(s); *max_div = reduce_f(&s->f[F_DIVU], 0); }
  return 0;
}
