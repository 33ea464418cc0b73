/*
 * mhd_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the fp64 ideal-MHD
 * Godunov step that is the hot path of arxiv 2510.24175 (gPLUTO, PAPER.md:146-155
 * §3.2: "boundary exchange/calculation, mapping of the conservative vectors to
 * primitive vectors, reconstruction ... of the cells interfaces values, solving
 * Riemann problem ..., computing the right hand side", repeated per Runge-Kutta
 * stage; divergence control by cleaning).
 *
 * The paper prints no equations; every formula follows the readings R1..R29 in
 * DESIGN.md §3 (which restate SURVEY.md §8(c) c.0-c.17: Miyoshi & Kusano 2005
 * HLLD, Dedner 2002 / Mignone & Tzeferacos 2010 GLM, van Leer MC, Heun RK2).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  It shares no code with the CUDA path (paper_2510_24175_b200/).
 *
 * Array layout at this interface: U[f][z][y][x], interior cells only, x fastest,
 * nvar = 8 + glm fields in the order (rho, mx, my, mz, E, Bx, By, Bz, psi).
 * All functions return 0 on success, nonzero on error (1 = bad argument,
 * 6 = unphysical state, see orc_counters.first_bad_cell / bad_stage).
 */
#ifndef MHD_ORACLE_H
#define MHD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n[3];        /* interior cells per axis; n[d]==1 => axis inactive (R7) */
  double lo[3], hi[3]; /* domain extent */
  int32_t bc_lo[3], bc_hi[3]; /* 0 periodic, 1 outflow (R18) */
  double gamma, cfl;
  int32_t limiter;     /* 0 minmod, 1 MC (c.5), 2 WENOZ (R31; ghost width 3) */
  int32_t riemann;     /* 0 HLL, 1 HLLD */
  int32_t glm;         /* 1 => 9 fields with GLM cleaning */
  int32_t stepper;     /* 0 SSP-RK2 (Heun, R2), 1 SSP-RK3 (Shu-Osher) */
  double glm_alpha;    /* 0.1 (R12) */
  double p_floor;      /* 1e-12 (R16) */
  int32_t ct;          /* 1: constrained transport: U fields 5..7 are the
                          face-centred b_x (face i-1/2), b_y (j-1/2), b_z (k-1/2); 3D periodic, glm 0 */
  int32_t pad2_;
} orc_config;

typedef struct {
  int64_t p_floors;      /* per (interior cell, stage) */
  int64_t plm_fallbacks; /* per (interior cell, active direction, stage) */
  int64_t hlld_to_hll;   /* per (face, stage) */
  int64_t first_bad_cell;/* lowest interior linear index (z*ny+y)*nx+x, or -1 */
  int32_t bad_stage;     /* 0 = dt pass, 1..3 = RK stage; -1 none */
  int32_t pad_;
} orc_counters;

/* counters must be reset by the caller before the first call (bad_stage = first_bad_cell = -1) */
void orc_counters_reset(orc_counters* cnt);
/* CT: discrete divergence sum_d (b_d(i+1) - b_d(i))/dx_d of the face field of interior U, per cell
 * (test helper for the div B pin; out has ncell entries). */
int orc_ct_divb(const orc_config* c, const double* U, double* out);
/* c.3: conservative -> primitive for one cell. Returns 1 if p was floored. */
int orc_cons2prim(const orc_config* c, const double* U, double* V);
/* c.4 energy of a primitive state (used by the tests for prim->cons round trips). */
double orc_total_energy(double gamma, const double* V);
/* c.4 fast magnetosonic speed. */
double orc_fast_speed(double gamma, double rho, double p, double bn, double bt1, double bt2);
/* WENO-Z face value between c and d from the cells (a, b, c, d, e) (R31). */
double orc_wenoz(double a, double b, double c, double d, double e);
/* c.5 limited slope. */
double orc_limited_slope(int32_t limiter, double dm, double dp);
/* c.6-c.10: one face flux in the normal frame (rho,vn,vt1,vt2,p,Bn,Bt1,Bt2[,psi]).
 * F receives nvar components in the normal frame.  Returns 1 if HLLD fell back to HLL. */
int orc_face_flux(const orc_config* c, const double* VL, const double* VR, double ch, double* F);
/* batched variant: VL/VR/F are [n][nvar] rows. returns number of HLL fallbacks. */
/* test-only: the HLLD wave fan of one face pair (speeds, branch flags, the six states and
 * the two side fluxes; layout in mhd_oracle.c) — 73 doubles */
void orc_hlld_fan(const orc_config* c, const double* VL, const double* VR, double ch, double* out);
int64_t orc_face_flux_batch(const orc_config* c, const double* VL, const double* VR, int64_t n,
                            double ch, double* F);
/* c.13: M = max_cells sum_d s_d/dx_d and ch = max_cells max_d s_d; dt = cfl/M. */
int orc_compute_dt(const orc_config* c, const double* U, double* dt, double* ch, orc_counters* cnt);
/* c.2-c.12: one full RK2 step in place on interior U, with the given dt and ch. */
int orc_step(const orc_config* c, double* U, double dt, double ch, orc_counters* cnt);
/* one RK stage operator S(U) (c.11), for tests of the stage operator alone. */
int orc_stage(const orc_config* c, const double* U, double* Uout, double dt, double ch, orc_counters* cnt);
/* c.14 driver: nsteps steps (t_end <= 0: no clamp).  dt_log has room for nsteps. */
int orc_run(const orc_config* c, double* U, int64_t nsteps, double t_end, double* dt_log,
            int64_t* steps_done, orc_counters* cnt);
/* number of OpenMP threads the oracle will use (1 if built without OpenMP) */
int orc_num_threads(void);
void orc_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
