/*
 * mhd_oracle.c — TEST INFRASTRUCTURE ONLY (see mhd_oracle.h).
 *
 * The plain CPU oracle of the fp64 ideal-MHD Godunov step of arxiv 2510.24175
 * (gPLUTO's 5-step RK pipeline, §3.2; double precision,
 * PAPER.md:179 §4.2; GLM divergence cleaning).
 *
 * The paper gives no formulas.  This file follows, step by step and in the
 * same order and association, the recipe written in DESIGN.md §3
 * ("Readings"), which restates SURVEY.md §8(c) c.0-c.17:
 *   c.2 ghost fill, c.3 cons->prim, c.4 face prim->cons + fast speed,
 *   c.5 PLM (minmod / MC), c.6 GLM interface pre-solve, c.7 physical flux,
 *   c.8 HLL (Miyoshi-Kusano eq. 67 speed bounds), c.9 HLLD (Miyoshi & Kusano
 *   2005), c.10 flux assembly, c.11 stage operator + RK2, c.12 GLM damping,
 *   c.13 CFL dt and c_h.
 * Arithmetic discipline (c.0 / DESIGN.md R-ARITH): compiled with
 * -ffp-contract=off and without -ffast-math; only + - * / sqrt fabs fmin fmax
 * per cell; every expression is evaluated exactly as parenthesised here.
 *
 * No blocking, fusion or reordering: each stage materialises the padded
 * state, the primitive array, the PLM face states and the face fluxes of
 * every direction, then applies the update.  OpenMP only splits the outer
 * loop of each pass; every output element is written by exactly one
 * iteration and the only reductions are integer sums and exact max/min, so
 * results are bitwise independent of the thread count.
 */
#include "mhd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_E_ARG 1
#define ORC_E_UNPHYSICAL 6

/* ------------------------------------------------------------------------ */
/* grid bookkeeping                                                          */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t n[3];   /* interior cells */
  int64_t g[3];   /* ghost width: 2 on active axes (PLM, c.1), 0 otherwise */
  int64_t m[3];   /* padded extent n + 2g */
  int act[3];     /* axis active (R7) */
  int nvar;       /* 8 + glm */
  double dx[3];   /* (hi-lo)/n, host double (c.1) */
} grid_t;

static int make_grid(const orc_config* c, grid_t* G) {
  if (!c) return ORC_E_ARG;
  if (!(c->gamma > 1.0) || !(c->cfl > 0.0 && c->cfl < 1.0)) return ORC_E_ARG;
  if (c->limiter < 0 || c->limiter > 2) return ORC_E_ARG;
  int nact = 0;
  for (int d = 0; d < 3; ++d) {
    if (c->n[d] < 1) return ORC_E_ARG;
    G->n[d] = c->n[d];
    G->act[d] = c->n[d] > 1;
    if (G->act[d] && c->n[d] < 4) return ORC_E_ARG;
    G->g[d] = G->act[d] ? (c->limiter == 2 ? 3 : 2) : 0; /* PLM 2, WENOZ 3 (R19) */
    G->m[d] = G->n[d] + 2 * G->g[d];
    if (!(c->hi[d] > c->lo[d])) return ORC_E_ARG;
    G->dx[d] = (c->hi[d] - c->lo[d]) / (double)c->n[d];
    nact += G->act[d];
  }
  if (nact == 0) return ORC_E_ARG;
  if (c->ct && (nact != 3 || c->glm)) return ORC_E_ARG;
  for (int d = 0; d < 3 && c->ct; ++d)
    if (c->bc_lo[d] != 0 || c->bc_hi[d] != 0) return ORC_E_ARG;
  G->nvar = 8 + (c->glm ? 1 : 0);
  return ORC_OK;
}

/* index of field f at interior coordinates (i,j,k); ghosts are negative or >= n */
static inline size_t P(const grid_t* G, int f, int64_t i, int64_t j, int64_t k) {
  return (((size_t)f * G->m[2] + (size_t)(k + G->g[2])) * G->m[1] + (size_t)(j + G->g[1])) * G->m[0] +
         (size_t)(i + G->g[0]);
}
static inline size_t padded_size(const grid_t* G) { return (size_t)G->nvar * G->m[0] * G->m[1] * G->m[2]; }
static inline int64_t interior_linear(const grid_t* G, int64_t i, int64_t j, int64_t k) {
  return (k * G->n[1] + j) * G->n[0] + i;
}

/* copy interior U[f][z][y][x] <-> padded */
static void load_interior(const grid_t* G, const double* U, double* Up) {
  for (int f = 0; f < G->nvar; ++f)
    for (int64_t k = 0; k < G->n[2]; ++k)
      for (int64_t j = 0; j < G->n[1]; ++j)
        for (int64_t i = 0; i < G->n[0]; ++i)
          Up[P(G, f, i, j, k)] = U[(((size_t)f * G->n[2] + k) * G->n[1] + j) * G->n[0] + i];
}
static void store_interior(const grid_t* G, const double* Up, double* U) {
  for (int f = 0; f < G->nvar; ++f)
    for (int64_t k = 0; k < G->n[2]; ++k)
      for (int64_t j = 0; j < G->n[1]; ++j)
        for (int64_t i = 0; i < G->n[0]; ++i)
          U[(((size_t)f * G->n[2] + k) * G->n[1] + j) * G->n[0] + i] = Up[P(G, f, i, j, k)];
}

/* ------------------------------------------------------------------------ */
/* c.2 ghost fill (row a1): periodic wrap or zero-gradient outflow, g cells   */
/* ------------------------------------------------------------------------ */
static void fill_ghosts(const orc_config* c, const grid_t* G, double* Up) {
  for (int d = 0; d < 3; ++d) {
    if (!G->act[d]) continue;
    const int64_t N = G->n[d], g = G->g[d];
    /* the two other axes, interior range (edge/corner ghosts are never read) */
    const int a = (d + 1) % 3, b = (d + 2) % 3;
    for (int f = 0; f < G->nvar; ++f)
      for (int64_t q = 0; q < G->n[b]; ++q)
        for (int64_t r = 0; r < G->n[a]; ++r) {
          int64_t idx[3];
          idx[a] = r;
          idx[b] = q;
#define AT(s) (*(idx[d] = (s), &Up[P(G, f, idx[0], idx[1], idx[2])]))
          for (int64_t m = 1; m <= g; ++m) {
            /* periodic: U[-m] = U[N-m], U[N-1+m] = U[m-1]; outflow: U[-m] = U[0], U[N-1+m] = U[N-1] */
            const double lo_src = (c->bc_lo[d] == 0) ? AT(N - m) : AT(0);
            AT(-m) = lo_src;
            const double hi_src = (c->bc_hi[d] == 0) ? AT(m - 1) : AT(N - 1);
            AT(N - 1 + m) = hi_src;
          }
#undef AT
        }
  }
}

/* ------------------------------------------------------------------------ */
/* WENO-Z reconstruction (the paper's scheme; */
/* Borges, Carmona, Costa & Don 2008 with the Jiang-Shu smoothness indicators; */
/* reading R31: eps = 1e-40, p = 2, linear weights 1/10, 6/10, 3/10).  The     */
/* value at the face between c and d from the 5 cells (a, b, c, d, e):         */
/* ------------------------------------------------------------------------ */
double orc_wenoz(double a, double b, double c, double d, double e) {
  const double eps = 1e-40;
  /* the indicators' terms in a mirror-symmetric association: W(e,d,c,b,a) forms the same
     t, u (u1 negated) in reverse order (R31) */
  const double t0 = (a + c) - 2.0 * b, u0 = (a + 3.0 * c) - 4.0 * b;
  const double t1 = (b + d) - 2.0 * c, u1 = b - d;
  const double t2 = (c + e) - 2.0 * d, u2 = (3.0 * c + e) - 4.0 * d;
  const double b0 = (13.0 / 12.0) * (t0 * t0) + 0.25 * (u0 * u0);
  const double b1 = (13.0 / 12.0) * (t1 * t1) + 0.25 * (u1 * u1);
  const double b2 = (13.0 / 12.0) * (t2 * t2) + 0.25 * (u2 * u2);
  const double tau = fabs(b0 - b2);
  const double r0 = tau / (b0 + eps), r1 = tau / (b1 + eps), r2 = tau / (b2 + eps);
  const double a0 = 0.1 * (1.0 + r0 * r0), a1 = 0.6 * (1.0 + r1 * r1), a2 = 0.3 * (1.0 + r2 * r2);
  const double p0 = (2.0 * a - 7.0 * b) + 11.0 * c; /* 6 x the candidate values */
  const double p1 = (5.0 * c - b) + 2.0 * d;
  const double p2 = (2.0 * c + 5.0 * d) - e;
  return ((a0 * p0 + a1 * p1) + a2 * p2) / (6.0 * ((a0 + a1) + a2));
}

/* ------------------------------------------------------------------------ */
/* c.3 conservative -> primitive (row a2)                                     */
/* ------------------------------------------------------------------------ */
int orc_cons2prim(const orc_config* c, const double* U, double* V) {
  const double gm1 = c->gamma - 1.0;
  const double rho = U[0], mx = U[1], my = U[2], mz = U[3], E = U[4];
  const double Bx = U[5], By = U[6], Bz = U[7];
  const double ir = 1.0 / rho;
  const double vx = mx * ir, vy = my * ir, vz = mz * ir;
  const double ke = 0.5 * ((mx * vx + my * vy) + mz * vz);
  const double me = 0.5 * ((Bx * Bx + By * By) + Bz * Bz);
  double p = gm1 * ((E - ke) - me);
  int floored = 0;
  if (p < c->p_floor) {
    p = c->p_floor;
    floored = 1;
  }
  V[0] = rho;
  V[1] = vx;
  V[2] = vy;
  V[3] = vz;
  V[4] = p;
  V[5] = Bx;
  V[6] = By;
  V[7] = Bz;
  if (c->glm) V[8] = U[8]; /* psi passes through */
  return floored;
}

static int bad_cell(const double* U, int nvar) {
  if (!(U[0] > 0.0)) return 1;
  for (int f = 0; f < nvar; ++f)
    if (!isfinite(U[f])) return 1;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* c.4 face-state energy and fast magnetosonic speed                          */
/* ------------------------------------------------------------------------ */
double orc_total_energy(double gamma, const double* V) {
  /* E = (p/(gamma-1) + 0.5 rho |v|^2) + 0.5 |B|^2, associated as c.4 */
  const double igm1 = 1.0 / (gamma - 1.0);
  const double kin2 = (V[1] * V[1] + V[2] * V[2]) + V[3] * V[3];
  const double bt_sq = V[6] * V[6] + V[7] * V[7];
  const double mag2 = V[5] * V[5] + bt_sq;
  return (V[4] * igm1 + (0.5 * V[0]) * kin2) + 0.5 * mag2;
}

double orc_fast_speed(double gamma, double rho, double p, double bn, double bt1, double bt2) {
  const double bt_sq = bt1 * bt1 + bt2 * bt2;
  const double ir = 1.0 / rho;
  const double a2 = (gamma * p) * ir;
  const double bn2 = (bn * bn) * ir;
  const double bt2n = bt_sq * ir;
  const double b2 = bn2 + bt2n;
  const double dd = (a2 - b2) * (a2 - b2) + (4.0 * a2) * bt2n; /* (a2+b2)^2 - 4 a2 bn2, never negative */
  return sqrt(0.5 * ((a2 + b2) + sqrt(dd)));
}

/* ------------------------------------------------------------------------ */
/* c.5 limiters                                                               */
/* ------------------------------------------------------------------------ */
double orc_limited_slope(int32_t limiter, double dm, double dp) {
  if (limiter == 0) { /* minmod */
    if (dm > 0.0 && dp > 0.0) return fmin(dm, dp);
    if (dm < 0.0 && dp < 0.0) return fmax(dm, dp);
    return 0.0;
  }
  /* monotonised central (van Leer 1977) */
  const double cc = 0.5 * (dm + dp);
  if (dm > 0.0 && dp > 0.0) return fmin(fmin(2.0 * dm, 2.0 * dp), cc);
  if (dm < 0.0 && dp < 0.0) return fmax(fmax(2.0 * dm, 2.0 * dp), cc);
  return 0.0;
}

/* ------------------------------------------------------------------------ */
/* c.6-c.10 face flux in the normal frame                                     */
/* ------------------------------------------------------------------------ */
typedef struct {
  double rho, vn, vt1, vt2, p, bn, bt1, bt2;
  double E, pt, cf;
  double U[8]; /* (rho, mn, mt1, mt2, E, Bn, Bt1, Bt2) */
  double F[8]; /* physical flux, c.7 */
} side_t;

/* c.4 + c.7 for one side; bn already replaced by Bm (c.6) */
static void side_state(double gamma, double igm1, const double* V, double bn, side_t* s) {
  s->rho = V[0];
  s->vn = V[1];
  s->vt1 = V[2];
  s->vt2 = V[3];
  s->p = V[4];
  s->bn = bn;
  s->bt1 = V[6];
  s->bt2 = V[7];
  /* c.4 */
  const double kin2 = (s->vn * s->vn + s->vt1 * s->vt1) + s->vt2 * s->vt2;
  const double bt_sq = s->bt1 * s->bt1 + s->bt2 * s->bt2;
  const double mag2 = s->bn * s->bn + bt_sq;
  s->E = (s->p * igm1 + (0.5 * s->rho) * kin2) + 0.5 * mag2;
  const double mn = s->rho * s->vn, mt1 = s->rho * s->vt1, mt2 = s->rho * s->vt2;
  s->pt = s->p + 0.5 * mag2;
  const double ir = 1.0 / s->rho;
  const double a2 = (gamma * s->p) * ir;
  const double bn2 = (s->bn * s->bn) * ir;
  const double bt2 = bt_sq * ir;
  const double b2 = bn2 + bt2;
  const double dd = (a2 - b2) * (a2 - b2) + (4.0 * a2) * bt2;
  s->cf = sqrt(0.5 * ((a2 + b2) + sqrt(dd)));
  s->U[0] = s->rho;
  s->U[1] = mn;
  s->U[2] = mt1;
  s->U[3] = mt2;
  s->U[4] = s->E;
  s->U[5] = s->bn;
  s->U[6] = s->bt1;
  s->U[7] = s->bt2;
  /* c.7 */
  const double fm = s->rho * s->vn;
  s->F[0] = fm;
  s->F[1] = (fm * s->vn + s->pt) - s->bn * s->bn;
  s->F[2] = fm * s->vt1 - s->bn * s->bt1;
  s->F[3] = fm * s->vt2 - s->bn * s->bt2;
  const double vB = (s->vn * s->bn + s->vt1 * s->bt1) + s->vt2 * s->bt2;
  s->F[4] = (s->E + s->pt) * s->vn - s->bn * vB;
  s->F[5] = 0.0;
  s->F[6] = s->bt1 * s->vn - s->bn * s->vt1;
  s->F[7] = s->bt2 * s->vn - s->bn * s->vt2;
}

/* c.8 HLL average of the 8 MHD components */
static void hll_flux(const side_t* L, const side_t* R, double SL, double SR, double* F) {
  const double isd = 1.0 / (SR - SL);
  for (int k = 0; k < 8; ++k) F[k] = ((SR * L->F[k] - SL * R->F[k]) + (SL * SR) * (R->U[k] - L->U[k])) * isd;
}

/* c.9 star state of one side (Miyoshi & Kusano 2005 eqs. 43-48) */
typedef struct {
  double sd, m, sm, rhos, vst1, vst2, bst1, bst2, vBs, Es;
  double Us[8];
} star_t;

static void star_state(const side_t* s, double S, double SM, double pts, double B, star_t* t) {
  t->sd = S - s->vn;
  t->m = s->rho * t->sd;
  t->sm = S - SM;
  t->rhos = t->m / t->sm;
  const double d = t->m * t->sm - B * B;
  if (fabs(d) < 1e-8 * pts) { /* degenerate (R6): no tangential jump */
    t->vst1 = s->vt1;
    t->vst2 = s->vt2;
    t->bst1 = s->bt1;
    t->bst2 = s->bt2;
  } else {
    const double id = 1.0 / d;
    const double cv = (B * (SM - s->vn)) * id;
    const double cb = (t->m * t->sd - B * B) * id;
    t->vst1 = s->vt1 - s->bt1 * cv;
    t->vst2 = s->vt2 - s->bt2 * cv;
    t->bst1 = s->bt1 * cb;
    t->bst2 = s->bt2 * cb;
  }
  const double vB = (s->vn * B + s->vt1 * s->bt1) + s->vt2 * s->bt2;
  t->vBs = (SM * B + t->vst1 * t->bst1) + t->vst2 * t->bst2;
  t->Es = (((t->sd * s->E - s->pt * s->vn) + pts * SM) + B * (vB - t->vBs)) / t->sm;
  t->Us[0] = t->rhos;
  t->Us[1] = t->rhos * SM;
  t->Us[2] = t->rhos * t->vst1;
  t->Us[3] = t->rhos * t->vst2;
  t->Us[4] = t->Es;
  t->Us[5] = B;
  t->Us[6] = t->bst1;
  t->Us[7] = t->bst2;
}

int orc_face_flux(const orc_config* c, const double* VLin, const double* VRin, double ch, double* F) {
  const double gamma = c->gamma;
  const double igm1 = 1.0 / (gamma - 1.0);
  /* c.6 GLM interface pre-solve (Dedner 2002 eq. 41 as used by Mignone & Tzeferacos 2010) */
  double Bm, psim = 0.0;
  if (c->glm) {
    const double hc = 0.5 * ch, ihc = 0.5 / ch;
    Bm = 0.5 * (VLin[5] + VRin[5]) - ihc * (VRin[8] - VLin[8]);
    psim = 0.5 * (VLin[8] + VRin[8]) - hc * (VRin[5] - VLin[5]);
  } else {
    Bm = 0.5 * (VLin[5] + VRin[5]);
  }
  side_t L, R;
  side_state(gamma, igm1, VLin, Bm, &L);
  side_state(gamma, igm1, VRin, Bm, &R);

  /* c.8 signal speeds (Miyoshi & Kusano 2005 eq. 67) */
  const double cmax = fmax(L.cf, R.cf);
  const double SL = fmin(L.vn, R.vn) - cmax;
  const double SR = fmax(L.vn, R.vn) + cmax;
  double Fm[8];
  int fell_back = 0;
  if (SL > 0.0) {
    memcpy(Fm, L.F, sizeof Fm);
  } else if (SR < 0.0) {
    memcpy(Fm, R.F, sizeof Fm);
  } else if (c->riemann == 0) {
    hll_flux(&L, &R, SL, SR, Fm);
  } else {
    /* c.9 HLLD */
    const double B = Bm;
    const double sdL = SL - L.vn, sdR = SR - R.vn;
    const double mL = L.rho * sdL, mR = R.rho * sdR;
    const double iden = 1.0 / (mR - mL);
    const double SM = (((mR * R.vn - mL * L.vn) - R.pt) + L.pt) * iden;               /* eq. 38 */
    const double pts = ((mR * L.pt - mL * R.pt) + (mL * mR) * (R.vn - L.vn)) * iden;  /* eq. 41 */
    if (!(SL < SM && SM < SR)) {
      hll_flux(&L, &R, SL, SR, Fm);
      fell_back = 1;
    } else {
      star_t sL, sR;
      star_state(&L, SL, SM, pts, B, &sL);
      star_state(&R, SR, SM, pts, B, &sR);
      const double srL = sqrt(sL.rhos), srR = sqrt(sR.rhos);
      const double SsL = SM - fabs(B) / srL; /* eq. 51 */
      const double SsR = SM + fabs(B) / srR;
      if (!(SL <= SsL && SsR <= SR)) { /* wave-ordering guard (R7) */
        hll_flux(&L, &R, SL, SR, Fm);
        fell_back = 1;
      } else {
        double FsL[8], FsR[8];
        for (int k = 0; k < 8; ++k) FsL[k] = L.F[k] + SL * (sL.Us[k] - L.U[k]); /* eq. 64 */
        for (int k = 0; k < 8; ++k) FsR[k] = R.F[k] + SR * (sR.Us[k] - R.U[k]);
        if (SsL >= 0.0) {
          memcpy(Fm, FsL, sizeof Fm);
        } else if (SM >= 0.0 || SsR >= 0.0) {
          /* double-star states, eqs. 59-63 */
          const double sg = (B >= 0.0) ? 1.0 : -1.0;
          const double is = 1.0 / (srL + srR);
          const double vss1 = ((srL * sL.vst1 + srR * sR.vst1) + (sR.bst1 - sL.bst1) * sg) * is;
          const double vss2 = ((srL * sL.vst2 + srR * sR.vst2) + (sR.bst2 - sL.bst2) * sg) * is;
          const double bss1 = ((srL * sR.bst1 + srR * sL.bst1) + ((srL * srR) * (sR.vst1 - sL.vst1)) * sg) * is;
          const double bss2 = ((srL * sR.bst2 + srR * sL.bst2) + ((srL * srR) * (sR.vst2 - sL.vst2)) * sg) * is;
          const double vBss = (SM * B + vss1 * bss1) + vss2 * bss2;
          if (SM >= 0.0) {
            const double EssL = sL.Es - (srL * (sL.vBs - vBss)) * sg;
            const double Uss[8] = {sL.rhos, sL.rhos * SM, sL.rhos * vss1, sL.rhos * vss2, EssL, B, bss1, bss2};
            for (int k = 0; k < 8; ++k) Fm[k] = FsL[k] + SsL * (Uss[k] - sL.Us[k]); /* eq. 65 */
          } else {
            const double EssR = sR.Es + (srR * (sR.vBs - vBss)) * sg;
            const double Uss[8] = {sR.rhos, sR.rhos * SM, sR.rhos * vss1, sR.rhos * vss2, EssR, B, bss1, bss2};
            for (int k = 0; k < 8; ++k) Fm[k] = FsR[k] + SsR * (Uss[k] - sR.Us[k]);
          }
        } else {
          memcpy(Fm, FsR, sizeof Fm);
        }
      }
    }
  }
  /* c.10 assembly */
  for (int k = 0; k < 8; ++k) F[k] = Fm[k];
  if (c->glm) {
    F[5] = psim;
    F[8] = (ch * ch) * Bm;
  } else {
    F[5] = 0.0;
  }
  return fell_back;
}

/* Test-only: the HLLD wave fan of one face pair (the same side_state / star_state as
 * orc_face_flux, the double-star states by the same expressions), so that tests can pin the
 * states themselves (integral consistency, jump conditions, the R6 / R7 branches):
 * out[0..4] = SL, S*L, SM, S*R, SR; out[5] = p_t*; out[6] = 0 fan built, 1 SM outside (SL, SR),
 * 2 wave-ordering guard, 3 supersonic (SL > 0 or SR < 0, no fan); out[7], out[8] = R6 degenerate
 * flag of the left / right star state; out[9 + 8 j + k] for j = 0..7: UL, U*L, U**L, U**R, U*R,
 * UR, FL, FR (the 8 MHD components, normal frame, B_n = Bm).  Entries not reached stay 0. */
void orc_hlld_fan(const orc_config* c, const double* VLin, const double* VRin, double ch, double* out) {
  memset(out, 0, 73 * sizeof(double));
  const double gamma = c->gamma;
  const double igm1 = 1.0 / (gamma - 1.0);
  double Bm;
  if (c->glm) {
    const double ihc = 0.5 / ch;
    Bm = 0.5 * (VLin[5] + VRin[5]) - ihc * (VRin[8] - VLin[8]);
  } else {
    Bm = 0.5 * (VLin[5] + VRin[5]);
  }
  side_t L, R;
  side_state(gamma, igm1, VLin, Bm, &L);
  side_state(gamma, igm1, VRin, Bm, &R);
  double* A = out + 9;
  for (int k = 0; k < 8; ++k) {
    A[0 * 8 + k] = L.U[k];
    A[5 * 8 + k] = R.U[k];
    A[6 * 8 + k] = L.F[k];
    A[7 * 8 + k] = R.F[k];
  }
  const double cmax = fmax(L.cf, R.cf);
  const double SL = fmin(L.vn, R.vn) - cmax;
  const double SR = fmax(L.vn, R.vn) + cmax;
  out[0] = SL;
  out[4] = SR;
  if (SL > 0.0 || SR < 0.0) {
    out[6] = 3.0;
    return;
  }
  const double B = Bm;
  const double sdL = SL - L.vn, sdR = SR - R.vn;
  const double mL = L.rho * sdL, mR = R.rho * sdR;
  const double iden = 1.0 / (mR - mL);
  const double SM = (((mR * R.vn - mL * L.vn) - R.pt) + L.pt) * iden;
  const double pts = ((mR * L.pt - mL * R.pt) + (mL * mR) * (R.vn - L.vn)) * iden;
  out[2] = SM;
  out[5] = pts;
  if (!(SL < SM && SM < SR)) {
    out[6] = 1.0;
    return;
  }
  star_t sL, sR;
  star_state(&L, SL, SM, pts, B, &sL);
  star_state(&R, SR, SM, pts, B, &sR);
  out[7] = fabs(sL.m * sL.sm - B * B) < 1e-8 * pts ? 1.0 : 0.0;
  out[8] = fabs(sR.m * sR.sm - B * B) < 1e-8 * pts ? 1.0 : 0.0;
  const double srL = sqrt(sL.rhos), srR = sqrt(sR.rhos);
  const double SsL = SM - fabs(B) / srL;
  const double SsR = SM + fabs(B) / srR;
  out[1] = SsL;
  out[3] = SsR;
  for (int k = 0; k < 8; ++k) {
    A[1 * 8 + k] = sL.Us[k];
    A[4 * 8 + k] = sR.Us[k];
  }
  if (!(SL <= SsL && SsR <= SR)) {
    out[6] = 2.0;
    return;
  }
  const double sg = (B >= 0.0) ? 1.0 : -1.0;
  const double is = 1.0 / (srL + srR);
  const double vss1 = ((srL * sL.vst1 + srR * sR.vst1) + (sR.bst1 - sL.bst1) * sg) * is;
  const double vss2 = ((srL * sL.vst2 + srR * sR.vst2) + (sR.bst2 - sL.bst2) * sg) * is;
  const double bss1 = ((srL * sR.bst1 + srR * sL.bst1) + ((srL * srR) * (sR.vst1 - sL.vst1)) * sg) * is;
  const double bss2 = ((srL * sR.bst2 + srR * sL.bst2) + ((srL * srR) * (sR.vst2 - sL.vst2)) * sg) * is;
  const double vBss = (SM * B + vss1 * bss1) + vss2 * bss2;
  const double EssL = sL.Es - (srL * (sL.vBs - vBss)) * sg;
  const double EssR = sR.Es + (srR * (sR.vBs - vBss)) * sg;
  const double UssL[8] = {sL.rhos, sL.rhos * SM, sL.rhos * vss1, sL.rhos * vss2, EssL, B, bss1, bss2};
  const double UssR[8] = {sR.rhos, sR.rhos * SM, sR.rhos * vss1, sR.rhos * vss2, EssR, B, bss1, bss2};
  for (int k = 0; k < 8; ++k) {
    A[2 * 8 + k] = UssL[k];
    A[3 * 8 + k] = UssR[k];
  }
}

int64_t orc_face_flux_batch(const orc_config* c, const double* VL, const double* VR, int64_t n, double ch,
                            double* F) {
  const int nvar = 8 + (c->glm ? 1 : 0);
  int64_t fb = 0;
  for (int64_t q = 0; q < n; ++q) fb += orc_face_flux(c, VL + q * nvar, VR + q * nvar, ch, F + q * nvar);
  return fb;
}

/* ------------------------------------------------------------------------ */
/* frame permutation (R8): x:(x,y,z), y:(y,z,x), z:(z,x,y)                    */
/* ------------------------------------------------------------------------ */
static void to_normal(int d, int nvar, const double* V, double* W) {
  const int n = d, t1 = (d + 1) % 3, t2 = (d + 2) % 3;
  W[0] = V[0];
  W[1] = V[1 + n];
  W[2] = V[1 + t1];
  W[3] = V[1 + t2];
  W[4] = V[4];
  W[5] = V[5 + n];
  W[6] = V[5 + t1];
  W[7] = V[5 + t2];
  if (nvar > 8) W[8] = V[8];
}
static void from_normal(int d, int nvar, const double* W, double* V) {
  const int n = d, t1 = (d + 1) % 3, t2 = (d + 2) % 3;
  V[0] = W[0];
  V[1 + n] = W[1];
  V[1 + t1] = W[2];
  V[1 + t2] = W[3];
  V[4] = W[4];
  V[5 + n] = W[5];
  V[5 + t1] = W[6];
  V[5 + t2] = W[7];
  if (nvar > 8) V[8] = W[8];
}

/* ------------------------------------------------------------------------ */
/* one RK stage operator S(U) = U - sum_d lambda_d (F_{d,i+1/2} - F_{d,i-1/2}) */
/* (c.2 -> c.3 -> c.5 -> c.6..c.10 -> c.11)                                   */
/* Up: padded input (interior set; ghosts are filled here).  Out: padded,     */
/* interior written.                                                          */
/* ------------------------------------------------------------------------ */
static int in_star(const grid_t* G, int64_t i, int64_t j, int64_t k) {
  /* every padded cell within the ghost width of the interior along at most one axis */
  int outside = (i < 0 || i >= G->n[0]) + (j < 0 || j >= G->n[1]) + (k < 0 || k >= G->n[2]);
  return outside <= 1;
}

static int stage_op(const orc_config* c, const grid_t* G, double* Up, double* Out, const double lam[3], double ch,
                    int stage, orc_counters* cnt) {
  const int nvar = G->nvar;
  const size_t np = padded_size(G);
  const size_t plane = (size_t)G->m[0] * G->m[1] * G->m[2];

  /* c.2 */
  fill_ghosts(c, G, Up);

  /* validity of the stage input (R16): lowest interior linear index */
  int64_t first_bad = INT64_MAX;
#pragma omp parallel for collapse(2) reduction(min : first_bad) schedule(static)
  for (int64_t k = 0; k < G->n[2]; ++k)
    for (int64_t j = 0; j < G->n[1]; ++j)
      for (int64_t i = 0; i < G->n[0]; ++i) {
        double u[9];
        for (int f = 0; f < nvar; ++f) u[f] = Up[P(G, f, i, j, k)];
        if (bad_cell(u, nvar) && interior_linear(G, i, j, k) < first_bad) first_bad = interior_linear(G, i, j, k);
      }
  if (first_bad != INT64_MAX) {
    if (cnt->bad_stage < 0) {
      cnt->bad_stage = stage;
      cnt->first_bad_cell = first_bad;
    }
    return ORC_E_UNPHYSICAL;
  }

  /* c.3 on every cell the star stencil touches */
  double* V = (double*)calloc(np, sizeof(double));
  int64_t floors = 0;
#pragma omp parallel for collapse(2) reduction(+ : floors) schedule(static)
  for (int64_t k = -G->g[2]; k < G->n[2] + G->g[2]; ++k)
    for (int64_t j = -G->g[1]; j < G->n[1] + G->g[1]; ++j)
      for (int64_t i = -G->g[0]; i < G->n[0] + G->g[0]; ++i) {
        if (!in_star(G, i, j, k)) continue;
        double u[9], v[9];
        for (int f = 0; f < nvar; ++f) u[f] = Up[P(G, f, i, j, k)];
        int fl = orc_cons2prim(c, u, v);
        for (int f = 0; f < nvar; ++f) V[P(G, f, i, j, k)] = v[f];
        if (fl && i >= 0 && i < G->n[0] && j >= 0 && j < G->n[1] && k >= 0 && k < G->n[2]) floors += 1;
      }
  cnt->p_floors += floors;

  /* c.5 + c.6..c.10 per active direction; F[d] holds, at cell index i, the flux through face i-1/2 */
  double* F[3] = {NULL, NULL, NULL};
  double* Vp = (double*)calloc(np, sizeof(double)); /* q+ : left state of face i+1/2 */
  double* Vm = (double*)calloc(np, sizeof(double)); /* q- : right state of face i-1/2 */
  int64_t fallbacks = 0, to_hll = 0;
  for (int d = 0; d < 3; ++d) {
    if (!G->act[d]) continue;
    F[d] = (double*)calloc(np, sizeof(double));
    int64_t off[3] = {0, 0, 0};
    off[d] = 1;
    /* reconstruction for cells -1..N along d, interior along the other axes */
    int64_t lo3[3] = {0, 0, 0}, hi3[3] = {G->n[0], G->n[1], G->n[2]};
    lo3[d] = -1;
    hi3[d] = G->n[d] + 1;
#pragma omp parallel for collapse(2) reduction(+ : fallbacks) schedule(static)
    for (int64_t k = lo3[2]; k < hi3[2]; ++k)
      for (int64_t j = lo3[1]; j < hi3[1]; ++j)
        for (int64_t i = lo3[0]; i < hi3[0]; ++i) {
          double qp[9], qm[9], q0[9];
          for (int f = 0; f < nvar; ++f) {
            const double qa = V[P(G, f, i - off[0], j - off[1], k - off[2])];
            const double qb = V[P(G, f, i, j, k)];
            const double qc = V[P(G, f, i + off[0], j + off[1], k + off[2])];
            q0[f] = qb;
            if (c->limiter == 2) { /* WENOZ: q+ from (i-2..i+2), q- from the mirrored stencil */
              const double qaa = V[P(G, f, i - 2 * off[0], j - 2 * off[1], k - 2 * off[2])];
              const double qcc = V[P(G, f, i + 2 * off[0], j + 2 * off[1], k + 2 * off[2])];
              qp[f] = orc_wenoz(qaa, qa, qb, qc, qcc);
              qm[f] = orc_wenoz(qcc, qc, qb, qa, qaa);
            } else { /* PLM (c.5) */
              const double dm = qb - qa, dp = qc - qb;
              const double s = orc_limited_slope(c->limiter, dm, dp);
              qp[f] = qb + 0.5 * s;
              qm[f] = qb - 0.5 * s;
            }
          }
          if (!(qp[0] > 0.0 && qm[0] > 0.0 && qp[4] > 0.0 && qm[4] > 0.0)) { /* positivity fallback (R17) */
            for (int f = 0; f < nvar; ++f) qp[f] = qm[f] = q0[f];
            const int64_t cd = (d == 0) ? i : (d == 1) ? j : k;
            if (cd >= 0 && cd < G->n[d]) fallbacks += 1;
          }
          for (int f = 0; f < nvar; ++f) {
            Vp[P(G, f, i, j, k)] = qp[f];
            Vm[P(G, f, i, j, k)] = qm[f];
          }
        }
    /* faces i-1/2 for i = 0..N: VL = V+[i-1], VR = V-[i] */
    int64_t fhi[3] = {G->n[0], G->n[1], G->n[2]};
    fhi[d] = G->n[d] + 1;
#pragma omp parallel for collapse(2) reduction(+ : to_hll) schedule(static)
    for (int64_t k = 0; k < fhi[2]; ++k)
      for (int64_t j = 0; j < fhi[1]; ++j)
        for (int64_t i = 0; i < fhi[0]; ++i) {
          double vl[9], vr[9], wl[9], wr[9], fn[9], fx[9];
          for (int f = 0; f < nvar; ++f) {
            vl[f] = Vp[P(G, f, i - off[0], j - off[1], k - off[2])];
            vr[f] = Vm[P(G, f, i, j, k)];
          }
          to_normal(d, nvar, vl, wl);
          to_normal(d, nvar, vr, wr);
          to_hll += orc_face_flux(c, wl, wr, ch, fn);
          from_normal(d, nvar, fn, fx);
          for (int f = 0; f < nvar; ++f) F[d][P(G, f, i, j, k)] = fx[f];
        }
  }
  cnt->plm_fallbacks += fallbacks;
  cnt->hlld_to_hll += to_hll;

  /* c.11 update: r = lx dFx; r = r + ly dFy; r = r + lz dFz; S(U) = U - r */
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t k = 0; k < G->n[2]; ++k)
    for (int64_t j = 0; j < G->n[1]; ++j)
      for (int64_t i = 0; i < G->n[0]; ++i)
        for (int f = 0; f < nvar; ++f) {
          double r = 0.0;
          int first = 1;
          for (int d = 0; d < 3; ++d) {
            if (!G->act[d]) continue;
            int64_t o[3] = {0, 0, 0};
            o[d] = 1;
            const double dF = F[d][P(G, f, i + o[0], j + o[1], k + o[2])] - F[d][P(G, f, i, j, k)];
            if (first) {
              r = lam[d] * dF;
              first = 0;
            } else {
              r = r + lam[d] * dF;
            }
          }
          const size_t q = P(G, f, i, j, k);
          Out[q] = Up[q] - r;
        }
  (void)plane;
  free(V);
  free(Vp);
  free(Vm);
  for (int d = 0; d < 3; ++d) free(F[d]);
  return ORC_OK;
}

void orc_counters_reset(orc_counters* cnt) {
  memset(cnt, 0, sizeof *cnt);
  cnt->bad_stage = -1;
  cnt->first_bad_cell = -1;
}

int orc_stage(const orc_config* c, const double* U, double* Uout, double dt, double ch, orc_counters* cnt) {
  grid_t G;
  int rc = make_grid(c, &G);
  if (rc) return rc;
  double lam[3];
  for (int d = 0; d < 3; ++d) lam[d] = dt / G.dx[d];
  double* Up = (double*)calloc(padded_size(&G), sizeof(double));
  double* Out = (double*)calloc(padded_size(&G), sizeof(double));
  load_interior(&G, U, Up);
  rc = stage_op(c, &G, Up, Out, lam, ch, 1, cnt);
  if (rc == ORC_OK) store_interior(&G, Out, Uout);
  free(Up);
  free(Out);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Constrained transport (the paper's weak-scaling div-B */
/* method, refs Evans & Hawley 1988, Londrillo & Del      */
/* Zanna 2004; reading R32).  3D, periodic, no GLM.  U fields 5..7 hold the   */
/* face-centred b_x at x-face i-1/2, b_y at y-face j-1/2, b_z at z-face k-1/2 */
/* of cell (i,j,k).  Per stage:                                              */
/*  1. cell-centred B = 0.5 (b(face -1/2) + b(face +1/2)) per component;     */
/*  2. c.3 cons->prim of (rho, m, E, B_cell);                                */
/*  3. reconstruction (c.5 / R31) of the primitives along each direction;    */
/*  4. at face i-1/2 the normal field of both states is the face value b;    */
/*     face solve c.6-c.10 without GLM (Bm = b): fluxes of rho, m, E and the */
/*     face EMFs (E = -v x B): x-face Ez = -F[By], Ey = F[Bz]; y-face        */
/*     Ex = -F[Bz], Ez = F[Bx]; z-face Ey = -F[Bx], Ex = F[By];              */
/*  5. edge EMFs, arithmetic 4-face average, e.g. at edge      */
/*     (i-1/2, j-1/2): Ez = 0.25 (((Ezx(i,j-1) + Ezx(i,j)) + Ezy(i-1,j)) +   */
/*     Ezy(i,j)) (faces of the first direction of the cyclic pair first);   */
/*  6. S(U): rho, m, E by c.11; face fields by Stokes,                        */
/*     bx -= ly (Ez(j+1/2) - Ez(j-1/2)) - lz (Ey(k+1/2) - Ey(k-1/2)),        */
/*     by -= lz (Ex(k+1/2) - Ex(k-1/2)) - lx (Ez(i+1/2) - Ez(i-1/2)),        */
/*     bz -= lx (Ey(i+1/2) - Ey(i-1/2)) - ly (Ex(j+1/2) - Ex(j-1/2)),        */
/*     each as b - ((la dEa) - (lb dEb)).  The discrete divergence of b is    */
/*     unchanged up to rounding.  N faces per periodic line (counters).       */
/* ------------------------------------------------------------------------ */
#define CTI(i, n) ((((i) % (n)) + (n)) % (n))

static size_t ct_at(const grid_t* G, int f, int64_t i, int64_t j, int64_t k) {
  return (((size_t)f * G->n[2] + CTI(k, G->n[2])) * G->n[1] + CTI(j, G->n[1])) * G->n[0] + CTI(i, G->n[0]);
}

/* cell-centred conservative vector (B from the face average) of cell (i,j,k) */
static void ct_cell_cons(const grid_t* G, const double* U, int64_t i, int64_t j, int64_t k, double* w) {
  for (int f = 0; f < 5; ++f) w[f] = U[ct_at(G, f, i, j, k)];
  w[5] = 0.5 * (U[ct_at(G, 5, i, j, k)] + U[ct_at(G, 5, i + 1, j, k)]);
  w[6] = 0.5 * (U[ct_at(G, 6, i, j, k)] + U[ct_at(G, 6, i, j + 1, k)]);
  w[7] = 0.5 * (U[ct_at(G, 7, i, j, k)] + U[ct_at(G, 7, i, j, k + 1)]);
}

int orc_ct_divb(const orc_config* c, const double* U, double* out) {
  grid_t G;
  int rc = make_grid(c, &G);
  if (rc) return rc;
  for (int64_t k = 0; k < G.n[2]; ++k)
    for (int64_t j = 0; j < G.n[1]; ++j)
      for (int64_t i = 0; i < G.n[0]; ++i)
        out[(k * G.n[1] + j) * G.n[0] + i] =
            ((U[ct_at(&G, 5, i + 1, j, k)] - U[ct_at(&G, 5, i, j, k)]) / G.dx[0] +
             (U[ct_at(&G, 6, i, j + 1, k)] - U[ct_at(&G, 6, i, j, k)]) / G.dx[1]) +
            (U[ct_at(&G, 7, i, j, k + 1)] - U[ct_at(&G, 7, i, j, k)]) / G.dx[2];
  return ORC_OK;
}

static int stage_op_ct(const orc_config* c, const grid_t* G, const double* Uin, double* Out, const double lam[3],
                       int stage, orc_counters* cnt) {
  const int64_t nx = G->n[0], ny = G->n[1], nz = G->n[2];
  const size_t ncell = (size_t)nx * ny * nz;
  const int wz = c->limiter == 2;

  /* validity of the stage input (R16) */
  int64_t first_bad = INT64_MAX;
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        double u[8];
        for (int f = 0; f < 8; ++f) u[f] = Uin[ct_at(G, f, i, j, k)];
        if (bad_cell(u, 8) && interior_linear(G, i, j, k) < first_bad) first_bad = interior_linear(G, i, j, k);
      }
  if (first_bad != INT64_MAX) {
    if (cnt->bad_stage < 0) {
      cnt->bad_stage = stage;
      cnt->first_bad_cell = first_bad;
    }
    return ORC_E_UNPHYSICAL;
  }

  /* 1-2: cell-centred primitives */
  double* V = (double*)calloc(8 * ncell, sizeof(double));
  int64_t floors = 0;
#pragma omp parallel for collapse(2) reduction(+ : floors) schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        double w[8], v[8];
        ct_cell_cons(G, Uin, i, j, k, w);
        floors += orc_cons2prim(c, w, v);
        for (int f = 0; f < 8; ++f) V[ct_at(G, f, i, j, k)] = v[f];
      }
  cnt->p_floors += floors;

  /* 3-4: per direction, reconstruction and the face solve at face i-1/2 of every cell */
  double* F[3];
  int64_t fallbacks = 0, to_hll = 0;
  for (int d = 0; d < 3; ++d) {
    F[d] = (double*)calloc(8 * ncell, sizeof(double));
    double* Vp = (double*)calloc(8 * ncell, sizeof(double));
    double* Vm = (double*)calloc(8 * ncell, sizeof(double));
    int64_t o[3] = {0, 0, 0};
    o[d] = 1;
#pragma omp parallel for collapse(2) reduction(+ : fallbacks) schedule(static)
    for (int64_t k = 0; k < nz; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          double qp[8], qm[8], q0[8];
          for (int f = 0; f < 8; ++f) {
            const double qa = V[ct_at(G, f, i - o[0], j - o[1], k - o[2])];
            const double qb = V[ct_at(G, f, i, j, k)];
            const double qc = V[ct_at(G, f, i + o[0], j + o[1], k + o[2])];
            q0[f] = qb;
            if (wz) {
              const double qaa = V[ct_at(G, f, i - 2 * o[0], j - 2 * o[1], k - 2 * o[2])];
              const double qcc = V[ct_at(G, f, i + 2 * o[0], j + 2 * o[1], k + 2 * o[2])];
              qp[f] = orc_wenoz(qaa, qa, qb, qc, qcc);
              qm[f] = orc_wenoz(qcc, qc, qb, qa, qaa);
            } else {
              const double s = orc_limited_slope(c->limiter, qb - qa, qc - qb);
              qp[f] = qb + 0.5 * s;
              qm[f] = qb - 0.5 * s;
            }
          }
          if (!(qp[0] > 0.0 && qm[0] > 0.0 && qp[4] > 0.0 && qm[4] > 0.0)) {
            for (int f = 0; f < 8; ++f) qp[f] = qm[f] = q0[f];
            fallbacks += 1;
          }
          for (int f = 0; f < 8; ++f) {
            Vp[ct_at(G, f, i, j, k)] = qp[f];
            Vm[ct_at(G, f, i, j, k)] = qm[f];
          }
        }
#pragma omp parallel for collapse(2) reduction(+ : to_hll) schedule(static)
    for (int64_t k = 0; k < nz; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          double vl[8], vr[8], wl[8], wr[8], fn[8], fx[8];
          for (int f = 0; f < 8; ++f) {
            vl[f] = Vp[ct_at(G, f, i - o[0], j - o[1], k - o[2])];
            vr[f] = Vm[ct_at(G, f, i, j, k)];
          }
          const double b = Uin[ct_at(G, 5 + d, i, j, k)]; /* the staggered normal field of face i-1/2 */
          vl[5 + d] = b;
          vr[5 + d] = b;
          to_normal(d, 8, vl, wl);
          to_normal(d, 8, vr, wr);
          to_hll += orc_face_flux(c, wl, wr, 0.0, fn);
          from_normal(d, 8, fn, fx);
          for (int f = 0; f < 8; ++f) F[d][ct_at(G, f, i, j, k)] = fx[f];
        }
    free(Vp);
    free(Vm);
  }
  cnt->plm_fallbacks += fallbacks;
  cnt->hlld_to_hll += to_hll;

  /* 5: edge EMFs.  Ez[i,j,k] at edge (i-1/2, j-1/2, k); Ex[i,j,k] at (i, j-1/2, k-1/2);
   * Ey[i,j,k] at (i-1/2, j, k-1/2).  Face EMFs from the induction fluxes (step 4). */
  double* Ez = (double*)calloc(ncell, sizeof(double));
  double* Ex = (double*)calloc(ncell, sizeof(double));
  double* Ey = (double*)calloc(ncell, sizeof(double));
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const size_t q = ct_at(G, 0, i, j, k);
        /* Ez: x faces (i-1/2) of rows j-1, j; y faces (j-1/2) of columns i-1, i */
        const double ezx0 = -F[0][ct_at(G, 6, i, j - 1, k)], ezx1 = -F[0][ct_at(G, 6, i, j, k)];
        const double ezy0 = F[1][ct_at(G, 5, i - 1, j, k)], ezy1 = F[1][ct_at(G, 5, i, j, k)];
        Ez[q] = 0.25 * (((ezx0 + ezx1) + ezy0) + ezy1);
        /* Ex: y faces (j-1/2) of planes k-1, k; z faces (k-1/2) of rows j-1, j */
        const double exy0 = -F[1][ct_at(G, 7, i, j, k - 1)], exy1 = -F[1][ct_at(G, 7, i, j, k)];
        const double exz0 = F[2][ct_at(G, 6, i, j - 1, k)], exz1 = F[2][ct_at(G, 6, i, j, k)];
        Ex[q] = 0.25 * (((exy0 + exy1) + exz0) + exz1);
        /* Ey: z faces (k-1/2) of columns i-1, i; x faces (i-1/2) of planes k-1, k */
        const double eyz0 = -F[2][ct_at(G, 5, i - 1, j, k)], eyz1 = -F[2][ct_at(G, 5, i, j, k)];
        const double eyx0 = F[0][ct_at(G, 7, i, j, k - 1)], eyx1 = F[0][ct_at(G, 7, i, j, k)];
        Ey[q] = 0.25 * (((eyz0 + eyz1) + eyx0) + eyx1);
      }

  /* 6: update */
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        for (int f = 0; f < 5; ++f) { /* c.11 */
          double r = lam[0] * (F[0][ct_at(G, f, i + 1, j, k)] - F[0][ct_at(G, f, i, j, k)]);
          r = r + lam[1] * (F[1][ct_at(G, f, i, j + 1, k)] - F[1][ct_at(G, f, i, j, k)]);
          r = r + lam[2] * (F[2][ct_at(G, f, i, j, k + 1)] - F[2][ct_at(G, f, i, j, k)]);
          const size_t q = ct_at(G, f, i, j, k);
          Out[q] = Uin[q] - r;
        }
        const size_t e = ct_at(G, 0, i, j, k);
        const double rbx = lam[1] * (Ez[ct_at(G, 0, i, j + 1, k)] - Ez[e]) - lam[2] * (Ey[ct_at(G, 0, i, j, k + 1)] - Ey[e]);
        const double rby = lam[2] * (Ex[ct_at(G, 0, i, j, k + 1)] - Ex[e]) - lam[0] * (Ez[ct_at(G, 0, i + 1, j, k)] - Ez[e]);
        const double rbz = lam[0] * (Ey[ct_at(G, 0, i + 1, j, k)] - Ey[e]) - lam[1] * (Ex[ct_at(G, 0, i, j + 1, k)] - Ex[e]);
        Out[ct_at(G, 5, i, j, k)] = Uin[ct_at(G, 5, i, j, k)] - rbx;
        Out[ct_at(G, 6, i, j, k)] = Uin[ct_at(G, 6, i, j, k)] - rby;
        Out[ct_at(G, 7, i, j, k)] = Uin[ct_at(G, 7, i, j, k)] - rbz;
      }
  free(V);
  for (int d = 0; d < 3; ++d) free(F[d]);
  free(Ez);
  free(Ex);
  free(Ey);
  return ORC_OK;
}

/* one RK step with CT (R30 weights, the same combination for every field) */
static int step_ct(const orc_config* c, const grid_t* G, double* U, const double lam[3], orc_counters* cnt) {
  const size_t n = 8 * (size_t)G->n[0] * G->n[1] * G->n[2];
  double* Ua = (double*)calloc(n, sizeof(double));
  double* Ub = (double*)calloc(n, sizeof(double));
  int rc = stage_op_ct(c, G, U, Ua, lam, 1, cnt); /* U1 = S(U^n) */
  if (rc == ORC_OK && c->stepper == 0) {
    rc = stage_op_ct(c, G, Ua, Ub, lam, 2, cnt);
    if (rc == ORC_OK)
      for (size_t q = 0; q < n; ++q) U[q] = 0.5 * (U[q] + Ub[q]);
  } else if (rc == ORC_OK) {
    const double a2 = 0.75, b2 = 0.25, a3 = 1.0 / 3.0, b3 = 2.0 / 3.0;
    rc = stage_op_ct(c, G, Ua, Ub, lam, 2, cnt);
    if (rc == ORC_OK) {
      for (size_t q = 0; q < n; ++q) Ub[q] = (a2 * U[q]) + (b2 * Ub[q]);
      rc = stage_op_ct(c, G, Ub, Ua, lam, 3, cnt);
    }
    if (rc == ORC_OK)
      for (size_t q = 0; q < n; ++q) U[q] = (a3 * U[q]) + (b3 * Ua[q]);
  }
  free(Ua);
  free(Ub);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* c.11-c.12: one RK step and the GLM damping                                 */
/*   SSP-RK2 (Heun, R2):  U* = S(U^n); U^{n+1} = 0.5 (U^n + S(U*))             */
/*   SSP-RK3 (Shu & Osher 1988; the paper's integrator; reading  */
/*   R30):  U1 = S(U^n); U2 = (3/4) U^n + (1/4) S(U1);                         */
/*          U^{n+1} = (1/3) U^n + (2/3) S(U2), each as (a*U^n) + (b*S)          */
/*   then psi^{n+1} <- psi^{n+1} * damp once per step (R12)                   */
/* ------------------------------------------------------------------------ */
int orc_step(const orc_config* c, double* U, double dt, double ch, orc_counters* cnt) {
  grid_t G;
  int rc = make_grid(c, &G);
  if (rc) return rc;
  if (!(dt > 0.0) || !isfinite(dt)) return ORC_E_ARG;
  if (c->glm && !(ch > 0.0)) return ORC_E_ARG;
  if (c->stepper != 0 && c->stepper != 1) return ORC_E_ARG;
  /* host scalars (R4) */
  double lam[3], dxmin = INFINITY;
  for (int d = 0; d < 3; ++d) {
    lam[d] = dt / G.dx[d];
    if (G.act[d] && G.dx[d] < dxmin) dxmin = G.dx[d];
  }
  const double damp = exp(-((c->glm_alpha * ch) * dt) / dxmin);
  if (c->ct) return step_ct(c, &G, U, lam, cnt);

  const size_t np = padded_size(&G);
  double* Un = (double*)calloc(np, sizeof(double));
  double* Ua = (double*)calloc(np, sizeof(double));
  double* Ub = (double*)calloc(np, sizeof(double));
  load_interior(&G, U, Un);
  rc = stage_op(c, &G, Un, Ua, lam, ch, 1, cnt); /* U* = S(U^n) */
  if (rc == ORC_OK && c->stepper == 0) {
    rc = stage_op(c, &G, Ua, Ub, lam, ch, 2, cnt); /* U** = S(U*) */
    if (rc == ORC_OK) {
      for (int f = 0; f < G.nvar; ++f)
        for (int64_t k = 0; k < G.n[2]; ++k)
          for (int64_t j = 0; j < G.n[1]; ++j)
            for (int64_t i = 0; i < G.n[0]; ++i) {
              const size_t q = P(&G, f, i, j, k);
              double u = 0.5 * (Un[q] + Ub[q]); /* U^{n+1} = (U^n + U**)/2 */
              if (f == 8) u = u * damp;         /* c.12 psi damping, once per step */
              Ub[q] = u;
            }
      store_interior(&G, Ub, U);
    }
  } else if (rc == ORC_OK) {
    const double a2 = 0.75, b2 = 0.25, a3 = 1.0 / 3.0, b3 = 2.0 / 3.0;
    rc = stage_op(c, &G, Ua, Ub, lam, ch, 2, cnt); /* S(U1) */
    if (rc == ORC_OK) {
      for (int f = 0; f < G.nvar; ++f)
        for (int64_t k = 0; k < G.n[2]; ++k)
          for (int64_t j = 0; j < G.n[1]; ++j)
            for (int64_t i = 0; i < G.n[0]; ++i) {
              const size_t q = P(&G, f, i, j, k);
              Ub[q] = (a2 * Un[q]) + (b2 * Ub[q]); /* U2 */
            }
      rc = stage_op(c, &G, Ub, Ua, lam, ch, 3, cnt); /* S(U2) */
    }
    if (rc == ORC_OK) {
      for (int f = 0; f < G.nvar; ++f)
        for (int64_t k = 0; k < G.n[2]; ++k)
          for (int64_t j = 0; j < G.n[1]; ++j)
            for (int64_t i = 0; i < G.n[0]; ++i) {
              const size_t q = P(&G, f, i, j, k);
              double u = (a3 * Un[q]) + (b3 * Ua[q]); /* U^{n+1} */
              if (f == 8) u = u * damp;
              Ua[q] = u;
            }
      store_interior(&G, Ua, U);
    }
  }
  free(Un);
  free(Ua);
  free(Ub);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* c.13 CFL dt and the GLM speed c_h                                          */
/* ------------------------------------------------------------------------ */
int orc_compute_dt(const orc_config* c, const double* U, double* dt, double* ch, orc_counters* cnt) {
  grid_t G;
  int rc = make_grid(c, &G);
  if (rc) return rc;
  double idx[3];
  for (int d = 0; d < 3; ++d) idx[d] = 1.0 / G.dx[d];
  const int nvar = G.nvar;
  const size_t ncell = (size_t)G.n[0] * G.n[1] * G.n[2];
  double M = 0.0, S = 0.0;
  int64_t first_bad = INT64_MAX;
#pragma omp parallel for collapse(2) reduction(max : M, S) reduction(min : first_bad) schedule(static)
  for (int64_t k = 0; k < G.n[2]; ++k)
    for (int64_t j = 0; j < G.n[1]; ++j)
      for (int64_t i = 0; i < G.n[0]; ++i) {
        const size_t lin = (size_t)interior_linear(&G, i, j, k);
        double u[9], v[9];
        for (int f = 0; f < nvar; ++f) u[f] = U[(size_t)f * ncell + lin];
        if (c->ct) ct_cell_cons(&G, U, i, j, k, u); /* CT: B from the face average (R32) */
        if (bad_cell(u, nvar)) {
          if ((int64_t)lin < first_bad) first_bad = (int64_t)lin;
          continue;
        }
        orc_cons2prim(c, u, v); /* floor applies; not counted (c.16) */
        double inv = 0.0, smax = 0.0;
        int first = 1;
        for (int d = 0; d < 3; ++d) {
          if (!G.act[d]) continue;
          const double cf = orc_fast_speed(c->gamma, v[0], v[4], v[5 + d], v[5 + (d + 1) % 3], v[5 + (d + 2) % 3]);
          const double s = fabs(v[1 + d]) + cf;
          if (first) {
            inv = s * idx[d];
            smax = s;
            first = 0;
          } else {
            inv = inv + s * idx[d];
            smax = fmax(smax, s);
          }
        }
        if (inv > M) M = inv;
        if (smax > S) S = smax;
      }
  if (first_bad != INT64_MAX) {
    if (cnt->bad_stage < 0) {
      cnt->bad_stage = 0;
      cnt->first_bad_cell = first_bad;
    }
    return ORC_E_UNPHYSICAL;
  }
  if (!isfinite(M) || !(M > 0.0)) return ORC_E_UNPHYSICAL;
  *dt = c->cfl / M;
  *ch = S;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* c.14 driver loop                                                           */
/* ------------------------------------------------------------------------ */
int orc_run(const orc_config* c, double* U, int64_t nsteps, double t_end, double* dt_log, int64_t* steps_done,
            orc_counters* cnt) {
  double t = 0.0;
  int64_t n = 0;
  int rc = ORC_OK;
  while (n < nsteps && (t_end <= 0.0 || t < t_end)) {
    double dt, ch;
    rc = orc_compute_dt(c, U, &dt, &ch, cnt);
    if (rc) break;
    if (t_end > 0.0 && t + dt > t_end) dt = t_end - t;
    rc = orc_step(c, U, dt, ch, cnt);
    if (rc) break;
    if (dt_log) dt_log[n] = dt;
    t = t + dt;
    n += 1;
  }
  if (steps_done) *steps_done = n;
  return rc;
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
