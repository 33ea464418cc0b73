/*
 * mhd.h — C ABI of libmhd: a B200-native (sm_100a) fp64 ideal-MHD Godunov step.
 *
 * The operation is gPLUTO's data-parallel hot path (arxiv 2510.24175): "boundary
 * exchange/calculation, mapping of the conservative vectors to primitive vectors,
 * reconstruction ... of the cells interfaces values, solving Riemann problem to calculate
 * the fluxes at the interfaces, computing the right hand side of the conservation law",
 * repeated for each Runge-Kutta stage (§3.2), with divergence cleaning
 * in double precision.  The exact recipe (PLM minmod/MC,
 * HLL/HLLD, GLM, SSP-RK2, CFL dt) is DESIGN.md §3; the call set is BASELINE.json's north
 * star ("mhd_create(grid,gamma,cfl,bc), mhd_set_state, mhd_compute_dt, mhd_step,
 * mhd_get_state, mhd_destroy") and SURVEY.md §8(b).
 *
 * Conventions
 *  - extern "C", fp64 only; every call returns an int status (MHD_OK = 0); nothing throws.
 *  - Layout at the ABI: U[f][z][y][x], x fastest, this rank's interior cells only,
 *    nvar = 8 + (glm != 0) fields in the order (rho, mx, my, mz, E, Bx, By, Bz, psi).
 *    Internally the library keeps padded [z][f][y][x] arrays with g ghost planes at each z
 *    end (g = 2 PLM, 3 WENO-Z, one more with CT) and no x/y ghost columns.
 *  - Ownership: the caller owns every host or device buffer it passes; the context owns
 *    the device state it allocates and its NCCL communicator.
 *  - Asynchrony: mhd_step is asynchronous with respect to the host (it enqueues on the
 *    context's stream); mhd_compute_dt, mhd_set_state, mhd_get_state and mhd_get_state_box
 *    synchronise; the *_async calls and mhd_io_join do not.
 *  - Errors are sticky: after MHD_E_UNPHYSICAL, MHD_E_CUDA or MHD_E_NCCL every call except
 *    mhd_get_state / mhd_get_diag / mhd_last_error / mhd_destroy returns MHD_E_STATE until
 *    the next successful mhd_set_state.
 *  - Collective semantics: with nranks > 1, mhd_create, mhd_compute_dt, mhd_step and
 *    mhd_destroy must be called by every rank in the same order (as with NCCL).  A
 *    synchronising call that sees neither progress nor an NCCL error for MHD_NCCL_TIMEOUT_S
 *    seconds (environment, default 600) aborts the communicator and returns the sticky
 *    MHD_E_NCCL (a neighbour rank that died or stopped calling).
 *  - A context is not thread-safe; different contexts are independent.
 */
#ifndef MHD_H
#define MHD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MHD_OK = 0,
  MHD_E_ARG = 1,        /* invalid argument (checked synchronously) */
  MHD_E_STATE = 2,      /* context in a sticky error state, or call out of order */
  MHD_E_CUDA = 3,       /* CUDA runtime error (message in mhd_last_error) */
  MHD_E_NCCL = 4,       /* NCCL error or timeout */
  MHD_E_NOMEM = 5,      /* device allocation failed */
  MHD_E_UNPHYSICAL = 6  /* rho <= 0 or non-finite state (see mhd_diag.first_bad_cell) */
};
enum { MHD_BC_PERIODIC = 0, MHD_BC_OUTFLOW = 1 };
enum { MHD_LIM_MINMOD = 0, MHD_LIM_MC = 1, MHD_LIM_WENOZ = 2 };  /* WENOZ: ghost width 3 (R31) */
enum { MHD_RS_HLL = 0, MHD_RS_HLLD = 1 };
enum { MHD_RK2 = 0, MHD_RK3 = 1 };

/* Global grid. n[d] == 1 makes axis d inactive (1D uses x; 2D uses x, y).  Active axes
 * need n[d] >= 4.  lo < hi on every axis.  DESIGN.md §3.1. */
typedef struct {
  int64_t n[3];
  double lo[3], hi[3];
} mhd_grid;

/* Boundary condition per axis and side.  Periodic must be set on both
 * sides of an axis.  With nranks > 1 the z axis must be periodic (slab ring). */
typedef struct {
  int32_t lo[3], hi[3];
} mhd_bc;

/* Scheme selection.  NULL => MC, HLLD, GLM on, RK2, alpha 0.1, floor 1e-12.
 * GLM is required when two or more axes are active. */
typedef struct {
  int32_t limiter;   /* MHD_LIM_* */
  int32_t riemann;   /* MHD_RS_* */
  int32_t glm;       /* 1: nvar = 9 with the psi field and c_h coupling */
  int32_t stepper;   /* MHD_RK2 (SSP-RK2, 2 stages, 2 state arrays) or MHD_RK3 (Shu-Osher
                        SSP-RK3, the paper's integrator PAPER.md:179; 3 stages, 3 arrays) */
  double glm_alpha;  /* psi damping exp(-alpha*ch*dt/dx_min), R12 */
  double p_floor;    /* pressure floor on primitives (counted), R16 */
  int32_t ct;        /* 1: constrained transport instead of GLM: glm = 0,
                        nvar = 8 with fields 5..7 = face-centred b_x (x-face i-1/2), b_y (j-1/2),
                        b_z (k-1/2); 3D, periodic on every axis, one GPU or z slabs */
  int32_t reserved;
} mhd_scheme;

/* Multi-GPU: z-slab decomposition over nranks GPUs.  NULL => 1 GPU, the
 * current CUDA device.  nranks must divide n[2] with n[2]/nranks >= the ghost width.  nccl_id comes from
 * mhd_nccl_get_unique_id on rank 0, broadcast by the caller (e.g. torch.distributed).
 * transport MHD_TRANSPORT_NCCL: one process per GPU, halos by ncclSend/ncclRecv overlapped
 * with the interior of each stage, dt by ncclAllReduce(max).
 * transport MHD_TRANSPORT_LOCAL: the nranks slabs live in ONE process on one device and are
 * stepped together by mhd_group_step / mhd_group_compute_dt (halos by device copies); it
 * exercises the identical decomposition, kernels and counters without NCCL (tests, 1 GPU). */
enum { MHD_TRANSPORT_NCCL = 0, MHD_TRANSPORT_LOCAL = 1 };
typedef struct {
  int32_t rank, nranks, device, transport;
  uint8_t nccl_id[128];
} mhd_dist;

/* Diagnostics (sums over all ranks after a synchronising call).  Counter ownership is
 * DESIGN.md §3.13. */
typedef struct {
  int64_t steps;          /* mhd_step calls completed */
  int64_t p_floors;       /* (interior cell, stage) pressure floors */
  int64_t plm_fallbacks;  /* (interior cell, direction, stage) first-order fallbacks */
  int64_t hlld_to_hll;    /* (face, stage) HLLD -> HLL fallbacks */
  int64_t first_bad_cell; /* lowest global interior linear index (z*ny+y)*nx+x, or -1 */
  int32_t bad_stage;      /* 0 dt pass or set_state, 1..3 RK stage, -1 none */
  int32_t reserved;
} mhd_diag;

typedef struct mhd_ctx mhd_ctx; /* opaque; created by mhd_create, freed by mhd_destroy */

/* rank 0 only; 128 bytes to broadcast to the other ranks before mhd_create. */
int mhd_nccl_get_unique_id(uint8_t out[128]);

/* Validates the arguments (MHD_E_ARG), plans the slab, allocates the padded state arrays
 * (U^n and U*; a third with MHD_RK3; the scratch of the CT and 3D WENO-Z stages) on the device
 * and, for nranks > 1, creates the NCCL communicator (collective).  gamma > 1, 0 < cfl < 1, each active extent >= 4, nx * ny * 9 < 2^31 (32-bit
 * offsets within a z plane).  *out receives the context (NULL on failure). */
int mhd_create(const mhd_grid* grid, double gamma, double cfl, const mhd_bc* bc,
               const mhd_scheme* scheme, const mhd_dist* dist, mhd_ctx** out);

/* Enqueue all further work on this CUDA stream (cudaStream_t as void*; NULL = default).
 * E.g. torch.cuda.current_stream().cuda_stream. */
int mhd_set_stream(mhd_ctx* ctx, void* cuda_stream);

/* This rank's interior block in global cell coordinates. */
int mhd_local_box(const mhd_ctx* ctx, int64_t off[3], int64_t ext[3]);

/* Bytes of device memory the context's state arrays and records take (the lazily allocated
 * async-I/O staging arrays excluded). */
int mhd_device_bytes(const mhd_ctx* ctx, size_t* bytes);

/* Copy a state in: U is [nvar][ext_z][ext_y][ext_x] (mhd_local_box), host memory when
 * on_device == 0 (pinned host memory makes the copy asynchronous-capable), device memory
 * otherwise.  Validates rho > 0, p > 0 and finiteness on the device (MHD_E_UNPHYSICAL with
 * the first bad cell); clears a sticky error; invalidates the cached dt. Synchronising. */
int mhd_set_state(mhd_ctx* ctx, const double* U, int32_t on_device);

/* Copy the state out, same layout as mhd_set_state.  Synchronising. */
int mhd_get_state(mhd_ctx* ctx, double* U, int32_t on_device);

/* CFL dt of the current state (row a6): dt = cfl / max_cells sum_d
 * (|v_d| + c_f,d)/dx_d, global over ranks (collective); also caches c_h = max_cells
 * max_d (|v_d| + c_f,d) for the next mhd_step.  Reports an unphysical state found by the
 * preceding mhd_step.  Host-synchronising (a 72-byte record stored into mapped host memory). */
int mhd_compute_dt(mhd_ctx* ctx, double* dt);

/* One SSP-RK2 (or RK3) step (rows a1-a5) with the given dt > 0 and the c_h cached
 * by the last mhd_compute_dt on this state (recomputed if the state changed since).
 * Collective with nranks > 1; asynchronous with respect to the host.  Also produces the
 * partial maxima the next mhd_compute_dt needs. */
int mhd_step(mhd_ctx* ctx, double dt);

/* In-process slab group (MHD_TRANSPORT_LOCAL): ctxs[r] is rank r of n, all on the current
 * device and the same stream (ctxs[0]'s).  mhd_group_compute_dt returns the global dt (max
 * over the slabs, exact) and caches c_h in every context; mhd_group_step runs, per RK stage,
 * the halo copies of every slab and then the stage kernel of every slab.  The group runs on
 * ctxs[0]'s stream: destroy the contexts in reverse rank order (rank 0 last). */
int mhd_group_compute_dt(mhd_ctx* const* ctxs, int32_t n, double* dt);
int mhd_group_step(mhd_ctx* const* ctxs, int32_t n, double dt);

/* Halo plan of a z slab (pure host logic, no GPU): the 4 transfers of one RK stage in posting
 * order, each as (peer rank or -1, 0 = send / 1 = recv, first storage plane, plane count);
 * storage planes are 0..nz_loc+2*ghost-1 with `ghost` ghost planes at each end (2 for PLM,
 * 3 for WENOZ, one more with CT).  Returns MHD_E_ARG on inconsistent arguments. */
int mhd_halo_plan(int32_t rank, int32_t nranks, int64_t nz_glob, int32_t z_periodic, int32_t ghost,
                  int32_t plan[4][4]);

/* Device bytes of the context's state arrays (U^n, U*, U2 with RK3, the CT / split-stage
 * scratch), each rounded up to 256 bytes: the size mhd_bind_workspace needs. */
int mhd_workspace_bytes(mhd_ctx* ctx, size_t* bytes);

/* Re-homes the context's state arrays into caller-owned device memory (e.g. a torch tensor from
 * the caching allocator): dev_ptr on the context's device, 256-byte aligned, >= the
 * mhd_workspace_bytes size.  The context frees the arrays it had allocated and only borrows
 * these (mhd_destroy never frees them; the caller keeps them alive until then).  The state is
 * cleared: call mhd_set_state next.  MHD_E_ARG on a short, misaligned or non-device buffer. */
int mhd_bind_workspace(mhd_ctx* ctx, void* dev_ptr, size_t bytes);

/* Pipelined host I/O (pinned host buffers, one full state each, caller-owned; the buffer must
 * stay valid and unmodified until mhd_io_join or the next call that waits on it):
 *  - mhd_set_state_async: starts the host->device copy of U ([nvar][z][y][x], as mhd_set_state)
 *    on the library's upload stream and returns; the next mhd_compute_dt / mhd_step /
 *    mhd_get_state* makes it the state (unpack + validation on the context's stream; an
 *    unphysical cell is reported by the next synchronising call, as a dt-pass error).
 *  - mhd_get_state_async: packs the current state (after all enqueued steps) into a staging
 *    array and starts its device->host copy into U on the download stream; returns at once.
 *  - mhd_io_join: makes the context's stream wait for every started copy (no host wait), so an
 *    event recorded on it afterwards, or cudaStreamSynchronize, covers them.
 * The copies of step n+1's input and step n-1's output overlap step n's kernels.  Two staging
 * arrays (2 x nvar x cells x 8 bytes) are allocated on first use (MHD_E_NOMEM if they do not
 * fit).  Not for in-process slab groups. */
int mhd_set_state_async(mhd_ctx* ctx, const double* U);
int mhd_get_state_async(mhd_ctx* ctx, double* U);
int mhd_io_join(mhd_ctx* ctx);

/* A sub-box of the current state: off/ext in global interior cell coordinates, inside this
 * rank's local block (mhd_local_box), every ext >= 1.  U: [nvar][ext_z][ext_y][ext_x], host
 * (on_device == 0) or device memory, owned by the caller.  Synchronising; MHD_E_ARG for a box
 * outside the block, MHD_E_STATE before mhd_set_state.  (For sampled checks and I/O of states
 * too large to copy out whole.) */
int mhd_get_state_box(mhd_ctx* ctx, const int64_t off[3], const int64_t ext[3], double* U, int32_t on_device);

/* The driver loop in native code (R26 / the oracle's orc_run): up to nsteps of
 * { dt = mhd_compute_dt; with t_end > 0 the step that would pass t_end takes dt = t_end - t;
 * mhd_step(dt); t = t + dt } while t < t_end (t_end <= 0: no end time).  dt_log (host, may be
 * NULL) receives the dts (capacity nsteps), *done the steps taken.  Collective with nranks > 1.
 * Returns the status of the first failing call (the steps before it stay done). */
int mhd_run(mhd_ctx* ctx, int64_t nsteps, double t_end, double* dt_log, int64_t* done);

/* Counters and the unphysical-state record.  On one GPU the counters are read back from the
 * device (synchronising) and include every completed step; with NCCL slabs they are the global
 * sums reduced by the last mhd_compute_dt (the collective). */
int mhd_get_diag(mhd_ctx* ctx, mhd_diag* diag);

/* Last error message of this context (valid until the next call on it); never NULL. */
const char* mhd_last_error(const mhd_ctx* ctx);

/* Frees what the context allocated, including its NCCL communicator.  NULL-safe. */
void mhd_destroy(mhd_ctx* ctx);

/* Test-only: the face solve of n independent face pairs in the
 * normal frame.  VL, VR, F are DEVICE pointers to [n][nvar] rows; ch is the GLM speed.
 * Enqueued on the context's stream, synchronised before return. *n_hll receives the
 * number of HLLD -> HLL fallbacks (may be NULL). */
int mhd_debug_face_flux(mhd_ctx* ctx, const double* VL, const double* VR, int64_t n, double ch,
                        double* F, int64_t* n_hll);

/* Kernel timing (measurement support for bench.py): while enabled, every RK
 * stage (class 0: all its launches — the fused kernel, or with slabs its interior launch, the
 * wait for the halo and its two boundary launches; the five launches of a split WENO-Z or CT
 * stage) and every dt pass (class 1: the dt kernel) is bracketed by one pair of CUDA events on
 * the context's stream.  enable: 0 off; 1 on with room for 1024 pairs; n > 1 on with room for n
 * pairs.  The events are created here, so none is created and nothing synchronises inside a
 * timed loop; units beyond the capacity are not recorded and make mhd_profile_read return
 * MHD_E_STATE (after filling ms/launches with what was recorded).  mhd_profile_read
 * synchronises, adds up the intervals recorded since enable, and returns total milliseconds
 * and recorded units per class.  Enabling resets the totals.  MHD_E_ARG for enable < 0. */
int mhd_profile_enable(mhd_ctx* ctx, int32_t enable);
int mhd_profile_read(mhd_ctx* ctx, double ms[2], int64_t launches[2]);
/* The same totals per class: index 0 the dt pass, 1..3 RK stage 1..3 (RK2 leaves 3 at zero),
 * so per-stage rooflines can be formed (stage 1 and stage 2 move different bytes); index 4 the
 * exposed halo wait of slab runs (per stage: from the end of the interior launch to the halo's
 * completion on the compute stream — the exchange time the interior did not hide; zero on one
 * slab).  The stage intervals include their halo wait. */
int mhd_profile_read_stages(mhd_ctx* ctx, double ms[5], int64_t units[5]);

/* Halo push (the z halo of each RK stage).  With the
 * environment variable MHD_HALO_PUSH=1 at mhd_create, a 3D slab context has each stage's last
 * kernel (the fused stage kernel; the update kernel of the split WENO-Z and CT stages) store
 * its g boundary planes also into the z neighbours' ghost planes of the next stage's input, so
 * the next stage needs no exchange (the fused stage then runs as one launch).  NCCL ranks: the state arrays are NCCL
 * symmetric windows (ncclMemAlloc, ncclCommWindowRegister; every neighbour must be reachable
 * by load/store, i.e. on the same node), and a one-CTA NCCL LSA barrier after every pushing
 * stage orders the ranks; the set-up is agreed over all ranks, and if any step of it fails on
 * any rank no rank pushes (the send/recv exchange stays in use; MHD_HALO_PUSH_FAULT=1..4 injects
 * such a failure, for tests).  In-process slab groups: the
 * neighbour slabs' arrays.  The first stage after a state change (mhd_set_state*,
 * mhd_bind_workspace) exchanges as before.  Results are bitwise those of the exchange.
 * Returns 1 if the context pushes, 0 if not, MHD_E_ARG for a null context.  With pushing NCCL
 * ranks mhd_bind_workspace fails with MHD_E_STATE (the arrays are windows). */
int mhd_halo_push(const mhd_ctx* ctx);

/* Library build identity, e.g. "libmhd sm_100a fused-v1". */
const char* mhd_version(void);

/* Test-only, no context: the branch-free division / reciprocal / square-root sequences of the
 * face solve (mhd_device.cuh; value-neutral) next to the IEEE operators, for
 * n pairs (a[i], b[i]).  a, b: DEVICE [n]; out: DEVICE [n][8] = (fast 1/b, 1.0/b, fast a/b,
 * a/b, fast sqrt(a), sqrt(a), fast |a|/b, |a|/b); ok: DEVICE [n] bit mask of the sequences
 * whose range test passed (bit 0 reciprocal, 1 division, 2 square root, 3 |a|/b — the last
 * defined for positive normal b only) — where a bit is set the fast value must equal the
 * IEEE one bitwise.  Runs on the current device's default stream and
 * synchronises.  MHD_E_ARG on NULL pointers or n < 0, MHD_E_CUDA on a launch error. */
int mhd_debug_fast_ops(const double* a, const double* b, int64_t n, double* out, int32_t* ok);

#ifdef __cplusplus
}
#endif
#endif /* MHD_H */
