// mhd_api.cu — host side of libmhd: the C ABI declared in include/mhd.h.
//
// Owns the device state (padded fp64 arrays U^n, U* [, U2 for RK3] and the CT / split-stage
// scratch; or borrowed from the caller, mhd_bind_workspace), the streams, the z-slab plan and
// the NCCL communicator; sequences one RK step as, per stage,
//   [z ghost planes of the stage input: copies / NCCL halo] -> stage kernel(s)
// (§3.2: boundary exchange, then the offloaded per-cell/per-face work, per
// Runge-Kutta stage; the boundary exchange is the only inter-GPU step), with the
// fused k_stage overlapping the halo with its interior planes; and the CFL reduction as
// k_dt -> ncclAllReduce(max) -> a 72-byte kernel store into mapped host memory.
// Also: pipelined host I/O (async set/get state), the native driver loop (mhd_run), the
// in-process slab group (decomposition tests on one GPU) and kernel timing.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost a pointer test unless a tool is attached

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "../../include/mhd.h"
#include "mhd_kernels.h"

using mhd::DtArgs;
using mhd::StageArgs;
using mhd::StageConsts;

struct mhd_ctx {
  // problem
  int64_t n[3];
  double lo[3], hi[3], dx[3], dxmin;
  int dim, nv;
  int bc_lo[3], bc_hi[3];
  mhd_scheme scheme;
  double gamma, cfl;
  // decomposition
  int rank, nranks, device;
  int nx, ny, nzl, gz;
  long long zoff;
  int up, down;  // ring neighbours along z (-1: none)
  // device state
  double* U0 = nullptr;  // U^n
  double* U1 = nullptr;  // U* (RK2) / U1 (RK3)
  double* U2 = nullptr;  // RK3 only: U2
  double* ctV = nullptr;                          // CT scratch: primitives
  double* ctF[3] = {nullptr, nullptr, nullptr};   // CT scratch: face fluxes
  bool split = false;                             // 3D GLM WENO-Z: the five-launch stage (mhd_split.cu)
  double* spF[3] = {nullptr, nullptr, nullptr};   // split scratch: face fluxes over (nx+1)(ny+1)(nz+1)
  size_t spF_elems = 0;
  cudaStream_t sp_aux[2] = {nullptr, nullptr};  // split stage: the y and z face kernels' streams
  cudaEvent_t sp_ev[3] = {nullptr, nullptr, nullptr};
  size_t arr_elems = 0;
  bool borrowed = false;  // the state arrays live in caller memory (mhd_bind_workspace)
  unsigned long long* dbuf = nullptr;  // [0,1] dt maxima bits, [2..4] counters, [5..8] bad slots, [20] debug
  unsigned long long* dred = nullptr;  // reduction scratch for nranks > 1 (the first 9 entries)
  unsigned long long* hbuf = nullptr;  // pinned host mirror
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  int transport = MHD_TRANSPORT_NCCL;
  // MHD_NCCL_SELF=1 (test/validation): one periodic 3D rank runs the slab schedule with its
  // z ghost planes exchanged through a one-rank NCCL communicator (send/recv to itself) and the
  // dt reduction through ncclAllReduce — the NCCL code path of the multi-GPU run, on one GPU
  bool nccl_self = false;
  cudaStream_t comm_stream = nullptr;            // NCCL halo exchange (overlaps the interior)
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  mhd_ctx* const* group = nullptr;                // MHD_TRANSPORT_LOCAL: the slabs of this group
  // halo push (MHD_HALO_PUSH=1; 3D slabs): each stage's last kernel stores its g boundary
  // planes into the z neighbours' ghost planes of the next stage's input, so the next stage
  // needs no exchange (the fused stage runs as one launch; §8).  NCCL ranks: the arrays are
  // symmetric windows, the peers' arrays plain pointers into NVLink peer memory, and a one-CTA
  // LSA barrier after each pushing stage orders the ranks (a state change must then be made on
  // every rank, as every caller here does); in-process slabs: the peer slabs' arrays, one
  // stream, and a state change of any slab invalidates the pushed planes of all (check_group).
  bool push = false;                              // the transport is set up for pushing
  bool push_valid = false;                        // the next stage's input ghost planes were pushed
  double* peer_dn[3] = {nullptr, nullptr, nullptr};  // down / up neighbour's U0, U1, U2
  double* peer_up[3] = {nullptr, nullptr, nullptr};
  int peer_dn_nz = 0;
  bool nccl_mem = false;                          // U0..U2 from ncclMemAlloc (windows)
  size_t nccl_mem_bytes = 0;
  ncclWindow_t win[3] = {nullptr, nullptr, nullptr};
  std::vector<unsigned char> devcomm;             // ncclDevComm (one LSA barrier), opaque here
  int nsm = 148;
  int kz = 32;
  // cached step state
  double ch = 0.0;
  bool ch_valid = false;
  bool has_state = false;
  int sticky = MHD_OK;
  mhd_diag diag;
  char err[512];
  // pipelined host I/O (mhd_set_state_async / mhd_get_state_async / mhd_io_join): staging
  // arrays in the ABI layout, copied on their own streams so the copies of one step overlap the
  // compute of its neighbours
  double* io_in = nullptr;
  double* io_out = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_in_copied = nullptr, ev_in_free = nullptr, ev_out_packed = nullptr, ev_out_copied = nullptr;
  bool in_pending = false;
  // kernel timing (mhd_profile_*)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_kind;  // one entry per recorded (start, stop) pair: its class
  // per timed class: 0 dt pass, 1..3 RK stage, 4 exposed halo wait (slabs: the compute stream's
  // wait for the halo after the interior launch)
  double prof_ms[5] = {0, 0, 0, 0, 0};
  int64_t prof_n[5] = {0, 0, 0, 0, 0};
  int64_t prof_dropped = 0;
  size_t prof_cap = 0;  // pairs the pool has room for (mhd_profile_enable)
};

namespace {

const char* kVersion = "libmhd sm_100a fused-stage-v2, split WENO-Z and CT stages (fp64, --fmad=false)";

int set_err(mhd_ctx* c, int code, const char* fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof c->err, fmt, ap);
    va_end(ap);
    if (code == MHD_E_UNPHYSICAL || code == MHD_E_CUDA || code == MHD_E_NCCL) c->sticky = code;
  }
  return code;
}

#define CUDA_OR_RETURN(ctx, call)                                                                   \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return set_err(ctx, MHD_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define NCCL_OR_RETURN(ctx, call)                                                                     \
  do {                                                                                                 \
    ncclResult_t r_ = (call);                                                                          \
    if (r_ != ncclSuccess) return set_err(ctx, MHD_E_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

size_t plane_elems(const mhd_ctx* c) { return (size_t)c->nv * c->nx * c->ny; }

// the context runs the slab schedule (a z halo exchange per stage): slabs, or the NCCL self test
bool slabbed(const mhd_ctx* c) { return c->nranks > 1 || c->nccl_self; }
// its halo and reductions go through an NCCL communicator
bool nccl_active(const mhd_ctx* c) {
  return c->comm && ((c->nranks > 1 && c->transport == MHD_TRANSPORT_NCCL) || c->nccl_self);
}
// the role (0 U^n, 1 U*/U1, 2 U2) of one of the context's state arrays
int role_of(const mhd_ctx* c, const double* p) { return p == c->U0 ? 0 : p == c->U1 ? 1 : 2; }
// MHD_HALO_PUSH=1 asks for the halo push (3D slabs: the fused, split WENO-Z and CT stages)
bool push_requested(const mhd_ctx* c) {
  const char* e = getenv("MHD_HALO_PUSH");
  return e && atoi(e) == 1 && c->dim == 3 && (c->nranks > 1 || c->nccl_self);
}

// Host wait for the context's stream.  With NCCL slabs the stream may wait on collectives of
// the other ranks: poll it together with ncclCommGetAsyncError and give up after
// MHD_NCCL_TIMEOUT_S seconds (default 600): the communicator is aborted and the context gets
// the sticky MHD_E_NCCL (a rank that died or stopped calling would otherwise hang every
// synchronising call; SPEC.md:106's neighbour timeout).
int sync_stream(mhd_ctx* c) {
  if (!nccl_active(c)) {
    CUDA_OR_RETURN(c, cudaStreamSynchronize(c->stream));
    return MHD_OK;
  }
  double limit = 600.0;
  if (const char* e = getenv("MHD_NCCL_TIMEOUT_S")) limit = atof(e) > 0.0 ? atof(e) : limit;
  const auto t0 = std::chrono::steady_clock::now();
  for (long spins = 0;; ++spins) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) return MHD_OK;
    if (q != cudaErrorNotReady) return set_err(c, MHD_E_CUDA, "stream: %s", cudaGetErrorString(q));
    ncclResult_t ae = ncclSuccess;
    if (ncclCommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      return set_err(c, MHD_E_NCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ae));
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      return set_err(c, MHD_E_NCCL, "NCCL timeout: no progress for %.0f s (a neighbour rank stopped?)", limit);
    }
    if (spins < 2000) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int check_sticky(mhd_ctx* c) {
  if (c->sticky != MHD_OK)
    return set_err(c, MHD_E_STATE, "context in error state %d; call mhd_set_state to recover", c->sticky);
  return MHD_OK;
}

StageConsts make_consts(const mhd_ctx* c, double dt, double ch) {
  StageConsts k;
  k.gamma = c->gamma;
  k.gm1 = c->gamma - 1.0;
  k.igm1 = 1.0 / (c->gamma - 1.0);
  k.p_floor = c->scheme.p_floor;
  k.hc = 0.5 * ch;
  k.ihc = 0.5 / ch;
  k.ch2 = ch * ch;
  for (int d = 0; d < 3; ++d) k.lam[d] = dt / c->dx[d];
  k.damp = std::exp(-((c->scheme.glm_alpha * ch) * dt) / c->dxmin);  // R12
  k.limiter = c->scheme.limiter;
  return k;
}

// the arrays and epilogue of RK stage `stage` (1-based) of the context's stepper (§3.11):
// RK2: S(U^n) -> U1;  0.5 (U^n + S(U1)) -> U^n
// RK3: S(U^n) -> U1;  (3/4) U^n + (1/4) S(U1) -> U2;  (1/3) U^n + (2/3) S(U2) -> U^n
struct StagePlan {
  double* in;
  double* out;
  int mode;
  double wa, wb;
  int last;
};
int nstages(const mhd_ctx* c) { return c->scheme.stepper == MHD_RK3 ? 3 : 2; }
StagePlan stage_plan(const mhd_ctx* c, int stage) {
  StagePlan p;
  p.wa = p.wb = 0.0;
  if (stage == 1) {
    p.in = c->U0;
    p.out = c->U1;
    p.mode = 0;
  } else if (c->scheme.stepper != MHD_RK3) {
    p.in = c->U1;
    p.out = c->U0;
    p.mode = 1;
  } else if (stage == 2) {
    p.in = c->U1;
    p.out = c->U2;
    p.mode = 2;
    p.wa = 0.75;
    p.wb = 0.25;
  } else {
    p.in = c->U2;
    p.out = c->U0;
    p.mode = 2;
    p.wa = 1.0 / 3.0;
    p.wb = 2.0 / 3.0;
  }
  p.last = stage == nstages(c);
  return p;
}

// a1 (z part).  Halo plan of one stage for a z slab with g ghost planes per side (PLM 2,
// WENO-Z 3): the transfers in posting order as (peer, 0 send / 1 recv, first storage plane,
// planes).  Storage planes: 0..g-1 bottom ghosts, g..nz+g-1 interior, nz+g..nz+2g-1 top
// ghosts.  Sends: top g interior planes -> up, bottom g interior planes -> down; receives:
// bottom ghosts <- down, top ghosts <- up.  The fixed
// posting order (send up, recv down, send down, recv up) pairs correctly with nranks = 2,
// where both neighbours are the same peer (NCCL matches per peer in posting order).
int halo_plan(int rank, int nranks, long long nz_glob, int z_periodic, int g, int plan[4][4]) {
  if (nranks < 1 || rank < 0 || rank >= nranks || g < 1 || nz_glob % nranks != 0 || nz_glob / nranks < g)
    return MHD_E_ARG;
  const int nz = (int)(nz_glob / nranks);
  const int up = (nranks > 1 && (z_periodic || rank < nranks - 1)) ? (rank + 1) % nranks : -1;
  const int down = (nranks > 1 && (z_periodic || rank > 0)) ? (rank + nranks - 1) % nranks : -1;
  const int rows[4][4] = {{up, 0, nz, g}, {down, 1, 0, g}, {down, 0, g, g}, {up, 1, nz + g, g}};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) plan[i][j] = rows[i][j];
  return MHD_OK;
}

// local part of the z ghost fill of array `which` (0: U^n, 1: U*): periodic wrap on one slab,
// zero-gradient copies at outflow domain ends
int fill_z_ghosts_local(mhd_ctx* c, double* U) {
  if (c->dim < 3) return MHD_OK;
  const size_t pe = plane_elems(c), pb = pe * sizeof(double);
  const int nz = c->nzl, g = c->gz;
  auto P = [&](int zs) { return U + (size_t)zs * pe; };
  const bool peri = c->bc_lo[2] == MHD_BC_PERIODIC;
  if (c->nranks == 1 && peri && !c->nccl_self) {  // U[-m] = U[N-m], U[N-1+m] = U[m-1]: two contiguous g-plane blocks
    CUDA_OR_RETURN(c, cudaMemcpyAsync(P(0), P(nz), g * pb, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_OR_RETURN(c, cudaMemcpyAsync(P(nz + g), P(g), g * pb, cudaMemcpyDeviceToDevice, c->stream));
  }
  for (int m = 0; m < g; ++m) {
    if (!peri && c->rank == 0)  // outflow: U[-m] = U[0]
      CUDA_OR_RETURN(c, cudaMemcpyAsync(P(m), P(g), pb, cudaMemcpyDeviceToDevice, c->stream));
    if (!peri && c->rank == c->nranks - 1)  // outflow: U[N-1+m] = U[N-1]
      CUDA_OR_RETURN(c, cudaMemcpyAsync(P(nz + g + m), P(nz + g - 1), pb, cudaMemcpyDeviceToDevice, c->stream));
  }
  return MHD_OK;
}

// exchange part by NCCL on the comm stream (after `ev_ready` on the compute stream); records
// `ev_halo` on the comm stream
int exchange_nccl(mhd_ctx* c, double* U) {
  const size_t pe = plane_elems(c);
  int plan[4][4];
  if (c->nccl_self) {  // the periodic wrap as the two-rank plan with both neighbours = this rank
    const int nz = c->nzl, g = c->gz;
    const int rows[4][4] = {{0, 0, nz, g}, {0, 1, 0, g}, {0, 0, g, g}, {0, 1, nz + g, g}};
    memcpy(plan, rows, sizeof plan);
  } else if (halo_plan(c->rank, c->nranks, c->n[2], c->bc_lo[2] == MHD_BC_PERIODIC, c->gz, plan)) {
    return set_err(c, MHD_E_ARG, "halo plan");
  }
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_ready, c->stream));
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
  NCCL_OR_RETURN(c, ncclGroupStart());
  for (int i = 0; i < 4; ++i) {
    if (plan[i][0] < 0) continue;
    double* p = U + (size_t)plan[i][2] * pe;
    const size_t cnt = (size_t)plan[i][3] * pe;
    if (plan[i][1] == 0)
      NCCL_OR_RETURN(c, ncclSend(p, cnt, ncclFloat64, plan[i][0], c->comm, c->comm_stream));
    else
      NCCL_OR_RETURN(c, ncclRecv(p, cnt, ncclFloat64, plan[i][0], c->comm, c->comm_stream));
  }
  NCCL_OR_RETURN(c, ncclGroupEnd());
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_halo, c->comm_stream));
  return MHD_OK;
}

// exchange part for an in-process group (MHD_TRANSPORT_LOCAL): the same plan and the same
// stream/event protocol as exchange_nccl (comm stream after `ev_ready`, `ev_halo` recorded
// after the last transfer), with each receive a device copy from the peer slab's array of the
// same role.  The group shares one compute stream, so `ev_ready` of a slab follows every launch
// of the previous stage of every slab.
int exchange_local(mhd_ctx* c, int stage) {
  const size_t pe = plane_elems(c), pb = pe * sizeof(double);
  const int g = c->gz;
  int plan[4][4];
  if (halo_plan(c->rank, c->nranks, c->n[2], c->bc_lo[2] == MHD_BC_PERIODIC, g, plan))
    return set_err(c, MHD_E_ARG, "halo plan");
  double* mine = stage_plan(c, stage).in;
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_ready, c->stream));
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
  for (int i = 0; i < 4; ++i) {
    if (plan[i][0] < 0 || plan[i][1] != 1) continue;  // receives only
    const mhd_ctx* peer = c->group[plan[i][0]];
    const double* theirs = stage_plan(peer, stage).in;
    // the peer sends its top g interior planes to its up neighbour, its bottom g to its down
    // neighbour: my bottom ghosts (recv from down) <- down's storage planes nz..nz+g-1; my top
    // ghosts (recv from up) <- up's storage planes g..2g-1
    const int src = (plan[i][2] == 0) ? peer->nzl : g;
    CUDA_OR_RETURN(c, cudaMemcpyAsync(mine + (size_t)plan[i][2] * pe, theirs + (size_t)src * pe, g * pb,
                                      cudaMemcpyDeviceToDevice, c->comm_stream));
  }
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_halo, c->comm_stream));
  return MHD_OK;
}

// the halo of stage `stage`'s input array (stage 1: U^n) on the comm stream, by the context's
// transport; `ev_halo` marks its completion
int exchange(mhd_ctx* c, int stage) {
  return c->transport == MHD_TRANSPORT_LOCAL ? exchange_local(c, stage) : exchange_nccl(c, stage_plan(c, stage).in);
}

// kernel timing: one (start, stop) event pair per timed unit — a whole RK stage (all its
// launches, including the wait for its halo) or a dt pass.  The pool is created by
// mhd_profile_enable; a unit beyond its capacity is not recorded (no event is created and
// nothing synchronises while a timed loop runs).
int prof_begin(mhd_ctx* c, int kind) {
  if (!c->prof) return -1;
  const size_t pair = c->ev_kind.size();
  if (pair >= c->prof_cap) {
    c->prof_dropped += 1;
    return -1;
  }
  cudaEventRecord(c->ev_pool[2 * pair], c->stream);
  c->ev_kind.push_back(kind);
  return (int)pair;
}
void prof_end(mhd_ctx* c, int pair) {
  if (pair >= 0) cudaEventRecord(c->ev_pool[2 * pair + 1], c->stream);
}
void prof_drain(mhd_ctx* c) {
  for (size_t i = 0; i < c->ev_kind.size(); ++i) {
    float ms = 0.f;
    cudaEventSynchronize(c->ev_pool[2 * i + 1]);
    cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]);
    c->prof_ms[c->ev_kind[i]] += ms;
    c->prof_n[c->ev_kind[i]] += 1;
  }
  c->ev_kind.clear();
}

// CT and split WENO-Z: the z ghost planes of stage `stage`'s input complete before the launches
// (periodic copy on one slab; the halo on slabs, waited for on the compute stream: these stages
// have no interior/boundary split)
int whole_fill_ghosts(mhd_ctx* c, int stage) {
  int rc = fill_z_ghosts_local(c, stage_plan(c, stage).in);
  if (rc) return rc;
  if (slabbed(c) && !(c->push && c->push_valid)) {  // (pushed: the neighbours stored them already)
    if ((rc = exchange(c, stage))) return rc;
    CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
  }
  return MHD_OK;
}

// the halo-push pointers of a launch writing `out` (null when the context does not push)
template <typename Args>
void set_push(const mhd_ctx* c, const double* out, Args& a) {
  a.push_dn = a.push_up = nullptr;
  a.push_dn_nz = 0;
  if (!c->push) return;
  const int r = role_of(c, out);
  a.push_dn = c->peer_dn[r];
  a.push_up = c->peer_up[r];
  a.push_dn_nz = c->peer_dn_nz;
}

int run_stage(mhd_ctx* c, int stage, const StageConsts& k, int zb, int ze) {
  const StagePlan sp = stage_plan(c, stage);
  StageArgs a;
  a.Uin = sp.in;
  a.Un = c->U0;
  a.Uout = sp.out;
  a.mode = sp.mode;
  a.wa = sp.wa;
  a.wb = sp.wb;
  a.last = sp.last;
  a.nx = c->nx;
  a.ny = c->ny;
  a.nz_loc = c->nzl;
  a.gz = c->gz;
  a.zoff = c->zoff;
  a.nz_glob = c->n[2];
  a.bcx[0] = c->bc_lo[0];
  a.bcx[1] = c->bc_hi[0];
  a.bcy[0] = c->bc_lo[1];
  a.bcy[1] = c->bc_hi[1];
  a.kz = c->kz;
  a.zb = zb;
  a.ze = ze;
  a.stage = stage;
  a.c = k;
  a.counters = c->dbuf + 2;
  a.bad = c->dbuf + 5;
  set_push(c, sp.out, a);  // the boundary planes also to the neighbours' ghost planes of sp.out
  cudaError_t e = mhd::launch_stage(c->dim, c->nv, c->scheme.riemann, a, c->stream);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "stage %d launch: %s", stage, cudaGetErrorString(e));
  return MHD_OK;
}

// One RK stage of the fused kernel on a slab, the schedule every multi-slab run uses (NCCL
// ranks and the in-process group alike, the boundary exchange overlapped with
// the interior): the local z ghost copies, then the halo on the comm stream while the interior
// planes [g, nz-g) run (their stencil reads no ghost plane), then — after `ev_halo` — the g + g
// boundary planes.  One slab: the ghost copies and one whole launch.  One profiling pair spans
// the stage.
// after a pushing stage: NCCL ranks order the stage against every rank's next one
int push_fence(mhd_ctx* c) {
  if (nccl_active(c)) {
    cudaError_t e = mhd::push_barrier(c->devcomm.data(), c->stream);
    if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "push barrier: %s", cudaGetErrorString(e));
  }
  c->push_valid = true;
  return MHD_OK;
}
int fused_stage_body(mhd_ctx* c, int stage, const StageConsts& k) {
  int rc = fill_z_ghosts_local(c, stage_plan(c, stage).in);
  if (rc) return rc;
  if (slabbed(c) && c->dim == 3 && c->push && c->push_valid) {
    // halo push: the input's ghost planes were stored by the neighbours' previous stage
    // (ordered by the barrier after it): one launch over the whole slab
    const int pr = prof_begin(c, stage);
    if ((rc = run_stage(c, stage, k, 0, c->nzl))) return rc;
    rc = push_fence(c);
    prof_end(c, pr);
    return rc;
  }
  if (slabbed(c) && c->dim == 3) {
    nvtxRangePushA("mhd halo exchange");
    rc = exchange(c, stage);
    nvtxRangePop();
    if (rc) return rc;
    const int pr = prof_begin(c, stage);
    const int g = c->gz;
    const int lo = g < c->nzl ? g : c->nzl, hi = c->nzl - g > lo ? c->nzl - g : lo;
    if ((rc = run_stage(c, stage, k, lo, hi))) return rc;
    // class 4 brackets the wait: its start completes with the interior launch, its end when the
    // halo has landed as well, so the pair measures the exchange time the interior did not hide
    const int pw = prof_begin(c, 4);
    CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
    prof_end(c, pw);
    if ((rc = run_stage(c, stage, k, 0, lo))) return rc;
    if ((rc = run_stage(c, stage, k, hi, c->nzl))) return rc;
    if (c->push && (rc = push_fence(c))) return rc;  // (the first stage after a state change)
    prof_end(c, pr);
    return MHD_OK;
  }
  const int pr = prof_begin(c, stage);
  rc = run_stage(c, stage, k, 0, c->nzl);
  prof_end(c, pr);
  return rc;
}
int fused_stage(mhd_ctx* c, int stage, const StageConsts& k) {
  nvtxRangePushA(stage == 1 ? "mhd stage 1" : stage == 2 ? "mhd stage 2" : "mhd stage 3");
  const int rc = fused_stage_body(c, stage, k);
  nvtxRangePop();
  return rc;
}

// the two auxiliary streams (and fork/join events) on which the split and CT stages run their
// y and z face kernels next to the x one (-1%)
int aux_streams(mhd_ctx* c) {
  if (c->sp_aux[0]) return MHD_OK;
  for (int i = 0; i < 2; ++i) CUDA_OR_RETURN(c, cudaStreamCreateWithFlags(&c->sp_aux[i], cudaStreamNonBlocking));
  for (int i = 0; i < 3; ++i) CUDA_OR_RETURN(c, cudaEventCreateWithFlags(&c->sp_ev[i], cudaEventDisableTiming));
  return MHD_OK;
}

// one CT stage (mhd_ct.cu): prim, three face passes, update with the RK epilogue
int run_ct_stage(mhd_ctx* c, int stage, const StageConsts& k) {
  const StagePlan sp = stage_plan(c, stage);
  mhd::CtArgs a;
  a.Uin = sp.in;
  a.Un = c->U0;
  a.Uout = sp.out;
  a.V = c->ctV;
  for (int d = 0; d < 3; ++d) a.F[d] = c->ctF[d];
  a.nx = c->nx;
  a.ny = c->ny;
  a.nz = c->nzl;
  a.gz = c->gz;
  a.G = c->gz - 1;
  a.zoff = c->zoff;
  a.stage = stage;
  a.mode = sp.mode;
  a.last = sp.last;
  a.wa = sp.wa;
  a.wb = sp.wb;
  a.c = k;
  a.counters = c->dbuf + 2;
  a.bad = c->dbuf + 5;
  set_push(c, sp.out, a);  // (the update kernel's epilogue)
  const int pr = prof_begin(c, stage);
  if (int rc_aux = aux_streams(c)) return rc_aux;
  cudaError_t e = mhd::launch_ct_stage(c->scheme.riemann, a, c->nsm, c->stream, c->sp_aux[0], c->sp_aux[1], c->sp_ev);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "ct stage %d: %s", stage, cudaGetErrorString(e));
  if (c->push)
    if (int rc = push_fence(c)) return rc;
  prof_end(c, pr);
  return MHD_OK;
}

// one WENO-Z stage of the 3D GLM path (mhd_split.cu); the z ghost planes of the input are filled
int run_split_stage(mhd_ctx* c, int stage, const StageConsts& k) {
  const StagePlan sp = stage_plan(c, stage);
  mhd::SplitArgs a;
  a.Uin = sp.in;
  a.Un = c->U0;
  a.Uout = sp.out;
  a.V = c->ctV;
  for (int d = 0; d < 3; ++d) a.F[d] = c->spF[d];
  a.nx = c->nx;
  a.ny = c->ny;
  a.nz = c->nzl;
  a.gz = c->gz;
  a.px = mhd::split_row_pitch(c->nx);
  a.zoff = c->zoff;
  a.nz_glob = c->n[2];
  a.bcx[0] = c->bc_lo[0];
  a.bcx[1] = c->bc_hi[0];
  a.bcy[0] = c->bc_lo[1];
  a.bcy[1] = c->bc_hi[1];
  a.stage = stage;
  a.mode = sp.mode;
  a.last = sp.last;
  a.wa = sp.wa;
  a.wb = sp.wb;
  a.c = k;
  a.counters = c->dbuf + 2;
  a.bad = c->dbuf + 5;
  set_push(c, sp.out, a);  // (the update kernel's epilogue)
  const int pr = prof_begin(c, stage);
  if (int rc_aux = aux_streams(c)) return rc_aux;
  cudaError_t e = mhd::launch_split_stage(c->scheme.riemann, a, c->nsm, c->stream, c->sp_aux[0], c->sp_aux[1], c->sp_ev);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "split stage %d: %s", stage, cudaGetErrorString(e));
  if (c->push)
    if (int rc = push_fence(c)) return rc;
  prof_end(c, pr);
  return MHD_OK;
}

// dt / c_h maxima of U^n into dbuf[0..1], reduced over ranks; reads back dbuf. Synchronising.
int reduce_and_read_(mhd_ctx* c);
int reduce_and_read(mhd_ctx* c) {
  nvtxRangePushA("mhd dt (k_dt + allreduce + read-back)");
  const int rc = reduce_and_read_(c);
  nvtxRangePop();
  return rc;
}
int reduce_and_read_(mhd_ctx* c) {
  CUDA_OR_RETURN(c, cudaMemsetAsync(c->dbuf, 0, 2 * sizeof(unsigned long long), c->stream));
  DtArgs d;
  d.U = c->U0;
  d.nx = c->nx;
  d.ny = c->ny;
  d.nz_loc = c->nzl;
  d.gz = c->gz;
  d.zoff = c->zoff;
  d.gamma = c->gamma;
  d.gm1 = c->gamma - 1.0;
  d.p_floor = c->scheme.p_floor;
  for (int i = 0; i < 3; ++i) d.idx[i] = 1.0 / c->dx[i];
  d.out = c->dbuf;
  d.bad = c->dbuf + 5;
  const int pr = prof_begin(c, 0);
  cudaError_t e = c->scheme.ct ? mhd::launch_ct_dt(d, c->nsm, c->stream) : mhd::launch_dt(c->dim, c->nv, d, c->nsm, c->stream);
  prof_end(c, pr);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "dt launch: %s", cudaGetErrorString(e));
  unsigned long long* src = c->dbuf;
  if (nccl_active(c)) {
    // maxima (exact on the int64 patterns of non-negative doubles), counter sums, bad-slot minima
    NCCL_OR_RETURN(c, ncclGroupStart());
    NCCL_OR_RETURN(c, ncclAllReduce(c->dbuf, c->dred, 2, ncclUint64, ncclMax, c->comm, c->stream));
    NCCL_OR_RETURN(c, ncclAllReduce(c->dbuf + 2, c->dred + 2, 3, ncclUint64, ncclSum, c->comm, c->stream));
    NCCL_OR_RETURN(c, ncclAllReduce(c->dbuf + 5, c->dred + 5, 4, ncclUint64, ncclMin, c->comm, c->stream));
    NCCL_OR_RETURN(c, ncclGroupEnd());
    src = c->dred;
  }
  // (a kernel store into the mapped pinned buffer, not a copy-engine transfer: see k_store_words)
  cudaError_t es = mhd::launch_store_words(c->hbuf, src, 9, c->stream);
  if (es != cudaSuccess) return set_err(c, MHD_E_CUDA, "dt read-back: %s", cudaGetErrorString(es));
  if (int rs = sync_stream(c)) return rs;
  c->diag.p_floors = (int64_t)c->hbuf[2];
  c->diag.plm_fallbacks = (int64_t)c->hbuf[3];
  c->diag.hlld_to_hll = (int64_t)c->hbuf[4];
  // time order of the records: stage 1 and stage 2 of the last step, then the dt pass
  for (int s : {1, 2, 3, 0}) {
    if (c->hbuf[5 + s] != ~0ULL) {
      c->diag.bad_stage = s;
      c->diag.first_bad_cell = (int64_t)c->hbuf[5 + s];
      return set_err(c, MHD_E_UNPHYSICAL, "unphysical state (stage %d, cell %lld)", s, (long long)c->hbuf[5 + s]);
    }
  }
  return MHD_OK;
}

int reset_device_records(mhd_ctx* c) {
  CUDA_OR_RETURN(c, cudaMemsetAsync(c->dbuf, 0, 5 * sizeof(unsigned long long), c->stream));
  CUDA_OR_RETURN(c, cudaMemsetAsync(c->dbuf + 5, 0xff, 4 * sizeof(unsigned long long), c->stream));
  return MHD_OK;
}

int io_setup(mhd_ctx* c) {
  if (c->io_in) return MHD_OK;
  const size_t bytes = plane_elems(c) * (size_t)c->nzl * sizeof(double);
  if (cudaMalloc(&c->io_in, bytes) != cudaSuccess || cudaMalloc(&c->io_out, bytes) != cudaSuccess) {
    cudaGetLastError();
    if (c->io_in) cudaFree(c->io_in);
    c->io_in = c->io_out = nullptr;
    return set_err(c, MHD_E_NOMEM, "async I/O: no room for two staging arrays (%zu bytes each)", bytes);
  }
  CUDA_OR_RETURN(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
  CUDA_OR_RETURN(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&c->ev_in_copied, &c->ev_in_free, &c->ev_out_packed, &c->ev_out_copied})
    CUDA_OR_RETURN(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return MHD_OK;
}

// a pending mhd_set_state_async takes effect on the compute stream: wait for its copy, unpack
// into U^n, validate (reported by the next synchronising call as an unphysical cell of the dt
// pass, like the synchronous path's), reset the per-state records
int apply_input(mhd_ctx* c) {
  if (!c->in_pending) return MHD_OK;
  c->in_pending = false;
  c->push_valid = false;
  c->sticky = MHD_OK;
  c->ch_valid = false;
  c->has_state = false;
  c->diag.first_bad_cell = -1;
  c->diag.bad_stage = -1;
  int rc = reset_device_records(c);
  if (rc) return rc;
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->stream, c->ev_in_copied, 0));
  cudaError_t e = mhd::launch_pack(c->io_in, c->U0, c->nv, c->nx, c->ny, c->nzl, c->gz, 1, c->nsm, c->stream);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "pack: %s", cudaGetErrorString(e));
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_in_free, c->stream));
  e = mhd::launch_validate(c->U0, c->nv, c->nx, c->ny, c->nzl, c->gz, c->zoff, c->gamma - 1.0, c->dbuf + 5, c->nsm,
                           c->stream, c->scheme.ct ? 0 : 1);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "validate: %s", cudaGetErrorString(e));
  c->has_state = true;
  return MHD_OK;
}

// every rank's verdict: the minimum of `ok` over the communicator
int agree(mhd_ctx* c, int ok) {
  int* d = nullptr;
  int h = ok;
  if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return 0;
  bool fine = cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
              ncclAllReduce(d, d, 1, ncclInt32, ncclMin, c->comm, c->stream) == ncclSuccess &&
              cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, c->stream) == cudaSuccess &&
              cudaStreamSynchronize(c->stream) == cudaSuccess;
  cudaFree(d);
  return fine ? h : 0;
}

// NCCL halo push: register the state arrays as symmetric windows, create the device
// communicator with one LSA barrier, and read the z neighbours' window addresses (NVLink peer
// memory; the rank itself for MHD_NCCL_SELF).  Every step is agreed over the ranks, so either
// all push or none does (then the send/recv exchange is used and the windows are released).
int push_setup_nccl(mhd_ctx* c) {
  // MHD_HALO_PUSH_FAULT=k (tests): step k of the set-up fails on this rank (1 the LSA check,
  // 2 the second window, 3 the device communicator, 4 the peer pointers)
  const char* fe = getenv("MHD_HALO_PUSH_FAULT");
  const int fault = fe ? atoi(fe) : 0;
  int ok = agree(c, mhd::lsa_team_size(c->comm) == c->nranks && fault != 1);  // neighbours load/store-accessible
  double* arr[3] = {c->U0, c->U1, c->U2};
  for (int r = 0; r < 3 && ok; ++r) {
    if (!arr[r]) continue;
    const int mine = !(fault == 2 && r == 1) &&
                     ncclCommWindowRegister(c->comm, arr[r], c->nccl_mem_bytes, &c->win[r], NCCL_WIN_COLL_SYMMETRIC) ==
                         ncclSuccess;
    if (!mine) c->win[r] = nullptr;
    ok = agree(c, mine);
  }
  if (ok) {
    c->devcomm.assign(mhd::devcomm_bytes(), 0);
    const bool made = fault != 3 && mhd::devcomm_create(c->comm, c->devcomm.data()) == 0;
    if (!made) c->devcomm.clear();
    ok = agree(c, made);  // (a communicator made here but not elsewhere is destroyed below)
  }
  if (ok) {
    double* p[6];
    void* w[3] = {c->win[0], c->win[1], c->win[2]};
    const int dn = c->nccl_self ? 0 : c->down, up = c->nccl_self ? 0 : c->up;
    ok = agree(c, fault != 4 && mhd::push_peer_pointers(w, dn, up, p, c->stream) == cudaSuccess);
    for (int r = 0; r < 3 && ok; ++r) {
      c->peer_dn[r] = p[2 * r];
      c->peer_up[r] = p[2 * r + 1];
    }
    c->peer_dn_nz = c->nzl;  // (equal slabs)
  }
  if (!ok) {  // release what was set up; the exchange stays the send/recv path
    cudaGetLastError();
    if (!c->devcomm.empty()) mhd::devcomm_destroy(c->comm, c->devcomm.data());
    c->devcomm.clear();
    for (int r = 0; r < 3; ++r)
      if (c->win[r]) ncclCommWindowDeregister(c->comm, c->win[r]);
    for (int r = 0; r < 3; ++r) c->win[r] = nullptr, c->peer_dn[r] = c->peer_up[r] = nullptr;
    return MHD_OK;
  }
  c->push = true;
  return MHD_OK;
}

}  // namespace

extern "C" {

const char* mhd_version(void) { return kVersion; }

int mhd_nccl_get_unique_id(uint8_t out[128]) {
  if (!out) return MHD_E_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return MHD_E_NCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return MHD_OK;
}

int mhd_create(const mhd_grid* grid, double gamma, double cfl, const mhd_bc* bc, const mhd_scheme* scheme,
               const mhd_dist* dist, mhd_ctx** out) {
  if (!out) return MHD_E_ARG;
  *out = nullptr;
  if (!grid || !bc) return MHD_E_ARG;
  if (!(gamma > 1.0) || !std::isfinite(gamma) || !(cfl > 0.0 && cfl < 1.0)) return MHD_E_ARG;
  mhd_ctx* c = new (std::nothrow) mhd_ctx();
  if (!c) return MHD_E_NOMEM;
  c->err[0] = 0;
  memset(&c->diag, 0, sizeof c->diag);
  c->diag.first_bad_cell = -1;
  c->diag.bad_stage = -1;
  int nact = 0;
  bool prefix = true;
  for (int d = 0; d < 3; ++d) {
    c->n[d] = grid->n[d];
    c->lo[d] = grid->lo[d];
    c->hi[d] = grid->hi[d];
    const bool act = grid->n[d] > 1;
    if (grid->n[d] < 1 || (act && grid->n[d] < 4) || !(grid->hi[d] > grid->lo[d]) || grid->n[d] > (1LL << 30)) {
      delete c;
      return MHD_E_ARG;
    }
    if (act && d > 0 && !(grid->n[d - 1] > 1)) prefix = false;
    nact += act;
    c->bc_lo[d] = bc->lo[d];
    c->bc_hi[d] = bc->hi[d];
    if ((bc->lo[d] != MHD_BC_PERIODIC && bc->lo[d] != MHD_BC_OUTFLOW) ||
        (bc->hi[d] != MHD_BC_PERIODIC && bc->hi[d] != MHD_BC_OUTFLOW) ||
        ((bc->lo[d] == MHD_BC_PERIODIC) != (bc->hi[d] == MHD_BC_PERIODIC))) {
      delete c;
      return MHD_E_ARG;
    }
    c->dx[d] = (grid->hi[d] - grid->lo[d]) / (double)grid->n[d];
  }
  if (nact == 0 || !prefix) {  // active axes must be x, then y, then z
    delete c;
    return MHD_E_ARG;
  }
  if (grid->n[0] * grid->n[1] * 9 >= (1LL << 31)) {  // the kernels keep 32-bit offsets within a z plane
    delete c;
    return MHD_E_ARG;
  }
  c->dim = nact;
  c->dxmin = INFINITY;
  for (int d = 0; d < c->dim; ++d) c->dxmin = c->dx[d] < c->dxmin ? c->dx[d] : c->dxmin;
  if (scheme) {
    c->scheme = *scheme;
  } else {
    c->scheme.limiter = MHD_LIM_MC;
    c->scheme.riemann = MHD_RS_HLLD;
    c->scheme.glm = 1;
    c->scheme.stepper = MHD_RK2;
    c->scheme.ct = 0;
    c->scheme.reserved = 0;
    c->scheme.glm_alpha = 0.1;
    c->scheme.p_floor = 1e-12;
  }
  if ((c->scheme.limiter != MHD_LIM_MINMOD && c->scheme.limiter != MHD_LIM_MC && c->scheme.limiter != MHD_LIM_WENOZ) ||
      (c->scheme.riemann != MHD_RS_HLL && c->scheme.riemann != MHD_RS_HLLD) || (c->scheme.glm != 0 && c->scheme.glm != 1) ||
      (c->scheme.stepper != MHD_RK2 && c->scheme.stepper != MHD_RK3) || (c->scheme.ct != 0 && c->scheme.ct != 1) ||
      (c->scheme.ct && (c->scheme.glm || c->dim != 3)) ||
      !(c->scheme.glm_alpha >= 0.0) || !std::isfinite(c->scheme.p_floor) || (c->dim >= 2 && !c->scheme.glm && !c->scheme.ct)) {
    delete c;
    return MHD_E_ARG;
  }
  c->gamma = gamma;
  c->cfl = cfl;
  c->nv = 8 + c->scheme.glm;
  c->rank = dist ? dist->rank : 0;
  c->nranks = dist ? dist->nranks : 1;
  if (c->scheme.ct) {  // CT: periodic on every axis (R32), one GPU or z slabs
    bool ok = true;
    for (int d = 0; d < 3; ++d) ok = ok && c->bc_lo[d] == MHD_BC_PERIODIC;
    if (!ok) {
      delete c;
      return MHD_E_ARG;
    }
  }
  if (dist && dist->transport != MHD_TRANSPORT_NCCL && dist->transport != MHD_TRANSPORT_LOCAL) {
    delete c;
    return MHD_E_ARG;
  }
  if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks || (c->nranks > 1 && c->dim < 3) ||
      (c->n[2] % c->nranks) != 0 || (c->dim == 3 && c->n[2] / c->nranks < 2)) {
    delete c;
    return MHD_E_ARG;
  }
  if (dist && dist->device >= 0) {
    if (cudaSetDevice(dist->device) != cudaSuccess) {
      delete c;
      return MHD_E_CUDA;
    }
  }
  cudaGetDevice(&c->device);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device);
  c->nx = (int)c->n[0];
  c->ny = (int)c->n[1];
  c->nzl = (int)(c->n[2] / c->nranks);
  c->zoff = (long long)c->nzl * c->rank;
  c->gz = c->dim == 3 ? (c->scheme.limiter == MHD_LIM_WENOZ ? 3 : 2) : 0;
  if (c->scheme.ct) c->gz += 1;  // the topmost reconstructed plane needs b_z one plane further
  // 3D GLM WENO-Z runs the five-launch stage (MHD_FUSED_WENOZ=1 keeps the fused kernel, for A/B)
  c->split = c->dim == 3 && !c->scheme.ct && c->scheme.limiter == MHD_LIM_WENOZ && c->nv == mhd::NVS;
  if (const char* f = getenv("MHD_FUSED_WENOZ")) if (atoi(f) == 1) c->split = false;
  if (c->dim == 3 && c->nzl < c->gz) {
    delete c;
    return MHD_E_ARG;
  }
  const bool zper = c->bc_lo[2] == MHD_BC_PERIODIC;
  c->up = (c->nranks > 1 && (zper || c->rank < c->nranks - 1)) ? (c->rank + 1) % c->nranks : -1;
  c->down = (c->nranks > 1 && (zper || c->rank > 0)) ? (c->rank + c->nranks - 1) % c->nranks : -1;
  // z chunk per CTA (3D): the CTAs of one stage launch run in waves of nsm x (resident CTAs
  // per SM); a chunk of kz planes costs ~kz + 1.5 plane-times (the prologue solves one extra z
  // face and converts 2 extra planes).  Pick the chunk count minimising waves x chunk cost
  // (small grids: enough CTAs to fill the GPU), ... (MHD_KZ overrides, for measurements).
  {
    const int ty = mhd::stage_tile_rows(c->dim, c->scheme.limiter);
    const long long tiles = (long long)((c->nx + 31) / 32) * ((c->ny + ty - 1) / ty);
    const long long slots = (long long)c->nsm * mhd::stage_ctas_per_sm(c->dim, c->nv, c->scheme.riemann, c->scheme.limiter);
    long long best_kz = c->nzl;
    double best = 1e300;
    for (long long chunks = 1; chunks <= c->nzl; ++chunks) {
      const long long kz = (c->nzl + chunks - 1) / chunks;
      const long long nch = (c->nzl + kz - 1) / kz;
      const long long waves = (tiles * nch + slots - 1) / slots;
      const double cost = (double)waves * ((double)kz + 1.5);
      if (cost < best - 1e-9) {
        best = cost;
        best_kz = kz;
      }
    }
    // ... capped at 96 planes (measured, profiles/r02_ab_kz.txt): once the grid has several waves
    // of CTAs, shorter chunks let the block scheduler even out the per-CTA time differences
    // (edge tiles, ragged rows) and dispatch the short remainder chunk last, which the uniform
    // model above does not see: 512^3 27.0 -> 25.8 ms per stage, 256^3 3.44 -> 3.39, 1024^3
    // 203.9 -> 202.4 (kz 64-128 all within 1% of 96)
    const long long kz_cap = 96;
    if (best_kz > kz_cap) best_kz = kz_cap;
    const char* env = getenv("MHD_KZ");
    if (env && atoi(env) > 0) best_kz = atoi(env) < c->nzl ? atoi(env) : c->nzl;
    c->kz = (int)(best_kz > 0 ? best_kz : 1);
  }
  c->arr_elems = plane_elems(c) * (size_t)(c->nzl + 2 * c->gz);
  c->transport = dist ? dist->transport : MHD_TRANSPORT_NCCL;
  if (const char* e = getenv("MHD_NCCL_SELF"))
    c->nccl_self = atoi(e) == 1 && c->nranks == 1 && c->dim == 3 && c->bc_lo[2] == MHD_BC_PERIODIC;
  const bool nccl_path = (c->nranks > 1 && c->transport == MHD_TRANSPORT_NCCL) || c->nccl_self;
  const bool want_push = push_requested(c);
  cudaError_t e1 = cudaSuccess, e2 = cudaSuccess;
  if (want_push && nccl_path) {  // the state arrays as NCCL symmetric windows (same size on every rank)
    c->nccl_mem = true;
    c->nccl_mem_bytes = (c->arr_elems * sizeof(double) + (2u << 20) - 1) / (2u << 20) * (2u << 20);
    double** arr[3] = {&c->U0, &c->U1, &c->U2};
    for (int r = 0; r < (c->scheme.stepper == MHD_RK3 ? 3 : 2); ++r)
      if (e1 == cudaSuccess && ncclMemAlloc((void**)arr[r], c->nccl_mem_bytes) != ncclSuccess) e1 = cudaErrorMemoryAllocation;
  } else {
    e1 = cudaMalloc(&c->U0, c->arr_elems * sizeof(double));
    e2 = cudaMalloc(&c->U1, c->arr_elems * sizeof(double));
    if (e1 == cudaSuccess && e2 == cudaSuccess && c->scheme.stepper == MHD_RK3)
      e2 = cudaMalloc(&c->U2, c->arr_elems * sizeof(double));
  }
  cudaError_t e3 = cudaMalloc(&c->dbuf, 24 * sizeof(unsigned long long));
  if (e1 == cudaSuccess && e2 == cudaSuccess && c->scheme.ct) {
    e2 = cudaMalloc(&c->ctV, c->arr_elems * sizeof(double));
    for (int d = 0; d < 3 && e2 == cudaSuccess; ++d) e2 = cudaMalloc(&c->ctF[d], c->arr_elems * sizeof(double));
  }
  if (e1 == cudaSuccess && e2 == cudaSuccess && c->split) {  // V (padded like U) + three face-flux arrays
    c->spF_elems = (size_t)mhd::split_row_pitch(c->nx) * (c->ny + 1) * (size_t)(c->nzl + 1) * mhd::NVS;
    e2 = cudaMalloc(&c->ctV, c->arr_elems * sizeof(double));
    for (int d = 0; d < 3 && e2 == cudaSuccess; ++d) e2 = cudaMalloc(&c->spF[d], c->spF_elems * sizeof(double));
  }
  cudaError_t e4 = cudaMallocHost(&c->hbuf, 24 * sizeof(unsigned long long));
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess) {
    mhd_destroy(c);
    return MHD_E_NOMEM;
  }
  c->dred = c->dbuf + 9;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    mhd_destroy(c);
    return MHD_E_CUDA;
  }
  c->own_stream = true;
  // zero the arrays so ghost planes never hold garbage
  cudaMemsetAsync(c->U0, 0, c->arr_elems * sizeof(double), c->stream);
  cudaMemsetAsync(c->U1, 0, c->arr_elems * sizeof(double), c->stream);
  if (c->U2) cudaMemsetAsync(c->U2, 0, c->arr_elems * sizeof(double), c->stream);
  if (reset_device_records(c) != MHD_OK || cudaStreamSynchronize(c->stream) != cudaSuccess) {
    mhd_destroy(c);
    return MHD_E_CUDA;
  }
  if (c->nranks > 1 || c->nccl_self) {  // the halo's stream and events (NCCL ranks and in-process slabs alike)
    if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming) != cudaSuccess) {
      mhd_destroy(c);
      return MHD_E_CUDA;
    }
  }
  if ((c->nranks > 1 && c->transport == MHD_TRANSPORT_NCCL) || c->nccl_self) {
    ncclUniqueId id;
    if (c->nccl_self) {
      if (ncclGetUniqueId(&id) != ncclSuccess) {
        mhd_destroy(c);
        return MHD_E_NCCL;
      }
    } else {
      memcpy(&id, dist->nccl_id, sizeof id);
    }
    if (ncclCommInitRank(&c->comm, c->nranks, id, c->rank) != ncclSuccess) {
      c->comm = nullptr;
      mhd_destroy(c);
      return MHD_E_NCCL;
    }
  }
  if (want_push && nccl_path) {
    const int rc = push_setup_nccl(c);
    if (rc) {
      mhd_destroy(c);
      return rc;
    }
  } else if (want_push && c->transport == MHD_TRANSPORT_LOCAL) {
    c->push = true;  // (the neighbour slabs' arrays are bound by the group calls)
  }
  *out = c;
  return MHD_OK;
}

int mhd_set_stream(mhd_ctx* c, void* s) {
  if (!c) return MHD_E_ARG;
  if (c->own_stream && c->stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  c->stream = (cudaStream_t)s;
  c->own_stream = false;
  return MHD_OK;
}

int mhd_local_box(const mhd_ctx* c, int64_t off[3], int64_t ext[3]) {
  if (!c || !off || !ext) return MHD_E_ARG;
  off[0] = 0;
  off[1] = 0;
  off[2] = c->zoff;
  ext[0] = c->nx;
  ext[1] = c->ny;
  ext[2] = c->nzl;
  return MHD_OK;
}

// the state arrays of a context in workspace order, with their sizes in doubles
struct WsArray {
  double** p;
  size_t n;
};
static int ws_arrays(mhd_ctx* c, WsArray out[10]) {
  int k = 0;
  out[k++] = {&c->U0, c->arr_elems};
  out[k++] = {&c->U1, c->arr_elems};
  if (c->scheme.stepper == MHD_RK3) out[k++] = {&c->U2, c->arr_elems};
  if (c->scheme.ct || c->split) out[k++] = {&c->ctV, c->arr_elems};
  for (int d = 0; d < 3; ++d) {
    if (c->scheme.ct) out[k++] = {&c->ctF[d], c->arr_elems};
    if (c->split) out[k++] = {&c->spF[d], c->spF_elems};
  }
  return k;
}
static size_t ws_round(size_t n) { return (n * sizeof(double) + 255) / 256 * 256; }

int mhd_workspace_bytes(mhd_ctx* c, size_t* bytes) {
  if (!c || !bytes) return MHD_E_ARG;
  WsArray a[10];
  const int n = ws_arrays(c, a);
  size_t b = 0;
  for (int i = 0; i < n; ++i) b += ws_round(a[i].n);
  *bytes = b;
  return MHD_OK;
}

int mhd_bind_workspace(mhd_ctx* c, void* dev_ptr, size_t bytes) {
  if (!c || !dev_ptr) return MHD_E_ARG;
  size_t need = 0;
  mhd_workspace_bytes(c, &need);
  if (bytes < need || ((uintptr_t)dev_ptr & 255)) return set_err(c, MHD_E_ARG, "workspace: %zu bytes, 256-byte aligned, needed", need);
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, dev_ptr) != cudaSuccess || at.type != cudaMemoryTypeDevice || at.device != c->device) {
    cudaGetLastError();
    return set_err(c, MHD_E_ARG, "workspace: not device memory of the context's device");
  }
  if (c->nccl_mem) return set_err(c, MHD_E_STATE, "workspace: the state arrays are NCCL windows (MHD_HALO_PUSH)");
  CUDA_OR_RETURN(c, cudaStreamSynchronize(c->stream));
  WsArray a[10];
  const int n = ws_arrays(c, a);
  char* p = static_cast<char*>(dev_ptr);
  for (int i = 0; i < n; ++i) {
    if (!c->borrowed && *a[i].p) cudaFree(*a[i].p);
    *a[i].p = reinterpret_cast<double*>(p);
    p += ws_round(a[i].n);
  }
  c->borrowed = true;
  c->push_valid = false;
  c->has_state = false;
  c->in_pending = false;
  c->ch_valid = false;
  CUDA_OR_RETURN(c, cudaMemsetAsync(dev_ptr, 0, need, c->stream));  // ghost planes never hold garbage
  CUDA_OR_RETURN(c, cudaStreamSynchronize(c->stream));
  return MHD_OK;
}

int mhd_device_bytes(const mhd_ctx* c, size_t* bytes) {
  if (!c || !bytes) return MHD_E_ARG;
  *bytes = ((c->U2 ? 3 : 2) + (c->ctV ? (c->split ? 1 : 4) : 0)) * c->arr_elems * sizeof(double) +
           3 * c->spF_elems * sizeof(double) + 24 * sizeof(unsigned long long);
  return MHD_OK;
}

int mhd_set_state(mhd_ctx* c, const double* U, int32_t on_device) {
  if (!c || !U) return MHD_E_ARG;
  c->in_pending = false;  // supersedes a pending mhd_set_state_async
  c->push_valid = false;
  const size_t n = plane_elems(c) * (size_t)c->nzl;
  c->sticky = MHD_OK;
  c->ch_valid = false;
  c->has_state = false;
  c->diag.first_bad_cell = -1;
  c->diag.bad_stage = -1;
  int rc = reset_device_records(c);
  if (rc) return rc;
  const double* src = U;
  if (!on_device) {
    CUDA_OR_RETURN(c, cudaMemcpyAsync(c->U1, U, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    src = c->U1;
  }
  cudaError_t e = mhd::launch_pack(src, c->U0, c->nv, c->nx, c->ny, c->nzl, c->gz, 1, c->nsm, c->stream);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "pack: %s", cudaGetErrorString(e));
  // (CT: the stored 5..7 are face fields, the pressure check of the cell-centred state is left
  // to the first mhd_compute_dt, which floors and counts like every stage)
  e = mhd::launch_validate(c->U0, c->nv, c->nx, c->ny, c->nzl, c->gz, c->zoff, c->gamma - 1.0, c->dbuf + 5, c->nsm,
                           c->stream, c->scheme.ct ? 0 : 1);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "validate: %s", cudaGetErrorString(e));
  CUDA_OR_RETURN(c, cudaMemcpyAsync(c->hbuf + 5, c->dbuf + 5, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                    c->stream));
  if (int rs = sync_stream(c)) return rs;
  if (c->hbuf[5] != ~0ULL) {
    c->diag.bad_stage = 0;
    c->diag.first_bad_cell = (int64_t)c->hbuf[5];
    c->sticky = MHD_E_UNPHYSICAL;
    CUDA_OR_RETURN(c, cudaMemsetAsync(c->dbuf + 5, 0xff, sizeof(unsigned long long), c->stream));
    return set_err(c, MHD_E_UNPHYSICAL, "set_state: unphysical cell %lld (rho<=0, p<=0 or non-finite)",
                   (long long)c->hbuf[5]);
  }
  c->has_state = true;
  return MHD_OK;
}

int mhd_get_state(mhd_ctx* c, double* U, int32_t on_device) {
  if (!c || !U) return MHD_E_ARG;
  int rc = apply_input(c);
  if (rc) return rc;
  if (!c->has_state) return set_err(c, MHD_E_STATE, "no state set");
  const size_t n = plane_elems(c) * (size_t)c->nzl;
  double* dst = on_device ? U : c->U1;
  cudaError_t e = mhd::launch_pack(c->U0, dst, c->nv, c->nx, c->ny, c->nzl, c->gz, 0, c->nsm, c->stream);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "unpack: %s", cudaGetErrorString(e));
  if (!on_device)
    CUDA_OR_RETURN(c, cudaMemcpyAsync(U, c->U1, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (int rs = sync_stream(c)) return rs;
  return MHD_OK;
}

int mhd_set_state_async(mhd_ctx* c, const double* U) {
  if (!c || !U) return MHD_E_ARG;
  if (c->transport == MHD_TRANSPORT_LOCAL && c->nranks > 1)
    return set_err(c, MHD_E_STATE, "in-process slab group: use mhd_set_state");
  int rc = io_setup(c);
  if (rc) return rc;
  const size_t bytes = plane_elems(c) * (size_t)c->nzl * sizeof(double);
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->h2d, c->ev_in_free, 0));  // the previous input was unpacked
  CUDA_OR_RETURN(c, cudaMemcpyAsync(c->io_in, U, bytes, cudaMemcpyHostToDevice, c->h2d));
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_in_copied, c->h2d));
  c->in_pending = true;
  return MHD_OK;
}

int mhd_get_state_async(mhd_ctx* c, double* U) {
  if (!c || !U) return MHD_E_ARG;
  int rc = apply_input(c);
  if (rc) return rc;
  if (!c->has_state) return set_err(c, MHD_E_STATE, "no state set");
  rc = io_setup(c);
  if (rc) return rc;
  const size_t bytes = plane_elems(c) * (size_t)c->nzl * sizeof(double);
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->stream, c->ev_out_copied, 0));  // the previous output left
  cudaError_t e = mhd::launch_pack(c->U0, c->io_out, c->nv, c->nx, c->ny, c->nzl, c->gz, 0, c->nsm, c->stream);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "unpack: %s", cudaGetErrorString(e));
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_out_packed, c->stream));
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->d2h, c->ev_out_packed, 0));
  CUDA_OR_RETURN(c, cudaMemcpyAsync(U, c->io_out, bytes, cudaMemcpyDeviceToHost, c->d2h));
  CUDA_OR_RETURN(c, cudaEventRecord(c->ev_out_copied, c->d2h));
  return MHD_OK;
}

int mhd_io_join(mhd_ctx* c) {
  if (!c) return MHD_E_ARG;
  if (!c->io_in) return MHD_OK;
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->stream, c->ev_in_copied, 0));
  CUDA_OR_RETURN(c, cudaStreamWaitEvent(c->stream, c->ev_out_copied, 0));
  return MHD_OK;
}

int mhd_get_state_box(mhd_ctx* c, const int64_t off[3], const int64_t ext[3], double* U, int32_t on_device) {
  if (!c || !off || !ext || !U) return MHD_E_ARG;
  int rc = apply_input(c);
  if (rc) return rc;
  if (!c->has_state) return set_err(c, MHD_E_STATE, "no state set");
  const int64_t lo[3] = {0, 0, c->zoff}, hi[3] = {c->nx, c->ny, c->zoff + c->nzl};
  for (int d = 0; d < 3; ++d)
    if (ext[d] < 1 || off[d] < lo[d] || off[d] + ext[d] > hi[d]) return set_err(c, MHD_E_ARG, "box outside the local block");
  const size_t pe = plane_elems(c), fs = (size_t)c->nx * c->ny;
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  for (int f = 0; f < c->nv; ++f)
    for (int64_t z = 0; z < ext[2]; ++z) {
      const double* src = c->U0 + (size_t)(off[2] - c->zoff + z + c->gz) * pe + (size_t)f * fs +
                          (size_t)off[1] * c->nx + (size_t)off[0];
      double* dst = U + ((size_t)f * ext[2] + (size_t)z) * (size_t)(ext[1] * ext[0]);
      CUDA_OR_RETURN(c, cudaMemcpy2DAsync(dst, (size_t)ext[0] * sizeof(double), src, (size_t)c->nx * sizeof(double),
                                          (size_t)ext[0] * sizeof(double), (size_t)ext[1], kind, c->stream));
    }
  if (int rs = sync_stream(c)) return rs;
  return MHD_OK;
}

int mhd_compute_dt(mhd_ctx* c, double* dt) {
  if (!c || !dt) return MHD_E_ARG;
  if (c->transport == MHD_TRANSPORT_LOCAL && c->nranks > 1)
    return set_err(c, MHD_E_STATE, "in-process slab group: use mhd_group_compute_dt");
  int rc = apply_input(c);
  if (rc) return rc;
  rc = check_sticky(c);
  if (rc) return rc;
  if (!c->has_state) return set_err(c, MHD_E_STATE, "no state set");
  if (c->scheme.ct && (rc = whole_fill_ghosts(c, 1))) return rc;  // cell-centred B_z needs plane nz
  rc = reduce_and_read(c);
  if (rc) return rc;
  double M, S;
  memcpy(&M, &c->hbuf[0], sizeof M);
  memcpy(&S, &c->hbuf[1], sizeof S);
  if (!std::isfinite(M) || !(M > 0.0)) {
    c->diag.bad_stage = 0;
    return set_err(c, MHD_E_UNPHYSICAL, "non-positive or non-finite signal speed maximum");
  }
  *dt = c->cfl / M;  // R13
  c->ch = S;         // R11
  c->ch_valid = true;
  return MHD_OK;
}

int mhd_step(mhd_ctx* c, double dt) {
  if (!c) return MHD_E_ARG;
  if (c->transport == MHD_TRANSPORT_LOCAL && c->nranks > 1)
    return set_err(c, MHD_E_STATE, "in-process slab group: use mhd_group_step");
  int rc = apply_input(c);
  if (rc) return rc;
  rc = check_sticky(c);
  if (rc) return rc;
  if (!c->has_state) return set_err(c, MHD_E_STATE, "no state set");
  if (!(dt > 0.0) || !std::isfinite(dt)) return set_err(c, MHD_E_ARG, "dt must be positive and finite");
  if (!c->ch_valid) {
    double tmp;
    rc = mhd_compute_dt(c, &tmp);
    if (rc) return rc;
  }
  if (c->scheme.glm && !(c->ch > 0.0)) return set_err(c, MHD_E_ARG, "c_h must be positive");
  const StageConsts k = make_consts(c, dt, c->ch);
  for (int stage = 1; stage <= nstages(c); ++stage) {
    if (c->scheme.ct || c->split) {
      if ((rc = whole_fill_ghosts(c, stage))) return rc;
      if ((rc = c->split ? run_split_stage(c, stage, k) : run_ct_stage(c, stage, k))) return rc;
    } else if ((rc = fused_stage(c, stage, k))) {
      return rc;
    }
  }
  c->ch_valid = false;
  c->diag.steps += 1;
  return MHD_OK;
}

int mhd_run(mhd_ctx* c, int64_t nsteps, double t_end, double* dt_log, int64_t* done) {
  if (!c || nsteps < 0 || !std::isfinite(t_end)) return MHD_E_ARG;
  int64_t n = 0;
  double t = 0.0;
  int rc = MHD_OK;
  while (n < nsteps && (t_end <= 0.0 || t < t_end)) {
    double dt = 0.0;
    if ((rc = mhd_compute_dt(c, &dt))) break;
    if (t_end > 0.0 && t + dt > t_end) dt = t_end - t;  // the last step lands on t_end
    if ((rc = mhd_step(c, dt))) break;
    if (dt_log) dt_log[n] = dt;
    ++n;
    t = t + dt;
  }
  if (done) *done = n;
  return rc;
}

int mhd_halo_plan(int32_t rank, int32_t nranks, int64_t nz_glob, int32_t z_periodic, int32_t ghost,
                  int32_t plan[4][4]) {
  if (!plan) return MHD_E_ARG;
  return halo_plan(rank, nranks, nz_glob, z_periodic, ghost, plan);
}

namespace {
int check_group(mhd_ctx* const* ctxs, int32_t n) {
  if (!ctxs || n < 1) return MHD_E_ARG;
  for (int r = 0; r < n; ++r) {
    mhd_ctx* c = ctxs[r];
    if (!c || c->nranks != n || c->rank != r || (n > 1 && c->transport != MHD_TRANSPORT_LOCAL)) return MHD_E_ARG;
    if (c->sticky != MHD_OK) return set_err(c, MHD_E_STATE, "context in error state %d", c->sticky);
    if (!c->has_state) return set_err(c, MHD_E_STATE, "no state set");
    c->group = ctxs;
    if (c->push) {  // in-process halo push: the neighbour slabs' arrays
      const mhd_ctx* dn = c->down >= 0 ? ctxs[c->down] : nullptr;
      const mhd_ctx* up = c->up >= 0 ? ctxs[c->up] : nullptr;
      if ((dn && !dn->push) || (up && !up->push)) return MHD_E_ARG;
      for (int q = 0; q < 3; ++q) {
        c->peer_dn[q] = dn ? (q == 0 ? dn->U0 : q == 1 ? dn->U1 : dn->U2) : nullptr;
        c->peer_up[q] = up ? (q == 0 ? up->U0 : q == 1 ? up->U1 : up->U2) : nullptr;
      }
      c->peer_dn_nz = dn ? dn->nzl : 0;
    }
    if (r > 0 && c->stream != ctxs[0]->stream) {  // one stream for the whole group
      if (c->own_stream && c->stream) {
        cudaStreamSynchronize(c->stream);
        cudaStreamDestroy(c->stream);
      }
      c->stream = ctxs[0]->stream;
      c->own_stream = false;
    }
  }
  // pushed ghost planes are valid only if no slab's state changed since the last pushing stage
  // (a slab's new interior planes are its neighbours' ghosts): all or none
  bool valid = true;
  for (int r = 0; r < n; ++r) valid = valid && ctxs[r]->push_valid;
  for (int r = 0; r < n; ++r) ctxs[r]->push_valid = valid;
  return MHD_OK;
}
}  // namespace

int mhd_group_compute_dt(mhd_ctx* const* ctxs, int32_t n, double* dt) {
  int rc = check_group(ctxs, n);
  if (rc || !dt) return rc ? rc : MHD_E_ARG;
  double M = 0.0, S = 0.0;
  if (ctxs[0]->scheme.ct) {  // CT: U^n ghost planes (cell-centred B_z of the last plane)
    for (int r = 0; r < n; ++r)
      if ((rc = whole_fill_ghosts(ctxs[r], 1))) return rc;
  }
  for (int r = 0; r < n; ++r) {  // exact maxima: the order over slabs does not matter
    mhd_ctx* c = ctxs[r];
    if ((rc = reduce_and_read(c))) return rc;
    double m, sx;
    memcpy(&m, &c->hbuf[0], sizeof m);
    memcpy(&sx, &c->hbuf[1], sizeof sx);
    M = m > M ? m : M;
    S = sx > S ? sx : S;
  }
  if (!std::isfinite(M) || !(M > 0.0)) return set_err(ctxs[0], MHD_E_UNPHYSICAL, "signal speed maximum");
  *dt = ctxs[0]->cfl / M;
  for (int r = 0; r < n; ++r) {
    ctxs[r]->ch = S;
    ctxs[r]->ch_valid = true;
  }
  return MHD_OK;
}

int mhd_group_step(mhd_ctx* const* ctxs, int32_t n, double dt) {
  int rc = check_group(ctxs, n);
  if (rc) return rc;
  if (!(dt > 0.0) || !std::isfinite(dt)) return MHD_E_ARG;
  for (int r = 0; r < n; ++r)
    if (!ctxs[r]->ch_valid) return set_err(ctxs[r], MHD_E_STATE, "call mhd_group_compute_dt first");
  // per stage, slab by slab, exactly the schedule of an NCCL rank's mhd_step (fused_stage /
  // whole_fill_ghosts with the device-copy halo on each slab's comm stream)
  for (int stage = 1; stage <= nstages(ctxs[0]); ++stage) {
    for (int r = 0; r < n; ++r) {
      mhd_ctx* c = ctxs[r];
      const StageConsts k = make_consts(c, dt, c->ch);
      if (c->scheme.ct || c->split) {
        if ((rc = whole_fill_ghosts(c, stage))) return rc;
        if ((rc = c->split ? run_split_stage(c, stage, k) : run_ct_stage(c, stage, k))) return rc;
      } else if ((rc = fused_stage(c, stage, k))) {
        return rc;
      }
    }
  }
  for (int r = 0; r < n; ++r) {
    ctxs[r]->ch_valid = false;
    ctxs[r]->diag.steps += 1;
  }
  return MHD_OK;
}

int mhd_get_diag(mhd_ctx* c, mhd_diag* d) {
  if (!c || !d) return MHD_E_ARG;
  // one rank (or an in-process group): refresh the counters from the device so that steps
  // since the last mhd_compute_dt are included; with NCCL slabs the global sums are the ones
  // reduced by the last mhd_compute_dt (a collective)
  if ((c->nranks == 1 || c->transport == MHD_TRANSPORT_LOCAL) && c->dbuf && c->stream != (cudaStream_t)-1) {
    if (cudaMemcpyAsync(c->hbuf + 2, c->dbuf + 2, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        c->stream) == cudaSuccess &&
        cudaStreamSynchronize(c->stream) == cudaSuccess) {
      c->diag.p_floors = (int64_t)c->hbuf[2];
      c->diag.plm_fallbacks = (int64_t)c->hbuf[3];
      c->diag.hlld_to_hll = (int64_t)c->hbuf[4];
    }
  }
  *d = c->diag;
  return MHD_OK;
}

const char* mhd_last_error(const mhd_ctx* c) { return c ? c->err : "null context"; }

void mhd_destroy(mhd_ctx* c) {
  if (!c) return;
  if (c->borrowed) {  // caller-owned: forget, never free
    c->U0 = c->U1 = c->U2 = c->ctV = nullptr;
    for (int d = 0; d < 3; ++d) c->ctF[d] = c->spF[d] = nullptr;
  }
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (int i = 0; i < 2; ++i)
    if (c->sp_aux[i]) {
      cudaStreamSynchronize(c->sp_aux[i]);
      cudaStreamDestroy(c->sp_aux[i]);
    }
  for (int i = 0; i < 3; ++i)
    if (c->sp_ev[i]) cudaEventDestroy(c->sp_ev[i]);
  if (c->h2d) cudaStreamSynchronize(c->h2d);
  if (c->d2h) cudaStreamSynchronize(c->d2h);
  if (c->io_in) cudaFree(c->io_in);
  if (c->io_out) cudaFree(c->io_out);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  for (cudaEvent_t e : {c->ev_in_copied, c->ev_in_free, c->ev_out_packed, c->ev_out_copied})
    if (e) cudaEventDestroy(e);
  if (c->comm && !c->devcomm.empty()) mhd::devcomm_destroy(c->comm, c->devcomm.data());
  for (int r = 0; r < 3; ++r)
    if (c->comm && c->win[r]) ncclCommWindowDeregister(c->comm, c->win[r]);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  for (double* u : {c->U0, c->U1, c->U2}) {
    if (!u) continue;
    if (c->nccl_mem) ncclMemFree(u);
    else cudaFree(u);
  }
  if (c->ctV) cudaFree(c->ctV);
  for (int d = 0; d < 3; ++d) {
    if (c->ctF[d]) cudaFree(c->ctF[d]);
    if (c->spF[d]) cudaFree(c->spF[d]);
  }
  if (c->dbuf) cudaFree(c->dbuf);
  if (c->hbuf) cudaFreeHost(c->hbuf);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  delete c;
}

int mhd_halo_push(const mhd_ctx* c) {
  if (!c) return MHD_E_ARG;
  return c->push ? 1 : 0;
}

int mhd_profile_enable(mhd_ctx* c, int32_t enable) {
  if (!c || enable < 0) return MHD_E_ARG;
  if (c->prof) prof_drain(c);
  c->prof = enable != 0;
  // the whole pool up front: none is created (and nothing drains) inside a timed loop
  const size_t pairs = enable > 1 ? (size_t)enable : 1024;
  while (c->prof && c->ev_pool.size() < 2 * pairs) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return set_err(c, MHD_E_CUDA, "profile: event pool");
    c->ev_pool.push_back(e);
  }
  c->prof_cap = pairs;
  c->ev_kind.clear();
  for (int i = 0; i < 5; ++i) {
    c->prof_ms[i] = 0.0;
    c->prof_n[i] = 0;
  }
  c->prof_dropped = 0;
  return MHD_OK;
}

int mhd_profile_read_stages(mhd_ctx* c, double ms[5], int64_t units[5]) {
  if (!c || !ms || !units) return MHD_E_ARG;
  prof_drain(c);
  for (int i = 0; i < 5; ++i) {
    ms[i] = c->prof_ms[i];
    units[i] = c->prof_n[i];
  }
  if (c->prof_dropped)
    return set_err(c, MHD_E_STATE, "profile: %lld timed units exceeded the event pool (mhd_profile_enable capacity)",
                   (long long)c->prof_dropped);
  return MHD_OK;
}

int mhd_profile_read(mhd_ctx* c, double ms[2], int64_t launches[2]) {
  if (!c || !ms || !launches) return MHD_E_ARG;
  double m4[5];
  int64_t n4[5];
  const int rc = mhd_profile_read_stages(c, m4, n4);
  ms[0] = m4[1] + m4[2] + m4[3];
  launches[0] = n4[1] + n4[2] + n4[3];
  ms[1] = m4[0];
  launches[1] = n4[0];
  return rc;
}

int mhd_debug_face_flux(mhd_ctx* c, const double* VL, const double* VR, int64_t n, double ch, double* F,
                        int64_t* n_hll) {
  if (!c || !VL || !VR || !F || n < 0) return MHD_E_ARG;
  if (n == 0) {
    if (n_hll) *n_hll = 0;
    return MHD_OK;
  }
  const StageConsts k = make_consts(c, 1.0, ch);
  unsigned long long* cnt = c->dbuf + 20;
  CUDA_OR_RETURN(c, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c->stream));
  cudaError_t e = mhd::launch_face_flux(c->nv, c->scheme.riemann, VL, VR, n, k, F, cnt, c->stream);
  if (e != cudaSuccess) return set_err(c, MHD_E_CUDA, "face flux: %s", cudaGetErrorString(e));
  CUDA_OR_RETURN(c, cudaMemcpyAsync(c->hbuf + 20, cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_RETURN(c, cudaStreamSynchronize(c->stream));
  if (n_hll) *n_hll = (int64_t)c->hbuf[20];
  return MHD_OK;
}

int mhd_debug_fast_ops(const double* a, const double* b, int64_t n, double* out, int32_t* ok) {
  if (!a || !b || !out || !ok || n < 0) return MHD_E_ARG;
  if (n == 0) return MHD_OK;
  if (mhd::launch_fast_ops(a, b, n, out, ok, 0) != cudaSuccess) return MHD_E_CUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? MHD_OK : MHD_E_CUDA;
}

}  // extern "C"
