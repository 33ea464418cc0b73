// mhd_kernels.cu — sm_100a kernels of the fp64 ideal-MHD Godunov step.
//
// Rows of SURVEY.md §8(a) → kernels:
//   a1 ghost fill   : x/y periodic/outflow resolved by index wrap/clamp inside the stage
//                     kernel (no ghost columns exist); z ghost planes (2 per side, 3 for
//                     WENO-Z) are filled by copies (1 GPU) or NCCL send/recv (slabs) in mhd_api.cu.
//   a2..a5          : k_stage — one fused kernel per RK stage: cons->prim, PLM (or WENO-Z in
//                     1D/2D), GLM pre-solve + HLL/HLLD face fluxes in x/y/z, flux divergence,
//                     the RK epilogue (RK2 average / RK3 weights) and psi damping.  (3D WENO-Z
//                     runs the split stage of mhd_split.cu; CT the stage of mhd_ct.cu.)
//   a6              : k_dt — CFL dt / c_h partial maxima (warp shuffle -> block -> int64
//                     atomicMax on non-negative doubles, exact and order-free).
//
// k_stage design: a CTA owns a 32 x TY column tile (TY cell warps + one edge
// warp) and marches over a chunk of z planes.  Lane = x (coalesced 256 B rows per field),
// warp = y row.  Shared memory holds the primitive plane k with a G-cell x/y halo (Vc), per
// column V+(k) in the z normal frame (Vpz) and the z fluxes of faces k-1/2, k+1/2 (Fz
// ping-pong), the y- and x-face fluxes of plane k (Fy, Fx), and q+ of the cells left of the
// tile (XP).  Each cell is reconstructed once along z (V+ carried) and along x (q+ passed to
// the next lane by shuffle); along y both cells of a face are reconstructed.  Every face is
// solved once per stage except the faces on tile edges in x and y (3%..5%), through one
// inlined, branch-free face solve (a face whose division / sqrt range tests fail is re-solved
// out of line with the IEEE operators, exact_face).
//
// All arithmetic is the recipe of DESIGN.md §3 (see mhd_device.cuh), built with
// --fmad=false so that results equal the CPU oracle bitwise.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <algorithm>
#include <mutex>
#include <climits>
#include <cstdlib>
#include <cstdint>

#include "mhd_device.cuh"
#include "mhd_kernels.h"

namespace mhd {

// ---------------------------------------------------------------------------------------
// indexing helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int wrap_index(int i, int n, int bclo, int bchi) {
  if (i < 0) return bclo == 0 ? (i + n >= 0 ? i + n : ((i % n) + n) % n) : 0;  // (% only when n < halo)
  if (i >= n) return bchi == 0 ? (i - n < n ? i - n : i % n) : n - 1;
  return i;
}

template <int NV>
__device__ __forceinline__ void load_cell(const double* __restrict__ U, size_t plane_off, size_t fstride,
                                          size_t cell, double* u) {
#pragma unroll
  for (int f = 0; f < NV; ++f) u[f] = __ldg(U + plane_off + f * fstride + cell);
}

// the NV fields of one cell: p points at field 0, fields are fs elements apart (the stage
// kernel keeps 32-bit field offsets from a per-plane 64-bit pointer: one IMAD.WIDE per load)
template <typename T>
__device__ __forceinline__ T* opaque(T* p) {  // hides the derivation of p: kept as a 64-bit base
  asm("mov.b64 %0, %0;" : "+l"(p));
  return p;
}
template <int NV>
__device__ __forceinline__ void load_fields(const double* __restrict__ p, int fs, double* u) {
  p = opaque(p);
#pragma unroll
  for (int f = 0; f < NV; ++f) u[f] = __ldg(p + f * fs);
}

__device__ __forceinline__ void prefetch_l2(const double* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l1(const double* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// ---------------------------------------------------------------------------------------
// face-state gathers (shared by the marching path and the exact re-solve below)
// ---------------------------------------------------------------------------------------
// The two states of an x (d = 0) or y (d = 1) face from the primitive plane Vc [NV][PH][PW]:
// face col-1/2 (x) or row-1/2 (y) of the tile cell (row, col); returns the right cell's
// positivity fallback.  Vc is read with the frame permutation folded into the field addresses
// (component n of the normal frame of direction d is field fo[n]); the reconstruction is
// component-wise, so reconstructing in the normal frame is value-identical.
template <int NV, int REC, int PH, int PW, int HY, int G>
__device__ __forceinline__ bool gather_xy(const double* Vc, int d, int row, int col, double* wl, double* wr) {
  constexpr int LIM = REC == 0 ? 0 : 1;
  const int s = (d == 0) ? 1 : PW;
  int fo[NV];
#pragma unroll
  for (int n = 0; n < NV; ++n) fo[n] = n;
  if (d == 1) {
    fo[1] = 2; fo[2] = 3; fo[3] = 1; fo[5] = 6; fo[6] = 7; fo[7] = 5;
  }
  double qa[NV], qb[NV], qc[NV], qd[NV], tmp[NV];
  if constexpr (REC == 2) {  // WENO-Z: left cell from v[-3..1], right cell from v[-2..2]
    double qaa[NV], qdd[NV];
#pragma unroll
    for (int n = 0; n < NV; ++n) {
      const double* base = Vc + (fo[n] * PH + row + HY) * PW + col + G;
      qaa[n] = base[-3 * s];
      qa[n] = base[-2 * s];
      qb[n] = base[-s];
      qc[n] = base[0];
      qd[n] = base[s];
      qdd[n] = base[2 * s];
    }
    weno_side<NV, true>(qaa, qa, qb, qc, qd, wl);        // left cell: V+
    return weno_side<NV, false>(qa, qb, qc, qd, qdd, wr);  // right cell: V-
  } else {
#pragma unroll
    for (int n = 0; n < NV; ++n) {
      const double* base = Vc + (fo[n] * PH + row + HY) * PW + col + G;
      qa[n] = base[-2 * s];
      qb[n] = base[-s];
      qc[n] = base[0];
      qd[n] = base[s];
    }
    plm_cell<NV, LIM>(qa, qb, qc, wl, tmp);       // left cell: V+
    return plm_cell<NV, LIM>(qb, qc, qd, tmp, wr);  // right cell: V-
  }
}

template <int NV>
__device__ __forceinline__ void convert_at(const double* __restrict__ Ucol, int fs, double gm1, double pf,
                                           double* v) {
  double u[NV];
  load_fields<NV>(Ucol, fs, u);
  cons2prim<NV>(u, v, gm1, pf);
}

// The two states of the z face k+1/2 of one column straight from the conservative planes
// (Ucol: the column's cell in storage plane 0): the same conversions and reconstructions as
// the marching path, which carries V+(k) in shared memory instead.
template <int NV, int REC>
__device__ __forceinline__ void gather_z(const double* __restrict__ Ucol, size_t pstride, int fs, int k,
                                         double gm1, double pf, double* wl, double* wr) {
  constexpr int LIM = REC == 0 ? 0 : 1;
  double qp[NV], qm[NV];
  auto at = [&](int kk) { return Ucol + (ptrdiff_t)kk * (ptrdiff_t)pstride; };
  if constexpr (REC == 2) {
    double q0[NV], q1[NV], q2[NV], q3[NV], q4[NV];
    convert_at<NV>(at(k - 2), fs, gm1, pf, q0);
    convert_at<NV>(at(k - 1), fs, gm1, pf, q1);
    convert_at<NV>(at(k), fs, gm1, pf, q2);
    convert_at<NV>(at(k + 1), fs, gm1, pf, q3);
    convert_at<NV>(at(k + 2), fs, gm1, pf, q4);
    weno_cell<NV>(q0, q1, q2, q3, q4, qp, qm);
    to_normal<NV, 2>(qp, wl);
    convert_at<NV>(at(k + 3), fs, gm1, pf, q0);
    weno_cell<NV>(q1, q2, q3, q4, q0, qp, qm);
    to_normal<NV, 2>(qm, wr);
  } else {
    double q0[NV], q1[NV], q2[NV];
    convert_at<NV>(at(k - 1), fs, gm1, pf, q0);
    convert_at<NV>(at(k), fs, gm1, pf, q1);
    convert_at<NV>(at(k + 1), fs, gm1, pf, q2);
    plm_cell<NV, LIM>(q0, q1, q2, qp, qm);
    to_normal<NV, 2>(qp, wl);
    convert_at<NV>(at(k + 2), fs, gm1, pf, q0);
    plm_cell<NV, LIM>(q1, q2, q0, qp, qm);
    to_normal<NV, 2>(qm, wr);
  }
}

// The face solve with the plain IEEE operators, its states re-derived: taken only when a
// range test of the branch-free operators failed (mhd_device.cuh).  Out of line so that the
// marching path keeps neither the inputs of its solve nor a second solve in its registers.
template <int NV>
struct FaceOut {
  double f[NV];
  int fell;
};
template <int NV, int RS, int REC, int PH, int PW, int HY, int G>
__device__ __noinline__ FaceOut<NV> exact_face(StageConsts c, const double* Vc, const double* Ucol, size_t pstride,
                                               int fs, int kplane, int d, int row, int col) {
  double vl[NV], vr[NV];
  if (d == 2) gather_z<NV, REC>(Ucol, pstride, fs, kplane, c.gm1, c.p_floor, vl, vr);
  else gather_xy<NV, REC, PH, PW, HY, G>(Vc, d, row, col, vl, vr);
  FaceOut<NV> o;
  bool unused = true;
  o.fell = face_flux_t<NV, RS, false>(vl, vr, c, o.f, unused);
  return o;
}

// ---------------------------------------------------------------------------------------
// TMA (sm_90+ bulk tensor copies) and mbarrier helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // visible to the async proxy
}
// one plane window [f][PH][PW] of the tensor at (x, y, 0, plane) into smem; completes on mb
__device__ __forceinline__ void tma_load_window(void* dst, const CUtensorMap* map, int x, int y, int plane,
                                                uint64_t* mb, uint32_t bytes) {
  // the CTA's generic-proxy accesses of dst (ordered before this thread by a barrier) happen
  // before the async-proxy writes of the copy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(0), "r"(plane), "r"(smem_u32(mb))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(mb)), "r"(parity)
        : "memory");
  } while (!done);
}

// ---------------------------------------------------------------------------------------
// fused stage kernel
#ifndef MHD_DT_PER_SM
#define MHD_DT_PER_SM 32 // k_dt blocks of 256 per SM in the grid (each loops over its planes)
#endif
#ifndef MHD_ZTMA
#define MHD_ZTMA 1
#endif
#ifndef MHD_EDGE_HALO
#define MHD_EDGE_HALO 1
#endif
#ifndef MHD_SKIP_RAGGED
#define MHD_SKIP_RAGGED 1  // the ragged warps of the last tile row skip the faces no cell needs
#endif
constexpr int kEdgeHalo = MHD_EDGE_HALO;  // TMA window: halo slots converted per edge-warp thread
#ifndef MHD_JOB_UNROLL
#define MHD_JOB_UNROLL 1
#endif
constexpr int kJobUnroll = MHD_JOB_UNROLL;  // face-job loop unrolling (1: one face-solve instance)
#ifndef MHD_OCC3
#define MHD_OCC3 2
#endif
// ---------------------------------------------------------------------------------------
template <int DIM, int NV, int TY, int G>
struct StageSmem {
  static constexpr int TX = 32;
  static constexpr int HY = DIM >= 2 ? G : 0;  // y halo rows (G = stencil half-width: PLM 2, WENOZ 3)
  static constexpr int PW = TX + 2 * G;
  static constexpr int PH = TY + 2 * HY;
  static constexpr int NT = 32 * (TY + 1);  // TY cell warps + 1 edge warp
  static constexpr int nVc = NV * PH * PW;
  static constexpr int nCol = (DIM == 3) ? NV * TY * TX : 0;  // Vpz, Fz[0], Fz[1] each
  static constexpr int nFy = (DIM >= 2) ? NV * (TY + 1) * TX : 0;
  static constexpr int FXP = TX + 2;  // x-flux row pitch (16-byte rows: a TMA box can fill it)
  static constexpr int nFx = NV * TY * FXP;
  static constexpr int nXP = NV * TY;  // q+ (x) of cell x0-1 per row, from the edge warp
  // Fy and Fx start on 128-byte boundaries (TMA destinations of the z staging, MHD_ZTMA)
  static constexpr int oFy = (nVc + 3 * nCol + 15) / 16 * 16;
  static constexpr int oFx = (oFy + nFy + 15) / 16 * 16;
  static constexpr size_t bytes = sizeof(double) * (size_t)(oFx + nFx + nXP);
};

#ifndef MHD_OCCW
#define MHD_OCCW 2
#endif
template <int DIM, int TY, int REC>
struct StageOcc {
  static constexpr int value = DIM == 3 ? (REC == 2 ? MHD_OCCW : MHD_OCC3) : (DIM == 2 ? 2 : 4);
};

// One CTA: a 32 x TY cell tile (TY "cell warps", lane = x) plus one "edge warp", marching
// over the z chunk [kb, ke).  Per plane k each warp runs a short loop of face jobs that all
// go through ONE inlined face solve (the HLLD solve is ~18 KB of SASS; one instance keeps the
// kernel resident in the instruction cache):
//   cell warp ty:  job 0 (3D)  z face k+1/2 of its column   (VL = V+(k) carried in smem)
//                  job 1 (2D+) y face ty-1/2 of its cell
//                  job 3       x face tx-1/2 of its cell
//   edge warp:     job 1 (2D+) the y faces of row TY-1/2 (one per column)
//                  job 2       the x faces of column TX-1/2 (one per row, lanes < TY)
// so every warp runs at most 3 face solves per plane and the per-plane barriers do not wait
// on a straggler.  Fluxes land in shared memory (Fz ping-pong, Fy, Fx); the update then forms
// r = lx dFx + ly dFy + lz dFz (DESIGN.md §3.11 order).
template <int DIM, int NV, int RS, int TY, int REC, bool TMA, bool PUSH = false>
__global__ void __launch_bounds__(32 * (TY + 1), (StageOcc<DIM, TY, REC>::value)) k_stage(const __grid_constant__ StageArgs a) {
  // REC: reconstruction, a compile-time choice (0 PLM minmod, 1 PLM MC, 2 WENO-Z)
  constexpr bool WZ = REC == 2;
  constexpr int LIM = REC == 0 ? 0 : 1;
  constexpr int G = WZ ? 3 : 2;  // reconstruction half-width: PLM 2, WENO-Z 3
  using S = StageSmem<DIM, NV, TY, G>;
  constexpr int TX = S::TX, HY = S::HY, PW = S::PW, PH = S::PH, NT = S::NT;
  constexpr int NC = 32 * TY;        // threads of the cell warps
  extern __shared__ __align__(128) double smem[];
  double* Vc = smem;                 // [NV][PH][PW] primitives of plane k (+halo); TMA destination
  double* Vpz = Vc + S::nVc;         // [NV][NC] V+ (z normal frame) of plane k   (3D)
  double* Fz = Vpz + S::nCol;        // [2][NV][NC] z fluxes, face k+1/2 in Fz[(k+1)&1] (3D)
  double* Fy = smem + S::oFy;        // [NV][TY+1][TX] y-face fluxes of plane k (2D/3D)
  double* Fx = smem + S::oFx;        // [NV][TY][FXP] x-face fluxes of plane k
  double* XP = Fx + S::nFx;          // [NV][TY] q+ along x of cell x0-1 of every row

  const StageConsts& c = a.c;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const bool cellw = ty < TY;        // warp-uniform
  const int nx = a.nx, ny = a.ny, nzl = a.nz_loc;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool own = cellw && gx < nx && gy < ny;
  const int fs = nx * ny;  // field stride in elements (mhd_create bounds nx*ny*nvar below 2^31)
  const size_t pstride = (size_t)fs * NV;
  const int kb = a.zb + blockIdx.z * a.kz;  // this CTA's z chunk inside [zb, ze)
  const int ke = min(kb + a.kz, a.ze);
  // rare events (floors, fallbacks, HLL fallbacks, bad cells) go to shared-memory counters by
  // atomics only when they happen: no registers held for them across the face solves
  __shared__ int s_cnt[3];
  __shared__ unsigned long long s_bad;
  __shared__ uint64_t s_mbar;  // TMA plane-window completion
  __shared__ uint64_t s_mbar2;  // TMA z-staging completion (ZT)
  constexpr bool tma = DIM == 3 && TMA;  // the plane window by TMA (a.tmap) instead of per-thread loads
  // ZT: the own-cell tiles of planes k+1 and k+2 for the z job of iteration k are staged by TMA
  // in the y- and x-flux buffers, which are dead from the end of the previous update (the
  // window barrier) to this plane's y and x jobs (each warp's flux writes cover exactly its own
  // staged rows, which its z job has already read); issued at the top of the iteration.  Same
  // time as the per-thread loads it replaces (3.43 ms; issued after the update behind one more
  // barrier instead: 3.60 ms)
  constexpr bool ZT = tma && !WZ && MHD_ZTMA;
  uint32_t zt_parity = 0;

  uint32_t tma_parity = 0;
  if (tid == 0) {
    s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
    s_bad = ULLONG_MAX;
    if (tma) mbar_init(&s_mbar, 1);
    if (ZT) mbar_init(&s_mbar2, 1);
  }
  __syncthreads();

  // own-cell offset (x, y wrapped for ragged lanes: they compute a valid duplicate and never store)
  const int wx = wrap_index(gx, nx, a.bcx[0], a.bcx[1]);
  const int wy = (DIM >= 2) ? wrap_index(gy, ny, a.bcy[0], a.bcy[1]) : 0;
  const int own_cell = wy * nx + wx;
  // 64-bit pointers to storage plane 0 of the interior; plane k starts k * pstride further
  const double* __restrict__ U0p = a.Uin + (size_t)a.gz * pstride;
  const double* __restrict__ Ucol = U0p + own_cell;  // the own column
  auto at = [&](const double* base, int k) { return base + (ptrdiff_t)k * (ptrdiff_t)pstride; };
  auto glin = [&](int k) -> unsigned long long {
    return ((unsigned long long)(a.zoff + k) * (unsigned long long)ny + (unsigned long long)gy) * (unsigned long long)nx +
           (unsigned long long)gx;
  };
  // conversion of the thread's own cell of plane k; `count` marks the one conversion per
  // (interior cell, stage) that counts floors and checks validity
  auto convert_own = [&](int k, double* v, bool count) {
    double u[NV];
    load_fields<NV>(at(Ucol, k), fs, u);
    const bool fl = cons2prim<NV>(u, v, c.gm1, c.p_floor);
    if (count && own) {
      if (fl) atomicAdd(&s_cnt[0], 1);
      if (bad_state<NV>(u)) atomicMin(&s_bad, glin(k));
    }
  };
  auto convert_any = [&](int k, int x, int y, double* v) {
    double u[NV];
    const int ix = wrap_index(x, nx, a.bcx[0], a.bcx[1]);
    const int iy = (DIM >= 2) ? wrap_index(y, ny, a.bcy[0], a.bcy[1]) : 0;
    load_fields<NV>(at(U0p, k) + (iy * nx + ix), fs, u);
    cons2prim<NV>(u, v, c.gm1, c.p_floor);
  };
  auto store_vc = [&](int r, int col, const double* v) {  // r: 0..PH-1, col: 0..PW-1
#pragma unroll
    for (int f = 0; f < NV; ++f) Vc[(f * PH + r) * PW + col] = v[f];
  };
  // plane k into Vc: interior (cell warps, own cell) + x halo of the TY rows + y halo of the
  // TX columns (all warps)
  auto load_plane = [&](int k, bool count_own) {
    if (cellw) {
      double v[NV];
      convert_own(k, v, count_own);
      store_vc(ty + HY, tx + G, v);
    }
    constexpr int NXH = 2 * G * TY;
    constexpr int NYH = (DIM >= 2) ? 2 * G * TX : 0;
    for (int h = (tid + 32) % NT; h < NXH + NYH; h += NT) {  // the edge warp takes the first slots
      double v[NV];
      if (h < NXH) {
        const int r = h / (2 * G), w = h % (2 * G);
        const int col = (w < G) ? w : TX + w;  // padded cols 0..G-1 | TX+G..TX+2G-1
        convert_any(k, x0 + col - G, y0 + r, v);
        store_vc(r + HY, col, v);
      } else {
        const int j = h - NXH, rs = j / TX, col = j % TX;
        const int r = (rs < G) ? rs : TY + rs;  // padded rows 0..G-1 | TY+G..TY+2G-1
        convert_any(k, x0 + col, y0 + r - HY, v);
        store_vc(r, col + G, v);
      }
    }
  };
  // The same plane window through TMA (3D): one elected thread copies the raw conservative
  // window [f][PH][PW] of plane k (halo and unused corners included; out-of-domain elements
  // zero-filled) into Vc, after the barrier that ends every read of Vc; each slot the face jobs
  // read is then converted in place from shared memory, or — out of the domain (periodic wrap,
  // outflow clamp, ragged tails) — from global memory as in load_plane.  tma_issue and
  // tma_convert bracket work that does not touch Vc (the update), which hides the copy.
  constexpr uint32_t kWinBytes = (uint32_t)(sizeof(double) * NV * PH * PW);
  auto tma_issue = [&](int k) {
    if (tid == 0) tma_load_window(Vc, &a.tmap, x0 - G, y0 - HY, a.gz + k, &s_mbar, kWinBytes);
  };
  constexpr uint32_t kFyBytes = (uint32_t)(sizeof(double) * NV * (TY + 1) * TX);
  constexpr uint32_t kFxBytes = (uint32_t)(sizeof(double) * NV * TY * S::FXP);
  auto zt_issue = [&](int kk) {  // raw U of planes kk (-> Fy) and kk + 1 (-> Fx), own tile
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&s_mbar2)),
                   "r"(kFyBytes + kFxBytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
          ::"r"(smem_u32(Fy)), "l"(&a.tmap_fy), "r"(x0), "r"(y0), "r"(0), "r"(a.gz + kk), "r"(smem_u32(&s_mbar2))
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
          ::"r"(smem_u32(Fx)), "l"(&a.tmap_fx), "r"(x0), "r"(y0), "r"(0), "r"(a.gz + kk + 1), "r"(smem_u32(&s_mbar2))
          : "memory");
    }
  };
  auto convert_slot = [&](int k, int r, int col) {  // Vc slot (r, col): global (x0 + col - G, y0 + r - HY)
    const int x = x0 + col - G, y = y0 + r - HY;
    double v[NV];
    if (x >= 0 && x < nx && y >= 0 && y < ny) {
      double u[NV];
#pragma unroll
      for (int f = 0; f < NV; ++f) u[f] = Vc[(f * PH + r) * PW + col];
      cons2prim<NV>(u, v, c.gm1, c.p_floor);
    } else {
      convert_any(k, x, y, v);
    }
    store_vc(r, col, v);
  };
  auto tma_convert = [&](int k) {
    mbar_wait(&s_mbar, tma_parity);
    tma_parity ^= 1u;
    if (cellw) convert_slot(k, ty + HY, tx + G);
    constexpr int NXH = 2 * G * TY;
    constexpr int NYH = 2 * G * TX;
    // halo slots: the edge warp (no update, no own cell) takes the first 32 * kEdgeHalo, the cell
    // threads the rest
    constexpr int E = 32 * kEdgeHalo < NXH + NYH ? 32 * kEdgeHalo : NXH + NYH;
    auto slot = [&](int h) {
      if (h < NXH) {
        const int r = h / (2 * G), w = h % (2 * G);
        convert_slot(k, r + HY, (w < G) ? w : TX + w);
      } else {
        const int j = h - NXH, rs = j / TX, col = j % TX;
        convert_slot(k, (rs < G) ? rs : TY + rs, col + G);
      }
    };
    if (!cellw) {
#pragma unroll 1
      for (int h = tid - NC; h < E; h += 32) slot(h);
    } else {
#pragma unroll 1
      for (int h = E + tid; h < NXH + NYH; h += NC) slot(h);
    }
  };

  // ------------------------------------------------------------------ prologue
  int kstart = kb;
  if constexpr (DIM == 3) {
    // V+(kb-1) into Vpz; V(kb-1) as the centre of Vc (read by the z job of iteration kb-1)
    if (cellw) {
      double qp[NV], qm[NV], qB[NV];
      if constexpr (WZ) {  // V+(kb-1) from V(kb-3..kb+1)
        double qAA[NV], qA[NV], qC[NV], qCC[NV];
        convert_own(kb - 3, qAA, false);
        convert_own(kb - 2, qA, false);
        convert_own(kb - 1, qB, false);
        convert_own(kb, qC, true);  // the counted conversions of planes kb, kb+1
        convert_own(kb + 1, qCC, kb + 1 < ke);
        weno_cell<NV>(qAA, qA, qB, qC, qCC, qp, qm);
      } else {  // V+(kb-1) from V(kb-2..kb)
        double qA[NV], qC[NV];
        convert_own(kb - 2, qA, false);
        convert_own(kb - 1, qB, false);
        convert_own(kb, qC, true);  // the counted conversion of plane kb
        plm_cell<NV, LIM>(qA, qB, qC, qp, qm);
      }
      double wp[NV];
      to_normal<NV, 2>(qp, wp);  // Vpz is kept in the z normal frame
#pragma unroll
      for (int f = 0; f < NV; ++f) Vpz[f * NC + tid] = wp[f];
      store_vc(ty + HY, tx + G, qB);
    }
    kstart = kb - 1;
    __syncthreads();
  } else {
    load_plane(kb, true);
    __syncthreads();
  }

  // ------------------------------------------------------------------ march over z
  for (int k = kstart; k < ke; ++k) {
    const bool full = k >= kb;  // k = kb-1 (3D) only solves the z face kb-1/2
    if (ZT && full) zt_issue(k + 1);  // (Fx, Fy are dead since the last update's barrier)
    if (DIM == 3 && cellw) {
      // latency hiding, one iteration ahead: the own cell of plane k+G+1 (the z job's newest
      // plane next iteration) into L1 and of plane k+G+2 into L2; U^n of plane k (the update,
      // stage 2) into L1
      const double* p2 = opaque(at(Ucol, k + G + 2 < nzl + a.gz ? k + G + 2 : k));
      const double* p1 = opaque(at(Ucol, k + G + 1 < nzl + a.gz ? k + G + 1 : k));
      const double* pn = opaque(at(a.Un + (size_t)a.gz * pstride + own_cell, k));
#pragma unroll
      for (int f = 0; f < NV; ++f) {
        prefetch_l2(p2 + f * fs);
        prefetch_l1(p1 + f * fs);
        if (full && a.mode != 0) prefetch_l1(pn + f * fs);
      }
    }
    if (full && !cellw) {
      // x faces: the cell warps reconstruct each cell once along x and pass q+ to the next
      // lane; the edge warp supplies q+ of the cells x0-1 (lane 0's left neighbours) and then
      // releases the cell warps' x jobs (named barrier 1: producer arrive / consumer sync)
      if (tx < TY) {
        double qa[NV], qb[NV], qc[NV], qp[NV];
        if constexpr (WZ) {
          double qaa[NV], qcc[NV];
#pragma unroll
          for (int f = 0; f < NV; ++f) {
            const double* base = Vc + (f * PH + tx + HY) * PW + G - 1;
            qaa[f] = base[-2];
            qa[f] = base[-1];
            qb[f] = base[0];
            qc[f] = base[1];
            qcc[f] = base[2];
          }
          weno_side<NV, true>(qaa, qa, qb, qc, qcc, qp);
        } else {
          double qm[NV];
#pragma unroll
          for (int f = 0; f < NV; ++f) {
            const double* base = Vc + (f * PH + tx + HY) * PW + G - 1;
            qa[f] = base[-1];
            qb[f] = base[0];
            qc[f] = base[1];
          }
          plm_cell<NV, LIM>(qa, qb, qc, qp, qm);
        }
#pragma unroll
        for (int f = 0; f < NV; ++f) XP[f * TY + tx] = qp[f];
      }
      asm volatile("bar.arrive 1, %0;" ::"r"(NT) : "memory");
    }
#pragma unroll kJobUnroll
    for (int job = 0; job <= 3; ++job) {
      // ---- select the face of this job (warp-uniform activity)
      int d = 0, row = ty, col = tx;
      bool active, cnt_right = false, cnt_face = false;
      // (MHD_SKIP_RAGGED: a cell warp whose row lies beyond ny — the ragged last tile row — solves
      // only the y face on the domain's top edge, the one face a valid cell needs)
      const bool ragged = MHD_SKIP_RAGGED && cellw && gy >= ny;  // warp-uniform
      if (job == 0) {
        active = DIM == 3 && cellw && !ragged;
        d = 2;
        cnt_right = own && k + 1 < ke;
        cnt_face = own && (k + 1 < ke || a.zoff + k + 1 == a.nz_glob);
      } else if (job == 1) {
        active = DIM >= 2 && full && !(ragged && gy > ny) && (cellw || !MHD_SKIP_RAGGED || y0 + TY <= ny);
        d = 1;
        if (cellw) {
          cnt_right = own;
          cnt_face = own || (gy == ny && gx < nx);
        } else {  // edge warp: y faces of row TY - 1/2
          row = TY;
          cnt_face = (y0 + TY == ny) && gx < nx;
        }
      } else if (job == 2) {  // edge warp: x faces of column TX - 1/2
        active = !cellw && full && tx < TY;
        d = 0;
        row = tx;
        col = TX;
        cnt_face = (x0 + TX == nx) && (y0 + tx < ny);
      } else {
        active = cellw && full && !ragged;
        d = 0;
        cnt_right = own;
        cnt_face = own || (gx == nx && gy < ny);
        if (ragged && full) {  // (the x job's named barrier with the edge warp still needs this warp)
          asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
          continue;
        }
      }
      if (!active) continue;
      // ---- gather the two face states (normal frame)
      double wl[NV], wr[NV];
      {
        bool fb;
        if (job == 0) {
          double q0[NV], q1[NV], q2[NV], qp[NV], qm[NV];
#pragma unroll
          for (int f = 0; f < NV; ++f) {
            q0[f] = Vc[(f * PH + ty + HY) * PW + tx + G];
            wl[f] = Vpz[f * NC + tid];
          }
          const bool staged = ZT && k != kstart;  // warp-uniform
          if (staged) mbar_wait(&s_mbar2, zt_parity);
          if (staged && own) {
            double u[NV];
#pragma unroll
            for (int f = 0; f < NV; ++f) u[f] = Fy[(f * (TY + 1) + ty) * TX + tx];
            cons2prim<NV>(u, q1, c.gm1, c.p_floor);
          } else {
            convert_own(k + 1, q1, false);
          }
          if constexpr (WZ) {  // cell k+1 from V(k-1..k+3); plane k+3 is first touched here
            double qm1[NV], q3[NV];
            convert_own(k - 1, qm1, false);
            convert_own(k + 2, q2, false);
            convert_own(k + 3, q3, k + 3 >= kb && k + 3 < ke);
            fb = weno_cell<NV>(qm1, q0, q1, q2, q3, qp, qm);
          } else {  // cell k+1 from V(k..k+2); plane k+2 is first touched here
            if (staged && own) {
              double u[NV];
#pragma unroll
              for (int f = 0; f < NV; ++f) u[f] = Fx[(f * TY + ty) * S::FXP + tx];
              const bool fl = cons2prim<NV>(u, q2, c.gm1, c.p_floor);
              if (k + 2 >= kb && k + 2 < ke) {  // the counted conversion of plane k+2 (convert_own's rule)
                if (fl) atomicAdd(&s_cnt[0], 1);
                if (bad_state<NV>(u)) atomicMin(&s_bad, glin(k + 2));
              }
            } else {
              convert_own(k + 2, q2, k + 2 >= kb && k + 2 < ke);
            }
            if (staged) zt_parity ^= 1u;
            fb = plm_cell<NV, LIM>(q0, q1, q2, qp, qm);
          }
          double wp[NV];
          to_normal<NV, 2>(qp, wp);
          to_normal<NV, 2>(qm, wr);
#pragma unroll
          for (int f = 0; f < NV; ++f) Vpz[f * NC + tid] = wp[f];
        } else if (job == 3) {
          // x face tx-1/2 (cell warps): own cell reconstructed once, left state from lane tx-1
          double qa[NV], qb[NV], qc[NV], qp[NV];
          if constexpr (WZ) {
            double qaa[NV], qcc[NV];
#pragma unroll
            for (int n = 0; n < NV; ++n) {
              const double* base = Vc + (n * PH + row + HY) * PW + col + G;
              qaa[n] = base[-2];
              qa[n] = base[-1];
              qb[n] = base[0];
              qc[n] = base[1];
              qcc[n] = base[2];
            }
            fb = weno_cell<NV>(qaa, qa, qb, qc, qcc, qp, wr);
          } else {
#pragma unroll
            for (int n = 0; n < NV; ++n) {
              const double* base = Vc + (n * PH + row + HY) * PW + col + G;
              qa[n] = base[-1];
              qb[n] = base[0];
              qc[n] = base[1];
            }
            fb = plm_cell<NV, LIM>(qa, qb, qc, qp, wr);
          }
          asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");  // XP written by the edge warp
#pragma unroll
          for (int n = 0; n < NV; ++n) {
            const double nb = __shfl_up_sync(0xffffffffu, qp[n], 1);
            wl[n] = (tx == 0) ? XP[n * TY + ty] : nb;
          }
        } else {
          fb = gather_xy<NV, REC, PH, PW, HY, G>(Vc, d, row, col, wl, wr);
        }
        if (fb && cnt_right) atomicAdd(&s_cnt[1], 1);
      }
      // ---- the face solve (single instance, branch-free division / square root)
      double fn[NV];
      bool ok = true;
      int fell = face_flux_t<NV, RS, true>(wl, wr, c, fn, ok);
      if (!ok) {
        // a range test of the branch-free operators failed (rare): the plain operators on the
        // same face, its two states re-derived from shared memory (x, y) or the planes (z)
        const FaceOut<NV> o = exact_face<NV, RS, REC, PH, PW, HY, G>(c, Vc, Ucol, pstride, fs, k, d, row, col);
#pragma unroll
        for (int f = 0; f < NV; ++f) fn[f] = o.f[f];
        fell = o.fell;
      }
      if (fell && cnt_face) atomicAdd(&s_cnt[2], 1);
      // ---- scatter (back to x,y,z components through the same field map)
      if (job == 0) {
        double fz[NV];
        from_normal<NV, 2>(fn, fz);
        double* dst = Fz + ((k + 1) & 1) * S::nCol;
#pragma unroll
        for (int f = 0; f < NV; ++f) dst[f * NC + tid] = fz[f];
      } else if (d == 1) {  // y frame (y, z, x): normal components n -> fields (0, 2, 3, 1, 4, 6, 7, 5, 8)
        double fy[NV];
        from_normal<NV, 1>(fn, fy);
#pragma unroll
        for (int f = 0; f < NV; ++f) Fy[(f * (TY + 1) + row) * TX + col] = fy[f];
      } else {
#pragma unroll
        for (int n = 0; n < NV; ++n) Fx[(n * TY + row) * S::FXP + col] = fn[n];
      }
    }
    if (!full) {  // 3D prologue iteration: bring plane kb into Vc
      __syncthreads();
      if (tma) {
        tma_issue(kb);
        tma_convert(kb);
      } else {
        load_plane(kb, false);
      }
      __syncthreads();
      continue;
    }
    // ---- advance the plane window (3D) and update.  After this barrier every read of Vc (the
    // face jobs) is done, so plane k+1 is loaded first: its conversions' L2 latency overlaps the
    // update, which reads only the flux buffers.  The next barrier publishes the window and
    // orders this update before the next plane's flux writes.
    // Update: S(U) = U - r, r = lx dFx (+ ly dFy) (+ lz dFz).  The pointwise loads of U and U^n
    // follow the barrier (held across it they would spill; both planes were prefetched into L1
    // at the top of the iteration).
    __syncthreads();
    if constexpr (DIM == 3) {
      if (k + 1 < ke) {
        if (tma) tma_issue(k + 1);
        else load_plane(k + 1, false);
      }
    }
    if (own) {  // (own: the cell is not wrapped, own_cell = gy * nx + gx)
      const size_t off = (size_t)a.gz * pstride + own_cell;
      const double* pu = opaque(at(a.Uin + off, k));
      const double* pn = opaque(at(a.Un + off, k));
      double* po = opaque(a.Uout + off + (ptrdiff_t)k * (ptrdiff_t)pstride);
      double u0[NV], un[NV];
#pragma unroll
      for (int f = 0; f < NV; ++f) {
        u0[f] = __ldg(pu + f * fs);
        un[f] = (a.mode != 0) ? pn[f * fs] : 0.0;
      }
      const double* fzn = Fz + ((k + 1) & 1) * S::nCol;
      const double* fzo = Fz + (k & 1) * S::nCol;
#pragma unroll
      for (int f = 0; f < NV; ++f) {
        double r = c.lam[0] * (Fx[(f * TY + ty) * S::FXP + tx + 1] - Fx[(f * TY + ty) * S::FXP + tx]);
        if constexpr (DIM >= 2) r = r + c.lam[1] * (Fy[(f * (TY + 1) + ty + 1) * TX + tx] - Fy[(f * (TY + 1) + ty) * TX + tx]);
        if constexpr (DIM == 3) r = r + c.lam[2] * (fzn[f * NC + tid] - fzo[f * NC + tid]);
        const double s = u0[f] - r;
        double v = s;
        if (a.mode == 1) v = 0.5 * (un[f] + s);                    // RK2: U^{n+1} = (U^n + U**)/2
        else if (a.mode == 2) v = (a.wa * un[f]) + (a.wb * s);     // RK3: (a U^n) + (b S(U))
        if (NV > 8 && f == NV - 1 && a.last) v = v * c.damp;       // GLM damping once per step
        po[f * fs] = v;
      }
      // halo push (the PUSH instances, 3D slabs; k is CTA-uniform, only boundary planes): the
      // values just stored, read back through L2 (not forwarded from registers, which would hold
      // them live across the loop) into the neighbours' ghost planes
      if (PUSH && a.push_dn && k < a.gz) {
        double* h = a.push_dn + (size_t)(a.push_dn_nz + a.gz + k) * pstride + own_cell;
#pragma unroll
        for (int f = 0; f < NV; ++f) h[f * fs] = __ldcg(po + f * fs);
      }
      if (PUSH && a.push_up && k >= nzl - a.gz) {
        double* h = a.push_up + (size_t)(k - (nzl - a.gz)) * pstride + own_cell;
#pragma unroll
        for (int f = 0; f < NV; ++f) h[f * fs] = __ldcg(po + f * fs);
      }
    }
    if constexpr (DIM == 3) {
      if (k + 1 < ke) {
        if (tma) tma_convert(k + 1);  // (after the update: the copy flew while it ran)
        __syncthreads();
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (s_bad != ULLONG_MAX) atomicMin(a.bad + a.stage, s_bad);
    if (s_cnt[0]) atomicAdd(a.counters + 0, (unsigned long long)s_cnt[0]);
    if (s_cnt[1]) atomicAdd(a.counters + 1, (unsigned long long)s_cnt[1]);
    if (s_cnt[2]) atomicAdd(a.counters + 2, (unsigned long long)s_cnt[2]);
  }
}

// ---------------------------------------------------------------------------------------
// a6: dt / c_h partial maxima over the interior of U (3.12)
// ---------------------------------------------------------------------------------------
template <int DIM, int NV>
__global__ void __launch_bounds__(256) k_dt(DtArgs a) {
  const int nx = a.nx, ny = a.ny, nzl = a.nz_loc;
  const int fs = nx * ny;  // (mhd_create bounds nx*ny*9 below 2^31)
  const size_t pstride = (size_t)fs * NV;
  double M = 0.0, Sx = 0.0;
  unsigned long long badidx = ULLONG_MAX;
  // planes over blockIdx.y, cells of a plane over x: 32-bit in-plane indices, no 64-bit division
  for (int k = blockIdx.y; k < nzl; k += gridDim.y) {
    const double* plane = a.U + (size_t)(k + a.gz) * pstride;
    for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < fs; cell += gridDim.x * blockDim.x) {
      double u[NV], v[NV];
      load_fields<NV>(plane + cell, fs, u);
      if (bad_state<NV>(u)) {
        badidx = min(badidx, (unsigned long long)((a.zoff + k) * (long long)fs + cell));
        continue;
      }
      cons2prim<NV>(u, v, a.gm1, a.p_floor);
      double inv = 0.0, smax = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const double cf = fast_speed(a.gamma, v[0], v[4], v[5 + d], v[5 + (d + 1) % 3], v[5 + (d + 2) % 3]);
        const double s = fabs(v[1 + d]) + cf;
        if (d == 0) {
          inv = s * a.idx[0];
          smax = s;
        } else {
          inv = inv + s * a.idx[d];
          smax = fmax(smax, s);
        }
      }
      M = fmax(M, inv);
      Sx = fmax(Sx, smax);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
    Sx = fmax(Sx, __shfl_xor_sync(0xffffffffu, Sx, o));
  }
  __shared__ double red[2][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][w] = M;
    red[1][w] = Sx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      M = fmax(M, red[0][i]);
      Sx = fmax(Sx, red[1][i]);
    }
    // non-negative doubles order like their int64 bit patterns: exact, order-free max
    atomicMax(a.out + 0, (unsigned long long)__double_as_longlong(M));
    atomicMax(a.out + 1, (unsigned long long)__double_as_longlong(Sx));
  }
  if (badidx != ULLONG_MAX) atomicMin(a.bad, badidx);
}

// ---------------------------------------------------------------------------------------
// layout conversion: ABI [f][z][y][x] (interior) <-> internal [z+gz][f][y][x]
// ---------------------------------------------------------------------------------------
__global__ void k_pack(const double* __restrict__ src, double* __restrict__ dst, int nv, int nx, int ny, int nzl,
                       int gz, int to_internal) {
  const size_t fstride = (size_t)nx * ny;
  const size_t n = fstride * nzl * nv;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    // i enumerates the ABI layout [f][z][cell]
    const size_t cell = i % fstride;
    const size_t zf = i / fstride;
    const size_t z = zf % nzl, f = zf / nzl;
    const size_t j = ((z + gz) * nv + f) * fstride + cell;
    if (to_internal)
      dst[j] = src[i];
    else
      dst[i] = src[j];
  }
}

// set_state validation: rho > 0, p > 0 (before any floor), all finite
template <int NV>
__global__ void k_validate(const double* __restrict__ U, int nx, int ny, int nzl, int gz, long long zoff, double gm1,
                           unsigned long long* bad, int check_p) {
  const size_t fstride = (size_t)nx * ny, pstride = fstride * NV, ncell = fstride * nzl;
  unsigned long long b = ULLONG_MAX;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < ncell; i += (size_t)gridDim.x * blockDim.x) {
    const size_t k = i / fstride, cell = i % fstride;
    double u[NV], v[NV];
    load_cell<NV>(U, (k + gz) * pstride, fstride, cell, u);
    bool bad = bad_state<NV>(u);
    if (!bad && check_p) {
      cons2prim<NV>(u, v, gm1, -1.0e300);
      bad = !(v[4] > 0.0);
    }
    if (bad) b = min(b, (unsigned long long)((zoff + k) * fstride + cell));
  }
  if (b != ULLONG_MAX) atomicMin(bad, b);
}

// test-only face solve of independent pairs
template <int NV, int RS>
__global__ void k_face_flux(const double* __restrict__ VL, const double* __restrict__ VR, long long n, StageConsts c,
                            double* __restrict__ F, unsigned long long* nhll) {
  int cnt = 0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    double wl[NV], wr[NV], fn[NV];
#pragma unroll
    for (int f = 0; f < NV; ++f) {
      wl[f] = VL[q * NV + f];
      wr[f] = VR[q * NV + f];
    }
    cnt += face_flux<NV, RS>(wl, wr, c, fn);
#pragma unroll
    for (int f = 0; f < NV; ++f) F[q * NV + f] = fn[f];
  }
  if (cnt) atomicAdd(nhll, (unsigned long long)cnt);
}

// n words of device memory into pinned (mapped) host memory by a kernel instead of a copy-engine
// transfer: the per-step dt read-back is not queued behind a large asynchronous device->host
// state copy on the same engine (mhd_get_state_async)
__global__ void k_store_words(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

cudaError_t launch_store_words(unsigned long long* host_dst, const unsigned long long* src, int n, cudaStream_t st) {
  k_store_words<<<1, 32, 0, st>>>(host_dst, src, n);
  return cudaGetLastError();
}

// test-only: the branch-free operator sequences next to the IEEE operators (mhd_device.cuh)
__global__ void k_fast_ops(const double* __restrict__ A, const double* __restrict__ B, long long n,
                           double* __restrict__ out, int* __restrict__ okm) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const double a = A[q], b = B[q];
    bool o0 = true, o1 = true, o2 = true, o3 = true;
    out[q * 8 + 0] = fast_rcp(b, o0);
    out[q * 8 + 1] = 1.0 / b;
    out[q * 8 + 2] = fast_div(a, b, div_rcp(b), o1);
    out[q * 8 + 3] = a / b;
    out[q * 8 + 4] = fast_sqrt(a, o2);
    out[q * 8 + 5] = sqrt(a);
    out[q * 8 + 6] = fast_div_b(fabs(a), b, o3);
    out[q * 8 + 7] = fabs(a) / b;
    okm[q] = (int)o0 | ((int)o1 << 1) | ((int)o2 << 2) | ((int)o3 << 3);
  }
}

cudaError_t launch_fast_ops(const double* A, const double* B, long long n, double* out, int* okm, cudaStream_t st) {
  const unsigned blocks = (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1);
  k_fast_ops<<<blocks < 4096u ? blocks : 4096u, 256, 0, st>>>(A, B, n, out, okm);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// host-side launchers (explicit instantiations)
// ---------------------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3D: the TMA descriptor of the stage input — a 4D fp64 tensor (x, y, field, storage plane) with
// the plane window of a tile (PW x PH x NV x 1) as its box.  TMA needs 16-byte row strides (nx
// even); otherwise, or with MHD_NO_TMA=1, the kernel loads the window with per-thread loads.
template <int NV>
static int encode_window_map(StageArgs& a, int PW, int PH, int TYZ) {
  static const bool off = [] { const char* e = getenv("MHD_NO_TMA"); return e && atoi(e) == 1; }();
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (off || !enc || (a.nx & 1)) return 0;
  const cuuint64_t dims[4] = {(cuuint64_t)a.nx, (cuuint64_t)a.ny, (cuuint64_t)NV, (cuuint64_t)(a.nz_loc + 2 * a.gz)};
  const cuuint64_t row = (cuuint64_t)a.nx * sizeof(double);
  const cuuint64_t strides[3] = {row, row * (cuuint64_t)a.ny, row * (cuuint64_t)a.ny * NV};
  const cuuint32_t box[4] = {(cuuint32_t)PW, (cuuint32_t)PH, (cuuint32_t)NV, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(a.Uin), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 0;
  if (TYZ > 0) {  // the z-staging boxes: [f][TY+1][32] and [f][TY][34]
    const cuuint32_t bfy[4] = {32, (cuuint32_t)(TYZ + 1), (cuuint32_t)NV, 1};
    const cuuint32_t bfx[4] = {34, (cuuint32_t)TYZ, (cuuint32_t)NV, 1};
    r = enc(&a.tmap_fy, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(a.Uin), dims, strides, bfy, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 0;
    r = enc(&a.tmap_fx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(a.Uin), dims, strides, bfx, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 0;
  }
  return 1;
}

// the TMA plane window is used by the 3D PLM kernels (the fused WENO-Z kernel, an A/B
// alternative to the split stage, keeps per-thread loads)
template <int DIM, int REC>
constexpr bool stage_tma() { return DIM == 3 && REC != 2; }

template <int DIM, int NV, int RS, int TY, int REC>
static cudaError_t launch_stage_t(const StageArgs& a0, cudaStream_t st) {
  using S = StageSmem<DIM, NV, TY, REC == 2 ? 3 : 2>;
  constexpr bool T = stage_tma<DIM, REC>();
  constexpr bool P = DIM == 3;  // (the halo push exists for 3D slabs only)
  if (a0.ze <= a0.zb) return cudaSuccess;
  StageArgs a = a0;
  a.tma = T ? encode_window_map<NV>(a, S::PW, S::PH, (MHD_ZTMA && REC != 2) ? TY : 0) : 0;
  // the PUSH instances only when this launch pushes: the others carry no trace of it
  const bool push = P && (a.push_dn || a.push_up);
  auto kern = a.tma ? (push ? k_stage<DIM, NV, RS, TY, REC, T, P> : k_stage<DIM, NV, RS, TY, REC, T, false>)
                    : (push ? k_stage<DIM, NV, RS, TY, REC, false, P> : k_stage<DIM, NV, RS, TY, REC, false, false>);
  // (the attribute is per device: set on every launch, a host-side call of ~1 us)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((a.nx + 31) / 32, (a.ny + TY - 1) / TY, (a.ze - a.zb + a.kz - 1) / a.kz);
  kern<<<grid, S::NT, S::bytes, st>>>(a);
  return cudaGetLastError();
}

#ifndef MHD_TY3
#define MHD_TY3 7
#endif
#ifndef MHD_TY2
#define MHD_TY2 5
#endif
#ifndef MHD_TYW3
#define MHD_TYW3 5
#endif
template <int REC>
static cudaError_t launch_stage_w(int dim, int nv, int riemann, const StageArgs& a, cudaStream_t st) {
  if (dim == 3) {
    constexpr int TY3 = REC == 2 ? MHD_TYW3 : MHD_TY3;
    if (riemann) return launch_stage_t<3, 9, 1, TY3, REC>(a, st);
    return launch_stage_t<3, 9, 0, TY3, REC>(a, st);
  }
  if (dim == 2) {
    if (riemann) return launch_stage_t<2, 9, 1, MHD_TY2, REC>(a, st);
    return launch_stage_t<2, 9, 0, MHD_TY2, REC>(a, st);
  }
  if (nv == 9) {
    if (riemann) return launch_stage_t<1, 9, 1, 1, REC>(a, st);
    return launch_stage_t<1, 9, 0, 1, REC>(a, st);
  }
  if (riemann) return launch_stage_t<1, 8, 1, 1, REC>(a, st);
  return launch_stage_t<1, 8, 0, 1, REC>(a, st);
}

cudaError_t launch_stage(int dim, int nv, int riemann, const StageArgs& a, cudaStream_t st) {
  // the reconstruction is a template parameter: 0 PLM minmod, 1 PLM MC, 2 WENO-Z (ghost width 3)
  if (a.c.limiter == 2) return launch_stage_w<2>(dim, nv, riemann, a, st);
  if (a.c.limiter == 1) return launch_stage_w<1>(dim, nv, riemann, a, st);
  return launch_stage_w<0>(dim, nv, riemann, a, st);
}

int stage_tile_rows(int dim, int limiter) {
  return dim == 3 ? (limiter == 2 ? MHD_TYW3 : MHD_TY3) : (dim == 2 ? MHD_TY2 : 1);
}

template <int DIM, int NV, int RS, int TY, int REC>
static int ctas_per_sm_t() {
  using S = StageSmem<DIM, NV, TY, REC == 2 ? 3 : 2>;
  auto kern = k_stage<DIM, NV, RS, TY, REC, stage_tma<DIM, REC>()>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, S::NT, S::bytes) != cudaSuccess) n = 1;
  return n > 0 ? n : 1;
}

int stage_ctas_per_sm(int dim, int nv, int riemann, int limiter) {
  if (limiter == 2) {
    if (dim == 3) return riemann ? ctas_per_sm_t<3, 9, 1, MHD_TYW3, 2>() : ctas_per_sm_t<3, 9, 0, MHD_TYW3, 2>();
    if (dim == 2) return riemann ? ctas_per_sm_t<2, 9, 1, MHD_TY2, 2>() : ctas_per_sm_t<2, 9, 0, MHD_TY2, 2>();
    return 1;
  }
  if (dim == 3) return riemann ? ctas_per_sm_t<3, 9, 1, MHD_TY3, 1>() : ctas_per_sm_t<3, 9, 0, MHD_TY3, 1>();
  if (dim == 2) return riemann ? ctas_per_sm_t<2, 9, 1, MHD_TY2, 1>() : ctas_per_sm_t<2, 9, 0, MHD_TY2, 1>();
  return 1;
}

cudaError_t launch_dt(int dim, int nv, const DtArgs& a, int nsm, cudaStream_t st) {
  // ~8 blocks of 256 per SM in total: x covers a plane (capped), y strides over the planes
  const size_t fs = (size_t)a.nx * a.ny, cap = (size_t)nsm * MHD_DT_PER_SM;
  const unsigned bx = (unsigned)std::max<size_t>(1, std::min<size_t>((fs + 255) / 256, cap));
  const unsigned by = (unsigned)std::max<size_t>(1, std::min<size_t>((size_t)a.nz_loc, cap / bx));
  const dim3 g(bx, by);
  if (dim == 3) k_dt<3, 9><<<g, 256, 0, st>>>(a);
  else if (dim == 2) k_dt<2, 9><<<g, 256, 0, st>>>(a);
  else if (nv == 9) k_dt<1, 9><<<g, 256, 0, st>>>(a);
  else k_dt<1, 8><<<g, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pack(const double* src, double* dst, int nv, int nx, int ny, int nzl, int gz, int to_internal,
                        int nsm, cudaStream_t st) {
  k_pack<<<nsm * 8, 256, 0, st>>>(src, dst, nv, nx, ny, nzl, gz, to_internal);
  return cudaGetLastError();
}

cudaError_t launch_validate(const double* U, int nv, int nx, int ny, int nzl, int gz, long long zoff, double gm1,
                            unsigned long long* bad, int nsm, cudaStream_t st, int check_p) {
  if (nv == 9) k_validate<9><<<nsm * 8, 256, 0, st>>>(U, nx, ny, nzl, gz, zoff, gm1, bad, check_p);
  else k_validate<8><<<nsm * 8, 256, 0, st>>>(U, nx, ny, nzl, gz, zoff, gm1, bad, check_p);
  return cudaGetLastError();
}

cudaError_t launch_face_flux(int nv, int riemann, const double* VL, const double* VR, long long n,
                             const StageConsts& c, double* F, unsigned long long* nhll, cudaStream_t st) {
  const unsigned blocks = (unsigned)((n + 127) / 128 > 0 ? (n + 127) / 128 : 1);
  if (nv == 9) {
    if (riemann) k_face_flux<9, 1><<<blocks, 128, 0, st>>>(VL, VR, n, c, F, nhll);
    else k_face_flux<9, 0><<<blocks, 128, 0, st>>>(VL, VR, n, c, F, nhll);
  } else {
    if (riemann) k_face_flux<8, 1><<<blocks, 128, 0, st>>>(VL, VR, n, c, F, nhll);
    else k_face_flux<8, 0><<<blocks, 128, 0, st>>>(VL, VR, n, c, F, nhll);
  }
  return cudaGetLastError();
}

}  // namespace mhd
