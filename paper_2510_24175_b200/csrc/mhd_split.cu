// mhd_split.cu — the WENO-Z stage of the GLM path as five plain launches (3D; SURVEY.md §8(f)
// row 3, DESIGN.md §5 "split stage").
//
// The fused k_stage keeps every intermediate on chip, which wins for PLM; a WENO-Z cell carries
// ~2x the reconstruction work and state, and the fused kernel runs 12 warps/SM at 168 registers.
// Here each step is its own high-occupancy kernel over HBM-resident intermediates (the same
// arithmetic, so the same bits):
//   k_sp_prim       cons -> prim of the planes [-3, nz+3) -> V (padded like U)
//   k_sp_face_x     x faces i-1/2, i in [0, nx]: each cell reconstructed once, q+ to the next lane
//                   by shuffle, the faces at 32-cell chunk starts in a second pass
//   k_sp_face_m<D>  y (D = 1) and z (D = 2) faces: a thread marches a 16-cell segment of a line,
//                   carrying q+ of the previous cell
//   k_sp_update     r = lx dFx + ly dFy + lz dFz (DESIGN.md §3.11 order), the RK epilogue, psi damping
// x/y boundaries by index wrap (periodic) or clamp (outflow), z by the ghost planes of U.
// Counters follow the fused kernel's owner rule: reconstruction fallbacks for the right cell of
// the faces of interior cells, HLL fallbacks for n+1 faces per line (z: the top face by the last
// slab only).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "mhd_device.cuh"
#include "mhd_kernels.h"

namespace mhd {

namespace {

struct SpIdx {
  int nx, ny, gz, nv;
  int bx0, bx1, by0, by1;  // 0 periodic, 1 outflow
  size_t fs, ps;           // field stride (nx*ny), plane stride (nv*fs)
  __device__ __forceinline__ int wx(int i) const {
    return i < 0 ? (bx0 ? 0 : i + nx) : (i >= nx ? (bx1 ? nx - 1 : i - nx) : i);
  }
  __device__ __forceinline__ int wy(int j) const {
    return j < 0 ? (by0 ? 0 : j + ny) : (j >= ny ? (by1 ? ny - 1 : j - ny) : j);
  }
  // field 0 of cell (i, j, k) of a padded [z+gz][f][y][x] array (x, y resolved by the BCs); the
  // fields follow int(fs) apart.  The pointer is made opaque so
  // that the field loads stay base + small offsets instead of a 64-bit index computation each
  template <typename T>
  __device__ __forceinline__ T* cell(T* base, int i, int j, int k) const {
    T* p = base + ((size_t)(k + gz) * ps + (size_t)(wy(j) * nx + wx(i)));
    asm("mov.b64 %0, %0;" : "+l"(p));
    return p;
  }
};

__device__ __forceinline__ SpIdx make_idx(const SplitArgs& a) {
  SpIdx X;
  X.nx = a.nx;
  X.ny = a.ny;
  X.gz = a.gz;
  X.nv = NVS;
  X.bx0 = a.bcx[0];
  X.bx1 = a.bcx[1];
  X.by0 = a.bcy[0];
  X.by1 = a.bcy[1];
  X.fs = (size_t)a.nx * a.ny;
  X.ps = X.fs * NVS;
  return X;
}

// face flux arrays: [k][f][j][i], rows of split_row_pitch(nx) >= nx + 1 (a multiple of 32: aligned
// rows), ny + 1 rows per plane, planes k in [0, nz]
__device__ __forceinline__ size_t fidx(const SplitArgs& a, int f, int i, int j, int k) {
  return (((size_t)k * NVS + f) * (size_t)(a.ny + 1) + j) * (size_t)a.px + i;
}

}  // namespace

// 1: primitives of the planes [-3, nz+3); floors and bad cells of the interior (owner rule)
__global__ void __launch_bounds__(256) k_sp_prim(SplitArgs a) {
  const SpIdx X = make_idx(a);
  const size_t n = X.fs * (a.nz + 6);
  int floors = 0;
  unsigned long long bad = ULLONG_MAX;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % a.nx), j = (int)((q / a.nx) % a.ny), k = (int)(q / X.fs) - 3;
    const bool interior = k >= 0 && k < a.nz;
    double u[NVS], v[NVS];
    const double* pu = X.cell(a.Uin, i, j, k);
    double* pv = X.cell(a.V, i, j, k);
    const int fs = (int)X.fs;
#pragma unroll
    for (int f = 0; f < NVS; ++f) u[f] = __ldg(pu + f * fs);
    if (interior && bad_state<NVS>(u))
      bad = min(bad, (unsigned long long)(((a.zoff + k) * a.ny + j) * (long long)a.nx + i));
    const bool fl = cons2prim<NVS>(u, v, a.c.gm1, a.c.p_floor);
    floors += (fl && interior) ? 1 : 0;
#pragma unroll
    for (int f = 0; f < NVS; ++f) pv[f * fs] = v[f];
  }
  if (floors) atomicAdd(a.counters + 0, (unsigned long long)floors);
  if (bad != ULLONG_MAX) atomicMin(a.bad + a.stage, bad);
}

// both WENO-Z states of cell (i,j,k) along D (the normal frame of D); returns the fallback
template <int D>
__device__ __forceinline__ bool sp_recon(const SplitArgs& a, const SpIdx& X, int i, int j, int k, double* qp,
                                         double* qm) {
  constexpr int oi = D == 0, oj = D == 1, ok = D == 2;
  double c[5][NVS], p[NVS], m[NVS];
  const int fs = (int)X.fs;
#pragma unroll
  for (int s = -2; s <= 2; ++s) {
    const double* v = X.cell(a.V, i + s * oi, j + s * oj, k + s * ok);
#pragma unroll
    for (int f = 0; f < NVS; ++f) c[s + 2][f] = v[f * fs];
  }
#ifndef MHD_SP_INL
#define MHD_SP_INL 0  // bit D: inline WENO-Z in the D-face kernel (round 2: all out of line, 8.40 vs 8.45 ms with x inline)
#endif
  const bool fb = weno_cell<NVS, (MHD_SP_INL >> D) & 1>(c[0], c[1], c[2], c[3], c[4], p, m);
  to_normal<NVS, D>(p, qp);
  to_normal<NVS, D>(m, qm);
  return fb;
}

// the face (vl | vr) in the normal frame of D -> F_D at face index (i, j, k); the HLL fallback
template <int D, int RS>
__device__ __forceinline__ int sp_solve_store(const SplitArgs& a, const double* vl, const double* vr, int i, int j,
                                              int k) {
  double fn[NVS], fx[NVS];
  const int fell = face_flux<NVS, RS, true>(vl, vr, a.c, fn);
  from_normal<NVS, D>(fn, fx);
  double* F = a.F[D] + fidx(a, 0, i, j, k);
  asm("mov.b64 %0, %0;" : "+l"(F));
  const int fst = (a.ny + 1) * a.px;  // field stride of the flux arrays
#pragma unroll
  for (int f = 0; f < NVS; ++f) F[f * fst] = fx[f];
  return fell;
}

#ifndef MHD_SP_SEG
#define MHD_SP_SEG 64
#endif
constexpr int kSpSeg = MHD_SP_SEG;
#ifndef MHD_SPP_PER_SM
#define MHD_SPP_PER_SM 64  // k_sp_prim blocks of 256 per SM
#endif
#ifndef MHD_SPF_PER_SM
#define MHD_SPF_PER_SM 32  // face-kernel blocks of 128 per SM
#endif
#ifndef MHD_SPU_PER_SM
#define MHD_SPU_PER_SM 256 // k_sp_update blocks of 256 per SM (grid-stride over the cells)
#endif  // faces per marching segment (at most; segments of a line are balanced)
#ifndef MHD_SP_BLOCK
#define MHD_SP_BLOCK 128  // face-kernel block size
#endif
constexpr int kSpB = MHD_SP_BLOCK;
#ifndef MHD_SP_MINB
#define MHD_SP_MINB 3  // 3 blocks of 128 per SM (<= 168 registers): +2% over no bound, 4 spills more
#endif

// y and z faces: lane = x (coalesced), a thread marches one 16-face segment of a line
template <int D, int RS>
__global__ void __launch_bounds__(kSpB, MHD_SP_MINB) k_sp_face_m(SplitArgs a) {
  const SpIdx X = make_idx(a);
  const int nb = D == 1 ? a.nz : a.ny;         // second line coordinate: k (y lines) or j (z lines)
  const int nm = D == 1 ? a.ny + 1 : a.nz + 1;  // faces per line
  const int nseg = (nm + kSpSeg - 1) / kSpSeg;
  const size_t n = (size_t)a.nx * nb * nseg;
  const int per = nm / nseg, rem = nm % nseg;  // segment sg: per + (sg < rem) faces
  const bool top_owner = a.zoff + a.nz == a.nz_glob;  // the domain's top z face is counted once
  int fbs = 0, hlls = 0;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % a.nx);
    const size_t r = q / a.nx;
    const int b = (int)(r % nb), sg = (int)(r / nb);
    const int m0 = sg * per + min(sg, rem), m1 = m0 + per + (sg < rem ? 1 : 0);
    double pl[NVS], qp[NVS], qm[NVS];
    if (D == 1) sp_recon<D>(a, X, i, m0 - 1, b, pl, qm);
    else sp_recon<D>(a, X, i, b, m0 - 1, pl, qm);  // q+ of the cell before the first face
    for (int m = m0; m < m1; ++m) {
      const int j = D == 1 ? m : b, k = D == 1 ? b : m;
      const bool fb = sp_recon<D>(a, X, i, j, k, qp, qm);  // (m = n: the ghost / wrapped cell)
      fbs += (fb && m < nm - 1) ? 1 : 0;
      const int fell = sp_solve_store<D, RS>(a, pl, qm, i, j, k);
      hlls += (fell && (D == 1 || m < nm - 1 || top_owner)) ? 1 : 0;
#pragma unroll
      for (int f = 0; f < NVS; ++f) pl[f] = qp[f];
    }
  }
  if (fbs) atomicAdd(a.counters + 1, (unsigned long long)fbs);
  if (hlls) atomicAdd(a.counters + 2, (unsigned long long)hlls);
}

// x faces i in [0, nx] of the rows (j, k).  A warp item covers the 32 cells 31t-1 .. 31t+30 of a
// row: every lane reconstructs its cell once; lanes 1..31 solve the faces i-1/2 with q+ of cell
// i-1 from lane l-1 (a shuffle).  Items overlap by one cell, so the faces at item starts need no
// second pass (the lane-0 cell is reconstructed twice: 1/32 of the work) and every read is a
// coalesced row segment that the neighbouring items also touch (L1/L2 hits, V read once from HBM).
template <int RS>
__global__ void __launch_bounds__(kSpB, MHD_SP_MINB) k_sp_face_x(SplitArgs a) {
  const SpIdx X = make_idx(a);
  const int nf = a.nx + 1, nch = (nf + 30) / 31;  // faces per row, items per row
  const size_t items = (size_t)nch * a.ny * a.nz;
  const int lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  int fbs = 0, hlls = 0;
  for (size_t w = gw; w < items; w += nw) {  // warp-uniform loop
    const int cx = (int)(w % nch);
    const size_t row = w / nch;
    const int j = (int)(row % a.ny), k = (int)(row / a.ny);
    const int i = cx * 31 - 1 + lane;  // (i < 0 or i > nx: the wrapped / clamped cell; i >= nx never counted)
    double qp[NVS], qm[NVS], pl[NVS];
    const bool fb = sp_recon<0>(a, X, i, j, k, qp, qm);
#pragma unroll
    for (int f = 0; f < NVS; ++f) pl[f] = __shfl_up_sync(0xffffffffu, qp[f], 1);
    if (lane > 0 && i <= a.nx) {  // face i-1/2, i in [0, nx]
      fbs += (fb && i < a.nx) ? 1 : 0;
      hlls += sp_solve_store<0, RS>(a, pl, qm, i, j, k) ? 1 : 0;
    }
  }
  if (fbs) atomicAdd(a.counters + 1, (unsigned long long)fbs);
  if (hlls) atomicAdd(a.counters + 2, (unsigned long long)hlls);
}

// flux divergence in the §3.11 order, the RK epilogue, psi damping on the last stage
__global__ void __launch_bounds__(256) k_sp_update(SplitArgs a) {
  const SpIdx X = make_idx(a);
  const size_t n = X.fs * a.nz;
  const double* lam = a.c.lam;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % a.nx), j = (int)((q / a.nx) % a.ny), k = (int)(q / X.fs);
    const int fs = (int)X.fs, fst = (a.ny + 1) * a.px, pl = NVS * fst;
    const double* fx = a.F[0] + fidx(a, 0, i, j, k);
    const double* fy = a.F[1] + fidx(a, 0, i, j, k);
    const double* fz = a.F[2] + fidx(a, 0, i, j, k);
    const double* pu = X.cell(a.Uin, i, j, k);
    const double* pn = X.cell(a.Un, i, j, k);
    double* po = X.cell(a.Uout, i, j, k);
    double v[NVS];  // every load before the first store (Uout may alias U^n)
#pragma unroll
    for (int f = 0; f < NVS; ++f) {
      double r = lam[0] * (__ldg(fx + f * fst + 1) - __ldg(fx + f * fst));
      r = r + lam[1] * (__ldg(fy + f * fst + a.px) - __ldg(fy + f * fst));
      r = r + lam[2] * (__ldg(fz + f * fst + pl) - __ldg(fz + f * fst));
      const double s = __ldg(pu + f * fs) - r;
      v[f] = s;
      if (a.mode == 1) v[f] = 0.5 * (pn[f * fs] + s);                 // RK2: U^{n+1} = (U^n + U**)/2
      else if (a.mode == 2) v[f] = (a.wa * pn[f * fs]) + (a.wb * s);  // RK3: (a U^n) + (b S(U))
    }
    if (a.last) v[NVS - 1] = v[NVS - 1] * a.c.damp;  // GLM damping once per step
#pragma unroll
    for (int f = 0; f < NVS; ++f) po[f * fs] = v[f];
    // halo push: a boundary plane also into the z neighbour's ghost plane
    const size_t cell = (size_t)j * a.nx + i;
    if (a.push_dn && k < a.gz) {
      double* h = a.push_dn + (size_t)(a.push_dn_nz + a.gz + k) * X.ps + cell;
#pragma unroll
      for (int f = 0; f < NVS; ++f) h[f * fs] = v[f];
    }
    if (a.push_up && k >= a.nz - a.gz) {
      double* h = a.push_up + (size_t)(k - (a.nz - a.gz)) * X.ps + cell;
#pragma unroll
      for (int f = 0; f < NVS; ++f) h[f * fs] = v[f];
    }
  }
}

cudaError_t launch_split_stage(int riemann, const SplitArgs& a, int nsm, cudaStream_t st, cudaStream_t aux1,
                               cudaStream_t aux2, cudaEvent_t* ev) {
  const size_t pc = (size_t)a.nx * a.ny;
  auto grid = [&](size_t n, int bs, int per_sm) {
    return (unsigned)std::max<size_t>(1, std::min<size_t>((n + bs - 1) / bs, (size_t)nsm * per_sm));
  };
  const size_t segy = (size_t)a.nx * a.nz * ((a.ny + 1 + kSpSeg - 1) / kSpSeg);
  const size_t segz = (size_t)a.nx * a.ny * ((a.nz + 1 + kSpSeg - 1) / kSpSeg);
  const size_t xw = (size_t)((a.nx + 1 + 30) / 31) * 32 * a.ny * a.nz;
  k_sp_prim<<<grid(pc * (a.nz + 6), 256, MHD_SPP_PER_SM), 256, 0, st>>>(a);
  // the three face kernels are independent (V in, their own F out): y and z on two auxiliary
  // streams, joined before the update, so one kernel's tail overlaps the others
  cudaStream_t s1 = aux1 ? aux1 : st, s2 = aux2 ? aux2 : st;
  if (aux1) {
    cudaEventRecord(ev[0], st);
    cudaStreamWaitEvent(s1, ev[0], 0);
    cudaStreamWaitEvent(s2, ev[0], 0);
  }
  if (riemann) {
    k_sp_face_x<1><<<grid(xw, kSpB, MHD_SPF_PER_SM), kSpB, 0, st>>>(a);
    k_sp_face_m<1, 1><<<grid(segy, kSpB, MHD_SPF_PER_SM), kSpB, 0, s1>>>(a);
    k_sp_face_m<2, 1><<<grid(segz, kSpB, MHD_SPF_PER_SM), kSpB, 0, s2>>>(a);
  } else {
    k_sp_face_x<0><<<grid(xw, kSpB, MHD_SPF_PER_SM), kSpB, 0, st>>>(a);
    k_sp_face_m<1, 0><<<grid(segy, kSpB, MHD_SPF_PER_SM), kSpB, 0, s1>>>(a);
    k_sp_face_m<2, 0><<<grid(segz, kSpB, MHD_SPF_PER_SM), kSpB, 0, s2>>>(a);
  }
  if (aux1) {
    cudaEventRecord(ev[1], s1);
    cudaEventRecord(ev[2], s2);
    cudaStreamWaitEvent(st, ev[1], 0);
    cudaStreamWaitEvent(st, ev[2], 0);
  }
  k_sp_update<<<grid(pc * a.nz, 256, MHD_SPU_PER_SM), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace mhd
