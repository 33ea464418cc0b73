// mhd_ct.cu — constrained transport path (R32).
//
// The paper's weak-scaling runs keep div B = 0 with constrained transport (
// Evans & Hawley 1988, Londrillo & Del Zanna 2004).  State: rho, m, E cell-centred, b_x / b_y /
// b_z on the x / y / z faces (face i-1/2 / j-1/2 / k-1/2 of cell (i,j,k)), 3D periodic, on one GPU
// or z slabs.  x/y are wrapped by index; z reads ghost planes (gz = G + 1 per side, G the
// reconstruction half-width: the topmost V plane needs b_z one plane further), filled by a
// periodic copy on one GPU or the slab halo exchange before every stage and dt pass.
// Per RK stage three kernels:
//   k_ct_prim    cell-centred B = face average, cons->prim -> V (8 fields)
//   k_ct_face_x, k_ct_face_m<D>: reconstruction along D (each cell once), normal field = the face
//                value, face solve -> F_D (the induction entries are the face EMFs)
//   k_ct_update  rho, m, E by the flux divergence; b by Stokes with edge EMFs averaged from the
//                four adjacent face EMFs (arithmetic); the RK epilogue.
// The arithmetic of every step follows the recipe of DESIGN.md R32 operation for
// operation (built with --fmad=false), so the two agree bitwise.
#include <cuda_runtime.h>

#include <climits>

#include "mhd_device.cuh"
#include "mhd_kernels.h"

#ifndef MHD_CT_WINL
#define MHD_CT_WINL true  // WENO-Z evaluator inlined in the CT face kernels
#endif

namespace mhd {

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

struct CtIdx {
  int nx, ny, nz, gz;
  size_t fs, ps;  // field stride (nx*ny), plane stride (8*fs)
  // cell (i, j, k) of field f: x, y wrapped (periodic), k in [-gz, nz + gz) (ghost planes)
  __device__ size_t at(int f, int i, int j, int k) const {
    return (size_t)(k + gz) * ps + (size_t)f * fs + (size_t)wrapi(j, ny) * nx + wrapi(i, nx);
  }
};
// decode q in [0, nx*ny*nk) into (i, j, k0 + kk).  (A 32-bit decode for grids below 2^32 cells
// measured 10% slower stages: profiles/r02_ab_fx.txt.)
__device__ __forceinline__ void ct_decode(size_t q, int nx, int ny, int k0, int& i, int& j, int& k) {
  i = (int)(q % nx);
  j = (int)((q / nx) % ny);
  k = k0 + (int)(q / ((size_t)nx * ny));
}

__device__ __forceinline__ void ct_cell_cons(const double* __restrict__ U, const CtIdx& X, int i, int j, int k,
                                             double* w) {
#pragma unroll
  for (int f = 0; f < 5; ++f) w[f] = __ldg(U + X.at(f, i, j, k));
  w[5] = 0.5 * (__ldg(U + X.at(5, i, j, k)) + __ldg(U + X.at(5, i + 1, j, k)));
  w[6] = 0.5 * (__ldg(U + X.at(6, i, j, k)) + __ldg(U + X.at(6, i, j + 1, k)));
  w[7] = 0.5 * (__ldg(U + X.at(7, i, j, k)) + __ldg(U + X.at(7, i, j, k + 1)));
}

// 1-2: cell-centred primitives of the planes [-G, nz + G) (V: the same padded layout); floors
// and bad cells are counted on the interior planes only (the owner rule)
__global__ void __launch_bounds__(256) k_ct_prim(CtArgs a) {
  const CtIdx X{a.nx, a.ny, a.nz, a.gz, (size_t)a.nx * a.ny, (size_t)a.nx * a.ny * 8};
  const size_t n = (size_t)a.nx * a.ny * (a.nz + 2 * a.G);
  int floors = 0;
  unsigned long long bad = ULLONG_MAX;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    int i, j, k;
    ct_decode(q, a.nx, a.ny, -a.G, i, j, k);
    const bool interior = k >= 0 && k < a.nz;
    double u[8], w[8], v[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) u[f] = __ldg(a.Uin + X.at(f, i, j, k));
    if (interior && bad_state<8>(u))
      bad = min(bad, (unsigned long long)(((a.zoff + k) * a.ny + j) * (long long)a.nx + i));
    ct_cell_cons(a.Uin, X, i, j, k, w);
    const bool fl = cons2prim<8>(w, v, a.c.gm1, a.c.p_floor);
    floors += (fl && interior) ? 1 : 0;
#pragma unroll
    for (int f = 0; f < 8; ++f) a.V[X.at(f, i, j, k)] = v[f];
  }
  if (floors) atomicAdd(a.counters + 0, (unsigned long long)floors);
  if (bad != ULLONG_MAX) atomicMin(a.bad + a.stage, bad);
}

// 3-4: faces along D: reconstruction, staggered normal field, face solve.  x/y faces on the
// planes [-1, nz] (the edge EMFs of the slab's end planes use the faces of the planes beyond),
// z faces k-1/2 for k in [0, nz]; counters for the faces of interior cells (the right cell's
// reconstruction fallback, R17; the solve's HLL fallback).  Every cell is reconstructed once
// per direction (both states from one WENO-Z indicator set or one PLM slope): the y and z
// kernels march along D carrying q+ of the previous cell, the x kernel passes q+ to the next
// lane and solves the faces at 32-cell chunk starts in a second pass.

// both states of cell (i,j,k) along D from V; returns the positivity fallback
template <int D, int REC>
__device__ __forceinline__ bool ct_recon(const CtArgs& a, const CtIdx& X, int i, int j, int k, double* qp,
                                         double* qm) {
  constexpr int oi = D == 0, oj = D == 1, ok = D == 2;
  constexpr int H = REC == 2 ? 2 : 1;
  double c[2 * H + 1][8];
#pragma unroll
  for (int s = -H; s <= H; ++s)
#pragma unroll
    for (int f = 0; f < 8; ++f) c[s + H][f] = a.V[X.at(f, i + s * oi, j + s * oj, k + s * ok)];
  if constexpr (REC == 2) return weno_cell<8, MHD_CT_WINL>(c[0], c[1], c[2], c[3], c[4], qp, qm);
  else return plm_cell<8, REC>(c[0], c[1], c[2], qp, qm);
}

// the face between vl (q+ of the cell before) and vr (q- of cell (i,j,k)) along D: staggered
// normal field, solve, F_D at (i,j,k); returns the HLL fallback.  vl, vr are modified.
template <int D, int RS>
__device__ __forceinline__ int ct_solve_store(const CtArgs& a, const CtIdx& X, double* vl, double* vr, int i, int j,
                                              int k) {
  const double b = __ldg(a.Uin + X.at(5 + D, i, j, k));  // the staggered normal field of this face
  vl[5 + D] = b;
  vr[5 + D] = b;
  double wl[8], wr[8], fn[8], fx[8];
  to_normal<8, D>(vl, wl);
  to_normal<8, D>(vr, wr);
  const int fell = face_flux<8, RS>(wl, wr, a.c, fn);
  from_normal<8, D>(fn, fx);
  double* F = a.F[D];
#pragma unroll
  for (int f = 0; f < 8; ++f) F[X.at(f, i, j, k)] = fx[f];
  return fell;
}

#ifndef MHD_CTU_PER_SM
#define MHD_CTU_PER_SM 64  // k_ct_prim / k_ct_update blocks of 256 per SM
#endif
#ifndef MHD_CT_SEG
#define MHD_CT_SEG 32
#endif
constexpr int kCtSeg = MHD_CT_SEG;  // cells per marching segment (one extra reconstruction per segment)
#ifndef MHD_CT_MINB
#define MHD_CT_MINB 4  // PLM: 4 blocks of 128 per SM (<= 128 registers): -3% CT-PLM stage time
#endif
#ifndef MHD_CT_MINB_W
#define MHD_CT_MINB_W 3  // WENO-Z: 3 blocks (<= 168 registers, fewer spills): 6.8-6.9 vs 7.05 ms (4 blocks)
#endif
template <int REC>
struct CtMinB {
  static constexpr int value = REC == 2 ? MHD_CT_MINB_W : MHD_CT_MINB;
};

// y (D = 1) and z (D = 2) faces: a thread marches a segment of one line (lane = x, coalesced)
template <int D, int RS, int REC>
__global__ void __launch_bounds__(128, CtMinB<REC>::value) k_ct_face_m(CtArgs a) {
  const CtIdx X{a.nx, a.ny, a.nz, a.gz, (size_t)a.nx * a.ny, (size_t)a.nx * a.ny * 8};
  const int nb = D == 1 ? a.nz + 2 : a.ny;     // second line coordinate: k + 1 (y) or j (z)
  const int nm = D == 1 ? a.ny : a.nz + 1;     // marched faces per line
  const int nseg = (nm + kCtSeg - 1) / kCtSeg;
  const size_t n = (size_t)a.nx * nb * nseg;
  int fbs = 0, hlls = 0;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % a.nx);
    const size_t r = q / a.nx;
    const int b = (int)(r % nb), sg = (int)(r / nb);
    const int m0 = sg * kCtSeg, m1 = min(m0 + kCtSeg, nm);
    auto cell = [&](int m, int& j, int& k) {
      if (D == 1) { j = m; k = b - 1; } else { j = b; k = m; }
    };
    double pl[8], qp[8], qm[8];
    int j, k;
    cell(m0 - 1, j, k);
    ct_recon<D, REC>(a, X, i, j, k, pl, qm);  // q+ of the cell before the segment's first face
    for (int m = m0; m < m1; ++m) {
      cell(m, j, k);
      const bool interior = k >= 0 && k < a.nz;
      const bool fb = ct_recon<D, REC>(a, X, i, j, k, qp, qm);
      fbs += (fb && interior) ? 1 : 0;
      hlls += (ct_solve_store<D, RS>(a, X, pl, qm, i, j, k) && interior) ? 1 : 0;
#pragma unroll
      for (int f = 0; f < 8; ++f) pl[f] = qp[f];
    }
  }
  if (fbs) atomicAdd(a.counters + 1, (unsigned long long)fbs);
  if (hlls) atomicAdd(a.counters + 2, (unsigned long long)hlls);
}

// x faces: warps over 32-cell chunks of the rows (j, k), k in [-1, nz]; lane l > 0 takes q+ of
// cell i-1 from lane l-1; the faces at chunk starts follow in a second pass, one per thread
template <int RS, int REC>
__global__ void __launch_bounds__(128, CtMinB<REC>::value) k_ct_face_x(CtArgs a) {
  const CtIdx X{a.nx, a.ny, a.nz, a.gz, (size_t)a.nx * a.ny, (size_t)a.nx * a.ny * 8};
  const int nch = (a.nx + 31) / 32;
  const size_t items = (size_t)nch * a.ny * (a.nz + 2);
  const int lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  int fbs = 0, hlls = 0;
  for (size_t w = gw; w < items; w += nw) {  // warp-uniform loop
    const int cx = (int)(w % nch);
    const size_t row = w / nch;
    const int j = (int)(row % a.ny), k = (int)(row / a.ny) - 1;
    const int i = cx * 32 + lane;  // (i >= nx: a wrapped duplicate, never stored)
    double qp[8], qm[8], pl[8];
    const bool fb = ct_recon<0, REC>(a, X, i, j, k, qp, qm);
#pragma unroll
    for (int f = 0; f < 8; ++f) pl[f] = __shfl_up_sync(0xffffffffu, qp[f], 1);
    if (lane > 0 && i < a.nx) {
      const bool interior = k >= 0 && k < a.nz;
      fbs += (fb && interior) ? 1 : 0;
      hlls += (ct_solve_store<0, RS>(a, X, pl, qm, i, j, k) && interior) ? 1 : 0;
    }
  }
  const size_t nt = (size_t)gridDim.x * blockDim.x;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < items; q += nt) {  // chunk starts
    const int cx = (int)(q % nch);
    const size_t row = q / nch;
    const int j = (int)(row % a.ny), k = (int)(row / a.ny) - 1;
    const int i = cx * 32;
    const bool interior = k >= 0 && k < a.nz;
    double pl[8], qm[8], t[8];
    ct_recon<0, REC>(a, X, i - 1, j, k, pl, t);
    const bool fb = ct_recon<0, REC>(a, X, i, j, k, t, qm);
    fbs += (fb && interior) ? 1 : 0;
    hlls += (ct_solve_store<0, RS>(a, X, pl, qm, i, j, k) && interior) ? 1 : 0;
  }
  if (fbs) atomicAdd(a.counters + 1, (unsigned long long)fbs);
  if (hlls) atomicAdd(a.counters + 2, (unsigned long long)hlls);
}

// edge EMFs (arithmetic average of the four adjacent face EMFs, R32)
__device__ __forceinline__ double ct_ez(const CtArgs& a, const CtIdx& X, int i, int j, int k) {  // edge (i-1/2, j-1/2)
  const double e0 = -a.F[0][X.at(6, i, j - 1, k)], e1 = -a.F[0][X.at(6, i, j, k)];
  const double e2 = a.F[1][X.at(5, i - 1, j, k)], e3 = a.F[1][X.at(5, i, j, k)];
  return 0.25 * (((e0 + e1) + e2) + e3);
}
__device__ __forceinline__ double ct_ex(const CtArgs& a, const CtIdx& X, int i, int j, int k) {  // edge (j-1/2, k-1/2)
  const double e0 = -a.F[1][X.at(7, i, j, k - 1)], e1 = -a.F[1][X.at(7, i, j, k)];
  const double e2 = a.F[2][X.at(6, i, j - 1, k)], e3 = a.F[2][X.at(6, i, j, k)];
  return 0.25 * (((e0 + e1) + e2) + e3);
}
__device__ __forceinline__ double ct_ey(const CtArgs& a, const CtIdx& X, int i, int j, int k) {  // edge (i-1/2, k-1/2)
  const double e0 = -a.F[2][X.at(5, i - 1, j, k)], e1 = -a.F[2][X.at(5, i, j, k)];
  const double e2 = a.F[0][X.at(7, i, j, k - 1)], e3 = a.F[0][X.at(7, i, j, k)];
  return 0.25 * (((e0 + e1) + e2) + e3);
}

// 5-6 + RK epilogue
__global__ void __launch_bounds__(256) k_ct_update(CtArgs a) {
  const CtIdx X{a.nx, a.ny, a.nz, a.gz, (size_t)a.nx * a.ny, (size_t)a.nx * a.ny * 8};
  const size_t n = (size_t)a.nx * a.ny * a.nz;
  const double* lam = a.c.lam;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    int i, j, k;
    ct_decode(q, a.nx, a.ny, 0, i, j, k);
    double s[8];
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      double r = lam[0] * (a.F[0][X.at(f, i + 1, j, k)] - a.F[0][X.at(f, i, j, k)]);
      r = r + lam[1] * (a.F[1][X.at(f, i, j + 1, k)] - a.F[1][X.at(f, i, j, k)]);
      r = r + lam[2] * (a.F[2][X.at(f, i, j, k + 1)] - a.F[2][X.at(f, i, j, k)]);
      s[f] = __ldg(a.Uin + X.at(f, i, j, k)) - r;
    }
    const double ez = ct_ez(a, X, i, j, k), ex = ct_ex(a, X, i, j, k), ey = ct_ey(a, X, i, j, k);
    const double rbx = lam[1] * (ct_ez(a, X, i, j + 1, k) - ez) - lam[2] * (ct_ey(a, X, i, j, k + 1) - ey);
    const double rby = lam[2] * (ct_ex(a, X, i, j, k + 1) - ex) - lam[0] * (ct_ez(a, X, i + 1, j, k) - ez);
    const double rbz = lam[0] * (ct_ey(a, X, i + 1, j, k) - ey) - lam[1] * (ct_ex(a, X, i, j + 1, k) - ex);
    s[5] = __ldg(a.Uin + X.at(5, i, j, k)) - rbx;
    s[6] = __ldg(a.Uin + X.at(6, i, j, k)) - rby;
    s[7] = __ldg(a.Uin + X.at(7, i, j, k)) - rbz;
    double v[8];  // every U^n load before the first store (Uout may alias U^n)
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      const size_t o = X.at(f, i, j, k);
      v[f] = s[f];
      if (a.mode == 1) v[f] = 0.5 * (a.Un[o] + s[f]);
      else if (a.mode == 2) v[f] = (a.wa * a.Un[o]) + (a.wb * s[f]);
    }
#pragma unroll
    for (int f = 0; f < 8; ++f) a.Uout[X.at(f, i, j, k)] = v[f];
    // halo push: a boundary plane also into the z neighbour's ghost plane
    const size_t cell = (size_t)j * a.nx + i;
    if (a.push_dn && k < a.gz) {
      double* h = a.push_dn + (size_t)(a.push_dn_nz + a.gz + k) * X.ps + cell;
#pragma unroll
      for (int f = 0; f < 8; ++f) h[f * X.fs] = v[f];
    }
    if (a.push_up && k >= a.nz - a.gz) {
      double* h = a.push_up + (size_t)(k - (a.nz - a.gz)) * X.ps + cell;
#pragma unroll
      for (int f = 0; f < 8; ++f) h[f * X.fs] = v[f];
    }
  }
}

template <int RS, int REC>
static cudaError_t launch_ct_t(const CtArgs& a, int nsm, cudaStream_t st, cudaStream_t aux1, cudaStream_t aux2,
                               cudaEvent_t* ev) {
  const size_t pc = (size_t)a.nx * a.ny;
  auto grid = [&](size_t n, int bs, int per_sm) {
    return (unsigned)std::max<size_t>(1, std::min<size_t>((n + bs - 1) / bs, (size_t)nsm * per_sm));
  };
  k_ct_prim<<<grid(pc * (a.nz + 2 * a.G), 256, MHD_CTU_PER_SM), 256, 0, st>>>(a);
  // the three face kernels are independent: y and z on two auxiliary streams, joined before
  // the update
  cudaStream_t s1 = aux1 ? aux1 : st, s2 = aux2 ? aux2 : st;
  if (aux1) {
    cudaEventRecord(ev[0], st);
    cudaStreamWaitEvent(s1, ev[0], 0);
    cudaStreamWaitEvent(s2, ev[0], 0);
  }
  k_ct_face_x<RS, REC><<<grid((size_t)((a.nx + 31) / 32) * 32 * a.ny * (a.nz + 2), 128, 32), 128, 0, st>>>(a);
  const size_t segy = (size_t)a.nx * (a.nz + 2) * ((a.ny + kCtSeg - 1) / kCtSeg);
  const size_t segz = (size_t)a.nx * a.ny * ((a.nz + 1 + kCtSeg - 1) / kCtSeg);
  k_ct_face_m<1, RS, REC><<<grid(segy, 128, 32), 128, 0, s1>>>(a);
  k_ct_face_m<2, RS, REC><<<grid(segz, 128, 32), 128, 0, s2>>>(a);
  if (aux1) {
    cudaEventRecord(ev[1], s1);
    cudaEventRecord(ev[2], s2);
    cudaStreamWaitEvent(st, ev[1], 0);
    cudaStreamWaitEvent(st, ev[2], 0);
  }
  k_ct_update<<<grid(pc * a.nz, 256, MHD_CTU_PER_SM), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_ct_stage(int riemann, const CtArgs& a, int nsm, cudaStream_t st, cudaStream_t aux1,
                            cudaStream_t aux2, cudaEvent_t* ev) {
  const int lim = a.c.limiter;
  if (riemann) {
    if (lim == 2) return launch_ct_t<1, 2>(a, nsm, st, aux1, aux2, ev);
    if (lim == 1) return launch_ct_t<1, 1>(a, nsm, st, aux1, aux2, ev);
    return launch_ct_t<1, 0>(a, nsm, st, aux1, aux2, ev);
  }
  if (lim == 2) return launch_ct_t<0, 2>(a, nsm, st, aux1, aux2, ev);
  if (lim == 1) return launch_ct_t<0, 1>(a, nsm, st, aux1, aux2, ev);
  return launch_ct_t<0, 0>(a, nsm, st, aux1, aux2, ev);
}

// dt / c_h maxima with the face-averaged B (3.12 with R32)
__global__ void __launch_bounds__(256) k_ct_dt(DtArgs a) {
  const CtIdx X{a.nx, a.ny, a.nz_loc, a.gz, (size_t)a.nx * a.ny, (size_t)a.nx * a.ny * 8};
  const size_t n = (size_t)a.nx * a.ny * a.nz_loc;
  double M = 0.0, Sx = 0.0;
  unsigned long long bad = ULLONG_MAX;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    int i, j, k;
    ct_decode(q, a.nx, a.ny, 0, i, j, k);
    double u[8], v[8];
    ct_cell_cons(a.U, X, i, j, k, u);  // (b_z of plane k + 1: the ghost plane above the last one)
    if (bad_state<8>(u)) {
      bad = min(bad, (unsigned long long)(((a.zoff + k) * a.ny + j) * (long long)a.nx + i));
      continue;
    }
    cons2prim<8>(u, v, a.gm1, a.p_floor);
    double inv = 0.0, smax = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
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
    for (int r = 1; r < (int)(blockDim.x >> 5); ++r) {
      M = fmax(M, red[0][r]);
      Sx = fmax(Sx, red[1][r]);
    }
    atomicMax(a.out + 0, (unsigned long long)__double_as_longlong(M));
    atomicMax(a.out + 1, (unsigned long long)__double_as_longlong(Sx));
  }
  if (bad != ULLONG_MAX) atomicMin(a.bad, bad);
}

cudaError_t launch_ct_dt(const DtArgs& a, int nsm, cudaStream_t st) {
  const size_t n = (size_t)a.nx * a.ny * a.nz_loc;
  const unsigned g = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)nsm * 32);
  k_ct_dt<<<g > 0 ? g : 1, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace mhd
