// mhd_kernels.h — internal interface between the host library (mhd_api.cu) and the kernels.
#pragma once
#include <cuda.h>  // CUtensorMap (the type only: the encoder is fetched through the runtime)
#include <cuda_runtime.h>

#include <cstdint>

#include "mhd_device.cuh"

namespace mhd {

// Internal state layout: [z + gz][f][y][x], x fastest, x/y unpadded (ghosts
// resolved by index wrap/clamp), gz = 2 ghost planes per side in 3D (0 otherwise).
struct StageArgs {
  // 3D: TMA descriptor of Uin as the 4D tensor [storage plane][field][y][x] (fp64, no swizzle),
  // box = one plane window of the CTA's tile with its x/y halo; set by launch_stage (tma = 1)
  alignas(64) CUtensorMap tmap;
  // 3D PLM (MHD_ZTMA): the own-cell tile of two planes for the next z job, boxes matching the
  // y- and x-flux buffers they are staged in ([f][TY+1][32] and [f][TY][34])
  alignas(64) CUtensorMap tmap_fy;
  alignas(64) CUtensorMap tmap_fx;
  int tma;
  const double* Uin;  // stage input, read with the stencil
  const double* Un;   // stage 2: U^n, read pointwise (aliases Uout)
  double* Uout;       // stage 1: U*, stage 2: U^n (in place)
  int nx, ny, nz_loc; // local interior extents
  int gz;             // z ghost planes per side
  long long zoff;     // global z offset of this slab
  long long nz_glob;  // global nz
  int bcx[2], bcy[2]; // 0 periodic, 1 outflow
  int kz;             // z planes per CTA
  int zb, ze;         // local z range of cells this launch updates (interior/boundary split)
  int stage;          // 1, 2 (, 3): selects the bad-cell slot
  int mode;           // epilogue: 0 S(U); 1 0.5 (U^n + S) (RK2); 2 (a U^n) + (b S) (RK3)
  int last;           // last stage of the step: apply the GLM damping
  double wa, wb;      // RK3 weights a, b
  StageConsts c;
  unsigned long long* counters;  // [p_floors, plm_fallbacks, hlld_to_hll]
  unsigned long long* bad;       // [4] lowest bad global linear index per stage (0 = dt pass)
  // halo push (3D slabs, MHD_HALO_PUSH): the z neighbours' arrays of Uout's role (storage plane
  // 0; peer memory: an NCCL symmetric window or an in-process slab), null where there is none.
  // Interior plane m < gz is also stored to the down neighbour's top ghost plane
  // push_dn_nz + gz + m, plane m >= nz_loc - gz to the up neighbour's bottom ghost plane
  // m - (nz_loc - gz): the next stage's z halo, written by this stage's epilogue
  double* push_dn;
  double* push_up;
  int push_dn_nz;
};

struct DtArgs {
  const double* U;
  int nx, ny, nz_loc, gz;
  long long zoff;
  double gamma, gm1, p_floor;
  double idx[3];
  unsigned long long* out;  // [2] bit patterns of max inv and max s
  unsigned long long* bad;  // stage-0 slot
};

cudaError_t launch_stage(int dim, int nv, int riemann, const StageArgs& a, cudaStream_t st);

// constrained transport (mhd_ct.cu): 3D, periodic, one GPU or z slabs, 8 fields (b on faces)
struct CtArgs {
  const double* Uin;  // stage input (padded [z+gz][8][y][x], z ghost planes filled)
  const double* Un;   // U^n for the RK epilogue
  double* Uout;
  double* V;          // scratch: cell-centred primitives
  double* F[3];       // scratch: face fluxes per direction (induction entries = face EMFs)
  int nx, ny, nz, gz;
  int G;              // reconstruction half-width (2 PLM, 3 WENO-Z); gz = G + 1
  long long zoff;     // global z offset of this slab (bad-cell indices)
  int stage, mode, last;
  double wa, wb;
  StageConsts c;
  unsigned long long* counters;  // [p_floors, plm_fallbacks, hlld_to_hll]
  unsigned long long* bad;       // [4] per stage
  double* push_dn;               // halo push, as in StageArgs (null: none)
  double* push_up;
  int push_dn_nz;
};
cudaError_t launch_ct_stage(int riemann, const CtArgs& a, int nsm, cudaStream_t st, cudaStream_t aux1,
                            cudaStream_t aux2, cudaEvent_t* ev);

// the WENO-Z stage of the 3D GLM path as five launches (mhd_split.cu)
constexpr int NVS = 9;
struct SplitArgs {
  const double* Uin;  // stage input (padded [z+gz][9][y][x], z ghost planes filled, gz = 3)
  const double* Un;   // U^n for the RK epilogue
  double* Uout;
  double* V;          // scratch: primitives, padded like U
  double* F[3];       // scratch: face fluxes [k][f][j][i], row pitch px, ny + 1 rows, k in [0, nz]
  int nx, ny, nz, gz;
  int px;             // split_row_pitch(nx)
  long long zoff, nz_glob;
  int bcx[2], bcy[2];
  int stage, mode, last;
  double wa, wb;
  StageConsts c;
  unsigned long long* counters;  // [p_floors, plm_fallbacks, hlld_to_hll]
  unsigned long long* bad;       // [4] per stage
  double* push_dn;               // halo push, as in StageArgs (null: none)
  double* push_up;
  int push_dn_nz;
};
cudaError_t launch_split_stage(int riemann, const SplitArgs& a, int nsm, cudaStream_t st, cudaStream_t aux1,
                               cudaStream_t aux2, cudaEvent_t* ev);
inline int split_row_pitch(int nx) { return (nx + 1 + 31) / 32 * 32; }
cudaError_t launch_ct_dt(const DtArgs& a, int nsm, cudaStream_t st);
// halo push over NCCL symmetric windows (mhd_push.cu); win: ncclWindow_t of U0, U1, U2 (or null)
cudaError_t push_peer_pointers(void* const win[3], int down, int up, double* out[6], cudaStream_t st);
cudaError_t push_barrier(const void* devcomm, cudaStream_t st);
size_t devcomm_bytes();
int devcomm_create(void* comm, void* out);
void devcomm_destroy(void* comm, const void* dc);
int lsa_team_size(void* comm);
int stage_tile_rows(int dim, int limiter);
int stage_ctas_per_sm(int dim, int nv, int riemann, int limiter);  // resident CTAs per SM of the stage kernel
cudaError_t launch_dt(int dim, int nv, const DtArgs& a, int nsm, cudaStream_t st);
cudaError_t launch_pack(const double* src, double* dst, int nv, int nx, int ny, int nzl, int gz, int to_internal,
                        int nsm, cudaStream_t st);
cudaError_t launch_validate(const double* U, int nv, int nx, int ny, int nzl, int gz, long long zoff, double gm1,
                            unsigned long long* bad, int nsm, cudaStream_t st, int check_p);
cudaError_t launch_store_words(unsigned long long* host_dst, const unsigned long long* src, int n, cudaStream_t st);
cudaError_t launch_fast_ops(const double* A, const double* B, long long n, double* out, int* okm, cudaStream_t st);
cudaError_t launch_face_flux(int nv, int riemann, const double* VL, const double* VR, long long n,
                             const StageConsts& c, double* F, unsigned long long* nhll, cudaStream_t st);

}  // namespace mhd
