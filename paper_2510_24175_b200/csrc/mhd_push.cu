// mhd_push.cu — the NCCL side of the halo push (MHD_HALO_PUSH): the stage
// kernel's epilogue stores its g boundary planes straight into the z neighbours' ghost planes
// (the halo of the next stage, here produced by the compute that precedes it
// instead of a separate exchange).  The state arrays are NCCL symmetric windows
// (ncclMemAlloc + ncclCommWindowRegister); this file turns them into plain peer pointers once,
// and provides the per-stage ordering point: a one-CTA LSA barrier over the node's ranks after
// each pushing stage, so that no rank starts the next stage before its neighbours' pushes have
// landed (and no rank pushes into an array a neighbour is still reading).
#include <nccl.h>
#include <nccl_device.h>

#include <cstring>

#include "mhd_kernels.h"

namespace mhd {

// peer pointers of the windows' storage plane 0: out[2 r] = down neighbour's, out[2 r + 1] = up
// neighbour's array of role r (U0, U1, U2); null for a missing window or neighbour
__global__ void k_peer_ptrs(ncclWindow_t w0, ncclWindow_t w1, ncclWindow_t w2, int down, int up, void** out) {
  const ncclWindow_t w[3] = {w0, w1, w2};
  for (int r = 0; r < 3; ++r) {
    out[2 * r] = (w[r] && down >= 0) ? ncclGetPeerPointer(w[r], 0, down) : nullptr;
    out[2 * r + 1] = (w[r] && up >= 0) ? ncclGetPeerPointer(w[r], 0, up) : nullptr;
  }
}

cudaError_t push_peer_pointers(void* const win[3], int down, int up, double* out[6], cudaStream_t st) {
  void** d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 6 * sizeof(void*), st);
  if (e != cudaSuccess) return e;
  k_peer_ptrs<<<1, 1, 0, st>>>((ncclWindow_t)win[0], (ncclWindow_t)win[1], (ncclWindow_t)win[2], down, up, d);
  void* h[6];
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  cudaStreamSynchronize(st);
  for (int i = 0; i < 6; ++i) out[i] = (double*)h[i];
  return e;
}

// every rank of the LSA team arrives and waits (release/acquire at system scope): the pushes
// of the stage launched before it on this stream, and of the same stage on every rank, are
// visible after it
__global__ void __launch_bounds__(128) k_push_barrier(ncclDevComm dc) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

cudaError_t push_barrier(const void* devcomm, cudaStream_t st) {
  k_push_barrier<<<1, 128, 0, st>>>(*(const ncclDevComm*)devcomm);
  return cudaGetLastError();
}

// host side: the device communicator with one LSA barrier (stored opaquely by the context)
size_t devcomm_bytes() { return sizeof(ncclDevComm); }
int devcomm_create(void* comm, void* out) {
  ncclDevCommRequirements req;
  memset(&req, 0, sizeof req);
  req.lsaBarrierCount = 1;
  return ncclDevCommCreate((ncclComm_t)comm, &req, (ncclDevComm*)out) == ncclSuccess ? 0 : -1;
}
void devcomm_destroy(void* comm, const void* dc) { ncclDevCommDestroy((ncclComm_t)comm, (const ncclDevComm*)dc); }
int lsa_team_size(void* comm) { return ncclTeamLsa((ncclComm_t)comm).nRanks; }

}  // namespace mhd
