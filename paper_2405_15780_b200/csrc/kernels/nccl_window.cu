// nccl_window.cu — peer pointers of an NCCL symmetric-memory window (NCCL 2.28
// device API): the UA_A2A_PEER transport's receive buffers are ncclMemAlloc'd,
// registered collectively with ncclCommWindowRegister(..., NCCL_WIN_COLL_SYMMETRIC),
// and every rank's copy is load/store-accessible over NVLink ("LSA").  One tiny
// kernel reads the window's per-peer addresses once per registration; the
// transport kernels (peer.cu, the attention epilogues) then store through them.
#include <nccl.h>
#include <nccl_device.h>

#include "../capi_internal.h"

namespace {

__global__ void lsa_ptrs_kernel(ncclWindow_t w, int P, void** out) {
  const int peer = threadIdx.x;
  if (peer < P) out[peer] = ncclGetPeerPointer(w, 0, peer);
}

}  // namespace

namespace ua_internal {

cudaError_t launch_lsa_ptrs(ncclWindow_t w, int P, void** out_dev, cudaStream_t stream) {
  lsa_ptrs_kernel<<<1, 32, 0, stream>>>(w, P, out_dev);
  return cudaGetLastError();
}

}  // namespace ua_internal
