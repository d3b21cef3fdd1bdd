// capi_internal.h — definitions shared by the C ABI translation units
// (capi.cpp: attention entry points; layer.cpp: the projection layer).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/ulysses_attn.h"
#include "kernels/attn_kernels.h"

struct ua_ctx {
  int P = 1;
  int rank = 0;
  int device = 0;
  ncclComm_t comm = nullptr;
  int64_t a2a_calls = 0;
  int64_t a2a_bytes = 0;
  // phase timing
  bool timing = false;
  struct Rec {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  // NVLink peer-store all-to-all (UA_A2A_PEER): library-owned buffers in NCCL
  // symmetric memory (ncclMemAlloc + ncclCommWindowRegister), load/store-accessible
  // from every rank (peer[k] = rank k's copy, peer[rank] = local).
  int a2a_mode = UA_A2A_NCCL;
  int deterministic = 0;  // ua_ctx_set_deterministic: query-stationary dQ, no cross-CTA reduction
  struct PeerBuf {
    void* local = nullptr;
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    void* peer[ua::kMaxPeers] = {};
  };
  PeerBuf flags, fwd_in, fwd_out, bwd_in, bwd_out;
  // Host-mapped error word of the bounded peer waits (peer.cu wait_copy_kernel):
  // peer_err_host != 0 after a wait timed out; peer_err is its device alias.
  int* peer_err_host = nullptr;
  int* peer_err = nullptr;
  int64_t step_fwd = 0, step_bwd = 0;
  cudaEvent_t get_event() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};


namespace ua_internal {
// Thread-local error detail + status (ua_last_error).
ua_status fail(ua_status s, const char* fmt, ...);
// Releases per-ctx state of the projection layer (layer.cpp; none at present); called by ua_ctx_destroy.
void layer_release(ua_ctx* ctx);
// UA_OK if the current device is an sm_100 GPU, else UA_ERR_UNSUPPORTED (no CPU fallback).
ua_status check_device();
// Writes the P per-rank addresses of window w (ncclGetPeerPointer) to out_dev[0..P) (kernels/nccl_window.cu).
cudaError_t launch_lsa_ptrs(ncclWindow_t w, int P, void** out_dev, cudaStream_t stream);
}  // namespace ua_internal

#define UA_CUDA(expr)                                                                                    \
  do {                                                                                                   \
    cudaError_t e_ = (expr);                                                                             \
    if (e_ != cudaSuccess) return ua_internal::fail(UA_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

#define UA_NCCL(expr)                                                                                     \
  do {                                                                                                    \
    ncclResult_t r_ = (expr);                                                                             \
    if (r_ != ncclSuccess) return ua_internal::fail(UA_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)

#define UA_TRY(expr)            \
  do {                          \
    ua_status s_ = (expr);      \
    if (s_ != UA_OK) return s_; \
  } while (0)
