/*
 * ulysses_attn.h — C ABI of the B200-native Ulysses sequence-parallel exact
 * attention library (libulysses_attn.so).
 *
 * What it computes.  PAPER.md P:165 (§2.5, "Sequence Parallel (SP)"):
 * DeepSpeed-Ulysses "partitions the input data along the sequence dimension",
 * then "employs an all-to-all collective communication to ensure that each GPU
 * receives a complete sequence, but only for a non-overlapping subset of the
 * attention heads", computes attention for those heads, and a second
 * all-to-all returns the result to sequence shards.  P:425 (§6.1): "two
 * all-to-all calls in the forward pass and two all-to-all calls + all reduce in
 * the backward pass per layer" (the all-reduce syncs weight gradients of the
 * model's projections; this op has no weights, so it issues exactly 2 + 2).
 * The local attention is exact softmax(Q K^T / sqrt(D)) V computed tile by
 * tile with an online softmax (§2.6 FlashAttention-2), so the N x N
 * score matrix never exists in memory.  No mask, no dropout, no bias.
 *
 * Conventions (all entry points):
 *  - Every tensor is caller-owned device memory (cudaMalloc / torch), dense
 *    row-major, 16-byte aligned.  The library never frees caller memory.
 *  - bf16 = IEEE bfloat16 (uint16 storage); fp32 = float.
 *  - Rank r of P owns tokens [r*N/P, (r+1)*N/P) ("sequence shard") and,
 *    after the all-to-all, heads [r*H/P, (r+1)*H/P) ("head shard").
 *  - scale = 1/sqrt(D); lse is the natural-log logsumexp of the scaled scores.
 *  - Calls are asynchronous and stream-ordered on `stream`.  For P > 1 they are
 *    COLLECTIVE: all P ranks call with identical (B, N, H, D, P) in the same
 *    order.  Shape validation happens on the host before anything is
 *    enqueued, so a shape error returns the same status on every rank and
 *    never hangs a peer.  In UA_A2A_PEER mode a peer that never signals (a
 *    rank that failed a per-rank check, died or diverged) is detected by a
 *    bounded device-side wait (60 s) and reported as UA_ERR_CUDA by the next
 *    call on that ctx; under UA_A2A_NCCL, NCCL's own error handling applies.
 *  - Errors: a non-UA_OK status; ua_last_error() returns a thread-local
 *    human-readable detail.  Asynchronous CUDA / NCCL faults surface as
 *    UA_ERR_CUDA / UA_ERR_NCCL on a later call.
 *  - There is no CPU fallback: without an sm_100 device every compute entry
 *    point fails with UA_ERR_UNSUPPORTED.
 */
#ifndef ULYSSES_ATTN_H_
#define ULYSSES_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ua_ctx ua_ctx; /* opaque: rank, P, device, NCCL communicator */
typedef struct CUstream_st* ua_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  UA_OK = 0,
  UA_ERR_INVALID_ARG = 1,       /* null / misaligned pointer, non-positive size, P != ctx P, workspace too small */
  UA_ERR_HEAD_DIVISIBILITY = 2, /* P > H or H % P != 0 (P:317 head limit) */
  UA_ERR_SEQ_DIVISIBILITY = 3,  /* N % P != 0; no padding */
  UA_ERR_UNSUPPORTED = 4,       /* D not in {32, 64, 72, 128}; N >= 2^31; no sm_100 device */
  UA_ERR_CUDA = 5,
  UA_ERR_NCCL = 6
} ua_status;

/* Library version string, e.g. "ulysses_attn 0.1 sm_100a". Never NULL. */
const char* ua_version(void);
const char* ua_status_string(ua_status s);
/* Detail of the last error on the calling thread ("" if none). */
const char* ua_last_error(void);

/* ------------------------------------------------------------- validation
 * Pure host check of a problem shape, no device access (S:238, S:244, S:248,
 * S:276).  Checked in this order: B, N, H, D, P >= 1 else
 * INVALID_ARG; P > H or H % P else HEAD_DIVISIBILITY; N % P else
 * SEQ_DIVISIBILITY; D not in {32,64,72,128} or N >= 2^31 else UNSUPPORTED. */
ua_status ua_validate(int64_t B, int64_t N, int H, int D, int P);

/* Workspace bytes the fwd / bwd calls need for this shape (0 for the forward
 * at P == 1).  Either output pointer may be NULL. */
ua_status ua_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* fwd_bytes, size_t* bwd_bytes);

/* ------------------------------------------------------------- context
 * ua_get_unique_id: rank 0 creates a 128-byte NCCL unique id; the caller
 * broadcasts it to the other ranks (e.g. over a torch.distributed group).
 * ua_ctx_create: binds the calling thread to `cuda_device` and, for P > 1,
 * creates the library's own NCCL communicator (ncclCommInitRank); `uid` is
 * ignored (may be NULL) when P == 1.  The ctx owns that communicator and is
 * released by ua_ctx_destroy.  ua_ctx_create and (once the peer transport has
 * run) ua_ctx_destroy are collective over the P ranks: the symmetric-memory
 * windows are registered and deregistered by all ranks together, so every rank
 * must call them. */
ua_status ua_get_unique_id(unsigned char uid[128]);
ua_status ua_ctx_create(const unsigned char* uid, int P, int rank, int cuda_device, ua_ctx** out);
ua_status ua_ctx_destroy(ua_ctx* ctx);
/* Per-ctx counters of collective traffic since creation (S:107-110 ledger):
 * a2a calls (a fused Q/K/V exchange counts as one call) and bytes this
 * rank sent to OTHER ranks. Either pointer may be NULL. */
ua_status ua_ctx_comm_stats(const ua_ctx* ctx, int64_t* a2a_calls, int64_t* a2a_bytes_sent);

/* Per-phase device timing (for benchmarks; off by default).  When enabled,
 * every fwd / bwd call records a CUDA event pair around each phase on the
 * call's stream.  ua_ctx_phase_times synchronises those events, ADDS the
 * elapsed milliseconds of each phase since the last query into ms[phase] and
 * launches[phase] (arrays of UA_NUM_PHASES, either may be NULL), and resets.
 * Phases: */
enum {
  UA_PHASE_PACK_FWD = 0,   /* sequence shard -> head chunks (q, k, v)      */
  UA_PHASE_A2A_FWD_IN,     /* all-to-all #1                                */
  UA_PHASE_ATTN_FWD,       /* attention forward kernel                     */
  UA_PHASE_A2A_FWD_OUT,    /* all-to-all #2                                */
  UA_PHASE_UNPACK_FWD,     /* head chunks -> out                           */
  UA_PHASE_PACK_BWD,       /* q, k, v, dO pack + Delta                     */
  UA_PHASE_A2A_BWD_IN,     /* all-to-all #3                                */
  UA_PHASE_ATTN_BWD,       /* attention backward kernel (+ dQ zeroing)     */
  UA_PHASE_DQ_FINALIZE,    /* fp32 dQ -> bf16                              */
  UA_PHASE_A2A_BWD_OUT,    /* all-to-all #4                                */
  UA_PHASE_UNPACK_BWD,     /* head chunks -> dq, dk, dv                    */
  UA_NUM_PHASES
};
ua_status ua_ctx_enable_timing(ua_ctx* ctx, int enable);

/* How the all-to-alls move data when P > 1:
 *  UA_A2A_NCCL  pack -> ncclSend/ncclRecv group -> unpack (default).
 *  UA_A2A_PEER  no NCCL on the data path: the pack kernel stores every head
 *               chunk straight into the owning GPU's receive buffer over
 *               NVLink, and the attention epilogues (O forward; dK, dV and the
 *               dQ finaliser backward) store each row straight into the token
 *               owner's buffer; completion is a system-scope flag per peer.
 *               The receive buffers are library-owned NCCL symmetric memory
 *               (ncclMemAlloc + ncclCommWindowRegister, collective, on first
 *               use per shape), addressed on every rank through the window's
 *               load/store-accessible peer pointers (NCCL >= 2.28).
 * Collective: every rank sets the same mode before its next call.
 * UA_ERR_UNSUPPORTED if P == 1 or the peer mappings cannot be created. */
enum { UA_A2A_NCCL = 0, UA_A2A_PEER = 1 };
ua_status ua_ctx_set_a2a_mode(ua_ctx* ctx, int mode);
ua_status ua_ctx_get_a2a_mode(const ua_ctx* ctx, int* mode);

/* Deterministic backward (in the first pass
 * "all matrices are the same" between the sequence-parallel and the
 * single-GPU run).  enable = 0 (default): dQ partial sums of the key tiles
 * are reduce-added into an fp32 accumulator by concurrent CTAs, so dQ may
 * differ in the last bits run to run.  enable != 0: dK, dV come from the
 * KV-stationary kernel without its dQ GEMM, and a second, query-stationary
 * kernel recomputes S and dP and sums dQ_i = sum_j dS_ij k_j over the key
 * tiles in ascending order in one accumulator (3 extra GEMMs per tile pair,
 * ~1.4x the backward flops), and every KV-stationary item sweeps the query
 * tiles from tile 0 whatever CTA runs it.  Ulysses: dq, dk, dv are then
 * bitwise reproducible and bitwise identical for every P (the same per-head
 * arithmetic in the same order).  LSS: bitwise reproducible for a given P
 * (its dK, dV are sums of P per-rank partials, so they depend on P).
 * Host-only setting, effective from the next call; every rank should set the
 * same value (the P-way identity needs it on all ranks). */
ua_status ua_ctx_set_deterministic(ua_ctx* ctx, int enable);
ua_status ua_ctx_get_deterministic(const ua_ctx* ctx, int* enable);
ua_status ua_ctx_phase_times(ua_ctx* ctx, double* ms, int64_t* launches);

/* ------------------------------------------------------------- forward
 * q, k, v : bf16 [B][N/P][H][D]   this rank's sequence shard (inputs)
 * out     : bf16 [B][N/P][H][D]   attention output, same shard (written)
 * lse     : fp32 [B][H/P][N]      logsumexp of this rank's HEAD shard over
 *                                 the full sequence (written; consumed by bwd)
 * workspace: device scratch of at least ua_workspace_size(...).fwd_bytes
 * P == 1: no communication; the kernels read q/k/v and write out in place.
 * P > 1 : pack -> all-to-all #1 (fused q,k,v) -> attention -> all-to-all #2
 *         -> unpack.  out must not alias q, k, v. */
ua_status ua_ulysses_attn_fwd(ua_ctx* ctx, const void* q, const void* k, const void* v, void* out, float* lse,
                              int64_t B, int64_t N, int H, int D, int P, void* workspace, size_t workspace_bytes,
                              ua_stream_t stream);

/* ------------------------------------------------------------- backward
 * Inputs: q, k, v, out, dout bf16 [B][N/P][H][D] (sequence shard; out is the
 * forward's output), lse fp32 [B][H/P][N] from the forward.
 * Outputs: dq, dk, dv bf16 [B][N/P][H][D] (gradients of the loss w.r.t. this
 * rank's shard of q, k, v).
 * Delta = rowsum(dout * out) is formed in fp32 in sequence space and shipped
 * with the all-to-all, so the backward needs no saved head-sharded state.
 * P > 1: pack(+Delta) -> all-to-all #3 -> attention bwd -> all-to-all #4 ->
 * unpack.  Outputs must not alias inputs. */
ua_status ua_ulysses_attn_bwd(ua_ctx* ctx, const void* q, const void* k, const void* v, const void* out,
                              const float* lse, const void* dout, void* dq, void* dk, void* dv, int64_t B, int64_t N,
                              int H, int D, int P, void* workspace, size_t workspace_bytes, ua_stream_t stream);

/* ------------------------------------------------------------- rank-local steps
 * The Ulysses path of ua_ulysses_attn_fwd / _bwd one step at a time, with no
 * communication: what ONE rank r of P computes between the all-to-alls
 * (§2.5; SURVEY §8(a) rows A1, A3, A6, B1, B3+B4, B6).  The fwd /
 * bwd entry points run exactly these internals; the all-to-all between them is
 * a byte-exact permutation (output[j] on rank i == input[i] on rank j),
 * so a caller holding every rank's buffers (e.g. a single-GPU test simulating P
 * ranks) can perform it with plain copies.  None of these calls needs a ctx;
 * all are stream-ordered and asynchronous; shapes are checked with
 * ua_validate(B, N, H, D, P) first, pointers must be non-NULL and 16-B aligned
 * (else UA_ERR_INVALID_ARG).  Layouts (elements, row-major, Hl = H/P, Nl = N/P):
 *
 * ua_pack_seq_to_head (A1; B1 with Delta): for w < ntensors (0..4)
 *   src[w] : bf16 [B][Nl][H][D]      this rank's sequence shard
 *   dst[w] : bf16 [P][Nl][B][Hl][D]  send chunk j = heads [j Hl, (j+1) Hl) of every local token
 *   dout, out, delta: all NULL, or all non-NULL: delta fp32 [P][Nl][B][Hl] =
 *            sum_d dout*out in fp32 (Delta_i = dO_i . O_i), packed like the
 *            tensors.  ntensors may be 0 when delta is requested.
 *   After the all-to-all, rank j's receive buffer [P][Nl][B][Hl][D] (chunk i
 *   from rank i) IS the head-shard tensor [N][B][Hl][D] the attention reads.
 * ua_unpack_head_to_seq (A6, B6): for w < ntensors (1..4)
 *   src[w] : bf16 [P][Nl][B][Hl][D]  chunk s = head block s, received from rank s
 *   dst[w] : bf16 [B][Nl][H][D]
 * ua_push_seq_to_head (A1+A2, B1+B3's input exchange fused; the UA_A2A_PEER
 * transport's kernel): stores rank `rank`'s chunks straight into every
 * destination's receive buffer: dst_rank[j] (j < P; device pointers this
 * process can write: a peer mapping, or local memory) holds
 * [ntensors][N][B][Hl][D] bf16 followed (if dout, out non-NULL) by Delta
 * [N][B][Hl] fp32; rank `rank`'s tokens land at rows [rank Nl, (rank+1) Nl).
 * No flag or fence is raised (the transport adds those).
 *
 * ua_head_attn_fwd (A3): exact attention of rank `rank`'s head shard
 * (heads [rank Hl, (rank+1) Hl)) over all N tokens:
 *   q, k, v : bf16 [N][B][Hl][D]     the all-to-all #1 receive buffers
 *   o       : bf16 [N][B][Hl][D]     = the all-to-all #2 send buffer (token block i -> rank i)
 *   lse     : fp32 [B][Hl][N]
 *   o_owner : NULL, or P pointers: then o must be NULL and the epilogue stores
 *             each output row straight into its token owner's [B][Nl][H][D]
 *             tensor o_owner[n / Nl] (A3 + A5 fused, UA_A2A_PEER).
 * ua_head_attn_bwd (B3 + B4): the backward of that head shard
 *   q, k, v, dout : bf16 [N][B][Hl][D];  lse fp32 [B][Hl][N];  delta fp32 [N][B][Hl]
 *   dq, dk, dv    : bf16 [N][B][Hl][D] (= the all-to-all #4 send buffers), or
 *   owners        : NULL, or 3P pointers (dq owners, dk owners, dv owners; each
 *                   [B][Nl][H][D]); then dq, dk, dv must be NULL and every row goes
 *                   straight to its token owner (B3 + B5 fused, UA_A2A_PEER).
 *   deterministic : as ua_ctx_set_deterministic.
 *   workspace     : >= ua_head_attn_bwd_workspace_size bytes (fp32 dQ accumulator
 *                   and the per-row (lse, Delta) table). */
ua_status ua_pack_seq_to_head(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t N, int H,
                              int D, int P, const void* dout, const void* out, float* delta, ua_stream_t stream);
ua_status ua_unpack_head_to_seq(const void* const* src, void* const* dst, int ntensors, int64_t B, int64_t N, int H,
                                int D, int P, ua_stream_t stream);
ua_status ua_push_seq_to_head(const void* const* src, int ntensors, void* const* dst_rank, int64_t B, int64_t N, int H,
                              int D, int P, int rank, const void* dout, const void* out, ua_stream_t stream);
ua_status ua_head_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t B, int64_t N,
                           int H, int D, int P, int rank, void* const* o_owner, ua_stream_t stream);
ua_status ua_head_attn_bwd_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* bytes);
ua_status ua_head_attn_bwd(const void* q, const void* k, const void* v, const void* dout, const float* lse,
                           const float* delta, void* dq, void* dk, void* dv, int64_t B, int64_t N, int H, int D, int P,
                           int rank, void* const* owners, int deterministic, void* workspace, size_t workspace_bytes,
                           ua_stream_t stream);

/* ------------------------------------------------------------- LSS chunking
 * One contiguous key segment ("Long Sequence Segmentation"):
 * exact attention of all N queries of a head-sharded problem over keys
 * [kv_begin, kv_end) only.  Operates on head-layout tensors (no comm):
 *   q, k, v : bf16 [B][N][Hx][D]   (Hx heads, e.g. one rank's head shard)
 *   o_seg   : fp32 [B][Hx][N][D]   segment output, normalised over the segment
 *   lse_seg : fp32 [B][Hx][N]      segment logsumexp
 * kv_begin must be a multiple of 128; 0 <= kv_begin < kv_end <= N. */
ua_status ua_attn_fwd_segment(const void* q, const void* k, const void* v, float* o_seg, float* lse_seg, int64_t B,
                              int64_t N, int Hx, int D, int64_t kv_begin, int64_t kv_end, ua_stream_t stream);
/* Exact merge (in place into a): lse_a <- logaddexp(lse_a, lse_b),
 * o_a <- e^{lse_a_old - lse} o_a + e^{lse_b - lse} o_b.  rows = B*Hx*N. */
ua_status ua_lse_merge(float* o_a, float* lse_a, const float* o_b, const float* lse_b, int64_t rows, int D,
                       ua_stream_t stream);
/* fp32 [B][Hx][N][D] -> bf16 [B][N][Hx][D] (final cast of a merged result). */
ua_status ua_f32_to_bf16_bnhd(const float* src, void* dst, int64_t B, int64_t N, int Hx, int D, ua_stream_t stream);

/* ------------------------------------------------------------- LSS sequence parallelism
 * The paper's other sequence-parallel strategy, Long Sequence Segmentation
 * (§1, §2.5: "sequences are divided into segments, with
 * each GPU computing a partial self-attention for its segment"; P:317, P:399:
 * it has no head limit, unlike Ulysses).  Reading (R14): rank r keeps
 * its contiguous query segment of ALL H heads; K and V of every rank are
 * gathered (one fused all-gather, 1 collective call); each rank computes exact
 * attention of its N/P queries over all N keys.  Backward: dQ stays local; dK,
 * dV partial sums over the local queries (fp32, all N keys) are summed over
 * ranks and scattered to the key owners (one fused reduce-scatter).  Per call
 * law: 1 collective in the forward, 2 in the backward (all-gather K/V again +
 * reduce-scatter); 0 at P = 1, where both reduce to plain attention.
 *   q, k, v, out, dout, dq, dk, dv : bf16 [B][N/P][H][D] (sequence shard)
 *   lse : fp32 [B][H][N/P]   (this rank's queries, all heads)
 * Constraints: N % P == 0, D in {32, 64, 72, 128}; any H >= 1 and any P (P > H is
 * allowed).  Same ownership / async / collective conventions as above.
 * Collective calls and bytes are counted in ua_ctx_comm_stats. */
ua_status ua_lss_validate(int64_t B, int64_t N, int H, int D, int P);
ua_status ua_lss_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* fwd_bytes, size_t* bwd_bytes);
ua_status ua_lss_attn_fwd(ua_ctx* ctx, const void* q, const void* k, const void* v, void* out, float* lse, int64_t B,
                          int64_t N, int H, int D, int P, void* workspace, size_t workspace_bytes, ua_stream_t stream);
ua_status ua_lss_attn_bwd(ua_ctx* ctx, const void* q, const void* k, const void* v, const void* out, const float* lse,
                          const void* dout, void* dq, void* dk, void* dv, int64_t B, int64_t N, int H, int D, int P,
                          void* workspace, size_t workspace_bytes, ua_stream_t stream);

/* LSS rank-local steps (no communication; the LSS analogue of the Ulysses
 * rank-local steps above, R14): what rank r computes between the collectives.
 *   q, out, dout, dq : bf16 [B][N/P][H][D]   this rank's query segment
 *   k_full, v_full   : bf16 [N][B][H][D]     every rank's keys / values in rank
 *                      order (the all-gather's output: rank p's tokens at rows
 *                      [p N/P, (p+1) N/P); for B == 1 each rank's [1][N/P][H][D]
 *                      shard is that block as is)
 *   lse              : fp32 [B][H][N/P]
 *   dk_part, dv_part : fp32 [N][B][H][D]     partial sums over THIS rank's
 *                      queries for all N keys (written; their sum over ranks,
 *                      scattered to the key owners, is dK, dV: the reduce-scatter)
 *   workspace        : >= ua_lss_rank_bwd_workspace_size bytes.
 * Constraints and errors as ua_lss_validate plus pointer checks. */
ua_status ua_lss_rank_fwd(const void* q, const void* k_full, const void* v_full, void* out, float* lse, int64_t B,
                          int64_t N, int H, int D, int P, ua_stream_t stream);
ua_status ua_lss_rank_bwd_workspace_size(int64_t B, int64_t N, int H, int D, int P, size_t* bytes);
ua_status ua_lss_rank_bwd(const void* q, const void* k_full, const void* v_full, const void* out, const float* lse,
                          const void* dout, void* dq, float* dk_part, float* dv_part, int64_t B, int64_t N, int H,
                          int D, int P, int deterministic, void* workspace, size_t workspace_bytes,
                          ua_stream_t stream);

/* ------------------------------------------------------------- attention layer
 * The rest of the paper's attention layer around the Ulysses attention
 * (SURVEY §8(f)-3): the Q/K/V and output projections and the SP group's
 * weight-gradient all-reduce (§5.4, §6.1: "two all-to-all
 * calls in the forward pass and two all-to-all calls + all reduce in the
 * backward pass per layer").  Reading (R16): bias-free projections,
 * y = x W^T, E = H * D, M = B * N/P tokens of this rank:
 *   forward   q|k|v = x Wq^T | x Wk^T | x Wv^T;  o = Ulysses attention;  y = o Wo^T
 *   backward  do = dy Wo, dWo = dy^T o;  (dq, dk, dv) = attention backward;
 *             dx = dq Wq + dk Wk + dv Wv;  dW_qkv = [dq^T x; dk^T x; dv^T x];
 *             dW_qkv and dWo summed over the P ranks (ONE fused NCCL all-reduce).
 *   x, y, dy, dx : bf16 [B][N/P][E]        (sequence shard)
 *   w_qkv        : bf16 [3E][E]            (rows: Wq, Wk, Wv; head h = rows h*D..h*D+D-1 of each)
 *   w_o          : bf16 [E][E]
 *   dw_qkv, dw_o : fp32 [3E][E], [E][E]    (full gradients, identical on every rank)
 *   saved        : caller-owned, ua_layer_sizes' saved_bytes: q, k, v, o, lse of the forward
 * GEMMs: this library's tcgen05 kernel (ua_gemm_bf16 below), bf16 operands, fp32 accumulation.
 * Collective calls per step: 2 forward, 3 backward (counted by ua_ctx_comm_stats).
 * Same validation (ua_validate) and conventions as the attention entry points. */
ua_status ua_layer_sizes(int64_t B, int64_t N, int H, int D, int P, size_t* saved_bytes, size_t* fwd_bytes,
                         size_t* bwd_bytes);
ua_status ua_layer_fwd(ua_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, void* y, void* saved,
                       int64_t B, int64_t N, int H, int D, int P, void* workspace, size_t workspace_bytes,
                       ua_stream_t stream);
ua_status ua_layer_bwd(ua_ctx* ctx, const void* x, const void* w_qkv, const void* w_o, const void* saved,
                       const void* dy, void* dx, float* dw_qkv, float* dw_o, int64_t B, int64_t N, int H, int D, int P,
                       void* workspace, size_t workspace_bytes, ua_stream_t stream);

/* The projection GEMM itself (sm_100a tcgen05, TMA, TMEM):
 *   C[M][N] = sum_{s < nseg} op(A[s]) op(B[s])   (fp32 accumulation; nseg 1..3
 *   concatenates the reduction dimension over separate buffers)
 *   a_mn = 0: A[s] bf16 [M][K] (op = identity);  a_mn = 1: A[s] bf16 [K][M] (op = transpose)
 *   b_mn = 0: B[s] bf16 [N][K] (op = transpose); b_mn = 1: B[s] bf16 [K][N] (op = identity)
 *   C: bf16 (c_f32 = 0) or fp32 [M][N].  Supported (a_mn, b_mn): (0,0) y = x W^T,
 *   (0,1) dx = g W, (1,1) dW = g^T x; else UA_ERR_CUDA (invalid value).
 * Pointers 16-B aligned; the leading dimensions (K, M or N) multiples of 8 elements.
 * M, N, K < 2^31.  Stream-ordered, asynchronous, no ctx. */
ua_status ua_gemm_bf16(int a_mn, int b_mn, int64_t M, int64_t N, int64_t K, const void* const* A, const void* const* B,
                       int nseg, void* C, int c_f32, ua_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* ULYSSES_ATTN_H_ */
