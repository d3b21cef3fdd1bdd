// attn_bwd_ws.cu — persistent, warp-specialised attention backward (sm_100a),
// D in {32, 64, 80 (= head dim 72 padded), 128}.
//
// Mathematics (FlashAttention-2's recompute backward):
//   P = exp(S - lse), dV += P^T dO, dS = P (dP - Delta), dK += scale dS^T Q,
//   dQ += scale dS K   (dQ partials reduced in fp32; scale applied later).
//
// Scheduling (the B200-specific part):
//  * persistent grid (<= one CTA per SM); work item = one 128-key tile of one
//    (b, h), items in head-major order, CTA c takes items c, c+G, ...  All
//    CTAs sweep their query tiles at the same rate, so at any moment they
//    touch a narrow window of Q / dO / dq rows of the same head (L2-resident
//    even at N = 188K, where one head's Q, dO and dq are ~96 MB).  Start tiles
//    are staggered over a window of kStagger tiles so only ~G/kStagger CTAs
//    reduce into the same dq tile at once.
//  * 16 warps: 0 TMA producer, 1 tcgen05.mma issuer, 4-7 elementwise for the
//    even 64-query half of each tile, 8-11 for the odd half, 12-15 dQ drain.
//    The halves have separate TMEM S^T / dP^T buffers, so the two elementwise
//    warpgroups and the tensor core work on different halves concurrently.
//  * Q / dO / (lse, Delta) arrive in a ring of 64-query half-tile slots; a
//    slot is released as soon as that half's dV / dK GEMMs are done.
//  * dQ: TMEM -> swizzled fp32 smem box -> TMA tensor reduce-add
//    (cp.reduce.async.bulk.tensor .add) into dq_acc.
//  * K, V stay in smem for the whole item (A operands of S^T, dP^T; B of dQ).
// TMEM (512 columns):  S^T[h] [64h, +64)  dP^T[h] [128+64h, +64)  dV [256, +D)
//   dK [256+D, +D)  dQ [256+2D, +D) for D <= 64.  D = 128 has no room for dQ:
//   it aliases dP^T [128, 256) and the next tile's dP^T GEMMs wait for the dQ
//   drain (the S^T GEMMs of the next tile run meanwhile).
// Variants (template kDq, macros):
//  * kDq = false (deterministic mode, ua_ctx_set_deterministic): no dQ GEMM /
//    staging / drain -- attn_bwd_dq.cu computes dQ query-stationary.  Every
//    item sweeps from query tile 0 (grid-independent dK / dV order).  For
//    D <= 80 the freed dQ columns hold a separate bf16 P^T per half (kSepP), the
//    next S^T GEMM is issued once S^T is in registers, and each half has two
//    elementwise warpgroups of 32 query columns (20 warps).
//  * UA_BWD_EW_SPLIT (off): the same 32-column split with the dQ path (24 warps).
//  * UA_BWD_KV_TMEM, UA_BWD_POLY_MOD, UA_BWD_STAGGER: see below.
#include <cstdio>
#include <cstdlib>

#include "attn_common.cuh"
#include "attn_kernels.h"
#include "trace.cuh"

#ifndef UA_BWD_POLY_MOD
#define UA_BWD_POLY_MOD 4   // every UA_BWD_POLY_MOD-th exp2 pair on the FMA pipe (0: none)
#endif
#ifndef UA_BWD_KV_TMEM
#define UA_BWD_KV_TMEM 1    // D <= 64: K, V copied into TMEM once per work item (TS MMAs)
#endif
#ifndef UA_BWD_SEP_P
#define UA_BWD_SEP_P 1      // dQ-less variant: separate TMEM P^T, next S^T under the exponentials
#endif
#ifndef UA_BWD_EW_SPLIT
#define UA_BWD_EW_SPLIT 0   // D <= 64 with dQ: two elementwise warpgroups of 32 query columns per half (24 warps); A/B: 853 vs 874 TFLOP/s at c4
#endif
#ifndef UA_BWD_DQ_LATE
#define UA_BWD_DQ_LATE 1    // issue the dQ GEMM after the next tile's S^T / dP^T GEMMs of the second half
#endif
#ifndef UA_BWD_BOX2
#define UA_BWD_BOX2 1       // D = 64: two dQ staging boxes (both halves of a tile's dQ reduced concurrently); A/B +8.6 % at N = 32K, = at c4
#endif
#ifndef UA_BWD_LDBATCH
#define UA_BWD_LDBATCH 0    // with dQ, no column split: all 64 S^T / dP^T columns of a half loaded with one wait (A/B: 838 vs 869 TFLOP/s at c4, spills)
#endif
#ifndef UA_BWD_SEP_POLY_MOD
#define UA_BWD_SEP_POLY_MOD 0   // same as UA_BWD_POLY_MOD for the separate-P^T variant (A/B: none is best)
#endif
#ifndef UA_BWD_PAIR
#define UA_BWD_PAIR 1       // clusters of 2 CTAs on adjacent key tiles of a head sharing each Q / dO half tile (TMA multicast)
#endif
#ifndef UA_BWD_DET_SLOTS
#define UA_BWD_DET_SLOTS 1  // dQ-less (deterministic) variant: no dS^T / staging buffers, their smem as ring slots
#endif
#ifndef UA_BWD_STAGGER
#define UA_BWD_STAGGER 16   // query-tile window the persistent CTAs' start tiles are spread over
#endif

namespace ua {

namespace {

template <int D, bool kDq = true>
struct BwdWsCfg {
  using G = TileGeom<D>;
  static constexpr int kThreads = 512;
  static constexpr int kStagger = UA_BWD_STAGGER;
  static constexpr bool kAliasDq = (256 + 3 * D) > 512;
  static constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + D;
  static constexpr uint32_t kColDQ = kAliasDq ? 128 : 256 + 2 * D;
  // D <= 64: K and V also live in TMEM (bf16 pairs, D/2 columns each) as the A
  // operands of S^T = K Q^T and dP^T = V dO^T, taking those reads off the smem port.
  static constexpr bool kKvTmem = UA_BWD_KV_TMEM && D <= 64;
  static constexpr uint32_t kColK = 256 + 3 * D, kColV = 256 + 3 * D + D / 2;
  static constexpr int kHalfBytes = 64 * D * 2;               // one [64][D] bf16 half tile
  // half-tile ring depth; UA_BWD_BOX2 trades one D == 64 slot for a second dQ staging box.
  // kDq = false (deterministic mode) with UA_BWD_DET_SLOTS: no dS^T or dQ staging buffers, their
  // shared memory goes to the ring (A/B at c4 and N = 32K: neutral, 795 vs 798 and 809 vs 811 TFLOP/s).
  static constexpr bool kDqBufs = kDq || !UA_BWD_DET_SLOTS;
  static constexpr int kSlots =
      !kDqBufs ? (D == 128 ? 4 : 8) : (D == 128 ? 3 : (D == 80 ? 4 : (UA_BWD_BOX2 && D == 64 ? 5 : 6)));
  static constexpr int kSlotBytes = 2 * kHalfBytes;            // Q_h + dO_h
  static constexpr int kNumDs = !kDqBufs ? 0 : (kAliasDq ? 1 : 2);   // dS^T smem buffers
  static constexpr int kDsBytes = 128 * 128 * 2;
  static constexpr int kStageBoxes =   // 16 KB fp32 staging boxes for dQ
      !kDqBufs ? 0 : ((D == 128 || (UA_BWD_BOX2 && D == 64)) ? 2 : 1);
  static constexpr int kBoxBytes = 128 * 32 * 4;
  static constexpr int kLsedBytes = 128 * 4;                   // per slot: 64 x -lse*log2e, 64 x -Delta
  static constexpr bool kPolyExp = UA_BWD_POLY_MOD > 0;
  static constexpr int kSmemBytes = 1024 + 2 * G::kTileBytes + kSlots * kSlotBytes + kNumDs * kDsBytes +
                                    kStageBoxes * kBoxBytes + kSlots * kLsedBytes + 512;
  // Without the dQ GEMM (deterministic mode) the dQ columns hold a separate bf16
  // P^T per half (32 columns each), so the next S^T GEMM can overwrite S^T as
  // soon as the elementwise warps have loaded it (D = 128 has no dQ columns).
  static constexpr uint32_t kColP = (kKvTmem && kColV + D / 2 + 64 <= 512) ? kColV + D / 2 : kColDQ;
  static constexpr bool kSepPFits = !kAliasDq && (kColP == kColDQ ? (kKvTmem ? kColK : 512u) : 512u) >= kColP + 64;
  static_assert(kSmemBytes <= 232448, "smem budget");
};

// Separate-P^T pipeline of the dQ-less variant (needs 64 spare TMEM columns).
template <int D, bool kDq>
__host__ __device__ constexpr bool ws_sep_p() { return !kDq && BwdWsCfg<D>::kSepPFits && UA_BWD_SEP_P; }
// Column split of the elementwise work: each 64-query half has two warpgroups of
// 32 query columns (kSepP: 20 warps; with the dQ drain warpgroup: 24 warps).
template <int D, bool kDq>
__host__ __device__ constexpr bool ws_ew_split() { return kDq && UA_BWD_EW_SPLIT && D <= 64; }
// Clusters of two CTAs that own key tiles 2m and 2m+1 of the same head and sweep
// the same query tiles in the same order: every Q / dO half tile is read from L2
// once per pair and multicast into both CTAs' ring slots (each CTA issues one of
// the two loads), halving the per-SM Q / dO L2 read traffic.
template <int D, bool kDq>
__host__ __device__ constexpr bool ws_pair() { return kDq && UA_BWD_PAIR; }
template <int D, bool kDq>
__host__ __device__ constexpr int ws_threads() {
  return ws_sep_p<D, kDq>() ? 640 : (ws_ew_split<D, kDq>() ? 768 : 512);
}

// kDq = false (deterministic mode): dK, dV only; dQ comes from the query-stationary
// attn_bwd_dq_kernel (attn_bwd_dq.cu), so no dS^T staging, dQ GEMM or reduction here.
template <int D, bool kDq>
__global__ void __launch_bounds__(ws_threads<D, kDq>(), 1) attn_bwd_ws_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdWsCfg<D, kDq>;
  constexpr bool kAlias = C::kAliasDq && kDq;   // dQ shares TMEM with dP^T (D = 128)
  constexpr bool kSepP = ws_sep_p<D, kDq>();
  constexpr bool kSplit = kSepP || ws_ew_split<D, kDq>();   // two elementwise warpgroups per half
  constexpr int kEwArrive = kSplit ? 256 : 128;   // arrivals per half on s_loaded / p_ready / ds_ready
  constexpr int kEwCols = kSplit ? 32 : 64;       // query columns per elementwise thread and half tile
  constexpr int kEwEnd = kSplit ? 20 : 12;        // first warp after the elementwise warpgroups
  constexpr bool kBatch = kDq && !kSplit && UA_BWD_LDBATCH;   // 128 data registers per elementwise thread
  constexpr bool kPair = ws_pair<D, kDq>();
  using G = TileGeom<D>;
  constexpr int kSl = C::kSlots;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-B aligned, stays in the shared window
  uint8_t* sK = smem;
  uint8_t* sV = sK + G::kTileBytes;
  uint8_t* sSlots = sV + G::kTileBytes;                        // [kSl] { Q_h, dO_h }
  uint8_t* sdS = sSlots + kSl * C::kSlotBytes;                 // [kNumDs] dS^T [128 keys][128 q], 2 SW128 atoms
  uint8_t* sStage = sdS + C::kNumDs * C::kDsBytes;             // [kStageBoxes] fp32 [128][32] SW128
  float* sLsed = reinterpret_cast<float*>(sStage + C::kStageBoxes * C::kBoxBytes);  // [kSl][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLsed + kSl * 128);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* dq_full = bars + 2;
  uint64_t* dq_empty = bars + 3;
  uint64_t* acc_full = bars + 4;
  uint64_t* acc_free = bars + 5;
  uint64_t* sdp_full = bars + 6;      // [2] per half
  uint64_t* ds_ready = bars + 8;      // [2] per half
  uint64_t* ds_free = bars + 10;      // [kNumDs]
  uint64_t* slot_full = bars + 12;    // [kSl]
  uint64_t* slot_empty = slot_full + kSl;
  uint64_t* kv_tmem = slot_empty + kSl;  // K, V copied into TMEM for this item
  uint64_t* dp_full = kv_tmem + 1;    // [2] kSepP: dP^T[h] computed (sdp_full then signals S^T alone)
  uint64_t* s_loaded = dp_full + 2;   // [2] kSepP: S^T[h] in registers, may be overwritten
  uint64_t* p_ready = s_loaded + 2;   // [2] kSepP: P^T[h] stored
  uint64_t* p_free = p_ready + 2;     // [2] kSepP: dV GEMM has read P^T[h]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_q = (p.n + 127) / 128;
  const int n_pad = n_q * 128;
  const int n_kt = (p.n_kv + 127) / 128;
  // Work units: one key tile (kPair: a pair of adjacent key tiles, one per CTA of
  // the cluster, both sweeping the same query tiles) of one (b, h), head-major.
  const int crank = kPair ? int(cluster_ctarank()) : 0;
  const int unit0 = kPair ? int(cluster_id_x()) : int(blockIdx.x);
  const int n_units_grid = kPair ? int(num_clusters_x()) : int(gridDim.x);
  const int n_kp = kPair ? (n_kt + 1) / 2 : n_kt;   // key tiles (pairs) per head; an odd tail pairs with an all-OOB tile
  const int n_items = p.batch * p.heads * n_kp;
  auto item_kt = [&](int u) { return kPair ? 2 * (u % n_kp) + crank : u % n_kp; };
  auto item_bh = [&](int u) { return u / n_kp; };
  // Deterministic mode (no dQ reduction to spread out): every item sweeps from
  // tile 0, so the dK / dV summation order does not depend on the grid (P-invariant).
  const int start = kDq ? int((int64_t(unit0) * C::kStagger) / n_units_grid) % n_q : 0;
  auto qslot = [&](int s) { return sSlots + s * C::kSlotBytes; };
  auto doslot = [&](int s) { return sSlots + s * C::kSlotBytes + C::kHalfBytes; };

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128);
    mbar_init(acc_full, 1);
    mbar_init(acc_free, 256);
    mbar_init(kv_tmem, 128);
    for (int h = 0; h < 2; ++h) {
      mbar_init(&sdp_full[h], 1);
      mbar_init(&ds_ready[h], kEwArrive);
      mbar_init(&dp_full[h], 1);
      mbar_init(&s_loaded[h], kEwArrive);
      mbar_init(&p_ready[h], kEwArrive);
      mbar_init(&p_free[h], 1);
    }
    for (int i = 0; i < C::kNumDs; ++i) mbar_init(&ds_free[i], 1);
    for (int s = 0; s < kSl; ++s) {
      mbar_init(&slot_full[s], 1);
      mbar_init(&slot_empty[s], kPair ? 2 : 1);   // kPair: released by both CTAs' MMAs (the slot is refilled for both)
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync();   // the peer's barriers exist before any multicast load / commit
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  // kSepP: 640 threads launch with 96 registers each; the producer / MMA
  // warpgroup gives 40 of them to the four elementwise warpgroups (56 + 4 x 104
  // <= 5 x 96: setmaxnreg.inc can only take what the CTA's own warps released).
  // Each role branch re-balances first thing so ptxas sees which limit applies.
// 24-warp split with dQ: 768 threads launch with 80 registers; 56 (producer / MMA)
// + 4 x 80 (elementwise) + 104 (dQ drain) = 6 x 80.
// kBatch (512 threads at 128): 56 + 2 x 168 (elementwise) + 112 (dQ drain) <= 4 x 128.
#define UA_BWD_REGS_LOW() do { if constexpr (kSplit || kBatch) setmaxnreg_dec<56>(); } while (0)
#define UA_BWD_REGS_HIGH() do { if constexpr (kSepP) setmaxnreg_inc<104>(); else if constexpr (kBatch) setmaxnreg_inc<168>(); } while (0)
#define UA_BWD_REGS_DRAIN() do { if constexpr (kSplit) setmaxnreg_inc<104>(); else if constexpr (kBatch) setmaxnreg_dec<112>(); } while (0)

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    UA_BWD_REGS_LOW();
    if (lane == 0) {
      tma_prefetch_desc(&p.tm_qh);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      tma_prefetch_desc(&p.tm_doh);
      int T = 0, it = 0;
      for (int item = unit0; item < n_items; item += n_units_grid, ++it) {
        const int kt = item_kt(item), bh = item_bh(item);
        const int b = bh / p.heads, h = bh % p.heads;
        if (it > 0) mbar_wait(kv_empty, (it - 1) & 1);
        mbar_arrive_expect_tx(kv_full, 2 * G::kTileBytes);
        for (int a = 0; a < G::kAtoms; ++a) {
          tma_load_4d(sK + a * G::kAtomBytes, &p.tm_k, kv_full, a * G::kAtomCols, kt * 128, h, b, kEvictFirst);
          tma_load_4d(sV + a * G::kAtomBytes, &p.tm_v, kv_full, a * G::kAtomCols, kt * 128, h, b, kEvictFirst);
        }
        const float* lsed_bh = reinterpret_cast<const float*>(p.lsed) + int64_t(bh) * n_pad * 2;
        for (int t = 0; t < n_q; ++t, ++T) {
          const int tile = (start + t) % n_q;
          const float* lsed_tile = lsed_bh + int64_t(tile) * 256;  // [128 nl][128 nd]
          for (int hh = 0; hh < 2; ++hh) {
            const int U = 2 * T + hh, s = U % kSl;
            UA_TEV(0, U, 1);
            if (U >= kSl) mbar_wait(&slot_empty[s], ((U / kSl) & 1) ^ 1);
            UA_TEV(0, U, 2);
            mbar_arrive_expect_tx(&slot_full[s], C::kSlotBytes + C::kLsedBytes);
            if constexpr (kPair) {  // Q_h (CTA 0) or dO_h (CTA 1), multicast into both CTAs' slot s
              for (int a = 0; a < G::kAtoms; ++a)
                tma_load_4d_mc((crank == 0 ? qslot(s) : doslot(s)) + a * 64 * G::kSw, crank == 0 ? &p.tm_qh : &p.tm_doh,
                               &slot_full[s], a * G::kAtomCols, tile * 128 + 64 * hh, h, b, uint16_t(3), kEvictLast);
            } else {
              for (int a = 0; a < G::kAtoms; ++a) {
                tma_load_4d(qslot(s) + a * 64 * G::kSw, &p.tm_qh, &slot_full[s], a * G::kAtomCols,
                            tile * 128 + 64 * hh, h, b, kEvictLast);
                tma_load_4d(doslot(s) + a * 64 * G::kSw, &p.tm_doh, &slot_full[s], a * G::kAtomCols,
                            tile * 128 + 64 * hh, h, b, kEvictLast);
              }
            }
            bulk_load(sLsed + s * 128, lsed_tile + 64 * hh, 256, &slot_full[s]);
            bulk_load(sLsed + s * 128 + 64, lsed_tile + 128 + 64 * hh, 256, &slot_full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    UA_BWD_REGS_LOW();
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16_f32(128, 64, false, false);  // S^T, dP^T half: N = 64 queries
      const uint32_t idesc_g = idesc_bf16_f32(128, D, false, true);    // dV, dK: A = TMEM, B MN-major
      const uint32_t idesc_q = idesc_bf16_f32(128, D, true, true);     // dQ: A, B MN-major
      const uint32_t sKa = smem_u32(sK), sVa = smem_u32(sV), sSa = smem_u32(sSlots), sdSa = smem_u32(sdS);
      auto q_at = [&](int U) { return sSa + (U % kSl) * C::kSlotBytes; };
      auto do_at = [&](int U) { return sSa + (U % kSl) * C::kSlotBytes + C::kHalfBytes; };
      auto wait_slot = [&](int U) {
        mbar_wait(&slot_full[U % kSl], (U / kSl) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int T, int hh) {   // S^T[hh] = K Q_h^T
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          if constexpr (C::kKvTmem)
            mma_ts(tbase + C::kColS + 64 * hh, tbase + C::kColK + kk * 8, kmajor_desc_r<D, 64>(q_at(2 * T + hh), kk),
                   idesc_s, kk > 0 ? 1u : 0u);
          else
            mma_ss(tbase + C::kColS + 64 * hh, kmajor_desc_r<D, 128>(sKa, kk),
                   kmajor_desc_r<D, 64>(q_at(2 * T + hh), kk), idesc_s, kk > 0 ? 1u : 0u);
        }
      };
      auto issue_dp = [&](int T, int hh) {  // dP^T[hh] = V dO_h^T
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          if constexpr (C::kKvTmem)
            mma_ts(tbase + C::kColDP + 64 * hh, tbase + C::kColV + kk * 8,
                   kmajor_desc_r<D, 64>(do_at(2 * T + hh), kk), idesc_s, kk > 0 ? 1u : 0u);
          else
            mma_ss(tbase + C::kColDP + 64 * hh, kmajor_desc_r<D, 128>(sVa, kk),
                   kmajor_desc_r<D, 64>(do_at(2 * T + hh), kk), idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sdp_full[hh]);
      };
      if constexpr (kSepP) {
        // S^T(T+1) right after the elementwise warps have loaded S^T(T); dV(T)
        // once P^T(T) is stored; dK(T) and then dP^T(T+1) once dS^T(T) is.
        auto issue_s1 = [&](int T1, int hh) {
          issue_s(T1, hh);
          mma_commit(&sdp_full[hh]);
        };
        auto issue_dp1 = [&](int T1, int hh) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            if constexpr (C::kKvTmem)
              mma_ts(tbase + C::kColDP + 64 * hh, tbase + C::kColV + kk * 8,
                     kmajor_desc_r<D, 64>(do_at(2 * T1 + hh), kk), idesc_s, kk > 0 ? 1u : 0u);
            else
              mma_ss(tbase + C::kColDP + 64 * hh, kmajor_desc_r<D, 128>(sVa, kk),
                     kmajor_desc_r<D, 64>(do_at(2 * T1 + hh), kk), idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(&dp_full[hh]);
        };
        int T = 0, it = 0;
        for (int item = unit0; item < n_items; item += n_units_grid, ++it) {
          mbar_wait(C::kKvTmem ? kv_tmem : kv_full, it & 1);
          tc_fence_after();
          for (int hh = 0; hh < 2; ++hh) {
            wait_slot(2 * T + hh);
            issue_s1(T, hh);
            issue_dp1(T, hh);
          }
          if (it > 0) {
            mbar_wait(acc_free, (it - 1) & 1);  // previous item's dV / dK drained
            tc_fence_after();
          }
          // Fixed issue order (half 0, then half 1, per tile): the dV / dK
          // summation order must not depend on timing.  (Issuing whichever half
          // is ready first measured no faster and breaks reproducibility.)
          for (int t = 0; t < n_q; ++t, ++T) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int U = 2 * T + hh;
              const bool more = t + 1 < n_q;
              if (more) {
                mbar_wait(&s_loaded[hh], T & 1);
                wait_slot(2 * (T + 1) + hh);
                issue_s1(T + 1, hh);
              }
              mbar_wait(&p_ready[hh], T & 1);
              tc_fence_after();
              const uint32_t acc = (t > 0 || hh > 0) ? 1u : 0u;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_ts(tbase + C::kColDV, tbase + C::kColP + 32 * hh + kk * 8, mnmajor_desc_r<D, 64>(do_at(U), kk),
                       idesc_g, (acc || kk > 0) ? 1u : 0u);
              mma_commit(&p_free[hh]);
              mbar_wait(&ds_ready[hh], T & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)  // dS^T queries [32g, 32g+32) were packed at column 32g
                mma_ts(tbase + C::kColDK, tbase + C::kColDP + 64 * hh + kk * 8 + (kk >= 2 ? 16 : 0),
                       mnmajor_desc_r<D, 64>(q_at(U), kk), idesc_g, (acc || kk > 0) ? 1u : 0u);
              mma_commit(&slot_empty[U % kSl]);
              if (more) issue_dp1(T + 1, hh);
            }
          }
          mma_commit(acc_full);
          mma_commit(kv_empty);
        }
      } else {
      int T = 0, it = 0;
      for (int item = unit0; item < n_items; item += n_units_grid, ++it) {
        mbar_wait(C::kKvTmem ? kv_tmem : kv_full, it & 1);
        tc_fence_after();
        // first tile of the item
        wait_slot(2 * T);
        issue_s(T, 0);
        if constexpr (!kAlias) issue_dp(T, 0);
        wait_slot(2 * T + 1);
        issue_s(T, 1);
        if constexpr (kAlias) {
          if (T > 0) {
            mbar_wait(dq_empty, (T - 1) & 1);
            tc_fence_after();
          }
          issue_dp(T, 0);
        }
        issue_dp(T, 1);
        if (it > 0) {
          mbar_wait(acc_free, (it - 1) & 1);  // previous item's dV / dK drained
          tc_fence_after();
        }
        for (int t = 0; t < n_q; ++t, ++T) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int U = 2 * T + hh;
            UA_TEV(1, T, 1 + 4 * hh);
            mbar_wait(&ds_ready[hh], T & 1);
            UA_TEV(1, T, 2 + 4 * hh);
            tc_fence_after();
            const uint32_t acc = (t > 0 || hh > 0) ? 1u : 0u;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts(tbase + C::kColDV, tbase + C::kColS + 64 * hh + kk * 8 + (kSplit && kk >= 2 ? 16 : 0),
                     mnmajor_desc_r<D, 64>(do_at(U), kk), idesc_g, (acc || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts(tbase + C::kColDK, tbase + C::kColDP + 64 * hh + kk * 8 + (kSplit && kk >= 2 ? 16 : 0),
                     mnmajor_desc_r<D, 64>(q_at(U), kk),
                     idesc_g, (acc || kk > 0) ? 1u : 0u);
            if constexpr (kPair)
              mma_commit_mc(&slot_empty[U % kSl], uint16_t(3));   // free in both CTAs' view of the slot
            else
              mma_commit(&slot_empty[U % kSl]);
            UA_TEV(1, T, 3 + 4 * hh);
            auto issue_dq = [&]() {  // dQ(T) = dS K
              if (!C::kAliasDq && T > 0) {
                UA_TEV(1, T, 9);
                mbar_wait(dq_empty, (T - 1) & 1);
                UA_TEV(1, T, 10);
                tc_fence_after();
              }
              const uint32_t ds = sdSa + (T % C::kNumDs) * C::kDsBytes;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                mma_ss(tbase + C::kColDQ, mnmajor_desc_r<128, 128>(ds, kk), mnmajor_desc_r<D, 128>(sKa, kk), idesc_q,
                       kk > 0 ? 1u : 0u);
              mma_commit(dq_full);
              UA_TEV(1, T, 11);
              mma_commit(&ds_free[T % C::kNumDs]);
            };
            // Without the dQ / dP^T aliasing, the next tile's S^T / dP^T GEMMs of this
            // half go first (their sdp_full commit then does not wait for the dQ GEMM,
            // which reads only smem and its own TMEM columns): UA_BWD_DQ_LATE.
            constexpr bool kDqLate = UA_BWD_DQ_LATE && !kAlias;
            if (kDq && hh == 1 && !kDqLate) issue_dq();
            if (t + 1 < n_q) {  // next tile, this half
              wait_slot(2 * (T + 1) + hh);
              issue_s(T + 1, hh);
              if constexpr (!kAlias) {
                issue_dp(T + 1, hh);
              } else if (hh == 1) {  // dP^T of the next tile overwrites the dQ region
                mbar_wait(dq_empty, T & 1);
                tc_fence_after();
                issue_dp(T + 1, 0);
                issue_dp(T + 1, 1);
              }
            }
            if (kDq && hh == 1 && kDqLate) issue_dq();
          }
        }
        mma_commit(acc_full);
        mma_commit(kv_empty);
      }
      }  // !kSepP
    }
    __syncwarp();
  } else if (warp >= 4 && warp < kEwEnd) {
    // ------------------------------------------------------------ elementwise (half hh)
    UA_BWD_REGS_HIGH();
    const int hh = kSplit ? (warp - 4) / 8 : (warp - 4) / 4;
    const int g = kSplit ? ((warp - 4) / 4) % 2 : 0;   // kSplit: query columns [32g, 32g+32) of the half
    const int quad = warp % 4;
    const int j = quad * 32 + lane;  // key row within the tile
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const uint32_t colS = C::kColS + 64 * hh + 32 * g, colDP = C::kColDP + 64 * hh + 32 * g;
    const float c = p.scale_log2;
    const float2 c2 = make_float2(c, c);
    int T = 0, it = 0;
    for (int item = unit0; item < n_items; item += n_units_grid, ++it) {
      const int kt = item_kt(item), bh = item_bh(item);
      const int b = bh / p.heads, h = bh % p.heads;
      if constexpr (C::kKvTmem) {
        if (hh == 0 && g == 0) {  // copy this item's K, V rows (row j per thread) into TMEM as bf16 pairs
          mbar_wait(kv_full, it & 1);
          const uint32_t sw = (uint32_t(j * G::kSw) >> 7) & uint32_t(G::kSw / 16 - 1);
          uint32_t rk[D / 2], rv[D / 2];
#pragma unroll
          for (int ch = 0; ch < D / 8; ++ch) {
            const uint32_t off = j * G::kSw + ((ch ^ sw) * 16);
            const uint4 k4 = *reinterpret_cast<const uint4*>(sK + off);
            const uint4 v4 = *reinterpret_cast<const uint4*>(sV + off);
            rk[4 * ch] = k4.x; rk[4 * ch + 1] = k4.y; rk[4 * ch + 2] = k4.z; rk[4 * ch + 3] = k4.w;
            rv[4 * ch] = v4.x; rv[4 * ch + 1] = v4.y; rv[4 * ch + 2] = v4.z; rv[4 * ch + 3] = v4.w;
          }
          if constexpr (D == 64) {
            tmem_st32(t_lane + C::kColK, rk);
            tmem_st32(t_lane + C::kColV, rv);
          } else {
            tmem_st16(t_lane + C::kColK, rk);
            tmem_st16(t_lane + C::kColV, rv);
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(kv_tmem);
        }
      }
      if constexpr (kSepP) {
        for (int t = 0; t < n_q; ++t, ++T) {
          const int U = 2 * T + hh, s = U % kSl;
          mbar_wait(&slot_full[s], (U / kSl) & 1);  // (lse, Delta) of this half landed
          mbar_wait(&sdp_full[hh], T & 1);          // S^T(T) computed
          tc_fence_after();
          const uint32_t nl_s = smem_u32(sLsed + s * 128 + 32 * g);
          const uint32_t nd_s = nl_s + 64 * 4;
          uint32_t rs[32];
          tmem_ld16(t_lane + colS, *reinterpret_cast<uint32_t(*)[16]>(rs));
          tmem_ld16(t_lane + colS + 16, *reinterpret_cast<uint32_t(*)[16]>(rs + 16));
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(&s_loaded[hh]);                  // the next S^T GEMM may overwrite S^T[hh]
          float pv[32];
          uint32_t pk_p[16];
#pragma unroll
          for (int x = 0; x < 32; x += 4) {
            const float4 nl = lds128(nl_s + x * 4);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float2 arg = __ffma2_rn(make_float2(__uint_as_float(rs[x + 2 * u]), __uint_as_float(rs[x + 2 * u + 1])),
                                            c2, u == 0 ? make_float2(nl.x, nl.y) : make_float2(nl.z, nl.w));
              const bool poly = UA_BWD_SEP_POLY_MOD > 0 &&
                                ((x / 2 + u) % (UA_BWD_SEP_POLY_MOD > 0 ? UA_BWD_SEP_POLY_MOD : 1)) == 1;
              const float2 pp = poly ? exp2_poly2(arg) : make_float2(ex2(arg.x), ex2(arg.y));
              pv[x + 2 * u] = pp.x;
              pv[x + 2 * u + 1] = pp.y;
              pk_p[x / 2 + u] = pack_bf16x2(pp.x, pp.y);
            }
          }
          if (T > 0) mbar_wait(&p_free[hh], (T - 1) & 1);  // dV(T-1) has read P^T[hh]
          tc_fence_after();
          tmem_st16(t_lane + C::kColP + 32 * hh + 16 * g, pk_p);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&p_ready[hh]);
          mbar_wait(&dp_full[hh], T & 1);           // dP^T(T) computed
          tc_fence_after();
          uint32_t rdA[16], rdB[16];
          tmem_ld16(t_lane + colDP, rdA);
          tmem_ld16(t_lane + colDP + 16, rdB);
          tmem_ld_wait();
          uint32_t pk_ds[16];
#pragma unroll
          for (int x = 0; x < 32; x += 4) {
            const uint32_t* rd = x < 16 ? rdA + x : rdB + (x - 16);
            const float4 nd = lds128(nd_s + x * 4);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float2 dd = __fadd2_rn(make_float2(__uint_as_float(rd[2 * u]), __uint_as_float(rd[2 * u + 1])),
                                           u == 0 ? make_float2(nd.x, nd.y) : make_float2(nd.z, nd.w));
              const float2 ds = __fmul2_rn(make_float2(pv[x + 2 * u], pv[x + 2 * u + 1]), dd);
              pk_ds[x / 2 + u] = pack_bf16x2(ds.x, ds.y);
            }
          }
          tmem_st16(t_lane + colDP, pk_ds);           // dS^T over this group's dP^T columns (all read)
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&ds_ready[hh]);
        }
      } else
      for (int t = 0; t < n_q; ++t, ++T) {
        const int U = 2 * T + hh, s = U % kSl;
        if (j == 0) UA_TEV(2 + hh, T, 1);
        mbar_wait(&slot_full[s], (U / kSl) & 1);  // (lse, Delta) of this half landed
        if (kDq && T >= C::kNumDs) mbar_wait(&ds_free[T % C::kNumDs], ((T / C::kNumDs) & 1) ^ 1);
        mbar_wait(&sdp_full[hh], T & 1);
        if (j == 0) UA_TEV(2 + hh, T, 2);
        tc_fence_after();
        const uint32_t atom = smem_u32(sdS + (T % C::kNumDs) * C::kDsBytes + hh * (128 * 128) + j * 128);
        const uint32_t nl_s = smem_u32(sLsed + s * 128 + 32 * g);
        const uint32_t nd_s = nl_s + 64 * 4;
#pragma unroll
        // TMEM loads software-pipelined: chunk k+1's S^T / dP^T columns are in
        // flight while chunk k is computed (P^T / dS^T stores only ever touch
        // columns already read).
        // kBatch: the half's 64 S^T and 64 dP^T columns in four loads and one
        // wait (all exponentials of the half independent); else two 16-column
        // buffers, chunk k+1 in flight while chunk k is computed.
        uint32_t rsv[kBatch ? 64 : 32], rdv[kBatch ? 64 : 32];
        if constexpr (kBatch) {
          tmem_ld32(t_lane + colS, rsv);
          tmem_ld32(t_lane + colS + 32, rsv + 32);
          tmem_ld32(t_lane + colDP, rdv);
          tmem_ld32(t_lane + colDP + 32, rdv + 32);
        } else {
          tmem_ld16(t_lane + colS, *reinterpret_cast<uint32_t(*)[16]>(rsv));
          tmem_ld16(t_lane + colDP, *reinterpret_cast<uint32_t(*)[16]>(rdv));
        }
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < kEwCols; cc += 16) {
          uint32_t* rs = kBatch ? rsv + cc : rsv + 16 * ((cc / 16) & 1);
          uint32_t* rd = kBatch ? rdv + cc : rdv + 16 * ((cc / 16) & 1);
          if (!kBatch && cc + 16 < kEwCols) {
            tmem_ld16(t_lane + colS + cc + 16, *reinterpret_cast<uint32_t(*)[16]>(rsv + 16 * (((cc / 16) & 1) ^ 1)));
            tmem_ld16(t_lane + colDP + cc + 16, *reinterpret_cast<uint32_t(*)[16]>(rdv + 16 * (((cc / 16) & 1) ^ 1)));
          }
          uint32_t pk_p[8], pk_ds[8];
#pragma unroll
          for (int x = 0; x < 16; x += 4) {
            const float4 nl = lds128(nl_s + (cc + x) * 4);
            const float4 nd = lds128(nd_s + (cc + x) * 4);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float2 arg = __ffma2_rn(make_float2(__uint_as_float(rs[x + 2 * u]), __uint_as_float(rs[x + 2 * u + 1])),
                                            c2, u == 0 ? make_float2(nl.x, nl.y) : make_float2(nl.z, nl.w));
              const bool poly = C::kPolyExp && ((x / 2 + u) % (UA_BWD_POLY_MOD > 0 ? UA_BWD_POLY_MOD : 1)) == 1;
              const float2 pp = poly ? exp2_poly2(arg) : make_float2(ex2(arg.x), ex2(arg.y));
              const float2 dd = __fadd2_rn(make_float2(__uint_as_float(rd[x + 2 * u]), __uint_as_float(rd[x + 2 * u + 1])),
                                           u == 0 ? make_float2(nd.x, nd.y) : make_float2(nd.z, nd.w));
              const float2 ds = __fmul2_rn(pp, dd);
              pk_p[x / 2 + u] = pack_bf16x2(pp.x, pp.y);
              pk_ds[x / 2 + u] = pack_bf16x2(ds.x, ds.y);
            }
          }
          tmem_st8(t_lane + colS + cc / 2, pk_p);
          tmem_st8(t_lane + colDP + cc / 2, pk_ds);
#pragma unroll
          for (int qd = 0; qd < 2 * int(kDq); ++qd) {
            const int chunk = (4 * g + (cc / 8) + qd) ^ (j & 7);
            sts128(atom + chunk * 16, pk_ds[4 * qd], pk_ds[4 * qd + 1], pk_ds[4 * qd + 2], pk_ds[4 * qd + 3]);
          }
          if (!kBatch && cc + 16 < kEwCols) tmem_ld_wait();
        }
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        if (j == 0) UA_TEV(2 + hh, T, 3);
        mbar_arrive(&ds_ready[hh]);
      }
      // ------------------------------------------------ dV (hh=0) / dK (hh=1) epilogue
      if (g != 0) continue;  // kSepP: the first warpgroup of each half drains dV / dK
      mbar_wait(acc_full, it & 1);
      tc_fence_after();
      const int krow = kt * 128 + j;
      const bool valid = krow < p.n_kv;
      const ViewArg& dst_v = hh == 0 ? p.dv : p.dk;
      const uint32_t col = hh == 0 ? C::kColDV : C::kColDK;
      const float sc = hh == 0 ? 1.f : p.scale;
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(dst_v.base) + b * dst_v.sb + h * dst_v.sh +
                           int64_t(krow) * dst_v.sn;
      const PeerOut& po = hh == 0 ? p.dv_peer : p.dk_peer;
      const int d_io = D % 32 == 0 ? D : p.d_io;  // columns >= d_io (padding of head dim 72) are not stored
      if (po.base[0] != nullptr && valid) {  // fused return all-to-all: the token owner's buffer
        const int owner = int(krow / po.nl);
        dst = reinterpret_cast<__nv_bfloat16*>(po.base[owner]) + ((b * po.nl + (krow - owner * po.nl)) * po.H + po.h0 + h) * d_io;
      }
      if (p.kv_f32) {  // fp32 partial sums (LSS: reduce-scattered across ranks afterwards)
        float* fdst = reinterpret_cast<float*>(dst_v.base) + b * dst_v.sb + h * dst_v.sh + int64_t(krow) * dst_v.sn;
#pragma unroll
        for (int cc = 0; cc < D; cc += 16) {
          uint32_t r[16];
          tmem_ld16(t_lane + col + cc, r);
          tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int x = 0; x < 16; x += 4)
              if (cc + x < d_io)
              *reinterpret_cast<float4*>(fdst + cc + x) =
                  make_float4(__uint_as_float(r[x]) * sc, __uint_as_float(r[x + 1]) * sc,
                              __uint_as_float(r[x + 2]) * sc, __uint_as_float(r[x + 3]) * sc);
          }
        }
      } else
#pragma unroll
      for (int cc = 0; cc < D; cc += 16) {
        uint32_t r[16];
        tmem_ld16(t_lane + col + cc, r);
        tmem_ld_wait();
        uint32_t pk[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) pk[x] = pack_bf16x2(__uint_as_float(r[2 * x]) * sc, __uint_as_float(r[2 * x + 1]) * sc);
        if (valid) {
          *reinterpret_cast<uint4*>(dst + cc) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          if (cc + 8 < d_io) *reinterpret_cast<uint4*>(dst + cc + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      tc_fence_before();
      mbar_arrive(acc_free);
    }
  } else if (kDq && warp >= kEwEnd) {
    // ------------------------------------------------------------ dQ drain
    const int quad = warp % 4;
    const int r = quad * 32 + lane;  // query row within the tile
    UA_BWD_REGS_DRAIN();
    const bool leader = threadIdx.x == kEwEnd * 32;
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    // columns held in registers per round; D = 80 drains 96 columns (3 boxes of 32: the
    // TMA reduce drops columns >= 72 as out of bounds, TMEM columns 496..511 are spare)
    constexpr int kCols = D == 128 ? 64 : (D == 80 ? 96 : D);
    constexpr int kRounds = D == 128 ? 2 : 1;
    int T = 0;
    for (int item = unit0; item < n_items; item += n_units_grid) {
      const int bh = item_bh(item);
      for (int t = 0; t < n_q; ++t, ++T) {
        const int tile = (start + t) % n_q;
        if (r == 0) UA_TEV(4, T, 1);
        mbar_wait(dq_full, T & 1);
        if (r == 0) UA_TEV(4, T, 2);
        tc_fence_after();
#pragma unroll
        for (int rd = 0; rd < kRounds; ++rd) {
          float acc[kCols];
#pragma unroll
          for (int cc = 0; cc < kCols; cc += 16) {
            uint32_t x[16];
            tmem_ld16(t_lane + C::kColDQ + rd * kCols + cc, x);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[cc + e] = __uint_as_float(x[e]);
          }
          if (rd == kRounds - 1) {
            tc_fence_before();
            mbar_arrive(dq_empty);
            if (r == 0) UA_TEV(4, T, 3);
          }
          // kCols / 32 boxes through kStageBoxes staging boxes
#pragma unroll
          for (int cb0 = 0; cb0 < kCols / 32; cb0 += C::kStageBoxes) {
            if (leader) bulk_wait_read<0>();   // previous reduction has read the staging boxes
            named_bar_sync(1, 128);
#pragma unroll
            for (int sb = 0; sb < C::kStageBoxes; ++sb) {
              const uint32_t srow = smem_u32(sStage + sb * C::kBoxBytes + r * 128);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const int e = 32 * (cb0 + sb) + 4 * q4;
                sts128f(srow + ((q4 ^ (r & 7)) * 16), acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
              }
            }
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (leader) {
#pragma unroll
              for (int sb = 0; sb < C::kStageBoxes; ++sb)
                tma_reduce_add_2d(&p.tm_dq, sStage + sb * C::kBoxBytes, rd * kCols + 32 * (cb0 + sb),
                                  bh * n_pad + tile * 128);
              bulk_commit();
            }
          }
        }
      }
    }
    if (leader) bulk_wait<0>();
  } else {
    UA_BWD_REGS_LOW();  // warps 2, 3 (and the idle dQ-drain warpgroup without the dQ GEMM)
  }
#undef UA_BWD_REGS_LOW
#undef UA_BWD_REGS_HIGH
#undef UA_BWD_REGS_DRAIN

  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync();   // no multicast load / commit may target a CTA that has exited
  if (warp == 1) tmem_free<512>(tbase);
}

template <int D, bool kDq>
cudaError_t launch_bwd_ws_impl(const BwdParams& p, cudaStream_t stream) {
  using C = BwdWsCfg<D, kDq>;
  const int num_sms = current_num_sms();
  if (num_sms <= 0) return cudaErrorNoDevice;
  cudaError_t e = set_max_smem(attn_bwd_ws_kernel<D, kDq>, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  const int n_kt = (p.n_kv + 127) / 128;
  constexpr bool kPair = ws_pair<D, kDq>();
  const int64_t units = int64_t(p.batch) * p.heads * (kPair ? (n_kt + 1) / 2 : n_kt);
#if UA_TRACE
  trace_reset();
#endif
  if constexpr (kPair) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(ws_threads<D, kDq>());
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int max_clusters = 0;   // co-resident pairs (an SM left alone in its GPC cannot host half of one)
    cfg.gridDim = dim3(2 * (num_sms / 2));
    e = cudaOccupancyMaxActiveClusters(&max_clusters, attn_bwd_ws_kernel<D, kDq>, &cfg);
    if (std::getenv("UA_VERBOSE"))
      std::fprintf(stderr, "[ua] attn_bwd_ws<%d>: %d SMs, max active clusters of 2: %d (%s)\n", D, num_sms,
                   max_clusters, cudaGetErrorString(e));
    if (e != cudaSuccess || max_clusters < 1) max_clusters = num_sms / 2;
    cudaGetLastError();
    const int64_t pairs = units < max_clusters ? units : max_clusters;
    cfg.gridDim = dim3(unsigned(2 * pairs));
    e = cudaLaunchKernelEx(&cfg, attn_bwd_ws_kernel<D, kDq>, p);
    if (e != cudaSuccess) return e;
  } else {
    const int grid = int(units < num_sms ? units : num_sms);
    attn_bwd_ws_kernel<D, kDq><<<grid, ws_threads<D, kDq>(), C::kSmemBytes, stream>>>(p);
  }
#if UA_TRACE
  trace_dump("bwd");
#endif
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_bwd_ws(const BwdParams& p, int D, cudaStream_t stream) {
  if (p.deterministic) {  // dK, dV here; dQ by the query-stationary kernel (no cross-CTA reduction)
    cudaError_t e = cudaSuccess;
    switch (D) {
      case 32: e = launch_bwd_ws_impl<32, false>(p, stream); break;
      case 64: e = launch_bwd_ws_impl<64, false>(p, stream); break;
      case 72: e = launch_bwd_ws_impl<80, false>(p, stream); break;
      case 128: e = launch_bwd_ws_impl<128, false>(p, stream); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    return launch_attn_bwd_dq(p, D, stream);
  }
  switch (D) {
    case 32: return launch_bwd_ws_impl<32, true>(p, stream);
    case 64: return launch_bwd_ws_impl<64, true>(p, stream);
    case 72: return launch_bwd_ws_impl<80, true>(p, stream);   // padded MMA head dim, p.d_io = 72
    case 128: return launch_bwd_ws_impl<128, true>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ua
