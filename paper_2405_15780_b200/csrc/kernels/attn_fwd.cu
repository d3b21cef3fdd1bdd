// attn_fwd.cu — exact attention forward for one head shard, sm_100a.
//
// Computes, for every (b, h) of the launch and query row i,
//   o_i = sum_j softmax_j(s_ij) v_j,  s_ij = q_i.k_j / sqrt(D),
//   lse_i = ln sum_j exp(s_ij)
// over the key range [kv_begin, kv_end): PAPER.md P:165 (§2.5, each GPU runs
// ordinary attention over the complete sequence for its head subset) computed
// FlashAttention-style (§2.6: tile the score matrix, never write it
// to HBM).  With kv_begin = 0, kv_end = N it is the full attention; a strict
// sub-range is one LSS segment merged later by lse_merge.
//
// Design (B200-first, not a port of any FA2/ROCm code):
//  * one CTA = 2 query tiles of 128 rows of one (b, h); 12 warps:
//      warp 0      TMA producer (Q once, K/V ring of kStages tiles)
//      warp 1      tcgen05.mma issuer (single elected thread) + TMEM owner
//      warps 4-7   softmax for query tile 0 (one row per thread)
//      warps 8-11  softmax for query tile 1
//  * TMEM (512 cols), D <= 64: S0 S1 [0,256) | P0 P1 [256,384) | O0 O1 [384,512).
//    S_t = Q_t K_j^T (SS MMA, M=128,N=128,K=D).  The softmax loads S_t into
//    registers and releases it (s_free), so S_t(j+1) is computed while it
//    exponentiates; it writes bf16 P_t (64 cols, packed pairs) and
//    O_t += P_t V_j runs as a TS MMA (A = P from TMEM, B = V from smem,
//    MN-major).  D = 128 has no room for separate P: S0 S1 | O0 O1, P
//    overwrites S_t in place and the two tiles ping-pong (one tile's GEMMs
//    under the other tile's softmax).
//  * online softmax in the log2 domain with a lazy max: the running max m used
//    for the exponent is only raised (and O, l rescaled) when a row's max grows
//    by more than 8 (a factor 256); the final o = O / l is exact either way
//    because O and l carry the same stale max.
#include "attn_common.cuh"
#include "attn_kernels.h"
#include "trace.cuh"

// Tuning knobs (defaults are the shipped configuration; scripts/ab.py builds
// variants with -D overrides).
#ifndef UA_FWD_SPLIT
#define UA_FWD_SPLIT 1      // D <= 64: the column-split kernel of attn_fwd_split.cu (4 softmax warpgroups)
#endif
#ifndef UA_FWD_SEP_P
#define UA_FWD_SEP_P 1      // separate TMEM P buffers when D <= 64: the next Q K^T overlaps this tile's softmax
#endif
#ifndef UA_FWD_POLY_MOD
#define UA_FWD_POLY_MOD 3   // every UA_FWD_POLY_MOD-th exp2 pair on the FMA pipe (0: none)
#endif
#ifndef UA_FWD_PINGPONG
#define UA_FWD_PINGPONG 0   // the two softmax warpgroups take turns for their exp2 phases (A/B: slower)
#endif
#ifndef UA_FWD_LDBATCH
#define UA_FWD_LDBATCH 1    // issue the four S chunk loads back to back with one wait
#endif
#ifndef UA_FWD_LATEP
#define UA_FWD_LATEP 0      // separate-P mode: exponentiate the whole tile before waiting for the P buffer
#endif
#ifndef UA_FWD_MAXNREG
#define UA_FWD_MAXNREG 224  // >0: setmaxnreg the softmax warpgroups up to this many registers (0: off)
#endif
#ifndef UA_FWD_POLY_MAXD
#define UA_FWD_POLY_MAXD 128  // largest head dim whose softmax offloads exp2 pairs to the FMA pipe (A/B at D = 128: +0.4-1.4 %)
#endif
#ifndef UA_FWD_RELOAD
#define UA_FWD_RELOAD 0     // two TMEM passes over S (max, then exp); A/B: slower, kept as an option
#endif

namespace ua {

namespace {

#ifndef UA_FWD_POLY16
#define UA_FWD_POLY16 4     // >0: this many of every 16 exp2 pairs on the FMA pipe, spread evenly (overrides POLY_MOD)
#endif

// Which of the 16 exp2 pairs of a 32-column chunk go to the FMA-pipe polynomial.
__device__ __forceinline__ constexpr bool poly_pair(int i) {
  if (UA_FWD_POLY16 > 0) return ((i + 1) * UA_FWD_POLY16) / 16 - (i * UA_FWD_POLY16) / 16 == 1;
  return UA_FWD_POLY_MOD > 0 && (i % (UA_FWD_POLY_MOD > 0 ? UA_FWD_POLY_MOD : 1)) == 1;
}

template <int D>
struct FwdCfg {
  using G = TileGeom<D>;
  static constexpr int kStages = D == 128 ? 2 : 3;
  static constexpr int kThreads = 384;
  static constexpr int kSmemTiles = (2 + 2 * kStages) * G::kTileBytes;
  static constexpr int kSmemBytes = 1024 + kSmemTiles + 256;
  // D <= 64: P gets its own TMEM columns (S0 S1 | P0 P1 | O0 O1 = 512), so the
  // next S = Q K^T can be issued as soon as the softmax has LOADED S instead of
  // after P.V consumed P.  D = 128: P aliases S (S0 S1 | O0 O1 = 512).
  static constexpr bool kSeparateP = UA_FWD_SEP_P && D <= 64;
  static constexpr uint32_t kColS = 0;                          // + t*128
  static constexpr uint32_t kColP = kSeparateP ? 256 : 0;       // + t*(kSeparateP ? 64 : 128)
  static constexpr uint32_t kPStride = kSeparateP ? 64 : 128;
  static constexpr uint32_t kColO = kSeparateP ? 384 : 256;     // + t*D
  static constexpr float kRescaleThreshold = 8.0f;  // log2 units
  static constexpr bool kPolyExp = D <= UA_FWD_POLY_MAXD;  // FMA-pipe exp2 share for head dims up to this
};

template <int D>
__global__ void __launch_bounds__(384, 1) attn_fwd_kernel(const __grid_constant__ FwdParams p) {
  using C = FwdCfg<D>;
  using G = TileGeom<D>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-B aligned, stays in the shared window
  uint8_t* sQ = smem;                                  // [2] tiles
  uint8_t* sK = sQ + 2 * G::kTileBytes;                // [kStages]
  uint8_t* sV = sK + kStages * G::kTileBytes;          // [kStages]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * G::kTileBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + kStages;
  uint64_t* kv_empty = v_full + kStages;
  uint64_t* s_full = kv_empty + kStages;  // [2]
  uint64_t* p_full = s_full + 2;          // [2]
  uint64_t* o_done = p_full + 2;          // [2]
  uint64_t* s_free = o_done + 2;          // [2] softmax has loaded S_t (kSeparateP)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = blockIdx.x * 256;
  const int kv_t0 = p.kv_begin / 128;
  const int n_kv = (p.kv_end - p.kv_begin + 127) / 128;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
      mbar_init(&o_done[t], 1);
      mbar_init(&s_free[t], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

#if UA_FWD_MAXNREG > 0
  // Registers to the softmax warpgroups (the producer / MMA warpgroup needs few);
  // each role branch re-balances first thing so ptxas sees which limit applies.
  constexpr int kRegsLow = ((65536 / 384 / 8 * 8) * 384 - 256 * UA_FWD_MAXNREG) / 128 / 8 * 8;
#define UA_FWD_REGS_LOW() setmaxnreg_dec<kRegsLow>()
#define UA_FWD_REGS_HIGH() setmaxnreg_inc<UA_FWD_MAXNREG>()
#else
#define UA_FWD_REGS_LOW() ((void)0)
#define UA_FWD_REGS_HIGH() ((void)0)
#endif

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    UA_FWD_REGS_LOW();
    if (elect_one()) {
      tma_prefetch_desc(&p.tm_q);
      tma_prefetch_desc(&p.tm_k);
      tma_prefetch_desc(&p.tm_v);
      mbar_arrive_expect_tx(q_full, 2 * G::kTileBytes);
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < G::kAtoms; ++a)
          tma_load_4d(sQ + t * G::kTileBytes + a * G::kAtomBytes, &p.tm_q, q_full, a * G::kAtomCols,
                      q0 + t * 128, h, b, kEvictFirst);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % kStages;
        UA_TEV(0, j, 1);
        if (j >= kStages) mbar_wait(&kv_empty[s], ((j / kStages) & 1) ^ 1);
        UA_TEV(0, j, 2);
        const int row = (kv_t0 + j) * 128;
        mbar_arrive_expect_tx(&k_full[s], G::kTileBytes);
        for (int a = 0; a < G::kAtoms; ++a)
          tma_load_4d(sK + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_k, &k_full[s], a * G::kAtomCols, row, h,
                      b, kEvictLast);
        mbar_arrive_expect_tx(&v_full[s], G::kTileBytes);
        for (int a = 0; a < G::kAtoms; ++a)
          tma_load_4d(sV + s * G::kTileBytes + a * G::kAtomBytes, &p.tm_v, &v_full[s], a * G::kAtomCols, row, h,
                      b, kEvictLast);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    UA_FWD_REGS_LOW();
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
      const uint32_t idesc_o = idesc_bf16_f32(128, D, false, true);
      const uint32_t sQa = smem_u32(sQ), sKa = smem_u32(sK), sVa = smem_u32(sV);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T
        const uint32_t qt = sQa + t * G::kTileBytes, kt = sKa + (j % kStages) * G::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tbase + C::kColS + t * 128, kmajor_desc<D>(qt, kk), kmajor_desc<D>(kt, kk), idesc_s,
                 kk > 0 ? 1u : 0u);
        mma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t(j) V_j
        const uint32_t vt = sVa + (j % kStages) * G::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tbase + C::kColO + t * D, tbase + C::kColP + t * C::kPStride + kk * 8, mnmajor_desc<D>(vt, kk),
                 idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&o_done[t]);
      };
      if constexpr (C::kSeparateP) {
        // S_t(j+1) as soon as softmax t has loaded S_t(j); P.V when P is stored.
        mbar_wait(&k_full[0], 0);
        tc_fence_after();
        issue_s(0, 0);
        issue_s(1, 0);
        for (int j = 0; j < n_kv; ++j) {
          UA_TEV(1, j, 1);
          if (j + 1 < n_kv) {
            mbar_wait(&k_full[(j + 1) % kStages], ((j + 1) / kStages) & 1);
            UA_TEV(1, j, 2);
            for (int t = 0; t < 2; ++t) {
              mbar_wait(&s_free[t], j & 1);
              tc_fence_after();
              issue_s(t, j + 1);
              UA_TEV(1, j, 3 + t);
            }
          }
          mbar_wait(&v_full[j % kStages], (j / kStages) & 1);
          UA_TEV(1, j, 5);
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&p_full[t], j & 1);
            tc_fence_after();
            issue_pv(t, j);
            UA_TEV(1, j, 6 + t);
          }
          mma_commit(&kv_empty[j % kStages]);
        }
      } else
      for (int j = 0; j <= n_kv; ++j) {
        const int s = j % kStages;
        if (j < n_kv) {
          UA_TEV(1, j, 1);
          mbar_wait(&k_full[s], (j / kStages) & 1);
          UA_TEV(1, j, 2);
          tc_fence_after();
        }
        for (int t = 0; t < 2; ++t) {
          if (j > 0) {  // O_t += P_t(j-1) V_{j-1}
            const int sp = (j - 1) % kStages;
            UA_TEV(1, j, 10 + t);
            mbar_wait(&p_full[t], (j - 1) & 1);
            UA_TEV(1, j, 12 + t);
            if (t == 0) mbar_wait(&v_full[sp], ((j - 1) / kStages) & 1);
            tc_fence_after();
            const uint32_t vt = sVa + sp * G::kTileBytes;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ts(tbase + C::kColO + t * D, tbase + C::kColS + t * 128 + kk * 8, mnmajor_desc<D>(vt, kk),
                     idesc_o, (j > 1 || kk > 0) ? 1u : 0u);
            mma_commit(&o_done[t]);
          }
          if (j < n_kv) {  // S_t = Q_t K_j^T
            const uint32_t qt = sQa + t * G::kTileBytes, kt = sKa + s * G::kTileBytes;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              mma_ss(tbase + C::kColS + t * 128, kmajor_desc<D>(qt, kk), kmajor_desc<D>(kt, kk), idesc_s,
                     kk > 0 ? 1u : 0u);
            mma_commit(&s_full[t]);
            UA_TEV(1, j, 14 + t);
          }
        }
        if (j > 0) mma_commit(&kv_empty[(j - 1) % kStages]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    UA_FWD_REGS_HIGH();
    const int t = (warp - 4) / 4;
    const int quad = warp % 4;                 // TMEM lane quadrant of this warp
    const int row = quad * 32 + lane;          // row within the query tile
    const int q_row = q0 + t * 128 + row;      // global query index
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const uint32_t colS = C::kColS + t * 128, colO = C::kColO + t * D;
    const uint32_t colP = C::kColP + t * C::kPStride;
    const float c = p.scale_log2;
    float m_use = -INFINITY, l = 0.f;
    // Exp-phase ping-pong: warpgroup t runs its exp2 / P-store phase only after
    // the other warpgroup finished its own (named barriers 1 and 2, 256
    // threads), so the two tiles' exponentials do not share the MUFU unit and
    // one tile's GEMMs run under the other tile's exponentials.
    const uint32_t bar_mine = 1 + t, bar_other = 2 - t;
    if (UA_FWD_PINGPONG && t == 1) named_bar_arrive(1, 256);  // tile 0 goes first

    for (int j = 0; j < n_kv; ++j) {
      if (row == 0) UA_TEV(2 + t, j, 1);
      mbar_wait(&s_full[t], j & 1);
      if (row == 0) UA_TEV(2 + t, j, 2);
      tc_fence_after();
      const int kv0 = p.kv_begin + j * 128;
      const bool tail = kv0 + 128 > p.kv_end;
#if UA_FWD_RELOAD
      // Two passes over S in TMEM (row max, then exponentials) so only one or
      // two 32-column chunks are live in registers: the register file then has
      // room for many independent exp2 chains in flight.
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int cc = 0; cc < 128; cc += 32) {
        uint32_t r[32];
        tmem_ld32(t_lane + colS + cc, r);
        tmem_ld_wait();
        if (tail) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (kv0 + cc + i >= p.kv_end) r[i] = __float_as_uint(-INFINITY);
        }
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            mx[u] = fmax3(mx[u], __uint_as_float(r[i + 2 * u]), __uint_as_float(r[i + 2 * u + 1]));
        }
      }
#else
      float sv[128];
#if UA_FWD_LDBATCH
      {  // all four 32-column loads in flight, one wait
        uint32_t r[128];
#pragma unroll
        for (int cc = 0; cc < 128; cc += 32) tmem_ld32(t_lane + colS + cc, r + cc);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 128; ++i) sv[i] = __uint_as_float(r[i]);
      }
#else
#pragma unroll
      for (int cc = 0; cc < 128; cc += 32) {
        uint32_t r[32];
        tmem_ld32(t_lane + colS + cc, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[cc + i] = __uint_as_float(r[i]);
      }
#endif
      if constexpr (C::kSeparateP) {  // S_t is in registers: the next Q K^T may overwrite it
        tc_fence_before();
        mbar_arrive(&s_free[t]);
      }
      if (row == 0) UA_TEV(2 + t, j, 3);
      if (tail) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (kv0 + i >= p.kv_end) sv[i] = -INFINITY;
      }
      // row max: 3-input FMNMX, 4 independent chains
      float mx[4] = {sv[0], sv[1], sv[2], sv[3]};
#pragma unroll
      for (int i = 4; i < 128; i += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mx[u] = fmax3(mx[u], sv[i + 2 * u], sv[i + 2 * u + 1]);
      }
#endif
      const float rmax = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3]));
      const float m_new = fmaxf(m_use, rmax * c);
      if (row == 0) UA_TEV(2 + t, j, 4);
      const bool need = m_new > m_use + C::kRescaleThreshold;
      const bool warp_need = __any_sync(0xffffffffu, need);
      const float alpha = need ? ex2(m_use - m_new) : 1.f;
      if (need) {
        m_use = m_new;
        l *= alpha;
      }
      // p = 2^(s*c - m): packed fp32x2 FFMA for the argument, MUFU ex2 or the
      // FMA-pipe polynomial for the power, packed FADD for the row sum.
      const float2 c2 = make_float2(c, c), nm2 = make_float2(-m_use, -m_use);
      float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      constexpr bool kLateP = C::kSeparateP && UA_FWD_LATEP && !UA_FWD_RELOAD;
      if (C::kSeparateP && !kLateP && j > 0) {  // P_t buffer free: PV_t(j-1) has consumed it
        mbar_wait(&o_done[t], (j - 1) & 1);
        tc_fence_after();
      }
      if (UA_FWD_PINGPONG) named_bar_sync(bar_mine, 256);
      if (row == 0) UA_TEV(2 + t, j, 5);
#if UA_FWD_RELOAD
      // software-pipelined: chunk k+1 is loaded from TMEM while chunk k is exponentiated
      uint32_t ra[32], rb[32];
      tmem_ld32(t_lane + colS, ra);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t* cur = (k & 1) ? rb : ra;
        uint32_t* nxt = (k & 1) ? ra : rb;
        if (k < 3) tmem_ld32(t_lane + colS + 32 * (k + 1), nxt);
        if (tail) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (kv0 + 32 * k + i >= p.kv_end) cur[i] = __float_as_uint(-INFINITY);
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(cur[2 * i]), __uint_as_float(cur[2 * i + 1])), c2, nm2);
          const bool poly = C::kPolyExp && poly_pair(i);
          const float2 pp = poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          ls[i & 1] = __fadd2_rn(ls[i & 1], pp);
          pk[i] = pack_bf16x2(pp.x, pp.y);
        }
        tmem_st16(t_lane + colP + 16 * k, pk);
        if (k < 3) tmem_ld_wait();
      }
      if constexpr (C::kSeparateP) {  // S_t fully consumed: the next Q K^T may overwrite it
        tc_fence_before();
        mbar_arrive(&s_free[t]);
      }
#else
      if constexpr (kLateP) {
        // All 128 exponentials into registers (64 packed words) first, so the
        // wait for PV_t(j-1) to release the P buffer hides under them.
        uint32_t pk[64];
#pragma unroll
        for (int cc = 0; cc < 128; cc += 32) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = __ffma2_rn(make_float2(sv[cc + 2 * i], sv[cc + 2 * i + 1]), c2, nm2);
            const bool poly = C::kPolyExp && poly_pair(i);
            const float2 pp = poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
            ls[i & 1] = __fadd2_rn(ls[i & 1], pp);
            pk[cc / 2 + i] = pack_bf16x2(pp.x, pp.y);
          }
        }
        if (j > 0) {
          mbar_wait(&o_done[t], (j - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int cc = 0; cc < 64; cc += 16) tmem_st16(t_lane + colP + cc, pk + cc);
      } else {
#pragma unroll
      for (int cc = 0; cc < 128; cc += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = __ffma2_rn(make_float2(sv[cc + 2 * i], sv[cc + 2 * i + 1]), c2, nm2);
          // a third of the pairs on the FMA pipe when the exp unit co-binds (D <= 64)
          const bool poly = C::kPolyExp && poly_pair(i);
          const float2 pp = poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          ls[i & 1] = __fadd2_rn(ls[i & 1], pp);
          pk[i] = pack_bf16x2(pp.x, pp.y);
        }
        tmem_st16(t_lane + colP + cc / 2, pk);
      }
      }
#endif
      l += (ls[0].x + ls[0].y) + (ls[1].x + ls[1].y);
      if (UA_FWD_PINGPONG) named_bar_arrive(bar_other, 256);
      // Lazy rescale of O_t, after PV_t(j-1) has completed (o_done).
      if (warp_need && j > 0) {
        mbar_wait(&o_done[t], (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc + 32 <= D; cc += 32) {
          uint32_t r[32];
          tmem_ld32(t_lane + colO + cc, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st32(t_lane + colO + cc, r);
        }
        if constexpr (D % 32 != 0) {  // D = 80: the last 16 columns (never touch the next tile's O)
          uint32_t r[16];
          tmem_ld16(t_lane + colO + D - 16, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st16(t_lane + colO + D - 16, r);
        }
      }
      if (row == 0) UA_TEV(2 + t, j, 6);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[t]);
      if (row == 0) UA_TEV(2 + t, j, 7);
    }

    if (UA_FWD_PINGPONG && t == 0) named_bar_sync(1, 256);  // consume tile 1's last hand-back

    // ------------------------------------------------------------ epilogue
    mbar_wait(&o_done[t], (n_kv - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l;
    const bool valid = q_row < p.n_q;
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o.base) + b * p.o.sb + h * p.o.sh + int64_t(q_row) * p.o.sn;
    // I/O head dim: == D except the padded D = 80 tile of head dim 72 (columns >= d_io are not stored)
    const int d_io = D % 32 == 0 ? D : p.d_io;
    if (p.o_peer.base[0] != nullptr && valid) {  // fused return all-to-all: store into the token owner's buffer
      const int owner = int(q_row / p.o_peer.nl);
      orow = reinterpret_cast<__nv_bfloat16*>(p.o_peer.base[owner]) +
             ((b * p.o_peer.nl + (q_row - owner * p.o_peer.nl)) * p.o_peer.H + p.o_peer.h0 + h) * d_io;
    }
#pragma unroll
    for (int cc = 0; cc < D; cc += 32) {
      uint32_t r[32];
      tmem_ld32(t_lane + colO + cc, r);
      tmem_ld_wait();
      if (p.o_f32 != nullptr) {
        if (valid) {
          float* frow = p.o_f32 + b * p.of_sb + h * p.of_sh + int64_t(q_row) * p.of_sn + cc;
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            if (cc + i < d_io)
              *reinterpret_cast<float4*>(frow + i) =
                  make_float4(__uint_as_float(r[i]) * inv_l, __uint_as_float(r[i + 1]) * inv_l,
                              __uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
        }
      } else {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]) * inv_l, __uint_as_float(r[2 * i + 1]) * inv_l);
        if (valid) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            if (cc + 2 * i < d_io)
              *reinterpret_cast<uint4*>(orow + cc + 2 * i) = make_uint4(pk[i], pk[i + 1], pk[i + 2], pk[i + 3]);
        }
      }
    }
    if (valid) p.lse[b * p.l_sb + h * p.l_sh + q_row] = (m_use + __log2f(l)) * kLn2;
  } else {
    UA_FWD_REGS_LOW();  // warps 2, 3: idle members of the producer / MMA warpgroup
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tbase);
}

template <int D>
cudaError_t launch_fwd_impl(const FwdParams& p, int B, int Hx, cudaStream_t stream) {
  using C = FwdCfg<D>;
  cudaError_t e = set_max_smem(attn_fwd_kernel<D>, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid((p.n_q + 255) / 256, Hx, B);
#if UA_TRACE
  trace_reset();
#endif
  attn_fwd_kernel<D><<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
#if UA_TRACE
  trace_dump("fwd");
#endif
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_fwd(const FwdParams& p, int D, int B, int Hx, cudaStream_t stream) {
#if UA_FWD_SPLIT
  if (D <= 64) return launch_attn_fwd_split(p, D, B, Hx, stream);   // column-split softmax (attn_fwd_split.cu)
#endif
  switch (D) {
    case 32: return launch_fwd_impl<32>(p, B, Hx, stream);
    case 64: return launch_fwd_impl<64>(p, B, Hx, stream);
    case 72: return launch_fwd_impl<80>(p, B, Hx, stream);   // padded MMA head dim, p.d_io = 72
    case 128: return launch_fwd_impl<128>(p, B, Hx, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ua
