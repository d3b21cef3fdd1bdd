// attn_fwd_split.cu — exact attention forward for D <= 64 with a column-split
// softmax (sm_100a).  Same result as attn_fwd.cu (§2.5,
// P:173-175 §2.6: per-head softmax(Q K^T / sqrt(D)) V over the key range
// [kv_begin, kv_end), online softmax, lse), different work split:
//
//  * At D <= 64 the softmax, not the tensor core, bounds the forward: per
//    128 x 128 score tile the tensor core needs 256 clocks (D = 64) but the
//    exponentials alone need 1024 MUFU slots.  attn_fwd.cu gives each query
//    tile one warpgroup (thread = row, 128 scores per thread), i.e. only two
//    softmax warps per SM sub-partition to hide the exp / FMA latency chains.
//  * Here each query tile has TWO warpgroups, one per 64-column half of the
//    score tile (warps w and w+4 share TMEM lanes 32 (w % 4)..+31).  Each
//    thread holds 64 scores; the halves exchange their partial row maxima
//    through shared memory (one named barrier per tile and key step), keep
//    partial row sums (combined once, at the end) and write their halves of
//    P.  Four softmax warps per sub-partition, same instruction count.
//  * 20 warps: 0 TMA producer, 1 tcgen05.mma issuer + TMEM owner, 2-3 idle
//    (register donors), 4-19 softmax: tile t = (w-4)/8, column half (w-4)/4 % 2.
//  * TMEM: S0 S1 [0,256) | P0 P1 [256,384) (bf16 pairs) | O0 O1 [384, 384+2D).
//    S_t(j+1) is issued as soon as both halves have loaded S_t(j); P.V when
//    both halves stored P_t(j).  Lazy max (rescale of O and l only when a row
//    max grows by more than 2^8), exact in the end (O and l share the max).
#include "attn_common.cuh"
#include "attn_kernels.h"

#ifndef UA_FWD_SPLIT_POLY16
#define UA_FWD_SPLIT_POLY16 4   // exp2 pairs of every 16 on the FMA-pipe polynomial
#endif
#ifndef UA_FWD_SPLIT_STAGES
#define UA_FWD_SPLIT_STAGES 4   // K / V ring depth (A/B at c4: 4 > 3 by 0.8 %, 2 -7 %)
#endif
#ifndef UA_FWD_SPLIT_REGS
#define UA_FWD_SPLIT_REGS 104   // setmaxnreg of the softmax warpgroups (0: off)
#endif

namespace ua {

namespace {

__device__ __forceinline__ constexpr bool split_poly_pair(int i) {
  return UA_FWD_SPLIT_POLY16 > 0 && ((i + 1) * UA_FWD_SPLIT_POLY16) / 16 - (i * UA_FWD_SPLIT_POLY16) / 16 == 1;
}

template <int D>
struct SplitCfg {
  using G = TileGeom<D>;
  static constexpr int kStages = UA_FWD_SPLIT_STAGES;
  static constexpr int kThreads = 640;
  static constexpr int kXchgBytes = 2 * 2 * 2 * 128 * 4;   // [tile][parity][half][row] partial maxima / sums
  static constexpr int kSmemBytes = 1024 + (2 + 2 * kStages) * G::kTileBytes + kXchgBytes + 256;
  static constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;  // + t*128, t*64, t*D
  static constexpr float kRescaleThreshold = 8.0f;  // log2 units
  static_assert(D <= 64, "column-split forward is for D <= 64 (TMEM: S, P, O of two tiles)");
};

template <int D>
__global__ void __launch_bounds__(640, 1) attn_fwd_split_kernel(const __grid_constant__ FwdParams p) {
  using C = SplitCfg<D>;
  using G = TileGeom<D>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                                  // [2] tiles
  uint8_t* sK = sQ + 2 * G::kTileBytes;                // [kStages]
  uint8_t* sV = sK + kStages * G::kTileBytes;          // [kStages]
  float* sX = reinterpret_cast<float*>(sV + kStages * G::kTileBytes);  // [2 t][2 parity][2 half][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sX) + C::kXchgBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + kStages;
  uint64_t* kv_empty = v_full + kStages;
  uint64_t* s_full = kv_empty + kStages;  // [2] S_t computed
  uint64_t* s_free = s_full + 2;          // [2] both halves have S_t in registers
  uint64_t* p_full = s_free + 2;          // [2] both halves stored P_t (and O_t is rescaled)
  uint64_t* o_done = p_full + 2;          // [2] P_t V done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

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
      mbar_init(&s_free[t], 256);
      mbar_init(&p_full[t], 256);
      mbar_init(&o_done[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

#if UA_FWD_SPLIT_REGS > 0
  constexpr int kRegsLow = 40;  // producer / MMA / idle warpgroup
  static_assert(128 * kRegsLow + 512 * UA_FWD_SPLIT_REGS <= (65536 / 640 / 8 * 8) * 640, "register pool");
#define UA_SPLIT_REGS_LOW() setmaxnreg_dec<kRegsLow>()
#define UA_SPLIT_REGS_HIGH() setmaxnreg_inc<UA_FWD_SPLIT_REGS>()
#else
#define UA_SPLIT_REGS_LOW() ((void)0)
#define UA_SPLIT_REGS_HIGH() ((void)0)
#endif

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    UA_SPLIT_REGS_LOW();
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
        if (j >= kStages) mbar_wait(&kv_empty[s], ((j / kStages) & 1) ^ 1);
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
    UA_SPLIT_REGS_LOW();
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
          mma_ts(tbase + C::kColO + t * D, tbase + C::kColP + t * 64 + kk * 8, mnmajor_desc<D>(vt, kk), idesc_o,
                 (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&o_done[t]);
      };
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {  // next S as soon as both halves hold this S in registers
          mbar_wait(&k_full[(j + 1) % kStages], ((j + 1) / kStages) & 1);
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&s_free[t], j & 1);
            tc_fence_after();
            issue_s(t, j + 1);
          }
        }
        mbar_wait(&v_full[j % kStages], (j / kStages) & 1);
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&p_full[t], j & 1);
          tc_fence_after();
          issue_pv(t, j);
        }
        mma_commit(&kv_empty[j % kStages]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax (tile t, column half hf)
    UA_SPLIT_REGS_HIGH();
    const int sw = warp - 4;
    const int t = sw / 8, hf = (sw / 4) % 2;
    const int quad = warp % 4;                 // TMEM lane quadrant
    const int row = quad * 32 + lane;          // row within the query tile
    const int q_row = q0 + t * 128 + row;
    const uint32_t t_lane = tbase + (uint32_t(quad * 32) << 16);
    const uint32_t colS = C::kColS + t * 128 + 64 * hf;
    const uint32_t colP = C::kColP + t * 64 + 32 * hf;
    const uint32_t colO = C::kColO + t * D;
    const uint32_t bar = 1 + t;                // named barrier of the tile's 256 softmax threads
    float* xbase = sX + t * (2 * 2 * 128);
    const float c = p.scale_log2;
    const float2 c2 = make_float2(c, c);
    float m_use = -INFINITY, l = 0.f;

    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      float sv[64];
      {
        uint32_t r[64];
        tmem_ld32(t_lane + colS, r);
        tmem_ld32(t_lane + colS + 32, r + 32);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 64; ++i) sv[i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      mbar_arrive(&s_free[t]);   // S_t(j) is in registers: S_t(j+1) may overwrite it
      const int kc0 = p.kv_begin + j * 128 + 64 * hf;
      if (kc0 + 64 > p.kv_end) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (kc0 + i >= p.kv_end) sv[i] = -INFINITY;
      }
      // partial row max over this half, exchanged with the other half
      float mx[4] = {sv[0], sv[1], sv[2], sv[3]};
#pragma unroll
      for (int i = 4; i < 64; i += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mx[u] = fmax3(mx[u], sv[i + 2 * u], sv[i + 2 * u + 1]);
      }
      const float pmax = fmax3(mx[0], mx[1], fmaxf(mx[2], mx[3]));
      float* xj = xbase + (j & 1) * (2 * 128);
      xj[hf * 128 + row] = pmax;
      named_bar_sync(bar, 256);
      const float rmax = fmaxf(pmax, xj[(1 - hf) * 128 + row]);
      const float m_new = fmaxf(m_use, rmax * c);
      const bool need = m_new > m_use + C::kRescaleThreshold;   // identical in both halves
      const bool warp_need = __any_sync(0xffffffffu, need);
      const float alpha = need ? ex2(m_use - m_new) : 1.f;
      if (need) {
        m_use = m_new;
        l *= alpha;
      }
      // p = 2^(s*c - m): FFMA2 for the argument, MUFU ex2 or the FMA-pipe polynomial, FADD2 row sum
      const float2 nm2 = make_float2(-m_use, -m_use);
      float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      uint32_t pk[32];
#pragma unroll
      for (int cc = 0; cc < 64; cc += 32) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = __ffma2_rn(make_float2(sv[cc + 2 * i], sv[cc + 2 * i + 1]), c2, nm2);
          const float2 pp = split_poly_pair(i) ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          ls[i & 1] = __fadd2_rn(ls[i & 1], pp);
          pk[cc / 2 + i] = pack_bf16x2(pp.x, pp.y);
        }
      }
      l += (ls[0].x + ls[0].y) + (ls[1].x + ls[1].y);
      if (j > 0) {  // P_t buffer free (P_t(j-1) V done), and O_t final for the rescale
        mbar_wait(&o_done[t], (j - 1) & 1);
        tc_fence_after();
      }
      tmem_st16(t_lane + colP, pk);
      tmem_st16(t_lane + colP + 16, pk + 16);
      if (hf == 0 && warp_need && j > 0) {  // lazy rescale of O_t (one half owns O)
#pragma unroll
        for (int cc = 0; cc < D; cc += 16) {
          uint32_t r[16];
          tmem_ld16(t_lane + colO + cc, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st16(t_lane + colO + cc, r);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[t]);
    }

    // ------------------------------------------------------------ epilogue
    // total row sum = both halves' partial sums (same max)
    float* xl = xbase + (n_kv & 1) * (2 * 128);   // parity n_kv: not read by any pending iteration
    xl[hf * 128 + row] = l;
    named_bar_sync(bar, 256);
    const float l_tot = l + xl[(1 - hf) * 128 + row];
    mbar_wait(&o_done[t], (n_kv - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l_tot;
    const bool valid = q_row < p.n_q;
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.o.base) + b * p.o.sb + h * p.o.sh + int64_t(q_row) * p.o.sn;
    if (p.o_peer.base[0] != nullptr && valid) {  // fused return all-to-all: the token owner's buffer
      const int owner = int(q_row / p.o_peer.nl);
      orow = reinterpret_cast<__nv_bfloat16*>(p.o_peer.base[owner]) +
             ((b * p.o_peer.nl + (q_row - owner * p.o_peer.nl)) * p.o_peer.H + p.o_peer.h0 + h) * D;
    }
    // each half stores D/2 columns of O
#pragma unroll
    for (int cc = hf * (D / 2); cc < (hf + 1) * (D / 2); cc += 16) {
      uint32_t r[16];
      tmem_ld16(t_lane + colO + cc, r);
      tmem_ld_wait();
      if (p.o_f32 != nullptr) {
        if (valid) {
          float* frow = p.o_f32 + b * p.of_sb + h * p.of_sh + int64_t(q_row) * p.of_sn + cc;
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(frow + i) =
                make_float4(__uint_as_float(r[i]) * inv_l, __uint_as_float(r[i + 1]) * inv_l,
                            __uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
        }
      } else {
        uint32_t pko[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          pko[i] = pack_bf16x2(__uint_as_float(r[2 * i]) * inv_l, __uint_as_float(r[2 * i + 1]) * inv_l);
        if (valid) {
          *reinterpret_cast<uint4*>(orow + cc) = make_uint4(pko[0], pko[1], pko[2], pko[3]);
          *reinterpret_cast<uint4*>(orow + cc + 8) = make_uint4(pko[4], pko[5], pko[6], pko[7]);
        }
      }
    }
    if (valid && hf == 0) p.lse[b * p.l_sb + h * p.l_sh + q_row] = (m_use + __log2f(l_tot)) * kLn2;
  } else {
    UA_SPLIT_REGS_LOW();  // warps 2, 3: idle members of the producer / MMA warpgroup
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tbase);
}

template <int D>
cudaError_t launch_split_impl(const FwdParams& p, int B, int Hx, cudaStream_t stream) {
  using C = SplitCfg<D>;
  cudaError_t e = set_max_smem(attn_fwd_split_kernel<D>, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid((p.n_q + 255) / 256, Hx, B);
  attn_fwd_split_kernel<D><<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_fwd_split(const FwdParams& p, int D, int B, int Hx, cudaStream_t stream) {
  switch (D) {
    case 32: return launch_split_impl<32>(p, B, Hx, stream);
    case 64: return launch_split_impl<64>(p, B, Hx, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ua
