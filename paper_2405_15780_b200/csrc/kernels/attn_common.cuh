// attn_common.cuh — shared definitions for the sm_100a attention kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "sm100_ptx.cuh"

namespace ua {

// Per-head-dim smem tile geometry.  A [128 rows][D] bf16 tile is stored as
// kAtoms column blocks ("atoms") of [128][kAtomCols], each row kSw bytes,
// swizzled by TMA: SWIZZLE_128B when 64 | D (64, 128), SWIZZLE_64B for D = 32,
// SWIZZLE_32B for D = 80 (the padded tile of head dim 72: five 16-column
// atoms, columns 72..79 zero-filled by TMA).  D here is the MMA head dim; the
// I/O head dim (72 for the padded case) travels in the kernel params.
template <int D>
struct TileGeom {
  static constexpr int kSw = D % 64 == 0 ? 128 : (D % 32 == 0 ? 64 : 32);  // swizzle span (bytes per atom row)
  static constexpr int kAtomCols = kSw / 2;                 // bf16 per atom row
  static constexpr int kAtoms = D / kAtomCols;              // atoms along D
  static constexpr int kAtomBytes = 128 * kSw;              // one atom of 128 rows
  static constexpr int kTileBytes = 128 * D * 2;            // whole [128][D] tile
  static constexpr uint32_t kLayout = kSw == 128 ? 2u : (kSw == 64 ? 4u : 6u);  // SWIZZLE_128B / 64B / 32B
  static constexpr uint32_t kSBO = 8 * kSw;                 // 8-row group stride
  static_assert(D % 16 == 0 && kAtoms * kAtomCols == D, "head dim");
};

// MMA head dim of an I/O head dim (72 -> 80: K and N must be multiples of 16).
constexpr int mma_dim(int d) { return (d + 15) / 16 * 16; }

// Generic smem descriptor (version 1, base offset 0).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (uint64_t(layout) << 61);
}

// Descriptor of the kk-th 16-wide K slice of a K-major [rows][D] tile.
template <int D>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t tile, int kk) {
  using G = TileGeom<D>;
  uint32_t off = ((kk * 16) / G::kAtomCols) * G::kAtomBytes + ((kk * 32) % G::kSw);
  return sdesc(tile + off, 16, G::kSBO, G::kLayout);
}

// Descriptor of rows [16 kk, 16 kk + 16) of a [128 rows][D] tile used as an
// MN-major operand (rows = K dimension of the MMA, D = its N or M dimension).
template <int D>
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t tile, int kk) {
  using G = TileGeom<D>;
  return sdesc(tile + kk * 16 * G::kSw, G::kAtomBytes, G::kSBO, G::kLayout);
}

// Same two descriptors for a tile of ROWS rows (atoms of ROWS x kSw bytes).
template <int D, int ROWS>
__device__ __forceinline__ uint64_t kmajor_desc_r(uint32_t tile, int kk) {
  using G = TileGeom<D>;
  uint32_t off = ((kk * 16) / G::kAtomCols) * (ROWS * G::kSw) + ((kk * 32) % G::kSw);
  return sdesc(tile + off, 16, G::kSBO, G::kLayout);
}
template <int D, int ROWS>
__device__ __forceinline__ uint64_t mnmajor_desc_r(uint32_t tile, int kk) {
  using G = TileGeom<D>;
  return sdesc(tile + kk * 16 * G::kSw, ROWS * G::kSw, G::kSBO, G::kLayout);
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

}  // namespace ua
