// Shared device-side definitions for the EBCC sm_100a path.
//
// Geometry, the spatial-orientation forest by formula (no N x 4 child table),
// MSB-first bitstream addressing and float64 helpers that round exactly like
// the reference's numpy expressions.  Everything float64 here is written with
// explicit __dadd_rn/__dmul_rn/__ddiv_rn so no FMA contraction can creep in
// (the library is also built with -fmad=false).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ebcc {

constexpr int kMaxLevels = 5;
constexpr int kHeader = 12;
constexpr int kZeroSentinel = -128;
constexpr int kMaxDecodePlanes = 64;
constexpr uint32_t kNone = 0xffffffffu;
constexpr int16_t kExpNone = -32768;  // exponent of 0: never significant

// CDF 9/7 lifting constants: the reference's double literals (dwt.py:23-30)
#define EBCC_ALPHA (-1.586134342059924)
#define EBCC_BETA (-0.052980118572961)
#define EBCC_GAMMA (0.882911075530934)
#define EBCC_DELTA (0.443506852043971)
#define EBCC_SCALE_LOW (1.1270436568907234)
#define EBCC_SCALE_HIGH (0.8773746085014191)

// Per-shape geometry, passed by value to kernels (dwt.py:82-92).
struct Geo {
  int rows, cols, levels;
  int64_t n;
  int lr[kMaxLevels + 1], lc[kMaxLevels + 1];  // ll_shapes[k]
};

__host__ __device__ inline int default_levels(int rows, int cols) {
  int m = rows < cols ? rows : cols;
  if (m < 2) return 1;
  int k = -1;
  while (m) { m >>= 1; k++; }
  int depth = k - 2;
  if (depth > kMaxLevels) depth = kMaxLevels;
  return depth < 1 ? 1 : depth;
}

__host__ __device__ inline int clamp_levels(int rows, int cols, int levels) {
  int m = rows < cols ? rows : cols;
  if (m < 2) m = 2;
  int k = -1;
  while (m) { m >>= 1; k++; }
  if (k < 1) k = 1;
  return levels < k ? levels : k;
}

inline Geo make_geo(int rows, int cols, int levels) {
  Geo g{};
  g.rows = rows; g.cols = cols; g.levels = levels;
  g.n = (int64_t)rows * cols;
  g.lr[0] = rows; g.lc[0] = cols;
  for (int k = 1; k <= levels; k++) {
    g.lr[k] = (g.lr[k - 1] + 1) / 2;
    g.lc[k] = (g.lc[k - 1] + 1) / 2;
  }
  for (int k = levels + 1; k <= kMaxLevels; k++) { g.lr[k] = g.lr[levels]; g.lc[k] = g.lc[levels]; }
  return g;
}

// Detail band rect (r0, c0, h, w) of orientation o (0 HL, 1 LH, 2 HH)
// created at `level` (dwt.py:68-79).
struct Rect { int r0, c0, h, w; };

__host__ __device__ inline Rect detail_rect(const Geo& g, int level, int o) {
  int ri = g.lr[level - 1], ci = g.lc[level - 1], rl = g.lr[level], cl = g.lc[level];
  if (o == 0) return {0, cl, rl, ci - cl};
  if (o == 1) return {rl, 0, ri - rl, cl};
  return {rl, cl, ri - rl, ci - cl};
}

// Children of a node in slot order, left-compacted (spiht.py:108-163).
// Returns the count and writes flat indices to ch[0..count).
__device__ __forceinline__ int tree_children(const Geo& g, int r, int c, uint32_t* ch) {
  const int L = g.levels;
  if (r < g.lr[L] && c < g.lc[L]) {
    // low-low root: same position in each coarsest detail band
    int m = 0;
#pragma unroll
    for (int o = 0; o < 3; o++) {
      Rect R = detail_rect(g, L, o);
      if (R.h > 0 && R.w > 0 && r < R.h && c < R.w)
        ch[m++] = (uint32_t)((R.r0 + r) * g.cols + (R.c0 + c));
    }
    return m;
  }
  // detail node: find its level k (largest k with the node inside box k-1)
  int k = 1;
  for (int kk = L; kk >= 1; kk--) {
    if (r < g.lr[kk - 1] && c < g.lc[kk - 1]) { k = kk; break; }
  }
  if (k < 2) return 0;
  int o = (r < g.lr[k]) ? 0 : ((c < g.lc[k]) ? 1 : 2);
  Rect P = detail_rect(g, k, o);
  Rect C = detail_rect(g, k - 1, o);
  int i = r - P.r0, j = c - P.c0;
  int m = 0;
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      int ci = 2 * i + a, cj = 2 * j + b;
      if (ci < C.h && cj < C.w) ch[m++] = (uint32_t)((C.r0 + ci) * g.cols + (C.c0 + cj));
    }
  return m;
}

// ---- MSB-first bitstream addressing over 32-bit words ----------------------
// Stream bit p lives in byte p>>3 at bit (7 - (p&7)).  In a little-endian u32
// word w (bytes 4w..4w+3) that is bit ((p>>3)&3)*8 + 7 - (p&7).
__host__ __device__ __forceinline__ uint32_t bit_mask_in_word(uint64_t p) {
  return 1u << ((((uint32_t)(p >> 3)) & 3u) * 8u + 7u - ((uint32_t)p & 7u));
}

__device__ __forceinline__ int read_bit(const uint32_t* words, uint64_t p, uint64_t limit) {
  if (p >= limit) return 0;
  return (__ldg(words + (p >> 5)) & bit_mask_in_word(p)) != 0;
}

// floor(log2(x)) for x > 0 finite (exact, subnormals included); kExpNone for 0
__device__ __forceinline__ int16_t exp_of(double x) {
  if (x == 0.0) return kExpNone;
  return (int16_t)ilogb(x);
}

// Top 32 bits of the 53-bit significand of |x| (hidden bit at bit 31).
__device__ __forceinline__ uint32_t mant32_of(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(fabs(x));
  uint64_t e = b >> 52;
  uint64_t m = b & ((1ull << 52) - 1);
  if (e) {
    m |= 1ull << 52;
  } else if (m) {
    while (!(m & (1ull << 52))) m <<= 1;
  }
  return (uint32_t)(m >> 21);
}

}  // namespace ebcc
