// Fused forward-DWT level kernel (dwt.py:136-155, 194-198): one launch does
// the row pass and the column pass of one level for every field of a batch.
//
// It mirrors the inverse level kernel (idwt_fused.cuh).  A CTA (256 threads)
// owns TW = 224 region columns x `th` region rows:
//
//  phase A (rows): one warp per (row, column group) holds 32 (s, d) pairs of
//     the row -- x[2j], x[2j+1] for j = j0-2 .. j0+29 -- and runs the four
//     lifting steps with warp shuffles (28 pairs come out valid), scales and
//     drops the row into an 8-row shared-memory chunk, s columns then d
//     columns per group ("patch columns");
//  phase B (columns): every thread streams down one patch column, carrying
//     the four lifting steps as a software pipeline in registers (loading row
//     pair m yields the finished pair m - 2), scales and stores s rows to the
//     upper and d rows to the lower half of the region.
//
// Borders: the reference clamps neighbour indices, which is whole-sample
// symmetric extension of the signal; every lifting step preserves that
// symmetry bit for bit (IEEE addition commutes), so out-of-range samples are
// loaded from their mirrored positions and the stencils run without branches
// (an odd-length line's missing last d sample becomes a mirrored "virtual"
// one that is computed but never stored).  All arithmetic is explicit
// __dadd_rn/__dmul_rn in numpy's evaluation order.
//
// The two separable passes it replaces ran at 3.4 IPC on index arithmetic
// (about 220 warp instructions per 32 points each); this kernel is bound by
// its 16 B/pt of HBM traffic.
#pragma once
#include "common.cuh"

namespace ebcc {
namespace fdwt {

constexpr int GROUPS = 4;
constexpr int GW = 56;               // region columns per group
constexpr int PC = 64;               // patch columns per group (32 s + 32 d)
constexpr int THREADS = GROUPS * PC;
constexpr int TW = GROUPS * GW;      // 224 region columns per CTA
constexpr int CH = 8;                // rows per shared-memory chunk
constexpr int KB = CH / 2;
constexpr int TH = 192;              // region rows per CTA (multiple of CH)

__device__ __forceinline__ int fold(int t, int n) {
  if (t >= 0 && t < n) return t;
  if (n == 1) return 0;
  int P = 2 * (n - 1);
  t %= P;
  if (t < 0) t += P;
  return t >= n ? P - t : t;
}

// region R x C (R, C > 1) of `in` (row stride cols, fields fstride apart) ->
// the same region of `out` in the [s | d] x [s | d] layout
#ifndef EBCC_FDWT_MINB
#define EBCC_FDWT_MINB 5  // 46 registers: 5 CTAs/SM hide the load -> shuffle -> barrier chain (148 fields: -0.6 ms vs 3)
#endif
__global__ void __launch_bounds__(THREADS, EBCC_FDWT_MINB)
    level_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t fstride, int cols,
                 int R, int C, int th) {
  extern __shared__ double dyn[];
  double (*rowbuf)[CH][THREADS + 1] = reinterpret_cast<double (*)[CH][THREADS + 1]>(dyn);
  const int f = blockIdx.z;
  const double* __restrict__ src = in + (int64_t)f * fstride;
  double* __restrict__ dst = out + (int64_t)f * fstride;
  const int nsR = (R + 1) / 2, ndR = R / 2, nsC = (C + 1) / 2, ndC = C / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Y0 = blockIdx.y * th;
  const int ylen = min(th, R - Y0);
  const int i0 = Y0 / 2;  // first row pair of the tile (Y0 is even)
  const int npairs = (ylen + 1) / 2;
  const int nchunks = (npairs + KB - 1) / KB;

  // phase A: warp w owns column group w % 4 and rows w / 4, w / 4 + 2, ...
  const int pg = warp % GROUPS, rsub = warp / GROUPS;
  const int gX0 = blockIdx.x * TW + pg * GW;
  const int ja = gX0 / 2 - 2 + lane;  // my pair of the row
  const int ca = fold(2 * ja, C), cb = fold(2 * ja + 1, C);
  // interior lanes: both samples in range and adjacent
  const int gbase = pg * PC;

  // phase B: my patch column
  const int grp = tid / PC, pcol = tid % PC, pl = pcol & 31;
  const bool is_d = pcol >= 32;
  const int jj = (blockIdx.x * TW + grp * GW) / 2 - 2 + pl;  // subband column index
  const bool col_ok = pl >= 2 && pl < 30 && jj >= 0 && jj < (is_d ? ndC : nsC);
  const int ocol = is_d ? nsC + jj : jj;
  double s0p = 0, d0p = 0, d1p = 0, s1p = 0, d2p = 0;

  int buf = 0;
  // load j: row pairs i0 - 2 + 4j .. i0 + 1 + 4j; its column steps finish
  // pairs i0 - 4 + 4j .. i0 - 1 + 4j (load 0 only warms the pipeline up)
  for (int j = 0; j <= nchunks; j++, buf ^= 1) {
    const int y0 = 2 * (i0 - 2 + KB * j);  // first region row of the load (may be out of range)
    // ---- phase A ----------------------------------------------------------
#pragma unroll
    for (int t = 0; t < CH / 2; t++) {
      const int r = rsub + 2 * t;
      const int y = fold(y0 + r, R);
      const double* row = src + (int64_t)y * cols;
      double s = row[ca], d = row[cb];
      // dwt.py:146-152
      double sn = __shfl_down_sync(0xffffffffu, s, 1);
      d = __dadd_rn(d, __dmul_rn(EBCC_ALPHA, __dadd_rn(s, sn)));
      double dp = __shfl_up_sync(0xffffffffu, d, 1);
      s = __dadd_rn(s, __dmul_rn(EBCC_BETA, __dadd_rn(dp, d)));
      sn = __shfl_down_sync(0xffffffffu, s, 1);
      d = __dadd_rn(d, __dmul_rn(EBCC_GAMMA, __dadd_rn(s, sn)));
      dp = __shfl_up_sync(0xffffffffu, d, 1);
      s = __dadd_rn(s, __dmul_rn(EBCC_DELTA, __dadd_rn(dp, d)));
      rowbuf[buf][r][gbase + lane] = __dmul_rn(s, EBCC_SCALE_LOW);
      rowbuf[buf][r][gbase + 32 + lane] = __dmul_rn(d, EBCC_SCALE_HIGH);
    }
    __syncthreads();
    // ---- phase B ----------------------------------------------------------
#pragma unroll
    for (int u = 0; u < KB; u++) {
      const double s0 = rowbuf[buf][2 * u][tid], d0 = rowbuf[buf][2 * u + 1][tid];
      // pair m = i0 - 2 + 4j + u arrives: finish pair m - 2
      const double d1 = __dadd_rn(d0p, __dmul_rn(EBCC_ALPHA, __dadd_rn(s0p, s0)));
      const double s1 = __dadd_rn(s0p, __dmul_rn(EBCC_BETA, __dadd_rn(d1p, d1)));
      const double d2 = __dadd_rn(d1p, __dmul_rn(EBCC_GAMMA, __dadd_rn(s1p, s1)));
      const double s2 = __dadd_rn(s1p, __dmul_rn(EBCC_DELTA, __dadd_rn(d2p, d2)));
      s0p = s0; d0p = d0; d1p = d1; s1p = s1; d2p = d2;
      const int k = i0 - 4 + KB * j + u;  // finished pair
      if (j > 0 && col_ok && k < i0 + npairs) {
        if (k < nsR) dst[(int64_t)k * cols + ocol] = __dmul_rn(s2, EBCC_SCALE_LOW);
        if (k < ndR) dst[(int64_t)(nsR + k) * cols + ocol] = __dmul_rn(d2, EBCC_SCALE_HIGH);
      }
    }
    // no trailing barrier: the next load writes the other buffer, and the
    // barrier after its phase A orders this phase B before that buffer's reuse
  }
}

// detail quadrants (and the LL quadrant too if `with_ll`) of region R x C
__global__ void copy_bands_kernel(const double* __restrict__ in, double* __restrict__ out,
                                  int64_t fstride, int cols, int R, int C, int with_ll) {
  const int f = blockIdx.z;
  const int nsR = (R + 1) / 2, nsC = (C + 1) / 2;
  const int y = blockIdx.y;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < C; x += gridDim.x * blockDim.x) {
    if (!with_ll && y < nsR && x < nsC) continue;
    const int64_t o = (int64_t)f * fstride + (int64_t)y * cols + x;
    out[o] = in[o];
  }
}

inline void launch_level(const double* in, double* out, int64_t fstride, int nfields, int cols,
                         int R, int C, cudaStream_t st) {
  static bool attr = false;
  constexpr size_t smem = sizeof(double) * 2 * CH * (THREADS + 1);
  if (!attr) {
    cudaFuncSetAttribute(level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  // shorter tiles on small levels so the grid still fills the machine
  int th = TH;
  const int64_t ct = (C + TW - 1) / TW;
  while (th > CH && ct * ((R + th - 1) / th) * nfields < 4 * 148) th /= 2;
  dim3 grid((unsigned)ct, (unsigned)((R + th - 1) / th), (unsigned)nfields);
  level_kernel<<<grid, THREADS, smem, st>>>(in, out, fstride, cols, R, C, th);
}

inline void copy_bands(const double* in, double* out, int64_t fstride, int nfields, int cols, int R,
                       int C, bool with_ll, cudaStream_t st) {
  dim3 grid((unsigned)((C + 255) / 256), (unsigned)R, (unsigned)nfields);
  copy_bands_kernel<<<grid, 256, 0, st>>>(in, out, fstride, cols, R, C, with_ll ? 1 : 0);
}

}  // namespace fdwt
}  // namespace ebcc
