// The CDF 9/7 lifting pass kernel (header so every TU can instantiate it
// with its own epilogue).  See dwt.cu for the design notes.
#pragma once
#include "dwt.cuh"

namespace ebcc {
namespace lift {


constexpr int HALO = 2;
#ifndef EBCC_ROW_TI
#define EBCC_ROW_TI 256
#endif
#ifndef EBCC_ROW_LINES
#define EBCC_ROW_LINES 4
#endif

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// One lifting step over the staged window.  X is updated from its own value
// and the neighbours of Y:  x[i] = x[i] (+|-) K*(y[a] + y[b]).
// For an s-step (updating s from d):  a = max(i-1,0), b = min(i, nd-1).
// For a d-step (updating d from s):   a = i,          b = min(i+1, ns-1).
template <bool SUB, bool UPDATE_S, int LINES, int SPAN>
__device__ __forceinline__ void lift_step(double (*x)[SPAN + 1], double (*y)[SPAN + 1], int lo, int xcount,
                                          int ycount, int ns, int nd, double K) {
  const int ylo = lo, yhi = lo + ycount - 1;
  for (int e = threadIdx.x; e < LINES * xcount; e += blockDim.x) {
    int line = e / xcount, k = e - line * xcount;
    int i = lo + k;  // global subband index
    int a, b;
    if (UPDATE_S) {
      a = i > 0 ? i - 1 : 0;
      b = i < nd ? i : nd - 1;
    } else {
      a = i;
      b = i + 1 < ns ? i + 1 : ns - 1;
    }
    a = clampi(a, ylo, yhi) - lo;
    b = clampi(b, ylo, yhi) - lo;
    double sum = __dadd_rn(y[line][a], y[line][b]);
    double t = __dmul_rn(K, sum);
    x[line][k] = SUB ? __dsub_rn(x[line][k], t) : __dadd_rn(x[line][k], t);
  }
}

// Generic pass.  Element (line L, position p) of the region lives at
// base + L*line_stride + p*elem_stride.  n = line length along the transform.
template <bool INVERSE, int LINES, int TI, class Epi>
__global__ void __launch_bounds__(256) lift_pass_kernel(const double* __restrict__ in,
                                                        double* __restrict__ out,
                                                        int64_t field_stride, int line_stride,
                                                        int elem_stride, int nlines, int n,
                                                        Epi epi_in) {
  constexpr int SPAN = TI + 2 * HALO;
  Epi epi = epi_in;  // per-thread copy: epilogues may accumulate
  __shared__ double s_sh[LINES][SPAN + 1];  // +1: odd row pitch, fewer bank conflicts
  __shared__ double d_sh[LINES][SPAN + 1];
  const int64_t fbase = (int64_t)blockIdx.z * field_stride;
  const int line0 = blockIdx.x * LINES;
  const int i0 = blockIdx.y * TI;
  const int ns = (n + 1) / 2, nd = n / 2;
  const double* src = in + fbase;
  double* dst = out + fbase;

  if (!epi.begin(blockIdx.z)) return;
  if (n == 1) {  // length-1 passthrough (dwt.py:140-141, 160-161)
    if (blockIdx.y == 0)
      for (int l = threadIdx.x; l < LINES; l += blockDim.x) {
        int line = line0 + l;
        if (line < nlines) {
          int64_t off = (int64_t)line * line_stride;
          epi.store(dst, blockIdx.z, off, src[off]);
        }
      }
    epi.finish(blockIdx.z);
    return;
  }
  if (i0 >= ns) { epi.finish(blockIdx.z); return; }
  // staged window [lo, hi] of subband indices (same window for s and d)
  const int lo = i0 - HALO > 0 ? i0 - HALO : 0;
  const int shi = (i0 + TI + HALO - 1) < ns - 1 ? (i0 + TI + HALO - 1) : ns - 1;
  const int dhi = (i0 + TI + HALO - 1) < nd - 1 ? (i0 + TI + HALO - 1) : nd - 1;
  const int scount = shi - lo + 1;
  const int dcount = dhi >= lo ? dhi - lo + 1 : 0;

  // load.  Map consecutive threads along whichever axis is contiguous.
  const bool lines_contig = (line_stride == 1);
  for (int e = threadIdx.x; e < LINES * SPAN; e += blockDim.x) {
    int l, k;
    if (lines_contig) { l = e % LINES; k = e / LINES; }
    else { k = e % SPAN; l = e / SPAN; }
    int line = line0 + l;
    if (line >= nlines) continue;
    int64_t lbase = (int64_t)line * line_stride;
    int i = lo + k;
    if (k < scount) {
      int p = INVERSE ? i : 2 * i;
      double v = src[lbase + (int64_t)p * elem_stride];
      s_sh[l][k] = INVERSE ? __ddiv_rn(v, EBCC_SCALE_LOW) : v;
    }
    if (k < dcount) {
      int p = INVERSE ? ns + i : 2 * i + 1;
      double v = src[lbase + (int64_t)p * elem_stride];
      d_sh[l][k] = INVERSE ? __ddiv_rn(v, EBCC_SCALE_HIGH) : v;
    }
  }
  __syncthreads();
  if (INVERSE) {
    lift_step<true, true, LINES, SPAN>(s_sh, d_sh, lo, scount, dcount, ns, nd, EBCC_DELTA);
    __syncthreads();
    lift_step<true, false, LINES, SPAN>(d_sh, s_sh, lo, dcount, scount, ns, nd, EBCC_GAMMA);
    __syncthreads();
    lift_step<true, true, LINES, SPAN>(s_sh, d_sh, lo, scount, dcount, ns, nd, EBCC_BETA);
    __syncthreads();
    lift_step<true, false, LINES, SPAN>(d_sh, s_sh, lo, dcount, scount, ns, nd, EBCC_ALPHA);
  } else {
    lift_step<false, false, LINES, SPAN>(d_sh, s_sh, lo, dcount, scount, ns, nd, EBCC_ALPHA);
    __syncthreads();
    lift_step<false, true, LINES, SPAN>(s_sh, d_sh, lo, scount, dcount, ns, nd, EBCC_BETA);
    __syncthreads();
    lift_step<false, false, LINES, SPAN>(d_sh, s_sh, lo, dcount, scount, ns, nd, EBCC_GAMMA);
    __syncthreads();
    lift_step<false, true, LINES, SPAN>(s_sh, d_sh, lo, scount, dcount, ns, nd, EBCC_DELTA);
  }
  __syncthreads();
  // store the tile's own indices [i0, i0+TI)
  const int kbeg = i0 - lo;
  for (int e = threadIdx.x; e < LINES * TI; e += blockDim.x) {
    int l, kk;
    if (lines_contig) { l = e % LINES; kk = e / LINES; }
    else { kk = e % TI; l = e / TI; }
    int line = line0 + l;
    if (line >= nlines) continue;
    int i = i0 + kk;
    int k = kbeg + kk;
    int64_t lbase = (int64_t)line * line_stride;
    if (i < ns) {
      double v = s_sh[l][k];
      int64_t p = INVERSE ? 2 * (int64_t)i : i;
      epi.store(dst, blockIdx.z, lbase + p * elem_stride,
                INVERSE ? v : __dmul_rn(v, EBCC_SCALE_LOW));
    }
    if (i < nd) {
      double v = d_sh[l][k];
      int64_t p = INVERSE ? 2 * (int64_t)i + 1 : (int64_t)ns + i;
      epi.store(dst, blockIdx.z, lbase + p * elem_stride,
                INVERSE ? v : __dmul_rn(v, EBCC_SCALE_HIGH));
    }
  }
  epi.finish(blockIdx.z);
}


template <bool INVERSE, class Epi>
inline void launch_pass_epi(const double* in, double* out, int64_t field_stride, int nfields, int cols,
                 int r, int c, bool along_cols, cudaStream_t st, const Epi& epi) {
  if (along_cols) {
    // lines = columns (contiguous across lines), transform length r
    constexpr int LINES = 32, TI = 64;
    dim3 grid((c + LINES - 1) / LINES, ((r + 1) / 2 + TI - 1) / TI, nfields);
    lift_pass_kernel<INVERSE, LINES, TI, Epi><<<grid, 256, 0, st>>>(in, out, field_stride, 1,
                                                                     cols, c, r, epi);
  } else {
    // rows: longer tiles (fewer halo samples and barriers per sample)
    constexpr int LINES = EBCC_ROW_LINES, TI = EBCC_ROW_TI;
    dim3 grid((r + LINES - 1) / LINES, ((c + 1) / 2 + TI - 1) / TI, nfields);
    lift_pass_kernel<INVERSE, LINES, TI, Epi><<<grid, 256, 0, st>>>(in, out, field_stride, cols,
                                                                     1, r, c, epi);
  }
}


}  // namespace lift
}  // namespace ebcc
