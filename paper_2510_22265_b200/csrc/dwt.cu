// CDF 9/7 lifting passes (forward analysis and inverse synthesis), float64,
// bit-exact against the reference (dwt.py:112-216).
//
// One launch = one 1D pass (all rows or all columns of the level-k region)
// for every field of a batch.  A CTA owns LINES lines x TI subband indices;
// it stages the s/d halves plus a 2-sample halo on each side in shared
// memory, runs the four lifting steps there (one __syncthreads per step),
// and writes the tile out.  Border behaviour is the reference's whole-sample
// mirror expressed as index clamping: left[i]=d[max(i-1,0)],
// right[i]=d[min(i,nd-1)], s_right[i]=s[min(i+1,ns-1)].  Halo samples whose
// neighbours fall outside the staged window are computed from clamped
// (wrong) neighbours but never feed an output sample.
//
// Passes ping-pong between two buffers; only the region is written, so after
// a (rows, cols) or (cols, rows) pair the data is back in the first buffer
// with the untouched detail bands still in place.
#include "lift.cuh"
#include "fdwt_fused.cuh"
#include <cstdlib>

namespace ebcc {

using lift::launch_pass_epi;

namespace {
template <bool INVERSE>
void launch_pass(const double* in, double* out, int64_t field_stride, int nfields, int cols,
                 int r, int c, bool along_cols, cudaStream_t st) {
  launch_pass_epi<INVERSE, StoreEpi>(in, out, field_stride, nfields, cols, r, c, along_cols, st,
                                     StoreEpi{});
}
}  // namespace

void forward_level(const double* a, double* b, int64_t field_stride, int nfields, const Geo& g,
                   int k, cudaStream_t st) {
  // dwt.py:194-198: rows then columns on region ll_shapes[k]; a -> b -> a
  int r = g.lr[k], c = g.lc[k];
  launch_pass<false>(a, b, field_stride, nfields, g.cols, r, c, false, st);
  launch_pass<false>(b, const_cast<double*>(a), field_stride, nfields, g.cols, r, c, true, st);
}

void inverse_level_cols(const double* a, double* b, int64_t field_stride, int nfields,
                        const Geo& g, int k, cudaStream_t st) {
  launch_pass<true>(a, b, field_stride, nfields, g.cols, g.lr[k], g.lc[k], true, st);
}

void inverse_level_rows(const double* b, double* a, int64_t field_stride, int nfields,
                        const Geo& g, int k, cudaStream_t st) {
  launch_pass<true>(b, a, field_stride, nfields, g.cols, g.lr[k], g.lc[k], false, st);
}

namespace {
// Every level by the fused row + column kernel (fdwt_fused.cuh).  A level
// cannot run in place (CTAs read their neighbours' halo), so the levels
// ping-pong: level k reads its region from the buffer level k-1 wrote (src
// for level 0) and writes all four quadrants to the other of a / b; what a
// level leaves in b is copied to a afterwards -- its detail bands, and the LL
// band too after the last level -- so the pyramid ends up in a.  Degenerate
// regions (a single row or column at some level) keep the separable passes.
bool fused_forward(const double* src, double* a, double* b, int64_t field_stride, int nfields,
                   const Geo& g, cudaStream_t st) {
  static const bool on = !(getenv("EBCC_FDWT") && getenv("EBCC_FDWT")[0] == '0');
  if (!on) return false;
  for (int k = 0; k < g.levels; k++)
    if (g.lr[k] < 2 || g.lc[k] < 2) return false;
  const double* cur = src;
  for (int k = 0; k < g.levels; k++) {
    double* out = (cur == a) ? b : a;
    fdwt::launch_level(cur, out, field_stride, nfields, g.cols, g.lr[k], g.lc[k], st);
    if (out != a)
      fdwt::copy_bands(out, a, field_stride, nfields, g.cols, g.lr[k], g.lc[k],
                       k == g.levels - 1, st);
    cur = out;
  }
  return true;
}
}  // namespace

void forward_dwt(double* a, double* b, int64_t field_stride, int nfields, const Geo& g,
                 cudaStream_t st) {
  if (fused_forward(a, a, b, field_stride, nfields, g, st)) return;
  for (int k = 0; k < g.levels; k++) forward_level(a, b, field_stride, nfields, g, k, st);
}

void forward_dwt_from(const double* src, double* a, double* b, int64_t field_stride, int nfields,
                      const Geo& g, cudaStream_t st) {
  if (fused_forward(src, a, b, field_stride, nfields, g, st)) return;
  // level 0: rows src -> b, columns b -> a (the whole array is the region)
  const int r = g.lr[0], c = g.lc[0];
  launch_pass<false>(src, b, field_stride, nfields, g.cols, r, c, false, st);
  launch_pass<false>(b, a, field_stride, nfields, g.cols, r, c, true, st);
  for (int k = 1; k < g.levels; k++) forward_level(a, b, field_stride, nfields, g, k, st);
}

void inverse_dwt(double* a, double* b, int64_t field_stride, int nfields, const Geo& g,
                 cudaStream_t st) {
  // dwt.py:211-215: coarse to fine, columns then rows; a -> b -> a
  for (int k = g.levels - 1; k >= 0; k--) {
    inverse_level_cols(a, b, field_stride, nfields, g, k, st);
    inverse_level_rows(b, a, field_stride, nfields, g, k, st);
  }
}

}  // namespace ebcc
