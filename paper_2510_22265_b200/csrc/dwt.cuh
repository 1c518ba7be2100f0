// Host entry points of the CDF 9/7 passes (dwt.cu).  All take a batch of
// `nfields` arrays laid out field_stride doubles apart.
#pragma once
#include "common.cuh"

namespace ebcc {

// Default pass epilogue: plain store.  Kernels call begin(field) once per CTA
// (false = skip the CTA), store(dst, field, offset, value) per output sample
// and finish(field) once per CTA (all threads).
struct StoreEpi {
  __device__ __forceinline__ bool begin(int) const { return true; }
  __device__ __forceinline__ void store(double* dst, int, int64_t off, double v) const { dst[off] = v; }
  __device__ __forceinline__ void finish(int) const {}
};


// whole forward transform: a holds the input and receives the pyramid; b is scratch
void forward_dwt(double* a, double* b, int64_t field_stride, int nfields, const Geo& g,
                 cudaStream_t st);
// the same with the input read from `src` (level 0's row pass reads it; level 0
// covers the whole array, so a needs no copy of the input first)
void forward_dwt_from(const double* src, double* a, double* b, int64_t field_stride, int nfields,
                      const Geo& g, cudaStream_t st);
// whole inverse transform: a holds the pyramid and receives the field; b is scratch
void inverse_dwt(double* a, double* b, int64_t field_stride, int nfields, const Geo& g,
                 cudaStream_t st);
// single inverse half-passes of level k (region ll_shapes[k]): cols a->b, rows b->a
void inverse_level_cols(const double* a, double* b, int64_t field_stride, int nfields,
                        const Geo& g, int k, cudaStream_t st);
void inverse_level_rows(const double* b, double* a, int64_t field_stride, int nfields,
                        const Geo& g, int k, cudaStream_t st);

}  // namespace ebcc
