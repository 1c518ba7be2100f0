// Quality metrics of the reference's benchmark harness on the GPU
// (pkg/src/ebcc/bench/metrics.py restated): point-wise error statistics
// (core.error_stats, core.py:189-207), the symmetric error histogram
// (metrics.py:78-99), mean SSIM with an 11x11 Gaussian window (metrics.py:
// 31-75) and the isotropic radial power spectrum (metrics.py:102-125).
//
// All arithmetic is float64 like the reference.  Error statistics and SSIM
// reduce in a fixed order (per-thread grid-stride sums, block trees,
// per-field trees) and are deterministic; spectrum annuli are summed with
// shared-memory atomics (order-dependent in the last bits).  All differ from
// numpy's pairwise / BLAS / pocketfft orders only in the last bits; maxima
// and histogram counts are exact.
#include <cufft.h>

#include <cmath>
#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "ctx.cuh"

namespace ebcc {
namespace {

constexpr int MB = 256;   // threads per metric block
constexpr int SB = 128;   // blocks per field for the streaming reductions
constexpr int kSsimW = 11;
constexpr double kSsimSigma = 1.5, kK1 = 0.01, kK2 = 0.03, kRangeFloor = 1e-30;

struct Fail {
  int code;
  std::string what;
};
#define MCK(x)                                                                     \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) throw Fail{EBCC_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// ---- per-context scratch ---------------------------------------------------
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      if (bytes == 0) bytes = 16;
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw Fail{EBCC_E_NOMEM, "metrics scratch allocation"};
      }
      cap = bytes;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};
struct MetricsWs {
  Buf a, b, part, aux, maps, fft;
  cufftHandle plan = 0;
  int plan_rows = 0, plan_cols = 0, plan_batch = 0;
};
std::mutex g_mu;
std::unordered_map<ebcc_ctx*, MetricsWs> g_ws;

MetricsWs& ws_of(ebcc_ctx* c) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_ws[c];
}

// input pointer on the device (copied from host unless flagged device-resident)
template <class T>
const T* device_input(const T* p, size_t count, int flags, Buf& b, cudaStream_t st) {
  if (flags & EBCC_INPUT_ON_DEVICE) return p;
  T* d = static_cast<T*>(b.get(sizeof(T) * count));
  MCK(cudaMemcpyAsync(d, p, sizeof(T) * count, cudaMemcpyHostToDevice, st));
  return d;
}

// ---- block reductions (fixed order) -------------------------------------------
template <class T, class Op>
__device__ T block_reduce(T v, T* sm, Op op) {
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sm[threadIdx.x] = op(sm[threadIdx.x], sm[threadIdx.x + s]);
    __syncthreads();
  }
  T r = sm[0];
  __syncthreads();
  return r;
}
struct MaxD { __device__ double operator()(double x, double y) const { return x > y ? x : y; } };
struct MinF { __device__ float operator()(float x, float y) const { return x < y ? x : y; } };
struct MaxF { __device__ float operator()(float x, float y) const { return x > y ? x : y; } };
struct SumD { __device__ double operator()(double x, double y) const { return __dadd_rn(x, y); } };
struct SumU { __device__ unsigned long long operator()(unsigned long long x, unsigned long long y) const { return x + y; } };

// ---- error statistics ----------------------------------------------------------
struct StatPart {
  double max_abs, sumsq;
  float amin, amax;
  unsigned long long neq;
};

__global__ void __launch_bounds__(MB) stats_kernel(const float* __restrict__ a,
                                                   const float* __restrict__ b, int64_t n,
                                                   StatPart* part) {
  const int f = blockIdx.y;
  const float* af = a + (int64_t)f * n;
  const float* bf = b + (int64_t)f * n;
  double mx = 0.0, ss = 0.0;
  float lo = INFINITY, hi = -INFINITY;
  unsigned long long neq = 0;
  for (int64_t i = (int64_t)blockIdx.x * MB + threadIdx.x; i < n; i += (int64_t)gridDim.x * MB) {
    const float x = af[i], y = bf[i];
    const double d = __dsub_rn((double)y, (double)x);  // b - a in float64
    const double ad = fabs(d);
    mx = ad > mx ? ad : mx;
    ss = __dadd_rn(ss, __dmul_rn(ad, ad));
    lo = x < lo ? x : lo;
    hi = x > hi ? x : hi;
    neq += x != y;
  }
  __shared__ double smd[MB];
  __shared__ float smf[MB];
  __shared__ unsigned long long smu[MB];
  StatPart P;
  P.max_abs = block_reduce(mx, smd, MaxD());
  P.sumsq = block_reduce(ss, smd, SumD());
  P.amin = block_reduce(lo, smf, MinF());
  P.amax = block_reduce(hi, smf, MaxF());
  P.neq = block_reduce(neq, smu, SumU());
  if (threadIdx.x == 0) part[(int64_t)f * gridDim.x + blockIdx.x] = P;
}

__global__ void __launch_bounds__(SB) stats_final(const StatPart* part, int nb, double* out) {
  const int f = blockIdx.x;
  StatPart P = threadIdx.x < nb ? part[(int64_t)f * nb + threadIdx.x]
                                : StatPart{0.0, 0.0, INFINITY, -INFINITY, 0ull};
  __shared__ double smd[SB];
  __shared__ float smf[SB];
  __shared__ unsigned long long smu[SB];
  const double mx = block_reduce(P.max_abs, smd, MaxD());
  const double ss = block_reduce(P.sumsq, smd, SumD());
  const float lo = block_reduce(P.amin, smf, MinF());
  const float hi = block_reduce(P.amax, smf, MaxF());
  const unsigned long long neq = block_reduce(P.neq, smu, SumU());
  if (threadIdx.x == 0) {
    double* o = out + (int64_t)f * 5;
    o[0] = mx;
    o[1] = (double)lo;
    o[2] = (double)hi;
    o[3] = ss;
    o[4] = (double)neq;
  }
}

// ---- error histogram (np.histogram with explicit edges: bins are
// [e_k, e_k+1), the last one closed) -------------------------------------------
__global__ void __launch_bounds__(MB) hist_kernel(const float* __restrict__ a,
                                                  const float* __restrict__ b, int64_t n,
                                                  const double* __restrict__ edges, int bins,
                                                  unsigned long long* counts) {
  const int f = blockIdx.y;
  extern __shared__ unsigned char hsm[];
  double* e = reinterpret_cast<double*>(hsm);
  unsigned int* c = reinterpret_cast<unsigned int*>(e + bins + 1);
  for (int i = threadIdx.x; i <= bins; i += MB) e[i] = edges[(int64_t)f * (bins + 1) + i];
  for (int i = threadIdx.x; i < bins; i += MB) c[i] = 0;
  __syncthreads();
  const float* af = a + (int64_t)f * n;
  const float* bf = b + (int64_t)f * n;
  for (int64_t i = (int64_t)blockIdx.x * MB + threadIdx.x; i < n; i += (int64_t)gridDim.x * MB) {
    const double d = __dsub_rn((double)bf[i], (double)af[i]);
    if (!(d >= e[0] && d <= e[bins])) continue;
    int lo = 0, hi = bins;  // last k with e[k] <= d
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (e[mid] <= d) lo = mid;
      else hi = mid;
    }
    atomicAdd(&c[lo], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += MB)
    if (c[i]) atomicAdd(&counts[(int64_t)f * bins + i], (unsigned long long)c[i]);
}

// ---- SSIM --------------------------------------------------------------------
struct SsimK {
  double k[kSsimW];
};

// horizontal 11-tap pass over a, b, a*a, b*b, a*b: maps[5][g][rows][cw]
__global__ void __launch_bounds__(MB) ssim_h_kernel(const float* __restrict__ a,
                                                    const float* __restrict__ b, int rows,
                                                    int cols, SsimK K, double* maps, int g) {
  const int f = blockIdx.y;
  const int cw = cols - (kSsimW - 1);
  const int64_t n = (int64_t)rows * cols, nw = (int64_t)rows * cw;
  const float* af = a + (int64_t)f * n;
  const float* bf = b + (int64_t)f * n;
  for (int64_t o = (int64_t)blockIdx.x * MB + threadIdx.x; o < nw; o += (int64_t)gridDim.x * MB) {
    const int r = (int)(o / cw), j = (int)(o - (int64_t)r * cw);
    const float* ar = af + (int64_t)r * cols + j;
    const float* br = bf + (int64_t)r * cols + j;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
    for (int t = 0; t < kSsimW; t++) {
      const double x = ar[t], y = br[t], w = K.k[t];
      s0 = __dadd_rn(s0, __dmul_rn(x, w));
      s1 = __dadd_rn(s1, __dmul_rn(y, w));
      s2 = __dadd_rn(s2, __dmul_rn(__dmul_rn(x, x), w));
      s3 = __dadd_rn(s3, __dmul_rn(__dmul_rn(y, y), w));
      s4 = __dadd_rn(s4, __dmul_rn(__dmul_rn(x, y), w));
    }
    const int64_t stride = (int64_t)g * nw;
    double* m = maps + (int64_t)f * nw + o;
    m[0] = s0;
    m[stride] = s1;
    m[2 * stride] = s2;
    m[3 * stride] = s3;
    m[4 * stride] = s4;
  }
}

// vertical 11-tap pass + the SSIM map, summed per block (fixed order)
__global__ void __launch_bounds__(MB) ssim_v_kernel(int rows, int cols, SsimK K,
                                                    const double* maps, int g,
                                                    const double* __restrict__ crange,
                                                    double* part) {
  const int f = blockIdx.y;
  const int cw = cols - (kSsimW - 1), rw = rows - (kSsimW - 1);
  const int64_t nw = (int64_t)rows * cw, nv = (int64_t)rw * cw;
  const int64_t stride = (int64_t)g * nw;
  const double* m = maps + (int64_t)f * nw;
  const double c1 = crange[2 * f], c2 = crange[2 * f + 1];
  double acc = 0.0;
  for (int64_t o = (int64_t)blockIdx.x * MB + threadIdx.x; o < nv; o += (int64_t)gridDim.x * MB) {
    const int i = (int)(o / cw), j = (int)(o - (int64_t)i * cw);
    double v[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int t = 0; t < kSsimW; t++) {
      const int64_t q = (int64_t)(i + t) * cw + j;
      const double w = K.k[t];
#pragma unroll
      for (int c = 0; c < 5; c++) v[c] = __dadd_rn(v[c], __dmul_rn(m[c * stride + q], w));
    }
    const double mu_a = v[0], mu_b = v[1];
    const double mu_aa = __dmul_rn(mu_a, mu_a), mu_bb = __dmul_rn(mu_b, mu_b);
    const double mu_ab = __dmul_rn(mu_a, mu_b);
    const double var_a = __dsub_rn(v[2], mu_aa), var_b = __dsub_rn(v[3], mu_bb);
    const double cov = __dsub_rn(v[4], mu_ab);
    const double num = __dmul_rn(__dadd_rn(__dmul_rn(2.0, mu_ab), c1),
                                 __dadd_rn(__dmul_rn(2.0, cov), c2));
    const double den = __dmul_rn(__dadd_rn(__dadd_rn(mu_aa, mu_bb), c1),
                                 __dadd_rn(__dadd_rn(var_a, var_b), c2));
    acc = __dadd_rn(acc, __ddiv_rn(num, den));
  }
  __shared__ double sm[MB];
  const double s = block_reduce(acc, sm, SumD());
  if (threadIdx.x == 0) part[(int64_t)f * gridDim.x + blockIdx.x] = s;
}

__global__ void __launch_bounds__(SB) sum_parts(const double* part, int nb, double* out) {
  const int f = blockIdx.x;
  __shared__ double sm[SB];
  const double v = threadIdx.x < nb ? part[(int64_t)f * nb + threadIdx.x] : 0.0;
  const double s = block_reduce(v, sm, SumD());
  if (threadIdx.x == 0) out[f] = s;
}

// ---- radial power spectrum --------------------------------------------------
__global__ void to_complex(const float* __restrict__ a, int64_t count, cufftDoubleComplex* z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = make_cuDoubleComplex((double)a[i], 0.0);
}

__global__ void __launch_bounds__(MB) spectrum_bin(const cufftDoubleComplex* __restrict__ z,
                                                   int64_t n, double rc,
                                                   const int32_t* __restrict__ idx, int kmax,
                                                   double* out) {
  const int f = blockIdx.y;
  extern __shared__ double bins[];
  for (int i = threadIdx.x; i < kmax; i += MB) bins[i] = 0.0;
  __syncthreads();
  const cufftDoubleComplex* zf = z + (int64_t)f * n;
  for (int64_t i = (int64_t)blockIdx.x * MB + threadIdx.x; i < n; i += (int64_t)gridDim.x * MB) {
    const int k = idx[i];
    if (k < 1 || k > kmax) continue;
    // spec = fft2(a) / (rows*cols); power = abs(spec)**2
    const double re = __ddiv_rn(zf[i].x, rc), im = __ddiv_rn(zf[i].y, rc);
    const double h = hypot(re, im);
    atomicAdd(&bins[k - 1], __dmul_rn(h, h));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kmax; i += MB)
    if (bins[i] != 0.0) atomicAdd(&out[(int64_t)f * kmax + i], bins[i]);
}

int blocks_for(int64_t n, int cap) {
  int64_t b = (n + MB - 1) / MB;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

SsimK ssim_kernel_weights() {
  // metrics.py:31-36: exp(-x^2 / (2 sigma^2)), normalised by its sum
  SsimK K;
  for (int t = 0; t < kSsimW; t++) {
    const double x = (double)(t - kSsimW / 2);
    K.k[t] = std::exp(-(x * x) / (2.0 * (kSsimSigma * kSsimSigma)));
  }
  // k.sum() in numpy's pairwise order for 11 elements: eight running
  // partials, combined as a tree, then the tail in sequence
  const double* k = K.k;
  double s = ((k[0] + k[1]) + (k[2] + k[3])) + ((k[4] + k[5]) + (k[6] + k[7]));
  for (int t = 8; t < kSsimW; t++) s += k[t];
  for (int t = 0; t < kSsimW; t++) K.k[t] /= s;
  return K;
}

template <class F>
int guarded(ebcc_ctx* c, F body) {
  if (!c) return EBCC_E_ARGUMENT;
  try {
    MCK(cudaSetDevice(ctx_device(c)));
    body();
    return EBCC_OK;
  } catch (Fail& e) {
    cudaGetLastError();
    return ctx_fail(c, e.code, e.what.c_str());
  }
}

}  // namespace

void metrics_release(ebcc_ctx* c) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_ws.find(c);
  if (it == g_ws.end()) return;
  MetricsWs& w = it->second;
  w.a.release();
  w.b.release();
  w.part.release();
  w.aux.release();
  w.maps.release();
  w.fft.release();
  if (w.plan) cufftDestroy(w.plan);
  g_ws.erase(it);
}

}  // namespace ebcc

using namespace ebcc;

extern "C" {

int ebcc_error_stats(ebcc_ctx* c, const float* orig, const float* rec, int64_t nfields,
                     int64_t n, int32_t flags, double* out) {
  if (!c || !orig || !rec || !out || nfields < 0 || n < 1)
    return c ? ctx_fail(c, EBCC_E_ARGUMENT, "bad arguments") : EBCC_E_ARGUMENT;
  if (nfields == 0) return EBCC_OK;
  return guarded(c, [&] {
    MetricsWs& w = ws_of(c);
    cudaStream_t st = ctx_stream(c);
    const size_t cnt = (size_t)nfields * n;
    const float* a = device_input(orig, cnt, flags, w.a, st);
    const float* b = device_input(rec, cnt, flags, w.b, st);
    const int nb = blocks_for(n, SB);
    StatPart* part = static_cast<StatPart*>(w.part.get(sizeof(StatPart) * nb * nfields));
    double* d_out = static_cast<double*>(w.aux.get(sizeof(double) * 5 * nfields));
    for (int64_t f0 = 0; f0 < nfields; f0 += 65535) {
      const int g = (int)std::min<int64_t>(65535, nfields - f0);
      stats_kernel<<<dim3(nb, g), MB, 0, st>>>(a + f0 * n, b + f0 * n, n, part + f0 * nb);
      stats_final<<<g, SB, 0, st>>>(part + f0 * nb, nb, d_out + f0 * 5);
    }
    MCK(cudaGetLastError());
    MCK(cudaMemcpyAsync(out, d_out, sizeof(double) * 5 * nfields, cudaMemcpyDeviceToHost, st));
    MCK(cudaStreamSynchronize(st));
  });
}

int ebcc_error_histogram(ebcc_ctx* c, const float* orig, const float* rec, int64_t nfields,
                         int64_t n, int32_t bins, const double* edges, int32_t flags,
                         int64_t* counts) {
  if (!c || !orig || !rec || !edges || !counts || nfields < 0 || n < 1 || bins < 1 ||
      bins > 65536)
    return c ? ctx_fail(c, EBCC_E_ARGUMENT, "bad arguments") : EBCC_E_ARGUMENT;
  if (nfields == 0) return EBCC_OK;
  return guarded(c, [&] {
    MetricsWs& w = ws_of(c);
    cudaStream_t st = ctx_stream(c);
    const size_t cnt = (size_t)nfields * n;
    const float* a = device_input(orig, cnt, flags, w.a, st);
    const float* b = device_input(rec, cnt, flags, w.b, st);
    const size_t eb = sizeof(double) * (bins + 1) * nfields;
    const size_t cb = sizeof(unsigned long long) * bins * nfields;
    char* aux = static_cast<char*>(w.aux.get(eb + cb));
    double* d_edges = reinterpret_cast<double*>(aux);
    unsigned long long* d_counts = reinterpret_cast<unsigned long long*>(aux + eb);
    MCK(cudaMemcpyAsync(d_edges, edges, eb, cudaMemcpyHostToDevice, st));
    MCK(cudaMemsetAsync(d_counts, 0, cb, st));
    const size_t smem = sizeof(double) * (bins + 1) + sizeof(unsigned int) * bins;
    if (smem > 48 * 1024)
      MCK(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nb = blocks_for(n, SB);
    for (int64_t f0 = 0; f0 < nfields; f0 += 65535) {
      const int g = (int)std::min<int64_t>(65535, nfields - f0);
      hist_kernel<<<dim3(nb, g), MB, smem, st>>>(a + f0 * n, b + f0 * n, n,
                                                 d_edges + f0 * (bins + 1), bins,
                                                 d_counts + f0 * bins);
    }
    MCK(cudaGetLastError());
    MCK(cudaMemcpyAsync(counts, d_counts, cb, cudaMemcpyDeviceToHost, st));
    MCK(cudaStreamSynchronize(st));
  });
}

int ebcc_ssim(ebcc_ctx* c, const float* orig, const float* rec, int64_t nfields, int32_t rows,
              int32_t cols, int32_t flags, double* out) {
  if (!c || !orig || !rec || !out || nfields < 0 || rows < kSsimW || cols < kSsimW)
    return c ? ctx_fail(c, EBCC_E_ARGUMENT, "bad arguments (fields must be at least 11x11)")
             : EBCC_E_ARGUMENT;
  if (nfields == 0) return EBCC_OK;
  return guarded(c, [&] {
    MetricsWs& w = ws_of(c);
    cudaStream_t st = ctx_stream(c);
    const int64_t n = (int64_t)rows * cols;
    const size_t cnt = (size_t)nfields * n;
    const float* a = device_input(orig, cnt, flags, w.a, st);
    const float* b = device_input(rec, cnt, flags, w.b, st);
    // range of the first argument and equality, from the statistics pass
    std::vector<double> stats(5 * nfields);
    {
      const int nb = blocks_for(n, SB);
      StatPart* part = static_cast<StatPart*>(w.part.get(sizeof(StatPart) * nb * nfields));
      double* d_out = static_cast<double*>(w.aux.get(sizeof(double) * 5 * nfields));
      for (int64_t f0 = 0; f0 < nfields; f0 += 65535) {
        const int g = (int)std::min<int64_t>(65535, nfields - f0);
        stats_kernel<<<dim3(nb, g), MB, 0, st>>>(a + f0 * n, b + f0 * n, n, part + f0 * nb);
        stats_final<<<g, SB, 0, st>>>(part + f0 * nb, nb, d_out + f0 * 5);
      }
      MCK(cudaGetLastError());
      MCK(cudaMemcpyAsync(stats.data(), d_out, sizeof(double) * 5 * nfields,
                          cudaMemcpyDeviceToHost, st));
      MCK(cudaStreamSynchronize(st));
    }
    const SsimK K = ssim_kernel_weights();
    const int cw = cols - (kSsimW - 1), rw = rows - (kSsimW - 1);
    const int64_t nw = (int64_t)rows * cw;
    // fields per group: five float64 maps each, at most ~2 GB of maps
    int64_t G = (int64_t)((2ll << 30) / (5 * 8 * nw));
    G = G < 1 ? 1 : (G > 65535 ? 65535 : G);
    const int nbv = blocks_for((int64_t)rw * cw, SB);
    for (int64_t f0 = 0; f0 < nfields; f0 += G) {
      const int g = (int)std::min<int64_t>(G, nfields - f0);
      double* maps = static_cast<double*>(w.maps.get(sizeof(double) * 5 * nw * g));
      std::vector<double> cr(2 * g);
      for (int k = 0; k < g; k++) {
        const double* s = &stats[5 * (f0 + k)];
        double range = s[2] - s[1];
        range = range > kRangeFloor ? range : kRangeFloor;
        cr[2 * k] = (kK1 * range) * (kK1 * range);
        cr[2 * k + 1] = (kK2 * range) * (kK2 * range);
      }
      char* aux = static_cast<char*>(w.aux.get(sizeof(double) * (2 * g + (size_t)nbv * g + g)));
      double* d_cr = reinterpret_cast<double*>(aux);
      double* d_part = d_cr + 2 * g;
      double* d_sum = d_part + (size_t)nbv * g;
      MCK(cudaMemcpyAsync(d_cr, cr.data(), sizeof(double) * 2 * g, cudaMemcpyHostToDevice, st));
      ssim_h_kernel<<<dim3(blocks_for(nw, 4 * SB), g), MB, 0, st>>>(a + f0 * n, b + f0 * n, rows,
                                                                     cols, K, maps, g);
      ssim_v_kernel<<<dim3(nbv, g), MB, 0, st>>>(rows, cols, K, maps, g, d_cr, d_part);
      sum_parts<<<g, SB, 0, st>>>(d_part, nbv, d_sum);
      MCK(cudaGetLastError());
      std::vector<double> sums(g);
      MCK(cudaMemcpyAsync(sums.data(), d_sum, sizeof(double) * g, cudaMemcpyDeviceToHost, st));
      MCK(cudaStreamSynchronize(st));
      for (int k = 0; k < g; k++) {
        const double* s = &stats[5 * (f0 + k)];
        // identical inputs score exactly 1 (metrics.py:61-62)
        out[f0 + k] = s[4] == 0.0 ? 1.0 : sums[k] / (double)((int64_t)rw * cw);
      }
    }
  });
}

int ebcc_radial_spectrum(ebcc_ctx* c, const float* data, int64_t nfields, int32_t rows,
                         int32_t cols, const int32_t* bin_idx, int32_t kmax, int32_t flags,
                         double* out) {
  if (!c || !data || !bin_idx || !out || nfields < 0 || rows < 1 || cols < 1 || kmax < 1 ||
      kmax > 65536)
    return c ? ctx_fail(c, EBCC_E_ARGUMENT, "bad arguments") : EBCC_E_ARGUMENT;
  if (nfields == 0) return EBCC_OK;
  return guarded(c, [&] {
    MetricsWs& w = ws_of(c);
    cudaStream_t st = ctx_stream(c);
    const int64_t n = (int64_t)rows * cols;
    const float* a = device_input(data, (size_t)nfields * n, flags, w.a, st);
    // the wavenumber map comes from the host (np.rint(np.hypot(...)) exactly)
    const int32_t* idx = device_input(bin_idx, (size_t)n, 0, w.b, st);
    int64_t G = (int64_t)((2ll << 30) / (16 * n));
    G = G < 1 ? 1 : (G > 65535 ? 65535 : G);
    if (G > nfields) G = nfields;
    double* d_out = static_cast<double*>(w.aux.get(sizeof(double) * kmax * nfields));
    MCK(cudaMemsetAsync(d_out, 0, sizeof(double) * kmax * nfields, st));
    const double rc = (double)rows * (double)cols;
    const size_t smem = sizeof(double) * kmax;
    if (smem > 48 * 1024)
      MCK(cudaFuncSetAttribute(spectrum_bin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int64_t f0 = 0; f0 < nfields; f0 += G) {
      const int g = (int)std::min<int64_t>(G, nfields - f0);
      cufftDoubleComplex* z =
          static_cast<cufftDoubleComplex*>(w.fft.get(sizeof(cufftDoubleComplex) * n * g));
      if (!w.plan || w.plan_rows != rows || w.plan_cols != cols || w.plan_batch != g) {
        if (w.plan) cufftDestroy(w.plan);
        w.plan = 0;
        int dims[2] = {rows, cols};
        if (cufftPlanMany(&w.plan, 2, dims, nullptr, 1, (int)n, nullptr, 1, (int)n, CUFFT_Z2Z, g) !=
            CUFFT_SUCCESS)
          throw Fail{EBCC_E_CUDA, "cufftPlanMany"};
        w.plan_rows = rows;
        w.plan_cols = cols;
        w.plan_batch = g;
      }
      if (cufftSetStream(w.plan, st) != CUFFT_SUCCESS) throw Fail{EBCC_E_CUDA, "cufftSetStream"};
      to_complex<<<blocks_for(n * g, 4096), MB, 0, st>>>(a + f0 * n, n * g, z);
      if (cufftExecZ2Z(w.plan, z, z, CUFFT_FORWARD) != CUFFT_SUCCESS)
        throw Fail{EBCC_E_CUDA, "cufftExecZ2Z"};
      spectrum_bin<<<dim3(blocks_for(n, SB), g), MB, smem, st>>>(z, n, rc, idx, kmax,
                                                                 d_out + f0 * kmax);
      MCK(cudaGetLastError());
    }
    MCK(cudaMemcpyAsync(out, d_out, sizeof(double) * kmax * nfields, cudaMemcpyDeviceToHost, st));
    MCK(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
