#include <algorithm>
// Field-level kernels of the EBCC path: the closed-form prefix decode and the
// feedback probes built on the lifting passes.
//
// Closed form: decoding B stream bits leaves coefficient c at
//   0                                   if its sign bit offset >= B
//   sign * floor(|c| / 2^m) * 2^m       otherwise,
// where m is the lowest plane whose refinement bit for c lies below B.  The
// refinement bit of plane p for LSP rank r is at refine_start[p] + r, so m is
// found by walking up from the significance plane through a 64-entry table.
// The result is an exact float64 built from the top `kept` mantissa bits.
// A probe = that decode + the inverse DWT + a reduction fused into the last
// row pass; no intermediate field is written at level 0.
#include "idwt_fused.cuh"
#include "lift.cuh"
#include "probe.cuh"

namespace ebcc {

namespace fused {
thread_local Level0Timer* g_level0_timer = nullptr;
}

namespace {

__device__ __forceinline__ unsigned int f32_key(float v) {
  unsigned int u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_f32(unsigned int k) {
  unsigned int u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// Signed zeros: numpy's float32 min/max keep one of several tied zeros by its
// SIMD lane order, which differs between CPUs (and between positions of the
// same data); this path pins "+0.0 preferred": the extremum is -0.0 only if
// the field holds no +0.0 (max already behaves so in key order; for min the
// two zero keys are swapped).  The oracle applies the same rule.
__device__ __forceinline__ unsigned int zswap(unsigned int k) {
  return k == 0x7fffffffu ? 0x80000000u : (k == 0x80000000u ? 0x7fffffffu : k);
}

__global__ void mm_init_kernel(unsigned int* mm, unsigned long long* first_bad, int nfields) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nfields) { mm[2 * f] = 0xffffffffu; mm[2 * f + 1] = 0u; first_bad[f] = ~0ull; }
}

// 16-byte loads where the field allows, one atomic pair per CTA (the warps'
// results meet in shared memory: thousands of warps hammering a field's two
// words had made this pass 8x slower than its HBM time)
__global__ void __launch_bounds__(256) minmax_kernel(const float* __restrict__ x, int64_t n,
                                                     unsigned int* mm,
                                                     unsigned long long* first_bad) {
  const int f = blockIdx.y;
  const float* xf = x + (int64_t)f * n;
  unsigned int lo = 0xffffffffu, hi = 0u;
  unsigned long long bad = ~0ull;
  auto take = [&](float v, int64_t i) {
    if (!isfinite(v)) bad = bad < (unsigned long long)i ? bad : (unsigned long long)i;
    const unsigned int k = f32_key(v);
    const unsigned int km = zswap(k);
    lo = km < lo ? km : lo;
    hi = k > hi ? k : hi;
  };
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  if (!(n & 3) && !((uintptr_t)xf & 15)) {
    const float4* x4 = reinterpret_cast<const float4*>(xf);
    for (int64_t i = t0; i < n / 4; i += nt) {
      const float4 v = x4[i];
      take(v.x, 4 * i); take(v.y, 4 * i + 1); take(v.z, 4 * i + 2); take(v.w, 4 * i + 3);
    }
  } else {
    for (int64_t i = t0; i < n; i += nt) take(xf[i], i);
  }
  if (bad != ~0ull) atomicMin(&first_bad[f], bad);  // core._check_finite, on device
  for (int o = 16; o; o >>= 1) {
    unsigned int a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  __shared__ unsigned int s_lo[8], s_hi[8];
  if ((threadIdx.x & 31) == 0) { s_lo[threadIdx.x >> 5] = lo; s_hi[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
      lo = s_lo[w] < lo ? s_lo[w] : lo;
      hi = s_hi[w] > hi ? s_hi[w] : hi;
    }
    atomicMin(&mm[2 * f], lo);
    atomicMax(&mm[2 * f + 1], hi);
  }
}

// core.normalize (core.py:161-180) + _ChunkCoder.eps_abs (pipeline.py:98)
__global__ void scalars_kernel(const unsigned int* mm, const unsigned long long* first_bad,
                               int nfields, double eps_rel, FieldScal* fs) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfields) return;
  double vmin = (double)key_f32(zswap(mm[2 * f])), vmax = (double)key_f32(mm[2 * f + 1]);
  double range = __dsub_rn(vmax, vmin);
  FieldScal s;
  s.vmin = vmin; s.vmax = vmax; s.range = range;
  s.range_inv = __drcp_rn(range);
  s.eps_rel = eps_rel;
  s.eps_abs = __dmul_rn(eps_rel, range);
  s.constant = range < 1e-30;
  s.pad = 0;
  s.first_bad = (long long)(first_bad[f] == ~0ull ? -1ll : (long long)first_bad[f]);
  fs[f] = s;
}

__global__ void normalize_kernel(const float* __restrict__ x, int64_t n, const FieldScal* fs,
                                 double* __restrict__ norm) {
  const int f = blockIdx.y;
  const FieldScal s = fs[f];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = (double)x[(int64_t)f * n + i];
    norm[(int64_t)f * n + i] = s.constant ? 0.0 : __ddiv_rn(__dsub_rn(v, s.vmin), s.range);
  }
}

__global__ void decode_coeffs_kernel(Meta m, const ProbeParam* __restrict__ prm,
                                     double* __restrict__ out, int64_t n) {
  const int f = blockIdx.y;
  const ProbeParam P = prm[f];
  if (!P.active) return;
  __shared__ uint32_t T[kMaxPlaneRecs];
  const int n_max = m.mo[f].n_max;
  int planes = P.planes, n_last = P.n_last;
  if (planes < 0) {
    planes = m.mo[f].planes_run;
    n_last = planes > 0 ? n_max - (planes - 1) : n_max;
  }
  fused::build_thresholds(T, m.planes + (int64_t)f * kMaxPlaneRecs, planes, P.B);
  const int64_t fo = (int64_t)f * m.stride;
  const uint32_t RB = fused::rank_bound(m.sprank + fo, m.mo[f].lsp_count, P.B);
  __syncthreads();
  const double off = P.midpoint ? scalbn(0.5, n_last) : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[(int64_t)f * n + i] = fused::decode_raw_scan(
        m.packed[fo + i], m.rank_hi ? (uint32_t)m.rank_hi[fo + i] << kRankBits : 0u, RB, planes,
        n_max, P.midpoint != 0, off, T);
}

// 8-byte probe records + sign offsets by rank (sprank preset to kNone)
__global__ void pack_meta_kernel(MachineBufs mb, uint2* packed, uint32_t* sprank,
                                 uint32_t* lspn, uint8_t* rank_hi) {
  const int f = blockIdx.y;
  const int64_t fo = (int64_t)f * mb.stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < mb.stride;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t sp = mb.sign_pos[fo + i];
    const uint32_t pi = mb.pinfo[fo + i];
    const uint32_t rank = sp == kNone ? 0xffffffffu : mb.lsp_rank[fo + i];
    packed[fo + i] = make_uint2((rank & kRankNone) | ((pi & 0x3fu) << kRankBits),
                                ((pi & 0x80u) << 24) | (mb.mant[fo + i] & 0x7fffffffu));
    if (rank_hi) rank_hi[fo + i] = (uint8_t)(rank >> kRankBits);
    if (sprank && sp != kNone) {  // (null: the encoder wrote both by rank already)
      sprank[fo + rank] = sp;
      if (lspn) lspn[fo + rank] = (uint32_t)i;
    }
  }
}

// ---- epilogues for the last (level-0 row) pass -----------------------------

__device__ __forceinline__ double denorm_err(const FieldScal& s, double dec, float orig) {
  // pipeline.py:116-119: rec = f32(vmin + dec*range); |f64(rec) - f64(orig)|
  float rec = __double2float_rn(__dadd_rn(s.vmin, __dmul_rn(dec, s.range)));
  return fabs(__dsub_rn((double)rec, (double)orig));
}

__device__ __forceinline__ void warp_flush(ProbeResult* r, unsigned long long cnt, double mx,
                                           bool do_count) {
  unsigned long long mxb = (unsigned long long)__double_as_longlong(mx);
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    unsigned long long y = __shfl_xor_sync(0xffffffffu, mxb, o);
    mxb = y > mxb ? y : mxb;
  }
  if ((threadIdx.x & 31) == 0) {
    if (do_count && cnt) atomicAdd(&r->count, cnt);
    atomicMax(&r->maxerr, mxb);
  }
}

// incremental probes: the CTA's tile total -> TileStat, the tile's flag
// (clean, or count stale when this probe did not count) and the result
__device__ __forceinline__ void tile_flush(ProbeResult* r, TileStat* t, volatile uint8_t* flag,
                                           unsigned long long cnt, double mx, bool do_count,
                                           bool aborted, bool add_count = true) {
  __shared__ unsigned long long s_cnt, s_mx;
  if (threadIdx.x == 0) { s_cnt = 0; s_mx = 0; }
  __syncthreads();
  unsigned long long mxb = (unsigned long long)__double_as_longlong(mx);
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    unsigned long long y = __shfl_xor_sync(0xffffffffu, mxb, o);
    mxb = y > mxb ? y : mxb;
  }
  if ((threadIdx.x & 31) == 0) {
    if (do_count && cnt) atomicAdd(&s_cnt, cnt);
    atomicMax(&s_mx, mxb);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (aborted) {  // the tile stopped early: recompute it on the next probe
      *flag = kTileDirty;
      atomicMax(&r->maxerr, s_mx);
      return;
    }
    t->count = s_cnt;
    t->maxerr = s_mx;
    *flag = do_count ? 0 : kTileCountStale;
    if (do_count && add_count && s_cnt) atomicAdd(&r->count, s_cnt);
    atomicMax(&r->maxerr, s_mx);
  }
}

// an error above eps_abs already recorded for chunk f by another CTA
__device__ __forceinline__ bool settled(const ProbeResult* r, double eps_abs) {
  const unsigned long long b = *reinterpret_cast<const volatile unsigned long long*>(&r->maxerr);
  return __longlong_as_double((long long)b) > eps_abs;
}

#ifndef EBCC_MINB_COUNT
#define EBCC_MINB_COUNT 3  // abortable count probes: 80 registers, no spills (measured -1.3% compress vs 4 CTAs/SM without abort)
#endif
// violations pushed so far: the count probes' abort test
__device__ __forceinline__ unsigned long long viol_seen(const ProbeResult* r) {
  return *reinterpret_cast<const volatile unsigned long long*>(&r->count);
}
// this CTA's count-probe violations (its tile total, incremental probes)
__device__ __forceinline__ unsigned int& tile_violations() {
  __shared__ unsigned int s_tile_viol;
  return s_tile_viol;
}

// COUNT: base-search probes (quantile count + max error); otherwise a
// pure-base feasibility probe (max error only).  Both abortable: a count
// probe stops once both of its answers are known to be "no" (ProbeParam)
template <bool COUNT>
struct BaseProbeEpi {
  const double* norm; const float* orig; const FieldScal* fs; const ProbeParam* prm;
  ProbeResult* res; int64_t n;
  unsigned long long cnt; double mx; FieldScal s;  // (cnt: unused, see cc)
  unsigned int cc;  // count: this lane's violations not yet pushed
  static constexpr bool count = COUNT;
  static constexpr bool kAbort = true;
  static constexpr int kMinBlocks = COUNT ? EBCC_MINB_COUNT : EBCC_MINB_EARLY;
  // masked path: only "some error exceeds eps_abs" is tracked; the reported
  // maximum is then +inf or 0 (every consumer only asks max_err <= eps_abs)
  bool bad;
  using Pre = float;
  __device__ Pre pre(int f, int64_t off) const { return orig[(int64_t)f * n + off]; }
  __device__ Pre pre_masked(int f, int64_t off) const { return pre(f, off); }
  // the level kernel stages the originals of a chunk's rows in shared memory
  static constexpr bool kStageOrig = true;
  __host__ __device__ const float* stage_src() const { return orig; }
  __device__ Pre pre_staged(int, int64_t, float o) const { return o; }
  __device__ bool begin(int v, int f) {  // probe v of chunk f
    cnt = 0; mx = 0.0; bad = false; cc = 0;
    if (count && threadIdx.x == 0) tile_violations() = 0;  // read after the chunk barriers
    if (!prm[v].active) return false;
    s = fs[f];
    return true;
  }
  __device__ double mxv() const { return bad ? (double)INFINITY : mx; }
  __device__ bool skip(int v) const {
    if (!prm[v].early || !settled(&res[v], s.eps_abs)) return false;
    return !count || (long long)viol_seen(&res[v]) > (long long)prm[v].vlim;
  }
  __device__ void put(double*, int f, int64_t off, double dec, float o) {
    if (count) {  // quantile search: the points missing |dec - norm| <= eps_rel
      // normalised value recomputed exactly like core.normalize (core.py:179)
      double nv = fused::div_exact(__dsub_rn((double)o, s.vmin), s.range, s.range_inv);
      cc += !(fabs(__dsub_rn(dec, nv)) <= s.eps_rel);
    }
    double e = denorm_err(s, dec, o);
    mx = fmax(e, mx);
  }
  // (count probes push their violations in chunk_done; the rest here)
  __device__ void finish(int f) {
    push(f, threadIdx.x & 31);
    warp_flush(&res[f], 0, mxv(), false);
  }
  // every lane computes; invalid lanes contribute nothing (no divergence)
  static constexpr bool kMasked = true, kProbe = true;
  __device__ void put_masked(int, int64_t, double dec, float o, bool valid) {
    if (count) {
      double nv = fused::div_exact(__dsub_rn((double)o, s.vmin), s.range, s.range_inv);
      cc += (valid && !(fabs(__dsub_rn(dec, nv)) <= s.eps_rel)) ? 1u : 0u;
    }
    bad |= valid && denorm_err(s, dec, o) > s.eps_abs;
  }
  // after every row chunk (whole warp): publish a first error above eps_abs
  // and, for count probes, the violations found since the last push
  __device__ void chunk_done(int v, int lane, bool& reported) {
    if (!reported && __any_sync(0xffffffffu, bad)) {
      if (lane == 0) report(v);
      reported = true;
    }
    push(v, lane);
  }
  // count probes: the warp's violations found since the last push
  __device__ void push(int v, int lane) {
    if (count && __any_sync(0xffffffffu, cc != 0)) {
      unsigned int d = cc;
      for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (lane == 0) {
        atomicAdd(&res[v].count, (unsigned long long)d);
        atomicAdd(&tile_violations(), d);
      }
      cc = 0;
    }
  }
  // incremental probes
  static constexpr bool kFinal = true;
  __device__ bool counting() const { return count; }
  __device__ void add_stored(int f, const TileStat& t) {
    if (count && t.count) atomicAdd(&res[f].count, t.count);
    atomicMax(&res[f].maxerr, t.maxerr);
  }
  __device__ void finish_inc(int f, TileStat* t, volatile uint8_t* flag, bool aborted) {
    unsigned long long tot = 0;
    if (count) {
      push(f, threadIdx.x & 31);
      __syncthreads();  // every warp's last push
      tot = threadIdx.x == 0 ? tile_violations() : 0;
    }
    tile_flush(&res[f], t, flag, tot, mxv(), count, aborted, false);
  }
  __device__ void report(int f) {
    atomicMax(&res[f].maxerr, (unsigned long long)__double_as_longlong((double)INFINITY));
  }
};

#ifndef EBCC_TRUNC_PREBASE
#define EBCC_TRUNC_PREBASE 1
#endif
struct TruncPre {
  double base;
  float orig;
};
// masked truncation epilogue: only the original is prefetched (register
// pressure); the base reconstruction is loaded at the put

struct TruncProbeEpi {
  const double* base; const float* orig; const FieldScal* fs; const ProbeParam* prm;
  ProbeResult* res; int64_t n;
  double mx; FieldScal s;
  bool bad;  // masked path (see BaseProbeEpi)
  static constexpr bool kAbort = true;
  // the midpoint decode + base add need more registers: 3 CTAs/SM, no spills
  static constexpr int kMinBlocks = EBCC_MINB_TRUNC;
  using Pre = TruncPre;
  __device__ Pre pre(int f, int64_t off) const {
    return {base[(int64_t)f * n + off], orig[(int64_t)f * n + off]};
  }
  __device__ bool begin(int v, int f) {  // probe v of chunk f
    mx = 0.0; bad = false;
    if (!prm[v].active) return false;
    s = fs[f];
    return true;
  }
  __device__ double mxv() const { return bad ? (double)INFINITY : mx; }
  __device__ bool skip(int f) const { return prm[f].early && settled(&res[f], s.eps_abs); }
  __device__ void put(double*, int f, int64_t off, double v, const Pre& p) {
    double rec = __dadd_rn(p.base, v);  // base_field + dequantized
    double e = denorm_err(s, rec, p.orig);
    mx = fmax(e, mx);
  }
  __device__ void finish(int f) { warp_flush(&res[f], 0, mxv(), false); }
  static constexpr bool kMasked = true, kProbe = true;
#if EBCC_TRUNC_PREBASE
  // both inputs prefetched before the row lifting (the kernel runs at 3
  // CTAs/SM, 80 registers: room for them)
  __device__ Pre pre_masked(int f, int64_t off) const { return pre(f, off); }
  static constexpr bool kStageOrig = true;
  __host__ __device__ const float* stage_src() const { return orig; }
  __device__ Pre pre_staged(int f, int64_t off, float o) const {
    return {base[(int64_t)f * n + off], o};
  }
  __device__ void put_masked(int, int64_t, double v, const Pre& p, bool valid) {
    const double rec = __dadd_rn(p.base, v);
    bad |= valid && denorm_err(s, rec, p.orig) > s.eps_abs;
  }
#else
  __device__ Pre pre_masked(int f, int64_t off) const { return {0.0, orig[(int64_t)f * n + off]}; }
  __device__ void put_masked(int f, int64_t off, double v, const Pre& p, bool valid) {
    const double rec = __dadd_rn(base[(int64_t)f * n + off], v);
    bad |= valid && denorm_err(s, rec, p.orig) > s.eps_abs;
  }
#endif
  static constexpr bool kFinal = true;
  __device__ bool counting() const { return false; }
  __device__ void chunk_done(int v, int lane, bool& reported) {
    if (!reported && __any_sync(0xffffffffu, bad)) {
      if (lane == 0) report(v);
      reported = true;
    }
  }
  __device__ void add_stored(int f, const TileStat& t) { atomicMax(&res[f].maxerr, t.maxerr); }
  __device__ void finish_inc(int f, TileStat* t, volatile uint8_t* flag, bool aborted) {
    tile_flush(&res[f], t, flag, 0, mxv(), false, aborted);
  }
  __device__ void report(int f) {
    atomicMax(&res[f].maxerr, (unsigned long long)__double_as_longlong((double)INFINITY));
  }
};

struct ResidueEpi {
  EBCC_NO_STAGE
  static constexpr bool kAbort = false;
  static constexpr int kMinBlocks = EBCC_MINB;
  static constexpr bool kMasked = false, kProbe = false;
  template <class P> __device__ void put_masked(int, int64_t, double, const P&, bool) {}
  __device__ auto pre_masked(int f, int64_t off) const { return pre(f, off); }
  const double* norm; double* base_dec; double* resid; const ProbeParam* prm; int64_t n;
  using Pre = double;
  __device__ Pre pre(int f, int64_t off) const { return norm[(int64_t)f * n + off]; }
  __device__ bool begin(int v, int) { return prm[v].active != 0; }
  __device__ bool skip(int) const { return false; }
  __device__ void put(double*, int f, int64_t off, double dec, double nv) {
    int64_t o = (int64_t)f * n + off;
    base_dec[o] = dec;
    resid[o] = __dsub_rn(nv, dec);  // nc.values - base_enc.decoded
  }
  __device__ void finish(int) {}
  bool bad = false;  // (probe epilogues only)
  __device__ void report(int) {}
};

struct StoreFieldEpi {
  EBCC_NO_STAGE
  static constexpr bool kAbort = false;
  static constexpr int kMinBlocks = EBCC_MINB;
  static constexpr bool kMasked = false, kProbe = false;
  template <class P> __device__ void put_masked(int, int64_t, double, const P&, bool) {}
  __device__ auto pre_masked(int f, int64_t off) const { return pre(f, off); }
  double* out; const ProbeParam* prm; int64_t n;
  using Pre = fused::NoPre;
  __device__ Pre pre(int, int64_t) const { return {}; }
  __device__ bool begin(int v, int) { return prm[v].active != 0; }
  __device__ bool skip(int) const { return false; }
  __device__ void put(double*, int f, int64_t off, double v, const Pre&) {
    out[(int64_t)f * n + off] = v;
  }
  __device__ void finish(int) {}
  bool bad = false;  // (probe epilogues only)
  __device__ void report(int) {}
};

struct AddDenormEpi {
  EBCC_NO_STAGE
  static constexpr bool kAbort = false;
  static constexpr int kMinBlocks = EBCC_MINB;
  static constexpr bool kMasked = false, kProbe = false;
  template <class P> __device__ void put_masked(int, int64_t, double, const P&, bool) {}
  __device__ auto pre_masked(int f, int64_t off) const { return pre(f, off); }
  const double* base; const FieldScal* fs; const ProbeParam* prm; float* out32; int64_t n;
  FieldScal s;
  using Pre = double;
  __device__ Pre pre(int f, int64_t off) const { return base[(int64_t)f * n + off]; }
  __device__ bool begin(int v, int f) {
    if (!prm[v].active) return false;
    s = fs[f];
    return true;
  }
  __device__ bool skip(int) const { return false; }
  __device__ void put(double*, int f, int64_t off, double v, double b) {
    int64_t o = (int64_t)f * n + off;
    double fld = __dadd_rn(b, v);
    out32[o] = __double2float_rn(__dadd_rn(s.vmin, __dmul_rn(fld, s.range)));
  }
  __device__ void finish(int) {}
  bool bad = false;  // (probe epilogues only)
  __device__ void report(int) {}
};

int grid_for(int64_t n, int cap = 2048) {
  int64_t b = (n + 255) / 256;
  return (int)(b > cap ? cap : (b < 1 ? 1 : b));
}

__global__ void denorm_kernel(const double* base, const FieldScal* fs, const uint8_t* active,
                              int64_t n, float* out32) {
  const int f = blockIdx.y;
  if (!active[f]) return;
  const FieldScal s = fs[f];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = (int64_t)f * n + i;
    out32[o] = __double2float_rn(__dadd_rn(s.vmin, __dmul_rn(base[o], s.range)));
  }
}

__global__ void fill_kernel(const FieldScal* fs, const uint8_t* active, int64_t n, float* out32) {
  const int f = blockIdx.y;
  if (!active[f]) return;
  const float v = (float)fs[f].vmin;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out32[(int64_t)f * n + i] = v;
}

// one CTA per part; bytes are MSB-first stream bytes = little-endian words
__global__ void pack_kernel(const PackPart* parts, uint8_t* out) {
  const PackPart P = parts[blockIdx.y];
  uint8_t* d = out + P.dst_off;
  const uint8_t* s = reinterpret_cast<const uint8_t*>(P.src);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.nbytes;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t v;
    if (i < (uint64_t)kHeader) {
      v = P.hdr[i];
    } else {
      uint64_t j = i - kHeader;
      v = s[j];
      uint64_t bit0 = j * 8;
      if (bit0 + 8 > P.bit_limit) {
        int keep = bit0 >= P.bit_limit ? 0 : (int)(P.bit_limit - bit0);
        v &= (uint8_t)(0xff00u >> keep);
      }
    }
    d[i] = v;
  }
}

__global__ void unpack_kernel(const UnpackPart* parts, const uint8_t* in) {
  const UnpackPart P = parts[blockIdx.y];
  uint8_t* d = reinterpret_cast<uint8_t*>(P.dst);
  uint64_t padded = (P.nbytes + 7) & ~7ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < padded;
       i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = i < P.nbytes ? in[P.src_off + i] : 0;
}

// container image: chunk i's record (25 bytes) then its payload
__global__ void container_kernel(const ContainerPart* parts, const uint8_t* records,
                                 const uint8_t* payload, uint8_t* out) {
  const int i = blockIdx.y;
  const ContainerPart P = parts[i];
  uint8_t* d = out + P.dst_off;
  const uint8_t* s = payload + P.src_off;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < P.len + 25;
       k += (int64_t)gridDim.x * blockDim.x)
    d[k] = k < 25 ? records[(int64_t)i * 25 + k] : s[k - 25];
}

}  // namespace

void assemble_container(const ContainerPart* parts, int nparts, const uint8_t* records,
                        const uint8_t* payload, uint8_t* out, cudaStream_t st) {
  for (int b = 0; b < nparts; b += 65535)
    container_kernel<<<dim3(64, std::min(65535, nparts - b)), 256, 0, st>>>(
        parts + b, records + (int64_t)b * 25, payload, out);
}

void ingest_normalize(const float* x, int64_t n, int nfields, double* norm, FieldScal* fs,
                      unsigned int* mm, double eps_rel, cudaStream_t st) {
  unsigned long long* first_bad = reinterpret_cast<unsigned long long*>(mm + 2 * nfields);
  mm_init_kernel<<<(nfields + 127) / 128, 128, 0, st>>>(mm, first_bad, nfields);
  // up to 128 CTAs per field: fills the machine for a single chunk, few
  // atomics per field for a batch
  minmax_kernel<<<dim3(grid_for(n / 4 + 1, 128), nfields), 256, 0, st>>>(x, n, mm, first_bad);
  scalars_kernel<<<(nfields + 127) / 128, 128, 0, st>>>(mm, first_bad, nfields, eps_rel, fs);
  normalize_kernel<<<dim3(grid_for(n, 1024), nfields), 256, 0, st>>>(x, n, fs, norm);
}

namespace {
// splitmix64
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double rand_double(uint64_t r, int emin, int emax) {
  // random sign, exponent in [emin, emax], random 52-bit significand
  int e = emin + (int)((r >> 52) % (uint64_t)(emax - emin + 1));
  uint64_t bits = ((uint64_t)(e + 1023) << 52) | (r & ((1ull << 52) - 1));
  if ((r >> 63) & 1) bits |= 1ull << 63;
  return __longlong_as_double((long long)bits);
}
__global__ void selftest_div_kernel(int64_t n, uint64_t seed, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t r1 = mix64(seed ^ (uint64_t)i), r2 = mix64(r1), r3 = mix64(r2);
    double x = rand_double(r1, -60, 60);
    if ((r3 & 15) == 0) x = (double)(int64_t)(r3 >> 40);  // integers, incl. 0
    // the two scale constants (inverse DWT)
    local += __double_as_longlong(fused::div_scale(x, EBCC_SCALE_LOW, EBCC_INV_SL)) !=
             __double_as_longlong(__ddiv_rn(x, EBCC_SCALE_LOW));
    local += __double_as_longlong(fused::div_scale(x, EBCC_SCALE_HIGH, EBCC_INV_SH)) !=
             __double_as_longlong(__ddiv_rn(x, EBCC_SCALE_HIGH));
    // runtime divisors (normalisation by the value range)
    double b = fabs(rand_double(r2, -40, 40));
    local += __double_as_longlong(fused::div_exact(x, b, __drcp_rn(b))) !=
             __double_as_longlong(__ddiv_rn(x, b));
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}
}  // namespace

void selftest_div(int64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t st) {
  selftest_div_kernel<<<148 * 8, 256, 0, st>>>(n, seed, bad);
}

void pack_meta(const MachineBufs& mb, uint2* packed, uint32_t* sprank, cudaStream_t st,
               uint32_t* lspn, uint8_t* rank_hi) {
  if (sprank) cudaMemsetAsync(sprank, 0xff, sizeof(uint32_t) * mb.stride * mb.nfields, st);
  pack_meta_kernel<<<dim3(grid_for(mb.stride, 1024), mb.nfields), 256, 0, st>>>(mb, packed,
                                                                                 sprank, lspn, rank_hi);
}

void decode_coeffs(const Meta& m, const ProbeParam* prm, double* a, int64_t n, int nfields,
                   cudaStream_t st) {
  decode_coeffs_kernel<<<dim3(grid_for(n, 1024), nfields), 256, 0, st>>>(m, prm, a, n);
}

void probe_base(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                int nfields, const double* norm, const float* orig, const FieldScal* fs,
                ProbeResult* res, cudaStream_t st, const Inc* inc, bool xe, bool early, int nphys) {
  // nfields probes; probe v reads chunk v % nphys (several per chunk: the
  // incremental path only)
  auto run = [&](auto e) {
    if (inc) fused::inverse_inc(m, prm, *inc, a, g, nfields, st, e, false, xe, nphys);
    else fused::inverse_fused(m, prm, a, b, g, nfields, st, e, false, xe);
  };
  if (early) run(BaseProbeEpi<false>{norm, orig, fs, prm, res, g.n, 0, 0.0, FieldScal{}, 0});
  else run(BaseProbeEpi<true>{norm, orig, fs, prm, res, g.n, 0, 0.0, FieldScal{}, 0});
}

void probe_trunc(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                 int nprobes, const double* base_dec, const float* orig, const FieldScal* fs,
                 ProbeResult* res, cudaStream_t st, const Inc* inc, bool xe, int nphys) {
  // probe v reads chunk v % nphys; several probes per chunk need the
  // incremental path (one LL buffer per probe)
  TruncProbeEpi e{base_dec, orig, fs, prm, res, g.n, 0.0, FieldScal{}};
  if (inc) fused::inverse_inc(m, prm, *inc, a, g, nprobes, st, e, true, xe, nphys);
  else fused::inverse_fused(m, prm, a, b, g, nprobes, st, e, true, xe);
}

// the level kernels' CTA tiling per level (fused::level_rows) and the
// persistent LL layout: level k >= 1 at columns coloff[k].. of an
// lr[1] x cols field, side by side
bool inc_geometry(const Geo& g, int nfields, Inc& inc) {
  IncGeo& ig = inc.ig;
  ig = IncGeo{};
  ig.levels = g.levels;
  ig.cols = g.cols;
  for (int k = 0; k <= kMaxLevels; k++) { ig.lr[k] = g.lr[k]; ig.lc[k] = g.lc[k]; }
  int off = 0;
  for (int k = 0; k < g.levels; k++) {
    IncLevel& lv = ig.lv[k];
    lv.R = g.lr[k];
    lv.C = g.lc[k];
    lv.th = fused::level_rows(g, k, nfields);
    lv.ct = (lv.C + fused::TW - 1) / fused::TW;
    lv.rt = (lv.R + lv.th - 1) / lv.th;
    lv.off = off;
    off += lv.ct * lv.rt;
  }
  ig.tiles = (off + 15) & ~15;
  ig.tiles0 = ig.lv[0].ct * ig.lv[0].rt;
  int c = 0;
  for (int k = 1; k < g.levels; k++) {
    inc.coloff[k] = c;
    c += g.lc[k];
  }
  inc.lstride = g.levels > 1 ? (int64_t)g.lr[1] * g.cols : 0;
  return c <= g.cols;
}

// worst-case flag / tile-stat sizes per field: the shortest tiles, which
// fused::level_rows picks for a batch of one chunk
void inc_capacity(const Geo& g, int64_t* tiles, int64_t* tiles0) {
  int64_t t = 0;
  for (int k = 0; k < g.levels; k++) {
    // the shortest tiles of either grid-size regime (level_rows)
    const int th = std::min(fused::level_rows(g, k, 1), fused::level_rows(g, k, fused::kSmallBatch + 1));
    int64_t n = (int64_t)((g.lc[k] + fused::TW - 1) / fused::TW) * ((g.lr[k] + th - 1) / th);
    if (k == 0) *tiles0 = n;
    t += n;
  }
  *tiles = (t + 15) & ~15ll;
}

void base_to_residue(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                     int nfields, const double* norm, double* base_dec, double* resid,
                     cudaStream_t st, bool xe) {
  ResidueEpi e{norm, base_dec, resid, prm, g.n};
  fused::inverse_fused(m, prm, a, b, g, nfields, st, e, false, xe);
}

void decode_field(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                  int nfields, double* out, cudaStream_t st, bool xe, bool midpoint) {
  StoreFieldEpi e{out, prm, g.n};
  fused::inverse_fused(m, prm, a, b, g, nfields, st, e, midpoint, xe);
}

void decode_field_add_denorm(const Meta& m, const ProbeParam* prm, double* a, double* b,
                             const Geo& g, int nfields, const double* base, const FieldScal* fs,
                             float* out32, cudaStream_t st, bool xe) {
  AddDenormEpi e{base, fs, prm, out32, g.n, FieldScal{}};
  fused::inverse_fused(m, prm, a, b, g, nfields, st, e, true, xe);
}

void denorm_only(const double* base, const FieldScal* fs, const uint8_t* active, int64_t n,
                 int nfields, float* out32, cudaStream_t st) {
  denorm_kernel<<<dim3(grid_for(n, 1024), nfields), 256, 0, st>>>(base, fs, active, n, out32);
}

void fill_constant(const FieldScal* fs, const uint8_t* active, int64_t n, int nfields,
                   float* out32, cudaStream_t st) {
  fill_kernel<<<dim3(grid_for(n, 1024), nfields), 256, 0, st>>>(fs, active, n, out32);
}

void pack_parts(const PackPart* parts, int nparts, uint8_t* out, cudaStream_t st) {
  for (int b = 0; b < nparts; b += 65535)
    pack_kernel<<<dim3(64, std::min(65535, nparts - b)), 256, 0, st>>>(parts + b, out);
}

void unpack_parts(const UnpackPart* parts, int nparts, const uint8_t* in, cudaStream_t st) {
  for (int b = 0; b < nparts; b += 65535)
    unpack_kernel<<<dim3(64, std::min(65535, nparts - b)), 256, 0, st>>>(parts + b, in);
}

}  // namespace ebcc
