// Data-parallel SPIHT coder for sm_100a (spiht.py:81-482 restated).
//
// The reference's coder is a list machine: per bit plane a LIP pass, LIS
// "waves" and a refinement pass, each a batch of list operations.  Here:
//
// * exponents replace magnitude compares: |c| >= 2^n  <=>  floor(log2|c|) >= n,
//   and the subtree maxima become integer max over exponents (e_d, e_l);
// * the machine (one CTA per field, 512 threads x 4 entries per tile) walks
//   the lists in order with block-wide scans, emitting significance/sign bits
//   at their exact stream offsets and recording, per coefficient, its LSP rank,
//   significance plane and sign-bit offset;
// * refinement bits are NOT produced by the machine: bit p of coefficient c
//   sits at refine_start[p] + lsp_rank[c], so a separate fully parallel kernel
//   writes (encode) or gathers (decode) them afterwards.
//
// The same machine runs as encoder (significance from exponents) or decoder
// (significance read from the stream at the offset the scan assigns), which is
// how the reference keeps encoder and decoder in lockstep.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "spiht.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace ebcc {

namespace {

#ifndef EBCC_MT
#define EBCC_MT 512
#endif
constexpr int MT = EBCC_MT;      // machine threads
#ifndef EBCC_MACH_CHILD_PREFETCH
#define EBCC_MACH_CHILD_PREFETCH 1  // 296 chunks: compress 134.0 -> 132.9 ms, 37: 23.9 -> 23.55
#endif
#ifndef EBCC_MACH_PRELOAD
#define EBCC_MACH_PRELOAD 1  // 148 chunks: decompress 16.3 -> 16.0 ms, compress the same
#endif
#ifndef EBCC_MI
// 2 entries per thread: the encoder and decoder machines run without register
// spills at 128 registers (4: 204 / 140 bytes of spill stores), same or
// slightly better times (474 chunks: decompress 57.2 -> 56.1 ms)
#define EBCC_MI 2
#endif
constexpr int MI = EBCC_MI;      // entries per thread per tile (16-bit scan lanes: MI*MT*4*4 < 2^16)
constexpr int TILE = MT * MI;    // 1024
constexpr int NW = MT / 32;
constexpr int STAGE_BITS = TILE * 4 + 64;  // children segment can be 4x the tile
constexpr int STAGE_WORDS = STAGE_BITS / 32 + 2;
constexpr uint32_t TYPE_B = 0x80000000u;

// ---------------------------------------------------------------------------
// tree tables
__device__ __forceinline__ uint64_t bitsat(uint64_t v, int at) { return v << at; }

// geometry node info: children count, has-grandchildren, band level/orientation
__global__ void tree_info_kernel(Geo g, uint64_t* ginfo) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  int r = (int)(idx / g.cols), c = (int)(idx - (int64_t)r * g.cols);
  uint32_t ch[4];
  int nc = tree_children(g, r, c, ch);
  int gc = 0;
  for (int s = 0; s < nc; s++) {
    uint32_t cc[4];
    int rr = (int)(ch[s] / g.cols), c2 = (int)(ch[s] - (uint32_t)rr * g.cols);
    gc |= tree_children(g, rr, c2, cc) > 0;
  }
  int level = 0, orient = 0;
  const int L = g.levels;
  if (!(r < g.lr[L] && c < g.lc[L])) {
    for (int kk = L; kk >= 1; kk--)
      if (r < g.lr[kk - 1] && c < g.lc[kk - 1]) { level = kk; break; }
    orient = (r < g.lr[level]) ? 0 : ((c < g.lc[level]) ? 1 : 2);
  }
  // 2x2 child block layout of detail nodes (children c0, c0+1, c0+cols, ...)
  int right = 0, bottom = 0;
  if (level >= 2 && nc > 0) {
    for (int s = 1; s < nc; s++) {
      right |= ch[s] == ch[0] + 1;
      bottom |= ch[s] == ch[0] + (uint32_t)g.cols;
    }
  }
  ginfo[idx] = (uint64_t)(uint32_t)idx | bitsat((uint64_t)nc, ninfo::NCH) |
               bitsat((uint64_t)right, ninfo::RIGHT) | bitsat((uint64_t)bottom, ninfo::BOTTOM) |
               bitsat((uint64_t)gc, ninfo::HASGC) | bitsat((uint64_t)level, ninfo::LEVEL) |
               bitsat((uint64_t)orient, ninfo::ORIENT) | bitsat(63, ninfo::RELC) |
               bitsat(63, ninfo::RELD) | bitsat(63, ninfo::RELL);
}

// children of an entry (spiht.py:108-163) from its level/orientation bits
__device__ __forceinline__ int entry_children(const Geo& g, uint64_t e, uint32_t* ch) {
  const uint32_t node = (uint32_t)e;
  const int r = (int)(node / (uint32_t)g.cols), c = (int)(node - (uint32_t)r * (uint32_t)g.cols);
  const int lev = (int)((e >> ninfo::LEVEL) & 7);
  int m = 0;
  if (lev == 0) {
#pragma unroll
    for (int o = 0; o < 3; o++) {
      Rect R = detail_rect(g, g.levels, o);
      if (R.h > 0 && R.w > 0 && r < R.h && c < R.w)
        ch[m++] = (uint32_t)((R.r0 + r) * g.cols + (R.c0 + c));
    }
    return m;
  }
  if (lev < 2) return 0;
  const int o = (int)((e >> ninfo::ORIENT) & 3);
  Rect P = detail_rect(g, lev, o), C = detail_rect(g, lev - 1, o);
  const int i = r - P.r0, j = c - P.c0;
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      int ci = 2 * i + a, cj = 2 * j + b;
      if (ci < C.h && cj < C.w) ch[m++] = (uint32_t)((C.r0 + ci) * g.cols + (C.c0 + cj));
    }
  return m;
}

// children of a detail node: c0 = 2 * node + K[level][orientation] (the 2x2
// block at (2i, 2j) of the next finer band), compacted like entry_children
__device__ __forceinline__ int entry_children_k(const Geo& g, const int64_t* K, uint64_t e,
                                                uint32_t* ch) {
  const int lev = (int)((e >> ninfo::LEVEL) & 7);
  if (lev == 0) {  // LL root: same position in each coarsest detail band, compacted
    const uint32_t node = (uint32_t)e;
    const int r = (int)(node / (uint32_t)g.cols), c = (int)(node - (uint32_t)r * (uint32_t)g.cols);
    uint32_t cand[3];
    bool ok[3];
#pragma unroll
    for (int o = 0; o < 3; o++) {
      const Rect R = detail_rect(g, g.levels, o);
      ok[o] = R.h > 0 && R.w > 0 && r < R.h && c < R.w;
      cand[o] = (uint32_t)((R.r0 + r) * g.cols + (R.c0 + c));
    }
    ch[0] = ok[0] ? cand[0] : (ok[1] ? cand[1] : cand[2]);
    ch[1] = ok[0] ? (ok[1] ? cand[1] : cand[2]) : cand[2];
    ch[2] = cand[2];
    ch[3] = 0;
    return (int)ok[0] + (int)ok[1] + (int)ok[2];
  }
  const int o = (int)((e >> ninfo::ORIENT) & 3);
  const uint32_t c0 = (uint32_t)(2 * (int64_t)(uint32_t)e + K[lev * 3 + o]);
  const uint32_t R = (uint32_t)((e >> ninfo::RIGHT) & 1), B = (uint32_t)((e >> ninfo::BOTTOM) & 1);
  const uint32_t cols = (uint32_t)g.cols;
  ch[0] = c0;
  ch[1] = R ? c0 + 1 : c0 + cols;
  ch[2] = c0 + cols;
  ch[3] = c0 + cols + 1;
  return (int)(1 + R + B + (R & B));
}

__device__ __forceinline__ int e_rel(uint64_t e, int at) { return (int)((e >> at) & 63); }
__device__ __forceinline__ int e_nch(uint64_t e) { return (int)((e >> ninfo::NCH) & 7); }
__device__ __forceinline__ int e_hasgc(uint64_t e) { return (int)((e >> ninfo::HASGC) & 1); }
__device__ __forceinline__ bool e_isb(uint64_t e) { return (e >> ninfo::TYPEB) & 1; }
__device__ __forceinline__ int e_neg(uint64_t e) { return (int)((e >> ninfo::NEG) & 1); }

// host replica of the children count (for the initial LIS)
int host_nchild(const Geo& g, int r, int c) {
  const int L = g.levels;
  if (r < g.lr[L] && c < g.lc[L]) {
    int m = 0;
    for (int o = 0; o < 3; o++) {
      Rect R = detail_rect(g, L, o);
      if (R.h > 0 && R.w > 0 && r < R.h && c < R.w) m++;
    }
    return m;
  }
  int k = 1;
  for (int kk = L; kk >= 1; kk--)
    if (r < g.lr[kk - 1] && c < g.lc[kk - 1]) { k = kk; break; }
  if (k < 2) return 0;
  int o = (r < g.lr[k]) ? 0 : ((c < g.lc[k]) ? 1 : 2);
  Rect P = detail_rect(g, k, o), C = detail_rect(g, k - 1, o);
  int i = r - P.r0, j = c - P.c0, m = 0;
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2; b++) m += (2 * i + a < C.h && 2 * j + b < C.w);
  return m;
}

// ---------------------------------------------------------------------------
// coefficient preparation: exponents, mantissas, signs, n_max
__global__ void coef_prepare_kernel(const double* __restrict__ coef, int64_t cstride, int64_t n,
                                    int16_t* ec, int16_t* ed, int16_t* el, uint32_t* mant,
                                    uint32_t* sign_pos, uint8_t* pinfo, int64_t stride,
                                    MachineOut* out) {
  const int f = blockIdx.y;
  const double* cf = coef + f * cstride;
  int best = kExpNone;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = cf[i];
    int16_t e = exp_of(v);
    int64_t o = f * stride + i;
    ec[o] = e;
    ed[o] = kExpNone;
    el[o] = kExpNone;
    mant[o] = v == 0.0 ? 0u : mant32_of(v);
    sign_pos[o] = kNone;
    pinfo[o] = v < 0.0 ? 0x80 : 0;
    best = e > best ? e : best;
  }
  for (int o = 16; o; o >>= 1) {
    int y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y > best ? y : best;
  }
  // one atomic per CTA (the warps meet in shared memory)
  __shared__ int s_best[32];
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)((blockDim.x + 31) >> 5); w++) best = s_best[w] > best ? s_best[w] : best;
    atomicMax(&out[f].n_max, best);
  }
}

// e_d / e_l for the parents of one level (spiht.py:182-195 over exponents)
__global__ void subtree_kernel(Geo g, int level, int16_t* ec, int16_t* ed, int16_t* el,
                               int64_t stride, int nfields) {
  // level >= 2: detail nodes of `level`; level == 0: the LL band
  int R, C;
  if (level == 0) { R = g.lr[g.levels]; C = g.lc[g.levels]; }
  else { R = g.lr[level - 1]; C = g.lc[level - 1]; }
  int64_t cnt = (int64_t)R * C;
  int f = blockIdx.y;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < cnt;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(idx / C), c = (int)(idx - (int64_t)r * C);
    if (level != 0 && r < g.lr[level] && c < g.lc[level]) continue;  // inside the coarser box
    uint32_t ch[4];
    int nc = tree_children(g, r, c, ch);
    int dm = kExpNone, lm = kExpNone;
    int64_t fo = (int64_t)f * stride;
    for (int s = 0; s < nc; s++) {
      int a = ec[fo + ch[s]], b = ed[fo + ch[s]];
      int m = a > b ? a : b;
      dm = m > dm ? m : dm;
      lm = b > lm ? b : lm;
    }
    int64_t o = fo + (int64_t)r * g.cols + c;
    ed[o] = (int16_t)dm;
    el[o] = (int16_t)lm;
  }
}

__device__ __forceinline__ uint64_t rel_of(int n_max, int e) {
  int r = n_max - e;
  return (uint64_t)(r < 0 ? 0 : (r > 63 ? 63 : r));
}

// per-field node info = geometry info + relative exponents + sign
__global__ void node_info_kernel(const uint64_t* __restrict__ ginfo, MachineBufs mb, int64_t n) {
  const int f = blockIdx.y;
  const int n_max = mb.out[f].n_max;
  const int64_t fo = (int64_t)f * mb.stride;
  const uint64_t clear = ~(bitsat(63, ninfo::RELC) | bitsat(63, ninfo::RELD) | bitsat(63, ninfo::RELL));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t e = ginfo[i] & clear;
    e |= bitsat(rel_of(n_max, mb.ec[fo + i]), ninfo::RELC);
    e |= bitsat(rel_of(n_max, mb.ed[fo + i]), ninfo::RELD);
    e |= bitsat(rel_of(n_max, mb.el[fo + i]), ninfo::RELL);
    e |= bitsat((uint64_t)(mb.pinfo[fo + i] >> 7), ninfo::NEG);
    mb.ninfo[fo + i] = e;
  }
}

// ---------------------------------------------------------------------------
// block scan of packed 4 x 16-bit counters (per-tile totals stay < 65536)
// One barrier per scan: every warp scans the NW warp totals itself, and
// consecutive scans alternate between two total buffers (`par`), so a fast
// warp's totals of the next scan cannot overwrite what a slow warp still
// reads (it would first have to pass the next scan's barrier).  The machines
// are barrier-bound (7 stall cycles per issue); the scan used to take three.
struct ScanSmem {
  uint64_t warp[2][NW];
};

__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t& total,
                                                         ScanSmem& sm, int& par) {
  static_assert(NW <= 32, "one warp scans the warp totals");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  uint64_t* wb = sm.warp[par];
  par ^= 1;
  if (lane == 31) wb[wid] = x;
  __syncthreads();
  uint64_t w = lane < NW ? wb[lane] : 0;
#pragma unroll
  for (int o = 1; o < NW; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
    if (lane >= o) w += y;
  }
  total = __shfl_sync(0xffffffffu, w, NW - 1);
  const uint64_t before = __shfl_sync(0xffffffffu, w, wid ? wid - 1 : 0);
  return (wid ? before : 0) + x - v;
}

__device__ __forceinline__ uint32_t lane16(uint64_t v, int k) { return (uint32_t)(v >> (16 * k)) & 0xffffu; }

// physical bits of a stream word holding stream positions [a, b) of it
// (MSB-first bytes in a little-endian word, bit_mask_in_word)
__device__ __forceinline__ uint32_t seg_mask(int a, int b) {
  uint32_t m = 0;
#pragma unroll
  for (int B = 0; B < 4; B++) {
    const int ja = min(max(a - 8 * B, 0), 8), jb = min(max(b - 8 * B, 0), 8);
    m |= ((0xffu >> ja) & ~(0xffu >> jb) & 0xffu) << (8 * B);
  }
  return m;
}
#ifndef EBCC_LIP_PREFIX
#define EBCC_LIP_PREFIX 1
#endif

// Cluster-wide exclusive scan: the CTAs of a cluster process consecutive
// sub-tiles of one list, so each thread's prefix is its block prefix plus the
// totals of the lower-ranked CTAs, exchanged through distributed shared
// memory with one cluster barrier (double-buffered slots).
struct ClusterScanOut {
  uint64_t ex;          // this thread's exclusive prefix over the cluster tile
  uint64_t total;       // cluster-tile total
  uint64_t cta_before;  // total of lower-ranked CTAs
  uint64_t cta_total;   // this CTA's total
};

__device__ __forceinline__ ClusterScanOut cluster_scan(uint64_t v, ScanSmem& sm, uint64_t* slots,
                                                       int& parity, const cg::cluster_group& cl,
                                                       int& spar) {
  ClusterScanOut o;
  uint64_t btot;
  uint64_t ex = block_exclusive_scan(v, btot, sm, spar);
  const unsigned n = cl.num_blocks();
  o.cta_total = btot;
  if (n == 1) {
    o.ex = ex; o.total = btot; o.cta_before = 0;
    return o;
  }
  if (threadIdx.x == 0) slots[parity] = btot;
  cl.sync();
  const unsigned rank = cl.block_rank();
  uint64_t before = 0, all = 0;
  for (unsigned r = 0; r < n; r++) {
    uint64_t t = *cl.map_shared_rank(&slots[parity], r);
    if (r < rank) before += t;
    all += t;
  }
  parity ^= 1;
  o.ex = before + ex;
  o.total = all;
  o.cta_before = before;
  return o;
}

// bit staging for one contiguous output segment [seg_start, seg_start + len)
struct Stage {
  uint32_t w[STAGE_WORDS];
};

__device__ __forceinline__ void stage_clear(Stage& s) {
  for (int i = threadIdx.x; i < STAGE_WORDS; i += MT) s.w[i] = 0;
}
__device__ __forceinline__ void stage_set(Stage& s, uint64_t seg_start, uint64_t p) {
  uint64_t w0 = seg_start >> 5;
  atomicOr(&s.w[(p >> 5) - w0], bit_mask_in_word(p));
}
__device__ __forceinline__ void stage_flush(Stage& s, uint64_t seg_start, uint64_t len,
                                            uint32_t* gw) {
  if (!len) return;
  uint64_t w0 = seg_start >> 5, w1 = (seg_start + len - 1) >> 5;
  for (uint64_t i = threadIdx.x; i <= w1 - w0; i += MT) {
    uint32_t v = s.w[i];
    if (!v) continue;
    // interior words belong to this segment alone: plain store
    if (i == 0 || i == w1 - w0) atomicOr(gw + w0 + i, v);
    else gw[w0 + i] = v;
  }
}

// ---------------------------------------------------------------------------
// the machine.  Encoder: significance from the entries' relative exponents;
// decoder: significance read from the stream at the scan-assigned offset.
// MINB = 2: 64 registers (spills) but two CTAs per SM -- for batches of more
// chunks than SMs (no clusters) the doubled warp count hides more of the
// machine's dependent-load latency than the spills cost (296 chunks:
// decompress 37.5 -> 34.6 ms, compress 167.7 -> 166 ms); small batches
// keep the spill-free 128-register machines (37 chunks: 5.4 vs 6.6 ms)
template <bool DECODE, int MINB = 1>
__global__ void __launch_bounds__(MT, MINB) machine_kernel(MachineBufs mb, Geo g, TreeTables tt,
                                                        int planes) {
  cg::cluster_group cl = cg::this_cluster();
  const int csize = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const int f = blockIdx.x / csize;
  if (mb.active && !mb.active[f]) return;  // uniform across the cluster
  if (!DECODE && mb.out[f].n_max == kExpNone) {  // all-zero pyramid: header-only stream
    if (crank == 0 && threadIdx.x == 0) {
      mb.out[f].planes_run = 0;
      mb.out[f].total_bits = 0;
      mb.out[f].overflow = 0;
      mb.out[f].lsp_count = 0;
    }
    return;
  }
  __shared__ ScanSmem ssm;
  __shared__ Stage st_a, st_b, st_c;
  __shared__ uint64_t slots[2];
  // encoder: the LIP passes are deferred to emit_lip; the machine only needs
  // |LIP_p| and the count K_p of LIP entries turning significant at plane p.
  // An entry appended while coding plane q with relc r is in the LIP for
  // planes q+1..r: difference counts over planes, summed across the cluster.
  __shared__ int s_diff[66];
  __shared__ int s_knew[64];
  // encoder: likewise the LIS as a history of kept entries; an entry kept at
  // plane q with significance plane r is an "old" entry for planes q+1..r
  __shared__ int s_ldiff[66];
  __shared__ long long s_bc[3];
  __shared__ int64_t s_K[8 * 3];  // child-block offsets per (level, orientation)
  int parity = 0, spar = 0;
  auto cscan = [&](uint64_t v) { return cluster_scan(v, ssm, slots, parity, cl, spar); };
  auto csync = [&]() {
    if (csize > 1) cl.sync();
    else __syncthreads();
  };

  const int64_t fo = (int64_t)f * mb.stride;
  uint32_t* sign_pos = mb.sign_pos + fo;
  uint32_t* lsp_rank = mb.lsp_rank + fo;
  uint8_t* pinfo = mb.pinfo + fo;
  const uint64_t* info = DECODE ? mb.ginfo : mb.ninfo + fo;
  uint64_t* lip = mb.lip + fo;
  uint64_t* lis_old = mb.lis0 + fo;
  uint64_t* lis_new = mb.lis1 + fo;
  uint64_t* wav_a = mb.w0 + fo;
  uint64_t* wav_b = mb.w1 + fo;
  uint32_t* lsp = mb.lsp + fo;
  uint32_t* sprank = (!DECODE && mb.sprank) ? mb.sprank + fo : nullptr;
  uint32_t* bits = mb.bits + (int64_t)f * mb.bit_stride;
  PlaneRec* prec = mb.planes + (int64_t)f * kMaxPlaneRecs;
  const int n_max = mb.out[f].n_max;
  const uint64_t limit = DECODE ? mb.limit[f] : ~0ull;
  const uint64_t bit_cap = (uint64_t)mb.bit_stride * 32;
  const uint64_t cap = (uint64_t)mb.stride;
  const uint64_t TYPEB = 1ull << ninfo::TYPEB;
  const bool leader = crank == 0 && threadIdx.x == 0;
  const uint64_t CT = (uint64_t)TILE * csize;      // entries per cluster tile
  const uint64_t my0 = (uint64_t)crank * TILE;      // my sub-tile offset

  if (threadIdx.x < 8 * 3) {
    const int lev = threadIdx.x / 3, o = threadIdx.x % 3;
    int64_t k = 0;
    if (lev >= 2 && lev <= g.levels) {
      const Rect P = detail_rect(g, lev, o), C = detail_rect(g, lev - 1, o);
      k = (int64_t)(C.r0 - 2 * P.r0) * g.cols + (C.c0 - 2 * P.c0);
    }
    s_K[threadIdx.x] = k;
  }
  __syncthreads();
  // initial lists (spiht.py:300-303); CTAs split the copy
  if (!DECODE) {
    for (int i = threadIdx.x; i < 66; i += MT) s_diff[i] = 0;
    for (int i = threadIdx.x; i < 66; i += MT) s_ldiff[i] = 0;
    for (int i = threadIdx.x; i < 64; i += MT) s_knew[i] = 0;
    __syncthreads();
    if (leader) {
      s_diff[0] = (int)tt.nroots;
      s_ldiff[0] = (int)tt.nlis_roots;
    }
  }
  for (int64_t i = (int64_t)crank * MT + threadIdx.x; i < tt.nroots; i += (int64_t)MT * csize) {
    const uint64_t e = info[tt.roots[i]];
    lip[i] = e;
    if (!DECODE) {
      const int r = e_rel(e, ninfo::RELC);
      atomicSub(&s_diff[r + 1], 1);
      atomicAdd(&s_knew[r], 1);
    }
  }
  uint8_t* hrel = DECODE ? nullptr : mb.hrel + (int64_t)f * ((mb.stride + 15) & ~15ll);
  for (int64_t i = (int64_t)crank * MT + threadIdx.x; i < tt.nlis_roots; i += (int64_t)MT * csize) {
    const uint64_t e = info[tt.lis_roots[i]];
    lis_old[i] = e;
    if (!DECODE) {
      const int r = e_rel(e, ninfo::RELD);
      hrel[i] = (uint8_t)r;
      atomicSub(&s_ldiff[r + 1], 1);
    }
  }
  uint64_t nlip = tt.nroots, nlis = tt.nlis_roots, nlsp = 0, pos = 0;
  uint64_t hlen = tt.nroots, lip_run = 0;  // encoder: LIP history length, |LIP_p|
  uint64_t hlis = tt.nlis_roots, lis_run = 0;  // encoder: LIS history length, old |LIS_p|
  int overflow = 0;
  int p = 0;
  csync();

#ifdef EBCC_MPROF
  unsigned long long mp_t = clock64(), mp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long mp_waves = 0, mp_tiles = 0, mp_ent = 0, mp_bucket = 0;
#define MPROF_MARK(k)                      \
  {                                        \
    unsigned long long t_ = clock64();     \
    mp_acc[k] += t_ - mp_t;                \
    mp_t = t_;                             \
  }
#else
#define MPROF_MARK(k)
#endif
  for (; p < planes; p++) {
    if (DECODE && pos >= limit) break;  // `while not src.depleted`
    const uint64_t refine_len = nlsp;
    if (leader) prec[p].start = (uint32_t)pos;

    if (!DECODE) {
      // ------------- LIP pass (encoder): counts only -----------------------
      if (threadIdx.x == 0) {
        long long d = 0, kk = 0;
        for (int r = 0; r < csize; r++) {
          d += *cl.map_shared_rank(&s_diff[p], r);
          kk += *cl.map_shared_rank(&s_knew[p], r);
        }
        s_bc[0] = d;
        s_bc[1] = kk;
      }
      __syncthreads();
      lip_run += (uint64_t)s_bc[0];
      const uint64_t K = (uint64_t)s_bc[1];
      if (leader) prec[p].lip_len = (uint32_t)lip_run;
      pos += lip_run + K;
      nlsp += K;
      nlip -= K;
    }
    // ---------------- LIP pass (decoder) ---------------------------------
    // The LIP's significance bits are one contiguous segment [pos, pos+nlip)
    // (bits past `limit` read as 0).  An entry's rank among the significant
    // ones is the number of set segment bits before its own: a per-word
    // prefix (one cluster scan over the segment's words) plus a popcount in
    // its word.  Survivors are compacted out of place (into the wave buffer,
    // which then becomes the LIP); no per-tile cluster barrier.
    if (DECODE && EBCC_LIP_PREFIX) {
      uint64_t K = 0;
      if (nlip) {
        const uint64_t seg0 = pos, seg1 = min(pos + nlip, limit);
        const uint64_t w0 = seg0 >> 5;
        const uint64_t nw = seg1 > seg0 ? ((seg1 - 1) >> 5) - w0 + 1 : 0;
        uint64_t* P = wav_b;  // exclusive prefix of set segment bits per word
        auto segcount = [&](uint64_t w) -> uint32_t {
          const uint64_t wb = (w0 + w) << 5;
          const int a = seg0 > wb ? (int)(seg0 - wb) : 0;
          const int b = seg1 < wb + 32 ? (int)(seg1 - wb) : 32;
          return __popc(__ldg(bits + w0 + w) & seg_mask(a, b));
        };
        const uint64_t per = (nw + csize - 1) / csize;
        const uint64_t wlo = min(nw, (uint64_t)crank * per), whi = min(nw, wlo + per);
        const uint64_t tper = (whi - wlo + MT - 1) / MT;
        const uint64_t tlo = min(whi, wlo + (uint64_t)threadIdx.x * tper);
        const uint64_t thi = min(whi, tlo + tper);
        uint64_t local = 0;
        for (uint64_t w = tlo; w < thi; w++) local += segcount(w);
        const ClusterScanOut cs = cscan(local);
        K = cs.total;
        uint64_t run = cs.ex;
        for (uint64_t w = tlo; w < thi; w++) {
          P[w] = run;
          run += segcount(w);
        }
        csync();  // every CTA's prefixes visible
        for (uint64_t i = (uint64_t)crank * MT + threadIdx.x; i < nlip; i += (uint64_t)MT * csize) {
          const uint64_t e = lip[i];
          const uint64_t q = pos + i;
          bool sig = false;
          uint64_t S = K;  // entries past `limit`: every set bit lies before them
          if (q < seg1) {
            const uint64_t wa = q >> 5;
            const uint32_t word = __ldg(bits + wa);
            const uint64_t wb = wa << 5;
            const int a = seg0 > wb ? (int)(seg0 - wb) : 0;
            S = P[wa - w0] + __popc(word & seg_mask(a, (int)(q - wb)));
            sig = (word & bit_mask_in_word(q)) != 0;
          }
          if (sig) {
            const uint64_t rank = nlsp + S, sp = pos + nlip + S;
            const uint32_t c = (uint32_t)e;
            lsp[rank] = c;
            lsp_rank[c] = (uint32_t)rank;
            if (sp < limit) {
              sign_pos[c] = (uint32_t)sp;
              pinfo[c] = (uint8_t)(p | (read_bit(bits, sp, limit) << 7));
            } else {
              pinfo[c] = (uint8_t)p;
            }
          } else {
            wav_a[i - S] = e;
          }
        }
      }
      pos += nlip + K;
      nlsp += K;
      nlip -= K;
      { uint64_t* t = lip; lip = wav_a; wav_a = t; }
      csync();  // compacted LIP visible cluster-wide before the LIS appends
    } else if (DECODE) {
      uint64_t K = 0;  // newly significant so far
      for (uint64_t base = 0; base < nlip; base += CT) {
        uint64_t ent[MI];
        int sig[MI];
        int cnt_sig = 0;
        const uint64_t i0 = base + my0 + (uint64_t)threadIdx.x * MI;
#pragma unroll
        for (int k = 0; k < MI; k++) {
          uint64_t i = i0 + k;
          sig[k] = 0;
          ent[k] = 0;
          if (i < nlip) {
            ent[k] = lip[i];
            sig[k] = DECODE ? read_bit(bits, pos + i, limit) : (e_rel(ent[k], ninfo::RELC) <= p);
            cnt_sig += sig[k];
          }
        }
        const ClusterScanOut cs = cscan((uint64_t)cnt_sig);
        const uint64_t ex = cs.ex, tot = cs.total;
        const uint64_t sub0 = base + my0;
        const uint64_t my_len = nlip > sub0 ? ((nlip - sub0) < TILE ? (nlip - sub0) : TILE) : 0;
        if (!DECODE) {
          stage_clear(st_a);
          stage_clear(st_b);
          __syncthreads();
          uint64_t sig_seg = pos + sub0, sgn_seg = pos + nlip + K + cs.cta_before;
          uint64_t r = ex;
#pragma unroll
          for (int k = 0; k < MI; k++) {
            if (!sig[k]) continue;
            stage_set(st_a, sig_seg, pos + i0 + k);
            if (e_neg(ent[k])) stage_set(st_b, sgn_seg, pos + nlip + K + r);
            r++;
          }
          __syncthreads();
          stage_flush(st_a, sig_seg, my_len, bits);
          stage_flush(st_b, sgn_seg, cs.cta_total, bits);
        }
        // newly significant -> LSP, metadata; survivors compacted in place
        // (every CTA of the cluster loaded its entries before the scan's barrier)
        uint64_t r = ex;
        uint64_t keep_before = (i0 - base) - ex;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MI; k++) {
          uint64_t i = i0 + k;
          if (i >= nlip) break;
          if (sig[k]) {
            uint64_t rank = nlsp + K + r;
            uint64_t sp = pos + nlip + K + r;
            uint32_t c = (uint32_t)ent[k];
            lsp[rank] = c;
            lsp_rank[c] = (uint32_t)rank;
            if (DECODE) {
              if (sp < limit) {
                sign_pos[c] = (uint32_t)sp;
                pinfo[c] = (uint8_t)(p | (read_bit(bits, sp, limit) << 7));
              } else {
                pinfo[c] = (uint8_t)p;
              }
            } else {
              sign_pos[c] = (uint32_t)sp;
              pinfo[c] = (uint8_t)((e_neg(ent[k]) << 7) | p);
              if (sprank) sprank[rank] = (uint32_t)sp;
            }
            r++;
          } else {
            lip[base - K + keep_before] = ent[k];
            keep_before++;
          }
        }
        K += tot;
        __syncthreads();
      }
      pos += nlip + K;
      nlsp += K;
      nlip -= K;
      csync();  // compaction visible cluster-wide before the LIS appends / next pass
    }

    MPROF_MARK(0);
    // ---------------- LIS waves ------------------------------------------
    {
      uint64_t nkeep = 0;
      const uint64_t* src = lis_old;
      uint64_t* dst = wav_a;
      uint64_t cnt = nlis;
      // encoder: the old entries' wave codes only those turning significant
      // now (relevant plane == p), gathered from the history in order; their
      // significance bits (and the old entries' zeros) are left to emit_lis
      bool w0 = false;
      uint64_t nbucket = 0;
      if (!DECODE) {
        if (threadIdx.x == 0) {
          long long d = 0;
          for (int r = 0; r < csize; r++) d += *cl.map_shared_rank(&s_ldiff[p], r);
          s_bc[2] = d;
        }
        __syncthreads();
        lis_run += (uint64_t)s_bc[2];
        if (leader) prec[p].lis_start = (uint32_t)pos;
        // each CTA scans a contiguous share of the history bytes
        const uint64_t per = ((hlis + csize - 1) / csize + 15) & ~15ull;
        const uint64_t lo = min(hlis, (uint64_t)crank * per), hi = min(hlis, lo + per);
        uint64_t* tmp = mb.lis1 + fo + lo;
        const uint32_t pp4 = 0x01010101u * (uint32_t)p;
        uint64_t n = 0;
        for (uint64_t base = lo; base < hi; base += (uint64_t)MT * 16) {
          const uint64_t i0 = base + (uint64_t)threadIdx.x * 16;
          uint32_t m = 0;
          if (i0 + 16 <= hi) {
            const uint4 v = *reinterpret_cast<const uint4*>(hrel + i0);
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const uint32_t x = __vcmpeq4(w4[q], pp4);
              m |= (((x >> 7) & 1u) | ((x >> 14) & 2u) | ((x >> 21) & 4u) | ((x >> 28) & 8u))
                   << (4 * q);
            }
          } else {
            for (int k = 0; k < 16; k++)
              if (i0 + k < hi && hrel[i0 + k] == (uint8_t)p) m |= 1u << k;
          }
          uint64_t tot;
          uint64_t o = n + block_exclusive_scan((uint64_t)__popc(m), tot, ssm, spar);
          while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            tmp[o] = lis_old[i0 + k];
            o++;
          }
          n += tot;
        }
        // concatenate the CTAs' matches into the wave list
        if (threadIdx.x == 0) slots[parity] = n;
        csync();
        uint64_t before = 0, all = 0;
        for (int r = 0; r < csize; r++) {
          const uint64_t t = csize > 1 ? *cl.map_shared_rank(&slots[parity], r) : slots[parity];
          if (r < crank) before += t;
          all += t;
        }
        parity ^= 1;
        for (uint64_t k = threadIdx.x; k < n; k += MT) wav_a[before + k] = tmp[k];
        csync();
        nbucket = all;
        src = wav_a;
        dst = wav_b;
        cnt = all;
        w0 = true;
      }
      MPROF_MARK(1);
#ifdef EBCC_MPROF
      mp_bucket += nbucket;
#endif
      const uint64_t hbase = hlis;
      while (cnt || w0) {
#ifdef EBCC_MPROF
        mp_waves++;
        mp_ent += cnt;
        mp_tiles += (cnt + CT - 1) / CT;
#endif
        // prepass: total children bits of significant type-A entries (the
        // sign bits follow all of the wave's children bits).  A wave of one
        // cluster tile gets it from the main pass's first scan instead.
        uint64_t TC = 0;
        const bool single = cnt <= CT;
        for (uint64_t base = 0; !single && base < cnt; base += CT) {
          uint64_t local = 0;
          const uint64_t i0 = base + my0 + (uint64_t)threadIdx.x * MI;
#pragma unroll
          for (int k = 0; k < MI; k++) {
            uint64_t i = i0 + k;
            if (i >= cnt) break;
            uint64_t e = src[i];
            if (e_isb(e)) continue;
            int s = DECODE ? read_bit(bits, pos + i, limit) : (e_rel(e, ninfo::RELD) <= p);
            if (s) local += e_nch(e);
          }
          TC += cscan(local).total;
        }
        MPROF_MARK(w0 ? 2 : 3);
        const uint64_t segw = w0 ? lis_run : cnt;  // entry significance bits
        const uint64_t ch_seg0 = pos + segw;       // children significance bits
        uint64_t sg_seg0 = pos + segw + TC;        // their sign bits (single: after scan 1)
        uint64_t ch_off = 0, sig_off = 0, nxt_off = 0;
#if EBCC_MACH_PRELOAD
        // the next tile's entries are loaded a tile ahead: their latency (the
        // head of each tile's dependent chain entry -> children -> node info
        // -> scan) hides behind the current tile's gathers and scans
        uint64_t pre[MI];
#pragma unroll
        for (int k = 0; k < MI; k++) {
          const uint64_t i = my0 + (uint64_t)threadIdx.x * MI + k;
          pre[k] = i < cnt ? src[i] : 0;
        }
#endif
        for (uint64_t base = 0; base < cnt; base += CT) {
          uint64_t ent[MI];
          int sig[MI], nch[MI], nxt[MI];
          uint32_t keep = 0, nchs = 0, nxts = 0;
          const uint64_t i0 = base + my0 + (uint64_t)threadIdx.x * MI;
#if EBCC_MACH_PRELOAD
          uint64_t cur[MI];
#pragma unroll
          for (int k = 0; k < MI; k++) {
            cur[k] = pre[k];
            const uint64_t i = i0 + CT + k;
            pre[k] = i < cnt ? src[i] : 0;
          }
#endif
#pragma unroll
          for (int k = 0; k < MI; k++) {
            uint64_t i = i0 + k;
            sig[k] = 0; nch[k] = 0; nxt[k] = 0; ent[k] = 0;
            if (i >= cnt) continue;
#if EBCC_MACH_PRELOAD
            uint64_t e = cur[k];
#else
            uint64_t e = src[i];
#endif
            ent[k] = e;
            bool isb = e_isb(e);
            sig[k] = DECODE ? read_bit(bits, pos + i, limit)
                            : (e_rel(e, isb ? ninfo::RELL : ninfo::RELD) <= p);
            if (!sig[k]) { keep++; continue; }
            if (!isb) {
              nch[k] = e_nch(e);
              nxt[k] = e_hasgc(e);
            } else {
              nxt[k] = -1;  // resolved below from the children's info
            }
            nchs += nch[k];
          }
          // children of significant entries (A: coded; B: next-wave sets)
          uint32_t chn[MI][4];
          uint64_t cin[MI][4];
          int nchild[MI];
#pragma unroll
          for (int k = 0; k < MI; k++) {
            nchild[k] = 0;
            if (!sig[k] || (!nch[k] && nxt[k] >= 0)) continue;
            const int m = entry_children_k(g, s_K, ent[k], chn[k]);
            nchild[k] = m;
#pragma unroll
            for (int s = 0; s < 4; s++)
              if (s < m) cin[k][s] = info[chn[k][s]];
            if (nxt[k] < 0) {
              int q = 0;
#pragma unroll
              for (int s = 0; s < 4; s++)
                if (s < m) q += e_nch(cin[k][s]) != 0;
              nxt[k] = q;
              nch[k] = 0;
            }
          }
#pragma unroll
          for (int k = 0; k < MI; k++) nxts += nxt[k] > 0 ? nxt[k] : 0;
          // children significance: the encoder knows it now (one scan for all
          // four counts); the decoder reads it at the offsets the first scan gives
          uint8_t chs[MI];  // bitmask of significant children
          uint32_t nsig = 0;
          if (!DECODE) {
#pragma unroll
            for (int k = 0; k < MI; k++) {
              chs[k] = 0;
#pragma unroll
              for (int s = 0; s < 4; s++) {
                if (s >= nch[k]) break;
                const int cs = e_rel(cin[k][s], ninfo::RELC) <= p;
                chs[k] |= (uint8_t)(cs << s);
                nsig += cs;
              }
            }
          }
          const ClusterScanOut s1 = cscan((uint64_t)keep | ((uint64_t)nchs << 16) |
                                          ((uint64_t)nxts << 32) |
                                          (DECODE ? 0ull : ((uint64_t)nsig << 48)));
          const uint64_t ex1 = s1.ex, tot1 = s1.total;
#if EBCC_MACH_PRELOAD && EBCC_MACH_CHILD_PREFETCH
          // encoder: the node info of the next tile's children on its way to
          // L2 (the preloaded entries have arrived behind the scan's barrier;
          // the per-field info array is not L2-resident, the decoder's shared
          // geometry table is)
          if (!DECODE) {
#pragma unroll
            for (int k = 0; k < MI; k++) {
              const uint64_t e = pre[k];
              const int lev = (int)((e >> ninfo::LEVEL) & 7);
              if (e && lev > 0 && e_rel(e, e_isb(e) ? ninfo::RELL : ninfo::RELD) <= p) {
                const int o = (int)((e >> ninfo::ORIENT) & 3);
                const uint32_t c0 = (uint32_t)(2 * (int64_t)(uint32_t)e + s_K[lev * 3 + o]);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(info + c0));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(info + c0 + (uint32_t)g.cols));
              }
            }
          }
#endif
          if (single) {
            TC = lane16(tot1, 1);
            sg_seg0 = pos + segw + TC;
          }
          uint64_t ex2, tot2, s2_before, s2_total;
          if (DECODE) {
            uint64_t cpos = ch_seg0 + ch_off + lane16(ex1, 1);
#pragma unroll
            for (int k = 0; k < MI; k++) {
              chs[k] = 0;
#pragma unroll
              for (int s = 0; s < 4; s++) {
                if (s >= nch[k]) break;
                const int cs = read_bit(bits, cpos, limit);
                chs[k] |= (uint8_t)(cs << s);
                nsig += cs;
                cpos++;
              }
            }
            const ClusterScanOut s2 = cscan((uint64_t)nsig);
            ex2 = s2.ex;
            tot2 = s2.total;
            s2_before = s2.cta_before;
            s2_total = s2.cta_total;
          } else {
            ex2 = lane16(ex1, 3);
            tot2 = lane16(tot1, 3);
            s2_before = lane16(s1.cta_before, 3);
            s2_total = lane16(s1.cta_total, 3);
          }
          const uint64_t sub0 = base + my0;
          const uint64_t my_len = cnt > sub0 ? ((cnt - sub0) < TILE ? (cnt - sub0) : TILE) : 0;
          if (!DECODE) {
            stage_clear(st_a);
            stage_clear(st_b);
            stage_clear(st_c);
            __syncthreads();
            uint64_t seg_a = pos + sub0;
            uint64_t seg_b = ch_seg0 + ch_off + lane16(s1.cta_before, 1);
            uint64_t seg_c = sg_seg0 + sig_off + s2_before;
            uint64_t cpos = ch_seg0 + ch_off + lane16(ex1, 1);
            uint64_t spos = sg_seg0 + sig_off + ex2;
#pragma unroll
            for (int k = 0; k < MI; k++) {
              if (sig[k] && !w0) stage_set(st_a, seg_a, pos + i0 + k);
#pragma unroll
              for (int s = 0; s < 4; s++) {
                if (s >= nch[k]) break;
                if ((chs[k] >> s) & 1) {
                  stage_set(st_b, seg_b, cpos);
                  if (e_neg(cin[k][s])) stage_set(st_c, seg_c, spos);
                  spos++;
                }
                cpos++;
              }
            }
            __syncthreads();
            if (!w0) stage_flush(st_a, seg_a, my_len, bits);
            stage_flush(st_b, seg_b, lane16(s1.cta_total, 1), bits);
            stage_flush(st_c, seg_c, s2_total, bits);
          }
          // list updates
          {
            uint64_t kp = nkeep + lane16(ex1, 0);
            uint64_t nx = nxt_off + lane16(ex1, 2);
            uint64_t sg = sig_off + ex2;                       // rank among sig children
            uint64_t ins = (ch_off + lane16(ex1, 1)) - sg;     // rank among insig children
#pragma unroll
            for (int k = 0; k < MI; k++) {
              uint64_t i = i0 + k;
              if (i >= cnt) break;
              uint64_t e = ent[k];
              if (!sig[k]) {
                if (DECODE) {
                  if (kp < cap) lis_new[kp] = e; else overflow = 1;
                } else {  // kept: appended to the LIS history
                  const uint64_t hi = hbase + kp;
                  const int r = e_rel(e, e_isb(e) ? ninfo::RELL : ninfo::RELD);
                  if (hi < cap) {
                    lis_old[hi] = e;
                    hrel[hi] = (uint8_t)r;
                  } else {
                    overflow = 1;
                  }
                  atomicSub(&s_ldiff[r + 1], 1);
                }
                kp++;
                continue;
              }
#pragma unroll
              for (int s = 0; s < 4; s++) {
                if (s >= nch[k]) break;
                uint32_t c = chn[k][s];
                if ((chs[k] >> s) & 1) {
                  uint64_t rank = nlsp + sg;
                  uint64_t sp = sg_seg0 + sg;
                  lsp[rank] = c;
                  lsp_rank[c] = (uint32_t)rank;
                  if (DECODE) {
                    if (sp < limit) {
                      sign_pos[c] = (uint32_t)sp;
                      pinfo[c] = (uint8_t)(p | (read_bit(bits, sp, limit) << 7));
                    } else {
                      pinfo[c] = (uint8_t)p;
                    }
                  } else {
                    sign_pos[c] = (uint32_t)sp;
                    pinfo[c] = (uint8_t)((e_neg(cin[k][s]) << 7) | p);
                    if (sprank) sprank[rank] = (uint32_t)sp;
                  }
                  sg++;
                } else {
                  uint64_t li = (DECODE ? nlip : hlen) + ins;
                  if (li < cap) lip[li] = cin[k][s]; else overflow = 1;
                  if (!DECODE) {
                    const int r = e_rel(cin[k][s], ninfo::RELC);
                    atomicSub(&s_diff[r + 1], 1);
                    atomicAdd(&s_knew[r], 1);
                  }
                  ins++;
                }
              }
              if (nxt[k] > 0) {
                if (!e_isb(e)) {
                  if (nx < cap) dst[nx] = e | TYPEB; else overflow = 1;
                  nx++;
                } else {
#pragma unroll
                  for (int s = 0; s < 4; s++)
                    if (s < nchild[k] && e_nch(cin[k][s])) {
                      if (nx < cap) dst[nx] = cin[k][s]; else overflow = 1;
                      nx++;
                    }
                }
              }
            }
          }
          nkeep += lane16(tot1, 0);
          ch_off += lane16(tot1, 1);
          nxt_off += lane16(tot1, 2);
          sig_off += tot2;
          __syncthreads();
        }
        pos += segw + TC + sig_off;
        nlsp += sig_off;
        nlip += TC - sig_off;
        if (!DECODE) {
          hlen += TC - sig_off;
          if (leader) s_diff[p + 1] += (int)(TC - sig_off);
        }
        cnt = nxt_off;
        MPROF_MARK(w0 ? 4 : 5);
        src = dst;
        dst = (dst == wav_a) ? wav_b : wav_a;
        w0 = false;
        csync();  // the next wave reads entries every CTA wrote
      }
      if (DECODE) {
        nlis = nkeep;
        uint64_t* t = lis_old; lis_old = lis_new; lis_new = t;
      } else {
        nlis = lis_run - nbucket + nkeep;
        hlis += nkeep;
        if (leader) s_ldiff[p + 1] += (int)nkeep;
      }
    }

    MPROF_MARK(6);
    // ---------------- refinement (positions only) ------------------------
    if (leader) {
      prec[p].refine_start = (uint32_t)pos;
      prec[p].refine_len = (uint32_t)refine_len;
    }
    pos += refine_len;
    if (leader) prec[p].lists_end = (uint32_t)(nlip + nlis + nlsp);
    if (!DECODE && pos > bit_cap) { overflow = 1; }
    if (pos > 0xffffffffull) overflow = 1;
    overflow = __syncthreads_or(overflow);
    if (csize > 1) overflow = cscan((uint64_t)(overflow && threadIdx.x == 0)).total != 0;
    if (overflow) { p++; break; }
  }
  if (leader) {
    mb.out[f].planes_run = p;
    mb.out[f].total_bits = (uint32_t)(pos > 0xffffffffull ? 0xffffffffull : pos);
    mb.out[f].overflow = overflow;
    mb.out[f].lsp_count = (uint32_t)nlsp;
    mb.out[f].hist_len = (uint32_t)hlen;
    mb.out[f].lis_hist_len = (uint32_t)hlis;
#ifdef EBCC_MPROF
    if (f == 0)
      printf("[mprof %s] planes %d lip %.0f bucket %.0f w0pre %.0f wpre %.0f w0main %.0f wmain %.0f "
             "tail %.0f kcyc | waves %llu tiles %llu entries %llu bucket %llu hlis %llu hlen %llu\n",
             DECODE ? "dec" : "enc", p, mp_acc[0] / 1e3, mp_acc[1] / 1e3, mp_acc[2] / 1e3,
             mp_acc[3] / 1e3, mp_acc[4] / 1e3, mp_acc[5] / 1e3, mp_acc[6] / 1e3, mp_waves,
             mp_tiles, mp_ent, mp_bucket, (unsigned long long)hlis, (unsigned long long)hlen);
#endif
  }
  // no CTA may exit while a peer can still read its shared memory (the last
  // cluster scan reads every CTA's slots through DSMEM)
  if (csize > 1) cl.sync();
}

// encoder refinement, word aligned.  Refinement bit of plane p for rank i
// sits at refine_start[p] + i for every plane after the coefficient's
// significance plane (that plane being < p is exactly i < refine_len[p]).
// A warp walks a contiguous run of 32-rank groups: each lane aligns its
// mantissa so bit 31-p is its plane-p bit, a 32x32 bit transpose (5 shuffle
// stages) hands lane p the plane-p ballot of the group, and output word w of
// plane p's segment (ranks 32w - o .. 32w - o + 31, o = refine_start[p] & 31)
// is a funnel shift of this group's and the previous group's masks.  Lane p
// stores plane p's word; only a segment's two edge words (shared with its
// neighbours) need an atomic.
__global__ void refine_write_kernel(MachineBufs mb, int planes) {
  const int f = blockIdx.y;
  if (mb.active && !mb.active[f]) return;
  const int64_t fo = (int64_t)f * mb.stride;
  const PlaneRec* prec = mb.planes + (int64_t)f * kMaxPlaneRecs;
  const int pr = mb.out[f].planes_run < planes ? mb.out[f].planes_run : planes;
  if (pr < 2) return;
  uint32_t* bits = mb.bits + (int64_t)f * mb.bit_stride;
  const int lane = threadIdx.x & 31;
  const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t maxlen = prec[pr - 1].refine_len;  // non-decreasing in p
  const uint32_t nw = maxlen / 32 + 2;
  const uint32_t run = (nw + nwarps - 1) / nwarps;
  const uint32_t wb = warp_global * run, we = min(nw, wb + run);
  if (wb >= we) return;
  for (int p0 = 0; p0 < pr; p0 += 32) {  // lane q <-> plane p0 + q
    const int pl = p0 + lane;
    const bool pon = pl >= 1 && pl < pr;
    const uint32_t rs = pon ? prec[pl].refine_start : 0u;
    const uint32_t rl = pon ? prec[pl].refine_len : 0u;
    const int o = (int)(rs & 31u);
    const uint32_t last = rl ? (uint32_t)(((uint64_t)rs + rl - 1) >> 5) : 0xffffffffu;
    auto group = [&](uint32_t g) -> uint32_t {
      const uint32_t i = g * 32 + lane;
      uint32_t a = 0;
      if (i < maxlen) {
        const uint32_t c = mb.lsp[fo + i];
        const uint32_t m = mb.mant[fo + c];
        const int d = p0 - (mb.pinfo[fo + c] & 0x3f);
        // bit 31-q of a = plane (p0+q) bit = m bit 31-(p0+q-ps), for p0+q > ps
        if (d <= 0) a = -d < 31 ? (m >> -d) & ((1u << (31 + d)) - 1u) : 0u;
        else a = d < 32 ? m << d : 0u;
      }
      uint32_t x = __brev(a);  // bit q <-> plane p0 + q
      // 32x32 transpose: lane q ends with bit l = lane l's bit q
#pragma unroll
      for (int j = 16; j >= 1; j >>= 1) {
        const uint32_t lo = j == 16 ? 0x0000ffffu : j == 8 ? 0x00ff00ffu : j == 4 ? 0x0f0f0f0fu
                          : j == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~lo) | ((y & ~lo) >> j)) : ((x & lo) | ((y & lo) << j));
      }
      return x;
    };
    uint32_t prev = wb > 0 ? group(wb - 1) : 0u;
    for (uint32_t w = wb; w < we; w++) {
      const uint32_t cur = group(w);
      // lane-order mask of output word w: bit q <-> rank 32w - o + q
      const uint32_t lm = o ? __funnelshift_l(prev, cur, o) : cur;
      prev = cur;
      if (pon && lm) {
        const uint32_t v = __byte_perm(__brev(lm), 0, 0x0123);
        const uint32_t wd = (rs >> 5) + w;
        if (w == 0 || wd == last) atomicOr(bits + wd, v);
        else bits[wd] = v;
      }
    }
  }
}

// decoder refinement gather: thread per LSP rank; bits past the stream
// limit read as zero exactly like _BitSource.take
__global__ void refine_gather_kernel(MachineBufs mb) {
  const int f = blockIdx.y;
  if (mb.active && !mb.active[f]) return;
  const int64_t fo = (int64_t)f * mb.stride;
  const PlaneRec* prec = mb.planes + (int64_t)f * kMaxPlaneRecs;
  const int pr = mb.out[f].planes_run;
  const uint32_t nlsp = mb.out[f].lsp_count;
  const uint64_t limit = mb.limit[f];
  const uint32_t* bits = mb.bits + (int64_t)f * mb.bit_stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)nlsp;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = mb.lsp[fo + i];
    if (mb.sign_pos[fo + c] == kNone) continue;  // sign never read: not placed
    int ps = mb.pinfo[fo + c] & 0x3f;
    uint32_t m = 0x80000000u;
    for (int p = ps + 1; p < pr && p - ps <= 31; p++) {
      if ((uint32_t)i >= prec[p].refine_len) break;
      uint64_t q = (uint64_t)prec[p].refine_start + (uint64_t)i;
      if (q >= limit) break;
      m |= (uint32_t)read_bit(bits, q, limit) << (31 - (p - ps));
    }
    mb.mant[fo + c] = m;
  }
}

// decompress: the refinement gather writes the probe records itself (probe.cuh:
// x = LSP rank | significance plane << 26, y = sign << 31 | significand bits)
// and the sign offsets by rank, instead of a significand array that
// pack_meta would re-read with the other per-coefficient arrays.  Records of
// coefficients whose sign was never read keep decode_init's all-ones
// ("never placed").  Narrow records only (ranks below 2^26 - 1).
__global__ void refine_gather_pack_kernel(MachineBufs mb, uint2* __restrict__ packed,
                                          uint32_t* __restrict__ sprank) {
  const int f = blockIdx.y;
  if (mb.active && !mb.active[f]) return;
  const int64_t fo = (int64_t)f * mb.stride;
  const PlaneRec* prec = mb.planes + (int64_t)f * kMaxPlaneRecs;
  const int pr = mb.out[f].planes_run;
  const uint32_t nlsp = mb.out[f].lsp_count;
  const uint64_t limit = mb.limit[f];
  const uint32_t* bits = mb.bits + (int64_t)f * mb.bit_stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)nlsp;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = mb.lsp[fo + i];
    const uint32_t sp = mb.sign_pos[fo + c];
    sprank[fo + i] = sp;  // kNone: sign never read (ranks >= lsp_count are never looked at)
    if (sp == kNone) continue;
    const uint32_t pi = mb.pinfo[fo + c];
    const int ps = pi & 0x3f;
    uint32_t m = 0;
    for (int p = ps + 1; p < pr && p - ps <= 31; p++) {
      if ((uint32_t)i >= prec[p].refine_len) break;
      uint64_t q = (uint64_t)prec[p].refine_start + (uint64_t)i;
      if (q >= limit) break;
      m |= (uint32_t)read_bit(bits, q, limit) << (31 - (p - ps));
    }
    packed[fo + c] = make_uint2(((uint32_t)i & 0x3ffffffu) | ((uint32_t)ps << 26),
                                ((pi & 0x80u) << 24) | m);
  }
}

// ---------------------------------------------------------------------------
// Deferred encoder LIP passes.  The LIP before plane p's pass is the LIP
// history H (roots, then every insignificant child in append order) filtered
// by relc >= p: entries leave the LIP at their significance plane and are
// appended in plane order (an entry appended while coding plane q has
// relc > q).  So entry i with relc r < planes_run has
//   significance bit at  start[r] + #{j < i : relc_j >= r}
//   sign bit at          start[r] + lip_len[r] + #{j < i : relc_j == r}
//   LSP rank             refine_len[r] + #{j < i : relc_j == r}
// (spiht.py's LIP pass, every plane at once): two rank-by-value counts over
// 64 relc buckets, from tile histograms, per-warp histograms and a bit-sliced
// in-warp compare.
constexpr int ET = 1024;        // emit threads per CTA
constexpr int EPT = 4;          // entries per thread
constexpr int ETILE = ET * EPT; // LIP-history entries per tile
constexpr int EVW = ETILE / 32; // 32-entry groups ("virtual warps") per tile

__device__ __forceinline__ bool emit_skip(const MachineBufs& mb, int f) {
  return (mb.active && !mb.active[f]) || mb.out[f].overflow;
}

// LIP history (relevant plane: relc) or LIS history (reld for type A, rell
// for type B entries)
template <bool LIS>
__device__ __forceinline__ uint32_t hist_len_of(const MachineBufs& mb, int f) {
  const uint32_t h = LIS ? mb.out[f].lis_hist_len : mb.out[f].hist_len;
  return (int64_t)h < mb.stride ? h : (uint32_t)mb.stride;
}
template <bool LIS>
__device__ __forceinline__ const uint64_t* hist_of(const MachineBufs& mb, int f) {
  return (LIS ? mb.lis0 : mb.lip) + (int64_t)f * mb.stride;
}
template <bool LIS>
__device__ __forceinline__ int hist_rel(uint64_t e) {
  return LIS ? e_rel(e, e_isb(e) ? ninfo::RELL : ninfo::RELD) : e_rel(e, ninfo::RELC);
}

// entry k of thread tid in a tile: sub-tile k, 32-entry group k*32 + warp
__device__ __forceinline__ int64_t emit_index(int64_t t0, int k) {
  return t0 + (int64_t)k * ET + threadIdx.x;
}

template <bool LIS>
__global__ void __launch_bounds__(ET) lip_hist_kernel(MachineBufs mb, uint32_t* hist, int tiles) {
  const int f = blockIdx.y;
  if (emit_skip(mb, f)) return;
  const uint32_t hlen = hist_len_of<LIS>(mb, f);
  const int64_t t0 = (int64_t)blockIdx.x * ETILE;
  if (t0 >= hlen) return;
  __shared__ uint32_t h[64];
  if (threadIdx.x < 64) h[threadIdx.x] = 0;
  const uint64_t* lip = hist_of<LIS>(mb, f);
  int bk[EPT];
#pragma unroll
  for (int k = 0; k < EPT; k++) {
    const int64_t i = emit_index(t0, k);
    bk[k] = i < hlen ? hist_rel<LIS>(lip[i]) : 64;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < EPT; k++) {
    const unsigned m = __match_any_sync(0xffffffffu, bk[k]);
    if (bk[k] < 64 && (int)(threadIdx.x & 31) == __ffs(m) - 1)
      atomicAdd(&h[bk[k]], (uint32_t)__popc(m));
  }
  __syncthreads();
  if (threadIdx.x < 64) hist[((int64_t)f * tiles + blockIdx.x) * 64 + threadIdx.x] = h[threadIdx.x];
}

// exclusive scan of the tile histograms over tiles, per bucket (in place)
template <bool LIS>
__global__ void __launch_bounds__(1024) lip_scan_kernel(MachineBufs mb, uint32_t* hist, int tiles) {
  const int f = blockIdx.x;
  if (emit_skip(mb, f)) return;
  const int ntiles = (int)((hist_len_of<LIS>(mb, f) + ETILE - 1) / ETILE);
  const int v = threadIdx.x & 63, sg = threadIdx.x >> 6;  // 16 segments of tiles
  const int per = (ntiles + 15) / 16;
  const int tb = sg * per, te = min(ntiles, tb + per);
  uint32_t* hf = hist + (int64_t)f * tiles * 64;
  uint32_t sum = 0;
  for (int t = tb; t < te; t++) sum += hf[(int64_t)t * 64 + v];
  __shared__ uint32_t seg[16][64];
  seg[sg][v] = sum;
  __syncthreads();
  uint32_t acc = 0;
  for (int q = 0; q < sg; q++) acc += seg[q][v];
  for (int t = tb; t < te; t++) {
    const uint32_t x = hf[(int64_t)t * 64 + v];
    hf[(int64_t)t * 64 + v] = acc;
    acc += x;
  }
}

template <bool LIS>
#ifndef EBCC_EMIT_MINB
#define EBCC_EMIT_MINB 2  // 32 registers, two 1024-thread CTAs per SM (148 fields: compress -0.7 ms)
#endif
__global__ void __launch_bounds__(ET, EBCC_EMIT_MINB) lip_emit_kernel(MachineBufs mb, const uint32_t* hist,
                                                      int tiles) {
  const int f = blockIdx.y;
  if (emit_skip(mb, f)) return;
  const uint32_t hlen = hist_len_of<LIS>(mb, f);
  const int64_t t0 = (int64_t)blockIdx.x * ETILE;
  if (t0 >= hlen) return;
  const int pr = mb.out[f].planes_run;
  const int64_t fo = (int64_t)f * mb.stride;
  __shared__ uint32_t wh[64][EVW + 1];  // [bucket][32-entry group], padded
  __shared__ uint32_t s_start[kMaxPlaneRecs], s_lip[kMaxPlaneRecs], s_ref[kMaxPlaneRecs];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < 64 * (EVW + 1); k += ET) (&wh[0][0])[k] = 0;
  if (tid < kMaxPlaneRecs) {
    const PlaneRec& R = mb.planes[(int64_t)f * kMaxPlaneRecs + tid];
    s_start[tid] = LIS ? R.lis_start : R.start;
    s_lip[tid] = R.lip_len;
    s_ref[tid] = R.refine_len;
  }
  uint64_t ent[EPT];
  int bk[EPT];
  unsigned mk[EPT];
#pragma unroll
  for (int k = 0; k < EPT; k++) {
    const int64_t i = emit_index(t0, k);
    ent[k] = i < hlen ? hist_of<LIS>(mb, f)[i] : 0;
  }
#pragma unroll
  for (int k = 0; k < EPT; k++) {
    const int64_t i = emit_index(t0, k);
    bk[k] = i < hlen ? hist_rel<LIS>(ent[k]) : 64;
    mk[k] = __match_any_sync(0xffffffffu, bk[k]);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < EPT; k++)
    if (bk[k] < 64 && lane == __ffs(mk[k]) - 1) wh[bk[k]][k * 32 + warp] = (uint32_t)__popc(mk[k]);
  __syncthreads();
  {  // exclusive over the groups (lane l owns groups EPT*l ..), on top of earlier tiles
    const uint32_t* tp = hist + ((int64_t)f * tiles + blockIdx.x) * 64;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int v = warp + 32 * h;
      uint32_t x[EPT], loc = 0;
#pragma unroll
      for (int j = 0; j < EPT; j++) { x[j] = wh[v][EPT * lane + j]; loc += x[j]; }
      uint32_t y = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
      }
      uint32_t run = tp[v] + y - loc;
#pragma unroll
      for (int j = 0; j < EPT; j++) { wh[v][EPT * lane + j] = run; run += x[j]; }
    }
  }
  __syncthreads();
  uint32_t* bits = mb.bits + (int64_t)f * mb.bit_stride;
  const uint64_t bit_cap = (uint64_t)mb.bit_stride * 32;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < EPT; k++) {
    const int b = bk[k];
    if (__all_sync(0xffffffffu, b >= pr)) continue;
    // bucket counts before this group, and their suffix sums (relc >= v)
    const int gi = k * 32 + warp;
    const uint32_t clo = wh[lane][gi], chi = wh[lane + 32][gi];
    uint32_t slo = clo, shi = chi;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yl = __shfl_down_sync(0xffffffffu, slo, o);
      const uint32_t yh = __shfl_down_sync(0xffffffffu, shi, o);
      if (lane + o < 32) { slo += yl; shi += yh; }
    }
    slo += __shfl_sync(0xffffffffu, shi, 0);
    const int src = b & 31;
    const uint32_t s_l = __shfl_sync(0xffffffffu, slo, src), s_h = __shfl_sync(0xffffffffu, shi, src);
    const uint32_t c_l = __shfl_sync(0xffffffffu, clo, src), c_h = __shfl_sync(0xffffffffu, chi, src);
    // in-group: lanes below me with relc == b / relc >= b (bit-sliced compare)
    unsigned eqm = 0xffffffffu, gtm = 0u;
#pragma unroll
    for (int q = 6; q >= 0; q--) {
      const unsigned B = __ballot_sync(0xffffffffu, (b >> q) & 1);
      if ((b >> q) & 1) {
        eqm &= B;
      } else {
        gtm |= eqm & B;
        eqm &= ~B;
      }
    }
    const bool on = b < pr;  // significant within the planes run (padding: b = 64)
    const uint64_t ge = (uint64_t)(b < 32 ? s_l : s_h) + (uint32_t)__popc((gtm | eqm) & lt);
    const uint64_t eq = (uint64_t)(b < 32 ? c_l : c_h) + (uint32_t)__popc(mk[k] & lt);
    const int neg = e_neg(ent[k]);
    const uint64_t sig = on ? (uint64_t)s_start[b] + ge : ~0ull;
    const uint64_t sp = on ? (uint64_t)s_start[b] + s_lip[b] + eq : ~0ull;
    // one atomic per distinct word per group
    {
      const uint32_t wd = on ? (uint32_t)(sig >> 5) : 0xffffffffu;
      const unsigned g = __match_any_sync(0xffffffffu, wd);
      const uint32_t v = __reduce_or_sync(g, on ? bit_mask_in_word(sig) : 0u);
      if (on && lane == __ffs(g) - 1 && sig < bit_cap) atomicOr(bits + wd, v);
    }
    if (LIS) continue;  // old LIS entries: significance bit only
    {
      const bool sn = on && neg;
      const uint32_t wd = sn ? (uint32_t)(sp >> 5) : 0xffffffffu;
      const unsigned g = __match_any_sync(0xffffffffu, wd);
      const uint32_t v = __reduce_or_sync(g, sn ? bit_mask_in_word(sp) : 0u);
      if (sn && lane == __ffs(g) - 1 && sp < bit_cap) atomicOr(bits + wd, v);
    }
    if (on) {
      const uint32_t c = (uint32_t)ent[k];
      const uint32_t rank = s_ref[b] + (uint32_t)eq;
      mb.lsp[fo + rank] = c;
      if (mb.sprank) mb.sprank[fo + rank] = (uint32_t)sp;
      mb.lsp_rank[fo + c] = rank;
      mb.sign_pos[fo + c] = (uint32_t)sp;
      mb.pinfo[fo + c] = (uint8_t)((neg << 7) | b);
    }
  }
}

void emit_lip_host(MachineBufs& mb, cudaStream_t st) {
  const int tiles = (int)((mb.stride + ETILE - 1) / ETILE);
  // the wave buffers are free once the machine is done: tile histograms
  uint32_t* hist = reinterpret_cast<uint32_t*>(mb.w0);
  lip_hist_kernel<false><<<dim3(tiles, mb.nfields), ET, 0, st>>>(mb, hist, tiles);
  lip_scan_kernel<false><<<mb.nfields, 1024, 0, st>>>(mb, hist, tiles);
  lip_emit_kernel<false><<<dim3(tiles, mb.nfields), ET, 0, st>>>(mb, hist, tiles);
  uint32_t* hist2 = reinterpret_cast<uint32_t*>(mb.w1);
  lip_hist_kernel<true><<<dim3(tiles, mb.nfields), ET, 0, st>>>(mb, hist2, tiles);
  lip_scan_kernel<true><<<mb.nfields, 1024, 0, st>>>(mb, hist2, tiles);
  lip_emit_kernel<true><<<dim3(tiles, mb.nfields), ET, 0, st>>>(mb, hist2, tiles);
}

// decoder init: nothing placed yet
// packed != null (gather_pack follows): the records start out "never placed"
// (all ones) and the significands are never materialised
__global__ void decode_init_kernel(MachineBufs mb, uint2* packed) {
  const int f = blockIdx.y;
  const int64_t fo = (int64_t)f * mb.stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < mb.stride;
       i += (int64_t)gridDim.x * blockDim.x) {
    mb.sign_pos[fo + i] = kNone;
    mb.pinfo[fo + i] = 0;
    if (packed) packed[fo + i] = make_uint2(0xffffffffu, 0xffffffffu);
    else mb.mant[fo + i] = 0;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
void build_tree_tables(const Geo& g, TreeTables& t, cudaStream_t st) {
  cudaMalloc(&t.ginfo, sizeof(uint64_t) * g.n);
  tree_info_kernel<<<(unsigned)((g.n + 255) / 256), 256, 0, st>>>(g, t.ginfo);
  // roots: LL row-major, then orphans per level L-1..1 and orientation (spiht.py:164-178)
  std::vector<uint32_t> roots, lis;
  int llr = g.lr[g.levels], llc = g.lc[g.levels];
  for (int i = 0; i < llr; i++)
    for (int j = 0; j < llc; j++) roots.push_back((uint32_t)(i * g.cols + j));
  for (int k = g.levels - 1; k >= 1; k--)
    for (int o = 0; o < 3; o++) {
      Rect C = detail_rect(g, k, o), P = detail_rect(g, k + 1, o);
      if (C.h <= 0 || C.w <= 0) continue;
      for (int i = 0; i < C.h; i++)
        for (int j = 0; j < C.w; j++)
          if (i / 2 >= P.h || j / 2 >= P.w) roots.push_back((uint32_t)((C.r0 + i) * g.cols + C.c0 + j));
    }
  for (uint32_t r : roots) {
    int rr = (int)(r / g.cols), cc = (int)(r % g.cols);
    if (host_nchild(g, rr, cc) > 0) lis.push_back(r);
  }
  t.nroots = (int64_t)roots.size();
  t.nlis_roots = (int64_t)lis.size();
  cudaMalloc(&t.roots, sizeof(uint32_t) * (roots.size() + 1));
  cudaMalloc(&t.lis_roots, sizeof(uint32_t) * (lis.size() + 1));
  cudaMemcpyAsync(t.roots, roots.data(), sizeof(uint32_t) * roots.size(), cudaMemcpyHostToDevice, st);
  if (!lis.empty())
    cudaMemcpyAsync(t.lis_roots, lis.data(), sizeof(uint32_t) * lis.size(), cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
}

void free_tree_tables(TreeTables& t) {
  cudaFree(t.ginfo); cudaFree(t.roots); cudaFree(t.lis_roots);
  t = TreeTables{};
}

void coef_prepare(const double* coef, int64_t field_stride, MachineBufs& mb, const Geo& g,
                  cudaStream_t st) {
  int blocks = (int)((g.n + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  dim3 grid(blocks, mb.nfields);
  coef_prepare_kernel<<<grid, 256, 0, st>>>(coef, field_stride, g.n, mb.ec, mb.ed, mb.el, mb.mant,
                                            mb.sign_pos, mb.pinfo, mb.stride, mb.out);
}

void subtree_exponents(MachineBufs& mb, const Geo& g, const TreeTables& tt, cudaStream_t st) {
  for (int k = 2; k <= g.levels; k++) {
    int64_t cnt = (int64_t)g.lr[k - 1] * g.lc[k - 1];
    int blocks = (int)((cnt + 255) / 256);
    if (blocks > 1024) blocks = 1024;
    subtree_kernel<<<dim3(blocks, mb.nfields), 256, 0, st>>>(g, k, mb.ec, mb.ed, mb.el, mb.stride,
                                                             mb.nfields);
  }
  int64_t cnt = (int64_t)g.lr[g.levels] * g.lc[g.levels];
  int blocks = (int)((cnt + 255) / 256);
  subtree_kernel<<<dim3(blocks, mb.nfields), 256, 0, st>>>(g, 0, mb.ec, mb.ed, mb.el, mb.stride,
                                                           mb.nfields);
  node_info_kernel<<<dim3((unsigned)std::min<int64_t>((g.n + 255) / 256, 2048), mb.nfields), 256, 0,
                     st>>>(tt.ginfo, mb, g.n);
}

// CTAs per field: the machine's time is per-entry work, so more CTAs per
// field help as long as every field's cluster is resident at once (clusters
// live inside one GPC, so e.g. 37 fields x 4 CTAs do not all fit on 148 SMs).
// the largest cluster (<= kMaxCluster CTAs) for which every chunk's cluster
// is resident at once: few large chunks get up to 7 CTAs each (the packed
// 16-bit scan lanes hold a cluster tile's children count, <= 4*TILE*size)
#ifndef EBCC_MAX_CLUSTER
// 15 CTAs (non-portable cluster size; 2 entries per thread leave the 16-bit
// scan lanes room): few chunks get more SMs per list machine (1 chunk:
// compress 5.8 -> 5.3 ms, decompress 1.6 -> 1.2 ms; 2 x 2881x5760: compress
// 50.3 -> 37.8 ms)
#define EBCC_MAX_CLUSTER 15
#endif
constexpr int kMaxCluster = EBCC_MAX_CLUSTER;
static_assert(4 * TILE * kMaxCluster < 65536, "16-bit scan lanes");
// clusters above 8 CTAs are non-portable: opt the machines in once
void allow_large_clusters() {
  static std::once_flag once;
  std::call_once(once, [] {
    if (kMaxCluster > 8) {
      cudaFuncSetAttribute(machine_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(machine_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaGetLastError();
    }
  });
}
int machine_cluster_size(bool decode, int nfields) {
  allow_large_clusters();
  if (const char* e = getenv("EBCC_MACHINE_CLUSTER")) {
    const int c = atoi(e);
    return c < 1 ? 1 : (c > kMaxCluster ? kMaxCluster : c);
  }
  static std::mutex mu;
  static std::unordered_map<int64_t, int> memo;
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t key = ((int64_t)dev << 40) | ((int64_t)decode << 32) | (uint32_t)nfields;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  int best = 1;
  for (int c = kMaxCluster; c >= 2; c--) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nfields * c), 1, 1);
    cfg.blockDim = dim3(MT, 1, 1);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t err = decode ? cudaOccupancyMaxActiveClusters(&n, machine_kernel<true>, &cfg)
                             : cudaOccupancyMaxActiveClusters(&n, machine_kernel<false>, &cfg);
    if (err != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (n >= nfields) {
      best = c;
      break;
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  memo[key] = best;
  return best;
}

void run_machine(bool decode, MachineBufs& mb, const Geo& g, const TreeTables& tt, int planes,
                 cudaStream_t st, int cluster) {
  allow_large_clusters();
  const int cs = cluster > 0 ? cluster : machine_cluster_size(decode, mb.nfields);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(mb.nfields * cs), 1, 1);
  cfg.blockDim = dim3(MT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const bool two_env = !(getenv("EBCC_MACH_TWO") && getenv("EBCC_MACH_TWO")[0] == '0');
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const bool two = two_env && cs == 1 && mb.nfields > sms;
  if (decode) {
    if (two) cudaLaunchKernelEx(&cfg, machine_kernel<true, 2>, mb, g, tt, planes);
    else cudaLaunchKernelEx(&cfg, machine_kernel<true>, mb, g, tt, planes);
  } else {
    if (two) cudaLaunchKernelEx(&cfg, machine_kernel<false, 2>, mb, g, tt, planes);
    else cudaLaunchKernelEx(&cfg, machine_kernel<false>, mb, g, tt, planes);
  }
}

void emit_lip(MachineBufs& mb, int planes, cudaStream_t st) {
  (void)planes;
  emit_lip_host(mb, st);
}

void write_refinement(MachineBufs& mb, int planes, cudaStream_t st) {
  int blocks = (int)((mb.stride / 32 + 7) / 8);
  if (blocks > 512) blocks = 512;
  if (blocks < 1) blocks = 1;
  refine_write_kernel<<<dim3(blocks, mb.nfields), 256, 0, st>>>(mb, planes);
}

void decode_init(MachineBufs& mb, cudaStream_t st, uint2* packed) {
  int blocks = (int)((mb.stride + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  decode_init_kernel<<<dim3(blocks, mb.nfields), 256, 0, st>>>(mb, packed);
}

void gather_pack(MachineBufs& mb, uint2* packed, uint32_t* sprank, cudaStream_t st) {
  int blocks = (int)((mb.stride + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  refine_gather_pack_kernel<<<dim3(blocks, mb.nfields), 256, 0, st>>>(mb, packed, sprank);
}

void gather_refinement(MachineBufs& mb, cudaStream_t st) {
  int blocks = (int)((mb.stride + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  refine_gather_kernel<<<dim3(blocks, mb.nfields), 256, 0, st>>>(mb);
}

}  // namespace ebcc
