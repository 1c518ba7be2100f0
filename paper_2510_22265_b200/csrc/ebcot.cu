// Opt-in JPEG2000-style base layer on the GPU (see ebcot.cuh for the codec
// and the stream layout; the CPU restatement is oracle/ebcot_oracle.c).
#include <algorithm>
#include <cstdio>
#include <vector>

#include "ebcot.cuh"

namespace ebcc {
namespace {

// ---- MQ coder (ITU-T T.800 Table C.2, Annex C) -----------------------------
__constant__ uint16_t kQe[47] = {
    0x5601, 0x3401, 0x1801, 0x0AC1, 0x0521, 0x0221, 0x5601, 0x5401, 0x4801, 0x3801,
    0x3001, 0x2401, 0x1C01, 0x1601, 0x5601, 0x5401, 0x5101, 0x4801, 0x3801, 0x3401,
    0x3001, 0x2801, 0x2401, 0x2201, 0x1C01, 0x1801, 0x1601, 0x1401, 0x1201, 0x1101,
    0x0AC1, 0x09C1, 0x08A1, 0x0521, 0x0441, 0x02A1, 0x0221, 0x0141, 0x0111, 0x0085,
    0x0049, 0x0025, 0x0015, 0x0009, 0x0005, 0x0001, 0x5601};
__constant__ uint8_t kNmps[47] = {1,  2,  3,  4,  5,  38, 7,  8,  9,  10, 11, 12, 13, 29, 15, 16,
                                  17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32,
                                  33, 34, 35, 36, 37, 38, 39, 40, 41, 42, 43, 44, 45, 45, 46};
__constant__ uint8_t kNlps[47] = {1,  6,  9,  12, 29, 33, 6,  14, 14, 14, 17, 18, 20, 21, 14, 14,
                                  15, 16, 17, 18, 19, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29,
                                  30, 31, 32, 33, 34, 35, 36, 37, 38, 39, 40, 41, 42, 43, 46};
// SWITCH is set only for states 0, 6 and 14
__device__ __forceinline__ bool mq_switch(int i) { return i == 0 || i == 6 || i == 14; }

constexpr int kCtx = 19, kCtxRL = 17, kCtxUni = 18;

struct Ctxs {
  uint8_t I[kCtx], mps[kCtx];
  __device__ void reset() {
    for (int i = 0; i < kCtx; i++) { I[i] = 0; mps[i] = 0; }
    I[0] = 4;
    I[kCtxRL] = 3;
    I[kCtxUni] = 46;
  }
};

struct MqEnc {
  uint32_t A, C;
  int CT, B;
  int64_t bp, cap;
  uint8_t* out;
  bool over;
  __device__ void init(uint8_t* o, int64_t c) {
    A = 0x8000; C = 0; CT = 12; B = 0; bp = -1; out = o; cap = c; over = false;
  }
  __device__ void put(int nb) {
    if (bp >= 0) {
      if (bp < cap) out[bp] = (uint8_t)B;
      else over = true;
    }
    bp++;
    B = nb;
  }
  __device__ void byteout() {
    if (B == 0xFF) {
      put((int)(C >> 20));
      C &= 0xFFFFF;
      CT = 7;
    } else if (C < 0x8000000) {
      put((int)(C >> 19));
      C &= 0x7FFFF;
      CT = 8;
    } else {
      B++;
      if (B == 0xFF) {
        C &= 0x7FFFFFF;
        put((int)(C >> 20));
        C &= 0xFFFFF;
        CT = 7;
      } else {
        put((int)(C >> 19));
        C &= 0x7FFFF;
        CT = 8;
      }
    }
  }
  __device__ void renorm() {
    do {
      A <<= 1;
      C <<= 1;
      CT--;
      if (CT == 0) byteout();
    } while ((A & 0x8000) == 0);
  }
  __device__ void code(Ctxs& s, int cx, int d) {
    const int st = s.I[cx];
    const uint32_t qe = kQe[st];
    A -= qe;
    if (d == s.mps[cx]) {
      if ((A & 0x8000) == 0) {
        if (A < qe) A = qe;
        else C += qe;
        s.I[cx] = kNmps[st];
        renorm();
      } else {
        C += qe;
      }
    } else {
      if (A < qe) C += qe;
      else A = qe;
      if (mq_switch(st)) s.mps[cx] ^= 1;
      s.I[cx] = kNlps[st];
      renorm();
    }
  }
  // returns the codeword length (a trailing 0xFF dropped)
  __device__ int64_t flush() {
    const uint32_t t = C + A;
    C |= 0xFFFF;
    if (C >= t) C -= 0x8000;
    C <<= CT;
    byteout();
    C <<= CT;
    byteout();
    if (bp >= 0) {
      if (bp < cap) out[bp] = (uint8_t)B;
      else over = true;
    }
    int64_t len = bp + 1;
    if (len > 0 && len <= cap && out[len - 1] == 0xFF) len--;
    return len;
  }
};

struct MqDec {
  uint32_t A, C;
  int CT;
  const uint8_t* d;
  int64_t n, bp;
  __device__ int byte(int64_t i) const { return i < n ? d[i] : 0xFF; }
  __device__ void bytein() {
    if (byte(bp) == 0xFF) {
      const int b1 = byte(bp + 1);
      if (b1 > 0x8F) {
        C += 0xFF00;
        CT = 8;
      } else {
        bp++;
        C += (uint32_t)b1 << 9;
        CT = 7;
      }
    } else {
      bp++;
      C += (uint32_t)byte(bp) << 8;
      CT = 8;
    }
  }
  __device__ void init(const uint8_t* data, int64_t len) {
    d = data; n = len; bp = 0;
    C = (uint32_t)byte(0) << 16;
    bytein();
    C <<= 7;
    CT -= 7;
    A = 0x8000;
  }
  __device__ void renorm() {
    do {
      if (CT == 0) bytein();
      A <<= 1;
      C <<= 1;
      CT--;
    } while ((A & 0x8000) == 0);
  }
  __device__ int decode(Ctxs& s, int cx) {
    const int st = s.I[cx];
    const uint32_t qe = kQe[st];
    int dd;
    A -= qe;
    if ((C >> 16) < qe) {  // LPS sub-interval: LPS exchange
      if (A < qe) {
        A = qe;
        dd = s.mps[cx];
        s.I[cx] = kNmps[st];
      } else {
        A = qe;
        dd = 1 - s.mps[cx];
        if (mq_switch(st)) s.mps[cx] ^= 1;
        s.I[cx] = kNlps[st];
      }
      renorm();
    } else {
      C -= qe << 16;
      if ((A & 0x8000) == 0) {  // MPS exchange
        if (A < qe) {
          dd = 1 - s.mps[cx];
          if (mq_switch(st)) s.mps[cx] ^= 1;
          s.I[cx] = kNlps[st];
        } else {
          dd = s.mps[cx];
          s.I[cx] = kNmps[st];
        }
        renorm();
      } else {
        dd = s.mps[cx];
      }
    }
    return dd;
  }
};

// ---- tier-1 contexts (T.800 Tables D.1, D.3, D.4) ---------------------------
// Per-sample state word: own flags in bits 0..3, the significance of the 8
// neighbours in bits 4..11 and the signs of the 4 edge neighbours in bits
// 12..15, kept up to date when a sample turns significant (one load per
// visit instead of nine; neighbours outside the code-block never count).
constexpr uint16_t F_SIG = 1, F_VIS = 2, F_REF = 4, F_NEG = 8;
constexpr int NB_W = 4, NB_E = 5, NB_N = 6, NB_S = 7, NB_NW = 8, NB_NE = 9, NB_SW = 10, NB_SE = 11;
constexpr uint16_t NSIG_MASK = 0x0FF0;

__device__ __forceinline__ int sig_ctx(int orient, int h, int v, int d) {
  if (orient == 1) { const int t = h; h = v; v = t; }
  if (orient == 2) {
    const int hv = h + v;
    if (d >= 3) return 8;
    if (d == 2) return hv >= 1 ? 7 : 6;
    if (d == 1) return hv >= 2 ? 5 : (hv == 1 ? 4 : 3);
    return hv >= 2 ? 2 : (hv == 1 ? 1 : 0);
  }
  if (h == 2) return 8;
  if (h == 1) return v >= 1 ? 7 : (d >= 1 ? 6 : 5);
  if (v == 2) return 4;
  if (v == 1) return 3;
  return d >= 2 ? 2 : (d == 1 ? 1 : 0);
}

// one code-block's view of the per-sample state: words stripe-major (the 4
// samples of a stripe column are one 8-byte word group); q / plow stay in
// the pyramid layout (base, cols)
struct Blk {
  uint16_t* f;     // the block's state words
  int64_t base;    // pyramid position of the block's (0, 0)
  int cols, h, w, orient;
  __device__ __forceinline__ int64_t idx(int y, int x) const {
    return ((int64_t)(y >> 2) * w + x) * 4 + (y & 3);
  }
  __device__ __forceinline__ uint16_t& ref(int y, int x) const { return f[idx(y, x)]; }
  __device__ __forceinline__ int word(int y, int x) const { return ref(y, x); }
  // the 4 words of stripe column (y0, x) (y0 a multiple of 4)
  __device__ __forceinline__ uint2 column(int y0, int x) const {
    return *reinterpret_cast<const uint2*>(f + idx(y0, x));
  }
  __device__ __forceinline__ int sig_context(int wd) const {
    const int hh = ((wd >> NB_W) & 1) + ((wd >> NB_E) & 1);
    const int vv = ((wd >> NB_N) & 1) + ((wd >> NB_S) & 1);
    const int dd = __popc((wd >> NB_NW) & 15);
    return sig_ctx(orient, hh, vv, dd);
  }
  __device__ __forceinline__ int sign_ctx(int wd, int& xr) const {
    auto contrib = [&](int sa, int sb) {
      int s = 0;
      if ((wd >> sa) & 1) s += ((wd >> (sa + 8)) & 1) ? -1 : 1;
      if ((wd >> sb) & 1) s += ((wd >> (sb + 8)) & 1) ? -1 : 1;
      return s > 0 ? 1 : (s < 0 ? -1 : 0);
    };
    const int hc = contrib(NB_W, NB_E), vc = contrib(NB_N, NB_S);
    int cx;
    xr = 0;
    if (hc == 1) cx = vc == 1 ? 13 : (vc == 0 ? 12 : 11);
    else if (hc == 0) { cx = vc == 0 ? 9 : 10; xr = vc == -1; }
    else { cx = vc == 1 ? 11 : (vc == 0 ? 12 : 13); xr = 1; }
    return cx;
  }
  __device__ __forceinline__ int mr_ctx(int wd) const {
    if (wd & F_REF) return 16;
    return (wd & NSIG_MASK) ? 15 : 14;
  }
  // (y, x) turns significant with sign neg: its own bit and its neighbours'
  __device__ __forceinline__ void set_sig(int y, int x, int neg) const {
    ref(y, x) |= F_SIG | (neg ? F_NEG : 0);
    auto nb = [&](int yy, int xx, int bit, bool edge) {
      if (yy < 0 || xx < 0 || yy >= h || xx >= w) return;
      uint16_t add = (uint16_t)(1u << bit);
      if (edge && neg) add |= (uint16_t)(1u << (bit + 8));
      ref(yy, xx) |= add;
    };
    nb(y, x - 1, NB_E, true);
    nb(y, x + 1, NB_W, true);
    nb(y - 1, x, NB_S, true);
    nb(y + 1, x, NB_N, true);
    nb(y - 1, x - 1, NB_SE, false);
    nb(y - 1, x + 1, NB_SW, false);
    nb(y + 1, x - 1, NB_NE, false);
    nb(y + 1, x + 1, NB_NW, false);
  }
};

// the symbol coder of one pass: encoder (lazily started codeword) or decoder
template <bool ENC>
struct PassCoder {
  MqEnc* e;
  MqDec* d;
  Ctxs* s;
  int64_t nsym;
  bool started;
  uint8_t* seg;
  int64_t segcap;
  const uint8_t* in;
  int64_t inlen;
  __device__ int code(int cx, int bit) {
    nsym++;
    if constexpr (ENC) {
      if (!started) { e->init(seg, segcap); started = true; }
      e->code(*s, cx, bit);
      return bit;
    } else {
      if (!started) { d->init(in, inlen); started = true; }
      return d->decode(*s, cx);
    }
  }
};

// One coding pass over a block (ptype 0 SP, 1 MR, 2 CU) at plane p.
// Encoder: q[] holds magnitude | sp << 30 | neg << 31 and gets the sp bit of
// samples turning significant; decoder: q[] accumulates the decoded bits and
// plow[] the lowest decoded plane.
template <bool ENC>
__device__ void run_pass(const Blk& b, uint32_t* q, int8_t* plow, int p, int ptype,
                         PassCoder<ENC>& c) {
  auto qi = [&](int y, int x) -> uint32_t& { return q[b.base + (int64_t)y * b.cols + x]; };
  auto pl = [&](int y, int x) -> int8_t& { return plow[b.base + (int64_t)y * b.cols + x]; };
  for (int y0 = 0; y0 < b.h; y0 += 4) {
    const int sh = b.h - y0 < 4 ? b.h - y0 : 4;
    for (int x = 0; x < b.w; x++) {
      {  // nothing to code in this stripe column: skip it with one load
        const uint2 cw = b.column(y0, x);
        const uint32_t wds[4] = {cw.x & 0xFFFFu, cw.x >> 16, cw.y & 0xFFFFu, cw.y >> 16};
        bool work = false;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          if (k >= sh) break;
          const uint32_t wd = wds[k];
          if (ptype == 0) work |= !(wd & F_SIG) && (wd & NSIG_MASK);
          else if (ptype == 1) work |= (wd & F_SIG) && !(wd & F_VIS);
          else work |= !(wd & (F_SIG | F_VIS));
        }
        if (!work) continue;
      }
      int y = y0;
      if (ptype == 2 && sh == 4) {  // cleanup run mode
        bool run_ok = true;
        for (int k = 0; k < 4 && run_ok; k++)
          if (b.word(y0 + k, x) & (F_SIG | F_VIS | NSIG_MASK)) run_ok = false;
        if (run_ok) {
          int first = 4;
          if (ENC)
            for (int k = 0; k < 4; k++)
              if ((qi(y0 + k, x) >> p) & 1) { first = k; break; }
          if (!c.code(kCtxRL, first < 4)) continue;
          if (ENC) {
            c.code(kCtxUni, (first >> 1) & 1);
            c.code(kCtxUni, first & 1);
          } else {
            first = c.code(kCtxUni, 0) << 1;
            first |= c.code(kCtxUni, 0);
          }
          const int yy = y0 + first;
          int xr;
          const int wd = b.word(yy, x);
          const int scx = b.sign_ctx(wd, xr);
          const int neg = ENC ? (int)(qi(yy, x) >> 31) : 0;
          const int sb = c.code(scx, neg ^ xr) ^ xr;
          if (!ENC) {
            qi(yy, x) |= 1u << p;
            pl(yy, x) = (int8_t)p;
          }
          b.set_sig(yy, x, sb);  // (cleanup significance: the sp bit stays 0)
          y = yy + 1;
        }
      }
      for (; y < y0 + sh; y++) {
        const int wd = b.word(y, x);
        if (ptype == 1) {  // magnitude refinement: significant before this plane
          if (!(wd & F_SIG) || (wd & F_VIS)) continue;
          const int cx = b.mr_ctx(wd);
          const int bit = c.code(cx, ENC ? (int)((qi(y, x) >> p) & 1) : 0);
          if (!ENC) {
            qi(y, x) |= (uint32_t)bit << p;
            pl(y, x) = (int8_t)p;
          }
          b.ref(y, x) |= F_REF;
          continue;
        }
        if (wd & F_SIG) continue;
        if (ptype == 0) {
          if (!(wd & NSIG_MASK)) continue;
          b.ref(y, x) |= F_VIS;
        } else if (wd & F_VIS) {
          continue;
        }
        const int cx = b.sig_context(wd);
        const int bit = c.code(cx, ENC ? (int)((qi(y, x) >> p) & 1) : 0);
        if (bit) {
          int xr;
          const int scx = b.sign_ctx(wd, xr);
          const int neg = ENC ? (int)(qi(y, x) >> 31) : 0;
          const int sb = c.code(scx, neg ^ xr) ^ xr;
          if (ENC) {
            if (ptype == 0) qi(y, x) |= 1u << 30;  // significant in a SP pass
          } else {
            qi(y, x) |= 1u << p;
            pl(y, x) = (int8_t)p;
          }
          b.set_sig(y, x, sb);
        }
      }
    }
  }
}

__device__ __forceinline__ void pass_of(int pt, int j, int& p, int& ptype) {
  if (j == 0) { p = pt; ptype = 2; return; }
  p = pt - 1 - (j - 1) / 3;
  ptype = (j - 1) % 3;
}
__device__ __forceinline__ int gidx(int p, int ptype) { return 3 * (kJ2Planes - 1 - p) + ptype; }
// pass index of block with top plane pt at global pass index g (-1: none)
__device__ __forceinline__ int pass_at(int pt, int g) {
  if (pt < 0) return -1;
  const int gt = gidx(pt, 2);
  if (g == gt) return 0;
  if (pt >= 1 && g >= gt + 1) return 1 + (g - (gt + 1));
  return -1;
}

__device__ __forceinline__ int leb_len(uint32_t v) {
  int n = 1;
  while (v >= 0x80) { v >>= 7; n++; }
  return n;
}

// ---- kernels -----------------------------------------------------------------
__global__ void nmax_kernel(const double* __restrict__ coef, int64_t n, int32_t* nmax,
                            const uint8_t* active) {
  const int f = blockIdx.y;
  if (active && !active[f]) return;
  int best = kExpNone;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = exp_of(coef[(int64_t)f * n + i]);
    best = e > best ? e : best;
  }
  for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(nmax + f, best);
}

__global__ void quantize_kernel(const double* __restrict__ coef, int64_t n, const int32_t* nmax,
                                uint32_t* qs, const uint8_t* active) {
  const int f = blockIdx.y;
  if (active && !active[f]) return;
  const int nm = nmax[f];
  const int e0 = nm - (kJ2Planes - 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double c = coef[(int64_t)f * n + i];
    uint32_t q = 0;
    if (nm != kExpNone) q = (uint32_t)floor(scalbn(fabs(c), -e0));
    qs[(int64_t)f * n + i] = q | (c < 0.0 ? 0x80000000u : 0u);
  }
}

// one thread per (field, code-block): all passes, one MQ codeword each
__global__ void __launch_bounds__(64) t1_encode_kernel(EbGeo eg, int cols, EbBufs b,
                                                       const uint8_t* active) {
  const int f = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= eg.nb || (active && !active[f])) return;
  const EbBlock B = eg.blocks[k];
  uint32_t* q = b.qs + (int64_t)f * b.n;
  Blk blk{b.flags + (int64_t)f * eg.state_stride + B.soff, (int64_t)B.r0 * cols + B.c0, cols,
          B.h, B.w, B.orient};
  for (int64_t i = 0; i < (int64_t)((B.h + 3) / 4) * 4 * B.w; i++) blk.f[i] = 0;
  uint32_t* uv = b.uval + ((int64_t)f * eg.nb + k) * kJ2Passes;
  for (int j = 0; j < kJ2Passes; j++) uv[j] = 0;
  if (b.nmax[f] == kExpNone) {
    b.ztab[(int64_t)f * eg.nb + k] = kJ2Planes;
    return;
  }
  uint32_t orq = 0;
  for (int y = 0; y < B.h; y++)
    for (int x = 0; x < B.w; x++) orq |= q[blk.base + (int64_t)y * cols + x] & 0xFFFFFFu;
  const int pt = orq ? 31 - __clz(orq) : -1;
  b.ztab[(int64_t)f * eg.nb + k] = (uint8_t)(pt < 0 ? kJ2Planes : kJ2Planes - 1 - pt);
  if (pt < 0) return;
  // codeword scratch: the block's share of the field's (kCwPerPoint bytes per sample)
  uint8_t* seg = b.cw + (int64_t)f * b.cw_stride + B.off * kCwPerPoint + (int64_t)k * kCwPerBlock;
  const int64_t segcap = (int64_t)B.h * B.w * kCwPerPoint + kCwPerBlock;
  Ctxs s;
  s.reset();
  MqEnc e;
  int64_t used = 0;
  const int np = 1 + 3 * pt;
  for (int j = 0; j < np; j++) {
    int p, ptype;
    pass_of(pt, j, p, ptype);
    if (ptype == 0)
      for (int y = 0; y < B.h; y++)
        for (int x = 0; x < B.w; x++) blk.ref(y, x) &= (uint16_t)~F_VIS;
    PassCoder<true> c{&e, nullptr, &s, 0, false, seg + used, segcap - used, nullptr, 0};
    run_pass<true>(blk, q, nullptr, p, ptype, c);
    if (c.started) {
      const int64_t len = e.flush();
      if (e.over || used + len > segcap) {
        atomicOr(b.status + f, 1);
        return;
      }
      uv[j] = (uint32_t)len + 1;
      used += len;
    }
  }
}

// one CTA per field: unit sizes by slot (global pass, block), scan, body
__global__ void __launch_bounds__(1024) assemble_kernel(EbGeo eg, int cols, EbBufs b,
                                                        const uint8_t* active) {
  const int f = blockIdx.x;
  if (active && !active[f]) return;
  const int nb = eg.nb;
  const int nslot = kJ2Slots * nb;
  uint32_t* cum = b.cum + (int64_t)f * (nslot + 1);
  uint8_t* body = b.body + (int64_t)f * b.body_stride;
  const uint8_t* zt = b.ztab + (int64_t)f * nb;
  const uint32_t* uval = b.uval + (int64_t)f * nb * kJ2Passes;
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  if (b.nmax[f] == kExpNone) {  // bare header: no body
    for (int i = threadIdx.x; i <= nslot; i += blockDim.x) cum[i] = 0;
    return;
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) body[i] = zt[i];
  __syncthreads();
  // cum[i] = bytes of slots < i (chunks of blockDim slots, block scan)
  for (int base = 0; base < nslot; base += blockDim.x) {
    const int i = base + threadIdx.x;
    uint32_t sz = 0;
    if (i < nslot) {
      const int g = i / nb, k = i - g * nb;
      const int pt = zt[k] >= kJ2Planes ? -1 : kJ2Planes - 1 - zt[k];
      const int j = pass_at(pt, g);
      if (j >= 0) {
        const uint32_t v = uval[(int64_t)k * kJ2Passes + j];
        sz = leb_len(v) + (v ? v - 1 : 0);
      }
    }
    uint32_t x = sz;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const uint32_t excl = carry + (w ? warp_tot[w - 1] : 0) + x - sz;
    if (i < nslot) cum[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + sz;
    __syncthreads();
  }
  if (threadIdx.x == 0) cum[nslot] = carry;
  if ((int64_t)nb + carry > b.body_stride) {
    if (threadIdx.x == 0) atomicOr(b.status + f, 2);
    return;
  }
  __syncthreads();
  // write the units: LEB128 value, then the codeword
  for (int i = threadIdx.x; i < nslot; i += blockDim.x) {
    const int g = i / nb, k = i - g * nb;
    const int pt = zt[k] >= kJ2Planes ? -1 : kJ2Planes - 1 - zt[k];
    const int j = pass_at(pt, g);
    if (j < 0) continue;
    uint32_t v = uval[(int64_t)k * kJ2Passes + j];
    uint8_t* o = body + nb + cum[i];
    const uint32_t len = v ? v - 1 : 0;
    do {
      uint8_t by = v & 0x7F;
      v >>= 7;
      if (v) by |= 0x80;
      *o++ = by;
    } while (v);
    if (len) {
      const EbBlock B = eg.blocks[k];
      // the block's codewords lie back to back in pass order
      int64_t off = 0;
      for (int jj = 0; jj < j; jj++) {
        const uint32_t vv = uval[(int64_t)k * kJ2Passes + jj];
        off += vv ? vv - 1 : 0;
      }
      const uint8_t* src =
          b.cw + (int64_t)f * b.cw_stride + B.off * kCwPerPoint + (int64_t)k * kCwPerBlock + off;
      for (uint32_t t = 0; t < len; t++) o[t] = src[t];
    }
  }
}

// closed form of a prefix: slot count j -> per block the last included
// global pass; a coefficient's value from its magnitude, sign and the pass
// (SP / CU) of its significance
__global__ void probe_decode_kernel(EbGeo eg, EbBufs b, const ProbeParam* __restrict__ prm,
                                    int nphys, double* out) {
  const int v = blockIdx.y;
  const int f = v % nphys;
  const ProbeParam P = prm[v];
  if (!P.active) return;
  const int nm = b.nmax[f];
  const int e0 = nm - (kJ2Planes - 1);
  const int nb = eg.nb;
  const int gt = (int)(P.B / (uint64_t)nb), kt = (int)(P.B % (uint64_t)nb);
  const uint32_t* q = b.qs + (int64_t)f * b.n;
  double* o = out + (int64_t)v * b.n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = q[i];
    const uint32_t mag = w & 0xFFFFFFu;
    double val = 0.0;
    if (nm != kExpNone && mag) {
      const int k = eg.blk_of[i];
      const int gmax = k < kt ? gt : gt - 1;
      const int ps = 31 - __clz(mag);
      const int gs = 3 * (kJ2Planes - 1 - ps) + ((w >> 30) & 1 ? 0 : 2);
      if (gs <= gmax) {
        int plo = ps;
        if (gmax >= 1) {
          const int pm = (kJ2Planes - 1) - (gmax - 1) / 3;
          plo = pm < 0 ? 0 : (pm < ps ? pm : ps);
        }
        const uint32_t m = mag >> plo;
        val = scalbn((double)(2 * m + 1), plo - 1 + e0);
        if (w >> 31) val = -val;
      }
    }
    o[i] = val;
  }
}

// decompress, step 1 (one thread per field): walk the units of the body
__global__ void parse_kernel(EbGeo eg, EbBufs b, const uint8_t* active) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= b.nfields || (active && !active[f])) return;
  const int nb = eg.nb;
  const uint8_t* body = b.body + (int64_t)f * b.body_stride;
  const int64_t len = (int64_t)b.body_len[f];
  int64_t* uo = b.uoff + (int64_t)f * nb * kJ2Passes;
  uint32_t* uv = b.uval + (int64_t)f * nb * kJ2Passes;
  for (int64_t i = 0; i < (int64_t)nb * kJ2Passes; i++) { uo[i] = -1; uv[i] = 0; }
  if (b.nmax[f] == kExpNone || len == 0) return;
  if (len < nb) { b.status[f] = 1; return; }
  int64_t pos = nb;
  for (int g = 0; g < kJ2Slots && pos < len; g++)
    for (int k = 0; k < nb && pos < len; k++) {
      const int z = body[k];
      if (z > kJ2Planes) { b.status[f] = 1; return; }
      const int pt = z == kJ2Planes ? -1 : kJ2Planes - 1 - z;
      const int j = pass_at(pt, g);
      if (j < 0) continue;
      uint64_t v = 0;
      int sh = 0;
      for (;;) {
        if (pos >= len || sh > 56) { b.status[f] = 1; return; }
        const uint8_t by = body[pos++];
        v |= (uint64_t)(by & 0x7F) << sh;
        sh += 7;
        if (!(by & 0x80)) break;
      }
      const int64_t cl = v ? (int64_t)v - 1 : 0;
      if (cl > len - pos) { b.status[f] = 1; return; }
      uo[(int64_t)k * kJ2Passes + j] = pos;
      uv[(int64_t)k * kJ2Passes + j] = (uint32_t)(v ? v : 0xFFFFFFFFu);  // 0xFFFFFFFF: present, no symbol
      pos += cl;
    }
  if (pos != len) b.status[f] = 1;
}

// decompress, step 2 (one thread per (field, block)): MQ-decode the present
// passes and reconstruct the block's coefficients
__global__ void __launch_bounds__(64) t1_decode_kernel(EbGeo eg, int cols, EbBufs b,
                                                       const uint8_t* active, double* out) {
  const int f = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= eg.nb || (active && !active[f])) return;
  const EbBlock B = eg.blocks[k];
  uint32_t* q = b.qs + (int64_t)f * b.n;
  int8_t* plow = b.plow + (int64_t)f * b.n;
  Blk blk{b.flags + (int64_t)f * eg.state_stride + B.soff, (int64_t)B.r0 * cols + B.c0, cols,
          B.h, B.w, B.orient};
  for (int64_t i = 0; i < (int64_t)((B.h + 3) / 4) * 4 * B.w; i++) blk.f[i] = 0;
  for (int y = 0; y < B.h; y++)
    for (int x = 0; x < B.w; x++) {
      const int64_t i = blk.base + (int64_t)y * cols + x;
      q[i] = 0;
      plow[i] = -1;
    }
  const int nm = b.nmax[f];
  const uint8_t* body = b.body + (int64_t)f * b.body_stride;
  if (nm != kExpNone && b.body_len[f] > 0) {
    const int z = body[k];
    const int pt = z >= kJ2Planes ? -1 : kJ2Planes - 1 - z;
    const int64_t* uo = b.uoff + ((int64_t)f * eg.nb + k) * kJ2Passes;
    const uint32_t* uv = b.uval + ((int64_t)f * eg.nb + k) * kJ2Passes;
    Ctxs s;
    s.reset();
    MqDec d;
    const int np = pt < 0 ? 0 : 1 + 3 * pt;
    for (int j = 0; j < np; j++) {
      if (uo[j] < 0) break;  // not in the prefix
      int p, ptype;
      pass_of(pt, j, p, ptype);
      if (ptype == 0)
        for (int y = 0; y < B.h; y++)
          for (int x = 0; x < B.w; x++) blk.ref(y, x) &= (uint16_t)~F_VIS;
      const bool sym = uv[j] != 0xFFFFFFFFu;
      PassCoder<false> c{nullptr, &d, &s, 0, false, nullptr, 0, body + uo[j],
                         sym ? (int64_t)uv[j] - 1 : 0};
      run_pass<false>(blk, q, plow, p, ptype, c);
      if ((c.nsym > 0) != sym) { b.status[f] = 1; return; }
    }
  }
  const int e0 = nm - (kJ2Planes - 1);
  double* o = out + (int64_t)f * b.n;
  for (int y = 0; y < B.h; y++)
    for (int x = 0; x < B.w; x++) {
      const int64_t i = blk.base + (int64_t)y * cols + x;
      const int wd = blk.word(y, x);
      double val = 0.0;
      if (wd & F_SIG) {
        const int pl = plow[i];
        const uint32_t m = q[i] >> pl;
        val = scalbn((double)(2 * m + 1), pl - 1 + e0);
        if (wd & F_NEG) val = -val;
      }
      o[i] = val;
    }
}

__device__ __forceinline__ double div_exact_rn(double x, double bb, double binv) {
  const double qq = __dmul_rn(x, binv);
  const double r = __fma_rn(-qq, bb, x);
  return copysign(__fma_rn(r, binv, qq), x);
}

__global__ void reduce_kernel(const double* __restrict__ dec, const float* __restrict__ orig,
                              const FieldScal* fs, const ProbeParam* prm, int64_t n, bool count,
                              ProbeResult* res) {
  const int f = blockIdx.y;
  if (!prm[f].active) return;
  const FieldScal s = fs[f];
  unsigned long long cnt = 0;
  double mx = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = dec[(int64_t)f * n + i];
    const float o = orig[(int64_t)f * n + i];
    if (count) {
      const double nv = div_exact_rn(__dsub_rn((double)o, s.vmin), s.range, s.range_inv);
      cnt += !(fabs(__dsub_rn(d, nv)) <= s.eps_rel);
    }
    const float rec = __double2float_rn(__dadd_rn(s.vmin, __dmul_rn(d, s.range)));
    mx = fmax(mx, fabs(__dsub_rn((double)rec, (double)o)));
  }
  unsigned long long mb = (unsigned long long)__double_as_longlong(mx);
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, mb, o);
    mb = y > mb ? y : mb;
  }
  if ((threadIdx.x & 31) == 0) {
    if (count && cnt) atomicAdd(&res[f].count, cnt);
    atomicMax(&res[f].maxerr, mb);
  }
}

__global__ void residue_kernel(const double* __restrict__ dec, const ProbeParam* prm, int64_t n,
                               double* base_dec, double* resid) {
  const int f = blockIdx.y;
  if (!prm[f].active) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)f * n + i;
    const double d = dec[o];
    base_dec[o] = d;
    resid[o] = __dsub_rn(resid[o], d);  // norm - base decode, in place
  }
}

__global__ void init_kernel(int32_t* nmax, int32_t* status, int nf) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) { nmax[f] = kExpNone; status[f] = 0; }
}

__global__ void nmax_copy_kernel(const int32_t* nmax, const int32_t* status, MachineOut* mo,
                                 int nf) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  MachineOut m{};
  m.n_max = nmax[f];
  m.overflow = status[f] != 0;
  mo[f] = m;
}

int grid_x(int64_t n, int cap = 1024) {
  const int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

}  // namespace

EbGeo ebcot_build_geo(const Geo& g, int32_t** blk_of_out, EbBlock** blocks_out, cudaStream_t st) {
  std::vector<EbBlock> bl;
  const int L = g.levels;
  for (int band = 0; band <= 3 * L; band++) {
    int r0, c0, h, w, orient;
    if (band == 0) {
      r0 = 0; c0 = 0; h = g.lr[L]; w = g.lc[L]; orient = 0;
    } else {
      const int k = L - (band - 1) / 3, o = (band - 1) % 3;
      const Rect R = detail_rect(g, k, o);
      r0 = R.r0; c0 = R.c0; h = R.h; w = R.w;
      orient = o == 0 ? 1 : (o == 1 ? 0 : 2);
    }
    if (h <= 0 || w <= 0) continue;
    for (int by = 0; by < h; by += kJ2Block)
      for (int bx = 0; bx < w; bx += kJ2Block)
        bl.push_back(EbBlock{r0 + by, c0 + bx, std::min(kJ2Block, h - by),
                             std::min(kJ2Block, w - bx), orient, 0, 0, 0});
  }
  int64_t acc = 0, sacc = 0;
  for (EbBlock& e : bl) {
    e.off = acc;
    acc += (int64_t)e.h * e.w;
    e.soff = sacc;
    sacc += (int64_t)((e.h + 3) / 4) * 4 * e.w;
  }
  std::vector<int32_t> of((size_t)g.n);
  for (int k = 0; k < (int)bl.size(); k++)
    for (int y = 0; y < bl[k].h; y++)
      for (int x = 0; x < bl[k].w; x++)
        of[(size_t)(bl[k].r0 + y) * g.cols + bl[k].c0 + x] = k;
  EbBlock* db = nullptr;
  int32_t* dof = nullptr;
  cudaMalloc(&db, sizeof(EbBlock) * std::max<size_t>(1, bl.size()));
  cudaMalloc(&dof, sizeof(int32_t) * (size_t)g.n);
  cudaMemcpyAsync(db, bl.data(), sizeof(EbBlock) * bl.size(), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dof, of.data(), sizeof(int32_t) * (size_t)g.n, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  *blk_of_out = dof;
  *blocks_out = db;
  return EbGeo{(int)bl.size(), db, dof, sacc};
}

void ebcot_encode(const double* coef, const EbGeo& eg, const Geo& g, EbBufs& b,
                  const uint8_t* active, cudaStream_t st) {
  const int nf = b.nfields;
  init_kernel<<<(nf + 255) / 256, 256, 0, st>>>(b.nmax, b.status, nf);
  nmax_kernel<<<dim3(grid_x(g.n), nf), 256, 0, st>>>(coef, g.n, b.nmax, active);
  quantize_kernel<<<dim3(grid_x(g.n), nf), 256, 0, st>>>(coef, g.n, b.nmax, b.qs, active);
  t1_encode_kernel<<<dim3((eg.nb + 63) / 64, nf), 64, 0, st>>>(eg, g.cols, b, active);
  assemble_kernel<<<nf, 1024, 0, st>>>(eg, g.cols, b, active);
}

void ebcot_probe_decode(const EbGeo& eg, const EbBufs& b, const ProbeParam* prm, int nprobes,
                        int nphys, double* out, cudaStream_t st) {
  probe_decode_kernel<<<dim3(grid_x(b.n), nprobes), 256, 0, st>>>(eg, b, prm, nphys, out);
}

void ebcot_stream_decode(const EbGeo& eg, const Geo& g, EbBufs& b, const uint8_t* active,
                         double* out, cudaStream_t st) {
  parse_kernel<<<(b.nfields + 31) / 32, 32, 0, st>>>(eg, b, active);
  t1_decode_kernel<<<dim3((eg.nb + 63) / 64, b.nfields), 64, 0, st>>>(eg, g.cols, b, active, out);
}

void ebcot_nmax_to(const EbBufs& b, MachineOut* mo, cudaStream_t st) {
  nmax_copy_kernel<<<(b.nfields + 255) / 256, 256, 0, st>>>(b.nmax, b.status, mo, b.nfields);
}

void ebcot_probe_reduce(const double* dec, const float* orig, const FieldScal* fs,
                        const ProbeParam* prm, int64_t n, int nfields, bool count,
                        ProbeResult* res, cudaStream_t st) {
  reduce_kernel<<<dim3(grid_x(n, 512), nfields), 256, 0, st>>>(dec, orig, fs, prm, n, count, res);
}

void ebcot_residue(const double* dec, const ProbeParam* prm, int64_t n, int nfields,
                   double* base_dec, double* resid, cudaStream_t st) {
  residue_kernel<<<dim3(grid_x(n), nfields), 256, 0, st>>>(dec, prm, n, base_dec, resid);
}

}  // namespace ebcc
