// Device-resident feedback controller: the reference's searches as
// per-chunk resumable state machines (see ctl.cuh).
//
// Each state machine is written as the reference's straight-line code with
// every memo access a suspension point: CTL_GET(KEY, LABEL) looks the key up
// and, if no probe has answered it yet, records LABEL, posts the probe and
// returns; the next advance re-enters the switch at LABEL (a Duff's-device
// coroutine; every variable that lives across a suspension is a CtlChunk
// field).  One thread advances one chunk; a controller launch is a single
// CTA that also sets the graph's conditional handles.
#include <cstdio>

#include "ctl.cuh"
#include "ebcot.cuh"

namespace ebcc {
namespace {

constexpr int kBasePlanes = 24, kDeepPlanes = 32;
static_assert(sizeof(CtlChunk) * kCtlSmemChunks <= 227 * 1024, "staged states exceed shared memory");
static_assert(sizeof(CtlChunk) % 8 == 0, "staged as 8-byte words");
constexpr int kSuspend = 1, kDone = 0;

// CPython float floor division (Objects/floatobject.c float_divmod), as
// base_codec.budget_for_ratio uses it: int(raw // ratio) != floor(raw / ratio)
__device__ double py_floordiv(double vx, double wx) {
  const double mod = fmod(vx, wx);
  double div = __ddiv_rn(__dsub_rn(vx, mod), wx);
  if (mod != 0.0 && ((wx < 0) != (mod < 0))) div = __dsub_rn(div, 1.0);
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
  } else {
    fl = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return fl;
}

__device__ __forceinline__ int64_t clamp_budget(const CtlChunk& s, int64_t b) {
  if (b > s.raw) b = s.raw;
  if (b < kHeader) b = kHeader;
  return b;
}
// base_codec.budget_for_ratio (base_codec.py:34-38), then _ChunkCoder's clamp
__device__ __forceinline__ int64_t ratio_budget(const CtlChunk& s, double ratio) {
  int64_t b = (int64_t)py_floordiv((double)s.raw, ratio);
  return clamp_budget(s, b > kHeader ? b : kHeader);
}
// J2 base: slots of the longest unit-aligned prefix within b bytes (-1: the
// bare header)
__device__ __forceinline__ int64_t eb_slots(const CtlChunk& s, int64_t b) {
  const int64_t room = b - kHeader - s.eb_sub;
  if (room < 0) return -1;
  int lo = 0, hi = s.eb_nslot;  // largest k with cum[k] <= room
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int64_t)s.eb_cum[mid] <= room) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ int64_t stream_len(const CtlChunk& s, int64_t b) {
  if (s.eb_cum) {
    const int64_t k = eb_slots(s, b);
    return k < 0 ? kHeader : kHeader + s.eb_sub + (int64_t)s.eb_cum[k];
  }
  const int64_t full = kHeader + (int64_t)((s.T_base + 7) / 8);
  return b < full ? b : full;
}
__device__ __forceinline__ int memo_find(const CtlChunk& s, int64_t b) {
  for (int i = 0; i < s.nmemo; i++)
    if (s.memo[i].budget == b) return i;
  return -1;
}
__device__ __forceinline__ int smemo_find(const CtlChunk& s, int64_t b) {
  for (int i = 0; i < s.nsmemo; i++)
    if (s.smemo[i].budget == b) return i;
  return -1;
}
// the memo entry of budget b; a speculative answer moves into the memo when
// the search asks for its budget (the reference's probe at that point)
__device__ int memo_get(CtlChunk& s, int64_t b) {
  const int i = memo_find(s, b);
  if (i >= 0) return i;
  const int j = smemo_find(s, b);
  if (j < 0) return -1;
  if (s.nmemo >= kCtlMemo) {
    s.status |= kCtlCapacity;
    return -1;
  }
  s.memo[s.nmemo] = s.smemo[j];
  return s.nmemo++;
}
__device__ __forceinline__ double q_of(const CtlChunk& s, int i) {
  return __ddiv_rn((double)s.memo[i].count, (double)s.n);
}
__device__ __forceinline__ bool pure_ok_at(const CtlChunk& s, int i) {
  return s.memo[i].maxerr <= s.eps_abs;
}
__device__ __forceinline__ int tmemo_find(const CtlChunk& s, int pi, int64_t t) {
  for (int i = 0; i < s.ntmemo[pi]; i++)
    if (s.tmemo[pi][i].t == t) return i;
  return -1;
}

// ---- _search_base (pipeline.py:142-199) -------------------------------------
// s.want_b / s.cur_b: the key and memo index of the access in progress
// (a suspension also sets s.bspec: the keys the next step asks whichever way
// this probe answers, for the speculative slots)
#define CTL_GET_B(KEY, LABEL)                           \
  s.want_b = (KEY);                                     \
  case LABEL:                                           \
    if ((s.cur_b = memo_get(s, s.want_b)) < 0) {        \
      s.pc_b = LABEL;                                   \
      base_spec(s, LABEL);                              \
      return kSuspend;                                  \
    }

// first step of the byte-exact refinement (pipeline.py:193-198 seeding, then
// _bisect_min_feasible) if the memo also held budget b with feasibility feas
// (-1: the bracket is already closed)
__device__ int64_t refine_first(const CtlChunk& s, int64_t b, bool feas) {
  int64_t hi = -1, lo = kHeader - 1;
  for (int i = 0; i < s.nmemo; i++)
    if (q_of(s, i) >= s.q && (hi < 0 || s.memo[i].budget < hi)) hi = s.memo[i].budget;
  if (feas && (hi < 0 || b < hi)) hi = b;
  for (int i = 0; i < s.nmemo; i++)
    if (q_of(s, i) < s.q && s.memo[i].budget < hi && s.memo[i].budget > lo) lo = s.memo[i].budget;
  if (!feas && b < hi && b > lo) lo = b;
  return hi - lo > 1 ? clamp_budget(s, (lo + hi) / 2) : -1;
}
// the ratio bisection's next key on [lo, hi], or the refinement's first
__device__ int64_t ratio_step(const CtlChunk& s, double lo, double hi, int64_t b, bool feas) {
  if (__dsub_rn(hi, lo) > s.tol) return ratio_budget(s, __dmul_rn(0.5, __dadd_rn(lo, hi)));
  return refine_first(s, b, feas);
}
// keys of the base search's next access for each answer of the probe at
// s.want_b (the code below, label by label; infeasible first)
__device__ void base_spec(CtlChunk& s, int label) {
  const int64_t b = s.want_b;
  int64_t k0 = -1, k1 = -1;
  switch (label) {
    case 1:  // r0: halve r_low / double r_high
      if (s.r0c > 1.0) k0 = ratio_budget(s, fmax(1.0, __ddiv_rn(s.r0c, 2.0)));
      k1 = s.r0c < s.r_cap ? ratio_budget(s, fmin(s.r_cap, __dmul_rn(s.r0c, 2.0)))
                           : ratio_step(s, s.r0c, s.r0c, b, true);
      break;
    case 2:  // r_low: halve again / bisect [r_low, r_high]
      if (s.r_low > 1.0) k0 = ratio_budget(s, fmax(1.0, __ddiv_rn(s.r_low, 2.0)));
      k1 = ratio_step(s, s.r_low, s.r_high, b, true);
      break;
    case 5:  // r_high: double again / bisect
      if (s.r_high < s.r_cap) {
        k1 = ratio_budget(s, fmin(s.r_cap, __dmul_rn(s.r_high, 2.0)));
        k0 = ratio_step(s, s.r_low, s.r_high, b, false);
      } else {
        k0 = ratio_step(s, s.r_low, s.r_high, b, false);
        k1 = ratio_step(s, s.r_low, s.r_high, b, true);
      }
      break;
    case 6:  // ratio bisection
      k0 = ratio_step(s, s.r_low, s.r_mid, b, false);
      k1 = ratio_step(s, s.r_mid, s.r_high, b, true);
      break;
    case 7:  // byte bisection
      if (s.hi_b - s.mid_b > 1) k0 = clamp_budget(s, (s.mid_b + s.hi_b) / 2);
      if (s.mid_b - s.lo_b > 1) k1 = clamp_budget(s, (s.lo_b + s.mid_b) / 2);
      break;
    default:
      break;
  }
  s.bspec[0] = k0;
  s.bspec[1] = k1;
}

__device__ int adv_base(CtlChunk& s) {
  switch (s.pc_b) {
    case 0:
      s.r_cap = fmax(1.0, __ddiv_rn((double)s.raw, (double)kHeader));
      s.r0c = fmin(fmax(s.r0, 1.0), s.r_cap);
      CTL_GET_B(ratio_budget(s, s.r0c), 1)
      s.q_a0 = q_of(s, s.cur_b);
      s.r_low = s.r_high = s.r0c;
      s.have = s.q_a0 >= s.q;
      s.q_a = s.q_a0;
      while (s.q_a < s.q && s.r_low > 1.0) {
        s.r_low = fmax(1.0, __ddiv_rn(s.r_low, 2.0));
        CTL_GET_B(ratio_budget(s, s.r_low), 2)
        s.q_a = q_of(s, s.cur_b);
      }
      if (s.q_a >= s.q) {
        CTL_GET_B(ratio_budget(s, s.r_low), 3)
        s.have = 1;
      }
      if (!s.have) {
        CTL_GET_B(ratio_budget(s, 1.0), 4)
        s.base_budget = s.memo[s.cur_b].budget;
        s.done_b = 1;
        s.pc_b = 99;
        return kDone;
      }
      s.q_a = s.q_a0;
      while (s.q_a > s.q && s.r_high < s.r_cap) {
        s.r_high = fmin(s.r_cap, __dmul_rn(s.r_high, 2.0));
        CTL_GET_B(ratio_budget(s, s.r_high), 5)
        s.q_a = q_of(s, s.cur_b);
      }
      while (__dsub_rn(s.r_high, s.r_low) > s.tol) {
        if (++s.guard > (1 << 20)) {  // the reference would spin forever here
          s.status |= kCtlCapacity;
          s.done_b = 1;
          s.pc_b = 99;
          return kDone;
        }
        s.r_mid = __dmul_rn(0.5, __dadd_rn(s.r_low, s.r_high));
        CTL_GET_B(ratio_budget(s, s.r_mid), 6)
        if (q_of(s, s.cur_b) < s.q) s.r_high = s.r_mid;
        else s.r_low = s.r_mid;
      }
      // byte-exact refinement seeded from every budget cached so far
      // (pipeline.py:193-198)
      s.hi_b = -1;
      s.lo_b = kHeader - 1;
      for (int i = 0; i < s.nmemo; i++)
        if (q_of(s, i) >= s.q && (s.hi_b < 0 || s.memo[i].budget < s.hi_b)) s.hi_b = s.memo[i].budget;
      for (int i = 0; i < s.nmemo; i++)
        if (q_of(s, i) < s.q && s.memo[i].budget < s.hi_b && s.memo[i].budget > s.lo_b)
          s.lo_b = s.memo[i].budget;
      // pipeline._bisect_min_feasible
      while (s.hi_b - s.lo_b > 1) {
        s.mid_b = (s.lo_b + s.hi_b) / 2;
        CTL_GET_B(clamp_budget(s, s.mid_b), 7)
        if (q_of(s, s.cur_b) >= s.q) s.hi_b = s.mid_b;
        else s.lo_b = s.mid_b;
      }
      CTL_GET_B(clamp_budget(s, s.hi_b), 8)
      s.base_budget = s.memo[s.cur_b].budget;
      s.done_b = 1;
      s.pc_b = 99;
      return kDone;
    default:
      return kDone;
  }
}

// ---- _search_pure (pipeline.py:215-236) ---------------------------------
#define CTL_GET_P(KEY, LABEL)                           \
  s.want_p = (KEY);                                     \
  case LABEL:                                           \
    if ((s.cur_p = memo_get(s, s.want_p)) < 0) {        \
      s.pc_p = LABEL;                                   \
      pure_spec(s, LABEL);                              \
      return kSuspend;                                  \
    }

// the pure-base bisection's first key after the bracket is seeded from the
// memo (the entries at kHeader and raw do not move it)
__device__ int64_t pure_first(const CtlChunk& s) {
  int64_t lo = kHeader, hi = s.raw;
  for (int i = 0; i < s.nmemo; i++)
    if (pure_ok_at(s, i) && s.memo[i].budget < hi) hi = s.memo[i].budget;
  for (int i = 0; i < s.nmemo; i++)
    if (s.memo[i].budget < hi && !pure_ok_at(s, i) && s.memo[i].budget > lo) lo = s.memo[i].budget;
  return hi - lo > 1 ? clamp_budget(s, (lo + hi) / 2) : -1;
}
__device__ void pure_spec(CtlChunk& s, int label) {
  int64_t k0 = -1, k1 = -1;
  switch (label) {
    case 1:
      k0 = clamp_budget(s, s.raw);
      k1 = pure_first(s);
      break;
    case 2:
      k0 = pure_first(s);
      break;
    case 3:
      if (s.hi_p - s.mid_p > 1) k0 = clamp_budget(s, (s.mid_p + s.hi_p) / 2);
      if (s.mid_p - s.lo_p > 1) k1 = clamp_budget(s, (s.lo_p + s.mid_p) / 2);
      break;
    default:
      break;
  }
  s.bspec[0] = k0;
  s.bspec[1] = k1;
}

__device__ int adv_pure(CtlChunk& s) {
  switch (s.pc_p) {
    case 0:
      s.p_lb = kHeader;
      s.p_ub = -1;
      CTL_GET_P(clamp_budget(s, kHeader), 1)
      if (pure_ok_at(s, s.cur_p)) {
        s.pure_budget = s.memo[s.cur_p].budget;
        s.done_p = 1;
        s.pc_p = 99;
        return kDone;
      }
      s.p_lb = kHeader + 1;
      CTL_GET_P(clamp_budget(s, s.raw), 2)
      if (!pure_ok_at(s, s.cur_p)) {
        s.pure_budget = -1;
        s.done_p = 1;
        s.pc_p = 99;
        return kDone;
      }
      s.lo_p = kHeader;
      s.hi_p = s.raw;
      // sorted(self._by_budget): every budget cached at this point
      s.ncached = s.nmemo;
      for (int i = 0; i < s.ncached; i++) {
        const int64_t b = s.memo[i].budget;
        int j = i;
        while (j > 0 && s.cached[j - 1] > b) {
          s.cached[j] = s.cached[j - 1];
          j--;
        }
        s.cached[j] = b;
      }
      for (int i = 0; i < s.ncached; i++)
        if (pure_ok_at(s, memo_find(s, s.cached[i])) && s.cached[i] < s.hi_p) s.hi_p = s.cached[i];
      for (int i = 0; i < s.ncached; i++)
        if (s.cached[i] < s.hi_p && !pure_ok_at(s, memo_find(s, s.cached[i])) &&
            s.cached[i] > s.lo_p)
          s.lo_p = s.cached[i];
      while (s.hi_p - s.lo_p > 1) {
        s.mid_p = (s.lo_p + s.hi_p) / 2;
        s.p_lb = stream_len(s, s.lo_p + 1);  // the answer's bracket (candidate pruning)
        s.p_ub = stream_len(s, s.hi_p);
        CTL_GET_P(clamp_budget(s, s.mid_p), 3)
        if (pure_ok_at(s, s.cur_p)) s.hi_p = s.mid_p;
        else s.lo_p = s.mid_p;
      }
      CTL_GET_P(clamp_budget(s, s.hi_p), 4)
      s.pure_budget = s.memo[s.cur_p].budget;
      s.done_p = 1;
      s.pc_p = 99;
      return kDone;
    default:
      return kDone;
  }
}

// ---- _truncation_search (pipeline.py:243-254), 24 then 32 planes ----------
#define CTL_GET_T(KEY, LABEL)                                     \
  s.want_t = (KEY);                                               \
  case LABEL:                                                     \
    if ((s.cur_t = tmemo_find(s, s.pass, s.want_t)) < 0) {        \
      s.pc_t = LABEL;                                             \
      return kSuspend;                                            \
    }                                                             \
    s.ntcalls++;

__device__ __forceinline__ double terr(const CtlChunk& s) { return s.tmemo[s.pass][s.cur_t].err; }

__device__ int adv_trunc(CtlChunk& s) {
  switch (s.pc_t) {
    case 0:
      s.pass = 0;
      while (s.pass < 2) {
        s.total_t = (int64_t)(((s.pass ? s.T32 : s.T24) + 7) / 8);
        s.t_lb = 0;
        s.t_ub = -1;
        s.spec[0] = s.total_t;      // a miss at err_at(0): 0, total and the
        s.spec[1] = s.total_t / 2;  // first midpoint are all needed
        CTL_GET_T(0, 1)
        if (terr(s) <= s.eps_abs) {
          s.trunc_t = 0;
          s.trunc_planes = s.pass ? kDeepPlanes : kBasePlanes;
          s.done_t = 1;
          s.pc_t = 99;
          return kDone;
        }
        s.spec[0] = s.total_t / 2;
        s.spec[1] = -1;
        CTL_GET_T(s.total_t, 2)
        if (!(terr(s) <= s.eps_abs)) {  // this planes variant cannot reach the bound
          s.pass++;
          continue;
        }
        s.lo_t = 0;
        s.hi_t = s.total_t;
        while (s.hi_t - s.lo_t > 1) {
          s.mid_t = (s.lo_t + s.hi_t) / 2;
          s.t_lb = s.lo_t + 1;
          s.t_ub = s.hi_t;
          s.spec[0] = s.mid_t - s.lo_t > 1 ? (s.lo_t + s.mid_t) / 2 : -1;
          s.spec[1] = s.hi_t - s.mid_t > 1 ? (s.mid_t + s.hi_t) / 2 : -1;
          CTL_GET_T(s.mid_t, 3)
          if (terr(s) <= s.eps_abs) s.hi_t = s.mid_t;
          else s.lo_t = s.mid_t;
        }
        s.trunc_t = s.hi_t;
        s.trunc_planes = s.pass ? kDeepPlanes : kBasePlanes;
        s.done_t = 1;
        s.pc_t = 99;
        return kDone;
      }
      s.trunc_t = -1;
      s.trunc_planes = 0;
      s.done_t = 1;
      s.pc_t = 99;
      return kDone;
    default:
      return kDone;
  }
}

// midpoint stopping plane of a decode of B bits of the `planes`-plane variant
// (decode_with_plane, spiht.py:426-478, incl. zero-padded phantom planes)
__device__ int n_last_of(const MachineOut& mo, const PlaneRec* pl, int planes, uint64_t B,
                         uint64_t T) {
  if (B == 0) return mo.n_max;
  if (B <= T) {
    int p = 0;
    for (int k = 0; k < planes; k++)
      if (pl[k].start < B) p = k;
    return mo.n_max - p;
  }
  const uint64_t L = pl[planes - 1].lists_end;
  int jmax;
  if (L == 0) {
    jmax = (kMaxDecodePlanes - 1) - planes;
  } else {
    const uint64_t j = (B - T + L - 1) / L - 1;
    const uint64_t cap = (uint64_t)((kMaxDecodePlanes - 1) - planes);
    jmax = (int)(j < cap ? j : cap);
  }
  return mo.n_max - (planes + jmax);
}

// counted: a base-search probe (its count field holds violations; a probe
// that stopped early reported more than vlim of them, so the count stored
// here is below the threshold exactly when the full count would be)
__device__ CtlEntry make_entry(const CtlChunk& s, int64_t b, const ProbeResult& r, bool counted) {
  double e;
  unsigned long long bits = r.maxerr;
  memcpy(&e, &bits, 8);
  const unsigned long long v = r.count;
  const unsigned long long hits = !counted ? 0ull : (v >= (unsigned long long)s.n ? 0ull : (unsigned long long)s.n - v);
  return CtlEntry{b, hits, e};
}
__device__ void memo_add(CtlChunk& s, int64_t b, const ProbeResult& r, bool counted) {
  if (memo_find(s, b) >= 0) return;
  if (s.nmemo >= kCtlMemo) {
    s.status |= kCtlCapacity;
    return;
  }
  s.memo[s.nmemo++] = make_entry(s, b, r, counted);
}
// a speculative answer (dropped when the side memo is full: the search then
// probes that budget itself)
__device__ void smemo_add(CtlChunk& s, int64_t b, const ProbeResult& r, bool counted) {
  if (memo_find(s, b) >= 0 || smemo_find(s, b) >= 0 || s.nsmemo >= kCtlSMemo) return;
  s.smemo[s.nsmemo++] = make_entry(s, b, r, counted);
}
// the speculative slots' requests for the access in flight at key `want`
template <class Req>
__device__ void post_spec(CtlChunk& s, int bslots, int64_t want, ProbeParam* ps, Req req) {
  for (int k = 1; k < bslots; k++) {
    const int64_t b2 = s.bspec[k - 1];
    s.bspend[k - 1] = -1;
    if (b2 < 0 || b2 == want || (k == 2 && b2 == s.bspec[0]) || memo_find(s, b2) >= 0 ||
        smemo_find(s, b2) >= 0)
      continue;
    s.bspend[k - 1] = b2;
    ps[k] = req(b2);
  }
}
// park the speculative slots' answers
__device__ void ingest_spec(CtlChunk& s, const CtlArgs& a, int f, bool counted) {
  for (int k = 1; k < a.bslots; k++) {
    if (s.bspend[k - 1] >= 0) smemo_add(s, s.bspend[k - 1], a.res[k * a.nfields + f], counted);
    s.bspend[k - 1] = -1;
  }
}
__device__ void tmemo_add(CtlChunk& s, int pi, int64_t t, const ProbeResult& r) {
  if (tmemo_find(s, pi, t) >= 0) return;
  if (s.ntmemo[pi] >= kCtlTMemo) {
    s.status |= kCtlCapacity;
    return;
  }
  double e;
  unsigned long long bits = r.maxerr;
  memcpy(&e, &bits, 8);
  s.tmemo[pi][s.ntmemo[pi]++] = CtlTEntry{t, e};
}

__device__ ProbeParam base_request(const CtlChunk& s, int64_t b, bool early) {
  ProbeParam p{};
  uint64_t B;
  if (s.eb_cum) {  // J2 base: the slots the prefix holds
    const int64_t k = eb_slots(s, b);
    B = k < 0 ? 0 : (uint64_t)k;
  } else {
    B = (uint64_t)(stream_len(s, b) - kHeader) * 8;
    if (B > s.T_base) B = s.T_base;
  }
  p.B = B;
  p.planes = kBasePlanes;
  p.active = 1;
  p.early = early;
  p.vlim = s.vlim;
  return p;
}

// smallest count c with c / n >= q (the reference's float64 compare), as the
// number of violations a count probe may see: n - c (-1: none reaches q)
__device__ int32_t violation_limit(int64_t n, double q) {
  const double dn = (double)n;
  int64_t c = (int64_t)floor(__dmul_rn(q, dn));
  if (c < 0) c = 0;
  if (c > n) c = n;
  while (c > 0 && __ddiv_rn((double)(c - 1), dn) >= q) c--;
  while (c <= n && __ddiv_rn((double)c, dn) < q) c++;
  return (int32_t)(n - c);
}

__device__ ProbeParam trunc_request(const CtlChunk& s, const CtlArgs& a, int f, int pi, int64_t t,
                                    bool early) {
  ProbeParam p{};
  const int P = pi ? kDeepPlanes : kBasePlanes;
  const uint64_t T = pi ? s.T32 : s.T24;
  const uint64_t Bfull = (uint64_t)t * 8;
  p.B = Bfull < T ? Bfull : T;
  p.planes = P;
  p.midpoint = 1;
  const MachineOut mo = a.mo_res[f];
  p.n_last = mo.n_max == kExpNone ? 0
                                   : n_last_of(mo, a.pl_res + (int64_t)f * kMaxPlaneRecs, P, Bfull, T);
  p.active = 1;
  p.early = early;
  return p;
}

// the controller is one CTA; `any` is or-reduced over it
__device__ __forceinline__ bool block_any(bool v) { return __syncthreads_or(v) != 0; }

// Few chunks: their states are staged through shared memory, so the one
// thread advancing a chunk pays shared-memory latency instead of a chain of
// dependent L2 misses (cold L1 at every launch).
extern __shared__ __align__(16) unsigned char ctl_sm[];
__device__ CtlChunk* stage_in(const CtlArgs& a) {
  if (!a.smem) return a.cs;
  const size_t words = sizeof(CtlChunk) / 8 * (size_t)a.nfields;
  const uint64_t* src = reinterpret_cast<const uint64_t*>(a.cs);
  uint64_t* dst = reinterpret_cast<uint64_t*>(ctl_sm);
  for (size_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  return reinterpret_cast<CtlChunk*>(ctl_sm);
}
__device__ void stage_out(const CtlArgs& a) {
  if (!a.smem) return;
  __syncthreads();
  const size_t words = sizeof(CtlChunk) / 8 * (size_t)a.nfields;
  const uint64_t* src = reinterpret_cast<const uint64_t*>(ctl_sm);
  uint64_t* dst = reinterpret_cast<uint64_t*>(a.cs);
  for (size_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}

__global__ void __launch_bounds__(1024) ctl_setup_kernel(CtlArgs a) {
  const CtlParams P = *a.prm_in;
  for (int f = threadIdx.x; f < a.nfields; f += blockDim.x) {
    const FieldScal fs = a.fs[f];
    const bool act = !fs.constant && fs.first_bad < 0;
    a.active[f] = act;
    MachineOut m{};
    m.n_max = kExpNone;
    a.mo_base[f] = m;
    a.mo_res[f] = m;
    CtlChunk& s = a.cs[f];
    s.n = a.n;
    s.raw = 4 * a.n;
    s.q = P.q;
    s.r0 = P.r0;
    s.tol = P.tol;
    s.eps_abs = fs.eps_abs;
    s.vlim = violation_limit(a.n, P.q);
    s.T_base = s.T24 = s.T32 = 0;
    s.active = act;
    s.status = 0;
    s.nmemo = 0;
    s.pend = 0;
    s.pend_budget = -1;
    s.pc_b = s.pc_p = s.pc_t = 0;
    s.guard = 0;
    s.done_b = s.done_p = s.done_t = act ? 0 : 1;
    s.base_budget = s.pure_budget = s.trunc_t = -1;
    s.trunc_planes = 0;
    s.ntcalls = 0;
    s.pure_pruned = s.trunc_pruned = 0;
    s.p_lb = kHeader;
    s.p_ub = -1;
    s.t_lb = 0;
    s.t_ub = -1;
    s.ntmemo[0] = s.ntmemo[1] = 0;
    for (int k = 0; k < kCtlSlots; k++) s.tpend[k] = -1;
    s.tpend_pi = 0;
    s.eb_cum = nullptr;
    s.eb_sub = s.eb_nslot = 0;
    s.nsmemo = 0;
    s.bspec[0] = s.bspec[1] = -1;
    for (int k = 0; k + 1 < kCtlSlots; k++) s.bspend[k] = -1;
  }
  if (threadIdx.x == 0) *a.stats = CtlStats{};
}

__global__ void __launch_bounds__(1024) ctl_base_kernel(CtlArgs a, int start, int set) {
  const bool early = a.prm_in->early != 0;
  bool any = false;
  CtlChunk* cs = stage_in(a);
  const int nf = a.nfields;
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    CtlChunk& s = cs[f];
    ProbeParam p[kCtlSlots] = {};
    if (s.active) {
      if (start) {
        s.T_base = a.mo_base[f].total_bits;
        if (a.mo_base[f].overflow) s.status |= kCtlCapacity;
        if (a.eb_cum) {  // J2 base: unit boundaries of the encoded stream
          s.eb_nslot = kJ2Slots * a.eb_nb;
          s.eb_cum = a.eb_cum + (int64_t)f * (s.eb_nslot + 1);
          s.eb_sub = a.eb_nmax[f] == kExpNone ? 0 : a.eb_nb;
        }
      }
      if (s.pend) {  // the probe that answered s.pend_budget
        memo_add(s, s.pend_budget, a.res[f], true);
        s.pend = 0;
      }
      ingest_spec(s, a, f, true);
      if (!s.done_b && !(s.status & kCtlCapacity) && adv_base(s) == kSuspend) {
        s.pend = 1;
        s.pend_budget = s.want_b;
        p[0] = base_request(s, s.want_b, early);
        post_spec(s, a.bslots, s.want_b, p, [&](int64_t b) { return base_request(s, b, early); });
        any = true;
      }
    }
    for (int k = 0; k < a.bslots; k++) {
      a.res[k * nf + f] = ProbeResult{};
      a.prm[k * nf + f] = p[k];
    }
  }
  stage_out(a);
  any = block_any(any);
  if (threadIdx.x == 0) {
    if (set & 1) cudaGraphSetConditional(a.h_loop, any ? 1u : 0u);
    if (set & 2) cudaGraphSetConditional(a.h_pure, any ? 1u : 0u);
    if (!start) a.stats->base_steps++;
    if (any) a.stats->base_probes++;
  }
}

__global__ void __launch_bounds__(1024) ctl_residue_kernel(CtlArgs a) {
  for (int f = threadIdx.x; f < a.nfields; f += blockDim.x) {
    const CtlChunk& s = a.cs[f];
    ProbeParam p{};
    if (s.active && s.base_budget >= 0) p = base_request(s, s.base_budget, false);
    a.prm[f] = p;
  }
}

__global__ void __launch_bounds__(1024) ctl_joint_kernel(CtlArgs a, int start, int set) {
  const CtlParams P = *a.prm_in;
  bool anyp = false, anyt = false;
  const int nf = a.nfields;
  if (start) {  // the residual stream's lengths; the searches start at the first step
    for (int f = threadIdx.x; f < nf; f += blockDim.x) {
      CtlChunk& s = a.cs[f];
      if (!s.active) continue;
      const MachineOut mo = a.mo_res[f];
      if (mo.overflow) s.status |= kCtlCapacity;
      if (mo.n_max != kExpNone) {
        s.T32 = mo.total_bits;
        s.T24 = a.pl_res[(int64_t)f * kMaxPlaneRecs + kBasePlanes].start;
      }
      // (a pure-base probe may be in flight: the joint loop ingests it)
      for (int k = 0; k < kCtlSlots; k++) s.tpend[k] = -1;
    }
    return;
  }
  CtlChunk* cs = stage_in(a);
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    CtlChunk& s = cs[f];
    ProbeParam pp[kCtlSlots] = {};
    ProbeParam tp[kCtlSlots] = {};
    const bool do_p = a.jmode & 1, do_t = a.jmode & 2;
    if (s.active) {
      if (do_p) {
        if (s.pend) {
          memo_add(s, s.pend_budget, a.res[f], false);
          s.pend = 0;
        }
        ingest_spec(s, a, f, false);
      }
      if (do_t) {
        for (int k = 0; k < a.slots; k++)
          if (s.tpend[k] >= 0) tmemo_add(s, s.tpend_pi, s.tpend[k], a.tres[k * nf + f]);
        for (int k = 0; k < kCtlSlots; k++) s.tpend[k] = -1;
      }
      bool p_open = false, t_open = false;
      if (do_p && !s.done_p && !(s.status & kCtlCapacity) && adv_pure(s) == kSuspend) {
        s.pend = 1;
        s.pend_budget = s.want_p;
        pp[0] = base_request(s, s.want_p, P.early != 0);
        post_spec(s, a.bslots, s.want_p, pp,
                  [&](int64_t b) { return base_request(s, b, P.early != 0); });
        p_open = true;
      }
      if (do_t && !s.done_t && !(s.status & kCtlCapacity) && adv_trunc(s) == kSuspend) {
        s.tpend_pi = s.pass;
        s.tpend[0] = s.want_t;
        tp[0] = trunc_request(s, a, f, s.pass, s.want_t, P.early != 0);
        // speculative slots: points the next step needs whichever way this
        // probe answers (same planes variant)
        for (int k = 0; k + 1 < a.slots && k < 2; k++) {
          const int64_t t2 = s.spec[k];
          if (t2 < 0 || t2 == s.want_t || tmemo_find(s, s.pass, t2) >= 0) continue;
          s.tpend[k + 1] = t2;
          tp[k + 1] = trunc_request(s, a, f, s.pass, t2, P.early != 0);
        }
        t_open = true;
      }
      if (P.prune && (p_open || t_open)) {
        // candidate pruning (pipeline.py:315-329 picks min((len, 0|1))): stop
        // a search whose candidate can no longer win; same chosen candidate
        const int64_t base_len = stream_len(s, s.base_budget);
        int64_t two_ub = -1, pure_ub = -1;
        if (s.trunc_planes) two_ub = base_len + kHeader + s.trunc_t;
        else if (t_open && s.t_ub >= 0) two_ub = base_len + kHeader + s.t_ub;
        if (s.done_p && s.pure_budget >= 0) pure_ub = stream_len(s, s.pure_budget);
        else if (p_open && s.p_ub >= 0) pure_ub = s.p_ub;
        const int64_t two_lb = base_len + kHeader + (t_open ? s.t_lb : 0);
        if (p_open && two_ub >= 0 && s.p_lb > two_ub) {
          s.done_p = 1;  // the two-layer candidate is strictly shorter
          s.pure_budget = -1;
          s.pure_pruned = 1;
          s.pend = 0;
          for (int k = 0; k < kCtlSlots; k++) pp[k] = ProbeParam{};
          for (int k = 0; k + 1 < kCtlSlots; k++) s.bspend[k] = -1;
          p_open = false;
        } else if (t_open && pure_ub >= 0 && two_lb >= pure_ub) {
          s.done_t = 1;  // pure-base is no longer (ties go to pure-base)
          s.trunc_pruned = 1;
          s.trunc_t = -1;
          s.trunc_planes = 0;
          for (int k = 0; k < kCtlSlots; k++) {
            s.tpend[k] = -1;
            tp[k] = ProbeParam{};
          }
          t_open = false;
        }
      }
      anyp |= p_open;
      anyt |= t_open;
    }
    for (int k = 0; do_p && k < a.bslots; k++) {
      a.prm[k * nf + f] = pp[k];
      a.res[k * nf + f] = ProbeResult{};
    }
    for (int k = 0; do_t && k < a.slots; k++) {
      a.tprm[k * nf + f] = tp[k];
      a.tres[k * nf + f] = ProbeResult{};
    }
  }
  stage_out(a);
  anyp = block_any(anyp);
  anyt = block_any(anyt);
  if (threadIdx.x == 0) {
    bool loop = anyp || anyt;
    // the pure-only loop stops once the residual is encoded; its last posted
    // probes still run (h_pure), and the joint loop ingests them
    if (a.jmode == 1 && *reinterpret_cast<volatile unsigned long long*>(&a.stats->stop)) loop = false;
    if (set & 1) cudaGraphSetConditional(a.h_loop, loop ? 1u : 0u);
    if (set & 2) cudaGraphSetConditional(a.h_pure, anyp ? 1u : 0u);
    if (set & 4) cudaGraphSetConditional(a.h_trunc, anyt ? 1u : 0u);
    a.stats->joint_steps++;
    if (anyp) a.stats->pure_probes++;
    if (anyt) a.stats->trunc_probes++;
  }
}

__global__ void __launch_bounds__(1024) ctl_finalize_kernel(CtlArgs a) {
  for (int f = threadIdx.x; f < a.nfields; f += blockDim.x) {
    const CtlChunk& s = a.cs[f];
    CtlOut o{};
    o.status = s.status;
    o.active = s.active;
    o.base_budget = s.base_budget;
    o.pure_budget = s.pure_budget;
    o.trunc_t = s.trunc_t;
    o.trunc_planes = s.trunc_planes;
    o.n_base_probes = s.nmemo;
    o.n_trunc_probes = s.ntcalls;
    o.pure_pruned = s.pure_pruned;
    o.trunc_pruned = s.trunc_pruned;
    o.T_base = s.T_base;
    o.T24 = s.T24;
    o.T32 = s.T32;
    o.len_base = s.active && s.base_budget >= 0 ? stream_len(s, s.base_budget) : -1;
    o.len_pure = s.active && s.pure_budget >= 0 ? stream_len(s, s.pure_budget) : -1;
    a.out[f] = o;
  }
}

inline int ctl_threads(int nfields) {
  int t = 32;
  while (t < nfields && t < 1024) t *= 2;
  return t;
}
// staged launches: more threads for the copies, the states' bytes of smem
inline int ctl_threads(const CtlArgs& a) { return a.smem ? 256 : ctl_threads(a.nfields); }
inline size_t ctl_smem(const CtlArgs& a) { return a.smem ? sizeof(CtlChunk) * a.nfields : 0; }
void ctl_smem_init() {
  static bool done = false;
  if (done) return;
  const int bytes = (int)(sizeof(CtlChunk) * kCtlSmemChunks);
  cudaFuncSetAttribute(ctl_base_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(ctl_joint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done = true;
}

}  // namespace

void ctl_setup(const CtlArgs& a, cudaStream_t st) {
  ctl_setup_kernel<<<1, ctl_threads(a.nfields), 0, st>>>(a);
}
bool ctl_smem_ok(int nfields) { return nfields <= kCtlSmemChunks; }
void ctl_base(const CtlArgs& a, bool start, int set, cudaStream_t st) {
  ctl_smem_init();
  ctl_base_kernel<<<1, ctl_threads(a), ctl_smem(a), st>>>(a, start ? 1 : 0, set);
}
void ctl_residue(const CtlArgs& a, cudaStream_t st) {
  ctl_residue_kernel<<<1, ctl_threads(a.nfields), 0, st>>>(a);
}
void ctl_joint(const CtlArgs& a, bool start, int set, cudaStream_t st) {
  ctl_smem_init();
  ctl_joint_kernel<<<1, ctl_threads(a), start ? 0 : ctl_smem(a), st>>>(a, start ? 1 : 0, set);
}
void ctl_finalize(const CtlArgs& a, cudaStream_t st) {
  ctl_finalize_kernel<<<1, ctl_threads(a.nfields), 0, st>>>(a);
}

}  // namespace ebcc
