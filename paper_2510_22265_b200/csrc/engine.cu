// Host runtime of the EBCC B200 path: device workspace, the batched feedback
// controller, and the C ABI declared in include/ebcc_gpu.h.
//
// Controller design.  The reference's searches (pipeline.py:142-254) are
// sequential and data dependent, and the emitted bytes depend on visiting
// exactly the same budgets in the same order.  Each chunk's
// search is therefore written here as ordinary straight-line code over a
// memo, restated from the reference; a memo miss throws NeedProbe.  Every
// step the controller *replays* each chunk's search from the top against its
// memo (microseconds of host work), collects the one missing probe per chunk,
// runs all of them as ONE batched device probe (decode -> IDWT -> reduction
// for every chunk at once), stores the two scalars per chunk, and repeats.
// The memo keeps insertion order so that replays see the exact snapshot the
// reference's dict iteration would (pipeline.py:193-198, 227-234).
//
// Phase order per chunk: base search, pure-base search, residual encode,
// truncation search.  The reference runs the truncation search before the
// pure search, but the truncation search never touches the base memo, so
// the order is observably identical, and running both base-memo searches
// first lets the residual encode reuse the base coefficient metadata arrays.
#include <omp.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ebcc_gpu.h"
#include "dwt.cuh"
#include "idwt_fused.cuh"
#include "ebcot.cuh"
#include "probe.cuh"
#include "spiht.cuh"
#include "ctx.cuh"
#include "ctl.cuh"

using namespace ebcc;

namespace {

constexpr int kBasePlanes = 24;   // spiht.DEFAULT_PLANES
constexpr int kDeepPlanes = 32;   // spiht.DEEP_PLANES

struct CudaFail {
  cudaError_t e;
  const char* what;
};

#define CK_STR2(x) #x
#define CK_STR(x) CK_STR2(x)
#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) throw CudaFail{e_, "engine.cu:" CK_STR(__LINE__) " " #x}; \
  } while (0)

// workspace allocations add their size here (Workspace::bytes)
thread_local int64_t* g_alloc_acc = nullptr;

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  // 256 bytes of slack behind every workspace buffer (vector loads of a
  // buffer's last partial granule stay inside the allocation)
  cudaError_t e = cudaMalloc(&p, sizeof(T) * count + 256);
  if (e != cudaSuccess) throw CudaFail{e, "cudaMalloc"};
  if (g_alloc_acc) *g_alloc_acc += (int64_t)(sizeof(T) * count);
  return static_cast<T*>(p);
}
struct AllocScope {  // count the device allocations of this scope into `acc`
  int64_t* prev;
  explicit AllocScope(int64_t* acc) : prev(g_alloc_acc) { g_alloc_acc = acc; }
  ~AllocScope() { g_alloc_acc = prev; }
};

// host memcpy split over a thread team (first-touch page faults of a fresh
// destination are spread over the team too)
void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  // host staging copies (pageable <-> page-locked) of 10-150 MB: a persistent
  // OpenMP team (spawning threads per call cost ~0.5 ms per 16 MB copy)
  static const int T = (int)std::max(1u, std::min(std::thread::hardware_concurrency(), 16u));
  if (bytes < (4u << 20) || T <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  {  // a fresh destination (a new bytes object) faults in 2 MiB pages
    const uintptr_t a = ((uintptr_t)dst + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
    const uintptr_t b = ((uintptr_t)dst + bytes) & ~(uintptr_t)((2u << 20) - 1);
    if (b > a) madvise((void*)a, b - a, MADV_HUGEPAGE);
  }
  size_t step = (bytes + T - 1) / T;
  step = (step + 4095) & ~size_t(4095);
#pragma omp parallel for num_threads(T) schedule(static)
  for (int t = 0; t < T; t++) {
    const size_t lo = (size_t)t * step;
    if (lo < bytes) memcpy((char*)dst + lo, (const char*)src + lo, std::min(step, bytes - lo));
  }
}

// fault in fresh pages with the thread team (one write per 4 KiB page)
void parallel_touch(void* dst, size_t bytes) {
  static const int T = (int)std::max(1u, std::min(std::thread::hardware_concurrency(), 16u));
  const size_t step = std::max<size_t>(((bytes + T - 1) / T + 4095) & ~size_t(4095), 4096);
#pragma omp parallel for num_threads(T) schedule(static)
  for (int t = 0; t < T; t++) {
    const size_t lo = (size_t)t * step;
    const size_t hi = std::min(bytes, lo + step);
    for (size_t o = lo; o < hi; o += 4096) static_cast<volatile char*>(dst)[o] = 0;
  }
}

bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// truncation probes per chunk and step: the bisection's next midpoint plus
// the two points one level further (one of which the next step needs)
constexpr int kTruncSlots = kCtlSlots;
// batches up to this many points speculate (slots beside each bisection
// midpoint): the GPU has slack at that size
constexpr int64_t kSpecPoints = 8ll << 20;
// ... and up to these the base / pure-base searches speculate too (measured:
// 1 or 2 fields of 721 x 1440 gain, 4 lose), and the pure-base search runs
// beside the residual encode (1 field gains, 2 lose)
constexpr int64_t kSpecBasePoints = 5ll << 19;
constexpr int64_t kSplitPoints = 5ll << 18;
struct IngestFail {};

// ---------------------------------------------------------------------------
struct Workspace {
  Geo g{};
  int cap = 0;  // fields
  // batches of at most spec_cap fields run kCtlSlots base-stream probes per
  // step (speculation); the base probe slots are sized for np0 probes
  int spec_cap = 0;
  int64_t np0 = 0;
  int64_t bytes = 0;  // device bytes held (allocations counted by AllocScope)
  float* x32 = nullptr;
  double *norm = nullptr, *A = nullptr, *B = nullptr, *base_dec = nullptr;
  int16_t *ec = nullptr, *ed = nullptr, *el = nullptr;
  uint32_t *mant = nullptr, *sign_pos = nullptr, *lsp_rank = nullptr;
  uint8_t* pinfo = nullptr;
  uint8_t* hrel = nullptr;
  uint2* packed = nullptr;
  uint2* packed2 = nullptr;      // residual metadata (built while the pure search runs)
  uint8_t* rank_hi = nullptr;    // wide chunks (probe.cuh): rank bits 26..31, base / residual
  uint8_t* rank_hi2 = nullptr;
  uint32_t* sprank = nullptr;    // sign bit offsets by LSP rank (base / residual)
  uint32_t* sprank2 = nullptr;
  double *A2 = nullptr, *B2 = nullptr;  // residual forward-DWT scratch
  uint64_t *lip = nullptr, *lis0 = nullptr, *lis1 = nullptr, *w0 = nullptr, *w1 = nullptr;
  uint32_t* lsp = nullptr;
  uint64_t* ninfo = nullptr;
  uint32_t *bits_base = nullptr, *bits_res = nullptr;
  int64_t words_base = 0, words_res = 0;
  PlaneRec *pl_base = nullptr, *pl_res = nullptr;
  MachineOut *mo_base = nullptr, *mo_res = nullptr;
  FieldScal* fs = nullptr;
  ProbeParam* prm = nullptr;
  ProbeResult* res = nullptr;
  uint8_t* tq_base = nullptr;  // per-probe decode tables (Meta::tq)
  uint8_t* tq_res = nullptr;
  uint64_t* limit = nullptr;
  uint8_t* active = nullptr;
  // incremental probes (probe.cuh): per stream (0 base, 1 residual) the
  // persistent LL levels, node by LSP rank, tile flags/results, plans, states
  double* Linc[2] = {nullptr, nullptr};
  uint32_t* lspn[2] = {nullptr, nullptr};
  uint8_t* iflags[2] = {nullptr, nullptr};
  TileStat* its[2] = {nullptr, nullptr};
  IncPlan* iplan[2] = {nullptr, nullptr};
  IncState* istate[2] = {nullptr, nullptr};
  unsigned long long* icomputed = nullptr;  // [2][kMaxLevels]
  int64_t inc_tiles = 0, inc_tiles0 = 0, inc_lstride = 0;
  // decompress: a second decoder state so the residual stream decodes
  // concurrently with the base stream (allocated on first use)
  struct DecSet {
    uint32_t *mant = nullptr, *sign_pos = nullptr, *lsp_rank = nullptr, *lsp = nullptr;
    uint8_t* pinfo = nullptr;
    uint64_t *lip = nullptr, *lis0 = nullptr, *lis1 = nullptr, *w0 = nullptr, *w1 = nullptr;
    uint64_t* limit = nullptr;
    uint8_t* active = nullptr;
  } dec2;
  unsigned int* mm = nullptr;
  // opt-in J2 base layer (ebcot.cuh), allocated on first use
  struct EbSet {
    EbBufs b{};
    EbGeo geo{};
    int32_t* blk_of = nullptr;
    EbBlock* blocks = nullptr;
    uint64_t* body_len = nullptr;
    double* ll = nullptr;  // second LL buffer of the fused probe levels (with B)
  } eb;
  // pinned host mirrors of the per-step control arrays
  TreeTables tt{};
  bool has_tt = false;
  // device controller (ctl.cuh): per-chunk search state, results, params
  CtlChunk* ctl = nullptr;
  CtlOut* ctl_out = nullptr;
  CtlParams* ctl_prm = nullptr;
  CtlStats* ctl_stats = nullptr;
  CtlOut* h_ctl_out = nullptr;     // pinned mirrors read once per batch
  FieldScal* h_fs = nullptr;
  CtlStats* h_ctl_stats = nullptr;
  CtlParams* h_ctl_prm = nullptr;
  MachineOut* h_mo = nullptr;      // base then residual machine outputs (2 x cap)
  // instantiated search graphs of this workspace, by batch shape
  struct SearchGraph {
    cudaGraphExec_t exec = nullptr;
    int nf = -1, slots = 0, prune = -1, early = -1, inc = -1, cluster = -1, j2 = -1;
  };
  std::vector<SearchGraph> graphs;

  void release() {
    for (SearchGraph& sg : graphs)
      if (sg.exec) cudaGraphExecDestroy(sg.exec);
    graphs.clear();
    void* cp[] = {ctl, ctl_out, ctl_prm, ctl_stats};
    for (void* p : cp)
      if (p) cudaFree(p);
    void* hp[] = {h_ctl_out, h_fs, h_ctl_stats, h_ctl_prm, h_mo};
    for (void* p : hp)
      if (p) cudaFreeHost(p);
    void* ptrs[] = {x32, norm, A, B, base_dec, ec, ed, el, mant, sign_pos, lsp_rank, pinfo, hrel,
                    packed, ninfo, rank_hi, rank_hi2,
                    packed2, sprank, sprank2, A2, B2,
                    lip, lis0, lis1, w0, w1, lsp, bits_base, bits_res, pl_base, pl_res,
                    mo_base, mo_res, fs, prm, res, tq_base, tq_res, limit, active, mm};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    for (int i = 0; i < 2; i++) {
      void* ip[] = {Linc[i], lspn[i], iflags[i], its[i], iplan[i], istate[i]};
      for (void* p : ip)
        if (p) cudaFree(p);
    }
    if (icomputed) cudaFree(icomputed);
    void* d2[] = {dec2.mant, dec2.sign_pos, dec2.lsp_rank, dec2.lsp, dec2.pinfo, dec2.lip,
                  dec2.lis0, dec2.lis1, dec2.w0, dec2.w1, dec2.limit, dec2.active};
    for (void* p : d2)
      if (p) cudaFree(p);
    if (has_tt) free_tree_tables(tt);
    void* ebp[] = {eb.b.qs, eb.b.flags, eb.b.plow, eb.b.cw, eb.b.uval, eb.b.uoff, eb.b.ztab,
                   eb.b.cum, eb.b.nmax, eb.b.status, eb.blk_of, eb.blocks, eb.body_len, eb.ll};
    for (void* p : ebp)
      if (p) cudaFree(p);
    *this = Workspace{};
  }
};

int64_t words_for(int64_t n, int planes) {
  // per plane <= |LIP|+|LSP| (<= n) + LIS bits (<= 2n/3); plus children and
  // sign bits (<= 2n over the whole stream)
  int64_t bits = (int64_t)planes * (n + (2 * n) / 3 + 8) + 2 * n + 1024;
  return bits / 32 + 64;
}

}  // namespace

struct ebcc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int64_t err_index = -1;   // flat element index of the last EBCC_E_INGEST
  Workspace ws;
  // workspaces of other chunk shapes, kept for reuse (calls alternating
  // between shapes - custom chunking, edge chunks - would otherwise free and
  // reallocate several GB per call); most recently parked last
  std::vector<Workspace> ws_cache;
  // pinned staging for pageable host buffers (copied by a thread team)
  uint8_t* h_stage = nullptr;
  // page-locked arena for the small host->device parameter copies of one
  // call: a pageable source would make cudaMemcpyAsync wait for the stream,
  // tying the host to the GPU at every copy
  uint8_t* h_arena = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  int64_t h_stage_cap = 0;
  // last compress result
  uint8_t* d_payload = nullptr;
  int64_t payload_cap = 0, payload_total = 0;
  PackPart* d_parts = nullptr;
  int parts_cap = 0;
  UnpackPart* d_unpack = nullptr;
  int unpack_cap = 0;
  uint8_t* d_stage = nullptr;
  int64_t stage_cap = 0;
  uint8_t* h_pay = nullptr;       // decompress: page-locked copy of a pageable payload
  int64_t h_pay_cap = 0;
  float* d_out = nullptr;
  int64_t out_cap = 0;
  // double buffers of the batch pipelines: compress stages batch i+1's
  // pageable input while batch i computes; decompress alternates its device
  // output and payload staging so batch i's device->host copy overlaps batch
  // i+1's decoders (ev_buf[k]: the last copy out of / into buffer k is done)
  uint8_t* h_stage2 = nullptr;
  int64_t h_stage2_cap = 0;
  uint8_t* h_pay2 = nullptr;
  int64_t h_pay2_cap = 0;
  float* d_out2 = nullptr;
  int64_t out2_cap = 0;
  cudaEvent_t ev_obuf[2] = {};
  cudaEvent_t ev_pbuf[2] = {};
  float* d_in2 = nullptr;         // compress: the next batch's input (device)
  int64_t in2_cap = 0;
  cudaEvent_t ev_in2 = nullptr, ev_in2_used = nullptr;
  uint8_t* d_cont = nullptr;      // container image (ebcc_fetch_container)
  int64_t cont_cap = 0;
  uint8_t* d_cmeta = nullptr;     // its records + parts
  int64_t cmeta_cap = 0;
  ebcc_stats stats{};
  fused::Level0Timer l0;
  cudaStream_t side = nullptr;   // high-priority stream for the overlapped residual encode
  cudaStream_t copy = nullptr;   // decompress: device->host copies of finished field groups
  cudaEvent_t ev_copy = nullptr;
  cudaEvent_t ev_in = nullptr;   // lanes: this lane's input copy has landed (CopyChain)
  std::vector<cudaEvent_t> ev_groups;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;
  cudaEvent_t ph[5] = {};  // EBCC_PROFILE=1: search-graph phase marks
  cudaEvent_t ev_f0 = nullptr, ev_f1 = nullptr;  // fork/join of the joint probe step
  cudaEvent_t cev0 = nullptr, cev1 = nullptr;    // per-call timing (batch loop)
  cudaEvent_t oev0 = nullptr, oev1 = nullptr;    // per-call timing (ebcc_compress)
  cudaEvent_t tm_a = nullptr, tm_b = nullptr;
  cudaStream_t cap[6] = {};      // graph capture streams (created on first use)
  cudaEvent_t tev[2] = {};       // base-encode timing
  cudaStream_t join = nullptr;   // caller's default stream the library stream follows
  cudaEvent_t ev_join = nullptr;
  std::vector<ebcc_ctx*> lanes;  // child contexts for concurrent sub-batches
  int machine_fields = 0;        // lanes: chunks whose machines run concurrently in total
  int last_batch = 0;            // chunks of the last compress batch (dev probe bench)
  // batch plans (chunks per device batch), cached per call shape so that
  // repeated calls neither query the free memory nor reallocate
  struct Plan {
    int rows = 0, cols = 0, levels = 0, lanes = 0, j2 = 0;
    int64_t nfields = -1, cap = 0;
    bool matches(const Geo& g, int64_t nf, int l, int j = 0) const {
      return rows == g.rows && cols == g.cols && levels == g.levels && nfields == nf && lanes == l &&
             j2 == j;
    }
  } cplan, dplan;
};

namespace {

// graph capture streams of a context (created on first use)
cudaStream_t cap_stream(ebcc_ctx* c, int k) {
  if (!c->cap[k]) CK(cudaStreamCreateWithFlags(&c->cap[k], cudaStreamNonBlocking));
  return c->cap[k];
}

// chunks past the 26-bit record rank keep rank bits 26..31 in a side byte
// (EBCC_WIDE_RECORDS=1 forces the layout for every chunk: parity tests)
bool wide_records(const Geo& g) {
  static const bool force = getenv("EBCC_WIDE_RECORDS") && getenv("EBCC_WIDE_RECORDS")[0] == '1';
  return force || g.n > kMaxNarrowPoints;
}

// make c->ws a workspace of geometry g holding at least nfields chunks; a
// new allocation takes max(nfields, want) chunks (want: the planned batch)
void ensure_workspace(ebcc_ctx* c, const Geo& g, int nfields, int want = 0) {
  Workspace& w = c->ws;
  bool same_geo = w.g.rows == g.rows && w.g.cols == g.cols && w.g.levels == g.levels;
  if (same_geo && w.cap >= nfields) return;
  if (!same_geo) {
    for (size_t i = 0; i < c->ws_cache.size(); i++) {
      Workspace& cw = c->ws_cache[i];
      if (cw.g.rows == g.rows && cw.g.cols == g.cols && cw.g.levels == g.levels) {
        if (cw.cap >= nfields) {
          // reuse it; the current one is parked as the most recently used
          Workspace found = cw;
          c->ws_cache.erase(c->ws_cache.begin() + i);
          if (w.cap > 0) c->ws_cache.push_back(w);
          w = found;
          return;
        }
        cw.release();  // too small for this call: never keep two of a shape
        c->ws_cache.erase(c->ws_cache.begin() + i);
        break;
      }
    }
    if (w.cap > 0) {  // park the current workspace, evicting the oldest
      static const size_t kKeep = getenv("EBCC_WS_CACHE") ? (size_t)atoi(getenv("EBCC_WS_CACHE")) : 3;
      c->ws_cache.push_back(w);
      w = Workspace{};
      while (c->ws_cache.size() > kKeep) {
        c->ws_cache.front().release();
        c->ws_cache.erase(c->ws_cache.begin());
      }
    }
  }
  int cap = std::max(std::max(nfields, want), same_geo ? w.cap : 0);
  w.release();
  w.g = g;
  w.cap = cap;
  AllocScope acc(&w.bytes);
  const int64_t N = g.n * cap;
  w.x32 = dalloc<float>(N);
  w.norm = dalloc<double>(N);
  w.A = dalloc<double>(N);
  w.B = dalloc<double>(N);
  w.base_dec = dalloc<double>(N);
  w.ec = dalloc<int16_t>(N);
  w.ed = dalloc<int16_t>(N);
  w.el = dalloc<int16_t>(N);
  w.mant = dalloc<uint32_t>(N);
  w.sign_pos = dalloc<uint32_t>(N);
  w.lsp_rank = dalloc<uint32_t>(N);
  w.pinfo = dalloc<uint8_t>(N);
  w.hrel = dalloc<uint8_t>((size_t)((g.n + 15) & ~15ll) * cap + 16);  // 16-B aligned per field
  w.packed = dalloc<uint2>(N);
  w.packed2 = dalloc<uint2>(N);
  if (wide_records(g)) {
    w.rank_hi = dalloc<uint8_t>(N);
    w.rank_hi2 = dalloc<uint8_t>(N);
  }
  w.sprank = dalloc<uint32_t>(N);
  w.sprank2 = dalloc<uint32_t>(N);
  w.A2 = dalloc<double>(N);
  w.B2 = dalloc<double>(N);
  w.lip = dalloc<uint64_t>(N);
  w.lis0 = dalloc<uint64_t>(N);
  w.lis1 = dalloc<uint64_t>(N);
  w.w0 = dalloc<uint64_t>(N);
  w.w1 = dalloc<uint64_t>(N);
  w.lsp = dalloc<uint32_t>(N);
  w.ninfo = dalloc<uint64_t>(N);
  w.words_base = words_for(g.n, kBasePlanes);
  w.words_res = words_for(g.n, kMaxDecodePlanes > kDeepPlanes ? kDeepPlanes : kDeepPlanes);
  w.bits_base = dalloc<uint32_t>(w.words_base * cap);
  w.bits_res = dalloc<uint32_t>(w.words_res * cap);
  w.pl_base = dalloc<PlaneRec>((size_t)kMaxPlaneRecs * cap);
  w.pl_res = dalloc<PlaneRec>((size_t)kMaxPlaneRecs * cap);
  w.mo_base = dalloc<MachineOut>(cap);
  w.mo_res = dalloc<MachineOut>(cap);
  w.fs = dalloc<FieldScal>(cap);
  w.spec_cap = (int)std::min<int64_t>(cap, std::max<int64_t>(1, kSpecPoints / g.n));
  w.np0 = std::max<int64_t>(cap, (int64_t)kCtlSlots * w.spec_cap);
  // per-probe decode tables: base-stream probes, truncation probes
  w.tq_base = dalloc<uint8_t>((size_t)kTqBytes * w.np0);
  w.tq_res = dalloc<uint8_t>((size_t)kTqBytes * kTruncSlots * cap);
  // parameter/result slots: np0 base-stream probes, then kTruncSlots x cap
  // truncation probes
  w.prm = dalloc<ProbeParam>(w.np0 + kTruncSlots * (size_t)cap);
  w.res = dalloc<ProbeResult>(w.np0 + kTruncSlots * (size_t)cap);
  w.limit = dalloc<uint64_t>(cap);
  w.active = dalloc<uint8_t>(cap);
  w.mm = dalloc<unsigned int>(4 * cap + 2);
  inc_capacity(g, &w.inc_tiles, &w.inc_tiles0);
  w.inc_lstride = g.levels > 1 ? (int64_t)g.lr[1] * g.cols : 1;
  for (int i = 0; i < 2; i++) {
    const size_t np = i ? (size_t)cap * kTruncSlots : (size_t)w.np0;  // probes per step
    w.Linc[i] = dalloc<double>((size_t)w.inc_lstride * np);
    w.lspn[i] = dalloc<uint32_t>(N);
    w.iflags[i] = dalloc<uint8_t>((size_t)w.inc_tiles * np);
    w.its[i] = dalloc<TileStat>((size_t)w.inc_tiles0 * np);
    w.iplan[i] = dalloc<IncPlan>(np);
    w.istate[i] = dalloc<IncState>(np);
    CK(cudaMemset(w.iflags[i], kTileDirty, (size_t)w.inc_tiles * np));
  }
  w.icomputed = dalloc<unsigned long long>(2 * kMaxLevels);
  w.ctl = dalloc<CtlChunk>(cap);
  w.ctl_out = dalloc<CtlOut>(cap);
  w.ctl_prm = dalloc<CtlParams>(1);
  w.ctl_stats = dalloc<CtlStats>(1);
  CK(cudaMallocHost(&w.h_ctl_out, sizeof(CtlOut) * cap));
  CK(cudaMallocHost(&w.h_fs, sizeof(FieldScal) * cap));
  CK(cudaMallocHost(&w.h_ctl_stats, sizeof(CtlStats)));
  CK(cudaMallocHost(&w.h_ctl_prm, sizeof(CtlParams)));
  CK(cudaMallocHost(&w.h_mo, sizeof(MachineOut) * 2 * cap));
  build_tree_tables(g, w.tt, c->stream);
  w.has_tt = true;
}

MachineBufs machine_bufs(Workspace& w, int nfields, bool residual) {
  MachineBufs mb{};
  mb.nfields = nfields;
  mb.stride = w.g.n;
  mb.bit_stride = residual ? w.words_res : w.words_base;
  mb.ec = w.ec; mb.ed = w.ed; mb.el = w.el;
  mb.mant = w.mant; mb.sign_pos = w.sign_pos; mb.lsp_rank = w.lsp_rank; mb.pinfo = w.pinfo;
  mb.lip = w.lip; mb.lis0 = w.lis0; mb.lis1 = w.lis1; mb.w0 = w.w0; mb.w1 = w.w1; mb.lsp = w.lsp;
  mb.ninfo = w.ninfo;
  mb.hrel = w.hrel;
  mb.ginfo = w.tt.ginfo;
  mb.bits = residual ? w.bits_res : w.bits_base;
  mb.planes = residual ? w.pl_res : w.pl_base;
  mb.out = residual ? w.mo_res : w.mo_base;
  mb.limit = w.limit;
  mb.active = w.active;
  return mb;
}

void ensure_dec2(Workspace& w) {
  if (w.dec2.mant) return;
  AllocScope acc(&w.bytes);
  const size_t N = (size_t)w.g.n * w.cap;
  w.dec2.mant = dalloc<uint32_t>(N);
  w.dec2.sign_pos = dalloc<uint32_t>(N);
  w.dec2.lsp_rank = dalloc<uint32_t>(N);
  w.dec2.lsp = dalloc<uint32_t>(N);
  w.dec2.pinfo = dalloc<uint8_t>(N);
  w.dec2.lip = dalloc<uint64_t>(N);
  w.dec2.lis0 = dalloc<uint64_t>(N);
  w.dec2.lis1 = dalloc<uint64_t>(N);
  w.dec2.w0 = dalloc<uint64_t>(N);
  w.dec2.w1 = dalloc<uint64_t>(N);
  w.dec2.limit = dalloc<uint64_t>(w.cap);
  w.dec2.active = dalloc<uint8_t>(w.cap);
}

// the residual decoder's state (decompress)
MachineBufs machine_bufs_dec2(Workspace& w, int nfields) {
  MachineBufs mb = machine_bufs(w, nfields, true);
  mb.mant = w.dec2.mant; mb.sign_pos = w.dec2.sign_pos; mb.lsp_rank = w.dec2.lsp_rank;
  mb.pinfo = w.dec2.pinfo; mb.lsp = w.dec2.lsp;
  mb.lip = w.dec2.lip; mb.lis0 = w.dec2.lis0; mb.lis1 = w.dec2.lis1;
  mb.w0 = w.dec2.w0; mb.w1 = w.dec2.w1;
  mb.limit = w.dec2.limit;
  mb.active = w.dec2.active;
  return mb;
}

Meta meta_of(Workspace& w, bool residual) {
  Meta m{};
  m.packed = residual ? w.packed2 : w.packed;
  m.rank_hi = residual ? w.rank_hi2 : w.rank_hi;
  m.sprank = residual ? w.sprank2 : w.sprank;
  m.planes = residual ? w.pl_res : w.pl_base;
  m.mo = residual ? w.mo_res : w.mo_base;
  m.stride = w.g.n;
  m.tq = residual ? w.tq_res : w.tq_base;
  return m;
}

// encode the pyramid currently in w.A (all fields): exponents, machine,
// refinement.  Returns per-field machine summaries and plane records.
struct PhaseClock;
void pc_mark(PhaseClock* pc, const char* name);
PhaseClock* g_pc = nullptr;
// EBCC_PROFILE=1: host-side split of the base/pure probe steps
struct StepProf {
  int64_t n = 0;
  double prep = 0, launch = 0, wait = 0, post = 0, timer = 0;
};
StepProf g_sp;
// EBCC_TRACE=1: per-lane host timeline of one compress (step completions,
// no extra synchronisation), printed when the call returns
struct Trace {
  bool on = false;
  std::mutex mu;
  std::chrono::steady_clock::time_point t0;
  struct Ev { int lane; const char* what; int i; double ms; };
  std::vector<Ev> ev;
  Trace() { on = getenv("EBCC_TRACE") && getenv("EBCC_TRACE")[0] == '1'; }
  void start() {
    if (!on) return;
    std::lock_guard<std::mutex> lk(mu);
    ev.clear();
    t0 = std::chrono::steady_clock::now();
  }
  void add(int lane, const char* what, int i) {
    if (!on) return;
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::lock_guard<std::mutex> lk(mu);
    ev.push_back({lane, what, i, ms});
  }
  void dump() {
    if (!on) return;
    std::lock_guard<std::mutex> lk(mu);
    for (int lane = 0; lane < 8; lane++) {
      std::string line;
      const char* prev = nullptr;
      int run = 0;
      double first = 0, lastms = 0;
      auto flush = [&]() {
        if (!prev) return;
        char b[96];
        if (run > 1) snprintf(b, sizeof b, " %s x%d [%.2f..%.2f]", prev, run, first, lastms);
        else snprintf(b, sizeof b, " %s@%.2f", prev, lastms);
        line += b;
      };
      for (auto& e : ev) {
        if (e.lane != lane) continue;
        if (prev && strcmp(prev, e.what) == 0) { run++; lastms = e.ms; continue; }
        flush();
        prev = e.what; run = 1; first = lastms = e.ms;
      }
      flush();
      if (!line.empty()) fprintf(stderr, "[ebcc trace lane %d]%s\n", lane, line.c_str());
    }
  }
};
Trace g_trace;
thread_local int g_lane = 0;

// EBCC_SLOWLOG=<ms>: report host intervals longer than that (tail-latency hunt)
struct SlowLog {
  double thr = -1;
  std::chrono::steady_clock::time_point last;
  SlowLog() {
    if (const char* e = getenv("EBCC_SLOWLOG")) thr = atof(e);
    last = std::chrono::steady_clock::now();
  }
  bool on() const { return thr >= 0; }
  void mark(const char* what, int i = -1) {
    g_trace.add(g_lane, what, i);
    if (thr < 0) return;
    auto now = std::chrono::steady_clock::now();
    double ms = std::chrono::duration<double, std::milli>(now - last).count();
    if (ms > thr) fprintf(stderr, "[ebcc slow] %s %d: %.2f ms\n", what, i, ms);
    last = now;
  }
};
thread_local SlowLog g_slow;
using SteadyClock = std::chrono::steady_clock;
inline double us_since(SteadyClock::time_point t) {
  return std::chrono::duration<double, std::micro>(SteadyClock::now() - t).count();
}

void h2d_small(ebcc_ctx* c, void* dst, const void* src, size_t n, cudaStream_t st);

// encode the pyramids in `coef` (all fields): exponents, machine (which
// skips all-zero pyramids itself), refinement, packed metadata.  Async on st.
// active == nullptr: the machine outputs and active flags were set on the
// device (ctl_setup) - nothing is copied from the host (graph-capturable)
void encode_launch(ebcc_ctx* c, int nfields, bool residual, int planes, const double* coef,
                   bool packed_residual, const std::vector<uint8_t>* active, cudaStream_t st,
                   int cluster = 0) {
  Workspace& w = c->ws;
  CK(cudaGetLastError());  // surface anything deferred from before this encode
  MachineBufs mb = machine_bufs(w, nfields, residual);
  // the stream's probe tables by LSP rank, written where the ranks are assigned
  mb.lsp = w.lspn[packed_residual ? 1 : 0];
  mb.sprank = packed_residual ? w.sprank2 : w.sprank;
  if (active) {
    std::vector<MachineOut> init(nfields);
    for (auto& m : init) { m = MachineOut{}; m.n_max = kExpNone; }
    h2d_small(c, mb.out, init.data(), sizeof(MachineOut) * nfields, st);
    h2d_small(c, w.active, active->data(), nfields, st);
  }
  CK(cudaMemsetAsync(mb.bits, 0, sizeof(uint32_t) * mb.bit_stride * nfields, st));
  coef_prepare(coef, w.g.n, mb, w.g, st);
  CK(cudaGetLastError());
  subtree_exponents(mb, w.g, w.tt, st);
  CK(cudaGetLastError());
  run_machine(false, mb, w.g, w.tt, planes, st, cluster);
  CK(cudaGetLastError());
  emit_lip(mb, planes, st);
  CK(cudaGetLastError());
  write_refinement(mb, planes, st);
  CK(cudaGetLastError());
  // (the encoder wrote the sign offsets and nodes by LSP rank itself:
  // MachineBufs::sprank, and its LSP list is the stream's lspn buffer)
  pack_meta(mb, packed_residual ? w.packed2 : w.packed, nullptr, st, nullptr,
            packed_residual ? w.rank_hi2 : w.rank_hi);
  c->stats.kernel_launches += 9 + w.g.levels;
  CK(cudaGetLastError());
}

// machine summaries + plane records of the last encode_launch (syncs st)
void encode_collect(ebcc_ctx* c, int nfields, bool residual, const std::vector<uint8_t>& active,
                    std::vector<MachineOut>& mo, std::vector<PlaneRec>& pl, cudaStream_t st) {
  MachineBufs mb = machine_bufs(c->ws, nfields, residual);
  CK(cudaMemcpyAsync(mo.data(), mb.out, sizeof(MachineOut) * nfields, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(pl.data(), mb.planes, sizeof(PlaneRec) * kMaxPlaneRecs * nfields,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int f = 0; f < nfields; f++)
    if (active[f] && mo[f].overflow) throw CudaFail{cudaErrorMemoryAllocation, "machine capacity"};
}

void encode_pyramids(ebcc_ctx* c, int nfields, bool residual, int planes,
                     const std::vector<uint8_t>& active, std::vector<MachineOut>& mo,
                     std::vector<PlaneRec>& pl) {
  // on the high-priority stream: the list machine needs whole SMs, and with
  // concurrent work (lanes) it must win them as they drain
  CK(cudaEventRecord(c->ev_a, c->stream));
  CK(cudaStreamWaitEvent(c->side, c->ev_a, 0));
  const int cluster = machine_cluster_size(false, std::max(nfields, c->machine_fields));
  encode_launch(c, nfields, residual, planes, c->ws.A, residual, &active, c->side, cluster);
  CK(cudaEventRecord(c->ev_b, c->side));
  CK(cudaStreamWaitEvent(c->stream, c->ev_b, 0));
  encode_collect(c, nfields, residual, active, mo, pl, c->stream);
}

void put_header(uint8_t* h, int n_max, int levels, int rows, int cols, bool j2 = false) {
  h[0] = j2 ? 'J' : 'S'; h[1] = j2 ? '2' : 'P';
  h[2] = (uint8_t)(int8_t)n_max;
  h[3] = (uint8_t)levels;
  uint32_t r = (uint32_t)rows, cc = (uint32_t)cols;
  memcpy(h + 4, &r, 4);
  memcpy(h + 8, &cc, 4);
}

// EBCC_PROFILE=1: host wall-clock per phase (stream synced at each mark)
struct PhaseClock {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0, last;
  std::string log;
  explicit PhaseClock(cudaStream_t s) : st(s) {
    const char* e = getenv("EBCC_PROFILE");
    on = e && *e == '1';
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* name) {
    if (!on) return;
    cudaStreamSynchronize(st);
    auto now = std::chrono::steady_clock::now();
    char buf[128];
    snprintf(buf, sizeof buf, " %s=%.2fms", name,
             std::chrono::duration<double, std::milli>(now - last).count());
    log += buf;
    last = now;
  }
  ~PhaseClock() {
    if (on && !log.empty()) fprintf(stderr, "[ebcc profile]%s\n", log.c_str());
    if (on && g_sp.n)
      fprintf(stderr, "[ebcc steps] base/pure steps %lld: per step prep %.1f launch %.1f wait %.1f "
              "post %.1f us\n", (long long)g_sp.n, g_sp.prep / g_sp.n, g_sp.launch / g_sp.n,
              g_sp.wait / g_sp.n, g_sp.post / g_sp.n);
    g_sp = StepProf{};
  }
};

void pc_mark(PhaseClock* pc, const char* name) {
  if (pc) pc->mark(name);
}

struct EventTimer {
  ebcc_ctx* c;
  double* acc;
  EventTimer(ebcc_ctx* c_, double* acc_);
  ~EventTimer();
};

EventTimer::EventTimer(ebcc_ctx* c_, double* acc_) : c(c_), acc(acc_) {
  cudaEventRecord(c->tm_a, c->stream);
}
EventTimer::~EventTimer() {
  cudaEventRecord(c->tm_b, c->stream);
  cudaEventSynchronize(c->tm_b);
  float ms = 0;
  cudaEventElapsedTime(&ms, c->tm_a, c->tm_b);
  *acc += ms;
}

// async H2D of a small host array through the page-locked arena
void arena_reset(ebcc_ctx* c) { c->arena_used = 0; }
void h2d_small(ebcc_ctx* c, void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return;
  size_t at = (c->arena_used + 63) & ~size_t(63);
  if (at + n > c->arena_cap) {
    // everything staged so far must have been consumed before reuse
    CK(cudaStreamSynchronize(c->stream));
    if (c->side) CK(cudaStreamSynchronize(c->side));
    at = 0;
    if (n > c->arena_cap) {
      if (c->h_arena) CK(cudaFreeHost(c->h_arena));
      c->h_arena = nullptr;
      c->arena_cap = 0;
      size_t cap = std::max<size_t>(n, 4u << 20);
      CK(cudaMallocHost(&c->h_arena, cap));
      c->arena_cap = cap;
    }
  }
  memcpy(c->h_arena + at, src, n);
  CK(cudaMemcpyAsync(dst, c->h_arena + at, n, cudaMemcpyHostToDevice, st));
  c->arena_used = at + n;
}

// a page-locked block of at least `bytes` held in (p, cap)
uint8_t* pinned_block(uint8_t*& p, int64_t& cap, int64_t bytes) {
  if (bytes > cap) {
    if (p) CK(cudaFreeHost(p));
    p = nullptr;
    cap = 0;
    CK(cudaMallocHost(&p, (size_t)bytes));
    cap = bytes;
  }
  return p;
}
template <class T>
T* device_block(T*& p, int64_t& cap, int64_t count) {
  if (count > cap) {
    if (p) CK(cudaFree(p));
    p = nullptr;
    cap = 0;
    p = dalloc<T>((size_t)count);
    cap = count;
  }
  return p;
}

uint8_t* host_stage(ebcc_ctx* c, int64_t bytes) {
  if (bytes > c->h_stage_cap) {
    if (c->h_stage) CK(cudaFreeHost(c->h_stage));
    c->h_stage = nullptr;
    c->h_stage_cap = 0;
    CK(cudaMallocHost(&c->h_stage, (size_t)bytes));
    c->h_stage_cap = bytes;
  }
  return c->h_stage;
}

// chunks per device batch: bounded by free HBM (and EBCC_MAX_BATCH, which the
// tests use to exercise the multi-batch path)
int64_t max_batch() {
  static const int64_t m = getenv("EBCC_MAX_BATCH") ? atoll(getenv("EBCC_MAX_BATCH")) : 4096;
  return m < 1 ? 1 : m;
}

// chunks per batch: free-memory bound, queried only when the workspace does
// not already cover the call (cudaMemGetInfo can stall for milliseconds)
int64_t plan_batch(ebcc_ctx* c, const Geo& g, int64_t want, int lanes, bool tree,
                   bool j2 = false);
int64_t balance(int64_t n, int64_t cap);

// feasibility-only probes may skip settled CTAs (EBCC_EARLY=0 disables)
bool early_ok() {
  static const bool on = !(getenv("EBCC_EARLY") && getenv("EBCC_EARLY")[0] == '0');
  return on;
}

// Add a conditional node (WHILE / IF on handle h) at the current capture
// point of `st` and capture its body from `bst` (a stream not capturing).
template <class F>
void add_conditional(cudaStream_t st, cudaStream_t bst, cudaGraphConditionalHandle h,
                     cudaGraphConditionalNodeType type, F fill) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t gr = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &gr, &deps, &nd));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = type;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, gr, deps, nd, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  CK(cudaStreamBeginCaptureToGraph(bst, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  fill(body, bst);
  cudaGraph_t out = nullptr;
  CK(cudaStreamEndCapture(bst, &out));
}

// the opt-in J2 base layer's buffers for nfields chunks of w's geometry
// (allocated on first use, for the workspace capacity); stream bodies live in
// bits_base (words_base words per chunk)
EbBufs& ensure_ebcot(Workspace& w, int nfields, cudaStream_t st) {
  Workspace::EbSet& e = w.eb;
  if (!e.blocks) {
    AllocScope acc(&w.bytes);  // (later batch plans see these bytes)
    e.geo = ebcot_build_geo(w.g, &e.blk_of, &e.blocks, st);
    CK(cudaGetLastError());
    const int64_t N = w.g.n * (int64_t)w.cap, nb = e.geo.nb, cap = w.cap;
    e.b.qs = dalloc<uint32_t>(N);
    e.b.flags = dalloc<uint16_t>(e.geo.state_stride * cap);
    e.b.plow = dalloc<int8_t>(N);
    e.b.cw_stride = w.g.n * kCwPerPoint + nb * kCwPerBlock;
    e.b.cw = dalloc<uint8_t>(cap * e.b.cw_stride);
    e.b.uval = dalloc<uint32_t>(cap * nb * kJ2Passes);
    e.b.uoff = dalloc<int64_t>(cap * nb * kJ2Passes);
    e.b.ztab = dalloc<uint8_t>(cap * nb);
    e.b.cum = dalloc<uint32_t>(cap * (kJ2Slots * nb + 1));
    e.b.nmax = dalloc<int32_t>(cap);
    e.b.status = dalloc<int32_t>(cap);
    e.body_len = dalloc<uint64_t>(cap);
    e.ll = dalloc<double>(N);
  }
  e.b.nfields = nfields;
  e.b.n = w.g.n;
  e.b.body = reinterpret_cast<uint8_t*>(w.bits_base);
  e.b.body_stride = w.words_base * 4;
  e.b.body_len = e.body_len;
  return e.b;
}

CtlArgs ctl_args(Workspace& w, int nfields, int slots) {
  CtlArgs a{};
  a.cs = w.ctl;
  a.out = w.ctl_out;
  a.prm_in = w.ctl_prm;
  a.stats = w.ctl_stats;
  a.fs = w.fs;
  a.mo_base = w.mo_base;
  a.mo_res = w.mo_res;
  a.pl_res = w.pl_res;
  a.active = w.active;
  a.prm = w.prm;
  a.res = w.res;
  a.tprm = w.prm + w.np0;
  a.tres = w.res + w.np0;
  a.nfields = nfields;
  a.slots = slots;
  a.bslots = 1;
  a.smem = ctl_smem_ok(nfields) ? 1 : 0;
  a.jmode = 3;
  a.n = w.g.n;
  return a;
}

// One compress batch of nfields (<= workspace capacity); x already in w.x32.
// in_groups > 0: the input arrives in that many field groups, group k
// complete when in_ev[k] fires (host input copied group by group); each
// group is normalised and transformed as soon as it lands.
//
// Eagerly enqueued: ingest + normalise, forward DWT, controller setup and
// the base encode.  Then ONE launch of the batch's search graph: the base
// quantile search (a conditional WHILE loop: controller step -> batched
// probe), the residue and the residual DWT + 32-plane encode, the joint
// pure-base + truncation searches (a WHILE loop whose two probe branches are
// IF nodes), and the copies of the candidate-choice inputs to the host.  The
// controller (ctl.cu) advances every chunk's search on the device and sets
// the loop conditions; the host synchronises once, after the graph, to pack
// the chosen prefixes.
int compress_batch(ebcc_ctx* c, int nfields, double eps_rel, double q, double r0, double tol,
                   bool prune,
                   ebcc_chunk_rec* recs, int64_t out_base_off, std::vector<PackPart>& parts,
                   std::vector<int64_t>& sizes, int in_groups = 0,
                   const cudaEvent_t* in_ev = nullptr, bool j2 = false) {
  Workspace& w = c->ws;
  const Geo& g = w.g;
  cudaStream_t st = c->stream;
  const int64_t N = g.n;
  c->last_batch = nfields;
  // ---- ingest + normalise (core.normalize) + forward DWT ----
  CK(cudaGetLastError());
  g_slow.mark("enter_batch");
  const bool grouped = in_groups > 0;
  if (!grouped) {
    ingest_normalize(w.x32, N, nfields, w.norm, w.fs, w.mm, eps_rel, st);
    forward_dwt_from(w.norm, w.A, w.B, N, nfields, g, st);
    c->stats.kernel_launches += 4 + 2 * g.levels;
  } else {
    // per group: normalise + forward DWT (the non-finite check is read after
    // the searches; a failing input only costs the wasted work)
    for (int k = 0; k < in_groups; k++) {
      const int a = (int)((int64_t)nfields * k / in_groups);
      const int b = (int)((int64_t)nfields * (k + 1) / in_groups);
      if (b <= a) continue;
      CK(cudaStreamWaitEvent(st, in_ev[k], 0));
      ingest_normalize(w.x32 + (int64_t)a * N, N, b - a, w.norm + (int64_t)a * N, w.fs + a,
                       w.mm + 4 * (int64_t)a, eps_rel, st);
      forward_dwt_from(w.norm + (int64_t)a * N, w.A + (int64_t)a * N, w.B + (int64_t)a * N, N,
                       b - a, g, st);
      c->stats.kernel_launches += 4 + 2 * g.levels;
    }
  }
  CK(cudaGetLastError());

  // ---- controller setup + base encode (eager, no host round trip) ----
  static const bool inc_env = !(getenv("EBCC_INC") && getenv("EBCC_INC")[0] == '0');
  static const int klim_div = getenv("EBCC_INC_KDIV") ? std::max(1, atoi(getenv("EBCC_INC_KDIV"))) : 16;
  // speculative truncation probes (the next bisection level's two points
  // beside each midpoint) while a lane's chunks leave the GPU slack
  // (EBCC_SPEC=1|2|3 forces the slot count)
  static const int spec_env =
      getenv("EBCC_SPEC") ? std::max(1, std::min(kTruncSlots, atoi(getenv("EBCC_SPEC")))) : 0;
  Inc inc_s[2];
  bool inc_ok = inc_env;
  for (int i = 0; i < 2; i++) {
    Inc& I = inc_s[i];
    I = Inc{};
    inc_ok = inc_geometry(g, nfields, I) && inc_ok;
    inc_ok = inc_ok && I.ig.tiles <= w.inc_tiles && I.ig.tiles0 <= w.inc_tiles0 &&
             (g.levels == 1 || I.lstride <= w.inc_lstride);
    I.flags = w.iflags[i];
    I.plan = w.iplan[i];
    I.state = w.istate[i];
    I.ts = w.its[i];
    I.lspn = w.lspn[i];
    I.computed = w.icomputed + i * kMaxLevels;
    I.klimit = (uint32_t)std::min<int64_t>(N / klim_div, 0xffffffffll);
    static const int dbg = getenv("EBCC_INC_LOG") ? atoi(getenv("EBCC_INC_LOG")) : 0;
    I.debug = dbg;
  }
  const Inc* inc_base = inc_ok ? &inc_s[0] : nullptr;
  const Inc* inc_res = inc_ok ? &inc_s[1] : nullptr;
  const int spec_auto = N * (int64_t)nfields <= kSpecPoints ? kTruncSlots : 1;
  const int TS = inc_res ? (spec_env ? spec_env : spec_auto) : 1;  // truncation probe slots
  const int ntp = TS * nfields;
  // base-stream probe slots: the base and pure-base searches speculate the
  // same way (SPIHT base, batches that fit the slot buffers)
  static const bool bspec_env = !(getenv("EBCC_BSPEC") && getenv("EBCC_BSPEC")[0] == '0');
  const int SB = (bspec_env && TS > 1 && !j2 && nfields <= w.spec_cap &&
                  N * (int64_t)nfields <= kSpecBasePoints) ? TS : 1;
  const int nbp = SB * nfields;
  *w.h_ctl_prm = CtlParams{q, r0, tol, prune ? 1 : 0, early_ok() ? 1 : 0, TS, 0};
  CK(cudaMemcpyAsync(w.ctl_prm, w.h_ctl_prm, sizeof(CtlParams), cudaMemcpyHostToDevice, st));
  CtlArgs a0 = ctl_args(w, nfields, TS);
  a0.bslots = SB;
  // opt-in J2 base layer (ebcot.cuh): its encoder, probes and residue
  EbBufs* eb = j2 ? &ensure_ebcot(w, nfields, st) : nullptr;
  const EbGeo egeo = w.eb.geo;
  Meta mj2{};  // J2 probes: the fused levels over the decoded f64 pyramid in A
  mj2.coef = w.A;
  mj2.mo = w.mo_base;
  mj2.stride = N;
  if (eb) {
    a0.eb_cum = eb->cum;
    a0.eb_nmax = eb->nmax;
    a0.eb_nb = egeo.nb;
  }
  ctl_setup(a0, st);
  const int cluster = machine_cluster_size(false, std::max(nfields, c->machine_fields));
  // on the high-priority stream: the list machine needs whole SMs, and with
  // concurrent work (lanes) it must win them as they drain
  CK(cudaEventRecord(c->ev_a, st));
  CK(cudaStreamWaitEvent(c->side, c->ev_a, 0));
  CK(cudaEventRecord(c->tev[0], c->side));
  if (eb) {
    ebcot_encode(w.A, egeo, g, *eb, w.active, c->side);
    ebcot_nmax_to(*eb, w.mo_base, c->side);
  } else {
    encode_launch(c, nfields, false, kBasePlanes, w.A, false, nullptr, c->side, cluster);
  }
  CK(cudaEventRecord(c->tev[1], c->side));
  CK(cudaEventRecord(c->ev_b, c->side));
  CK(cudaStreamWaitEvent(st, c->ev_b, 0));
  c->stats.kernel_launches += 2;
  g_slow.mark("base_encode_issued");

  // ---- the search graph (built once per batch shape of this workspace) ----
  const int early = early_ok() ? 1 : 0;
  Workspace::SearchGraph* sg = nullptr;
  for (Workspace::SearchGraph& x : w.graphs)
    if (x.nf == nfields && x.slots == TS && x.prune == (int)prune && x.early == early &&
        x.inc == (int)inc_ok && x.cluster == cluster && x.j2 == (int)j2)
      sg = &x;
  // EBCC_GRAPHS=0: the same sequence issued eagerly, the loop conditions read
  // back by the host after every controller step (profiling only: ncu does
  // not descend into conditional graph nodes)
  static const bool graphs = !(getenv("EBCC_GRAPHS") && getenv("EBCC_GRAPHS")[0] == '0');
  if (!graphs) {
    Meta mbase = meta_of(w, false), mres = meta_of(w, true);
    for (int i = 0; i < 2; i++)
      CK(cudaMemsetAsync(w.istate[i], 0, sizeof(IncState) * (i ? ntp : nbp), st));
    CK(cudaMemsetAsync(w.icomputed, 0, sizeof(unsigned long long) * 2 * kMaxLevels, st));
    auto base_probe = [&](bool early_p) {
      if (eb) {  // J2 base: closed-form prefix decode, then the fused probe levels
        ebcot_probe_decode(egeo, *eb, w.prm, nfields, nfields, w.A, st);
        probe_base(mj2, w.prm, w.B, w.eb.ll, g, nfields, w.norm, w.x32, w.fs, w.res, st,
                   nullptr, true, early_p);
        return;
      }
      probe_base(mbase, w.prm, inc_base ? w.Linc[0] : w.A, w.B, g, nbp, w.norm, w.x32,
                 w.fs, w.res, st, inc_base, false, early_p, nfields);
    };
    auto stats_now = [&]() {
      CK(cudaMemcpyAsync(w.h_ctl_stats, w.ctl_stats, sizeof(CtlStats), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      return *w.h_ctl_stats;
    };
    ctl_base(a0, true, 0, st);
    fused::g_level0_timer = &c->l0;
    base_probe(false);
    fused::g_level0_timer = nullptr;
    unsigned long long seen = stats_now().base_probes;
    for (;;) {
      ctl_base(a0, false, 0, st);
      const CtlStats cs = stats_now();
      if (cs.base_probes == seen) break;
      seen = cs.base_probes;
      base_probe(false);
    }
    ctl_residue(a0, st);
    if (eb) {
      ebcot_probe_decode(egeo, *eb, w.prm, nfields, nfields, w.A, st);
      base_to_residue(mj2, w.prm, w.B, w.eb.ll, g, nfields, w.norm, w.base_dec, w.norm, st);
    } else {
      // (like the probes: a normalised field's exponents stay in the normal range)
      base_to_residue(mbase, w.prm, w.A, w.B, g, nfields, w.norm, w.base_dec, w.norm, st, false);
    }
    forward_dwt_from(w.norm, w.A2, w.B2, N, nfields, g, st);
    CK(cudaEventRecord(c->ev_s0, st));
    encode_launch(c, nfields, true, kDeepPlanes, w.A2, true, nullptr, st, cluster);
    CK(cudaEventRecord(c->ev_s1, st));
    ctl_joint(a0, true, 0, st);
    CtlStats prev = stats_now();
    for (;;) {
      ctl_joint(a0, false, 0, st);
      const CtlStats cs = stats_now();
      const bool anyp = cs.pure_probes != prev.pure_probes;
      const bool anyt = cs.trunc_probes != prev.trunc_probes;
      prev = cs;
      if (!anyp && !anyt) break;
      if (anyt)
        probe_trunc(mres, w.prm + w.np0, inc_res ? w.Linc[1] : w.A2, w.B2, g, ntp, w.base_dec,
                    w.x32, w.fs, w.res + w.np0, st, inc_res, false, nfields);
      if (anyp) base_probe(true);
    }
    ctl_finalize(a0, st);
    CK(cudaMemcpyAsync(w.h_ctl_out, w.ctl_out, sizeof(CtlOut) * nfields, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(w.h_fs, w.fs, sizeof(FieldScal) * nfields, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(w.h_mo, w.mo_base, sizeof(MachineOut) * nfields, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(w.h_mo + w.cap, w.mo_res, sizeof(MachineOut) * nfields,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(w.h_ctl_stats, w.ctl_stats, sizeof(CtlStats), cudaMemcpyDeviceToHost, st));
  } else if (!sg) {
    Meta mbase = meta_of(w, false), mres = meta_of(w, true);
    cudaStream_t s0 = cap_stream(c, 0), s1 = cap_stream(c, 1), s2 = cap_stream(c, 2),
                 s3 = cap_stream(c, 3), s4 = cap_stream(c, 4), s5 = cap_stream(c, 5);
    CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
    cudaStreamCaptureStatus cst;
    cudaGraph_t top = nullptr;
    CK(cudaStreamGetCaptureInfo(s0, &cst, nullptr, &top, nullptr, nullptr));
    // incremental-probe state is invalid at the batch start
    for (int i = 0; i < 2; i++)
      CK(cudaMemsetAsync(w.istate[i], 0, sizeof(IncState) * (i ? ntp : nbp), s0));
    CK(cudaMemsetAsync(w.icomputed, 0, sizeof(unsigned long long) * 2 * kMaxLevels, s0));
    auto base_probe = [&](cudaStream_t ps, bool early_p) {
      if (eb) {  // J2 base: closed-form prefix decode, then the fused probe levels
        ebcot_probe_decode(egeo, *eb, w.prm, nfields, nfields, w.A, ps);
        probe_base(mj2, w.prm, w.B, w.eb.ll, g, nfields, w.norm, w.x32, w.fs, w.res, ps,
                   nullptr, true, early_p);
        return;
      }
      probe_base(mbase, w.prm, inc_base ? w.Linc[0] : w.A, w.B, g, nbp, w.norm, w.x32,
                 w.fs, w.res, ps, inc_base, false, early_p, nfields);
    };
    // base quantile search: start (T_base, first requests), the first probe
    // (its level-0 kernel timed for the roofline), then the loop
    fused::timer_record(c->ph[0], s0);
    CtlArgs ab = a0;
    ctl_base(ab, true, 0, s0);
    fused::g_level0_timer = &c->l0;
    base_probe(s0, false);
    fused::g_level0_timer = nullptr;
    cudaGraphConditionalHandle hb;
    CK(cudaGraphConditionalHandleCreate(&hb, top, 1, cudaGraphCondAssignDefault));
    add_conditional(s0, s1, hb, cudaGraphCondTypeWhile, [&](cudaGraph_t body, cudaStream_t bs) {
      cudaGraphConditionalHandle hp;
      CK(cudaGraphConditionalHandleCreate(&hp, body, 0, 0));
      CtlArgs al = a0;
      al.h_loop = hb;
      al.h_pure = hp;
      ctl_base(al, false, 3, bs);
      add_conditional(bs, s3, hp, cudaGraphCondTypeIf,
                      [&](cudaGraph_t, cudaStream_t is) { base_probe(is, false); });
    });
    // residue = norm - base decode at the chosen budget; residual DWT +
    // 32-plane encode (the 24-plane variant is its prefix)
    fused::timer_record(c->ph[1], s0);
    // small batches (speculating, the GPU has slack): the pure-base search
    // needs only the base stream, so it runs as its own loop beside the
    // residue, the residual DWT and the residual encode, and hands over to
    // the joint loop (candidate pruning) when the encode is done; the residue
    // decode takes its parameters and decode tables from the (idle)
    // truncation slots
    const bool split = SB > 1 && N * (int64_t)nfields <= kSplitPoints;
    if (split) {
      CK(cudaEventRecord(c->ev_f0, s0));
      CK(cudaStreamWaitEvent(s5, c->ev_f0, 0));
      cudaGraphConditionalHandle hq;
      CK(cudaGraphConditionalHandleCreate(&hq, top, 1, cudaGraphCondAssignDefault));
      add_conditional(s5, s1, hq, cudaGraphCondTypeWhile, [&](cudaGraph_t body, cudaStream_t bs) {
        cudaGraphConditionalHandle hp;
        CK(cudaGraphConditionalHandleCreate(&hp, body, 0, 0));
        CtlArgs al = a0;
        al.jmode = 1;
        al.h_loop = hq;
        al.h_pure = hp;
        ctl_joint(al, false, 3, bs);
        add_conditional(bs, s3, hp, cudaGraphCondTypeIf,
                        [&](cudaGraph_t, cudaStream_t is) { base_probe(is, true); });
      });
    }
    {
      CtlArgs ar = a0;
      Meta mr = mbase;
      if (split) {
        ar.prm = a0.tprm;
        mr.tq = w.tq_res;
      }
      ctl_residue(ar, s0);
      if (eb) {
        ebcot_probe_decode(egeo, *eb, ar.prm, nfields, nfields, w.A, s0);
        base_to_residue(mj2, ar.prm, w.B, w.eb.ll, g, nfields, w.norm, w.base_dec, w.norm, s0);
      } else {
        base_to_residue(mr, ar.prm, w.A, w.B, g, nfields, w.norm, w.base_dec, w.norm, s0, false);
      }
    }
    forward_dwt_from(w.norm, w.A2, w.B2, N, nfields, g, s0);
    fused::timer_record(c->ev_s0, s0);
    encode_launch(c, nfields, true, kDeepPlanes, w.A2, true, nullptr, s0, cluster);
    fused::timer_record(c->ev_s1, s0);
    if (split) {
      CK(cudaMemsetAsync(&w.ctl_stats->stop, 1, sizeof(unsigned long long), s0));
      fused::timer_record(c->ph[4], s5);
      CK(cudaEventRecord(c->ev_f1, s5));
      CK(cudaStreamWaitEvent(s0, c->ev_f1, 0));
    }
    // pure-base search (unless done above) and truncation search (24 planes,
    // then 32): each step probes both kinds of candidates as two concurrent
    // IF branches
    ctl_joint(a0, true, 0, s0);
    cudaGraphConditionalHandle hj;
    CK(cudaGraphConditionalHandleCreate(&hj, top, 1, cudaGraphCondAssignDefault));
    add_conditional(s0, s1, hj, cudaGraphCondTypeWhile, [&](cudaGraph_t body, cudaStream_t bs) {
      cudaGraphConditionalHandle hp, ht;
      CK(cudaGraphConditionalHandleCreate(&hp, body, 0, 0));
      CK(cudaGraphConditionalHandleCreate(&ht, body, 0, 0));
      CtlArgs al = a0;
      al.h_loop = hj;
      al.h_pure = hp;
      al.h_trunc = ht;
      ctl_joint(al, false, 7, bs);
      CK(cudaEventRecord(c->ev_f0, bs));
      CK(cudaStreamWaitEvent(s2, c->ev_f0, 0));
      add_conditional(s2, s4, ht, cudaGraphCondTypeIf, [&](cudaGraph_t, cudaStream_t is) {
        probe_trunc(mres, w.prm + w.np0, inc_res ? w.Linc[1] : w.A2, w.B2, g, ntp, w.base_dec,
                    w.x32, w.fs, w.res + w.np0, is, inc_res, false, nfields);
      });
      add_conditional(bs, s3, hp, cudaGraphCondTypeIf,
                      [&](cudaGraph_t, cudaStream_t is) { base_probe(is, true); });
      CK(cudaEventRecord(c->ev_f1, s2));
      CK(cudaStreamWaitEvent(bs, c->ev_f1, 0));
    });
    fused::timer_record(c->ph[2], s0);
    ctl_finalize(a0, s0);
    CK(cudaMemcpyAsync(w.h_ctl_out, w.ctl_out, sizeof(CtlOut) * nfields, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(w.h_fs, w.fs, sizeof(FieldScal) * nfields, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(w.h_mo, w.mo_base, sizeof(MachineOut) * nfields, cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(w.h_mo + w.cap, w.mo_res, sizeof(MachineOut) * nfields,
                       cudaMemcpyDeviceToHost, s0));
    CK(cudaMemcpyAsync(w.h_ctl_stats, w.ctl_stats, sizeof(CtlStats), cudaMemcpyDeviceToHost, s0));
    fused::timer_record(c->ph[3], s0);
    cudaGraph_t gr = nullptr;
    CK(cudaStreamEndCapture(s0, &gr));
    Workspace::SearchGraph ng;
    ng.nf = nfields; ng.slots = TS; ng.prune = prune; ng.early = early; ng.inc = inc_ok;
    ng.cluster = cluster; ng.j2 = j2;
    CK(cudaGraphInstantiate(&ng.exec, gr, 0));
    cudaGraphDestroy(gr);
    w.graphs.push_back(ng);
    sg = &w.graphs.back();
    g_slow.mark("graph_built");
  }
  if (graphs) CK(cudaGraphLaunch(sg->exec, st));
  CK(cudaStreamSynchronize(st));
  g_slow.mark("searches_done");
  g_trace.add(g_lane, "searches_done", -1);

  // ---- instrumentation ----
  {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, c->tev[0], c->tev[1]) == cudaSuccess) c->stats.ms_encode += ms;
    if (cudaEventElapsedTime(&ms, c->ev_s0, c->ev_s1) == cudaSuccess) c->stats.ms_encode += ms;
    static const bool prof = getenv("EBCC_PROFILE") && getenv("EBCC_PROFILE")[0] == '1';
    if (prof && graphs) {
      float t[6] = {};
      cudaEventElapsedTime(&t[0], c->tev[0], c->tev[1]);
      cudaEventElapsedTime(&t[1], c->ph[0], c->ph[1]);
      cudaEventElapsedTime(&t[2], c->ph[1], c->ev_s0);
      cudaEventElapsedTime(&t[3], c->ev_s0, c->ev_s1);
      cudaEventElapsedTime(&t[4], c->ev_s1, c->ph[2]);
      cudaEventElapsedTime(&t[5], c->ph[2], c->ph[3]);
      const CtlStats cs = *w.h_ctl_stats;
      float tp = -1;
      if (SB > 1 && N * (int64_t)nfields <= kSplitPoints) cudaEventElapsedTime(&tp, c->ph[1], c->ph[4]);
      if (tp >= 0) fprintf(stderr, "[ebcc phases] pure-base loop beside the residual encode: %.3f ms\n", tp);
      fprintf(stderr,
              "[ebcc phases] %d fields: base encode %.3f | base search %.3f (%llu steps) | "
              "residue+dwt %.3f | residual encode %.3f | joint search %.3f (%llu steps) | "
              "finalize %.3f ms\n",
              nfields, t[0], t[1], cs.base_steps, t[2], t[3], t[4], cs.joint_steps, t[5]);
    }
    if (cudaEventElapsedTime(&ms, c->l0.a, c->l0.b) == cudaSuccess) {
      c->stats.ms_probe_kernel += ms;
      c->stats.probe_kernel_count++;
      c->stats.probe_kernel_fields += nfields;
    }
    cudaGetLastError();
    const CtlStats cs = *w.h_ctl_stats;
    c->stats.probe_launches += 1 + (int64_t)(cs.base_steps + cs.joint_steps);
    c->stats.kernel_launches += 4 + (int64_t)(cs.base_steps + cs.joint_steps) +
                                (int64_t)(1 + cs.base_probes + cs.pure_probes + cs.trunc_probes) *
                                    (g.levels + 1) +
                                2 * g.levels + 10 + g.levels;
  }

  // ---- ingest errors, then candidate choice (pipeline.py:315-329) + parts ----
  const FieldScal* fs = w.h_fs;
  for (int f = 0; f < nfields; f++)
    if (fs[f].first_bad >= 0) {
      c->err_index = (int64_t)f * N + fs[f].first_bad;
      throw IngestFail{};
    }
  int status = EBCC_OK;
  const MachineOut* bmo = w.h_mo;
  const MachineOut* rmo = w.h_mo + w.cap;
  int64_t probed = 0;
  for (int f = 0; f < nfields; f++) {
    ebcc_chunk_rec& r = recs[f];
    const CtlOut& o = w.h_ctl_out[f];
    memset(&r, 0, sizeof(r));
    r.vmin = fs[f].vmin;
    r.vmax = fs[f].vmax;
    r.n_base_probes = o.n_base_probes;
    r.n_trunc_probes = o.n_trunc_probes;
    probed += o.n_base_probes + o.n_trunc_probes;
    if (fs[f].constant) {
      r.mode = EBCC_MODE_CONSTANT;
      sizes.push_back(0);
      continue;
    }
    if (o.status & kCtlCapacity)
      throw CudaFail{cudaErrorMemoryAllocation, "search state capacity (memo / list / loop guard)"};
    // (the controller's stream lengths: the budget's bytes, or for a J2
    // base the longest unit-aligned prefix)
    const int64_t pure_len = o.pure_budget >= 0 ? o.len_pure : -1;
    const int64_t base_len = o.len_base;
    const int64_t two_len = o.trunc_t >= 0 ? base_len + kHeader + o.trunc_t : -1;
    if (pure_len < 0 && two_len < 0) {
      r.status = EBCC_E_RESIDUAL;
      status = EBCC_E_RESIDUAL;
      sizes.push_back(0);
      continue;
    }
    const int base_nmax = bmo[f].n_max;
    if (base_nmax < -128 || base_nmax > 127 ||
        (rmo[f].n_max != kExpNone && (rmo[f].n_max < -128 || rmo[f].n_max > 127)))
      throw CudaFail{cudaErrorInvalidValue, "stream exponent out of int8 range"};
    int64_t off = out_base_off;
    for (int64_t z : sizes) off += z;
    PackPart bp{};
    bp.src = w.bits_base + (int64_t)f * w.words_base;  // (J2: the stream body)
    bp.bit_limit = ~0ull;
    put_header(bp.hdr, base_nmax == kExpNone ? kZeroSentinel : base_nmax, g.levels, g.rows,
               g.cols, j2);
    if (pure_len >= 0 && (two_len < 0 || pure_len <= two_len)) {
      r.mode = EBCC_MODE_PURE_BASE;
      r.base_len = pure_len;
      r.resid_len = 0;
      bp.dst_off = (uint64_t)off;
      bp.nbytes = (uint64_t)pure_len;
      parts.push_back(bp);
      sizes.push_back(pure_len);
    } else {
      r.mode = EBCC_MODE_TWO_LAYER;
      r.base_len = base_len;
      r.resid_len = kHeader + o.trunc_t;
      r.resid_planes = o.trunc_planes;
      bp.dst_off = (uint64_t)off;
      bp.nbytes = (uint64_t)base_len;
      parts.push_back(bp);
      PackPart rp{};
      rp.src = w.bits_res + (int64_t)f * w.words_res;
      rp.dst_off = (uint64_t)(off + base_len);
      rp.nbytes = (uint64_t)(kHeader + o.trunc_t);
      rp.bit_limit = o.trunc_planes == kBasePlanes ? o.T24 : o.T32;
      const int rn = rmo[f].n_max == kExpNone ? kZeroSentinel : rmo[f].n_max;
      put_header(rp.hdr, rn, g.levels, g.rows, g.cols);
      parts.push_back(rp);
      sizes.push_back(two_len);
    }
  }
  if (inc_ok) {
    unsigned long long comp[2 * kMaxLevels];
    CK(cudaMemcpy(comp, w.icomputed, sizeof comp, cudaMemcpyDeviceToHost));
    c->stats.tiles_computed += (int64_t)(comp[0] + comp[kMaxLevels]);
    c->stats.tiles_probed += probed * inc_s[0].ig.tiles0;
  }
  return status;
}

int fail(ebcc_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

}  // namespace

// order the library stream after the caller's default stream (set_stream(0))
void join_caller(ebcc_ctx* c) {
  if (!c || !c->join) return;
  if (!c->ev_join) cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  cudaEventRecord(c->ev_join, c->join);
  cudaStreamWaitEvent(c->stream, c->ev_join, 0);
}

namespace ebcc {
cudaStream_t ctx_stream(ebcc_ctx* c) {
  join_caller(c);
  return c->stream;
}
int ctx_device(ebcc_ctx* c) { return c->device; }
int ctx_fail(ebcc_ctx* c, int code, const char* msg) { return fail(c, code, msg); }
}  // namespace ebcc

// ===========================================================================
// C ABI
extern "C" {

int ebcc_abi_version(void) { return EBCC_ABI_VERSION; }

int ebcc_create(int32_t device, ebcc_ctx** out) {
  if (!out) return EBCC_E_ARGUMENT;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return EBCC_E_CUDA;
  ebcc_ctx* c = new ebcc_ctx();
  c->device = device;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete c; return EBCC_E_CUDA; }
  cudaEventCreate(&c->l0.a);
  cudaEventCreate(&c->l0.b);
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_f0, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_f1, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming);
    cudaEventCreate(&c->cev0);
    cudaEventCreate(&c->cev1);
    cudaEventCreate(&c->oev0);
    cudaEventCreate(&c->oev1);
    cudaEventCreate(&c->ev_s0);
    cudaEventCreate(&c->ev_s1);
    for (cudaEvent_t& e : c->ph) cudaEventCreate(&e);
    cudaEventCreate(&c->tm_a);
    cudaEventCreate(&c->tm_b);
    cudaEventCreate(&c->tev[0]);
    cudaEventCreate(&c->tev[1]);
  }
  c->own_stream = true;
  *out = c;
  return EBCC_OK;
}

void ebcc_destroy(ebcc_ctx* c) {
  if (!c) return;
  metrics_release(c);
  for (ebcc_ctx* l : c->lanes) ebcc_destroy(l);
  c->lanes.clear();
  cudaSetDevice(c->device);
  c->ws.release();
  for (Workspace& cw : c->ws_cache) cw.release();
  c->ws_cache.clear();
  if (c->d_payload) cudaFree(c->d_payload);
  if (c->d_parts) cudaFree(c->d_parts);
  if (c->d_unpack) cudaFree(c->d_unpack);
  if (c->d_stage) cudaFree(c->d_stage);
  if (c->d_out) cudaFree(c->d_out);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->h_arena) cudaFreeHost(c->h_arena);
  if (c->h_pay) cudaFreeHost(c->h_pay);
  if (c->h_stage2) cudaFreeHost(c->h_stage2);
  if (c->h_pay2) cudaFreeHost(c->h_pay2);
  if (c->d_out2) cudaFree(c->d_out2);
  if (c->d_in2) cudaFree(c->d_in2);
  for (cudaEvent_t e : {c->ev_in2, c->ev_in2_used})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_obuf[0], c->ev_obuf[1], c->ev_pbuf[0], c->ev_pbuf[1]})
    if (e) cudaEventDestroy(e);
  if (c->d_cont) cudaFree(c->d_cont);
  if (c->d_cmeta) cudaFree(c->d_cmeta);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->l0.a) cudaEventDestroy(c->l0.a);
  if (c->l0.b) cudaEventDestroy(c->l0.b);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->ev_copy) cudaEventDestroy(c->ev_copy);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  for (cudaEvent_t e : c->ev_groups) cudaEventDestroy(e);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->ev_f0) cudaEventDestroy(c->ev_f0);
  if (c->ev_f1) cudaEventDestroy(c->ev_f1);
  for (cudaEvent_t e : {c->cev0, c->cev1, c->oev0, c->oev1})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ph)
    if (e) cudaEventDestroy(e);
  if (c->ev_s0) cudaEventDestroy(c->ev_s0);
  if (c->ev_s1) cudaEventDestroy(c->ev_s1);
  if (c->tm_a) cudaEventDestroy(c->tm_a);
  if (c->tm_b) cudaEventDestroy(c->tm_b);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (cudaEvent_t e : c->tev)
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : c->cap)
    if (s) cudaStreamDestroy(s);
  delete c;
}

int ebcc_set_stream(ebcc_ctx* c, void* s) {
  if (!c) return EBCC_E_ARGUMENT;
  cudaStream_t cs = static_cast<cudaStream_t>(s);
  if (cs == nullptr || cs == cudaStreamLegacy || cs == cudaStreamPerThread) {
    // the legacy / per-thread default stream cannot be captured into CUDA
    // graphs: the library keeps a stream of its own and orders it after the
    // caller's stream at every call (results are complete when a call returns)
    if (!c->own_stream) {
      if (cudaSetDevice(c->device) != cudaSuccess ||
          cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
        return fail(c, EBCC_E_CUDA, "cannot create the library stream");
      c->own_stream = true;
    }
    c->join = cs == nullptr ? cudaStreamLegacy : cs;
    return EBCC_OK;
  }
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  c->stream = cs;
  c->own_stream = false;
  c->join = nullptr;
  return EBCC_OK;
}

const char* ebcc_last_error(const ebcc_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t ebcc_last_error_index(const ebcc_ctx* c) { return c ? c->err_index : -1; }

int ebcc_get_stats(const ebcc_ctx* c, ebcc_stats* out) {
  if (!c || !out) return EBCC_E_ARGUMENT;
  *out = c->stats;
  return EBCC_OK;
}

}  // extern "C"

namespace {
// compress nfields chunks on one context; the packed payload is left in
// c->d_payload (c->payload_total bytes), per-chunk sizes in `sizes`
// device bytes held by the workspaces of a context tree (the context and its
// lanes); `caches` adds the parked workspaces of other chunk shapes
int64_t tree_held(const ebcc_ctx* c, bool caches) {
  int64_t b = c->ws.bytes;
  if (caches)
    for (const Workspace& w : c->ws_cache) b += w.bytes;
  for (const ebcc_ctx* l : c->lanes) b += tree_held(l, caches);
  return b;
}
void tree_drop_caches(ebcc_ctx* c) {
  for (Workspace& w : c->ws_cache) w.release();
  c->ws_cache.clear();
  for (ebcc_ctx* l : c->lanes) tree_drop_caches(l);
}
// device bytes per chunk of a workspace of geometry g (measured from an
// existing one, incl. the decompress decoder state; else ~262 B/pt), plus
// the call's own payload / output buffers (~12 B/pt)
int64_t per_field_bytes(const ebcc_ctx* c, const Geo& g) {
  auto same = [&](const Workspace& w) {
    return w.cap > 0 && w.g.rows == g.rows && w.g.cols == g.cols && w.g.levels == g.levels;
  };
  int64_t pf = g.n * 262 + (1 << 16);
  auto take = [&](const Workspace& w) {
    if (!same(w)) return;
    int64_t b = w.bytes / w.cap + (w.dec2.mant ? 0 : g.n * 57);
    pf = std::max<int64_t>(b, g.n * 64);
  };
  take(c->ws);
  for (const ebcc_ctx* l : c->lanes) take(l->ws);
  return pf + 20 * g.n;  // + payload, two output / input buffers
}
// chunks per device batch for `lanes` concurrent sub-batches of up to `want`
// chunks each: 85% of (free HBM + what this tree's workspaces hold) minus a
// 1 GiB reserve, split evenly.  `tree` = every lane's workspace may be
// reallocated (compress); otherwise only c->ws (decompress).
int64_t plan_batch(ebcc_ctx* c, const Geo& g, int64_t want, int lanes, bool tree, bool j2) {
  want = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, 4096), max_batch()));
  // the opt-in J2 base layer's buffers (ensure_ebcot): ~24 B/pt + per-block tables
  const int64_t pf = per_field_bytes(c, g) + (j2 ? g.n * 26 + (1 << 20) : 0);
  auto cap_now = [&]() {
    size_t freeb = 0, totalb = 0;
    CK(cudaMemGetInfo(&freeb, &totalb));
    const double avail = (double)freeb + (double)(tree ? tree_held(c, false) : c->ws.bytes) -
                         (double)(1ll << 30);
    return (int64_t)(avail * 0.85 / std::max(1, lanes) / (double)pf);
  };
  int64_t cap = cap_now();
  if (cap < want && tree_held(c, true) > tree_held(c, false)) {
    tree_drop_caches(c);  // parked workspaces of other shapes give way
    cap = cap_now();
  }
  return cap < 1 ? 1 : (cap > want ? want : cap);
}
// balanced batches: ceil(n / cap) batches of near-equal size
int64_t balance(int64_t n, int64_t cap) {
  if (n <= 0) return 1;
  const int64_t nb = (n + cap - 1) / cap;
  return (n + nb - 1) / nb;
}

// lanes: their input copies run one after another (lane k's copy starts
// when lane k-1's has finished), so lane 0 computes while lane 1's input is
// still arriving instead of every lane waiting for the whole input
struct CopyChain {
  std::atomic<int> issued{0};  // lanes whose copy (and its event) are enqueued
  std::vector<cudaEvent_t> done;
};

int compress_impl(ebcc_ctx* c, const float* fields, int64_t nfields, int32_t rows, int32_t cols,
                  double eps_rel, double q, double r0, double search_tol, int32_t flags,
                  ebcc_chunk_rec* recs, std::vector<int64_t>& sizes, cudaEvent_t start_after,
                  int64_t plan_cap, CopyChain* chain = nullptr, int lane = 0) {
  struct ChainRelease {  // a lane that fails before its copy must not stall the next
    CopyChain* ch; int k; bool done = false;
    ~ChainRelease() {
      if (!ch || done) return;
      while (ch->issued.load() < k) std::this_thread::yield();
      ch->issued.store(k + 1);
    }
  } chain_release{chain, lane};
  c->stats = ebcc_stats{};
  c->err.clear();
  try {
    CK(cudaSetDevice(c->device));
    CK(cudaGetLastError());
    cudaStream_t st = c->stream;
    if (start_after) CK(cudaStreamWaitEvent(st, start_after, 0));
    int levels = clamp_levels(rows, cols, default_levels(rows, cols));
    Geo g = make_geo(rows, cols, levels);
    const int64_t cap = balance(nfields, plan_cap);
    cudaEvent_t t0 = c->cev0, t1 = c->cev1;
    cudaEventRecord(t0, st);
    std::vector<PackPart> parts;
    sizes.clear();
    int status = EBCC_OK;
    g_slow.mark("compress_setup");
    // host input, several batches: while batch i computes, a helper thread
    // stages batch i+1 (pageable input: into the other page-locked block) and
    // uploads it on the copy stream into a second device buffer; batch i+1
    // then starts with a device-to-device copy instead of waiting for PCIe
    const bool host_in = !(flags & EBCC_INPUT_ON_DEVICE);
    struct Prefetch {
      std::thread t;
      int64_t f0 = -1;
      cudaError_t err = cudaSuccess;
      ~Prefetch() { if (t.joinable()) t.join(); }
    } pf;
    int stage_k = 0;
    auto stage_buf = [&](int k, int64_t bytes) {
      return k ? pinned_block(c->h_stage2, c->h_stage2_cap, bytes) : host_stage(c, bytes);
    };
    if (host_in && cap < nfields) {
      if (!c->copy) {
        CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming));
      }
      for (cudaEvent_t* e : {&c->ev_in2, &c->ev_in2_used})
        if (!*e) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    for (int64_t f0 = 0; f0 < nfields; f0 += cap) {
      int nb = (int)std::min<int64_t>(cap, nfields - f0);
      ensure_workspace(c, g, nb, (int)cap);
      g_slow.mark("ensure_workspace");
      CK(cudaGetLastError());
      const float* src = fields + f0 * g.n;
      const size_t in_bytes = sizeof(float) * g.n * nb;
      const bool prefetched = pf.f0 == f0;
      if (prefetched) {
        pf.t.join();
        pf.f0 = -1;
        if (pf.err != cudaSuccess) throw CudaFail{pf.err, "input prefetch"};
        CK(cudaStreamWaitEvent(st, c->ev_in2, 0));
        CK(cudaMemcpyAsync(c->ws.x32, c->d_in2, in_bytes, cudaMemcpyDeviceToDevice, st));
        CK(cudaEventRecord(c->ev_in2_used, st));
        g_trace.add(g_lane, "in_prefetched", (int)f0);
      }
      // pageable input not prefetched (the first batch): staged group by
      // group below, each group's upload issued as soon as it is staged
      const float* stage_from = nullptr;
      if (!prefetched && host_in && is_pageable(src)) {
        CK(cudaGetLastError());
        uint8_t* stg = stage_buf(stage_k, (int64_t)in_bytes);
        CK(cudaGetLastError());
        stage_from = src;
        src = reinterpret_cast<const float*>(stg);
        stage_k ^= 1;
      }
      CK(cudaGetLastError());
      const bool chained = chain && f0 == 0 && !(flags & EBCC_INPUT_ON_DEVICE);
      if (stage_from && chained && lane > 0) {
        // a later lane's upload queues behind the earlier lanes': stage it
        // whole now, concurrently with theirs
        parallel_memcpy(const_cast<float*>(src), stage_from, in_bytes);
        stage_from = nullptr;
        g_trace.add(g_lane, "in_staged", (int)f0);
      }
      // host input: copied in field groups on the copy stream, each group
      // transformed as soon as it lands (compress_batch)
      static const int in_groups_env =
          getenv("EBCC_IN_GROUPS") ? std::max(1, atoi(getenv("EBCC_IN_GROUPS"))) : 4;
      const int in_groups = (!host_in || prefetched) ? 0 : std::min(in_groups_env, nb);
      cudaStream_t cst = in_groups ? c->copy : st;
      if (in_groups && !c->copy) {
        CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming));
        cst = c->copy;
      }
      while ((int)c->ev_groups.size() < in_groups) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_groups.push_back(e);
      }
      if (in_groups) CK(cudaStreamWaitEvent(cst, c->cev0, 0));  // after this call's start
      if (chained && lane > 0) {
        while (chain->issued.load() < lane) std::this_thread::yield();
        CK(cudaStreamWaitEvent(cst, chain->done[lane - 1], 0));
      }
      if (in_groups) {
        for (int k = 0; k < in_groups; k++) {
          const int64_t a = (int64_t)nb * k / in_groups, b = (int64_t)nb * (k + 1) / in_groups;
          if (b > a && stage_from)
            parallel_memcpy(const_cast<float*>(src) + a * g.n, stage_from + a * g.n,
                            sizeof(float) * g.n * (b - a));
          if (b > a)
            CK(cudaMemcpyAsync(c->ws.x32 + a * g.n, src + a * g.n, sizeof(float) * g.n * (b - a),
                               cudaMemcpyHostToDevice, cst));
          CK(cudaEventRecord(c->ev_groups[k], cst));
        }
        if (stage_from) g_trace.add(g_lane, "in_staged", (int)f0);
      } else if (!prefetched) {
        if (stage_from) parallel_memcpy(const_cast<float*>(src), stage_from, in_bytes);
        CK(cudaMemcpyAsync(c->ws.x32, src, in_bytes,
                           (flags & EBCC_INPUT_ON_DEVICE) ? cudaMemcpyDeviceToDevice
                                                          : cudaMemcpyHostToDevice,
                           st));
      }
      if (chained) {
        CK(cudaEventRecord(chain->done[lane], cst));
        chain->issued.store(lane + 1);
        chain_release.done = true;
      }
      // next batch: stage + upload behind this batch's compute
      const int64_t f1 = f0 + cap;
      if (host_in && f1 < nfields) {
        const int64_t nb1 = std::min<int64_t>(cap, nfields - f1);
        const size_t nbytes = sizeof(float) * g.n * nb1;
        const float* nsrc = fields + f1 * g.n;
        uint8_t* nstg = nullptr;
        if (is_pageable(nsrc)) {
          nstg = stage_buf(stage_k, (int64_t)nbytes);
          stage_k ^= 1;
        }
        float* dst = device_block(c->d_in2, c->in2_cap, g.n * cap);
        // the upload may overwrite d_in2 once this batch's copy out of it ran
        if (prefetched) CK(cudaStreamWaitEvent(c->copy, c->ev_in2_used, 0));
        const int dev = c->device;
        cudaStream_t cp = c->copy;
        cudaEvent_t done_ev = c->ev_in2;
        Prefetch* pp = &pf;
        pf.err = cudaSuccess;
        pf.t = std::thread([=] {
          const float* s = nsrc;
          if (nstg) {
            parallel_memcpy(nstg, nsrc, nbytes);
            s = reinterpret_cast<const float*>(nstg);
          }
          cudaError_t e = cudaSetDevice(dev);
          if (e == cudaSuccess) e = cudaMemcpyAsync(dst, s, nbytes, cudaMemcpyHostToDevice, cp);
          if (e == cudaSuccess) e = cudaEventRecord(done_ev, cp);
          pp->err = e;
        });
        pf.f0 = f1;
      }
      std::vector<PackPart> bparts;
      int64_t done = 0;
      for (int64_t z : sizes) done += z;
      std::vector<int64_t> bsizes;
      int s;
      try {
        s = compress_batch(c, nb, eps_rel, q, r0, search_tol, !(flags & EBCC_FULL_SEARCH),
                           recs + f0, done, bparts, bsizes, in_groups, c->ev_groups.data(),
                           (flags & EBCC_BASE_EBCOT) != 0);
      } catch (IngestFail&) {
        c->err_index += f0 * g.n;
        return fail(c, EBCC_E_INGEST, "non-finite value in the input");
      }
      if (s != EBCC_OK) status = s;
      g_slow.mark("batch_searches");
      // pack this batch now: the stream buffers are reused by the next batch
      int64_t bytes = done;
      for (int64_t z : bsizes) bytes += z;
      if (bytes > c->payload_cap) {
        // grow, preserving what earlier batches packed
        uint8_t* nbuf = dalloc<uint8_t>((size_t)std::max<int64_t>(bytes * 2, 1 << 20));
        if (c->d_payload && done) CK(cudaMemcpyAsync(nbuf, c->d_payload, done, cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
        if (c->d_payload) cudaFree(c->d_payload);
        c->d_payload = nbuf;
        c->payload_cap = std::max<int64_t>(bytes * 2, 1 << 20);
      }
      if (!bparts.empty()) {
        if ((int)bparts.size() > c->parts_cap) {
          if (c->d_parts) cudaFree(c->d_parts);
          c->parts_cap = (int)bparts.size() * 2;
          c->d_parts = dalloc<PackPart>(c->parts_cap);
        }
        h2d_small(c, c->d_parts, bparts.data(), sizeof(PackPart) * bparts.size(), st);
        pack_parts(c->d_parts, (int)bparts.size(), c->d_payload, st);
        c->stats.kernel_launches++;
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
      }
      sizes.insert(sizes.end(), bsizes.begin(), bsizes.end());
      g_slow.mark("batch_pack");
      g_trace.add(g_lane, "packed", (int)f0);
    }
    int64_t total = 0;
    for (int64_t f = 0; f < nfields; f++) total += sizes[f];
    c->payload_total = total;
    cudaEventRecord(t1, st);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    c->stats.ms_total = ms;
    c->stats.ms_other = ms - c->stats.ms_encode - c->stats.ms_probe;
    return status;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, e.e == cudaErrorMemoryAllocation ? EBCC_E_NOMEM : EBCC_E_CUDA,
                std::string(e.what) + ": " + cudaGetErrorString(e.e));
  } catch (std::exception& e) {
    return fail(c, EBCC_E_CUDA, e.what());
  }
}

int lanes_for(int64_t nfields, int64_t npoints) {
  const char* e = getenv("EBCC_LANES");
  // two concurrent sub-batches hide one lane's latency-bound list machine and
  // host turnaround behind the other's probes: measured -6.5% compress time
  // for 37 x 721x1440 (mean 42.1 vs 45.1 ms, p99 45 ms over 100 runs)
  // large chunks (configs[3]: 2881x5760): the list machines of a few chunks
  // leave most SMs idle, so up to three lanes pay off already from two chunks
  // (10 chunks: 129.7 -> 122.7 ms; 2 chunks: 51.8 -> 49.6 ms)
  int want = e ? atoi(e) : (npoints >= (4 << 20) ? 3 : (nfields >= 16 ? 2 : 1));
  if (want < 1) want = 1;
  if (want > nfields) want = (int)std::max<int64_t>(1, nfields);
  return want;
}

ebcc_ctx* lane_ctx(ebcc_ctx* c, int k);

void add_stats(ebcc_stats& a, const ebcc_stats& b) {
  a.kernel_launches += b.kernel_launches;
  a.ms_encode += b.ms_encode;
  a.ms_probe += b.ms_probe;
  a.probe_launches += b.probe_launches;
  a.ms_probe_kernel += b.ms_probe_kernel;
  a.probe_kernel_count += b.probe_kernel_count;
  a.probe_kernel_fields += b.probe_kernel_fields;
  a.tiles_computed += b.tiles_computed;
  a.tiles_probed += b.tiles_probed;
}

}  // namespace

extern "C" int ebcc_create(int32_t device, ebcc_ctx** out);
extern "C" void ebcc_destroy(ebcc_ctx* c);

namespace {
ebcc_ctx* lane_ctx(ebcc_ctx* c, int k) {
  while ((int)c->lanes.size() <= k) {
    ebcc_ctx* child = nullptr;
    if (ebcc_create(c->device, &child) != EBCC_OK) throw CudaFail{cudaErrorUnknown, "lane create"};
    c->lanes.push_back(child);
  }
  return c->lanes[k];
}
}  // namespace

extern "C" int ebcc_compress(ebcc_ctx* c, const float* fields, int64_t nfields, int32_t rows,
                             int32_t cols, double eps_rel, double q, double r0,
                             double search_tol, int32_t flags, ebcc_chunk_rec* recs,
                             uint8_t* payload, int64_t payload_cap, int64_t* payload_offsets,
                             int64_t* payload_total) {
  if (!c || !fields || !recs || nfields < 0 || rows < 1 || cols < 1)
    return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  // EbccParams.validate (pipeline.py:54-62)
  if (!(eps_rel > 0.0 && eps_rel < 1.0))
    return fail(c, EBCC_E_ARGUMENT, "epsilon_rel must be in (0, 1)");
  if (!(q > 0.0 && q <= 1.0)) return fail(c, EBCC_E_ARGUMENT, "q must be in (0, 1]");
  if (r0 < 1.0) return fail(c, EBCC_E_ARGUMENT, "r0 must be >= 1");
  if (!(search_tol > 0.0)) return fail(c, EBCC_E_ARGUMENT, "search_tol must be positive");
  if ((int64_t)rows * cols > kMaxChunkPoints)
    return fail(c, EBCC_E_ARGUMENT, "chunk too large (at most 2^32 - 2 points)");
  c->err.clear();
  c->err_index = -1;
  arena_reset(c);  // the previous call ended synchronised
  try {
    CK(cudaSetDevice(c->device));
    join_caller(c);
    const int L = lanes_for(nfields, (int64_t)rows * cols);
    const int64_t n = (int64_t)rows * cols;
    {
      const int levels = clamp_levels(rows, cols, default_levels(rows, cols));
      const Geo g = make_geo(rows, cols, levels);
      for (int k = 0; k < (L > 1 ? L : 0); k++) lane_ctx(c, k);  // the tree the plan covers
      const int j2 = (flags & EBCC_BASE_EBCOT) ? 1 : 0;
      if (!c->cplan.matches(g, nfields, L, j2)) {
        c->cplan.cap = plan_batch(c, g, (nfields + L - 1) / L, L, true, j2 != 0);
        c->cplan.rows = g.rows; c->cplan.cols = g.cols; c->cplan.levels = g.levels;
        c->cplan.nfields = nfields; c->cplan.lanes = L; c->cplan.j2 = j2;
      }
    }
    const int64_t plan_cap = c->cplan.cap;
    g_trace.start();
    struct TraceDump { ~TraceDump() { g_trace.dump(); } } trace_dump;
    std::vector<int64_t> sizes;
    int status = EBCC_OK;
    cudaEvent_t t0 = c->oev0, t1 = c->oev1;
    CK(cudaEventRecord(t0, c->stream));
    ebcc_stats total_stats{};
    if (L == 1) {
      status = compress_impl(c, fields, nfields, rows, cols, eps_rel, q, r0, search_tol, flags,
                             recs, sizes, nullptr, plan_cap);
      total_stats = c->stats;
      if (status != EBCC_OK && status != EBCC_E_RESIDUAL) return status;
    } else {
      // concurrent sub-batches: each lane (own stream + workspace + host
      // thread) runs the whole pipeline on a contiguous block of chunks, so
      // one lane's latency-bound list machine overlaps another's probes
      std::vector<ebcc_ctx*> ls(L);
      for (int k = 0; k < L; k++) {
        ls[k] = lane_ctx(c, k);
        ls[k]->machine_fields = (int)nfields;  // every lane's clusters resident at once
      }
      std::vector<int64_t> lo(L + 1);
      for (int k = 0; k <= L; k++) lo[k] = nfields * k / L;
      std::vector<std::vector<int64_t>> lsz(L);
      std::vector<int> lst(L, EBCC_OK);
      std::vector<std::thread> th;
      CopyChain chain;
      for (int k = 0; k < L; k++) chain.done.push_back(ls[k]->ev_in);
      for (int k = 0; k < L; k++)
        th.emplace_back([&, k] {
          cudaSetDevice(c->device);
          g_lane = k;
          lst[k] = compress_impl(ls[k], fields + lo[k] * n, lo[k + 1] - lo[k], rows, cols, eps_rel,
                                 q, r0, search_tol, flags, recs + lo[k], lsz[k], t0, plan_cap,
                                 &chain, k);
        });
      for (auto& t : th) t.join();
      for (int k = 0; k < L; k++) {
        if (lst[k] != EBCC_OK && lst[k] != EBCC_E_RESIDUAL) {
          c->err = ls[k]->err;
          c->err_index = ls[k]->err_index + lo[k] * n;
          return lst[k];
        }
        if (lst[k] == EBCC_E_RESIDUAL) status = EBCC_E_RESIDUAL;
        sizes.insert(sizes.end(), lsz[k].begin(), lsz[k].end());
        add_stats(total_stats, ls[k]->stats);
      }
      // gather the lanes' payloads into this context's buffer
      int64_t tot = 0;
      for (int64_t z : sizes) tot += z;
      if (tot > c->payload_cap) {
        if (c->d_payload) cudaFree(c->d_payload);
        c->payload_cap = std::max<int64_t>(tot * 2, 1 << 20);
        c->d_payload = dalloc<uint8_t>((size_t)c->payload_cap);
      }
      int64_t off = 0;
      for (int k = 0; k < L; k++) {
        if (ls[k]->payload_total)
          CK(cudaMemcpyAsync(c->d_payload + off, ls[k]->d_payload, ls[k]->payload_total,
                             cudaMemcpyDeviceToDevice, c->stream));
        off += ls[k]->payload_total;
      }
    }
    int64_t total = 0;
    for (int64_t f = 0; f < nfields; f++) {
      if (payload_offsets) payload_offsets[f] = total;
      total += sizes[f];
    }
    c->payload_total = total;
    if (payload_total) *payload_total = total;
    CK(cudaEventRecord(t1, c->stream));
    CK(cudaEventSynchronize(t1));
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    c->stats = total_stats;
    c->stats.lanes = L;
    c->stats.ms_total = ms;
    c->stats.ms_other = ms - c->stats.ms_encode / L - c->stats.ms_probe / L;
    if (status != EBCC_OK) {
      for (int64_t f = 0; f < nfields; f++)
        if (recs[f].status == EBCC_E_RESIDUAL)
          return fail(c, EBCC_E_RESIDUAL,
                      "chunk " + std::to_string(f) + ": no encoding reaches epsilon_rel");
    }
    if (payload && total > 0) {
      if (total > payload_cap) return fail(c, EBCC_E_CAPACITY, "payload buffer too small");
      CK(cudaMemcpyAsync(payload, c->d_payload, total,
                         (flags & EBCC_OUTPUT_ON_DEVICE) ? cudaMemcpyDeviceToDevice
                                                         : cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, e.e == cudaErrorMemoryAllocation ? EBCC_E_NOMEM : EBCC_E_CUDA,
                std::string(e.what) + ": " + cudaGetErrorString(e.e));
  }
}

extern "C" {

int ebcc_fetch_payload(ebcc_ctx* c, uint8_t* payload, int64_t cap, int32_t flags) {
  if (!c || !payload) return EBCC_E_ARGUMENT;
  if (cap < c->payload_total) return fail(c, EBCC_E_CAPACITY, "payload buffer too small");
  if (!c->payload_total) return EBCC_OK;
  cudaError_t e = cudaMemcpyAsync(payload, c->d_payload, c->payload_total,
                                  (flags & EBCC_OUTPUT_ON_DEVICE) ? cudaMemcpyDeviceToDevice
                                                                  : cudaMemcpyDeviceToHost,
                                  c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return e == cudaSuccess ? EBCC_OK : fail(c, EBCC_E_CUDA, cudaGetErrorString(e));
}

int ebcc_fetch_container(ebcc_ctx* c, const uint8_t* header42, const uint8_t* records25,
                         int64_t n, uint8_t* out, int64_t cap, int32_t flags, int64_t* out_len) {
  const bool body = (flags & EBCC_CONTAINER_BODY) != 0;  // records + payloads only
  if (!c || (!header42 && !body) || !out || n < 0 || (n && !records25))
    return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  const int64_t hlen = body ? 0 : 42;
  const int64_t total = hlen + 25 * n + c->payload_total;
  if (out_len) *out_len = total;
  if (cap < total) return fail(c, EBCC_E_CAPACITY, "container buffer too small");
  std::vector<ContainerPart> parts((size_t)n);
  int64_t src = 0, dst = hlen;
  for (int64_t i = 0; i < n; i++) {
    uint32_t bl, rl;
    memcpy(&bl, records25 + 25 * i + 17, 4);
    memcpy(&rl, records25 + 25 * i + 21, 4);
    parts[i] = ContainerPart{src, dst, (int64_t)bl + rl};
    src += (int64_t)bl + rl;
    dst += 25 + (int64_t)bl + rl;
  }
  if (src != c->payload_total)
    return fail(c, EBCC_E_ARGUMENT, "records do not match the last compress call's payload");
  try {
    CK(cudaSetDevice(c->device));
    join_caller(c);
    cudaStream_t st = c->stream;
    if (total > c->cont_cap) {
      if (c->d_cont) CK(cudaFree(c->d_cont));
      c->d_cont = nullptr;
      c->cont_cap = 0;
      c->d_cont = dalloc<uint8_t>((size_t)total);
      c->cont_cap = total;
    }
    const int64_t mb = (int64_t)sizeof(ContainerPart) * n + 25 * n + 16;
    if (mb > c->cmeta_cap) {
      if (c->d_cmeta) CK(cudaFree(c->d_cmeta));
      c->d_cmeta = nullptr;
      c->cmeta_cap = 0;
      c->d_cmeta = dalloc<uint8_t>((size_t)mb);
      c->cmeta_cap = mb;
    }
    ContainerPart* d_parts = reinterpret_cast<ContainerPart*>(c->d_cmeta);
    uint8_t* d_recs = c->d_cmeta + sizeof(ContainerPart) * n;
    if (!body) CK(cudaMemcpyAsync(c->d_cont, header42, 42, cudaMemcpyHostToDevice, st));
    if (n) {
      CK(cudaMemcpyAsync(d_parts, parts.data(), sizeof(ContainerPart) * n, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(d_recs, records25, 25 * n, cudaMemcpyHostToDevice, st));
      assemble_container(d_parts, (int)n, d_recs, c->d_payload, c->d_cont, st);
      CK(cudaGetLastError());
    }
    if (flags & EBCC_OUTPUT_ON_DEVICE) {
      CK(cudaMemcpyAsync(out, c->d_cont, total, cudaMemcpyDeviceToDevice, st));
    } else if (is_pageable(out)) {
      // pageable destination (a fresh bytes object): device->host copies of
      // 64 MiB pieces into two page-locked blocks, each piece copied on by the
      // thread team while the next one crosses PCIe
      constexpr int64_t kPiece = 64ll << 20;
      uint8_t* blk[2] = {host_stage(c, std::min(total, kPiece)),
                         total > kPiece ? pinned_block(c->h_stage2, c->h_stage2_cap, kPiece)
                                        : nullptr};
      for (int k = 0; k < 2; k++)
        if (!c->ev_pbuf[k]) CK(cudaEventCreateWithFlags(&c->ev_pbuf[k], cudaEventDisableTiming));
      const int64_t pieces = (total + kPiece - 1) / kPiece;
      auto issue = [&](int64_t i) {
        const int64_t o = i * kPiece, len = std::min(kPiece, total - o);
        CK(cudaMemcpyAsync(blk[i & 1], c->d_cont + o, len, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(c->ev_pbuf[i & 1], st));
      };
      issue(0);
      for (int64_t i = 0; i < pieces; i++) {
        if (i + 1 < pieces) issue(i + 1);
        CK(cudaEventSynchronize(c->ev_pbuf[i & 1]));
        const int64_t o = i * kPiece, len = std::min(kPiece, total - o);
        parallel_memcpy(out + o, blk[i & 1], (size_t)len);
      }
    } else {
      CK(cudaMemcpyAsync(out, c->d_cont, total, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, e.e == cudaErrorMemoryAllocation ? EBCC_E_NOMEM : EBCC_E_CUDA,
                std::string(e.what) + ": " + cudaGetErrorString(e.e));
  }
}

int ebcc_decompress(ebcc_ctx* c, const uint8_t* payload, const int64_t* offsets,
                    const ebcc_chunk_rec* recs, int64_t nfields, int32_t rows, int32_t cols,
                    int32_t levels, int32_t flags, float* out) {
  if (!c || !recs || !out || nfields < 0 || rows < 1 || cols < 1 || levels < 1 ||
      levels > kMaxLevels)
    return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  if ((int64_t)rows * cols > kMaxChunkPoints)
    return fail(c, EBCC_E_ARGUMENT, "chunk too large (at most 2^32 - 2 points)");
  c->stats = ebcc_stats{};
  c->err.clear();
  arena_reset(c);  // the previous call ended synchronised
  g_trace.start();
  struct TraceDump { ~TraceDump() { g_trace.dump(); } } trace_dump;
  g_slow.mark("dec_enter");
  try {
    CK(cudaSetDevice(c->device));
    join_caller(c);
    cudaStream_t st = c->stream;
    Geo g = make_geo(rows, cols, levels);
    cudaEvent_t t0 = c->cev0, t1 = c->cev1;
    cudaEventRecord(t0, st);
    // decompress borrows lane 0's workspace (idle between compress calls)
    // instead of holding a second one of its own
    struct LaneWs {
      ebcc_ctx* c;
      explicit LaneWs(ebcc_ctx* c_) : c(c_) {
        if (!c->lanes.empty()) std::swap(c->ws, c->lanes[0]->ws);
      }
      ~LaneWs() {
        if (!c->lanes.empty()) std::swap(c->ws, c->lanes[0]->ws);
      }
    } lane_ws(c);
    // J2 base streams (the opt-in layer) need the ebcot buffers: the first
    // stream's magic decides the plan
    int j2_plan = 0;
    for (int64_t i = 0; i < nfields; i++) {
      if (recs[i].mode == EBCC_MODE_CONSTANT || recs[i].base_len < 2) continue;
      uint8_t mg[2] = {0, 0};
      if (flags & EBCC_INPUT_ON_DEVICE)
        CK(cudaMemcpy(mg, payload + offsets[i], 2, cudaMemcpyDeviceToHost));
      else
        memcpy(mg, payload + offsets[i], 2);
      j2_plan = mg[0] == 'J' && mg[1] == '2';
      break;
    }
    if (!c->dplan.matches(g, nfields, 1, j2_plan)) {
      c->dplan.cap = plan_batch(c, g, nfields, 1, false, j2_plan != 0);
      c->dplan.rows = g.rows; c->dplan.cols = g.cols; c->dplan.levels = g.levels;
      c->dplan.nfields = nfields; c->dplan.lanes = 1; c->dplan.j2 = j2_plan;
    }
    // Several batches: whole waves of list machines.  A batch's base and
    // residual decoder machines are one CTA per chunk each, resident two per
    // SM, so a batch of a multiple of the SM count fills every wave (2,368
    // chunks in 7 balanced batches of 338 = 1.14 waves each took 297 ms, in
    // 16 batches of 148 they take 257 ms); otherwise balanced batches.
    int64_t cap = balance(nfields, c->dplan.cap);
    {
      // EBCC_DEC_WAVES: 0 = balanced batches, k > 0 = at most k x SM count per batch
      // (one SM count per batch measured best: 257 ms; two 264, balanced 338s 297)
      static const int waves = getenv("EBCC_DEC_WAVES") ? atoi(getenv("EBCC_DEC_WAVES")) : 1;
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
      const int64_t lim = std::min<int64_t>(c->dplan.cap, (int64_t)waves * sms);
      if (waves > 0 && nfields > lim && lim >= sms) cap = lim / sms * sms;
    }
    g_slow.mark("dec_meminfo");
    for (int k = 0; k < 2; k++) {
      if (!c->ev_obuf[k]) CK(cudaEventCreateWithFlags(&c->ev_obuf[k], cudaEventDisableTiming));
      if (!c->ev_pbuf[k]) CK(cudaEventCreateWithFlags(&c->ev_pbuf[k], cudaEventDisableTiming));
    }
    // batch b uses output / payload staging buffers b & 1 (double buffers:
    // no host wait between batches; the call synchronises once at the end)
    int bk = 0;
    bool used[2] = {false, false};
    for (int64_t f0 = 0; f0 < nfields; f0 += cap, bk ^= 1) {
      int nb = (int)std::min<int64_t>(cap, nfields - f0);
      ensure_workspace(c, g, nb, (int)cap);
      g_slow.mark("dec_workspace");
      Workspace& w = c->ws;
      // gather this batch's payload bytes into a staging buffer
      int64_t lo = INT64_MAX, hi = 0;
      for (int i = 0; i < nb; i++) {
        const ebcc_chunk_rec& r = recs[f0 + i];
        if (r.mode == EBCC_MODE_CONSTANT) continue;
        int64_t o = offsets[f0 + i];
        lo = std::min(lo, o);
        hi = std::max(hi, o + r.base_len + r.resid_len);
      }
      std::vector<UnpackPart> up;
      std::vector<MachineOut> bmo(nb), rmo(nb);
      std::vector<uint64_t> blim(nb, 0), rlim(nb, 0);
      std::vector<uint8_t> bact(nb, 0), ract(nb, 0), pure(nb, 0), cst(nb, 0);
      std::vector<FieldScal> fsv(nb);
      int j2 = -1;  // base streams of the batch: 0 SPIHT ('SP'), 1 J2 (opt-in layer)
      // stream headers of device-resident payloads: all copied, one wait
      uint8_t* hdrs = nullptr;
      if (flags & EBCC_INPUT_ON_DEVICE) {
        hdrs = host_stage(c, (int64_t)2 * kHeader * nb);
        for (int i = 0; i < nb; i++) {
          const ebcc_chunk_rec& r = recs[f0 + i];
          if (r.mode == EBCC_MODE_CONSTANT || r.base_len < kHeader) continue;
          CK(cudaMemcpyAsync(hdrs + 2 * kHeader * i, payload + offsets[f0 + i], kHeader,
                             cudaMemcpyDeviceToHost, st));
          if (r.mode == EBCC_MODE_TWO_LAYER && r.resid_len >= kHeader)
            CK(cudaMemcpyAsync(hdrs + 2 * kHeader * i + kHeader,
                               payload + offsets[f0 + i] + r.base_len, kHeader,
                               cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
      }
      for (int i = 0; i < nb; i++) {
        const ebcc_chunk_rec& r = recs[f0 + i];
        fsv[i] = FieldScal{};
        fsv[i].vmin = r.vmin; fsv[i].vmax = r.vmax; fsv[i].range = r.vmax - r.vmin;
        fsv[i].range_inv = fsv[i].range != 0.0 ? 1.0 / fsv[i].range : 0.0;
        bmo[i] = MachineOut{}; rmo[i] = MachineOut{};
        bmo[i].n_max = kExpNone; rmo[i].n_max = kExpNone;
        if (r.mode == EBCC_MODE_CONSTANT) { cst[i] = 1; continue; }
        if (r.base_len < kHeader || (r.mode == EBCC_MODE_TWO_LAYER && r.resid_len > 0 && r.resid_len < kHeader))
          return fail(c, EBCC_E_FORMAT, "stream shorter than header");
        const uint8_t* bh = (flags & EBCC_INPUT_ON_DEVICE) ? hdrs + 2 * kHeader * i
                                                            : payload + offsets[f0 + i];
        const int is_j2 = bh[0] == 'J' && bh[1] == '2';
        if (j2 >= 0 && is_j2 != j2)
          return fail(c, EBCC_E_FORMAT, "mixed base stream formats in one chunk shape");
        j2 = is_j2;
        int nb_max = (int8_t)bh[2];
        bmo[i].n_max = nb_max == kZeroSentinel ? kExpNone : nb_max;
        blim[i] = (uint64_t)(r.base_len - kHeader) * 8;
        bact[i] = nb_max != kZeroSentinel;
        up.push_back(UnpackPart{(uint64_t)(offsets[f0 + i] + kHeader - lo),
                                (uint64_t)(r.base_len - kHeader),
                                w.bits_base + (int64_t)i * w.words_base});
        if (r.mode == EBCC_MODE_TWO_LAYER && r.resid_len > 0) {
          const uint8_t* rh = (flags & EBCC_INPUT_ON_DEVICE)
                                  ? hdrs + 2 * kHeader * i + kHeader
                                  : payload + offsets[f0 + i] + r.base_len;
          int rn = (int8_t)rh[2];
          rmo[i].n_max = rn == kZeroSentinel ? kExpNone : rn;
          rlim[i] = (uint64_t)(r.resid_len - kHeader) * 8;
          ract[i] = 1;
          up.push_back(UnpackPart{(uint64_t)(offsets[f0 + i] + r.base_len + kHeader - lo),
                                  (uint64_t)(r.resid_len - kHeader),
                                  w.bits_res + (int64_t)i * w.words_res});
        } else {
          pure[i] = 1;
        }
        if ((int64_t)((r.base_len - kHeader + 3) / 4) + 2 > w.words_base ||
            (ract[i] && (int64_t)((r.resid_len - kHeader + 3) / 4) + 2 > w.words_res))
          return fail(c, EBCC_E_FORMAT, "stream longer than any encoder output");
      }
      h2d_small(c, w.fs, fsv.data(), sizeof(FieldScal) * nb, st);
      if (hi > lo) {
        int64_t span = hi - lo;
        if (span > c->stage_cap) {
          if (c->d_stage) cudaFree(c->d_stage);
          c->d_stage = dalloc<uint8_t>(span);
          c->stage_cap = span;
        }
        const uint8_t* psrc = payload + lo;
        // (registering the caller's pageable buffer in place instead was
        // measured slower: 457 -> 952+ ms device time for 2,368 fields)
        if (!(flags & EBCC_INPUT_ON_DEVICE) && is_pageable(psrc)) {
          // a pageable source would make the copy synchronous through the
          // driver's small bounce buffers: stage it (thread team) into a
          // page-locked block of this context instead
          // the block's previous upload (two batches ago) must have landed
          if (used[bk]) CK(cudaEventSynchronize(c->ev_pbuf[bk]));
          uint8_t* hp = bk ? pinned_block(c->h_pay2, c->h_pay2_cap, span)
                           : pinned_block(c->h_pay, c->h_pay_cap, span);
          // staged in 64 MiB pieces, each uploaded as soon as it is staged
          // (the first batch's upload overlaps its own staging)
          constexpr int64_t kPiece = 64ll << 20;
          for (int64_t o = 0; o < span; o += kPiece) {
            const int64_t len = std::min(kPiece, span - o);
            parallel_memcpy(hp + o, psrc + o, (size_t)len);
            CK(cudaMemcpyAsync(c->d_stage + o, hp + o, len, cudaMemcpyHostToDevice, st));
          }
        } else {
          CK(cudaMemcpyAsync(c->d_stage, psrc, span,
                             (flags & EBCC_INPUT_ON_DEVICE) ? cudaMemcpyDeviceToDevice
                                                            : cudaMemcpyHostToDevice,
                             st));
        }
        CK(cudaEventRecord(c->ev_pbuf[bk], st));
        if ((int)up.size() > c->unpack_cap) {
          if (c->d_unpack) cudaFree(c->d_unpack);
          c->unpack_cap = (int)up.size() * 2;
          c->d_unpack = dalloc<UnpackPart>(c->unpack_cap);
        }
        g_trace.add(0, "dec_payload_staged", -1);
        h2d_small(c, c->d_unpack, up.data(), sizeof(UnpackPart) * up.size(), st);
        unpack_parts(c->d_unpack, (int)up.size(), c->d_stage, st);
        c->stats.kernel_launches++;
      }
      std::vector<ProbeParam> prm(nb);
      float* dst = out + f0 * g.n;
      float* out_dev = dst;
      if (!(flags & EBCC_OUTPUT_ON_DEVICE)) {
        // (a second buffer only when there is a next batch to overlap)
        out_dev = (bk && nfields > cap) ? device_block(c->d_out2, c->out2_cap, g.n * nb)
                                        : device_block(c->d_out, c->out_cap, g.n * nb);
        // its previous device->host copy (two batches ago) must be done
        if (used[bk]) CK(cudaStreamWaitEvent(st, c->ev_obuf[bk], 0));
      }
      used[bk] = true;
      // two decodes: the residual stream (midpoint) on the high-priority side
      // stream with its own decoder state, concurrently with the base stream
      // (lower bound) on `st`; joined before the residual field is added to
      // the base field
      bool any_res = false;
      for (int i = 0; i < nb; i++) any_res |= ract[i] != 0;
      if (any_res) {
        ensure_dec2(w);
        MachineBufs rb = machine_bufs_dec2(w, nb);
        CK(cudaEventRecord(c->ev_a, st));  // streams unpacked
        CK(cudaStreamWaitEvent(c->side, c->ev_a, 0));
        h2d_small(c, rb.out, rmo.data(), sizeof(MachineOut) * nb, c->side);
        h2d_small(c, w.dec2.limit, rlim.data(), sizeof(uint64_t) * nb, c->side);
        std::vector<uint8_t> mact(nb);
        for (int i = 0; i < nb; i++) mact[i] = ract[i] && rmo[i].n_max != kExpNone;
        h2d_small(c, w.dec2.active, mact.data(), nb, c->side);
        decode_init(rb, c->side, w.rank_hi2 ? nullptr : w.packed2);
        // one CTA per chunk: fits beside the base machine's clusters
        // (EBCC_DEC_RES_CLUSTER: A/B runs)
        static const int res_cluster =
            getenv("EBCC_DEC_RES_CLUSTER") ? std::max(1, atoi(getenv("EBCC_DEC_RES_CLUSTER"))) : 1;
        run_machine(true, rb, g, w.tt, kMaxDecodePlanes, c->side, res_cluster);
        if (w.rank_hi2) {  // wide records: significands, then pack_meta
          gather_refinement(rb, c->side);
          pack_meta(rb, w.packed2, w.sprank2, c->side, nullptr, w.rank_hi2);
        } else {
          gather_pack(rb, w.packed2, w.sprank2, c->side);
        }
        CK(cudaEventRecord(c->ev_b, c->side));
        c->stats.kernel_launches += 4;
      }
      if (j2 == 1) {
        // opt-in J2 base layer: parse the units, MQ-decode every code-block,
        // inverse DWT into base_dec (all-zero streams decode to zeros)
        EbBufs& eb = ensure_ebcot(w, nb, st);
        std::vector<int32_t> enm(nb);
        std::vector<uint64_t> blen(nb, 0);
        std::vector<uint8_t> eact(nb);
        for (int i = 0; i < nb; i++) {
          enm[i] = bmo[i].n_max;
          eact[i] = !cst[i];
          if (!cst[i]) blen[i] = (uint64_t)(recs[f0 + i].base_len - kHeader);
        }
        h2d_small(c, eb.nmax, enm.data(), sizeof(int32_t) * nb, st);
        h2d_small(c, w.eb.body_len, blen.data(), sizeof(uint64_t) * nb, st);
        h2d_small(c, w.active, eact.data(), nb, st);
        CK(cudaMemsetAsync(eb.status, 0, sizeof(int32_t) * nb, st));
        ebcot_stream_decode(w.eb.geo, g, eb, w.active, w.base_dec, st);
        inverse_dwt(w.base_dec, w.B, g.n, nb, g, st);
        c->stats.kernel_launches += 2 + 2 * g.levels;
        std::vector<int32_t> est(nb);
        CK(cudaMemcpyAsync(est.data(), eb.status, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int i = 0; i < nb; i++)
          if (est[i]) return fail(c, EBCC_E_FORMAT, "malformed J2 base stream");
      } else {
        MachineBufs mb = machine_bufs(w, nb, false);
        h2d_small(c, mb.out, bmo.data(), sizeof(MachineOut) * nb, st);
        h2d_small(c, const_cast<uint64_t*>(w.limit), blim.data(), sizeof(uint64_t) * nb, st);
        std::vector<uint8_t> mact(nb);
        for (int i = 0; i < nb; i++) mact[i] = bact[i] && bmo[i].n_max != kExpNone;
        h2d_small(c, w.active, mact.data(), nb, st);
        decode_init(mb, st, w.rank_hi ? nullptr : w.packed);
        run_machine(true, mb, g, w.tt, kMaxDecodePlanes, st);
        if (w.rank_hi) {
          gather_refinement(mb, st);
          pack_meta(mb, w.packed, w.sprank, st, nullptr, w.rank_hi);
        } else {
          gather_pack(mb, w.packed, w.sprank, st);
        }
        c->stats.kernel_launches += 4;
      }
      g_trace.add(0, "dec_machines_issued", -1);
      bool res_joined = false;  // st has waited for the residual decoder
      bool xe_b = false, xe_r = false;  // stream exponents outside the normal range
      for (int i = 0; i < nb; i++) {
        if (bact[i] && bmo[i].n_max != kExpNone) xe_b |= exps_extreme(bmo[i].n_max);
        if (ract[i] && rmo[i].n_max != kExpNone) xe_r |= exps_extreme(rmo[i].n_max);
      }
      // IDWT + denormalise in field groups; with a page-locked host
      // destination each group's device->host copy (copy stream) overlaps
      // the next group's IDWT
      const bool to_host = !(flags & EBCC_OUTPUT_ON_DEVICE);
      const bool pageable = to_host && is_pageable(dst);
      static const int groups_env =
          getenv("EBCC_DEC_GROUPS") ? std::max(1, atoi(getenv("EBCC_DEC_GROUPS"))) : 4;
      const int G = (to_host && !pageable && nb >= 2 * groups_env) ? groups_env : 1;
      if (G > 1 && !c->copy) {
        CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming));
      }
      while ((int)c->ev_groups.size() < G) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_groups.push_back(e);
      }
      for (int j = 0; j < G; j++) {
        const int a = (int)((int64_t)nb * j / G), b = (int)((int64_t)nb * (j + 1) / G);
        bool g_res = false;
        std::vector<uint8_t> gpure(nb, 0), gcst(nb, 0);
        for (int i = 0; i < nb; i++) {
          const bool in = i >= a && i < b;
          prm[i] = ProbeParam{};
          prm[i].B = ~0ull;
          prm[i].planes = -1;
          prm[i].active = in && !cst[i];
          g_res |= in && ract[i];
          gpure[i] = in && pure[i];
          gcst[i] = in && cst[i];
        }
        h2d_small(c, w.prm, prm.data(), sizeof(ProbeParam) * nb, st);
        if (j2 != 1) {  // (a J2 base field is already in base_dec)
          decode_field(meta_of(w, false), w.prm, w.A, w.B, g, nb, w.base_dec, st, xe_b);
          c->stats.kernel_launches += g.levels;
        }
        CK(cudaGetLastError());
        if (g_slow.on()) {
          CK(cudaStreamSynchronize(st));
          g_slow.mark("dec_base");
        }
        if (g_res) {
          if (!res_joined) CK(cudaStreamWaitEvent(st, c->ev_b, 0));
          res_joined = true;
          for (int i = 0; i < nb; i++) {
            prm[i] = ProbeParam{};
            prm[i].B = ~0ull;
            prm[i].planes = -1;
            prm[i].midpoint = 1;
            prm[i].active = i >= a && i < b && ract[i];
          }
          h2d_small(c, w.prm, prm.data(), sizeof(ProbeParam) * nb, st);
          decode_field_add_denorm(meta_of(w, true), w.prm, w.A, w.B, g, nb, w.base_dec, w.fs,
                                  out_dev, st, xe_r);
          c->stats.kernel_launches += g.levels;
          CK(cudaGetLastError());
        }
        h2d_small(c, w.active, gpure.data(), nb, st);
        denorm_only(w.base_dec, w.fs, w.active, g.n, nb, out_dev, st);
        h2d_small(c, w.active, gcst.data(), nb, st);  // stream-ordered after denorm_only
        fill_constant(w.fs, w.active, g.n, nb, out_dev, st);
        c->stats.kernel_launches += 2;
        CK(cudaGetLastError());
        if (G > 1) {
          CK(cudaEventRecord(c->ev_groups[j], st));
          CK(cudaStreamWaitEvent(c->copy, c->ev_groups[j], 0));
          CK(cudaMemcpyAsync(dst + (int64_t)a * g.n, out_dev + (int64_t)a * g.n,
                             sizeof(float) * g.n * (b - a), cudaMemcpyDeviceToHost, c->copy));
        }
      }
      g_trace.add(0, "dec_idwt_issued", -1);
      if (any_res && !res_joined) CK(cudaStreamWaitEvent(st, c->ev_b, 0));
      if (G > 1) {
        CK(cudaEventRecord(c->ev_obuf[bk], c->copy));
      } else if (to_host) {
        const size_t ob = sizeof(float) * g.n * nb;
        if (pageable) {
          uint8_t* stg = host_stage(c, (int64_t)ob);
          CK(cudaMemcpyAsync(stg, out_dev, ob, cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          parallel_memcpy(dst, stg, ob);
        } else {
          CK(cudaMemcpyAsync(dst, out_dev, ob, cudaMemcpyDeviceToHost, st));
        }
        CK(cudaEventRecord(c->ev_obuf[bk], st));
      }
      if (g_slow.on()) CK(cudaStreamSynchronize(st));
    }
    if (c->copy) {  // the last batches' device->host copies
      CK(cudaEventRecord(c->ev_copy, c->copy));
      CK(cudaStreamWaitEvent(st, c->ev_copy, 0));
    }
    CK(cudaStreamSynchronize(st));
    g_trace.add(0, "dec_batches_done", -1);
    cudaEventRecord(t1, st);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    c->stats.ms_total = ms;
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, e.e == cudaErrorMemoryAllocation ? EBCC_E_NOMEM : EBCC_E_CUDA,
                std::string(e.what) + ": " + cudaGetErrorString(e.e));
  } catch (std::exception& e) {
    return fail(c, EBCC_E_CUDA, e.what());
  }
}

int ebcc_dwt(ebcc_ctx* c, const double* in, double* out, int64_t nfields, int32_t rows,
             int32_t cols, int32_t levels, int32_t inverse) {
  if (!c || !in || !out || nfields < 1 || rows < 1 || cols < 1 || levels < 1 ||
      levels > kMaxLevels)
    return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  try {
    CK(cudaSetDevice(c->device));
    if (!inverse) levels = clamp_levels(rows, cols, levels);
    Geo g = make_geo(rows, cols, levels);
    ensure_workspace(c, g, (int)nfields);
    Workspace& w = c->ws;
    CK(cudaMemcpyAsync(w.A, in, sizeof(double) * g.n * nfields, cudaMemcpyHostToDevice, c->stream));
    if (inverse) inverse_dwt(w.A, w.B, g.n, (int)nfields, g, c->stream);
    else forward_dwt(w.A, w.B, g.n, (int)nfields, g, c->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, w.A, sizeof(double) * g.n * nfields, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, EBCC_E_CUDA, std::string(e.what) + ": " + cudaGetErrorString(e.e));
  }
}

int ebcc_spiht_encode(ebcc_ctx* c, const double* coeffs, int32_t rows, int32_t cols,
                      int32_t levels, int32_t planes, uint8_t* out, int64_t cap, int64_t* len) {
  if (!c || !coeffs || !out || rows < 1 || cols < 1 || levels < 1 || levels > kMaxLevels ||
      planes < 1 || planes > kDeepPlanes || cap < kHeader)
    return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  if ((int64_t)rows * cols > kMaxChunkPoints) return fail(c, EBCC_E_ARGUMENT, "chunk too large");
  try {
    CK(cudaSetDevice(c->device));
    Geo g = make_geo(rows, cols, levels);
    ensure_workspace(c, g, 1);
    Workspace& w = c->ws;
    CK(cudaMemcpyAsync(w.A, coeffs, sizeof(double) * g.n, cudaMemcpyHostToDevice, c->stream));
    std::vector<uint8_t> act(1, 1);
    std::vector<MachineOut> mo(1);
    std::vector<PlaneRec> pl(kMaxPlaneRecs);
    encode_pyramids(c, 1, true, planes, act, mo, pl);
    uint8_t hdr[kHeader];
    if (mo[0].n_max == kExpNone) {
      put_header(hdr, kZeroSentinel, levels, rows, cols);
      memcpy(out, hdr, kHeader);
      *len = kHeader;
      return EBCC_OK;
    }
    int64_t nbytes = kHeader + (int64_t)((mo[0].total_bits + 7) / 8);
    *len = nbytes;
    if (nbytes > cap) return fail(c, EBCC_E_CAPACITY, "output buffer too small");
    put_header(out, mo[0].n_max, levels, rows, cols);
    if (nbytes > kHeader)
      CK(cudaMemcpy(out + kHeader, w.bits_res, nbytes - kHeader, cudaMemcpyDeviceToHost));
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, EBCC_E_CUDA, std::string(e.what) + ": " + cudaGetErrorString(e.e));
  }
}

namespace {
// ebcc_spiht_decode / ebcc_decode_field: decoder machine on one stream prefix,
// then either the coefficients (decode_coeffs) or the field through the
// production fused inverse transform (decode_field)
int decode_one(ebcc_ctx* c, const uint8_t* data, int64_t len, int64_t prefix_len, int32_t rows,
               int32_t cols, double* coeffs_out, int32_t* n_last, double* field_out,
               int32_t midpoint);
}  // namespace

int ebcc_spiht_decode(ebcc_ctx* c, const uint8_t* data, int64_t len, int64_t prefix_len,
                      int32_t rows, int32_t cols, double* coeffs_out, int32_t* n_last) {
  if (!c || !data || !coeffs_out || !n_last || rows < 1 || cols < 1)
    return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  return decode_one(c, data, len, prefix_len, rows, cols, coeffs_out, n_last, nullptr, 0);
}

int ebcc_decode_field(ebcc_ctx* c, const uint8_t* data, int64_t len, int64_t prefix_len,
                      int32_t rows, int32_t cols, int32_t midpoint, double* field_out) {
  if (!c || !data || !field_out || rows < 1 || cols < 1)
    return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  int32_t nl = 0;
  return decode_one(c, data, len, prefix_len, rows, cols, nullptr, &nl, field_out, midpoint);
}

}  // extern "C"

namespace {
int decode_one(ebcc_ctx* c, const uint8_t* data, int64_t len, int64_t prefix_len, int32_t rows,
               int32_t cols, double* coeffs_out, int32_t* n_last, double* field_out,
               int32_t midpoint) {
  if ((int64_t)rows * cols > kMaxChunkPoints) return fail(c, EBCC_E_ARGUMENT, "chunk too large");
  if (len < kHeader || data[0] != 'S' || data[1] != 'P') return fail(c, EBCC_E_FORMAT, "bad header");
  int levels = data[3];
  uint32_t hr, hc;
  memcpy(&hr, data + 4, 4);
  memcpy(&hc, data + 8, 4);
  if ((int)hr != rows || (int)hc != cols || levels < 1 || levels > kMaxLevels)
    return fail(c, EBCC_E_FORMAT, "header does not match");
  if (prefix_len < 0 || prefix_len > len) prefix_len = len;
  try {
    CK(cudaSetDevice(c->device));
    Geo g = make_geo(rows, cols, levels);
    ensure_workspace(c, g, 1);
    Workspace& w = c->ws;
    cudaStream_t st = c->stream;
    int nm = (int8_t)data[2];
    std::vector<MachineOut> mo(1);
    mo[0] = MachineOut{};
    mo[0].n_max = nm == kZeroSentinel ? kExpNone : nm;
    uint64_t lim = prefix_len > kHeader ? (uint64_t)(prefix_len - kHeader) * 8 : 0;
    int64_t pbytes = prefix_len > kHeader ? prefix_len - kHeader : 0;
    if ((pbytes + 3) / 4 + 2 > w.words_res) return fail(c, EBCC_E_FORMAT, "stream too long");
    CK(cudaMemsetAsync(w.bits_res, 0, sizeof(uint32_t) * w.words_res, st));
    if (pbytes) CK(cudaMemcpyAsync(w.bits_res, data + kHeader, pbytes, cudaMemcpyHostToDevice, st));
    MachineBufs mb = machine_bufs(w, 1, true);
    CK(cudaMemcpyAsync(mb.out, mo.data(), sizeof(MachineOut), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.limit, &lim, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    uint8_t act = nm != kZeroSentinel;
    CK(cudaMemcpyAsync(w.active, &act, 1, cudaMemcpyHostToDevice, st));
    decode_init(mb, st, w.rank_hi2 ? nullptr : w.packed2);
    run_machine(true, mb, g, w.tt, kMaxDecodePlanes, st);
    if (w.rank_hi2) {
      gather_refinement(mb, st);
      pack_meta(mb, w.packed2, w.sprank2, st, nullptr, w.rank_hi2);
    } else {
      gather_pack(mb, w.packed2, w.sprank2, st);
    }
    ProbeParam p{};
    p.B = ~0ull; p.planes = -1; p.active = 1;
    // (an all-zero stream has no n_last: dequantized_field adds no offset)
    p.midpoint = (midpoint && nm != kZeroSentinel) ? 1 : 0;
    CK(cudaMemcpyAsync(w.prm, &p, sizeof(p), cudaMemcpyHostToDevice, st));
    if (field_out) {
      decode_field(meta_of(w, true), w.prm, w.A, w.B, g, 1, w.base_dec, st,
                   nm != kZeroSentinel && exps_extreme(nm), p.midpoint != 0);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(field_out, w.base_dec, sizeof(double) * g.n, cudaMemcpyDeviceToHost, st));
    } else {
      decode_coeffs(meta_of(w, true), w.prm, w.A, g.n, 1, st);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(coeffs_out, w.A, sizeof(double) * g.n, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(mo.data(), mb.out, sizeof(MachineOut), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (nm == kZeroSentinel) *n_last = -999;
    else *n_last = mo[0].planes_run > 0 ? nm - (mo[0].planes_run - 1) : nm;
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, EBCC_E_CUDA, std::string(e.what) + ": " + cudaGetErrorString(e.e));
  }
}
}  // namespace

extern "C" {

// page-locked result blocks: size-keyed free list, bounded cache
namespace {
std::mutex g_pin_mu;
std::multimap<int64_t, void*> g_pin_free;
std::unordered_map<void*, int64_t> g_pin_size;
int64_t g_pin_cached = 0;
// freed page-locked blocks kept for reuse: up to a quarter of host RAM
// (pinning a 9.8 GB result block costs seconds; reusing it nothing)
int64_t pin_cache_max() {
  static const int64_t m = [] {
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGE_SIZE);
    const int64_t ram = pages > 0 && psz > 0 ? (int64_t)pages * psz : (int64_t)32 << 30;
    return std::max<int64_t>((int64_t)8 << 30, ram / 4);
  }();
  return m;
}

// A page-locked block: anonymous mmap (transparent huge pages), first-touched
// by the host thread team, then cudaHostRegister'ed.  Measured on a B200 box
// for 9.8 GB: cudaHostAlloc 6.8 s; register of touched memory 0.2 s.
void* pin_block_alloc(size_t bytes) {
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return nullptr;
  madvise(p, bytes, MADV_HUGEPAGE);
  parallel_touch(p, bytes);
  if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) != cudaSuccess) {
    cudaGetLastError();
    munmap(p, bytes);
    return nullptr;
  }
  return p;
}
void pin_block_free(void* p, size_t bytes) {
  cudaHostUnregister(p);
  munmap(p, bytes);
}

void pin_release_cached_locked() {
  for (auto& kv : g_pin_free) {
    g_pin_size.erase(kv.second);
    pin_block_free(kv.second, (size_t)kv.first);
  }
  g_pin_free.clear();
  g_pin_cached = 0;
}
}  // namespace

int ebcc_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return EBCC_E_ARGUMENT;
  if (bytes == 0) bytes = 1;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  auto it = g_pin_free.lower_bound(bytes);
  if (it != g_pin_free.end() && it->first <= 2 * bytes) {
    *out = it->second;
    g_pin_cached -= it->first;
    g_pin_free.erase(it);
    return EBCC_OK;
  }
  void* p = pin_block_alloc((size_t)bytes);
  if (!p) {
    pin_release_cached_locked();
    p = pin_block_alloc((size_t)bytes);
    if (!p) return EBCC_E_NOMEM;
  }
  g_pin_size[p] = bytes;
  *out = p;
  return EBCC_OK;
}

void ebcc_host_cache_trim(void) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  pin_release_cached_locked();
}

int ebcc_host_free(void* p) {
  if (!p) return EBCC_OK;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  auto it = g_pin_size.find(p);
  if (it == g_pin_size.end()) return EBCC_E_ARGUMENT;
  g_pin_free.insert({it->second, p});
  g_pin_cached += it->second;
  while (g_pin_cached > pin_cache_max() && !g_pin_free.empty()) {
    auto v = g_pin_free.begin();  // smallest first
    g_pin_cached -= v->first;
    g_pin_size.erase(v->second);
    pin_block_free(v->second, (size_t)v->first);
    g_pin_free.erase(v);
  }
  return EBCC_OK;
}

// developer instrumentation: time full (non-incremental) base probes of the
// last compress batch on this context (single-lane calls) at B = frac * T_base
int ebcc_dev_probe_bench(ebcc_ctx* c, double frac, int32_t iters, int32_t early, double* us_l0,
                         double* us_probe) {
  if (!c || iters < 1 || !us_l0 || !us_probe) return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  Workspace& w = c->ws;
  const int nf = c->last_batch;
  if (nf < 1 || !w.packed) return fail(c, EBCC_E_ARGUMENT, "no compress batch on this context");
  try {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    std::vector<MachineOut> mo(nf);
    CK(cudaMemcpy(mo.data(), w.mo_base, sizeof(MachineOut) * nf, cudaMemcpyDeviceToHost));
    std::vector<ProbeParam> prm(nf);
    for (int f = 0; f < nf; f++) {
      prm[f] = ProbeParam{};
      prm[f].B = (uint64_t)(frac * mo[f].total_bits);
      prm[f].planes = kBasePlanes;
      prm[f].active = mo[f].n_max != kExpNone;
      prm[f].early = early;
    }
    CK(cudaMemcpy(w.prm, prm.data(), sizeof(ProbeParam) * nf, cudaMemcpyHostToDevice));
    Meta mb = meta_of(w, false);
    bool xe = false;
    for (int f = 0; f < nf; f++)
      if (mo[f].n_max != kExpNone) xe |= exps_extreme(mo[f].n_max);
    double l0 = 0, all = 0;
    for (int it = 0; it < iters + 1; it++) {
      CK(cudaMemsetAsync(w.res, 0, sizeof(ProbeResult) * nf, st));
      CK(cudaEventRecord(c->tm_a, st));
      fused::g_level0_timer = &c->l0;
      probe_base(mb, w.prm, w.A, w.B, w.g, nf, w.norm, w.x32, w.fs, w.res, st, nullptr, xe,
                 early != 0);
      fused::g_level0_timer = nullptr;
      CK(cudaEventRecord(c->tm_b, st));
      CK(cudaStreamSynchronize(st));
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, c->l0.a, c->l0.b);
      cudaEventElapsedTime(&b, c->tm_a, c->tm_b);
      if (it > 0) { l0 += a; all += b; }
    }
    *us_l0 = 1e3 * l0 / iters;
    *us_probe = 1e3 * all / iters;
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, EBCC_E_CUDA, std::string(e.what) + ": " + cudaGetErrorString(e.e));
  }
}

// container.read_file's record walk (container.py:82-145): records are
// variable-length (25 B + payload), so the walk is sequential; a native loop
// over 2,368 records takes microseconds (the Python loop: ~10 ms).
int ebcc_parse_records(const uint8_t* data, int64_t len, int64_t count, uint8_t* records25,
                       int64_t* offsets, int64_t* err_offset, int32_t* err_aux) {
  if (!data || count < 0 || (count && (!records25 || !offsets)) || !err_offset || !err_aux)
    return EBCC_E_ARGUMENT;
  *err_offset = -1;
  *err_aux = 0;
  int64_t pos = 42;
  for (int64_t i = 0; i < count; i++) {
    if (pos + 25 > len) { *err_offset = pos; *err_aux = 1; return EBCC_E_FORMAT; }
    const uint8_t mode = data[pos];
    if (mode > 2) { *err_offset = pos; *err_aux = 2; return EBCC_E_FORMAT; }
    memcpy(records25 + 25 * i, data + pos, 25);
    uint32_t bl, rl;
    memcpy(&bl, data + pos + 17, 4);
    memcpy(&rl, data + pos + 21, 4);
    pos += 25;
    const int64_t n = (int64_t)bl + (int64_t)rl;
    if (pos + n > len) { *err_offset = pos; *err_aux = 3; return EBCC_E_FORMAT; }
    offsets[i] = pos;
    pos += n;
  }
  if (pos != len) { *err_offset = pos; *err_aux = 4; return EBCC_E_FORMAT; }
  return EBCC_OK;
}

// decompress_chunk's stream-header checks (pipeline.py:336-353,
// spiht.parse_header spiht.py:67-78) for same-shape chunks: 'SP' magic,
// positive dims equal to (rows, cols), levels >= 1 and <= 5, residual levels
// equal to the base's.  *levels = the common level count (0 if every chunk is
// constant); EBCC_E_FORMAT names the first bad chunk in *bad (its exact
// reference message is produced by the caller); a chunk whose level count
// differs from the first one's returns EBCC_E_ARGUMENT (mixed depths).
int ebcc_check_streams(const uint8_t* data, int64_t len, const uint8_t* records25,
                       const int64_t* offsets, int64_t n, int32_t rows, int32_t cols,
                       int32_t* levels, int64_t* bad) {
  if (!data || n < 0 || (n && (!records25 || !offsets)) || !levels || !bad) return EBCC_E_ARGUMENT;
  *levels = 0;
  *bad = -1;
  // base streams may also be 'J2' (the opt-in JPEG2000-style layer)
  auto hdr_ok = [&](int64_t off, int64_t ln, int* lv, bool base) {
    if (ln < kHeader || off < 0 || off + ln > len) return false;
    const uint8_t* h = data + off;
    if (!(h[0] == 'S' && h[1] == 'P') && !(base && h[0] == 'J' && h[1] == '2')) return false;
    uint32_t r, c;
    memcpy(&r, h + 4, 4);
    memcpy(&c, h + 8, 4);
    if (r < 1 || c < 1 || h[3] < 1) return false;
    if ((int64_t)r != rows || (int64_t)c != cols) return false;
    *lv = h[3];
    return true;
  };
  for (int64_t i = 0; i < n; i++) {
    const uint8_t* rec = records25 + 25 * i;
    const int mode = rec[0];
    if (mode == EBCC_MODE_CONSTANT) continue;
    uint32_t bl, rl;
    memcpy(&bl, rec + 17, 4);
    memcpy(&rl, rec + 21, 4);
    int lv = 0, rlv = 0;
    if (!hdr_ok(offsets[i], bl, &lv, true)) { *bad = i; return EBCC_E_FORMAT; }
    if (mode == EBCC_MODE_TWO_LAYER && rl > 0 &&
        (!hdr_ok(offsets[i] + bl, rl, &rlv, false) || rlv != lv)) { *bad = i; return EBCC_E_FORMAT; }
    if (lv > 5) { *bad = i; return EBCC_E_FORMAT; }
    if (*levels && lv != *levels) { *bad = i; return EBCC_E_ARGUMENT; }
    *levels = lv;
  }
  return EBCC_OK;
}

int ebcc_selftest_div(ebcc_ctx* c, int64_t n, uint64_t seed, int64_t* mismatches) {
  if (!c || !mismatches || n < 1) return fail(c, EBCC_E_ARGUMENT, "bad arguments");
  try {
    CK(cudaSetDevice(c->device));
    unsigned long long* d = dalloc<unsigned long long>(1);
    CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->stream));
    selftest_div(n, seed, d, c->stream);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d);
    *mismatches = (int64_t)h;
    return EBCC_OK;
  } catch (CudaFail& e) {
    cudaGetLastError();
    return fail(c, EBCC_E_CUDA, std::string(e.what) + ": " + cudaGetErrorString(e.e));
  }
}

}  // extern "C"
