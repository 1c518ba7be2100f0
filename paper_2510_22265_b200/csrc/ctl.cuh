// Device-resident feedback controller (ctl.cu).
//
// The reference's three searches - _search_base (pipeline.py:142-199),
// _search_pure (215-236) and _truncation_search (243-254) - restated as
// per-chunk resumable state machines that live in device memory and are
// advanced by one thread per chunk between two batched probes.  A state
// machine runs straight-line until it needs a memo entry that does not exist
// yet; it then posts that probe (a ProbeParam) and suspends.  The loop
//   while (any chunk posted a probe) { probe all posted; advance all }
// is a CUDA graph with conditional WHILE nodes whose condition the advance
// kernel sets on the device: no host round trip between probes.
//
// Straight-line execution is what the reference does, so the memo at every
// point holds exactly the entries the reference's dict holds there; the
// seeding loops over "all cached budgets" (pipeline.py:193-198, 227-234)
// need no replay bookkeeping.  Budgets use CPython float floor division
// (base_codec.py:38); ratios, q and errors are the same doubles as the
// reference's.
#pragma once
#include <cuda_runtime.h>

#include "probe.cuh"
#include "spiht.cuh"

namespace ebcc {

constexpr int kCtlMemo = 256;    // distinct base budgets per chunk
constexpr int kCtlTMemo = 160;   // truncation offsets per planes variant
constexpr int kCtlSlots = 3;     // probes per chunk and step of each search
constexpr int kCtlSMemo = 64;    // speculative base-memo entries per chunk
constexpr int kCtlSmemChunks = 12;  // chunk states a controller CTA stages in shared memory

struct CtlEntry {
  int64_t budget;
  unsigned long long count;
  double maxerr;
};
struct CtlTEntry {
  int64_t t;
  double err;
};

// status bits of a chunk's controller
constexpr int kCtlCapacity = 1;  // a memo or a loop guard overflowed

struct CtlChunk {
  // --- inputs (ctl_setup / ctl_*_start) ---
  int64_t n, raw;
  double q, r0, tol, eps_abs;
  uint64_t T_base, T24, T32;
  int32_t active;        // not constant, finite input
  int32_t status;
  int32_t vlim, pad_v;   // violations a count probe may see and still reach q
  // opt-in J2 base layer (ebcot.cuh): the stream served for a budget is the
  // longest unit-aligned prefix; eb_cum[k] = body bytes of the first k slots
  const uint32_t* eb_cum;  // null: SPIHT base (prefix = the budget's bytes)
  int32_t eb_sub, eb_nslot;  // block-table bytes (0: all-zero pyramid), slots
  // --- base memo (shared by the base and the pure-base searches) ---
  int32_t nmemo, pend;   // pend: memo budget of the probe in flight (-1 none)
  int64_t pend_budget;
  CtlEntry memo[kCtlMemo];
  // speculative base-memo probes (the budgets the base / pure-base search
  // asks next whichever way the probe in flight answers): answers park here
  // and move into `memo` only when the search asks for that budget, so the
  // memo always holds exactly the reference's entries
  int64_t bspec[2];                // next-step keys of the access in progress (-1 none)
  int64_t bspend[kCtlSlots - 1];   // their probes in flight (-1 none)
  int32_t nsmemo, pad_s;
  CtlEntry smemo[kCtlSMemo];
  // --- the access each coroutine is at: key and memo index ---
  int64_t want_b, want_p, want_t;
  int32_t cur_b, cur_p, cur_t, pad1;
  // --- _search_base ---
  int32_t pc_b, guard;
  double r_cap, r0c, q_a0, q_a, r_low, r_high, r_mid;
  int32_t have, done_b;
  int64_t lo_b, hi_b, mid_b, base_budget;
  // --- _search_pure ---
  int32_t pc_p, done_p, ci, ncached;
  int64_t lo_p, hi_p, mid_p, pure_budget;
  int64_t p_lb, p_ub;
  int32_t pure_pruned, pad0;
  int64_t cached[kCtlMemo];
  // --- _truncation_search (24, then 32 planes) ---
  int32_t pc_t, pass, done_t, ntcalls, ncalls_pass, trunc_planes;
  int64_t lo_t, hi_t, mid_t, total_t, trunc_t;
  int64_t t_lb, t_ub;
  int64_t spec[2];
  int32_t trunc_pruned, tpend_pi;
  int64_t tpend[kCtlSlots];       // offsets of the truncation probes in flight (-1 none)
  int32_t ntmemo[2];
  CtlTEntry tmemo[2][kCtlTMemo];
};

// per-chunk result the host reads once per batch
struct CtlOut {
  int32_t status;        // kCtlCapacity bits
  int32_t active;
  int64_t base_budget, pure_budget, trunc_t;
  int32_t trunc_planes;
  int32_t n_base_probes, n_trunc_probes;
  int32_t pure_pruned, trunc_pruned;
  int32_t pad;
  uint64_t T_base, T24, T32;
  int64_t len_base, len_pure;  // stream lengths of the chosen budgets (-1: none)
};

// per-call parameters (device resident, written before each batch)
struct CtlParams {
  double q, r0, tol;
  int32_t prune, early, slots, pad;
};

// counters of one batch (instrumentation)
struct CtlStats {  // controller steps, and steps that launched probes of each kind
  unsigned long long base_steps, joint_steps, base_probes, pure_probes, trunc_probes;
  // nonzero once the residual encode has finished: a pure-base loop running
  // beside it hands its (suspended) search to the joint loop
  unsigned long long stop;
};

struct CtlArgs {
  CtlChunk* cs;
  CtlOut* out;
  const CtlParams* prm_in;
  CtlStats* stats;
  const FieldScal* fs;
  MachineOut* mo_base;
  MachineOut* mo_res;
  const PlaneRec* pl_res;
  uint8_t* active;
  ProbeParam* prm;        // base-stream probes (bslots x nfields, probe v -> chunk v % nfields)
  ProbeResult* res;
  ProbeParam* tprm;       // truncation probes (slots x nfields, probe v -> chunk v % nfields)
  ProbeResult* tres;
  int nfields;
  int slots;              // truncation probe slots
  int bslots;             // base-stream probe slots (1: no speculation)
  int smem;               // the chunks' states fit the controller CTA's shared memory
  int jmode;              // ctl_joint advances: 1 the pure-base search, 2 truncation, 3 both
  int64_t n;
  cudaGraphConditionalHandle h_loop;   // WHILE condition of the current loop
  cudaGraphConditionalHandle h_pure;   // IF: the pure-base branch has probes
  cudaGraphConditionalHandle h_trunc;  // IF: the truncation branch has probes
  // opt-in J2 base layer: per chunk (eb_nb * 72 + 1) cumulative unit bytes,
  // n_max (null: SPIHT base)
  const uint32_t* eb_cum;
  const int32_t* eb_nmax;
  int eb_nb;
};

// CtlArgs::smem may be set (the states fit the controller's shared memory)
bool ctl_smem_ok(int nfields);
// active flags, machine-output init and controller state of every chunk
void ctl_setup(const CtlArgs& a, cudaStream_t st);
// `set` selects the conditional handles a launch writes: 1 h_loop, 2 h_pure,
// 4 h_trunc (a launch outside a handle's graph writes none).
// base search: start (T_base) + ingest the last probe's results + advance +
// post the next probes
void ctl_base(const CtlArgs& a, bool start, int set, cudaStream_t st);
// ProbeParam of the chosen base budget for base_to_residue
void ctl_residue(const CtlArgs& a, cudaStream_t st);
// pure-base + truncation searches: start = T24 / T32 only; otherwise ingest
// + advance the searches `jmode` selects + candidate pruning + post.  A
// pure-only loop (jmode 1) may run beside the residual encode: it touches no
// truncation state, and its answer is never pruned (the truncation search,
// run after it, is pruned against it)
void ctl_joint(const CtlArgs& a, bool start, int set, cudaStream_t st);
// candidate-choice inputs of every chunk into CtlOut
void ctl_finalize(const CtlArgs& a, cudaStream_t st);

}  // namespace ebcc
