// Field-level kernels: ingest/normalise, closed-form prefix decode, the
// feedback probes (decode -> IDWT -> fused reduction), residue formation,
// decompress tails and payload (un)packing (probe.cu).
#pragma once
#include "common.cuh"
#include "spiht.cuh"

namespace ebcc {

// per-field scalars shared by all probes
struct FieldScal {
  double vmin, vmax, range;  // range = vmax - vmin (float64, like the reference)
  double range_inv;          // RN(1/range), for the FMA-corrected exact division
  double eps_rel, eps_abs;
  int32_t constant;
  int32_t pad;
  long long first_bad;       // first non-finite element of the chunk, -1 if none
};

// what one probe decodes
struct ProbeParam {
  uint64_t B;          // stream bits available: positions < B were read
  int32_t planes;      // refinement planes present (24/32 variant); -1: take
                       // planes_run / n_last from the decoder machine
  int32_t midpoint;    // add sign * 2^(n_last-1) (residual layer)
  int32_t n_last;
  int32_t active;
  // the caller only needs max_err <= eps_abs (pure-base and truncation
  // probes): CTAs starting after another CTA has already seen an error above
  // eps_abs skip their work.  Base-search (count) probes: the caller only
  // needs count/n >= q and max_err <= eps_abs; once more than `vlim` points
  // miss eps_rel and an error above eps_abs was seen, both answers are "no"
  // and the probe may stop likewise.
  int32_t early;
  int32_t vlim;        // count probes: n - (smallest count c with c/n >= q)
};

struct ProbeResult {
  // count probes: #points with !(|dec - norm| <= eps_rel), pushed by the
  // warps as they find them (a probe that stopped early holds more than vlim)
  unsigned long long count;
  unsigned long long maxerr;  // bits of max |f32(denorm(rec)) - orig| (non-negative double)
};

// Per-coefficient closed-form metadata packed for the probes: one 16-byte
// load per coefficient = {sign bit offset, LSP rank, top-32 significand bits,
// pinfo (plane index | sign << 7)}.
// Per-coefficient probe record, 8 bytes (the dominant probe stream):
//   x = LSP rank (26 bits; kRankNone = never placed) | significance plane << 26
//   y = negative << 31 | the 31 significand bits after the leading one
// The sign bit offset is not stored: it grows with the LSP rank, so "sign bit
// read within B bits" is rank < R(B), R(B) found once per probe by a binary
// search over the sign offsets in rank order (Meta::sprank).
// Chunks of more than 2^26 - 2 points ("wide" chunks) keep the record and
// store the rank's bits 26..31 in a side byte per coefficient (rank_hi; a
// never-placed coefficient has rank 2^32 - 1); their level kernels are the
// XE instantiations, which read the byte (one more byte load per sample).
constexpr uint32_t kRankBits = 26;
constexpr uint32_t kRankNone = (1u << kRankBits) - 1;
constexpr int64_t kMaxNarrowPoints = (int64_t)kRankNone - 1;
// bit offsets and LSP ranks are 32-bit: chunks up to 2^32 - 2 points (a
// stream that outgrows 2^32 bits is reported as a capacity error)
constexpr int64_t kMaxChunkPoints = (int64_t)0xfffffffe;

struct Meta {  // one field = `stride` entries
  const uint2* packed;
  const uint8_t* rank_hi;  // wide chunks: rank bits 26..31 per coefficient (else null)
  // non-null: the coefficients are this f64 pyramid (stride `stride`), not
  // closed-form decodes of records (the opt-in J2 base layer's probes; the
  // XE instantiations read it, like rank_hi)
  const double* coef;
  const uint32_t* sprank;  // sign bit offset by LSP rank (kNone: sign not read)
  const PlaneRec* planes;
  const MachineOut* mo;
  int64_t stride;
  // per-probe decode tables, kTqBytes per field (64 plane thresholds + the
  // rank-bucket table), built once per probe by inverse_fused's first kernel
  uint8_t* tq;
};
constexpr int kTqBytes = 64 * 4 + 2048 + 16;  // thresholds, bucket table, R(B)
constexpr int kTqRankOffset = 64 * 4 + 2048;

// ---- incremental probes ----------------------------------------------------
// Consecutive probes of one chunk's search read B and B' stream bits of the
// same stream.  A coefficient's decoded value changes only if its sign bit or
// one of its refinement bits lies in [min(B,B'), max(B,B')): the LSP ranks of
// the sign-offset range plus, per plane, one contiguous rank range of the
// refinement segment.  Every IDWT level is deterministic, so an output tile
// whose inputs did not change is bit-identical to the previous probe's: the
// probe recomputes only the tiles reachable from the changed coefficients,
// keeping each level's LL output (and level 0's per-tile count / max error)
// from the previous probe of the same stream.
constexpr int kIncMaxIv = kMaxPlaneRecs + 1;
struct IncState {        // the last probe of this chunk on this stream
  uint64_t B;
  int32_t planes, midpoint, n_last, valid;
};
struct IncPlan {         // this probe: changed LSP ranks as intervals
  int32_t full;          // recompute everything (no state, or too many changes)
  int32_t niv;
  uint32_t K;            // changed ranks in total
  int32_t dense0;        // so many changes that every level-0 tile is taken as dirty
  uint32_t start[kIncMaxIv];
  uint32_t pre[kIncMaxIv + 1];
};
struct TileStat {        // level-0 tile result of the last computation
  unsigned long long count, maxerr;
};
// tile flag bits: the tile must be recomputed / its count is not valid
constexpr uint8_t kTileDirty = 1, kTileCountStale = 2;
struct IncLevel {        // the level kernel's CTA tiling of region k
  int off;               // first flag of level k within a field's flags
  int ct, rt, th;        // column tiles (TW columns each), row tiles, rows per tile
  int R, C;
};
struct IncGeo {
  int levels, tiles;     // tiles = flag bytes per field
  int tiles0;            // level-0 tiles (TileStat entries per field)
  int cols;
  int lr[kMaxLevels + 1], lc[kMaxLevels + 1];
  IncLevel lv[kMaxLevels];
};
struct Inc {
  uint8_t* flags;              // per field: IncGeo::tiles
  IncPlan* plan;               // per field
  IncState* state;             // per field
  TileStat* ts;                // per field: IncGeo::tiles0
  const uint32_t* lspn;        // node by LSP rank (Meta::stride per field)
  unsigned long long* computed;  // [kMaxLevels] tiles computed (instrumentation)
  int64_t lstride;             // per-field stride of the persistent LL buffer
  uint32_t klimit;             // more changed ranks than this: recompute in full
  int32_t debug;               // EBCC_INC_LOG: per-probe plan of chunk 0 (printf)
  int coloff[kMaxLevels + 1];  // column offset of level k's LL output in it
  IncGeo ig;
};

// GPU self-test: FMA-corrected exact divisions vs __ddiv_rn on n random cases
void selftest_div(int64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t st);

// build Meta::packed from the machine's per-coefficient arrays
void pack_meta(const MachineBufs& mb, uint2* packed, uint32_t* sprank, cudaStream_t st,
               uint32_t* lspn = nullptr, uint8_t* rank_hi = nullptr);

// f32 input -> per-field vmin/vmax/constant flag/first non-finite index and
// the float64 normalised field.  `mm` holds 2*nfields u32 + nfields u64.
void ingest_normalize(const float* x, int64_t n, int nfields, double* norm, FieldScal* fs,
                      unsigned int* mm, double eps_rel, cudaStream_t st);

// closed-form prefix decode into coefficient buffer `a`
void decode_coeffs(const Meta& m, const ProbeParam* prm, double* a, int64_t n, int nfields,
                   cudaStream_t st);

// base probe: decode (lower bound) -> IDWT -> count & max error
void probe_base(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                int nfields, const double* norm, const float* orig, const FieldScal* fs,
                ProbeResult* res, cudaStream_t st, const Inc* inc = nullptr, bool xe = true,
                bool early = false, int nphys = -1);

// residual probe: decode (midpoint) -> IDWT -> + base -> max error
void probe_trunc(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                 int nprobes, const double* base_dec, const float* orig, const FieldScal* fs,
                 ProbeResult* res, cudaStream_t st, const Inc* inc = nullptr, bool xe = true,
                 int nphys = -1);

// some exponent n_max - p (p < 64 planes) outside the normal float64 range:
// the level kernels' decode then keeps its scalbn path
inline bool exps_extreme(int n_max) { return n_max - 63 <= -1022 || n_max >= 1024; }

// tiling of the incremental probes (the level kernels' CTA grids); false if
// the persistent LL layout does not fit (the probes then run in full)
bool inc_geometry(const Geo& g, int nfields, Inc& inc);
void inc_capacity(const Geo& g, int64_t* tiles, int64_t* tiles0);

// decode the chosen base prefix; write base_dec and resid = norm - base_dec
void base_to_residue(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                     int nfields, const double* norm, double* base_dec, double* resid,
                     cudaStream_t st, bool xe = true);

// decompress: decode a stream to a float64 field (out), optionally midpoint
void decode_field(const Meta& m, const ProbeParam* prm, double* a, double* b, const Geo& g,
                  int nfields, double* out, cudaStream_t st, bool xe = true,
                  bool midpoint = false);
// decompress: residual decode fused with base add + denormalise to f32
void decode_field_add_denorm(const Meta& m, const ProbeParam* prm, double* a, double* b,
                             const Geo& g, int nfields, const double* base, const FieldScal* fs,
                             float* out32, cudaStream_t st, bool xe = true);
// decompress: f32(vmin + base*range) for fields without residual (gate: active)
void denorm_only(const double* base, const FieldScal* fs, const uint8_t* active, int64_t n,
                 int nfields, float* out32, cudaStream_t st);
// decompress: constant chunks (gate: active)
void fill_constant(const FieldScal* fs, const uint8_t* active, int64_t n, int nfields,
                   float* out32, cudaStream_t st);

// payload pack: for each part, copy header (12 B from hdr) + stream bytes
struct PackPart {
  uint64_t dst_off;      // byte offset in the packed output
  uint64_t nbytes;       // total bytes incl. 12-byte header
  uint64_t bit_limit;    // stream bits >= this are zeroed (padding of a shorter variant)
  const uint32_t* src;   // stream words
  uint8_t hdr[16];
};
void pack_parts(const PackPart* parts, int nparts, uint8_t* out, cudaStream_t st);

// payload unpack: scatter stream bytes (after the header) into word buffers
struct UnpackPart {
  uint64_t src_off;      // offset of the stream's first payload byte in `in`
  uint64_t nbytes;       // payload bytes (excluding header)
  uint32_t* dst;         // word buffer (zero-padded to a word)
};
void unpack_parts(const UnpackPart* parts, int nparts, const uint8_t* in, cudaStream_t st);

// container image (container.py:44-73): record i (25 B, records + 25 i) at
// dst_off, its payload (len bytes at payload + src_off) right after
struct ContainerPart {
  int64_t src_off;
  int64_t dst_off;
  int64_t len;
};
void assemble_container(const ContainerPart* parts, int nparts, const uint8_t* records,
                        const uint8_t* payload, uint8_t* out, cudaStream_t st);

}  // namespace ebcc
