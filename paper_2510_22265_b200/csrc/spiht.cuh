// SPIHT list machine and its helpers (spiht.cu).
#pragma once
#include "common.cuh"

namespace ebcc {

// Per-plane record written by the machine, index p = n_max - n.
struct PlaneRec {
  uint32_t start;         // bit offset where plane p begins
  uint32_t refine_start;  // bit offset of plane p's refinement segment
  uint32_t refine_len;    // |LSP| at the start of plane p
  uint32_t lists_end;     // |LIP| + |LIS| + |LSP| after plane p
  uint32_t lip_len;       // |LIP| at the start of plane p (encoder)
  uint32_t lis_start;     // bit offset of plane p's first LIS wave (encoder)
  uint32_t pad[2];
};

constexpr int kMaxPlaneRecs = 64;

// Per-field machine state summary (device resident).
struct MachineOut {
  int32_t n_max;          // input (encode: computed by coef_prepare)
  int32_t planes_run;     // planes entered
  uint32_t total_bits;    // bit position after the last plane
  int32_t overflow;       // list or bit-buffer capacity exceeded
  uint32_t lsp_count;     // |LSP| at the end
  uint32_t hist_len;      // encoder: entries ever appended to the LIP
  uint32_t lis_hist_len;  // encoder: entries ever kept in the LIS
  uint32_t pad;
};

// List entries are 64-bit "node info" words carrying everything the machine
// needs about a node, so list passes stream instead of gathering:
//   bits  0..31 node (flat index)
//   bits 32..37 relc = clamp(n_max - floor(log2|c|), 0, 63)   (63: never)
//   bits 38..43 reld  (same, for the max over all descendants)
//   bits 44..49 rell  (same, for the max over grandchildren and below)
//   bit  50     coefficient is negative
//   bits 51..53 number of children; bit 54 has grandchildren
//   bit  55     LIS entry of type B
//   bits 56..58 band level (0 = LL, 1..5 detail); bits 59..60 orientation
//   bits 61, 62 a detail node's 2x2 child block has its right column / bottom row
// "significant at plane index p" is simply rel <= p.
namespace ninfo {
constexpr int RELC = 32, RELD = 38, RELL = 44, NEG = 50, NCH = 51, HASGC = 54, TYPEB = 55,
              LEVEL = 56, ORIENT = 59, RIGHT = 61, BOTTOM = 62;
}

// Batched buffers, all fields `stride` elements apart (bits: bit_stride words).
struct MachineBufs {
  int nfields;
  int64_t stride;            // elements per field for per-coefficient arrays
  int64_t bit_stride;        // words per field in the bit buffer
  // per coefficient
  int16_t* ec; int16_t* ed; int16_t* el;
  uint32_t* mant; uint32_t* sign_pos; uint32_t* lsp_rank; uint8_t* pinfo;
  uint64_t* ninfo;           // per-field node info (encode)
  const uint64_t* ginfo;     // geometry-only node info (decode; shared by all fields)
  // lists (capacity `stride` each)
  uint64_t* lip; uint64_t* lis0; uint64_t* lis1; uint64_t* w0; uint64_t* w1; uint32_t* lsp;
  // encoder, optional: sign bit offset by LSP rank, written with the LSP
  // entry (Meta::sprank; pack_meta then has nothing to scatter)
  uint32_t* sprank;
  uint8_t* hrel;             // encoder: significance plane of each LIS history entry
  // stream bits
  uint32_t* bits;
  PlaneRec* planes;          // [nfields][kMaxPlaneRecs]
  MachineOut* out;           // [nfields]
  const uint64_t* limit;     // decode: per-field bit limit (8 * payload bytes)
  const uint8_t* active;     // optional per-field gate (nullptr = all)
};

// geometry-wide tables (shared by every field of a batch)
struct TreeTables {
  uint64_t* ginfo;       // geometry node info (nchild, has_gc, level, orientation)
  uint32_t* roots;       // LIP initial order
  uint32_t* lis_roots;   // roots with children (initial LIS, type A)
  int64_t nroots, nlis_roots;
};

void build_tree_tables(const Geo& g, TreeTables& t, cudaStream_t st);  // allocates device memory
void free_tree_tables(TreeTables& t);

// coefficient exponents / mantissas / signs + per-field n_max
void coef_prepare(const double* coef, int64_t field_stride, MachineBufs& mb, const Geo& g,
                  cudaStream_t st);
// e_d / e_l bottom-up, then the per-field node info words
void subtree_exponents(MachineBufs& mb, const Geo& g, const TreeTables& tt, cudaStream_t st);
// the list machine (one CTA per field)
// cluster > 0 forces the CTAs per field (1..4); 0 picks by batch size
void run_machine(bool decode, MachineBufs& mb, const Geo& g, const TreeTables& tt, int planes,
                 cudaStream_t st, int cluster = 0);
// CTAs per chunk the machine uses when `concurrent_fields` chunks' clusters
// must be resident at once (cudaOccupancyMaxActiveClusters; EBCC_MACHINE_CLUSTER)
int machine_cluster_size(bool decode, int concurrent_fields);
// encoder: the deferred LIP passes and old-LIS significance bits (fully
// parallel over the LIP / LIS histories);
// must run after run_machine(decode=false) and before write_refinement
void emit_lip(MachineBufs& mb, int planes, cudaStream_t st);
// encoder refinement bits (fully parallel over LSP)
void write_refinement(MachineBufs& mb, int planes, cudaStream_t st);
// decoder: reset per-coefficient metadata before run_machine(decode=true)
// packed != null: records preset to "never placed" for gather_pack
void decode_init(MachineBufs& mb, cudaStream_t st, uint2* packed = nullptr);
// decompress (narrow records): refinement gather straight into the probe
// records + sign offsets by rank (replaces gather_refinement + pack_meta)
void gather_pack(MachineBufs& mb, uint2* packed, uint32_t* sprank, cudaStream_t st);
// decoder: gather refinement bits into mant[] (in LSP order)
void gather_refinement(MachineBufs& mb, cudaStream_t st);

}  // namespace ebcc
