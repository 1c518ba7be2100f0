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
};

constexpr int kMaxPlaneRecs = 64;

// Per-field machine state summary (device resident).
struct MachineOut {
  int32_t n_max;          // input (encode: computed by coef_prepare)
  int32_t planes_run;     // planes entered
  uint32_t total_bits;    // bit position after the last plane
  int32_t overflow;       // list or bit-buffer capacity exceeded
  uint32_t lsp_count;     // |LSP| at the end
  uint32_t pad[3];
};

// Batched buffers, all fields `stride` elements apart (bits: bit_stride words).
struct MachineBufs {
  int nfields;
  int64_t stride;            // elements per field for per-coefficient arrays
  int64_t bit_stride;        // words per field in the bit buffer
  // per coefficient
  int16_t* ec; int16_t* ed; int16_t* el;
  uint32_t* mant; uint32_t* sign_pos; uint32_t* lsp_rank; uint8_t* pinfo;
  // lists (capacity `stride` each)
  uint32_t* lip; uint32_t* lis0; uint32_t* lis1; uint32_t* w0; uint32_t* w1; uint32_t* lsp;
  // stream bits
  uint32_t* bits;
  PlaneRec* planes;          // [nfields][kMaxPlaneRecs]
  MachineOut* out;           // [nfields]
  const uint64_t* limit;     // decode: per-field bit limit (8 * payload bytes)
  const uint8_t* active;     // optional per-field gate (nullptr = all)
};

// geometry-wide tables (shared by every field of a batch)
struct TreeTables {
  uint8_t* flags;        // nchild | has_grandchild << 3
  uint32_t* roots;       // LIP initial order
  uint32_t* lis_roots;   // roots with children (initial LIS, type A)
  int64_t nroots, nlis_roots;
};

void build_tree_tables(const Geo& g, TreeTables& t, cudaStream_t st);  // allocates device memory
void free_tree_tables(TreeTables& t);

// coefficient exponents / mantissas / signs + per-field n_max
void coef_prepare(const double* coef, int64_t field_stride, MachineBufs& mb, const Geo& g,
                  cudaStream_t st);
// e_d / e_l bottom-up
void subtree_exponents(MachineBufs& mb, const Geo& g, const TreeTables& tt, cudaStream_t st);
// the list machine (one CTA per field)
void run_machine(bool decode, MachineBufs& mb, const Geo& g, const TreeTables& tt, int planes,
                 cudaStream_t st);
// encoder refinement bits (fully parallel over LSP)
void write_refinement(MachineBufs& mb, int planes, cudaStream_t st);
// decoder: reset per-coefficient metadata before run_machine(decode=true)
void decode_init(MachineBufs& mb, cudaStream_t st);
// decoder: gather refinement bits into mant[] (in LSP order)
void gather_refinement(MachineBufs& mb, cudaStream_t st);

}  // namespace ebcc
