// Opt-in JPEG2000-style base layer ("ebcot" base codec, ebcot.cu).
//
// The reference's base layer is DWT + SPIHT; the paper's was JPEG2000
// through OpenJPEG, which the reference leaves out
// (SPEC.md:261).  This codec restores a JPEG2000-style base layer as an
// opt-in (container version 2): the same CDF 9/7 pyramid, deadzone
// quantisation with one step 2^(n_max-23), EBCOT tier-1 coding of 64x64
// code-blocks with the T.800 MQ coder (one coding pass per MQ codeword), and
// a stream of coding-pass units in (global pass, code-block) order, so that
// every budget is served by a unit-aligned byte prefix.  PARITY IS UNPINNED
// (no reference implementation exists); the CPU oracle oracle/ebcot_oracle.c
// restates the same algorithm and the GPU streams must equal its bytes.
//
// GPU mapping: quantisation and the closed-form probe decode are one thread
// per coefficient; tier-1 coding (inherently sequential inside a code-block)
// is one thread per code-block, thousands of code-blocks per batch; stream
// assembly is one CTA per chunk (a block scan over the unit sizes).
#pragma once
#include "common.cuh"
#include "probe.cuh"
#include "spiht.cuh"

namespace ebcc {

constexpr int kJ2Planes = 24;
constexpr int kJ2Block = 64;
constexpr int kJ2Passes = 1 + 3 * (kJ2Planes - 1);   // passes of a block with 24 planes
constexpr int kJ2Slots = 3 * kJ2Planes;              // global pass indices

struct EbBlock {
  int r0, c0, h, w;
  int orient;  // 0 LL / LH, 1 HL (H and V swapped), 2 HH
  int pad;
  int64_t off;   // samples of the blocks before it (its codeword scratch offset)
  int64_t soff;  // its tier-1 state words: stripe-major, ceil(h/4) * 4 * w
};

// geometry tables (one set per chunk shape)
struct EbGeo {
  int nb;                   // code-blocks
  const EbBlock* blocks;    // [nb]
  const int32_t* blk_of;    // [n] code-block of each pyramid position
  int64_t state_stride;     // tier-1 state words per field (sum of the blocks' soff spans)
};

// per-batch buffers (all fields `n` coefficients apart)
struct EbBufs {
  int nfields;
  int64_t n;
  uint32_t* qs;        // [f][n] magnitude | significance-in-SP << 30 | negative << 31
  uint16_t* flags;     // [f][state_stride] tier-1 state words (own flags, neighbours'
                       // significance / signs), stripe-major per code-block
  int8_t* plow;        // [f][n] decoder: lowest decoded plane
  uint8_t* cw;         // [f][cw_stride] per-block codeword scratch
  int64_t cw_stride;   // n * kCwPerPoint + nb * kCwPerBlock bytes per field
  uint32_t* uval;      // [f][nb][kJ2Passes] unit values (0: no symbol, else len + 1)
  int64_t* uoff;       // [f][nb][kJ2Passes] decoder: codeword offsets in the body
  uint8_t* ztab;       // [f][nb] leading zero planes (24: empty block)
  uint32_t* cum;       // [f][kJ2Slots * nb + 1] body bytes after the block table, by slot
  int32_t* nmax;       // [f] n_max (kExpNone: all zero)
  int32_t* status;     // [f] capacity overflow (encoder) / format error (decoder)
  uint8_t* body;       // [f][body_stride] stream body = block table + units (after the header)
  int64_t body_stride; // bytes per field
  const uint64_t* body_len;  // decoder: body bytes present per field
};
constexpr int kCwPerPoint = 8;    // codeword scratch bytes per coefficient (MQ output <= ~3 bits/pt)
constexpr int kCwPerBlock = 512;  // plus per block (pass terminations of tiny blocks)

// host-built geometry tables (device memory; free with ebcot_free_geo)
EbGeo ebcot_build_geo(const Geo& g, int32_t** blk_of_out, EbBlock** blocks_out, cudaStream_t st);

// encode the pyramids in `coef` (f64, field stride n): n_max, quantisation,
// tier-1 coding and stream assembly; `active` gates fields (null = all)
void ebcot_encode(const double* coef, const EbGeo& eg, const Geo& g, EbBufs& b,
                  const uint8_t* active, cudaStream_t st);

// closed-form decode of probe v's prefix (ProbeParam::B = slots included)
// into the f64 pyramid `out` (stride n); chunk v % nphys
void ebcot_probe_decode(const EbGeo& eg, const EbBufs& b, const ProbeParam* prm, int nprobes,
                        int nphys, double* out, cudaStream_t st);

// decompress: parse the stream bodies and MQ-decode every code-block into
// the f64 pyramid `out`; nmax[] holds each field's header n_max
void ebcot_stream_decode(const EbGeo& eg, const Geo& g, EbBufs& b, const uint8_t* active,
                         double* out, cudaStream_t st);
// copy the fields' n_max into MachineOut::n_max (the packer's stream headers)
void ebcot_nmax_to(const EbBufs& b, MachineOut* mo, cudaStream_t st);

// probe epilogue on a decoded normalised field: count = #points with
// !(|dec - norm| <= eps_rel) (count probes), maxerr of the f32 denormalised
// reconstruction (ProbeResult, like the SPIHT probes')
void ebcot_probe_reduce(const double* dec, const float* orig, const FieldScal* fs,
                        const ProbeParam* prm, int64_t n, int nfields, bool count,
                        ProbeResult* res, cudaStream_t st);

// base_dec = dec; resid = norm - dec (pipeline.py:300)
void ebcot_residue(const double* dec, const ProbeParam* prm, int64_t n, int nfields,
                   double* base_dec, double* resid, cudaStream_t st);

}  // namespace ebcc
