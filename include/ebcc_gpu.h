/* ebcc_gpu.h — C ABI of the B200-native EBCC chunk path (libebcc_gpu.so).
 *
 * The library replaces the reference's per-chunk pipeline behind its own
 * Python API: everything above the two batch calls (ebcc.api.compress /
 * decompress, the container writer/reader, tiling and ingest validation)
 * stays host Python, byte-identical to the reference.
 *
 *   ebcc_compress    replaces pipeline.compress_grid's per-chunk loop
 *                    (pkg/src/ebcc/pipeline.py:358-367) over a batch of
 *                    same-shape chunks: compress_chunk (pipeline.py:277-329)
 *                    with its base-quantile search (142-199), pure-base search
 *                    (215-236), residual encode + truncation search (243-254,
 *                    303-309) and candidate choice (315-329), all on device.
 *   ebcc_decompress  replaces pipeline.decompress_grid's per-chunk loop
 *                    (pipeline.py:370-379) -> decompress_chunk (332-355).
 *
 * Plain pointers and sizes only; no exceptions cross the boundary.  Every
 * call returns an EBCC_* status; ebcc_last_error() has the message.
 */
#ifndef EBCC_GPU_H
#define EBCC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EBCC_ABI_VERSION 1

/* status codes (mirroring pkg/src/ebcc/errors.py) */
#define EBCC_OK 0
#define EBCC_E_ARGUMENT 1      /* ArgumentError  (pipeline.py:54-62)            */
#define EBCC_E_FORMAT 2        /* FormatError    (pipeline.py:336-353)          */
#define EBCC_E_RESIDUAL 3      /* ResidualInsufficient (pipeline.py:322-325)    */
#define EBCC_E_CAPACITY 4      /* payload buffer too small; see payload_total  */
#define EBCC_E_CUDA 5          /* CUDA runtime failure -> EbccError              */
#define EBCC_E_NOMEM 6         /* device allocation failed                     */
#define EBCC_E_INGEST 7        /* IngestError: non-finite input (core.py:74-79) */

/* flags */
#define EBCC_INPUT_ON_DEVICE 1   /* `fields` / `payload` are device pointers  */
#define EBCC_OUTPUT_ON_DEVICE 2  /* `payload` / `out` are device pointers     */
#define EBCC_FULL_SEARCH 4       /* compress: run every probe of the reference's
                                    searches (no candidate pruning; same bytes,
                                    n_base_probes / n_trunc_probes equal the
                                    reference's probe counts)                 */
#define EBCC_CONTAINER_BODY 8    /* ebcc_fetch_container: records + payloads
                                    only (no 42-byte file header; header42 may
                                    be NULL) - one rank's span of a container
                                    assembled by several processes           */
#define EBCC_BASE_EBCOT 16       /* compress: the opt-in JPEG2000-style base
                                    layer ('J2' streams: deadzone quantisation,
                                    EBCOT tier-1 + MQ coder; container
                                    version 2).  The reference has no such
                                    layer: parity unpinned.
                                    decompress recognises 'J2' streams by
                                    their magic.                              */

/* Chunk modes (pipeline.py:38-41). */
#define EBCC_MODE_CONSTANT 0
#define EBCC_MODE_PURE_BASE 1
#define EBCC_MODE_TWO_LAYER 2

/* One chunk's record: the container record fields (container.py:26-27)
 * plus search statistics. */
typedef struct {
  int32_t mode;
  int32_t status;          /* per-chunk status (EBCC_OK / EBCC_E_RESIDUAL)   */
  double vmin, vmax;       /* chunk extrema (float32 values held as double)  */
  int64_t base_len;        /* bytes of base stream in the payload            */
  int64_t resid_len;       /* bytes of residual stream in the payload        */
  int32_t n_base_probes;   /* distinct base budgets evaluated (P_base)       */
  int32_t n_trunc_probes;  /* residual truncation evaluations (P_trunc)      */
  int32_t resid_planes;    /* 24 or 32 when TWO_LAYER                        */
  int32_t reserved;
} ebcc_chunk_rec;

typedef struct ebcc_ctx ebcc_ctx;

int ebcc_abi_version(void);

/* One context per device (and per host thread using it). */
int ebcc_create(int32_t device, ebcc_ctx **out);
void ebcc_destroy(ebcc_ctx *ctx);
/* Run on this cudaStream_t (default: the context's own stream). */
int ebcc_set_stream(ebcc_ctx *ctx, void *cuda_stream);
const char *ebcc_last_error(const ebcc_ctx *ctx);
/* After EBCC_E_INGEST: flat index (into the `fields` array of the call) of the
 * first non-finite value, in C order; -1 otherwise. */
int64_t ebcc_last_error_index(const ebcc_ctx *ctx);

/* Compress `nfields` row-major float32 chunks of rows x cols each, laid out
 * back to back (chunk i at fields + i*rows*cols).  Parameters are the
 * reference's EbccParams as Python doubles (pipeline.py:44-62).
 * Payload of chunk i is written at payload + payload_offsets[i]
 * (base_len + resid_len bytes); payload_total receives the sum.  When
 * payload_cap is too small the call returns EBCC_E_CAPACITY with records and
 * payload_total filled; call ebcc_fetch_payload with a larger buffer.
 * A chunk for which no candidate reaches the bound has status
 * EBCC_E_RESIDUAL and the call returns EBCC_E_RESIDUAL. */
int ebcc_compress(ebcc_ctx *ctx, const float *fields, int64_t nfields, int32_t rows,
                  int32_t cols, double eps_rel, double q, double r0, double search_tol,
                  int32_t flags, ebcc_chunk_rec *recs, uint8_t *payload, int64_t payload_cap,
                  int64_t *payload_offsets, int64_t *payload_total);

/* Copy the payload of the last ebcc_compress call. */
int ebcc_fetch_payload(ebcc_ctx *ctx, uint8_t *payload, int64_t payload_cap, int32_t flags);

/* Write the reference container image of the last ebcc_compress call
 * (container.py:44-73 write_file): the caller's 42-byte file header, then per
 * chunk its caller-built 25-byte record followed by its payload.  Assembled
 * on the device, then one device->host (or device->device) copy into `out`.
 * out_len receives 42 + 25 * nchunks + payload_total. */
int ebcc_fetch_container(ebcc_ctx *ctx, const uint8_t *header42, const uint8_t *records25,
                         int64_t nchunks, uint8_t *out, int64_t cap, int32_t flags,
                         int64_t *out_len);

/* Host-side container indexing (container.py:82-145, pipeline.py:336-353),
 * native so a 2,368-chunk container is indexed in microseconds:
 *   ebcc_parse_records  walks the `count` records after the 42-byte header:
 *                       copies each 25-byte record to records25 and the
 *                       absolute payload offset to offsets.  EBCC_E_FORMAT
 *                       with *err_offset and *err_aux = 1 truncated record,
 *                       2 unknown mode, 3 truncated payload, 4 trailing bytes
 *                       (the reference's FormatError offsets).
 *   ebcc_check_streams  the stream-header checks of decompress_chunk for
 *                       same-shape chunks; *levels = common level count;
 *                       EBCC_E_FORMAT names the first bad chunk in *bad,
 *                       EBCC_E_ARGUMENT a chunk of a different depth. */
int ebcc_parse_records(const uint8_t *data, int64_t len, int64_t count, uint8_t *records25,
                       int64_t *offsets, int64_t *err_offset, int32_t *err_aux);
int ebcc_check_streams(const uint8_t *data, int64_t len, const uint8_t *records25,
                       const int64_t *offsets, int64_t n, int32_t rows, int32_t cols,
                       int32_t *levels, int64_t *bad);

/* Page-locked host blocks for result arrays, from a per-process cache so that
 * repeated calls do not pay cudaHostAlloc.  Device->host copies into them run
 * at full PCIe/C2C speed without a staging hop. */
int ebcc_host_alloc(int64_t bytes, void **out);
int ebcc_host_free(void *ptr);
/* Release every freed block the cache holds. */
void ebcc_host_cache_trim(void);

/* Decompress `nfields` same-shape chunks.  recs[i].mode/vmin/vmax/base_len/
 * resid_len come from the container; chunk i's payload starts at
 * payload + payload_offsets[i].  `levels` is the level count stored in the
 * streams' headers.  Writes nfields*rows*cols float32 to `out`. */
int ebcc_decompress(ebcc_ctx *ctx, const uint8_t *payload, const int64_t *payload_offsets,
                    const ebcc_chunk_rec *recs, int64_t nfields, int32_t rows, int32_t cols,
                    int32_t levels, int32_t flags, float *out);

/* Unit-level entry points (host pointers), each the device counterpart of a
 * reference function, used by the parity tests:
 *   ebcc_dwt          dwt.forward_dwt / dwt.inverse_dwt (dwt.py:178-216) on
 *                     nfields rows x cols float64 arrays; `levels` as given
 *                     (forward clamps like clamp_levels).
 *   ebcc_spiht_encode spiht.spiht_encode(pyramid, planes=planes) unbudgeted
 *                     (spiht.py:271-358); budgeted streams are byte prefixes.
 *   ebcc_spiht_decode spiht.decode_with_plane(data, prefix_len)
 *                     (spiht.py:403-482): coefficients + n_last (-999: None).
 *   ebcc_decode_field base_codec.dequantized_field(data, prefix_len, midpoint)
 *                     (base_codec.py:70-84): the decoded prefix through the
 *                     PRODUCTION inverse transform (the fused level kernels
 *                     of decompress and the probes, closed-form decode on
 *                     load) into a float64 field. */
int ebcc_dwt(ebcc_ctx *ctx, const double *in, double *out, int64_t nfields, int32_t rows,
             int32_t cols, int32_t levels, int32_t inverse);
int ebcc_spiht_encode(ebcc_ctx *ctx, const double *coeffs, int32_t rows, int32_t cols,
                      int32_t levels, int32_t planes, uint8_t *out, int64_t cap, int64_t *len);
int ebcc_spiht_decode(ebcc_ctx *ctx, const uint8_t *data, int64_t len, int64_t prefix_len,
                      int32_t rows, int32_t cols, double *coeffs_out, int32_t *n_last);
int ebcc_decode_field(ebcc_ctx *ctx, const uint8_t *data, int64_t len, int64_t prefix_len,
                      int32_t rows, int32_t cols, int32_t midpoint, double *field_out);

/* Quality metrics of the reference's benchmark harness (pkg/src/ebcc/bench/
 * metrics.py), float64 on the device, for nfields fields of n (= rows*cols)
 * float32 values each; `orig`/`rec` are host pointers unless flags has
 * EBCC_INPUT_ON_DEVICE.  Statistics and SSIM reduce in a fixed order.
 *   ebcc_error_stats      core.error_stats (core.py:189-207) ingredients, per
 *                         field 5 doubles: max|rec-orig|, min(orig),
 *                         max(orig), sum (rec-orig)^2, count(orig != rec).
 *   ebcc_error_histogram  metrics.error_histogram (metrics.py:78-99) counts for
 *                         caller-given edges (nfields x (bins+1), np.linspace);
 *                         bins [e_k, e_k+1), the last closed; exact counts.
 *   ebcc_ssim             metrics.ssim (metrics.py:47-75): mean SSIM, 11x11
 *                         Gaussian (sigma 1.5), range from `orig`, 1 for
 *                         identical fields; rows, cols >= 11.
 *   ebcc_radial_spectrum  metrics.radial_power_spectrum (metrics.py:102-125):
 *                         |fft2(a)/(rows*cols)|^2 summed per wavenumber annulus;
 *                         bin_idx (rows*cols, host) is the rounded isotropic
 *                         wavenumber of each mode (bins 1..kmax kept). */
int ebcc_error_stats(ebcc_ctx *ctx, const float *orig, const float *rec, int64_t nfields,
                     int64_t n, int32_t flags, double *out);
int ebcc_error_histogram(ebcc_ctx *ctx, const float *orig, const float *rec, int64_t nfields,
                         int64_t n, int32_t bins, const double *edges, int32_t flags,
                         int64_t *counts);
int ebcc_ssim(ebcc_ctx *ctx, const float *orig, const float *rec, int64_t nfields, int32_t rows,
              int32_t cols, int32_t flags, double *out);
int ebcc_radial_spectrum(ebcc_ctx *ctx, const float *data, int64_t nfields, int32_t rows,
                         int32_t cols, const int32_t *bin_idx, int32_t kmax, int32_t flags,
                         double *out);

/* Self-test of the FMA-corrected exact divisions used by the kernels
 * (x / SCALE_LOW, x / SCALE_HIGH, x / range) against IEEE __ddiv_rn on n
 * random operands; *mismatches must be 0. */
int ebcc_selftest_div(ebcc_ctx *ctx, int64_t n, uint64_t seed, int64_t *mismatches);

/* Developer instrumentation: time full base probes (decode + inverse DWT +
 * count / max-error reduction) of the last single-lane compress batch on
 * this context at B = frac * (full base stream bits); averages over iters. */
int ebcc_dev_probe_bench(ebcc_ctx *ctx, double frac, int32_t iters, int32_t early,
                         double *us_level0, double *us_probe);

/* Instrumentation for bench.py: kernels launched and device milliseconds
 * (CUDA events on the library stream) of the last call, split by stage. */
typedef struct {
  int64_t kernel_launches;
  double ms_total;
  double ms_encode;     /* DWT + SPIHT encodes                       */
  double ms_probe;      /* feedback probes (decode + IDWT + reduce)  */
  double ms_other;
  int64_t probe_launches;     /* probe steps (batched over fields)   */
  double ms_probe_kernel;     /* summed duration of the dominant probe kernels */
  int64_t probe_kernel_count;
  int64_t probe_kernel_fields; /* chunks covered by those launches, summed */
  int64_t lanes;               /* concurrent sub-batches the call used */
  int64_t tiles_computed;      /* level-0 probe tiles recomputed (incremental probes) */
  int64_t tiles_probed;        /* level-0 probe tiles the probes covered */
} ebcc_stats;

int ebcc_get_stats(const ebcc_ctx *ctx, ebcc_stats *out);

#ifdef __cplusplus
}
#endif
#endif
