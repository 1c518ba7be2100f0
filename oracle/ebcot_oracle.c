/* CPU oracle of the opt-in JPEG2000-style base layer ("ebcot" base codec).
 *
 * TEST INFRASTRUCTURE ONLY (see ebcc_oracle.h).  The reference has no
 * JPEG2000 base layer (the paper used OpenJPEG),
 * so PARITY IS UNPINNED: this file is an independent scalar restatement of
 * the published algorithms (ITU-T T.800 Annex C MQ coder, Annex D EBCOT
 * tier-1 coding) in the layout this repository defines, against which the
 * CUDA codec (paper_2510_22265_b200/csrc/ebcot.cu) is checked byte for byte.
 *
 * Stream ("J2") = 12-byte header like SPIHT's ('J','2', n_max i8, levels u8,
 * rows u32, cols u32), then - unless the stream is the bare header - one byte
 * per code-block (leading all-zero bit-planes, 24 = empty block), then the
 * coding-pass units in inclusion order.  Quantisation: deadzone, one step
 * 2^(n_max-23) for every subband (24 bit-planes, like the SPIHT base layer).
 * Code-blocks: 64x64 per subband (LL, then levels coarse to fine, HL/LH/HH),
 * row-major inside a subband.  Per code-block: cleanup pass on its top plane,
 * then significance-propagation / magnitude-refinement / cleanup per plane,
 * 19 contexts (T.800 Tables D.1-D.4), stripes of 4 rows, every pass its own
 * MQ codeword (termination on each pass).  Unit order: global pass index
 * G = 3*(23 - plane) + {SP 0, MR 1, CU 2}, then code-block index.  A unit is
 * a LEB128 value v (0: the pass codes no symbol; else a codeword of v-1
 * bytes) followed by the codeword.  A budget keeps the longest unit-aligned
 * prefix that fits (at least the bare header).  Reconstruction: midpoint of
 * the interval the decoded bits leave, sign * (2m+1) * 2^(p_low-1) * step.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ebcc_oracle.h"

#define J2_PLANES 24
#define CB 64
#define HDR 12
#define MAXLEV 5
#define ZERO_SENT (-128)

/* ---- MQ coder (T.800 Table C.2 and Annex C procedures) --------------- */
static const uint16_t QE[47] = {
    0x5601, 0x3401, 0x1801, 0x0AC1, 0x0521, 0x0221, 0x5601, 0x5401, 0x4801, 0x3801,
    0x3001, 0x2401, 0x1C01, 0x1601, 0x5601, 0x5401, 0x5101, 0x4801, 0x3801, 0x3401,
    0x3001, 0x2801, 0x2401, 0x2201, 0x1C01, 0x1801, 0x1601, 0x1401, 0x1201, 0x1101,
    0x0AC1, 0x09C1, 0x08A1, 0x0521, 0x0441, 0x02A1, 0x0221, 0x0141, 0x0111, 0x0085,
    0x0049, 0x0025, 0x0015, 0x0009, 0x0005, 0x0001, 0x5601};
static const uint8_t NMPS[47] = {1,  2,  3,  4,  5,  38, 7,  8,  9,  10, 11, 12, 13, 29, 15, 16,
                                 17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32,
                                 33, 34, 35, 36, 37, 38, 39, 40, 41, 42, 43, 44, 45, 45, 46};
static const uint8_t NLPS[47] = {1,  6,  9,  12, 29, 33, 6,  14, 14, 14, 17, 18, 20, 21, 14, 14,
                                 15, 16, 17, 18, 19, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29,
                                 30, 31, 32, 33, 34, 35, 36, 37, 38, 39, 40, 41, 42, 43, 46};
static const uint8_t SWITCHB[47] = {1, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 1, 0,
                                    0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                                    0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};

#define NCTX 19
#define CTX_RL 17
#define CTX_UNI 18

typedef struct { uint8_t I[NCTX], mps[NCTX]; } ctxs_t;

static void ctx_reset(ctxs_t *s) {
  memset(s, 0, sizeof(*s));
  s->I[0] = 4;
  s->I[CTX_RL] = 3;
  s->I[CTX_UNI] = 46;
}

typedef struct {
  uint32_t A, C;
  int CT;
  int B;          /* byte at position bp (bp == -1: the dummy byte) */
  int64_t bp;
  uint8_t *out;   /* the pass's codeword */
} mqe_t;

static void mqe_init(mqe_t *e, uint8_t *out) {
  e->A = 0x8000; e->C = 0; e->CT = 12; e->B = 0; e->bp = -1; e->out = out;
}

static void mqe_put(mqe_t *e, int nb) { /* commit B, move to the next byte */
  if (e->bp >= 0) e->out[e->bp] = (uint8_t)e->B;
  e->bp++;
  e->B = nb;
}

static void mqe_byteout(mqe_t *e) {
  if (e->B == 0xFF) {
    mqe_put(e, (int)(e->C >> 20));
    e->C &= 0xFFFFF;
    e->CT = 7;
  } else if (e->C < 0x8000000) {
    mqe_put(e, (int)(e->C >> 19));
    e->C &= 0x7FFFF;
    e->CT = 8;
  } else {
    e->B++;
    if (e->B == 0xFF) {
      e->C &= 0x7FFFFFF;
      mqe_put(e, (int)(e->C >> 20));
      e->C &= 0xFFFFF;
      e->CT = 7;
    } else {
      mqe_put(e, (int)(e->C >> 19));
      e->C &= 0x7FFFF;
      e->CT = 8;
    }
  }
}

static void mqe_renorm(mqe_t *e) {
  do {
    e->A <<= 1;
    e->C <<= 1;
    e->CT--;
    if (e->CT == 0) mqe_byteout(e);
  } while ((e->A & 0x8000) == 0);
}

static void mqe_code(mqe_t *e, ctxs_t *s, int cx, int d) {
  const uint32_t qe = QE[s->I[cx]];
  e->A -= qe;
  if (d == s->mps[cx]) { /* CODEMPS */
    if ((e->A & 0x8000) == 0) {
      if (e->A < qe) e->A = qe;
      else e->C += qe;
      s->I[cx] = NMPS[s->I[cx]];
      mqe_renorm(e);
    } else {
      e->C += qe;
    }
  } else { /* CODELPS */
    if (e->A < qe) e->C += qe;
    else e->A = qe;
    if (SWITCHB[s->I[cx]]) s->mps[cx] = (uint8_t)(1 - s->mps[cx]);
    s->I[cx] = NLPS[s->I[cx]];
    mqe_renorm(e);
  }
}

/* FLUSH (SETBITS + two byte-outs); returns the codeword length without a
 * trailing 0xFF */
static int64_t mqe_flush(mqe_t *e) {
  const uint32_t t = e->C + e->A;
  e->C |= 0xFFFF;
  if (e->C >= t) e->C -= 0x8000;
  e->C <<= e->CT;
  mqe_byteout(e);
  e->C <<= e->CT;
  mqe_byteout(e);
  if (e->bp >= 0) e->out[e->bp] = (uint8_t)e->B;
  int64_t len = e->bp + 1;
  if (len > 0 && e->out[len - 1] == 0xFF) len--;
  return len;
}

typedef struct {
  uint32_t A, C;
  int CT;
  const uint8_t *d;
  int64_t n, bp;
} mqd_t;

static int mqd_byte(const mqd_t *m, int64_t i) { return i < m->n ? m->d[i] : 0xFF; }

static void mqd_bytein(mqd_t *m) {
  if (mqd_byte(m, m->bp) == 0xFF) {
    const int b1 = mqd_byte(m, m->bp + 1);
    if (b1 > 0x8F) {
      m->C += 0xFF00;
      m->CT = 8;
    } else {
      m->bp++;
      m->C += (uint32_t)b1 << 9;
      m->CT = 7;
    }
  } else {
    m->bp++;
    m->C += (uint32_t)mqd_byte(m, m->bp) << 8;
    m->CT = 8;
  }
}

static void mqd_init(mqd_t *m, const uint8_t *d, int64_t n) {
  m->d = d; m->n = n; m->bp = 0;
  m->C = (uint32_t)mqd_byte(m, 0) << 16;
  mqd_bytein(m);
  m->C <<= 7;
  m->CT -= 7;
  m->A = 0x8000;
}

static void mqd_renorm(mqd_t *m) {
  do {
    if (m->CT == 0) mqd_bytein(m);
    m->A <<= 1;
    m->C <<= 1;
    m->CT--;
  } while ((m->A & 0x8000) == 0);
}

static int mqd_decode(mqd_t *m, ctxs_t *s, int cx) {
  const uint32_t qe = QE[s->I[cx]];
  int d;
  m->A -= qe;
  if ((m->C >> 16) < qe) { /* the LPS sub-interval (the bottom Qe): LPS exchange */
    if (m->A < qe) {
      m->A = qe;
      d = s->mps[cx];
      s->I[cx] = NMPS[s->I[cx]];
    } else {
      m->A = qe;
      d = 1 - s->mps[cx];
      if (SWITCHB[s->I[cx]]) s->mps[cx] = (uint8_t)(1 - s->mps[cx]);
      s->I[cx] = NLPS[s->I[cx]];
    }
    mqd_renorm(m);
  } else {
    m->C -= qe << 16;
    if ((m->A & 0x8000) == 0) { /* MPS exchange */
      if (m->A < qe) {
        d = 1 - s->mps[cx];
        if (SWITCHB[s->I[cx]]) s->mps[cx] = (uint8_t)(1 - s->mps[cx]);
        s->I[cx] = NLPS[s->I[cx]];
      } else {
        d = s->mps[cx];
        s->I[cx] = NMPS[s->I[cx]];
      }
      mqd_renorm(m);
    } else {
      d = s->mps[cx];
    }
  }
  return d;
}

/* exported for the MQ round-trip test: n symbols in n contexts (cx[i] < 19) */
int64_t eo_mq_encode(const uint8_t *bits, const uint8_t *cx, int64_t n, uint8_t *out) {
  ctxs_t s;
  ctx_reset(&s);
  mqe_t e;
  mqe_init(&e, out);
  for (int64_t i = 0; i < n; i++) mqe_code(&e, &s, cx[i], bits[i]);
  return mqe_flush(&e);
}

void eo_mq_decode(const uint8_t *data, int64_t len, const uint8_t *cx, int64_t n, uint8_t *bits) {
  ctxs_t s;
  ctx_reset(&s);
  mqd_t m;
  mqd_init(&m, data, len);
  for (int64_t i = 0; i < n; i++) bits[i] = (uint8_t)mqd_decode(&m, &s, cx[i]);
}

/* ---- geometry: subbands and code-blocks ----------------------------- */
typedef struct {
  int r0, c0, h, w;   /* code-block rectangle in the Mallat layout */
  int orient;         /* 0 LL/LH, 1 HL (H and V swapped), 2 HH */
} cblk_t;

static void shapes(int rows, int cols, int levels, int *lr, int *lc) {
  lr[0] = rows; lc[0] = cols;
  for (int k = 1; k <= levels; k++) { lr[k] = (lr[k - 1] + 1) / 2; lc[k] = (lc[k - 1] + 1) / 2; }
}

/* the code-blocks in stream order; returns their count */
int eo_ebcot_blocks(int rows, int cols, int levels, int *out5, int cap) {
  int lr[MAXLEV + 1], lc[MAXLEV + 1];
  shapes(rows, cols, levels, lr, lc);
  int n = 0;
  for (int band = 0; band <= 3 * levels; band++) {
    int r0, c0, h, w, orient;
    if (band == 0) { r0 = 0; c0 = 0; h = lr[levels]; w = lc[levels]; orient = 0; }
    else {
      const int k = levels - (band - 1) / 3, o = (band - 1) % 3;
      const int ri = lr[k - 1], ci = lc[k - 1], rl = lr[k], cl = lc[k];
      if (o == 0) { r0 = 0; c0 = cl; h = rl; w = ci - cl; orient = 1; }
      else if (o == 1) { r0 = rl; c0 = 0; h = ri - rl; w = cl; orient = 0; }
      else { r0 = rl; c0 = cl; h = ri - rl; w = ci - cl; orient = 2; }
    }
    if (h <= 0 || w <= 0) continue;
    for (int by = 0; by < h; by += CB)
      for (int bx = 0; bx < w; bx += CB) {
        if (out5 && n < cap) {
          int *b = out5 + 5 * n;
          b[0] = r0 + by; b[1] = c0 + bx;
          b[2] = h - by < CB ? h - by : CB;
          b[3] = w - bx < CB ? w - bx : CB;
          b[4] = orient;
        }
        n++;
      }
  }
  return n;
}

static cblk_t *blocks_of(int rows, int cols, int levels, int *nb) {
  int n = eo_ebcot_blocks(rows, cols, levels, NULL, 0);
  int *t = malloc(sizeof(int) * 5 * (n ? n : 1));
  eo_ebcot_blocks(rows, cols, levels, t, n);
  cblk_t *b = malloc(sizeof(cblk_t) * (n ? n : 1));
  for (int i = 0; i < n; i++) {
    b[i].r0 = t[5 * i]; b[i].c0 = t[5 * i + 1]; b[i].h = t[5 * i + 2]; b[i].w = t[5 * i + 3];
    b[i].orient = t[5 * i + 4];
  }
  free(t);
  *nb = n;
  return b;
}

/* ---- contexts (T.800 Tables D.1, D.3, D.4) --------------------------- */
static int sig_ctx(int orient, int h, int v, int d) {
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

/* code-block state: flags per sample */
#define F_SIG 1
#define F_VIS 2   /* coded in this plane's significance-propagation pass */
#define F_REF 4   /* refined at least once */
#define F_NEG 8   /* sign (valid once significant) */

typedef struct {
  int h, w, orient;
  uint8_t *f;      /* h * w flags */
} blk_t;

static inline int flg(const blk_t *b, int y, int x) {
  if (y < 0 || x < 0 || y >= b->h || x >= b->w) return 0;
  return b->f[y * b->w + x];
}

static void neigh(const blk_t *b, int y, int x, int *h, int *v, int *d) {
  *h = (flg(b, y, x - 1) & F_SIG) + (flg(b, y, x + 1) & F_SIG);
  *v = (flg(b, y - 1, x) & F_SIG) + (flg(b, y + 1, x) & F_SIG);
  *d = (flg(b, y - 1, x - 1) & F_SIG) + (flg(b, y - 1, x + 1) & F_SIG) +
       (flg(b, y + 1, x - 1) & F_SIG) + (flg(b, y + 1, x + 1) & F_SIG);
}

static int sgn_contrib(const blk_t *b, int y0, int x0, int y1, int x1) {
  int s = 0;
  const int a = flg(b, y0, x0), c = flg(b, y1, x1);
  if (a & F_SIG) s += (a & F_NEG) ? -1 : 1;
  if (c & F_SIG) s += (c & F_NEG) ? -1 : 1;
  return s > 0 ? 1 : (s < 0 ? -1 : 0);
}

/* sign context and xor bit */
static int sign_ctx(const blk_t *b, int y, int x, int *xr) {
  const int hc = sgn_contrib(b, y, x - 1, y, x + 1), vc = sgn_contrib(b, y - 1, x, y + 1, x);
  int cx, xo = 0;
  if (hc == 1) cx = vc == 1 ? 13 : (vc == 0 ? 12 : 11);
  else if (hc == 0) { cx = vc == 0 ? 9 : 10; xo = vc == -1; }
  else { cx = vc == 1 ? 11 : (vc == 0 ? 12 : 13); xo = 1; }
  if (hc == 1) xo = 0;
  *xr = xo;
  return cx;
}

static int mr_ctx(const blk_t *b, int y, int x) {
  if (flg(b, y, x) & F_REF) return 16;
  int h, v, d;
  neigh(b, y, x, &h, &v, &d);
  return (h + v + d) ? 15 : 14;
}

/* ---- tier-1: one code-block, encoder and decoder share the pass logic - */
/* coder callback: enc != NULL -> code symbol `bit`; else decode one */
typedef struct {
  mqe_t *e; mqd_t *d; ctxs_t *s; int64_t nsym;
  uint8_t *segbuf; int started; const uint8_t *seg; int64_t seglen;
} coder_t;

static int code_bit(coder_t *c, int cx, int bit) {
  c->nsym++;
  if (c->e) {
    if (!c->started) { mqe_init(c->e, c->segbuf); c->started = 1; }
    mqe_code(c->e, c->s, cx, bit);
    return bit;
  }
  if (!c->started) { mqd_init(c->d, c->seg, c->seglen); c->started = 1; }
  return mqd_decode(c->d, c->s, cx);
}

/* one pass over the block.  ptype 0 SP, 1 MR, 2 CU.  Encoder: q holds the
 * magnitudes; decoder: q is built up (bits OR'ed in), plow[] tracks the
 * lowest decoded plane of each significant sample. */
static void run_pass(blk_t *b, uint32_t *q, int8_t *plow, int p, int ptype, coder_t *c) {
  const int enc = c->e != NULL;
  for (int y0 = 0; y0 < b->h; y0 += 4) {
    const int sh = b->h - y0 < 4 ? b->h - y0 : 4;
    for (int x = 0; x < b->w; x++) {
      int y = y0;
      if (ptype == 2 && sh == 4) { /* cleanup run mode */
        int run_ok = 1;
        for (int k = 0; k < 4 && run_ok; k++) {
          const int fl = b->f[(y0 + k) * b->w + x];
          int h, v, d;
          neigh(b, y0 + k, x, &h, &v, &d);
          if ((fl & (F_SIG | F_VIS)) || h + v + d) run_ok = 0;
        }
        if (run_ok) {
          int first = 4;
          if (enc)
            for (int k = 0; k < 4; k++)
              if ((q[(y0 + k) * b->w + x] >> p) & 1) { first = k; break; }
          const int any = code_bit(c, CTX_RL, first < 4);
          if (!any) continue;
          if (enc) {
            code_bit(c, CTX_UNI, (first >> 1) & 1);
            code_bit(c, CTX_UNI, first & 1);
          } else {
            first = code_bit(c, CTX_UNI, 0) << 1;
            first |= code_bit(c, CTX_UNI, 0);
          }
          const int yy = y0 + first, i = yy * b->w + x;
          int xr;
          const int scx = sign_ctx(b, yy, x, &xr);
          const int neg = enc ? ((b->f[i] & F_NEG) != 0) : 0;
          const int sb = code_bit(c, scx, neg ^ xr) ^ xr;
          if (!enc) { q[i] |= 1u << p; plow[i] = (int8_t)p; if (sb) b->f[i] |= F_NEG; }
          b->f[i] |= F_SIG;
          y = yy + 1;
        }
      }
      for (; y < y0 + sh; y++) {
        const int i = y * b->w + x;
        const int fl = b->f[i];
        if (ptype == 1) { /* MR: significant before this plane */
          if (!(fl & F_SIG) || (fl & F_VIS)) continue;
          const int cx = mr_ctx(b, y, x);
          const int bit = code_bit(c, cx, enc ? (int)((q[i] >> p) & 1) : 0);
          if (!enc) { q[i] |= (uint32_t)bit << p; plow[i] = (int8_t)p; }
          b->f[i] |= F_REF;
          continue;
        }
        if (fl & F_SIG) continue;
        int h, v, d;
        neigh(b, y, x, &h, &v, &d);
        if (ptype == 0) {
          if (h + v + d == 0) continue;
          b->f[i] |= F_VIS;
        } else if (fl & F_VIS) {
          continue;
        }
        const int cx = sig_ctx(b->orient, h, v, d);
        const int bit = code_bit(c, cx, enc ? (int)((q[i] >> p) & 1) : 0);
        if (bit) {
          int xr;
          const int scx = sign_ctx(b, y, x, &xr);
          const int neg = enc ? ((fl & F_NEG) != 0) : 0;
          const int sb = code_bit(c, scx, neg ^ xr) ^ xr;
          if (!enc) { q[i] |= 1u << p; plow[i] = (int8_t)p; if (sb) b->f[i] |= F_NEG; }
          b->f[i] |= F_SIG;
        }
      }
    }
  }
}

/* pass sequence of a block with top plane pt: CU(pt), then SP/MR/CU below */
static int block_passes(int pt) { return pt < 0 ? 0 : 1 + 3 * pt; }
static void pass_of(int pt, int j, int *p, int *ptype) {
  if (j == 0) { *p = pt; *ptype = 2; return; }
  *p = pt - 1 - (j - 1) / 3;
  *ptype = (j - 1) % 3;
}
static int gidx(int p, int ptype) { return 3 * (J2_PLANES - 1 - p) + ptype; }

static int floor_log2_dbl(double x) { int e; frexp(x, &e); return e - 1; }

static void put_hdr(uint8_t *o, int nmax, int levels, int rows, int cols) {
  o[0] = 'J'; o[1] = '2'; o[2] = (uint8_t)(int8_t)nmax; o[3] = (uint8_t)levels;
  uint32_t r = (uint32_t)rows, c = (uint32_t)cols;
  memcpy(o + 4, &r, 4);
  memcpy(o + 8, &c, 4);
}

static int leb_put(uint8_t *o, uint64_t v) {
  int n = 0;
  do {
    uint8_t b = v & 0x7F;
    v >>= 7;
    if (v) b |= 0x80;
    o[n++] = b;
  } while (v);
  return n;
}

static int leb_get(const uint8_t *d, int64_t len, int64_t *pos, uint64_t *v) {
  uint64_t x = 0;
  int sh = 0;
  for (;;) {
    if (*pos >= len || sh > 56) return -1;
    const uint8_t b = d[(*pos)++];
    x |= (uint64_t)(b & 0x7F) << sh;
    sh += 7;
    if (!(b & 0x80)) break;
  }
  *v = x;
  return 0;
}

/* Encode a pyramid (Mallat layout, rows x cols) to the J2 stream truncated to
 * max_bytes (< 0: the whole stream).  Returns the length or -EO_E_*. */
int64_t eo_ebcot_encode(const double *coeffs, int rows, int cols, int levels, int64_t max_bytes,
                        uint8_t *out, int64_t cap) {
  const int64_t n = (int64_t)rows * cols;
  if (cap < HDR) return -EO_E_CAPACITY;
  double mx = 0.0;
  for (int64_t i = 0; i < n; i++) {
    const double a = fabs(coeffs[i]);
    if (a > mx) mx = a;
  }
  if (mx == 0.0) {
    put_hdr(out, ZERO_SENT, levels, rows, cols);
    return HDR;
  }
  const int nmax = floor_log2_dbl(mx);
  const int e0 = nmax - (J2_PLANES - 1);
  put_hdr(out, nmax, levels, rows, cols);
  int nb;
  cblk_t *bl = blocks_of(rows, cols, levels, &nb);
  /* per block: passes as (length field, codeword) */
  typedef struct { int pt, np; uint32_t *v; uint8_t **cw; } benc_t;
  benc_t *be = calloc(nb, sizeof(benc_t));
  for (int k = 0; k < nb; k++) {
    const cblk_t *cb = &bl[k];
    const int m = cb->h * cb->w;
    uint32_t *q = malloc(sizeof(uint32_t) * m);
    blk_t b = {cb->h, cb->w, cb->orient, calloc(m, 1)};
    uint32_t orq = 0;
    for (int y = 0; y < cb->h; y++)
      for (int x = 0; x < cb->w; x++) {
        const double c = coeffs[(int64_t)(cb->r0 + y) * cols + cb->c0 + x];
        const uint32_t qq = (uint32_t)floor(ldexp(fabs(c), -e0));
        q[y * cb->w + x] = qq;
        if (c < 0) b.f[y * cb->w + x] |= F_NEG;
        orq |= qq;
      }
    const int pt = orq ? floor_log2_dbl((double)orq) : -1;
    be[k].pt = pt;
    be[k].np = block_passes(pt);
    be[k].v = calloc(be[k].np ? be[k].np : 1, sizeof(uint32_t));
    be[k].cw = calloc(be[k].np ? be[k].np : 1, sizeof(uint8_t *));
    ctxs_t s;
    ctx_reset(&s);
    mqe_t e;
    uint8_t *seg = malloc((size_t)m * 4 + 64);
    for (int j = 0; j < be[k].np; j++) {
      int p, ptype;
      pass_of(pt, j, &p, &ptype);
      coder_t c = {&e, NULL, &s, 0, seg, 0, NULL, 0};
      if (ptype == 0)
        for (int i = 0; i < m; i++) b.f[i] &= ~F_VIS;
      run_pass(&b, q, NULL, p, ptype, &c);
      if (c.started) {
        const int64_t len = mqe_flush(&e);
        be[k].v[j] = (uint32_t)len + 1;
        be[k].cw[j] = malloc(len ? len : 1);
        memcpy(be[k].cw[j], seg, len);
      }
    }
    free(seg);
    free(q);
    free(b.f);
  }
  /* bare header if the block table does not fit */
  int64_t pos = HDR;
  if (max_bytes >= 0 && max_bytes < HDR + nb) goto done;
  if (cap < HDR + nb) { pos = -EO_E_CAPACITY; goto done; }
  for (int k = 0; k < nb; k++) out[HDR + k] = (uint8_t)(be[k].pt < 0 ? J2_PLANES : J2_PLANES - 1 - be[k].pt);
  pos = HDR + nb;
  /* units by (global pass index, block) */
  for (int g = 0; g < 3 * J2_PLANES; g++) {
    for (int k = 0; k < nb; k++) {
      const int pt = be[k].pt;
      if (pt < 0) continue;
      const int gtop = gidx(pt, 2);
      int j;
      if (g == gtop) j = 0;
      else if (g > gtop + 0 && g >= gidx(pt - 1, 0) && pt >= 1) j = 1 + (g - gidx(pt - 1, 0));
      else continue;
      if (j >= be[k].np) continue;
      uint8_t lb[10];
      const int ln = leb_put(lb, be[k].v[j]);
      const int64_t ulen = ln + (be[k].v[j] ? be[k].v[j] - 1 : 0);
      if (max_bytes >= 0 && pos + ulen > max_bytes) goto done;
      if (pos + ulen > cap) { pos = -EO_E_CAPACITY; goto done; }
      memcpy(out + pos, lb, ln);
      if (be[k].v[j] > 1) memcpy(out + pos + ln, be[k].cw[j], be[k].v[j] - 1);
      pos += ulen;
    }
  }
done:
  for (int k = 0; k < nb; k++) {
    for (int j = 0; j < be[k].np; j++) free(be[k].cw[j]);
    free(be[k].cw);
    free(be[k].v);
  }
  free(be);
  free(bl);
  return pos;
}

/* Decode a J2 stream (or prefix) to coefficients (midpoint reconstruction). */
int eo_ebcot_decode(const uint8_t *data, int64_t len, int rows, int cols, double *out) {
  if (len < HDR || data[0] != 'J' || data[1] != '2') return EO_E_FORMAT;
  const int nmax = (int8_t)data[2], levels = data[3];
  uint32_t hr, hc;
  memcpy(&hr, data + 4, 4);
  memcpy(&hc, data + 8, 4);
  if ((int)hr != rows || (int)hc != cols || levels < 1 || levels > MAXLEV) return EO_E_FORMAT;
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = 0; i < n; i++) out[i] = 0.0;
  if (nmax == ZERO_SENT || len == HDR) return EO_OK;
  const int e0 = nmax - (J2_PLANES - 1);
  int nb;
  cblk_t *bl = blocks_of(rows, cols, levels, &nb);
  if (len < HDR + nb) { free(bl); return EO_E_FORMAT; }
  /* pass segments of every block */
  int *pt = malloc(sizeof(int) * nb);
  int64_t *soff = malloc(sizeof(int64_t) * nb * (1 + 3 * J2_PLANES));
  int64_t *slen = malloc(sizeof(int64_t) * nb * (1 + 3 * J2_PLANES));
  int *nin = calloc(nb, sizeof(int));  /* passes present in the prefix */
  for (int k = 0; k < nb; k++) {
    const int z = data[HDR + k];
    if (z > J2_PLANES) { free(bl); free(pt); free(soff); free(slen); free(nin); return EO_E_FORMAT; }
    pt[k] = z == J2_PLANES ? -1 : J2_PLANES - 1 - z;
  }
  int64_t pos = HDR + nb;
  int st = EO_OK;
  for (int g = 0; g < 3 * J2_PLANES && pos < len; g++)
    for (int k = 0; k < nb && pos < len; k++) {
      if (pt[k] < 0) continue;
      const int gtop = gidx(pt[k], 2);
      int j;
      if (g == gtop) j = 0;
      else if (pt[k] >= 1 && g >= gidx(pt[k] - 1, 0)) j = 1 + (g - gidx(pt[k] - 1, 0));
      else continue;
      if (j >= block_passes(pt[k])) continue;
      uint64_t v;
      if (leb_get(data, len, &pos, &v)) { st = EO_E_FORMAT; goto out; }
      const int64_t cl = v ? (int64_t)v - 1 : -1;
      if (cl > len - pos) { st = EO_E_FORMAT; goto out; }
      soff[(int64_t)k * (1 + 3 * J2_PLANES) + j] = pos;
      slen[(int64_t)k * (1 + 3 * J2_PLANES) + j] = cl;
      nin[k] = j + 1;
      pos += cl > 0 ? cl : 0;
    }
  if (pos != len) st = EO_E_FORMAT;  /* a prefix ends on a unit boundary */
  for (int k = 0; k < nb && st == EO_OK; k++) {
    const cblk_t *cb = &bl[k];
    const int m = cb->h * cb->w;
    uint32_t *q = calloc(m, sizeof(uint32_t));
    int8_t *plow = malloc(m);
    memset(plow, -1, m);
    blk_t b = {cb->h, cb->w, cb->orient, calloc(m, 1)};
    ctxs_t s;
    ctx_reset(&s);
    mqd_t d;
    for (int j = 0; j < nin[k]; j++) {
      int p, ptype;
      pass_of(pt[k], j, &p, &ptype);
      const int64_t sl = slen[(int64_t)k * (1 + 3 * J2_PLANES) + j];
      coder_t c = {NULL, &d, &s, 0, NULL, 0, data + soff[(int64_t)k * (1 + 3 * J2_PLANES) + j],
                   sl > 0 ? sl : 0};
      if (ptype == 0)
        for (int i = 0; i < m; i++) b.f[i] &= ~F_VIS;
      run_pass(&b, q, plow, p, ptype, &c);
      if ((c.nsym > 0) != (sl >= 0)) { st = EO_E_FORMAT; break; }
    }
    for (int y = 0; y < cb->h; y++)
      for (int x = 0; x < cb->w; x++) {
        const int i = y * cb->w + x;
        if (!(b.f[i] & F_SIG)) continue;
        const int pl = plow[i];
        const uint32_t mm = q[i] >> pl;
        double v = ldexp((double)(2 * mm + 1), pl - 1 + e0);
        out[(int64_t)(cb->r0 + y) * cols + cb->c0 + x] = (b.f[i] & F_NEG) ? -v : v;
      }
    free(q);
    free(plow);
    free(b.f);
  }
out:
  free(bl); free(pt); free(soff); free(slen); free(nin);
  return st;
}
