/* CPU oracle for the EBCC chunk path — TEST INFRASTRUCTURE ONLY.
 *
 * A scalar C restatement of the reference Python/numpy algorithm, written
 * from its behaviour and cited function by function.
 * It is deliberately naive where the reference is naive (every base-budget
 * probe re-runs the forward DWT and the budgeted SPIHT encode, exactly like
 * base_codec.base_encode_budget does), so that timing it is timing the
 * reference's algorithm on host cores.
 *
 * Compile with -ffp-contract=off: every float64 expression below must round
 * once per operation in the reference's (numpy's) evaluation order.
 */
#include "ebcc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* dwt.py:23-30 — identical double literals */
static const double ALPHA = -1.586134342059924;
static const double BETA = -0.052980118572961;
static const double GAMMA = 0.882911075530934;
static const double DELTA = 0.443506852043971;
static const double SCALE_LOW = 1.1270436568907234;
static const double SCALE_HIGH = 0.8773746085014191;

#define MAX_LEVELS 5
#define HEADER_SIZE 12
#define ZERO_SENTINEL (-128)
#define MAX_DECODE_PLANES 64
#define NLAST_NONE (-999)

static int floor_log2_int(int m) { /* floor(log2(m)) for m >= 1 */
  int k = -1;
  while (m) { m >>= 1; k++; }
  return k;
}

/* dwt.py:35-41 */
int eo_default_levels(int rows, int cols) {
  int m = rows < cols ? rows : cols;
  if (m < 2) return 1;
  int depth = floor_log2_int(m) - 2;
  if (depth > MAX_LEVELS) depth = MAX_LEVELS;
  return depth < 1 ? 1 : depth;
}

/* dwt.py:44-48 */
int eo_clamp_levels(int rows, int cols, int levels) {
  int m = rows < cols ? rows : cols;
  if (m < 2) m = 2;
  int cap = floor_log2_int(m);
  if (cap < 1) cap = 1;
  return levels < cap ? levels : cap;
}

/* dwt.py:82-92: ll[k] = ceil(ll[k-1]/2) */
static void ll_shapes(int rows, int cols, int levels, int *lr, int *lc) {
  lr[0] = rows; lc[0] = cols;
  for (int k = 1; k <= levels; k++) {
    lr[k] = (lr[k - 1] + 1) / 2;
    lc[k] = (lc[k - 1] + 1) / 2;
  }
}

/* dwt.py:68-79: rects (r0, c0, h, w) of HL/LH/HH created at `level` */
static void detail_rect(const int *lr, const int *lc, int level, int o, int *r0, int *c0,
                        int *h, int *w) {
  int ri = lr[level - 1], ci = lc[level - 1], rl = lr[level], cl = lc[level];
  if (o == 0) { *r0 = 0; *c0 = cl; *h = rl; *w = ci - cl; }
  else if (o == 1) { *r0 = rl; *c0 = 0; *h = ri - rl; *w = cl; }
  else { *r0 = rl; *c0 = cl; *h = ri - rl; *w = ci - cl; }
}

/* ---- 1D lifting on a contiguous line (dwt.py:112-175) ---------------- */

static void analyze_line(double *x, int n, double *s, double *d) {
  if (n == 1) return; /* length-1 passthrough, no scaling (dwt.py:140-141) */
  int ns = (n + 1) / 2, nd = n / 2;
  for (int i = 0; i < ns; i++) s[i] = x[2 * i];
  for (int i = 0; i < nd; i++) d[i] = x[2 * i + 1];
  /* d += ALPHA*(s + s_right) ; s_right[i] = s[min(i+1, ns-1)] */
  for (int i = 0; i < nd; i++) {
    double sr = s[i + 1 < ns ? i + 1 : ns - 1];
    d[i] = d[i] + ALPHA * (s[i] + sr);
  }
  /* s += BETA*(left + right); left[i]=d[max(i-1,0)], right[i]=d[min(i,nd-1)] */
  for (int i = 0; i < ns; i++) {
    double l = d[i > 0 ? i - 1 : 0], r = d[i < nd ? i : nd - 1];
    s[i] = s[i] + BETA * (l + r);
  }
  for (int i = 0; i < nd; i++) {
    double sr = s[i + 1 < ns ? i + 1 : ns - 1];
    d[i] = d[i] + GAMMA * (s[i] + sr);
  }
  for (int i = 0; i < ns; i++) {
    double l = d[i > 0 ? i - 1 : 0], r = d[i < nd ? i : nd - 1];
    s[i] = s[i] + DELTA * (l + r);
  }
  for (int i = 0; i < ns; i++) x[i] = s[i] * SCALE_LOW;
  for (int i = 0; i < nd; i++) x[ns + i] = d[i] * SCALE_HIGH;
}

static void synthesize_line(double *y, int n, double *s, double *d) {
  if (n == 1) return;
  int ns = (n + 1) / 2, nd = n - ns;
  for (int i = 0; i < ns; i++) s[i] = y[i] / SCALE_LOW;
  for (int i = 0; i < nd; i++) d[i] = y[ns + i] / SCALE_HIGH;
  for (int i = 0; i < ns; i++) {
    double l = d[i > 0 ? i - 1 : 0], r = d[i < nd ? i : nd - 1];
    s[i] = s[i] - DELTA * (l + r);
  }
  for (int i = 0; i < nd; i++) {
    double sr = s[i + 1 < ns ? i + 1 : ns - 1];
    d[i] = d[i] - GAMMA * (s[i] + sr);
  }
  for (int i = 0; i < ns; i++) {
    double l = d[i > 0 ? i - 1 : 0], r = d[i < nd ? i : nd - 1];
    s[i] = s[i] - BETA * (l + r);
  }
  for (int i = 0; i < nd; i++) {
    double sr = s[i + 1 < ns ? i + 1 : ns - 1];
    d[i] = d[i] - ALPHA * (s[i] + sr);
  }
  for (int i = 0; i < ns; i++) y[2 * i] = s[i];
  for (int i = 0; i < nd; i++) y[2 * i + 1] = d[i];
}

/* dwt.py:178-199: per level, all rows then all columns */
void eo_forward_dwt(double *a, int rows, int cols, int levels) {
  int lr[72], lc[72];
  levels = eo_clamp_levels(rows, cols, levels);
  ll_shapes(rows, cols, levels, lr, lc);
  int mx = rows > cols ? rows : cols;
  double *line = malloc(sizeof(double) * mx), *s = malloc(sizeof(double) * mx),
         *d = malloc(sizeof(double) * mx);
  for (int k = 0; k < levels; k++) {
    int r = lr[k], c = lc[k];
    for (int i = 0; i < r; i++) analyze_line(a + (int64_t)i * cols, c, s, d);
    for (int j = 0; j < c; j++) {
      for (int i = 0; i < r; i++) line[i] = a[(int64_t)i * cols + j];
      analyze_line(line, r, s, d);
      for (int i = 0; i < r; i++) a[(int64_t)i * cols + j] = line[i];
    }
  }
  free(line); free(s); free(d);
}

/* dwt.py:202-216: coarse to fine, columns then rows */
void eo_inverse_dwt(double *a, int rows, int cols, int levels) {
  int lr[72], lc[72];
  ll_shapes(rows, cols, levels, lr, lc);
  int mx = rows > cols ? rows : cols;
  double *line = malloc(sizeof(double) * mx), *s = malloc(sizeof(double) * mx),
         *d = malloc(sizeof(double) * mx);
  for (int k = levels - 1; k >= 0; k--) {
    int r = lr[k], c = lc[k];
    for (int j = 0; j < c; j++) {
      for (int i = 0; i < r; i++) line[i] = a[(int64_t)i * cols + j];
      synthesize_line(line, r, s, d);
      for (int i = 0; i < r; i++) a[(int64_t)i * cols + j] = line[i];
    }
    for (int i = 0; i < r; i++) synthesize_line(a + (int64_t)i * cols, c, s, d);
  }
  free(line); free(s); free(d);
}

/* ---- spatial-orientation forest (spiht.py:81-179) -------------------- */

typedef struct {
  int rows, cols, levels;
  int32_t *children; /* [n][4], left-compacted, -1 = none */
  uint8_t *nchild, *has_grandchild;
  int32_t *roots;
  int64_t nroots;
  /* bottom-up evaluation order for subtree maxima (parent_groups) */
  int32_t *group_nodes;
  int64_t ngroup_nodes;
} tree_t;

static void tree_free(tree_t *t) {
  free(t->children); free(t->nchild); free(t->has_grandchild); free(t->roots);
  free(t->group_nodes);
}

static int tree_build(tree_t *t, int rows, int cols, int levels) {
  int lr[72], lc[72];
  int64_t n = (int64_t)rows * cols;
  ll_shapes(rows, cols, levels, lr, lc);
  t->rows = rows; t->cols = cols; t->levels = levels;
  t->children = malloc(sizeof(int32_t) * 4 * n);
  t->nchild = calloc(n, 1);
  t->has_grandchild = calloc(n, 1);
  t->roots = malloc(sizeof(int32_t) * n);
  t->group_nodes = malloc(sizeof(int32_t) * n);
  if (!t->children || !t->nchild || !t->has_grandchild || !t->roots || !t->group_nodes)
    return EO_E_NOMEM;
  for (int64_t i = 0; i < 4 * n; i++) t->children[i] = -1;
  t->ngroup_nodes = 0;
  /* same-orientation links: parent band at level k feeds level k-1 */
  for (int k = 2; k <= levels; k++) {
    for (int o = 0; o < 3; o++) {
      int pr0, pc0, ph, pw, cr0, cc0, ch, cw;
      detail_rect(lr, lc, k, o, &pr0, &pc0, &ph, &pw);
      detail_rect(lr, lc, k - 1, o, &cr0, &cc0, &ch, &cw);
      if (ph <= 0 || pw <= 0) continue;
      for (int i = 0; i < ph; i++)
        for (int j = 0; j < pw; j++) t->group_nodes[t->ngroup_nodes++] = (pr0 + i) * cols + pc0 + j;
      if (ch <= 0 || cw <= 0) continue;
      for (int i = 0; i < ph; i++)
        for (int j = 0; j < pw; j++) {
          int32_t pid = (pr0 + i) * cols + pc0 + j;
          int slot = 0;
          for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++, slot++) {
              int ci = 2 * i + a, cj = 2 * j + b;
              if (ci < ch && cj < cw) t->children[4 * (int64_t)pid + slot] = (cr0 + ci) * cols + cc0 + cj;
            }
        }
    }
  }
  /* low-low roots parent the same position of each coarsest detail band */
  int llr = lr[levels], llc = lc[levels];
  for (int o = 0; o < 3; o++) {
    int r0, c0, h, w;
    detail_rect(lr, lc, levels, o, &r0, &c0, &h, &w);
    if (h <= 0 || w <= 0) continue;
    int hh = llr < h ? llr : h, ww = llc < w ? llc : w;
    for (int i = 0; i < hh; i++)
      for (int j = 0; j < ww; j++) t->children[4 * (int64_t)(i * cols + j) + o] = (r0 + i) * cols + c0 + j;
  }
  for (int i = 0; i < llr; i++)
    for (int j = 0; j < llc; j++) t->group_nodes[t->ngroup_nodes++] = i * cols + j;
  /* left-compact the child slots (stable) and count them */
  for (int64_t p = 0; p < n; p++) {
    int32_t tmp[4];
    int m = 0;
    for (int s = 0; s < 4; s++)
      if (t->children[4 * p + s] >= 0) tmp[m++] = t->children[4 * p + s];
    for (int s = 0; s < 4; s++) t->children[4 * p + s] = s < m ? tmp[s] : -1;
    t->nchild[p] = (uint8_t)m;
  }
  for (int64_t p = 0; p < n; p++) {
    int g = 0;
    for (int s = 0; s < t->nchild[p]; s++) g |= t->nchild[t->children[4 * p + s]] > 0;
    t->has_grandchild[p] = (uint8_t)g;
  }
  /* roots: LL row-major, then orphans per level k = L-1..1 and orientation */
  t->nroots = 0;
  for (int i = 0; i < llr; i++)
    for (int j = 0; j < llc; j++) t->roots[t->nroots++] = i * cols + j;
  for (int k = levels - 1; k >= 1; k--) {
    for (int o = 0; o < 3; o++) {
      int r0, c0, h, w, pr0, pc0, ph, pw;
      detail_rect(lr, lc, k, o, &r0, &c0, &h, &w);
      detail_rect(lr, lc, k + 1, o, &pr0, &pc0, &ph, &pw);
      if (h <= 0 || w <= 0) continue;
      for (int i = 0; i < h; i++)
        for (int j = 0; j < w; j++)
          if (i / 2 >= ph || j / 2 >= pw) t->roots[t->nroots++] = (r0 + i) * cols + c0 + j;
    }
  }
  return EO_OK;
}

/* spiht.py:182-195 */
static void subtree_maxima(const double *val, const tree_t *t, double *dmax, double *lmax) {
  int64_t n = (int64_t)t->rows * t->cols;
  memset(dmax, 0, sizeof(double) * n);
  memset(lmax, 0, sizeof(double) * n);
  for (int64_t g = 0; g < t->ngroup_nodes; g++) {
    int32_t p = t->group_nodes[g];
    double dm = 0.0, lm = 0.0;
    for (int s = 0; s < t->nchild[p]; s++) {
      int32_t c = t->children[4 * (int64_t)p + s];
      double v = val[c] > dmax[c] ? val[c] : dmax[c];
      if (v > dm) dm = v;
      if (dmax[c] > lm) lm = dmax[c];
    }
    dmax[p] = dm;
    lmax[p] = lm;
  }
}

/* ---- growable lists -------------------------------------------------- */

typedef struct { int32_t *v; int64_t n, cap; } ilist;
typedef struct { int32_t *node; uint8_t *isb; int64_t n, cap; } slist;

static void il_push(ilist *l, int32_t x) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 1024;
    l->v = realloc(l->v, sizeof(int32_t) * l->cap);
  }
  l->v[l->n++] = x;
}
static void sl_push(slist *l, int32_t x, uint8_t b) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 1024;
    l->node = realloc(l->node, sizeof(int32_t) * l->cap);
    l->isb = realloc(l->isb, l->cap);
  }
  l->node[l->n] = x;
  l->isb[l->n++] = b;
}
static void sl_free(slist *l) { free(l->node); free(l->isb); memset(l, 0, sizeof(*l)); }

/* ---- bit sink (spiht.py:202-222) ------------------------------------- */

typedef struct {
  uint8_t *buf;
  int64_t cap_bytes, total, budget; /* budget < 0: unbudgeted */
  int overflow;
} sink_t;

/* returns 1 when the budget is reached (encoding stops exactly there) */
static int sink_put(sink_t *s, int bit) {
  if (s->budget >= 0 && s->total >= s->budget) return 1;
  int64_t byte = s->total >> 3;
  if (byte >= s->cap_bytes) { s->overflow = 1; return 1; }
  if (bit) s->buf[byte] |= (uint8_t)(0x80u >> (s->total & 7));
  s->total++;
  return s->budget >= 0 && s->total >= s->budget;
}

static int floor_log2_d(double x) { int e; frexp(x, &e); return e - 1; }

static void put_header(uint8_t *out, int n_max, int levels, int rows, int cols) {
  out[0] = 'S'; out[1] = 'P';
  out[2] = (uint8_t)(int8_t)n_max;
  out[3] = (uint8_t)levels;
  uint32_t r = (uint32_t)rows, c = (uint32_t)cols;
  memcpy(out + 4, &r, 4);
  memcpy(out + 8, &c, 4);
}

/* spiht.py:271-358 */
int64_t eo_spiht_encode(const double *coeffs, int rows, int cols, int levels,
                        int64_t max_bytes, int planes, uint8_t *out, int64_t cap) {
  if (max_bytes >= 0 && max_bytes < HEADER_SIZE) return -EO_E_ARGUMENT;
  if (cap < HEADER_SIZE) return -EO_E_CAPACITY;
  int64_t n = (int64_t)rows * cols;
  double *val = malloc(sizeof(double) * n);
  double top = 0.0;
  for (int64_t i = 0; i < n; i++) {
    val[i] = fabs(coeffs[i]);
    if (val[i] > top) top = val[i];
  }
  if (top == 0.0) {
    put_header(out, ZERO_SENTINEL, levels, rows, cols);
    free(val);
    return HEADER_SIZE;
  }
  int n_max = floor_log2_d(top);
  put_header(out, n_max, levels, rows, cols);
  tree_t tr;
  memset(&tr, 0, sizeof(tr));
  if (tree_build(&tr, rows, cols, levels)) { free(val); tree_free(&tr); return -EO_E_NOMEM; }
  double *dmax = malloc(sizeof(double) * n), *lmax = malloc(sizeof(double) * n);
  subtree_maxima(val, &tr, dmax, lmax);

  sink_t sk = {out + HEADER_SIZE, cap - HEADER_SIZE, 0,
               max_bytes < 0 ? -1 : (max_bytes - HEADER_SIZE) * 8, 0};
  memset(out + HEADER_SIZE, 0, (size_t)(cap - HEADER_SIZE));

  ilist lip = {0}, lsp = {0}, newly = {0}, achild = {0};
  slist lis = {0}, wave = {0}, next = {0}, keep = {0};
  for (int64_t i = 0; i < tr.nroots; i++) {
    il_push(&lip, tr.roots[i]);
    if (tr.nchild[tr.roots[i]]) sl_push(&lis, tr.roots[i], 0);
  }
  uint8_t *sigbuf = malloc(n + 1);

  for (int pl = 0; pl < planes; pl++) {
    int nn = n_max - pl;
    double t = ldexp(1.0, nn);
    int64_t refine_end = lsp.n;
    /* insignificant pixels: all significance bits, then signs */
    if (lip.n) {
      newly.n = 0;
      for (int64_t i = 0; i < lip.n; i++) {
        int sg = val[lip.v[i]] >= t;
        if (sink_put(&sk, sg)) goto done;
        if (sg) il_push(&newly, lip.v[i]);
      }
      for (int64_t i = 0; i < newly.n; i++)
        if (sink_put(&sk, coeffs[newly.v[i]] < 0)) goto done;
      int64_t w = 0;
      for (int64_t i = 0; i < lip.n; i++)
        if (!(val[lip.v[i]] >= t)) lip.v[w++] = lip.v[i];
      lip.n = w;
      for (int64_t i = 0; i < newly.n; i++) il_push(&lsp, newly.v[i]);
    }
    /* insignificant sets, in waves */
    keep.n = 0;
    wave.n = 0;
    for (int64_t i = 0; i < lis.n; i++) sl_push(&wave, lis.node[i], lis.isb[i]);
    while (wave.n) {
      for (int64_t j = 0; j < wave.n; j++) {
        int32_t p = wave.node[j];
        int sg = wave.isb[j] ? lmax[p] >= t : dmax[p] >= t;
        sigbuf[j] = (uint8_t)sg;
        if (sink_put(&sk, sg)) goto done;
        if (!sg) sl_push(&keep, p, wave.isb[j]);
      }
      /* children of significant type-A sets: significance bits, then signs */
      achild.n = 0;
      for (int64_t j = 0; j < wave.n; j++) {
        if (!sigbuf[j] || wave.isb[j]) continue;
        int32_t p = wave.node[j];
        for (int s = 0; s < tr.nchild[p]; s++) {
          int32_t c = tr.children[4 * (int64_t)p + s];
          il_push(&achild, c);
          if (sink_put(&sk, val[c] >= t)) goto done;
        }
      }
      newly.n = 0;
      for (int64_t i = 0; i < achild.n; i++)
        if (val[achild.v[i]] >= t) il_push(&newly, achild.v[i]);
      for (int64_t i = 0; i < newly.n; i++)
        if (sink_put(&sk, coeffs[newly.v[i]] < 0)) goto done;
      for (int64_t i = 0; i < newly.n; i++) il_push(&lsp, newly.v[i]);
      for (int64_t i = 0; i < achild.n; i++)
        if (!(val[achild.v[i]] >= t)) il_push(&lip, achild.v[i]);
      /* next wave, in entry order (spiht.py:361-388) */
      next.n = 0;
      for (int64_t j = 0; j < wave.n; j++) {
        if (!sigbuf[j]) continue;
        int32_t p = wave.node[j];
        if (!wave.isb[j]) {
          if (tr.has_grandchild[p]) sl_push(&next, p, 1);
        } else {
          for (int s = 0; s < tr.nchild[p]; s++) {
            int32_t c = tr.children[4 * (int64_t)p + s];
            if (tr.nchild[c]) sl_push(&next, c, 0);
          }
        }
      }
      slist tmp = wave; wave = next; next = tmp;
    }
    { slist tmp = lis; lis = keep; keep = tmp; }
    /* refinement of previously significant coefficients */
    for (int64_t i = 0; i < refine_end; i++) {
      int64_t qv = (int64_t)floor(val[lsp.v[i]] / t);
      if (sink_put(&sk, (int)(qv & 1))) goto done;
    }
  }
done:;
  int overflow = sk.overflow;
  int64_t total = sk.total;
  free(val); free(dmax); free(lmax); free(sigbuf);
  free(lip.v); free(lsp.v); free(newly.v); free(achild.v);
  sl_free(&lis); sl_free(&wave); sl_free(&next); sl_free(&keep);
  tree_free(&tr);
  if (overflow) return -EO_E_CAPACITY;
  return HEADER_SIZE + (total + 7) / 8;
}

/* ---- decoder (spiht.py:225-254, 403-482) ----------------------------- */

typedef struct { const uint8_t *p; int64_t nbits, pos; } src_t;

/* take one bit; past the end returns 0 and does not advance */
static inline int src_bit(src_t *s) {
  if (s->pos >= s->nbits) return 0;
  int b = (s->p[s->pos >> 3] >> (7 - (s->pos & 7))) & 1;
  s->pos++;
  return b;
}

int eo_spiht_decode(const uint8_t *data, int64_t len, int64_t prefix_len, int rows,
                    int cols, double *coeffs_out, int *n_last_out) {
  if (len < HEADER_SIZE) return EO_E_FORMAT;
  if (data[0] != 'S' || data[1] != 'P') return EO_E_FORMAT;
  int n_max = (int8_t)data[2];
  int levels = data[3];
  uint32_t hr, hc;
  memcpy(&hr, data + 4, 4);
  memcpy(&hc, data + 8, 4);
  if (hr < 1 || hc < 1 || levels < 1) return EO_E_FORMAT;
  if (levels > 64) return EO_E_FORMAT; /* far beyond any encoder output */
  if ((int)hr != rows || (int)hc != cols) return EO_E_FORMAT;
  if (prefix_len < 0 || prefix_len > len) prefix_len = len;
  int64_t n = (int64_t)rows * cols;
  for (int64_t i = 0; i < n; i++) coeffs_out[i] = 0.0;
  if (n_max == ZERO_SENTINEL) { *n_last_out = NLAST_NONE; return EO_OK; }
  src_t src = {data + HEADER_SIZE, prefix_len > HEADER_SIZE ? (prefix_len - HEADER_SIZE) * 8 : 0, 0};
  tree_t tr;
  memset(&tr, 0, sizeof(tr));
  if (tree_build(&tr, rows, cols, levels)) { tree_free(&tr); return EO_E_NOMEM; }
  double *mag = calloc(n, sizeof(double)), *sgn = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; i++) sgn[i] = 1.0;
  ilist lip = {0}, lsp = {0}, newly = {0}, achild = {0};
  slist lis = {0}, wave = {0}, next = {0}, keep = {0};
  uint8_t *sig = malloc(n + 1), *csig = malloc(4 * n + 1);
  for (int64_t i = 0; i < tr.nroots; i++) {
    il_push(&lip, tr.roots[i]);
    if (tr.nchild[tr.roots[i]]) sl_push(&lis, tr.roots[i], 0);
  }
  int n_floor = n_max - MAX_DECODE_PLANES, nn = n_max, n_last = n_max;
  while (!(src.pos >= src.nbits) && nn > n_floor) {
    n_last = nn;
    double t = ldexp(1.0, nn);
    int64_t refine_end = lsp.n;
    if (lip.n) {
      newly.n = 0;
      for (int64_t i = 0; i < lip.n; i++) {
        sig[i] = (uint8_t)src_bit(&src);
        if (sig[i]) il_push(&newly, lip.v[i]);
      }
      for (int64_t i = 0; i < newly.n; i++) {
        if (src.pos < src.nbits) {
          int b = src_bit(&src);
          mag[newly.v[i]] = t;
          sgn[newly.v[i]] = 1.0 - 2.0 * b;
        }
        il_push(&lsp, newly.v[i]);
      }
      int64_t w = 0;
      for (int64_t i = 0; i < lip.n; i++)
        if (!sig[i]) lip.v[w++] = lip.v[i];
      lip.n = w;
    }
    keep.n = 0;
    wave.n = 0;
    for (int64_t i = 0; i < lis.n; i++) sl_push(&wave, lis.node[i], lis.isb[i]);
    while (wave.n) {
      for (int64_t j = 0; j < wave.n; j++) {
        sig[j] = (uint8_t)src_bit(&src);
        if (!sig[j]) sl_push(&keep, wave.node[j], wave.isb[j]);
      }
      achild.n = 0;
      for (int64_t j = 0; j < wave.n; j++) {
        if (!sig[j] || wave.isb[j]) continue;
        int32_t p = wave.node[j];
        for (int s = 0; s < tr.nchild[p]; s++) {
          csig[achild.n] = (uint8_t)src_bit(&src);
          il_push(&achild, tr.children[4 * (int64_t)p + s]);
        }
      }
      newly.n = 0;
      for (int64_t i = 0; i < achild.n; i++)
        if (csig[i]) il_push(&newly, achild.v[i]);
      for (int64_t i = 0; i < newly.n; i++) {
        if (src.pos < src.nbits) {
          int b = src_bit(&src);
          mag[newly.v[i]] = t;
          sgn[newly.v[i]] = 1.0 - 2.0 * b;
        }
        il_push(&lsp, newly.v[i]);
      }
      for (int64_t i = 0; i < achild.n; i++)
        if (!csig[i]) il_push(&lip, achild.v[i]);
      next.n = 0;
      for (int64_t j = 0; j < wave.n; j++) {
        if (!sig[j]) continue;
        int32_t p = wave.node[j];
        if (!wave.isb[j]) {
          if (tr.has_grandchild[p]) sl_push(&next, p, 1);
        } else {
          for (int s = 0; s < tr.nchild[p]; s++) {
            int32_t c = tr.children[4 * (int64_t)p + s];
            if (tr.nchild[c]) sl_push(&next, c, 0);
          }
        }
      }
      slist tmp = wave; wave = next; next = tmp;
    }
    { slist tmp = lis; lis = keep; keep = tmp; }
    for (int64_t i = 0; i < refine_end; i++) {
      int b = src_bit(&src);
      mag[lsp.v[i]] = mag[lsp.v[i]] + (double)b * t;
    }
    nn--;
  }
  for (int64_t i = 0; i < n; i++) coeffs_out[i] = sgn[i] * mag[i];
  *n_last_out = n_last;
  free(mag); free(sgn); free(sig); free(csig);
  free(lip.v); free(lsp.v); free(newly.v); free(achild.v);
  sl_free(&lis); sl_free(&wave); sl_free(&next); sl_free(&keep);
  tree_free(&tr);
  return EO_OK;
}

/* dequantized_field (base_codec.py:70-83) */
/* opt-in JPEG2000-style base layer (ebcot_oracle.c): 0 SPIHT, 1 EBCOT */
static int g_base_codec = 0;
void eo_set_base_codec(int codec) { g_base_codec = codec; }

static int dequantized_field(const uint8_t *data, int64_t len, int64_t prefix_len, int rows,
                             int cols, int midpoint, double *out) {
  if (len >= 2 && data[0] == 'J' && data[1] == '2') { /* EBCOT base stream */
    int st = eo_ebcot_decode(data, prefix_len < 0 ? len : prefix_len, rows, cols, out);
    if (st) return st;
    eo_inverse_dwt(out, rows, cols, data[3]);
    return EO_OK;
  }
  int n_last;
  int st = eo_spiht_decode(data, len, prefix_len, rows, cols, out, &n_last);
  if (st) return st;
  int64_t n = (int64_t)rows * cols;
  if (midpoint && n_last != NLAST_NONE) {
    double off = ldexp(0.5, n_last);
    for (int64_t i = 0; i < n; i++) {
      double sg = out[i] > 0 ? 1.0 : (out[i] < 0 ? -1.0 : 0.0);
      out[i] = out[i] + sg * off;
    }
  }
  eo_inverse_dwt(out, rows, cols, data[3]);
  return EO_OK;
}

/* CPython float floor division (Objects/floatobject.c float_divmod) */
static double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) div -= 1.0;
  }
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (div - fl > 0.5) fl += 1.0;
  } else {
    fl = copysign(0.0, vx / wx);
  }
  return fl;
}

/* base_codec.py:34-38 */
int64_t eo_budget_for_ratio(int rows, int cols, double ratio) {
  if (ratio < 1.0) return -1;
  double raw = (double)((int64_t)rows * cols * 4);
  int64_t b = (int64_t)py_floordiv(raw, ratio);
  return b > HEADER_SIZE ? b : HEADER_SIZE;
}

static int64_t stream_cap(int64_t n) { return HEADER_SIZE + 16 * n + 64; }

/* base_codec.py:41-61 */
int64_t eo_base_encode_budget(const double *norm, int rows, int cols, int64_t budget,
                              double eps, uint8_t *out, int64_t cap, double *q_out,
                              double *decoded) {
  if (!(eps > 0.0 && eps < 1.0)) return -EO_E_ARGUMENT;
  int64_t n = (int64_t)rows * cols;
  int levels = eo_default_levels(rows, cols);
  levels = eo_clamp_levels(rows, cols, levels);
  double *pyr = malloc(sizeof(double) * n);
  memcpy(pyr, norm, sizeof(double) * n);
  eo_forward_dwt(pyr, rows, cols, levels);
  int64_t len = g_base_codec == 1 ? eo_ebcot_encode(pyr, rows, cols, levels, budget, out, cap)
                                   : eo_spiht_encode(pyr, rows, cols, levels, budget, 24, out, cap);
  free(pyr);
  if (len < 0) return len;
  int st = dequantized_field(out, len, -1, rows, cols, 0, decoded);
  if (st) return -st;
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; i++) cnt += fabs(decoded[i] - norm[i]) <= eps;
  *q_out = (double)cnt / (double)n;
  return len;
}

/* ---- pipeline (pipeline.py:87-329) ---------------------------------- */

typedef struct {
  int64_t budget, len;
  double q, maxerr;
  int pure_known;
} memo_t;

typedef struct {
  const float *orig;
  const double *norm;
  double vmin, vmax, eps_abs, eps_rel;
  int rows, cols;
  int64_t n, raw;
  memo_t *memo;
  int nmemo, capmemo;
  uint8_t *sbuf;
  int64_t scap;
  double *dec;
  int64_t *tb; double *tq; int tcap;
  int status;
} coder_t;

/* pipeline.py:116-119: max |f32(vmin + v*range) - orig| in float64 */
static double max_err(const coder_t *c, const double *dec) {
  double range = c->vmax - c->vmin, m = 0.0;
  for (int64_t i = 0; i < c->n; i++) {
    float rec = (float)(c->vmin + dec[i] * range);
    double e = fabs((double)rec - (double)c->orig[i]);
    if (e > m) m = e;
  }
  return m;
}

/* _ChunkCoder.at_budget (pipeline.py:105-110) */
static memo_t *at_budget(coder_t *c, int64_t budget) {
  if (budget > c->raw) budget = c->raw;
  if (budget < HEADER_SIZE) budget = HEADER_SIZE;
  for (int i = 0; i < c->nmemo; i++)
    if (c->memo[i].budget == budget) return &c->memo[i];
  double q;
  int64_t len = eo_base_encode_budget(c->norm, c->rows, c->cols, budget, c->eps_rel, c->sbuf,
                                      c->scap, &q, c->dec);
  if (len < 0) { c->status = (int)-len; len = HEADER_SIZE; q = 0.0; }
  if (c->nmemo == c->capmemo) {
    c->capmemo = c->capmemo ? 2 * c->capmemo : 64;
    c->memo = realloc(c->memo, sizeof(memo_t) * c->capmemo);
  }
  memo_t *m = &c->memo[c->nmemo];
  if (c->tb && c->nmemo < c->tcap) { c->tb[c->nmemo] = budget; c->tq[c->nmemo] = q; }
  c->nmemo++;
  m->budget = budget; m->len = len; m->q = q;
  m->maxerr = max_err(c, c->dec); /* what pure_ok would compute from the cached decode */
  m->pure_known = 0;
  return m;
}

static memo_t *at_ratio(coder_t *c, double ratio) {
  return at_budget(c, eo_budget_for_ratio(c->rows, c->cols, ratio));
}

static int pure_ok(coder_t *c, int64_t budget) {
  memo_t *m = at_budget(c, budget);
  m->pure_known = 1;
  return m->maxerr <= c->eps_abs;
}

/* pipeline.py:142-199; returns the chosen budget */
static int64_t search_base(coder_t *c, double q, double r0_param, double tol) {
  double r_cap = (double)c->raw / (double)HEADER_SIZE;
  if (r_cap < 1.0) r_cap = 1.0;
  double r0 = r0_param > 1.0 ? r0_param : 1.0;
  if (r0 > r_cap) r0 = r_cap;
  memo_t *e0 = at_ratio(c, r0);
  int64_t b0 = e0->budget;
  double q_a0 = e0->q;
  double r_low = r0, r_high = r0;
  int have_ef = q_a0 >= q;
  double q_a = q_a0;
  while (q_a < q && r_low > 1.0) {
    r_low = r_low / 2.0;
    if (r_low < 1.0) r_low = 1.0;
    q_a = at_ratio(c, r_low)->q;
  }
  if (q_a >= q) { at_ratio(c, r_low); have_ef = 1; }
  if (!have_ef) return at_ratio(c, 1.0)->budget;
  (void)b0;
  q_a = q_a0;
  while (q_a > q && r_high < r_cap) {
    r_high = r_high * 2.0;
    if (r_high > r_cap) r_high = r_cap;
    q_a = at_ratio(c, r_high)->q;
  }
  while (r_high - r_low > tol) {
    double r_mid = 0.5 * (r_low + r_high);
    if (at_ratio(c, r_mid)->q < q) r_high = r_mid;
    else r_low = r_mid;
  }
  /* byte-exact refinement seeded from the memo */
  int64_t hi = -1, lo = HEADER_SIZE - 1;
  for (int i = 0; i < c->nmemo; i++)
    if (c->memo[i].q >= q && (hi < 0 || c->memo[i].budget < hi)) hi = c->memo[i].budget;
  for (int i = 0; i < c->nmemo; i++)
    if (c->memo[i].q < q && c->memo[i].budget < hi && c->memo[i].budget > lo) lo = c->memo[i].budget;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) / 2;
    if (at_budget(c, mid)->q >= q) hi = mid;
    else lo = mid;
  }
  return hi;
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return x < y ? -1 : x > y;
}

/* pipeline.py:215-236; returns the budget or -1 for None */
static int64_t search_pure(coder_t *c) {
  if (pure_ok(c, HEADER_SIZE)) return HEADER_SIZE;
  if (!pure_ok(c, c->raw)) return -1;
  int64_t lo = HEADER_SIZE, hi = c->raw;
  int nc = c->nmemo;
  int64_t *cached = malloc(sizeof(int64_t) * nc);
  for (int i = 0; i < nc; i++) cached[i] = c->memo[i].budget;
  qsort(cached, nc, sizeof(int64_t), cmp_i64);
  for (int i = 0; i < nc; i++)
    if (pure_ok(c, cached[i]) && cached[i] < hi) hi = cached[i];
  for (int i = 0; i < nc; i++)
    if (cached[i] < hi && !pure_ok(c, cached[i]) && cached[i] > lo) lo = cached[i];
  free(cached);
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) / 2;
    if (pure_ok(c, mid)) hi = mid;
    else lo = mid;
  }
  return hi;
}

int eo_compress_chunk(const float *values, int rows, int cols, double eps_rel, double q,
                      double r0, double search_tol, eo_chunk_result *res, uint8_t *payload,
                      int64_t payload_cap, int64_t *trace_budgets, double *trace_q,
                      int trace_cap, int64_t *trace_trunc, int trunc_cap) {
  memset(res, 0, sizeof(*res));
  /* EbccParams.validate (pipeline.py:54-62) */
  if (!(eps_rel > 0.0 && eps_rel < 1.0) || !(q > 0.0 && q <= 1.0) || r0 < 1.0 ||
      !(search_tol > 0.0)) {
    res->status = EO_E_ARGUMENT;
    return EO_E_ARGUMENT;
  }
  int64_t n = (int64_t)rows * cols;
  /* core.normalize (core.py:161-180) */
  float fmin = values[0], fmax = values[0];
  int pos_zero = 0;
  for (int64_t i = 0; i < n; i++) {
    if (values[i] < fmin) fmin = values[i];
    if (values[i] > fmax) fmax = values[i];
    if (values[i] == 0.0f && !signbit(values[i])) pos_zero = 1;
  }
  /* tied signed zeros: numpy keeps one by its SIMD lane order (CPU-dependent);
   * pinned here (and on the GPU) as "+0.0 preferred" */
  if (fmin == 0.0f) fmin = pos_zero ? 0.0f : -0.0f;
  if (fmax == 0.0f) fmax = pos_zero ? 0.0f : -0.0f;
  double vmin = fmin, vmax = fmax, vrange = vmax - vmin;
  res->vmin = vmin; res->vmax = vmax;
  if (vrange < 1e-30) { res->mode = 0; return EO_OK; }
  double *norm = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; i++) norm[i] = ((double)values[i] - vmin) / vrange;

  coder_t c;
  memset(&c, 0, sizeof(c));
  c.orig = values; c.norm = norm; c.vmin = vmin; c.vmax = vmax;
  c.eps_rel = eps_rel; c.eps_abs = eps_rel * (vmax - vmin);
  c.rows = rows; c.cols = cols; c.n = n; c.raw = n * 4;
  c.scap = stream_cap(n);
  c.sbuf = malloc(c.scap);
  c.dec = malloc(sizeof(double) * n);
  c.tb = trace_budgets; c.tq = trace_q; c.tcap = trace_cap;

  int levels = eo_clamp_levels(rows, cols, eo_default_levels(rows, cols));
  int64_t base_budget = search_base(&c, q, r0, search_tol);
  /* recover the chosen base encoding (a memo hit in the reference) */
  double qq;
  double *base_dec = malloc(sizeof(double) * n);
  uint8_t *base_stream = malloc(c.scap);
  int64_t base_len = eo_base_encode_budget(norm, rows, cols, base_budget, eps_rel, base_stream,
                                           c.scap, &qq, base_dec);

  /* two-layer candidate (pipeline.py:300-309) */
  double *resid = malloc(sizeof(double) * n), *rec = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; i++) resid[i] = norm[i] - base_dec[i];
  eo_forward_dwt(resid, rows, cols, levels);
  int64_t rcap = stream_cap(n) * 2;
  uint8_t *rstream = malloc(rcap);
  int64_t two_t = -1, rlen = 0;
  int ntr = 0;
  int planes_used = 0;
  for (int pass = 0; pass < 2 && two_t < 0; pass++) {
    int planes = pass == 0 ? 24 : 32;
    rlen = eo_spiht_encode(resid, rows, cols, levels, -1, planes, rstream, rcap);
    if (rlen < 0) { c.status = (int)-rlen; break; }
    int64_t total = rlen - HEADER_SIZE;
    /* _truncation_search (pipeline.py:243-254) */
#define ERR_AT(tt, outv)                                                          \
    do {                                                                          \
      if (trace_trunc && ntr < trunc_cap) trace_trunc[ntr] = (tt);                \
      ntr++;                                                                      \
      dequantized_field(rstream, rlen, HEADER_SIZE + (tt), rows, cols, 1, rec);   \
      for (int64_t i_ = 0; i_ < n; i_++) rec[i_] = base_dec[i_] + rec[i_];        \
      (outv) = max_err(&c, rec);                                                  \
    } while (0)
    double e;
    ERR_AT(0, e);
    if (e <= c.eps_abs) { two_t = 0; planes_used = planes; break; }
    ERR_AT(total, e);
    if (e > c.eps_abs) continue;
    int64_t lo = 0, hi = total;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) / 2;
      ERR_AT(mid, e);
      if (e <= c.eps_abs) hi = mid;
      else lo = mid;
    }
    two_t = hi;
    planes_used = planes;
#undef ERR_AT
  }

  /* pure-base candidate */
  int64_t pure_budget = search_pure(&c);
  int64_t pure_len = -1;
  for (int i = 0; i < c.nmemo && pure_budget >= 0; i++)
    if (c.memo[i].budget == pure_budget) pure_len = c.memo[i].len;

  res->n_base_probes = c.nmemo;
  res->n_trunc_probes = ntr;
  int status = c.status;
  if (status == EO_OK) {
    int64_t two_len = two_t >= 0 ? base_len + HEADER_SIZE + two_t : -1;
    if (pure_budget < 0 && two_t < 0) {
      status = EO_E_RESIDUAL;
    } else if (pure_budget >= 0 && (two_t < 0 || pure_len <= two_len)) {
      res->mode = 1;
      res->base_len = pure_len;
      res->resid_len = 0;
      if (pure_len > payload_cap) status = EO_E_CAPACITY;
      else {
        double qp;
        eo_base_encode_budget(norm, rows, cols, pure_budget, eps_rel, payload, pure_len + 16, &qp,
                              c.dec);
      }
    } else {
      res->mode = 2;
      res->base_len = base_len;
      res->resid_len = HEADER_SIZE + two_t;
      res->resid_planes = planes_used;
      if (two_len > payload_cap) status = EO_E_CAPACITY;
      else {
        memcpy(payload, base_stream, base_len);
        memcpy(payload + base_len, rstream, HEADER_SIZE + two_t);
      }
    }
  }
  res->status = status;
  free(norm); free(c.sbuf); free(c.dec); free(c.memo); free(base_dec); free(base_stream);
  free(resid); free(rec); free(rstream);
  return status;
}

int eo_decompress_chunk(int mode, double vmin, double vmax, const uint8_t *payload,
                        int64_t base_len, int64_t resid_len, int rows, int cols, float *out) {
  int64_t n = (int64_t)rows * cols;
  if (mode == 0) {
    for (int64_t i = 0; i < n; i++) out[i] = (float)vmin;
    return EO_OK;
  }
  double *field = malloc(sizeof(double) * n);
  int st = dequantized_field(payload, base_len, -1, rows, cols, 0, field);
  if (st) { free(field); return st; }
  if (mode == 2 && resid_len > 0) {
    double *r = malloc(sizeof(double) * n);
    st = dequantized_field(payload + base_len, resid_len, -1, rows, cols, 1, r);
    if (st) { free(field); free(r); return st; }
    for (int64_t i = 0; i < n; i++) field[i] = field[i] + r[i];
    free(r);
  }
  double range = vmax - vmin;
  for (int64_t i = 0; i < n; i++) out[i] = (float)(vmin + field[i] * range);
  free(field);
  return EO_OK;
}
