/* bitlamb_oracle.c — TEST INFRASTRUCTURE ONLY (see bitlamb_oracle.h).
 *
 * Clean-room C restatement of the reference algorithm, function by function.
 * Every routine cites the reference file:line (relative to
 * /root/reference/proj) it restates.  Arithmetic follows the reference's
 * evaluation order operation by operation; in the f32 build every elementwise
 * operation is rounded to float, per-step scalars are formed in double exactly
 * as the reference forms them and rounded to float once, and reductions
 * accumulate in double.
 */
#include "bitlamb_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef OC_REAL_FLOAT
#define OC_TILE_ORDER 1
#define R(x) ((float)(x))
#define OC_FABS(x) fabsf(x)
#else
#define OC_TILE_ORDER 0
#define R(x) ((double)(x))
#define OC_FABS(x) fabs(x)
#endif

/* OpenMP: elementwise maps and per-tile / per-block partial sums run in
 * parallel; every reduction still combines its partials in the canonical
 * order (serially), so results are independent of the thread count.  Small
 * vectors stay serial. */
#ifdef _OPENMP
#define OC_PAR _Pragma("omp parallel for schedule(static) if (n_ > 65536)")
#else
#define OC_PAR
#endif

static _Thread_local char g_err[512];

/* Reusable scratch (grow-only, one buffer per role) and parallel copies: at
 * BERT-Large sizes fresh 1.3 GB allocations and serial memcpy dominated the
 * checker's run time.  Roles never nest with themselves. */
enum { S_PAD, S_CORR, S_DEC, S_WBITS, S_INBOX, S_AVG, S_CORR2, S_DEC2, S_SBITS, S_RESULT, S_STREAMS,
       S_MG, S_REC, S_U, S_LAVG, S_COUNT };
static void* g_scr[S_COUNT];
static size_t g_scr_n[S_COUNT];
static void* scratch(int role, size_t bytes) {
  if (bytes + 64u > g_scr_n[role]) {
    free(g_scr[role]);
    g_scr[role] = malloc(bytes + 64u);
    g_scr_n[role] = bytes + 64u;
  }
  return g_scr[role];
}
static void pcopy(void* dst, const void* src, size_t bytes) {
  const size_t blk = (size_t)1 << 22, nb = (bytes + blk - 1u) / blk;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) if (nb > 4)
#endif
  for (size_t b = 0; b < nb; ++b) {
    const size_t o = b * blk, k = bytes - o < blk ? bytes - o : blk;
    memcpy((char*)dst + o, (const char*)src + o, k);
  }
}

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* oc_last_error(void) { return g_err; }
int oc_real_bytes(void) { return (int)sizeof(oc_real); }

static int oc_isfinite(oc_real x) { return isfinite(x) ? 1 : 0; }

/* ------------------------------------------------------------------------ */
/* Reductions.                                                               */
/* ------------------------------------------------------------------------ */
enum { SUM_ABS = 0, SUM_SQ = 1 };

static double term(oc_real x, int kind) {
  const double d = (double)x;
  return kind == SUM_ABS ? fabs(d) : d * d; /* d*d exact for float inputs */
}

#if OC_TILE_ORDER
/* Canonical B200 order (DESIGN.md §4 "tile-tree"): a segment is cut into
 * 4096-element tiles of 32 rows x 128; lane l (0..31) accumulates, in double,
 * elements 4l..4l+3 of every row in (row, element) order; the 32 lane sums are
 * combined by the xor butterfly (16,8,4,2,1); tile partials are combined by
 * 1024 ascending stripes followed by two butterfly levels.  This is exactly
 * what kernels.cu computes with warp shuffles. */
static double butterfly32(double* a) {
  double b[32];
  for (int s = 16; s >= 1; s >>= 1) {
    for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ s];
    memcpy(a, b, sizeof b);
  }
  return a[0];
}

static double tile_partial(const oc_real* x, uint64_t len, uint64_t t, int kind) {
  double acc[32];
  for (int l = 0; l < 32; ++l) acc[l] = 0.0;
  const uint64_t base = t * 4096u;
  if (base + 4096u <= len) { /* full tile: same order, no bounds test */
    const oc_real* xt = x + base;
    for (int r = 0; r < 32; ++r)
      for (int l = 0; l < 32; ++l)
        for (int q = 0; q < 4; ++q) acc[l] += term(xt[128 * r + 4 * l + q], kind);
    return butterfly32(acc);
  }
  for (int r = 0; r < 32; ++r) {
    for (int l = 0; l < 32; ++l) {
      for (int q = 0; q < 4; ++q) {
        const uint64_t i = base + 128u * (uint64_t)r + 4u * (uint64_t)l + (uint64_t)q;
        if (i < len) acc[l] += term(x[i], kind);
      }
    }
  }
  return butterfly32(acc);
}

static double combine_partials(const double* p, uint64_t T) {
  double* stripe = calloc(1024, sizeof(double));
  for (uint64_t t = 0; t < T; ++t) stripe[t % 1024u] += p[t];
  double warp[32];
  for (int w = 0; w < 32; ++w) warp[w] = butterfly32(stripe + 32 * w);
  free(stripe);
  return butterfly32(warp);
}

static double canonical_sum(const oc_real* x, uint64_t len, int kind) {
  const uint64_t T = (len + 4095u) / 4096u;
  if (T == 0) return 0.0;
  double* p = malloc(T * sizeof(double));
  const uint64_t n_ = len;
  OC_PAR
  for (uint64_t t = 0; t < T; ++t) p[t] = tile_partial(x, len, t, kind);
  const double s = combine_partials(p, T);
  free(p);
  return s;
}
#else
/* Reference order: kernels.cpp:134-150 (blocked_sum, kReduceBlock = 4096):
 * serial left-to-right inside each block, block partials summed in order. */
static double serial_sum(const oc_real* x, uint64_t lo, uint64_t hi, int kind) {
  double acc = 0.0;
  for (uint64_t i = lo; i < hi; ++i) acc += term(x[i], kind);
  return acc;
}

static double canonical_sum(const oc_real* x, uint64_t len, int kind) {
  if (len <= 4096u) return serial_sum(x, 0, len, kind);
  const uint64_t nb = (len + 4095u) / 4096u, n_ = len;
  double* part = malloc(nb * sizeof(double));
  OC_PAR
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t lo = b * 4096u;
    const uint64_t hi = lo + 4096u < len ? lo + 4096u : len;
    part[b] = serial_sum(x, lo, hi, kind);
  }
  double acc = 0.0;
  for (uint64_t b = 0; b < nb; ++b) acc += part[b]; /* block partials in order */
  free(part);
  return acc;
}
#endif

double oc_canonical_sum(const oc_real* x, uint64_t len, int kind) {
  return canonical_sum(x, len, kind);
}

/* kernels.cpp:185-198 max_abs_ratio (start 0, |a|/max(b, floor)) */
static double max_abs_ratio(const oc_real* a, const oc_real* b, uint64_t n,
                            double floor_) {
  const oc_real fl = R(floor_);
  oc_real m = 0;
  const uint64_t n_ = n;
#ifdef _OPENMP
#pragma omp parallel if (n_ > 65536)
#endif
  {
    oc_real mt = 0; /* maxima are order-free: per-thread, then combined by the same rule */
#ifdef _OPENMP
#pragma omp for schedule(static) nowait
#endif
    for (uint64_t i = 0; i < n; ++i) {
      const oc_real den = b[i] < fl ? fl : b[i]; /* std::max(b[i], floor) */
      const oc_real q = OC_FABS(a[i]) / den;
      mt = mt < q ? q : mt; /* std::max(m, q) */
    }
#ifdef _OPENMP
#pragma omp critical
#endif
    m = m < mt ? mt : m;
  }
  return (double)m;
}

/* kernels.cpp:172-183 max_abs */
static double max_abs(const oc_real* v, uint64_t n) {
  oc_real m = 0;
  const uint64_t n_ = n;
#ifdef _OPENMP
#pragma omp parallel if (n_ > 65536)
#endif
  {
    oc_real mt = 0;
#ifdef _OPENMP
#pragma omp for schedule(static) nowait
#endif
    for (uint64_t i = 0; i < n; ++i) {
      const oc_real a = OC_FABS(v[i]);
      mt = mt < a ? a : mt; /* std::max(m, std::abs(x)) */
    }
#ifdef _OPENMP
#pragma omp critical
#endif
    m = m < mt ? mt : m;
  }
  return (double)m;
}

static int all_finite(const oc_real* v, uint64_t n) {
  int ok = 1;
  const uint64_t n_ = n;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) reduction(&& : ok) if (n_ > 65536)
#endif
  for (uint64_t i = 0; i < n; ++i) ok = ok && oc_isfinite(v[i]);
  return ok;
}

/* vector_ops.cpp:25-28 */
static double clip(double x, double a, double b) {
  const double lo = x < a ? a : x; /* std::max(x, a) */
  return b < lo ? b : lo;          /* std::min(lo, b) */
}

/* ------------------------------------------------------------------------ */
/* Compression (compression.cpp).                                           */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint8_t* bits; /* ceil(len/8) bytes, LSB-first, pad bits zero (:40) */
  oc_real scale;
  uint64_t len;
} oc_block;

/* compression.cpp:37-60 CompressedBlock::compress */
static int block_compress(const oc_real* v, uint64_t len, oc_block* b) {
  b->len = len;
  const uint64_t nbytes = (len + 7u) / 8u, n_ = len;
  OC_PAR
  for (uint64_t y = 0; y < nbytes; ++y) { /* byte-parallel, as compression.cpp:42-53 */
    uint8_t byte = 0;
    for (uint64_t i = 8u * y; i < 8u * y + 8u && i < len; ++i)
      if (v[i] >= 0) byte |= (uint8_t)(1u << (i & 7u));
    b->bits[y] = byte;
  }
  const double s = len == 0 ? 0.0 : canonical_sum(v, len, SUM_ABS) / (double)len;
  b->scale = R(s);
  if (!oc_isfinite(b->scale)) {
    return fail(OC_INVALID_ARGUMENT, "compress: input vector is not finite");
  }
  return OC_OK;
}

static int bit_at(const uint8_t* bits, uint64_t i) { return (bits[i >> 3] >> (i & 7u)) & 1; }

/* compression.cpp:68-81 decompress_into */
static void block_decompress(const uint8_t* bits, oc_real s, uint64_t len, oc_real* out) {
  const uint64_t n_ = len;
  OC_PAR
  for (uint64_t i = 0; i < len; ++i) out[i] = s == 0 ? (oc_real)0 : (bit_at(bits, i) ? s : -s);
}

/* compression.cpp:91-99 serialize: sign bytes then LE float32 scale */
static void block_serialize(const oc_block* b, uint8_t* out) {
  const uint64_t nb = (b->len + 7u) / 8u;
  memcpy(out, b->bits, nb);
  const float f = (float)b->scale;
  uint32_t u;
  memcpy(&u, &f, 4);
  for (int k = 0; k < 4; ++k) out[nb + k] = (uint8_t)((u >> (8 * k)) & 0xffu);
}

/* In-memory message between the oracle's phases: sign bytes followed by the
 * scale in native precision (the reference passes the double scale in-process,
 * comm_sim.hpp:141; only serialize() rounds it to float).  For the f32 build
 * this is byte-identical to serialize(). */
static uint64_t ipkt_bytes(uint64_t len) { return (len + 7u) / 8u + sizeof(oc_real); }

static void block_store(const oc_block* b, uint8_t* out) {
  const uint64_t nb = (b->len + 7u) / 8u;
  memcpy(out, b->bits, nb);
  memcpy(out + nb, &b->scale, sizeof(oc_real));
}

static oc_real stored_scale(const uint8_t* pkt, uint64_t len) {
  oc_real s;
  memcpy(&s, pkt + (len + 7u) / 8u, sizeof(oc_real));
  return s;
}

static void stored_to_wire(const uint8_t* pkt, uint64_t len, uint8_t* out) {
  oc_block b;
  b.bits = (uint8_t*)pkt;
  b.len = len;
  b.scale = stored_scale(pkt, len);
  block_serialize(&b, out);
}

/* compression.cpp:166-198 compress_with_feedback (span form).  corrected is
 * scratch of len.  kind 0 = one-bit, 1 = identity. */
static int compress_with_feedback(const oc_real* v, oc_real* delta, uint64_t len, int kind,
                                  double es, oc_real* corrected, oc_block* out) {
  const oc_real a = R(1.0), b = R(es);
  const uint64_t n_ = len;
  OC_PAR
  for (uint64_t i = 0; i < len; ++i) corrected[i] = a * v[i] + b * delta[i]; /* :181 */
  if (kind == 1) {                                                           /* :184-188 */
    for (uint64_t i = 0; i < len; ++i) delta[i] = 0;
    out->len = len;
    out->scale = 0;
    return OC_OK;
  }
  int st = block_compress(corrected, len, out); /* :182 */
  if (st) return st;
  const oc_real s = out->scale;
  OC_PAR
  for (uint64_t i = 0; i < len; ++i) { /* :190-196 */
    const oc_real rec = bit_at(out->bits, i) ? s : -s;
    delta[i] = v[i] + delta[i] - rec;
  }
  return OC_OK;
}

int oc_compress_with_feedback(const oc_real* v, oc_real* delta, uint64_t d, int kind,
                              double es, uint8_t* bytes, double* scale,
                              oc_real* decompressed) {
  oc_block b;
  b.bits = calloc((d + 7u) / 8u + 1u, 1);
  oc_real* corr = malloc((d + 1u) * sizeof(oc_real));
  int st = compress_with_feedback(v, delta, d, kind, es, corr, &b);
  if (st == OC_OK) {
    if (kind == 1) {
      memcpy(decompressed, corr, d * sizeof(oc_real));
      *scale = 0.0;
    } else {
      block_serialize(&b, bytes);
      *scale = (double)b.scale;
      block_decompress(b.bits, b.scale, d, decompressed);
    }
  }
  free(b.bits);
  free(corr);
  return st;
}

/* comm_sim.cpp:36-48 */
int oc_volume_reduction(double w, double bb, double cb, double* out) {
  if (!(w >= 0.0 && w <= 1.0))
    return fail(OC_INVALID_ARGUMENT, "volume_reduction: warmup_ratio must be in [0, 1]");
  if (!(bb > 0.0)) return fail(OC_INVALID_ARGUMENT, "volume_reduction: baseline_bits must be > 0");
  if (!(cb >= 0.0))
    return fail(OC_INVALID_ARGUMENT, "volume_reduction: compressed bits must be >= 0");
  const double denom = w + (1.0 - w) * cb / bb;
  *out = denom == 0.0 ? INFINITY : 1.0 / denom;
  return OC_OK;
}

/* ------------------------------------------------------------------------ */
/* SimCluster (comm_sim.cpp).                                               */
/* ------------------------------------------------------------------------ */
typedef struct {
  double delta_l2, delta_linf, corrected_linf, max_delta_linf, max_corrected_linf;
} oc_stats;

typedef struct {
  int n, kind, baseline_bits, verify;
  double tol;
  uint64_t dim, padded, chunk;
  oc_real* werr;      /* n x padded   (:60) */
  oc_real* serr;      /* n x chunk    (:61) */
  double* wcmax;      /* n: max|corrected| of worker_corrected_ (:62), kept as its maximum only */
  uint8_t* wpk;       /* [worker][server] serialized packets of the last call */
  uint8_t* spk;       /* [server] serialized server packets of the last call */
  oc_stats* wstats;   /* n */
  oc_stats* sstats;   /* n */
  uint64_t ledger[6]; /* gather, scatter, lossless, baseline, ncomp, nloss */
  uint64_t checks;
} oc_cluster;

/* comm_sim.cpp:50-66 */
int oc_cluster_new(int n, uint64_t dim, int kind, int baseline_bits, int verify, void** out) {
  if (n < 1) return fail(OC_INVALID_ARGUMENT, "SimCluster: need at least one worker");
  if (dim < 1) return fail(OC_INVALID_ARGUMENT, "SimCluster: dim must be >= 1");
  if (baseline_bits < 1) return fail(OC_INVALID_ARGUMENT, "SimCluster: baseline bits must be >= 1");
  oc_cluster* c = calloc(1, sizeof *c);
  c->n = n;
  c->kind = kind;
  c->baseline_bits = baseline_bits;
  c->verify = verify;
  c->tol = 1e-12;
  c->dim = dim;
  c->padded = (dim + (uint64_t)n - 1u) / (uint64_t)n * (uint64_t)n;
  c->chunk = c->padded / (uint64_t)n;
  c->werr = calloc((size_t)n * c->padded, sizeof(oc_real));
  c->serr = calloc((size_t)n * c->chunk, sizeof(oc_real));
  c->wcmax = calloc((size_t)n, sizeof(double));
  c->wpk = calloc((size_t)n * (size_t)n * ipkt_bytes(c->chunk), 1);
  c->spk = calloc((size_t)n * ipkt_bytes(c->chunk), 1);
  c->wstats = calloc((size_t)n, sizeof(oc_stats));
  c->sstats = calloc((size_t)n, sizeof(oc_stats));
  *out = c;
  return OC_OK;
}

void oc_cluster_set_tolerance(void* cv, double tol) { ((oc_cluster*)cv)->tol = tol; }

void oc_cluster_free(void* cv) {
  oc_cluster* c = cv;
  if (!c) return;
  free(c->werr);
  free(c->serr);
  free(c->wcmax);
  free(c->wpk);
  free(c->spk);
  free(c->wstats);
  free(c->sstats);
  free(c);
}

uint64_t oc_cluster_padded(void* c) { return ((oc_cluster*)c)->padded; }
uint64_t oc_cluster_chunk(void* c) { return ((oc_cluster*)c)->chunk; }

/* comm_sim.cpp:68-79 */
static uint64_t chunk_real_elems(const oc_cluster* c, uint64_t j) {
  const uint64_t begin = j * c->chunk;
  if (begin >= c->dim) return 0;
  return c->chunk < c->dim - begin ? c->chunk : c->dim - begin;
}

static uint64_t chunk_payload_bits(const oc_cluster* c, uint64_t j) {
  const uint64_t real = chunk_real_elems(c, j);
  if (real == 0) return 0;
  if (c->kind == 0) return real + 32u;
  return real * (uint64_t)c->baseline_bits;
}

/* comm_sim.cpp:83-106 */
static int verify_chunk(const oc_cluster* c, const oc_real* corrected, const oc_real* dec,
                        const oc_real* delta_new, uint64_t len) {
  for (uint64_t k = 0; k < len; ++k) {
    const double lhs = (double)corrected[k];
    const double rhs = (double)dec[k] + (double)delta_new[k];
    double denom = fabs(lhs);
    if (fabs((double)dec[k]) > denom) denom = fabs((double)dec[k]);
    if (1e-300 > denom) denom = 1e-300;
    if (fabs(lhs - rhs) > c->tol * denom) {
      return fail(OC_LOGIC,
                  "error-compensation identity violated at element %llu: |%.17g - %.17g| "
                  "exceeds relative tolerance %g",
                  (unsigned long long)k, lhs, rhs, c->tol);
    }
  }
  return OC_OK;
}

static void stats_update(oc_stats* s, double l2, double linf, double cinf) {
  s->delta_l2 = l2;
  s->delta_linf = linf;
  s->corrected_linf = cinf;
  if (linf > s->max_delta_linf) s->max_delta_linf = linf;
  if (cinf > s->max_corrected_linf) s->max_corrected_linf = cinf;
}

/* Worker phase of comm_sim.cpp:133-149 for one worker: padded copy, then every
 * chunk compressed with its slice of the worker residual.  packets: n slots of
 * ipkt_bytes(chunk) (in-memory layout).  corr_max (may be NULL) receives
 * max|corrected| over the padded stream (the endpoint statistic of :108-118). */
static int worker_phase(const oc_real* input, uint64_t dim, int n, int kind, oc_real* werr,
                        double es, uint8_t* packets, double* corr_max, const oc_cluster* vc) {
  const uint64_t padded = (dim + (uint64_t)n - 1u) / (uint64_t)n * (uint64_t)n;
  const uint64_t chunk = padded / (uint64_t)n;
  oc_real* p = scratch(S_PAD, (padded + 1u) * sizeof(oc_real)); /* :136-137 padded_input */
  pcopy(p, input, dim * sizeof(oc_real));
  for (uint64_t k = dim; k < padded; ++k) p[k] = 0;
  oc_real* corr = scratch(S_CORR, (chunk + 1u) * sizeof(oc_real)); /* one chunk at a time */
  double cmax = 0.0;
  oc_real* dec = scratch(S_DEC, (chunk + 1u) * sizeof(oc_real));
  oc_block b;
  b.bits = scratch(S_WBITS, (chunk + 7u) / 8u + 1u);
  int st = OC_OK;
  for (int j = 0; j < n && st == OC_OK; ++j) {
    const uint64_t off = (uint64_t)j * chunk;
    st = compress_with_feedback(p + off, werr + off, chunk, kind, es, corr, &b);
    if (st) break;
    if (corr_max) {
      const double mj = max_abs(corr, chunk);
      cmax = cmax < mj ? mj : cmax;
    }
    if (kind == 0) block_store(&b, packets + (size_t)j * ipkt_bytes(chunk));
    if (vc && vc->verify && es == 1.0) { /* :145-147 */
      if (kind == 0) block_decompress(b.bits, b.scale, chunk, dec);
      else memcpy(dec, corr, chunk * sizeof(oc_real));
      st = verify_chunk(vc, corr, dec, werr + off, chunk);
    }
  }
  if (corr_max) *corr_max = cmax;
  return st;
}

int oc_worker_compress(const oc_real* stream, uint64_t dim, int n, oc_real* werr, double es,
                       uint8_t* packets) {
  return worker_phase(stream, dim, n, 0, werr, es, packets, NULL, NULL);
}

/* Server phase of comm_sim.cpp:158-181 for one chunk: ascending-worker
 * decompress_accumulate (compression.cpp:83-89, skipped when scale == 0),
 * scale(1/n) (:164), then compression with the server residual. */
static int server_avg(const uint8_t* packets, uint64_t chunk, int n, oc_real* avg) {
  const double inv_n = 1.0 / (double)n;
  const uint64_t n_ = chunk;
  double sc[64];
  for (int i = 0; i < n && i < 64; ++i)
    sc[i] = (double)stored_scale(packets + (size_t)i * ipkt_bytes(chunk), chunk);
  OC_PAR
  for (uint64_t k = 0; k < chunk; ++k) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      const uint8_t* pk = packets + (size_t)i * ipkt_bytes(chunk);
      const double s = i < 64 ? sc[i] : (double)stored_scale(pk, chunk);
      if (s == 0.0) continue;
      acc += bit_at(pk, k) ? s : -s;
    }
    avg[k] = R(acc * inv_n);
  }
  return OC_OK;
}

int oc_server_reduce(const uint8_t* packets, uint64_t chunk, int n, oc_real* serr, double es,
                     uint8_t* out_packet) {
  oc_real* avg = scratch(S_AVG, (chunk + 1u) * sizeof(oc_real));
  oc_real* corr = scratch(S_CORR2, (chunk + 1u) * sizeof(oc_real));
  oc_block b;
  b.bits = scratch(S_SBITS, (chunk + 7u) / 8u + 1u);
  server_avg(packets, chunk, n, avg);
  int st = compress_with_feedback(avg, serr, chunk, 0, es, corr, &b);
  if (st == OC_OK) block_store(&b, out_packet);
  return st;
}

void oc_decompress(const uint8_t* packet, uint64_t len, oc_real* out) {
  block_decompress(packet, stored_scale(packet, len), len, out);
}

/* comm_sim.cpp:120-203 */
static int cluster_compressed(oc_cluster* c, const oc_real* inputs, double es, oc_real* out) {
  const int n = c->n;
  const uint64_t P = c->padded, ch = c->chunk, pb = ipkt_bytes(ch);
  int st = OC_OK;
  oc_real* result = scratch(S_RESULT, (P + 1u) * sizeof(oc_real)); /* every chunk is written */
  if (c->kind == 1) {
    /* Identity compressor: dense messages, residuals stay zero. */
    oc_real* corr_all = malloc(((size_t)n * P + 1u) * sizeof(oc_real));
    for (int i = 0; i < n; ++i) {
      oc_real* p = calloc(P + 1u, sizeof(oc_real));
      memcpy(p, inputs + (size_t)i * c->dim, c->dim * sizeof(oc_real));
      oc_block b;
      for (int j = 0; j < n; ++j) {
        compress_with_feedback(p + (uint64_t)j * ch, c->werr + (size_t)i * P + (uint64_t)j * ch, ch,
                               1, es, corr_all + (size_t)i * P + (uint64_t)j * ch, &b);
      }
      c->wcmax[i] = max_abs(corr_all + (size_t)i * P, P);
      free(p);
    }
    oc_real* avg = malloc((ch + 1u) * sizeof(oc_real));
    oc_real* corr = malloc((ch + 1u) * sizeof(oc_real));
    for (int j = 0; j < n; ++j) {
      for (uint64_t k = 0; k < ch; ++k) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += (double)corr_all[(size_t)i * P + (uint64_t)j * ch + k];
        avg[k] = R(acc * (1.0 / (double)n));
      }
      oc_block b;
      compress_with_feedback(avg, c->serr + (size_t)j * ch, ch, 1, es, corr, &b);
      memcpy(result + (uint64_t)j * ch, corr, ch * sizeof(oc_real));
      stats_update(&c->sstats[j], sqrt(canonical_sum(c->serr + (size_t)j * ch, ch, SUM_SQ)),
                   max_abs(c->serr + (size_t)j * ch, ch), max_abs(corr, ch));
    }
    free(avg);
    free(corr);
    free(corr_all);
  } else {
    for (int i = 0; i < n && st == OC_OK; ++i) {
      st = worker_phase(inputs + (size_t)i * c->dim, c->dim, n, 0, c->werr + (size_t)i * P, es,
                        c->wpk + (size_t)i * (size_t)n * pb, &c->wcmax[i], c);
    }
    uint8_t* inbox = scratch(S_INBOX, (size_t)n * pb);
    oc_real* avg = scratch(S_AVG, (ch + 1u) * sizeof(oc_real));
    oc_real* corr = scratch(S_CORR2, (ch + 1u) * sizeof(oc_real));
    oc_real* dec = scratch(S_DEC2, (ch + 1u) * sizeof(oc_real));
    oc_block b;
    b.bits = scratch(S_SBITS, (ch + 7u) / 8u + 1u);
    for (int j = 0; j < n && st == OC_OK; ++j) {
      for (int i = 0; i < n; ++i)
        pcopy(inbox + (size_t)i * pb, c->wpk + ((size_t)i * (size_t)n + (size_t)j) * pb, pb);
      server_avg(inbox, ch, n, avg);
      oc_real* se = c->serr + (size_t)j * ch;
      st = compress_with_feedback(avg, se, ch, 0, es, corr, &b);
      if (st) break;
      block_store(&b, c->spk + (size_t)j * pb);
      block_decompress(b.bits, b.scale, ch, dec);
      if (c->verify && es == 1.0) st = verify_chunk(c, corr, dec, se, ch);
      pcopy(result + (uint64_t)j * ch, dec, ch * sizeof(oc_real));
      stats_update(&c->sstats[j], sqrt(canonical_sum(se, ch, SUM_SQ)), max_abs(se, ch),
                   max_abs(corr, ch));
    }
  }
  if (st == OC_OK) {
    for (int i = 0; i < n; ++i) { /* :108-118 refresh_endpoint_stats */
      const oc_real* we = c->werr + (size_t)i * P;
      stats_update(&c->wstats[i], sqrt(canonical_sum(we, P, SUM_SQ)), max_abs(we, P), c->wcmax[i]);
    }
    uint64_t bits = 0; /* :189-197 ledger */
    for (int j = 0; j < n; ++j) bits += chunk_payload_bits(c, (uint64_t)j);
    c->ledger[0] += (uint64_t)(n - 1) * bits;
    c->ledger[1] += (uint64_t)(n - 1) * bits;
    c->ledger[3] += 2u * (uint64_t)(n - 1) * c->dim * (uint64_t)c->baseline_bits;
    c->ledger[4] += 1;
    if (c->verify && es == 1.0) c->checks += (uint64_t)n * (uint64_t)n + (uint64_t)n;
    pcopy(out, result, c->dim * sizeof(oc_real)); /* :202 truncate to dim */
  }
  return st;
}

int oc_cluster_compressed_allreduce_n(void* cv, const oc_real* inputs, int n_inputs, uint64_t len,
                                      double es, oc_real* out) {
  oc_cluster* c = cv;
  if ((uint64_t)n_inputs != (uint64_t)c->n)
    return fail(OC_DIMENSION, "compressed_allreduce: worker count: size mismatch (%d vs %d)",
                n_inputs, c->n);
  if (len != c->dim)
    return fail(OC_DIMENSION, "compressed_allreduce: input length: size mismatch (%llu vs %llu)",
                (unsigned long long)len, (unsigned long long)c->dim);
  return cluster_compressed(c, inputs, es, out);
}

int oc_cluster_compressed_allreduce(void* cv, const oc_real* inputs, double es, oc_real* out) {
  oc_cluster* c = cv;
  return cluster_compressed(c, inputs, es, out);
}

/* comm_sim.cpp:205-232 */
int oc_cluster_lossless_allreduce(void* cv, const oc_real* inputs, oc_real* out) {
  oc_cluster* c = cv;
  const double inv_n = 1.0 / (double)c->n;
  const uint64_t n_ = c->dim;
  OC_PAR
  for (uint64_t k = 0; k < c->dim; ++k) {
    double acc = 0.0;
    for (int i = 0; i < c->n; ++i) acc += (double)inputs[(size_t)i * c->dim + k];
    out[k] = R(acc * inv_n);
  }
  const uint64_t bits =
      2u * (uint64_t)(c->n - 1) * c->dim * (uint64_t)c->baseline_bits;
  c->ledger[2] += bits;
  c->ledger[3] += bits;
  c->ledger[5] += 1;
  return OC_OK;
}

void oc_cluster_worker_error(void* cv, int i, oc_real* out) {
  oc_cluster* c = cv;
  pcopy(out, c->werr + (size_t)i * c->padded, c->padded * sizeof(oc_real));
}

void oc_cluster_server_error(void* cv, int j, oc_real* out) {
  oc_cluster* c = cv;
  pcopy(out, c->serr + (size_t)j * c->chunk, c->chunk * sizeof(oc_real));
}

void oc_cluster_ledger(void* cv, uint64_t* out) { memcpy(out, ((oc_cluster*)cv)->ledger, 48); }

void oc_cluster_stats(void* cv, double* out) {
  oc_cluster* c = cv;
  int k = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const oc_stats* s = pass == 0 ? c->wstats : c->sstats;
    for (int i = 0; i < c->n; ++i) {
      out[k++] = s[i].delta_l2;
      out[k++] = s[i].delta_linf;
      out[k++] = s[i].corrected_linf;
      out[k++] = s[i].max_delta_linf;
      out[k++] = s[i].max_corrected_linf;
    }
  }
}

uint64_t oc_cluster_compensation_checks(void* c) { return ((oc_cluster*)c)->checks; }

int oc_cluster_packet(void* cv, int worker, int server, uint8_t* bytes) {
  oc_cluster* c = cv;
  const uint64_t pb = ipkt_bytes(c->chunk);
  stored_to_wire(c->wpk + ((size_t)worker * (size_t)c->n + (size_t)server) * pb, c->chunk, bytes);
  return OC_OK;
}

int oc_cluster_server_packet(void* cv, int server, uint8_t* bytes) {
  oc_cluster* c = cv;
  const uint64_t pb = ipkt_bytes(c->chunk);
  stored_to_wire(c->spk + (size_t)server * pb, c->chunk, bytes);
  return OC_OK;
}

/* ------------------------------------------------------------------------ */
/* Optimizer (optimizers.cpp).                                              */
/* ------------------------------------------------------------------------ */
enum { V_LAMB = 0, V_ADAM = 1, V_ONEBIT_LAMB = 2, V_BASIC = 3, V_ONEBIT_ADAM = 4 };

typedef struct {
  double beta1, beta2, beta3, eta, c_min, c_max, r_min, r_max, r_thr, wd, floor_;
  uint64_t total, warmup;
  int scaled_ef;
} oc_hp;

typedef struct {
  int variant, L, frozen, has_vf, has_mprev;
  oc_hp hp;
  uint64_t d;
  uint64_t* off; /* L+1 (FusedLayout, fusion.cpp:26-36) */
  oc_real *x, *m, *v, *vf, *mprev;
  double *c_avg, *r_prev, *coeff;
  double c_mean_prev, c_mean_prev2;
} oc_opt;

/* optimizers.cpp:60-74 HyperParams::validate */
static int validate(const oc_hp* h) {
  if (!(h->beta1 >= 0.0 && h->beta1 < 1.0)) return fail(OC_CONFIG, "beta1 must be in [0, 1)");
  if (!(h->beta2 >= 0.0 && h->beta2 < 1.0)) return fail(OC_CONFIG, "beta2 must be in [0, 1)");
  if (!(h->beta3 >= 0.0 && h->beta3 < 1.0)) return fail(OC_CONFIG, "beta3 must be in [0, 1)");
  if (!(h->eta > 0.0)) return fail(OC_CONFIG, "eta must be > 0");
  if (!(h->c_min <= h->c_max)) return fail(OC_CONFIG, "c_min must not exceed c_max");
  if (!(h->r_min <= h->r_max)) return fail(OC_CONFIG, "r_min must not exceed r_max");
  if (!(h->r_thr > 0.0 && h->r_thr < 1.0)) return fail(OC_CONFIG, "r_threshold must be in (0, 1)");
  if (!(h->wd >= 0.0)) return fail(OC_CONFIG, "weight_decay must be >= 0");
  if (!(h->floor_ > 0.0)) return fail(OC_CONFIG, "division_floor must be > 0");
  if (h->warmup > h->total) return fail(OC_CONFIG, "warmup_steps must not exceed total_steps");
  return OC_OK;
}

/* optimizers.cpp:76-97 */
int oc_opt_new(int variant, const uint64_t* sizes, int L, const double* hp, uint64_t total,
               uint64_t warmup, int scaled_ef, void** out) {
  oc_hp h = {hp[0], hp[1], hp[2], hp[3], hp[4], hp[5], hp[6], hp[7], hp[8], hp[9], hp[10],
             total, warmup, scaled_ef};
  int st = validate(&h);
  if (st) return st;
  if (L < 1) return fail(OC_INVALID_ARGUMENT, "Optimizer: need at least one layer");
  for (int l = 0; l < L; ++l)
    if (sizes[l] == 0) return fail(OC_INVALID_ARGUMENT, "Optimizer: layer size must be > 0");
  oc_opt* o = calloc(1, sizeof *o);
  o->variant = variant;
  o->L = L;
  o->hp = h;
  o->off = malloc(((size_t)L + 1u) * sizeof(uint64_t));
  o->off[0] = 0;
  for (int l = 0; l < L; ++l) o->off[l + 1] = o->off[l] + sizes[l];
  o->d = o->off[L];
  o->x = calloc(o->d + 1u, sizeof(oc_real));
  o->m = calloc(o->d + 1u, sizeof(oc_real));
  o->v = calloc(o->d + 1u, sizeof(oc_real));
  o->vf = calloc(o->d + 1u, sizeof(oc_real));
  o->mprev = calloc(o->d + 1u, sizeof(oc_real));
  o->c_avg = calloc((size_t)L, sizeof(double));
  o->r_prev = malloc((size_t)L * sizeof(double));
  o->coeff = malloc((size_t)L * sizeof(double));
  for (int l = 0; l < L; ++l) {
    o->r_prev[l] = 1.0;
    o->coeff[l] = 1.0; /* MomentumScales::uniform */
  }
  o->c_mean_prev = o->c_mean_prev2 = 1.0;
  *out = o;
  return OC_OK;
}

void oc_opt_free(void* ov) {
  oc_opt* o = ov;
  if (!o) return;
  free(o->off);
  free(o->x);
  free(o->m);
  free(o->v);
  free(o->vf);
  free(o->mprev);
  free(o->c_avg);
  free(o->r_prev);
  free(o->coeff);
  free(o);
}

/* Elementwise maps, kernels.cpp:226-305 (each product/sum rounded to real). */
static void axpby(oc_real* y, double a, double b, const oc_real* x, uint64_t n) {
  const oc_real A = R(a), B = R(b);
  const uint64_t n_ = n;
  OC_PAR
  for (uint64_t i = 0; i < n; ++i) y[i] = A * y[i] + B * x[i];
}
static void axpby_square(oc_real* y, double a, double b, const oc_real* x, uint64_t n) {
  const oc_real A = R(a), B = R(b);
  const uint64_t n_ = n;
  OC_PAR
  for (uint64_t i = 0; i < n; ++i) y[i] = A * y[i] + B * x[i] * x[i];
}
static void linear_combine(oc_real* dst, double a, const oc_real* x, double b, const oc_real* y,
                           uint64_t n) {
  const oc_real A = R(a), B = R(b);
  const uint64_t n_ = n;
  OC_PAR
  for (uint64_t i = 0; i < n; ++i) dst[i] = A * x[i] + B * y[i];
}
static void precondition(oc_real* dst, const oc_real* m, const oc_real* v, double eta, uint64_t n) {
  const oc_real E = R(eta);
  const uint64_t n_ = n;
  OC_PAR
  for (uint64_t i = 0; i < n; ++i) {
#ifdef OC_REAL_FLOAT
    dst[i] = m[i] / (sqrtf(v[i]) + E);
#else
    dst[i] = m[i] / (sqrt(v[i]) + E);
#endif
  }
}
static void axpy(oc_real* y, double a, const oc_real* x, uint64_t n) {
  const oc_real A = R(a);
  const uint64_t n_ = n;
  OC_PAR
  for (uint64_t i = 0; i < n; ++i) y[i] += A * x[i];
}
static void scale_vec(oc_real* v, double a, uint64_t n) {
  const oc_real A = R(a);
  const uint64_t n_ = n;
  OC_PAR
  for (uint64_t i = 0; i < n; ++i) v[i] *= A;
}

static int is_two_stage(int v) { return v == V_ONEBIT_LAMB || v == V_BASIC || v == V_ONEBIT_ADAM; }

/* optimizers.cpp:140-177 lamb_step */
static void lamb_step(oc_opt* o, const oc_real* g, double lr, int track, double* tr) {
  const int L = o->L;
  const oc_hp* h = &o->hp;
  for (int l = 0; l < L; ++l) {
    const uint64_t a = o->off[l], n = o->off[l + 1] - a;
    oc_real *x = o->x + a, *m = o->m + a, *v = o->v + a;
    axpby(m, h->beta1, 1.0 - h->beta1, g + a, n);
    axpby_square(v, h->beta2, 1.0 - h->beta2, g + a, n);
    oc_real* u = scratch(S_U, (n + 1u) * sizeof(oc_real));
    precondition(u, m, v, h->eta, n);
    if (h->wd > 0.0) axpy(u, h->wd, x, n);
    const double xn = sqrt(canonical_sum(x, n, SUM_SQ));
    const double un = sqrt(canonical_sum(u, n, SUM_SQ));
    double c;
    if (un == 0.0) c = xn > 0.0 ? h->c_max : clip(1.0, h->c_min, h->c_max);
    else c = clip(xn / un, h->c_min, h->c_max);
    axpy(x, -lr * c, u, n);
    if (track) o->c_avg[l] = h->beta3 * o->c_avg[l] + (1.0 - h->beta3) * c;
    tr[l] = c;
    tr[L + l] = 1.0;
    tr[2 * L + l] = sqrt(canonical_sum(v, n, SUM_SQ));
    tr[3 * L + l] = 1.0;
  }
}

/* optimizers.cpp:179-200 adam_step */
static void adam_step(oc_opt* o, const oc_real* g, double lr, double* tr) {
  const int L = o->L;
  const oc_hp* h = &o->hp;
  for (int l = 0; l < L; ++l) {
    const uint64_t a = o->off[l], n = o->off[l + 1] - a;
    oc_real *x = o->x + a, *m = o->m + a, *v = o->v + a;
    axpby(m, h->beta1, 1.0 - h->beta1, g + a, n);
    axpby_square(v, h->beta2, 1.0 - h->beta2, g + a, n);
    oc_real* u = scratch(S_U, (n + 1u) * sizeof(oc_real));
    precondition(u, m, v, h->eta, n);
    if (h->wd > 0.0) axpy(u, h->wd, x, n);
    axpy(x, -lr, u, n);
    tr[l] = 1.0;
    tr[L + l] = 1.0;
    tr[2 * L + l] = sqrt(canonical_sum(v, n, SUM_SQ));
    tr[3 * L + l] = 1.0;
  }
}

/* optimizers.cpp:202-224 finalize_warmup; fusion.cpp:107-125 compute_scales */
static void finalize_warmup(oc_opt* o) {
  const int L = o->L;
  pcopy(o->vf, o->v, o->d * sizeof(oc_real));
  o->has_vf = 1;
  if (o->variant == V_ONEBIT_LAMB) {
    pcopy(o->mprev, o->m, o->d * sizeof(oc_real));
    o->has_mprev = 1;
  }
  if (o->variant == V_ONEBIT_ADAM) {
    for (int l = 0; l < L; ++l) o->coeff[l] = 1.0;
  } else {
    double* mag = malloc((size_t)L * sizeof(double));
    double ref = 0.0;
    for (int l = 0; l < L; ++l) {
      const uint64_t a = o->off[l], n = o->off[l + 1] - a;
      const double mean = canonical_sum(o->m + a, n, SUM_ABS) / (double)n; /* mean_abs */
      mag[l] = mean < o->hp.floor_ ? o->hp.floor_ : mean; /* std::max(mean, floor) */
      ref += mag[l];
    }
    ref /= (double)L;
    for (int l = 0; l < L; ++l) o->coeff[l] = ref / mag[l];
    free(mag);
  }
  double c_mean = 0.0;
  for (int l = 0; l < L; ++l) c_mean += o->variant == V_ONEBIT_ADAM ? 1.0 : o->c_avg[l];
  c_mean /= (double)L;
  const double cm = c_mean < o->hp.floor_ ? o->hp.floor_ : c_mean;
  o->c_mean_prev = o->c_mean_prev2 = cm;
  o->frozen = 1;
}

/* optimizers.cpp:231-332 compressed_step */
static int compressed_step(oc_opt* o, oc_cluster* c, const oc_real* grads, int n, double lr,
                           double* tr) {
  const int L = o->L;
  const oc_hp* h = &o->hp;
  const uint64_t d = o->d;
  if (!o->frozen)
    return fail(OC_STAGE_ORDER,
                "compression-stage step before warmup finalized: frozen variance, c_avg and "
                "momentum snapshot are missing");
  if (n != c->n)
    return fail(OC_DIMENSION, "compressed step: worker count: size mismatch (%d vs %d)", n, c->n);
  oc_real* streams = scratch(S_STREAMS, ((size_t)n * d + 1u) * sizeof(oc_real));
  for (int i = 0; i < n; ++i) { /* :248-255 */
    for (int l = 0; l < L; ++l) {
      const uint64_t a = o->off[l], len = o->off[l + 1] - a;
      const double co = o->coeff[l];
      linear_combine(streams + (size_t)i * d + a, co * h->beta1, o->m + a, co * (1.0 - h->beta1),
                     grads + (size_t)i * d + a, len);
    }
  }
  const double es = h->scaled_ef ? o->c_mean_prev2 / o->c_mean_prev : 1.0; /* :226-229 */
  oc_real* mg = scratch(S_MG, (d + 1u) * sizeof(oc_real));
  int st = cluster_compressed(c, streams, es, mg);
  if (st) return st;
  for (int l = 0; l < L; ++l) { /* fusion.cpp:139-145 remove_scaling */
    const uint64_t a = o->off[l];
    scale_vec(mg + a, 1.0 / o->coeff[l], o->off[l + 1] - a);
  }
  double c_sum = 0.0;
  for (int l = 0; l < L; ++l) {
    const uint64_t a = o->off[l], len = o->off[l + 1] - a;
    oc_real *x = o->x + a, *m = o->m + a, *v = o->v + a, *vf = o->vf + a, *mp = o->mprev + a;
    const oc_real* mgl = mg + a;
    double cc = 1.0, r = 1.0, pre = 1.0;
    if (o->variant == V_ONEBIT_LAMB) {
      if (!o->has_mprev) {
        return fail(OC_STAGE_ORDER, "compressed step: momentum snapshot missing");
      }
      oc_real* rec = scratch(S_REC, (len + 1u) * sizeof(oc_real));
      const double inv = 1.0 / (1.0 - h->beta1);
      linear_combine(rec, inv, mgl, -h->beta1 * inv, mp, len); /* :284-287 */
      if (!all_finite(rec, len)) {
        return fail(OC_RUNTIME, "non-finite reconstructed gradient for layer 'layer%d'", l);
      }
      axpby_square(v, h->beta2, 1.0 - h->beta2, rec, len); /* :294 */
      pre = max_abs_ratio(vf, v, len, h->floor_); /* :296 */
      r = clip(pre, (1.0 - h->r_thr) * o->r_prev[l], (1.0 + h->r_thr) * o->r_prev[l]);
      r = clip(r, h->r_min, h->r_max);
      cc = r * o->c_avg[l];
    } else if (o->variant == V_BASIC) {
      cc = o->c_avg[l];
    }
    if (!o->has_vf) {
      return fail(OC_STAGE_ORDER, "compressed step: frozen variance missing");
    }
    oc_real* u = scratch(S_U, (len + 1u) * sizeof(oc_real));
    precondition(u, mgl, vf, h->eta, len); /* :308-312 */
    if (h->wd > 0.0) axpy(u, h->wd, x, len);
    axpy(x, -lr * cc, u, len); /* :313 */
    if (o->variant == V_ONEBIT_LAMB) {
      pcopy(mp, mgl, len * sizeof(oc_real));
      o->r_prev[l] = r;
    }
    pcopy(m, mgl, len * sizeof(oc_real));
    c_sum += cc;
    tr[l] = cc;
    tr[L + l] = r;
    tr[2 * L + l] = sqrt(canonical_sum(v, len, SUM_SQ));
    tr[3 * L + l] = pre;
  }
  o->c_mean_prev2 = o->c_mean_prev;
  const double cm = c_sum / (double)L;
  o->c_mean_prev = cm < h->floor_ ? h->floor_ : cm;
  return OC_OK;
}

/* optimizers.cpp:334-364 Optimizer::step.  grads: n x d fused. */
int oc_opt_step(void* ov, void* cv, const oc_real* grads, int n, uint64_t t, double lr,
                double* tr, int* compressed) {
  oc_opt* o = ov;
  oc_cluster* c = cv;
  *compressed = 0;
  if (n < 1) return fail(OC_INVALID_ARGUMENT, "step: no worker gradients");
  for (int i = 0; i < n; ++i) { /* :99-117 check_gradients */
    for (int l = 0; l < o->L; ++l) {
      const uint64_t a = o->off[l];
      if (!all_finite(grads + (size_t)i * o->d + a, o->off[l + 1] - a))
        return fail(OC_RUNTIME, "non-finite gradient at step %llu, worker %d, layer 'layer%d'",
                    (unsigned long long)t, i, l);
    }
  }
  if (n != c->n) return fail(OC_DIMENSION, "step: worker count: size mismatch (%d vs %d)", n, c->n);
  if (c->dim != o->d)
    return fail(OC_DIMENSION, "compressed_allreduce: input length: size mismatch (%llu vs %llu)",
                (unsigned long long)o->d, (unsigned long long)c->dim);
  if (!is_two_stage(o->variant) || t < o->hp.warmup) {
    oc_real* avg = scratch(S_LAVG, (o->d + 1u) * sizeof(oc_real));
    oc_cluster_lossless_allreduce(c, grads, avg); /* :119-138 average_lossless */
    if (o->variant == V_ADAM || o->variant == V_ONEBIT_ADAM) adam_step(o, avg, lr, tr);
    else lamb_step(o, avg, lr, o->variant != V_LAMB, tr);
    if (is_two_stage(o->variant) && t + 1u == o->hp.warmup) finalize_warmup(o);
    return OC_OK;
  }
  int st = compressed_step(o, c, grads, n, lr, tr);
  if (st == OC_OK) *compressed = 1;
  return st;
}

void oc_opt_get(void* ov, int which, oc_real* out) {
  oc_opt* o = ov;
  const oc_real* src = which == 0 ? o->x : which == 1 ? o->m : which == 2 ? o->v
                     : which == 3 ? o->vf : o->mprev;
  pcopy(out, src, o->d * sizeof(oc_real));
}

void oc_opt_set(void* ov, int which, const oc_real* in) {
  oc_opt* o = ov;
  oc_real* dst = which == 0 ? o->x : which == 1 ? o->m : which == 2 ? o->v
               : which == 3 ? o->vf : o->mprev;
  pcopy(dst, in, o->d * sizeof(oc_real));
  if (which == 3) o->has_vf = 1;
  if (which == 4) o->has_mprev = 1;
}

void oc_opt_get_scalars(void* ov, double* out) {
  oc_opt* o = ov;
  const int L = o->L;
  for (int l = 0; l < L; ++l) {
    out[l] = o->c_avg[l];
    out[L + l] = o->r_prev[l];
    out[2 * L + l] = o->coeff[l];
  }
}

void oc_opt_set_scalars(void* ov, const double* in) {
  oc_opt* o = ov;
  for (int l = 0; l < o->L; ++l) {
    o->c_avg[l] = in[l];
    o->r_prev[l] = in[o->L + l];
  }
}

int oc_opt_frozen(void* o) { return ((oc_opt*)o)->frozen; }
