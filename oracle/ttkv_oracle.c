/*
 * ttkv_oracle.c -- CPU restatement of the TTKV decode hot path (plain C).
 * TEST INFRASTRUCTURE ONLY (see ttkv_oracle.h).  Compile with
 * -ffp-contract=off: the reference's fp64 sums must not be FMA-contracted.
 */
#include "ttkv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Sizes and accounting                                                      */
/* ------------------------------------------------------------------------ */

/* tier_store.cpp:36-44 (fast_capacity) */
size_t tko_fast_capacity(size_t budget, size_t d_kv, size_t bytes_fp, size_t block_size) {
  if (d_kv == 0 || bytes_fp == 0 || block_size == 0) return 0;
  size_t tokens = budget / (d_kv * bytes_fp);
  tokens -= tokens % block_size;
  if (tokens < block_size) return 0;
  return tokens;
}

/* quantizer.cpp:12-15 */
size_t tko_packed_bytes(size_t count, unsigned bits) {
  if (bits == 16) return count * sizeof(float);
  return (count * bits + 7) / 8;
}

/* quantizer.cpp:17-20 */
static size_t modeled_bytes(size_t count, unsigned bits) {
  if (bits == 16) return count * 2;
  return (count * bits + 7) / 8;
}

/* quantizer.cpp:172-180 (== QuantizedBlock::modeled_payload_bytes 117-124 for
 * a full block) */
size_t tko_modeled_block_bytes(size_t block_size, size_t d_k, size_t d_v,
                               unsigned key_bits, unsigned value_bits) {
  size_t bytes = modeled_bytes(block_size * d_k, key_bits) +
                 modeled_bytes(block_size * d_v, value_bits);
  if (key_bits != 16) bytes += 4 * d_k;
  if (value_bits != 16) bytes += 4 * d_v;
  return bytes;
}

/* ------------------------------------------------------------------------ */
/* Quantizer                                                                 */
/* ------------------------------------------------------------------------ */

/* quantizer.cpp:22-32 (pack_codes): LSB-first over the flat row-major index */
static void pack_codes(const uint16_t* codes, size_t count, unsigned bits, uint8_t* out) {
  memset(out, 0, tko_packed_bytes(count, bits));
  size_t bitpos = 0;
  for (size_t i = 0; i < count; ++i) {
    for (unsigned b = 0; b < bits; ++b)
      if (codes[i] & (1u << b)) out[(bitpos + b) / 8] |= (uint8_t)(1u << ((bitpos + b) % 8));
    bitpos += bits;
  }
}

/* quantizer.cpp:34-47 (unpack_codes) */
static void unpack_codes(const uint8_t* in, size_t count, unsigned bits, uint16_t* codes) {
  size_t bitpos = 0;
  for (size_t i = 0; i < count; ++i) {
    uint16_t code = 0;
    for (unsigned b = 0; b < bits; ++b)
      if (in[(bitpos + b) / 8] & (1u << ((bitpos + b) % 8))) code |= (uint16_t)(1u << b);
    codes[i] = code;
    bitpos += bits;
  }
}

/* quantizer.cpp:51-88 (quantize_tensor).  std::min/std::max semantics:
 * min(a,b) = (b < a) ? b : a ; max(a,b) = (a < b) ? b : a. */
void tko_quantize_tensor(const float* data, size_t rows, size_t dim, unsigned bits,
                         float* params, uint8_t* packed) {
  if (bits == 16) {
    memcpy(packed, data, rows * dim * sizeof(float));
    return;
  }
  const double levels = (double)((1u << bits) - 1);
  uint16_t* codes = (uint16_t*)calloc(rows * dim ? rows * dim : 1, sizeof(uint16_t));
  for (size_t c = 0; c < dim; ++c) {
    float lo = INFINITY, hi = -INFINITY;
    for (size_t r = 0; r < rows; ++r) {
      const float x = data[r * dim + c];
      lo = (x < lo) ? x : lo;
      hi = (hi < x) ? x : hi;
    }
    if (hi == lo) {
      params[2 * c] = 1.0f;
      params[2 * c + 1] = lo;
      continue;
    }
    const float scale = (float)(((double)hi - (double)lo) / levels);
    params[2 * c] = scale;
    params[2 * c + 1] = lo;
    for (size_t r = 0; r < rows; ++r) {
      double q = round(((double)data[r * dim + c] - (double)lo) / (double)scale);
      /* std::clamp(q, 0.0, levels) */
      if (q < 0.0) q = 0.0;
      else if (levels < q) q = levels;
      codes[r * dim + c] = (uint16_t)q;
    }
  }
  pack_codes(codes, rows * dim, bits, packed);
  free(codes);
}

/* quantizer.cpp:90-113 (dequantize_tensor) */
void tko_dequantize_tensor(const uint8_t* packed, size_t rows, size_t dim,
                           unsigned bits, const float* params, float* out) {
  if (bits == 16) {
    memcpy(out, packed, rows * dim * sizeof(float));
    return;
  }
  uint16_t* codes = (uint16_t*)malloc((rows * dim ? rows * dim : 1) * sizeof(uint16_t));
  unpack_codes(packed, rows * dim, bits, codes);
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < dim; ++c)
      out[r * dim + c] = (float)((double)codes[r * dim + c] * (double)params[2 * c] +
                                 (double)params[2 * c + 1]);
  free(codes);
}

/* quantizer.cpp:141-148 */
void tko_centroid(const float* keys, size_t rows, size_t d_k, float* out) {
  for (size_t c = 0; c < d_k; ++c) {
    double sum = 0.0;
    for (size_t r = 0; r < rows; ++r) sum += (double)keys[r * d_k + c];
    out[c] = (float)(sum / (double)rows);
  }
}

/* ------------------------------------------------------------------------ */
/* Relevance                                                                 */
/* ------------------------------------------------------------------------ */

/* relevance.cpp:19-27 */
double tko_score_block(const float* q, const float* c, size_t d) {
  double s = 0.0;
  for (size_t i = 0; i < d; ++i) s += (double)q[i] * (double)c[i];
  return s;
}

/* relevance.cpp:10-17 */
size_t tko_resolve(int has_top_k, size_t top_k, double fraction, size_t n) {
  if (has_top_k) return top_k < n ? top_k : n;
  if (!(fraction > 0.0 && fraction <= 1.0)) return (size_t)-1;
  const size_t k = (size_t)ceil(fraction * (double)n);
  return k < n ? k : n;
}

typedef struct {
  uint64_t id;
  double score;
} block_score;

/* relevance.cpp:34-38 comparator: score desc, then block_id desc. */
static int cmp_block_score(const void* pa, const void* pb) {
  const block_score* a = (const block_score*)pa;
  const block_score* b = (const block_score*)pb;
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  if (a->id != b->id) return a->id > b->id ? -1 : 1;
  return 0;
}

/* relevance.cpp:29-43.  The comparator is a total order on distinct ids, so
 * qsort's instability cannot change the result of std::stable_sort. */
void tko_select_top_k(const double* scores, const uint64_t* ids, size_t n, size_t k,
                      uint64_t* out) {
  block_score* v = (block_score*)malloc((n ? n : 1) * sizeof(block_score));
  for (size_t i = 0; i < n; ++i) {
    v[i].id = ids ? ids[i] : i;
    v[i].score = scores[i];
  }
  qsort(v, n, sizeof(block_score), cmp_block_score);
  for (size_t i = 0; i < k && i < n; ++i) out[i] = v[i].id;
  free(v);
}

/* ------------------------------------------------------------------------ */
/* Serialization (quantizer.cpp:248-274)                                     */
/* ------------------------------------------------------------------------ */

static uint8_t* put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) *p++ = (uint8_t)((v >> (8 * i)) & 0xff);
  return p;
}
static uint8_t* put_f32(uint8_t* p, float f) {
  uint32_t v;
  memcpy(&v, &f, 4);
  return put_le(p, v, 4);
}

size_t tko_serialize_block(uint64_t block_id, uint64_t first_pos, uint64_t last_pos,
                           uint32_t token_count, uint32_t d_k, uint32_t d_v,
                           unsigned key_bits, unsigned value_bits,
                           const float* key_params, const float* value_params,
                           const float* centroid, const uint8_t* packed_k,
                           const uint8_t* packed_v, uint8_t* out) {
  const size_t nkp = key_bits == 16 ? 0 : d_k;
  const size_t nvp = value_bits == 16 ? 0 : d_v;
  const size_t kb = tko_packed_bytes((size_t)token_count * d_k, key_bits);
  const size_t vb = tko_packed_bytes((size_t)token_count * d_v, value_bits);
  const size_t total = 4 + 2 + 8 * 3 + 4 * 3 + 2 * 2 + 8 * (nkp + nvp) + 4 * d_k + 8 + kb + 8 + vb;
  if (!out) return total;
  uint8_t* p = out;
  *p++ = 'T'; *p++ = 'T'; *p++ = 'K'; *p++ = 'V';
  p = put_le(p, 1, 2);
  p = put_le(p, block_id, 8);
  p = put_le(p, first_pos, 8);
  p = put_le(p, last_pos, 8);
  p = put_le(p, token_count, 4);
  p = put_le(p, d_k, 4);
  p = put_le(p, d_v, 4);
  p = put_le(p, key_bits, 2);
  p = put_le(p, value_bits, 2);
  for (size_t c = 0; c < nkp; ++c) { p = put_f32(p, key_params[2 * c]); p = put_f32(p, key_params[2 * c + 1]); }
  for (size_t c = 0; c < nvp; ++c) { p = put_f32(p, value_params[2 * c]); p = put_f32(p, value_params[2 * c + 1]); }
  for (size_t c = 0; c < d_k; ++c) p = put_f32(p, centroid[c]);
  p = put_le(p, kb, 8);
  memcpy(p, packed_k, kb); p += kb;
  p = put_le(p, vb, 8);
  memcpy(p, packed_v, vb); p += vb;
  return (size_t)(p - out);
}

/* ------------------------------------------------------------------------ */
/* Engine (tier_store.cpp + engine.cpp)                                      */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t first_pos;
  uint8_t* packed_k;
  uint8_t* packed_v;
  float* k_params;
  float* v_params;
  float* centroid;
} slow_block;

struct tko_engine {
  tko_config cfg;
  /* fast tier: tokens [fast_first, next_pos), stored from index fast_off */
  float* fk;
  float* fv;
  size_t fcap, fast_off, fast_n;
  uint64_t next_pos;
  slow_block* slow;
  size_t n_slow, slow_cap;
};

tko_engine* tko_engine_create(const tko_config* cfg) {
  if (!cfg || cfg->d_k == 0 || cfg->d_v == 0 || cfg->block_size == 0 || cfg->l_fast < cfg->block_size)
    return NULL;
  tko_engine* e = (tko_engine*)calloc(1, sizeof(tko_engine));
  e->cfg = *cfg;
  e->fcap = 2 * (cfg->l_fast + cfg->block_size) + 8;
  e->fk = (float*)malloc(e->fcap * cfg->d_k * sizeof(float));
  e->fv = (float*)malloc(e->fcap * cfg->d_v * sizeof(float));
  return e;
}

void tko_engine_destroy(tko_engine* e) {
  if (!e) return;
  for (size_t i = 0; i < e->n_slow; ++i) {
    free(e->slow[i].packed_k); free(e->slow[i].packed_v);
    free(e->slow[i].k_params); free(e->slow[i].v_params); free(e->slow[i].centroid);
  }
  free(e->slow); free(e->fk); free(e->fv); free(e);
}

/* tier_store.cpp:49-67 (append_token; sequencing is implicit here) */
static void append_token(tko_engine* e, const float* key, const float* value) {
  const size_t dk = e->cfg.d_k, dv = e->cfg.d_v;
  if (e->fast_off + e->fast_n == e->fcap) { /* compact */
    memmove(e->fk, e->fk + e->fast_off * dk, e->fast_n * dk * sizeof(float));
    memmove(e->fv, e->fv + e->fast_off * dv, e->fast_n * dv * sizeof(float));
    e->fast_off = 0;
  }
  memcpy(e->fk + (e->fast_off + e->fast_n) * dk, key, dk * sizeof(float));
  memcpy(e->fv + (e->fast_off + e->fast_n) * dv, value, dv * sizeof(float));
  e->fast_n++;
  e->next_pos++;
}

/* tier_store.cpp:69 */
static int eviction_pending(const tko_engine* e) { return e->fast_n > e->cfg.l_fast; }

/* tier_store.cpp:71-98 + quantize_block quantizer.cpp:126-155 */
static void evict_and_compress(tko_engine* e) {
  const tko_config* c = &e->cfg;
  const size_t n = c->block_size, dk = c->d_k, dv = c->d_v;
  if (e->n_slow == e->slow_cap) {
    e->slow_cap = e->slow_cap ? 2 * e->slow_cap : 64;
    e->slow = (slow_block*)realloc(e->slow, e->slow_cap * sizeof(slow_block));
  }
  slow_block* b = &e->slow[e->n_slow];
  const float* keys = e->fk + e->fast_off * dk;
  const float* vals = e->fv + e->fast_off * dv;
  b->first_pos = e->next_pos - e->fast_n;
  b->centroid = (float*)malloc(dk * sizeof(float));
  tko_centroid(keys, n, dk, b->centroid);
  b->packed_k = (uint8_t*)malloc(tko_packed_bytes(n * dk, c->key_bits) + 1);
  b->packed_v = (uint8_t*)malloc(tko_packed_bytes(n * dv, c->value_bits) + 1);
  b->k_params = (float*)calloc(2 * dk, sizeof(float));
  b->v_params = (float*)calloc(2 * dv, sizeof(float));
  tko_quantize_tensor(keys, n, dk, c->key_bits, b->k_params, b->packed_k);
  tko_quantize_tensor(vals, n, dv, c->value_bits, b->v_params, b->packed_v);
  e->n_slow++;
  e->fast_off += n;
  e->fast_n -= n;
}

/* engine.cpp:15-20 */
int tko_engine_prefill(tko_engine* e, const float* keys, const float* values, size_t n) {
  for (size_t t = 0; t < n; ++t) {
    append_token(e, keys + t * e->cfg.d_k, values + t * e->cfg.d_v);
    while (eviction_pending(e)) evict_and_compress(e);
  }
  return 0;
}

/* attention.hpp:17-61, AttentionAccumulator<double> */
typedef struct {
  double scale, running_max, den;
  double* wv;
  size_t d_v, absorbed;
} accum;

static void acc_init(accum* a, size_t d_v, double scale) {
  a->scale = scale;
  a->running_max = -INFINITY;
  a->den = 0.0;
  a->wv = (double*)calloc(d_v, sizeof(double));
  a->d_v = d_v;
  a->absorbed = 0;
}

/* attention.hpp:29-50 */
static void acc_absorb(accum* a, const float* q, const float* keys, const float* values,
                       size_t rows, size_t d_k) {
  for (size_t r = 0; r < rows; ++r) {
    double s = 0.0;
    const float* k = keys + r * d_k;
    for (size_t i = 0; i < d_k; ++i) s += (double)q[i] * (double)k[i];
    s *= a->scale;
    if (s > a->running_max) {
      const double rescale = exp(a->running_max - s);
      a->den *= rescale;
      for (size_t i = 0; i < a->d_v; ++i) a->wv[i] *= rescale;
      a->running_max = s;
    }
    const double w = exp(s - a->running_max);
    a->den += w;
    const float* v = values + r * a->d_v;
    for (size_t i = 0; i < a->d_v; ++i) a->wv[i] += w * (double)v[i];
    a->absorbed++;
  }
}

int tko_engine_decode_step(tko_engine* e, const float* q, size_t G, int mode,
                           const float* key, const float* value, double* out,
                           uint64_t* fetched, size_t fetched_cap, size_t* n_fetched,
                           size_t* n_scored, double* bytes_modeled,
                           size_t* union_blocks, int* evicted) {
  const tko_config* c = &e->cfg;
  const size_t dk = c->d_k, dv = c->d_v, B = c->block_size;
  if (G == 0) return -1;
  const int smode = mode & 1;         /* selection: per-head / group-shared */
  const int literal = (mode >> 1) & 1; /* EngineOptions::literal_additive_merge */
  append_token(e, key, value); /* engine.cpp:28 */
  const double scale = 1.0 / sqrt((double)dk); /* engine.cpp:30 */
  const size_t n = e->n_slow;
  const size_t k = tko_resolve(c->has_top_k, c->top_k, c->fetch_fraction, n);
  if (k == (size_t)-1) return -2;
  if (n_scored) *n_scored = n;

  double* scores = (double*)malloc((n ? n : 1) * sizeof(double));
  uint64_t* sel = (uint64_t*)malloc((k ? k : 1) * sizeof(uint64_t));
  float* dk_buf = (float*)malloc(B * dk * sizeof(float));
  float* dv_buf = (float*)malloc(B * dv * sizeof(float));
  uint8_t* in_union = (uint8_t*)calloc(n ? n : 1, 1);
  float* qshared = (float*)calloc(dk, sizeof(float));
  if (smode == 1)
    for (size_t g = 0; g < G; ++g)
      for (size_t i = 0; i < dk; ++i) qshared[i] += q[g * dk + i];

  double bytes = 0.0;
  const size_t blk_bytes = tko_modeled_block_bytes(B, dk, dv, c->key_bits, c->value_bits);
  for (size_t g = 0; g < G; ++g) {
    const float* qg = q + g * dk;
    accum acc;
    acc_init(&acc, dv, scale);
    /* engine.cpp:36-40: fast tier including the new token */
    for (size_t t = 0; t < e->fast_n; ++t)
      acc_absorb(&acc, qg, e->fk + (e->fast_off + t) * dk, e->fv + (e->fast_off + t) * dv, 1, dk);
    /* engine.cpp:44-48: literal additive merge keeps the fast partition's
     * normalized output and sums every block's normalized output onto it */
    double* lit = NULL;
    if (literal) {
      lit = (double*)calloc(dv, sizeof(double));
      for (size_t i = 0; i < dv; ++i) lit[i] = acc.wv[i] / acc.den;
    }
    /* engine.cpp:51-58 */
    const float* qs = (smode == 1) ? qshared : qg;
    for (size_t b = 0; b < n; ++b) scores[b] = tko_score_block(qs, e->slow[b].centroid, dk);
    tko_select_top_k(scores, NULL, n, k, sel);
    /* engine.cpp:61-83 */
    for (size_t i = 0; i < k; ++i) {
      const slow_block* b = &e->slow[sel[i]];
      in_union[sel[i]] = 1;
      bytes += (double)blk_bytes;
      tko_dequantize_tensor(b->packed_k, B, dk, c->key_bits, b->k_params, dk_buf);
      tko_dequantize_tensor(b->packed_v, B, dv, c->value_bits, b->v_params, dv_buf);
      if (literal) { /* engine.cpp:67-72 */
        accum part;
        acc_init(&part, dv, scale);
        acc_absorb(&part, qg, dk_buf, dv_buf, B, dk);
        for (size_t j = 0; j < dv; ++j) lit[j] += part.wv[j] / part.den;
        free(part.wv);
      } else {
        acc_absorb(&acc, qg, dk_buf, dv_buf, B, dk);
      }
    }
    /* attention.hpp:54-61 */
    for (size_t i = 0; i < dv; ++i) out[g * dv + i] = literal ? lit[i] : acc.wv[i] / acc.den;
    free(acc.wv);
    free(lit);
    if (fetched)
      for (size_t i = 0; i < k && i < fetched_cap; ++i) fetched[g * fetched_cap + i] = sel[i];
    if (n_fetched) n_fetched[g] = k;
  }
  if (bytes_modeled) *bytes_modeled = bytes / (double)G; /* per head, as one Engine reports */
  if (union_blocks) {
    size_t u = 0;
    for (size_t b = 0; b < n; ++b) u += in_union[b];
    *union_blocks = u;
  }
  int ev = 0;
  while (eviction_pending(e)) { /* engine.cpp:88-91 */
    evict_and_compress(e);
    ev = 1;
  }
  if (evicted) *evicted = ev;
  free(scores); free(sel); free(dk_buf); free(dv_buf); free(in_union); free(qshared);
  return 0;
}

size_t tko_engine_slow_blocks(const tko_engine* e) { return e->n_slow; }
size_t tko_engine_fast_tokens(const tko_engine* e) { return e->fast_n; }
size_t tko_engine_appended(const tko_engine* e) { return (size_t)e->next_pos; }
const float* tko_engine_centroid(const tko_engine* e, size_t i) {
  return i < e->n_slow ? e->slow[i].centroid : NULL;
}

size_t tko_engine_serialize_block(const tko_engine* e, size_t i, uint8_t* out) {
  if (i >= e->n_slow) return 0;
  const slow_block* b = &e->slow[i];
  const tko_config* c = &e->cfg;
  return tko_serialize_block(i, b->first_pos, b->first_pos + c->block_size - 1,
                             (uint32_t)c->block_size, (uint32_t)c->d_k, (uint32_t)c->d_v,
                             c->key_bits, c->value_bits, b->k_params, b->v_params,
                             b->centroid, b->packed_k, b->packed_v, out);
}

/* ------------------------------------------------------------------------ */
/* Dense oracle (reference.cpp:12-51)                                        */
/* ------------------------------------------------------------------------ */

int tko_dense_attention(const float* q, size_t d_k, const float* keys,
                        const float* values, size_t rows, size_t d_v, double* out) {
  if (rows == 0) return -1;
  const double scale = 1.0 / sqrt((double)d_k);
  double* logits = (double*)malloc(rows * sizeof(double));
  double mx = -INFINITY;
  for (size_t r = 0; r < rows; ++r) {
    double s = 0.0;
    for (size_t j = 0; j < d_k; ++j) s += (double)q[j] * (double)keys[r * d_k + j];
    logits[r] = s * scale;
    mx = (mx < logits[r]) ? logits[r] : mx;
  }
  for (size_t j = 0; j < d_v; ++j) out[j] = 0.0;
  double den = 0.0;
  for (size_t r = 0; r < rows; ++r) {
    const double w = exp(logits[r] - mx);
    den += w;
    for (size_t j = 0; j < d_v; ++j) out[j] += w * (double)values[r * d_v + j];
  }
  for (size_t j = 0; j < d_v; ++j) out[j] /= den;
  free(logits);
  return 0;
}

double tko_relative_error(const double* a, const double* b, size_t n) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < n; ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return den > 0 ? sqrt(num / den) : sqrt(num);
}

/* ------------------------------------------------------------------------ */
/* Workload generator (workload.cpp:12-95)                                   */
/* ------------------------------------------------------------------------ */

/* std::mt19937_64 (the standard's parameters) */
void tko_gauss_seed(tko_gauss* g, uint64_t seed) {
  g->mt[0] = seed;
  for (size_t i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + i;
  g->idx = 312;
  g->has_spare = 0;
  g->spare = 0.0;
}

uint64_t tko_mt_next(tko_gauss* g) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  static const uint64_t A = 0xB5026F5AA96619E9ULL;
  if (g->idx >= 312) {
    for (size_t i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      g->mt[i] = g->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* workload.cpp:12-26 */
double tko_gauss_next(tko_gauss* g) {
  if (g->has_spare) {
    g->has_spare = 0;
    return g->spare;
  }
  const double inv = 0x1.0p-53;
  const double u1 = ((double)(tko_mt_next(g) >> 11) + 1.0) * inv;
  const double u2 = (double)(tko_mt_next(g) >> 11) * inv;
  const double r = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.141592653589793 * u2;
  g->spare = r * sin(theta);
  g->has_spare = 1;
  return r * cos(theta);
}

/* workload.cpp:42-95 */
int tko_generate_workload(int needle, size_t ctx, size_t T, size_t d_k, size_t d_v,
                          uint64_t seed, size_t needle_block_position,
                          double needle_strength, float* pre_k, float* pre_v,
                          float* dec_k, float* dec_v, float* dec_q, float* needle_dir) {
  const size_t span = 128; /* kNeedleSpanTokens, workload.hpp:10 */
  if (ctx < 1 || d_k == 0 || d_v == 0) return -1;
  if (needle && (needle_block_position * span + span > ctx || needle_strength <= 0)) return -1;
  tko_gauss g;
  tko_gauss_seed(&g, seed);
  float* u = (float*)malloc(d_k * sizeof(float));
  const float uval = 1.0f / sqrtf((float)d_k);
  for (size_t i = 0; i < d_k; ++i) u[i] = uval;
  if (needle && needle_dir) memcpy(needle_dir, u, d_k * sizeof(float));
  const size_t nf = needle_block_position * span, nl = nf + span;
  const double mean_mag = needle_strength / sqrt((double)span);
  for (size_t p = 0; p < ctx + T; ++p) {
    float* kk = p < ctx ? pre_k + p * d_k : dec_k + (p - ctx) * d_k;
    float* vv = p < ctx ? pre_v + p * d_v : dec_v + (p - ctx) * d_v;
    const int in_needle = needle && p >= nf && p < nl;
    for (size_t i = 0; i < d_k; ++i) {
      double x = tko_gauss_next(&g);
      if (in_needle) x += mean_mag * (double)u[i];
      kk[i] = (float)x;
    }
    for (size_t i = 0; i < d_v; ++i) vv[i] = (float)tko_gauss_next(&g);
    if (p >= ctx) {
      float* qq = dec_q + (p - ctx) * d_k;
      if (needle) memcpy(qq, u, d_k * sizeof(float));
      else
        for (size_t i = 0; i < d_k; ++i) qq[i] = (float)tko_gauss_next(&g);
    }
  }
  free(u);
  return 0;
}
