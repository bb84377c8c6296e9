/*
 * ttkv_oracle.h -- CPU restatement of the TTKV decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the checker.
 * The product path (paper_2604_19769_b200/) never links or calls it.
 *
 * Every function restates one reference function; the citation is given as
 * /root/reference/proj/<path>:<lines>.  The restatement is pinned by
 *   (1) the reference's own golden vectors (tests/test_oracle_golden.py), and
 *   (2) the unmodified reference compiled into oracle/_ref/ (oracle/Makefile),
 *       compared byte-for-byte / bit-for-bit in tests/test_oracle_vs_ref.py,
 *   (3) fixtures generated from oracle/_ref under tests/golden/.
 *
 * Build flags must keep IEEE semantics: -O2 -ffp-contract=off (no FMA
 * contraction).
 */
#ifndef TTKV_ORACLE_H
#define TTKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  size_t d_k, d_v;
  size_t block_size;
  size_t l_fast;          /* fast-tier capacity in tokens (tko_fast_capacity) */
  unsigned key_bits, value_bits;
  int has_top_k;
  size_t top_k;
  double fetch_fraction;
} tko_config;

/* tier_store.cpp:36-44.  Returns 0 when the budget holds < one block. */
size_t tko_fast_capacity(size_t budget, size_t d_kv, size_t bytes_fp, size_t block_size);

/* quantizer.cpp:12-15 (actual stored bytes; 16-bit = raw float32). */
size_t tko_packed_bytes(size_t count, unsigned bits);
/* quantizer.cpp:17-20, 172-180: modeled bytes of one block. */
size_t tko_modeled_block_bytes(size_t block_size, size_t d_k, size_t d_v,
                               unsigned key_bits, unsigned value_bits);

/* quantizer.cpp:51-88 (+ pack_codes 22-32).  params = {scale, zp} x dim,
 * nothing written for bits == 16 (payload = raw float32 bytes). */
void tko_quantize_tensor(const float* data, size_t rows, size_t dim, unsigned bits,
                         float* params, uint8_t* packed);
/* quantizer.cpp:90-113 (+ unpack_codes 34-47). */
void tko_dequantize_tensor(const uint8_t* packed, size_t rows, size_t dim,
                           unsigned bits, const float* params, float* out);
/* quantizer.cpp:141-148: pre-quantization key mean. */
void tko_centroid(const float* keys, size_t rows, size_t d_k, float* out);

/* relevance.cpp:19-27 */
double tko_score_block(const float* q, const float* c, size_t d);
/* relevance.cpp:10-17.  Returns (size_t)-1 on ConfigError. */
size_t tko_resolve(int has_top_k, size_t top_k, double fraction, size_t n);
/* relevance.cpp:29-43: ids[i] = block ids, order (score desc, id desc). */
void tko_select_top_k(const double* scores, const uint64_t* ids, size_t n,
                      size_t k, uint64_t* out);

/* Serialized block (quantizer.cpp:248-274) -- returns bytes written, or the
 * required size when out == NULL. */
size_t tko_serialize_block(uint64_t block_id, uint64_t first_pos, uint64_t last_pos,
                           uint32_t token_count, uint32_t d_k, uint32_t d_v,
                           unsigned key_bits, unsigned value_bits,
                           const float* key_params, const float* value_params,
                           const float* centroid, const uint8_t* packed_k,
                           const uint8_t* packed_v, uint8_t* out);

/* ---- Engine: a stream of KV shared by G query heads -------------------- */
typedef struct tko_engine tko_engine;

/* Returns NULL if the config is invalid. */
tko_engine* tko_engine_create(const tko_config* cfg);
void tko_engine_destroy(tko_engine* e);

/* engine.cpp:15-20 */
int tko_engine_prefill(tko_engine* e, const float* keys, const float* values, size_t n);

/* engine.cpp:22-93 generalised to G query heads on one KV stream.
 *   mode 0 (per-head): head g == one reference Engine fed q_g.
 *   mode 1 (group-shared): selection scored with q' = sum_g q_g (float,
 *          sequential g), every head attends that set.
 *   mode | 2: EngineOptions::literal_additive_merge (engine.cpp:44-48, 67-72).
 * out: G x d_v doubles.  fetched: G x cap ids (schedule order), n_fetched[G].
 * Returns 0, or a negative code on shape/config errors. */
int tko_engine_decode_step(tko_engine* e, const float* q, size_t G, int mode,
                           const float* key, const float* value, double* out,
                           uint64_t* fetched, size_t fetched_cap, size_t* n_fetched,
                           size_t* n_scored, double* bytes_modeled,
                           size_t* union_blocks, int* evicted);

size_t tko_engine_slow_blocks(const tko_engine* e);
size_t tko_engine_fast_tokens(const tko_engine* e);
size_t tko_engine_appended(const tko_engine* e);
/* Serialized bytes of slow block i (reference format). */
size_t tko_engine_serialize_block(const tko_engine* e, size_t i, uint8_t* out);
const float* tko_engine_centroid(const tko_engine* e, size_t i);

/* ---- Dense oracle (reference.cpp:12-51) ---------------------------------- */
int tko_dense_attention(const float* q, size_t d_k, const float* keys,
                        const float* values, size_t rows, size_t d_v, double* out);
double tko_relative_error(const double* a, const double* b, size_t n);

/* ---- Workload generator (workload.cpp:12-95; mt19937_64 + Box-Muller) ---- */
typedef struct {
  uint64_t mt[312];
  size_t idx;
  double spare;
  int has_spare;
} tko_gauss;
void tko_gauss_seed(tko_gauss* g, uint64_t seed);
uint64_t tko_mt_next(tko_gauss* g);
double tko_gauss_next(tko_gauss* g);

/* generate_workload (Gaussian or planted-needle).  Arrays are caller-owned:
 * pre_k [ctx x d_k], pre_v [ctx x d_v], dec_k [T x d_k], dec_v [T x d_v],
 * dec_q [T x d_k], needle_dir [d_k] (needle only; may be NULL). */
int tko_generate_workload(int needle, size_t ctx, size_t T, size_t d_k, size_t d_v,
                          uint64_t seed, size_t needle_block_position,
                          double needle_strength, float* pre_k, float* pre_v,
                          float* dec_k, float* dec_v, float* dec_q, float* needle_dir);

#ifdef __cplusplus
}
#endif
#endif
