/*
 * kvref — CPU restatement of the bytes the DualPath KV loading path moves.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the CPU baseline; the product path never calls it.
 *
 * The reference carries byte counts only ("No tensor contents; blocks carry
 * sizes only"), so the contents are a builder extension pinned
 * here and checked bit-for-bit against the GPU path:
 *
 *   - Full Block layout [L][T][b]: L Layer Blocks concatenated
 *     (ClusterConfig::layer_block_bytes / full_block_bytes,
 *     proj/include/pdsim/types.hpp:33-39);
 *   - content word(p, w) = splitmix64((p << 32 | w) ^ seed * 0xD1B54A32D192ED03)
 *     for Full Block p of the store and 8-byte word w;
 *   - per-layer hit transfer of a request = tokens [0, C) of Layer Block l of
 *     each of its ceil(C/T) Full Blocks (start_hit_transfer moves kvb_layer(C)
 *     = C*b bytes per layer, proj/src/desim.cpp:569-571, :612-621;
 *     blocks_for, proj/src/types.cpp:55-60), into pool[l][slot][T][b];
 *   - Layer Block hash H = sum_i splitmix64(word_i + (i+1) * golden) mod 2^64.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ull
#define SEED_MUL 0xD1B54A32D192ED03ull

typedef struct kv_geom {
  int32_t n_layer;
  int32_t block_tokens;
  int64_t bytes_per_token_layer;
} kv_geom;

/* same field order/meaning as dp_job in include/dualpath/kv_abi.h */
typedef struct kv_job {
  const int64_t* src_fb;
  const int32_t* dst_slot;
  int64_t n_tokens;
  int32_t n_blk;
  int32_t layer_begin;
  int32_t layer_end;
  int32_t ticket;
} kv_job;

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline int64_t lb_bytes(const kv_geom* g) {
  return (int64_t)g->block_tokens * g->bytes_per_token_layer;
}
static inline int64_t fb_bytes(const kv_geom* g) { return lb_bytes(g) * g->n_layer; }

uint64_t kvref_splitmix64(uint64_t x) { return splitmix64(x); }

uint64_t kvref_word(uint64_t seed, int64_t fb, int64_t w) {
  return splitmix64((((uint64_t)fb) << 32 | (uint64_t)w) ^ (seed * SEED_MUL));
}

/* Fill Full Blocks [fb0, fb0 + n) of a store image (n * FB bytes at out). */
void kvref_fill_store(const kv_geom* g, uint64_t seed, int64_t fb0, int64_t n, uint8_t* out) {
  const int64_t words = fb_bytes(g) / 8;
  uint64_t* o = (uint64_t*)out;
  for (int64_t p = 0; p < n; ++p)
    for (int64_t w = 0; w < words; ++w) o[p * words + w] = kvref_word(seed, fb0 + p, w);
}

/* Expected bytes of Layer Block `layer` of Full Block `fb` (first ntok tokens). */
void kvref_layer_block(const kv_geom* g, uint64_t seed, int64_t fb, int32_t layer, int64_t ntok,
                       uint8_t* out) {
  const int64_t w0 = (int64_t)layer * lb_bytes(g) / 8;
  const int64_t nw = ntok * g->bytes_per_token_layer / 8;
  uint64_t* o = (uint64_t*)out;
  for (int64_t i = 0; i < nw; ++i) o[i] = kvref_word(seed, fb, w0 + i);
}

/* H of a byte range (n_words words). */
uint64_t kvref_hash_words(const uint64_t* words, int64_t n_words) {
  uint64_t h = 0;
  for (int64_t i = 0; i < n_words; ++i) h += splitmix64(words[i] + (uint64_t)(i + 1) * GOLDEN);
  return h;
}

/* H of the expected Layer Block, generated from the content formula alone. */
uint64_t kvref_layer_block_hash(const kv_geom* g, uint64_t seed, int64_t fb, int32_t layer,
                                int64_t ntok) {
  const int64_t w0 = (int64_t)layer * lb_bytes(g) / 8;
  const int64_t nw = ntok * g->bytes_per_token_layer / 8;
  uint64_t h = 0;
  for (int64_t i = 0; i < nw; ++i)
    h += splitmix64(kvref_word(seed, fb, w0 + i) + (uint64_t)(i + 1) * GOLDEN);
  return h;
}

/* Prefill stand-in digest (K5, dp_prefill_attend in include/dualpath/kv_abi.h):
 *   sum_{q in [q_begin, q_begin + bsz)} sum_{t < cached} sum_i Q[q][i] * K[t][i]   (mod 2^64)
 * over unsigned bytes i < b, K[t] = token t of Layer Block `layer` of Full
 * Block fb[t / T], Q[q] the procedural query bytes.  Restated as the inner
 * product of the per-lane column sums (exact: the same integer mod 2^64),
 * so the check costs (bsz + cached) * b instead of bsz * cached * b. */
#define QUERY_MUL 0xA24BAED4963EE407ull
uint64_t kvref_query_word(uint64_t seed, uint32_t req, int32_t layer, int64_t q, int64_t w) {
  const uint64_t base = splitmix64((((uint64_t)req << 20) | (uint64_t)layer) ^ (seed * QUERY_MUL));
  return splitmix64(base ^ (((uint64_t)q << 16) | (uint64_t)w));
}

uint64_t kvref_attend_digest(const kv_geom* g, uint64_t seed, const int64_t* fb, int64_t cached,
                             uint32_t req, int32_t layer, int64_t q_begin, int64_t bsz) {
  const int64_t b = g->bytes_per_token_layer;
  uint64_t* kcol = (uint64_t*)calloc((size_t)b, sizeof(uint64_t));
  uint64_t* qcol = (uint64_t*)calloc((size_t)b, sizeof(uint64_t));
  if (!kcol || !qcol) {
    free(kcol);
    free(qcol);
    return 0;
  }
  const int64_t lw0 = (int64_t)layer * lb_bytes(g) / 8;
  for (int64_t t = 0; t < cached; ++t) {
    const int64_t blk = t / g->block_tokens, within = t % g->block_tokens;
    for (int64_t w = 0; w < b / 8; ++w) {
      const uint64_t word = kvref_word(seed, fb[blk], lw0 + within * (b / 8) + w);
      for (int k = 0; k < 8; ++k) kcol[8 * w + k] += (word >> (8 * k)) & 0xff;
    }
  }
  for (int64_t q = q_begin; q < q_begin + bsz; ++q)
    for (int64_t w = 0; w < b / 8; ++w) {
      const uint64_t word = kvref_query_word(seed, req, layer, q, w);
      for (int k = 0; k < 8; ++k) qcol[8 * w + k] += (word >> (8 * k)) & 0xff;
    }
  uint64_t d = 0;
  for (int64_t i = 0; i < b; ++i) d += qcol[i] * kcol[i];
  free(kcol);
  free(qcol);
  return d;
}

/* Restated hit transfer: move each job's Layer Blocks from a store image
 * into a pool image [n_layer][n_slots][T][b] with memcpy (serial). */
int kvref_gather(const kv_geom* g, const uint8_t* store, int64_t store_fb, const kv_job* jobs,
                 int32_t n_jobs, uint8_t* pool, int32_t n_slots) {
  const int64_t lb = lb_bytes(g), fb = fb_bytes(g);
  for (int32_t j = 0; j < n_jobs; ++j) {
    const kv_job* job = &jobs[j];
    for (int32_t l = job->layer_begin; l < job->layer_end; ++l)
      for (int32_t k = 0; k < job->n_blk; ++k) {
        int64_t ntok = job->n_tokens - (int64_t)k * g->block_tokens;
        if (ntok > g->block_tokens) ntok = g->block_tokens;
        if (ntok <= 0) continue;
        const int64_t f = job->src_fb[k];
        const int32_t s = job->dst_slot[k];
        if (f < 0 || f >= store_fb || s < 0 || s >= n_slots) return -1;
        memcpy(pool + ((int64_t)l * n_slots + s) * lb, store + f * fb + (int64_t)l * lb,
               (size_t)(ntok * g->bytes_per_token_layer));
      }
  }
  return 0;
}

/* Multi-threaded CPU gather (the CPU baseline of the same byte movement):
 * Layer Blocks of all jobs are split round-robin over `threads` workers. */
typedef struct gather_arg {
  const kv_geom* g;
  const uint8_t* store;
  const kv_job* jobs;
  int32_t n_jobs;
  uint8_t* pool;
  int32_t n_slots;
  int tid, nthreads;
  int64_t bytes;
} gather_arg;

static void* gather_worker(void* p) {
  gather_arg* a = (gather_arg*)p;
  const int64_t lb = lb_bytes(a->g), fbb = fb_bytes(a->g);
  int64_t idx = 0;
  for (int32_t j = 0; j < a->n_jobs; ++j) {
    const kv_job* job = &a->jobs[j];
    for (int32_t l = job->layer_begin; l < job->layer_end; ++l)
      for (int32_t k = 0; k < job->n_blk; ++k, ++idx) {
        if (idx % a->nthreads != a->tid) continue;
        int64_t ntok = job->n_tokens - (int64_t)k * a->g->block_tokens;
        if (ntok > a->g->block_tokens) ntok = a->g->block_tokens;
        if (ntok <= 0) continue;
        const size_t n = (size_t)(ntok * a->g->bytes_per_token_layer);
        memcpy(a->pool + ((int64_t)l * a->n_slots + job->dst_slot[k]) * lb,
               a->store + job->src_fb[k] * fbb + (int64_t)l * lb, n);
        a->bytes += (int64_t)n;
      }
  }
  return NULL;
}

int64_t kvref_gather_mt(const kv_geom* g, const uint8_t* store, const kv_job* jobs, int32_t n_jobs,
                        uint8_t* pool, int32_t n_slots, int threads) {
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  gather_arg* args = (gather_arg*)calloc((size_t)threads, sizeof(gather_arg));
  for (int t = 0; t < threads; ++t) {
    gather_arg a = {g, store, jobs, n_jobs, pool, n_slots, t, threads, 0};
    args[t] = a;
    pthread_create(&th[t], NULL, gather_worker, &args[t]);
  }
  int64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    total += args[t].bytes;
  }
  free(th);
  free(args);
  return total;
}
