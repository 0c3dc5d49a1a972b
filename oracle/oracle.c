/*
 * oracle.c — plain, slow, obviously-correct CPU oracle (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs, never by the product path.
 * Shares no code with paper_2105_07829_b200/csrc.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (no -ffast-math,
 * no FMA contraction) so every float operation below is one IEEE-754
 * binary32/binary64 operation, rounded to nearest-even, in source order.
 *
 * Parity status: every function here is pinned by
 * tests/test_oracle_*.py; none is "parity unpinned".
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3"). Reading R13: the counter-based generator the
 * dithering and random-k compressors draw from.
 * Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt). */
static void mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; round++) {
    if (round > 0) {            /* key schedule: Weyl sequence bump */
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
    mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R13: element j of chunk c at step t draws word (j mod 4) of
 * Philox(ctr = (floor(j/4), c, t, stage<<31 | rank), key = (lo32(seed), hi32(seed))).
 * stage 0 = worker push (rank = worker i), stage 1 = server pull (rank 0). */
uint32_t orc_rng_word(uint64_t seed, uint64_t j, uint32_t chunk, uint32_t t,
                      uint32_t stage, uint32_t rank) {
  uint32_t ctr[4] = {(uint32_t)(j / 4), chunk, t, (stage << 31) | rank};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  orc_philox4x32_10(ctr, key, out);
  return out[j % 4];
}

/* ------------------------------------------------------------------------ */
/* Reading R6 (norm reduction order; the paper is silent): pairwise summation
 * in fp64 — S(lo, len) = len == 1 ? a[lo] : S(lo, len/2) + S(lo + len/2, len/2)
 * over the input padded with +0 to the next power of two. */
static double pairwise(const double* a, uint64_t n, uint64_t lo, uint64_t len) {
  if (len == 1) return lo < n ? a[lo] : 0.0;
  return pairwise(a, n, lo, len / 2) + pairwise(a, n, lo + len / 2, len / 2);
}

double orc_pairwise_sum(const double* a, uint64_t n) {
  uint64_t P = 1;
  while (P < n) P <<= 1;
  return pairwise(a, n, 0, P);
}

/* ||x||_1 in fp64 ("||v||_1"), R6 order. */
static double l1_norm(const float* x, uint64_t L) {
  double* a = (double*)malloc(sizeof(double) * (L ? L : 1));
  for (uint64_t j = 0; j < L; j++) a[j] = (double)fabsf(x[j]);
  double s = orc_pairwise_sum(a, L);
  free(a);
  return s;
}

/* ||x||_2 rounded to fp32 (R12: the dithering norm). The squares of fp32
 * values are exact in fp64. */
static float l2_norm_f32(const float* x, uint64_t L) {
  double* a = (double*)malloc(sizeof(double) * (L ? L : 1));
  for (uint64_t j = 0; j < L; j++) a[j] = (double)x[j] * (double)x[j];
  double s = orc_pairwise_sum(a, L);
  free(a);
  return (float)sqrt(s);
}

/* ------------------------------------------------------------------------ */
/* little-endian byte helpers ("all integers little-endian") */
static void put_u32(uint8_t* p, uint32_t v) { for (int b = 0; b < 4; b++) p[b] = (uint8_t)(v >> (8 * b)); }
static void put_u64(uint8_t* p, uint64_t v) { for (int b = 0; b < 8; b++) p[b] = (uint8_t)(v >> (8 * b)); }
static uint32_t get_u32(const uint8_t* p) { uint32_t v = 0; for (int b = 0; b < 4; b++) v |= (uint32_t)p[b] << (8 * b); return v; }
static uint64_t get_u64(const uint8_t* p) { uint64_t v = 0; for (int b = 0; b < 8; b++) v |= (uint64_t)p[b] << (8 * b); return v; }
static void put_f32(uint8_t* p, float f) { uint32_t u; memcpy(&u, &f, 4); put_u32(p, u); }
static float get_f32(const uint8_t* p) { uint32_t u = get_u32(p); float f; memcpy(&f, &u, 4); return f; }
/* bit field of `nbits` bits at bit offset `pos`, LSB-first */
static void put_bits(uint8_t* base, uint64_t pos, uint32_t nbits, uint32_t v) {
  for (uint32_t b = 0; b < nbits; b++) {
    uint64_t q = pos + b;
    if ((v >> b) & 1u) base[q >> 3] |= (uint8_t)(1u << (q & 7));
  }
}
static uint32_t get_bits(const uint8_t* base, uint64_t pos, uint32_t nbits) {
  uint32_t v = 0;
  for (uint32_t b = 0; b < nbits; b++) {
    uint64_t q = pos + b;
    v |= (uint32_t)((base[q >> 3] >> (q & 7)) & 1u) << b;
  }
  return v;
}

/* ------------------------------------------------------------------------ */
/* R8: fractional k -> k = max(1, floor(L * k_num / k_den)) in integers. */
uint64_t orc_topk_k(const orc_comp* c, uint64_t L) {
  uint64_t k = (L * (uint64_t)c->k_num) / (uint64_t)c->k_den;
  return k < 1 ? 1 : k;
}

/* R23: a sparse value in binary16 (PAPER.md:648 counts 16-bit values): the
 * fp32 value saturated to the largest finite half, +-65504, then rounded to
 * nearest even (the C compiler's float -> _Float16 conversion). */
static uint16_t f32_to_f16(float v) {
  if (v > 65504.0f) v = 65504.0f;
  if (v < -65504.0f) v = -65504.0f;
  _Float16 h = (_Float16)v;
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static float f16_to_f32(uint16_t u) {
  _Float16 h;
  memcpy(&h, &u, 2);
  return (float)h;
}

/* Closed-form payload sizes. */
uint64_t orc_payload_bytes(const orc_comp* c, int raw, uint64_t L) {
  if (raw || c->kind == ORC_NONE) return 4 * L;
  switch (c->kind) {
    case ORC_SCALED_SIGN: return 4 + (L + 7) / 8;
    case ORC_TOP_K:
    case ORC_RANDOM_K: return 8 + (c->f16 ? 6 : 8) * orc_topk_k(c, L);
    case ORC_LINEAR_DITHER:
    case ORC_NATURAL_DITHER: return 4 + (c->bits * L + 7) / 8;
  }
  return 0;
}

/* ---- sparse selection helpers ---- */
typedef struct { float mag; uint32_t key; uint64_t j; } sel_item;

/* top-k order (R9): |q| descending, then index ascending */
static int cmp_topk(const void* a, const void* b) {
  const sel_item* x = (const sel_item*)a;
  const sel_item* y = (const sel_item*)b;
  if (x->mag > y->mag) return -1;
  if (x->mag < y->mag) return 1;
  return x->j < y->j ? -1 : (x->j > y->j ? 1 : 0);
}
/* random-k order (R10): Philox key ascending, then index ascending */
static int cmp_randk(const void* a, const void* b) {
  const sel_item* x = (const sel_item*)a;
  const sel_item* y = (const sel_item*)b;
  if (x->key < y->key) return -1;
  if (x->key > y->key) return 1;
  return x->j < y->j ? -1 : (x->j > y->j ? 1 : 0);
}
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* ------------------------------------------------------------------------ */
int orc_compress(const orc_comp* c, int raw, const float* x, uint64_t L, uint64_t seed,
                 uint32_t chunk, uint32_t t, uint32_t stage, uint32_t rank, uint8_t* out) {
  memset(out, 0, orc_payload_bytes(c, raw, L));
  if (raw || c->kind == ORC_NONE) {
    /* identity: raw fp32 values */
    for (uint64_t j = 0; j < L; j++) put_f32(out + 4 * j, x[j]);
    return 0;
  }
  switch (c->kind) {
    case ORC_SCALED_SIGN: {
      /* C(v) = ||v||_1 / d * sign(v), with d = L (R1) and
       * sign(0) = +1 (R2). Payload: [f32 s][bit j = 1 iff v_j >= 0]. */
      float s = (float)(l1_norm(x, L) / (double)L);
      put_f32(out, s);
      for (uint64_t j = 0; j < L; j++)
        if (!(x[j] < 0.0f)) put_bits(out + 4, j, 1, 1);
      return 0;
    }
    case ORC_TOP_K:
    case ORC_RANDOM_K: {
      /* top-k: the k largest |v_j| (ties R9);
       * random-k: k indices with the smallest Philox keys (R10). */
      uint64_t k = orc_topk_k(c, L);
      if (k > L) return 1;
      sel_item* it = (sel_item*)malloc(sizeof(sel_item) * L);
      for (uint64_t j = 0; j < L; j++) {
        it[j].mag = fabsf(x[j]);
        it[j].key = c->kind == ORC_RANDOM_K ? orc_rng_word(seed, j, chunk, t, stage, rank) : 0;
        it[j].j = j;
      }
      qsort(it, L, sizeof(sel_item), c->kind == ORC_TOP_K ? cmp_topk : cmp_randk);
      uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * k);
      for (uint64_t i = 0; i < k; i++) idx[i] = it[i].j;
      qsort(idx, k, sizeof(uint64_t), cmp_u64);          /* indices ascending */
      put_u64(out, k);
      float scale = 1.0f;
      int scaled = c->kind == ORC_RANDOM_K && c->randk_scaled;
      if (scaled) scale = (float)((double)L / (double)k);  /* unbiased d/k */
      for (uint64_t i = 0; i < k; i++) {
        put_u32(out + 8 + 4 * i, (uint32_t)idx[i]);
        float val = scaled ? x[idx[i]] * scale : x[idx[i]];
        if (c->f16) {                                     /* R23 */
          uint16_t h = f32_to_f16(val);
          memcpy(out + 8 + 4 * k + 2 * i, &h, 2);
        } else {
          put_f32(out + 8 + 4 * k + 4 * i, val);
        }
      }
      free(idx);
      free(it);
      return 0;
    }
    case ORC_LINEAR_DITHER: {
      /* QSGD-style linear dithering:
       * s levels on [0, 1] of |v|/||v||_2, stochastic rounding (R11-R13). */
      uint32_t b = c->bits;
      if (b < 2 || b > 8) return 1;
      float sl = (float)((1u << (b - 1)) - 1u);
      float N = l2_norm_f32(x, L);
      put_f32(out, N);
      for (uint64_t j = 0; j < L; j++) {
        uint32_t sign = !(x[j] < 0.0f);
        uint32_t level = 0;
        if (N != 0.0f) {
          float inv = sl / N;
          float r = fabsf(x[j]) * inv;
          if (r > sl) r = sl;
          float l = floorf(r);
          float f = r - l;
          float u = (float)(orc_rng_word(seed, j, chunk, t, stage, rank) >> 8) * 0x1p-24f;
          level = (uint32_t)l + (u < f ? 1u : 0u);
        }
        put_bits(out + 4, (uint64_t)b * j, b, sign | (level << 1));
      }
      return 0;
    }
    case ORC_NATURAL_DITHER: {
      /* natural dithering (Horvath et al.):
       * levels {0} U {2^-(cmax-c) : c = 1..cmax}, cmax = 2^(b-1) - 1 (R11). */
      uint32_t b = c->bits;
      if (b < 2 || b > 8) return 1;
      int cmax = (int)((1u << (b - 1)) - 1u);
      float lmin = ldexpf(1.0f, -(cmax - 1));
      float N = l2_norm_f32(x, L);
      put_f32(out, N);
      for (uint64_t j = 0; j < L; j++) {
        uint32_t sign = !(x[j] < 0.0f);
        uint32_t code = 0;
        if (N != 0.0f) {
          float r = fabsf(x[j]) / N;
          if (r > 1.0f) r = 1.0f;
          float u = (float)(orc_rng_word(seed, j, chunk, t, stage, rank) >> 8) * 0x1p-24f;
          if (r >= lmin) {
            int ex;
            frexpf(r, &ex);                  /* r = m * 2^ex, m in [0.5, 1) */
            int e_lo = ex - 1;               /* lo = 2^e_lo <= r < 2^(e_lo+1) */
            float lo = ldexpf(1.0f, e_lo);
            float pup = r / lo - 1.0f;
            int e_lev = (u < pup) ? e_lo + 1 : e_lo;
            code = (uint32_t)(cmax + e_lev);  /* level 2^e_lev = 2^-(cmax - code) */
          } else {
            float pup = r / lmin;
            code = (u < pup) ? 1u : 0u;
          }
        }
        put_bits(out + 4, (uint64_t)b * j, b, sign | (code << 1));
      }
      return 0;
    }
  }
  return 1;
}

int orc_decompress(const orc_comp* c, int raw, const uint8_t* in, uint64_t L, float* out) {
  if (raw || c->kind == ORC_NONE) {
    for (uint64_t j = 0; j < L; j++) out[j] = get_f32(in + 4 * j);
    return 0;
  }
  switch (c->kind) {
    case ORC_SCALED_SIGN: {
      float s = get_f32(in);
      for (uint64_t j = 0; j < L; j++) out[j] = get_bits(in + 4, j, 1) ? s : -s;
      return 0;
    }
    case ORC_TOP_K:
    case ORC_RANDOM_K: {
      uint64_t k = get_u64(in);
      for (uint64_t j = 0; j < L; j++) out[j] = 0.0f;
      uint64_t prev = 0;
      for (uint64_t i = 0; i < k; i++) {
        uint64_t j = get_u32(in + 8 + 4 * i);
        if (j >= L || (i > 0 && j <= prev)) return 1;   /* malformed */
        if (c->f16) {
          uint16_t h;
          memcpy(&h, in + 8 + 4 * k + 2 * i, 2);
          out[j] = f16_to_f32(h);
        } else {
          out[j] = get_f32(in + 8 + 4 * k + 4 * i);
        }
        prev = j;
      }
      return 0;
    }
    case ORC_LINEAR_DITHER: {
      uint32_t b = c->bits;
      float sl = (float)((1u << (b - 1)) - 1u);
      float N = get_f32(in);
      float unit = N / sl;
      for (uint64_t j = 0; j < L; j++) {
        uint32_t code = get_bits(in + 4, (uint64_t)b * j, b);
        float mag = (float)(code >> 1) * unit;
        out[j] = (code & 1u) ? mag : -mag;
      }
      return 0;
    }
    case ORC_NATURAL_DITHER: {
      uint32_t b = c->bits;
      int cmax = (int)((1u << (b - 1)) - 1u);
      float N = get_f32(in);
      for (uint64_t j = 0; j < L; j++) {
        uint32_t code = get_bits(in + 4, (uint64_t)b * j, b);
        uint32_t cl = code >> 1;
        float level = cl == 0 ? 0.0f : ldexpf(1.0f, -(cmax - (int)cl));
        float mag = level * N;
        out[j] = (code & 1u) ? mag : -mag;
      }
      return 0;
    }
  }
  return 1;
}

/* ------------------------------------------------------------------------ */
/* Chunk plan: R3 (tensors with 4*numel < threshold bytes stay raw, one unit
 * each) and R1 (compressed tensors split into units of
 * chunk_elems; 0 = whole tensor). Chunk ids are global, in tensor order. */
int64_t orc_plan(const orc_cfg* cfg, orc_chunk* chunks, int64_t cap) {
  int64_t nc = 0;
  for (uint32_t ti = 0; ti < cfg->num_tensors; ti++) {
    uint64_t L = cfg->numel[ti];
    if (L == 0) return -1;
    int raw = (4 * L < cfg->threshold_bytes) || cfg->comp.kind == ORC_NONE;
    uint64_t unit = (raw || cfg->chunk_elems == 0) ? L : cfg->chunk_elems;
    for (uint64_t s = 0; s < L; s += unit) {
      if (chunks && nc < cap) {
        chunks[nc].tensor = ti;
        chunks[nc].offset = cfg->offset[ti] + s;
        chunks[nc].len = (L - s < unit) ? (L - s) : unit;
        chunks[nc].raw = raw;
      }
      nc++;
    }
  }
  return nc;
}

/* ------------------------------------------------------------------------ */
void orc_push_pull(uint32_t n, uint64_t D, const float* g, float* out) {
  /* Alg. 1: p_t = (1/n) sum_i g_{t,i}; fp64 accumulation in rank order (R5). */
  for (uint64_t j = 0; j < D; j++) {
    double acc = 0.0;
    for (uint32_t i = 0; i < n; i++) acc += (double)g[(uint64_t)i * D + j];
    out[j] = (float)(acc * (1.0 / (double)n));
  }
}

void orc_adam(uint64_t L, const float* gt, float* m, float* v, float* x, uint32_t t,
              float lr, float beta1, float beta2, float eps, float wd) {
  /* Alg. 5 lines 12-16 and the x update with the
   * direction r + lambda x (PAPER.md:292-295 with the LANS normalisation
   * left to NEXT #1): reading R15. The bias corrections (1 - beta^t) are
   * formed once per step in fp64 and rounded to fp32 (R16); lines 14-15
   * divide by them, as the paper writes. */
  float omb1 = (float)(1.0 - (double)beta1);
  float omb2 = (float)(1.0 - (double)beta2);
  float bc1 = (float)(1.0 - pow((double)beta1, (double)t));
  float bc2 = (float)(1.0 - pow((double)beta2, (double)t));
  for (uint64_t j = 0; j < L; j++) {
    float g = gt[j];
    m[j] = beta1 * m[j] + omb1 * g;                 /* line 12 */
    v[j] = beta2 * v[j] + omb2 * (g * g);           /* line 13 */
    float mh = m[j] / bc1;                          /* line 14: m / (1 - beta1^t) */
    float vh = v[j] / bc2;                          /* line 15: v / (1 - beta2^t) */
    float r = mh / (sqrtf(vh) + eps);               /* line 16 */
    x[j] = x[j] - lr * (r + wd * x[j]);             /* line 18 (Adam core) */
  }
}

/* NAG, the optimizer every compressor is applied to in the CNN experiments
 * ("All the compression methods are applied to NAG"), in the
 * form of SPEC.md:393 with weight decay folded into the gradient as in the
 * SGD of the paper's training recipe (reading R24):
 *   g = g~ + lambda x;  v = mu v + g;  x = x - eta (g + mu v). */
void orc_nag(uint64_t L, const float* gt, float* vel, float* x, float lr, float mu, float wd) {
  for (uint64_t j = 0; j < L; j++) {
    float g = gt[j] + wd * x[j];
    vel[j] = mu * vel[j] + g;
    x[j] = x[j] - lr * (g + mu * vel[j]);
  }
}

/* LANS block update (CLAN, Alg. 5 lines 12-18; the same
 * step as Alg. 2 lines 8-14), in the paper's order:
 *   m, v, m~, v~ as in orc_adam (lines 12-15, R16);
 *   line 16: r = m~ / (sqrt(v~) + eps),  c = g~ / (sqrt(v~) + eps);
 *   line 17: d~ = phi(||x_b||) [ beta1 (r + lambda x)/||r + lambda x||
 *                               + (1 - beta1)(c + lambda x)/||c + lambda x|| ];
 *   line 18: x = x - eta d~.
 * Reading R22: the three block norms are fp64 pairwise sums (R6)
 * of the exact fp64 squares of the fp32 values, square-rooted in fp64;
 * phi(z) = min(max(fl32(||x_b||), alpha_l), alpha_u); the two
 * per-block coefficients a = fl32(phi * beta1 / ||r + lambda x||) and
 * b = fl32(phi * (1 - beta1) / ||c + lambda x||) are formed in fp64, and a
 * zero norm makes its term zero; per element, in fp32,
 * d = a u + b w and x = x - eta d. */
void orc_lans_block(uint64_t L, const float* gt, float* m, float* v, float* x, uint32_t t,
                    float lr, float beta1, float beta2, float eps, float wd, float alpha_l,
                    float alpha_u) {
  float omb1 = (float)(1.0 - (double)beta1);
  float omb2 = (float)(1.0 - (double)beta2);
  float bc1 = (float)(1.0 - pow((double)beta1, (double)t));
  float bc2 = (float)(1.0 - pow((double)beta2, (double)t));
  float* u = (float*)malloc(sizeof(float) * (size_t)(L ? L : 1));
  float* w = (float*)malloc(sizeof(float) * (size_t)(L ? L : 1));
  double* sq = (double*)malloc(sizeof(double) * (size_t)(L ? L : 1));
  for (uint64_t j = 0; j < L; j++) {
    float g = gt[j];
    m[j] = beta1 * m[j] + omb1 * g;                 /* line 12 */
    v[j] = beta2 * v[j] + omb2 * (g * g);           /* line 13 */
    float mh = m[j] / bc1;                          /* line 14 */
    float vh = v[j] / bc2;                          /* line 15 */
    float den = sqrtf(vh) + eps;
    float r = mh / den;                             /* line 16: r */
    float c = g / den;                              /* line 16: c */
    u[j] = r + wd * x[j];                           /* r + lambda x */
    w[j] = c + wd * x[j];                           /* c + lambda x */
  }
  for (uint64_t j = 0; j < L; j++) sq[j] = (double)x[j] * (double)x[j];
  double nx = sqrt(orc_pairwise_sum(sq, L));
  for (uint64_t j = 0; j < L; j++) sq[j] = (double)u[j] * (double)u[j];
  double nu = sqrt(orc_pairwise_sum(sq, L));
  for (uint64_t j = 0; j < L; j++) sq[j] = (double)w[j] * (double)w[j];
  double nw = sqrt(orc_pairwise_sum(sq, L));
  float phi = (float)nx;
  if (phi < alpha_l) phi = alpha_l;
  if (phi > alpha_u) phi = alpha_u;
  float a = nu > 0.0 ? (float)((double)phi * (double)beta1 / nu) : 0.0f;
  float b = nw > 0.0 ? (float)((double)phi * (1.0 - (double)beta1) / nw) : 0.0f;
  for (uint64_t j = 0; j < L; j++) {
    float d = a * u[j] + b * w[j];                  /* line 17 */
    x[j] = x[j] - lr * d;                           /* line 18 */
  }
  free(u); free(w); free(sq);
}

/* ------------------------------------------------------------------------ */
/* Host threads for orc_round (OpenMP over units; 1 = plain serial). Units are
 * independent in Alg. 3/4 (each worker compresses each unit on its own, the
 * server aggregates each unit on its own, the update is per element / per
 * block), so the result does not depend on the thread count. */
static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int orc_get_threads(void) { return g_threads; }

int orc_round(const orc_cfg* cfg, uint64_t D, const float* grads, float* e, float* et,
              float* m, float* v, float* x, uint32_t t, float lr,
              uint8_t* delta_out, uint8_t* p_out, float* gtilde_out) {
  int64_t nc = orc_plan(cfg, NULL, 0);
  if (nc < 0 || cfg->n < 1 || t < 1) return 1;
  orc_chunk* ch = (orc_chunk*)malloc(sizeof(orc_chunk) * (size_t)(nc ? nc : 1));
  orc_plan(cfg, ch, nc);
  const orc_comp* C = &cfg->comp;
  uint32_t n = cfg->n;

  /* payload stream: chunk c at byte offset poff[c], no padding */
  uint64_t* poff = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nc + 1));
  poff[0] = 0;
  for (int64_t c = 0; c < nc; c++) poff[c + 1] = poff[c] + orc_payload_bytes(C, ch[c].raw, ch[c].len);
  uint64_t total = poff[nc];
  uint8_t* delta = (uint8_t*)malloc((size_t)((n * total) > 0 ? n * total : 1));
  uint8_t* pbuf = (uint8_t*)malloc((size_t)(total ? total : 1));
  float* gall = cfg->optimizer == 1 ? (float*)calloc((size_t)(D ? D : 1), sizeof(float)) : NULL;
  int err = 0;

  /* ---- workers (Alg. 4 lines 5-7; Alg. 3 line 4),
   * every (worker i, unit c) on its own */
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads) reduction(|: err)
  for (int64_t w = 0; w < (int64_t)n * nc; w++) {
    uint32_t i = (uint32_t)(w / nc);
    int64_t c = w % nc;
    const float* g = grads + (uint64_t)i * D;
    float* ei = e + (uint64_t)i * D;
    uint64_t L = ch[c].len, o = ch[c].offset;
    int ef = C->use_ef && !ch[c].raw;     /* raw units carry no EF (R3) */
    float* q = (float*)malloc(sizeof(float) * L);
    float* dec = (float*)malloc(sizeof(float) * L);
    for (uint64_t j = 0; j < L; j++) q[j] = ef ? g[o + j] + ei[o + j] : g[o + j];  /* q = g + e */
    uint8_t* d = delta + (uint64_t)i * total + poff[c];
    err |= orc_compress(C, ch[c].raw, q, L, cfg->seed, (uint32_t)c, t, 0, i, d);  /* delta = C(q) */
    if (ef) {
      err |= orc_decompress(C, 0, d, L, dec);
      for (uint64_t j = 0; j < L; j++) ei[o + j] = q[j] - dec[j];                  /* e = q - delta */
    }
    free(q); free(dec);
  }

  /* ---- server (Alg. 4 lines 10-13; Alg. 3 lines 7-8), every unit
   * on its own, then the workers' g~ = dec(p) and the adaptive update (Alg. 5 l.12-18) */
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads) reduction(|: err)
  for (int64_t c = 0; c < nc; c++) {
    if (err) continue;
    uint64_t L = ch[c].len, o = ch[c].offset, off = poff[c];
    int ef = C->use_ef && !ch[c].raw;
    float* q = (float*)malloc(sizeof(float) * L);
    float* dec = (float*)malloc(sizeof(float) * L);
    float* gt = (float*)malloc(sizeof(float) * L);
    double* acc = (double*)malloc(sizeof(double) * L);
    for (uint64_t j = 0; j < L; j++) acc[j] = 0.0;
    for (uint32_t i = 0; i < n; i++) {              /* pull delta_i, sum in rank order (R5) */
      err |= orc_decompress(C, ch[c].raw, delta + (uint64_t)i * total + off, L, dec);
      for (uint64_t j = 0; j < L; j++) acc[j] += (double)dec[j];
    }
    for (uint64_t j = 0; j < L; j++)                /* Delta = (1/n) sum + e~ */
      q[j] = (float)(acc[j] * (1.0 / (double)n) + (ef ? (double)et[o + j] : 0.0));
    err |= orc_compress(C, ch[c].raw, q, L, cfg->seed, (uint32_t)c, t, 1, 0, pbuf + off);  /* p = C(Delta) */
    err |= orc_decompress(C, ch[c].raw, pbuf + off, L, gt);
    if (ef)
      for (uint64_t j = 0; j < L; j++) et[o + j] = q[j] - gt[j];                     /* e~ = Delta - p */
    /* ---- workers: g~ = dec(p), then the adaptive update (Alg. 5 l.12-18) */
    if (cfg->optimizer == 1)
      memcpy(gall + o, gt, sizeof(float) * L);      /* LANS: per-block update after all chunks */
    else if (cfg->optimizer == 2)
      orc_nag(L, gt, m + o, x + o, lr, cfg->momentum, cfg->weight_decay);   /* velocity in m */
    else
      orc_adam(L, gt, m + o, v + o, x + o, t, lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay);
    if (gtilde_out) memcpy(gtilde_out + o, gt, sizeof(float) * L);
    free(q); free(dec); free(gt); free(acc);
  }

  if (!err && cfg->optimizer == 1) {                /* LANS: one block per tensor */
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t b = 0; b < (int64_t)cfg->num_tensors; b++) {
      uint64_t o = cfg->offset[b], L = cfg->numel[b];
      orc_lans_block(L, gall + o, m + o, v + o, x + o, t, lr, cfg->beta1, cfg->beta2, cfg->eps,
                     cfg->weight_decay, cfg->alpha_l, cfg->alpha_u);
    }
  }
  free(gall);
  if (!err && delta_out) memcpy(delta_out, delta, (size_t)(n * total));
  if (!err && p_out) memcpy(p_out, pbuf, (size_t)total);
  free(delta); free(pbuf); free(poff); free(ch);
  return err;
}
