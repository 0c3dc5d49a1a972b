/*
 * oracle.h — plain, slow CPU oracle for the compressed aggregation + update
 * step of arXiv 2105.07829 (CLAN / BytePS-Compress).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2105_07829_b200/csrc, include/bpc.h) and never includes them.
 *
 * Every function follows the paper's statement, citing PAPER.md lines:
 *   Alg. 3 compress_push_pull
 *   Alg. 4 compress_ef_push_pull
 *   Alg. 5 CLAN (lines 12-16 + x update, Adam core)
 *   scaled sign
 *   top-k / random-k / dithering
 *   operator fusion (O(k) EF)      PAPER.md:501-502 (the oracle does NOT fuse;
 *                                  it computes e = q - dec(C(q)) literally)
 *   size threshold
 * Where the paper is silent the oracle takes DESIGN.md §3 reading R<n>.
 * Floating point is fp32 where the paper's objects are fp32 gradients
 * and fp64 for every accumulation (R5, R6).
 */
#ifndef BPC_ORACLE_H
#define BPC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Compressor kinds; numeric ids follow the SPEC wire ids. */
enum { ORC_NONE = 0, ORC_SCALED_SIGN = 2, ORC_TOP_K = 3, ORC_RANDOM_K = 4,
       ORC_LINEAR_DITHER = 5, ORC_NATURAL_DITHER = 6 };

typedef struct {
  int32_t kind;
  uint32_t k_num, k_den;   /* sparse kinds: k = max(1, floor(L*k_num/k_den)) (R8) */
  uint32_t bits;           /* dither bits including the sign bit, 2..8 (R11) */
  int32_t randk_scaled;    /* random-k: 1 = values * L/k (unbiased, Alg. 3); 0 = unscaled (R10) */
  int32_t use_ef;          /* Alg. 5 use_ef */
  int32_t f16;             /* sparse kinds: values as IEEE binary16 (PAPER.md:648's 333x, R23) */
} orc_comp;

typedef struct {
  uint32_t n;                    /* number of workers n (Alg. 3/4) */
  uint64_t seed;                 /* Philox key (R13) */
  uint32_t num_tensors;
  const uint64_t* numel;         /* per tensor element count */
  const uint64_t* offset;        /* per tensor element offset in the flat buffer */
  uint64_t chunk_elems;          /* compression unit (R1); 0 = whole tensor */
  uint64_t threshold_bytes;      /* PAPER.md:505 size threshold (R3) */
  orc_comp comp;
  float beta1, beta2, eps, weight_decay;   /* Alg. 5 inputs, R15 */
  int32_t optimizer;             /* 0: Adam core (R15); 1: LANS block-normalised update (R22);
                                    2: NAG (R24) */
  float alpha_l, alpha_u;        /* LANS: phi = clamp(., alpha_l, alpha_u) */
  float momentum;                /* NAG: mu in [0, 1) */
} orc_cfg;

typedef struct {
  uint32_t tensor;     /* tensor index */
  uint64_t offset;     /* flat element offset of the chunk's first element */
  uint64_t len;        /* L, elements in the compression unit */
  int32_t raw;         /* 1: below the size threshold -> NONE compressor */
} orc_chunk;

/* ---- primitives ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* Philox word for element j of chunk c, step t, stage (0 push / 1 pull), rank (R13). */
uint32_t orc_rng_word(uint64_t seed, uint64_t j, uint32_t chunk, uint32_t t,
                      uint32_t stage, uint32_t rank);
double orc_pairwise_sum(const double* a, uint64_t n);   /* R6 */

/* ---- compression operators on one unit of length L ---- */
uint64_t orc_topk_k(const orc_comp* c, uint64_t L);
uint64_t orc_payload_bytes(const orc_comp* c, int raw, uint64_t L);
/* C(x) -> payload (orc_payload_bytes bytes). Returns 0 on success. */
int orc_compress(const orc_comp* c, int raw, const float* x, uint64_t L, uint64_t seed,
                 uint32_t chunk, uint32_t t, uint32_t stage, uint32_t rank, uint8_t* payload);
/* dec(payload) -> out[0..L). Returns 0 on success, nonzero if malformed. */
int orc_decompress(const orc_comp* c, int raw, const uint8_t* payload, uint64_t L, float* out);

/* ---- plan ---- */
/* Fills chunks (capacity cap); returns the chunk count, or -1 on a bad config. */
int64_t orc_plan(const orc_cfg* cfg, orc_chunk* chunks, int64_t cap);

/* ---- one bulk-synchronous round (Alg. 5 with Alg. 3 or 4) ----
 * grads: n rows of D floats (worker i's gradient g_{t,i});
 * e: n rows of D floats (worker errors e_{t,i}); etilde: D floats (server error);
 * m, v, x: D floats; t: step counter (>= 1).
 * delta_out (optional): n rows of payload_total bytes (worker payloads, chunk order,
 * no padding); p_out (optional): payload_total bytes (server payloads).
 * gtilde_out (optional): D floats, dec(p) (elements outside every chunk untouched). */
int orc_round(const orc_cfg* cfg, uint64_t D, const float* grads, float* e, float* etilde,
              float* m, float* v, float* x, uint32_t t, float lr,
              uint8_t* delta_out, uint8_t* p_out, float* gtilde_out);

/* Host threads of orc_round (OpenMP over units, default 1); the result is the
 * same for every thread count (units are independent). */
void orc_set_threads(int n);
int orc_get_threads(void);

/* Alg. 1 push_pull: p = (1/n) sum_i g_i with fp64 accumulation. */
void orc_push_pull(uint32_t n, uint64_t D, const float* grads, float* out);

/* Alg. 5 lines 12-15 + x update (Adam core, R15/R16) on one vector. */
/* LANS / CLAN update of one block G_b (Alg. 5 lines 12-18, PAPER.md:285-295;
 * Alg. 2), reading R22. */
void orc_lans_block(uint64_t L, const float* gtilde, float* m, float* v, float* x, uint32_t t,
                    float lr, float beta1, float beta2, float eps, float wd, float alpha_l,
                    float alpha_u);
/* Nesterov momentum (NAG) on the aggregated gradient, R24. */
void orc_nag(uint64_t L, const float* gtilde, float* vel, float* x, float lr, float mu, float wd);
void orc_adam(uint64_t L, const float* gtilde, float* m, float* v, float* x, uint32_t t,
              float lr, float beta1, float beta2, float eps, float weight_decay);

#ifdef __cplusplus
}
#endif
#endif
