/*
 * bpc.h — C ABI of the B200-native compressed aggregation + update step of
 * arXiv 2105.07829 (CLAN / BytePS-Compress), libbpc.so.
 *
 * The four calls of the hot path follow the paper's statement of the problem:
 *   bpc_compress   Alg. 4 lines 5-7 / Alg. 3 line 4:
 *                  on worker i, q = g + e; push delta = C(q); e = q - delta.
 *   bpc_aggregate  Alg. 4 lines 9-13 / Alg. 3 lines 6-9:
 *                  servers pull delta_i, Delta = (1/n) sum_i delta_i + e~, p = C(Delta),
 *                  e~ = Delta - p, push p to each worker. Here every GPU is the server
 *                  of its own shard of chunks ("More Servers"):
 *                  an all-to-all of compressed payloads, the server kernel, then an
 *                  all-gather of the re-compressed p, over NVLink peer memory fused
 *                  into the kernels (default) or NCCL (bpc_exchange_mode).
 *   bpc_step       Alg. 5 lines 12-16 + x update, Adam core
 *                  (R15): g~ = dec(p) decoded inside the update kernel.
 * bpc_aggregate = bpc_exchange_push; bpc_server; bpc_exchange_pull.
 *
 * Conventions (all calls):
 *  - Every call returns bpc_status; nothing throws or aborts across the ABI.
 *  - Host-detectable errors (NULL pointers, sizes, k > L, bad bits, misaligned
 *    offsets, call order) return before anything is enqueued and leave the
 *    state unchanged.  Device-side errors (non-finite gradients when
 *    check_finite, async CUDA/NCCL errors) surface at bpc_sync.
 *  - Pointers named d_* are DEVICE pointers (fp32, caller-owned, borrowed):
 *    the caller keeps them valid until cfg.cuda_stream has passed the work
 *    enqueued on them.  host_* are host pointers.  The context owns its
 *    worker error e, server error e~ (owned shard only), m, v, t and all
 *    payload buffers.
 *  - All device work is enqueued on cfg.cuda_stream (borrowed), in call order.
 *  - CUDA graphs: one step's calls (compress .. step, any world size, either
 *    exchange) may be captured once on cfg.cuda_stream and replayed; each replay
 *    is the next step.  The step counter t and the per-kernel-family launch and
 *    exchange epochs live in device memory and advance inside the kernels (the
 *    step's last update launch advances t), so no host value is baked into the
 *    graph.  The bias corrections of step t come from a device table built at
 *    bpc_init (R16).  bpc_sync, bpc_copy_state / load_state, get / set_step and
 *    bpc_get_timing synchronise and must stay outside a capture; timing must be
 *    off while capturing.
 *  - Call order per step: compress -> aggregate (or push, server, pull) -> step;
 *    out-of-order calls return BPC_ERR_BAD_STATE.  A context is not thread-safe.
 *  - Step counter t starts at 1 and advances in bpc_step's last kernel
 *    (SPEC.md:362, 411).
 *  - There is no CPU fallback: without a usable sm_100 device bpc_init fails
 *    with BPC_ERR_CUDA.
 */
#ifndef BPC_H
#define BPC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BPC_OK = 0,
  BPC_ERR_INVALID_ARGUMENT = 1,
  BPC_ERR_SIZE_MISMATCH = 2,
  BPC_ERR_EMPTY_BLOCK = 3,       /* a tensor with numel 0 */
  BPC_ERR_K_TOO_LARGE = 4,       /* resolved k > L */
  BPC_ERR_UNSUPPORTED_KIND = 5,
  BPC_ERR_BAD_STATE = 6,         /* call order / mode */
  BPC_ERR_NONFINITE = 7,         /* gradients must be finite */
  BPC_ERR_CUDA = 8,
  BPC_ERR_NCCL = 9,
  BPC_ERR_OUT_OF_MEMORY = 10
} bpc_status;

/* Compressor ids = SPEC wire ids. */
typedef enum {
  BPC_NONE = 0,            /* identity (Alg. 1 recovery) */
  BPC_SCALED_SIGN = 2,     /* ||v||_1/L * sign(v) per unit (R1, R2) */
  BPC_TOP_K = 3,           /* k largest |v|, ties to the lowest index (R8, R9) */
  BPC_RANDOM_K = 4,        /* k smallest Philox keys (R10) */
  BPC_LINEAR_DITHER = 5,   /* QSGD-style, s = 2^(bits-1)-1 levels (R11-R13) */
  BPC_NATURAL_DITHER = 6   /* power-of-two levels (R11-R13) */
} bpc_kind;

typedef struct {
  int32_t kind;            /* bpc_kind */
  uint32_t k_num, k_den;   /* sparse kinds: k = max(1, floor(L*k_num/k_den)) per unit, k_num <= k_den */
  uint32_t bits;           /* dither bits including the sign bit, 2..8 */
  int32_t randk_scaled;    /* random-k: 1 = values * L/k (unbiased); 0 = unscaled */
  int32_t use_ef;          /* Alg. 5 use_ef: 1 = Alg. 4 (error feedback), 0 = Alg. 3 */
  int32_t f16_values;      /* sparse kinds: 1 = values as IEEE binary16, saturated to +-65504,
                              round to nearest even (PAPER.md:648's 333x payload; DESIGN.md
                              R23); payload [u64 k][k x u32 index][k x f16]; 0 = fp32 (R20) */
} bpc_compressor;

typedef struct {
  int32_t world_size;            /* n workers = n GPUs (one process per GPU) */
  int32_t rank;                  /* this process's rank, 0..n-1 */
  int32_t device;                /* CUDA device ordinal this context runs on */
  void* cuda_stream;             /* cudaStream_t, borrowed; NULL = default stream */
  const uint8_t* nccl_unique_id; /* 128 bytes from bpc_get_unique_id() on rank 0, broadcast by
                                    the caller; NULL when world_size == 1 or for an external
                                    exchange (then only bpc_server and the buffer API are usable
                                    for the exchange, bpc_aggregate returns BPC_ERR_BAD_STATE) */
  uint64_t seed;                 /* Philox key for random-k / dithering (R13) */
  uint32_t num_tensors;
  const uint64_t* tensor_numel;  /* host array [num_tensors], each >= 1 */
  const uint64_t* tensor_offset; /* host array [num_tensors], element offsets into the flat
                                    buffers, multiples of 4 (16-byte aligned), non-overlapping */
  uint64_t chunk_elems;          /* compression unit (R1): a power of two in [2^14, 2^18];
                                    0 = default 2^18 */
  uint64_t size_threshold_bytes; /* tensors with 4*numel < threshold stay raw fp32 (R3) */
  bpc_compressor comp;
  float beta1, beta2, eps, weight_decay;   /* Alg. 5 inputs; weight_decay = lambda (R15) */
  int32_t check_finite;          /* 1: flag non-finite gradients (reported by bpc_sync) */
  int32_t exchange;              /* bpc_exchange_mode requested for A4/A8 when world_size > 1 */
  int32_t optimizer;             /* bpc_optimizer applied by bpc_step */
  float lans_alpha_l, lans_alpha_u;  /* LANS: phi(z) = min(max(z, alpha_l), alpha_u),
                                        0 < alpha_l <= alpha_u */
  float momentum;                /* NAG: mu in [0, 1) */
  int32_t unit_mode;             /* compression unit: 0 = chunks of chunk_elems (R1); 1 = one unit
                                    per tensor, the paper's granularity (NEXT #4),
                                    tensors <= 2^27 elements: scaled sign / dithering / NONE run
                                    two passes (slice partials, a per-unit tree, the emitting pass;
                                    20 B/element for onebit+EF); top-k / random-k units longer
                                    than 2^18 take a multi-CTA radix select over the unit */
} bpc_config;

/* The update of bpc_step (A9).
 * BPC_OPT_ADAM: Alg. 5 lines 12-16 and x = x - lr (r + weight_decay x)
 *   (R15, R16), one fused pass (24 B/element + payload).
 * BPC_OPT_LANS: CLAN proper, Alg. 5 lines 12-18 (Alg. 2
 *   PAPER.md:157-163): per block G_b = one tensor,
 *   d = phi(||x_b||) [beta1 (r + lambda x)/||r + lambda x|| + (1 - beta1)(c + lambda x)/||c + lambda x||],
 *   c = g~/(sqrt(v~) + eps), x = x - lr d (reading R22).  Two streaming passes
 *   plus one CTA per block for the norms (36 B/element + 2 payload reads);
 *   every tensor must have <= 2^25 elements (else BPC_ERR_INVALID_ARGUMENT).
 * BPC_OPT_NAG: Nesterov momentum, the optimizer every compressor is applied to
 *   in the paper's CNN runs (R24): g = g~ + lambda x,
 *   v = momentum v + g, x = x - lr (g + momentum v); the velocity lives in the
 *   BPC_BUF_M buffer, BPC_BUF_V is unused (16 B/element + payload). */
typedef enum { BPC_OPT_ADAM = 0, BPC_OPT_LANS = 1, BPC_OPT_NAG = 2 } bpc_optimizer;

/* Transport of the exchange steps A4 (push) and A8 (pull), world_size > 1.
 * BPC_EXCHANGE_P2P: every rank maps its peers' RECV / P / flag buffers with CUDA
 *   IPC (handles all-gathered over the NCCL communicator at init); flags are
 *   per-step epochs released with system-scope stores and waited on with
 *   acquire loads inside the kernels.
 *   - norm-based kinds (NONE, SCALED_SIGN, dithering), fused into the kernels:
 *     bpc_compress stores each payload straight into its owner's RECV slot
 *     over NVLink (SEND is not written) and releases the push flags;
 *     bpc_server waits for every rank's push, writes p into its own P segment
 *     and releases the pull flags; bpc_step waits for them and bulk-copies
 *     each chunk's p from its owner's P over NVLink.  bpc_exchange_push/pull
 *     launch nothing; P holds valid bytes for the owned segment only.
 *   - sparse kinds (top-k, random-k): bpc_exchange_push/pull run a copy
 *     kernel that stores the segments into the peers' RECV / P over NVLink and
 *     releases the flags; bpc_server / bpc_step start with a one-warp kernel
 *     that waits for the peers' flags (SEND and P fully valid).
 *   If the peer mappings cannot be opened on every rank, init falls back to
 *   BPC_EXCHANGE_NCCL (bpc_get_exchange reports what is in use).
 * BPC_EXCHANGE_NCCL: grouped ncclSend/ncclRecv (all-to-all, all-gather). */
/* BPC_EXCHANGE_NVLS: BPC_EXCHANGE_P2P with the pull (A8) through NVLink SHARP
 * multicast: P is a VMM allocation bound to one multicast
 * object over the ranks' devices; the server kernel stores each owned unit's p
 * once through the multicast mapping (multimem.st), the switch writes it into
 * every rank's P, and the update kernel reads every p from local HBM.  Set up
 * at bpc_init (collective: rank 0 creates the object and hands its POSIX fd to
 * the other processes over an abstract unix socket) or bpc_connect_local
 * (distinct devices); it applies to the fused kinds (scaled sign, dithering,
 * NONE).  Where multicast is unavailable (no NVSwitch multicast support, a
 * shared device, a failed step on any rank) the group keeps BPC_EXCHANGE_P2P;
 * bpc_get_exchange reports BPC_EXCHANGE_NVLS only when it is in use. */
typedef enum { BPC_EXCHANGE_P2P = 0, BPC_EXCHANGE_NCCL = 1, BPC_EXCHANGE_NVLS = 2 } bpc_exchange_mode;

typedef struct bpc_ctx bpc_ctx;

/* Buffers a caller may inspect (bpc_buffer / bpc_copy_state / bpc_load_state). */
typedef enum {
  BPC_BUF_SEND = 0,        /* worker payloads delta, grouped by owner rank (device; not
                              written by the fused P2P exchange: see RECV) */
  BPC_BUF_RECV = 1,        /* this owner's n received payload slots (device) */
  BPC_BUF_P = 2,           /* server payloads p, same layout as SEND (device; fused P2P
                              exchange: only this rank's owned segment) */
  BPC_BUF_WORKER_ERR = 3,  /* e, fp32, flat layout of the gradient */
  BPC_BUF_SERVER_ERR = 4,  /* e~ of the owned chunks, fp32, compact (chunk server_err_offset) */
  BPC_BUF_M = 5,           /* first moment m, flat */
  BPC_BUF_V = 6            /* second moment v, flat */
} bpc_buffer_id;

typedef struct {
  uint32_t tensor;           /* tensor index */
  int32_t raw;               /* 1: below threshold, NONE payload */
  uint32_t owner;            /* rank that acts as this chunk's server */
  uint32_t k;                /* sparse k of the unit (0 otherwise) */
  uint64_t offset;           /* flat element offset of the unit */
  uint64_t len;              /* L */
  uint64_t payload_offset;   /* byte offset in SEND and P */
  uint64_t payload_bytes;    /* closed-form payload size (unpadded) */
  uint64_t recv_offset;      /* byte offset inside each RECV slot (owner only) */
  uint64_t server_err_offset;/* element offset in SERVER_ERR (owner only, compressed + use_ef) */
} bpc_chunk_info;

typedef struct {
  uint32_t num_chunks, num_compressed, num_owned;
  uint32_t cluster_ctas;     /* CTAs per compression unit (chunk_elems / 2^14) */
  uint64_t flat_elems;       /* D = max(offset + numel) */
  uint64_t send_bytes;       /* SEND / P buffer size */
  uint64_t recv_slot_bytes;  /* bytes per RECV slot (= this rank's SEND segment) */
  uint64_t server_err_elems; /* SERVER_ERR length */
  uint64_t payload_total;    /* sum of unpadded payload bytes (wire volume per direction) */
} bpc_plan_summary;

bpc_status bpc_get_unique_id(uint8_t out[128]);

/* Validates cfg, builds the chunk plan (R1, R3) and owner map (LPT over server cost,
 * DESIGN.md §7), allocates e, e~, m, v (zeroed) and payload buffers on cfg.device,
 * and creates the NCCL communicator when cfg.nccl_unique_id is given (collective
 * over all ranks). */
bpc_status bpc_init(const bpc_config* cfg, bpc_ctx** out);
/* Host-only planning (no device needed): fills the summary and, if infos != NULL,
 * up to cap chunk records, exactly as bpc_init would. */
bpc_status bpc_plan(const bpc_config* cfg, bpc_plan_summary* summary, bpc_chunk_info* infos,
                    uint32_t cap);

/* Single-process exchange group: wires n contexts of THIS process (index r =
 * rank r, world_size n, created with nccl_unique_id = NULL, before their first
 * step) into one BPC_EXCHANGE_P2P group with direct device pointers instead of
 * CUDA IPC.  Contexts on distinct devices get peer access enabled (both
 * directions; BPC_ERR_CUDA if the devices cannot reach each other).  The
 * kernels then run exactly the multi-process P2P exchange (fused stores into
 * the owners' RECV, release / acquire flags, bulk reads of the owners' P).
 * Issue order: every rank's call of one phase before any rank's next phase
 * (compress x n, exchange_push x n, server x n, exchange_pull x n, step x n),
 * because a phase's kernels wait on flags released by the previous phase of
 * every rank; contexts that share a device must also share one stream, or a
 * persistent kernel spinning on a flag can hold the SMs its producer needs.
 * bpc_aggregate on one context is then invalid (it would wait on peers'
 * later phases).  Finalize only after every context's stream has drained.
 * Errors: BPC_ERR_INVALID_ARGUMENT (NULL, n < 2 or n > 64), BPC_ERR_BAD_STATE
 * (wrong world size / rank order, NCCL id given, already stepped),
 * BPC_ERR_SIZE_MISMATCH (plans differ). */
bpc_status bpc_connect_local(bpc_ctx* const* ctxs, int32_t n);

/* d_grad / d_params: device memory of cfg.device (or managed), 16-byte aligned,
 * >= plan flat_elems fp32 values; otherwise BPC_ERR_INVALID_ARGUMENT before
 * anything is enqueued. */
bpc_status bpc_compress(bpc_ctx* ctx, const float* d_grad);          /* A1-A3 */
bpc_status bpc_aggregate(bpc_ctx* ctx);                              /* A4-A8 */
bpc_status bpc_exchange_push(bpc_ctx* ctx);                          /* A4 all-to-all */
bpc_status bpc_server(bpc_ctx* ctx);                                 /* A5-A7 */
bpc_status bpc_exchange_pull(bpc_ctx* ctx);                          /* A8 all-gather */
bpc_status bpc_step(bpc_ctx* ctx, float* d_params, float lr);        /* A9, t += 1 */
bpc_status bpc_sync(bpc_ctx* ctx);   /* drain the stream; surface async CUDA/NCCL/non-finite */
/* Frees the context.  With the multi-process P2P exchange this is collective
 * (an NCCL all-reduce orders every rank's frees after all peers' last reads of
 * its buffers): every rank must call it. */
bpc_status bpc_finalize(bpc_ctx* ctx);

bpc_status bpc_get_plan(const bpc_ctx* ctx, bpc_plan_summary* out);
bpc_status bpc_get_chunk(const bpc_ctx* ctx, uint32_t chunk, bpc_chunk_info* out);
/* Segment of peer r inside SEND / P: [*offset, *offset + *bytes). */
bpc_status bpc_peer_segment(const bpc_ctx* ctx, int32_t peer, uint64_t* offset, uint64_t* bytes);
bpc_status bpc_buffer(const bpc_ctx* ctx, int32_t which, void** d_ptr, uint64_t* bytes);
/* Synchronous copies of a buffer to / from host memory (bytes must equal its size). */
bpc_status bpc_copy_state(bpc_ctx* ctx, int32_t which, void* host_dst, uint64_t bytes);
bpc_status bpc_load_state(bpc_ctx* ctx, int32_t which, const void* host_src, uint64_t bytes);
/* Exchange transport in use (bpc_exchange_mode; BPC_EXCHANGE_NCCL also when
 * world_size == 1 or for an external exchange, where no transport runs). */
bpc_status bpc_get_exchange(const bpc_ctx* ctx, int32_t* mode);
/* The device step counter t: get waits for cfg.cuda_stream to drain and reads it;
 * set (t >= 1, else BPC_ERR_INVALID_ARGUMENT) writes it in stream order and
 * waits (resume after bpc_load_state of e, e~, m, v). */
bpc_status bpc_get_step(const bpc_ctx* ctx, uint32_t* t);
bpc_status bpc_set_step(bpc_ctx* ctx, uint32_t t);

/* Per-kernel device timing with CUDA events on cfg.cuda_stream.
 * Kernel ids: 0 worker compress, 1 server, 2 update, 3 exchange push, 4 exchange pull. */
enum { BPC_TIMER_COMPRESS = 0, BPC_TIMER_SERVER = 1, BPC_TIMER_UPDATE = 2,
       BPC_TIMER_PUSH = 3, BPC_TIMER_PULL = 4, BPC_NUM_TIMERS = 5 };
bpc_status bpc_set_timing(bpc_ctx* ctx, int32_t enable);   /* resets the accumulators */
/* Accumulated milliseconds and launch counts since bpc_set_timing(ctx, 1); synchronizes. */
bpc_status bpc_get_timing(bpc_ctx* ctx, float ms[BPC_NUM_TIMERS], uint32_t count[BPC_NUM_TIMERS]);
/* Number of libbpc kernels launched since init (for the bench's gpu_launches). */
uint64_t bpc_launch_count(const bpc_ctx* ctx);

const char* bpc_status_string(bpc_status s);
const char* bpc_last_error(const bpc_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
