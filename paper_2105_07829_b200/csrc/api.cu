// api.cu — the libbpc C ABI (include/bpc.h): validation, chunk plan, owner map,
// buffers, the NCCL exchange and the kernel launches of one step.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "bpc.h"
#include "kernels.h"
#include "nvls.h"

#include <unistd.h>

#include <memory>

namespace {
using namespace bpc;

constexpr uint64_t kSlice = 16384;   // == SLICE of the cluster kernels
constexpr uint32_t kStreamSlice = 8192;   // == CSL of the streaming kernels

// compressors whose worker step runs in the streaming kernel (unit norm, no selection)
bool stream_worker(int kind) {
  return kind == BPC_NONE || kind == BPC_SCALED_SIGN || kind == BPC_LINEAR_DITHER || kind == BPC_NATURAL_DITHER;
}

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct PlanChunk {
  bpc_chunk_info info;
};

struct Plan {
  std::vector<bpc_chunk_info> chunks;
  uint32_t cs = 16;
  uint64_t D = 0;
  std::vector<uint64_t> seg_off, seg_bytes;   // per peer segment of SEND / P
  uint64_t send_bytes = 0, etl_elems = 0, payload_total = 0;
  uint32_t num_compressed = 0, num_owned = 0;
};

// k = max(1, floor(L * num / den))  (R8)
uint64_t sparse_k(const bpc_compressor& c, uint64_t L) {
  const uint64_t k = (L * (uint64_t)c.k_num) / (uint64_t)c.k_den;
  return k < 1 ? 1 : k;
}

// closed-form payload sizes
uint64_t payload_size(const bpc_compressor& c, bool raw, uint64_t L) {
  if (raw || c.kind == BPC_NONE) return 4 * L;
  switch (c.kind) {
    case BPC_SCALED_SIGN: return 4 + (L + 7) / 8;
    case BPC_TOP_K:
    case BPC_RANDOM_K: return 8 + (c.f16_values ? 6 : 8) * sparse_k(c, L);
    case BPC_LINEAR_DITHER:
    case BPC_NATURAL_DITHER: return 4 + ((uint64_t)c.bits * L + 7) / 8;
  }
  return 0;
}

bpc_status make_plan(const bpc_config* cfg, Plan* P, std::string* err) {
  auto fail = [&](bpc_status s, const char* msg) {
    *err = msg;
    return s;
  };
  if (!cfg) return fail(BPC_ERR_INVALID_ARGUMENT, "cfg is NULL");
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size)
    return fail(BPC_ERR_INVALID_ARGUMENT, "bad world_size / rank");
  if (cfg->num_tensors < 1 || !cfg->tensor_numel || !cfg->tensor_offset)
    return fail(BPC_ERR_INVALID_ARGUMENT, "no tensors");
  const bpc_compressor& C = cfg->comp;
  switch (C.kind) {
    case BPC_NONE: case BPC_SCALED_SIGN: break;
    case BPC_TOP_K: case BPC_RANDOM_K:
      if (C.k_num < 1 || C.k_den < 1) return fail(BPC_ERR_INVALID_ARGUMENT, "k_num/k_den must be >= 1");
      if (C.k_num > C.k_den) return fail(BPC_ERR_K_TOO_LARGE, "k fraction > 1");
      break;
    case BPC_LINEAR_DITHER: case BPC_NATURAL_DITHER:
      if (C.bits < 2 || C.bits > 8) return fail(BPC_ERR_INVALID_ARGUMENT, "dither bits must be 2..8");
      break;
    default: return fail(BPC_ERR_UNSUPPORTED_KIND, "unknown compressor kind");
  }
  if (C.f16_values != 0 && !(C.f16_values == 1 && (C.kind == BPC_TOP_K || C.kind == BPC_RANDOM_K)))
    return fail(BPC_ERR_INVALID_ARGUMENT, "f16_values is 0 or 1, and 1 only for top-k / random-k");
  if (!(cfg->beta1 > 0.f && cfg->beta1 < 1.f && cfg->beta2 > 0.f && cfg->beta2 < 1.f))
    return fail(BPC_ERR_INVALID_ARGUMENT, "betas must lie in (0, 1)");
  if (!(cfg->eps >= 0.f) || !(cfg->weight_decay >= 0.f))
    return fail(BPC_ERR_INVALID_ARGUMENT, "eps and weight_decay must be >= 0");
  if (cfg->exchange != BPC_EXCHANGE_P2P && cfg->exchange != BPC_EXCHANGE_NCCL && cfg->exchange != BPC_EXCHANGE_NVLS)
    return fail(BPC_ERR_INVALID_ARGUMENT, "unknown exchange mode");
  if (cfg->optimizer != BPC_OPT_ADAM && cfg->optimizer != BPC_OPT_LANS && cfg->optimizer != BPC_OPT_NAG)
    return fail(BPC_ERR_INVALID_ARGUMENT, "unknown optimizer");
  if (cfg->optimizer == BPC_OPT_NAG && !(cfg->momentum >= 0.f && cfg->momentum < 1.f))
    return fail(BPC_ERR_INVALID_ARGUMENT, "NAG momentum must lie in [0, 1)");
  if (cfg->optimizer == BPC_OPT_LANS && !(cfg->lans_alpha_l > 0.f && cfg->lans_alpha_l <= cfg->lans_alpha_u))
    return fail(BPC_ERR_INVALID_ARGUMENT, "LANS needs 0 < alpha_l <= alpha_u");
  if (cfg->unit_mode != 0 && cfg->unit_mode != 1) return fail(BPC_ERR_INVALID_ARGUMENT, "unit_mode is 0 or 1");
  uint64_t ce = cfg->chunk_elems ? cfg->chunk_elems : (1ull << 18);
  if (ce < kSlice || ce > 16 * kSlice || (ce & (ce - 1)))
    return fail(BPC_ERR_INVALID_ARGUMENT, "chunk_elems must be a power of two in [2^14, 2^18]");
  P->cs = (uint32_t)(ce / kSlice);
  // tensors: numel >= 1, offsets 16-byte aligned, disjoint
  std::vector<std::pair<uint64_t, uint64_t>> iv;
  P->D = 0;
  for (uint32_t t = 0; t < cfg->num_tensors; t++) {
    const uint64_t L = cfg->tensor_numel[t], o = cfg->tensor_offset[t];
    if (L == 0) return fail(BPC_ERR_EMPTY_BLOCK, "tensor with numel 0");
    if (L >= (1ull << 31)) return fail(BPC_ERR_INVALID_ARGUMENT, "tensor numel >= 2^31");
    if (cfg->unit_mode == 1 && stream_worker(C.kind) && L > (uint64_t)kStreamSlice * UNIT_MAX_SLICES)
      return fail(BPC_ERR_INVALID_ARGUMENT, "per-tensor unit of a norm-based kind larger than 2^27 elements");
    if (cfg->optimizer == BPC_OPT_LANS && L > 4096ull * LANS_MAX_TILES)
      return fail(BPC_ERR_INVALID_ARGUMENT, "LANS block (tensor) larger than 2^25 elements");
    if (o % 4) return fail(BPC_ERR_INVALID_ARGUMENT, "tensor offsets must be multiples of 4 elements");
    iv.push_back({o, o + L});
    P->D = std::max(P->D, o + L);
  }
  std::sort(iv.begin(), iv.end());
  for (size_t i = 1; i < iv.size(); i++)
    if (iv[i].first < iv[i - 1].second) return fail(BPC_ERR_SIZE_MISMATCH, "tensors overlap");
  // chunk plan: raw below threshold (R3), else units of chunk_elems (R1)
  P->chunks.clear();
  P->num_compressed = 0;
  for (uint32_t t = 0; t < cfg->num_tensors; t++) {
    const uint64_t L = cfg->tensor_numel[t];
    const bool raw = (4 * L < cfg->size_threshold_bytes) || C.kind == BPC_NONE;
    const uint64_t unit = (raw || cfg->unit_mode == 1) ? L : ce;   // per-tensor units
    for (uint64_t s = 0; s < L; s += unit) {
      bpc_chunk_info ci = {};
      ci.tensor = t;
      ci.raw = raw;
      ci.offset = cfg->tensor_offset[t] + s;
      ci.len = std::min(unit, L - s);
      ci.k = (!raw && (C.kind == BPC_TOP_K || C.kind == BPC_RANDOM_K)) ? (uint32_t)sparse_k(C, ci.len) : 0;
      ci.payload_bytes = payload_size(C, raw, ci.len);
      P->chunks.push_back(ci);
      if (!raw) P->num_compressed++;
    }
  }
  // owner map: LPT (largest first) over the server cost model
  const uint32_t n = (uint32_t)cfg->world_size;
  std::vector<std::pair<uint64_t, uint32_t>> cost;
  for (uint32_t c = 0; c < P->chunks.size(); c++) {
    const auto& ci = P->chunks[c];
    const uint64_t pb = ci.payload_bytes;
    const uint64_t w = ci.raw ? (4 * n * ci.len + 4 * ci.len) : (n * pb + 8 * ci.len * (C.use_ef ? 1 : 0) + pb);
    cost.push_back({w, c});
  }
  std::sort(cost.begin(), cost.end(), [](auto a, auto b) {
    return a.first != b.first ? a.first > b.first : a.second < b.second;
  });
  std::vector<uint64_t> load(n, 0);
  for (auto& wc : cost) {
    uint32_t best = 0;
    for (uint32_t r = 1; r < n; r++)
      if (load[r] < load[best]) best = r;
    load[best] += wc.first;
    P->chunks[wc.second].owner = best;
  }
  // payload layout grouped by owner, 16-byte slots with >= 4 spare bytes
  P->seg_off.assign(n, 0);
  P->seg_bytes.assign(n, 0);
  P->payload_total = 0;
  uint64_t off = 0;
  for (uint32_t r = 0; r < n; r++) {
    P->seg_off[r] = off;
    for (auto& ci : P->chunks) {
      if (ci.owner != r) continue;
      ci.payload_offset = off;
      ci.recv_offset = off - P->seg_off[r];
      off += round_up(ci.payload_bytes + 4, 16);
      P->payload_total += ci.payload_bytes;
    }
    P->seg_bytes[r] = off - P->seg_off[r];
  }
  P->send_bytes = off;
  // compact server error for the owned compressed chunks
  P->etl_elems = 0;
  P->num_owned = 0;
  for (auto& ci : P->chunks) {
    if (ci.owner != (uint32_t)cfg->rank) continue;
    P->num_owned++;
    if (!ci.raw && C.use_ef) {
      ci.server_err_offset = P->etl_elems;
      P->etl_elems += round_up(ci.len, 4);
    }
  }
  return BPC_OK;
}

void fill_summary(const Plan& P, int rank, bpc_plan_summary* s) {
  s->num_chunks = (uint32_t)P.chunks.size();
  s->num_compressed = P.num_compressed;
  s->num_owned = P.num_owned;
  s->cluster_ctas = P.cs;
  s->flat_elems = P.D;
  s->send_bytes = P.send_bytes;
  s->recv_slot_bytes = P.seg_bytes[rank];
  s->server_err_elems = P.etl_elems;
  s->payload_total = P.payload_total;
}

}  // namespace

struct bpc_ctx {
  bpc_config cfg;
  std::vector<uint64_t> numel, offset;
  Plan plan;
  cudaStream_t stream = nullptr;
  float *e = nullptr, *etl = nullptr, *m = nullptr, *v = nullptr;
  uint8_t *send = nullptr, *recv = nullptr, *pbuf = nullptr;
  uint64_t recv_bytes = 0;
  DevChunk* d_chunks = nullptr;
  uint32_t *d_witems = nullptr, *d_sitems = nullptr;
  Tile* d_utiles = nullptr;
  uint2* d_ent = nullptr;     // sparse kinds: payload entries per 2048-element half tile
  uint32_t n_witems = 0, n_sitems = 0, n_utiles = 0;
  // sparse kinds (kernels_sparse.cu), per side (0 worker, 1 server): chunk -> unit,
  // candidate thresholds, counters, candidate lists
  uint32_t* d_chunk2u[2] = {nullptr, nullptr};
  uint32_t* d_guess[2] = {nullptr, nullptr};
  uint32_t* d_scnt[2] = {nullptr, nullptr};         // candidates per slice (streaming pass)
  uint32_t* d_first_slice[2] = {nullptr, nullptr};  // per unit: its first slice
  uint2* d_cand[2] = {nullptr, nullptr};
  uint32_t* d_cand_off[2] = {nullptr, nullptr};
  uint32_t sel_cap[2] = {0, 0};                  // CTA select kernel: candidates in shared memory
  uint32_t* d_big[2] = {nullptr, nullptr};       // units handed from the warp to the CTA select
  uint2* d_apply_blk = nullptr;                  // server: 256-entry blocks of the ranks' entries
  uint32_t n_apply_blk = 0;
  // per-tensor units longer than SEL_LMAX, per side: the large-unit select path
  uint32_t* d_large_units[2] = {nullptr, nullptr};
  uint2* d_lslices[2] = {nullptr, nullptr};
  uint32_t* d_lslice_first[2] = {nullptr, nullptr};
  uint32_t* d_lstate[2] = {nullptr, nullptr};
  uint32_t* d_lhist[2] = {nullptr, nullptr};
  uint2* d_lcnt[2] = {nullptr, nullptr};
  uint2* d_loff[2] = {nullptr, nullptr};
  uint32_t n_large[2] = {0, 0}, n_lslices[2] = {0, 0};
  float* d_sdelta = nullptr;   // server Delta of the owned units (sparse kinds without EF)
  unsigned int* d_flag = nullptr;
  // streaming worker (norm-based compressors): slices, partials, unit counters
  Slice* d_wslices = nullptr;
  uint32_t n_wslices = 0;
  double* d_wpartials = nullptr;
  unsigned long long* d_wcounters = nullptr;
  // streaming server (owned units)
  Slice* d_sslices = nullptr;
  uint32_t n_sslices = 0;
  double* d_spartials = nullptr;
  unsigned long long* d_scounters = nullptr;
  int num_sms = 148;
  ncclComm_t comm = nullptr;
  // peer-memory exchange (BPC_EXCHANGE_P2P): peers' IPC-mapped RECV / P / flags
  int32_t exchange = BPC_EXCHANGE_NCCL;
  unsigned long long* d_xflags = nullptr;   // [2n]: push slots [0, n), pull slots [n, 2n)
  std::vector<uint8_t*> peer_recv, peer_p;
  std::vector<unsigned long long*> peer_flags;
  bool local_group = false;   // bpc_connect_local: peers are contexts of this process (direct pointers)
  // BPC_EXCHANGE_NVLS: P bound to a multicast object (nvls.cu); the server
  // stores p through pbuf_mc, every rank reads it from its own P
  bool nvls = false;
  bool nvls_copy = false;            // the multicast by a copy kernel after the server (else in the server)
  NvlsMap nv;
  std::shared_ptr<uint64_t> nv_mc;   // the multicast handle (released with the last reference)
  uint8_t* pbuf_mc = nullptr;
  uint8_t* pbuf_cm = nullptr;        // the cudaMalloc'd P the NVLS one replaced
  uint8_t uid[128] = {};             // the NCCL unique id (names the handle socket)
  // LANS (BPC_OPT_LANS): per update tile partial sums, per block coefficients
  double* d_lans_part = nullptr;
  // per-tensor units (unit_mode 1): per side, unit tables and totals
  uint32_t *d_wufirst = nullptr, *d_wuns = nullptr, *d_sufirst = nullptr, *d_suns = nullptr;
  double *d_wutotal = nullptr, *d_sutotal = nullptr;
  uint32_t n_wunits = 0, n_sunits = 0;
  float2* d_lans_coef = nullptr;
  uint32_t* d_blk_tile = nullptr;
  int push_grid = 1, pull_grid = 1;
  // device-side step state: the step counter t and the launch / exchange epochs
  // live in HBM and advance inside the kernels, so a captured step replays
  DevState* d_st = nullptr;
  float4* d_bct = nullptr;   // bias corrections per step (R16), see BiasTab
  uint32_t nbct = 0;
  int32_t bconv = 0;
  int phase = 0;   // 0 compress, 1 push, 2 server, 3 pull, 4 step
  bool timing = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> events;
  uint64_t launches = 0;
  std::string err;
};

namespace {

bpc_status cuda_fail(bpc_ctx* c, cudaError_t e, const char* what) {
  if (c) c->err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? BPC_ERR_OUT_OF_MEMORY : BPC_ERR_CUDA;
}
#define CK(call, what)                                 \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, what); \
  } while (0)
#define NK(call, what)                                              \
  do {                                                              \
    ncclResult_t _r = (call);                                       \
    if (_r != ncclSuccess) {                                        \
      ctx->err = std::string(what) + ": " + ncclGetErrorString(_r); \
      return BPC_ERR_NCCL;                                          \
    }                                                               \
  } while (0)

// Every entry point runs on the context's device and restores the caller's
// current device on return (a process may drive contexts on several GPUs).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// A caller buffer handed to the kernels: device memory of the context's device
// (or managed), 16-byte aligned (the kernels bulk-copy it with cp.async.bulk).
bpc_status check_user_ptr(bpc_ctx* ctx, const void* p, const char* what) {
  if (!p) {
    ctx->err = std::string(what) + " is NULL";
    return BPC_ERR_INVALID_ARGUMENT;
  }
  if (reinterpret_cast<uintptr_t>(p) & 15u) {
    ctx->err = std::string(what) + " is not 16-byte aligned";
    return BPC_ERR_INVALID_ARGUMENT;
  }
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    ctx->err = std::string(what) + " is not a CUDA pointer";
    return BPC_ERR_INVALID_ARGUMENT;
  }
  const bool ok = a.type == cudaMemoryTypeManaged || (a.type == cudaMemoryTypeDevice && a.device == ctx->cfg.device);
  if (!ok) {
    ctx->err = std::string(what) + " is not device memory of the context's device";
    return BPC_ERR_INVALID_ARGUMENT;
  }
  return BPC_OK;
}

void timer_begin(bpc_ctx* ctx, int id, cudaEvent_t* ev) {
  if (!ctx->timing) return;
  cudaEventCreate(ev);
  cudaEventRecord(*ev, ctx->stream);
  (void)id;
}
void timer_end(bpc_ctx* ctx, int id, cudaEvent_t b) {
  if (!ctx->timing) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, ctx->stream);
  ctx->events.push_back({id, {b, e}});
}

template <class T>
bpc_status upload(bpc_ctx* ctx, T** dst, const std::vector<T>& src) {
  if (src.empty()) return BPC_OK;
  CK(cudaMalloc((void**)dst, sizeof(T) * src.size()), "cudaMalloc table");
  CK(cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice), "upload table");
  return BPC_OK;
}

void free_ctx(bpc_ctx* ctx) {
  if (!ctx) return;
  if (ctx->local_group) {   // direct pointers into the other contexts: nothing to close
    ctx->peer_recv.clear();
    ctx->peer_p.clear();
    ctx->peer_flags.clear();
  }
  for (auto* v : {&ctx->peer_recv, &ctx->peer_p})
    for (int r = 0; r < (int)v->size(); r++)
      if ((*v)[r] && r != ctx->cfg.rank) cudaIpcCloseMemHandle((*v)[r]);
  for (int r = 0; r < (int)ctx->peer_flags.size(); r++)
    if (ctx->peer_flags[r] && r != ctx->cfg.rank) cudaIpcCloseMemHandle(ctx->peer_flags[r]);
  if (ctx->d_xflags) cudaFree(ctx->d_xflags);
  for (void* q : {(void*)ctx->d_lans_part, (void*)ctx->d_lans_coef, (void*)ctx->d_blk_tile,
                  (void*)ctx->d_wufirst, (void*)ctx->d_wuns, (void*)ctx->d_sufirst, (void*)ctx->d_suns,
                  (void*)ctx->d_wutotal, (void*)ctx->d_sutotal})
    if (q) cudaFree(q);
  for (void* q : {(void*)ctx->d_st, (void*)ctx->d_bct})
    if (q) cudaFree(q);
  if (ctx->nvls) {   // P is the unicast mapping of the multicast-bound allocation
    nvls_release(&ctx->nv);
    ctx->nv_mc.reset();
    ctx->pbuf = ctx->pbuf_cm;
  }
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (void* p : {(void*)ctx->e, (void*)ctx->etl, (void*)ctx->m, (void*)ctx->v, (void*)ctx->send,
                  (void*)ctx->pbuf, (void*)ctx->d_chunks, (void*)ctx->d_witems, (void*)ctx->d_sitems,
                  (void*)ctx->d_utiles, (void*)ctx->d_ent, (void*)ctx->d_flag, (void*)ctx->d_sdelta,
                  (void*)ctx->d_chunk2u[0], (void*)ctx->d_chunk2u[1], (void*)ctx->d_guess[0], (void*)ctx->d_guess[1],
                  (void*)ctx->d_scnt[0], (void*)ctx->d_scnt[1], (void*)ctx->d_first_slice[0],
                  (void*)ctx->d_first_slice[1], (void*)ctx->d_cand[0], (void*)ctx->d_cand[1],
                  (void*)ctx->d_cand_off[0], (void*)ctx->d_cand_off[1], (void*)ctx->d_big[0], (void*)ctx->d_big[1],
                  (void*)ctx->d_apply_blk, (void*)ctx->d_large_units[0], (void*)ctx->d_large_units[1],
                  (void*)ctx->d_lslices[0], (void*)ctx->d_lslices[1], (void*)ctx->d_lslice_first[0],
                  (void*)ctx->d_lslice_first[1], (void*)ctx->d_lstate[0], (void*)ctx->d_lstate[1],
                  (void*)ctx->d_lhist[0], (void*)ctx->d_lhist[1], (void*)ctx->d_lcnt[0], (void*)ctx->d_lcnt[1],
                  (void*)ctx->d_loff[0], (void*)ctx->d_loff[1],
                  (void*)ctx->d_wslices, (void*)ctx->d_wpartials, (void*)ctx->d_wcounters,
                  (void*)ctx->d_sslices, (void*)ctx->d_spartials, (void*)ctx->d_scounters})
    if (p) cudaFree(p);
  if (ctx->recv && ctx->recv != ctx->send) cudaFree(ctx->recv);
  for (auto& ev : ctx->events) {
    cudaEventDestroy(ev.second.first);
    cudaEventDestroy(ev.second.second);
  }
  delete ctx;
}

// The peer arrays are filled (peers' RECV / P / flags): switch to the P2P
// exchange and size the copy grids of the sparse kinds' exchange kernels.
void finish_p2p(bpc_ctx* ctx) {
  const int n = ctx->cfg.world_size, rank = ctx->cfg.rank;
  const Plan& P = ctx->plan;
  ctx->exchange = BPC_EXCHANGE_P2P;
  ctx->peer_recv[rank] = ctx->recv;
  ctx->peer_p[rank] = ctx->pbuf;
  ctx->peer_flags[rank] = ctx->d_xflags;
  // copy grids: one 32 KB round (512 threads x 4 x 16 B) per CTA, <= 2 CTAs per SM
  auto grid_for = [&](uint64_t bytes) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(2ull * ctx->num_sms, (bytes + 32767) / 32768));
  };
  ctx->push_grid = grid_for(P.send_bytes);
  ctx->pull_grid = grid_for((uint64_t)(n - 1) * P.seg_bytes[rank]);
}

// BPC_EXCHANGE_P2P setup (collective over all ranks, after the communicator
// exists): export RECV, P and the flag array as CUDA IPC handles, all-gather
// them over NCCL, open the peers' handles, and agree (all-reduce min) that every
// rank could open all of them.  Any failure leaves the context on NCCL.
// min over ranks of v (NCCL all-reduce on the context's stream); false if the
// collective itself failed
bool agree_min(bpc_ctx* ctx, int32_t* v) {
  int32_t* d = nullptr;
  bool ok = cudaMalloc((void**)&d, 4) == cudaSuccess && cudaMemcpy(d, v, 4, cudaMemcpyHostToDevice) == cudaSuccess &&
            ncclAllReduce(d, d, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream) == ncclSuccess &&
            cudaStreamSynchronize(ctx->stream) == cudaSuccess && cudaMemcpy(v, d, 4, cudaMemcpyDeviceToHost) == cudaSuccess;
  if (d) cudaFree(d);
  (void)cudaGetLastError();
  return ok;
}

// swap P for the unicast mapping of a multicast-bound allocation
void nvls_adopt(bpc_ctx* ctx, const NvlsMap& m, std::shared_ptr<uint64_t> mc) {
  ctx->nvls = true;
  // default: the server kernel stores p through the multicast mapping itself;
  // BPC_NVLS_MODE=copy: it writes the local P and one copy kernel multicasts this
  // rank's whole segment with 16-byte multimem stores (measured slower at N = 2:
  // C5 2.458 vs 2.396 ms, C4 1.110 vs 1.006 ms; kept for measurements)
  const char* mode = getenv("BPC_NVLS_MODE");
  ctx->nvls_copy = mode && strcmp(mode, "copy") == 0;
  ctx->nv = m;
  ctx->nv_mc = std::move(mc);
  ctx->pbuf_cm = ctx->pbuf;
  ctx->pbuf = reinterpret_cast<uint8_t*>(m.uc);
  ctx->pbuf_mc = reinterpret_cast<uint8_t*>(m.mc);
  cudaMemset(ctx->pbuf, 0, m.size);
}

std::shared_ptr<uint64_t> mc_ref(uint64_t h) {
  return std::shared_ptr<uint64_t>(new uint64_t(h), [](uint64_t* p) {
    nvls_release_handle(*p);
    delete p;
  });
}

// BPC_EXCHANGE_NVLS between processes (collective): rank 0 creates the multicast
// object and serves its fd over an abstract unix socket named after the NCCL
// unique id; every rank adds its device, then binds and maps its P.  Every
// step is agreed over the communicator: all ranks adopt it or none does.
void setup_nvls_mp(bpc_ctx* ctx) {
  const int n = ctx->cfg.world_size, rank = ctx->cfg.rank, dev = ctx->cfg.device;
  std::string err;
  char tag[48];
  uint64_t h0 = 1469598103934665603ull;   // FNV-1a of the unique id
  for (int i = 0; i < 128; i++) h0 = (h0 ^ ctx->uid[i]) * 1099511628211ull;
  snprintf(tag, sizeof(tag), "%016llx", (unsigned long long)h0);
  int32_t ok = nvls_supported(dev) ? 1 : 0;
  uint64_t size = 0;
  if (ok && !nvls_size(n, dev, ctx->plan.send_bytes, &size, &err)) ok = 0;
  if (!agree_min(ctx, &ok) || !ok) return;
  uint64_t mc = 0;
  int fd = -1, lsock = -1;
  if (rank == 0) {
    ok = nvls_create(n, size, &mc, &err) && nvls_export(mc, &fd, &err) && (lsock = fd_listen(tag, &err)) >= 0;
  }
  if (!agree_min(ctx, &ok) || !ok) {   // rank 0 is listening (or nobody proceeds)
    if (lsock >= 0) close(lsock);
    if (fd >= 0) close(fd);
    if (mc) nvls_release_handle(mc);
    return;
  }
  if (rank == 0) {
    ok = fd_serve(lsock, fd, n - 1, &err) ? 1 : 0;
    close(lsock);
    close(fd);
  } else {
    fd = fd_fetch(tag, 30.0, &err);
    ok = fd >= 0 && nvls_import(fd, &mc, &err);
    if (fd >= 0) close(fd);
  }
  std::shared_ptr<uint64_t> ref = mc ? mc_ref(mc) : nullptr;
  if (ok && !nvls_add_device(mc, dev, &err)) ok = 0;
  if (!agree_min(ctx, &ok) || !ok) return;   // every device added before any bind
  NvlsMap m;
  if (!nvls_bind_map(mc, dev, size, &m, &err)) ok = 0;
  int32_t all = ok;
  if (!agree_min(ctx, &all) || !all) {
    nvls_release(&m);
    if (!err.empty()) ctx->err = "NVLS setup: " + err;
    return;
  }
  nvls_adopt(ctx, m, ref);
}

bpc_status setup_p2p(bpc_ctx* ctx) {
  const int n = ctx->cfg.world_size, rank = ctx->cfg.rank;
  const Plan& P = ctx->plan;
  cudaError_t ce;
  // the multicast pull (fused kinds only: the sparse kinds' copy kernels write
  // into the peers' P)
  if (ctx->cfg.exchange == BPC_EXCHANGE_NVLS && stream_worker(ctx->cfg.comp.kind)) setup_nvls_mp(ctx);
  CK(cudaMalloc((void**)&ctx->d_xflags, 16ull * n), "alloc exchange flags");
  CK(cudaMemset(ctx->d_xflags, 0, 16ull * n), "zero exchange flags");
  struct Rec {
    cudaIpcMemHandle_t h[3];
    int32_t ok;
    int32_t pad[3];
  };
  Rec mine = {};
  mine.ok = n <= P2P_MAXJ;
  // (with NVLS nobody reads a peer's P: it is not exported, and a VMM allocation
  // could not be)
  void* bufs[3] = {ctx->recv, ctx->nvls ? nullptr : ctx->pbuf, ctx->d_xflags};
  for (int i = 0; i < 3 && mine.ok; i++)
    if (bufs[i] && cudaIpcGetMemHandle(&mine.h[i], bufs[i]) != cudaSuccess) mine.ok = 0;
  (void)cudaGetLastError();
  uint8_t* d_all = nullptr;
  int32_t* d_ok = nullptr;
  CK(cudaMalloc((void**)&d_all, sizeof(Rec) * n), "alloc handle exchange");
  CK(cudaMalloc((void**)&d_ok, 4), "alloc handle exchange");
  std::vector<Rec> all(n);
  bpc_status st = BPC_OK;
  int32_t ok = 0;
  do {
    if ((ce = cudaMemcpy(d_all + sizeof(Rec) * rank, &mine, sizeof(Rec), cudaMemcpyHostToDevice)) != cudaSuccess) {
      st = cuda_fail(ctx, ce, "handle upload");
      break;
    }
    ncclResult_t r = ncclAllGather(d_all + sizeof(Rec) * rank, d_all, sizeof(Rec), ncclUint8, ctx->comm, ctx->stream);
    if (r != ncclSuccess || (ce = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) {
      ctx->err = "IPC handle all-gather failed";
      st = BPC_ERR_NCCL;
      break;
    }
    if ((ce = cudaMemcpy(all.data(), d_all, sizeof(Rec) * n, cudaMemcpyDeviceToHost)) != cudaSuccess) {
      st = cuda_fail(ctx, ce, "handle download");
      break;
    }
    ok = 1;
    for (int q = 0; q < n; q++) ok &= all[q].ok;
    ctx->peer_recv.assign(n, nullptr);
    ctx->peer_p.assign(n, nullptr);
    ctx->peer_flags.assign(n, nullptr);
    for (int q = 0; q < n && ok; q++) {
      if (q == rank) continue;
      void* ptr[3] = {nullptr, nullptr, nullptr};
      for (int i = 0; i < 3 && ok; i++)
        if ((i != 1 || !ctx->nvls) &&
            cudaIpcOpenMemHandle(&ptr[i], all[q].h[i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
          ok = 0;
      ctx->peer_recv[q] = (uint8_t*)ptr[0];
      ctx->peer_p[q] = (uint8_t*)ptr[1];
      ctx->peer_flags[q] = (unsigned long long*)ptr[2];
    }
    (void)cudaGetLastError();
    // every rank must take the same transport
    if ((ce = cudaMemcpy(d_ok, &ok, 4, cudaMemcpyHostToDevice)) != cudaSuccess) {
      st = cuda_fail(ctx, ce, "agreement upload");
      break;
    }
    r = ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream);
    if (r != ncclSuccess || cudaStreamSynchronize(ctx->stream) != cudaSuccess ||
        cudaMemcpy(&ok, d_ok, 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
      ctx->err = "transport agreement failed";
      st = BPC_ERR_NCCL;
      break;
    }
  } while (0);
  cudaFree(d_all);
  cudaFree(d_ok);
  if (st != BPC_OK) return st;
  if (ok) finish_p2p(ctx);
  return BPC_OK;
}

// The exchange is fused into the streaming kernels (worker stores into the
// owners' RECV, server into every rank's P) for the norm-based kinds; the
// sparse kinds use the copy kernels in bpc_exchange_push / pull.
bool fused_exchange(const bpc_ctx* ctx) {
  return ctx->exchange == BPC_EXCHANGE_P2P && stream_worker(ctx->cfg.comp.kind);
}
// launch bookkeeping of one kernel of family `fam` (EP_*): epochs and the step
// counter are read and advanced on the device (DevState)
PeerSync peer_sync(const bpc_ctx* ctx, int fam) {
  PeerSync s = {};
  s.st = ctx->d_st;
  s.fam = fam;
  s.wait_fam = -1;
  s.sig_fam = -1;
  s.n = (uint32_t)ctx->cfg.world_size;
  s.self = (uint32_t)ctx->cfg.rank;
  return s;
}
// wait for exchange family `fam` (EP_PUSH: slots [0, n); EP_PULL: [n, 2n)) in
// this rank's flag array
void set_wait(const bpc_ctx* ctx, PeerSync* s, int fam) {
  s->wait_fam = fam;
  s->wflags = ctx->d_xflags;
  s->wslot0 = fam == EP_PUSH ? 0u : (uint32_t)ctx->cfg.world_size;
}
// release exchange family `fam` into this rank's slot of every peer's flag array
void set_signal(const bpc_ctx* ctx, PeerSync* s, int fam) {
  const int n = ctx->cfg.world_size, rank = ctx->cfg.rank;
  s->sig_fam = fam;
  for (int r = 0; r < n; r++) s->sflag[r] = r == rank ? nullptr : ctx->peer_flags[r];
  s->sslot = (uint32_t)((fam == EP_PUSH ? 0 : n) + rank);
}

// Streaming worker / server launch: one pass, or (per-tensor units) partials,
// unit tree, then the emitting pass
cudaError_t launch_stream_side(bpc_ctx* ctx, bool server, StreamParams& q) {
  const int kind = ctx->cfg.comp.kind;
  auto go = [&]() { return server ? launch_server_stream(kind, q, ctx->num_sms, ctx->stream)
                                  : launch_worker_stream(kind, q, ctx->num_sms, ctx->stream); };
  if (ctx->cfg.unit_mode != 1) {
    q.pass = 0;
    ctx->launches++;
    return go();
  }
  UnitTreeParams ut = {};
  ut.part = q.partials;
  ut.first = server ? ctx->d_sufirst : ctx->d_wufirst;
  ut.ns = server ? ctx->d_suns : ctx->d_wuns;
  ut.nunits = server ? ctx->n_sunits : ctx->n_wunits;
  ut.total = server ? ctx->d_sutotal : ctx->d_wutotal;
  q.pass = 1;
  const int sig = q.sync.sig_fam;   // the exchange is released by pass 2 only
  q.sync.sig_fam = -1;
  cudaError_t e = go();
  if (e == cudaSuccess) e = launch_unit_tree(ut, ctx->stream);
  q.pass = 2;
  q.sync.sig_fam = sig;
  q.unit_total = ut.total;
  if (e == cudaSuccess) e = go();
  ctx->launches += 3;
  return e;
}

// sparse kinds, one side: prep (server entries, candidate threshold), the
// streaming pass (cstream_kernel<C_TOPK / C_RANDK>: q / Delta, candidates, raw
// units), then the exact selection and payload (kernels_sparse.cu)
bpc_status launch_sparse_side(bpc_ctx* ctx, const SparseParams& p, const float* d_grad) {
  const int kind = ctx->cfg.comp.kind;
  CK(launch_sparse_prep(kind, p, ctx->stream), "sparse prep launch");
  StreamParams q = {};
  q.grad = d_grad;
  q.err = p.vals;
  q.out = p.out;
  q.recv = p.recv;
  q.slot_bytes = p.slot_bytes;
  q.chunks = ctx->d_chunks;
  q.slices = p.slices;
  q.n_slices = p.n_slices;
  q.partials = p.server ? ctx->d_spartials : ctx->d_wpartials;
  q.counters = p.server ? ctx->d_scounters : ctx->d_wcounters;
  q.n = p.n;
  q.inv_n = p.inv_n;
  q.rank = p.server ? 0u : (uint32_t)ctx->cfg.rank;
  q.stage = p.stage;
  q.seed = p.seed;
  q.bits = 1;
  q.use_ef = p.use_ef;
  q.check_finite = p.server ? 0 : p.check_finite;
  q.flag = ctx->d_flag;
  q.sync = peer_sync(ctx, p.server ? EP_SERVER : EP_WORKER);
  q.sp_chunk2u = p.chunk2u;
  q.sp_guess = p.guess;
  q.sp_scnt = p.scnt;
  q.sp_cand = p.cand;
  q.sp_cand_off = p.cand_off;
  cudaError_t e = p.server ? launch_server_stream(kind, q, ctx->num_sms, ctx->stream)
                           : launch_worker_stream(kind, q, ctx->num_sms, ctx->stream);
  CK(e, "sparse streaming launch");
  CK(launch_sparse_select(kind, p, ctx->stream), "sparse select launch");
  ctx->launches += 4;
  return BPC_OK;
}

SparseParams sparse_params(bpc_ctx* ctx, int side) {
  SparseParams p = {};
  p.chunks = ctx->d_chunks;
  p.items = side ? ctx->d_sitems : ctx->d_witems;
  p.n_units = side ? ctx->n_sitems : ctx->n_witems;
  p.slices = side ? ctx->d_sslices : ctx->d_wslices;
  p.n_slices = side ? ctx->n_sslices : ctx->n_wslices;
  p.chunk2u = ctx->d_chunk2u[side];
  p.guess = ctx->d_guess[side];
  p.scnt = ctx->d_scnt[side];
  p.first_slice = ctx->d_first_slice[side];
  p.cand = ctx->d_cand[side];
  p.cand_off = ctx->d_cand_off[side];
  p.n = (uint32_t)ctx->cfg.world_size;
  p.inv_n = 1.0 / (double)ctx->cfg.world_size;
  p.st = ctx->d_st;
  p.stage = side ? 1u : 0u;
  p.rrank = side ? 0u : (uint32_t)ctx->cfg.rank;
  p.seed = ctx->cfg.seed;
  p.server = side;
  p.randk_scaled = ctx->cfg.comp.randk_scaled;
  p.use_ef = ctx->cfg.comp.use_ef;
  p.f16 = ctx->cfg.comp.f16_values;
  p.check_finite = ctx->cfg.check_finite;
  p.flag = ctx->d_flag;
  p.sel_cap = ctx->sel_cap[side];
  p.big = ctx->d_big[side];
  p.apply_blk = ctx->d_apply_blk;
  p.n_apply_blk = side ? ctx->n_apply_blk : 0;
  p.large_units = ctx->d_large_units[side];
  p.n_large = ctx->n_large[side];
  p.lslices = ctx->d_lslices[side];
  p.n_lslices = ctx->n_lslices[side];
  p.lslice_first = ctx->d_lslice_first[side];
  p.lstate = ctx->d_lstate[side];
  p.lhist = ctx->d_lhist[side];
  p.lcnt = ctx->d_lcnt[side];
  p.loff = ctx->d_loff[side];
  p.large_grid = 2u * (uint32_t)ctx->num_sms;
  return p;
}

}  // namespace

extern "C" {

const char* bpc_status_string(bpc_status s) {
  switch (s) {
    case BPC_OK: return "ok";
    case BPC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case BPC_ERR_SIZE_MISMATCH: return "size mismatch";
    case BPC_ERR_EMPTY_BLOCK: return "empty block";
    case BPC_ERR_K_TOO_LARGE: return "k too large";
    case BPC_ERR_UNSUPPORTED_KIND: return "unsupported compressor kind";
    case BPC_ERR_BAD_STATE: return "bad state (call order / mode)";
    case BPC_ERR_NONFINITE: return "non-finite gradient";
    case BPC_ERR_CUDA: return "CUDA error";
    case BPC_ERR_NCCL: return "NCCL error";
    case BPC_ERR_OUT_OF_MEMORY: return "out of device memory";
  }
  return "unknown status";
}

const char* bpc_last_error(const bpc_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

bpc_status bpc_get_unique_id(uint8_t out[128]) {
  if (!out) return BPC_ERR_INVALID_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return BPC_ERR_NCCL;
  static_assert(sizeof(id) == 128, "NCCL unique id size");
  memcpy(out, &id, 128);
  return BPC_OK;
}

bpc_status bpc_plan(const bpc_config* cfg, bpc_plan_summary* summary, bpc_chunk_info* infos, uint32_t cap) {
  Plan P;
  std::string err;
  const bpc_status s = make_plan(cfg, &P, &err);
  if (s != BPC_OK) return s;
  if (summary) fill_summary(P, cfg->rank, summary);
  if (infos)
    for (uint32_t i = 0; i < cap && i < P.chunks.size(); i++) infos[i] = P.chunks[i];
  return BPC_OK;
}

bpc_status bpc_init(const bpc_config* cfg, bpc_ctx** out) {
  if (!out) return BPC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  bpc_ctx* ctx = new bpc_ctx();
  std::string err;
  bpc_status s = make_plan(cfg, &ctx->plan, &err);
  if (s != BPC_OK) {
    delete ctx;
    return s;
  }
  ctx->cfg = *cfg;
  ctx->numel.assign(cfg->tensor_numel, cfg->tensor_numel + cfg->num_tensors);
  ctx->offset.assign(cfg->tensor_offset, cfg->tensor_offset + cfg->num_tensors);
  ctx->cfg.tensor_numel = ctx->numel.data();
  ctx->cfg.tensor_offset = ctx->offset.data();
  ctx->cfg.nccl_unique_id = nullptr;
  ctx->stream = (cudaStream_t)cfg->cuda_stream;
  auto bail = [&](bpc_status st) {
    free_ctx(ctx);
    return st;
  };
  // device: must be sm_100 (no CPU fallback)
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) return bail(BPC_ERR_CUDA);
  DeviceGuard dg(cfg->device);   // restores the caller's device on return
  {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != cfg->device) return bail(BPC_ERR_CUDA);
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10) return bail(BPC_ERR_CUDA);
  const Plan& P = ctx->plan;
  const uint32_t n = (uint32_t)cfg->world_size;
  const uint32_t rank = (uint32_t)cfg->rank;
  const uint64_t D = round_up(P.D, 4);
  auto alloc = [&](void** p, uint64_t bytes) -> cudaError_t {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) e = cudaMemset(*p, 0, bytes);
    return e;
  };
  cudaError_t ce;
  if ((ce = alloc((void**)&ctx->e, 4 * D)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc e"));
  if ((ce = alloc((void**)&ctx->etl, 4 * P.etl_elems)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc e~"));
  if ((ce = alloc((void**)&ctx->m, 4 * D)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc m"));
  if ((ce = alloc((void**)&ctx->v, 4 * D)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc v"));
  if ((ce = alloc((void**)&ctx->send, P.send_bytes)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc send"));
  if ((ce = alloc((void**)&ctx->pbuf, P.send_bytes)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc p"));
  if (n == 1) {
    ctx->recv = ctx->send;   // the worker's payloads are the server's input
    ctx->recv_bytes = P.send_bytes;
  } else {
    ctx->recv_bytes = n * P.seg_bytes[rank];
    if ((ce = alloc((void**)&ctx->recv, ctx->recv_bytes)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc recv"));
  }
  if ((ce = alloc((void**)&ctx->d_flag, 4)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc flag"));
  // step state (t = 1, epochs 0) and the bias-correction table (R16): rows for
  // t = 1.. until both fl32(1 - beta^t) reach 1.0f, at most 2^20 rows
  if ((ce = alloc((void**)&ctx->d_st, sizeof(DevState))) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc step state"));
  {
    const uint32_t one = 1;
    if ((ce = cudaMemcpy(&ctx->d_st->t, &one, 4, cudaMemcpyHostToDevice)) != cudaSuccess)
      return bail(cuda_fail(ctx, ce, "init step state"));
    std::vector<float4> bct;
    const double b1 = (double)cfg->beta1, b2 = (double)cfg->beta2;
    ctx->bconv = 0;
    for (uint32_t t = 1; t <= (1u << 20); t++) {
      float4 r;
      r.x = (float)(1.0 - std::pow(b1, (double)t));
      r.y = (float)(1.0 - std::pow(b2, (double)t));
      r.z = 1.0f / r.x;   // RN(1 / bc): IEEE fp32 division on the host
      r.w = 1.0f / r.y;
      bct.push_back(r);
      if (r.x == 1.0f && r.y == 1.0f) {
        ctx->bconv = 1;
        break;
      }
    }
    ctx->nbct = (uint32_t)bct.size();
    if ((ce = alloc((void**)&ctx->d_bct, 16ull * bct.size())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc bias table"));
    if ((ce = cudaMemcpy(ctx->d_bct, bct.data(), 16ull * bct.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return bail(cuda_fail(ctx, ce, "upload bias table"));
  }
  // device tables
  std::vector<DevChunk> dch(P.chunks.size());
  std::vector<uint32_t> witems, sitems;
  std::vector<Tile> utiles;
  std::vector<uint32_t> blk_tile;   // first update tile of each tensor
  const bool sparse_kind = !stream_worker(cfg->comp.kind);
  uint64_t sd_elems = 0;            // server Delta scratch (sparse kinds without EF)
  for (uint32_t c = 0; c < P.chunks.size(); c++) {
    const auto& ci = P.chunks[c];
    DevChunk& d = dch[c];
    d.off = ci.offset;
    d.pay = ci.payload_offset;
    d.recv = ci.recv_offset;
    d.etl = ci.server_err_offset;
    d.len = (uint32_t)ci.len;
    d.k = ci.k;
    d.id = c;
    d.raw = ci.raw ? 1 : 0;
    d.owner = ci.owner;
    const bool mine = ci.owner == rank;
    if (!ci.raw) {
      witems.push_back(c);
      if (mine) sitems.push_back(c);
      if (mine && sparse_kind && !cfg->comp.use_ef) {   // the server's Delta lives in the scratch
        d.etl = sd_elems;
        sd_elems += round_up(ci.len, 4);
      }
    }
    if (blk_tile.size() <= ci.tensor) blk_tile.resize(ci.tensor + 1, (uint32_t)utiles.size());
    for (uint64_t s0 = 0; s0 < ci.len; s0 += 4096) {
      // pad = block (tensor) index: LANS reduces per block (tiles of a tensor are contiguous)
      Tile tl = {c, (uint32_t)s0, (uint32_t)std::min<uint64_t>(4096, ci.len - s0), ci.tensor};
      utiles.push_back(tl);
    }
  }
  if ((s = upload(ctx, &ctx->d_chunks, dch)) != BPC_OK) return bail(s);
  if ((s = upload(ctx, &ctx->d_witems, witems)) != BPC_OK) return bail(s);
  if ((s = upload(ctx, &ctx->d_sitems, sitems)) != BPC_OK) return bail(s);
  if ((s = upload(ctx, &ctx->d_utiles, utiles)) != BPC_OK) return bail(s);
  if (sparse_kind && (ce = alloc((void**)&ctx->d_ent, 16ull * utiles.size())) != cudaSuccess)
    return bail(cuda_fail(ctx, ce, "alloc entry ranges"));
  ctx->n_witems = (uint32_t)witems.size();
  ctx->n_sitems = (uint32_t)sitems.size();
  if (sparse_kind) {
    // per side: chunk -> unit, and each unit's candidate list: one index-ordered
    // sub-list per 2^13-element slice of cs entries, cs ~ 3x the expected
    // candidates of a slice + 32 (the guess keeps ~1.5-5 k candidates per unit;
    // the server also lists the n ranks' k entries); an overflowing slice sends
    // its unit to the exact whole-unit path
    for (int side = 0; side < 2; side++) {
      const std::vector<uint32_t>& items = side ? sitems : witems;
      std::vector<uint32_t> c2u(P.chunks.size(), 0xffffffffu), off(items.size() + 1, 0), first(items.size(), 0);
      for (uint32_t u = 0; u < items.size(); u++) {
        const auto& ci = P.chunks[items[u]];
        const uint64_t L = ci.len, k = ci.k, ns = (L + kStreamSlice - 1) / kStreamSlice;
        double expect;   // candidates of the unit
        if (cfg->comp.kind == BPC_RANDOM_K) expect = (double)k + 8.0 * std::sqrt((double)k) + 64.0;
        else if (side && !cfg->comp.use_ef) expect = (double)n * k;   // nonzero Delta only
        else expect = (double)sparse_sample_rank((uint32_t)k, (uint32_t)L) * (double)L / 4096.0 + (side ? (double)n * k : 0.0);
        const double per = std::min<double>((double)kStreamSlice, expect * (double)kStreamSlice / (double)L);
        uint64_t cs = L <= 4096 ? L : (uint64_t)std::ceil(3.0 * per + 32.0);
        cs = std::min<uint64_t>(cs, kStreamSlice);
        c2u[items[u]] = u;
        off[u + 1] = off[u] + (uint32_t)(ns * cs);
        if (L <= SEL_LMAX) ctx->sel_cap[side] = std::max<uint32_t>(ctx->sel_cap[side], (uint32_t)std::min<uint64_t>(L, ns * cs));
      }
      // the units' first slices in this side's slice table (same construction as below)
      {
        uint32_t si = 0;
        for (uint32_t c = 0; c < P.chunks.size(); c++) {
          const auto& ci = P.chunks[c];
          if (side == 1 && ci.owner != rank) continue;
          if (c2u[c] != 0xffffffffu) first[c2u[c]] = si;
          si += (uint32_t)((ci.len + kStreamSlice - 1) / kStreamSlice);
        }
        if ((ce = alloc((void**)&ctx->d_scnt[side], 4ull * std::max<uint32_t>(si, 1))) != cudaSuccess)
          return bail(cuda_fail(ctx, ce, "alloc slice counts"));
      }
      // a power of two: the CTA select pads nothing, but the bound keeps its shared
      // memory fixed
      uint32_t sc = 1;
      while (sc < ctx->sel_cap[side]) sc <<= 1;
      ctx->sel_cap[side] = std::min<uint32_t>(sc, SEL_CAP);
      if ((s = upload(ctx, &ctx->d_chunk2u[side], c2u)) != BPC_OK) return bail(s);
      if ((s = upload(ctx, &ctx->d_cand_off[side], off)) != BPC_OK) return bail(s);
      if ((s = upload(ctx, &ctx->d_first_slice[side], first)) != BPC_OK) return bail(s);
      if ((ce = alloc((void**)&ctx->d_guess[side], 4ull * items.size())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc guesses"));
      if ((ce = alloc((void**)&ctx->d_cand[side], 8ull * off.back())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc candidates"));
      if ((ce = alloc((void**)&ctx->d_big[side], 4ull * items.size())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc select flags"));
    }
    if ((ce = alloc((void**)&ctx->d_sdelta, 4ull * sd_elems)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc Delta scratch"));
  }
  ctx->n_utiles = (uint32_t)utiles.size();
  if (cfg->optimizer == BPC_OPT_LANS) {
    blk_tile.push_back((uint32_t)utiles.size());   // [num_tensors + 1]
    if ((s = upload(ctx, &ctx->d_blk_tile, blk_tile)) != BPC_OK) return bail(s);
    if ((ce = alloc((void**)&ctx->d_lans_part, 24ull * utiles.size())) != cudaSuccess)
      return bail(cuda_fail(ctx, ce, "alloc LANS partials"));
    if ((ce = alloc((void**)&ctx->d_lans_coef, 8ull * cfg->num_tensors)) != cudaSuccess)
      return bail(cuda_fail(ctx, ce, "alloc LANS coefficients"));
  }
  // streaming-worker slices: compressed units in 2^13-element slices (multi-slice
  // units combine partials through global memory), raw units as plain tiles
  // (the server's: only the units this rank owns)
  for (int side = 0; side < 2; side++) {
    std::vector<Slice> sl;
    std::vector<uint32_t> ufirst, uns;
    uint32_t units = 0, parts = 0;
    for (uint32_t c = 0; c < P.chunks.size(); c++) {
      const auto& ci = P.chunks[c];
      if (side == 1 && ci.owner != rank) continue;
      const uint32_t L = (uint32_t)ci.len;
      const uint32_t ns = (L + kStreamSlice - 1) / kStreamSlice;
      for (uint32_t s0 = 0, k = 0; s0 < L; s0 += kStreamSlice, k++) {
        Slice x = {c, s0, std::min<uint32_t>(kStreamSlice, L - s0), ci.raw ? 0u : ns, k, units, parts, 0};
        sl.push_back(x);
      }
      if (!ci.raw && ns > 1) {
        ufirst.push_back(parts);
        uns.push_back(ns);
        units++;
        parts += ns;
      }
    }
    Slice** dsl = side ? &ctx->d_sslices : &ctx->d_wslices;
    double** dp = side ? &ctx->d_spartials : &ctx->d_wpartials;
    unsigned long long** dc = side ? &ctx->d_scounters : &ctx->d_wcounters;
    if ((s = upload(ctx, dsl, sl)) != BPC_OK) return bail(s);
    (side ? ctx->n_sslices : ctx->n_wslices) = (uint32_t)sl.size();
    if ((ce = alloc((void**)dp, 8ull * parts)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc partials"));
    if ((ce = alloc((void**)dc, 8ull * units)) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc counters"));
    if (cfg->unit_mode == 1) {
      if ((s = upload(ctx, side ? &ctx->d_sufirst : &ctx->d_wufirst, ufirst)) != BPC_OK) return bail(s);
      if ((s = upload(ctx, side ? &ctx->d_suns : &ctx->d_wuns, uns)) != BPC_OK) return bail(s);
      if ((ce = alloc((void**)(side ? &ctx->d_sutotal : &ctx->d_wutotal), 8ull * units)) != cudaSuccess)
        return bail(cuda_fail(ctx, ce, "alloc unit totals"));
      (side ? ctx->n_sunits : ctx->n_wunits) = units;
    }
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  if (sparse_kind) {
    // server: the ranks' entries in 256-entry blocks (sparse_apply)
    std::vector<uint2> ab;
    for (uint32_t u = 0; u < sitems.size(); u++) {
      const uint64_t ne = (uint64_t)n * P.chunks[sitems[u]].k;
      for (uint64_t f = 0; f < ne; f += 256) ab.push_back(make_uint2(u, (uint32_t)f));
    }
    if ((s = upload(ctx, &ctx->d_apply_blk, ab)) != BPC_OK) return bail(s);
    ctx->n_apply_blk = (uint32_t)ab.size();
    // per side: units longer than SEL_LMAX and their slices (same order as the slice tables)
    for (int side = 0; side < 2; side++) {
      const std::vector<uint32_t>& items = side ? sitems : witems;
      std::vector<uint32_t> lunits, lfirst;
      std::vector<uint2> lsl;
      std::vector<int32_t> lu_of(P.chunks.size(), -1);
      for (uint32_t u = 0; u < items.size(); u++)
        if (P.chunks[items[u]].len > SEL_LMAX) {
          lu_of[items[u]] = (int32_t)lunits.size();
          lunits.push_back(u);
        }
      uint32_t si = 0;
      int32_t cur = -1;
      for (uint32_t c = 0; c < P.chunks.size(); c++) {
        const auto& ci = P.chunks[c];
        if (side == 1 && ci.owner != rank) continue;
        for (uint64_t s0 = 0; s0 < ci.len; s0 += kStreamSlice, si++) {
          if (lu_of[c] < 0) continue;
          if (lu_of[c] != cur) {
            cur = lu_of[c];
            lfirst.push_back((uint32_t)lsl.size());
          }
          lsl.push_back(make_uint2(si, (uint32_t)lu_of[c]));
        }
      }
      lfirst.push_back((uint32_t)lsl.size());
      ctx->n_large[side] = (uint32_t)lunits.size();
      ctx->n_lslices[side] = (uint32_t)lsl.size();
      if (lunits.empty()) continue;
      if ((s = upload(ctx, &ctx->d_large_units[side], lunits)) != BPC_OK) return bail(s);
      if ((s = upload(ctx, &ctx->d_lslices[side], lsl)) != BPC_OK) return bail(s);
      if ((s = upload(ctx, &ctx->d_lslice_first[side], lfirst)) != BPC_OK) return bail(s);
      if ((ce = alloc((void**)&ctx->d_lstate[side], 32ull * lunits.size())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc large state"));
      if ((ce = alloc((void**)&ctx->d_lhist[side], 1024ull * lunits.size())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc large hist"));
      if ((ce = alloc((void**)&ctx->d_lcnt[side], 8ull * lsl.size())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc large counts"));
      if ((ce = alloc((void**)&ctx->d_loff[side], 8ull * lsl.size())) != cudaSuccess) return bail(cuda_fail(ctx, ce, "alloc large offsets"));
    }
  }
  if ((ce = cudaDeviceSynchronize()) != cudaSuccess) return bail(cuda_fail(ctx, ce, "init sync"));
  // NCCL communicator (collective over all ranks)
  if (cfg->nccl_unique_id && n > 1) {
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, 128);
    memcpy(ctx->uid, cfg->nccl_unique_id, 128);
    ncclResult_t r = ncclCommInitRank(&ctx->comm, (int)n, id, (int)rank);
    if (r != ncclSuccess) {
      ctx->comm = nullptr;
      return bail(BPC_ERR_NCCL);
    }
    if ((cfg->exchange == BPC_EXCHANGE_P2P || cfg->exchange == BPC_EXCHANGE_NVLS) && (s = setup_p2p(ctx)) != BPC_OK)
      return bail(s);
  }
  *out = ctx;
  return BPC_OK;
}

bpc_status bpc_connect_local(bpc_ctx* const* ctxs, int32_t n) {
  if (!ctxs || n < 2 || n > P2P_MAXJ) return BPC_ERR_INVALID_ARGUMENT;
  for (int r = 0; r < n; r++) {
    bpc_ctx* c = ctxs[r];
    if (!c) return BPC_ERR_INVALID_ARGUMENT;
    if (c->cfg.world_size != n || c->cfg.rank != r || c->comm || c->local_group || c->phase != 0 ||
        c->launches != 0) {
      c->err = "bpc_connect_local: needs fresh contexts of world_size n, rank r at index r, no NCCL id";
      return BPC_ERR_BAD_STATE;
    }
    const Plan& a = c->plan;
    const Plan& b = ctxs[0]->plan;
    if (a.chunks.size() != b.chunks.size() || a.send_bytes != b.send_bytes || a.seg_bytes != b.seg_bytes) {
      c->err = "bpc_connect_local: the contexts' plans differ";
      return BPC_ERR_SIZE_MISMATCH;
    }
  }
  // peer access between distinct devices (both directions)
  for (int a = 0; a < n; a++)
    for (int b = 0; b < n; b++) {
      const int da = ctxs[a]->cfg.device, db = ctxs[b]->cfg.device;
      if (da == db) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, da, db) != cudaSuccess || !can) {
        ctxs[a]->err = "bpc_connect_local: no peer access between the contexts' devices";
        return BPC_ERR_CUDA;
      }
      DeviceGuard dg(da);
      const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(ctxs[a], e, "peer access");
      (void)cudaGetLastError();
    }
  for (int r = 0; r < n; r++) {
    bpc_ctx* ctx = ctxs[r];
    DeviceGuard dg(ctx->cfg.device);
    if (!ctx->d_xflags) {
      CK(cudaMalloc((void**)&ctx->d_xflags, 16ull * n), "alloc exchange flags");
      CK(cudaMemset(ctx->d_xflags, 0, 16ull * n), "zero exchange flags");
    }
  }
  // BPC_EXCHANGE_NVLS: one multicast object over the group's devices (distinct
  // devices only; otherwise the group keeps the peer reads of p)
  bool want = stream_worker(ctxs[0]->cfg.comp.kind);
  for (int r = 0; r < n && want; r++) {
    want = ctxs[r]->cfg.exchange == BPC_EXCHANGE_NVLS && nvls_supported(ctxs[r]->cfg.device);
    for (int q = 0; q < r && want; q++) want = ctxs[q]->cfg.device != ctxs[r]->cfg.device;
  }
  if (want) {
    std::string err;
    uint64_t size = 0, mc = 0;
    bool ok = nvls_size(n, ctxs[0]->cfg.device, ctxs[0]->plan.send_bytes, &size, &err) &&
              nvls_create(n, size, &mc, &err);
    std::shared_ptr<uint64_t> ref = ok ? mc_ref(mc) : nullptr;
    for (int r = 0; r < n && ok; r++) ok = nvls_add_device(mc, ctxs[r]->cfg.device, &err);
    std::vector<NvlsMap> maps(n);
    for (int r = 0; r < n && ok; r++) {
      DeviceGuard dg(ctxs[r]->cfg.device);
      ok = nvls_bind_map(mc, ctxs[r]->cfg.device, size, &maps[r], &err);
    }
    if (ok) {
      for (int r = 0; r < n; r++) {
        DeviceGuard dg(ctxs[r]->cfg.device);
        nvls_adopt(ctxs[r], maps[r], ref);
      }
    } else {
      for (int r = 0; r < n; r++) nvls_release(&maps[r]);
      ctxs[0]->err = "NVLS setup: " + err;   // informational: the group keeps the peer reads
    }
  }
  for (int r = 0; r < n; r++) {
    bpc_ctx* ctx = ctxs[r];
    ctx->peer_recv.assign(n, nullptr);
    ctx->peer_p.assign(n, nullptr);
    ctx->peer_flags.assign(n, nullptr);
    for (int q = 0; q < n; q++) {
      ctx->peer_recv[q] = ctxs[q]->recv;
      ctx->peer_p[q] = ctxs[q]->pbuf;
      ctx->peer_flags[q] = ctxs[q]->d_xflags;
    }
    ctx->local_group = true;
    finish_p2p(ctx);
  }
  for (int r = 0; r < n; r++) {
    DeviceGuard dg(ctxs[r]->cfg.device);
    bpc_ctx* ctx = ctxs[r];
    CK(cudaDeviceSynchronize(), "connect sync");
  }
  return BPC_OK;
}

bpc_status bpc_compress(bpc_ctx* ctx, const float* d_grad) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  if (ctx->phase != 0) return BPC_ERR_BAD_STATE;
  DeviceGuard dg(ctx->cfg.device);
  if (bpc_status st = check_user_ptr(ctx, d_grad, "d_grad")) return st;
  cudaEvent_t b = nullptr;
  timer_begin(ctx, BPC_TIMER_COMPRESS, &b);
  if (stream_worker(ctx->cfg.comp.kind)) {
    StreamParams q = {};
    q.grad = d_grad;
    q.err = ctx->e;
    q.out = ctx->send;
    q.chunks = ctx->d_chunks;
    q.slices = ctx->d_wslices;
    q.n_slices = ctx->n_wslices;
    q.partials = ctx->d_wpartials;
    q.counters = ctx->d_wcounters;
    q.n = (uint32_t)ctx->cfg.world_size;
    q.inv_n = 1.0 / (double)ctx->cfg.world_size;
    q.rank = (uint32_t)ctx->cfg.rank;
    q.stage = 0;
    q.seed = ctx->cfg.seed;
    q.bits = ctx->cfg.comp.bits;
    q.use_ef = ctx->cfg.comp.use_ef;
    q.check_finite = ctx->cfg.check_finite;
    q.flag = ctx->d_flag;
    q.sync = peer_sync(ctx, EP_WORKER);
    if (fused_exchange(ctx)) {   // fused push: payloads go straight to the owners' RECV slots
      const Plan& P = ctx->plan;
      q.ndst = (uint32_t)ctx->cfg.world_size;
      for (int r = 0; r < ctx->cfg.world_size; r++)
        q.dst[r] = ctx->peer_recv[r] + (uint64_t)ctx->cfg.rank * P.seg_bytes[r];
      set_signal(ctx, &q.sync, EP_PUSH);
    }
    CK(launch_stream_side(ctx, false, q), "worker stream launch");
  } else {
    SparseParams p = sparse_params(ctx, 0);
    p.grad = d_grad;
    p.vals = ctx->e;
    p.out = ctx->send;
    if (bpc_status st = launch_sparse_side(ctx, p, d_grad)) return st;
  }
  timer_end(ctx, BPC_TIMER_COMPRESS, b);
  ctx->phase = 1;
  return BPC_OK;
}

bpc_status bpc_exchange_push(bpc_ctx* ctx) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  if (ctx->phase != 1) return BPC_ERR_BAD_STATE;
  DeviceGuard dg(ctx->cfg.device);
  const int n = ctx->cfg.world_size, rank = ctx->cfg.rank;
  if (n > 1 && (ctx->comm || ctx->local_group) && !fused_exchange(ctx)) {
    const Plan& P = ctx->plan;
    cudaEvent_t b = nullptr;
    timer_begin(ctx, BPC_TIMER_PUSH, &b);
    const uint64_t slot = P.seg_bytes[rank];
    if (ctx->exchange == BPC_EXCHANGE_P2P) {
      // segment r of SEND -> slot `rank` of owner r's RECV (the local one included),
      // then release the push flag on every peer; bpc_server waits for the peers'
      // flags before its first read of RECV
      P2PParams q = {};
      for (int r = 0; r < n; r++) {
        if (!P.seg_bytes[r]) continue;
        q.src[q.njobs] = ctx->send + P.seg_off[r];
        q.dst[q.njobs] = ctx->peer_recv[r] + (uint64_t)rank * P.seg_bytes[r];
        q.len[q.njobs++] = P.seg_bytes[r];
      }
      q.sync = peer_sync(ctx, EP_PUSH);
      set_signal(ctx, &q.sync, EP_PUSH);
      CK(launch_p2p_copy(q, ctx->push_grid, ctx->stream), "push copy launch");
      ctx->launches += 1;
    } else {
      NK(ncclGroupStart(), "group start");
      for (int r = 0; r < n; r++) {
        if (r == rank) continue;
        if (P.seg_bytes[r]) NK(ncclSend(ctx->send + P.seg_off[r], P.seg_bytes[r], ncclUint8, r, ctx->comm, ctx->stream), "send");
        if (slot) NK(ncclRecv(ctx->recv + r * slot, slot, ncclUint8, r, ctx->comm, ctx->stream), "recv");
      }
      NK(ncclGroupEnd(), "group end");
      if (slot) CK(cudaMemcpyAsync(ctx->recv + rank * slot, ctx->send + P.seg_off[rank], slot,
                                   cudaMemcpyDeviceToDevice, ctx->stream), "self copy");
    }
    timer_end(ctx, BPC_TIMER_PUSH, b);
  }
  // n == 1: RECV aliases SEND.  n > 1 without a communicator: the caller performed
  // the exchange through bpc_buffer / bpc_peer_segment (external exchange).
  ctx->phase = 2;
  return BPC_OK;
}

// sparse kinds over the P2P exchange: one warp waits for every peer's release of
// exchange family `fam` (EP_PUSH / EP_PULL) at this rank's own epoch of it
// (advanced by this rank's copy kernel) before the consumer kernel reads
static bpc_status launch_flag_wait(bpc_ctx* ctx, int fam, const char* what) {
  P2PWait w = {};
  const int slot0 = fam == EP_PUSH ? 0 : ctx->cfg.world_size;
  for (int r = 0; r < ctx->cfg.world_size; r++)
    if (r != ctx->cfg.rank) w.slots[w.nslots++] = slot0 + r;
  w.flags = ctx->d_xflags;
  w.st = ctx->d_st;
  w.fam = fam;
  CK(launch_p2p_wait(w, ctx->stream), what);
  ctx->launches++;
  return BPC_OK;
}
static bool sparse_p2p(const bpc_ctx* ctx) {
  return ctx->cfg.world_size > 1 && ctx->exchange == BPC_EXCHANGE_P2P && !fused_exchange(ctx);
}

bpc_status bpc_server(bpc_ctx* ctx) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  if (ctx->phase != 2) return BPC_ERR_BAD_STATE;
  DeviceGuard dg(ctx->cfg.device);
  // n == 1: RECV aliases SEND, recv offsets equal payload offsets (one segment)
  const uint64_t slot = ctx->cfg.world_size == 1 ? 0 : ctx->plan.seg_bytes[ctx->cfg.rank];
  cudaEvent_t b = nullptr;
  timer_begin(ctx, BPC_TIMER_SERVER, &b);
  if (stream_worker(ctx->cfg.comp.kind)) {
    StreamParams q = {};
    q.err = ctx->etl;
    q.out = ctx->pbuf;
    q.recv = ctx->recv;
    q.slot_bytes = slot;
    q.chunks = ctx->d_chunks;
    q.slices = ctx->d_sslices;
    q.n_slices = ctx->n_sslices;
    q.partials = ctx->d_spartials;
    q.counters = ctx->d_scounters;
    q.n = (uint32_t)ctx->cfg.world_size;
    q.inv_n = 1.0 / (double)ctx->cfg.world_size;
    q.rank = 0;
    q.stage = 1;
    q.seed = ctx->cfg.seed;
    q.bits = ctx->cfg.comp.bits;
    q.use_ef = ctx->cfg.comp.use_ef;
    q.flag = ctx->d_flag;
    // stage the ranks' payload bytes of a slice in shared memory when a 3+-deep
    // ring still fits (<= 48 KB of pieces per stage)
    const uint32_t bb = ctx->cfg.comp.kind == BPC_SCALED_SIGN ? 1u : ctx->cfg.comp.bits;
    q.piece_stride = (uint32_t)round_up((uint64_t)kStreamSlice * bb / 8 + 32, 16);
    q.stage_payload = (uint64_t)q.piece_stride * q.n <= 49152 && ctx->cfg.world_size <= 32;
    q.sync = peer_sync(ctx, EP_SERVER);
    const bool mcopy = fused_exchange(ctx) && ctx->nvls && ctx->nvls_copy;
    if (fused_exchange(ctx)) {   // wait for every rank's push; p stays in the local P; signal
      set_wait(ctx, &q.sync, EP_PUSH);
      if (!mcopy) set_signal(ctx, &q.sync, EP_PULL);   // (NVLS copy: the copy kernel signals)
      if (ctx->nvls && !mcopy) q.mc_out = ctx->pbuf_mc;   // ... or goes to every rank's P (multicast)
      if (ctx->n_sslices == 0 && !mcopy) {   // owns no chunk: no server launch, only the signal
        P2PParams e = {};
        e.sync = peer_sync(ctx, EP_PULL);
        set_signal(ctx, &e.sync, EP_PULL);
        CK(launch_p2p_copy(e, 1, ctx->stream), "pull signal launch");
        ctx->launches++;
      }
    }
    CK(launch_stream_side(ctx, true, q), "server stream launch");
    if (mcopy) {   // this rank's p segment (contiguous, 16-byte slots) to every rank's P, then signal
      const Plan& P = ctx->plan;
      const int rank = ctx->cfg.rank;
      P2PParams e = {};
      if (P.seg_bytes[rank]) {
        e.src[0] = ctx->pbuf + P.seg_off[rank];
        e.dst[0] = ctx->pbuf_mc + P.seg_off[rank];
        e.len[0] = P.seg_bytes[rank];
        e.njobs = 1;
      }
      e.mc = 1;
      e.sync = peer_sync(ctx, EP_PULL);
      set_signal(ctx, &e.sync, EP_PULL);
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(2ull * ctx->num_sms, (P.seg_bytes[rank] + 32767) / 32768));
      CK(launch_p2p_copy(e, grid, ctx->stream), "multicast copy launch");
      ctx->launches++;
    }
  } else {
    if (sparse_p2p(ctx)) {   // every rank's delta has landed in RECV
      if (bpc_status st = launch_flag_wait(ctx, EP_PUSH, "push wait launch")) return st;
    }
    SparseParams p = sparse_params(ctx, 1);
    p.recv = ctx->recv;
    p.slot_bytes = slot;
    p.vals = ctx->cfg.comp.use_ef ? ctx->etl : ctx->d_sdelta;
    p.out = ctx->pbuf;
    if (bpc_status st = launch_sparse_side(ctx, p, nullptr)) return st;
  }
  timer_end(ctx, BPC_TIMER_SERVER, b);
  ctx->phase = 3;
  return BPC_OK;
}

bpc_status bpc_exchange_pull(bpc_ctx* ctx) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  if (ctx->phase != 3) return BPC_ERR_BAD_STATE;
  DeviceGuard dg(ctx->cfg.device);
  const int n = ctx->cfg.world_size, rank = ctx->cfg.rank;
  if (n > 1 && (ctx->comm || ctx->local_group) && !fused_exchange(ctx)) {
    const Plan& P = ctx->plan;
    cudaEvent_t b = nullptr;
    timer_begin(ctx, BPC_TIMER_PULL, &b);
    if (ctx->exchange == BPC_EXCHANGE_P2P) {
      // my segment of P -> the same offset of every peer's P, then release the pull
      // flag on every peer; bpc_step waits for the peers' flags before it decodes
      P2PParams q = {};
      for (int r = 0; r < n; r++) {
        if (r == rank) continue;
        if (P.seg_bytes[rank]) {
          q.src[q.njobs] = ctx->pbuf + P.seg_off[rank];
          q.dst[q.njobs] = ctx->peer_p[r] + P.seg_off[rank];
          q.len[q.njobs++] = P.seg_bytes[rank];
        }
      }
      q.sync = peer_sync(ctx, EP_PULL);
      set_signal(ctx, &q.sync, EP_PULL);
      CK(launch_p2p_copy(q, ctx->pull_grid, ctx->stream), "pull copy launch");
      ctx->launches += 1;
    } else {
      NK(ncclGroupStart(), "group start");
      for (int r = 0; r < n; r++) {
        if (r == rank) continue;
        if (P.seg_bytes[rank]) NK(ncclSend(ctx->pbuf + P.seg_off[rank], P.seg_bytes[rank], ncclUint8, r, ctx->comm, ctx->stream), "send");
        if (P.seg_bytes[r]) NK(ncclRecv(ctx->pbuf + P.seg_off[r], P.seg_bytes[r], ncclUint8, r, ctx->comm, ctx->stream), "recv");
      }
      NK(ncclGroupEnd(), "group end");
    }
    timer_end(ctx, BPC_TIMER_PULL, b);
  }
  ctx->phase = 4;
  return BPC_OK;
}

bpc_status bpc_aggregate(bpc_ctx* ctx) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  if (ctx->cfg.world_size > 1 && !ctx->comm && !ctx->local_group) return BPC_ERR_BAD_STATE;
  bpc_status s = bpc_exchange_push(ctx);
  if (s != BPC_OK) return s;
  if ((s = bpc_server(ctx)) != BPC_OK) return s;
  return bpc_exchange_pull(ctx);
}

bpc_status bpc_step(bpc_ctx* ctx, float* d_params, float lr) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  if (ctx->phase != 4) return BPC_ERR_BAD_STATE;
  DeviceGuard dg(ctx->cfg.device);
  if (bpc_status st = check_user_ptr(ctx, d_params, "d_params")) return st;
  const bpc_config& c = ctx->cfg;
  UpdateParams p = {};
  p.pbuf = ctx->pbuf;
  p.chunks = ctx->d_chunks;
  p.tiles = ctx->d_utiles;
  p.n_tiles = ctx->n_utiles;
  p.m = ctx->m;
  p.v = ctx->v;
  p.x = d_params;
  p.beta1 = c.beta1;
  p.beta2 = c.beta2;
  p.omb1 = (float)(1.0 - (double)c.beta1);
  p.omb2 = (float)(1.0 - (double)c.beta2);
  // bias corrections 1 - beta^t of the device's t, fp64 then one rounding (R16)
  p.bias.bct = ctx->d_bct;
  p.bias.nbct = ctx->nbct;
  p.bias.conv = ctx->bconv;
  p.bias.beta1 = (double)c.beta1;
  p.bias.beta2 = (double)c.beta2;
  p.eps = c.eps;
  p.lr = lr;
  p.wd = c.weight_decay;
  p.bits = c.comp.bits;
  p.f16 = c.comp.f16_values;
  p.mu = c.momentum;
  p.sync = peer_sync(ctx, EP_UPDATE);
  if (fused_exchange(ctx)) {   // wait for every owner's p, then read it from the owner's P
    set_wait(ctx, &p.sync, EP_PULL);
    // NVLS: the server multicast p into every rank's P, so every owner's p is local
    for (int r = 0; r < c.world_size; r++) p.psrc[r] = ctx->nvls ? ctx->pbuf : ctx->peer_p[r];
  }
  cudaEvent_t b = nullptr;
  timer_begin(ctx, BPC_TIMER_UPDATE, &b);
  if (sparse_p2p(ctx)) {   // every owner's p has landed in P
    if (bpc_status st = launch_flag_wait(ctx, EP_PULL, "pull wait launch")) return st;
  }
  const bool sparse = c.comp.kind == BPC_TOP_K || c.comp.kind == BPC_RANDOM_K;
  if (sparse) {   // each half tile's payload entries, for the update's scatter
    p.ent = ctx->d_ent;
    CK(launch_sparse_ranges(p, ctx->d_ent, ctx->stream), "entry ranges launch");
    ctx->launches++;
  }
  auto pass = [&](int mode) -> cudaError_t {
    p.mode = mode;
    return launch_update_stream(c.comp.kind, p, ctx->num_sms, ctx->stream);
  };
  if (c.optimizer == BPC_OPT_LANS) {
    // LANS (R22): m, v + per-tile block sums; per-block coefficients; x
    p.lans_part = ctx->d_lans_part;
    p.lans_coef = ctx->d_lans_coef;
    CK(pass(1), "LANS pass 1 launch");
    LansCoefParams lc = {};
    lc.part = ctx->d_lans_part;
    lc.blk_tile = ctx->d_blk_tile;
    lc.nblk = c.num_tensors;
    lc.coef = ctx->d_lans_coef;
    lc.beta1 = c.beta1;
    lc.alpha_l = c.lans_alpha_l;
    lc.alpha_u = c.lans_alpha_u;
    CK(launch_lans_coef(lc, ctx->stream), "LANS coefficient launch");
    p.sync.inc_t = 1;   // the step's last launch advances t
    CK(pass(2), "LANS pass 2 launch");
    ctx->launches += 3;
  } else {
    p.sync.inc_t = 1;
    CK(pass(c.optimizer == BPC_OPT_NAG ? 3 : 0), "update launch");
    ctx->launches++;
  }
  timer_end(ctx, BPC_TIMER_UPDATE, b);
  ctx->phase = 0;
  return BPC_OK;
}

bpc_status bpc_sync(bpc_ctx* ctx) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->cfg.device);
  CK(cudaStreamSynchronize(ctx->stream), "stream sync");
  if (ctx->comm) {
    ncclResult_t ar;
    if (ncclCommGetAsyncError(ctx->comm, &ar) != ncclSuccess || ar != ncclSuccess) {
      ctx->err = "NCCL async error";
      return BPC_ERR_NCCL;
    }
  }
  unsigned int flag = 0;
  CK(cudaMemcpy(&flag, ctx->d_flag, 4, cudaMemcpyDeviceToHost), "flag read");
  if (flag) {
    CK(cudaMemset(ctx->d_flag, 0, 4), "flag reset");
    ctx->err = "non-finite gradient";
    return BPC_ERR_NONFINITE;
  }
  return BPC_OK;
}

bpc_status bpc_finalize(bpc_ctx* ctx) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->cfg.device);
  bpc_status st = BPC_OK;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->comm && ctx->exchange == BPC_EXCHANGE_P2P) {
    // Collective teardown: a peer's last update may still be reading this
    // rank's P (or its last push writing this rank's RECV) over NVLink after
    // this rank's stream drained.  An all-reduce over the communicator, run
    // after every rank's stream drained, orders the frees after all of them.
    int32_t* d = nullptr;
    if (cudaMalloc((void**)&d, 4) == cudaSuccess && cudaMemsetAsync(d, 0, 4, ctx->stream) == cudaSuccess &&
        ncclAllReduce(d, d, 1, ncclInt32, ncclSum, ctx->comm, ctx->stream) == ncclSuccess) {
      if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = BPC_ERR_CUDA;
    } else {
      st = BPC_ERR_NCCL;
    }
    if (d) cudaFree(d);
  }
  free_ctx(ctx);
  return st;
}

bpc_status bpc_get_plan(const bpc_ctx* ctx, bpc_plan_summary* out) {
  if (!ctx || !out) return BPC_ERR_INVALID_ARGUMENT;
  fill_summary(ctx->plan, ctx->cfg.rank, out);
  return BPC_OK;
}

bpc_status bpc_get_chunk(const bpc_ctx* ctx, uint32_t chunk, bpc_chunk_info* out) {
  if (!ctx || !out || chunk >= ctx->plan.chunks.size()) return BPC_ERR_INVALID_ARGUMENT;
  *out = ctx->plan.chunks[chunk];
  return BPC_OK;
}

bpc_status bpc_peer_segment(const bpc_ctx* ctx, int32_t peer, uint64_t* offset, uint64_t* bytes) {
  if (!ctx || !offset || !bytes || peer < 0 || peer >= ctx->cfg.world_size) return BPC_ERR_INVALID_ARGUMENT;
  *offset = ctx->plan.seg_off[peer];
  *bytes = ctx->plan.seg_bytes[peer];
  return BPC_OK;
}

static bool buffer_of(const bpc_ctx* ctx, int32_t which, void** p, uint64_t* bytes) {
  const uint64_t D = round_up(ctx->plan.D, 4);
  switch (which) {
    case BPC_BUF_SEND: *p = ctx->send; *bytes = ctx->plan.send_bytes; return true;
    case BPC_BUF_RECV: *p = ctx->recv; *bytes = ctx->recv_bytes; return true;
    case BPC_BUF_P: *p = ctx->pbuf; *bytes = ctx->plan.send_bytes; return true;
    case BPC_BUF_WORKER_ERR: *p = ctx->e; *bytes = 4 * D; return true;
    case BPC_BUF_SERVER_ERR: *p = ctx->etl; *bytes = 4 * ctx->plan.etl_elems; return true;
    case BPC_BUF_M: *p = ctx->m; *bytes = 4 * D; return true;
    case BPC_BUF_V: *p = ctx->v; *bytes = 4 * D; return true;
  }
  return false;
}

bpc_status bpc_buffer(const bpc_ctx* ctx, int32_t which, void** d_ptr, uint64_t* bytes) {
  if (!ctx || !d_ptr || !bytes) return BPC_ERR_INVALID_ARGUMENT;
  return buffer_of(ctx, which, d_ptr, bytes) ? BPC_OK : BPC_ERR_INVALID_ARGUMENT;
}

bpc_status bpc_copy_state(bpc_ctx* ctx, int32_t which, void* host_dst, uint64_t bytes) {
  void* p;
  uint64_t b;
  if (!ctx || !host_dst || !buffer_of(ctx, which, &p, &b)) return BPC_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->cfg.device);
  if (bytes != b) return BPC_ERR_SIZE_MISMATCH;
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  if (b) CK(cudaMemcpy(host_dst, p, b, cudaMemcpyDeviceToHost), "copy state");
  return BPC_OK;
}

bpc_status bpc_load_state(bpc_ctx* ctx, int32_t which, const void* host_src, uint64_t bytes) {
  void* p;
  uint64_t b;
  if (!ctx || !host_src || !buffer_of(ctx, which, &p, &b)) return BPC_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->cfg.device);
  if (bytes != b) return BPC_ERR_SIZE_MISMATCH;
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  if (which == BPC_BUF_SERVER_ERR && !stream_worker(ctx->cfg.comp.kind) && b) {
    // sparse kinds: the server reads Delta = fl32(0 + e~) as e~ itself, which holds
    // for every e~ it writes (never -0); a loaded -0 is stored as the +0 it decodes to
    std::vector<uint32_t> w(b / 4);
    memcpy(w.data(), host_src, b);
    for (auto& x : w)
      if (x == 0x80000000u) x = 0;
    CK(cudaMemcpy(p, w.data(), b, cudaMemcpyHostToDevice), "load state");
    return BPC_OK;
  }
  if (b) CK(cudaMemcpy(p, host_src, b, cudaMemcpyHostToDevice), "load state");
  return BPC_OK;
}

bpc_status bpc_get_exchange(const bpc_ctx* ctx, int32_t* mode) {
  if (!ctx || !mode) return BPC_ERR_INVALID_ARGUMENT;
  *mode = (ctx->exchange == BPC_EXCHANGE_P2P && ctx->nvls) ? BPC_EXCHANGE_NVLS : ctx->exchange;
  return BPC_OK;
}

// t lives on the device (DevState): read / written in the context's stream order
bpc_status bpc_get_step(const bpc_ctx* cctx, uint32_t* t) {
  if (!cctx || !t) return BPC_ERR_INVALID_ARGUMENT;
  bpc_ctx* ctx = const_cast<bpc_ctx*>(cctx);   // error text only
  DeviceGuard dg(ctx->cfg.device);
  CK(cudaMemcpyAsync(t, &ctx->d_st->t, 4, cudaMemcpyDeviceToHost, ctx->stream), "step read");
  CK(cudaStreamSynchronize(ctx->stream), "step read sync");
  return BPC_OK;
}

bpc_status bpc_set_step(bpc_ctx* ctx, uint32_t t) {
  if (!ctx || t < 1) return BPC_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->cfg.device);
  CK(cudaMemcpyAsync(&ctx->d_st->t, &t, 4, cudaMemcpyHostToDevice, ctx->stream), "step write");
  CK(cudaStreamSynchronize(ctx->stream), "step write sync");
  return BPC_OK;
}

bpc_status bpc_set_timing(bpc_ctx* ctx, int32_t enable) {
  if (!ctx) return BPC_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->cfg.device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& ev : ctx->events) {
    cudaEventDestroy(ev.second.first);
    cudaEventDestroy(ev.second.second);
  }
  ctx->events.clear();
  ctx->timing = enable != 0;
  return BPC_OK;
}

bpc_status bpc_get_timing(bpc_ctx* ctx, float ms[BPC_NUM_TIMERS], uint32_t count[BPC_NUM_TIMERS]) {
  if (!ctx || !ms || !count) return BPC_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->cfg.device);
  for (int i = 0; i < BPC_NUM_TIMERS; i++) {
    ms[i] = 0.f;
    count[i] = 0;
  }
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  for (auto& ev : ctx->events) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ev.second.first, ev.second.second), "elapsed");
    ms[ev.first] += t;
    count[ev.first]++;
  }
  return BPC_OK;
}

uint64_t bpc_launch_count(const bpc_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
