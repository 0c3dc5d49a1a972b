// kernels.h — device-side tables and host launchers of libbpc (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace bpc {

constexpr int P2P_MAXJ = 64;   // max world size of the peer-memory exchange

// Step-varying values of a context live in device memory: every kernel reads
// the ones it needs when it starts, and the last CTA of a launch advances them.
// No kernel parameter changes from step to step, so a CUDA graph of a step
// replays correctly (any world size, fused exchange included).
enum { EP_WORKER = 0, EP_SERVER = 1, EP_UPDATE = 2, EP_PUSH = 3, EP_PULL = 4 };
struct DevState {
  uint32_t t;                  // Alg. 5 step counter, >= 1
  uint32_t ep[7];              // launch epochs per family (EP_*); push / pull = exchange epochs
  unsigned long long done[8];  // per-family CTA arrivals of the running launch (the last CTA resets)
};
// Bias corrections of step t (R16): bct[t - 1] = (fl32(1 - b1^t), fl32(1 - b2^t),
// RN(1 / bc1), RN(1 / bc2)) formed on the host in fp64; past nbct both are 1.0f
// (conv = 1) or the table was capped (conv = 0: computed on the device)
struct BiasTab {
  const float4* bct;
  uint32_t nbct;
  int32_t conv;
  double beta1, beta2;
};
__device__ __forceinline__ float4 bias_of(const BiasTab& b, uint32_t t) {
  if (t <= b.nbct) return b.bct[t - 1];
  if (b.conv) return make_float4(1.f, 1.f, 1.f, 1.f);
  const float b1 = (float)(1.0 - pow(b.beta1, (double)t)), b2 = (float)(1.0 - pow(b.beta2, (double)t));
  return make_float4(b1, b2, 1.f / b1, 1.f / b2);
}

// Launch bookkeeping and the fused NVLink exchange of one kernel launch:
//  epoch  - E = st->ep[fam] + 1 for this launch; the last CTA (done counter
//           reaching the grid size) stores it;
//  wait   - wait_fam >= 0: before its first load of exchanged bytes the kernel
//           waits until wflags[wslot0 + r] >= st->ep[wait_fam] for every rank
//           r != self (system-scope acquire of the producers' release);
//  signal - sig_fam >= 0: after its last store the last CTA releases
//           st->ep[sig_fam] + 1 into slot sslot of every peer's flag array
//           (sflag[r]; null for self) and stores it;
//  inc_t  - the last CTA advances st->t (the step's final update launch).
struct PeerSync {
  DevState* st;
  int32_t fam, wait_fam, sig_fam, inc_t;
  const unsigned long long* wflags;
  uint32_t wslot0;
  unsigned long long* sflag[P2P_MAXJ];
  uint32_t sslot;
  uint32_t n, self;
};

// one compression unit (chunk) as the kernels see it
struct DevChunk {
  uint64_t off;    // flat element offset
  uint64_t pay;    // byte offset of its payload in SEND / P
  uint64_t recv;   // byte offset inside each RECV slot (owned chunks)
  uint64_t etl;    // element offset in SERVER_ERR (owned, compressed, use_ef)
  uint32_t len;    // L
  uint32_t k;      // sparse k
  uint32_t id;     // global chunk id (Philox counter word 1)
  uint32_t raw;    // 1 = NONE payload
  uint32_t owner;  // server rank of the chunk
  uint32_t pad;
};

// a piece of a chunk processed by one CTA (raw tiles, update tiles)
struct Tile {
  uint32_t chunk;  // index into the chunk table
  uint32_t start;  // first element, relative to the chunk
  uint32_t len;
  uint32_t pad;
};

struct UpdateParams {
  const uint8_t* pbuf;
  const DevChunk* chunks;
  const Tile* tiles;
  uint32_t n_tiles;
  float* m;
  float* v;
  float* x;
  float beta1, beta2, omb1, omb2, eps, lr, wd;
  BiasTab bias;           // bc = fl32(1 - beta^t) of the step (R16) and RN(1 / bc) (divc)
  uint32_t bits;
  int32_t mode;           // 0 Adam core; LANS (R22): 1 = pass 1 (m, v, block sums), 2 = pass 2 (x);
                          // 3 NAG (R24, velocity in m)
  int32_t f16;            // sparse kinds: binary16 values (R23)
  float mu;               // NAG momentum (mode 3, R24)
  double* lans_part;      // LANS pass 1: per update tile the pairwise sums of x^2, u^2, w^2
  const float2* lans_coef;  // LANS pass 2: per block (a, b) coefficients
  const uint2* ent;       // sparse kinds: per 2048-element half tile (first payload entry, entries)
                          // (sparse_ranges_kernel)
  PeerSync sync;          // fused exchange: wait for the owners' p (pull) ...
  const uint8_t* psrc[P2P_MAXJ];   // ... and read chunk payloads from psrc[owner] (P of each rank)
};

// a 2^13-element slice of a unit for the streaming worker / server kernels
struct Slice {
  uint32_t chunk;       // index into the chunk table
  uint32_t start;       // first element, relative to the chunk
  uint32_t len;
  uint32_t nslices;     // slices in this unit (0 = raw tile: no reduction)
  uint32_t sidx;        // index of this slice inside its unit
  uint32_t unit;        // unit counter index (multi-slice units)
  uint32_t unit_first;  // first partial of the unit
  uint32_t pad;
};

struct StreamParams {
  const float* grad;      // worker: g
  float* err;             // worker: e; server: e~ (compact)
  uint8_t* out;           // worker: SEND; server: P
  const uint8_t* recv;    // server: RECV
  uint64_t slot_bytes;
  const DevChunk* chunks;
  const Slice* slices;
  uint32_t n_slices;
  double* partials;       // per-slice tree partials of multi-slice units
  unsigned long long* counters;   // per-unit published-slice counters (monotonic: a unit is
                                  // complete at E x nslices, E = this launch's epoch)
  uint32_t n;
  double inv_n;
  uint32_t rank, stage;
  uint64_t seed;
  uint32_t bits;
  int32_t use_ef, check_finite;
  unsigned int* flag;
  uint32_t stage_payload;   // server: stage the n ranks' payload pieces in smem
  uint32_t piece_stride;    // server: bytes per staged piece
  uint32_t nstages, stage_a, stage_b;   // ring geometry (set by the launcher)
  uint32_t defer;                       // emit deferral D (set by the launcher)
  uint32_t rk[20];          // Philox round keys of the seed (set by the launcher, R13)
  // per-tensor units (NEXT #4): two passes.  pass 0: single pass
  // (units <= 32 slices, cross-CTA unit totals); pass 1: produce + publish the
  // slice partials only; pass 2: produce again and emit with unit_total[unit]
  uint32_t pass;
  const double* unit_total;
  // fused exchange (BPC_EXCHANGE_P2P, n > 1):
  //  worker: ndst = n, the payload of a chunk owned by r goes to dst[r] +
  //          chunk.recv (slot `rank` of r's RECV, IPC-mapped), then signals push;
  //  server: waits for every push, stores p to the local P, then signals pull
  //          (the update kernels read it from there over NVLink);
  //          with mc_out (BPC_EXCHANGE_NVLS) p is stored through the multicast
  //          mapping of P instead (multimem.st: every rank's P holds it).
  uint8_t* dst[P2P_MAXJ];
  uint32_t ndst;
  uint8_t* mc_out;
  PeerSync sync;
  // sparse kinds (top-k, random-k): this side's candidate lists (kernels_sparse.cu)
  const uint32_t* sp_chunk2u;
  const uint32_t* sp_guess;
  uint32_t* sp_scnt;          // candidates per slice (of this side's slice table)
  uint2* sp_cand;             // unit u's list at sp_cand_off[u]: one sub-list of (cap / nslices) per slice,
                              // entries (index, select key)
  const uint32_t* sp_cand_off;
};

// sparse kinds (kernels_sparse.cu): prep -> streaming pass (kernels_cstream.cu) -> select, per side
struct SparseParams {
  const float* grad;        // worker: g (flat)
  float* vals;              // worker: e (flat; use_ef); server: e~ (use_ef) or the Delta scratch
                            // (compact, DevChunk.etl)
  uint8_t* out;             // worker: SEND; server: P
  const uint8_t* recv;      // server: RECV (n slots)
  uint64_t slot_bytes;
  const DevChunk* chunks;
  const uint32_t* items;    // this side's compressed units (chunk indices)
  uint32_t n_units;
  const Slice* slices;      // this side's 2^13-element slices (compressed and raw units)
  uint32_t n_slices;
  const uint32_t* chunk2u;  // chunk -> unit index of this side
  uint32_t* guess;          // [n_units] candidate thresholds
  uint32_t* scnt;           // candidates per slice of this side's slice table (written by the streaming pass)
  uint2* cand;              // candidates (index, select key), unit u at [cand_off[u], cand_off[u + 1]): slice s of
                            // the unit owns the index-ordered sub-list [s cs, s cs + min(scnt, cs)),
                            // cs = (cand_off[u + 1] - cand_off[u]) / nslices
  const uint32_t* cand_off; // [n_units + 1]
  const uint32_t* first_slice;  // [n_units] the unit's first slice in this side's slice table
  uint32_t n;
  double inv_n;
  const DevState* st;        // the step counter t (Philox counter word 2, R13)
  uint32_t stage, rrank;     // Philox counter words (R13): stage 0 push (rank), 1 pull (0)
  uint64_t seed;
  int32_t server, randk_scaled, use_ef, f16, check_finite;
  unsigned int* flag;
  uint32_t sel_cap;         // CTA select kernel: candidates held in shared memory, a power of two <= SEL_CAP
  uint32_t* big;            // [n_units] units the warp select hands to the CTA select (it resets them)
  const uint2* apply_blk;   // server: (unit, first entry) of each 256-entry block of the ranks' entries
  uint32_t n_apply_blk;
  // per-tensor units longer than SEL_LMAX (the large path)
  const uint32_t* large_units;   // [n_large] unit indices
  uint32_t n_large;
  const uint2* lslices;          // (slice index, large unit) of every slice of the large units, by unit
  uint32_t n_lslices;
  const uint32_t* lslice_first;  // [n_large + 1]
  uint32_t* lstate;              // [8 n_large] radix-select state
  uint32_t* lhist;               // [256 n_large]
  uint2* lcnt;                   // [n_lslices] (keys > T, keys == T)
  uint2* loff;                   // [n_lslices] (first output position, T-ties before)
  uint32_t large_grid;
};
constexpr uint32_t SEL_CAP = 16384;     // max candidates a select CTA holds in shared memory
constexpr uint32_t SEL_LMAX = 1u << 18; // longer units (per-tensor) take the large-unit path
// the sample rank of the top-k guess (host: capacity; device: the guess)
__host__ __device__ inline uint32_t sparse_sample_rank(uint32_t k, uint32_t L) {
  const double mu = (double)k * 4096.0 / (double)L;
  return (uint32_t)ceil(mu + 3.0 * sqrt(mu) + 6.0);
}
cudaError_t launch_sparse_prep(int kind, const SparseParams& p, cudaStream_t s);
cudaError_t launch_sparse_select(int kind, const SparseParams& p, cudaStream_t s);
size_t sparse_select_smem(uint32_t sel_cap);

// peer-memory exchange (kernels_p2p.cu)
struct P2PParams {
  const uint8_t* src[P2P_MAXJ];
  uint8_t* dst[P2P_MAXJ];           // local or a peer's IPC-mapped buffer
  uint64_t len[P2P_MAXJ];           // bytes, multiples of 16
  int njobs;
  int mc;                           // dst is a multicast mapping (BPC_EXCHANGE_NVLS): multimem.st.v4
  PeerSync sync;                    // fam = sig_fam = EP_PUSH / EP_PULL: the copy's epoch, released to the peers
};
struct P2PWait {
  const unsigned long long* flags;  // this rank's flag array
  int slots[P2P_MAXJ];
  int nslots;
  const DevState* st;               // wait until every slot >= st->ep[fam]
  int fam;
};

// LANS block coefficients (R22): one CTA per block reduces its tiles' partial
// sums (pairwise, padded to a power of two) and writes (a, b)
struct LansCoefParams {
  const double* part;        // [3 * n_tiles]
  const uint32_t* blk_tile;  // per block: first tile index; blk_tile[nblk] = n_tiles
  uint32_t nblk;
  float2* coef;              // [nblk]
  float beta1, alpha_l, alpha_u;
};
cudaError_t launch_lans_coef(const LansCoefParams& p, cudaStream_t s);
constexpr uint32_t LANS_MAX_TILES = 8192;   // tiles per block (2^25 elements)

// per-tensor units: unit u's total = pairwise tree over its slice partials
// part[first[u] .. first[u] + ns[u]) padded to a power of two (R6)
struct UnitTreeParams {
  const double* part;
  const uint32_t* first;
  const uint32_t* ns;
  uint32_t nunits;
  double* total;
};
cudaError_t launch_unit_tree(const UnitTreeParams& p, cudaStream_t s);
constexpr uint32_t UNIT_MAX_SLICES = 16384;   // 2^27 elements per unit

// host launchers (return the launch error)
cudaError_t launch_p2p_copy(const P2PParams& p, int grid, cudaStream_t s);
cudaError_t launch_p2p_wait(const P2PWait& w, cudaStream_t s);
cudaError_t launch_worker_stream(int kind, const StreamParams& p, int grid, cudaStream_t s);
cudaError_t launch_server_stream(int kind, const StreamParams& p, int grid, cudaStream_t s);
cudaError_t launch_update_stream(int kind, const UpdateParams& p, int grid, cudaStream_t s);
size_t cstream_smem();
size_t update_stream_smem();
// sparse kinds: p.ent of every half tile (binary searches of the tile bounds in
// the chunk's ascending payload indices), before update_stream
cudaError_t launch_sparse_ranges(const UpdateParams& p, uint2* ent, cudaStream_t s);

}  // namespace bpc
