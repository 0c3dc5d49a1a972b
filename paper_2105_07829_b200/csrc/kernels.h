// kernels.h — device-side tables and host launchers of libbpc (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace bpc {

constexpr int P2P_MAXJ = 64;   // max world size of the peer-memory exchange

// Fused NVLink exchange inside a streaming kernel (BPC_EXCHANGE_P2P):
//  wait   - before its first load of exchanged bytes, the kernel waits until
//           wflags[wslot0 + r] >= wepoch for every rank r != self (system-scope
//           acquire of the producers' release);
//  signal - after its last store, the last CTA releases sepoch into slot sslot
//           of every peer's flag array (sflag[r], IPC-mapped; null for self).
struct PeerSync {
  const unsigned long long* wflags;   // null: no wait
  uint32_t wslot0, wepoch;
  unsigned long long* done;           // CTA counter (monotonic: sepoch * grid); null: no signal
  unsigned long long* sflag[P2P_MAXJ];
  uint32_t sslot, sepoch;
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
  float beta1, beta2, omb1, omb2, bc1, bc2, eps, lr, wd;   // bc = fl32(1 - beta^t), R16
  float ibc1, ibc2;       // RN(1 / bc): the divisions by bc run as Markstein's correction (divc)
  uint32_t bits;
  int32_t mode;           // 0 Adam core; LANS (R22): 1 = pass 1 (m, v, block sums), 2 = pass 2 (x);
                          // 3 NAG (R24, velocity in m)
  int32_t f16;            // sparse kinds: binary16 values (R23)
  float mu;               // NAG momentum (mode 3, R24)
  double* lans_part;      // LANS pass 1: per update tile the pairwise sums of x^2, u^2, w^2
  const float2* lans_coef;  // LANS pass 2: per block (a, b) coefficients
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
  unsigned long long* counters;   // per-unit published-slice counters (monotonic)
  uint32_t epoch;         // launch number: a unit is complete at epoch * nslices
  uint32_t n;
  double inv_n;
  uint32_t t, rank, stage;
  uint64_t seed;
  uint32_t bits;
  int32_t use_ef, check_finite;
  unsigned int* flag;
  uint32_t stage_payload;   // server: stage the n ranks' payload pieces in smem
  uint32_t piece_stride;    // server: bytes per staged piece
  uint32_t nstages, stage_a, stage_b;   // ring geometry (set by the launcher)
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
  //          (the update kernels read it from there over NVLink).
  uint8_t* dst[P2P_MAXJ];
  uint32_t ndst;
  PeerSync sync;
};

// sparse kinds (kernels_sparse.cu): guess -> stream -> select, per side
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
  uint32_t* cnt;            // [n_units] candidate counters (the select kernel resets them)
  uint32_t* cand;           // candidate indices, unit u at [cand_off[u], cand_off[u + 1])
  const uint32_t* cand_off; // [n_units + 1]
  uint32_t n;
  double inv_n;
  uint32_t t, stage, rrank;  // Philox counter words (R13): stage 0 push (rank), 1 pull (0)
  uint64_t seed;
  int32_t server, randk_scaled, use_ef, f16, check_finite;
  unsigned int* flag;
  uint32_t sel_cap;         // CTA select kernel: candidates held in shared memory, a power of two <= SEL_CAP
  uint32_t* big;            // [n_units] units the warp select hands to the CTA select (it resets them)
};
constexpr uint32_t SEL_CAP = 16384;     // max candidates a select CTA holds in shared memory
// the sample rank of the top-k guess (host: capacity; device: the guess)
__host__ __device__ inline uint32_t sparse_sample_rank(uint32_t k, uint32_t L) {
  const double mu = (double)k * 4096.0 / (double)L;
  return (uint32_t)ceil(mu + 3.0 * sqrt(mu) + 6.0);
}
cudaError_t launch_sparse(int kind, const SparseParams& p, int grid, cudaStream_t s);
size_t sparse_select_smem(uint32_t sel_cap);

// peer-memory exchange (kernels_p2p.cu)
struct P2PParams {
  const uint8_t* src[P2P_MAXJ];
  uint8_t* dst[P2P_MAXJ];           // local or a peer's IPC-mapped buffer
  uint64_t len[P2P_MAXJ];           // bytes, multiples of 16
  int njobs;
  unsigned long long* peer_flag[P2P_MAXJ];   // peers' flag arrays (IPC-mapped)
  int npeers;
  int slot;                         // flag slot this launch releases on every peer
  uint32_t epoch;
  unsigned long long* done;         // local CTA counter (monotonic: epoch * grid)
};
struct P2PWait {
  const unsigned long long* flags;  // this rank's flag array
  int slots[P2P_MAXJ];
  int nslots;
  uint32_t epoch;
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
cudaError_t launch_update(int kind, const UpdateParams& p, cudaStream_t s);

}  // namespace bpc
