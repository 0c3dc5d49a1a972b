// kernels_compress.cu — worker compress and server
// decompress-sum-recompress (A5-A7) for the sparse kinds, top-k (R9) and
// random-k (R10), on sm_100a.
//
// One thread-block cluster per compression unit (chunk of <= cs * 2^14
// elements, R1): CTA r of the cluster owns slice
// [r * 2^14, (r + 1) * 2^14) of the unit and keeps it on chip (64 KB of shared
// memory) between the unit-wide selection and the write-back, so every HBM
// byte is read and written once:
//   worker  q = g + e (Alg. 4 l.5) -> C(q) (l.6) -> e = q - dec (l.7)
//   server  Delta = (1/n) sum_i dec(delta_i) + e~ (l.10)
//           -> p = C(Delta) (l.11) -> e~ = Delta - dec(p) (l.13)
// The exact selection of the k largest keys runs over the cluster through
// DSMEM (histogram bins, candidate gather, tie cut), with a
// 4 x 8-bit radix select as the fallback.  Raw (below-threshold) units ride the
// same launch as plain tiles.  The norm-based kinds run in kernels_cstream.cu.
#include "device.cuh"

namespace bpc {

enum { K_TOPK = 3, K_RANDK = 4 };

constexpr int FNB = 1024;   // bins of the sparse kinds' 10-bit key histogram
constexpr int FCAP = FNB / 2;   // candidate capacity: CTA 0 keeps (key, index) pairs in fh
constexpr int SELCAP = 512;     // small-k emit: a CTA's selected (index, value) pairs in bsum / hist

struct __align__(16) Smem {
  float4 q[SLICE / 4];      // the slice of q (worker) or Delta (server)
  union {
    uint32_t fh[FNB];       // sparse kinds: 10-bit key histogram (DSMEM), then CTA 0's candidate
                            // keys [0, FCAP) and their indices [FCAP, 2 FCAP)
  };
  union {
    uint32_t bsum[FNB];     // sparse: this CTA's share of the cluster-wide histogram (DSMEM)
    struct {
      uint32_t hist[2][256];   // sparse fallback: radix-select histograms (DSMEM)
      uint32_t tot[256];
    };
  };
  uint32_t cnt[2];          // (#key > T, #key == T) of this slice (DSMEM); small k: cnt[0] = #selected
  uint32_t scan[NWARP + 1];
  uint32_t info[8];
  uint32_t btot;            // sum of bsum (DSMEM)
  uint32_t ccount;          // candidates gathered into CTA 0 (DSMEM atomics)
  uint64_t qbar;            // whole-slice bulk copy of g (worker) / e~ (server) into q
};

// Thread 0 bulk-copies the whole 64 KB slice src[0, SLICE) into sm.q (TMA,
// completes on sm.qbar); the caller waits with slice_wait().  The bytes arrive
// while the threads load the rest of their inputs through registers.
__device__ __forceinline__ void slice_bulk_load(Smem& sm, const float* src) {
  if (threadIdx.x == 0) {
    mbar_init(&sm.qbar, 1);
    fence_mbar_init();
    constexpr uint32_t PIECE = SLICE * 4 / 4;
    mbar_arrive_expect_tx(&sm.qbar, SLICE * 4);
#pragma unroll
    for (int i = 0; i < 4; i++)
      tma_load_1d(reinterpret_cast<uint8_t*>(sm.q) + i * PIECE, reinterpret_cast<const uint8_t*>(src) + i * PIECE,
                  PIECE, &sm.qbar);
  }
}
__device__ __forceinline__ void slice_wait(Smem& sm) {
  __syncthreads();   // the barrier's init is visible
  mbar_wait(&sm.qbar, 0);
}

size_t compress_smem_bytes() { return sizeof(Smem); }

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* scan, uint32_t& total) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) scan[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < NWARP ? scan[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NWARP) scan[lane] = wi - w;
    if (lane == NWARP - 1) scan[NWARP] = wi;
  }
  __syncthreads();
  const uint32_t r = scan[warp] + incl - v;
  total = scan[NWARP];
  __syncthreads();
  return r;
}

// key of an element for the "k largest keys, lowest index first" selection:
// top-k: |q| bits (R9); random-k: ~Philox word (k smallest words, R10)
template <int KIND>
__device__ __forceinline__ uint4 keys4(float4 q, uint32_t j, const CompressParams& p, uint32_t id,
                                       uint32_t stage, uint32_t rrank) {
  if (KIND == K_TOPK) {
    return make_uint4(__float_as_uint(q.x) & 0x7fffffffu, __float_as_uint(q.y) & 0x7fffffffu,
                      __float_as_uint(q.z) & 0x7fffffffu, __float_as_uint(q.w) & 0x7fffffffu);
  } else {
    const uint4 w = rng4(p.seed, j >> 2, id, p.t, stage, rrank);
    return make_uint4(~w.x, ~w.y, ~w.z, ~w.w);
  }
}
__device__ __forceinline__ uint32_t getu(const uint4& v, int u) {
  return u == 0 ? v.x : (u == 1 ? v.y : (u == 2 ? v.z : v.w));
}

// ---------------------------------------------------------------- producers
// worker: q = g + e (use_ef) or q = g; slice -> sm.q; the round-0 10-bit key
// histogram of the selection (emit_sparse) is built here, on the fly, instead
// of in a separate pass
template <int HISTK>
__device__ __forceinline__ void produce_worker(const CompressParams& p, const DevChunk& c, Smem& sm,
                                               uint32_t s0) {
  const float* g = p.grad + c.off;
  const float* e = p.err + c.off;
  const uint32_t L = c.len;
  bool bad = false;
  auto finish = [&](int it, float4 g4, float4 e4) {
    if (p.check_finite) bad |= !(isfinite(g4.x) && isfinite(g4.y) && isfinite(g4.z) && isfinite(g4.w));
    // padding lanes are 0 + 0 = +0
    const float4 q = p.use_ef ? make_float4(fadd(g4.x, e4.x), fadd(g4.y, e4.y), fadd(g4.z, e4.z), fadd(g4.w, e4.w))
                              : g4;
    sm.q[it * NT + threadIdx.x] = q;
    if (HISTK) {
      constexpr int DSH = HISTK == K_TOPK ? 21 : 22;
      const uint32_t j = s0 + 4 * (it * NT + threadIdx.x);
      if (j < L) {
        const uint4 kq = keys4<HISTK>(q, j, p, c.id, 0u, p.rank);
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (j + u < L) atomicAdd(&sm.fh[(getu(kq, u) >> DSH) & (FNB - 1)], 1u);
      }
    }
  };
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (s0 + SLICE <= L) {
    // whole slice valid: g lands in sm.q by one bulk copy while each thread
    // loads its e in batches of B (B 16-byte loads in flight), then q = g + e in place
    slice_bulk_load(sm, g + s0);
    constexpr int B = 8;
    float4 e4[B];
#pragma unroll
    for (int b = 0; b < B; b++) e4[b] = p.use_ef ? ld4(e + s0 + 4 * (b * NT + threadIdx.x)) : z;
    slice_wait(sm);
#pragma unroll
    for (int it0 = 0; it0 < IT; it0 += B) {
      float4 en[B];
      if (it0 + B < IT) {
#pragma unroll
        for (int b = 0; b < B; b++) en[b] = p.use_ef ? ld4(e + s0 + 4 * ((it0 + B + b) * NT + threadIdx.x)) : z;
      }
#pragma unroll
      for (int b = 0; b < B; b++) finish(it0 + b, sm.q[(it0 + b) * NT + threadIdx.x], e4[b]);
      if (it0 + B < IT) {
#pragma unroll
        for (int b = 0; b < B; b++) e4[b] = en[b];
      }
    }
  } else {
#pragma unroll 2
    for (int it = 0; it < IT; it++) {
      const uint32_t j = s0 + 4 * (it * NT + threadIdx.x);
      const float4 g4 = j < L ? load4_masked(g, j, L) : z;
      const float4 e4 = (p.use_ef && j < L) ? load4_masked(e, j, L) : z;
      finish(it, g4, e4);
    }
  }
  if (bad) atomicOr(p.flag, 1u);
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// server, sparse kinds: Delta_j = (float)(sum over ranks holding j of val * (1/n) + e~_j)
// (adding the implicit zeros of the other ranks leaves an fp64 sum that starts at +0 unchanged)
__device__ __forceinline__ void produce_server_sparse(const CompressParams& p, const DevChunk& c,
                                                      Smem& sm, uint32_t s0) {
  const uint32_t L = c.len, k = c.k;
  const float* et = p.etl + c.etl;
  float* sq = reinterpret_cast<float*>(sm.q);
  auto base = [&](int it, float4 e4) {
    float4 d;
    d.x = mean_plus(0.0, p.inv_n, (double)e4.x);
    d.y = mean_plus(0.0, p.inv_n, (double)e4.y);
    d.z = mean_plus(0.0, p.inv_n, (double)e4.z);
    d.w = mean_plus(0.0, p.inv_n, (double)e4.w);
    sm.q[it * NT + threadIdx.x] = d;
  };
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (p.use_ef && s0 + SLICE <= L) {
    // whole slice valid: e~ lands in sm.q by one bulk copy, Delta formed in place
    slice_bulk_load(sm, et + s0);
    slice_wait(sm);
#pragma unroll 4
    for (int it = 0; it < IT; it++) base(it, sm.q[it * NT + threadIdx.x]);
  } else {
#pragma unroll 2
    for (int it = 0; it < IT; it++) {
      const uint32_t j = s0 + 4 * (it * NT + threadIdx.x);
      base(it, (p.use_ef && j < L) ? load4_masked(et, j, L) : z);
    }
  }
  __syncthreads();
  const uint32_t jlo = s0, jhi = min(s0 + (uint32_t)SLICE, L);
  if (jlo >= jhi) return;
  for (uint32_t r = 0; r < p.n; r++) {
    const uint8_t* pl = p.recv + r * p.slot_bytes + c.recv;
    const uint32_t* idx = reinterpret_cast<const uint32_t*>(pl + 8);
    const uint8_t* val = pl + 8 + 4ull * k;
    const uint32_t lo = warp_lower_bound(idx, k, jlo), hi = warp_lower_bound(idx, k, jhi);
    for (uint32_t e = lo + threadIdx.x; e < hi; e += NT) {
      const uint32_t j = idx[e];
      bool first = true;
      for (uint32_t r2 = 0; r2 < r && first; r2++) {
        const uint32_t* idx2 = reinterpret_cast<const uint32_t*>(p.recv + r2 * p.slot_bytes + c.recv + 8);
        const uint32_t pos = lower_bound_u32(idx2, k, j);
        first = !(pos < k && idx2[pos] == j);
      }
      if (!first) continue;
      double acc = 0.0;
      acc += (double)get_val(val, e, p.f16);
      for (uint32_t r2 = r + 1; r2 < p.n; r2++) {
        const uint8_t* pl2 = p.recv + r2 * p.slot_bytes + c.recv;
        const uint32_t* idx2 = reinterpret_cast<const uint32_t*>(pl2 + 8);
        const uint32_t pos = lower_bound_u32(idx2, k, j);
        if (pos < k && idx2[pos] == j) acc += (double)get_val(pl2 + 8 + 4ull * k, pos, p.f16);
      }
      const double ev = p.use_ef ? (double)et[j] : 0.0;
      sq[j - s0] = mean_plus(acc, p.inv_n, ev);
    }
  }
  __syncthreads();
}

template <int KIND>
__device__ void emit_sparse(const CompressParams& p, const DevChunk& c, Smem& sm, uint32_t s0,
                            uint32_t crank, uint8_t* pay, float* errp, uint32_t stage, uint32_t rrank,
                            bool prehist) {
  const uint32_t L = c.len, k = c.k, cs = p.cs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t prefix = 0, pmask = 0, kk = k, tie_cut = 0;
  bool selected = false;
  // ---- fast exact select of the k-th largest key over the unit (cluster):
  // (1) 10-bit histogram of the top key bits per slice (plain smem atomics);
  // (2) CTA r sums bins [r B, r B + B) over the cluster (DSMEM), B = 1024 / cs;
  // (3) every CTA scans the block totals and that block's bins from the top to
  //     find the bin holding the k-th largest key and the count above it;
  // (4) the bin's keys (a few hundred for gradients) are gathered into CTA 0
  //     (DSMEM atomics), which ranks them exactly; T and the number of T-ties to
  //     take are read back by every CTA.  A bin larger than the capacity (e.g. a
  //     unit of equal values) falls back to the 4 x 8-bit radix select below.
  {
    constexpr int DSH = KIND == K_TOPK ? 21 : 22;   // |q| bits have bit 31 clear; Philox keys use all 32
    if (threadIdx.x == 0) sm.ccount = 0;
    // up to two 10-bit rounds: round 1 histograms only the keys of round 0's bin
    uint32_t bin = 0, above = 0, cnt = 0, dsh = DSH;
    for (int round = 0; round < 2; round++) {
      dsh = DSH - 10 * round;
      const uint32_t pbin = bin;   // round 1: keys with (key >> DSH) == pbin
      const bool built = round == 0 && prehist;   // round 0 built by the producer
      if (!built) {
        for (uint32_t b = threadIdx.x; b < (uint32_t)FNB; b += NT) sm.fh[b] = 0;
        __syncthreads();
      }
#pragma unroll 2
      for (int it = 0; it < IT && !built; it++) {
        const uint32_t i4 = it * NT + threadIdx.x;
        const uint32_t j = s0 + 4 * i4;
        if (j >= L) continue;
        const uint4 kq = keys4<KIND>(sm.q[i4], j, p, c.id, stage, rrank);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const uint32_t key = getu(kq, u);
          if (j + u < L && (round == 0 || (key >> DSH) == pbin))
            atomicAdd(&sm.fh[(key >> dsh) & (FNB - 1)], 1u);
        }
      }
      cluster_sync_all();   // histograms visible to the cluster
      const uint32_t B = FNB / cs;
      uint32_t bt = 0;
      for (uint32_t b = threadIdx.x; b < B; b += NT) {
        uint32_t s = 0;
        for (uint32_t r = 0; r < cs; r++) s += dsmem(sm.fh, r)[crank * B + b];
        sm.bsum[b] = s;
        bt += s;
      }
      bt = __reduce_add_sync(0xffffffffu, bt);
      if (threadIdx.x == 0) sm.btot = 0;
      __syncthreads();
      if (lane == 0) atomicAdd(&sm.btot, bt);
      cluster_sync_all();   // block sums visible
      if (warp == 0) {
        // warp-parallel scan from the top: lane l holds block cs-1-l (one DSMEM
        // round trip), then that block's bins 32 at a time
        auto incl_scan = [&](uint32_t v) {
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
          }
          return v;
        };
        const uint32_t t = (uint32_t)lane < cs ? *dsmem(&sm.btot, cs - 1 - lane) : 0u;
        const uint32_t ti = incl_scan(t);
        const uint32_t hitb = __ballot_sync(0xffffffffu, (uint32_t)lane < cs && above + ti >= k);
        const int lb = __ffs(hitb) - 1;   // exists: the unit holds >= k keys of this round
        const uint32_t blk = cs - 1 - (uint32_t)lb;
        uint32_t ab = above + __shfl_sync(0xffffffffu, ti - t, lb);
        const uint32_t* bs = dsmem(sm.bsum, blk);
        uint32_t bn = 0, cn = 0;
        for (int top = (int)B - 1; top >= 0; top -= 32) {
          const int b = top - lane;
          const uint32_t v = b >= 0 ? bs[b] : 0u;
          const uint32_t vi = incl_scan(v);
          const uint32_t hit = __ballot_sync(0xffffffffu, b >= 0 && ab + vi >= k);
          if (hit) {
            const int lh = __ffs(hit) - 1;
            bn = blk * B + (uint32_t)(top - lh);
            cn = __shfl_sync(0xffffffffu, v, lh);
            ab += __shfl_sync(0xffffffffu, vi - v, lh);
            break;
          }
          ab += __shfl_sync(0xffffffffu, vi, 31);
        }
        if (lane == 0) {
          sm.info[4] = round == 0 ? bn : ((pbin << 10) | bn);
          sm.info[5] = ab;
          sm.info[6] = cn;
        }
      }
      __syncthreads();
      bin = sm.info[4];
      above = sm.info[5];
      cnt = sm.info[6];
      __syncthreads();
      // refine while the bin is large: CTA 0 ranks the candidates in O(C^2 / NT)
      if (cnt <= 256u) break;   // cluster-uniform
    }
    // candidates: the keys with (key >> dsh) == bin, with their unit indices
    if (cnt <= (uint32_t)FCAP) {   // cluster-uniform
      uint32_t* cand = dsmem(sm.fh, 0u);
      uint32_t* ccount = dsmem(&sm.ccount, 0u);
#pragma unroll 2
      for (int it = 0; it < IT; it++) {
        const uint32_t i4 = it * NT + threadIdx.x;
        const uint32_t j = s0 + 4 * i4;
        if (j >= L) continue;
        const uint4 kq = keys4<KIND>(sm.q[i4], j, p, c.id, stage, rrank);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const uint32_t key = getu(kq, u);
          if (j + u < L && (key >> dsh) == bin) {
            const uint32_t slot = atomicAdd(ccount, 1u);
            cand[slot] = key;
            cand[FCAP + slot] = j + u;
          }
        }
      }
      cluster_sync_all();   // candidates gathered in CTA 0
      if (crank == 0) {
        const uint32_t kk2 = k - above;   // rank of the k-th largest inside the bin
        for (uint32_t a = threadIdx.x; a < cnt; a += NT) {
          const uint32_t ka = sm.fh[a];
          uint32_t gt = 0, eq = 0;
          uint32_t b2 = 0;
          for (; b2 + 4 <= cnt; b2 += 4) {   // 4 keys per shared-memory broadcast
            const uint4 kb = *reinterpret_cast<const uint4*>(&sm.fh[b2]);
            gt += (kb.x > ka) + (kb.y > ka) + (kb.z > ka) + (kb.w > ka);
            eq += (kb.x == ka) + (kb.y == ka) + (kb.z == ka) + (kb.w == ka);
          }
          for (; b2 < cnt; b2++) {
            const uint32_t kb = sm.fh[b2];
            gt += kb > ka;
            eq += kb == ka;
          }
          if (gt < kk2 && kk2 <= gt + eq) {   // ka is the kk2-th largest (all such threads agree)
            sm.info[2] = ka;
            sm.info[3] = kk2 - gt;
          }
        }
        __syncthreads();
        // tie cut: the (kk2 - gt)-th smallest index among the candidates equal to T
        const uint32_t T0 = sm.info[2], need = sm.info[3];
        for (uint32_t a = threadIdx.x; a < cnt; a += NT) {
          if (sm.fh[a] != T0) continue;
          const uint32_t ia = sm.fh[FCAP + a];
          uint32_t below = 0;
          for (uint32_t b2 = 0; b2 < cnt; b2++) below += sm.fh[b2] == T0 && sm.fh[FCAP + b2] < ia;
          if (below + 1 == need) sm.info[7] = ia;
        }
      }
      cluster_sync_all();   // T published by CTA 0
      if (threadIdx.x == 0) {
        sm.info[0] = *dsmem(&sm.info[2], 0u);
        sm.info[1] = *dsmem(&sm.info[3], 0u);
        sm.info[4] = *dsmem(&sm.info[7], 0u);
      }
      __syncthreads();
      prefix = sm.info[0];
      kk = sm.info[1];
      tie_cut = sm.info[4];
      selected = true;
      __syncthreads();
    }
  }
  // ---- fallback: radix select of the k-th largest key over the whole unit (cluster)
  if (!selected) cluster_sync_all();   // peers may still read bsum, which hist / tot alias
  for (int pass = 0; pass < 4 && !selected; pass++) {
    const int shift = 24 - 8 * pass;
    uint32_t* h = sm.hist[pass & 1];
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll 2
    for (int it = 0; it < IT; it++) {
      const uint32_t i4 = it * NT + threadIdx.x;
      const uint32_t j = s0 + 4 * i4;
      uint4 kq = make_uint4(0, 0, 0, 0);
      if (j < L) kq = keys4<KIND>(sm.q[i4], j, p, c.id, stage, rrank);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t key = getu(kq, u);
        const bool part = (j + u < L) && ((key & pmask) == prefix);
        const uint32_t dig = part ? ((key >> shift) & 255u) : (0x100u | (uint32_t)lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        if (part && (__ffs(peers) - 1) == lane) atomicAdd(&h[dig], (uint32_t)__popc(peers));
      }
    }
    cluster_sync_all();
    if (threadIdx.x < 256) {
      uint32_t s = 0;
      for (uint32_t r = 0; r < cs; r++) s += dsmem(h, r)[threadIdx.x];
      sm.tot[threadIdx.x] = s;
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t c8[8], S = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        c8[i] = sm.tot[255 - 8 * lane - i];
        S += c8[i];
      }
      uint32_t incl = S;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl = incl - S;
      if (excl < kk && kk <= incl) {
        uint32_t above = excl;
#pragma unroll
        for (int i = 0; i < 8; i++) {
          if (above + c8[i] >= kk) {
            sm.info[0] = 255 - 8 * lane - i;
            sm.info[1] = above;
            break;
          }
          above += c8[i];
        }
      }
    }
    __syncthreads();
    prefix |= sm.info[0] << shift;
    pmask |= 0xFFu << shift;
    kk -= sm.info[1];
    __syncthreads();
  }
  const uint32_t T = prefix;   // the k-th largest key; take kk of the keys equal to T (lowest index)
  const bool scaled = KIND == K_RANDK && p.randk_scaled;
  const float scale = (float)((double)L / (double)k);
  uint32_t* idx_out = reinterpret_cast<uint32_t*>(pay + 8);
  uint8_t* val_out = pay + 8 + 4ull * k;   // fp32, or binary16 values (R23)
  if (selected && k <= (uint32_t)SELCAP) {   // cluster-uniform
    // ---- small k: the selected entries are key > T, or key == T at index <= tie_cut.
    // One pass writes the error and collects this slice's (index, value) pairs in
    // shared memory (bsum / hist, no longer read by peers); a cluster prefix of the
    // per-slice counts and a rank by index place them in ascending order.
    uint32_t* sidx = sm.bsum;
    float* sval = reinterpret_cast<float*>(sm.bsum) + SELCAP;
    if (threadIdx.x == 0) sm.cnt[0] = 0;
    __syncthreads();
    for (int it = 0; it < IT; it++) {
      const uint32_t i4 = it * NT + threadIdx.x;
      const uint32_t j = s0 + 4 * i4;
      const float4 q = sm.q[i4];
      float4 ev = q;
      uint32_t selm = 0;
      if (j < L) {
        const uint4 kq = keys4<KIND>(q, j, p, c.id, stage, rrank);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const uint32_t key = getu(kq, u);
          if (j + u < L && (key > T || (key == T && j + u <= tie_cut))) selm |= 1u << u;
        }
      }
      const uint32_t nsel = __popc(selm);
      const uint32_t wsum = __reduce_add_sync(0xffffffffu, nsel);
      if (wsum) {
        uint32_t incl = nsel;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        uint32_t base = 0;
        if (lane == 31) base = atomicAdd(&sm.cnt[0], incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        uint32_t pos = base + incl - nsel;
#pragma unroll
        for (int u = 0; u < 4; u++)
          if ((selm >> u) & 1u) {
            const float qu = get(q, u);
            const float val = quant_val(scaled ? fmul(qu, scale) : qu, p.f16);   // R23
            sidx[pos] = j + u;
            sval[pos] = val;
            set(ev, u, fsub(qu, val));
            pos++;
          }
      }
      if (errp && j < L) store4_masked(errp, j, L, ev);
    }
    cluster_sync_all();   // per-slice counts visible
    uint32_t base = 0;
    for (uint32_t r = 0; r < crank; r++) base += *dsmem(&sm.cnt[0], r);
    const uint32_t m = sm.cnt[0];
    for (uint32_t a = threadIdx.x; a < m; a += NT) {
      const uint32_t ia = sidx[a];
      uint32_t rank = 0;
      for (uint32_t b2 = 0; b2 < m; b2++) rank += sidx[b2] < ia;
      idx_out[base + rank] = ia;
      put_val(val_out, base + rank, sval[a], p.f16);
    }
    cluster_arrive_relaxed();   // done with peers' smem; the matching wait is at kernel exit
    if (crank == 0 && threadIdx.x == 0) *reinterpret_cast<uint64_t*>(pay) = (uint64_t)k;
    return;
  }
  // ---- per-slice counts -> cluster prefix
  if (threadIdx.x < 2) sm.cnt[threadIdx.x] = 0;
  __syncthreads();
  {
    uint32_t ngt = 0, neq = 0;
    for (int it = 0; it < IT; it++) {
      const uint32_t i4 = it * NT + threadIdx.x;
      const uint32_t j = s0 + 4 * i4;
      if (j >= L) continue;
      const uint4 kq = keys4<KIND>(sm.q[i4], j, p, c.id, stage, rrank);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        if (j + u < L) {
          const uint32_t key = getu(kq, u);
          ngt += key > T;
          neq += key == T;
        }
      }
    }
    ngt = __reduce_add_sync(0xffffffffu, ngt);
    neq = __reduce_add_sync(0xffffffffu, neq);
    if (lane == 0) {
      atomicAdd(&sm.cnt[0], ngt);
      atomicAdd(&sm.cnt[1], neq);
    }
  }
  cluster_sync_all();
  if (threadIdx.x == 0) {
    uint32_t eqb = 0, selb = 0;
    for (uint32_t r = 0; r < crank; r++) {
      const uint32_t* cr = dsmem(sm.cnt, r);
      const uint32_t g = cr[0], e = cr[1];
      selb += g + min(e, kk > eqb ? kk - eqb : 0u);
      eqb += e;
    }
    sm.info[2] = selb;
    sm.info[3] = min(sm.cnt[1], kk > eqb ? kk - eqb : 0u);
  }
  __syncthreads();
  cluster_arrive_relaxed();   // done with peers' smem; the matching wait is at kernel exit
  const uint32_t take_eq = sm.info[3];
  uint32_t sel_run = sm.info[2], eq_run = 0;
  // ---- ordered compaction (index ascending) + error write
  for (int it = 0; it < IT; it++) {
    const uint32_t i4 = it * NT + threadIdx.x;
    const uint32_t j = s0 + 4 * i4;
    const float4 q = sm.q[i4];
    uint32_t gtm = 0, eqm = 0;
    if (j < L) {
      const uint4 kq = keys4<KIND>(q, j, p, c.id, stage, rrank);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t key = getu(kq, u);
        if (j + u < L) {
          gtm |= (uint32_t)(key > T) << u;
          eqm |= (uint32_t)(key == T) << u;
        }
      }
    }
    float4 ev = q;
    if (__syncthreads_or((int)(gtm | eqm))) {
      uint32_t te, ts;
      const uint32_t ee = block_excl_scan(__popc(eqm), sm.scan, te);
      uint32_t selm = gtm, rr = eq_run + ee;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if ((eqm >> u) & 1u) {
          if (rr < take_eq) selm |= 1u << u;
          rr++;
        }
      uint32_t pos = sel_run + block_excl_scan(__popc(selm), sm.scan, ts);
#pragma unroll
      for (int u = 0; u < 4; u++)
        if ((selm >> u) & 1u) {
          const float qu = get(q, u);
          const float val = quant_val(scaled ? fmul(qu, scale) : qu, p.f16);   // R23
          idx_out[pos] = j + u;
          put_val(val_out, pos, val, p.f16);
          set(ev, u, fsub(qu, val));
          pos++;
        }
      eq_run += te;
      sel_run += ts;
    }
    if (errp && j < L) store4_masked(errp, j, L, ev);
  }
  if (crank == 0 && threadIdx.x == 0) *reinterpret_cast<uint64_t*>(pay) = (uint64_t)k;
}

// ---------------------------------------------------------------- raw tiles
template <bool SERVER>
__device__ __forceinline__ void raw_tile(const CompressParams& p, const Tile& tl) {
  const DevChunk c = p.chunks[tl.chunk];
  float* out = reinterpret_cast<float*>(p.out + c.pay);
  const uint32_t L = c.len;
  bool bad = false;
  for (uint32_t i = threadIdx.x; 4 * i < tl.len; i += NT) {
    const uint32_t j = tl.start + 4 * i;
    float4 v;
    if (!SERVER) {
      v = load4_masked(p.grad + c.off, j, L);   // raw units: delta = g, no EF (R3)
      if (p.check_finite) bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    } else {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      for (uint32_t r = 0; r < p.n; r++) {
        const float4 d = load4_masked(reinterpret_cast<const float*>(p.recv + r * p.slot_bytes + c.recv), j, L);
        a0 += (double)d.x; a1 += (double)d.y; a2 += (double)d.z; a3 += (double)d.w;
      }
      v = make_float4(mean_plus(a0, p.inv_n, 0.0), mean_plus(a1, p.inv_n, 0.0),
                      mean_plus(a2, p.inv_n, 0.0), mean_plus(a3, p.inv_n, 0.0));
    }
    store4_masked(out, j, L, v);
  }
  if (bad) atomicOr(p.flag, 1u);
}

// ---------------------------------------------------------------- the kernel
template <int KIND, bool SERVER>
__global__ void __launch_bounds__(NT, 3) compress_kernel(const __grid_constant__ CompressParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t cid = blockIdx.x / p.cs;
  const uint32_t crank = cta_rank_in_cluster();
  if (cid >= p.n_items) {   // cluster-uniform: raw tiles, no cluster barriers
    const uint32_t ti = (cid - p.n_items) * p.cs + crank;
    if (ti < p.n_raw_tiles) raw_tile<SERVER>(p, p.raw_tiles[ti]);
    return;
  }
  {
    const DevChunk c = p.chunks[p.items[cid]];
    const uint32_t s0 = crank * SLICE;
    uint8_t* pay = p.out + c.pay;
    float* errp = p.use_ef ? (SERVER ? p.etl + c.etl : p.err + c.off) : nullptr;
    const uint32_t stage = SERVER ? 1u : 0u;
    const uint32_t rrank = SERVER ? 0u : p.rank;
    if (SERVER) {
      produce_server_sparse(p, c, sm, s0);
    } else {
      for (uint32_t b = threadIdx.x; b < (uint32_t)FNB; b += NT) sm.fh[b] = 0;
      __syncthreads();
      produce_worker<KIND>(p, c, sm, s0);
    }
    __syncthreads();
    emit_sparse<KIND>(p, c, sm, s0, crank, pay, errp, stage, rrank, !SERVER);
    cluster_wait();   // no CTA exits while a peer may still read its shared memory
  }
}

template <int KIND, bool SERVER>
static cudaError_t launch_t(const CompressParams& p, cudaStream_t s) {
  const uint32_t nclusters = p.n_items + (p.n_raw_tiles + p.cs - 1) / p.cs;
  if (nclusters == 0) return cudaSuccess;
  auto fn = compress_kernel<KIND, SERVER>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * p.cs);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = sizeof(Smem);
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = p.cs;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, p);
}

template <int KIND, bool SERVER>
static cudaError_t max_clusters_t(uint32_t cs, int* out) {
  auto fn = compress_kernel<KIND, SERVER>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = sizeof(Smem);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cs;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, fn, &cfg);
}

// the cluster kernels serve the sparse kinds (top-k, random-k) and their raw
// units; the norm-based kinds run in the streaming kernels (kernels_cstream.cu)
#define BPC_DISPATCH(KIND_, SERVER_, CALL)                                     \
  switch (KIND_) {                                                             \
    case K_TOPK: return SERVER_ ? CALL(K_TOPK, true) : CALL(K_TOPK, false);    \
    case K_RANDK: return SERVER_ ? CALL(K_RANDK, true) : CALL(K_RANDK, false); \
  }                                                                            \
  return cudaErrorInvalidValue;

cudaError_t launch_compress(int kind, bool server, const CompressParams& p, cudaStream_t s) {
#define CALL_LAUNCH(K, S) launch_t<K, S>(p, s)
  BPC_DISPATCH(kind, server, CALL_LAUNCH)
#undef CALL_LAUNCH
}

cudaError_t compress_max_active_clusters(int kind, bool server, uint32_t cs, int* out) {
#define CALL_MAX(K, S) max_clusters_t<K, S>(cs, out)
  BPC_DISPATCH(kind, server, CALL_MAX)
#undef CALL_MAX
}

}  // namespace bpc
