// kernels_sparse.cu — worker compress and server
// decompress-sum-recompress (A5-A7) for the sparse kinds, top-k (R9) and
// random-k (R10), on sm_100a.  Per side:
//
//   sparse_prep    one CTA per unit.  Server: applies the n ranks' payload
//                  entries, Delta_j = fl32(fl64(sum_i dec_i,j) (1/n) + e~_j)
//                  (Alg. 4 l.10; R5), in place at those j only:
//                  elsewhere Delta_j = fl32(0 + e~_j) = e~_j, because e~ is
//                  never -0 (see the dense pass).  Both sides: a candidate
//                  threshold G_u (top-k: about the m-th largest key of a
//                  4096-element sample of q / Delta, m = mu + 3 sqrt(mu) + 6,
//                  mu = k S / L; random-k: the uniform keys' quantile
//                  1 - (k + 8 sqrt(k) + 64) / L).  G only decides which elements
//                  are examined exactly; any G gives the same result.
//   streaming     cstream_kernel<C_TOPK / C_RANDK> (kernels_cstream.cu): the TMA
//                  pipeline of the norm kinds.  Worker: q = g + e (Alg. 4 l.5,
//                  PAPER.md:241), e := q (bulk store), raw units copied.  Server:
//                  reads Delta (e~ + the applied entries; 4 B/element), raw units
//                  averaged.  Every element with key >= G_u joins its slice's
//                  index-ordered sub-list of the unit's candidates as (index,
//                  key), so the select reads the lists contiguously and gathers
//                  values only for the k selected elements.
//   sparse_select  if the unit has k <= c <= cap candidates, every element
//                  outside them has key < G <= T (the k-th largest key), so the
//                  exact selection (keys desc, index asc, R9/R10) is a radix
//                  select over the c candidates: one 128-thread CTA per unit
//                  (c <= 4096, k <= 512), else one 512-thread CTA per unit
//                  (c <= SEL_CAP), else an exact
//                  radix select + ordered compaction over the whole unit.  Emits
//                  the payload [u64 k][k idx asc][k val] (l.6 / l.11) and the
//                  operator-fused EF update e_j = q_j - val_j at the k selected
//                  indices only (l.7 / l.13).
// HBM per element: worker 12 B (g, e read, e written), server 4 B (Delta read).
#include "device.cuh"

namespace bpc {

enum { SP_TOPK = 3, SP_RANDK = 4 };

constexpr int SG_NT = 256;        // prep kernel threads
constexpr int SG_S = 4096;        // sample size (16 runs of 256)
constexpr int SE_NT = 512;        // CTA select kernel threads
constexpr uint32_t SW_CAP = 4096; // unit select: max candidates
constexpr uint32_t SW_KMAX = 512; // unit select: max k
constexpr int SA_NT = 256;        // server apply: entries per block

__device__ __forceinline__ uint32_t topk_key(float v) { return __float_as_uint(v) & 0x7fffffffu; }
template <int KIND>
__device__ __forceinline__ uint32_t sel_key(float v, uint32_t j, const SparseParams& p, uint32_t id) {
  if (KIND == SP_TOPK) return topk_key(v);
  // random-k: the k smallest Philox words = the k largest complements (R10); t is
  // the step counter in device memory (read-only in these kernels, L1-resident)
  const uint4 w = rng4(p.seed, j >> 2, id, p.st->t, p.stage, p.rrank);
  const uint32_t u = j & 3u;
  return ~(u == 0 ? w.x : (u == 1 ? w.y : (u == 2 ? w.z : w.w)));
}

// the unit's values V_j after the dense pass: worker q (e if use_ef, else g),
// server Delta (e~ if use_ef, else the zero-based scratch)
__device__ __forceinline__ const float* unit_values(const SparseParams& p, const DevChunk& c) {
  return p.server ? p.vals + c.etl : (p.use_ef ? p.vals + c.off : p.grad + c.off);
}

// ---------------------------------------------------------------- helpers
// histogram increment with warp aggregation: lanes holding the same bin add once
// (the top digits of the keys near a unit's threshold share a handful of bins,
// so plain shared-memory atomics would serialise)
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin, bool valid) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t act = __activemask();
  const uint32_t peers = __match_any_sync(act, valid ? bin : (0x80000000u | lane));
  if (valid && (uint32_t)(__ffs(peers) - 1) == lane) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}

// one warp: the bin of hist[0, 256) holding the kk-th largest key counting from
// the top bin; returns (bin, keys in higher bins) in every lane
__device__ __forceinline__ uint2 warp_find_bin256(const uint32_t* hist, uint32_t kk) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t c8[8], s = 0;   // lane l: bins 255 - 8 l - i
#pragma unroll
  for (int i = 0; i < 8; i++) {
    c8[i] = hist[255 - 8 * lane - i];
    s += c8[i];
  }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  const uint32_t excl = incl - s;
  uint32_t bin = 0, ab = 0;
  const bool mine = excl < kk && kk <= incl;
  if (mine) {
    uint32_t a = excl;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (a + c8[i] >= kk) {
        bin = 255 - 8 * lane - i;
        ab = a;
        break;
      }
      a += c8[i];
    }
  }
  const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
  return make_uint2(__shfl_sync(0xffffffffu, bin, src), __shfl_sync(0xffffffffu, ab, src));
}

template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* scan, uint32_t* total) {
  constexpr int NW = NT / 32;
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
    const uint32_t w = lane < NW ? scan[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NW) scan[lane] = wi - w;
    if (lane == NW - 1) scan[NW] = wi;
  }
  __syncthreads();
  const uint32_t r = scan[warp] + incl - v;
  *total = scan[NW];
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint32_t lower_bound_u(const uint32_t* a, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ bool holds(const uint32_t* a, uint32_t n, uint32_t j, uint32_t* pos) {
  *pos = lower_bound_u(a, n, j);
  return *pos < n && a[*pos] == j;
}

// rank r's payload of unit c: [u64 k][k idx][k val]
__device__ __forceinline__ const uint8_t* rank_payload(const SparseParams& p, const DevChunk& c, uint32_t r) {
  return p.recv + r * p.slot_bytes + c.recv;
}

// ================================================================ prep
// server: the ranks' entries, one thread per entry; block b covers entries
// [first, first + 256) of unit apply_blk[b].x's n k entries (rank-major)
template <int KIND>
__global__ void __launch_bounds__(SA_NT) sparse_apply_kernel(const __grid_constant__ SparseParams p) {
  const uint2 blk = p.apply_blk[blockIdx.x];
  const uint32_t u = blk.x;
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t k = c.k, n = p.n;
  float* V = const_cast<float*>(unit_values(p, c));
  const uint32_t i = blk.y + threadIdx.x;
  if (i >= n * k) return;
  const uint32_t r = i / k, e = i - r * k;
  auto idx_of = [&](uint32_t rr) { return reinterpret_cast<const uint32_t*>(rank_payload(p, c, rr) + 8); };
  const uint32_t j = idx_of(r)[e];
  // the first rank holding j sums every holder in rank order (R5)
  uint32_t pos;
  for (uint32_t r2 = 0; r2 < r; r2++)
    if (holds(idx_of(r2), k, j, &pos)) return;
  double acc = 0.0;
  acc += (double)get_val(rank_payload(p, c, r) + 8 + 4ull * k, e, p.f16);
  for (uint32_t r2 = r + 1; r2 < n; r2++)
    if (holds(idx_of(r2), k, j, &pos)) acc += (double)get_val(rank_payload(p, c, r2) + 8 + 4ull * k, pos, p.f16);
  V[j] = mean_plus(acc, p.inv_n, (double)V[j]);   // no EF: V is the zeroed scratch
}

// the candidate threshold of each unit
template <int KIND>
__global__ void __launch_bounds__(SG_NT) sparse_prep_kernel(const __grid_constant__ SparseParams p) {
  __shared__ uint32_t red[SG_NT / 32];
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t pick[2];
  const uint32_t u = blockIdx.x;
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t L = c.len, k = c.k;
  float* V = const_cast<float*>(unit_values(p, c));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (KIND == SP_TOPK && p.server && !p.use_ef) {   // Delta is +0 outside the ranks' entries
    if (threadIdx.x == 0) p.guess[u] = 1u;
    return;
  }
  // ---- candidate threshold
  uint32_t G;
  if (KIND == SP_RANDK) {
    // uniform 32-bit keys: expected candidates k + 8 sqrt(k) + 64
    const double want = (double)k + 8.0 * sqrt((double)k) + 64.0;
    G = want >= (double)L ? 0u : (uint32_t)fmin(4294967295.0, floor((1.0 - want / (double)L) * 4294967296.0));
  } else {
    // 16 runs of 256 (or the whole unit when L <= 4096); all loads in flight
    const uint32_t S = L < (uint32_t)SG_S ? L : (uint32_t)SG_S;
    uint32_t key[16];
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const uint32_t s = threadIdx.x + r * SG_NT;
      key[r] = 0;
      if (s < S) {
        const uint32_t pos = L <= (uint32_t)SG_S ? s : (uint32_t)(((uint64_t)r * (L - 256)) / 15) + threadIdx.x;
        float v;
        if (p.server) {
          v = V[pos];   // Delta (entries applied above; Delta = e~ elsewhere)
        } else {
          const float g = p.grad[c.off + pos];
          v = p.use_ef ? fadd(g, p.vals[c.off + pos]) : g;
        }
        key[r] = topk_key(v);
      }
    }
    // the m-th largest sample key, its bits 30..10 by two radix passes (11 + 10
    // bits, shared-memory histograms): G is the lower edge of the 2^-13-wide
    // magnitude bin holding it, the largest multiple of 2^10 with >= m sample
    // keys at or above it
    const uint32_t m = L <= (uint32_t)SG_S ? k : (uint32_t)min(S, sparse_sample_rank(k, L));
    uint32_t g = 0, rank = m;
    for (int pass = 0; pass < 2; pass++) {
      const int sh = pass ? 10 : 20, nb = pass ? 1024 : 2048, per = nb / SG_NT;
      for (int b = threadIdx.x; b < nb; b += SG_NT) hist[b] = 0;
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const uint32_t sidx = threadIdx.x + r * SG_NT;
        if (sidx < S && (pass == 0 || (key[r] >> 20) == (g >> 20)))
          atomicAdd(&hist[(key[r] >> sh) & (uint32_t)(nb - 1)], 1u);
      }
      __syncthreads();
      // thread t owns bins nb - 1 - per t - j (descending): block scan of the counts
      // from the top; the owner of the rank-th largest publishes (bin, keys above it)
      uint32_t tot = 0;
      for (int j = 0; j < per; j++) tot += hist[nb - 1 - per * threadIdx.x - j];
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (lane == 31) red[warp] = incl;
      __syncthreads();
      for (int w = 0; w < warp; w++) incl += red[w];
      const uint32_t before = incl - tot;
      if (before < rank && rank <= incl) {
        uint32_t run = before;
        for (int j = 0; j < per; j++) {
          const uint32_t cj = hist[nb - 1 - per * threadIdx.x - j];
          if (run + cj >= rank) {
            pick[0] = (uint32_t)(nb - 1 - per * threadIdx.x - j);
            pick[1] = run;
            break;
          }
          run += cj;
        }
      }
      __syncthreads();
      g |= pick[0] << sh;
      rank -= pick[1];
      __syncthreads();   // hist, red and pick are reused by the next pass
    }
    // key 0 (magnitude +-0) is never a useful threshold: with fewer than k nonzero
    // values the select kernel takes its exact whole-unit path
    G = g > 1u ? g : 1u;
  }
  if (threadIdx.x == 0) p.guess[u] = G;
}

// ================================================================ select
// The unit's candidates are index-ordered per slice and the slices are in index
// order, so the concatenated list is sorted by index: after the radix select of
// T, one ordered pass (ties counted in index order) emits the payload -- no sort.

// server without EF: the scratch goes back to all-zero (only the ranks' entries
// were written by sparse_apply), by `nt` threads from `tid`
__device__ __forceinline__ void clear_scratch(const SparseParams& p, const DevChunk& c, float* V, uint32_t tid,
                                              uint32_t nt) {
  for (uint32_t i = tid; i < p.n * c.k; i += nt) {
    const uint32_t r = i / c.k, e = i - r * c.k;
    V[reinterpret_cast<const uint32_t*>(rank_payload(p, c, r) + 8)[e]] = 0.f;
  }
}

// one payload entry (position pos) of the selected index j with its value q
__device__ __forceinline__ void emit_entry(const SparseParams& p, float* V, uint8_t* pay, uint32_t k, uint32_t pos,
                                           uint32_t j, float q, bool scaled, float scale) {
  const float val = quant_val(scaled ? fmul(q, scale) : q, p.f16);   // R23
  reinterpret_cast<uint32_t*>(pay + 8)[pos] = j;
  put_val(pay + 8 + 4ull * k, pos, val, p.f16);
  if (p.use_ef) V[j] = fsub(q, val);   // e = q - dec (operator fusion: O(k))
}

// the unit's candidate count (sum over its slices, each at most cs) and whether
// a slice overflowed its sub-list
__device__ __forceinline__ uint32_t unit_ns(const DevChunk& c) { return (c.len + 8191u) / 8192u; }

// ---- one small CTA (SU_NT threads) per unit: c <= SW_CAP candidates, k <= SW_KMAX
constexpr int SU_NT = 128;                 // threads of the unit select
constexpr int SU_W = SU_NT / 32;
constexpr int SU_R = SW_CAP / SU_NT;       // candidates per thread (registers)
struct UnitSel {
  uint32_t idx[SW_CAP];   // candidate indices, ascending
  uint32_t key[SW_CAP];   // keys, then the selected indices
  uint32_t x[SW_CAP];     // the keys still sharing T's prefix (the threshold search)
  uint32_t sbase[33];     // the sub-lists' offsets in the concatenated list; [32] = count
  uint32_t red[4][SU_W];  // per-warp partials of the block reductions
};

// block reductions over SU_NT threads (all threads call; a barrier inside)
__device__ __forceinline__ uint32_t su_sum(uint32_t v, uint32_t (&red)[SU_W], uint32_t lane, uint32_t w) {
  v = __reduce_add_sync(0xffffffffu, v);
  if (lane == 0) red[w] = v;
  __syncthreads();
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < SU_W; i++) t += red[i];
  return t;
}

template <int KIND>
__global__ void __launch_bounds__(SU_NT) sparse_select_unit_kernel(const __grid_constant__ SparseParams p) {
  extern __shared__ __align__(16) unsigned char suraw[];
  UnitSel& s = *reinterpret_cast<UnitSel*>(suraw);
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t u = blockIdx.x;
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t L = c.len, k = c.k;
  if (L > SEL_LMAX) return;   // per-tensor unit: the large-unit path (sparse_large_*)
  const uint32_t ns = unit_ns(c), cs = (p.cand_off[u + 1] - p.cand_off[u]) / ns;
  if (w == 0) {   // lane l: slice l's count (a chunk unit has <= 32 slices)
    const uint32_t sc = lane < ns ? p.scnt[p.first_slice[u] + lane] : 0u;
    const bool ovf = __any_sync(0xffffffffu, sc > cs);
    uint32_t incl = sc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    s.sbase[lane] = incl - sc;
    if (lane == 31) s.sbase[32] = ovf ? 0xffffffffu : incl;
  }
  __syncthreads();
  const uint32_t cnt = s.sbase[32];
  if (cnt == 0xffffffffu || cnt < k || cnt > SW_CAP || k > SW_KMAX) {
    if (tid == 0) p.big[u] = 1;   // the CTA select kernel takes this unit
    return;
  }
  float* V = const_cast<float*>(unit_values(p, c));
  uint8_t* pay = p.out + c.pay;
  const uint2* cand = p.cand + p.cand_off[u];
  // the sub-lists (index, key), concatenated in slice order (= index order): warp
  // w takes slices w, w + 4, ..; two entries per lane and slice, 16 loads in flight
  {
    uint2 v[16];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t sl = w + SU_W * q;
      const uint32_t n_sl = sl < ns ? (sl + 1 < ns ? s.sbase[sl + 1] : cnt) - s.sbase[sl] : 0u;
      v[2 * q] = lane < n_sl ? cand[sl * cs + lane] : make_uint2(0u, 0u);
      v[2 * q + 1] = lane + 32 < n_sl ? cand[sl * cs + lane + 32] : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t sl = w + SU_W * q;
      if (sl >= ns) continue;
      const uint32_t b_sl = s.sbase[sl], n_sl = (sl + 1 < ns ? s.sbase[sl + 1] : cnt) - b_sl;
      if (lane < n_sl) {
        s.idx[b_sl + lane] = v[2 * q].x;
        s.key[b_sl + lane] = v[2 * q].y;
      }
      if (lane + 32 < n_sl) {
        s.idx[b_sl + lane + 32] = v[2 * q + 1].x;
        s.key[b_sl + lane + 32] = v[2 * q + 1].y;
      }
      for (uint32_t i = lane + 64; i < n_sl; i += 32) {
        const uint2 e = cand[sl * cs + i];
        s.idx[b_sl + i] = e.x;
        s.key[b_sl + i] = e.y;
      }
    }
  }
  __syncthreads();
  // T = the k-th largest key, bit by bit from the top over the keys that still
  // share T's prefix: a bit on which they all agree is taken as it is; a bit
  // that splits them is decided by one count, and the chosen half is compacted
  // into x[] (the set is first read into registers, so the writes are safe)
  const uint32_t* A = s.key;
  uint32_t na = cnt, above = 0, prefix = 0;
  uint32_t andv, orv;
  {
    uint32_t x0 = 0xffffffffu, x1 = 0u;
    for (uint32_t i = tid; i < na; i += SU_NT) {
      x0 &= A[i];
      x1 |= A[i];
    }
    x0 = __reduce_and_sync(0xffffffffu, x0);
    x1 = __reduce_or_sync(0xffffffffu, x1);
    if (lane == 0) {
      s.red[0][w] = x0;
      s.red[1][w] = x1;
    }
    __syncthreads();
    andv = 0xffffffffu;
    orv = 0u;
#pragma unroll
    for (int i = 0; i < SU_W; i++) {
      andv &= s.red[0][i];
      orv |= s.red[1][i];
    }
    __syncthreads();
  }
  for (int bit = 31; bit >= 0; bit--) {
    const uint32_t m = 1u << bit;
    if (!((andv ^ orv) & m)) {   // every key left agrees on this bit
      prefix |= andv & m;
      continue;
    }
    uint32_t r[SU_R];
    uint32_t c1 = 0;
#pragma unroll
    for (int j = 0; j < SU_R; j++) {
      if (SU_NT * (uint32_t)j >= na) break;   // (uniform: the loops run ceil(na / SU_NT) times)
      const uint32_t i = tid + SU_NT * j;
      r[j] = i < na ? A[i] : 0u;
      c1 += (i < na && (r[j] & m)) ? 1u : 0u;
    }
    const uint32_t cset = su_sum(c1, s.red[2], lane, w);   // (barrier: every read of A done)
    const bool take1 = above + cset >= k;   // the k-th largest has this bit set
    if (take1) prefix |= m;
    else above += cset;
    // keep the chosen half: warp counts -> warp bases -> ballot positions
    uint32_t kept = 0;
#pragma unroll
    for (int j = 0; j < SU_R; j++) {
      if (SU_NT * (uint32_t)j >= na) break;
      const uint32_t i = tid + SU_NT * j;
      kept += (i < na && (((r[j] & m) != 0) == take1)) ? 1u : 0u;
    }
    kept = __reduce_add_sync(0xffffffffu, kept);
    if (lane == 0) s.red[3][w] = kept;
    __syncthreads();
    uint32_t base = 0, total = 0;
#pragma unroll
    for (int i = 0; i < SU_W; i++) {
      base += (uint32_t)i < w ? s.red[3][i] : 0u;
      total += s.red[3][i];
    }
    uint32_t x0 = 0xffffffffu, x1 = 0u;
#pragma unroll
    for (int j = 0; j < SU_R; j++) {
      if (SU_NT * (uint32_t)j >= na) break;
      const uint32_t i = tid + SU_NT * j;
      const bool keep = i < na && (((r[j] & m) != 0) == take1);
      const uint32_t bl = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        s.x[base + __popc(bl & ((1u << lane) - 1))] = r[j];
        x0 &= r[j];
        x1 |= r[j];
      }
      base += __popc(bl);
    }
    x0 = __reduce_and_sync(0xffffffffu, x0);
    x1 = __reduce_or_sync(0xffffffffu, x1);
    if (lane == 0) {
      s.red[0][w] = x0;
      s.red[1][w] = x1;
    }
    __syncthreads();
    andv = 0xffffffffu;
    orv = 0u;
#pragma unroll
    for (int i = 0; i < SU_W; i++) {
      andv &= s.red[0][i];
      orv |= s.red[1][i];
    }
    A = s.x;
    na = total;
    __syncthreads();   // red[] is reused
  }
  const uint32_t T = prefix;
  const uint32_t need = k - above;   // T-ties to take (lowest indices first)
  // ordered pass over the index-sorted candidates, SU_NT at a time: the selected
  // indices, in order, compacted to the front of key[] (read before any write)
  uint32_t eq_run = 0, out_run = 0;
  for (uint32_t i0 = 0; i0 < cnt; i0 += SU_NT) {
    const uint32_t i = i0 + tid;
    const uint32_t key = i < cnt ? s.key[i] : 0u;
    const uint32_t ix = i < cnt ? s.idx[i] : 0u;
    const bool eq = i < cnt && key == T;
    const uint32_t be = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) s.red[0][w] = __popc(be);
    __syncthreads();
    uint32_t eb = eq_run, et = 0;
#pragma unroll
    for (int q = 0; q < SU_W; q++) {
      eb += (uint32_t)q < w ? s.red[0][q] : 0u;
      et += s.red[0][q];
    }
    const uint32_t er = eb + __popc(be & ((1u << lane) - 1));
    const bool sel = i < cnt && (key > T || (eq && er < need));
    const uint32_t bs = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) s.red[1][w] = __popc(bs);
    __syncthreads();
    uint32_t ob = out_run, ot = 0;
#pragma unroll
    for (int q = 0; q < SU_W; q++) {
      ob += (uint32_t)q < w ? s.red[1][q] : 0u;
      ot += s.red[1][q];
    }
    if (sel) s.key[ob + __popc(bs & ((1u << lane) - 1))] = ix;   // position <= i0 < later reads
    eq_run += et;
    out_run += ot;
    __syncthreads();
  }
  // emit, value reads batched 4 deep per thread
  const bool scaled = KIND == SP_RANDK && p.randk_scaled;
  const float scale = (float)((double)L / (double)k);
  for (uint32_t i0 = 0; i0 < k; i0 += 4 * SU_NT) {
    float qv[4];
    uint32_t jj[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const uint32_t i = i0 + SU_NT * r + tid;
      jj[r] = i < k ? s.key[i] : 0u;
      qv[r] = i < k ? V[jj[r]] : 0.f;
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const uint32_t i = i0 + SU_NT * r + tid;
      if (i < k) emit_entry(p, V, pay, k, i, jj[r], qv[r], scaled, scale);
    }
  }
  __syncthreads();
  if (p.server && !p.use_ef) clear_scratch(p, c, V, tid, SU_NT);
  if (tid == 0) *reinterpret_cast<uint64_t*>(pay) = (uint64_t)k;
}

// ---- one CTA per unit: larger candidate lists, or the exact whole-unit path
struct SelSmem {
  uint32_t hist[256];
  uint32_t info[4];
  uint32_t scan[SE_NT / 32 + 1];
  uint32_t sbase[33];   // the sub-lists' offsets in the concatenated list
};

// the rank-th largest (1-based) key over `n` keys given by key_of(i), 4 x 8-bit
// digits; returns the key, *above = keys strictly larger
template <class KeyOf>
__device__ uint32_t block_kth_largest(KeyOf key_of, uint32_t n, uint32_t rank, SelSmem& sm, uint32_t* above) {
  uint32_t prefix = 0, pmask = 0, kk = rank, ab = 0;
  for (int pass = 0; pass < 4; pass++) {
    const int sh = 24 - 8 * pass;
    for (uint32_t b = threadIdx.x; b < 256; b += SE_NT) sm.hist[b] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += SE_NT) {
      const uint32_t key = key_of(i);
      hist_add(sm.hist, (key >> sh) & 255u, (key & pmask) == prefix);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const uint2 fb = warp_find_bin256(sm.hist, kk);
      if (threadIdx.x == 0) {
        sm.info[0] = fb.x;
        sm.info[1] = fb.y;
      }
    }
    __syncthreads();
    prefix |= sm.info[0] << sh;
    pmask |= 0xffu << sh;
    kk -= sm.info[1];
    ab += sm.info[1];
    __syncthreads();
  }
  *above = ab;
  return prefix;
}

// ordered emission over `n` index-ascending items (4 consecutive per thread per
// round): item i is selected if key > T, or key == T among the first `need`
// T-ties in index order
template <class ItemOf>
__device__ void block_ordered_emit(ItemOf item_of, uint32_t n, uint32_t T, uint32_t need, SelSmem& sm,
                                   const SparseParams& p, float* V, uint8_t* pay, uint32_t k, bool scaled,
                                   float scale) {
  uint32_t eq_run = 0, out_run = 0;
  for (uint32_t base = 0; base < n; base += 4 * SE_NT) {
    const uint32_t i0 = base + 4 * threadIdx.x;
    uint32_t jj[4], gtm = 0, eqm = 0;
    float qv[4];
#pragma unroll
    for (int e = 0; e < 4; e++) {
      jj[e] = 0;
      qv[e] = 0.f;
      if (i0 + e < n) {
        uint32_t key;
        item_of(i0 + e, &jj[e], &key, &qv[e]);
        gtm |= (uint32_t)(key > T) << e;
        eqm |= (uint32_t)(key == T) << e;
      }
    }
    uint32_t teq;
    const uint32_t er = block_excl_scan_u32<SE_NT>(__popc(eqm), sm.scan, &teq);
    uint32_t selm = gtm, rr = eq_run + er;
#pragma unroll
    for (int e = 0; e < 4; e++)
      if ((eqm >> e) & 1u) {
        if (rr < need) selm |= 1u << e;
        rr++;
      }
    uint32_t tsel;
    uint32_t pos = out_run + block_excl_scan_u32<SE_NT>(__popc(selm), sm.scan, &tsel);
#pragma unroll
    for (int e = 0; e < 4; e++)
      if ((selm >> e) & 1u) emit_entry(p, V, pay, k, pos++, jj[e], qv[e], scaled, scale);
    eq_run += teq;
    out_run += tsel;
  }
}

template <int KIND>
__global__ void __launch_bounds__(SE_NT) sparse_select_kernel(const __grid_constant__ SparseParams p) {
  // dynamic: [sel_cap] candidate indices | [sel_cap] keys
  extern __shared__ __align__(16) uint32_t sx[];
  __shared__ SelSmem sm;
  const uint32_t u = blockIdx.x;
  if (!p.big[u]) return;   // the warp kernel selected this unit
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t L = c.len, k = c.k;
  float* V = const_cast<float*>(unit_values(p, c));
  uint8_t* pay = p.out + c.pay;
  const bool scaled = KIND == SP_RANDK && p.randk_scaled;
  const float scale = (float)((double)L / (double)k);
  const uint32_t ns = unit_ns(c), cs = (p.cand_off[u + 1] - p.cand_off[u]) / ns;
  const uint2* cand = p.cand + p.cand_off[u];
  if (threadIdx.x < 32) {   // the sub-lists' offsets (ns <= 32)
    const uint32_t lane = threadIdx.x;
    const uint32_t sc = lane < ns ? p.scnt[p.first_slice[u] + lane] : 0u;
    const bool ovf = __any_sync(0xffffffffu, sc > cs);
    uint32_t incl = sc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    sm.sbase[lane] = incl - sc;
    if (lane == 31) sm.sbase[32] = ovf ? 0xffffffffu : incl;
  }
  __syncthreads();
  const uint32_t cnt = sm.sbase[32];
  const uint32_t SC = p.sel_cap;
  uint32_t above, T;
  if (cnt != 0xffffffffu && cnt >= k && cnt <= SC) {
    // ---- exact selection among the candidates (every other key < G <= T)
    uint32_t* ci = sx;
    uint32_t* ck = sx + SC;
    for (uint32_t sl = 0; sl < ns; sl++) {
      const uint32_t b0 = sm.sbase[sl], n_sl = (sl + 1 < ns ? sm.sbase[sl + 1] : cnt) - b0;
      for (uint32_t i = threadIdx.x; i < n_sl; i += SE_NT) {
        const uint2 e = cand[sl * cs + i];
        ci[b0 + i] = e.x;
        ck[b0 + i] = e.y;
      }
    }
    __syncthreads();
    T = block_kth_largest([&](uint32_t i) { return ck[i]; }, cnt, k, sm, &above);
    block_ordered_emit(
        [&](uint32_t i, uint32_t* j, uint32_t* key, float* q) {
          *j = ci[i];
          *key = ck[i];
          *q = V[*j];
        },
        cnt, T, k - above, sm, p, V, pay, k, scaled, scale);
  } else {
    // ---- exact over the whole unit
    T = block_kth_largest(
        [&](uint32_t j) { return sel_key<KIND>(KIND == SP_TOPK ? V[j] : 0.f, j, p, c.id); }, L, k, sm, &above);
    block_ordered_emit(
        [&](uint32_t i, uint32_t* j, uint32_t* key, float* q) {
          *j = i;
          *q = V[i];
          *key = sel_key<KIND>(*q, i, p, c.id);
        },
        L, T, k - above, sm, p, V, pay, k, scaled, scale);
  }
  __syncthreads();
  if (p.server && !p.use_ef) clear_scratch(p, c, V, threadIdx.x, SE_NT);
  if (threadIdx.x == 0) {
    *reinterpret_cast<uint64_t*>(pay) = (uint64_t)k;
    p.big[u] = 0;
  }
}

// ================================================================ large units
// Per-tensor units (NEXT #4) can hold 10^8 elements with k ~ 10^5:
// T is found by a multi-CTA radix select over the unit's candidates (or over the
// whole unit when they do not suffice), then the selection is emitted in index
// order by a count / scan / compaction over the unit's 2^13-element slices.
// lstate[8 u + .]: 0 prefix, 1 pmask, 2 kk, 3 above, 4 work mode (1 = candidates)

template <int KIND>
__device__ __forceinline__ uint32_t large_key(const SparseParams& p, const DevChunk& c, const float* V, uint32_t j) {
  return sel_key<KIND>(KIND == SP_TOPK ? V[j] : 0.f, j, p, c.id);
}

// per large unit: the candidates suffice (no sub-list overflow, >= k of them)?
__global__ void sparse_large_init(const __grid_constant__ SparseParams p) {
  __shared__ uint32_t tot, ovf;
  const uint32_t lu = blockIdx.x, u = p.large_units[lu];
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t ns = unit_ns(c), cs = (p.cand_off[u + 1] - p.cand_off[u]) / ns;
  if (threadIdx.x == 0) tot = ovf = 0;
  __syncthreads();
  uint32_t t = 0, o = 0;
  for (uint32_t s = threadIdx.x; s < ns; s += blockDim.x) {
    const uint32_t sc = p.scnt[p.first_slice[u] + s];
    t += sc;
    o |= sc > cs;
  }
  atomicAdd(&tot, t);
  if (o) atomicOr(&ovf, 1u);
  __syncthreads();
  if (threadIdx.x == 0) p.lstate[8 * lu + 4] = (!ovf && tot >= c.k) ? 1u : 0u;
}

// radix-select histogram pass over the large units' candidates (mode 1: the
// sub-lists, slice by slice) or whole units (mode 0)
template <int KIND>
__global__ void __launch_bounds__(256) sparse_large_hist(const __grid_constant__ SparseParams p, int pass) {
  __shared__ uint32_t h[256];
  const int sh = 24 - 8 * pass;
  for (uint32_t lu = 0; lu < p.n_large; lu++) {
    const uint32_t u = p.large_units[lu];
    const DevChunk c = p.chunks[p.items[u]];
    const float* V = unit_values(p, c);
    const bool cand = p.lstate[8 * lu + 4] != 0;
    const uint32_t prefix = pass ? p.lstate[8 * lu + 0] : 0u, pmask = pass ? p.lstate[8 * lu + 1] : 0u;
    h[threadIdx.x] = 0;
    __syncthreads();
    if (cand) {
      const uint32_t ns = unit_ns(c), cs = (p.cand_off[u + 1] - p.cand_off[u]) / ns;
      for (uint32_t sl = blockIdx.x; sl < ns; sl += gridDim.x) {
        const uint32_t n_sl = p.scnt[p.first_slice[u] + sl];
        for (uint32_t i = threadIdx.x; i < n_sl; i += 256) {
          const uint32_t key = p.cand[p.cand_off[u] + sl * cs + i].y;
          hist_add(h, (key >> sh) & 255u, (key & pmask) == prefix);
        }
      }
    } else {
      for (uint32_t j = blockIdx.x * 256 + threadIdx.x; j < c.len; j += gridDim.x * 256) {
        const uint32_t key = large_key<KIND>(p, c, V, j);
        hist_add(h, (key >> sh) & 255u, (key & pmask) == prefix);
      }
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(p.lhist + 256 * lu + threadIdx.x, h[threadIdx.x]);
    __syncthreads();
  }
}

// one warp per large unit: the bin holding the kk-th largest key; clears the histogram
__global__ void sparse_large_find(const __grid_constant__ SparseParams p, int pass) {
  const uint32_t lu = blockIdx.x;
  const int sh = 24 - 8 * pass;
  uint32_t* st = p.lstate + 8 * lu;
  const uint32_t u = p.large_units[lu];
  const uint32_t kk = pass ? st[2] : p.chunks[p.items[u]].k;
  const uint2 fb = warp_find_bin256(p.lhist + 256 * lu, kk);
  __syncwarp();
  for (uint32_t b = threadIdx.x; b < 256; b += 32) p.lhist[256 * lu + b] = 0;
  if (threadIdx.x == 0) {
    st[0] = (pass ? st[0] : 0u) | (fb.x << sh);
    st[1] = (pass ? st[1] : 0u) | (0xffu << sh);
    st[2] = kk - fb.y;
    st[3] = (pass ? st[3] : 0u) + fb.y;
  }
}

// per slice of a large unit: keys above T and equal to T
template <int KIND>
__global__ void __launch_bounds__(SE_NT) sparse_large_count(const __grid_constant__ SparseParams p) {
  __shared__ uint32_t red[2][SE_NT / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t ls = blockIdx.x; ls < p.n_lslices; ls += gridDim.x) {
    const uint2 us = p.lslices[ls];   // (slice index, large unit)
    const Slice sl = p.slices[us.x];
    const DevChunk c = p.chunks[sl.chunk];
    const float* V = unit_values(p, c);
    const uint32_t T = p.lstate[8 * us.y + 0];
    uint32_t gt = 0, eq = 0;
    for (uint32_t o = threadIdx.x; o < sl.len; o += SE_NT) {
      const uint32_t key = large_key<KIND>(p, c, V, sl.start + o);
      gt += key > T;
      eq += key == T;
    }
    gt = __reduce_add_sync(0xffffffffu, gt);
    eq = __reduce_add_sync(0xffffffffu, eq);
    if (lane == 0) {
      red[0][warp] = gt;
      red[1][warp] = eq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t a = 0, b = 0;
      for (int w = 0; w < SE_NT / 32; w++) {
        a += red[0][w];
        b += red[1][w];
      }
      p.lcnt[ls] = make_uint2(a, b);
    }
    __syncthreads();
  }
}

// one CTA per large unit: each slice's first output position and the T-ties
// before it (ties go to the lowest indices: the first `need` in index order)
__global__ void __launch_bounds__(SE_NT) sparse_large_scan(const __grid_constant__ SparseParams p) {
  __shared__ uint32_t scan[SE_NT / 32 + 1];
  const uint32_t lu = blockIdx.x;
  const uint32_t u = p.large_units[lu];
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t need = c.k - p.lstate[8 * lu + 3];
  uint32_t out_run = 0, eq_run = 0;
  const uint32_t s0 = p.lslice_first[lu], s1 = p.lslice_first[lu + 1];
  for (uint32_t b0 = s0; b0 < s1; b0 += SE_NT) {
    const uint32_t ls = b0 + threadIdx.x;
    const uint2 ce = ls < s1 ? p.lcnt[ls] : make_uint2(0, 0);
    uint32_t teq;
    const uint32_t eb = eq_run + block_excl_scan_u32<SE_NT>(ce.y, scan, &teq);
    const uint32_t take = eb >= need ? 0u : min(ce.y, need - eb);
    uint32_t tsel;
    const uint32_t ob = out_run + block_excl_scan_u32<SE_NT>(ce.x + take, scan, &tsel);
    if (ls < s1) p.loff[ls] = make_uint2(ob, eb);
    out_run += tsel;
    eq_run += teq;
  }
  if (threadIdx.x == 0) *reinterpret_cast<uint64_t*>(p.out + c.pay) = (uint64_t)c.k;
}

// per slice of a large unit: the selected elements in index order -> payload,
// EF fix-ups; 16 consecutive elements per thread
template <int KIND>
__global__ void __launch_bounds__(SE_NT) sparse_large_emit(const __grid_constant__ SparseParams p) {
  __shared__ uint32_t scan[SE_NT / 32 + 1];
  const bool scaled = KIND == SP_RANDK && p.randk_scaled;
  for (uint32_t ls = blockIdx.x; ls < p.n_lslices; ls += gridDim.x) {
    const uint2 us = p.lslices[ls];
    const Slice sl = p.slices[us.x];
    const DevChunk c = p.chunks[sl.chunk];
    float* V = const_cast<float*>(unit_values(p, c));
    const uint32_t T = p.lstate[8 * us.y + 0];
    const uint32_t need = c.k - p.lstate[8 * us.y + 3];
    const uint2 off = p.loff[ls];   // (first output position, T-ties before this slice)
    const float scale = (float)((double)c.len / (double)c.k);
    uint8_t* pay = p.out + c.pay;
    const uint32_t j0 = sl.start + 16 * threadIdx.x;
    uint32_t gtm = 0, eqm = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) {
      if (16 * threadIdx.x + e < sl.len) {
        const uint32_t key = large_key<KIND>(p, c, V, j0 + e);
        gtm |= (uint32_t)(key > T) << e;
        eqm |= (uint32_t)(key == T) << e;
      }
    }
    uint32_t teq;
    uint32_t rr = off.y + block_excl_scan_u32<SE_NT>(__popc(eqm), scan, &teq);
    uint32_t selm = gtm;
#pragma unroll
    for (int e = 0; e < 16; e++)
      if ((eqm >> e) & 1u) {
        if (rr < need) selm |= 1u << e;
        rr++;
      }
    uint32_t tsel;
    uint32_t pos = off.x + block_excl_scan_u32<SE_NT>(__popc(selm), scan, &tsel);
    for (uint32_t m = selm; m; m &= m - 1) {
      const uint32_t j = j0 + (uint32_t)(__ffs(m) - 1);
      const float q = V[j];
      const float val = quant_val(scaled ? fmul(q, scale) : q, p.f16);   // R23
      reinterpret_cast<uint32_t*>(pay + 8)[pos] = j;
      put_val(pay + 8 + 4ull * c.k, pos, val, p.f16);
      if (p.use_ef) V[j] = fsub(q, val);
      pos++;
    }
    __syncthreads();
  }
}

// after the emit: the no-EF server's scratch cleared
__global__ void sparse_large_done(const __grid_constant__ SparseParams p) {
  const uint32_t lu = blockIdx.x;
  const uint32_t u = p.large_units[lu];
  const DevChunk c = p.chunks[p.items[u]];
  if (p.server && !p.use_ef) clear_scratch(p, c, const_cast<float*>(unit_values(p, c)), threadIdx.x, blockDim.x);
}

// ================================================================ launchers
size_t sparse_select_smem(uint32_t sel_cap) { return 2ull * sel_cap * sizeof(uint32_t); }

template <int KIND>
static cudaError_t launch_prep_t(const SparseParams& p, cudaStream_t s) {
  if (!p.n_units) return cudaSuccess;
  if (p.server && p.n_apply_blk) {
    sparse_apply_kernel<KIND><<<p.n_apply_blk, SA_NT, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  sparse_prep_kernel<KIND><<<p.n_units, SG_NT, 0, s>>>(p);
  return cudaGetLastError();
}

template <int KIND>
static cudaError_t launch_select_t(const SparseParams& p, cudaStream_t s) {
  if (!p.n_units) return cudaSuccess;
  const size_t ws = sizeof(UnitSel);
  cudaError_t e = cudaFuncSetAttribute(sparse_select_unit_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws);
  if (e != cudaSuccess) return e;
  sparse_select_unit_kernel<KIND><<<p.n_units, SU_NT, ws, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t smem = sparse_select_smem(p.sel_cap);
  e = cudaFuncSetAttribute(sparse_select_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sparse_select_kernel<KIND><<<p.n_units, SE_NT, smem, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (p.n_large) {   // per-tensor units
    sparse_large_init<<<p.n_large, 256, 0, s>>>(p);
    for (int pass = 0; pass < 4; pass++) {
      sparse_large_hist<KIND><<<p.large_grid, 256, 0, s>>>(p, pass);
      sparse_large_find<<<p.n_large, 32, 0, s>>>(p, pass);
    }
    sparse_large_count<KIND><<<p.large_grid, SE_NT, 0, s>>>(p);
    sparse_large_scan<<<p.n_large, SE_NT, 0, s>>>(p);
    sparse_large_emit<KIND><<<p.large_grid, SE_NT, 0, s>>>(p);
    sparse_large_done<<<p.n_large, 256, 0, s>>>(p);
    e = cudaGetLastError();
  }
  return e;
}

cudaError_t launch_sparse_prep(int kind, const SparseParams& p, cudaStream_t s) {
  switch (kind) {
    case SP_TOPK: return launch_prep_t<SP_TOPK>(p, s);
    case SP_RANDK: return launch_prep_t<SP_RANDK>(p, s);
  }
  return cudaErrorInvalidValue;
}
cudaError_t launch_sparse_select(int kind, const SparseParams& p, cudaStream_t s) {
  switch (kind) {
    case SP_TOPK: return launch_select_t<SP_TOPK>(p, s);
    case SP_RANDK: return launch_select_t<SP_RANDK>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bpc
