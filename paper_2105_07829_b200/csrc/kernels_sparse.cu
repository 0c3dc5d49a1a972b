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
//   sparse_dense   persistent CTAs over 2^13-element slices, HBM streaming.
//                  Worker: q = g + e (Alg. 4 l.5), e := q (use_ef),
//                  raw units copied.  Server: reads Delta (e~ + the applied
//                  entries; 4 B/element), raw units averaged.  Every element
//                  with key >= G_u joins the unit's candidate list (gathered per
//                  slice in shared memory, one global append per slice).
//   sparse_select  if the unit has k <= c <= cap candidates, every element
//                  outside them has key < G <= T (the k-th largest key), so the
//                  exact selection (keys desc, index asc, R9/R10) is a radix
//                  select over the c candidates: one WARP per unit (c <= 4096,
//                  k <= 512), else one CTA per unit (c <= SEL_CAP), else an exact
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
constexpr int SS_NT = 512;        // dense kernel threads (16 elements per thread per slice)
constexpr int SS_CAND = 1024;     // candidates a dense CTA gathers per slice before one global append
constexpr int SE_NT = 512;        // CTA select kernel threads
constexpr int SW_WARPS = 4;       // warp select: units (warps) per CTA
constexpr uint32_t SW_CAP = 4096; // warp select: max candidates
constexpr uint32_t SW_KMAX = 512; // warp select: max k
constexpr int PREP_IDX = 4096;    // server prep: rank index entries staged in shared memory

__device__ __forceinline__ uint32_t topk_key(float v) { return __float_as_uint(v) & 0x7fffffffu; }
template <int KIND>
__device__ __forceinline__ uint32_t sel_key(float v, uint32_t j, const SparseParams& p, uint32_t id) {
  if (KIND == SP_TOPK) return topk_key(v);
  // random-k: the k smallest Philox words = the k largest complements (R10)
  const uint4 w = rng4(p.seed, j >> 2, id, p.t, p.stage, p.rrank);
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

// ascending bitonic sort of a[0, n) in shared memory, n a power of two, by
// `nt` threads (tid in [0, nt)); `sync` orders the stages
template <class Sync>
__device__ __forceinline__ void bitonic_sort(uint32_t* a, uint32_t n, uint32_t tid, uint32_t nt, Sync sync) {
  for (uint32_t size = 2; size <= n; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < n / 2; i += nt) {
        const uint32_t lo = 2 * i - (i & (stride - 1));
        const uint32_t hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint32_t x = a[lo], y = a[hi];
        if ((x > y) == up) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      sync();
    }
  }
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
template <int KIND>
__global__ void __launch_bounds__(SG_NT) sparse_prep_kernel(const __grid_constant__ SparseParams p) {
  __shared__ uint32_t sidx[PREP_IDX];   // server: the ranks' index lists, when they fit
  __shared__ uint32_t red[SG_NT / 32];
  __shared__ uint32_t scnt;
  const uint32_t u = blockIdx.x;
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t L = c.len, k = c.k;
  float* V = const_cast<float*>(unit_values(p, c));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool topk_noef_server = KIND == SP_TOPK && p.server && !p.use_ef;
  // ---- server: Delta_j at the ranks' entries (rank order, fp64, R5)
  if (p.server) {
    const uint32_t n = p.n;
    const bool staged = (uint64_t)n * k <= (uint64_t)PREP_IDX;
    if (staged) {
      for (uint32_t i = threadIdx.x; i < n * k; i += SG_NT) {
        const uint32_t r = i / k, e = i - r * k;
        sidx[i] = reinterpret_cast<const uint32_t*>(rank_payload(p, c, r) + 8)[e];
      }
    }
    if (threadIdx.x == 0) scnt = 0;
    __syncthreads();
    auto idx_of = [&](uint32_t r) -> const uint32_t* {
      return staged ? sidx + r * k : reinterpret_cast<const uint32_t*>(rank_payload(p, c, r) + 8);
    };
    uint32_t* cand = p.cand + p.cand_off[u];
    const uint32_t cap = p.cand_off[u + 1] - p.cand_off[u];
    for (uint32_t i = threadIdx.x; i < n * k; i += SG_NT) {
      const uint32_t r = i / k, e = i - r * k;
      const uint32_t j = idx_of(r)[e];
      // the first rank holding j sums every holder in rank order
      bool first = true;
      uint32_t pos;
      for (uint32_t r2 = 0; r2 < r && first; r2++) first = !holds(idx_of(r2), k, j, &pos);
      if (!first) continue;
      double acc = 0.0;
      acc += (double)get_val(rank_payload(p, c, r) + 8 + 4ull * k, e, p.f16);
      for (uint32_t r2 = r + 1; r2 < n; r2++)
        if (holds(idx_of(r2), k, j, &pos)) acc += (double)get_val(rank_payload(p, c, r2) + 8 + 4ull * k, pos, p.f16);
      const float d = mean_plus(acc, p.inv_n, (double)V[j]);   // no EF: V is the zeroed scratch
      V[j] = d;
      if (topk_noef_server && d != 0.f) {   // no dense pass: the candidates are the nonzero Delta
        const uint32_t s = atomicAdd(&scnt, 1u);
        if (s < cap) cand[s] = j;
      }
    }
    __syncthreads();
    if (topk_noef_server) {
      if (threadIdx.x == 0) {
        p.cnt[u] = scnt;
        p.guess[u] = 1u;
      }
      return;
    }
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
    // the m-th largest sample key, bit by bit from the top (22 bits: G is the
    // lower edge of a 2^-13-wide magnitude bin holding it, G <= that key)
    const uint32_t m = L <= (uint32_t)SG_S ? k : (uint32_t)min(S, sparse_sample_rank(k, L));
    uint32_t g = 0;
    for (int bit = 30; bit >= 10; bit--) {
      const uint32_t t = g | (1u << bit);
      uint32_t cnt = 0;
#pragma unroll
      for (int r = 0; r < 16; r++) cnt += key[r] >= t;
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0) red[warp] = cnt;
      __syncthreads();
      uint32_t tot = 0;
#pragma unroll
      for (int w = 0; w < SG_NT / 32; w++) tot += red[w];
      __syncthreads();
      if (tot >= m) g = t;
    }
    // key 0 (magnitude +-0) is never a useful threshold: with fewer than k nonzero
    // values the select kernel takes its exact whole-unit path
    G = g > 1u ? g : 1u;
  }
  if (threadIdx.x == 0) p.guess[u] = G;
}

// ================================================================ dense
template <int KIND, bool SERVER>
__global__ void __launch_bounds__(SS_NT, 2) sparse_dense_kernel(const __grid_constant__ SparseParams p) {
  __shared__ uint32_t scand[SS_CAND];   // the slice's candidates (unit indices)
  __shared__ uint32_t scnt, sbase;
  bool bad = false;
  for (uint32_t si = blockIdx.x; si < p.n_slices; si += gridDim.x) {
    const Slice sl = p.slices[si];
    const DevChunk c = p.chunks[sl.chunk];
    const uint32_t L = c.len, s0 = sl.start, len = sl.len;
    if (sl.nslices == 0) {   // ---- raw unit: worker payload = g (no EF, R3); server: the ranks' mean
      float* out = reinterpret_cast<float*>(p.out + c.pay);
      for (uint32_t i = threadIdx.x; 4 * i < len; i += SS_NT) {
        const uint32_t j = s0 + 4 * i;
        float4 v;
        if (!SERVER) {
          v = load4_masked(p.grad + c.off, j, L);
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
      continue;
    }
    if (SERVER && KIND == SP_TOPK && !p.use_ef) continue;   // candidates listed by the prep kernel
    const uint32_t u = p.chunk2u[sl.chunk];
    const uint32_t G = p.guess[u];
    float* V = const_cast<float*>(unit_values(p, c));
    float4 q[4];
    if (!SERVER) {
      float4 g4[4], e4[4];
#pragma unroll
      for (int it = 0; it < 4; it++) {   // all loads in flight first
        const uint32_t j = s0 + 4 * (threadIdx.x + it * SS_NT);
        const bool in = 4 * (threadIdx.x + it * SS_NT) < len;
        g4[it] = e4[it] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (in) {
          g4[it] = j + 4 <= L ? ldg4_stream(p.grad + c.off + j) : load4_masked(p.grad + c.off, j, L);
          if (p.use_ef) e4[it] = j + 4 <= L ? ldg4_stream(p.vals + c.off + j) : load4_masked(p.vals + c.off, j, L);
        }
      }
#pragma unroll
      for (int it = 0; it < 4; it++) {
        const uint32_t j = s0 + 4 * (threadIdx.x + it * SS_NT);
        if (p.check_finite)
          bad |= !(isfinite(g4[it].x) && isfinite(g4[it].y) && isfinite(g4[it].z) && isfinite(g4[it].w));
        q[it] = p.use_ef ? make_float4(fadd(g4[it].x, e4[it].x), fadd(g4[it].y, e4[it].y), fadd(g4[it].z, e4[it].z),
                                       fadd(g4[it].w, e4[it].w))
                         : g4[it];
        if (p.use_ef && 4 * (threadIdx.x + it * SS_NT) < len) {   // e := q (the selected get e = q - val later)
          if (j + 4 <= L) st4(V + j, q[it]);
          else store4_masked(V, j, L, q[it]);
        }
      }
    } else if (KIND == SP_TOPK || p.use_ef) {
      // Delta = e~ with the entries applied.  e~ is never -0 (every write is +0 +
      // x, x - x, or a mean that starts at +0), except after bpc_load_state of a
      // -0: Delta = fl32(0 + e~) is then +0, fixed here (read-only otherwise)
#pragma unroll
      for (int it = 0; it < 4; it++) {
        const uint32_t f = threadIdx.x + it * SS_NT;
        const uint32_t j = s0 + 4 * f;
        q[it] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (4 * f < len) q[it] = j + 4 <= L ? ldg4_stream(V + j) : load4_masked(V, j, L);
      }
#pragma unroll
      for (int it = 0; it < 4; it++) {
        const uint32_t j = s0 + 4 * (threadIdx.x + it * SS_NT);
#pragma unroll
        for (int e = 0; e < 4; e++)
          if (__float_as_uint(get(q[it], e)) == 0x80000000u && j + e < L) {
            set(q[it], e, 0.f);
            V[j + e] = 0.f;
          }
      }
    } else {
#pragma unroll
      for (int it = 0; it < 4; it++) q[it] = make_float4(0.f, 0.f, 0.f, 0.f);   // random-k, no EF: keys only
    }
    // ---- candidates: key >= G, gathered per slice in shared memory, then one
    // global append per slice (a unit's slices run on many CTAs at once)
    if (threadIdx.x == 0) scnt = 0;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < 4; it++) {
      const uint32_t f = threadIdx.x + it * SS_NT;
      const uint32_t j = s0 + 4 * f;
      uint32_t m = 0;
      if (4 * f < len) {
#pragma unroll
        for (int e = 0; e < 4; e++)
          if (j + e < L && sel_key<KIND>(get(q[it], e), j + e, p, c.id) >= G) m |= 1u << e;
      }
      if (__ballot_sync(0xffffffffu, m != 0u)) {
#pragma unroll
        for (int e = 0; e < 4; e++)
          if ((m >> e) & 1u) {
            const uint32_t pos = atomicAdd(&scnt, 1u);
            if (pos < (uint32_t)SS_CAND) scand[pos] = j + e;
          }
      }
    }
    __syncthreads();
    const uint32_t ns = scnt;
    if (ns) {
      const uint32_t cap = p.cand_off[u + 1] - p.cand_off[u];
      if (threadIdx.x == 0)   // more than SS_CAND: the list is incomplete, push the count past cap
        sbase = atomicAdd(p.cnt + u, ns > (uint32_t)SS_CAND ? ns + cap + 1 : ns);
      __syncthreads();
      uint32_t* cand = p.cand + p.cand_off[u];
      for (uint32_t i = threadIdx.x; i < ns && i < (uint32_t)SS_CAND; i += SS_NT)
        if (sbase + i < cap) cand[sbase + i] = scand[i];
    }
    __syncthreads();   // scnt / scand / sbase reused by the next slice
  }
  if (bad) atomicOr(p.flag, 1u);
}

// ================================================================ select
__device__ __forceinline__ void emit_one(const SparseParams& p, float* V, uint8_t* pay, uint32_t k, uint32_t pos,
                                         uint32_t j, bool scaled, float scale) {
  const float q = V[j];
  const float val = quant_val(scaled ? fmul(q, scale) : q, p.f16);   // R23
  reinterpret_cast<uint32_t*>(pay + 8)[pos] = j;
  put_val(pay + 8 + 4ull * k, pos, val, p.f16);
  if (p.use_ef) V[j] = fsub(q, val);   // e = q - dec (operator fusion: O(k))
}

// server without EF: the scratch goes back to all-zero (only the ranks' entries
// were written by the prep kernel), by `nt` threads from `tid`
__device__ __forceinline__ void clear_scratch(const SparseParams& p, const DevChunk& c, float* V, uint32_t tid,
                                              uint32_t nt) {
  for (uint32_t i = tid; i < p.n * c.k; i += nt) {
    const uint32_t r = i / c.k, e = i - r * c.k;
    V[reinterpret_cast<const uint32_t*>(rank_payload(p, c, r) + 8)[e]] = 0.f;
  }
}

// ---- one warp per unit: the candidate path for c <= SW_CAP, k <= SW_KMAX
struct WarpSel {
  uint32_t idx[SW_CAP];   // candidate indices; bit 31 = selected, bit 30 = T-tie
  uint32_t key[SW_CAP];   // keys, then the T-tie / selection lists
  uint32_t hist[256];
};

template <int KIND>
__global__ void __launch_bounds__(32 * SW_WARPS) sparse_select_warp_kernel(const __grid_constant__ SparseParams p) {
  extern __shared__ __align__(16) unsigned char swraw[];
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * SW_WARPS + w;
  if (u >= p.n_units) return;
  WarpSel& s = reinterpret_cast<WarpSel*>(swraw)[w];
  const DevChunk c = p.chunks[p.items[u]];
  const uint32_t L = c.len, k = c.k;
  const uint32_t cap = p.cand_off[u + 1] - p.cand_off[u];
  const uint32_t cnt = p.cnt[u];
  if (!(cnt >= k && cnt <= cap && cnt <= SW_CAP && k <= SW_KMAX)) {
    if (lane == 0) p.big[u] = 1;   // the CTA select kernel takes this unit
    return;
  }
  float* V = const_cast<float*>(unit_values(p, c));
  uint8_t* pay = p.out + c.pay;
  const uint32_t* cand = p.cand + p.cand_off[u];
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint32_t j = cand[i];
    s.idx[i] = j;
    s.key[i] = sel_key<KIND>(KIND == SP_TOPK ? V[j] : 0.f, j, p, c.id);
  }
  __syncwarp();
  // k-th largest key: 4 x 8-bit radix select
  uint32_t prefix = 0, pmask = 0, kk = k, above = 0;
  for (int pass = 0; pass < 4; pass++) {
    const int sh = 24 - 8 * pass;
#pragma unroll
    for (int i = 0; i < 8; i++) s.hist[lane + 32 * i] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint32_t key = s.key[i];
      hist_add(s.hist, (key >> sh) & 255u, (key & pmask) == prefix);
    }
    __syncwarp();
    const uint2 fb = warp_find_bin256(s.hist, kk);
    __syncwarp();
    prefix |= fb.x << sh;
    pmask |= 0xffu << sh;
    kk -= fb.y;
    above += fb.y;
  }
  const uint32_t T = prefix, need = k - above;   // T-ties to take, lowest indices first
  uint32_t neq = 0;
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint32_t key = s.key[i];
    if (key > T) s.idx[i] |= 0x80000000u;
    else if (key == T) {
      s.idx[i] |= 0x40000000u;
      neq++;
    }
  }
  neq = __reduce_add_sync(0xffffffffu, neq);
  __syncwarp();
  uint32_t cut = 0xffffffffu;
  if (need < neq) {   // the need-th smallest index among the T-ties (sorted in key[])
    uint32_t base = 0;
    for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool t = i < cnt && (s.idx[i] & 0x40000000u);
      const uint32_t b = __ballot_sync(0xffffffffu, t);
      if (t) s.key[base + __popc(b & ((1u << lane) - 1))] = s.idx[i] & 0x3fffffffu;
      base += __popc(b);
    }
    uint32_t P = 1;
    while (P < neq) P <<= 1;
    for (uint32_t i = neq + lane; i < P; i += 32) s.key[i] = 0xffffffffu;
    __syncwarp();
    bitonic_sort(s.key, P, lane, 32, [] { __syncwarp(); });
    cut = s.key[need - 1];
    __syncwarp();
  }
  // the k selected indices into key[], then sorted ascending
  uint32_t base = 0;
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t x = i < cnt ? s.idx[i] : 0u;
    const bool sel = i < cnt && ((x & 0x80000000u) || ((x & 0x40000000u) && (x & 0x3fffffffu) <= cut));
    const uint32_t b = __ballot_sync(0xffffffffu, sel);
    if (sel) s.key[base + __popc(b & ((1u << lane) - 1))] = x & 0x3fffffffu;
    base += __popc(b);
  }
  uint32_t P = 1;
  while (P < k) P <<= 1;
  for (uint32_t i = k + lane; i < P; i += 32) s.key[i] = 0xffffffffu;
  __syncwarp();
  bitonic_sort(s.key, P, lane, 32, [] { __syncwarp(); });
  const bool scaled = KIND == SP_RANDK && p.randk_scaled;
  const float scale = (float)((double)L / (double)k);
  for (uint32_t i = lane; i < k; i += 32) emit_one(p, V, pay, k, i, s.key[i], scaled, scale);
  __syncwarp();
  if (p.server && !p.use_ef) clear_scratch(p, c, V, lane, 32);
  if (lane == 0) {
    *reinterpret_cast<uint64_t*>(pay) = (uint64_t)k;
    p.cnt[u] = 0;   // the next step's dense pass appends from 0
  }
}

// ---- one CTA per unit: larger candidate lists, or the exact whole-unit path
struct SelSmem {
  uint32_t hist[256];
  uint32_t info[4];
  uint32_t scan[SE_NT / 32 + 1];
};

__device__ __forceinline__ uint32_t block_compact(const uint32_t* a, uint32_t n, uint32_t mask, uint32_t* out,
                                                  uint32_t* counter) {
  if (threadIdx.x == 0) *counter = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += SE_NT)
    if (a[i] & mask) out[atomicAdd(counter, 1u)] = a[i] & 0x3fffffffu;
  __syncthreads();
  const uint32_t m = *counter;
  __syncthreads();
  return m;
}

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

template <int KIND>
__global__ void __launch_bounds__(SE_NT) sparse_select_kernel(const __grid_constant__ SparseParams p) {
  // dynamic: [sel_cap] candidate indices | [sel_cap] keys / lists
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
  const uint32_t cap = p.cand_off[u + 1] - p.cand_off[u];
  const uint32_t cnt = p.cnt[u];
  const uint32_t* cand = p.cand + p.cand_off[u];
  const uint32_t SC = p.sel_cap;
  if (cnt >= k && cnt <= cap && cnt <= SC) {
    // ---- exact selection among the candidates (every other key < G <= T)
    uint32_t* ci = sx;        // indices; bit 31 = selected, bit 30 = T-tie
    uint32_t* ck = sx + SC;   // keys, then the T-tie / selection lists
    for (uint32_t i = threadIdx.x; i < cnt; i += SE_NT) {
      const uint32_t j = cand[i];
      ci[i] = j;
      ck[i] = sel_key<KIND>(KIND == SP_TOPK ? V[j] : 0.f, j, p, c.id);
    }
    __syncthreads();
    uint32_t above;
    const uint32_t T = block_kth_largest([&](uint32_t i) { return ck[i]; }, cnt, k, sm, &above);
    const uint32_t need = k - above;
    for (uint32_t i = threadIdx.x; i < cnt; i += SE_NT) {
      const uint32_t key = ck[i];
      if (key > T) ci[i] |= 0x80000000u;
      else if (key == T) ci[i] |= 0x40000000u;
    }
    __syncthreads();
    const uint32_t neq = block_compact(ci, cnt, 0x40000000u, ck, &sm.info[2]);
    uint32_t cut = 0xffffffffu;
    if (need < neq) {
      uint32_t P = 1;
      while (P < neq) P <<= 1;
      for (uint32_t i = neq + threadIdx.x; i < P; i += SE_NT) ck[i] = 0xffffffffu;
      __syncthreads();
      bitonic_sort(ck, P, threadIdx.x, SE_NT, [] { __syncthreads(); });
      cut = ck[need - 1];
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += SE_NT) {
      const uint32_t x = ci[i];
      if ((x & 0x40000000u) && (x & 0x3fffffffu) <= cut) ci[i] = x | 0x80000000u;
    }
    __syncthreads();
    const uint32_t ns = block_compact(ci, cnt, 0x80000000u, ck, &sm.info[2]);   // == k
    uint32_t P = 1;
    while (P < ns) P <<= 1;
    for (uint32_t i = ns + threadIdx.x; i < P; i += SE_NT) ck[i] = 0xffffffffu;
    __syncthreads();
    bitonic_sort(ck, P, threadIdx.x, SE_NT, [] { __syncthreads(); });
    for (uint32_t i = threadIdx.x; i < k; i += SE_NT) emit_one(p, V, pay, k, i, ck[i], scaled, scale);
  } else {
    // ---- exact over the whole unit: radix select of T over all L keys, then an
    // ordered compaction (index ascending) with the tie cut
    uint32_t above;
    const uint32_t T = block_kth_largest(
        [&](uint32_t j) { return sel_key<KIND>(KIND == SP_TOPK ? V[j] : 0.f, j, p, c.id); }, L, k, sm, &above);
    const uint32_t need = k - above;   // take the `need` lowest-index T-ties
    uint32_t eq_run = 0, out_run = 0;
    for (uint32_t base = 0; base < L; base += 4 * SE_NT) {   // 4 consecutive elements per thread
      const uint32_t j0 = base + 4 * threadIdx.x;
      uint32_t gtm = 0, eqm = 0;
#pragma unroll
      for (int e = 0; e < 4; e++) {
        if (j0 + e < L) {
          const uint32_t key = sel_key<KIND>(KIND == SP_TOPK ? V[j0 + e] : 0.f, j0 + e, p, c.id);
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
        if ((selm >> e) & 1u) emit_one(p, V, pay, k, pos++, j0 + e, scaled, scale);
      eq_run += teq;
      out_run += tsel;
    }
  }
  __syncthreads();
  if (p.server && !p.use_ef) clear_scratch(p, c, V, threadIdx.x, SE_NT);
  if (threadIdx.x == 0) {
    *reinterpret_cast<uint64_t*>(pay) = (uint64_t)k;
    p.cnt[u] = 0;   // the next step's dense pass appends from 0
    p.big[u] = 0;
  }
}

// ================================================================ launchers
size_t sparse_select_smem(uint32_t sel_cap) { return 2ull * sel_cap * sizeof(uint32_t); }

template <int KIND>
static cudaError_t launch_sparse_t(const SparseParams& p, int grid, cudaStream_t s) {
  cudaError_t e;
  if (p.n_units) {
    sparse_prep_kernel<KIND><<<p.n_units, SG_NT, 0, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (p.n_slices) {
    const unsigned g = (unsigned)std::min<uint32_t>((uint32_t)grid, p.n_slices);
    if (p.server) sparse_dense_kernel<KIND, true><<<g, SS_NT, 0, s>>>(p);
    else sparse_dense_kernel<KIND, false><<<g, SS_NT, 0, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (p.n_units) {
    const size_t ws = sizeof(WarpSel) * SW_WARPS;
    e = cudaFuncSetAttribute(sparse_select_warp_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws);
    if (e != cudaSuccess) return e;
    sparse_select_warp_kernel<KIND><<<(p.n_units + SW_WARPS - 1) / SW_WARPS, 32 * SW_WARPS, ws, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t smem = sparse_select_smem(p.sel_cap);
    e = cudaFuncSetAttribute(sparse_select_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sparse_select_kernel<KIND><<<p.n_units, SE_NT, smem, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_sparse(int kind, const SparseParams& p, int grid, cudaStream_t s) {
  switch (kind) {
    case SP_TOPK: return launch_sparse_t<SP_TOPK>(p, grid, s);
    case SP_RANDK: return launch_sparse_t<SP_RANDK>(p, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bpc
