// kernels_stream.cu — persistent, warp-specialised, TMA-pipelined streaming
// kernels (sm_100a).  One CTA per SM; the last warp is the PRODUCER: it reads
// the work descriptors, stages them in shared memory and issues 1-D bulk
// copies (cp.async.bulk -> UBLKCP, mbarrier complete_tx) up to ST stages ahead;
// 16 CONSUMER warps wait on full[s], compute, and release empty[s].  Descriptor
// latency never reaches the consumers and the copy engine keeps ~130 KB of
// reads in flight per SM.
//
// update_stream: g~ = dec(p) from the staged payload bytes,
// then Alg. 5 lines 12-16 + x update (R15/R16)
// on the staged m, v, x tile; results stored straight to HBM.
//
// worker_stream (A1-A3 for the norm-based compressors: scaled sign, linear /
// natural dithering, raw units): per 2^13-element slice q = g + e in shared
// memory (Alg. 4 l.5) and the slice's pairwise-tree partial
// (R6); a unit spanning several slices combines its partials through global
// memory (release add on a per-unit counter, acquire spin).  The emit of slice
// i-1 (sign bits / codes + e = q - dec, l.6-7) is deferred behind the produce
// of slice i so the wait overlaps useful work.  All CTAs are co-resident
// (cooperative launch) and every CTA publishes a slice before it waits on an
// earlier one, so the waits cannot deadlock.
#include <type_traits>

#include "device.cuh"

namespace bpc {

enum { S_NONE = 0, S_SIGN = 2, S_TOPK = 3, S_RANDK = 4, S_LDITHER = 5, S_NDITHER = 6 };

constexpr int CW = 16;                 // consumer warps
constexpr int CNT = 32 * CW;           // consumer threads
constexpr int SNT = CNT + 64;          // + 1 producer warp + 1 reducer warp (LANS pass 1)

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumers_sync() {   // named barrier over the consumer warps
  asm volatile("bar.sync 1, %0;" ::"n"(CNT) : "memory");
}

// ============================================================== update_stream
constexpr int UST = 3;                      // stages
// Work items: 4096-element update tiles (LANS: its block sums are per 4096-tile,
// R22), or their 2048-element halves (Adam, NAG): a 2048 item needs half the
// shared memory, so two CTAs share an SM -- 32 consumer warps hide the latency
// of the exact division / root sequences (8 per 4 elements) that 16 could not

struct UDesc {
  uint64_t off;    // flat element offset of the chunk
  uint32_t e0, ne; // sparse kinds: the item's payload entries [e0, e0 + ne)
  uint32_t k;      // sparse kinds: the chunk's k
  const uint8_t* pay;   // the chunk's payload (local P, or the owner's P over NVLink)
  uint32_t start;  // tile start (chunk-relative)
  uint32_t len;
  uint32_t L;
  uint32_t raw;
  uint32_t pofs;   // byte offset of the tile's first payload field inside the staged piece
  uint32_t tile;   // global tile index (LANS partials)
  float ca, cb;    // LANS pass 2: the tile's block coefficients (R22)
};

template <int T>
struct __align__(128) USmem {
  float4 m[UST][T / 4];
  float4 v[UST][T / 4];
  float4 x[UST][T / 4];
  float4 pay[UST][T / 4];         // payload piece: raw fp32 tile, or sign / code bits
  float4 head[UST];               // the payload's first 16 bytes: scale (sign) / norm (dither)
  UDesc desc[UST];
  uint64_t full[UST], empty[UST];
  uint64_t sums[UST];             // LANS pass 1: the consumers' warp subtrees of stage s are in red[s]
  double red[UST][3][T / 16];     // LANS pass 1: 16-element subtrees of x^2, u^2, w^2
};


// LANS (R22): u = r + lambda x, w = c + lambda x with r = m~/(sqrt(v~)+eps),
// c = g~/(sqrt(v~)+eps), from the already-updated m, v (the oracle's order)
__device__ __forceinline__ void lans_uw(float g, float m, float v, float x, const UpdateParams& p, const float4 bc,
                                        float& u, float& w) {
  const float den = fadd(fsqrt0(divc(v, bc.y, bc.w)), p.eps);
  u = fadd(fdiv_pos(divc(m, bc.x, bc.z), den), fmul(p.wd, x));
  w = fadd(fdiv_pos(g, den), fmul(p.wd, x));
}

// FUSED: wait for the owners' p (fused NVLink exchange), then bulk-copy each
// chunk's payload straight from its owner's P (p.psrc[owner], IPC-mapped).
// MODE 0: Adam core (A9).  LANS (NEXT #1, R22) runs two passes:
// MODE 1: m, v updated and stored; per tile the fp64 pairwise subtrees of
//         x^2, u^2, w^2 (a reducer warp writes p.lans_part[3 tile + q]);
// MODE 2: u, w recomputed from the stored m, v; x -= lr (a u + b w) with the
//         tile's block coefficients (p.lans_coef, from lans_coef_kernel).
// MODE 3: NAG (R24): g = g~ + lambda x, m = mu m + g (m holds the velocity),
//         x -= lr (g + mu m); v is neither read nor written (16 B/element).
template <int KIND, bool FUSED, int MODE, int T>
__global__ void __launch_bounds__(SNT, T == UTILE ? 1 : 2) update_stream(const __grid_constant__ UpdateParams p) {
  static_assert(T == UTILE || (T == UTILE / 2 && MODE != 1 && MODE != 2), "LANS works on whole tiles");
  constexpr int UK = T / 4 / CNT;   // float4 per consumer thread per item
  constexpr uint32_t SPLIT = UTILE / T;
  extern __shared__ __align__(128) unsigned char sraw[];
  USmem<T>& sm = *reinterpret_cast<USmem<T>*>(sraw);
  const uint32_t G = gridDim.x;
  const uint32_t n_items = p.n_tiles * SPLIT;
  const uint32_t mine = n_items > blockIdx.x ? (n_items - blockIdx.x + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool SPARSE = KIND == S_TOPK || KIND == S_RANDK;
  const int b = (KIND == S_SIGN || SPARSE) ? 1 : (int)p.bits;
  if (threadIdx.x == 0) {
    for (int s = 0; s < UST; s++) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], MODE == 1 ? CW + 1 : CW);
      mbar_init(&sm.sums[s], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait_and_release();
  const LaunchEp ep = launch_begin(p.sync);
  const float4 bc = bias_of(p.bias, ep.t);   // the step's bias corrections (R16)
  if (warp == CW) {   // ---------------- producer
    if (lane == 0) {
      if (FUSED) peer_wait(p.sync, ep);   // fused exchange: every owner's p has landed in P
      for (uint32_t i = 0; i < mine; i++) {
        const int s = i % UST;
        if (i >= (uint32_t)UST) mbar_wait(&sm.empty[s], ((i / UST) - 1) & 1);
        const uint32_t item = blockIdx.x + i * G;
        Tile tl = p.tiles[item / SPLIT];
        if (SPLIT > 1) {   // half h of the tile (the second half of a short tile may be empty)
          const uint32_t h = item % SPLIT, s0 = h * T;
          tl.len = tl.len > s0 ? min(tl.len - s0, (uint32_t)T) : 0u;
          tl.start += s0;
        }
        const DevChunk c = p.chunks[tl.chunk];
        const uint8_t* pay = (FUSED ? p.psrc[c.owner] : p.pbuf) + c.pay;
        const uint32_t nvb = (tl.len & ~3u) * 4u;
        UDesc d;
        d.off = c.off;
        d.pay = pay;
        d.start = tl.start;
        d.len = tl.len;
        d.L = c.len;
        d.raw = c.raw;
        d.tile = item;
        if (SPARSE) {   // the item's entries (T = UTILE: both halves of the tile)
          const uint2 e = p.ent[SPLIT > 1 ? item : 2 * item];
          d.e0 = e.x;
          d.ne = SPLIT > 1 ? e.y : e.y + p.ent[2 * item + 1].y;
          d.k = c.k;
        }
        if (MODE == 2) {
          const float2 cf = p.lans_coef[tl.pad];   // Tile.pad = block (tensor) index
          d.ca = cf.x;
          d.cb = cf.y;
        }
        const uint8_t* psrc;
        uint32_t pbytes, hbytes = 0;
        if (tl.len == 0) {   // empty half: nothing to load, the phase completes at once
          psrc = pay;
          pbytes = 0;
          d.pofs = 0;
        } else if (c.raw || KIND == S_NONE) {
          psrc = pay + 4ull * tl.start;
          pbytes = nvb;
          d.pofs = 0;
        } else if (SPARSE) {   // the consumers scatter the item's entries (L2-resident P)
          psrc = pay;
          pbytes = 0;
          d.pofs = 0;
        } else {
          const uint64_t s0 = 4 + (uint64_t)tl.start * b / 8;                  // first field byte
          const uint64_t e0 = 4 + ((uint64_t)(tl.start + tl.len) * b + 7) / 8;  // end byte
          const uint64_t a0 = s0 & ~15ull, a1 = (e0 + 15) & ~15ull;           // inside the 16-B slot
          psrc = pay + a0;
          pbytes = (uint32_t)(a1 - a0);
          d.pofs = (uint32_t)(s0 - a0);
          hbytes = 16;
        }
        sm.desc[s] = d;
        mbar_arrive_expect_tx(&sm.full[s], (MODE == 3 ? 2 : 3) * nvb + pbytes + hbytes);
        if (hbytes) tma_load_1d(&sm.head[s], pay, 16, &sm.full[s]);
        if (nvb) {
          tma_load_1d(sm.m[s], p.m + c.off + tl.start, nvb, &sm.full[s]);
          if (MODE != 3) tma_load_1d(sm.v[s], p.v + c.off + tl.start, nvb, &sm.full[s]);
          tma_load_1d(sm.x[s], p.x + c.off + tl.start, nvb, &sm.full[s]);
        }
        if (pbytes) tma_load_1d(sm.pay[s], psrc, pbytes, &sm.full[s]);
      }
    }
    return;
  }
  if (warp == CW + 1) {   // ---------------- reducer (LANS pass 1 only)
    if (MODE == 1) {
      for (uint32_t i = 0; i < mine; i++) {
        const int s = i % UST;
        mbar_wait(&sm.sums[s], (i / UST) & 1);
        const uint32_t tile = sm.desc[s].tile;
#pragma unroll
        for (int q = 0; q < 3; q++) {   // tile total: pairwise tree over its 256 subtrees (R6)
          const double* r8 = &sm.red[s][q][8 * lane];   // lane l: elements [128 l, 128 l + 128)
          const double a = ((r8[0] + r8[1]) + (r8[2] + r8[3])) + ((r8[4] + r8[5]) + (r8[6] + r8[7]));
          const double t = warp_tree(a);
          if (lane == 0) p.lans_part[3ull * tile + q] = t;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
      }
    }
    return;
  }
  // ---------------- consumers
  const float sl = (float)((1u << (p.bits - 1)) - 1u);
  const int cmax = (1 << (p.bits - 1)) - 1;
  for (uint32_t i = 0; i < mine; i++) {
    const int s = i % UST;
    // the tile's bytes: a short sleep between polls keeps the waiting warps off
    // the issue slots of the ones computing (a tile streams in ~2 us)
    mbar_wait_backoff(&sm.full[s], (i / UST) & 1, 64);
    const UDesc d = sm.desc[s];
    const uint32_t nvec = d.len >> 2;
    float* m = p.m + d.off;
    float* v = p.v + d.off;
    float* x = p.x + d.off;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(sm.pay[s]) + d.pofs);
    const float hdr = *reinterpret_cast<const float*>(&sm.head[s]);
    const float unit = fdiv(hdr, sl);
    float* gts = reinterpret_cast<float*>(sm.pay[s]);   // sparse: the item's decoded g~ (T floats)
    if (SPARSE && !d.raw && d.len) {
      // zero the item, scatter its entries (indices ascending, inside [start, start + len)),
      // then every thread reads its own float4s
#pragma unroll
      for (int k = 0; k < UK; k++) sm.pay[s][threadIdx.x + k * CNT] = make_float4(0.f, 0.f, 0.f, 0.f);
      consumers_sync();
      const uint32_t* idx = reinterpret_cast<const uint32_t*>(d.pay + 8);
      const uint8_t* val = d.pay + 8 + 4ull * d.k;   // fp32, or binary16 values (R23)
      for (uint32_t e = threadIdx.x; e < d.ne; e += CNT) {
        const uint32_t q = d.e0 + e;
        gts[idx[q] - d.start] = get_val(val, q, p.f16);
      }
      consumers_sync();
    }
#pragma unroll
    for (int k = 0; k < UK; k++) {
      const uint32_t f = threadIdx.x + k * CNT;   // float4 index inside the tile
      const bool in = 4 * f < d.len;
      if (MODE != 1 && !in) continue;
      const uint32_t j = d.start + 4 * f;
      float4 g4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!in) {
      } else if (d.raw || KIND == S_NONE) {
        g4 = f < nvec ? sm.pay[s][f] : load4_masked(reinterpret_cast<const float*>(d.pay), j, d.L);
      } else if (KIND == S_SIGN) {
        const float h = hdr;
        const uint32_t nib = (words[f >> 3] >> ((f & 7) * 4)) & 15u;
        g4 = make_float4(nib & 1u ? h : -h, nib & 2u ? h : -h, nib & 4u ? h : -h, nib & 8u ? h : -h);
      } else if (SPARSE) {
        g4 = sm.pay[s][f];
      } else {
        const uint32_t field = load_field(words, (uint64_t)b * 4 * f, 4 * b);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const uint32_t code = (field >> (b * u)) & ((1u << b) - 1u);
          float mag;
          if (KIND == S_LDITHER) {
            mag = fmul((float)(code >> 1), unit);
          } else {
            const uint32_t cl = code >> 1;
            mag = fmul(cl == 0 ? 0.f : __uint_as_float((uint32_t)(127 - (cmax - (int)cl)) << 23), hdr);
          }
          set(g4, u, (code & 1u) ? mag : -mag);
        }
      }
      float4 m4 = make_float4(0.f, 0.f, 0.f, 0.f), v4 = m4, x4 = m4;
      if (f < nvec) {
        m4 = sm.m[s][f];
        if (MODE != 3) v4 = sm.v[s][f];
        x4 = sm.x[s][f];
      } else if (in) {   // ragged tail of a unit: not covered by the 16-byte bulk copies
        m4 = load4_masked(m, j, d.L);
        if (MODE != 3) v4 = load4_masked(v, j, d.L);
        x4 = load4_masked(x, j, d.L);
      }
      if (MODE == 0) {
        adam4(g4, m4, v4, x4, p, bc);
        if (f < nvec) {
          st4(m + j, m4);
          st4(v + j, v4);
          st4(x + j, x4);
        } else {
          store4_masked(m, j, d.L, m4);
          store4_masked(v, j, d.L, v4);
          store4_masked(x, j, d.L, x4);
        }
      } else if (MODE == 1) {
        float4 u4, w4;
#pragma unroll
        for (int e = 0; e < 4; e++) {
          float mm = get(m4, e), vv = get(v4, e);
          const float g = get(g4, e);
          mm = fadd(fmul(p.beta1, mm), fmul(p.omb1, g));            // line 12
          vv = fadd(fmul(p.beta2, vv), fmul(p.omb2, fmul(g, g)));   // line 13
          set(m4, e, mm);
          set(v4, e, vv);
          float uu, ww;
          lans_uw(g, mm, vv, get(x4, e), p, bc, uu, ww);
          const bool valid = in && j + e < d.L;   // padding contributes +0 to the block sums
          set(u4, e, valid ? uu : 0.f);
          set(w4, e, valid ? ww : 0.f);
          if (!valid) set(x4, e, 0.f);
        }
        if (in) {
          if (f < nvec) {
            st4(m + j, m4);
            st4(v + j, v4);
          } else {
            store4_masked(m, j, d.L, m4);
            store4_masked(v, j, d.L, v4);
          }
        }
        // two butterfly levels: lanes 4q hold the 16-element subtree 8 (k CW + warp) + q
        // of tile elements [16 i, 16 i + 16); the reducer warp completes the tree
        double tx = leaf4_sq(x4), tu = leaf4_sq(u4), tw = leaf4_sq(w4);
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          tx = tx + __shfl_xor_sync(0xffffffffu, tx, o);
          tu = tu + __shfl_xor_sync(0xffffffffu, tu, o);
          tw = tw + __shfl_xor_sync(0xffffffffu, tw, o);
        }
        if ((lane & 3) == 0) {
          const uint32_t i16 = 8 * (k * CW + warp) + (lane >> 2);
          sm.red[s][0][i16] = tx;
          sm.red[s][1][i16] = tu;
          sm.red[s][2][i16] = tw;
        }
      } else if (MODE == 3) {   // NAG (R24)
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const float xx = get(x4, e);
          const float g = fadd(get(g4, e), fmul(p.wd, xx));
          const float vel = fadd(fmul(p.mu, get(m4, e)), g);
          set(m4, e, vel);
          set(x4, e, fsub(xx, fmul(p.lr, fadd(g, fmul(p.mu, vel)))));
        }
        if (f < nvec) {
          st4(m + j, m4);
          st4(x + j, x4);
        } else {
          store4_masked(m, j, d.L, m4);
          store4_masked(x, j, d.L, x4);
        }
      } else {   // MODE 2
#pragma unroll
        for (int e = 0; e < 4; e++) {
          float uu, ww;
          lans_uw(get(g4, e), get(m4, e), get(v4, e), get(x4, e), p, bc, uu, ww);
          const float dd = fadd(fmul(d.ca, uu), fmul(d.cb, ww));   // line 17
          set(x4, e, fsub(get(x4, e), fmul(p.lr, dd)));           // line 18
        }
        if (f < nvec) st4(x + j, x4);
        else store4_masked(x, j, d.L, x4);
      }
    }
    if (SPARSE) {   // generic-proxy writes of pay[s] before the next bulk copy into it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) {
      if (MODE == 1) mbar_arrive(&sm.sums[s]);    // red[s] written (release)
      mbar_arrive(&sm.empty[s]);                  // this warp is done with stage s
    }
  }
  consumers_sync();   // every consumer's stores issued: the launch may count this CTA done
  launch_end(p.sync, ep, threadIdx.x == 0);
}

size_t update_stream_smem() { return sizeof(USmem<UTILE>); }

cudaError_t launch_update_stream(int kind, const UpdateParams& p, int grid, cudaStream_t st) {
  if (p.n_tiles == 0) return cudaSuccess;
  auto go = [&](auto fn, size_t smem, uint32_t per_sm, uint32_t split) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<uint32_t>((uint32_t)grid * per_sm, p.n_tiles * split));
    cfg.blockDim = dim3(SNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // prologue overlaps the predecessor
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, p);
  };
  const bool f = p.sync.wait_fam >= 0;
  auto pick = [&](auto kind_tag) -> cudaError_t {
    constexpr int K = decltype(kind_tag)::value;
    constexpr int H = UTILE / 2;
    const size_t sh = sizeof(USmem<H>), sf = sizeof(USmem<UTILE>);
    switch (p.mode * 2 + (f ? 1 : 0)) {
      case 0: return go(update_stream<K, false, 0, H>, sh, 2, 2);
      case 1: return go(update_stream<K, true, 0, H>, sh, 2, 2);
      case 2: return go(update_stream<K, false, 1, UTILE>, sf, 1, 1);
      case 3: return go(update_stream<K, true, 1, UTILE>, sf, 1, 1);
      case 4: return go(update_stream<K, false, 2, UTILE>, sf, 1, 1);
      case 5: return go(update_stream<K, true, 2, UTILE>, sf, 1, 1);
      case 6: return go(update_stream<K, false, 3, H>, sh, 2, 2);
      case 7: return go(update_stream<K, true, 3, H>, sh, 2, 2);
    }
    return cudaErrorInvalidValue;
  };
  switch (kind) {
    case S_NONE: return pick(std::integral_constant<int, S_NONE>{});
    case S_SIGN: return pick(std::integral_constant<int, S_SIGN>{});
    case S_LDITHER: return pick(std::integral_constant<int, S_LDITHER>{});
    case S_NDITHER: return pick(std::integral_constant<int, S_NDITHER>{});
    case S_TOPK: return pick(std::integral_constant<int, S_TOPK>{});
    case S_RANDK: return pick(std::integral_constant<int, S_RANDK>{});
  }
  return cudaErrorInvalidValue;
}

// one thread per 2048-element half tile: its entries in the chunk's ascending
// payload indices, [lower_bound(start), lower_bound(start + len))
__global__ void sparse_ranges_kernel(const __grid_constant__ UpdateParams p, uint2* ent) {
  const uint32_t item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= 2 * p.n_tiles) return;
  Tile tl = p.tiles[item >> 1];
  const uint32_t s0 = (item & 1) * (UTILE / 2);
  tl.len = tl.len > s0 ? min(tl.len - s0, (uint32_t)(UTILE / 2)) : 0u;
  tl.start += s0;
  const DevChunk c = p.chunks[tl.chunk];
  if (c.raw || tl.len == 0) {
    ent[item] = make_uint2(0u, 0u);
    return;
  }
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(p.pbuf + c.pay + 8);
  auto lb = [&](uint32_t key) {
    uint32_t lo = 0, n = c.k;
    while (n > 0) {
      const uint32_t h = n >> 1;
      if (__ldg(idx + lo + h) < key) {
        lo += h + 1;
        n -= h + 1;
      } else {
        n = h;
      }
    }
    return lo;
  };
  const uint32_t a = lb(tl.start), e = lb(tl.start + tl.len);
  ent[item] = make_uint2(a, e - a);
}

cudaError_t launch_sparse_ranges(const UpdateParams& p, uint2* ent, cudaStream_t s) {
  const uint32_t n = 2 * p.n_tiles;
  if (!n) return cudaSuccess;
  sparse_ranges_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, ent);
  return cudaGetLastError();
}


}  // namespace bpc
