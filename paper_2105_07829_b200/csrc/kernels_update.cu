// kernels_update.cu — fused decompress + adaptive update:
// g~ = dec(p) decoded on the fly from the all-gathered server payloads, then
// Alg. 5 lines 12-16 and x <- x - eta (r + lambda x)
// (R15), one streaming pass over m, v, x (24 B/element + payload).
#include "device.cuh"

namespace bpc {

enum { U_NONE = 0, U_SIGN = 2, U_TOPK = 3, U_RANDK = 4, U_LDITHER = 5, U_NDITHER = 6 };


// LANS (R22): u = r + lambda x, w = c + lambda x from the updated m, v
__device__ __forceinline__ void lans_uw1(float g, float m, float v, float x, const UpdateParams& p,
                                         const float4 bc, float& u, float& w) {
  const float den = fadd(fsqrt0(divc(v, bc.y, bc.w)), p.eps);
  u = fadd(fdiv_pos(divc(m, bc.x, bc.z), den), fmul(p.wd, x));
  w = fadd(fdiv_pos(g, den), fmul(p.wd, x));
}

// MODE 0: Adam core; LANS (R22) MODE 1: m, v + the tile's pairwise sums of
// x^2, u^2, w^2 -> p.lans_part; MODE 2: x -= lr (a u + b w)   (see update_stream)
template <int KIND, int MODE>
__global__ void __launch_bounds__(UNT, 4) update_kernel(const __grid_constant__ UpdateParams p) {
  constexpr bool SPARSE = KIND == U_TOPK || KIND == U_RANDK;
  __shared__ float gts[SPARSE ? UTILE : 1];
  __shared__ double red[MODE == 1 ? 3 : 1][32];
  const LaunchEp ep = launch_begin(p.sync);
  const float4 bc = bias_of(p.bias, ep.t);   // the step's bias corrections (R16)
  const Tile tl = p.tiles[blockIdx.x];
  const DevChunk c = p.chunks[tl.chunk];
  const uint8_t* pay = p.pbuf + c.pay;
  const uint32_t L = c.len;
  float* m = p.m + c.off;
  float* v = p.v + c.off;
  float* x = p.x + c.off;
  const bool raw = c.raw != 0;
  const int b = (int)p.bits;
  // full tiles (the common case): unconditional 16-byte loads, 3 * UIT in flight per
  // thread, issued before the sparse payload search so its latency overlaps them
  const bool full = tl.len == UTILE;
  float4 m4[UIT], v4[UIT], x4[UIT];
#pragma unroll
  for (int it = 0; it < UIT; it++) {
    const uint32_t i4 = it * UNT + threadIdx.x;
    const uint32_t j = tl.start + 4 * i4;
    m4[it] = v4[it] = x4[it] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (full) {
      m4[it] = ld4(m + j);
      if (MODE != 3) v4[it] = ld4(v + j);
      x4[it] = ld4(x + j);
    } else if (4 * i4 < tl.len) {
      m4[it] = load4_masked(m, j, L);
      if (MODE != 3) v4[it] = load4_masked(v, j, L);
      x4[it] = load4_masked(x, j, L);
    }
  }
  if constexpr (SPARSE) {
    if (!raw) {
      for (uint32_t i = threadIdx.x; i < UTILE; i += UNT) gts[i] = 0.f;
      __syncthreads();
      const uint32_t k = c.k;
      const uint32_t* idx = reinterpret_cast<const uint32_t*>(pay + 8);
      const uint8_t* val = pay + 8 + 4ull * k;   // fp32, or binary16 values (R23)
      const uint32_t lo = warp_lower_bound(idx, k, tl.start);
      for (uint32_t e = lo + threadIdx.x; e < k; e += UNT) {
        const uint32_t j = idx[e];
        if (j >= tl.start + tl.len) break;
        gts[j - tl.start] = get_val(val, e, p.f16);
      }
      __syncthreads();
    }
  }
  const float hdr = raw ? 0.f : *reinterpret_cast<const float*>(pay);
  const float sl = (float)((1u << (b - 1)) - 1u);
  const int cmax = (1 << (b - 1)) - 1;
  const float unit = fdiv(hdr, sl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2 cf = make_float2(0.f, 0.f);
  if (MODE == 2) cf = p.lans_coef[tl.pad];   // Tile.pad = block (tensor) index
#pragma unroll
  for (int it = 0; it < UIT; it++) {
    const uint32_t i4 = it * UNT + threadIdx.x;
    const uint32_t j = tl.start + 4 * i4;
    const bool in = full || 4 * i4 < tl.len;
    if (MODE != 1 && !in) continue;
    float4 g4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!in) {
    } else if (raw || KIND == U_NONE) {
      g4 = full ? ld4(reinterpret_cast<const float*>(pay) + j) : load4_masked(reinterpret_cast<const float*>(pay), j, L);
    } else if (KIND == U_SIGN) {
      const uint32_t nib = (reinterpret_cast<const uint32_t*>(pay + 4)[j >> 5] >> (j & 31)) & 15u;
      g4 = make_float4(nib & 1u ? hdr : -hdr, nib & 2u ? hdr : -hdr, nib & 4u ? hdr : -hdr,
                       nib & 8u ? hdr : -hdr);
    } else if (SPARSE) {
      g4 = *reinterpret_cast<const float4*>(&gts[4 * i4]);
    } else {
      const uint32_t field = load_field(reinterpret_cast<const uint32_t*>(pay + 4), (uint64_t)b * j, 4 * b);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t code = (field >> (b * u)) & ((1u << b) - 1u);
        float mag;
        if (KIND == U_LDITHER) {
          mag = fmul((float)(code >> 1), unit);
        } else {
          const uint32_t cl = code >> 1;
          mag = fmul(cl == 0 ? 0.f : __uint_as_float((uint32_t)(127 - (cmax - (int)cl)) << 23), hdr);
        }
        set(g4, u, (code & 1u) ? mag : -mag);
      }
    }
    if (MODE == 0) {
      adam4(g4, m4[it], v4[it], x4[it], p, bc);
      if (full) {
        st4(m + j, m4[it]);
        st4(v + j, v4[it]);
        st4(x + j, x4[it]);
      } else {
        store4_masked(m, j, L, m4[it]);
        store4_masked(v, j, L, v4[it]);
        store4_masked(x, j, L, x4[it]);
      }
    } else if (MODE == 1) {
      float4 u4, w4, xv = x4[it];
#pragma unroll
      for (int e = 0; e < 4; e++) {
        float mm = get(m4[it], e), vv = get(v4[it], e);
        const float g = get(g4, e);
        mm = fadd(fmul(p.beta1, mm), fmul(p.omb1, g));            // line 12
        vv = fadd(fmul(p.beta2, vv), fmul(p.omb2, fmul(g, g)));   // line 13
        set(m4[it], e, mm);
        set(v4[it], e, vv);
        float uu, ww;
        lans_uw1(g, mm, vv, get(xv, e), p, bc, uu, ww);
        const bool valid = in && j + e < L;   // padding contributes +0 to the block sums
        set(u4, e, valid ? uu : 0.f);
        set(w4, e, valid ? ww : 0.f);
        if (!valid) set(xv, e, 0.f);
      }
      if (in) {
        if (full) {
          st4(m + j, m4[it]);
          st4(v + j, v4[it]);
        } else {
          store4_masked(m, j, L, m4[it]);
          store4_masked(v, j, L, v4[it]);
        }
      }
      // subtree it * 8 + warp covers tile elements [128 (it * 8 + warp), + 128)
      const double tx = warp_tree(leaf4_sq(xv));
      const double tu = warp_tree(leaf4_sq(u4));
      const double tw = warp_tree(leaf4_sq(w4));
      if (lane == 0) {
        red[0][it * 8 + warp] = tx;
        red[MODE == 1 ? 1 : 0][it * 8 + warp] = tu;
        red[MODE == 1 ? 2 : 0][it * 8 + warp] = tw;
      }
    } else if (MODE == 3) {   // NAG (R24): velocity in m
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const float xx = get(x4[it], e);
        const float g = fadd(get(g4, e), fmul(p.wd, xx));
        const float vel = fadd(fmul(p.mu, get(m4[it], e)), g);
        set(m4[it], e, vel);
        set(x4[it], e, fsub(xx, fmul(p.lr, fadd(g, fmul(p.mu, vel)))));
      }
      if (full) {
        st4(m + j, m4[it]);
        st4(x + j, x4[it]);
      } else {
        store4_masked(m, j, L, m4[it]);
        store4_masked(x, j, L, x4[it]);
      }
    } else {   // MODE 2
#pragma unroll
      for (int e = 0; e < 4; e++) {
        float uu, ww;
        lans_uw1(get(g4, e), get(m4[it], e), get(v4[it], e), get(x4[it], e), p, bc, uu, ww);
        const float dd = fadd(fmul(cf.x, uu), fmul(cf.y, ww));   // line 17
        set(x4[it], e, fsub(get(x4[it], e), fmul(p.lr, dd)));    // line 18
      }
      if (full) st4(x + j, x4[it]);
      else store4_masked(x, j, L, x4[it]);
    }
  }
  if (MODE == 1) {   // tile totals: pairwise tree over the 32 subtrees (R6)
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < 3; q++) {
        const double t = warp_tree(red[MODE == 1 ? q : 0][lane]);
        if (lane == 0) p.lans_part[3ull * blockIdx.x + q] = t;
      }
    }
  }
  __syncthreads();   // the CTA's stores issued: count it done
  launch_end(p.sync, ep, threadIdx.x == 0);
}

// LANS block coefficients (R22): CTA b sums its tiles' partials in pairwise
// order over the tile count padded to a power of two (= the pairwise tree over
// the block padded to a power of two: tiles are 4096-aligned inside a block),
// then phi = clamp(fl32(||x_b||)), a = fl32(phi beta1 / ||u_b||),
// b = fl32(phi (1 - beta1) / ||w_b||), a zero norm -> 0.
__global__ void __launch_bounds__(1024) lans_coef_kernel(const __grid_constant__ LansCoefParams p) {
  extern __shared__ double acc[];   // [3][LANS_MAX_TILES]: x^2, u^2, w^2 reduced together
  const uint32_t b = blockIdx.x;
  const uint32_t first = p.blk_tile[b], T = p.blk_tile[b + 1] - first;
  uint32_t P = 1;
  while (P < T) P <<= 1;
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x)
#pragma unroll
    for (int q = 0; q < 3; q++) acc[q * LANS_MAX_TILES + i] = i < T ? p.part[3ull * (first + i) + q] : 0.0;
  __syncthreads();
  for (uint32_t st = 1; st < P; st <<= 1) {
    for (uint32_t i = threadIdx.x * 2 * st; i < P; i += blockDim.x * 2 * st)
#pragma unroll
      for (int q = 0; q < 3; q++) acc[q * LANS_MAX_TILES + i] = acc[q * LANS_MAX_TILES + i] + acc[q * LANS_MAX_TILES + i + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double nx = sqrt(acc[0]), nu = sqrt(acc[LANS_MAX_TILES]), nw = sqrt(acc[2 * LANS_MAX_TILES]);
    float phi = (float)nx;
    phi = fminf(fmaxf(phi, p.alpha_l), p.alpha_u);
    const float a = nu > 0.0 ? (float)((double)phi * (double)p.beta1 / nu) : 0.f;
    const float bb = nw > 0.0 ? (float)((double)phi * (1.0 - (double)p.beta1) / nw) : 0.f;
    p.coef[b] = make_float2(a, bb);
  }
}

cudaError_t launch_lans_coef(const LansCoefParams& p, cudaStream_t s) {
  if (p.nblk == 0) return cudaSuccess;
  const size_t smem = 3 * sizeof(double) * LANS_MAX_TILES;
  cudaError_t e = cudaFuncSetAttribute(lans_coef_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  lans_coef_kernel<<<p.nblk, 1024, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_update(int kind, const UpdateParams& p, cudaStream_t s) {
  if (p.n_tiles == 0) return cudaSuccess;
  const dim3 grid(p.n_tiles), block(UNT);
#define BPC_UPD(K)                                                       \
  case K:                                                                \
    if (p.mode == 0) update_kernel<K, 0><<<grid, block, 0, s>>>(p);      \
    else if (p.mode == 1) update_kernel<K, 1><<<grid, block, 0, s>>>(p); \
    else if (p.mode == 2) update_kernel<K, 2><<<grid, block, 0, s>>>(p); \
    else update_kernel<K, 3><<<grid, block, 0, s>>>(p);                  \
    break;
  switch (kind) {
    BPC_UPD(U_NONE)
    BPC_UPD(U_SIGN)
    BPC_UPD(U_TOPK)
    BPC_UPD(U_RANDK)
    BPC_UPD(U_LDITHER)
    BPC_UPD(U_NDITHER)
    default: return cudaErrorInvalidValue;
  }
#undef BPC_UPD
  return cudaGetLastError();
}

}  // namespace bpc
