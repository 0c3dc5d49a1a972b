// kernels_update.cu — fused decompress + adaptive update:
// g~ = dec(p) decoded on the fly from the all-gathered server payloads, then
// Alg. 5 lines 12-16 and x <- x - eta (r + lambda x)
// (R15), one streaming pass over m, v, x (24 B/element + payload).
#include "device.cuh"

namespace bpc {

enum { U_NONE = 0, U_SIGN = 2, U_TOPK = 3, U_RANDK = 4, U_LDITHER = 5, U_NDITHER = 6 };

__device__ __forceinline__ void adam1(float g, float& m, float& v, float& x, const UpdateParams& p) {
  m = fadd(fmul(p.beta1, m), fmul(p.omb1, g));                 // line 12
  v = fadd(fmul(p.beta2, v), fmul(p.omb2, fmul(g, g)));        // line 13
  const float mh = fmul(m, p.bc1);                             // line 14 (bc1 = fl32(1/(1-b1^t)), R21)
  const float vh = fmul(v, p.bc2);                             // line 15
  const float r = fdiv(mh, fadd(__fsqrt_rn(vh), p.eps));       // line 16
  x = fsub(x, fmul(p.lr, fadd(r, fmul(p.wd, x))));             // x update (Adam core)
}

template <int KIND>
__global__ void __launch_bounds__(UNT) update_kernel(const __grid_constant__ UpdateParams p) {
  constexpr bool SPARSE = KIND == U_TOPK || KIND == U_RANDK;
  __shared__ float gts[SPARSE ? UTILE : 1];
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
    if (full) {
      m4[it] = ld4(m + j);
      v4[it] = ld4(v + j);
      x4[it] = ld4(x + j);
    } else if (4 * i4 < tl.len) {
      m4[it] = load4_masked(m, j, L);
      v4[it] = load4_masked(v, j, L);
      x4[it] = load4_masked(x, j, L);
    }
  }
  if constexpr (SPARSE) {
    if (!raw) {
      for (uint32_t i = threadIdx.x; i < UTILE; i += UNT) gts[i] = 0.f;
      __syncthreads();
      const uint32_t k = c.k;
      const uint32_t* idx = reinterpret_cast<const uint32_t*>(pay + 8);
      const float* val = reinterpret_cast<const float*>(pay + 8 + 4ull * k);
      const uint32_t lo = warp_lower_bound(idx, k, tl.start);
      for (uint32_t e = lo + threadIdx.x; e < k; e += UNT) {
        const uint32_t j = idx[e];
        if (j >= tl.start + tl.len) break;
        gts[j - tl.start] = val[e];
      }
      __syncthreads();
    }
  }
  const float hdr = raw ? 0.f : *reinterpret_cast<const float*>(pay);
  const float sl = (float)((1u << (b - 1)) - 1u);
  const int cmax = (1 << (b - 1)) - 1;
  const float unit = fdiv(hdr, sl);
#pragma unroll
  for (int it = 0; it < UIT; it++) {
    const uint32_t i4 = it * UNT + threadIdx.x;
    const uint32_t j = tl.start + 4 * i4;
    if (!full && 4 * i4 >= tl.len) continue;
    float4 g4;
    if (raw || KIND == U_NONE) {
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
    adam1(g4.x, m4[it].x, v4[it].x, x4[it].x, p);
    adam1(g4.y, m4[it].y, v4[it].y, x4[it].y, p);
    adam1(g4.z, m4[it].z, v4[it].z, x4[it].z, p);
    adam1(g4.w, m4[it].w, v4[it].w, x4[it].w, p);
    if (full) {
      st4(m + j, m4[it]);
      st4(v + j, v4[it]);
      st4(x + j, x4[it]);
    } else {
      store4_masked(m, j, L, m4[it]);
      store4_masked(v, j, L, v4[it]);
      store4_masked(x, j, L, x4[it]);
    }
  }
}

cudaError_t launch_update(int kind, const UpdateParams& p, cudaStream_t s) {
  if (p.n_tiles == 0) return cudaSuccess;
  const dim3 grid(p.n_tiles), block(UNT);
  switch (kind) {
    case U_NONE: update_kernel<U_NONE><<<grid, block, 0, s>>>(p); break;
    case U_SIGN: update_kernel<U_SIGN><<<grid, block, 0, s>>>(p); break;
    case U_TOPK: update_kernel<U_TOPK><<<grid, block, 0, s>>>(p); break;
    case U_RANDK: update_kernel<U_RANDK><<<grid, block, 0, s>>>(p); break;
    case U_LDITHER: update_kernel<U_LDITHER><<<grid, block, 0, s>>>(p); break;
    case U_NDITHER: update_kernel<U_NDITHER><<<grid, block, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace bpc
