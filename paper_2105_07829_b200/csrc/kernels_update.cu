// kernels_update.cu — the LANS block coefficients (NEXT #1, R22) between the
// two update passes.  The update itself (A9, every kind) is update_stream in
// kernels_stream.cu.
#include "device.cuh"

namespace bpc {

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

}  // namespace bpc
