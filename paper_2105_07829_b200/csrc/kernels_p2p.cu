// kernels_p2p.cu — the exchange steps A4 (push delta to the owners) and A8
// (broadcast p) over NVLink peer memory: every rank maps
// its peers' RECV, P and flag buffers with CUDA IPC, stores its payload bytes
// straight into them from SM warps (16-byte st.global over NVLink), then
// publishes a per-step epoch into each peer's flag array with a system-scope
// release.  The consumer side waits with system-scope acquire loads.  No NCCL
// call, no staging copy on the receiver.
#include "device.cuh"

namespace bpc {

// Copy job j: bytes [src_j, src_j + len_j) -> dst_j (all 16-byte aligned).  The
// grid strides over all jobs' 16-byte words; afterwards the last CTA to finish
// releases `epoch` into flag slot `slot` of every peer.
__global__ void __launch_bounds__(512) p2p_copy_signal(const __grid_constant__ P2PParams p) {
  const LaunchEp ep = launch_begin(p.sync);   // fam = sig_fam: the exchange epoch of this copy
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int jb = 0; jb < p.njobs; jb++) {
    const uint64_t nw = p.len[jb] / 16;
    const int4* s = reinterpret_cast<const int4*>(p.src[jb]);
    int4* d = reinterpret_cast<int4*>(p.dst[jb]);
    uint64_t w = g0;
    auto put = [&](uint64_t i, int4 v) {
      if (p.mc) mm_st_v4(d + i, make_float4(__int_as_float(v.x), __int_as_float(v.y), __int_as_float(v.z),
                                            __int_as_float(v.w)));
      else d[i] = v;
    };
    for (; w + 3 * stride < nw; w += 4 * stride) {   // 4 independent 16-byte copies in flight
      const int4 a = __ldg(s + w), b = __ldg(s + w + stride), c = __ldg(s + w + 2 * stride),
                 e = __ldg(s + w + 3 * stride);
      put(w, a);
      put(w + stride, b);
      put(w + 2 * stride, c);
      put(w + 3 * stride, e);
    }
    for (; w < nw; w += stride) put(w, __ldg(s + w));
  }
  // make this CTA's peer (or multicast) stores visible system-wide; the last CTA
  // releases the epoch
  if (p.mc) asm volatile("fence.proxy.alias;" ::: "memory");
  __threadfence_system();
  __syncthreads();
  launch_end(p.sync, ep, threadIdx.x == 0);
}

// One warp waits until flags[i] >= the epoch of family `fam` for every listed slot.
__global__ void p2p_wait(const __grid_constant__ P2PWait w) {
  const int lane = threadIdx.x;
  const unsigned long long epoch = w.st->ep[w.fam];
  for (int i = lane; i < w.nslots; i += 32) {
    const unsigned long long* f = w.flags + w.slots[i];
    const long long t0 = clock64();
    for (uint32_t it = 1; ld_relaxed_sys(f) < epoch; it++) {
      __nanosleep(100);
      if ((it & 63) == 0 && clock64() - t0 > BPC_WATCHDOG_CYCLES)
        watchdog_fire("p2p flag", (uint32_t)w.slots[i], 0, ld_relaxed_sys(f), epoch);
    }
    (void)ld_acquire_sys(f);
  }
  __syncwarp();
  __threadfence_system();
}

cudaError_t launch_p2p_copy(const P2PParams& p, int grid, cudaStream_t s) {
  p2p_copy_signal<<<grid, 512, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_p2p_wait(const P2PWait& w, cudaStream_t s) {
  p2p_wait<<<1, 32, 0, s>>>(w);
  return cudaGetLastError();
}

}  // namespace bpc
