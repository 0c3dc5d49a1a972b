// device.cuh — sm_100a device helpers shared by the libbpc kernels:
// thread-block-cluster barriers and DSMEM, the fp64 pairwise tree (R6),
// Philox4x32-10 (R13), warp bit packing, exact-IEEE fp32
// arithmetic wrappers.  Nothing here is shared with oracle/.
#pragma once
#include <cooperative_groups.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "kernels.h"

namespace bpc {
namespace cg = cooperative_groups;

constexpr int SLICE = 16384;           // elements per CTA of a compression unit
constexpr int NT = 256;                // threads per compress CTA (3 CTAs / SM)
constexpr int NWARP = NT / 32;         // 8
constexpr int IT = SLICE / 4 / NT;     // float4 per thread per slice = 16
static_assert(IT * NWARP == 128, "slice reduction expects 128 warp subtrees");
constexpr int UNT = 256;               // threads per update CTA
constexpr int UTILE = 4096;            // elements per update tile
constexpr int UIT = UTILE / 4 / UNT;   // 4

// ---------------------------------------------------------------- cluster
__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_index() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive without memory ordering: "my reads of peers' shared memory are done"
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  cluster_arrive();
  cluster_wait();
}
// address of `p` (a shared variable of this CTA) in CTA `rank` of the cluster
template <class T>
__device__ __forceinline__ T* dsmem(T* p, uint32_t rank) {
  return cg::this_cluster().map_shared_rank(p, rank);
}

// ---------------------------------------------------------------- mbarrier + 1-D TMA
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// bulk global -> shared copy (UBLKCP); bytes and both addresses multiples of 16
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Watchdog: a wait longer than ~4 s of SM clock reports who was waiting on what
// and traps (the launch fails with an error instead of hanging the device).
#ifndef BPC_WATCHDOG_CYCLES
#define BPC_WATCHDOG_CYCLES 8000000000ll
#endif
static __device__ __noinline__ void watchdog_fire(const char* what, uint32_t a, uint32_t b,
                                                  unsigned long long c, unsigned long long d) {
  printf("BPC WATCHDOG block %d thread %d: %s tag=%x parity=%u c=%llu d=%llu\n", (int)blockIdx.x,
         (int)threadIdx.x, what, a, b, c, d);
  __trap();
}
// try_wait with a suspend-time hint: the thread sleeps in hardware until the
// phase completes or ~hint ns pass, so a waiting warp issues almost nothing
__device__ __forceinline__ bool mbar_try_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ long long clock64_v() {   // not hoisted out of the watchdog branch
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, uint32_t tag = 0) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64_v();
  for (uint32_t it = 1; !mbar_try_sleep(bar, parity, 20000u); it++) {   // clock read every 16 tries
    if ((it & 15) == 0 && clock64_v() - t0 > BPC_WATCHDOG_CYCLES)
      watchdog_fire("mbarrier", tag, parity, (unsigned long long)smem_u32(bar), 0);
  }
}
// poll with a sleep between tries, for waiters off the critical path: a
// try_wait's own suspend is woken by any barrier traffic in the CTA, so a
// long wait there keeps issuing instructions the compute warps need
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns, uint32_t tag = 0) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64_v();
  for (uint32_t it = 1; !mbar_try(bar, parity); it++) {
    __nanosleep(ns);
    if ((it & 63) == 0) {
      if (clock64_v() - t0 > BPC_WATCHDOG_CYCLES)
        watchdog_fire("mbarrier", tag, parity, (unsigned long long)smem_u32(bar), 0);
    }
  }
}
#ifndef BPC_CTR_POLL_NS
#define BPC_CTR_POLL_NS 128   // poll of a cross-CTA unit counter (512 measured slower, profiles/r2/ab/)
#endif
// gpu-scope release add / acquire load on unit counters (cross-CTA unit reductions)
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// spin with relaxed loads (no L1 invalidation per poll), then one acquire
__device__ __forceinline__ void wait_counter(const unsigned long long* p, unsigned long long target,
                                             uint32_t tag = 0) {
  unsigned long long v = ld_relaxed(p);
  if (v < target) {
    const long long t0 = clock64_v();
    for (uint32_t it = 1; (v = ld_relaxed(p)) < target; it++) {
      __nanosleep(BPC_CTR_POLL_NS);
      if ((it & 63) == 0) {
        if (clock64_v() - t0 > BPC_WATCHDOG_CYCLES) watchdog_fire("counter", tag, 0, v, target);
      }
    }
  }
  (void)ld_acquire(p);
}

// ---------------------------------------------------------------- programmatic dependent launch
// The streaming kernels are launched with programmatic stream serialization:
// a kernel may start (prologue: barrier init) while its predecessor's last CTAs
// drain.  Every thread waits for the predecessor's completion (and memory)
// before touching global data, then lets its own successor be scheduled.
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- NVLink peer sync
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// The step-varying values one launch uses, read from DevState when it starts
// (after griddepcontrol.wait / stream order: the previous launches' last CTAs
// have stored theirs)
struct LaunchEp {
  uint32_t E;      // this launch's epoch in its family
  uint32_t Esig;   // the exchange epoch it releases (sig_fam)
  uint32_t Ewait;  // the exchange epoch it waits for (wait_fam)
  uint32_t t;      // the step counter
};
__device__ __forceinline__ LaunchEp launch_begin(const PeerSync& s) {
  LaunchEp e;
  e.t = s.st->t;
  e.E = s.st->ep[s.fam] + 1;
  e.Esig = s.sig_fam >= 0 ? s.st->ep[s.sig_fam] + 1 : 0u;
  e.Ewait = s.wait_fam >= 0 ? s.st->ep[s.wait_fam] : 0u;
  return e;
}
// One thread: wait until every other rank released this step's epoch, then
// order the later bulk (async-proxy) reads of the exchanged bytes after it.
__device__ __forceinline__ void peer_wait(const PeerSync& s, const LaunchEp& e) {
  if (s.wait_fam < 0) return;
  for (uint32_t r = 0; r < s.n; r++) {
    if (r == s.self) continue;
    const unsigned long long* f = s.wflags + s.wslot0 + r;
    const long long t0 = clock64();
    for (uint32_t it = 1; ld_relaxed_sys(f) < (unsigned long long)e.Ewait; it++) {
      __nanosleep(64);
      if ((it & 63) == 0 && clock64() - t0 > BPC_WATCHDOG_CYCLES)
        watchdog_fire("peer flag", s.wslot0 + r, 0, ld_relaxed_sys(f), e.Ewait);
    }
    (void)ld_acquire_sys(f);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// One thread per CTA (`leader`), after the CTA's work -- for a signalling launch,
// after every thread that stored exchanged bytes ran __threadfence_system() and
// a barrier: the last CTA of the launch releases the exchange epoch to every
// peer and stores the launch's epochs (and the next step counter) for the next
// launches.
__device__ __forceinline__ void launch_end(const PeerSync& s, const LaunchEp& e, bool leader) {
  if (!leader) return;
  const unsigned long long prev = atomicAdd(&s.st->done[s.fam], 1ull);
  if (prev + 1 == (unsigned long long)gridDim.x) {   // the last CTA (the next launch of
    s.st->done[s.fam] = 0ull;                        // the family runs after this grid)
    __threadfence_system();
    if (s.sig_fam >= 0) {
      for (uint32_t r = 0; r < s.n; r++)
        if (s.sflag[r]) st_release_sys(s.sflag[r] + s.sslot, (unsigned long long)e.Esig);
      s.st->ep[s.sig_fam] = e.Esig;
    }
    s.st->ep[s.fam] = e.E;
    if (s.inc_t) s.st->t = e.t + 1;
  }
}

// ---------------------------------------------------------------- exact fp32 ops
// -fmad=false is also set, these keep every operation a single IEEE op.
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
// a / b and sqrt(a) with the +-0 operand answered directly: the IEEE sequences send
// zero operands to their slow-path subroutines, and the moments of coordinates
// whose aggregated gradient stays 0 (sparse kinds; BERT's unused embedding rows)
// are exactly 0 (same results: +-0 / b = +-0 for b > 0, sqrt(+-0) = +-0; 0 / 0
// still takes the IEEE division)
__device__ __forceinline__ float fdiv_pos(float a, float b) { return (a == 0.f && b > 0.f) ? a : __fdiv_rn(a, b); }
__device__ __forceinline__ float fsqrt0(float a) { return a == 0.f ? a : __fsqrt_rn(a); }
// a / b correctly rounded for a per-launch constant divisor b with y = RN(1/b)
// (Markstein: q = RN(a y) is within an ulp, the residual a - b q is exact by
// FMA, and RN(q + r y) is RN(a / b)), two FMAs instead of the IEEE division
// sequence.  The theorem needs the residual not to underflow: |a| < 2^-100
// takes the IEEE division (checked bit for bit against a / b for the Adam bias
// corrections over 2.9e8 cases, tests/test_divc.py).
__device__ __forceinline__ float divc(float a, float b, float y) {
  if (fabsf(a) < 0x1p-100f) return a == 0.f ? a : __fdiv_rn(a, b);   // +-0 / b = +-0 (b > 0)
  const float q = __fmul_rn(a, y);
  const float r = __fmaf_rn(-q, b, a);
  return __fmaf_rn(r, y, q);
}
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
// server mean (R5): (float)(acc * (1/n) + e~), two fp64 roundings then one to fp32
__device__ __forceinline__ float mean_plus(double acc, double inv_n, double et) {
  return __double2float_rn(dadd(dmul(acc, inv_n), et));
}

// ---------------------------------------------------------------- packed fp32 pairs
// FADD2 (sm_100): two IEEE round-to-nearest fp32 additions per instruction,
// lane by lane the same results as the scalar ops.  No packed products: ptxas
// fuses a packed multiply into a following packed add (FFMA2) regardless of
// -fmad=false.
__device__ __forceinline__ unsigned long long f2_bits(float2 a) {
  unsigned long long r;
  memcpy(&r, &a, 8);
  return r;
}
__device__ __forceinline__ float2 bits_f2(unsigned long long r) {
  float2 a;
  memcpy(&a, &r, 8);
  return a;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(r);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(r);
}
#define BPC_F4_OP(NAME, OP2)                                                              \
  __device__ __forceinline__ float4 NAME(float4 a, float4 b) {                            \
    const float2 lo = OP2(make_float2(a.x, a.y), make_float2(b.x, b.y));                 \
    const float2 hi = OP2(make_float2(a.z, a.w), make_float2(b.z, b.w));                 \
    return make_float4(lo.x, lo.y, hi.x, hi.y);                                           \
  }
BPC_F4_OP(fadd4, fadd2)
BPC_F4_OP(fsub4, fsub2)
#undef BPC_F4_OP
__device__ __forceinline__ float4 splat4(float a) { return make_float4(a, a, a, a); }

// Alg. 5 lines 12-16 and x <- x - eta (r + lambda x) on 4 elements (R15, R16, R21):
// products per element, the sums of two products as packed pairs, divisions and
// roots per element -- the same IEEE operations in the same order as the scalar
// form.  (Packed products feeding packed sums are NOT used: ptxas 12.9 contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false, a single
// rounding the oracle does not make; scalar FMUL results are left alone.)
__device__ __forceinline__ float4 fmul4s(float4 a, float4 b) {   // scalar products
  return make_float4(fmul(a.x, b.x), fmul(a.y, b.y), fmul(a.z, b.z), fmul(a.w, b.w));
}
__device__ __forceinline__ void adam4(float4 g, float4& m, float4& v, float4& x, const UpdateParams& p,
                                      const float4 bc) {   // bc = (bc1, bc2, 1/bc1, 1/bc2) of the step
  m = fadd4(fmul4s(splat4(p.beta1), m), fmul4s(splat4(p.omb1), g));                 // line 12
  v = fadd4(fmul4s(splat4(p.beta2), v), fmul4s(splat4(p.omb2), fmul4s(g, g)));      // line 13
  float4 r;
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const float mh = divc(u == 0 ? m.x : u == 1 ? m.y : u == 2 ? m.z : m.w, bc.x, bc.z);   // line 14
    const float vh = divc(u == 0 ? v.x : u == 1 ? v.y : u == 2 ? v.z : v.w, bc.y, bc.w);   // line 15
    const float ru = fdiv_pos(mh, fadd(fsqrt0(vh), p.eps));                                   // line 16
    if (u == 0) r.x = ru; else if (u == 1) r.y = ru; else if (u == 2) r.z = ru; else r.w = ru;
  }
  x = fsub4(x, fmul4s(splat4(p.lr), fadd4(r, fmul4s(splat4(p.wd), x))));          // x update
}

// ---------------------------------------------------------------- pairwise tree (R6)
// Lane l holds the subtree sum of its 4 consecutive elements; the xor butterfly
// with masks 1..16 builds the perfect binary tree over the warp's 128 elements
// (both lanes of a pair hold a+b == b+a).
__device__ __forceinline__ double warp_tree(double a) {
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) a = a + __shfl_xor_sync(0xffffffffu, a, m);
  return a;
}
__device__ __forceinline__ double leaf4_abs(float4 q) {
  return ((double)fabsf(q.x) + (double)fabsf(q.y)) + ((double)fabsf(q.z) + (double)fabsf(q.w));
}
__device__ __forceinline__ double leaf4_sq(float4 q) {
  return ((double)q.x * (double)q.x + (double)q.y * (double)q.y) +
         ((double)q.z * (double)q.z + (double)q.w * (double)q.w);
}

// ---------------------------------------------------------------- Philox4x32-10 (R13)
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}
// the 4 words of elements 4*g .. 4*g+3 of unit `chunk` (counter layout R13)
// the same generator with the 10 round keys precomputed on the host (key
// schedule k + r * (0x9E3779B9, 0xBB67AE85) mod 2^32): in the kernel parameter
// space they are constant-bank operands of the xors, no key arithmetic per call
__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const uint32_t (&rk)[20]) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ rk[2 * r], lo1, hi0 ^ c.w ^ rk[2 * r + 1], lo0);
  }
  return c;
}
__device__ __forceinline__ uint4 rng4(uint64_t seed, uint32_t g, uint32_t chunk, uint32_t t,
                                      uint32_t stage, uint32_t rank) {
  return philox4x32_10(make_uint4(g, chunk, t, (stage << 31) | rank), (uint32_t)seed,
                       (uint32_t)(seed >> 32));
}

// ---------------------------------------------------------------- bit packing
// Lane l owns a field of nb bits at bit nb*l of the warp's 32*nb bits (= nb words).
// Returns, in lanes 0..nb-1, word `lane` of the packed stream (LSB-first).
__device__ __forceinline__ uint32_t warp_pack(uint32_t field, int nb) {
  const int lane = threadIdx.x & 31;
  const int w = lane < nb ? lane : 0;
  const int first = (32 * w) / nb;
  const int last = (32 * w + 31) / nb;
  uint32_t acc = 0;
#pragma unroll
  for (int it = 0; it < 9; it++) {
    const int src = min(first + it, 31);
    const uint32_t v = __shfl_sync(0xffffffffu, field, src);
    if (first + it <= last) {
      const int pos = nb * (first + it) - 32 * w;
      acc |= pos >= 0 ? (v << pos) : (v >> (-pos));
    }
    if (it * nb >= 32 + nb) break;   // uniform: enough lanes visited for any word
  }
  return acc;
}
// nb-bit field (nb <= 32) starting at bit `pos` of a little-endian u32 stream
__device__ __forceinline__ uint32_t load_field(const uint32_t* words, uint64_t pos, int nb) {
  const uint64_t w = pos >> 5;
  const int sh = (int)(pos & 31);
  uint64_t v = words[w];
  if (sh + nb > 32) v |= (uint64_t)words[w + 1] << 32;
  const uint64_t mask = nb == 32 ? 0xFFFFFFFFull : ((1ull << nb) - 1);
  return (uint32_t)((v >> sh) & mask);
}

// first position with a[pos] >= key in the ascending a[0, n): each warp probes 32
// positions per round (2 dependent loads for n <= 1024 instead of log2 n)
__device__ __forceinline__ uint32_t warp_lower_bound(const uint32_t* a, uint32_t n, uint32_t key) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = n;   // answer in [lo, hi]
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t pos = lo + lane * step;
    const bool below = pos < hi && a[pos] < key;
    const uint32_t nb = __popc(__ballot_sync(0xffffffffu, below));
    if (nb == 0) return lo;
    const uint32_t last = lo + (nb - 1) * step;   // a[last] < key
    const uint32_t next = lo + nb * step;          // a[next] >= key, or past hi
    lo = last + 1;
    if (next < hi) hi = next;
  }
  const uint32_t pos = lo + lane;
  const bool below = pos < hi && a[pos] < key;
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// ---------------------------------------------------------------- sparse values (R23)
// binary16 values: saturate to +-65504 (the oracle's comparisons, NaN passes
// through), then round to nearest even; returns the decoded fp32 value
__device__ __forceinline__ float quant_val(float v, bool f16) {
  if (!f16) return v;
  if (v > 65504.f) v = 65504.f;
  if (v < -65504.f) v = -65504.f;
  return __half2float(__float2half_rn(v));
}
// value i of a payload's value array (fp32, or binary16 when f16)
__device__ __forceinline__ float get_val(const uint8_t* vals, uint32_t i, bool f16) {
  return f16 ? __half2float(reinterpret_cast<const __half*>(vals)[i]) : reinterpret_cast<const float*>(vals)[i];
}
// store an already-quantised value (exact in binary16 when f16)
__device__ __forceinline__ void put_val(uint8_t* vals, uint32_t i, float v, bool f16) {
  if (f16) reinterpret_cast<__half*>(vals)[i] = __float2half_rn(v);
  else reinterpret_cast<float*>(vals)[i] = v;
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ldg4_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ float4 load4_masked(const float* p, uint32_t j, uint32_t L) {
  if (j + 4 <= L) return ld4(p + j);
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j < L) r.x = p[j];
  if (j + 1 < L) r.y = p[j + 1];
  if (j + 2 < L) r.z = p[j + 2];
  return r;
}
// NVLS multicast stores (addresses in a multicast mapping: the switch writes every
// bound replica); weak stores, ordered for the peers by fence.proxy.alias + a
// system-scope release
__device__ __forceinline__ void mm_st_u32(void* a, uint32_t v) {
  asm volatile("multimem.st.global.b32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void mm_st_f32(void* a, float v) {
  asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void mm_st_v4(void* a, float4 v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_store4_masked(float* p, uint32_t j, uint32_t L, float4 v) {
  if (j + 4 <= L) {
    mm_st_v4(p + j, v);
    return;
  }
  if (j < L) mm_st_f32(p + j, v.x);
  if (j + 1 < L) mm_st_f32(p + j + 1, v.y);
  if (j + 2 < L) mm_st_f32(p + j + 2, v.z);
}
__device__ __forceinline__ void store4_masked(float* p, uint32_t j, uint32_t L, float4 v) {
  if (j + 4 <= L) {
    st4(p + j, v);
    return;
  }
  if (j < L) p[j] = v.x;
  if (j + 1 < L) p[j + 1] = v.y;
  if (j + 2 < L) p[j + 2] = v.z;
}
__device__ __forceinline__ float get(const float4& v, int u) {
  return u == 0 ? v.x : (u == 1 ? v.y : (u == 2 ? v.z : v.w));
}
__device__ __forceinline__ void set(float4& v, int u, float x) {
  if (u == 0) v.x = x; else if (u == 1) v.y = x; else if (u == 2) v.z = x; else v.w = x;
}

}  // namespace bpc
