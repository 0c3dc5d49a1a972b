// kernels_cstream.cu — persistent, warp-specialised worker and server kernels
// for the norm-based compressors (scaled sign, linear / natural dithering) and
// raw units (sm_100a).
//
//   worker: q = g + e (Alg. 4 l.5),
//           delta = C(q) (l.6), e = q - dec(delta) (l.7)
//   server  (A5-A7): Delta = (1/n) sum_i dec(delta_i) + e~ (l.10),
//           p = C(Delta) (l.11), e~ = Delta - dec(p) (l.13)
//
// One CTA per SM walks 2^13-element slices of its units.  Shared memory holds
// two rings sized at launch:
//   HELD ring  (NH x 32 KB)  q (worker: g lands here by TMA, q = g + e in place)
//                            or Delta (server), kept until the slice is emitted;
//                            the emit overwrites it with the error e / e~ (or it
//                            holds a raw unit's values), which the producer
//                            writes back with one bulk store (TMA, full sectors);
//   INPUT ring (NI x SI)     e (worker) or the n ranks' payload bytes (server),
//                            released as soon as the slice is produced.
// Warps:
//   PRODUCER   reads the slice descriptors, issues the 1-D bulk loads
//              (cp.async.bulk -> UBLKCP, one mbarrier complete_tx per slice) and
//              the bulk stores of emitted slices (cp.async.bulk.global.shared);
//   4 REDUCERS (slice i -> reducer i % 4) complete each unit's fp64 pairwise-tree
//              total (R6): a multi-slice unit publishes one partial per
//              slice (release add on a per-unit counter) and each slice's reducer
//              waits (relaxed spin + one acquire) for the unit, then reduces it;
//   16 CONSUMERS produce slice i (q or Delta, slice partial) and then emit slice
//              i - D (sign bits / codes + error) once its total is ready,
//              D = NH - 2 <= 3, so the cross-CTA wait overlaps useful work.
//
// Consumer layout (round 2): warp w owns elements [512 w, 512 w + 512) of a
// slice and lane l the 16 contiguous elements [512 w + 16 l, + 16), i.e. float4
// groups 4 l' .. 4 l' + 3 (l' = 32 w + l).  So a lane's 16 elements are one
// subtree of R6's pairwise tree (15 fp64 adds in registers, then a 5-level
// butterfly for the warp's 512), its 16 sign bits are one half-word of the
// payload and its 16 codes one 16 b-bit field: no cross-lane packing loops.
// The lane visits its groups in the rotated order k = (s + (l >> 1)) & 3,
// s = 0..3: eight consecutive lanes then touch eight distinct 16-byte bank
// groups, so the 16-byte shared-memory accesses are conflict-free although the
// lanes are 64 bytes apart (a plain order would be 4-way conflicted).
// All CTAs are co-resident (cooperative launch) and every slice's partial is
// published before its CTA waits on an earlier unit, so the waits cannot
// deadlock.  Each mbarrier has a single in-order waiter group; the reducers,
// run out of order (slice i -> reducer i % 4) but each waits on its slice's
// held-stage barrier, which cannot run a phase ahead of it.
#include <cstdlib>
#include <type_traits>

#include "device.cuh"

namespace bpc {

enum { C_NONE = 0, C_SIGN = 2, C_TOPK = 3, C_RANDK = 4, C_LDITHER = 5, C_NDITHER = 6 };

constexpr int CCW = 16;                  // consumer warps
constexpr int CCNT = 32 * CCW;           // consumer threads
constexpr int CPROD = CCW;               // producer warp index
constexpr int CRED = CCW + 1;            // first reducer warp index
constexpr int CRW = 4;                   // reducer warps (slice i -> reducer i % CRW)
constexpr int CSNT = CCNT + 32 + 32 * CRW;   // + producer + reducers
constexpr int CMAXH = 8;                 // max held stages
constexpr int CNI = 2;                   // input stages
constexpr int CMAXD = 3;                 // max emit deferral (D = 4 measured slower for the server)
constexpr int CRED_R = CMAXD + 1;        // ring of the consumer warps' slice subtrees (>= D + 1)
#ifndef BPC_RED_POLL_NS
#define BPC_RED_POLL_NS 200    // reducer poll of the slice-produced barrier (1000: C2 server +2.5 %)
#endif
constexpr int CSL = 8192;                // elements per slice
constexpr int CLE = 16;                  // elements per consumer lane per slice
constexpr int CUNITSL = (1 << 18) / CSL; // max slices per unit (32)
static_assert(CSL == CCNT * CLE, "one slice = 16 elements per consumer lane");

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

struct CDesc {
  uint64_t off;        // worker: flat element offset of the chunk
  uint64_t pay;        // payload byte offset (SEND / P)
  uint64_t recv;       // server: offset inside each RECV slot
  uint64_t etl;        // server: e~ element offset
  uint32_t start, len, L, id;
  uint32_t nslices, sidx, unit, unit_first;
  uint32_t pofs;       // server: byte offset of the slice's first field inside a staged piece
  uint32_t staged;     // server: payload pieces staged in smem
  uint32_t owner;      // server rank of the chunk (worker: fused push destination)
  uint32_t gsl;        // the slice's index in this side's slice table
  uint32_t sp_u, sp_g, sp_cs;   // sparse kinds: unit index, candidate threshold, sub-list capacity
};

struct __align__(128) CHead {
  uint64_t fullI[CNI], emptyI[CNI], emptyH[CMAXH], tready[CMAXH];
  uint64_t pready[CMAXH];   // slice in held stage s produced (its reducer waits on it)
  uint64_t pfin;            // fused exchange: the producer's last bulk store has completed
  CDesc desc[CMAXH];
  double red[CRED_R][CCW];  // the consumer warps' 512-element subtrees of slice i at i % CRED_R
  uint32_t wcnt[2 * CCW];   // sparse kinds: candidates per consumer warp of the emitting slice (2 buffers)
  double part[CMAXH];
  float4 dv[CMAXH];         // the slice's unit scalars from its total (reducer): sign (s);
                            // dithering (N, RN(s_l / N) or 0, RN(N / s_l))
};

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(CCNT) : "memory");
}
// bulk shared -> global copy (UBLKCP), tracked by the issuing thread's bulk groups
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {   // sources of every committed store read
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {        // every committed store complete
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 128-bit field helpers (a lane's 16 b-bit codes, b <= 8)
struct U128 {
  uint64_t lo, hi;
};
__device__ __forceinline__ uint32_t u128_get(const U128& a, uint32_t s) {   // bits [s, s + 32)
  uint64_t v;
  if (s == 0) v = a.lo;
  else if (s < 64) v = (a.lo >> s) | (a.hi << (64 - s));
  else v = a.hi >> (s - 64);
  return (uint32_t)v;
}
__device__ __forceinline__ void u128_or(U128& a, uint32_t x, uint32_t s) {   // a |= x << s (s < 128)
  const uint64_t v = x;
  if (s < 64) {
    a.lo |= v << s;
    if (s > 32) a.hi |= v >> (64 - s);
  } else {
    a.hi |= v << (s - 64);
  }
}
__device__ __forceinline__ U128 u128_shr(const U128& a, uint32_t s) {   // s < 64
  if (s == 0) return a;
  return U128{(a.lo >> s) | (a.hi << (64 - s)), a.hi >> s};
}
// shifts by a warp-uniform amount s < 128 (uniform branches only)
__device__ __forceinline__ U128 u128_shl_u(const U128& a, uint32_t s) {
  if (s == 0) return a;
  if (s < 64) return U128{a.lo << s, (a.hi << s) | (a.lo >> (64 - s))};
  return U128{0, a.lo << (s - 64)};
}
__device__ __forceinline__ U128 u128_shr_u(const U128& a, uint32_t s) {
  if (s == 0) return a;
  if (s < 64) return U128{(a.lo >> s) | (a.hi << (64 - s)), a.hi >> s};
  return U128{a.hi >> (s - 64), 0};
}
// rotate a w-bit field (w <= 128, bits above w zero) left by a uniform r < w
__device__ __forceinline__ U128 u128_rotl_u(const U128& a, uint32_t r, uint32_t w) {
  const U128 x = u128_shl_u(a, r), y = u128_shr_u(a, w - r);
  U128 m = u128_shl_u(U128{~0ull, ~0ull}, 128 - w);
  m = u128_shr_u(m, 128 - w);   // low w bits
  return U128{(x.lo | y.lo) & m.lo, (x.hi | y.hi) & m.hi};
}
// a |= x << s for a warp-uniform s < 128 (x < 2^32)
__device__ __forceinline__ U128 u128_or_u(const U128& a, uint32_t x, uint32_t s) {
  const U128 v = u128_shl_u(U128{x, 0}, s);
  return U128{a.lo | v.lo, a.hi | v.hi};
}
__device__ __forceinline__ U128 u128_sel(bool c, const U128& a, const U128& b) {
  return U128{c ? a.lo : b.lo, c ? a.hi : b.hi};
}
// the lane's 16 codes in element order (group k at bit 4 b k) from the per-step
// group fields f0 (bits 4 b s for step s, group k = (s + rot) & 3): rotate left by
// 4 b rot = 4 b (rot & 1) + 8 b (rot & 2) / 2 with uniform amounts and per-lane selects
__device__ __forceinline__ U128 unrotate_field(const U128& f0, uint32_t rot, uint32_t gb) {
  const uint32_t w = 4 * gb;
  U128 f = u128_sel(rot & 1u, u128_rotl_u(f0, gb, w), f0);
  return u128_sel(rot & 2u, u128_rotl_u(f, 2 * gb, w), f);
}
// the inverse: step s's group at bit 4 b s (f's bits at and above 4 gb, the next
// lane's codes of a loaded field, are dropped first)
__device__ __forceinline__ U128 rotate_field(const U128& fin, uint32_t rot, uint32_t gb) {
  const uint32_t w = 4 * gb;
  const U128 m = u128_shr_u(U128{~0ull, ~0ull}, 128 - w);
  const U128 f{fin.lo & m.lo, fin.hi & m.hi};
  U128 g = u128_sel(rot & 1u, u128_rotl_u(f, w - gb, w), f);
  return u128_sel(rot & 2u, u128_rotl_u(g, w - 2 * gb, w), g);
}

// inv = fl32(s / N), or 0 when N = 0: then every q of the unit is +-0, r = 0 and
// the level is 0 without a branch (N = 0 implies all-zero q: q*q is exact in fp64)
__device__ __forceinline__ uint32_t lin_code_c(float q, float sl, float inv, uint32_t w) {
  const uint32_t sign = !(q < 0.f);
  const float r = fminf(fmul(fabsf(q), inv), sl);
  const float l = floorf(r);
  const float f = fsub(r, l);
  const float u = (float)(w >> 8) * 0x1p-24f;
  const uint32_t level = (uint32_t)l + (u < f ? 1u : 0u);
  return sign | (level << 1);
}
__device__ __forceinline__ uint32_t nat_code_c(float q, float N, int cmax, float lmin, uint32_t w) {
  const uint32_t sign = !(q < 0.f);
  uint32_t code = 0;
  if (N != 0.f) {
    const float r = fminf(fdiv_pos(fabsf(q), N), 1.0f);
    const float u = (float)(w >> 8) * 0x1p-24f;
    if (r >= lmin) {
      const int eb = (int)(__float_as_uint(r) >> 23);
      const float lo = __uint_as_float((uint32_t)eb << 23);
      const float pup = fsub(fdiv_pos(r, lo), 1.0f);
      const int e_lev = (u < pup) ? eb - 127 + 1 : eb - 127;
      code = (uint32_t)(cmax + e_lev);
    } else {
      code = (u < fdiv_pos(r, lmin)) ? 1u : 0u;
    }
  }
  return sign | (code << 1);
}
// |dec| of a dithering code
template <int KIND>
__device__ __forceinline__ float dither_mag(uint32_t code, float hdr, float unit, int cmax) {
  if (KIND == C_LDITHER) return fmul((float)(code >> 1), unit);
  const uint32_t cl = code >> 1;
  return fmul(cl == 0 ? 0.f : __uint_as_float((uint32_t)(127 - (cmax - (int)cl)) << 23), hdr);
}

// FUSED (n > 1, BPC_EXCHANGE_P2P): the worker stores its payloads straight into
// the owners' RECV slots over NVLink and releases the push flags; the server
// waits for every rank's push before its first load and releases the pull
// flags after its last store (the update kernels read p from the owners' P).
// BITS: dithering bits as a compile-time constant (the paper's 3 / 5 / 7-bit runs,
// every shift of the code packing is then an immediate), or 0 =
// p.bits at run time
// X: 0 plain, 1 FUSED (n > 1, BPC_EXCHANGE_P2P), 2 the server at n = 1 (N1: one
// rank's payload, Delta = dec + e~ in fp32; the general n-rank code is not built)
template <int KIND, bool SERVER, int X, int BITS>
__global__ void __launch_bounds__(CSNT, 1) cstream_kernel(const __grid_constant__ StreamParams p) {
  constexpr bool FUSED = X == 1;
  constexpr bool N1 = SERVER && X == 2;
  extern __shared__ __align__(128) unsigned char sraw[];
  CHead& hd = *reinterpret_cast<CHead*>(sraw);
  const uint32_t NH = p.nstages;          // held stages
  const uint32_t D = p.defer;              // emit deferral, <= NH - 2 and <= CMAXD
  const uint32_t SI = p.stage_b;          // bytes per input stage
  const uint32_t SIE = p.stage_a;         // byte offset of the e region inside an input stage
  unsigned char* held = sraw + sizeof(CHead);
  unsigned char* input = held + (size_t)NH * CSL * 4;
  auto H = [&](uint32_t s) { return reinterpret_cast<float4*>(held + (size_t)s * CSL * 4); };
  // server input stage: [n x 16-byte payload heads][n payload pieces]
  const uint32_t HB = SERVER ? (16 * p.n + 127) / 128 * 128 : 0;
  auto IH = [&](uint32_t t) { return input + (size_t)t * SI; };               // payload heads
  auto I = [&](uint32_t t) { return input + (size_t)t * SI + HB; };          // payload pieces
  auto IE = [&](uint32_t t) { return reinterpret_cast<float4*>(input + (size_t)t * SI + SIE); };
  const uint32_t G = gridDim.x;
  const uint32_t mine = p.n_slices > blockIdx.x ? (p.n_slices - blockIdx.x + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // SPARSE (top-k, random-k; kernels_sparse.cu brackets this launch): the
  // streaming pass of a compressed unit computes q (worker) / reads Delta
  // (server) and lists the candidates with key >= G_u; the exact selection and
  // the payload follow in sparse_select
  constexpr bool SPARSE = KIND == C_TOPK || KIND == C_RANDK;
  const int b = (KIND == C_SIGN || SPARSE) ? 1 : (BITS ? BITS : (int)p.bits);   // bits per element in the payload stream
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NH; s++) {
      mbar_init(&hd.emptyH[s], CCW);
      mbar_init(&hd.tready[s], 1);
      mbar_init(&hd.pready[s], SPARSE ? 1 : CCW);   // every consumer warp (its subtree, its q)
    }
    for (uint32_t t = 0; t < (uint32_t)CNI; t++) {
      mbar_init(&hd.fullI[t], 1);
      mbar_init(&hd.emptyI[t], CCW);
    }
    mbar_init(&hd.pfin, 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait_and_release();
  const LaunchEp ep = launch_begin(p.sync);   // this launch's epoch, the step counter t

  // ===================================================== producer
  if (warp == CPROD) {
    if (lane == 0) {
      if (SERVER && FUSED) peer_wait(p.sync, ep);   // fused exchange: every rank's delta has landed in RECV
      // write-back of emitted slice ie (its held stage): the error e / e~, or a raw
      // unit's payload (worker: g; server: the mean), 16-byte-aligned part
      auto flush = [&](uint32_t ie) {
        const uint32_t hs = ie % NH;
        mbar_wait_backoff(&hd.emptyH[hs], (ie / NH) & 1, 128, 0x1000000u | ie);   // consumers emitted slice ie
        if (p.pass == 1) return;
        const CDesc& o = hd.desc[hs];
        const uint32_t nvb = (o.len & ~3u) * 4u;
        if (!nvb) return;
        uint8_t* dst = nullptr;
        if (o.nslices == 0) {
          if (SERVER && FUSED && p.mc_out) return;   // NVLS: the consumers multicast raw payloads
          uint8_t* pay = (!SERVER && FUSED) ? p.dst[o.owner] + o.recv : p.out + o.pay;
          dst = pay + 4ull * o.start;
        } else if (p.use_ef && !(SPARSE && SERVER)) {   // the sparse server only reads Delta
          dst = reinterpret_cast<uint8_t*>(p.err + (SERVER ? o.etl : o.off) + o.start);
        }
        if (dst) bulk_store(dst, H(hs), nvb);
      };
      // descriptors of the next slice are loaded before the stage waits, so their
      // latency overlaps the wait instead of delaying the bulk copies
      Slice sl_next = mine ? p.slices[blockIdx.x] : Slice{};
      DevChunk c_next = mine ? p.chunks[sl_next.chunk] : DevChunk{};
      for (uint32_t i = 0; i < mine; i++) {
        const uint32_t hs = i % NH, t = i % CNI;
        const Slice sl = sl_next;
        const DevChunk c = c_next;
        if (i + 1 < mine) {
          sl_next = p.slices[blockIdx.x + (i + 1) * G];
          c_next = p.chunks[sl_next.chunk];
        }
        // stage hs held slice i - NH, flushed one iteration ago: its store must
        // have read the stage before new bytes land there
        if (i >= NH) bulk_wait_read_all();
        if (i >= (uint32_t)CNI) mbar_wait_backoff(&hd.emptyI[t], ((i / CNI) - 1) & 1, 128, 0x1100000u | i);
        CDesc d;
        d.off = c.off;
        d.pay = c.pay;
        d.recv = c.recv;
        d.etl = c.etl;
        d.start = sl.start;
        d.len = sl.len;
        d.L = c.len;
        d.id = c.id;
        d.nslices = sl.nslices;
        d.sidx = sl.sidx;
        d.unit = sl.unit;
        d.unit_first = sl.unit_first;
        d.pofs = 0;
        d.staged = 0;
        d.owner = c.owner;
        d.gsl = blockIdx.x + i * G;
        if (SPARSE && sl.nslices) {
          d.sp_u = p.sp_chunk2u[sl.chunk];
          d.sp_g = p.sp_guess[d.sp_u];
          d.sp_cs = (p.sp_cand_off[d.sp_u + 1] - p.sp_cand_off[d.sp_u]) / sl.nslices;   // per-slice sub-list
        }
        const uint32_t nvb = (sl.len & ~3u) * 4u;
        const bool comp = sl.nslices > 0;
        uint32_t tx = 0;
        uint64_t a0 = 0, a1 = 0;
        if (!SERVER) {
          tx = (p.use_ef && comp) ? 2 * nvb : nvb;
        } else if (comp && SPARSE) {
          tx = nvb;         // Delta (e~ + the applied entries, or the scratch) lands in the held stage
        } else if (comp) {
          const uint64_t s0 = 4 + (uint64_t)sl.start * b / 8;
          const uint64_t e0 = 4 + ((uint64_t)(sl.start + sl.len) * b + 7) / 8;
          a0 = s0 & ~15ull;
          a1 = (e0 + 15) & ~15ull;
          d.pofs = (uint32_t)(s0 - a0);
          d.staged = p.stage_payload;
          if (p.use_ef) tx += nvb;   // e~ lands in the held stage; Delta is formed in place
          if (d.staged) tx += p.n * (uint32_t)(a1 - a0);
          tx += 16 * p.n;   // each rank's payload head (scale / norm) by bulk copy
        } else {
          tx = nvb;         // raw unit: rank 0's fp32 values land in the held stage
        }
        hd.desc[hs] = d;
        mbar_arrive_expect_tx(&hd.fullI[t], tx);
        if (!SERVER) {
          if (nvb) {
            tma_load_1d(H(hs), p.grad + c.off + sl.start, nvb, &hd.fullI[t]);
            if (p.use_ef && comp) tma_load_1d(IE(t), p.err + c.off + sl.start, nvb, &hd.fullI[t]);
          }
        } else if (!comp) {
          if (nvb) tma_load_1d(H(hs), p.recv + c.recv + 4ull * sl.start, nvb, &hd.fullI[t]);
        } else if (SPARSE) {
          if (nvb) tma_load_1d(H(hs), p.err + c.etl + sl.start, nvb, &hd.fullI[t]);
        } else {
          if (p.use_ef && nvb) tma_load_1d(H(hs), p.err + c.etl + sl.start, nvb, &hd.fullI[t]);
          for (uint32_t r = 0; r < p.n; r++)
            tma_load_1d(IH(t) + 16 * r, p.recv + r * p.slot_bytes + c.recv, 16, &hd.fullI[t]);
          if (d.staged)
            for (uint32_t r = 0; r < p.n; r++)
              tma_load_1d(I(t) + r * p.piece_stride, p.recv + r * p.slot_bytes + c.recv + a0,
                          (uint32_t)(a1 - a0), &hd.fullI[t]);
        }
        // flush the slice whose stage the next iteration reuses (store issued now,
        // its smem read waited for only then)
        if (i + 1 >= NH && i + 1 < mine) flush(i + 1 - NH);
      }
      for (uint32_t ie = mine > NH ? mine - NH : 0; ie < mine; ie++) flush(ie);
      bulk_wait_all();
      if (FUSED && p.pass != 1) {   // raw payloads stored into peers' RECV: visible before the signal
        __threadfence_system();
        mbar_arrive1(&hd.pfin);
      }
    }
    return;
  }

  // ===================================================== reducers
  if (warp >= CRED) {
    if (SPARSE) return;   // no unit norm: the emit does not wait for a total
    // the emit's scalars from the unit total, once per slice (not per lane):
    // scaled sign s = fl32(||q||_1 / L); dithering N = fl32(sqrt(||q||^2))
    // (R12), s_l / N and N / s_l with IEEE divisions
    const float rslv = (float)((1u << ((BITS ? BITS : (int)p.bits) - 1)) - 1u);
    auto publish = [&](uint32_t hs, double total) {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      if (KIND == C_SIGN) {
        r.x = __double2float_rn(total / (double)hd.desc[hs].L);
      } else if (KIND == C_LDITHER || KIND == C_NDITHER) {
        const float N = __double2float_rn(sqrt(total));
        r = make_float4(N, N != 0.f ? fdiv(rslv, N) : 0.f, fdiv(N, rslv), 0.f);
      }
      hd.dv[hs] = r;
    };
    for (uint32_t i = warp - CRED; i < mine; i += CRW) {
      const uint32_t hs = i % NH;
      // slice i produced.  Cannot alias: slice i + NH needs stage hs back, which
      // needs this reducer's tready arrive for slice i first.
      // the emit of slice i runs D slices later; a slept poll (200 ns) keeps the
      // waiting warps off the issue slots the consumers need.  A 1 us poll
      // delayed the unit totals: onebit server +2.5 % (C2), +2 % (C5)
      mbar_wait_backoff(&hd.pready[hs], (i / NH) & 1, BPC_RED_POLL_NS, 0x2000000u | i);
      const uint32_t ns = SPARSE ? 0u : hd.desc[hs].nslices;   // sparse kinds: no unit norm
      if (ns > 0) {   // the slice partial: pairwise tree over the 16 consumer warps' subtrees
        double r = lane < CCW ? hd.red[i % CRED_R][lane] : 0.0;
#pragma unroll
        for (int m = 1; m < CCW; m <<= 1) r = r + __shfl_xor_sync(0xffffffffu, r, m);
        if (lane == 0) hd.part[hs] = r;
        __syncwarp();
      }
      if (ns > 1 && p.pass == 1) {   // per-tensor units, pass 1: publish the partial only
        if (lane == 0) p.partials[hd.desc[hs].unit_first + hd.desc[hs].sidx] = hd.part[hs];
      } else if (ns > 1 && p.pass == 2) {   // pass 2: the unit's total from unit_tree_kernel
        if (lane == 0) publish(hs, __ldcg(p.unit_total + hd.desc[hs].unit));
      } else if (ns > 1) {
        if (lane == 0) {
          // publish this slice's partial, then wait for the unit's other slices
          const CDesc& d = hd.desc[hs];
          p.partials[d.unit_first + d.sidx] = hd.part[hs];
          red_release_add(p.counters + d.unit, 1ull);
          wait_counter(p.counters + d.unit, (unsigned long long)ep.E * ns, 0x3000000u | i);
        }
        __syncwarp();
        // unit total: pairwise tree over its slices, zero-padded to CUNITSL (R6)
        const double* P = p.partials + hd.desc[hs].unit_first;
        double v;
        if (CUNITSL == 64) {   // lane l holds the 2-slice subtree (2l, 2l+1)
          const uint32_t l0 = 2 * lane, l1 = 2 * lane + 1;
          v = (l0 < ns ? __ldcg(P + l0) : 0.0) + (l1 < ns ? __ldcg(P + l1) : 0.0);
        } else {
          v = (uint32_t)lane < ns ? __ldcg(P + lane) : 0.0;
        }
        v = warp_tree(v);
        if (lane == 0) publish(hs, v);
      } else if (ns == 1 && lane == 0) {
        publish(hs, hd.part[hs]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&hd.tready[hs]);
    }
    return;
  }

  // ===================================================== consumers
  const float slv = (float)((1u << (b - 1)) - 1u);
  const int cmax = (1 << (b - 1)) - 1;
  const float lmin = __uint_as_float((uint32_t)(127 - (cmax - 1)) << 23);
  const uint32_t cmask = (1u << b) - 1u;
  const uint32_t gbits = 4u * (uint32_t)b;                  // bits of one float4 group's codes
  const uint32_t gmask = gbits == 32 ? 0xFFFFFFFFu : (1u << gbits) - 1u;
  const uint32_t stage_id = SERVER ? 1u : 0u;
  const uint32_t rng_rank = SERVER ? 0u : p.rank;
  const uint32_t rot = ((uint32_t)lane >> 1) & 3u;         // conflict-free group order (header)
  const uint32_t lf = 128u * warp + 4u * lane;              // the lane's first float4 in a slice
  const uint32_t lq = 32u * warp + lane;                    // lane index within the slice
  const uint32_t lbit = 16u * (uint32_t)b * lq;             // first bit of the lane's field in the slice stream
  bool bad = false;

  // the lane's 16 b-bit field of a payload stream whose slice starts at `words`
  // (32-bit aligned); words at index >= sw are not read (they are not payload)
  auto load_lane_field = [&](const uint32_t* words, uint32_t sw) -> U128 {
    const uint32_t w0 = lbit >> 5;
    uint32_t wv[4];
#pragma unroll
    for (int c = 0; c < 4; c++) wv[c] = (w0 + c < sw) ? words[w0 + c] : 0u;
    U128 a{(uint64_t)wv[0] | ((uint64_t)wv[1] << 32), (uint64_t)wv[2] | ((uint64_t)wv[3] << 32)};
    return u128_shr(a, lbit & 31u);
  };

  // A slice is FULL when it holds CSL elements of its unit: no bounds checks, no
  // tail loads (the ragged-tail code runs only for a unit's last slice).
  // ---------------- produce: q (worker) / Delta (server) of a slice + its warp subtrees
  auto produce = [&](auto full_tag, uint32_t i, uint32_t t, const CDesc& d, float4* val, bool comp) {
    constexpr bool FULL = decltype(full_tag)::value;
    const uint32_t nvec = d.len >> 2;
    const uint32_t sw = (uint32_t)(((uint64_t)d.len * b + 31) / 32);   // payload words of the slice
    const bool lane_any = FULL || 16u * lq < d.len;
    double lv[4];
    // server, n = 1: rank 0's field of the lane (sign: one half-word), read once
    U128 fld{0, 0};
    float h0 = 0.f;
    if (N1 && comp && lane_any) {
      h0 = *reinterpret_cast<const float*>(IH(t));
      const uint32_t* words = d.staged ? reinterpret_cast<const uint32_t*>(I(t) + d.pofs)
                                       : reinterpret_cast<const uint32_t*>(p.recv + d.recv + 4 +
                                                                           (uint64_t)d.start * b / 8);
      if (KIND == C_SIGN) fld.lo = reinterpret_cast<const uint16_t*>(words)[lq];
      else fld = rotate_field(load_lane_field(words, sw), rot, gbits);   // step s's group at bit 4 b s
    }
    const float unit0 = KIND == C_SIGN ? 0.f : fdiv(h0, slv);
#pragma unroll
    for (int s = 0; s < 4; s++) {
      const uint32_t k = (s + rot) & 3u;
      const uint32_t f = lf + k;
      const uint32_t j = d.start + 4 * f;
      const bool inv4 = FULL || f < nvec;   // a whole float4 inside the 16-byte bulk copies
      const bool any = FULL || 4 * f < d.len;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      bool wr = false;
      if (!SERVER) {
        const bool ef = p.use_ef && comp;
        float4 g4 = q, e4 = q;
        if (inv4) {
          g4 = val[f];
          if (ef) e4 = IE(t)[f];
        } else if (any) {   // ragged tail (not in the 16-byte bulk copy)
          g4 = load4_masked(p.grad + d.off, j, d.L);
          if (ef) e4 = load4_masked(p.err + d.off, j, d.L);
          wr = true;
        }
        if (p.check_finite) bad |= !(isfinite(g4.x) && isfinite(g4.y) && isfinite(g4.z) && isfinite(g4.w));
        if (ef) {
          q = fadd4(g4, e4);
          wr = any;
        } else {
          q = g4;
        }
      } else if (SPARSE && comp && any) {
        // Delta as sparse_apply left it (e~ + the ranks' entries; Delta = fl32(0 + e~)
        // = e~ elsewhere: e~ never holds -0, bpc_load_state stores -0 as +0)
        q = inv4 ? val[f] : load4_masked(p.err + d.etl, j, d.L);
        wr = !inv4;
      } else if (any) {
        wr = true;
        if (!comp) {   // raw unit: mean of the ranks' fp32 values (rank 0's staged in val)
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          for (uint32_t r = 0; r < (N1 ? 1u : p.n); r++) {
            const float4 x4 = (r == 0 && inv4)
                                  ? val[f]
                                  : load4_masked(reinterpret_cast<const float*>(p.recv + r * p.slot_bytes + d.recv), j, d.L);
            acc[0] += (double)x4.x;
            acc[1] += (double)x4.y;
            acc[2] += (double)x4.z;
            acc[3] += (double)x4.w;
          }
          if (FULL || j < d.L) q.x = mean_plus(acc[0], p.inv_n, 0.0);
          if (FULL || j + 1 < d.L) q.y = mean_plus(acc[1], p.inv_n, 0.0);
          if (FULL || j + 2 < d.L) q.z = mean_plus(acc[2], p.inv_n, 0.0);
          if (FULL || j + 3 < d.L) q.w = mean_plus(acc[3], p.inv_n, 0.0);
        } else if (N1) {
          // n = 1: Delta = fl32(fl64(dec * 1.0) + fl64(e~)) equals the fp32 sum
          // fl32(dec + e~): the fp64 sum of two fp32 values is exact unless their
          // exponents differ by more than 29, and then both roundings return the
          // larger operand.  One fp32 add instead of four conversions.
          float4 e4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p.use_ef) e4 = inv4 ? val[f] : load4_masked(p.err + d.etl, j, d.L);
          float4 dec;
          if (KIND == C_SIGN) {
            // sign: h >= +0, and for h = 0 both decodes are +0 (the fp64 sum of the
            // oracle starts at +0, so -0 never survives): one add per element
            const float hneg = h0 == 0.f ? 0.f : -h0;
            const uint32_t nib = (uint32_t)(fld.lo >> (4 * k)) & 15u;
            dec = make_float4(nib & 1u ? h0 : hneg, nib & 2u ? h0 : hneg, nib & 4u ? h0 : hneg,
                              nib & 8u ? h0 : hneg);
          } else {
            const uint32_t x = u128_get(fld, gbits * s) & gmask;
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const uint32_t code = (x >> (b * u)) & cmask;
              const float mag = dither_mag<KIND>(code, h0, unit0, cmax);
              set(dec, u, (code & 1u) ? mag : -mag);
            }
            // acc = +0.0 + dec (turns -0 into +0, as the fp64 sum does), then + e~
            dec = fadd4(make_float4(0.f, 0.f, 0.f, 0.f), dec);
          }
          const float4 dsum = fadd4(dec, e4);
          q = FULL ? dsum : make_float4(j < d.L ? dsum.x : 0.f, j + 1 < d.L ? dsum.y : 0.f,
                                        j + 2 < d.L ? dsum.z : 0.f, j + 3 < d.L ? dsum.w : 0.f);
        } else {
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          for (uint32_t r = 0; r < p.n; r++) {
            const float h = *reinterpret_cast<const float*>(IH(t) + 16 * r);
            const uint32_t* words =
                d.staged ? reinterpret_cast<const uint32_t*>(I(t) + r * p.piece_stride + d.pofs)
                         : reinterpret_cast<const uint32_t*>(p.recv + r * p.slot_bytes + d.recv + 4 +
                                                             (uint64_t)d.start * b / 8);
            // this group's 4 codes: bits [lbit + 4 b k, + 4 b) of the slice stream
            const uint32_t pos = lbit + gbits * k;
            const uint32_t w0 = pos >> 5;
            const uint32_t lo = words[w0];
            const uint32_t hi = (w0 + 1 < sw) ? words[w0 + 1] : 0u;
            const uint32_t x = (uint32_t)((((uint64_t)hi << 32) | lo) >> (pos & 31)) & gmask;
            const float unit = KIND == C_SIGN ? 0.f : fdiv(h, slv);
            const double hd64 = (double)h;   // sign: one conversion per rank, not per element
#pragma unroll
            for (int u = 0; u < 4; u++) {
              double dec;
              if (KIND == C_SIGN) {
                dec = ((x >> u) & 1u) ? hd64 : -hd64;
              } else {
                const uint32_t code = (x >> (b * u)) & cmask;
                const float mag = dither_mag<KIND>(code, h, unit, cmax);
                dec = (double)((code & 1u) ? mag : -mag);
              }
              if (FULL || j + u < d.L) acc[u] += dec;
            }
          }
          float4 e4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p.use_ef) e4 = inv4 ? val[f] : load4_masked(p.err + d.etl, j, d.L);
          if (FULL || j < d.L) q.x = mean_plus(acc[0], p.inv_n, (double)e4.x);
          if (FULL || j + 1 < d.L) q.y = mean_plus(acc[1], p.inv_n, (double)e4.y);
          if (FULL || j + 2 < d.L) q.z = mean_plus(acc[2], p.inv_n, (double)e4.z);
          if (FULL || j + 3 < d.L) q.w = mean_plus(acc[3], p.inv_n, (double)e4.w);
        }
      }
      if (wr) val[f] = q;
      lv[s] = (comp && !SPARSE) ? (KIND == C_SIGN ? leaf4_abs(q) : leaf4_sq(q)) : 0.0;
    }
    if (comp && !SPARSE) {
      // the lane's 16-element subtree: groups (0, 1) and (2, 3) pair up; in step
      // order that is (s0, s1), (s2, s3) for an even rotation and (s3, s0),
      // (s1, s2) for an odd one (IEEE + is commutative)
      const bool odd = rot & 1u;
      const double x1 = odd ? lv[3] : lv[1], y1 = odd ? lv[1] : lv[3];
      const double a = warp_tree((lv[0] + x1) + (lv[2] + y1));   // the warp's 512 elements
      // slot i % CRED_R is free: its previous slice i - CRED_R was emitted by this
      // warp (iteration i - 1 emitted slice i - 1 - D >= i - CRED_R, in order),
      // which waited for that slice's reducer
      if (lane == 0) hd.red[i % CRED_R][warp] = a;
    }
  };

  // ---------------- emit: payload (sign bits / codes) + error of a slice (into the
  // held stage; the producer bulk-stores it), raw units: ragged tail only
  auto emit = [&](auto full_tag, const CDesc& d, float4* val, uint8_t* pay, const float4 dv) {
    constexpr bool FULL = decltype(full_tag)::value;
    const bool MC = SERVER && FUSED && p.mc_out != nullptr;   // pay is in the multicast mapping
    const uint32_t L = d.L;
    const uint32_t nvec = d.len >> 2;
    if (d.nslices == 0) {   // raw unit: the producer bulk-stores [0, nvec); the ragged float4 here
      if (MC) {   // NVLS: the consumers store the whole raw payload through the multicast mapping
#pragma unroll
        for (int s = 0; s < 4; s++) {
          const uint32_t f = lf + ((s + rot) & 3u);
          if (FULL || 4 * f < d.len) mm_store4_masked(reinterpret_cast<float*>(pay), d.start + 4 * f, L, val[f]);
        }
      } else if (!FULL && (d.len & 3u)) {
#pragma unroll
        for (int s = 0; s < 4; s++) {
          const uint32_t f = lf + ((s + rot) & 3u);
          if (f == nvec) store4_masked(reinterpret_cast<float*>(pay), d.start + 4 * f, L, val[f]);
        }
      }
      return;
    }
    float* errp = p.use_ef ? (SERVER ? p.err + d.etl : p.err + d.off) : nullptr;
    if (SPARSE) {
      // the unit's candidates: key >= G_u (top-k |q| bits, R9; random-k the
      // complemented Philox word, R10), in index order into this slice's own
      // sub-list of the unit's list (lanes own contiguous elements: a scan of the
      // lanes' counts in lane order is the index order) + the slice's count.
      // q stays in the held stage: it is the worker's new e (bulk-stored)
      const uint32_t u = d.sp_u, G = d.sp_g;
      uint32_t mask = 0;   // bit 4 k + e: element 16 lq + 4 k + e of the slice
#pragma unroll
      for (int s = 0; s < 4; s++) {
        const uint32_t k = (s + rot) & 3u;
        const uint32_t f = lf + k;
        const uint32_t j = d.start + 4 * f;
        if (!(FULL || 4 * f < d.len)) continue;
        const float4 q = val[f];
        if (!SERVER && errp && !FULL && f >= (d.len >> 2)) store4_masked(errp, j, L, q);   // ragged: not bulk-stored
        uint4 key;
        if (KIND == C_TOPK) {
          key = make_uint4(__float_as_uint(q.x) & 0x7fffffffu, __float_as_uint(q.y) & 0x7fffffffu,
                           __float_as_uint(q.z) & 0x7fffffffu, __float_as_uint(q.w) & 0x7fffffffu);
        } else {
          const uint4 w = philox4x32_10_rk(make_uint4(j >> 2, d.id, ep.t, (stage_id << 31) | rng_rank), p.rk);
          key = make_uint4(~w.x, ~w.y, ~w.z, ~w.w);
        }
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const uint32_t ke = e == 0 ? key.x : e == 1 ? key.y : e == 2 ? key.z : key.w;
          if (ke >= G && (FULL || j + e < L)) mask |= 1u << (4 * k + e);
        }
      }
      const uint32_t cnt = __popc(mask);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t* wc = hd.wcnt + CCW * (d.gsl & 1);   // double-buffered: one barrier per slice
      if (lane == 31) wc[warp] = incl;
      cons_sync();
      uint32_t wi = lane < CCW ? wc[lane] : 0u;   // warps' counts: inclusive scan over 16 lanes
#pragma unroll
      for (int o = 1; o < CCW; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      const uint32_t wbefore = warp ? __shfl_sync(0xffffffffu, wi, warp - 1) : 0u;
      const uint32_t total = __shfl_sync(0xffffffffu, wi, CCW - 1);
      uint32_t before = incl - cnt + wbefore;
      // sub-list of slice sidx: cs entries at cand_off[u] + sidx cs
      const uint32_t cs = d.sp_cs;
      uint2* sub = p.sp_cand + p.sp_cand_off[u] + d.sidx * cs;
      const uint32_t j0 = d.start + 16 * lq;
      const float* vq = reinterpret_cast<const float*>(val + lf);   // the lane's 16 values, element order
      for (uint32_t m = mask; m; m &= m - 1) {
        // each entry carries its key, so the select never gathers the unit's values
        // (candidates are rare: the key is re-formed here, a Philox call for random-k)
        const uint32_t bpos = (uint32_t)(__ffs(m) - 1), j = j0 + bpos;
        uint32_t key;
        if (KIND == C_TOPK) {
          key = __float_as_uint(vq[bpos]) & 0x7fffffffu;
        } else {
          const uint4 w = philox4x32_10_rk(make_uint4(j >> 2, d.id, ep.t, (stage_id << 31) | rng_rank), p.rk);
          const uint32_t e = j & 3u;
          key = ~(e == 0 ? w.x : (e == 1 ? w.y : (e == 2 ? w.z : w.w)));
        }
        if (before < cs) sub[before] = make_uint2(j, key);
        before++;
      }
      if (threadIdx.x == 0) p.sp_scnt[d.gsl] = total;   // > cs: the list overflowed
    } else if (KIND == C_SIGN) {
      const float sc = dv.x;
      const float nsc = -sc;
      uint32_t m16 = 0;
#pragma unroll
      for (int s = 0; s < 4; s++) {
        const uint32_t k = (s + rot) & 3u;
        const uint32_t f = lf + k;
        const uint32_t j = d.start + 4 * f;
        if (!(FULL || 4 * f < d.len)) continue;
        const float4 q = val[f];
        uint32_t nib = 0;
        float4 m;
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const bool bit = !(get(q, u) < 0.f);
          if (bit && (FULL || j + u < L)) nib |= 1u << u;
          set(m, u, bit ? nsc : sc);   // e = q - dec: q - s or q + s
        }
        if (errp) {
          const float4 ev = fadd4(q, m);
          val[f] = ev;
          if (!FULL && f >= nvec) store4_masked(errp, j, L, ev);   // ragged float4 (not bulk-stored)
        }
        m16 |= nib << (4 * k);
      }
      // lane pairs (2m, 2m+1) hold the two halves of payload word m of the warp
      const uint32_t other = __shfl_xor_sync(0xffffffffu, m16, 1);
      const uint32_t wi = (d.start >> 5) + (lq >> 1);
      if (!(lane & 1) && (FULL || wi < (L + 31) / 32))
      {
        uint32_t* w = reinterpret_cast<uint32_t*>(pay + 4) + wi;
        if (MC) mm_st_u32(w, m16 | (other << 16));
        else *w = m16 | (other << 16);
      }
      if (d.sidx == 0 && threadIdx.x == 0) {
        if (MC) mm_st_f32(pay, sc);
        else *reinterpret_cast<float*>(pay) = sc;
      }
    } else if (KIND == C_LDITHER || KIND == C_NDITHER) {
      const float N = dv.x, inv = dv.y, unit = dv.z;
      U128 fld{0, 0};   // the lane's 16 codes in element order
#pragma unroll
      for (int s = 0; s < 4; s++) {
        const uint32_t k = (s + rot) & 3u;
        const uint32_t f = lf + k;
        const uint32_t j = d.start + 4 * f;
        if (!(FULL || 4 * f < d.len)) continue;
        const float4 q = val[f];
        const uint4 w4 = philox4x32_10_rk(make_uint4(j >> 2, d.id, ep.t, (stage_id << 31) | rng_rank), p.rk);
        uint32_t g = 0, codes[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const uint32_t w = u == 0 ? w4.x : (u == 1 ? w4.y : (u == 2 ? w4.z : w4.w));
          const float qu = get(q, u);
          codes[u] = KIND == C_LDITHER ? lin_code_c(qu, slv, inv, w) : nat_code_c(qu, N, cmax, lmin, w);
          if (FULL || j + u < L) g |= codes[u] << (b * u);   // code < 2^b
        }
        fld = u128_or_u(fld, g, gbits * s);
        if (errp) {   // EF runs only; no error arithmetic otherwise
          float4 m;
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const float mag = dither_mag<KIND>(codes[u], N, unit, cmax);
            set(m, u, (codes[u] & 1u) ? -mag : mag);   // e = q - dec
          }
          const float4 ev = fadd4(q, m);
          val[f] = ev;
          if (!FULL && f >= nvec) store4_masked(errp, j, L, ev);
        }
      }
      fld = unrotate_field(fld, rot, gbits);
      // store the lane's 16 b bits at bit lbit of the slice stream.  Odd b: lane
      // 2m+1 starts at bit 16 of the word lane 2m ends in; it hands its first 16
      // bits to lane 2m, which stores that shared word
      uint32_t* out = reinterpret_cast<uint32_t*>(pay + 4) + (uint32_t)((uint64_t)d.start * b / 32);
      const uint32_t nwu = (uint32_t)(((uint64_t)b * L + 31) / 32 - (uint64_t)d.start * b / 32);   // words left in the unit
      uint32_t w0 = lbit >> 5, nw = (uint32_t)b / 2;
      if (b & 1) {
        const uint32_t nb16 = __shfl_xor_sync(0xffffffffu, (uint32_t)fld.lo & 0xFFFFu, 1);
        if (lane & 1) {
          fld = u128_shr(fld, 16);
          w0 += 1;
        } else {
          u128_or(fld, nb16, 16u * b);
          nw += 1;
        }
      }
#pragma unroll
      for (uint32_t c = 0; c < 4; c++)
        if (c < nw && (FULL || w0 + c < nwu)) {
          if (MC) mm_st_u32(out + w0 + c, u128_get(fld, 32 * c));
          else out[w0 + c] = u128_get(fld, 32 * c);
        }
      if (d.sidx == 0 && threadIdx.x == 0) {
        if (MC) mm_st_f32(pay, N);
        else *reinterpret_cast<float*>(pay) = N;
      }
    }
  };

  // ring positions as running counters (no division by the run-time NH per slice):
  // produce slice i in held stage ph (phase bit phb), input stage pt (phase ptb);
  // emit slice i - D in held stage eh (phase ehb)
  uint32_t ph = 0, phb = 0, pt = 0, ptb = 0, eh = 0, ehb = 0;
  for (uint32_t i = 0; i < mine + D; i++) {
    // ---------------- produce slice i
    if (i < mine) {
      const uint32_t hs = ph, t = pt;
      mbar_wait(&hd.fullI[t], ptb, 0x4000000u | i);
      const CDesc d = hd.desc[hs];
      const bool comp = d.nslices > 0;
      if (d.len == CSL) produce(BoolC<true>{}, i, t, d, H(hs), comp);
      else produce(BoolC<false>{}, i, t, d, H(hs), comp);
      __syncwarp();
      if (lane == 0) mbar_arrive1(&hd.emptyI[t]);   // input stage consumed by this warp
      if (++pt == (uint32_t)CNI) {
        pt = 0;
        ptb ^= 1;
      }
      if (++ph == NH) {
        ph = 0;
        phb ^= 1;
      }
      // release: this warp's subtree (and q) to the slice's reducer, which forms the
      // slice partial; the consumer warps never wait for each other
      if (!SPARSE && lane == 0) mbar_arrive1(&hd.pready[hs]);
    }
    // ---------------- emit slice i - D
    if (i >= D) {
      const uint32_t ie = i - D;
      const uint32_t hs = eh;
      const CDesc d = hd.desc[hs];
      // payload destination: worker -> the owner's RECV slot (fused push) or SEND;
      // server -> the local P
      uint8_t* const pay = (!SERVER && FUSED) ? p.dst[d.owner] + d.recv
                           : (SERVER && FUSED && p.mc_out) ? p.mc_out + d.pay : p.out + d.pay;
      // every slice (raw included) waits for its reducer before the stage is
      // recycled: keeps each mbarrier at most one phase ahead of its waiters
      if (!SPARSE) mbar_wait(&hd.tready[hs], ehb, 0x5000000u | ie);
      const float4 dv = hd.dv[hs];
      if (p.pass == 1) {
        // per-tensor units, pass 1: nothing to emit (pass 2 re-produces the slice)
      } else if (d.len == CSL) {
        emit(BoolC<true>{}, d, H(hs), pay, dv);
      } else {
        emit(BoolC<false>{}, d, H(hs), pay, dv);
      }
      fence_proxy_async();   // this thread's smem writes before the producer's bulk store
      __syncwarp();
      if (lane == 0) mbar_arrive1(&hd.emptyH[hs]);   // this warp is done with held stage hs
      if (++eh == NH) {
        eh = 0;
        ehb ^= 1;
      }
    }
  }
  if (bad) atomicOr(p.flag, 1u);
  // fused exchange: this step's payload bytes are released to the peers by the
  // launch's last CTA; every launch stores its epoch there
  if (FUSED && p.pass != 1) {
    // NVLS: order this thread's multicast stores (another virtual alias of the
    // peers' P) before the release of the pull epoch
    if (SERVER && p.mc_out) asm volatile("fence.proxy.alias;" ::: "memory");
    __threadfence_system();
  }
  cons_sync();
  if (threadIdx.x == 0 && FUSED && p.pass != 1) mbar_wait(&hd.pfin, 0, 0x6000000u);   // the producer's raw stores landed
  launch_end(p.sync, ep, threadIdx.x == 0);
}

// ring geometry for a launch: input-stage size and layout, number of held stages
static void cstream_geometry(bool server, const StreamParams& p, uint32_t* sie, uint32_t* si, uint32_t* nh,
                             size_t* smem) {
  const uint32_t slice_bytes = CSL * 4;
  uint32_t pieces = 0, ebytes = 0;
  if (!server) {
    ebytes = p.use_ef ? slice_bytes : 0;                                              // e
  } else {
    pieces = p.stage_payload ? (uint32_t)((p.n * p.piece_stride + 127) / 128 * 128) : 0;   // payload pieces
    ebytes = 0;                                   // e~ (and raw rank-0 values) land in the held stage
  }
  const uint32_t heads = server ? (16 * p.n + 127) / 128 * 128 : 0;   // payload heads
  *sie = heads + pieces;
  *si = heads + pieces + ebytes;
  const size_t budget = 227 * 1024 - sizeof(CHead) - 1024;
  uint32_t n = (uint32_t)((budget - (size_t)CNI * (*si)) / slice_bytes);
  *nh = n > (uint32_t)CMAXH ? (uint32_t)CMAXH : n;
  *smem = sizeof(CHead) + (size_t)(*nh) * slice_bytes + (size_t)CNI * (*si);
}

template <bool SERVER>
static cudaError_t launch_cstream_t(int kind, StreamParams p, int grid, cudaStream_t st) {
  if (p.n_slices == 0) return cudaSuccess;
  size_t smem;
  cstream_geometry(SERVER, p, &p.stage_a, &p.stage_b, &p.nstages, &smem);
  for (int r = 0; r < 10; r++) {   // Philox4x32-10 key schedule of the seed (R13)
    p.rk[2 * r] = (uint32_t)p.seed + (uint32_t)r * 0x9E3779B9u;
    p.rk[2 * r + 1] = (uint32_t)(p.seed >> 32) + (uint32_t)r * 0xBB67AE85u;
  }
  if (p.nstages < 3) return cudaErrorInvalidConfiguration;   // deferral >= 1 needs 3 held stages
  {
    // D = NH - 2 <= CMAXD for the norm kinds (the emit waits for the unit total);
    // 1 for the sparse kinds, which wait for nothing (measured: C3 1.101 ms at
    // D = 1, 1.123 at D = 3); BPC_CSTREAM_DEFER overrides it for measurements
    uint32_t dmax = (kind == C_TOPK || kind == C_RANDK) ? 1u : (uint32_t)CMAXD;
    if (const char* e = getenv("BPC_CSTREAM_DEFER")) dmax = (uint32_t)atoi(e);
    if (dmax < 1) dmax = 1;
    if (dmax > (uint32_t)CMAXD) dmax = CMAXD;
    p.defer = std::min<uint32_t>(p.nstages - 2, dmax);
  }
  auto go = [&](auto fn) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<uint32_t>((uint32_t)grid, p.n_slices));
    cfg.blockDim = dim3(CSNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident: the unit waits need it
    a[0].val.cooperative = 1;
    a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // prologue overlaps the predecessor
    a[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, fn, p);
  };
  const bool fused = p.ndst > 0 || p.sync.wait_fam >= 0;
  const int x = fused ? 1 : (SERVER && p.n == 1 ? 2 : 0);
  auto pick = [&](auto k_tag, auto b_tag) -> cudaError_t {
    constexpr int K = decltype(k_tag)::value, B = decltype(b_tag)::value;
    if (x == 1) return go(cstream_kernel<K, SERVER, 1, B>);
    if (SERVER && x == 2) return go(cstream_kernel<K, SERVER, SERVER ? 2 : 0, B>);
    return go(cstream_kernel<K, SERVER, 0, B>);
  };
  auto dither = [&](auto kind_tag) -> cudaError_t {
    switch (p.bits) {
      case 3: return pick(kind_tag, std::integral_constant<int, 3>{});
      case 5: return pick(kind_tag, std::integral_constant<int, 5>{});
      case 7: return pick(kind_tag, std::integral_constant<int, 7>{});
    }
    return pick(kind_tag, std::integral_constant<int, 0>{});
  };
  switch (kind) {
    case C_NONE: return pick(std::integral_constant<int, C_NONE>{}, std::integral_constant<int, 0>{});
    case C_SIGN: return pick(std::integral_constant<int, C_SIGN>{}, std::integral_constant<int, 0>{});
    case C_TOPK:   // sparse: no fused exchange
      return x == 2 ? go(cstream_kernel<C_TOPK, SERVER, SERVER ? 2 : 0, 0>) : go(cstream_kernel<C_TOPK, SERVER, 0, 0>);
    case C_RANDK:
      return x == 2 ? go(cstream_kernel<C_RANDK, SERVER, SERVER ? 2 : 0, 0>) : go(cstream_kernel<C_RANDK, SERVER, 0, 0>);
    case C_LDITHER: return dither(std::integral_constant<int, C_LDITHER>{});
    case C_NDITHER: return dither(std::integral_constant<int, C_NDITHER>{});
  }
  return cudaErrorInvalidValue;
}

size_t cstream_smem() { return sizeof(CHead); }

// per-tensor units: one CTA per unit sums its slice partials in pairwise order
// over the slice count padded to a power of two (slices are 8192-aligned in the
// unit, so this is R6's tree of the padded unit)
__global__ void __launch_bounds__(1024) unit_tree_kernel(const __grid_constant__ UnitTreeParams p) {
  extern __shared__ double acc[];   // [UNIT_MAX_SLICES]
  const uint32_t u = blockIdx.x, first = p.first[u], T = p.ns[u];
  uint32_t P = 1;
  while (P < T) P <<= 1;
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) acc[i] = i < T ? p.part[first + i] : 0.0;
  __syncthreads();
  for (uint32_t st = 1; st < P; st <<= 1) {
    for (uint32_t i = threadIdx.x * 2 * st; i < P; i += blockDim.x * 2 * st) acc[i] = acc[i] + acc[i + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) p.total[u] = acc[0];
}

cudaError_t launch_unit_tree(const UnitTreeParams& p, cudaStream_t s) {
  if (p.nunits == 0) return cudaSuccess;
  const size_t smem = sizeof(double) * UNIT_MAX_SLICES;
  cudaError_t e = cudaFuncSetAttribute(unit_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  unit_tree_kernel<<<p.nunits, 1024, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_worker_stream(int kind, const StreamParams& p, int grid, cudaStream_t st) {
  return launch_cstream_t<false>(kind, p, grid, st);
}
cudaError_t launch_server_stream(int kind, const StreamParams& p, int grid, cudaStream_t st) {
  return launch_cstream_t<true>(kind, p, grid, st);
}

}  // namespace bpc
