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
//   INPUT ring (NI x SI)     e (worker) or e~ and the n ranks' payload bytes
//                            (server), released as soon as the slice is produced.
// Warps:
//   PRODUCER   reads the slice descriptors and issues the 1-D bulk copies
//              (cp.async.bulk -> UBLKCP, one mbarrier complete_tx per slice);
//   4 REDUCERS (slice i -> reducer i % 4) complete each unit's fp64 pairwise-tree
//              total (R6): a multi-slice unit publishes one partial per
//              slice (release add on a per-unit counter) and each slice's reducer
//              waits (relaxed spin + one acquire) for the unit, then reduces it;
//   16 CONSUMERS produce slice i (q or Delta, slice partial) and then emit slice
//              i - D (codes + error) once its total is ready, D = NH - 2 <= 3, so
//              the cross-CTA wait overlaps the produce of D later slices.
// All CTAs are co-resident (cooperative launch) and every slice's partial is
// published before its CTA waits on an earlier unit, so the waits cannot
// deadlock.  Each mbarrier has a single in-order waiter group; the reducers,
// run out of order (slice i -> reducer i % 4) but each waits on its slice's
// held-stage barrier, which cannot run a phase ahead of it.
#include "device.cuh"

namespace bpc {

enum { C_NONE = 0, C_SIGN = 2, C_LDITHER = 5, C_NDITHER = 6 };

constexpr int CCW = 16;                  // consumer warps
constexpr int CCNT = 32 * CCW;           // consumer threads
constexpr int CPROD = CCW;               // producer warp index
constexpr int CRED = CCW + 1;            // first reducer warp index
constexpr int CRW = 4;                   // reducer warps (slice i -> reducer i % CRW)
constexpr int CSNT = CCNT + 32 + 32 * CRW;   // + producer + reducers
constexpr int CMAXH = 8;                 // max held stages
constexpr int CNI = 2;                   // input stages
constexpr int CMAXD = 3;                 // max emit deferral
constexpr int CSL = 8192;                // elements per slice
constexpr int CK = CSL / 4 / CCNT;       // float4 per consumer thread per slice
constexpr int CNRED = CK * CCW;          // 128-element warp subtrees per slice (64)
constexpr int CUNITSL = (1 << 18) / CSL; // max slices per unit (32)
static_assert(CNRED == 32 || CNRED == 64, "slice tree expects 32 or 64 warp subtrees");

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
};

struct __align__(128) CHead {
  uint64_t fullI[CNI], emptyI[CNI], emptyH[CMAXH], tready[CMAXH];
  uint64_t pready[CMAXH];   // slice in held stage s produced (its reducer waits on it)
  CDesc desc[CMAXH];
  double red[2][CNRED];
  double part[CMAXH];
  double total[CMAXH];
};

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(CCNT) : "memory");
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
    const float r = fminf(fdiv(fabsf(q), N), 1.0f);
    const float u = (float)(w >> 8) * 0x1p-24f;
    if (r >= lmin) {
      const int eb = (int)(__float_as_uint(r) >> 23);
      const float lo = __uint_as_float((uint32_t)eb << 23);
      const float pup = fsub(fdiv(r, lo), 1.0f);
      const int e_lev = (u < pup) ? eb - 127 + 1 : eb - 127;
      code = (uint32_t)(cmax + e_lev);
    } else {
      code = (u < fdiv(r, lmin)) ? 1u : 0u;
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
template <int KIND, bool SERVER, bool FUSED>
__global__ void __launch_bounds__(CSNT, 1) cstream_kernel(const __grid_constant__ StreamParams p) {
  extern __shared__ __align__(128) unsigned char sraw[];
  CHead& hd = *reinterpret_cast<CHead*>(sraw);
  const uint32_t NH = p.nstages;          // held stages
  const uint32_t D = NH - 2 < (uint32_t)CMAXD ? NH - 2 : (uint32_t)CMAXD;   // emit deferral
  const uint32_t SI = p.stage_b;          // bytes per input stage
  const uint32_t SIE = p.stage_a;         // byte offset of the e / e~ region inside an input stage
  unsigned char* held = sraw + sizeof(CHead);
  unsigned char* input = held + (size_t)NH * CSL * 4;
  auto H = [&](uint32_t s) { return reinterpret_cast<float4*>(held + (size_t)s * CSL * 4); };
  // server input stage: [n x 16-byte payload heads][n payload pieces][e~]
  const uint32_t HB = SERVER ? (16 * p.n + 127) / 128 * 128 : 0;
  auto IH = [&](uint32_t t) { return input + (size_t)t * SI; };               // payload heads
  auto I = [&](uint32_t t) { return input + (size_t)t * SI + HB; };          // payload pieces
  auto IE = [&](uint32_t t) { return reinterpret_cast<float4*>(input + (size_t)t * SI + SIE); };
  const uint32_t G = gridDim.x;
  const uint32_t mine = p.n_slices > blockIdx.x ? (p.n_slices - blockIdx.x + G - 1) / G : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = KIND == C_SIGN ? 1 : (int)p.bits;       // bits per element in the payload stream
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < NH; s++) {
      mbar_init(&hd.emptyH[s], CCW);
      mbar_init(&hd.tready[s], 1);
      mbar_init(&hd.pready[s], 1);
    }
    for (uint32_t t = 0; t < (uint32_t)CNI; t++) {
      mbar_init(&hd.fullI[t], 1);
      mbar_init(&hd.emptyI[t], CCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait_and_release();

  // ===================================================== producer
  if (warp == CPROD) {
    if (lane == 0) {
      if (SERVER && FUSED) peer_wait(p.sync);   // fused exchange: every rank's delta has landed in RECV
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
        if (i >= NH) mbar_wait(&hd.emptyH[hs], ((i / NH) - 1) & 1, 0x1000000u | i);
        if (i >= (uint32_t)CNI) mbar_wait(&hd.emptyI[t], ((i / CNI) - 1) & 1, 0x1100000u | i);
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
        const uint32_t nvb = (sl.len & ~3u) * 4u;
        const bool comp = sl.nslices > 0;
        uint32_t tx = 0;
        uint64_t a0 = 0, a1 = 0;
        if (!SERVER) {
          tx = (p.use_ef && comp) ? 2 * nvb : nvb;
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
        } else {
          if (p.use_ef && nvb) tma_load_1d(H(hs), p.err + c.etl + sl.start, nvb, &hd.fullI[t]);
          for (uint32_t r = 0; r < p.n; r++)
            tma_load_1d(IH(t) + 16 * r, p.recv + r * p.slot_bytes + c.recv, 16, &hd.fullI[t]);
          if (d.staged)
            for (uint32_t r = 0; r < p.n; r++)
              tma_load_1d(I(t) + r * p.piece_stride, p.recv + r * p.slot_bytes + c.recv + a0,
                          (uint32_t)(a1 - a0), &hd.fullI[t]);
        }
      }
    }
    return;
  }

  // ===================================================== reducers
  if (warp >= CRED) {
    for (uint32_t i = warp - CRED; i < mine; i += CRW) {
      const uint32_t hs = i % NH;
      // slice i produced.  Cannot alias: slice i + NH needs stage hs back, which
      // needs this reducer's tready arrive for slice i first.
      mbar_wait_backoff(&hd.pready[hs], (i / NH) & 1, 200, 0x2000000u | i);
      const uint32_t ns = hd.desc[hs].nslices;
      if (ns > 1 && p.pass == 1) {   // per-tensor units, pass 1: publish the partial only
        if (lane == 0) p.partials[hd.desc[hs].unit_first + hd.desc[hs].sidx] = hd.part[hs];
      } else if (ns > 1 && p.pass == 2) {   // pass 2: the unit's total from unit_tree_kernel
        if (lane == 0) hd.total[hs] = __ldcg(p.unit_total + hd.desc[hs].unit);
      } else if (ns > 1) {
        if (lane == 0) {
          // publish this slice's partial, then wait for the unit's other slices
          const CDesc& d = hd.desc[hs];
          p.partials[d.unit_first + d.sidx] = hd.part[hs];
          red_release_add(p.counters + d.unit, 1ull);
          wait_counter(p.counters + d.unit, (unsigned long long)p.epoch * ns, 0x3000000u | i);
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
        if (lane == 0) hd.total[hs] = v;
      } else if (ns == 1 && lane == 0) {
        hd.total[hs] = hd.part[hs];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&hd.tready[hs]);
    }
    return;
  }

  // ===================================================== consumers
  const int nb = 4 * b;
  const float slv = (float)((1u << (p.bits - 1)) - 1u);
  const int cmax = (1 << (p.bits - 1)) - 1;
  const float lmin = __uint_as_float((uint32_t)(127 - (cmax - 1)) << 23);
  const uint32_t cmask = (1u << b) - 1u;
  const uint32_t stage_id = SERVER ? 1u : 0u;
  const uint32_t rng_rank = SERVER ? 0u : p.rank;
  bool bad = false;

  // A slice is FULL when it holds CSL elements of its unit: no bounds checks, no
  // tail loads (the ragged-tail code runs only for a unit's last slice).
  // ---------------- produce: q (worker) / Delta (server) of a slice + its warp subtrees
  auto produce = [&](auto full_tag, uint32_t i, uint32_t t, const CDesc& d, float4* val, bool comp) {
    constexpr bool FULL = decltype(full_tag)::value;
    const uint32_t nvec = d.len >> 2;
#pragma unroll
    for (int k = 0; k < CK; k++) {
      const uint32_t f = threadIdx.x + k * CCNT;
      const uint32_t j = d.start + 4 * f;
      const bool inv4 = FULL || f < nvec;   // a whole float4 inside the 16-byte bulk copies
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!SERVER) {
        const bool ef = p.use_ef && comp;
        float4 g4 = q, e4 = q;
        if (inv4) {
          g4 = val[f];
          if (ef) e4 = IE(t)[f];
        } else if (4 * f < d.len) {   // ragged tail (not in the 16-byte bulk copy)
          g4 = load4_masked(p.grad + d.off, j, d.L);
          if (ef) e4 = load4_masked(p.err + d.off, j, d.L);
        }
        if (p.check_finite) bad |= !(isfinite(g4.x) && isfinite(g4.y) && isfinite(g4.z) && isfinite(g4.w));
        q = ef ? make_float4(fadd(g4.x, e4.x), fadd(g4.y, e4.y), fadd(g4.z, e4.z), fadd(g4.w, e4.w)) : g4;
      } else if (FULL || 4 * f < d.len) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (!comp) {   // raw unit: mean of the ranks' fp32 values (rank 0's staged in val)
          for (uint32_t r = 0; r < p.n; r++) {
            const float4 x4 = (r == 0 && inv4)
                                  ? val[f]
                                  : load4_masked(reinterpret_cast<const float*>(p.recv + r * p.slot_bytes + d.recv), j, d.L);
            acc[0] += (double)x4.x;
            acc[1] += (double)x4.y;
            acc[2] += (double)x4.z;
            acc[3] += (double)x4.w;
          }
        } else if (p.n == 1) {
          // n = 1: Delta = fl32(fl64(dec * 1.0) + fl64(e~)) equals the fp32 sum
          // fl32(dec + e~): the fp64 sum of two fp32 values is exact unless their
          // exponents differ by more than 29, and then both roundings return the
          // larger operand.  One fp32 add instead of four conversions.
          const float h = *reinterpret_cast<const float*>(IH(t));
          // staged words are read with shared-memory loads (no generic pointer merge)
          uint32_t field;
          if (d.staged) {
            const uint32_t* words = reinterpret_cast<const uint32_t*>(I(t) + d.pofs);
            field = KIND == C_SIGN ? ((words[f >> 3] >> ((f & 7) * 4)) & 15u)
                                   : load_field(words, (uint64_t)b * 4 * f, nb);
          } else {
            const uint32_t* words =
                reinterpret_cast<const uint32_t*>(p.recv + d.recv + 4 + (uint64_t)d.start * b / 8);
            field = KIND == C_SIGN ? ((words[f >> 3] >> ((f & 7) * 4)) & 15u)
                                   : load_field(words, (uint64_t)b * 4 * f, nb);
          }
          const float unit = KIND == C_SIGN ? 0.f : fdiv(h, slv);
          // sign: h >= +0, and for h = 0 both decodes are +0 (the fp64 sum of the
          // oracle starts at +0, so -0 never survives): one add per element
          const float hneg = h == 0.f ? 0.f : -h;
          float4 e4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p.use_ef) e4 = inv4 ? val[f] : load4_masked(p.err + d.etl, j, d.L);
#pragma unroll
          for (int u = 0; u < 4; u++) {
            float dsum;
            if (KIND == C_SIGN) {
              dsum = fadd(((field >> u) & 1u) ? h : hneg, get(e4, u));
            } else {
              const uint32_t code = (field >> (b * u)) & cmask;
              const float mag = dither_mag<KIND>(code, h, unit, cmax);
              // acc = +0.0 + dec (turns -0 into +0, as the fp64 sum does), then + e~
              dsum = fadd(fadd(0.f, (code & 1u) ? mag : -mag), get(e4, u));
            }
            if (FULL || j + u < d.L) set(q, u, dsum);
          }
        } else {
          for (uint32_t r = 0; r < p.n; r++) {
            const float h = *reinterpret_cast<const float*>(IH(t) + 16 * r);
            const uint32_t* words =
                d.staged ? reinterpret_cast<const uint32_t*>(I(t) + r * p.piece_stride + d.pofs)
                         : reinterpret_cast<const uint32_t*>(p.recv + r * p.slot_bytes + d.recv + 4 +
                                                             (uint64_t)d.start * b / 8);
            const uint32_t field = KIND == C_SIGN ? ((words[f >> 3] >> ((f & 7) * 4)) & 15u)
                                                  : load_field(words, (uint64_t)b * 4 * f, nb);
            const float unit = KIND == C_SIGN ? 0.f : fdiv(h, slv);
            const double hd64 = (double)h;   // sign: one conversion per rank, not per element
#pragma unroll
            for (int u = 0; u < 4; u++) {
              double dec;
              if (KIND == C_SIGN) {
                dec = ((field >> u) & 1u) ? hd64 : -hd64;
              } else {
                const uint32_t code = (field >> (b * u)) & cmask;
                const float mag = dither_mag<KIND>(code, h, unit, cmax);
                dec = (double)((code & 1u) ? mag : -mag);
              }
              if (FULL || j + u < d.L) acc[u] += dec;
            }
          }
        }
        if (!comp || p.n != 1) {
          float4 e4 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (comp && p.use_ef) e4 = inv4 ? val[f] : load4_masked(p.err + d.etl, j, d.L);
          if (FULL || j < d.L) q.x = mean_plus(acc[0], p.inv_n, (double)e4.x);
          if (FULL || j + 1 < d.L) q.y = mean_plus(acc[1], p.inv_n, (double)e4.y);
          if (FULL || j + 2 < d.L) q.z = mean_plus(acc[2], p.inv_n, (double)e4.z);
          if (FULL || j + 3 < d.L) q.w = mean_plus(acc[3], p.inv_n, (double)e4.w);
        }
      }
      val[f] = q;
      if (comp) {
        const double a = warp_tree(KIND == C_SIGN ? leaf4_abs(q) : leaf4_sq(q));
        if (lane == 0) hd.red[i & 1][k * CCW + warp] = a;   // subtree of slice elements [128 m, 128 m + 128)
      }
    }
  };

  // ---------------- emit: payload (sign bits / codes / raw fp32) + error of a slice
  auto emit = [&](auto full_tag, const CDesc& d, const float4* val, uint8_t* pay, double total) {
    constexpr bool FULL = decltype(full_tag)::value;
    const uint32_t L = d.L;
    if (d.nslices == 0) {   // raw unit: fp32 payload (worker: g, no EF; server: the mean)
#pragma unroll
      for (int k = 0; k < CK; k++) {
        const uint32_t f = threadIdx.x + k * CCNT;
        if (FULL) st4(reinterpret_cast<float*>(pay) + d.start + 4 * f, val[f]);
        else if (4 * f < d.len) store4_masked(reinterpret_cast<float*>(pay), d.start + 4 * f, L, val[f]);
      }
      return;
    }
    float* errp = p.use_ef ? (SERVER ? p.err + d.etl : p.err + d.off) : nullptr;
    if (KIND == C_SIGN) {
      const float sc = __double2float_rn(total / (double)L);
#pragma unroll
      for (int k = 0; k < CK; k++) {
        const uint32_t f = threadIdx.x + k * CCNT;
        const uint32_t j = d.start + 4 * f;
        const float4 q = val[f];
        uint32_t nib = 0;
        float4 ev;
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const float qu = get(q, u);
          const bool bit = !(qu < 0.f);
          if (bit && (FULL || j + u < L)) nib |= 1u << u;
          set(ev, u, bit ? fsub(qu, sc) : fadd(qu, sc));
        }
        if (errp) {
          if (FULL) st4(errp + j, ev);
          else if (j < L) store4_masked(errp, j, L, ev);
        }
        uint32_t w = nib << (4 * (lane & 7));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((lane & 7) == 0 && (FULL || j < L)) reinterpret_cast<uint32_t*>(pay + 4)[j >> 5] = w;
      }
      if (d.sidx == 0 && threadIdx.x == 0) *reinterpret_cast<float*>(pay) = sc;
    } else if (KIND == C_LDITHER || KIND == C_NDITHER) {
      const float N = __double2float_rn(sqrt(total));
      const float inv = N != 0.f ? fdiv(slv, N) : 0.f;
      const float unit = fdiv(N, slv);
      const uint64_t nwords = ((uint64_t)b * L + 31) / 32;
#pragma unroll
      for (int k = 0; k < CK; k++) {
        const uint32_t f = threadIdx.x + k * CCNT;
        const uint32_t j = d.start + 4 * f;
        const float4 q = val[f];
        uint32_t field = 0;
        if (FULL || j < L) {
          const uint4 w4 = philox4x32_10_rk(make_uint4(j >> 2, d.id, p.t, (stage_id << 31) | rng_rank), p.rk);
          float4 ev;
          uint32_t codes[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const uint32_t w = u == 0 ? w4.x : (u == 1 ? w4.y : (u == 2 ? w4.z : w4.w));
            const float qu = get(q, u);
            const uint32_t code = KIND == C_LDITHER ? lin_code_c(qu, slv, inv, w)
                                                    : nat_code_c(qu, N, cmax, lmin, w);
            if (FULL || j + u < L) field |= (code & cmask) << (b * u);
            codes[u] = code;
          }
          if (errp) {   // e = q - dec (EF runs only); no error arithmetic otherwise
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const float mag = dither_mag<KIND>(codes[u], N, unit, cmax);
              set(ev, u, fsub(get(q, u), (codes[u] & 1u) ? mag : -mag));
            }
            if (FULL) st4(errp + j, ev);
            else store4_masked(errp, j, L, ev);
          }
        }
        const uint32_t wd = warp_pack(field, nb);
        const uint64_t wbase = (uint64_t)(d.start + 4 * (k * CCNT + 32 * warp)) / 32 * b;
        if (lane < nb && (FULL || wbase + lane < nwords)) reinterpret_cast<uint32_t*>(pay + 4)[wbase + lane] = wd;
      }
      if (d.sidx == 0 && threadIdx.x == 0) *reinterpret_cast<float*>(pay) = N;
    }
  };

  for (uint32_t i = 0; i < mine + D; i++) {
    // ---------------- produce slice i
    if (i < mine) {
      const uint32_t hs = i % NH, t = i % CNI;
      mbar_wait(&hd.fullI[t], (i / CNI) & 1, 0x4000000u | i);
      const CDesc d = hd.desc[hs];
      const bool comp = d.nslices > 0;
      if (d.len == CSL) produce(BoolC<true>{}, i, t, d, H(hs), comp);
      else produce(BoolC<false>{}, i, t, d, H(hs), comp);
      __syncwarp();
      if (lane == 0) mbar_arrive1(&hd.emptyI[t]);   // input stage consumed by this warp
      cons_sync();                                    // all q written, red complete
      if (warp == 0) {
        if (comp) {
          const double r = warp_tree(CNRED == 64 ? hd.red[i & 1][2 * lane] + hd.red[i & 1][2 * lane + 1]
                                                 : hd.red[i & 1][lane]);
          if (lane == 0) hd.part[hs] = r;   // the slice's reducer publishes it
        }
        if (lane == 0) mbar_arrive1(&hd.pready[hs]);   // release: q and part[hs] visible to the reducer
      }
    }
    // ---------------- emit slice i - D
    if (i >= D) {
      const uint32_t ie = i - D;
      const uint32_t hs = ie % NH;
      const CDesc d = hd.desc[hs];
      // payload destination: worker -> the owner's RECV slot (fused push) or SEND;
      // server -> the local P
      uint8_t* const pay = (!SERVER && FUSED) ? p.dst[d.owner] + d.recv : p.out + d.pay;
      // every slice (raw included) waits for its reducer before the stage is
      // recycled: keeps each mbarrier at most one phase ahead of its waiters
      mbar_wait(&hd.tready[hs], (ie / NH) & 1, 0x5000000u | ie);
      const double total = hd.total[hs];
      if (p.pass == 1) {
        // per-tensor units, pass 1: nothing to emit (pass 2 re-produces the slice)
      } else if (d.len == CSL) {
        emit(BoolC<true>{}, d, H(hs), pay, total);
      } else {
        emit(BoolC<false>{}, d, H(hs), pay, total);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&hd.emptyH[hs]);   // this warp is done with held stage hs
    }
  }
  if (bad) atomicOr(p.flag, 1u);
  if (FUSED && p.pass != 1) {   // fused exchange: release this step's payload bytes to the peers
    __threadfence_system();
    cons_sync();
    peer_signal(p.sync, threadIdx.x == 0);
  }
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
  const bool fused = p.ndst > 0 || p.sync.wflags != nullptr;
  switch (kind) {
    case C_NONE: return fused ? go(cstream_kernel<C_NONE, SERVER, true>) : go(cstream_kernel<C_NONE, SERVER, false>);
    case C_SIGN: return fused ? go(cstream_kernel<C_SIGN, SERVER, true>) : go(cstream_kernel<C_SIGN, SERVER, false>);
    case C_LDITHER:
      return fused ? go(cstream_kernel<C_LDITHER, SERVER, true>) : go(cstream_kernel<C_LDITHER, SERVER, false>);
    case C_NDITHER:
      return fused ? go(cstream_kernel<C_NDITHER, SERVER, true>) : go(cstream_kernel<C_NDITHER, SERVER, false>);
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
