// gcx_span_dev.cuh — device code of the span kernels (gcx_span.cu, gcx_span_pieces.cu):
// helpers, the element arithmetic, the K1 / K3 / fused-owner kernel templates.
#pragma once
// gcx_span.cu — K1 "span" kernel: single-vector quantize (codec::quantize,
// /root/reference/proj/src/codec.cpp:24-69) for buckets of 32, 64 and 128,
// the configuration of C1 and of every default plan (model.hpp default 4/128).
//
// Work decomposition: a WARP owns a tile of 4096 consecutive elements and a
// LANE owns a span (row) of 128 consecutive elements of it (one bucket of 128,
// two of 64, four of 32), so both passes of the reference algorithm are
// lane-local:
//   pass 1  the sequential FP64 sum of squares of each bucket (codec.cpp:41-48)
//           over the lane's row, in index order (RN(sq + v*v) == fma(v,v,sq):
//           the square of a float is exact in FP64);
//   pass 2  level + stochastic rounding + sign of every element
//           (codec.cpp:50-64) and LSB-first packing into (bits+1)-bit fields
//           (codec.cpp:97-124): a row is 4 whole 32-element groups and a group
//           owns exactly W = bits+1 whole 32-bit words, so the fields are
//           shifted into registers at compile-time positions.
//
// Data movement (Blackwell-native).  The tile is staged as 4 QUARTERS (element
// columns [32g, 32g+32) of all 32 rows); each quarter is ONE 2-D TMA tensor
// copy (box 32 x 32 floats, rows 512 B apart in HBM, UTMALDG) into a 4 KB
// shared slot with the 128-byte swizzle, so the lane-per-row LDS.128 reads of
// both passes are bank-conflict free.  Each warp cycles 5 slots: the slot of
// group g is refilled with the next quarter as soon as group g is quantized,
// so the next tile streams in one group ahead and pass 1 of a tile waits only
// on quarters issued a group earlier.  Completion is counted on one mbarrier
// per slot.  The packed words of a tile are written to a shared buffer and
// leave with one bulk store (cp.async.bulk global <- shared).  Key prefixes
// T(i) (gcx_make_prefix) use the span key layout (span_key_pos): per tile and
// group, 1024 high words ordered [quad][lane][4] then the 1024 low words, so
// each lane's next four keys are one coalesced 16-byte load per word half;
// they ride one group ahead in registers.
//
// Bit-exactness: the arithmetic is gcx_device.cuh's.  The
// FP32 -> FP64 conversion is cvt (exact for zeros and subnormals), so the fast
// path covers every finite input; a bucket holding a non-finite input (its
// FP64 sum is then non-finite) and a group with an ambiguous key compare
// (probability ~3 * 2^-32 per element) are recomputed by the exact
// per-element path (quantize_field on the full 64-bit key).  The ragged last
// tile is staged zero-filled (zeros add nothing to a norm and quantize to 0).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cmath>
#include <cstring>
#include <mutex>

#include "gcx.h"
#include "gcx_device.cuh"
#include "gcx_plan.cuh"

namespace gcx_span {

using namespace gcx_dev;
using gcx_plan::span_key_pos;
using gcx_plan::span_key_slot;

constexpr uint32_t kSpan = 128;          // elements per lane row
constexpr uint32_t kWTile = 32 * kSpan;  // elements per warp tile
constexpr uint32_t kSlots = 5;           // quarter slots per warp (4 KB each)
constexpr uint32_t kSlotFloats = 32 * 32;
#ifndef GCX_SPAN_WARPS
#define GCX_SPAN_WARPS 4
#endif
constexpr int kWarps = GCX_SPAN_WARPS;
#ifndef GCX_SMALL_TILES_PER_SM
#define GCX_SMALL_TILES_PER_SM 2  // tables of at most this many tiles per SM: CTA-per-tile kernels
#endif

// per-warp shared memory: kSlots swizzled quarter slots, the packed output
// words of one tile (128 groups x W words), kSlots mbarriers; 1 KB aligned
// (the 128-byte swizzle pattern repeats every 1024 bytes)
__host__ __device__ constexpr uint32_t out_words(uint32_t W) { return 128u * W; }
__host__ __device__ constexpr uint32_t warp_smem_bytes(uint32_t W) {
  return (kSlots * kSlotFloats * 4 + out_words(W) * 4 + kSlots * 8 + 1023) & ~1023u;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SPAN_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SPAN_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 2-D TMA tensor copy global -> shared (UTMALDG), completion on `bar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// bulk copy shared -> global (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__host__ __device__ __forceinline__ uint64_t mix64h(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Element e (0..31) of row r in a swizzled quarter slot: the 16-byte chunk
// e/4 of the row's 128 bytes sits at chunk (e/4) ^ (r % 8) (TMA SWIZZLE_128B).
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t e) {
  return r * 32u + ((((e >> 2) ^ (r & 7u)) << 2) | (e & 3u));
}

// a lane's row of the tile: its 4 quarter slots and the row index
struct RowView {
  const float* slot[4];
  uint32_t r;
  __device__ __forceinline__ float at(uint32_t e) const { return slot[e >> 5][swz(r, e & 31u)]; }
};

// One element of codec::quantize on the fast path (finite v in a bucket with
// a non-zero norm).  As quantize_field32 (gcx_device.cuh) with two changes:
//  * no clamp: norm >= |v| makes a <= 1 and x <= s, and x == s exactly gives
//    fl == 0, so the key never rounds past s;
//  * `h` is the key's top word BEFORE the final `z ^= z >> 31` of mix64
//    (util.hpp:18): the true top word K = h ^ (h >> 31) differs from h by at
//    most 1, so K < fl <=> h < fl whenever h is not within 1 of fl; those
//    elements (mn <= 2 after the group) take the exact path.
// The FP32 -> FP64 conversion is exact for zeros and subnormals: a zero gives
// x = 0, fl = 0, level 0, never rounded up; the sign is signbit(v) (-0.0 -> 1).
template <uint32_t BITS>
__device__ __forceinline__ uint32_t span_field(uint32_t u, double nd, double y, uint32_t h,
                                               uint32_t& mn) {
  constexpr double S2 = double((1u << BITS) - 1) * 4294967296.0;
  const double av = fabs(double(__uint_as_float(u)));
  const double q0 = __dmul_rn(av, y);
  const double r = __fma_rn(-nd, q0, av);
  const double a = __fma_rn(r, y, q0);
  const double X = __dmul_rn(a, S2);
  const double T = __dadd_rz(X, 4503599627370496.0);
  const uint32_t fl = uint32_t(__double2loint(T));
  const uint32_t lv = uint32_t(__double2hiint(T)) - 0x43300000u;
  mn = min(mn, h - fl + 1u);
  const uint32_t l = lv + (h < fl ? 1u : 0u);
  return l | ((u >> 31) << BITS);
}

// top word of mix64(seed ^ T) before the final xorshift (see span_field)
__device__ __forceinline__ uint32_t key_hraw_from_prefix(uint32_t lo, uint32_t hi, uint32_t s_lo,
                                                         uint32_t s_hi, const HashK& k) {
  lo ^= s_lo;
  hi ^= s_hi;
  asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(lo), "+r"(hi));
  xorshift_v<GCX_HASH_HV>(lo, hi, GCX_HASH_HV == 1 ? 30u : k.k30, k.m30);
  mul64c(lo, hi, 0x1ce4e5b9u, 0xbf58476du);
  xorshift_v<GCX_HASH_HV>(lo, hi, GCX_HASH_HV == 1 ? 27u : k.k27, k.m27);
  return __umulhi(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
}

__device__ __forceinline__ uint32_t key_hraw_inline(uint32_t i, uint32_t b, uint32_t s_lo,
                                                    uint32_t s_hi, const HashK& k) {
  uint32_t lo, hi;
  draw_prefix<GCX_HASH_HV>(i, b, k, lo, hi);
  return key_hraw_from_prefix(lo, hi, s_lo, s_hi, k);
}

template <uint32_t W>
__device__ __forceinline__ void put_field(uint32_t (&w)[W], uint32_t j, uint32_t f) {
  const uint32_t bit = j * W, m = bit >> 5, sh = bit & 31u;
  w[m] |= f << sh;
  if (sh + W > 32) w[m + 1] |= f >> (32 - sh);
}

// exact per-element path for group g of a lane's row (any inputs); writes the
// group's W words to w.  Keys: prefix table words of the tile (hi at
// ph[quad*128 + lane*4 + k], lo 4096 words later) or inline hashing.
// key sources of the span K1 kernels
constexpr int kKmInline = 0;  // three SplitMix64 finalizers per element
constexpr int kKmTable = 1;   // full keys from a per-step table (gcx_make_keys*), span layout
constexpr int kKmPrefix = 2;  // seed-independent prefixes T(i), span layout: one finalizer

template <uint32_t BITS, int LGB, int KM>
__device__ __noinline__ void span_group_exact(RowView rv, uint32_t g, uint32_t i0, uint32_t nu,
                                              uint64_t seed, const uint32_t* ph, uint32_t lane,
                                              uint32_t* w) {
  constexpr uint32_t W = BITS + 1, S = (1u << BITS) - 1;
  uint32_t acc[W];
  for (uint32_t m = 0; m < W; ++m) acc[m] = 0u;
  if (nu != 0u) {  // all-zero bucket: every field 0, sign too (codec.cpp:50)
    const Opq opq = make_opq();
    const double nd = f32abs_to_f64(nu);
    const double y = __drcp_rn(nd);
    for (uint32_t j = 0; j < 32; ++j) {
      uint32_t hl, hh;
      if (KM != kKmInline) {  // ph: the tile's first key word (span_key_pos)
        const uint32_t pos = g * 2048u + (j >> 2) * 128u + lane * 4u + (j & 3u);
        if (KM == kKmTable) {
          hh = ph[pos];
          hl = ph[pos + 1024];
        } else {
          const uint64_t z = (uint64_t(ph[pos]) << 32 | ph[pos + 1024]) ^ seed;
          const uint64_t h = mix64h(z);
          hl = uint32_t(h);
          hh = uint32_t(h >> 32);
        }
      } else {
        const uint32_t i = i0 + j;
        draw_key(i, 0u, i >> LGB, 0u, uint32_t(seed), uint32_t(seed >> 32), opq, hl, hh);
      }
      const uint32_t f = quantize_field(__float_as_uint(rv.at(g * 32 + j)), nd, y, double(S), S,
                                        int(BITS), hl, hh);
      const uint32_t bit = j * W, m = bit >> 5, sh = bit & 31u;
      acc[m] |= f << sh;
      if (sh + W > 32) acc[m + 1] |= f >> (32 - sh);
    }
  }
  for (uint32_t m = 0; m < W; ++m) w[m] = acc[m];
}

// exact sequential norm of elements [e0, e0+cnt) of a row (any inputs) +
// first non-finite index (codec.cpp:41-48, :43-45)
static __device__ __noinline__ uint32_t span_norm_exact(RowView rv, uint32_t e0, uint32_t cnt, uint32_t i0,
                                                 unsigned long long* bad) {
  double sq = 0.0;
  uint32_t first_bad = ~0u;
  for (uint32_t j = 0; j < cnt; ++j) {
    const uint32_t ua = __float_as_uint(rv.at(e0 + j)) & 0x7FFFFFFFu;
    if (ua >= 0x7F800000u && first_bad == ~0u) first_bad = j;
    const double d = f32abs_to_f64_nb(ua);
    sq = __fma_rn(d, d, sq);
  }
  if (first_bad != ~0u && bad != nullptr) atomicMin(bad, (unsigned long long)(i0 + first_bad));
  return __float_as_uint(__double2float_rn(__dsqrt_rn(sq)));
}

// Pass 1 for buckets of 2^LGB > 128 elements (RPB = 2^(LGB-7) consecutive
// rows per bucket): the bucket's first lane runs the reference's sequential
// FP64 chain over its RPB rows (codec.cpp:41-48) and every lane gets its
// row's bucket norm by shuffle.  first_bad (lead lanes): the bucket-relative
// index of the first non-finite input, or ~0.
template <int LGB>
__device__ __forceinline__ void span_pass1_big(const RowView& rv, uint32_t lane, uint32_t& nu,
                                               bool& careful, uint32_t& first_bad) {
  constexpr uint32_t RPB = 1u << (LGB - 7);
  const bool lead = (lane & (RPB - 1u)) == 0;
  double sq = 0.0;
  first_bad = ~0u;
  if (lead) {
#pragma unroll 1
    for (uint32_t k = 0; k < RPB; ++k) {
      const uint32_t row = lane + k;
#pragma unroll
      for (uint32_t g = 0; g < 4; ++g) {
        const float* rp = rv.slot[g] + row * 32u;
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(rp + ((q ^ (row & 7u)) << 2));
          double d = double(v.x);
          sq = __fma_rn(d, d, sq);
          d = double(v.y);
          sq = __fma_rn(d, d, sq);
          d = double(v.z);
          sq = __fma_rn(d, d, sq);
          d = double(v.w);
          sq = __fma_rn(d, d, sq);
        }
      }
    }
  }
  const bool c = lead && (uint32_t(__double2hiint(sq)) & 0x7FF00000u) == 0x7FF00000u;
  uint32_t v = 0u;
  if (lead) {
    if (c) {  // exact sums and the first non-finite input, row by row
      double sx = 0.0;
      for (uint32_t k = 0; k < RPB; ++k) {
        RowView rk = rv;
        rk.r = lane + k;
        for (uint32_t e = 0; e < kSpan; ++e) {
          const uint32_t ua = __float_as_uint(rk.at(e)) & 0x7FFFFFFFu;
          if (ua >= 0x7F800000u && first_bad == ~0u) first_bad = k * kSpan + e;
          const double d = f32abs_to_f64_nb(ua);
          sx = __fma_rn(d, d, sx);
        }
      }
      v = __float_as_uint(__double2float_rn(__dsqrt_rn(sx)));
    } else {
      v = __float_as_uint(__double2float_rn(__dsqrt_rn(sq)));
    }
  }
  const uint32_t src = lane & ~(RPB - 1u);
  nu = __shfl_sync(0xffffffffu, v, src);
  careful = __shfl_sync(0xffffffffu, c ? 1u : 0u, src) != 0u;
}

struct SpanArgs {
  const float* x;
  uint32_t n;
  uint32_t nfull;  // full warp tiles
  uint64_t seed;
  const uint32_t* prefix;  // span-layout prefix table (words) or nullptr
  float* norms;
  uint32_t* packed;
  unsigned long long* bad;
  bool tma;     // x 16-byte aligned and the tensor map describes its full rows
  bool p_al16;  // packed 16-byte aligned: bulk store
};

__device__ __forceinline__ uint4 ldg_nc_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float4 lds_v4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// pass 2 of one group on the fast path; returns false when the group needs the
// exact path (ambiguous key compare).  Keys ride one group ahead in a ring of
// 8 quads: the group's 32 key words are hashed first, then the next group's
// keys (kn, or nothing when kn == nullptr) are loaded into the ring, then the
// elements are quantized — the loads are volatile so they stay ahead of the
// shared-memory reads and get a whole group of work to land.
template <uint32_t BITS, int LGB, int KM>
__device__ __forceinline__ bool span_group_fast(const float* slot, uint32_t lane, uint32_t i0,
                                                uint32_t nu, uint32_t s_lo, uint32_t s_hi,
                                                const HashK& shk, uint32_t (&w)[BITS + 1],
                                                uint4 (&kh)[8], uint4 (&kl)[8], const uint4* kn) {
  constexpr uint32_t W = BITS + 1;
  const uint32_t b = i0 >> LGB;
  const float* row = slot + lane * 32u;
  const uint32_t key = lane & 7u;
  uint32_t hh[32];
  if (KM == kKmPrefix) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      hh[4 * q + 0] = key_hraw_from_prefix(kl[q].x, kh[q].x, s_lo, s_hi, shk);
      hh[4 * q + 1] = key_hraw_from_prefix(kl[q].y, kh[q].y, s_lo, s_hi, shk);
      hh[4 * q + 2] = key_hraw_from_prefix(kl[q].z, kh[q].z, s_lo, s_hi, shk);
      hh[4 * q + 3] = key_hraw_from_prefix(kl[q].w, kh[q].w, s_lo, s_hi, shk);
    }
  } else if (KM == kKmTable) {  // the final key's top word (the compare window covers it)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      hh[4 * q + 0] = kh[q].x;
      hh[4 * q + 1] = kh[q].y;
      hh[4 * q + 2] = kh[q].z;
      hh[4 * q + 3] = kh[q].w;
    }
  }
  if (KM != kKmInline && kn != nullptr) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      kh[q] = ldg_nc_v4(kn + q * 32);
      if (KM == kKmPrefix) kl[q] = ldg_nc_v4(kn + 256 + q * 32);
    }
  }
  const double nd = f32abs_to_f64(nu);
  const double y = __drcp_rn(nd);
  uint32_t mn = ~0u;
#pragma unroll
  for (int m = 0; m < int(W); ++m) w[m] = 0u;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 v = lds_v4(row + ((uint32_t(q) ^ key) << 2));
    const uint32_t u[4] = {__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z),
                           __float_as_uint(v.w)};
    if (KM == kKmInline) {
#pragma unroll
      for (int k = 0; k < 4; ++k) hh[4 * q + k] = key_hraw_inline(i0 + 4 * q + k, b, s_lo, s_hi, shk);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      put_field<W>(w, uint32_t(4 * q + k), span_field<BITS>(u[k], nd, y, hh[4 * q + k], mn));
  }
  return mn > 2u;
}

template <uint32_t BITS, int LGB, bool PREFIX>
__global__ void __launch_bounds__(32 * kWarps, 1)
    k_span(const __grid_constant__ CUtensorMap tmap, SpanArgs A) {
  constexpr uint32_t W = BITS + 1;
  constexpr uint32_t BL = 1u << LGB;                         // bucket length
  constexpr uint32_t NB = BL <= kSpan ? kSpan / BL : 1u;      // buckets per row (1, 2, 4)
  constexpr uint32_t GPB = BL <= kSpan ? BL / 32 : 4u;        // groups per bucket in a row
  extern __shared__ __align__(1024) unsigned char span_smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  unsigned char* base = span_smem + warp * warp_smem_bytes(W);
  float* slots = reinterpret_cast<float*>(base);
  uint32_t* outw = reinterpret_cast<uint32_t*>(base + kSlots * kSlotFloats * 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kSlots * kSlotFloats * 4 + out_words(W) * 4);
  const uint32_t gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  const uint32_t ntiles = A.nfull + (A.n > A.nfull * kWTile ? 1u : 0u);
  const HashK shk = make_hashk();
  const uint32_t s_lo = uint32_t(A.seed), s_hi = uint32_t(A.seed >> 32);

  if (lane == 0) {
    for (uint32_t s = 0; s < kSlots; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // Quarter Q of this warp's work = quarter Q % 4 of its (Q / 4)-th tile; it
  // lives in slot Q % 5, whose mbarrier completes its (Q / 5)-th phase.
  auto issue = [&](uint32_t Q) {
    const uint32_t t = gw + (Q >> 2) * nw, g = Q & 3u;
    if (t >= ntiles) return;
    const uint32_t s = Q % kSlots;
    float* dst = slots + s * kSlotFloats;
    if (A.tma && t < A.nfull) {
      if (lane == 0) {
        fence_async_smem();  // this slot's generic reads precede the async write
        mbar_arrive_expect_tx(bars + s, kSlotFloats * 4);
        tma_load_2d(dst, &tmap, int32_t(g * 32), int32_t(t * 32), bars + s);
      }
    } else {  // unaligned input or the ragged last tile: zero-filled register copy
      const uint64_t t0 = uint64_t(t) * kWTile;
      for (uint32_t r = 0; r < 32; ++r) {
        const uint64_t i = t0 + r * kSpan + g * 32 + lane;
        dst[swz(r, lane)] = i < A.n ? A.x[i] : 0.0f;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + s);
    }
  };
  auto wait_q = [&](uint32_t Q) { mbar_wait(bars + Q % kSlots, (Q / kSlots) & 1u); };

  uint4 kh[8], kl[8];
  if (PREFIX && gw < ntiles) {
    const uint4* k0 = reinterpret_cast<const uint4*>(A.prefix + uint64_t(gw) * 8192u) + lane;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      kh[q] = __ldg(k0 + q * 32);
      kl[q] = __ldg(k0 + 256 + q * 32);
    }
  }
  for (uint32_t Q = 0; Q < kSlots; ++Q) issue(Q);

  uint32_t j = 0;
  for (uint32_t t = gw; t < ntiles; t += nw, ++j) {
    const bool more = t + nw < ntiles;
    const bool full = t < A.nfull;
    const uint32_t i_lane = t * kWTile + lane * kSpan;  // first element of the row
    RowView rv;
#pragma unroll
    for (uint32_t g = 0; g < 4; ++g) rv.slot[g] = slots + ((4 * j + g) % kSlots) * kSlotFloats;
    rv.r = lane;

    // ---- pass 1: sequential FP64 norms of the row's buckets, quarter by quarter ----
    uint32_t nu[NB];
    bool careful[NB];
    if constexpr (BL > kSpan) {  // a bucket spans rows: its first lane sums them
#pragma unroll
      for (uint32_t g = 0; g < 4; ++g) wait_q(4 * j + g);
      uint32_t fb;
      span_pass1_big<LGB>(rv, lane, nu[0], careful[0], fb);
      if ((lane & (BL / kSpan - 1u)) == 0) {
        if (fb != ~0u && A.bad != nullptr) atomicMin(A.bad, (unsigned long long)(i_lane + fb));
        if (full || i_lane < A.n) A.norms[i_lane >> LGB] = __uint_as_float(nu[0]);
      }
    } else {
      double sq = 0.0;
#pragma unroll
      for (uint32_t g = 0; g < 4; ++g) {
        wait_q(4 * j + g);
        const float* row = rv.slot[g] + lane * 32u;
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(row + ((q ^ (lane & 7u)) << 2));
          // exact conversion for every finite float; a non-finite input makes
          // sq non-finite (squares of floats cannot overflow FP64)
          double d = double(v.x);
          sq = __fma_rn(d, d, sq);
          d = double(v.y);
          sq = __fma_rn(d, d, sq);
          d = double(v.z);
          sq = __fma_rn(d, d, sq);
          d = double(v.w);
          sq = __fma_rn(d, d, sq);
        }
        if ((g * 32 + 32) % BL == 0) {  // bucket r complete
          const uint32_t r = (g * 32) / BL;
          const bool c = (uint32_t(__double2hiint(sq)) & 0x7FF00000u) == 0x7FF00000u;
          const uint32_t v = c ? span_norm_exact(rv, r * BL, BL, i_lane + r * BL, A.bad)
                               : __float_as_uint(__double2float_rn(__dsqrt_rn(sq)));
#pragma unroll
          for (uint32_t rr = 0; rr < NB; ++rr)
            if (rr == r) {
              nu[rr] = v;
              careful[rr] = c;
            }
          if (full || i_lane + r * BL < A.n) A.norms[(i_lane >> LGB) + r] = __uint_as_float(v);
          sq = 0.0;
        }
      }
    }

    // ---- pass 2: quantize + pack the row's 4 groups ----
    if (A.p_al16 && lane == 0) bulk_wait_read0();  // previous tile's bulk store has read outw
    __syncwarp();
    // key ring: group 0 of this tile was loaded during the previous tile (or
    // before the loop); group g+1 (or group 0 of the next tile) loads during g
    const uint4* kp = PREFIX ? reinterpret_cast<const uint4*>(A.prefix + uint64_t(t) * 8192u) + lane
                             : nullptr;
    const uint4* kp_next =
        PREFIX && more ? reinterpret_cast<const uint4*>(A.prefix + uint64_t(t + nw) * 8192u) + lane
                       : nullptr;
#pragma unroll 1
    for (uint32_t g = 0; g < 4; ++g) {
      const uint32_t r = g / GPB;
      uint32_t nug = nu[0];
      bool car = careful[0];
#pragma unroll
      for (uint32_t rr = 1; rr < NB; ++rr)
        if (r == rr) {
          nug = nu[rr];
          car = careful[rr];
        }
      const uint32_t i0 = i_lane + g * 32;
      const uint4* kn = g < 3 ? kp + (g + 1) * 512 : kp_next;
      if (PREFIX && lane == 0) {  // keys two groups ahead into L2 (the ring loads then hit L2)
        const uint4* k2 = g < 2 ? kp + (g + 2) * 512 : (kp_next ? kp_next + (g - 2) * 512 : nullptr);
        if (k2 != nullptr) prefetch_l2(k2 - lane, 8192);
      }
      const float* slot = slots + ((4 * j + g) % kSlots) * kSlotFloats;
      // The fast path always runs (its result is discarded for an all-zero or
      // non-finite bucket), so the key ring flows through one code path; the
      // exact path writes its words itself, so no local-memory result merges
      // into registers the key-ring loads are pending on.
      uint32_t* wout = outw + (lane * 4 + g) * W;
      uint32_t w[W];
      const bool ok = span_group_fast<BITS, LGB, PREFIX ? kKmPrefix : kKmInline>(
                          slot, lane, i0, nug, s_lo, s_hi, shk, w, kh, kl, kn) &&
                      nug != 0u && !car;
      if (ok) {
#pragma unroll
        for (int m = 0; m < int(W); ++m) wout[m] = w[m];
      } else {
        span_group_exact<BITS, LGB, PREFIX ? kKmPrefix : kKmInline>(rv, g, i0, nug, A.seed,
                                            PREFIX ? A.prefix + uint64_t(t) * 8192u : nullptr, lane,
                                            wout);
      }
      __syncwarp();               // every lane is done with this slot
      issue(4 * j + g + kSlots);  // refill it: the quarter kSlots ahead
    }
    __syncwarp();
    uint32_t* dstw = A.packed + uint64_t(t) * out_words(W);
    if (A.p_al16 && full) {
      fence_async_smem();
      __syncwarp();
      if (lane == 0) bulk_s2g(dstw, outw, out_words(W) * 4);
    } else {  // only the words the vector owns (gcx_packed_capacity)
      const uint32_t nwords =
          full ? out_words(W) : uint32_t((uint64_t(A.n - t * kWTile) * W + 31) / 32);
      for (uint32_t e = lane; e < nwords; e += 32) dstw[e] = outw[e];
    }
    __syncwarp();  // outw free for reuse
  }
  if (A.p_al16 && lane == 0) bulk_wait0();  // bulk stores complete before exit
}

// ---------------------------------------------------------------------------
// K1 span over a piece table (gcx_encode_pieces: SRA stage 1, the owner's
// re-encode, the engine's buffers) whose quantized pieces all share one
// (bits, bucket in {32, 64, 128}) — GCX_F_SPAN_ENC from gcx_plan_tiles.  Same
// passes and key ring as k_span; per tile the piece is located in the tile
// prefix (pieces are piece-local: bucket and key indices restart at every
// piece, codec.cpp:60 via collectives.cpp:143-163).  Tiles are staged by
// zero-filling cp.async copies (piece offsets are arbitrary, so no tensor map
// describes them), completion counted on the slot's mbarrier
// (cp.async.mbarrier.arrive.noinc, one arrival per lane).  Raw pieces are
// copied into the message by the warp.  Keys: inline, or span-layout
// prefixes at run offset p.keys (gcx_plan_keys / gcx_make_key_prefix).
// ---------------------------------------------------------------------------
// Raw pieces (CodecMode::uncompressed) travel as f32.  A warp (or CTA) copies
// or folds a tile of them with 16-byte accesses and 4 loads in flight per
// lane: a lane-strided scalar loop keeps one dependent load per iteration in
// flight and made a warp with a 4096-element raw tile the kernel's straggler.
__device__ __forceinline__ void raw_copy(const float* __restrict__ in, float* __restrict__ out,
                                         uint32_t count, float div, float recip, bool pow2,
                                         uint32_t tid, uint32_t nthreads) {
  if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0) {
    const uint32_t n4 = count >> 2;
    const float4* i4 = reinterpret_cast<const float4*>(in);
    float4* o4 = reinterpret_cast<float4*>(out);
#pragma unroll 4
    for (uint32_t k = tid; k < n4; k += nthreads) {
      float4 v = __ldcs(i4 + k);
      v.x = apply_divisor(v.x, div, recip, pow2);
      v.y = apply_divisor(v.y, div, recip, pow2);
      v.z = apply_divisor(v.z, div, recip, pow2);
      v.w = apply_divisor(v.w, div, recip, pow2);
      __stcs(o4 + k, v);
    }
    for (uint32_t e = (n4 << 2) + tid; e < count; e += nthreads)
      out[e] = apply_divisor(__ldcs(in + e), div, recip, pow2);
  } else {
#pragma unroll 8
    for (uint32_t e = tid; e < count; e += nthreads)
      out[e] = apply_divisor(__ldcs(in + e), div, recip, pow2);
  }
}

struct SpanPiecesArgs {
  gcx_plan::PlanView pv;
  uint32_t flags;
  uint64_t seed;
  const unsigned long long* seed_dev;  // GCX_F_SEED_DEVICE: the launch seed, read on the device
  const float* src;      // the input (FOLD: the owner's raw values)
  uint8_t* msg;          // the message written (FOLD: the owner's broadcast message)
  const uint32_t* keys;  // span-layout prefix words or nullptr (inline)
  unsigned long long* bad;
  // FOLD (SRA owner step): peer id's message for this chunk sits in receive
  // slot (id < me ? id : id - 1) at recv + slot * slot_stride
  const uint8_t* recv;
  uint64_t slot_stride;
  uint32_t nodes, me;
};

// The table's launch seed: a kernel argument, or (GCX_F_SEED_DEVICE: a step
// replayed from a CUDA graph) a word in device memory written earlier on the
// stream (gcx_sra_step_seeds)
__device__ __forceinline__ uint64_t launch_seed(const SpanPiecesArgs& A) {
  return A.seed_dev != nullptr ? *A.seed_dev : A.seed;
}

// Widths 5-8: a chunk's table would have F = 2^(bits+1) > 32 entries, so each
// element's value is computed from its own field instead (dequant_field:
// RN32(RN64(RN64(norm * level) / s)), signed, then finalize's divisor) — four
// independent FP64 chains per lane per chunk.  `win` is the lane's 4W-bit
// window (at most 36 bits: two words).
//
// RN32(RN64(nl / s)) for nl = RN64(norm * level) (exact): q0 = RN(nl * RN(1/s))
// is within 3 ulp of RN64(nl / s) (RN(1/s) and the product each carry a
// relative error <= 2^-53), so the two round to the same float unless q0's 29
// dropped bits lie within a few ulp of the halfway point 2^28, or q0 is below
// the normal float range; only then is dequant_field's correction step taken.
__device__ __forceinline__ float wide_mag(double nl, double sd, double ys) {
  const double q0 = __dmul_rn(nl, ys);
  const uint32_t hi = uint32_t(__double2hiint(q0)), lo = uint32_t(__double2loint(q0));
  if ((lo & 0x1FFFFFFFu) - 0x0FFFFFF8u < 16u || hi - 1u < 0x380FFFFFu) {  // rare
    const double q = __fma_rn(__fma_rn(-sd, q0, nl), ys, q0);
    return f64pos_to_f32_rn(q);
  }
  return __double2float_rn(q0);  // nl = 0 (level 0) lands here: +0
}

template <uint32_t BITS>
__device__ __forceinline__ void wide_values(uint64_t win, double nd, float div, float recip, bool pow2,
                                            float (&v)[4]) {
  constexpr uint32_t W = BITS + 1, S = (1u << BITS) - 1;
  const double sd = double(S), ys = 1.0 / double(S);  // RN(1/s), as __drcp_rn
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t f = uint32_t(win >> (k * W)) & ((1u << W) - 1u);
    const float m = wide_mag(__dmul_rn(nd, u32_to_f64(f & S)), sd, ys);
    v[k] = apply_divisor((f >> BITS) && (f & S) ? -m : m, div, recip, pow2);
  }
}

__device__ __forceinline__ uint64_t lane_window2(uint32_t w0, uint32_t w1, uint32_t qsh, bool two) {
  return (two ? (uint64_t(w1) << 32) | w0 : uint64_t(w0)) >> qsh;
}

__device__ __forceinline__ uint64_t lane_window(const uint32_t* cw, uint32_t qsh, bool two) {
  return lane_window2(cw[0], two ? cw[1] : 0u, qsh, two);
}

// The SRA owner's fold of one tile (collectives.cpp:266-279) straight into
// the K1 staging slots: row r of the tile (one bucket of 128) is decoded from
// every peer's payload warp-wide — lane l owns elements 4l..4l+3, the peer's
// table for the row's bucket lives one entry per lane (as k_dspan), so a
// value is one shuffle — and added in ascending node id with the owner's raw
// values (f32, the reference's order).  The aggregate is stored swizzled into
// slot l/8, where the span K1 passes read it.  Row r+1's loads (the peers'
// norms and packed windows, the owner's raw quad) are issued before row r is
// folded.  Widths 5-8 compute each value from its field (wide_values).
// Buckets 128 / 512; nodes <= 8.
template <uint32_t BITS, int LGB>
__device__ __forceinline__ void fold_tile(const SpanPiecesArgs& A, const gcx_piece& p,
                                          uint32_t start, uint32_t count, float* slots,
                                          uint32_t lane, uint32_t r0 = 0, uint32_t r1 = 32,
                                          uint32_t rstep = 1) {
  constexpr uint32_t W = BITS + 1, S = (1u << BITS) - 1, F = 2u << BITS;
  const uint32_t f = lane & (F - 1u), level = f & S, sign = f >> BITS;
  const double dl = double(level);
  const double sd = double(S), ys = __drcp_rn(sd);
  const uint32_t qbit = 4 * W * lane, qw = qbit >> 5, qsh = qbit & 31u;
  const bool two = qsh + 4 * W > 32;
  const uint32_t nodes = A.nodes, me = A.me;
  struct RowLoads {
    uint32_t nu[8], w0[8], w1[8];
    float4 own;
  };
  auto load_row = [&](uint32_t r, RowLoads& L) {
    const uint32_t vr = count > r * 128u ? min(128u, count - r * 128u) : 0u;
    const uint32_t e_row = start + r * 128u;
    const bool quad = 4 * lane < vr;
    L.own = make_float4(0.f, 0.f, 0.f, 0.f);
    if (quad) {
      const float* o = A.src + p.src + e_row + 4 * lane;
      if (4 * lane + 4 <= vr && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
        L.own = __ldg(reinterpret_cast<const float4*>(o));
      } else {
        L.own.x = __ldg(o);
        if (4 * lane + 1 < vr) L.own.y = __ldg(o + 1);
        if (4 * lane + 2 < vr) L.own.z = __ldg(o + 2);
        if (4 * lane + 3 < vr) L.own.w = __ldg(o + 3);
      }
    }
#pragma unroll
    for (uint32_t id = 0; id < 8; ++id) {
      L.nu[id] = 0u;
      L.w0[id] = 0u;
      L.w1[id] = 0u;
      if (id < nodes && id != me && vr > 0) {
        const uint8_t* m = A.recv + uint64_t(id < me ? id : id - 1) * A.slot_stride;
        L.nu[id] = __ldg(reinterpret_cast<const uint32_t*>(m + p.norms) + (e_row >> LGB));
        if (quad) {
          const uint32_t* wp = reinterpret_cast<const uint32_t*>(m + p.packed) + (e_row >> 5) * W + qw;
          L.w0[id] = __ldg(wp);
          if (two) L.w1[id] = __ldg(wp + 1);
        }
      }
    }
  };
  RowLoads cur;
  load_row(r0, cur);
#pragma unroll 1
  for (uint32_t r = r0; r < r1; r += rstep) {
    if (r * 128u >= count) {  // the rest of this lane set's rows lie past the piece: zeros
      for (; r < r1; r += rstep)
        *reinterpret_cast<float4*>(slots + (lane >> 3) * kSlotFloats + r * 32u +
                                   (((lane & 7u) ^ (r & 7u)) << 2)) = make_float4(0.f, 0.f, 0.f, 0.f);
      break;
    }
    RowLoads nxt;
    if (r + rstep < r1) load_row(r + rstep, nxt);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    // every peer's table entry first (absent peers give 0), unconditionally:
    // eight independent FP64 chains the scheduler can overlap
    float entry[8];
    if constexpr (F <= 32) {
#pragma unroll
      for (uint32_t id = 0; id < 8; ++id) {
        // this lane's entry of peer id's table for the row's bucket (dequant_field)
        const double nl = __dmul_rn(double(__uint_as_float(cur.nu[id])), dl);  // exact
        const double q0 = __dmul_rn(nl, ys);
        const double q = __fma_rn(__fma_rn(-sd, q0, nl), ys, q0);
        const float m = __double2float_rn(q);
        entry[id] = level == 0 ? 0.0f : (sign ? -m : m);
      }
    }
#pragma unroll
    for (uint32_t id = 0; id < 8; ++id) {
      if (id >= nodes) break;
      float x[4];
      if (id == me) {
        x[0] = cur.own.x;
        x[1] = cur.own.y;
        x[2] = cur.own.z;
        x[3] = cur.own.w;
      } else if constexpr (F > 32) {  // widths 5-8: per-element values
        wide_values<BITS>(lane_window2(cur.w0[id], cur.w1[id], qsh, two),
                          double(__uint_as_float(cur.nu[id])), 1.0f, 1.0f, false, x);
      } else {
        const uint32_t win = two ? __funnelshift_r(cur.w0[id], cur.w1[id], qsh) : (cur.w0[id] >> qsh);
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = __shfl_sync(0xffffffffu, entry[id], (win >> (k * W)) & (F - 1u));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = id == 0 ? x[k] : __fadd_rn(acc[k], x[k]);
    }
    // elements past the piece stay 0 (zero-filled tile)
    const uint32_t vr = count > r * 128u ? min(128u, count - r * 128u) : 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (4 * lane + k >= vr) acc[k] = 0.0f;
    float* dst = slots + (lane >> 3) * kSlotFloats + r * 32u + ((((lane & 7u) ^ (r & 7u))) << 2);
    *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    cur = nxt;
  }
}

__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4z(void* smem, const void* gmem, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <uint32_t BITS, int LGB, int KM, bool FOLD>
__global__ void __launch_bounds__(32 * kWarps, 1) k_span_pieces(SpanPiecesArgs A) {
  static_assert(!FOLD || (BITS <= 4 && LGB >= 7), "the fused fold needs bits <= 4 and bucket >= 128");
  constexpr uint32_t W = BITS + 1;
  constexpr uint32_t BL = 1u << LGB;
  constexpr uint32_t NB = BL <= kSpan ? kSpan / BL : 1u;
  constexpr uint32_t GPB = BL <= kSpan ? BL / 32 : 4u;
  extern __shared__ __align__(1024) unsigned char span_smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  unsigned char* base = span_smem + warp * warp_smem_bytes(W);
  float* slots = reinterpret_cast<float*>(base);
  uint32_t* outw = reinterpret_cast<uint32_t*>(base + kSlots * kSlotFloats * 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kSlots * kSlotFloats * 4 + out_words(W) * 4);
  const uint32_t gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
  const uint32_t ntiles = A.pv.ntiles;
  const HashK shk = make_hashk();
  const bool piece_seeds = (A.flags & GCX_F_PIECE_SEEDS) != 0;

  if (lane == 0) {
    for (uint32_t s = 0; s < kSlots; ++s) mbar_init(bars + s, 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // Tile contexts: each tile is located once (locate_warp searches the tile
  // prefix) and kept in the warp's shared slot `memo` until the next tile is
  // located: the quarters of a tile are issued back to back and the main
  // loop's look-ahead asks for the tile the last issue located.
  __shared__ gcx_plan::TileCtx memo_all[kWarps];
  __shared__ uint32_t memo_t[kWarps];
  gcx_plan::TileCtx& memo = memo_all[warp];
  if (lane == 0) memo_t[warp] = ~0u;
  __syncwarp();
  auto ctx_of = [&](uint32_t t, gcx_plan::TileCtx& c) {
    if (memo_t[warp] == t) {
      c = memo;
      return;
    }
    gcx_plan::locate_warp(A.pv, t, c);
    __syncwarp();
    if (lane == 0) {
      memo = c;
      memo_t[warp] = t;
    }
    __syncwarp();
  };
  // quarter Q = quarter Q % 4 of this warp's (Q / 4)-th tile, slot Q % 5
  auto issue = [&](uint32_t Q) {
    if (FOLD) return;  // the fold writes the slots itself
    const uint32_t t = gw + (Q >> 2) * nw, g = Q & 3u;
    if (t >= ntiles) return;
    gcx_plan::TileCtx c;
    ctx_of(t, c);
    uint64_t* bar = bars + Q % kSlots;
    if (c.p.bits > 0) {
      float* dst = slots + (Q % kSlots) * kSlotFloats;
      const float* x = A.src + c.p.src + c.start + g * 32;
      if ((reinterpret_cast<uintptr_t>(A.src + c.p.src) & 15u) == 0) {
#pragma unroll
        for (uint32_t m = 0; m < 8; ++m) {  // lanes 8r'..8r'+7: one row's 128 bytes
          const uint32_t r = 4 * m + (lane >> 3), ch = lane & 7u;
          const uint32_t e = r * kSpan + g * 32 + ch * 4;
          const uint32_t nb = e >= c.count ? 0u : min(4u, c.count - e) * 4u;
          cp_async16z(dst + r * 32 + ((ch ^ (r & 7u)) << 2), nb ? x + r * kSpan + ch * 4 : A.src, nb);
        }
      } else {
        for (uint32_t r = 0; r < 32; ++r) {
          const uint32_t e = r * kSpan + g * 32 + lane;
          cp_async4z(dst + swz(r, lane), e < c.count ? x + r * kSpan + lane : A.src, e < c.count ? 4u : 0u);
        }
      }
    }
    cp_async_mbar_arrive(bar);  // raw tiles: the phase completes at once
  };
  auto wait_q = [&](uint32_t Q) { mbar_wait(bars + Q % kSlots, (Q / kSlots) & 1u); };
  auto key_group = [&](const gcx_plan::TileCtx& c, uint32_t g) -> const uint4* {
    return reinterpret_cast<const uint4*>(A.keys) + ((c.p.keys + c.start) >> 12) * 2048 + g * 512 + lane;
  };

  uint4 kh[8], kl[8];
  gcx_plan::TileCtx cur;
  if (gw < ntiles) {
    ctx_of(gw, cur);
    if (KM != kKmInline && cur.p.bits > 0) {
      const uint4* k0 = key_group(cur, 0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        kh[q] = __ldg(k0 + q * 32);
        if (KM == kKmPrefix) kl[q] = __ldg(k0 + 256 + q * 32);
      }
    }
  }
  for (uint32_t Q = 0; Q < kSlots; ++Q) issue(Q);

  uint32_t j = 0;
  for (uint32_t t = gw; t < ntiles; t += nw, ++j) {
    const bool more = t + nw < ntiles;
    gcx_plan::TileCtx nxt;
    if (more) ctx_of(t + nw, nxt);
    const gcx_piece& p = cur.p;
    if (p.bits == 0) {  // raw piece: its f32 values are the payload (collectives.cpp:153-158)
      const float* xs = A.src + p.src + cur.start;
      float* d = reinterpret_cast<float*>(A.msg + p.norms) + cur.start;
      if (FOLD) {  // the raw fold, ascending id (collectives.cpp:268-279)
#pragma unroll 4
        for (uint32_t e = lane; e < cur.count; e += 32) {
          float acc = 0.0f;
          for (uint32_t id = 0; id < A.nodes; ++id) {
            const float x =
                id == A.me ? __ldg(xs + e)
                           : __ldg(reinterpret_cast<const float*>(
                                 A.recv + uint64_t(id < A.me ? id : id - 1) * A.slot_stride + p.norms) +
                                 cur.start + e);
            acc = id == 0 ? x : __fadd_rn(acc, x);
          }
          d[e] = acc;
        }
      } else {
        raw_copy(xs, d, cur.count, 1.0f, 1.0f, true, lane, 32);
      }
      if (KM != kKmInline && more && nxt.p.bits > 0) {  // the key ring's next group
        const uint4* kn = key_group(nxt, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          kh[q] = __ldg(kn + q * 32);
          if (KM == kKmPrefix) kl[q] = __ldg(kn + 256 + q * 32);
        }
      }
#pragma unroll 1
      for (uint32_t g = 0; g < 4; ++g) {
        __syncwarp();
        issue(4 * j + g + kSlots);
      }
      cur = nxt;
      continue;
    }
    const uint64_t seed = piece_seeds ? p.seed : launch_seed(A);
    const uint32_t s_lo = uint32_t(seed), s_hi = uint32_t(seed >> 32);
    const bool full = cur.count == kWTile;
    const uint32_t i_lane = cur.start + lane * kSpan;  // piece-local first element of the row
    uint32_t* norms = reinterpret_cast<uint32_t*>(A.msg + p.norms);
    const unsigned long long pkey = uint64_t(cur.pidx) << 40;
    RowView rv;
#pragma unroll
    for (uint32_t g = 0; g < 4; ++g) rv.slot[g] = slots + (FOLD ? g : (4 * j + g) % kSlots) * kSlotFloats;
    rv.r = lane;
    if (FOLD) {
      if constexpr (FOLD) fold_tile<BITS, LGB>(A, p, cur.start, cur.count, slots, lane);
      __syncwarp();
    }

    // ---- pass 1 ----
    uint32_t nu[NB];
    bool careful[NB];
    if constexpr (BL > kSpan) {  // a bucket spans rows: its first lane sums them
      if (!FOLD) {
#pragma unroll
        for (uint32_t g = 0; g < 4; ++g) wait_q(4 * j + g);
      }
      uint32_t fb;
      span_pass1_big<LGB>(rv, lane, nu[0], careful[0], fb);
      if ((lane & (BL / kSpan - 1u)) == 0) {
        if (fb != ~0u && A.bad != nullptr) atomicMin(A.bad, pkey | (i_lane + fb));
        if (i_lane < p.len) norms[i_lane >> LGB] = nu[0];
      }
    } else {
      double sq = 0.0;
#pragma unroll
      for (uint32_t g = 0; g < 4; ++g) {
        if (!FOLD) wait_q(4 * j + g);
        const float* row = rv.slot[g] + lane * 32u;
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(row + ((q ^ (lane & 7u)) << 2));
          double d = double(v.x);
          sq = __fma_rn(d, d, sq);
          d = double(v.y);
          sq = __fma_rn(d, d, sq);
          d = double(v.z);
          sq = __fma_rn(d, d, sq);
          d = double(v.w);
          sq = __fma_rn(d, d, sq);
        }
        if ((g * 32 + 32) % BL == 0) {
          const uint32_t r = (g * 32) / BL;
          const bool c = (uint32_t(__double2hiint(sq)) & 0x7FF00000u) == 0x7FF00000u;
          uint32_t v;
          if (c) {
            v = span_norm_exact(rv, r * BL, BL, 0u, nullptr);
            if (A.bad != nullptr) {  // first non-finite: (piece << 40) | piece-local index
              for (uint32_t e = 0; e < BL; ++e)
                if ((__float_as_uint(rv.at(r * BL + e)) & 0x7FFFFFFFu) >= 0x7F800000u) {
                  atomicMin(A.bad, pkey | (i_lane + r * BL + e));
                  break;
                }
            }
          } else {
            v = __float_as_uint(__double2float_rn(__dsqrt_rn(sq)));
          }
#pragma unroll
          for (uint32_t rr = 0; rr < NB; ++rr)
            if (rr == r) {
              nu[rr] = v;
              careful[rr] = c;
            }
          if (i_lane + r * BL < p.len) norms[(i_lane >> LGB) + r] = v;
          sq = 0.0;
        }
      }
    }

    // ---- pass 2 ----
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
    const uint4* kp = KM != kKmInline ? key_group(cur, 0) : nullptr;
    const uint4* kp_next = KM != kKmInline && more && nxt.p.bits > 0 ? key_group(nxt, 0) : nullptr;
#pragma unroll 1
    for (uint32_t g = 0; g < 4; ++g) {
      const uint32_t r = g / GPB;
      uint32_t nug = nu[0];
      bool car = careful[0];
#pragma unroll
      for (uint32_t rr = 1; rr < NB; ++rr)
        if (r == rr) {
          nug = nu[rr];
          car = careful[rr];
        }
      const uint32_t i0 = i_lane + g * 32;
      const uint4* kn = g < 3 ? kp + (g + 1) * 512 : kp_next;
      const float* slot = rv.slot[g];
      uint32_t* wout = outw + (lane * 4 + g) * W;
      uint32_t w[W];
      const bool ok = span_group_fast<BITS, LGB, KM>(slot, lane, i0, nug, s_lo, s_hi, shk, w, kh,
                                                         kl, kn) &&
                      nug != 0u && !car;
      if (ok) {
#pragma unroll
        for (int m = 0; m < int(W); ++m) wout[m] = w[m];
      } else {
        span_group_exact<BITS, LGB, KM>(
            rv, g, i0, nug, seed,
            KM != kKmInline ? A.keys + ((p.keys + cur.start) >> 12) * 8192u : nullptr, lane, wout);
      }
      __syncwarp();
      issue(4 * j + g + kSlots);
    }
    __syncwarp();
    uint32_t* dstw = reinterpret_cast<uint32_t*>(A.msg + p.packed) + uint64_t(cur.start >> 5) * W;
    if (full && (reinterpret_cast<uintptr_t>(dstw) & 15u) == 0) {
      fence_async_smem();
      __syncwarp();
      if (lane == 0) bulk_s2g(dstw, outw, out_words(W) * 4);
    } else {
      const uint32_t nwords = (cur.count * W + 31) / 32;
      for (uint32_t e = lane; e < nwords; e += 32) dstw[e] = outw[e];
    }
    __syncwarp();
    cur = nxt;
  }
  if (lane == 0) bulk_wait0();
}


// ---------------------------------------------------------------------------
// K3 span decode (codec::dequantize, codec.cpp:71-95, + finalize's average,
// collectives.cpp:213-228) for bits <= 4 and power-of-two buckets of 128 ..
// 4096 (C1 and the default plans).  A warp owns a tile of 4096 elements = 32
// chunks of 128; every chunk lies in one bucket, so the chunk's signed
// dequantization table has F = 2^(bits+1) <= 32 entries and lives one entry
// per LANE: lane k computes entry f = k % F once per chunk (one FP64 RN(norm *
// level / s) per lane, bit-exact as dequant_field), and each element's value
// is one warp shuffle from the lane holding its field.  No shared-memory
// table, no bank conflicts.  Lane l decodes elements 4l..4l+3 of each chunk
// (its 4W-bit window of the chunk's packed words, staged per tile in shared
// memory by coalesced 16-byte loads) and writes them with one coalesced
// 16-byte streaming store: the kernel moves C(n) + 4n bytes and little else.
// ---------------------------------------------------------------------------
constexpr int kDWarps = 8;
#ifndef GCX_DSPAN_MINB
#define GCX_DSPAN_MINB 4
#endif

struct DspanArgs {
  const float* norms;
  const uint32_t* packed;
  float* out;
  uint32_t n;
  float div, recip;
  bool pow2;
};

template <uint32_t BITS, uint32_t LGB>
__global__ void __launch_bounds__(32 * kDWarps, GCX_DSPAN_MINB) k_dspan(DspanArgs A) {
  constexpr uint32_t W = BITS + 1, S = (1u << BITS) - 1, F = 2u << BITS;
  constexpr uint32_t TW = 128u * W;               // packed words per tile
  constexpr uint32_t NBT = kWTile >> LGB;         // buckets per tile (1..32)
  constexpr uint32_t BSH = LGB - 7;               // chunks per bucket = 2^BSH
  __shared__ __align__(16) uint32_t words_all[kDWarps][TW];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t* words = words_all[warp];
  const uint32_t gw = blockIdx.x * kDWarps + warp, nw = gridDim.x * kDWarps;
  const uint32_t ntiles = (A.n + kWTile - 1) / kWTile;
  const uint32_t nwords = uint32_t((uint64_t(A.n) * W + 31) / 32);  // gcx_packed_capacity / 4
  const uint32_t nbk = (A.n + (1u << LGB) - 1) >> LGB;
  // this lane's table entry: field f = level | sign << BITS
  const uint32_t f = lane & (F - 1u), level = f & S, sign = f >> BITS;
  const double dl = double(level);
  const double sd = double(S), ys = __drcp_rn(sd);
  // this lane's 4W-bit window inside every chunk
  const uint32_t qbit = 4 * W * lane, qw = qbit >> 5, qsh = qbit & 31u;
  const bool two = qsh + 4 * W > 32;
  for (uint32_t t = gw; t < ntiles; t += nw) {
    const uint32_t e0 = t * kWTile;
    const bool full = e0 + kWTile <= A.n;
    // stage the tile's packed words (coalesced 16-byte loads) and its norms
    const uint32_t* src = A.packed + uint64_t(t) * TW;
    const uint32_t b0 = e0 >> LGB;
    const uint32_t nreg =
        lane < NBT && b0 + lane < nbk ? __ldg(reinterpret_cast<const uint32_t*>(A.norms) + b0 + lane) : 0u;
    if (full) {
      uint4 st[W];
#pragma unroll
      for (uint32_t k = 0; k < W; ++k) st[k] = __ldcs(reinterpret_cast<const uint4*>(src) + k * 32 + lane);
#pragma unroll
      for (uint32_t k = 0; k < W; ++k) reinterpret_cast<uint4*>(words)[k * 32 + lane] = st[k];
    } else {
      for (uint32_t k = lane; k < TW; k += 32) words[k] = t * TW + k < nwords ? src[k] : 0u;
    }
    __syncwarp();
    float* out = A.out + e0 + 4 * lane;
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15u) == 0 && full;
    if constexpr (F > 32) {  // widths 5-8: per-element values (wide_values)
#pragma unroll 4
      for (uint32_t c = 0; c < 32; ++c) {
        if (!full && e0 + c * 128 >= A.n) break;
        const double nd = double(__uint_as_float(__shfl_sync(0xffffffffu, nreg, c >> BSH)));
        float v[4];
        wide_values<BITS>(lane_window(words + c * 4 * W + qw, qsh, two), nd, A.div, A.recip, A.pow2, v);
        float* o = out + c * 128;
        if (vec) {
          __stcs(reinterpret_cast<float4*>(o), make_float4(v[0], v[1], v[2], v[3]));
        } else {
          const uint32_t e = e0 + c * 128 + 4 * lane;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (e + k < A.n) __stcs(o + k, v[k]);
        }
      }
      __syncwarp();
      continue;
    }
    // batches of 8 chunks: the batch's table entries (one per bucket it
    // touches: RN32(RN64(RN64(norm * level) / s)), /N, signed) are 1..8
    // independent FP64 chains, then the chunks are decoded by shuffles
    constexpr uint32_t CB = 8;
    constexpr uint32_t NEB = (CB >> BSH) > 0 ? (CB >> BSH) : 1;
#pragma unroll
    for (uint32_t bb = 0; bb < 32 / CB; ++bb) {
      if (!full && e0 + bb * CB * 128 >= A.n) break;
      float entry[NEB];
#pragma unroll
      for (uint32_t i = 0; i < NEB; ++i) {
        const uint32_t nu = __shfl_sync(0xffffffffu, nreg, ((bb * CB) >> BSH) + i);
        const double nl = __dmul_rn(double(__uint_as_float(nu)), dl);  // exact
        const double q0 = __dmul_rn(nl, ys);
        const double q = __fma_rn(__fma_rn(-sd, q0, nl), ys, q0);  // RN(nl / s), see dequant_field
        const float m = apply_divisor(__double2float_rn(q), A.div, A.recip, A.pow2);
        entry[i] = level == 0 ? 0.0f : (sign ? -m : m);
      }
#pragma unroll
      for (uint32_t cc = 0; cc < CB; ++cc) {
        const uint32_t c = bb * CB + cc;
        if (!full && e0 + c * 128 >= A.n) break;
        const uint32_t* cw = words + c * 4 * W + qw;
        const uint32_t win = two ? __funnelshift_r(cw[0], cw[1], qsh) : (cw[0] >> qsh);
        const float en = entry[NEB > 1 ? (cc >> BSH) : 0];
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[k] = __shfl_sync(0xffffffffu, en, (win >> (k * W)) & (F - 1u));
        float* o = out + c * 128;
        if (vec) {
          __stcs(reinterpret_cast<float4*>(o), make_float4(v[0], v[1], v[2], v[3]));
        } else {
          const uint32_t e = e0 + c * 128 + 4 * lane;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (e + k < A.n) __stcs(o + k, v[k]);
        }
      }
    }
    __syncwarp();  // words[] is restaged by the next tile
  }
}

using DspanFn = void (*)(DspanArgs);

template <uint32_t BITS>
inline DspanFn pick_dspan_lgb(uint32_t lgb) {
  switch (lgb) {
    case 7: return k_dspan<BITS, 7>;
    case 8: return k_dspan<BITS, 8>;
    case 9: return k_dspan<BITS, 9>;
    case 10: return k_dspan<BITS, 10>;
    case 11: return k_dspan<BITS, 11>;
    case 12: return k_dspan<BITS, 12>;
    default: return nullptr;
  }
}

static inline DspanFn pick_dspan(int bits, uint32_t lgb) {
  switch (bits) {
    case 1: return pick_dspan_lgb<1>(lgb);
    case 2: return pick_dspan_lgb<2>(lgb);
    case 3: return pick_dspan_lgb<3>(lgb);
    case 4: return pick_dspan_lgb<4>(lgb);
    case 5: return pick_dspan_lgb<5>(lgb);
    case 6: return pick_dspan_lgb<6>(lgb);
    case 7: return pick_dspan_lgb<7>(lgb);
    case 8: return pick_dspan_lgb<8>(lgb);
    default: return nullptr;
  }
}

// K3 span decode of one tile of a piece (gcx_decode_pieces): as k_dspan with
// the bucket size a runtime property of the piece (one table entry per chunk,
// recomputed when the chunk starts a new bucket) and piece-relative offsets.
template <uint32_t BITS>
__device__ __forceinline__ void dspan_piece_tile(const gcx_piece& p, uint32_t start, uint32_t count,
                                                 const uint8_t* __restrict__ msg,
                                                 float* __restrict__ dst, float div, float recip,
                                                 bool pow2, uint32_t* words, uint32_t lane,
                                                 uint32_t c_lo = 0, uint32_t c_hi = 32) {
  constexpr uint32_t W = BITS + 1, S = (1u << BITS) - 1, F = 2u << BITS;
  constexpr uint32_t TW = 128u * W;
  const uint32_t f = lane & (F - 1u), level = f & S, sign = f >> BITS;
  const double dl = double(level);
  const double sd = double(S), ys = __drcp_rn(sd);
  const uint32_t qbit = 4 * W * lane, qw = qbit >> 5, qsh = qbit & 31u;
  const bool two = qsh + 4 * W > 32;
  const uint32_t lgb = 31 - __clz(p.bucket), bshift = lgb - 7;
  const bool full = count == kWTile;
  const uint32_t* src =
      reinterpret_cast<const uint32_t*>(msg + p.packed) + uint64_t(start >> 5) * W;
  const uint32_t nbk = uint32_t((p.len + p.bucket - 1) >> lgb);
  const uint32_t b0 = start >> lgb;
  const uint32_t nreg = lane < (kWTile >> lgb) && b0 + lane < nbk
                            ? __ldg(reinterpret_cast<const uint32_t*>(msg + p.norms) + b0 + lane)
                            : 0u;
  if (c_lo == 0 && c_hi == 32 && full && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
    uint4 st[W];
#pragma unroll
    for (uint32_t k = 0; k < W; ++k) st[k] = __ldcs(reinterpret_cast<const uint4*>(src) + k * 32 + lane);
#pragma unroll
    for (uint32_t k = 0; k < W; ++k) reinterpret_cast<uint4*>(words)[k * 32 + lane] = st[k];
  } else {  // the words of chunks [c_lo, c_hi) (a lane's window stays inside its chunk)
    const uint32_t nw = (count * W + 31) / 32;
    const uint32_t k1 = min(TW, c_hi * 4 * W);
    for (uint32_t k = c_lo * 4 * W + lane; k < k1; k += 32) words[k] = k < nw ? src[k] : 0u;
  }
  __syncwarp();
  float* out = dst + p.src + start + 4 * lane;
  const bool vec = full && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  if constexpr (F > 32) {  // widths 5-8: per-element values (wide_values)
#pragma unroll 4
    for (uint32_t c = c_lo; c < c_hi; ++c) {
      if (c * 128 >= count) break;
      const double nd = double(__uint_as_float(__shfl_sync(0xffffffffu, nreg, c >> bshift)));
      float v[4];
      wide_values<BITS>(lane_window(words + c * 4 * W + qw, qsh, two), nd, div, recip, pow2, v);
      float* o = out + c * 128;
      if (vec) {
        __stcs(reinterpret_cast<float4*>(o), make_float4(v[0], v[1], v[2], v[3]));
      } else {
        const uint32_t e = c * 128 + 4 * lane;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (e + k < count) __stcs(o + k, v[k]);
      }
    }
    __syncwarp();
    return;
  }
  // batches of 8 chunks: 8 independent FP64 chains for the batch's table
  // entries (one per chunk; chunks of one bucket compute the same entry),
  // then 8 chunks decoded by shuffles
#pragma unroll 1
  for (uint32_t c0 = c_lo; c0 < c_hi; c0 += 8) {
    if (c0 * 128 >= count) break;
    const uint32_t bb8 = c0;  // first chunk of the batch
    float entry[8];
#pragma unroll
    for (uint32_t cc = 0; cc < 8; ++cc) {
      const uint32_t nu = __shfl_sync(0xffffffffu, nreg, min(bb8 + cc, 31u) >> bshift);
      const double nl = __dmul_rn(double(__uint_as_float(nu)), dl);  // exact
      const double q0 = __dmul_rn(nl, ys);
      const double q = __fma_rn(__fma_rn(-sd, q0, nl), ys, q0);  // RN(nl / s), see dequant_field
      const float m = apply_divisor(__double2float_rn(q), div, recip, pow2);
      entry[cc] = level == 0 ? 0.0f : (sign ? -m : m);
    }
#pragma unroll
    for (uint32_t cc = 0; cc < 8; ++cc) {
      const uint32_t c = bb8 + cc;
      if (c >= c_hi || c * 128 >= count) break;
      const uint32_t* cw = words + c * 4 * W + qw;
      const uint32_t win = two ? __funnelshift_r(cw[0], cw[1], qsh) : (cw[0] >> qsh);
      float v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __shfl_sync(0xffffffffu, entry[cc], (win >> (k * W)) & (F - 1u));
      float* o = out + c * 128;
      if (vec) {
        __stcs(reinterpret_cast<float4*>(o), make_float4(v[0], v[1], v[2], v[3]));
      } else {
        const uint32_t e = c * 128 + 4 * lane;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (e + k < count) __stcs(o + k, v[k]);
      }
    }
  }
  __syncwarp();  // words[] is restaged by the next tile
}



// ---------------------------------------------------------------------------
// Fused SRA owner step, CTA per tile (k_span_fold_cta): the owner's chunk is
// 1/N of a buffer (476 tiles for ResNet-50 buffer 0 at N = 8), too few tiles
// for one warp per tile to hide the fold's latency, so the four warps of a CTA
// share each tile:
//   A  warp w folds rows 8w..8w+7 into the swizzled slots (fold_tile);
//   B  warp 0: the sequential FP64 norms, lane per row; warps 1-3 load keys;
//   C  warp w quantizes group w (elements [32w, 32w+32)) of every row;
//   D  the tile's packed words leave with one bulk store.
// ---------------------------------------------------------------------------
constexpr int kFoldWarps = 4;
#ifndef GCX_FOLD_MINB
#define GCX_FOLD_MINB 4  // resident CTAs per SM (registers <= 128): the owner chunk fits one wave
#endif

// FOLD = false is the same CTA-per-tile K1 fed from `src` (phase A stages
// rows 8w..8w+7 by coalesced loads): the small-message form of k_span_pieces,
// whose one-warp tiles leave a short table latency-bound (bucket 128 only).
#ifndef GCX_FOLD_PEER_MAJOR
#define GCX_FOLD_PEER_MAJOR 4  // node counts up to this take the peer-major fold (widths <= 4)
#endif
// The CTA owner step's fold (widths <= 4) peer-major: a warp's 8 rows
// (warp, warp + 4, ...), in two passes of 4, are folded one peer at a time in
// ascending node id (collectives.cpp:268-279; the owner's raw quads at id ==
// me), so a peer's receive slot is addressed once per pass, its 4 rows'
// norms and packed windows are loaded together (12 independent loads), and
// the next peer's loads are in flight while this peer is decoded.  Per row and peer: the
// lane's table entry (one FP64 dequant_field evaluation) and four shuffles.
template <uint32_t BITS, int LGB>
__device__ __forceinline__ void fold_rows_peer_major(const SpanPiecesArgs& A, const gcx_piece& p,
                                                     uint32_t start, uint32_t count, float* slots,
                                                     uint32_t lane, uint32_t warp) {
  constexpr uint32_t W = BITS + 1, S = (1u << BITS) - 1, F = 2u << BITS;
  constexpr uint32_t RB = 16u / kFoldWarps;  // rows per pass (two passes: 8 rows per warp)
  const uint32_t f = lane & (F - 1u), level = f & S, sign = f >> BITS;
  const double dl = double(level);
  const double sd = double(S), ys = __drcp_rn(sd);
  const uint32_t qbit = 4 * W * lane, qw = qbit >> 5, qsh = qbit & 31u;
  const bool two = qsh + 4 * W > 32;
  const uint32_t nodes = A.nodes, me = A.me;
  struct PeerLoads {
    uint32_t nu[RB], w0[RB], w1[RB];
  };
#pragma unroll 1
  for (uint32_t half = 0; half < 2; ++half) {
  const uint32_t w0r = warp + half * RB * kFoldWarps;  // this pass's first row
  auto vrow = [&](uint32_t j) {
    const uint32_t r = w0r + j * kFoldWarps;
    return count > r * 128u ? min(128u, count - r * 128u) : 0u;
  };
  auto load_peer = [&](uint32_t id, PeerLoads& L) {
    const uint8_t* m = A.recv + uint64_t(id < me ? id : id - 1) * A.slot_stride;
    const uint32_t* nb = reinterpret_cast<const uint32_t*>(m + p.norms);
    const uint32_t* wb = reinterpret_cast<const uint32_t*>(m + p.packed) + qw;
#pragma unroll
    for (uint32_t j = 0; j < RB; ++j) {
      const uint32_t vr = vrow(j);
      const uint32_t e_row = start + (w0r + j * kFoldWarps) * 128u;
      L.nu[j] = vr > 0 ? __ldg(nb + (e_row >> LGB)) : 0u;
      const bool quad = 4 * lane < vr;
      L.w0[j] = quad ? __ldg(wb + (e_row >> 5) * W) : 0u;
      L.w1[j] = quad && two ? __ldg(wb + (e_row >> 5) * W + 1) : 0u;
    }
  };
  float acc[RB][4];
  PeerLoads cur, nxt;
  const uint32_t first = me == 0 ? 1u : 0u;
  load_peer(first, cur);
#pragma unroll
  for (uint32_t id = 0; id < 8; ++id) {
    if (id >= nodes) break;
    if (id == me) {  // the owner's raw values
#pragma unroll
      for (uint32_t j = 0; j < RB; ++j) {
        const uint32_t vr = vrow(j);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (4 * lane < vr) {
          const float* o = A.src + p.src + start + (w0r + j * kFoldWarps) * 128u + 4 * lane;
          if (4 * lane + 4 <= vr && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
            v = __ldg(reinterpret_cast<const float4*>(o));
          } else {
            v.x = __ldg(o);
            if (4 * lane + 1 < vr) v.y = __ldg(o + 1);
            if (4 * lane + 2 < vr) v.z = __ldg(o + 2);
            if (4 * lane + 3 < vr) v.w = __ldg(o + 3);
          }
        }
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[j][k] = id == 0 ? x[k] : __fadd_rn(acc[j][k], x[k]);
      }
      continue;
    }
    const uint32_t nid = id + 1 == me ? id + 2 : id + 1;
    if (nid < nodes) load_peer(nid, nxt);
#pragma unroll
    for (uint32_t j = 0; j < RB; ++j) {
      // this lane's entry of the peer's table for row j's bucket (dequant_field)
      const double nl = __dmul_rn(double(__uint_as_float(cur.nu[j])), dl);  // exact
      const double q0 = __dmul_rn(nl, ys);
      const double q = __fma_rn(__fma_rn(-sd, q0, nl), ys, q0);
      const float mg = __double2float_rn(q);
      const float entry = level == 0 ? 0.0f : (sign ? -mg : mg);
      const uint32_t win = two ? __funnelshift_r(cur.w0[j], cur.w1[j], qsh) : (cur.w0[j] >> qsh);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = __shfl_sync(0xffffffffu, entry, (win >> (k * W)) & (F - 1u));
        acc[j][k] = id == 0 ? x : __fadd_rn(acc[j][k], x);
      }
    }
    cur = nxt;
  }
#pragma unroll
  for (uint32_t j = 0; j < RB; ++j) {
    const uint32_t r = w0r + j * kFoldWarps, vr = vrow(j);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (4 * lane + k >= vr) acc[j][k] = 0.0f;  // past the piece: the zero-filled tile
    float* dst = slots + (lane >> 3) * kSlotFloats + r * 32u + (((lane & 7u) ^ (r & 7u)) << 2);
    *reinterpret_cast<float4*>(dst) = make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
  }
  }  // half
}

template <uint32_t BITS, int LGB, int KM, bool FOLD, bool PM = false>
__global__ void __launch_bounds__(32 * kFoldWarps, GCX_FOLD_MINB) k_span_fold_cta(SpanPiecesArgs A) {
  constexpr uint32_t W = BITS + 1;
  extern __shared__ __align__(1024) unsigned char span_smem[];
  float* slots = reinterpret_cast<float*>(span_smem);                       // 4 x 4 KB
  uint32_t* outw = reinterpret_cast<uint32_t*>(span_smem + 4 * kSlotFloats * 4);  // 128 W
  uint32_t* nus = outw + out_words(W);                                      // 32 norms
  uint32_t* cars = nus + 32;                                                 // 32 flags
  __shared__ gcx_plan::TileCtx ctx_s;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const HashK shk = make_hashk();
  for (uint32_t t = blockIdx.x; t < A.pv.ntiles; t += gridDim.x) {
    if (warp == 0) {
      gcx_plan::TileCtx c;
      gcx_plan::locate_warp(A.pv, t, c);
      if (lane == 0) ctx_s = c;
    }
    __syncthreads();
    const gcx_plan::TileCtx cur = ctx_s;
    const gcx_piece& p = cur.p;
    if (p.bits == 0 && !FOLD) {  // raw piece: its f32 values are the payload
      raw_copy(A.src + p.src + cur.start, reinterpret_cast<float*>(A.msg + p.norms) + cur.start,
               cur.count, 1.0f, 1.0f, true, threadIdx.x, 32 * kFoldWarps);
      __syncthreads();
      continue;
    }
    if (p.bits == 0) {  // raw piece: the raw fold, ascending id (collectives.cpp:268-279)
      const float* xs = A.src + p.src + cur.start;
      float* d = reinterpret_cast<float*>(A.msg + p.norms) + cur.start;
#pragma unroll 4
      for (uint32_t e = threadIdx.x; e < cur.count; e += 32 * kFoldWarps) {
        float acc = 0.0f;
        for (uint32_t id = 0; id < A.nodes; ++id) {
          const float x =
              id == A.me ? __ldg(xs + e)
                         : __ldg(reinterpret_cast<const float*>(
                               A.recv + uint64_t(id < A.me ? id : id - 1) * A.slot_stride + p.norms) +
                               cur.start + e);
          acc = id == 0 ? x : __fadd_rn(acc, x);
        }
        d[e] = acc;
      }
      __syncthreads();
      continue;
    }
    const uint64_t seed = (A.flags & GCX_F_PIECE_SEEDS) ? p.seed : launch_seed(A);
    const uint32_t s_lo = uint32_t(seed), s_hi = uint32_t(seed >> 32);
    // A: fold (or stage) rows 8w..8w+7
    if constexpr (FOLD) {
      // rows warp, warp+4, ...: a short tile's rows spread over all four warps
      // PM (few peers, widths <= 4): peer-major; else the row-major fold with
      // its one-row-ahead loads (faster at N = 8)
      if constexpr (PM && (2u << BITS) <= 32)
        fold_rows_peer_major<BITS, LGB>(A, p, cur.start, cur.count, slots, lane, warp);
      else
        fold_tile<BITS, LGB>(A, p, cur.start, cur.count, slots, lane, warp, 32, kFoldWarps);
    } else {
      const float* xs = A.src + p.src + cur.start;
      const bool al = (reinterpret_cast<uintptr_t>(A.src + p.src) & 15u) == 0;
#pragma unroll
      for (uint32_t r = warp; r < 32; r += kFoldWarps) {  // rows spread over the warps
        const uint32_t e = r * 128u + 4 * lane;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e + 4 <= cur.count && al) {
          v = __ldcs(reinterpret_cast<const float4*>(xs + e));
        } else {
          if (e < cur.count) v.x = xs[e];
          if (e + 1 < cur.count) v.y = xs[e + 1];
          if (e + 2 < cur.count) v.z = xs[e + 2];
          if (e + 3 < cur.count) v.w = xs[e + 3];
        }
        *reinterpret_cast<float4*>(slots + (lane >> 3) * kSlotFloats + r * 32u +
                                   (((lane & 7u) ^ (r & 7u)) << 2)) = v;
      }
    }
    __syncthreads();
    RowView rv;
#pragma unroll
    for (uint32_t g = 0; g < 4; ++g) rv.slot[g] = slots + g * kSlotFloats;
    rv.r = lane;
    const uint32_t i_lane = cur.start + lane * kSpan;
    // B: norms (warp 0), keys (every warp, its group)
    uint4 kh[8], kl[8];
    const uint4* kg = KM != kKmInline ? reinterpret_cast<const uint4*>(A.keys) +
                                            ((p.keys + cur.start) >> 12) * 2048 + warp * 512 + lane
                                      : nullptr;
    if (KM != kKmInline) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        kh[q] = __ldg(kg + q * 32);
        if (KM == kKmPrefix) kl[q] = __ldg(kg + 256 + q * 32);
      }
    }
    if (warp == 0) {
      uint32_t v;
      bool c;
      if constexpr (LGB > 7) {  // a bucket spans rows: its first lane sums them
        uint32_t fb;
        span_pass1_big<LGB>(rv, lane, v, c, fb);
        if ((lane & ((1u << (LGB - 7)) - 1u)) == 0) {
          if (fb != ~0u && A.bad != nullptr)
            atomicMin(A.bad, (uint64_t(cur.pidx) << 40) | (i_lane + fb));
          if (i_lane < p.len) reinterpret_cast<uint32_t*>(A.msg + p.norms)[i_lane >> LGB] = v;
        }
      } else {
        double sq = 0.0;
#pragma unroll
        for (uint32_t g = 0; g < 4; ++g) {
          const float* row = rv.slot[g] + lane * 32u;
#pragma unroll
          for (uint32_t q = 0; q < 8; ++q) {
            const float4 x = *reinterpret_cast<const float4*>(row + ((q ^ (lane & 7u)) << 2));
            double d = double(x.x);
            sq = __fma_rn(d, d, sq);
            d = double(x.y);
            sq = __fma_rn(d, d, sq);
            d = double(x.z);
            sq = __fma_rn(d, d, sq);
            d = double(x.w);
            sq = __fma_rn(d, d, sq);
          }
        }
        c = (uint32_t(__double2hiint(sq)) & 0x7FF00000u) == 0x7FF00000u;
        if (c) {
          v = span_norm_exact(rv, 0, 128, 0u, nullptr);
          if (A.bad != nullptr)
            for (uint32_t e = 0; e < 128; ++e)
              if ((__float_as_uint(rv.at(e)) & 0x7FFFFFFFu) >= 0x7F800000u) {
                atomicMin(A.bad, (uint64_t(cur.pidx) << 40) | (i_lane + e));
                break;
              }
        } else {
          v = __float_as_uint(__double2float_rn(__dsqrt_rn(sq)));
        }
        if (i_lane < p.len) reinterpret_cast<uint32_t*>(A.msg + p.norms)[i_lane >> 7] = v;
      }
      nus[lane] = v;
      cars[lane] = c ? 1u : 0u;
      if (lane == 0) bulk_wait_read0();  // the previous tile's bulk store has read outw
    }
    __syncthreads();
    // C: group `warp` of every row
    {
      const uint32_t g = warp;
      const uint32_t nug = nus[lane];
      const bool car = cars[lane] != 0u;
      const uint32_t i0 = i_lane + g * 32;
      uint32_t* wout = outw + (lane * 4 + g) * W;
      uint32_t w[W];
      const bool ok = span_group_fast<BITS, LGB, KM>(rv.slot[g], lane, i0, nug, s_lo, s_hi, shk, w, kh,
                                                   kl, nullptr) &&
                      nug != 0u && !car;
      if (ok) {
#pragma unroll
        for (int m = 0; m < int(W); ++m) wout[m] = w[m];
      } else {
        span_group_exact<BITS, LGB, KM>(
            rv, g, i0, nug, seed,
            KM != kKmInline ? A.keys + ((p.keys + cur.start) >> 12) * 8192u : nullptr, lane, wout);
      }
    }
    __syncthreads();
    // D: the packed words
    uint32_t* dstw = reinterpret_cast<uint32_t*>(A.msg + p.packed) + uint64_t(cur.start >> 5) * W;
    if (cur.count == kWTile && (reinterpret_cast<uintptr_t>(dstw) & 15u) == 0) {
      if (threadIdx.x == 0) {
        fence_async_smem();
        bulk_s2g(dstw, outw, out_words(W) * 4);
      }
    } else {
      const uint32_t nwords = (cur.count * W + 31) / 32;
      for (uint32_t e = threadIdx.x; e < nwords; e += 32 * kFoldWarps) dstw[e] = outw[e];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) bulk_wait0();
}

}  // namespace gcx_span
