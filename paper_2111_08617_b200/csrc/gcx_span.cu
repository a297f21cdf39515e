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

#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "gcx_span.h"
#include "gcx_span_dev.cuh"

namespace gcx_span {

__global__ void __launch_bounds__(256) k_span_prefix(uint32_t n, uint32_t lgb, uint32_t ntiles,
                                                     uint4* __restrict__ table) {
  // thread per 4 consecutive high-word positions (one uint4 of highs, one of lows)
  const uint64_t total = uint64_t(ntiles) * 1024u;  // uint4 of high words
  for (uint64_t u = blockIdx.x * 256ull + threadIdx.x; u < total; u += uint64_t(gridDim.x) * 256u) {
    const uint64_t pos = ((u >> 8) << 11) | ((u & 255u) << 2);  // first high word of the uint4
    const uint64_t t0 = span_key_slot(pos);
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = t0 + k;
      const uint64_t z = i < n ? mix64h(uint64_t(i >> lgb) ^ mix64h(i)) : 0ull;
      hi[k] = uint32_t(z >> 32);
      lo[k] = uint32_t(z);
    }
    table[pos >> 2] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    table[(pos >> 2) + 256] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// WIDE: some piece has widths 5-8 (GCX_F_SPAN_DEC_WIDE; 9-word chunks)
// A work item is 1/2^lgs of a tile (chunks [c_lo, c_hi)): when the table has
// about one tile per warp, a tile's decode is a chain of dependent latencies
// (locate, stage, 32 chunks) that splitting shortens.
template <bool WIDE>
__global__ void __launch_bounds__(32 * kDWarps) k_dspan_pieces(gcx_plan::PlanView pv,
                                                               const uint8_t* __restrict__ msg,
                                                               float* __restrict__ dst, float div,
                                                               float recip, bool pow2, uint32_t lgs) {
  __shared__ __align__(16) uint32_t words_all[kDWarps][128 * (WIDE ? 9 : 5)];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t* words = words_all[warp];
  const uint32_t nw = gridDim.x * kDWarps, nitems = pv.ntiles << lgs, cp = 32u >> lgs;
  for (uint32_t u = blockIdx.x * kDWarps + warp; u < nitems; u += nw) {
    gcx_plan::TileCtx c;
    gcx_plan::locate_warp(pv, u >> lgs, c);
    const gcx_piece& p = c.p;
    const uint32_t c_lo = (u & ((1u << lgs) - 1u)) * cp, c_hi = c_lo + cp;
    if (c_lo * 128u >= c.count) continue;
    switch (p.bits) {
      case 0: {  // raw piece: f32 payload at p.norms, divided (finalize's average)
        const uint32_t e0 = c.start + c_lo * 128u;
        raw_copy(reinterpret_cast<const float*>(msg + p.norms) + e0, dst + p.src + e0,
                 min(c.count - c_lo * 128u, cp * 128u), div, recip, pow2, lane, 32);
        break;
      }
#define GCX_DSPAN_CASE(B) \
      case B: dspan_piece_tile<B>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      GCX_DSPAN_CASE(1)
      GCX_DSPAN_CASE(2)
      GCX_DSPAN_CASE(3)
      GCX_DSPAN_CASE(4)
#undef GCX_DSPAN_CASE
#define GCX_DSPAN_CASE(B) \
      case B: if constexpr (WIDE) dspan_piece_tile<B>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      GCX_DSPAN_CASE(5)
      GCX_DSPAN_CASE(6)
      GCX_DSPAN_CASE(7)
      GCX_DSPAN_CASE(8)
#undef GCX_DSPAN_CASE
      default: break;
    }
  }
}

// Short tables (a small message): a CTA of 8 warps per tile, warp w decoding
// chunks 4w..4w+3, so one tile's latency is an eighth of a warp's.
template <bool WIDE>
__global__ void __launch_bounds__(32 * kDWarps) k_dspan_pieces_small(gcx_plan::PlanView pv,
                                                                     const uint8_t* __restrict__ msg,
                                                                     float* __restrict__ dst,
                                                                     float div, float recip,
                                                                     bool pow2) {
  __shared__ __align__(16) uint32_t words[128 * (WIDE ? 9 : 5) + 4];
  __shared__ gcx_plan::TileCtx ctx_s;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint32_t t = blockIdx.x; t < pv.ntiles; t += gridDim.x) {
    if (warp == 0) {
      gcx_plan::TileCtx c;
      gcx_plan::locate_warp(pv, t, c);
      if (lane == 0) ctx_s = c;
    }
    __syncthreads();
    const gcx_plan::TileCtx c = ctx_s;
    const gcx_piece& p = c.p;
    const uint32_t c_lo = 4 * warp, c_hi = 4 * warp + 4;
    switch (p.bits) {
      case 0:
        raw_copy(reinterpret_cast<const float*>(msg + p.norms) + c.start, dst + p.src + c.start,
                 c.count, div, recip, pow2, threadIdx.x, 32 * kDWarps);
        break;
      case 1: dspan_piece_tile<1>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      case 2: dspan_piece_tile<2>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      case 3: dspan_piece_tile<3>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      case 4: dspan_piece_tile<4>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      case 5: if constexpr (WIDE) dspan_piece_tile<5>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      case 6: if constexpr (WIDE) dspan_piece_tile<6>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      case 7: if constexpr (WIDE) dspan_piece_tile<7>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      case 8: if constexpr (WIDE) dspan_piece_tile<8>(p, c.start, c.count, msg, dst, div, recip, pow2, words, lane, c_lo, c_hi); break;
      default: break;
    }
    __syncthreads();
  }
}

using SpanFn = void (*)(const __grid_constant__ CUtensorMap, SpanArgs);

template <uint32_t BITS>
SpanFn pick_lgb(int lgb, bool prefix) {
  switch (lgb) {
    case 5: return prefix ? k_span<BITS, 5, true> : k_span<BITS, 5, false>;
    case 6: return prefix ? k_span<BITS, 6, true> : k_span<BITS, 6, false>;
    case 7: return prefix ? k_span<BITS, 7, true> : k_span<BITS, 7, false>;
    case 9: return prefix ? k_span<BITS, 9, true> : k_span<BITS, 9, false>;
    default: return nullptr;
  }
}

SpanFn pick(int bits, int lgb, bool prefix) {
  switch (bits) {
    case 1: return pick_lgb<1>(lgb, prefix);
    case 2: return pick_lgb<2>(lgb, prefix);
    case 3: return pick_lgb<3>(lgb, prefix);
    case 4: return pick_lgb<4>(lgb, prefix);
    case 5: return pick_lgb<5>(lgb, prefix);
    case 6: return pick_lgb<6>(lgb, prefix);
    case 7: return pick_lgb<7>(lgb, prefix);
    case 8: return pick_lgb<8>(lgb, prefix);
    default: return nullptr;
  }
}

int lgb_of(uint64_t bucket) {
  return bucket == 32 ? 5 : bucket == 64 ? 6 : bucket == 128 ? 7 : bucket == 512 ? 9 : -1;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// The vector's full 128-element rows as a 2-D tensor {128, rows}; box {32, 32}
// = one quarter of a warp tile, 128-byte swizzle.
bool make_tmap(const float* x, uint64_t rows, CUtensorMap* map) {
  EncodeFn fn = encode_fn();
  if (fn == nullptr || rows == 0) return false;
  const cuuint64_t dims[2] = {kSpan, rows};
  const cuuint64_t strides[1] = {kSpan * 4};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace gcx_span


using namespace gcx_span;

bool gcx_span_supported(uint64_t bucket) { return lgb_of(bucket) > 0; }

uint64_t gcx_span_prefix_slots(uint64_t n) { return (n + kWTile - 1) / kWTile * kWTile; }

cudaError_t gcx_span_make_prefix(uint64_t n, uint64_t bucket, unsigned long long* table,
                                 int sms, cudaStream_t st) {
  const int lgb = lgb_of(bucket);
  if (lgb < 0) return cudaErrorInvalidValue;
  const uint32_t ntiles = uint32_t((n + kWTile - 1) / kWTile);
  const uint64_t threads = uint64_t(ntiles) * 1024u;
  const uint64_t blocks = (threads + 255) / 256;
  const uint32_t grid = uint32_t(blocks < uint64_t(sms) * 8 ? blocks : uint64_t(sms) * 8);
  k_span_prefix<<<grid > 0 ? grid : 1, 256, 0, st>>>(uint32_t(n), uint32_t(lgb), ntiles,
                                                      reinterpret_cast<uint4*>(table));
  return cudaGetLastError();
}

cudaError_t gcx_span_quantize(const float* x, uint64_t n, int bits, uint64_t bucket, uint64_t seed,
                              const unsigned long long* prefix, float* norms, uint8_t* packed,
                              unsigned long long* bad, int sms, cudaStream_t st) {
  const int lgb = lgb_of(bucket);
  SpanFn fn = pick(bits, lgb, prefix != nullptr);
  if (fn == nullptr) return cudaErrorInvalidValue;
  const uint32_t W = uint32_t(bits) + 1;
  const size_t smem = size_t(kWarps) * warp_smem_bytes(W);
  static thread_local int occ[9][8][2] = {};
  int& o = occ[bits][lgb][prefix != nullptr];
  if (o == 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 32 * kWarps, smem);
    if (e != cudaSuccess) return e;
    if (o < 1) o = 1;
  }
  SpanArgs a;
  a.x = x;
  a.n = uint32_t(n);
  a.nfull = uint32_t(n / kWTile);
  a.seed = seed;
  a.prefix = reinterpret_cast<const uint32_t*>(prefix);
  a.norms = norms;
  a.packed = reinterpret_cast<uint32_t*>(packed);
  a.bad = bad;
  a.p_al16 = (reinterpret_cast<uintptr_t>(packed) & 15u) == 0;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  a.tma = (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && a.nfull > 0 &&
          make_tmap(x, uint64_t(a.nfull) * 32, &map);
  const uint32_t tiles = uint32_t((n + kWTile - 1) / kWTile);
  uint32_t grid = (tiles + kWarps - 1) / kWarps;
  if (grid > uint32_t(sms * o)) grid = uint32_t(sms * o);
  if (grid == 0) grid = 1;
  fn<<<grid, 32 * kWarps, smem, st>>>(map, a);
  return cudaGetLastError();
}

bool gcx_span_decode_supported(int bits, uint64_t bucket) {
  return bits >= 1 && bits <= 8 && bucket >= 128 && bucket <= kWTile && (bucket & (bucket - 1)) == 0;
}

cudaError_t gcx_span_dequantize(const float* norms, const uint8_t* packed, uint64_t n, int bits,
                                uint64_t bucket, float* out, float divisor, int sms,
                                cudaStream_t st) {
  if (!gcx_span_decode_supported(bits, bucket)) return cudaErrorInvalidValue;
  if (reinterpret_cast<uintptr_t>(packed) & 15u) return cudaErrorInvalidValue;
  uint32_t lgb = 0;
  while ((1ull << lgb) < bucket) ++lgb;
  DspanFn fn = pick_dspan(bits, lgb);
  if (fn == nullptr) return cudaErrorInvalidValue;
  static thread_local int occ[9][13] = {};
  int& o = occ[bits][lgb];
  if (o == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 32 * kDWarps, 0);
    if (e != cudaSuccess) return e;
    if (o < 1) o = 1;
  }
  DspanArgs a;
  a.norms = norms;
  a.packed = reinterpret_cast<const uint32_t*>(packed);
  a.out = out;
  a.n = uint32_t(n);
  a.div = divisor;
  a.recip = 1.0f / divisor;
  int e2 = 0;
  a.pow2 = std::frexp(divisor, &e2) == 0.5f;
  const uint32_t tiles = uint32_t((n + kWTile - 1) / kWTile);
  uint32_t grid = (tiles + kDWarps - 1) / kDWarps;
  if (grid > uint32_t(sms * o)) grid = uint32_t(sms * o);
  if (grid == 0) grid = 1;
  fn<<<grid, 32 * kDWarps, 0, st>>>(a);
  return cudaGetLastError();
}

bool gcx_span_decode_piece_ok(int bits, uint64_t bucket) {
  return bits == 0 || gcx_span_decode_supported(bits, bucket);
}

cudaError_t gcx_span_decode_pieces(const gcx_piece* pieces, const uint32_t* tile_prefix,
                                   uint32_t npieces, uint32_t ntiles, const uint8_t* msg,
                                   float* dst, float divisor, bool wide, int sms, cudaStream_t st) {
  static thread_local int occ[2] = {0, 0};
  int& o = occ[wide];
  if (o == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &o, wide ? k_dspan_pieces<true> : k_dspan_pieces<false>, 32 * kDWarps, 0);
    if (e != cudaSuccess) return e;
    if (o < 1) o = 1;
  }
  gcx_plan::PlanView pv{pieces, tile_prefix, npieces, ntiles, {}};
  int e2 = 0;
  const bool pow2 = std::frexp(divisor, &e2) == 0.5f;
  if (ntiles <= uint32_t(sms) * GCX_SMALL_TILES_PER_SM) {  // short table: CTA per tile
    auto fn = wide ? k_dspan_pieces_small<true> : k_dspan_pieces_small<false>;
    fn<<<ntiles, 32 * kDWarps, 0, st>>>(pv, msg, dst, divisor, 1.0f / divisor, pow2);
    return cudaGetLastError();
  }
  // wide tables with fewer than 2 tiles per resident warp decode half tiles
  // (C3 8b/512 N = 8: -6 % per step); narrow tables measured no gain from
  // splitting (1/2/4/8 parts on C2 / C3 2b).  GCX_DSPAN_SPLIT=k forces 2^k
  // parts (measurement)
  const uint64_t slots = uint64_t(sms) * uint64_t(o) * kDWarps;
  uint32_t lgs = wide && uint64_t(ntiles) < 2 * slots ? 1u : 0u;
  static const int forced = [] {
    const char* e = std::getenv("GCX_DSPAN_SPLIT");
    return e != nullptr ? std::atoi(e) : -1;
  }();
  if (forced >= 0 && forced <= 3) lgs = uint32_t(forced);
  if ((uint64_t(ntiles) << lgs) > 0xFFFFFFFFull) lgs = 0;
  const uint64_t items = uint64_t(ntiles) << lgs;
  uint32_t grid = uint32_t((items + kDWarps - 1) / kDWarps);
  if (grid > uint32_t(sms * o)) grid = uint32_t(sms * o);
  if (grid == 0) grid = 1;
  auto fn = wide ? k_dspan_pieces<true> : k_dspan_pieces<false>;
  fn<<<grid, 32 * kDWarps, 0, st>>>(pv, msg, dst, divisor, 1.0f / divisor, pow2, lgs);
  return cudaGetLastError();
}

