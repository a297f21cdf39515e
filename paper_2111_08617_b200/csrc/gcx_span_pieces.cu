// gcx_span_pieces.cu — host launchers of the piece-table span K1, the
// CTA-per-tile K1 for short tables and the fused SRA owner step
// (kernels in gcx_span_dev.cuh; C-ABI routing in gcx_kernels.cu).
#include <cuda_runtime.h>

#include <cstdint>

#include "gcx_span.h"
#include "gcx_span_dev.cuh"

using namespace gcx_span;

using SpanPiecesFn = void (*)(SpanPiecesArgs);

template <uint32_t BITS, int LGB>
SpanPiecesFn pick_pieces_km(int km) {
  switch (km) {
    case kKmTable: return k_span_pieces<BITS, LGB, kKmTable, false>;
    case kKmPrefix: return k_span_pieces<BITS, LGB, kKmPrefix, false>;
    default: return k_span_pieces<BITS, LGB, kKmInline, false>;
  }
}

#ifndef GCX_FOLD_CTA
#define GCX_FOLD_CTA 1  // the fused owner step: 1 = CTA per tile, 0 = warp per tile
#endif
template <int LGB>
static SpanPiecesFn pick_fold_lgb(int bits, bool prefix) {
  if (GCX_FOLD_CTA) {
    switch (bits) {
      case 1: return prefix ? k_span_fold_cta<1, LGB, kKmPrefix, true> : k_span_fold_cta<1, LGB, kKmInline, true>;
      case 2: return prefix ? k_span_fold_cta<2, LGB, kKmPrefix, true> : k_span_fold_cta<2, LGB, kKmInline, true>;
      case 3: return prefix ? k_span_fold_cta<3, LGB, kKmPrefix, true> : k_span_fold_cta<3, LGB, kKmInline, true>;
      case 4: return prefix ? k_span_fold_cta<4, LGB, kKmPrefix, true> : k_span_fold_cta<4, LGB, kKmInline, true>;
      case 5: return prefix ? k_span_fold_cta<5, LGB, kKmPrefix, true> : k_span_fold_cta<5, LGB, kKmInline, true>;
      case 6: return prefix ? k_span_fold_cta<6, LGB, kKmPrefix, true> : k_span_fold_cta<6, LGB, kKmInline, true>;
      case 7: return prefix ? k_span_fold_cta<7, LGB, kKmPrefix, true> : k_span_fold_cta<7, LGB, kKmInline, true>;
      case 8: return prefix ? k_span_fold_cta<8, LGB, kKmPrefix, true> : k_span_fold_cta<8, LGB, kKmInline, true>;
      default: return nullptr;
    }
  }
  switch (bits) {
    case 1: return prefix ? k_span_pieces<1, LGB, kKmPrefix, true> : k_span_pieces<1, LGB, kKmInline, true>;
    case 2: return prefix ? k_span_pieces<2, LGB, kKmPrefix, true> : k_span_pieces<2, LGB, kKmInline, true>;
    case 3: return prefix ? k_span_pieces<3, LGB, kKmPrefix, true> : k_span_pieces<3, LGB, kKmInline, true>;
    case 4: return prefix ? k_span_pieces<4, LGB, kKmPrefix, true> : k_span_pieces<4, LGB, kKmInline, true>;
    default: return nullptr;
  }
}

// the peer-major fold (few peers, widths <= 4)
template <int LGB>
static SpanPiecesFn pick_fold_pm_lgb(int bits, bool prefix) {
  switch (bits) {
    case 1: return prefix ? k_span_fold_cta<1, LGB, kKmPrefix, true, true> : k_span_fold_cta<1, LGB, kKmInline, true, true>;
    case 2: return prefix ? k_span_fold_cta<2, LGB, kKmPrefix, true, true> : k_span_fold_cta<2, LGB, kKmInline, true, true>;
    case 3: return prefix ? k_span_fold_cta<3, LGB, kKmPrefix, true, true> : k_span_fold_cta<3, LGB, kKmInline, true, true>;
    case 4: return prefix ? k_span_fold_cta<4, LGB, kKmPrefix, true, true> : k_span_fold_cta<4, LGB, kKmInline, true, true>;
    default: return nullptr;
  }
}

static SpanPiecesFn pick_fold(int bits, int lgb, bool prefix, bool pm) {
  if (pm && GCX_FOLD_CTA && bits <= 4) {
    switch (lgb) {
      case 7: return pick_fold_pm_lgb<7>(bits, prefix);
      case 9: return pick_fold_pm_lgb<9>(bits, prefix);
      default: return nullptr;
    }
  }
  switch (lgb) {
    case 7: return pick_fold_lgb<7>(bits, prefix);
    case 9: return pick_fold_lgb<9>(bits, prefix);
    default: return nullptr;
  }
}

template <uint32_t BITS>
SpanPiecesFn pick_pieces_lgb(int lgb, int km) {
  switch (lgb) {
    case 5: return pick_pieces_km<BITS, 5>(km);
    case 6: return pick_pieces_km<BITS, 6>(km);
    case 7: return pick_pieces_km<BITS, 7>(km);
    case 9: return pick_pieces_km<BITS, 9>(km);
    default: return nullptr;
  }
}

static SpanPiecesFn pick_pieces(int bits, int lgb, int km) {
  switch (bits) {
    case 1: return pick_pieces_lgb<1>(lgb, km);
    case 2: return pick_pieces_lgb<2>(lgb, km);
    case 3: return pick_pieces_lgb<3>(lgb, km);
    case 4: return pick_pieces_lgb<4>(lgb, km);
    case 5: return pick_pieces_lgb<5>(lgb, km);
    case 6: return pick_pieces_lgb<6>(lgb, km);
    case 7: return pick_pieces_lgb<7>(lgb, km);
    case 8: return pick_pieces_lgb<8>(lgb, km);
    default: return nullptr;
  }
}


template <uint32_t BITS, int LGB>
static SpanPiecesFn pick_small_km(int km) {
  switch (km) {
    case kKmTable: return k_span_fold_cta<BITS, LGB, kKmTable, false>;
    case kKmPrefix: return k_span_fold_cta<BITS, LGB, kKmPrefix, false>;
    default: return k_span_fold_cta<BITS, LGB, kKmInline, false>;
  }
}

template <int LGB>
static SpanPiecesFn pick_small_lgb(int bits, int km) {
  switch (bits) {
    case 1: return pick_small_km<1, LGB>(km);
    case 2: return pick_small_km<2, LGB>(km);
    case 3: return pick_small_km<3, LGB>(km);
    case 4: return pick_small_km<4, LGB>(km);
    case 5: return pick_small_km<5, LGB>(km);
    case 6: return pick_small_km<6, LGB>(km);
    case 7: return pick_small_km<7, LGB>(km);
    case 8: return pick_small_km<8, LGB>(km);
    default: return nullptr;
  }
}

static SpanPiecesFn pick_small(int bits, int lgb, int km) {
  switch (lgb) {
    case 7: return pick_small_lgb<7>(bits, km);
    case 9: return pick_small_lgb<9>(bits, km);
    default: return nullptr;
  }
}

// K1 for short tables (a small message's chunks): a CTA of 4 warps per tile
static cudaError_t span_small_encode(const gcx_piece* pieces, const uint32_t* tile_prefix,
                                     uint32_t npieces, uint32_t ntiles, uint32_t flags,
                                     uint64_t seed, const float* src, uint8_t* msg,
                                     const unsigned long long* keys, unsigned long long* bad,
                                     int bits, int lgb, int km, int sms, cudaStream_t st) {
  SpanPiecesFn fn = pick_small(bits, lgb, km);
  if (fn == nullptr) return cudaErrorInvalidValue;
  const uint32_t W = uint32_t(bits) + 1;
  const size_t smem = size_t(4 * kSlotFloats * 4 + out_words(W) * 4 + 64 * 4);
  static thread_local bool cfg[9][13][3] = {};
  if (!cfg[bits][lgb][km]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    cfg[bits][lgb][km] = true;
  }
  SpanPiecesArgs a;
  a.pv = gcx_plan::PlanView{pieces, tile_prefix, npieces, ntiles, {}};
  a.flags = flags;
  a.seed = seed;
  a.seed_dev = (flags & GCX_F_SEED_DEVICE) ? reinterpret_cast<const unsigned long long*>(seed)
                                           : nullptr;
  a.src = src;
  a.msg = msg;
  a.keys = reinterpret_cast<const uint32_t*>(keys);
  a.bad = bad;
  a.recv = nullptr;
  a.slot_stride = 0;
  a.nodes = 0;
  a.me = 0;
  uint32_t grid = ntiles;
  if (grid > uint32_t(sms * GCX_FOLD_MINB)) grid = uint32_t(sms * GCX_FOLD_MINB);
  fn<<<grid > 0 ? grid : 1, 32 * kFoldWarps, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t gcx_span_encode_pieces(const gcx_piece* pieces, const uint32_t* tile_prefix,
                                   uint32_t npieces, uint32_t ntiles, uint32_t flags, uint64_t seed,
                                   const float* src, uint8_t* msg, const unsigned long long* keys,
                                   unsigned long long* bad, int sms, cudaStream_t st) {
  const int bits = int((flags >> GCX_F_SPAN_BITS_SHIFT) & 15u);
  const int lgb = int((flags >> GCX_F_SPAN_LGB_SHIFT) & 15u);
  const int km = keys == nullptr ? kKmInline : (flags & GCX_F_KEY_PREFIX) ? kKmPrefix : kKmTable;
  if ((lgb == 7 || lgb == 9) && ntiles <= uint32_t(sms) * GCX_SMALL_TILES_PER_SM)
    return span_small_encode(pieces, tile_prefix, npieces, ntiles, flags, seed, src, msg, keys, bad,
                             bits, lgb, km, sms, st);
  SpanPiecesFn fn = pick_pieces(bits, lgb, km);
  if (fn == nullptr) return cudaErrorInvalidValue;
  const size_t smem = size_t(kWarps) * warp_smem_bytes(uint32_t(bits) + 1);
  static thread_local int occ[9][8][3] = {};
  int& o = occ[bits][lgb][km];
  if (o == 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 32 * kWarps, smem);
    if (e != cudaSuccess) return e;
    if (o < 1) o = 1;
  }
  SpanPiecesArgs a;
  a.pv = gcx_plan::PlanView{pieces, tile_prefix, npieces, ntiles, {}};
  a.flags = flags;
  a.seed = seed;
  a.seed_dev = (flags & GCX_F_SEED_DEVICE) ? reinterpret_cast<const unsigned long long*>(seed)
                                           : nullptr;
  a.src = src;
  a.msg = msg;
  a.keys = reinterpret_cast<const uint32_t*>(keys);
  a.bad = bad;
  a.recv = nullptr;
  a.slot_stride = 0;
  a.nodes = 0;
  a.me = 0;
  uint32_t grid = (ntiles + kWarps - 1) / kWarps;
  if (grid > uint32_t(sms * o)) grid = uint32_t(sms * o);
  if (grid == 0) grid = 1;
  fn<<<grid, 32 * kWarps, smem, st>>>(a);
  return cudaGetLastError();
}

bool gcx_span_fold_ok(uint32_t flags, uint32_t nodes) {
  const uint32_t bits = (flags >> GCX_F_SPAN_BITS_SHIFT) & 15u;
  const uint32_t lgb = (flags >> GCX_F_SPAN_LGB_SHIFT) & 15u;
  return (flags & GCX_F_SPAN_ENC) && bits >= 1 && bits <= 8 && (lgb == 7 || lgb == 9) && nodes >= 2 &&
         nodes <= 8;
}

cudaError_t gcx_span_fold_encode(const gcx_piece* pieces, const uint32_t* tile_prefix,
                                 uint32_t npieces, uint32_t ntiles, uint32_t flags,
                                 const uint8_t* recv, uint64_t slot_stride, const float* own,
                                 uint32_t nodes, uint32_t me, uint64_t seed, uint8_t* bcast,
                                 const unsigned long long* prefix, unsigned long long* bad, int sms,
                                 cudaStream_t st) {
  if (!gcx_span_fold_ok(flags, nodes) || me >= nodes) return cudaErrorInvalidValue;
  const int bits = int((flags >> GCX_F_SPAN_BITS_SHIFT) & 15u);
  const int lgb = int((flags >> GCX_F_SPAN_LGB_SHIFT) & 15u);
  const bool pm = nodes <= GCX_FOLD_PEER_MAJOR && bits <= 4;
  SpanPiecesFn fn = pick_fold(bits, lgb, prefix != nullptr, pm);
  if (fn == nullptr) return cudaErrorInvalidValue;
  const uint32_t W = uint32_t(bits) + 1;
  const size_t smem = GCX_FOLD_CTA ? size_t(4 * kSlotFloats * 4 + out_words(W) * 4 + 64 * 4)
                                   : size_t(kWarps) * warp_smem_bytes(W);
  const int threads = GCX_FOLD_CTA ? 32 * kFoldWarps : 32 * kWarps;
  static thread_local int occ[9][13][2][2] = {};
  int& o = occ[bits][lgb][prefix != nullptr][pm];
  if (o == 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem);
    if (e != cudaSuccess) return e;
    if (o < 1) o = 1;
  }
  SpanPiecesArgs a;
  a.pv = gcx_plan::PlanView{pieces, tile_prefix, npieces, ntiles, {}};
  a.flags = flags | (prefix != nullptr ? GCX_F_KEY_PREFIX : 0u);
  a.seed = seed;
  a.seed_dev = (flags & GCX_F_SEED_DEVICE) ? reinterpret_cast<const unsigned long long*>(seed)
                                           : nullptr;
  a.src = own;
  a.msg = bcast;
  a.keys = reinterpret_cast<const uint32_t*>(prefix);
  a.bad = bad;
  a.recv = recv;
  a.slot_stride = slot_stride;
  a.nodes = nodes;
  a.me = me;
  uint32_t grid = GCX_FOLD_CTA ? ntiles : (ntiles + kWarps - 1) / kWarps;
  if (grid > uint32_t(sms * o)) grid = uint32_t(sms * o);
  if (grid == 0) grid = 1;
  fn<<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

