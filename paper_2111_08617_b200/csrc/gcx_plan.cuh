// gcx_plan.cuh — tile decomposition of a piece table (gcx_plan_tiles), shared
// by the kernels of gcx_kernels.cu and gcx_span.cu.
#pragma once

#include <cstdint>

#include "gcx.h"

namespace gcx_plan {

constexpr uint32_t kTile = GCX_TILE;
constexpr uint32_t kMaxBuckets = 256;  // buckets per tile

__host__ __device__ __forceinline__ uint32_t tile_elems(const gcx_piece& p) {
  if (p.bits == 0 || p.bucket > kTile) return kTile;
  uint32_t nb = kTile / p.bucket;
  if (nb > kMaxBuckets) nb = kMaxBuckets;
  return nb * p.bucket;
}

struct PlanView {
  const gcx_piece* pieces;  // device table or nullptr (then `one`)
  const uint32_t* prefix;
  uint32_t npieces;
  uint32_t ntiles;
  gcx_piece one;
};

struct TileCtx {
  gcx_piece p;
  uint32_t pidx;
  uint32_t start;  // piece-local first element of the tile (pieces < 2^32)
  uint32_t count;  // elements in the tile
};

// Tile -> (piece, first element).  The piece containing tile t is found by a
// warp-wide search of the tile prefix: 32 probes per step, so a table of P
// pieces takes ceil(log32 P) dependent loads instead of log2 P.  Call with
// all 32 lanes of one warp; every lane gets the result.
__device__ __forceinline__ void locate_warp(const PlanView& pv, uint32_t t, TileCtx& c) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t k;
  if (pv.pieces == nullptr) {
    c.p = pv.one;
    c.pidx = 0;
    k = t;
  } else {
    uint32_t lo = 0, hi = pv.npieces;  // prefix[lo] <= t < prefix[hi]
    while (hi - lo > 1) {
      const uint32_t span = hi - lo;
      const uint32_t step = (span + 31) / 32;
      const uint32_t probe = min(lo + lane * step, hi - 1);
      const bool le = __ldg(pv.prefix + probe) <= t;
      const uint32_t ballot = __ballot_sync(0xffffffffu, le);
      // probes are increasing; the last lane with prefix <= t bounds the piece
      const int last = 31 - __clz(ballot);
      const uint32_t nlo = min(lo + uint32_t(last) * step, hi - 1);
      hi = min(hi, nlo + step);
      lo = nlo;
    }
    c.p = pv.pieces[lo];
    c.pidx = lo;
    k = t - __ldg(pv.prefix + lo);
  }
  const uint32_t T = tile_elems(c.p);
  c.start = k * T;
  const uint64_t rem = c.p.len - c.start;
  c.count = rem < T ? uint32_t(rem) : T;
}

// Span key layout (prefix and key tables of the span K1 kernels): slot t of
// a run (runs start on multiples of 4096 slots) = element t of a piece; with
// tile T = t >> 12, row r = (t >> 7) & 31, quad q = (t >> 2) & 31, k = t & 3,
// its high word sits in block b = 4T + q/8 (2048 words: 1024 high words, then
// the 1024 low words) at (q % 8) * 128 + r * 4 + k.  Blocks of 1024 slots with
// high words first are also the lane-group layout's (key_pos), so slot-wise
// passes (gcx_make_keys_prefixed) serve both.
__host__ __device__ __forceinline__ uint64_t span_key_pos(uint64_t t) {
  const uint64_t q = (t >> 2) & 31u;
  return (((t >> 12) * 4 + (q >> 3)) << 11) | ((q & 7u) << 7) | (((t >> 7) & 31u) << 2) | (t & 3u);
}
// inverse for a high-word position u (u & 2047 < 1024)
__host__ __device__ __forceinline__ uint64_t span_key_slot(uint64_t u) {
  const uint64_t blk = u >> 11, w = u & 1023u;
  const uint64_t q = (blk & 3u) * 8 + (w >> 7);
  return ((blk >> 2) << 12) | (((w >> 2) & 31u) << 7) | (q << 2) | (w & 3u);
}

}  // namespace gcx_plan
