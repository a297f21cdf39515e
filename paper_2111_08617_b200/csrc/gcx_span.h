// gcx_span.h — internal interface of the span K1 kernel (gcx_span.cu) used by
// the C-ABI in gcx_kernels.cu.  Not part of the public boundary (include/gcx.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "gcx.h"

// buckets the span kernel handles (32, 64, 128)
bool gcx_span_supported(uint64_t bucket);
// prefix-table slots (8 bytes each) of an n-element vector in span layout
uint64_t gcx_span_prefix_slots(uint64_t n);
cudaError_t gcx_span_make_prefix(uint64_t n, uint64_t bucket, unsigned long long* table, int sms,
                                 cudaStream_t st);
// prefix == nullptr: keys hashed inline (three SplitMix64 finalizers)
cudaError_t gcx_span_quantize(const float* x, uint64_t n, int bits, uint64_t bucket, uint64_t seed,
                              const unsigned long long* prefix, float* norms, uint8_t* packed,
                              unsigned long long* bad, int sms, cudaStream_t st);
// K3 span decode: bits 1..4, power-of-two buckets 128..4096; packed 16-byte aligned
bool gcx_span_decode_supported(int bits, uint64_t bucket);
cudaError_t gcx_span_dequantize(const float* norms, const uint8_t* packed, uint64_t n, int bits,
                                uint64_t bucket, float* out, float divisor, int sms,
                                cudaStream_t st);
// K3 span decode over a piece table whose pieces are all raw or
// span-decodable (gcx_plan_tiles sets GCX_F_SPAN_DEC); wide: some piece has
// widths 5-8 (GCX_F_SPAN_DEC_WIDE)
bool gcx_span_decode_piece_ok(int bits, uint64_t bucket);
cudaError_t gcx_span_decode_pieces(const gcx_piece* pieces, const uint32_t* tile_prefix,
                                   uint32_t npieces, uint32_t ntiles, const uint8_t* msg,
                                   float* dst, float divisor, bool wide, int sms, cudaStream_t st);
// K1 span over a piece table with GCX_F_SPAN_ENC (bits and log2 bucket in the
// flags); keys == nullptr: hashed inline; with GCX_F_KEY_PREFIX span-layout
// prefixes, else a span-layout key table for this seed
cudaError_t gcx_span_encode_pieces(const gcx_piece* pieces, const uint32_t* tile_prefix,
                                   uint32_t npieces, uint32_t ntiles, uint32_t flags, uint64_t seed,
                                   const float* src, uint8_t* msg, const unsigned long long* keys,
                                   unsigned long long* bad, int sms, cudaStream_t st);
// Fused SRA owner step, fold + hop-1 re-encode (GCX_F_SPAN_ENC tables with
// bits <= 4, bucket 128, 2 <= nodes <= 8); prefix: the table's span-layout key
// prefixes, or nullptr to hash inline
bool gcx_span_fold_ok(uint32_t flags, uint32_t nodes);
cudaError_t gcx_span_fold_encode(const gcx_piece* pieces, const uint32_t* tile_prefix,
                                 uint32_t npieces, uint32_t ntiles, uint32_t flags,
                                 const uint8_t* recv, uint64_t slot_stride, const float* own,
                                 uint32_t nodes, uint32_t me, uint64_t seed, uint8_t* bcast,
                                 const unsigned long long* prefix, unsigned long long* bad, int sms,
                                 cudaStream_t st);
