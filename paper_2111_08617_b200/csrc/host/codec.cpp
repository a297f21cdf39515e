// codec.cpp — gcomm::codec façade over gcx_quantize / gcx_dequantize.
// Reference: /root/reference/proj/src/codec.cpp (API and error behaviour).
// quantize/dequantize run on the GPU; pack/unpack/serialize/parse are the
// byte-format utilities of the same API (host-side format code, no math).
#include <cmath>
#include <cstring>
#include <mutex>

#include "devmem.hpp"
#include "gcomm.hpp"

namespace gcomm {

std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) { return mix64(a ^ mix64(b)); }

double uniform01(std::uint64_t seed, std::uint64_t a, std::uint64_t b) {
  return static_cast<double>(mix64(seed ^ mix64(a ^ mix64(b))) >> 11) * 0x1.0p-53;
}

float normal01(std::uint64_t seed, std::uint64_t idx) {
  double u1 = uniform01(seed, idx, 0x6e5fULL);
  double u2 = uniform01(seed, idx, 0x7a21ULL);
  if (u1 < 1e-300) u1 = 1e-300;
  return static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2));
}

std::uint64_t fnv1a64(std::span<const std::uint8_t> bytes) {
  std::uint64_t h = 0xcbf29ce484222325ULL;
  for (std::uint8_t b : bytes) {
    h ^= b;
    h *= 0x100000001b3ULL;
  }
  return h;
}

std::uint64_t fnv1a64(const std::string& text) {
  return fnv1a64(std::span<const std::uint8_t>(
      reinterpret_cast<const std::uint8_t*>(text.data()), text.size()));
}

namespace codec {

using detail::cuda_check;
using detail::DeviceBuffer;

void QuantParams::validate() const {
  if (bits < 1 || bits > 8)
    throw std::invalid_argument("quantization bits must be in [1, 8], got " +
                                std::to_string(bits));
  if (bucket_size == 0) throw std::invalid_argument("bucket size must be positive");
}

static std::size_t bucket_count(std::size_t n, std::size_t bucket) {
  return (n + bucket - 1) / bucket;
}

namespace {

// per-thread scratch so repeated host-API calls do not re-allocate
struct Scratch {
  DeviceBuffer x, norms, packed, bad, out;
  detail::Stream stream;
};

Scratch& scratch() {
  detail::require_device();
  static thread_local Scratch s;
  return s;
}

void gcx_check(int rc) {
  if (rc == GCX_E_INVALID) throw std::invalid_argument(gcx_last_error());
  if (rc != GCX_OK) throw std::runtime_error(gcx_last_error());
}

}  // namespace

CompressedChunk quantize(std::span<const float> values, const QuantParams& params) {
  params.validate();
  const std::size_t n = values.size();
  CompressedChunk chunk;
  chunk.element_count = n;
  chunk.params = params;
  if (n == 0) return chunk;
  Scratch& s = scratch();
  const std::size_t nb = bucket_count(n, params.bucket_size);
  const std::size_t cap = gcx_packed_capacity(n, params.bits);
  s.x.ensure(4 * n);
  s.norms.ensure(4 * nb);
  s.packed.ensure(cap);
  s.bad.ensure(8);
  cudaStream_t st = s.stream.get();
  cuda_check(cudaMemcpyAsync(s.x.get(), values.data(), 4 * n, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemsetAsync(s.bad.get(), 0xFF, 8, st), "memset");
  gcx_check(gcx_quantize(s.x.get<float>(), n, params.bits, params.bucket_size, params.seed,
                         s.norms.get<float>(), s.packed.get<std::uint8_t>(),
                         s.bad.get<unsigned long long>(), st));
  chunk.bucket_norms.resize(nb);
  chunk.packed_levels.resize(gcx_packed_bytes(n, params.bits));
  std::uint64_t bad = 0;
  cuda_check(cudaMemcpyAsync(&bad, s.bad.get(), 8, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(chunk.bucket_norms.data(), s.norms.get(), 4 * nb,
                             cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(chunk.packed_levels.data(), s.packed.get(),
                             chunk.packed_levels.size(), cudaMemcpyDeviceToHost, st), "D2H");
  s.stream.sync();
  if (bad != ~0ULL)
    throw std::invalid_argument("non-finite gradient value at index " +
                                std::to_string(bad & ((1ULL << 40) - 1)));
  return chunk;
}

std::vector<float> dequantize(const CompressedChunk& chunk) {
  chunk.params.validate();
  const std::size_t n = chunk.element_count;
  const std::size_t bucket = chunk.params.bucket_size;
  if (chunk.bucket_norms.size() != bucket_count(n, bucket))
    throw std::runtime_error("bucket norm count does not match element count");
  const std::size_t need = gcx_packed_bytes(n, chunk.params.bits);
  if (chunk.packed_levels.size() < need)
    throw std::runtime_error("packed payload shorter than element count requires");
  std::vector<float> out(n);
  if (n == 0) return out;
  Scratch& s = scratch();
  const std::size_t cap = gcx_packed_capacity(n, chunk.params.bits);
  s.norms.ensure(4 * chunk.bucket_norms.size());
  s.packed.ensure(cap);
  s.out.ensure(4 * n);
  cudaStream_t st = s.stream.get();
  if (cap > need) cuda_check(cudaMemsetAsync(s.packed.get<char>() + need, 0, cap - need, st), "memset");
  cuda_check(cudaMemcpyAsync(s.norms.get(), chunk.bucket_norms.data(), 4 * chunk.bucket_norms.size(),
                             cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(s.packed.get(), chunk.packed_levels.data(), need,
                             cudaMemcpyHostToDevice, st), "H2D");
  gcx_check(gcx_dequantize(s.norms.get<float>(), s.packed.get<std::uint8_t>(), n,
                           chunk.params.bits, bucket, s.out.get<float>(), st));
  cuda_check(cudaMemcpyAsync(out.data(), s.out.get(), 4 * n, cudaMemcpyDeviceToHost, st), "D2H");
  s.stream.sync();
  return out;
}

// codec.cpp:158-193 on the GPU (gcx_topk_compress): accumulate, select by
// (|acc| desc, index asc), sort the winners' indices, zero them in the residual
SparseChunk topk_compress(std::span<const float> values, std::size_t k, ErrorFeedbackState& state) {
  const std::size_t n = values.size();
  if (k < 1 || k > n)
    throw std::invalid_argument("topk k must be in [1, length], got " + std::to_string(k));
  if (state.residual.size() != n)
    throw std::invalid_argument("error feedback state length does not match input");
  Scratch& s = scratch();
  cudaStream_t st = s.stream.get();
  s.x.ensure(4 * n);
  s.out.ensure(4 * n);  // residual / accumulator
  s.norms.ensure(4 * k);  // values
  s.packed.ensure(4 * k);  // indices
  s.bad.ensure(8);
  static thread_local DeviceBuffer work;
  const std::uint64_t wb = gcx_topk_scratch_bytes(n);
  work.ensure(wb);
  cuda_check(cudaMemcpyAsync(s.x.get(), values.data(), 4 * n, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(s.out.get(), state.residual.data(), 4 * n, cudaMemcpyHostToDevice, st),
             "H2D");
  cuda_check(cudaMemsetAsync(s.bad.get(), 0xFF, 8, st), "memset");
  const int rc = gcx_topk_compress(s.x.get<float>(), n, k, s.out.get<float>(),
                                   s.packed.get<std::uint32_t>(), s.norms.get<float>(), work.get(), wb,
                                   s.bad.get<unsigned long long>(), st);
  if (rc == GCX_E_INVALID) throw std::invalid_argument(gcx_stats_last_error());
  if (rc != GCX_OK) throw std::runtime_error(gcx_stats_last_error());
  std::uint64_t bad = 0;
  std::vector<std::uint32_t> idx(k);
  SparseChunk chunk;
  chunk.original_length = n;
  chunk.k = k;
  chunk.values.resize(k);
  std::vector<float> residual(n);
  cuda_check(cudaMemcpyAsync(&bad, s.bad.get(), 8, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(idx.data(), s.packed.get(), 4 * k, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(chunk.values.data(), s.norms.get(), 4 * k, cudaMemcpyDeviceToHost, st),
             "D2H");
  cuda_check(cudaMemcpyAsync(residual.data(), s.out.get(), 4 * n, cudaMemcpyDeviceToHost, st), "D2H");
  s.stream.sync();
  if (bad != ~0ULL)  // codec.cpp:170-172 (the state is left untouched)
    throw std::invalid_argument("non-finite gradient value at index " + std::to_string(bad));
  chunk.indices.assign(idx.begin(), idx.end());
  state.residual = std::move(residual);
  return chunk;
}

// codec.cpp:195-209: validation on the host, the scatter on the GPU
std::vector<float> topk_decompress(const SparseChunk& chunk) {
  if (chunk.indices.size() != chunk.values.size() || chunk.indices.size() != chunk.k)
    throw std::runtime_error("sparse chunk index/value arity mismatch");
  for (std::size_t i = 0; i < chunk.k; ++i) {
    if (chunk.indices[i] >= chunk.original_length)
      throw std::runtime_error("sparse index out of range");
    if (i > 0 && chunk.indices[i] <= chunk.indices[i - 1])
      throw std::runtime_error("sparse indices must be strictly increasing");
  }
  const std::size_t n = chunk.original_length, k = chunk.k;
  std::vector<float> out(n);
  if (n == 0) return out;
  Scratch& s = scratch();
  cudaStream_t st = s.stream.get();
  s.out.ensure(4 * n);
  s.norms.ensure(4 * k + 4);
  s.packed.ensure(4 * k + 4);
  std::vector<std::uint32_t> idx(chunk.indices.begin(), chunk.indices.end());
  if (k) {
    cuda_check(cudaMemcpyAsync(s.packed.get(), idx.data(), 4 * k, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(s.norms.get(), chunk.values.data(), 4 * k, cudaMemcpyHostToDevice, st),
               "H2D");
  }
  gcx_check(gcx_topk_densify(s.packed.get<std::uint32_t>(), s.norms.get<float>(), k, n,
                             s.out.get<float>(), st));
  cuda_check(cudaMemcpyAsync(out.data(), s.out.get(), 4 * n, cudaMemcpyDeviceToHost, st), "D2H");
  s.stream.sync();
  return out;
}

// Byte-format utilities (codec.cpp:97-149): the field layout of the packed
// stream, exposed so the packing identity can be checked without the GPU.
std::vector<std::uint8_t> pack_levels(std::span<const std::uint32_t> levels,
                                      std::span<const std::uint8_t> signs, int bits) {
  if (bits < 1 || bits > 8) throw std::invalid_argument("pack width out of range");
  if (levels.size() != signs.size())
    throw std::invalid_argument("levels/signs length mismatch");
  const int width = bits + 1;
  const std::uint32_t max_level = (1u << bits) - 1;
  std::vector<std::uint8_t> out((levels.size() * width + 7) / 8, 0);
  for (std::size_t i = 0; i < levels.size(); ++i) {
    if (levels[i] > max_level) throw std::invalid_argument("level exceeds representable range");
    const std::uint32_t field = levels[i] | (std::uint32_t(signs[i] ? 1 : 0) << bits);
    const std::size_t bit = i * width;
    for (int k = 0; k < width; ++k)
      if (field >> k & 1u) out[(bit + k) >> 3] |= std::uint8_t(1u << ((bit + k) & 7));
  }
  return out;
}

void unpack_levels(std::span<const std::uint8_t> packed, std::size_t count, int bits,
                   std::vector<std::uint32_t>& levels, std::vector<std::uint8_t>& signs) {
  if (bits < 1 || bits > 8) throw std::invalid_argument("pack width out of range");
  const int width = bits + 1;
  if (packed.size() < (count * width + 7) / 8)
    throw std::runtime_error("packed payload shorter than element count requires");
  levels.assign(count, 0);
  signs.assign(count, 0);
  for (std::size_t i = 0; i < count; ++i) {
    std::uint32_t field = 0;
    const std::size_t bit = i * width;
    for (int k = 0; k < width; ++k)
      field |= std::uint32_t(packed[(bit + k) >> 3] >> ((bit + k) & 7) & 1u) << k;
    levels[i] = field & ((1u << bits) - 1);
    signs[i] = std::uint8_t(field >> bits & 1u);
  }
}

std::size_t compressed_size_bytes(std::size_t element_count, const QuantParams& params) {
  params.validate();
  return gcx_compressed_size(element_count, params.bits, params.bucket_size);
}

static constexpr std::size_t kHeaderBytes = 4 + 1 + 4 + 8;

static void put_le(std::vector<std::uint8_t>& out, std::uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(std::uint8_t(v >> (8 * i)));
}

static std::uint64_t get_le(const std::uint8_t* p, int bytes) {
  std::uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= std::uint64_t(p[i]) << (8 * i);
  return v;
}

std::vector<std::uint8_t> serialize(const CompressedChunk& chunk) {
  std::vector<std::uint8_t> out;
  out.reserve(serialized_size_bytes(chunk.element_count, chunk.params));
  put_le(out, std::uint32_t(chunk.element_count), 4);
  out.push_back(std::uint8_t(chunk.params.bits));
  put_le(out, std::uint32_t(chunk.params.bucket_size), 4);
  put_le(out, chunk.params.seed, 8);
  for (float norm : chunk.bucket_norms) {
    std::uint32_t b;
    std::memcpy(&b, &norm, 4);
    put_le(out, b, 4);
  }
  out.insert(out.end(), chunk.packed_levels.begin(), chunk.packed_levels.end());
  return out;
}

CompressedChunk parse_chunk(std::span<const std::uint8_t> bytes) {
  if (bytes.size() < kHeaderBytes)
    throw std::runtime_error("compressed chunk truncated: header incomplete");
  CompressedChunk chunk;
  chunk.element_count = get_le(bytes.data(), 4);
  chunk.params.bits = bytes[4];
  chunk.params.bucket_size = get_le(bytes.data() + 5, 4);
  chunk.params.seed = get_le(bytes.data() + 9, 8);
  chunk.params.validate();
  const std::size_t buckets =
      chunk.element_count == 0 ? 0 : bucket_count(chunk.element_count, chunk.params.bucket_size);
  const std::size_t packed = (chunk.element_count * (chunk.params.bits + 1) + 7) / 8;
  if (bytes.size() < kHeaderBytes + 4 * buckets + packed)
    throw std::runtime_error("compressed chunk truncated: payload incomplete");
  chunk.bucket_norms.resize(buckets);
  for (std::size_t b = 0; b < buckets; ++b) {
    const std::uint32_t v = std::uint32_t(get_le(bytes.data() + kHeaderBytes + 4 * b, 4));
    std::memcpy(&chunk.bucket_norms[b], &v, 4);
  }
  const auto* body = bytes.data() + kHeaderBytes + 4 * buckets;
  chunk.packed_levels.assign(body, body + packed);
  return chunk;
}

std::size_t serialized_size_bytes(std::size_t element_count, const QuantParams& params) {
  return kHeaderBytes + compressed_size_bytes(element_count, params);
}

}  // namespace codec
}  // namespace gcomm
