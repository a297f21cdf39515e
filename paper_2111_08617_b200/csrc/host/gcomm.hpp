// gcomm.hpp — C++ host façade of the B200 path, mirroring the reference's
// public API (/root/reference/proj/include/gcomm/{codec,collectives,model}.hpp)
// so a caller of the reference can switch by relinking.  Everything numeric
// runs on the GPU through the C-ABI in include/gcx.h; this layer owns device
// memory, streams, piece tables and NCCL.  There is no CPU fallback: without
// a CUDA device every compute entry point throws std::runtime_error.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <regex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "gcx.h"

namespace gcomm {

// include/gcomm/util.hpp:14-29 (host copies for seeds / keys)
std::uint64_t mix64(std::uint64_t z);
std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b);
double uniform01(std::uint64_t seed, std::uint64_t a, std::uint64_t b);
float normal01(std::uint64_t seed, std::uint64_t idx);
std::uint64_t fnv1a64(std::span<const std::uint8_t> bytes);
std::uint64_t fnv1a64(const std::string& text);

namespace codec {

// include/gcomm/codec.hpp:12-26
struct QuantParams {
  int bits = 4;
  std::size_t bucket_size = 128;
  std::uint64_t seed = 0;
  int levels() const { return (1 << bits) - 1; }
  void validate() const;  // std::invalid_argument, codec.cpp:13-18
};

struct CompressedChunk {
  std::size_t element_count = 0;
  QuantParams params;
  std::vector<float> bucket_norms;
  std::vector<std::uint8_t> packed_levels;
};

CompressedChunk quantize(std::span<const float> values, const QuantParams& params);
std::vector<float> dequantize(const CompressedChunk& chunk);
std::vector<std::uint8_t> pack_levels(std::span<const std::uint32_t> levels,
                                      std::span<const std::uint8_t> signs, int bits);
void unpack_levels(std::span<const std::uint8_t> packed, std::size_t count, int bits,
                   std::vector<std::uint32_t>& levels, std::vector<std::uint8_t>& signs);
std::size_t compressed_size_bytes(std::size_t element_count, const QuantParams& params);
std::vector<std::uint8_t> serialize(const CompressedChunk& chunk);
CompressedChunk parse_chunk(std::span<const std::uint8_t> bytes);
std::size_t serialized_size_bytes(std::size_t element_count, const QuantParams& params);

// include/gcomm/codec.hpp:28-42, 59-61: TopK selection with error feedback
struct SparseChunk {
  std::size_t original_length = 0;
  std::size_t k = 0;
  std::vector<std::size_t> indices;
  std::vector<float> values;
};

struct ErrorFeedbackState {
  std::vector<float> residual;
  ErrorFeedbackState() = default;
  explicit ErrorFeedbackState(std::size_t length) : residual(length, 0.0f) {}
};

SparseChunk topk_compress(std::span<const float> values, std::size_t k, ErrorFeedbackState& state);
std::vector<float> topk_decompress(const SparseChunk& chunk);

}  // namespace codec

namespace model {

// include/gcomm/model.hpp:13-103
enum class LayerKind { weight, bias, norm, embedding, other };
LayerKind layer_kind_from_string(const std::string& s);
std::string to_string(LayerKind kind);

struct LayerSpec {
  std::string name;
  std::size_t elements = 0;
  LayerKind kind = LayerKind::weight;
};

enum class CodecMode { quantize, topk, uncompressed };

struct LayerCodec {
  CodecMode mode = CodecMode::quantize;
  int bits = 4;
  std::size_t bucket_size = 128;
  std::size_t k = 0;
};

struct CompressionPlan {
  LayerCodec defaults;
  std::vector<std::pair<std::string, LayerCodec>> overrides;
  LayerCodec resolve(const std::string& layer_name) const;
  void set(const std::string& layer_name, const LayerCodec& codec);
  void validate() const;
  static CompressionPlan from_json(const std::string& text);
  std::string to_json() const;
};

struct FilterRules {
  std::vector<LayerKind> exclude_kinds{LayerKind::bias, LayerKind::norm};
  std::size_t min_elements = 4096;
  std::vector<std::string> exclude_patterns;
  void compile();
  bool excluded(const LayerSpec& layer) const;

 private:
  std::vector<std::regex> compiled_;
  bool compiled_ready_ = false;
};

struct BufferSegment {
  std::size_t tensor_index = 0;
  std::size_t layer_offset = 0;
  std::size_t buffer_offset = 0;
  std::size_t length = 0;
};

struct FusedBuffer {
  std::vector<BufferSegment> segments;
  std::size_t total_elements = 0;
  std::size_t capacity_bytes = 0;
};

std::vector<FusedBuffer> pack_fused_buffers(const std::vector<std::size_t>& tensor_elements,
                                            std::size_t capacity_bytes);

}  // namespace model

namespace collectives {

enum class Topology { sra, ring, tree };
Topology topology_from_string(const std::string& s);
std::string to_string(Topology topology);
enum class ReduceOp { sum, average };

// include/gcomm/collectives.hpp:23-42
struct Segment {
  std::size_t offset = 0;
  std::size_t length = 0;
  model::CodecMode mode = model::CodecMode::quantize;
  int bits = 4;
  std::size_t bucket_size = 128;
};

// include/gcomm/simnet.hpp:43-57.  Byte counters are the reference's wire
// bytes (17-byte headers included) so they compare 1:1; device_time_s is
// the CUDA-event time of the call (the reference reports virtual time).
struct StepTrace {
  std::vector<std::uint64_t> bytes_sent;
  std::vector<std::uint64_t> bytes_received;
  std::uint64_t message_count = 0;
  std::uint64_t rounds = 0;
  double device_time_s = 0.0;
  std::uint64_t compress_calls = 0;
  std::uint64_t decompress_calls = 0;
  std::uint64_t max_compress_depth = 0;
  std::uint64_t device_bytes_sent = 0;  // bytes actually moved by our layout (all nodes)
  std::uint64_t total_bytes_sent() const;
  std::uint64_t total_bytes_received() const;
  void accumulate(const StepTrace& other);
};

struct ReduceRequest {
  std::vector<std::vector<float>> inputs;
  std::vector<Segment> segments;
  Topology topology = Topology::sra;
  ReduceOp op = ReduceOp::sum;
  std::uint64_t step_seed = 0;
};

struct ReduceResult {
  std::vector<std::vector<float>> outputs;
  StepTrace trace;
};

std::uint64_t hop_seed(std::uint64_t step_seed, std::uint64_t hop, std::uint64_t node);
std::uint64_t latency_rounds(Topology topology, std::size_t nodes);
void validate_request(const ReduceRequest& req, std::size_t nodes);

// Owner chunk bounds (collectives.cpp:106-122) and per-chunk piece layouts
// with their device payload offsets.
struct ChunkLayout {
  std::size_t lo = 0, hi = 0;
  std::vector<gcx_piece> pieces;  // src absolute; norms/packed relative to the chunk message
  std::uint64_t msg_bytes = 0;    // device message size (16-byte aligned pieces)
  std::uint64_t wire_bytes = 0;   // reference wire size (serialize per piece)
  std::size_t quantized_pieces = 0;
  bool any_quantized() const { return quantized_pieces > 0; }
};

struct SraLayout {
  std::size_t d = 0, nodes = 0;
  std::vector<std::size_t> bounds;
  std::vector<ChunkLayout> chunks;
  std::vector<std::uint64_t> gather_offset;  // chunk c message offset in a full-layout buffer
  std::uint64_t gather_bytes = 0;
};

std::vector<std::size_t> chunk_boundaries(std::size_t d, std::size_t nodes,
                                          const std::vector<Segment>& segments);
SraLayout make_layout(std::size_t d, std::size_t nodes, const std::vector<Segment>& segments);
StepTrace sra_trace(const SraLayout& layout);

// Drop-in for collectives::allreduce(request, SimNet&) (collectives.cpp:475-494):
// all `nodes` run on the current GPU (one process), the exchange is
// device-local.  Outputs are bit-identical to the reference's.
ReduceResult allreduce(const ReduceRequest& request, std::size_t nodes);

// Drop-in for collectives::sparse_allreduce(chunks, op, SimNet&)
// (collectives.cpp:533-603): every node's sparse chunk is densified and the
// dense vectors summed in ascending node order on this GPU (÷N for average).
ReduceResult sparse_allreduce(const std::vector<codec::SparseChunk>& chunks, ReduceOp op,
                              std::size_t nodes);

// ---------------- one process per GPU (NCCL over NVLink) ----------------
class Communicator {
 public:
  static std::vector<std::uint8_t> unique_id();  // ncclGetUniqueId (128 bytes)
  Communicator(int rank, int nranks, const std::vector<std::uint8_t>& id);
  ~Communicator();
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  int rank() const { return rank_; }
  int size() const { return nranks_; }
  void* handle() const { return comm_; }

 private:
  int rank_ = 0, nranks_ = 1;
  void* comm_ = nullptr;
};

// Per-rank SRA over NCCL for one fixed buffer layout: K1 encode -> grouped
// send/recv (all-to-all) -> K2 fold+requant -> grouped send/recv
// (all-gather) -> K3 decode.  Buffers and device piece tables are built once.
class DeviceReducer {
 public:
  DeviceReducer(Communicator& comm, std::size_t d, std::vector<Segment> segments);
  ~DeviceReducer();
  // in/out: device pointers to d floats (may alias); stream: cudaStream_t
  void allreduce(const float* in, float* out, std::uint64_t step_seed, ReduceOp op,
                 void* stream);
  const SraLayout& layout() const { return layout_; }
  StepTrace trace() const;
  std::uint64_t device_bytes_sent() const;
  int launches_per_call() const;

 private:
  struct Impl;
  Communicator& comm_;
  SraLayout layout_;
  std::unique_ptr<Impl> impl_;
};

}  // namespace collectives
}  // namespace gcomm
