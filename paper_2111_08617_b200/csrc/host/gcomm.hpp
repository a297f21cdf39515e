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

// ---------------- one process per GPU ----------------
// One rank's view of the exchange fabric.  DeviceReducer drives its two SRA
// rounds (collectives.cpp:255,264 / :289,297 in the reference) through this
// interface, so every offset, slot and message size is computed once and the
// fabric only moves bytes:
//   Communicator       NCCL grouped ncclSend/ncclRecv over NVLink (production)
//   LoopbackTransport  N in-process ranks on ONE GPU, one host thread each;
//                      a round is a device-to-device copy from the sender's
//                      buffer into the receiver's (same descriptors, same
//                      matching rule as NCCL), so the production per-rank
//                      path runs at N > 1 on a single B200.
struct PeerTransfer {
  int peer = 0;
  const void* src = nullptr;  // sends: the bytes to send
  void* dst = nullptr;        // receives: where they land
  std::uint64_t bytes = 0;
};

class Transport {
 public:
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual std::string kind() const = 0;
  // One round, issued on `stream` (a cudaStream_t) with NCCL grouped
  // semantics: when the stream reaches the end of the round every receive
  // buffer holds its message and every send buffer may be reused.  Each
  // (sender, receiver) pair carries at most one message per round; sizes
  // must agree on both sides (std::runtime_error otherwise).
  virtual void exchange(const std::vector<PeerTransfer>& sends,
                        const std::vector<PeerTransfer>& recvs, void* stream) = 0;
  // A transport over the same ranks whose rounds are independent of this
  // one's (a separate stream of messages), for per-buffer pipelining.
  // Collective: every rank calls it, in the same order.
  virtual std::unique_ptr<Transport> split() = 0;
  // Raise asynchronous fabric errors (ncclCommGetAsyncError).
  virtual void check_async() {}
};

class Communicator : public Transport {
 public:
  static std::vector<std::uint8_t> unique_id();  // ncclGetUniqueId (128 bytes)
  Communicator(int rank, int nranks, const std::vector<std::uint8_t>& id);
  ~Communicator() override;
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  int rank() const override { return rank_; }
  int size() const override { return nranks_; }
  std::string kind() const override { return "nccl"; }
  void exchange(const std::vector<PeerTransfer>& sends, const std::vector<PeerTransfer>& recvs,
                void* stream) override;
  std::unique_ptr<Transport> split() override;  // ncclCommSplit(color 0, key rank)
  void check_async() override;
  void* handle() const { return comm_; }

 private:
  Communicator(int rank, int nranks, void* comm) : rank_(rank), nranks_(nranks), comm_(comm) {}
  int rank_ = 0, nranks_ = 1;
  void* comm_ = nullptr;
};

// Shared state of N loopback ranks (one per host thread, one device).
class LoopbackHub {
 public:
  explicit LoopbackHub(int nranks, double timeout_s = 120.0);
  ~LoopbackHub();
  LoopbackHub(const LoopbackHub&) = delete;
  LoopbackHub& operator=(const LoopbackHub&) = delete;
  int size() const { return n_; }
  void exchange(int rank, const std::vector<PeerTransfer>& sends,
                const std::vector<PeerTransfer>& recvs, void* stream);
  std::shared_ptr<LoopbackHub> child(int rank);  // the rank's next split
  std::uint64_t rounds() const { return rounds_; }
  std::uint64_t bytes_moved() const { return bytes_; }

 private:
  void barrier();
  struct Impl;
  int n_;
  double timeout_s_;
  std::unique_ptr<Impl> impl_;
  std::uint64_t rounds_ = 0, bytes_ = 0;
};

class LoopbackTransport : public Transport {
 public:
  LoopbackTransport(std::shared_ptr<LoopbackHub> hub, int rank);
  int rank() const override { return rank_; }
  int size() const override { return hub_->size(); }
  std::string kind() const override { return "loopback"; }
  void exchange(const std::vector<PeerTransfer>& sends, const std::vector<PeerTransfer>& recvs,
                void* stream) override {
    hub_->exchange(rank_, sends, recvs, stream);
  }
  std::unique_ptr<Transport> split() override;
  const std::shared_ptr<LoopbackHub>& hub() const { return hub_; }

 private:
  std::shared_ptr<LoopbackHub> hub_;
  int rank_;
};

// The byte-level plan of one rank's two SRA rounds, from the layout alone
// (every rank derives it without talking to the others; the reference's
// node program sends/receives at collectives.cpp:255,264 and :289,297).
// Offsets are into the rank's three device buffers: `send` (its compressed
// share of every other chunk, at gather offsets), `recv` (N-1 slots of
// recv_stride bytes: the chunk from node src lands in slot
// src < me ? src : src-1) and `gather` (every owner's aggregate at its
// gather offset; the rank's own is the round-2 send).
enum class Region { send = 0, recv = 1, gather = 2 };
struct PlannedTransfer {
  int peer = 0;
  Region region = Region::send;
  std::uint64_t offset = 0;
  std::uint64_t bytes = 0;
};
struct ExchangePlan {
  std::uint64_t recv_stride = 0;
  std::vector<PlannedTransfer> sends[2], recvs[2];  // [round]
};
ExchangePlan sra_exchange_plan(const SraLayout& layout, std::size_t me);

// Segment-table checks shared by validate_request and DeviceReducer
// (collectives.cpp:77-102): contiguous cover of [0, d), no empty or topk
// segments, valid QuantParams, bucket sizes that fit the 32-bit piece field.
void validate_segments(const std::vector<Segment>& segments, std::size_t d);

// Per-rank SRA for one fixed buffer layout: K1 encode -> round 1 (all-to-all
// of compressed chunks) -> K2 fold + hop-1 re-encode -> round 2 (variable-size
// all-gather) -> K3 decode (+ average).  Buffers, device piece tables and key
// prefixes are built once.  Not reentrant (like the reference's SimNet and an
// NCCL communicator); concurrent buffers use separate reducers on split
// transports.
class DeviceReducer {
 public:
  DeviceReducer(Transport& transport, std::size_t d, std::vector<Segment> segments);
  ~DeviceReducer();
  // in/out: device pointers to d floats (may alias); stream: cudaStream_t.
  // Non-finite inputs of quantized pieces are recorded on the device (the
  // reference's codec.cpp:43-45 check) and raised by poll().
  void allreduce(const float* in, float* out, std::uint64_t step_seed, ReduceOp op,
                 void* stream);
  // Raise std::invalid_argument("non-finite gradient value at index i") if
  // the last completed call saw one, and the transport's async errors.
  // wait = false: only if that call has finished on the device (no sync).
  // Returns whether the last call has completed.
  bool poll(bool wait);
  // Graph-replayable steps: from now on allreduce() ignores step_seed and
  // takes the step seed H(H(base_seed, step), buffer) (engine.cpp:208-209)
  // from a device-resident counter that starts at next_step and advances on
  // the device every call, so a step captured in a CUDA graph (NCCL
  // transport) replays with fresh keys.  Span tables only.
  void use_device_seeds(std::uint64_t base_seed, std::uint64_t buffer, std::uint64_t next_step);
  std::uint64_t device_step() const;  // the counter (synchronous read)
  // After a captured step's replay has completed: raise its non-finite /
  // transport errors (poll() covers eager calls).
  void check_replay();
  std::size_t elements() const { return layout_.d; }
  const SraLayout& layout() const { return layout_; }
  StepTrace trace() const;
  std::uint64_t device_bytes_sent() const;
  int launches_per_call() const;
  Transport& transport() const { return transport_; }

 private:
  struct Impl;
  Transport& transport_;
  SraLayout layout_;
  std::unique_ptr<Impl> impl_;
};

}  // namespace collectives
}  // namespace gcomm
