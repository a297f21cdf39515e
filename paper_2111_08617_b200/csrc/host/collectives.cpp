// collectives.cpp — compressed SRA allreduce on B200.
// Reference: /root/reference/proj/src/collectives.cpp (run_sra :230-310,
// chunk_boundaries :106-122, pieces_for :124-140, finalize :213-228,
// allreduce :475-494).  Two drivers share the layout code:
//   allreduce(request, nodes)  all nodes on the current GPU (drop-in for the
//                              reference's single-process allreduce(req, net))
//   DeviceReducer              one rank per GPU, NCCL grouped send/recv over
//                              NVLink for the two exchange rounds.
#include <nvtx3/nvToolsExt.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "devmem.hpp"
#include "gcomm.hpp"

namespace gcomm::collectives {

using detail::align_up;
using detail::cuda_check;
using detail::DeviceBuffer;

namespace {

void gcx_check(int rc) {
  if (rc == GCX_E_INVALID) throw std::invalid_argument(gcx_last_error());
  if (rc != GCX_OK) throw std::runtime_error(gcx_last_error());
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}

constexpr std::uint64_t kMsgAlign = 256;

}  // namespace

Topology topology_from_string(const std::string& s) {
  if (s == "sra") return Topology::sra;
  if (s == "ring") return Topology::ring;
  if (s == "tree") return Topology::tree;
  throw std::invalid_argument("unknown topology: " + s);
}

std::string to_string(Topology topology) {
  switch (topology) {
    case Topology::sra: return "sra";
    case Topology::ring: return "ring";
    case Topology::tree: return "tree";
  }
  return "sra";
}

// collectives.cpp:29-31
std::uint64_t hop_seed(std::uint64_t step_seed, std::uint64_t hop, std::uint64_t node) {
  return hash_combine(step_seed, hash_combine(hop, node));
}

// collectives.cpp:33-45
std::uint64_t latency_rounds(Topology topology, std::size_t nodes) {
  if (nodes <= 1) return 0;
  switch (topology) {
    case Topology::sra: return 2;
    case Topology::ring: return 2 * (nodes - 1);
    case Topology::tree: {
      std::size_t levels = 0;
      while ((std::size_t{1} << levels) < nodes) ++levels;
      return 2 * levels;
    }
  }
  return 0;
}

std::uint64_t StepTrace::total_bytes_sent() const {
  std::uint64_t t = 0;
  for (auto b : bytes_sent) t += b;
  return t;
}

std::uint64_t StepTrace::total_bytes_received() const {
  std::uint64_t t = 0;
  for (auto b : bytes_received) t += b;
  return t;
}

void StepTrace::accumulate(const StepTrace& o) {
  if (bytes_sent.size() < o.bytes_sent.size()) bytes_sent.resize(o.bytes_sent.size(), 0);
  if (bytes_received.size() < o.bytes_received.size())
    bytes_received.resize(o.bytes_received.size(), 0);
  for (std::size_t i = 0; i < o.bytes_sent.size(); ++i) bytes_sent[i] += o.bytes_sent[i];
  for (std::size_t i = 0; i < o.bytes_received.size(); ++i)
    bytes_received[i] += o.bytes_received[i];
  message_count += o.message_count;
  rounds += o.rounds;
  device_time_s += o.device_time_s;
  compress_calls += o.compress_calls;
  decompress_calls += o.decompress_calls;
  max_compress_depth = std::max(max_compress_depth, o.max_compress_depth);
  device_bytes_sent += o.device_bytes_sent;
}

// collectives.cpp:77-102 (same messages)
void validate_segments(const std::vector<Segment>& segments, std::size_t d) {
  std::size_t cursor = 0;
  for (const auto& seg : segments) {
    if (seg.offset != cursor)
      throw std::invalid_argument("segments must cover the buffer contiguously");
    if (seg.length == 0) throw std::invalid_argument("zero-length segment");
    if (seg.mode == model::CodecMode::topk)
      throw std::invalid_argument("topk segments use the sparse path");
    if (seg.mode == model::CodecMode::quantize) {
      codec::QuantParams p;
      p.bits = seg.bits;
      p.bucket_size = seg.bucket_size;
      p.validate();
      if (seg.bucket_size > 0xFFFFFFFFull)
        throw std::invalid_argument("bucket size must fit 32 bits");
    }
    cursor += seg.length;
  }
  if (cursor != d)
    throw std::invalid_argument("segments cover " + std::to_string(cursor) +
                                " elements but buffers hold " + std::to_string(d));
}

void validate_request(const ReduceRequest& req, std::size_t nodes) {
  if (req.inputs.size() != nodes)
    throw std::invalid_argument("expected one input buffer per node");
  const std::size_t d = req.inputs.empty() ? 0 : req.inputs[0].size();
  for (const auto& in : req.inputs)
    if (in.size() != d) throw std::invalid_argument("input buffers must have equal lengths");
  validate_segments(req.segments, d);
}

// collectives.cpp:106-122
std::vector<std::size_t> chunk_boundaries(std::size_t d, std::size_t nodes,
                                          const std::vector<Segment>& segments) {
  std::vector<std::size_t> bounds(nodes + 1, 0);
  bounds[nodes] = d;
  for (std::size_t k = 1; k < nodes; ++k) {
    std::size_t p = d * k / nodes;
    for (const auto& seg : segments) {
      if (p >= seg.offset && p < seg.offset + seg.length) {
        if (seg.mode == model::CodecMode::quantize)
          p = seg.offset + ((p - seg.offset) / seg.bucket_size) * seg.bucket_size;
        break;
      }
    }
    bounds[k] = std::max(bounds[k - 1], p);
  }
  return bounds;
}

// pieces_for (collectives.cpp:124-140) + the device payload layout of a
// chunk message: 16-byte aligned norms / packed / raw regions per piece.
SraLayout make_layout(std::size_t d, std::size_t nodes, const std::vector<Segment>& segments) {
  SraLayout L;
  L.d = d;
  L.nodes = nodes;
  L.bounds = chunk_boundaries(d, nodes, segments);
  L.chunks.resize(nodes);
  L.gather_offset.resize(nodes);
  std::uint64_t goff = 0;
  for (std::size_t c = 0; c < nodes; ++c) {
    ChunkLayout& ch = L.chunks[c];
    ch.lo = L.bounds[c];
    ch.hi = L.bounds[c + 1];
    std::uint64_t off = 0;
    for (const auto& seg : segments) {
      const std::size_t a = std::max(ch.lo, seg.offset);
      const std::size_t b = std::min(ch.hi, seg.offset + seg.length);
      if (a >= b) continue;
      gcx_piece p{};
      p.src = a;
      p.len = b - a;
      if (seg.mode == model::CodecMode::quantize) {
        p.bits = seg.bits;
        p.bucket = std::uint32_t(seg.bucket_size);
        p.norms = off;
        const std::uint64_t nb = (p.len + seg.bucket_size - 1) / seg.bucket_size;
        p.packed = align_up(off + 4 * nb, 16);
        off = align_up(p.packed + gcx_packed_capacity(p.len, p.bits), 16);
        ch.wire_bytes += 17 + gcx_compressed_size(p.len, p.bits, seg.bucket_size);
        ch.quantized_pieces += 1;
      } else {
        p.bits = 0;
        p.bucket = 0;
        p.norms = off;
        p.packed = off;
        off = align_up(off + 4 * p.len, 16);
        ch.wire_bytes += 4 * p.len;
      }
      ch.pieces.push_back(p);
    }
    ch.msg_bytes = off;
    L.gather_offset[c] = goff;
    goff += align_up(off, kMsgAlign);
  }
  L.gather_bytes = goff;
  return L;
}

// Reference-equivalent accounting of one SRA step (simnet.hpp:43-57 as
// run_sra fills it): wire bytes with 17-byte headers, 2N(N-1) messages.
StepTrace sra_trace(const SraLayout& L) {
  StepTrace t;
  const std::size_t N = L.nodes;
  t.bytes_sent.assign(N, 0);
  t.bytes_received.assign(N, 0);
  if (N <= 1) return t;
  std::uint64_t q_total = 0, all_wire = 0;
  bool any_q = false;
  for (const auto& ch : L.chunks) {
    q_total += ch.quantized_pieces;
    all_wire += ch.wire_bytes;
    any_q = any_q || ch.any_quantized();
  }
  for (std::size_t me = 0; me < N; ++me) {
    const std::uint64_t mine = L.chunks[me].wire_bytes;
    t.bytes_sent[me] = (all_wire - mine) + (N - 1) * mine;
    t.bytes_received[me] = (N - 1) * mine + (all_wire - mine);
  }
  t.message_count = 2 * N * (N - 1);
  t.rounds = 2;
  t.compress_calls = N * q_total;
  t.decompress_calls = (2 * N - 1) * q_total;
  t.max_compress_depth = any_q ? 2 : 0;
  for (std::size_t me = 0; me < N; ++me) {
    std::uint64_t dev = 0;
    for (std::size_t c = 0; c < N; ++c)
      if (c != me) dev += L.chunks[c].msg_bytes + L.chunks[me].msg_bytes;
    t.device_bytes_sent += dev;
  }
  return t;
}

namespace {

// A device piece table with its tile prefix (and, for tables quantized under
// one seed, its key-table plan), uploaded into one blob.
struct Table;
bool onestep_table(const Table& t);
// Shared key tables (N > 2 stage 1) take the span K1 in key-table mode
// (default; 4 % faster per rank at N = 8 than the CTA K1 once raw tiles were
// vectorised); GCX_SPAN_SHARED=0 restores the lane-group layout + CTA K1
// (measurement switch)
bool span_shared_tables() {
  static const bool v = [] {
    const char* e = std::getenv("GCX_SPAN_SHARED");
    return e == nullptr || e[0] != '0';
  }();
  return v;
}

struct Table {
  std::vector<gcx_piece> pieces;
  std::vector<std::uint32_t> prefix;
  std::uint32_t ntiles = 0;
  std::uint32_t flags = 0;
  std::size_t dev_off = 0;  // byte offsets in the blob
  std::size_t pre_off = 0;
  std::vector<gcx_keygroup> groups;
  std::uint64_t key_len = 0;  // key-table entries this table needs
  std::size_t grp_off = 0;
  // with_keys: plan key runs; keep_span: keep the span key layout even when
  // the table is not a one-step table (an owner table fed to the fused fold)
  void plan(bool with_keys = false, bool keep_span = false) {
    prefix.assign(pieces.size() + 1, 0);
    const std::int64_t nt =
        gcx_plan_tiles(pieces.data(), std::uint32_t(pieces.size()), prefix.data(), &flags);
    if (nt < 0) gcx_check(int(nt));
    ntiles = std::uint32_t(nt);
    groups.clear();
    key_len = 0;
    for (auto& p : pieces) p.keys = ~0ULL;
    if (with_keys && !pieces.empty()) {
      auto plan_keys = [&](int layout) {
        groups.resize(pieces.size());
        std::uint32_t ng = 0;
        const std::int64_t len =
            gcx_plan_keys_layout(pieces.data(), std::uint32_t(pieces.size()), groups.data(),
                                 std::uint32_t(groups.size()), &ng, layout);
        if (len < 0) gcx_check(int(len));
        groups.resize(ng);
        key_len = std::uint64_t(len);
      };
      plan_keys(GCX_KEYS_AUTO);
      // Span tables keep the span key layout (prefix one-step or key-table
      // mode of the span K1); with GCX_SPAN_SHARED=0 tables whose key slots
      // are read by several pieces (N > 2 stage 1) fall back to the two-step
      // key table + CTA K1, in the lane-group layout without GCX_F_SPAN_ENC.
      if ((flags & GCX_F_SPAN_ENC) && !onestep_table(*this) && !keep_span && !span_shared_tables()) {
        flags &= ~(GCX_F_SPAN_ENC | (0xFFu << GCX_F_SPAN_BITS_SHIFT));
        plan_keys(GCX_KEYS_LANE_GROUP);
      }
    }
  }
};

struct TableBlob {
  DeviceBuffer buf;
  void upload(std::vector<Table*> tables) {
    std::size_t off = 0;
    for (Table* t : tables) {
      t->dev_off = off;
      off = align_up(off + sizeof(gcx_piece) * std::max<std::size_t>(1, t->pieces.size()), 16);
      t->pre_off = off;
      off = align_up(off + 4 * t->prefix.size(), 16);
      t->grp_off = off;
      off = align_up(off + sizeof(gcx_keygroup) * t->groups.size() + 16, 16);
    }
    std::vector<std::uint8_t> host(off, 0);
    for (Table* t : tables) {
      if (!t->pieces.empty())
        std::memcpy(host.data() + t->dev_off, t->pieces.data(), sizeof(gcx_piece) * t->pieces.size());
      std::memcpy(host.data() + t->pre_off, t->prefix.data(), 4 * t->prefix.size());
      if (!t->groups.empty())
        std::memcpy(host.data() + t->grp_off, t->groups.data(),
                    sizeof(gcx_keygroup) * t->groups.size());
    }
    buf.reset(off);
    cuda_check(cudaMemcpy(buf.get(), host.data(), off, cudaMemcpyHostToDevice), "table upload");
  }
  const gcx_piece* pieces(const Table& t) const {
    return reinterpret_cast<const gcx_piece*>(buf.get<std::uint8_t>() + t.dev_off);
  }
  const std::uint32_t* prefix(const Table& t) const {
    return reinterpret_cast<const std::uint32_t*>(buf.get<std::uint8_t>() + t.pre_off);
  }
  const gcx_keygroup* groups(const Table& t) const {
    return reinterpret_cast<const gcx_keygroup*>(buf.get<std::uint8_t>() + t.grp_off);
  }
};

// Device time of the kernels issued between construction and end_ms() on
// st (the single-GPU drivers' device_time_s).  GCX_EMUL_GRAPH=1 captures
// the region as a CUDA graph and launches it once, so the events bracket
// device work only -- what a graph-replayed per-rank step runs
// (DeviceReducer::use_device_seeds); by default the region is timed as
// issued, host launch gaps included.
struct TimedRegion {
  cudaStream_t st;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool graph;
  explicit TimedRegion(cudaStream_t s) : st(s) {
    const char* e = std::getenv("GCX_EMUL_GRAPH");
    graph = e != nullptr && e[0] == '1';
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    if (graph)
      cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed), "begin capture");
    else
      cuda_check(cudaEventRecord(e0, st), "event record");
  }
  float end_ms() {
    if (graph) {
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ge = nullptr;
      cuda_check(cudaStreamEndCapture(st, &g), "end capture");
      cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
      cuda_check(cudaGraphUpload(ge, st), "graph upload");
      cuda_check(cudaEventRecord(e0, st), "event record");
      cuda_check(cudaGraphLaunch(ge, st), "graph launch");
      cuda_check(cudaEventRecord(e1, st), "event record");
      cuda_check(cudaStreamSynchronize(st), "sync");
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    } else {
      cuda_check(cudaEventRecord(e1, st), "event record");
      cuda_check(cudaEventSynchronize(e1), "sync");
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
  }
  ~TimedRegion() {
    cudaStreamCaptureStatus c = cudaStreamCaptureStatusNone;
    if (graph && cudaStreamIsCapturing(st, &c) == cudaSuccess && c != cudaStreamCaptureStatusNone) {
      cudaGraph_t g = nullptr;  // an exception left the capture open: close and drop it
      if (cudaStreamEndCapture(st, &g) == cudaSuccess && g) cudaGraphDestroy(g);
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
  TimedRegion(const TimedRegion&) = delete;
  TimedRegion& operator=(const TimedRegion&) = delete;
};

// K1 over a table quantized under one seed: draw the shared key runs once
// (gcx_make_keys), then norms + quantize + pack reading keys from the table
// (from the table's stored key prefixes when given: one finalizer per slot)
// A table whose key slots are NOT shared between pieces (one owner chunk, or
// N = 2's single peer chunk) and is large is quantized in ONE launch straight
// from the prefixes (K1 hashes mix64(seed ^ T) per element): the separate
// key-table pass would hash every slot once anyway and adds its traffic.
// Shared tables (N > 2 send tables: N-1 pieces read each slot) and small
// tables (the CTA K1 has the lower latency) keep the two-step path.
// Measured on B200, 4-bit/128: N = 2 at 16/64 MiB 78 -> 71 / 222 -> 187 us
// per rank one-step; 4 MiB and below, two-step is 7-9 us faster.
// GCX_ONESTEP_MIN_SLOTS overrides the size threshold (measurement).
std::uint64_t onestep_min_slots() {
  static const std::uint64_t v = [] {
    const char* e = std::getenv("GCX_ONESTEP_MIN_SLOTS");
    return e != nullptr ? std::strtoull(e, nullptr, 10) : std::uint64_t{1} << 20;
  }();
  return v;
}

bool onestep(const Table& t) {
  std::uint64_t q = 0;
  for (const auto& p : t.pieces)
    if (p.bits > 0) q += p.len;
  return t.key_len >= onestep_min_slots() && 2 * q < 3 * t.key_len;
}

bool onestep_table(const Table& t) { return onestep(t); }

// seed_dev (a graph-replayable step): the seed is read on the device from
// *seed_dev (GCX_F_SEED_DEVICE), span tables with key prefixes only.
void encode(const TableBlob& blob, const Table& t, std::uint64_t seed, const float* src,
            std::uint8_t* msg, unsigned long long* keys, unsigned long long* bad,
            cudaStream_t st, const unsigned long long* key_prefix = nullptr,
            const unsigned long long* seed_dev = nullptr) {
  const bool use_keys = keys != nullptr && t.key_len > 0;
  const std::uint32_t fdev = seed_dev != nullptr ? GCX_F_SEED_DEVICE : 0u;
  const std::uint64_t sarg = seed_dev != nullptr ? reinterpret_cast<std::uint64_t>(seed_dev) : seed;
  if (use_keys && key_prefix != nullptr && onestep(t)) {
    gcx_check(gcx_encode_pieces(blob.pieces(t), blob.prefix(t), std::uint32_t(t.pieces.size()),
                                t.ntiles, t.flags | GCX_F_KEY_PREFIX | fdev, sarg, src, msg,
                                key_prefix, bad, st));
    return;
  }
  if (use_keys && key_prefix != nullptr && seed_dev != nullptr)
    gcx_check(gcx_make_keys_prefixed_dev(t.key_len, seed_dev, key_prefix, keys, st));
  else if (use_keys && key_prefix != nullptr)
    gcx_check(gcx_make_keys_prefixed(t.key_len, seed, key_prefix, keys, st));
  else if (use_keys && seed_dev != nullptr)
    throw std::invalid_argument("device-resident seeds need the table's key prefixes");
  else if (use_keys)
    gcx_check(gcx_make_keys(blob.groups(t), std::uint32_t(t.groups.size()), t.key_len, seed, keys,
                            st));
  gcx_check(gcx_encode_pieces(blob.pieces(t), blob.prefix(t), std::uint32_t(t.pieces.size()),
                              t.ntiles, t.flags | fdev, sarg, src, msg, use_keys ? keys : nullptr,
                              bad, st));
}

// The owner's fold + hop-1 re-encode (collectives.cpp:266-284): one fused
// launch when the table qualifies (gcx_sra_fold_encode: span K1 fed by the
// fold, the aggregate never in HBM), else fold into `out` and encode it.
void owner_step(const TableBlob& blob, const Table& t, const std::uint8_t* recv,
                std::uint64_t slot_stride, const float* own, std::size_t nodes, std::size_t me,
                std::uint64_t seed, std::uint8_t* bcast, float* out, unsigned long long* keys,
                unsigned long long* bad, cudaStream_t st, const unsigned long long* key_prefix,
                const unsigned long long* seed_dev = nullptr) {
  const bool pre = key_prefix != nullptr && t.key_len > 0;
  if ((t.flags & GCX_F_SPAN_ENC) && nodes <= 8) {
    gcx_check(gcx_sra_fold_encode(
        blob.pieces(t), blob.prefix(t), std::uint32_t(t.pieces.size()), t.ntiles,
        t.flags | (pre ? GCX_F_KEY_PREFIX : 0u) | (seed_dev != nullptr ? GCX_F_SEED_DEVICE : 0u),
        recv, slot_stride, own, std::uint32_t(nodes), std::uint32_t(me),
        seed_dev != nullptr ? reinterpret_cast<std::uint64_t>(seed_dev) : seed, bcast, out,
        pre ? key_prefix : nullptr, bad, st));
    return;
  }
  gcx_check(gcx_fold_pieces(blob.pieces(t), blob.prefix(t), std::uint32_t(t.pieces.size()),
                            t.ntiles, t.flags, recv, slot_stride, own, std::uint32_t(nodes),
                            std::uint32_t(me), out, st));
  encode(blob, t, seed, out, bcast, keys, bad, st, key_prefix, seed_dev);
}

Table shifted(const std::vector<gcx_piece>& src, std::uint64_t delta) {
  Table t;
  t.pieces = src;
  for (auto& p : t.pieces) {
    p.norms += delta;
    p.packed += delta;
  }
  return t;
}

void append(Table& t, const std::vector<gcx_piece>& src, std::uint64_t delta) {
  for (gcx_piece p : src) {
    p.norms += delta;
    p.packed += delta;
    t.pieces.push_back(p);
  }
}

[[noreturn]] void throw_non_finite(const Table& t, std::uint64_t key) {
  const std::uint64_t local = key & ((1ULL << 40) - 1);
  (void)t;
  throw std::invalid_argument("non-finite gradient value at index " + std::to_string(local));
}

// quantized pieces of a piece list (for the reference's call counters)
std::uint64_t quantized(const std::vector<gcx_piece>& ps) {
  std::uint64_t q = 0;
  for (const auto& p : ps) q += p.bits > 0 ? 1 : 0;
  return q;
}

void encode_inline(const TableBlob& blob, const Table& t, std::uint64_t seed, const float* src,
                   std::uint8_t* msg, std::uint64_t msg_bytes, unsigned long long* bad,
                   cudaStream_t st) {
  if (t.flags & GCX_F_NEEDS_ZERO)
    cuda_check(cudaMemsetAsync(msg, 0, msg_bytes, st), "memset");
  gcx_check(gcx_encode_pieces(blob.pieces(t), blob.prefix(t), std::uint32_t(t.pieces.size()),
                              t.ntiles, t.flags, seed, src, msg, nullptr, bad, st));
}

void decode_into(const TableBlob& blob, const Table& t, const std::uint8_t* msg, float* dst,
                 float divisor, cudaStream_t st) {
  gcx_check(gcx_decode_pieces(blob.pieces(t), blob.prefix(t), std::uint32_t(t.pieces.size()),
                              t.ntiles, t.flags, msg, dst, divisor, st));
}

// run_ring (collectives.cpp:312-386) with every node on this GPU: the
// reduce-scatter carries a chunk around the ring, each stop decoding the
// partial, adding its local values and re-encoding (hop seed (t, me)); the
// owner encodes its finished chunk once (hop N-1) and the bytes travel
// verbatim, so every node decodes the same payload.
ReduceResult allreduce_ring(const ReduceRequest& req, std::size_t N) {
  const std::size_t d = req.inputs[0].size();
  const SraLayout L = make_layout(d, N, req.segments);
  std::vector<Table> loc(N), full(N);
  std::uint64_t max_msg = 16;
  for (std::size_t c = 0; c < N; ++c) {
    loc[c].pieces = L.chunks[c].pieces;
    for (auto& p : loc[c].pieces) p.src -= L.bounds[c];  // chunk-local
    full[c].pieces = L.chunks[c].pieces;                  // buffer offsets
    loc[c].plan();
    full[c].plan();
    max_msg = std::max<std::uint64_t>(max_msg, L.chunks[c].msg_bytes);
  }
  std::vector<Table*> all;
  for (std::size_t c = 0; c < N; ++c) {
    all.push_back(&loc[c]);
    all.push_back(&full[c]);
  }
  TableBlob blob;
  blob.upload(all);
  std::size_t max_chunk = 1;
  for (std::size_t c = 0; c < N; ++c)
    max_chunk = std::max(max_chunk, L.bounds[c + 1] - L.bounds[c]);
  const std::uint64_t mstride = align_up(max_msg, kMsgAlign);

  detail::Stream stream;
  cudaStream_t st = stream.get();
  DeviceBuffer in(4 * d * N + 16), out(4 * d * N + 16), carry(4 * max_chunk * N + 16),
      msg(mstride * N + 16), gather(L.gather_bytes + 16), bad(8 * N * N + 16);
  for (std::size_t k = 0; k < N; ++k)
    cuda_check(cudaMemcpyAsync(in.get<float>() + k * d, req.inputs[k].data(), 4 * d,
                               cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemsetAsync(bad.get(), 0xFF, bad.size(), st), "memset");
  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0), "event");
  cuda_check(cudaEventCreate(&e1), "event");
  cudaEventRecord(e0, st);
  auto chunk_at = [N](std::size_t j, std::size_t back) { return (j + N - back % N) % N; };
  auto* badp = bad.get<unsigned long long>();
  auto cbuf = [&](std::size_t me) { return carry.get<float>() + me * max_chunk; };
  auto mbuf = [&](std::size_t me) { return msg.get<std::uint8_t>() + me * mstride; };
  for (std::size_t me = 0; me < N; ++me) {
    const std::size_t c = chunk_at(me, 1);
    cuda_check(cudaMemcpyAsync(cbuf(me), in.get<float>() + me * d + L.bounds[c],
                               4 * (L.bounds[c + 1] - L.bounds[c]), cudaMemcpyDeviceToDevice, st),
               "D2D");
  }
  for (std::size_t t = 0; t + 1 < N; ++t) {
    for (std::size_t me = 0; me < N; ++me) {  // every node sends right
      const std::size_t c = chunk_at(me, 1 + t);
      encode_inline(blob, loc[c], hop_seed(req.step_seed, t, me), cbuf(me), mbuf(me),
                    L.chunks[c].msg_bytes, badp + t * N + me, st);
    }
    for (std::size_t me = 0; me < N; ++me) {  // and folds what came from the left
      const std::size_t left = (me + N - 1) % N, c = chunk_at(me, 2 + t);
      decode_into(blob, loc[c], mbuf(left), cbuf(me), 1.0f, st);
      gcx_check(gcx_add_f32(cbuf(me), in.get<float>() + me * d + L.bounds[c],
                            L.bounds[c + 1] - L.bounds[c], st));
    }
  }
  const float divisor = req.op == ReduceOp::average ? float(N) : 1.0f;
  for (std::size_t me = 0; me < N; ++me)  // owners: chunk me, hop N-1
    encode_inline(blob, loc[me], hop_seed(req.step_seed, N - 1, me), cbuf(me),
                  gather.get<std::uint8_t>() + L.gather_offset[me], L.chunks[me].msg_bytes,
                  badp + (N - 1) * N + me, st);
  for (std::size_t me = 0; me < N; ++me)
    for (std::size_t c = 0; c < N; ++c)
      decode_into(blob, full[c], gather.get<std::uint8_t>() + L.gather_offset[c],
                  out.get<float>() + me * d, divisor, st);
  cudaEventRecord(e1, st);
  ReduceResult result;
  result.outputs.assign(N, std::vector<float>(d));
  for (std::size_t k = 0; k < N; ++k)
    cuda_check(cudaMemcpyAsync(result.outputs[k].data(), out.get<float>() + k * d, 4 * d,
                               cudaMemcpyDeviceToHost, st), "D2H");
  std::vector<std::uint64_t> badh(N * N);
  cuda_check(cudaMemcpyAsync(badh.data(), bad.get(), 8 * N * N, cudaMemcpyDeviceToHost, st), "D2H");
  stream.sync();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (std::size_t k = 0; k < N * N; ++k)
    if (badh[k] != ~0ULL) throw_non_finite(loc[0], badh[k]);
  // the reference's counters (collectives.cpp:340-384)
  StepTrace tr;
  tr.bytes_sent.assign(N, 0);
  tr.bytes_received.assign(N, 0);
  for (std::size_t me = 0; me < N; ++me) {
    const std::size_t right = (me + 1) % N;
    for (std::size_t t = 0; t + 1 < N; ++t) {
      const std::uint64_t rs = L.chunks[chunk_at(me, 1 + t)].wire_bytes;  // reduce-scatter
      const std::uint64_t ag = L.chunks[chunk_at(me, t)].wire_bytes;      // forwarded gather
      tr.bytes_sent[me] += rs + ag;
      tr.bytes_received[right] += rs + ag;
      tr.compress_calls += quantized(L.chunks[chunk_at(me, 1 + t)].pieces);
      tr.decompress_calls += quantized(L.chunks[chunk_at(me, 2 + t)].pieces) +
                             quantized(L.chunks[chunk_at(me, 1 + t)].pieces);
    }
    tr.compress_calls += quantized(L.chunks[me].pieces);
    tr.decompress_calls += quantized(L.chunks[me].pieces);
  }
  tr.message_count = 2 * N * (N - 1);
  tr.rounds = 2 * (N - 1);
  // compression depth as the reference propagates it (message notes)
  {
    auto q = [&](std::size_t c) -> std::uint64_t { return quantized(L.chunks[c].pieces) ? 1 : 0; };
    std::vector<std::uint64_t> carry_d(N, 0), sent(N);
    for (std::size_t t = 0; t + 1 < N; ++t) {
      for (std::size_t me = 0; me < N; ++me) sent[me] = carry_d[me] + q(chunk_at(me, 1 + t));
      for (std::size_t me = 0; me < N; ++me) carry_d[me] = sent[(me + N - 1) % N];
    }
    for (std::size_t me = 0; me < N; ++me)
      tr.max_compress_depth = std::max(tr.max_compress_depth, carry_d[me] + q(me));
  }
  tr.device_time_s = ms * 1e-3;
  result.trace = tr;
  return result;
}

// run_tree (collectives.cpp:388-471): binary reduction toward node 0 with a
// re-encode at every level (hop seed (level, me)), then the root encodes
// once (hop `levels`) and every node decodes the same bytes.
ReduceResult allreduce_tree(const ReduceRequest& req, std::size_t N) {
  const std::size_t d = req.inputs[0].size();
  const SraLayout L1 = make_layout(d, 1, req.segments);  // one chunk = the full piece list
  Table full;
  full.pieces = L1.chunks[0].pieces;
  full.plan();
  TableBlob blob;
  blob.upload({&full});
  std::size_t levels = 0;
  while ((std::size_t{1} << levels) < N) ++levels;
  const std::uint64_t mbytes = std::max<std::uint64_t>(L1.chunks[0].msg_bytes, 16);
  const std::uint64_t mstride = align_up(mbytes, kMsgAlign);

  detail::Stream stream;
  cudaStream_t st = stream.get();
  DeviceBuffer acc(4 * d * N + 16), tmp(4 * d + 16), msg(mstride * (N + 1) + 16),
      out(4 * d * N + 16), bad(8 * (N + 1) + 16);
  for (std::size_t k = 0; k < N; ++k)
    cuda_check(cudaMemcpyAsync(acc.get<float>() + k * d, req.inputs[k].data(), 4 * d,
                               cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemsetAsync(bad.get(), 0xFF, bad.size(), st), "memset");
  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0), "event");
  cuda_check(cudaEventCreate(&e1), "event");
  cudaEventRecord(e0, st);
  auto* badp = bad.get<unsigned long long>();
  auto abuf = [&](std::size_t me) { return acc.get<float>() + me * d; };
  auto mbuf = [&](std::size_t me) { return msg.get<std::uint8_t>() + me * mstride; };
  std::vector<bool> sent(N, false);
  for (std::size_t l = 0; l < levels; ++l) {
    const std::size_t stride = std::size_t{1} << l, group = stride << 1;
    for (std::size_t me = 0; me < N; ++me)
      if (!sent[me] && me % group == stride) {
        encode_inline(blob, full, hop_seed(req.step_seed, l, me), abuf(me), mbuf(me), mbytes,
                      badp + me, st);
        sent[me] = true;
      }
    for (std::size_t me = 0; me < N; ++me)
      if (!sent[me] && me % group == 0 && me + stride < N) {
        decode_into(blob, full, mbuf(me + stride), tmp.get<float>(), 1.0f, st);
        gcx_check(gcx_add_f32(abuf(me), tmp.get<float>(), d, st));
      }
  }
  const float divisor = req.op == ReduceOp::average ? float(N) : 1.0f;
  encode_inline(blob, full, hop_seed(req.step_seed, levels, 0), abuf(0), mbuf(N), mbytes, badp + N,
                st);
  for (std::size_t me = 0; me < N; ++me)
    decode_into(blob, full, mbuf(N), out.get<float>() + me * d, divisor, st);
  cudaEventRecord(e1, st);
  ReduceResult result;
  result.outputs.assign(N, std::vector<float>(d));
  for (std::size_t k = 0; k < N; ++k)
    cuda_check(cudaMemcpyAsync(result.outputs[k].data(), out.get<float>() + k * d, 4 * d,
                               cudaMemcpyDeviceToHost, st), "D2H");
  std::vector<std::uint64_t> badh(N + 1);
  cuda_check(cudaMemcpyAsync(badh.data(), bad.get(), 8 * (N + 1), cudaMemcpyDeviceToHost, st), "D2H");
  stream.sync();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (std::size_t k = 0; k <= N; ++k)
    if (badh[k] != ~0ULL) throw_non_finite(full, badh[k]);
  StepTrace tr;
  tr.bytes_sent.assign(N, 0);
  tr.bytes_received.assign(N, 0);
  const std::uint64_t w = L1.chunks[0].wire_bytes, q = quantized(full.pieces);
  for (std::size_t me = 1; me < N; ++me) {  // one upward message per non-root node
    const std::size_t parent = me & (me - 1);
    tr.bytes_sent[me] += w;
    tr.bytes_received[parent] += w;
    tr.bytes_sent[parent] += w;  // and the broadcast back down the same edge
    tr.bytes_received[me] += w;
  }
  tr.message_count = 2 * (N - 1);
  tr.rounds = 2 * levels;
  {  // compression depth: upward notes, then the root's broadcast note
    const std::uint64_t qq = q ? 1 : 0;
    std::vector<std::uint64_t> depth(N, 0);
    std::vector<bool> up(N, false);
    for (std::size_t l = 0; l < levels; ++l) {
      const std::size_t stride = std::size_t{1} << l, group = stride << 1;
      for (std::size_t me = 0; me < N; ++me)
        if (!up[me] && me % group == stride) {
          up[me] = true;
          tr.max_compress_depth = std::max(tr.max_compress_depth, depth[me] + qq);
          depth[me - stride] = std::max(depth[me - stride], depth[me] + qq);
        }
    }
    tr.max_compress_depth = std::max(tr.max_compress_depth, depth[0] + qq);
  }
  tr.compress_calls = N * q;
  tr.decompress_calls = (2 * N - 1) * q;
  tr.device_time_s = ms * 1e-3;
  result.trace = tr;
  return result;
}

}  // namespace

// ---------------------------------------------------------------------------
// sparse path (collectives.cpp:533-603), all nodes on one GPU
// ---------------------------------------------------------------------------
ReduceResult sparse_allreduce(const std::vector<codec::SparseChunk>& chunks, ReduceOp op,
                              std::size_t nodes) {
  if (chunks.size() != nodes) throw std::invalid_argument("expected one sparse chunk per node");
  const std::size_t d = chunks.empty() ? 0 : chunks[0].original_length;
  for (const auto& c : chunks)
    if (c.original_length != d)
      throw std::invalid_argument("sparse chunks disagree on vector length");
  ReduceResult result;
  if (nodes == 1) {
    result.outputs.assign(1, codec::topk_decompress(chunks[0]));
    result.trace.bytes_sent.assign(1, 0);
    result.trace.bytes_received.assign(1, 0);
    return result;
  }
  for (const auto& c : chunks) {  // parse_sparse / topk_decompress validation
    if (c.indices.size() != c.values.size() || c.indices.size() != c.k)
      throw std::runtime_error("sparse chunk index/value arity mismatch");
    for (std::size_t i = 0; i < c.k; ++i) {
      if (c.indices[i] >= d) throw std::runtime_error("sparse index out of range");
      if (i > 0 && c.indices[i] <= c.indices[i - 1])
        throw std::runtime_error("sparse indices must be strictly increasing");
    }
  }
  detail::require_device();
  detail::Stream stream;
  cudaStream_t st = stream.get();
  std::size_t kmax = 1;
  for (const auto& c : chunks) kmax = std::max(kmax, c.k);
  DeviceBuffer out(4 * d + 16), dense(4 * d + 16), idx(4 * kmax + 16), val(4 * kmax + 16);
  cuda_check(cudaMemsetAsync(out.get(), 0, 4 * d, st), "memset");
  std::vector<std::uint32_t> hidx;
  for (std::size_t id = 0; id < nodes; ++id) {  // out[i] += dense_id[i], ascending id
    const auto& c = chunks[id];
    hidx.assign(c.indices.begin(), c.indices.end());
    if (c.k) {
      cuda_check(cudaMemcpyAsync(idx.get(), hidx.data(), 4 * c.k, cudaMemcpyHostToDevice, st), "H2D");
      cuda_check(cudaMemcpyAsync(val.get(), c.values.data(), 4 * c.k, cudaMemcpyHostToDevice, st),
                 "H2D");
    }
    gcx_check(gcx_topk_densify(idx.get<std::uint32_t>(), val.get<float>(), c.k, d,
                               dense.get<float>(), st));
    gcx_check(gcx_add_f32(out.get<float>(), dense.get<float>(), d, st));
    stream.sync();  // hidx is reused
  }
  if (op == ReduceOp::average) gcx_check(gcx_div_f32(out.get<float>(), d, float(nodes), st));
  std::vector<float> host(d);
  cuda_check(cudaMemcpyAsync(host.data(), out.get(), 4 * d, cudaMemcpyDeviceToHost, st), "D2H");
  stream.sync();
  result.outputs.assign(nodes, host);  // every node sums the same chunks in the same order
  StepTrace& tr = result.trace;
  tr.bytes_sent.assign(nodes, 0);
  tr.bytes_received.assign(nodes, 0);
  for (std::size_t me = 0; me < nodes; ++me) {
    const std::uint64_t b = 8 + 8 * chunks[me].k;  // serialize_sparse
    tr.bytes_sent[me] = (nodes - 1) * b;
    for (std::size_t r = 0; r < nodes; ++r)
      if (r != me) tr.bytes_received[r] += b;
  }
  tr.message_count = nodes * (nodes - 1);
  tr.rounds = 1;
  return result;
}

// ---------------------------------------------------------------------------
// all nodes on one GPU
// ---------------------------------------------------------------------------
ReduceResult allreduce(const ReduceRequest& req, std::size_t nodes) {
  if (nodes < 1) throw std::invalid_argument("simnet needs at least one node");
  if (nodes > 64) throw std::invalid_argument("simnet supports at most 64 nodes");
  validate_request(req, nodes);
  ReduceResult result;
  if (nodes == 1) {  // collectives.cpp:479-486: identity, nothing compressed
    result.outputs = req.inputs;
    result.trace.bytes_sent.assign(1, 0);
    result.trace.bytes_received.assign(1, 0);
    return result;
  }
  detail::require_device();
  if (req.topology == Topology::ring) return allreduce_ring(req, nodes);
  if (req.topology == Topology::tree) return allreduce_tree(req, nodes);
  const std::size_t N = nodes, d = req.inputs[0].size();
  const SraLayout L = make_layout(d, N, req.segments);

  // mailbox arena: chunk c holds N-1 slots of stride S_c (one per sender)
  std::vector<std::uint64_t> slot_stride(N), mbase(N);
  std::uint64_t arena = 0;
  for (std::size_t c = 0; c < N; ++c) {
    slot_stride[c] = align_up(std::max<std::uint64_t>(L.chunks[c].msg_bytes, 16), kMsgAlign);
    mbase[c] = arena;
    arena += slot_stride[c] * (N - 1);
  }
  std::vector<Table> send(N), own(N), dec(N);
  std::uint32_t flags = 0;
  std::uint64_t key_len = 0;
  for (std::size_t id = 0; id < N; ++id) {
    for (std::size_t c = 0; c < N; ++c) {
      if (c != id) {
        const std::uint64_t slot = id < c ? id : id - 1;
        append(send[id], L.chunks[c].pieces, mbase[c] + slot * slot_stride[c]);
      }
      append(dec[id], L.chunks[c].pieces, L.gather_offset[c]);  // own chunk too
    }
    own[id] = shifted(L.chunks[id].pieces, 0);
    send[id].plan(true);
    own[id].plan(true, /*keep_span=*/true);
    dec[id].plan();
    flags |= send[id].flags | own[id].flags;
    key_len = std::max({key_len, send[id].key_len, own[id].key_len});
  }
  std::vector<Table*> all;
  for (std::size_t k = 0; k < N; ++k) {
    all.push_back(&send[k]);
    all.push_back(&own[k]);
    all.push_back(&dec[k]);
  }
  TableBlob blob;
  blob.upload(all);

  detail::Stream stream;
  cudaStream_t st = stream.get();
  DeviceBuffer in(4 * d * N + 16), out(4 * d * N + 16), mail(arena + 16),
      gather(L.gather_bytes + 16), bad(16 * N), keys(8 * key_len + 16);
  for (std::size_t k = 0; k < N; ++k)
    cuda_check(cudaMemcpyAsync(in.get<float>() + k * d, req.inputs[k].data(), 4 * d,
                               cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemsetAsync(bad.get(), 0xFF, 16 * N, st), "memset");
  if (flags & GCX_F_NEEDS_ZERO) {
    cuda_check(cudaMemsetAsync(mail.get(), 0, mail.size(), st), "memset");
    cuda_check(cudaMemsetAsync(gather.get(), 0, gather.size(), st), "memset");
  }
  // each node's persistent state, as a DeviceReducer holds it: the
  // seed-independent key prefixes of its send and owner tables
  std::vector<DeviceBuffer> kpre(2 * N);
  for (std::size_t k = 0; k < N; ++k) {
    const Table* tt[2] = {&send[k], &own[k]};
    for (int r = 0; r < 2; ++r) {
      kpre[2 * k + r].reset(8 * tt[r]->key_len + 16);
      gcx_check(gcx_make_key_prefix(blob.groups(*tt[r]), std::uint32_t(tt[r]->groups.size()),
                                    tt[r]->key_len, kpre[2 * k + r].get<unsigned long long>(), st));
    }
  }
  TimedRegion timed(st);
  auto* badp = bad.get<unsigned long long>();
  auto* kp = keys.get<unsigned long long>();
  const float divisor = req.op == ReduceOp::average ? float(N) : 1.0f;
  // stage 1 (scatter): every sender encodes its share of every other chunk
  for (std::size_t id = 0; id < N; ++id)
    encode(blob, send[id], hop_seed(req.step_seed, 0, id), in.get<float>() + id * d,
           mail.get<std::uint8_t>(), kp, badp + id, st, kpre[2 * id].get<unsigned long long>());
  // owners: ascending-id fold into out, re-encode with the hop-1 seed
  for (std::size_t c = 0; c < N; ++c) {
    owner_step(blob, own[c], mail.get<std::uint8_t>() + mbase[c], slot_stride[c],
               in.get<float>() + c * d, N, c, hop_seed(req.step_seed, 1, c),
               gather.get<std::uint8_t>() + L.gather_offset[c], out.get<float>() + c * d, kp,
               badp + N + c, st, kpre[2 * c + 1].get<unsigned long long>());
  }
  // stage 2 (all-gather): everyone decodes every owner's bytes (own included)
  for (std::size_t id = 0; id < N; ++id)
    gcx_check(gcx_decode_pieces(blob.pieces(dec[id]), blob.prefix(dec[id]),
                                std::uint32_t(dec[id].pieces.size()), dec[id].ntiles,
                                dec[id].flags, gather.get<std::uint8_t>(),
                                out.get<float>() + id * d, divisor, st));
  const float ms = timed.end_ms();
  result.outputs.assign(N, std::vector<float>(d));
  for (std::size_t k = 0; k < N; ++k)
    cuda_check(cudaMemcpyAsync(result.outputs[k].data(), out.get<float>() + k * d, 4 * d,
                               cudaMemcpyDeviceToHost, st), "D2H");
  std::vector<std::uint64_t> badh(2 * N);
  cuda_check(cudaMemcpyAsync(badh.data(), bad.get(), 16 * N, cudaMemcpyDeviceToHost, st), "D2H");
  stream.sync();
  for (std::size_t k = 0; k < 2 * N; ++k)
    if (badh[k] != ~0ULL) throw_non_finite(k < N ? send[k] : own[k - N], badh[k]);
  result.trace = sra_trace(L);
  result.trace.device_time_s = ms * 1e-3;
  return result;
}

// ---------------------------------------------------------------------------
// transports
// ---------------------------------------------------------------------------
std::vector<std::uint8_t> Communicator::unique_id() {
  ncclUniqueId id;
  nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
  return std::vector<std::uint8_t>(reinterpret_cast<std::uint8_t*>(&id),
                                   reinterpret_cast<std::uint8_t*>(&id) + sizeof(id));
}

Communicator::Communicator(int rank, int nranks, const std::vector<std::uint8_t>& id)
    : rank_(rank), nranks_(nranks) {
  if (id.size() != sizeof(ncclUniqueId)) throw std::invalid_argument("bad NCCL unique id size");
  detail::require_device();
  ncclUniqueId uid;
  std::memcpy(&uid, id.data(), sizeof(uid));
  ncclComm_t comm;
  nccl_check(ncclCommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  comm_ = comm;
}

Communicator::~Communicator() {
  if (comm_) ncclCommDestroy(static_cast<ncclComm_t>(comm_));
}

void Communicator::exchange(const std::vector<PeerTransfer>& sends,
                            const std::vector<PeerTransfer>& recvs, void* stream) {
  ncclComm_t comm = static_cast<ncclComm_t>(comm_);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  nccl_check(ncclGroupStart(), "ncclGroupStart");
  for (const auto& t : sends)
    nccl_check(ncclSend(t.src, t.bytes, ncclUint8, t.peer, comm, st), "ncclSend");
  for (const auto& t : recvs)
    nccl_check(ncclRecv(t.dst, t.bytes, ncclUint8, t.peer, comm, st), "ncclRecv");
  nccl_check(ncclGroupEnd(), "ncclGroupEnd");
}

std::unique_ptr<Transport> Communicator::split() {
  ncclComm_t child = nullptr;
  nccl_check(ncclCommSplit(static_cast<ncclComm_t>(comm_), 0, rank_, &child, nullptr),
             "ncclCommSplit");
  return std::unique_ptr<Transport>(new Communicator(rank_, nranks_, child));
}

void Communicator::check_async() {
  ncclResult_t r = ncclSuccess;
  nccl_check(ncclCommGetAsyncError(static_cast<ncclComm_t>(comm_), &r), "ncclCommGetAsyncError");
  if (r != ncclSuccess && r != ncclInProgress)
    throw std::runtime_error(std::string("NCCL asynchronous error: ") + ncclGetErrorString(r));
}

struct LoopbackHub::Impl {
  struct Posted {
    std::vector<PeerTransfer> sends, recvs;
  };
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  std::uint64_t gen = 0;
  std::vector<Posted> posted;
  std::vector<cudaEvent_t> ready, done;
  std::vector<std::shared_ptr<LoopbackHub>> children;
  std::vector<std::size_t> nsplit;
};

LoopbackHub::LoopbackHub(int nranks, double timeout_s)
    : n_(nranks), timeout_s_(timeout_s), impl_(std::make_unique<Impl>()) {
  if (nranks < 1) throw std::invalid_argument("loopback needs at least one rank");
  impl_->posted.resize(nranks);
  impl_->ready.assign(nranks, nullptr);
  impl_->done.assign(nranks, nullptr);
  impl_->nsplit.assign(nranks, 0);
}

LoopbackHub::~LoopbackHub() {
  for (auto e : impl_->ready)
    if (e) cudaEventDestroy(e);
  for (auto e : impl_->done)
    if (e) cudaEventDestroy(e);
}

void LoopbackHub::barrier() {
  Impl& I = *impl_;
  std::unique_lock<std::mutex> lk(I.mu);
  const std::uint64_t g = I.gen;
  if (++I.arrived == n_) {
    I.arrived = 0;
    ++I.gen;
    I.cv.notify_all();
    return;
  }
  if (!I.cv.wait_for(lk, std::chrono::duration<double>(timeout_s_), [&] { return I.gen != g; }))
    throw std::runtime_error("loopback transport: peers did not reach the exchange within " +
                             std::to_string(timeout_s_) + " s");
}

std::shared_ptr<LoopbackHub> LoopbackHub::child(int rank) {
  Impl& I = *impl_;
  std::lock_guard<std::mutex> lk(I.mu);
  const std::size_t k = I.nsplit.at(std::size_t(rank))++;
  while (I.children.size() <= k) I.children.push_back(std::make_shared<LoopbackHub>(n_, timeout_s_));
  return I.children[k];
}

// One round for `rank` (its own host thread).  Sends are matched to
// receives exactly as NCCL matches grouped ncclSend/ncclRecv (one message per
// ordered pair, equal sizes); every rank checks the whole round, so a
// mismatch raises the same error on all of them.  The receiver copies from
// the sender's buffer after the sender's stream reached the round (event
// `ready`), and the sender's stream continues only after every receiver
// copied (event `done`): the send buffer is reusable and the receive buffer
// full when the stream leaves the round.
void LoopbackHub::exchange(int rank, const std::vector<PeerTransfer>& sends,
                           const std::vector<PeerTransfer>& recvs, void* stream) {
  Impl& I = *impl_;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(st, &cap), "cudaStreamIsCapturing");
  if (cap != cudaStreamCaptureStatusNone)  // its rounds are host rendezvous between threads
    throw std::logic_error("the loopback transport cannot be captured in a CUDA graph");
  const std::size_t me = std::size_t(rank);
  if (!I.ready[me]) {
    cuda_check(cudaEventCreateWithFlags(&I.ready[me], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&I.done[me], cudaEventDisableTiming), "event");
  }
  I.posted[me].sends = sends;
  I.posted[me].recvs = recvs;
  cuda_check(cudaEventRecord(I.ready[me], st), "event record");
  barrier();
  auto find = [](const std::vector<PeerTransfer>& v, int peer) -> const PeerTransfer* {
    const PeerTransfer* hit = nullptr;
    for (const auto& t : v)
      if (t.peer == peer) {
        if (hit) throw std::runtime_error("loopback transport: two messages for one peer in a round");
        hit = &t;
      }
    return hit;
  };
  for (int r = 0; r < n_; ++r)
    for (const auto& rv : I.posted[std::size_t(r)].recvs) {
      if (rv.peer < 0 || rv.peer >= n_ || rv.peer == r)
        throw std::runtime_error("loopback transport: bad peer " + std::to_string(rv.peer));
      const PeerTransfer* sd = find(I.posted[std::size_t(rv.peer)].sends, r);
      if (!sd || sd->bytes != rv.bytes)
        throw std::runtime_error("loopback transport: rank " + std::to_string(r) + " expects " +
                                 std::to_string(rv.bytes) + " bytes from rank " +
                                 std::to_string(rv.peer) + ", which sends " +
                                 (sd ? std::to_string(sd->bytes) : std::string("nothing")));
    }
  for (int r = 0; r < n_; ++r)
    for (const auto& sd : I.posted[std::size_t(r)].sends)
      if (sd.peer < 0 || sd.peer >= n_ || !find(I.posted[std::size_t(sd.peer)].recvs, r))
        throw std::runtime_error("loopback transport: rank " + std::to_string(r) +
                                 " sends to rank " + std::to_string(sd.peer) +
                                 ", which posted no receive");
  std::uint64_t moved = 0;
  for (const auto& rv : recvs) {
    const PeerTransfer* sd = find(I.posted[std::size_t(rv.peer)].sends, rank);
    cuda_check(cudaStreamWaitEvent(st, I.ready[std::size_t(rv.peer)], 0), "stream wait");
    if (rv.bytes)
      cuda_check(cudaMemcpyAsync(rv.dst, sd->src, rv.bytes, cudaMemcpyDeviceToDevice, st),
                 "loopback copy");
    moved += rv.bytes;
  }
  cuda_check(cudaEventRecord(I.done[me], st), "event record");
  barrier();
  for (const auto& sd : sends)
    cuda_check(cudaStreamWaitEvent(st, I.done[std::size_t(sd.peer)], 0), "stream wait");
  std::lock_guard<std::mutex> lk(I.mu);
  bytes_ += moved;
  if (rank == 0) ++rounds_;
}

LoopbackTransport::LoopbackTransport(std::shared_ptr<LoopbackHub> hub, int rank)
    : hub_(std::move(hub)), rank_(rank) {
  if (!hub_) throw std::invalid_argument("loopback transport needs a hub");
  if (rank < 0 || rank >= hub_->size())
    throw std::invalid_argument("loopback rank " + std::to_string(rank) + " outside [0, " +
                                std::to_string(hub_->size()) + ")");
}

std::unique_ptr<Transport> LoopbackTransport::split() {
  return std::make_unique<LoopbackTransport>(hub_->child(rank_), rank_);
}

ExchangePlan sra_exchange_plan(const SraLayout& L, std::size_t me) {
  const std::size_t N = L.nodes;
  ExchangePlan P;
  if (N <= 1) return P;
  const std::uint64_t m_me = L.chunks[me].msg_bytes;
  P.recv_stride = align_up(std::max<std::uint64_t>(m_me, 16), kMsgAlign);
  for (std::size_t j = 1; j < N; ++j) {
    const std::size_t peer = (me + j) % N, src = (me + N - j) % N;
    // round 1: my share of owner `peer`'s chunk; owner me receives src's share
    if (L.chunks[peer].msg_bytes)
      P.sends[0].push_back({int(peer), Region::send, L.gather_offset[peer], L.chunks[peer].msg_bytes});
    if (m_me)
      P.recvs[0].push_back({int(src), Region::recv, (src < me ? src : src - 1) * P.recv_stride, m_me});
    // round 2: my compressed aggregate to everybody; src's aggregate to me
    if (m_me) P.sends[1].push_back({int(peer), Region::gather, L.gather_offset[me], m_me});
    if (L.chunks[src].msg_bytes)
      P.recvs[1].push_back({int(src), Region::gather, L.gather_offset[src], L.chunks[src].msg_bytes});
  }
  return P;
}

// ---------------------------------------------------------------------------
// one rank per GPU
// ---------------------------------------------------------------------------
struct DeviceReducer::Impl {
  Table send, own, dec;
  TableBlob blob;
  DeviceBuffer send_buf, recv_buf, gather_buf, bad, keys;
  DeviceBuffer prefix_send, prefix_own;  // seed-independent key prefixes, built once
  std::uint64_t recv_stride = 0;
  std::uint32_t flags = 0;
  ExchangePlan plan;
  std::vector<PeerTransfer> sends[2], recvs[2];  // the plan as device pointers
  // non-finite flags of the last call, copied to pinned host memory at its end
  unsigned long long* host_bad = nullptr;
  cudaEvent_t done = nullptr;
  bool pending = false;
  // device-resident step seeds (use_device_seeds): {base, step, buffer, me,
  // hop-0 seed, hop-1 seed}, advanced on the device every call
  DeviceBuffer seed_state;
  bool dev_seeds = false;
  ~Impl() {
    if (host_bad) cudaFreeHost(host_bad);
    if (done) cudaEventDestroy(done);
  }
};

DeviceReducer::DeviceReducer(Transport& transport, std::size_t d, std::vector<Segment> segments)
    : transport_(transport), impl_(std::make_unique<Impl>()) {
  validate_segments(segments, d);
  const std::size_t N = std::size_t(transport.size()), me = std::size_t(transport.rank());
  layout_ = make_layout(d, N, segments);
  if (N == 1) return;
  detail::require_device();
  Impl& I = *impl_;
  for (std::size_t c = 0; c < N; ++c) {
    if (c != me) append(I.send, layout_.chunks[c].pieces, layout_.gather_offset[c]);
    append(I.dec, layout_.chunks[c].pieces, layout_.gather_offset[c]);  // own chunk too
  }
  I.own = shifted(layout_.chunks[me].pieces, 0);
  I.send.plan(true);
  I.own.plan(true, /*keep_span=*/true);
  I.dec.plan();
  I.flags = I.send.flags | I.own.flags;
  I.blob.upload({&I.send, &I.own, &I.dec});
  I.keys.reset(8 * std::max(I.send.key_len, I.own.key_len) + 16);
  I.prefix_send.reset(8 * I.send.key_len + 16);
  I.prefix_own.reset(8 * I.own.key_len + 16);
  gcx_check(gcx_make_key_prefix(I.blob.groups(I.send), std::uint32_t(I.send.groups.size()),
                                I.send.key_len, I.prefix_send.get<unsigned long long>(), nullptr));
  gcx_check(gcx_make_key_prefix(I.blob.groups(I.own), std::uint32_t(I.own.groups.size()),
                                I.own.key_len, I.prefix_own.get<unsigned long long>(), nullptr));
  cuda_check(cudaDeviceSynchronize(), "key prefixes");
  I.plan = sra_exchange_plan(layout_, me);
  I.recv_stride = I.plan.recv_stride;
  I.send_buf.reset(layout_.gather_bytes + 16);
  I.gather_buf.reset(layout_.gather_bytes + 16);
  I.recv_buf.reset(I.recv_stride * (N - 1) + 16);
  I.bad.reset(16);
  cuda_check(cudaMemset(I.bad.get(), 0xFF, 16), "memset");
  cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&I.host_bad), 16, cudaHostAllocDefault),
             "cudaHostAlloc");
  I.host_bad[0] = I.host_bad[1] = ~0ULL;
  cuda_check(cudaEventCreateWithFlags(&I.done, cudaEventDisableTiming), "event");
  std::uint8_t* base[3] = {I.send_buf.get<std::uint8_t>(), I.recv_buf.get<std::uint8_t>(),
                           I.gather_buf.get<std::uint8_t>()};
  for (int r = 0; r < 2; ++r) {
    for (const auto& t : I.plan.sends[r])
      I.sends[r].push_back({t.peer, base[int(t.region)] + t.offset, nullptr, t.bytes});
    for (const auto& t : I.plan.recvs[r])
      I.recvs[r].push_back({t.peer, nullptr, base[int(t.region)] + t.offset, t.bytes});
  }
  if (I.flags & GCX_F_NEEDS_ZERO) {
    cuda_check(cudaMemset(I.send_buf.get(), 0, I.send_buf.size()), "memset");
    cuda_check(cudaMemset(I.gather_buf.get(), 0, I.gather_buf.size()), "memset");
  }
}

DeviceReducer::~DeviceReducer() = default;

namespace {
// NVTX range over one phase of the per-rank step (host-side issue; nsys /
// ncu --nvtx show them around the phase's launches)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

void DeviceReducer::allreduce(const float* in, float* out, std::uint64_t step_seed, ReduceOp op,
                              void* stream) {
  NvtxRange step_range("gcx.sra.step");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const std::size_t N = layout_.nodes, me = std::size_t(transport_.rank()), d = layout_.d;
  if (N == 1) {  // collectives.cpp:479-486: identity, nothing compressed
    if (in != out)
      cuda_check(cudaMemcpyAsync(out, in, 4 * d, cudaMemcpyDeviceToDevice, st), "copy");
    return;
  }
  Impl& I = *impl_;
  const float divisor = op == ReduceOp::average ? float(N) : 1.0f;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(st, &cap), "cudaStreamIsCapturing");
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (capturing && !I.dev_seeds)  // a replay would repeat this step's keys
    throw std::logic_error("capturing a DeviceReducer step needs use_device_seeds()");
  const unsigned long long* seed0 = nullptr;
  const unsigned long long* seed1 = nullptr;
  if (I.dev_seeds) {  // step_seed is not used: the device counter supplies it
    gcx_check(gcx_sra_step_seeds(I.seed_state.get<unsigned long long>(), st));
    seed0 = I.seed_state.get<unsigned long long>() + 4;
    seed1 = seed0 + 1;
  }
  cuda_check(cudaMemsetAsync(I.bad.get(), 0xFF, 16, st), "memset");
  if (I.flags & GCX_F_NEEDS_ZERO) {
    cuda_check(cudaMemsetAsync(I.send_buf.get(), 0, I.send_buf.size(), st), "memset");
    cuda_check(cudaMemsetAsync(I.gather_buf.get<std::uint8_t>() + layout_.gather_offset[me], 0,
                               layout_.chunks[me].msg_bytes, st), "memset");
  }
  auto* bad = I.bad.get<unsigned long long>();
  auto* keys = I.keys.get<unsigned long long>();
  // K1: my share of every other owner's chunk, seed hop_seed(step, 0, me)
  // (collectives.cpp:252-253)
  {
    NvtxRange r("gcx.sra.k1_scatter");
    encode(I.blob, I.send, hop_seed(step_seed, 0, me), in, I.send_buf.get<std::uint8_t>(), keys,
           bad, st, I.prefix_send.get<unsigned long long>(), seed0);
  }
  // round 1: all-to-all of compressed chunks (collectives.cpp:255, :264)
  {
    NvtxRange r("gcx.sra.exchange_scatter");
    transport_.exchange(I.sends[0], I.recvs[0], st);
  }
  // K2: ascending-id fold into out, then re-encode with the hop-1 seed
  // (collectives.cpp:266-284)
  std::uint8_t* bcast = I.gather_buf.get<std::uint8_t>() + layout_.gather_offset[me];
  {
    NvtxRange r("gcx.sra.owner_fold_encode");
    owner_step(I.blob, I.own, I.recv_buf.get<std::uint8_t>(), I.recv_stride, in, N, me,
               hop_seed(step_seed, 1, me), bcast, out, keys, bad + 1, st,
               I.prefix_own.get<unsigned long long>(), seed1);
  }
  // round 2: variable-size all-gather of the owners' compressed aggregates
  // (collectives.cpp:289, :297)
  {
    NvtxRange r("gcx.sra.exchange_allgather");
    transport_.exchange(I.sends[1], I.recvs[1], st);
  }
  // K3: decode every owner's chunk (own included) (+ average)
  {
    NvtxRange r("gcx.sra.k3_decode");
    gcx_check(gcx_decode_pieces(I.blob.pieces(I.dec), I.blob.prefix(I.dec),
                                std::uint32_t(I.dec.pieces.size()), I.dec.ntiles, I.dec.flags,
                                I.gather_buf.get<std::uint8_t>(), out, divisor, st));
  }
  cuda_check(cudaMemcpyAsync(I.host_bad, I.bad.get(), 16, cudaMemcpyDeviceToHost, st), "D2H");
  if (capturing) return;  // each replay copies its flags; check_replay() reads them
  cuda_check(cudaEventRecord(I.done, st), "event record");
  I.pending = true;
}

void DeviceReducer::use_device_seeds(std::uint64_t base_seed, std::uint64_t buffer,
                                     std::uint64_t next_step) {
  const std::size_t N = layout_.nodes;
  if (N == 1) return;  // identity: no keys drawn
  Impl& I = *impl_;
  if (!(I.send.flags & GCX_F_SPAN_ENC) || !(I.own.flags & GCX_F_SPAN_ENC) || N > 8)
    throw std::invalid_argument(
        "device-resident seeds need span tables (one bits/bucket in {32, 64, 128, 512}) and "
        "at most 8 nodes");
  if (I.seed_state.size() == 0) I.seed_state.reset(8 * 8);
  const std::uint64_t h[6] = {base_seed, next_step, buffer, std::uint64_t(transport_.rank()), 0,
                              0};
  cuda_check(cudaMemcpy(I.seed_state.get(), h, sizeof(h), cudaMemcpyHostToDevice), "H2D");
  I.dev_seeds = true;
}

std::uint64_t DeviceReducer::device_step() const {
  const Impl& I = *impl_;
  if (!I.dev_seeds) return 0;
  std::uint64_t h[2] = {0, 0};
  cuda_check(cudaMemcpy(h, I.seed_state.get(), sizeof(h), cudaMemcpyDeviceToHost), "D2H");
  return h[1];
}

void DeviceReducer::check_replay() {
  if (layout_.nodes <= 1) return;
  Impl& I = *impl_;
  for (int k = 0; k < 2; ++k)
    if (I.host_bad[k] != ~0ULL) {
      const unsigned long long key = I.host_bad[k];
      I.host_bad[0] = I.host_bad[1] = ~0ULL;
      throw_non_finite(k == 0 ? I.send : I.own, key);
    }
  transport_.check_async();
}

bool DeviceReducer::poll(bool wait) {
  if (layout_.nodes <= 1 || !impl_->pending) return true;
  Impl& I = *impl_;
  for (;;) {
    const cudaError_t q = cudaEventQuery(I.done);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) cuda_check(q, "cudaEventQuery");
    transport_.check_async();
    if (!wait) return false;
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  I.pending = false;
  for (int k = 0; k < 2; ++k)
    if (I.host_bad[k] != ~0ULL) {
      const unsigned long long key = I.host_bad[k];
      I.host_bad[0] = I.host_bad[1] = ~0ULL;
      throw_non_finite(k == 0 ? I.send : I.own, key);
    }
  return true;
}

StepTrace DeviceReducer::trace() const { return sra_trace(layout_); }

std::uint64_t DeviceReducer::device_bytes_sent() const {
  const std::size_t N = layout_.nodes, me = std::size_t(transport_.rank());
  std::uint64_t b = 0;
  for (std::size_t c = 0; c < N; ++c)
    if (c != me) b += layout_.chunks[c].msg_bytes + layout_.chunks[me].msg_bytes;
  return b;
}

int DeviceReducer::launches_per_call() const {
  if (layout_.nodes <= 1) return 0;
  // per encode (stage 1, owner re-encode): make_keys + K1b (+ norm pre-pass,
  // big-bucket norms, generic K1b as the flags require); fold; decode
  int enc = 2;
  if (impl_->flags & GCX_F_NORM_PASS) ++enc;
  if (impl_->flags & GCX_F_LANE_GROUP) ++enc;
  if (impl_->flags & GCX_F_BIG_BUCKETS) ++enc;
  if (impl_->flags & GCX_F_ODD_BUCKETS) ++enc;
  const int odd = (impl_->flags & GCX_F_ODD_BUCKETS) ? 1 : 0;  // generic fold / decode too
  return 2 * enc + 2 * (1 + odd) + (impl_->dev_seeds ? 1 : 0);  // + gcx_sra_step_seeds
}

}  // namespace gcomm::collectives
