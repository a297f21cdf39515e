// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference sources, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/.
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline), never product code.
//
// It exposes the reference's own codec (src/codec.cpp:24-95) and its SRA
// allreduce through SimNet (src/collectives.cpp:475-494) so the tests can
// validate oracle/cgx_oracle.c against the real thing and bench.py can time
// the reference CPU path.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "gcomm/codec.hpp"
#include "gcomm/collectives.hpp"
#include "gcomm/simnet.hpp"
#include "gcomm/util.hpp"

namespace {
thread_local std::string g_err;
}

extern "C" {

struct ref_segment {
  std::uint64_t offset, length;
  std::int32_t mode, bits;
  std::uint64_t bucket;
};

const char* ref_last_error() { return g_err.c_str(); }

// returns 0 ok, -1 error (message in ref_last_error)
int ref_quantize(const float* v, std::uint64_t n, int bits, std::uint64_t bucket,
                 std::uint64_t seed, float* norms, std::uint8_t* packed) {
  try {
    gcomm::codec::QuantParams p;
    p.bits = bits;
    p.bucket_size = bucket;
    p.seed = seed;
    auto c = gcomm::codec::quantize(std::span<const float>(v, n), p);
    std::memcpy(norms, c.bucket_norms.data(), 4 * c.bucket_norms.size());
    std::memcpy(packed, c.packed_levels.data(), c.packed_levels.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_dequantize(const float* norms, const std::uint8_t* packed, std::uint64_t n, int bits,
                   std::uint64_t bucket, float* out) {
  try {
    gcomm::codec::CompressedChunk c;
    c.element_count = n;
    c.params.bits = bits;
    c.params.bucket_size = bucket;
    const std::size_t nb = n ? (n + bucket - 1) / bucket : 0;
    c.bucket_norms.assign(norms, norms + nb);
    c.packed_levels.assign(packed, packed + (n * (bits + 1) + 7) / 8);
    auto v = gcomm::codec::dequantize(c);
    std::memcpy(out, v.data(), 4 * v.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

std::uint64_t ref_serialize(const float* v, std::uint64_t n, int bits, std::uint64_t bucket,
                            std::uint64_t seed, std::uint8_t* out) {
  gcomm::codec::QuantParams p;
  p.bits = bits;
  p.bucket_size = bucket;
  p.seed = seed;
  auto bytes = gcomm::codec::serialize(gcomm::codec::quantize(std::span<const float>(v, n), p));
  std::memcpy(out, bytes.data(), bytes.size());
  return bytes.size();
}

// SRA allreduce through the reference's SimNet with `nodes` threads.
// outputs: nodes pointers to d floats. bytes_sent: nodes entries.
int ref_allreduce_topo(const float* const* inputs, std::uint64_t nodes, std::uint64_t d,
                       const ref_segment* segs, std::uint64_t nsegs, std::uint64_t step_seed,
                       int op, int topology, float* const* outputs, std::uint64_t* bytes_sent,
                       std::uint64_t* counters);

int ref_allreduce(const float* const* inputs, std::uint64_t nodes, std::uint64_t d,
                  const ref_segment* segs, std::uint64_t nsegs, std::uint64_t step_seed, int op,
                  float* const* outputs, std::uint64_t* bytes_sent, std::uint64_t* counters) {
  return ref_allreduce_topo(inputs, nodes, d, segs, nsegs, step_seed, op, 0, outputs, bytes_sent,
                            counters);
}

// topology: 0 = sra, 1 = ring, 2 = tree (collectives.hpp Topology order)
int ref_allreduce_topo(const float* const* inputs, std::uint64_t nodes, std::uint64_t d,
                       const ref_segment* segs, std::uint64_t nsegs, std::uint64_t step_seed,
                       int op, int topology, float* const* outputs, std::uint64_t* bytes_sent,
                       std::uint64_t* counters) {
  try {
    gcomm::collectives::ReduceRequest req;
    req.inputs.resize(nodes);
    for (std::uint64_t n = 0; n < nodes; ++n) req.inputs[n].assign(inputs[n], inputs[n] + d);
    for (std::uint64_t s = 0; s < nsegs; ++s) {
      gcomm::collectives::Segment seg;
      seg.offset = segs[s].offset;
      seg.length = segs[s].length;
      seg.mode = static_cast<gcomm::model::CodecMode>(segs[s].mode);
      seg.bits = segs[s].bits;
      seg.bucket_size = segs[s].bucket;
      req.segments.push_back(seg);
    }
    req.topology = topology == 1   ? gcomm::collectives::Topology::ring
                   : topology == 2 ? gcomm::collectives::Topology::tree
                                   : gcomm::collectives::Topology::sra;
    req.op = op ? gcomm::collectives::ReduceOp::average : gcomm::collectives::ReduceOp::sum;
    req.step_seed = step_seed;
    gcomm::simnet::SimNetConfig cfg;
    cfg.nodes = nodes;
    gcomm::simnet::SimNet net(cfg);
    auto res = gcomm::collectives::allreduce(req, net);
    for (std::uint64_t n = 0; n < nodes; ++n) {
      std::memcpy(outputs[n], res.outputs[n].data(), 4 * d);
      if (bytes_sent) bytes_sent[n] = res.trace.bytes_sent[n];
    }
    if (counters) {
      counters[0] = res.trace.compress_calls;
      counters[1] = res.trace.decompress_calls;
      counters[2] = res.trace.message_count;
      counters[3] = res.trace.rounds;
      counters[4] = res.trace.max_compress_depth;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// codec::topk_compress (codec.cpp:158-193); residual is updated in place
int ref_topk_compress(const float* v, std::uint64_t n, std::uint64_t k, float* residual,
                      std::uint64_t* idx_out, float* val_out) {
  try {
    gcomm::codec::ErrorFeedbackState st;
    st.residual.assign(residual, residual + n);
    auto c = gcomm::codec::topk_compress(std::span<const float>(v, n), k, st);
    for (std::size_t i = 0; i < c.k; ++i) {
      idx_out[i] = c.indices[i];
      val_out[i] = c.values[i];
    }
    std::memcpy(residual, st.residual.data(), 4 * n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// collectives::sparse_allreduce over SimNet (collectives.cpp:533-603)
int ref_sparse_allreduce(std::uint64_t nodes, std::uint64_t d, const std::uint64_t* ks,
                         const std::uint64_t* const* idx, const float* const* vals, int op,
                         float* const* outputs, std::uint64_t* bytes_sent) {
  try {
    std::vector<gcomm::codec::SparseChunk> chunks(nodes);
    for (std::uint64_t r = 0; r < nodes; ++r) {
      chunks[r].original_length = d;
      chunks[r].k = ks[r];
      chunks[r].indices.assign(idx[r], idx[r] + ks[r]);
      chunks[r].values.assign(vals[r], vals[r] + ks[r]);
    }
    gcomm::simnet::SimNetConfig cfg;
    cfg.nodes = nodes;
    gcomm::simnet::SimNet net(cfg);
    auto res = gcomm::collectives::sparse_allreduce(
        chunks, op ? gcomm::collectives::ReduceOp::average : gcomm::collectives::ReduceOp::sum, net);
    for (std::uint64_t r = 0; r < nodes; ++r) {
      std::memcpy(outputs[r], res.outputs[r].data(), 4 * d);
      if (bytes_sent) bytes_sent[r] = res.trace.bytes_sent[r];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

std::uint64_t ref_hop_seed(std::uint64_t s, std::uint64_t hop, std::uint64_t node) {
  return gcomm::collectives::hop_seed(s, hop, node);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Engine (src/engine.cpp) through SimNet, for end-to-end engine / adaptive
// parity.  Inputs: node r, layer t, step k get
//   scales[t] * normal01(hash_combine(hash_combine(hash_combine(tag, k), r), t), i).
// digests[k] = FNV-1a of node 0's outputs of step k, layers concatenated
// (all nodes are checked identical).  events: the engine's JSONL log.
// ---------------------------------------------------------------------------
#include "gcomm/engine.hpp"

extern "C" int ref_engine_run(int nodes, int nlayers, const char** names, const std::uint64_t* sizes,
                              const int* kinds, const float* scales, int steps, std::uint64_t tag,
                              const char* plan_json, const char* adaptive_json,
                              std::uint64_t step_seed, std::uint64_t fuse_limit,
                              std::uint64_t* digests, char* events, std::uint64_t events_cap) {
  try {
    using namespace gcomm;
    engine::EngineConfig cfg;
    cfg.nodes = nodes;
    cfg.step_seed = step_seed;
    if (fuse_limit) cfg.fuse_limit_bytes = fuse_limit;
    if (plan_json && *plan_json) cfg.plan = model::CompressionPlan::from_json(plan_json);
    if (adaptive_json && *adaptive_json) {
      cfg.plan_source = engine::PlanSource::adaptive;
      cfg.adaptive = adaptive::AdaptiveConfig::from_json(adaptive_json);
    }
    simnet::SimNetConfig net;
    net.nodes = nodes;
    engine::Engine eng(cfg, net);
    for (int k = 0; k < steps; ++k) {
      for (int r = 0; r < nodes; ++r)
        for (int t = 0; t < nlayers; ++t) {
          model::GradientTensor g;
          g.layer.name = names[t];
          g.layer.elements = sizes[t];
          g.layer.kind = static_cast<model::LayerKind>(kinds[t]);
          g.values.resize(sizes[t]);
          const std::uint64_t key = hash_combine(hash_combine(hash_combine(tag, k), r), t);
          for (std::uint64_t i = 0; i < sizes[t]; ++i) g.values[i] = scales[t] * normal01(key, i);
          eng.submit(r, std::move(g));
        }
      std::vector<std::uint8_t> bytes0;
      for (int r = 0; r < nodes; ++r) {
        auto out = eng.flush(r);
        std::vector<std::uint8_t> bytes;
        for (const auto& g : out) {
          const auto* p = reinterpret_cast<const std::uint8_t*>(g.values.data());
          bytes.insert(bytes.end(), p, p + 4 * g.values.size());
        }
        if (r == 0) bytes0 = std::move(bytes);
        else if (bytes != bytes0) throw std::runtime_error("replicas disagree");
      }
      digests[k] = fnv1a64(bytes0);
    }
    const std::string ev = eng.events_json();
    if (events && events_cap) {
      const std::size_t n = std::min<std::size_t>(ev.size(), events_cap - 1);
      std::memcpy(events, ev.data(), n);
      events[n] = 0;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
