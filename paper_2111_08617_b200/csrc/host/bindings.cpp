// bindings.cpp — pybind11 module `_gcomm`: the C++ host façade (gcomm.hpp)
// exposed with the reference's names, so Python tests read like
// /root/reference/proj/tests/*.cpp.  Large vectors cross as numpy arrays.
// Exceptions keep their reference types: std::invalid_argument -> ValueError,
// std::runtime_error -> RuntimeError.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>

#include "engine.hpp"
#include "gcomm.hpp"

namespace py = pybind11;
using namespace gcomm;

namespace {

using farr = py::array_t<float, py::array::c_style | py::array::forcecast>;
using u8arr = py::array_t<std::uint8_t, py::array::c_style | py::array::forcecast>;
using u32arr = py::array_t<std::uint32_t, py::array::c_style | py::array::forcecast>;

template <class T>
py::array_t<T> to_np(const std::vector<T>& v) {
  py::array_t<T> a(v.size());
  if (!v.empty()) std::memcpy(a.mutable_data(), v.data(), v.size() * sizeof(T));
  return a;
}

template <class T, class A>
std::vector<T> from_np(const A& a) {
  return std::vector<T>(a.data(), a.data() + a.size());
}

std::vector<std::uint8_t> bytes_like(py::object o) {
  if (py::isinstance<py::bytes>(o)) {
    std::string s = o.cast<std::string>();
    return std::vector<std::uint8_t>(s.begin(), s.end());
  }
  return from_np<std::uint8_t>(o.cast<u8arr>());
}

}  // namespace

PYBIND11_MODULE(_gcomm, m) {
  m.doc() = "B200 compressed-allreduce host facade (gcomm:: API over libgcx.so)";

  // ---- util.hpp ----
  m.def("mix64", &mix64);
  m.def("hash_combine", &hash_combine);
  m.def("uniform01", &uniform01);
  m.def("normal01", &normal01);
  m.def("fnv1a64", [](py::object o) {
    if (py::isinstance<py::str>(o)) return fnv1a64(o.cast<std::string>());
    py::buffer_info b = py::buffer(o).request();
    return fnv1a64(std::span<const std::uint8_t>(static_cast<const std::uint8_t*>(b.ptr),
                                                 std::size_t(b.size * b.itemsize)));
  });

  // ---- codec ----
  py::class_<codec::QuantParams>(m, "QuantParams")
      .def(py::init([](int bits, std::size_t bucket, std::uint64_t seed) {
             codec::QuantParams p;
             p.bits = bits;
             p.bucket_size = bucket;
             p.seed = seed;
             return p;
           }),
           py::arg("bits") = 4, py::arg("bucket_size") = 128, py::arg("seed") = 0)
      .def_readwrite("bits", &codec::QuantParams::bits)
      .def_readwrite("bucket_size", &codec::QuantParams::bucket_size)
      .def_readwrite("seed", &codec::QuantParams::seed)
      .def("levels", &codec::QuantParams::levels)
      .def("validate", &codec::QuantParams::validate);

  py::class_<codec::CompressedChunk>(m, "CompressedChunk")
      .def(py::init<>())
      .def_readwrite("element_count", &codec::CompressedChunk::element_count)
      .def_readwrite("params", &codec::CompressedChunk::params)
      .def_property(
          "bucket_norms", [](const codec::CompressedChunk& c) { return to_np(c.bucket_norms); },
          [](codec::CompressedChunk& c, farr a) { c.bucket_norms = from_np<float>(a); })
      .def_property(
          "packed_levels", [](const codec::CompressedChunk& c) { return to_np(c.packed_levels); },
          [](codec::CompressedChunk& c, u8arr a) { c.packed_levels = from_np<std::uint8_t>(a); });

  m.def("quantize", [](farr v, const codec::QuantParams& p) {
    return codec::quantize(std::span<const float>(v.data(), std::size_t(v.size())), p);
  });
  m.def("dequantize", [](const codec::CompressedChunk& c) { return to_np(codec::dequantize(c)); });

  py::class_<codec::SparseChunk>(m, "SparseChunk")
      .def(py::init<>())
      .def_readwrite("original_length", &codec::SparseChunk::original_length)
      .def_readwrite("k", &codec::SparseChunk::k)
      .def_property(
          "indices",
          [](const codec::SparseChunk& c) {
            std::vector<std::uint64_t> v(c.indices.begin(), c.indices.end());
            return to_np(v);
          },
          [](codec::SparseChunk& c, py::array_t<std::uint64_t, py::array::c_style | py::array::forcecast> a) {
            c.indices.assign(a.data(), a.data() + a.size());
          })
      .def_property(
          "values", [](const codec::SparseChunk& c) { return to_np(c.values); },
          [](codec::SparseChunk& c, farr a) { c.values = from_np<float>(a); });
  py::class_<codec::ErrorFeedbackState>(m, "ErrorFeedbackState")
      .def(py::init<>())
      .def(py::init<std::size_t>())
      .def_property(
          "residual", [](const codec::ErrorFeedbackState& e) { return to_np(e.residual); },
          [](codec::ErrorFeedbackState& e, farr a) { e.residual = from_np<float>(a); });
  m.def("topk_compress", [](farr v, std::size_t k, codec::ErrorFeedbackState& state) {
    return codec::topk_compress(std::span<const float>(v.data(), std::size_t(v.size())), k, state);
  });
  m.def("topk_decompress", [](const codec::SparseChunk& c) { return to_np(codec::topk_decompress(c)); });
  m.def("pack_levels", [](u32arr levels, u8arr signs, int bits) {
    return to_np(codec::pack_levels(std::span<const std::uint32_t>(levels.data(), levels.size()),
                                    std::span<const std::uint8_t>(signs.data(), signs.size()), bits));
  });
  m.def("unpack_levels", [](py::object packed, std::size_t count, int bits) {
    const auto bytes = bytes_like(packed);
    std::vector<std::uint32_t> levels;
    std::vector<std::uint8_t> signs;
    codec::unpack_levels(bytes, count, bits, levels, signs);
    return py::make_tuple(to_np(levels), to_np(signs));
  });
  m.def("compressed_size_bytes", &codec::compressed_size_bytes);
  m.def("serialized_size_bytes", &codec::serialized_size_bytes);
  m.def("serialize", [](const codec::CompressedChunk& c) {
    const auto b = codec::serialize(c);
    return py::bytes(reinterpret_cast<const char*>(b.data()), b.size());
  });
  m.def("parse_chunk", [](py::object bytes) { return codec::parse_chunk(bytes_like(bytes)); });

  // ---- model ----
  py::enum_<model::LayerKind>(m, "LayerKind")
      .value("weight", model::LayerKind::weight)
      .value("bias", model::LayerKind::bias)
      .value("norm", model::LayerKind::norm)
      .value("embedding", model::LayerKind::embedding)
      .value("other", model::LayerKind::other);
  m.def("layer_kind_from_string", &model::layer_kind_from_string);
  py::enum_<model::CodecMode>(m, "CodecMode")
      .value("quantize", model::CodecMode::quantize)
      .value("topk", model::CodecMode::topk)
      .value("uncompressed", model::CodecMode::uncompressed);
  py::class_<model::LayerSpec>(m, "LayerSpec")
      .def(py::init([](std::string name, std::size_t elements, model::LayerKind kind) {
             return model::LayerSpec{std::move(name), elements, kind};
           }),
           py::arg("name") = "", py::arg("elements") = 0, py::arg("kind") = model::LayerKind::weight)
      .def_readwrite("name", &model::LayerSpec::name)
      .def_readwrite("elements", &model::LayerSpec::elements)
      .def_readwrite("kind", &model::LayerSpec::kind);
  py::class_<model::LayerCodec>(m, "LayerCodec")
      .def(py::init([](model::CodecMode mode, int bits, std::size_t bucket, std::size_t k) {
             return model::LayerCodec{mode, bits, bucket, k};
           }),
           py::arg("mode") = model::CodecMode::quantize, py::arg("bits") = 4,
           py::arg("bucket_size") = 128, py::arg("k") = 0)
      .def_readwrite("mode", &model::LayerCodec::mode)
      .def_readwrite("bits", &model::LayerCodec::bits)
      .def_readwrite("bucket_size", &model::LayerCodec::bucket_size)
      .def_readwrite("k", &model::LayerCodec::k);
  py::class_<model::CompressionPlan>(m, "CompressionPlan")
      .def(py::init<>())
      .def_readwrite("defaults", &model::CompressionPlan::defaults)
      .def_readwrite("overrides", &model::CompressionPlan::overrides)
      .def("resolve", &model::CompressionPlan::resolve)
      .def("set", &model::CompressionPlan::set)
      .def("validate", &model::CompressionPlan::validate)
      .def_static("from_json", &model::CompressionPlan::from_json)
      .def("to_json", &model::CompressionPlan::to_json);
  py::class_<model::FilterRules>(m, "FilterRules")
      .def(py::init<>())
      .def_readwrite("exclude_kinds", &model::FilterRules::exclude_kinds)
      .def_readwrite("min_elements", &model::FilterRules::min_elements)
      .def_readwrite("exclude_patterns", &model::FilterRules::exclude_patterns)
      .def("compile", &model::FilterRules::compile)
      .def("excluded", &model::FilterRules::excluded);
  py::class_<model::BufferSegment>(m, "BufferSegment")
      .def_readonly("tensor_index", &model::BufferSegment::tensor_index)
      .def_readonly("layer_offset", &model::BufferSegment::layer_offset)
      .def_readonly("buffer_offset", &model::BufferSegment::buffer_offset)
      .def_readonly("length", &model::BufferSegment::length);
  py::class_<model::FusedBuffer>(m, "FusedBuffer")
      .def_readonly("segments", &model::FusedBuffer::segments)
      .def_readonly("total_elements", &model::FusedBuffer::total_elements)
      .def_readonly("capacity_bytes", &model::FusedBuffer::capacity_bytes);
  m.def("pack_fused_buffers", &model::pack_fused_buffers);

  // ---- collectives ----
  py::enum_<collectives::Topology>(m, "Topology")
      .value("sra", collectives::Topology::sra)
      .value("ring", collectives::Topology::ring)
      .value("tree", collectives::Topology::tree);
  py::enum_<collectives::ReduceOp>(m, "ReduceOp")
      .value("sum", collectives::ReduceOp::sum)
      .value("average", collectives::ReduceOp::average);
  py::class_<collectives::Segment>(m, "Segment")
      .def(py::init([](std::size_t off, std::size_t len, model::CodecMode mode, int bits,
                       std::size_t bucket) {
             return collectives::Segment{off, len, mode, bits, bucket};
           }),
           py::arg("offset") = 0, py::arg("length") = 0,
           py::arg("mode") = model::CodecMode::quantize, py::arg("bits") = 4,
           py::arg("bucket_size") = 128)
      .def_readwrite("offset", &collectives::Segment::offset)
      .def_readwrite("length", &collectives::Segment::length)
      .def_readwrite("mode", &collectives::Segment::mode)
      .def_readwrite("bits", &collectives::Segment::bits)
      .def_readwrite("bucket_size", &collectives::Segment::bucket_size);
  py::class_<collectives::StepTrace>(m, "StepTrace")
      .def(py::init<>())
      .def_readonly("bytes_sent", &collectives::StepTrace::bytes_sent)
      .def_readonly("bytes_received", &collectives::StepTrace::bytes_received)
      .def_readonly("message_count", &collectives::StepTrace::message_count)
      .def_readonly("rounds", &collectives::StepTrace::rounds)
      .def_readonly("device_time_s", &collectives::StepTrace::device_time_s)
      .def_readonly("compress_calls", &collectives::StepTrace::compress_calls)
      .def_readonly("decompress_calls", &collectives::StepTrace::decompress_calls)
      .def_readonly("max_compress_depth", &collectives::StepTrace::max_compress_depth)
      .def_readonly("device_bytes_sent", &collectives::StepTrace::device_bytes_sent)
      .def("total_bytes_sent", &collectives::StepTrace::total_bytes_sent)
      .def("total_bytes_received", &collectives::StepTrace::total_bytes_received)
      .def("accumulate", &collectives::StepTrace::accumulate);
  py::class_<collectives::ReduceRequest>(m, "ReduceRequest")
      .def(py::init<>())
      .def_property(
          "inputs",
          [](const collectives::ReduceRequest& r) {
            py::list l;
            for (const auto& v : r.inputs) l.append(to_np(v));
            return l;
          },
          [](collectives::ReduceRequest& r, py::list l) {
            r.inputs.clear();
            for (auto item : l) r.inputs.push_back(from_np<float>(item.cast<farr>()));
          })
      .def_readwrite("segments", &collectives::ReduceRequest::segments)
      .def_readwrite("topology", &collectives::ReduceRequest::topology)
      .def_readwrite("op", &collectives::ReduceRequest::op)
      .def_readwrite("step_seed", &collectives::ReduceRequest::step_seed);
  py::class_<collectives::ReduceResult>(m, "ReduceResult")
      .def_property_readonly("outputs",
                             [](const collectives::ReduceResult& r) {
                               py::list l;
                               for (const auto& v : r.outputs) l.append(to_np(v));
                               return l;
                             })
      .def_readonly("trace", &collectives::ReduceResult::trace);
  m.def("hop_seed", &collectives::hop_seed);
  m.def("latency_rounds", &collectives::latency_rounds);
  m.def("chunk_boundaries", &collectives::chunk_boundaries);
  m.def("sra_layout", [](std::size_t d, std::size_t nodes,
                         const std::vector<collectives::Segment>& segs) {
    const auto L = collectives::make_layout(d, nodes, segs);
    py::dict out;
    out["bounds"] = L.bounds;
    out["gather_offset"] = L.gather_offset;
    out["gather_bytes"] = L.gather_bytes;
    std::vector<std::uint64_t> msg, wire, q;
    py::list pieces;
    for (const auto& ch : L.chunks) {
      msg.push_back(ch.msg_bytes);
      wire.push_back(ch.wire_bytes);
      q.push_back(ch.quantized_pieces);
      py::list pl;
      for (const auto& p : ch.pieces)
        pl.append(py::make_tuple(p.src, p.len, p.norms, p.packed, p.bucket, p.bits));
      pieces.append(pl);
    }
    out["msg_bytes"] = msg;
    out["wire_bytes"] = wire;
    out["quantized_pieces"] = q;
    out["pieces"] = pieces;
    const auto tr = collectives::sra_trace(L);
    out["bytes_sent"] = tr.bytes_sent;
    return out;
  });
  m.def("sra_exchange_plan", [](std::size_t d, std::size_t nodes, std::size_t me,
                                std::vector<collectives::Segment> segs) {
    collectives::validate_segments(segs, d);
    const auto L = collectives::make_layout(d, nodes, segs);
    const auto P = collectives::sra_exchange_plan(L, me);
    static const char* region[] = {"send", "recv", "gather"};
    py::dict out;
    out["recv_stride"] = P.recv_stride;
    out["gather_offset"] = L.gather_offset;
    out["gather_bytes"] = L.gather_bytes;
    py::list rounds;
    for (int r = 0; r < 2; ++r) {
      py::list sends, recvs;
      for (const auto& t : P.sends[r])
        sends.append(py::make_tuple(t.peer, region[int(t.region)], t.offset, t.bytes));
      for (const auto& t : P.recvs[r])
        recvs.append(py::make_tuple(t.peer, region[int(t.region)], t.offset, t.bytes));
      py::dict rd;
      rd["sends"] = sends;
      rd["recvs"] = recvs;
      rounds.append(rd);
    }
    out["rounds"] = rounds;
    return out;
  }, py::arg("elements"), py::arg("nodes"), py::arg("me"), py::arg("segments"));
  m.def("allreduce", &collectives::allreduce, py::arg("request"), py::arg("nodes"),
        py::call_guard<py::gil_scoped_release>());
  m.def("sparse_allreduce", &collectives::sparse_allreduce, py::arg("chunks"), py::arg("op"),
        py::arg("nodes"), py::call_guard<py::gil_scoped_release>());

  py::class_<collectives::Transport>(m, "Transport")
      .def("rank", &collectives::Transport::rank)
      .def("size", &collectives::Transport::size)
      .def("kind", &collectives::Transport::kind)
      .def("split", &collectives::Transport::split, py::call_guard<py::gil_scoped_release>())
      .def("check_async", &collectives::Transport::check_async);
  py::class_<collectives::Communicator, collectives::Transport>(m, "Communicator")
      .def(py::init([](int rank, int nranks, py::bytes id) {
             std::string s = id;
             std::vector<std::uint8_t> v(s.begin(), s.end());
             py::gil_scoped_release nogil;
             return std::make_unique<collectives::Communicator>(rank, nranks, v);
           }),
           py::arg("rank"), py::arg("nranks"), py::arg("unique_id"))
      .def_static("unique_id", []() {
        const auto id = collectives::Communicator::unique_id();
        return py::bytes(reinterpret_cast<const char*>(id.data()), id.size());
      });
  py::class_<collectives::LoopbackHub, std::shared_ptr<collectives::LoopbackHub>>(m, "LoopbackHub")
      .def(py::init<int, double>(), py::arg("nranks"), py::arg("timeout_s") = 120.0)
      .def("size", &collectives::LoopbackHub::size)
      .def("rounds", &collectives::LoopbackHub::rounds)
      .def("bytes_moved", &collectives::LoopbackHub::bytes_moved)
      .def("transport", [](std::shared_ptr<collectives::LoopbackHub> hub, int rank) {
        return std::make_unique<collectives::LoopbackTransport>(hub, rank);
      }, py::arg("rank"));
  py::class_<collectives::LoopbackTransport, collectives::Transport>(m, "LoopbackTransport")
      .def(py::init<std::shared_ptr<collectives::LoopbackHub>, int>(), py::arg("hub"),
           py::arg("rank"))
      .def_property_readonly("hub", &collectives::LoopbackTransport::hub);
  py::class_<collectives::DeviceReducer>(m, "DeviceReducer")
      .def(py::init<collectives::Transport&, std::size_t, std::vector<collectives::Segment>>(),
           py::arg("transport"), py::arg("elements"), py::arg("segments"), py::keep_alive<1, 2>())
      .def(
          "allreduce",
          [](collectives::DeviceReducer& r, std::uintptr_t in, std::uintptr_t out,
             std::uint64_t elements, std::uint64_t step_seed, collectives::ReduceOp op,
             std::uintptr_t stream) {
            // the reducer's layout is fixed: a buffer of another length would
            // be read and written out of bounds (advisor finding, ddp hook)
            if (elements != r.elements())
              throw std::invalid_argument("buffer holds " + std::to_string(elements) +
                                          " elements but the reducer was built for " +
                                          std::to_string(r.elements()));
            py::gil_scoped_release nogil;  // loopback ranks rendezvous across threads
            r.allreduce(reinterpret_cast<const float*>(in), reinterpret_cast<float*>(out),
                        step_seed, op, reinterpret_cast<void*>(stream));
          },
          py::arg("in_ptr"), py::arg("out_ptr"), py::arg("elements"), py::arg("step_seed"),
          py::arg("op"), py::arg("stream") = 0)
      .def("poll", &collectives::DeviceReducer::poll, py::arg("wait") = true,
           py::call_guard<py::gil_scoped_release>())
      .def("use_device_seeds", &collectives::DeviceReducer::use_device_seeds,
           py::arg("base_seed"), py::arg("buffer"), py::arg("next_step"))
      .def("device_step", &collectives::DeviceReducer::device_step)
      .def("check_replay", &collectives::DeviceReducer::check_replay)
      .def("elements", &collectives::DeviceReducer::elements)
      .def("trace", &collectives::DeviceReducer::trace)
      .def("device_bytes_sent", &collectives::DeviceReducer::device_bytes_sent)
      .def("launches_per_call", &collectives::DeviceReducer::launches_per_call)
      .def_property_readonly("bounds",
                             [](const collectives::DeviceReducer& r) { return r.layout().bounds; });

  // ---- adaptive ----
  py::class_<adaptive::LayerStats>(m, "LayerStats")
      .def(py::init<>())
      .def_readwrite("name", &adaptive::LayerStats::name)
      .def_readwrite("elements", &adaptive::LayerStats::elements)
      .def_readwrite("l2_norm", &adaptive::LayerStats::l2_norm)
      .def_readwrite("top_fraction_norm", &adaptive::LayerStats::top_fraction_norm);
  py::class_<adaptive::StatsCollector>(m, "StatsCollector")
      .def(py::init<double>(), py::arg("top_fraction") = 0.01)
      .def("add", [](adaptive::StatsCollector& c, const std::string& layer, farr v) {
        c.add(layer, std::span<const float>(v.data(), std::size_t(v.size())));
      })
      .def("add_device",
           [](adaptive::StatsCollector& c, const std::string& layer, std::uintptr_t ptr,
              std::size_t n, std::uintptr_t stream) {
             c.add_device(layer, reinterpret_cast<const float*>(ptr), n,
                          reinterpret_cast<void*>(stream));
           },
           py::arg("layer"), py::arg("ptr"), py::arg("n"), py::arg("stream") = 0)
      .def("finish_step", &adaptive::StatsCollector::finish_step)
      .def("steps", &adaptive::StatsCollector::steps)
      .def("stats", &adaptive::StatsCollector::stats)
      .def("snapshots",
           [](const adaptive::StatsCollector& c) {
             py::dict d;
             for (const auto& kv : c.snapshots()) d[py::str(kv.first)] = to_np(kv.second);
             return d;
           })
      .def("clear", &adaptive::StatsCollector::clear);
  py::class_<adaptive::AdaptiveConfig>(m, "AdaptiveConfig")
      .def(py::init<>())
      .def_readwrite("method", &adaptive::AdaptiveConfig::method)
      .def_readwrite("palette", &adaptive::AdaptiveConfig::palette)
      .def_readwrite("alpha", &adaptive::AdaptiveConfig::alpha)
      .def_readwrite("top_fraction", &adaptive::AdaptiveConfig::top_fraction)
      .def_readwrite("bucket_size", &adaptive::AdaptiveConfig::bucket_size)
      .def_readwrite("reference_bits", &adaptive::AdaptiveConfig::reference_bits)
      .def_readwrite("clusters", &adaptive::AdaptiveConfig::clusters)
      .def_readwrite("stats_period", &adaptive::AdaptiveConfig::stats_period)
      .def_readwrite("stats_window", &adaptive::AdaptiveConfig::stats_window)
      .def_readwrite("pair_buckets", &adaptive::AdaptiveConfig::pair_buckets)
      .def_readwrite("seed", &adaptive::AdaptiveConfig::seed)
      .def_readwrite("probe_seed", &adaptive::AdaptiveConfig::probe_seed)
      .def("validate", &adaptive::AdaptiveConfig::validate)
      .def_static("from_json", &adaptive::AdaptiveConfig::from_json)
      .def("to_json", &adaptive::AdaptiveConfig::to_json);
  py::class_<adaptive::PlanDecision>(m, "PlanDecision")
      .def(py::init<>())
      .def_readwrite("bits", &adaptive::PlanDecision::bits)
      .def_readwrite("buckets", &adaptive::PlanDecision::buckets)
      .def_readwrite("within_budget", &adaptive::PlanDecision::within_budget)
      .def_readwrite("plan_error", &adaptive::PlanDecision::plan_error)
      .def_readwrite("baseline_error", &adaptive::PlanDecision::baseline_error)
      .def_readwrite("compression_ratio", &adaptive::PlanDecision::compression_ratio)
      .def("to_compression_plan", &adaptive::PlanDecision::to_compression_plan)
      .def("to_json", &adaptive::PlanDecision::to_json);
  auto snaps_from = [](py::dict d) {
    std::map<std::string, std::vector<float>> m;
    for (auto kv : d) m[kv.first.cast<std::string>()] = from_np<float>(kv.second.cast<farr>());
    return m;
  };
  m.def("assign_bits_linear", &adaptive::assign_bits_linear);
  m.def("assign_bits_kmeans", &adaptive::assign_bits_kmeans);
  m.def("plan_error", [snaps_from](py::dict snaps, const std::map<std::string, int>& bits,
                                   const std::map<std::string, std::size_t>& buckets,
                                   const adaptive::AdaptiveConfig& cfg) {
    return adaptive::plan_error(snaps_from(snaps), bits, buckets, cfg);
  });
  m.def("build_plan", [snaps_from](const std::vector<adaptive::LayerStats>& stats, py::dict snaps,
                                   const adaptive::AdaptiveConfig& cfg) {
    return adaptive::build_plan(stats, snaps_from(snaps), cfg);
  });

  // ---- engine ----
  py::register_exception<engine::ProtocolError>(m, "ProtocolError", PyExc_RuntimeError);
  py::register_exception<engine::OrderingError>(m, "OrderingError", PyExc_RuntimeError);
  py::enum_<engine::PlanSource>(m, "PlanSource")
      .value("static_plan", engine::PlanSource::static_plan)
      .value("adaptive", engine::PlanSource::adaptive);
  py::class_<engine::EngineConfig>(m, "EngineConfig")
      .def(py::init<>())
      .def_readwrite("nodes", &engine::EngineConfig::nodes)
      .def_readwrite("fuse_limit_bytes", &engine::EngineConfig::fuse_limit_bytes)
      .def_readwrite("cycle_time_s", &engine::EngineConfig::cycle_time_s)
      .def_readwrite("topology", &engine::EngineConfig::topology)
      .def_readwrite("plan_source", &engine::EngineConfig::plan_source)
      .def_readwrite("plan", &engine::EngineConfig::plan)
      .def_readwrite("adaptive", &engine::EngineConfig::adaptive)
      .def_readwrite("filters", &engine::EngineConfig::filters)
      .def_readwrite("step_seed", &engine::EngineConfig::step_seed)
      .def("validate", &engine::EngineConfig::validate);
  py::class_<engine::GradientTensor>(m, "GradientTensor")
      .def(py::init([](model::LayerSpec layer, farr values) {
        return engine::GradientTensor{std::move(layer), from_np<float>(values)};
      }))
      .def_readwrite("layer", &engine::GradientTensor::layer)
      .def_property_readonly("values", [](const engine::GradientTensor& g) { return to_np(g.values); });
  py::class_<engine::EngineEvent>(m, "EngineEvent")
      .def_readonly("step", &engine::EngineEvent::step)
      .def_readonly("event", &engine::EngineEvent::event)
      .def_readonly("payload", &engine::EngineEvent::payload);
  py::class_<engine::PlanSwap>(m, "PlanSwap")
      .def_readonly("step", &engine::PlanSwap::step)
      .def_readonly("decision", &engine::PlanSwap::decision);
  py::class_<engine::Engine>(m, "Engine")
      .def(py::init<engine::EngineConfig>())
      .def("submit", &engine::Engine::submit)
      .def("flush", &engine::Engine::flush)
      .def("steps_completed", &engine::Engine::steps_completed)
      .def("last_trace", &engine::Engine::last_trace)
      .def("total_trace", &engine::Engine::total_trace)
      .def("active_plan", &engine::Engine::active_plan)
      .def("events", &engine::Engine::events)
      .def("events_json", &engine::Engine::events_json)
      .def("plan_history", &engine::Engine::plan_history);
}
