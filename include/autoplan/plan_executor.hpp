// Native (C++) execution of a reference execution plan: the forward pass of
// the graph document (proj/src/graph_ir.cpp:449-573) under the plan document
// plan_to_json writes (proj/src/planner.cpp:455-600), on a MeshRuntime
// (simulated mesh or one NCCL rank). Header-only over the drop-in layout API
// and the C-ABI; parses JSON with nlohmann/json (the reference's own JSON
// dependency -- put its include directory on the path).
//
// What runs, mirroring insert_comm_nodes (planner.cpp:218-352):
//   * every edge whose producer spec differs from what the consumer needs is
//     converted with the reference's path (find_transform_path), collapsed
//     into one exchange (APL_FUSE_CHAIN) or step by step; one conversion per
//     (producer, target spec), shared by its consumers (planner.cpp:299-305);
//   * matmul nodes run their named strategy (intraop.cpp:141-234) as tcgen05
//     GEMMs on the shards, with the partial-sum all-reduce (`<host>.ar`,
//     planner.cpp:263-282); a GELU consuming a non-partial matmul output in
//     the same layout is fused into the GEMM epilogue;
//   * the output node collects to RR (intraop.cpp:469-482).
// The Python PlanExecutor (paper_2302_02599_b200/executor.py) is the same
// algorithm plus the backward pass; tests/test_cpp_plan_executor.py checks
// the two produce identical bytes.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <nlohmann/json.hpp>
#include <set>
#include <string>
#include <vector>

#include "autoplan/execute.hpp"
#include "autoplan/matmul_strategies.hpp"

namespace autoplan {

class PlanExecutor {
 public:
  PlanExecutor(MeshRuntime& rt, const DeviceMesh& mesh, const std::string& graph_json,
               const std::string& plan_json, bool fuse_chain = true)
      : rt_(rt), mesh_(mesh), fuse_(fuse_chain) {
    int n = 0, first = 0, nl = 0, dist = 0;
    apl_detail::check(apl_mesh_info(rt_.get(), &n, &first, &nl, &dist));
    num_local_ = nl;
    const nlohmann::json g = nlohmann::json::parse(graph_json);
    const nlohmann::json p = nlohmann::json::parse(plan_json);
    output_ = g.at("output").get<std::string>();
    for (const auto& node : g.at("nodes")) {
      Node nd;
      nd.id = node.at("id").get<std::string>();
      nd.kind = node.at("kind").get<std::string>();
      for (const auto& in : node.at("inputs")) nd.inputs.push_back(in.at(0).get<std::string>());
      // shapes: declared outputs, else the shape rules of graph_ir.cpp:189-373
      if (!node.at("outputs").empty()) {
        const auto& o = node.at("outputs").at(0);
        nd.meta.shape = o.at("shape").get<std::vector<int64_t>>();
        nd.meta.dtype_bytes = o.at("dtype_bytes").get<int>();
      } else if (nd.kind == "matmul") {
        const TensorMeta& a = nodes_.at(nd.inputs.at(0)).meta;
        const TensorMeta& b = nodes_.at(nd.inputs.at(1)).meta;
        nd.meta = a;
        nd.meta.shape.back() = b.shape.back();
      } else if (nd.kind == "elementwise-unary" || nd.kind == "output") {
        nd.meta = nodes_.at(nd.inputs.at(0)).meta;
      } else {
        throw SchemaError("node kind '" + nd.kind + "' is not executable");
      }
      const auto& pn = p.at("nodes").at(nd.id);
      nd.spec = ShardingSpec::parse(pn.at("spec").get<std::string>(), mesh_.rank());
      if (nd.kind == "matmul") {
        nd.strategy = find_matmul_strategy(pn.at("strategy").get<std::string>(),
                                           nodes_.at(nd.inputs.at(0)).meta,
                                           nodes_.at(nd.inputs.at(1)).meta, mesh_);
        if (!(nd.strategy.output_spec == nd.spec))
          throw ShapeError(nd.id + ": plan spec differs from its strategy's output spec");
      }
      order_.push_back(nd.id);
      for (const auto& in : nd.inputs) consumers_[in].push_back(nd.id);
      nodes_.emplace(nd.id, std::move(nd));
    }
  }

  PlanExecutor(const PlanExecutor&) = delete;
  PlanExecutor& operator=(const PlanExecutor&) = delete;
  ~PlanExecutor() {
    for (auto& [key, bufs] : buffers_)
      for (void* b : bufs) cudaFree(b);
    for (auto& [key, w] : workspaces_) cudaFree(w.first);
  }

  int num_local() const { return num_local_; }
  const ShardingSpec& spec(const std::string& id) const { return nodes_.at(id).spec; }
  const TensorMeta& meta(const std::string& id) const { return nodes_.at(id).meta; }

  // feeds: for every placeholder / parameter, its local shards (one device
  // pointer per local device) in the node's plan spec. Returns the output's
  // local shards (replicated), owned by the executor, valid until the next
  // forward. Stream-ordered on `stream` (a cudaStream_t).
  std::vector<void*> forward(const std::map<std::string, std::vector<const void*>>& feeds,
                             void* stream) {
    std::map<std::string, std::vector<const void*>> values;
    std::map<std::string, std::vector<const void*>> converted;
    std::set<std::string> fused;
    std::vector<void*> result;
    for (const std::string& id : order_) {
      const Node& nd = nodes_.at(id);
      if (nd.kind == "placeholder" || nd.kind == "parameter") {
        const auto& f = feeds.at(id);
        if (static_cast<int>(f.size()) != num_local_)
          throw ShapeError(id + ": expected one shard per local device");
        values[id] = f;
        continue;
      }
      std::vector<std::vector<const void*>> ins;
      for (size_t slot = 0; slot < nd.inputs.size(); ++slot) {
        const std::string& src = nd.inputs[slot];
        const ShardingSpec want = required_spec(nd, slot);
        const ShardingSpec& have = nodes_.at(src).spec;
        if (have == want) {
          ins.push_back(values.at(src));
          continue;
        }
        const std::string key = src + ">" + want.to_string();
        if (!converted.count(key)) converted[key] = convert(src, values.at(src), have, want, stream);
        ins.push_back(converted.at(key));
      }
      if (nd.kind == "matmul") {
        const std::string gelu = fusable_gelu(nd);
        auto out = buffers(id, nd.spec, nd.meta);
        const OpStrategy& st = nd.strategy;
        apl_matmul_strategy c{};
        c.a = apl_detail::to_c(st.input_specs.at(0));
        c.b = apl_detail::to_c(st.input_specs.at(1));
        c.c = apl_detail::to_c(st.output_spec);
        c.partial_sum = st.partial_sum ? 1 : 0;
        c.nreduce = static_cast<int32_t>(st.reduce_axes.size());
        for (size_t i = 0; i < st.reduce_axes.size(); ++i) c.reduce_axes[i] = st.reduce_axes[i];
        const apl_meta am = apl_detail::to_c(nodes_.at(nd.inputs[0]).meta);
        const apl_meta bm = apl_detail::to_c(nodes_.at(nd.inputs[1]).meta);
        apl_detail::check(apl_sharded_matmul_ex(
            rt_.get(), &c, &am, &bm, ins[0].data(), ins[1].data(), out.data(), APL_B_KN,
            nd.meta.dtype_bytes == 4 ? APL_F32 : APL_BF16,
            gelu.empty() ? APL_EPI_NONE : APL_EPI_GELU, nullptr, stream));
        if (!gelu.empty()) fused.insert(gelu);
        values[id] = as_const(out);
      } else if (nd.kind == "elementwise-unary") {
        if (fused.count(id)) {
          values[id] = ins[0];
          continue;
        }
        auto out = buffers(id, nd.spec, nd.meta);
        const size_t count = static_cast<size_t>(nd.spec.per_device_bytes(nd.meta, mesh_) /
                                                 nd.meta.dtype_bytes);
        for (int d = 0; d < num_local_; ++d)
          apl_detail::check(apl_gelu(ins[0][d], out[d], count,
                                     nd.meta.dtype_bytes == 4 ? APL_F32 : APL_BF16, stream));
        values[id] = as_const(out);
      } else {  // output: already collected to RR by the conversion above
        values[id] = ins[0];
        if (id == output_)
          for (const void* v : ins[0]) result.push_back(const_cast<void*>(v));
      }
    }
    return result;
  }

 private:
  struct Node {
    std::string id, kind;
    std::vector<std::string> inputs;
    TensorMeta meta;
    ShardingSpec spec;
    OpStrategy strategy;
  };

  ShardingSpec required_spec(const Node& nd, size_t slot) const {
    if (nd.kind == "matmul") return nd.strategy.input_specs.at(slot);
    if (nd.kind == "output")
      return ShardingSpec::replicated(static_cast<int>(nd.meta.shape.size()), mesh_.rank());
    return nd.spec;  // elementwise: the node's layout mirrored onto its input
  }

  std::string fusable_gelu(const Node& mm) const {
    auto it = consumers_.find(mm.id);
    if (it == consumers_.end() || it->second.size() != 1 || mm.strategy.partial_sum) return "";
    const Node& g = nodes_.at(it->second[0]);
    return g.kind == "elementwise-unary" && g.spec == mm.spec ? g.id : "";
  }

  static std::vector<const void*> as_const(const std::vector<void*>& v) {
    return std::vector<const void*>(v.begin(), v.end());
  }

  std::vector<void*> buffers(const std::string& key, const ShardingSpec& spec,
                             const TensorMeta& meta) {
    auto it = buffers_.find(key);
    if (it != buffers_.end()) return it->second;
    const size_t bytes = static_cast<size_t>(spec.per_device_bytes(meta, mesh_));
    std::vector<void*> bufs(static_cast<size_t>(num_local_));
    for (auto& b : bufs)
      if (cudaMalloc(&b, bytes < 256 ? 256 : bytes) != cudaSuccess)
        throw RuntimeFailure(APL_ERR_CUDA, "cudaMalloc of a plan value failed");
    buffers_.emplace(key, bufs);
    return bufs;
  }

  std::vector<const void*> convert(const std::string& src, const std::vector<const void*>& in,
                                   const ShardingSpec& have, const ShardingSpec& want,
                                   void* stream) {
    const TensorMeta& m = nodes_.at(src).meta;
    const TransformPath path = find_transform_path(have, want, mesh_, m);
    auto out = buffers(src + ">" + want.to_string(), want, m);
    const std::string wkey = src + ">" + want.to_string();
    auto w = workspaces_.find(wkey);
    if (w == workspaces_.end()) {
      const size_t bytes = workspace_bytes(rt_, path, m, fuse_);
      void* ws = nullptr;
      if (cudaMalloc(&ws, bytes < 256 ? 256 : bytes) != cudaSuccess)
        throw RuntimeFailure(APL_ERR_CUDA, "cudaMalloc of a conversion workspace failed");
      w = workspaces_.emplace(wkey, std::make_pair(ws, bytes)).first;
    }
    execute(rt_, path, m, in.data(), out.data(), w->second.first, w->second.second, fuse_,
            stream);
    return as_const(out);
  }

  MeshRuntime& rt_;
  DeviceMesh mesh_;
  bool fuse_;
  int num_local_ = 1;
  std::string output_;
  std::vector<std::string> order_;
  std::map<std::string, Node> nodes_;
  std::map<std::string, std::vector<std::string>> consumers_;
  std::map<std::string, std::vector<void*>> buffers_;
  std::map<std::string, std::pair<void*, size_t>> workspaces_;
};

}  // namespace autoplan
