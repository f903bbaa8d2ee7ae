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
//   * the transformer-block kinds of gpt_block.json run their named strategy
//     on the local shards (intraop.cpp:280-450): reshape = a view, transpose /
//     layernorm / softmax / embedding / elementwise = block_ops kernels,
//     batched matmul = one grouped tcgen05 GEMM per device (+ the split-k
//     all-reduce); the attention chain scale -> u8 mask -> softmax runs as
//     one pass and a sharded embedding table is read from its owners' blocks
//     (simulated mesh) exactly when the Python executor does so;
//   * the output node collects to RR (intraop.cpp:469-482).
// Unary functions are bound by the Python executor's rule (u8 input: not;
// "scale" id behind a batched matmul: 1/sqrt(k); else GELU).
// The Python PlanExecutor (paper_2302_02599_b200/executor.py) is the same
// algorithm plus the backward pass; tests/test_cpp_plan_executor.py checks
// the two produce identical bytes.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <nlohmann/json.hpp>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "autoplan/execute.hpp"
#include "autoplan/matmul_strategies.hpp"

namespace autoplan {

class PlanExecutor {
  struct Node;

 public:
  PlanExecutor(MeshRuntime& rt, const DeviceMesh& mesh, const std::string& graph_json,
               const std::string& plan_json, bool fuse_chain = true)
      : rt_(rt), mesh_(mesh), fuse_(fuse_chain) {
    init(nlohmann::json::parse(graph_json), nlohmann::json::parse(plan_json));
  }

  // From the reference planner's in-memory result: its ComputationGraph
  // (graph_ir.hpp:110-124, GraphNode :92-104) and ExecutionPlan
  // (planner.hpp:99-122), whose node_plans (NodePlan, intraop.hpp:120-127)
  // give every node's output spec and strategy and whose mesh is the
  // DeviceMesh. Templated on both types, so this header needs none of the
  // planner's headers (any types with these members work); the node kinds
  // are named through the reference's own to_string(NodeKind)
  // (graph_ir.cpp:408-413), found by argument-dependent lookup.
  template <class Graph, class Plan,
            class = decltype(std::declval<const Plan&>().node_plans,
                             std::declval<const Graph&>().nodes)>
  PlanExecutor(MeshRuntime& rt, const Graph& graph, const Plan& plan, bool fuse_chain = true)
      : rt_(rt), mesh_(plan.mesh), fuse_(fuse_chain) {
    nlohmann::json g, p;
    g["output"] = graph.output;
    g["nodes"] = nlohmann::json::array();
    for (const auto& n : graph.nodes) {
      nlohmann::json j;
      j["id"] = n.id;
      j["kind"] = std::string(to_string(n.kind));
      j["inputs"] = nlohmann::json::array();
      for (const auto& in : n.inputs) j["inputs"].push_back({in.node, in.out_index});
      j["outputs"] = nlohmann::json::array();
      for (const auto& o : n.outputs)
        j["outputs"].push_back({{"shape", o.shape}, {"dtype_bytes", o.dtype_bytes}});
      j["attrs"] = {{"target_shape", n.attrs.target_shape},
                    {"perm", n.attrs.perm},
                    {"axis", n.attrs.axis}};
      g["nodes"].push_back(std::move(j));
    }
    p["nodes"] = nlohmann::json::object();
    for (const auto& np : plan.node_plans)
      p["nodes"][np.node] = {{"spec", np.spec.to_string()},
                             {"strategy", np.strategy},
                             {"partial_sum", np.partial_sum},
                             {"reduce_axes", np.reduce_axes}};
    init(g, p);
  }

 private:
  void init(const nlohmann::json& g, const nlohmann::json& p) {
    int n = 0, first = 0, nl = 0, dist = 0;
    apl_detail::check(apl_mesh_info(rt_.get(), &n, &first, &nl, &dist));
    num_local_ = nl;
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
      } else if (nd.kind == "batched-matmul") {
        const TensorMeta& a = nodes_.at(nd.inputs.at(0)).meta;
        const TensorMeta& b = nodes_.at(nd.inputs.at(1)).meta;
        nd.meta = a;
        nd.meta.shape = {a.shape.at(0), a.shape.at(1), b.shape.at(2)};
      } else if (nd.kind == "elementwise-unary" || nd.kind == "output" ||
                 nd.kind == "layernorm" || nd.kind == "softmax") {
        nd.meta = nodes_.at(nd.inputs.at(0)).meta;
      } else if (nd.kind == "elementwise-binary") {
        nd.meta = nodes_.at(nd.inputs.at(0)).meta;
        nd.meta.dtype_bytes =
            std::max(nd.meta.dtype_bytes, nodes_.at(nd.inputs.at(1)).meta.dtype_bytes);
      } else if (nd.kind == "reshape") {
        nd.meta = nodes_.at(nd.inputs.at(0)).meta;
        nd.meta.shape = node.at("attrs").at("target_shape").get<std::vector<int64_t>>();
      } else if (nd.kind == "transpose") {
        const TensorMeta& in = nodes_.at(nd.inputs.at(0)).meta;
        nd.meta = in;
        nd.perm = node.at("attrs").at("perm").get<std::vector<int64_t>>();
        for (size_t i = 0; i < nd.perm.size(); ++i)
          nd.meta.shape[i] = in.shape.at(static_cast<size_t>(nd.perm[i]));
      } else if (nd.kind == "embedding-lookup") {
        const TensorMeta& ids = nodes_.at(nd.inputs.at(0)).meta;
        const TensorMeta& table = nodes_.at(nd.inputs.at(1)).meta;
        nd.meta = table;
        nd.meta.shape = ids.shape;
        nd.meta.shape.push_back(table.shape.at(1));
      } else {
        throw SchemaError("node kind '" + nd.kind + "' is not executable");
      }
      // attributes are read whether or not the outputs were declared (an
      // in-memory graph after infer_meta carries every node's outputs)
      if (nd.kind == "transpose")
        nd.perm = node.at("attrs").at("perm").get<std::vector<int64_t>>();
      if (node.contains("attrs") && node.at("attrs").contains("axis"))
        nd.axis = node.at("attrs").at("axis").get<int64_t>();
      const auto& pn = p.at("nodes").at(nd.id);
      nd.spec = ShardingSpec::parse(pn.at("spec").get<std::string>(), mesh_.rank());
      const std::string name = pn.at("strategy").get<std::string>();
      if (nd.kind == "matmul" || nd.kind == "batched-matmul") {
        nd.strategy = find_matmul_strategy(name, nodes_.at(nd.inputs.at(0)).meta,
                                           nodes_.at(nd.inputs.at(1)).meta, mesh_,
                                           nd.kind == "batched-matmul");
        if (!(nd.strategy.output_spec == nd.spec))
          throw ShapeError(nd.id + ": plan spec differs from its strategy's output spec");
        nd.in_specs = nd.strategy.input_specs;
      } else if (nd.kind != "placeholder" && nd.kind != "parameter") {
        nd.in_specs = input_specs(nd, name);
      }
      order_.push_back(nd.id);
      for (const auto& in : nd.inputs) consumers_[in].push_back(nd.id);
      nodes_.emplace(nd.id, std::move(nd));
    }
    for (auto& [id, nd] : nodes_)
      if (nd.kind == "elementwise-unary") bind_unary(nd);
    find_attention_chains();
  }

 public:

  PlanExecutor(const PlanExecutor&) = delete;
  PlanExecutor& operator=(const PlanExecutor&) = delete;
  ~PlanExecutor() {
    for (auto& [key, bufs] : buffers_)
      for (void* b : bufs) cudaFree(b);
    for (auto& [key, w] : workspaces_) cudaFree(w.first);
  }

  int num_local() const { return num_local_; }

  // backward() computes in bf16 (gradient buffers, GELU / softmax /
  // layernorm backward kernels, transposes of 2-byte elements), so a
  // training forward refuses plans whose differentiable values -- parameters
  // and computed nodes; u8 masks and placeholders (ids, inputs) are not
  // differentiated -- have any other width, instead of reading fp32 buffers
  // as bf16.
  void check_trainable() const {
    for (const auto& id : order_) {
      const Node& nd = nodes_.at(id);
      if (nd.kind == "placeholder" || nd.meta.dtype_bytes == 1) continue;
      if (nd.meta.dtype_bytes != 2)
        throw PlanError("backward supports bf16 plans only: node '" + id + "' has dtype_bytes " +
                        std::to_string(nd.meta.dtype_bytes));
    }
  }
  const ShardingSpec& spec(const std::string& id) const { return nodes_.at(id).spec; }
  const TensorMeta& meta(const std::string& id) const { return nodes_.at(id).meta; }
  // placeholders and parameters, in graph order (what forward() must be fed)
  std::vector<std::string> sources() const {
    std::vector<std::string> out;
    for (const auto& id : order_) {
      const std::string& k = nodes_.at(id).kind;
      if (k == "placeholder" || k == "parameter") out.push_back(id);
    }
    return out;
  }

  // feeds: for every placeholder / parameter, its local shards (one device
  // pointer per local device) in the node's plan spec. Returns the output's
  // local shards (replicated), owned by the executor, valid until the next
  // forward. Stream-ordered on `stream` (a cudaStream_t).
  // train = true keeps what backward() reads (the Python executor's rule:
  // matmul / batched-matmul / layernorm operands as consumed, GELU
  // pre-activations -- a fused GELU's epilogue stores it -- softmax outputs,
  // embedding ids) and runs the attention chain unfused.
  std::vector<void*> forward(const std::map<std::string, std::vector<const void*>>& feeds,
                             void* stream, bool train = false) {
    if (train) check_trainable();
    saved_.clear();
    trained_ = train;
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
      if (!train && attn_members_.count(id)) continue;  // inside the fused softmax below
      if (auto ch = attn_.find(id); !train && ch != attn_.end()) {
        auto out = buffers(id, nd.spec, nd.meta);
        const auto& x = values.at(ch->second.x);
        const auto& m = values.at(ch->second.mask);
        const auto sh = local_shape(nd.spec, nd.meta);
        const int64_t w = sh.back(), rows = numel(sh) / w;
        for (int d = 0; d < num_local_; ++d)
          apl_detail::check(apl_softmax_ex(x[d], out[d], rows, w, ch->second.alpha, m[d],
                                           kMaskFill, dtype_of(nd.meta), stream));
        values[id] = as_const(out);
        continue;
      }
      const bool gather_t = nd.kind == "embedding-lookup" && gatherable_table(nd);
      std::vector<std::vector<const void*>> ins;
      for (size_t slot = 0; slot < nd.inputs.size(); ++slot) {
        const std::string& src = nd.inputs[slot];
        const ShardingSpec want = required_spec(nd, slot);
        const ShardingSpec& have = nodes_.at(src).spec;
        if (have == want || (slot == 1 && gather_t)) {
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
        std::vector<void*> pre;
        if (train) {
          saved_[id] = {ins[0], ins[1]};
          if (!gelu.empty()) {  // one pass writes GELU(acc) and keeps acc for backward
            pre = buffers(id + ".pre", nd.spec, nd.meta);
            saved_[gelu] = {as_const(pre)};
          }
        }
        apl_detail::check(apl_sharded_matmul_ex(
            rt_.get(), &c, &am, &bm, ins[0].data(), ins[1].data(), out.data(), APL_B_KN,
            nd.meta.dtype_bytes == 4 ? APL_F32 : APL_BF16,
            gelu.empty() ? APL_EPI_NONE : (pre.empty() ? APL_EPI_GELU : APL_EPI_GELU_SAVE),
            pre.empty() ? nullptr : pre.data(), stream));
        if (!gelu.empty()) fused.insert(gelu);
        values[id] = as_const(out);
      } else if (nd.kind == "elementwise-unary") {
        if (fused.count(id)) {
          values[id] = ins[0];
          continue;
        }
        auto out = buffers(id, nd.spec, nd.meta);
        const size_t count = static_cast<size_t>(numel(local_shape(nd.spec, nd.meta)));
        for (int d = 0; d < num_local_; ++d) {
          if (nd.unary == Unary::kGelu)
            apl_detail::check(apl_gelu(ins[0][d], out[d], count, dtype_of(nd.meta), stream));
          else if (nd.unary == Unary::kScale)
            apl_detail::check(
                apl_scale(ins[0][d], out[d], count, nd.alpha, dtype_of(nd.meta), stream));
          else
            apl_detail::check(apl_mask_not(ins[0][d], out[d], count, stream));
        }
        if (train && nd.unary == Unary::kGelu) saved_[id] = {ins[0]};  // the pre-activation
        values[id] = as_const(out);
      } else if (nd.kind == "output") {  // already collected to RR by the conversion above
        values[id] = ins[0];
        if (id == output_)
          for (const void* v : ins[0]) result.push_back(const_cast<void*>(v));
      } else if (nd.kind == "reshape") {  // a view: the plan's rewritten local shape
        values[id] = ins[0];
      } else if (nd.kind == "embedding-lookup" && gather_t) {
        values[id] = lookup_gathered_table(nd, ins[0], values.at(nd.inputs[1]), stream);
        if (train) saved_[id] = {ins[0]};
      } else {
        values[id] = block_node(nd, ins, stream);
        if (train) {
          if (nd.kind == "batched-matmul" || nd.kind == "layernorm") saved_[id] = ins;
          else if (nd.kind == "embedding-lookup") saved_[id] = {ins[0]};
          else if (nd.kind == "softmax") saved_[id] = {values[id]};
        }
      }
    }
    return result;
  }

  // Backward of the last forward(train = true): grad_out = the output's
  // gradient, one bf16 RR shard per local device. Returns every parameter's
  // gradient (fp32, in its plan spec), owned by the executor -- the
  // Python PlanExecutor.backward algorithm step for step (same kernels, same
  // order, same bytes): reverse graph walk, per-node input gradients in the
  // layouts the strategy consumed, partial sums reduced where they are made,
  // reverse conversions back to the producers' layouts, out-of-place sums for
  // values with several consumers.
  std::map<std::string, std::vector<void*>> backward(const std::vector<const void*>& grad_out,
                                                     void* stream) {
    if (!trained_) throw PlanError("backward() needs a preceding forward(train = true)");
    if (static_cast<int>(grad_out.size()) != num_local_)
      throw ShapeError("grad_out: expected one shard per local device");
    gcount_ = 0;
    const Node& out = nodes_.at(output_);
    const std::string src = out.inputs.at(0);
    std::map<std::string, Grad> grads;
    grads[src] = convert_grad(src, Grad{grad_out, 2}, required_spec(out, 0), nodes_.at(src).spec,
                              stream);
    std::set<std::string> done;
    auto wants = [&](const std::string& id) {
      const std::string& k = nodes_.at(id).kind;
      return k != "placeholder";  // parameters and every computed value
    };
    auto add = [&](const std::string& id, const Grad& g) {
      auto it = grads.find(id);
      if (it == grads.end()) {
        grads[id] = g;
        return;
      }
      if (it->second.eb != g.eb) throw PlanError(id + ": gradient dtypes differ");
      const size_t count = static_cast<size_t>(numel(local_shape(nodes_.at(id).spec,
                                                                 nodes_.at(id).meta)));
      const size_t bytes = count * static_cast<size_t>(g.eb);
      std::vector<const void*> sum;
      for (int d = 0; d < num_local_; ++d) {
        void* o = grad_buf(bytes);
        apl_detail::check(apl_add(it->second.p[d], g.p[d], 0, o, count, 1.f,
                                  g.eb == 4 ? APL_F32 : APL_BF16, stream));
        sum.push_back(o);
      }
      it->second.p = sum;
    };
    for (auto r = order_.rbegin(); r != order_.rend(); ++r) {
      const std::string& id = *r;
      if (done.count(id) || !grads.count(id)) continue;
      const Node& nd = nodes_.at(id);
      const Grad dy = grads.at(id);
      if (nd.kind == "matmul") {
        const OpStrategy& st = nd.strategy;
        const auto& sv = saved_.at(id);
        const std::string a_src = nd.inputs[0], b_src = nd.inputs[1];
        const Node& an = nodes_.at(a_src);
        std::string a_target = a_src;
        const std::vector<const void*>* aux = nullptr;
        auto cons = consumers_.find(a_src);
        if (an.kind == "elementwise-unary" && an.unary == Unary::kGelu &&
            an.spec == st.input_specs[0] && cons != consumers_.end() &&
            cons->second.size() == 1 && saved_.count(a_src)) {
          aux = &saved_.at(a_src)[0];
          a_target = an.inputs[0];
          done.insert(a_src);
        }
        const bool need_a = wants(a_target), need_b = wants(b_src);
        const TensorMeta& am = nodes_.at(a_src).meta;
        const TensorMeta& bm = nodes_.at(b_src).meta;
        std::vector<void*> ga, gb;
        if (need_a)
          for (int d = 0; d < num_local_; ++d)
            ga.push_back(grad_buf(static_cast<size_t>(numel(local_shape(st.input_specs[0], am))) *
                                  2));
        if (need_b)
          for (int d = 0; d < num_local_; ++d)
            gb.push_back(grad_buf(static_cast<size_t>(numel(local_shape(st.input_specs[1], bm))) *
                                  4));
        if (need_a || need_b) {
          apl_matmul_strategy c = to_c_strategy(st);
          const apl_meta amc = apl_detail::to_c(am), bmc = apl_detail::to_c(bm);
          apl_detail::check(apl_sharded_matmul_backward(
              rt_.get(), &c, &amc, &bmc, sv[0].data(), sv[1].data(), dy.p.data(),
              need_a ? ga.data() : nullptr, need_b ? gb.data() : nullptr, APL_B_KN,
              aux ? APL_EPI_DGELU : APL_EPI_NONE, aux ? aux->data() : nullptr, APL_F32, stream));
        }
        if (need_a)
          add(a_target, convert_grad(a_target, Grad{as_const(ga), 2}, st.input_specs[0],
                                     nodes_.at(a_target).spec, stream));
        if (need_b)
          add(b_src, convert_grad(b_src, Grad{as_const(gb), 4}, st.input_specs[1],
                                  nodes_.at(b_src).spec, stream));
      } else if (nd.kind == "elementwise-unary" && nd.unary == Unary::kGelu) {
        const std::string x = nd.inputs[0];
        const auto& pre = saved_.at(id)[0];
        const size_t count = static_cast<size_t>(numel(local_shape(nd.spec, nd.meta)));
        std::vector<const void*> dx;
        for (int d = 0; d < num_local_; ++d) {
          void* o = grad_buf(count * 2);
          apl_detail::check(apl_gelu_backward(dy.p[d], pre[d], o, count, APL_BF16, stream));
          dx.push_back(o);
        }
        add(x, convert_grad(x, Grad{dx, 2}, nd.spec, nodes_.at(x).spec, stream));
      } else if (nd.kind != "output" && nd.kind != "placeholder" && nd.kind != "parameter") {
        for (auto& [slot, g, layout] : block_backward(nd, dy, wants, stream)) {
          const std::string& in = nd.inputs[static_cast<size_t>(slot)];
          add(in, convert_grad(in, g, layout, nodes_.at(in).spec, stream));
        }
      }
    }
    std::map<std::string, std::vector<void*>> result;
    for (auto& [id, g] : grads)
      if (nodes_.at(id).kind == "parameter") {
        std::vector<void*> v;
        for (const void* q : g.p) v.push_back(const_cast<void*>(q));
        result[id] = v;
      }
    return result;
  }

 private:
  struct Grad {
    std::vector<const void*> p;
    int eb = 2;  // element bytes: 2 bf16 (activations), 4 fp32 (parameters)
  };

  static apl_matmul_strategy to_c_strategy(const OpStrategy& st) {
    apl_matmul_strategy c{};
    c.a = apl_detail::to_c(st.input_specs.at(0));
    c.b = apl_detail::to_c(st.input_specs.at(1));
    c.c = apl_detail::to_c(st.output_spec);
    c.partial_sum = st.partial_sum ? 1 : 0;
    c.nreduce = static_cast<int32_t>(st.reduce_axes.size());
    for (size_t i = 0; i < st.reduce_axes.size(); ++i) c.reduce_axes[i] = st.reduce_axes[i];
    return c;
  }

  // gradient scratch: one cached buffer per allocation index of a backward
  // pass (the sequence repeats every step, so buffers are reused)
  void* grad_buf(size_t bytes) {
    const std::string key = "grad#" + std::to_string(gcount_++);
    auto it = workspaces_.find(key);
    if (it != workspaces_.end() && it->second.second >= bytes) return it->second.first;
    if (it != workspaces_.end()) {
      cudaFree(it->second.first);
      workspaces_.erase(it);
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes < 256 ? 256 : bytes) != cudaSuccess)
      throw RuntimeFailure(APL_ERR_CUDA, "cudaMalloc of a gradient buffer failed");
    workspaces_.emplace(key, std::make_pair(p, bytes));
    return p;
  }

  void* grad_zeros(size_t bytes, void* stream) {
    void* p = grad_buf(bytes);
    if (cudaMemsetAsync(p, 0, bytes, static_cast<cudaStream_t>(stream)) != cudaSuccess)
      throw RuntimeFailure(APL_ERR_CUDA, "memset of a gradient accumulator failed");
    return p;
  }

  // A gradient held in `have` into `want`: the reverse conversion (a layout
  // conversion is the identity on the global tensor; its adjoint is too).
  Grad convert_grad(const std::string& id, const Grad& g, const ShardingSpec& have,
                    const ShardingSpec& want, void* stream) {
    if (have == want) return g;
    TensorMeta m = nodes_.at(id).meta;
    m.dtype_bytes = g.eb;
    const CachedPath& cp = cached_path(id, have, want, m);
    const size_t out_b = static_cast<size_t>(want.per_device_bytes(m, mesh_));
    std::vector<void*> out;
    for (int d = 0; d < num_local_; ++d) out.push_back(grad_buf(out_b));
    void* ws = grad_buf(cp.ws < 256 ? 256 : cp.ws);
    execute(rt_, cp.path, m, g.p.data(), out.data(), ws, cp.ws, fuse_, stream);
    return Grad{as_const(out), g.eb};
  }

  struct SlotGrad {
    int slot;
    Grad g;
    ShardingSpec layout;
  };

  // input gradients of one block node (PlanExecutor._block_backward)
  template <typename Wants>
  std::vector<SlotGrad> block_backward(const Node& nd, const Grad& dy, Wants wants,
                                       void* stream) {
    std::vector<SlotGrad> out;
    const auto ls = local_shape(nd.spec, nd.meta);
    const size_t count = static_cast<size_t>(numel(ls));
    if (nd.kind == "reshape") {
      out.push_back({0, dy, required_spec(nd, 0)});
    } else if (nd.kind == "transpose") {
      // dx = dy permuted back: inverse permutation of the output's layout
      std::vector<int64_t> inv(nd.perm.size());
      for (size_t k = 0; k < nd.perm.size(); ++k) inv[static_cast<size_t>(nd.perm[k])] = static_cast<int64_t>(k);
      std::vector<const void*> dx;
      for (int d = 0; d < num_local_; ++d) {
        void* o = grad_buf(count * 2);
        permute(dy.p[d], o, ls, inv, 2, stream);
        dx.push_back(o);
      }
      out.push_back({0, Grad{dx, 2}, required_spec(nd, 0)});
    } else if (nd.kind == "elementwise-unary") {
      if (nd.unary == Unary::kScale && wants(nd.inputs[0])) {
        std::vector<const void*> dx;
        for (int d = 0; d < num_local_; ++d) {
          void* o = grad_buf(count * 2);
          apl_detail::check(apl_scale(dy.p[d], o, count, nd.alpha, APL_BF16, stream));
          dx.push_back(o);
        }
        out.push_back({0, Grad{dx, 2}, required_spec(nd, 0)});
      }
    } else if (nd.kind == "elementwise-binary") {
      for (int slot = 0; slot < 2; ++slot) {
        const std::string& in = nd.inputs[static_cast<size_t>(slot)];
        if (nodes_.at(in).meta.dtype_bytes != 1 && wants(in))
          out.push_back({slot, dy, required_spec(nd, static_cast<size_t>(slot))});
      }
    } else if (nd.kind == "softmax") {
      const auto& y = saved_.at(nd.id)[0];
      const int64_t so = axis_outer(ls, nd.axis), sn = ls[axis_of(ls, nd.axis)],
                    si = numel(ls) / (so * sn);
      std::vector<const void*> dx;
      for (int d = 0; d < num_local_; ++d) {
        void* o = grad_buf(count * 2);
        apl_detail::check(
            apl_softmax_axis_backward(y[d], dy.p[d], o, so, sn, si, 1.f, APL_BF16, stream));
        dx.push_back(o);
      }
      out.push_back({0, Grad{dx, 2}, required_spec(nd, 0)});
    } else if (nd.kind == "layernorm") {
      const auto& sv = saved_.at(nd.id);
      const int64_t h = ls.back(), rows = numel(ls) / h;
      const bool has_g = sv.size() > 1, has_b = sv.size() > 2;
      std::vector<const void*> dx;
      std::vector<void*> dg, db;
      for (int d = 0; d < num_local_; ++d) {
        void* o = grad_buf(count * 2);
        void* g = has_g ? grad_zeros(static_cast<size_t>(h) * 4, stream) : nullptr;
        void* b = has_b ? grad_zeros(static_cast<size_t>(h) * 4, stream) : nullptr;
        size_t sb = 0;
        if (has_g || has_b) apl_detail::check(apl_layernorm_backward_scratch(rows, h, &sb));
        void* stats = has_g || has_b ? grad_buf(sb) : nullptr;
        apl_detail::check(apl_layernorm_backward_ex(sv[0][d], has_g ? sv[1][d] : nullptr,
                                                    dy.p[d], o, static_cast<float*>(g),
                                                    static_cast<float*>(b), stats, sb, rows, h,
                                                    1e-5f, APL_BF16, stream));
        dx.push_back(o);
        if (has_g) dg.push_back(g);
        if (has_b) db.push_back(b);
      }
      out.push_back({0, Grad{dx, 2}, required_spec(nd, 0)});
      std::set<int> axes_set;
      const ShardingSpec in0 = required_spec(nd, 0);
      for (size_t k = 0; k + 1 < in0.dims.size(); ++k)
        for (int a : in0.dims[k].axes) axes_set.insert(a);
      std::vector<int32_t> axes(axes_set.begin(), axes_set.end());
      for (int slot = 1; slot <= 2; ++slot) {
        std::vector<void*>& pg = slot == 1 ? dg : db;
        if (pg.empty() || !wants(nd.inputs[static_cast<size_t>(slot)])) continue;
        if (!axes.empty())
          apl_detail::check(apl_all_reduce(rt_.get(), axes.data(), static_cast<int>(axes.size()),
                                           pg.data(), static_cast<size_t>(h), APL_F32, stream));
        out.push_back({slot, Grad{as_const(pg), 4}, required_spec(nd, static_cast<size_t>(slot))});
      }
    } else if (nd.kind == "embedding-lookup") {
      const auto& ids = saved_.at(nd.id)[0];
      const std::string& tab = nd.inputs[1];
      const ShardingSpec tspec = required_spec(nd, 1);
      const ShardingSpec& tplan = nodes_.at(tab).spec;
      const TensorMeta& tm = nodes_.at(tab).meta;
      const int64_t n = numel(ls) / ls.back();
      int nn = 0, first = 0, nl = 0, dist = 0;
      apl_detail::check(apl_mesh_info(rt_.get(), &nn, &first, &nl, &dist));
      if (wants(tab) && !dist && tspec.dims[1].replicated() && !(tplan == tspec)) {
        // reduce-scatter fused: each owner block from every distinct id block
        const ShardingSpec ispec = required_spec(nd, 0);
        std::map<std::vector<int64_t>, int> srcs;
        for (int d = 0; d < num_local_; ++d) {
          std::vector<int64_t> key;
          for (const auto& dim : ispec.dims) key.push_back(block_index(dim, d).first);
          srcs.emplace(key, d);
        }
        std::vector<int> order;
        for (auto& [k, d] : srcs) order.push_back(d);
        std::sort(order.begin(), order.end());
        std::vector<const int64_t*> sid;
        std::vector<const void*> sdy;
        for (int d : order) {
          sid.push_back(static_cast<const int64_t*>(ids[d]));
          sdy.push_back(dy.p[d]);
        }
        const int64_t vocab = tm.shape[0], width = tm.shape[1];
        std::vector<const void*> blks;
        for (int d = 0; d < num_local_; ++d) {
          const auto [iv, nv] = block_index(tplan.dims[0], d);
          const auto [ih, nh] = block_index(tplan.dims[1], d);
          const int64_t rows = vocab / nv, cols = width / nh;
          void* blk = grad_zeros(static_cast<size_t>(rows * cols) * 4, stream);
          apl_detail::check(apl_embedding_backward_block(
              sid.data(), sdy.data(), static_cast<int>(sid.size()), n, ls.back(),
              static_cast<float*>(blk), iv * rows, rows, ih * cols, cols, APL_BF16, stream));
          blks.push_back(blk);
        }
        out.push_back({1, Grad{blks, 4}, tplan});
      } else if (wants(tab)) {
        const auto ts = local_shape(tspec, tm);
        std::vector<void*> dt;
        for (int d = 0; d < num_local_; ++d) {
          void* t = grad_zeros(static_cast<size_t>(numel(ts)) * 4, stream);
          apl_detail::check(apl_embedding_backward(static_cast<const int64_t*>(ids[d]), n,
                                                   dy.p[d], static_cast<float*>(t), ts[0], ts[1],
                                                   APL_BF16, stream));
          dt.push_back(t);
        }
        std::set<int> axes_set;
        for (const auto& dim : required_spec(nd, 0).dims)
          for (int a : dim.axes) axes_set.insert(a);
        std::vector<int32_t> axes(axes_set.begin(), axes_set.end());
        if (!axes.empty())
          apl_detail::check(apl_all_reduce(rt_.get(), axes.data(), static_cast<int>(axes.size()),
                                           dt.data(), static_cast<size_t>(numel(ts)), APL_F32,
                                           stream));
        out.push_back({1, Grad{as_const(dt), 4}, tspec});
      }
    } else if (nd.kind == "batched-matmul") {
      const OpStrategy& st = nd.strategy;
      if (st.partial_sum) throw PlanError("backward of split-k batched matmul strategies");
      const auto& sv = saved_.at(nd.id);
      const auto as = local_shape(required_spec(nd, 0), nodes_.at(nd.inputs[0]).meta);
      const auto bs = local_shape(required_spec(nd, 1), nodes_.at(nd.inputs[1]).meta);
      const int64_t nb = as[0], m = as[1], k = as[2], nn = bs[2];
      auto bmm = [&](const void* a, const void* b, void* o, int64_t M, int64_t N, int64_t K,
                     int64_t lda, int64_t ldb, int a_layout, int b_layout, int64_t a_step,
                     int64_t b_step) {
        std::vector<const void*> A, B;
        std::vector<void*> Cp;
        for (int64_t i = 0; i < nb; ++i) {
          A.push_back(static_cast<const char*>(a) + i * a_step * 2);
          B.push_back(static_cast<const char*>(b) + i * b_step * 2);
          Cp.push_back(static_cast<char*>(o) + i * M * N * 2);
        }
        apl_detail::check(apl_gemm_bf16_grouped_ex(A.data(), B.data(), Cp.data(),
                                                   static_cast<int>(nb), M, N, K, lda, ldb, N,
                                                   a_layout, b_layout, APL_BF16, stream));
      };
      if (wants(nd.inputs[0])) {  // dA = dC . B^T
        std::vector<void*> da;
        for (int d = 0; d < num_local_; ++d) {
          void* o = grad_buf(static_cast<size_t>(nb * m * k) * 2);
          bmm(dy.p[d], sv[1][d], o, m, k, nn, nn, nn, APL_A_MK, APL_B_NK, m * nn, k * nn);
          da.push_back(o);
        }
        if (!st.output_spec.dims[2].axes.empty()) {
          std::vector<int32_t> axes(st.output_spec.dims[2].axes.begin(),
                                    st.output_spec.dims[2].axes.end());
          apl_detail::check(apl_all_reduce(rt_.get(), axes.data(), static_cast<int>(axes.size()),
                                           da.data(), static_cast<size_t>(nb * m * k), APL_BF16,
                                           stream));
        }
        out.push_back({0, Grad{as_const(da), 2}, required_spec(nd, 0)});
      }
      if (wants(nd.inputs[1])) {  // dB = A^T . dC
        std::vector<void*> db;
        for (int d = 0; d < num_local_; ++d) {
          void* o = grad_buf(static_cast<size_t>(nb * k * nn) * 2);
          bmm(sv[0][d], dy.p[d], o, k, nn, m, k, nn, APL_A_KM, APL_B_KN, m * k, m * nn);
          db.push_back(o);
        }
        if (!st.output_spec.dims[1].axes.empty()) {
          std::vector<int32_t> axes(st.output_spec.dims[1].axes.begin(),
                                    st.output_spec.dims[1].axes.end());
          apl_detail::check(apl_all_reduce(rt_.get(), axes.data(), static_cast<int>(axes.size()),
                                           db.data(), static_cast<size_t>(nb * k * nn), APL_BF16,
                                           stream));
        }
        out.push_back({1, Grad{as_const(db), 2}, required_spec(nd, 1)});
      }
    } else {
      throw PlanError("backward through " + nd.kind + " (" + nd.id + ")");
    }
    return out;
  }

  static constexpr float kMaskFill = -1e4f;  // additive attention mask
  enum class Unary { kGelu, kScale, kNot };

  struct Node {
    std::string id, kind;
    std::vector<std::string> inputs;
    TensorMeta meta;
    ShardingSpec spec;
    OpStrategy strategy;
    std::vector<ShardingSpec> in_specs;
    std::vector<int64_t> perm;
    int64_t axis = -1;
    Unary unary = Unary::kGelu;
    float alpha = 1.f;
  };

  struct Chain {
    std::string x, mask;
    float alpha;
  };

  static int64_t numel(const std::vector<int64_t>& s) {
    int64_t n = 1;
    for (int64_t e : s) n *= e;
    return n;
  }
  static int dtype_of(const TensorMeta& m) { return m.dtype_bytes == 4 ? APL_F32 : APL_BF16; }

  std::vector<int64_t> local_shape(const ShardingSpec& spec, const TensorMeta& m) const {
    std::vector<int64_t> out = m.shape;
    for (size_t k = 0; k < out.size(); ++k)
      for (int a : spec.dims[k].axes) out[k] /= mesh_.shape[static_cast<size_t>(a)];
    return out;
  }

  // row-major device -> coordinate (cluster.hpp:56); a free computation, so
  // this header also compiles against the reference's own DeviceMesh
  std::vector<int64_t> mesh_coord(int64_t device) const {
    std::vector<int64_t> c(mesh_.shape.size());
    for (size_t k = c.size(); k-- > 0;) {
      c[k] = device % mesh_.shape[k];
      device /= mesh_.shape[k];
    }
    return c;
  }

  // (index, count) of `device`'s block along a dim sharded over dim.axes
  std::pair<int64_t, int64_t> block_index(const DimSpec& dim, int64_t device) const {
    const auto c = mesh_coord(device);
    int64_t idx = 0, cnt = 1;
    for (int a : dim.axes) {
      idx = idx * mesh_.shape[static_cast<size_t>(a)] + c[static_cast<size_t>(a)];
      cnt *= mesh_.shape[static_cast<size_t>(a)];
    }
    return {idx, cnt};
  }

  // a device holding block (i, j) of a rank-2 spec (mixed radix, first axis
  // most significant)
  int64_t block_owner(const ShardingSpec& spec, int64_t i, int64_t j) const {
    std::vector<int64_t> coord(static_cast<size_t>(mesh_.rank()), 0);
    const int64_t idx[2] = {i, j};
    for (int k = 0; k < 2; ++k) {
      int64_t v = idx[k];
      const auto& axes = spec.dims[static_cast<size_t>(k)].axes;
      for (auto a = axes.rbegin(); a != axes.rend(); ++a) {
        coord[static_cast<size_t>(*a)] = v % mesh_.shape[static_cast<size_t>(*a)];
        v /= mesh_.shape[static_cast<size_t>(*a)];
      }
    }
    int64_t d = 0;  // row-major coordinate -> device (cluster.hpp:56)
    for (size_t k = 0; k < coord.size(); ++k) d = d * mesh_.shape[k] + coord[k];
    return d;
  }

  // input layouts of a non-matmul node's named strategy (intraop.cpp:280-450)
  std::vector<ShardingSpec> input_specs(const Node& nd, const std::string& name) const {
    const int mr = mesh_.rank();
    if (nd.kind == "output")
      return {ShardingSpec::replicated(static_cast<int>(nd.meta.shape.size()), mr)};
    if (nd.kind == "reshape" || nd.kind == "transpose" || nd.kind == "softmax" ||
        nd.kind == "layernorm") {
      const ShardingSpec in = ShardingSpec::parse(name.substr(name.find(':') + 1), mr);
      std::vector<ShardingSpec> out = {in};
      if (nd.kind == "layernorm")
        for (size_t i = 1; i < nd.inputs.size(); ++i)
          out.push_back(ShardingSpec::replicated(1, mr));
      return out;
    }
    if (nd.kind == "embedding-lookup") {
      const size_t ri = nodes_.at(nd.inputs.at(0)).meta.shape.size();
      ShardingSpec ids = ShardingSpec::replicated(static_cast<int>(ri), mr);
      for (size_t k = 0; k < ri; ++k) ids.dims[k] = nd.spec.dims[k];
      ShardingSpec table = ShardingSpec::replicated(2, mr);
      table.dims[1] = nd.spec.dims[ri];
      return {ids, table};
    }
    return std::vector<ShardingSpec>(nd.inputs.size(), nd.spec);  // elementwise
  }

  static size_t axis_of(const std::vector<int64_t>& shape, int64_t axis) {
    const int64_t r = static_cast<int64_t>(shape.size());
    return static_cast<size_t>(axis < 0 ? axis + r : axis);
  }
  // product of the extents before the softmax axis
  static int64_t axis_outer(const std::vector<int64_t>& shape, int64_t axis) {
    int64_t o = 1;
    for (size_t k = 0; k < axis_of(shape, axis); ++k) o *= shape[k];
    return o;
  }
  // any transpose of a local shard (graph_ir.cpp:270-290); the last-two swap
  // takes the tiled 2-D transpose kernel
  static void permute(const void* x, void* y, const std::vector<int64_t>& in_shape,
                      const std::vector<int64_t>& perm, int elem_bytes, void* stream) {
    const size_t r = perm.size();
    bool last2 = r >= 2 && perm[r - 2] == static_cast<int64_t>(r - 1) &&
                 perm[r - 1] == static_cast<int64_t>(r - 2);
    for (size_t i = 0; last2 && i + 2 < r; ++i) last2 = perm[i] == static_cast<int64_t>(i);
    if (last2) {
      const int64_t rows = in_shape[r - 2], cols = in_shape[r - 1];
      const int64_t batch = numel(in_shape) / std::max<int64_t>(1, rows * cols);
      apl_detail::check(apl_transpose(x, y, batch, rows, cols, elem_bytes, stream));
      return;
    }
    apl_detail::check(apl_permute(x, y, static_cast<int>(r), in_shape.data(), perm.data(),
                                  elem_bytes, stream));
  }

  void bind_unary(Node& nd) const {
    const Node& src = nodes_.at(nd.inputs.at(0));
    if (src.meta.dtype_bytes == 1) {
      nd.unary = Unary::kNot;
    } else if (nd.id.find("scale") != std::string::npos && src.kind == "batched-matmul") {
      nd.unary = Unary::kScale;
      const double k = static_cast<double>(nodes_.at(src.inputs.at(0)).meta.shape.back());
      nd.alpha = static_cast<float>(1.0 / std::sqrt(k));
    } else if (src.kind == "matmul" || nd.id.find("gelu") != std::string::npos) {
      nd.unary = Unary::kGelu;  // the MLP activation (fc1 -> act)
    } else {
      // the graph does not name the function: refuse to guess (the Python
      // executor takes an explicit unary= binding for such graphs)
      throw SchemaError(nd.id + ": elementwise-unary consuming a " + src.kind +
                        " node has no known function binding");
    }
  }

  // scale -> u8 additive mask -> last-axis softmax, no conversion on the way
  void find_attention_chains() {
    auto single = [&](const std::string& id) {
      auto it = consumers_.find(id);
      return it != consumers_.end() && it->second.size() == 1;
    };
    for (const auto& [id, sm] : nodes_) {
      if (sm.kind != "softmax" ||
          (sm.axis != -1 && sm.axis != static_cast<int64_t>(sm.meta.shape.size()) - 1))
        continue;
      const Node& b = nodes_.at(sm.inputs.at(0));
      if (b.kind != "elementwise-binary" || !single(b.id) || !(b.spec == sm.in_specs.at(0)))
        continue;
      int mslot = -1, nmask = 0;
      for (int k = 0; k < 2; ++k)
        if (nodes_.at(b.inputs[static_cast<size_t>(k)]).meta.dtype_bytes == 1) {
          mslot = k;
          ++nmask;
        }
      if (nmask != 1) continue;
      const Node& u = nodes_.at(b.inputs[static_cast<size_t>(1 - mslot)]);
      const Node& m = nodes_.at(b.inputs[static_cast<size_t>(mslot)]);
      if (u.kind != "elementwise-unary" || !single(u.id) || u.unary != Unary::kScale) continue;
      const Node& x = nodes_.at(u.inputs.at(0));
      if (!(u.spec == b.in_specs[static_cast<size_t>(1 - mslot)]) ||
          !(m.spec == b.in_specs[static_cast<size_t>(mslot)]) || !(x.spec == u.in_specs.at(0)))
        continue;
      attn_[id] = Chain{x.id, m.id, u.alpha};
      attn_members_.insert(u.id);
      attn_members_.insert(b.id);
    }
  }

  ShardingSpec required_spec(const Node& nd, size_t slot) const { return nd.in_specs.at(slot); }

  std::string fusable_gelu(const Node& mm) const {
    auto it = consumers_.find(mm.id);
    if (it == consumers_.end() || it->second.size() != 1 || mm.strategy.partial_sum ||
        mm.kind != "matmul")
      return "";
    const Node& g = nodes_.at(it->second[0]);
    return g.kind == "elementwise-unary" && g.unary == Unary::kGelu && g.spec == mm.spec ? g.id
                                                                                        : "";
  }

  // an embedding whose sharded table is read from its owners' blocks
  // (simulated mesh; the Python executor's auto rule)
  bool gatherable_table(const Node& nd) const {
    int n = 0, first = 0, nl = 0, dist = 0;
    apl_detail::check(apl_mesh_info(rt_.get(), &n, &first, &nl, &dist));
    if (dist) return false;
    const ShardingSpec& have = nodes_.at(nd.inputs.at(1)).spec;
    if (have == required_spec(nd, 1)) return false;
    int64_t nb = 1;
    for (const auto& d : have.dims)
      for (int a : d.axes) nb *= mesh_.shape[static_cast<size_t>(a)];
    return nb <= 64;
  }

  std::vector<const void*> lookup_gathered_table(const Node& nd,
                                                 const std::vector<const void*>& ids,
                                                 const std::vector<const void*>& table,
                                                 void* stream) {
    const Node& t = nodes_.at(nd.inputs.at(1));
    const ShardingSpec& have = t.spec;
    const ShardingSpec want = required_spec(nd, 1);
    const int64_t vocab = t.meta.shape.at(0), width = t.meta.shape.at(1);
    const int64_t nvb = block_index(have.dims[0], 0).second;
    const int64_t nhb = block_index(have.dims[1], 0).second;
    std::vector<const void*> blocks;
    for (int64_t i = 0; i < nvb; ++i)
      for (int64_t j = 0; j < nhb; ++j) blocks.push_back(table.at(static_cast<size_t>(
          block_owner(have, i, j))));
    auto out = buffers(nd.id, nd.spec, nd.meta);
    const auto ls = local_shape(nd.spec, nd.meta);
    const int64_t n = numel(ls) / ls.back();
    for (int d = 0; d < num_local_; ++d) {
      const auto [j, nw] = block_index(want.dims[1], d);
      apl_detail::check(apl_embedding_lookup_blocks(
          static_cast<const int64_t*>(ids[d]), n, blocks.data(), static_cast<int>(nvb),
          static_cast<int>(nhb), vocab, width, j * (width / nw), ls.back(), t.meta.dtype_bytes,
          out[d], stream));
    }
    return as_const(out);
  }

  std::vector<const void*> block_node(const Node& nd,
                                      const std::vector<std::vector<const void*>>& ins,
                                      void* stream) {
    auto out = buffers(nd.id, nd.spec, nd.meta);
    const auto ls = local_shape(nd.spec, nd.meta);
    const int dt = dtype_of(nd.meta);
    if (nd.kind == "embedding-lookup") {
      const Node& t = nodes_.at(nd.inputs[1]);
      const auto ts = local_shape(required_spec(nd, 1), t.meta);
      const int64_t n = numel(ls) / ls.back();
      for (int d = 0; d < num_local_; ++d)
        apl_detail::check(apl_embedding_lookup(static_cast<const int64_t*>(ins[0][d]), n,
                                               ins[1][d], ts[0], ts[1], t.meta.dtype_bytes,
                                               out[d], stream));
    } else if (nd.kind == "layernorm") {
      const int64_t w = ls.back(), rows = numel(ls) / w;
      for (int d = 0; d < num_local_; ++d)
        apl_detail::check(apl_layernorm(ins[0][d], ins.size() > 1 ? ins[1][d] : nullptr,
                                        ins.size() > 2 ? ins[2][d] : nullptr, out[d], rows, w,
                                        1e-5f, dt, stream));
    } else if (nd.kind == "softmax") {
      // the softmax axis is replicated under every strategy (intraop.cpp:368-384)
      const int64_t o = axis_outer(ls, nd.axis), n = ls[axis_of(ls, nd.axis)],
                    i = numel(ls) / (o * n);
      for (int d = 0; d < num_local_; ++d)
        apl_detail::check(apl_softmax_axis(ins[0][d], out[d], o, n, i, dt, stream));
    } else if (nd.kind == "transpose") {
      const auto is = local_shape(required_spec(nd, 0), nodes_.at(nd.inputs[0]).meta);
      for (int d = 0; d < num_local_; ++d)
        permute(ins[0][d], out[d], is, nd.perm, nd.meta.dtype_bytes, stream);
    } else if (nd.kind == "elementwise-binary") {
      int a = 0, b = 1;
      if (nodes_.at(nd.inputs[0]).meta.dtype_bytes == 1) std::swap(a, b);
      const bool mask = nodes_.at(nd.inputs[static_cast<size_t>(b)]).meta.dtype_bytes == 1;
      const size_t count = static_cast<size_t>(numel(ls));
      for (int d = 0; d < num_local_; ++d)
        apl_detail::check(apl_add(ins[static_cast<size_t>(a)][d], ins[static_cast<size_t>(b)][d],
                                  mask ? 1 : 0, out[d], count, mask ? kMaskFill : 1.f, dt,
                                  stream));
    } else if (nd.kind == "batched-matmul") {
      const auto as = local_shape(required_spec(nd, 0), nodes_.at(nd.inputs[0]).meta);
      const int64_t nb = as[0], m = as[1], k = as[2], n = ls[2];
      const int64_t ea = nodes_.at(nd.inputs[0]).meta.dtype_bytes, eo = nd.meta.dtype_bytes;
      for (int d = 0; d < num_local_; ++d) {
        std::vector<const void*> A, B;
        std::vector<void*> Cp;
        for (int64_t i = 0; i < nb; ++i) {
          A.push_back(static_cast<const char*>(ins[0][d]) + i * m * k * ea);
          B.push_back(static_cast<const char*>(ins[1][d]) + i * k * n * ea);
          Cp.push_back(static_cast<char*>(out[d]) + i * m * n * eo);
        }
        apl_detail::check(apl_gemm_bf16_grouped_ex(A.data(), B.data(), Cp.data(),
                                                   static_cast<int>(nb), m, n, k, k, n, n,
                                                   APL_A_MK, APL_B_KN, dt, stream));
      }
      if (nd.strategy.partial_sum) {
        std::vector<int32_t> axes(nd.strategy.reduce_axes.begin(), nd.strategy.reduce_axes.end());
        apl_detail::check(apl_all_reduce(rt_.get(), axes.data(), static_cast<int>(axes.size()),
                                         out.data(), static_cast<size_t>(numel(ls)), dt,
                                         stream));
      }
    } else {
      throw SchemaError("node kind '" + nd.kind + "' is not executable");
    }
    return as_const(out);
  }

  // The reference path and its workspace size per (value, have -> want,
  // element size), searched once: later steps (and every backward pass)
  // convert without touching the host planner.
  struct CachedPath {
    TransformPath path;
    size_t ws;
  };
  const CachedPath& cached_path(const std::string& id, const ShardingSpec& have,
                                const ShardingSpec& want, const TensorMeta& m) {
    const std::string key = id + "|" + have.to_string() + ">" + want.to_string() + "|" +
                            std::to_string(m.dtype_bytes);
    auto it = paths_.find(key);
    if (it == paths_.end()) {
      TransformPath p = find_transform_path(have, want, mesh_, m);
      const size_t ws = workspace_bytes(rt_, p, m, fuse_);
      it = paths_.emplace(key, CachedPath{std::move(p), ws}).first;
    }
    return it->second;
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
    const CachedPath& cp = cached_path(src, have, want, m);
    const TransformPath& path = cp.path;
    auto out = buffers(src + ">" + want.to_string(), want, m);
    const std::string wkey = src + ">" + want.to_string();
    auto w = workspaces_.find(wkey);
    if (w == workspaces_.end()) {
      const size_t bytes = cp.ws;
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
  std::map<std::string, Chain> attn_;
  std::set<std::string> attn_members_;
  std::map<std::string, std::vector<std::vector<const void*>>> saved_;
  bool trained_ = false;
  int gcount_ = 0;
  std::map<std::string, std::vector<void*>> buffers_;
  std::map<std::string, std::pair<void*, size_t>> workspaces_;
  std::map<std::string, CachedPath> paths_;
};

}  // namespace autoplan
