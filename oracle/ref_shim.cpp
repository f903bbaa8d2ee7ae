// ref_shim.cpp — C entry points over the REFERENCE autoplan library
// (test infrastructure only; see oracle/Makefile).
//
// Linked against the reference's own translation units compiled straight
// from /root/reference/proj/src (never copied into this repo) into
// oracle/_ref/libautoplan_ref.so. Used by tests/ to check the drop-in host
// API step-for-step against the real reference, by tests/golden/make_golden.py
// to write the committed golden paths, and by bench.py --impl reference to
// time the reference planner on the GPU box's host.
//
// Calls wrapped (reference file:line):
//   ShardingSpec::parse / to_string / valid_for  src/layout.cpp:79-160
//   one_step_transforms                          src/layout.cpp:162-221
//   dim_diff / heuristic_diff                    src/layout.cpp:223-251
//   find_transform_path / conversion_cost        src/layout.cpp:253-329
//   PathCache::get                               src/layout.cpp:331-346
//   collective_cost                              src/cluster.cpp:374-400
//   mesh_to_json / mesh_from_json                src/cluster.cpp:417-450
//   testutil::all_valid_specs / bfs_min_steps /
//   replay_path_error                            tests/helpers.hpp:245-363
//   matmul strategy catalog (generate_strategies) src/intraop.cpp:141-234,497-555,719-767
#include <chrono>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "autoplan/cluster.hpp"
#include "autoplan/errors.hpp"
#include "autoplan/graph_ir.hpp"
#include "autoplan/intraop.hpp"
#include "autoplan/layout.hpp"
#include "helpers.hpp"

using namespace autoplan;

namespace {

int code_of(const std::exception& e) {
  if (dynamic_cast<const SchemaError*>(&e)) return 1;
  if (dynamic_cast<const AxisError*>(&e)) return 2;
  if (dynamic_cast<const ShapeError*>(&e)) return 3;
  if (dynamic_cast<const RankMismatchError*>(&e)) return 4;
  if (dynamic_cast<const InfeasibleError*>(&e)) return 5;
  if (dynamic_cast<const PlanError*>(&e)) return 9;
  return 10;
}

int put(const std::string& s, char* out, size_t cap) {
  if (s.size() + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

DeviceMesh mesh_of(const int64_t* m, int mr) {
  return DeviceMesh::uniform(std::vector<int64_t>(m, m + mr), 1e-5, 1e-9, 1e12);
}

TensorMeta meta_of(const int64_t* shape, int rank, int dtype_bytes) {
  TensorMeta t;
  t.shape.assign(shape, shape + rank);
  t.dtype_bytes = dtype_bytes;
  return t;
}

std::string render_path(const TransformPath& p) {
  std::ostringstream os;
  for (const TransformStep& s : p.steps)
    os << static_cast<int>(s.kind) << " " << s.tensor_dim << " " << s.target_dim << " "
       << s.mesh_axis << " " << s.result.to_string() << "\n";
  char buf[64];
  std::snprintf(buf, sizeof(buf), "cost %.17g\n", p.comm_cost_s);
  os << buf;
  return os.str();
}

}  // namespace

extern "C" {

// Path as text: one "kind tensor_dim target_dim mesh_axis result" line per
// step, then "cost <%.17g>". Returns 0, a PlanError class code, or -1
// (buffer too small).
int ref_find_path(const int64_t* mesh, int mr, const int64_t* shape, int rank, int eb,
                  const char* src, const char* tgt, char* out, size_t cap) {
  try {
    DeviceMesh m = mesh_of(mesh, mr);
    TensorMeta t = meta_of(shape, rank, eb);
    TransformPath p = find_transform_path(ShardingSpec::parse(src, mr), ShardingSpec::parse(tgt, mr), m, t);
    conversion_cost(p, m, t);
    return put(render_path(p), out, cap);
  } catch (const std::exception& e) {
    put(e.what(), out, cap);
    return code_of(e);
  }
}

int ref_one_step(const int64_t* mesh, int mr, const int64_t* shape, int rank, int eb,
                 const char* spec, char* out, size_t cap) {
  try {
    auto r = one_step_transforms(ShardingSpec::parse(spec, mr), mesh_of(mesh, mr), meta_of(shape, rank, eb));
    std::ostringstream os;
    for (auto& [next, s] : r)
      os << static_cast<int>(s.kind) << " " << s.tensor_dim << " " << s.target_dim << " "
         << s.mesh_axis << " " << next.to_string() << "\n";
    return put(os.str(), out, cap);
  } catch (const std::exception& e) {
    put(e.what(), out, cap);
    return code_of(e);
  }
}

int ref_all_valid_specs(const int64_t* mesh, int mr, const int64_t* shape, int rank, int eb,
                        char* out, size_t cap) {
  try {
    std::ostringstream os;
    for (const ShardingSpec& s : testutil::all_valid_specs(meta_of(shape, rank, eb), mesh_of(mesh, mr)))
      os << s.to_string() << "\n";
    return put(os.str(), out, cap);
  } catch (const std::exception& e) {
    put(e.what(), out, cap);
    return code_of(e);
  }
}

int ref_bfs_min_steps(const int64_t* mesh, int mr, const int64_t* shape, int rank, int eb,
                      const char* src, const char* tgt) {
  try {
    return testutil::bfs_min_steps(ShardingSpec::parse(src, mr), ShardingSpec::parse(tgt, mr),
                                   mesh_of(mesh, mr), meta_of(shape, rank, eb));
  } catch (const std::exception&) {
    return -2;
  }
}

int ref_dim_diff(const int* a, int na, const int* b, int nb, double* out) {
  DimSpec x, y;
  x.axes.assign(a, a + na);
  y.axes.assign(b, b + nb);
  *out = dim_diff(x, y);
  return 0;
}

int ref_heuristic_diff(int mr, const char* a, const char* b, double* out) {
  try {
    *out = heuristic_diff(ShardingSpec::parse(a, mr), ShardingSpec::parse(b, mr));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_collective_cost(const int64_t* mesh, int mr, const int* axes, int naxes, int kind,
                        double bytes, double* out) {
  try {
    *out = collective_cost(mesh_of(mesh, mr), std::vector<int>(axes, axes + naxes),
                           static_cast<CollectiveKind>(kind), bytes);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_spec_valid(const int64_t* mesh, int mr, const int64_t* shape, int rank, int eb,
                   const char* spec) {
  try {
    return ShardingSpec::parse(spec, mr).valid_for(meta_of(shape, rank, eb), mesh_of(mesh, mr)) ? 1 : 0;
  } catch (const std::exception& e) {
    return -code_of(e);
  }
}

// Reference mesh_from_json -> mesh_to_json round trip of a document
// (cluster.cpp:417-450): 0 and the canonical dump, or the error class code
// and message.
int ref_mesh_json(const char* text, char* out, size_t cap) {
  try {
    const DeviceMesh m = mesh_from_json(nlohmann::json::parse(text));
    return put(mesh_to_json(m).dump(), out, cap);
  } catch (const nlohmann::json::exception& e) {
    put(e.what(), out, cap);
    return 11;
  } catch (const std::exception& e) {
    put(e.what(), out, cap);
    return code_of(e);
  }
}

// Mean seconds per uncached find_transform_path + conversion_cost call
// (`hits` = 0) or per cached PathCache::get (`hits` = 1), over `iters` calls.
double ref_time_paths(const int64_t* mesh, int mr, const int64_t* shape, int rank, int eb,
                      const char* src, const char* tgt, int iters, int hits) {
  DeviceMesh m = mesh_of(mesh, mr);
  TensorMeta t = meta_of(shape, rank, eb);
  ShardingSpec a = ShardingSpec::parse(src, mr), b = ShardingSpec::parse(tgt, mr);
  PathCache cache;
  cache.get(a, b, m, t);
  volatile double sink = 0;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) {
    if (hits) {
      sink = sink + cache.get(a, b, m, t).comm_cost_s;
    } else {
      TransformPath p = find_transform_path(a, b, m, t);
      sink = sink + conversion_cost(p, m, t);
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count() / iters;
}

}  // extern "C"

// ---- strategy catalog and planner (config 5) -------------------------------
#include "autoplan/planner.hpp"

extern "C" {

// generate_strategies for one node of a graph document (intraop.cpp:719-767):
// one line per strategy "name|in0|in1|out|partial|reduce axes|compute|comm|mem".
int ref_node_strategies(const char* graph_json, const char* node_id, const int64_t* mesh,
                        int mr, double flops, char* out, size_t cap) {
  try {
    ComputationGraph g = parse_graph_text(graph_json);
    infer_meta(g);
    DeviceMesh m = DeviceMesh::uniform(std::vector<int64_t>(mesh, mesh + mr), 1e-5, 1e-9, flops);
    std::ostringstream os;
    char buf[128];
    for (const OpStrategy& s : generate_strategies(g, g.node(node_id), m)) {
      os << s.name << "|";
      for (const ShardingSpec& in : s.input_specs) os << in.to_string() << "|";
      os << s.output_spec.to_string() << "|" << (s.partial_sum ? 1 : 0) << "|";
      for (size_t i = 0; i < s.reduce_axes.size(); ++i) os << (i ? "," : "") << s.reduce_axes[i];
      std::snprintf(buf, sizeof(buf), "|%.17g|%.17g|%lld\n", s.compute_time_s, s.comm_time_s,
                    static_cast<long long>(s.memory_bytes));
      os << buf;
    }
    return put(os.str(), out, cap);
  } catch (const std::exception& e) {
    put(e.what(), out, cap);
    return code_of(e);
  }
}

// Full planner run (sweep, planner.cpp:91-212) on a uniform mesh; writes the
// version-1 plan document (plan_to_json, planner.cpp:455-600).
int ref_plan(const char* graph_json, const int64_t* mesh, int mr, double alpha, double beta_inv,
             double flops, int64_t device_budget_bytes, char* out, size_t cap) {
  try {
    ComputationGraph g = parse_graph_text(graph_json);
    infer_meta(g);
    DeviceMesh m = DeviceMesh::uniform(std::vector<int64_t>(mesh, mesh + mr), alpha, beta_inv, flops);
    ExecutionPlan plan = sweep(g, m, device_budget_bytes);
    return put(plan_to_json(plan).dump(1), out, cap);
  } catch (const std::exception& e) {
    put(e.what(), out, cap);
    return code_of(e);
  }
}

}  // extern "C"
