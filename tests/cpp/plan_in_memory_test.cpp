// The reference planner running on the drop-in, its in-memory plan executed
// by the native PlanExecutor:
//
//   * the reference's OWN graph_ir / intraop / ckpt / planner translation
//     units (compiled from /root/reference by oracle/Makefile) are linked
//     against libapl.so INSTEAD of the reference's layout.cpp / cluster.cpp
//     -- the drop-in supplies ShardingSpec, find_transform_path, PathCache,
//     DeviceMesh, collective_cost ... to the reference's solvers;
//   * sweep() (planner.cpp:91-212) produces the ExecutionPlan in memory and
//     plan_to_json of it must equal the golden plan the all-reference build
//     wrote (tests/golden/plans/, make_plans.py);
//   * with a directory argument, PlanExecutor(rt, graph, plan) -- the
//     reference's ComputationGraph and ExecutionPlan objects, no JSON --
//     runs the forward pass on a simulated mesh and writes device 0's
//     output replica to <dir>/out.bin (operands <dir>/<id>.bin as in
//     plan_executor_test.cpp).
//
//   plan_in_memory_test <graph.json> <AxB> <budget_bytes> <golden_plan.json> [dir]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "autoplan/planner.hpp"        // the reference's planner (its headers first on -I)
#include "autoplan/plan_executor.hpp"  // ours

using namespace autoplan;

static std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

int main(int argc, char** argv) {
  if (argc != 5 && argc != 6) {
    std::fprintf(stderr, "usage: plan_in_memory_test graph.json AxB budget golden.json [dir]\n");
    return 2;
  }
  ComputationGraph g = parse_graph_text(slurp(argv[1]));
  infer_meta(g);
  const DeviceMesh mesh =
      DeviceMesh::uniform(parse_mesh_shape(argv[2]), 3e-6, 1.0 / 900e9, 1.65e15);
  const int64_t budget = std::stoll(argv[3]);
  const ExecutionPlan plan = sweep(g, mesh, budget);
  const nlohmann::json mine = plan_to_json(plan);
  const nlohmann::json golden = nlohmann::json::parse(slurp(argv[4]));
  if (mine != golden) {
    std::cerr << "plan differs from the golden (all-reference) plan\n";
    std::cerr << nlohmann::json::diff(golden, mine).dump(1).substr(0, 2000) << "\n";
    return 1;
  }
  std::cout << "plan == golden: " << plan.node_plans.size() << " node plans, "
            << plan.inserted_comm_nodes.size() << " comm insertions\n";
  if (argc == 5) return 0;

  const std::string dir = argv[5];
  MeshRuntime rt = MeshRuntime::Simulated(plan.mesh, 0);
  PlanExecutor ex(rt, g, plan);  // the in-memory objects, no JSON in between
  std::map<std::string, std::vector<const void*>> feeds;
  std::vector<void*> owned;
  for (const std::string& id : ex.sources()) {
    const TensorMeta& m = ex.meta(id);
    const ShardingSpec& s = ex.spec(id);
    const std::string data = slurp(dir + "/" + id + ".bin");
    const size_t rank = m.shape.size();
    const int64_t eb = m.dtype_bytes;
    std::vector<const void*> shards;
    for (int64_t d = 0; d < plan.mesh.num_devices(); ++d) {
      std::vector<int64_t> c(plan.mesh.shape.size());  // row-major coordinate
      for (int64_t k = static_cast<int64_t>(c.size()) - 1, v = d; k >= 0; --k) {
        c[static_cast<size_t>(k)] = v % plan.mesh.shape[static_cast<size_t>(k)];
        v /= plan.mesh.shape[static_cast<size_t>(k)];
      }
      std::vector<int64_t> blk(rank, 0), loc(rank);
      int64_t total = 1;
      for (size_t k = 0; k < rank; ++k) {
        int64_t cnt = 1;
        for (int a : s.dims[k].axes) {
          blk[k] = blk[k] * plan.mesh.shape[a] + c[a];
          cnt *= plan.mesh.shape[a];
        }
        loc[k] = m.shape[k] / cnt;
        total *= loc[k];
      }
      std::vector<char> host(static_cast<size_t>(total * eb));
      const int64_t run = loc[rank - 1];
      std::vector<int64_t> idx(rank, 0);
      for (int64_t r = 0; r < total / run; ++r) {
        int64_t off = 0;
        for (size_t k = 0; k < rank; ++k)
          off = off * m.shape[k] + blk[k] * loc[k] + (k + 1 < rank ? idx[k] : 0);
        std::memcpy(host.data() + r * run * eb, data.data() + off * eb,
                    static_cast<size_t>(run * eb));
        for (size_t k = rank - 1; k-- > 0;) {
          if (++idx[k] < loc[k]) break;
          idx[k] = 0;
        }
      }
      void* dptr = nullptr;
      cudaMalloc(&dptr, host.size() < 256 ? 256 : host.size());
      cudaMemcpy(dptr, host.data(), host.size(), cudaMemcpyHostToDevice);
      owned.push_back(dptr);
      shards.push_back(dptr);
    }
    feeds[id] = shards;
  }
  cudaStream_t stream;
  cudaStreamCreate(&stream);
  std::vector<void*> out = ex.forward(feeds, stream, false);
  cudaStreamSynchronize(stream);
  const TensorMeta& om = ex.meta(g.output);
  size_t bytes = static_cast<size_t>(om.dtype_bytes);
  for (int64_t e : om.shape) bytes *= static_cast<size_t>(e);
  std::vector<char> host(bytes);
  if (cudaMemcpy(host.data(), out.at(0), bytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
    std::fprintf(stderr, "copy-back failed\n");
    return 1;
  }
  std::ofstream(dir + "/out.bin", std::ios::binary).write(host.data(), static_cast<long>(bytes));
  for (void* p : owned) cudaFree(p);
  std::cout << "in-memory plan executed on " << plan.mesh.num_devices() << " simulated devices\n";
  return 0;
}
