// Runs a reference plan with the native C++ PlanExecutor on a simulated mesh:
//   plan_executor_test <graph.json> <plan.json> <mesh AxB> <dir>
// reads <dir>/<id>.bin (global row-major bf16 tensors of every placeholder
// and parameter), shards them on the host by each node's plan spec, runs the
// forward pass and writes device 0's output replica to <dir>/out.bin.
#include <cuda_runtime.h>

#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "autoplan/plan_executor.hpp"

using namespace autoplan;

static std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

int main(int argc, char** argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: plan_executor_test graph.json plan.json AxB dir\n");
    return 2;
  }
  const std::string dir = argv[4];
  const DeviceMesh mesh = DeviceMesh::uniform(parse_mesh_shape(argv[3]));
  MeshRuntime rt = MeshRuntime::Simulated(mesh, 0);
  PlanExecutor ex(rt, mesh, slurp(argv[1]), slurp(argv[2]));
  std::map<std::string, std::vector<const void*>> feeds;
  std::vector<void*> owned;
  for (const std::string id : {"x", "w1", "w2"}) {
    const TensorMeta& m = ex.meta(id);
    const ShardingSpec& s = ex.spec(id);
    const std::string data = slurp(dir + "/" + id + ".bin");
    const int64_t rows = m.shape[0], cols = m.shape[1], eb = m.dtype_bytes;
    std::vector<const void*> shards;
    for (int64_t d = 0; d < mesh.num_devices(); ++d) {
      const auto c = mesh.coord_of(d);
      int64_t blk[2], cnt[2];
      for (int k = 0; k < 2; ++k) {
        blk[k] = 0;
        cnt[k] = 1;
        for (int a : s.dims[k].axes) {
          blk[k] = blk[k] * mesh.shape[a] + c[a];
          cnt[k] *= mesh.shape[a];
        }
      }
      const int64_t lr = rows / cnt[0], lc = cols / cnt[1];
      std::vector<char> host(static_cast<size_t>(lr * lc * eb));
      for (int64_t r = 0; r < lr; ++r)
        std::memcpy(host.data() + r * lc * eb,
                    data.data() + ((blk[0] * lr + r) * cols + blk[1] * lc) * eb,
                    static_cast<size_t>(lc * eb));
      void* dptr = nullptr;
      cudaMalloc(&dptr, host.size());
      cudaMemcpy(dptr, host.data(), host.size(), cudaMemcpyHostToDevice);
      owned.push_back(dptr);
      shards.push_back(dptr);
    }
    feeds[id] = shards;
  }
  cudaStream_t stream;
  cudaStreamCreate(&stream);
  std::vector<void*> out;
  for (int i = 0; i < 2; ++i) out = ex.forward(feeds, stream);  // second call reuses buffers
  cudaStreamSynchronize(stream);
  const TensorMeta& om = ex.meta("out");
  size_t bytes = static_cast<size_t>(om.dtype_bytes);
  for (int64_t e : om.shape) bytes *= static_cast<size_t>(e);
  std::vector<char> host(bytes);
  if (cudaMemcpy(host.data(), out.at(0), bytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
    std::fprintf(stderr, "copy-back failed\n");
    return 1;
  }
  std::ofstream(dir + "/out.bin", std::ios::binary).write(host.data(), static_cast<long>(bytes));
  for (void* p : owned) cudaFree(p);
  std::cout << "plan executed on " << mesh.num_devices() << " simulated devices\n";
  return 0;
}
