// Runs a reference plan with the native C++ PlanExecutor on a simulated mesh:
//   plan_executor_test <graph.json> <plan.json> <mesh AxB> <dir>
// reads <dir>/<id>.bin (global row-major tensors of every placeholder and
// parameter, any rank and element size), shards them on the host by each
// node's plan spec, runs the forward pass and writes device 0's output
// replica to <dir>/out.bin. With "train" it runs forward + backward against
// <dir>/dy.bin and writes every parameter gradient to <dir>/grad_<id>.bin.
// Distributed mode (env APL_TEST_RANK, APL_TEST_IDFILE = a 128-byte NCCL
// unique id): this process is one rank of the mesh on the NCCL transport
// (MeshRuntime::Distributed), feeds only its own shards and writes its
// output replica / gradient shards as out_r<rank>.bin / grad_<id>_r<rank>.bin.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
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
  if (argc != 5 && argc != 6) {
    std::fprintf(stderr, "usage: plan_executor_test graph.json plan.json AxB dir [train]\n");
    return 2;
  }
  const bool train = argc == 6 && std::string(argv[5]) == "train";
  const std::string dir = argv[4];
  const DeviceMesh mesh = DeviceMesh::uniform(parse_mesh_shape(argv[3]));
  const char* rank_env = std::getenv("APL_TEST_RANK");
  const bool dist = rank_env != nullptr;
  const int64_t my_rank = dist ? std::atoll(rank_env) : 0;
  std::string nccl_id;
  if (dist) nccl_id = slurp(std::getenv("APL_TEST_IDFILE"));
  MeshRuntime rt = dist ? MeshRuntime::Distributed(
                              mesh, static_cast<int>(my_rank),
                              reinterpret_cast<const uint8_t*>(nccl_id.data()), 0)
                        : MeshRuntime::Simulated(mesh, 0);
  const std::string sfx = dist ? "_r" + std::to_string(my_rank) : "";
  PlanExecutor ex(rt, mesh, slurp(argv[1]), slurp(argv[2]));
  std::map<std::string, std::vector<const void*>> feeds;
  std::vector<void*> owned;
  for (const std::string& id : ex.sources()) {
    const TensorMeta& m = ex.meta(id);
    const ShardingSpec& s = ex.spec(id);
    const std::string data = slurp(dir + "/" + id + ".bin");
    const size_t rank = m.shape.size();
    const int64_t eb = m.dtype_bytes;
    std::vector<const void*> shards;
    for (int64_t d = dist ? my_rank : 0; d < (dist ? my_rank + 1 : mesh.num_devices()); ++d) {
      const auto c = mesh.coord_of(d);
      std::vector<int64_t> blk(rank, 0), loc(rank);
      int64_t total = 1;
      for (size_t k = 0; k < rank; ++k) {
        int64_t cnt = 1;
        for (int a : s.dims[k].axes) {
          blk[k] = blk[k] * mesh.shape[a] + c[a];
          cnt *= mesh.shape[a];
        }
        loc[k] = m.shape[k] / cnt;
        total *= loc[k];
      }
      // copy the block run by run (runs = the local extent of the last dim)
      std::vector<char> host(static_cast<size_t>(total * eb));
      const int64_t run = loc[rank - 1];
      std::vector<int64_t> idx(rank, 0);
      for (int64_t r = 0; r < total / run; ++r) {
        int64_t off = 0;
        for (size_t k = 0; k < rank; ++k)
          off = off * m.shape[k] + blk[k] * loc[k] + (k + 1 < rank ? idx[k] : 0);
        std::memcpy(host.data() + r * run * eb, data.data() + off * eb,
                    static_cast<size_t>(run * eb));
        for (size_t k = rank - 1; k-- > 0;) {  // next run: odometer over the leading dims
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
  std::vector<void*> out;
  std::map<std::string, std::vector<void*>> grads;
  std::vector<void*> dys;
  if (train) {  // <dir>/dy.bin: the output gradient (global bf16), replicated
    const std::string dy = slurp(dir + "/dy.bin");
    for (int64_t d = 0; d < (dist ? 1 : mesh.num_devices()); ++d) {
      void* p = nullptr;
      cudaMalloc(&p, dy.size());
      cudaMemcpy(p, dy.data(), dy.size(), cudaMemcpyHostToDevice);
      dys.push_back(p);
    }
  }
  for (int i = 0; i < 2; ++i) {  // the second step reuses every buffer
    out = ex.forward(feeds, stream, train);
    if (train) grads = ex.backward(std::vector<const void*>(dys.begin(), dys.end()), stream);
  }
  cudaStreamSynchronize(stream);
  const TensorMeta& om = ex.meta("out");
  size_t bytes = static_cast<size_t>(om.dtype_bytes);
  for (int64_t e : om.shape) bytes *= static_cast<size_t>(e);
  std::vector<char> host(bytes);
  if (cudaMemcpy(host.data(), out.at(0), bytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
    std::fprintf(stderr, "copy-back failed\n");
    return 1;
  }
  std::ofstream(dir + "/out" + sfx + ".bin", std::ios::binary)
      .write(host.data(), static_cast<long>(bytes));
  for (auto& [id, shards] : grads) {  // grad_<id>.bin: fp32 shards in device order
    const TensorMeta& m = ex.meta(id);
    TensorMeta m4 = m;
    m4.dtype_bytes = 4;
    const size_t sb = static_cast<size_t>(ex.spec(id).per_device_bytes(m4, mesh));
    std::ofstream f(dir + "/grad_" + id + sfx + ".bin", std::ios::binary);
    std::vector<char> h(sb);
    for (void* p : shards) {
      cudaMemcpy(h.data(), p, sb, cudaMemcpyDeviceToHost);
      f.write(h.data(), static_cast<long>(sb));
    }
  }
  for (void* p : dys) cudaFree(p);
  for (void* p : owned) cudaFree(p);
  if (dist)
    std::cout << "plan executed as rank " << my_rank << " of " << mesh.num_devices()
              << " over NCCL\n";
  else
    std::cout << "plan executed on " << mesh.num_devices() << " simulated devices\n";
  return 0;
}
