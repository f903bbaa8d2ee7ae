// apl_convert: the reference CLI's `plan convert` (proj/tools/plan_main.cpp:
// 98-109 options, 179-202 output) on the drop-in layout API, plus the
// execute mode SURVEY 2 row 8 asks for: run the conversion on B200 shards.
//
//   apl_convert --from S0R --to RS0 --mesh 2x2 --shape 1024x1024 [--dtype-bytes 4]
//               [--execute [--stepwise] [--iters N] [--device D]]
//
// Without --execute the output is the reference's, line for line. With it,
// the conversion runs on a simulated mesh (every mesh device a buffer on
// one GPU): source shards are filled with a byte pattern, converted, then
// converted back along the reverse path; the tool checks the round trip is
// bit-exact and reports the device time and HBM GB/s of the forward pass.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

#include "autoplan/execute.hpp"
#include "autoplan/layout.hpp"

namespace {

void usage() {
  std::fprintf(stderr,
               "usage: apl_convert --from SPEC --to SPEC --mesh AxB --shape XxY "
               "[--dtype-bytes N] [--execute [--stepwise] [--iters N] [--device D]]\n");
  std::exit(2);
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(3);
  }
}

int64_t local_bytes(const autoplan::ShardingSpec& s, const autoplan::DeviceMesh& mesh,
                    const autoplan::TensorMeta& meta) {
  return s.per_device_bytes(meta, mesh);
}

}  // namespace

int main(int argc, char** argv) {
  std::string from, to, mesh_arg, shape_arg;
  int dtype_bytes = 4, iters = 20, device = 0;
  bool execute = false, stepwise = false;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage();
      return argv[++i];
    };
    if (a == "--from") from = val();
    else if (a == "--to") to = val();
    else if (a == "--mesh") mesh_arg = val();
    else if (a == "--shape") shape_arg = val();
    else if (a == "--dtype-bytes") dtype_bytes = std::atoi(val().c_str());
    else if (a == "--execute") execute = true;
    else if (a == "--stepwise") stepwise = true;
    else if (a == "--iters") iters = std::atoi(val().c_str());
    else if (a == "--device") device = std::atoi(val().c_str());
    else usage();
  }
  if (from.empty() || to.empty() || mesh_arg.empty() || shape_arg.empty()) usage();
  try {
    // plan_main.cpp:179-202
    autoplan::DeviceMesh mesh = autoplan::DeviceMesh::uniform(autoplan::parse_mesh_shape(mesh_arg));
    autoplan::TensorMeta meta;
    meta.shape = autoplan::parse_mesh_shape(shape_arg);
    meta.dtype_bytes = dtype_bytes;
    autoplan::ShardingSpec src = autoplan::ShardingSpec::parse(from, mesh.rank());
    autoplan::ShardingSpec tgt = autoplan::ShardingSpec::parse(to, mesh.rank());
    autoplan::TransformPath path = autoplan::find_transform_path(src, tgt, mesh, meta);
    double cost = autoplan::conversion_cost(path, mesh, meta);
    std::cout << src.to_string() << " -> " << tgt.to_string() << ": " << path.steps.size()
              << " step(s), " << cost << " s\n";
    autoplan::ShardingSpec cur = src;
    for (const autoplan::TransformStep& step : path.steps) {
      std::cout << "  " << autoplan::to_string(step.kind) << " dim " << step.tensor_dim;
      if (step.target_dim >= 0) std::cout << " -> dim " << step.target_dim;
      std::cout << " axis " << step.mesh_axis << ": " << cur.to_string() << " -> "
                << step.result.to_string() << '\n';
      cur = step.result;
    }
    if (!execute) return 0;

    // ---- execute mode: forward + reverse on a simulated mesh, bit-exact check
    autoplan::TransformPath back = autoplan::find_transform_path(tgt, src, mesh, meta);
    autoplan::MeshRuntime rt = autoplan::MeshRuntime::Simulated(mesh, device);
    const int64_t n = mesh.num_devices();
    const int64_t in_b = local_bytes(src, mesh, meta), out_b = local_bytes(tgt, mesh, meta);
    std::vector<void*> ins(n), outs(n), backs(n);
    std::vector<uint8_t> pattern(static_cast<size_t>(in_b));
    for (int64_t d = 0; d < n; ++d) {
      cuda_ok(cudaMalloc(&ins[d], static_cast<size_t>(in_b)), "cudaMalloc");
      cuda_ok(cudaMalloc(&outs[d], static_cast<size_t>(out_b)), "cudaMalloc");
      cuda_ok(cudaMalloc(&backs[d], static_cast<size_t>(in_b)), "cudaMalloc");
    }
    // Source shards: devices holding the same block (replicas) must hold the
    // same bytes, so fill by block index, not device index.
    for (int64_t d = 0; d < n; ++d) {
      const auto c = mesh.coord_of(d);
      uint64_t block = 0;
      for (const auto& dim : src.dims)
        for (int a : dim.axes) block = block * static_cast<uint64_t>(mesh.shape[a]) + c[a];
      uint64_t x = 0x9E3779B97F4A7C15ull * (block + 1);
      for (auto& b : pattern) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        b = static_cast<uint8_t>(x);
      }
      cuda_ok(cudaMemcpy(ins[d], pattern.data(), pattern.size(), cudaMemcpyHostToDevice), "H2D");
    }
    const bool fuse = !stepwise;
    const size_t ws1 = autoplan::workspace_bytes(rt, path, meta, fuse);
    const size_t ws2 = autoplan::workspace_bytes(rt, back, meta, fuse);
    void* ws = nullptr;
    cuda_ok(cudaMalloc(&ws, std::max<size_t>(std::max(ws1, ws2), 256)), "cudaMalloc");
    cudaStream_t stream;
    cuda_ok(cudaStreamCreate(&stream), "stream");
    autoplan::execute(rt, path, meta, ins.data(), outs.data(), ws, ws1, fuse, stream);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, stream);
    for (int i = 0; i < iters; ++i)
      autoplan::execute(rt, path, meta, ins.data(), outs.data(), ws, ws1, fuse, stream);
    cudaEventRecord(e1, stream);
    autoplan::execute(rt, back, meta, outs.data(), backs.data(), ws, ws2, fuse, stream);
    cuda_ok(cudaStreamSynchronize(stream), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= static_cast<float>(std::max(iters, 1));
    bool ok = true;
    std::vector<uint8_t> a(static_cast<size_t>(in_b)), b(static_cast<size_t>(in_b));
    for (int64_t d = 0; d < n && ok; ++d) {
      cuda_ok(cudaMemcpy(a.data(), ins[d], a.size(), cudaMemcpyDeviceToHost), "D2H");
      cuda_ok(cudaMemcpy(b.data(), backs[d], b.size(), cudaMemcpyDeviceToHost), "D2H");
      ok = std::memcmp(a.data(), b.data(), a.size()) == 0;
    }
    const double bytes = static_cast<double>(n) * static_cast<double>(in_b + out_b);
    std::cout << "execute (" << (fuse ? "collapsed" : "stepwise") << ", " << n
              << " simulated devices): " << ms * 1e3 << " us per conversion, "
              << bytes / (ms * 1e-3) / 1e9 << " GB/s (shard bytes read + written); round trip "
              << (ok ? "bit-exact" : "MISMATCH") << '\n';
    for (int64_t d = 0; d < n; ++d) {
      cudaFree(ins[d]);
      cudaFree(outs[d]);
      cudaFree(backs[d]);
    }
    cudaFree(ws);
    return ok ? 0 : 1;
  } catch (const autoplan::InfeasibleError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;  // plan_main.cpp:256-265
  } catch (const autoplan::PlanError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 3;
  }
}
