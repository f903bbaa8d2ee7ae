// Device-mesh geometry and the collective vocabulary (drop-in subset).
//
// Same names and signatures as the reference's cluster header
// (proj/include/autoplan/cluster.hpp:46-98) for the parts the layout hot path
// touches: CollectiveKind, DeviceMesh, parse_mesh_shape, collective_cost.
// The topology parser / greedy mesh builder (cluster.cpp:129-372) is planning
// code outside the hot path and is not part of this build.
//
// Placement contract used by the runtime: mesh coordinates map to ranks in
// row-major order (cluster.hpp:56), i.e. rank = sum_i c_i * prod_{j>i} n_j.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "autoplan/errors.hpp"

namespace autoplan {

enum class CollectiveKind {
  kAllGather,
  kAllReduce,
  kReduceScatter,
  kAllToAll,
  kShardSlice,  // local: no bytes cross a link
};

// "all-gather", "all-reduce", "reduce-scatter", "all-to-all", "shard-slice".
const char* to_string(CollectiveKind kind);

struct DeviceMesh {
  std::vector<int64_t> shape;
  std::vector<std::string> assignment;  // row-major coordinate -> device name
  std::vector<double> axis_alpha;       // seconds of latency per axis
  std::vector<double> axis_beta_inv;    // seconds per byte per axis
  double device_flops_per_s = 0;
  std::vector<std::string> warnings;

  int rank() const { return static_cast<int>(shape.size()); }
  int64_t num_devices() const;
  int64_t axis_extent(int axis) const;  // AxisError when out of range
  std::string shape_string() const;     // e.g. "2x4"

  // Row-major coordinate <-> linear device index helpers (runtime side).
  std::vector<int64_t> coord_of(int64_t device) const;
  int64_t device_of(const std::vector<int64_t>& coord) const;

  static DeviceMesh uniform(const std::vector<int64_t>& shape, double alpha = 1e-5,
                            double beta_inv = 1e-9, double device_flops_per_s = 1e12);
};

// "2x4" -> {2, 4}; SchemaError on malformed text.
std::vector<int64_t> parse_mesh_shape(const std::string& text);

// Alpha-beta ring price of one collective over the product of `axes`; the
// slowest axis sets alpha and beta. `bytes` is the per-participant payload.
double collective_cost(const DeviceMesh& mesh, const std::vector<int>& axes,
                       CollectiveKind kind, double bytes);

std::string mesh_report(const DeviceMesh& mesh);

}  // namespace autoplan

// Mesh round-trip helpers (reference cluster.hpp:93-96, cluster.cpp:417-450):
// solution and plan documents embed the mesh. Declared when nlohmann/json is
// on the include path (the reference's own JSON library); libapl.so is built
// with it and exports both. Same fields, same SchemaError cases.
#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
namespace autoplan {
nlohmann::json mesh_to_json(const DeviceMesh& mesh);
DeviceMesh mesh_from_json(const nlohmann::json& doc);
}  // namespace autoplan
#endif
