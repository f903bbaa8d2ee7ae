// DimSpec / ShardingSpec value semantics.
//
// Behavioural parity targets (reference file:line):
//   DimSpec::to_string           proj/src/layout.cpp:65-70
//   ShardingSpec::parse          proj/src/layout.cpp:79-119 (same error classes
//                                and the same checks, in the same order)
//   used_axes / shard_count      proj/src/layout.cpp:127-140
//   per_device_bytes             proj/src/layout.cpp:142-145 (integer division)
//   valid_for                    proj/src/layout.cpp:147-160
#include <algorithm>

#include "autoplan/layout.hpp"

namespace autoplan {

namespace {

int64_t extent_product(const DeviceMesh& mesh, const std::vector<int>& axes) {
  int64_t p = 1;
  for (int a : axes) p *= mesh.axis_extent(a);
  return p;
}

bool is_digit(char ch) { return ch >= '0' && ch <= '9'; }

}  // namespace

std::string DimSpec::to_string() const {
  if (axes.empty()) return "R";
  std::string text(1, 'S');
  for (int a : axes) text += std::to_string(a);
  return text;
}

ShardingSpec ShardingSpec::replicated(int tensor_rank, int mesh_rank) {
  ShardingSpec spec;
  spec.mesh_rank = mesh_rank;
  spec.dims.assign(static_cast<size_t>(tensor_rank), DimSpec{});
  return spec;
}

ShardingSpec ShardingSpec::parse(const std::string& text, int mesh_rank) {
  ShardingSpec spec;
  spec.mesh_rank = mesh_rank;
  std::vector<char> taken(static_cast<size_t>(std::max(mesh_rank, 0)), 0);
  const size_t n = text.size();
  size_t at = 0;
  while (at < n) {
    const char head = text[at++];
    if (head == 'R') {
      spec.dims.push_back(DimSpec{});
      continue;
    }
    if (head != 'S') {
      throw SchemaError("unexpected character '" + std::string(1, head) +
                        "' in sharding spec '" + text + "'");
    }
    DimSpec dim;
    for (; at < n && is_digit(text[at]); ++at) {
      const int axis = text[at] - '0';
      if (axis >= mesh_rank) {
        throw AxisError("mesh axis " + std::to_string(axis) +
                        " out of range for mesh rank " + std::to_string(mesh_rank));
      }
      if (taken[static_cast<size_t>(axis)]) {
        throw AxisError("mesh axis " + std::to_string(axis) +
                        " used more than once in spec '" + text + "'");
      }
      taken[static_cast<size_t>(axis)] = 1;
      dim.axes.push_back(axis);
    }
    if (dim.axes.empty()) {
      throw SchemaError("'S' without mesh axes in sharding spec '" + text + "'");
    }
    spec.dims.push_back(std::move(dim));
  }
  if (spec.dims.empty()) throw SchemaError("empty sharding spec");
  return spec;
}

std::string ShardingSpec::to_string() const {
  std::string text;
  for (const DimSpec& d : dims) text += d.to_string();
  return text;
}

std::vector<int> ShardingSpec::used_axes() const {
  std::vector<int> all;
  for (const DimSpec& d : dims) all.insert(all.end(), d.axes.begin(), d.axes.end());
  std::sort(all.begin(), all.end());
  return all;
}

int64_t ShardingSpec::shard_count(const DeviceMesh& mesh) const {
  int64_t count = 1;
  for (const DimSpec& d : dims) count *= extent_product(mesh, d.axes);
  return count;
}

int64_t ShardingSpec::per_device_bytes(const TensorMeta& meta, const DeviceMesh& mesh) const {
  return meta.bytes() / shard_count(mesh);
}

bool ShardingSpec::valid_for(const TensorMeta& meta, const DeviceMesh& mesh) const {
  if (dims.size() != meta.shape.size()) return false;
  if (mesh_rank != mesh.rank()) return false;
  std::vector<char> taken(static_cast<size_t>(mesh_rank), 0);
  for (size_t d = 0; d < dims.size(); ++d) {
    int64_t split = 1;
    for (int a : dims[d].axes) {
      if (a < 0 || a >= mesh_rank || taken[static_cast<size_t>(a)]) return false;
      taken[static_cast<size_t>(a)] = 1;
      split *= mesh.shape[static_cast<size_t>(a)];
    }
    if (meta.shape[d] % split != 0) return false;
  }
  return true;
}

}  // namespace autoplan
