// DeviceMesh geometry, mesh-shape parsing and alpha-beta collective pricing.
//
// Behavioural parity targets (reference file:line):
//   DeviceMesh::uniform        proj/src/cluster.cpp:195-205
//   parse_mesh_shape           proj/src/cluster.cpp:207-227
//   collective_cost            proj/src/cluster.cpp:374-400 (same float order)
//   to_string(CollectiveKind)  proj/src/cluster.cpp:118-127
#include <algorithm>
#include <cctype>
#include <sstream>

#include "autoplan/cluster.hpp"

namespace autoplan {

const char* to_string(CollectiveKind kind) {
  static const char* const kNames[] = {"all-gather", "all-reduce", "reduce-scatter",
                                       "all-to-all", "shard-slice"};
  const int k = static_cast<int>(kind);
  return (k >= 0 && k < 5) ? kNames[k] : "?";
}

int64_t DeviceMesh::num_devices() const {
  int64_t total = 1;
  for (int64_t e : shape) total *= e;
  return total;
}

int64_t DeviceMesh::axis_extent(int axis) const {
  if (axis < 0 || axis >= rank()) {
    throw AxisError("mesh axis " + std::to_string(axis) + " is outside a rank-" +
                    std::to_string(rank()) + " mesh");
  }
  return shape[static_cast<size_t>(axis)];
}

std::string DeviceMesh::shape_string() const {
  std::string text;
  for (size_t i = 0; i < shape.size(); ++i) {
    if (i != 0) text.push_back('x');
    text += std::to_string(shape[i]);
  }
  return text;
}

std::vector<int64_t> DeviceMesh::coord_of(int64_t device) const {
  std::vector<int64_t> coord(shape.size(), 0);
  for (int i = rank() - 1; i >= 0; --i) {
    coord[static_cast<size_t>(i)] = device % shape[static_cast<size_t>(i)];
    device /= shape[static_cast<size_t>(i)];
  }
  return coord;
}

int64_t DeviceMesh::device_of(const std::vector<int64_t>& coord) const {
  int64_t device = 0;
  for (size_t i = 0; i < shape.size(); ++i) device = device * shape[i] + coord[i];
  return device;
}

DeviceMesh DeviceMesh::uniform(const std::vector<int64_t>& shape, double alpha,
                               double beta_inv, double device_flops_per_s) {
  DeviceMesh mesh;
  mesh.shape = shape;
  mesh.axis_alpha = std::vector<double>(shape.size(), alpha);
  mesh.axis_beta_inv = std::vector<double>(shape.size(), beta_inv);
  mesh.device_flops_per_s = device_flops_per_s;
  const int64_t count = mesh.num_devices();
  mesh.assignment.reserve(static_cast<size_t>(count));
  for (int64_t d = 0; d < count; ++d) mesh.assignment.push_back("d" + std::to_string(d));
  return mesh;
}

std::vector<int64_t> parse_mesh_shape(const std::string& text) {
  auto bad = [&]() { return SchemaError("malformed mesh shape '" + text + "' (want e.g. 2x4)"); };
  if (text.empty()) throw SchemaError("empty mesh shape");
  std::vector<int64_t> extents;
  size_t pos = 0;
  while (true) {
    size_t end = text.find('x', pos);
    std::string field = text.substr(pos, end == std::string::npos ? std::string::npos : end - pos);
    // Digits only (std::stoll-compatible leading whitespace/sign is not a
    // documented form; a sign would be rejected by the >=1 rule anyway).
    if (field.empty()) throw bad();
    int64_t value = 0;
    try {
      size_t used = 0;
      value = std::stoll(field, &used);
      if (used == 0) throw bad();
    } catch (const std::exception&) {
      throw bad();
    }
    if (value < 1) throw bad();
    extents.push_back(value);
    if (end == std::string::npos) break;
    pos = end + 1;
  }
  return extents;
}

double collective_cost(const DeviceMesh& mesh, const std::vector<int>& axes,
                       CollectiveKind kind, double bytes) {
  if (bytes < 0) throw PlanError("collective payload must be non-negative");
  double group = 1, alpha = 0, beta_inv = 0;
  for (int a : axes) {
    group *= static_cast<double>(mesh.axis_extent(a));
    alpha = std::max(alpha, mesh.axis_alpha[static_cast<size_t>(a)]);
    beta_inv = std::max(beta_inv, mesh.axis_beta_inv[static_cast<size_t>(a)]);
  }
  if (kind == CollectiveKind::kShardSlice || group <= 1) return 0.0;
  // Ring model: (p-1) latency hops, (p-1)/p of the payload on the wire.
  const double hops = group - 1.0;
  const double wire = (group - 1.0) / group * bytes * beta_inv;
  if (kind == CollectiveKind::kAllReduce) return 2.0 * hops * alpha + 2.0 * wire;
  return hops * alpha + wire;
}

std::string mesh_report(const DeviceMesh& mesh) {
  std::ostringstream os;
  os << "mesh shape: " << mesh.shape_string() << "\n";
  for (int a = 0; a < mesh.rank(); ++a) {
    os << "axis " << a << ": extent " << mesh.shape[static_cast<size_t>(a)] << ", alpha "
       << mesh.axis_alpha[static_cast<size_t>(a)] << " s, beta_inv "
       << mesh.axis_beta_inv[static_cast<size_t>(a)] << " s/B\n";
  }
  os << "assignment (row-major):";
  for (const std::string& name : mesh.assignment) os << " " << name;
  os << "\n";
  for (const std::string& w : mesh.warnings) os << "warning: " << w << "\n";
  return os.str();
}

#if __has_include(<nlohmann/json.hpp>)
// Document form of a mesh (cluster.cpp:417-450): the five tabled fields;
// `warnings` is diagnostic and not serialised.
nlohmann::json mesh_to_json(const DeviceMesh& mesh) {
  nlohmann::json doc;
  doc["shape"] = mesh.shape;
  doc["assignment"] = mesh.assignment;
  doc["axis_alpha"] = mesh.axis_alpha;
  doc["axis_beta_inv"] = mesh.axis_beta_inv;
  doc["device_flops_per_s"] = mesh.device_flops_per_s;
  return doc;
}

DeviceMesh mesh_from_json(const nlohmann::json& doc) {
  if (!doc.is_object()) throw SchemaError("mesh document must be an object");
  DeviceMesh mesh;
  try {
    doc.at("shape").get_to(mesh.shape);
    doc.at("assignment").get_to(mesh.assignment);
    doc.at("axis_alpha").get_to(mesh.axis_alpha);
    doc.at("axis_beta_inv").get_to(mesh.axis_beta_inv);
    mesh.device_flops_per_s = doc.at("device_flops_per_s").get<double>();
  } catch (const nlohmann::json::exception& e) {
    throw SchemaError(std::string("malformed mesh document: ") + e.what());
  }
  int64_t devices = 1;
  for (const int64_t n : mesh.shape) {
    if (n < 1) throw SchemaError("mesh extents must be positive");
    devices *= n;
  }
  const size_t r = mesh.shape.size();
  if (static_cast<int64_t>(mesh.assignment.size()) != devices || mesh.axis_alpha.size() != r ||
      mesh.axis_beta_inv.size() != r)
    throw SchemaError("mesh document fields have inconsistent sizes");
  return mesh;
}
#endif

}  // namespace autoplan
