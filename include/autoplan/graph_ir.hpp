// Tensor metadata (drop-in subset of the reference graph IR).
//
// Only TensorMeta (proj/include/autoplan/graph_ir.hpp:33-43) is on the layout
// hot path; the graph parser / profiler are analysis code outside this build.
#pragma once

#include <cstdint>
#include <vector>

namespace autoplan {

struct TensorMeta {
  std::vector<int64_t> shape;
  int dtype_bytes = 4;  // one of {1, 2, 4, 8} (graph_ir.cpp:81-84)
  bool requires_grad = false;

  int64_t rank() const { return static_cast<int64_t>(shape.size()); }
  int64_t num_elements() const {
    int64_t n = 1;
    for (int64_t e : shape) n *= e;
    return n;
  }
  int64_t bytes() const { return num_elements() * dtype_bytes; }

  bool operator==(const TensorMeta&) const = default;
};

}  // namespace autoplan
