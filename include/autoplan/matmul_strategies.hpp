// Sharded-matmul strategy catalog (drop-in subset of the reference intra-op
// module, proj/include/autoplan/intraop.hpp:34-49 and
// proj/src/intraop.cpp:141-234, 497-555, 582-591).
//
// The runtime executes these strategies (apl_sharded_matmul); the catalog is
// here so a plan document that names a strategy ("split-mk@0:1,0") can be
// decoded into its input/output specs and reduce axes without the solver.
// Names, order, divisibility filter, dedup and the replicated fallback match
// the reference; tests/test_strategies.py compares against oracle/_ref.
#pragma once

#include <string>
#include <vector>

#include "autoplan/cluster.hpp"
#include "autoplan/graph_ir.hpp"
#include "autoplan/layout.hpp"

namespace autoplan {

// The reference's own definition when its intraop.hpp is already included
// (a caller mixing the reference planner with this drop-in); the layouts
// are identical (intraop.hpp:34-49).
#ifndef AUTOPLAN_INTRAOP_HPP_
struct OpStrategy {
  std::string node;
  std::string name;
  std::vector<ShardingSpec> input_specs;
  ShardingSpec output_spec;
  bool partial_sum = false;
  std::vector<int> reduce_axes;
  double compute_time_s = 0;
  double comm_time_s = 0;
  double bwd_compute_time_s = 0;
  double bwd_comm_time_s = 0;
  int64_t comm_buffer_bytes = 0;
  int64_t memory_bytes = 0;
};
#endif

// Every valid strategy of C[..m.., n] = A[..m.., k] . B[k, n] (batched ==
// false) or C[b,m,n] = A[b,m,k] . B[b,k,n] (batched == true) on `mesh`, in
// the reference's order, priced like the reference (FLOP model of
// graph_ir.cpp:665-690, all-reduce on the output shard).
std::vector<OpStrategy> matmul_strategies(const TensorMeta& a, const TensorMeta& b,
                                          const DeviceMesh& mesh, bool batched = false);

// Product of the extents of every mesh axis any operand uses.
int64_t engaged_devices(const OpStrategy& strategy, const DeviceMesh& mesh);

// Looks a strategy up by name; throws MissingStrategyError when absent.
OpStrategy find_matmul_strategy(const std::string& name, const TensorMeta& a,
                                const TensorMeta& b, const DeviceMesh& mesh,
                                bool batched = false);

}  // namespace autoplan
