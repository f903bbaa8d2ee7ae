// Matmul strategy catalog.
//
// Behavioural parity targets (reference file:line):
//   candidate generation     proj/src/intraop.cpp:141-234 (names, order)
//   finalize                 proj/src/intraop.cpp:497-555 (fallback appended last,
//                            validity filter, first-seen dedup on specs+reduce
//                            axes, FLOP/all-reduce pricing)
//   engaged_devices          proj/src/intraop.cpp:582-591
//   matmul FLOPs             proj/src/graph_ir.cpp:669-688 (2mkn, bwd 2x)
#include <set>
#include <utility>

#include "autoplan/matmul_strategies.hpp"

namespace autoplan {

namespace {

using Placement = std::vector<std::pair<int, std::vector<int>>>;

ShardingSpec placed(int rank, int mesh_rank, const Placement& p) {
  ShardingSpec s = ShardingSpec::replicated(rank, mesh_rank);
  for (const auto& [dim, axes] : p) s.dims[static_cast<size_t>(dim)].axes = axes;
  return s;
}

std::string digits(const std::vector<int>& axes) {
  std::string t;
  for (int a : axes) t += std::to_string(a);
  return t;
}

std::string dedup_key(const OpStrategy& s) {
  std::string k;
  for (const ShardingSpec& in : s.input_specs) k += in.to_string() + "|";
  k += ">" + s.output_spec.to_string();
  for (int a : s.reduce_axes) k += "+" + std::to_string(a);
  return k;
}

}  // namespace

int64_t engaged_devices(const OpStrategy& s, const DeviceMesh& mesh) {
  std::set<int> axes;
  for (const ShardingSpec& in : s.input_specs)
    for (int a : in.used_axes()) axes.insert(a);
  for (int a : s.output_spec.used_axes()) axes.insert(a);
  int64_t n = 1;
  for (int a : axes) n *= mesh.axis_extent(a);
  return n;
}

std::vector<OpStrategy> matmul_strategies(const TensorMeta& a, const TensorMeta& b,
                                          const DeviceMesh& mesh, bool batched) {
  const int mr = mesh.rank();
  const int ra = static_cast<int>(a.rank());
  const int rb = static_cast<int>(b.rank());
  TensorMeta c = a;  // output meta: A's leading dims + B's last dim
  c.shape.back() = b.shape.back();
  const int rc = static_cast<int>(c.rank());

  std::vector<OpStrategy> raw;
  auto add = [&](std::string name, const Placement& pa, const Placement& pb,
                 const Placement& pc, std::vector<int> reduce) {
    OpStrategy s;
    s.name = std::move(name);
    s.input_specs = {placed(ra, mr, pa), placed(rb, mr, pb)};
    s.output_spec = placed(rc, mr, pc);
    s.partial_sum = !reduce.empty();
    s.reduce_axes = std::move(reduce);
    raw.push_back(std::move(s));
  };

  // single axes, then ascending two-axis groups
  std::vector<std::vector<int>> groups;
  for (int x = 0; x < mr; ++x) groups.push_back({x});
  for (int x = 0; x < mr; ++x)
    for (int y = x + 1; y < mr; ++y) groups.push_back({x, y});

  if (!batched) {
    const int kd = ra - 1, nd = rc - 1;
    for (const auto& g : groups) {
      const std::string t = digits(g);
      for (int i = 0; i + 2 <= ra; ++i)
        add("split-m@" + std::to_string(i) + ":" + t, {{i, g}}, {}, {{i, g}}, {});
      add("split-n:" + t, {}, {{1, g}}, {{nd, g}}, {});
      add("split-k:" + t, {{kd, g}}, {{0, g}}, {}, g);
    }
    for (int x = 0; x < mr; ++x) {
      for (int y = 0; y < mr; ++y) {
        if (x == y) continue;
        const std::string t = std::to_string(x) + "," + std::to_string(y);
        for (int i = 0; i + 2 <= ra; ++i) {
          const std::string at = std::to_string(i);
          add("split-mn@" + at + ":" + t, {{i, {x}}}, {{1, {y}}}, {{i, {x}}, {nd, {y}}}, {});
          add("split-mk@" + at + ":" + t, {{i, {x}}, {kd, {y}}}, {{0, {y}}}, {{i, {x}}}, {y});
        }
        add("split-nk:" + t, {{kd, {y}}}, {{0, {y}}, {1, {x}}}, {{nd, {x}}}, {y});
        if (x < y) {
          for (int i = 0; i + 2 <= ra; ++i)
            for (int j = i + 1; j + 2 <= ra; ++j)
              add("split-mm@" + std::to_string(i) + "," + std::to_string(j) + ":" + t,
                  {{i, {x}}, {j, {y}}}, {}, {{i, {x}}, {j, {y}}}, {});
        }
      }
    }
  } else {
    for (const auto& g : groups) {
      const std::string t = digits(g);
      add("split-b:" + t, {{0, g}}, {{0, g}}, {{0, g}}, {});
      add("split-m:" + t, {{1, g}}, {}, {{1, g}}, {});
      add("split-n:" + t, {}, {{2, g}}, {{2, g}}, {});
      add("split-k:" + t, {{2, g}}, {{1, g}}, {}, g);
    }
    for (int x = 0; x < mr; ++x) {
      for (int y = 0; y < mr; ++y) {
        if (x == y) continue;
        const std::string t = std::to_string(x) + "," + std::to_string(y);
        add("split-bm:" + t, {{0, {x}}, {1, {y}}}, {{0, {x}}}, {{0, {x}}, {1, {y}}}, {});
        add("split-bn:" + t, {{0, {x}}}, {{0, {x}}, {2, {y}}}, {{0, {x}}, {2, {y}}}, {});
        add("split-bk:" + t, {{0, {x}}, {2, {y}}}, {{0, {x}}, {1, {y}}}, {{0, {x}}}, {y});
        add("split-mn:" + t, {{1, {x}}}, {{2, {y}}}, {{1, {x}}, {2, {y}}}, {});
        add("split-mk:" + t, {{1, {x}}, {2, {y}}}, {{1, {y}}}, {{1, {x}}}, {y});
        add("split-nk:" + t, {{2, {y}}}, {{1, {y}}, {2, {x}}}, {{2, {x}}}, {y});
      }
    }
  }
  add("replicated", {}, {}, {}, {});

  // FLOP model (graph_ir.cpp:669-688) and output bytes.
  double m = 1;
  for (int i = 0; i + 1 < ra; ++i) m *= static_cast<double>(a.shape[static_cast<size_t>(i)]);
  const double flops = batched ? 2.0 * static_cast<double>(a.shape[0]) *
                                     static_cast<double>(a.shape[1]) *
                                     static_cast<double>(a.shape[2]) *
                                     static_cast<double>(b.shape[2])
                               : 2.0 * m * static_cast<double>(a.shape.back()) *
                                     static_cast<double>(b.shape[1]);
  const int64_t out_bytes = c.bytes();
  const double rate = mesh.device_flops_per_s;

  std::vector<OpStrategy> out;
  std::set<std::string> seen;
  for (OpStrategy& s : raw) {
    if (!s.input_specs[0].valid_for(a, mesh) || !s.input_specs[1].valid_for(b, mesh) ||
        !s.output_spec.valid_for(c, mesh))
      continue;
    if (!seen.insert(dedup_key(s)).second) continue;
    const int64_t engaged = engaged_devices(s, mesh);
    if (rate > 0) {
      s.compute_time_s = flops / static_cast<double>(engaged) / rate;
      s.bwd_compute_time_s = 2.0 * flops / static_cast<double>(engaged) / rate;
    }
    const int64_t shards = s.output_spec.shard_count(mesh);
    s.memory_bytes = out_bytes / shards;
    if (s.partial_sum) {
      const double buffer = static_cast<double>(out_bytes / shards);
      s.comm_time_s = collective_cost(mesh, s.reduce_axes, CollectiveKind::kAllReduce, buffer);
      s.comm_buffer_bytes = static_cast<int64_t>(buffer);
      s.bwd_comm_time_s = s.comm_time_s;
    }
    out.push_back(std::move(s));
  }
  return out;
}

OpStrategy find_matmul_strategy(const std::string& name, const TensorMeta& a,
                                const TensorMeta& b, const DeviceMesh& mesh, bool batched) {
  for (OpStrategy& s : matmul_strategies(a, b, mesh, batched))
    if (s.name == name) return s;
  throw MissingStrategyError("no valid matmul strategy named '" + name + "' for these shapes");
}

}  // namespace autoplan
