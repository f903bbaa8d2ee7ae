// Neighbour generation, heuristic, best-first path search, pricing, cache.
//
// Behavioural parity targets (reference file:line):
//   one_step_transforms   proj/src/layout.cpp:162-221  (generation order, validity
//                         filter, first-seen dedup)
//   dim_diff              proj/src/layout.cpp:223-237
//   heuristic_diff        proj/src/layout.cpp:239-251
//   find_transform_path   proj/src/layout.cpp:253-316  (ShapeError on invalid ends,
//                         (score, sequence) min-order, close-on-generate,
//                         stop-on-generate, InfeasibleError when exhausted)
//   conversion_cost       proj/src/layout.cpp:318-329  (bytes = shard before step)
//   PathCache             proj/src/layout.cpp:331-362
//
// Differences that do not change results: states are keyed by a compact
// byte string instead of an ostringstream rendering, and the open list is an
// explicit binary heap over (score, sequence) pairs.
#include <algorithm>
#include <queue>
#include <unordered_set>

#include "autoplan/layout.hpp"

namespace autoplan {

namespace {

// Unambiguous compact state key: axis bytes per dim, 0xFF terminates a dim.
std::string state_key(const ShardingSpec& spec) {
  std::string key;
  key.reserve(spec.dims.size() * 3);
  for (const DimSpec& d : spec.dims) {
    for (int a : d.axes) key.push_back(static_cast<char>(a & 0x7F));
    key.push_back(static_cast<char>(0xFF));
  }
  return key;
}

void require_rank(const ShardingSpec& spec, const TensorMeta& meta) {
  if (static_cast<int64_t>(spec.tensor_rank()) != meta.rank()) {
    throw RankMismatchError("sharding spec rank " + std::to_string(spec.tensor_rank()) +
                            " does not match tensor rank " + std::to_string(meta.rank()));
  }
}

TransformStep make_step(CollectiveKind kind, int dim, int target, int axis) {
  TransformStep s;
  s.kind = kind;
  s.tensor_dim = dim;
  s.target_dim = target;
  s.mesh_axis = axis;
  return s;
}

}  // namespace

std::vector<std::pair<ShardingSpec, TransformStep>> one_step_transforms(
    const ShardingSpec& spec, const DeviceMesh& mesh, const TensorMeta& meta) {
  require_rank(spec, meta);
  std::vector<std::pair<ShardingSpec, TransformStep>> out;
  std::unordered_set<std::string> keys;
  auto offer = [&](ShardingSpec candidate, TransformStep step) {
    if (!candidate.valid_for(meta, mesh)) return;
    if (!keys.insert(state_key(candidate)).second) return;
    step.result = candidate;
    out.emplace_back(std::move(candidate), std::move(step));
  };

  const int rank = spec.tensor_rank();
  std::vector<char> in_use(static_cast<size_t>(std::max(spec.mesh_rank, 0)), 0);
  for (const DimSpec& d : spec.dims)
    for (int a : d.axes)
      if (a >= 0 && a < spec.mesh_rank) in_use[static_cast<size_t>(a)] = 1;

  // 1. gathers: drop the trailing axis of each sharded dim.
  for (int d = 0; d < rank; ++d) {
    const auto& axes = spec.dims[static_cast<size_t>(d)].axes;
    if (axes.empty()) continue;
    ShardingSpec next = spec;
    next.dims[static_cast<size_t>(d)].axes.pop_back();
    offer(std::move(next), make_step(CollectiveKind::kAllGather, d, -1, axes.back()));
  }
  // 2. slices: append any free axis to any dim.
  for (int d = 0; d < rank; ++d) {
    for (int a = 0; a < spec.mesh_rank; ++a) {
      if (in_use[static_cast<size_t>(a)]) continue;
      ShardingSpec next = spec;
      next.dims[static_cast<size_t>(d)].axes.push_back(a);
      offer(std::move(next), make_step(CollectiveKind::kShardSlice, d, -1, a));
    }
  }
  // 3. all-to-alls: move a dim's trailing axis onto another dim.
  for (int d = 0; d < rank; ++d) {
    const auto& axes = spec.dims[static_cast<size_t>(d)].axes;
    if (axes.empty()) continue;
    const int moved = axes.back();
    for (int t = 0; t < rank; ++t) {
      if (t == d) continue;
      ShardingSpec next = spec;
      next.dims[static_cast<size_t>(d)].axes.pop_back();
      next.dims[static_cast<size_t>(t)].axes.push_back(moved);
      offer(std::move(next), make_step(CollectiveKind::kAllToAll, d, t, moved));
    }
  }
  return out;
}

double dim_diff(const DimSpec& src, const DimSpec& tgt, const DimDiffWeights& w) {
  const size_t limit = std::min(src.axes.size(), tgt.axes.size());
  size_t prefix = 0;
  while (prefix < limit && src.axes[prefix] == tgt.axes[prefix]) ++prefix;
  // Everything past the shared prefix is gathered off, then sliced back on.
  const double gathers = static_cast<double>(src.axes.size() - prefix);
  const double slices = static_cast<double>(tgt.axes.size() - prefix);
  const double ops = gathers + slices;
  double score = gathers * w.all_gather + slices * w.shard;
  if (ops > 1) score += w.step_penalty * (ops - 1);
  return score;
}

double heuristic_diff(const ShardingSpec& src, const ShardingSpec& tgt,
                      const DimDiffWeights& w) {
  if (src.tensor_rank() != tgt.tensor_rank()) {
    throw RankMismatchError("cannot compare sharding specs of ranks " +
                            std::to_string(src.tensor_rank()) + " and " +
                            std::to_string(tgt.tensor_rank()));
  }
  double sum = 0;
  for (size_t d = 0; d < src.dims.size(); ++d) sum += dim_diff(src.dims[d], tgt.dims[d], w);
  return sum;
}

TransformPath find_transform_path(const ShardingSpec& src, const ShardingSpec& tgt,
                                  const DeviceMesh& mesh, const TensorMeta& meta,
                                  const DimDiffWeights& w) {
  if (!src.valid_for(meta, mesh))
    throw ShapeError("source sharding spec " + src.to_string() + " is not valid for the tensor/mesh");
  if (!tgt.valid_for(meta, mesh))
    throw ShapeError("target sharding spec " + tgt.to_string() + " is not valid for the tensor/mesh");

  TransformPath path;
  path.source = src;
  path.target = tgt;
  if (src == tgt) return path;

  // Search tree stored flat; `via[i]` is the step that produced state i from
  // state `from[i]`.
  std::vector<ShardingSpec> state{src};
  std::vector<int> from{-1};
  std::vector<TransformStep> via(1);
  std::unordered_set<std::string> closed{state_key(src)};
  const std::string goal = state_key(tgt);

  using Entry = std::pair<double, int>;  // (score, sequence number == state index)
  std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> frontier;
  frontier.emplace(heuristic_diff(src, tgt, w), 0);

  int reached = -1;
  while (reached < 0 && !frontier.empty()) {
    const int at = frontier.top().second;
    frontier.pop();
    const ShardingSpec here = state[static_cast<size_t>(at)];
    for (auto& [next, step] : one_step_transforms(here, mesh, meta)) {
      std::string key = state_key(next);
      if (!closed.insert(key).second) continue;
      const int id = static_cast<int>(state.size());
      state.push_back(next);
      from.push_back(at);
      via.push_back(step);
      if (key == goal) {
        reached = id;
        break;
      }
      frontier.emplace(heuristic_diff(next, tgt, w), id);
    }
  }
  if (reached < 0) {
    throw InfeasibleError("no conversion path from " + src.to_string() + " to " +
                          tgt.to_string());
  }
  for (int i = reached; i > 0; i = from[static_cast<size_t>(i)]) path.steps.push_back(via[static_cast<size_t>(i)]);
  std::reverse(path.steps.begin(), path.steps.end());
  return path;
}

double conversion_cost(TransformPath& path, const DeviceMesh& mesh, const TensorMeta& meta) {
  double seconds = 0;
  const ShardingSpec* before = &path.source;
  for (const TransformStep& s : path.steps) {
    const int64_t shard_bytes = before->per_device_bytes(meta, mesh);
    seconds += collective_cost(mesh, {s.mesh_axis}, s.kind, static_cast<double>(shard_bytes));
    before = &s.result;
  }
  path.comm_cost_s = seconds;
  return seconds;
}

TransformPath PathCache::get(const ShardingSpec& src, const ShardingSpec& tgt,
                             const DeviceMesh& mesh, const TensorMeta& meta) {
  std::string key = state_key(src);
  key.push_back('|');
  key += state_key(tgt);
  key.push_back('|');
  key += mesh.shape_string();
  key.push_back('|');
  for (int64_t e : meta.shape) {
    key += std::to_string(e);
    key.push_back(',');
  }
  key.push_back('|');
  key += std::to_string(meta.dtype_bytes);

  std::lock_guard<std::mutex> hold(mutex_);
  if (auto hit = cache_.find(key); hit != cache_.end()) return hit->second;
  TransformPath path = find_transform_path(src, tgt, mesh, meta);
  conversion_cost(path, mesh, meta);
  ++searches_;
  cache_.emplace(std::move(key), path);
  return path;
}

void PathCache::clear() {
  std::lock_guard<std::mutex> hold(mutex_);
  cache_.clear();
  searches_ = 0;
}

size_t PathCache::searches() const {
  std::lock_guard<std::mutex> hold(mutex_);
  return searches_;
}

size_t PathCache::size() const {
  std::lock_guard<std::mutex> hold(mutex_);
  return cache_.size();
}

}  // namespace autoplan
