// C++ drop-in check: code written against the reference's layout API
// (proj/include/autoplan/layout.hpp) compiles against include/autoplan and
// links libapl.so unchanged. Mirrors proj/tests/test_layout.cpp cases.
#include <cstdio>
#include <set>
#include <string>

#include "autoplan/execute.hpp"
#include "autoplan/layout.hpp"

using namespace autoplan;

static int failures = 0;
#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      ++failures;                                                 \
    }                                                             \
  } while (0)

int main(int argc, char** argv) {
  const bool has_gpu = argc > 1 && std::string(argv[1]) == "--gpu";
  const TensorMeta square{{8, 8}, 4, false};
  const DeviceMesh mesh = DeviceMesh::uniform({2, 4}, 1e-5, 1e-9, 1e12);

  CHECK(ShardingSpec::parse("S10R", 2).to_string() == "S10R");
  bool threw = false;
  try {
    ShardingSpec::parse("S9R", 2);
  } catch (const AxisError&) {
    threw = true;
  }
  CHECK(threw);

  std::set<std::string> names;
  for (auto& [spec, step] : one_step_transforms(ShardingSpec::parse("S0R", 2), mesh, square))
    names.insert(spec.to_string());
  CHECK((names == std::set<std::string>{"RR", "S0S1", "S01R", "RS0"}));

  TransformPath p = find_transform_path(ShardingSpec::parse("S0R", 2), ShardingSpec::parse("RS0", 2),
                                        mesh, square);
  CHECK(p.steps.size() == 1 && p.steps[0].kind == CollectiveKind::kAllToAll &&
        p.steps[0].tensor_dim == 0 && p.steps[0].target_dim == 1 && p.steps[0].mesh_axis == 0);

  const DeviceMesh m4 = DeviceMesh::uniform({4}, 1e-5, 1e-9, 1e12);
  const TensorMeta big{{1024, 1024}, 4, false};
  TransformPath g = find_transform_path(ShardingSpec::parse("S0R", 1), ShardingSpec::replicated(2, 1),
                                        m4, big);
  const double want = 3e-5 + 0.75 * 1048576 * 1e-9;
  const double got = conversion_cost(g, m4, big);
  CHECK(got > want * (1 - 1e-12) && got < want * (1 + 1e-12));

  PathCache cache;
  cache.get(ShardingSpec::parse("S0R", 2), ShardingSpec::parse("RS0", 2), mesh, square);
  cache.get(ShardingSpec::parse("S0R", 2), ShardingSpec::parse("RS0", 2), mesh, square);
  CHECK(cache.searches() == 1 && cache.size() == 1);

  // Runtime surface: on a CPU-only host creating a device mesh must fail
  // loudly (no fallback); on a GPU host it must succeed.
  bool failed = false;
  try {
    MeshRuntime rt = MeshRuntime::Simulated(mesh, 0);
    CHECK(workspace_bytes(rt, p, square, true) == 0);
  } catch (const RuntimeFailure& e) {
    failed = true;
  }
  CHECK(failed != has_gpu);
  if (failures == 0) std::puts("drop-in ok");
  return failures == 0 ? 0 : 1;
}
