// C++ caller surface of the runtime: executes autoplan::TransformPath /
// sharded-matmul strategies on device data through the C-ABI (apl.h).
//
// This is what a reference-side caller adds next to layout.hpp (SURVEY §8b
// "Who calls it"): the planner's comm-insertion pass (reference
// planner.cpp:218-352), `plan convert` (plan_main.cpp:179-202) or any C++
// executor walking CommInsertion records. Header-only; link libapl.so.
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "apl.h"
#include "autoplan/layout.hpp"

namespace autoplan {

class RuntimeFailure : public PlanError {
 public:
  RuntimeFailure(int code, const std::string& what) : PlanError(what), code(code) {}
  int code;
};

namespace apl_detail {

inline void check(int rc) {
  if (rc == APL_OK) return;
  const std::string msg = apl_last_error();
  switch (rc) {
    case APL_ERR_SCHEMA: throw SchemaError(msg);
    case APL_ERR_AXIS: throw AxisError(msg);
    case APL_ERR_SHAPE: throw ShapeError(msg);
    case APL_ERR_RANK: throw RankMismatchError(msg);
    case APL_ERR_INFEASIBLE: throw InfeasibleError(msg);
    default: throw RuntimeFailure(rc, msg);
  }
}

inline apl_spec to_c(const ShardingSpec& s) {
  apl_spec out;
  std::memset(&out, 0, sizeof(out));
  out.rank = s.tensor_rank();
  out.mesh_rank = s.mesh_rank;
  for (int d = 0; d < s.tensor_rank(); ++d) {
    const auto& axes = s.dims[static_cast<size_t>(d)].axes;
    out.naxes[d] = static_cast<int32_t>(axes.size());
    for (size_t i = 0; i < axes.size(); ++i) out.axes[d][i] = axes[i];
  }
  return out;
}

inline apl_meta to_c(const TensorMeta& m) {
  apl_meta out;
  std::memset(&out, 0, sizeof(out));
  out.rank = static_cast<int32_t>(m.shape.size());
  out.dtype_bytes = m.dtype_bytes;
  for (size_t i = 0; i < m.shape.size(); ++i) out.shape[i] = m.shape[i];
  return out;
}

inline apl_mesh_desc to_c(const DeviceMesh& m) {
  apl_mesh_desc out;
  std::memset(&out, 0, sizeof(out));
  out.ndim = m.rank();
  for (int i = 0; i < m.rank(); ++i) {
    out.shape[i] = m.shape[static_cast<size_t>(i)];
    out.alpha[i] = m.axis_alpha[static_cast<size_t>(i)];
    out.beta_inv[i] = m.axis_beta_inv[static_cast<size_t>(i)];
  }
  return out;
}

inline std::vector<apl_step> to_c(const std::vector<TransformStep>& steps) {
  std::vector<apl_step> out(steps.size());
  for (size_t i = 0; i < steps.size(); ++i) {
    out[i].kind = static_cast<int32_t>(steps[i].kind);
    out[i].tensor_dim = steps[i].tensor_dim;
    out[i].target_dim = steps[i].target_dim;
    out[i].mesh_axis = steps[i].mesh_axis;
    out[i].result = to_c(steps[i].result);
  }
  return out;
}

}  // namespace apl_detail

// Owns an apl_mesh: Simulated(mesh) puts every mesh device on one GPU;
// Distributed(mesh, rank, nccl_id) is one process per GPU.
class MeshRuntime {
 public:
  static MeshRuntime Simulated(const DeviceMesh& mesh, int cuda_device = 0) {
    MeshRuntime rt;
    const apl_mesh_desc d = apl_detail::to_c(mesh);
    apl_detail::check(apl_mesh_create_local(&d, cuda_device, &rt.handle_));
    return rt;
  }
  static MeshRuntime Distributed(const DeviceMesh& mesh, int rank, const uint8_t* nccl_id,
                                 int cuda_device) {
    MeshRuntime rt;
    const apl_mesh_desc d = apl_detail::to_c(mesh);
    apl_detail::check(apl_mesh_create_nccl(&d, rank, nccl_id, cuda_device, &rt.handle_));
    return rt;
  }
  MeshRuntime(MeshRuntime&& o) noexcept : handle_(o.handle_) { o.handle_ = nullptr; }
  MeshRuntime& operator=(MeshRuntime&& o) noexcept {
    std::swap(handle_, o.handle_);
    return *this;
  }
  MeshRuntime(const MeshRuntime&) = delete;
  ~MeshRuntime() {
    if (handle_) apl_mesh_destroy(handle_);
  }
  apl_mesh* get() const { return handle_; }

 private:
  MeshRuntime() = default;
  apl_mesh* handle_ = nullptr;
};

// Workspace bytes execute() needs for this path.
inline size_t workspace_bytes(MeshRuntime& rt, const TransformPath& path, const TensorMeta& meta,
                              bool fuse_chain) {
  const apl_spec s = apl_detail::to_c(path.source), t = apl_detail::to_c(path.target);
  const apl_meta m = apl_detail::to_c(meta);
  const auto steps = apl_detail::to_c(path.steps);
  size_t bytes = 0;
  apl_detail::check(apl_path_workspace_bytes(rt.get(), &s, &t, steps.data(),
                                             static_cast<int>(steps.size()), &m,
                                             fuse_chain ? APL_FUSE_CHAIN : APL_STEPWISE, &bytes));
  return bytes;
}

// Executes `path` on device shards: `in`/`out` hold one pointer per local
// mesh device (all devices on a simulated mesh, this rank's on a distributed
// one); stream-ordered on `stream` (a cudaStream_t).
inline void execute(MeshRuntime& rt, const TransformPath& path, const TensorMeta& meta,
                    const void* const* in, void* const* out, void* workspace,
                    size_t workspace_bytes, bool fuse_chain, void* stream) {
  const apl_spec s = apl_detail::to_c(path.source), t = apl_detail::to_c(path.target);
  const apl_meta m = apl_detail::to_c(meta);
  const auto steps = apl_detail::to_c(path.steps);
  apl_detail::check(apl_run_path(rt.get(), &s, &t, steps.data(), static_cast<int>(steps.size()),
                                 &m, in, out, workspace, workspace_bytes,
                                 fuse_chain ? APL_FUSE_CHAIN : APL_STEPWISE, stream));
}

}  // namespace autoplan
