// C-ABI (include/apl.h) over the autoplan host API and the device runtime.
// Exceptions never cross: each entry point maps the PlanError hierarchy
// (reference errors.hpp:25-108) and runtime failures onto apl_status codes.
#include "apl.h"

#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "autoplan/layout.hpp"
#include "autoplan/matmul_strategies.hpp"
#include "runtime/runtime.hpp"

using autoplan::CollectiveKind;
using autoplan::DeviceMesh;
using autoplan::ShardingSpec;
using autoplan::TensorMeta;
using autoplan::TransformPath;
using autoplan::TransformStep;

struct apl_path_cache {
  autoplan::PathCache cache;
};
struct apl_mesh {
  apl::Mesh impl;
};
struct apl_conversion {
  apl::Conversion impl;  // holds a pointer to its mesh: destroy before the mesh
};

namespace {

thread_local std::string g_last_error;

struct ArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int guarded(F&& body) {
  try {
    body();
    g_last_error.clear();
    return APL_OK;
  } catch (const autoplan::SchemaError& e) {
    g_last_error = e.what();
    return APL_ERR_SCHEMA;
  } catch (const autoplan::AxisError& e) {
    g_last_error = e.what();
    return APL_ERR_AXIS;
  } catch (const autoplan::ShapeError& e) {
    g_last_error = e.what();
    return APL_ERR_SHAPE;
  } catch (const autoplan::RankMismatchError& e) {
    g_last_error = e.what();
    return APL_ERR_RANK;
  } catch (const autoplan::InfeasibleError& e) {
    g_last_error = e.what();
    return APL_ERR_INFEASIBLE;
  } catch (const autoplan::PlanError& e) {
    g_last_error = e.what();
    return APL_ERR_PLAN;
  } catch (const apl::RuntimeError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const ArgError& e) {
    g_last_error = e.what();
    return APL_ERR_ARG;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return APL_ERR_INTERNAL;
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw ArgError(what);
}

ShardingSpec to_spec(const apl_spec* s) {
  need(s != nullptr, "null spec");
  need(s->rank >= 1 && s->rank <= APL_MAX_DIMS, "spec rank outside [1, APL_MAX_DIMS]");
  need(s->mesh_rank >= 0 && s->mesh_rank <= APL_MAX_MESH, "spec mesh rank outside [0, APL_MAX_MESH]");
  ShardingSpec out;
  out.mesh_rank = s->mesh_rank;
  out.dims.resize(static_cast<size_t>(s->rank));
  for (int d = 0; d < s->rank; ++d) {
    need(s->naxes[d] >= 0 && s->naxes[d] <= APL_MAX_MESH, "axis count out of range");
    for (int i = 0; i < s->naxes[d]; ++i) out.dims[static_cast<size_t>(d)].axes.push_back(s->axes[d][i]);
  }
  return out;
}

void from_spec(const ShardingSpec& s, apl_spec* out) {
  need(s.tensor_rank() <= APL_MAX_DIMS, "tensor rank above APL_MAX_DIMS");
  std::memset(out, 0, sizeof(*out));
  out->rank = s.tensor_rank();
  out->mesh_rank = s.mesh_rank;
  for (int d = 0; d < s.tensor_rank(); ++d) {
    const auto& axes = s.dims[static_cast<size_t>(d)].axes;
    need(axes.size() <= APL_MAX_MESH, "too many axes on one dim");
    out->naxes[d] = static_cast<int32_t>(axes.size());
    for (size_t i = 0; i < axes.size(); ++i) out->axes[d][i] = axes[i];
  }
}

TensorMeta to_meta(const apl_meta* m) {
  need(m != nullptr, "null meta");
  need(m->rank >= 1 && m->rank <= APL_MAX_DIMS, "meta rank outside [1, APL_MAX_DIMS]");
  need(m->dtype_bytes == 1 || m->dtype_bytes == 2 || m->dtype_bytes == 4 || m->dtype_bytes == 8,
       "dtype_bytes must be one of {1,2,4,8}");
  TensorMeta t;
  t.dtype_bytes = m->dtype_bytes;
  for (int i = 0; i < m->rank; ++i) {
    need(m->shape[i] >= 1, "tensor extents must be positive");
    t.shape.push_back(m->shape[i]);
  }
  return t;
}

DeviceMesh to_mesh(const apl_mesh_desc* m) {
  need(m != nullptr, "null mesh");
  need(m->ndim >= 1 && m->ndim <= APL_MAX_MESH, "mesh rank outside [1, APL_MAX_MESH]");
  DeviceMesh mesh = DeviceMesh::uniform(std::vector<int64_t>(m->shape, m->shape + m->ndim));
  for (int i = 0; i < m->ndim; ++i) {
    need(m->shape[i] >= 1, "mesh extents must be positive");
    mesh.axis_alpha[static_cast<size_t>(i)] = m->alpha[i];
    mesh.axis_beta_inv[static_cast<size_t>(i)] = m->beta_inv[i];
  }
  return mesh;
}

void from_step(const TransformStep& s, apl_step* out) {
  out->kind = static_cast<int32_t>(s.kind);
  out->tensor_dim = s.tensor_dim;
  out->target_dim = s.target_dim;
  out->mesh_axis = s.mesh_axis;
  from_spec(s.result, &out->result);
}

TransformStep to_step(const apl_step* s) {
  need(s->kind >= 0 && s->kind <= APL_SHARD_SLICE, "bad step kind");
  TransformStep t;
  t.kind = static_cast<CollectiveKind>(s->kind);
  t.tensor_dim = s->tensor_dim;
  t.target_dim = s->target_dim;
  t.mesh_axis = s->mesh_axis;
  t.result = to_spec(&s->result);
  return t;
}

std::vector<TransformStep> to_steps(const apl_step* steps, int n) {
  need(n >= 0 && (n == 0 || steps != nullptr), "bad step array");
  std::vector<TransformStep> out;
  for (int i = 0; i < n; ++i) out.push_back(to_step(&steps[i]));
  return out;
}

void emit_path(const TransformPath& p, apl_step* steps, int cap, int* nsteps, double* cost) {
  need(nsteps != nullptr, "null nsteps");
  *nsteps = static_cast<int>(p.steps.size());
  if (cost) *cost = p.comm_cost_s;
  need(static_cast<int>(p.steps.size()) <= cap, "step capacity too small");
  for (size_t i = 0; i < p.steps.size(); ++i) from_step(p.steps[i], &steps[i]);
}

autoplan::DimDiffWeights weights_of(const double* w) {
  autoplan::DimDiffWeights out;
  if (w) {
    out.all_gather = w[0];
    out.shard = w[1];
    out.all_to_all = w[2];
    out.step_penalty = w[3];
  }
  return out;
}

}  // namespace

extern "C" {

int apl_version(void) { return 101; }  // 101: apl_layernorm_backward_ex

const char* apl_last_error(void) { return g_last_error.c_str(); }

int apl_mesh_desc_uniform(const int64_t* shape, int ndim, apl_mesh_desc* out) {
  return guarded([&] {
    need(shape && out && ndim >= 1 && ndim <= APL_MAX_MESH, "bad mesh shape");
    std::memset(out, 0, sizeof(*out));
    out->ndim = ndim;
    for (int i = 0; i < ndim; ++i) {
      need(shape[i] >= 1, "mesh extents must be positive");
      out->shape[i] = shape[i];
      out->alpha[i] = 1e-5;
      out->beta_inv[i] = 1e-9;
    }
  });
}

int apl_mesh_to_json(const apl_mesh_desc* mesh, double device_flops_per_s, char* buf,
                     size_t cap, size_t* len) {
  return guarded([&] {
    need(len, "null out");
    DeviceMesh m = to_mesh(mesh);
    m.device_flops_per_s = device_flops_per_s;
    const std::string text = autoplan::mesh_to_json(m).dump();
    *len = text.size();
    if (buf != nullptr) {
      need(cap > text.size(), "buffer too small");
      std::memcpy(buf, text.c_str(), text.size() + 1);
    }
  });
}

int apl_mesh_from_json(const char* text, apl_mesh_desc* out, double* device_flops_per_s) {
  return guarded([&] {
    need(text && out, "null argument");
    nlohmann::json doc;
    try {
      doc = nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
      throw autoplan::SchemaError(std::string("mesh document is not JSON: ") + e.what());
    }
    const DeviceMesh m = autoplan::mesh_from_json(doc);
    need(m.rank() >= 1 && m.rank() <= APL_MAX_MESH, "mesh rank outside [1, APL_MAX_MESH]");
    std::memset(out, 0, sizeof(*out));
    out->ndim = m.rank();
    for (int i = 0; i < m.rank(); ++i) {
      out->shape[i] = m.shape[static_cast<size_t>(i)];
      out->alpha[i] = m.axis_alpha[static_cast<size_t>(i)];
      out->beta_inv[i] = m.axis_beta_inv[static_cast<size_t>(i)];
    }
    if (device_flops_per_s) *device_flops_per_s = m.device_flops_per_s;
  });
}

int apl_parse_mesh_shape(const char* text, int64_t* shape, int cap, int* ndim) {
  return guarded([&] {
    need(text && shape && ndim, "null argument");
    auto v = autoplan::parse_mesh_shape(text);
    *ndim = static_cast<int>(v.size());
    need(static_cast<int>(v.size()) <= cap, "mesh shape capacity too small");
    for (size_t i = 0; i < v.size(); ++i) shape[i] = v[i];
  });
}

int apl_spec_parse(const char* text, int mesh_rank, apl_spec* out) {
  return guarded([&] {
    need(text && out, "null argument");
    from_spec(ShardingSpec::parse(text, mesh_rank), out);
  });
}

int apl_spec_to_string(const apl_spec* spec, char* buf, size_t cap) {
  return guarded([&] {
    const std::string s = to_spec(spec).to_string();
    need(buf && cap > s.size(), "string buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int apl_spec_valid(const apl_spec* spec, const apl_mesh_desc* mesh, const apl_meta* meta,
                   int* valid) {
  return guarded([&] {
    need(valid, "null out");
    *valid = to_spec(spec).valid_for(to_meta(meta), to_mesh(mesh)) ? 1 : 0;
  });
}

int apl_spec_per_device_bytes(const apl_spec* spec, const apl_mesh_desc* mesh,
                              const apl_meta* meta, int64_t* bytes) {
  return guarded([&] {
    need(bytes, "null out");
    *bytes = to_spec(spec).per_device_bytes(to_meta(meta), to_mesh(mesh));
  });
}

int apl_one_step_transforms(const apl_spec* spec, const apl_mesh_desc* mesh,
                            const apl_meta* meta, apl_step* out, int cap, int* count) {
  return guarded([&] {
    need(count, "null count");
    auto r = autoplan::one_step_transforms(to_spec(spec), to_mesh(mesh), to_meta(meta));
    *count = static_cast<int>(r.size());
    need(static_cast<int>(r.size()) <= cap && (r.empty() || out), "step capacity too small");
    for (size_t i = 0; i < r.size(); ++i) from_step(r[i].second, &out[i]);
  });
}

int apl_dim_diff(const int32_t* src_axes, int nsrc, const int32_t* tgt_axes, int ntgt,
                 const double* weights4, double* out) {
  return guarded([&] {
    need(out && nsrc >= 0 && ntgt >= 0, "bad argument");
    autoplan::DimSpec a, b;
    for (int i = 0; i < nsrc; ++i) a.axes.push_back(src_axes[i]);
    for (int i = 0; i < ntgt; ++i) b.axes.push_back(tgt_axes[i]);
    *out = autoplan::dim_diff(a, b, weights_of(weights4));
  });
}

int apl_heuristic_diff(const apl_spec* src, const apl_spec* tgt, const double* weights4,
                       double* out) {
  return guarded([&] {
    need(out, "null out");
    *out = autoplan::heuristic_diff(to_spec(src), to_spec(tgt), weights_of(weights4));
  });
}

int apl_find_transform_path(const apl_mesh_desc* mesh, const apl_spec* src, const apl_spec* tgt,
                            const apl_meta* meta, apl_step* steps, int cap, int* nsteps,
                            double* comm_cost_s) {
  return guarded([&] {
    const DeviceMesh m = to_mesh(mesh);
    const TensorMeta t = to_meta(meta);
    TransformPath p = autoplan::find_transform_path(to_spec(src), to_spec(tgt), m, t);
    autoplan::conversion_cost(p, m, t);
    emit_path(p, steps, cap, nsteps, comm_cost_s);
  });
}

int apl_collective_cost(const apl_mesh_desc* mesh, const int32_t* axes, int naxes, int kind,
                        double bytes, double* out) {
  return guarded([&] {
    need(out && naxes >= 0 && kind >= 0 && kind <= APL_SHARD_SLICE, "bad argument");
    std::vector<int> ax(axes, axes + naxes);
    *out = autoplan::collective_cost(to_mesh(mesh), ax, static_cast<CollectiveKind>(kind), bytes);
  });
}

int apl_path_cache_create(apl_path_cache** out) {
  return guarded([&] {
    need(out, "null out");
    *out = new apl_path_cache();
  });
}

int apl_path_cache_destroy(apl_path_cache* cache) {
  return guarded([&] { delete cache; });
}

int apl_path_cache_get(apl_path_cache* cache, const apl_mesh_desc* mesh, const apl_spec* src,
                       const apl_spec* tgt, const apl_meta* meta, apl_step* steps, int cap,
                       int* nsteps, double* comm_cost_s) {
  return guarded([&] {
    need(cache, "null cache");
    TransformPath p = cache->cache.get(to_spec(src), to_spec(tgt), to_mesh(mesh), to_meta(meta));
    emit_path(p, steps, cap, nsteps, comm_cost_s);
  });
}

int apl_path_cache_stats(const apl_path_cache* cache, size_t* searches, size_t* size) {
  return guarded([&] {
    need(cache, "null cache");
    if (searches) *searches = cache->cache.searches();
    if (size) *size = cache->cache.size();
  });
}

int apl_path_cache_clear(apl_path_cache* cache) {
  return guarded([&] {
    need(cache, "null cache");
    cache->cache.clear();
  });
}

int apl_plan_pieces(const apl_mesh_desc* mesh, const apl_spec* src, const apl_spec* tgt,
                    const apl_meta* meta, int device, int role, apl_piece* out, int cap,
                    int* count) {
  return guarded([&] {
    need(count, "null count");
    const DeviceMesh m = to_mesh(mesh);
    const TensorMeta t = to_meta(meta);
    const ShardingSpec s = to_spec(src), g = to_spec(tgt);
    if (!s.valid_for(t, m)) throw autoplan::ShapeError("source spec invalid for tensor/mesh");
    if (!g.valid_for(t, m)) throw autoplan::ShapeError("target spec invalid for tensor/mesh");
    need(device >= 0 && device < m.num_devices(), "device index out of range");
    auto pieces = role == 0 ? apl::pieces_for_receiver(s, g, m, t, device)
                            : apl::pieces_for_sender(s, g, m, t, device);
    *count = static_cast<int>(pieces.size());
    need(static_cast<int>(pieces.size()) <= cap && (pieces.empty() || out), "piece capacity too small");
    for (size_t i = 0; i < pieces.size(); ++i) {
      apl_piece& o = out[i];
      std::memset(&o, 0, sizeof(o));
      o.sender = static_cast<int32_t>(pieces[i].sender);
      o.receiver = static_cast<int32_t>(pieces[i].receiver);
      for (size_t d = 0; d < pieces[i].ext.size(); ++d) {
        o.src_lo[d] = pieces[i].src_lo[d];
        o.dst_lo[d] = pieces[i].dst_lo[d];
        o.ext[d] = pieces[i].ext[d];
      }
    }
  });
}

int apl_mesh_create_local(const apl_mesh_desc* mesh, int cuda_device, apl_mesh** out) {
  return guarded([&] {
    need(out, "null out");
    DeviceMesh m = to_mesh(mesh);
    need(m.num_devices() <= APL_MAX_LOCAL, "simulated meshes hold at most APL_MAX_LOCAL devices");
    int n = 0;
    apl::check_cuda(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    need(cuda_device >= 0 && cuda_device < n, "cuda device index out of range");
    auto* h = new apl_mesh();
    h->impl.geo = std::move(m);
    h->impl.device = cuda_device;
    *out = h;
  });
}

int apl_nccl_unique_id(uint8_t* out128) {
  return guarded([&] {
    need(out128, "null out");
    static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
    ncclUniqueId id;
    apl::check_nccl(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int apl_mesh_create_nccl(const apl_mesh_desc* mesh, int rank, const uint8_t* nccl_id,
                         int cuda_device, apl_mesh** out) {
  apl_mesh* h = nullptr;
  int rc = guarded([&] {
    need(out && nccl_id, "null argument");
    DeviceMesh m = to_mesh(mesh);
    const int64_t world = m.num_devices();
    need(rank >= 0 && rank < world, "rank out of range");
    apl::check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    h = new apl_mesh();
    apl::Mesh& x = h->impl;
    x.geo = std::move(m);
    x.device = cuda_device;
    x.distributed = true;
    x.rank = rank;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    apl::check_nccl(ncclCommInitRank(&x.world, static_cast<int>(world), id, rank), "ncclCommInitRank");
    // One communicator per non-empty axis subset: color = coordinates off the
    // subset, key = mixed-radix coordinate on it (axis order).
    const int r = x.geo.rank();
    const auto coord = x.geo.coord_of(rank);
    for (uint32_t mask = 1; mask < (1u << r); ++mask) {
      int64_t color = 0, key = 0;
      for (int a = 0; a < r; ++a) {
        const int64_t n = x.geo.shape[static_cast<size_t>(a)];
        if (mask & (1u << a)) key = key * n + coord[static_cast<size_t>(a)];
        else color = color * n + coord[static_cast<size_t>(a)];
      }
      ncclComm_t c = nullptr;
      apl::check_nccl(ncclCommSplit(x.world, static_cast<int>(color), static_cast<int>(key), &c, nullptr),
                      "ncclCommSplit");
      x.sub[mask] = c;
    }
    *out = h;
  });
  if (rc != APL_OK) delete h;
  return rc;
}

int apl_mesh_create_peer(const apl_mesh_desc* mesh, int rank, int cuda_device, apl_mesh** out) {
  return guarded([&] {
    need(out, "null out");
    DeviceMesh m = to_mesh(mesh);
    need(rank >= 0 && rank < m.num_devices(), "rank out of range");
    need(m.num_devices() <= APL_MAX_LOCAL, "peer meshes hold at most APL_MAX_LOCAL ranks");
    apl::check_cuda(cudaSetDevice(cuda_device), "cudaSetDevice");
    auto* h = new apl_mesh();
    h->impl.geo = std::move(m);
    h->impl.device = cuda_device;
    h->impl.distributed = true;
    h->impl.rank = rank;
    *out = h;
  });
}

int apl_peer_alloc(apl_mesh* mesh, size_t bytes, void** ptr, uint8_t* handle64) {
  return guarded([&] {
    need(mesh && ptr && handle64 && bytes > 0, "bad argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "unexpected IPC handle size");
    apl::check_cuda(cudaSetDevice(mesh->impl.device), "cudaSetDevice");
    void* p = nullptr;
    apl::check_cuda(cudaMalloc(&p, bytes), "cudaMalloc(peer buffer)");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      apl::check_cuda(e, "cudaIpcGetMemHandle");
    }
    std::lock_guard<std::mutex> hold(mesh->impl.mu);
    mesh->impl.peer_buffers[p] = true;
    std::memcpy(handle64, &h, sizeof(h));
    *ptr = p;
  });
}

int apl_peer_open(apl_mesh* mesh, const uint8_t* handle64, void** ptr) {
  return guarded([&] {
    need(mesh && ptr && handle64, "bad argument");
    apl::check_cuda(cudaSetDevice(mesh->impl.device), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    void* p = nullptr;
    apl::check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess),
                    "cudaIpcOpenMemHandle");
    std::lock_guard<std::mutex> hold(mesh->impl.mu);
    mesh->impl.peer_buffers[p] = false;
    *ptr = p;
  });
}

int apl_run_pull(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt, const apl_meta* meta,
                 const void* const* peer_in, void* out, void* stream) {
  return guarded([&] {
    need(mesh && peer_in && out, "null argument");
    apl::run_pull(mesh->impl, to_spec(src), to_spec(tgt), to_meta(meta), peer_in, out,
                  static_cast<cudaStream_t>(stream));
  });
}

int apl_run_pull_sync(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                      const apl_meta* meta, const void* const* peer_in, void* out,
                      const apl_peer_sync* sync, void* stream) {
  return guarded([&] {
    need(mesh && peer_in && out && sync, "null argument");
    apl::PeerSyncArgs a{sync->peer_flags, sync->local_flags, sync->counter, sync->epoch,
                        static_cast<uint64_t>(sync->timeout_ms) * 1000000ull};
    apl::run_pull_sync(mesh->impl, to_spec(src), to_spec(tgt), to_meta(meta), peer_in, out, a,
                       static_cast<cudaStream_t>(stream));
  });
}

int apl_run_push_sync(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                      const apl_meta* meta, const void* in, void* const* peer_out,
                      const apl_peer_sync* sync, void* stream) {
  return guarded([&] {
    need(mesh && in && peer_out && sync, "null argument");
    apl::PeerSyncArgs a{sync->peer_flags, sync->local_flags, sync->counter, sync->epoch,
                        static_cast<uint64_t>(sync->timeout_ms) * 1000000ull};
    apl::run_push_sync(mesh->impl, to_spec(src), to_spec(tgt), to_meta(meta), in, peer_out, a,
                       static_cast<cudaStream_t>(stream));
  });
}

int apl_exchange_peers(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                       const apl_meta* meta, int32_t* senders, int* n_senders, int32_t* readers,
                       int* n_readers) {
  return guarded([&] {
    need(mesh && n_senders && n_readers, "null argument");
    need(mesh->impl.distributed, "needs a distributed mesh");
    const autoplan::ShardingSpec s = to_spec(src), t = to_spec(tgt);
    const autoplan::TensorMeta m = to_meta(meta);
    if (!s.valid_for(m, mesh->impl.geo) || !t.valid_for(m, mesh->impl.geo))
      throw apl::RuntimeError(APL_ERR_SHAPE, "spec is not valid for the tensor/mesh");
    auto ex = apl::get_exchange(mesh->impl, s, t, m);
    *n_senders = static_cast<int>(ex->pull_senders.size());
    *n_readers = static_cast<int>(ex->pull_readers.size());
    for (size_t i = 0; senders && i < ex->pull_senders.size(); ++i) senders[i] = ex->pull_senders[i];
    for (size_t i = 0; readers && i < ex->pull_readers.size(); ++i) readers[i] = ex->pull_readers[i];
  });
}

int apl_peer_flags_store(void* const* remote_flags, int n, int slot, uint32_t epoch,
                         void* stream) {
  return guarded([&] {
    need(n >= 0 && n <= 64, "at most 64 flag arrays");
    need(remote_flags || n == 0, "null flag table");
    need(slot >= 0, "bad slot");
    std::vector<uint32_t*> p(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      need(remote_flags[i] != nullptr, "null flag array");
      p[static_cast<size_t>(i)] = static_cast<uint32_t*>(remote_flags[i]);
    }
    apl::check_cuda(apl::launch_flag_store(p.data(), n, slot, epoch,
                                           static_cast<cudaStream_t>(stream)),
                    "flag store launch");
  });
}

int apl_peer_flags_wait(const void* local_flags, const int32_t* slots, int n, uint32_t epoch,
                        uint32_t timeout_ms, void* stream) {
  return guarded([&] {
    need(n >= 0 && n <= 64, "at most 64 flags");
    need(local_flags && (slots || n == 0), "null argument");
    std::vector<int> s(slots, slots + n);
    for (int v : s) need(v >= 0, "bad slot");
    apl::check_cuda(apl::launch_flag_wait(static_cast<const uint32_t*>(local_flags), s.data(), n,
                                          epoch, uint64_t{timeout_ms} * 1000000ull,
                                          static_cast<cudaStream_t>(stream)),
                    "flag wait launch");
  });
}

int apl_peer_gemm_scatter(const void* A, const void* B, void* const* owner_slabs, int owners,
                          int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
                          int b_layout, void* stream) {
  return guarded([&] {
    need(A && B && owner_slabs, "null argument");
    need(owners >= 1 && owners <= 8, "1..8 owners");
    need(b_layout == APL_B_NK || b_layout == APL_B_KN, "unknown B layout");
    need(M > 0 && N > 0 && K > 0 && M <= INT32_MAX && N <= INT32_MAX && K <= INT32_MAX,
         "extents out of range");
    need(M % owners == 0 && (M / owners) % 128 == 0, "M / owners must be a multiple of 128");
    for (int q = 0; q < owners; ++q) need(owner_slabs[q] != nullptr, "null owner slab");
    apl::check_cuda(apl::gemm_bf16_scatter(A, B, owner_slabs, owners, static_cast<int>(M),
                                           static_cast<int>(N), static_cast<int>(K),
                                           static_cast<int>(lda), static_cast<int>(ldb),
                                           b_layout == APL_B_KN, static_cast<cudaStream_t>(stream)),
                    "GEMM scatter launch");
  });
}

int apl_peer_allreduce(void* const* members, int P, size_t count, int dtype, void* stream) {
  return guarded([&] {
    need(members && P >= 1 && P <= 8, "1..8 members");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    for (int r = 0; r < P; ++r) need(members[r] != nullptr, "null member buffer");
    apl::check_cuda(apl::launch_peer_allreduce(members, P, static_cast<int64_t>(count), dtype,
                                               static_cast<cudaStream_t>(stream)),
                    "peer all-reduce launch");
  });
}

int apl_peer_reduce_gather(const float* staging, int P, int64_t slab_elems, void* const* outs,
                           int nout, int out_dtype, void* stream) {
  return guarded([&] {
    need(staging && outs, "null argument");
    need(P >= 1 && nout >= 1 && nout <= 8, "bad group size");
    need(slab_elems > 0 && slab_elems % 4 == 0, "slab must hold a multiple of 4 elements");
    need(out_dtype == APL_F32 || out_dtype == APL_BF16, "output dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_reduce_gather(staging, P, slab_elems, outs, nout,
                                              out_dtype == APL_F32,
                                              static_cast<cudaStream_t>(stream)),
                    "reduce-gather launch");
  });
}

int apl_mesh_destroy(apl_mesh* mesh) {
  return guarded([&] { delete mesh; });
}

int apl_mesh_health(apl_mesh* mesh, int* state) {
  return guarded([&] {
    need(mesh && state, "null argument");
    apl::Mesh& m = mesh->impl;
    *state = 0;
    if (m.aborted) {
      *state = static_cast<int>(ncclInvalidUsage);
      return;
    }
    auto poll = [&](ncclComm_t c) {
      if (c == nullptr || (*state != 0 && *state != static_cast<int>(ncclInProgress))) return;
      ncclResult_t r = ncclSuccess;
      apl::check_nccl(ncclCommGetAsyncError(c, &r), "ncclCommGetAsyncError");
      if (r != ncclSuccess) *state = static_cast<int>(r);
    };
    poll(m.world);
    for (auto& [mask, c] : m.sub) poll(c);
  });
}

int apl_mesh_abort(apl_mesh* mesh) {
  return guarded([&] {
    need(mesh, "null mesh");
    apl::Mesh& m = mesh->impl;
    if (m.aborted) return;
    m.aborted = true;
    for (auto& [mask, c] : m.sub)
      if (c != nullptr) ncclCommAbort(c);
    if (m.world != nullptr) ncclCommAbort(m.world);
  });
}

int apl_mesh_info(const apl_mesh* mesh, int* num_devices, int* first_local, int* num_local,
                  int* is_distributed) {
  return guarded([&] {
    need(mesh, "null mesh");
    const apl::Mesh& m = mesh->impl;
    if (num_devices) *num_devices = static_cast<int>(m.geo.num_devices());
    if (first_local) *first_local = m.distributed ? m.rank : 0;
    if (num_local) *num_local = m.num_local();
    if (is_distributed) *is_distributed = m.distributed ? 1 : 0;
  });
}

int apl_path_workspace_bytes(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                             const apl_step* steps, int nsteps, const apl_meta* meta,
                             unsigned flags, size_t* bytes) {
  return guarded([&] {
    need(mesh && bytes, "null argument");
    const ShardingSpec s = to_spec(src), g = to_spec(tgt);
    const TensorMeta t = to_meta(meta);
    if (!s.valid_for(t, mesh->impl.geo) || !g.valid_for(t, mesh->impl.geo))
      throw autoplan::ShapeError("spec is not valid for the tensor/mesh");
    *bytes = apl::path_workspace(mesh->impl, s, g, to_steps(steps, nsteps), t,
                                 (flags & APL_FUSE_CHAIN) != 0);
  });
}

int apl_run_step(apl_mesh* mesh, const apl_spec* src, const apl_step* step, const apl_meta* meta,
                 const void* const* in, void* const* out, void* ws, size_t ws_bytes,
                 void* stream) {
  return guarded([&] {
    need(mesh && step && in && out, "null argument");
    const TransformStep s = to_step(step);
    apl::run_path(mesh->impl, to_spec(src), s.result, {s}, to_meta(meta), in, out, ws, ws_bytes,
                  false, static_cast<cudaStream_t>(stream));
  });
}

int apl_run_path(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt, const apl_step* steps,
                 int nsteps, const apl_meta* meta, const void* const* in, void* const* out,
                 void* ws, size_t ws_bytes, unsigned flags, void* stream) {
  return guarded([&] {
    need(mesh && in && out, "null argument");
    apl::run_path(mesh->impl, to_spec(src), to_spec(tgt), to_steps(steps, nsteps), to_meta(meta),
                  in, out, ws, ws_bytes, (flags & APL_FUSE_CHAIN) != 0,
                  static_cast<cudaStream_t>(stream));
  });
}

int apl_exchange_traffic(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                         const apl_meta* meta, int64_t* hbm_read, int64_t* hbm_write,
                         int64_t* wire_in) {
  return guarded([&] {
    need(mesh, "null mesh");
    const ShardingSpec s = to_spec(src), g = to_spec(tgt);
    const TensorMeta t = to_meta(meta);
    if (!s.valid_for(t, mesh->impl.geo) || !g.valid_for(t, mesh->impl.geo))
      throw autoplan::ShapeError("spec is not valid for the tensor/mesh");
    auto ex = apl::get_exchange(mesh->impl, s, g, t);
    int64_t r = 0, w = 0;
    for (const auto* list : {&ex->host_copies, &ex->host_pre, &ex->host_post})
      for (const apl::CopyDesc& c : *list) {
        r += c.bytes();
        w += c.bytes() * c.ndst;
      }
    if (hbm_read) *hbm_read = r;
    if (hbm_write) *hbm_write = w;
    if (wire_in) *wire_in = ex->wire_bytes_in;
  });
}

int apl_conversion_create(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                          const apl_step* steps, int nsteps, const apl_meta* meta,
                          unsigned flags, apl_conversion** out) {
  return guarded([&] {
    need(mesh && out, "null argument");
    auto* c = new apl_conversion();
    try {
      c->impl = apl::prepare_conversion(mesh->impl, to_spec(src), to_spec(tgt),
                                        to_steps(steps, nsteps), to_meta(meta),
                                        (flags & APL_FUSE_CHAIN) != 0);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int apl_conversion_workspace(const apl_conversion* conv, size_t* bytes) {
  return guarded([&] {
    need(conv && bytes, "null argument");
    *bytes = apl::conversion_workspace(conv->impl);
  });
}

int apl_conversion_run(apl_conversion* conv, const void* const* in, void* const* out, void* ws,
                       size_t ws_bytes, void* stream) {
  return guarded([&] {
    need(conv && in && out, "null argument");
    apl::run_conversion(conv->impl, in, out, ws, ws_bytes, static_cast<cudaStream_t>(stream));
  });
}

int apl_conversion_destroy(apl_conversion* conv) {
  return guarded([&] { delete conv; });
}

int apl_exchange_engine(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                        const apl_meta* meta, int* engine) {
  return guarded([&] {
    need(mesh && engine, "null argument");
    const ShardingSpec s = to_spec(src), g = to_spec(tgt);
    const TensorMeta t = to_meta(meta);
    if (!s.valid_for(t, mesh->impl.geo) || !g.valid_for(t, mesh->impl.geo))
      throw autoplan::ShapeError("spec is not valid for the tensor/mesh");
    auto ex = apl::get_exchange(mesh->impl, s, g, t);
    const auto& host = mesh->impl.distributed ? ex->host_pre : ex->host_copies;
    const int vec = apl::natural_vec(host);
    *engine = apl::tile_eligible(host, vec) ? 2 : apl::bulk_eligible(host, vec) ? 1 : 0;
  });
}

namespace {

std::string copies_json(const std::vector<apl::CopyDesc>& v) {
  std::string j = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    const apl::CopyDesc& c = v[i];
    if (i) j += ",";
    j += "{\"src_buf\":" + std::to_string(c.src_buf) + ",\"dst_buf\":" + std::to_string(c.dst_buf) +
         ",\"src_off\":" + std::to_string(c.src_off) + ",\"dst_off\":" + std::to_string(c.dst_off) +
         ",\"run_bytes\":" + std::to_string(c.run_bytes) + ",\"ext\":[";
    for (int d = 0; d < c.nouter; ++d) j += (d ? "," : "") + std::to_string(c.ext[d]);
    j += "],\"src_stride\":[";
    for (int d = 0; d < c.nouter; ++d) j += (d ? "," : "") + std::to_string(c.src_stride[d]);
    j += "],\"dst_stride\":[";
    for (int d = 0; d < c.nouter; ++d) j += (d ? "," : "") + std::to_string(c.dst_stride[d]);
    j += "],\"ksplit\":" + std::to_string(c.ksplit) +
         ",\"split_src_step\":" + std::to_string(c.split_src_step) + ",\"split_dst\":[";
    for (int d = 0; d < c.ksplit && c.ksplit > 1; ++d)
      j += (d ? "," : "") + std::to_string(c.split_dst[d]);
    j += "],\"split_dst_off\":[";
    for (int d = 0; d < c.ksplit && c.ksplit > 1; ++d)
      j += (d ? "," : "") + std::to_string(c.split_dst_off[d]);
    j += "]}";
  }
  return j + "]";
}

std::string xfers_json(const std::vector<apl::Exchange::Xfer>& v) {
  std::string j = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) j += ",";
    j += "[" + std::to_string(v[i].peer) + "," + (v[i].direct ? "1" : "0") + "," +
         std::to_string(v[i].offset) + "," + std::to_string(v[i].bytes) + "]";
  }
  return j + "]";
}

// The distributed executor's schedule of one hop for this rank.
std::string exchange_json(const apl::Exchange& ex) {
  std::string j = "{\"pre\":" + copies_json(ex.host_pre) + ",\"post\":" + copies_json(ex.host_post) +
                  ",\"sends\":" + xfers_json(ex.sends) + ",\"recvs\":" + xfers_json(ex.recvs) +
                  ",\"send_staging\":" + std::to_string(ex.send_staging) +
                  ",\"recv_staging\":" + std::to_string(ex.recv_staging) +
                  ",\"workspace\":" + std::to_string(apl::exchange_workspace(ex)) +
                  ",\"in_bytes\":" + std::to_string(ex.in_bytes) +
                  ",\"out_bytes\":" + std::to_string(ex.out_bytes);
  if (ex.ag_axis >= 0)
    j += ",\"allgather\":{\"axis\":" + std::to_string(ex.ag_axis) +
         ",\"direct\":" + (ex.ag_direct ? "1" : "0") + "}";
  if (ex.a2a_axis >= 0)
    j += ",\"alltoall\":{\"axis\":" + std::to_string(ex.a2a_axis) +
         ",\"chunk\":" + std::to_string(ex.a2a_chunk) +
         ",\"direct_send\":" + (ex.a2a_direct_send ? "1" : "0") +
         ",\"direct_recv\":" + (ex.a2a_direct_recv ? "1" : "0") + "}";
  return j + "}";
}

void emit(const std::string& j, char* out, size_t cap, size_t* len) {
  *len = j.size() + 1;
  need(out != nullptr && cap >= j.size() + 1, "output buffer too small");
  std::memcpy(out, j.c_str(), j.size() + 1);
}

}  // namespace

int apl_exchange_schedule_json(const apl_mesh_desc* mesh, int rank, const apl_spec* src,
                               const apl_spec* tgt, const apl_meta* meta, char* out, size_t cap,
                               size_t* len) {
  return guarded([&] {
    need(len, "null len");
    apl::Mesh dry;  // no communicators: schedule compilation is host-only
    dry.geo = to_mesh(mesh);
    dry.distributed = true;
    need(rank >= 0 && rank < dry.geo.num_devices(), "rank out of range");
    dry.rank = rank;
    const ShardingSpec s = to_spec(src), g = to_spec(tgt);
    const TensorMeta t = to_meta(meta);
    if (!s.valid_for(t, dry.geo) || !g.valid_for(t, dry.geo))
      throw autoplan::ShapeError("spec is not valid for the tensor/mesh");
    emit(exchange_json(*apl::get_exchange(dry, s, g, t)), out, cap, len);
  });
}

int apl_conversion_schedule_json(const apl_mesh_desc* mesh, int rank, const apl_spec* src,
                                 const apl_spec* tgt, const apl_step* steps, int nsteps,
                                 const apl_meta* meta, unsigned flags, char* out, size_t cap,
                                 size_t* len) {
  return guarded([&] {
    need(len, "null len");
    need(nsteps >= 0 && (steps || nsteps == 0), "bad steps");
    apl::Mesh dry;  // host-only compilation of a distributed rank's conversion
    dry.geo = to_mesh(mesh);
    dry.distributed = true;
    need(rank >= 0 && rank < dry.geo.num_devices(), "rank out of range");
    dry.rank = rank;
    std::vector<autoplan::TransformStep> st;
    for (int i = 0; i < nsteps; ++i) st.push_back(to_step(&steps[i]));
    apl::Conversion cv = apl::prepare_conversion(dry, to_spec(src), to_spec(tgt), st,
                                                 to_meta(meta), (flags & APL_FUSE_CHAIN) != 0);
    std::string j = "{\"hops\":[";
    for (size_t i = 0; i < cv.hops.size(); ++i) j += (i ? "," : "") + exchange_json(*cv.hops[i]);
    j += "],\"inter_bytes\":" + std::to_string(cv.inter_bytes) +
         ",\"staging\":" + std::to_string(cv.staging) + "}";
    emit(j, out, cap, len);
  });
}
int apl_all_reduce(apl_mesh* mesh, const int32_t* axes, int naxes, void* const* bufs,
                   size_t count, int dtype, void* stream) {
  return guarded([&] {
    need(mesh && bufs && (naxes == 0 || axes), "null argument");
    need(dtype >= APL_F32 && dtype <= APL_F16, "bad dtype");
    apl::all_reduce(mesh->impl, std::vector<int>(axes, axes + naxes), bufs, count, dtype,
                    static_cast<cudaStream_t>(stream));
  });
}

int apl_matmul_strategies(const apl_mesh_desc* mesh, const apl_meta* a_meta,
                          const apl_meta* b_meta, int batched, double device_flops_per_s,
                          apl_strategy_info* out, int cap, int* count) {
  return guarded([&] {
    need(count, "null count");
    DeviceMesh m = to_mesh(mesh);
    m.device_flops_per_s = device_flops_per_s;
    const TensorMeta a = to_meta(a_meta), b = to_meta(b_meta);
    need(batched ? (a.rank() == 3 && b.rank() == 3) : (a.rank() >= 2 && b.rank() == 2),
         "matmul wants A[..m.., k] . B[k, n] (or rank-3 batched operands)");
    const auto all = autoplan::matmul_strategies(a, b, m, batched != 0);
    *count = static_cast<int>(all.size());
    need(static_cast<int>(all.size()) <= cap && (all.empty() || out), "capacity too small");
    for (size_t i = 0; i < all.size(); ++i) {
      const autoplan::OpStrategy& s = all[i];
      apl_strategy_info& o = out[i];
      std::memset(&o, 0, sizeof(o));
      need(s.name.size() < sizeof(o.name), "strategy name too long");
      std::memcpy(o.name, s.name.c_str(), s.name.size() + 1);
      from_spec(s.input_specs[0], &o.strategy.a);
      from_spec(s.input_specs[1], &o.strategy.b);
      from_spec(s.output_spec, &o.strategy.c);
      o.strategy.partial_sum = s.partial_sum ? 1 : 0;
      o.strategy.nreduce = static_cast<int32_t>(s.reduce_axes.size());
      for (size_t j = 0; j < s.reduce_axes.size(); ++j) o.strategy.reduce_axes[j] = s.reduce_axes[j];
      o.compute_time_s = s.compute_time_s;
      o.comm_time_s = s.comm_time_s;
      o.bwd_compute_time_s = s.bwd_compute_time_s;
      o.bwd_comm_time_s = s.bwd_comm_time_s;
      o.comm_buffer_bytes = s.comm_buffer_bytes;
      o.memory_bytes = s.memory_bytes;
    }
  });
}

int apl_gemm_force_plan(int pair, int bn, int streamk) {
  return guarded([&] {
    need(pair >= -1 && pair <= 1 && (bn == -1 || bn == 128 || bn == 256) && streamk >= -1 &&
             streamk <= 4,
         "pair in {-1, 0, 1}, bn in {-1, 128, 256}, streamk in {-1, 0, 1} or an aligned "
         "split-K factor 2..4");
    apl::gemm_force_plan(pair, bn, streamk);
  });
}

int apl_gemm_trace(void* buf, size_t bytes) {
  return guarded([&] {
    need(buf == nullptr || bytes >= 16 * sizeof(uint64_t), "trace buffer smaller than one CTA's slots");
    apl::gemm_trace(buf, bytes);
  });
}

int apl_gemm_bf16(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                  int64_t lda, int64_t ldb, int64_t ldc, int b_layout, int out_dtype,
                  int epilogue, void* stream) {
  return guarded([&] {
    need(A && B && C, "null operand");
    need(M >= 0 && N >= 0 && K >= 0 && M <= INT32_MAX && N <= INT32_MAX && K <= INT32_MAX,
         "extents out of range");
    need(b_layout == APL_B_NK || b_layout == APL_B_KN, "unknown B layout");
    const bool kn = b_layout == APL_B_KN;
    need(lda >= K && ldb >= (kn ? N : K) && ldc >= N, "leading dimensions too small");
    need(out_dtype == APL_F32 || out_dtype == APL_BF16, "output dtype must be f32 or bf16");
    need(epilogue == APL_EPI_NONE || epilogue == APL_EPI_GELU, "unknown epilogue");
    apl::check_cuda(apl::gemm_bf16(A, B, C, static_cast<int>(M), static_cast<int>(N),
                                   static_cast<int>(K), static_cast<int>(lda),
                                   static_cast<int>(ldb), static_cast<int>(ldc), kn,
                                   out_dtype == APL_F32, epilogue == APL_EPI_GELU,
                                   static_cast<cudaStream_t>(stream)),
                    "apl_gemm_bf16");
  });
}

int apl_gemm_bf16_grouped(const void* const* A, const void* const* B, void* const* C,
                          int groups, int reduce, int64_t M, int64_t N, int64_t K, int64_t lda,
                          int64_t ldb, int64_t ldc, int b_layout, int out_dtype, int epilogue,
                          const void* const* aux, void* stream) {
  return guarded([&] {
    need(A && B && C, "null operand table");
    need(groups >= 1 && reduce >= 1 && reduce <= 8, "groups >= 1, 1 <= reduce <= 8");
    need(M > 0 && N > 0 && K > 0 && M <= INT32_MAX && N <= INT32_MAX && K <= INT32_MAX,
         "extents out of range");
    need(b_layout == APL_B_NK || b_layout == APL_B_KN, "unknown B layout");
    const bool kn = b_layout == APL_B_KN;
    need(lda >= K && ldb >= (kn ? N : K) && ldc >= N, "leading dimensions too small");
    need(out_dtype == APL_F32 || out_dtype == APL_BF16, "output dtype must be f32 or bf16");
    need(epilogue >= APL_EPI_NONE && epilogue <= APL_EPI_GELU_SAVE, "unknown epilogue");
    need(epilogue < APL_EPI_DGELU || aux != nullptr, "epilogue needs aux buffers");
    for (int i = 0; i < groups * reduce; ++i) need(A[i] && B[i], "null operand");
    for (int i = 0; i < groups; ++i) need(C[i] != nullptr, "null output");
    apl::check_cuda(apl::gemm_bf16_grouped(A, B, C, groups, reduce, 1, static_cast<int>(M),
                                           static_cast<int>(N), static_cast<int>(K),
                                           static_cast<int>(lda), static_cast<int>(ldb),
                                           static_cast<int>(ldc), kn, out_dtype == APL_F32,
                                           epilogue, false, aux, static_cast<int>(ldc),
                                           static_cast<cudaStream_t>(stream)),
                    "grouped GEMM launch");
  });
}

int apl_sharded_matmul_ex(apl_mesh* mesh, const apl_matmul_strategy* strategy,
                          const apl_meta* a_meta, const apl_meta* b_meta, const void* const* A,
                          const void* const* B, void* const* C, int b_layout, int out_dtype,
                          int epilogue, void* const* aux, void* stream) {
  return guarded([&] {
    need(mesh && strategy && A && B && C, "null argument");
    need(b_layout == APL_B_NK || b_layout == APL_B_KN, "unknown B layout");
    need(out_dtype == APL_F32 || out_dtype == APL_BF16, "output dtype must be f32 or bf16");
    need(epilogue == APL_EPI_NONE || epilogue == APL_EPI_GELU || epilogue == APL_EPI_GELU_SAVE,
         "unknown epilogue");
    need(epilogue != APL_EPI_GELU_SAVE || (aux != nullptr && out_dtype == APL_BF16),
         "APL_EPI_GELU_SAVE needs aux buffers and bf16 output");
    need(strategy->nreduce >= 0 && strategy->nreduce <= APL_MAX_MESH, "bad reduce axis count");
    apl::MatmulStrategy s;
    s.a = to_spec(&strategy->a);
    s.b = to_spec(&strategy->b);
    s.c = to_spec(&strategy->c);
    s.partial_sum = strategy->partial_sum != 0;
    for (int i = 0; i < strategy->nreduce; ++i) s.reduce_axes.push_back(strategy->reduce_axes[i]);
    need(s.partial_sum == !s.reduce_axes.empty(), "partial_sum iff reduce axes are given");
    apl::sharded_matmul(mesh->impl, s, to_meta(a_meta), to_meta(b_meta), A, B, C,
                        b_layout == APL_B_KN, out_dtype, epilogue,
                        static_cast<cudaStream_t>(stream), aux);
  });
}

int apl_sharded_matmul(apl_mesh* mesh, const apl_matmul_strategy* strategy,
                       const apl_meta* a_meta, const apl_meta* b_meta, const void* const* A,
                       const void* const* B, void* const* C, int b_layout, int out_dtype,
                       int epilogue, void* stream) {
  if (epilogue == APL_EPI_GELU_SAVE) {
    g_last_error = "APL_EPI_GELU_SAVE needs apl_sharded_matmul_ex (aux buffers)";
    return APL_ERR_ARG;
  }
  return apl_sharded_matmul_ex(mesh, strategy, a_meta, b_meta, A, B, C, b_layout, out_dtype,
                               epilogue, nullptr, stream);
}

int apl_gelu_inplace(void* buf, size_t count, int dtype, void* stream) {
  return guarded([&] {
    need(buf || count == 0, "null buffer");
    need(dtype >= APL_F32 && dtype <= APL_F16, "bad dtype");
    apl::check_cuda(apl::launch_gelu_inplace(buf, count, dtype, static_cast<cudaStream_t>(stream)),
                    "gelu launch");
  });
}

int apl_gelu(const void* x, void* y, size_t count, int dtype, void* stream) {
  return guarded([&] {
    need((x && y) || count == 0, "null buffer");
    need(dtype >= APL_F32 && dtype <= APL_F16, "bad dtype");
    apl::check_cuda(apl::launch_gelu(x, y, count, dtype, static_cast<cudaStream_t>(stream)),
                    "gelu launch");
  });
}

int apl_gelu_backward(const void* dy, const void* x, void* dx, size_t count, int dtype,
                      void* stream) {
  return guarded([&] {
    need((dy && x && dx) || count == 0, "null buffer");
    need(dtype >= APL_F32 && dtype <= APL_F16, "bad dtype");
    apl::check_cuda(
        apl::launch_gelu_backward(dy, x, dx, count, dtype, static_cast<cudaStream_t>(stream)),
        "gelu backward launch");
  });
}

int apl_embedding_lookup(const int64_t* ids, int64_t n, const void* table, int64_t vocab,
                         int64_t width, int elem_bytes, void* out, void* stream) {
  return guarded([&] {
    need(n >= 0 && width >= 0 && vocab >= 0, "negative extent");
    need((ids && table && out) || n == 0 || width == 0, "null buffer");
    need(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
         "elem_bytes must be 1, 2, 4 or 8");
    apl::check_cuda(apl::launch_embedding(ids, n, table, vocab, width, elem_bytes, out,
                                          static_cast<cudaStream_t>(stream)),
                    "embedding launch");
  });
}

int apl_embedding_lookup_blocks(const int64_t* ids, int64_t n, const void* const* blocks,
                                int vocab_blocks, int hidden_blocks, int64_t vocab, int64_t width,
                                int64_t col_begin, int64_t cols, int elem_bytes, void* out,
                                void* stream) {
  return guarded([&] {
    need(n >= 0 && vocab >= 0 && width > 0 && cols >= 0, "bad extents");
    need(vocab_blocks >= 1 && hidden_blocks >= 1 && vocab_blocks * hidden_blocks <= 64,
         "1..64 table blocks");
    need(vocab % vocab_blocks == 0 && width % hidden_blocks == 0,
         "blocks must split the table evenly");
    need(col_begin >= 0 && col_begin + cols <= width, "column slice outside the table");
    need((ids && blocks && out) || n == 0 || cols == 0, "null buffer");
    for (int i = 0; blocks && i < vocab_blocks * hidden_blocks; ++i)
      need(blocks[i] != nullptr, "null table block");
    need(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
         "elem_bytes must be 1, 2, 4 or 8");
    apl::check_cuda(apl::launch_embedding_blocks(ids, n, blocks, vocab_blocks, hidden_blocks,
                                                 vocab, width, col_begin, cols, elem_bytes, out,
                                                 static_cast<cudaStream_t>(stream)),
                    "embedding launch");
  });
}

int apl_layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows,
                  int64_t width, float eps, int dtype, void* stream) {
  return guarded([&] {
    need(rows >= 0 && width > 0, "bad extents");
    need((x && y) || rows == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_layernorm(x, gamma, beta, y, rows, width, eps, dtype,
                                          static_cast<cudaStream_t>(stream)),
                    "layernorm launch");
  });
}

int apl_softmax_ex(const void* x, void* y, int64_t rows, int64_t width, float alpha,
                   const void* mask, float fill, int dtype, void* stream) {
  return guarded([&] {
    need(rows >= 0 && width > 0, "bad extents");
    need((x && y) || rows == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_softmax(x, y, rows, width, alpha, mask, fill, dtype,
                                        static_cast<cudaStream_t>(stream)),
                    "softmax launch");
  });
}

int apl_softmax(const void* x, void* y, int64_t rows, int64_t width, int dtype, void* stream) {
  return apl_softmax_ex(x, y, rows, width, 1.f, nullptr, 0.f, dtype, stream);
}

int apl_transpose(const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
                  int elem_bytes, void* stream) {
  return guarded([&] {
    need(batch >= 0 && rows >= 0 && cols >= 0 && rows <= INT32_MAX && cols <= INT32_MAX,
         "extents out of range");
    need((x && y) || batch * rows * cols == 0, "null buffer");
    need(x != y, "transpose is out of place");
    need(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
         "elem_bytes must be 1, 2, 4 or 8");
    apl::check_cuda(apl::launch_transpose(x, y, batch, rows, cols, elem_bytes,
                                          static_cast<cudaStream_t>(stream)),
                    "transpose launch");
  });
}

int apl_permute(const void* x, void* y, int rank, const int64_t* shape, const int64_t* perm,
                int elem_bytes, void* stream) {
  return guarded([&] {
    need(rank >= 1 && rank <= 8 && shape != nullptr && perm != nullptr, "rank must be 1..8");
    bool seen[8] = {};
    int64_t numel = 1;
    for (int d = 0; d < rank; ++d) {
      need(perm[d] >= 0 && perm[d] < rank && !seen[perm[d]], "perm is not a permutation");
      seen[perm[d]] = true;
      need(shape[d] >= 0, "negative extent");
      numel *= shape[d];
    }
    need((x && y) || numel == 0, "null buffer");
    need(x != y || numel == 0, "permute is out of place");
    need(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
         "elem_bytes must be 1, 2, 4 or 8");
    apl::check_cuda(apl::launch_permute(x, y, rank, shape, perm, elem_bytes,
                                        static_cast<cudaStream_t>(stream)),
                    "permute launch");
  });
}

int apl_softmax_axis(const void* x, void* y, int64_t outer, int64_t len, int64_t inner,
                     int dtype, void* stream) {
  return guarded([&] {
    need(outer >= 0 && len > 0 && inner > 0, "bad extents");
    need((x && y) || outer == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    if (inner == 1) {
      apl::check_cuda(apl::launch_softmax(x, y, outer, len, 1.f, nullptr, 0.f, dtype,
                                          static_cast<cudaStream_t>(stream)),
                      "softmax launch");
      return;
    }
    apl::check_cuda(apl::launch_softmax_axis(x, y, outer, len, inner, dtype,
                                             static_cast<cudaStream_t>(stream)),
                    "softmax (axis) launch");
  });
}

int apl_softmax_axis_backward(const void* y, const void* dy, void* dx, int64_t outer,
                              int64_t len, int64_t inner, float alpha, int dtype, void* stream) {
  return guarded([&] {
    need(outer >= 0 && len > 0 && inner > 0, "bad extents");
    need((y && dy && dx) || outer == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    if (inner == 1) {
      apl::check_cuda(apl::launch_softmax_backward(y, dy, dx, outer, len, alpha, dtype,
                                                   static_cast<cudaStream_t>(stream)),
                      "softmax backward launch");
      return;
    }
    apl::check_cuda(apl::launch_softmax_axis_backward(y, dy, dx, outer, len, inner, alpha, dtype,
                                                      static_cast<cudaStream_t>(stream)),
                    "softmax (axis) backward launch");
  });
}

int apl_scale(const void* x, void* y, size_t count, float alpha, int dtype, void* stream) {
  return guarded([&] {
    need((x && y) || count == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(
        apl::launch_scale(x, y, count, alpha, dtype, static_cast<cudaStream_t>(stream)),
        "scale launch");
  });
}

int apl_add(const void* a, const void* b, int b_mask, void* y, size_t count, float alpha,
            int dtype, void* stream) {
  return guarded([&] {
    need((a && b && y) || count == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_add(a, b, b_mask != 0, y, count, alpha, dtype,
                                    static_cast<cudaStream_t>(stream)),
                    "add launch");
  });
}

int apl_layernorm_backward(const void* x, const void* gamma, const void* dy, void* dx,
                           float* dgamma, float* dbeta, void* stats, int64_t rows, int64_t width,
                           float eps, int dtype, void* stream) {
  return guarded([&] {
    need(rows >= 0 && width > 0, "bad extents");
    need((x && dy && dx) || rows == 0, "null buffer");
    need((dgamma == nullptr && dbeta == nullptr) || stats != nullptr || rows == 0,
         "parameter gradients need the per-row stats scratch");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_layernorm_backward(x, gamma, dy, dx, dgamma, dbeta, stats, rows,
                                                   width, eps, dtype,
                                                   static_cast<cudaStream_t>(stream)),
                    "layernorm backward launch");
  });
}

int apl_layernorm_backward_ex(const void* x, const void* gamma, const void* dy, void* dx,
                              float* dgamma, float* dbeta, void* stats, size_t stats_bytes,
                              int64_t rows, int64_t width, float eps, int dtype, void* stream) {
  if ((dgamma != nullptr || dbeta != nullptr) && rows > 0 && width > 0 &&
      stats_bytes < apl::layernorm_backward_scratch_bytes(rows, width)) {
    g_last_error = "stats scratch smaller than apl_layernorm_backward_scratch()";
    return APL_ERR_ARG;
  }
  return apl_layernorm_backward(x, gamma, dy, dx, dgamma, dbeta, stats, rows, width, eps, dtype,
                                stream);
}

int apl_layernorm_backward_scratch(int64_t rows, int64_t width, size_t* bytes) {
  return guarded([&] {
    need(rows >= 0 && width > 0 && bytes != nullptr, "bad arguments");
    *bytes = apl::layernorm_backward_scratch_bytes(rows, width);
  });
}

int apl_softmax_backward(const void* y, const void* dy, void* dx, int64_t rows, int64_t width,
                         float alpha, int dtype, void* stream) {
  return guarded([&] {
    need(rows >= 0 && width > 0, "bad extents");
    need((y && dy && dx) || rows == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_softmax_backward(y, dy, dx, rows, width, alpha, dtype,
                                                 static_cast<cudaStream_t>(stream)),
                    "softmax backward launch");
  });
}

int apl_embedding_backward(const int64_t* ids, int64_t n, const void* dy, float* dtable,
                           int64_t vocab, int64_t width, int dtype, void* stream) {
  return guarded([&] {
    need(n >= 0 && vocab >= 0 && width >= 0, "negative extent");
    need((ids && dy && dtable) || n == 0 || width == 0, "null buffer");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_embedding_backward(ids, n, dy, dtable, vocab, width, dtype,
                                                   static_cast<cudaStream_t>(stream)),
                    "embedding backward launch");
  });
}

int apl_embedding_backward_block(const int64_t* const* ids, const void* const* dy, int nsrc,
                                 int64_t n, int64_t dy_width, float* dblock, int64_t v0,
                                 int64_t rows, int64_t c0, int64_t cols, int dtype, void* stream) {
  return guarded([&] {
    need(nsrc >= 0 && nsrc <= 64, "0..64 sources");
    need(n >= 0 && rows >= 0 && cols >= 0 && c0 >= 0 && c0 + cols <= dy_width, "bad extents");
    need((ids && dy && dblock) || nsrc == 0 || n == 0, "null buffer");
    for (int i = 0; ids && dy && i < nsrc; ++i) need(ids[i] && dy[i], "null source");
    need(dtype == APL_F32 || dtype == APL_BF16, "dtype must be f32 or bf16");
    apl::check_cuda(apl::launch_embedding_backward_block(ids, dy, nsrc, n, dy_width, dblock, v0,
                                                         rows, c0, cols, dtype,
                                                         static_cast<cudaStream_t>(stream)),
                    "embedding backward launch");
  });
}

int apl_gemm_bf16_grouped_ex(const void* const* A, const void* const* B, void* const* C,
                             int groups, int64_t M, int64_t N, int64_t K, int64_t lda,
                             int64_t ldb, int64_t ldc, int a_layout, int b_layout, int out_dtype,
                             void* stream) {
  return guarded([&] {
    need(A && B && C && groups >= 1, "null operand table");
    need(M > 0 && N > 0 && K > 0 && M <= INT32_MAX && N <= INT32_MAX && K <= INT32_MAX,
         "extents out of range");
    need(a_layout == APL_A_MK || a_layout == APL_A_KM, "unknown A layout");
    need(b_layout == APL_B_NK || b_layout == APL_B_KN, "unknown B layout");
    const bool kn = b_layout == APL_B_KN, km = a_layout == APL_A_KM;
    need(lda >= (km ? M : K) && ldb >= (kn ? N : K) && ldc >= N, "leading dimensions too small");
    need(out_dtype == APL_F32 || out_dtype == APL_BF16, "output dtype must be f32 or bf16");
    for (int i = 0; i < groups; ++i) need(A[i] && B[i] && C[i], "null operand");
    apl::check_cuda(apl::gemm_bf16_grouped(A, B, C, groups, 1, 1, static_cast<int>(M),
                                           static_cast<int>(N), static_cast<int>(K),
                                           static_cast<int>(lda), static_cast<int>(ldb),
                                           static_cast<int>(ldc), kn, out_dtype == APL_F32,
                                           APL_EPI_NONE, km, nullptr, static_cast<int>(ldc),
                                           static_cast<cudaStream_t>(stream)),
                    "grouped GEMM launch");
  });
}

int apl_mask_not(const void* x, void* y, size_t count, void* stream) {
  return guarded([&] {
    need((x && y) || count == 0, "null buffer");
    apl::check_cuda(apl::launch_mask_not(x, y, count, static_cast<cudaStream_t>(stream)),
                    "mask launch");
  });
}

int apl_sharded_matmul_backward(apl_mesh* mesh, const apl_matmul_strategy* strategy,
                                const apl_meta* a_meta, const apl_meta* b_meta,
                                const void* const* A, const void* const* B,
                                const void* const* dC, void* const* dA, void* const* dB,
                                int b_layout, int dA_epilogue, const void* const* aux,
                                int dB_dtype, void* stream) {
  return guarded([&] {
    need(mesh && strategy && dC, "null argument");
    need(dA == nullptr || B != nullptr, "dA needs B");
    need(dB == nullptr || A != nullptr, "dB needs A");
    need(b_layout == APL_B_NK || b_layout == APL_B_KN, "unknown B layout");
    need(dA_epilogue == APL_EPI_NONE || dA_epilogue == APL_EPI_DGELU, "unknown dA epilogue");
    need(dA_epilogue != APL_EPI_DGELU || aux != nullptr, "APL_EPI_DGELU needs aux");
    need(dB_dtype == APL_F32 || dB_dtype == APL_BF16, "dB dtype must be f32 or bf16");
    need(strategy->nreduce >= 0 && strategy->nreduce <= APL_MAX_MESH, "bad reduce axis count");
    apl::MatmulStrategy s;
    s.a = to_spec(&strategy->a);
    s.b = to_spec(&strategy->b);
    s.c = to_spec(&strategy->c);
    s.partial_sum = strategy->partial_sum != 0;
    for (int i = 0; i < strategy->nreduce; ++i) s.reduce_axes.push_back(strategy->reduce_axes[i]);
    apl::sharded_matmul_backward(mesh->impl, s, to_meta(a_meta), to_meta(b_meta), A, B, dC, dA,
                                 dB, b_layout == APL_B_KN, dA_epilogue == APL_EPI_DGELU, aux,
                                 dB_dtype, static_cast<cudaStream_t>(stream));
  });
}

int apl_launch_count(uint64_t* launches) {
  return guarded([&] {
    need(launches, "null out");
    *launches = apl::launch_count();
  });
}

}  // extern "C"
