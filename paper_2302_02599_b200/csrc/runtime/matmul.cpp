// Sharded-matmul strategy execution: local tcgen05 GEMM on each device's
// shards, partial-sum all-reduce over the strategy's reduce axes, epilogue.
//
// Strategy semantics follow the reference catalog (proj/src/intraop.cpp:
// 141-234): C[..m.., n] = A[..m.., k] . B[k, n] with the input/output specs
// of the strategy; partial_sum strategies (split-k and the k-containing
// pairs) leave per-device partial sums that are reduced over reduce_axes
// (priced at intraop.cpp:544-551, inserted as <host>.ar nodes at
// planner.cpp:263-282).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "apl.h"
#include "runtime.hpp"

namespace apl {

void sharded_matmul(Mesh& mesh, const MatmulStrategy& s, const autoplan::TensorMeta& a_meta,
                    const autoplan::TensorMeta& b_meta, const void* const* A,
                    const void* const* B, void* const* C, bool b_kn, int out_dtype, int epilogue,
                    cudaStream_t stream, void* const* aux) {
  NvtxRange range("apl.sharded_matmul");
  const bool save = epilogue == APL_EPI_GELU_SAVE;
  if (save && (aux == nullptr || out_dtype != APL_BF16))
    throw RuntimeError(APL_ERR_ARG, "GELU_SAVE needs bf16 output and aux buffers");
  const auto& geo = mesh.geo;
  // matmul: A[..m.., k] . B[k, n];  batched matmul: A[b, m, k] . B[b, k, n]
  const bool batched = b_meta.rank() == 3;
  if (batched ? a_meta.rank() != 3 : (b_meta.rank() != 2 || a_meta.rank() < 2))
    throw RuntimeError(APL_ERR_SHAPE, "matmul wants A[..m.., k] . B[k, n] or A[b,m,k] . B[b,k,n]");
  if (a_meta.dtype_bytes != 2 || b_meta.dtype_bytes != 2)
    throw RuntimeError(APL_ERR_ARG, "matmul operands must be bf16");
  const size_t kb = batched ? 1 : 0;  // contraction dim of B
  if (a_meta.shape.back() != b_meta.shape[kb] || (batched && a_meta.shape[0] != b_meta.shape[0]))
    throw RuntimeError(APL_ERR_SHAPE, "contraction / batch extents differ");
  autoplan::TensorMeta c_meta = a_meta;
  c_meta.shape.back() = b_meta.shape.back();
  c_meta.dtype_bytes = out_dtype == APL_F32 ? 4 : 2;
  if (!s.a.valid_for(a_meta, geo) || !s.b.valid_for(b_meta, geo) || !s.c.valid_for(c_meta, geo))
    throw RuntimeError(APL_ERR_SHAPE, "strategy specs are not valid for these tensors");
  const auto la = local_shape(s.a, geo, a_meta);
  const auto lb = local_shape(s.b, geo, b_meta);
  const auto lc = local_shape(s.c, geo, c_meta);
  int64_t batch = 1, m = 1;
  if (batched) {
    batch = la[0];
    m = la[1];
    if (lb[0] != batch || lc[0] != batch || lc[1] != m)
      throw RuntimeError(APL_ERR_SHAPE, "A, B and C shards disagree on b / m");
  } else {
    for (size_t i = 0; i + 1 < la.size(); ++i) {
      m *= la[i];
      if (la[i] != lc[i]) throw RuntimeError(APL_ERR_SHAPE, "A and C shards disagree on m dims");
    }
  }
  const int64_t k = la.back(), n = lb.back();
  if (lb[kb] != k || lc.back() != n)
    throw RuntimeError(APL_ERR_SHAPE, "local shards do not form a matmul");
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX)
    throw RuntimeError(APL_ERR_ARG, "local GEMM extents exceed int32");
  const int nl = mesh.num_local();
  const int eb_c = out_dtype == APL_F32 ? 4 : 2;
  // Simulated mesh + partial sums: the GEMM and its all-reduce are ONE
  // kernel — each reduction group's tile accumulates every member's K slice
  // in TMEM (fp32, member order) and the epilogue writes the finished tile
  // (GELU applied to the full sum) to every member. APL_FUSED_AR=0 keeps the
  // two-pass form (GEMM writes partials, reduce_groups sums them).
  static const bool fused_ar_enabled = [] {
    const char* e = std::getenv("APL_FUSED_AR");
    return e == nullptr || std::string(e) != "0";
  }();
  if (s.partial_sum && !mesh.distributed && batch == 1 && fused_ar_enabled && !save) {
    const auto groups = axis_groups(geo, s.reduce_axes);
    const int gsize = static_cast<int>(groups[0].size());
    if (gsize <= 8) {
      std::vector<const void*> pa, pb;
      std::vector<void*> pc;
      for (const auto& g : groups)
        for (int d : g) {
          pa.push_back(A[d]);
          pb.push_back(B[d]);
          pc.push_back(C[d]);
        }
      check_cuda(gemm_bf16_grouped(pa.data(), pb.data(), pc.data(),
                                   static_cast<int>(groups.size()), gsize, gsize,
                                   static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                                   static_cast<int>(k), static_cast<int>(b_kn ? n : k),
                                   static_cast<int>(n), b_kn, out_dtype == APL_F32,
                                   epilogue == APL_EPI_GELU, stream),
                 "fused GEMM + all-reduce launch");
      return;
    }
  }
  const bool fuse_gelu = (epilogue == APL_EPI_GELU || save) && !s.partial_sum;
  // Every local device (and every batch element) has the same shard shapes:
  // all problems go through the persistent batched launcher together (a
  // simulated mesh runs its 8 GEMMs as one launch).
  std::vector<const void*> pa, pb;
  std::vector<void*> pc;
  for (int d = 0; d < nl; ++d)
    for (int64_t i = 0; i < batch; ++i) {
      pa.push_back(static_cast<const char*>(A[d]) + i * m * k * 2);
      pb.push_back(static_cast<const char*>(B[d]) + i * k * n * 2);
      pc.push_back(static_cast<char*>(C[d]) + i * m * n * eb_c);
    }
  std::vector<const void*> px;
  if (save && fuse_gelu)
    for (int d = 0; d < nl; ++d)
      for (int64_t i = 0; i < batch; ++i)
        px.push_back(static_cast<const char*>(aux[d]) + i * m * n * 2);
  check_cuda(gemm_bf16_grouped(pa.data(), pb.data(), pc.data(), static_cast<int>(pa.size()), 1, 1,
                               static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                               static_cast<int>(k), static_cast<int>(b_kn ? n : k),
                               static_cast<int>(n), b_kn, out_dtype == APL_F32,
                               fuse_gelu ? (save ? 3 : 1) : 0, false,
                               px.empty() ? nullptr : px.data(), static_cast<int>(n), stream),
             "tcgen05 GEMM launch");
  const size_t count = static_cast<size_t>(batch * m * n);
  if (s.partial_sum) {
    all_reduce(mesh, s.reduce_axes, C, count, out_dtype, stream);
    for (int d = 0; d < nl && (epilogue == APL_EPI_GELU || save); ++d) {
      if (save)  // the full sum is the pre-activation
        check_cuda(cudaMemcpyAsync(aux[d], C[d], count * 2, cudaMemcpyDeviceToDevice, stream),
                   "save pre-activation");
      check_cuda(launch_gelu_inplace(C[d], count, out_dtype, stream), "gelu launch");
    }
  }
}

namespace {

// Local GEMM extents of a strategy: batch, m (all m dims flattened), k, n.
struct LocalDims {
  int64_t batch = 1, m = 1, k = 0, n = 0;
};

LocalDims local_dims(const Mesh& mesh, const MatmulStrategy& s, const autoplan::TensorMeta& a_meta,
                     const autoplan::TensorMeta& b_meta) {
  const auto& geo = mesh.geo;
  const bool batched = b_meta.rank() == 3;
  if (batched ? a_meta.rank() != 3 : (b_meta.rank() != 2 || a_meta.rank() < 2))
    throw RuntimeError(APL_ERR_SHAPE, "matmul wants A[..m.., k] . B[k, n] or A[b,m,k] . B[b,k,n]");
  if (a_meta.dtype_bytes != 2 || b_meta.dtype_bytes != 2)
    throw RuntimeError(APL_ERR_ARG, "matmul operands must be bf16");
  const size_t kb = batched ? 1 : 0;
  if (a_meta.shape.back() != b_meta.shape[kb] || (batched && a_meta.shape[0] != b_meta.shape[0]))
    throw RuntimeError(APL_ERR_SHAPE, "contraction / batch extents differ");
  autoplan::TensorMeta c_meta = a_meta;
  c_meta.shape.back() = b_meta.shape.back();
  if (!s.a.valid_for(a_meta, geo) || !s.b.valid_for(b_meta, geo) || !s.c.valid_for(c_meta, geo))
    throw RuntimeError(APL_ERR_SHAPE, "strategy specs are not valid for these tensors");
  const auto la = local_shape(s.a, geo, a_meta);
  const auto lb = local_shape(s.b, geo, b_meta);
  const auto lc = local_shape(s.c, geo, c_meta);
  LocalDims d;
  if (batched) {
    d.batch = la[0];
    d.m = la[1];
    if (lb[0] != d.batch || lc[0] != d.batch || lc[1] != d.m)
      throw RuntimeError(APL_ERR_SHAPE, "A, B and C shards disagree on b / m");
  } else {
    for (size_t i = 0; i + 1 < la.size(); ++i) {
      d.m *= la[i];
      if (la[i] != lc[i]) throw RuntimeError(APL_ERR_SHAPE, "A and C shards disagree on m dims");
    }
  }
  d.k = la.back();
  d.n = lb.back();
  if (lb[kb] != d.k || lc.back() != d.n)
    throw RuntimeError(APL_ERR_SHAPE, "local shards do not form a matmul");
  if (d.m > INT32_MAX || d.n > INT32_MAX || d.k > INT32_MAX)
    throw RuntimeError(APL_ERR_ARG, "local GEMM extents exceed int32");
  return d;
}

// One backward GEMM over every local device (and batch element), with the
// sum over `partial_axes`: on a simulated mesh fused into the GEMM (each
// group's tile accumulates every member's contraction slice, the epilogue
// writes every member), otherwise GEMM + all_reduce.
struct BwdGemm {
  int M, N, K, lda, ldb, ldc;
  bool a_km, b_kn, out_f32;
  int epi;
  int64_t a_step, b_step, c_step, aux_step;  // bytes per batch element
};

void run_bwd_gemm(Mesh& mesh, const BwdGemm& g, int64_t batch, const void* const* A,
                  const void* const* B, void* const* C, const void* const* aux,
                  const std::vector<int>& partial_axes, cudaStream_t stream) {
  const int nl = mesh.num_local();
  static const bool fused_ar_enabled = [] {
    const char* e = std::getenv("APL_FUSED_AR");
    return e == nullptr || std::string(e) != "0";
  }();
  if (!partial_axes.empty() && !mesh.distributed && batch == 1 && fused_ar_enabled) {
    const auto groups = axis_groups(mesh.geo, partial_axes);
    const int gsize = static_cast<int>(groups[0].size());
    if (gsize <= 8) {
      std::vector<const void*> pa, pb, px;
      std::vector<void*> pc;
      for (const auto& grp : groups) {
        px.push_back(aux ? aux[grp[0]] : nullptr);  // aux is replicated over the group
        for (int d : grp) {
          pa.push_back(A[d]);
          pb.push_back(B[d]);
          pc.push_back(C[d]);
        }
      }
      check_cuda(gemm_bf16_grouped(pa.data(), pb.data(), pc.data(),
                                   static_cast<int>(groups.size()), gsize, gsize, g.M, g.N, g.K,
                                   g.lda, g.ldb, g.ldc, g.b_kn, g.out_f32, g.epi, g.a_km,
                                   aux ? px.data() : nullptr, g.ldc, stream),
                 "fused backward GEMM + all-reduce launch");
      return;
    }
  }
  std::vector<const void*> pa, pb, px;
  std::vector<void*> pc;
  for (int d = 0; d < nl; ++d)
    for (int64_t i = 0; i < batch; ++i) {
      pa.push_back(static_cast<const char*>(A[d]) + i * g.a_step);
      pb.push_back(static_cast<const char*>(B[d]) + i * g.b_step);
      pc.push_back(static_cast<char*>(C[d]) + i * g.c_step);
      px.push_back(aux ? static_cast<const char*>(aux[d]) + i * g.aux_step : nullptr);
    }
  check_cuda(gemm_bf16_grouped(pa.data(), pb.data(), pc.data(), static_cast<int>(pa.size()), 1, 1,
                               g.M, g.N, g.K, g.lda, g.ldb, g.ldc, g.b_kn, g.out_f32, g.epi,
                               g.a_km, aux ? px.data() : nullptr, g.ldc, stream),
             "backward GEMM launch");
  if (!partial_axes.empty())
    all_reduce(mesh, partial_axes, C, static_cast<size_t>(batch) * g.M * g.N,
               g.out_f32 ? APL_F32 : APL_BF16, stream);
}

}  // namespace

void sharded_matmul_backward(Mesh& mesh, const MatmulStrategy& s,
                             const autoplan::TensorMeta& a_meta,
                             const autoplan::TensorMeta& b_meta, const void* const* A,
                             const void* const* B, const void* const* dC, void* const* dA,
                             void* const* dB, bool b_kn, bool dgelu, const void* const* aux,
                             int dB_dtype, cudaStream_t stream) {
  NvtxRange range("apl.sharded_matmul_backward");
  const LocalDims d = local_dims(mesh, s, a_meta, b_meta);
  const bool batched = b_meta.rank() == 3;
  if (dgelu && aux == nullptr) throw RuntimeError(APL_ERR_ARG, "GELU backward needs aux");
  if (dB_dtype != APL_F32 && dB_dtype != APL_BF16)
    throw RuntimeError(APL_ERR_ARG, "dB dtype must be f32 or bf16");
  // Which mesh axes each gradient is partial over (C = A . B with C's dims
  // [..m.., n]): dA sums over n, so over the axes sharding C's n dim; dB
  // sums over m, so over the axes sharding C's m dims (batch dims excluded).
  std::vector<int> n_axes = s.c.dims.back().axes, m_axes;
  for (size_t i = batched ? 1 : 0; i + 1 < s.c.dims.size(); ++i)
    m_axes.insert(m_axes.end(), s.c.dims[i].axes.begin(), s.c.dims[i].axes.end());
  std::sort(n_axes.begin(), n_axes.end());
  std::sort(m_axes.begin(), m_axes.end());
  const int m = static_cast<int>(d.m), k = static_cast<int>(d.k), n = static_cast<int>(d.n);
  if (dA != nullptr) {
    // dA[m, k] = dC[m, n] . B^T: B [k, n] stored row-major is the Bt form of
    // the operand B^T; B stored transposed [n, k] is its row-major form.
    BwdGemm g{m, k, n, n, b_kn ? n : k, k, false, !b_kn, false,
              dgelu ? 2 : 0, int64_t{m} * n * 2, int64_t{k} * n * 2, int64_t{m} * k * 2,
              int64_t{m} * k * 2};
    run_bwd_gemm(mesh, g, d.batch, dC, B, dA, dgelu ? aux : nullptr, n_axes, stream);
  }
  if (dB != nullptr) {
    const bool f32 = dB_dtype == APL_F32;
    const int eb = f32 ? 4 : 2;
    if (b_kn) {
      // dB[k, n] = A^T . dC: A [m, k] read as the MN-major operand A^T.
      BwdGemm g{k, n, m, k, n, n, true, true, f32, 0, int64_t{m} * k * 2, int64_t{m} * n * 2,
                int64_t{k} * n * eb, 0};
      run_bwd_gemm(mesh, g, d.batch, A, dC, dB, nullptr, m_axes, stream);
    } else {
      // dBt[n, k] = dC^T . A: dC [m, n] read as the MN-major operand dC^T.
      BwdGemm g{n, k, m, n, k, k, true, true, f32, 0, int64_t{m} * n * 2, int64_t{m} * k * 2,
                int64_t{n} * k * eb, 0};
      run_bwd_gemm(mesh, g, d.batch, dC, A, dB, nullptr, m_axes, stream);
    }
  }
}

}  // namespace apl
