// Partial-sum all-reduce on a simulated (single-GPU) mesh.
//
// Each axis group of the mesh holds `group_size` partial buffers; every
// member ends with the same sum, accumulated in fp32 in member order and
// rounded once (so results are identical across members and independent of
// thread scheduling). HBM-bound: reads group_size x count and writes
// group_size x count elements per group.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

namespace apl {

extern std::atomic<uint64_t> g_launches;

namespace {

constexpr int kMaxMembers = 64;

struct ReduceArgs {
  void* bufs[kMaxMembers];
  int members[kMaxMembers];
  int groups;
  int group_size;
};

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <>
__device__ __forceinline__ __half from_f<__half>(float x) { return __float2half_rn(x); }

// VEC elements per thread per iteration, moved as one 16-byte access when
// VEC * sizeof(T) == 16.
template <typename T, int VEC>
__global__ void __launch_bounds__(256) reduce_groups(const __grid_constant__ ReduceArgs a,
                                                     int64_t nvec) {
  struct alignas(sizeof(T) * VEC) Pack {
    T v[VEC];
  };
  const int g = blockIdx.y;
  const int* mem = a.members + g * a.group_size;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nvec;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = 0.f;
    for (int j = 0; j < a.group_size; ++j) {
      const Pack p = reinterpret_cast<const Pack*>(a.bufs[mem[j]])[i];
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[k] += to_f(p.v[k]);
    }
    Pack o;
#pragma unroll
    for (int k = 0; k < VEC; ++k) o.v[k] = from_f<T>(acc[k]);
    for (int j = 0; j < a.group_size; ++j) reinterpret_cast<Pack*>(a.bufs[mem[j]])[i] = o;
  }
}

template <typename T>
cudaError_t launch_typed(const ReduceArgs& a, size_t count, bool aligned, cudaStream_t stream) {
  constexpr int kVec = 16 / sizeof(T);
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_group = std::max(1, (sms * 8) / std::max(1, a.groups));
  if (aligned && count % kVec == 0) {
    const int64_t nvec = static_cast<int64_t>(count / kVec);
    const int64_t want = (nvec + 255) / 256;
    dim3 grid(static_cast<unsigned>(std::min<int64_t>(want, per_group)), a.groups);
    reduce_groups<T, kVec><<<grid, 256, 0, stream>>>(a, nvec);
  } else {
    const int64_t nvec = static_cast<int64_t>(count);
    const int64_t want = (nvec + 255) / 256;
    dim3 grid(static_cast<unsigned>(std::min<int64_t>(want, per_group)), a.groups);
    reduce_groups<T, 1><<<grid, 256, 0, stream>>>(a, nvec);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_allreduce_local(void* const* bufs, const int* members, int groups,
                                   int group_size, size_t count, int dtype,
                                   cudaStream_t stream) {
  if (groups * group_size > kMaxMembers) return cudaErrorInvalidValue;
  ReduceArgs a{};
  bool aligned = true;
  for (int i = 0; i < groups * group_size; ++i) {
    a.members[i] = i;
    a.bufs[i] = bufs[members[i]];
    aligned = aligned && (reinterpret_cast<uintptr_t>(a.bufs[i]) % 16 == 0);
  }
  a.groups = groups;
  a.group_size = group_size;
  switch (dtype) {
    case 0:
      return launch_typed<float>(a, count, aligned, stream);
    case 1:
      return launch_typed<__nv_bfloat16>(a, count, aligned, stream);
    case 2:
      return launch_typed<__half>(a, count, aligned, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

namespace {

__device__ __forceinline__ float gelu_f(float v) {
  return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
}
__device__ __forceinline__ float gelu_grad_f(float v) {
  return 0.5f * (1.f + erff(v * 0.70710678118654752f)) +
         v * 0.3989422804014327f * __expf(-0.5f * v * v);
}

// y = GELU(x) (dy == nullptr) or y = dy * GELU'(x), 16-byte vectors of
// 16 / sizeof(T) elements per thread per iteration (scalar tail).
template <typename T>
__global__ void __launch_bounds__(256) gelu_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                   const T* __restrict__ dy, int64_t n,
                                                   int64_t nv) {
  constexpr int VEC = 16 / sizeof(T);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += stride) {
    uint4 xv = reinterpret_cast<const uint4*>(x)[i], gv;
    if (dy != nullptr) gv = reinterpret_cast<const uint4*>(dy)[i];
    const T* xe = reinterpret_cast<const T*>(&xv);
    const T* ge = reinterpret_cast<const T*>(&gv);
    uint4 ov;
    T* oe = reinterpret_cast<T*>(&ov);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const float v = to_f(xe[k]);
      oe[k] = from_f<T>(dy != nullptr ? to_f(ge[k]) * gelu_grad_f(v) : gelu_f(v));
    }
    reinterpret_cast<uint4*>(y)[i] = ov;
  }
  for (int64_t i = nv * VEC + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const float v = to_f(x[i]);
    y[i] = from_f<T>(dy != nullptr ? to_f(dy[i]) * gelu_grad_f(v) : gelu_f(v));
  }
}

template <typename T>
cudaError_t gelu_typed(const void* x, void* y, const void* dy, size_t count, cudaStream_t stream) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                         reinterpret_cast<uintptr_t>(dy)) & 15) == 0;
  const size_t vec = 16 / sizeof(T);
  const int64_t nv = aligned ? static_cast<int64_t>(count / vec) : 0;  // else all scalar
  const int grid = static_cast<int>(std::min<size_t>((count / vec + 255) / 256 + 1, 148 * 8));
  gelu_kernel<T><<<grid, 256, 0, stream>>>(static_cast<const T*>(x), static_cast<T*>(y),
                                           static_cast<const T*>(dy), static_cast<int64_t>(count),
                                           nv);
  return cudaGetLastError();
}

cudaError_t gelu_dispatch(const void* x, void* y, const void* dy, size_t count, int dtype,
                          cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  cudaError_t e;
  switch (dtype) {
    case 0:
      e = gelu_typed<float>(x, y, dy, count, stream);
      break;
    case 1:
      e = gelu_typed<__nv_bfloat16>(x, y, dy, count, stream);
      break;
    case 2:
      e = gelu_typed<__half>(x, y, dy, count, stream);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return e;
}

}  // namespace

// Exact-erf GELU over a buffer (the epilogue of partial-sum strategies,
// applied once the all-reduce has produced the full sums).
cudaError_t launch_gelu_inplace(void* buf, size_t count, int dtype, cudaStream_t stream) {
  return gelu_dispatch(buf, buf, nullptr, count, dtype, stream);
}

// y = GELU(x) out of place (training forward keeps the pre-activation x).
cudaError_t launch_gelu(const void* x, void* y, size_t count, int dtype, cudaStream_t stream) {
  return gelu_dispatch(x, y, nullptr, count, dtype, stream);
}

// dx = dy * GELU'(x) (backward of an unfused elementwise GELU node).
cudaError_t launch_gelu_backward(const void* dy, const void* x, void* dx, size_t count, int dtype,
                                 cudaStream_t stream) {
  return gelu_dispatch(x, dx, dy, count, dtype, stream);
}

uint64_t launch_count() { return g_launches.load(); }

}  // namespace apl
