// Device-side epoch flags for the peer-memory exchange (no host barrier, no
// NCCL): every rank owns a small IPC-exported flag array that its peers
// write into over NVLink.
//
//   flags[r][slot]  slot p          : "rank p's source shard of epoch e is written"
//                   slot P + p      : "rank p finished reading epoch e's sources"
//
// An exchange at epoch e on rank r is, in stream order:
//   store(ready, e) to every peer -> wait(all ready >= e) -> pull kernel ->
//   store(done, e) to every peer
// and before r overwrites its source for epoch e+1: wait(all done >= e).
// Stores are st.release.sys after a system fence (the producer's writes and
// the pull's reads completed at the preceding kernel boundary); waits spin on
// ld.acquire.sys with a nanosleep back-off and trap after a timeout instead of
// hanging the GPU.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

namespace apl {

extern std::atomic<uint64_t> g_launches;

constexpr int kMaxFlagPeers = 64;

struct FlagPtrs {
  uint32_t* p[kMaxFlagPeers];
};
struct FlagSlots {
  int s[kMaxFlagPeers];
};

namespace {

__global__ void flag_store_kernel(const __grid_constant__ FlagPtrs ptrs, int n, int slot,
                                  uint32_t epoch) {
  __threadfence_system();
  const int i = threadIdx.x;
  if (i < n)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(ptrs.p[i] + slot), "r"(epoch)
                 : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void flag_wait_kernel(const uint32_t* flags, const __grid_constant__ FlagSlots slots,
                                 int n, uint32_t epoch, uint64_t timeout_ns) {
  const int i = threadIdx.x;
  if (i < n) {
    const uint32_t* f = flags + slots.s[i];
    const uint64_t t0 = global_ns();
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;  // wrap-safe v >= epoch
      __nanosleep(256);
      if (global_ns() - t0 > timeout_ns) __trap();  // a lost peer: fail, do not hang
    }
  }
  __syncthreads();
}

struct OutPtrs {
  void* p[8];
};

// Owner side of the fused all-reduce: sum the P fp32 partial slabs this rank
// received (in rank order: deterministic, and only the owner computes its
// rows, so every replica gets identical bytes) and write the result into
// every rank's output at this rank's rows (peer stores = the all-gather).
__global__ void __launch_bounds__(256) reduce_gather_kernel(const float* __restrict__ staging,
                                                            int P, int64_t slab4,
                                                            const __grid_constant__ OutPtrs outs,
                                                            int nout, int out_f32) {
  const float4* st = reinterpret_cast<const float4*>(staging);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < slab4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = __ldg(st + i);
    for (int r = 1; r < P; ++r) {
      const float4 b = __ldg(st + r * slab4 + i);
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    if (out_f32) {
      for (int q = 0; q < nout; ++q) reinterpret_cast<float4*>(outs.p[q])[i] = a;
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      uint2 v;
      v.x = *reinterpret_cast<uint32_t*>(&lo);
      v.y = *reinterpret_cast<uint32_t*>(&hi);
      for (int q = 0; q < nout; ++q) reinterpret_cast<uint2*>(outs.p[q])[i] = v;
    }
  }
}

// In-place all-reduce of this rank's block across the P members of a group:
// bufs.p[r] = member r's tensor at this rank's block (peer-mapped). Each
// rank owns one block: it reads the block from every member, sums in member
// order in fp32 (deterministic; only the owner computes the block, so every
// member ends with identical bytes) and writes the sum back to every member.
// Blocks of different owners never overlap, so no two kernels race.
template <typename T>
__global__ void __launch_bounds__(256) peer_allreduce_kernel(const __grid_constant__ OutPtrs bufs,
                                                             int P, int64_t n) {
  constexpr int VEC = 16 / sizeof(T);
  const int64_t nv = n / VEC;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t i = tid; i < nv; i += stride) {
    float acc[VEC];
    for (int r = 0; r < P; ++r) {
      const uint4 u = reinterpret_cast<const uint4*>(bufs.p[r])[i];
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[k] = (r == 0 ? 0.f : acc[k]) + static_cast<float>(e[k]);
    }
    uint4 o;
    T* oe = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int k = 0; k < VEC; ++k) oe[k] = static_cast<T>(acc[k]);
    for (int r = 0; r < P; ++r) reinterpret_cast<uint4*>(bufs.p[r])[i] = o;
  }
  for (int64_t i = nv * VEC + tid; i < n; i += stride) {
    float acc = 0.f;
    for (int r = 0; r < P; ++r) acc += static_cast<float>(static_cast<const T*>(bufs.p[r])[i]);
    for (int r = 0; r < P; ++r) static_cast<T*>(bufs.p[r])[i] = static_cast<T>(acc);
  }
}

}  // namespace

cudaError_t launch_peer_allreduce(void* const* members, int P, int64_t count, int dtype,
                                  cudaStream_t stream) {
  if (P < 1 || P > 8 || count < 0) return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  OutPtrs b{};
  bool aligned = true;
  for (int r = 0; r < P; ++r) {
    b.p[r] = members[r];
    aligned = aligned && (reinterpret_cast<uintptr_t>(members[r]) & 15) == 0;
  }
  if (!aligned) return cudaErrorMisalignedAddress;
  const int grid = static_cast<int>(std::min<int64_t>((count / 4 + 255) / 256 + 1, 148 * 8));
  if (dtype == 0)
    peer_allreduce_kernel<float><<<grid, 256, 0, stream>>>(b, P, count);
  else if (dtype == 1)
    peer_allreduce_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(b, P, count);
  else
    return cudaErrorInvalidValue;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_reduce_gather(const float* staging, int P, int64_t slab_elems,
                                 void* const* outs, int nout, bool out_f32, cudaStream_t stream) {
  if (P < 1 || nout < 1 || nout > 8 || slab_elems % 4) return cudaErrorInvalidValue;
  OutPtrs o{};
  for (int q = 0; q < nout; ++q) o.p[q] = outs[q];
  const int64_t slab4 = slab_elems / 4;
  const int grid = static_cast<int>(std::min<int64_t>((slab4 + 255) / 256, 148 * 8));
  reduce_gather_kernel<<<grid, 256, 0, stream>>>(staging, P, slab4, o, nout, out_f32 ? 1 : 0);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_flag_store(uint32_t* const* remote, int n, int slot, uint32_t epoch,
                              cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (n > kMaxFlagPeers) return cudaErrorInvalidValue;
  FlagPtrs p{};
  for (int i = 0; i < n; ++i) p.p[i] = remote[i];
  flag_store_kernel<<<1, 64, 0, stream>>>(p, n, slot, epoch);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_flag_wait(const uint32_t* flags, const int* slots, int n, uint32_t epoch,
                             uint64_t timeout_ns, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (n > kMaxFlagPeers) return cudaErrorInvalidValue;
  FlagSlots s{};
  for (int i = 0; i < n; ++i) s.s[i] = slots[i];
  flag_wait_kernel<<<1, 64, 0, stream>>>(flags, s, n, epoch, timeout_ns);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace apl
