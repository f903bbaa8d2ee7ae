// Batched N-D box copy kernel (sm_100a). See box_copy.cuh for the model.
//
// Roofline: HBM. Algorithmic bytes per launch = 2 x sum of descriptor bytes
// (every byte is read once and written once). Design points:
//  * persistent grid (a multiple of the SM count), each CTA sweeping chunks
//    of blockDim * U units; U independent 128-bit loads are issued before
//    any store so every thread keeps U x 16 B in flight;
//  * the chunk's descriptor is staged in shared memory once per chunk, so
//    the per-unit address math is two multiply-high divisions per outer dim
//    against smem-resident constants (no per-unit global descriptor loads
//    unless a chunk straddles two descriptors);
//  * loads use the non-coherent streaming path (ld.global.nc.L1::no_allocate),
//    stores are plain 128-bit st.global (data is consumed by the next kernel
//    or a collective, so it should stay in L2 when it fits).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <stdexcept>
#include <string>

#include "box_copy.cuh"

namespace apl {

std::atomic<uint64_t> g_launches{0};

namespace {

template <int V>
struct Vec;
template <>
struct Vec<16> {
  using T = uint4;
};
template <>
struct Vec<8> {
  using T = uint2;
};
template <>
struct Vec<4> {
  using T = uint32_t;
};
template <>
struct Vec<2> {
  using T = uint16_t;
};
template <>
struct Vec<1> {
  using T = uint8_t;
};

__device__ __forceinline__ uint4 load_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 load_stream(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t load_stream(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint16_t load_stream(const uint16_t* p) { return __ldg(p); }
__device__ __forceinline__ uint8_t load_stream(const uint8_t* p) { return __ldg(p); }

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.div == 1 ? n : (__umulhi(n, f.mul) >> f.shr);
}

// Resolves unit `local` of descriptor `c` into (src, dst) byte offsets.
template <int V>
__device__ __forceinline__ void resolve(const DevCopy& c, uint32_t local, int64_t& so,
                                        int64_t& dd) {
  uint32_t row = fdiv(local, c.units_per_run);
  const uint32_t col = local - row * c.units_per_run.div;
  so = c.src_off + static_cast<int64_t>(col) * V;
  dd = c.dst_off + static_cast<int64_t>(col) * V;
  for (int i = c.nouter - 1; i >= 0; --i) {
    const uint32_t q = fdiv(row, c.ext[i]);
    const uint32_t r = row - q * c.ext[i].div;
    so += static_cast<int64_t>(r) * c.src_stride[i];
    dd += static_cast<int64_t>(r) * c.dst_stride[i];
    row = q;
  }
}

template <int V, int U>
__global__ void __launch_bounds__(256, 4)
    box_copy_kernel(const DevCopy* __restrict__ table, int ntasks, int64_t total,
                    const __grid_constant__ PtrTable ptrs) {
  using T = typename Vec<V>::T;
  __shared__ DevCopy s_desc;
  __shared__ int s_task;
  __shared__ int64_t s_next_begin;
  const int64_t chunk = static_cast<int64_t>(blockDim.x) * U;

  for (int64_t base = static_cast<int64_t>(blockIdx.x) * chunk; base < total;
       base += static_cast<int64_t>(gridDim.x) * chunk) {
    if (threadIdx.x == 0) {
      int lo = 0, hi = ntasks - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (table[mid].unit_begin <= base) lo = mid;
        else hi = mid - 1;
      }
      s_task = lo;
      s_next_begin = (lo + 1 < ntasks) ? table[lo + 1].unit_begin : total;
    }
    __syncthreads();
    const int t0 = s_task;
    {
      const uint32_t* g = reinterpret_cast<const uint32_t*>(table + t0);
      uint32_t* s = reinterpret_cast<uint32_t*>(&s_desc);
      for (int w = threadIdx.x; w < static_cast<int>(sizeof(DevCopy) / 4); w += blockDim.x)
        s[w] = g[w];
    }
    __syncthreads();
    const int64_t next_begin = s_next_begin;

    T v[U];
    char* dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t g = base + static_cast<int64_t>(u) * blockDim.x + threadIdx.x;
      dst[u] = nullptr;
      if (g < total) {
        int64_t so, dd;
        const char* sp;
        char* dp;
        if (g < next_begin) {
          resolve<V>(s_desc, static_cast<uint32_t>(g - s_desc.unit_begin), so, dd);
          sp = ptrs.src[s_desc.src_buf];
          dp = ptrs.dst[s_desc.dst_buf];
        } else {  // chunk straddles descriptors: walk forward in global
          int t = t0 + 1;
          while (t + 1 < ntasks && table[t + 1].unit_begin <= g) ++t;
          const DevCopy& c = table[t];
          resolve<V>(c, static_cast<uint32_t>(g - c.unit_begin), so, dd);
          sp = ptrs.src[c.src_buf];
          dp = ptrs.dst[c.dst_buf];
        }
        v[u] = load_stream(reinterpret_cast<const T*>(sp + so));
        dst[u] = dp + dd;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u] != nullptr) *reinterpret_cast<T*>(dst[u]) = v[u];
    __syncthreads();  // s_desc is rewritten by the next chunk
  }
}

int g_num_sms = 0;

}  // namespace

FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.div = d;
  if (d <= 1) {
    f.div = 1;
    return f;
  }
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;  // ceil(log2 d)
  const uint64_t p = 31 + l;
  f.mul = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
  f.shr = static_cast<uint32_t>(p - 32);
  return f;
}

int sm_count() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

cudaError_t launch_box_copy(const DevCopy* d_table, int ntasks, int64_t total_units,
                            int vec_bytes, const PtrTable& ptrs, cudaStream_t stream) {
  if (ntasks <= 0 || total_units <= 0) return cudaSuccess;
  constexpr int kThreads = 256;
  constexpr int kUnroll = 4;
  const int64_t chunk = static_cast<int64_t>(kThreads) * kUnroll;
  const int64_t chunks = (total_units + chunk - 1) / chunk;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 4;  // 4 resident CTAs per SM
  const int grid = static_cast<int>(std::min(chunks, cap));
  switch (vec_bytes) {
    case 16:
      box_copy_kernel<16, kUnroll><<<grid, kThreads, 0, stream>>>(d_table, ntasks, total_units, ptrs);
      break;
    case 8:
      box_copy_kernel<8, kUnroll><<<grid, kThreads, 0, stream>>>(d_table, ntasks, total_units, ptrs);
      break;
    case 4:
      box_copy_kernel<4, kUnroll><<<grid, kThreads, 0, stream>>>(d_table, ntasks, total_units, ptrs);
      break;
    case 2:
      box_copy_kernel<2, kUnroll><<<grid, kThreads, 0, stream>>>(d_table, ntasks, total_units, ptrs);
      break;
    default:
      box_copy_kernel<1, kUnroll><<<grid, kThreads, 0, stream>>>(d_table, ntasks, total_units, ptrs);
      break;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace apl
