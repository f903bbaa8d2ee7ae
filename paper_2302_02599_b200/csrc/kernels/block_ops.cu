// The non-GEMM node kinds of the reference's transformer-block graph
// (proj/tests/fixtures/gpt_block.json; kinds graph_ir.cpp:40-46, shape rules
// graph_ir.cpp:240-345), run on one device's shard. Every strategy the
// reference generates for them keeps the op local (intraop.cpp:280-450: the
// softmax / layernorm axis stays replicated, an embedding shards the lookup
// batch or the table's hidden dim, a transpose permutes the spec with the
// data), so these kernels never communicate: the plan executor converts
// their inputs first.
//
// All HBM-bound; fp32 math, bf16 / f32 / u8 storage:
//   embedding  : rows of the table gathered per id       (width x eb read + written per id);
//                from a sharded table's owner blocks directly (all-gather fused)
//   layernorm  : warp per row, mean / var / affine        (row read once into registers
//   softmax    : warp per row, max, exp-sum, normalise     up to 256 x 16 B, else streamed
//                                                          from L1 in 3 / 2 passes; written once)
//   transpose  : [batch, R, C] -> [batch, C, R], 64 x 64 shared-memory tiles with
//                16-byte vectors on both sides (32 x 32 scalar tiles for ragged shapes)
//   scale / add / not : 16-byte vectors, grid-stride
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

namespace apl {

extern std::atomic<uint64_t> g_launches;
int sm_count();

namespace {

__device__ __forceinline__ float ld(const float* p) { return *p; }
__device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void st(float* p, float v) { *p = v; }
__device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// V contiguous elements per access: 16-byte vectors when the row allows, else 1.
// The alignment makes the access one LDG/STG.128 instead of V narrow ones.
template <typename T, int V>
struct alignas(sizeof(T) * V) Vec {
  T v[V];
};

template <typename T, int V>
__device__ __forceinline__ void load_row(const T* row, int64_t i, float (&f)[V]) {
  const Vec<T, V> x = reinterpret_cast<const Vec<T, V>*>(row)[i];
#pragma unroll
  for (int k = 0; k < V; ++k) f[k] = ld(&x.v[k]);
}

template <typename T, int V>
__device__ __forceinline__ void store_row(T* row, int64_t i, const float (&f)[V]) {
  Vec<T, V> x;
#pragma unroll
  for (int k = 0; k < V; ++k) st(&x.v[k], f[k]);
  reinterpret_cast<Vec<T, V>*>(row)[i] = x;
}

// ---- embedding lookup: out[t, :] = table[ids[t], :] ------------------------
// Ids outside [0, vocab) produce a zero row (the reference plans the op and
// does not define out-of-range lookups).
template <typename W>
__global__ void __launch_bounds__(256) embedding_kernel(const int64_t* __restrict__ ids, int64_t n,
                                                        const W* __restrict__ table, int64_t vocab,
                                                        int64_t words, W* __restrict__ out) {
  const int64_t total = n * words;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += stride) {
    const int64_t t = i / words, w = i - t * words;
    const int64_t id = __ldg(ids + t);
    W v{};
    if (id >= 0 && id < vocab) v = table[id * words + w];
    out[i] = v;
  }
}

// ---- embedding lookup from a sharded table, all-gather fused ----------------
// The table is a grid of [vocab_blocks x hidden_blocks] equal blocks, each
// contiguous [vb_rows, hb_words] in its owner's buffer (a simulated mesh's
// shard, or a peer-mapped shard); out[t, :] = table[ids[t], col0 : col0 +
// out_words] read straight from the owners: the gather of the whole table
// every device would otherwise materialise is never written.
constexpr int kMaxBlocks = 64;
struct TableBlocks {
  const void* p[kMaxBlocks];
};

template <typename W>
__global__ void __launch_bounds__(256) embedding_blocks_kernel(
    const int64_t* __restrict__ ids, int64_t n, const __grid_constant__ TableBlocks blocks,
    int hidden_blocks, int64_t vb_rows, int64_t hb_words, int64_t vocab, int64_t col0,
    int64_t out_words, W* __restrict__ out) {
  // a warp per id: the owner block row is found once, then the output row is
  // copied run by run (one run per hidden block it spans), no per-word division
  const int lane = threadIdx.x % 32;
  for (int64_t t = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    W* orow = out + t * out_words;
    const int64_t id = __ldg(ids + t);
    if (id < 0 || id >= vocab) {
      for (int64_t w = lane; w < out_words; w += 32) orow[w] = W{};
      continue;
    }
    const int64_t vb = id / vb_rows, r = id - vb * vb_rows;
    for (int64_t w = 0; w < out_words;) {
      const int64_t col = col0 + w, hb = col / hb_words, off = col - hb * hb_words;
      const int64_t len = min(hb_words - off, out_words - w);
      const W* src = static_cast<const W*>(blocks.p[vb * hidden_blocks + hb]) + r * hb_words + off;
      for (int64_t k = lane; k < len; k += 32) orow[w + k] = src[k];
      w += len;
    }
  }
}

// ---- layernorm over the last dim ----------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(256) layernorm_kernel(const T* __restrict__ x,
                                                        const T* __restrict__ gamma,
                                                        const T* __restrict__ beta,
                                                        T* __restrict__ y, int64_t rows,
                                                        int64_t width, float eps) {
  const int lane = threadIdx.x % 32;
  const int64_t nv = width / V;
  const float inv_w = 1.f / static_cast<float>(width);
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const T* xr = x + r * width;
    T* yr = y + r * width;
    float s = 0.f;
    for (int64_t i = lane; i < nv; i += 32) {
      float f[V];
      load_row<T, V>(xr, i, f);
#pragma unroll
      for (int k = 0; k < V; ++k) s += f[k];
    }
    const float mean = warp_sum(s) * inv_w;
    float q = 0.f;
    for (int64_t i = lane; i < nv; i += 32) {
      float f[V];
      load_row<T, V>(xr, i, f);
#pragma unroll
      for (int k = 0; k < V; ++k) q += (f[k] - mean) * (f[k] - mean);
    }
    const float rstd = rsqrtf(warp_sum(q) * inv_w + eps);
    for (int64_t i = lane; i < nv; i += 32) {
      float f[V], g[V], b[V];
      load_row<T, V>(xr, i, f);
      if (gamma != nullptr) load_row<T, V>(gamma, i, g);
      if (beta != nullptr) load_row<T, V>(beta, i, b);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        float v = (f[k] - mean) * rstd;
        if (gamma != nullptr) v *= g[k];
        if (beta != nullptr) v += b[k];
        f[k] = v;
      }
      store_row<T, V>(yr, i, f);
    }
  }
}

// ---- softmax over the last dim ------------------------------------------
// Attention pre-op fused in: softmax(alpha * x + fill * mask), mask a u8
// [rows, width] (or null); alpha = 1 / null mask is the plain softmax.
template <int V>
__device__ __forceinline__ void pre_op(float (&f)[V], const uint8_t* mrow, int64_t i, float alpha,
                                       float fill) {
  if (mrow != nullptr) {
    const Vec<uint8_t, V> m = reinterpret_cast<const Vec<uint8_t, V>*>(mrow)[i];
#pragma unroll
    for (int k = 0; k < V; ++k) f[k] = alpha * f[k] + fill * static_cast<float>(m.v[k]);
  } else if (alpha != 1.f) {
#pragma unroll
    for (int k = 0; k < V; ++k) f[k] *= alpha;
  }
}

template <typename T, int V>
__global__ void __launch_bounds__(256) softmax_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                      int64_t rows, int64_t width, float alpha,
                                                      const uint8_t* __restrict__ mask,
                                                      float fill) {
  const int lane = threadIdx.x % 32;
  const int64_t nv = width / V;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const T* xr = x + r * width;
    T* yr = y + r * width;
    const uint8_t* mr = mask != nullptr ? mask + r * width : nullptr;
    float m = -INFINITY, s = 0.f;  // online max / sum per lane
    for (int64_t i = lane; i < nv; i += 32) {
      float f[V];
      load_row<T, V>(xr, i, f);
      pre_op<V>(f, mr, i, alpha, fill);
      float mv = f[0];
#pragma unroll
      for (int k = 1; k < V; ++k) mv = fmaxf(mv, f[k]);
      const float nm = fmaxf(m, mv);
      s *= __expf(m - nm);
#pragma unroll
      for (int k = 0; k < V; ++k) s += __expf(f[k] - nm);
      m = nm;
    }
    const float gm = warp_max(m);
    const float gs = warp_sum(m == -INFINITY ? 0.f : s * __expf(m - gm));
    const float inv = 1.f / gs;
    for (int64_t i = lane; i < nv; i += 32) {
      float f[V];
      load_row<T, V>(xr, i, f);
      pre_op<V>(f, mr, i, alpha, fill);
#pragma unroll
      for (int k = 0; k < V; ++k) f[k] = __expf(f[k] - gm) * inv;
      store_row<T, V>(yr, i, f);
    }
  }
}

// ---- [batch, R, C] -> [batch, C, R] -------------------------------------
template <typename W>
__global__ void __launch_bounds__(256) transpose_kernel(const W* __restrict__ x, W* __restrict__ y,
                                                        int64_t batch, int R, int C) {
  __shared__ W tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int64_t b = blockIdx.z; b < batch; b += gridDim.z) {
    const W* xb = x + b * R * static_cast<int64_t>(C);
    W* yb = y + b * R * static_cast<int64_t>(C);
    for (int j = threadIdx.y; j < 32; j += 8) {
      const int r = r0 + j, c = c0 + threadIdx.x;
      if (r < R && c < C) tile[j][threadIdx.x] = xb[static_cast<int64_t>(r) * C + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
      const int c = c0 + j, r = r0 + threadIdx.x;
      if (r < R && c < C) yb[static_cast<int64_t>(c) * R + r] = tile[threadIdx.x][j];
    }
    __syncthreads();
  }
}

// ---- row-cached variants: rows of up to 32 x NV x V elements are loaded once
// into registers (every load of the row in flight together), then reduced and
// written -- one HBM round trip of latency per row instead of three.
template <typename T, int V, int NV>
__global__ void __launch_bounds__(256) layernorm_cached_kernel(
    const T* __restrict__ x, const T* __restrict__ gamma, const T* __restrict__ beta,
    T* __restrict__ y, int64_t rows, int64_t width, float eps) {
  const int lane = threadIdx.x % 32;
  const int nv = static_cast<int>(width / V);
  const float inv_w = 1.f / static_cast<float>(width);
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const T* xr = x + r * width;
    float c[NV][V];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
        load_row<T, V>(xr, i, c[j]);
#pragma unroll
        for (int k = 0; k < V; ++k) s += c[j][k];
      }
    }
    const float mean = warp_sum(s) * inv_w;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (lane + 32 * j < nv)
#pragma unroll
        for (int k = 0; k < V; ++k) q += (c[j][k] - mean) * (c[j][k] - mean);
    const float rstd = rsqrtf(warp_sum(q) * inv_w + eps);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
        float g[V], b[V];
        if (gamma != nullptr) load_row<T, V>(gamma, i, g);
        if (beta != nullptr) load_row<T, V>(beta, i, b);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          float v = (c[j][k] - mean) * rstd;
          if (gamma != nullptr) v *= g[k];
          if (beta != nullptr) v += b[k];
          c[j][k] = v;
        }
        store_row<T, V>(y + r * width, i, c[j]);
      }
    }
  }
}

template <typename T, int V, int NV>
__global__ void __launch_bounds__(256) softmax_cached_kernel(const T* __restrict__ x,
                                                             T* __restrict__ y, int64_t rows,
                                                             int64_t width, float alpha,
                                                             const uint8_t* __restrict__ mask,
                                                             float fill) {
  const int lane = threadIdx.x % 32;
  const int nv = static_cast<int>(width / V);
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const T* xr = x + r * width;
    const uint8_t* mr = mask != nullptr ? mask + r * width : nullptr;
    float c[NV][V];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
        load_row<T, V>(xr, i, c[j]);
        pre_op<V>(c[j], mr, i, alpha, fill);
#pragma unroll
        for (int k = 0; k < V; ++k) m = fmaxf(m, c[j][k]);
      }
    }
    m = warp_max(m);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (lane + 32 * j < nv)
#pragma unroll
        for (int k = 0; k < V; ++k) {
          c[j][k] = __expf(c[j][k] - m);
          s += c[j][k];
        }
    const float inv = 1.f / warp_sum(s);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
#pragma unroll
        for (int k = 0; k < V; ++k) c[j][k] *= inv;
        store_row<T, V>(y + r * width, i, c[j]);
      }
    }
  }
}

// ---- software-pipelined row kernels ------------------------------------------
// A warp per row, the row held in registers as raw 16-byte vectors (4 regs per
// 8 bf16 / 4 fp32 elements, unpacked to fp32 on use), and the NEXT row's loads
// issued before the current row's reductions: every warp keeps a row of reads
// in flight through its whole compute phase. The r01 row-cached kernels
// stalled on long_scoreboard with half the warps resident (fp32 row registers
// limit occupancy), so HBM saw a bubble per row.
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ldg_stream8(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_stream4(const void* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// No "memory" clobber: volatile asm keeps these stores in program order with
// the volatile prefetch loads, while ordinary loads (gamma / beta, L1 hits)
// may still be scheduled across them instead of serialising behind each store.
__device__ __forceinline__ void stg16(void* p, const uint4& v);
__device__ __forceinline__ void stg16_cs(void* p, const uint4& v) {  // streaming (evict-first)
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w));
}
// Output sinks of the row functions: 0 st.global, 1 st.global.cs
// (evict-first), 2 the streamed kernel's shared-memory slab (stored to HBM
// by a TMA bulk store).
__device__ __forceinline__ void stg16(void* p, const uint4& v, int sink) {
  if (sink == 2) *reinterpret_cast<uint4*>(p) = v;
  else if (sink == 1) stg16_cs(p, v);
  else stg16(p, v);
}
__device__ __forceinline__ void stg16(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w));
}

__device__ __forceinline__ float ex2_ftz(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

template <typename T>
struct Raw;  // 16-byte vector <-> fp32
template <>
struct Raw<__nv_bfloat16> {
  static constexpr int V = 8;
  using Mask = uint2;  // 8 mask bytes
  __device__ static void unpack(const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  __device__ static uint4 pack(const float (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ static Mask load_mask(const uint8_t* p) { return ldg_stream8(p); }
  __device__ static float mask_at(const Mask& m, int k) {
    return static_cast<float>(((k < 4 ? m.x : m.y) >> (8 * (k & 3))) & 0xFFu);
  }
};
template <>
struct Raw<float> {
  static constexpr int V = 4;
  using Mask = uint32_t;  // 4 mask bytes
  __device__ static void unpack(const uint4& u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
  }
  __device__ static uint4 pack(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
  __device__ static Mask load_mask(const uint8_t* p) { return ldg_stream4(p); }
  __device__ static float mask_at(const Mask& m, int k) {
    return static_cast<float>((m >> (8 * k)) & 0xFFu);
  }
};

// ---- per-row math, shared by the prefetching register kernels and the
// TMA-streamed ones (identical arithmetic, so either engine's output is the
// same bytes). A warp owns one row held as NV raw 16-byte vectors per lane.

// softmax(alpha * x + fill * mask) of one row of width <= 32 * NV * V.
template <typename T, int NV, bool kMask>
__device__ __forceinline__ void softmax_row(const uint4 (&cur)[NV],
                                            const typename Raw<T>::Mask (&mc)[NV], int lane,
                                            int nv, float alpha, float fill, T* __restrict__ yrow,
                                            int cs = 0) {
  using R = Raw<T>;
  constexpr int V = R::V;
  float f[NV][V];
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (lane + 32 * j < nv) {
      R::unpack(cur[j], f[j]);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if constexpr (kMask) f[j][k] = fmaf(alpha, f[j][k], fill * R::mask_at(mc[j], k));
        else f[j][k] *= alpha;
        m = fmaxf(m, f[j][k]);
      }
    }
  m = warp_max(m);
  const float ml = m * 1.4426950408889634f;
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (lane + 32 * j < nv)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        f[j][k] = ex2_ftz(fmaf(f[j][k], 1.4426950408889634f, -ml));
        s += f[j][k];
      }
  const float inv = 1.f / warp_sum(s);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i = lane + 32 * j;
    if (i < nv) {
#pragma unroll
      for (int k = 0; k < V; ++k) f[j][k] *= inv;
      stg16(yrow + static_cast<int64_t>(i) * V, R::pack(f[j]), cs);
    }
  }
}

// Shared-memory slot of parameter element c in the lane-interleaved fp32
// layout load_param<.., true> reads (V elements per 16-byte vector i; vector
// i belongs to lane i % 32).
template <int V>
__device__ __forceinline__ int64_t gb_index(int64_t c) {
  const int64_t i = c / V, k = c % V;
  return (((i >> 5) * (V / 4) + k / 4) * 32 + (i & 31)) * 4 + (k & 3);
}

// gamma / beta of vector i: the bf16 / fp32 parameter in global memory
// (kGB32 = false) or its fp32 copy staged in shared memory (kGB32 = true);
// the same fp32 values either way.
template <typename T, int V, bool kGB32>
__device__ __forceinline__ void load_param(const void* p, int i, float (&f)[V]) {
  if constexpr (kGB32) {
    // staged lane-interleaved (gb_index): a warp's float4 loads are contiguous,
    // so each LDS.128 is conflict-free
    const float* q = static_cast<const float*>(p);
#pragma unroll
    for (int u = 0; u < V / 4; ++u) {
      const float4 v =
          *reinterpret_cast<const float4*>(q + ((((i >> 5) * (V / 4) + u) << 5) + (i & 31)) * 4);
      f[4 * u] = v.x;
      f[4 * u + 1] = v.y;
      f[4 * u + 2] = v.z;
      f[4 * u + 3] = v.w;
    }
  } else {
    load_row<T, V>(static_cast<const T*>(p), i, f);
  }
}

// layernorm of one row; two-pass mean / variance from the registers (the
// same arithmetic as ln_bwd_row, so backward's recomputed statistics equal
// forward's bit for bit). The row is unpacked to fp32 once and normalised
// in FMA form, y = x * (rstd g) + (b - mean rstd g): three FP32 ops per
// element where (x - mean) * rstd * g + b took four plus two re-unpacks --
// the streamed kernel is issue-bound (ncu r02: issue slots 75% busy).
template <typename T, int NV, bool kGB32, bool kKeepF32>
__device__ __forceinline__ void ln_row(const uint4 (&cur)[NV], int lane, int nv, float inv_w,
                                       float eps, const void* __restrict__ gamma,
                                       const void* __restrict__ beta, T* __restrict__ yrow,
                                       int cs = 0) {
  using R = Raw<T>;
  constexpr int V = R::V;
  // kKeepF32: the row unpacked once and kept in fp32 registers (streamed
  // kernel, registers to spare); else re-unpacked per pass (prefetch kernel,
  // whose occupancy is its registers). Unpacking is exact: same bytes.
  float keep[kKeepF32 ? NV : 1][V];
  auto row = [&](int j, float (&f)[V]) {
    if constexpr (kKeepF32) {
#pragma unroll
      for (int k = 0; k < V; ++k) f[k] = keep[j][k];
    } else {
      R::unpack(cur[j], f);
    }
  };
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (lane + 32 * j < nv) {
      float f[V];
      R::unpack(cur[j], f);
      if constexpr (kKeepF32) {
#pragma unroll
        for (int k = 0; k < V; ++k) keep[j][k] = f[k];
      }
#pragma unroll
      for (int k = 0; k < V; ++k) s += f[k];
    }
  const float mean = warp_sum(s) * inv_w;
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (lane + 32 * j < nv) {
      float f[V];
      row(j, f);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float c = f[k] - mean;
        q += c * c;
      }
    }
  const float rstd = rsqrtf(warp_sum(q) * inv_w + eps);
  const float nm = -mean;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i = lane + 32 * j;
    if (i < nv) {
      float f[V], g[V], b[V];
      row(j, f);
      if (gamma != nullptr) load_param<T, V, kGB32>(gamma, i, g);
      if (beta != nullptr) load_param<T, V, kGB32>(beta, i, b);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float a = gamma != nullptr ? rstd * g[k] : rstd;
        const float c = fmaf(nm, a, beta != nullptr ? b[k] : 0.f);
        f[k] = fmaf(f[k], a, c);
      }
      stg16(yrow + static_cast<int64_t>(i) * V, R::pack(f), cs);
    }
  }
}

// layernorm backward of one row: dx and (lane 0) the row's (mean, rstd),
// computed exactly as ln_row does.
template <typename T, int NV, bool kGB32>
__device__ __forceinline__ void ln_bwd_row(const uint4 (&cx)[NV], const uint4 (&cd)[NV], int lane,
                                           int nv, float inv_w, float eps,
                                           const void* __restrict__ gamma, T* __restrict__ dxrow,
                                           float2* __restrict__ stat, int cs = 0) {
  using R = Raw<T>;
  constexpr int V = R::V;
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (lane + 32 * j < nv) {
      float f[V];
      R::unpack(cx[j], f);
#pragma unroll
      for (int k = 0; k < V; ++k) s += f[k];
    }
  const float mean = warp_sum(s) * inv_w;
  float q = 0.f, sa = 0.f, sax = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (lane + 32 * j < nv) {
      float f[V], d[V], g[V];
      R::unpack(cx[j], f);
      R::unpack(cd[j], d);
      if (gamma != nullptr) load_param<T, V, kGB32>(gamma, lane + 32 * j, g);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float c = f[k] - mean;
        const float gd = gamma != nullptr ? g[k] * d[k] : d[k];
        q += c * c;
        sa += gd;
        sax += gd * c;
      }
    }
  const float rstd = rsqrtf(warp_sum(q) * inv_w + eps);
  const float a = warp_sum(sa) * inv_w;
  const float b = rstd * warp_sum(sax) * inv_w;  // mean(g.dy.xhat)
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i = lane + 32 * j;
    if (i < nv) {
      float f[V], d[V], g[V];
      R::unpack(cx[j], f);
      R::unpack(cd[j], d);
      if (gamma != nullptr) load_param<T, V, kGB32>(gamma, i, g);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float gd = gamma != nullptr ? g[k] * d[k] : d[k];
        f[k] = rstd * (gd - a - (f[k] - mean) * rstd * b);
      }
      stg16(dxrow + static_cast<int64_t>(i) * V, R::pack(f), cs);
    }
  }
  if (lane == 0 && stat != nullptr) *stat = make_float2(mean, rstd);
}

// ---- prefetching register kernels: the NEXT row's loads issued before the
// current row's reductions.

// softmax(alpha * x + fill * mask) over rows of width <= 32 * NV * V.
template <typename T, int NV, bool kMask>
__global__ void __launch_bounds__(256) softmax_pipe_kernel(const T* __restrict__ x,
                                                           T* __restrict__ y, int64_t rows,
                                                           int64_t width, float alpha,
                                                           const uint8_t* __restrict__ mask,
                                                           float fill) {
  using R = Raw<T>;
  constexpr int V = R::V;
  const int lane = threadIdx.x % 32;
  const int nv = static_cast<int>(width / V);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x / 32;
  int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  uint4 cur[NV], nxt[NV];
  typename R::Mask mc[NV], mn[NV];
  auto load = [&](int64_t row, uint4 (&d)[NV], typename R::Mask (&m)[NV]) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
        d[j] = ldg_stream(x + row * width + static_cast<int64_t>(i) * V);
        if constexpr (kMask) m[j] = R::load_mask(mask + row * width + static_cast<int64_t>(i) * V);
      }
    }
  };
  if (r < rows) load(r, cur, mc);
  for (; r < rows; r += stride) {
    if (r + stride < rows) load(r + stride, nxt, mn);
    softmax_row<T, NV, kMask>(cur, mc, lane, nv, alpha, fill, y + r * width);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      cur[j] = nxt[j];
      if constexpr (kMask) mc[j] = mn[j];
    }
  }
}

// layernorm forward, rows of width <= 32 * NV * V.
template <typename T, int NV>
__global__ void __launch_bounds__(256) layernorm_pipe_kernel(
    const T* __restrict__ x, const T* __restrict__ gamma, const T* __restrict__ beta,
    T* __restrict__ y, int64_t rows, int64_t width, float eps) {
  using R = Raw<T>;
  constexpr int V = R::V;
  const int lane = threadIdx.x % 32;
  const int nv = static_cast<int>(width / V);
  const float inv_w = 1.f / static_cast<float>(width);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x / 32;
  int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  uint4 cur[NV], nxt[NV];
  auto load = [&](int64_t row, uint4 (&d)[NV]) {
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (lane + 32 * j < nv) d[j] = ldg_stream(x + row * width + static_cast<int64_t>(lane + 32 * j) * V);
  };
  if (r < rows) load(r, cur);
  for (; r < rows; r += stride) {
    if (r + stride < rows) load(r + stride, nxt);
    ln_row<T, NV, false, false>(cur, lane, nv, inv_w, eps, gamma, beta, y + r * width);
#pragma unroll
    for (int j = 0; j < NV; ++j) cur[j] = nxt[j];
  }
}

// layernorm backward (dx and the per-row statistics for the parameter pass),
// x and dy of the next row prefetched.
template <typename T, int NV>
__global__ void __launch_bounds__(256) layernorm_bwd_pipe_kernel(
    const T* __restrict__ x, const T* __restrict__ gamma, const T* __restrict__ dy,
    T* __restrict__ dx, float2* __restrict__ stats, int64_t rows, int64_t width, float eps) {
  using R = Raw<T>;
  constexpr int V = R::V;
  const int lane = threadIdx.x % 32;
  const int nv = static_cast<int>(width / V);
  const float inv_w = 1.f / static_cast<float>(width);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x / 32;
  int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  uint4 cx[NV], cd[NV], nx[NV], nd[NV];
  auto load = [&](int64_t row, uint4 (&a)[NV], uint4 (&b)[NV]) {
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (lane + 32 * j < nv) {
        const int64_t o = row * width + static_cast<int64_t>(lane + 32 * j) * V;
        a[j] = ldg_stream(x + o);
        b[j] = ldg_stream(dy + o);
      }
  };
  if (r < rows) load(r, cx, cd);
  for (; r < rows; r += stride) {
    if (r + stride < rows) load(r + stride, nx, nd);
    ln_bwd_row<T, NV, false>(cx, cd, lane, nv, inv_w, eps, gamma, dx + r * width,
                      stats != nullptr ? stats + r : nullptr);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      cx[j] = nx[j];
      cd[j] = nd[j];
    }
  }
}

// ---- TMA-streamed row kernels -------------------------------------------------
// The register-prefetch kernels keep one row per warp in flight, so their
// bytes in flight are capped by registers (occupancy): the layernorm pair
// measured 0.74 / 0.72 of the HBM roofline with it (r02). Here the loads
// leave the register file: a producer warp streams slabs of kRsRows
// contiguous rows (every input of the row op: x, dy, the u8 mask) into a
// ring of shared-memory stages with cp.async.bulk (one bulk copy per input
// per slab, completion counted on the stage's mbarrier), and kRsRows
// consumer warps each take one row of the slab from shared memory, free the
// stage, and run the same per-row math, storing straight to HBM. Bytes in
// flight per SM = resident CTAs x stages x slab bytes, independent of the
// math's register footprint.
constexpr int kRsRows = 8;            // consumer warps = rows per slab
constexpr int kRsMaxStages = 8;
constexpr int kRsBudget = 72 * 1024;  // stage ring per CTA: 3 CTAs per SM

enum RowOp { kRowLn = 0, kRowSoftmax = 1, kRowMaskedSoftmax = 2, kRowLnBwd = 3 };

struct RowStreamArgs {
  const void* in0;      // x (layernorm, softmax) / x (layernorm backward)
  const void* in1;      // dy (layernorm backward)
  const uint8_t* mask;  // u8 mask (masked softmax)
  const void* gamma;
  const void* beta;
  void* out;
  float2* stats;
  int64_t rows, width;
  float eps, alpha, fill;
  int stages;
  uint32_t row0, row1, rowm;      // bytes per row of each input (0: absent)
  uint32_t off1, offm, stage;     // offsets inside a stage, stage bytes
  uint32_t params;                // bytes of fp32 gamma + beta staged before the ring
  int policy;                     // bit 0: evict-first bulk loads; bit 1: streaming stores
};

__device__ __forceinline__ void rs_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void rs_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                        bool evict_first) {
  if (evict_first) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
        "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))), "l"(pol)
        : "memory");
    return;
  }
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}

// kTS = false: consumers store their rows with st.global and free the stage
// right after reading it. kTS = true: consumers write the result over their
// input row in shared memory and a storer warp writes the slab back with one
// cp.async.bulk store (TMA both ways, like the bulk copy engine); the stage
// is freed once that store has read it.
// Position in the stage ring (slot, mbarrier phase), advanced per slab
// without integer division.
struct RsRing {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++s == n) {
      s = 0;
      ph ^= 1u;
    }
  }
};

template <typename T, int NV, int kOp, int kMinBlocks, bool kTS>
__global__ void __launch_bounds__(32 * (kRsRows + 1 + kTS), kMinBlocks)
    row_stream_kernel(const __grid_constant__ RowStreamArgs a) {
  using R = Raw<T>;
  constexpr int V = R::V;
  extern __shared__ __align__(128) uint8_t rs_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(rs_smem);
  uint64_t* empty = full + kRsMaxStages;
  uint64_t* done = empty + kRsMaxStages;  // kTS: consumers -> storer
  // [barriers 256 B][fp32 gamma][fp32 beta][stage ring]
  float* g32 = reinterpret_cast<float*>(rs_smem + 256);
  float* b32 = g32 + (a.width / V + 31) / 32 * 32 * V;  // gb_index spans whole lane groups
  uint8_t* data = rs_smem + 256 + a.params;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t slabs = (a.rows + kRsRows - 1) / kRsRows;
  if constexpr (kOp == kRowLn || kOp == kRowLnBwd) {
    for (int64_t c = threadIdx.x; c < a.width; c += blockDim.x) {
      if (a.gamma != nullptr) g32[gb_index<V>(c)] = ld(static_cast<const T*>(a.gamma) + c);
      if (a.beta != nullptr) b32[gb_index<V>(c)] = ld(static_cast<const T*>(a.beta) + c);
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&full[s])))
                   : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&empty[s]))),
                   "r"(kTS ? 1 : kRsRows)
                   : "memory");
      if constexpr (kTS)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&done[s]))),
                     "r"(kRsRows)
                     : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kRsRows) {  // producer
    if (lane == 0) {
      RsRing ring;
      for (int64_t slab = blockIdx.x; slab < slabs; slab += gridDim.x, ring.next(a.stages)) {
        const int s = ring.s;
        rs_wait(&empty[s], ring.ph ^ 1);
        const int64_t r0 = slab * kRsRows;
        const int64_t left = a.rows - r0;
        const uint32_t nr = static_cast<uint32_t>(left < kRsRows ? left : kRsRows);
        uint8_t* st = data + static_cast<size_t>(s) * a.stage;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&full[s]))),
                     "r"(nr * (a.row0 + a.row1 + a.rowm))
                     : "memory");
        const bool ef = a.policy & 1;
        rs_bulk(st, static_cast<const uint8_t*>(a.in0) + r0 * a.row0, nr * a.row0, &full[s], ef);
        if (a.row1)
          rs_bulk(st + a.off1, static_cast<const uint8_t*>(a.in1) + r0 * a.row1, nr * a.row1,
                  &full[s], ef);
        if (a.rowm) rs_bulk(st + a.offm, a.mask + r0 * a.rowm, nr * a.rowm, &full[s], ef);
      }
    }
    return;
  }
  if constexpr (kTS) {
    if (warp == kRsRows + 1) {  // storer: slab s back to HBM, then free its stage
      if (lane == 0) {
        RsRing ring;
        int prev = -1;
        for (int64_t slab = blockIdx.x; slab < slabs; slab += gridDim.x, ring.next(a.stages)) {
          const int s = ring.s;
          rs_wait(&done[s], ring.ph);
          const int64_t r0 = slab * kRsRows;
          const int64_t left = a.rows - r0;
          const uint32_t nr = static_cast<uint32_t>(left < kRsRows ? left : kRsRows);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                           static_cast<uint8_t*>(a.out) + r0 * a.row0),
                       "r"(static_cast<uint32_t>(
                           __cvta_generic_to_shared(data + static_cast<size_t>(s) * a.stage))),
                       "r"(nr * a.row0)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          // at most this slab's store still reading shared memory: the previous
          // slab's stage is free
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          if (prev >= 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(&empty[prev])))
                         : "memory");
          prev = s;
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
      return;
    }
  }
  const int nv = static_cast<int>(a.width / V);
  const float inv_w = 1.f / static_cast<float>(a.width);
  RsRing ring;
  for (int64_t slab = blockIdx.x; slab < slabs; slab += gridDim.x, ring.next(a.stages)) {
    const int s = ring.s;
    rs_wait(&full[s], ring.ph);
    const int64_t r = slab * kRsRows + warp;
    const bool live = r < a.rows;
    uint8_t* st = data + static_cast<size_t>(s) * a.stage;
    uint4 c0[NV], c1[NV];
    typename R::Mask mc[NV];
    if (live) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int i = lane + 32 * j;
        if (i < nv) {
          c0[j] = *reinterpret_cast<const uint4*>(st + warp * a.row0 + i * 16);
          if constexpr (kOp == kRowLnBwd)
            c1[j] = *reinterpret_cast<const uint4*>(st + a.off1 + warp * a.row1 + i * 16);
          if constexpr (kOp == kRowMaskedSoftmax)
            mc[j] = *reinterpret_cast<const typename R::Mask*>(st + a.offm + warp * a.rowm +
                                                              i * sizeof(typename R::Mask));
        }
      }
    }
    if constexpr (!kTS) {
      // the row is in registers: release the stage to the producer
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&empty[s])))
                     : "memory");
      if (!live) continue;
    }
    if (live) {
      // kTS: the result overwrites this warp's input row in the stage
      T* out = kTS ? reinterpret_cast<T*>(st + warp * a.row0) : static_cast<T*>(a.out) + r * a.width;
      const int sink = kTS ? 2 : ((a.policy & 2) ? 1 : 0);
      if constexpr (kOp == kRowLn) {
        ln_row<T, NV, true, true>(c0, lane, nv, inv_w, a.eps, a.gamma != nullptr ? g32 : nullptr,
                                  a.beta != nullptr ? b32 : nullptr, out, sink);
      } else if constexpr (kOp == kRowLnBwd) {
        ln_bwd_row<T, NV, true>(c0, c1, lane, nv, inv_w, a.eps,
                                a.gamma != nullptr ? g32 : nullptr, out,
                                a.stats != nullptr ? a.stats + r : nullptr, sink);
      } else {
        softmax_row<T, NV, kOp == kRowMaskedSoftmax>(c0, mc, lane, nv, a.alpha, a.fill, out,
                                                     sink);
      }
    }
    if constexpr (kTS) {
      // generic-proxy writes -> visible to the bulk store (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&done[s])))
                     : "memory");
    }
  }
}
// softmax backward, y and dy of the next row prefetched.
template <typename T, int NV>
__global__ void __launch_bounds__(256) softmax_bwd_pipe_kernel(const T* __restrict__ y,
                                                               const T* __restrict__ dy,
                                                               T* __restrict__ dx, int64_t rows,
                                                               int64_t width, float alpha) {
  using R = Raw<T>;
  constexpr int V = R::V;
  const int lane = threadIdx.x % 32;
  const int nv = static_cast<int>(width / V);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x / 32;
  int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  uint4 cy[NV], cd[NV], ny[NV], nd[NV];
  auto load = [&](int64_t row, uint4 (&a)[NV], uint4 (&b)[NV]) {
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (lane + 32 * j < nv) {
        const int64_t o = row * width + static_cast<int64_t>(lane + 32 * j) * V;
        a[j] = ldg_stream(y + o);
        b[j] = ldg_stream(dy + o);
      }
  };
  if (r < rows) load(r, cy, cd);
  for (; r < rows; r += stride) {
    if (r + stride < rows) load(r + stride, ny, nd);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (lane + 32 * j < nv) {
        float a[V], d[V];
        R::unpack(cy[j], a);
        R::unpack(cd[j], d);
#pragma unroll
        for (int k = 0; k < V; ++k) s += a[k] * d[k];
      }
    s = warp_sum(s);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
        float a[V], d[V];
        R::unpack(cy[j], a);
        R::unpack(cd[j], d);
#pragma unroll
        for (int k = 0; k < V; ++k) a[k] = alpha * a[k] * (d[k] - s);
        stg16(dx + r * width + static_cast<int64_t>(i) * V, R::pack(a));
      }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      cy[j] = ny[j];
      cd[j] = nd[j];
    }
  }
}


// ---- general transpose (any permutation) and softmax over any axis ----------
// The graph format's transpose carries an arbitrary `perm` and softmax an
// `axis` (graph_ir.cpp:270-290); the block plans only use the last-two swap
// and the last axis (the kernels above), these cover the rest.

constexpr int kMaxPermDims = 8;
struct PermArgs {
  int rank;
  int64_t out_shape[kMaxPermDims];   // output extents
  int64_t in_stride[kMaxPermDims];   // input element stride of output dim d (x dim perm[d])
  int64_t out_stride[kMaxPermDims];  // output element strides (row-major)
};

// perm[r-1] == r-1: the last dim stays innermost, so each output row is one
// contiguous input row -- a warp copies it (16-byte vectors when aligned).
template <typename W>
__global__ void __launch_bounds__(256) permute_rows_kernel(const W* __restrict__ x,
                                                           W* __restrict__ y, int64_t rows,
                                                           int64_t row_words,
                                                           const __grid_constant__ PermArgs a) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * blockDim.x / 32;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += warps) {
    int64_t rem = r, in_off = 0;  // a.in_stride in W words
    for (int d = a.rank - 2; d >= 0; --d) {  // output coordinates of row r, minor first
      const int64_t c = rem % a.out_shape[d];
      rem /= a.out_shape[d];
      in_off += c * a.in_stride[d];
    }
    const W* from = x + in_off;
    W* to = y + r * row_words;
    for (int64_t i = lane; i < row_words; i += 32) to[i] = from[i];
  }
}

// General case: the input's last dim (contiguous in x) and input dim q =
// perm[r-1] (contiguous in y) form a 32 x 32 shared-memory tile, so reads
// are coalesced along x's last dim and writes along y's; every other dim
// is a batch index. a.in_stride / a.out_stride here are indexed by INPUT dim.
template <typename E>
__global__ void __launch_bounds__(256) permute_tile_kernel(const E* __restrict__ x,
                                                           E* __restrict__ y, int q, int last,
                                                           int64_t nq, int64_t nl, int64_t batch,
                                                           const __grid_constant__ PermArgs a) {
  __shared__ E tile[32][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  const int64_t tiles_l = (nl + 31) / 32, tiles_q = (nq + 31) / 32;
  for (int64_t t = blockIdx.x; t < batch * tiles_q * tiles_l; t += gridDim.x) {
    int64_t b = t / (tiles_q * tiles_l);
    const int64_t tt = t % (tiles_q * tiles_l);
    const int64_t q0 = (tt / tiles_l) * 32, l0 = (tt % tiles_l) * 32;
    // batch index over the input dims other than q and last, minor first
    int64_t in_base = 0, out_base = 0;
    for (int d = a.rank - 1; d >= 0; --d) {
      if (d == q || d == last) continue;
      const int64_t c = b % a.out_shape[d];  // out_shape holds INPUT extents here
      b /= a.out_shape[d];
      in_base += c * a.in_stride[d];
      out_base += c * a.out_stride[d];
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
      const int64_t qi = q0 + i, li = l0 + tx;
      if (qi < nq && li < nl) tile[i][tx] = x[in_base + qi * a.in_stride[q] + li];
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
      const int64_t li = l0 + i, qi = q0 + tx;
      if (qi < nq && li < nl) y[out_base + li * a.out_stride[last] + qi] = tile[tx][i];
    }
  }
}

// softmax over the middle dim of [outer, len, inner] (inner > 1): a thread per
// (outer, inner) column, consecutive threads on consecutive inner indices so
// every pass is coalesced; one online max/sum pass, one normalising pass.
template <typename T>
__global__ void __launch_bounds__(256) softmax_axis_kernel(const T* __restrict__ x,
                                                           T* __restrict__ y, int64_t outer,
                                                           int64_t len, int64_t inner) {
  const int64_t cols = outer * inner;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cols;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = c / inner, i = c % inner;
    const T* xc = x + o * len * inner + i;
    T* yc = y + o * len * inner + i;
    float m = -INFINITY, s = 0.f;
    for (int64_t k = 0; k < len; ++k) {
      const float v = ld(xc + k * inner);
      const float nm = fmaxf(m, v);
      s = s * __expf(m - nm) + __expf(v - nm);
      m = nm;
    }
    const float inv = 1.f / s;
    for (int64_t k = 0; k < len; ++k) st(yc + k * inner, __expf(ld(xc + k * inner) - m) * inv);
  }
}

// its backward from the output: dx = alpha * y * (dy - sum_k dy * y)
template <typename T>
__global__ void __launch_bounds__(256) softmax_axis_bwd_kernel(const T* __restrict__ y,
                                                               const T* __restrict__ dy,
                                                               T* __restrict__ dx, int64_t outer,
                                                               int64_t len, int64_t inner,
                                                               float alpha) {
  const int64_t cols = outer * inner;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cols;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t base = (c / inner) * len * inner + c % inner;
    float s = 0.f;
    for (int64_t k = 0; k < len; ++k) s += ld(y + base + k * inner) * ld(dy + base + k * inner);
    for (int64_t k = 0; k < len; ++k) {
      const int64_t o = base + k * inner;
      st(dx + o, alpha * ld(y + o) * (ld(dy + o) - s));
    }
  }
}

// ---- backward ---------------------------------------------------------------
// layernorm: dx = rstd * (g.dy - mean(g.dy) - xhat * mean(g.dy.xhat)), warp per
// row: one pass for the four row sums (mean / rstd recomputed from x, kept per
// row for the column pass), one for dx;
// dgamma += sum_rows dy.xhat, dbeta += sum_rows dy in a second, column pass.
template <typename T, int V>
__global__ void __launch_bounds__(256) layernorm_bwd_kernel(
    const T* __restrict__ x, const T* __restrict__ gamma, const T* __restrict__ dy,
    T* __restrict__ dx, float2* __restrict__ stats, int64_t rows, int64_t width, float eps) {
  const int lane = threadIdx.x % 32;
  const int64_t nv = width / V;
  const float inv_w = 1.f / static_cast<float>(width);
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const T* xr = x + r * width;
    const T* gr = dy + r * width;
    // one pass over (x, dy) for all four row sums: sum x, sum x^2, sum g.dy,
    // sum g.dy.x (mean / var / the two projections follow from them)
    float sx = 0.f, sxx = 0.f, sa = 0.f, sax = 0.f;
    for (int64_t i = lane; i < nv; i += 32) {
      float f[V], d[V], g[V];
      load_row<T, V>(xr, i, f);
      load_row<T, V>(gr, i, d);
      if (gamma != nullptr) load_row<T, V>(gamma, i, g);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float gd = gamma != nullptr ? g[k] * d[k] : d[k];
        sx += f[k];
        sxx += f[k] * f[k];
        sa += gd;
        sax += gd * f[k];
      }
    }
    const float mean = warp_sum(sx) * inv_w;
    const float var = fmaxf(warp_sum(sxx) * inv_w - mean * mean, 0.f);
    const float rstd = rsqrtf(var + eps);
    const float a = warp_sum(sa) * inv_w;
    const float b = rstd * (warp_sum(sax) * inv_w - mean * a);  // mean(g.dy.xhat)
    for (int64_t i = lane; i < nv; i += 32) {
      float f[V], d[V], g[V];
      load_row<T, V>(xr, i, f);
      load_row<T, V>(gr, i, d);
      if (gamma != nullptr) load_row<T, V>(gamma, i, g);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float gd = gamma != nullptr ? g[k] * d[k] : d[k];
        f[k] = rstd * (gd - a - (f[k] - mean) * rstd * b);
      }
      store_row<T, V>(dx + r * width, i, f);
    }
    if (lane == 0 && stats != nullptr) stats[r] = make_float2(mean, rstd);
  }
}

// dgamma[c] += sum_r dy[r,c] * xhat[r,c], dbeta[c] += sum_r dy[r,c]: a 32-column
// strip per warp lane group, row chunks across blockIdx.y, partials per chunk.
template <typename T>
__global__ void __launch_bounds__(256) layernorm_param_grad_kernel(
    const T* __restrict__ x, const T* __restrict__ dy, const float2* __restrict__ stats,
    float* __restrict__ part, int64_t rows, int64_t width, int64_t rows_per_chunk) {
  const int64_t c = blockIdx.x * 32 + threadIdx.x;
  const int64_t r0 = blockIdx.y * rows_per_chunk;
  const int64_t r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
  float sg = 0.f, sb = 0.f;
  if (c < width)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += blockDim.y) {
      const float2 st = stats[r];
      const float d = ld(dy + r * width + c);
      sg += d * (ld(x + r * width + c) - st.x) * st.y;
      sb += d;
    }
  __shared__ float red[2][8][33];
  red[0][threadIdx.y][threadIdx.x] = sg;
  red[1][threadIdx.y][threadIdx.x] = sb;
  __syncthreads();
  if (threadIdx.y == 0 && c < width) {
    for (int j = 1; j < blockDim.y; ++j) {
      sg += red[0][j][threadIdx.x];
      sb += red[1][j][threadIdx.x];
    }
    // per-chunk partials, summed in chunk order by the next kernel: no
    // atomics, so the parameter gradients are bit-reproducible
    part[blockIdx.y * width + c] = sg;
    part[(gridDim.y + blockIdx.y) * width + c] = sb;
  }
}

__global__ void __launch_bounds__(256) layernorm_param_reduce_kernel(
    const float* __restrict__ part, int64_t chunks, int64_t width, float* __restrict__ dgamma,
    float* __restrict__ dbeta) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= width) return;
  float sg = 0.f, sb = 0.f;
  for (int64_t j = 0; j < chunks; ++j) {
    sg += part[j * width + c];
    sb += part[(chunks + j) * width + c];
  }
  if (dgamma != nullptr) dgamma[c] += sg;
  if (dbeta != nullptr) dbeta[c] += sb;
}

int64_t layernorm_param_chunks(int64_t rows, int64_t width) {
  const int64_t strips = (width + 31) / 32;
  return std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64, (148 * 8 + strips - 1) / strips));
}

// softmax: dx = alpha * y * (dy - sum(dy * y)) per row (alpha: the fused
// attention scale's chain rule; 1 for a plain softmax)
template <typename T, int V>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const T* __restrict__ y,
                                                          const T* __restrict__ dy,
                                                          T* __restrict__ dx, int64_t rows,
                                                          int64_t width, float alpha) {
  const int lane = threadIdx.x % 32;
  const int64_t nv = width / V;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const T* yr = y + r * width;
    const T* gr = dy + r * width;
    float s = 0.f;
    for (int64_t i = lane; i < nv; i += 32) {
      float a[V], d[V];
      load_row<T, V>(yr, i, a);
      load_row<T, V>(gr, i, d);
#pragma unroll
      for (int k = 0; k < V; ++k) s += a[k] * d[k];
    }
    s = warp_sum(s);
    for (int64_t i = lane; i < nv; i += 32) {
      float a[V], d[V];
      load_row<T, V>(yr, i, a);
      load_row<T, V>(gr, i, d);
#pragma unroll
      for (int k = 0; k < V; ++k) a[k] = alpha * a[k] * (d[k] - s);
      store_row<T, V>(dx + r * width, i, a);
    }
  }
}

// ---- embedding backward: deterministic, id-sorted -------------------------
// dtable[id, :] += sum of dy[t, :] over the tokens t with ids[t] == id.
// Instead of fp32 atomics (whose summation order -- and so the bytes --
// changes run to run when ids repeat), every (source e, token t) gets the
// unique key (id << 32 | e * n + t); a radix sort groups the keys by id with
// the tokens in ascending order, and one warp per distinct id sums its tokens
// in that order and updates the row once. The result is bit-reproducible.
// The same path serves the fused reduce-scatter form (an owner's block of
// vocab rows [v0, v0 + rows) x columns [c0, c0 + cols), sources from every
// device); ids outside the block get a sentinel key that sorts last.
struct EmbSources {
  const int64_t* ids[kMaxBlocks];
  const void* dy[kMaxBlocks];
};

__global__ void __launch_bounds__(256) embedding_keys_kernel(const __grid_constant__ EmbSources src,
                                                             int nsrc, int64_t n, int64_t v0,
                                                             int64_t rows,
                                                             uint64_t* __restrict__ keys) {
  const int64_t total = static_cast<int64_t>(nsrc) * n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(i / n);
    const int64_t id = __ldg(src.ids[e] + (i - e * n)) - v0;
    keys[i] = (id >= 0 && id < rows) ? (static_cast<uint64_t>(id) << 32) | static_cast<uint64_t>(i)
                                     : ~uint64_t{0};
  }
}

template <typename T>
__global__ void __launch_bounds__(256) embedding_accum_kernel(
    const uint64_t* __restrict__ keys, int64_t m, const __grid_constant__ EmbSources src,
    int64_t n, int64_t dy_width, float* __restrict__ dblock, int64_t rows, int64_t c0,
    int64_t cols) {
  const int lane = threadIdx.x % 32;
  for (int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const uint64_t k = keys[p];
    const int64_t id = static_cast<int64_t>(k >> 32);
    if (id >= rows) continue;                             // sentinel (outside the block)
    if (p > 0 && (keys[p - 1] >> 32) == k >> 32) continue;  // not the first token of its id
    int64_t q_end = p + 1;
    while (q_end < m && (keys[q_end] >> 32) == k >> 32) ++q_end;
    float* out = dblock + id * cols;
    for (int64_t c = lane; c < cols; c += 32) {
      float acc = 0.f;
      for (int64_t q = p; q < q_end; ++q) {  // tokens in ascending (source, token) order
        const int64_t i = static_cast<int64_t>(keys[q] & 0xffffffffu);
        const int e = static_cast<int>(i / n);
        acc += ld(static_cast<const T*>(src.dy[e]) + (i - e * n) * dy_width + c0 + c);
      }
      out[c] += acc;
    }
  }
}

// Vectorised transpose: 64 x 64 element tiles, every global access a 16-byte
// vector along a row (input rows on the way in, output rows on the way out);
// the shared tile is padded by one 4-byte word per row against bank conflicts.
template <typename W>
__global__ void __launch_bounds__(256) transpose_vec_kernel(const W* __restrict__ x,
                                                            W* __restrict__ y, int64_t batch,
                                                            int R, int C) {
  constexpr int E = 16 / sizeof(W);  // elements per vector
  constexpr int T = 64;
  constexpr int PAD = sizeof(W) >= 4 ? 1 : 4 / sizeof(W);
  __shared__ W tile[T][T + PAD];
  const int c0 = blockIdx.x * T, r0 = blockIdx.y * T;
  constexpr int VPR = T / E;  // vectors per tile row
  for (int64_t b = blockIdx.z; b < batch; b += gridDim.z) {
    const W* xb = x + b * R * static_cast<int64_t>(C);
    W* yb = y + b * R * static_cast<int64_t>(C);
    for (int v = threadIdx.x; v < T * VPR; v += blockDim.x) {
      const int i = v / VPR, j = (v % VPR) * E;  // tile row, first column
      const int r = r0 + i, c = c0 + j;
      if (r < R && c < C) {
        const Vec<W, E> in = *reinterpret_cast<const Vec<W, E>*>(xb + static_cast<int64_t>(r) * C + c);
#pragma unroll
        for (int k = 0; k < E; ++k) tile[i][j + k] = in.v[k];
      }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < T * VPR; v += blockDim.x) {
      const int i = v / VPR, j = (v % VPR) * E;  // output tile row (= input column), first col
      const int c = c0 + i, r = r0 + j;
      if (c < C && r < R) {
        Vec<W, E> out;
#pragma unroll
        for (int k = 0; k < E; ++k) out.v[k] = tile[j + k][i];
        *reinterpret_cast<Vec<W, E>*>(yb + static_cast<int64_t>(c) * R + r) = out;
      }
    }
    __syncthreads();
  }
}

// ---- elementwise ----------------------------------------------------------
// y = alpha * x
template <typename T, int V>
__global__ void __launch_bounds__(256) scale_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                    int64_t nv, float alpha) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float f[V];
    load_row<T, V>(x, i, f);
#pragma unroll
    for (int k = 0; k < V; ++k) f[k] *= alpha;
    store_row<T, V>(y, i, f);
  }
}

// y = a + alpha * b, b of the same type or a u8 mask (B = uint8_t)
template <typename T, typename B, int V>
__global__ void __launch_bounds__(256) add_kernel(const T* __restrict__ a, const B* __restrict__ b,
                                                  T* __restrict__ y, int64_t nv, float alpha) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float f[V];
    load_row<T, V>(a, i, f);
    const Vec<B, V> bv = reinterpret_cast<const Vec<B, V>*>(b)[i];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float g;
      if constexpr (sizeof(B) == 1) g = static_cast<float>(bv.v[k]);
      else g = ld(&bv.v[k]);
      f[k] += alpha * g;
    }
    store_row<T, V>(y, i, f);
  }
}

__global__ void __launch_bounds__(256) not_kernel(const uint8_t* __restrict__ x,
                                                  uint8_t* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = x[i] == 0 ? 1 : 0;
}

int grid_for(int64_t threads) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((threads + 255) / 256, 148 * 16)));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

cudaError_t done() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Grid of a prefetching row kernel: exactly the CTAs that are resident at
// once (SMs x occupancy), so every warp walks many rows with its prefetch
// always in flight instead of paying an unhidden first-row load per short
// CTA lifetime; never more warps than rows.
template <typename... Args>
int pipe_grid(void (*kernel)(Args...), int64_t rows) {
  static std::mutex mu;
  static std::map<const void*, int> occ_of;
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  int occ;
  {
    std::lock_guard<std::mutex> hold(mu);
    auto it = occ_of.find(reinterpret_cast<const void*>(kernel));
    if (it == occ_of.end()) {
      int o = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, 256, 0) != cudaSuccess || o < 1)
        o = 1;
      it = occ_of.emplace(reinterpret_cast<const void*>(kernel), o).first;
    }
    occ = it->second;
  }
  const int64_t need = (rows * 32 + 255) / 256;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t{sms} * occ)));
}

// APL_ROW_PIPE=0 selects the r01 row kernels (A/B of the prefetching ones).
bool pipe_rows_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("APL_ROW_PIPE");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

// Row engine per op (r02 measurements, 128 Ki rows x 1024 bf16, fraction of
// the HBM copy peak, profiles/r02_block_ops_*.jsonl): layernorm 0.80 streamed
// vs 0.73 register-prefetch, its backward 0.84 vs 0.71, masked softmax 0.87
// vs 0.82 -- the streamed kernel wins where the row math's registers cap
// the prefetch kernel's bytes in flight; plain softmax 0.80 vs 0.92 -- there
// the prefetch kernel's occupancy suffices and it pays no barrier traffic.
// APL_ROW_ENGINE=stream / pipe forces one engine for every op (A/B, tests).
int row_engine_forced() {  // -1 policy, 0 pipe, 1 stream
  static const int v = [] {
    const char* e = std::getenv("APL_ROW_ENGINE");
    if (e == nullptr) return -1;
    if (std::strcmp(e, "pipe") == 0) return 0;
    if (std::strcmp(e, "stream") == 0) return 1;
    return -1;
  }();
  return v;
}
bool row_stream_enabled(bool plain_softmax = false) {
  const int f = row_engine_forced();
  return f < 0 ? !plain_softmax : f == 1;
}

constexpr uint32_t align128(uint32_t v) { return (v + 127u) & ~127u; }

// One TMA-streamed row launch; cudaErrorNotSupported when the slab does not
// fit two stages (the caller falls back to the register kernels).
template <typename T, int NV, int kOp, bool kTS>
cudaError_t launch_row_stream(RowStreamArgs a, cudaStream_t s) {
  // layernorm keeps its row in fp32 registers: 2 CTAs per SM (<= 113 regs)
  constexpr int kMin = (kTS || kOp == kRowLn || (kOp == kRowLnBwd && NV >= 4)) ? 2 : 3;
  constexpr int kThreads = 32 * (kRsRows + 1 + kTS);
  auto kern = row_stream_kernel<T, NV, kOp, kMin, kTS>;
  a.off1 = align128(kRsRows * a.row0);
  a.offm = align128(a.off1 + kRsRows * a.row1);
  a.stage = align128(a.offm + kRsRows * a.rowm);
  static const int budget = [] {  // APL_RS_BUDGET_KB: stage-ring bytes per CTA (probe)
    const char* e = std::getenv("APL_RS_BUDGET_KB");
    return e ? std::max(16, std::min(200, std::atoi(e))) * 1024 : kRsBudget;
  }();
  a.stages = std::min<int>(kRsMaxStages, budget / static_cast<int>(a.stage));
  if (a.stages < 2) return cudaErrorNotSupported;
  static const int policy = [] {  // APL_RS_POLICY: cache-policy probe bits (see RowStreamArgs)
    const char* e = std::getenv("APL_RS_POLICY");
    return e ? std::atoi(e) : 0;
  }();
  a.policy = policy;
  constexpr int kV = 16 / static_cast<int>(sizeof(T));
  a.params = (kOp == kRowLn || kOp == kRowLnBwd)
                 ? align128(static_cast<uint32_t>(2 * ((a.width / kV + 31) / 32 * 32 * kV) *
                                                  sizeof(float)))
                 : 0u;
  const int smem = 256 + static_cast<int>(a.params) + a.stages * static_cast<int>(a.stage);
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ_of;
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  int occ;
  {
    std::lock_guard<std::mutex> hold(mu);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kern), smem);
    auto it = occ_of.find(key);
    if (it == occ_of.end()) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           std::min(227 * 1024, 256 + 8192 + std::max(budget, kRsBudget)));
      int o = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, smem) !=
              cudaSuccess ||
          o < 1)
        o = 1;
      it = occ_of.emplace(key, o).first;
    }
    occ = it->second;
  }
  const int64_t slabs = (a.rows + kRsRows - 1) / kRsRows;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(slabs, int64_t{sms} * occ)));
  kern<<<grid, kThreads, smem, s>>>(a);
  return cudaSuccess;
}

// Store path of the streamed kernel per op (r02, fraction of the HBM copy
// peak): softmax / masked softmax write back with TMA bulk stores (0.92 /
// 0.93 vs 0.79 / 0.89 with st.global); layernorm and its backward with
// st.global (0.78 / 0.92 vs 0.73-0.74 / 0.89), whose longer row math holds a
// TMA-store stage too long. APL_RS_STORE=tma / stg forces one (A/B, tests).
bool row_stream_tma_store(int op) {
  static const int forced = [] {
    const char* e = std::getenv("APL_RS_STORE");
    if (e == nullptr) return -1;
    return std::strcmp(e, "stg") == 0 ? 0 : std::strcmp(e, "tma") == 0 ? 1 : -1;
  }();
  return forced >= 0 ? forced == 1 : (op == kRowSoftmax || op == kRowMaskedSoftmax);
}

template <typename T, int kOp>
cudaError_t row_stream_nv(int nv, const RowStreamArgs& a, cudaStream_t s) {
  if (row_stream_tma_store(kOp)) {
    if (nv == 1) return launch_row_stream<T, 1, kOp, true>(a, s);
    if (nv == 2) return launch_row_stream<T, 2, kOp, true>(a, s);
    return launch_row_stream<T, 4, kOp, true>(a, s);
  }
  if (nv == 1) return launch_row_stream<T, 1, kOp, false>(a, s);
  if (nv == 2) return launch_row_stream<T, 2, kOp, false>(a, s);
  return launch_row_stream<T, 4, kOp, false>(a, s);
}

// Streams rows of <= 4 16-byte vectors per lane; the inputs must be 16-byte
// aligned with 16-byte rows (the mask's rows too).
template <typename T>
cudaError_t row_stream(int op, int nv, const RowStreamArgs& a, cudaStream_t s) {
  switch (op) {
    case kRowLn: return row_stream_nv<T, kRowLn>(nv, a, s);
    case kRowSoftmax: return row_stream_nv<T, kRowSoftmax>(nv, a, s);
    case kRowMaskedSoftmax: return row_stream_nv<T, kRowMaskedSoftmax>(nv, a, s);
    default: return row_stream_nv<T, kRowLnBwd>(nv, a, s);
  }
}

struct SoftmaxPre {
  float alpha = 1.f;
  const uint8_t* mask = nullptr;
  float fill = 0.f;
};

template <typename T, int V, int NV>
void rowwise_cached(bool softmax, const T* X, const T* G, const T* B, T* Y, int64_t rows,
                    int64_t width, float eps, const SoftmaxPre& p, int grid, cudaStream_t s) {
  if (softmax)
    softmax_cached_kernel<T, V, NV><<<grid, 256, 0, s>>>(X, Y, rows, width, p.alpha, p.mask,
                                                         p.fill);
  else layernorm_cached_kernel<T, V, NV><<<grid, 256, 0, s>>>(X, G, B, Y, rows, width, eps);
}

template <typename T>
cudaError_t rowwise(bool softmax, const void* x, const void* g, const void* b, void* y,
                    int64_t rows, int64_t width, float eps, cudaStream_t s,
                    const SoftmaxPre& p = SoftmaxPre{}) {
  constexpr int V = 16 / sizeof(T);
  const bool vec = width % V == 0 && aligned16(x) && aligned16(y) && (!g || aligned16(g)) &&
                   (!b || aligned16(b)) && reinterpret_cast<uintptr_t>(p.mask) % V == 0;
  const int grid = grid_for(rows * 32);
  auto X = static_cast<const T*>(x);
  auto Y = static_cast<T*>(y);
  auto G = static_cast<const T*>(g);
  auto B = static_cast<const T*>(b);
  const int64_t per_lane = vec ? (width / V + 31) / 32 : 0;  // vectors each lane holds
  if (per_lane >= 1 && per_lane <= 4 && row_stream_enabled(softmax && p.mask == nullptr) &&
      (p.mask == nullptr || (width % 16 == 0 && aligned16(p.mask)))) {
    const bool masked = p.mask != nullptr;
    RowStreamArgs a{};
    a.in0 = x;
    a.mask = p.mask;
    a.gamma = g;
    a.beta = b;
    a.out = y;
    a.rows = rows;
    a.width = width;
    a.eps = eps;
    a.alpha = p.alpha;
    a.fill = p.fill;
    a.row0 = static_cast<uint32_t>(width * sizeof(T));
    a.rowm = masked ? static_cast<uint32_t>(width) : 0u;
    const int op = !softmax ? kRowLn : masked ? kRowMaskedSoftmax : kRowSoftmax;
    const int nv = per_lane == 1 ? 1 : per_lane == 2 ? 2 : 4;
    if (row_stream<T>(op, nv, a, s) != cudaErrorNotSupported) return done();
  }
  if (per_lane >= 1 && per_lane <= 4 && pipe_rows_enabled()) {
    const bool masked = p.mask != nullptr;
    const int nv = per_lane == 1 ? 1 : per_lane == 2 ? 2 : 4;
#define APL_ROW_PIPE(NVC)                                                                    \
    if (!softmax)                                                                            \
      layernorm_pipe_kernel<T, NVC><<<pipe_grid(layernorm_pipe_kernel<T, NVC>, rows), 256, 0,  \
                                      s>>>(X, G, B, Y, rows, width, eps);                      \
    else if (masked)                                                                         \
      softmax_pipe_kernel<T, NVC, true><<<pipe_grid(softmax_pipe_kernel<T, NVC, true>, rows),  \
                                          256, 0, s>>>(X, Y, rows, width, p.alpha, p.mask,     \
                                                       p.fill);                                \
    else                                                                                     \
      softmax_pipe_kernel<T, NVC, false><<<pipe_grid(softmax_pipe_kernel<T, NVC, false>, rows), \
                                           256, 0, s>>>(X, Y, rows, width, p.alpha, nullptr,   \
                                                        0.f);
    if (nv == 1) { APL_ROW_PIPE(1) }
    else if (nv == 2) { APL_ROW_PIPE(2) }
    else { APL_ROW_PIPE(4) }
#undef APL_ROW_PIPE
    return done();
  }
  if (per_lane >= 1 && per_lane <= 8) {
    if (per_lane == 1) rowwise_cached<T, V, 1>(softmax, X, G, B, Y, rows, width, eps, p, grid, s);
    else if (per_lane == 2) rowwise_cached<T, V, 2>(softmax, X, G, B, Y, rows, width, eps, p, grid, s);
    else if (per_lane <= 4) rowwise_cached<T, V, 4>(softmax, X, G, B, Y, rows, width, eps, p, grid, s);
    else rowwise_cached<T, V, 8>(softmax, X, G, B, Y, rows, width, eps, p, grid, s);
    return done();
  }
  if (softmax) {
    if (vec) softmax_kernel<T, V><<<grid, 256, 0, s>>>(X, Y, rows, width, p.alpha, p.mask, p.fill);
    else softmax_kernel<T, 1><<<grid, 256, 0, s>>>(X, Y, rows, width, p.alpha, p.mask, p.fill);
  } else {
    if (vec) layernorm_kernel<T, V><<<grid, 256, 0, s>>>(X, G, B, Y, rows, width, eps);
    else layernorm_kernel<T, 1><<<grid, 256, 0, s>>>(X, G, B, Y, rows, width, eps);
  }
  return done();
}

template <typename T>
cudaError_t scale_typed(const void* x, void* y, size_t count, float alpha, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const int64_t n = static_cast<int64_t>(count);
  if (n % V == 0 && aligned16(x) && aligned16(y))
    scale_kernel<T, V><<<grid_for(n / V), 256, 0, s>>>(static_cast<const T*>(x), static_cast<T*>(y),
                                                       n / V, alpha);
  else
    scale_kernel<T, 1><<<grid_for(n), 256, 0, s>>>(static_cast<const T*>(x), static_cast<T*>(y), n,
                                                   alpha);
  return done();
}

template <typename T>
cudaError_t add_typed(const void* a, const void* b, bool b_mask, void* y, size_t count, float alpha,
                      cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const int64_t n = static_cast<int64_t>(count);
  // a u8 operand moves V bytes per access: keep it 4-byte aligned at least
  const bool vec = n % V == 0 && aligned16(a) && aligned16(y) &&
                   (b_mask ? (reinterpret_cast<uintptr_t>(b) % V == 0) : aligned16(b));
  auto A = static_cast<const T*>(a);
  auto Y = static_cast<T*>(y);
  if (b_mask) {
    auto Bm = static_cast<const uint8_t*>(b);
    if (vec) add_kernel<T, uint8_t, V><<<grid_for(n / V), 256, 0, s>>>(A, Bm, Y, n / V, alpha);
    else add_kernel<T, uint8_t, 1><<<grid_for(n), 256, 0, s>>>(A, Bm, Y, n, alpha);
  } else {
    auto Bt = static_cast<const T*>(b);
    if (vec) add_kernel<T, T, V><<<grid_for(n / V), 256, 0, s>>>(A, Bt, Y, n / V, alpha);
    else add_kernel<T, T, 1><<<grid_for(n), 256, 0, s>>>(A, Bt, Y, n, alpha);
  }
  return done();
}

}  // namespace

cudaError_t launch_embedding(const int64_t* ids, int64_t n, const void* table, int64_t vocab,
                             int64_t width, int elem_bytes, void* out, cudaStream_t s) {
  if (n == 0 || width == 0) return cudaSuccess;
  const int64_t row = width * elem_bytes;
  if (row % 16 == 0 && aligned16(table) && aligned16(out))
    embedding_kernel<uint4><<<grid_for(n * row / 16), 256, 0, s>>>(
        ids, n, static_cast<const uint4*>(table), vocab, row / 16, static_cast<uint4*>(out));
  else if (row % 4 == 0 && reinterpret_cast<uintptr_t>(table) % 4 == 0 &&
           reinterpret_cast<uintptr_t>(out) % 4 == 0)
    embedding_kernel<uint32_t><<<grid_for(n * row / 4), 256, 0, s>>>(
        ids, n, static_cast<const uint32_t*>(table), vocab, row / 4, static_cast<uint32_t*>(out));
  else
    embedding_kernel<uint8_t><<<grid_for(n * row), 256, 0, s>>>(
        ids, n, static_cast<const uint8_t*>(table), vocab, row, static_cast<uint8_t*>(out));
  return done();
}

cudaError_t launch_embedding_blocks(const int64_t* ids, int64_t n, const void* const* blocks,
                                    int vocab_blocks, int hidden_blocks, int64_t vocab,
                                    int64_t width, int64_t col_begin, int64_t cols,
                                    int elem_bytes, void* out, cudaStream_t s) {
  if (n == 0 || cols == 0) return cudaSuccess;
  if (vocab_blocks < 1 || hidden_blocks < 1 || vocab_blocks * hidden_blocks > kMaxBlocks ||
      vocab % vocab_blocks || width % hidden_blocks)
    return cudaErrorInvalidValue;
  TableBlocks tb{};
  uintptr_t align = reinterpret_cast<uintptr_t>(out);
  for (int i = 0; i < vocab_blocks * hidden_blocks; ++i) {
    tb.p[i] = blocks[i];
    align |= reinterpret_cast<uintptr_t>(blocks[i]);
  }
  const int64_t vb_rows = vocab / vocab_blocks;
  const int64_t hb = width / hidden_blocks * elem_bytes, c0 = col_begin * elem_bytes,
                nc = cols * elem_bytes;
  // the widest word every block row, the output slice and all bases divide
  int wb = 16;
  while (wb > 1 && ((hb | c0 | nc) % wb || align % wb)) wb >>= 1;
  switch (wb) {
    case 16:
      embedding_blocks_kernel<uint4><<<grid_for(n * 32), 256, 0, s>>>(
          ids, n, tb, hidden_blocks, vb_rows, hb / 16, vocab, c0 / 16, nc / 16,
          static_cast<uint4*>(out));
      break;
    case 8:
      embedding_blocks_kernel<uint2><<<grid_for(n * 32), 256, 0, s>>>(
          ids, n, tb, hidden_blocks, vb_rows, hb / 8, vocab, c0 / 8, nc / 8,
          static_cast<uint2*>(out));
      break;
    case 4:
      embedding_blocks_kernel<uint32_t><<<grid_for(n * 32), 256, 0, s>>>(
          ids, n, tb, hidden_blocks, vb_rows, hb / 4, vocab, c0 / 4, nc / 4,
          static_cast<uint32_t*>(out));
      break;
    case 2:
      embedding_blocks_kernel<uint16_t><<<grid_for(n * 32), 256, 0, s>>>(
          ids, n, tb, hidden_blocks, vb_rows, hb / 2, vocab, c0 / 2, nc / 2,
          static_cast<uint16_t*>(out));
      break;
    default:
      embedding_blocks_kernel<uint8_t><<<grid_for(n * 32), 256, 0, s>>>(
          ids, n, tb, hidden_blocks, vb_rows, hb, vocab, c0, nc, static_cast<uint8_t*>(out));
      break;
  }
  return done();
}

cudaError_t launch_layernorm(const void* x, const void* gamma, const void* beta, void* y,
                             int64_t rows, int64_t width, float eps, int dtype, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  if (dtype == 0) return rowwise<float>(false, x, gamma, beta, y, rows, width, eps, s);
  if (dtype == 1) return rowwise<__nv_bfloat16>(false, x, gamma, beta, y, rows, width, eps, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_softmax(const void* x, void* y, int64_t rows, int64_t width, float alpha,
                           const void* mask, float fill, int dtype, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  SoftmaxPre p;
  p.alpha = alpha;
  p.mask = static_cast<const uint8_t*>(mask);
  p.fill = fill;
  if (dtype == 0) return rowwise<float>(true, x, nullptr, nullptr, y, rows, width, 0.f, s, p);
  if (dtype == 1)
    return rowwise<__nv_bfloat16>(true, x, nullptr, nullptr, y, rows, width, 0.f, s, p);
  return cudaErrorInvalidValue;
}

cudaError_t launch_permute(const void* x, void* y, int rank, const int64_t* shape,
                           const int64_t* perm, int elem_bytes, cudaStream_t s) {
  int64_t numel = 1;
  for (int d = 0; d < rank; ++d) numel *= shape[d];
  if (numel == 0) return cudaSuccess;
  int64_t in_stride[kMaxPermDims];  // row-major element strides of x
  in_stride[rank - 1] = 1;
  for (int d = rank - 2; d >= 0; --d) in_stride[d] = in_stride[d + 1] * shape[d + 1];
  PermArgs a{};
  a.rank = rank;
  const int last = rank - 1;
  if (perm[last] == last) {  // rows stay contiguous: a row copy
    for (int d = 0; d < rank; ++d) {
      a.out_shape[d] = shape[perm[d]];
      a.in_stride[d] = in_stride[perm[d]];
    }
    const int64_t row_bytes = shape[last] * elem_bytes, rows = numel / shape[last];
    const bool v16 = row_bytes % 16 == 0 && aligned16(x) && aligned16(y);
    const int w = v16 ? 16 : elem_bytes;
    for (int d = 0; d < rank; ++d) a.in_stride[d] = a.in_stride[d] * elem_bytes / w;
    const int grid = grid_for(rows * 32);
    switch (w) {
      case 16: permute_rows_kernel<uint4><<<grid, 256, 0, s>>>(static_cast<const uint4*>(x), static_cast<uint4*>(y), rows, row_bytes / 16, a); break;
      case 8: permute_rows_kernel<uint64_t><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(x), static_cast<uint64_t*>(y), rows, row_bytes / 8, a); break;
      case 4: permute_rows_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(x), static_cast<uint32_t*>(y), rows, row_bytes / 4, a); break;
      case 2: permute_rows_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(x), static_cast<uint16_t*>(y), rows, row_bytes / 2, a); break;
      default: permute_rows_kernel<uint8_t><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(x), static_cast<uint8_t*>(y), rows, row_bytes, a); break;
    }
    return done();
  }
  // tile case: strides indexed by INPUT dim; out_shape carries input extents
  int64_t out_dim_stride[kMaxPermDims];  // row-major strides of y
  out_dim_stride[rank - 1] = 1;
  for (int d = rank - 2; d >= 0; --d) out_dim_stride[d] = out_dim_stride[d + 1] * shape[perm[d + 1]];
  for (int d = 0; d < rank; ++d) {
    a.out_shape[d] = shape[d];
    a.in_stride[d] = in_stride[d];
  }
  for (int d = 0; d < rank; ++d) a.out_stride[perm[d]] = out_dim_stride[d];
  const int q = static_cast<int>(perm[last]);
  const int64_t nq = shape[q], nl = shape[last], batch = numel / (nq * nl);
  const int64_t tiles = batch * ((nq + 31) / 32) * ((nl + 31) / 32);
  const int grid = static_cast<int>(std::min<int64_t>(tiles, int64_t{sm_count()} * 16));
  switch (elem_bytes) {
    case 1: permute_tile_kernel<uint8_t><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(x), static_cast<uint8_t*>(y), q, last, nq, nl, batch, a); break;
    case 2: permute_tile_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(x), static_cast<uint16_t*>(y), q, last, nq, nl, batch, a); break;
    case 4: permute_tile_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(x), static_cast<uint32_t*>(y), q, last, nq, nl, batch, a); break;
    default: permute_tile_kernel<uint64_t><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(x), static_cast<uint64_t*>(y), q, last, nq, nl, batch, a); break;
  }
  return done();
}

cudaError_t launch_softmax_axis(const void* x, void* y, int64_t outer, int64_t len, int64_t inner,
                                int dtype, cudaStream_t s) {
  if (outer * len * inner == 0) return cudaSuccess;
  const int grid = grid_for(outer * inner);
  if (dtype == 0)
    softmax_axis_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x),
                                                    static_cast<float*>(y), outer, len, inner);
  else
    softmax_axis_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), outer, len, inner);
  return done();
}

cudaError_t launch_softmax_axis_backward(const void* y, const void* dy, void* dx, int64_t outer,
                                         int64_t len, int64_t inner, float alpha, int dtype,
                                         cudaStream_t s) {
  if (outer * len * inner == 0) return cudaSuccess;
  const int grid = grid_for(outer * inner);
  if (dtype == 0)
    softmax_axis_bwd_kernel<float><<<grid, 256, 0, s>>>(
        static_cast<const float*>(y), static_cast<const float*>(dy), static_cast<float*>(dx),
        outer, len, inner, alpha);
  else
    softmax_axis_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(y), static_cast<const __nv_bfloat16*>(dy),
        static_cast<__nv_bfloat16*>(dx), outer, len, inner, alpha);
  return done();
}

cudaError_t launch_transpose(const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
                             int elem_bytes, cudaStream_t s) {
  if (batch == 0 || rows == 0 || cols == 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32),
                  static_cast<unsigned>(std::min<int64_t>(batch, 65535)));
  const dim3 block(32, 8);
  const int R = static_cast<int>(rows), C = static_cast<int>(cols);
  // whole 16-byte vectors along both input and output rows
  const int E = 16 / elem_bytes;
  if (elem_bytes <= 8 && rows % E == 0 && cols % E == 0 && aligned16(x) && aligned16(y)) {
    const dim3 g(static_cast<unsigned>((cols + 63) / 64), static_cast<unsigned>((rows + 63) / 64),
                 static_cast<unsigned>(std::min<int64_t>(batch, 65535)));
    switch (elem_bytes) {
      case 1:
        transpose_vec_kernel<uint8_t><<<g, 256, 0, s>>>(static_cast<const uint8_t*>(x),
                                                        static_cast<uint8_t*>(y), batch, R, C);
        break;
      case 2:
        transpose_vec_kernel<uint16_t><<<g, 256, 0, s>>>(static_cast<const uint16_t*>(x),
                                                         static_cast<uint16_t*>(y), batch, R, C);
        break;
      case 4:
        transpose_vec_kernel<uint32_t><<<g, 256, 0, s>>>(static_cast<const uint32_t*>(x),
                                                         static_cast<uint32_t*>(y), batch, R, C);
        break;
      default:
        transpose_vec_kernel<uint64_t><<<g, 256, 0, s>>>(static_cast<const uint64_t*>(x),
                                                         static_cast<uint64_t*>(y), batch, R, C);
        break;
    }
    return done();
  }
  switch (elem_bytes) {
    case 1:
      transpose_kernel<uint8_t><<<grid, block, 0, s>>>(static_cast<const uint8_t*>(x),
                                                       static_cast<uint8_t*>(y), batch, R, C);
      break;
    case 2:
      transpose_kernel<uint16_t><<<grid, block, 0, s>>>(static_cast<const uint16_t*>(x),
                                                        static_cast<uint16_t*>(y), batch, R, C);
      break;
    case 4:
      transpose_kernel<uint32_t><<<grid, block, 0, s>>>(static_cast<const uint32_t*>(x),
                                                        static_cast<uint32_t*>(y), batch, R, C);
      break;
    case 8:
      transpose_kernel<uint64_t><<<grid, block, 0, s>>>(static_cast<const uint64_t*>(x),
                                                        static_cast<uint64_t*>(y), batch, R, C);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return done();
}

cudaError_t launch_scale(const void* x, void* y, size_t count, float alpha, int dtype,
                         cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (dtype == 0) return scale_typed<float>(x, y, count, alpha, s);
  if (dtype == 1) return scale_typed<__nv_bfloat16>(x, y, count, alpha, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_add(const void* a, const void* b, bool b_mask, void* y, size_t count,
                       float alpha, int dtype, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (dtype == 0) return add_typed<float>(a, b, b_mask, y, count, alpha, s);
  if (dtype == 1) return add_typed<__nv_bfloat16>(a, b, b_mask, y, count, alpha, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_mask_not(const void* x, void* y, size_t count, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  const int64_t n = static_cast<int64_t>(count);
  not_kernel<<<grid_for(n), 256, 0, s>>>(static_cast<const uint8_t*>(x), static_cast<uint8_t*>(y),
                                         n);
  return done();
}

namespace {

template <typename T>
cudaError_t layernorm_bwd_typed(const void* x, const void* gamma, const void* dy, void* dx,
                                float* dgamma, float* dbeta, float2* stats, int64_t rows,
                                int64_t width, float eps, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const bool vec = width % V == 0 && aligned16(x) && aligned16(dy) && aligned16(dx) &&
                   (!gamma || aligned16(gamma));
  const int grid = grid_for(rows * 32);
  auto X = static_cast<const T*>(x);
  auto G = static_cast<const T*>(gamma);
  auto D = static_cast<const T*>(dy);
  auto O = static_cast<T*>(dx);
  // rows of up to 4 vectors per lane: the prefetching register kernel (raw
  // 16-byte vectors keep its occupancy up; the r01 fp32-register variant
  // halved it and measured 0.54 of the roofline); longer rows stream.
  const int64_t per_lane = vec ? (width / V + 31) / 32 : 0;
  bool streamed = false;
  if (per_lane >= 1 && per_lane <= 4 && row_stream_enabled()) {
    RowStreamArgs a{};
    a.in0 = x;
    a.in1 = dy;
    a.gamma = gamma;
    a.out = dx;
    a.stats = stats;
    a.rows = rows;
    a.width = width;
    a.eps = eps;
    a.row0 = a.row1 = static_cast<uint32_t>(width * sizeof(T));
    const int nv = per_lane == 1 ? 1 : per_lane == 2 ? 2 : 4;
    streamed = row_stream<T>(kRowLnBwd, nv, a, s) != cudaErrorNotSupported;
  }
  if (streamed) {
  } else if (per_lane >= 1 && per_lane <= 4 && pipe_rows_enabled()) {
    if (per_lane == 1)
      layernorm_bwd_pipe_kernel<T, 1><<<pipe_grid(layernorm_bwd_pipe_kernel<T, 1>, rows), 256, 0,
                                        s>>>(X, G, D, O, stats, rows, width, eps);
    else if (per_lane == 2)
      layernorm_bwd_pipe_kernel<T, 2><<<pipe_grid(layernorm_bwd_pipe_kernel<T, 2>, rows), 256, 0,
                                        s>>>(X, G, D, O, stats, rows, width, eps);
    else
      layernorm_bwd_pipe_kernel<T, 4><<<pipe_grid(layernorm_bwd_pipe_kernel<T, 4>, rows), 256, 0,
                                        s>>>(X, G, D, O, stats, rows, width, eps);
  } else if (vec) {
    layernorm_bwd_kernel<T, V><<<grid, 256, 0, s>>>(X, G, D, O, stats, rows, width, eps);
  } else {
    layernorm_bwd_kernel<T, 1><<<grid, 256, 0, s>>>(X, G, D, O, stats, rows, width, eps);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (dgamma != nullptr || dbeta != nullptr) {
    const int64_t strips = (width + 31) / 32;
    const int64_t chunks = layernorm_param_chunks(rows, width);
    const int64_t per = (rows + chunks - 1) / chunks;
    // partials live after the per-row stats in the scratch (16-byte aligned)
    float* part = reinterpret_cast<float*>(stats + ((rows + 1) / 2) * 2);
    layernorm_param_grad_kernel<T><<<dim3(static_cast<unsigned>(strips),
                                          static_cast<unsigned>(chunks)),
                                     dim3(32, 8), 0, s>>>(X, D, stats, part, rows, width, per);
    layernorm_param_reduce_kernel<<<static_cast<unsigned>((width + 255) / 256), 256, 0, s>>>(
        part, chunks, width, dgamma, dbeta);
    g_launches.fetch_add(2, std::memory_order_relaxed);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t softmax_bwd_typed(const void* y, const void* dy, void* dx, int64_t rows,
                              int64_t width, float alpha, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  const bool vec = width % V == 0 && aligned16(y) && aligned16(dy) && aligned16(dx);
  const int grid = grid_for(rows * 32);
  auto Y = static_cast<const T*>(y);
  auto D = static_cast<const T*>(dy);
  auto O = static_cast<T*>(dx);
  const int64_t per_lane = vec ? (width / V + 31) / 32 : 0;
  if (per_lane >= 1 && per_lane <= 4 && pipe_rows_enabled()) {
    if (per_lane == 1)
      softmax_bwd_pipe_kernel<T, 1><<<pipe_grid(softmax_bwd_pipe_kernel<T, 1>, rows), 256, 0, s>>>(
          Y, D, O, rows, width, alpha);
    else if (per_lane == 2)
      softmax_bwd_pipe_kernel<T, 2><<<pipe_grid(softmax_bwd_pipe_kernel<T, 2>, rows), 256, 0, s>>>(
          Y, D, O, rows, width, alpha);
    else
      softmax_bwd_pipe_kernel<T, 4><<<pipe_grid(softmax_bwd_pipe_kernel<T, 4>, rows), 256, 0, s>>>(
          Y, D, O, rows, width, alpha);
  } else if (vec) {
    softmax_bwd_kernel<T, V><<<grid, 256, 0, s>>>(Y, D, O, rows, width, alpha);
  } else {
    softmax_bwd_kernel<T, 1><<<grid, 256, 0, s>>>(Y, D, O, rows, width, alpha);
  }
  return done();
}

}  // namespace

// stats: layernorm_backward_scratch_bytes(rows, width) of scratch -- the
// per-row (mean, rstd) float2s, then the per-chunk parameter partials --
// needed when dgamma / dbeta are requested (apl_layernorm_backward_ex checks
// the size).
cudaError_t launch_layernorm_backward(const void* x, const void* gamma, const void* dy, void* dx,
                                      float* dgamma, float* dbeta, void* stats, int64_t rows,
                                      int64_t width, float eps, int dtype, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  auto st = static_cast<float2*>(stats);
  if (dtype == 0)
    return layernorm_bwd_typed<float>(x, gamma, dy, dx, dgamma, dbeta, st, rows, width, eps, s);
  if (dtype == 1)
    return layernorm_bwd_typed<__nv_bfloat16>(x, gamma, dy, dx, dgamma, dbeta, st, rows, width,
                                              eps, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_softmax_backward(const void* y, const void* dy, void* dx, int64_t rows,
                                    int64_t width, float alpha, int dtype, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  if (dtype == 0) return softmax_bwd_typed<float>(y, dy, dx, rows, width, alpha, s);
  if (dtype == 1) return softmax_bwd_typed<__nv_bfloat16>(y, dy, dx, rows, width, alpha, s);
  return cudaErrorInvalidValue;
}

namespace {

cudaError_t embedding_backward_sorted(const EmbSources& src, int nsrc, int64_t n, int64_t dy_width,
                                      float* dblock, int64_t v0, int64_t rows, int64_t c0,
                                      int64_t cols, int dtype, cudaStream_t s) {
  const int64_t m = static_cast<int64_t>(nsrc) * n;
  if (m >= (int64_t{1} << 32) - 1 || rows >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
  if (dtype != 0 && dtype != 1) return cudaErrorInvalidValue;
  int id_bits = 1;
  while ((int64_t{1} << id_bits) <= rows) ++id_bits;  // the sentinel's id field exceeds rows
  const int end_bit = 32 + id_bits;
  size_t temp = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, temp, static_cast<const uint64_t*>(nullptr),
                                                 static_cast<uint64_t*>(nullptr), m, 0, end_bit, s);
  if (e != cudaSuccess) return e;
  const size_t kb = (static_cast<size_t>(m) * 8 + 255) / 256 * 256;
  void* scratch = nullptr;
  if ((e = cudaMallocAsync(&scratch, 2 * kb + temp, s)) != cudaSuccess) return e;
  uint64_t* k_in = static_cast<uint64_t*>(scratch);
  uint64_t* k_out = reinterpret_cast<uint64_t*>(static_cast<char*>(scratch) + kb);
  void* t = static_cast<char*>(scratch) + 2 * kb;
  embedding_keys_kernel<<<grid_for(m), 256, 0, s>>>(src, nsrc, n, v0, rows, k_in);
  e = cub::DeviceRadixSort::SortKeys(t, temp, k_in, k_out, m, 0, end_bit, s);
  if (e == cudaSuccess) {
    if (dtype == 0)
      embedding_accum_kernel<float><<<grid_for(m * 32), 256, 0, s>>>(k_out, m, src, n, dy_width,
                                                                    dblock, rows, c0, cols);
    else
      embedding_accum_kernel<__nv_bfloat16><<<grid_for(m * 32), 256, 0, s>>>(
          k_out, m, src, n, dy_width, dblock, rows, c0, cols);
  }
  const cudaError_t f = cudaFreeAsync(scratch, s);
  return e != cudaSuccess ? e : f;
}

}  // namespace

cudaError_t launch_embedding_backward(const int64_t* ids, int64_t n, const void* dy,
                                      float* dtable, int64_t vocab, int64_t width, int dtype,
                                      cudaStream_t s) {
  if (n == 0 || width == 0) return cudaSuccess;
  EmbSources src{};
  src.ids[0] = ids;
  src.dy[0] = dy;
  const cudaError_t e =
      embedding_backward_sorted(src, 1, n, width, dtable, 0, vocab, 0, width, dtype, s);
  return e != cudaSuccess ? e : done();
}

cudaError_t launch_embedding_backward_block(const int64_t* const* ids, const void* const* dy,
                                            int nsrc, int64_t n, int64_t dy_width, float* dblock,
                                            int64_t v0, int64_t rows, int64_t c0, int64_t cols,
                                            int dtype, cudaStream_t s) {
  if (nsrc == 0 || n == 0 || rows == 0 || cols == 0) return cudaSuccess;
  if (nsrc > kMaxBlocks) return cudaErrorInvalidValue;
  EmbSources src{};
  for (int i = 0; i < nsrc; ++i) {
    src.ids[i] = ids[i];
    src.dy[i] = dy[i];
  }
  const cudaError_t e =
      embedding_backward_sorted(src, nsrc, n, dy_width, dblock, v0, rows, c0, cols, dtype, s);
  return e != cudaSuccess ? e : done();
}

size_t layernorm_backward_scratch_bytes(int64_t rows, int64_t width) {
  const int64_t chunks = layernorm_param_chunks(rows, width);
  return static_cast<size_t>(((rows + 1) / 2) * 2 * 8 + 2 * chunks * width * 4);
}

}  // namespace apl
