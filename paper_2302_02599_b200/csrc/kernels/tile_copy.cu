// TMA tensor-tile copy engine (sm_100a): the strided box copies whose rows
// are short (64 B .. 2 KiB -- the all-to-all pack/unpack of small inner
// dims, where one cp.async.bulk per row is issue-bound and LDG pays address
// math per 16 bytes) move as 2-D..5-D TMA tiles: one
// cp.async.bulk.tensor load of a [rows x run] box into shared memory, one
// tensor store of the same box per destination. The hardware walks the
// strides; the SMs only pick boxes.
//
// Each descriptor becomes a source tensor map and one map per destination
// (UINT64 elements, dims = [run/8, ext innermost .. outermost], byte strides
// from the descriptor), passed in kernel parameter space together with the
// box grid of every descriptor. One CTA per SM, two warps: lane 0 of warp 0
// loads boxes into a ring of kStages 16 KiB stages (mbarrier complete_tx),
// lane 0 of warp 1 stores them and frees a stage once its shared-memory
// reads are done (bulk wait_group.read). Partial boxes at the edges: TMA
// zero-fills the load and clips the store.
// Roofline: HBM, algorithmic bytes = bytes read once + bytes written.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "tile_copy.cuh"

namespace apl {

extern std::atomic<uint64_t> g_launches;
int sm_count();

namespace {

constexpr int kStages = 12;
constexpr int kSmemBytes = kStages * kTileBoxBytes + 1024;

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.div == 1 ? n : (__umulhi(n, f.mul) >> f.shr);
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}

struct Box {
  int d;        // descriptor
  int c[5];     // element coordinates of the box origin
};

__device__ __forceinline__ void locate(const TileArgs& a, int64_t u, int& cur, Box& b) {
  while (cur + 1 < a.ndesc && a.d[cur + 1].unit_begin <= u) ++cur;
  const TileDesc& t = a.d[cur];
  uint32_t r = static_cast<uint32_t>(u - t.unit_begin);
  b.d = cur;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const uint32_t q = fdiv(r, t.nb[i]);
    const uint32_t k = r - q * t.nb[i].div;
    b.c[i] = static_cast<int>(k) * t.box[i];
    r = q;
  }
}

__device__ __forceinline__ void tile_load(int rank, uint32_t dst, const CUtensorMap* map,
                                          uint32_t bar, const int (&c)[5]) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1])
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2])
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3])
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
          "l"(m), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
          : "memory");
      break;
  }
}

__device__ __forceinline__ void tile_store(int rank, const CUtensorMap* map, uint32_t src,
                                           const int (&c)[5]) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::
                       "l"(m), "r"(src), "r"(c[0]), "r"(c[1])
                   : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
          "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2])
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::
              "l"(m),
          "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3])
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::
              "l"(m),
          "r"(src), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
          : "memory");
      break;
  }
}

__global__ void __launch_bounds__(64, 1) tile_copy_kernel(const __grid_constant__ TileArgs a) {
  extern __shared__ __align__(128) uint8_t raw[];
  uint8_t* stage = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 127) &
                                              ~uintptr_t(127));
  __shared__ uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (lane != 0) return;
  const int64_t step = gridDim.x;
  if (warp == 0) {  // loader
    int cur = 0, i = 0;
    for (int64_t u = a.first + blockIdx.x; u < a.total; u += step, ++i) {
      const int s = i % kStages;
      bar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
      Box b;
      locate(a, u, cur, b);
      const TileDesc& t = a.d[b.d];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       saddr(&full[s])),
                   "r"(t.box_bytes)
                   : "memory");
      tile_load(t.rank, saddr(stage + s * kTileBoxBytes), &a.maps[t.src_map], saddr(&full[s]),
                b.c);
    }
  } else {  // storer
    int cur = 0, i = 0, prev = -1;
    for (int64_t u = a.first + blockIdx.x; u < a.total; u += step, ++i) {
      const int s = i % kStages;
      bar_wait(&full[s], (i / kStages) & 1);
      Box b;
      locate(a, u, cur, b);
      const TileDesc& t = a.d[b.d];
      for (int j = 0; j < t.ndst; ++j)
        tile_store(t.rank, &a.maps[t.dst_map + j], saddr(stage + s * kTileBoxBytes), b.c);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // the previous stage's shared-memory reads are done once at most this
      // stage's group is still reading
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      if (prev >= 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&empty[prev]))
                     : "memory");
      prev = s;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

}  // namespace

int tile_smem_bytes() { return kSmemBytes; }

cudaError_t launch_tile_copy(const TileArgs& args, cudaStream_t stream) {
  if (args.total <= args.first) return cudaSuccess;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tile_copy_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int64_t units = args.total - args.first;
  const int grid = static_cast<int>(std::min<int64_t>(units, sm_count()));
  tile_copy_kernel<<<grid, 64, kSmemBytes, stream>>>(args);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace apl
