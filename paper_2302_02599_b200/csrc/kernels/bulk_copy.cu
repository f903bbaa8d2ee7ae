// TMA bulk copy engine for descriptor tables whose contiguous runs are long
// (>= kBulkMinRun bytes, 16-byte aligned): the SMs only compute addresses,
// the Tensor Memory Accelerator moves the bytes.
//
// Work unit = one segment of <= kBulkSeg bytes of one run (row). A CTA has
// two warps and a ring of kStages stages of 32 segments:
//   warp 0 (loader): lane i resolves unit 32*b+i, issues
//     cp.async.bulk.shared::cluster.global.mbarrier::complete_tx into the
//     stage slot i; lane 0 arms the stage's mbarrier with the batch's bytes;
//   warp 1 (storer): after the mbarrier completes, lane i issues one
//     cp.async.bulk.global.shared::cta per destination of its unit (fan-out
//     descriptors read HBM once and store to every receiver), commits the
//     bulk group and frees the stage once its shared-memory reads finished
//     (cp.async.bulk.wait_group.read).
// Roofline: HBM, algorithmic bytes = bytes read once + bytes written.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "box_copy.cuh"

namespace apl {

extern std::atomic<uint64_t> g_launches;
int sm_count();

namespace {

constexpr int kStages = 3;
constexpr int kStageBytes = 32 * kBulkSeg;
constexpr int kBulkSmemTasks = 64;  // descriptors per launch, staged in smem
constexpr int kTableBytes = kBulkSmemTasks * static_cast<int>(sizeof(DevCopy));
constexpr int kSmemBytes = kTableBytes + kStages * kStageBytes + 128;

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

struct Unit {
  const DevCopy* d;
  int64_t so, dd;
  uint32_t bytes;
};

__device__ __forceinline__ int find_task(const DevCopy* table, int ntasks, int64_t u) {
  int lo = 0, hi = ntasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (table[mid].unit_begin <= u) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Unit u -> descriptor, source/destination byte offsets, segment length.
// `cur` is the lane's descriptor cursor: units only move forward, so only
// the entries after it are searched.
__device__ __forceinline__ bool resolve_unit(const DevCopy* table, int ntasks, int64_t total,
                                             int64_t u, int& cur, Unit& out) {
  if (u >= total) return false;
  if (cur + 1 < ntasks && table[cur + 1].unit_begin <= u)
    cur = cur + 1 + find_task(table + cur + 1, ntasks - cur - 1, u);
  const DevCopy& c = table[cur];
  const uint32_t local = static_cast<uint32_t>(u - c.unit_begin);
  uint32_t row = fdiv(local, c.units_per_run);
  const uint32_t seg = local - row * c.units_per_run.div;
  int64_t so = c.src_off + static_cast<int64_t>(seg) * kBulkSeg;
  int64_t dd = c.dst_off + static_cast<int64_t>(seg) * kBulkSeg;
  for (int i = c.nouter - 1; i >= 0; --i) {
    const uint32_t q = fdiv(row, c.ext[i]);
    const uint32_t r = row - q * c.ext[i].div;
    so += static_cast<int64_t>(r) * c.src_stride[i];
    dd += static_cast<int64_t>(r) * c.dst_stride[i];
    row = q;
  }
  const int64_t left = c.run_bytes - static_cast<int64_t>(seg) * kBulkSeg;
  out.d = &c;
  out.so = so;
  out.dd = dd;
  out.bytes = static_cast<uint32_t>(left < kBulkSeg ? left : kBulkSeg);
  return true;
}

__global__ void __launch_bounds__(64, 1)
    bulk_copy_kernel(const DevCopy* __restrict__ table, int ntasks, int64_t first, int64_t total,
                     int evict_first, const __grid_constant__ PtrTable ptrs) {
  // Shared memory: [descriptor table (this launch's <= kBulkSmemTasks)] [ring].
  // The table is staged once per CTA so unit resolution is a broadcast smem
  // search, not a chain of dependent global loads per batch.
  extern __shared__ __align__(128) uint8_t raw[];
  const DevCopy* tab = reinterpret_cast<const DevCopy*>(raw);
  uint8_t* stage = raw + kTableBytes;
  __shared__ uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  {
    stage_table(table, ntasks, raw);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t batches = (total - first + 31) / 32;
  // Batches go round-robin over the CTAs; a lane's units only move forward,
  // so its descriptor cursor is advanced by a search over later entries.
  int cur = 0;
  if (warp == 0) {  // loader
    int i = 0;
    for (int64_t b = blockIdx.x; b < batches; b += gridDim.x, ++i) {
      const int s = i % kStages;
      bar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
      Unit u;
      const bool ok = resolve_unit(tab, ntasks, total, first + b * 32 + lane, cur, u);
      uint32_t bytes = ok ? u.bytes : 0;
      uint32_t sum = bytes;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         saddr(&full[s])),
                     "r"(sum)
                     : "memory");
      __syncwarp();
      if (ok) {
        const char* src = ptrs.src[u.d->src_buf] + u.so;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(saddr(stage + s * kStageBytes + lane * kBulkSeg)),
            "l"(src), "r"(bytes), "r"(saddr(&full[s]))
            : "memory");
      }
    }
  } else {  // storer
    // Outputs of >= 64 MiB: stores marked evict-first (+3-7% at 64 MiB-1 GiB).
    uint64_t policy = 0;
    if (evict_first)
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int i = 0, prev = -1;
    for (int64_t b = blockIdx.x; b < batches; b += gridDim.x, ++i) {
      const int s = i % kStages;
      bar_wait(&full[s], (i / kStages) & 1);
      Unit u;
      if (resolve_unit(tab, ntasks, total, first + b * 32 + lane, cur, u)) {
        const uint32_t from = saddr(stage + s * kStageBytes + lane * kBulkSeg);
        for (int j = 0; j < u.d->ndst; ++j) {
          char* dst = ptrs.dst[u.d->dst_bufs[j]] + u.dd;
          if (evict_first)
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                    dst),
                "r"(from), "r"(u.bytes), "l"(policy)
                : "memory");
          else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                         "r"(from), "r"(u.bytes)
                         : "memory");
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // The stage before this one has been read out of shared memory once at
      // most one bulk group (this stage's) is still reading.
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      if (prev >= 0 && lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&empty[prev]))
                     : "memory");
      prev = s;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

}  // namespace

int bulk_smem_bytes() { return kSmemBytes; }

cudaError_t launch_bulk_copy(const DevCopy* d_table, const int64_t* begins, int ntasks,
                             int64_t total_units, const PtrTable& ptrs, cudaStream_t stream,
                             int64_t write_bytes) {
  if (ntasks <= 0 || total_units <= 0) return cudaSuccess;
  static const int ef_env = [] {
    const char* e = std::getenv("APL_COPY_CS");
    return e ? std::atoi(e) : -1;
  }();
  const int ef = ef_env >= 0 ? ef_env : (write_bytes >= (int64_t{64} << 20) ? 1 : 0);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(bulk_copy_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  for (int k = 0; k < ntasks; k += kBulkSmemTasks) {
    const int m = std::min(kBulkSmemTasks, ntasks - k);
    const int64_t first = begins[k];
    const int64_t end = k + m < ntasks ? begins[k + m] : total_units;
    const int64_t batches = (end - first + 31) / 32;
    const int grid = static_cast<int>(std::min<int64_t>(batches, sm_count()));
    bulk_copy_kernel<<<grid, 64, kSmemBytes, stream>>>(d_table + k, m, first, end, ef, ptrs);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace apl
