// Batched N-D box copy: the one data-moving kernel behind shard-slice,
// all-gather unpack, all-to-all pack/unpack, collapsed-chain redistribution
// and the simulated-mesh exchange.
//
// A launch executes a table of copy descriptors. Each descriptor moves
// rows x run bytes, where a row is addressed by up to 7 outer indices
// (strides in bytes on both sides) and the run is contiguous on both sides.
// A descriptor may fan out to several destination buffers at the same
// offset (one read, `ndst` writes): on a simulated mesh every receiver of a
// replicated block takes the same bytes, so they are read from HBM once.
// The work is flattened into "units" of V bytes (V = 16 whenever every run,
// stride, offset and base pointer allows it), so one persistent grid sweeps
// all descriptors with coalesced 128-bit loads/stores regardless of how the
// pieces are shaped.
#pragma once

#include <cstdint>

namespace apl {

constexpr int kCopyMaxOuter = 7;
constexpr int kCopyMaxPtrs = 66;  // 64 simulated devices + 2 staging buffers
constexpr int kCopyMaxFan = 8;    // destinations per descriptor
constexpr int kCopySmemTasks = 128;  // descriptors per LDG launch (staged in smem)

// Division by a runtime-invariant uint32 via multiply-high (n < 2^31).
struct FastDiv {
  uint32_t div = 1, mul = 0, shr = 0;
};

struct DevCopy {
  int64_t unit_begin;  // prefix sum of units over the table
  int64_t src_off, dst_off;
  int64_t src_stride[kCopyMaxOuter], dst_stride[kCopyMaxOuter];
  FastDiv ext[kCopyMaxOuter];
  FastDiv units_per_run;
  int32_t src_buf, nouter, ndst;
  uint8_t dst_bufs[kCopyMaxFan];
  int32_t ksplit;     // > 1: split descriptor (see below)
  int64_t run_bytes;  // bulk (TMA) tables: run length, units are kBulkSeg segments
  // Split descriptor (short-run transposes): one source row holds ksplit
  // adjacent chunks of run bytes (split_src_step apart); chunk j goes to
  // destination buffer dst_bufs[j] at dst_offs[j]. Units enumerate
  // (row, chunk, column) row-major, so consecutive lanes read one whole
  // source row (ksplit * run bytes, contiguous) and every destination still
  // receives its contiguous run — the smem-free form of a tile transpose for
  // rows of a few bytes per receiver.
  FastDiv split_div;  // units per chunk (the run's unit count)
  int64_t split_src_step;
  int64_t dst_offs[kCopyMaxFan];
};

static_assert(sizeof(DevCopy) % 16 == 0, "descriptors are staged in smem as uint4");

// TMA bulk engine (bulk_copy.cu): rows of >= kBulkMinRun contiguous bytes
// move as cp.async.bulk global->smem->global segments of <= kBulkSeg bytes.
constexpr int kBulkSeg = 2048;
constexpr int kBulkMinRun = 2048;  // r01 run probe: shorter runs are faster on LDG

#ifdef __CUDACC__
// Stages a launch's descriptor table in shared memory with asynchronous
// 16-byte copies: every load is in flight at once, so staging costs one
// memory round trip instead of one per loop trip (a plain load/store loop
// measured ~0.13 us per descriptor at 64 threads per CTA). Caller syncs.
__device__ __forceinline__ void stage_table(const DevCopy* table, int ntasks, void* smem) {
  const char* g = reinterpret_cast<const char*>(table);
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n16 = ntasks * static_cast<int>(sizeof(DevCopy) / 16);
  for (int w = threadIdx.x; w < n16; w += blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s + 16 * w), "l"(g + 16 * w)
                 : "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
}
#endif

struct PtrTable {
  const char* src[kCopyMaxPtrs];
  char* dst[kCopyMaxPtrs];
};

// Device-side ordering of a fused peer exchange (box_pull_sync_kernel).
// Flag arrays hold uint32 epochs: slot p = "rank p's source of this epoch is
// written", slot P + p = "rank p finished reading its sources".
constexpr int kPeerMaxRanks = 64;
struct PeerSync {
  // kPush: the table writes into peers' outputs (remote stores), so every
  // CTA fences at system scope before the last one announces done.
  enum : int { kAnnounce = 1, kDone = 2, kPush = 4 };
  uint32_t* remote[kPeerMaxRanks];   // every peer's flag array (mapped here)
  const uint32_t* local;             // this rank's flag array
  unsigned int* counter;             // zeroed device counter (last-CTA election)
  int32_t wait_slot[kPeerMaxRanks];  // ready slots of the ranks this pull reads from
  int32_t n_remote, n_wait, ready_slot, done_slot, mode;
  uint32_t epoch;
  uint64_t timeout_ns;
};

}  // namespace apl
