// Batched N-D box copy kernel (sm_100a). See box_copy.cuh for the model.
//
// Roofline: HBM. Algorithmic bytes per launch = sum over descriptors of
// (bytes read once + bytes written to each destination). Design points:
//  * persistent grid (a multiple of the SM count), each CTA sweeping chunks
//    of blockDim * U units; U independent 128-bit loads are issued before
//    any store so every thread keeps U x 16 B in flight;
//  * the chunk's descriptor is staged in shared memory once per chunk and
//    then held in registers (the kernel is specialised on the largest outer
//    rank NO of the table), so the per-unit address math is one multiply-
//    high division per outer dim plus the run division;
//  * fan-out descriptors: one load, up to 8 stores (replicated targets on a
//    simulated mesh read their source bytes once);
//  * loads use the non-coherent streaming path (ld.global.nc.L1::no_allocate),
//    stores are plain 128-bit st.global (data is consumed by the next kernel
//    or a collective, so it should stay in L2 when it fits).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
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

// Coherent (weak, L1-bypassing) loads for the fused peer exchange: its
// sources are written by other GPUs while the kernel is already running
// (it acquires their ready flags first), so the non-coherent path is not
// allowed there.
template <typename T>
__device__ __forceinline__ T load_coherent(const T* p) {
  return *reinterpret_cast<const volatile T*>(p);
}
template <>
__device__ __forceinline__ uint4 load_coherent<uint4>(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
template <>
__device__ __forceinline__ uint2 load_coherent<uint2>(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
  return r;
}

// Stores; `cs` = cache-streaming (evict-first) for outputs far larger than L2.
template <typename T>
__device__ __forceinline__ void store_v(T* p, const T& v, bool cs) {
  *p = v;
}
template <>
__device__ __forceinline__ void store_v<uint4>(uint4* p, const uint4& v, bool cs) {
  if (cs)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  else
    *p = v;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.div == 1 ? n : (__umulhi(n, f.mul) >> f.shr);
}

// Generic resolution straight from a (global or shared) descriptor: source
// offset and destination offset relative to the descriptor's first
// destination buffer (a split unit's chunk lands in its own buffer, folded
// in as the difference of the two base addresses).
template <int V, bool SPLIT>
__device__ __forceinline__ void resolve(const DevCopy& c, uint32_t local, const PtrTable& ptrs,
                                        int64_t& so, int64_t& dd) {
  uint32_t row = fdiv(local, c.units_per_run);
  uint32_t col = local - row * c.units_per_run.div;
  if (SPLIT && c.ksplit > 1) {
    const uint32_t j = fdiv(col, c.split_div);
    col -= j * c.split_div.div;
    so = c.src_off + static_cast<int64_t>(j) * c.split_src_step + static_cast<int64_t>(col) * V;
    dd = c.dst_offs[j] + (ptrs.dst[c.dst_bufs[j]] - ptrs.dst[c.dst_bufs[0]]) +
         static_cast<int64_t>(col) * V;
  } else {
    so = c.src_off + static_cast<int64_t>(col) * V;
    dd = c.dst_off + static_cast<int64_t>(col) * V;
  }
  for (int i = c.nouter - 1; i >= 0; --i) {
    const uint32_t q = fdiv(row, c.ext[i]);
    const uint32_t r = row - q * c.ext[i].div;
    so += static_cast<int64_t>(r) * c.src_stride[i];
    dd += static_cast<int64_t>(r) * c.dst_stride[i];
    row = q;
  }
}

template <int V, int U, int NO, bool SPLIT, bool COHERENT>
__device__ __forceinline__ void box_copy_body(const DevCopy* __restrict__ table, int ntasks,
                                              int64_t first, int64_t total, int lockstep,
                                              const PtrTable& ptrs) {
  using T = typename Vec<V>::T;
  constexpr int NR = NO > 0 ? NO : 1;
  // The launch's descriptor table (<= kCopySmemTasks entries) is staged in
  // shared memory once per CTA -- one round trip -- after which every thread
  // resolves its chunk with a broadcast binary search in smem: no per-chunk
  // global-memory latency chain and no block barrier inside the loop.
  // Units [first, total) of the table are this launch's.
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  {
    stage_table(table, ntasks, dyn_smem);
    __syncthreads();
  }
  const DevCopy* tab = reinterpret_cast<const DevCopy*>(dyn_smem);
  const int64_t chunk = static_cast<int64_t>(blockDim.x) * U;

  // Chunks go round-robin over the CTAs (the grid sweeps the table front to
  // back together, which keeps DRAM pages and TLB entries shared; a
  // contiguous range per CTA measured 2-5% slower). A CTA's chunks only move
  // forward, so each lookup is a binary search over the table entries at or
  // after the previous chunk's.
  // (lockstep bit 2: contiguous chunk range per CTA instead)
  const int64_t nchunks = (total - first + chunk - 1) / chunk;
  int64_t ci, cend, cstep;
  if (lockstep & 4) {
    const int64_t span = (nchunks + gridDim.x - 1) / gridDim.x;
    ci = static_cast<int64_t>(blockIdx.x) * span;
    cend = ci + span < nchunks ? ci + span : nchunks;
    cstep = 1;
  } else {
    ci = blockIdx.x;
    cend = nchunks;
    cstep = gridDim.x;
  }
  int lo = 0;
  for (; ci < cend; ci += cstep) {
    const int64_t base = first + ci * chunk;
    if (lo + 1 < ntasks && tab[lo + 1].unit_begin <= base) {
      int hi = ntasks - 1;
      ++lo;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tab[mid].unit_begin <= base) lo = mid;
        else hi = mid - 1;
      }
    }
    const int t0 = lo;
    const int64_t next_begin = (lo + 1 < ntasks) ? tab[lo + 1].unit_begin : total;
    const DevCopy& D = tab[lo];
    const bool cs = (lockstep & 2) != 0;
    // Register copy of the chunk's descriptor.
    const int64_t begin = D.unit_begin;
    const FastDiv upr = D.units_per_run;
    const int64_t soff = D.src_off, doff = D.dst_off;
    const int nout = D.nouter;
    const int ndst = D.ndst;
    const int ks = D.ksplit;  // uniform per chunk
    const FastDiv sdiv = D.split_div;
    const int64_t sstep = D.split_src_step;
    FastDiv ext[NR];
    int64_t sst[NR], dst_[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      ext[i] = D.ext[i];
      sst[i] = D.src_stride[i];
      dst_[i] = D.dst_stride[i];
    }
    const char* sp0 = ptrs.src[D.src_buf];
    // destination buffer ids, 4 per register; pointers come from the param bank at store time
    uint32_t dbuf[2];
    std::memcpy(dbuf, D.dst_bufs, sizeof(dbuf));

    T v[U];
    int64_t dd[U];  // offset from the first destination buffer's base
    int slow_task[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t g = base + static_cast<int64_t>(u) * blockDim.x + threadIdx.x;
      slow_task[u] = -2;  // -2: nothing, -1: fast path, >= 0: descriptor index
      if (g < total) {
        int64_t so;
        const char* sp;
        if (g < next_begin) {
          uint32_t row = fdiv(static_cast<uint32_t>(g - begin), upr);
          uint32_t col = static_cast<uint32_t>(g - begin) - row * upr.div;
          if (SPLIT && ks > 1) {
            const uint32_t j = fdiv(col, sdiv);
            col -= j * sdiv.div;
            so = soff + static_cast<int64_t>(j) * sstep + static_cast<int64_t>(col) * V;
            dd[u] = D.dst_offs[j] + (ptrs.dst[D.dst_bufs[j]] - ptrs.dst[D.dst_bufs[0]]) +
                    static_cast<int64_t>(col) * V;
          } else {
            so = soff + static_cast<int64_t>(col) * V;
            dd[u] = doff + static_cast<int64_t>(col) * V;
          }
          if constexpr (NO > 0) {
#pragma unroll
            for (int i = NO - 1; i >= 0; --i) {
              if (i < nout) {
                const uint32_t q = fdiv(row, ext[i]);
                const uint32_t r = row - q * ext[i].div;
                so += static_cast<int64_t>(r) * sst[i];
                dd[u] += static_cast<int64_t>(r) * dst_[i];
                row = q;
              }
            }
          }
          sp = sp0;
          slow_task[u] = -1;
        } else {  // chunk straddles descriptors: walk forward
          int t = t0 + 1;
          while (t + 1 < ntasks && tab[t + 1].unit_begin <= g) ++t;
          const DevCopy& c = tab[t];
          resolve<V, SPLIT>(c, static_cast<uint32_t>(g - c.unit_begin), ptrs, so, dd[u]);
          sp = ptrs.src[c.src_buf];
          slow_task[u] = t;
        }
        if constexpr (COHERENT)
          v[u] = load_coherent(reinterpret_cast<const T*>(sp + so));
        else
          v[u] = load_stream(reinterpret_cast<const T*>(sp + so));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (slow_task[u] == -1) {
        // split descriptors have ndst == 1 (their chunks are folded into dd)
#pragma unroll
        for (int j = 0; j < kCopyMaxFan; ++j)
          if (j < ndst)
            store_v(reinterpret_cast<T*>(ptrs.dst[(dbuf[j >> 2] >> (8 * (j & 3))) & 0xFF] + dd[u]),
                    v[u], cs);
      } else if (slow_task[u] >= 0) {
        const DevCopy& c = tab[slow_task[u]];
        for (int j = 0; j < c.ndst; ++j)
          *reinterpret_cast<T*>(ptrs.dst[c.dst_bufs[j]] + dd[u]) = v[u];
      }
    }
    if (lockstep & 1) __syncthreads();
  }
}

template <int V, int U, int NO, int MINB, bool SPLIT>
__global__ void __launch_bounds__(256, MINB)
    box_copy_kernel(const DevCopy* __restrict__ table, int ntasks, int64_t first, int64_t total,
                    int lockstep, const __grid_constant__ PtrTable ptrs) {
  box_copy_body<V, U, NO, SPLIT, false>(table, ntasks, first, total, lockstep, ptrs);
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The whole peer exchange of one rank in ONE launch (box_copy.cuh,
// PeerSync): CTA 0 announces this rank's source (stores `ready` into every
// peer's flag array), every CTA acquires the ready flags of the ranks it
// actually reads from, the copy body pulls over peer pointers with coherent
// loads, and the last CTA to finish announces `done` to every peer.
template <int V, int U, int NO, int MINB>
__global__ void __launch_bounds__(256, MINB)
    box_pull_sync_kernel(const DevCopy* __restrict__ table, int ntasks, int64_t first,
                         int64_t total, int lockstep, const __grid_constant__ PtrTable ptrs,
                         const __grid_constant__ PeerSync sync) {
  const int t = threadIdx.x;
  if (sync.mode & PeerSync::kAnnounce) {
    if (blockIdx.x == 0 && t < sync.n_remote) {
      __threadfence_system();  // the source (written by earlier kernels) before the flag
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sync.remote[t] + sync.ready_slot),
                   "r"(sync.epoch)
                   : "memory");
    }
    if (t < sync.n_wait) {
      const uint32_t* f = sync.local + sync.wait_slot[t];
      const uint64_t t0 = global_ns();
      while (true) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (static_cast<int32_t>(v - sync.epoch) >= 0) break;  // wrap-safe v >= epoch
        __nanosleep(128);
        if (global_ns() - t0 > sync.timeout_ns) __trap();  // a lost peer: fail, do not hang
      }
    }
    __syncthreads();
  }
  box_copy_body<V, U, NO, false, true>(table, ntasks, first, total, lockstep, ptrs);
  if (sync.mode & PeerSync::kDone) {
    __syncthreads();  // every load of this CTA has returned (its stores consumed them)
    __shared__ unsigned int last;
    if (t == 0) {
      if (sync.mode & PeerSync::kPush) __threadfence_system();  // remote stores visible
      else __threadfence();
      last = atomicAdd(sync.counter, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (last) {
      if (t == 0) *sync.counter = 0;  // stream-serial reuse by the next exchange
      if (t < sync.n_remote) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sync.remote[t] + sync.done_slot),
                     "r"(sync.epoch)
                     : "memory");
      }
    }
  }
}

int g_num_sms = 0;

}  // namespace
int sm_count();
namespace {

// Tiling variants (16-byte path; narrower vectors always use variant 0):
//   0: U=8  @ 2 CTAs/SM (128 regs, no spills)
//   1: U=4  @ 4 CTAs/SM   -- plain contiguous runs (r01 sweep: 96% of copy peak)
//   2: U=16 @ 1 CTA/SM    -- fan-out tables (one load, many stores: 92%)
//   3: U=8  @ 3 CTAs/SM   -- strided boxes (the r01 copy sweep's pick; variant 1
//                            measured ahead of it at every size since)
// The launch picks by table shape (profiles/r01_copy_sweep.md) and size;
// APL_COPY_VARIANT forces one, APL_COPY_CTAS_PER_SM overrides the grid.
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// Launch-bound regime (r01 crossover probe, profiles/r01_crossover.jsonl):
// below 8 MiB read by a fan-out gather, or 64 MiB moved by a strided table,
// U=4 @ 4 CTAs/SM finishes first (AG fan-out of 1 MiB: 4.6 vs 12.4 us;
// 256 B-run all-to-all of 16 MiB: 8.3 vs 9.2 us); the wide variants only pay
// off once the launch streams.
// Strided tables: U=4 @ 4 CTAs/SM as well (r01 short-row probe: 0.92 vs
// 0.85 for U=8 @ 3 on 256 B rows at 512 MiB, ahead at every size measured,
// profiles/r01_short_row_probe.jsonl); U=8 @ 3 stays selectable (variant 3).
// Fan-out tables (r02 knob sweep, profiles/r02_copy_variant_probe.jsonl,
// and the every-pair sweep, r02_pairs_*.jsonl): U=16 @ 1 CTA/SM only wins
// for wide (>= 4-way) fan-outs (config 2's S0R->RR 0.91 vs 0.87; S1R->RR
// on 2x4 0.93 vs 0.89; the 8-way S0S1->RR of strided 4 KiB runs 0.90 vs
// 0.87). Narrow fan-outs (2-way: a target replicated over one mesh axis of
// 2, or a 4x-replicated source feeding 8 receivers) went from 0.65-0.76
// with it to 0.87-0.98 with U=8 @ 2 CTAs/SM, which keeps twice the loads
// in flight per SM.
int copy_variant(int max_outer, int max_fan, int64_t write_bytes) {
  static int forced = env_int("APL_COPY_VARIANT", -1);
  if (forced >= 0) return forced;
  (void)max_outer;
  if (max_fan > 1) {
    if (write_bytes / max_fan < (int64_t{8} << 20)) return 1;
    return max_fan >= 4 ? 2 : 0;
  }
  return 1;
}

template <int V, int U, int MINB, bool SPLIT = false>
void launch_vu(int no, int64_t total, const DevCopy* t, const int64_t* begins, int n,
               const PtrTable& p, cudaStream_t s, bool lock, bool streaming, bool spanning) {
  constexpr int kThreads = 256;
  static int ctas_per_sm = env_int("APL_COPY_CTAS_PER_SM", MINB);
  // Tables larger than kCopySmemTasks run as consecutive launches over
  // slices of the table (each slice's units keep their global numbering).
  for (int k = 0; k < n; k += kCopySmemTasks) {
    const int m = std::min(kCopySmemTasks, n - k);
    const int64_t first = begins[k];
    const int64_t end = k + m < n ? begins[k + m] : total;
    const int64_t chunk = int64_t{kThreads} * U;
    const int64_t chunks = (end - first + chunk - 1) / chunk;
    const int grid = static_cast<int>(
        std::min<int64_t>(chunks, static_cast<int64_t>(sm_count()) * ctas_per_sm));
    const size_t smem = static_cast<size_t>(m) * sizeof(DevCopy);
    // Block barrier per chunk (warps write each chunk together): +7% on
    // plain and fan-out copies, -3% on strided boxes (r01 lock probe).
    static const int forced_lock = env_int("APL_COPY_LOCKSTEP", -1);
    // Cache-streaming stores for single-destination launches writing far
    // at least half of L2 (+2-3% on 64 MiB-1 GiB copies; -1% on fan-out, so not there).
    static const int cs_env = env_int("APL_COPY_CS", -1);
    const bool cs = cs_env >= 0 ? cs_env != 0 : streaming;
    // Contiguous chunk range per CTA for strided single-destination launches
    // of >= 512 MiB (r01 span probe: +5% at 1 GiB with 64 pieces, -1..7% at
    // 128 MiB, where round-robin keeps the grid on shared DRAM pages).
    static const int span_env = env_int("APL_COPY_SPAN", -1);
    const bool span = span_env >= 0 ? span_env != 0 : (no > 0 && spanning);
    const int lockstep =
        (forced_lock >= 0 ? forced_lock : (lock ? 1 : 0)) | (cs ? 2 : 0) | (span ? 4 : 0);
    const DevCopy* tk = t + k;
    switch (no) {
      case 0:
        box_copy_kernel<V, U, 0, MINB, SPLIT><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p);
        break;
      case 1:
        box_copy_kernel<V, U, 1, MINB, SPLIT><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p);
        break;
      case 2:
        box_copy_kernel<V, U, 2, MINB, SPLIT><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p);
        break;
      case 3:
        box_copy_kernel<V, U, 3, MINB, SPLIT><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p);
        break;
      default:
        box_copy_kernel<V, U, kCopyMaxOuter, MINB, SPLIT>
            <<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p);
        break;
    }
  }
}

template <int V>
void launch_v(int no, int fan, bool split, int64_t total_units, const DevCopy* t,
              const int64_t* begins, int n, const PtrTable& p, cudaStream_t s, int64_t wbytes) {
  const bool streaming = fan == 1 && wbytes >= (int64_t{64} << 20);
  const bool spanning = fan == 1 && wbytes >= (int64_t{512} << 20);
  const bool lock = fan > 1 || no == 0;
  // Split tables get their own instantiation so the chunk arithmetic does
  // not cost the common kernels registers (U=8 @ 2 CTAs/SM: no spills).
  if (split) return launch_vu<V, 8, 2, true>(no, total_units, t, begins, n, p, s, lock, streaming, spanning);
  if constexpr (V == 16) {
    switch (copy_variant(no, fan, wbytes)) {
      case 1:
        return launch_vu<V, 4, 4>(no, total_units, t, begins, n, p, s, lock, streaming, spanning);
      case 2:
        return launch_vu<V, 16, 1>(no, total_units, t, begins, n, p, s, lock, streaming, spanning);
      case 3:
        return launch_vu<V, 8, 3>(no, total_units, t, begins, n, p, s, lock, streaming, spanning);
      default:
        break;
    }
  }
  launch_vu<V, 8, 2>(no, total_units, t, begins, n, p, s, lock, streaming, spanning);
}

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

namespace {

template <int V, int U, int MINB>
void launch_pull_sync_v(int no, int64_t total, const DevCopy* t, const int64_t* begins, int n,
                        const PtrTable& p, const PeerSync& sync, cudaStream_t s) {
  constexpr int kThreads = 256;
  // An exchange with nothing to move still runs (grid 1): its flags order
  // the epoch for every peer.
  const int slices = n > 0 ? (n + kCopySmemTasks - 1) / kCopySmemTasks : 1;
  for (int sl = 0; sl < slices; ++sl) {
    const int k = sl * kCopySmemTasks;
    const int m = n > 0 ? std::min(kCopySmemTasks, n - k) : 0;
    const int64_t first = n > 0 ? begins[k] : 0;
    const int64_t end = k + m < n ? begins[k + m] : total;
    const int64_t chunk = int64_t{kThreads} * U;
    const int64_t chunks = std::max<int64_t>(1, (end - first + chunk - 1) / chunk);
    // APL_PULL_GRID_CAP: at most this many CTAs per launch (the single-process
    // loopback harness runs every rank's kernel concurrently on one GPU, so
    // each must leave room for the others to be resident).
    static const int cap = env_int("APL_PULL_GRID_CAP", 0);
    int64_t g = std::min<int64_t>(chunks, static_cast<int64_t>(sm_count()) * MINB);
    if (cap > 0) g = std::min<int64_t>(g, cap);
    const int grid = static_cast<int>(g);
    const size_t smem = static_cast<size_t>(m) * sizeof(DevCopy);
    PeerSync y = sync;
    y.mode = (sl == 0 ? (sync.mode & PeerSync::kAnnounce) : 0) |
             (sl + 1 == slices ? (sync.mode & PeerSync::kDone) : 0);
    const DevCopy* tk = t + k;
    const int lockstep = no == 0 ? 1 : 0;
    switch (no) {
      case 0:
        box_pull_sync_kernel<V, U, 0, MINB><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p, y);
        break;
      case 1:
        box_pull_sync_kernel<V, U, 1, MINB><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p, y);
        break;
      case 2:
        box_pull_sync_kernel<V, U, 2, MINB><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p, y);
        break;
      case 3:
        box_pull_sync_kernel<V, U, 3, MINB><<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p, y);
        break;
      default:
        box_pull_sync_kernel<V, U, kCopyMaxOuter, MINB>
            <<<grid, kThreads, smem, s>>>(tk, m, first, end, lockstep, p, y);
        break;
    }
  }
}

}  // namespace

// One launch per fused peer exchange (tables over kCopySmemTasks descriptors
// take one launch per slice: the first announces and acquires, the last
// announces done).
cudaError_t launch_box_pull_sync(const DevCopy* d_table, const int64_t* begins, int ntasks,
                                 int64_t total_units, int vec_bytes, int max_outer,
                                 const PtrTable& ptrs, const PeerSync& sync, cudaStream_t stream) {
  if (sync.n_remote > kPeerMaxRanks || sync.n_wait > kPeerMaxRanks) return cudaErrorInvalidValue;
  switch (ntasks > 0 ? vec_bytes : 16) {
    case 16:
      launch_pull_sync_v<16, 4, 4>(max_outer, total_units, d_table, begins, ntasks, ptrs, sync, stream);
      break;
    case 8:
      launch_pull_sync_v<8, 8, 2>(max_outer, total_units, d_table, begins, ntasks, ptrs, sync, stream);
      break;
    case 4:
      launch_pull_sync_v<4, 8, 2>(max_outer, total_units, d_table, begins, ntasks, ptrs, sync, stream);
      break;
    case 2:
      launch_pull_sync_v<2, 8, 2>(max_outer, total_units, d_table, begins, ntasks, ptrs, sync, stream);
      break;
    default:
      launch_pull_sync_v<1, 8, 2>(max_outer, total_units, d_table, begins, ntasks, ptrs, sync, stream);
      break;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_box_copy(const DevCopy* d_table, const int64_t* begins, int ntasks,
                            int64_t total_units, int vec_bytes, int max_outer, int max_fan, bool split,
                            const PtrTable& ptrs, cudaStream_t stream, int64_t write_bytes) {
  if (ntasks <= 0 || total_units <= 0) return cudaSuccess;
  switch (vec_bytes) {
    case 16:
      launch_v<16>(max_outer, max_fan, split, total_units, d_table, begins, ntasks, ptrs, stream, write_bytes);
      break;
    case 8:
      launch_v<8>(max_outer, max_fan, split, total_units, d_table, begins, ntasks, ptrs, stream, write_bytes);
      break;
    case 4:
      launch_v<4>(max_outer, max_fan, split, total_units, d_table, begins, ntasks, ptrs, stream, write_bytes);
      break;
    case 2:
      launch_v<2>(max_outer, max_fan, split, total_units, d_table, begins, ntasks, ptrs, stream, write_bytes);
      break;
    default:
      launch_v<1>(max_outer, max_fan, split, total_units, d_table, begins, ntasks, ptrs, stream, write_bytes);
      break;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace apl
