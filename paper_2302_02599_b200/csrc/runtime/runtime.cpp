// Device runtime: exchange compilation and execution on simulated (1 GPU)
// and distributed (NCCL, one process per GPU) meshes.
#include "runtime.hpp"

#include <algorithm>
#include <numeric>
#include <cstdlib>
#include <cstring>

#include <cuda.h>

#include "apl.h"
#include <nvtx3/nvToolsExt.h>

namespace apl {

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }


namespace {

constexpr int64_t kAlign = 256;
constexpr int64_t kMaxUnitsPerDesc = int64_t{1} << 30;  // keeps kernel indices in uint32

int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

int pow2_vec(int64_t g) {
  for (int v = 16; v > 1; v >>= 1)
    if (g % v == 0) return v;
  return 1;
}

int ptr_align(const void* p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  for (int v = 16; v > 1; v >>= 1)
    if (a % static_cast<uintptr_t>(v) == 0) return v;
  return 1;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Splits descriptors whose unit count would overflow the kernel's 32-bit
// per-descriptor index.
void split_large(const CopyDesc& d, int vec, std::vector<CopyDesc>& out) {
  const int64_t upr = d.run_bytes / vec * d.ksplit;
  int64_t rows = 1;
  for (int i = 0; i < d.nouter; ++i) rows *= d.ext[i];
  if (upr * rows <= kMaxUnitsPerDesc) {
    out.push_back(d);
    return;
  }
  if (upr > kMaxUnitsPerDesc / 4) {
    // One very long run: cut it into 2^24-unit runs (+ a remainder).
    const int64_t piece = (int64_t{1} << 24) * vec;
    const int64_t whole = d.run_bytes / piece;
    const int64_t rest = d.run_bytes - whole * piece;
    if (d.nouter == 0) {
      CopyDesc a = d;
      a.run_bytes = piece;
      a.nouter = 1;
      a.ext[0] = whole;
      a.src_stride[0] = piece;
      a.dst_stride[0] = piece;
      split_large(a, vec, out);
      if (rest > 0) {
        CopyDesc b = d;
        b.src_off += whole * piece;
        b.dst_off += whole * piece;
        b.run_bytes = rest;
        out.push_back(b);
      }
      return;
    }
    // Peel the outermost index and recurse on each row.
    for (int64_t i = 0; i < d.ext[0]; ++i) {
      CopyDesc r = d;
      r.src_off += i * d.src_stride[0];
      r.dst_off += i * d.dst_stride[0];
      r.nouter = d.nouter - 1;
      for (int j = 0; j < r.nouter; ++j) {
        r.ext[j] = d.ext[j + 1];
        r.src_stride[j] = d.src_stride[j + 1];
        r.dst_stride[j] = d.dst_stride[j + 1];
      }
      split_large(r, vec, out);
    }
    return;
  }
  // Split the outermost dim into slabs small enough.
  const int64_t inner = upr * rows / d.ext[0];
  const int64_t slab = std::max<int64_t>(1, kMaxUnitsPerDesc / inner);
  for (int64_t i = 0; i < d.ext[0]; i += slab) {
    CopyDesc r = d;
    r.ext[0] = std::min(slab, d.ext[0] - i);
    r.src_off += i * d.src_stride[0];
    r.dst_off += i * d.dst_stride[0];
    split_large(r, vec, out);
  }
}

}  // namespace

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw RuntimeError(APL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw RuntimeError(APL_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

int natural_vec(const std::vector<CopyDesc>& descs) {
  int64_t g = 16;
  for (const CopyDesc& d : descs) {
    g = std::gcd(g, d.run_bytes);
    g = std::gcd(g, d.src_off);
    g = std::gcd(g, d.dst_off);
    for (int i = 0; i < d.nouter; ++i) {
      g = std::gcd(g, d.src_stride[i]);
      g = std::gcd(g, d.dst_stride[i]);
    }
    if (d.ksplit > 1) {
      g = std::gcd(g, d.split_src_step);
      for (int j = 0; j < d.ksplit; ++j) g = std::gcd(g, d.split_dst_off[j]);
    }
  }
  return pow2_vec(g);
}

namespace {

int copy_engine_forced() {  // APL_COPY_ENGINE = ldg | bulk | tile, unset = auto
  static const int forced = [] {
    const char* e = std::getenv("APL_COPY_ENGINE");
    if (e == nullptr) return -1;
    const std::string v(e);
    return v == "bulk" ? 1 : v == "ldg" ? 0 : v == "tile" ? 2 : -1;
  }();
  return forced;
}

constexpr int64_t kSmallCopyBytes = int64_t{8} << 20;   // below: LDG small-launch variant
constexpr int64_t kFanRingMaxBytes = int64_t{64} << 20;  // fan-out gathers on the ring below
constexpr int64_t kTileMinBytes = int64_t{64} << 20;     // TMA tensor tiles from (when on)

// The tile engine's place in the automatic policy: the deep-box rule below
// (r02), or every eligible table with APL_TILE_AUTO=1.
// r01 short-row probe (profiles/r01_short_row_probe.jsonl): for strided rows
// of 64 B - 1 KiB the LDG kernel at U=4 @ 4 CTAs/SM matches the tensor tiles
// at 128 MiB (0.84 vs 0.85) and beats them from 512 MiB (0.92 vs 0.88 at
// 256 B rows; 0.81 vs 0.72 at 128 B) and on the rank-3 2x2x2 case (0.94 vs
// 0.91). The engine stays available (APL_COPY_ENGINE=tile) and tested.
bool tile_auto_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("APL_TILE_AUTO");
    return e != nullptr && std::string(e) == "1";
  }();
  return on;
}

// APL_TILE_AUTO=0: never pick the tiles automatically (not even by the
// deep-box rule below).
bool tile_rule_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("APL_TILE_AUTO");
    return e == nullptr || std::string(e) != "0";
  }();
  return on;
}

// The deep-box rule: tables whose bytes mostly sit in descriptors with two
// or more outer dims left after merging and short runs. The LDG kernel
// resolves every 16-byte chunk through one FastDiv per level (~157
// instructions per chunk at NO = 2 against ~117 at NO = 1, ncu), and on
// these boxes it stalls at 0.65-0.69 of the copy peak where the tensor
// tiles move a whole box per TMA instruction. Every-pair sweep of the
// rank-3 2x2x2 mesh, tiles vs LDG (profiles/r02_pairs_222_r3_*.jsonl):
//   129-256 B runs: tiles ahead on 1,530 of 1,557 such pairs, +13% mean;
//   65-128 B runs: ahead only when the source rows are dense and the
//     destination is strided (strided 128 B reads: -14% worst);
//   <= 64 B runs: no rule (strided 64 B writes on tiles lose up to 35%).
bool deep_short_box(const CopyDesc& d) {
  if (d.nouter < 2) return false;
  const int64_t inner = d.nouter - 1;  // ext/stride index of the innermost outer dim
  if (d.run_bytes > 128 && d.run_bytes <= 256) return true;
  return d.run_bytes > 64 && d.run_bytes <= 128 && d.src_stride[inner] == d.run_bytes &&
         d.dst_stride[inner] != d.run_bytes;
}

bool deep_short_boxes(const std::vector<CopyDesc>& descs) {
  int64_t deep = 0, all = 0;
  for (const CopyDesc& d : descs) {
    const int64_t b = d.bytes();
    all += b;
    if (deep_short_box(d)) deep += b;
  }
  return all > 0 && 2 * deep >= all;
}

}  // namespace

int64_t copy_read_bytes(const std::vector<CopyDesc>& descs) {
  int64_t r = 0;
  for (const CopyDesc& d : descs) r += d.bytes();
  return r;
}

bool bulk_eligible(const std::vector<CopyDesc>& descs, int vec) {
  const int forced = copy_engine_forced();
  if (vec != 16 || descs.empty() || forced == 0 || forced == 2) return false;
  bool strided = false, fan = false;
  for (const CopyDesc& d : descs) {
    if (d.bytes() == 0) continue;
    if (d.run_bytes < (forced == 1 ? 16 : kBulkMinRun) || d.run_bytes % 16 || d.ksplit > 1)
      return false;
    strided = strided || d.nouter > 0;
    fan = fan || d.ndst > 1;
  }
  if (forced == 1) return true;
  // r01 sweep (profiles/r01_copy_engines.md): the TMA ring wins on strided
  // rows (all-to-all packs: 97% vs 80% of copy peak); the LDG kernel keeps
  // plain contiguous copies (95% vs 94%) and fan-out gathers (90% vs 89%).
  // By size (profiles/r01_crossover.jsonl): under 8 MiB read the LDG kernel's
  // small-launch variant finishes first (4 MiB 2 KiB-row all-to-all: 4.2 vs
  // 5.8 us); fan-out gathers of 8-64 MiB run faster on the ring (16 MiB
  // all-gather: 24.6 vs 30.6 us; equal at 64 MiB).
  const int64_t r = copy_read_bytes(descs);
  if (r < kSmallCopyBytes) return false;
  if (fan) return !strided && r < kFanRingMaxBytes;
  return strided;
}

namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_tiled() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    // by version first (the unversioned query can resolve differently under
    // tools that interpose the driver, e.g. compute-sanitizer)
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && p != nullptr)
      return reinterpret_cast<EncodeTiled>(p);
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiled>(nullptr);
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// Tensor geometry of a descriptor for the tile engine: dim 0 = the run in
// 8-byte elements, dims 1.. = the outer dims innermost first.
struct TileGeo {
  int rank;
  cuuint64_t dim[5];
  cuuint32_t box[5];
  int64_t nb[5];
};

TileGeo tile_geo(const CopyDesc& d) {
  TileGeo g{};
  g.rank = 1 + d.nouter;
  g.dim[0] = static_cast<cuuint64_t>(d.run_bytes / 8);
  for (int k = 1; k < g.rank; ++k) g.dim[k] = static_cast<cuuint64_t>(d.ext[d.nouter - k]);
  g.box[0] = static_cast<cuuint32_t>(std::min<cuuint64_t>(g.dim[0], 256));
  const int64_t rows = kTileBoxBytes / (int64_t{g.box[0]} * 8);
  g.box[1] = static_cast<cuuint32_t>(std::min<int64_t>({static_cast<int64_t>(g.dim[1]), 256, rows}));
  for (int k = 2; k < g.rank; ++k) g.box[k] = 1;
  for (int k = 0; k < 5; ++k)
    g.nb[k] = k < g.rank ? (static_cast<int64_t>(g.dim[k]) + g.box[k] - 1) / g.box[k] : 1;
  return g;
}

bool encode_map(CUtensorMap* map, const TileGeo& g, const char* base, const int64_t* stride_outer,
                int nouter) {
  EncodeTiled enc = encode_tiled();
  if (enc == nullptr) return false;
  cuuint64_t strides[4];
  for (int k = 1; k < g.rank; ++k) strides[k - 1] = static_cast<cuuint64_t>(stride_outer[nouter - k]);
  const cuuint32_t elem[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, static_cast<cuuint32_t>(g.rank),
             const_cast<char*>(base), g.dim, strides, g.box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void build_tile_launches(const CompiledCopies& c, const PtrTable& ptrs) {
  c.tile_launches.clear();
  TileArgs cur;
  std::memset(&cur, 0, sizeof(cur));
  int nmaps = 0;
  int64_t units = 0;
  auto flush = [&] {
    if (cur.ndesc == 0) return;
    cur.total = units;
    c.tile_launches.push_back(cur);
    std::memset(&cur, 0, sizeof(cur));
    nmaps = 0;
  };
  for (const CopyDesc& d : c.tile_descs) {
    if (cur.ndesc == kTileMaxDesc || nmaps + 1 + d.ndst > kTileMaxMaps) flush();
    if (cur.ndesc == 0) cur.first = units;
    const TileGeo g = tile_geo(d);
    TileDesc& t = cur.d[cur.ndesc++];
    t.unit_begin = units;
    int64_t n = 1;
    for (int k = 0; k < 5; ++k) {
      t.nb[k] = make_fastdiv(static_cast<uint32_t>(g.nb[k]));
      t.box[k] = k < g.rank ? static_cast<int>(g.box[k]) : 1;
      n *= g.nb[k];
    }
    t.rank = g.rank;
    t.box_bytes = static_cast<int>(int64_t{g.box[0]} * 8 * g.box[1]);
    t.src_map = nmaps;
    if (!encode_map(&cur.maps[nmaps++], g, ptrs.src[d.src_buf] + d.src_off, d.src_stride,
                    d.nouter))
      throw RuntimeError(APL_ERR_CUDA, "cuTensorMapEncodeTiled failed (source)");
    t.dst_map = nmaps;
    t.ndst = d.ndst;
    for (int j = 0; j < d.ndst; ++j) {
      const int buf = j == 0 ? d.dst_buf : d.extra_dst[j - 1];
      if (!encode_map(&cur.maps[nmaps++], g, ptrs.dst[buf] + d.dst_off, d.dst_stride, d.nouter))
        throw RuntimeError(APL_ERR_CUDA, "cuTensorMapEncodeTiled failed (destination)");
    }
    units += n;
  }
  flush();
  c.tile_ptrs = ptrs;
  c.tile_cached = true;
}

}  // namespace

bool tile_eligible(const std::vector<CopyDesc>& descs, int vec) {
  const int forced = copy_engine_forced();
  if (vec != 16 || descs.empty() || forced == 0 || forced == 1) return false;
  if (encode_tiled() == nullptr) return false;
  for (const CopyDesc& d : descs) {
    if (d.bytes() == 0) continue;
    if (d.ksplit > 1 || d.ndst > kTileMaxFan || d.nouter < 1 || d.nouter > 4) return false;
    if (d.run_bytes % 16 || d.run_bytes < 64 || d.src_off % 16 || d.dst_off % 16) return false;
    if (forced != 2 && d.run_bytes >= kBulkMinRun) return false;  // the bulk ring's regime
    for (int i = 0; i < d.nouter; ++i) {
      if (d.src_stride[i] % 16 || d.dst_stride[i] % 16 || d.ext[i] > (int64_t{1} << 31))
        return false;
    }
  }
  // under 64 MiB the tiles' fixed cost (~12 us: tensor-map fetches, ring
  // ramp) loses to the LDG kernel's small-launch variant (16 MiB 256 B-run
  // all-to-all: 8.3 vs 13.8 us; profiles/r01_crossover.jsonl)
  if (forced != 2 && copy_read_bytes(descs) < kTileMinBytes) return false;
  return forced == 2 || tile_auto_enabled() || (tile_rule_enabled() && deep_short_boxes(descs));
}

CompiledCopies compile_copies(const std::vector<CopyDesc>& descs, int vec, bool bulk, bool tile) {
  CompiledCopies cc;
  cc.vec = vec;
  cc.bulk = bulk;
  if (tile) {
    cc.tile = true;
    for (const CopyDesc& d : descs)
      if (d.bytes() > 0) {
        cc.tile_descs.push_back(d);
        cc.bytes += d.bytes();
        cc.write_bytes += d.bytes() * d.ndst;
      }
    return cc;
  }
  std::vector<CopyDesc> flat;
  for (const CopyDesc& d : descs)
    if (d.bytes() > 0) split_large(d, vec, flat);
  if (flat.empty()) return cc;
  static const int slabs = [] {  // experiment knob: cut every descriptor into row slabs
    const char* e = std::getenv("APL_SLABS");
    return e ? std::atoi(e) : 0;
  }();
  if (slabs > 1) {
    std::vector<CopyDesc> cut;
    for (const CopyDesc& d : flat) {
      if (d.nouter == 0 || d.ext[0] < slabs) {
        cut.push_back(d);
        continue;
      }
      const int64_t per = (d.ext[0] + slabs - 1) / slabs;
      for (int64_t i = 0; i < d.ext[0]; i += per) {
        CopyDesc r = d;
        r.ext[0] = std::min(per, d.ext[0] - i);
        r.src_off += i * d.src_stride[0];
        r.dst_off += i * d.dst_stride[0];
        cut.push_back(r);
      }
    }
    flat.swap(cut);
  }
  std::vector<DevCopy> host(flat.size());
  int64_t units = 0;
  for (size_t i = 0; i < flat.size(); ++i) {
    const CopyDesc& d = flat[i];
    DevCopy& h = host[i];
    std::memset(&h, 0, sizeof(h));
    h.unit_begin = units;
    h.src_off = d.src_off;
    h.dst_off = d.dst_off;
    h.src_buf = d.src_buf;
    h.ndst = d.ndst;
    h.dst_bufs[0] = static_cast<uint8_t>(d.dst_buf);
    for (int j = 1; j < d.ndst; ++j) h.dst_bufs[j] = static_cast<uint8_t>(d.extra_dst[j - 1]);
    h.nouter = d.nouter;
    cc.max_outer = std::max(cc.max_outer, d.nouter);
    cc.max_fan = std::max(cc.max_fan, d.ndst);
    int64_t upr = bulk ? (d.run_bytes + kBulkSeg - 1) / kBulkSeg : d.run_bytes / vec;
    h.ksplit = d.ksplit;
    cc.split = cc.split || d.ksplit > 1;
    if (d.ksplit > 1) {  // units of one row: ksplit chunks of upr units
      h.split_div = make_fastdiv(static_cast<uint32_t>(upr));
      h.split_src_step = d.split_src_step;
      for (int j = 0; j < d.ksplit; ++j) {
        h.dst_bufs[j] = static_cast<uint8_t>(d.split_dst[j]);
        h.dst_offs[j] = d.split_dst_off[j];
      }
      upr *= d.ksplit;
    }
    h.units_per_run = make_fastdiv(static_cast<uint32_t>(upr));
    h.run_bytes = d.run_bytes;
    int64_t rows = 1;
    for (int j = 0; j < d.nouter; ++j) {
      h.ext[j] = make_fastdiv(static_cast<uint32_t>(d.ext[j]));
      h.src_stride[j] = d.src_stride[j];
      h.dst_stride[j] = d.dst_stride[j];
      rows *= d.ext[j];
    }
    units += upr * rows;
    cc.bytes += d.bytes();
    cc.write_bytes += d.bytes() * d.ndst;
  }
  cc.ntasks = static_cast<int>(host.size());
  cc.total_units = units;
  for (const DevCopy& h : host) cc.begins.push_back(h.unit_begin);
  check_cuda(cudaMalloc(&cc.table, host.size() * sizeof(DevCopy)), "cudaMalloc(copy table)");
  check_cuda(cudaMemcpy(cc.table, host.data(), host.size() * sizeof(DevCopy),
                        cudaMemcpyHostToDevice),
             "cudaMemcpy(copy table)");
  return cc;
}

void free_copies(CompiledCopies& c) {
  if (c.table != nullptr) cudaFree(c.table);
  c = CompiledCopies{};
}

void run_copies(const CompiledCopies& c, const PtrTable& ptrs, cudaStream_t stream) {
  if (c.empty()) return;
  if (c.tile) {
    if (!c.tile_cached || std::memcmp(&c.tile_ptrs, &ptrs, sizeof(PtrTable)) != 0)
      build_tile_launches(c, ptrs);
    for (const TileArgs& a : c.tile_launches)
      check_cuda(launch_tile_copy(a, stream), "tile copy launch");
    return;
  }
  if (c.bulk) {
    check_cuda(launch_bulk_copy(c.table, c.begins.data(), c.ntasks, c.total_units, ptrs, stream,
                                c.write_bytes), "bulk copy launch");
    return;
  }
  check_cuda(launch_box_copy(c.table, c.begins.data(), c.ntasks, c.total_units, c.vec, c.max_outer, c.max_fan, c.split, ptrs,
                             stream, c.write_bytes),
             "box_copy launch");
}

Mesh::~Mesh() {
  for (auto& [key, ex] : exchanges) {
    for (auto* m : {&ex->copies, &ex->pre, &ex->post, &ex->pull, &ex->push})
      for (auto& [v, c] : *m) free_copies(c);
  }
  for (auto& [ptr, owned] : peer_buffers)
    if (owned) cudaFree(ptr);
    else cudaIpcCloseMemHandle(ptr);
  if (!aborted) {
    for (auto& [mask, comm] : sub) ncclCommDestroy(comm);
    if (world != nullptr) ncclCommDestroy(world);
  }
}

std::shared_ptr<Exchange> get_exchange(Mesh& mesh, const autoplan::ShardingSpec& src,
                                       const autoplan::ShardingSpec& tgt,
                                       const autoplan::TensorMeta& meta) {
  std::string key = src.to_string() + ">" + tgt.to_string() + "|";
  for (int64_t e : meta.shape) key += std::to_string(e) + ",";
  key += "|" + std::to_string(meta.dtype_bytes);
  {
    std::lock_guard<std::mutex> hold(mesh.mu);
    auto it = mesh.exchanges.find(key);
    if (it != mesh.exchanges.end()) return it->second;
  }
  auto ex = std::make_shared<Exchange>();
  const int eb = meta.dtype_bytes;
  const std::vector<int64_t> ls = local_shape(src, mesh.geo, meta);
  const std::vector<int64_t> lt = local_shape(tgt, mesh.geo, meta);
  ex->in_bytes = src.per_device_bytes(meta, mesh.geo);
  ex->out_bytes = tgt.per_device_bytes(meta, mesh.geo);

  if (!mesh.distributed) {
    // Receivers taking the identical box from the same sender at the same
    // local offset (replicated targets) share one fan-out descriptor, so the
    // source bytes are read from HBM once.
    std::map<std::vector<int64_t>, size_t> group;
    for (int64_t q = 0; q < mesh.geo.num_devices(); ++q) {
      for (const Piece& p : pieces_for_receiver(src, tgt, mesh.geo, meta, q)) {
        if (p.sender != q) ex->wire_bytes_in += p.elements() * eb;
        std::vector<int64_t> key{p.sender};
        key.insert(key.end(), p.src_lo.begin(), p.src_lo.end());
        key.insert(key.end(), p.dst_lo.begin(), p.dst_lo.end());
        key.insert(key.end(), p.ext.begin(), p.ext.end());
        auto it = group.find(key);
        if (it != group.end() && ex->host_copies[it->second].ndst < CopyDesc::kMaxFan) {
          CopyDesc& c = ex->host_copies[it->second];
          c.extra_dst[c.ndst - 1] = static_cast<int>(q);
          ++c.ndst;
          continue;
        }
        group[key] = ex->host_copies.size();
        ex->host_copies.push_back(make_copy(static_cast<int>(p.sender), ls, p.src_lo,
                                            static_cast<int>(q), lt, p.dst_lo, p.ext, eb));
      }
    }
    merge_splits(ex->host_copies);
  } else {
    const int64_t me = mesh.rank;
    // Source buffer ids: 0 = in, 1 = recv staging. Destination: 0 = out, 1 = send staging.
    for (const Piece& p : pieces_for_receiver(src, tgt, mesh.geo, meta, me)) {
      // Peer-pull form of the same piece: source buffer id = sender rank in
      // the table of peer-mapped source shards.
      ex->host_pull.push_back(make_copy(static_cast<int>(p.sender), ls, p.src_lo, 0, lt, p.dst_lo,
                                        p.ext, eb));
      if (p.sender != me &&
          std::find(ex->pull_senders.begin(), ex->pull_senders.end(), p.sender) ==
              ex->pull_senders.end())
        ex->pull_senders.push_back(static_cast<int>(p.sender));
      const int64_t bytes = p.elements() * eb;
      if (p.sender == me) {
        ex->host_pre.push_back(make_copy(0, ls, p.src_lo, 0, lt, p.dst_lo, p.ext, eb));
        continue;
      }
      ex->wire_bytes_in += bytes;
      if (box_contiguous(lt, p.ext)) {
        ex->recvs.push_back({static_cast<int>(p.sender), true, box_offset(lt, p.dst_lo) * eb, bytes});
      } else {
        const int64_t off = ex->recv_staging;
        std::vector<int64_t> zero(p.ext.size(), 0);
        CopyDesc c = make_copy(1, p.ext, zero, 0, lt, p.dst_lo, p.ext, eb);
        c.src_off += off;
        ex->host_post.push_back(c);
        ex->recvs.push_back({static_cast<int>(p.sender), false, off, bytes});
        ex->recv_staging = align_up(off + bytes);
      }
    }
    for (const Piece& p : pieces_for_sender(src, tgt, mesh.geo, meta, me)) {
      if (p.receiver == me) continue;
      if (std::find(ex->pull_readers.begin(), ex->pull_readers.end(), p.receiver) ==
          ex->pull_readers.end())
        ex->pull_readers.push_back(static_cast<int>(p.receiver));
      const int64_t bytes = p.elements() * eb;
      ex->wire_bytes_out += bytes;
      if (box_contiguous(ls, p.ext)) {
        ex->sends.push_back({static_cast<int>(p.receiver), true, box_offset(ls, p.src_lo) * eb, bytes});
      } else {
        const int64_t off = ex->send_staging;
        std::vector<int64_t> zero(p.ext.size(), 0);
        CopyDesc c = make_copy(0, ls, p.src_lo, 1, p.ext, zero, p.ext, eb);
        c.dst_off += off;
        ex->host_pre.push_back(c);
        ex->sends.push_back({static_cast<int>(p.receiver), false, off, bytes});
        ex->send_staging = align_up(off + bytes);
      }
    }
    merge_splits(ex->host_pre);
    // Push form: the pieces the pull form's receivers take from this rank
    // (the same sender choice, so pull and push move identical bytes).
    // Receivers taking the identical box at the same offset (replicated
    // targets) share one fan-out descriptor: the source is read once.
    std::map<std::vector<int64_t>, size_t> group;
    for (int64_t q = 0; q < mesh.geo.num_devices(); ++q)
      for (const Piece& p : pieces_for_receiver(src, tgt, mesh.geo, meta, q)) {
        if (p.sender != me) continue;
        std::vector<int64_t> key(p.src_lo);
        key.insert(key.end(), p.dst_lo.begin(), p.dst_lo.end());
        key.insert(key.end(), p.ext.begin(), p.ext.end());
        auto it = group.find(key);
        if (it != group.end() && ex->host_push[it->second].ndst < CopyDesc::kMaxFan) {
          CopyDesc& c = ex->host_push[it->second];
          c.extra_dst[c.ndst - 1] = static_cast<int>(q);
          ++c.ndst;
          continue;
        }
        group[key] = ex->host_push.size();
        ex->host_push.push_back(make_copy(0, ls, p.src_lo, static_cast<int>(q), lt, p.dst_lo,
                                          p.ext, eb));
      }
  }
  std::lock_guard<std::mutex> hold(mesh.mu);
  ex->label = key;
  auto [it, fresh] = mesh.exchanges.emplace(key, ex);
  return it->second;
}

std::shared_ptr<Exchange> get_allgather(Mesh& mesh, const autoplan::ShardingSpec& src,
                                        const autoplan::TransformStep& step,
                                        const autoplan::TensorMeta& meta) {
  std::string key = "AG|" + src.to_string() + ">" + step.result.to_string() + "|" +
                    std::to_string(step.tensor_dim) + "," + std::to_string(step.mesh_axis) + "|";
  for (int64_t e : meta.shape) key += std::to_string(e) + ",";
  key += "|" + std::to_string(meta.dtype_bytes);
  {
    std::lock_guard<std::mutex> hold(mesh.mu);
    auto it = mesh.exchanges.find(key);
    if (it != mesh.exchanges.end()) return it->second;
  }
  auto ex = std::make_shared<Exchange>();
  const int eb = meta.dtype_bytes;
  const std::vector<int64_t> ls = local_shape(src, mesh.geo, meta);
  const std::vector<int64_t> lt = local_shape(step.result, mesh.geo, meta);
  const int d = step.tensor_dim;
  const int64_t n = mesh.geo.shape[static_cast<size_t>(step.mesh_axis)];
  ex->in_bytes = src.per_device_bytes(meta, mesh.geo);
  ex->out_bytes = step.result.per_device_bytes(meta, mesh.geo);
  ex->ag_axis = step.mesh_axis;
  int64_t outer = 1;
  for (int i = 0; i < d; ++i) outer *= ls[static_cast<size_t>(i)];
  ex->ag_direct = outer == 1;  // [n][1..][L][Q] == [1..][n*L][Q]
  ex->wire_bytes_in = (n - 1) * ex->in_bytes;
  ex->wire_bytes_out = (n - 1) * ex->in_bytes;
  if (!ex->ag_direct) {
    // block j (coordinate j on the axis, the least significant digit of
    // dims[d]) -> offset j * L along dim d of the output
    std::vector<int64_t> zero(ls.size(), 0);
    for (int64_t j = 0; j < n; ++j) {
      std::vector<int64_t> lo(ls.size(), 0);
      lo[static_cast<size_t>(d)] = j * ls[static_cast<size_t>(d)];
      CopyDesc c = make_copy(1, ls, zero, 0, lt, lo, ls, eb);
      c.src_off += j * ex->in_bytes;
      ex->host_post.push_back(c);
    }
    ex->recv_staging = align_up(n * ex->in_bytes);
  }
  std::lock_guard<std::mutex> hold(mesh.mu);
  ex->label = key;
  auto [it, fresh] = mesh.exchanges.emplace(key, ex);
  return it->second;
}

std::shared_ptr<Exchange> get_alltoall(Mesh& mesh, const autoplan::ShardingSpec& src,
                                       const autoplan::TransformStep& step,
                                       const autoplan::TensorMeta& meta) {
  std::string key = "A2A|" + src.to_string() + ">" + step.result.to_string() + "|" +
                    std::to_string(step.tensor_dim) + "," + std::to_string(step.target_dim) +
                    "," + std::to_string(step.mesh_axis) + "|";
  for (int64_t e : meta.shape) key += std::to_string(e) + ",";
  key += "|" + std::to_string(meta.dtype_bytes);
  {
    std::lock_guard<std::mutex> hold(mesh.mu);
    auto it = mesh.exchanges.find(key);
    if (it != mesh.exchanges.end()) return it->second;
  }
  auto ex = std::make_shared<Exchange>();
  const int eb = meta.dtype_bytes;
  const std::vector<int64_t> ls = local_shape(src, mesh.geo, meta);
  const std::vector<int64_t> lt = local_shape(step.result, mesh.geo, meta);
  const size_t d = static_cast<size_t>(step.tensor_dim), d2 = static_cast<size_t>(step.target_dim);
  const int64_t n = mesh.geo.shape[static_cast<size_t>(step.mesh_axis)];
  ex->in_bytes = src.per_device_bytes(meta, mesh.geo);
  ex->out_bytes = step.result.per_device_bytes(meta, mesh.geo);
  ex->a2a_axis = step.mesh_axis;
  ex->a2a_chunk = ex->in_bytes / n;
  // chunk j = `in` with dim d2 cut to its j-th 1/n (peer j's part)
  std::vector<int64_t> chunk = ls;
  chunk[d2] /= n;
  int64_t before_d2 = 1, before_d = 1;
  for (size_t i = 0; i < d2; ++i) before_d2 *= ls[i];
  for (size_t i = 0; i < d; ++i) before_d *= lt[i];
  ex->a2a_direct_send = before_d2 == 1;  // `in` is [n][chunk] already
  ex->a2a_direct_recv = before_d == 1;   // [n][chunk] lands as `out`
  const std::vector<int64_t> zero(ls.size(), 0);
  for (int64_t j = 0; j < n; ++j) {
    if (!ex->a2a_direct_send) {
      std::vector<int64_t> lo(ls.size(), 0);
      lo[d2] = j * chunk[d2];
      CopyDesc c = make_copy(0, ls, lo, 1, chunk, zero, chunk, eb);
      c.dst_off += j * ex->a2a_chunk;
      ex->host_pre.push_back(c);
    }
    if (!ex->a2a_direct_recv) {  // block from coordinate j -> offset j * L along d
      std::vector<int64_t> lo(lt.size(), 0);
      lo[d] = j * chunk[d];
      CopyDesc c = make_copy(1, chunk, zero, 0, lt, lo, chunk, eb);
      c.src_off += j * ex->a2a_chunk;
      ex->host_post.push_back(c);
    }
  }
  if (!ex->a2a_direct_send) ex->send_staging = align_up(ex->in_bytes);
  if (!ex->a2a_direct_recv) ex->recv_staging = align_up(ex->out_bytes);
  ex->wire_bytes_in = (n - 1) * ex->a2a_chunk;
  ex->wire_bytes_out = (n - 1) * ex->a2a_chunk;
  merge_splits(ex->host_pre);
  std::lock_guard<std::mutex> hold(mesh.mu);
  ex->label = key;
  auto [it, fresh] = mesh.exchanges.emplace(key, ex);
  return it->second;
}

size_t exchange_workspace(const Exchange& ex) {
  return static_cast<size_t>(align_up(ex.send_staging) + align_up(ex.recv_staging));
}

namespace {

const CompiledCopies& compiled_for(std::map<int, CompiledCopies>& cache,
                                   const std::vector<CopyDesc>& host, int vec) {
  const bool tile = tile_eligible(host, vec);
  const bool bulk = !tile && bulk_eligible(host, vec);
  const int key = vec + (bulk ? 1000 : 0) + (tile ? 2000 : 0);
  auto it = cache.find(key);
  if (it == cache.end()) it = cache.emplace(key, compile_copies(host, vec, bulk, tile)).first;
  return it->second;
}

}  // namespace

void run_exchange(Mesh& mesh, Exchange& ex, const void* const* in, void* const* out, void* ws,
                  size_t ws_bytes, cudaStream_t stream) {
  NvtxRange range(ex.label.c_str());
  DeviceGuard guard(mesh.device);
  const int nl = mesh.num_local();
  if (!mesh.distributed) {
    PtrTable t{};
    int align = natural_vec(ex.host_copies);
    for (int i = 0; i < nl; ++i) {
      t.src[i] = static_cast<const char*>(in[i]);
      t.dst[i] = static_cast<char*>(out[i]);
      align = std::min({align, ptr_align(in[i]), ptr_align(out[i])});
    }
    std::lock_guard<std::mutex> hold(mesh.mu);
    run_copies(compiled_for(ex.copies, ex.host_copies, align), t, stream);
    return;
  }
  if (mesh.aborted) throw RuntimeError(APL_ERR_NCCL, "mesh communicators were aborted");
  if (ws_bytes < exchange_workspace(ex))
    throw RuntimeError(APL_ERR_ARG, "workspace smaller than apl_path_workspace_bytes");
  char* send = static_cast<char*>(ws);
  char* recv = send + align_up(ex.send_staging);
  PtrTable t{};
  t.src[0] = static_cast<const char*>(in[0]);
  t.src[1] = recv;
  t.dst[0] = static_cast<char*>(out[0]);
  t.dst[1] = send;
  if (ex.a2a_axis >= 0) {  // pack, one ncclAlltoAll on the axis communicator, unpack
    auto comm = mesh.sub.find(1u << ex.a2a_axis);
    if (comm == mesh.sub.end())
      throw RuntimeError(APL_ERR_NCCL, "no communicator for mesh axis " +
                                           std::to_string(ex.a2a_axis));
    const int palign = std::min({ptr_align(in[0]), ptr_align(out[0]), ptr_align(ws)});
    if (!ex.a2a_direct_send) {
      std::lock_guard<std::mutex> hold(mesh.mu);
      run_copies(compiled_for(ex.pre, ex.host_pre, std::min(palign, natural_vec(ex.host_pre))), t,
                 stream);
    }
    check_nccl(ncclAlltoAll(ex.a2a_direct_send ? in[0] : static_cast<const void*>(send),
                            ex.a2a_direct_recv ? out[0] : static_cast<void*>(recv),
                            static_cast<size_t>(ex.a2a_chunk), ncclInt8, comm->second, stream),
               "ncclAlltoAll");
    if (!ex.a2a_direct_recv) {
      std::lock_guard<std::mutex> hold(mesh.mu);
      run_copies(compiled_for(ex.post, ex.host_post, std::min(palign, natural_vec(ex.host_post))),
                 t, stream);
    }
    return;
  }
  if (ex.ag_axis >= 0) {  // one NCCL all-gather on the axis communicator (+ unpack)
    auto comm = mesh.sub.find(1u << ex.ag_axis);
    if (comm == mesh.sub.end())
      throw RuntimeError(APL_ERR_NCCL, "no communicator for mesh axis " +
                                           std::to_string(ex.ag_axis));
    check_nccl(ncclAllGather(in[0], ex.ag_direct ? out[0] : static_cast<void*>(recv),
                             static_cast<size_t>(ex.in_bytes), ncclInt8, comm->second, stream),
               "ncclAllGather");
    if (!ex.ag_direct) {
      const int palign = std::min(ptr_align(out[0]), ptr_align(ws));
      std::lock_guard<std::mutex> hold(mesh.mu);
      run_copies(compiled_for(ex.post, ex.host_post, std::min(palign, natural_vec(ex.host_post))),
                 t, stream);
    }
    return;
  }
  const int palign = std::min({ptr_align(in[0]), ptr_align(out[0]), ptr_align(ws)});
  {
    std::lock_guard<std::mutex> hold(mesh.mu);
    run_copies(compiled_for(ex.pre, ex.host_pre, std::min(palign, natural_vec(ex.host_pre))), t,
               stream);
  }
  if (!ex.sends.empty() || !ex.recvs.empty()) {
    check_nccl(ncclGroupStart(), "ncclGroupStart");
    for (const auto& s : ex.sends) {
      const char* p = s.direct ? static_cast<const char*>(in[0]) + s.offset : send + s.offset;
      check_nccl(ncclSend(p, static_cast<size_t>(s.bytes), ncclInt8, s.peer, mesh.world, stream),
                 "ncclSend");
    }
    for (const auto& r : ex.recvs) {
      char* p = r.direct ? static_cast<char*>(out[0]) + r.offset : recv + r.offset;
      check_nccl(ncclRecv(p, static_cast<size_t>(r.bytes), ncclInt8, r.peer, mesh.world, stream),
                 "ncclRecv");
    }
    check_nccl(ncclGroupEnd(), "ncclGroupEnd");
  }
  {
    std::lock_guard<std::mutex> hold(mesh.mu);
    run_copies(compiled_for(ex.post, ex.host_post, std::min(palign, natural_vec(ex.host_post))),
               t, stream);
  }
}

void run_pull(Mesh& mesh, const autoplan::ShardingSpec& src, const autoplan::ShardingSpec& tgt,
              const autoplan::TensorMeta& meta, const void* const* peer_in, void* out,
              cudaStream_t stream) {
  if (!mesh.distributed) throw RuntimeError(APL_ERR_ARG, "peer pull needs a distributed mesh");
  if (!src.valid_for(meta, mesh.geo) || !tgt.valid_for(meta, mesh.geo))
    throw RuntimeError(APL_ERR_SHAPE, "spec is not valid for the tensor/mesh");
  const int64_t p = mesh.geo.num_devices();
  if (p > kCopyMaxPtrs) throw RuntimeError(APL_ERR_ARG, "mesh too large for one pull launch");
  DeviceGuard guard(mesh.device);
  auto ex = get_exchange(mesh, src, tgt, meta);
  NvtxRange range(ex->label.c_str());
  PtrTable t{};
  int align = std::min(natural_vec(ex->host_pull), ptr_align(out));
  for (int64_t i = 0; i < p; ++i) {
    t.src[i] = static_cast<const char*>(peer_in[i]);
    align = std::min(align, ptr_align(peer_in[i]));
  }
  t.dst[0] = static_cast<char*>(out);
  std::lock_guard<std::mutex> hold(mesh.mu);
  // Peer loads stay on the LDG/STG engine (plain ld.global through the
  // peer aperture, L2-bypassing over NVLink).
  auto it = ex->pull.find(align);
  if (it == ex->pull.end()) it = ex->pull.emplace(align, compile_copies(ex->host_pull, align, false)).first;
  run_copies(it->second, t, stream);
}

void run_pull_sync(Mesh& mesh, const autoplan::ShardingSpec& src,
                   const autoplan::ShardingSpec& tgt, const autoplan::TensorMeta& meta,
                   const void* const* peer_in, void* out, const PeerSyncArgs& sync,
                   cudaStream_t stream) {
  if (!mesh.distributed) throw RuntimeError(APL_ERR_ARG, "peer pull needs a distributed mesh");
  if (!src.valid_for(meta, mesh.geo) || !tgt.valid_for(meta, mesh.geo))
    throw RuntimeError(APL_ERR_SHAPE, "spec is not valid for the tensor/mesh");
  const int64_t p = mesh.geo.num_devices();
  if (p > kCopyMaxPtrs || p > kPeerMaxRanks)
    throw RuntimeError(APL_ERR_ARG, "mesh too large for one pull launch");
  if (sync.flags == nullptr || sync.local_flags == nullptr || sync.counter == nullptr)
    throw RuntimeError(APL_ERR_ARG, "null flag arrays / counter");
  DeviceGuard guard(mesh.device);
  auto ex = get_exchange(mesh, src, tgt, meta);
  NvtxRange range(ex->label.c_str());
  PtrTable t{};
  int align = std::min(natural_vec(ex->host_pull), ptr_align(out));
  for (int64_t i = 0; i < p; ++i) {
    t.src[i] = static_cast<const char*>(peer_in[i]);
    align = std::min(align, ptr_align(peer_in[i]));
  }
  t.dst[0] = static_cast<char*>(out);
  PeerSync y{};
  for (int64_t q = 0; q < p; ++q) {
    if (q == mesh.rank) continue;
    y.remote[y.n_remote++] = static_cast<uint32_t*>(sync.flags[q]);
  }
  for (int s : ex->pull_senders) y.wait_slot[y.n_wait++] = s;
  y.local = static_cast<const uint32_t*>(sync.local_flags);
  y.counter = static_cast<unsigned int*>(sync.counter);
  y.ready_slot = mesh.rank;
  y.done_slot = static_cast<int32_t>(p) + mesh.rank;
  y.mode = PeerSync::kAnnounce | PeerSync::kDone;
  y.epoch = sync.epoch;
  y.timeout_ns = sync.timeout_ns;
  std::lock_guard<std::mutex> hold(mesh.mu);
  auto it = ex->pull.find(align);
  if (it == ex->pull.end())
    it = ex->pull.emplace(align, compile_copies(ex->host_pull, align, false)).first;
  const CompiledCopies& c = it->second;
  check_cuda(launch_box_pull_sync(c.table, c.begins.data(), c.ntasks, c.total_units, c.vec,
                                  c.max_outer, t, y, stream),
             "fused peer exchange launch");
}

void run_push_sync(Mesh& mesh, const autoplan::ShardingSpec& src,
                   const autoplan::ShardingSpec& tgt, const autoplan::TensorMeta& meta,
                   const void* in, void* const* peer_out, const PeerSyncArgs& sync,
                   cudaStream_t stream) {
  if (!mesh.distributed) throw RuntimeError(APL_ERR_ARG, "peer push needs a distributed mesh");
  if (!src.valid_for(meta, mesh.geo) || !tgt.valid_for(meta, mesh.geo))
    throw RuntimeError(APL_ERR_SHAPE, "spec is not valid for the tensor/mesh");
  const int64_t p = mesh.geo.num_devices();
  if (p > kCopyMaxPtrs || p > kPeerMaxRanks)
    throw RuntimeError(APL_ERR_ARG, "mesh too large for one push launch");
  if (sync.flags == nullptr || sync.local_flags == nullptr || sync.counter == nullptr)
    throw RuntimeError(APL_ERR_ARG, "null flag arrays / counter");
  DeviceGuard guard(mesh.device);
  auto ex = get_exchange(mesh, src, tgt, meta);
  NvtxRange range(ex->label.c_str());
  PtrTable t{};
  int align = std::min(natural_vec(ex->host_push), ptr_align(in));
  t.src[0] = static_cast<const char*>(in);
  for (int64_t i = 0; i < p; ++i) {
    t.dst[i] = static_cast<char*>(peer_out[i]);
    align = std::min(align, ptr_align(peer_out[i]));
  }
  PeerSync y{};
  for (int64_t q = 0; q < p; ++q) {
    if (q == mesh.rank) continue;
    y.remote[y.n_remote++] = static_cast<uint32_t*>(sync.flags[q]);
  }
  // the receivers of this rank's pieces must have entered this epoch (their
  // previous output is consumed) before it is overwritten
  for (int r : ex->pull_readers) y.wait_slot[y.n_wait++] = r;
  y.local = static_cast<const uint32_t*>(sync.local_flags);
  y.counter = static_cast<unsigned int*>(sync.counter);
  y.ready_slot = mesh.rank;
  y.done_slot = static_cast<int32_t>(p) + mesh.rank;
  y.mode = PeerSync::kAnnounce | PeerSync::kDone | PeerSync::kPush;
  y.epoch = sync.epoch;
  y.timeout_ns = sync.timeout_ns;
  std::lock_guard<std::mutex> hold(mesh.mu);
  auto it = ex->push.find(align);
  if (it == ex->push.end())
    it = ex->push.emplace(align, compile_copies(ex->host_push, align, false)).first;
  const CompiledCopies& c = it->second;
  check_cuda(launch_box_pull_sync(c.table, c.begins.data(), c.ntasks, c.total_units, c.vec,
                                  c.max_outer, t, y, stream),
             "peer push launch");
}

namespace {

// Checks the steps replay src -> tgt with the reference step semantics
// (the same contract as reference tests/helpers.hpp:282-339).
void validate_steps(const autoplan::ShardingSpec& src, const autoplan::ShardingSpec& tgt,
                    const std::vector<autoplan::TransformStep>& steps,
                    const autoplan::DeviceMesh& geo, const autoplan::TensorMeta& meta) {
  using autoplan::CollectiveKind;
  autoplan::ShardingSpec cur = src;
  for (size_t i = 0; i < steps.size(); ++i) {
    const auto& s = steps[i];
    const int r = cur.tensor_rank();
    bool ok = s.tensor_dim >= 0 && s.tensor_dim < r;
    if (ok) {
      auto& axes = cur.dims[static_cast<size_t>(s.tensor_dim)].axes;
      switch (s.kind) {
        case CollectiveKind::kAllGather:
          ok = !axes.empty() && axes.back() == s.mesh_axis;
          if (ok) axes.pop_back();
          break;
        case CollectiveKind::kShardSlice: {
          const auto used = cur.used_axes();
          ok = s.mesh_axis >= 0 && s.mesh_axis < cur.mesh_rank &&
               std::find(used.begin(), used.end(), s.mesh_axis) == used.end();
          if (ok) axes.push_back(s.mesh_axis);
          break;
        }
        case CollectiveKind::kAllToAll:
          ok = s.target_dim >= 0 && s.target_dim < r && s.target_dim != s.tensor_dim &&
               !axes.empty() && axes.back() == s.mesh_axis;
          if (ok) {
            axes.pop_back();
            cur.dims[static_cast<size_t>(s.target_dim)].axes.push_back(s.mesh_axis);
          }
          break;
        default:
          ok = false;
      }
    }
    if (!ok || !(cur == s.result) || !cur.valid_for(meta, geo))
      throw RuntimeError(APL_ERR_ARG, "step " + std::to_string(i) +
                                          " does not replay from " + src.to_string());
  }
  if (!(cur == tgt))
    throw RuntimeError(APL_ERR_ARG, "steps end at " + cur.to_string() + ", not " +
                                        tgt.to_string());
}

}  // namespace

Conversion prepare_conversion(Mesh& mesh, const autoplan::ShardingSpec& src,
                              const autoplan::ShardingSpec& tgt,
                              const std::vector<autoplan::TransformStep>& steps,
                              const autoplan::TensorMeta& meta, bool fuse) {
  if (!src.valid_for(meta, mesh.geo) || !tgt.valid_for(meta, mesh.geo))
    throw RuntimeError(APL_ERR_SHAPE, "spec is not valid for the tensor/mesh");
  validate_steps(src, tgt, steps, mesh.geo, meta);
  Conversion cv;
  cv.mesh = &mesh;
  // Distributed meshes run an all-gather step as ONE ncclAllGather and an
  // all-to-all step as ONE ncclAlltoAll on the step's mesh-axis
  // communicator (also when the path is that single step); a collapsed
  // multi-step chain stays one point-to-point exchange.
  const bool ag_single = mesh.distributed && steps.size() == 1 &&
                         (steps[0].kind == autoplan::CollectiveKind::kAllGather ||
                          steps[0].kind == autoplan::CollectiveKind::kAllToAll);
  if ((fuse || steps.size() <= 1) && !ag_single) {
    cv.hops.push_back(get_exchange(mesh, src, tgt, meta));
    cv.staging = static_cast<int64_t>(exchange_workspace(*cv.hops[0]));
    return cv;
  }
  const autoplan::ShardingSpec* cur = &src;
  for (size_t i = 0; i < steps.size(); ++i) {
    const auto kind = steps[i].kind;
    auto ex = !mesh.distributed ? get_exchange(mesh, *cur, steps[i].result, meta)
              : kind == autoplan::CollectiveKind::kAllGather
                  ? get_allgather(mesh, *cur, steps[i], meta)
              : kind == autoplan::CollectiveKind::kAllToAll
                  ? get_alltoall(mesh, *cur, steps[i], meta)
                  : get_exchange(mesh, *cur, steps[i].result, meta);
    cv.staging = std::max<int64_t>(cv.staging, static_cast<int64_t>(exchange_workspace(*ex)));
    if (i + 1 < steps.size())
      cv.inter_bytes = std::max(cv.inter_bytes, align_up(ex->out_bytes) * mesh.num_local());
    cv.hops.push_back(std::move(ex));
    cur = &steps[i].result;
  }
  return cv;
}

size_t conversion_workspace(const Conversion& cv) {
  return static_cast<size_t>(2 * cv.inter_bytes + cv.staging);
}

void run_conversion(Conversion& cv, const void* const* in, void* const* out, void* ws,
                    size_t ws_bytes, cudaStream_t stream) {
  NvtxRange range(cv.hops.size() == 1 ? "apl.convert" : "apl.convert.stepwise");
  Mesh& mesh = *cv.mesh;
  if (ws_bytes < conversion_workspace(cv))
    throw RuntimeError(APL_ERR_ARG, "workspace smaller than apl_path_workspace_bytes");
  if (cv.hops.size() == 1) {
    run_exchange(mesh, *cv.hops[0], in, out, ws, ws_bytes, stream);
    return;
  }
  const int nl = mesh.num_local();
  char* region[2] = {static_cast<char*>(ws), static_cast<char*>(ws) + cv.inter_bytes};
  char* staging = static_cast<char*>(ws) + 2 * cv.inter_bytes;
  std::vector<const void*> cur_in(in, in + nl);
  std::vector<void*> next(static_cast<size_t>(nl));
  for (size_t i = 0; i < cv.hops.size(); ++i) {
    const bool last = i + 1 == cv.hops.size();
    if (last) {
      for (int j = 0; j < nl; ++j) next[static_cast<size_t>(j)] = out[j];
    } else {
      const int64_t stride = align_up(cv.hops[i]->out_bytes);
      for (int j = 0; j < nl; ++j) next[static_cast<size_t>(j)] = region[i % 2] + j * stride;
    }
    run_exchange(mesh, *cv.hops[i], cur_in.data(), next.data(), staging,
                 static_cast<size_t>(cv.staging), stream);
    for (int j = 0; j < nl; ++j) cur_in[static_cast<size_t>(j)] = next[static_cast<size_t>(j)];
  }
}

size_t path_workspace(Mesh& mesh, const autoplan::ShardingSpec& src,
                      const autoplan::ShardingSpec& tgt,
                      const std::vector<autoplan::TransformStep>& steps,
                      const autoplan::TensorMeta& meta, bool fuse) {
  return conversion_workspace(prepare_conversion(mesh, src, tgt, steps, meta, fuse));
}

void run_path(Mesh& mesh, const autoplan::ShardingSpec& src, const autoplan::ShardingSpec& tgt,
              const std::vector<autoplan::TransformStep>& steps,
              const autoplan::TensorMeta& meta, const void* const* in, void* const* out,
              void* ws, size_t ws_bytes, bool fuse, cudaStream_t stream) {
  Conversion cv = prepare_conversion(mesh, src, tgt, steps, meta, fuse);
  run_conversion(cv, in, out, ws, ws_bytes, stream);
}

void all_reduce(Mesh& mesh, const std::vector<int>& axes, void* const* bufs, size_t count,
                int dtype, cudaStream_t stream) {
  NvtxRange range("apl.all_reduce");
  DeviceGuard guard(mesh.device);
  uint32_t mask = 0;
  for (int a : axes) {
    if (a < 0 || a >= mesh.geo.rank()) throw RuntimeError(APL_ERR_AXIS, "reduce axis out of range");
    mask |= 1u << a;
  }
  if (mask == 0 || count == 0) return;
  if (mesh.distributed) {
    if (mesh.aborted) throw RuntimeError(APL_ERR_NCCL, "mesh communicators were aborted");
    ncclDataType_t t = dtype == APL_F32 ? ncclFloat32 : dtype == APL_BF16 ? ncclBfloat16 : ncclFloat16;
    check_nccl(ncclAllReduce(bufs[0], bufs[0], count, t, ncclSum, mesh.sub.at(mask), stream),
               "ncclAllReduce");
    return;
  }
  const auto groups = axis_groups(mesh.geo, axes);
  std::vector<int> members;
  for (const auto& g : groups) members.insert(members.end(), g.begin(), g.end());
  check_cuda(launch_allreduce_local(bufs, members.data(), static_cast<int>(groups.size()),
                                    static_cast<int>(groups[0].size()), count, dtype, stream),
             "all-reduce launch");
}

std::vector<std::vector<int>> axis_groups(const autoplan::DeviceMesh& geo,
                                          const std::vector<int>& axes) {
  // Devices sharing every coordinate off `axes`; members ordered by their
  // mixed-radix coordinate on `axes` (row-major order preserves it).
  uint32_t mask = 0;
  for (int a : axes) mask |= 1u << a;
  const int64_t p = geo.num_devices();
  int64_t gsize = 1;
  for (int a = 0; a < geo.rank(); ++a)
    if (mask & (1u << a)) gsize *= geo.shape[static_cast<size_t>(a)];
  std::vector<std::vector<int>> groups(static_cast<size_t>(p / gsize));
  for (int64_t d = 0; d < p; ++d) {
    const auto c = geo.coord_of(d);
    int64_t off = 0;
    for (int a = 0; a < geo.rank(); ++a)
      if (!(mask & (1u << a))) off = off * geo.shape[static_cast<size_t>(a)] + c[static_cast<size_t>(a)];
    groups[static_cast<size_t>(off)].push_back(static_cast<int>(d));
  }
  return groups;
}

}  // namespace apl
