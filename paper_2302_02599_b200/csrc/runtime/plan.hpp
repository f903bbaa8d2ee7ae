// Data-placement geometry and exchange planning (host side, no CUDA).
//
// Placement: dim d of a tensor sharded over axes
// (a_1..a_m) is split into N_d = prod n_{a_i} equal blocks and the device at
// coordinate c holds block s_d = mixed radix (c_{a_1}, .., c_{a_m}), a_1 most
// significant. Every reference step (layout.cpp:178-219) is then a pure
// per-axis-group collective, and the bytes a device ends with depend only on
// (tensor, target spec, mesh) — which is what lets a chain be collapsed into
// one exchange without changing a single output byte.
#pragma once

#include <cstdint>
#include <vector>

#include "autoplan/layout.hpp"

namespace apl {

using autoplan::DeviceMesh;
using autoplan::ShardingSpec;
using autoplan::TensorMeta;

constexpr int kMaxDims = 8;

// Local (per-device) shard shape of `meta` under `spec`.
std::vector<int64_t> local_shape(const ShardingSpec& spec, const DeviceMesh& mesh,
                                 const TensorMeta& meta);

// Global lower corner of the block device `device` holds under `spec`.
std::vector<int64_t> block_origin(const ShardingSpec& spec, const DeviceMesh& mesh,
                                  const TensorMeta& meta, int64_t device);

struct Piece {
  int64_t sender = 0;
  int64_t receiver = 0;
  std::vector<int64_t> src_lo, dst_lo, ext;  // local coordinates / extents
  int64_t elements() const {
    int64_t n = 1;
    for (int64_t e : ext) n *= e;
    return n;
  }
};

// Pieces `receiver` needs for a direct src->tgt redistribution, ordered by
// sender index. The sender of each piece is the source replica agreeing with
// the receiver on every axis `src` does not use.
std::vector<Piece> pieces_for_receiver(const ShardingSpec& src, const ShardingSpec& tgt,
                                       const DeviceMesh& mesh, const TensorMeta& meta,
                                       int64_t receiver);

// Pieces `sender` must provide, ordered by receiver index (same pieces as
// the receiver view, seen from the other end).
std::vector<Piece> pieces_for_sender(const ShardingSpec& src, const ShardingSpec& tgt,
                                     const DeviceMesh& mesh, const TensorMeta& meta,
                                     int64_t sender);

// A strided byte copy: `rows` (outer dims, up to kMaxDims-1, innermost last)
// of `run_bytes` contiguous bytes each.
struct CopyDesc {
  static constexpr int kMaxFan = 8;
  int src_buf = 0;  // index into the launch's source pointer table
  int dst_buf = 0;  // index into the launch's destination pointer table
  int ndst = 1;     // fan-out: the same bytes also land in extra_dst[0..ndst-2]
  int extra_dst[kMaxFan - 1] = {};
  // Split form (ksplit > 1): chunk j of each source row (src_off + j *
  // split_src_step) goes to buffer split_dst[j] at split_dst_off[j].
  int ksplit = 1;
  int64_t split_src_step = 0;
  int split_dst[kMaxFan] = {};
  int64_t split_dst_off[kMaxFan] = {};
  int64_t src_off = 0, dst_off = 0;  // bytes
  int64_t run_bytes = 0;
  int nouter = 0;
  int64_t ext[kMaxDims - 1] = {};
  int64_t src_stride[kMaxDims - 1] = {};  // bytes
  int64_t dst_stride[kMaxDims - 1] = {};  // bytes
  int64_t bytes() const {  // bytes read (= written per destination)
    int64_t n = run_bytes * ksplit;
    for (int i = 0; i < nouter; ++i) n *= ext[i];
    return n;
  }
};

// Copy of box `ext` from (src_shape, src_lo) to (dst_shape, dst_lo) with
// adjacent dims merged whenever both sides are contiguous across them.
CopyDesc make_copy(int src_buf, const std::vector<int64_t>& src_shape,
                   const std::vector<int64_t>& src_lo, int dst_buf,
                   const std::vector<int64_t>& dst_shape, const std::vector<int64_t>& dst_lo,
                   const std::vector<int64_t>& ext, int elem_bytes);

// Merges descriptors with short runs (< 64 B) that read adjacent chunks of
// the same source rows (same buffer, outer extents and strides, source
// offsets run_bytes apart) into split descriptors of up to 8 chunks.
void merge_splits(std::vector<CopyDesc>& descs);

// True when the box is one contiguous run inside an array of `shape`.
bool box_contiguous(const std::vector<int64_t>& shape, const std::vector<int64_t>& ext);
int64_t box_offset(const std::vector<int64_t>& shape, const std::vector<int64_t>& lo);

// Mesh axes along which sender and receiver differ for some piece of this
// redistribution (the collective's group axes).
std::vector<int> active_axes(const ShardingSpec& src, const ShardingSpec& tgt,
                             const DeviceMesh& mesh, const TensorMeta& meta);

}  // namespace apl
