// Exchange planning for layout conversions (host side).
//
// The step semantics this restates are the reference's layout pass
// (proj/src/layout.cpp:178-219, spec level) applied to data with the SURVEY
// Appendix A placement; see oracle/apl_oracle.c for the independent CPU
// restatement the GPU results are checked against.
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <string>
#include <stdexcept>

namespace apl {

namespace {

int64_t split_of(const autoplan::DimSpec& dim, const DeviceMesh& mesh) {
  int64_t p = 1;
  for (int a : dim.axes) p *= mesh.shape[static_cast<size_t>(a)];
  return p;
}

// Writes block index `s` of `dim` back into mesh coordinates (last-listed
// axis is the least significant digit).
void scatter_block_index(const autoplan::DimSpec& dim, const DeviceMesh& mesh, int64_t s,
                         std::vector<int64_t>& coord) {
  for (size_t i = dim.axes.size(); i-- > 0;) {
    const int a = dim.axes[i];
    const int64_t n = mesh.shape[static_cast<size_t>(a)];
    coord[static_cast<size_t>(a)] = s % n;
    s /= n;
  }
}

std::vector<int64_t> row_major_strides(const std::vector<int64_t>& shape) {
  std::vector<int64_t> st(shape.size(), 1);
  for (size_t i = shape.size(); i-- > 1;) st[i - 1] = st[i] * shape[i];
  return st;
}

}  // namespace

std::vector<int64_t> local_shape(const ShardingSpec& spec, const DeviceMesh& mesh,
                                 const TensorMeta& meta) {
  std::vector<int64_t> out(meta.shape.size());
  for (size_t d = 0; d < meta.shape.size(); ++d)
    out[d] = meta.shape[d] / split_of(spec.dims[d], mesh);
  return out;
}

std::vector<int64_t> block_origin(const ShardingSpec& spec, const DeviceMesh& mesh,
                                  const TensorMeta& meta, int64_t device) {
  const std::vector<int64_t> coord = mesh.coord_of(device);
  std::vector<int64_t> lo(meta.shape.size());
  for (size_t d = 0; d < meta.shape.size(); ++d) {
    int64_t s = 0;
    for (int a : spec.dims[d].axes)
      s = s * mesh.shape[static_cast<size_t>(a)] + coord[static_cast<size_t>(a)];
    lo[d] = s * (meta.shape[d] / split_of(spec.dims[d], mesh));
  }
  return lo;
}

std::vector<Piece> pieces_for_receiver(const ShardingSpec& src, const ShardingSpec& tgt,
                                       const DeviceMesh& mesh, const TensorMeta& meta,
                                       int64_t receiver) {
  const size_t k = meta.shape.size();
  const std::vector<int64_t> ls = local_shape(src, mesh, meta);
  const std::vector<int64_t> lt = local_shape(tgt, mesh, meta);
  const std::vector<int64_t> ot = block_origin(tgt, mesh, meta, receiver);
  const std::vector<int64_t> home = mesh.coord_of(receiver);

  // Per dim: the source block indices overlapping the receiver's target range.
  std::vector<int64_t> first(k), count(k);
  int64_t combos = 1;
  for (size_t d = 0; d < k; ++d) {
    if (lt[d] == 0 || ls[d] == 0) return {};
    first[d] = ot[d] / ls[d];
    count[d] = (ot[d] + lt[d] - 1) / ls[d] - first[d] + 1;
    combos *= count[d];
  }
  std::vector<Piece> out;
  out.reserve(static_cast<size_t>(combos));
  std::vector<int64_t> idx(k, 0);
  for (int64_t c = 0; c < combos; ++c) {
    int64_t rest = c;
    for (size_t d = k; d-- > 0;) {
      idx[d] = first[d] + rest % count[d];
      rest /= count[d];
    }
    std::vector<int64_t> coord = home;
    Piece p;
    p.receiver = receiver;
    p.src_lo.resize(k);
    p.dst_lo.resize(k);
    p.ext.resize(k);
    for (size_t d = 0; d < k; ++d) {
      scatter_block_index(src.dims[d], mesh, idx[d], coord);
      const int64_t s_lo = idx[d] * ls[d];
      const int64_t lo = std::max(ot[d], s_lo);
      const int64_t hi = std::min(ot[d] + lt[d], s_lo + ls[d]);
      p.src_lo[d] = lo - s_lo;
      p.dst_lo[d] = lo - ot[d];
      p.ext[d] = hi - lo;
    }
    p.sender = mesh.device_of(coord);
    out.push_back(std::move(p));
  }
  std::stable_sort(out.begin(), out.end(),
                   [](const Piece& a, const Piece& b) { return a.sender < b.sender; });
  return out;
}

std::vector<Piece> pieces_for_sender(const ShardingSpec& src, const ShardingSpec& tgt,
                                     const DeviceMesh& mesh, const TensorMeta& meta,
                                     int64_t sender) {
  const size_t k = meta.shape.size();
  const std::vector<int64_t> ls = local_shape(src, mesh, meta);
  const std::vector<int64_t> lt = local_shape(tgt, mesh, meta);
  const std::vector<int64_t> os = block_origin(src, mesh, meta, sender);
  const std::vector<int64_t> home = mesh.coord_of(sender);
  const std::vector<int> free_axes = src.used_axes();

  int64_t combos = 1;
  for (int a : free_axes) combos *= mesh.shape[static_cast<size_t>(a)];
  std::vector<Piece> out;
  for (int64_t c = 0; c < combos; ++c) {
    std::vector<int64_t> coord = home;
    int64_t rest = c;
    for (size_t i = free_axes.size(); i-- > 0;) {
      const int a = free_axes[i];
      coord[static_cast<size_t>(a)] = rest % mesh.shape[static_cast<size_t>(a)];
      rest /= mesh.shape[static_cast<size_t>(a)];
    }
    const int64_t receiver = mesh.device_of(coord);
    const std::vector<int64_t> ot = block_origin(tgt, mesh, meta, receiver);
    Piece p;
    p.sender = sender;
    p.receiver = receiver;
    p.src_lo.resize(k);
    p.dst_lo.resize(k);
    p.ext.resize(k);
    bool empty = false;
    for (size_t d = 0; d < k && !empty; ++d) {
      const int64_t lo = std::max(os[d], ot[d]);
      const int64_t hi = std::min(os[d] + ls[d], ot[d] + lt[d]);
      if (hi <= lo) {
        empty = true;
        break;
      }
      p.src_lo[d] = lo - os[d];
      p.dst_lo[d] = lo - ot[d];
      p.ext[d] = hi - lo;
    }
    if (!empty) out.push_back(std::move(p));
  }
  std::stable_sort(out.begin(), out.end(),
                   [](const Piece& a, const Piece& b) { return a.receiver < b.receiver; });
  return out;
}

bool box_contiguous(const std::vector<int64_t>& shape, const std::vector<int64_t>& ext) {
  // Contiguous iff: unit extents, then at most one partial dim, then full dims.
  size_t i = 0;
  while (i < shape.size() && ext[i] == 1) ++i;
  if (i == shape.size()) return true;
  ++i;  // the (possibly partial) leading non-unit dim
  for (; i < shape.size(); ++i)
    if (ext[i] != shape[i]) return false;
  return true;
}

int64_t box_offset(const std::vector<int64_t>& shape, const std::vector<int64_t>& lo) {
  const std::vector<int64_t> st = row_major_strides(shape);
  int64_t off = 0;
  for (size_t i = 0; i < shape.size(); ++i) off += lo[i] * st[i];
  return off;
}

CopyDesc make_copy(int src_buf, const std::vector<int64_t>& src_shape,
                   const std::vector<int64_t>& src_lo, int dst_buf,
                   const std::vector<int64_t>& dst_shape, const std::vector<int64_t>& dst_lo,
                   const std::vector<int64_t>& ext, int elem_bytes) {
  const size_t k = ext.size();
  const std::vector<int64_t> ss = row_major_strides(src_shape);
  const std::vector<int64_t> ds = row_major_strides(dst_shape);

  CopyDesc c;
  c.src_buf = src_buf;
  c.dst_buf = dst_buf;
  c.src_off = box_offset(src_shape, src_lo) * elem_bytes;
  c.dst_off = box_offset(dst_shape, dst_lo) * elem_bytes;

  struct Dim {
    int64_t e, s, d;
  };
  std::vector<Dim> dims;  // outer -> inner, unit extents dropped
  for (size_t i = 0; i < k; ++i)
    if (ext[i] != 1) dims.push_back({ext[i], ss[i], ds[i]});

  // Contiguous run: innermost dims with unit stride on both sides.
  int64_t run = 1;
  while (!dims.empty() && dims.back().s == run && dims.back().d == run) {
    run *= dims.back().e;
    dims.pop_back();
  }
  c.run_bytes = run * elem_bytes;

  // Merge remaining outer dims where both sides are dense across them.
  std::vector<Dim> merged;
  for (size_t i = dims.size(); i-- > 0;) {
    if (!merged.empty()) {
      Dim& inner = merged.back();
      if (dims[i].s == inner.e * inner.s && dims[i].d == inner.e * inner.d) {
        inner.e *= dims[i].e;
        continue;
      }
    }
    merged.push_back(dims[i]);
  }
  std::reverse(merged.begin(), merged.end());
  if (merged.size() > static_cast<size_t>(kMaxDims - 1))
    throw std::runtime_error("copy descriptor exceeds the supported rank");
  c.nouter = static_cast<int>(merged.size());
  for (size_t i = 0; i < merged.size(); ++i) {
    c.ext[i] = merged[i].e;
    c.src_stride[i] = merged[i].s * elem_bytes;
    c.dst_stride[i] = merged[i].d * elem_bytes;
  }
  return c;
}

void merge_splits(std::vector<CopyDesc>& descs) {
  static const int64_t kShortRun = [] {  // APL_SPLIT_RUN: experiment knob
    const char* e = std::getenv("APL_SPLIT_RUN");
    return e ? std::atoll(e) : int64_t{64};
  }();
  static const bool enabled = [] {
    const char* e = std::getenv("APL_SPLIT");  // "0" disables (A/B measurements)
    return e == nullptr || std::string(e) != "0";
  }();
  if (!enabled) return;
  // Bucket candidates by everything but the source offset / destination.
  std::map<std::vector<int64_t>, std::vector<size_t>> buckets;
  for (size_t i = 0; i < descs.size(); ++i) {
    const CopyDesc& d = descs[i];
    if (d.run_bytes >= kShortRun || d.ndst != 1 || d.ksplit != 1 || d.nouter == 0) continue;
    std::vector<int64_t> key{d.src_buf, d.run_bytes, d.nouter};
    for (int j = 0; j < d.nouter; ++j) {
      key.push_back(d.ext[j]);
      key.push_back(d.src_stride[j]);
      key.push_back(d.dst_stride[j]);
    }
    buckets[key].push_back(i);
  }
  std::vector<char> gone(descs.size(), 0);
  std::vector<CopyDesc> merged;
  for (auto& [key, idx] : buckets) {
    std::sort(idx.begin(), idx.end(),
              [&](size_t a, size_t b) { return descs[a].src_off < descs[b].src_off; });
    size_t i = 0;
    while (i < idx.size()) {
      // Longest run of chunks exactly run_bytes apart, at most kMaxFan.
      size_t j = i + 1;
      while (j < idx.size() && j - i < static_cast<size_t>(CopyDesc::kMaxFan) &&
             descs[idx[j]].src_off == descs[idx[j - 1]].src_off + descs[idx[i]].run_bytes)
        ++j;
      if (j - i >= 2) {
        CopyDesc s = descs[idx[i]];
        s.ksplit = static_cast<int>(j - i);
        s.split_src_step = s.run_bytes;
        for (size_t t = i; t < j; ++t) {
          s.split_dst[t - i] = descs[idx[t]].dst_buf;
          s.split_dst_off[t - i] = descs[idx[t]].dst_off;
          gone[idx[t]] = 1;
        }
        merged.push_back(s);
      }
      i = j;
    }
  }
  if (merged.empty()) return;
  std::vector<CopyDesc> out;
  for (size_t i = 0; i < descs.size(); ++i)
    if (!gone[i]) out.push_back(descs[i]);
  out.insert(out.end(), merged.begin(), merged.end());
  descs.swap(out);
}

std::vector<int> active_axes(const ShardingSpec& src, const ShardingSpec& tgt,
                             const DeviceMesh& mesh, const TensorMeta& meta) {
  std::vector<char> differs(mesh.shape.size(), 0);
  for (int64_t q = 0; q < mesh.num_devices(); ++q) {
    const std::vector<int64_t> cq = mesh.coord_of(q);
    for (const Piece& p : pieces_for_receiver(src, tgt, mesh, meta, q)) {
      if (p.sender == q) continue;
      const std::vector<int64_t> cp = mesh.coord_of(p.sender);
      for (size_t a = 0; a < cq.size(); ++a)
        if (cp[a] != cq[a]) differs[a] = 1;
    }
  }
  std::vector<int> axes;
  for (size_t a = 0; a < differs.size(); ++a)
    if (differs[a]) axes.push_back(static_cast<int>(a));
  return axes;
}

}  // namespace apl
