// TMA tensor-tile copy engine (tile_copy.cu): descriptors with short strided
// rows move as 2-D..5-D tensor boxes. Host and device share these layouts.
#pragma once

#include <cuda.h>

#include <cstdint>

#include "box_copy.cuh"

namespace apl {

constexpr int kTileBoxBytes = 16384;  // one shared-memory stage = one box
constexpr int kTileMaxDesc = 40;      // descriptors per launch (parameter space)
constexpr int kTileMaxMaps = 88;      // tensor maps per launch (source + destinations)
constexpr int kTileMaxFan = 4;

// One descriptor's box grid: units enumerate boxes with dim 0 fastest.
struct TileDesc {
  int64_t unit_begin;
  FastDiv nb[5];     // boxes per tensor dim
  int box[5];        // box extent per dim (elements; dims >= 2 are 1)
  int rank;          // tensor rank 2..5
  int src_map;       // index into TileArgs::maps
  int dst_map;       // first destination map (ndst consecutive)
  int ndst;
  int box_bytes;     // full box (TMA counts zero-filled OOB elements too)
};

struct TileArgs {
  CUtensorMap maps[kTileMaxMaps];
  TileDesc d[kTileMaxDesc];
  int ndesc;
  int64_t first, total;  // this launch's units [first, total)
};

static_assert(sizeof(TileArgs) <= 32000, "kernel parameter space");

}  // namespace apl
