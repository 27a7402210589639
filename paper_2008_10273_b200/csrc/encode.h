// Host-side, bit-exact encoder primitives (the inverses of parse.h):
// MSB-first bit writer, LEB128, tANS symbol payloads (entropy.py:68-172,
// 219-308), subdivision trees (subdivision.py:76-130,178-181).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "common.h"

namespace hivc {

// bits.BitWriter (bits.py:10-38)
struct BitWriter {
    std::vector<uint8_t> bytes;
    uint64_t acc = 0;
    int nbits = 0;
    void write(uint64_t value, int count);  // count <= 32
    uint64_t size_bits() const { return bytes.size() * 8 + (uint64_t)nbits; }
    void append_to(std::vector<uint8_t>& out) const;  // final partial byte zero-padded
};

void write_uvarint(std::vector<uint8_t>& out, uint64_t v);

// entropy.normalize_counts (entropy.py:68-106)
std::vector<int64_t> normalize_counts(const std::vector<int64_t>& hist, int table_log);
// entropy.encode_symbols (entropy.py:255-273); table_log < 0: automatic (entropy.py:243-252)
void encode_symbols(const int64_t* symbols, size_t n, int table_log, std::vector<uint8_t>& out);
// entropy.encode_signed_values (entropy.py:294-308)
void encode_signed_values(const int64_t* values, size_t n, int table_log, std::vector<uint8_t>& out);

}  // namespace hivc

namespace hivc {

// subdivision.subdivide_by_error (subdivision.py:76-130) with the error of
// region_ssd (one plane) or joint_ssd_error (several planes, subdivision.py:
// 133-144), float64 sums in numpy's association order (sum_region below);
// optional min_error early stop.  Appends the preorder tree bits to `bits`
// (serialize_tree, subdivision.py:178-181) and returns the preorder leaves
// (x, y, w, h) — SubdivisionTree.leaves().
struct Rect4 {
    int32_t x, y, w, h;
};
void subdivide_by_error(const double* const* planes, int nplanes, int32_t W, int32_t H, int64_t target,
                        bool use_min_error, double min_error, BitWriter& bits, std::vector<Rect4>& leaves);

// np.sum(plane[y:y+h, x:x+w]) for a C-contiguous float64 plane of width W:
// one pairwise sum when the view is contiguous, else numpy's buffered
// reduction (whole-row chunks of at most 8192 elements, each pairwise summed
// and accumulated in order).
double sum_region(const double* plane, int32_t W, int32_t x, int32_t y, int32_t w, int32_t h);
// numpy's pairwise summation of n contiguous doubles
double np_pairwise(const double* a, int64_t n);

}  // namespace hivc

namespace hivc {

// codec._plan_group (codec.py:118-137) for every raster 8x8 tile of h x w
// integer residual planes: coded[t] = 0 when the tile is zero in all planes;
// otherwise the tile's subdivision tree with min(points, bh*bw) leaves
// (joint SSD over the planes), its preorder bits (tree_bits[16 t ..], MSB
// first, tree_nbits[t] bits) and its 8x8 mask word (bit y*8+x at each leaf's
// floor midpoint, subdivision.py:147-152).  Tiles run on `threads` threads.
void plan_residual_tiles(const int64_t* const* planes, int nplanes, int32_t h, int32_t w, int32_t points,
                         int threads, uint8_t* coded, uint64_t* masks, uint8_t* tree_bits, uint8_t* tree_nbits);

}  // namespace hivc
