// Host-side, bit-exact parsing of the HIVC container and payloads.
//
// Everything here is sequential integer work (MSB-first bit reads, LEB128,
// tANS state machine, preorder subdivision trees).  It runs on the CPU and
// produces compact, device-ready descriptions of each frame (mask point
// lists, flow trees, coded-block masks and quantised symbols); the float
// work happens in the CUDA kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "common.h"

namespace hivc {

// MSB-first reader with a hard bit limit (reference bits.py:41-78), with a
// 64-bit look-ahead buffer: the next `avail` bits sit at the top of `buf`.
struct BitReader {
    const uint8_t* d;
    size_t nbytes;
    uint64_t limit;
    uint64_t pos = 0;
    uint64_t buf = 0;
    int avail = 0;
    size_t next = 0;
    BitReader(const uint8_t* data, size_t nb, uint64_t nbits) : d(data), nbytes(nb), limit(nbits) {
        if (nbits > (uint64_t)nb * 8) fail(HIVC_E_TRUNCATED_STREAM, "bit length exceeds buffer");
    }
    inline void refill() {
        while (avail <= 56 && next < nbytes) {
            buf |= (uint64_t)d[next++] << (56 - avail);
            avail += 8;
        }
    }
    void seek(uint64_t bitpos) {  // absolute bit position
        pos = bitpos;
        next = (size_t)(bitpos >> 3);
        buf = 0;
        avail = 0;
        refill();
        const int drop = (int)(bitpos & 7);
        if (drop && avail >= drop) {
            buf <<= drop;
            avail -= drop;
        }
    }
    inline uint32_t bit() {
        if (pos >= limit) fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
        if (avail == 0) refill();
        const uint32_t b = (uint32_t)(buf >> 63);
        buf <<= 1;
        --avail;
        ++pos;
        return b;
    }
    // the next 12 bits without consuming them (zeros past the data)
    inline uint32_t peek12() {
        if (avail < 12) refill();
        return (uint32_t)(buf >> 52);
    }
    // consume n <= 12 bits known to lie inside the limit (after peek12)
    inline void skip(int n) {
        buf <<= n;
        avail -= n;
        pos += (uint64_t)n;
    }
    inline uint32_t take(int n) {  // n <= 32
        if (n == 0) return 0;
        if (pos + (uint64_t)n > limit) fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
        if (avail < n) refill();
        const uint32_t v = (uint32_t)(buf >> (64 - n));
        buf <<= n;
        avail -= n;
        pos += (uint64_t)n;
        return v;
    }
};

// Preorder walk of one serialised subdivision tree (subdivision.py:198-222):
// bit 1 halves the longer side (ties halve the width, first half rounded up),
// bit 0 is a leaf -> on_leaf(x, y, w, h).  The explicit stack never holds
// more than (tree depth + 1) rectangles.
template <class F>
inline void walk_tree(BitReader& rd, int32_t w, int32_t h, F&& on_leaf) {
    int32_t st[4 * 130];
    int sp = 0;
    st[0] = 0;
    st[1] = 0;
    st[2] = w;
    st[3] = h;
    sp = 1;
    while (sp) {
        --sp;
        const int32_t x = st[4 * sp], y = st[4 * sp + 1], rw = st[4 * sp + 2], rh = st[4 * sp + 3];
        if (rd.bit()) {
            if (rw == 1 && rh == 1) fail(HIVC_E_SUBDIVISION, "split of a single pixel");
            if (sp + 2 > 130) fail(HIVC_E_SUBDIVISION, "subdivision tree too deep");
            int32_t* a = st + 4 * sp;
            if (rh > rw) {
                const int32_t t = (rh + 1) / 2;
                a[0] = x, a[1] = y + t, a[2] = rw, a[3] = rh - t;  // second child, popped last
                a[4] = x, a[5] = y, a[6] = rw, a[7] = t;
            } else {
                const int32_t t = (rw + 1) / 2;
                a[0] = x + t, a[1] = y, a[2] = rw - t, a[3] = rh;
                a[4] = x, a[5] = y, a[6] = t, a[7] = rh;
            }
            sp += 2;
        } else {
            on_leaf(x, y, rw, rh);
        }
    }
}

uint64_t read_uvarint(const uint8_t* d, size_t len, size_t& pos);

// tANS decode tables for one normalised distribution (entropy.py:108-130).
// Entry: symbol, bit count nb and base = x << nb, so the next state is
// base | the next nb bits (fse_decode, entropy.py:175-211).
struct FseTable {
    struct Entry {
        uint32_t base;
        uint16_t sym;
        uint8_t nb;
    };
    int table_log = 0;
    std::vector<Entry> dec;
    void build(const std::vector<uint64_t>& counts, int table_log);
};

// entropy.decode_symbols (entropy.py:276-291); returns next position.
size_t decode_symbols(const uint8_t* d, size_t len, size_t pos, std::vector<int32_t>& out);
// entropy.decode_signed_values (entropy.py:311-338); returns next position.
size_t decode_signed_values(const uint8_t* d, size_t len, size_t pos, std::vector<int32_t>& out);

struct Rect {
    int32_t x, y, w, h;
};
// Preorder leaves of one serialised tree (subdivision.py:198-222 / 183-195).
void parse_tree_leaves(BitReader& rd, int32_t w, int32_t h, std::vector<Rect>& leaves);

// Flow tree flattened for device traversal.  Nodes in preorder: node i has
// code = nodes[2i] (0 leaf, 1 split on x, 2 split on y) in the low 2 bits and
// the absolute split coordinate above; nodes[2i+1] = right child index for a
// split (the left child is i+1) or the leaf's value index.
void parse_flow_tree(BitReader& rd, int32_t w, int32_t h, std::vector<int32_t>& nodes, int32_t& nleaves,
                     std::vector<Rect>* leaves = nullptr);

// One flow component (flow._decompress_plane, flow.py:343-356): leaf
// rectangles in preorder and their dequantised values (quantize.py:78-82),
// with the reference's error classes in its order; returns the next position.
size_t parse_flow_component(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int levels,
                            std::vector<Rect>& leaves, std::vector<double>& vals);

struct StreamHeader {
    int32_t width, height, frame_count, fps_num, fps_den, gop_size, channels;
    int32_t intra_levels, flow_levels, residual_levels;
};
constexpr size_t HEADER_SIZE = 22;
StreamHeader parse_header(const uint8_t* d, size_t len);
// read_stream (bitstream.py:132-154): GOP payload (offset, length) list.
void split_gops(const uint8_t* d, size_t len, const StreamHeader& h, std::vector<std::pair<size_t, size_t>>& gops);

// ---------------------------------------------------------------- frame payloads

struct IntraJob {
    // one mask per tree (Y; shared chroma tree when channels == 3)
    std::vector<int32_t> pts[2];    // raster-sorted flat indices of mask points
    std::vector<double> vals[3];    // per channel, raster order of its mask's points
    int nchan = 1;
    std::vector<int32_t> idx[3];    // scratch: quantised values
    std::vector<uint64_t> local;    // scratch: per-subtree bitmaps
};
// prediction.decode_intra (prediction.py:185-208), parse half; returns next pos.
size_t parse_intra(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int channels, int levels,
                   IntraJob& job, std::vector<uint64_t>& scratch_bits);

struct FlowJob {
    std::vector<int32_t> nodes[2];   // u, v trees
    std::vector<double> vals[2];
    // per 8x8 tile: index of the leaf covering the whole tile (< 0x8000), else
    // 0x8000 + the deepest node containing the tile (the device walks the tree
    // per pixel from there), or 0xFFFF (walk from the root)
    std::vector<uint16_t> tiles[2];
};
// flow.decompress_flow (flow.py:343-372); returns next pos.
size_t parse_flow(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int levels, FlowJob& job);

struct ResidualGroup {
    int nplanes = 1;
    int32_t nblocks = 0;
    int32_t npoints = 0;                  // mask points over all blocks (one plane)
    std::vector<uint64_t> tile_words;     // bit (t % 64) of word t/64 = tile t coded
    std::vector<int32_t> word_prefix;     // coded tiles before word i
    std::vector<uint64_t> block_mask;     // per coded block, bit y*8+x
    std::vector<int32_t> block_off;       // per coded block, first point index
    std::vector<int32_t> c_sym;           // plane-major: nplanes * npoints
    std::vector<int32_t> a_sym;           // plane-major: nplanes * nblocks
};
struct ResidualJob {
    bool zero = true;                     // marker 0: all-zero residual
    double c_scale = 1.0, a_scale = 1.0;  // c_fp / 65536, a_fp / 65536
    int ngroups = 0;
    ResidualGroup g[2];
};
// codec._decode_residual (codec.py:248-340), parse half; returns next pos.
size_t parse_residual(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int channels, ResidualJob& job);

}  // namespace hivc
