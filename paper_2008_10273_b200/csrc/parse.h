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

// MSB-first reader with a hard bit limit (reference bits.py:41-78).
struct BitReader {
    const uint8_t* d;
    size_t nbytes;
    uint64_t limit;
    uint64_t pos = 0;
    BitReader(const uint8_t* data, size_t nb, uint64_t nbits) : d(data), nbytes(nb), limit(nbits) {
        if (nbits > (uint64_t)nb * 8) fail(HIVC_E_TRUNCATED_STREAM, "bit length exceeds buffer");
    }
    inline uint32_t bit() {
        if (pos + 1 > limit) fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
        uint32_t b = (d[pos >> 3] >> (7 - (pos & 7))) & 1u;
        ++pos;
        return b;
    }
    inline uint32_t take(int n) {  // n <= 32
        if (n == 0) return 0;
        if (pos + (uint64_t)n > limit) fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
        uint64_t byte = pos >> 3;
        int off = (int)(pos & 7);
        uint64_t v = 0;
        for (int i = 0; i < 5; ++i) v = (v << 8) | (byte + i < nbytes ? d[byte + i] : 0u);
        pos += (uint64_t)n;
        return (uint32_t)((v >> (40 - off - n)) & ((1ull << n) - 1));
    }
};

uint64_t read_uvarint(const uint8_t* d, size_t len, size_t& pos);

// tANS decode tables for one normalised distribution (entropy.py:108-130).
struct FseTable {
    int table_log = 0;
    std::vector<uint16_t> sym;
    std::vector<uint32_t> x;
    std::vector<uint8_t> nb;
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
void parse_flow_tree(BitReader& rd, int32_t w, int32_t h, std::vector<int32_t>& nodes, int32_t& nleaves);

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
};
// prediction.decode_intra (prediction.py:185-208), parse half; returns next pos.
size_t parse_intra(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int channels, int levels,
                   IntraJob& job, std::vector<uint64_t>& scratch_bits);

struct FlowJob {
    std::vector<int32_t> nodes[2];   // u, v trees
    std::vector<double> vals[2];
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
