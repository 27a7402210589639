// Bit-exact host parsing of HIVC payloads.  Reference citations per function.
#include "parse.h"

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>

#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

namespace hivc {

// bit-reversed bytes: MSB-first bitmap byte -> LSB-first tile bits
static const struct BitRev {
    uint8_t t[256];
    constexpr BitRev() : t() {
        for (int i = 0; i < 256; ++i) {
            int r = 0;
            for (int b = 0; b < 8; ++b)
                if (i & (1 << b)) r |= 1 << (7 - b);
            t[i] = (uint8_t)r;
        }
    }
    uint8_t operator[](int i) const { return t[i]; }
} kBitReverse;

static inline uint32_t rd_u32(const uint8_t* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}
static inline uint16_t rd_u16(const uint8_t* p) {
    uint16_t v;
    std::memcpy(&v, p, 2);
    return v;
}

uint64_t read_uvarint(const uint8_t* d, size_t len, size_t& pos) {  // bits.py:95-108
    uint64_t v = 0;
    int shift = 0;
    while (true) {
        if (pos >= len) fail(HIVC_E_TRUNCATED_STREAM, "varint runs past end of buffer");
        uint8_t b = d[pos++];
        if (shift == 63 && (b & 0x7F) > 1) v = ~0ull;  // >= 2^64: saturate (only ever fails later checks)
        else if (shift < 64) v |= (uint64_t)(b & 0x7F) << shift;
        if (!(b & 0x80)) return v;
        shift += 7;
        if (shift > 63) fail(HIVC_E_ARGUMENT, "varint too long");
    }
}

void FseTable::build(const std::vector<uint64_t>& counts, int tl) {  // entropy.py:108-130
    table_log = tl;
    const uint32_t size = 1u << tl;
    uint64_t total = 0;
    for (uint64_t c : counts) {
        total += c;
        if (c > size || total > size) fail(HIVC_E_ENTROPY, "normalized counts must sum to table size");
    }
    if (total != size) fail(HIVC_E_ENTROPY, "normalized counts must sum to table size");
    const uint32_t step = (size >> 1) + (size >> 3) + 3;
    std::vector<uint16_t> sym(size, 0);
    uint32_t k = 0;
    for (size_t s = 0; s < counts.size(); ++s)
        for (uint64_t j = 0; j < counts[s]; ++j) sym[(k++ * step) & (size - 1)] = (uint16_t)s;
    std::vector<uint32_t> next(counts.size());
    for (size_t s = 0; s < counts.size(); ++s) next[s] = (uint32_t)counts[s];
    dec.resize(size);
    for (uint32_t slot = 0; slot < size; ++slot) {
        const uint32_t xv = next[sym[slot]]++;
        const int bl = 32 - __builtin_clz(xv);  // xv >= 1
        const int nb = tl + 1 - bl;             // 0 <= nb <= tl
        dec[slot] = {xv << nb, sym[slot], (uint8_t)nb};
    }
}

namespace {
// MSB-first reader for the hot entropy loops: a 64-bit window refilled eight
// bytes at a time, no per-read limit check (reads past the data see zeros);
// the caller compares the consumed bit count with the limit once, which
// raises the same error a bit-by-bit reader would (fse_decode's loop has no
// other failure, entropy.py:175-211).
struct FastBits {
    const uint8_t* d;
    size_t nbytes, next = 0;
    uint64_t buf = 0;
    int avail = 0;
    FastBits(const uint8_t* p, size_t n) : d(p), nbytes(n) { refill(); }
    inline void refill() {
        if (avail > 56) return;
        if (next + 8 <= nbytes) {
            uint64_t v;
            std::memcpy(&v, d + next, 8);
            v = __builtin_bswap64(v);
            buf |= v >> avail;  // the partial byte below the whole ones is re-ORed identically next time
            const int nb = (63 - avail) >> 3;
            next += (size_t)nb;
            avail += nb * 8;
        } else {
            while (avail <= 56) {
                const uint64_t b = next < nbytes ? d[next] : 0;
                buf |= b << (56 - avail);
                ++next;
                avail += 8;
            }
        }
    }
    inline uint32_t take(int n) {  // 0 <= n <= 32, avail >= n
        const uint32_t v = n ? (uint32_t)(buf >> (64 - n)) : 0u;
        buf <<= n;
        avail -= n;
        return v;
    }
};
}  // namespace

size_t decode_symbols(const uint8_t* d, size_t len, size_t pos, std::vector<int32_t>& out) {
    // header: entropy.py:227-240
    if (pos >= len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    int tl = d[pos++];
    if (tl < 5 || tl > 12) fail(HIVC_E_ENTROPY, "bad table_log " + std::to_string(tl));
    uint64_t nsym = read_uvarint(d, len, pos);
    if (nsym == 0 || nsym > (1ull << tl)) fail(HIVC_E_ENTROPY, "bad alphabet size");
    std::vector<uint64_t> counts(nsym);
    for (uint64_t i = 0; i < nsym; ++i) counts[i] = read_uvarint(d, len, pos);
    // body: entropy.py:276-291
    if (pos + 10 > len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    uint32_t count = rd_u32(d + pos);
    uint32_t state = rd_u16(d + pos + 4);
    uint32_t bit_len = rd_u32(d + pos + 6);
    pos += 10;
    if (count > (1u << 28)) fail(HIVC_E_ENTROPY, "implausible symbol count " + std::to_string(count));
    size_t nbytes = ((size_t)bit_len + 7) / 8;
    if (pos + nbytes > len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    FseTable t;
    t.build(counts, tl);
    out.resize(count);
    if (count) {  // fse_decode, entropy.py:175-211
        const uint32_t size = 1u << tl;
        if (state < size || state >= 2 * size) fail(HIVC_E_ENTROPY, "corrupt stream: initial state out of range");
        FastBits rd(d + pos, nbytes);
        const FseTable::Entry* tab = t.dec.data();
        int32_t* o = out.data();
        uint64_t used = 0;
        for (uint32_t i = 0; i < count; ++i) {
            const FseTable::Entry e = tab[state - size];
            o[i] = e.sym;
            if (rd.avail < 12) rd.refill();  // nb <= table_log <= 12
            state = e.base + rd.take(e.nb);
            used += e.nb;
        }
        if (used > bit_len) fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
        if (state != size) fail(HIVC_E_ENTROPY, "corrupt stream: final state mismatch");
    }
    return pos + nbytes;
}

size_t decode_signed_values(const uint8_t* d, size_t len, size_t pos, std::vector<int32_t>& out) {
    // entropy.py:311-338: the category symbols, then the raw extra bits
    pos = decode_symbols(d, len, pos, out);
    if (pos + 4 > len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    uint32_t bit_len = rd_u32(d + pos);
    pos += 4;
    size_t nbytes = ((size_t)bit_len + 7) / 8;
    if (pos + nbytes > len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    uint64_t sum = 0;
    bool bad = false;
    for (int32_t c : out) {
        bad |= c > 16;
        sum += (uint64_t)c;
    }
    if (bad) fail(HIVC_E_ENTROPY, "bad category in stream");
    if (sum != bit_len) fail(HIVC_E_ENTROPY, "extra-bits length mismatch");
    FastBits rd(d + pos, nbytes);
    for (int32_t& v : out) {  // category -> value in place (from_category, entropy.py:52-60)
        const int k = v;
        if (rd.avail < 16) rd.refill();
        const int32_t e = (int32_t)rd.take(k);
        v = k == 0 ? 0 : (e >= (1 << (k - 1)) ? e : e - (1 << k) + 1);
    }
    return pos + nbytes;
}

// Residual block trees of full 8x8 tiles (codec.py:300-303, subdivision.py:
// 198-222) decoded by table: for every 12-bit look-ahead, the mask of the tree
// it starts with and the tree's bit count, when the tree ends within those 12
// bits and never splits a single pixel (nbits 0 otherwise: the bit-by-bit walk
// handles it, and raises the reference's error when there is one).  A K = 4
// tree is 7 bits.
static const struct BlockTreeLut {
    uint64_t mask[4096];
    uint8_t nbits[4096];
    BlockTreeLut() {
        for (uint32_t v = 0; v < 4096; ++v) {
            int32_t st[4 * 32];
            int sp = 1, used = 0;
            st[0] = 0, st[1] = 0, st[2] = 8, st[3] = 8;
            uint64_t m = 0;
            bool ok = true;
            while (sp && ok) {
                --sp;
                const int32_t x = st[4 * sp], y = st[4 * sp + 1], rw = st[4 * sp + 2], rh = st[4 * sp + 3];
                if (used == 12) {
                    ok = false;
                    break;
                }
                const int b = (v >> (11 - used)) & 1;
                ++used;
                if (b) {
                    if (rw == 1 && rh == 1) {
                        ok = false;
                        break;
                    }
                    int32_t* a = st + 4 * sp;
                    if (rh > rw) {
                        const int32_t t = (rh + 1) / 2;
                        a[0] = x, a[1] = y + t, a[2] = rw, a[3] = rh - t;
                        a[4] = x, a[5] = y, a[6] = rw, a[7] = t;
                    } else {
                        const int32_t t = (rw + 1) / 2;
                        a[0] = x + t, a[1] = y, a[2] = rw - t, a[3] = rh;
                        a[4] = x, a[5] = y, a[6] = t, a[7] = rh;
                    }
                    sp += 2;
                } else {
                    m |= 1ull << ((y + rh / 2) * 8 + (x + rw / 2));
                }
            }
            mask[v] = ok ? m : 0;
            nbits[v] = ok ? (uint8_t)used : 0;
        }
    }
} kBlockTree;

void parse_tree_leaves(BitReader& rd, int32_t w, int32_t h, std::vector<Rect>& leaves) {
    walk_tree(rd, w, h, [&](int32_t x, int32_t y, int32_t rw, int32_t rh) { leaves.push_back({x, y, rw, rh}); });
}

void parse_flow_tree(BitReader& rd, int32_t w, int32_t h, std::vector<int32_t>& nodes, int32_t& nleaves,
                     std::vector<Rect>* leaves) {
    if (leaves) leaves->clear();
    // Same preorder walk as parse_tree_leaves (subdivision.py:183-195), but
    // recording the split structure.  The stack carries the index of the
    // parent whose right-child slot the popped rectangle fills (-1: none).
    struct Item {
        Rect r;
        int32_t parent_right;
    };
    std::vector<Item> st;
    st.push_back({{0, 0, w, h}, -1});
    nodes.clear();
    nleaves = 0;
    while (!st.empty()) {
        Item it = st.back();
        st.pop_back();
        int32_t idx = (int32_t)(nodes.size() / 2);
        if (it.parent_right >= 0) nodes[2 * it.parent_right + 1] = idx;
        const Rect& r = it.r;
        if (rd.bit()) {
            if (r.w == 1 && r.h == 1) fail(HIVC_E_SUBDIVISION, "cannot split a single pixel");
            if (r.h > r.w) {
                int32_t a = (r.h + 1) / 2;
                nodes.push_back(((r.y + a) << 2) | 2);
                nodes.push_back(-1);
                st.push_back({{r.x, r.y + a, r.w, r.h - a}, idx});
                st.push_back({{r.x, r.y, r.w, a}, -1});
            } else {
                int32_t a = (r.w + 1) / 2;
                nodes.push_back(((r.x + a) << 2) | 1);
                nodes.push_back(-1);
                st.push_back({{r.x + a, r.y, r.w - a, r.h}, idx});
                st.push_back({{r.x, r.y, a, r.h}, -1});
            }
        } else {
            nodes.push_back(0);
            nodes.push_back(nleaves++);
            if (leaves) leaves->push_back(r);
        }
    }
}

// Tile -> covering leaf map.  A tile inside one leaf gets the leaf's value
// index (< 0x8000); a tile straddling leaves gets 0x8000 + the deepest node
// whose rectangle contains the whole tile (the device walks from there), or
// 0xFFFF (walk from the root) when the indices do not fit 15 bits.  One
// preorder descent hands each node the block of tiles lying wholly inside
// it: a split passes its children the tiles wholly on their side and keeps
// the (at most one) row or column of tiles its split line crosses; a leaf
// takes all of its block.  Tiles are clipped to the plane (edge tiles).
static void flow_tile_map(const std::vector<int32_t>& nodes, int32_t nleaves, int32_t w, int32_t h,
                          std::vector<uint16_t>& tiles) {
    const int nbx = (w + 7) / 8, nby = (h + 7) / 8;
    tiles.assign((size_t)nbx * nby, 0xFFFF);
    if (nleaves >= 0x8000) return;  // all: per-pixel walk from the root
    struct Blk {
        int32_t node, tx0, tx1, ty0, ty1;
    };
    std::vector<Blk> st;
    st.push_back({0, 0, nbx, 0, nby});
    auto fill = [&](int32_t tx0, int32_t tx1, int32_t ty0, int32_t ty1, uint16_t v) {
        for (int32_t ty = ty0; ty < ty1; ++ty)
            std::fill(tiles.begin() + (size_t)ty * nbx + tx0, tiles.begin() + (size_t)ty * nbx + tx1, v);
    };
    while (!st.empty()) {
        const Blk b = st.back();
        st.pop_back();
        if (b.tx0 >= b.tx1 || b.ty0 >= b.ty1) continue;
        const int32_t a = nodes[2 * (size_t)b.node];
        const int code = a & 3, c = a >> 2;
        if (code == 0) {
            fill(b.tx0, b.tx1, b.ty0, b.ty1, (uint16_t)nodes[2 * (size_t)b.node + 1]);
            continue;
        }
        const uint16_t here = b.node < 0x7FFF ? (uint16_t)(0x8000 + b.node) : (uint16_t)0xFFFF;
        const int32_t left = b.node + 1, right = nodes[2 * (size_t)b.node + 1];
        if (code == 1) {  // x split: tiles with min(w, 8tx + 8) <= c go left, 8tx >= c right
            int32_t lo = std::min(c / 8, b.tx1), hi = std::max(std::min((c + 7) / 8, b.tx1), b.tx0);
            if (lo < b.tx0) lo = b.tx0;
            if (std::min(w, 8 * lo + 8) <= c) ++lo;  // (only when c is a multiple of 8 or at the clipped edge)
            lo = std::min(lo, b.tx1);
            hi = std::max(hi, lo);
            st.push_back({right, hi, b.tx1, b.ty0, b.ty1});
            st.push_back({left, b.tx0, lo, b.ty0, b.ty1});
            fill(lo, hi, b.ty0, b.ty1, here);
        } else {  // y split
            int32_t lo = std::min(c / 8, b.ty1), hi = std::max(std::min((c + 7) / 8, b.ty1), b.ty0);
            if (lo < b.ty0) lo = b.ty0;
            if (std::min(h, 8 * lo + 8) <= c) ++lo;
            lo = std::min(lo, b.ty1);
            hi = std::max(hi, lo);
            st.push_back({right, b.tx0, b.tx1, hi, b.ty1});
            st.push_back({left, b.tx0, b.tx1, b.ty0, lo});
            fill(b.tx0, b.tx1, lo, hi, here);
        }
    }
}

StreamHeader parse_header(const uint8_t* d, size_t len) {  // bitstream.py:102-121, 80-91
    if (len < HEADER_SIZE) fail(HIVC_E_TRUNCATED, "stream shorter than header");
    if (std::memcmp(d, "HIVC", 4) != 0) fail(HIVC_E_BAD_MAGIC, "not a compressed video stream");
    if (d[4] != 1) fail(HIVC_E_UNSUPPORTED_VERSION, "stream version " + std::to_string(d[4]) + ", expected 1");
    StreamHeader h;
    h.width = rd_u16(d + 5);
    h.height = rd_u16(d + 7);
    h.frame_count = (int32_t)rd_u32(d + 9);
    h.fps_num = rd_u16(d + 13);
    h.fps_den = rd_u16(d + 15);
    h.gop_size = d[17];
    h.channels = d[18];
    h.intra_levels = d[19] + 1;
    h.flow_levels = d[20] + 1;
    h.residual_levels = d[21];
    if (rd_u32(d + 9) > 0x7fffffffu) fail(HIVC_E_BITSTREAM, "frame count out of range");
    if (h.width < 1 || h.height < 1) fail(HIVC_E_BITSTREAM, "bad frame dimensions");
    if (h.channels != 1 && h.channels != 3) fail(HIVC_E_BITSTREAM, "channels must be 1 or 3");
    if (h.gop_size < 1) fail(HIVC_E_BITSTREAM, "gop_size out of range");
    if (h.intra_levels < 2 || h.flow_levels < 2) fail(HIVC_E_BITSTREAM, "quantizer levels out of range");
    if (h.residual_levels < 3 || h.residual_levels % 2 == 0)
        fail(HIVC_E_BITSTREAM, "residual_levels must be odd and >= 3");
    if (h.fps_num < 1 || h.fps_den < 1) fail(HIVC_E_BITSTREAM, "bad frame rate");
    return h;
}

void split_gops(const uint8_t* d, size_t len, const StreamHeader& h, std::vector<std::pair<size_t, size_t>>& gops) {
    size_t pos = HEADER_SIZE;  // bitstream.py:132-154
    gops.clear();
    while (pos < len) {
        if (pos + 4 > len) fail(HIVC_E_TRUNCATED, "group length prefix cut short");
        size_t n = rd_u32(d + pos);
        pos += 4;
        if (pos + n > len)
            fail(HIVC_E_TRUNCATED, "group payload " + std::to_string(gops.size()) + " cut short (" +
                                       std::to_string(len - pos) + " of " + std::to_string(n) + " bytes present)");
        gops.push_back({pos, n});
        pos += n;
    }
    size_t want = h.frame_count ? ((size_t)h.frame_count + h.gop_size - 1) / h.gop_size : 0;
    if (gops.size() != want)
        fail(HIVC_E_LENGTH_MISMATCH, "stream holds " + std::to_string(gops.size()) + " groups, header implies " +
                                         std::to_string(want));
}

// ---------------------------------------------------------------- intra payload

// Preorder walk of an intra mask tree (subdivision.py:198-222) with the
// current rectangle in registers: a split bit continues into the first child
// and pushes the second, a leaf bit ORs the leaf centre into the mask bitmap
// (prediction.py:117-119) and pops — selected without branches, since split
// and leaf bits alternate unpredictably.  Rectangles are packed 4 x 16 bits.
// Bits come from a look-ahead buffer without per-bit limit checks: reads past
// the tree's bit length see zeros (leaves, so the walk winds down) and the
// length is checked once at the end — and before reporting a bad split, so
// the error is the one a bit-by-bit reader raises first.  The bitmap has
// `stride` bits per row and its origin at plane pixel (x0, y0).
static uint64_t intra_tree_walk(const uint8_t* d, size_t nbytes, uint64_t nbits, uint64_t start, int32_t x, int32_t y,
                                int32_t w, int32_t h, int32_t x0, int32_t y0, size_t stride, uint64_t* bits,
                                size_t& nleaves) {
    constexpr int kCap = 128;  // >= log2(area) + 1 pending rectangles: unreachable (areas halve)
    uint64_t st[kCap + 2];
    size_t next = (size_t)(start >> 3);
    uint64_t buf = 0;
    int avail = 0;
    auto refill = [&]() {
        while (avail <= 56) {
            const uint64_t v = next < nbytes ? d[next] : 0;
            ++next;
            buf |= v << (56 - avail);
            avail += 8;
        }
    };
    refill();
    {
        const int drop = (int)(start & 7);
        buf <<= drop;
        avail -= drop;
    }
    uint64_t used = 0;
    uint64_t cur = (uint64_t)(uint16_t)x | (uint64_t)(uint16_t)y << 16 | (uint64_t)(uint16_t)w << 32 |
                   (uint64_t)(uint16_t)h << 48;
    int sp = 1;  // st[0] is a sentinel (never popped: the walk ends first)
    st[0] = 0;
    size_t nl = 0;
    for (;;) {
        if (avail == 0) refill();
        const uint32_t b = (uint32_t)(buf >> 63);
        buf <<= 1;
        --avail;
        ++used;
        const int32_t cx = (int32_t)(cur & 0xFFFF), cy = (int32_t)((cur >> 16) & 0xFFFF);
        const int32_t cw = (int32_t)((cur >> 32) & 0xFFFF), ch = (int32_t)(cur >> 48);
        if (b & (uint32_t)(cw == 1) & (uint32_t)(ch == 1)) {
            if (start + used > nbits) fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
            fail(HIVC_E_SUBDIVISION, "split of a single pixel");
        }
        const size_t i = (size_t)(cy + (ch >> 1) - y0) * stride + (size_t)(cx + (cw >> 1) - x0);
        bits[i >> 6] |= (uint64_t)(b ^ 1u) << (i & 63);
        nl += b ^ 1u;
        if (!b && sp == 1) break;
        const bool sh = ch > cw;  // halve the longer side, ties halve the width; first half rounded up
        const int32_t t = ((sh ? ch : cw) + 1) >> 1;
        const uint64_t first = sh ? (cur & 0x0000FFFFFFFFFFFFull) | (uint64_t)t << 48
                                  : (cur & 0xFFFF0000FFFFFFFFull) | (uint64_t)t << 32;
        const uint64_t second = sh ? (cur + ((uint64_t)t << 16)) - ((uint64_t)t << 48)
                                   : (cur + (uint64_t)t) - ((uint64_t)t << 32);
        const uint64_t popped = st[sp - 1];
        st[sp] = second;
        cur = b ? first : popped;
        sp += (int)(2 * b) - 1;
        if (sp > kCap) fail(HIVC_E_SUBDIVISION, "subdivision tree too deep");
    }
    if (start + used > nbits) fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
    nleaves = nl;
    return start + used;
}

// Excess tables over MSB-first bytes: a leaf bit (0) counts +1, a split (1)
// -1; a preorder subtree ends at the first bit where its excess reaches +1.
static const struct ExcessTables {
    int8_t net[256], maxp[256];
    ExcessTables() {
        for (int v = 0; v < 256; ++v) {
            int c = 0, m = -100;
            for (int k = 7; k >= 0; --k) {
                c += ((v >> k) & 1) ? -1 : 1;
                m = std::max(m, c);
            }
            net[v] = (int8_t)c;
            maxp[v] = (int8_t)m;
        }
    }
} kExcess;

// First bit after the preorder subtree that starts at bit s.
static uint64_t subtree_skip(const uint8_t* d, uint64_t nbits, uint64_t s) {
    uint64_t pos = s;
    int c = 0;
    while (pos < nbits) {
        if ((pos & 7) == 0 && pos + 8 <= nbits) {
            const uint8_t v = d[pos >> 3];
            if (c + kExcess.maxp[v] < 1) {
                c += kExcess.net[v];
                pos += 8;
                continue;
            }
        }
        c += ((d[pos >> 3] >> (7 - (pos & 7))) & 1) ? -1 : 1;
        ++pos;
        if (c == 1) return pos;
    }
    fail(HIVC_E_TRUNCATED_STREAM, "bit stream exhausted");
}

struct TreeTask {
    uint64_t start;
    int32_t x, y, w, h;
    size_t off = 0, stride = 0, nleaves = 0;  // local bitmap (words) and its row stride (bits)
    uint64_t end = 0;                         // first bit after the walked subtree
};

// Cut the tree at depth `depth` into independent subtrees (preorder).
static void tree_tasks(const uint8_t* d, uint64_t nbits, uint64_t s, int32_t x, int32_t y, int32_t w, int32_t h,
                       int depth, std::vector<TreeTask>& out) {
    if (depth == 0 || s >= nbits || !((d[s >> 3] >> (7 - (s & 7))) & 1) || (w == 1 && h == 1)) {
        out.push_back({s, x, y, w, h});
        return;
    }
    int32_t ax, ay, aw, ah, bx, by, bw, bh;
    if (h > w) {
        const int32_t t = (h + 1) / 2;
        ax = x, ay = y, aw = w, ah = t, bx = x, by = y + t, bw = w, bh = h - t;
    } else {
        const int32_t t = (w + 1) / 2;
        ax = x, ay = y, aw = t, ah = h, bx = x + t, by = y, bw = w - t, bh = h;
    }
    tree_tasks(d, nbits, s + 1, ax, ay, aw, ah, depth - 1, out);
    tree_tasks(d, nbits, subtree_skip(d, nbits, s + 1), bx, by, bw, bh, depth - 1, out);
}

// OR a (w x h) bitmap with a row stride of `stride` bits into the plane bitmap at (x0, y0).
static void merge_rect_bits(const uint64_t* src, size_t stride, int32_t x0, int32_t y0, int32_t w, int32_t h,
                            int32_t W, uint64_t* dst, size_t dst_words) {
    const size_t nw = ((size_t)w + 63) / 64;
    for (int32_t r = 0; r < h; ++r) {
        const uint64_t* row = src + (size_t)r * (stride / 64);
        const size_t g = (size_t)(y0 + r) * W + x0;
        for (size_t k = 0; k < nw; ++k) {
            uint64_t v = row[k];
            if (!v) continue;
            const size_t rem = (size_t)w - 64 * k;
            if (rem < 64) v &= (1ull << rem) - 1;
            const size_t gb = g + 64 * k, gw = gb >> 6, sh = gb & 63;
            dst[gw] |= v << sh;
            if (sh && gw + 1 < dst_words) dst[gw + 1] |= v >> (64 - sh);
        }
    }
}

// Run fn(i) for i in [0, n) on up to nthreads threads (the caller included).
// Helper threads run at a lower priority (nice +3) than the decode's parse
// workers: they soak up idle cores without delaying the smaller planes'
// parses that gate the first solve batch.
static void helper_priority() { setpriority(PRIO_PROCESS, (id_t)syscall(SYS_gettid), 3); }

template <class F>
static void parallel_for(int n, int nthreads, F&& fn) {
    std::atomic<int> next{0};
    auto body = [&]() {
        for (int i; (i = next.fetch_add(1)) < n;) fn(i);
    };
    std::vector<std::thread> th;
    for (int t = 1; t < std::min(n, nthreads); ++t)
        th.emplace_back([&]() {
            helper_priority();
            body();
        });
    body();
    for (auto& t : th) t.join();
}

// prediction._read_tree (prediction.py:149-159): returns the end of the tree payload
static size_t intra_tree_span(const uint8_t* d, size_t len, size_t pos, uint32_t& nbits) {
    if (pos + 4 > len) fail(HIVC_E_TRUNCATED_STREAM, "intra payload truncated");
    nbits = rd_u32(d + pos);
    const size_t nbytes = ((size_t)nbits + 7) / 8;
    if (pos + 4 + nbytes > len) fail(HIVC_E_TRUNCATED_STREAM, "intra payload truncated");
    return pos + 4 + nbytes;
}

// Sequential: mask bitmap of one tree (the exact reference error on a bad stream).
static size_t intra_tree_seq(const uint8_t* d, size_t pos, uint32_t nbits, int32_t h, int32_t w,
                             std::vector<uint64_t>& bits) {
    bits.assign(((size_t)h * w + 63) / 64, 0);
    size_t nleaves = 0;
    intra_tree_walk(d + pos + 4, ((size_t)nbits + 7) / 8, nbits, 0, 0, 0, w, h, 0, 0, (size_t)w, bits.data(), nleaves);
    return nleaves;
}

// Parallel: cut at depth 5 (32 subtrees), walk them into local bitmaps on
// `threads` threads, merge; any failure reruns the sequential walk so the
// error is the one a preorder walk meets first.
static size_t intra_tree_par(const uint8_t* d, size_t pos, uint32_t nbits, int32_t h, int32_t w, int threads,
                             std::vector<uint64_t>& bits, std::vector<uint64_t>& local) {
    const uint8_t* tb = d + pos + 4;
    const size_t nbytes = ((size_t)nbits + 7) / 8;
    std::vector<TreeTask> tasks;
    try {
        tree_tasks(tb, nbits, 0, 0, 0, w, h, 5, tasks);
    } catch (const Error&) {
        return intra_tree_seq(d, pos, nbits, h, w, bits);
    }
    size_t words = 0;
    for (TreeTask& t : tasks) {
        t.stride = ((size_t)t.w + 63) / 64 * 64;
        t.off = words;
        words += (size_t)t.h * (t.stride / 64);
    }
    local.assign(words, 0);
    std::atomic<bool> bad{false};
    parallel_for((int)tasks.size(), threads, [&](int i) {
        TreeTask& t = tasks[i];
        try {
            t.end = intra_tree_walk(tb, nbytes, nbits, t.start, t.x, t.y, t.w, t.h, t.x, t.y, t.stride,
                                    local.data() + t.off, t.nleaves);
        } catch (const Error&) {
            bad = true;
        }
    });
    if (bad) return intra_tree_seq(d, pos, nbits, h, w, bits);
    bits.assign(((size_t)h * w + 63) / 64, 0);
    size_t nleaves = 0;
    for (const TreeTask& t : tasks) {
        merge_rect_bits(local.data() + t.off, t.stride, t.x, t.y, t.w, t.h, w, bits.data(), bits.size());
        nleaves += t.nleaves;
    }
    return nleaves;
}

// A gray plane's tree walked by the parse thread (+ `extra` tree threads for
// large planes) and the value-decode helper together: the parse thread cuts
// the tree into subtrees and starts walking them while the helper decodes the
// entropy-coded values (decode_vals), after which the helper takes the
// remaining subtrees.  The two sections of a 540p I-frame (~0.2 ms of values,
// ~0.5 ms of tree) then end together instead of the tree alone gating the
// solve.  Any failure reruns the sequential walk (the reference's error, in
// stream order).
template <class V>
static size_t intra_tree_coop(const uint8_t* d, size_t pos, uint32_t nbits, int32_t h, int32_t w,
                              std::vector<uint64_t>& bits, std::vector<uint64_t>& local, int depth, int extra,
                              bool renice, V&& decode_vals) {
    const uint8_t* tb = d + pos + 4;
    const size_t nbytes = ((size_t)nbits + 7) / 8;
    std::vector<TreeTask> tasks;
    std::atomic<int> state{0};  // 0: cutting, 1: tasks ready, 2: cut failed
    std::atomic<int> next{0};
    std::atomic<bool> bad{false};
    auto run = [&]() {
        for (int i; (i = next.fetch_add(1)) < (int)tasks.size();) {
            TreeTask& t = tasks[i];
            try {
                t.end = intra_tree_walk(tb, nbytes, nbits, t.start, t.x, t.y, t.w, t.h, t.x, t.y, t.stride,
                                        local.data() + t.off, t.nleaves);
            } catch (const Error&) {
                bad = true;
            }
        }
    };
    auto wait_run = [&]() {
        int st;
        while ((st = state.load(std::memory_order_acquire)) == 0) std::this_thread::yield();
        if (st == 1) run();
    };
    std::thread helper([&]() {
        if (renice) helper_priority();
        decode_vals();
        wait_run();
    });
    std::vector<std::thread> more;  // tree threads from the start (large planes)
    for (int e = 0; e < extra; ++e)
        more.emplace_back([&]() {
            helper_priority();
            wait_run();
        });
    bool cut = true;
    try {
        tree_tasks(tb, nbits, 0, 0, 0, w, h, depth, tasks);
    } catch (const Error&) {
        cut = false;
    }
    if (cut) {
        size_t words = 0;
        for (TreeTask& t : tasks) {
            t.stride = ((size_t)t.w + 63) / 64 * 64;
            t.off = words;
            words += (size_t)t.h * (t.stride / 64);
        }
        local.assign(words, 0);
        state.store(1, std::memory_order_release);
        run();
    } else {
        state.store(2, std::memory_order_release);
    }
    helper.join();
    for (auto& t : more) t.join();
    if (!cut || bad) return intra_tree_seq(d, pos, nbits, h, w, bits);
    bits.assign(((size_t)h * w + 63) / 64, 0);
    size_t nleaves = 0;
    for (const TreeTask& t : tasks) {
        merge_rect_bits(local.data() + t.off, t.stride, t.x, t.y, t.w, t.h, w, bits.data(), bits.size());
        nleaves += t.nleaves;
    }
    return nleaves;
}

// Raster-ordered mask points (flat indices) of a bitmap; `threads` ranges in parallel.
static void intra_points(const std::vector<uint64_t>& bits, size_t nleaves, std::vector<int32_t>& pts, int threads) {
    const size_t nw = bits.size();
    const int nr = threads > 1 ? threads * 4 : 1;
    std::vector<size_t> base(nr + 1, 0);
    auto range = [&](int r, size_t& a, size_t& b) {
        a = nw * r / nr;
        b = nw * (r + 1) / nr;
    };
    parallel_for(nr, threads, [&](int r) {
        size_t a, b, c = 0;
        range(r, a, b);
        for (size_t i = a; i < b; ++i) c += (size_t)__builtin_popcountll(bits[i]);
        base[r + 1] = c;
    });
    for (int r = 0; r < nr; ++r) base[r + 1] += base[r];
    if (base[nr] != nleaves) fail(HIVC_E_SUBDIVISION, "mask leaf count mismatch");
    pts.resize(nleaves);
    parallel_for(nr, threads, [&](int r) {
        size_t a, b;
        range(r, a, b);
        int32_t* o = pts.data() + base[r];
        for (size_t wi = a; wi < b; ++wi) {
            uint64_t v = bits[wi];
            while (v) {
                *o++ = (int32_t)(wi * 64 + __builtin_ctzll(v));
                v &= v - 1;
            }
        }
    });
}

// End of an entropy.decode_symbols payload without decoding it (entropy.py:227-240, 276-291).
static size_t symbols_span(const uint8_t* d, size_t len, size_t pos) {
    if (pos >= len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    const int tl = d[pos++];
    if (tl < 5 || tl > 12) fail(HIVC_E_ENTROPY, "bad table_log " + std::to_string(tl));
    const uint64_t nsym = read_uvarint(d, len, pos);
    if (nsym == 0 || nsym > (1ull << tl)) fail(HIVC_E_ENTROPY, "bad alphabet size");
    for (uint64_t i = 0; i < nsym; ++i) read_uvarint(d, len, pos);
    if (pos + 10 > len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    const uint32_t bit_len = rd_u32(d + pos + 6);
    pos += 10;
    const size_t nbytes = ((size_t)bit_len + 7) / 8;
    if (pos + nbytes > len) fail(HIVC_E_TRUNCATED_STREAM, "entropy payload truncated");
    return pos + nbytes;
}

// prediction._decode_plane_values (prediction.py:133-139): lo/hi, then the symbols.
static size_t intra_values_span(const uint8_t* d, size_t len, size_t pos) {
    if (pos + 4 > len) fail(HIVC_E_TRUNCATED_STREAM, "intra payload truncated");
    return symbols_span(d, len, pos + 4);
}

static void intra_symbols(const uint8_t* d, size_t len, size_t pos, std::vector<int32_t>& idx) {
    decode_symbols(d, len, pos + 4, idx);
}

static void intra_dequantize(const uint8_t* d, size_t pos, int levels, const std::vector<int32_t>& idx, size_t npts,
                             std::vector<double>& out) {
    // uniform_dequantize (quantize.py:78-82)
    int16_t lo, hi;
    std::memcpy(&lo, d + pos, 2);
    std::memcpy(&hi, d + pos + 2, 2);
    const double flo = lo, fhi = hi;
    if (!(flo < fhi)) fail(HIVC_E_QUANTIZE, "need lo < hi");
    const double step = (fhi - flo) / (double)(levels - 1);
    // f.ravel()[points] = values (prediction.py:205): numpy broadcasts a
    // single value, any other length mismatch is a ValueError.
    if (idx.size() != npts && idx.size() != 1)
        fail(HIVC_E_ARGUMENT, "shape mismatch: " + std::to_string(idx.size()) + " values for " +
                                  std::to_string(npts) + " mask points");
    out.resize(npts);
    for (size_t i = 0; i < npts; ++i) out[i] = flo + (double)idx[idx.size() == 1 ? 0 : i] * step;
}

size_t parse_intra(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int channels, int levels,
                   IntraJob& job, std::vector<uint64_t>& bits) {
    // prediction.decode_intra (prediction.py:185-200).  The payload is
    // [tree Y][values Y] (+ [tree chroma][values Cb][values Cr]); the section
    // bounds come from the length fields, so the entropy-coded value planes
    // decode on a helper thread while the trees are walked (large planes:
    // each tree cut into 16 subtrees walked on several threads).
    const int ntrees = channels == 3 ? 2 : 1;
    uint32_t tbits[2] = {0, 0};
    size_t tpos[2] = {0, 0}, vpos[3] = {0, 0, 0};
    size_t p = pos;
    tpos[0] = p;
    p = intra_tree_span(d, len, p, tbits[0]);
    vpos[0] = p;
    p = intra_values_span(d, len, p);
    if (ntrees == 2) {
        tpos[1] = p;
        p = intra_tree_span(d, len, p, tbits[1]);
        for (int c = 1; c < 3; ++c) {
            vpos[c] = p;
            p = intra_values_span(d, len, p);
        }
    }
    const size_t end = p;
    const size_t npx = (size_t)h * w;
    static const int kHw = (int)std::max(1u, std::thread::hardware_concurrency());
    // (the decoder already runs one parse per GOP on its own thread: only the
    // largest planes, whose I-frame parse is on the critical path, fan out)
    static const int kTreeThreads = [] {
        const char* e = debug_opt("tree_threads");
        return e ? std::max(1, atoi(e)) : 3;
    }();
    static const int kTreeThreadsSmall = [] {
        const char* e = debug_opt("tree_threads_small");
        return e ? std::max(1, atoi(e)) : 1;
    }();
    const int tree_threads = npx >= (1u << 20) ? std::min(kTreeThreads, kHw)
                             : npx >= (1u << 18) ? std::min(kTreeThreadsSmall, kHw)
                                                 : 1;
    std::vector<int32_t>* idx = job.idx;
    std::exception_ptr verr[3], terr[2];
    auto decode_vals = [&]() {
        for (int c = 0; c < channels; ++c) {
            try {
                intra_symbols(d, len, vpos[c], idx[c]);
            } catch (...) {
                verr[c] = std::current_exception();
            }
        }
    };
    std::thread helper;
    const bool par = npx >= (1u << 18) && kHw > 1;
    if (par && ntrees == 1) {
        // gray: the value-decode helper joins the tree walk once the values are done
        // (540p: the parse thread + the helper; >= 1 Mpx: tree_threads from the start)
        try {
            const size_t nl = intra_tree_coop(d, tpos[0], tbits[0], h, w, bits, job.local, tree_threads > 1 ? 5 : 3,
                                              tree_threads - 1, tree_threads > 1, decode_vals);
            intra_points(bits, nl, job.pts[0], tree_threads);
        } catch (...) {
            terr[0] = std::current_exception();
        }
        if (terr[0]) std::rethrow_exception(terr[0]);
        if (verr[0]) std::rethrow_exception(verr[0]);
        intra_dequantize(d, vpos[0], levels, idx[0], job.pts[0].size(), job.vals[0]);
        job.nchan = 1;
        return end;
    }
    if (par)
        helper = std::thread([&]() {
            helper_priority();
            decode_vals();
        });
    for (int t = 0; t < ntrees; ++t) {
        try {
            const size_t nl = tree_threads > 1 ? intra_tree_par(d, tpos[t], tbits[t], h, w, tree_threads, bits, job.local)
                                               : intra_tree_seq(d, tpos[t], tbits[t], h, w, bits);
            intra_points(bits, nl, job.pts[t], tree_threads);
        } catch (...) {
            terr[t] = std::current_exception();
        }
    }
    if (par)
        helper.join();
    else
        decode_vals();
    // errors in stream order: tree Y, values Y, tree chroma, values Cb, values Cr
    if (terr[0]) std::rethrow_exception(terr[0]);
    if (verr[0]) std::rethrow_exception(verr[0]);
    intra_dequantize(d, vpos[0], levels, idx[0], job.pts[0].size(), job.vals[0]);
    job.nchan = 1;
    if (ntrees == 2) {
        if (terr[1]) std::rethrow_exception(terr[1]);
        for (int c = 1; c < 3; ++c) {
            if (verr[c]) std::rethrow_exception(verr[c]);
            intra_dequantize(d, vpos[c], 2 * levels - 1, idx[c], job.pts[1].size(), job.vals[c]);
        }
        job.nchan = 3;
    }
    return end;
}

// ---------------------------------------------------------------- flow payload

size_t parse_flow(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int levels, FlowJob& job) {
    for (int c = 0; c < 2; ++c) {  // flow._decompress_plane (flow.py:343-356)
        if (pos + 12 > len) fail(HIVC_E_TRUNCATED_STREAM, "flow payload truncated");
        float lo, hi;
        std::memcpy(&lo, d + pos, 4);
        std::memcpy(&hi, d + pos + 4, 4);
        uint32_t nbits = rd_u32(d + pos + 8);
        pos += 12;
        size_t nbytes = ((size_t)nbits + 7) / 8;
        if (pos + nbytes > len) fail(HIVC_E_TRUNCATED_STREAM, "flow payload truncated");
        BitReader rd(d + pos, nbytes, nbits);
        int32_t nleaves = 0;
        parse_flow_tree(rd, w, h, job.nodes[c], nleaves, nullptr);
        flow_tile_map(job.nodes[c], nleaves, w, h, job.tiles[c]);
        pos += nbytes;
        std::vector<int32_t> idx;
        pos = decode_symbols(d, len, pos, idx);
        double flo = lo, fhi = hi;
        if (!(flo < fhi)) fail(HIVC_E_QUANTIZE, "need lo < hi");
        double step = (fhi - flo) / (double)(levels - 1);
        if ((int64_t)idx.size() != nleaves) fail(HIVC_E_SUBDIVISION, "leaf value count mismatch");
        job.vals[c].resize(idx.size());
        for (size_t i = 0; i < idx.size(); ++i) job.vals[c][i] = flo + (double)idx[i] * step;
    }
    for (int c = 0; c < 2; ++c)  // FlowField.__post_init__ (flow.py:45-49)
        for (double v : job.vals[c])
            if (!std::isfinite(v)) fail(HIVC_E_FLOW, "non-finite flow values");
    return pos;
}

size_t parse_flow_component(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int levels,
                            std::vector<Rect>& leaves, std::vector<double>& vals) {
    if (pos + 12 > len) fail(HIVC_E_TRUNCATED_STREAM, "flow payload truncated");
    float lo, hi;
    std::memcpy(&lo, d + pos, 4);
    std::memcpy(&hi, d + pos + 4, 4);
    uint32_t nbits = rd_u32(d + pos + 8);
    pos += 12;
    size_t nbytes = ((size_t)nbits + 7) / 8;
    if (pos + nbytes > len) fail(HIVC_E_TRUNCATED_STREAM, "flow payload truncated");
    BitReader rd(d + pos, nbytes, nbits);
    leaves.clear();
    parse_tree_leaves(rd, w, h, leaves);  // deserialize_tree (flow.py:351-352)
    pos += nbytes;
    std::vector<int32_t> idx;
    pos = decode_symbols(d, len, pos, idx);
    double flo = lo, fhi = hi;
    if (!(flo < fhi)) fail(HIVC_E_QUANTIZE, "need lo < hi");  // uniform_dequantize (quantize.py:78-82)
    const double step = (fhi - flo) / (double)(levels - 1);
    // paint_leaf_values (subdivision.py:162-170)
    if (idx.size() != leaves.size()) fail(HIVC_E_SUBDIVISION, "leaf value count mismatch");
    vals.resize(idx.size());
    for (size_t i = 0; i < idx.size(); ++i) vals[i] = flo + (double)idx[i] * step;
    return pos;
}

// ---------------------------------------------------------------- residual payload

size_t parse_residual(const uint8_t* d, size_t len, size_t pos, int32_t h, int32_t w, int channels, ResidualJob& job) {
    // codec._decode_residual (codec.py:248-340), parse half
    const int32_t nbx = (w + 7) / 8, nby = (h + 7) / 8;
    const size_t ntiles = (size_t)nbx * nby;
    const size_t nskip = (ntiles + 7) / 8;
    if (pos + 1 > len) fail(HIVC_E_TRUNCATED, "residual payload truncated");
    uint8_t marker = d[pos++];
    job.ngroups = 0;
    if (marker == 0) {
        job.zero = true;
        return pos;
    }
    if (marker != 1) fail(HIVC_E_CODEC, "bad residual payload marker");
    job.zero = false;
    if (pos + 8 > len) fail(HIVC_E_TRUNCATED, "residual payload truncated");
    uint32_t c_fp = rd_u32(d + pos), a_fp = rd_u32(d + pos + 4);
    pos += 8;
    if (c_fp == 0 || a_fp == 0) fail(HIVC_E_CODEC, "zero coefficient scale");
    job.c_scale = c_fp / 65536.0;
    job.a_scale = a_fp / 65536.0;
    const int groups[2] = {1, 2};
    const int ng = channels == 3 ? 2 : 1;
    std::vector<Rect> leaves;
    for (int gi = 0; gi < ng; ++gi) {
        ResidualGroup& g = job.g[gi];
        g.nplanes = groups[gi];
        if (pos + nskip > len) fail(HIVC_E_TRUNCATED, "residual payload truncated");
        // skip bitmap, MSB-first (np.unpackbits, codec.py:285-289)
        const size_t nwords = (ntiles + 63) / 64;
        g.tile_words.assign(nwords, 0);
        g.word_prefix.assign(nwords, 0);
        for (size_t byte = 0; byte < nskip; ++byte) {  // tile 8j+i = bit 7-i of byte j
            uint64_t v = kBitReverse[d[pos + byte]];
            if (!v) continue;
            if (byte == nskip - 1 && (ntiles & 7)) v &= (1u << (ntiles & 7)) - 1u;  // np.unpackbits(...)[:ntiles]
            g.tile_words[byte >> 3] |= v << ((byte & 7) * 8);
        }
        pos += nskip;
        int32_t acc = 0;
        for (size_t i = 0; i < nwords; ++i) {
            g.word_prefix[i] = acc;
            acc += __builtin_popcountll(g.tile_words[i]);
        }
        g.nblocks = acc;
        if (pos + 4 > len) fail(HIVC_E_TRUNCATED, "residual payload truncated");
        uint32_t tree_bits = rd_u32(d + pos);
        pos += 4;
        size_t tnb = ((size_t)tree_bits + 7) / 8;
        if (pos + tnb > len) fail(HIVC_E_TRUNCATED, "residual payload truncated");
        BitReader rd(d + pos, tnb, tree_bits);
        pos += tnb;
        g.block_mask.resize(g.nblocks);
        g.block_off.resize(g.nblocks);
        int32_t b = 0, npts = 0;
        for (size_t wi = 0; wi < nwords; ++wi) {
            uint64_t bits = g.tile_words[wi];
            while (bits) {
                size_t t = wi * 64 + __builtin_ctzll(bits);
                bits &= bits - 1;
                int32_t ty = (int32_t)(t / nbx), tx = (int32_t)(t % nbx);
                int32_t bh = std::min(8, h - ty * 8), bw = std::min(8, w - tx * 8);
                uint64_t m = 0;  // parse_mask per coded tile (codec.py:300-303)
                bool done = false;
                if (bw == 8 && bh == 8) {
                    const uint32_t v = rd.peek12();
                    const int nb = kBlockTree.nbits[v];
                    if (nb && rd.pos + (uint64_t)nb <= rd.limit) {
                        m = kBlockTree.mask[v];
                        rd.skip(nb);
                        done = true;
                    }
                }
                if (!done)
                    walk_tree(rd, bw, bh, [&](int32_t x, int32_t y, int32_t rw, int32_t rh) {
                        m |= 1ull << ((y + rh / 2) * 8 + (x + rw / 2));
                    });
                g.block_mask[b] = m;
                g.block_off[b] = npts;
                npts += __builtin_popcountll(m);
                ++b;
            }
        }
        g.npoints = npts;
        pos = decode_signed_values(d, len, pos, g.c_sym);
        pos = decode_signed_values(d, len, pos, g.a_sym);
        if (g.c_sym.size() != (size_t)npts * g.nplanes || g.a_sym.size() != (size_t)g.nblocks * g.nplanes)
            fail(HIVC_E_CODEC, "residual payload inconsistent with block masks");
    }
    job.ngroups = ng;
    return pos;
}

}  // namespace hivc
