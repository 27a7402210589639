// Encoder primitives, bit-exact with the reference (see encode.h).
#include "encode.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <cstdlib>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>

namespace hivc {

void BitWriter::write(uint64_t value, int count) {
    if (count <= 0) return;
    acc = (acc << count) | (value & ((1ull << count) - 1ull));
    nbits += count;
    while (nbits >= 8) {
        nbits -= 8;
        bytes.push_back((uint8_t)((acc >> nbits) & 0xFF));
    }
    acc &= (nbits ? ((1ull << nbits) - 1ull) : 0ull);
}

void BitWriter::append_to(std::vector<uint8_t>& out) const {
    out.insert(out.end(), bytes.begin(), bytes.end());
    if (nbits) out.push_back((uint8_t)(acc << (8 - nbits)));
}

void write_uvarint(std::vector<uint8_t>& out, uint64_t v) {
    for (;;) {
        const uint8_t byte = v & 0x7F;
        v >>= 7;
        if (v) {
            out.push_back(byte | 0x80);
        } else {
            out.push_back(byte);
            return;
        }
    }
}

std::vector<int64_t> normalize_counts(const std::vector<int64_t>& hist, int table_log) {
    if (table_log < 5 || table_log > 12) fail(HIVC_E_ENTROPY, "table_log out of range [5, 12]");
    const size_t n = hist.size();
    if (n == 0) fail(HIVC_E_ENTROPY, "bad histogram");
    double total = 0.0;  // np.sum of a float64 copy (exact: integer counts << 2^53)
    int64_t present = 0;
    for (int64_t c : hist) {
        if (c < 0) fail(HIVC_E_ENTROPY, "bad histogram");
        total += (double)c;
        present += c > 0;
    }
    if (total <= 0) fail(HIVC_E_ENTROPY, "histogram has no counts");
    const int64_t size = 1ll << table_log;
    if (present > size) fail(HIVC_E_ENTROPY, "alphabet larger than table");
    std::vector<double> ideal(n);
    std::vector<int64_t> norm(n);
    int64_t sum = 0;
    for (size_t i = 0; i < n; ++i) {
        ideal[i] = (double)hist[i] / total * (double)size;  // hist / total * size
        norm[i] = (int64_t)std::floor(ideal[i]);
        if (hist[i] > 0 && norm[i] == 0) norm[i] = 1;
        sum += norm[i];
    }
    int64_t diff = size - sum;
    if (diff > 0) {
        // np.lexsort((arange, -remainder)): remainder descending, index ascending
        std::vector<double> rem(n);
        for (size_t i = 0; i < n; ++i) rem[i] = ideal[i] - std::floor(ideal[i]);
        std::vector<size_t> order(n);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return -rem[a] < -rem[b]; });
        size_t i = 0;
        while (diff > 0) {
            const size_t s = order[i % n];
            if (hist[s] > 0) {
                ++norm[s];
                --diff;
            }
            ++i;
        }
    }
    while (diff < 0) {  // decrement the largest count (smallest index on ties) among those > 1
        size_t best = n;
        for (size_t s = 0; s < n; ++s)
            if (norm[s] > 1 && (best == n || norm[s] > norm[best])) best = s;
        --norm[best];
        ++diff;
    }
    return norm;
}

namespace {

int bit_length(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

int auto_table_log(size_t alphabet, size_t n) {  // entropy.py:243-252
    const int need = alphabet > 1 ? std::max(1, bit_length(alphabet - 1)) : 1;
    int tl = std::max(5, need + 1);
    if (n >= 4096) tl = std::max(tl, 10);
    if (n >= 65536) tl = std::max(tl, 11);
    return std::min(tl, 12);
}

}  // namespace

void encode_symbols(const int64_t* symbols, size_t n, int table_log, std::vector<uint8_t>& out) {
    std::vector<int64_t> hist;
    if (n) {
        int64_t mx = 0;
        for (size_t i = 0; i < n; ++i) {
            if (symbols[i] < 0) fail(HIVC_E_ENTROPY, "symbols must be nonnegative");
            mx = std::max(mx, symbols[i]);
        }
        hist.assign((size_t)mx + 1, 0);
        for (size_t i = 0; i < n; ++i) ++hist[(size_t)symbols[i]];
    } else {
        hist.assign(1, 1);
    }
    if (table_log < 0) table_log = auto_table_log(hist.size(), n);
    const std::vector<int64_t> counts = normalize_counts(hist, table_log);
    const uint32_t size = 1u << table_log;
    BitWriter w;
    uint32_t state = size;
    if (n) {
        // FseTable (entropy.py:108-141): spread the symbols; for symbol s the
        // x values counts[s] .. 2 counts[s] - 1 go to its slots in slot order
        const uint32_t step = (size >> 1) + (size >> 3) + 3;
        std::vector<uint32_t> spread(size);
        uint32_t k = 0;
        for (size_t s = 0; s < counts.size(); ++s)
            for (int64_t j = 0; j < counts[s]; ++j) spread[(k++ * step) & (size - 1)] = (uint32_t)s;
        std::vector<uint32_t> base(counts.size() + 1, 0);
        for (size_t s = 0; s < counts.size(); ++s) base[s + 1] = base[s] + (uint32_t)counts[s];
        std::vector<uint32_t> slot_of(size), next(counts.size(), 0);  // slot_of[base[s] + (x - counts[s])]
        for (uint32_t slot = 0; slot < size; ++slot) {
            const uint32_t s = spread[slot];
            slot_of[base[s] + next[s]++] = slot;
        }
        // fse_encode (entropy.py:148-172): symbols in reverse, chunks written in reverse
        std::vector<std::pair<uint32_t, int>> chunks(n);
        for (size_t i = n; i-- > 0;) {
            const uint32_t s = (uint32_t)symbols[i];
            const uint32_t c = (uint32_t)counts[s];
            if (c == 0) fail(HIVC_E_ENTROPY, "symbol " + std::to_string(s) + " absent from table");
            int nb = bit_length(state) - bit_length(c);
            if ((state >> nb) >= 2 * c)
                ++nb;
            else if (nb > 0 && (state >> nb) < c)
                --nb;
            chunks[n - 1 - i] = {state & ((1u << nb) - 1u), nb};
            state = size + slot_of[base[s] + ((state >> nb) - c)];
        }
        for (size_t i = n; i-- > 0;) w.write(chunks[i].first, chunks[i].second);
    }
    out.push_back((uint8_t)table_log);  // _encode_header (entropy.py:219-224)
    write_uvarint(out, counts.size());
    for (int64_t c : counts) write_uvarint(out, (uint64_t)c);
    const uint32_t cnt = (uint32_t)n;
    const uint16_t st = (uint16_t)state;
    const uint32_t bl = (uint32_t)w.size_bits();
    uint8_t hdr[10];
    std::memcpy(hdr, &cnt, 4);
    std::memcpy(hdr + 4, &st, 2);
    std::memcpy(hdr + 6, &bl, 4);
    out.insert(out.end(), hdr, hdr + 10);
    w.append_to(out);
}

void encode_signed_values(const int64_t* values, size_t n, int table_log, std::vector<uint8_t>& out) {
    std::vector<int64_t> cats(n);
    BitWriter extra;
    for (size_t i = 0; i < n; ++i) {  // to_category (entropy.py:40-49)
        const int64_t v = values[i];
        const int64_t a = v < 0 ? -v : v;
        if (a > (1 << 15) - 1) fail(HIVC_E_ENTROPY, "magnitude overflow: " + std::to_string(v));
        if (v == 0) {
            cats[i] = 0;
            continue;
        }
        const int k = bit_length((uint64_t)a);
        cats[i] = k;
        extra.write((uint64_t)(v > 0 ? v : v + (1ll << k) - 1), k);
    }
    encode_symbols(cats.data(), n, table_log, out);
    const uint32_t bl = (uint32_t)extra.size_bits();
    uint8_t b4[4];
    std::memcpy(b4, &bl, 4);
    out.insert(out.end(), b4, b4 + 4);
    extra.append_to(out);
}

}  // namespace hivc

// ---------------------------------------------------------------- subdivision

#include <queue>

namespace hivc {

double np_pairwise(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

namespace {

thread_local std::vector<double> t_buf;

// Large regions are summed on several threads.  Both of numpy's orders split
// into independent pieces combined in a fixed order (the two halves of a
// pairwise recursion; the per-chunk sums of a buffered reduction, accumulated
// in sequence), so the parallel sums are bit-identical to the serial ones.
constexpr int64_t kParMin = 1 << 16;
int enc_threads() {
    static const int n = [] {
        const char* e = debug_opt("enc_threads");
        int v = e ? std::atoi(e) : 8;
        return std::max(1, std::min(v, (int)std::max(1u, std::thread::hardware_concurrency())));
    }();
    return n;
}

// Persistent helpers: fork_join(nt, fn) runs fn(0) here and fn(1..nt-1) on the
// pool.  Pool threads never wait on other tasks (no nested fork_join), so
// concurrent callers (several GOPs encoding at once) cannot deadlock.
class EncPool {
  public:
    explicit EncPool(int n) {
        for (int i = 0; i < n; ++i)
            th_.emplace_back([this] {
                for (;;) {
                    std::function<void()> f;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                        if (stop_ && q_.empty()) return;
                        f = std::move(q_.front());
                        q_.pop_front();
                    }
                    f();
                }
            });
    }
    ~EncPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(f));
        }
        cv_.notify_one();
    }

  private:
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    bool stop_ = false;
};

EncPool& enc_pool() {
    static EncPool* pool = new EncPool(enc_threads() - 1);  // leaked on purpose: no join at exit
    return *pool;
}

template <class F>
void fork_join(int nt, F&& fn) {
    if (nt <= 1) {
        fn(0);
        return;
    }
    std::atomic<int> left{nt - 1};
    std::mutex m;
    std::condition_variable cv;
    for (int t = 1; t < nt; ++t)
        enc_pool().submit([&, t] {
            fn(t);
            if (left.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> lk(m);
                cv.notify_all();
            }
        });
    fn(0);
    std::unique_lock<std::mutex> lk(m);
    cv.wait(lk, [&] { return left.load() == 0; });
}

// the top `depth` levels of numpy's pairwise recursion as independent segments
void pw_segments(int64_t off, int64_t n, int depth, std::vector<std::pair<int64_t, int64_t>>& segs) {
    if (depth == 0 || n < kParMin) {
        segs.push_back({off, n});
        return;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    pw_segments(off, n2, depth - 1, segs);
    pw_segments(off + n2, n - n2, depth - 1, segs);
}

double pw_combine(int64_t n, int depth, const double*& vals) {
    if (depth == 0 || n < kParMin) return *vals++;
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const double l = pw_combine(n2, depth - 1, vals);
    const double r = pw_combine(n - n2, depth - 1, vals);
    return l + r;
}

double np_pairwise_par(const double* a, int64_t n, int par) {
    if (par <= 1 || n < kParMin) return np_pairwise(a, n);
    int depth = 0;
    while ((1 << (depth + 1)) <= par) ++depth;
    std::vector<std::pair<int64_t, int64_t>> segs;
    pw_segments(0, n, depth, segs);
    std::vector<double> part(segs.size());
    const int nt = std::min<int>(par, (int)segs.size());
    fork_join(nt, [&](int t) {
        for (size_t k = (size_t)t; k < segs.size(); k += (size_t)nt) part[k] = np_pairwise(a + segs[k].first, segs[k].second);
    });
    const double* v = part.data();
    return pw_combine(n, depth, v);
}

double sum_region_par(const double* plane, int32_t W, int32_t x, int32_t y, int32_t w, int32_t h, int par) {
    const int64_t n = (int64_t)w * h;
    if (w == W || h == 1) return np_pairwise_par(plane + (int64_t)y * W + x, n, par);  // contiguous view
    if (par <= 1 || n < kParMin || w > 8192) return sum_region(plane, W, x, y, w, h);
    const int32_t rpc = std::max<int32_t>(1, 8192 / w);
    const int32_t nchunks = (h + rpc - 1) / rpc;
    std::vector<double> part((size_t)nchunks);
    const int nt = std::min<int>(par, nchunks);
    fork_join(nt, [&](int t) {
        std::vector<double>& buf = t_buf;
        buf.resize((size_t)rpc * w);
        for (int32_t k = t; k < nchunks; k += nt) {
            const int32_t r0 = k * rpc, rr = std::min(rpc, h - r0);
            for (int32_t r = 0; r < rr; ++r)
                std::memcpy(buf.data() + (size_t)r * w, plane + (int64_t)(y + r0 + r) * W + x, (size_t)w * sizeof(double));
            part[(size_t)k] = np_pairwise(buf.data(), (int64_t)rr * w);
        }
    });
    double acc = 0.0;
    for (double v : part) acc += v;
    return acc;
}

}  // namespace

double sum_region(const double* plane, int32_t W, int32_t x, int32_t y, int32_t w, int32_t h) {
    const int64_t n = (int64_t)w * h;
    if (w == W || h == 1) return np_pairwise(plane + (int64_t)y * W + x, n);  // contiguous view
    const int32_t rows_per_chunk = std::max<int32_t>(1, 8192 / w);
    double acc = 0.0;
    if (w > 8192) {  // (not reached for planes <= 8192 wide)
        for (int32_t r = 0; r < h; ++r) acc += np_pairwise(plane + (int64_t)(y + r) * W + x, w);
        return acc;
    }
    t_buf.resize((size_t)rows_per_chunk * w);
    for (int32_t r0 = 0; r0 < h; r0 += rows_per_chunk) {
        const int32_t rr = std::min(rows_per_chunk, h - r0);
        for (int32_t r = 0; r < rr; ++r)
            std::memcpy(t_buf.data() + (size_t)r * w, plane + (int64_t)(y + r0 + r) * W + x, (size_t)w * sizeof(double));
        acc += np_pairwise(t_buf.data(), (int64_t)rr * w);
    }
    return acc;
}

namespace {

// float(np.sum((region - region.mean()) ** 2)) (subdivision.py:133-135)
thread_local std::vector<double> t_dev;
double region_ssd(const double* plane, int32_t W, int32_t x, int32_t y, int32_t w, int32_t h) {
    const int64_t n = (int64_t)w * h;
    const int par = n >= kParMin ? enc_threads() : 1;
    const double mean = sum_region_par(plane, W, x, y, w, h, par) / (double)n;
    t_dev.resize((size_t)n);
    double* d = t_dev.data();
    auto rows = [&](int32_t r0, int32_t r1) {
        for (int32_t r = r0; r < r1; ++r) {
            const double* row = plane + (int64_t)(y + r) * W + x;
            for (int32_t c = 0; c < w; ++c) {
                const double v = row[c] - mean;
                d[(int64_t)r * w + c] = v * v;
            }
        }
    };
    if (par > 1) {
        const int nt = std::min<int>(par, h);
        fork_join(nt, [&](int t) { rows((int32_t)((int64_t)h * t / nt), (int32_t)((int64_t)h * (t + 1) / nt)); });
    } else {
        rows(0, h);
    }
    return np_pairwise_par(d, n, par);
}

struct Node {
    Rect4 r;
    int32_t first = -1, second = -1;  // children (node indices) once split
};

struct Entry {
    double neg_err;
    int32_t y, x;
    int64_t seq;
    int32_t node;
    bool operator>(const Entry& o) const {  // heapq order on (-err, y, x, seq)
        if (neg_err != o.neg_err) return neg_err > o.neg_err;
        if (y != o.y) return y > o.y;
        if (x != o.x) return x > o.x;
        return seq > o.seq;
    }
};

}  // namespace

void subdivide_by_error(const double* const* planes, int nplanes, int32_t W, int32_t H, int64_t target,
                        bool use_min_error, double min_error, BitWriter& bits, std::vector<Rect4>& leaves) {
    if (target < 1) fail(HIVC_E_SUBDIVISION, "target_points must be >= 1");
    if (target > (int64_t)W * H) fail(HIVC_E_SUBDIVISION, "target_points exceeds pixel count");
    auto error = [&](const Rect4& r) -> double {
        if (r.w == 1 && r.h == 1) return -1.0;
        if (nplanes == 1) return region_ssd(planes[0], W, r.x, r.y, r.w, r.h);
        double s = 0.0;  // sum(region_ssd(p) for p in planes)
        for (int i = 0; i < nplanes; ++i) s += region_ssd(planes[i], W, r.x, r.y, r.w, r.h);
        return s;
    };
    std::vector<Node> nodes;
    nodes.reserve((size_t)std::min<int64_t>(2 * target, 1 << 26));
    nodes.push_back({{0, 0, W, H}});
    std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
    int64_t seq = 0;
    heap.push({-error(nodes[0].r), 0, 0, seq, 0});
    int64_t n_leaves = 1;
    while (n_leaves < target) {
        const Entry e = heap.top();
        heap.pop();
        if (use_min_error && -e.neg_err <= min_error) break;
        const Rect4 r = nodes[e.node].r;
        Rect4 a, b;  // split_children (subdivision.py:25-35)
        if (r.h > r.w) {
            const int32_t t = (r.h + 1) / 2;
            a = {r.x, r.y, r.w, t};
            b = {r.x, r.y + t, r.w, r.h - t};
        } else {
            const int32_t t = (r.w + 1) / 2;
            a = {r.x, r.y, t, r.h};
            b = {r.x + t, r.y, r.w - t, r.h};
        }
        if (r.w == 1 && r.h == 1) fail(HIVC_E_SUBDIVISION, "cannot split a single pixel");
        const int32_t ia = (int32_t)nodes.size();
        nodes.push_back({a});
        nodes.push_back({b});
        nodes[e.node].first = ia;
        nodes[e.node].second = ia + 1;
        ++seq;
        heap.push({-error(a), a.y, a.x, seq, ia});
        ++seq;
        heap.push({-error(b), b.y, b.x, seq, ia + 1});
        ++n_leaves;
    }
    // preorder serialisation (subdivision.py:115-129) + leaves
    std::vector<int32_t> stack{0};
    leaves.clear();
    while (!stack.empty()) {
        const int32_t i = stack.back();
        stack.pop_back();
        if (nodes[i].first < 0) {
            bits.write(0, 1);
            leaves.push_back(nodes[i].r);
        } else {
            bits.write(1, 1);
            stack.push_back(nodes[i].second);
            stack.push_back(nodes[i].first);
        }
    }
}

}  // namespace hivc

// ---------------------------------------------------------------- residual tile plans

#include <atomic>
#include <mutex>
#include <thread>

namespace hivc {

void plan_residual_tiles(const int64_t* const* planes, int nplanes, int32_t h, int32_t w, int32_t points,
                         int threads, uint8_t* coded, uint64_t* masks, uint8_t* tree_bits, uint8_t* tree_nbits) {
    if (nplanes < 1 || nplanes > 2) fail(HIVC_E_ARGUMENT, "a residual channel group has 1 or 2 planes");
    if (points < 1 || points > 48) fail(HIVC_E_ARGUMENT, "residual points must lie in [1, 48]");
    const int32_t nbx = (w + 7) / 8, nby = (h + 7) / 8;
    const int64_t ntiles = (int64_t)nbx * nby;
    std::atomic<int64_t> next{0};
    std::atomic<bool> failed{false};
    std::string err;
    int err_code = 0;
    std::mutex err_mu;
    auto body = [&]() {
        double tile[2][64];
        const double* tp[2] = {tile[0], tile[1]};
        BitWriter bw;
        std::vector<Rect4> leaves;
        try {
            for (;;) {
                const int64_t base = next.fetch_add(64);
                if (base >= ntiles || failed.load(std::memory_order_relaxed)) break;
                for (int64_t t = base; t < std::min<int64_t>(base + 64, ntiles); ++t) {
                    const int32_t y0 = (int32_t)(t / nbx) * 8, x0 = (int32_t)(t % nbx) * 8;
                    const int32_t bh = std::min(8, h - y0), bwid = std::min(8, w - x0);
                    bool any = false;
                    for (int p = 0; p < nplanes; ++p)
                        for (int32_t r = 0; r < bh; ++r)
                            for (int32_t c = 0; c < bwid; ++c) {
                                const int64_t v = planes[p][(int64_t)(y0 + r) * w + x0 + c];
                                tile[p][r * bwid + c] = (double)v;
                                any |= v != 0;
                            }
                    coded[t] = any;
                    masks[t] = 0;
                    tree_nbits[t] = 0;
                    if (!any) continue;
                    bw.bytes.clear();
                    bw.acc = 0;
                    bw.nbits = 0;
                    subdivide_by_error(tp, nplanes, bwid, bh, std::min<int64_t>(points, (int64_t)bh * bwid), false,
                                       0.0, bw, leaves);
                    uint64_t m = 0;
                    for (const Rect4& l : leaves) m |= 1ull << ((l.y + l.h / 2) * 8 + (l.x + l.w / 2));
                    masks[t] = m;
                    tree_nbits[t] = (uint8_t)bw.size_bits();
                    std::vector<uint8_t> out;
                    bw.append_to(out);
                    std::memset(tree_bits + 16 * t, 0, 16);
                    std::memcpy(tree_bits + 16 * t, out.data(), out.size());
                }
            }
        } catch (const Error& e) {
            std::lock_guard<std::mutex> lk(err_mu);
            if (!failed.exchange(true)) {
                err = e.what();
                err_code = e.code;
            }
        }
    };
    const int nt = std::max(1, std::min<int>(threads, (int)((ntiles + 255) / 256)));
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) th.emplace_back(body);
    body();
    for (auto& t : th) t.join();
    if (failed) fail(err_code, err);
}

}  // namespace hivc

// ---------------------------------------------------------------- C ABI

#include "hivc_b200.h"

namespace {

int put_payload(const std::vector<uint8_t>& v, uint8_t* out, size_t cap, size_t* size) {
    *size = v.size();
    if (out && v.size() <= cap) std::memcpy(out, v.data(), v.size());
    return HIVC_OK;
}

}  // namespace

extern "C" {

int hivc_encode_symbols(const int64_t* symbols, size_t n, int32_t table_log, uint8_t* out, size_t cap,
                        size_t* size) {
    return hivc::guarded([&] {
        std::vector<uint8_t> v;
        hivc::encode_symbols(symbols, n, table_log, v);
        put_payload(v, out, cap, size);
    });
}

int hivc_normalize_counts(const int64_t* hist, size_t n, int32_t table_log, int64_t* out) {
    return hivc::guarded([&] {
        std::vector<int64_t> h(hist, hist + n);
        const std::vector<int64_t> c = hivc::normalize_counts(h, table_log);
        std::copy(c.begin(), c.end(), out);
    });
}

int hivc_encode_signed_values(const int64_t* values, size_t n, int32_t table_log, uint8_t* out, size_t cap,
                              size_t* size) {
    return hivc::guarded([&] {
        std::vector<uint8_t> v;
        hivc::encode_signed_values(values, n, table_log, v);
        put_payload(v, out, cap, size);
    });
}

int hivc_subdivide(const double* const* planes, int32_t nplanes, int32_t width, int32_t height, int64_t target,
                   int32_t use_min_error, double min_error, uint8_t* bits, uint64_t* nbits, int32_t* rects,
                   size_t* nleaves) {
    return hivc::guarded([&] {
        if (nplanes < 1 || width < 1 || height < 1) hivc::fail(HIVC_E_ARGUMENT, "bad subdivision arguments");
        hivc::BitWriter bw;
        std::vector<hivc::Rect4> leaves;
        hivc::subdivide_by_error(planes, nplanes, width, height, target, use_min_error != 0, min_error, bw, leaves);
        std::vector<uint8_t> b;
        bw.append_to(b);
        std::memcpy(bits, b.data(), b.size());
        *nbits = bw.size_bits();
        std::memcpy(rects, leaves.data(), leaves.size() * sizeof(hivc::Rect4));
        *nleaves = leaves.size();
    });
}

int hivc_region_means(const double* plane, int32_t width, int32_t height, const int32_t* rects, size_t n,
                      double* out) {
    return hivc::guarded([&] {
        for (size_t i = 0; i < n; ++i) {
            const int32_t* r = rects + 4 * i;
            if (r[2] < 1 || r[3] < 1 || r[0] < 0 || r[1] < 0 || r[0] + r[2] > width || r[1] + r[3] > height)
                hivc::fail(HIVC_E_ARGUMENT, "rectangle outside the plane");
            out[i] = hivc::sum_region(plane, width, r[0], r[1], r[2], r[3]) / (double)((int64_t)r[2] * r[3]);
        }
    });
}

int hivc_gather_tiles(const int64_t* const* planes, int32_t nplanes, int32_t h, int32_t w, const int64_t* tiles,
                      size_t n, double* out) {
    return hivc::guarded([&] {
        const int32_t nbx = (w + 7) / 8, nby = (h + 7) / 8;
        for (int p = 0; p < nplanes; ++p)
            for (size_t i = 0; i < n; ++i) {
                const int64_t t = tiles[i];
                if (t < 0 || t >= (int64_t)nbx * nby) hivc::fail(HIVC_E_ARGUMENT, "tile index out of range");
                const int32_t y0 = (int32_t)(t / nbx) * 8, x0 = (int32_t)(t % nbx) * 8;
                const int32_t bh = std::min(8, h - y0), bw = std::min(8, w - x0);
                double* o = out + ((size_t)p * n + i) * 64;
                for (int k = 0; k < 64; ++k) o[k] = 0.0;
                for (int32_t r = 0; r < bh; ++r)
                    for (int32_t c = 0; c < bw; ++c) o[r * 8 + c] = (double)planes[p][(int64_t)(y0 + r) * w + x0 + c];
            }
    });
}

int hivc_plan_residual_tiles(const int64_t* const* planes, int32_t nplanes, int32_t h, int32_t w, int32_t points,
                             int32_t threads, uint8_t* coded, uint64_t* masks, uint8_t* tree_bits,
                             uint8_t* tree_nbits) {
    return hivc::guarded([&] {
        const int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
        hivc::plan_residual_tiles(planes, nplanes, h, w, points, nt, coded, masks, tree_bits, tree_nbits);
    });
}

}  // extern "C"
