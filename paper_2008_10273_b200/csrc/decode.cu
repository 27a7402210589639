// codec.decode (codec.py:484-563) on the GPU.
//
// GOPs are independent (prev resets per GOP, codec.py:496), so the GOP
// range is dealt round-robin to decode lanes.  Each lane is a host thread
// with its own CUDA stream: it parses a whole GOP on the CPU (bit-exact,
// parse.cpp), packs the compact frame descriptions into pinned staging,
// ships them with ONE host->device copy, and queues the GOP's kernels —
// intra: scatter + pyramid + cascadic CG (inpaint.cu) + fused finalize;
// inter: fused warp/residual/finalize (recon.cu).  Parsing of GOP k+1
// overlaps the GPU work of GOP k (double-buffered staging).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>

#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

#include "decode.h"

namespace hivc {

namespace {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

inline uint32_t rd_u32(const uint8_t* p) {
    uint32_t v;
    std::memcpy(&v, p, 4);
    return v;
}


// Host parse time per stage: summed seconds (every occurrence, all threads)
// and the occurrences' intervals (absolute now_s() times) for the stage's
// wall-clock share (codec.py:509-562 stage semantics, see decode_streams).
struct HostTimes {
    double intra_parse = 0, flow_parse = 0, residual_parse = 0;
    std::vector<std::pair<double, double>> iv[3];  // intra, flow, residual
    void add(const HostTimes& o) {
        intra_parse += o.intra_parse;
        flow_parse += o.flow_parse;
        residual_parse += o.residual_parse;
        for (int k = 0; k < 3; ++k) iv[k].insert(iv[k].end(), o.iv[k].begin(), o.iv[k].end());
    }
};

// Length of the union of intervals.
double union_length(std::vector<std::pair<double, double>> v) {
    std::sort(v.begin(), v.end());
    double tot = 0, a = 0, b = -1e300;
    for (auto& x : v) {
        if (x.first > b) {
            if (b > a) tot += b - a;
            a = x.first;
            b = x.second;
        } else {
            b = std::max(b, x.second);
        }
    }
    if (b > a) tot += b - a;
    return tot;
}

// Frame records of one GOP payload, parsed one at a time (codec.decode's frame
// loop, codec.py:496-556; record layout bitstream.py:157-196).
struct GopCursor {
    const uint8_t* p;
    size_t n, pos = 2;
    const StreamHeader& hd;
    std::string gs;
    int nframes = 0, next = 0;
    GopCursor(const uint8_t* data, size_t len, const StreamHeader& h, int gi)
        : p(data), n(len), hd(h), gs(std::to_string(gi)) {
        if (n < 2) fail(HIVC_E_TRUNCATED, "group " + gs + " payload too small");
        uint16_t nf;
        std::memcpy(&nf, p, 2);
        nframes = nf;
    }
    void parse(FrameJob& J, HostTimes& ht, std::vector<uint64_t>& bits) {
        const int fi = next++;
        if (pos + 5 > n) fail(HIVC_E_TRUNCATED, "frame record cut short in group " + gs);
        uint8_t ftype = p[pos];
        uint32_t plen = rd_u32(p + pos + 1);
        pos += 5;
        if (ftype > 1) fail(HIVC_E_CODEC, "unknown frame type " + std::to_string(ftype));
        if (pos + plen > n) fail(HIVC_E_TRUNCATED, "prediction payload cut short in group " + gs);
        const uint8_t* pd = p + pos;
        pos += plen;
        size_t used;
        double t0 = now_s();
        J.type = ftype;
        if (ftype == 0) {
            used = parse_intra(pd, plen, 0, hd.height, hd.width, hd.channels, hd.intra_levels, J.intra, bits);
            const double t1 = now_s();
            ht.intra_parse += t1 - t0;
            ht.iv[0].push_back({t0, t1});
        } else {
            if (fi == 0) fail(HIVC_E_CODEC, "group " + gs + " starts with an inter frame");
            used = parse_flow(pd, plen, 0, hd.height, hd.width, hd.flow_levels, J.flow);
            const double t1 = now_s();
            ht.flow_parse += t1 - t0;
            ht.iv[1].push_back({t0, t1});
        }
        if (used != plen) fail(HIVC_E_CODEC, "prediction payload length mismatch in group " + gs);
        if (pos + 4 > n) fail(HIVC_E_TRUNCATED, "frame record cut short in group " + gs);
        uint32_t rlen = rd_u32(p + pos);
        pos += 4;
        if (pos + rlen > n) fail(HIVC_E_TRUNCATED, "residual payload cut short in group " + gs);
        t0 = now_s();
        used = parse_residual(p + pos, rlen, 0, hd.height, hd.width, hd.channels, J.res);
        const double t1 = now_s();
        ht.residual_parse += t1 - t0;
        ht.iv[2].push_back({t0, t1});
        if (used != rlen) fail(HIVC_E_CODEC, "residual payload length mismatch in group " + gs);
        pos += rlen;
    }
    void finish() const {
        if (pos != n) fail(HIVC_E_CODEC, "trailing bytes in group " + gs);
    }
};

void parse_gop(const uint8_t* p, size_t n, const StreamHeader& hd, int gi, std::vector<FrameJob>& jobs, HostTimes& ht,
               std::vector<uint64_t>& bits) {
    GopCursor cur(p, n, hd, gi);
    jobs.resize(cur.nframes);
    for (int fi = 0; fi < cur.nframes; ++fi) cur.parse(jobs[fi], ht, bits);
    cur.finish();
}

// Frame-record layout of one GOP payload (codec.py:494-556; record =
// [u8 type][u32 pred_len][pred][u32 res_len][res]), found from the length
// fields alone: rec[i] = start of record i for every record that fits, plus
// the start of the first one that does not.  `complete` records fit
// structurally (<= the u16 frame count); `end` follows the last of them.
// Output buffers are sized by `complete`, never by the unchecked count, and
// the records can be parsed in parallel (each from its own start).
struct GopLayout {
    int nframes = 0, complete = 0;
    size_t end = 2;
    std::vector<size_t> rec;
};

void scan_gop(const uint8_t* p, size_t n, GopLayout& L) {
    L.rec.clear();
    L.nframes = L.complete = 0;
    L.end = 2;
    if (n < 2) return;
    uint16_t nf;
    std::memcpy(&nf, p, 2);
    L.nframes = nf;
    size_t pos = 2;
    for (int fi = 0; fi < nf; ++fi) {
        L.rec.push_back(pos);
        if (pos + 5 > n) break;
        const uint64_t q = (uint64_t)pos + 5 + rd_u32(p + pos + 1);
        if (q + 4 > n) break;
        const uint64_t e = q + 4 + rd_u32(p + q);
        if (e > n) break;
        pos = (size_t)e;
        L.complete = fi + 1;
        L.end = pos;
    }
}

// Bump allocator over the pinned staging buffer.
struct Packer {
    uint8_t* base = nullptr;
    size_t off = 0;
    bool measure = true;
    template <class T>
    size_t put(const std::vector<T>& v) {
        off = (off + 15) & ~size_t(15);
        size_t o = off;
        if (!measure && !v.empty()) std::memcpy(base + o, v.data(), v.size() * sizeof(T));
        off += v.size() * sizeof(T);
        return o;
    }
};

struct FrameOffsets {
    size_t pts[2], vals[3];
    size_t nodes[2], fvals[2], ftiles[2];
    size_t g[2][6];
};

void pack_frame(Packer& pk, const FrameJob& J, FrameOffsets& o) {
    if (J.type == 0) {
        int ntrees = J.intra.nchan == 3 ? 2 : 1;
        for (int t = 0; t < ntrees; ++t) o.pts[t] = pk.put(J.intra.pts[t]);
        for (int c = 0; c < J.intra.nchan; ++c) o.vals[c] = pk.put(J.intra.vals[c]);
    } else {
        for (int c = 0; c < 2; ++c) {
            o.nodes[c] = pk.put(J.flow.nodes[c]);
            o.fvals[c] = pk.put(J.flow.vals[c]);
            o.ftiles[c] = pk.put(J.flow.tiles[c]);
        }
    }
    for (int gi = 0; gi < J.res.ngroups; ++gi) {
        const ResidualGroup& G = J.res.g[gi];
        o.g[gi][0] = pk.put(G.tile_words);
        o.g[gi][1] = pk.put(G.word_prefix);
        o.g[gi][2] = pk.put(G.block_mask);
        o.g[gi][3] = pk.put(G.block_off);
        o.g[gi][4] = pk.put(G.c_sym);
        o.g[gi][5] = pk.put(G.a_sym);
    }
}

template <class T>
const T* at(const uint8_t* base, size_t off) {
    return reinterpret_cast<const T*>(base + off);
}

}  // namespace

// ---------------------------------------------------------------- slots

void Slot::init(int dev) {
    if (stream) return;
    device = dev;
    // (a higher priority for the P-frame streams than for the solver stream
    // measured slower: 4270 vs 4400 frames/s; a higher priority for the solver
    // (and pre) streams measured no faster: profiles/r02n_ab_prio.txt)
    static const bool prio = debug_opt("p_prio") != nullptr;
    if (prio) {
        int lo = 0, hi = 0;
        CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_CHECK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, hi));
    } else {
        CUDA_CHECK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    }
    CUDA_CHECK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    for (auto& e : up_ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : frame_ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&out_free, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&intra_ready, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&intra_done, cudaEventDisableTiming));
    ws.pack_bands = true;  // batched solves run side by side: throughput mode
}

void Slot::reserve_planes(int h, int w, int channels) {
    size_t n = (size_t)h * w;
    if (n <= plane_px && channels <= chans) return;
    CUDA_CHECK(cudaStreamSynchronize(stream));
    for (int c = 0; c < 3; ++c) {
        if (f[c]) cudaFree(f[c]);
        if (u[c]) cudaFree(u[c]);
        f[c] = u[c] = nullptr;
        for (int k = 0; k < 2; ++k) {
            if (ring[k][c]) cudaFree(ring[k][c]);
            ring[k][c] = nullptr;
        }
    }
    for (int t = 0; t < 2; ++t) {
        if (m[t]) cudaFree(m[t]);
        m[t] = nullptr;
    }
    for (int c = 0; c < channels; ++c) {
        CUDA_CHECK(cudaMalloc(&f[c], n * sizeof(double)));
        CUDA_CHECK(cudaMalloc(&u[c], n * sizeof(double)));
        if (channels == 3)
            for (int k = 0; k < 2; ++k) CUDA_CHECK(cudaMalloc(&ring[k][c], n * sizeof(int16_t)));
    }
    for (int t = 0; t < (channels == 3 ? 2 : 1); ++t) CUDA_CHECK(cudaMalloc(&m[t], n));
    plane_px = n;
    chans = channels;
}

void Slot::stage_begin_call(size_t min_bytes) {
    // the previous call has synchronised: consolidate into one block
    size_t want = std::max(min_bytes, stage_used + stage_used / 4);
    if (stage.size() != 1 || stage[0].cap < want) {
        for (auto& b : stage) {
            if (b.host) cudaFreeHost(b.host);
            if (b.dev) cudaFree(b.dev);
        }
        stage.clear();
        StageBlock b;
        b.cap = std::max(want, (size_t)1 << 20);
        CUDA_CHECK(cudaHostAlloc(&b.host, b.cap, cudaHostAllocDefault));
        CUDA_CHECK(cudaMalloc(&b.dev, b.cap));
        stage.push_back(b);
    }
    stage_off = 0;
    stage_used = 0;
}

void Slot::stage_alloc(size_t bytes, uint8_t*& host, uint8_t*& dev) {
    bytes = (bytes + 255) & ~size_t(255);
    if (stage.empty() || stage_off + bytes > stage.back().cap) {  // chain a block (no wait, no free mid-call)
        StageBlock b;
        b.cap = std::max(bytes, stage.empty() ? (size_t)1 << 20 : 2 * stage.back().cap);
        CUDA_CHECK(cudaHostAlloc(&b.host, b.cap, cudaHostAllocDefault));
        CUDA_CHECK(cudaMalloc(&b.dev, b.cap));
        stage.push_back(b);
        stage_off = 0;
    }
    host = stage.back().host + stage_off;
    dev = stage.back().dev + stage_off;
    stage_off += bytes;
    stage_used += bytes;
}

void Slot::reserve_gop_out(size_t bytes) {
    if (bytes <= gop_out_cap) return;
    CUDA_CHECK(cudaStreamSynchronize(copy));
    if (gop_out) cudaFree(gop_out);
    CUDA_CHECK(cudaMalloc(&gop_out, bytes));
    gop_out_cap = bytes;
}

Slot::~Slot() {
    if (stream) cudaStreamSynchronize(stream);
    if (copy) cudaStreamSynchronize(copy);
    for (int c = 0; c < 3; ++c) {
        if (f[c]) cudaFree(f[c]);
        if (u[c]) cudaFree(u[c]);
        for (int k = 0; k < 2; ++k)
            if (ring[k][c]) cudaFree(ring[k][c]);
    }
    for (int t = 0; t < 2; ++t)
        if (m[t]) cudaFree(m[t]);
    if (gop_out) cudaFree(gop_out);
    for (auto& b : stage) {
        if (b.host) cudaFreeHost(b.host);
        if (b.dev) cudaFree(b.dev);
    }
    for (auto& e : frame_ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {out_free, intra_ready, intra_done})
        if (e) cudaEventDestroy(e);
    if (up) cudaStreamSynchronize(up);
    for (auto& e : up_ev)
        if (e) cudaEventDestroy(e);
    if (up) cudaStreamDestroy(up);
    if (copy) cudaStreamDestroy(copy);
    if (stream) cudaStreamDestroy(stream);
}

Context::~Context() {
    slots.clear();
    probe.reset();
    if (d_status) cudaFree(d_status);
    if (op_hi) cudaFree(op_hi);
    if (solver) cudaStreamDestroy(solver);
    for (cudaStream_t p : pre)
        if (p) cudaStreamDestroy(p);
    if (stream) cudaStreamDestroy(stream);
}

// Host-only parse of a whole stream (no GPU): per frame 8 int64 —
// type, intra mask points (Y), flow leaves u, flow leaves v, residual marker,
// coded blocks (group 0), mask points (group 0), coded blocks (group 1).
void parse_stream_stats(const uint8_t* data, size_t len, std::vector<int64_t>& stats, double* seconds) {
    const double t0 = now_s();
    StreamHeader hd = parse_header(data, len);
    std::vector<std::pair<size_t, size_t>> gops;
    split_gops(data, len, hd, gops);
    std::vector<FrameJob> jobs;
    std::vector<uint64_t> bits;
    HostTimes ht;
    stats.clear();
    for (size_t g = 0; g < gops.size(); ++g) {
        parse_gop(data + gops[g].first, gops[g].second, hd, (int)g, jobs, ht, bits);
        for (const FrameJob& J : jobs) {
            int64_t leaves[2] = {0, 0};
            for (int c = 0; c < 2 && J.type == 1; ++c) leaves[c] = (int64_t)J.flow.vals[c].size();
            stats.push_back(J.type);
            stats.push_back(J.type == 0 ? (int64_t)J.intra.pts[0].size() : 0);
            stats.push_back(leaves[0]);
            stats.push_back(leaves[1]);
            stats.push_back(J.res.zero ? 0 : 1);
            stats.push_back(J.res.ngroups > 0 ? J.res.g[0].nblocks : 0);
            stats.push_back(J.res.ngroups > 0 ? J.res.g[0].npoints : 0);
            stats.push_back(J.res.ngroups > 1 ? J.res.g[1].nblocks : 0);
        }
    }
    if (seconds) *seconds = now_s() - t0;
}

void gop_frame_counts(const uint8_t* data, size_t len, std::vector<int32_t>& counts) {
    StreamHeader hd = parse_header(data, len);
    std::vector<std::pair<size_t, size_t>> gops;
    split_gops(data, len, hd, gops);
    counts.resize(gops.size());
    GopLayout lay;
    for (size_t g = 0; g < gops.size(); ++g) {
        if (gops[g].second < 2) fail(HIVC_E_TRUNCATED, "group " + std::to_string(g) + " payload too small");
        // frames whose records fit (= the u16 count on a valid stream): a corrupt
        // count cannot size the output beyond the frames the payload can hold
        scan_gop(data + gops[g].first, gops[g].second, lay);
        counts[g] = lay.complete;
    }
}

// ---------------------------------------------------------------- decode

namespace {

struct StreamJob {
    const uint8_t* data = nullptr;
    size_t len = 0;
    StreamHeader hd{};
    std::vector<std::pair<size_t, size_t>> gops;
    std::vector<size_t> frame_base;  // first output frame of each GOP (relative to gop_begin)
    uint8_t* out = nullptr;
    int gop_begin = 0, gop_end = 0;
};

struct EvRec {
    cudaEvent_t first = nullptr, second = nullptr;
    int stream = 0, gop = 0, frame = 0;
};
using EvPairs = std::vector<EvRec>;

double drain(EvPairs& v, cudaEvent_t origin, char kind, int lane, std::string* timeline,
             std::vector<std::pair<double, double>>* iv = nullptr) {
    double t = 0;
    for (auto& e : v) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e.first, e.second);
        t += ms * 1e-3;
        if (iv) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, origin, e.first);
            cudaEventElapsedTime(&b, origin, e.second);
            iv->push_back({a * 1e-3, b * 1e-3});
        }
        if (timeline) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, origin, e.first);
            cudaEventElapsedTime(&b, origin, e.second);
            char line[160];
            std::snprintf(line, sizeof line, "%d,%c,%d,%d,%d,%.1f,%.1f\n", lane, kind, e.stream, e.gop, e.frame,
                          a * 1e3, b * 1e3);
            *timeline += line;
        }
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    v.clear();
    return t;
}

// One (stream, GOP) of a decode call.  Its frame records are parsed by any
// pool thread (frame 0 in the intra phase, every later record as its own
// task); frames are launched on the item's stream strictly in order by
// whichever thread completes the parsed prefix (try_launch, under `mu`).
struct Item {
    int stream = 0, gop = 0, group = 0;
    Slot* slot = nullptr;
    GopLayout lay;
    int nf = 0;
    std::unique_ptr<std::mutex> mu;  // launch state, errors, host times
    std::vector<uint8_t> parsed;     // per frame: record parsed (under mu)
    int next_launch = 1;             // next P frame to launch (under mu)
    bool head_done = false;          // I-frame finalize + frame 0 copy queued (under mu)
    bool finished = false;           // every frame launched, `done` recorded (under mu)
    int err_frame = 1 << 30;         // frame of the recorded error (the earliest wins)
    const double* qtab = nullptr;  // device dequantisation table (ResDev::qtab), shipped with frame 0
    FrameArgs a0;  // I-frame finalize (frame 0)
    uint8_t* gop_dev = nullptr;
    uint8_t* gop_host = nullptr;
    bool solve0 = false;  // frame 0 staged and waiting for the batched solve
    int code = HIVC_OK;
    std::string msg;
    HostTimes ht;
    int64_t h2d = 0, d2h = 0, inter_frames = 0, intra_frames = 0;
    EvPairs ev_inter, ev_intra, ev_ifin;
    cudaEvent_t done = nullptr;
    bool issued = false;  // its I-frame solve is queued (under mu)
    double h_i0 = 0, h_i1 = 0, h_issue = 0, h_p0 = 0, h_p1 = 0;  // host timeline (HIVC_TIMELINE)
};

// Same-shape items whose I-frame solves are issued as batches: as soon as
// kMinBatch of them are parsed (a packed band level runs up to 4 side by
// side), and the rest when the last one is.  3 measured better than 4 for
// config 3 (three runs each on one box: 5828-5912 vs 5679-5770 frames/s,
// e2e 5337-5454 vs 4915-5012; profiles/r02_summary.md).
constexpr int kMinBatch = 3;
struct Group {
    int h = 0, w = 0, c = 0;
    std::vector<int> items;
    std::mutex mu;
    int pending = 0;         // items whose intra phase has not finished (under mu)
    std::vector<int> ready;  // parsed, not yet issued (under mu)
};

// Record an error of frame fi; the reference decodes in order, so the
// earliest failing frame's error is the one it raises.
void fail_item(Item& it, int code, const std::string& msg, int fi = 0) {
    std::lock_guard<std::mutex> lk(*it.mu);
    if (it.code == HIVC_OK || fi < it.err_frame) {
        it.code = code;
        it.msg = msg;
        it.err_frame = fi;
    }
}

// Pack frames [fi, fi + cnt) of the item into the next staging buffer and ship them.
const uint8_t* stage_chunk(Slot& L, Item& it, size_t fi, int cnt, FrameOffsets* offs,
                           const std::vector<double>* table = nullptr, size_t* table_off = nullptr) {
    Packer pk;
    for (int k = 0; k < cnt; ++k) pack_frame(pk, it.slot->jobs[fi + k], offs[k]);
    if (table) *table_off = pk.put(*table);
    uint8_t *host, *dev;
    L.stage_alloc(pk.off + 16, host, dev);
    pk.base = host;
    pk.off = 0;
    pk.measure = false;
    for (int k = 0; k < cnt; ++k) pack_frame(pk, it.slot->jobs[fi + k], offs[k]);
    if (table) pk.put(*table);
    // upload on the slot's own copy stream; the compute stream waits for it
    CUDA_CHECK(cudaMemcpyAsync(dev, host, pk.off, cudaMemcpyHostToDevice, L.up));
    cudaEvent_t ue = L.up_ev[L.up_next++ % Slot::kUpEv];
    CUDA_CHECK(cudaEventRecord(ue, L.up));
    CUDA_CHECK(cudaStreamWaitEvent(L.stream, ue, 0));
    it.h2d += (int64_t)pk.off;
    return dev;
}

// Frame arguments of frame fi (prediction source, residual, outputs).
FrameArgs frame_args(Slot& L, const StreamHeader& hd, Item& it, size_t fi, const FrameOffsets& o, const uint8_t* dev) {
    const int h = hd.height, w = hd.width, C = hd.channels;
    const size_t N = (size_t)h * w, frame_bytes = N * C;
    const FrameJob& J = it.slot->jobs[fi];
    FrameArgs A;
    A.h = h;
    A.w = w;
    A.channels = C;
    uint8_t* fr = it.gop_dev + fi * frame_bytes;
    uint8_t* frprev = fi ? it.gop_dev + (fi - 1) * frame_bytes : nullptr;
    for (int c = 0; c < C; ++c) {
        if (C == 1) {
            A.recon[c] = fr;  // gray: the reconstruction IS the output frame
            A.prev[c] = frprev;
        } else {
            A.recon[c] = L.ring[fi & 1][c];
            A.prev[c] = L.ring[(fi + 1) & 1][c];
            A.rgb[c] = fr + c * N;
        }
        A.u[c] = L.u[c];
    }
    ResDev& RD = A.res;
    RD.ngroups = J.res.zero ? 0 : J.res.ngroups;
    RD.dz_step = 127.0 / (double)((hd.residual_levels - 1) / 2);  // quantize.py:43-47
    RD.c_scale = J.res.c_scale;
    RD.a_scale = J.res.a_scale;
    RD.qtab = it.qtab;
    for (int g = 0; g < RD.ngroups; ++g) {
        const ResidualGroup& G = J.res.g[g];
        ResGroupDev& D = RD.g[g];
        D.nplanes = G.nplanes;
        D.nblocks = G.nblocks;
        D.npoints = G.npoints;
        D.tile_words = at<uint64_t>(dev, o.g[g][0]);
        D.word_prefix = at<int32_t>(dev, o.g[g][1]);
        D.block_mask = at<uint64_t>(dev, o.g[g][2]);
        D.block_off = at<int32_t>(dev, o.g[g][3]);
        D.c_sym = at<int32_t>(dev, o.g[g][4]);
        D.a_sym = at<int32_t>(dev, o.g[g][5]);
    }
    if (J.type == 1)
        for (int c = 0; c < 2; ++c) {
            A.flow.nodes[c] = at<int32_t>(dev, o.nodes[c]);
            A.flow.vals[c] = at<double>(dev, o.fvals[c]);
            A.flow.tiles[c] = at<uint16_t>(dev, o.ftiles[c]);
            A.flow.nleaves[c] = (int)J.flow.vals[c].size();
        }
    return A;
}

// f = 0 with the intra values scattered at the mask points (prediction.py:203-208), on the slot stream.
void scatter_intra(Context& ctx, Slot& L, const StreamHeader& hd, const FrameJob& J, const FrameOffsets& o,
                   const uint8_t* dev) {
    const size_t N = (size_t)hd.height * hd.width;
    for (int c = 0; c < hd.channels; ++c) {
        const int t = c == 0 ? 0 : 1;
        CUDA_CHECK(cudaMemsetAsync(L.f[c], 0, N * sizeof(double), L.stream));
        if (c <= 1) CUDA_CHECK(cudaMemsetAsync(L.m[t], 0, N, L.stream));
        launch_scatter(at<int32_t>(dev, o.pts[t]), at<double>(dev, o.vals[c]), (int)J.intra.pts[t].size(), L.f[c],
                       c <= 1 ? L.m[t] : nullptr, L.stream);
        ctx.launches += 1;
    }
}

struct CallState {
    Context& ctx;
    std::vector<StreamJob>& streams;
    std::vector<Item>& items;
    std::deque<Group>& groups;
    bool out_on_device;  // frames written straight into `out` (out_mode 1)
    bool timed;
    cudaEvent_t origin;
    double t0;     // host clock at the origin event
    int out_mode;  // 0 host, 1 device, 2 device through per-frame staged copies (peer / IPC destinations)
};

// A finished frame leaves the slot's GOP buffer on the copy stream while the
// next frames decode: D2H into host frames (out_mode 0), or device-to-device
// into a peer GPU's frame buffer over NVLink (out_mode 2: the multi-GPU
// gather fused into the decode, frame by frame).
void copy_out(CallState& cs, Slot& L, Item& it, size_t fi, size_t frame_bytes) {
    if (cs.out_on_device) return;
    cudaEvent_t fe = L.frame_ev[L.frame_ev_next++ % Slot::kFrameEv];
    CUDA_CHECK(cudaEventRecord(fe, L.stream));
    CUDA_CHECK(cudaStreamWaitEvent(L.copy, fe, 0));
    const bool d2d = cs.out_mode == 2;
    CUDA_CHECK(cudaMemcpyAsync(it.gop_host + fi * frame_bytes, it.gop_dev + fi * frame_bytes, frame_bytes,
                               d2d ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, L.copy));
    if (!d2d) it.d2h += (int64_t)frame_bytes;
}

// Solve the staged I-frames of items idx (same shape): pyramid + cluster
// levels on a side stream, grid levels on the solver stream; each item's
// intra_done is recorded as soon as its own solve is complete (the finest
// levels run one solve after another), so its finalize and P frames start
// while the batch's later solves still run.  Callers hold ctx.solver_mu.
void issue_solves(CallState& cs, const std::vector<int>& idx, const StreamHeader& hd) {
    Context& ctx = cs.ctx;
    const int h = hd.height, w = hd.width, C = hd.channels;
    const cudaStream_t pre = ctx.pre[ctx.pre_next++ % Context::kPre];
    for (size_t b0 = 0; b0 < idx.size(); b0 += kMaxBatch) {
        const int K = (int)std::min<size_t>(kMaxBatch, idx.size() - b0);
        for (int j = 0; j < K; ++j) CUDA_CHECK(cudaStreamWaitEvent(pre, cs.items[idx[b0 + j]].slot->intra_ready, 0));
        EvRec r;
        if (cs.timed) {
            const Item& i0 = cs.items[idx[b0]];
            r.stream = i0.stream;
            r.gop = i0.gop;
            CUDA_CHECK(cudaEventCreate(&r.first));
            CUDA_CHECK(cudaEventCreate(&r.second));
            CUDA_CHECK(cudaEventRecord(r.first, pre));
        }
        int64_t launches = 0;
        for (int c = 0; c < C; ++c) {
            SolveJob sj[kMaxBatch];
            for (int j = 0; j < K; ++j) {
                Slot& L = *cs.items[idx[b0 + j]].slot;
                sj[j] = {&L.ws, L.f[c], L.m[c == 0 ? 0 : 1], L.u[c], c == C - 1 ? L.intra_done : nullptr};
            }
            solve_batch_async(sj, K, h, w, 1e-4, 160, ctx.solver, &launches, cs.timed ? &ctx.probe : nullptr, pre);
        }
        ctx.launches += launches;
        if (cs.timed) {  // the batch interval (stage sums stay per batch), kept with its first item
            CUDA_CHECK(cudaEventRecord(r.second, ctx.solver));
            cs.items[idx[b0]].ev_intra.push_back(r);
        }
        for (int j = 0; j < K; ++j) cs.items[idx[b0 + j]].solve0 = false;
    }
}

// I-frame finalize (rint / clip / RCT of the inpainted planes + residual) on the slot stream.
void finalize_intra(CallState& cs, Item& it, const FrameArgs& A, int frame) {
    Slot& L = *it.slot;
    CUDA_CHECK(cudaStreamWaitEvent(L.stream, L.intra_done, 0));
    EvRec r;
    r.stream = it.stream;
    r.gop = it.gop;
    r.frame = frame;
    if (cs.timed) {
        CUDA_CHECK(cudaEventCreate(&r.first));
        CUDA_CHECK(cudaEventCreate(&r.second));
        CUDA_CHECK(cudaEventRecord(r.first, L.stream));
    }
    launch_frame(A, false, L.stream);
    cs.ctx.launches += 1;
    if (cs.timed) {
        CUDA_CHECK(cudaEventRecord(r.second, L.stream));
        it.ev_ifin.push_back(r);
    }
}

// The item's last frame is queued: its device span ends there (and, with
// host output, with its last D2H copy).  Callers hold it.mu or run alone.
void finish_item(CallState& cs, Item& it) {
    Slot& L = *it.slot;
    if (!cs.out_on_device) {
        cudaEventRecord(L.out_free, L.copy);
        cudaStreamWaitEvent(L.stream, L.out_free, 0);
    }
    cudaEventRecord(it.done, L.stream);
    it.finished = true;
    it.h_p1 = now_s() - cs.t0;
}

// Queue everything of the item that can go now, in frame order: the I-frame
// finalize once its solve is issued, then every parsed P frame of the
// unbroken prefix (one staged upload, kernel and copy-out each).
void try_launch(CallState& cs, Item& it) {
    std::lock_guard<std::mutex> lk(*it.mu);
    if (!it.issued || it.finished) return;
    const StreamHeader& hd = cs.streams[it.stream].hd;
    Slot& L = *it.slot;
    const size_t frame_bytes = (size_t)hd.height * hd.width * hd.channels;
    int fi = 0;
    try {
        CUDA_CHECK(cudaSetDevice(L.device));
        if (it.nf > 0 && it.err_frame > 0 && !it.head_done) {
            finalize_intra(cs, it, it.a0, 0);
            copy_out(cs, L, it, 0, frame_bytes);
            it.head_done = true;
        }
        while (it.next_launch < it.nf && it.parsed[it.next_launch] && it.next_launch < it.err_frame) {
            fi = it.next_launch;
            FrameOffsets o[1];
            const uint8_t* dev = stage_chunk(L, it, (size_t)fi, 1, o);
            const FrameJob& J = L.jobs[fi];
            FrameArgs A = frame_args(L, hd, it, (size_t)fi, o[0], dev);
            EvRec e;
            e.stream = it.stream;
            e.gop = it.gop;
            e.frame = fi;
            if (cs.timed) {
                CUDA_CHECK(cudaEventCreate(&e.first));
                CUDA_CHECK(cudaEventCreate(&e.second));
                CUDA_CHECK(cudaEventRecord(e.first, L.stream));
            }
            if (J.type == 0) {
                // an intra frame inside the GOP: solved alone on the solver stream
                scatter_intra(cs.ctx, L, hd, J, o[0], dev);
                CUDA_CHECK(cudaEventRecord(L.intra_ready, L.stream));
                {
                    std::lock_guard<std::mutex> sl(cs.ctx.solver_mu);
                    issue_solves(cs, std::vector<int>{(int)(&it - cs.items.data())}, hd);
                }
                finalize_intra(cs, it, A, fi);
                it.intra_frames += 1;
            } else {
                static const int prep = debug_opt("p_repeat") ? std::atoi(debug_opt("p_repeat")) : 1;
                for (int rep = 0; rep < prep; ++rep) launch_frame(A, true, L.stream);
                cs.ctx.launches += 1;
                it.inter_frames += 1;
            }
            if (cs.timed) {
                CUDA_CHECK(cudaEventRecord(e.second, L.stream));
                it.ev_inter.push_back(e);
            }
            copy_out(cs, L, it, (size_t)fi, frame_bytes);
            ++it.next_launch;
        }
        if (it.next_launch >= it.nf && it.code == HIVC_OK) finish_item(cs, it);
    } catch (const Error& e) {
        if (it.code == HIVC_OK || fi < it.err_frame) it.code = e.code, it.msg = e.what(), it.err_frame = fi;
    } catch (const std::exception& e) {
        if (it.code == HIVC_OK || fi < it.err_frame) it.code = HIVC_E_ARGUMENT, it.msg = e.what(), it.err_frame = fi;
    }
}

// A cursor over the item's GOP payload positioned at record fi.
GopCursor cursor_at(CallState& cs, const Item& it, int fi) {
    const StreamJob& S = cs.streams[it.stream];
    GopCursor cur(S.data + S.gops[it.gop].first, S.gops[it.gop].second, S.hd, it.gop);
    cur.pos = it.lay.rec[fi];
    cur.next = fi;
    return cur;
}

// Phase 1 of an item: parse + ship its I-frame, scatter the mask values; the
// last item of a shape group issues the group's batched solves.
void intra_phase(CallState& cs, Item& it) {
    std::vector<uint64_t>& bits = it.slot->bits;
    const StreamJob& S = cs.streams[it.stream];
    const StreamHeader& hd = S.hd;
    Slot& L = *it.slot;
    const size_t frame_bytes = (size_t)hd.height * hd.width * hd.channels;
    it.h_i0 = now_s() - cs.t0;
    try {
        CUDA_CHECK(cudaSetDevice(L.device));
        CUDA_CHECK(cudaStreamWaitEvent(L.stream, cs.origin, 0));
        CUDA_CHECK(cudaStreamWaitEvent(L.copy, cs.origin, 0));
        CUDA_CHECK(cudaStreamWaitEvent(L.up, cs.origin, 0));
        it.gop_dev = cs.out_on_device ? S.out + S.frame_base[it.gop] * frame_bytes : L.gop_out;
        it.gop_host = cs.out_on_device ? nullptr : S.out + S.frame_base[it.gop] * frame_bytes;
        if (!cs.out_on_device) CUDA_CHECK(cudaStreamWaitEvent(L.stream, L.out_free, 0));  // last call's copies
        if (S.gops[it.gop].second < 2) fail(HIVC_E_TRUNCATED, "group " + std::to_string(it.gop) + " payload too small");
        if (it.nf > 0) {
            GopCursor cur = cursor_at(cs, it, 0);
            HostTimes ht;
            cur.parse(L.jobs[0], ht, bits);  // frame 0 must be intra (codec.py:503)
            if (it.nf == 1) cur.finish();
            {
                std::lock_guard<std::mutex> lk0(*it.mu);
                it.ht.add(ht);
            }
            FrameOffsets o[1];
            std::vector<double> qt(255);  // s * dz_step / 127 for |s| <= 127 (quantize.py:43-47, codec.py:316-321)
            const double dz = 127.0 / (double)((hd.residual_levels - 1) / 2);
            for (int k = 0; k < 255; ++k) qt[k] = (double)(k - 127) * dz / 127.0;
            size_t qoff = 0;
            const uint8_t* dev = stage_chunk(L, it, 0, 1, o, &qt, &qoff);
            it.qtab = reinterpret_cast<const double*>(dev + qoff);
            scatter_intra(cs.ctx, L, hd, L.jobs[0], o[0], dev);
            CUDA_CHECK(cudaEventRecord(L.intra_ready, L.stream));
            it.a0 = frame_args(L, hd, it, 0, o[0], dev);
            it.intra_frames += 1;
            it.solve0 = true;
        } else {
            GopCursor(S.data + S.gops[it.gop].first, S.gops[it.gop].second, hd, it.gop).finish();
        }
    } catch (const Error& e) {
        fail_item(it, e.code, e.what(), 0);
    } catch (const std::exception& e) {
        fail_item(it, HIVC_E_ARGUMENT, e.what(), 0);
    }
    it.h_i1 = now_s() - cs.t0;
    Group& g = cs.groups[it.group];
    std::vector<int> batch;
    {
        std::lock_guard<std::mutex> lk(g.mu);
        const int self = (int)(&it - cs.items.data());
        if (it.code == HIVC_OK && it.solve0) g.ready.push_back(self);
        --g.pending;
        static const int min_batch = [] {
            const char* e = debug_opt("min_batch");
            return e ? std::max(1, std::atoi(e)) : kMinBatch;
        }();
        // (never leave a lone straggler behind a batch: its cluster levels could
        // not start until the batch's full-GPU levels are done)
        if (g.pending == 0 || ((int)g.ready.size() >= min_batch && g.pending >= 2)) batch.swap(g.ready);
    }
    if (!batch.empty()) {
        for (int i : batch) cs.items[i].h_issue = now_s() - cs.t0;
        try {
            std::lock_guard<std::mutex> lk(cs.ctx.solver_mu);
            CUDA_CHECK(cudaSetDevice(cs.ctx.device));
            issue_solves(cs, batch, hd);
        } catch (const Error& e) {
            for (int i : batch) fail_item(cs.items[i], e.code, e.what(), 0);
        } catch (const std::exception& e) {
            for (int i : batch) fail_item(cs.items[i], HIVC_E_ARGUMENT, e.what(), 0);
        }
    }
    // the batch (and a failed / empty item itself) may now launch their frames
    auto release = [&](Item& x) {
        {
            std::lock_guard<std::mutex> lk(*x.mu);
            x.issued = true;
        }
        try_launch(cs, x);
    };
    for (int i : batch) release(cs.items[i]);
    bool solo;  // not waiting for a solve (failed, or no frames)
    {
        std::lock_guard<std::mutex> lk(*it.mu);
        solo = !(it.err_frame > 0 && it.solve0) || it.nf == 0;
    }
    if (solo) release(it);
}

// Phase 2, one task per later frame record: parse it (bit-exact host C++),
// then launch whatever prefix of the item is ready.
void frame_task(CallState& cs, Item& it, int fi) {
    {
        std::lock_guard<std::mutex> lk(*it.mu);
        if (it.code != HIVC_OK && it.err_frame <= fi) return;  // an earlier frame failed: the reference stops there
        if (it.h_p0 == 0) it.h_p0 = now_s() - cs.t0;
    }
    HostTimes ht;
    try {
        GopCursor cur = cursor_at(cs, it, fi);
        std::vector<uint64_t> bits;  // (an intra record inside the GOP)
        cur.parse(it.slot->jobs[fi], ht, bits);
        if (fi == it.nf - 1) cur.finish();
    } catch (const Error& e) {
        fail_item(it, e.code, e.what(), fi);
        return;
    } catch (const std::exception& e) {
        fail_item(it, HIVC_E_ARGUMENT, e.what(), fi);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(*it.mu);
        it.parsed[fi] = 1;
        it.ht.add(ht);
    }
    try_launch(cs, it);
}

}  // namespace

// Persistent decode workers: created once, parked between calls, so a call's
// parse workers all start within microseconds instead of one thread creation
// after another (the first I-frame parses gate the first solve batch).  A pool
// thread may lower its scheduling priority during a call (frame tasks); it
// returns to nice 0 before the next call, and when the process is not allowed
// to raise it back, `renice_ok()` turns false and later calls keep it.
class WorkerPool {
   public:
    static WorkerPool& get() {
        static WorkerPool p;
        return p;
    }
    static std::atomic<bool>& renice_ok() {
        static std::atomic<bool> ok{true};
        return ok;
    }
    // fn(true) on n - 1 pool threads and fn(false) on the caller; false when
    // the pool is busy with another call (the caller then makes its own threads)
    bool run(int n, const std::function<void(bool)>& fn) {
        if (getpid() != pid_) return false;  // a forked child has none of the parent's threads
        std::unique_lock<std::mutex> busy(run_mu_, std::try_to_lock);
        if (!busy.owns_lock()) return false;
        {
            std::lock_guard<std::mutex> lk(mu_);
            while ((int)th_.size() < n - 1) {
                const int idx = (int)th_.size();
                th_.emplace_back([this, idx]() { loop(idx); });
            }
            job_ = &fn;
            want_ = n - 1;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(false);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&]() { return pending_ == 0; });
        job_ = nullptr;
        return true;
    }
    ~WorkerPool() {
        if (getpid() != pid_) {  // not ours to join
            for (auto& t : th_) t.detach();
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }

   private:
    void loop(int idx) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(bool)>* job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&]() { return stop_ || (gen_ != seen && idx < want_); });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            (*job)(true);
            // back to the default priority for the next call's I-frame parses
            const pid_t tid = (pid_t)syscall(SYS_gettid);
            if (getpriority(PRIO_PROCESS, (id_t)tid) != 0 && setpriority(PRIO_PROCESS, (id_t)tid, 0) != 0)
                renice_ok() = false;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_cv_.notify_all();
            }
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> th_;
    const std::function<void(bool)>* job_ = nullptr;
    int want_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
    const pid_t pid_ = getpid();
};

void decode_streams(Context& ctx, int nstreams, const uint8_t* const* data, const size_t* len, const int* gop_begin,
                    const int* gop_end, uint8_t* const* out, int out_mode, double* stage_seconds) {
    const bool out_on_device = out_mode == 1;
    double t_all = now_s();
    std::vector<StreamJob> streams(nstreams);
    std::vector<Item> items;
    int max_h = 1, max_w = 1, max_c = 1;
    size_t max_gop_bytes = 1;
    for (int k = 0; k < nstreams; ++k) {
        StreamJob& S = streams[k];
        S.data = data[k];
        S.len = len[k];
        S.out = out[k];
        S.hd = parse_header(S.data, S.len);
        split_gops(S.data, S.len, S.hd, S.gops);
        const int ngops = (int)S.gops.size();
        S.gop_begin = gop_begin ? std::max(0, gop_begin[k]) : 0;
        S.gop_end = (!gop_end || gop_end[k] < 0 || gop_end[k] > ngops) ? ngops : gop_end[k];
        if (S.gop_begin > S.gop_end) fail(HIVC_E_ARGUMENT, "bad GOP range");
        S.frame_base.assign(ngops + 1, 0);
        size_t acc = 0;
        const size_t frame_bytes = (size_t)S.hd.height * S.hd.width * S.hd.channels;
        for (int g = S.gop_begin; g < S.gop_end; ++g) {
            S.frame_base[g] = acc;
            Item it;
            it.stream = k;
            it.gop = g;
            scan_gop(S.data + S.gops[g].first, S.gops[g].second, it.lay);
            it.nf = it.lay.nframes;
            // outputs hold the frames whose records fit (gop_frame_counts): a
            // corrupt count fails in stream order instead of sizing buffers
            acc += (size_t)it.lay.complete;
            max_gop_bytes = std::max(max_gop_bytes, (size_t)it.lay.complete * frame_bytes);
            it.mu = std::make_unique<std::mutex>();
            items.push_back(std::move(it));
        }
        max_h = std::max(max_h, S.hd.height);
        max_w = std::max(max_w, S.hd.width);
        max_c = std::max(max_c, S.hd.channels);
    }
    const int n = (int)items.size();
    // smallest planes first: their I-frames parse fastest, so their batch is
    // issued (and on the GPU) first while the large planes are still parsing
    std::stable_sort(items.begin(), items.end(), [&](const Item& a, const Item& b) {
        const StreamHeader &ha = streams[a.stream].hd, &hb = streams[b.stream].hd;
        return (int64_t)ha.height * ha.width * ha.channels < (int64_t)hb.height * hb.width * hb.channels;
    });
    // shape groups: their I-frame solves are batched
    std::deque<Group> groups;
    for (int i = 0; i < n; ++i) {
        const StreamHeader& hd = streams[items[i].stream].hd;
        int gi = -1;
        for (size_t g = 0; g < groups.size(); ++g)
            if (groups[g].h == hd.height && groups[g].w == hd.width && groups[g].c == hd.channels) gi = (int)g;
        if (gi < 0) {
            groups.emplace_back();
            gi = (int)groups.size() - 1;
            groups[gi].h = hd.height;
            groups[gi].w = hd.width;
            groups[gi].c = hd.channels;
        }
        items[i].group = gi;
        groups[gi].items.push_back(i);
    }
    for (auto& g : groups) g.pending = (int)g.items.size();
    CUDA_CHECK(cudaSetDevice(ctx.device));
    if (!ctx.solver) CUDA_CHECK(cudaStreamCreateWithFlags(&ctx.solver, cudaStreamNonBlocking));
    for (cudaStream_t& p : ctx.pre)
        if (!p) CUDA_CHECK(cudaStreamCreateWithFlags(&p, cudaStreamNonBlocking));
    while ((int)ctx.slots.size() < n) ctx.slots.push_back(std::make_unique<Slot>());
    for (int i = 0; i < n; ++i) {
        Slot& L = *ctx.slots[i];
        L.init(ctx.device);
        L.reserve_planes(max_h, max_w, max_c);
        L.ws.reserve(max_h, max_w, ctx.device);
        if (!out_on_device) L.reserve_gop_out(max_gop_bytes);
        L.stage_begin_call((size_t)4 * max_h * max_w * max_c + 65536);
        items[i].slot = &L;
        CUDA_CHECK(cudaEventCreate(&items[i].done));
        const size_t nrec = items[i].lay.rec.size();
        if (L.jobs.size() < nrec) L.jobs.resize(nrec);
        items[i].parsed.assign(std::max<size_t>(nrec, 1), 0);
    }
    const bool timed = (stage_seconds != nullptr && ctx.stage_events) || debug_opt("timeline");
    cudaEvent_t origin;
    CUDA_CHECK(cudaEventCreate(&origin));
    CUDA_CHECK(cudaEventRecord(origin, ctx.stream));
    CUDA_CHECK(cudaStreamWaitEvent(ctx.solver, origin, 0));
    for (cudaStream_t p : ctx.pre) CUDA_CHECK(cudaStreamWaitEvent(p, origin, 0));
    CallState cs{ctx, streams, items, groups, out_on_device, timed, origin, now_s(), out_mode};
    // task list: every item's intra phase (in batch-issue order), then one task
    // per later frame record, item by item.  Frame records parse independently
    // (each from its own start, GopLayout), so a GOP's P frames are parsed by
    // several threads and are all ready when its I-frame solve completes; a
    // pool thread that reaches the frame tasks drops its scheduling priority
    // (the large I-frames still being parsed gate the next solve batch).
    std::vector<std::pair<int, int>> tasks;
    for (int i = 0; i < n; ++i) tasks.push_back({i, 0});
    for (int i = 0; i < n; ++i) {
        // records 1..complete-1 fit; record `complete` (when short of nf) is parsed
        // too, so the error is the one its own parse meets first
        const int last = std::min(items[i].nf - 1, items[i].lay.complete);
        for (int fi = 1; fi <= last; ++fi) tasks.push_back({i, fi});
    }
    const int ntasks = (int)tasks.size();
    std::atomic<int> next_task{0};
    auto worker = [&](bool pool) {
        bool low = false;
        for (int t; (t = next_task.fetch_add(1)) < ntasks;) {
            const auto [i, fi] = tasks[t];
            if (fi == 0) {
                intra_phase(cs, items[i]);
            } else {
                if (pool && !low && WorkerPool::renice_ok()) {
                    setpriority(PRIO_PROCESS, (id_t)syscall(SYS_gettid), 10);
                    low = true;
                }
                frame_task(cs, items[i], fi);
            }
        }
    };
    static const int kMaxWorkers = [] {
        const char* e = debug_opt("workers");
        // one process per GPU (torchrun): the ranks of a node share its cores
        const char* lws = std::getenv("LOCAL_WORLD_SIZE");
        const int ranks = lws ? std::max(1, std::atoi(lws)) : 1;
        const int hw = std::max(2, (int)std::thread::hardware_concurrency() / ranks);
        // half the hardware threads: each large I-frame parse also runs tree
        // and value helper threads (measured on 16 cores: 8 workers beat 16 by 3 %)
        return e ? std::max(1, std::min(64, std::atoi(e))) : std::max(2, std::min(hw / 2, 32));
    }();
    const int nworkers = std::max(1, std::min(ntasks, kMaxWorkers));
    if (nworkers == 1 || n == 0) {
        worker(false);
    } else if (!WorkerPool::get().run(nworkers, worker)) {
        std::vector<std::thread> th;
        for (int l = 0; l < nworkers; ++l) th.emplace_back(worker, true);
        for (auto& t : th) t.join();
    }
    // items that stopped early (an error) end here
    for (auto& it : items)
        if (!it.finished) finish_item(cs, it);
    double span = 0;
    for (auto& it : items) {
        cudaStreamSynchronize(it.slot->stream);
        cudaStreamSynchronize(it.slot->copy);
        cudaStreamSynchronize(it.slot->up);
        float ms = 0;
        if (cudaEventElapsedTime(&ms, origin, it.done) == cudaSuccess) span = std::max(span, (double)ms * 1e-3);
    }
    cudaStreamSynchronize(ctx.solver);
    std::string timeline;
    std::string* tl = debug_opt("timeline") ? &timeline : nullptr;
    double gpu_intra = 0, gpu_inter = 0, gpu_ifin = 0;
    std::vector<std::pair<double, double>> dev_iv[3];  // solves, P frames, I-frame finalize (s from origin)
    for (int i = 0; i < n; ++i) {
        Item& it = items[i];
        gpu_intra += drain(it.ev_intra, origin, 'I', i, tl, &dev_iv[0]);
        gpu_inter += drain(it.ev_inter, origin, 'P', i, tl, &dev_iv[1]);
        gpu_ifin += drain(it.ev_ifin, origin, 'F', i, tl, &dev_iv[2]);
        if (tl) {  // item completion (incl. its last D2H copy in host-output mode)
            float d = 0;
            cudaEventElapsedTime(&d, origin, it.done);
            char line[96];
            std::snprintf(line, sizeof line, "%d,D,%d,%d,0,%.1f,%.1f\n", i, it.stream, it.gop, d * 1e3, d * 1e3);
            *tl += line;
        }
        cudaEventDestroy(it.done);
        if (tl) {
            char line[200];
            std::snprintf(line, sizeof line, "%d,H,%d,%d,0,%.1f,%.1f\n%d,Q,%d,%d,0,%.1f,%.1f\n", i, it.stream, it.gop,
                          it.h_i0 * 1e6, it.h_i1 * 1e6, i, it.stream, it.gop, it.h_p0 * 1e6, it.h_p1 * 1e6);
            *tl += line;
        }
    }
    cudaEventDestroy(origin);
    if (tl) {
        if (FILE* f = std::fopen(debug_opt("timeline"), "a")) {
            std::fputs(timeline.c_str(), f);
            std::fprintf(f, "-\n");
            std::fclose(f);
        }
    }
    CgTotals cg;
    if (timed) ctx.probe.harvest(cg);
    // the first failing (stream, GOP) in stream order wins (the reference decodes sequentially)
    int worst = -1;
    for (int i = 0; i < n; ++i)
        if (items[i].code != HIVC_OK &&
            (worst < 0 ||
             std::make_pair(items[i].stream, items[i].gop) < std::make_pair(items[worst].stream, items[worst].gop)))
            worst = i;
    if (worst >= 0) fail(items[worst].code, items[worst].msg);
    CUDA_CHECK(cudaGetLastError());
    for (const StreamJob& S : streams) {
        if (S.gop_begin == 0 && S.gop_end == (int)S.gops.size()) {  // codec.py:558-561
            size_t total = 0;
            for (auto& g : S.gops) {
                uint16_t nf;
                std::memcpy(&nf, S.data + g.first, 2);
                total += nf;
            }
            if (total != (size_t)S.hd.frame_count)
                fail(HIVC_E_CODEC, "decoded " + std::to_string(total) + " frames, header promised " +
                                       std::to_string(S.hd.frame_count));
        }
    }
    HostTimes ht;
    {
        std::lock_guard<std::mutex> g(ctx.stats_mu);
        CgTotals& T = ctx.cg;
        T.solves += cg.solves;
        T.pixel_iters += cg.pixel_iters;
        T.pixel_levels += cg.pixel_levels;
        T.grid_launches += cg.grid_launches;
        T.grid_seconds += cg.grid_seconds;
        T.grid_pixel_iters += cg.grid_pixel_iters;
        T.grid_pixels += cg.grid_pixels;
        for (auto& it : items) {
            ctx.h2d_bytes += it.h2d;
            ctx.d2h_bytes += it.d2h;
            ctx.inter_frames += it.inter_frames;
            ctx.intra_frames += it.intra_frames;
            ht.add(it.ht);
        }
        ctx.inter_seconds += gpu_inter;
    }
    if (stage_seconds) {
        // The reference times its stages one after another (codec.py:509-562);
        // here they overlap across GOPs, host threads and streams.  Each stage
        // reports its wall-clock share: the union of its occurrences'
        // intervals (so no stage exceeds `total`):
        //   intra_solve        host intra-payload parse + the batched device solves
        //   flow_parse         host flow-payload parse
        //   warp               the fused P-frame kernels (warp + residual + rint/clip)
        //   residual_parse     host residual-payload parse
        //   residual_transform the I-frame finalize kernels (block rebuild + add + rint/clip)
        //   finalize           0 here: fused into the two kernels above (codec.decode adds the
        //                      host Frame construction)
        auto rel = [&](const std::vector<std::pair<double, double>>& v) {
            std::vector<std::pair<double, double>> r;
            for (auto& x : v) r.push_back({x.first - cs.t0, x.second - cs.t0});
            return r;
        };
        std::vector<std::pair<double, double>> intra = rel(ht.iv[0]);
        intra.insert(intra.end(), dev_iv[0].begin(), dev_iv[0].end());
        double s[8] = {union_length(intra), union_length(rel(ht.iv[1])), union_length(dev_iv[1]),
                       union_length(rel(ht.iv[2])), union_length(dev_iv[2]), 0, 0, 0};
        s[6] = now_s() - t_all;
        s[7] = span;
        std::memcpy(stage_seconds, s, sizeof(s));
    }
}

}  // namespace hivc
