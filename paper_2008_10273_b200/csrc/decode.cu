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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

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

struct FrameJob {
    int type = 0;  // 0 intra, 1 inter
    IntraJob intra;
    FlowJob flow;
    ResidualJob res;
};

struct HostTimes {
    double intra_parse = 0, flow_parse = 0, residual_parse = 0;
};

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
            ht.intra_parse += now_s() - t0;
        } else {
            if (fi == 0) fail(HIVC_E_CODEC, "group " + gs + " starts with an inter frame");
            used = parse_flow(pd, plen, 0, hd.height, hd.width, hd.flow_levels, J.flow);
            ht.flow_parse += now_s() - t0;
        }
        if (used != plen) fail(HIVC_E_CODEC, "prediction payload length mismatch in group " + gs);
        if (pos + 4 > n) fail(HIVC_E_TRUNCATED, "frame record cut short in group " + gs);
        uint32_t rlen = rd_u32(p + pos);
        pos += 4;
        if (pos + rlen > n) fail(HIVC_E_TRUNCATED, "residual payload cut short in group " + gs);
        t0 = now_s();
        used = parse_residual(p + pos, rlen, 0, hd.height, hd.width, hd.channels, J.res);
        ht.residual_parse += now_s() - t0;
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

// ---------------------------------------------------------------- lanes

void Lane::reserve_planes(int h, int w, int channels) {
    size_t n = (size_t)h * w;
    if (n <= plane_px && channels <= chans) return;
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

void Lane::reserve_stage(int slot, size_t bytes) {
    if (bytes <= stage_cap[slot]) return;
    if (host_stage[slot]) cudaFreeHost(host_stage[slot]);
    if (dev_stage[slot]) cudaFree(dev_stage[slot]);
    size_t cap = bytes + bytes / 4 + 4096;
    CUDA_CHECK(cudaHostAlloc(&host_stage[slot], cap, cudaHostAllocDefault));
    CUDA_CHECK(cudaMalloc(&dev_stage[slot], cap));
    stage_cap[slot] = cap;
}

void Lane::reserve_gop_out(size_t bytes) {
    if (!copy) {
        CUDA_CHECK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
        for (auto& e : frame_ev) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : out_free) CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (bytes <= gop_out_cap) return;
    CUDA_CHECK(cudaStreamSynchronize(copy));
    for (int k = 0; k < 2; ++k) {
        if (gop_out[k]) cudaFree(gop_out[k]);
        CUDA_CHECK(cudaMalloc(&gop_out[k], bytes));
    }
    gop_out_cap = bytes;
}

Lane::~Lane() {
    if (stream) cudaStreamSynchronize(stream);
    if (copy) cudaStreamSynchronize(copy);
    for (int c = 0; c < 3; ++c) {
        if (f[c]) cudaFree(f[c]);
        if (u[c]) cudaFree(u[c]);
        for (int k = 0; k < 2; ++k)
            if (ring[k][c]) cudaFree(ring[k][c]);
    }
    for (int t = 0; t < 2; ++t) {
        if (m[t]) cudaFree(m[t]);
        if (gop_out[t]) cudaFree(gop_out[t]);
    }
    for (int t = 0; t < kStage; ++t) {
        if (host_stage[t]) cudaFreeHost(host_stage[t]);
        if (dev_stage[t]) cudaFree(dev_stage[t]);
        if (staged[t]) cudaEventDestroy(staged[t]);
    }
    if (copy) cudaStreamSynchronize(copy);
    for (auto& e : frame_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : out_free)
        if (e) cudaEventDestroy(e);
    if (copy) cudaStreamDestroy(copy);
    if (stream) cudaStreamDestroy(stream);
}

Context::~Context() {
    lanes.clear();
    if (d_status) cudaFree(d_status);
    if (op_hi) cudaFree(op_hi);
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
    for (size_t g = 0; g < gops.size(); ++g) {
        if (gops[g].second < 2) fail(HIVC_E_TRUNCATED, "group " + std::to_string(g) + " payload too small");
        uint16_t nf;
        std::memcpy(&nf, data + gops[g].first, 2);
        counts[g] = nf;
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

struct WorkItem {
    int stream, gop;
};

struct LaneResult {
    int code = HIVC_OK;
    int stream = -1, gop = -1;
    std::string msg;
    HostTimes ht;
    double gpu_intra = 0, gpu_inter = 0, gpu_ifinal = 0;
    int64_t h2d = 0, d2h = 0;
    int64_t inter_frames = 0, intra_frames = 0;
    CgTotals cg;
    std::string timeline;  // HIVC_TIMELINE rows: kind,stream,gop,frame,t0_us,t1_us (from the decode origin)
};

struct EvRec {
    cudaEvent_t first = nullptr, second = nullptr;
    int stream = 0, gop = 0, frame = 0;
};
using EvPairs = std::vector<EvRec>;

double drain(EvPairs& v, cudaEvent_t origin, char kind, std::string* timeline) {
    double t = 0;
    for (auto& e : v) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e.first, e.second);
        t += ms * 1e-3;
        if (timeline) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, origin, e.first);
            cudaEventElapsedTime(&b, origin, e.second);
            char line[128];
            std::snprintf(line, sizeof line, "%c,%d,%d,%d,%.1f,%.1f\n", kind, e.stream, e.gop, e.frame, a * 1e3, b * 1e3);
            *timeline += line;
        }
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    v.clear();
    return t;
}

void decode_gop(Context& ctx, Lane& L, const StreamJob& S, int gi, bool out_on_device, bool timed, LaneResult& R,
                std::vector<FrameJob>& jobs, std::vector<uint64_t>& bits, int& slot, EvPairs& ev_intra,
                EvPairs& ev_inter, EvPairs& ev_ifin) {
    const StreamHeader& hd = S.hd;
    const int h = hd.height, w = hd.width, C = hd.channels;
    const size_t N = (size_t)h * w;
    const size_t frame_bytes = N * C;
    GopCursor cur(S.data + S.gops[gi].first, S.gops[gi].second, hd, gi);
    const int nf = cur.nframes;
    if ((int)jobs.size() < nf) jobs.resize(nf);
    cudaStream_t s = L.stream;
    uint8_t* gop_dev = out_on_device ? S.out + S.frame_base[gi] * frame_bytes : L.gop_out[slot];
    uint8_t* gop_host = out_on_device ? nullptr : S.out + S.frame_base[gi] * frame_bytes;
    if (!out_on_device) CUDA_CHECK(cudaStreamWaitEvent(s, L.out_free[slot], 0));  // copies out of this slot done
    // Parse and ship in chunks: the I-frame alone, so its solve runs while the
    // host parses the P frames, then kChunk P frames at a time.
    constexpr int kChunk = 2;
    FrameOffsets offs[kChunk];
    size_t fi = 0;
    while ((int)fi < nf) {
        const int cnt = fi == 0 ? 1 : std::min(kChunk, nf - (int)fi);
        for (int k = 0; k < cnt; ++k) cur.parse(jobs[fi + k], R.ht, bits);
        if ((int)fi + cnt == nf) cur.finish();
        // pack the compact frame descriptions: measure, then write into pinned staging
        Packer pk;
        for (int k = 0; k < cnt; ++k) pack_frame(pk, jobs[fi + k], offs[k]);
        const int b = L.stage_next++ % Lane::kStage;
        if (L.staged[b]) CUDA_CHECK(cudaEventSynchronize(L.staged[b]));
        L.reserve_stage(b, pk.off + 16);
        pk.base = L.host_stage[b];
        pk.off = 0;
        pk.measure = false;
        for (int k = 0; k < cnt; ++k) pack_frame(pk, jobs[fi + k], offs[k]);
        CUDA_CHECK(cudaMemcpyAsync(L.dev_stage[b], L.host_stage[b], pk.off, cudaMemcpyHostToDevice, s));
        R.h2d += (int64_t)pk.off;
        if (!L.staged[b]) CUDA_CHECK(cudaEventCreateWithFlags(&L.staged[b], cudaEventDisableTiming));
        CUDA_CHECK(cudaEventRecord(L.staged[b], s));
        const uint8_t* dev = L.dev_stage[b];
        for (int k = 0; k < cnt; ++k, ++fi) {
            const FrameJob& J = jobs[fi];
            const FrameOffsets& o = offs[k];
            FrameArgs A;
            A.h = h;
            A.w = w;
            A.channels = C;
            uint8_t* fr = gop_dev + fi * frame_bytes;
            uint8_t* frprev = fi ? gop_dev + (fi - 1) * frame_bytes : nullptr;
            for (int c = 0; c < C; ++c) {
                if (C == 1) {
                    A.recon[c] = fr;  // gray: the reconstruction IS the output frame
                    A.prev[c] = frprev;
                } else {
                    A.recon[c] = L.ring[fi & 1][c];
                    A.prev[c] = L.ring[(fi + 1) & 1][c];
                    A.rgb[c] = fr + c * N;
                }
            }
            ResDev& RD = A.res;
            RD.ngroups = J.res.zero ? 0 : J.res.ngroups;
            RD.dz_step = 127.0 / (double)((hd.residual_levels - 1) / 2);  // quantize.py:43-47
            RD.c_scale = J.res.c_scale;
            RD.a_scale = J.res.a_scale;
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
            EvRec e;
            e.stream = R.stream;
            e.gop = gi;
            e.frame = (int)fi;
            auto ev_begin = [&]() {
                if (!timed) return;
                CUDA_CHECK(cudaEventCreate(&e.first));
                CUDA_CHECK(cudaEventCreate(&e.second));
                CUDA_CHECK(cudaEventRecord(e.first, s));
            };
            auto ev_end = [&](EvPairs& v) {
                if (!timed) return;
                CUDA_CHECK(cudaEventRecord(e.second, s));
                v.push_back(e);
            };
            ev_begin();
            (J.type == 0 ? R.intra_frames : R.inter_frames) += 1;
            if (J.type == 0) {
                // intra: f = 0 with the values scattered at the mask points, then solve (prediction.py:203-208)
                int64_t launches = 0;
                for (int c = 0; c < C; ++c) {
                    int t = c == 0 ? 0 : 1;
                    const auto& pts = J.intra.pts[t];
                    CUDA_CHECK(cudaMemsetAsync(L.f[c], 0, N * sizeof(double), s));
                    if (c <= 1) CUDA_CHECK(cudaMemsetAsync(L.m[t], 0, N, s));
                    launch_scatter(at<int32_t>(dev, o.pts[t]), at<double>(dev, o.vals[c]), (int)pts.size(), L.f[c],
                                   c <= 1 ? L.m[t] : nullptr, s);
                    ++launches;
                    solve_homogeneous_async(L.ws, s, L.f[c], L.m[t], h, w, 1e-4, 160, L.u[c], &launches,
                                            timed ? &L.probe : nullptr);
                    A.u[c] = L.u[c];
                }
                ctx.launches += launches;
                ev_end(ev_intra);
                ev_begin();
                launch_frame(A, false, s);
                ctx.launches += 1;
                ev_end(ev_ifin);
            } else {
                for (int c = 0; c < 2; ++c) {
                    A.flow.nodes[c] = at<int32_t>(dev, o.nodes[c]);
                    A.flow.vals[c] = at<double>(dev, o.fvals[c]);
                    A.flow.tiles[c] = at<uint16_t>(dev, o.ftiles[c]);
                }
                launch_frame(A, true, s);
                ctx.launches += 1;
                ev_end(ev_inter);
            }
            if (!out_on_device) {  // frame fi is final: copy it out while fi+1 decodes
                cudaEvent_t fe = L.frame_ev[L.frame_ev_next++ % Lane::kFrameEv];
                CUDA_CHECK(cudaEventRecord(fe, s));
                CUDA_CHECK(cudaStreamWaitEvent(L.copy, fe, 0));
                CUDA_CHECK(cudaMemcpyAsync(gop_host + fi * frame_bytes, fr, frame_bytes, cudaMemcpyDeviceToHost, L.copy));
                R.d2h += (int64_t)frame_bytes;
            }
        }
    }
    if (!out_on_device) CUDA_CHECK(cudaEventRecord(L.out_free[slot], L.copy));
    slot ^= 1;
}

void run_lane(Context& ctx, Lane& L, const std::vector<StreamJob>& streams, const std::vector<WorkItem>& items,
              std::atomic<size_t>& next_item, bool out_on_device, bool timed, cudaEvent_t origin, cudaEvent_t done,
              LaneResult& R) {
    std::vector<FrameJob> jobs;
    std::vector<uint64_t> bits;
    EvPairs ev_intra, ev_inter, ev_ifin;
    int slot = 0;
    try {
        CUDA_CHECK(cudaSetDevice(L.device));
        CUDA_CHECK(cudaStreamWaitEvent(L.stream, origin, 0));
        bool any = false;
        for (size_t i; (i = next_item.fetch_add(1)) < items.size();) {  // largest planes first, first free lane
            const WorkItem& it = items[i];
            any = true;
            R.stream = it.stream;
            R.gop = it.gop;
            decode_gop(ctx, L, streams[it.stream], it.gop, out_on_device, timed, R, jobs, bits, slot, ev_intra,
                       ev_inter, ev_ifin);
        }
        if (!out_on_device && any)  // the span ends with the last D2H copy
            CUDA_CHECK(cudaStreamWaitEvent(L.stream, L.out_free[slot ^ 1], 0));
        CUDA_CHECK(cudaEventRecord(done, L.stream));
        CUDA_CHECK(cudaStreamSynchronize(L.stream));
        std::string* tl = std::getenv("HIVC_TIMELINE") ? &R.timeline : nullptr;
        R.gpu_intra = drain(ev_intra, origin, 'I', tl);
        R.gpu_inter = drain(ev_inter, origin, 'P', tl);
        R.gpu_ifinal = drain(ev_ifin, origin, 'F', tl);
        L.probe.harvest(R.cg);
    } catch (const Error& e) {
        R.code = e.code;
        R.msg = e.what();
        cudaEventRecord(done, L.stream);
        cudaStreamSynchronize(L.stream);
        if (L.copy) cudaStreamSynchronize(L.copy);
    } catch (const std::exception& e) {
        R.code = HIVC_E_ARGUMENT;
        R.msg = e.what();
        cudaEventRecord(done, L.stream);
        cudaStreamSynchronize(L.stream);
        if (L.copy) cudaStreamSynchronize(L.copy);
    }
}

}  // namespace

void decode_streams(Context& ctx, int nstreams, const uint8_t* const* data, const size_t* len, const int* gop_begin,
                    const int* gop_end, uint8_t* const* out, bool out_on_device, double* stage_seconds) {
    double t_all = now_s();
    std::vector<StreamJob> streams(nstreams);
    std::vector<WorkItem> items;
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
            uint16_t nf = 0;
            if (S.gops[g].second >= 2) std::memcpy(&nf, S.data + S.gops[g].first, 2);
            acc += nf;
            max_gop_bytes = std::max(max_gop_bytes, nf * frame_bytes);
            items.push_back({k, g});
        }
        max_h = std::max(max_h, S.hd.height);
        max_w = std::max(max_w, S.hd.width);
        max_c = std::max(max_c, S.hd.channels);
    }
    // largest planes first so lanes finish together
    std::stable_sort(items.begin(), items.end(), [&](const WorkItem& a, const WorkItem& b) {
        const StreamHeader &ha = streams[a.stream].hd, &hb = streams[b.stream].hd;
        return (int64_t)ha.height * ha.width * ha.channels > (int64_t)hb.height * hb.width * hb.channels;
    });
    static const int kMaxLanes = [] {
        const char* e = std::getenv("HIVC_LANES");
        return e ? std::max(1, std::min(32, std::atoi(e))) : 8;
    }();
    int nlanes = std::max(1, std::min((int)items.size(), kMaxLanes));
    CUDA_CHECK(cudaSetDevice(ctx.device));
    while ((int)ctx.lanes.size() < nlanes) {
        auto L = std::make_unique<Lane>();
        L->device = ctx.device;
        CUDA_CHECK(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking));
        ctx.lanes.push_back(std::move(L));
    }
    for (int l = 0; l < nlanes; ++l) {
        Lane& L = *ctx.lanes[l];
        L.reserve_planes(max_h, max_w, max_c);
        L.ws.reserve(max_h, max_w, ctx.device);
        L.ws.pack_bands = true;  // lanes solve side by side: throughput mode
        if (!out_on_device) L.reserve_gop_out(max_gop_bytes);
        // staging sized up front (an I-frame of a typical mask fits), so a lane
        // meeting its first large chunk does not reallocate (cudaFree syncs the device)
        for (int b = 0; b < Lane::kStage; ++b) L.reserve_stage(b, (size_t)2 * max_h * max_w * max_c + 65536);
    }
    std::atomic<size_t> next_item{0};
    std::vector<LaneResult> res(nlanes);
    const bool timed = (stage_seconds != nullptr && ctx.stage_events) || std::getenv("HIVC_TIMELINE");
    // device-side span: every lane waits on `origin`, records `done[l]` after its last copy
    cudaEvent_t origin;
    CUDA_CHECK(cudaEventCreate(&origin));
    std::vector<cudaEvent_t> done(nlanes);
    for (auto& e : done) CUDA_CHECK(cudaEventCreate(&e));
    CUDA_CHECK(cudaEventRecord(origin, ctx.stream));
    if (nlanes == 1) {
        run_lane(ctx, *ctx.lanes[0], streams, items, next_item, out_on_device, timed, origin, done[0], res[0]);
    } else {
        std::vector<std::thread> th;
        for (int l = 0; l < nlanes; ++l)
            th.emplace_back(run_lane, std::ref(ctx), std::ref(*ctx.lanes[l]), std::cref(streams), std::cref(items),
                            std::ref(next_item), out_on_device, timed, origin, done[l], std::ref(res[l]));
        for (auto& t : th) t.join();
    }
    double span = 0;
    for (auto& e : done) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, origin, e) == cudaSuccess) span = std::max(span, (double)ms * 1e-3);
        cudaEventDestroy(e);
    }
    cudaEventDestroy(origin);
    // the first failing (stream, GOP) in stream order wins (the reference decodes sequentially)
    int worst = -1;
    for (int l = 0; l < nlanes; ++l)
        if (res[l].code != HIVC_OK &&
            (worst < 0 || std::make_pair(res[l].stream, res[l].gop) < std::make_pair(res[worst].stream, res[worst].gop)))
            worst = l;
    if (worst >= 0) fail(res[worst].code, res[worst].msg);
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
    if (const char* tl = std::getenv("HIVC_TIMELINE")) {  // debug: append lane,kind,stream,gop,frame,t0,t1
        if (FILE* f = std::fopen(tl, "a")) {
            for (int l = 0; l < nlanes; ++l) {
                size_t a = 0;
                const std::string& t = res[l].timeline;
                while (a < t.size()) {
                    size_t b = t.find('\n', a);
                    std::fprintf(f, "%d,%s\n", l, t.substr(a, b - a).c_str());
                    a = b + 1;
                }
            }
            std::fprintf(f, "-\n");
            std::fclose(f);
        }
    }
    for (auto& r : res) {
        ctx.h2d_bytes += r.h2d;
        ctx.d2h_bytes += r.d2h;
        std::lock_guard<std::mutex> g(ctx.stats_mu);
        CgTotals& T = ctx.cg;
        T.solves += r.cg.solves;
        T.pixel_iters += r.cg.pixel_iters;
        T.pixel_levels += r.cg.pixel_levels;
        T.grid_launches += r.cg.grid_launches;
        T.grid_seconds += r.cg.grid_seconds;
        T.grid_pixel_iters += r.cg.grid_pixel_iters;
        T.grid_pixels += r.cg.grid_pixels;
        ctx.inter_frames += r.inter_frames;
        ctx.inter_seconds += r.gpu_inter;
        ctx.intra_frames += r.intra_frames;
    }
    if (stage_seconds) {
        double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (auto& r : res) {
            s[0] += r.ht.intra_parse + r.gpu_intra;
            s[1] += r.ht.flow_parse;
            s[2] += r.gpu_inter;
            s[3] += r.ht.residual_parse;
            s[4] += r.gpu_ifinal;
        }
        s[6] = now_s() - t_all;
        s[7] = span;
        std::memcpy(stage_seconds, s, sizeof(s));
    }
}

}  // namespace hivc
