// Stream decoder: GOP-parallel host parsing, batched I-frame solves, per-GOP P-frame streams.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <memory>
#include <mutex>
#include <vector>

#include "brox.h"
#include "inpaint.h"
#include "parse.h"
#include "recon.h"

namespace hivc {

// Parsed description of one frame record (host side).
struct FrameJob {
    int type = 0;  // 0 intra, 1 inter
    IntraJob intra;
    FlowJob flow;
    ResidualJob res;
};

// Device state of one work item (one GOP of one stream) of a decode call;
// a call uses slots [0, items).  The slot's stream carries the item's
// uploads, the I-frame scatter and the P-frame chain; its I-frame solve runs
// batched with the other items' on the context's solver stream.
struct Slot {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr;  // host output: D2H of finished frames
    cudaStream_t up = nullptr;    // H2D of frame descriptions (never queued behind the solves)
    static constexpr int kUpEv = 16;
    cudaEvent_t up_ev[kUpEv] = {};
    int up_next = 0;
    InpaintWorkspace ws;
    size_t plane_px = 0;
    int chans = 0;
    double* f[3] = {nullptr, nullptr, nullptr};
    uint8_t* m[2] = {nullptr, nullptr};
    double* u[3] = {nullptr, nullptr, nullptr};
    int16_t* ring[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    // staging arena (pinned host block + device block): every chunk of frame
    // descriptions of a call gets its own range, so a worker never waits for
    // the GPU to free a buffer; a call that outgrows the block chains a new
    // one and the next call starts with one block of the combined size
    struct StageBlock {
        uint8_t* host = nullptr;
        uint8_t* dev = nullptr;
        size_t cap = 0;
    };
    std::vector<StageBlock> stage;
    size_t stage_off = 0, stage_used = 0;
    void stage_begin_call(size_t min_bytes);
    void stage_alloc(size_t bytes, uint8_t*& host, uint8_t*& dev);
    uint8_t* gop_out = nullptr;  // host-output mode: the GOP's frames on the device
    size_t gop_out_cap = 0;
    static constexpr int kFrameEv = 8;
    cudaEvent_t frame_ev[kFrameEv] = {};
    int frame_ev_next = 0;
    cudaEvent_t out_free = nullptr;     // last D2H out of gop_out
    cudaEvent_t intra_ready = nullptr;  // I-frame f / mask planes in place (slot stream)
    cudaEvent_t intra_done = nullptr;   // I-frame solved and finalised (solver stream)
    // host scratch kept across calls (capacity reuse: no page faults per call)
    std::vector<FrameJob> jobs;
    std::vector<uint64_t> bits;
    void init(int dev);
    void reserve_planes(int h, int w, int channels);
    void reserve_gop_out(size_t bytes);
    ~Slot();
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;  // function-level API stream
    InpaintWorkspace ws;            // function-level solver scratch
    BroxWorkspace brox;             // flow_brox scratch
    std::vector<std::unique_ptr<Slot>> slots;
    cudaStream_t solver = nullptr;  // every batched (grid-barrier) solve of a decode call, in order
    static constexpr int kPre = 4;
    cudaStream_t pre[kPre] = {};  // pyramid + cluster levels of a batch (side streams, round robin)
    int pre_next = 0;             // (under solver_mu)
    std::mutex solver_mu;           // one batch's launches stay contiguous on the solver stream
    CgProbe probe;                  // solver-stream launches (stage timing on)
    std::atomic<int64_t> launches{0};
    std::atomic<int64_t> h2d_bytes{0}, d2h_bytes{0};
    bool stage_events = true;  // per-frame CUDA events for the stage breakdown
    std::mutex stats_mu;
    CgTotals cg;               // accumulated over timed decodes
    int64_t inter_frames = 0, intra_frames = 0;
    double inter_seconds = 0;  // device time of the fused P-frame kernels
    int* d_status = nullptr;
    float* op_hi = nullptr;  // shared-layout block operator (tf32 head, then tail), config 2a
    uint64_t op_mask = 0;
    ~Context();
};

// Decode GOP ranges of several streams in one pass (work items = (stream,
// GOP), parsed by a pool of host threads; I-frame solves batched per shape).  stage_seconds (nullable, 8 doubles): the 7
// reference timing keys + the device-side span (first lane start -> last lane end).
void decode_streams(Context& ctx, int nstreams, const uint8_t* const* data, const size_t* len, const int* gop_begin,
                    const int* gop_end, uint8_t* const* out, int out_mode, double* stage_seconds);

// Host-only parse of every frame record (8 int64 per frame, see decode.cu).
void parse_stream_stats(const uint8_t* data, size_t len, std::vector<int64_t>& stats, double* seconds);

// Frames per GOP (u16 at the head of each GOP payload, codec.py:494).
void gop_frame_counts(const uint8_t* data, size_t len, std::vector<int32_t>& counts);

}  // namespace hivc
