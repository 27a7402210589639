// Stream decoder: GOP-parallel host parsing feeding per-lane CUDA streams.
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

// One decode lane: a CUDA stream, a solver workspace and double-buffered
// staging (pinned host + device) for the compact frame descriptions.
struct Lane {
    int device = 0;
    cudaStream_t stream = nullptr;
    InpaintWorkspace ws;
    size_t plane_px = 0;
    int chans = 0;
    double* f[3] = {nullptr, nullptr, nullptr};
    uint8_t* m[2] = {nullptr, nullptr};
    double* u[3] = {nullptr, nullptr, nullptr};
    int16_t* ring[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    // ring of pinned staging buffers: one per shipped chunk of frame descriptions
    static constexpr int kStage = 4;
    uint8_t* host_stage[kStage] = {};
    uint8_t* dev_stage[kStage] = {};
    size_t stage_cap[kStage] = {};
    cudaEvent_t staged[kStage] = {};
    int stage_next = 0;
    uint8_t* gop_out[2] = {nullptr, nullptr};  // device frame buffers when output goes to the host
    size_t gop_out_cap = 0;
    // host output: each finished frame is copied D2H on `copy` while the lane
    // stream decodes the next one; out_free[slot] = last copy out of gop_out[slot]
    cudaStream_t copy = nullptr;
    static constexpr int kFrameEv = 8;
    cudaEvent_t frame_ev[kFrameEv] = {};
    cudaEvent_t out_free[2] = {nullptr, nullptr};
    int frame_ev_next = 0;
    CgProbe probe;
    void reserve_planes(int h, int w, int channels);
    void reserve_stage(int slot, size_t bytes);
    void reserve_gop_out(size_t bytes);
    ~Lane();
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;  // function-level API stream
    InpaintWorkspace ws;            // function-level solver scratch
    BroxWorkspace brox;             // flow_brox scratch
    std::vector<std::unique_ptr<Lane>> lanes;
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

// Decode GOP ranges of several streams in one pass (one lane per host thread,
// work items = (stream, GOP)).  stage_seconds (nullable, 8 doubles): the 7
// reference timing keys + the device-side span (first lane start -> last lane end).
void decode_streams(Context& ctx, int nstreams, const uint8_t* const* data, const size_t* len, const int* gop_begin,
                    const int* gop_end, uint8_t* const* out, bool out_on_device, double* stage_seconds);

// Host-only parse of every frame record (8 int64 per frame, see decode.cu).
void parse_stream_stats(const uint8_t* data, size_t len, std::vector<int64_t>& stats, double* seconds);

// Frames per GOP (u16 at the head of each GOP payload, codec.py:494).
void gop_frame_counts(const uint8_t* data, size_t len, std::vector<int32_t>& counts);

}  // namespace hivc
