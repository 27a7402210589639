// extern "C" entry points declared in include/hivc_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "blockgemm.h"
#include "brox.h"
#include "decode.h"
#include "inpaint.h"
#include "parse.h"
#include "recon.h"

struct hivc_ctx {
    hivc::Context c;
};

namespace hivc {
static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace hivc

using hivc::guarded;

extern "C" {

const char* hivc_last_error(void) { return hivc::g_last_error.c_str(); }

const char* hivc_version(void) {
    return "hivc_b200 1.0 (sm_100a, float64 replay of the reference decoder, -fmad=false)";
}

int hivc_ctx_create(int device, hivc_ctx** out) {
    return guarded([&] {
        if (!out) hivc::fail(HIVC_E_ARGUMENT, "null out pointer");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0)
            hivc::fail(HIVC_E_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
        if (device < 0 || device >= n) hivc::fail(HIVC_E_ARGUMENT, "bad device index");
        CUDA_CHECK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            hivc::fail(HIVC_E_CUDA, "this library is built for sm_100a (B200); device is sm_" +
                                        std::to_string(prop.major) + std::to_string(prop.minor));
        auto* c = new hivc_ctx();
        c->c.device = device;
        CUDA_CHECK(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
        CUDA_CHECK(cudaMalloc(&c->c.d_status, 64 * sizeof(int)));
        *out = c;
    });
}

int hivc_ctx_destroy(hivc_ctx* ctx) {
    return guarded([&] { delete ctx; });
}

void* hivc_ctx_stream(hivc_ctx* ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }

int hivc_ctx_synchronize(hivc_ctx* ctx) {
    return guarded([&] {
        CUDA_CHECK(cudaSetDevice(ctx->c.device));
        CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
    });
}

int64_t hivc_ctx_launch_count(hivc_ctx* ctx) { return ctx ? ctx->c.launches.load() : 0; }

int hivc_parse_header(const uint8_t* data, size_t len, hivc_stream_info* info) {
    return guarded([&] {
        hivc::StreamHeader h = hivc::parse_header(data, len);
        std::vector<std::pair<size_t, size_t>> gops;
        hivc::split_gops(data, len, h, gops);
        info->width = h.width;
        info->height = h.height;
        info->frame_count = h.frame_count;
        info->fps_num = h.fps_num;
        info->fps_den = h.fps_den;
        info->gop_size = h.gop_size;
        info->channels = h.channels;
        info->intra_levels = h.intra_levels;
        info->flow_levels = h.flow_levels;
        info->residual_levels = h.residual_levels;
        info->gop_count = (int32_t)gops.size();
    });
}

int hivc_gop_frame_counts(const uint8_t* data, size_t len, int32_t* counts, int32_t cap, int32_t* ngops) {
    return guarded([&] {
        std::vector<int32_t> c;
        hivc::gop_frame_counts(data, len, c);
        *ngops = (int32_t)c.size();
        for (int32_t i = 0; i < cap && i < (int32_t)c.size(); ++i) counts[i] = c[i];
    });
}

int hivc_parse_stream(const uint8_t* data, size_t len, int64_t* stats, int64_t cap, int64_t* nframes,
                      double* seconds) {
    return guarded([&] {
        std::vector<int64_t> s;
        hivc::parse_stream_stats(data, len, s, seconds);
        *nframes = (int64_t)(s.size() / 8);
        for (int64_t i = 0; i < cap && i < (int64_t)s.size(); ++i) stats[i] = s[i];
    });
}

static int parse_sym_common(bool signed_vals, const uint8_t* data, size_t len, size_t pos, int64_t* out, size_t cap,
                            size_t* count, size_t* next_pos) {
    return guarded([&] {
        std::vector<int32_t> v;
        size_t np = signed_vals ? hivc::decode_signed_values(data, len, pos, v) : hivc::decode_symbols(data, len, pos, v);
        *count = v.size();
        if (next_pos) *next_pos = np;
        for (size_t i = 0; i < cap && i < v.size(); ++i) out[i] = v[i];
    });
}

int hivc_parse_symbols(const uint8_t* data, size_t len, size_t pos, int64_t* out, size_t cap, size_t* count,
                       size_t* next_pos) {
    return parse_sym_common(false, data, len, pos, out, cap, count, next_pos);
}

int hivc_parse_signed_values(const uint8_t* data, size_t len, size_t pos, int64_t* out, size_t cap, size_t* count,
                             size_t* next_pos) {
    return parse_sym_common(true, data, len, pos, out, cap, count, next_pos);
}

int hivc_parse_tree(const uint8_t* data, size_t nbytes, uint64_t nbits, uint64_t bit_offset, int32_t width,
                    int32_t height, int32_t* rects, size_t cap, size_t* nleaves, uint64_t* bits_used) {
    return guarded([&] {
        hivc::BitReader rd(data, nbytes, nbits);
        rd.seek(bit_offset);
        std::vector<hivc::Rect> leaves;
        hivc::parse_tree_leaves(rd, width, height, leaves);
        *nleaves = leaves.size();
        if (bits_used) *bits_used = rd.pos - bit_offset;
        for (size_t i = 0; i < cap && i < leaves.size(); ++i) {
            rects[4 * i] = leaves[i].x;
            rects[4 * i + 1] = leaves[i].y;
            rects[4 * i + 2] = leaves[i].w;
            rects[4 * i + 3] = leaves[i].h;
        }
    });
}

int hivc_homog_solve(hivc_ctx* ctx, const double* f, const uint8_t* mask, int32_t h, int32_t w, double tol,
                     int32_t max_iter, int32_t strict, double* u, int32_t* level_sizes, int32_t* level_iters,
                     int32_t* nlevels) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        if (h < 1 || w < 1) hivc::fail(HIVC_E_INPAINTING, "plane/mask shape mismatch");
        if (strict && !(tol > 0)) hivc::fail(HIVC_E_INPAINTING, "tol must be positive");
        if (max_iter < 0) max_iter = 0;
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        // empty-mask check (homogeneous.py:177-178)
        {
            size_t n = (size_t)h * w;
            // reuse the workspace byte buffer? keep it simple: reduce on host copy of the mask
            std::vector<uint8_t> hm(n);
            CUDA_CHECK(cudaMemcpyAsync(hm.data(), mask, n, cudaMemcpyDeviceToHost, C.stream));
            CUDA_CHECK(cudaStreamSynchronize(C.stream));
            bool any = false;
            for (uint8_t b : hm)
                if (b) {
                    any = true;
                    break;
                }
            if (!any) hivc::fail(HIVC_E_INPAINTING, "empty inpainting mask");
        }
        C.ws.reserve(h, w, C.device);
        int64_t launches = 0;
        int L = hivc::solve_homogeneous_async(C.ws, C.stream, f, mask, h, w, tol, max_iter, u, &launches);
        std::vector<std::pair<int, int>> shapes;
        hivc::pyramid_shapes(h, w, shapes);
        std::vector<int> it(L);
        CUDA_CHECK(cudaMemcpyAsync(it.data(), C.ws.iters, L * sizeof(int), cudaMemcpyDeviceToHost, C.stream));
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
        if ((hivc::debug_opt("cg_trace") || hivc::debug_opt("cg_trace_cluster")) && C.ws.trace) {
            // phase timing of the finest level (CTA 0, thread 0): mean ns per phase
            std::vector<unsigned long long> tr(hivc::kTraceLen);
            CUDA_CHECK(cudaMemcpy(tr.data(), C.ws.trace, tr.size() * 8, cudaMemcpyDeviceToHost));
            {  // arrival spread at the first reduction: max - min arrival, release - last arrival
                double spread = 0, rel = 0;
                int nk = 0;
                for (int k = 2; k < 255 && tr[(k + 1) * 8] != 0; ++k) {
                    unsigned long long lo = ~0ull, hi = 0;
                    for (int b = 0; b < 160; ++b) {
                        unsigned long long t = tr[2048 + k * 160 + b];
                        if (!t) continue;
                        lo = std::min(lo, t);
                        hi = std::max(hi, t);
                    }
                    if (!hi) continue;
                    spread += (double)(hi - lo);
                    rel += (double)tr[k * 8 + 3] - (double)hi;
                    ++nk;
                }
                if (nk) fprintf(stderr, "[cg trace] arrival spread %.0f ns | last arrival -> CTA0 released+summed %.0f ns\n",
                                spread / nk, rel / nk);
            }
            double acc[6] = {0, 0, 0, 0, 0, 0}, acc6 = 0, acc7 = 0;
            int n = 0;
            for (int k = 2; k < 255 && tr[(k + 1) * 8] != 0; ++k, ++n) {
                const unsigned long long* t = &tr[k * 8];
                acc[0] += (double)(t[1] - t[0]);
                acc[1] += (double)(t[2] - t[1]);
                acc[2] += (double)(t[3] - t[2]);
                acc[3] += (double)(t[4] - t[3]);
                acc[4] += (double)(t[5] - t[4]);
                acc[5] += (double)(tr[(k + 1) * 8] - t[5]);
                if (t[6]) acc6 += (double)(t[6] - t[4]);
                if (t[7]) acc7 += (double)(t[7] - t[0]);
            }
            if (n)
                fprintf(stderr,
                        "[cg trace] %d iters: halo+p %.0f ns | stencil %.0f | reduce1 %.0f | phase2 %.0f | reduce2 %.0f "
                        "(arrive + x update %.0f) | tail %.0f | halo loads+stores %.0f\n",
                        n, acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n, acc[4] / n, acc6 / n, acc[5] / n, acc7 / n);
        }
        if (nlevels) *nlevels = L;
        for (int i = 0; i < L && i < 32; ++i) {
            auto s = shapes[L - 1 - i];
            if (level_sizes) level_sizes[i] = s.first * s.second;
            if (level_iters) level_iters[i] = it[i];
        }
        if (strict) {
            double rel = hivc::strict_relative_residual(C.ws, C.stream, u, f, mask, h, w, &launches);
            if (rel >= 0 && rel > tol) {
                char buf[128];
                snprintf(buf, sizeof(buf), "relative residual %.3e > tol %.3e", rel, tol);
                C.launches += launches;
                hivc::fail(HIVC_E_CONVERGENCE, buf);
            }
        }
        C.launches += launches;
    });
}

int hivc_poisson_interior(hivc_ctx* ctx, const double* w_full, const uint8_t* mask, int32_t h, int32_t w,
                          double tol, int32_t max_iter, double* z, int32_t* iters) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        if (h < 1 || w < 1) hivc::fail(HIVC_E_INPAINTING, "plane/mask shape mismatch");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        C.ws.reserve(h, w, C.device);
        int64_t launches = 0;
        int it = hivc::solve_poisson_interior(C.ws, C.stream, w_full, mask, h, w, tol, max_iter, z, &launches);
        C.launches += launches;
        if (iters) *iters = it;
    });
}

int hivc_mask_adjoint(hivc_ctx* ctx, const double* w_full, const double* z, const int32_t* pts, int32_t npts,
                      int32_t h, int32_t w, double* out) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        hivc::launch_mask_adjoint(w_full, z, pts, npts, h, w, out, C.stream);
        C.launches += 1;
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
    });
}

int hivc_flow_component(hivc_ctx* ctx, const uint8_t* data, size_t len, size_t pos, int32_t h, int32_t w,
                        int32_t levels, double* out, size_t* next_pos) {
    return guarded([&] {
        if (h < 1 || w < 1 || levels < 2) hivc::fail(HIVC_E_ARGUMENT, "bad flow plane shape or levels");
        std::vector<hivc::Rect> leaves;
        std::vector<double> vals;
        const size_t next = hivc::parse_flow_component(data, len, pos, h, w, levels, leaves, vals);
        static_assert(sizeof(hivc::Rect) == 16, "Rect is four int32");
        if (!ctx) {  // host plane
            for (size_t i = 0; i < leaves.size(); ++i) {
                const hivc::Rect& r = leaves[i];
                for (int32_t y = r.y; y < r.y + r.h; ++y) std::fill_n(out + (size_t)y * w + r.x, r.w, vals[i]);
            }
        } else {  // device plane: one upload, one launch
            hivc::Context& C = ctx->c;
            CUDA_CHECK(cudaSetDevice(C.device));
            const size_t n = leaves.size(), rb = n * sizeof(hivc::Rect);
            void* tmp = nullptr;
            CUDA_CHECK(cudaMallocAsync(&tmp, rb + n * sizeof(double), C.stream));
            CUDA_CHECK(cudaMemcpyAsync(tmp, leaves.data(), rb, cudaMemcpyHostToDevice, C.stream));
            CUDA_CHECK(cudaMemcpyAsync((char*)tmp + rb, vals.data(), n * sizeof(double), cudaMemcpyHostToDevice,
                                       C.stream));
            hivc::launch_paint_leaves((const int32_t*)tmp, (const double*)((char*)tmp + rb), (int)n, w, out, C.stream);
            C.launches += 1;
            CUDA_CHECK(cudaFreeAsync(tmp, C.stream));
            CUDA_CHECK(cudaStreamSynchronize(C.stream));
        }
        if (next_pos) *next_pos = next;
    });
}

int hivc_warp(hivc_ctx* ctx, const double* const* src, int32_t nplanes, const double* u, const double* v, int32_t h,
              int32_t w, double* const* dst) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        hivc::launch_warp(src, nplanes, u, v, h, w, dst, C.stream);
        C.launches += (nplanes + 7) / 8;
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
    });
}

int hivc_block_reconstruct(hivc_ctx* ctx, const double* mc, const double* a, const double* eig, int32_t n,
                           double* out) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        hivc::launch_block_reconstruct(mc, a, eig, n, out, C.stream);
        C.launches += n > 0;
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
    });
}

int hivc_block_fit(hivc_ctx* ctx, const double* f_blocks, const uint64_t* masks, int32_t n, double* c_out,
                   double* a_out) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        CUDA_CHECK(cudaMemsetAsync(C.d_status, 0, sizeof(int), C.stream));
        hivc::launch_block_fit(f_blocks, masks, n, c_out, a_out, C.d_status, C.stream);
        C.launches += n > 0;
        int st = 0;
        CUDA_CHECK(cudaMemcpyAsync(&st, C.d_status, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
        if (st == 1) hivc::fail(HIVC_E_PSEUDODIFF, "block mask needs at least one point");
        if (st == 2) hivc::fail(HIVC_E_PSEUDODIFF, "singular coefficient system");
    });
}

int hivc_residual_keep(hivc_ctx* ctx, int32_t npl, const double* const* c, const double* const* a,
                       const double* const* fb, const uint64_t* words, int32_t n, int32_t levels,
                       int32_t bits_per_sym, double c_scale, double a_scale, double lam, int32_t* const* q,
                       int32_t* const* qa, double* const* rec, uint8_t* keep) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        if (npl < 1 || npl > 2) hivc::fail(HIVC_E_ARGUMENT, "a residual channel group has 1 or 2 planes");
        if (levels < 3 || levels % 2 == 0) hivc::fail(HIVC_E_QUANTIZE, "dead-zone levels must be odd and >= 3");
        if (!(c_scale > 0) || !(a_scale > 0)) hivc::fail(HIVC_E_QUANTIZE, "global_scale must be positive");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        hivc::KeepArgs A{};
        for (int i = 0; i < npl; ++i) {
            A.c[i] = c[i];
            A.a[i] = a[i];
            A.fb[i] = fb[i];
            A.q[i] = q[i];
            A.qa[i] = qa[i];
            A.rec[i] = rec[i];
        }
        A.words = words;
        A.n = n;
        A.npl = npl;
        A.lmax = (levels - 1) / 2;
        A.bits_per_sym = bits_per_sym;
        A.c_scale = c_scale;
        A.a_scale = a_scale;
        A.step = 127.0 / (double)((levels - 1) / 2);  // quantize.deadzone_step
        A.lam = lam;
        A.keep = keep;
        hivc::launch_residual_keep(A, C.stream);
        C.launches += n > 0;
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
    });
}

int hivc_block_operator(hivc_ctx* ctx, const float* plane, int32_t h, int32_t w, uint64_t mask, float* out) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        if (C.op_mask != mask || !C.op_hi) {
            std::vector<double> R;
            hivc::shared_block_operator(mask, R);
            std::vector<float> hi(64 * 64), lo(64 * 64);
            for (int i = 0; i < 64 * 64; ++i) {
                float f = (float)R[i];
                uint32_t u;
                std::memcpy(&u, &f, 4);
                u &= 0xFFFFE000u;  // tf32 head
                float fh;
                std::memcpy(&fh, &u, 4);
                hi[i] = fh;
                lo[i] = (float)(R[i] - (double)fh);
            }
            // row-major hi, lo; then both again in the canonical K-major UMMA layout
            // (core matrix (n/8, k/4) at 128 B, rows 16 B apart) for a single bulk copy
            std::vector<float> kl(2 * 64 * 64);
            for (int n = 0; n < 64; ++n)
                for (int k = 0; k < 64; ++k) {
                    const size_t off = ((size_t)((n >> 3) * 16 + (k >> 2)) * 128 + (n & 7) * 16 + (k & 3) * 4) / 4;
                    kl[off] = hi[n * 64 + k];
                    kl[4096 + off] = lo[n * 64 + k];
                }
            if (!C.op_hi) CUDA_CHECK(cudaMalloc(&C.op_hi, 4 * 64 * 64 * sizeof(float)));
            CUDA_CHECK(cudaMemcpy(C.op_hi, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
            CUDA_CHECK(cudaMemcpy(C.op_hi + 64 * 64, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice));
            CUDA_CHECK(cudaMemcpy(C.op_hi + 2 * 64 * 64, kl.data(), kl.size() * 4, cudaMemcpyHostToDevice));
            C.op_mask = mask;
        }
        int dev_sms = 0;
        CUDA_CHECK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, C.device));
        hivc::launch_block_operator_tc(plane, out, h, w, C.op_hi, C.op_hi + 64 * 64, dev_sms, C.stream,
                                       C.op_hi + 2 * 64 * 64);
        C.launches += 1;
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
    });
}

int hivc_block_perblock(hivc_ctx* ctx, const float* plane, int32_t h, int32_t w, const uint64_t* masks, float* out) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        CUDA_CHECK(cudaMemsetAsync(C.d_status, 0, 2 * sizeof(int), C.stream));
        hivc::launch_block_perblock(plane, out, h, w, masks, C.d_status, C.stream);
        C.launches += 1;
        int st2[2] = {0, 0};
        CUDA_CHECK(cudaMemcpyAsync(st2, C.d_status, 2 * sizeof(int), cudaMemcpyDeviceToHost, C.stream));
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
        int st = st2[0];
        if (st == 0 && st2[1]) {  // blocks with more than 8 points: the one-thread kernel for those
            hivc::launch_block_perblock(plane, out, h, w, masks, C.d_status, C.stream, false, true);
            C.launches += 1;
            CUDA_CHECK(cudaMemcpyAsync(&st, C.d_status, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
            CUDA_CHECK(cudaStreamSynchronize(C.stream));
        }
        if (st == 4) {  // a block has more than 16 points: the wide-system variant for all blocks
            CUDA_CHECK(cudaMemsetAsync(C.d_status, 0, sizeof(int), C.stream));
            hivc::launch_block_perblock(plane, out, h, w, masks, C.d_status, C.stream, true);
            C.launches += 1;
            CUDA_CHECK(cudaMemcpyAsync(&st, C.d_status, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
            CUDA_CHECK(cudaStreamSynchronize(C.stream));
        }
        if (st == 1) hivc::fail(HIVC_E_PSEUDODIFF, "block mask needs at least one point");
        if (st == 2) hivc::fail(HIVC_E_PSEUDODIFF, "singular coefficient system");
    });
}

int hivc_brox(hivc_ctx* ctx, const double* frame_t, const double* frame_prev, int32_t h, int32_t w,
              const hivc_brox_params* params, const double* taps_presmooth, int32_t ntaps_presmooth,
              const double* taps_antialias, int32_t ntaps_antialias, double* u, double* v) {
    return guarded([&] {
        if (!ctx || !params) hivc::fail(HIVC_E_ARGUMENT, "null argument");
        if (h < 2 || w < 2) hivc::fail(HIVC_E_FLOW, "flow needs planes of at least 2x2");
        if (ntaps_presmooth > 63 || ntaps_antialias > 63 || ntaps_antialias < 1)
            hivc::fail(HIVC_E_ARGUMENT, "Gaussian radius out of range");
        if (!(params->pyramid_scale > 0 && params->pyramid_scale < 1))
            hivc::fail(HIVC_E_FLOW, "pyramid_scale must lie in (0, 1)");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        hivc::BroxParamsC P;
        P.alpha = params->alpha;
        P.gamma = params->gamma;
        P.pyramid_scale = params->pyramid_scale;
        P.min_size = params->min_size;
        P.warps = params->warps;
        P.fixed_point_iters = params->fixed_point_iters;
        P.solver_iters = params->solver_iters;
        P.eps = params->eps;
        P.presmooth_sigma = params->presmooth_sigma;
        int64_t launches = 0;
        hivc::brox_flow(C.brox, C.stream, frame_t, frame_prev, h, w, P, taps_presmooth, ntaps_presmooth, taps_antialias,
                        ntaps_antialias, u, v, &launches);
        C.launches += launches;
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
    });
}

int hivc_horn_schunck(hivc_ctx* ctx, const double* frame_t, const double* frame_prev, int32_t h, int32_t w,
                      double alpha, int32_t iterations, double* u, double* v) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null argument");
        if (h < 2 || w < 2) hivc::fail(HIVC_E_FLOW, "flow needs planes of at least 2x2");
        if (iterations < 0) hivc::fail(HIVC_E_ARGUMENT, "iterations must be >= 0");
        hivc::Context& C = ctx->c;
        CUDA_CHECK(cudaSetDevice(C.device));
        int64_t launches = 0;
        hivc::horn_schunck_flow(C.brox, C.stream, frame_t, frame_prev, h, w, alpha, iterations, u, v, &launches);
        C.launches += launches;
        CUDA_CHECK(cudaStreamSynchronize(C.stream));
    });
}

// ---------------------------------------------------------------- peer frame buffers (multi-GPU gather)

int hivc_peer_alloc(int32_t device, size_t bytes, void** ptr, uint8_t* ipc_handle) {
    return guarded([&] {
        CUDA_CHECK(cudaSetDevice(device));
        CUDA_CHECK(cudaMalloc(ptr, std::max<size_t>(bytes, 1)));
        cudaIpcMemHandle_t h;
        CUDA_CHECK(cudaIpcGetMemHandle(&h, *ptr));
        std::memcpy(ipc_handle, &h, sizeof(h));
    });
}

int hivc_peer_open(int32_t device, const uint8_t* ipc_handle, void** ptr) {
    return guarded([&] {
        CUDA_CHECK(cudaSetDevice(device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, ipc_handle, sizeof(h));
        CUDA_CHECK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int hivc_peer_close(void* ptr) {
    return guarded([&] { CUDA_CHECK(cudaIpcCloseMemHandle(ptr)); });
}

int hivc_peer_free(void* ptr) {
    return guarded([&] { CUDA_CHECK(cudaFree(ptr)); });
}

int hivc_memcpy(void* dst, const void* src, size_t bytes) {
    return guarded([&] { CUDA_CHECK(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault)); });
}

static int out_mode_of(int32_t v) {
    if (v < 0 || v > 2) hivc::fail(HIVC_E_ARGUMENT, "out_on_device must be 0 (host), 1 (device) or 2 (staged device)");
    return v;
}

int hivc_decode(hivc_ctx* ctx, const uint8_t* data, size_t len, int32_t gop_begin, int32_t gop_end, uint8_t* out,
                int32_t out_on_device, double* stage_seconds) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        CUDA_CHECK(cudaSetDevice(ctx->c.device));
        int gb = gop_begin, ge = gop_end;
        hivc::decode_streams(ctx->c, 1, &data, &len, &gb, &ge, &out, out_mode_of(out_on_device), stage_seconds);
    });
}

int hivc_decode_multi(hivc_ctx* ctx, int32_t nstreams, const uint8_t* const* data, const size_t* len,
                      const int32_t* gop_begin, const int32_t* gop_end, uint8_t* const* out, int32_t out_on_device,
                      double* stage_seconds) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        if (nstreams < 1) hivc::fail(HIVC_E_ARGUMENT, "no streams");
        CUDA_CHECK(cudaSetDevice(ctx->c.device));
        hivc::decode_streams(ctx->c, nstreams, data, len, gop_begin, gop_end, out, out_mode_of(out_on_device),
                             stage_seconds);
    });
}

int hivc_ctx_bytes(hivc_ctx* ctx, int64_t* h2d, int64_t* d2h) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        if (h2d) *h2d = ctx->c.h2d_bytes.load();
        if (d2h) *d2h = ctx->c.d2h_bytes.load();
    });
}

int hivc_ctx_decode_stats(hivc_ctx* ctx, double* out, int32_t reset) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        hivc::Context& C = ctx->c;
        std::lock_guard<std::mutex> g(C.stats_mu);
        const hivc::CgTotals& T = C.cg;
        double v[10] = {(double)T.solves,        (double)T.pixel_iters,      (double)T.pixel_levels,
                        (double)T.grid_launches, T.grid_seconds,             (double)T.grid_pixel_iters,
                        (double)T.grid_pixels,   (double)C.inter_frames,     C.inter_seconds,
                        (double)C.intra_frames};
        std::memcpy(out, v, sizeof(v));
        if (reset) {
            C.cg = hivc::CgTotals{};
            C.inter_frames = C.intra_frames = 0;
            C.inter_seconds = 0;
        }
    });
}

int hivc_ctx_set_stage_timing(hivc_ctx* ctx, int32_t enable) {
    return guarded([&] {
        if (!ctx) hivc::fail(HIVC_E_ARGUMENT, "null context");
        ctx->c.stage_events = enable != 0;
    });
}

}  // extern "C"
