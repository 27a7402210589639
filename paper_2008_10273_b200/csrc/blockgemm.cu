// Config-2 block pseudodifferential microbench kernels (reference
// pseudodiff.py:218-279, codec.py:140-153): fit the Green's-function
// coefficients of every 8x8 residual block at its mask points and rebuild the
// block, u = G M c + a.
//
// (a) one mask layout shared by all blocks: fit + rebuild is a fixed linear
//     map of the block's 64 samples, rec = R f with the 64x64 operator
//         R[:, pos] = G[:, pos] S^-1[:K, :K] + 1 S^-1[K, :K]
//     (S the bordered (K+1)^2 system, computed once on the host in float64).
//     Applied to all blocks as ONE dense contraction on the 5th-gen tensor
//     cores: tcgen05.mma kind::tf32, M=128 blocks x N=64 x K=64, accumulator
//     in TMEM, 3xTF32 split precision (A_hi B_hi + A_hi B_lo + A_lo B_hi) so
//     the result carries ~fp32 accuracy (single-pass TF32 fails the 1e-3 bar,
//     SURVEY §0).  Operands are staged in shared memory in the canonical
//     K-major no-swizzle UMMA layout (8-row x 16-byte core matrices).
// (b) per-block masks: every block solves its own bordered system in shared
//     memory (float64) and rebuilds G[:, pos] c + a.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "aan_constants.h"
#include "blockgemm.h"
#include "func_attr.h"
#include "inpaint.h"

namespace hivc {

namespace {

constexpr int kTileM = 128;  // blocks per tile (UMMA M)
constexpr int kN = 64;       // outputs per block (UMMA N)
constexpr int kK = 64;       // samples per block (UMMA K total)
constexpr int kThreadsG = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// canonical K-major SWIZZLE_NONE offset (bytes) of element (row, k) of an
// operand with 64 K-elements per row: core matrix (row/8, k/4) is 128 B,
// core matrices of one row group are consecutive along K (LBO = 128 B),
// row groups are 16 core matrices apart (SBO = 2048 B)
__device__ __forceinline__ uint32_t kmajor_off(int row, int k) {
    return (uint32_t)(((row >> 3) * 16 + (k >> 2)) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
    return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, N=64, M=128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

}  // namespace

// rec[b] = R f[b] for every 8x8 block b of the plane (f32 in/out), 3xTF32 on tcgen05.
__global__ void __launch_bounds__(kThreadsG, 2)
    block_operator_tc_kernel(const float* __restrict__ plane, float* __restrict__ out, int h, int w,
                             const float* __restrict__ r_hi, const float* __restrict__ r_lo, int nblocks, int vec) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* a_hi = smem;                        // 128 x 64 f32 = 32 KB
    uint8_t* a_lo = smem + 32768;                // 32 KB
    uint8_t* b_hi = smem + 65536;                // 64 x 64 f32 = 16 KB
    uint8_t* b_lo = smem + 65536 + 16384;        // 16 KB
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nbx = (w + 7) >> 3;
    const int ntiles = (nblocks + kTileM - 1) / kTileM;

    // operator halves, K-major (row n of R = output pixel n, k = input pixel):
    // every thread issues its 16 float4 loads before the first store (one round trip)
    {
        float4 vh[8], vl[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            vh[i] = __ldg(reinterpret_cast<const float4*>(r_hi) + tid + kThreadsG * i);
            vl[i] = __ldg(reinterpret_cast<const float4*>(r_lo) + tid + kThreadsG * i);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = 4 * (tid + kThreadsG * i), n = e / kK, k = e % kK;
            *reinterpret_cast<float4*>(b_hi + kmajor_off(n, k)) = vh[i];
            *reinterpret_cast<float4*>(b_lo + kmajor_off(n, k)) = vl[i];
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(kN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    uint32_t phase = 0;

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // ---- stage the tile's blocks: A = f (row m = block tile*128 + m, 64 samples), split hi/lo.
        // Thread m loads its own block (8 rows x 2 float4, all issued before use).
        {
            const int b = tile * kTileM + tid;
            const int by = b / nbx, bx = b % nbx, y0 = by * 8, x0 = bx * 8;
            float4 v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (b < nblocks) {
                if (vec && y0 + 8 <= h && x0 + 8 <= w) {
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const float4* src = reinterpret_cast<const float4*>(plane + (size_t)(y0 + r) * w + x0);
                        v[2 * r] = __ldg(src);
                        v[2 * r + 1] = __ldg(src + 1);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int y = y0 + (j >> 1), x = x0 + (j & 1) * 4;
                        float t[4] = {0.f, 0.f, 0.f, 0.f};
                        for (int q = 0; q < 4; ++q)
                            if (y < h && x + q < w) t[q] = __ldg(plane + (size_t)y * w + x + q);
                        v[j] = make_float4(t[0], t[1], t[2], t[3]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {  // samples k = 4j .. 4j+3 (row j/2 of the block)
                const float4 hv = make_float4(tf32_hi(v[j].x), tf32_hi(v[j].y), tf32_hi(v[j].z), tf32_hi(v[j].w));
                const float4 lv = make_float4(v[j].x - hv.x, v[j].y - hv.y, v[j].z - hv.z, v[j].w - hv.w);
                *reinterpret_cast<float4*>(a_hi + kmajor_off(tid, 4 * j)) = hv;
                *reinterpret_cast<float4*>(a_lo + kmajor_off(tid, 4 * j)) = lv;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy smem writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
            uint32_t acc = 0;
#pragma unroll
            for (int kb = 0; kb < kK / 8; ++kb) {  // K = 8 tf32 per MMA = 2 core matrices
                const uint32_t off = kb * 2 * 128;
                mma_tf32(tmem, smem_desc(ah + off, 128, 2048), smem_desc(bh + off, 128, 2048), acc);
                acc = 1;
                mma_tf32(tmem, smem_desc(ah + off, 128, 2048), smem_desc(bl + off, 128, 2048), 1);
                mma_tf32(tmem, smem_desc(al + off, 128, 2048), smem_desc(bh + off, 128, 2048), 1);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&mbar)));
        }
        // ---- wait for the accumulator
        {
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(done)
                    : "r"(smem_u32(&mbar)), "r"(phase));
            }
            phase ^= 1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;");
        // ---- epilogue: warp w reads TMEM lanes 32w..32w+31 (= blocks), 64 columns
        const int m = warp * 32 + lane;
        const int b = tile * kTileM + m;
        const int by = b / nbx, bx = b % nbx;
#pragma unroll
        for (int c0 = 0; c0 < kN; c0 += 16) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            if (b < nblocks) {
                if (vec && by * 8 + 8 <= h && bx * 8 + 8 <= w) {  // two block rows, 4 float4 stores
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const int n = c0 + j;
                        float4* dst = reinterpret_cast<float4*>(out + (size_t)(by * 8 + (n >> 3)) * w + bx * 8 + (n & 7));
                        *dst = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                           __uint_as_float(v[j + 3]));
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        int n = c0 + j;
                        int y = by * 8 + (n >> 3), x = bx * 8 + (n & 7);
                        if (y < h && x < w) out[(size_t)y * w + x] = __uint_as_float(v[j]);
                    }
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();  // TMEM and smem reused by the next tile
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kN));
}

// The same contraction fed by TMA, persistent, with the next tile's load in
// flight while the current one is split, multiplied and stored.  The plane is
// viewed as a rank-3 tensor (8 floats of a block row, blocks along the image
// row at 32 B, image rows at w*4 B); ONE cp.async.bulk.tensor per tile brings
// 128 consecutive blocks of a block row x 8 image rows (32 KB) into shared
// memory with the 32-byte swizzle, which is the canonical K-major SW32 UMMA
// layout for A (row = block, 32 B = the block's 8 pixels of one image row =
// the 8 tf32 K-elements of one MMA): image row r feeds MMA k-step r with its
// descriptor at tile + r * 4096 (SBO 256 B between 8-block groups).  Blocks
// past the row end are zero-filled by TMA and not stored.  3xTF32 as above:
// the split into A_hi / A_lo is an elementwise pass over the (swizzled) tile,
// so both halves keep the layout.  Tiles: (block row, 128-block span).
namespace {
constexpr int kTmaTile = 128 * 64 * 4;  // bytes of one A tile (fp32)

__device__ __forceinline__ uint64_t smem_desc_sw32(uint32_t addr, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;  // LBO (unused for a swizzled K-major operand one atom wide)
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    d |= (uint64_t)6 << 61;  // layout type SWIZZLE_32B
    return d;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_tile(const CUtensorMap* tmap, uint32_t dst, uint32_t bar, int bj0, int y0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kTmaTile) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(dst),
        "l"(tmap), "r"(0), "r"(bj0), "r"(y0), "r"(bar)
        : "memory");
}
}  // namespace

__global__ void __launch_bounds__(kThreadsG, 1)
    block_operator_tma_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ out, int h, int w,
                              const float* __restrict__ r_kl) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* raw[2] = {smem, smem + kTmaTile};     // TMA destinations (fp32 tiles)
    uint8_t* a_hi = smem + 2 * kTmaTile;           // split halves, same swizzled layout
    uint8_t* a_lo = smem + 3 * kTmaTile;
    uint8_t* b_hi = smem + 4 * kTmaTile;           // 64 x 64 operator, K-major, no swizzle
    uint8_t* b_lo = b_hi + 16384;
    __shared__ __align__(8) uint64_t full[2];
    __shared__ __align__(8) uint64_t mma_bar;
    __shared__ __align__(8) uint64_t op_bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nbx = w >> 3, nby = h >> 3;
    const int spans = (nbx + kTileM - 1) / kTileM;
    const int ntiles = nby * spans;
    auto tile_coords = [&](int t, int& bj0, int& by) {
        by = t / spans;
        bj0 = (t - by * spans) * kTileM;
    };
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mma_bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&op_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        // the operator halves, already in the K-major layout (host), as one bulk copy
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&op_bar)), "r"(32768)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(b_hi)),
                     "l"(r_kl), "r"(32768), "r"(smem_u32(&op_bar))
                     : "memory");
        // the first two tiles' loads go out before anything else
        for (int s = 0; s < 2; ++s) {
            const int t = blockIdx.x + s * gridDim.x;
            if (t < ntiles) {
                int bj0, by;
                tile_coords(t, bj0, by);
                tma_load_tile(&tmap, smem_u32(raw[s]), smem_u32(&full[s]), bj0, by * 8);
            }
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(kN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it & 1;
        int bj0, by;
        tile_coords(t, bj0, by);
        mbar_wait(smem_u32(&full[st]), (uint32_t)((it >> 1) & 1));
        // ---- split the landed tile into tf32 hi / lo halves (elementwise: the layout is kept)
        {
            const float4* src = reinterpret_cast<const float4*>(raw[st]);
            float4* dh = reinterpret_cast<float4*>(a_hi);
            float4* dl = reinterpret_cast<float4*>(a_lo);
#pragma unroll 4
            for (int i = tid; i < kTmaTile / 16; i += kThreadsG) {
                const float4 v = src[i];
                const float4 hv = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                dh[i] = hv;
                dl[i] = make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;");
        __syncthreads();
        if (it == 0) mbar_wait(smem_u32(&op_bar), 0);
        if (tid == 0) {
            // raw[st] is consumed: the tile two ahead goes out now
            const int tn = t + 2 * gridDim.x;
            if (tn < ntiles) {
                int nb0, nby2;
                tile_coords(tn, nb0, nby2);
                tma_load_tile(&tmap, smem_u32(raw[st]), smem_u32(&full[st]), nb0, nby2 * 8);
            }
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
            for (int kb = 0; kb < kK / 8; ++kb) {  // image row kb of the blocks = k 8kb .. 8kb+7
                const uint64_t dah = smem_desc_sw32(ah + kb * 4096, 256), dal = smem_desc_sw32(al + kb * 4096, 256);
                const uint32_t boff = kb * 2 * 128;
                mma_tf32(tmem, dah, smem_desc(bh + boff, 128, 2048), kb > 0);
                mma_tf32(tmem, dah, smem_desc(bl + boff, 128, 2048), 1);
                mma_tf32(tmem, dal, smem_desc(bh + boff, 128, 2048), 1);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&mma_bar)));
        }
        mbar_wait(smem_u32(&mma_bar), (uint32_t)(it & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        // ---- epilogue: warp w reads TMEM lanes 32w..32w+31 (= blocks), 64 columns (= pixels)
        const int m = warp * 32 + lane;
        const int bx = bj0 + m;
#pragma unroll
        for (int c0 = 0; c0 < kN; c0 += 16) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            if (bx < nbx) {
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    const int n = c0 + j;
                    float4* dst = reinterpret_cast<float4*>(out + (size_t)(by * 8 + (n >> 3)) * w + bx * 8 + (n & 7));
                    *dst = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                       __uint_as_float(v[j + 3]));
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();  // TMEM and the split halves are reused by the next tile
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kN));
}

// (b) per-block masks: bordered solve in shared memory (float64), then
// rec = G[:, pos] c + a (pseudodiff.py:218-240, 266-272), one warp per block.
constexpr int kPbWarps = 4;

// LD: row stride of the bordered system (K <= LD - 2).  The LD = 18 variant
// (K <= 16: every block of a 5 % mask in practice) needs ~10 KB of shared
// memory per CTA instead of ~140 KB, so 16 CTAs per SM run instead of one; a
// block with more points flags status 4 and the host reruns with LD = 66.
template <int LD>
__global__ void __launch_bounds__(kPbWarps * 32)
    block_perblock_kernel(const float* __restrict__ plane, float* __restrict__ out, int h, int w,
                          const uint64_t* __restrict__ masks, int nblocks, int* status, int min_k) {
    extern __shared__ double sm[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * kPbWarps + wid;
    if (b >= nblocks) return;
    double* M = sm + (size_t)wid * (LD - 1) * LD;
    double* fb = sm + (size_t)kPbWarps * (LD - 1) * LD + wid * 64;
    int* pos = reinterpret_cast<int*>(sm + (size_t)kPbWarps * ((LD - 1) * LD + 64)) + wid * 64;
    const uint64_t mask = masks[b];
    const int K = __popcll(mask);
    if (K > 0 && K <= min_k) return;  // (done by block_schur8_kernel)
    const int nbx = (w + 7) >> 3;
    const int by = b / nbx, bx = b % nbx;
    for (int k = lane; k < 64; k += 32) {
        int y = by * 8 + (k >> 3), x = bx * 8 + (k & 7);
        fb[k] = (y < h && x < w) ? (double)plane[(size_t)y * w + x] : 0.0;
    }
    if (K == 0) {
        if (lane == 0) atomicExch(status, 1);
        return;
    }
    if (K > LD - 2) {  // does not fit this variant
        if (lane == 0) atomicExch(status, 4);
        return;
    }
    for (int j = lane; j < 64; j += 32)
        if ((mask >> j) & 1ull) pos[__popcll(mask & ((1ull << j) - 1ull))] = j;
    __syncwarp();
    const int N = K + 1;
    for (int e = lane; e < N * N; e += 32) {
        int i = e / N, j = e % N;
        M[i * LD + j] = (i < K && j < K) ? kGreens64[pos[i] * 64 + pos[j]] : ((i == K && j == K) ? 0.0 : 1.0);
    }
    for (int i = lane; i < N; i += 32) M[i * LD + N] = i < K ? fb[pos[i]] : 0.0;
    __syncwarp();
    for (int col = 0; col < N; ++col) {
        int piv = col;
        double best = -1.0;
        for (int i = col; i < N; ++i) {
            double v = fabs(M[i * LD + col]);
            if (v > best) {
                best = v;
                piv = i;
            }
        }
        if (best == 0.0) {
            if (lane == 0) atomicExch(status, 2);
            return;
        }
        if (piv != col)
            for (int j = lane; j <= N; j += 32) {
                double t = M[col * LD + j];
                M[col * LD + j] = M[piv * LD + j];
                M[piv * LD + j] = t;
            }
        __syncwarp();
        const double d = M[col * LD + col];
        for (int i = col + 1; i < N; ++i) {
            const double l = M[i * LD + col] / d;
            for (int j = col + 1 + lane; j <= N; j += 32) M[i * LD + j] = M[i * LD + j] - l * M[col * LD + j];
            __syncwarp();
        }
    }
    if (lane == 0)
        for (int i = N - 1; i >= 0; --i) {
            double s = M[i * LD + N];
            for (int j = i + 1; j < N; ++j) s = s - M[i * LD + j] * M[j * LD + N];
            M[i * LD + N] = s / M[i * LD + i];
        }
    __syncwarp();
    const double a = M[K * LD + N];
    for (int n = lane; n < 64; n += 32) {
        double acc = 0.0;
        for (int i = 0; i < K; ++i) acc = acc + kGreens64[n * 64 + pos[i]] * M[i * LD + N];
        int y = by * 8 + (n >> 3), x = bx * 8 + (n & 7);
        if (y < h && x < w) out[(size_t)y * w + x] = (float)(acc + a);
    }
}

// Config 2b: the bordered system [[G_KK, 1], [1^T, 0]] [c; a] = [f_K; 0] of
// every block solved through its Schur complement — G_KK (a principal
// submatrix of the positive semi-definite Green's matrix whose null space is
// the constant block, so positive definite for K < 64) is factored
// G_KK = L L^T, then y = G_KK^-1 f, z = G_KK^-1 1, a = 1^T y / 1^T z and
// c = y - a z (the unique solution of the reference's system,
// pseudodiff.py:218-263; rounding differs from LAPACK's pivoted LU at the
// 1e-13 level); rec = G[:, pos] c + a.
// Eight lanes per block (four blocks per warp) for blocks of up to kSL
// points: lane j owns rows j and j + 8 of the Cholesky factor, which lives in
// shared memory with the block's points and right-hand sides, and every loop
// runs to K (no unrolling to the worst case: a typical block has 1-6
// points).  G_KK = L L^T column by column, forward and backward substitution
// for y = G^-1 f and z = G^-1 1, a = sum y / sum z, c = y - a z; lane j then
// rebuilds pixel column j of the block, reading the symmetric Green's matrix
// along rows (G[p][n] in place of G[n][p]: conflict-free).  Blocks with more
// points are flagged (status[1]) for the warp-per-block kernel above.
constexpr int kSL = 16;
constexpr int kS8Warps = 8;
constexpr int kSGroup = kSL * (kSL + 1) / 2 + 3 * kSL;  // doubles per block: packed L, y, z, positions

__global__ void __launch_bounds__(kS8Warps * 32) block_schur8_kernel(const float* __restrict__ plane,
                                                                     float* __restrict__ out, int h, int w,
                                                                     const uint64_t* __restrict__ masks,
                                                                     int nblocks, int* status,
                                                                     const double* __restrict__ G) {
    // G: the 64 x 64 Green's matrix in global memory (L1-resident: 32 KB, read along rows)
    extern __shared__ double s8[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, grp = lane >> 3, j = lane & 7;
    const unsigned gm = 0xFFu << (8 * grp);
    const int b = (blockIdx.x * kS8Warps + wid) * 4 + grp;
    if (b >= nblocks) return;  // (whole 8-lane groups)
    const uint64_t mask = __ldg(masks + b);
    const int K = __popcll(mask);
    if (K == 0) {
        if (j == 0) atomicExch(status, 1);
        return;
    }
    if (K > kSL) {  // the one-thread kernel takes these
        if (j == 0) atomicOr(status + 1, 1);
        return;
    }
    double* L = s8 + (size_t)(wid * 4 + grp) * kSGroup;
    double* Y = L + kSL * (kSL + 1) / 2;
    auto T = [](int i, int k) { return i * (i + 1) / 2 + k; };  // packed lower triangle
    double* Z = Y + kSL;
    int* P = reinterpret_cast<int*>(Z + kSL);
    const int nbx = (w + 7) >> 3;
    const int by = b / nbx, bx = b - by * nbx;
    for (int i = j; i < K; i += 8) {  // point i: the i-th set bit, its sample, rhs 1
        uint64_t m = mask;
        for (int t = 0; t < i; ++t) m &= m - 1;
        const int p = __ffsll((long long)m) - 1;
        P[i] = p;
        const int yy = by * 8 + (p >> 3), xx = bx * 8 + (p & 7);
        Y[i] = (yy < h && xx < w) ? (double)__ldg(plane + (size_t)yy * w + xx) : 0.0;
        Z[i] = 1.0;
    }
    __syncwarp(gm);
    // G_KK = L L^T, column by column
    bool bad = false;
    for (int c = 0; c < K; ++c) {
        const int pc = P[c];
        if (j == (c & 7)) {
            double d = G[pc * 64 + pc];
            for (int k = 0; k < c; ++k) d = d - L[T(c, k)] * L[T(c, k)];
            bad |= !(d > 0.0);
            L[T(c, c)] = sqrt(fmax(d, 1e-300));
        }
        __syncwarp(gm);
        const double lcc = L[T(c, c)];
        for (int i = j; i < K; i += 8)
            if (i > c) {
                double v = G[pc * 64 + P[i]];  // = G[p_i][p_c] (symmetric)
                for (int k = 0; k < c; ++k) v = v - L[T(i, k)] * L[T(c, k)];
                L[T(i, c)] = v / lcc;
            }
        __syncwarp(gm);
    }
    if (__any_sync(gm, bad)) {
        if (j == 0) atomicExch(status, 2);
        return;
    }
    // forward: L u = f (and 1), then backward: L^T x = u
    for (int c = 0; c < K; ++c) {
        const double lcc = L[T(c, c)];
        if (j == (c & 7)) {
            Y[c] = Y[c] / lcc;
            Z[c] = Z[c] / lcc;
        }
        __syncwarp(gm);
        const double yc = Y[c], zc = Z[c];
        for (int i = j; i < K; i += 8)
            if (i > c) {
                const double l = L[T(i, c)];
                Y[i] = Y[i] - l * yc;
                Z[i] = Z[i] - l * zc;
            }
        __syncwarp(gm);
    }
    for (int c = K - 1; c >= 0; --c) {
        const double lcc = L[T(c, c)];
        if (j == (c & 7)) {
            Y[c] = Y[c] / lcc;
            Z[c] = Z[c] / lcc;
        }
        __syncwarp(gm);
        const double yc = Y[c], zc = Z[c];
        for (int i = j; i < c; i += 8) {
            const double l = L[T(c, i)];
            Y[i] = Y[i] - l * yc;
            Z[i] = Z[i] - l * zc;
        }
        __syncwarp(gm);
    }
    double sy = 0.0, sz = 0.0;
    for (int i = 0; i < K; ++i) {
        sy += Y[i];
        sz += Z[i];
    }
    const double a = sy / sz;
    // lane j rebuilds pixel column j: rec[r][j] = sum_i G[p_i][r*8 + j] (y_i - a z_i) + a
    double acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0.0;
    for (int i = 0; i < K; ++i) {
        const double ci = Y[i] - a * Z[i];
        const double* g = G + P[i] * 64 + j;
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r] = acc[r] + g[r * 8] * ci;
    }
    const int xx = bx * 8 + j;
    if (xx < w)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int yy = by * 8 + r;
            if (yy < h) out[(size_t)yy * w + xx] = (float)(acc[r] + a);
        }
}

// ---------------------------------------------------------------- host

// R = G[:, pos] S^-1[:K,:K] + 1 S^-1[K,:K] scattered to the mask columns (float64, Gauss-Jordan)
void shared_block_operator(uint64_t mask, std::vector<double>& R) {
    std::vector<int> pos;
    for (int j = 0; j < 64; ++j)
        if ((mask >> j) & 1ull) pos.push_back(j);
    const int K = (int)pos.size();
    if (K == 0) fail(HIVC_E_PSEUDODIFF, "block mask needs at least one point");
    const int N = K + 1;
    std::vector<double> S((size_t)N * 2 * N, 0.0);  // [S | I]
    for (int i = 0; i < N; ++i) {
        for (int j = 0; j < N; ++j)
            S[(size_t)i * 2 * N + j] =
                (i < K && j < K) ? kGreens64Host[pos[i] * 64 + pos[j]] : ((i == K && j == K) ? 0.0 : 1.0);
        S[(size_t)i * 2 * N + N + i] = 1.0;
    }
    for (int c = 0; c < N; ++c) {
        int piv = c;
        for (int i = c + 1; i < N; ++i)
            if (std::fabs(S[(size_t)i * 2 * N + c]) > std::fabs(S[(size_t)piv * 2 * N + c])) piv = i;
        if (S[(size_t)piv * 2 * N + c] == 0.0) fail(HIVC_E_PSEUDODIFF, "singular coefficient system");
        if (piv != c)
            for (int j = 0; j < 2 * N; ++j) std::swap(S[(size_t)c * 2 * N + j], S[(size_t)piv * 2 * N + j]);
        double d = S[(size_t)c * 2 * N + c];
        for (int j = 0; j < 2 * N; ++j) S[(size_t)c * 2 * N + j] /= d;
        for (int i = 0; i < N; ++i) {
            if (i == c) continue;
            double l = S[(size_t)i * 2 * N + c];
            if (l != 0.0)
                for (int j = 0; j < 2 * N; ++j) S[(size_t)i * 2 * N + j] -= l * S[(size_t)c * 2 * N + j];
        }
    }
    auto inv = [&](int i, int j) { return S[(size_t)i * 2 * N + N + j]; };
    R.assign(64 * 64, 0.0);
    for (int n = 0; n < 64; ++n)
        for (int j = 0; j < K; ++j) {
            double acc = inv(K, j);  // constant term a = S^-1[K, :K] f_K
            for (int i = 0; i < K; ++i) acc += kGreens64Host[n * 64 + pos[i]] * inv(i, j);
            R[(size_t)n * 64 + pos[j]] = acc;
        }
}

void launch_block_operator_tc(const float* plane, float* out, int h, int w, const float* r_hi, const float* r_lo,
                              int num_sms, cudaStream_t s, const float* r_kl) {
    const int nblocks = ((h + 7) / 8) * ((w + 7) / 8);
    const int ntiles = (nblocks + kTileM - 1) / kTileM;
    const size_t smem = 65536 + 32768;
    ensure_func_attr((const void*)block_operator_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // the TMA-fed persistent kernel: whole 8x8 blocks, 16-byte aligned rows
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        cudaGetLastError();
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (r_kl && encode && h % 8 == 0 && w % 8 == 0 && (uintptr_t)plane % 16 == 0 && (uintptr_t)out % 16 == 0) {
        CUtensorMap tmap;
        const cuuint64_t dims[3] = {8, (cuuint64_t)(w / 8), (cuuint64_t)h};
        const cuuint64_t strides[2] = {32, (cuuint64_t)w * 4};
        const cuuint32_t box[3] = {8, (cuuint32_t)kTileM, 8};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(plane), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
            const size_t tsmem = 4 * (size_t)kTmaTile + 32768 + 1024;
            ensure_func_attr((const void*)block_operator_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tsmem);
            const int tiles = (h / 8) * ((w / 8 + kTileM - 1) / kTileM);
            block_operator_tma_kernel<<<std::min(tiles, num_sms), kThreadsG, tsmem, s>>>(tmap, out, h, w, r_kl);
            CUDA_CHECK(cudaGetLastError());
            return;
        }
    }
    const int vec = (w % 4 == 0) && ((uintptr_t)plane % 16 == 0) && ((uintptr_t)out % 16 == 0);
    // two CTAs per SM (96 KB smem, 64 TMEM columns each): one tile per CTA at 1080p, loads of one
    // CTA overlap the MMA / epilogue of the other
    block_operator_tc_kernel<<<std::min(ntiles, 2 * num_sms), kThreadsG, smem, s>>>(plane, out, h, w, r_hi, r_lo, nblocks,
                                                                             vec);
    CUDA_CHECK(cudaGetLastError());
}

// The Green's matrix in global memory, once per device.
static const double* greens_device() {
    static std::mutex mu;
    static std::map<int, double*> per_dev;
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    double*& p = per_dev[dev];
    if (!p) {
        CUDA_CHECK(cudaMalloc(&p, 4096 * sizeof(double)));
        CUDA_CHECK(cudaMemcpy(p, kGreens64Host, 4096 * sizeof(double), cudaMemcpyHostToDevice));
    }
    return p;
}

void launch_block_perblock(const float* plane, float* out, int h, int w, const uint64_t* masks, int* status,
                           cudaStream_t s, bool wide, bool second_pass) {
    const int nblocks = ((h + 7) / 8) * ((w + 7) / 8);
    auto go = [&](auto kernel, int ld, int min_k) {
        const size_t smem =
            (size_t)kPbWarps * ((ld - 1) * ld + 64) * sizeof(double) + kPbWarps * 64 * sizeof(int);
        ensure_func_attr((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kernel<<<(nblocks + kPbWarps - 1) / kPbWarps, kPbWarps * 32, smem, s>>>(plane, out, h, w, masks, nblocks,
                                                                                  status, min_k);
    };
    if (wide) {
        go(block_perblock_kernel<66>, 66, 0);
    } else if (second_pass) {  // the blocks block_schur8_kernel flagged (K > kSL): a warp each, K <= 16
        go(block_perblock_kernel<18>, 18, kSL);
    } else {
        const size_t smem = (size_t)(kS8Warps * 4 * kSGroup) * sizeof(double);
        ensure_func_attr((const void*)block_schur8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int per_cta = kS8Warps * 4;
        block_schur8_kernel<<<(nblocks + per_cta - 1) / per_cta, kS8Warps * 32, smem, s>>>(plane, out, h, w, masks,
                                                                                          nblocks, status,
                                                                                          greens_device());
    }
    CUDA_CHECK(cudaGetLastError());
}

}  // namespace hivc
