// gemm_sm100.cu — K3: tcgen05 / TMEM / TMA quantized GEMM for the three HALO
// matmuls (Y = X W^T, dX = E W, dW = E^T X), sm_100a.
//
// Reference: qmatmul, quantize.hpp:339-380.  The INT8 per-tensor path
// accumulates exactly in integers and rescales once:
//     c = float(double(acc) * (double(sa) * double(sb)))        (:356-370)
// tcgen05.mma kind::i8 accumulates s32 in TMEM — exact, since
// |acc| <= K * 127^2 < 2^31 for K <= 133,144 — and the epilogue performs the
// same two roundings in fp64, so outputs are bit-identical to the reference.
// E4M3 runs kind::f8f6f4 with an fp32 accumulator (tolerance parity: the
// reference dequantizes and accumulates in double, :377-379).
//
// Operand layouts (no transposed copies are ever materialised):
//   F  Y  = Xq  Wq^T : A K-major [b][m],  B K-major [n][m]
//   E  dX = Ehq Wq   : A K-major [bp][n], B MN-major [n][m]
//   G  dW = Eq^T Xq  : A MN-major [b][n], B MN-major [b][m]   (K = tokens)
// 8-bit MN-major operands are legal for tcgen05 (instruction descriptor bits
// 15/16), so the reference's transpose_quantized (quantize.hpp:297-334)
// disappears into the TMA box orientation + UMMA descriptor.
//
// Structure (one CTA per SM, persistent, warp-specialised, 256 threads):
//   warp 0      TMA producer: 4-stage ring of {A 128x128 B, B 256x128 B}
//               tiles, 128 B swizzle, mbarrier complete_tx
//   warp 1      MMA issuer: one thread issues 4 x tcgen05.mma (K = 32 B each)
//               per stage into a 128 x 256 s32 TMEM accumulator; commits
//               free smem stages and publish finished accumulators
//   warp 2      TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4-7   epilogue: tcgen05.ld 32 lanes x 32 columns, fp64 rescale,
//               fp32 / bf16 / raw-s32 stores; overlaps the next tile's MMAs
//               through the double-buffered accumulator.
#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

namespace halo_b200 {

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK;  // 16 KB
constexpr int B_STAGE_BYTES = BN * BK;  // 32 KB
constexpr int GEMM_THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 16;  // tile raster: 16 M-tiles share each B panel in L2
constexpr size_t GEMM_SMEM = 1024 /*align slack*/ + STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 256;

struct GemmArgs {
    int M, N, K;
    int a_kmajor, b_kmajor;
    int fmt;        // 0 int8, 1 e4m3
    int out_kind;   // 0 fp32, 1 bf16, 2 raw s32
    const float* sa;
    const float* sb;
    void* out;
    // fused epilogue Hadamard (K4): blockwise FWHT of block 2^xf_lb along N
    // (the tile's 256 columns hold whole blocks), reference stage order, then
    // one multiply by xf_norm.  0 = none.
    int xf_lb;
    float xf_norm;
    // transposed store: out is [n_valid][M] row-major (C^T), rows >= n_valid
    // of C^T (N-index) are dropped (take_rows after the left transform)
    int out_trans;
    int n_valid;
};

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
template <int FMT>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (FMT == FMT_INT8) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
            : "memory");
    }
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
        "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
        "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void ep_bfly(float& a, float& b) {
    const float x = a, y = b;
    a = x + y;
    b = x - y;
}
__device__ __forceinline__ void ep_bfly2(float& a0, float& a1, float& b0, float& b1) {
    const float2 x = make_float2(a0, a1), y = make_float2(b0, b1);
    const float2 s = __fadd2_rn(x, y), d = __fadd2_rn(x, make_float2(-y.x, -y.y));
    a0 = s.x;
    a1 = s.y;
    b0 = d.x;
    b1 = d.y;
}

// store 8 consecutive N-columns (col0..col0+7) of one C row
__device__ __forceinline__ void ep_store8(const GemmArgs& p, int row, int col0, const float (&v)[8]) {
    if (!p.out_trans) {
        if (row >= p.M || col0 >= p.N) return;
        if (p.out_kind == 0) {
            float* o = static_cast<float*>(p.out) + (int64_t)row * p.N + col0;
            if (col0 + 8 <= p.N && (p.N % 4) == 0) {
                reinterpret_cast<float4*>(o)[0] = make_float4(v[0], v[1], v[2], v[3]);
                reinterpret_cast<float4*>(o)[1] = make_float4(v[4], v[5], v[6], v[7]);
            } else {
                
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (col0 + j < p.N) o[j] = v[j];
            }
        } else {
            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + (int64_t)row * p.N + col0;
            if (col0 + 8 <= p.N && (p.N % 8) == 0) store8(o, v);
            else
                {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (col0 + j < p.N) o[j] = __float2bfloat16_rn(v[j]);
            }
        }
    } else {
        // C^T[col][row]: consecutive lanes = consecutive rows -> 128 B per store
        if (row >= p.M) return;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = col0 + j;
            if (c < p.n_valid) {
                if (p.out_kind == 0) static_cast<float*>(p.out)[(int64_t)c * p.M + row] = v[j];
                else static_cast<__nv_bfloat16*>(p.out)[(int64_t)c * p.M + row] = __float2bfloat16_rn(v[j]);
            }
        }
    }
}

// UMMA shared-memory descriptor, SWIZZLE_128B, sm_100 version bits.
//   K-major : SBO = 1024 B (8 rows x 128 B), LBO unused
//   MN-major: LBO = stride between 128-element MN chunks, SBO = 1024 B
//             (8 k-rows x 128 B)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

// instruction descriptor (kind::i8 / kind::f8f6f4, dense)
__host__ __device__ constexpr uint32_t make_idesc(int fmt, int a_mn, int b_mn, int M, int N) {
    return (uint32_t)((fmt == FMT_INT8 ? 2u : 1u) << 4)         // D format: s32 / f32
           | (uint32_t)((fmt == FMT_INT8 ? 1u : 0u) << 7)       // A: signed int8 / e4m3
           | (uint32_t)((fmt == FMT_INT8 ? 1u : 0u) << 10)      // B
           | (uint32_t)(a_mn ? 1u : 0u) << 15 | (uint32_t)(b_mn ? 1u : 0u) << 16 |
           (uint32_t)(N >> 3) << 17 | (uint32_t)(M >> 4) << 24;
}

__device__ __forceinline__ void tile_coords(int t, int mt, int nt, int& mb, int& nb) {
    const int per_group = GROUP_M * nt;
    const int g = t / per_group;
    const int first = g * GROUP_M;
    const int gsize = min(GROUP_M, mt - first);
    const int r = t - g * per_group;
    mb = first + r % gsize;
    nb = r / gsize;
}

template <int FMT>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = bars + 2 * STAGES + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = (p.M + BM - 1) / BM, nt = (p.N + BN - 1) / BN;
    const int ntiles = mt * nt;
    const int nkb = (p.K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ============================ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mb, nb;
                tile_coords(t, mt, nt, mb, nb);
                const int m0 = mb * BM, n0 = nb * BN;
                for (int kb = 0; kb < nkb; ++kb) {
                    const int k0 = kb * BK;
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
                    uint8_t* a_dst = sA + stage * A_STAGE_BYTES;
                    uint8_t* b_dst = sB + stage * B_STAGE_BYTES;
                    if (p.a_kmajor) tma_load_2d(a_dst, &tmA, &full[stage], k0, m0);
                    else tma_load_2d(a_dst, &tmA, &full[stage], m0, k0);
                    if (p.b_kmajor) {
                        tma_load_2d(b_dst, &tmB, &full[stage], k0, n0);
                    } else {
                        tma_load_2d(b_dst, &tmB, &full[stage], n0, k0);
                        tma_load_2d(b_dst + B_STAGE_BYTES / 2, &tmB, &full[stage], n0 + 128, k0);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = make_idesc(FMT, !p.a_kmajor, !p.b_kmajor, BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * A_STAGE_BYTES);
                    const uint32_t b_addr = smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k) {
                        // K-major: +32 B along the swizzled row; MN-major: +32 k-rows = 4 KB
                        const uint64_t ad = p.a_kmajor ? make_desc(a_addr + k * 32, 16, 1024)
                                                       : make_desc(a_addr + k * 4096, A_STAGE_BYTES, 1024);
                        const uint64_t bd = p.b_kmajor ? make_desc(b_addr + k * 32, 16, 1024)
                                                       : make_desc(b_addr + k * 4096, B_STAGE_BYTES / 2, 1024);
                        tc_mma<FMT>(tmem_d, ad, bd, idesc, (kb | k) ? 1u : 0u);
                    }
                    tc_commit(&empty[stage]);  // smem stage free once these MMAs retire
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tc_commit(&tfull[acc]);  // accumulator complete
            }
        }
    } else if (warp >= 4) {
        // ============================ epilogue
        const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
        const double ss = (double)(*p.sa) * (double)(*p.sb);
        const float ssf = (float)ss;
        int local = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
            int mb, nb;
            tile_coords(t, mt, nt, mb, nb);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row = mb * BM + ew * 32 + lane;
            const bool row_ok = row < p.M;
            const uint32_t tacc = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
            if (p.xf_lb > 0) {
                // ---- fused FWHT along N (hadamard.hpp:136-177 order): pass 1
                // runs stages len = 1..16 on each 32-column chunk and parks the
                // fp32 result back in TMEM; pass 2 gathers 8 columns from each
                // chunk (tcgen05.ld x8) for stages len = 32, 64, 128.
                const int B = 1 << p.xf_lb;
                const bool two_pass = B > 32;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tacc + c * 32, r);
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if constexpr (FMT == FMT_INT8) v[j] = (float)((double)(int32_t)r[j] * ss);
                        else v[j] = __uint_as_float(r[j]) * ssf;
                    }
#pragma unroll
                    for (int j = 0; j < 32; j += 2) ep_bfly(v[j], v[j + 1]);  // len 1 (B >= 2)
#pragma unroll
                    for (int t = 1; t < 5; ++t) {
                        const int len = 1 << t;
                        if (len < B) {
#pragma unroll
                            for (int j = 0; j < 32; j += 2)
                                if ((j & len) == 0) ep_bfly2(v[j], v[j + 1], v[j + len], v[j + len + 1]);
                        }
                    }
                    if (two_pass) {
                        tmem_st32(tacc + c * 32, v);
                    } else {
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            float o[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) o[j] = v[8 * g + j] * p.xf_norm;
                            ep_store8(p, row, nb * BN + c * 32 + 8 * g, o);
                        }
                    }
                }
                if (two_pass) {
                    tmem_wait_st();
#pragma unroll 1
                    for (int g = 0; g < 4; ++g) {
                        float u[8][8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            uint32_t r[8];
                            tmem_ld8(tacc + c * 32 + g * 8, r);
#pragma unroll
                            for (int j = 0; j < 8; ++j) u[c][j] = __uint_as_float(r[j]);
                        }
                        tmem_wait_ld();
#pragma unroll
                        for (int t = 0; t < 3; ++t) {
                            const int h = 1 << t;
                            if ((32 << t) < B) {
#pragma unroll
                                for (int c = 0; c < 8; ++c)
                                    if ((c & h) == 0)
#pragma unroll
                                        for (int j = 0; j < 8; j += 2)
                                            ep_bfly2(u[c][j], u[c][j + 1], u[c + h][j], u[c + h][j + 1]);
                            }
                        }
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            float o[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) o[j] = u[c][j] * p.xf_norm;
                            ep_store8(p, row, nb * BN + c * 32 + 8 * g, o);
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                continue;
            }
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c * 32, r);
                const int col0 = nb * BN + c * 32;
                if (!row_ok || col0 >= p.N) continue;
                const bool full_chunk = (col0 + 32 <= p.N) && (p.N % 8 == 0);  // 16 B aligned rows
                if (p.out_kind == 2) {
                    int32_t* o = static_cast<int32_t*>(p.out) + (int64_t)row * p.N + col0;
                    if (full_chunk) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<int4*>(o + j) = make_int4(r[j], r[j + 1], r[j + 2], r[j + 3]);
                    } else {
                        
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < p.N) o[j] = (int32_t)r[j];
                    }
                    continue;
                }
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if constexpr (FMT == FMT_INT8) v[j] = (float)((double)(int32_t)r[j] * ss);
                    else v[j] = __uint_as_float(r[j]) * ssf;
                }
                if (p.out_kind == 0) {
                    float* o = static_cast<float*>(p.out) + (int64_t)row * p.N + col0;
                    if (full_chunk) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    } else {
                        
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < p.N) o[j] = v[j];
                    }
                } else {
                    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + (int64_t)row * p.N + col0;
                    if (full_chunk) {
#pragma unroll
                        for (int j = 0; j < 32; j += 8) store8(o + j, v + j);
                    } else {
                        
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < p.N) o[j] = __float2bfloat16_rn(v[j]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

// ------------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 get_encode();

// 2-D tensor map with 128 B swizzle (shared with fwht3.cu): element type
// `dtype` (0 fp32, 1 bf16, 2 uint8), row length `inner` elements (= 128 B),
// `outer` rows, box {inner, box_outer}, zero OOB fill.
bool encode_2d_sw128(CUtensorMap* map, int dtype, const void* base, uint64_t inner, uint64_t outer,
                     uint32_t box_outer) {
    auto enc = get_encode();
    if (!enc) return false;
    const int esz = dtype == 0 ? 4 : dtype == 1 ? 2 : 1;
    const CUtensorMapDataType dt = dtype == 0   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * esz};
    const cuuint32_t box[2] = {(cuuint32_t)inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// 2-D uint8 tensor map: inner dim `inner` (contiguous), outer dim `outer`,
// box {128, box_outer}, 128 B swizzle, zero OOB fill.
static bool encode_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
    auto enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner};
    const cuuint32_t box[2] = {128, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int run_gemm(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
             int b_kmajor, const float* sa, const float* sb, void* out, int out_kind, cudaStream_t st) {
    return run_gemm_x(fmt, A, B, M, N, K, a_kmajor, b_kmajor, sa, sb, out, out_kind, 0, 1.0f, 0, N, st);
}

int run_gemm_x(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
               int b_kmajor, const float* sa, const float* sb, void* out, int out_kind, int xf_lb, float xf_norm,
               int out_trans, int64_t n_valid, cudaStream_t st) {
    if (xf_lb < 0 || xf_lb > 8) return -1;  // the 256-column tile must hold whole blocks
    if ((xf_lb > 0 || out_trans) && out_kind == 2) return -1;
    if (M <= 0 || N <= 0 || K <= 0) return -1;
    if (M > INT32_MAX / 2 || N > INT32_MAX / 2 || K > INT32_MAX / 2) return -1;
    // TMA: global strides must be multiples of 16 bytes
    if ((a_kmajor ? K : M) % 16 != 0 || (b_kmajor ? K : N) % 16 != 0) return -1;
    if (out_kind == 2 && fmt != FMT_INT8) return -1;
    CUtensorMap ma, mb;
    const bool ok_a = a_kmajor ? encode_map(&ma, A, K, M, BM) : encode_map(&ma, A, M, K, BK);
    const bool ok_b = b_kmajor ? encode_map(&mb, B, K, N, BN) : encode_map(&mb, B, N, K, BK);
    if (!ok_a || !ok_b) return -2;
    GemmArgs args{(int)M, (int)N, (int)K, a_kmajor, b_kmajor, fmt, out_kind, sa, sb, out,
                  xf_lb, xf_norm, out_trans, (int)(n_valid < N ? n_valid : N)};
    const int tiles = (int)(((M + BM - 1) / BM) * ((N + BN - 1) / BN));
    const int grid = tiles < num_sms() ? tiles : num_sms();
    if (fmt == FMT_INT8) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_gemm<FMT_INT8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
            attr = true;
        }
        k_gemm<FMT_INT8><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(ma, mb, args);
    } else {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_gemm<FMT_E4M3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
            attr = true;
        }
        k_gemm<FMT_E4M3><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(ma, mb, args);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace halo_b200
