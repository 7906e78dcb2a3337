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

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

namespace halo_b200 {

// Per-CTA tile: 128 rows (TMEM lanes) x 256 columns.  CG = 2 pairs two CTAs
// of a cluster on one 256 x 256 tile with cta_group::2 MMAs: each CTA loads
// its 128 rows of A and HALF of B (128 of the 256 N-rows), so the L2->SM
// operand traffic per MAC drops by a third (48 -> 32 KB per CTA per k-block).
constexpr int BM = 128, BN = 256, BK = 128;
constexpr int A_STAGE_BYTES = BM * BK;  // 16 KB
template <int CG>
struct GemmCfg {
    static constexpr int B_ROWS = BN / CG;                       // B rows loaded per CTA
    static constexpr int B_STAGE_BYTES = B_ROWS * BK;            // 32 / 16 KB
    static constexpr int STAGES = CG == 1 ? 4 : 6;
    static constexpr int TILE_M = BM * CG;                       // rows per (pair) tile
};
constexpr int GEMM_THREADS = 384;  // 4 control warps + 8 epilogue warps
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 16;  // tile raster: 16 M-tiles share each B panel in L2
constexpr int EPI_WARPS = 8;
constexpr int STG_BYTES = EPI_WARPS * 32 * 32 * 4;  // epilogue staging: 32 rows x 32 fp32 per warp
template <int CG>
constexpr size_t gemm_smem() {
    return 1024 /*align slack*/ + GemmCfg<CG>::STAGES * (A_STAGE_BYTES + GemmCfg<CG>::B_STAGE_BYTES) + STG_BYTES + 256;
}
static_assert(gemm_smem<1>() <= 232448 && gemm_smem<2>() <= 232448, "smem budget");

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
    int dbg_skip_epi;  // HALO_GEMM_DEBUG_SKIP_EPI=1: epilogue only releases TMEM (timing experiments)
    int tma_store;     // C written by TMA boxes of 32 rows x 128 B (tmC); else coalesced STG flush
    // Granularity::row scales on non-contracted dims (nullptr = per tensor):
    // sa_vec[M] per row of C, sb_vec[N] per column of C
    const float* sa_vec;
    const float* sb_vec;
    // sharded operands (HQ-FSDP without an all-gather): A / B split into
    // *_shards equal parts of *_len rows along K (*_along_k) or along M / N,
    // each part behind its own tensor map in global memory (parts may live
    // in peer GPUs' HBM, reached over NVLink).  0 shards = tmA / tmB.
    const CUtensorMap* a_maps;
    int a_shards, a_len, a_along_k;
    const CUtensorMap* b_maps;
    int b_shards, b_len, b_along_k;
    // scattered C (HQ-FSDP gradient reduce-scatter fused into the G GEMM):
    // rows [i*c_len, (i+1)*c_len) of C go through c_maps[i] -- this rank's
    // slot in the receive buffer of the rank owning those rows, possibly a
    // peer GPU's HBM (TMA stores over NVLink).  0 parts = tmC.
    const CUtensorMap* c_maps;
    int c_parts, c_len;
    // SwiGLU epilogue (the up projection of a Llama MLP): C = u (bf16) and
    // h = silu(g) * u into tmH, g [M][N] bf16 read from HBM (glu_g != null);
    // glu_res: residual epilogue instead, C = RN_bf16(g + RN_bf16(acc)) (the
    // block's y = h + MLP(.) as torch adds two bf16 tensors), no tmH
    const __nv_bfloat16* glu_g;
    int glu_res;
};

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_commit_mc2(uint64_t* bar) {
    // arrive on the barrier at this offset in BOTH CTAs of the pair
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-CTA TMA: data lands in this CTA's smem, completion bytes go to the
// leader CTA's mbarrier (cluster address)
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}

template <int FMT, int CG>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (CG == 2) {
        if constexpr (FMT == FMT_INT8) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
                : "memory");
        } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
                : "memory");
        }
        return;
    }
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

// split form: issue now, consume after tmem_wait32 (which ties the registers
// to the wait so the compiler cannot read them early)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait32(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])::"memory");
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
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
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

// ---- epilogue staging: a warp's 32 rows x 32 fp32 columns (4 KB), the
// 16 B chunks XOR-swizzled by row so that both the row-per-lane writes and
// the chunk-per-lane reads are bank-conflict free; the flush then writes
// whole sectors (8 lanes cover one 128 B row of fp32 per instruction)
// instead of one scattered 16 B piece per lane and row.
__device__ __forceinline__ int stg_phys(int row, int k) { return k ^ (row & 7); }

// 8 values = staged chunks 2*seg, 2*seg+1 of this lane's row
__device__ __forceinline__ void stg_put(float* S, int lane, int seg, const float* v8) {
    float4* R = reinterpret_cast<float4*>(S + lane * 32);
    R[stg_phys(lane, 2 * seg)] = make_float4(v8[0], v8[1], v8[2], v8[3]);
    R[stg_phys(lane, 2 * seg + 1)] = make_float4(v8[4], v8[5], v8[6], v8[7]);
}

// staged (row r, chunk k) -> C[row0 + r][col_base + (k>>1)*cstride + (k&1)*4 .. +3]
__device__ __forceinline__ void stg_flush(const GemmArgs& p, const float* S, int lane, int row0, int col_base,
                                          int cstride) {
    const int k = lane & 7;
    const int col = col_base + (k >> 1) * cstride + (k & 1) * 4;
    const bool full = col + 4 <= p.N && (p.N % 4) == 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int r = 4 * t + (lane >> 3);
        const float4 a = reinterpret_cast<const float4*>(S + r * 32)[stg_phys(r, k)];
        const int row = row0 + r;
        if (row >= p.M || col >= p.N) continue;
        const int64_t off = (int64_t)row * p.N + col;
        const float v[4] = {a.x, a.y, a.z, a.w};
        if (p.out_kind == 1) {
            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + off;
            if (full) {
                *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w));
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (col + j < p.N) o[j] = __float2bfloat16_rn(v[j]);
            }
        } else {  // fp32, or raw s32 bits
            float* o = static_cast<float*>(p.out) + off;
            if (full) {
                *reinterpret_cast<float4*>(o) = a;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (col + j < p.N) o[j] = v[j];
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
    // A/B type: kind::i8 1 = signed; kind::f8f6f4 0 = E4M3, and for FP6 E3M2
    // held in bits 7:2 of each byte the type code 2 -- measured on this B200
    // (tools/fp6_probe.py: code 2 with MSB-aligned E3M2 reproduces every
    // 64 x 64 code product exactly; the other codes / alignments do not)
    return (uint32_t)((fmt == FMT_INT8 ? 2u : 1u) << 4)                           // D format: s32 / f32
           | (uint32_t)((fmt == FMT_INT8 ? 1u : fmt == FMT_E3M2 ? 2u : 0u) << 7)  // A
           | (uint32_t)((fmt == FMT_INT8 ? 1u : fmt == FMT_E3M2 ? 2u : 0u) << 10) // B
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

template <int FMT, int CG>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmH, GemmArgs p) {
    using C = GemmCfg<CG>;
    // SwiGLU epilogue: one operand stage fewer, its smem doubles the
    // epilogue staging (u and h boxes side by side)
    const bool glu = p.glu_g != nullptr && !p.glu_res;
    const int STAGES = glu ? C::STAGES - 1 : C::STAGES;
    const int stg_bytes = glu ? 2 * STG_BYTES : STG_BYTES;
    constexpr int B_STAGE_BYTES = C::B_STAGE_BYTES;
    extern __shared__ uint8_t smem_raw[];
    // 1024 B alignment (128 B swizzle atoms) by pointer arithmetic on the
    // __shared__ array, so generic-pointer accesses stay LDS/STS (identical
    // offsets in both CTAs of a pair, as cta_group::2 requires)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
    // epilogue staging (1 KB aligned: 128 B-swizzled TMA-store boxes), then barriers
    float* stg = reinterpret_cast<float*>(sB + STAGES * B_STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES + stg_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = bars + 2 * STAGES + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;  // pair (cluster) index
    const int mt = (p.M + C::TILE_M - 1) / C::TILE_M, nt = (p.N + BN - 1) / BN;
    const int ntiles = mt * nt;
    const int nkb = (p.K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        // shard maps were written to global memory by the host (copy
        // engine): acquire them for the tensormap proxy before first use
        for (int i = 0; i < p.a_shards; ++i)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p.a_maps + i) : "memory");
        for (int i = 0; i < p.b_shards; ++i)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p.b_maps + i) : "memory");
        for (int i = 0; i < p.c_parts; ++i)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p.c_maps + i) : "memory");
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], EPI_WARPS * CG);  // every epilogue warp of the pair
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote signal
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // setup above overlaps the previous kernel's tail (PDL); no global
    // access before this point
    pdl_wait();
    pdl_trigger();

    if (warp == 0) {
        // ============================ TMA producer (both CTAs of a pair)
        if (lane == 0) {
            // pair mode: bytes of BOTH CTAs complete on the leader's barrier,
            // which alone carries the expect_tx
            const uint32_t full_leader0 = CG == 2 ? mapa_rank(&full[0], 0) : 0u;
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                int mb, nb;
                tile_coords(t, mt, nt, mb, nb);
                const int m0 = mb * C::TILE_M + (int)rank * BM, n0 = nb * BN + (int)rank * C::B_ROWS;
                // operand shards split along M / N: fixed for the tile
                const CUtensorMap* mapA = &tmA;
                const CUtensorMap* mapB = &tmB;
                int am = m0, bn = n0;
                if (p.a_shards && !p.a_along_k) {
                    const int i = m0 / p.a_len;
                    mapA = p.a_maps + i;
                    am = m0 - i * p.a_len;
                }
                if (p.b_shards && !p.b_along_k) {
                    const int i = n0 / p.b_len;
                    mapB = p.b_maps + i;
                    bn = n0 - i * p.b_len;
                }
                for (int kb = 0; kb < nkb; ++kb) {
                    const int k0 = kb * BK;
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a_dst = sA + stage * A_STAGE_BYTES;
                    uint8_t* b_dst = sB + stage * B_STAGE_BYTES;
                    if constexpr (CG == 2) {
                        if (leader) mbar_expect_tx(&full[stage], 2 * (A_STAGE_BYTES + B_STAGE_BYTES));
                        const uint32_t fb = full_leader0 + stage * 8;
                        // operand shards split along K: the k-block's part
                        const CUtensorMap* ma = mapA;
                        const CUtensorMap* mb = mapB;
                        int ak = k0, bk = k0;
                        if (p.a_shards && p.a_along_k) {
                            const int i = k0 / p.a_len;
                            ma = p.a_maps + i;
                            ak = k0 - i * p.a_len;
                        }
                        if (p.b_shards && p.b_along_k) {
                            const int i = k0 / p.b_len;
                            mb = p.b_maps + i;
                            bk = k0 - i * p.b_len;
                        }
                        if (p.a_kmajor) tma_load_2d_2sm(a_dst, ma, fb, ak, am);
                        else tma_load_2d_2sm(a_dst, ma, fb, am, ak);
                        if (p.b_kmajor) tma_load_2d_2sm(b_dst, mb, fb, bk, bn);
                        else tma_load_2d_2sm(b_dst, mb, fb, bn, bk);
                    } else {
                        mbar_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
                        if (p.a_kmajor) tma_load_2d(a_dst, &tmA, &full[stage], k0, m0);
                        else tma_load_2d(a_dst, &tmA, &full[stage], m0, k0);
                        if (p.b_kmajor) {
                            tma_load_2d(b_dst, &tmB, &full[stage], k0, n0);
                        } else {
                            tma_load_2d(b_dst, &tmB, &full[stage], n0, k0);
                            tma_load_2d(b_dst + B_STAGE_BYTES / 2, &tmB, &full[stage], n0 + 128, k0);
                        }
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer (the leader CTA of a pair)
        if (lane == 0 && leader) {
            const uint32_t idesc = make_idesc(FMT, !p.a_kmajor, !p.b_kmajor, C::TILE_M, BN);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = cid; t < ntiles; t += ncl, ++local) {
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
                                                       : make_desc(b_addr + k * 4096, 128 * BK, 1024);
                        tc_mma<FMT, CG>(tmem_d, ad, bd, idesc, (kb | k) ? 1u : 0u);
                    }
                    // smem stage free (in both CTAs) once these MMAs retire
                    if constexpr (CG == 2) tc_commit_mc2(&empty[stage]);
                    else tc_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if constexpr (CG == 2) tc_commit_mc2(&tfull[acc]);  // accumulator complete (both halves)
                else tc_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        // ============================ epilogue (8 warps)
        // warp w reads TMEM lanes 32*(w%4).. (its row quadrant q) and owns the
        // column half h of the 256-column accumulator
        const int ew = warp - 4;
        const int q = ew & 3, h = ew >> 2;
        float* S = stg + ew * (glu ? 2 : 1) * (32 * 32);
        const float sa = *p.sa, sb = *p.sb;
        const double ss = (double)sa * (double)sb;
        const float ssf = (float)ss;
        // ss = s_hi + s_lo exactly (a product of two floats has <= 48 bits)
        const float s_hi = __fmul_rn(sa, sb), s_lo = __fmaf_rn(sa, sb, -s_hi);
        // raw accumulator -> output value.  INT8: the reference's
        // float(double(acc) * (double(sa) * double(sb))) (quantize.hpp:356-370)
        // on the fp32 pipe: for |acc| < 2^24, P = acc*s_hi + acc*s_lo as p + t
        // (t's rounding error <= 2^-47 |p|), c = RN(p + t), certified when the
        // residual P - c lies more than 2^-16 half-ulps inside the rounding
        // interval (then neither the fp32 rounding nor the reference's
        // intermediate fp64 rounding, 2^-53, can land elsewhere).  A lane
        // with an uncertified element (about 2^-16 of them, |acc| >= 2^24, or
        // acc == 0) redoes its 32 values with the fp64 formula.
        auto cvt = [&](const uint32_t (&r)[32], float (&v)[32], int row_, int col0_) {
            if (p.out_kind == 2) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                return;
            }
            if (p.sa_vec || p.sb_vec) {
                // per-row / per-column scales: the same formula with the
                // element's scale pair, float(double(acc) * (double(sa_i) * double(sb_j)))
                const float sai = p.sa_vec ? (row_ < p.M ? __ldg(p.sa_vec + row_) : 0.f) : sa;
                if constexpr (FMT == FMT_INT8) {
                    int viol = -1;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float sbj = p.sb_vec ? (col0_ + j < p.N ? __ldg(p.sb_vec + col0_ + j) : 0.f) : sb;
                        const float shi = __fmul_rn(sai, sbj), slo = __fmaf_rn(sai, sbj, -shi);
                        const int A = (int)r[j];
                        const float af = __int2float_rn(A);
                        const float pp = __fmul_rn(af, shi);
                        const float t = __fmaf_rn(af, slo, __fmaf_rn(af, shi, -pp));
                        const float c = __fadd_rn(pp, t);
                        const float rr = __fadd_rn(__fadd_rn(pp, -c), t);
                        const int thr = (int)(__float_as_uint(c) & 0x7F800000u) - (24 << 23) - 0x100;
                        viol = max(viol, max((int)(__float_as_uint(rr) & 0x7FFFFFFFu) - thr, abs(A) - 0xFFFFFF));
                        v[j] = c;
                    }
                    if (viol >= 0) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float sbj = p.sb_vec ? (col0_ + j < p.N ? __ldg(p.sb_vec + col0_ + j) : 0.f) : sb;
                            v[j] = (float)((double)(int32_t)r[j] * ((double)sai * (double)sbj));
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float sbj = p.sb_vec ? (col0_ + j < p.N ? __ldg(p.sb_vec + col0_ + j) : 0.f) : sb;
                        v[j] = __uint_as_float(r[j]) * __fmul_rn(sai, sbj);
                    }
                }
                return;
            }
            if constexpr (FMT == FMT_INT8) {
                // pairs on the packed fp32 pipe (FMUL2/FFMA2/FADD2); per element
                // the integer test |rr| < half-ulp(c) * (1 - 2^-16)
                int viol = -1;    // max of (|rr| bits - threshold bits)
                float amx = 0.f;  // max |acc| (exactness of RN(acc) needs |acc| < 2^24)
                const float2 shi2 = make_float2(s_hi, s_hi), slo2 = make_float2(s_lo, s_lo);
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    const float2 af = make_float2(__int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]));
                    const float2 pp = __fmul2_rn(af, shi2);
                    const float2 e = __ffma2_rn(af, shi2, make_float2(-pp.x, -pp.y));  // exact product error
                    const float2 t = __ffma2_rn(af, slo2, e);
                    const float2 c = __fadd2_rn(pp, t);
                    const float2 rr = __fadd2_rn(__fadd2_rn(pp, make_float2(-c.x, -c.y)), t);  // pp - c exact
                    const int d0 = (int)(__float_as_uint(rr.x) & 0x7FFFFFFFu) -
                                   (int)(__float_as_uint(c.x) & 0x7F800000u) + ((24 << 23) + 0x100);
                    const int d1 = (int)(__float_as_uint(rr.y) & 0x7FFFFFFFu) -
                                   (int)(__float_as_uint(c.y) & 0x7F800000u) + ((24 << 23) + 0x100);
                    viol = max(viol, max(d0, d1));
                    amx = fmaxf(amx, fmaxf(fabsf(af.x), fabsf(af.y)));
                    v[j] = c.x;
                    v[j + 1] = c.y;
                }
                if (viol >= 0 || amx >= 16777216.0f) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = (float)((double)(int32_t)r[j] * ss);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * ssf;
            }
        };
        // 32 final values of this lane's row, columns col0..col0+31 (chunk c
        // of the tile) -> C.  TMA path: stage a 32-row x 128 B box (fp32: one
        // chunk; bf16: chunks c, c+1 side by side) 128 B-swizzled, then one
        // elected lane issues the bulk tensor store.
        auto store_chunk = [&](const float (&v)[32], int c, int row0_, int col0) {
            if (p.dbg_skip_epi == 7) {
                // timing experiment: direct per-lane row stores (no smem staging)
                const int rr_ = row0_ + lane;
                if (rr_ < p.M) {
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        float o[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) o[j] = v[8 * g + j];
                        if (p.out_kind == 1) store8(static_cast<__nv_bfloat16*>(p.out) + (int64_t)rr_ * p.N + col0 + 8 * g, o);
                        else {
                            float* d = static_cast<float*>(p.out) + (int64_t)rr_ * p.N + col0 + 8 * g;
                            reinterpret_cast<float4*>(d)[0] = make_float4(o[0], o[1], o[2], o[3]);
                            reinterpret_cast<float4*>(d)[1] = make_float4(o[4], o[5], o[6], o[7]);
                        }
                    }
                }
                return;
            }
            if (p.tma_store) {
                uint4* R = reinterpret_cast<uint4*>(S) + lane * 8;
                if (p.out_kind == 1) {
                    if ((c & 1) == 0) {
                        if (lane == 0) bulk_wait_read0();
                        __syncwarp();
                    }
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        R[(4 * (c & 1) + g) ^ (lane & 7)] =
                            make_uint4(pack_bf16x2(v[8 * g], v[8 * g + 1]), pack_bf16x2(v[8 * g + 2], v[8 * g + 3]),
                                       pack_bf16x2(v[8 * g + 4], v[8 * g + 5]), pack_bf16x2(v[8 * g + 6], v[8 * g + 7]));
                    if (c & 1) {
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmC, S, col0 - 32, row0_);
                            bulk_commit();
                        }
                    }
                } else {
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        R[k ^ (lane & 7)] = make_uint4(__float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                                                       __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3]));
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (p.c_parts) {  // the owner's receive slot (fp32 partial of this rank)
                            const int i = row0_ / p.c_len;
                            tma_store_2d(p.c_maps + i, S, col0, row0_ - i * p.c_len);
                        } else {
                            tma_store_2d(&tmC, S, col0, row0_);
                        }
                        bulk_commit();
                    }
                }
            } else {
#pragma unroll
                for (int g = 0; g < 4; ++g) stg_put(S, lane, g, v + 8 * g);
                __syncwarp();
                stg_flush(p, S, lane, row0_, col0, 8);
                __syncwarp();
            }
        };
        const uint32_t tempty_leader0 = CG == 2 ? mapa_rank(&tempty[0], 0) : 0u;
        int local = 0;
        for (int t = cid; t < ntiles; t += ncl, ++local) {
            int mb, nb;
            tile_coords(t, mt, nt, mb, nb);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            const int row0 = mb * C::TILE_M + (int)rank * BM + q * 32;
            const int row = row0 + lane;
            // SwiGLU epilogue: this lane's row of g, the first chunk fetched
            // while the tile's mainloop still runs (rows >= M read row M-1;
            // their outputs are clipped by the TMA store)
            // (two chunks in flight: chunk i+2's load issues when chunk i is consumed)
            const uint4* grow = nullptr;
            uint4 gq[2][4];
            if (p.glu_g) {
                grow = reinterpret_cast<const uint4*>(p.glu_g + (int64_t)min(row, p.M - 1) * p.N + nb * BN) + 16 * h;
#pragma unroll
                for (int k = 0; k < 8; ++k) gq[k >> 2][k & 3] = __ldg(grow + k);
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
            if (p.dbg_skip_epi == 1) {
            } else if (p.glu_g) {
                // ---- SwiGLU epilogue: u = the bf16 output, h = silu(g) * u
                // exactly as k_swiglu_fwd computes it from bf16 g and u; u and
                // h leave as 32-row x 128 B boxes (chunks c, c+1) from the two
                // 4 KB halves of the warp's staging buffer
                uint4* RU = reinterpret_cast<uint4*>(S) + lane * 8;
                uint4* RH = RU + 256;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int c = 4 * h + i;
                    uint4 gc[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) gc[k] = gq[i & 1][k];
                    if (i + 2 < 4 && p.dbg_skip_epi != 8) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) gq[i & 1][k] = __ldg(grow + 4 * (i + 2) + k);
                    }
                    uint32_t r[32];
                    tmem_ld32(tacc + c * 32, r);
                    float v[32];
                    cvt(r, v, row, nb * BN + c * 32);
                    if ((c & 1) == 0) {
                        if (lane == 0) bulk_wait_read0();
                        __syncwarp();
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t gw[4] = {gc[k].x, gc[k].y, gc[k].z, gc[k].w};
                        uint32_t uw[4], hw[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uw[j] = pack_bf16x2(v[8 * k + 2 * j], v[8 * k + 2 * j + 1]);
                            if (p.glu_res)  // y = RN(res + RN(acc))
                                uw[j] = pack_bf16x2(__uint_as_float(gw[j] << 16) + __uint_as_float(uw[j] << 16),
                                                    __uint_as_float(gw[j] & 0xFFFF0000u) +
                                                        __uint_as_float(uw[j] & 0xFFFF0000u));
                            else if (p.dbg_skip_epi == 9)  // timing experiment: no silu
                                hw[j] = uw[j] ^ gw[j];
                            else
                                hw[j] = pack_bf16x2(swiglu_fwd1(__uint_as_float(gw[j] << 16), __uint_as_float(uw[j] << 16)),
                                                    swiglu_fwd1(__uint_as_float(gw[j] & 0xFFFF0000u),
                                                                __uint_as_float(uw[j] & 0xFFFF0000u)));
                        }
                        const int slot = (4 * (c & 1) + k) ^ (lane & 7);
                        RU[slot] = make_uint4(uw[0], uw[1], uw[2], uw[3]);
                        if (!p.glu_res) RH[slot] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    }
                    if (c & 1) {
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmC, S, nb * BN + (c - 1) * 32, row0);
                            if (!p.glu_res) tma_store_2d(&tmH, S + 1024, nb * BN + (c - 1) * 32, row0);
                            bulk_commit();
                        }
                    }
                }
            } else if (p.dbg_skip_epi == 4) {
                // timing experiment: TMEM loads + conversion, no stores
                uint32_t x = 0;
#pragma unroll 1
                for (int c = 4 * h; c < 4 * h + 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tacc + c * 32, r);
                    float v[32];
                    cvt(r, v, row, nb * BN + c * 32);
#pragma unroll
                    for (int j = 0; j < 32; ++j) x ^= __float_as_uint(v[j]);
                }
                if (x == 0x9E3779B9u) static_cast<int*>(p.out)[0] = 1;
            } else if (p.dbg_skip_epi == 5) {
                // timing experiment: TMEM loads + staging + stores of the raw bits, no conversion
#pragma unroll 1
                for (int c = 4 * h; c < 4 * h + 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tacc + c * 32, r);
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
#pragma unroll
                    for (int g = 0; g < 4; ++g) stg_put(S, lane, g, v + 8 * g);
                    __syncwarp();
                    stg_flush(p, S, lane, row0, nb * BN + c * 32, 8);
                    __syncwarp();
                }
            } else if (p.xf_lb > 0) {
                // ---- fused FWHT along N (hadamard.hpp:136-177 order): pass 1
                // runs stages len = 1..16 on each 32-column chunk (this warp's
                // 4 chunks) and parks the fp32 result back in TMEM; pass 2
                // gathers 8 columns from each of the 8 chunks (tcgen05.ld x8;
                // this warp's 2 of the 4 column groups) for len = 32, 64, 128.
                const int B = 1 << p.xf_lb;
                const bool two_pass = B > 32;
#pragma unroll 1
                for (int c = 4 * h; c < 4 * h + 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tacc + c * 32, r);
                    float v[32];
                    cvt(r, v, row, nb * BN + c * 32);
#pragma unroll
                    for (int j = 0; j < 32; j += 2) ep_bfly(v[j], v[j + 1]);  // len 1 (B >= 2)
#pragma unroll
                    for (int tt = 1; tt < 5; ++tt) {
                        const int len = 1 << tt;
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
                        for (int j = 0; j < 32; ++j) v[j] *= p.xf_norm;
                        if (p.out_trans) {
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                float o[8];
#pragma unroll
                                for (int j = 0; j < 8; ++j) o[j] = v[8 * g + j];
                                ep_store8(p, row, nb * BN + c * 32 + 8 * g, o);
                            }
                        } else {
                            store_chunk(v, c, row0, nb * BN + c * 32);
                        }
                    }
                }
                if (two_pass) {
                    tmem_wait_st();
                    // both column halves of this row quadrant must be in TMEM
                    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
#pragma unroll 1
                    for (int g = 2 * h; g < 2 * h + 2; ++g) {
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
                        for (int tt = 0; tt < 3; ++tt) {
                            const int hh = 1 << tt;
                            if ((32 << tt) < B) {
#pragma unroll
                                for (int c = 0; c < 8; ++c)
                                    if ((c & hh) == 0)
#pragma unroll
                                        for (int j = 0; j < 8; j += 2)
                                            ep_bfly2(u[c][j], u[c][j + 1], u[c + hh][j], u[c + hh][j + 1]);
                            }
                        }
#pragma unroll
                        for (int c = 0; c < 8; ++c)
#pragma unroll
                            for (int j = 0; j < 8; ++j) u[c][j] *= p.xf_norm;
                        if (p.out_trans) {
#pragma unroll
                            for (int c = 0; c < 8; ++c) ep_store8(p, row, nb * BN + c * 32 + 8 * g, u[c]);
                        } else {
                            // final values back into TMEM; pass 3 stores whole chunks
#pragma unroll
                            for (int c = 0; c < 8; ++c) tmem_st8(tacc + c * 32 + g * 8, u[c]);
                        }
                    }
                    if (!p.out_trans) {
                        tmem_wait_st();
                        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
#pragma unroll 1
                        for (int c = 4 * h; c < 4 * h + 4; ++c) {
                            uint32_t r[32];
                            tmem_ld32(tacc + c * 32, r);
                            float v[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                            store_chunk(v, c, row0, nb * BN + c * 32);
                        }
                    }
                }
            } else {
                // ---- plain epilogue: this warp's 4 chunks of 32 columns
#pragma unroll 1
                for (int c = 4 * h; c < 4 * h + 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(tacc + c * 32, r);
                    float v[32];
                    cvt(r, v, row, nb * BN + c * 32);
                    store_chunk(v, c, row0, nb * BN + c * 32);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader0 + acc * 8);
                else mbar_arrive(&tempty[acc]);
            }
        }
        if (lane == 0) bulk_wait0();  // staged boxes fully written before the CTA leaves
    }

    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();  // no CTA leaves while its peer may still signal it
    tc_fence_after();
    if (warp == 2) {
        if constexpr (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
        else
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

// 2-D tensor map, no swizzle, zero OOB fill: `inner` contiguous elements per
// row, `outer` rows `row_bytes` apart, box {box_inner, box_outer}
bool encode_2d_plain(CUtensorMap* map, int dtype, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                     uint32_t box_inner, uint32_t box_outer) {
    auto enc = get_encode();
    if (!enc) return false;
    const CUtensorMapDataType dt = dtype == 0   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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
    return run_gemm_v(fmt, A, B, M, N, K, a_kmajor, b_kmajor, sa, nullptr, sb, nullptr, out, out_kind, xf_lb, xf_norm,
                      out_trans, n_valid, st);
}

namespace {
thread_local const ShardSpec* t_shard_a = nullptr;
thread_local const ShardSpec* t_shard_b = nullptr;
thread_local const ScatterSpec* t_scatter_c = nullptr;
}  // namespace

ShardScope::ShardScope(const ShardSpec* a, const ShardSpec* b, const ScatterSpec* c) {
    t_shard_a = a;
    t_shard_b = b;
    t_scatter_c = c;
}
ShardScope::~ShardScope() {
    t_shard_a = nullptr;
    t_shard_b = nullptr;
    t_scatter_c = nullptr;
}
bool ShardScope::active() { return t_shard_a || t_shard_b || t_scatter_c; }

namespace {
thread_local const void* t_glu_g = nullptr;
thread_local void* t_glu_h = nullptr;
thread_local bool t_glu_used = false;
}  // namespace
GluScope::GluScope(const void* g, void* h) {
    t_glu_g = g;
    t_glu_h = h;
    t_glu_used = false;
}
GluScope::~GluScope() {
    t_glu_g = nullptr;
    t_glu_h = nullptr;
}
bool GluScope::used() { return t_glu_used; }

bool encode_scatter_maps(void* const* recv, int parts, int slot, int64_t len, int64_t cols, CUtensorMap* out) {
    auto enc = get_encode();
    if (!enc) return false;
    for (int i = 0; i < parts; ++i) {
        float* base = static_cast<float*>(recv[i]) + (int64_t)slot * len * cols;
        const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)len};
        const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
        const cuuint32_t box[2] = {32, 32};
        const cuuint32_t estr[2] = {1, 1};
        if (enc(&out[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

bool encode_shard_maps(const uint8_t* const* parts, int n, int64_t inner, int64_t rows, CUtensorMap* out) {
    for (int i = 0; i < n; ++i)
        if (!encode_map(&out[i], parts[i], (uint64_t)inner, (uint64_t)rows, 128)) return false;
    return true;
}

int run_gemm_v(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
               int b_kmajor, const float* sa, const float* sa_vec, const float* sb, const float* sb_vec, void* out,
               int out_kind, int xf_lb, float xf_norm, int out_trans, int64_t n_valid, cudaStream_t st) {
    fmt = code_format(fmt);
    if ((sa_vec || sb_vec) && (xf_lb > 0 || out_trans || out_kind == 2)) return -1;
    const ShardSpec* sha = t_shard_a;
    const ShardSpec* shb = t_shard_b;
    const ScatterSpec* scc = t_scatter_c;
    // scattered C: fp32, row-major, every 32-row TMA box inside one part
    if (scc && (out_kind != 0 || out_trans || sa_vec || sb_vec || scc->parts < 1 || scc->len % 256 ||
                (int64_t)scc->parts * scc->len != M || (N * 4) % 16))
        return -1;
    static const float kOne = 1.0f;
    static float* d_one = nullptr;
    if (!sa || !sb) {  // vector-only call: the tensor scale slot still needs a valid device word
        if (!d_one) {
            cudaMalloc(&d_one, sizeof(float));
            cudaMemcpy(d_one, &kOne, sizeof(float), cudaMemcpyHostToDevice);
        }
        if (!sa) sa = d_one;
        if (!sb) sb = d_one;
    }
    if (xf_lb < 0 || xf_lb > 8) return -1;  // the 256-column tile must hold whole blocks
    if ((xf_lb > 0 || out_trans) && out_kind == 2) return -1;
    if (M <= 0 || N <= 0 || K <= 0) return -1;
    if (M > INT32_MAX / 2 || N > INT32_MAX / 2 || K > INT32_MAX / 2) return -1;
    // TMA: global strides must be multiples of 16 bytes
    if ((a_kmajor ? K : M) % 16 != 0 || (b_kmajor ? K : N) % 16 != 0) return -1;
    if (out_kind == 2 && fmt != FMT_INT8) return -1;
    GemmArgs args{(int)M, (int)N, (int)K, a_kmajor, b_kmajor, fmt, out_kind, sa, sb, out,
                  xf_lb, xf_norm, out_trans, (int)(n_valid < N ? n_valid : N), 0, 0, sa_vec, sb_vec};
    static const int dbg = [] {
        const char* e = getenv("HALO_GEMM_DEBUG_SKIP_EPI");
        return e ? atoi(e) : 0;
    }();
    args.dbg_skip_epi = dbg;

    // HALO_GEMM_CG=1 pins the single-CTA kernel (A/B runs)
    static const int cg_env = [] {
        const char* e = getenv("HALO_GEMM_CG");
        return e ? atoi(e) : 2;
    }();
    const int cg = (cg_env == 1 || num_sms() < 2) ? 1 : 2;
    CUtensorMap ma, mb;
    const int b_box = BN / cg;
    // sharded operands: the parts' maps (box 128 x 128) replace tmA / tmB;
    // every tile / k-block must fall inside one part
    auto shard_ok = [&](const ShardSpec* sh, int64_t mn, int tile) {
        if (!sh) return true;
        if (cg != 2 || sh->n < 1 || sh->n > 64 || sh->len <= 0) return false;
        const int64_t total = sh->along_k ? K : mn;
        return (int64_t)sh->n * sh->len == total && sh->len % (sh->along_k ? BK : tile) == 0;
    };
    if (!shard_ok(sha, M, BM * 2) || !shard_ok(shb, N, BN)) return -1;
    const bool ok_a = sha ? true : a_kmajor ? encode_map(&ma, A, K, M, BM) : encode_map(&ma, A, M, K, BK);
    const bool ok_b = shb ? true : b_kmajor ? encode_map(&mb, B, K, N, b_box) : encode_map(&mb, B, N, K, BK);
    if (!ok_a || !ok_b) return -2;
    if (sha) ma = sha->maps_host0;
    if (sha) args.a_maps = sha->maps, args.a_shards = sha->n, args.a_len = (int)sha->len, args.a_along_k = sha->along_k;
    if (shb) mb = shb->maps_host0;
    if (shb) args.b_maps = shb->maps, args.b_shards = shb->n, args.b_len = (int)shb->len, args.b_along_k = shb->along_k;
    // C via TMA stores when the row pitch is a multiple of 16 B (HALO_GEMM_TMA_STORE=0 disables)
    static const int tma_store_env = [] {
        const char* e = getenv("HALO_GEMM_TMA_STORE");
        return e ? atoi(e) : 1;
    }();
    CUtensorMap mc, mh;
    std::memset(&mc, 0, sizeof(mc));
    std::memset(&mh, 0, sizeof(mh));
    const int esz = out_kind == 1 ? 2 : 4;
    args.tma_store = 0;
    if (t_glu_g) {
        // SwiGLU epilogue: u and h as 32-row x 128 B boxes (128 B swizzle)
        // (t_glu_h null: the residual epilogue, C only)
        if (out_kind != 1 || out_trans || xf_lb || scc || N % BN || (uintptr_t)out % 16 ||
            (uintptr_t)t_glu_g % 16 || (uintptr_t)t_glu_h % 16 || !tma_store_env)
            return -1;
        auto enc = get_encode();
        const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        const cuuint64_t strides[1] = {(cuuint64_t)N * 2};
        const cuuint32_t box[2] = {64, 32};
        const cuuint32_t estr[2] = {1, 1};
        for (int i = 0; i < (t_glu_h ? 2 : 1); ++i)
            if (!enc || enc(i ? &mh : &mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, i ? t_glu_h : out, dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return -2;
        args.tma_store = 1;
        args.glu_g = static_cast<const __nv_bfloat16*>(t_glu_g);
        args.glu_res = t_glu_h ? 0 : 1;
        t_glu_used = true;
    } else if (scc) {
        mc = scc->maps_host0;
        args.tma_store = 1;
        args.c_maps = scc->maps;
        args.c_parts = scc->parts;
        args.c_len = (int)scc->len;
    } else if (tma_store_env && !out_trans && ((int64_t)N * esz) % 16 == 0 && (uintptr_t)out % 16 == 0) {
        auto enc = get_encode();
        const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        const cuuint64_t strides[1] = {(cuuint64_t)N * esz};
        const cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 32};
        const cuuint32_t estr[2] = {1, 1};
        const CUtensorMapDataType dt = out_kind == 1   ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                       : out_kind == 2 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        if (enc && enc(&mc, dt, 2, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
            args.tma_store = 1;
    }
    const int64_t tile_m = (int64_t)BM * cg;
    const int tiles = (int)(((M + tile_m - 1) / tile_m) * ((N + BN - 1) / BN));
    if (cg == 1) {
        const int grid = tiles < num_sms() ? tiles : num_sms();
        auto kern = fmt == FMT_INT8 ? k_gemm<FMT_INT8, 1> : fmt == FMT_E3M2 ? k_gemm<FMT_E3M2, 1> : k_gemm<FMT_E4M3, 1>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem<1>());
        kern<<<grid, GEMM_THREADS, gemm_smem<1>(), st>>>(ma, mb, mc, mh, args);
    } else {
        auto kern = fmt == FMT_INT8 ? k_gemm<FMT_INT8, 2> : fmt == FMT_E3M2 ? k_gemm<FMT_E3M2, 2> : k_gemm<FMT_E4M3, 2>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem<2>());
        // persistent: as many co-resident pairs as the GPCs can host
        static int max_pairs[3] = {0, 0, 0};
        int& mp = max_pairs[fmt == FMT_INT8 ? 0 : fmt == FMT_E3M2 ? 2 : 1];
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(GEMM_THREADS, 1, 1);
        cfg.dynamicSmemBytes = gemm_smem<2>();
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (!mp) {
            cfg.gridDim = dim3(num_sms(), 1, 1);
            if (cudaOccupancyMaxActiveClusters(&mp, kern, &cfg) != cudaSuccess || mp < 1) mp = num_sms() / 2;
        }
        const int grid = 2 * (tiles < mp ? tiles : mp);
        cfg.gridDim = dim3(grid, 1, 1);
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mh, args);
        if (le != cudaSuccess) return (int)le;
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace halo_b200
