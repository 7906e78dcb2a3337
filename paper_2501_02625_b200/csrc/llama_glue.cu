// llama_glue.cu — the transformer-block glue around the HALO projections,
// one HBM pass each (the eager torch chains they replace launch 6-12 kernels
// apiece): RMSNorm forward / backward (with the gain gradient) and rotary
// position embedding applied to the fused qkv projection output.
//
// RMSNorm (rmsnorm.hpp:27-100): y = x * r * g, r = 1/sqrt(S/D + eps) with
// S = sum_j x_j^2 accumulated in double, D = dim when `mean` (Llama) or 1
// (the reference's x/||x||, eps 0).  In the reference form y (and dx) are
// evaluated in double as rmsnorm.hpp does (double(x) * r, then *
// double(g)); the Llama form multiplies in fp32.  Backward: dx_k = r g_k dy_k - (r^3 x_k / D) * sum_j g_j dy_j x_j
// (= rmsnorm_backward's (e' - x_hat <x_hat, e'>) / ||x|| for D = 1, eps 0),
// dg_j = sum_rows dy_j x_j r (rmsnorm_gain_gradient) via per-CTA partial rows
// reduced in a fixed order (deterministic).
//
// RoPE (Llama-3, theta 500000): on each query / key head of the qkv row
// [q heads | k heads | v heads] x head_dim, pairs (i, i + hd/2):
//   o1 = t1 c - t2 s,  o2 = t2 c + t1 s,   c, s = cos / sin(pos * inv_freq_i)
// in fp32 from a per-(position, i) fp32 table; v passes through.  Backward is
// the transpose rotation.
#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

namespace halo_b200 {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int NORM_WARPS = 8;

// one warp per row; a lane owns 8-element groups g = lane, lane + 32, ...
// EXACT (the reference form): y = float(double(x) * r * double(g)) as
// rmsnorm.hpp:38-42; otherwise (Llama) the fp32 product (x * r) * g.
// ADD: the input row is h = RN_bf16(x + res) (torch's bf16 add), written to
// hout and normalised -- the residual add fused into the norm's first pass.
template <typename OutT, bool EXACT, bool ADD = false>
__global__ void __launch_bounds__(32 * NORM_WARPS) k_rmsnorm_fwd(const __nv_bfloat16* __restrict__ x,
                                                                  const float* __restrict__ gain, OutT* __restrict__ y,
                                                                  float* __restrict__ rstd, int64_t rows, int dim,
                                                                  double div, double eps,
                                                                  const __nv_bfloat16* __restrict__ res = nullptr,
                                                                  __nv_bfloat16* __restrict__ hout = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * NORM_WARPS + (threadIdx.x >> 5);
    if (row >= rows) return;
    const __nv_bfloat16* xr = (ADD ? hout : x) + row * dim;  // pass 2 reads h back (this thread wrote it)
    double s = 0.0;
    for (int c = lane * 8; c < dim; c += 256) {
        float v[8];
        if constexpr (ADD) {
            float a[8], b[8];
            load8(x + row * dim + c, a);
            load8(res + row * dim + c, b);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(__float2bfloat16_rn(a[j] + b[j]));
            store8(hout + row * dim + c, v);
        } else {
            load8(xr + c, v);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) s += (double)v[j] * (double)v[j];
    }
    s = warp_sum(s);
    // a zero row with eps == 0 (rmsnorm.hpp:35-36 raises numeric_error) gives
    // r = inf and non-finite outputs, which the next HALO quantizer flags
    const double r = 1.0 / sqrt(s / div + eps);
    if (lane == 0 && rstd) rstd[row] = (float)r;
    const float rf = (float)r;
    OutT* yr = y + row * dim;
    for (int c = lane * 8; c < dim; c += 256) {
        float v[8], o[8];
        load8(xr + c, v);
        const float4 g0 = __ldg(reinterpret_cast<const float4*>(gain + c));
        const float4 g1 = __ldg(reinterpret_cast<const float4*>(gain + c) + 1);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (EXACT) o[j] = (float)(((double)v[j] * r) * (double)g[j]);
            else o[j] = (v[j] * rf) * g[j];
        }
        if constexpr (sizeof(OutT) == 2) store8(reinterpret_cast<__nv_bfloat16*>(yr + c), o);
        else store8(reinterpret_cast<float*>(yr + c), o);
    }
}

// A CTA owns BWD_ROWS rows.  Phase 1 (warp per row): dot = sum_j g dy x
// (double) and r -> shared memory.  Phase 2 (column-parallel, coalesced 16 B
// per thread and row): dx for every (row, column) and the gain-gradient
// partial sum over the CTA's rows in a fixed order (deterministic), written
// to part[blockIdx.x].  The second read of x / dy hits L2.  Phase 2 walks
// its rows UNROLL at a time with every load issued before the math, so a
// thread keeps 2 * UNROLL 16-byte requests in flight.
constexpr int BWD_ROWS = 8;
constexpr int BWD_UNROLL = 4;
// RES: dx = RN_bf16(RN_bf16(dx_norm) + dres) -- the autograd engine's bf16
// accumulation of the residual-stream gradient, fused into the store.
template <typename DyT, bool EXACT, bool RES = false>
__global__ void __launch_bounds__(32 * NORM_WARPS) k_rmsnorm_bwd(const __nv_bfloat16* __restrict__ x,
                                                                  const DyT* __restrict__ dy,
                                                                  const float* __restrict__ gain,
                                                                  const float* __restrict__ rstd,
                                                                  __nv_bfloat16* __restrict__ dx,
                                                                  float* __restrict__ part, int64_t rows, int dim,
                                                                  double div,
                                                                  const __nv_bfloat16* __restrict__ dres = nullptr) {
    __shared__ double kr[BWD_ROWS];
    __shared__ double rr[BWD_ROWS];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BWD_ROWS;
    const int nr = (int)(rows - row0 < BWD_ROWS ? rows - row0 : BWD_ROWS);
    for (int i = w; i < nr; i += NORM_WARPS) {
        const int64_t row = row0 + i;
        const __nv_bfloat16* xr = x + row * dim;
        const DyT* dr = dy + row * dim;
        double dot = 0.0;
        for (int c = lane * 8; c < dim; c += 256) {
            float v[8], d[8];
            load8(xr + c, v);
            load8(dr + c, d);
            const float4 g0 = __ldg(reinterpret_cast<const float4*>(gain + c));
            const float4 g1 = __ldg(reinterpret_cast<const float4*>(gain + c) + 1);
            const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
            for (int j = 0; j < 8; ++j) dot += (double)g[j] * (double)d[j] * (double)v[j];
        }
        dot = warp_sum(dot);
        if (lane == 0) {
            const double r = (double)rstd[row];
            rr[i] = r;
            kr[i] = r * r * r * dot / div;
        }
    }
    __syncthreads();
    for (int c = threadIdx.x * 8; c < dim; c += blockDim.x * 8) {
        const float4 g0 = __ldg(reinterpret_cast<const float4*>(gain + c));
        const float4 g1 = __ldg(reinterpret_cast<const float4*>(gain + c) + 1);
        const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        double accd[EXACT ? 8 : 1];
        if constexpr (EXACT) {
#pragma unroll
            for (int j = 0; j < 8; ++j) accd[j] = 0.0;
        }
        // rows in order (the gain-gradient partial sums stay deterministic)
        auto one_row = [&](int i, const float (&v)[8], const float (&d)[8], const float (&e)[8]) {
            const int64_t row = row0 + i;
            float o[8];
            const double r = rr[i], k = kr[i];
            const float rf = (float)r, kf = (float)k;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if constexpr (EXACT) {
                    o[j] = (float)(r * (double)g[j] * (double)d[j] - k * (double)v[j]);
                    accd[j] += (double)d[j] * (double)v[j] * r;
                } else {
                    o[j] = rf * g[j] * d[j] - kf * v[j];
                    acc[j] += d[j] * v[j] * rf;
                }
                if constexpr (RES) o[j] = __bfloat162float(__float2bfloat16_rn(o[j])) + e[j];
            }
            store8(dx + row * dim + c, o);
        };
        int i = 0;
        for (; i + BWD_UNROLL <= nr; i += BWD_UNROLL) {
            float v[BWD_UNROLL][8], d[BWD_UNROLL][8], e[BWD_UNROLL][RES ? 8 : 1];
#pragma unroll
            for (int u = 0; u < BWD_UNROLL; ++u) {
                load8(x + (row0 + i + u) * dim + c, v[u]);
                load8(dy + (row0 + i + u) * dim + c, d[u]);
                if constexpr (RES) load8(dres + (row0 + i + u) * dim + c, e[u]);
            }
#pragma unroll
            for (int u = 0; u < BWD_UNROLL; ++u) {
                float e8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if constexpr (RES)
#pragma unroll
                    for (int j = 0; j < 8; ++j) e8[j] = e[u][j];
                one_row(i + u, v[u], d[u], e8);
            }
        }
        for (; i < nr; ++i) {
            float v[8], d[8], e8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            load8(x + (row0 + i) * dim + c, v);
            load8(dy + (row0 + i) * dim + c, d);
            if constexpr (RES) load8(dres + (row0 + i) * dim + c, e8);
            one_row(i, v, d, e8);
        }
        if constexpr (EXACT) {
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = (float)accd[j];
        }
        store8(part + (int64_t)blockIdx.x * dim + c, acc);
    }
}

// dgain[c] = the partials summed in double, deterministically in two levels:
// level 1 sums each group of SUM_GROUP consecutive partials in order (every
// (group, column) a thread: the whole GPU streams the partials), level 2 the
// group sums in order (a short latency chain per column)
constexpr int SUM_GROUP = 16;
__global__ void __launch_bounds__(256) k_sum_rows1(const float* __restrict__ part, int nparts, int dim,
                                                   double* __restrict__ gsum) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= dim) return;
    const int i0 = blockIdx.y * SUM_GROUP, i1 = min(i0 + SUM_GROUP, nparts);
    float q[SUM_GROUP];
#pragma unroll
    for (int u = 0; u < SUM_GROUP; ++u) q[u] = i0 + u < i1 ? __ldg(part + (int64_t)(i0 + u) * dim + c) : 0.f;
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < SUM_GROUP; ++u)
        if (i0 + u < i1) s += (double)q[u];
    gsum[(int64_t)blockIdx.y * dim + c] = s;
}
__global__ void __launch_bounds__(64) k_sum_rows2(const double* __restrict__ gsum, int ngroups, int dim,
                                                  float* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= dim) return;
    double s = 0.0;
    int i = 0;
    for (; i + 16 <= ngroups; i += 16) {
        double q[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) q[u] = gsum[(int64_t)(i + u) * dim + c];
#pragma unroll
        for (int u = 0; u < 16; ++u) s += q[u];
    }
    for (; i < ngroups; ++i) s += gsum[(int64_t)i * dim + c];
    out[c] = (float)s;
}

// RoPE over the qkv rows: one thread per (row, head of q/k, 8-pair group)
__global__ void __launch_bounds__(256) k_rope(const __nv_bfloat16* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                              const float* __restrict__ cs, int64_t rows, int seq, int nrot,
                                              int nall, int hd, int backward) {
    const int half = hd / 2, groups = half / 8;
    const int64_t per_row = (int64_t)nall * groups;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * per_row) return;
    const int64_t row = idx / per_row;
    const int rem = (int)(idx % per_row);
    const int head = rem / groups, g = rem % groups;
    const int64_t base = row * (int64_t)nall * hd + (int64_t)head * hd + g * 8;
    float t1[8], t2[8], o1[8], o2[8];
    load8(in + base, t1);
    load8(in + base + half, t2);
    if (head < nrot) {
        const int pos = (int)(row % seq);
        const float* c = cs + ((int64_t)pos * half + g * 8) * 2;  // (cos, sin) pairs
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float cj = c[2 * j], sj = c[2 * j + 1];
            if (!backward) {
                o1[j] = t1[j] * cj - t2[j] * sj;
                o2[j] = t2[j] * cj + t1[j] * sj;
            } else {
                o1[j] = t1[j] * cj + t2[j] * sj;
                o2[j] = t2[j] * cj - t1[j] * sj;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            o1[j] = t1[j];
            o2[j] = t2[j];
        }
    }
    store8(out + base, o1);
    store8(out + base + half, o2);
}

}  // namespace

bool run_rmsnorm_fwd(const void* x, const float* gain, void* y, int y_dtype, float* rstd, int64_t rows, int dim,
                     bool mean, double eps, cudaStream_t st, const void* res, void* hout) {
    if (dim % 8 || dim <= 0 || (!res) != (!hout)) return false;
    const unsigned grid = (unsigned)((rows + NORM_WARPS - 1) / NORM_WARPS);
    const double div = mean ? (double)dim : 1.0;
    auto xp = static_cast<const __nv_bfloat16*>(x);
    auto rp = static_cast<const __nv_bfloat16*>(res);
    auto hp = static_cast<__nv_bfloat16*>(hout);
    // the reference form (x/||x||, eps 0) evaluates y in double like rmsnorm.hpp
    const bool exact = !mean;
#define HALO_NF(T, E, A) k_rmsnorm_fwd<T, E, A><<<grid, 32 * NORM_WARPS, 0, st>>>(xp, gain, static_cast<T*>(y), rstd, rows, dim, div, eps, rp, hp)
    if (res) {
        if (y_dtype != DT_BF16 || exact) return false;  // the Llama block form only
        HALO_NF(__nv_bfloat16, false, true);
    } else if (y_dtype == DT_BF16) {
        if (exact) HALO_NF(__nv_bfloat16, true, false); else HALO_NF(__nv_bfloat16, false, false);
    } else {
        if (exact) HALO_NF(float, true, false); else HALO_NF(float, false, false);
    }
#undef HALO_NF
    return true;
}

// floats: the per-CTA partials, then the level-1 group sums (doubles)
int64_t rmsnorm_bwd_scratch(int64_t rows, int dim) {
    const int64_t parts = (rows + BWD_ROWS - 1) / BWD_ROWS, groups = (parts + SUM_GROUP - 1) / SUM_GROUP;
    return parts * dim + 2 * groups * dim + 2;
}

bool run_rmsnorm_bwd(const void* x, const void* dy, int dy_dtype, const float* gain, const float* rstd, void* dx,
                     float* dgain, float* scratch, int64_t rows, int dim, bool mean, cudaStream_t st, const void* dres) {
    if (dim % 8 || dim <= 0) return false;
    const unsigned grid = (unsigned)((rows + BWD_ROWS - 1) / BWD_ROWS);
    const double div = mean ? (double)dim : 1.0;
    auto xp = static_cast<const __nv_bfloat16*>(x);
    auto dxp = static_cast<__nv_bfloat16*>(dx);
    auto rp = static_cast<const __nv_bfloat16*>(dres);
    const bool exact = !mean;
#define HALO_NB(T, E, R) k_rmsnorm_bwd<T, E, R><<<grid, 32 * NORM_WARPS, 0, st>>>(xp, static_cast<const T*>(dy), gain, rstd, dxp, scratch, rows, dim, div, rp)
    if (dres) {
        if (exact) return false;  // the Llama block form only
        if (dy_dtype == DT_BF16) HALO_NB(__nv_bfloat16, false, true); else HALO_NB(float, false, true);
    } else if (dy_dtype == DT_BF16) {
        if (exact) HALO_NB(__nv_bfloat16, true, false); else HALO_NB(__nv_bfloat16, false, false);
    } else {
        if (exact) HALO_NB(float, true, false); else HALO_NB(float, false, false);
    }
#undef HALO_NB
    const int groups = (int)((grid + SUM_GROUP - 1) / SUM_GROUP);
    // 8-byte aligned group sums after the partials
    double* gsum = reinterpret_cast<double*>(scratch + (((int64_t)grid * dim + 1) & ~(int64_t)1));
    k_sum_rows1<<<dim3((dim + 255) / 256, groups), 256, 0, st>>>(scratch, (int)grid, dim, gsum);
    k_sum_rows2<<<(dim + 63) / 64, 64, 0, st>>>(gsum, groups, dim, dgain);
    return true;
}

bool run_rope(const void* in, void* out, const float* cs, int64_t rows, int seq, int nrot, int nall, int hd,
              bool backward, cudaStream_t st) {
    if (hd % 16 || nrot > nall || seq <= 0) return false;
    const int64_t n = rows * (int64_t)nall * (hd / 16);
    if (n == 0) return true;
    k_rope<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(in),
                                                        static_cast<__nv_bfloat16*>(out), cs, rows, seq, nrot, nall,
                                                        hd, backward ? 1 : 0);
    return true;
}

}  // namespace halo_b200
