// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" shim over the UNMODIFIED reference headers at
// /root/reference/proj/include/halo (header-only C++20).  oracle/Makefile
// compiles this file against those headers where they lie (-I, no copy) into
// oracle/_ref/libhalo_ref.so.  It is used (a) to pin the C restatement in
// oracle/halo_oracle.c, (b) to generate tests/golden/*.npz, and (c) as the
// bench.py `--impl reference` CPU arm.  Nothing in the product links it.
//
// Block-size extension: a right transform with block B is the
// reference transform_right applied to the row-major buffer viewed as
// (rows*d/B) x B; a left transform with block B is transform_left applied to
// each contiguous B-row slab.  With B == d both are the reference verbatim.

#include <halo/hadamard.hpp>
#include <halo/halo_linear.hpp>
#include <halo/hqfsdp.hpp>
#include <halo/quantize.hpp>
#include <halo/rmsnorm.hpp>
#include <halo/tensor.hpp>

#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

using namespace halo;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const numeric_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Tensor make(const float* p, index_t r, index_t c) {
    Tensor t(r, c);
    if (r * c) std::memcpy(t.data(), p, sizeof(float) * size_t(r * c));
    return t;
}

void put(const Tensor& t, float* out) {
    if (t.size()) std::memcpy(out, t.data(), sizeof(float) * size_t(t.size()));
}

NumericFormat fmt_of(int f) { return static_cast<NumericFormat>(f); }

Granularity gran_of(int g) {
    switch (g) {
    case 1: return Granularity::row();
    case 2: return Granularity::column();
    case 4: return Granularity::mx();
    default: return Granularity::tensor();
    }
}

// right transform with block B (hadamard.hpp:194-197 on the reshaped view)
Tensor right_blocked(const Tensor& a, index_t block, bool ht) {
    const index_t B = block ? block : a.cols();
    Tensor v = make(a.data(), a.rows() * a.cols() / B, B);
    const HadamardSpec spec = build_spec(B);
    Tensor r = ht ? transform_right_ht(v, spec) : transform_right(v, spec);
    Tensor out(a.rows(), a.cols());
    put(r, out.data());
    return out;
}

// left transform with block B (hadamard.hpp:208-216 per B-row slab)
Tensor left_blocked(const Tensor& a, index_t block, bool h) {
    const index_t B = block ? block : a.rows();
    const HadamardSpec spec = build_spec(B);
    Tensor out(a.rows(), a.cols());
    for (index_t s = 0; s < a.rows(); s += B) {
        Tensor slab = make(a.row(s), B, a.cols());
        Tensor r = h ? transform_left_h(slab, spec) : transform_left(slab, spec);
        std::memcpy(out.row(s), r.data(), sizeof(float) * size_t(r.size()));
    }
    return out;
}

QuantizedTensor qt_from(const float* codes, index_t r, index_t c, int fmt, float scale) {
    QuantizedTensor q;
    q.format = fmt_of(fmt);
    q.granularity = Granularity::tensor();
    q.rows = r;
    q.cols = c;
    q.codes.assign(codes, codes + r * c);
    q.scales = {scale};
    return q;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_is_supported_hadamard_dim(long long d) { return is_supported_hadamard_dim(d) ? 1 : 0; }
long long ref_next_supported_hadamard_dim(long long d) { return next_supported_hadamard_dim(d); }

int ref_fwht_rows(float* a, long long rows, long long cols, long long block) {
    return guard([&] { put(right_blocked(make(a, rows, cols), block, false), a); });
}

int ref_fwht_rows_ht(float* a, long long rows, long long cols, long long block) {
    return guard([&] { put(right_blocked(make(a, rows, cols), block, true), a); });
}

int ref_fwht_cols(float* a, long long rows, long long cols, long long block) {
    return guard([&] { put(left_blocked(make(a, rows, cols), block, false), a); });
}

double ref_round_code(double x, int fmt) { return detail::round_code(x, fmt_of(fmt)); }

int ref_quantize(const float* a, long long rows, long long cols, int fmt, int gran, int supplied,
                 float* scales, float* codes) {
    return guard([&] {
        const Tensor t = make(a, rows, cols);
        std::vector<float> sv;
        QuantizedTensor q;
        if (supplied) {
            const index_t groups = detail::group_count(gran_of(gran), rows, cols);
            sv.assign(scales, scales + groups);
            q = quantize(t, fmt_of(fmt), gran_of(gran), &sv);
        } else {
            q = quantize(t, fmt_of(fmt), gran_of(gran));
        }
        std::memcpy(codes, q.codes.data(), sizeof(float) * q.codes.size());
        std::memcpy(scales, q.scales.data(), sizeof(float) * q.scales.size());
    });
}

// qmatmul(a, b, transpose_b) quantize.hpp:339-380 on per-tensor operands.
// A is M x K row-major codes; B is N x K (transpose_b) or K x N codes.
int ref_qmatmul(const float* A, const float* B, long long M, long long N, long long K,
                int transpose_b, int fmt, float sa, float sb, float* out) {
    return guard([&] {
        const QuantizedTensor qa = qt_from(A, M, K, fmt, sa);
        const QuantizedTensor qb = transpose_b ? qt_from(B, N, K, fmt, sb) : qt_from(B, K, N, fmt, sb);
        put(qmatmul(qa, qb, transpose_b != 0), out);
    });
}

// The HALO layer.  block == 0 (or == m with a batch the reference supports)
// runs HaloLinearLayer verbatim (halo_linear.hpp:227-462); otherwise the
// same sequence is composed from reference primitives with blocked
// transforms, following error_path / gradient_path line by line.
// gran 0 = Granularity::tensor(), 1 = ::row(), 2 = ::column() (quantize.hpp:73-80);
// sx / sw receive the first scale of each operand.
int ref_linear_g(int level, int fmt, long long block, int gran, long long b, long long m, long long n,
                 const float* X, const float* W, const float* EY, float* Y, float* EX, float* GW,
                 float* xq, float* sx, float* wq, float* sw) {
    return guard([&] {
        const Tensor x = make(X, b, m), w = make(W, n, m), ey = make(EY, b, n);
        const Granularity g = gran_of(gran);
        const HaloScheme scheme = level == 0 ? halo0(fmt_of(fmt), g) : level == 1 ? halo1(fmt_of(fmt), g)
                                                                                 : halo2(fmt_of(fmt), g);
        if (block == 0) {
            HaloLinearLayer layer(w, scheme);
            SavedContext ctx;
            put(layer.forward(x, ctx), Y);
            const auto back = layer.backward(ctx, ey);
            put(back.e_x, EX);
            put(back.grad_w, GW);
            std::memcpy(xq, ctx.xq.codes.data(), sizeof(float) * ctx.xq.codes.size());
            std::memcpy(wq, ctx.wq.codes.data(), sizeof(float) * ctx.wq.codes.size());
            *sx = ctx.xq.scales[0];
            *sw = ctx.wq.scales[0];
            return;
        }
        const NumericFormat f = fmt_of(fmt);
        // forward :288-299
        const QuantizedTensor qx = quantize(level ? right_blocked(x, block, false) : x, f, g);
        const QuantizedTensor qw = quantize(level ? right_blocked(w, block, false) : w, f, g);
        put(qmatmul(qx, qw, true), Y);
        // error path :381-413
        const QuantizedTensor qe = quantize(ey, f, g);
        Tensor prod;
        if (level == 2) {
            const index_t bp = (b + block - 1) / block * block;
            const Tensor padded = bp == b ? ey : pad_rows(ey, bp);
            const QuantizedTensor qeh = quantize(left_blocked(padded, block, true), f, g);
            prod = qmatmul(qeh, qw);
            prod = left_blocked(prod, block, false);
            if (prod.rows() != b) prod = take_rows(prod, b);
        } else {
            prod = qmatmul(qe, qw);
        }
        if (level >= 1) prod = right_blocked(prod, block, true);
        put(prod, EX);
        // gradient path :418-439
        // MX blocks do not transpose: quantize the transpose itself (:427-431)
        Tensor gw = qmatmul(g.kind == GranularityKind::MxBlock ? quantize(transpose(ey), f, g) : transpose_quantized(qe),
                            qx);
        if (level >= 1) gw = right_blocked(gw, block, true);
        put(gw, GW);
        std::memcpy(xq, qx.codes.data(), sizeof(float) * qx.codes.size());
        std::memcpy(wq, qw.codes.data(), sizeof(float) * qw.codes.size());
        *sx = qx.scales[0];
        *sw = qw.scales[0];
    });
}

int ref_linear(int level, int fmt, long long block, long long b, long long m, long long n,
               const float* X, const float* W, const float* EY, float* Y, float* EX, float* GW,
               float* xq, float* sx, float* wq, float* sw) {
    return ref_linear_g(level, fmt, block, 0, b, m, n, X, W, EY, Y, EX, GW, xq, sx, wq, sw);
}

// HQ-FSDP forward gather (hqfsdp.hpp:131-148, 204-237): codes of the padded
// rotated weight ((rows padded to a multiple of world) x cols), its global
// scale and the per-rank local absmaxes.
int ref_fsdp_gather(long long world, const float* W, long long rows, long long cols, int fmt,
                    int hadamard, float* codes, float* scale, double* local_absmax) {
    return guard([&] {
        WorldConfig wc;
        wc.world_size = world;
        auto p = shard(make(W, rows, cols), wc, fmt_of(fmt));
        CommLedger ledger;
        const QuantizedTensor q = quantized_all_gather(p, hadamard != 0, ledger);
        std::memcpy(codes, q.codes.data(), sizeof(float) * q.codes.size());
        *scale = q.scales[0];
        for (index_t r = 0; r < world; ++r) local_absmax[r] = p.local_absmax[size_t(r)];
        const QuantizedTensor again = backward_regather(p, hadamard != 0, ledger);
        if (again.codes != q.codes) throw std::logic_error("regather mismatch");
    });
}

// hqfsdp.hpp:271-300: grads is world x (rows x cols); shards out is
// world x (shard_rows x cols) with shard_rows = ceil(rows/world).
int ref_reduce_scatter(long long world, const float* grads, long long rows, long long cols,
                       float* shards_out) {
    return guard([&] {
        WorldConfig wc;
        wc.world_size = world;
        auto p = shard(Tensor(rows, cols), wc, NumericFormat::Int8);
        std::vector<Tensor> per;
        for (index_t r = 0; r < world; ++r) per.push_back(make(grads + r * rows * cols, rows, cols));
        CommLedger ledger;
        const auto shards = reduce_scatter_grads(per, p, ledger);
        for (index_t r = 0; r < world; ++r)
            put(shards[size_t(r)], shards_out + r * p.shard_rows * cols);
    });
}

// tensor.hpp:433-445
void ref_randn(float* out, long long n, unsigned long long seed, double stddev) {
    Rng rng(seed);
    for (long long i = 0; i < n; ++i) out[i] = static_cast<float>(rng.normal() * stddev);
}

// tensor.hpp:464-493 (columns or rows axis, explicit channels)
int ref_inject_outliers(float* a, long long rows, long long cols, const long long* channels,
                        long long nch, double mag, int axis_rows) {
    return guard([&] {
        OutlierProfile p;
        p.channels.assign(channels, channels + nch);
        p.magnification = mag;
        p.axis = axis_rows ? Axis::Rows : Axis::Columns;
        put(inject_outliers(make(a, rows, cols), p), a);
    });
}

// CPU baseline arm: `threads` independent copies of one HALO fwd+bwd on a
// (b x m -> n) sample, each on its own thread, through ref_linear.  Returns
// wall seconds for the whole batch of copies.
double ref_time_linear(int level, int fmt, long long block, long long b, long long m, long long n,
                       int threads) {
    auto work = [&](int t) {
        std::vector<float> X(size_t(b * m)), W(size_t(n * m)), EY(size_t(b * n)), Y(size_t(b * n)),
            EX(size_t(b * m)), GW(size_t(n * m)), xq(size_t(b * m)), wq(size_t(n * m));
        ref_randn(X.data(), b * m, 1 + 10 * t, 1.0);
        ref_randn(W.data(), n * m, 2 + 10 * t, 1.0 / std::sqrt(double(m)));
        ref_randn(EY.data(), b * n, 3 + 10 * t, 1e-3);
        float sx, sw;
        ref_linear(level, fmt, block, b, m, n, X.data(), W.data(), EY.data(), Y.data(), EX.data(),
                   GW.data(), xq.data(), &sx, wq.data(), &sw);
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

// write_quantized_tensor / read_quantized_tensor (quantize.hpp:405-474):
// codes as the reference's float code values, granularity kind 0/1/2
int ref_write_quantized(const char* path, int fmt, int gran, long long rows, long long cols, const float* codes,
                        const float* scales, long long nscales) {
    return guard([&] {
        QuantizedTensor q;
        q.format = static_cast<NumericFormat>(fmt);
        q.granularity.kind = static_cast<GranularityKind>(gran);
        q.rows = rows;
        q.cols = cols;
        q.codes.assign(codes, codes + rows * cols);
        q.scales.assign(scales, scales + nscales);
        write_quantized_tensor(std::string(path), q);
    });
}

int ref_read_quantized_info(const char* path, int* fmt, int* gran, long long* rows, long long* cols,
                            long long* nscales) {
    return guard([&] {
        const QuantizedTensor q = read_quantized_tensor(std::string(path));
        *fmt = static_cast<int>(q.format);
        *gran = static_cast<int>(q.granularity.kind);
        *rows = q.rows;
        *cols = q.cols;
        *nscales = static_cast<long long>(q.scales.size());
    });
}

int ref_read_quantized(const char* path, float* codes, float* scales) {
    return guard([&] {
        const QuantizedTensor q = read_quantized_tensor(std::string(path));
        std::memcpy(codes, q.codes.data(), sizeof(float) * q.codes.size());
        std::memcpy(scales, q.scales.data(), sizeof(float) * q.scales.size());
    });
}

// rmsnorm_forward / rmsnorm_backward / rmsnorm_gain_gradient (rmsnorm.hpp:27-100)
int ref_rmsnorm(const float* x, const float* gain, const float* e, long long rows, long long dim, float* y,
                float* dx, float* dgain) {
    return guard([&] {
        const Tensor X = make(x, rows, dim), G = make(gain, 1, dim), E = make(e, rows, dim);
        put(rmsnorm_forward(X, &G), y);
        put(rmsnorm_backward(X, E, &G), dx);
        put(rmsnorm_gain_gradient(X, E), dgain);
    });
}

} // extern "C"
