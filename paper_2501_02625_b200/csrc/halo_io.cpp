// halo_io.cpp — the reference's quantized-tensor file format (HALT
// container, tensor_io.hpp:1-135; write_quantized_tensor /
// read_quantized_tensor, quantize.hpp:405-474) for the device code layouts,
// so an exported (WH)_Q (export_inference_weights, halo_linear.hpp:332-338)
// is readable by the reference and vice versa.
//
//   "HALT" | u32 version 1 | u8 dtype (2 = int8 codes, 3 = f32 codes) |
//   u8 rank 2 | u64 rows | u64 cols | u8 NumericFormat | u8 GranularityKind |
//   u32 block_rows | u32 block_cols | u64 n_scales | f32 scales[n] |
//   codes: int8 bytes (Int8) or f32 grid values (Fp8E4M3, Fp6E3M2)
//
// All integers little-endian.  Device code layouts: INT8 two's complement,
// OCP E4M3 bytes, E3M2 codes in bits 7:2.  Host buffers in and out (the
// caller moves device codes); pure host code.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/halo_b200.h"

namespace halo_b200 {
void set_last_error(const char* msg);
}

namespace {

halo_status io_fail(const std::string& m) {
    halo_b200::set_last_error(m.c_str());
    return HALO_ERR_IO;
}

float e4m3_value(uint8_t b) {
    const int s = b >> 7, e = (b >> 3) & 15, m = b & 7;
    float v = e == 0 ? std::ldexp((float)m, -9) : std::ldexp(1.0f + m / 8.0f, e - 7);
    return s ? -v : v;
}
float e3m2_value(uint8_t code6) {
    const int s = (code6 >> 5) & 1, e = (code6 >> 2) & 7, m = code6 & 3;
    float v = e == 0 ? std::ldexp((float)m, -4) : std::ldexp(1.0f + m / 4.0f, e - 3);
    return s ? -v : v;
}
// device byte -> code value (the reference's QuantizedTensor::codes)
float code_value(int fmt, uint8_t b) {
    if (fmt == HALO_FMT_INT8) return (float)(int8_t)b;
    if (fmt == HALO_FMT_FP8_E4M3) return e4m3_value(b);
    return e3m2_value(b >> 2);
}
// code value -> device byte; false if the value is not on the grid
bool code_byte(int fmt, float v, uint8_t* out) {
    if (fmt == HALO_FMT_INT8) {
        if (!(v >= -127.0f && v <= 127.0f) || v != std::nearbyint(v)) return false;
        *out = (uint8_t)(int8_t)v;
        return true;
    }
    if (v == 0.0f) {  // the reference stores +0 (round_minifloat adds +0.0)
        *out = 0;
        return true;
    }
    const int n = fmt == HALO_FMT_FP8_E4M3 ? 256 : 64;
    for (int c = 0; c < n; ++c) {
        if (fmt == HALO_FMT_FP8_E4M3 && (c & 0x7f) == 0x7f) continue;  // NaN encodings
        const float g = fmt == HALO_FMT_FP8_E4M3 ? e4m3_value((uint8_t)c) : e3m2_value((uint8_t)c);
        if (g == v) {
            *out = fmt == HALO_FMT_FP8_E4M3 ? (uint8_t)c : (uint8_t)(c << 2);
            return true;
        }
    }
    return false;
}

int64_t group_count(int gran, int64_t rows, int64_t cols) {
    return gran == HALO_GRAN_TENSOR ? 1 : gran == HALO_GRAN_ROW ? rows : cols;
}

struct Reader {
    FILE* f;
    bool ok = true;
    uint64_t le(int n) {
        uint64_t v = 0;
        for (int i = 0; i < n; ++i) {
            const int c = std::fgetc(f);
            if (c == EOF) {
                ok = false;
                return 0;
            }
            v |= (uint64_t)(uint8_t)c << (8 * i);
        }
        return v;
    }
};
void put_le(std::vector<uint8_t>& b, uint64_t v, int n) {
    for (int i = 0; i < n; ++i) b.push_back((uint8_t)(v >> (8 * i)));
}

struct Header {
    int dtype, fmt, gran;
    int64_t rows, cols, block_rows, block_cols, nscales;
};

halo_status read_header(FILE* f, Header* h) {
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "HALT", 4) != 0)
        return io_fail("tensor file: bad magic");
    Reader r{f};
    const uint32_t ver = (uint32_t)r.le(4);
    if (!r.ok) return io_fail("tensor file: truncated");
    if (ver != 1) return io_fail("tensor file: unsupported version " + std::to_string(ver));
    h->dtype = (int)r.le(1);
    const int rank = (int)r.le(1);
    h->rows = (int64_t)r.le(8);
    h->cols = (int64_t)r.le(8);
    if (!r.ok) return io_fail("tensor file: truncated");
    if (h->dtype > 3) return io_fail("tensor file: unknown dtype code " + std::to_string(h->dtype));
    if (rank != 2) return io_fail("tensor file: unsupported rank " + std::to_string(rank));
    if (h->dtype != 2 && h->dtype != 3) return io_fail("tensor file: not a quantized payload");
    h->fmt = (int)r.le(1);
    h->gran = (int)r.le(1);
    h->block_rows = (int64_t)r.le(4);
    h->block_cols = (int64_t)r.le(4);
    h->nscales = (int64_t)r.le(8);
    if (!r.ok) return io_fail("tensor file: truncated");
    if (h->fmt > 5) return io_fail("tensor file: unknown format code");
    if (h->gran > 4) return io_fail("tensor file: unknown granularity code");
    return HALO_OK;
}

}  // namespace

extern "C" halo_status halo_quantized_tensor_write(const char* path, int32_t format, int32_t granularity, int64_t rows,
                                                   int64_t cols, const uint8_t* codes, const float* scales,
                                                   int64_t n_scales) {
    if (!path || (rows * cols > 0 && !codes) || !scales) return io_fail("write_quantized_tensor: null argument");
    if (format != HALO_FMT_INT8 && format != HALO_FMT_FP8_E4M3 && format != HALO_FMT_FP6_E3M2)
        return io_fail("write_quantized_tensor: format must be int8, fp8_e4m3 or fp6_e3m2");
    if (granularity != HALO_GRAN_TENSOR && granularity != HALO_GRAN_ROW && granularity != HALO_GRAN_COLUMN)
        return io_fail("write_quantized_tensor: tensor, row or column granularity");
    if (rows < 0 || cols < 0 || n_scales != group_count(granularity, rows, cols))
        return io_fail("write_quantized_tensor: scale count does not match granularity");
    const bool i8 = format == HALO_FMT_INT8;
    std::vector<uint8_t> b;
    b.reserve(64 + (size_t)n_scales * 4 + (size_t)(rows * cols) * (i8 ? 1 : 4));
    b.insert(b.end(), {'H', 'A', 'L', 'T'});
    put_le(b, 1, 4);
    put_le(b, i8 ? 2 : 3, 1);
    put_le(b, 2, 1);
    put_le(b, (uint64_t)rows, 8);
    put_le(b, (uint64_t)cols, 8);
    put_le(b, (uint64_t)format, 1);  // halo_format ids are NumericFormat's (quantize.hpp:22-29)
    put_le(b, (uint64_t)granularity, 1);  // HALO_GRAN_* are GranularityKind's (:65-71)
    put_le(b, 0, 4);
    put_le(b, 0, 4);
    put_le(b, (uint64_t)n_scales, 8);
    for (int64_t i = 0; i < n_scales; ++i) {
        uint32_t u;
        std::memcpy(&u, scales + i, 4);
        put_le(b, u, 4);
    }
    const int64_t n = rows * cols;
    if (i8) {
        b.insert(b.end(), codes, codes + n);
    } else {
        for (int64_t i = 0; i < n; ++i) {
            const float v = code_value(format, codes[i]);
            uint32_t u;
            std::memcpy(&u, &v, 4);
            put_le(b, u, 4);
        }
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) return io_fail(std::string("cannot open ") + path + " for writing");
    const bool ok = std::fwrite(b.data(), 1, b.size(), f) == b.size();
    const bool closed = std::fclose(f) == 0;
    if (!ok || !closed) return io_fail(std::string("write failed for ") + path);
    return HALO_OK;
}

extern "C" halo_status halo_quantized_tensor_info(const char* path, int32_t* format, int32_t* granularity,
                                                  int64_t* rows, int64_t* cols, int64_t* n_scales) {
    if (!path) return io_fail("read_quantized_tensor: null path");
    FILE* f = std::fopen(path, "rb");
    if (!f) return io_fail(std::string("cannot open ") + path);
    Header h;
    const halo_status s = read_header(f, &h);
    std::fclose(f);
    if (s != HALO_OK) return s;
    if (format) *format = h.fmt;
    if (granularity) *granularity = h.gran;
    if (rows) *rows = h.rows;
    if (cols) *cols = h.cols;
    if (n_scales) *n_scales = h.nscales;
    return HALO_OK;
}

extern "C" halo_status halo_quantized_tensor_read(const char* path, uint8_t* codes, float* scales) {
    if (!path) return io_fail("read_quantized_tensor: null path");
    FILE* f = std::fopen(path, "rb");
    if (!f) return io_fail(std::string("cannot open ") + path);
    Header h;
    halo_status s = read_header(f, &h);
    auto done = [&](halo_status st) {
        std::fclose(f);
        return st;
    };
    if (s != HALO_OK) return done(s);
    if (h.fmt != HALO_FMT_INT8 && h.fmt != HALO_FMT_FP8_E4M3 && h.fmt != HALO_FMT_FP6_E3M2)
        return done(io_fail("read_quantized_tensor: format has no device code layout (int8, fp8_e4m3, fp6_e3m2)"));
    if (h.gran > HALO_GRAN_COLUMN)
        return done(io_fail("read_quantized_tensor: block / mx granularity has no device layout"));
    if (h.nscales != group_count(h.gran, h.rows, h.cols))
        return done(io_fail("tensor file: scale count does not match granularity"));
    if ((h.dtype == 2) != (h.fmt == HALO_FMT_INT8))
        return done(io_fail("tensor file: payload dtype does not match the format"));
    Reader r{f};
    for (int64_t i = 0; i < h.nscales; ++i) {
        const uint32_t u = (uint32_t)r.le(4);
        std::memcpy(scales + i, &u, 4);
    }
    const int64_t n = h.rows * h.cols;
    if (h.dtype == 2) {
        if (n && std::fread(codes, 1, (size_t)n, f) != (size_t)n) r.ok = false;
    } else {
        for (int64_t i = 0; i < n && r.ok; ++i) {
            const uint32_t u = (uint32_t)r.le(4);
            float v;
            std::memcpy(&v, &u, 4);
            if (r.ok && !code_byte(h.fmt, v, codes + i))
                return done(io_fail("tensor file: code value off the format grid at element " + std::to_string(i)));
        }
    }
    if (!r.ok) return done(io_fail("tensor file: truncated"));
    return done(HALO_OK);
}
