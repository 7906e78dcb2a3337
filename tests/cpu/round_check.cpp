// Compiles the device quantizer header on the host and compares it with the
// oracle's double-precision round_code (quantize.hpp:152-180) on
// random, grid-midpoint and saturation inputs.  Prints "mismatches N total T".
#include "../../paper_2501_02625_b200/csrc/quant_round.cuh"
#include "../../oracle/halo_oracle.h"
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
using namespace halo_b200;

static long long bad = 0, total = 0;

static void check(float x, float s, int fmt) {
    const float inv = 1.0f / s;
    const double want = orc_round_code((double)x / (double)s, fmt);
    ++total;
    if (fmt == ORC_INT8) {
        const int8_t got = quant_int8(x, s, inv);
        uint32_t sl;
        int8_t fast = (int8_t)quant_int8_try(x, inv, sl);
        if (sl) fast = quant_int8(x, s, inv);
        if (quant_int8_fast(x, s, inv) != fast) fast = 99;
        uint32_t sr;
        int8_t fr = (int8_t)quant_int8_try_r(x, s, inv, half_margin(s), sr);
        if (sr) fr = quant_int8(x, s, inv);
        if (fr != fast) fast = 98;
        if ((double)got != want || (double)fast != want) {
            if (bad < 5) printf("int8 x=%a s=%a got %d fast %d want %g\n", x, s, got, fast, want);
            ++bad;
        }
    } else if (fmt == ORC_FP6_E3M2) {
        const uint8_t got = quant_e3m2(x, s, inv);
        const float wv = (float)want;
        // the 6-bit code of the oracle's grid value: decode every code, match
        uint8_t wb = 0xFF;
        for (int c = 0; c < 64; ++c)
            if (e3m2_to_float((uint8_t)c) == wv && !(wv == 0.0f && c != 0)) { wb = (uint8_t)c; break; }
        if (got != wb) {
            if (bad < 5) printf("e3m2 x=%a s=%a got %02x want %02x (%g)\n", x, s, got, wb, want);
            ++bad;
        }
    } else {
        const uint8_t got = quant_e4m3(x, s, inv);
        uint32_t sl;
        uint8_t fast = quant_e4m3_try(x, inv, sl);
        if (sl) fast = quant_e4m3(x, s, inv);
        if (quant_e4m3_fast(x, s, inv) != fast) fast = 0xFF;
        float wf = (float)want; uint8_t wb; orc_codes_to_e4m3(&wf, 1, &wb);
        if (got != wb || fast != wb) {
            if (bad < 5) printf("e4m3 x=%a s=%a got %02x fast %02x want %02x (%g)\n", x, s, got, fast, wb, want);
            ++bad;
        }
    }
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 10000000;
    std::mt19937_64 g(12345);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int fmt = 0; fmt < 3; ++fmt) {
        const double fmax = fmt == 0 ? 127.0 : fmt == 1 ? 448.0 : 28.0;
        // 1) random scales, values spread over the whole code range
        for (long long i = 0; i < n; ++i) {
            const float s = (float)std::ldexp(1.0 + u(g), (int)(u(g) * 40) - 30);
            const float x = (float)((u(g) * 2 - 1) * fmax * 1.02 * s);
            check(x, s, fmt);
        }
        // 2) values at / next to every exact midpoint q+1/2 (and minifloat
        //    midpoints), for random scales: x = mid*s rounded, and its
        //    float neighbours.
        std::vector<double> mids;
        if (fmt == 0) { for (int q = -128; q <= 127; ++q) mids.push_back(q + 0.5); }
        else if (fmt == 2) {
            std::vector<double> grid;
            for (int c = 0; c < 32; ++c) grid.push_back(e3m2_to_float((uint8_t)c));
            grid.push_back(32.0);
            for (size_t k = 0; k + 1 < grid.size(); ++k) { mids.push_back(0.5 * (grid[k] + grid[k + 1])); mids.push_back(-0.5 * (grid[k] + grid[k + 1])); }
        } else {
            std::vector<double> grid;
            for (int b = 0; b < 127; ++b) { uint8_t c = (uint8_t)b; grid.push_back(orc_e4m3_to_float(c)); }
            grid.push_back(480.0);
            for (size_t k = 0; k + 1 < grid.size(); ++k) { mids.push_back(0.5 * (grid[k] + grid[k + 1])); mids.push_back(-0.5 * (grid[k] + grid[k + 1])); }
        }
        for (long long i = 0; i < n / 20; ++i) {
            const float s = (float)std::ldexp(1.0 + u(g), (int)(u(g) * 40) - 30);
            for (double m : mids) {
                const float x = (float)(m * (double)s);
                check(x, s, fmt);
                check(std::nextafter(x, 1e30f), s, fmt);
                check(std::nextafter(x, -1e30f), s, fmt);
            }
        }
        // 3) exact ties: scale a power of two so mid*s is exact
        for (int e = -20; e <= 20; ++e) {
            const float s = std::ldexp(1.0f, e);
            for (double m : mids) { check((float)(m * s), s, fmt); check((float)(m * s * 1.5), s * 1.5f, fmt); }
        }
        // 4) saturation and zeros
        for (float s : {1.0f, 0.25f, 3.0f}) {
            for (float x : {0.0f, -0.0f, 1e-30f, -1e-30f, 1e6f, -1e6f, 127.5f, -127.5f, 464.0f, -464.0f, 448.0f, 447.9f,
                            28.0f, 29.9f, 30.0f, -30.0f, 31.0f, 32.0f, 0.03125f, -0.03125f, 0.09375f})
                check(x * s, s, fmt);
        }
    }
    printf("mismatches %lld total %lld\n", bad, total);
    return bad != 0;
}
