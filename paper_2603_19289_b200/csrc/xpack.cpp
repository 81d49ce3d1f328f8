// xpack.cpp — lossless exponent packing of bf16 expert blocks (format in
// engine.h, "xp12").  Host side: xp_pack at store fill, xp_unpack for tests and
// partial rewrites; the device decoder is k_xp_unpack (kernels.cu), run on the
// copy stream between the H2D of the packed block and the slot's ready flag.
//
// Why: every expert miss moves the expert's bf16 block over PCIe (the link is
// the bottleneck of the offloaded decode).  Sign and mantissa
// are incompressible, but the 8-bit exponent of weights drawn around a fixed
// scale spans a few binades; a 4-bit code relative to a per-block base, with
// an escape list for the rare values outside the 15-binade window, carries
// every weight in 12 bits.  The slots in HBM hold the plain bf16 block, so no
// compute kernel changes and parity is untouched (lossless by construction,
// checked by tests/test_capi.py round trips and the bit-exact GPU tests).
#include "engine.h"

#include <cstring>

namespace smoe {

long long xp_pack(const uint16_t* raw, long long n, uint8_t* out, long long cap) {
    if (n <= 0 || n % 8 != 0) return 0;
    // base: the 15-binade window [base, base + 14] (base >= 1: zeros and
    // subnormals always escape) holding the most weights, so a few outliers
    // never push the Gaussian bulk out of the window
    long long hist[256] = {0};
    for (long long i = 0; i < n; ++i) ++hist[(raw[i] >> 7) & 0xff];
    long long win = 0;
    for (int e = 1; e <= 15; ++e) win += hist[e];
    int base = 1;
    long long best = win;
    for (int b = 2; b + 14 <= 255; ++b) {
        win += hist[b + 14] - hist[b - 1];
        if (win >= best) {
            best = win;
            base = b;
        }
    }
    const long long nesc = n - best;
    const long long bytes = xp_bytes(n, nesc);
    if (bytes > n * 2 * 7 / 8 || bytes > cap) return 0;
    const uint32_t hdr[4] = {kXpMagic, static_cast<uint32_t>(base), static_cast<uint32_t>(nesc),
                             static_cast<uint32_t>(n / 8)};
    std::memcpy(out, hdr, sizeof hdr);
    uint8_t* codes = out + kXpHeader;
    uint8_t* sm = codes + n / 2;
    uint8_t* esc = sm + n;
    long long k = 0;
    for (long long i = 0; i < n; i += 2) {
        uint8_t pair = 0;
        for (int j = 0; j < 2; ++j) {
            const uint16_t v = raw[i + j];
            const int e = (v >> 7) & 0xff;
            int c = e - base;
            if (c < 0 || c > 14) {
                c = 15;
                const uint32_t idx = static_cast<uint32_t>(i + j);
                std::memcpy(esc + 8 * k, &idx, 4);
                std::memcpy(esc + 8 * k + 4, &v, 2);
                std::memset(esc + 8 * k + 6, 0, 2);
                ++k;
            }
            pair |= static_cast<uint8_t>(c << (4 * j));
            sm[i + j] = static_cast<uint8_t>(((v >> 8) & 0x80) | (v & 0x7f));
        }
        codes[i / 2] = pair;
    }
    return bytes;
}

void xp_unpack(const uint8_t* in, uint16_t* out) {
    uint32_t hdr[4];
    std::memcpy(hdr, in, sizeof hdr);
    if (hdr[0] != kXpMagic) throw std::runtime_error("xp_unpack: not a packed expert block");
    const int base = static_cast<int>(hdr[1]);
    const long long nesc = hdr[2], n = static_cast<long long>(hdr[3]) * 8;
    const uint8_t* codes = in + kXpHeader;
    const uint8_t* sm = codes + n / 2;
    const uint8_t* esc = sm + n;
    for (long long i = 0; i < n; ++i) {
        const int c = (codes[i / 2] >> (4 * (i & 1))) & 15;
        const uint8_t b = sm[i];
        out[i] = static_cast<uint16_t>(((b & 0x80) << 8) | ((base + c) << 7) | (b & 0x7f));
    }
    for (long long k = 0; k < nesc; ++k) {
        uint32_t idx;
        uint16_t v;
        std::memcpy(&idx, esc + 8 * k, 4);
        std::memcpy(&v, esc + 8 * k + 4, 2);
        if (idx >= n) throw std::runtime_error("xp_unpack: escape index out of range");
        out[idx] = v;
    }
}

}  // namespace smoe
