// xpack.cpp — lossless exponent packing of bf16 expert blocks (format in
// engine.h, "xp11").  Host side: xp_pack at store fill, xp_unpack for tests and
// partial rewrites; the device decoder is k_xp_unpack (kernels.cu), run on the
// copy lane between the H2D of the packed block and the slot's ready flag.
//
// Why: every expert miss moves the expert's bf16 block over PCIe (the link is
// the bottleneck of the offloaded decode).  Sign and mantissa
// are incompressible, but the 8-bit exponent of weights drawn around a fixed
// scale spans a few binades, so it is coded with a 2-bit primary code (the
// block's three most frequent exponents) and a 4-bit secondary code for the
// rest, with an escape list for what the secondary window misses.  The slots
// in HBM hold the plain bf16 block, so no compute kernel changes and parity is
// untouched (lossless by construction, checked by tests/test_xpack.py round
// trips and the bit-exact GPU tests).
#include "engine.h"

#include <algorithm>
#include <cstring>

namespace smoe {

long long xp_pack(const uint16_t* raw, long long n, uint8_t* out, long long cap) {
    if (n <= 0 || n % kXpGroup != 0) return 0;
    long long hist[256] = {0};
    for (long long i = 0; i < n; ++i) ++hist[(raw[i] >> 7) & 0xff];
    // primary: the three most frequent exponents (ties: lower exponent)
    int p[3] = {-1, -1, -1};
    for (int k = 0; k < 3; ++k)
        for (int e = 0; e < 256; ++e) {
            if (e == p[0] || e == p[1]) continue;
            if (p[k] < 0 || hist[e] > hist[p[k]]) p[k] = e;
        }
    int prim[256];
    std::fill(prim, prim + 256, -1);
    for (int k = 0; k < 3; ++k) prim[p[k]] = k;
    // secondary window: the 15 binades [base, base + 14], base >= 1, holding
    // the most non-primary weights (zeros and subnormals always escape)
    long long rest[256];
    for (int e = 0; e < 256; ++e) rest[e] = prim[e] >= 0 ? 0 : hist[e];
    long long win = 0;
    for (int e = 1; e <= 15; ++e) win += rest[e];
    int base = 1;
    long long best = win;
    for (int b = 2; b + 14 <= 255; ++b) {
        win += rest[b + 14] - rest[b - 1];
        if (win > best) {
            best = win;
            base = b;
        }
    }
    long long nsec = 0;
    for (int e = 0; e < 256; ++e) nsec += rest[e];
    const long long nesc = nsec - best;
    const long long bytes = xp_bytes(n, nsec, nesc);
    if (bytes > n * 2 * 7 / 8 || bytes > cap) return 0;
    std::memset(out, 0, static_cast<size_t>(xp_off_sm(n, nsec)));
    const uint32_t hdr[8] = {kXpMagic, static_cast<uint32_t>(n / kXpGroup), static_cast<uint32_t>(nsec),
                             static_cast<uint32_t>(nesc), static_cast<uint32_t>(p[0]), static_cast<uint32_t>(p[1]),
                             static_cast<uint32_t>(p[2]), static_cast<uint32_t>(base)};
    std::memcpy(out, hdr, sizeof hdr);
    uint8_t* pc = out + kXpHeader;
    uint8_t* gr = out + xp_off_groups(n);
    uint8_t* sc = out + xp_off_sec(n);
    uint8_t* sm = out + xp_off_sm(n, nsec);
    uint8_t* esc = out + xp_off_esc(n, nsec);
    long long k = 0, ke = 0;
    for (long long i = 0; i < n; ++i) {
        if (i % kXpGroup == 0) {
            const uint32_t g = static_cast<uint32_t>(k);
            std::memcpy(gr + 4 * (i / kXpGroup), &g, 4);
        }
        const uint16_t v = raw[i];
        const int e = (v >> 7) & 0xff;
        int c = prim[e];
        if (c < 0) {
            c = 3;
            int s2 = e - base;
            if (e == 0 || s2 < 0 || s2 > 14) {
                s2 = 15;
                const uint32_t idx = static_cast<uint32_t>(i);
                std::memcpy(esc + 8 * ke, &idx, 4);
                std::memcpy(esc + 8 * ke + 4, &v, 2);
                std::memset(esc + 8 * ke + 6, 0, 2);
                ++ke;
            }
            sc[k / 2] |= static_cast<uint8_t>(s2 << (4 * (k & 1)));
            ++k;
        }
        pc[i / 4] |= static_cast<uint8_t>(c << (2 * (i % 4)));
        sm[i] = static_cast<uint8_t>(((v >> 8) & 0x80) | (v & 0x7f));
    }
    return bytes;
}

void xp_unpack(const uint8_t* in, uint16_t* out) {
    uint32_t hdr[8];
    std::memcpy(hdr, in, sizeof hdr);
    if (hdr[0] != kXpMagic) throw std::runtime_error("xp_unpack: not a packed expert block");
    const long long n = static_cast<long long>(hdr[1]) * kXpGroup, nsec = hdr[2], nesc = hdr[3];
    const int p[3] = {static_cast<int>(hdr[4]), static_cast<int>(hdr[5]), static_cast<int>(hdr[6])};
    const int base = static_cast<int>(hdr[7]);
    const uint8_t* pc = in + kXpHeader;
    const uint8_t* sc = in + xp_off_sec(n);
    const uint8_t* sm = in + xp_off_sm(n, nsec);
    const uint8_t* esc = in + xp_off_esc(n, nsec);
    long long k = 0;
    for (long long i = 0; i < n; ++i) {
        const int c = (pc[i / 4] >> (2 * (i % 4))) & 3;
        int e;
        if (c < 3) {
            e = p[c];
        } else {
            const int s2 = (sc[k / 2] >> (4 * (k & 1))) & 15;
            ++k;
            e = base + s2;  // s2 == 15: patched from the escape list below
        }
        const uint8_t b = sm[i];
        out[i] = static_cast<uint16_t>(((b & 0x80) << 8) | ((e & 0xff) << 7) | (b & 0x7f));
    }
    for (long long q = 0; q < nesc; ++q) {
        uint32_t idx;
        uint16_t v;
        std::memcpy(&idx, esc + 8 * q, 4);
        std::memcpy(&v, esc + 8 * q + 4, 2);
        if (idx >= n) throw std::runtime_error("xp_unpack: escape index out of range");
        out[idx] = v;
    }
}

}  // namespace smoe
