// philox_plane.cuh -- Philox4x32-10 blocks of the PLANE engine's bit-plane
// draws (counter {site, t_lo, t_hi, group << 4 | block}, run key schedule in
// the kernel's constant bank), with the parts that are constant over a colour
// phase or shared by the blocks of one site computed once.
#pragma once

#include <stdint.h>

#include "philox.cuh"

namespace tg {

// The PLANE kernels take both halves of a Philox product from one 32x32->64
// multiply (IMAD.WIDE.U32): measured +0.5 ... +1.2 % on the fused kernels once
// the compare chains were shortened (profiles/r2/ab_mulwide_s5.txt); the FLOAT
// and SLOT kernels keep the split form of philox.cuh (-2.5 % with the wide one).
#ifndef TG_PLANE_MULWIDE
#define TG_PLANE_MULWIDE 1
#endif
__device__ __forceinline__ void mulhilo_p(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if TG_PLANE_MULWIDE
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
#else
    hi = __umulhi(a, b);
    lo = a * b;
#endif
}

// Philox4x32-10 for the plane counters {site, t_lo, t_hi, group << 4 | blk}
// with t and the key fixed for a colour phase: the products of round 1 on
// (t_hi) and of round 2 on the resulting constant are per-phase constants
// (PhiloxT), and the two unconditional blocks of a site share round 1's
// product on `site` and round 3's on the site-only word.  Output identical
// to philox4x32_10_ks (tests compare every plane draw with the oracle).
struct PhiloxT {
    uint32_t c0, c1x;  // round-1 words 0, 1 (c1x = word 1 ^ round-2 key 0)
    uint32_t h0x, l0;  // round-2 hi(M0 * c0) ^ round-2 key 1, lo(M0 * c0)
};

__device__ __forceinline__ PhiloxT philox_t(uint32_t tlo, uint32_t thi, const uint32_t* ks) {
    PhiloxT P;
    const uint32_t hi1 = __umulhi(kPhiloxM1, thi), lo1 = kPhiloxM1 * thi;
    P.c0 = hi1 ^ tlo ^ ks[0];
    P.c1x = lo1 ^ ks[2];
    P.h0x = __umulhi(kPhiloxM0, P.c0) ^ ks[3];
    P.l0 = kPhiloxM0 * P.c0;
    return P;
}

// Rounds 3..10 from the round-2 output.
__device__ __forceinline__ u32x4 philox_rounds_3_10(u32x4 c, const uint32_t* ks) {
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo_p(kPhiloxM0, c.x, hi0, lo0);
        mulhilo_p(kPhiloxM1, c.z, hi1, lo1);
        c = u32x4{hi1 ^ c.y ^ ks[2 * r], lo1, hi0 ^ c.w ^ ks[2 * r + 1], lo0};
    }
    return c;
}

// One block: counter word 3 = g.
__device__ __forceinline__ u32x4 philox_plane(uint32_t site, uint32_t g, const PhiloxT& P,
                                              const uint32_t* ks) {
    const uint32_t hs = __umulhi(kPhiloxM0, site), ls = kPhiloxM0 * site;
    const uint32_t y2 = hs ^ g ^ ks[1];                  // round 1 (words 0, 1 are P.c0, lo1)
    const uint32_t hq = __umulhi(kPhiloxM1, y2), lq = kPhiloxM1 * y2;
    return philox_rounds_3_10(u32x4{hq ^ P.c1x, lq, P.h0x ^ ls, P.l0}, ks);  // round 2
}

// The two blocks g0, g0 | 1 of one site.
__device__ __forceinline__ void philox_plane2(uint32_t site, uint32_t g0, const PhiloxT& P,
                                              const uint32_t* ks, u32x4& r0, u32x4& r1) {
    const uint32_t hs = __umulhi(kPhiloxM0, site), ls = kPhiloxM0 * site;
    const uint32_t z2 = P.h0x ^ ls;                      // round-2 word 2, shared
    const uint32_t ya = hs ^ g0 ^ ks[1], yb = hs ^ (g0 | 1u) ^ ks[1];
    const uint32_t hqa = __umulhi(kPhiloxM1, ya), lqa = kPhiloxM1 * ya;
    const uint32_t hqb = __umulhi(kPhiloxM1, yb), lqb = kPhiloxM1 * yb;
    // round 3: M1 * z2 shared
    const uint32_t h3 = __umulhi(kPhiloxM1, z2), l3 = kPhiloxM1 * z2;
    const uint32_t xa = hqa ^ P.c1x, xb = hqb ^ P.c1x;
    const uint32_t h0a = __umulhi(kPhiloxM0, xa), l0a = kPhiloxM0 * xa;
    const uint32_t h0b = __umulhi(kPhiloxM0, xb), l0b = kPhiloxM0 * xb;
    u32x4 a{h3 ^ lqa ^ ks[4], l3, h0a ^ P.l0 ^ ks[5], l0a};
    u32x4 b{h3 ^ lqb ^ ks[4], l3, h0b ^ P.l0 ^ ks[5], l0b};
#pragma unroll
    for (int r = 3; r < 10; ++r) {
        uint32_t p0, q0, p1, q1, s0, t0, s1, t1;
        mulhilo_p(kPhiloxM0, a.x, p0, q0);
        mulhilo_p(kPhiloxM1, a.z, p1, q1);
        mulhilo_p(kPhiloxM0, b.x, s0, t0);
        mulhilo_p(kPhiloxM1, b.z, s1, t1);
        a = u32x4{p1 ^ a.y ^ ks[2 * r], q1, p0 ^ a.w ^ ks[2 * r + 1], q0};
        b = u32x4{s1 ^ b.y ^ ks[2 * r], t1, s0 ^ b.w ^ ks[2 * r + 1], t0};
    }
    r0 = a;
    r1 = b;
}


// N blocks of one site, counter word 3 = g[j]: rounds 1-3 share the site's
// round-1 product and the round-2 word-2 product (philox_plane2 for N = 2).
// WIDE1: also the shared first-round products as one wide multiply each
// (plane_c5.cu: +1.3 %; the word-local kernel loses 1.4 % with it).
template <int N, bool WIDE1 = false>
__device__ __forceinline__ void philox_planeN(uint32_t site, const uint32_t (&g)[N], const PhiloxT& P,
                                              const uint32_t* ks, u32x4 (&o)[N]) {
    uint32_t hs, ls, h3, l3;
    if (WIDE1) mulhilo_p(kPhiloxM0, site, hs, ls);
    else { hs = __umulhi(kPhiloxM0, site); ls = kPhiloxM0 * site; }
    const uint32_t z2 = P.h0x ^ ls;
    if (WIDE1) mulhilo_p(kPhiloxM1, z2, h3, l3);
    else { h3 = __umulhi(kPhiloxM1, z2); l3 = kPhiloxM1 * z2; }
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const uint32_t y = hs ^ g[j] ^ ks[1];
        uint32_t hq, lq, h0, l0;
        if (WIDE1) mulhilo_p(kPhiloxM1, y, hq, lq);
        else { hq = __umulhi(kPhiloxM1, y); lq = kPhiloxM1 * y; }
        const uint32_t x = hq ^ P.c1x;
        if (WIDE1) mulhilo_p(kPhiloxM0, x, h0, l0);
        else { h0 = __umulhi(kPhiloxM0, x); l0 = kPhiloxM0 * x; }
        o[j] = u32x4{h3 ^ lq ^ ks[4], l3, h0 ^ P.l0 ^ ks[5], l0};
    }
#pragma unroll
    for (int r = 3; r < 10; ++r) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            uint32_t p0, q0, p1, q1;
            mulhilo_p(kPhiloxM0, o[j].x, p0, q0);
            mulhilo_p(kPhiloxM1, o[j].z, p1, q1);
            o[j] = u32x4{p1 ^ o[j].y ^ ks[2 * r], q1, p0 ^ o[j].w ^ ks[2 * r + 1], q0};
        }
    }
}

}  // namespace tg
