// plane_device.cuh -- bit-sliced device helpers of the PLANE engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.cuh"

namespace tg {

// ------------------------------------------------------------ helpers

// One LOP3 with an explicit truth table (a = 0xF0, b = 0xCC, c = 0xAA).
template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

#ifndef TG_CMP8
#define TG_CMP8 1
#endif

__device__ __forceinline__ uint32_t sel(uint32_t m, uint32_t a1, uint32_t a0) {
#if TG_CMP8
    return lop3<0xCA>(m, a1, a0);  // (m & a1) | (~m & a0) as one instruction
#else
    return (m & a1) | (~m & a0);
#endif
}

// Select, per lane bit, leaves[class(lane)] where class bits are cb[0..B).
template <int B>
__device__ __forceinline__ uint32_t mux_tree(const uint32_t* cb, const uint32_t* leaves) {
    constexpr int L = 1 << B;
    uint32_t v[L < 4 ? 4 : L];
    if constexpr (L >= 4) {
#pragma unroll
        for (int q = 0; q < L / 4; ++q) {
            const uint4 t = __ldg(reinterpret_cast<const uint4*>(leaves) + q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < L; ++q) v[q] = __ldg(leaves + q);
    }
#pragma unroll
    for (int lvl = 0; lvl < B; ++lvl) {
#pragma unroll
        for (int c = 0; c < (L >> (lvl + 1)); ++c) v[c] = sel(cb[lvl], v[2 * c + 1], v[2 * c]);
    }
    return v[0];
}

// Add a one-bit-per-lane mask to a bit-sliced counter of NB bits.
template <int NB>
__device__ __forceinline__ void bs_add(uint32_t* c, uint32_t v) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const uint32_t carry = c[b] & v;
        c[b] ^= v;
        v = carry;
    }
}

// 32x32 bit-matrix transpose across a warp (row = lane): five block-swap
// stages; the partner's row is rotated into place and bit-selected.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t m = 0x0000FFFFu;
#pragma unroll
    for (int j = 16; j; j >>= 1, m ^= (m << j)) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        const bool hi = (lane & j) != 0;
        const uint32_t rot = __funnelshift_l(y, y, hi ? 32 - j : j);  // y >> j / y << j, wrapped
        const uint32_t keep = hi ? ~m : m;
        x = (x & keep) | (rot & ~keep);
    }
    return x;
}


template <int WV>
__device__ __forceinline__ void load_row(const uint32_t* p, uint32_t (&r)[WV]) {
    if constexpr (WV % 4 == 0) {
#pragma unroll
        for (int q = 0; q < WV / 4; ++q) {
            const uint4 v = reinterpret_cast<const uint4*>(p)[q];
            r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
        }
    } else if constexpr (WV == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        r[0] = v.x; r[1] = v.y;
    } else {
#pragma unroll
        for (int q = 0; q < WV; ++q) r[q] = p[q];
    }
}

template <int WV>
__device__ __forceinline__ void store_row(uint32_t* p, const uint32_t (&r)[WV]) {
    if constexpr (WV % 4 == 0) {
#pragma unroll
        for (int q = 0; q < WV / 4; ++q)
            reinterpret_cast<uint4*>(p)[q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    } else if constexpr (WV == 2) {
        *reinterpret_cast<uint2*>(p) = make_uint2(r[0], r[1]);
    } else {
#pragma unroll
        for (int q = 0; q < WV; ++q) p[q] = r[q];
    }
}

// Lazy MSB-first comparison of the 53-bit uniforms of 32 lanes against the
// lanes' thresholds, 4 planes per Philox4x32-10 block.
template <int B>
__device__ __forceinline__ void compare_block(const uint32_t* cb, const uint32_t* kpb, int ncl,
                                              int blk, const u32x4& r, uint32_t& und,
                                              uint32_t& lt) {
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int b = blk * 4 + q;
        if (b < kKPlanes) {
            const uint32_t tb = mux_tree<B>(cb, kpb + b * ncl);
            lt |= und & tb & ~rr[q];
            und &= ~(tb ^ rr[q]);
        }
    }
}


// compare_block with a one-level threshold select between two adjacent
// classes (k01[0] for lanes with c clear, k01[1] with c set), one 8-byte load
// per plane.
__device__ __forceinline__ void compare_block_sel(uint32_t c, const uint32_t* k01, int ncl, int blk,
                                                  const u32x4& r, uint32_t& und, uint32_t& lt) {
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int b = blk * 4 + q;
        if (b < kKPlanes) {
            const uint2 kk = __ldg(reinterpret_cast<const uint2*>(k01 + b * ncl));
            const uint32_t tb = sel(c, kk.y, kk.x);
            lt |= und & tb & ~rr[q];
            und &= ~(tb ^ rr[q]);
        }
    }
}

// The 8 unconditional planes (0 = most significant) of the lazy comparison in
// two 3-input chains, two instructions per plane: walking the planes from
// the least significant one up, "less than so far" needs no "equal so far"
// term (lt' = ~r t | ~(r ^ t) lt), and the undecided lanes are the AND of the
// planes' equalities.  Same (lt, und) as eight MSB-first steps from (0, u);
// `lt` is only meaningful on the lanes of u.
__device__ __forceinline__ void compare8(const uint32_t (&t)[8], const uint32_t (&r)[8], uint32_t u,
                                         uint32_t& und, uint32_t& lt) {
    uint32_t l = t[7] & ~r[7], e = u;
#pragma unroll
    for (int b = 6; b >= 0; --b) l = lop3<0x8E>(r[b], t[b], l);
#pragma unroll
    for (int b = 0; b < 8; ++b) e = lop3<0x90>(e, r[b], t[b]);
    lt = l;
    und = e;
}

// compare8 with the one-level threshold select of compare4_sel.
__device__ __forceinline__ void compare8_sel(uint32_t c, const uint4& k2a, const uint4& k2b, const uint4& k3a,
                                             const uint4& k3b, const u32x4& r0, const u32x4& r1, uint32_t u,
                                             uint32_t& und, uint32_t& lt) {
    const uint32_t t[8] = {sel(c, k3a.x, k2a.x), sel(c, k3a.y, k2a.y), sel(c, k3a.z, k2a.z), sel(c, k3a.w, k2a.w),
                           sel(c, k3b.x, k2b.x), sel(c, k3b.y, k2b.y), sel(c, k3b.z, k2b.z), sel(c, k3b.w, k2b.w)};
    const uint32_t r[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    compare8(t, r, u, und, lt);
}

// Pruned compare of 4 planes with thresholds already in registers: lanes
// with c set compare against class-3 planes k3, the others against k2.
__device__ __forceinline__ void compare4_sel(uint32_t c, const uint4& k2, const uint4& k3,
                                             const u32x4& r, uint32_t& und, uint32_t& lt) {
    const uint32_t t0 = sel(c, k3.x, k2.x), t1 = sel(c, k3.y, k2.y);
    const uint32_t t2 = sel(c, k3.z, k2.z), t3 = sel(c, k3.w, k2.w);
    lt |= und & t0 & ~r.x; und &= ~(t0 ^ r.x);
    lt |= und & t1 & ~r.y; und &= ~(t1 ^ r.y);
    lt |= und & t2 & ~r.z; und &= ~(t2 ^ r.z);
    lt |= und & t3 & ~r.w; und &= ~(t3 ^ r.w);
}

}  // namespace tg
