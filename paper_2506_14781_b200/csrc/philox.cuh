// philox.cuh -- counter-based Philox4x32-10 and the stream-keying contract,
// host+device.  The same functions run in the sweep/swap kernels and in the
// host-side swap replay, so every draw is a pure function of
// (seed, purpose, index, counter).
//
// Keying restates the reference's seed derivation (rng.hpp:13-40:
// derive_seed = mix64(mix64(master ^ mix64(purpose)) ^ index)); the engine
// std::mt19937_64 (rng.hpp:82) is replaced by Philox4x32-10 (pinned against
// cuRAND's implementation by tests/golden/philox_kat.json).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD inline
#endif

namespace tg {

enum : uint64_t {
    kPurposeReplica = 1,
    kPurposeSwap = 2,
    kPurposeInit = 3,
    kPurposeProbe = 4,   // schedule probe chains (rng.hpp:27)
    kPurposeRepeat = 5,  // J-column baseline repeats (rng.hpp:28)
    kPurposePlane = 8,
    kPurposePack = 9,    // FLOAT engine packed draws (oracle/philox_ref.h tgo_pack_u53)
};

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

TG_HD uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

TG_HD uint64_t derive_seed(uint64_t master, uint64_t purpose, uint64_t index) {
    return mix64(mix64(master ^ mix64(purpose)) ^ index);
}

struct u32x4 {
    uint32_t x, y, z, w;
};

#ifndef TG_MULWIDE
#define TG_MULWIDE 0
#endif
TG_HD void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if defined(__CUDA_ARCH__) && TG_MULWIDE
    // one 32x32->64 multiply (IMAD.WIDE.U32) for both halves
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
#elif defined(__CUDA_ARCH__)
    hi = __umulhi(a, b);
    lo = a * b;
#else
    const uint64_t p = (uint64_t)a * b;
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
#endif
}

TG_HD u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(kPhiloxM0, c.x, hi0, lo0);
        mulhilo(kPhiloxM1, c.z, hi1, lo1);
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return c;
}

// Philox4x32-10 with a precomputed key schedule ks[2r], ks[2r+1] = key of
// round r.  With ks in the kernel's constant bank (compile-time offsets) the
// rounds need no key additions at all: the XOR takes the constant operand.
TG_HD u32x4 philox4x32_10_ks(u32x4 c, const uint32_t* ks) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(kPhiloxM0, c.x, hi0, lo0);
        mulhilo(kPhiloxM1, c.z, hi1, lo1);
        c = u32x4{hi1 ^ c.y ^ ks[2 * r], lo1, hi0 ^ c.w ^ ks[2 * r + 1], lo0};
    }
    return c;
}

TG_HD void philox_key_schedule(uint64_t key, uint32_t ks[20]) {
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int r = 0; r < 10; ++r) {
        ks[2 * r] = k0;
        ks[2 * r + 1] = k1;
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
}

// n-th 64-bit output of stream(seed): counter n>>1, words (0,1) or (2,3).
TG_HD uint64_t stream_bits(uint64_t seed, uint64_t n) {
    const uint64_t blk = n >> 1;
    const u32x4 o = philox4x32_10(u32x4{(uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u},
                                  (uint32_t)seed, (uint32_t)(seed >> 32));
    return (n & 1) ? ((uint64_t)o.z | ((uint64_t)o.w << 32))
                   : ((uint64_t)o.x | ((uint64_t)o.y << 32));
}

// Digest term of spin i (caller order) being +1.
TG_HD uint64_t digest_term(uint64_t i) { return mix64(i + 1); }

}  // namespace tg
