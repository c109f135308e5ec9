/*
 * oracle/philox_ref.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never
 * the product path).  Plain-C restatement of the random-stream contract the
 * B200 engine and every oracle share.
 *
 *   mix64 / derive_seed   restate /root/reference/proj/include/tempergrid/rng.hpp:13-40
 *                         (SplitMix64 finalizer; derive_seed = mix64(mix64(m ^ mix64(p)) ^ idx)).
 *   StreamPurpose values  rng.hpp:23-31 (replica=1, swap=2, init=3, ...) plus one
 *                         new purpose, PLANE=8, for the bit-plane sweep draws.
 *   philox4x32_10         the published Philox4x32-10 bijection (Salmon et al.,
 *                         SC'11), identical to cuRAND's curand_Philox4x32_10
 *                         (/usr/local/cuda/include/curand_philox4x32_x.h:160-186);
 *                         pinned by tests/golden/philox_kat.json.
 *
 * Stream semantics (replaces the std::mt19937_64 engine of rng.hpp:82; every
 * derived draw of rng.hpp:50-79 keeps its formula):
 *   stream(seed): key = {lo32(seed), hi32(seed)}; the n-th 64-bit output is
 *     c = philox(ctr = {lo32(n>>1), hi32(n>>1), 0, 0}, key)
 *     bits_n = (n even) ? c0 | c1<<32 : c2 | c3<<32
 *   uniform01 = (bits >> 11) * 2^-53        (rng.hpp:53-55)
 *   spin      = (bits >> 63) ? +1 : -1      (rng.hpp:79)
 *
 * Bit-plane draws (engine "plane"): the 53-bit uniform of physical state
 * m = 32*grp + lane at sweep t, site i is
 *   U53 = sum_{b=0..52} bit_lane( philox(ctr={i, lo32(t), hi32(t), (b>>2) | grp<<4},
 *                                       key(derive_seed(seed, PLANE, 0)))[b&3] ) << (52-b)
 *   u   = U53 * 2^-53.
 * One key per run (the stream identity of a 32-replica group lives in the
 * counter), so the device key schedule is a compile-time-addressed constant.
 *
 * Packed draws (engine "float"): the 53-bit uniform of physical state m at
 * sweep t, site i is U53 = hi16 << 37 | lo37 with
 *   hi16 = halfword (m & 7) of philox(ctr={i, lo32(t), hi32(t), (m>>3) | 1<<30}, key)
 *          (halfword h = bits 16*(h&1) .. +15 of word h>>1): one block serves
 *          8 consecutive states, whose decisions are nearly always settled
 *          by these 16 bits;
 *   lo37 = low 37 bits of (c0 | c1<<32) of philox(ctr={i, lo32(t), hi32(t), m | 2<<30}, key),
 * key = derive_seed(seed, PACK, 0).
 */
#ifndef TG_PHILOX_REF_H
#define TG_PHILOX_REF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TGO_PURPOSE_REPLICA = 1,
    TGO_PURPOSE_SWAP = 2,
    TGO_PURPOSE_INIT = 3,
    TGO_PURPOSE_PROBE = 4,
    TGO_PURPOSE_REPEAT = 5,
    TGO_PURPOSE_SAMPLING = 6,
    TGO_PURPOSE_BOOTSTRAP = 7,
    TGO_PURPOSE_PLANE = 8,
    TGO_PURPOSE_PACK = 9
};

static inline uint64_t tgo_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t tgo_derive_seed(uint64_t master, uint64_t purpose, uint64_t index) {
    const uint64_t p = tgo_mix64(purpose);
    return tgo_mix64(tgo_mix64(master ^ p) ^ index);
}

static inline void tgo_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                                     uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* n-th 64-bit output of stream(seed). */
static inline uint64_t tgo_stream_bits(uint64_t seed, uint64_t n) {
    const uint64_t blk = n >> 1;
    const uint32_t ctr[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    tgo_philox4x32_10(ctr, key, o);
    return (n & 1) ? ((uint64_t)o[2] | ((uint64_t)o[3] << 32))
                   : ((uint64_t)o[0] | ((uint64_t)o[1] << 32));
}

static inline double tgo_u53_to_unit(uint64_t u53) { return (double)u53 * 0x1.0p-53; }

/* 53-bit plane-assembled uniform of lane `lane` of 32-replica group `grp`
 * under run key `pkey` = derive_seed(seed, PLANE, 0), at sweep t, site i
 * (see header comment). */
static inline uint64_t tgo_plane_u53(uint64_t pkey, uint32_t grp, uint64_t t, uint32_t site, int lane) {
    const uint32_t key[2] = {(uint32_t)pkey, (uint32_t)(pkey >> 32)};
    uint64_t u = 0;
    for (int blk = 0; blk < 14; ++blk) {
        const uint32_t ctr[4] = {site, (uint32_t)t, (uint32_t)(t >> 32), (uint32_t)blk | (grp << 4)};
        uint32_t o[4];
        tgo_philox4x32_10(ctr, key, o);
        for (int w = 0; w < 4; ++w) {
            const int b = blk * 4 + w;
            if (b >= 53) break;
            u |= (uint64_t)((o[w] >> lane) & 1u) << (52 - b);
        }
    }
    return u;
}

/* Packed-draw 53-bit uniform of physical state m at sweep t, site i under run
 * key `pkey` = derive_seed(seed, PACK, 0) (see header comment). */
static inline uint64_t tgo_pack_u53(uint64_t pkey, uint32_t m, uint64_t t, uint32_t site) {
    const uint32_t key[2] = {(uint32_t)pkey, (uint32_t)(pkey >> 32)};
    uint32_t o[4];
    const uint32_t c1[4] = {site, (uint32_t)t, (uint32_t)(t >> 32), (m >> 3) | (1u << 30)};
    tgo_philox4x32_10(c1, key, o);
    const uint32_t h = m & 7u;
    const uint64_t hi16 = (o[h >> 1] >> (16u * (h & 1u))) & 0xFFFFu;
    const uint32_t c2[4] = {site, (uint32_t)t, (uint32_t)(t >> 32), m | (2u << 30)};
    tgo_philox4x32_10(c2, key, o);
    const uint64_t lo37 = ((uint64_t)o[0] | ((uint64_t)o[1] << 32)) & ((1ull << 37) - 1ull);
    return (hi16 << 37) | lo37;
}

/* Order-independent, position-keyed digest of a spin configuration:
 * sum over +1 spins of mix64(i + 1), mod 2^64. */
static inline uint64_t tgo_digest_term(uint64_t i) { return tgo_mix64(i + 1); }

#ifdef __cplusplus
}
#endif

#endif /* TG_PHILOX_REF_H */
