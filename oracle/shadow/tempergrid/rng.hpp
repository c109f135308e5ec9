// oracle/shadow/tempergrid/rng.hpp -- TEST INFRASTRUCTURE ONLY.
//
// Drop-in shadow for /root/reference/proj/include/tempergrid/rng.hpp used to
// build oracle "O2": the unmodified reference sources compiled with
// `-I oracle/shadow` placed before the reference include directory, so that
// every `#include "tempergrid/rng.hpp"` of the reference resolves here.
//
// It keeps the reference's public surface byte-compatible -- detail::mix64,
// StreamPurpose, derive_seed (rng.hpp:13-40) and every RngStream member
// (rng.hpp:47-83) with the same formulas for uniform01, below, normal and
// spin -- and replaces only the engine: std::mt19937_64 (rng.hpp:82) becomes
// the counter-based Philox4x32-10 stream of oracle/philox_ref.h, so the k-th
// bits() of stream(seed) is a pure function of (seed, k).  The reference fed
// through this header consumes exactly the draws the B200 engine computes.
#pragma once

#include <cmath>
#include <cstdint>

#include "../../philox_ref.h"

namespace tempergrid {

namespace detail {

inline std::uint64_t mix64(std::uint64_t z) { return tgo_mix64(z); }

}  // namespace detail

enum class StreamPurpose : std::uint64_t {
    replica = 1,
    swap = 2,
    init = 3,
    probe = 4,
    repeat = 5,
    sampling = 6,
    bootstrap = 7,
};

inline std::uint64_t derive_seed(std::uint64_t master, StreamPurpose purpose,
                                 std::uint64_t index) {
    return tgo_derive_seed(master, static_cast<std::uint64_t>(purpose), index);
}

class RngStream {
public:
    RngStream() : seed_(0), n_(0) {}
    explicit RngStream(std::uint64_t seed) : seed_(seed), n_(0) {}

    std::uint64_t bits() { return tgo_stream_bits(seed_, n_++); }

    double uniform01() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }

    std::uint64_t below(std::uint64_t n) {
        const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        std::uint64_t x;
        do {
            x = bits();
        } while (x >= limit);
        return x % n;
    }

    double normal() {
        double u1;
        do {
            u1 = uniform01();
        } while (u1 <= 0.0);
        const double u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        return r * std::cos(6.283185307179586476925286766559 * u2);
    }

    int spin() { return (bits() >> 63) ? 1 : -1; }

    // Shadow-only introspection (not used by the reference sources).
    std::uint64_t seed() const { return seed_; }
    std::uint64_t position() const { return n_; }

private:
    std::uint64_t seed_;
    std::uint64_t n_;
};

}  // namespace tempergrid
