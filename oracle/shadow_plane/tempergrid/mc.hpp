// oracle/shadow_plane/tempergrid/mc.hpp -- TEST INFRASTRUCTURE ONLY.
//
// Shadow of the reference sweep interface (/root/reference/proj/include/
// tempergrid/mc.hpp:13-30) for the "O2-plane" oracle build.  Same functions
// and SweepState members as the reference, plus two trailing members that
// travel with a configuration when engine.cpp swaps states
// (std::swap(a.state, b.state), engine.cpp:160,182): the physical state id
// and its sweep counter.  They let oracle/alt_sweep.cpp key bit-plane draws
// by physical state, the association the B200 "msc" engine uses.
#pragma once

#include <cstdint>

#include "tempergrid/constraints.hpp"
#include "tempergrid/ising.hpp"
#include "tempergrid/rng.hpp"

namespace tempergrid {

struct SweepState {
    SpinState spins;
    LocalFields local;
    double f = 0.0;
    double g = 0.0;
    int plane_id = -1;           // physical state id, adopted at first sweep
    std::uint64_t plane_t = 0;   // sweeps performed by this configuration
};

SweepState make_sweep_state(const EffectiveModel& view, SpinState spins);
void refresh_sweep_state(const EffectiveModel& view, SweepState& state);
void metropolis_sweep(const EffectiveModel& view, double beta,
                      SweepState& state, RngStream& rng);

}  // namespace tempergrid
