// oracle/alt_sweep.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Replacement translation unit for /root/reference/proj/src/mc.cpp, linked in
// its place to build the O2 variants that the reference does not ship:
//   ALT_RULE=1   heat-bath (Gibbs / p-bit) update, s_i = +1 iff u < sigma(2 beta h_i),
//                with the reference's one-draw-per-spin contract and f/g bookkeeping
//                (mc.cpp:21-35, test_mc.cpp:52-61);
//   ALT_PLANE=1  bit-plane draws keyed by physical state (philox_ref.h), the RNG
//                association of the B200 PLANE engine.  Needs the shadow SweepState
//                of oracle/shadow_plane/tempergrid/mc.hpp.
//   ALT_PLANE=2  packed draws keyed by physical state (philox_ref.h tgo_pack_u53),
//                the RNG association of the B200 FLOAT engine (same shadow).
// make_sweep_state / refresh_sweep_state restate mc.cpp:7-19 unchanged.
#include <cmath>
#include <cstdint>
#include <vector>

#include "tempergrid/mc.hpp"

#ifndef ALT_RULE
#define ALT_RULE 0
#endif
#ifndef ALT_PLANE
#define ALT_PLANE 0
#endif

namespace tgref_ctx {
// Installed by ref_harness.cpp around each run_2dpt call (plane builds only):
// the master seed and replica count, so a slot stream's seed can be mapped
// back to its slot index (derive_seed is a bijection of the index).
thread_local std::uint64_t master = 0;
thread_local int n_replicas = 0;
}  // namespace tgref_ctx

namespace tempergrid {

SweepState make_sweep_state(const EffectiveModel& view, SpinState spins) {
    SweepState state;
    state.spins = std::move(spins);
    refresh_sweep_state(view, state);
    return state;
}

void refresh_sweep_state(const EffectiveModel& view, SweepState& state) {
    state.local = local_fields(view.merged, state.spins);
    const EnergyBreakdown eb = energy_breakdown(view, state.spins);
    state.f = eb.f;
    state.g = eb.g;
}

namespace {

#if ALT_PLANE
int slot_of_seed(std::uint64_t seed) {
    for (int r = 0; r < tgref_ctx::n_replicas; ++r)
        if (derive_seed(tgref_ctx::master, StreamPurpose::replica, r) == seed) return r;
    return -1;
}
#endif

}  // namespace

void metropolis_sweep(const EffectiveModel& view, double beta, SweepState& state,
                      RngStream& rng) {
    const int n = view.merged.n_spins();
#if ALT_PLANE
    // Every configuration sweeps first in the slot it was created in, so the
    // slot stream seen at its first sweep names the physical state.
    if (state.plane_id < 0) state.plane_id = slot_of_seed(rng.seed());
    const std::uint64_t pkey = tgo_derive_seed(tgref_ctx::master,
                                               ALT_PLANE == 2 ? TGO_PURPOSE_PACK : TGO_PURPOSE_PLANE, 0);
    const std::uint32_t grp = (std::uint32_t)(state.plane_id >> 5);
    const int lane = state.plane_id & 31;
    const std::uint64_t t = state.plane_t++;
#endif
    for (int i = 0; i < n; ++i) {
        const double local_i = state.local[i];
        const double de = 2.0 * static_cast<double>(state.spins[i]) * local_i;
#if ALT_PLANE == 2
        const double u = tgo_u53_to_unit(tgo_pack_u53(pkey, (std::uint32_t)state.plane_id, t, (std::uint32_t)i));
        (void)grp; (void)lane;
#elif ALT_PLANE
        const double u = tgo_u53_to_unit(tgo_plane_u53(pkey, grp, t, (std::uint32_t)i, lane));
#else
        const double u = rng.uniform01();
#endif
#if ALT_RULE == 0
        const bool flip = de <= 0.0 || u < std::exp(-beta * de);
#else
        const double p = 1.0 / (1.0 + std::exp(-2.0 * beta * local_i));
        const Spin nv = u < p ? Spin{1} : Spin{-1};
        const bool flip = nv != state.spins[i];
#endif
        if (flip) {
            const double dg = view.constraints.delta_flip(state.spins, i);
            apply_flip(view.merged, state.spins, i, state.local);
            state.f += de - view.penalty * dg;
            state.g += dg;
        }
    }
}

}  // namespace tempergrid
