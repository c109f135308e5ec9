// plane_sweep.cu -- PLANE engine sweep kernel (multi-spin coding), compiled
// once per update rule (-DTG_PLANE_RULE=0 Metropolis, =1 heat bath).
//
// Restates metropolis_sweep (/root/reference/proj/src/mc.cpp:21-35) over the
// canonical colour order for J = +-1, h = 0 instances: bit l of word w at a
// site is the spin of physical replica 32w+l; a lane's flip probability is
// replaced by its 53-bit threshold K (exact host-side exp, engine.cpp
// semantics) compared MSB-first against bit planes of Philox draws.
#include <cooperative_groups.h>
#include <cuda_pipeline.h>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"
#include "plane_device.cuh"
#include "plane_round.cuh"

namespace cg = cooperative_groups;

#ifndef TG_PLANE_RULE
#define TG_PLANE_RULE 0
#endif
#define TG_CAT2(a, b) a##b
#define TG_CAT(a, b) TG_CAT2(a, b)

namespace tg {

// In-warp compaction of undecided (site, word) pairs in the FAST/prefetch path
// (TAIL = 2 below; TAIL = 0: each word runs its own lazy loop).
constexpr int kPfTail = 2;

// One thread = one site of the chunk; all WV words (32 replicas each) of the
// site row [wb, wb+WV) are loaded as one vector, updated, stored back.
template <int NCB, int NQB, int RULE, int WV, int TAIL, int PF = 0>
__device__ __forceinline__ void plane_site(const PlaneArgs& a, const Chunk& ch, const PlaneType& ty,
                                           int wb, uint64_t t, bool count, int lower,
                                           int (&acc_c)[WV], int (&acc_q)[WV],
                                           const uint32_t* pfrow = nullptr,
                                           const int32_t* pfidx = nullptr) {
    constexpr int DCM = (1 << NCB) - 1;
    constexpr int DQM = (1 << NQB) - 1;
    constexpr int B = NCB + NQB;
    const int lane = threadIdx.x & 31;
    const int dc = ty.dc, dq = ty.dq, deg = dc + dq;
    const bool valid = lane < ch.len;
    const int site = ch.start + lane;
    const int Wp = a.W;

    uint32_t s[WV];
    uint32_t x[DCM > 0 ? DCM : 1][WV];
    uint32_t y[DQM > 0 ? DQM : 1][WV];
    uint32_t lowx = 0, lowy = 0;
#pragma unroll
    for (int w = 0; w < WV; ++w) s[w] = 0u;
    if (valid) {
        // rows come from global memory, or from this warp's shared-memory
        // stage filled by cp.async one chunk ahead (PF): row r of lane l at
        // pfrow[(r*32 + l)*WV], neighbour entries at pfidx[k*32 + l]
        if constexpr (PF) load_row<WV>(pfrow + (size_t)lane * WV, s);
        else load_row<WV>(a.spins + (size_t)site * Wp + wb, s);
        const int32_t* nb = a.nbr + ch.nbr_base + (size_t)lane * deg;
#pragma unroll
        for (int k = 0; k < DCM; ++k) {
            if (k < dc) {
                const int32_t e = PF ? pfidx[k * 32 + lane] : __ldg(nb + k);
                const int j = e & 0x7fffffff;
                const uint32_t neg = e < 0 ? 0xffffffffu : 0u;
                if constexpr (PF) load_row<WV>(pfrow + (size_t)((1 + k) * 32 + lane) * WV, x[k]);
                else load_row<WV>(a.spins + (size_t)j * Wp + wb, x[k]);
#pragma unroll
                for (int w = 0; w < WV; ++w) x[k][w] ^= neg;  // bit: J_ij s_j = +1
                lowx |= (uint32_t)(j < lower) << k;
            } else {
#pragma unroll
                for (int w = 0; w < WV; ++w) x[k][w] = 0u;
            }
        }
#pragma unroll
        for (int k = 0; k < DQM; ++k) {
            if (k < dq) {
                const int j = PF ? pfidx[(dc + k) * 32 + lane] : __ldg(nb + dc + k);
                if constexpr (PF) load_row<WV>(pfrow + (size_t)((1 + dc + k) * 32 + lane) * WV, y[k]);
                else load_row<WV>(a.spins + (size_t)j * Wp + wb, y[k]);
                lowy |= (uint32_t)(j < lower) << k;
            } else {
#pragma unroll
                for (int w = 0; w < WV; ++w) y[k][w] = 0u;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < (DCM > 0 ? DCM : 1); ++k)
#pragma unroll
            for (int w = 0; w < WV; ++w) x[k][w] = 0u;
#pragma unroll
        for (int k = 0; k < (DQM > 0 ? DQM : 1); ++k)
#pragma unroll
            for (int w = 0; w < WV; ++w) y[k][w] = 0u;
    }
    const int ncl = ty.ncl;
    uint32_t ns[WV];
    if constexpr (TAIL == 2) {
        // ---- pass 1: class bits and the first 8 planes of every word
        uint32_t cbw[WV][B > 0 ? B : 1], alw[WV], undw[WV], ltw[WV];
        const bool pruned = (RULE == 0 && NQB == 0 && NCB == 2 && dc == 3);
        const uint32_t thi = (uint32_t)(t >> 32), tlo = (uint32_t)t;
        const int ncl = ty.ncl;
#pragma unroll
        for (int w = 0; w < WV; ++w) {
#pragma unroll
            for (int b = 0; b < (B > 0 ? B : 1); ++b) cbw[w][b] = 0u;
#pragma unroll
            for (int k = 0; k < DCM; ++k)
                if (k < dc) bs_add<NCB>(cbw[w], RULE == 0 ? ~(s[w] ^ x[k][w]) : x[k][w]);
#pragma unroll
            for (int k = 0; k < DQM; ++k)
                if (k < dq) bs_add<NQB>(cbw[w] + NCB, RULE == 0 ? ~(s[w] ^ y[k][w]) : y[k][w]);
            const uint32_t* kpb = a.kp + (size_t)(wb + w) * a.kpw + ty.kp_off;
            const uint32_t act = valid ? a.active[wb + w] : 0u;
            alw[w] = mux_tree<B>(cbw[w], kpb + kKPlanes * ncl) & act;
            undw[w] = act & ~alw[w];
            ltw[w] = 0u;
            const uint32_t grp4 = (uint32_t)(a.w_global0 + wb + w) << 4;
            const u32x4 r0 = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | 0u}, a.pks);
            const u32x4 r1 = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | 1u}, a.pks);
            if (pruned) {
                const uint4* kc2 = reinterpret_cast<const uint4*>(
                    a.kpc + ((size_t)(wb + w) * a.n_types + ch.type) * 128);
                compare4_sel(cbw[w][0], __ldg(kc2 + 0), __ldg(kc2 + 16), r0, undw[w], ltw[w]);
                compare4_sel(cbw[w][0], __ldg(kc2 + 1), __ldg(kc2 + 17), r1, undw[w], ltw[w]);
            } else {
                compare_block<B>(cbw[w], kpb, ncl, 0, r0, undw[w], ltw[w]);
                compare_block<B>(cbw[w], kpb, ncl, 1, r1, undw[w], ltw[w]);
            }
        }
        // ---- pass 2: (thread, word) pairs still undecided are packed onto
        // consecutive lanes and finish the lazy comparison together, one pair
        // per lane, instead of each word dragging the whole warp through
        // further Philox blocks.
        uint32_t pend[WV];
        int off[WV + 1];
        off[0] = 0;
#pragma unroll
        for (int w = 0; w < WV; ++w) {
            pend[w] = __ballot_sync(0xffffffffu, undw[w] != 0u);
            off[w + 1] = off[w] + __popc(pend[w]);
        }
        const int P = off[WV];
        for (int b0 = 0; b0 < P; b0 += 32) {
            const int pi = b0 + lane;
            const bool mine = pi < P;
            int pw = 0;
#pragma unroll
            for (int w = 1; w < WV; ++w) pw += (pi >= off[w]) ? 1 : 0;
            int src = 0;
            if (mine) {  // rank-th set bit of pend[pw]
                uint32_t mm = 0u;
                int r = pi;
#pragma unroll
                for (int w = 0; w < WV; ++w) if (w == pw) { mm = pend[w]; r -= off[w]; }
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) {
                    const int c = __popc(mm & ((1u << st) - 1u));
                    if (r >= c) { r -= c; mm >>= st; src += st; }
                }
            }
            uint32_t u = 0u, cbp[B > 0 ? B : 1];
#pragma unroll
            for (int b = 0; b < (B > 0 ? B : 1); ++b) cbp[b] = 0u;
#pragma unroll
            for (int w = 0; w < WV; ++w) {
                const uint32_t v = __shfl_sync(0xffffffffu, undw[w], src);
                if (w == pw) u = v;
#pragma unroll
                for (int b = 0; b < (B > 0 ? B : 1); ++b) {
                    const uint32_t cv = __shfl_sync(0xffffffffu, cbw[w][b], src);
                    if (w == pw) cbp[b] = cv;
                }
            }
            if (!mine) u = 0u;
            const int psite = ch.start + src;
            const uint32_t pgrp4 = (uint32_t)(a.w_global0 + wb + pw) << 4;
            const uint32_t* kpb = a.kp + (size_t)(wb + pw) * a.kpw + ty.kp_off;
            const uint4* kc2 = reinterpret_cast<const uint4*>(
                a.kpc + ((size_t)(wb + pw) * a.n_types + ch.type) * 128);
            uint32_t lx = 0u;
#pragma unroll 1
            for (int blk = 2; blk < 14; ++blk) {
                if (!__any_sync(0xffffffffu, u)) break;
                const u32x4 r = philox4x32_10_ks(u32x4{(uint32_t)psite, tlo, thi, pgrp4 | (uint32_t)blk}, a.pks);
                if (pruned) compare4_sel(cbp[0], __ldg(kc2 + blk), __ldg(kc2 + 16 + blk), r, u, lx);
                else compare_block<B>(cbp, kpb, ncl, blk, r, u, lx);
            }
            // return each pair's extra "take" lanes to its owner
#pragma unroll
            for (int w = 0; w < WV; ++w) {
                const int mypi = off[w] + __popc(pend[w] & ((1u << lane) - 1u));
                const int dst = mypi - b0;
                const uint32_t v = __shfl_sync(0xffffffffu, lx, dst & 31);
                if (undw[w] != 0u && dst >= 0 && dst < 32) ltw[w] |= v;
            }
        }
        // ---- pass 3: new words, energy counts
#pragma unroll
        for (int w = 0; w < WV; ++w) {
            const uint32_t act = valid ? a.active[wb + w] : 0u;
            const uint32_t take = (alw[w] | ltw[w]) & act;
            ns[w] = RULE == 0 ? (s[w] ^ take) : ((s[w] & ~act) | take);
            if (count) {
                if constexpr (NCB > 0) {
                    uint32_t m[NCB];
#pragma unroll
                    for (int b = 0; b < NCB; ++b) m[b] = 0u;
#pragma unroll
                    for (int k = 0; k < DCM; ++k)
                        if (k < dc && ((lowx >> k) & 1u)) bs_add<NCB>(m, (ns[w] ^ x[k][w]) & act);
                    int tot = 0;
#pragma unroll
                    for (int b = 0; b < NCB; ++b)
                        if (__any_sync(0xffffffffu, m[b])) tot += __popc(warp_transpose32(m[b])) << b;
                    acc_c[w] += tot;
                }
                if constexpr (NQB > 0) {
                    uint32_t m[NQB];
#pragma unroll
                    for (int b = 0; b < NQB; ++b) m[b] = 0u;
#pragma unroll
                    for (int k = 0; k < DQM; ++k)
                        if (k < dq && ((lowy >> k) & 1u)) bs_add<NQB>(m, (ns[w] ^ y[k][w]) & act);
                    int tot = 0;
#pragma unroll
                    for (int b = 0; b < NQB; ++b)
                        if (__any_sync(0xffffffffu, m[b])) tot += __popc(warp_transpose32(m[b])) << b;
                    acc_q[w] += tot;
                }
            }
        }
    } else {
#pragma unroll
    for (int w = 0; w < WV; ++w) {
        uint32_t cb[B > 0 ? B : 1];
#pragma unroll
        for (int b = 0; b < (B > 0 ? B : 1); ++b) cb[b] = 0u;
#pragma unroll
        for (int k = 0; k < DCM; ++k)
            if (k < dc) bs_add<NCB>(cb, RULE == 0 ? ~(s[w] ^ x[k][w]) : x[k][w]);
#pragma unroll
        for (int k = 0; k < DQM; ++k)
            if (k < dq) bs_add<NQB>(cb + NCB, RULE == 0 ? ~(s[w] ^ y[k][w]) : y[k][w]);
        const uint32_t* kpb = a.kp + (size_t)(wb + w) * a.kpw + ty.kp_off;
        const uint32_t act = valid ? a.active[wb + w] : 0u;
        const uint32_t always = mux_tree<B>(cb, kpb + kKPlanes * ncl) & act;
        // Metropolis without chain partners: de = 2(2 n_c - dc) > 0 only for
        // n_c > dc/2; for dc <= 3 those classes differ in bit 0 at most, so
        // the threshold of an undecided lane is a 1-level select.
        const bool pruned = (RULE == 0 && NQB == 0 && NCB == 2 && dc == 3);
        uint32_t und = act & ~always;
        uint32_t lt = 0;
        const uint32_t thi = (uint32_t)(t >> 32), tlo = (uint32_t)t;
        const uint32_t grp4 = (uint32_t)(a.w_global0 + wb + w) << 4;  // stream id in the counter
        // The first two blocks (8 planes) are almost always needed by some
        // lane of the warp: issue them unconditionally as independent chains.
        const u32x4 r0 = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | 0u}, a.pks);
        const u32x4 r1 = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | 1u}, a.pks);
        // class-major planes of the two threshold classes (pruned types)
        const uint4* kc2 = reinterpret_cast<const uint4*>(
            a.kpc + ((size_t)(wb + w) * a.n_types + ch.type) * 128);
        if (pruned) {
            compare4_sel(cb[0], __ldg(kc2 + 0), __ldg(kc2 + 16), r0, und, lt);
            compare4_sel(cb[0], __ldg(kc2 + 1), __ldg(kc2 + 17), r1, und, lt);
        } else {
            compare_block<B>(cb, kpb, ncl, 0, r0, und, lt);
            compare_block<B>(cb, kpb, ncl, 1, r1, und, lt);
        }
        {
#pragma unroll 1
            for (int blk = 2; blk < 14; ++blk) {
                if (!__any_sync(0xffffffffu, und)) break;
                const u32x4 r = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | (uint32_t)blk}, a.pks);
                if (pruned) compare4_sel(cb[0], __ldg(kc2 + blk), __ldg(kc2 + 16 + blk), r, und, lt);
                else compare_block<B>(cb, kpb, ncl, blk, r, und, lt);
            }
        }
        const uint32_t take = (always | lt) & act;
        ns[w] = RULE == 0 ? (s[w] ^ take) : ((s[w] & ~act) | take);
        if (count) {
            // unsatisfied bonds to lower-colour neighbours, counted once per
            // edge at its higher-colour endpoint, summed per replica lane.
            if constexpr (NCB > 0) {
                uint32_t m[NCB];
#pragma unroll
                for (int b = 0; b < NCB; ++b) m[b] = 0u;
#pragma unroll
                for (int k = 0; k < DCM; ++k)
                    if (k < dc && ((lowx >> k) & 1u)) bs_add<NCB>(m, (ns[w] ^ x[k][w]) & act);
                int tot = 0;
#pragma unroll
                for (int b = 0; b < NCB; ++b)
                    if (__any_sync(0xffffffffu, m[b])) tot += __popc(warp_transpose32(m[b])) << b;
                acc_c[w] += tot;
            }
            if constexpr (NQB > 0) {
                uint32_t m[NQB];
#pragma unroll
                for (int b = 0; b < NQB; ++b) m[b] = 0u;
#pragma unroll
                for (int k = 0; k < DQM; ++k)
                    if (k < dq && ((lowy >> k) & 1u)) bs_add<NQB>(m, (ns[w] ^ y[k][w]) & act);
                int tot = 0;
#pragma unroll
                for (int b = 0; b < NQB; ++b)
                    if (__any_sync(0xffffffffu, m[b])) tot += __popc(warp_transpose32(m[b])) << b;
                acc_q[w] += tot;
            }
        }
    }
    }
    if (valid) store_row<WV>(a.spins + (size_t)site * Wp + wb, ns);
}

// FAST = 1: only site types with cost degree <= 3 and chain degree <= 1
// (the config-5 graphs); the host picks the kernel from the type table.
template <int RULE, int WV, int FAST, int TAIL>
__device__ __forceinline__ void plane_dispatch(const PlaneArgs& a, const Chunk& ch, int wb,
                                               uint64_t t, bool count, int lower,
                                               int (&acc_c)[WV], int (&acc_q)[WV]) {
    const PlaneType& ty = a.ty[ch.type];
#define TG_CASE(C, Q) \
    case (C) * 4 + (Q): plane_site<C, Q, RULE, WV, TAIL>(a, ch, ty, wb, t, count, lower, acc_c, acc_q); break;
    if constexpr (FAST) {
        switch (ty.ncb * 4 + ty.nqb) {
            TG_CASE(0, 0) TG_CASE(0, 1)
            TG_CASE(1, 0) TG_CASE(1, 1) TG_CASE(2, 0) TG_CASE(2, 1)
            default: break;
        }
    } else {
        switch (ty.ncb * 4 + ty.nqb) {
            TG_CASE(0, 0) TG_CASE(0, 1) TG_CASE(0, 2)
            TG_CASE(1, 0) TG_CASE(1, 1) TG_CASE(1, 2)
            TG_CASE(2, 0) TG_CASE(2, 1) TG_CASE(2, 2)
            TG_CASE(3, 0) TG_CASE(3, 1) TG_CASE(3, 2)
            default: break;
        }
    }
#undef TG_CASE
}

// One colour phase of one sweep over this warp's items; unsatisfied-bond
// counts (last sweep of a round) go to cnt_c/cnt_q.
template <int RULE, int WV, int FAST>
__device__ __forceinline__ void plane_phase(const PlaneArgs& a, int c, uint64_t t, bool count,
                                            int gidx, int ngroups, int wb,
                                            int32_t* cnt_c, int32_t* cnt_q) {
    int acc_c[WV], acc_q[WV];
#pragma unroll
    for (int w = 0; w < WV; ++w) { acc_c[w] = 0; acc_q[w] = 0; }
    const int c0 = a.chunk_off[c];
    const int n_chunks = a.chunk_off[c + 1] - c0;
    const int lower = a.color_start[c];
    count = count && lower > 0;  // colour 0 has no lower-colour neighbours: nothing to count
    for (int item = gidx; item < n_chunks; item += ngroups) {
        const Chunk ch = a.chunks[c0 + item];
        plane_dispatch<RULE, WV, FAST, 0>(a, ch, wb, t, count, lower, acc_c, acc_q);
    }
    if (count) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int w = 0; w < WV; ++w) {
            const int m = (wb + w) * 32 + lane;
            if (m < a.local_states) {
                if (acc_c[w]) atomicAdd(cnt_c + m, acc_c[w]);
                if (acc_q[w]) atomicAdd(cnt_q + m, acc_q[w]);
            }
        }
    }
}


// Software-pipelined phase for the FAST site types (deg <= 4) with WV = 4:
// while chunk k is computed, the neighbour entries and the five 16-byte rows
// of chunk k+1 stream into this warp's other shared-memory stage with
// cp.async (LDGSTS) -- the L2 latency of the random neighbour gathers is
// hidden behind a chunk of Philox/compare work instead of stalling the warp.
constexpr int kPfRows = 5;                     // own row + up to 4 neighbours
template <int WV>
__host__ __device__ constexpr int pf_stage_words() { return kPfRows * 32 * WV + 4 * 32; }  // rows + neighbour entries
template <int RULE, int WV>
__device__ __forceinline__ void plane_phase_pf(const PlaneArgs& a, int c, uint64_t t, bool count,
                                               int gidx, int ngroups, int wb, int32_t* cnt_c,
                                               int32_t* cnt_q, uint32_t* pf) {
    constexpr int kStage = pf_stage_words<WV>();
    int acc_c[WV], acc_q[WV];
#pragma unroll
    for (int w = 0; w < WV; ++w) { acc_c[w] = 0; acc_q[w] = 0; }
    const int c0 = a.chunk_off[c];
    const int n_chunks = a.chunk_off[c + 1] - c0;
    const int lower = a.color_start[c];
    count = count && lower > 0;
    const int lane = threadIdx.x & 31;
    const int Wp = a.W;
    auto issue = [&](int item, int stage) {
        const Chunk ch = a.chunks[c0 + item];
        const PlaneType& ty = a.ty[ch.type];
        const int deg = ty.dc + ty.dq;
        uint32_t* rows = pf + stage * kStage;
        int32_t* idx = reinterpret_cast<int32_t*>(rows + kPfRows * 32 * WV);
        if (lane < ch.len) {
            const int site = ch.start + lane;
            __pipeline_memcpy_async(rows + lane * WV, a.spins + (size_t)site * Wp + wb, 4 * WV);
            for (int k = 0; k < deg; ++k) {
                const int32_t e = __ldg(a.nbr + ch.nbr_base + lane * deg + k);
                idx[k * 32 + lane] = e;
                __pipeline_memcpy_async(rows + ((1 + k) * 32 + lane) * WV,
                                        a.spins + (size_t)(e & 0x7fffffff) * Wp + wb, 4 * WV);
            }
        }
        __pipeline_commit();
        return ch;
    };
    int item = gidx;
    Chunk cur{};
    if (item < n_chunks) cur = issue(item, 0);
    int k = 0;
    while (item < n_chunks) {
        const int nxt = item + ngroups;
        Chunk next{};
        if (nxt < n_chunks) next = issue(nxt, (k + 1) & 1);
        else __pipeline_commit();
        __pipeline_wait_prior(1);
        __syncwarp();
        const uint32_t* rows = pf + (k & 1) * kStage;
        const int32_t* idx = reinterpret_cast<const int32_t*>(rows + kPfRows * 32 * WV);
        const PlaneType& ty = a.ty[cur.type];
        switch (ty.ncb * 4 + ty.nqb) {
            case 0 * 4 + 0: plane_site<0, 0, RULE, WV, kPfTail, 1>(a, cur, ty, wb, t, count, lower, acc_c, acc_q, rows, idx); break;
            case 0 * 4 + 1: plane_site<0, 1, RULE, WV, kPfTail, 1>(a, cur, ty, wb, t, count, lower, acc_c, acc_q, rows, idx); break;
            case 1 * 4 + 0: plane_site<1, 0, RULE, WV, kPfTail, 1>(a, cur, ty, wb, t, count, lower, acc_c, acc_q, rows, idx); break;
            case 1 * 4 + 1: plane_site<1, 1, RULE, WV, kPfTail, 1>(a, cur, ty, wb, t, count, lower, acc_c, acc_q, rows, idx); break;
            case 2 * 4 + 0: plane_site<2, 0, RULE, WV, kPfTail, 1>(a, cur, ty, wb, t, count, lower, acc_c, acc_q, rows, idx); break;
            case 2 * 4 + 1: plane_site<2, 1, RULE, WV, kPfTail, 1>(a, cur, ty, wb, t, count, lower, acc_c, acc_q, rows, idx); break;
            default: break;
        }
        __syncwarp();
        cur = next;
        item = nxt;
        ++k;
    }
    __pipeline_wait_prior(0);
    if (count) {
#pragma unroll
        for (int w = 0; w < WV; ++w) {
            const int m = (wb + w) * 32 + lane;
            if (m < a.local_states) {
                if (acc_c[w]) atomicAdd(cnt_c + m, acc_c[w]);
                if (acc_q[w]) atomicAdd(cnt_q + m, acc_q[w]);
            }
        }
    }
}

// Sweep-only cooperative kernel (multi-GPU path): all sweeps of one round;
// the (f, g) exchange and the swap run after it.  Work item = (chunk of <= 32
// same-type sites of one colour, pass of WV words).
template <int RULE, int WV>
__global__ void __launch_bounds__(kPlaneThreads, 1)
plane_sweep_kernel(const __grid_constant__ PlaneArgs a, int64_t t0, int n_sweeps) {
    if (a.rs) t0 = a.rs->round * n_sweeps;
    cg::grid_group grid = cg::this_grid();
    const int wpb = blockDim.x >> 5;
    // each block owns one pass of WV words (block-uniform Philox keys); the
    // blocks of a pass split its chunks (host: gridDim % passes == 0)
    const int passes = a.W / WV;
    const int wb = (int)(blockIdx.x % passes) * WV;
    const int gidx = (int)(blockIdx.x / passes) * wpb + (threadIdx.x >> 5);
    const int ngroups = (int)(gridDim.x / passes) * wpb;
    for (int sw = 0; sw < n_sweeps; ++sw) {
        const uint64_t t = (uint64_t)(t0 + sw);
        const bool count = (sw == n_sweeps - 1);
        for (int c = 0; c < a.n_colors; ++c) {
            plane_phase<RULE, WV, 0>(a, c, t, count, gidx, ngroups, wb, a.cnt_c, a.cnt_q);
            grid.sync();
        }
    }
    // Per-replica f and g (reference units) from the unsatisfied-bond counts:
    // f = -(m - 2 u_c) for J = +-1, h = 0; g = sum (s_a - s_b)^2 = 4 u_q.
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < a.local_states;
         m += gridDim.x * blockDim.x) {
        const int uc = a.cnt_c[m], uq = a.cnt_q[m];
        a.f_loc[m] = -((double)a.m_cost - 2.0 * (double)uc);
        a.g_loc[m] = 4.0 * (double)uq;
        a.cnt_c[m] = 0;
        a.cnt_q[m] = 0;
    }
}

// Persistent single-GPU kernel: n_rounds whole rounds of run_2dpt
// (engine.cpp:121-216) without leaving the device.  Per round: sps sweeps
// (one grid barrier per colour phase), then every block derives all
// replicas' (f, g) from the bond counts, replays the identical swap phase on
// its shared-memory copy of the labels, and rebuilds its share of the
// threshold planes; block 0 publishes labels, counters and the record; one
// more grid barrier closes the round.
template <int RULE, int WV, int FAST>
__global__ void __launch_bounds__(FAST ? kPlaneThreadsFast : kPlaneThreads,
                                  FAST ? (WV == 2 ? 2 : kPlaneMinBlocksFast) : 1)
plane_rounds_kernel(const __grid_constant__ PlaneArgs a, const __grid_constant__ RoundArgs r) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm_d[];
    double* s_f = sm_d;
    double* s_g = sm_d + r.R;
    int32_t* s_slot = reinterpret_cast<int32_t*>(sm_d + 2 * r.R);
    int32_t* s_state = s_slot + r.R;
    char* sm_pf = reinterpret_cast<char*>(s_state + r.R + (r.R & 1));  // cp.async row stages
    uint32_t* pfbuf = reinterpret_cast<uint32_t*>(sm_pf) +
                      (size_t)(threadIdx.x >> 5) * 2 * pf_stage_words<WV == 2 ? 2 : 4>();
    const int tid = threadIdx.x;
    const int wpb = blockDim.x >> 5;
    const int warp = tid >> 5;
    const int passes = a.W / WV;
    const int wb = (int)(blockIdx.x % passes) * WV;
    const int gidx = (int)(blockIdx.x / passes) * wpb + warp;
    const int ngroups = (int)(gridDim.x / passes) * wpb;
    for (int m = tid; m < r.R; m += blockDim.x) {
        s_slot[m] = r.slot_state[m];
        s_state[m] = r.state_slot[m];
    }
    uint64_t swap_base = r.swap_base0;
    for (int k = 0; k < r.n_rounds; ++k) {
        const int64_t round = r.round0 + k;
        const int par = (int)(round & 1);
        int32_t* cc = r.cnt + (size_t)par * 2 * r.cnt_stride;
        int32_t* cq = cc + r.cnt_stride;
        for (int sw = 0; sw < r.sps; ++sw) {
            const uint64_t t = (uint64_t)((round - 1) * r.sps + sw);
            const bool count = (sw == r.sps - 1);
            for (int c = 0; c < a.n_colors; ++c) {
                if constexpr (FAST && (WV == 4 || WV == 2))
                    plane_phase_pf<RULE, WV>(a, c, t, count, gidx, ngroups, wb, cc, cq, pfbuf);
                else plane_phase<RULE, WV, FAST>(a, c, t, count, gidx, ngroups, wb, cc, cq);
                grid.sync();
            }
        }
        round_epilogue(a, r, RoundSmem{s_f, s_g, s_slot, s_state}, k, round, cc, cq, swap_base, 0);
    }
}

template __global__ void plane_sweep_kernel<TG_PLANE_RULE, 1>(const __grid_constant__ PlaneArgs, int64_t, int);
template __global__ void plane_sweep_kernel<TG_PLANE_RULE, 2>(const __grid_constant__ PlaneArgs, int64_t, int);
template __global__ void plane_sweep_kernel<TG_PLANE_RULE, 4>(const __grid_constant__ PlaneArgs, int64_t, int);
template __global__ void plane_rounds_kernel<TG_PLANE_RULE, 1, 0>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);
template __global__ void plane_rounds_kernel<TG_PLANE_RULE, 2, 0>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);
template __global__ void plane_rounds_kernel<TG_PLANE_RULE, 4, 0>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);
template __global__ void plane_rounds_kernel<TG_PLANE_RULE, 4, 1>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);
template __global__ void plane_rounds_kernel<TG_PLANE_RULE, 2, 1>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);
template __global__ void plane_rounds_kernel<TG_PLANE_RULE, 1, 1>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);



void* TG_CAT(plane_rounds_fn_r, TG_PLANE_RULE)(int wv, int fast) {
    if (wv >= 4) return fast ? (void*)plane_rounds_kernel<TG_PLANE_RULE, 4, 1>
                             : (void*)plane_rounds_kernel<TG_PLANE_RULE, 4, 0>;
    if (wv >= 2) return fast ? (void*)plane_rounds_kernel<TG_PLANE_RULE, 2, 1>
                             : (void*)plane_rounds_kernel<TG_PLANE_RULE, 2, 0>;
    return fast ? (void*)plane_rounds_kernel<TG_PLANE_RULE, 1, 1>
                : (void*)plane_rounds_kernel<TG_PLANE_RULE, 1, 0>;
}

void* TG_CAT(plane_sweep_fn_r, TG_PLANE_RULE)(int wv) {
    return wv >= 4 ? (void*)plane_sweep_kernel<TG_PLANE_RULE, 4>
                   : (wv >= 2 ? (void*)plane_sweep_kernel<TG_PLANE_RULE, 2>
                              : (void*)plane_sweep_kernel<TG_PLANE_RULE, 1>);
}

}  // namespace tg
