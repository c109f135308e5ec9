// plane_c5.cu -- the config-5 fused round kernel of the PLANE engine
// (Metropolis): two 32-replica words per thread, chain-free and chain sites
// in separate item loops.
//
// Both update rules (Metropolis; heat bath, the north star's p-bit rule).
// Same contract, and therefore the same trajectories bit for bit, as
// plane_tpw_rounds_kernel / plane_rounds_kernel: the reference sweep
// (mc.cpp:21-35) over the canonical colour order, thresholds
// K = ceil(T * 2^53) compared MSB-first against bit planes of Philox4x32-10
// draws with counter {site, t_lo, t_hi, group << 4 | block}, labels permuted
// by the swap phase (plane_round.cuh).  It applies to instances whose sites
// all have cost degree 3 (J = +-1, h = 0) and chain degree 0 or 1 with a
// proper 2-colouring (BASELINE config 5): every neighbour of a colour-1 site
// is colour 0, so the unsatisfied bonds a colour-1 site leaves behind are c if
// it flips and 3 - c otherwise (c = satisfied bonds before the update).
//
// Work layout: thread = (site, word pair); a warp item is S = 64 / W
// consecutive sites x the W / 2 word pairs of their rows (lane = site * W/2 +
// pair), so each row load is one 8-byte access per lane and W/2 lanes cover a
// whole 32-byte row.  Per colour phase the chain-free sites and the chain
// sites (contiguous in the canonical order) are walked by two loops, so every
// item is of one kind and no per-item type test or straddling exists.  Per
// thread and phase: the class-2/3 threshold planes 0-7 of both words in
// registers, 4 Philox blocks per chain-free item (the two unconditional blocks
// of each word, sharing the site's round-1/2/3 products), the 8 unconditional
// planes compared in two 3-input LOP3 chains (plane_device.cuh compare8).
// (Site, word)s still undecided after 8 planes -- chain-free and chain sites
// alike -- go to a per-warp shared-memory queue (one 16-byte record) resolved
// 32 at a time, one per lane (c5_drain, c5_drain_chain).  The bit-sliced bond
// counters are flushed once per phase (and every kC5FlushAt items).
// plane_c5_sweep_kernel is the sweep-only form for the unfused round loop.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"
#include "philox_plane.cuh"
#include "plane_device.cuh"
#include "plane_round.cuh"

namespace cg = cooperative_groups;

namespace tg {

constexpr int kC5VB = 8;  // vertical counter planes (<= 255 per lane between flushes)
constexpr int kC5FlushAt = 80;  // items (<= 3 bonds each) between flushes of the cost-bond counters

extern __shared__ __align__(16) int c5_sm[];

// Dynamic shared memory: queues [warps][kC5QCap] int4 | s_cc[32W] | s_cq[32W]
// | the round block (labels, energies) of plane_round.cuh.
__device__ __forceinline__ int4* c5_queue(int warp) {
    return reinterpret_cast<int4*>(c5_sm) + warp * kC5QCap;
}
__device__ __forceinline__ int* c5_cnt() { return c5_sm + (kC5Threads / 32) * kC5QCap * 4 + kMaxWordsArg * 36; }
// threshold planes staged per round for the chain-free type: Metropolis,
// class-2/3 planes 0-7 of every word, [4][W] uint4 (k2 planes 0-3, 4-7, k3
// planes 0-3, 4-7); heat bath, planes 0-7 and the "always" word of its 4
// classes, [9][W] uint4 (x..w = classes 0..3) -- part-major: the words of one
// warp's pairs are 32 bytes apart, so an LDS.128 is conflict-free
__device__ __forceinline__ uint4* c5_thr() { return reinterpret_cast<uint4*>(c5_sm + (kC5Threads / 32) * kC5QCap * 4); }

// V += m (2-bit bit-sliced value) in kC5VB-bit vertical arithmetic.
template <int NB>
__device__ __forceinline__ void c5_vadd(uint32_t (&V)[kC5VB], uint32_t m0, uint32_t m1) {
    uint32_t carry = 0u;
#pragma unroll
    for (int b = 0; b < kC5VB; ++b) {
        const uint32_t x = V[b];
        if (b < NB) {
            const uint32_t y = b == 0 ? m0 : m1;
            V[b] = x ^ y ^ carry;
            carry = (x & y) | (carry & (x ^ y));
        } else {
            V[b] = x ^ carry;
            carry = x & carry;
        }
    }
}

// Per-replica totals of the warp's vertical counters of word `j` of each
// lane's pair, added into s_cnt[(2 * pair + j) * 32 + replica]; V is
// cleared.  Lanes holding the same pair (lane = p * WP + pair) are summed by
// a butterfly; the sums' planes are packed S per 32x32 transpose, after which
// lane l reads replica l's bits of every pair.
template <int LOGWP>
__device__ __noinline__ void c5_vflush(uint4 lo, uint4 hi, int j, int* s_cnt) {
    constexpr int WP = 1 << LOGWP, LOGS = 5 - LOGWP, S = 1 << LOGS;
    constexpr int NB = kC5VB + LOGS;
    constexpr int NQ = (NB + S - 1) / S;
    const int lane = threadIdx.x & 31;
    uint32_t E[NB];
    const uint32_t V[kC5VB] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int b = 0; b < NB; ++b) E[b] = b < kC5VB ? V[b] : 0u;
#pragma unroll
    for (int lv = 0; lv < LOGS; ++lv) {
        uint32_t carry = 0u;
#pragma unroll
        for (int b = 0; b <= kC5VB + lv && b < NB; ++b) {
            const uint32_t x = E[b];
            const uint32_t o = __shfl_xor_sync(0xffffffffu, x, WP << lv);
            E[b] = x ^ o ^ carry;
            carry = (x & o) | (carry & (x ^ o));
        }
    }
    const int p_me = lane >> LOGWP;
    uint32_t T[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        uint32_t v = 0u;
#pragma unroll
        for (int p = 0; p < S; ++p)
            if (q * S + p < NB) v = (p == p_me) ? E[q * S + p] : v;
        T[q] = warp_transpose32(v);
    }
#pragma unroll
    for (int w = 0; w < WP; ++w) {
        int val = 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
#pragma unroll
            for (int p = 0; p < S; ++p)
                if (q * S + p < NB) val += (int)((T[q] >> (p * WP + w)) & 1u) << (q * S + p);
        }
        if (val) atomicAdd(s_cnt + (2 * w + j) * 32 + lane, val);
    }
}

__device__ __forceinline__ void c5_flush(uint32_t (&V)[kC5VB], int logWP, int j, int* s_cnt) {
    const uint4 lo = make_uint4(V[0], V[1], V[2], V[3]), hi = make_uint4(V[4], V[5], V[6], V[7]);
    switch (logWP) {
        case 0: c5_vflush<0>(lo, hi, j, s_cnt); break;
        case 1: c5_vflush<1>(lo, hi, j, s_cnt); break;
        case 2: c5_vflush<2>(lo, hi, j, s_cnt); break;
        case 3: c5_vflush<3>(lo, hi, j, s_cnt); break;
        default: c5_vflush<4>(lo, hi, j, s_cnt); break;
    }
#pragma unroll
    for (int b = 0; b < kC5VB; ++b) V[b] = 0u;
}

// Resolve queue entries [base, base + n) (n <= 32) of the calling warp, one
// per lane: Philox blocks 2.. of the entry's (site, word), threshold planes
// 8.. of its word, late decisions applied to the stored word (same warp, after
// __syncwarp) and, when counting, the unsatisfied-bond correction.
// Metropolis: undecided lanes are class 2 | 3 (c = 2 + c0), planes from kpc,
// a late flip changes the lane's unsatisfied bonds by 2c - 3 = 1 + 2 c0.
// Heat bath: 4 classes (c = c0 + 2 c1 +1 contributions), planes from kp, a
// late +1 (provisionally -1) changes them by 3 - 2c.
template <int RULE>
__device__ __noinline__ void c5_drain(const PlaneArgs& a, int base, int n, uint32_t tlo, uint32_t thi,
                                      int t30, bool count, int* s_cc) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    const bool mine = lane < n;
    int4 e = make_int4(0, 0, 0, 0);
    if (mine) e = c5_queue(threadIdx.x >> 5)[base + lane];
    const uint32_t site = (uint32_t)e.x & 0x07ffffffu;
    const int w = (int)((uint32_t)e.x >> 27);
    uint32_t und = (uint32_t)e.y;
    const uint32_t c0 = (uint32_t)e.z, c1 = (uint32_t)e.w;
    const uint32_t grp4 = (uint32_t)(a.w_global0 + w) << 4;
    const uint4* kc2 = reinterpret_cast<const uint4*>(a.kpc + ((size_t)w * a.n_types + t30) * 128);
    const uint4* kh = reinterpret_cast<const uint4*>(a.kp + (size_t)w * a.kpw + a.ty[t30].kp_off);
    uint32_t lt = 0u;
    const PhiloxT P = philox_t(tlo, thi, a.pks);
#pragma unroll 1
    for (int blk = 2; blk < 14; ++blk) {
        if (!__any_sync(0xffffffffu, und)) break;
        const u32x4 r = philox_plane(site, grp4 | (uint32_t)blk, P, a.pks);
        if (RULE == 0) {
            compare4_sel(c0, __ldg(kc2 + blk), __ldg(kc2 + 16 + blk), r, und, lt);
        } else {
            const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int b = blk * 4 + q;
                if (b < kKPlanes) {
                    const uint4 T = __ldg(kh + b);  // the 4 classes of plane b
                    const uint32_t tb = sel(c1, sel(c0, T.w, T.z), sel(c0, T.y, T.x));
                    lt |= und & tb & ~rr[q];
                    und &= ~(tb ^ rr[q]);
                }
            }
        }
    }
    if (lt) {
        if (RULE == 0) a.spins[(size_t)site * a.W + w] ^= lt;
        else a.spins[(size_t)site * a.W + w] |= lt;
        if (count) {
            uint32_t ex = lt;
            while (ex) {
                const int l = __ffs(ex) - 1;
                ex &= ex - 1;
                const int cl = (int)((c0 >> l) & 1u) + 2 * (int)((c1 >> l) & 1u);
                atomicAdd(s_cc + w * 32 + l, RULE == 0 ? 1 + 2 * (int)((c0 >> l) & 1u) : 3 - 2 * cl);
            }
        }
    }
    __syncwarp();
}

#ifndef TG_C5_QDEFER
#define TG_C5_QDEFER 1
#endif

// c5_drain for chain sites (8 classes: c = c0 + 2 c1 cost bits, q = chain
// bit).  The record carries the cost bits; the chain bit is recomputed from
// the stored rows (the partner has the other colour, and the own word's
// undecided lanes still hold their old spin under Metropolis).  A late flip
// changes the lane's unsatisfied cost bonds by 2c - 3 (heat bath, late +1:
// 3 - 2c) and its unsatisfied chain bond by +1 if it was satisfied, else -1.
template <int RULE>
__device__ __noinline__ void c5_drain_chain(const PlaneArgs& a, int base, int n, uint32_t tlo, uint32_t thi,
                                            int t31, bool count, int* s_cc, int* s_cq) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    const bool mine = lane < n;
    int4 e = make_int4(0, 0, 0, 0);
    if (mine) e = c5_queue(threadIdx.x >> 5)[base + lane];
    const uint32_t site = (uint32_t)e.x & 0x07ffffffu;
    const int w = (int)((uint32_t)e.x >> 27);
    uint32_t und = (uint32_t)e.y;
    uint32_t cb[3] = {(uint32_t)e.z, (uint32_t)e.w, 0u};
    uint32_t* own = a.spins + (size_t)site * a.W + w;
    if (mine) {
        const uint32_t y = a.spins[(size_t)((uint32_t)__ldg(&a.nbr4[site].w)) + w];
        cb[2] = RULE == 0 ? ~(*own ^ y) : y;
    }
    const uint32_t grp4 = (uint32_t)(a.w_global0 + w) << 4;
    const uint32_t* kpb = a.kp + (size_t)w * a.kpw + a.ty[t31].kp_off;
    uint32_t lt = 0u;
    const PhiloxT P = philox_t(tlo, thi, a.pks);
#pragma unroll 1
    for (int blk = 2; blk < 14; ++blk) {
        if (!__any_sync(0xffffffffu, und)) break;
        const u32x4 r = philox_plane(site, grp4 | (uint32_t)blk, P, a.pks);
        compare_block<3>(cb, kpb, 8, blk, r, und, lt);
    }
    if (lt) {
        if (RULE == 0) *own ^= lt;
        else *own |= lt;
        if (count) {
            uint32_t ex = lt;
            while (ex) {
                const int l = __ffs(ex) - 1;
                ex &= ex - 1;
                const int cl = (int)((cb[0] >> l) & 1u) + 2 * (int)((cb[1] >> l) & 1u);
                const int q = (int)((cb[2] >> l) & 1u);
                atomicAdd(s_cc + w * 32 + l, RULE == 0 ? 2 * cl - 3 : 3 - 2 * cl);
                atomicAdd(s_cq + w * 32 + l, RULE == 0 ? (q ? 1 : -1) : (q ? -1 : 1));
            }
        }
    }
    __syncwarp();
}

// Per-thread constants of a colour phase.
struct C5Ctx {
    uint32_t act[2];
    uint32_t g[4];                         // Philox word 3 of the 4 unconditional blocks
    uint32_t tlo, thi;
    PhiloxT P;
};

// One colour phase: chain-free items, then chain items.
template <int RULE>
__device__ __forceinline__ void c5_phase(const PlaneArgs& a, int c, uint64_t t, bool count, int gw,
                                         int nw, int logW, uint32_t (&V0)[kC5VB], uint32_t (&V1)[kC5VB],
                                         int t30, int t31, int nfree) {
    int* s_cc = c5_cnt();
    int* s_cq = s_cc + 32 * a.W;
    const int lane = threadIdx.x & 31;
    const int logWP = logW - 1;
    const int WP = 1 << logWP;
    const int S = 32 >> logWP;               // sites per item
    const int wp = lane & (WP - 1), sl = lane >> logWP;
    const int w0 = 2 * wp;
    const int cs = a.color_start[c], ce = a.color_start[c + 1];
    const int cf = cs + nfree;               // first chain site of the colour
    count = count && c == 1;
    C5Ctx K;
    // staged per round, part-major so the word pairs of a warp hit distinct
    // banks: Metropolis [k2a, k2b, k3a, k3b][word]; heat bath [9][word]
    const uint4* thr = c5_thr() + w0;
    const int W = 1 << logW;
    K.act[0] = a.active[w0];
    K.act[1] = a.active[w0 + 1];
    const uint32_t g0 = (uint32_t)(a.w_global0 + w0) << 4;
    K.g[0] = g0; K.g[1] = g0 | 1u; K.g[2] = g0 + 16u; K.g[3] = (g0 + 16u) | 1u;
    K.tlo = (uint32_t)t;
    K.thi = (uint32_t)(t >> 32);
    K.P = philox_t(K.tlo, K.thi, a.pks);
    const char* base = reinterpret_cast<const char*>(a.spins + w0);
#ifndef TG_ADDR32
#define TG_ADDR32 1
#endif
    // off: word offset of a row (index << logW) below 2^30 (host check), flag
    // bits 30-31 of an nbr4 entry fall off the 32-bit byte offset
    auto row = [&](uint32_t off) -> uint2 {
#if TG_ADDR32
        return *reinterpret_cast<const uint2*>(base + (uint32_t)(off << 2));
#else
        return *reinterpret_cast<const uint2*>(base + (size_t)(off & 0x7fffffffu) * 4u);
#endif
    };
    int qn = 0;
    int since = 0;  // items added to V0 / V1 since their last flush
    // ---------------------------------------------------------- chain-free
    {
        const int n_it = (nfree + S - 1) / S;
        auto entries = [&](int i) -> int4 {
            int4 v = make_int4(0, 0, 0, 0);
            if (i < n_it) {
                const int st = cs + i * S + sl;
                if (st < cf) v = __ldg(a.nbr4 + st);
            }
            return v;
        };
        struct Rows { uint2 s, x0, x1, x2; };
        auto rows = [&](int i, const int4& e) -> Rows {
            Rows q{make_uint2(0u, 0u), make_uint2(0u, 0u), make_uint2(0u, 0u), make_uint2(0u, 0u)};
            const int st = cs + i * S + sl;
            if (i < n_it && st < cf) {
                q.s = row((uint32_t)st << logW);
                q.x0 = row((uint32_t)e.x);
                q.x1 = row((uint32_t)e.y);
                q.x2 = row((uint32_t)e.z);
            }
            return q;
        };
        int it = gw;
        // software pipeline: the rows of the next item and the entries of the
        // one after it are in flight while the current item computes
        int4 en = entries(it);
        Rows rn = rows(it, en);
        int4 en2 = entries(it + nw);
        for (; it < n_it; it += nw) {
            const int4 e = en;
            const Rows q = rn;
            const uint32_t site = (uint32_t)(cs + it * S + sl);
            const bool valid = (int)site < cf;
            en = en2;
            rn = rows(it + nw, en);
            en2 = entries(it + 2 * nw);
            const uint2 s = q.s, x0 = q.x0, x1 = q.x1, x2 = q.x2;
            u32x4 r[4];
            philox_planeN<4, true>(site, K.g, K.P, a.pks, r);
            const uint32_t m0s = (uint32_t)(e.x >> 31), m1s = (uint32_t)(e.y >> 31), m2s = (uint32_t)(e.z >> 31);
            uint32_t und[2], ns[2], cl0[2], cl1[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t sj = j ? s.y : s.x;
                // Metropolis: satisfied bonds (J_ik s_i s_k = +1); heat bath:
                // +1 contributions (J_ik s_k = +1)
                const uint32_t b0 = (j ? x0.y : x0.x) ^ m0s, b1 = (j ? x1.y : x1.x) ^ m1s,
                               b2 = (j ? x2.y : x2.x) ^ m2s;
                const uint32_t a0 = RULE == 0 ? ~(sj ^ b0) : b0, a1 = RULE == 0 ? ~(sj ^ b1) : b1,
                               a2 = RULE == 0 ? ~(sj ^ b2) : b2;
                const uint32_t c0 = a0 ^ a1 ^ a2;
                const uint32_t c1 = (a0 & a1) | (a2 & (a0 ^ a1));
                const uint32_t act = valid ? K.act[j] : 0u;
                uint32_t u, lt = 0u, take;
                if (RULE == 0) {
                    u = c1 & act;  // classes 0, 1 (de < 0): always taken
#if TG_CMP8
                    compare8_sel(c0, thr[j], thr[W + j], thr[2 * W + j], thr[3 * W + j], r[2 * j], r[2 * j + 1],
                                 u, u, lt);
                    take = act & (~c1 | lt);
#else
                    compare4_sel(c0, thr[j], thr[2 * W + j], r[2 * j], u, lt);
                    compare4_sel(c0, thr[W + j], thr[3 * W + j], r[2 * j + 1], u, lt);
                    take = (~c1 & act) | lt;
#endif
                    ns[j] = sj ^ take;
                } else {
                    const uint4* tj = thr + j;
                    const uint4 L = tj[8 * W];
                    const uint32_t always = sel(c1, sel(c0, L.w, L.z), sel(c0, L.y, L.x)) & act;
                    u = act & ~always;
                    const uint32_t rr[8] = {r[2 * j].x, r[2 * j].y, r[2 * j].z, r[2 * j].w,
                                            r[2 * j + 1].x, r[2 * j + 1].y, r[2 * j + 1].z, r[2 * j + 1].w};
#if TG_CMP8
                    uint32_t tb[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const uint4 T = tj[b * W];
                        tb[b] = sel(c1, sel(c0, T.w, T.z), sel(c0, T.y, T.x));
                    }
                    compare8(tb, rr, u, u, lt);  // lt beyond u: covered by `always` / masked by act
#else
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const uint4 T = tj[b * W];
                        const uint32_t tb = sel(c1, sel(c0, T.w, T.z), sel(c0, T.y, T.x));
                        lt |= u & tb & ~rr[b];
                        u &= ~(tb ^ rr[b]);
                    }
#endif
                    take = (always | lt) & act;  // new spin +1 (undecided lanes provisionally -1)
                    ns[j] = (sj & ~act) | take;
                }
                und[j] = u;
                if (count) {  // unsatisfied bonds after the update (all neighbours lower)
                    uint32_t m0, m1;
                    if (RULE == 0) {
                        m0 = ~(c0 ^ take) & act;
                        m1 = ~(c1 ^ take) & act;
                    } else {
                        const uint32_t u0 = ns[j] ^ b0, u1 = ns[j] ^ b1, u2 = ns[j] ^ b2;
                        m0 = (u0 ^ u1 ^ u2) & act;
                        m1 = ((u0 & u1) | (u2 & (u0 ^ u1))) & act;
                    }
                    if (j == 0) c5_vadd<2>(V0, m0, m1);
                    else c5_vadd<2>(V1, m0, m1);
                }
                cl0[j] = c0;
                cl1[j] = c1;
            }
            if (valid)
                *reinterpret_cast<uint2*>(const_cast<char*>(base) + (uint32_t)(site << (logW + 2))) =
                    make_uint2(ns[0], ns[1]);
            // deferred tail: pairs with lanes still undecided after 8 planes
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t pend = __ballot_sync(0xffffffffu, und[j] != 0u);
                if (pend) {
                    if (und[j])  // {site | word << 27, undecided lanes, class bits}
                        c5_queue(threadIdx.x >> 5)[qn + __popc(pend & ((1u << lane) - 1u))] =
                            make_int4((int)(site | ((uint32_t)(w0 + j) << 27)), (int)und[j], (int)cl0[j],
                                      (int)cl1[j]);
                    qn += __popc(pend);
                }
            }
            if (qn >= 32) {
                qn -= 32;
                c5_drain<RULE>(a, qn, 32, K.tlo, K.thi, t30, count, s_cc);
            }
            if (count && ++since == kC5FlushAt) {  // 8-plane counters: at most 3 per item
                c5_flush(V0, logWP, 0, s_cc);
                c5_flush(V1, logWP, 1, s_cc);
                since = 0;
            }
        }
    }
    // ---------------------------------------------------------- chain sites
    const int nq = ce - cf;
    const int n_itq = (nq + S - 1) / S;
    auto centry = [&](int i) -> int4 {
        int4 v = make_int4(0, 0, 0, 0);
        if (i < n_itq) {
            const int st = cf + i * S + sl;
            if (st < ce) v = __ldg(a.nbr4 + st);
        }
        return v;
    };
    struct CRows { uint2 s, x0, x1, x2, y; };
    auto crows = [&](int i, const int4& e) -> CRows {
        const uint2 z = make_uint2(0u, 0u);
        CRows q{z, z, z, z, z};
        const int st = cf + i * S + sl;
        if (i < n_itq && st < ce) {
            q.s = row((uint32_t)st << logW);
            q.x0 = row((uint32_t)e.x);
            q.x1 = row((uint32_t)e.y);
            q.x2 = row((uint32_t)e.z);
            q.y = row((uint32_t)e.w);
        }
        return q;
    };
    while (qn > 0) {
        const int n = qn < 32 ? qn : 32;
        qn -= n;
        c5_drain<RULE>(a, qn, n, K.tlo, K.thi, t30, count, s_cc);
    }
    if (nq > 0) {
        const int n_it = n_itq;
        const uint32_t* kpb0 = a.kp + (size_t)w0 * a.kpw + a.ty[t31].kp_off;
        const uint32_t* kpb1 = kpb0 + a.kpw;
        uint32_t Q0[kC5VB], Q1[kC5VB];
#pragma unroll
        for (int b = 0; b < kC5VB; ++b) { Q0[b] = 0u; Q1[b] = 0u; }
        for (int it = gw; it < n_it; it += nw) {
            const uint32_t site = (uint32_t)(cf + it * S + sl);
            const bool valid = (int)site < ce;
            // (a software pipeline of these loads as in the chain-free loop was
            // measured 1.3 % slower: profiles/r2/ab_c5_flush_chainpipe.txt)
            const int4 e = centry(it);
            const CRows cq_ = crows(it, e);
            const uint2 s = cq_.s, x0 = cq_.x0, x1 = cq_.x1, x2 = cq_.x2, y = cq_.y;
            u32x4 r[4];
            philox_planeN<4, true>(site, K.g, K.P, a.pks, r);
            const uint32_t m0s = (uint32_t)(e.x >> 31), m1s = (uint32_t)(e.y >> 31), m2s = (uint32_t)(e.z >> 31);
            uint32_t ns[2];
            uint32_t undq[2] = {0u, 0u}, clq0[2] = {0u, 0u}, clq1[2] = {0u, 0u};
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t sj = j ? s.y : s.x;
                const uint32_t b0 = (j ? x0.y : x0.x) ^ m0s, b1 = (j ? x1.y : x1.x) ^ m1s,
                               b2 = (j ? x2.y : x2.x) ^ m2s;
                const uint32_t a0 = RULE == 0 ? ~(sj ^ b0) : b0, a1 = RULE == 0 ? ~(sj ^ b1) : b1,
                               a2 = RULE == 0 ? ~(sj ^ b2) : b2;
                const uint32_t yj = j ? y.y : y.x;
                const uint32_t cb[3] = {a0 ^ a1 ^ a2, (a0 & a1) | (a2 & (a0 ^ a1)), RULE == 0 ? ~(sj ^ yj) : yj};
                const uint32_t act = valid ? K.act[j] : 0u;
                const uint32_t* kpb = j ? kpb1 : kpb0;
                const uint32_t always = mux_tree<3>(cb, kpb + kKPlanes * 8) & act;
                uint32_t u = act & ~always, lt = 0u;
#if TG_CMP8
                {
                    const uint32_t rr[8] = {r[2 * j].x, r[2 * j].y, r[2 * j].z, r[2 * j].w,
                                            r[2 * j + 1].x, r[2 * j + 1].y, r[2 * j + 1].z, r[2 * j + 1].w};
                    uint32_t tb[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b) tb[b] = mux_tree<3>(cb, kpb + b * 8);
                    compare8(tb, rr, u, u, lt);  // lt beyond u: covered by `always` / masked by act
                }
#else
                compare_block<3>(cb, kpb, 8, 0, r[2 * j], u, lt);
                compare_block<3>(cb, kpb, 8, 1, r[2 * j + 1], u, lt);
#endif
#if TG_C5_QDEFER
                lt &= ~u;  // undecided lanes: provisionally not taken, resolved by c5_drain_chain
                undq[j] = u;
                clq0[j] = cb[0];
                clq1[j] = cb[1];
#else
#pragma unroll 1
                for (int blk = 2; blk < 14; ++blk) {
                    if (!__any_sync(0xffffffffu, u)) break;
                    const u32x4 rb = philox_plane(site, K.g[2 * j] | (uint32_t)blk, K.P, a.pks);
                    compare_block<3>(cb, kpb, 8, blk, rb, u, lt);
                }
#endif
                const uint32_t take = (always | lt) & act;
                ns[j] = RULE == 0 ? sj ^ take : (sj & ~act) | take;
                if (count) {
                    const uint32_t mq = (ns[j] ^ yj) & act;  // chain bond unsatisfied after the update
                    uint32_t m0, m1;
                    if (RULE == 0) {
                        m0 = ~(cb[0] ^ take) & act;
                        m1 = ~(cb[1] ^ take) & act;
                    } else {
                        const uint32_t u0 = ns[j] ^ b0, u1 = ns[j] ^ b1, u2 = ns[j] ^ b2;
                        m0 = (u0 ^ u1 ^ u2) & act;
                        m1 = ((u0 & u1) | (u2 & (u0 ^ u1))) & act;
                    }
                    if (j == 0) {
                        c5_vadd<2>(V0, m0, m1);
                        c5_vadd<1>(Q0, mq, 0u);
                    } else {
                        c5_vadd<2>(V1, m0, m1);
                        c5_vadd<1>(Q1, mq, 0u);
                    }
                }
            }
            if (valid)
                *reinterpret_cast<uint2*>(const_cast<char*>(base) + (uint32_t)(site << (logW + 2))) =
                    make_uint2(ns[0], ns[1]);
#if TG_C5_QDEFER
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t pend = __ballot_sync(0xffffffffu, undq[j] != 0u);
                if (pend) {
                    if (undq[j])  // {site | word << 27, undecided lanes, cost class bits}
                        c5_queue(threadIdx.x >> 5)[qn + __popc(pend & ((1u << lane) - 1u))] =
                            make_int4((int)(site | ((uint32_t)(w0 + j) << 27)), (int)undq[j], (int)clq0[j],
                                      (int)clq1[j]);
                    qn += __popc(pend);
                }
            }
            if (qn >= 32) {
                qn -= 32;
                c5_drain_chain<RULE>(a, qn, 32, K.tlo, K.thi, t31, count, s_cc, s_cq);
            }
#endif
            if (count && ++since == kC5FlushAt) {
                c5_flush(V0, logWP, 0, s_cc);
                c5_flush(V1, logWP, 1, s_cc);
                c5_flush(Q0, logWP, 0, s_cq);
                c5_flush(Q1, logWP, 1, s_cq);
                since = 0;
            }
        }
#if TG_C5_QDEFER
        while (qn > 0) {
            const int n = qn < 32 ? qn : 32;
            qn -= n;
            c5_drain_chain<RULE>(a, qn, n, K.tlo, K.thi, t31, count, s_cc, s_cq);
        }
#endif
        if (count) {
            c5_flush(Q0, logWP, 0, s_cq);
            c5_flush(Q1, logWP, 1, s_cq);
        }
    }
    if (count) {  // one flush of the cost-bond counters per phase (chain-free + chain items)
        c5_flush(V0, logWP, 0, s_cc);
        c5_flush(V1, logWP, 1, s_cc);
    }
}

// Persistent single-GPU kernel: n_rounds whole rounds of run_2dpt
// (engine.cpp:121-216); one grid barrier per colour phase, the round epilogue
// (plane_round.cuh) closes each round.
template <int RULE>
__global__ void __launch_bounds__(kC5Threads, kC5MinBlocks)
plane_c5_rounds_kernel(const __grid_constant__ PlaneArgs a, const __grid_constant__ RoundArgs r) {
    cg::grid_group grid = cg::this_grid();
    const int nrep = a.W * 32;
    int* s_cc = c5_cnt();
    int* s_cq = s_cc + nrep;
    const RoundSmem s = round_smem(s_cq + nrep, r.R);
    const int logW = r.log_w;
    const int gw = blockIdx.x * (kC5Threads >> 5) + (threadIdx.x >> 5);
    const int nw = r.n_warps;
    // site types: t30 = cost 3 / no chain, t31 = cost 3 / one chain partner
    int t30 = 0, t31 = 0;
    for (int ty = 0; ty < a.n_types; ++ty) {
        if (a.ty[ty].dq == 0) t30 = ty;
        else t31 = ty;
    }
    for (int m = threadIdx.x; m < 2 * nrep; m += blockDim.x) s_cc[m] = 0;
    round_load_labels(r, s);
    __syncthreads();
    uint32_t V0[kC5VB], V1[kC5VB];
#pragma unroll
    for (int b = 0; b < kC5VB; ++b) { V0[b] = 0u; V1[b] = 0u; }
    uint64_t swap_base = r.swap_base0;
    for (int k = 0; k < r.n_rounds; ++k) {
        const int64_t round = r.round0 + k;
        const int par = (int)(round & 1);
        int32_t* cc = r.cnt + (size_t)par * 2 * r.cnt_stride;
        int32_t* cq = cc + r.cnt_stride;
        {   // this round's thresholds of the chain-free type (the epilogue's grid barrier precedes)
            uint4* th = c5_thr();
            if (RULE == 0) {  // class-2/3 planes 0-7
                for (int q = threadIdx.x; q < 4 * a.W; q += blockDim.x) {
                    const int part = q / a.W, w = q % a.W;
                    th[q] = reinterpret_cast<const uint4*>(a.kpc + ((size_t)w * a.n_types + t30) * 128)
                        [(part & 1) + 16 * (part >> 1)];
                }
            } else {          // 4 classes: planes 0-7 and "always"
                const int kp0 = a.ty[t30].kp_off;
                for (int q = threadIdx.x; q < 9 * a.W; q += blockDim.x) {
                    const int b = q / a.W, w = q % a.W;
                    th[q] = *reinterpret_cast<const uint4*>(a.kp + (size_t)w * a.kpw + kp0 + (b < 8 ? b : kKPlanes) * 4);
                }
            }
            __syncthreads();
        }
        for (int sw = 0; sw < r.sps; ++sw) {
            const uint64_t t = (uint64_t)((round - 1) * r.sps + sw);
            const bool count = (sw == r.sps - 1);
            for (int c = 0; c < 2; ++c) {
                c5_phase<RULE>(a, c, t, count, gw, nw, logW, V0, V1, t30, t31, r.c5_nfree[c]);
                if (count && c == 1) {
                    __syncthreads();
                    for (int m = threadIdx.x; m < nrep; m += blockDim.x) {
                        const int vc = s_cc[m], vqv = s_cq[m];
                        if (vc) { atomicAdd(cc + m, vc); s_cc[m] = 0; }
                        if (vqv) { atomicAdd(cq + m, vqv); s_cq[m] = 0; }
                    }
                }
                grid.sync();
            }
        }
        round_epilogue(a, r, s, k, round, cc, cq, swap_base, 2 * r.sps);
    }
}

// Sweep-only kernel of the unfused round loop (multi-GPU ranks, full-grid
// records; same contract as plane_tpw_sweep_kernel): n_sweeps sweeps over the
// rank's words with the thresholds the swap kernel left in a.kp / a.kpc,
// then the rank's per-replica (f, g) into a.f_loc / a.g_loc (counters
// re-zeroed); the (f, g) exchange and the swap phase run after it.
template <int RULE>
__global__ void __launch_bounds__(kC5Threads, kC5MinBlocks)
plane_c5_sweep_kernel(const __grid_constant__ PlaneArgs a, int64_t t0, int n_sweeps, int nfree0, int nfree1) {
    if (a.rs) t0 = a.rs->round * n_sweeps;
    cg::grid_group grid = cg::this_grid();
    const int nrep = a.W * 32;
    int* s_cc = c5_cnt();
    int* s_cq = s_cc + nrep;
    const int logW = __ffs(a.W) - 1;
    const int gw = blockIdx.x * (kC5Threads >> 5) + (threadIdx.x >> 5);
    const int nw = gridDim.x * (kC5Threads >> 5);
    int t30 = 0, t31 = 0;
    for (int ty = 0; ty < a.n_types; ++ty) {
        if (a.ty[ty].dq == 0) t30 = ty;
        else t31 = ty;
    }
    for (int m = threadIdx.x; m < 2 * nrep; m += blockDim.x) s_cc[m] = 0;
    {   // thresholds of the chain-free type (the labels are fixed for the whole launch)
        uint4* th = c5_thr();
        if (RULE == 0) {
            for (int q = threadIdx.x; q < 4 * a.W; q += blockDim.x) {
                const int part = q / a.W, w = q % a.W;
                th[q] = reinterpret_cast<const uint4*>(a.kpc + ((size_t)w * a.n_types + t30) * 128)
                    [(part & 1) + 16 * (part >> 1)];
            }
        } else {
            const int kp0 = a.ty[t30].kp_off;
            for (int q = threadIdx.x; q < 9 * a.W; q += blockDim.x) {
                const int b = q / a.W, w = q % a.W;
                th[q] = *reinterpret_cast<const uint4*>(a.kp + (size_t)w * a.kpw + kp0 + (b < 8 ? b : kKPlanes) * 4);
            }
        }
    }
    __syncthreads();
    uint32_t V0[kC5VB], V1[kC5VB];
#pragma unroll
    for (int b = 0; b < kC5VB; ++b) { V0[b] = 0u; V1[b] = 0u; }
    for (int sw = 0; sw < n_sweeps; ++sw) {
        const uint64_t t = (uint64_t)(t0 + sw);
        const bool count = (sw == n_sweeps - 1);
        for (int c = 0; c < 2; ++c) {
            c5_phase<RULE>(a, c, t, count, gw, nw, logW, V0, V1, t30, t31, c ? nfree1 : nfree0);
            if (count && c == 1) {
                __syncthreads();
                for (int m = threadIdx.x; m < nrep; m += blockDim.x) {
                    const int vc = s_cc[m], vqv = s_cq[m];
                    if (vc) { atomicAdd(a.cnt_c + m, vc); s_cc[m] = 0; }
                    if (vqv) { atomicAdd(a.cnt_q + m, vqv); s_cq[m] = 0; }
                }
            }
            grid.sync();
        }
    }
    // f = -(m - 2 u_c) for J = +-1, h = 0; g = sum (s_a - s_b)^2 = 4 u_q
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < a.local_states; m += gridDim.x * blockDim.x) {
        const int uc = a.cnt_c[m], uq = a.cnt_q[m];
        a.f_loc[m] = -((double)a.m_cost - 2.0 * (double)uc);
        a.g_loc[m] = 4.0 * (double)uq;
        a.cnt_c[m] = 0;
        a.cnt_q[m] = 0;
    }
}

template __global__ void plane_c5_sweep_kernel<0>(const __grid_constant__ PlaneArgs, int64_t, int, int, int);
template __global__ void plane_c5_sweep_kernel<1>(const __grid_constant__ PlaneArgs, int64_t, int, int, int);

void* plane_c5_sweep_fn(int rule) {
    return rule ? (void*)plane_c5_sweep_kernel<1> : (void*)plane_c5_sweep_kernel<0>;
}

template __global__ void plane_c5_rounds_kernel<0>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);
template __global__ void plane_c5_rounds_kernel<1>(const __grid_constant__ PlaneArgs, const __grid_constant__ RoundArgs);

void* plane_c5_fn(int rule) {
    return rule ? (void*)plane_c5_rounds_kernel<1> : (void*)plane_c5_rounds_kernel<0>;
}

}  // namespace tg
