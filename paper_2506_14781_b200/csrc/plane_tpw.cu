// plane_tpw.cu -- PLANE engine fused round kernel, one thread per
// (site, 32-replica word).  Compiled once per update rule (-DTG_PLANE_RULE).
//
// Same contract as plane_rounds_kernel (plane_sweep.cu) and therefore the
// same trajectories bit for bit: the reference sweep (mc.cpp:21-35) over the
// canonical colour order, thresholds K = ceil(T * 2^53) compared MSB-first
// against bit planes of Philox4x32-10 draws with counter
// {site, t_lo, t_hi, group << 4 | block}, labels permuted by the swap phase.
//
// Layout of the work: a warp item is S = 32 / W consecutive sites of one
// chunk (same colour, same site type) x all W words of their rows; lane =
// site_in_item * W + word, so a warp's loads of a row are W consecutive
// words (coalesced) and every thread keeps ONE word for the whole launch:
// its lane mask, Philox group and threshold-plane block are per-thread
// constants.  Few live registers per thread -> 2 CTAs x 512 threads per SM.
//
// Energy bookkeeping: on the last sweep of a round every site adds its
// unsatisfied bonds to lower-colour neighbours (each bond counted once, at
// its higher-colour end) into per-thread VERTICAL bit-sliced counters (8 bit
// planes, bit l = replica l of the thread's word); they are reduced to
// per-replica integers once per colour phase (butterfly across the lanes of
// one word, packed 32x32 bit transposes) into shared-memory counters, then
// one global atomic per replica and block.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"
#include "plane_device.cuh"
#include "philox_plane.cuh"

#ifndef TG_PLANE_RULE
#define TG_PLANE_RULE 0
#endif
#define TG_CAT2(a, b) a##b
#define TG_CAT(a, b) TG_CAT2(a, b)

namespace cg = cooperative_groups;

namespace tg {

// Stage timer (variant builds only, -DTG_TPW_PROF=1): block 0 records
// %globaltimer at the stages of the first 64 rounds of a launch; every block
// records the latest "all items of this phase done" time (atomicMax).
#ifndef TG_TPW_PROF
#define TG_TPW_PROF 0
#endif
#if TG_TPW_PROF
__device__ unsigned long long g_tpw_prof[64][16];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TPW_STAMP(k, s) do { if ((k) < 64 && blockIdx.x == 0 && threadIdx.x == 0) g_tpw_prof[k][s] = gtimer(); } while (0)
#define TPW_MAXSTAMP(k, s) do { __syncthreads(); if ((k) < 64 && threadIdx.x == 0) atomicMax(&g_tpw_prof[k][s], gtimer()); } while (0)
#define TPW_EPI_STAMP(k, s) TPW_STAMP(k, s)
#else
#define TPW_STAMP(k, s) do {} while (0)
#define TPW_MAXSTAMP(k, s) do {} while (0)
#endif
}  // namespace tg
#include "plane_round.cuh"
namespace tg {

#ifndef TG_TPW_DYN_K
#define TG_TPW_DYN_K 1
#endif
constexpr int kTpwDynK = TG_TPW_DYN_K;  // items per warp left to the dynamic tail
constexpr int kVB = kTpwVB;  // planes of the per-thread vertical bond counters (max 255)

// V += m (NB-bit bit-sliced value) in kVB-bit vertical arithmetic.
template <int NB>
__device__ __forceinline__ void vadd(uint32_t (&V)[kVB], const uint32_t* m) {
    uint32_t carry = 0u;
#pragma unroll
    for (int b = 0; b < kVB; ++b) {
        const uint32_t x = V[b];
        if (b < NB) {
            const uint32_t y = m[b];
            V[b] = x ^ y ^ carry;
            carry = (x & y) | (carry & (x ^ y));
        } else {
            V[b] = x ^ carry;
            carry = x & carry;
        }
    }
}

static_assert(kTpwVB == 8, "vflush_v passes 8 counter planes");
// Per-replica totals of the warp's vertical counters, added into
// s_cnt[w * 32 + l]; V is cleared.  Lanes sharing a word (lane = p * W + w)
// are summed by a butterfly; the sum's planes are then packed S per 32x32
// transpose (row p * W + w carries plane q * S + p of word w), after which
// lane l reads replica l's bits of every word.
template <int LOGW>
__device__ __forceinline__ void vflush_w(uint32_t (&V)[kVB], int* s_cnt) {
    constexpr int W = 1 << LOGW, LOGS = 5 - LOGW, S = 1 << LOGS;
    constexpr int NB = kVB + LOGS;          // planes of the per-word sum
    constexpr int NQ = (NB + S - 1) / S;    // packed transposes
    const int lane = threadIdx.x & 31;
    uint32_t E[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) E[b] = b < kVB ? V[b] : 0u;
#pragma unroll
    for (int b = 0; b < kVB; ++b) V[b] = 0u;
#pragma unroll
    for (int lv = 0; lv < LOGS; ++lv) {
        uint32_t carry = 0u;
#pragma unroll
        for (int b = 0; b <= kVB + lv && b < NB; ++b) {
            const uint32_t x = E[b];
            const uint32_t o = __shfl_xor_sync(0xffffffffu, x, W << lv);
            E[b] = x ^ o ^ carry;
            carry = (x & o) | (carry & (x ^ o));
        }
    }
    const int p_me = lane >> LOGW;
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
    for (int w = 0; w < W; ++w) {
        int val = 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if constexpr (S == 4) {
                const uint32_t x = (T[q] >> w) & 0x01010101u;
                val += (int)((x * 0x01020408u) >> 24) << (4 * q);
            } else {
#pragma unroll
                for (int p = 0; p < S; ++p)
                    val += (int)((T[q] >> (p * W + w)) & 1u) << (q * S + p);
            }
        }
        if (val) atomicAdd(s_cnt + w * 32 + lane, val);
    }
}

// Counters passed by value (registers through the call, no local-memory
// copy of the caller's array); the caller clears its counters.
static __device__ __noinline__ void vflush_v(uint4 lo, uint4 hi, int logW, int* s_cnt) {
    uint32_t V[kVB] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    switch (logW) {
        case 0: vflush_w<0>(V, s_cnt); break;
        case 1: vflush_w<1>(V, s_cnt); break;
        case 2: vflush_w<2>(V, s_cnt); break;
        case 3: vflush_w<3>(V, s_cnt); break;
        case 4: vflush_w<4>(V, s_cnt); break;
        default: vflush_w<5>(V, s_cnt); break;
    }
}

__device__ __forceinline__ void vflush(uint32_t (&V)[kVB], int logW, int* s_cnt) {
    vflush_v(make_uint4(V[0], V[1], V[2], V[3]), make_uint4(V[4], V[5], V[6], V[7]), logW, s_cnt);
#pragma unroll
    for (int b = 0; b < kVB; ++b) V[b] = 0u;
}

// Deferred tail of the lazy comparison (Metropolis, cost degree 3, no chain:
// the dominant site type).  After the two unconditional Philox blocks (8
// planes) a (site, word) pair still has undecided lanes with probability
// ~6 %; instead of dragging the whole warp through further blocks for it, the
// pair is queued in the warp's shared-memory queue with the provisional word
// (undecided lanes not taken) already stored, and resolved later 32 pairs at
// a time, one per lane: same planes, same thresholds, so the same decisions.
// Lanes taken late are XORed into the stored word (same warp, after
// __syncwarp) and their bond counts corrected: a flip turns the m_l
// unsatisfied lower bonds counted for lane l into nlow - m_l.
// Dynamic shared memory of the kernel, fixed layout (compile-time offsets;
// kTpwThreads threads): tail queues [warps][6][kTpwQCap] (site, meta =
// w | type << 5 | count << 10 | nlow << 11, und, class bit 0, the counted
// 2-bit unsatisfied lower bonds m0/m1), chain vertical counters
// [kVB][threads], per-replica counters [2][32W], then the round block.
extern __shared__ __align__(16) int tpw_sm[];
enum { kQSite, kQMeta, kQUnd, kQC0, kQM0, kQM1, kQC1, kQFields };
__device__ __forceinline__ int* tq(int warp, int field) {
    return tpw_sm + (warp * kQFields + field) * kTpwQCap;
}
static_assert(kQFields == kTpwQFields, "queue layout");
constexpr int kTpwSmVq = (kTpwThreads / 32) * kQFields * kTpwQCap;
// heat bath, config-5 path: planes 0-7 and the "always" word of the 4
// classes of the chain-free type, [9][W] uint4, staged once per colour phase
constexpr int kTpwSmHb = kTpwSmVq + kVB * kTpwThreads;
constexpr int kTpwSmCnt = kTpwSmHb + kTpwHbWords;

// Resolve entries [base, base + n) of the warp's queue (n <= 32).
template <int RULE>
static __device__ __noinline__ void tpw_drain(const PlaneArgs& a, int base, int n, uint32_t tlo,
                                              uint32_t thi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int* s_cc = tpw_sm + kTpwSmCnt;
    __syncwarp();
    const bool mine = lane < n;
    const int e = base + lane;
    int site = 0, meta = 0;
    uint32_t und = 0u, c0 = 0u, c1 = 0u;
    if (mine) {
        site = tq(warp, kQSite)[e];
        meta = tq(warp, kQMeta)[e];
        und = (uint32_t)tq(warp, kQUnd)[e];
        c0 = (uint32_t)tq(warp, kQC0)[e];
        if (RULE == 1) c1 = (uint32_t)tq(warp, kQC1)[e];
    }
    const int w = meta & 31, type = (meta >> 5) & 31;
    const uint32_t grp4 = (uint32_t)(a.w_global0 + w) << 4;
    const uint4* kc2 = reinterpret_cast<const uint4*>(a.kpc + ((size_t)w * a.n_types + type) * 128);
    uint32_t lt = 0u;
    const PhiloxT P = philox_t(tlo, thi, a.pks);
#pragma unroll 1
    for (int blk = 2; blk < 14; ++blk) {
        if (!__any_sync(0xffffffffu, und)) break;
        const u32x4 r = philox_plane((uint32_t)site, grp4 | (uint32_t)blk, P, a.pks);
        if (RULE == 0) {
            compare4_sel(c0, __ldg(kc2 + blk), __ldg(kc2 + 16 + blk), r, und, lt);
        } else {  // 4 classes, plane-major leaves of kp
            const uint32_t cb[2] = {c0, c1};
            compare_block<2>(cb, a.kp + (size_t)w * a.kpw + a.ty[type].kp_off, 4, blk, r, und, lt);
        }
    }
    if (lt) {
        // Metropolis: late flips; heat bath: late "up" (the provisional word has them down)
        if (RULE == 0) a.spins[(size_t)site * a.W + w] ^= lt;
        else a.spins[(size_t)site * a.W + w] |= lt;
        if ((meta >> 10) & 1) {
            const uint32_t m0 = (uint32_t)tq(warp, kQM0)[e], m1 = (uint32_t)tq(warp, kQM1)[e];
            const int nlow = (meta >> 11) & 7;
            uint32_t ex = lt;
            while (ex) {
                const int l = __ffs(ex) - 1;
                ex &= ex - 1;
                const int ml = (int)((m0 >> l) & 1u) + 2 * (int)((m1 >> l) & 1u);
                const int d = nlow - 2 * ml;
                if (d) atomicAdd(s_cc + w * 32 + l, d);
            }
        }
    }
    __syncwarp();
}

// One (site, word) update.  cb = bit-sliced class counters (satisfied bonds
// for Metropolis, +1 contributions for heat bath), as in plane_site.
template <int NCB, int NQB, int RULE>
__device__ __forceinline__ void tpw_site(const PlaneArgs& a, const Chunk& ch, const PlaneType& ty,
                                         int pos, int w, uint32_t act_w, uint32_t grp4, uint32_t tlo,
                                         uint32_t thi, bool count, int lower, uint32_t (&Vc)[kVB],
                                         int& qn) {
    constexpr int DCM = (1 << NCB) - 1;
    constexpr int DQM = (1 << NQB) - 1;
    constexpr int B = NCB + NQB;
    const int dc = ty.dc, dq = ty.dq, deg = dc + dq;
    const bool valid = pos < ch.len;
    const int site = ch.start + pos;
    const int W = a.W;
    uint32_t s = 0u, x[DCM > 0 ? DCM : 1], y[DQM > 0 ? DQM : 1];
    uint32_t lowx = 0u, lowy = 0u;
#pragma unroll
    for (int k = 0; k < (DCM > 0 ? DCM : 1); ++k) x[k] = 0u;
#pragma unroll
    for (int k = 0; k < (DQM > 0 ? DQM : 1); ++k) y[k] = 0u;
    if (valid) {
        s = a.spins[(size_t)site * W + w];
        const int32_t* nb = a.nbr + ch.nbr_base + pos * deg;
#pragma unroll
        for (int k = 0; k < DCM; ++k) {
            if (k < dc) {
                const int32_t e = __ldg(nb + k);
                const int j = e & 0x7fffffff;
                x[k] = a.spins[(size_t)j * W + w] ^ (uint32_t)(e >> 31);  // bit: J_ij s_j = +1
                lowx |= (uint32_t)(j < lower) << k;
            }
        }
#pragma unroll
        for (int k = 0; k < DQM; ++k) {
            if (k < dq) {
                const int j = __ldg(nb + dc + k);
                y[k] = a.spins[(size_t)j * W + w];
                lowy |= (uint32_t)(j < lower) << k;
            }
        }
    }
    uint32_t cb[B > 0 ? B : 1];
#pragma unroll
    for (int b = 0; b < (B > 0 ? B : 1); ++b) cb[b] = 0u;
#pragma unroll
    for (int k = 0; k < DCM; ++k)
        if (k < dc) bs_add<NCB>(cb, RULE == 0 ? ~(s ^ x[k]) : x[k]);
#pragma unroll
    for (int k = 0; k < DQM; ++k)
        if (k < dq) bs_add<NQB>(cb + NCB, RULE == 0 ? ~(s ^ y[k]) : y[k]);
    const uint32_t act = valid ? act_w : 0u;
    const uint32_t* kpb = a.kp + (size_t)w * a.kpw + ty.kp_off;
    const int ncl = ty.ncl;
    // Metropolis, cost degree 3, no chain: classes 0, 1 (de < 0) are always
    // taken; flag bit 0 says classes 2, 3 are never "always" for any label,
    // so the undecided lanes are exactly class 2 | 3 and one select picks
    // their threshold plane.
    const bool fastp = RULE == 0 && NQB == 0 && NCB == 2 && (ty.pad & 1);
    uint32_t always;
    if (fastp) always = ~cb[1] & act;
    else always = mux_tree<B>(cb, kpb + kKPlanes * ncl) & act;
    uint32_t und = act & ~always, lt = 0u;
    const uint4* kc2 = reinterpret_cast<const uint4*>(a.kpc + ((size_t)w * a.n_types + ch.type) * 128);
    {
        const u32x4 r0 = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | 0u}, a.pks);
        const u32x4 r1 = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | 1u}, a.pks);
        if (fastp) {
            compare4_sel(cb[0], __ldg(kc2 + 0), __ldg(kc2 + 16), r0, und, lt);
            compare4_sel(cb[0], __ldg(kc2 + 1), __ldg(kc2 + 17), r1, und, lt);
        } else {
            compare_block<B>(cb, kpb, ncl, 0, r0, und, lt);
            compare_block<B>(cb, kpb, ncl, 1, r1, und, lt);
        }
    }
    uint32_t pend = 0u;
    if (fastp) {
        pend = __ballot_sync(0xffffffffu, und != 0u);  // -> deferred tail
    } else {
#pragma unroll 1
        for (int blk = 2; blk < 14; ++blk) {
            if (!__any_sync(0xffffffffu, und)) break;
            const u32x4 r = philox4x32_10_ks(u32x4{(uint32_t)site, tlo, thi, grp4 | (uint32_t)blk}, a.pks);
            compare_block<B>(cb, kpb, ncl, blk, r, und, lt);
        }
    }
    const uint32_t take = (always | lt) & act;
    const uint32_t ns = RULE == 0 ? (s ^ take) : ((s & ~act) | take);
    if (valid) a.spins[(size_t)site * W + w] = ns;
    uint32_t m[NCB > 0 ? NCB : 1];
    m[0] = 0u;
    if (count) {
        if constexpr (NCB > 0) {
            // all cost neighbours lower (bipartite colour 1): unsatisfied after
            // the update = c if taken (Metropolis flip), dc - c = ~c otherwise
            const bool all_low = RULE == 0 && dc == DCM &&
                                 __all_sync(0xffffffffu, !valid || lowx == (uint32_t)DCM);
            if (all_low) {
#pragma unroll
                for (int b = 0; b < NCB; ++b) m[b] = ~(cb[b] ^ take) & act;
            } else {
#pragma unroll
                for (int b = 0; b < NCB; ++b) m[b] = 0u;
#pragma unroll
                for (int k = 0; k < DCM; ++k)
                    if (k < dc) bs_add<NCB>(m, (ns ^ x[k]) & act & (0u - ((lowx >> k) & 1u)));
            }
            vadd<NCB>(Vc, m);
        }
        if constexpr (NQB > 0) {
            uint32_t mq[NQB];
#pragma unroll
            for (int b = 0; b < NQB; ++b) mq[b] = 0u;
#pragma unroll
            for (int k = 0; k < DQM; ++k)
                if (k < dq) bs_add<NQB>(mq, (ns ^ y[k]) & act & (0u - ((lowy >> k) & 1u)));
            // chain counters live in shared memory (chain sites are few)
            uint32_t* vq = reinterpret_cast<uint32_t*>(tpw_sm + kTpwSmVq) + threadIdx.x;
            uint32_t V[kVB];
#pragma unroll
            for (int b = 0; b < kVB; ++b) V[b] = vq[b * kTpwThreads];
            vadd<NQB>(V, mq);
#pragma unroll
            for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = V[b];
        }
    }
    if constexpr (RULE == 0 && NQB == 0 && NCB == 2) {
        if (pend) {
            if (und) {
                const int e = qn + __popc(pend & ((1u << (threadIdx.x & 31)) - 1u));
                const int warp = threadIdx.x >> 5;
                tq(warp, kQSite)[e] = site;
                tq(warp, kQMeta)[e] = w | (ch.type << 5) | ((int)count << 10) | (__popc(lowx) << 11);
                tq(warp, kQUnd)[e] = (int)und;
                tq(warp, kQC0)[e] = (int)cb[0];
                tq(warp, kQM0)[e] = (int)m[0];
                tq(warp, kQM1)[e] = (int)m[1];
            }
            qn += __popc(pend);
        }
    }
}

// Config-5 site types, Metropolis (the FAST kernel): cost degree exactly 3,
// chain degree DQ in {0, 1}, 32-bit indexing, per-thread constants in K.
// DQ = 0 types carry flag bit 0 (classes 2, 3 never "always"), so
// always = (c < 2) and the undecided lanes compare against the class-2/3
// planes with one select; their tail is deferred to the warp queue.  ALLLOW:
// every neighbour has a lower colour (colour 1 of a 2-colouring), so the
// unsatisfied bonds after the update are c if taken, 3 - c = ~c otherwise.
struct C5K {
    uint4 k2a, k2b, k3a, k3b;  // planes 0-7 of classes 2 and 3 (word w, the cost-3 chain-free type)
    uint32_t kc2;          // word offset of word w's class-2/3 planes in kpc (w * n_types * 128)
    uint32_t kpw;          // word offset of word w's block in kp (w * kpw)
    uint32_t act_w, grp4, tlo, thi;
    PhiloxT P;
    int w, logW, lower;
    int t30, t31;          // type ids of the chain-free and the chain sites
};

// An item's row words (own, cost neighbours, chain partner), gathered at the
// top of the item loop before the next item's prefetches are issued.
struct C5Rows {
    uint32_t s, x0, x1, x2, y0;
};

template <int RULE, int DQ, bool ALLLOW>
__device__ __forceinline__ void c5_site(const PlaneArgs& a, const C5K& K, int tyi,
                                        const PlaneType& ty, uint32_t site, bool valid, bool count,
                                        uint32_t (&Vc)[kVB], int& qn, int32_t e0, int32_t e1,
                                        int32_t e2, int32_t e3, const C5Rows& R) {
    const uint32_t j0 = (uint32_t)e0 & 0x7fffffffu, j1 = (uint32_t)e1 & 0x7fffffffu,
                   j2 = (uint32_t)e2 & 0x7fffffffu, jq = (uint32_t)e3;
    uint32_t s = R.s, x0 = R.x0, x1 = R.x1, x2 = R.x2, y0 = R.y0;
    u32x4 r0, r1;
    philox_plane2(site, K.grp4, K.P, a.pks, r0, r1);
    x0 ^= (uint32_t)(e0 >> 31);  // bit: J_ij s_j = +1
    x1 ^= (uint32_t)(e1 >> 31);
    x2 ^= (uint32_t)(e2 >> 31);
    uint32_t lowx = 7u, lowy = 1u;
    if (!ALLLOW) {  // j are row offsets (index << log2 W)
        const int lw = K.lower << K.logW;
        lowx = (uint32_t)((int)j0 < lw) | ((uint32_t)((int)j1 < lw) << 1) | ((uint32_t)((int)j2 < lw) << 2);
        lowy = (uint32_t)((int)jq < lw);
    }
    // class counters: satisfied bonds (Metropolis) / +1 contributions (heat bath)
    const uint32_t a0 = RULE == 0 ? ~(s ^ x0) : x0, a1 = RULE == 0 ? ~(s ^ x1) : x1,
                   a2 = RULE == 0 ? ~(s ^ x2) : x2;
    const uint32_t c0 = a0 ^ a1 ^ a2;
    const uint32_t c1 = (a0 & a1) | (a2 & (a0 ^ a1));
    const uint32_t act = valid ? K.act_w : 0u;
    uint32_t always, und, lt = 0u;
    const uint32_t* kpb = a.kp + K.kpw + ty.kp_off;
    uint32_t cb[3] = {c0, c1, DQ ? (RULE == 0 ? ~(s ^ y0) : y0) : 0u};
    // heat bath, chain-free sites: planes 0-7 and "always" of the 4 classes
    // from the per-phase shared-memory stage [9][W] (uint4 = classes 0..3)
    const uint4* hb = reinterpret_cast<const uint4*>(tpw_sm + kTpwSmHb) + K.w;
    if (DQ == 0) {
        if (RULE == 0) {
            always = ~c1 & act;
            und = c1 & act;
        } else {
            const uint4 L = hb[8 << K.logW];
            always = sel(c1, sel(c0, L.w, L.z), sel(c0, L.y, L.x)) & act;
            und = act & ~always;
        }
    } else {
        always = mux_tree<3>(cb, kpb + kKPlanes * 8) & act;
        und = act & ~always;
    }
    {
        if (DQ == 0) {
            if (RULE == 0) {
                compare4_sel(c0, K.k2a, K.k3a, r0, und, lt);
                compare4_sel(c0, K.k2b, K.k3b, r1, und, lt);
            } else {
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const uint4 L = hb[b << K.logW];
                    const uint32_t tb = sel(c1, sel(c0, L.w, L.z), sel(c0, L.y, L.x));
                    const uint32_t rb = b == 0 ? r0.x : b == 1 ? r0.y : b == 2 ? r0.z : b == 3 ? r0.w
                                      : b == 4 ? r1.x : b == 5 ? r1.y : b == 6 ? r1.z : r1.w;
                    lt |= und & tb & ~rb;
                    und &= ~(tb ^ rb);
                }
            }
        } else {
            compare_block<3>(cb, kpb, 8, 0, r0, und, lt);
            compare_block<3>(cb, kpb, 8, 1, r1, und, lt);
        }
    }
    uint32_t pend = 0u;
    if (DQ == 0) {
        pend = __ballot_sync(0xffffffffu, und != 0u);  // -> deferred tail
    } else {
#pragma unroll 1
        for (int blk = 2; blk < 14; ++blk) {
            if (!__any_sync(0xffffffffu, und)) break;
            const u32x4 r = philox_plane(site, K.grp4 | (uint32_t)blk, K.P, a.pks);
            compare_block<3>(cb, kpb, 8, blk, r, und, lt);
        }
    }
    const uint32_t take = (always | lt) & act;
    // Metropolis: taken lanes flip; heat bath: taken lanes +1, the others -1
    // (undecided lanes provisionally -1, raised by the drain when taken)
    const uint32_t ns = RULE == 0 ? (s ^ take) : ((s & ~act) | take);
    if (valid) a.spins[K.w + (site << K.logW)] = ns;
    uint32_t m[2] = {0u, 0u};
    if (count) {
        if (RULE == 0 && ALLLOW) {
            m[0] = ~(c0 ^ take) & act;
            m[1] = ~(c1 ^ take) & act;
        } else {
            bs_add<2>(m, (ns ^ x0) & act & (0u - (lowx & 1u)));
            bs_add<2>(m, (ns ^ x1) & act & (0u - ((lowx >> 1) & 1u)));
            bs_add<2>(m, (ns ^ x2) & act & (0u - ((lowx >> 2) & 1u)));
        }
        vadd<2>(Vc, m);
        if (DQ) {
            uint32_t mq[1] = {(ns ^ y0) & act & (0u - lowy)};
            uint32_t* vq = reinterpret_cast<uint32_t*>(tpw_sm + kTpwSmVq) + threadIdx.x;
            uint32_t V[kVB];
#pragma unroll
            for (int b = 0; b < kVB; ++b) V[b] = vq[b * kTpwThreads];
            vadd<1>(V, mq);
#pragma unroll
            for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = V[b];
        }
    }
    if (DQ == 0 && pend) {
        if (und) {
            const int e = qn + __popc(pend & ((1u << (threadIdx.x & 31)) - 1u));
            const int warp = threadIdx.x >> 5;
            tq(warp, kQSite)[e] = (int)site;
            tq(warp, kQMeta)[e] = K.w | (tyi << 5) | ((int)count << 10) |
                                  ((ALLLOW ? 3 : __popc(lowx)) << 11);
            tq(warp, kQUnd)[e] = (int)und;
            tq(warp, kQC0)[e] = (int)c0;
            tq(warp, kQM0)[e] = (int)m[0];
            tq(warp, kQM1)[e] = (int)m[1];
            if (RULE == 1) tq(warp, kQC1)[e] = (int)c1;
        }
        qn += __popc(pend);
    }
}

// Heat bath, config-5 path: stage planes 0-7 and "always" of the chain-free
// type's 4 classes for every word, [9][W] uint4, once per round (thresholds
// change only in the round epilogue; the caller's grid barrier precedes this).
__device__ __forceinline__ void tpw_stage_hb(const PlaneArgs& a) {
    int t30 = 0;
    for (int ty = 0; ty < a.n_types; ++ty)
        if (a.ty[ty].dq == 0) t30 = ty;
    uint4* hb = reinterpret_cast<uint4*>(tpw_sm + kTpwSmHb);
    const int kp0 = a.ty[t30].kp_off, W = a.W;
    for (int q = threadIdx.x; q < 9 * W; q += blockDim.x) {
        const int b = q / W, ww = q % W;
        hb[q] = *reinterpret_cast<const uint4*>(a.kp + (size_t)ww * a.kpw + kp0 + (b < 8 ? b : kKPlanes) * 4);
    }
    __syncthreads();
}

// FAST colour phase (config-5 types): chunk descriptors two items ahead,
// neighbour entries one item ahead, so an item's gathers depend only on
// registers when it starts.
template <int RULE>
__device__ __forceinline__ void tpw_phase_c5(const PlaneArgs& a, int c, uint64_t t, bool count,
                                             int gw, int nw, int logW, uint32_t (&Vc)[kVB],
                                             int flush_every, int* work = nullptr) {
    int* s_cc = tpw_sm + kTpwSmCnt;
    int* s_cq = s_cc + 32 * a.W;
    uint32_t* vq = reinterpret_cast<uint32_t*>(tpw_sm + kTpwSmVq) + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int W = 1 << logW, S = 32 >> logW;
    const int w = lane & (W - 1), sl = lane >> logW;
    const int lower = a.color_start[c];
    count = count && lower > 0;  // colour 0 has no lower-colour neighbours
    const bool alllow = a.n_colors == 2 && c == 1;  // proper 2-colouring: every neighbour is colour 0
    C5K K;
    K.kc2 = (uint32_t)(w * a.n_types * 128);
    K.kpw = (uint32_t)(w * a.kpw);
    K.t30 = K.t31 = 0;  // FAST kernels: at most one type of each
    for (int ty = 0; ty < a.n_types; ++ty) {
        if (a.ty[ty].dq == 0) K.t30 = ty;
        else K.t31 = ty;
    }
    if (RULE == 0) {
        const uint4* kc = reinterpret_cast<const uint4*>(a.kpc + K.kc2) + K.t30 * 32;
        K.k2a = kc[0];
        K.k2b = kc[1];
        K.k3a = kc[16];
        K.k3b = kc[17];
    }  // heat bath: planes 0-7 of the chain-free type's classes were staged at round start
    K.act_w = a.active[w];
    K.grp4 = (uint32_t)(a.w_global0 + w) << 4;
    K.tlo = (uint32_t)t;
    K.thi = (uint32_t)(t >> 32);
    K.P = philox_t(K.tlo, K.thi, a.pks);
    K.w = w;
    K.logW = logW;
    K.lower = lower;
    int since = 0, qn = 0;
    // items: S consecutive sites of the colour x the W words of their rows,
    // strided over the warps (chain sites, costlier, sit together in the
    // canonical order).  The padded neighbour table is indexed by site and
    // flags chain-free sites (bit 31 of the 4th entry), so no chunk table is
    // read; an item straddling the chain-free / chain boundary runs both
    // paths with complementary lane masks.  Entries are loaded one item ahead.
    const int cs = a.color_start[c], ce = a.color_start[c + 1];
    const int n_it = (ce - cs + S - 1) / S;
    const PlaneType& ty0 = a.ty[K.t30];
    const PlaneType& ty1 = a.ty[K.t31];
    auto entries = [&](int it, int4& e) {
        const int site = cs + it * S + sl;
        e = make_int4(0, 0, 0, (int)0x80000000u);
        if (it < n_it && site < ce) e = __ldg(a.nbr4 + site);  // one 16-byte load
    };
    // Static strided items for all but about one item per warp; the tail is
    // handed out by a per-phase counter (work != nullptr), so warps that
    // finish early take the remaining items instead of idling at the barrier.
    const int n_static = work ? (n_it / nw - kTpwDynK > 0 ? (n_it / nw - kTpwDynK) * nw : 0) : n_it;
    const int lane_ = threadIdx.x & 31;
    auto next_of = [&](int it) {
        const int nx = it + nw;
        if (nx < n_static || !work) return nx;
        int v = 0;
        if (lane_ == 0) v = n_static + atomicAdd(work, 1);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    int item = gw < n_static ? gw : next_of(gw - nw);
    int4 en;
    entries(item, en);
    for (int nxt; item < n_it; item = nxt) {
        nxt = next_of(item);
        const int4 e = en;
        const uint32_t site = (uint32_t)(cs + item * S + sl);
        const bool valid = (int)site < ce;
        const bool hasq = valid && !((uint32_t)e.w & 0x80000000u);
        C5Rows R{0u, 0u, 0u, 0u, 0u};
        if (valid) {  // gathers first: in flight during the prefetch and the Philox blocks
            const uint32_t* sp = a.spins + w;
            R.s = sp[site << logW];
            R.x0 = sp[(uint32_t)e.x & 0x7fffffffu];  // nbr4 entries are row offsets
            R.x1 = sp[(uint32_t)e.y & 0x7fffffffu];
            R.x2 = sp[(uint32_t)e.z & 0x7fffffffu];
            if (hasq) R.y0 = sp[(uint32_t)e.w];
        }
        entries(nxt, en);
        // one call site per path; both run (complementary lanes) only when
        // the item straddles the chain-free / chain boundary
        const bool v0 = valid && !hasq;
        if (__any_sync(0xffffffffu, v0)) {
            if (alllow) c5_site<RULE, 0, true>(a, K, K.t30, ty0, site, v0, count, Vc, qn, e.x, e.y, e.z, e.w, R);
            else c5_site<RULE, 0, false>(a, K, K.t30, ty0, site, v0, count, Vc, qn, e.x, e.y, e.z, e.w, R);
        }
        if (__any_sync(0xffffffffu, hasq))
            c5_site<RULE, 1, false>(a, K, K.t31, ty1, site, hasq, count, Vc, qn, e.x, e.y, e.z, e.w, R);
        if (qn >= 32) {
            qn -= 32;
            tpw_drain<RULE>(a, qn, 32, K.tlo, K.thi);
        }
        if (count && ++since >= flush_every) {  // keep the 8-bit vertical counters from overflowing
            vflush(Vc, logW, s_cc);
            uint32_t V[kVB], any = 0u;
#pragma unroll
            for (int b = 0; b < kVB; ++b) { V[b] = vq[b * kTpwThreads]; any |= V[b]; }
            if (__any_sync(0xffffffffu, any)) {
                vflush(V, logW, s_cq);
#pragma unroll
                for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = 0u;
            }
            since = 0;
        }
    }
    while (qn > 0) {
        const int n = qn < 32 ? qn : 32;
        qn -= n;
        tpw_drain<RULE>(a, qn, n, K.tlo, K.thi);
    }
    if (count) {
        vflush(Vc, logW, s_cc);
        uint32_t V[kVB], any = 0u;
#pragma unroll
        for (int b = 0; b < kVB; ++b) { V[b] = vq[b * kTpwThreads]; any |= V[b]; }
        if (__any_sync(0xffffffffu, any)) {
            vflush(V, logW, s_cq);
#pragma unroll
            for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = 0u;
        }
    }
}

// One colour phase over this warp's items.
template <int RULE, int FAST>
__device__ __forceinline__ void tpw_phase(const PlaneArgs& a, int c, uint64_t t, bool count, int gw,
                                          int nw, int logW, uint32_t (&Vc)[kVB], int flush_every) {
    int* s_cc = tpw_sm + kTpwSmCnt;
    int* s_cq = s_cc + 32 * a.W;
    uint32_t* vq = reinterpret_cast<uint32_t*>(tpw_sm + kTpwSmVq) + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int W = 1 << logW, S = 32 >> logW;
    const int w = lane & (W - 1), sl = lane >> logW;
    const uint32_t act_w = a.active[w];
    const uint32_t grp4 = (uint32_t)(a.w_global0 + w) << 4;
    const uint32_t thi = (uint32_t)(t >> 32), tlo = (uint32_t)t;
    const int c0 = a.chunk_off[c];
    const int n_items = (a.chunk_off[c + 1] - c0) << logW;
    const int lower = a.color_start[c];
    count = count && lower > 0;  // colour 0 has no lower-colour neighbours
    int since = 0, qn = 0;
    int item = gw;
    Chunk nxt{};
    if (item < n_items) nxt = a.chunks[c0 + (item >> logW)];
    while (item < n_items) {
        const Chunk ch = nxt;
        const int p0 = (item & (W - 1)) * S;
        item += nw;
        if (item < n_items) nxt = a.chunks[c0 + (item >> logW)];  // prefetch the next descriptor
        if (p0 >= ch.len) continue;
        const PlaneType& ty = a.ty[ch.type];
#define TG_TCASE(C, Q)                                                                               \
    case (C) * 4 + (Q):                                                                              \
        tpw_site<C, Q, RULE>(a, ch, ty, p0 + sl, w, act_w, grp4, tlo, thi, count, lower, Vc, qn); \
        break;
        {
            switch (ty.ncb * 4 + ty.nqb) {
                TG_TCASE(0, 0) TG_TCASE(0, 1) TG_TCASE(0, 2)
                TG_TCASE(1, 0) TG_TCASE(1, 1) TG_TCASE(1, 2)
                TG_TCASE(2, 0) TG_TCASE(2, 1) TG_TCASE(2, 2)
                TG_TCASE(3, 0) TG_TCASE(3, 1) TG_TCASE(3, 2)
                default: break;
            }
        }
#undef TG_TCASE
        if (qn >= 32) {
            qn -= 32;
            tpw_drain<RULE>(a, qn, 32, tlo, thi);
        }
        if (count && ++since >= flush_every) {  // keep the 8-bit vertical counters from overflowing
            vflush(Vc, logW, s_cc);
            uint32_t V[kVB], any = 0u;
#pragma unroll
            for (int b = 0; b < kVB; ++b) { V[b] = vq[b * kTpwThreads]; any |= V[b]; }
            if (__any_sync(0xffffffffu, any)) {
                vflush(V, logW, s_cq);
#pragma unroll
                for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = 0u;
            }
            since = 0;
        }
    }
    while (qn > 0) {
        const int n = qn < 32 ? qn : 32;
        qn -= n;
        tpw_drain<RULE>(a, qn, n, tlo, thi);
    }
    if (count) {
        vflush(Vc, logW, s_cc);
        // chain counters: only warps that met chain sites
        uint32_t V[kVB], any = 0u;
#pragma unroll
        for (int b = 0; b < kVB; ++b) { V[b] = vq[b * kTpwThreads]; any |= V[b]; }
        if (__any_sync(0xffffffffu, any)) {
            vflush(V, logW, s_cq);
#pragma unroll
            for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = 0u;
        }
    }
}

// Persistent single-GPU kernel: n_rounds whole rounds of run_2dpt
// (engine.cpp:121-216); one grid barrier per colour phase, the round
// epilogue (plane_round.cuh) closes each round.
template <int RULE, int FAST>
__global__ void __launch_bounds__(kTpwThreads, kTpwMinBlocks)
plane_tpw_rounds_kernel(const __grid_constant__ PlaneArgs a, const __grid_constant__ RoundArgs r) {
    cg::grid_group grid = cg::this_grid();
    const int nrep = a.W * 32;
    int* s_cc = tpw_sm + kTpwSmCnt;
    int* s_cq = s_cc + nrep;
    const RoundSmem s = round_smem(s_cq + nrep, r.R);
    uint32_t* vq = reinterpret_cast<uint32_t*>(tpw_sm + kTpwSmVq) + threadIdx.x;
    // launch constants as kernel parameters (host-computed): when register
    // pressure makes the compiler rematerialise them inside the item loop a
    // constant-bank load is all it costs
    const int logW = r.log_w;
    const int gw = blockIdx.x * (kTpwThreads >> 5) + (threadIdx.x >> 5);
    const int nw = r.n_warps;
    const int flush_every = r.flush_every;  // <= 255 / (max bonds per item): 8-bit counters
    for (int m = threadIdx.x; m < 2 * nrep; m += blockDim.x) s_cc[m] = 0;
#pragma unroll
    for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = 0u;
    round_load_labels(r, s);
    __syncthreads();
    uint32_t Vc[kVB];
#pragma unroll
    for (int b = 0; b < kVB; ++b) Vc[b] = 0u;
    uint64_t swap_base = r.swap_base0;
    for (int k = 0; k < r.n_rounds; ++k) {
        const int64_t round = r.round0 + k;
        const int par = (int)(round & 1);
        int32_t* cc = r.cnt + (size_t)par * 2 * r.cnt_stride;
        int32_t* cq = cc + r.cnt_stride;
        TPW_STAMP(k, 0);
        if (FAST && RULE == 1) tpw_stage_hb(a);
        for (int sw = 0; sw < r.sps; ++sw) {
            const uint64_t t = (uint64_t)((round - 1) * r.sps + sw);
            const bool count = (sw == r.sps - 1);
            for (int c = 0; c < a.n_colors; ++c) {
                if constexpr (FAST)
                    tpw_phase_c5<RULE>(a, c, t, count, gw, nw, logW, Vc, flush_every,
                                       r.work ? r.work + (size_t)(par * a.n_colors + c) * r.sps + sw : nullptr);
                else tpw_phase<RULE, FAST>(a, c, t, count, gw, nw, logW, Vc, flush_every);
                TPW_STAMP(k, 1 + 3 * (c & 1));
                TPW_MAXSTAMP(k, 2 + 3 * (c & 1));
                if (count && a.color_start[c] > 0) {
                    __syncthreads();
                    for (int m = threadIdx.x; m < nrep; m += blockDim.x) {
                        const int vc = s_cc[m], vqv = s_cq[m];
                        if (vc) { atomicAdd(cc + m, vc); s_cc[m] = 0; }
                        if (vqv) { atomicAdd(cq + m, vqv); s_cq[m] = 0; }
                    }
                }
                grid.sync();
                TPW_STAMP(k, 3 + 3 * (c & 1));
            }
        }
        round_epilogue(a, r, s, k, round, cc, cq, swap_base, a.n_colors * r.sps);
        TPW_STAMP(k, 7);
    }
}

// Sweep-only variant (multi-GPU, full-grid records): n_sweeps sweeps, then
// every replica's (f, g) in reference units from the bond counts (which it
// zeroes); the (f, g) exchange and the swap phase run after it.
template <int RULE, int FAST>
__global__ void __launch_bounds__(kTpwThreads, kTpwMinBlocks)
plane_tpw_sweep_kernel(const __grid_constant__ PlaneArgs a, int64_t t0, int n_sweeps) {
    if (a.rs) t0 = a.rs->round * n_sweeps;
    cg::grid_group grid = cg::this_grid();
    const int nrep = a.W * 32;
    int* s_cc = tpw_sm + kTpwSmCnt;
    int* s_cq = s_cc + nrep;
    uint32_t* vq = reinterpret_cast<uint32_t*>(tpw_sm + kTpwSmVq) + threadIdx.x;
    const int logW = __ffs(a.W) - 1;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int flush_every = FAST ? 255 / 3 : 255 / 7;
    for (int m = threadIdx.x; m < 2 * nrep; m += blockDim.x) s_cc[m] = 0;
#pragma unroll
    for (int b = 0; b < kVB; ++b) vq[b * kTpwThreads] = 0u;
    __syncthreads();
    uint32_t Vc[kVB];
#pragma unroll
    for (int b = 0; b < kVB; ++b) Vc[b] = 0u;
    if (FAST && RULE == 1) tpw_stage_hb(a);  // labels are fixed for the whole launch
    for (int sw = 0; sw < n_sweeps; ++sw) {
        const uint64_t t = (uint64_t)(t0 + sw);
        const bool count = (sw == n_sweeps - 1);
        for (int c = 0; c < a.n_colors; ++c) {
            if constexpr (FAST) tpw_phase_c5<RULE>(a, c, t, count, gw, nw, logW, Vc, flush_every);
            else tpw_phase<RULE, FAST>(a, c, t, count, gw, nw, logW, Vc, flush_every);
            if (count && a.color_start[c] > 0) {
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

template __global__ void plane_tpw_sweep_kernel<TG_PLANE_RULE, 0>(const __grid_constant__ PlaneArgs, int64_t, int);
template __global__ void plane_tpw_sweep_kernel<TG_PLANE_RULE, 1>(const __grid_constant__ PlaneArgs, int64_t, int);

void* TG_CAT(plane_tpw_sweep_fn_r, TG_PLANE_RULE)(int fast) {
    return fast ? (void*)plane_tpw_sweep_kernel<TG_PLANE_RULE, 1>
                : (void*)plane_tpw_sweep_kernel<TG_PLANE_RULE, 0>;
}

template __global__ void plane_tpw_rounds_kernel<TG_PLANE_RULE, 0>(const __grid_constant__ PlaneArgs,
                                                                   const __grid_constant__ RoundArgs);
template __global__ void plane_tpw_rounds_kernel<TG_PLANE_RULE, 1>(const __grid_constant__ PlaneArgs,
                                                                   const __grid_constant__ RoundArgs);

#if TG_TPW_PROF && TG_PLANE_RULE == 0
extern "C" int tg_debug_tpw_prof(unsigned long long* dst) {
    return (int)cudaMemcpyFromSymbol(dst, g_tpw_prof, sizeof(g_tpw_prof));
}
extern "C" int tg_debug_tpw_prof_reset() {
    static unsigned long long z[64][16] = {};
    return (int)cudaMemcpyToSymbol(g_tpw_prof, z, sizeof(z));
}
#endif

void* TG_CAT(plane_tpw_fn_r, TG_PLANE_RULE)(int fast) {
    return fast ? (void*)plane_tpw_rounds_kernel<TG_PLANE_RULE, 1>
                : (void*)plane_tpw_rounds_kernel<TG_PLANE_RULE, 0>;
}


}  // namespace tg
