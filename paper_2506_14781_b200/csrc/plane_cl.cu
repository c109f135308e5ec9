// plane_cl.cu -- the cluster-per-word fused round kernel of the PLANE engine
// (config 5 at small and medium N: 2^14 .. 2^18 sites).
//
// Same contract, and therefore the same trajectories bit for bit, as
// plane_c5_rounds_kernel: the reference sweep (mc.cpp:21-35) over the
// canonical colour order, thresholds K = ceil(T * 2^53) compared MSB-first
// against bit planes of Philox4x32-10 draws with counter {site, t_lo, t_hi,
// group << 4 | block}, the swap phase of engine.cpp:148-187 replayed on
// labels.  What changes is the decomposition.  The replicas of different
// 32-replica words never interact inside a sweep, so every word gets its own
// thread-block cluster (C CTAs on C SMs of one GPC):
//   * a colour phase ends with a hardware cluster barrier (barrier.cluster,
//     ~0.2 us) instead of a grid barrier (~1.3 us): words run ahead of one
//     another inside a round;
//   * each CTA owns fixed slices of the four site ranges (colour x chain-free /
//     chain); their neighbour entries are staged once per launch into its
//     shared memory by TMA bulk copies (cp.async.bulk + mbarrier), which takes
//     the entry -> row dependent load out of every update;
//   * the unsatisfied-bond counts of a word are reduced through distributed
//     shared memory (atomics on the cluster leader's shared memory) and
//     published by the leader as one tagged 64-bit word per replica {round,
//     chain count, cost count}; the only grid-wide step of a round is that
//     (f, g) exchange -- every CTA polls the 32 W words (the data is its own
//     flag: no fence, no second round trip) -- after which every CTA replays
//     the swap phase and rebuilds the threshold planes of its own word in its
//     own shared memory (ktab, betas, penalties staged there as well);
//   * the target digest / snapshot is taken by the cluster that holds the
//     target replica, each CTA over the sites it updates itself.
// thread = (site, word); per-warp deferred-tail queue as in plane_c5.cu.
//
// Two launch modes share the kernel (template GROUP).  Cluster mode is the one
// described above.  On B200 one GPC hosts no cluster larger than 10 CTAs when
// 8 are needed, so cluster mode runs on 80 of the 148 SMs; group mode gives a
// word G = floor(SMs / W) CTAs of an ordinary cooperative launch (144 SMs for
// 8 words): the word's colour-phase barrier is then a software barrier on a
// per-word global counter and the counts are reduced with global atomics.
// The hardware barrier wins at 2^14 sites, the extra SMs from 2^15 up.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"
#include "philox_plane.cuh"
#include "plane_device.cuh"
#include "plane_round.cuh"

namespace cg = cooperative_groups;

namespace tg {

// Stage timer (variant builds only, -DTG_CL_PROF=1): thread 0 of block 0
// records %globaltimer at the stages of the first 64 rounds of a launch.
#ifndef TG_CL_PROF
#define TG_CL_PROF 0
#endif
#if TG_CL_PROF
__device__ unsigned long long g_cl_prof[64][16];
#define CL_STAMP(k, s)                                                                  \
    do {                                                                                \
        if ((k) < 64 && blockIdx.x == 0 && threadIdx.x == 0) {                          \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                       \
            g_cl_prof[k][s] = t_;                                                       \
        }                                                                               \
    } while (0)
__device__ int g_cl_k;
#define CL_SETK(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_cl_k = (k); } while (0)
#else
#define CL_STAMP(k, s) do {} while (0)
#define CL_SETK(k) do {} while (0)
#endif

extern __shared__ __align__(16) int cl_sm[];

// Dynamic shared memory (kernels.cuh cl_smem_bytes): queues [warps][kClQCap]
// int4 | kp of the word [kpw] | kpc of the word [n_types][128] | Philox key
// schedule [24] | local counts [64] | cluster totals [64] | mbarrier | betas
// [I] | penalties [J] | accepted swaps [np + nb] | labels + energies
// (plane_round.cuh) | ktab [R][row]
// (when it fits) | staged neighbour entries.
struct ClSmem {
    int4* queue;
    uint32_t* kp;
    uint32_t* kpc;
    uint32_t* pks;
    int* loc;
    int* tot;
    unsigned long long* mbar;
    double* betas;
    double* pens;
    int* acc;               // accepted swaps of this launch [np + nb]
    RoundSmem rs;
    const uint64_t* ktab;   // shared-memory copy, or the global table
    int4* stage;
};

// wpt: words per thread (1 or 2): kp | kpc | loc | tot hold one block per word
__device__ __forceinline__ ClSmem cl_smem(const PlaneArgs& a, const RoundArgs& r, int wpt) {
    ClSmem s;
    int* p = cl_sm;
    s.queue = reinterpret_cast<int4*>(p);
    p += (kClThreads / 32) * kClQCap * 4;
    s.kp = reinterpret_cast<uint32_t*>(p);
    p += wpt * ((a.kpw + 3) & ~3);
    s.kpc = reinterpret_cast<uint32_t*>(p);
    p += wpt * a.n_types * 128;
    s.pks = reinterpret_cast<uint32_t*>(p);
    p += 24;
    s.loc = p;
    p += wpt * 64;
    s.tot = p;
    p += wpt * 64;
    s.mbar = reinterpret_cast<unsigned long long*>(p);
    p += 4;
    s.betas = reinterpret_cast<double*>(p);
    p += 2 * ((r.I + 1) & ~1);
    s.pens = reinterpret_cast<double*>(p);
    p += 2 * ((r.J + 1) & ~1);
    s.acc = p;
    p += (r.I * (r.J > 1 ? r.J - 1 : 0) + (r.I > 1 ? r.I - 1 : 0) * r.J + 3) & ~3;
    s.rs = round_smem(p, r.R);
    p += (int)((round_smem_bytes(r.R) + 15) / 16) * 4;
    s.ktab = r.ktab;
    if (r.cl_ktab) {
        s.ktab = reinterpret_cast<const uint64_t*>(p);
        p += ((2 * r.R * r.ktab_row + 3) & ~3);
    }
    s.stage = reinterpret_cast<int4*>(p);
    return s;
}

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared memory of this CTA, completion on `bar`.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_gpu_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Group mode: barrier of the G CTAs of one word on the word's global counter
// (monotonic: `target` = G x barriers so far); the fence of thread 0 after the
// CTA barrier publishes the CTA's spin stores (read with ld.cg by the peers).
__device__ __forceinline__ void cl_group_sync(unsigned int* bar, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_gpu_u32(bar) < target) {}
    }
    __syncthreads();
}

// ------------------------------------------------------------ thresholds

// 8-class select from shared-memory leaves (chain sites: class = c0 + 2 c1 + 4 q).
__device__ __forceinline__ uint32_t cl_mux8(const uint32_t* cb, const uint32_t* leaves) {
    const uint4 lo = *reinterpret_cast<const uint4*>(leaves);
    const uint4 hi = *reinterpret_cast<const uint4*>(leaves + 4);
    const uint32_t a = sel(cb[1], sel(cb[0], lo.w, lo.z), sel(cb[0], lo.y, lo.x));
    const uint32_t b = sel(cb[1], sel(cb[0], hi.w, hi.z), sel(cb[0], hi.y, hi.x));
    return sel(cb[2], b, a);
}

__device__ __forceinline__ void cl_compare8(const uint32_t* cb, const uint32_t* kpb, int blk,
                                            const u32x4& r, uint32_t& und, uint32_t& lt) {
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int b = blk * 4 + q;
        if (b < kKPlanes) {
            const uint32_t tb = cl_mux8(cb, kpb + b * 8);
            lt |= und & tb & ~rr[q];
            und &= ~(tb ^ rr[q]);
        }
    }
}

// Threshold planes of word w for the labels in s_state, into this CTA's
// shared memory (and the global tables when to_global): one warp per (type,
// class); plane b = bit 52 - b of the lanes' thresholds by two 32x32
// transposes (plane_round.cuh).
// w0: the CTA's first word, wpt its word count (word w0 + j fills block j).
__device__ __forceinline__ void cl_build_planes(const PlaneArgs& a, const RoundArgs& r,
                                                const int32_t* s_state, int w0, int wpt, const ClSmem& S,
                                                bool to_global) {
    const int lane = threadIdx.x & 31;
    int combos = 0;
    for (int ty = 0; ty < a.n_types; ++ty) combos += a.ty[ty].ncl;
    const int kpw4 = (a.kpw + 3) & ~3;
    for (int job = threadIdx.x >> 5; job < combos * wpt; job += blockDim.x >> 5) {
        const int jw = job / combos, w = w0 + jw;
        int c = job % combos, ty = 0;
        while (c >= a.ty[ty].ncl) { c -= a.ty[ty].ncl; ++ty; }
        const PlaneType& pt = a.ty[ty];
        const int m = w * 32 + lane;
        const bool live = m < a.local_states;
        uint64_t K = 0;
        if (live) K = S.ktab[(size_t)s_state[m] * r.ktab_row + pt.ktab_off + c];
        const uint32_t th = warp_transpose32((uint32_t)(K >> 21));
        const uint32_t tl = warp_transpose32((uint32_t)(K << 11));
        const uint32_t alw = __ballot_sync(0xffffffffu, live && K >= (1ull << 53));
        const int bh = 31 - lane, bl = 63 - lane;
        const bool cls = c == 2 || c == 3;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            if (g == 1 && !to_global) break;
            uint32_t* dst = (g ? r.kp + (size_t)w * a.kpw : S.kp + jw * kpw4) + pt.kp_off + c;
            uint32_t* dstc = (g ? r.kpc + (size_t)w * a.n_types * 128 : S.kpc + jw * a.n_types * 128) + ty * 128 +
                             (c - 2) * 64;
            dst[bh * pt.ncl] = th;
            if (cls) dstc[bh] = th;
            if (lane >= 11) {
                dst[bl * pt.ncl] = tl;
                if (cls) dstc[bl] = tl;
            }
            if (lane == 0) dst[kKPlanes * pt.ncl] = alw;
        }
    }
}

// ------------------------------------------------------------ counters

// V += m (NB-bit bit-sliced value) in NP-plane vertical arithmetic.
template <int NB, int NP>
__device__ __forceinline__ void cl_vadd(uint32_t (&V)[NP], uint32_t m0, uint32_t m1) {
    uint32_t carry = 0u;
#pragma unroll
    for (int b = 0; b < NP; ++b) {
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

// Warp total of the lanes' NP-plane vertical counters (all lanes hold the
// same word): bit-sliced butterfly all-reduce, after which every lane holds
// every plane and lane l reads replica l's count.  Added into dst[l].
template <int NP>
__device__ __noinline__ void cl_vflush(uint4 lo, uint4 hi, int* dst) {  // by value: V stays in registers
    const int lane = threadIdx.x & 31;
    const uint32_t Vin[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t E[NP + 5];
#pragma unroll
    for (int b = 0; b < NP + 5; ++b) E[b] = b < NP ? Vin[b] : 0u;
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        uint32_t carry = 0u;
#pragma unroll
        for (int b = 0; b <= NP + lv && b < NP + 5; ++b) {
            const uint32_t x = E[b];
            const uint32_t o = __shfl_xor_sync(0xffffffffu, x, 1 << lv);
            E[b] = x ^ o ^ carry;
            carry = (x & o) | (carry & (x ^ o));
        }
    }
    int val = 0;
#pragma unroll
    for (int b = 0; b < NP + 5; ++b) val += (int)((E[b] >> lane) & 1u) << b;
    if (val) atomicAdd(dst + lane, val);
}

template <int NP>
__device__ __forceinline__ void cl_flush(uint32_t (&V)[NP], int* dst) {
    if constexpr (NP == 8)
        cl_vflush<NP>(make_uint4(V[0], V[1], V[2], V[3]), make_uint4(V[4], V[5], V[6], V[7]), dst);
    else
        cl_vflush<NP>(make_uint4(V[0], V[1], V[2], V[3]), make_uint4(0u, 0u, 0u, 0u), dst);
#pragma unroll
    for (int b = 0; b < NP; ++b) V[b] = 0u;
}

// ------------------------------------------------------------ deferred tail

// Resolve queue entries [0, n) (n <= 32) of `queue`, one per lane
// (plane_c5.cu c5_drain): Philox blocks 2.. of the entry's (site, word),
// threshold planes 8.. of the word, late decisions applied to the stored word
// and, when counting, the unsatisfied-bond correction.  Bit 30 of the entry's
// site field selects the thread's second word (strides kcs / khs of its
// threshold blocks).  Everything it reads but the spin word is in shared memory.
template <int RULE>
__device__ __noinline__ void cl_drain(uint32_t* spins_w, int logW, const int4* queue, const uint32_t* ks,
                                      const uint4* kc2, const uint4* kh, int kcs, int khs, int* loc,
                                      uint32_t grp4, int n, uint32_t tlo, uint32_t thi, bool count) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    int4 e = make_int4(0, 0, 0, 0);
    if (lane < n) e = queue[lane];
    const uint32_t site = (uint32_t)e.x & 0x3fffffffu;
    const int jw = (int)(((uint32_t)e.x >> 30) & 1u);
    uint32_t und = (uint32_t)e.y;
    const uint32_t c0 = (uint32_t)e.z, c1 = (uint32_t)e.w;
    kc2 += jw * kcs;
    kh += jw * khs;
    loc += jw * 64;
    grp4 += (uint32_t)jw << 4;
    uint32_t lt = 0u;
    const PhiloxT P = philox_t(tlo, thi, ks);
#pragma unroll 1
    for (int blk = 2; blk < 14; ++blk) {
        if (!__any_sync(0xffffffffu, und)) break;
        const u32x4 r = philox_plane(site, grp4 | (uint32_t)blk, P, ks);
        if (RULE == 0) {
            compare4_sel(c0, kc2[blk], kc2[16 + blk], r, und, lt);
        } else {
            const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int b = blk * 4 + q;
                if (b < kKPlanes) {
                    const uint4 T = kh[b];  // the 4 classes of plane b
                    const uint32_t tb = sel(c1, sel(c0, T.w, T.z), sel(c0, T.y, T.x));
                    lt |= und & tb & ~rr[q];
                    und &= ~(tb ^ rr[q]);
                }
            }
        }
    }
    if (lt) {
        uint32_t* p = spins_w + ((size_t)site << logW) + jw;
        const uint32_t old = __ldcg(p);
        *p = RULE == 0 ? old ^ lt : old | lt;
        if (count) {
            uint32_t ex = lt;
            while (ex) {
                const int l = __ffs(ex) - 1;
                ex &= ex - 1;
                const int b0 = (int)((c0 >> l) & 1u), b1 = (int)((c1 >> l) & 1u);
                atomicAdd(loc + l, RULE == 0 ? 1 + 2 * b0 : 3 - 2 * (b0 + 2 * b1));
            }
        }
    }
    __syncwarp();
}

// ------------------------------------------------------------ site slices

// Slice of the site range [b, e) that CTA `rank` of a C-CTA cluster updates
// (multiples of 32 sites).
__device__ __forceinline__ void cl_slice(int b, int e, int rank, int C, int& lo, int& hi) {
    int per = (e - b + C - 1) / C;
    per = (per + 31) & ~31;
    lo = b + rank * per;
    hi = lo + per < e ? lo + per : e;
    if (lo > e) lo = e;
    if (hi < lo) hi = lo;
}

// One row load of the thread's WPT words (an 8-byte access for a word pair).
template <int WPT>
__device__ __forceinline__ void cl_row(const uint32_t* p, uint32_t (&v)[WPT]) {
    if constexpr (WPT == 2) {
        const uint2 t = __ldcg(reinterpret_cast<const uint2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = __ldcg(p);
    }
}

// ------------------------------------------------------------ colour phase

// One colour phase of this CTA: its chain-free slice [flo, fhi), then its
// chain slice [qlo, qhi); fent / qent address the slices' staged entries by
// site (null: the global table).  thread = (site, WPT words from word w0).
template <int RULE, int NP, int WPT>
__device__ __forceinline__ void cl_phase(const PlaneArgs& a, const RoundArgs& r, const ClSmem& S, int w0,
                                         uint64_t t, bool count, int t30, int t31, uint32_t (&V)[WPT][NP],
                                         uint32_t (&Q)[WPT][NP], int flo, int fhi, const int4* fent, int qlo,
                                         int qhi, const int4* qent) {
    constexpr int kFlushAt = NP == 8 ? 85 : 5;  // items between flushes: 3 bonds each, NP-bit counters
    const int lane = threadIdx.x & 31;
    const int logW = r.log_w;
    uint32_t act_w[WPT];
#pragma unroll
    for (int j = 0; j < WPT; ++j) act_w[j] = a.active[w0 + j];
    const uint32_t g0 = (uint32_t)(a.w_global0 + w0) << 4;
    uint32_t gg[2 * WPT];  // Philox word 3 of the unconditional blocks
#pragma unroll
    for (int j = 0; j < WPT; ++j) { gg[2 * j] = g0 + 16u * j; gg[2 * j + 1] = (g0 + 16u * j) | 1u; }
    const uint32_t tlo = (uint32_t)t, thi = (uint32_t)(t >> 32);
    const PhiloxT P = philox_t(tlo, thi, a.pks);
    uint32_t* base = a.spins + w0;
    // row at word offset `off` (< 2^30: n <= 2^18 sites): 32-bit byte offset,
    // the flag bits 30-31 of an nbr4 entry fall off the shift
    auto rowp = [&](uint32_t off) -> uint32_t* {
        return reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(base) + (uint32_t)(off << 2));
    };
    int4* queue = S.queue + (threadIdx.x >> 5) * kClQCap;
    const int kcs = a.n_types * 32, khs = ((a.kpw + 3) & ~3) >> 2;  // uint4 strides between the words' blocks
    const uint4* kc = reinterpret_cast<const uint4*>(S.kpc + t30 * 128);
    const uint4* kh = reinterpret_cast<const uint4*>(S.kp + a.ty[t30].kp_off);
    int qn = 0;
    int since = 0;
    // ---------------------------------------------------------- chain-free
    {
        uint4 k2a, k2b, k3a, k3b;  // one word per thread: its class-2/3 planes 0-7 stay in registers
        if (RULE == 0 && WPT == 1) { k2a = kc[0]; k2b = kc[1]; k3a = kc[16]; k3b = kc[17]; }
        // software pipeline: the rows of the next site and the entry of the
        // one after it are in flight while the current site computes
        auto entry = [&](int st) -> int4 {
            int4 v = make_int4(0, 0, 0, 0);
            if (st < fhi) v = fent ? fent[st] : __ldg(a.nbr4 + st);
            return v;
        };
        struct Rows { uint32_t s[WPT], x0[WPT], x1[WPT], x2[WPT]; };
        auto rows = [&](int st, const int4& en) -> Rows {
            Rows q;
#pragma unroll
            for (int j = 0; j < WPT; ++j) { q.s[j] = 0u; q.x0[j] = 0u; q.x1[j] = 0u; q.x2[j] = 0u; }
            if (st < fhi) {
                cl_row<WPT>(rowp((uint32_t)st << logW), q.s);
                cl_row<WPT>(rowp((uint32_t)en.x), q.x0);
                cl_row<WPT>(rowp((uint32_t)en.y), q.x1);
                cl_row<WPT>(rowp((uint32_t)en.z), q.x2);
            }
            return q;
        };
        const int first = flo + (int)(threadIdx.x & ~31u) + lane;
        int4 en = entry(first);
        Rows rn = rows(first, en);
        int4 en2 = entry(first + kClThreads);
        for (int b0 = flo + (int)(threadIdx.x & ~31u); b0 < fhi; b0 += kClThreads) {
            const int site = b0 + lane;
            const bool valid = site < fhi;
            const int4 e = en;
            const Rows q = rn;
            en = en2;
            rn = rows(site + kClThreads, en);
            en2 = entry(site + 2 * kClThreads);
            u32x4 rr4[2 * WPT];
            philox_planeN<2 * WPT>((uint32_t)site, gg, P, a.pks, rr4);
            const uint32_t m0s = (uint32_t)(e.x >> 31), m1s = (uint32_t)(e.y >> 31), m2s = (uint32_t)(e.z >> 31);
            uint32_t und[WPT], nsv[WPT], cl0[WPT], cl1[WPT];
#pragma unroll
            for (int j = 0; j < WPT; ++j) {
                const uint32_t s = q.s[j];
                const uint32_t bb0 = q.x0[j] ^ m0s, bb1 = q.x1[j] ^ m1s, bb2 = q.x2[j] ^ m2s;
                const uint32_t a0 = RULE == 0 ? ~(s ^ bb0) : bb0, a1 = RULE == 0 ? ~(s ^ bb1) : bb1,
                               a2 = RULE == 0 ? ~(s ^ bb2) : bb2;
                const uint32_t c0 = a0 ^ a1 ^ a2;
                const uint32_t c1 = (a0 & a1) | (a2 & (a0 ^ a1));
                const uint32_t act = valid ? act_w[j] : 0u;
                const u32x4 r0 = rr4[2 * j], r1 = rr4[2 * j + 1];
                uint32_t u, lt = 0u, take, ns;
                if (RULE == 0) {
                    u = c1 & act;  // classes 0, 1 (de <= 0): always taken
#if TG_CMP8
                    if (WPT == 1) {
                        compare8_sel(c0, k2a, k2b, k3a, k3b, r0, r1, u, u, lt);
                    } else {
                        const uint4* kj = kc + j * kcs;
                        compare8_sel(c0, kj[0], kj[1], kj[16], kj[17], r0, r1, u, u, lt);
                    }
                    take = act & (~c1 | lt);
#else
                    if (WPT == 1) {
                        compare4_sel(c0, k2a, k3a, r0, u, lt);
                        compare4_sel(c0, k2b, k3b, r1, u, lt);
                    } else {
                        const uint4* kj = kc + j * kcs;
                        compare4_sel(c0, kj[0], kj[16], r0, u, lt);
                        compare4_sel(c0, kj[1], kj[17], r1, u, lt);
                    }
                    take = (~c1 & act) | lt;
#endif
                    ns = s ^ take;
                } else {
                    const uint4* kj = kh + j * khs;
                    const uint4 L = kj[kKPlanes];
                    const uint32_t always = sel(c1, sel(c0, L.w, L.z), sel(c0, L.y, L.x)) & act;
                    u = act & ~always;
                    const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#if TG_CMP8
                    uint32_t tb[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const uint4 T = kj[b];
                        tb[b] = sel(c1, sel(c0, T.w, T.z), sel(c0, T.y, T.x));
                    }
                    compare8(tb, rr, u, u, lt);  // lt beyond u: covered by `always` / masked by act
#else
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const uint4 T = kj[b];
                        const uint32_t tb = sel(c1, sel(c0, T.w, T.z), sel(c0, T.y, T.x));
                        lt |= u & tb & ~rr[b];
                        u &= ~(tb ^ rr[b]);
                    }
#endif
                    take = (always | lt) & act;  // new spin +1 (undecided lanes provisionally -1)
                    ns = (s & ~act) | take;
                }
                if (count) {  // unsatisfied bonds after the update (all neighbours are colour 0)
                    uint32_t m0, m1;
                    if (RULE == 0) {
                        m0 = ~(c0 ^ take) & act;
                        m1 = ~(c1 ^ take) & act;
                    } else {
                        const uint32_t u0 = ns ^ bb0, u1 = ns ^ bb1, u2 = ns ^ bb2;
                        m0 = (u0 ^ u1 ^ u2) & act;
                        m1 = ((u0 & u1) | (u2 & (u0 ^ u1))) & act;
                    }
                    cl_vadd<2, NP>(V[j], m0, m1);
                }
                und[j] = u;
                nsv[j] = ns;
                cl0[j] = c0;
                cl1[j] = c1;
            }
            if (count && ++since == kFlushAt) {
#pragma unroll
                for (int j = 0; j < WPT; ++j) cl_flush<NP>(V[j], S.loc + j * 64);
                since = 0;
            }
            if (valid) {
                if constexpr (WPT == 2)
                    *reinterpret_cast<uint2*>(rowp((uint32_t)site << logW)) = make_uint2(nsv[0], nsv[1]);
                else
                    *rowp((uint32_t)site << logW) = nsv[0];
            }
            // deferred tail: (site, word)s with lanes still undecided after 8 planes
#pragma unroll
            for (int j = 0; j < WPT; ++j) {
                const uint32_t pend = __ballot_sync(0xffffffffu, und[j] != 0u);
                if (pend) {
                    if (und[j])
                        queue[qn + __popc(pend & ((1u << lane) - 1u))] =
                            make_int4((int)((uint32_t)site | ((uint32_t)j << 30)), (int)und[j], (int)cl0[j],
                                      (int)cl1[j]);
                    qn += __popc(pend);
                    if (qn >= 32) {
                        qn -= 32;
                        cl_drain<RULE>(base, logW, queue + qn, S.pks, kc, kh, kcs, khs, S.loc, g0, 32, tlo, thi,
                                       count);
                    }
                }
            }
        }
        if (count) CL_STAMP(g_cl_k, 9);
        if (qn > 0) cl_drain<RULE>(base, logW, queue, S.pks, kc, kh, kcs, khs, S.loc, g0, qn, tlo, thi, count);
        if (count) CL_STAMP(g_cl_k, 10);
    }
    // ---------------------------------------------------------- chain sites
    {
        const int kpw4 = (a.kpw + 3) & ~3;
        // the last warps take the chain sites: they have the fewest chain-free sites
        for (int b0 = qlo + (int)((kClThreads - 32) - (threadIdx.x & ~31u)); b0 < qhi; b0 += kClThreads) {
            const int site = b0 + lane;
            const bool valid = site < qhi;
            int4 e = make_int4(0, 0, 0, 0);
            uint32_t s[WPT], x0[WPT], x1[WPT], x2[WPT], y[WPT];
#pragma unroll
            for (int j = 0; j < WPT; ++j) { s[j] = 0u; x0[j] = 0u; x1[j] = 0u; x2[j] = 0u; y[j] = 0u; }
            if (valid) {
                e = qent ? qent[site] : __ldg(a.nbr4 + site);
                cl_row<WPT>(rowp((uint32_t)site << logW), s);
                cl_row<WPT>(rowp((uint32_t)e.x), x0);
                cl_row<WPT>(rowp((uint32_t)e.y), x1);
                cl_row<WPT>(rowp((uint32_t)e.z), x2);
                cl_row<WPT>(rowp((uint32_t)e.w), y);
            }
            u32x4 rr4[2 * WPT];
            philox_planeN<2 * WPT>((uint32_t)site, gg, P, a.pks, rr4);
            const uint32_t m0s = (uint32_t)(e.x >> 31), m1s = (uint32_t)(e.y >> 31), m2s = (uint32_t)(e.z >> 31);
            uint32_t nsv[WPT];
#pragma unroll
            for (int j = 0; j < WPT; ++j) {
                const uint32_t* kpb = S.kp + j * kpw4 + a.ty[t31].kp_off;
                const uint32_t bb0 = x0[j] ^ m0s, bb1 = x1[j] ^ m1s, bb2 = x2[j] ^ m2s;
                const uint32_t a0 = RULE == 0 ? ~(s[j] ^ bb0) : bb0, a1 = RULE == 0 ? ~(s[j] ^ bb1) : bb1,
                               a2 = RULE == 0 ? ~(s[j] ^ bb2) : bb2;
                const uint32_t cb[3] = {a0 ^ a1 ^ a2, (a0 & a1) | (a2 & (a0 ^ a1)),
                                        RULE == 0 ? ~(s[j] ^ y[j]) : y[j]};
                const uint32_t act = valid ? act_w[j] : 0u;
                const uint32_t always = cl_mux8(cb, kpb + kKPlanes * 8) & act;
                uint32_t u = act & ~always, lt = 0u;
#if TG_CMP8
                {
                    const u32x4 r0 = rr4[2 * j], r1 = rr4[2 * j + 1];
                    const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
                    uint32_t tb[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b) tb[b] = cl_mux8(cb, kpb + b * 8);
                    compare8(tb, rr, u, u, lt);  // lt beyond u: covered by `always` / masked by act
                }
#else
                cl_compare8(cb, kpb, 0, rr4[2 * j], u, lt);
                cl_compare8(cb, kpb, 1, rr4[2 * j + 1], u, lt);
#endif
#pragma unroll 1
                for (int blk = 2; blk < 14; ++blk) {
                    if (!__any_sync(0xffffffffu, u)) break;
                    const u32x4 rb = philox_plane((uint32_t)site, gg[2 * j] | (uint32_t)blk, P, S.pks);
                    cl_compare8(cb, kpb, blk, rb, u, lt);
                }
                const uint32_t take = (always | lt) & act;
                const uint32_t ns = RULE == 0 ? s[j] ^ take : (s[j] & ~act) | take;
                if (count) {
                    const uint32_t mq = (ns ^ y[j]) & act;  // chain bond unsatisfied after the update
                    uint32_t m0, m1;
                    if (RULE == 0) {
                        m0 = ~(cb[0] ^ take) & act;
                        m1 = ~(cb[1] ^ take) & act;
                    } else {
                        const uint32_t u0 = ns ^ bb0, u1 = ns ^ bb1, u2 = ns ^ bb2;
                        m0 = (u0 ^ u1 ^ u2) & act;
                        m1 = ((u0 & u1) | (u2 & (u0 ^ u1))) & act;
                    }
                    cl_vadd<2, NP>(V[j], m0, m1);
                    cl_vadd<1, NP>(Q[j], mq, 0u);
                }
                nsv[j] = ns;
            }
            if (count && ++since == kFlushAt) {
#pragma unroll
                for (int j = 0; j < WPT; ++j) {
                    cl_flush<NP>(V[j], S.loc + j * 64);
                    cl_flush<NP>(Q[j], S.loc + j * 64 + 32);
                }
                since = 0;
            }
            if (valid) {
                if constexpr (WPT == 2)
                    *reinterpret_cast<uint2*>(rowp((uint32_t)site << logW)) = make_uint2(nsv[0], nsv[1]);
                else
                    *rowp((uint32_t)site << logW) = nsv[0];
            }
        }
    }
    if (count) CL_STAMP(g_cl_k, 11);
    if (count) {
#pragma unroll
        for (int j = 0; j < WPT; ++j) {
            cl_flush<NP>(V[j], S.loc + j * 64);
            if (qhi > qlo) cl_flush<NP>(Q[j], S.loc + j * 64 + 32);
        }
    }
}

// ------------------------------------------------------------ the kernel

// n_rounds whole rounds of run_2dpt (engine.cpp:121-216).  Grid = W / WPT
// clusters (or groups) of C CTAs, all co-resident.  NP: planes of the
// per-thread vertical bond counters (4 when a thread updates <= 5 sites per
// phase, else 8); GROUP: software word barrier instead of clusters; WPT: words
// per thread (2: the word pair shares the site's Philox products and row
// sectors, as in plane_c5.cu).
template <int RULE, int NP, int GROUP, int WPT>
__global__ void __launch_bounds__(kClThreads, 1)
plane_cl_rounds_kernel(const __grid_constant__ PlaneArgs a, const __grid_constant__ RoundArgs r) {
    cg::cluster_group cluster = cg::this_cluster();
    const int C = GROUP ? r.cl_size : (int)cluster.num_blocks();
    const int nrep = a.W * 32;
    if (C != r.cl_size) {  // the launch lost its cluster attribute (seen under a profiler): report, touch nothing
        if (blockIdx.x == 0 && threadIdx.x == 0) r.cl_x[2 * nrep] = 1ull;
        return;
    }
    const int rank = GROUP ? (int)(blockIdx.x % C) : (int)cluster.block_rank();
    const int wq = blockIdx.x / C;       // the CTA's word group
    const int w0 = wq * WPT;             // its first word
    unsigned int* gbar = r.cl_bar + wq * 32;  // group mode: the word group's barrier counter (own 128-byte line)
    unsigned int gtarget = 0;
    const int tid = threadIdx.x, lane = tid & 31;
    const ClSmem S = cl_smem(a, r, WPT);
    const RoundSmem s = S.rs;
    const int np = r.I * (r.J > 1 ? r.J - 1 : 0);
    const int nb = (r.I > 1 ? r.I - 1 : 0) * r.J;
    int t30 = 0, t31 = 0;
    for (int ty = 0; ty < a.n_types; ++ty) {
        if (a.ty[ty].dq == 0) t30 = ty;
        else t31 = ty;
    }
    // this CTA's slices of the four site ranges (colour x {chain-free, chain})
    int flo[2], fhi[2], qlo[2], qhi[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int cs = a.color_start[c], ce = a.color_start[c + 1], cf = cs + r.c5_nfree[c];
        cl_slice(cs, cf, rank, C, flo[c], fhi[c]);
        cl_slice(cf, ce, rank, C, qlo[c], qhi[c]);
    }
    const int off_f1 = fhi[0] - flo[0], off_q0 = off_f1 + fhi[1] - flo[1], off_q1 = off_q0 + qhi[0] - qlo[0];
    const int n_stage = off_q1 + qhi[1] - qlo[1];
    const int4* fent[2] = {nullptr, nullptr};
    const int4* qent[2] = {nullptr, nullptr};
    if (r.cl_stage) {
        fent[0] = S.stage - flo[0];
        fent[1] = S.stage + off_f1 - flo[1];
        qent[0] = S.stage + off_q0 - qlo[0];
        qent[1] = S.stage + off_q1 - qlo[1];
    }
    // ---- launch prologue: staged entries (TMA), tables, labels, this word group's planes
    if (tid == 0) {
        mbar_init(S.mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (r.cl_stage && tid == 0) {
        mbar_expect_tx(S.mbar, (uint32_t)n_stage * 16u);
        if (fhi[0] > flo[0]) tma_bulk_g2s(S.stage, a.nbr4 + flo[0], (uint32_t)(fhi[0] - flo[0]) * 16u, S.mbar);
        if (fhi[1] > flo[1]) tma_bulk_g2s(S.stage + off_f1, a.nbr4 + flo[1], (uint32_t)(fhi[1] - flo[1]) * 16u, S.mbar);
        if (qhi[0] > qlo[0]) tma_bulk_g2s(S.stage + off_q0, a.nbr4 + qlo[0], (uint32_t)(qhi[0] - qlo[0]) * 16u, S.mbar);
        if (qhi[1] > qlo[1]) tma_bulk_g2s(S.stage + off_q1, a.nbr4 + qlo[1], (uint32_t)(qhi[1] - qlo[1]) * 16u, S.mbar);
    }
    for (int m = tid; m < 128 * WPT; m += blockDim.x) S.loc[m] = 0;  // loc + tot
    if (tid < 20) S.pks[tid] = a.pks[tid];
    for (int m = tid; m < r.I; m += blockDim.x) S.betas[m] = r.betas[m];
    for (int m = tid; m < r.J; m += blockDim.x) S.pens[m] = r.pens[m];
    for (int m = tid; m < np + nb; m += blockDim.x) S.acc[m] = 0;
    if (r.cl_ktab) {
        uint64_t* kt = const_cast<uint64_t*>(S.ktab);
        for (int m = tid; m < r.R * r.ktab_row; m += blockDim.x) kt[m] = r.ktab[m];
    }
    round_load_labels(r, s);
    __syncthreads();
    cl_build_planes(a, r, s.state, w0, WPT, S, false);
    if (r.cl_stage) mbar_wait(S.mbar, 0);
    __syncthreads();
    int* tot0 = S.tot;
    if (!GROUP) {
        cluster.sync();  // every CTA of the cluster has zeroed its totals
        tot0 = cluster.map_shared_rank(S.tot, 0);
    }
    uint32_t V[WPT][NP], Q[WPT][NP];
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
#pragma unroll
        for (int b = 0; b < NP; ++b) { V[j][b] = 0u; Q[j][b] = 0u; }
    }
    uint64_t swap_base = r.swap_base0;
    const int n_groups = a.W / WPT;
    for (int k = 0; k < r.n_rounds; ++k) {
        const int64_t round = r.round0 + k;
        unsigned long long* xw = r.cl_x + (size_t)(k & 1) * nrep;  // exchange words of this parity
        const unsigned long long tag = (unsigned long long)((k + 1) & 0xffff);
        int* gt = r.cl_gtot + ((size_t)(k & 1) * n_groups + wq) * 64 * WPT;  // group mode: this group's totals
        CL_SETK(k);
        CL_STAMP(k, 0);
        for (int sw = 0; sw < r.sps; ++sw) {
            const uint64_t t = (uint64_t)((round - 1) * r.sps + sw);
            const bool count = (sw == r.sps - 1);
            cl_phase<RULE, NP, WPT>(a, r, S, w0, t, false, t30, t31, V, Q, flo[0], fhi[0], fent[0], qlo[0],
                                    qhi[0], qent[0]);
            CL_STAMP(k, 1);
            if (GROUP) cl_group_sync(gbar, gtarget += (unsigned)C);
            else cluster.sync();
            CL_STAMP(k, 2);
            cl_phase<RULE, NP, WPT>(a, r, S, w0, t, count, t30, t31, V, Q, flo[1], fhi[1], fent[1], qlo[1],
                                    qhi[1], qent[1]);
            CL_STAMP(k, 3);
            if (count) {  // word totals through distributed shared memory (group mode: global atomics)
                __syncthreads();
                if (tid < 64 * WPT) {
                    const int v = S.loc[tid];
                    if (v) {
                        atomicAdd(GROUP ? gt + tid : tot0 + tid, v);
                        S.loc[tid] = 0;
                    }
                }
            }
            if (GROUP) cl_group_sync(gbar, gtarget += (unsigned)C);
            else cluster.sync();
            CL_STAMP(k, 4);
        }
        // ---- (f, g) exchange: the leader publishes the words' counts, tagged with the round
        if (rank == 0 && tid < 32 * WPT) {
            const int jw = tid >> 5, l = tid & 31;
            unsigned long long cc, cq;
            if (GROUP) {
                cc = (unsigned long long)(uint32_t)__ldcg(gt + jw * 64 + l);
                cq = (unsigned long long)(uint32_t)__ldcg(gt + jw * 64 + 32 + l);
                gt[jw * 64 + l] = 0;       // this parity's totals are next added to two rounds on
                gt[jw * 64 + 32 + l] = 0;
            } else {
                cc = (unsigned long long)(uint32_t)S.tot[jw * 64 + l];
                cq = (unsigned long long)(uint32_t)S.tot[jw * 64 + 32 + l];
                S.tot[jw * 64 + l] = 0;
                S.tot[jw * 64 + 32 + l] = 0;
            }
            st_relaxed_gpu(xw + (w0 + jw) * 32 + l, tag << 48 | cq << 24 | cc);
        }
        // everything of this thread's swap attempt that does not depend on the energies (slots,
        // labels, coefficients, the draw) is done while the words arrive
        const int n_att = (int)round_attempts(r.I, r.J, round);
        SwapPrep sp{};
        if (tid < n_att)
            sp = swap_prepare(r.I, r.J, S.betas, S.pens, round, tid, s.slot,
                              swap_uniform(r.swap_seed, swap_base, tid));
        CL_STAMP(k, 13);
        for (int m = tid; m < r.R; m += blockDim.x) {
            unsigned long long v;
            do { v = ld_relaxed_gpu(xw + m); } while ((v >> 48) != tag);
            s.f[m] = -((double)a.m_cost - 2.0 * (double)(uint32_t)(v & 0xffffffull));
            s.g[m] = 4.0 * (double)(uint32_t)((v >> 24) & 0xffffffull);
        }
        __syncthreads();
        CL_STAMP(k, 5);
        // ---- swap phase (engine.cpp:148-187), replayed identically by every CTA
        for (int q = tid; q < n_att; q += blockDim.x) {
            if (q != tid)
                sp = swap_prepare(r.I, r.J, S.betas, S.pens, round, q, s.slot,
                                  swap_uniform(r.swap_seed, swap_base, q));
            if (swap_decide(sp, s.f, s.g)) {
                // the attempts of a round touch disjoint slot pairs
                s.slot[sp.slot_a] = sp.sb;
                s.slot[sp.slot_b] = sp.sa;
                s.state[sp.sb] = sp.slot_a;
                s.state[sp.sa] = sp.slot_b;
                S.acc[sp.is_p ? sp.counter : np + sp.counter] += 1;  // one attempt per counter and round
            }
        }
        swap_base += (uint64_t)n_att;
        CL_STAMP(k, 12);
        __syncthreads();
        const int tg = s.slot[r.R - 1];
        CL_STAMP(k, 6);
        if (blockIdx.x == 0) {
            if (tid == 0) {  // record, engine.cpp:189-208 (digest added atomically by the target's group)
                TgRecordDev* rec = reinterpret_cast<TgRecordDev*>(r.rec) + k;
                rec->round = round;
                rec->sweep_count = round * r.sps;
                rec->f = s.f[tg];
                rec->g = s.g[tg];
                rec->feasible = s.g[tg] == 0.0 ? 1 : 0;
                rec->target_state = tg;
            }
            if ((r.rec_flags & 8) && r.rec_acc) {
                int64_t* dst = r.rec_acc + (size_t)k * (np + nb);
                for (int q = tid; q < np; q += blockDim.x) dst[q] = r.acc_p[q] + S.acc[q];
                for (int q = tid; q < nb; q += blockDim.x) dst[np + q] = r.acc_b[q] + S.acc[np + q];
            }
            if (k == r.n_rounds - 1) {  // labels, energies and counters after the launch's last round (same thread per counter as above)
                for (int m = tid; m < r.R; m += blockDim.x) {
                    r.slot_state[m] = s.slot[m];
                    r.state_slot[m] = s.state[m];
                    r.f_all[m] = s.f[m];
                    r.g_all[m] = s.g[m];
                }
                for (int q = tid; q < np; q += blockDim.x) r.acc_p[q] += S.acc[q];
                for (int q = tid; q < nb; q += blockDim.x) r.acc_b[q] += S.acc[np + q];
            }
        }
        // ---- threshold planes of this CTA's words for the new labels
        cl_build_planes(a, r, s.state, w0, WPT, S, rank == 0 && k == r.n_rounds - 1);
        CL_STAMP(k, 7);
        // ---- target digest / snapshot: the target's word group, each CTA over its own sites
        if ((r.rec_flags & 3) && (tg >> 5) / WPT == wq) {
            uint64_t dsum = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int lo = q < 2 ? flo[q & 1] : qlo[q & 1], hi = q < 2 ? fhi[q & 1] : qhi[q & 1];
                for (int i = lo + tid; i < hi; i += blockDim.x) {
                    const uint32_t wv = __ldcg(a.spins + (size_t)i * a.W + (tg >> 5));
                    const int ci = r.perm[i];
                    const bool up = (wv >> (tg & 31)) & 1u;
                    if (r.rec_flags & 2) r.rec_states[(size_t)k * a.n + ci] = up ? 1 : -1;
                    if (up) dsum += digest_term((uint64_t)ci);
                }
            }
            if (r.rec_flags & 1) {
#pragma unroll
                for (int o = 16; o; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
                if (lane == 0 && dsum)
                    atomicAdd(reinterpret_cast<unsigned long long*>(
                                  &(reinterpret_cast<TgRecordDev*>(r.rec) + k)->digest),
                              (unsigned long long)dsum);
            }
        }
        __syncthreads();
        CL_STAMP(k, 8);
    }
    if (!GROUP) cluster.sync();  // no CTA exits while a peer may still address its shared memory
}

#define TG_CL_INST(R, P, G, T) \
    template __global__ void plane_cl_rounds_kernel<R, P, G, T>(const __grid_constant__ PlaneArgs, \
                                                                const __grid_constant__ RoundArgs);
TG_CL_INST(0, 4, 0, 1) TG_CL_INST(1, 4, 0, 1) TG_CL_INST(0, 8, 0, 1) TG_CL_INST(1, 8, 0, 1)
TG_CL_INST(0, 4, 1, 1) TG_CL_INST(1, 4, 1, 1) TG_CL_INST(0, 8, 1, 1) TG_CL_INST(1, 8, 1, 1)
TG_CL_INST(0, 4, 1, 2) TG_CL_INST(1, 4, 1, 2) TG_CL_INST(0, 8, 1, 2) TG_CL_INST(1, 8, 1, 2)
#undef TG_CL_INST

// small: 4-plane counters; group: software word barrier; pair: two words per thread (group mode only)
void* plane_cl_fn(int rule, int small, int group, int pair) {
#define TG_CL_PICK(G, T)                                                                               \
    (small ? (rule ? (void*)plane_cl_rounds_kernel<1, 4, G, T> : (void*)plane_cl_rounds_kernel<0, 4, G, T>) \
           : (rule ? (void*)plane_cl_rounds_kernel<1, 8, G, T> : (void*)plane_cl_rounds_kernel<0, 8, G, T>))
    if (group && pair) return TG_CL_PICK(1, 2);
    if (group) return TG_CL_PICK(1, 1);
    return TG_CL_PICK(0, 1);
#undef TG_CL_PICK
}

}  // namespace tg

#if TG_CL_PROF
extern "C" int tg_debug_cl_prof(unsigned long long* dst) {
    return (int)cudaMemcpyFromSymbol(dst, tg::g_cl_prof, sizeof(tg::g_cl_prof));
}
#endif
