// slot_fast.cu -- FLOAT engine: the float-coupling sweep (configs 2-4) with
// packed draws keyed by physical replica.
//
// Same update as the reference sweep (mc.cpp:21-35: u < exp(-beta de) /
// heat bath u < sigma(2 beta h), one uniform per spin) over the canonical
// colour order, in the SLOT v2 batch layout (spins int8 [instance][site][Rp],
// labels permuted by slot2_swap_kernel).  Differences from SLOT v2:
//
// * RNG association: the 53-bit uniform of physical replica m at sweep t,
//   site i is hi16 << 37 | lo37 (oracle/philox_ref.h tgo_pack_u53): hi16 is
//   halfword m & 7 of one Philox4x32-10 block per (site, sweep, 8 replicas),
//   lo37 comes from a per-replica block that is only generated when the 16
//   leading bits cannot settle the decision.  One block serves 8 updates.
// * Thread = (site, 8 consecutive replicas): one 8-byte load per row, the
//   site's entries, field and couplings shared by its 8 replicas.
// * Certified FP32 decisions: FP32 field and exp with the error band of
//   slot_engine.cu s2_update; u lies in [hi16 2^-16, (hi16 + 1) 2^-16), so the
//   decision is taken from the 16 bits when that interval clears the band and
//   falls back to the reference's FP64 expression with all 53 bits otherwise
//   (probability ~1e-4): decisions equal the FP64 ones.
// * Energies: per-thread FP64 partials of the lower-colour bonds, flushed as
//   2^-40 fixed-point integers with integer atomics (order-independent, so
//   runs are bit-reproducible), converted to (f, g) after the last sweep.
//
// Work layout: lanes per site LPS = min(32, Rp / 8); a warp item is
// SPW = 32 / LPS sites (Rp < 256) or one site and one of NGS = Rp / 256
// 256-replica group sets; every warp keeps one group set for the launch and
// walks a contiguous range of its colour's items, so a lane's instance (its
// labels and accumulators) changes rarely.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tg {

__device__ __forceinline__ int sf_find_instance(const int* pref, int B, int item) {
    int lo = 0, hi = B;  // pref[lo] <= item < pref[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pref[mid] <= item) lo = mid; else hi = mid;
    }
    return lo;
}

// w with its sign flipped where byte `k` (0..3) of `word` is negative (spin -1)
__device__ __forceinline__ float sf_signed(float w, uint32_t word, int k) {
    return __int_as_float(__float_as_int(w) ^ ((word << (24 - 8 * k)) & 0x80000000u));
}

#ifndef TG_SF_FASTDEC
#define TG_SF_FASTDEC 2  // 2: one-comparison certified decisions; 0: the previous accept / reject predicates (A/B)
#endif

// 2^x, one MUFU.EX2 (relative error 2^-22; results below 2^-126 flush to zero,
// which the decisions below treat as "smaller than every nonzero prefix").
__device__ __forceinline__ float sf_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sf_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// FP64 decision of one replica with all 53 bits (the semantics the FP32 path
// certifies): local field in the reference's merged-CSR order
// (constraints.cpp:122-140, ising.cpp:79-88), then mc.cpp:27-29 / heat bath.
__device__ __forceinline__ int sf_exact(const S2Args& a, const SInst& in, const int8_t* sp, int i, int r,
                                     int si8, uint64_t u53, double beta, double two_p, int rule) {
    double local = a.h[in.h_off + i];
    const int e0 = a.off[in.csr_off + i], e1 = a.off[in.csr_off + i + 1];
    for (int e = e0; e < e1; ++e) {
        const int q = in.nbr_off + e;
        const double wgt = a.w[q] + (double)a.cm[q] * two_p;
        local += wgt * (double)sp[(size_t)a.nbr[q] * a.Rp + r];
    }
    const double u = (double)u53 * 0x1.0p-53;
    if (rule == 0) {
        const double de = 2.0 * (double)si8 * local;
        return (de <= 0.0 || u < exp(-beta * de)) ? -si8 : si8;
    }
    const double p = 1.0 / (1.0 + exp(-2.0 * beta * local));
    return u < p ? 1 : -1;
}

// Per-thread accumulators of one instance: FP64 cost energy and chain-bond
// counts of the thread's 8 replicas, flushed as fixed point.
__device__ __forceinline__ void sf_flush(const S2Args& a, int b, int m0, double (&fl)[8], uint32_t (&g16)[4]) {
    long long* fx = a.fx + (size_t)b * a.Rp + m0;
    int* gx = a.gx + (size_t)b * a.Rp + m0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int gj = (int)((g16[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
        if (fl[j] != 0.0) atomicAdd(reinterpret_cast<unsigned long long*>(fx + j),
                                    (unsigned long long)__double2ll_rn(fl[j] * 0x1.0p40));
        if (gj) atomicAdd(gx + j, gj);
        fl[j] = 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) g16[j] = 0u;
}

template <int RULE, int DEG, int D>
__global__ void __launch_bounds__(kSlotFThreads, 1)
slotf_sweep_kernel(const __grid_constant__ S2Args a, int64_t t0, int n_sweeps, int do_energy) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
    const int nw = gridDim.x * wpb;
    const int ngs = a.fngs, lps = a.flps, spw = a.fspw;
    const int gs = gw % ngs, wi = gw / ngs, nwi = nw / ngs;  // host: nw % ngs == 0
    const int sub = lane / lps;
    const int grp = gs * 32 + lane % lps;                   // replicas 8 grp .. 8 grp + 7
    const bool lane_on = sub < spw && grp * 8 < a.Rp;
    const int m0 = grp * 8;
    const unsigned Rp = (unsigned)a.Rp;
    for (int swp = 0; swp < n_sweeps; ++swp) {
        const uint64_t t = (uint64_t)(t0 + swp);
        const uint32_t tlo = (uint32_t)t, thi = (uint32_t)(t >> 32);
        const bool count = do_energy && swp == n_sweeps - 1;
        double fl[8];
        uint32_t g16[4];  // chain counters, two replicas per word (16-bit lanes)
        int since = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) fl[j] = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) g16[j] = 0u;
        for (int c = 0; c < a.max_colors; ++c) {
            const int* pref = a.fitem_pref + (size_t)c * (a.B + 1);
            const int total = pref[a.B];
            const int lo = (int)((long long)wi * total / nwi), hi = (int)((long long)(wi + 1) * total / nwi);
            int b = -1, b_end = 0;
            int cs = 0, ce = 0, p0 = 0;
            float bt[8], tp[8];       // beta, 2P of the lanes' replicas (current instance)
            uint32_t k0 = 0, k1 = 0;  // the instance's pack key
            float tol = 0.f, c1 = 0.f;  // de dead band; band coefficient of T (p)
            const SInst* in = nullptr;
            for (int item = lo; item < hi; ++item) {
                if (item >= b_end) {  // next instance (flush the previous one's energies)
                    if (count && b >= 0 && lane_on) sf_flush(a, b, m0, fl, g16);
                    since = 0;
                    b = (b < 0) ? sf_find_instance(pref, a.B, item) : b + 1;
                    while (pref[b + 1] <= item) ++b;
                    b_end = pref[b + 1];
                    p0 = pref[b];
                    in = a.inst + b;
                    cs = a.color_start[in->color_off + c];
                    ce = a.color_start[in->color_off + c + 1];
                    k0 = (uint32_t)in->pkey;
                    k1 = (uint32_t)(in->pkey >> 32);
                    {   // error band of slot_engine.cu s2_update: T (2 eb + |x| 2^-19 + 2^-18),
                        // heat bath eb + |y| 2^-19 + 2^-18, eb = 2 beta_max eps
                        const float eb = 2.0f * in->beta_max * in->eps;
                        tol = 2.0f * in->eps;
                        c1 = RULE == 0 ? 2.0f * eb + 0x1.0p-18f : eb + 0x1.0p-18f;
#if TG_SF_FASTDEC == 2
                        if (in->beta_max * in->eps > 0.125f) c1 = 0x1.0p+100f;  // nothing certified: all FP64
#endif
                    }
                    if (lane_on) {
                        const float4* lp = reinterpret_cast<const float4*>(a.lab + (size_t)b * a.Rp + m0);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float4 v = lp[q];
                            bt[2 * q] = v.x; tp[2 * q] = v.y; bt[2 * q + 1] = v.z; tp[2 * q + 1] = v.w;
#if TG_SF_FASTDEC == 2
                            // -2 beta log2(e): exp(-2 beta s l) = 2^(bt s l)
                            bt[2 * q] *= -2.885390081777927f;
                            bt[2 * q + 1] *= -2.885390081777927f;
#endif
                        }
                    }
                }
                const int i = cs + (item - p0) * spw + sub;
                if (!lane_on || i >= ce) continue;
                int8_t* sp = a.spins + in->spin_off;
                // the site's entries {j | cm << 28 | fwd << 27, float J}
                const int2* ep = a.entp + in->entp_off + (size_t)i * D;
                int2 e[D];
#pragma unroll
                for (int q = 0; q < D / 2; ++q) {
                    const int4 v = __ldg(reinterpret_cast<const int4*>(ep) + q);
                    e[2 * q] = make_int2(v.x, v.y);
                    e[2 * q + 1] = make_int2(v.z, v.w);
                }
                uint2 rk[DEG];
#pragma unroll
                for (int k = 0; k < DEG; ++k)
                    rk[k] = *reinterpret_cast<const uint2*>(sp + (size_t)(unsigned)(e[k].x & 0x07ffffff) * Rp + m0);
                uint2* own = reinterpret_cast<uint2*>(sp + (size_t)(unsigned)i * Rp + m0);
                const uint2 s0 = *own;
                const float h32 = __ldg(a.h32 + in->h_off + i);
                const u32x4 o = philox4x32_10(u32x4{(uint32_t)i, tlo, thi, (uint32_t)grp | (1u << 30)}, k0, k1);
                // field of the 8 replicas: cost couplings (item-uniform J) and
                // chain multiplicities times the replica's 2P
                float l[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) l[j] = h32;
#pragma unroll
                for (int k = 0; k < DEG; ++k) {
                    const float jk = __int_as_float(e[k].y);
                    const int cmk = (e[k].x >> 28) & 15;
                    if (jk != 0.0f) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) l[j] += sf_signed(jk, j < 4 ? rk[k].x : rk[k].y, j & 3);
                    }
                    if (cmk) {
                        const float cf = (float)cmk;
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            l[j] = fmaf(sf_signed(cf, j < 4 ? rk[k].x : rk[k].y, j & 3), tp[j], l[j]);
                    }
                }
                // certified decisions from the 16-bit prefix; undecided replicas
                // (|u - T| inside the error band) take the FP64 path below
                uint32_t fm0 = 0u, fm1 = 0u;  // bytes to flip (0xFE: +1 <-> -1)
                uint32_t und = 0u;
#if TG_SF_FASTDEC == 2
                // One comparison per replica.  With w = T - uf0 (T = exp(-beta de)
                // resp. the heat-bath p; uf0 = hi16 2^-16 <= u < uf0 + 2^-16) and
                // A = band + 2^-16: u < T is certain when w >= A, u >= T is
                // certain when w <= -A, and only |w| < A goes to the FP64 path
                // (probability ~2^-15).  Metropolis needs no test of the sign
                // of de: for de <= eps the band (>= T 4 beta_max eps, host
                // guarantees beta_max eps <= 1/8) puts T + A above 1 > uf0, so a
                // rejection is never certified there, and a certified
                // acceptance is right for either sign.  The exponent is clamped
                // at 2^64 (de < 0 deep: accepted for every u) so T stays finite; a
                // T flushed to zero (below 2^-126) leaves A = 2^-16, so the bucket
                // of hi16 = 0 stays undecided and every other one is rejected.
                float mu = -1.0f;  // max over replicas of A - |w|: > 0 <=> someone undecided
                auto decide = [&](int j, float& w, float& A) {
                    const uint32_t ow = j < 4 ? s0.x : s0.y;
                    const float hwf = __uint2float_rn(((j < 2 ? o.x : j < 4 ? o.y : j < 6 ? o.z : o.w) >> (16 * (j & 1))) & 0xFFFFu);
                    if (RULE == 0) {
                        const float x2 = fminf(bt[j] * sf_signed(l[j], ow, j & 3), 64.0f);  // -2 beta s l log2(e)
                        const float T = sf_ex2(x2);
                        A = fmaf(T, fmaf(fabsf(x2), 0x1.62e430p-20f, c1), 0x1.0p-16f);
                        w = fmaf(hwf, -0x1.0p-16f, T);
                    } else {
                        const float y2 = bt[j] * l[j];                     // -2 beta l log2(e)
                        const float p = sf_rcp(1.0f + sf_ex2(y2));
                        A = fmaf(fabsf(y2), 0x1.62e430p-20f, c1 + 0x1.0p-16f);
                        w = fmaf(hwf, -0x1.0p-16f, p);
                    }
                };
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float w, A;
                    decide(j, w, A);
                    const uint32_t ow = j < 4 ? s0.x : s0.y;
                    const int bj = j & 3;
                    bool flip;
                    if (RULE == 0) flip = w >= A;                      // u < T certain
                    else {
                        const bool up = ((ow >> (8 * bj + 7)) & 1u) == 0u;  // current spin +1
                        flip = up ? (w <= -A) : (w >= A);
                    }
                    if (flip) {
                        if (j < 4) fm0 |= 0xFEu << (8 * bj);
                        else fm1 |= 0xFEu << (8 * bj);
                    }
                    mu = fmaxf(mu, A - fabsf(w));
                }
                if (mu > 0.0f) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float w, A;
                        decide(j, w, A);
                        if (fabsf(w) < A) und |= 1u << j;
                    }
                }
#else
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t ow = j < 4 ? s0.x : s0.y;
                    const int bj = j & 3;
                    const float lj = l[j];
                    const uint32_t hw = ((j < 2 ? o.x : j < 4 ? o.y : j < 6 ? o.z : o.w) >> (16 * (j & 1))) & 0xFFFFu;
                    const float uf0 = __uint2float_rn(hw) * 0x1.0p-16f;
                    const float uf1 = uf0 + 0x1.0p-16f;
                    bool flip, undec;
                    if (RULE == 0) {
                        const float de = 2.0f * sf_signed(lj, ow, bj);  // 2 s_i l
                        const float x = -bt[j] * de;
                        const float T = __expf(x);
                        const float band = T * fmaf(fabsf(x), 0x1.0p-19f, c1);
                        const bool pos = de > tol;
                        const bool acc = de < -tol || (pos && uf1 + band <= T);
                        const bool rej = pos && uf0 >= T + band;
                        flip = acc;
                        undec = !(acc || rej);
                    } else {  // heat bath: new spin +1 iff u < sigma(2 beta l)
                        const float y = 2.0f * bt[j] * lj;
                        const float p = __frcp_rn(1.0f + __expf(-y));
                        const float band = fmaf(fabsf(y), 0x1.0p-19f, c1);
                        const bool up = ((ow >> (8 * bj + 7)) & 1u) == 0u;  // current spin +1
                        const bool nup = uf1 + band <= p, ndown = uf0 >= p + band;
                        flip = up ? ndown : nup;
                        undec = !(nup || ndown);
                    }
                    if (flip) {
                        if (j < 4) fm0 |= 0xFEu << (8 * bj);
                        else fm1 |= 0xFEu << (8 * bj);
                    }
                    und |= (uint32_t)undec << j;
                }
#endif
                while (und) {  // FP64 with all 53 bits (rare)
                    const int j = __ffs(und) - 1;
                    und &= und - 1;
                    const int m = m0 + j;
                    const uint32_t ow = j < 4 ? s0.x : s0.y;
                    const int bj = j & 3;
                    const uint32_t ox = j < 2 ? o.x : j < 4 ? o.y : j < 6 ? o.z : o.w;
                    const uint32_t hw = (ox >> (16 * (j & 1))) & 0xFFFFu;
                    const u32x4 q2 = philox4x32_10(u32x4{(uint32_t)i, tlo, thi, (uint32_t)m | (2u << 30)}, k0, k1);
                    const uint64_t u53 = ((uint64_t)hw << 37) |
                                         (((uint64_t)q2.x | ((uint64_t)q2.y << 32)) & ((1ull << 37) - 1ull));
                    const int si8 = ((ow >> (8 * bj + 7)) & 1u) ? -1 : 1;
                    const int nv = sf_exact(a, *in, sp, i, m, si8, u53, a.sbeta[(size_t)b * a.Rp + m],
                                            a.stwop[(size_t)b * a.Rp + m], RULE);
                    if (nv != si8) {
                        if (j < 4) fm0 |= 0xFEu << (8 * bj);
                        else fm1 |= 0xFEu << (8 * bj);
                    }
                }
                const uint2 s1 = make_uint2(s0.x ^ fm0, s0.y ^ fm1);
                if (fm0 | fm1) *own = s1;
                if (count) {  // bonds to lower-colour neighbours (each bond once) and the field
                    uint2 gb = make_uint2(0u, 0u);  // unsatisfied chain bonds x multiplicity, per byte
#pragma unroll
                    for (int k = 0; k < DEG; ++k) {
                        const int jn = e[k].x & 0x07ffffff;
                        if (jn >= cs) continue;
                        const int cmk = (e[k].x >> 28) & 15;
                        const uint32_t dx = s1.x ^ rk[k].x, dy = s1.y ^ rk[k].y;  // bytes 0xFE where s_i != s_k
                        if (__int_as_float(e[k].y) != 0.0f) {
                            const double nwk = -a.wp[in->entp_off + (size_t)i * D + k];  // -J s_i s_k, s_i = s_k
                            const int hi = __double2hiint(nwk), lo = __double2loint(nwk);
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const uint32_t d = j < 4 ? dx : dy;
                                fl[j] += __hiloint2double(hi ^ (int)((d << (24 - 8 * (j & 3))) & 0x80000000u), lo);
                            }
                        }
                        if (cmk) {
                            gb.x += ((dx >> 7) & 0x01010101u) * (uint32_t)cmk;
                            gb.y += ((dy >> 7) & 0x01010101u) * (uint32_t)cmk;
                        }
                    }
                    g16[0] += __byte_perm(gb.x, 0u, 0x4140);
                    g16[1] += __byte_perm(gb.x, 0u, 0x4342);
                    g16[2] += __byte_perm(gb.y, 0u, 0x4140);
                    g16[3] += __byte_perm(gb.y, 0u, 0x4342);
                    const double h64 = a.h[in->h_off + i];
                    if (h64 != 0.0) {
                        const int hi = __double2hiint(-h64), lo = __double2loint(-h64);  // -h_i s_i
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const uint32_t w = j < 4 ? s1.x : s1.y;
                            fl[j] += __hiloint2double(hi ^ (int)((w << (24 - 8 * (j & 3))) & 0x80000000u), lo);
                        }
                    }
                    if (++since >= 1024) {  // 16-bit chain counters: flush well before overflow
                        sf_flush(a, b, m0, fl, g16);
                        since = 0;
                    }
                }
            }
            if (count && b >= 0 && lane_on) sf_flush(a, b, m0, fl, g16);
            grid.sync();
        }
    }
    if (!do_energy) return;
    // (f, g) of every replica: f = cost energy, g = 4 x unsatisfied chain bonds
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.B * a.R; q += gridDim.x * blockDim.x) {
        const int b = q / a.R, r = q % a.R;
        const size_t x = (size_t)b * a.Rp + r;
        a.f[q] = (double)a.fx[x] * 0x1.0p-40;
        a.g[q] = 4.0 * (double)a.gx[x];
        a.fx[x] = 0;
        a.gx[x] = 0;
    }
}

template __global__ void slotf_sweep_kernel<0, 3, 4>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slotf_sweep_kernel<1, 3, 4>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slotf_sweep_kernel<0, 4, 4>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slotf_sweep_kernel<1, 4, 4>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slotf_sweep_kernel<0, 8, 8>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slotf_sweep_kernel<1, 8, 8>(const __grid_constant__ S2Args, int64_t, int, int);

// deg: the batch's largest merged degree (<= 8)
void* slotf_sweep_fn(int rule, int deg) {
    if (deg <= 3) return rule ? (void*)slotf_sweep_kernel<1, 3, 4> : (void*)slotf_sweep_kernel<0, 3, 4>;
    if (deg <= 4) return rule ? (void*)slotf_sweep_kernel<1, 4, 4> : (void*)slotf_sweep_kernel<0, 4, 4>;
    return rule ? (void*)slotf_sweep_kernel<1, 8, 8> : (void*)slotf_sweep_kernel<0, 8, 8>;
}

}  // namespace tg
