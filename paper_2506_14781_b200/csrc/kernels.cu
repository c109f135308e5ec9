// kernels.cu -- sm_100a kernels of the 2D-PT hot path.
//
//   plane_sweep_kernel   multi-spin-coded chromatic sweeps (PLANE engine)
//   slot_sweep_kernel    int8 / FP64 chromatic sweeps, one CTA per replica (SLOT engine)
//   swap_kernel          P / beta label swaps, round record, threshold-plane rebuild
//   extract_kernel       target-state digest / snapshot for the trace
//   *_init_kernel        initial configurations (engine.cpp:98-106)
//
// Reference semantics restated: metropolis_sweep (mc.cpp:21-35), swap phases
// and record (engine.cpp:121-216).  See DESIGN.md for layouts and rooflines.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tg {

// ------------------------------------------------------------ helpers

__device__ __forceinline__ uint32_t sel(uint32_t m, uint32_t a1, uint32_t a0) {
    return (m & a1) | (~m & a0);
}

// Select, per lane bit, leaves[class(lane)] where class bits are cb[0..B).
template <int B>
__device__ __forceinline__ uint32_t mux_tree(const uint32_t* cb, const uint32_t* leaves) {
    constexpr int L = 1 << B;
    uint32_t v[L < 4 ? 4 : L];
    if constexpr (L >= 4) {
#pragma unroll
        for (int q = 0; q < L / 4; ++q) {
            const uint4 t = __ldg(reinterpret_cast<const uint4*>(leaves) + q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < L; ++q) v[q] = __ldg(leaves + q);
    }
#pragma unroll
    for (int lvl = 0; lvl < B; ++lvl) {
#pragma unroll
        for (int c = 0; c < (L >> (lvl + 1)); ++c) v[c] = sel(cb[lvl], v[2 * c + 1], v[2 * c]);
    }
    return v[0];
}

// Add a one-bit-per-lane mask to a bit-sliced counter of NB bits.
template <int NB>
__device__ __forceinline__ void bs_add(uint32_t* c, uint32_t v) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const uint32_t carry = c[b] & v;
        c[b] ^= v;
        v = carry;
    }
}

// Add a 3-bit bit-sliced number (m0,m1,m2) into a kVPlanes vertical counter.
__device__ __forceinline__ void vc_add3(uint32_t (&v)[kVPlanes], uint32_t m0, uint32_t m1,
                                        uint32_t m2) {
    uint32_t carry = v[0] & m0;
    v[0] ^= m0;
    {
        const uint32_t t = v[1] ^ m1;
        const uint32_t c = (v[1] & m1) | (t & carry);
        v[1] = t ^ carry;
        carry = c;
    }
    {
        const uint32_t t = v[2] ^ m2;
        const uint32_t c = (v[2] & m2) | (t & carry);
        v[2] = t ^ carry;
        carry = c;
    }
#pragma unroll
    for (int p = 3; p < kVPlanes; ++p) {
        const uint32_t t = v[p] & carry;
        v[p] ^= carry;
        carry = t;
    }
}

// 32x32 bit-matrix transpose across a warp (row = lane).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x) {
    const int lane = threadIdx.x & 31;
    uint32_t m = 0x0000FFFFu;
#pragma unroll
    for (int j = 16; j; j >>= 1, m ^= (m << j)) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
    }
    return x;
}

// Per-lane totals of a warp's vertical counters -> atomics per replica.
__device__ __forceinline__ void vc_flush(uint32_t (&v)[kVPlanes], int32_t* cnt, int w,
                                         int local_states) {
    uint32_t any = 0;
#pragma unroll
    for (int p = 0; p < kVPlanes; ++p) any |= v[p];
    if (!__any_sync(0xffffffffu, any)) return;
    int total = 0;
#pragma unroll
    for (int p = 0; p < kVPlanes; ++p) {
        total += __popc(warp_transpose32(v[p])) << p;
        v[p] = 0;
    }
    const int m = w * 32 + (threadIdx.x & 31);
    if (total && m < local_states) atomicAdd(cnt + m, total);
}

// ---------------------------------------------------- plane engine sweep

// One warp updates the 32 sites of chunk `ch` for the 32 replicas of word w.
template <int NCB, int NQB, int RULE>
__device__ __forceinline__ void plane_chunk(const PlaneArgs& a, const Chunk ch, int w, uint64_t t,
                                            bool count, int lower, uint32_t (&vc)[kVPlanes],
                                            uint32_t (&vq)[kVPlanes], uint32_t k0, uint32_t k1) {
    constexpr int DCM = (1 << NCB) - 1;
    constexpr int DQM = (1 << NQB) - 1;
    constexpr int B = NCB + NQB;
    const int lane = threadIdx.x & 31;
    const PlaneType ty = a.types[ch.type];
    const int dc = ty.dc, dq = ty.dq, deg = dc + dq;
    const bool valid = lane < ch.len;
    const int site = ch.start + lane;
    const int W = a.W;

    uint32_t s = 0;
    uint32_t x[DCM > 0 ? DCM : 1];
    uint32_t y[DQM > 0 ? DQM : 1];
    uint32_t cb[B > 0 ? B : 1];
#pragma unroll
    for (int b = 0; b < (B > 0 ? B : 1); ++b) cb[b] = 0u;
    uint32_t lowx = 0, lowy = 0;  // bit k: neighbour k has a lower colour
    if (valid) {
        s = a.spins[(size_t)site * W + w];
        const int32_t* nb = a.nbr + ch.nbr_base + (size_t)lane * deg;
#pragma unroll
        for (int k = 0; k < DCM; ++k) {
            x[k] = 0u;
            if (k < dc) {
                const int32_t e = __ldg(nb + k);
                const int j = e & 0x7fffffff;
                const uint32_t neg = e < 0 ? 0xffffffffu : 0u;
                x[k] = a.spins[(size_t)j * W + w] ^ neg;  // bit: J_ij s_j = +1
                lowx |= (uint32_t)(j < lower) << k;
                const uint32_t v = RULE == 0 ? ~(s ^ x[k]) : x[k];
                bs_add<NCB>(cb, v);
            }
        }
#pragma unroll
        for (int k = 0; k < DQM; ++k) {
            y[k] = 0u;
            if (k < dq) {
                const int j = __ldg(nb + dc + k);
                y[k] = a.spins[(size_t)j * W + w];
                lowy |= (uint32_t)(j < lower) << k;
                const uint32_t v = RULE == 0 ? ~(s ^ y[k]) : y[k];
                bs_add<NQB>(cb + NCB, v);
            }
        }
    }
    const uint32_t* kpb = a.kp + (size_t)w * a.kpw + ty.kp_off;
    const int ncl = ty.ncl;
    const uint32_t act = valid ? __ldg(a.active + w) : 0u;
    const uint32_t always = mux_tree<B>(cb, kpb + kKPlanes * ncl) & act;
    uint32_t und = act & ~always;
    uint32_t lt = 0;
#pragma unroll 1
    for (int blk = 0; blk < 14; ++blk) {
        if (!__any_sync(0xffffffffu, und)) break;
        const u32x4 r = philox4x32_10(
            u32x4{(uint32_t)site, (uint32_t)t, (uint32_t)(t >> 32), (uint32_t)blk}, k0, k1);
        const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int b = blk * 4 + q;
            if (b < kKPlanes) {
                const uint32_t tb = mux_tree<B>(cb, kpb + b * ncl);
                lt |= und & tb & ~rr[q];
                und &= ~(tb ^ rr[q]);
            }
        }
    }
    const uint32_t take = (always | lt) & act;
    const uint32_t ns = RULE == 0 ? (s ^ take) : ((s & ~act) | take);
    if (valid) a.spins[(size_t)site * W + w] = ns;

    if (count) {
        uint32_t m[3] = {0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < DCM; ++k)
            if (valid && k < dc && ((lowx >> k) & 1u)) bs_add<3>(m, (ns ^ x[k]) & act);
        vc_add3(vc, m[0], m[1], m[2]);
        uint32_t q[3] = {0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < DQM; ++k)
            if (valid && k < dq && ((lowy >> k) & 1u)) bs_add<3>(q, (ns ^ y[k]) & act);
        vc_add3(vq, q[0], q[1], q[2]);
    }
}

template <int RULE>
__device__ __forceinline__ void plane_dispatch(const PlaneArgs& a, const Chunk ch, int ncb, int nqb,
                                               int w, uint64_t t, bool count, int lower,
                                               uint32_t (&vc)[kVPlanes], uint32_t (&vq)[kVPlanes],
                                               uint32_t k0, uint32_t k1) {
#define TG_CASE(C, Q) \
    case (C) * 4 + (Q): plane_chunk<C, Q, RULE>(a, ch, w, t, count, lower, vc, vq, k0, k1); break;
    switch (ncb * 4 + nqb) {
        TG_CASE(0, 0) TG_CASE(0, 1) TG_CASE(0, 2)
        TG_CASE(1, 0) TG_CASE(1, 1) TG_CASE(1, 2)
        TG_CASE(2, 0) TG_CASE(2, 1) TG_CASE(2, 2)
        TG_CASE(3, 0) TG_CASE(3, 1) TG_CASE(3, 2)
        default: break;
    }
#undef TG_CASE
}

template <int RULE>
__global__ void __launch_bounds__(kPlaneThreads, 1)
plane_sweep_kernel(PlaneArgs a, int64_t t0, int n_sweeps) {
    cg::grid_group grid = cg::this_grid();
    const int wpb = blockDim.x >> 5;
    const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
    const int nw = gridDim.x * wpb;  // host guarantees nw % W == 0
    const int w = gw % a.W;
    const uint2 key = a.wkey[w];
    for (int sw = 0; sw < n_sweeps; ++sw) {
        const uint64_t t = (uint64_t)(t0 + sw);
        const bool count = (sw == n_sweeps - 1);
        for (int c = 0; c < a.n_colors; ++c) {
            uint32_t vc[kVPlanes], vq[kVPlanes];
#pragma unroll
            for (int p = 0; p < kVPlanes; ++p) { vc[p] = 0u; vq[p] = 0u; }
            const int c0 = a.chunk_off[c];
            const int items = (a.chunk_off[c + 1] - c0) * a.W;
            const int lower = a.color_start[c];
            int done = 0;
            for (int item = gw; item < items; item += nw) {
                const Chunk ch = a.chunks[c0 + item / a.W];
                const PlaneType& ty = a.types[ch.type];
                plane_dispatch<RULE>(a, ch, ty.ncb, ty.nqb, w, t, count, lower, vc, vq, key.x,
                                     key.y);
                if (count && ++done == 32) {
                    vc_flush(vc, a.cnt_c, w, a.local_states);
                    vc_flush(vq, a.cnt_q, w, a.local_states);
                    done = 0;
                }
            }
            if (count) {
                vc_flush(vc, a.cnt_c, w, a.local_states);
                vc_flush(vq, a.cnt_q, w, a.local_states);
            }
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

template __global__ void plane_sweep_kernel<0>(PlaneArgs, int64_t, int);
template __global__ void plane_sweep_kernel<1>(PlaneArgs, int64_t, int);

void* plane_sweep_fn(int rule) {
    return rule == 0 ? (void*)plane_sweep_kernel<0> : (void*)plane_sweep_kernel<1>;
}

// ----------------------------------------------------- slot engine sweep

__device__ __forceinline__ void slot_update(const SlotArgs& a, int8_t* s, int i, uint64_t u53,
                                            double beta, double two_p) {
    double local = a.h[i];
    const int e0 = a.off[i], e1 = a.off[i + 1];
    for (int e = e0; e < e1; ++e) {
        const double wgt = a.w[e] + (double)a.cm[e] * two_p;
        local += wgt * (double)s[a.nbr[e]];
    }
    const double si = (double)s[i];
    const double u = (double)u53 * 0x1.0p-53;
    if (a.rule == 0) {
        const double de = 2.0 * si * local;
        if (de <= 0.0 || u < exp(-beta * de)) s[i] = (int8_t)-s[i];
    } else {
        const double p = 1.0 / (1.0 + exp(-2.0 * beta * local));
        s[i] = u < p ? (int8_t)1 : (int8_t)-1;
    }
}

__global__ void __launch_bounds__(kSlotThreads)
slot_sweep_kernel(SlotArgs a, int64_t t0, int n_sweeps) {
    extern __shared__ int8_t sm[];
    const int m = blockIdx.x;  // local state
    const int n = a.n;
    int8_t* s = sm;
    int8_t* gs = a.spins + (size_t)m * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = gs[i];
    const int slot = a.state_slot[a.state0 + m];
    const double beta = a.betas[slot / a.J];
    const double two_p = 2.0 * a.pens[slot % a.J];
    const uint64_t key = a.slot_key[slot];
    const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    __syncthreads();
    for (int sw = 0; sw < n_sweeps; ++sw) {
        const uint64_t base = (uint64_t)(t0 + sw) * (uint64_t)n;  // draw index of spin 0
        for (int c = 0; c < a.n_colors; ++c) {
            const int cs = a.color_start[c], ce = a.color_start[c + 1];
            if (ce > cs) {
                const uint64_t q0 = (base + cs) >> 1, q1 = (base + ce - 1) >> 1;
                for (uint64_t q = q0 + threadIdx.x; q <= q1; q += blockDim.x) {
                    const u32x4 o =
                        philox4x32_10(u32x4{(uint32_t)q, (uint32_t)(q >> 32), 0u, 0u}, k0, k1);
                    const int64_t i0 = (int64_t)(2 * q - base);
                    if (i0 >= cs && i0 < ce)
                        slot_update(a, s, (int)i0, ((uint64_t)o.x | ((uint64_t)o.y << 32)) >> 11,
                                    beta, two_p);
                    if (i0 + 1 >= cs && i0 + 1 < ce)
                        slot_update(a, s, (int)i0 + 1,
                                    ((uint64_t)o.z | ((uint64_t)o.w << 32)) >> 11, beta, two_p);
                }
            }
            __syncthreads();
        }
    }
    // f = -sum_{i<j} J s_i s_j - sum h s (ising.cpp:70-77), g = sum (s_a - s_b)^2
    double fl = 0.0, gl = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double si = (double)s[i];
        fl -= a.h[i] * si;
        for (int e = a.off[i]; e < a.off[i + 1]; ++e) {
            const int j = a.nbr[e];
            if (j > i) {
                const double sj = (double)s[j];
                fl -= a.w[e] * si * sj;
                const double d = si - sj;
                gl += (double)a.cm[e] * d * d;
            }
        }
        gs[i] = s[i];
    }
    __shared__ double red_f[kSlotThreads / 32], red_g[kSlotThreads / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        fl += __shfl_xor_sync(0xffffffffu, fl, o);
        gl += __shfl_xor_sync(0xffffffffu, gl, o);
    }
    if ((threadIdx.x & 31) == 0) { red_f[threadIdx.x >> 5] = fl; red_g[threadIdx.x >> 5] = gl; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double F = 0.0, G = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { F += red_f[q]; G += red_g[q]; }
        a.f_loc[m] = F;
        a.g_loc[m] = G;
    }
}

void* slot_sweep_fn() { return (void*)slot_sweep_kernel; }

// ------------------------------------------------------------ swap kernel

__global__ void __launch_bounds__(kSwapThreads) swap_kernel(SwapArgs a, int64_t round,
                                                            uint64_t swap_base, int rec_idx,
                                                            int rec_flags) {
    const int64_t n_att = round_attempts(a.I, a.J, round);
    for (int k = threadIdx.x; k < n_att; k += blockDim.x) {
        int sa, sb, ctr, is_p;
        const int acc = swap_attempt(a.I, a.J, a.betas, a.pens, round, k, a.f_all, a.g_all,
                                     a.slot_state, a.swap_seed, swap_base, sa, sb, ctr, is_p);
        if (acc) {  // pairs are disjoint: no two attempts touch one slot
            const int xa = a.slot_state[sa], xb = a.slot_state[sb];
            a.slot_state[sa] = xb;
            a.slot_state[sb] = xa;
            a.state_slot[xb] = sa;
            a.state_slot[xa] = sb;
            if (is_p) a.acc_p[ctr] += 1; else a.acc_b[ctr] += 1;
        }
    }
    __syncthreads();
    // record (engine.cpp:189-208): the target is grid slot I*J-1
    if (threadIdx.x == 0) {
        TgRecordDev* r = reinterpret_cast<TgRecordDev*>(a.rec) + rec_idx;
        const int tgt = a.slot_state[a.R - 1];
        r->round = round;
        r->f = a.f_all[tgt];
        r->g = a.g_all[tgt];
        r->feasible = a.g_all[tgt] == 0.0 ? 1 : 0;
        r->target_state = tgt;
        r->digest = 0ull;
    }
    if ((rec_flags & 8) && a.rec_acc) {
        const int np = a.I * (a.J > 1 ? a.J - 1 : 0);
        const int nb = (a.I > 1 ? a.I - 1 : 0) * a.J;
        int64_t* dst = a.rec_acc + (size_t)rec_idx * (np + nb);
        for (int k = threadIdx.x; k < np; k += blockDim.x) dst[k] = a.acc_p[k];
        for (int k = threadIdx.x; k < nb; k += blockDim.x) dst[np + k] = a.acc_b[k];
    }
    if (!a.plane) return;
    // Rebuild the threshold planes of this rank's words for the new labels:
    // bit l of plane b of (w, type, class) = bit (52-b) of K(slot(32w+l), type, class).
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    int combos = 0;
    for (int ty = 0; ty < a.n_types; ++ty) combos += a.types[ty].ncl;
    const int total = a.W * combos;
    for (int job = warp; job < total; job += nwarps) {
        const int w = job / combos;
        int c = job % combos, ty = 0;
        while (c >= a.types[ty].ncl) { c -= a.types[ty].ncl; ++ty; }
        const PlaneType pt = a.types[ty];
        const int m = w * 32 + lane;  // local state
        uint64_t K = 0;
        bool live = false;
        if (m < a.local_states) {
            const int slot = a.state_slot[a.state0 + m];
            K = a.ktab[(size_t)slot * a.ktab_row + pt.ktab_off + c];
            live = true;
        }
        uint32_t* dst = a.kp + (size_t)w * a.kpw + pt.kp_off + c;
        for (int b = 0; b < kKPlanes; ++b) {
            const uint32_t word = __ballot_sync(0xffffffffu, live && ((K >> (52 - b)) & 1ull));
            if (lane == 0) dst[b * pt.ncl] = word;
        }
        const uint32_t alw = __ballot_sync(0xffffffffu, live && K >= (1ull << 53));
        if (lane == 0) dst[kKPlanes * pt.ncl] = alw;
    }
}

// -------------------------------------------------------- extract kernel

__global__ void extract_kernel(ExtractArgs e) {
    const int tgt_slot_count = e.all_slots ? e.R : 1;
    const long long total = (long long)tgt_slot_count * e.n;
    uint64_t dsum = 0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const int sl = e.all_slots ? (int)(q / e.n) : e.R - 1;
        const int i = (int)(q % e.n);
        const int m = e.slot_state[sl] - e.state0;  // local index of the state
        int8_t v = 0;
        if (m >= 0 && m < e.local_states) {
            if (e.plane) v = ((e.spins32[(size_t)i * e.W + (m >> 5)] >> (m & 31)) & 1u) ? 1 : -1;
            else v = e.spins8[(size_t)m * e.n + i];
        }
        const int ci = e.perm[i];  // caller index
        if (e.states) e.states[(size_t)(e.all_slots ? sl : 0) * e.n + ci] = v;
        if (!e.all_slots && v > 0) dsum += digest_term((uint64_t)ci);
    }
    if (e.digest) {
#pragma unroll
        for (int o = 16; o; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        if ((threadIdx.x & 31) == 0 && dsum)
            atomicAdd(reinterpret_cast<unsigned long long*>(e.digest), (unsigned long long)dsum);
    }
}

// ------------------------------------------------------------- init kernels

__global__ void plane_init_kernel(uint32_t* spins, int n, int W, int local_states, int state0,
                                  uint64_t seed) {
    const long long total = (long long)n * W;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(q / W), w = (int)(q % W);
        uint32_t word = 0;
        for (int l = 0; l < 32; ++l) {
            const int m = w * 32 + l;
            if (m >= local_states) break;
            const uint64_t key = derive_seed(seed, kPurposeInit, (uint64_t)(state0 + m));
            if (stream_bits(key, (uint64_t)i) >> 63) word |= 1u << l;  // rng.hpp:79
        }
        spins[q] = word;
    }
}

__global__ void slot_init_kernel(int8_t* spins, int n, int local_states, int state0, uint64_t seed) {
    const long long total = (long long)n * local_states;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const int m = (int)(q / n), i = (int)(q % n);
        const uint64_t key = derive_seed(seed, kPurposeInit, (uint64_t)(state0 + m));
        spins[q] = (stream_bits(key, (uint64_t)i) >> 63) ? (int8_t)1 : (int8_t)-1;
    }
}

}  // namespace tg
