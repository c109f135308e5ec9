// kernels.cu -- sm_100a kernels of the 2D-PT hot path.
//
//   (plane_sweep_kernel lives in plane_sweep.cu, one object per update rule)
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
#include "plane_device.cuh"

namespace cg = cooperative_groups;

namespace tg {

void* plane_sweep_fn_r0(int wv);
void* plane_sweep_fn_r1(int wv);
void* plane_sweep_fn(int rule, int wv) { return rule == 0 ? plane_sweep_fn_r0(wv) : plane_sweep_fn_r1(wv); }
void* plane_rounds_fn_r0(int wv, int fast);
void* plane_rounds_fn_r1(int wv, int fast);
void* plane_tpw_fn_r0(int fast);
void* plane_tpw_fn_r1(int fast);
void* plane_tpw_fn(int rule, int fast) { return rule == 0 ? plane_tpw_fn_r0(fast) : plane_tpw_fn_r1(fast); }
__global__ void k_gen_chunks(const __grid_constant__ RunTable rt, Chunk* chunks) {
    const int total = rt.cpref[rt.n];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
        int q = 0;
        while (rt.cpref[q + 1] <= k) ++q;  // runs are few
        const int s0 = rt.start[q] + 32 * (k - rt.cpref[q]);
        chunks[k] = Chunk{s0, min(32, rt.start[q] + rt.cnt[q] - s0), rt.type[q], 0};
    }
}

cudaError_t plane_gen_chunks(const RunTable& rt, Chunk* chunks, cudaStream_t st) {
    const int total = rt.cpref[rt.n];
    if (total > 0) k_gen_chunks<<<(total + 255) / 256, 256, 0, st>>>(rt, chunks);
    return cudaGetLastError();
}

// Per-site padded neighbour table of the tpw config-5 path (one warp per chunk).
__global__ void k_tpw_nbr4(const Chunk* chunks, int n_chunks, TypeDq tdq, const int32_t* nbr, int logW,
                           int4* out) {
    const int lane = threadIdx.x & 31;
    for (int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n_chunks;
         q += gridDim.x * (blockDim.x >> 5)) {
        const Chunk ch = chunks[q];
        if (lane >= ch.len) continue;
        const int dq = tdq.dq[ch.type];
        const int32_t* e = nbr + ch.nbr_base + lane * (3 + dq);
        auto sh = [&](int32_t v) {
            return (int)((((uint32_t)v & 0x7fffffffu) << logW) | ((uint32_t)v & 0x80000000u));
        };
        // bit 31 of the 4th entry: no chain partner
        out[ch.start + lane] = make_int4(sh(e[0]), sh(e[1]), sh(e[2]), dq ? sh(e[3]) : (int)0x80000000u);
    }
}

cudaError_t tpw_build_nbr4(const Chunk* chunks, int n_chunks, TypeDq tdq, const int32_t* nbr, int logW,
                           int4* out, cudaStream_t st) {
    if (n_chunks > 0) k_tpw_nbr4<<<(n_chunks + 7) / 8, 256, 0, st>>>(chunks, n_chunks, tdq, nbr, logW, out);
    return cudaGetLastError();
}

void* plane_tpw_sweep_fn_r0(int fast);
void* plane_tpw_sweep_fn_r1(int fast);
void* plane_tpw_sweep_fn(int rule, int fast) {
    return rule == 0 ? plane_tpw_sweep_fn_r0(fast) : plane_tpw_sweep_fn_r1(fast);
}
void* plane_rounds_fn(int rule, int wv, int fast) {
    return rule == 0 ? plane_rounds_fn_r0(wv, fast) : plane_rounds_fn_r1(wv, fast);
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

// FP32 fast path with a certified fallback: the FP32 local field, exponent and
// uniform carry explicit error bounds (eps_local from the host, ulp terms for
// the products, __expf and the u53 -> float rounding).  When the FP32 decision
// is certain it equals the FP64 decision of slot_update; otherwise (a band of
// relative width ~1e-5 around the threshold) the FP64 path decides.  Results
// are therefore identical to the all-FP64 kernel.
__device__ __forceinline__ void slot_update_fast(const SlotArgs& a, int8_t* s, int i, uint64_t u53,
                                                 double beta, double two_p, float beta32,
                                                 float two_p32) {
    const int e0 = __ldg(a.off + i), e1 = __ldg(a.off + i + 1);
    float l32 = __ldg(a.h32 + i);
    for (int e = e0; e < e1; ++e) {
        const int2 v = __ldg(a.ent + e);
        const float wgt = __int_as_float(v.y) + (float)(v.x >> 28) * two_p32;
        l32 = fmaf(wgt, (float)s[v.x & 0x0fffffff], l32);
    }
    const float si = (float)s[i];
    const float uf = (float)u53 * 0x1.0p-53f;            // rel. error <= 2^-24
    const float eb = 2.0f * a.beta_max * a.eps_local;      // bound on the exponent error from the field
    if (a.rule == 0) {
        const float de32 = 2.0f * si * l32;
        const float tol = 2.0f * a.eps_local;
        if (de32 < -tol) { s[i] = (int8_t)-s[i]; return; }  // de64 <= 0 for sure
        if (de32 > tol) {
            const float x = -beta32 * de32;
            const float T = __expf(x);
            const float band = T * (2.0f * eb + fabsf(x) * 0x1.0p-19f + 0x1.0p-18f) + uf * 0x1.0p-22f;
            if (uf < T - band) { s[i] = (int8_t)-s[i]; return; }
            if (uf > T + band) return;
        }
    } else {
        const float y = 2.0f * beta32 * l32;
        const float p = __frcp_rn(1.0f + __expf(-y));
        const float band = eb + fabsf(y) * 0x1.0p-19f + 0x1.0p-18f + uf * 0x1.0p-22f;
        if (uf < p - band) { s[i] = 1; return; }
        if (uf > p + band) { s[i] = -1; return; }
    }
    slot_update(a, s, i, u53, beta, two_p);  // near the threshold: decide in FP64
}

__global__ void __launch_bounds__(kSlotThreads)
slot_sweep_kernel(SlotArgs a, int64_t t0, int n_sweeps) {
    if (a.rs) t0 = a.rs->round * n_sweeps;
    extern __shared__ int8_t sm[];
    const int m = blockIdx.x;  // local state
    const int n = a.n;
    int8_t* s = sm;
    int8_t* gs = a.spins + (size_t)m * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = gs[i];
    const int slot = a.state_slot[a.state0 + m];
    const double beta = a.betas[slot / a.J];
    const double two_p = 2.0 * a.pens[slot % a.J];
    const float beta32 = (float)beta, two_p32 = (float)two_p;
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
                        slot_update_fast(a, s, (int)i0, ((uint64_t)o.x | ((uint64_t)o.y << 32)) >> 11,
                                         beta, two_p, beta32, two_p32);
                    if (i0 + 1 >= cs && i0 + 1 < ce)
                        slot_update_fast(a, s, (int)i0 + 1,
                                         ((uint64_t)o.z | ((uint64_t)o.w << 32)) >> 11, beta, two_p,
                                         beta32, two_p32);
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

// ---------------------------------------------- slot engine, padded degree

// Fixed-degree variant: every site has D padded entries, so the field and
// energy loops unroll without branches.  Same decisions as slot_update_fast.
template <int D>
__device__ __forceinline__ void slot_update_d(const SlotArgs& a, int8_t* s, int i, uint64_t u53,
                                              double beta, double two_p, float beta32,
                                              float two_p32) {
    const int2* ep = a.entp + (size_t)i * D;
    float l32 = __ldg(a.h32 + i);
#pragma unroll
    for (int k = 0; k < D; k += 2) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(ep + k));
        const float w0 = __int_as_float(v.y) + (float)((v.x >> 28) & 15) * two_p32;
        const float w1 = __int_as_float(v.w) + (float)((v.z >> 28) & 15) * two_p32;
        l32 = fmaf(w0, (float)s[v.x & 0x07ffffff], l32);
        l32 = fmaf(w1, (float)s[v.z & 0x07ffffff], l32);
    }
    const float si = (float)s[i];
    const float uf = (float)u53 * 0x1.0p-53f;
    const float eb = 2.0f * a.beta_max * a.eps_local;
    if (a.rule == 0) {
        const float de32 = 2.0f * si * l32;
        const float tol = 2.0f * a.eps_local;
        if (de32 < -tol) { s[i] = (int8_t)-s[i]; return; }
        if (de32 > tol) {
            const float x = -beta32 * de32;
            const float T = __expf(x);
            const float band = T * (2.0f * eb + fabsf(x) * 0x1.0p-19f + 0x1.0p-18f) + uf * 0x1.0p-22f;
            if (uf < T - band) { s[i] = (int8_t)-s[i]; return; }
            if (uf > T + band) return;
        }
    } else {
        const float y = 2.0f * beta32 * l32;
        const float p = __frcp_rn(1.0f + __expf(-y));
        const float band = eb + fabsf(y) * 0x1.0p-19f + 0x1.0p-18f + uf * 0x1.0p-22f;
        if (uf < p - band) { s[i] = 1; return; }
        if (uf > p + band) { s[i] = -1; return; }
    }
    slot_update(a, s, i, u53, beta, two_p);  // near the threshold: decide in FP64
}

template <int D>
__global__ void __launch_bounds__(kSlotThreads)
slot_sweep_kernel_d(SlotArgs a, int64_t t0, int n_sweeps) {
    if (a.rs) t0 = a.rs->round * n_sweeps;
    extern __shared__ int8_t sm[];
    const int m = blockIdx.x;
    const int n = a.n;
    int8_t* s = sm;
    int8_t* gs = a.spins + (size_t)m * n;
    {   // 16-byte staging of the configuration (rows are 16-byte aligned iff n % 16 == 0)
        const int n16 = (n & 15) ? 0 : (n >> 4);
        for (int q = threadIdx.x; q < n16; q += blockDim.x)
            reinterpret_cast<int4*>(s)[q] = reinterpret_cast<const int4*>(gs)[q];
        for (int i = (n16 << 4) + threadIdx.x; i < n; i += blockDim.x) s[i] = gs[i];
    }
    const int slot = a.state_slot[a.state0 + m];
    const double beta = a.betas[slot / a.J];
    const double two_p = 2.0 * a.pens[slot % a.J];
    const float beta32 = (float)beta, two_p32 = (float)two_p;
    const uint64_t key = a.slot_key[slot];
    const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    __syncthreads();
    for (int sw = 0; sw < n_sweeps; ++sw) {
        const uint64_t base = (uint64_t)(t0 + sw) * (uint64_t)n;
        for (int c = 0; c < a.n_colors; ++c) {
            const int cs = a.color_start[c], ce = a.color_start[c + 1];
            if (ce > cs) {
                const uint64_t q0 = (base + cs) >> 1, q1 = (base + ce - 1) >> 1;
                for (uint64_t q = q0 + threadIdx.x; q <= q1; q += blockDim.x) {
                    const u32x4 o =
                        philox4x32_10(u32x4{(uint32_t)q, (uint32_t)(q >> 32), 0u, 0u}, k0, k1);
                    const int64_t i0 = (int64_t)(2 * q - base);
                    if (i0 >= cs && i0 < ce)
                        slot_update_d<D>(a, s, (int)i0, ((uint64_t)o.x | ((uint64_t)o.y << 32)) >> 11,
                                         beta, two_p, beta32, two_p32);
                    if (i0 + 1 >= cs && i0 + 1 < ce)
                        slot_update_d<D>(a, s, (int)i0 + 1, ((uint64_t)o.z | ((uint64_t)o.w << 32)) >> 11,
                                         beta, two_p, beta32, two_p32);
                }
            }
            __syncthreads();
        }
    }
    // f, g over forward edges (bit 27), FP64 cost weights
    double fl = 0.0, gl = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double si = (double)s[i];
        fl -= a.h[i] * si;
        const int2* ep = a.entp + (size_t)i * D;
        const double* wp = a.wp + (size_t)i * D;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int2 v = __ldg(ep + k);
            const double sj = (double)s[v.x & 0x07ffffff];
            const bool fwd = (v.x >> 27) & 1;
            const double cmf = (double)((v.x >> 28) & 15);
            const double d = si - sj;
            fl -= fwd ? __ldg(wp + k) * si * sj : 0.0;
            gl += fwd ? cmf * d * d : 0.0;
        }
    }
    {
        const int n16 = (n & 15) ? 0 : (n >> 4);
        for (int q = threadIdx.x; q < n16; q += blockDim.x)
            reinterpret_cast<int4*>(gs)[q] = reinterpret_cast<const int4*>(s)[q];
        for (int i = (n16 << 4) + threadIdx.x; i < n; i += blockDim.x) gs[i] = s[i];
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

void* slot_sweep_fn_d(int D) {
    return D == 4 ? (void*)slot_sweep_kernel_d<4> : (D == 8 ? (void*)slot_sweep_kernel_d<8> : nullptr);
}


// ------------------------------------------------------------ swap kernel

__global__ void __launch_bounds__(kSwapThreads) swap_kernel(SwapArgs a, int64_t round,
                                                            uint64_t swap_base, int rec_idx,
                                                            int rec_flags) {
    if (a.rs) {
        round = a.rs->round + 1;
        swap_base = a.rs->swap_base;
        rec_idx = a.rs->filled;
    }
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
    // every thread read the round state before the barrier above: advance it for the
    // kernels that follow (extract_kernel indexes with filled - 1, the next sweep with round)
    if (a.tick && threadIdx.x == 0) {
        a.tick->swap_base = swap_base + (uint64_t)n_att;
        a.tick->round = round;
        a.tick->filled = rec_idx + 1;
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
        uint32_t* dstc = (c == 2 || c == 3) ? a.kpc + ((size_t)w * a.n_types + ty) * 128 + (c - 2) * 64
                                            : nullptr;
        for (int b = 0; b < kKPlanes; ++b) {
            const uint32_t word = __ballot_sync(0xffffffffu, live && ((K >> (52 - b)) & 1ull));
            if (lane == 0) {
                dst[b * pt.ncl] = word;
                if (dstc) dstc[b] = word;
            }
        }
        const uint32_t alw = __ballot_sync(0xffffffffu, live && K >= (1ull << 53));
        if (lane == 0) dst[kKPlanes * pt.ncl] = alw;
    }
}

// Threshold planes of this rank's words for the current labels, one warp per
// (word, type, class) job over the whole grid (the unfused round loop runs it
// after swap_kernel, which then skips its own single-block rebuild).  Plane b
// holds bit 52 - b of the lanes' 53-bit thresholds: two 32x32 transposes
// (plane_round.cuh) instead of 53 ballots.
__global__ void __launch_bounds__(256) plane_rebuild_kernel(SwapArgs a) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nw = gridDim.x * (blockDim.x >> 5);
    int combos = 0;
    for (int ty = 0; ty < a.n_types; ++ty) combos += a.types[ty].ncl;
    const int total = a.W * combos;
    for (int job = gw; job < total; job += nw) {
        const int w = job / combos;
        int c = job % combos, ty = 0;
        while (c >= a.types[ty].ncl) { c -= a.types[ty].ncl; ++ty; }
        const PlaneType pt = a.types[ty];
        const int m = w * 32 + lane;  // local state
        uint64_t K = 0;
        const bool live = m < a.local_states;
        if (live) K = a.ktab[(size_t)a.state_slot[a.state0 + m] * a.ktab_row + pt.ktab_off + c];
        uint32_t* dst = a.kp + (size_t)w * a.kpw + pt.kp_off + c;
        uint32_t* dstc = (c == 2 || c == 3) ? a.kpc + ((size_t)w * a.n_types + ty) * 128 + (c - 2) * 64
                                            : nullptr;
        const uint32_t th = warp_transpose32((uint32_t)(K >> 21));
        const uint32_t tl = warp_transpose32((uint32_t)(K << 11));
        const int bh = 31 - lane, bl = 63 - lane;
        dst[bh * pt.ncl] = th;
        if (dstc) dstc[bh] = th;
        if (lane >= 11) {
            dst[bl * pt.ncl] = tl;
            if (dstc) dstc[bl] = tl;
        }
        const uint32_t alw = __ballot_sync(0xffffffffu, live && K >= (1ull << 53));
        if (lane == 0) dst[kKPlanes * pt.ncl] = alw;
    }
}

// -------------------------------------------------------- extract kernel

// Advance the device round counters after a round of the unfused loop.
__global__ void round_tick_kernel(RoundState* rs, int I, int J) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const int64_t round = rs->round + 1;
        rs->swap_base += (uint64_t)round_attempts(I, J, round);
        rs->round = round;
        rs->filled += 1;
    }
}

__global__ void extract_kernel(ExtractArgs e) {
    if (e.rs) {  // this round's slot of the chunk's state ring and digest array
        const int k = e.rs->filled - e.rs_back;  // rs_back: swap_kernel already advanced the round state
        if (e.states) e.states += (size_t)k * e.per_state;
        if (e.digest) e.digest += k;
    }
    const int tgt_slot_count = e.all_slots ? e.R : 1;
    const long long total = (long long)tgt_slot_count * e.n;
    uint64_t dsum = 0;
    if (!e.all_slots) {
        // the target slot only (every round of a traced run): one label lookup, 32-bit
        // indexing, four independent gathers in flight per thread
        const int m = e.slot_state[e.R - 1] - e.state0;
        const bool here = m >= 0 && m < e.local_states;
        const int stride = gridDim.x * blockDim.x;
        for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < e.n; i0 += 4 * stride) {
            int8_t v[4] = {0, 0, 0, 0};
            int ci[4] = {0, 0, 0, 0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * stride;
                if (i >= e.n) continue;
                if (here) {
                    if (e.plane) v[u] = ((e.spins32[(size_t)i * e.W + (m >> 5)] >> (m & 31)) & 1u) ? 1 : -1;
                    else v[u] = e.spins8[(size_t)m * e.n + i];
                }
                ci[u] = e.perm[i];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (i0 + u * stride >= e.n) continue;
                if (e.states) e.states[ci[u]] = v[u];
                if (v[u] > 0) dsum += digest_term((uint64_t)ci[u]);
            }
        }
    } else
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
        if (sl == e.R - 1 && v > 0) dsum += digest_term((uint64_t)ci);  // the target slot's digest
    }
    if (e.digest) {
#pragma unroll
        for (int o = 16; o; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        if ((threadIdx.x & 31) == 0 && dsum)
            atomicAdd(reinterpret_cast<unsigned long long*>(e.digest), (unsigned long long)dsum);
    }
}

// ------------------------------------------------------------- init kernels

// random_state (ising.cpp:15-19) of every local replica, bit-packed: one warp
// per (site pair, word); lane l is replica 32 w + l, whose init stream gives
// the draws of sites 2p and 2p+1 from ONE Philox block (rng.hpp:79: the spin
// is the top bit), and two ballots pack the 32 replicas into the words.
__global__ void plane_init_kernel(uint32_t* spins, int n, int W, int local_states, int state0,
                                  uint64_t seed) {
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int npairs = (n + 1) >> 1;
    // a warp keeps one word (its lanes' init keys, key schedule in registers)
    // when the warp count allows: then p advances by nw / W with no division
    const bool fixed_w = nw % W == 0;
    const int items = npairs * W;  // <= 2^19 * 32
    int w = gw % W;
    uint32_t ks[20];
    philox_key_schedule(derive_seed(seed, kPurposeInit, (uint64_t)(state0 + w * 32 + lane)), ks);
    const int dp = nw / W;
    int p = gw / W;
    if (fixed_w) {
        // two independent site pairs per iteration (two Philox blocks in flight)
        const bool live = w * 32 + lane < local_states;
        for (int it = gw; it < items; it += 2 * nw, p += 2 * dp) {
            const bool two = it + nw < items;
            const u32x4 o = philox4x32_10_ks(u32x4{(uint32_t)p, 0u, 0u, 0u}, ks);
            const u32x4 o2 = philox4x32_10_ks(u32x4{(uint32_t)(p + dp), 0u, 0u, 0u}, ks);
            const uint32_t w0 = __ballot_sync(0xffffffffu, live && (o.y >> 31));   // draw 2p
            const uint32_t w1 = __ballot_sync(0xffffffffu, live && (o.w >> 31));   // draw 2p + 1
            const uint32_t w2 = __ballot_sync(0xffffffffu, live && (o2.y >> 31));
            const uint32_t w3 = __ballot_sync(0xffffffffu, live && (o2.w >> 31));
            if (lane == 0) {
                spins[(size_t)(2 * p) * W + w] = w0;
                if (2 * p + 1 < n) spins[(size_t)(2 * p + 1) * W + w] = w1;
                if (two) {
                    const int q = p + dp;
                    spins[(size_t)(2 * q) * W + w] = w2;
                    if (2 * q + 1 < n) spins[(size_t)(2 * q + 1) * W + w] = w3;
                }
            }
        }
        return;
    }
    for (int it = gw; it < items; it += nw) {
        w = it % W;
        p = it / W;
        philox_key_schedule(derive_seed(seed, kPurposeInit, (uint64_t)(state0 + w * 32 + lane)), ks);
        const u32x4 o = philox4x32_10_ks(u32x4{(uint32_t)p, 0u, 0u, 0u}, ks);
        const bool live = w * 32 + lane < local_states;
        const uint32_t w0 = __ballot_sync(0xffffffffu, live && (o.y >> 31));  // draw 2p
        const uint32_t w1 = __ballot_sync(0xffffffffu, live && (o.w >> 31));  // draw 2p + 1
        if (lane == 0) {
            spins[(size_t)(2 * p) * W + w] = w0;
            if (2 * p + 1 < n) spins[(size_t)(2 * p + 1) * W + w] = w1;
        }
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
