// slot_engine.cu -- SLOT engine v2: replica-fastest int8 layout, batched
// instances, cooperative persistent sweep kernel.
//
// Restates metropolis_sweep (/root/reference/proj/src/mc.cpp:21-35) with the
// reference's per-slot RNG association (engine.cpp:98-107): the update of
// spin i in sweep t of the replica at grid slot r draws output t*N+i of
// stream(derive_seed(seed, replica, r)).  Layout spins[b][site][Rp] (Rp = I*J
// rounded up to 32): a warp updates one site of one instance for 32
// replicas, so the site's neighbour list is a warp-uniform broadcast load and
// each neighbour gather is one coalesced 32-byte sector.  Any number of
// independent instances (config 3's batch) share one launch; every instance
// keeps its own structure, schedule, seed, labels, counters and records, so a
// batch equals independent run_2dpt calls instance by instance.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tg {

__device__ __forceinline__ int find_instance(const int* pref, int B, int item) {
    int lo = 0, hi = B;  // pref[lo] <= item < pref[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pref[mid] <= item) lo = mid; else hi = mid;
    }
    return lo;
}

// FP64 decision (the semantics all fast paths must reproduce): local field
// in the reference's merged-CSR order (constraints.cpp:122-140, ising.cpp:79-88).
__device__ __forceinline__ int8_t s2_exact(const S2Args& a, const SInst& in, const int8_t* sp, int i,
                                           int r, int8_t si8, uint64_t u53, double beta,
                                           double two_p) {
    double local = a.h[in.h_off + i];
    const int e0 = a.off[in.csr_off + i], e1 = a.off[in.csr_off + i + 1];
    for (int e = e0; e < e1; ++e) {
        const int q = in.nbr_off + e;
        const double wgt = a.w[q] + (double)a.cm[q] * two_p;
        local += wgt * (double)sp[(size_t)a.nbr[q] * a.Rp + r];
    }
    const double si = (double)si8;
    const double u = (double)u53 * 0x1.0p-53;
    if (a.rule == 0) {
        const double de = 2.0 * si * local;
        return (de <= 0.0 || u < exp(-beta * de)) ? (int8_t)-si8 : si8;
    }
    const double p = 1.0 / (1.0 + exp(-2.0 * beta * local));
    return u < p ? (int8_t)1 : (int8_t)-1;
}

// One update of spin i for replica r: certified FP32 decision with FP64
// fallback (error bounds as in kernels.cu slot_update_fast).  Returns the new
// spin; on the counting sweep adds the bonds to lower-colour neighbours to
// (fl, gl) (each edge once, at its higher-colour endpoint).
template <int D>
__device__ __forceinline__ void s2_update(const S2Args& a, const SInst& in, int8_t* sp, int i, int r,
                                          uint64_t u53, double beta, double two_p, float beta32,
                                          float two_p32, bool count, int lower, double& fl,
                                          double& gl) {
    const int2* ep = a.entp + in.entp_off + i * D;
    const unsigned Rp = (unsigned)a.Rp;
    int4 v[D / 2];
#pragma unroll
    for (int k = 0; k < D / 2; ++k) v[k] = __ldg(reinterpret_cast<const int4*>(ep) + k);
    int8_t sn[D];
#pragma unroll
    for (int k = 0; k < D / 2; ++k) {
        sn[2 * k] = sp[(unsigned)(v[k].x & 0x07ffffff) * Rp + r];
        sn[2 * k + 1] = sp[(unsigned)(v[k].z & 0x07ffffff) * Rp + r];
    }
    float l32 = __ldg(a.h32 + in.h_off + i);
#pragma unroll
    for (int k = 0; k < D / 2; ++k) {
        const float w0 = __int_as_float(v[k].y) + (float)((v[k].x >> 28) & 15) * two_p32;
        const float w1 = __int_as_float(v[k].w) + (float)((v[k].z >> 28) & 15) * two_p32;
        l32 = fmaf(w0, (float)sn[2 * k], l32);
        l32 = fmaf(w1, (float)sn[2 * k + 1], l32);
    }
    int8_t* cell = sp + (unsigned)i * Rp + r;
    const int8_t si8 = *cell;
    const float si = (float)si8;
    const float uf = (float)u53 * 0x1.0p-53f;
    const float eb = 2.0f * in.beta_max * in.eps;
    int decided = 0;  // 1: take, -1: keep / set -1, 2: set +1 (heat bath)
    int8_t nv = si8;
    if (a.rule == 0) {
        const float de32 = 2.0f * si * l32;
        const float tol = 2.0f * in.eps;
        if (de32 < -tol) { nv = (int8_t)-si8; decided = 1; }
        else if (de32 > tol) {
            const float x = -beta32 * de32;
            const float T = __expf(x);
            const float band = T * (2.0f * eb + fabsf(x) * 0x1.0p-19f + 0x1.0p-18f) + uf * 0x1.0p-22f;
            if (uf < T - band) { nv = (int8_t)-si8; decided = 1; }
            else if (uf > T + band) decided = 1;
        }
    } else {
        const float y = 2.0f * beta32 * l32;
        const float p = __frcp_rn(1.0f + __expf(-y));
        const float band = eb + fabsf(y) * 0x1.0p-19f + 0x1.0p-18f + uf * 0x1.0p-22f;
        if (uf < p - band) { nv = 1; decided = 1; }
        else if (uf > p + band) { nv = -1; decided = 1; }
    }
    if (!decided) nv = s2_exact(a, in, sp, i, r, si8, u53, beta, two_p);
    if (nv != si8) *cell = nv;
    if (count) {
        const double sv = (double)nv;
        fl -= a.h[in.h_off + i] * sv;
        const double* wp = a.wp + in.entp_off + i * D;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int x = (k & 1) ? v[k >> 1].z : v[k >> 1].x;
            const int j = x & 0x07ffffff;
            if (j < lower) {
                const double sj = (double)sn[k];
                fl -= __ldg(wp + k) * sv * sj;
                const double d = sv - sj;
                gl += (double)((x >> 28) & 15) * d * d;
            }
        }
    }
}

// Fixed-order reduction of the per-warp energy partials into out_f/out_g
// [B*R] (one warp per replica, lanes take strided partials, then a fixed
// shuffle tree); clears the partials for the next sweep.
__device__ __forceinline__ void s2_reduce(const S2Args& a, int gw, int lane, int nsub, double* out_f,
                                          double* out_g) {
    for (int idx = gw; idx < a.B * a.R; idx += gridDim.x * (blockDim.x >> 5)) {
        const int b = idx / a.R, rr = idx % a.R;
        double F = 0.0, G = 0.0;
        for (int q = lane; q < nsub; q += 32) {
            double* pf = a.part_f + ((size_t)b * nsub + q) * a.Rp + rr;
            double* pg = a.part_g + ((size_t)b * nsub + q) * a.Rp + rr;
            F += *pf;
            G += *pg;
            *pf = 0.0;
            *pg = 0.0;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            F += __shfl_xor_sync(0xffffffffu, F, o);
            G += __shfl_xor_sync(0xffffffffu, G, o);
        }
        if (lane == 0) {
            out_f[idx] = F;
            out_g[idx] = G;
        }
    }
}

// Persistent cooperative kernel: the sweeps of one round for every instance
// of the batch.  Each warp keeps one replica group (its lanes = replicas
// 32*gi .. 32*gi+31 of every instance), so a lane's slot label, beta, 2P and
// stream key are loaded once per instance instead of per update.
template <int D, bool HIST>
__global__ void __launch_bounds__(kSlot2Threads, 2)
slot2_sweep_kernel(const __grid_constant__ S2Args a, int64_t t0, int n_sweeps, int do_energy) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
    const int gi = gw % a.G;           // replica group of this warp (host: warps % G == 0)
    const int sw = gw / a.G, nsub = a.nsub;
    const int r = gi * 32 + lane;
    const bool live = r < a.R;
    for (int swp = 0; swp < n_sweeps; ++swp) {
        const uint64_t t = (uint64_t)(t0 + swp);
        const bool hist = HIST && (int64_t)t >= a.hist_t0;
        const bool count = (do_energy && swp == n_sweeps - 1) || hist;
        int cur_b = -1;
        double beta = 0.0, two_p = 0.0;
        uint64_t key = 0;
        double fl = 0.0, gl = 0.0;
        for (int c = 0; c < a.max_colors; ++c) {
            const int* pref = a.item_pref + (size_t)c * (a.B + 1);
            const int total = pref[a.B];
            // items rise monotonically: advance the instance instead of searching
            int b = sw < total ? find_instance(pref, a.B, sw) : 0;
            int b_end = pref[b + 1];
            for (int item = sw; item < total; item += nsub) {
                while (item >= b_end) b_end = pref[++b + 1];
                const SInst& in = a.inst[b];
                if (b != cur_b) {
                    if (count && cur_b >= 0) {  // flush the previous instance's partial sums
                        a.part_f[((size_t)cur_b * nsub + sw) * a.Rp + r] += fl;
                        a.part_g[((size_t)cur_b * nsub + sw) * a.Rp + r] += gl;
                        fl = 0.0; gl = 0.0;
                    }
                    cur_b = b;
                    beta = a.sbeta[(size_t)b * a.Rp + r];
                    two_p = a.stwop[(size_t)b * a.Rp + r];
                    key = a.skey[(size_t)b * a.Rp + r];
                }
                if (c >= in.n_colors) continue;
                const int cs = a.color_start[in.color_off + c], ce = a.color_start[in.color_off + c + 1];
                if (ce <= cs) continue;
                const uint64_t base = t * (uint64_t)in.n;
                const uint64_t q = ((base + cs) >> 1) + (uint64_t)(item - pref[b]);
                if (q > ((base + ce - 1) >> 1) || !live) continue;
                const u32x4 o = philox4x32_10(u32x4{(uint32_t)q, (uint32_t)(q >> 32), 0u, 0u},
                                              (uint32_t)key, (uint32_t)(key >> 32));
                int8_t* sp = a.spins + in.spin_off;
                const int64_t i0 = (int64_t)(2 * q - base);
                if (i0 >= cs && i0 < ce)
                    s2_update<D>(a, in, sp, (int)i0, r, ((uint64_t)o.x | ((uint64_t)o.y << 32)) >> 11,
                                 beta, two_p, (float)beta, (float)two_p, count, cs, fl, gl);
                if (i0 + 1 >= cs && i0 + 1 < ce)
                    s2_update<D>(a, in, sp, (int)i0 + 1, r, ((uint64_t)o.z | ((uint64_t)o.w << 32)) >> 11,
                                 beta, two_p, (float)beta, (float)two_p, count, cs, fl, gl);
            }
            grid.sync();
        }
        if (count && cur_b >= 0) {
            a.part_f[((size_t)cur_b * nsub + sw) * a.Rp + r] += fl;
            a.part_g[((size_t)cur_b * nsub + sw) * a.Rp + r] += gl;
        }
        if (HIST && hist) {  // probe: this sweep's (f, g) of every replica into the history
            grid.sync();
            const size_t row = (size_t)((int64_t)t - a.hist_t0) * a.B * a.R;
            s2_reduce(a, gw, lane, nsub, a.hist_f + row, a.hist_g + row);
            grid.sync();
        }
    }
    if (!do_energy) return;
    grid.sync();
    s2_reduce(a, gw, lane, nsub, a.f, a.g);
}

template __global__ void slot2_sweep_kernel<4, false>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slot2_sweep_kernel<8, false>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slot2_sweep_kernel<16, false>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slot2_sweep_kernel<4, true>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slot2_sweep_kernel<8, true>(const __grid_constant__ S2Args, int64_t, int, int);
template __global__ void slot2_sweep_kernel<16, true>(const __grid_constant__ S2Args, int64_t, int, int);

// hist = the probe variant (per-sweep energies into a history)
void* slot2_sweep_fn(int D, bool hist) {
    if (hist)
        return D <= 4 ? (void*)slot2_sweep_kernel<4, true>
                      : (D <= 8 ? (void*)slot2_sweep_kernel<8, true> : (void*)slot2_sweep_kernel<16, true>);
    return D <= 4 ? (void*)slot2_sweep_kernel<4, false>
                  : (D <= 8 ? (void*)slot2_sweep_kernel<8, false> : (void*)slot2_sweep_kernel<16, false>);
}

// One block per instance: that instance's swap phase, record and counters.
__global__ void __launch_bounds__(kSwapThreads)
slot2_swap_kernel(const __grid_constant__ S2Swap s, int64_t round, uint64_t swap_base, int rec_idx,
                  int rec_flags) {
    const int b = blockIdx.x;
    const int R = s.R, I = s.I, J = s.J;
    const int np = I * (J > 1 ? J - 1 : 0), nb = (I > 1 ? I - 1 : 0) * J;
    int32_t* slot_state = s.slot_state + b * R;
    int32_t* state_slot = s.state_slot + b * R;
    const double* f = s.f + b * R;
    const double* g = s.g + b * R;
    int64_t* acc_p = s.acc_p + (size_t)b * np;
    int64_t* acc_b = s.acc_b + (size_t)b * nb;
    const int64_t n_att = round_attempts(I, J, round);
    for (int k = threadIdx.x; k < n_att; k += blockDim.x) {
        int sa, sb, ctr, is_p;
        if (swap_attempt(I, J, s.betas + b * I, s.pens + b * J, round, k, f, g, slot_state,
                         s.swap_seed[b], swap_base, sa, sb, ctr, is_p)) {
            const int xa = slot_state[sa], xb = slot_state[sb];
            slot_state[sa] = xb;
            slot_state[sb] = xa;
            state_slot[xb] = sa;
            state_slot[xa] = sb;
            if (is_p) acc_p[ctr] += 1; else acc_b[ctr] += 1;
        }
    }
    __syncthreads();
    for (int m = threadIdx.x; m < R; m += blockDim.x) {  // label tables of each physical replica
        const int sl = state_slot[m];
        s.sbeta[(size_t)b * s.Rp + m] = s.betas[b * I + sl / J];
        s.stwop[(size_t)b * s.Rp + m] = 2.0 * s.pens[b * J + sl % J];
        s.skey[(size_t)b * s.Rp + m] = s.slot_key[(size_t)b * R + sl];
        if (s.lab)  // FLOAT engine: FP32 (beta, 2P) of the slot
            s.lab[(size_t)b * s.Rp + m] = make_float2((float)s.betas[b * I + sl / J],
                                                      (float)(2.0 * s.pens[b * J + sl % J]));
    }
    if (threadIdx.x == 0) {
        TgRecordDev* rec = reinterpret_cast<TgRecordDev*>(s.rec) + (size_t)b * s.rec_cap + rec_idx;
        const int tgt = slot_state[R - 1];
        rec->round = round;
        rec->f = f[tgt];
        rec->g = g[tgt];
        rec->feasible = g[tgt] == 0.0 ? 1 : 0;
        rec->target_state = tgt;
        rec->digest = 0ull;
    }
    if ((rec_flags & 8) && s.rec_acc) {
        int64_t* dst = s.rec_acc + ((size_t)b * s.rec_cap + rec_idx) * (np + nb);
        for (int k = threadIdx.x; k < np; k += blockDim.x) dst[k] = acc_p[k];
        for (int k = threadIdx.x; k < nb; k += blockDim.x) dst[np + k] = acc_b[k];
    }
}

// Target-state digest / snapshot (or every slot) per instance, caller order.
__global__ void slot2_extract_kernel(const __grid_constant__ S2Args a, const __grid_constant__ S2Swap s,
                                     int rec_idx, int all_slots) {
    const int b = blockIdx.y;
    const SInst& in = a.inst[b];
    const int slots = all_slots ? a.R : 1;
    const long long total = (long long)slots * in.n;
    uint64_t dsum = 0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const int sl = all_slots ? (int)(q / in.n) : a.R - 1;
        const int i = (int)(q % in.n);
        const int m = s.slot_state[b * a.R + sl];
        const int8_t v = a.spins[in.spin_off + (size_t)i * a.Rp + m];
        const int ci = s.perm[in.h_off + i];
        if (s.rec_states) {
            int8_t* dst = s.rec_states + (size_t)in.state_off * slots * s.rec_cap +
                          (size_t)rec_idx * in.n * slots;
            dst[(size_t)(all_slots ? sl : 0) * in.n + ci] = v;
        }
        if (!all_slots && v > 0) dsum += digest_term((uint64_t)ci);
    }
    if (s.rec && !all_slots) {
#pragma unroll
        for (int o = 16; o; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        if ((threadIdx.x & 31) == 0 && dsum) {
            TgRecordDev* rec = reinterpret_cast<TgRecordDev*>(s.rec) + (size_t)b * s.rec_cap + rec_idx;
            atomicAdd(reinterpret_cast<unsigned long long*>(&rec->digest), (unsigned long long)dsum);
        }
    }
}

__global__ void slot2_init_kernel(const __grid_constant__ S2Args a, const uint64_t* init_keys) {
    const int b = blockIdx.y;
    const SInst& in = a.inst[b];
    const long long total = (long long)in.n * a.Rp;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(q / a.Rp), m = (int)(q % a.Rp);
        int8_t v = 1;
        if (m < a.R) {  // random_state with replica m's init stream (engine.cpp:100-101,
                        // schedule.cpp:30-31 for probes), draw i
            const uint64_t key = init_keys[(size_t)b * a.R + m];
            v = (stream_bits(key, (uint64_t)i) >> 63) ? (int8_t)1 : (int8_t)-1;
        }
        a.spins[in.spin_off + q] = v;
    }
}

}  // namespace tg

namespace tg {

// One block per instance, after the round's swaps: decode the target replica
// (decode, constraints.cpp:149-160: majority over each logical spin's copies,
// ties to the first copy, infeasible when chain-adjacent copies differ), add it
// to the instance's histogram (kl_curve, analysis.cpp:224-226) and evaluate
// kl_divergence (oracle.cpp:178-195) of the accumulated histogram -- every
// histogram bin in parallel, combined in a fixed tree order.
__global__ void __launch_bounds__(1024)
slot2_kl_kernel(const __grid_constant__ S2Args a, const int32_t* slot_state,
                const __grid_constant__ KLArgs k, int64_t round) {
    __shared__ unsigned s_enc;
    __shared__ int s_feas;
    __shared__ double s_red[32];
    const int b = blockIdx.x;
    const SInst& in = a.inst[b];
    const int tgt = slot_state[(size_t)b * a.R + a.R - 1];
    const int8_t* sp = a.spins + in.spin_off;
    if (threadIdx.x == 0) { s_enc = 0u; s_feas = 1; }
    __syncthreads();
    const int* map = k.map + (size_t)b * k.ncopies;
    for (int u = threadIdx.x; u < k.n_logical; u += blockDim.x) {
        const int q0 = k.map_off[u], q1 = k.map_off[u + 1];
        int sum = 0, feas = 1;
        int8_t prev = 0;
        for (int q = q0; q < q1; ++q) {
            const int8_t v = sp[(size_t)map[q] * a.Rp + tgt];
            sum += v;
            if (q > q0 && v != prev) feas = 0;
            prev = v;
        }
        const int8_t first = sp[(size_t)map[q0] * a.Rp + tgt];
        const int bit = sum != 0 ? (sum > 0) : (first > 0);
        if (bit) atomicOr(&s_enc, 1u << u);
        if (!feas) s_feas = 0;
    }
    __syncthreads();
    uint32_t* hist = k.hist + (size_t)b * k.K;
    if (threadIdx.x == 0 && (s_feas || !k.discard)) {
        hist[s_enc] += 1u;
        k.total[b] += 1ull;
    }
    __syncthreads();
    const unsigned long long T = k.total[b];
    double acc = 0.0;
    if (T > 0) {
        const double inv_t = (double)T;
        for (int e = threadIdx.x; e < k.K; e += blockDim.x) {
            const uint32_t c = hist[e];
            if (!c) continue;
            const double ph = (double)c / inv_t;
            const double pe = k.p[e];
            if (pe <= 0.0) { atomicExch(k.error, 1); continue; }
            acc += ph * log(ph / pe);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0 && round >= 1 && round <= k.cap) {
            k.kl[(size_t)b * k.cap + round - 1] = T > 0 ? v : __longlong_as_double(0x7ff8000000000000ll);
            k.samples[(size_t)b * k.cap + round - 1] = (int64_t)T;
        }
    }
}

// Per-replica (f, g) after a round's sweeps, as a separate deterministic pass
// (used when the fused per-warp partials of the sweep kernel would not fit:
// large batches).  Stage 1: block (slice s, replica group g, instance b), 8
// warps; warp w sums sites s_lo + w, s_lo + w + 8, ... of the slice in order
// (field term, and every edge at its higher-index endpoint), the 8 warp sums
// are combined in warp order.  Stage 2 adds the slices in order.
__global__ void __launch_bounds__(256)
slot2_energy_kernel(const __grid_constant__ S2Args a, int n_slices, double* part) {
    __shared__ double sf[8][32], sg[8][32];
    const int b = blockIdx.z, g = blockIdx.y, sl = blockIdx.x;
    const SInst& in = a.inst[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = g * 32 + lane;
    const int per = (in.n + n_slices - 1) / n_slices;
    const int lo = sl * per, hi = min(in.n, lo + per);
    const int8_t* sp = a.spins + in.spin_off;
    const int D = in.D;
    double fl = 0.0, gl = 0.0;
    if (r < a.R) {
        for (int i = lo + warp; i < hi; i += 8) {
            const double sv = (double)sp[(size_t)i * a.Rp + r];
            fl -= a.h[in.h_off + i] * sv;
            const int2* ep = a.entp + in.entp_off + (size_t)i * D;
            const double* wp = a.wp + in.entp_off + (size_t)i * D;
            for (int k = 0; k < D; ++k) {
                const int x = __ldg(&ep[k].x);
                const int j = x & 0x07ffffff;
                if (j < i) {
                    const double sj = (double)sp[(size_t)j * a.Rp + r];
                    fl -= __ldg(wp + k) * sv * sj;
                    const double d = sv - sj;
                    gl += (double)((x >> 28) & 15) * d * d;
                }
            }
        }
    }
    sf[warp][lane] = fl;
    sg[warp][lane] = gl;
    __syncthreads();
    if (warp == 0 && r < a.R) {
        double F = 0.0, G = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) { F += sf[w][lane]; G += sg[w][lane]; }
        const size_t o = ((size_t)b * n_slices + sl) * a.R + r;
        part[2 * o] = F;
        part[2 * o + 1] = G;
    }
}

__global__ void slot2_energy_sum_kernel(const __grid_constant__ S2Args a, int n_slices, const double* part) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= a.B * a.R) return;
    const int b = idx / a.R, r = idx % a.R;
    double F = 0.0, G = 0.0;
    for (int sl = 0; sl < n_slices; ++sl) {
        const size_t o = ((size_t)b * n_slices + sl) * a.R + r;
        F += part[2 * o];
        G += part[2 * o + 1];
    }
    a.f[idx] = F;
    a.g[idx] = G;
}

// Probe moments (schedule.cpp:34-51): the four pooled sums over the history in
// the reference's order (chain-major, then sweep), one thread per sum, with
// unfused FP64 arithmetic as on the host.
__global__ void probe_moments_kernel(const double* hist_f, const double* hist_g, int R, int kept,
                                     double penalty, double* out) {
    const int k = threadIdx.x;
    if (k >= 4) return;
    double acc = 0.0;
    for (int c = 0; c < R; ++c)
        for (int s = 0; s < kept; ++s) {
            const double f = hist_f[(size_t)s * R + c], g = hist_g[(size_t)s * R + c];
            const double e = __dadd_rn(f, __dmul_rn(penalty, g));
            const double x = k == 0 ? e : (k == 1 ? __dmul_rn(e, e) : (k == 2 ? g : __dmul_rn(g, g)));
            acc = __dadd_rn(acc, x);
        }
    out[k] = acc;
}

}  // namespace tg
