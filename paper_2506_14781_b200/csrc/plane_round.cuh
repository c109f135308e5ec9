// plane_round.cuh -- the device-side round epilogue of the fused PLANE
// kernels (plane_sweep.cu, plane_tpw.cu): per-replica (f, g) from the
// unsatisfied-bond counts, the swap phase replayed identically by every
// block on its shared-memory labels (engine.cpp:148-187), counters, the trace
// record (engine.cpp:189-208), the threshold planes of the new labels and the
// optional target-state digest / snapshot.
#pragma once

#include <cooperative_groups.h>

#include "engine.cuh"
#include "kernels.cuh"
#include "plane_device.cuh"

namespace tg {

struct RoundSmem {
    double* f;
    double* g;
    int32_t* slot;
    int32_t* state;
};

// Bytes of the label/energy block at the start of dynamic shared memory.
__host__ __device__ inline size_t round_smem_bytes(int R) {
    return (size_t)R * (2 * sizeof(double) + 2 * sizeof(int32_t)) + 8;
}

__device__ __forceinline__ RoundSmem round_smem(void* base, int R) {
    RoundSmem s;
    s.f = reinterpret_cast<double*>(base);
    s.g = s.f + R;
    s.slot = reinterpret_cast<int32_t*>(s.g + R);
    s.state = s.slot + R;
    return s;
}

__device__ __forceinline__ void round_load_labels(const RoundArgs& r, RoundSmem s) {
    for (int m = threadIdx.x; m < r.R; m += blockDim.x) {
        s.slot[m] = r.slot_state[m];
        s.state[m] = r.state_slot[m];
    }
}

// Everything after the sweeps of round `round` (k-th of this launch).  The
// caller's grid barrier after the last colour phase makes cc/cq final; this
// function ends with the round's closing grid barrier.  n_work: entries of
// r.work per parity (dynamic chunk counters), zeroed for the next round.
__device__ __forceinline__ void round_epilogue(const PlaneArgs& a, const RoundArgs& r, RoundSmem s,
                                               int k, int64_t round, const int32_t* cc,
                                               const int32_t* cq, uint64_t& swap_base, int n_work) {
    namespace cg = cooperative_groups;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int wpb = blockDim.x >> 5;
    const int gw = blockIdx.x * wpb + (tid >> 5);
    const int nw = gridDim.x * wpb;
    const int par = (int)(round & 1);
    const int np = r.I * (r.J > 1 ? r.J - 1 : 0);
    const int nb = (r.I > 1 ? r.I - 1 : 0) * r.J;
    // (f, g) of every replica, reference units: f = -(m - 2 u_c), g = 4 u_q
    for (int m = tid; m < r.R; m += blockDim.x) {
        s.f[m] = -((double)a.m_cost - 2.0 * (double)cc[m]);
        s.g[m] = 4.0 * (double)cq[m];
    }
    __syncthreads();
    // swap phase (engine.cpp:148-187), replayed identically by every block
    const int64_t n_att = round_attempts(r.I, r.J, round);
    for (int q = tid; q < n_att; q += blockDim.x) {
        int sa, sb, ctr, is_p;
        if (swap_attempt(r.I, r.J, r.betas, r.pens, round, q, s.f, s.g, s.slot, r.swap_seed,
                         swap_base, sa, sb, ctr, is_p)) {
            const int xa = s.slot[sa], xb = s.slot[sb];
            s.slot[sa] = xb;
            s.slot[sb] = xa;
            s.state[xb] = sa;
            s.state[xa] = sb;
            if (blockIdx.x == 0) {
                if (is_p) r.acc_p[ctr] += 1; else r.acc_b[ctr] += 1;
            }
        }
    }
    swap_base += (uint64_t)n_att;
    __syncthreads();
#ifdef TPW_EPI_STAMP
    TPW_EPI_STAMP(k, 8);
#endif
    if (blockIdx.x == 0) {
        // counters of the other parity are free again: zero them
        int32_t* other = r.cnt + (size_t)(par ^ 1) * 2 * r.cnt_stride;
        for (int m = tid; m < 2 * r.cnt_stride; m += blockDim.x) other[m] = 0;
        if (r.work) {
            int* ow = r.work + (size_t)(par ^ 1) * n_work;
            for (int m = tid; m < n_work; m += blockDim.x) ow[m] = 0;
        }
        for (int m = tid; m < r.R; m += blockDim.x) {
            r.slot_state[m] = s.slot[m];
            r.state_slot[m] = s.state[m];
            r.f_all[m] = s.f[m];
            r.g_all[m] = s.g[m];
        }
        if (tid == 0) {  // record, engine.cpp:189-208
            TgRecordDev* rec = reinterpret_cast<TgRecordDev*>(r.rec) + k;
            const int tg = s.slot[r.R - 1];
            rec->round = round;
            rec->sweep_count = round * r.sps;
            rec->f = s.f[tg];
            rec->g = s.g[tg];
            rec->feasible = s.g[tg] == 0.0 ? 1 : 0;
            rec->target_state = tg;
        }
        if ((r.rec_flags & 8) && r.rec_acc) {
            int64_t* dst = r.rec_acc + (size_t)k * (np + nb);
            for (int q = tid; q < np; q += blockDim.x) dst[q] = r.acc_p[q];
            for (int q = tid; q < nb; q += blockDim.x) dst[np + q] = r.acc_b[q];
        }
    }
    // threshold planes for the new labels: warp job = (word, type, class).
    // Plane b (b = 0..52) holds bit 52-b of the lanes' 53-bit thresholds:
    // the 32x32 transpose of the words K >> 21 gives lane j plane 31-j, that
    // of K << 11 gives lane j >= 11 plane 63-j (two transposes instead of 53
    // ballots).
    {
        int combos = 0;
        for (int ty = 0; ty < a.n_types; ++ty) combos += a.ty[ty].ncl;
        const int total = a.W * combos;
        for (int job = gw; job < total; job += nw) {
            const int w = job / combos;
            int c = job % combos, ty = 0;
            while (c >= a.ty[ty].ncl) { c -= a.ty[ty].ncl; ++ty; }
            const PlaneType& pt = a.ty[ty];
            const int m = w * 32 + lane;
            uint64_t K = 0;
            const bool live = m < a.local_states;
            if (live) K = r.ktab[(size_t)s.state[m] * r.ktab_row + pt.ktab_off + c];
            uint32_t* dst = r.kp + (size_t)w * a.kpw + pt.kp_off + c;
            uint32_t* dstc = (c == 2 || c == 3)
                ? r.kpc + ((size_t)w * a.n_types + ty) * 128 + (c - 2) * 64 : nullptr;
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
#ifdef TPW_EPI_STAMP
    TPW_EPI_STAMP(k, 9);
#endif
    // target-state digest / snapshot for the trace (optional)
    if (r.rec_flags & 3) {
        const int tg = s.slot[r.R - 1];
        uint64_t dsum = 0;
        // four independent row loads in flight per thread (the pass is a
        // latency-bound gather of one word per site)
        const int stride = gridDim.x * blockDim.x;
        for (int i0 = blockIdx.x * blockDim.x + tid; i0 < a.n; i0 += 4 * stride) {
            uint32_t wv[4];
            int ci[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * stride;
                wv[u] = i < a.n ? a.spins[(size_t)i * a.W + (tg >> 5)] : 0u;
                ci[u] = i < a.n ? r.perm[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * stride;
                if (i >= a.n) break;
                const bool up = (wv[u] >> (tg & 31)) & 1u;
                if (r.rec_flags & 2) r.rec_states[(size_t)k * a.n + ci[u]] = up ? 1 : -1;
                if (up) dsum += digest_term((uint64_t)ci[u]);
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
#ifdef TPW_EPI_STAMP
    TPW_EPI_STAMP(k, 10);
#endif
    cg::this_grid().sync();
}

}  // namespace tg
