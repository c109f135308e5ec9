// prep.cu -- instance preprocessing on the device for the PLANE engine.
//
// The host used to validate the instance, colour it greedily in index order,
// relabel it (canonical order) and build the internal CSR --
// about 110 ms of single-threaded host work at N = 2^20, more than five times
// the 100-round sweep it prepares.  Everything that touches O(N + E) data runs
// here instead; the host only sees O(colours x site types) summaries.
//
//   validate   IsingModel / ConstraintSet checks (ising.cpp:21-46,
//              constraints.cpp:16-26) as one flag word; on a violation the
//              caller re-runs the host validator to produce the reference's
//              exact message (error path only).
//   adjacency  cost + chain CSR in caller order, rows sorted (deterministic),
//              duplicate couplings detected per row.
//   colour     greedy index-order colouring (colour(i) = mex of the colours of
//              i's lower-index neighbours) as a fixpoint: a node is coloured as
//              soon as all its lower neighbours are, which yields exactly the
//              sequential greedy result; rounds run inside one cooperative
//              kernel.  Graphs whose dependency chains are longer than the
//              round budget are finished on the host from the partial result.
//   order      stable radix sort of (colour, chain degree, cost degree) keys --
//              the same stable counting sort as the host canonical order.
//   csr        internal-order rows (cost entries first with the J<0 sign bit,
//              then chain entries), and the (key) run-length summary the host
//              turns into site types and 32-site chunks.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "engine.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tg {

namespace {

__global__ void k_check_couplings(int n, int m, const int* ci, const int* cj, const double* w,
                                  int* degc, unsigned* bad) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
        int x = ci[k], y = cj[k];
        if (x > y) { const int t = x; x = y; y = t; }
        if (x == y || x < 0 || y >= n || !isfinite(w[k])) {
            atomicOr(bad, kPrepBadCoupling);
            continue;
        }
        if (!(w[k] == 1.0 || w[k] == -1.0) && !(*(volatile unsigned*)bad & kPrepNotPM1))
            atomicOr(bad, kPrepNotPM1);  // set once; later threads see it and skip the atomic
        atomicAdd(&degc[x], 1);
        atomicAdd(&degc[y], 1);
    }
}

__global__ void k_check_pairs(int n, int np, const int* pa, const int* pb, int* degq, unsigned* bad) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < np; k += gridDim.x * blockDim.x) {
        int x = pa[k], y = pb[k];
        if (x > y) { const int t = x; x = y; y = t; }
        if (x == y || x < 0 || y >= n) {
            atomicOr(bad, kPrepBadPair);
            continue;
        }
        atomicAdd(&degq[x], 1);
        atomicAdd(&degq[y], 1);
    }
}

__global__ void k_degrees(int n, const double* h, const int* degc, const int* degq, int* deg,
                          unsigned* bad, int* maxd) {
    int mc = 0, mq = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (!isfinite(h[i])) atomicOr(bad, kPrepBadField);
        if (h[i] != 0.0 && !(*(volatile unsigned*)bad & kPrepNonzeroField)) atomicOr(bad, kPrepNonzeroField);
        deg[i] = degc[i] + degq[i];
        mc = max(mc, degc[i]);
        mq = max(mq, degq[i]);
    }
    mc = __reduce_max_sync(0xffffffffu, mc);
    mq = __reduce_max_sync(0xffffffffu, mq);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&maxd[0], mc);
        atomicMax(&maxd[1], mq);
    }
}

// rows: [off[i], off[i] + degc[i]) cost entries (neighbour | J<0 sign bit),
// then degq[i] chain entries
__global__ void k_scatter(int n, int m, int np, const int* ci, const int* cj, const double* w,
                          const int* pa, const int* pb, int* curc, int* curq, int* adj) {
    const int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
        const int x = ci[k], y = cj[k];
        const int sgn = w[k] < 0.0 ? (int)0x80000000u : 0;
        adj[atomicAdd(&curc[x], 1)] = y | sgn;
        adj[atomicAdd(&curc[y], 1)] = x | sgn;
    }
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < np; k += stride) {
        const int x = pa[k], y = pb[k];
        adj[atomicAdd(&curq[x], 1)] = y;
        adj[atomicAdd(&curq[y], 1)] = x;
    }
}

__device__ __forceinline__ void sort_segment(int* a, int len) {
    for (int p = 1; p < len; ++p) {  // insertion sort on the neighbour index (rows are short)
        const int v = a[p];
        const int key = v & 0x7fffffff;
        int q = p - 1;
        while (q >= 0 && (a[q] & 0x7fffffff) > key) {
            a[q + 1] = a[q];
            --q;
        }
        a[q + 1] = v;
    }
}

__global__ void k_sort_rows(int n, const int* off, const int* degc, int* adj, unsigned* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int* row = adj + off[i];
        const int dc = degc[i], d = off[i + 1] - off[i];
        sort_segment(row, dc);
        sort_segment(row + dc, d - dc);
        for (int p = 1; p < dc; ++p)
            if ((row[p] & 0x7fffffff) == (row[p - 1] & 0x7fffffff)) atomicOr(bad, kPrepDuplicate);
    }
}

// Greedy index-order colouring as a fixpoint inside one cooperative kernel.
// ctr[0..2]: per-round counts of still-uncoloured nodes, ctr[3..5]: per-round
// "more than 64 colours" flags -- rotating slots, so every thread takes the
// same break decision from values that are final after the round's grid sync.
__global__ void k_colour(int n, const int* off, const int* adj, int* color, int* ctr, int max_rounds,
                         int* status) {
    cg::grid_group grid = cg::this_grid();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    volatile int* vc = color;
    int round = 0;
    for (; round < max_rounds; ++round) {
        int left = 0;
        bool ovf = false;
        for (int i = tid; i < n; i += stride) {
            if (vc[i] >= 0) continue;
            unsigned long long used = 0ull;
            bool ready = true;
            for (int e = off[i]; e < off[i + 1]; ++e) {
                const int j = adj[e] & 0x7fffffff;
                if (j >= i) continue;
                const int c = vc[j];
                if (c < 0) { ready = false; break; }
                if (c >= 63) { ovf = true; ready = false; break; }  // 64+ colours: host path
                used |= 1ull << c;
            }
            if (!ready) { ++left; continue; }
            vc[i] = __ffsll((long long)~used) - 1;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) left += __shfl_xor_sync(0xffffffffu, left, o);
        const bool any_ovf = __any_sync(0xffffffffu, ovf);
        if ((threadIdx.x & 31) == 0) {
            if (left) atomicAdd(&ctr[round % 3], left);
            if (any_ovf) atomicExch(&ctr[3 + round % 3], 1);
        }
        grid.sync();
        // slot r % 3 is read by everyone between sync r and sync r+1; it was
        // reset in round r-2 and is reset again in round r+1 (after sync r+1)
        const int remaining = *(volatile int*)&ctr[round % 3];
        const int overflow = *(volatile int*)&ctr[3 + round % 3];
        if (tid == 0) {
            ctr[(round + 2) % 3] = 0;
            ctr[3 + (round + 2) % 3] = 0;
        }
        if (overflow) {
            if (tid == 0) status[0] |= 2;
            break;
        }
        if (remaining == 0) break;
    }
    if (tid == 0) status[1] = round;
}

__global__ void k_keys(int n, const int* color, const int* degc, const int* degq, const int* maxd,
                       unsigned* key, int* idx, int* ncol) {
    const int mc = maxd[0], mq = maxd[1];
    int mx = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int c = color[i];
        key[i] = (unsigned)((c * (mq + 1) + degq[i]) * (mc + 1) + degc[i]);
        idx[i] = i;
        mx = max(mx, c);
    }
    mx = __reduce_max_sync(0xffffffffu, mx);  // one atomic per warp, not per thread
    if ((threadIdx.x & 31) == 0) atomicMax(ncol, mx + 1);
}

__global__ void k_inverse(int n, const int* order, const int* deg, int* inv, int* deg_int) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = order[k];
        inv[i] = k;
        deg_int[k] = deg[i];
    }
}

__global__ void k_internal_rows(int n, const int* order, const int* inv, const int* off, const int* adj,
                                const int* base, int* nbr) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = order[k];
        const int d = off[i + 1] - off[i];
        for (int e = 0; e < d; ++e) {
            const int v = adj[off[i] + e];
            nbr[base[k] + e] = inv[v & 0x7fffffff] | (v & (int)0x80000000u);
        }
    }
}

__global__ void k_chunk_bases(int n_chunks, Chunk* chunks, const int* base) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_chunks; q += gridDim.x * blockDim.x)
        chunks[q].nbr_base = base[chunks[q].start];
}

int grid_for(int count, int sms) { return std::max(1, std::min((count + 255) / 256, sms * 8)); }

__global__ void k_chain_cursors(int n, const int* off, const int* degc, int* curc, int* curq) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        curc[i] = off[i];
        curq[i] = off[i] + degc[i];
    }
}

// stream-ordered temporaries, released on the stream when the pool goes out of scope
struct Tmp {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Tmp(cudaStream_t s) : st(s) {}
    template <class T>
    T* get(size_t count) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, sizeof(T) * std::max<size_t>(count, 1), st) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Tmp() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

}  // namespace

#define PK(x)                                    \
    do {                                         \
        cudaError_t e_ = (x);                    \
        if (e_ != cudaSuccess) return e_;        \
    } while (0)
#define PA(p)                                                   \
    do {                                                        \
        if (!(p)) return cudaErrorMemoryAllocation;             \
    } while (0)

cudaError_t plane_prep_device(const PrepIn& in, const PrepOut& o, PrepSummary& r, cudaStream_t st,
                              int sms) {
    const int n = in.n, m = in.m, np = in.np;
    Tmp T(st);
    const int gb = grid_for(std::max(std::max(m, np), n), sms);
    int* degc = T.get<int>(n);
    int* degq = T.get<int>(n);
    int* deg = T.get<int>(n + 1);
    int* off = T.get<int>(n + 1);
    unsigned* bad = T.get<unsigned>(1);
    int* small = T.get<int>(12);  // maxd[2], status[2], ctr[6], ncol
    PA(degc); PA(degq); PA(deg); PA(off); PA(bad); PA(small);
    int* maxd = small;
    int* status = small + 2;
    int* ctr = small + 4;
    int* ncol = small + 10;
    PK(cudaMemsetAsync(degc, 0, sizeof(int) * n, st));
    PK(cudaMemsetAsync(degq, 0, sizeof(int) * n, st));
    PK(cudaMemsetAsync(deg, 0, sizeof(int) * (n + 1), st));
    PK(cudaMemsetAsync(bad, 0, sizeof(unsigned), st));
    PK(cudaMemsetAsync(small, 0, sizeof(int) * 12, st));
    if (m) k_check_couplings<<<gb, 256, 0, st>>>(n, m, in.ci, in.cj, in.w, degc, bad);
    if (np) k_check_pairs<<<gb, 256, 0, st>>>(n, np, in.pa, in.pb, degq, bad);
    k_degrees<<<gb, 256, 0, st>>>(n, in.h, degc, degq, deg, bad, maxd);
    PK(cudaGetLastError());
    unsigned h_bad = 0;
    int h_maxd[2] = {0, 0};
    PK(cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, st));
    PK(cudaMemcpyAsync(h_maxd, maxd, sizeof h_maxd, cudaMemcpyDeviceToHost, st));
    PK(cudaStreamSynchronize(st));
    r.info = h_bad & ~kPrepErrors;
    r.bad = h_bad & kPrepErrors;
    if (r.bad) return cudaSuccess;
    r.max_dc = h_maxd[0];
    r.max_dq = h_maxd[1];

    // caller-order CSR: cost entries (sign bit) then chain entries, rows sorted
    size_t tb = 0;
    PK(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, off, n + 1, st));
    void* tmp = T.get<char>(tb);
    PA(tmp);
    PK(cub::DeviceScan::ExclusiveSum(tmp, tb, deg, off, n + 1, st));
    int* curc = T.get<int>(n);
    int* curq = T.get<int>(n);
    int* adj = T.get<int>((size_t)2 * (m + np));
    PA(curc); PA(curq); PA(adj);
    k_chain_cursors<<<gb, 256, 0, st>>>(n, off, degc, curc, curq);
    k_scatter<<<gb, 256, 0, st>>>(n, m, np, in.ci, in.cj, in.w, in.pa, in.pb, curc, curq, adj);
    k_sort_rows<<<gb, 256, 0, st>>>(n, off, degc, adj, bad);
    PK(cudaGetLastError());

    // greedy colouring fixpoint (cooperative: all blocks resident)
    int* color = T.get<int>(n);
    PA(color);
    PK(cudaMemsetAsync(color, 0xff, sizeof(int) * n, st));
    int per_sm = 0;
    PK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_colour, 256, 0));
    const int cgrid = std::max(1, std::min(per_sm * sms, (n + 255) / 256));
    int max_rounds = kPrepColourRounds;
    {
        int nn = n;
        void* args[] = {&nn, &off, &adj, &color, &ctr, &max_rounds, &status};
        PK(cudaLaunchCooperativeKernel((const void*)k_colour, dim3(cgrid), dim3(256), args, 0, st));
    }
    int h_status[2] = {0, 0};
    PK(cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, st));
    PK(cudaMemcpyAsync(h_status, status, sizeof h_status, cudaMemcpyDeviceToHost, st));
    PK(cudaStreamSynchronize(st));
    r.bad = h_bad & kPrepErrors;
    r.colour_rounds = h_status[1];
    if (r.bad) return cudaSuccess;
    if ((h_status[0] & 2) || h_status[1] >= max_rounds) {
        r.colour_incomplete = true;
        return cudaSuccess;
    }

    // canonical order: stable sort of (colour, chain degree, cost degree) keys
    unsigned* key = T.get<unsigned>(n);
    unsigned* key_sorted = T.get<unsigned>(n);
    int* idx = T.get<int>(n);
    PA(key); PA(key_sorted); PA(idx);
    k_keys<<<gb, 256, 0, st>>>(n, color, degc, degq, maxd, key, idx, ncol);
    PK(cudaGetLastError());
    const unsigned long long kmax = 64ull * (h_maxd[1] + 1) * (h_maxd[0] + 1);
    int end_bit = 1;
    while ((1ull << end_bit) < kmax && end_bit < 32) ++end_bit;
    tb = 0;
    PK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key_sorted, idx, o.order, n, 0, end_bit, st));
    tmp = T.get<char>(tb);
    PA(tmp);
    PK(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key_sorted, idx, o.order, n, 0, end_bit, st));
    int* deg_int = T.get<int>(n + 1);
    PA(deg_int);
    PK(cudaMemsetAsync(deg_int + n, 0, sizeof(int), st));
    k_inverse<<<gb, 256, 0, st>>>(n, o.order, deg, o.inv, deg_int);
    tb = 0;
    PK(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg_int, o.base, n + 1, st));
    tmp = T.get<char>(tb);
    PA(tmp);
    PK(cub::DeviceScan::ExclusiveSum(tmp, tb, deg_int, o.base, n + 1, st));
    k_internal_rows<<<gb, 256, 0, st>>>(n, o.order, o.inv, off, adj, o.base, o.nbr);
    PK(cudaGetLastError());

    // (colour, dq, dc) runs -> site types and chunks on the host
    unsigned* rk = T.get<unsigned>(n);
    int* rc = T.get<int>(n);
    int* nruns = T.get<int>(1);
    PA(rk); PA(rc); PA(nruns);
    tb = 0;
    PK(cub::DeviceRunLengthEncode::Encode(nullptr, tb, key_sorted, rk, rc, nruns, n, st));
    tmp = T.get<char>(tb);
    PA(tmp);
    PK(cub::DeviceRunLengthEncode::Encode(tmp, tb, key_sorted, rk, rc, nruns, n, st));
    int h_runs = 0, h_ncol = 0;
    // the run count is bounded by the key range: when that bound is small, the
    // runs come back with the counts in the same synchronisation
    const size_t bound = (size_t)std::min<unsigned long long>((unsigned long long)n, kmax);
    const bool eager = bound <= kPrepEagerRuns;
    if (eager) {
        r.run_keys.resize(bound);
        r.run_counts.resize(bound);
        PK(cudaMemcpyAsync(r.run_keys.data(), rk, sizeof(unsigned) * bound, cudaMemcpyDeviceToHost, st));
        PK(cudaMemcpyAsync(r.run_counts.data(), rc, sizeof(int) * bound, cudaMemcpyDeviceToHost, st));
    }
    PK(cudaMemcpyAsync(&h_runs, nruns, sizeof(int), cudaMemcpyDeviceToHost, st));
    PK(cudaMemcpyAsync(&h_ncol, ncol, sizeof(int), cudaMemcpyDeviceToHost, st));
    PK(cudaStreamSynchronize(st));
    r.n_colors = h_ncol;
    if (eager) {
        r.run_keys.resize(h_runs);
        r.run_counts.resize(h_runs);
        return cudaSuccess;
    }
    r.run_keys.resize(h_runs);
    r.run_counts.resize(h_runs);
    PK(cudaMemcpyAsync(r.run_keys.data(), rk, sizeof(unsigned) * h_runs, cudaMemcpyDeviceToHost, st));
    PK(cudaMemcpyAsync(r.run_counts.data(), rc, sizeof(int) * h_runs, cudaMemcpyDeviceToHost, st));
    PK(cudaStreamSynchronize(st));
    return cudaSuccess;
}

cudaError_t plane_chunk_bases(Chunk* chunks, int n_chunks, const int* base, cudaStream_t st, int sms) {
    if (n_chunks > 0) k_chunk_bases<<<grid_for(n_chunks, sms), 256, 0, st>>>(n_chunks, chunks, base);
    return cudaGetLastError();
}

}  // namespace tg
