// host_common.cu -- validation, canonical order, host copies, thresholds, error plumbing (C ABI support).
#include "host.cuh"

#include <dlfcn.h>

namespace tgh {

thread_local std::string g_create_error;
thread_local cudaStream_t t_alloc_stream = nullptr;

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a{};
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
        a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
        a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
        a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
        a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
        a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
        a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.AllReduce &&
               a.GroupStart && a.GroupEnd && a.GetErrorString;
        return a;
    }();
    return api;
}

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw TgFail{code, buf};
}

// Greedy colouring in index order and canonical order (see tg_canonical_order).
void canonical(int n, const std::vector<int>& ci, const std::vector<int>& cj,
               const std::vector<int>& pa, const std::vector<int>& pb, std::vector<int>& order,
               std::vector<int>& color, int& n_colors) {
    std::vector<int> dc(n, 0), dq(n, 0), off(n + 1, 0);
    for (size_t k = 0; k < ci.size(); ++k) { dc[ci[k]]++; dc[cj[k]]++; }
    for (size_t k = 0; k < pa.size(); ++k) { dq[pa[k]]++; dq[pb[k]]++; }
    for (int i = 0; i < n; ++i) off[i + 1] = off[i] + dc[i] + dq[i];
    std::vector<int> adj(off[n]), cur(off.begin(), off.end() - 1);
    for (size_t k = 0; k < ci.size(); ++k) { adj[cur[ci[k]]++] = cj[k]; adj[cur[cj[k]]++] = ci[k]; }
    for (size_t k = 0; k < pa.size(); ++k) { adj[cur[pa[k]]++] = pb[k]; adj[cur[pb[k]]++] = pa[k]; }
    color.assign(n, 0);
    std::vector<char> used(n + 2, 0);
    n_colors = 0;
    for (int i = 0; i < n; ++i) {
        for (int k = off[i]; k < off[i + 1]; ++k) if (adj[k] < i) used[color[adj[k]]] = 1;
        int c = 0;
        while (used[c]) ++c;
        color[i] = c;
        n_colors = std::max(n_colors, c + 1);
        for (int k = off[i]; k < off[i + 1]; ++k) if (adj[k] < i) used[color[adj[k]]] = 0;
    }
    // stable counting sort by (colour, chain degree, cost degree)
    int mq = 0, mc = 0;
    for (int i = 0; i < n; ++i) { mq = std::max(mq, dq[i]); mc = std::max(mc, dc[i]); }
    const size_t nk = (size_t)n_colors * (mq + 1) * (mc + 1);
    std::vector<int> bucket(nk + 1, 0), keyv(n);
    for (int i = 0; i < n; ++i) {
        keyv[i] = (color[i] * (mq + 1) + dq[i]) * (mc + 1) + dc[i];
        bucket[keyv[i] + 1]++;
    }
    for (size_t k = 0; k < nk; ++k) bucket[k + 1] += bucket[k];
    order.resize(n);
    for (int i = 0; i < n; ++i) order[bucket[keyv[i]]++] = i;
}

// IsingModel / ConstraintSet validation (ising.cpp:21-46, constraints.cpp:16-26)
void load_problem(BatchInst& bi, int n, int n_couplings, const int32_t* ci, const int32_t* cj,
                  const double* w, const double* fields, int n_pairs, const int32_t* pa,
                  const int32_t* pb) {
    if (n <= 0) fail(TG_ERR_CONFIG, "model: n_spins must be positive");
    if (n_couplings < 0 || n_pairs < 0) fail(TG_ERR_CONFIG, "model: negative counts");
    std::vector<int> a(n_couplings), b(n_couplings), qa(n_pairs), qb(n_pairs);
    std::vector<int> row(n + 1, 0);
    for (int k = 0; k < n_couplings; ++k) {
        int x = ci[k], y = cj[k];
        if (x == y) fail(TG_ERR_CONFIG, "model: self-loop on spin %d", x);
        if (x > y) std::swap(x, y);
        if (x < 0 || y >= n) fail(TG_ERR_CONFIG, "model: coupling index out of range: (%d, %d)", x, y);
        if (!std::isfinite(w[k])) fail(TG_ERR_CONFIG, "model: coupling weights must be finite");
        a[k] = x;
        b[k] = y;
        row[x + 1]++;
    }
    {   // duplicate check in O(E): bucket the upper endpoints by lower endpoint
        // (counting sort), then sort each short bucket; the reported pair is the
        // smallest duplicate, as after the reference's full sort (ising.cpp:37-46)
        for (int i = 0; i < n; ++i) row[i + 1] += row[i];
        std::vector<int> cur(row.begin(), row.end() - 1), ys(n_couplings);
        for (int k = 0; k < n_couplings; ++k) ys[cur[a[k]]++] = b[k];
        for (int i = 0; i < n; ++i) {
            int* p0 = ys.data() + row[i];
            int* p1 = ys.data() + row[i + 1];
            if (p1 - p0 < 2) continue;
            std::sort(p0, p1);
            for (int* q = p0 + 1; q < p1; ++q)
                if (*q == q[-1]) fail(TG_ERR_CONFIG, "model: duplicate coupling (%d, %d)", i, *q);
        }
    }
    for (int k = 0; k < n_pairs; ++k) {
        int x = pa[k], y = pb[k];
        if (x == y) fail(TG_ERR_CONFIG, "constraint: pair on a single spin %d", x);
        if (x > y) std::swap(x, y);
        if (x < 0 || y >= n) fail(TG_ERR_CONFIG, "constraint: index out of range: (%d, %d)", x, y);
        qa[k] = x;
        qb[k] = y;
    }
    bi.n = n;
    bi.ci = a;
    bi.cj = b;
    bi.cw.assign(w, w + n_couplings);
    bi.h.assign(n, 0.0);
    if (fields) for (int i = 0; i < n; ++i) bi.h[i] = fields[i];
    for (double x : bi.h) if (!std::isfinite(x)) fail(TG_ERR_CONFIG, "model: fields must be finite");
    bi.pa = qa;
    bi.pb = qb;
}

void check_vec(const std::vector<double>& v, const char* what) {  // engine.cpp:41-52
    if (v.empty()) fail(TG_ERR_CONFIG, "%s vector must be non-empty", what);
    for (double x : v) if (!std::isfinite(x)) fail(TG_ERR_CONFIG, "%s entries must be finite", what);
    for (size_t k = 1; k < v.size(); ++k)
        if (v[k] <= v[k - 1]) fail(TG_ERR_CONFIG, "%s vector must be strictly increasing", what);
}

void ensure_host_arrays(tg_ctx& c);

// 53-bit acceptance threshold: the draw u = U53 * 2^-53 accepts iff U53 < K;
// K >= 2^53 encodes "always" (u < 1).  Reference expressions of mc.cpp:27-28
// (Metropolis) and of the heat-bath rule, evaluated with the host libm.
uint64_t threshold_metropolis(double beta, double de) {
    if (de <= 0.0) return 1ull << 53;
    const double T = std::exp(-beta * de);
    if (!(T < 1.0)) return 1ull << 53;  // beta <= 0: accepted for every uniform (no overflowing cast)
    return (uint64_t)std::ceil(T * 0x1.0p53);
}
uint64_t threshold_heat_bath(double beta, double local) {
    const double p = 1.0 / (1.0 + std::exp(-2.0 * beta * local));
    return (uint64_t)std::ceil(p * 0x1.0p53);
}

void build_plane_rest(tg_ctx& c, std::vector<PlaneType>& types, const std::vector<int>& chunk_off);

// Host copies of the instance (indices normalised i < j as IsingModel /
// ConstraintSet store them), fetched from the device copy on first use by a
// host-side path (SLOT engine, batches, probes, the J-column baseline).
void ensure_host_arrays(tg_ctx& c) {
    if (c.host_arrays) return;
    cudaStream_t st = c.stream;
    c.ci.resize(c.m); c.cj.resize(c.m); c.cw.resize(c.m); c.h.resize(c.n);
    c.pa.resize(c.np); c.pb.resize(c.np);
    if (c.m) {
        CK(cudaMemcpyAsync(c.ci.data(), c.d_raw_ci.p, sizeof(int) * c.m, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c.cj.data(), c.d_raw_cj.p, sizeof(int) * c.m, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c.cw.data(), c.d_raw_w.p, sizeof(double) * c.m, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(c.h.data(), c.d_raw_h.p, sizeof(double) * c.n, cudaMemcpyDeviceToHost, st));
    if (c.np) {
        CK(cudaMemcpyAsync(c.pa.data(), c.d_raw_pa.p, sizeof(int) * c.np, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c.pb.data(), c.d_raw_pb.p, sizeof(int) * c.np, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    for (int k = 0; k < c.m; ++k)
        if (c.ci[k] > c.cj[k]) std::swap(c.ci[k], c.cj[k]);
    for (int k = 0; k < c.np; ++k)
        if (c.pa[k] > c.pb[k]) std::swap(c.pa[k], c.pb[k]);
    c.host_arrays = true;
}

// Host copies of the canonical order (order / inv / color) for host-side
// paths, from the device prep when it ran.
void ensure_host_canonical(tg_ctx& c) {
    if (c.host_canonical) return;
    const int n = c.n;
    c.order.resize(n);
    c.inv.resize(n);
    CK(cudaMemcpyAsync(c.order.data(), c.d_order_dev.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(c.inv.data(), c.d_inv_dev.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    c.color.assign(n, 0);
    for (int col = 0; col < c.n_colors; ++col)
        for (int k = c.color_start[col]; k < c.color_start[col + 1]; ++k) c.color[c.order[k]] = col;
    c.host_canonical = true;
}

// PLANE engine structure from the device prep: site types and 32-site chunks
// from the (colour, chain degree, cost degree) run summary; rows stay on the
// device.  Same types / chunks / rows as the host construction below.

}  // namespace tgh
