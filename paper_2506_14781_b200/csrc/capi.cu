// capi.cu -- host driver behind the C ABI (include/tempergrid_b200.h).
//
// Owns the device copy of one ConstrainedProblem in canonical colour order,
// the replica grid labels, and the round loop of run_2dpt
// (/root/reference/proj/src/engine.cpp:83-219): per round one sweep launch
// (all sweeps_per_swap sweeps, every colour phase), the (f, g) exchange
// (NCCL all-gather when the grid is split over GPUs), one swap/record launch,
// and an optional target-state extract; records drain to the caller's sink
// in round order.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <thread>
#include <vector>
#include <limits>

#include "../../include/tempergrid_b200.h"
#include "engine.cuh"
#include "kernels.cuh"

using namespace tg;

namespace {

thread_local std::string g_create_error;

// NCCL is resolved at run time (dlopen) and only when a context spans more
// than one GPU: linking it would pin whichever libnccl.so.2 loads first into
// the process, and PyTorch needs its own bundled build.  Under torchrun,
// PyTorch is imported first, so its copy is the one dlopen returns.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

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

struct TgFail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw TgFail{code, buf};
}

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) fail(TG_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                    __FILE__, __LINE__);                                       \
    } while (0)
#define NK(x)                                                                                  \
    do {                                                                                       \
        if (!nccl().ok) fail(TG_ERR_CUDA, "NCCL library (libnccl.so.2) not available");         \
        ncclResult_t r_ = (x);                                                                 \
        if (r_ != ncclSuccess) fail(TG_ERR_CUDA, "%s: %s", #x, nccl().GetErrorString(r_));      \
    } while (0)

// Device buffers come from the device's stream-ordered memory pool on the
// stream of the context being served (set by guard() / create_impl): freed
// memory stays in the pool, so the next context's allocations -- e.g. the next
// run_2dpt call -- cost microseconds instead of cudaMalloc / cudaFree.
thread_local cudaStream_t t_alloc_stream = nullptr;

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s_ = nullptr;
    void alloc(size_t count) {
        release();
        n = count;
        s_ = t_alloc_stream;
        if (count) CK(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, s_));
    }
    void upload(const std::vector<T>& v, cudaStream_t s) {
        alloc(v.size());
        if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
    }
    void upload(const T* src, size_t count, cudaStream_t s) {
        alloc(count);
        if (count) CK(cudaMemcpyAsync(p, src, sizeof(T) * count, cudaMemcpyHostToDevice, s));
    }
    void copy_from(const DBuf<T>& o, cudaStream_t s) {
        alloc(o.n);
        if (o.n) CK(cudaMemcpyAsync(p, o.p, sizeof(T) * o.n, cudaMemcpyDeviceToDevice, s));
    }
    void zero(cudaStream_t s) {
        if (n) CK(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
    }
    void release() {
        if (p) cudaFreeAsync(p, s_);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
};

// Owns the context stream; declared before every DBuf member of tg_ctx, so it
// is destroyed after them (their stream-ordered frees are queued on a live
// stream) and drains the stream before destroying it.
struct StreamOwner {
    cudaStream_t s = nullptr;
    ~StreamOwner() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

// TG_HOST_TIMING=1: host-side phase timings on stderr (e2e breakdown).
struct HostTimer {
    const char* what;
    std::chrono::steady_clock::time_point t0;
    bool on;
    explicit HostTimer(const char* w) : what(w), t0(std::chrono::steady_clock::now()),
                                        on(std::getenv("TG_HOST_TIMING") != nullptr) {}
    ~HostTimer() {
        if (on)
            std::fprintf(stderr, "[tg host] %-28s %9.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

int nbits(int d) {
    int b = 0;
    while ((1 << b) <= d) ++b;
    return d == 0 ? 0 : b;
}


struct BatchInst {
    int n = 0;
    std::vector<int> ci, cj, pa, pb;
    std::vector<double> cw, h, betas, pens;
    uint64_t seed = 1;
};

struct S2Prep {
    int n = 0, n_colors = 0, D = 4;
    std::vector<int> order, inv, color, color_start, off;
    std::vector<int32_t> nbr;
    std::vector<double> w, h;
    std::vector<int8_t> cm;
    std::vector<float> h32;
    std::vector<int2> entp;
    std::vector<double> wp;
    float eps = 0.f, beta_max = 0.f;
};


struct Slot2 {
    int B = 0, I = 0, J = 0, R = 0, Rp = 0, G = 0, D = 4, max_colors = 0, slots = 1;
    int rec_cap = 0, grid = 0, nsub = 1;
    tg_run_config cfg{};
    std::vector<S2Prep> prep;
    DBuf<double> d_sbeta, d_stwop;
    DBuf<uint64_t> d_skey;
    std::vector<int> state_off;
    DBuf<SInst> d_inst;
    DBuf<int2> d_entp;
    DBuf<double> d_wp, d_w, d_h, d_betas, d_pens, d_part_f, d_part_g, d_f, d_g;
    DBuf<int> d_off, d_cstart, d_item_pref, d_energy_pref, d_perm;
    DBuf<int32_t> d_nbr, d_slot_state, d_state_slot;
    DBuf<int8_t> d_cm, d_spins, d_rec_states;
    DBuf<float> d_h32;
    DBuf<uint64_t> d_keys, d_swap_seed, d_seeds;
    DBuf<int64_t> d_acc_p, d_acc_b, d_rec_acc;
    DBuf<TgRecordDev> d_rec;
    std::vector<TgRecordDev> h_rec;
    std::vector<int64_t> h_acc;
    std::vector<int8_t> h_states;
    int64_t rounds_done = 0;
    uint64_t swap_base = 0;
    bool ready = false;
    // schedule probes (schedule.cpp:18-52): independent chains, no swaps,
    // one stream per chain for the initial state and the sweeps
    bool probe = false;
    DBuf<uint64_t> d_init_keys;
    DBuf<double> d_hist_f, d_hist_g, d_moments;
    std::vector<SInst> h_inst;
    // separate energy pass (large batches): slices per instance, partials
    bool sep_energy = false;
    int e_slices = 1;
    DBuf<double> d_epart;
    // KL observer buffers
    bool kl_on = false;
    int64_t kl_cap = 0;
    DBuf<int> d_kl_off, d_kl_map, d_kl_err;
    DBuf<double> d_kl_p, d_kl;
    DBuf<uint32_t> d_kl_hist;
    DBuf<unsigned long long> d_kl_total;
    DBuf<int64_t> d_kl_samples;
    uint64_t probe_gen = 0;
    int probe_chains = 0, probe_rule = -1;
};

}  // namespace

struct tg_ctx {
    std::string err;
    int device = 0, rank = 0, world = 1;
    int sms = 0;
    StreamOwner stream_owner;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    bool profiling = false;

    // problem (caller order) + canonical relabel
    bool have_problem = false;
    uint64_t problem_gen = 0;
    int n = 0;
    std::vector<int> ci, cj, pa, pb;
    std::vector<double> cw, h;
    std::vector<int> order, inv, color;  // order[k] = caller index at internal k
    int n_colors = 0;
    std::vector<int> color_start;
    // canonical order + internal CSR computed on the device at set_problem
    // (prep.cu); the host copies of order / inv / color are materialised only
    // when a host-side path needs them (ensure_host_canonical)
    bool dev_prep = false, host_canonical = false, host_arrays = false;
    int m = 0, np = 0;
    PrepSummary prep;
    DBuf<int> d_raw_ci, d_raw_cj, d_raw_pa, d_raw_pb;  // caller arrays as given
    DBuf<double> d_raw_w, d_raw_h;
    DBuf<int> d_order_dev, d_inv_dev, d_base_dev, d_nbr_dev;

    bool have_schedule = false;
    std::vector<double> betas, pens;

    // run state
    bool initialised = false;
    tg_run_config cfg{};
    int engine = 0;
    int I = 0, J = 0, R = 0, R_local = 0, state0 = 0, W = 0;
    int64_t rounds_done = 0;
    uint64_t swap_base = 0;
    int kpw = 0, ktab_row = 0, n_types = 0, m_cost = 0, WV = 1;
    std::vector<PlaneType> h_types;
    std::vector<uint32_t> h_active;
    std::vector<uint2> h_wkey;
    int plane_grid = 0, plane_block = kPlaneThreads;
    int fused_grid = 0, fused_fast = 0, fused_block = kPlaneThreads, fused_wv = 4;
    size_t fused_smem = 0;
    size_t slot_smem = 0;

    DBuf<double> d_betas, d_pens, d_f, d_g;
    DBuf<int32_t> d_slot_state, d_state_slot, d_perm;
    DBuf<int64_t> d_acc_p, d_acc_b, d_rec_acc;
    DBuf<TgRecordDev> d_rec;
    DBuf<int8_t> d_rec_states;
    // plane
    DBuf<uint32_t> d_spins32, d_kp, d_kpc, d_active;
    DBuf<int32_t> d_nbr, d_cnt_c, d_cnt_q, d_cnt2;
    DBuf<int> d_work;
    DBuf<Chunk> d_chunks;
    DBuf<int> d_chunk_off, d_color_start;
    DBuf<PlaneType> d_types;
    DBuf<uint2> d_wkey;
    DBuf<uint64_t> d_ktab;
    // slot
    DBuf<int8_t> d_spins8, d_cm;
    DBuf<int> d_off;
    DBuf<int32_t> d_snbr;
    DBuf<double> d_sw, d_h;
    DBuf<int2> d_ent, d_entp;
    DBuf<double> d_wp;
    int slot_D = 0;
    DBuf<float> d_h32;
    float slot_eps = 0.0f, slot_beta_max = 0.0f;
    DBuf<uint64_t> d_slot_key;

    // decoded-sample KL observer (analysis.cpp:215-241), SLOT engine v2
    struct {
        bool on = false;
        int n_logical = 0, discard = 0;
        std::vector<int> copy_off, copies;   // caller physical indices, chain order
        std::vector<double> probs;           // exact logical Boltzmann, 2^n_logical
    } kl;

    // SLOT engine v2 (single instance and batches)
    std::vector<BatchInst> batch;
    Slot2 s2;
    bool use_s2 = false;

    int rec_cap = 0;
    std::vector<TgRecordDev> h_rec;
    std::vector<int8_t> h_states;
    std::vector<int64_t> h_acc;
    std::vector<cudaEvent_t> ev;
    double last_sweep_ms = 0, last_swap_ms = 0;
    int64_t sweep_launches = 0, other_launches = 0;

    ~tg_ctx() {
        t_alloc_stream = stream;
        for (auto e : ev) cudaEventDestroy(e);
        if (comm) nccl().CommDestroy(comm);
        // members free their buffers on `stream`; stream_owner destroys it last
    }
};

extern "C" int tg_partition(int n_replicas, int rank, int world, int engine, int32_t* state0,
                            int32_t* count);

namespace {

template <class F>
int guard(tg_ctx* ctx, F&& f) {
    if (ctx) t_alloc_stream = ctx->stream;
    try {
        f();
        if (ctx) ctx->err.clear();
        return TG_OK;
    } catch (const TgFail& e) {
        if (ctx) ctx->err = e.msg; else g_create_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what(); else g_create_error = e.what();
        return TG_ERR_INTERNAL;
    }
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

bool plane_eligible(tg_ctx& c, std::string* why) {
    if (c.dev_prep) {
        if (c.prep.info & kPrepNotPM1) { if (why) *why = "couplings must be +-1"; return false; }
        if (c.prep.info & kPrepNonzeroField) { if (why) *why = "fields must be 0"; return false; }
        if (c.prep.max_dc > kMaxDC || c.prep.max_dq > kMaxDQ) { if (why) *why = "degree bound exceeded"; return false; }
        return true;
    }
    ensure_host_arrays(c);
    for (double w : c.cw) if (!(w == 1.0 || w == -1.0)) { if (why) *why = "couplings must be +-1"; return false; }
    for (double x : c.h) if (x != 0.0) { if (why) *why = "fields must be 0"; return false; }
    std::vector<int> dc(c.n, 0), dq(c.n, 0);
    for (size_t k = 0; k < c.ci.size(); ++k) { dc[c.ci[k]]++; dc[c.cj[k]]++; }
    for (size_t k = 0; k < c.pa.size(); ++k) { dq[c.pa[k]]++; dq[c.pb[k]]++; }
    for (int i = 0; i < c.n; ++i)
        if (dc[i] > kMaxDC || dq[i] > kMaxDQ) { if (why) *why = "degree bound exceeded"; return false; }
    return true;
}

// 53-bit acceptance threshold: the draw u = U53 * 2^-53 accepts iff U53 < K;
// K >= 2^53 encodes "always" (u < 1).  Reference expressions of mc.cpp:27-28
// (Metropolis) and of the heat-bath rule, evaluated with the host libm.
uint64_t threshold_metropolis(double beta, double de) {
    if (de <= 0.0) return 1ull << 53;
    const double T = std::exp(-beta * de);
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
void build_plane_structure_device(tg_ctx& c, std::vector<PlaneType>& types, std::vector<Chunk>& chunks,
                                  std::vector<int>& chunk_off) {
    const PrepSummary& P = c.prep;
    const int mq1 = P.max_dq + 1, mc1 = P.max_dc + 1;
    std::vector<int> tid_of((kMaxDC + 1) * (kMaxDQ + 1), -1);
    chunk_off.assign(c.n_colors + 1, 0);
    int start = 0, cur_col = -1;
    for (size_t q = 0; q < P.run_keys.size(); ++q) {
        const unsigned key = P.run_keys[q];
        const int cnt = P.run_counts[q];
        const int dc = (int)(key % mc1), dq = (int)((key / mc1) % mq1), col = (int)(key / ((unsigned)mc1 * mq1));
        while (cur_col < col) chunk_off[++cur_col] = (int)chunks.size();
        const int tkey = dc * (kMaxDQ + 1) + dq;
        if (tid_of[tkey] < 0) {
            PlaneType t{};
            t.dc = dc;
            t.dq = dq;
            t.ncb = nbits(dc);
            t.nqb = nbits(dq);
            t.ncl = std::max(4, 1 << (t.ncb + t.nqb));
            tid_of[tkey] = (int)types.size();
            types.push_back(t);
        }
        for (int s0 = start; s0 < start + cnt; s0 += 32)
            chunks.push_back(Chunk{s0, std::min(32, start + cnt - s0), tid_of[tkey], 0});
        start += cnt;
    }
    while (cur_col < c.n_colors) chunk_off[++cur_col] = (int)chunks.size();
    chunk_off[c.n_colors] = (int)chunks.size();
}

void build_plane(tg_ctx& c) {
    HostTimer tm_("build_plane");
    cudaStream_t st = c.stream;
    const int n = c.n;
    if (c.dev_prep) {
        std::vector<PlaneType> types;
        std::vector<Chunk> chunks;
        std::vector<int> chunk_off;
        build_plane_structure_device(c, types, chunks, chunk_off);
        c.d_nbr.copy_from(c.d_nbr_dev, st);
        c.d_chunks.upload(chunks, st);
        CK(plane_chunk_bases(c.d_chunks.p, (int)chunks.size(), c.d_base_dev.p, st, c.sms));
        build_plane_rest(c, types, chunk_off);
        return;
    }
    ensure_host_arrays(c);
    ensure_host_canonical(c);
    // internal adjacency as flat CSR (cost entries carry the J<0 sign bit)
    std::vector<int> dcv(n, 0), dqv(n, 0);
    for (size_t k = 0; k < c.ci.size(); ++k) { dcv[c.inv[c.ci[k]]]++; dcv[c.inv[c.cj[k]]]++; }
    for (size_t k = 0; k < c.pa.size(); ++k) { dqv[c.inv[c.pa[k]]]++; dqv[c.inv[c.pb[k]]]++; }
    std::vector<int> base(n + 1, 0);
    for (int i = 0; i < n; ++i) base[i + 1] = base[i] + dcv[i] + dqv[i];
    std::vector<int32_t> nbr(base[n]);
    {
        std::vector<int> cc(n), cq(n);
        for (int i = 0; i < n; ++i) { cc[i] = base[i]; cq[i] = base[i] + dcv[i]; }
        for (size_t k = 0; k < c.ci.size(); ++k) {
            const int x = c.inv[c.ci[k]], y = c.inv[c.cj[k]];
            const int32_t sgn = c.cw[k] < 0 ? (int32_t)0x80000000u : 0;
            nbr[cc[x]++] = y | sgn;
            nbr[cc[y]++] = x | sgn;
        }
        for (size_t k = 0; k < c.pa.size(); ++k) {
            const int x = c.inv[c.pa[k]], y = c.inv[c.pb[k]];
            nbr[cq[x]++] = y;
            nbr[cq[y]++] = x;
        }
    }
    // site types (cost degree, chain degree)
    std::vector<int> tid_of((kMaxDC + 1) * (kMaxDQ + 1), -1);
    std::vector<int> site_type(n);
    std::vector<PlaneType> types;
    for (int i = 0; i < n; ++i) {
        const int key = dcv[i] * (kMaxDQ + 1) + dqv[i];
        if (tid_of[key] < 0) {
            PlaneType t{};
            t.dc = dcv[i];
            t.dq = dqv[i];
            t.ncb = nbits(t.dc);
            t.nqb = nbits(t.dq);
            t.ncl = std::max(4, 1 << (t.ncb + t.nqb));
            tid_of[key] = (int)types.size();
            types.push_back(t);
        }
        site_type[i] = tid_of[key];
    }
    // chunks (colour-major; the canonical order keeps types contiguous)
    std::vector<Chunk> chunks;
    std::vector<int> chunk_off(c.n_colors + 1, 0);
    for (int col = 0; col < c.n_colors; ++col) {
        chunk_off[col] = (int)chunks.size();
        int i = c.color_start[col];
        const int end = c.color_start[col + 1];
        while (i < end) {
            const int ty = site_type[i];
            int j = i;
            while (j < end && j - i < 32 && site_type[j] == ty) ++j;
            chunks.push_back(Chunk{i, j - i, ty, base[i]});
            i = j;
        }
    }
    chunk_off[c.n_colors] = (int)chunks.size();
    c.d_nbr.upload(nbr, st);
    c.d_chunks.upload(chunks, st);
    build_plane_rest(c, types, chunk_off);
}

// Everything after the site types and chunks: threshold tables, words, keys,
// masks, buffers and the cooperative grids.
void build_plane_rest(tg_ctx& c, std::vector<PlaneType>& types, const std::vector<int>& chunk_off) {
    cudaStream_t st = c.stream;
    const int n = c.n;
    if ((int)types.size() > kMaxTypes) fail(TG_ERR_RESOURCE, "plane engine: too many site types");
    int kpw = 0, krow = 0;
    for (auto& t : types) {
        t.kp_off = kpw;
        t.ktab_off = krow;
        kpw += kKWords * t.ncl;
        krow += t.ncl;
    }
    c.kpw = kpw;
    c.ktab_row = krow;
    c.n_types = (int)types.size();
    // words, keys, masks: rows padded to a whole number of WV-word passes
    const int w_log = (c.R_local + 31) / 32;
    c.WV = w_log > 2 ? 4 : w_log;
    if (const char* e = std::getenv("TG_PLANE_WV")) {  // tuning override: 1, 2 or 4
        const int v = std::atoi(e);
        if (v == 1 || v == 2 || v == 4) c.WV = std::min(v, w_log > 2 ? 4 : (w_log > 1 ? 2 : 1));
    }
    c.W = (w_log + c.WV - 1) / c.WV * c.WV;
    if (c.W > kMaxWordsArg) fail(TG_ERR_RESOURCE, "plane engine: %d replicas per rank exceed %d", c.R_local, 32 * kMaxWordsArg);
    std::vector<uint32_t> active(c.W, 0u);
    std::vector<uint2> wkey(c.W);
    for (int w = 0; w < c.W; ++w) {
        for (int l = 0; l < 32; ++l) if (w * 32 + l < c.R_local) active[w] |= 1u << l;
        const uint64_t k = derive_seed(c.cfg.seed, kPurposePlane, (uint64_t)(c.state0 / 32 + w));
        wkey[w] = make_uint2((uint32_t)k, (uint32_t)(k >> 32));
    }
    // thresholds per (slot, type, class)
    std::vector<uint64_t> ktab((size_t)c.R * krow, 0ull);
    for (int slot = 0; slot < c.R; ++slot) {
        const double beta = c.betas[slot / c.J], P = c.pens[slot % c.J];
        for (const auto& t : types) {
            for (int cl = 0; cl < t.ncl; ++cl) {
                const int ncnt = cl & ((1 << t.ncb) - 1);
                const int qcnt = cl >> t.ncb;
                uint64_t K = 0;
                if (ncnt <= t.dc && qcnt <= t.dq) {
                    // s_i * local_i (Metropolis, counts of satisfied bonds) or
                    // local_i (heat bath, counts of +1 contributions)
                    const double v = (double)(2 * ncnt - t.dc) + 2.0 * P * (double)(2 * qcnt - t.dq);
                    K = c.cfg.rule == TG_RULE_METROPOLIS ? threshold_metropolis(beta, 2.0 * v)
                                                         : threshold_heat_bath(beta, v);
                }
                ktab[(size_t)slot * krow + t.ktab_off + cl] = K;
            }
        }
    }
    c.m_cost = c.m;
    c.d_chunk_off.upload(chunk_off, st);
    c.d_color_start.upload(c.color_start, st);
    c.d_types.upload(types, st);
    c.h_types = types;
    c.h_active = active;
    c.h_wkey = wkey;
    c.d_ktab.upload(ktab, st);
    c.d_kp.alloc((size_t)c.W * kpw);
    c.d_kp.zero(st);
    c.d_kpc.alloc((size_t)c.W * c.n_types * 128);
    c.d_kpc.zero(st);
    c.d_spins32.alloc((size_t)n * c.W);
    c.d_cnt_c.alloc((size_t)c.W * 32);
    c.d_cnt_q.alloc((size_t)c.W * 32);
    c.d_cnt_c.zero(st);
    c.d_cnt_q.zero(st);
    c.d_cnt2.alloc((size_t)4 * c.W * 32);
    c.d_cnt2.zero(st);
    c.d_work.alloc((size_t)2 * c.n_colors * std::max(1, c.W));
    c.d_work.zero(st);
    // cooperative grid: a multiple of W warps, all blocks co-resident
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)plane_sweep_fn(c.cfg.rule, c.WV),
                                                     kPlaneThreads, 0));
    if (per_sm < 1) fail(TG_ERR_RESOURCE, "plane engine: kernel does not fit on an SM");
    int blocks = per_sm * c.sms;
    const int wpb = kPlaneThreads / 32;
    const int passes = c.W / c.WV;
    blocks -= blocks % passes;  // each block owns one pass of WV words
    if (blocks < passes) fail(TG_ERR_RESOURCE, "plane engine: cannot tile %d words", c.W);
    c.plane_grid = blocks;
    // fused round-loop kernel (single GPU)
    c.fused_fast = 1;
    for (const auto& t : types) if (t.ncb > 2 || t.nqb > 1) c.fused_fast = 0;
    // FAST: specialised kernel for site types with cost degree <= 3 and chain
    // degree <= 1 (config 5), cp.async row prefetch; TG_PLANE_FAST=0 disables.
    if (const char* e = std::getenv("TG_PLANE_FAST")) c.fused_fast = c.fused_fast && std::atoi(e) != 0;
    c.fused_grid = 0;
    if (c.world == 1 && c.R <= 2048) {
        c.fused_wv = c.WV;
        if (const char* e = std::getenv("TG_PLANE_LOOP")) if (std::atoi(e)) c.fused_wv = 0;
        const void* fn = plane_rounds_fn(c.cfg.rule, c.fused_wv, c.fused_fast);
        c.fused_block = c.fused_fast ? kPlaneThreadsFast : kPlaneThreads;
        const size_t pf_words = c.fused_fast && (c.fused_wv == 4 || c.fused_wv == 2)
                                    ? (size_t)2 * (5 * 32 * c.fused_wv + 4 * 32) : 0;
        const size_t tail_words = c.fused_fast && (c.fused_wv == 4 || c.fused_wv == 2)
                                      ? 0 : std::max<size_t>(kTailCap * 7, (size_t)2 * c.W * 32);
        c.fused_smem = (size_t)c.R * (2 * sizeof(double) + 2 * sizeof(int32_t)) + 8 +
                       (size_t)(c.fused_block / 32) * std::max(pf_words, tail_words) * sizeof(int32_t);
        if (c.fused_smem > 48 * 1024)
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.fused_smem));
        int fb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fb, fn, c.fused_block, c.fused_smem));
        if (fb >= 1) {
            int g = fb * c.sms;
            const int fp = c.fused_wv ? passes : 1;
            g -= g % fp;
            if (g >= fp) c.fused_grid = g;
        }
    }
}

void build_slot(tg_ctx& c) {
    ensure_host_arrays(c);
    ensure_host_canonical(c);
    cudaStream_t st = c.stream;
    const int n = c.n;
    if (n > 200 * 1024) fail(TG_ERR_RESOURCE, "slot engine: %d spins exceed shared memory", n);
    // merged adjacency (cost weight J, chain multiplicity) in increasing
    // neighbour order, like the reference's merged CSR (constraints.cpp:122-140)
    struct E { uint64_t key; double w; int cm; };
    std::vector<E> ent;
    ent.reserve(2 * (c.ci.size() + c.pa.size()));
    for (size_t k = 0; k < c.ci.size(); ++k) {
        const uint64_t x = (uint64_t)c.inv[c.ci[k]], y = (uint64_t)c.inv[c.cj[k]];
        ent.push_back({x << 32 | y, c.cw[k], 0});
        ent.push_back({y << 32 | x, c.cw[k], 0});
    }
    for (size_t k = 0; k < c.pa.size(); ++k) {
        const uint64_t x = (uint64_t)c.inv[c.pa[k]], y = (uint64_t)c.inv[c.pb[k]];
        ent.push_back({x << 32 | y, 0.0, 1});
        ent.push_back({y << 32 | x, 0.0, 1});
    }
    std::stable_sort(ent.begin(), ent.end(), [](const E& p, const E& q) { return p.key < q.key; });
    std::vector<int> off(n + 1, 0);
    std::vector<int32_t> nbr;
    std::vector<double> w;
    std::vector<int8_t> cm;
    for (size_t k = 0; k < ent.size();) {
        size_t q = k;
        double wsum = 0.0;
        int csum = 0;
        while (q < ent.size() && ent[q].key == ent[k].key) { wsum += ent[q].w; csum += ent[q].cm; ++q; }
        const int i = (int)(ent[k].key >> 32);
        nbr.push_back((int32_t)(ent[k].key & 0xffffffffu));
        w.push_back(wsum);
        cm.push_back((int8_t)csum);
        off[i + 1]++;
        k = q;
    }
    for (int i = 0; i < n; ++i) off[i + 1] += off[i];
    std::vector<double> hi(n);
    for (int i = 0; i < n; ++i) hi[i] = c.h[c.order[i]];
    // FP32 fast-path tables and the bound on |local_fp32 - local_fp64|
    if (n >= (1 << 28)) fail(TG_ERR_RESOURCE, "slot engine: too many spins for the packed CSR");
    std::vector<int2> ent2(nbr.size());
    std::vector<float> h32(n);
    double pmax = 0.0, bmax = 0.0, eps = 0.0;
    for (double p : c.pens) pmax = std::max(pmax, p);
    for (double b : c.betas) bmax = std::max(bmax, std::fabs(b));
    for (int i = 0; i < n; ++i) {
        h32[i] = (float)hi[i];
        double S = std::fabs(hi[i]);
        for (int e = off[i]; e < off[i + 1]; ++e) {
            const float wf = (float)w[e];
            int bits;
            std::memcpy(&bits, &wf, 4);
            ent2[e] = make_int2(nbr[e] | ((int)cm[e] << 28), bits);
            S += std::fabs(w[e]) + (double)cm[e] * 2.0 * pmax;
        }
        eps = std::max(eps, (double)(off[i + 1] - off[i] + 3) * S * 0x1.0p-22);
    }
    // padded fixed-degree copy (D = 4 or 8) for the unrolled kernel
    int maxdeg = 0;
    for (int i = 0; i < n; ++i) maxdeg = std::max(maxdeg, off[i + 1] - off[i]);
    c.slot_D = maxdeg <= 4 ? 4 : (maxdeg <= 8 ? 8 : 0);
    if (n >= (1 << 27)) c.slot_D = 0;
    if (const char* e = std::getenv("TG_SLOT_GENERAL")) if (std::atoi(e)) c.slot_D = 0;
    if (c.slot_D) {
        const int D = c.slot_D;
        std::vector<int2> entp((size_t)n * D);
        std::vector<double> wp((size_t)n * D, 0.0);
        for (int i = 0; i < n; ++i) {
            for (int k = 0; k < D; ++k) entp[(size_t)i * D + k] = make_int2(i, 0);  // pad: w = 0
            for (int e = off[i]; e < off[i + 1]; ++e) {
                const int k = e - off[i];
                int2 v = ent2[e];
                if (nbr[e] > i) v.x |= 1 << 27;  // forward edge, counted once in (f, g)
                entp[(size_t)i * D + k] = v;
                wp[(size_t)i * D + k] = w[e];
            }
        }
        c.d_entp.upload(entp, st);
        c.d_wp.upload(wp, st);
    }
    c.slot_eps = (float)(eps * 1.0001 + 1e-30);
    c.slot_beta_max = (float)(bmax * 1.0001);
    c.d_ent.upload(ent2, st);
    c.d_h32.upload(h32, st);
    std::vector<uint64_t> keys(c.R);
    for (int r = 0; r < c.R; ++r) keys[r] = derive_seed(c.cfg.seed, kPurposeReplica, (uint64_t)r);
    c.d_off.upload(off, st);
    c.d_snbr.upload(nbr, st);
    c.d_sw.upload(w, st);
    c.d_cm.upload(cm, st);
    c.d_h.upload(hi, st);
    c.d_color_start.upload(c.color_start, st);
    c.d_slot_key.upload(keys, st);
    c.d_spins8.alloc((size_t)c.R_local * n);
    c.slot_smem = (size_t)n;
    CK(cudaFuncSetAttribute((const void*)slot_sweep_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)std::max<size_t>(c.slot_smem, 48 * 1024)));
    if (c.slot_D)
        CK(cudaFuncSetAttribute(slot_sweep_fn_d(c.slot_D), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(c.slot_smem, 48 * 1024)));
}

PlaneArgs plane_args(tg_ctx& c) {
    PlaneArgs a{};
    a.n = c.n;
    a.W = c.W;
    a.n_colors = c.n_colors;
    a.local_states = c.R_local;
    a.rule = c.cfg.rule;
    a.n_types = c.n_types;
    a.kpw = c.kpw;
    a.m_cost = c.m_cost;
    a.spins = c.d_spins32.p;
    a.nbr = c.d_nbr.p;
    a.chunks = c.d_chunks.p;
    a.chunk_off = c.d_chunk_off.p;
    a.color_start = c.d_color_start.p;
    for (int q = 0; q < c.n_types && q < kMaxTypes; ++q) a.ty[q] = c.h_types[q];
    for (int w = 0; w < c.W && w < kMaxWordsArg; ++w) a.active[w] = c.h_active[w];
    philox_key_schedule(derive_seed(c.cfg.seed, kPurposePlane, 0), a.pks);
    a.state_slot = c.d_state_slot.p;
    a.ktab = c.d_ktab.p;
    a.ktab_row = c.ktab_row;
    a.w_global0 = c.state0 / 32;
    a.kp = c.d_kp.p;
    a.kpc = c.d_kpc.p;
    a.cnt_c = c.d_cnt_c.p;
    a.cnt_q = c.d_cnt_q.p;
    a.f_loc = c.d_f.p + c.state0;
    a.g_loc = c.d_g.p + c.state0;
    return a;
}

SlotArgs slot_args(tg_ctx& c) {
    SlotArgs a{};
    a.n = c.n;
    a.n_colors = c.n_colors;
    a.local_states = c.R_local;
    a.state0 = c.state0;
    a.rule = c.cfg.rule;
    a.I = c.I;
    a.J = c.J;
    a.spins = c.d_spins8.p;
    a.off = c.d_off.p;
    a.nbr = c.d_snbr.p;
    a.w = c.d_sw.p;
    a.cm = c.d_cm.p;
    a.h = c.d_h.p;
    a.ent = c.d_ent.p;
    a.entp = c.d_entp.p;
    a.wp = c.d_wp.p;
    a.D = c.slot_D;
    a.h32 = c.d_h32.p;
    a.eps_local = c.slot_eps;
    a.beta_max = c.slot_beta_max;
    a.color_start = c.d_color_start.p;
    a.betas = c.d_betas.p;
    a.pens = c.d_pens.p;
    a.state_slot = c.d_state_slot.p;
    a.slot_key = c.d_slot_key.p;
    a.f_loc = c.d_f.p + c.state0;
    a.g_loc = c.d_g.p + c.state0;
    return a;
}

SwapArgs swap_args(tg_ctx& c) {
    SwapArgs a{};
    a.I = c.I;
    a.J = c.J;
    a.R = c.R;
    a.betas = c.d_betas.p;
    a.pens = c.d_pens.p;
    a.f_all = c.d_f.p;
    a.g_all = c.d_g.p;
    a.slot_state = c.d_slot_state.p;
    a.state_slot = c.d_state_slot.p;
    a.acc_p = c.d_acc_p.p;
    a.acc_b = c.d_acc_b.p;
    a.swap_seed = derive_seed(c.cfg.seed, kPurposeSwap, 0);
    a.rec = c.d_rec.p;
    a.rec_cap = c.rec_cap;
    a.rec_acc = c.d_rec_acc.p;
    a.plane = c.engine == TG_ENGINE_PLANE;
    a.W = c.W;
    a.state0 = c.state0;
    a.local_states = c.R_local;
    a.n_types = c.n_types;
    a.kpw = c.kpw;
    a.types = c.d_types.p;
    a.ktab = c.d_ktab.p;
    a.ktab_row = c.ktab_row;
    a.kp = c.d_kp.p;
    a.kpc = c.d_kpc.p;
    return a;
}

void launch_sweep(tg_ctx& c, int64_t t0) {
    const int sps = (int)c.cfg.sweeps_per_swap;
    if (c.engine == TG_ENGINE_PLANE) {
        PlaneArgs a = plane_args(c);
        int64_t t = t0;
        int nsw = sps;
        void* args[] = {&a, &t, &nsw};
        CK(cudaLaunchCooperativeKernel(plane_sweep_fn(c.cfg.rule, c.WV), dim3(c.plane_grid),
                                       dim3(kPlaneThreads), args, 0, c.stream));
    } else {
        SlotArgs a = slot_args(c);
        int64_t t = t0;
        int nsw = sps;
        void* args[] = {&a, &t, &nsw};
        CK(cudaLaunchKernel(c.slot_D ? slot_sweep_fn_d(c.slot_D) : slot_sweep_fn(), dim3(c.R_local),
                            dim3(kSlotThreads), args, c.slot_smem, c.stream));
    }
    c.sweep_launches++;
}

// Labels and thresholds for the current slot assignment: run the swap
// kernel's plane-rebuild with a round that attempts nothing.
void rebuild_planes(tg_ctx& c) {
    if (c.engine != TG_ENGINE_PLANE) return;
    SwapArgs a = swap_args(c);
    // round 1 of a 1x1-like schedule attempts nothing: fake I=J=1 for the swap part
    a.I = 1;
    a.J = 1;
    swap_kernel<<<1, kSwapThreads, 0, c.stream>>>(a, 1, 0, c.rec_cap, 0);
    CK(cudaGetLastError());
}

void s2_build(tg_ctx& c, const tg_run_config* cfg);

void do_init(tg_ctx& c, const tg_run_config* cfg) {
    HostTimer tm_("init (total)");
    if (!c.have_problem) fail(TG_ERR_CONFIG, "run: no problem set");
    if (!c.have_schedule) fail(TG_ERR_CONFIG, "run: no schedule set");
    if (cfg->sweeps_per_swap < 1) fail(TG_ERR_CONFIG, "run: sweeps_per_swap must be >= 1");
    if (cfg->total_sweeps < cfg->sweeps_per_swap)
        fail(TG_ERR_CONFIG, "run: total_sweeps must be >= sweeps_per_swap");
    if (cfg->rule != TG_RULE_METROPOLIS && cfg->rule != TG_RULE_HEAT_BATH)
        fail(TG_ERR_CONFIG, "run: unknown update rule %d", cfg->rule);
    c.cfg = *cfg;
    if (c.cfg.record_every < 1) c.cfg.record_every = 1;
    c.I = (int)c.betas.size();
    c.J = (int)c.pens.size();
    c.R = c.I * c.J;
    std::string why;
    int eng = cfg->engine;
    if (eng == TG_ENGINE_AUTO)
        eng = (!c.kl.on && plane_eligible(c, nullptr)) ? TG_ENGINE_PLANE : TG_ENGINE_SLOT;
    if (c.kl.on && (eng != TG_ENGINE_SLOT || c.world != 1 || std::getenv("TG_SLOT_V1")))
        fail(TG_ERR_CONFIG, "kl decoder: needs the single-GPU SLOT engine");
    if (eng == TG_ENGINE_PLANE && !plane_eligible(c, &why))
        fail(TG_ERR_CONFIG, "plane engine: instance not eligible (%s)", why.c_str());
    if (eng != TG_ENGINE_PLANE && eng != TG_ENGINE_SLOT) fail(TG_ERR_CONFIG, "unknown engine %d", eng);
    c.engine = eng;
    {
        int32_t s0 = 0, cnt = 0;
        if (tg_partition(c.R, c.rank, c.world, eng, &s0, &cnt) != TG_OK)
            fail(TG_ERR_CONFIG, "grid of %d replicas does not split over %d ranks%s", c.R, c.world,
                 eng == TG_ENGINE_PLANE ? " in 32-replica words" : "");
        c.state0 = s0;
        c.R_local = cnt;
    }
    cudaStream_t st = c.stream;
    CK(cudaSetDevice(c.device));
    c.use_s2 = false;
    if (eng == TG_ENGINE_SLOT && c.world == 1 && !std::getenv("TG_SLOT_V1")) {
        // single instance = batch of one on the replica-fastest SLOT engine
        BatchInst bi;
        ensure_host_arrays(c);
        bi.n = c.n; bi.ci = c.ci; bi.cj = c.cj; bi.pa = c.pa; bi.pb = c.pb;
        bi.cw = c.cw; bi.h = c.h; bi.betas = c.betas; bi.pens = c.pens; bi.seed = cfg->seed;
        c.batch.assign(1, bi);
        c.s2.probe = false;
        s2_build(c, &c.cfg);
        c.use_s2 = true;
        c.rounds_done = 0;
        c.initialised = true;
        return;
    }
    c.d_betas.upload(c.betas, st);
    c.d_pens.upload(c.pens, st);
    c.d_f.alloc(c.R);
    c.d_g.alloc(c.R);
    c.d_f.zero(st);
    c.d_g.zero(st);
    std::vector<int32_t> ident(c.R);
    for (int r = 0; r < c.R; ++r) ident[r] = r;
    c.d_slot_state.upload(ident, st);
    c.d_state_slot.upload(ident, st);
    if (c.dev_prep) c.d_perm.copy_from(c.d_order_dev, st);
    else c.d_perm.upload(c.order, st);
    const int np = c.I * std::max(0, c.J - 1), nb = std::max(0, c.I - 1) * c.J;
    c.d_acc_p.alloc(std::max(np, 1));
    c.d_acc_b.alloc(std::max(nb, 1));
    c.d_acc_p.zero(st);
    c.d_acc_b.zero(st);
    // record ring
    const int flags = c.cfg.record_flags;
    size_t per_state = (flags & TG_REC_GRID) ? (size_t)c.R * c.n : ((flags & TG_REC_STATE) ? (size_t)c.n : 0);
    int cap = 1024;
    if (per_state) cap = (int)std::max<size_t>(1, std::min<size_t>(1024, (size_t)(256u << 20) / per_state));
    c.rec_cap = cap;
    c.d_rec.alloc(cap + 1);  // +1: scratch entry for table rebuilds
    c.d_rec_acc.release();
    if (flags & TG_REC_COUNTERS) c.d_rec_acc.alloc((size_t)(cap + 1) * (np + nb + 1));
    c.d_rec_states.release();
    if (per_state) c.d_rec_states.alloc((size_t)cap * per_state);
    c.h_rec.resize(cap);
    c.h_states.resize((size_t)cap * per_state);
    c.h_acc.resize((flags & TG_REC_COUNTERS) ? (size_t)cap * (np + nb + 1) : 0);
    if (eng == TG_ENGINE_PLANE) build_plane(c); else build_slot(c);
    // initial configurations (engine.cpp:98-106)
    if (eng == TG_ENGINE_PLANE) {
        plane_init_kernel<<<c.sms * 4, 256, 0, st>>>(c.d_spins32.p, c.n, c.W, c.R_local, c.state0, c.cfg.seed);
    } else {
        slot_init_kernel<<<c.sms * 4, 256, 0, st>>>(c.d_spins8.p, c.n, c.R_local, c.state0, c.cfg.seed);
    }
    CK(cudaGetLastError());
    rebuild_planes(c);
    c.rounds_done = 0;
    c.swap_base = 0;
    c.initialised = true;
    CK(cudaStreamSynchronize(st));
}

struct SinkCtx {
    tg_sink_fn fn;
    void* user;
};

struct BatchSinkCtx {
    tg_batch_sink_fn fn;
    void* user;
};

void s2_build(tg_ctx& c, const tg_run_config* cfg);
void s2_advance(tg_ctx& c, int64_t n_rounds, const BatchSinkCtx& sink);

void drain(tg_ctx& c, int filled, int64_t first_round, const SinkCtx& sink) {
    if (filled <= 0) return;
    cudaStream_t st = c.stream;
    CK(cudaMemcpyAsync(c.h_rec.data(), c.d_rec.p, sizeof(TgRecordDev) * filled, cudaMemcpyDeviceToHost, st));
    const int flags = c.cfg.record_flags;
    const size_t per_state = (flags & TG_REC_GRID) ? (size_t)c.R * c.n : ((flags & TG_REC_STATE) ? (size_t)c.n : 0);
    if (per_state)
        CK(cudaMemcpyAsync(c.h_states.data(), c.d_rec_states.p, per_state * filled, cudaMemcpyDeviceToHost, st));
    const int np = c.I * std::max(0, c.J - 1), nb = std::max(0, c.I - 1) * c.J;
    if (flags & TG_REC_COUNTERS)
        CK(cudaMemcpyAsync(c.h_acc.data(), c.d_rec_acc.p, sizeof(int64_t) * (size_t)filled * (np + nb),
                           cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!sink.fn) return;
    // split counters into P / beta arrays
    std::vector<int64_t> ap((size_t)filled * np), ab((size_t)filled * nb);
    if (flags & TG_REC_COUNTERS)
        for (int k = 0; k < filled; ++k) {
            std::copy_n(c.h_acc.data() + (size_t)k * (np + nb), np, ap.data() + (size_t)k * np);
            std::copy_n(c.h_acc.data() + (size_t)k * (np + nb) + np, nb, ab.data() + (size_t)k * nb);
        }
    std::vector<tg_record> out;
    std::vector<int8_t> outs;
    std::vector<int64_t> oap, oab;
    for (int k = 0; k < filled; ++k) {
        const int64_t round = first_round + k;
        if (round % c.cfg.record_every != 0) continue;
        const TgRecordDev& d = c.h_rec[k];
        tg_record r;
        r.round = round;
        r.sweep_count = round * c.cfg.sweeps_per_swap;
        r.f = d.f;
        r.g = d.g;
        r.feasible = d.feasible;
        r.target_state = d.target_state;
        r.digest = d.digest;
        out.push_back(r);
        if (per_state) outs.insert(outs.end(), c.h_states.begin() + (size_t)k * per_state,
                                   c.h_states.begin() + (size_t)(k + 1) * per_state);
        if (flags & TG_REC_COUNTERS) {
            oap.insert(oap.end(), ap.begin() + (size_t)k * np, ap.begin() + (size_t)(k + 1) * np);
            oab.insert(oab.end(), ab.begin() + (size_t)k * nb, ab.begin() + (size_t)(k + 1) * nb);
        }
    }
    if (out.empty()) return;
    const int rc = sink.fn(sink.user, out.data(), (int64_t)out.size(), per_state ? outs.data() : nullptr,
                           (flags & TG_REC_COUNTERS) ? oap.data() : nullptr,
                           (flags & TG_REC_COUNTERS) ? oab.data() : nullptr);
    if (rc) fail(TG_ERR_SINK, "record sink requested stop at round %lld", (long long)(first_round + filled - 1));
}

// Device time of the sweep launches and of everything between them for the
// `filled` rounds of the current chunk (events recorded without host syncs).
void profile_chunk(tg_ctx& c, int filled, double& sweep_ms, double& other_ms) {
    CK(cudaEventRecord(c.ev[2 * filled], c.stream));
    CK(cudaEventSynchronize(c.ev[2 * filled]));
    for (int k = 0; k < filled; ++k) {
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, c.ev[2 * k], c.ev[2 * k + 1]));
        CK(cudaEventElapsedTime(&b, c.ev[2 * k + 1], c.ev[2 * k + 2]));
        sweep_ms += a;
        other_ms += b;
    }
}

// Single-GPU plane engine: whole rounds inside one persistent kernel per
// record chunk (no host round trip, no separate swap launch).
void do_advance_fused(tg_ctx& c, int64_t n_rounds, const SinkCtx& sink) {
    cudaStream_t st = c.stream;
    const int flags = c.cfg.record_flags;
    if (c.profiling && c.ev.size() < 2) {
        for (auto e : c.ev) cudaEventDestroy(e);
        c.ev.assign(2, nullptr);
        for (auto& e : c.ev) CK(cudaEventCreate(&e));
    }
    double sweep_ms = 0;
    int64_t left = n_rounds;
    while (left > 0) {
        const int n = (int)std::min<int64_t>(left, c.rec_cap);
        CK(cudaMemsetAsync(c.d_rec.p, 0, sizeof(TgRecordDev) * n, st));
        PlaneArgs a = plane_args(c);
        RoundArgs r{};
        r.I = c.I; r.J = c.J; r.R = c.R; r.sps = (int)c.cfg.sweeps_per_swap;
        r.round0 = c.rounds_done + 1;
        r.n_rounds = n;
        r.rec_flags = flags & (TG_REC_DIGEST | TG_REC_STATE | TG_REC_COUNTERS);
        r.swap_base0 = c.swap_base;
        r.swap_seed = derive_seed(c.cfg.seed, kPurposeSwap, 0);
        r.betas = c.d_betas.p; r.pens = c.d_pens.p;
        r.slot_state = c.d_slot_state.p; r.state_slot = c.d_state_slot.p;
        r.acc_p = c.d_acc_p.p; r.acc_b = c.d_acc_b.p;
        r.f_all = c.d_f.p; r.g_all = c.d_g.p;
        r.cnt = c.d_cnt2.p; r.cnt_stride = c.W * 32;
        // dynamic chunk grabbing measured 3% slower than the static split (r1); opt in
        r.work = (std::getenv("TG_PLANE_DYNAMIC") ? c.d_work.p : nullptr);
        r.ktab = c.d_ktab.p; r.ktab_row = c.ktab_row; r.kp = c.d_kp.p; r.kpc = c.d_kpc.p;
        r.rec = c.d_rec.p; r.rec_acc = c.d_rec_acc.p;
        r.rec_states = (flags & TG_REC_STATE) ? c.d_rec_states.p : nullptr;
        r.perm = c.d_perm.p;
        void* args[] = {&a, &r};
        if (c.profiling) CK(cudaEventRecord(c.ev[0], st));
        CK(cudaLaunchCooperativeKernel(plane_rounds_fn(c.cfg.rule, c.fused_wv, c.fused_fast),
                                       dim3(c.fused_grid), dim3(c.fused_block), args, c.fused_smem, st));
        if (c.profiling) CK(cudaEventRecord(c.ev[1], st));
        c.sweep_launches++;
        const int64_t first = c.rounds_done + 1;
        for (int k = 0; k < n; ++k) c.swap_base += (uint64_t)round_attempts(c.I, c.J, first + k);
        c.rounds_done += n;
        left -= n;
        drain(c, n, first, sink);
        if (c.profiling) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
            sweep_ms += ms;
        }
    }
    CK(cudaStreamSynchronize(st));
    c.last_sweep_ms = sweep_ms;
    c.last_swap_ms = 0;
}

int single_sink_adapter(void* user, int32_t, const tg_record* recs, int64_t n, const int8_t* st,
                        const int64_t* ap, const int64_t* ab) {
    const SinkCtx* sc = static_cast<const SinkCtx*>(user);
    return sc->fn ? sc->fn(sc->user, recs, n, st, ap, ab) : 0;
}

void do_advance(tg_ctx& c, int64_t n_rounds, const SinkCtx& sink) {
    if (!c.initialised) fail(TG_ERR_CONFIG, "advance: context not initialised (tg_init)");
    if (c.use_s2) {
        SinkCtx sc = sink;
        s2_advance(c, n_rounds, BatchSinkCtx{sink.fn ? &single_sink_adapter : nullptr, &sc});
        c.rounds_done = c.s2.rounds_done;
        return;
    }
    if (c.engine == TG_ENGINE_PLANE && c.world == 1 && c.fused_grid > 0 &&
        !(c.cfg.record_flags & TG_REC_GRID)) {
        do_advance_fused(c, n_rounds, sink);
        return;
    }
    cudaStream_t st = c.stream;
    const int flags = c.cfg.record_flags;
    const bool need_extract = (flags & (TG_REC_DIGEST | TG_REC_STATE | TG_REC_GRID)) != 0;
    const size_t per_state = (flags & TG_REC_GRID) ? (size_t)c.R * c.n : ((flags & TG_REC_STATE) ? (size_t)c.n : 0);
    SwapArgs sa = swap_args(c);
    const int sps = (int)c.cfg.sweeps_per_swap;
    if (c.profiling && (int)c.ev.size() < 2 * c.rec_cap + 1) {
        for (auto e : c.ev) cudaEventDestroy(e);
        c.ev.assign(2 * c.rec_cap + 1, nullptr);
        for (auto& e : c.ev) CK(cudaEventCreate(&e));
    }
    double sweep_ms = 0, swap_ms = 0;
    int filled = 0;
    int64_t first_round = c.rounds_done + 1;
    for (int64_t k = 0; k < n_rounds; ++k) {
        const int64_t round = c.rounds_done + 1;
        if (c.profiling) CK(cudaEventRecord(c.ev[2 * filled], st));
        launch_sweep(c, (round - 1) * sps);
        if (c.profiling) CK(cudaEventRecord(c.ev[2 * filled + 1], st));
        if (c.world > 1) {
            NK(nccl().GroupStart());
            NK(nccl().AllGather(c.d_f.p + c.state0, c.d_f.p, c.R_local, ncclDouble, c.comm, st));
            NK(nccl().AllGather(c.d_g.p + c.state0, c.d_g.p, c.R_local, ncclDouble, c.comm, st));
            NK(nccl().GroupEnd());
        }
        swap_kernel<<<1, kSwapThreads, 0, st>>>(sa, round, c.swap_base, filled, flags);
        CK(cudaGetLastError());
        c.other_launches++;
        if (need_extract) {
            ExtractArgs e{};
            e.n = c.n;
            e.R = c.R;
            e.W = c.W;
            e.plane = c.engine == TG_ENGINE_PLANE;
            e.all_slots = (flags & TG_REC_GRID) ? 1 : 0;
            e.local_states = c.R_local;
            e.state0 = c.state0;
            e.slot_state = c.d_slot_state.p;
            e.spins32 = c.d_spins32.p;
            e.spins8 = c.d_spins8.p;
            e.perm = c.d_perm.p;
            e.states = per_state ? c.d_rec_states.p + (size_t)filled * per_state : nullptr;
            uint64_t* dg = (flags & TG_REC_DIGEST) ? &c.d_rec.p[filled].digest : nullptr;
            e.digest = dg;
            const long long total = (long long)(e.all_slots ? c.R : 1) * c.n;
            const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)c.sms * 8);
            extract_kernel<<<std::max(blocks, 1), 256, 0, st>>>(e);
            CK(cudaGetLastError());
            c.other_launches++;
            if (c.world > 1) {
                if (dg) NK(nccl().AllReduce(dg, dg, 1, ncclUint64, ncclSum, c.comm, st));
                if (e.states) NK(nccl().AllReduce(e.states, e.states, per_state, ncclInt8, ncclSum, c.comm, st));
            }
        }
        c.swap_base += (uint64_t)round_attempts(c.I, c.J, round);
        c.rounds_done = round;
        ++filled;
        if (filled == c.rec_cap) {
            if (c.profiling) profile_chunk(c, filled, sweep_ms, swap_ms);
            drain(c, filled, first_round, sink);
            filled = 0;
            first_round = c.rounds_done + 1;
        }
    }
    if (c.profiling && filled) profile_chunk(c, filled, sweep_ms, swap_ms);
    drain(c, filled, first_round, sink);
    CK(cudaStreamSynchronize(st));
    c.last_sweep_ms = sweep_ms;
    c.last_swap_ms = swap_ms;
}

// ------------------------------------------------ SLOT engine v2 (host side)

// One instance prepared for the device: canonical order, merged CSR (FP64
// fallback), padded degree-D entries (FP32 fast path + forward-edge flags),
// and the FP32 error bound (see kernels.cu slot_update_fast).
// Error bands of the certified FP32 decision path (slot_engine.cu s2_update)
// for fields bounded by |h| + sum |w| + 2 pmax * chain multiplicity at
// inverse temperatures up to bmax.
void s2_bands(S2Prep& P, double bmax, double pmax) {
    double eps = 0.0;
    for (int i = 0; i < P.n; ++i) {
        double S = std::fabs(P.h[i]);
        for (int e = P.off[i]; e < P.off[i + 1]; ++e)
            S += std::fabs(P.w[e]) + (double)P.cm[e] * 2.0 * pmax;
        eps = std::max(eps, (double)(P.off[i + 1] - P.off[i] + 3) * S * 0x1.0p-22);
    }
    P.eps = (float)(eps * 1.0001 + 1e-30);
    P.beta_max = (float)(bmax * 1.0001);
}

void s2_prepare(S2Prep& P, const BatchInst& bi) {
    const int n = bi.n;
    P.n = n;
    canonical(n, bi.ci, bi.cj, bi.pa, bi.pb, P.order, P.color, P.n_colors);
    P.inv.assign(n, 0);
    for (int k = 0; k < n; ++k) P.inv[P.order[k]] = k;
    P.color_start.assign(P.n_colors + 1, 0);
    for (int k = 0; k < n; ++k) P.color_start[P.color[P.order[k]] + 1]++;
    for (int q = 0; q < P.n_colors; ++q) P.color_start[q + 1] += P.color_start[q];
    struct E { uint64_t key; double w; int cm; };
    std::vector<E> ent;
    ent.reserve(2 * (bi.ci.size() + bi.pa.size()));
    for (size_t k = 0; k < bi.ci.size(); ++k) {
        const uint64_t x = (uint64_t)P.inv[bi.ci[k]], y = (uint64_t)P.inv[bi.cj[k]];
        ent.push_back({x << 32 | y, bi.cw[k], 0});
        ent.push_back({y << 32 | x, bi.cw[k], 0});
    }
    for (size_t k = 0; k < bi.pa.size(); ++k) {
        const uint64_t x = (uint64_t)P.inv[bi.pa[k]], y = (uint64_t)P.inv[bi.pb[k]];
        ent.push_back({x << 32 | y, 0.0, 1});
        ent.push_back({y << 32 | x, 0.0, 1});
    }
    std::stable_sort(ent.begin(), ent.end(), [](const E& p, const E& q) { return p.key < q.key; });
    P.off.assign(n + 1, 0);
    P.nbr.clear(); P.w.clear(); P.cm.clear();
    for (size_t k = 0; k < ent.size();) {
        size_t q = k;
        double ws = 0.0;
        int cs = 0;
        while (q < ent.size() && ent[q].key == ent[k].key) { ws += ent[q].w; cs += ent[q].cm; ++q; }
        P.nbr.push_back((int32_t)(ent[k].key & 0xffffffffu));
        P.w.push_back(ws);
        P.cm.push_back((int8_t)cs);
        P.off[(int)(ent[k].key >> 32) + 1]++;
        k = q;
    }
    for (int i = 0; i < n; ++i) P.off[i + 1] += P.off[i];
    int maxdeg = 0;
    for (int i = 0; i < n; ++i) maxdeg = std::max(maxdeg, P.off[i + 1] - P.off[i]);
    if (maxdeg > 16) fail(TG_ERR_RESOURCE, "slot engine: merged degree %d > 16", maxdeg);
    if (n >= (1 << 27)) fail(TG_ERR_RESOURCE, "slot engine: %d spins exceed the packed index", n);
    P.D = maxdeg <= 4 ? 4 : (maxdeg <= 8 ? 8 : 16);
    double pmax = 0.0, bmax = 0.0;
    for (double p : bi.pens) pmax = std::max(pmax, p);
    for (double b : bi.betas) bmax = std::max(bmax, std::fabs(b));
    P.h.resize(n);
    P.h32.resize(n);
    P.entp.assign((size_t)n * P.D, make_int2(0, 0));
    P.wp.assign((size_t)n * P.D, 0.0);
    for (int i = 0; i < n; ++i) {
        P.h[i] = bi.h[P.order[i]];
        P.h32[i] = (float)P.h[i];
        for (int k = 0; k < P.D; ++k) P.entp[(size_t)i * P.D + k] = make_int2(i, 0);  // pad: weight 0
        for (int e = P.off[i]; e < P.off[i + 1]; ++e) {
            const float wf = (float)P.w[e];
            int bits;
            std::memcpy(&bits, &wf, 4);
            int x = P.nbr[e] | ((int)P.cm[e] << 28);
            if (P.nbr[e] > i) x |= 1 << 27;
            P.entp[(size_t)i * P.D + (e - P.off[i])] = make_int2(x, bits);
            P.wp[(size_t)i * P.D + (e - P.off[i])] = P.w[e];
        }
    }
    s2_bands(P, bmax, pmax);
}

S2Args s2_args(tg_ctx& c) {
    Slot2& S = c.s2;
    S2Args a{};
    a.B = S.B; a.I = S.I; a.J = S.J; a.R = S.R; a.Rp = S.Rp; a.G = S.G;
    a.rule = S.cfg.rule; a.max_colors = S.max_colors;
    a.inst = S.d_inst.p; a.spins = S.d_spins.p; a.entp = S.d_entp.p; a.wp = S.d_wp.p;
    a.off = S.d_off.p; a.nbr = S.d_nbr.p; a.w = S.d_w.p; a.cm = S.d_cm.p;
    a.h = S.d_h.p; a.h32 = S.d_h32.p; a.color_start = S.d_cstart.p;
    a.item_pref = S.d_item_pref.p; a.energy_pref = S.d_energy_pref.p;
    a.betas = S.d_betas.p; a.pens = S.d_pens.p; a.state_slot = S.d_state_slot.p;
    a.slot_key = S.d_keys.p; a.part_f = S.d_part_f.p; a.part_g = S.d_part_g.p;
    a.f = S.d_f.p; a.g = S.d_g.p;
    a.sbeta = S.d_sbeta.p; a.stwop = S.d_stwop.p; a.skey = S.d_skey.p; a.nsub = S.nsub;
    return a;
}

KLArgs kl_args(tg_ctx& c) {
    Slot2& S = c.s2;
    KLArgs k{};
    k.n_logical = c.kl.n_logical;
    k.K = 1 << c.kl.n_logical;
    k.discard = c.kl.discard;
    k.ncopies = (int)c.kl.copies.size();
    k.map_off = S.d_kl_off.p;
    k.map = S.d_kl_map.p;
    k.p = S.d_kl_p.p;
    k.hist = S.d_kl_hist.p;
    k.total = S.d_kl_total.p;
    k.kl = S.d_kl.p;
    k.samples = S.d_kl_samples.p;
    k.cap = S.kl_cap;
    k.error = S.d_kl_err.p;
    return k;
}

S2Swap s2_swap(tg_ctx& c) {
    Slot2& S = c.s2;
    S2Swap s{};
    s.R = S.R; s.I = S.I; s.J = S.J; s.rec_cap = S.rec_cap;
    s.betas = S.d_betas.p; s.pens = S.d_pens.p; s.f = S.d_f.p; s.g = S.d_g.p;
    s.slot_state = S.d_slot_state.p; s.state_slot = S.d_state_slot.p;
    s.acc_p = S.d_acc_p.p; s.acc_b = S.d_acc_b.p; s.swap_seed = S.d_swap_seed.p;
    s.rec = S.d_rec.p; s.rec_acc = S.d_rec_acc.p; s.rec_states = S.d_rec_states.p;
    s.perm = S.d_perm.p;
    s.sbeta = S.d_sbeta.p; s.stwop = S.d_stwop.p; s.skey = S.d_skey.p;
    s.slot_key = S.d_keys.p; s.Rp = S.Rp;
    return s;
}

void s2_build(tg_ctx& c, const tg_run_config* cfg) {
    Slot2& S = c.s2;
    cudaStream_t st = c.stream;
    const int B = (int)c.batch.size();
    if (B < 1) fail(TG_ERR_CONFIG, "batch: no instances");
    S.B = B;
    S.I = (int)c.batch[0].betas.size();
    S.J = (int)c.batch[0].pens.size();
    for (const auto& bi : c.batch)
        if ((int)bi.betas.size() != S.I || (int)bi.pens.size() != S.J)
            fail(TG_ERR_CONFIG, "batch: every instance needs the same I x J grid shape");
    S.R = S.I * S.J;
    S.Rp = (S.R + 31) / 32 * 32;
    S.G = S.Rp / 32;
    S.cfg = *cfg;
    if (S.cfg.record_every < 1) S.cfg.record_every = 1;
    S.prep.assign(B, S2Prep{});
    S.state_off.clear();
    for (int b = 0; b < B; ++b) {
        const BatchInst& x = c.batch[b];
        const BatchInst* y = b ? &c.batch[b - 1] : nullptr;
        if (y && x.n == y->n && x.ci == y->ci && x.cj == y->cj && x.cw == y->cw && x.h == y->h &&
            x.pa == y->pa && x.pb == y->pb)
            S.prep[b] = S.prep[b - 1];  // repeats of one instance (J-column baseline)
        else
            s2_prepare(S.prep[b], x);
    }
    int D = 4;
    for (const auto& P : S.prep) D = std::max(D, P.D);
    S.D = D;
    // concatenate
    std::vector<SInst> inst(B);
    std::vector<int2> entp;
    std::vector<double> wp, w, h, betas, pens;
    std::vector<int> off, cstart, perm;
    std::vector<int32_t> nbr;
    std::vector<int8_t> cm;
    std::vector<float> h32;
    std::vector<uint64_t> keys((size_t)B * S.R), swap_seed(B), seeds(B);
    long long spin_off = 0;
    int chunk_off = 0, state_off = 0, max_colors = 0;
    for (int b = 0; b < B; ++b) {
        S2Prep& P = S.prep[b];
        SInst& in = inst[b];
        in.n = P.n;
        in.D = D;
        in.n_colors = P.n_colors;
        in.color_off = (int)cstart.size();
        cstart.insert(cstart.end(), P.color_start.begin(), P.color_start.end());
        in.spin_off = spin_off;
        spin_off += (long long)P.n * S.Rp;
        in.entp_off = (int)entp.size();
        for (int i = 0; i < P.n; ++i)
            for (int k = 0; k < D; ++k) {
                entp.push_back(k < P.D ? P.entp[(size_t)i * P.D + k] : make_int2(i, 0));
                wp.push_back(k < P.D ? P.wp[(size_t)i * P.D + k] : 0.0);
            }
        in.csr_off = (int)off.size();
        off.insert(off.end(), P.off.begin(), P.off.end());
        in.nbr_off = (int)nbr.size();
        nbr.insert(nbr.end(), P.nbr.begin(), P.nbr.end());
        w.insert(w.end(), P.w.begin(), P.w.end());
        cm.insert(cm.end(), P.cm.begin(), P.cm.end());
        in.h_off = (int)h.size();
        h.insert(h.end(), P.h.begin(), P.h.end());
        h32.insert(h32.end(), P.h32.begin(), P.h32.end());
        perm.insert(perm.end(), P.order.begin(), P.order.end());
        in.n_chunks = (P.n + 31) / 32;
        in.chunk_off = chunk_off;
        chunk_off += in.n_chunks;
        in.state_off = state_off;
        S.state_off.push_back(state_off);
        state_off += P.n;
        in.eps = P.eps;
        in.beta_max = P.beta_max;
        max_colors = std::max(max_colors, P.n_colors);
        betas.insert(betas.end(), c.batch[b].betas.begin(), c.batch[b].betas.end());
        pens.insert(pens.end(), c.batch[b].pens.begin(), c.batch[b].pens.end());
        seeds[b] = c.batch[b].seed;
        for (int r = 0; r < S.R; ++r)
            keys[(size_t)b * S.R + r] = S.probe ? derive_seed(c.batch[b].seed, kPurposeProbe, (uint64_t)r)
                                                : derive_seed(c.batch[b].seed, kPurposeReplica, (uint64_t)r);
        swap_seed[b] = derive_seed(c.batch[b].seed, kPurposeSwap, 0);
    }
    S.max_colors = max_colors;
    // item prefix tables: per colour, per instance, upper bound of Philox pairs x groups
    std::vector<int> item_pref((size_t)max_colors * (B + 1), 0), energy_pref(B + 1, 0);
    for (int col = 0; col < max_colors; ++col)
        for (int b = 0; b < B; ++b) {
            const S2Prep& P = S.prep[b];
            const int len = col < P.n_colors ? P.color_start[col + 1] - P.color_start[col] : 0;
            const int ub = len > 0 ? (len + 3) / 2 : 0;
            item_pref[(size_t)col * (B + 1) + b + 1] = item_pref[(size_t)col * (B + 1) + b] + ub;
        }
    for (int b = 0; b < B; ++b) energy_pref[b + 1] = energy_pref[b] + inst[b].n_chunks * S.G;
    S.d_inst.upload(inst, st);
    S.h_inst = inst;
    S.d_entp.upload(entp, st);
    S.d_wp.upload(wp, st);
    S.d_off.upload(off, st);
    S.d_nbr.upload(nbr, st);
    S.d_w.upload(w, st);
    S.d_cm.upload(cm, st);
    S.d_h.upload(h, st);
    S.d_h32.upload(h32, st);
    S.d_cstart.upload(cstart, st);
    S.d_item_pref.upload(item_pref, st);
    S.d_energy_pref.upload(energy_pref, st);
    S.d_betas.upload(betas, st);
    S.d_pens.upload(pens, st);
    S.d_keys.upload(keys, st);
    S.d_swap_seed.upload(swap_seed, st);
    S.d_seeds.upload(seeds, st);
    {   // init streams: engine.cpp:100-101 (purpose init, per replica), or for a
        // probe the chain's own stream from draw 0 (schedule.cpp:30-31)
        std::vector<uint64_t> ik((size_t)B * S.R);
        for (int b = 0; b < B; ++b)
            for (int r = 0; r < S.R; ++r)
                ik[(size_t)b * S.R + r] = S.probe ? keys[(size_t)b * S.R + r]
                                                  : derive_seed(c.batch[b].seed, kPurposeInit, (uint64_t)r);
        S.d_init_keys.upload(ik, st);
    }
    S.d_perm.upload(perm, st);
    S.d_spins.alloc((size_t)spin_off);
    // cooperative grid: whole warps per replica group
    {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, slot2_sweep_fn(S.D), kSlot2Threads, 0));
        if (per_sm < 1) fail(TG_ERR_RESOURCE, "slot engine: sweep kernel does not fit on an SM");
        int blocks = per_sm * c.sms;
        const int wpb = kSlot2Threads / 32;
        // no more warps than the widest colour phase can use (small instances)
        long long need = 0;
        for (int col = 0; col < max_colors; ++col)
            need = std::max<long long>(need, (long long)item_pref[(size_t)col * (B + 1) + B] * S.G);
        need = std::max<long long>(need, (long long)B * S.R);  // energy reduction: one warp per replica
        blocks = (int)std::min<long long>(blocks, (need + wpb - 1) / wpb);
        blocks = std::max(blocks, 1);
        while (blocks > 1 && (blocks * wpb) % S.G != 0) --blocks;
        if ((blocks * wpb) % S.G != 0) {  // round up instead (still co-resident if under the limit)
            blocks = (S.G + wpb - 1) / wpb * wpb / wpb;
            while ((blocks * wpb) % S.G != 0) ++blocks;
            if (blocks > per_sm * c.sms) fail(TG_ERR_RESOURCE, "slot engine: cannot tile %d replica groups", S.G);
        }
        S.grid = blocks;
        S.nsub = blocks * wpb / S.G;
    }
    // fused per-warp energy partials cost B x nsub x Rp doubles of traffic per
    // round; past a few MB a separate pass over the spins is cheaper
    S.sep_energy = (size_t)B * S.nsub * S.Rp * 16 > ((size_t)8 << 20) || std::getenv("TG_SLOT_SEP_ENERGY");
    if (S.sep_energy) {
        S.e_slices = std::max(1, (c.sms * 8) / std::max(1, B * S.G));
        S.d_epart.alloc((size_t)2 * B * S.e_slices * S.R);
    }
    S.d_part_f.alloc(S.sep_energy ? 0 : (size_t)B * S.nsub * S.Rp);
    S.d_part_g.alloc(S.sep_energy ? 0 : (size_t)B * S.nsub * S.Rp);
    S.d_part_f.zero(st);
    S.d_part_g.zero(st);
    {
        std::vector<double> sb((size_t)B * S.Rp, 0.0), stp((size_t)B * S.Rp, 0.0);
        std::vector<uint64_t> sk((size_t)B * S.Rp, 0);
        for (int b = 0; b < B; ++b)
            for (int r = 0; r < S.R; ++r) {
                sb[(size_t)b * S.Rp + r] = c.batch[b].betas[r / S.J];
                stp[(size_t)b * S.Rp + r] = 2.0 * c.batch[b].pens[r % S.J];
                sk[(size_t)b * S.Rp + r] = keys[(size_t)b * S.R + r];
            }
        S.d_sbeta.upload(sb, st);
        S.d_stwop.upload(stp, st);
        S.d_skey.upload(sk, st);
    }
    S.d_f.alloc((size_t)B * S.R);
    S.d_g.alloc((size_t)B * S.R);
    std::vector<int32_t> ident((size_t)B * S.R);
    for (int b = 0; b < B; ++b)
        for (int r = 0; r < S.R; ++r) ident[(size_t)b * S.R + r] = r;
    S.d_slot_state.upload(ident, st);
    S.d_state_slot.upload(ident, st);
    const int np = S.I * std::max(0, S.J - 1), nb = std::max(0, S.I - 1) * S.J;
    S.d_acc_p.alloc((size_t)B * std::max(np, 1));
    S.d_acc_b.alloc((size_t)B * std::max(nb, 1));
    S.d_acc_p.zero(st);
    S.d_acc_b.zero(st);
    // records
    const int flags = S.cfg.record_flags;
    S.slots = (flags & TG_REC_GRID) ? S.R : 1;
    const size_t per_round_states = (flags & (TG_REC_STATE | TG_REC_GRID)) ? (size_t)state_off * S.slots : 0;
    int cap = 1024;
    if (per_round_states) cap = (int)std::max<size_t>(1, std::min<size_t>(1024, (size_t)(256u << 20) / per_round_states));
    S.rec_cap = cap;
    S.d_rec.alloc((size_t)B * cap);
    S.d_rec_acc.release();
    if (flags & TG_REC_COUNTERS) S.d_rec_acc.alloc((size_t)B * cap * (np + nb + 1));
    S.d_rec_states.release();
    if (per_round_states) S.d_rec_states.alloc(per_round_states * cap);
    S.h_rec.resize((size_t)B * cap);
    S.h_acc.resize((flags & TG_REC_COUNTERS) ? (size_t)B * cap * (np + nb + 1) : 0);
    S.h_states.resize(per_round_states * cap);
    // decoded-sample KL observer
    S.kl_on = c.kl.on && !S.probe;
    if (S.kl_on) {
        const int nc = (int)c.kl.copies.size(), K = 1 << c.kl.n_logical;
        std::vector<int> map((size_t)B * nc);
        for (int b = 0; b < B; ++b)
            for (int q = 0; q < nc; ++q) {
                const int x = c.kl.copies[q];
                if (x < 0 || x >= S.prep[b].n) fail(TG_ERR_CONFIG, "kl decoder: copy %d out of range", x);
                map[(size_t)b * nc + q] = S.prep[b].inv[x];
            }
        S.d_kl_off.upload(c.kl.copy_off, st);
        S.d_kl_map.upload(map, st);
        S.d_kl_p.upload(c.kl.probs, st);
        S.d_kl_hist.alloc((size_t)B * K);
        S.d_kl_hist.zero(st);
        S.d_kl_total.alloc(B);
        S.d_kl_total.zero(st);
        S.kl_cap = std::max<int64_t>(1, cfg->total_sweeps / std::max<int64_t>(1, cfg->sweeps_per_swap));
        S.d_kl.alloc((size_t)B * S.kl_cap);
        S.d_kl_samples.alloc((size_t)B * S.kl_cap);
        S.d_kl_err.alloc(1);
        S.d_kl_err.zero(st);
    }
    // initial configurations (engine.cpp:98-106)
    S2Args a = s2_args(c);
    slot2_init_kernel<<<dim3(c.sms * 4, B), 256, 0, st>>>(a, S.d_init_keys.p);
    CK(cudaGetLastError());
    S.rounds_done = 0;
    S.swap_base = 0;
    S.ready = true;
    CK(cudaStreamSynchronize(st));
}

void s2_drain(tg_ctx& c, int filled, int64_t first_round, const BatchSinkCtx& sink) {
    Slot2& S = c.s2;
    if (filled <= 0) return;
    cudaStream_t st = c.stream;
    const int B = S.B, cap = S.rec_cap, flags = S.cfg.record_flags;
    const int np = S.I * std::max(0, S.J - 1), nb = std::max(0, S.I - 1) * S.J;
    CK(cudaMemcpy2DAsync(S.h_rec.data(), sizeof(TgRecordDev) * cap, S.d_rec.p, sizeof(TgRecordDev) * cap,
                         sizeof(TgRecordDev) * filled, B, cudaMemcpyDeviceToHost, st));
    if (flags & TG_REC_COUNTERS)
        CK(cudaMemcpy2DAsync(S.h_acc.data(), sizeof(int64_t) * cap * (np + nb), S.d_rec_acc.p,
                             sizeof(int64_t) * cap * (np + nb), sizeof(int64_t) * filled * (np + nb), B,
                             cudaMemcpyDeviceToHost, st));
    if (S.d_rec_states.p) CK(cudaMemcpyAsync(S.h_states.data(), S.d_rec_states.p, S.h_states.size(),
                                             cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!sink.fn) return;
    for (int b = 0; b < B; ++b) {
        const int n = S.prep[b].n;
        const size_t per = (size_t)n * S.slots;
        std::vector<tg_record> out;
        std::vector<int8_t> outs;
        std::vector<int64_t> oap, oab;
        for (int k = 0; k < filled; ++k) {
            const int64_t round = first_round + k;
            if (round % S.cfg.record_every != 0) continue;
            const TgRecordDev& d = S.h_rec[(size_t)b * cap + k];
            tg_record r;
            r.round = round;
            r.sweep_count = round * S.cfg.sweeps_per_swap;
            r.f = d.f; r.g = d.g; r.feasible = d.feasible; r.target_state = d.target_state;
            r.digest = d.digest;
            out.push_back(r);
            if (S.d_rec_states.p) {
                const int8_t* src = S.h_states.data() + (size_t)S.state_off[b] * S.slots * cap +
                                    (size_t)k * per;
                outs.insert(outs.end(), src, src + per);
            }
            if (flags & TG_REC_COUNTERS) {
                const int64_t* src = S.h_acc.data() + ((size_t)b * cap + k) * (np + nb);
                oap.insert(oap.end(), src, src + np);
                oab.insert(oab.end(), src + np, src + np + nb);
            }
        }
        if (out.empty()) continue;
        const int rc = sink.fn(sink.user, b, out.data(), (int64_t)out.size(),
                               S.d_rec_states.p ? outs.data() : nullptr,
                               (flags & TG_REC_COUNTERS) ? oap.data() : nullptr,
                               (flags & TG_REC_COUNTERS) ? oab.data() : nullptr);
        if (rc) fail(TG_ERR_SINK, "record sink requested stop (instance %d)", b);
    }
}

void s2_advance(tg_ctx& c, int64_t n_rounds, const BatchSinkCtx& sink) {
    Slot2& S = c.s2;
    if (!S.ready) fail(TG_ERR_CONFIG, "advance: batch not initialised");
    cudaStream_t st = c.stream;
    const int flags = S.cfg.record_flags;
    const int sps = (int)S.cfg.sweeps_per_swap;
    if (c.profiling && c.ev.size() < 2) {
        for (auto e : c.ev) cudaEventDestroy(e);
        c.ev.assign(2, nullptr);
        for (auto& e : c.ev) CK(cudaEventCreate(&e));
    }
    S2Args a = s2_args(c);
    S2Swap s = s2_swap(c);
    double sweep_ms = 0.0;
    int filled = 0;
    int64_t first = S.rounds_done + 1;
    for (int64_t k = 0; k < n_rounds; ++k) {
        const int64_t round = S.rounds_done + 1;
        int64_t t0 = (round - 1) * sps;
        int nsw = sps, de = S.sep_energy ? 0 : 1;
        void* args[] = {&a, &t0, &nsw, &de};
        if (c.profiling) CK(cudaEventRecord(c.ev[0], st));
        CK(cudaLaunchCooperativeKernel(slot2_sweep_fn(S.D), dim3(S.grid), dim3(kSlot2Threads), args, 0, st));
        if (c.profiling) CK(cudaEventRecord(c.ev[1], st));
        c.sweep_launches++;
        if (S.sep_energy) {
            slot2_energy_kernel<<<dim3(S.e_slices, S.G, S.B), 256, 0, st>>>(a, S.e_slices, S.d_epart.p);
            slot2_energy_sum_kernel<<<(S.B * S.R + 255) / 256, 256, 0, st>>>(a, S.e_slices, S.d_epart.p);
            CK(cudaGetLastError());
            c.other_launches += 2;
        }
        slot2_swap_kernel<<<S.B, kSwapThreads, 0, st>>>(s, round, S.swap_base, filled, flags);
        CK(cudaGetLastError());
        c.other_launches++;
        if (S.kl_on) {
            slot2_kl_kernel<<<S.B, 1024, 0, st>>>(a, S.d_slot_state.p, kl_args(c), round);
            CK(cudaGetLastError());
            c.other_launches++;
        }
        if (flags & (TG_REC_DIGEST | TG_REC_STATE | TG_REC_GRID)) {
            slot2_extract_kernel<<<dim3(std::max(1, c.sms / 2), S.B), 256, 0, st>>>(
                a, s, filled, (flags & TG_REC_GRID) ? 1 : 0);
            CK(cudaGetLastError());
            c.other_launches++;
        }
        if (c.profiling && (k + 1 == n_rounds || (k & 63) == 63)) {
            // sampled: one sweep launch in 64 (and the last) is timed, scaled to all
            CK(cudaEventSynchronize(c.ev[1]));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
            const int64_t span = (k & 63) + 1;
            sweep_ms += ms * (double)span;
        }
        S.swap_base += (uint64_t)round_attempts(S.I, S.J, round);
        S.rounds_done = round;
        if (++filled == S.rec_cap) {
            s2_drain(c, filled, first, sink);
            filled = 0;
            first = S.rounds_done + 1;
        }
    }
    s2_drain(c, filled, first, sink);
    CK(cudaStreamSynchronize(st));
    c.last_sweep_ms = sweep_ms;
    if (S.kl_on) {
        int e = 0;
        CK(cudaMemcpy(&e, S.d_kl_err.p, sizeof e, cudaMemcpyDeviceToHost));
        if (e) fail(TG_ERR_CONFIG, "kl: target has zero mass on an observed state");
    }
}


void s2_get_state(tg_ctx& c, int b, int slot, int8_t* out) {
    Slot2& S = c.s2;
    if (!S.ready) fail(TG_ERR_CONFIG, "get_state: not initialised");
    if (b < 0 || b >= S.B) fail(TG_ERR_CONFIG, "instance %d out of range", b);
    if (slot < 0 || slot >= S.R) fail(TG_ERR_CONFIG, "get_state: slot %d out of range", slot);
    int32_t m = 0;
    CK(cudaMemcpyAsync(&m, S.d_slot_state.p + (size_t)b * S.R + slot, sizeof(int32_t),
                       cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    const S2Prep& P = S.prep[b];
    std::vector<int8_t> col(P.n);
    long long off = 0;
    for (int q = 0; q < b; ++q) off += (long long)S.prep[q].n * S.Rp;
    CK(cudaMemcpy2DAsync(col.data(), 1, S.d_spins.p + off + m, S.Rp, 1, P.n, cudaMemcpyDeviceToHost,
                         c.stream));
    CK(cudaStreamSynchronize(c.stream));
    for (int i = 0; i < P.n; ++i) out[P.order[i]] = col[i];
}

void s2_counters(tg_ctx& c, int b, int64_t* attempts_p, int64_t* accepts_p, int64_t* attempts_b,
                 int64_t* accepts_b) {
    Slot2& S = c.s2;
    if (!S.ready) fail(TG_ERR_CONFIG, "get_counters: not initialised");
    if (b < 0 || b >= S.B) fail(TG_ERR_CONFIG, "instance %d out of range", b);
    const int np = S.I * std::max(0, S.J - 1), nb = std::max(0, S.I - 1) * S.J;
    if (accepts_p && np)
        CK(cudaMemcpyAsync(accepts_p, S.d_acc_p.p + (size_t)b * np, sizeof(int64_t) * np,
                           cudaMemcpyDeviceToHost, c.stream));
    if (accepts_b && nb)
        CK(cudaMemcpyAsync(accepts_b, S.d_acc_b.p + (size_t)b * nb, sizeof(int64_t) * nb,
                           cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    std::vector<int64_t> ap(np, 0), ab(nb, 0);
    for (int64_t r = 1; r <= S.rounds_done; ++r) {
        int even, dp, db;
        round_phase(S.I, S.J, r, even, dp, db);
        if (dp) for (int i = 0; i < S.I; ++i) for (int p = even; p + 1 < S.J; p += 2) ap[i * (S.J - 1) + p]++;
        if (db) for (int j = 0; j < S.J; ++j) for (int q = even; q + 1 < S.I; q += 2) ab[q * S.J + j]++;
    }
    if (attempts_p) std::copy(ap.begin(), ap.end(), attempts_p);
    if (attempts_b) std::copy(ab.begin(), ab.end(), attempts_b);
}

void s2_energies(tg_ctx& c, int b, double* f, double* g) {
    Slot2& S = c.s2;
    std::vector<double> fs(S.R), gs(S.R);
    std::vector<int32_t> ss(S.R);
    CK(cudaMemcpyAsync(fs.data(), S.d_f.p + (size_t)b * S.R, sizeof(double) * S.R, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(gs.data(), S.d_g.p + (size_t)b * S.R, sizeof(double) * S.R, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(ss.data(), S.d_slot_state.p + (size_t)b * S.R, sizeof(int32_t) * S.R,
                       cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    for (int q = 0; q < S.R; ++q) {
        if (f) f[q] = fs[ss[q]];
        if (g) g[q] = gs[ss[q]];
    }
}
}  // namespace

// ================================================================ C ABI

namespace {

// ---------------------------------------------------------------- probes
// probe_population (schedule.cpp:18-52) on the device: the chains are the
// replicas of a one-instance SLOT-engine batch that never swaps.  The batch is
// built once per (problem, n_chains, rule); every probe re-keys the chains'
// streams (derive_seed(seed, probe, c), drawing the initial state from draw 0
// and the sweeps from draw n on), re-initialises them, and runs all its sweeps
// in ONE cooperative launch that writes each kept sweep's (f, g) of every chain
// into a history; probe_moments_kernel pools the history in the reference's
// order.  The host only evaluates the closing formulas.
void probe_run(tg_ctx& c, double beta, double penalty, int n_chains, int sweeps, uint64_t seed,
               int rule, tg_probe_stats* out) {
    if (n_chains < 2) fail(TG_ERR_CONFIG, "probe: need at least 2 chains");
    if (sweeps < 2) fail(TG_ERR_CONFIG, "probe: need at least 2 sweeps");
    if (!c.have_problem) fail(TG_ERR_CONFIG, "probe: no problem set (tg_set_problem)");
    if (!(penalty >= 0.0)) fail(TG_ERR_CONFIG, "build_effective: penalty must be >= 0");
    if (rule != TG_RULE_METROPOLIS && rule != TG_RULE_HEAT_BATH)
        fail(TG_ERR_CONFIG, "probe: unknown update rule %d", rule);
    if (c.world != 1) fail(TG_ERR_CONFIG, "probe: single-GPU contexts only");
    Slot2& S = c.s2;
    cudaStream_t st = c.stream;
    if (!S.ready || !S.probe || S.probe_gen != c.problem_gen || S.probe_chains != n_chains ||
        S.probe_rule != rule) {
        BatchInst bi;
        bi.n = c.n;
        ensure_host_arrays(c);
        bi.ci = c.ci; bi.cj = c.cj; bi.cw = c.cw; bi.h = c.h; bi.pa = c.pa; bi.pb = c.pb;
        bi.betas.assign(n_chains, beta);
        bi.pens.assign(1, penalty);
        bi.seed = seed;
        c.batch.assign(1, std::move(bi));
        tg_run_config cfg{};
        cfg.total_sweeps = 1;
        cfg.sweeps_per_swap = 1;
        cfg.rule = rule;
        cfg.engine = TG_ENGINE_SLOT;
        cfg.record_every = 1;
        c.use_s2 = false;
        c.initialised = false;
        S.probe = true;
        s2_build(c, &cfg);
        c.batch.clear();
        S.probe_gen = c.problem_gen;
        S.probe_chains = n_chains;
        S.probe_rule = rule;
    }
    const int R = S.R, Rp = S.Rp, n = S.prep[0].n;
    // per-probe labels: beta, 2P, stream keys; error bands for this (beta, P)
    s2_bands(S.prep[0], std::fabs(beta), penalty);
    S.h_inst[0].eps = S.prep[0].eps;
    S.h_inst[0].beta_max = S.prep[0].beta_max;
    S.d_inst.upload(S.h_inst, st);
    std::vector<double> sb(Rp, 0.0), stp(Rp, 0.0);
    std::vector<uint64_t> sk(Rp, 0), keys(R);
    for (int r = 0; r < R; ++r) {
        keys[r] = derive_seed(seed, kPurposeProbe, (uint64_t)r);
        sb[r] = beta;
        stp[r] = 2.0 * penalty;
        sk[r] = keys[r];
    }
    S.d_sbeta.upload(sb, st);
    S.d_stwop.upload(stp, st);
    S.d_skey.upload(sk, st);
    S.d_keys.upload(keys, st);
    S.d_init_keys.upload(keys, st);
    const int burn_in = sweeps / 2, kept = sweeps - burn_in;
    S.d_hist_f.alloc((size_t)kept * R);
    S.d_hist_g.alloc((size_t)kept * R);
    S.d_moments.alloc(4);
    S2Args a = s2_args(c);
    slot2_init_kernel<<<dim3(c.sms * 4, 1), 256, 0, st>>>(a, S.d_init_keys.p);
    CK(cudaGetLastError());
    a.hist_f = S.d_hist_f.p;
    a.hist_g = S.d_hist_g.p;
    a.hist_t0 = 1 + burn_in;      // sweep s uses draws (s+1)*n + i: t = s + 1
    int64_t t0 = 1;
    int nsw = sweeps, de = 0;
    void* args[] = {&a, &t0, &nsw, &de};
    CK(cudaLaunchCooperativeKernel(slot2_sweep_fn(S.D, true), dim3(S.grid), dim3(kSlot2Threads), args, 0, st));
    probe_moments_kernel<<<1, 32, 0, st>>>(S.d_hist_f.p, S.d_hist_g.p, R, kept, penalty, S.d_moments.p);
    CK(cudaGetLastError());
    c.sweep_launches += 1;
    c.other_launches += 2;
    double sum[4];
    CK(cudaMemcpyAsync(sum, S.d_moments.p, sizeof sum, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    (void)n;
    // schedule.cpp:43-51
    const double inv = 1.0 / static_cast<double>((int64_t)kept * n_chains);
    out->row = out->column = 0;
    out->beta = beta;
    out->penalty = penalty;
    out->mean_g = sum[2] * inv;
    const double mean_e = sum[0] * inv;
    out->sigma_e = std::sqrt(std::max(0.0, sum[1] * inv - mean_e * mean_e));
    out->sigma_g = std::sqrt(std::max(0.0, sum[3] * inv - out->mean_g * out->mean_g));
}

double median_of(std::vector<double> v) {  // schedule.cpp:57-60 (lower median)
    std::sort(v.begin(), v.end());
    return v[(v.size() - 1) / 2];
}

// build_schedule (schedule.cpp:77-163) with every probe on the device.
void build_schedule(tg_ctx& c, const tg_schedule_config& cfg, std::vector<double>& betas,
                    std::vector<double>& pens, std::vector<tg_probe_stats>& stats, bool& exhausted) {
    // check_config, schedule.cpp:62-73
    if (cfg.beta0 <= 0.0) fail(TG_ERR_CONFIG, "schedule: beta0 must be > 0");
    if (cfg.p0 < 0.0) fail(TG_ERR_CONFIG, "schedule: P0 must be >= 0");
    if (cfg.i_max < 1 || cfg.j_max < 1) fail(TG_ERR_CONFIG, "schedule: I_max and J_max must be >= 1");
    if (cfg.alpha_beta <= 0.0 || cfg.alpha_p <= 0.0) fail(TG_ERR_CONFIG, "schedule: learning rates must be > 0");
    if (cfg.replica_budget < 1) fail(TG_ERR_CONFIG, "schedule: replica budget must be >= 1");
    if ((long long)cfg.i_max * cfg.j_max > cfg.replica_budget)
        fail(TG_ERR_CONFIG, "schedule: I_max * J_max exceeds replica budget");
    if (!c.have_problem) fail(TG_ERR_CONFIG, "schedule: no problem set (tg_set_problem)");
    const double sigma_min = cfg.sigma_min > 0.0 ? cfg.sigma_min : 0.5 * std::sqrt((double)c.n);
    const double p_cap = 2.0 * cfg.p0 + 1.0;
    uint64_t probe_counter = 0;
    auto run_probe = [&](double beta, double penalty) {
        tg_probe_stats s;
        probe_run(c, beta, penalty, cfg.n_chains, cfg.sweeps_per_probe,
                  derive_seed(cfg.seed, kPurposeProbe, probe_counter++), cfg.rule, &s);
        return s;
    };
    auto p_increment = [&](double beta, double sigma_g) {
        return std::min(cfg.alpha_p / (beta * std::max(sigma_g, 1e-300)), p_cap);
    };
    pens.assign(1, cfg.p0);
    stats.clear();
    exhausted = false;
    std::vector<std::vector<double>> beta_columns;
    std::map<std::pair<int, int>, double> proposals;
    std::vector<double> column = {cfg.beta0};
    tg_probe_stats last{};
    for (int i = 0;; ++i) {
        last = run_probe(column[i], cfg.p0);
        last.row = i;
        last.column = 0;
        stats.push_back(last);
        if (last.sigma_e <= sigma_min) break;
        proposals[{i, 1}] = cfg.p0 + p_increment(column[i], last.sigma_g);
        if (i + 1 >= cfg.i_max) break;
        column.push_back(column[i] + cfg.alpha_beta / last.sigma_e);
    }
    beta_columns.push_back(column);
    const int n_rows = (int)column.size();
    if (last.mean_g >= 0.5) {
        if (proposals.empty()) proposals[{0, 1}] = cfg.p0 + p_increment(cfg.beta0, last.sigma_g);
        for (int j = 1;; ++j) {
            std::vector<double> next_p;
            for (const auto& kv : proposals)
                if (kv.first.second == j) next_p.push_back(kv.second);
            if ((long long)(j + 1) * n_rows > cfg.replica_budget || j >= cfg.j_max) {
                exhausted = true;
                break;
            }
            const double prev = pens.back();
            pens.push_back(std::max(median_of(next_p), prev + 1e-9 * (1.0 + std::fabs(prev))));
            column.assign(1, cfg.beta0);
            for (int i = 0; i < n_rows; ++i) {
                last = run_probe(column[i], pens[j]);
                last.row = i;
                last.column = j;
                stats.push_back(last);
                const auto base = proposals.find({i, j});
                proposals[{i, j + 1}] = (base != proposals.end() ? base->second : pens[j]) +
                                        p_increment(column[i], last.sigma_g);
                if (i + 1 < n_rows)
                    column.push_back(column[i] + cfg.alpha_beta / std::max(last.sigma_e, sigma_min));
            }
            beta_columns.push_back(column);
            if (last.mean_g < 0.5) break;
        }
    }
    betas.resize(n_rows);
    for (int i = 0; i < n_rows; ++i) {
        std::vector<double> row;
        for (const auto& col : beta_columns) row.push_back(col[i]);
        betas[i] = median_of(row);
    }
}

}  // namespace

extern "C" {

int tg_abi_version(void) { return TG_ABI_VERSION; }

static int create_impl(int device, int rank, int world, const void* nccl_id, tg_ctx** out) {
    HostTimer tm_("create");
    if (!out) return TG_ERR_CONFIG;
    *out = nullptr;
    tg_ctx* c = new tg_ctx();
    const int rc = guard(nullptr, [&] {
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            fail(TG_ERR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
        if (device < 0 || device >= count) fail(TG_ERR_CONFIG, "device %d out of range", device);
        c->device = device;
        c->rank = rank;
        c->world = world;
        CK(cudaSetDevice(device));
        int major = 0, minor = 0;  // attribute queries: microseconds, unlike cudaGetDeviceProperties
        CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
        if (major < 10)
            fail(TG_ERR_CUDA, "device %d is sm_%d%d; this build targets sm_100a", device, major, minor);
        CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->stream_owner.s = c->stream;
        t_alloc_stream = c->stream;
        static bool pool_set[64] = {};
        if (device < 64 && !pool_set[device]) {  // keep freed pool memory for the next context
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t keep = ~0ull;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
            pool_set[device] = true;
        }
        if (world > 1) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            NK(nccl().CommInitRank(&c->comm, world, id, rank));
        }
    });
    if (rc != TG_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return TG_OK;
}

int tg_create(int device, tg_ctx** out) { return create_impl(device, 0, 1, nullptr, out); }

int tg_create_distributed(int device, int rank, int world_size, const void* nccl_id, tg_ctx** out) {
    if (world_size < 1 || rank < 0 || rank >= world_size || (world_size > 1 && !nccl_id)) {
        g_create_error = "tg_create_distributed: bad rank/world/id";
        return TG_ERR_CONFIG;
    }
    return create_impl(device, rank, world_size, nccl_id, out);
}

int tg_nccl_unique_id(void* out128) {
    ncclUniqueId id;
    if (!nccl().ok || nccl().GetUniqueId(&id) != ncclSuccess) return TG_ERR_CUDA;
    std::memcpy(out128, &id, sizeof(id));
    return TG_OK;
}

void tg_destroy(tg_ctx* ctx) {
    HostTimer tm_("destroy");
    delete ctx;
}

size_t tg_last_error(const tg_ctx* ctx, char* buf, size_t len) {
    const std::string& s = ctx ? ctx->err : g_create_error;
    if (buf && len) {
        const size_t k = std::min(len - 1, s.size());
        std::memcpy(buf, s.data(), k);
        buf[k] = '\0';
    }
    return s.size();
}

int tg_set_problem(tg_ctx* ctx, int n, int n_couplings, const int32_t* ci, const int32_t* cj,
                   const double* w, const double* fields, int n_pairs, const int32_t* pa,
                   const int32_t* pb) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        HostTimer tm_("set_problem (total)");
        if (n <= 0) fail(TG_ERR_CONFIG, "model: n_spins must be positive");
        if (n_couplings < 0 || n_pairs < 0) fail(TG_ERR_CONFIG, "model: negative counts");
        tg_ctx& c = *ctx;
        cudaStream_t st = c.stream;
        CK(cudaSetDevice(c.device));
        c.have_problem = false;
        c.dev_prep = c.host_canonical = false;
        // validation, colouring, canonical order and the internal CSR on the
        // device (prep.cu); the raw caller arrays go up once
        PrepSummary P;
        {
            HostTimer t2_("set_problem: device prep");
            DBuf<int>& dci = c.d_raw_ci; DBuf<int>& dcj = c.d_raw_cj;
            DBuf<int>& dpa = c.d_raw_pa; DBuf<int>& dpb = c.d_raw_pb;
            DBuf<double>& dw = c.d_raw_w; DBuf<double>& dh = c.d_raw_h;
            dci.upload(ci, n_couplings, st);
            dcj.upload(cj, n_couplings, st);
            dw.upload(w, n_couplings, st);
            std::vector<double> hz;
            if (!fields) hz.assign(n, 0.0);
            dh.upload(fields ? fields : hz.data(), n, st);
            dpa.upload(pa, n_pairs, st);
            dpb.upload(pb, n_pairs, st);
            c.d_order_dev.alloc(n);
            c.d_inv_dev.alloc(n);
            c.d_base_dev.alloc((size_t)n + 1);
            c.d_nbr_dev.alloc((size_t)2 * ((size_t)n_couplings + n_pairs));
            PrepIn in{n, n_couplings, n_pairs, dci.p, dcj.p, dw.p, dh.p, dpa.p, dpb.p};
            PrepOut out{c.d_order_dev.p, c.d_inv_dev.p, c.d_base_dev.p, c.d_nbr_dev.p};
            CK(plane_prep_device(in, out, P, st, c.sms));
        }
        HostTimer t3_("set_problem: finish");
        if (P.bad) {  // the host validator produces the reference's message
            BatchInst bi;
            load_problem(bi, n, n_couplings, ci, cj, w, fields, n_pairs, pa, pb);
            fail(TG_ERR_INTERNAL, "device validation rejected an instance the host accepts (flags %u)", P.bad);
        }
        c.n = n;
        c.m = n_couplings;
        c.np = n_pairs;
        c.host_arrays = false;  // host copies are fetched from the device when a host path needs them
        if (P.colour_incomplete) {  // dependency chains beyond the device round budget
            ensure_host_arrays(c);
            canonical(n, c.ci, c.cj, c.pa, c.pb, c.order, c.color, c.n_colors);
            c.inv.assign(n, 0);
            for (int k = 0; k < n; ++k) c.inv[c.order[k]] = k;
            c.color_start.assign(c.n_colors + 1, 0);
            for (int k = 0; k < n; ++k) c.color_start[c.color[c.order[k]] + 1]++;
            for (int q = 0; q < c.n_colors; ++q) c.color_start[q + 1] += c.color_start[q];
            c.host_canonical = true;
            c.d_order_dev.release();
            c.d_inv_dev.release();
            c.d_base_dev.release();
            c.d_nbr_dev.release();
        } else {
            c.n_colors = P.n_colors;
            c.color_start.assign(c.n_colors + 1, 0);
            const unsigned mq1 = P.max_dq + 1, mc1 = P.max_dc + 1;
            for (size_t q = 0; q < P.run_keys.size(); ++q)
                c.color_start[P.run_keys[q] / (mq1 * mc1) + 1] += P.run_counts[q];
            for (int q = 0; q < c.n_colors; ++q) c.color_start[q + 1] += c.color_start[q];
            c.prep = std::move(P);
            c.dev_prep = true;
        }
        ctx->have_problem = true;
        ++ctx->problem_gen;
        ctx->initialised = false;
    });
}

int tg_set_schedule(tg_ctx* ctx, int n_betas, const double* betas, int n_penalties,
                    const double* penalties) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        std::vector<double> b(betas, betas + std::max(n_betas, 0));
        std::vector<double> p(penalties, penalties + std::max(n_penalties, 0));
        check_vec(b, "beta");
        check_vec(p, "penalty");
        for (double x : p) if (x < 0.0) fail(TG_ERR_CONFIG, "build_effective: penalty must be >= 0");
        ctx->betas = b;
        ctx->pens = p;
        ctx->have_schedule = true;
        ctx->initialised = false;
    });
}

int tg_init(tg_ctx* ctx, const tg_run_config* cfg) {
    if (!ctx || !cfg) return TG_ERR_CONFIG;
    return guard(ctx, [&] { do_init(*ctx, cfg); });
}

int tg_advance(tg_ctx* ctx, int64_t n_rounds, tg_sink_fn sink, void* user) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] { do_advance(*ctx, n_rounds, SinkCtx{sink, user}); });
}

int tg_run(tg_ctx* ctx, const tg_run_config* cfg, tg_sink_fn sink, void* user) {
    if (!ctx || !cfg) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        do_init(*ctx, cfg);
        HostTimer tm_("advance (all rounds)");
        do_advance(*ctx, cfg->total_sweeps / cfg->sweeps_per_swap, SinkCtx{sink, user});
    });
}

int tg_get_state(tg_ctx* ctx, int slot, int8_t* out) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        HostTimer tm_("get_state");
        tg_ctx& c = *ctx;
        if (c.use_s2) { s2_get_state(c, 0, slot, out); return; }
        if (!c.initialised) fail(TG_ERR_CONFIG, "get_state: context not initialised");
        if (slot < 0 || slot >= c.R) fail(TG_ERR_CONFIG, "get_state: slot %d out of range", slot);
        // reuse the extract kernel on a one-slot view: temporarily point slot R-1 at `slot`
        std::vector<int32_t> ss(c.R);
        CK(cudaMemcpyAsync(ss.data(), c.d_slot_state.p, sizeof(int32_t) * c.R, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        DBuf<int32_t> view;
        std::vector<int32_t> v(c.R, ss[slot]);
        view.upload(v, c.stream);
        DBuf<int8_t> dst;
        dst.alloc(c.n);
        ExtractArgs e{};
        e.n = c.n;
        e.R = c.R;
        e.W = c.W;
        e.plane = c.engine == TG_ENGINE_PLANE;
        e.all_slots = 0;
        e.local_states = c.R_local;
        e.state0 = c.state0;
        e.slot_state = view.p;
        e.spins32 = c.d_spins32.p;
        e.spins8 = c.d_spins8.p;
        e.perm = c.d_perm.p;
        e.states = dst.p;
        e.digest = nullptr;
        extract_kernel<<<std::max(1, std::min((c.n + 255) / 256, c.sms * 8)), 256, 0, c.stream>>>(e);
        CK(cudaGetLastError());
        if (c.world > 1) NK(nccl().AllReduce(dst.p, dst.p, c.n, ncclInt8, ncclSum, c.comm, c.stream));
        CK(cudaMemcpyAsync(out, dst.p, c.n, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    });
}

int tg_get_counters(tg_ctx* ctx, int64_t* attempts_p, int64_t* accepts_p, int64_t* attempts_b,
                    int64_t* accepts_b) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        tg_ctx& c = *ctx;
        if (c.use_s2) { s2_counters(c, 0, attempts_p, accepts_p, attempts_b, accepts_b); return; }
        if (!c.initialised) fail(TG_ERR_CONFIG, "get_counters: context not initialised");
        const int np = c.I * std::max(0, c.J - 1), nb = std::max(0, c.I - 1) * c.J;
        if (accepts_p && np) CK(cudaMemcpyAsync(accepts_p, c.d_acc_p.p, sizeof(int64_t) * np, cudaMemcpyDeviceToHost, c.stream));
        if (accepts_b && nb) CK(cudaMemcpyAsync(accepts_b, c.d_acc_b.p, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        std::vector<int64_t> ap(np, 0), ab(nb, 0);
        for (int64_t r = 1; r <= c.rounds_done; ++r) {
            int even, dp, db;
            round_phase(c.I, c.J, r, even, dp, db);
            if (dp) for (int i = 0; i < c.I; ++i) for (int p = even; p + 1 < c.J; p += 2) ap[i * (c.J - 1) + p]++;
            if (db) for (int j = 0; j < c.J; ++j) for (int b = even; b + 1 < c.I; b += 2) ab[b * c.J + j]++;
        }
        if (attempts_p) std::copy(ap.begin(), ap.end(), attempts_p);
        if (attempts_b) std::copy(ab.begin(), ab.end(), attempts_b);
    });
}

int tg_get_energies(tg_ctx* ctx, double* f, double* g) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        tg_ctx& c = *ctx;
        if (c.use_s2) { s2_energies(c, 0, f, g); return; }
        if (!c.initialised) fail(TG_ERR_CONFIG, "get_energies: context not initialised");
        std::vector<double> fs(c.R), gs(c.R);
        std::vector<int32_t> ss(c.R);
        CK(cudaMemcpyAsync(fs.data(), c.d_f.p, sizeof(double) * c.R, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(gs.data(), c.d_g.p, sizeof(double) * c.R, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(ss.data(), c.d_slot_state.p, sizeof(int32_t) * c.R, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        for (int s = 0; s < c.R; ++s) {
            if (f) f[s] = fs[ss[s]];
            if (g) g[s] = gs[ss[s]];
        }
    });
}

int tg_get_info(tg_ctx* ctx, tg_info* info) {
    if (!ctx || !info) return TG_ERR_CONFIG;
    std::memset(info, 0, sizeof(*info));
    info->engine = ctx->engine;
    info->n_colors = ctx->n_colors;
    info->n_replicas = ctx->R;
    info->local_replicas = ctx->R_local;
    info->words = ctx->W;
    info->device_sms = ctx->sms;
    info->rounds_done = ctx->rounds_done;
    info->last_sweep_ms = ctx->last_sweep_ms;
    info->last_swap_ms = ctx->last_swap_ms;
    info->sweep_launches = ctx->sweep_launches;
    info->other_launches = ctx->other_launches;
    return TG_OK;
}

void* tg_stream(tg_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int tg_set_profiling(tg_ctx* ctx, int on) {
    if (!ctx) return TG_ERR_CONFIG;
    ctx->profiling = on != 0;
    return TG_OK;
}

int tg_batch_clear(tg_ctx* ctx) {
    if (!ctx) return TG_ERR_CONFIG;
    ctx->batch.clear();
    ctx->s2.ready = false;
    ctx->use_s2 = false;
    return TG_OK;
}

int tg_batch_add(tg_ctx* ctx, int n, int n_couplings, const int32_t* ci, const int32_t* cj,
                 const double* w, const double* fields, int n_pairs, const int32_t* pa,
                 const int32_t* pb, int n_betas, const double* betas, int n_penalties,
                 const double* penalties, uint64_t seed, int32_t* index) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        BatchInst bi;
        load_problem(bi, n, n_couplings, ci, cj, w, fields, n_pairs, pa, pb);
        bi.betas.assign(betas, betas + std::max(n_betas, 0));
        bi.pens.assign(penalties, penalties + std::max(n_penalties, 0));
        check_vec(bi.betas, "beta");
        check_vec(bi.pens, "penalty");
        for (double x : bi.pens) if (x < 0.0) fail(TG_ERR_CONFIG, "build_effective: penalty must be >= 0");
        bi.seed = seed;
        ctx->batch.push_back(std::move(bi));
        ctx->s2.ready = false;
        if (index) *index = (int32_t)ctx->batch.size() - 1;
    });
}

int tg_batch_init(tg_ctx* ctx, const tg_run_config* cfg) {
    if (!ctx || !cfg) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        if (cfg->sweeps_per_swap < 1) fail(TG_ERR_CONFIG, "run: sweeps_per_swap must be >= 1");
        if (cfg->total_sweeps < cfg->sweeps_per_swap)
            fail(TG_ERR_CONFIG, "run: total_sweeps must be >= sweeps_per_swap");
        if (cfg->rule != TG_RULE_METROPOLIS && cfg->rule != TG_RULE_HEAT_BATH)
            fail(TG_ERR_CONFIG, "run: unknown update rule %d", cfg->rule);
        if (cfg->engine != TG_ENGINE_AUTO && cfg->engine != TG_ENGINE_SLOT)
            fail(TG_ERR_CONFIG, "batch: only the SLOT engine runs batches");
        if (ctx->world != 1) fail(TG_ERR_CONFIG, "batch: single-GPU contexts only");
        ctx->use_s2 = false;
        ctx->initialised = false;
        ctx->s2.probe = false;
        s2_build(*ctx, cfg);
        ctx->rounds_done = 0;
    });
}

int tg_batch_advance(tg_ctx* ctx, int64_t n_rounds, tg_batch_sink_fn sink, void* user) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        if (!ctx->s2.ready || ctx->s2.probe) fail(TG_ERR_CONFIG, "batch: not initialised (tg_batch_init)");
        s2_advance(*ctx, n_rounds, BatchSinkCtx{sink, user});
        ctx->rounds_done = ctx->s2.rounds_done;
    });
}

int tg_batch_run(tg_ctx* ctx, const tg_run_config* cfg, tg_batch_sink_fn sink, void* user) {
    const int rc = tg_batch_init(ctx, cfg);
    if (rc != TG_OK) return rc;
    return tg_batch_advance(ctx, cfg->total_sweeps / cfg->sweeps_per_swap, sink, user);
}

int tg_batch_get_state(tg_ctx* ctx, int instance, int slot, int8_t* out) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] { s2_get_state(*ctx, instance, slot, out); });
}

int tg_batch_get_counters(tg_ctx* ctx, int instance, int64_t* attempts_p, int64_t* accepts_p,
                          int64_t* attempts_b, int64_t* accepts_b) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] { s2_counters(*ctx, instance, attempts_p, accepts_p, attempts_b, accepts_b); });
}

namespace {
struct JColumnMerge {
    tg_baseline_record* out;
    int64_t rounds;
    int64_t feasible_total, sample_total;
};

int jcolumn_sink(void* user, int32_t, const tg_record* recs, int64_t n, const int8_t*, const int64_t*,
                 const int64_t*) {
    auto* m = static_cast<JColumnMerge*>(user);
    for (int64_t k = 0; k < n; ++k) {
        const tg_record& r = recs[k];
        if (r.round < 1 || r.round > m->rounds) return 1;
        tg_baseline_record& b = m->out[r.round - 1];
        ++b.n_total;
        ++m->sample_total;
        if (r.feasible) {
            ++b.n_feasible;
            ++m->feasible_total;
            if (!b.any_feasible || r.f < b.best_f) b.best_f = r.f;
            b.any_feasible = 1;
        }
    }
    return 0;
}
}  // namespace

int tg_run_jcolumn(tg_ctx* ctx, int n_betas, const double* betas, double p_fixed, int j_repeats,
                   const tg_run_config* cfg, tg_baseline_record* out, int64_t out_cap,
                   double* feasible_fraction) {
    if (!ctx || !cfg) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        // engine.cpp:224-225
        if (!(p_fixed > 0.0)) fail(TG_ERR_CONFIG, "baseline: P must be positive");
        if (j_repeats < 1) fail(TG_ERR_CONFIG, "baseline: repeats must be >= 1");
        if (!ctx->have_problem) fail(TG_ERR_CONFIG, "baseline: no problem set (tg_set_problem)");
        if (cfg->sweeps_per_swap < 1) fail(TG_ERR_CONFIG, "run: sweeps_per_swap must be >= 1");
        if (cfg->total_sweeps < cfg->sweeps_per_swap)
            fail(TG_ERR_CONFIG, "run: total_sweeps must be >= sweeps_per_swap");
        const int64_t rounds = cfg->total_sweeps / cfg->sweeps_per_swap;
        if (!out || out_cap < rounds) fail(TG_ERR_CONFIG, "baseline: output holds %lld of %lld rounds",
                                           (long long)out_cap, (long long)rounds);
        BatchInst proto;
        proto.n = ctx->n;
        ensure_host_arrays(*ctx);
        proto.ci = ctx->ci;
        proto.cj = ctx->cj;
        proto.cw = ctx->cw;
        proto.h = ctx->h;
        proto.pa = ctx->pa;
        proto.pb = ctx->pb;
        proto.betas.assign(betas, betas + std::max(n_betas, 0));
        proto.pens.assign(1, p_fixed);
        check_vec(proto.betas, "beta");
        ctx->batch.clear();
        for (int rep = 0; rep < j_repeats; ++rep) {
            ctx->batch.push_back(proto);
            ctx->batch.back().seed = derive_seed(cfg->seed, kPurposeRepeat, (uint64_t)rep);
        }
        for (int64_t k = 0; k < rounds; ++k) {
            tg_baseline_record& b = out[k];
            b.round = k + 1;
            b.sweep_count = (k + 1) * cfg->sweeps_per_swap;
            b.best_f = std::numeric_limits<double>::quiet_NaN();
            b.any_feasible = b.n_feasible = b.n_total = b.reserved = 0;
        }
        tg_run_config c2 = *cfg;
        c2.record_flags = 0;  // f, g, feasible only (store_target_only, engine.cpp:239)
        c2.record_every = 1;
        c2.engine = TG_ENGINE_SLOT;
        if (cfg->engine != TG_ENGINE_AUTO && cfg->engine != TG_ENGINE_SLOT)
            fail(TG_ERR_CONFIG, "baseline: only the SLOT engine runs batches");
        if (ctx->world != 1) fail(TG_ERR_CONFIG, "baseline: single-GPU contexts only");
        JColumnMerge m{out, rounds, 0, 0};
        ctx->use_s2 = false;
        ctx->initialised = false;
        ctx->s2.probe = false;
        s2_build(*ctx, &c2);
        s2_advance(*ctx, rounds, BatchSinkCtx{&jcolumn_sink, &m});
        ctx->batch.clear();
        if (feasible_fraction)
            *feasible_fraction = m.sample_total == 0 ? 0.0 : (double)m.feasible_total / (double)m.sample_total;
    });
}

int tg_set_kl_decoder(tg_ctx* ctx, int n_logical, int n_couplings, const int32_t* li,
                      const int32_t* lj, const double* lw, const double* lh, double beta,
                      const int32_t* copy_offsets, const int32_t* copies, int discard_infeasible) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        // IsingModel validation (ising.cpp:21-46) of the logical model
        BatchInst lm;
        load_problem(lm, n_logical, n_couplings, li, lj, lw, lh, 0, nullptr, nullptr);
        if (n_logical > 20)
            fail(TG_ERR_RESOURCE, "kl decoder: %d logical spins (device histogram limit 20)", n_logical);
        if (!copy_offsets || !copies) fail(TG_ERR_CONFIG, "kl decoder: missing copy map");
        std::vector<int> off(copy_offsets, copy_offsets + n_logical + 1);
        if (off[0] != 0) fail(TG_ERR_CONFIG, "kl decoder: copy offsets must start at 0");
        for (int u = 0; u < n_logical; ++u)
            if (off[u + 1] <= off[u]) fail(TG_ERR_CONFIG, "kl decoder: logical spin %d has no copies", u);
        // enumerate_boltzmann (oracle.cpp:86-165): couplings sorted (i, j) as the
        // IsingModel stores them, energy = -sum w s_i s_j - sum h s_i, max-shifted
        // exponentials summed in encoding order
        std::vector<int> idx(lm.ci.size());
        for (size_t q = 0; q < idx.size(); ++q) idx[q] = (int)q;
        std::sort(idx.begin(), idx.end(), [&](int x, int y) {
            return lm.ci[x] != lm.ci[y] ? lm.ci[x] < lm.ci[y] : lm.cj[x] < lm.cj[y];
        });
        const size_t K = (size_t)1 << n_logical;
        std::vector<double> pr(K);
        double max_log = -std::numeric_limits<double>::infinity();
        for (size_t enc = 0; enc < K; ++enc) {
            double e = 0.0;
            for (int q : idx) {
                const double si = ((enc >> lm.ci[q]) & 1) ? 1.0 : -1.0;
                const double sj = ((enc >> lm.cj[q]) & 1) ? 1.0 : -1.0;
                e -= lm.cw[q] * si * sj;
            }
            for (int i = 0; i < n_logical; ++i) e -= lm.h[i] * (((enc >> i) & 1) ? 1.0 : -1.0);
            pr[enc] = e;
            max_log = std::max(max_log, -beta * e);
        }
        double sum = 0.0;
        for (size_t enc = 0; enc < K; ++enc) {
            pr[enc] = std::exp(-beta * pr[enc] - max_log);
            sum += pr[enc];
        }
        for (auto& p : pr) p /= sum;
        ctx->kl.on = true;
        ctx->kl.n_logical = n_logical;
        ctx->kl.discard = discard_infeasible ? 1 : 0;
        ctx->kl.copy_off = off;
        ctx->kl.copies.assign(copies, copies + off[n_logical]);
        ctx->kl.probs = std::move(pr);
        ctx->initialised = false;
    });
}

int tg_clear_kl_decoder(tg_ctx* ctx) {
    if (!ctx) return TG_ERR_CONFIG;
    ctx->kl.on = false;
    ctx->initialised = false;
    return TG_OK;
}

int tg_get_kl_curve(tg_ctx* ctx, int instance, int64_t first_round, int64_t n, double* kl,
                    int64_t* samples) {
    if (!ctx) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        Slot2& S = ctx->s2;
        if (!S.ready || !S.kl_on) fail(TG_ERR_CONFIG, "kl: no decoded run on this context");
        if (instance < 0 || instance >= S.B) fail(TG_ERR_CONFIG, "instance %d out of range", instance);
        if (first_round < 1 || n < 0 || first_round - 1 + n > std::min<int64_t>(S.kl_cap, S.rounds_done))
            fail(TG_ERR_CONFIG, "kl: rounds [%lld, %lld) not recorded", (long long)first_round,
                 (long long)(first_round + n));
        const size_t off = (size_t)instance * S.kl_cap + (size_t)(first_round - 1);
        if (kl) CK(cudaMemcpy(kl, S.d_kl.p + off, sizeof(double) * n, cudaMemcpyDeviceToHost));
        if (samples) CK(cudaMemcpy(samples, S.d_kl_samples.p + off, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    });
}

int tg_probe_population(tg_ctx* ctx, double beta, double penalty, int n_chains, int sweeps,
                        uint64_t seed, int rule, tg_probe_stats* out) {
    if (!ctx || !out) return TG_ERR_CONFIG;
    return guard(ctx, [&] { probe_run(*ctx, beta, penalty, n_chains, sweeps, seed, rule, out); });
}

int tg_build_schedule(tg_ctx* ctx, const tg_schedule_config* cfg, double* betas, int betas_cap,
                      int* n_betas, double* penalties, int penalties_cap, int* n_penalties,
                      tg_probe_stats* stats, int stats_cap, int* n_stats, int* budget_exhausted) {
    if (!ctx || !cfg) return TG_ERR_CONFIG;
    return guard(ctx, [&] {
        std::vector<double> b, p;
        std::vector<tg_probe_stats> st;
        bool ex = false;
        build_schedule(*ctx, *cfg, b, p, st, ex);
        if ((int)b.size() > betas_cap || (int)p.size() > penalties_cap)
            fail(TG_ERR_CONFIG, "schedule: output arrays hold %d betas / %d penalties, need %d / %d",
                 betas_cap, penalties_cap, (int)b.size(), (int)p.size());
        std::copy(b.begin(), b.end(), betas);
        std::copy(p.begin(), p.end(), penalties);
        if (n_betas) *n_betas = (int)b.size();
        if (n_penalties) *n_penalties = (int)p.size();
        if (stats) std::copy_n(st.begin(), std::min<size_t>(st.size(), (size_t)std::max(stats_cap, 0)), stats);
        if (n_stats) *n_stats = (int)st.size();
        if (budget_exhausted) *budget_exhausted = ex ? 1 : 0;
    });
}

int tg_canonical_order(int n, int n_couplings, const int32_t* ci, const int32_t* cj, int n_pairs,
                       const int32_t* pa, const int32_t* pb, int32_t* order, int32_t* color,
                       int32_t* n_colors) {
    return guard(nullptr, [&] {
        if (n <= 0) fail(TG_ERR_CONFIG, "model: n_spins must be positive");
        std::vector<int> a(ci, ci + n_couplings), b(cj, cj + n_couplings), x(pa, pa + n_pairs), y(pb, pb + n_pairs);
        for (int k = 0; k < n_couplings; ++k)
            if (a[k] < 0 || a[k] >= n || b[k] < 0 || b[k] >= n || a[k] == b[k]) fail(TG_ERR_CONFIG, "bad coupling");
        for (int k = 0; k < n_pairs; ++k)
            if (x[k] < 0 || x[k] >= n || y[k] < 0 || y[k] >= n || x[k] == y[k]) fail(TG_ERR_CONFIG, "bad pair");
        std::vector<int> ord, col;
        int nc = 0;
        canonical(n, a, b, x, y, ord, col, nc);
        for (int i = 0; i < n; ++i) {
            if (order) order[i] = ord[i];
            if (color) color[i] = col[i];
        }
        if (n_colors) *n_colors = nc;
    });
}

double tg_p_swap_probability(double beta, double d_penalty, double dg) {
    const double x = beta * d_penalty * dg;
    return x >= 0.0 ? 1.0 : std::exp(x);
}
double tg_beta_swap_probability(double d_beta, double d_energy) {
    const double x = d_beta * d_energy;
    return x >= 0.0 ? 1.0 : std::exp(x);
}
double tg_general_swap_probability(double beta_a, double beta_b, double de_a, double de_b) {
    const double x = beta_a * de_a + beta_b * de_b;
    return x >= 0.0 ? 1.0 : std::exp(x);
}

int tg_partition(int n_replicas, int rank, int world, int engine, int32_t* state0, int32_t* count) {
    if (n_replicas < 1 || world < 1 || rank < 0 || rank >= world) return TG_ERR_CONFIG;
    if (n_replicas % world != 0) return TG_ERR_CONFIG;
    const int per = n_replicas / world;
    if (engine == TG_ENGINE_PLANE && world > 1 && per % 32 != 0) return TG_ERR_CONFIG;
    if (state0) *state0 = rank * per;
    if (count) *count = per;
    return TG_OK;
}

int tg_swap_phase_host(int n_betas, const double* betas, int n_penalties, const double* penalties,
                       int64_t round, int /*direction*/, uint64_t seed, uint64_t swap_base,
                       const double* f_state, const double* g_state, int32_t* slot_state,
                       int64_t* accepts_p, int64_t* accepts_b) {
    const int I = n_betas, J = n_penalties;
    if (I < 1 || J < 1 || round < 1) return TG_ERR_CONFIG;
    const uint64_t swap_seed = derive_seed(seed, kPurposeSwap, 0);
    const int64_t n_att = round_attempts(I, J, round);
    for (int k = 0; k < n_att; ++k) {
        int sa, sb, ctr, is_p;
        if (swap_attempt(I, J, betas, penalties, round, k, f_state, g_state, slot_state, swap_seed,
                         swap_base, sa, sb, ctr, is_p)) {
            std::swap(slot_state[sa], slot_state[sb]);
            if (is_p) { if (accepts_p) accepts_p[ctr]++; }
            else if (accepts_b) accepts_b[ctr]++;
        }
    }
    return TG_OK;
}

}  // extern "C"
