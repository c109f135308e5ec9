// host.cuh -- internal declarations shared by the host-side translation units
// of the engine library (capi.cu = the C ABI entry points; host_*.cu = the
// drivers behind them).  Not installed, not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <atomic>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/tempergrid_b200.h"
#include "engine.cuh"
#include "kernels.cuh"

namespace tgh {

using namespace tg;


extern thread_local std::string g_create_error;

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

const NcclApi& nccl();

struct TgFail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...);

// Run `work` on the calling thread and up to nt - 1 helper threads.  Helper
// creation may fail (pids / cgroup limits): the threads already started are
// always joined and the caller's own run of `work` covers the rest (`work`
// pulls its items from a shared counter).
template <class F>
void run_pool(int nt, F& work) {
    std::vector<std::thread> pool;
    struct Joiner {
        std::vector<std::thread>& p;
        ~Joiner() { for (auto& th : p) if (th.joinable()) th.join(); }
    } joiner{pool};
    for (int t = 1; t < nt; ++t) {
        try {
            pool.emplace_back(work);
        } catch (...) {
            break;
        }
    }
    work();
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
extern thread_local cudaStream_t t_alloc_stream;

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
// Uninitialised host staging buffer for device-to-host record copies: a
// std::vector's zero-fill of a large ring (e.g. 64 instances x 1024 rounds of
// acceptance counters, 250 MB) cost ~80 ms per run before any data arrived.
template <class T>
struct HostVec {
    std::unique_ptr<T[]> p;
    size_t n = 0;
    void resize(size_t m) {
        if (m != n) {
            p.reset(m ? new T[m] : nullptr);
            n = m;
        }
    }
    T* data() { return p.get(); }
    const T* data() const { return p.get(); }
    size_t size() const { return n; }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
    T* begin() { return p.get(); }
    T* end() { return p.get() + n; }
};

// NVTX range for the host-side phases (sweep launches, swap / exchange,
// record drains): visible in Nsight timelines, free when no tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

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

inline int nbits(int d) {
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
    HostVec<TgRecordDev> h_rec;
    HostVec<int64_t> h_acc;
    HostVec<int8_t> h_states;
    int64_t rounds_done = 0;
    uint64_t swap_base = 0;
    bool ready = false;
    // schedule probes (schedule.cpp:18-52): independent chains, no swaps,
    // one stream per chain for the initial state and the sweeps
    bool probe = false;
    // FLOAT engine (slot_fast.cu): packed draws, certified FP32 decisions
    bool fast = false;
    int fdeg = 4, flps = 32, fspw = 1, fngs = 1;
    DBuf<float2> d_lab;
    DBuf<long long> d_fx;
    DBuf<int> d_gx, d_fitem_pref;
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


}  // namespace tgh

using namespace tg;
using namespace tgh;

struct tg_ctx {
    std::string err;
    int device = 0, rank = 0, world = 1;
    int sms = 0;
    StreamOwner stream_owner;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    bool dist = false;  // exchange over NCCL: world > 1, or a 1-rank communicator under TG_DIST_SELFTEST
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
    int fused_tpw = 0, tpw_fast = 0;
    int fused_c5 = 0;                // config-5 kernel (plane_c5.cu) for the fused round loop
    int c5_nfree[2] = {0, 0};        // chain-free sites of colours 0, 1
    int fused_cl = 0;                // cluster-per-word kernel (plane_cl.cu) instead of plane_c5
    int cl_size = 0, cl_stage = 0;   // CTAs per cluster; neighbour entries staged in shared memory
    int cl_ktab = 0, cl_small = 0;   // ktab staged in shared memory; <= 5 sites per thread and phase
    int cl_group = 0;                // software word barrier on G = cl_size CTAs per word (no clusters)
    int cl_pair = 0;                 // ... with two words per thread (G CTAs per word pair)
    int tpw_sweep_grid = 0;          // sweep-only tpw kernel grid (0: plane_sweep_kernel)
    int c5_sweep_grid = 0;           // sweep-only config-5 kernel grid (0: the tpw / plane sweep kernels)
    size_t c5_sweep_smem = 0;
    size_t tpw_sweep_smem = 0;
    const char* sweep_kernel = "";   // dominant sweep kernel of the last advance (tg_info)     // thread-per-(site, word) kernel (plane_tpw.cu) instead of plane_rounds_kernel
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
    DBuf<int4> d_nbr4;
    DBuf<unsigned long long> d_clx;  // cluster kernel: tagged (f, g) exchange words [2 parities][32 W] + error word
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
    HostVec<TgRecordDev> h_rec;
    HostVec<int8_t> h_states;
    HostVec<int64_t> h_acc;
    std::vector<cudaEvent_t> ev;
    double last_sweep_ms = 0, last_swap_ms = 0;
    int64_t sweep_launches = 0, other_launches = 0;
    // unfused round loop (multi-GPU, full-grid records): device round state,
    // per-chunk target digests, CUDA graphs of whole chunks keyed by length
    DBuf<RoundState> d_rstate;
    DBuf<uint64_t> d_dig;
    HostVec<uint64_t> h_dig;
    RoundState h_rstate{};
    std::map<int, cudaGraphExec_t> graphs;
    bool graphs_ok = true;
    int64_t graph_launches = 0;
    void clear_graphs() {
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
        graphs.clear();
    }

    ~tg_ctx() {
        t_alloc_stream = stream;
        clear_graphs();
        for (auto e : ev) cudaEventDestroy(e);
        if (comm) nccl().CommDestroy(comm);
        // members free their buffers on `stream`; stream_owner destroys it last
    }
};

extern "C" int tg_partition(int n_replicas, int rank, int world, int engine, int32_t* state0,
                            int32_t* count);

namespace tgh {


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

struct SinkCtx {
    tg_sink_fn fn;
    void* user;
};

struct BatchSinkCtx {
    tg_batch_sink_fn fn;
    void* user;
};

// ---- host drivers (definitions in host_*.cu)
void canonical(int n, const std::vector<int>& ci, const std::vector<int>& cj,
               const std::vector<int>& pa, const std::vector<int>& pb, std::vector<int>& order,
               std::vector<int>& color, int& n_colors);
void load_problem(BatchInst& bi, int n, int n_couplings, const int32_t* ci, const int32_t* cj,
                  const double* w, const double* fields, int n_pairs, const int32_t* pa,
                  const int32_t* pb);
void check_vec(const std::vector<double>& v, const char* what);
bool plane_eligible(tg_ctx& c, std::string* why);
uint64_t threshold_metropolis(double beta, double de);
uint64_t threshold_heat_bath(double beta, double local);
void ensure_host_arrays(tg_ctx& c);
void ensure_host_canonical(tg_ctx& c);
void build_plane_structure_device(tg_ctx& c, std::vector<PlaneType>& types, std::vector<Chunk>& chunks,
                                  std::vector<int>& chunk_off);
void build_plane(tg_ctx& c);
void build_plane_types_device(tg_ctx& c, std::vector<PlaneType>& types, std::vector<int>& chunk_off,
                              RunTable& rt);
void build_plane_rest(tg_ctx& c, std::vector<PlaneType>& types, const std::vector<int>& chunk_off);
void build_slot(tg_ctx& c);
PlaneArgs plane_args(tg_ctx& c);
SlotArgs slot_args(tg_ctx& c);
SwapArgs swap_args(tg_ctx& c);
void launch_sweep(tg_ctx& c, int64_t t0, const RoundState* rs = nullptr);
void rebuild_planes(tg_ctx& c);
void do_init(tg_ctx& c, const tg_run_config* cfg);
void drain(tg_ctx& c, int filled, int64_t first_round, const SinkCtx& sink, bool dig_array = false);
void profile_chunk(tg_ctx& c, int filled, double& sweep_ms, double& other_ms);
void do_advance_fused(tg_ctx& c, int64_t n_rounds, const SinkCtx& sink);
int single_sink_adapter(void* user, int32_t, const tg_record* recs, int64_t n, const int8_t* st,
                        const int64_t* ap, const int64_t* ab);
void do_advance(tg_ctx& c, int64_t n_rounds, const SinkCtx& sink);
void s2_bands(S2Prep& P, double bmax, double pmax);
void s2_prepare(S2Prep& P, const BatchInst& bi);
S2Args s2_args(tg_ctx& c);
KLArgs kl_args(tg_ctx& c);
S2Swap s2_swap(tg_ctx& c);
void s2_build(tg_ctx& c, const tg_run_config* cfg);
void s2_drain(tg_ctx& c, int filled, int64_t first_round, const BatchSinkCtx& sink);
void s2_advance(tg_ctx& c, int64_t n_rounds, const BatchSinkCtx& sink);
void s2_get_state(tg_ctx& c, int b, int slot, int8_t* out);
void s2_counters(tg_ctx& c, int b, int64_t* attempts_p, int64_t* accepts_p, int64_t* attempts_b,
                 int64_t* accepts_b);
void s2_energies(tg_ctx& c, int b, double* f, double* g);
void probe_run(tg_ctx& c, double beta, double penalty, int n_chains, int sweeps, uint64_t seed,
               int rule, tg_probe_stats* out);
double median_of(std::vector<double> v);
void build_schedule(tg_ctx& c, const tg_schedule_config& cfg, std::vector<double>& betas,
                    std::vector<double>& pens, std::vector<tg_probe_stats>& stats, bool& exhausted);

}  // namespace tgh
