// capi.cu -- the C ABI entry points (include/tempergrid_b200.h).
//
// A tg_ctx owns the device copy of one ConstrainedProblem in canonical colour
// order, the replica grid labels and the round loop of run_2dpt
// (/root/reference/proj/src/engine.cpp:83-219).  The drivers behind these
// entry points live in host_*.cu (host.cuh): instance validation and the
// device preprocessing (host_common.cu, prep.cu), the PLANE and SLOT engines
// (host_plane.cu, host_slot.cu), the round loop and record draining
// (host_run.cu), schedule probes (host_extras.cu).  Every entry point runs
// under guard(): C++ exceptions become status codes + tg_last_error.
#include <thread>

#include "host.cuh"

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
        // TG_DIST_SELFTEST=1 with an id and world == 1: a one-rank communicator, and the
        // engine takes the multi-GPU round loop (sweep launches, NCCL all-gather /
        // all-reduce inside the captured graph) so that path runs on a single GPU
        const bool selftest = world == 1 && nccl_id && std::getenv("TG_DIST_SELFTEST") &&
                              std::atoi(std::getenv("TG_DIST_SELFTEST")) != 0;
        if (world > 1 || selftest) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            NK(nccl().CommInitRank(&c->comm, world, id, rank));
            c->dist = true;
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
        // the extract kernel's one-slot mode reads slot R-1: a grid truncated
        // after `slot` makes that the slot asked for (state looked up on device)
        DBuf<int8_t> dst;
        dst.alloc(c.n);
        ExtractArgs e{};
        e.n = c.n;
        e.R = slot + 1;
        e.W = c.W;
        e.plane = c.engine == TG_ENGINE_PLANE;
        e.all_slots = 0;
        e.local_states = c.R_local;
        e.state0 = c.state0;
        e.slot_state = c.d_slot_state.p;
        e.spins32 = c.d_spins32.p;
        e.spins8 = c.d_spins8.p;
        e.perm = c.d_perm.p;
        e.states = dst.p;
        e.digest = nullptr;
        extract_kernel<<<std::max(1, std::min((c.n + 255) / 256, c.sms * 8)), 256, 0, c.stream>>>(e);
        CK(cudaGetLastError());
        if (c.dist) NK(nccl().AllReduce(dst.p, dst.p, c.n, ncclInt8, ncclSum, c.comm, c.stream));
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
    std::snprintf(info->sweep_kernel, sizeof(info->sweep_kernel), "%s", ctx->sweep_kernel);
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
    HostTimer tm_("batch: add");
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
        if (cfg->engine != TG_ENGINE_AUTO && cfg->engine != TG_ENGINE_SLOT && cfg->engine != TG_ENGINE_FLOAT)
            fail(TG_ERR_CONFIG, "batch: only the SLOT and FLOAT engines run batches");
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
