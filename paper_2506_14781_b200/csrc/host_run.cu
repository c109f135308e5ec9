// host_run.cu -- run_2dpt round loop on the host side: init, record draining, the per-round launch sequence and the NCCL (f, g) exchange.
#include "host.cuh"

namespace tgh {

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

void launch_sweep(tg_ctx& c, int64_t t0, const RoundState* rs) {
    const int sps = (int)c.cfg.sweeps_per_swap;
    if (c.engine == TG_ENGINE_PLANE) {
        PlaneArgs a = plane_args(c);
        a.rs = rs;
        int64_t t = t0;
        int nsw = sps;
        void* args[] = {&a, &t, &nsw};
        if (c.c5_sweep_grid > 0) {
            int nf0 = c.c5_nfree[0], nf1 = c.c5_nfree[1];
            void* args5[] = {&a, &t, &nsw, &nf0, &nf1};
            c.sweep_kernel = "plane_c5_sweep_kernel";
            CK(cudaLaunchCooperativeKernel(plane_c5_sweep_fn(c.cfg.rule), dim3(c.c5_sweep_grid), dim3(kC5Threads),
                                           args5, c.c5_sweep_smem, c.stream));
        } else if (c.tpw_sweep_grid > 0) {
            c.sweep_kernel = "plane_tpw_sweep_kernel";
            CK(cudaLaunchCooperativeKernel(plane_tpw_sweep_fn(c.cfg.rule, c.tpw_fast), dim3(c.tpw_sweep_grid),
                                           dim3(kTpwThreads), args, c.tpw_sweep_smem, c.stream));
        } else {
            c.sweep_kernel = "plane_sweep_kernel";
            CK(cudaLaunchCooperativeKernel(plane_sweep_fn(c.cfg.rule, c.WV), dim3(c.plane_grid),
                                           dim3(kPlaneThreads), args, 0, c.stream));
        }
    } else {
        SlotArgs a = slot_args(c);
        a.rs = rs;
        int64_t t = t0;
        int nsw = sps;
        void* args[] = {&a, &t, &nsw};
        c.sweep_kernel = "slot_sweep_kernel";
        CK(cudaLaunchKernel(c.slot_D ? slot_sweep_fn_d(c.slot_D) : slot_sweep_fn(), dim3(c.R_local),
                            dim3(kSlotThreads), args, c.slot_smem, c.stream));
    }
    c.sweep_launches++;
}

// Labels and thresholds for the current slot assignment: run the swap
// kernel's plane-rebuild with a round that attempts nothing.
void do_init(tg_ctx& c, const tg_run_config* cfg) {
    HostTimer tm_("init (total)");
    c.clear_graphs();  // captured kernel arguments point at the previous buffers
    c.graphs_ok = true;
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
    if (c.kl.on && ((eng != TG_ENGINE_SLOT && eng != TG_ENGINE_FLOAT) || c.world != 1 || std::getenv("TG_SLOT_V1")))
        fail(TG_ERR_CONFIG, "kl decoder: needs the single-GPU SLOT or FLOAT engine");
    if (eng == TG_ENGINE_PLANE && !plane_eligible(c, &why))
        fail(TG_ERR_CONFIG, "plane engine: instance not eligible (%s)", why.c_str());
    if (eng == TG_ENGINE_FLOAT && c.world != 1) fail(TG_ERR_CONFIG, "float engine: single-GPU contexts only");
    if (eng != TG_ENGINE_PLANE && eng != TG_ENGINE_SLOT && eng != TG_ENGINE_FLOAT)
        fail(TG_ERR_CONFIG, "unknown engine %d", eng);
    c.engine = eng;
    {
        int32_t s0 = 0, cnt = 0;
        if (tg_partition(c.R, c.rank, c.world, eng == TG_ENGINE_FLOAT ? TG_ENGINE_SLOT : eng, &s0, &cnt) != TG_OK)
            fail(TG_ERR_CONFIG, "grid of %d replicas does not split over %d ranks%s", c.R, c.world,
                 eng == TG_ENGINE_PLANE ? " in 32-replica words" : "");
        c.state0 = s0;
        c.R_local = cnt;
    }
    cudaStream_t st = c.stream;
    CK(cudaSetDevice(c.device));
    c.use_s2 = false;
    if ((eng == TG_ENGINE_SLOT && c.world == 1 && !c.dist && !std::getenv("TG_SLOT_V1")) || eng == TG_ENGINE_FLOAT) {
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
        plane_init_kernel<<<c.sms * 16, 256, 0, st>>>(c.d_spins32.p, c.n, c.W, c.R_local, c.state0, c.cfg.seed);
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

void drain(tg_ctx& c, int filled, int64_t first_round, const SinkCtx& sink, bool dig_array) {
    if (filled <= 0) return;
    cudaStream_t st = c.stream;
    CK(cudaMemcpyAsync(c.h_rec.data(), c.d_rec.p, sizeof(TgRecordDev) * filled, cudaMemcpyDeviceToHost, st));
    if (dig_array) {  // unfused loop: digests gathered (and all-reduced) in d_dig
        c.h_dig.resize(c.rec_cap);
        CK(cudaMemcpyAsync(c.h_dig.data(), c.d_dig.p, sizeof(uint64_t) * filled, cudaMemcpyDeviceToHost, st));
    }
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
        r.digest = dig_array ? c.h_dig[k] : d.digest;
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
    if (c.engine == TG_ENGINE_PLANE && c.world == 1 && !c.dist && c.fused_grid > 0 &&
        !(c.cfg.record_flags & TG_REC_GRID)) {
        do_advance_fused(c, n_rounds, sink);
        return;
    }
    cudaStream_t st = c.stream;
    const int flags = c.cfg.record_flags;
    const bool need_extract = (flags & (TG_REC_DIGEST | TG_REC_STATE | TG_REC_GRID)) != 0;
    const size_t per_state = (flags & TG_REC_GRID) ? (size_t)c.R * c.n : ((flags & TG_REC_STATE) ? (size_t)c.n : 0);
    if (c.profiling && (int)c.ev.size() < 2 * c.rec_cap + 1) {
        c.clear_graphs();  // graphs record the events they were captured with
        for (auto e : c.ev) cudaEventDestroy(e);
        c.ev.assign(2 * c.rec_cap + 1, nullptr);
        for (auto& e : c.ev) CK(cudaEventCreate(&e));
    }
    if (c.d_rstate.n < 1) c.d_rstate.alloc(1);
    if (c.d_dig.n < (size_t)c.rec_cap) c.d_dig.alloc(c.rec_cap);
    // every kernel of a round reads the device round state (round, swap-stream
    // position, record slot); round_tick_kernel advances it, so the launch
    // sequence of a chunk is the same every time and is replayed as a graph
    SwapArgs sa = swap_args(c);
    sa.rs = c.d_rstate.p;
    SwapArgs sa_noplane = sa;  // the swap kernel leaves the plane rebuild to plane_rebuild_kernel
    sa_noplane.plane = 0;
    sa_noplane.tick = c.d_rstate.p;  // and advances the round state (no separate tick launch)
    const int rebuild_blocks = std::max(1, std::min(c.sms, (c.W * 16 + 7) / 8));
    ExtractArgs e{};
    if (need_extract) {
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
        e.states = per_state ? c.d_rec_states.p : nullptr;
        e.digest = (flags & TG_REC_DIGEST) ? c.d_dig.p : nullptr;
        e.rs = c.d_rstate.p;
        e.rs_back = 1;
        e.per_state = per_state;
    }
    const long long ex_total = (long long)(e.all_slots ? c.R : 1) * c.n;
    const int ex_blocks = std::max(1, (int)std::min<long long>((ex_total + 255) / 256, (long long)c.sms * 8));
    NvtxRange nv_("tg: unfused rounds");
    auto one_round = [&](int k, bool capturing) {
        if (c.profiling)
            CK(capturing ? cudaEventRecordWithFlags(c.ev[2 * k], st, cudaEventRecordExternal)
                         : cudaEventRecord(c.ev[2 * k], st));
        launch_sweep(c, 0, c.d_rstate.p);
        if (c.profiling)
            CK(capturing ? cudaEventRecordWithFlags(c.ev[2 * k + 1], st, cudaEventRecordExternal)
                         : cudaEventRecord(c.ev[2 * k + 1], st));
        if (c.dist) {
            NvtxRange nx_("tg: (f, g) all-gather");
            NK(nccl().GroupStart());
            NK(nccl().AllGather(c.d_f.p + c.state0, c.d_f.p, c.R_local, ncclDouble, c.comm, st));
            NK(nccl().AllGather(c.d_g.p + c.state0, c.d_g.p, c.R_local, ncclDouble, c.comm, st));
            NK(nccl().GroupEnd());
        }
        swap_kernel<<<1, kSwapThreads, 0, st>>>(sa_noplane, 0, 0, 0, flags);
        CK(cudaGetLastError());
        if (sa.plane) {  // threshold planes of the new labels, grid-wide
            plane_rebuild_kernel<<<rebuild_blocks, 256, 0, st>>>(sa);
            CK(cudaGetLastError());
        }
        if (need_extract) {
            extract_kernel<<<ex_blocks, 256, 0, st>>>(e);
            CK(cudaGetLastError());
        }
    };
    const int per_round_other = 1 + (need_extract ? 1 : 0) + (sa.plane ? 1 : 0);
    // a graph of n rounds (captured once per chunk length); none if capture fails
    auto graph_for = [&](int n) -> cudaGraphExec_t {
        // Direct launches by default: measured on B200 (tools/dist_selftest_rate.py) a round of
        // the unfused loop is ~23 us shorter launched directly (the host runs ahead of these
        // 20-100 us kernels) than replayed as graph nodes; TG_GRAPHS=1 replays captured chunks.
        const char* ge = std::getenv("TG_GRAPHS");
        if (!c.graphs_ok || !ge || !std::atoi(ge) || std::getenv("TG_NO_GRAPHS")) return nullptr;
        auto it = c.graphs.find(n);
        if (it != c.graphs.end()) return it->second;
        const int64_t sl0 = c.sweep_launches;
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ex = nullptr;
        bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            try {
                for (int k = 0; k < n; ++k) one_round(k, true);
            } catch (const TgFail&) {
                ok = false;
            }
            ok = (cudaStreamEndCapture(st, &g) == cudaSuccess) && ok && g != nullptr;
        }
        if (ok) ok = cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();  // a failed capture leaves no sticky error
        c.sweep_launches = sl0;
        if (!ok) {
            c.graphs_ok = false;
            return nullptr;
        }
        c.graphs[n] = ex;
        return ex;
    };
    double sweep_ms = 0, swap_ms = 0;
    int64_t left = n_rounds;
    while (left > 0) {
        const int n = (int)std::min<int64_t>(left, c.rec_cap);
        const int64_t first_round = c.rounds_done + 1;
        c.h_rstate = RoundState{c.rounds_done, c.swap_base, 0, 0};
        CK(cudaMemcpyAsync(c.d_rstate.p, &c.h_rstate, sizeof(RoundState), cudaMemcpyHostToDevice, st));
        if (flags & TG_REC_DIGEST) CK(cudaMemsetAsync(c.d_dig.p, 0, sizeof(uint64_t) * n, st));
        if (cudaGraphExec_t gx = graph_for(n)) {
            CK(cudaGraphLaunch(gx, st));
            c.graph_launches++;
            c.sweep_launches += n;
        } else {
            for (int k = 0; k < n; ++k) one_round(k, false);
        }
        c.other_launches += (int64_t)n * per_round_other;
        for (int k = 0; k < n; ++k) c.swap_base += (uint64_t)round_attempts(c.I, c.J, first_round + k);
        c.rounds_done += n;
        left -= n;
        if (c.dist) {
            // target digests and snapshots: every rank wrote zeros for states it
            // does not hold, one all-reduce per chunk instead of one per round
            if (flags & TG_REC_DIGEST) NK(nccl().AllReduce(c.d_dig.p, c.d_dig.p, n, ncclUint64, ncclSum, c.comm, st));
            if (per_state)
                NK(nccl().AllReduce(c.d_rec_states.p, c.d_rec_states.p, per_state * n, ncclInt8, ncclSum, c.comm, st));
        }
        if (c.profiling) profile_chunk(c, n, sweep_ms, swap_ms);
        NvtxRange nr_("tg: drain records");
        drain(c, n, first_round, sink, (flags & TG_REC_DIGEST) != 0);
    }
    CK(cudaStreamSynchronize(st));
    c.last_sweep_ms = sweep_ms;
    c.last_swap_ms = swap_ms;
}


}  // namespace tgh
