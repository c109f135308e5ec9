// host_slot.cu -- SLOT engine host drivers: v1 (multi-GPU) structure and arguments, v2 (single GPU and batches) build / advance / read-back.
#include "host.cuh"

namespace tgh {

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
    {
        // = std::stable_sort by key (row x, then column y): a stable counting
        // sort by row, then a stable insertion sort inside each (short) row
        std::vector<int> pos(n + 1, 0);
        for (const E& e : ent) pos[(e.key >> 32) + 1]++;
        for (int i = 0; i < n; ++i) pos[i + 1] += pos[i];
        std::vector<E> srt(ent.size());
        std::vector<int> fill(pos.begin(), pos.end() - 1);
        for (const E& e : ent) srt[fill[e.key >> 32]++] = e;
        for (int i = 0; i < n; ++i)
            for (int a = pos[i] + 1; a < pos[i + 1]; ++a) {
                const E v = srt[a];
                int b = a - 1;
                while (b >= pos[i] && srt[b].key > v.key) { srt[b + 1] = srt[b]; --b; }
                srt[b + 1] = v;
            }
        ent.swap(srt);
    }
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
    {
        // = std::stable_sort by key (row x, then column y): a stable counting
        // sort by row, then a stable insertion sort inside each (short) row
        std::vector<int> pos(n + 1, 0);
        for (const E& e : ent) pos[(e.key >> 32) + 1]++;
        for (int i = 0; i < n; ++i) pos[i + 1] += pos[i];
        std::vector<E> srt(ent.size());
        std::vector<int> fill(pos.begin(), pos.end() - 1);
        for (const E& e : ent) srt[fill[e.key >> 32]++] = e;
        for (int i = 0; i < n; ++i)
            for (int a = pos[i] + 1; a < pos[i + 1]; ++a) {
                const E v = srt[a];
                int b = a - 1;
                while (b >= pos[i] && srt[b].key > v.key) { srt[b + 1] = srt[b]; --b; }
                srt[b + 1] = v;
            }
        ent.swap(srt);
    }
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
    a.lab = S.d_lab.p; a.fx = S.d_fx.p; a.gx = S.d_gx.p; a.fitem_pref = S.d_fitem_pref.p;
    a.flps = S.flps; a.fspw = S.fspw; a.fngs = S.fngs;
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
    s.lab = S.fast ? S.d_lab.p : nullptr;
    return s;
}

void s2_build(tg_ctx& c, const tg_run_config* cfg) {
    HostTimer tm_("batch: s2_build");
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
    S.fast = cfg->engine == TG_ENGINE_FLOAT && !S.probe;
    S.prep.assign(B, S2Prep{});
    S.state_off.clear();
    std::unique_ptr<HostTimer> tsec(new HostTimer("batch: s2_build prepare"));
    // per-instance host preprocessing (canonical order, merged CSR, padded
    // entries): independent instances run on host threads; repeats of one
    // instance (J-column baseline) copy the previous instance's result
    std::vector<char> dup(B, 0);
    std::vector<int> todo;
    for (int b = 0; b < B; ++b) {
        const BatchInst& x = c.batch[b];
        const BatchInst* y = b ? &c.batch[b - 1] : nullptr;
        dup[b] = y && x.n == y->n && x.ci == y->ci && x.cj == y->cj && x.cw == y->cw && x.h == y->h &&
                 x.pa == y->pa && x.pb == y->pb;
        if (!dup[b]) todo.push_back(b);
    }
    {
        const int nt = (int)std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                            std::min<size_t>(todo.size(), 32)));
        std::vector<std::exception_ptr> err(B);
        std::atomic<int> next{0};
        auto work = [&] {
            for (int k; (k = next.fetch_add(1)) < (int)todo.size();) {
                const int b = todo[k];
                try {
                    s2_prepare(S.prep[b], c.batch[b]);
                } catch (...) {
                    err[b] = std::current_exception();
                }
            }
        };
        run_pool(nt, work);
        for (int b = 0; b < B; ++b)  // the first failing instance's error, as a sequential loop would
            if (err[b]) std::rethrow_exception(err[b]);
    }
    for (int b = 1; b < B; ++b)
        if (dup[b]) {
            // same graph, possibly another schedule: the FP32 error bands
            // depend on this instance's own max |beta| and max P
            S.prep[b] = S.prep[b - 1];
            double pmax = 0.0, bmax = 0.0;
            for (double p : c.batch[b].pens) pmax = std::max(pmax, p);
            for (double be : c.batch[b].betas) bmax = std::max(bmax, std::fabs(be));
            s2_bands(S.prep[b], bmax, pmax);
        }
    int D = 4;
    for (const auto& P : S.prep) D = std::max(D, P.D);
    S.D = D;
    tsec.reset(new HostTimer("batch: s2_build concatenate"));
    // concatenate
    std::vector<SInst> inst(B);
    // the padded entry arrays are the largest: allocated without value-init so
    // their pages are first touched by the filling threads below
    std::unique_ptr<int2[]> entp;
    std::unique_ptr<double[]> wp;
    std::vector<double> w, h, betas, pens;
    std::vector<int> off, cstart, perm;
    std::vector<int32_t> nbr;
    std::vector<int8_t> cm;
    std::vector<float> h32;
    std::vector<uint64_t> keys((size_t)B * S.R), swap_seed(B), seeds(B);
    long long spin_off = 0;
    int chunk_off = 0, state_off = 0, max_colors = 0;
    // offsets of every instance in each concatenated array, then the copies
    // on host threads (instances are independent)
    struct Cat { size_t cst, ent, off, nbr, w, cm, h, h32, perm; };
    std::vector<Cat> at(B + 1, Cat{0, 0, 0, 0, 0, 0, 0, 0, 0});
    for (int b = 0; b < B; ++b) {
        const S2Prep& P = S.prep[b];
        const Cat& a = at[b];
        at[b + 1] = Cat{a.cst + P.color_start.size(), a.ent + (size_t)P.n * D, a.off + P.off.size(),
                        a.nbr + P.nbr.size(), a.w + P.w.size(), a.cm + P.cm.size(), a.h + P.h.size(),
                        a.h32 + P.h32.size(), a.perm + P.order.size()};
    }
    // the device table keeps 32-bit offsets (entp_off, csr_off, nbr_off, h_off)
    if (at[B].ent > (size_t)INT_MAX || at[B].off > (size_t)INT_MAX || at[B].nbr > (size_t)INT_MAX ||
        at[B].h > (size_t)INT_MAX)
        fail(TG_ERR_RESOURCE, "batch: concatenated instance arrays exceed 2^31 entries");
    cstart.resize(at[B].cst);
    entp.reset(new int2[std::max<size_t>(at[B].ent, 1)]);
    wp.reset(new double[std::max<size_t>(at[B].ent, 1)]);
    off.resize(at[B].off);
    nbr.resize(at[B].nbr);
    w.resize(at[B].w);
    cm.resize(at[B].cm);
    h.resize(at[B].h);
    h32.resize(at[B].h32);
    perm.resize(at[B].perm);
    for (int b = 0; b < B; ++b) {
        S2Prep& P = S.prep[b];
        SInst& in = inst[b];
        in.n = P.n;
        in.D = D;
        in.n_colors = P.n_colors;
        in.color_off = (int)at[b].cst;
        in.spin_off = spin_off;
        spin_off += (long long)P.n * S.Rp;
        in.entp_off = (int)at[b].ent;
        in.csr_off = (int)at[b].off;
        in.nbr_off = (int)at[b].nbr;
        in.h_off = (int)at[b].h;
        in.n_chunks = (P.n + 31) / 32;
        in.chunk_off = chunk_off;
        chunk_off += in.n_chunks;
        in.state_off = state_off;
        S.state_off.push_back(state_off);
        state_off += P.n;
        in.eps = P.eps;
        in.beta_max = P.beta_max;
        in.pkey = derive_seed(c.batch[b].seed, kPurposePack, 0);
        max_colors = std::max(max_colors, P.n_colors);
        betas.insert(betas.end(), c.batch[b].betas.begin(), c.batch[b].betas.end());
        pens.insert(pens.end(), c.batch[b].pens.begin(), c.batch[b].pens.end());
        seeds[b] = c.batch[b].seed;
        for (int r = 0; r < S.R; ++r)
            keys[(size_t)b * S.R + r] = S.probe ? derive_seed(c.batch[b].seed, kPurposeProbe, (uint64_t)r)
                                                : derive_seed(c.batch[b].seed, kPurposeReplica, (uint64_t)r);
        swap_seed[b] = derive_seed(c.batch[b].seed, kPurposeSwap, 0);
    }
    {
        auto fill = [&](int b) {
            const S2Prep& P = S.prep[b];
            const Cat& a = at[b];
            std::copy(P.color_start.begin(), P.color_start.end(), cstart.begin() + a.cst);
            int2* ep = entp.get() + a.ent;
            double* wq = wp.get() + a.ent;
            for (int i = 0; i < P.n; ++i)
                for (int k = 0; k < D; ++k) {
                    *ep++ = k < P.D ? P.entp[(size_t)i * P.D + k] : make_int2(i, 0);
                    *wq++ = k < P.D ? P.wp[(size_t)i * P.D + k] : 0.0;
                }
            std::copy(P.off.begin(), P.off.end(), off.begin() + a.off);
            std::copy(P.nbr.begin(), P.nbr.end(), nbr.begin() + a.nbr);
            std::copy(P.w.begin(), P.w.end(), w.begin() + a.w);
            std::copy(P.cm.begin(), P.cm.end(), cm.begin() + a.cm);
            std::copy(P.h.begin(), P.h.end(), h.begin() + a.h);
            std::copy(P.h32.begin(), P.h32.end(), h32.begin() + a.h32);
            std::copy(P.order.begin(), P.order.end(), perm.begin() + a.perm);
        };
        const int nt = (int)std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                            (unsigned)std::min(B, 16)));
        std::atomic<int> next{0};
        auto work = [&] {
            for (int b; (b = next.fetch_add(1)) < B;) fill(b);
        };
        run_pool(nt, work);
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
    tsec.reset(new HostTimer("batch: s2_build uploads"));
    S.d_inst.upload(inst, st);
    S.h_inst = inst;
    S.d_entp.upload(entp.get(), at[B].ent, st);
    S.d_wp.upload(wp.get(), at[B].ent, st);
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
    tsec.reset(new HostTimer("batch: s2_build grid/rest"));
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
    if (S.fast) {
        // FLOAT engine: lanes per site, sites per warp item, 256-replica group
        // sets; warp items per colour and instance (prefix sums)
        int maxdeg = 0;
        for (const auto& P : S.prep)
            for (int i = 0; i < P.n; ++i) maxdeg = std::max(maxdeg, P.off[i + 1] - P.off[i]);
        if (maxdeg > 8) fail(TG_ERR_RESOURCE, "float engine: merged degree %d > 8", maxdeg);
        S.fdeg = maxdeg <= 3 && D == 4 ? 3 : (maxdeg <= 4 && D == 4 ? 4 : 8);
        if (S.fdeg == 8 && D != 8) fail(TG_ERR_RESOURCE, "float engine: padded degree %d", D);
        const int g8 = S.Rp / 8;
        S.flps = std::min(32, g8);
        S.fspw = 32 / S.flps;
        S.fngs = (g8 + 31) / 32;
        std::vector<int> fpref((size_t)max_colors * (B + 1), 0);
        for (int col = 0; col < max_colors; ++col)
            for (int b = 0; b < B; ++b) {
                const S2Prep& P = S.prep[b];
                const int len = col < P.n_colors ? P.color_start[col + 1] - P.color_start[col] : 0;
                fpref[(size_t)col * (B + 1) + b + 1] = fpref[(size_t)col * (B + 1) + b] + (len + S.fspw - 1) / S.fspw;
            }
        S.d_fitem_pref.upload(fpref, st);
        const void* fn = slotf_sweep_fn(S.cfg.rule, S.fdeg);
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSlotFThreads, 0));
        if (per_sm < 1) fail(TG_ERR_RESOURCE, "float engine: sweep kernel does not fit on an SM");
        const int wpb = kSlotFThreads / 32;
        long long need = 0;  // no more warps than the widest colour phase can use
        for (int col = 0; col < max_colors; ++col)
            need = std::max<long long>(need, (long long)fpref[(size_t)col * (B + 1) + B] * S.fngs);
        int blocks = (int)std::min<long long>((long long)per_sm * c.sms, (need + wpb - 1) / wpb);
        blocks = std::max(blocks, 1);
        while (blocks > 1 && (blocks * wpb) % S.fngs != 0) --blocks;
        if ((blocks * wpb) % S.fngs != 0) fail(TG_ERR_RESOURCE, "float engine: cannot tile %d group sets", S.fngs);
        S.grid = blocks;
        S.d_fx.alloc((size_t)B * S.Rp);
        S.d_gx.alloc((size_t)B * S.Rp);
        S.d_fx.zero(st);
        S.d_gx.zero(st);
        std::vector<float2> lab((size_t)B * S.Rp, make_float2(0.f, 0.f));
        for (int b = 0; b < B; ++b)
            for (int r = 0; r < S.R; ++r)
                lab[(size_t)b * S.Rp + r] = make_float2((float)c.batch[b].betas[r / S.J],
                                                        (float)(2.0 * c.batch[b].pens[r % S.J]));
        S.d_lab.upload(lab, st);
    } else {
        S.d_lab.release();
        S.d_fx.release();
        S.d_gx.release();
    }
    // fused per-warp energy partials cost B x nsub x Rp doubles of traffic per
    // round; past a few MB a separate pass over the spins is cheaper
    S.sep_energy = !S.fast && ((size_t)B * S.nsub * S.Rp * 16 > ((size_t)8 << 20) || std::getenv("TG_SLOT_SEP_ENERGY"));
    if (S.sep_energy) {
        S.e_slices = std::max(1, (c.sms * 8) / std::max(1, B * S.G));
        S.d_epart.alloc((size_t)2 * B * S.e_slices * S.R);
    }
    S.d_part_f.alloc(S.sep_energy || S.fast ? 0 : (size_t)B * S.nsub * S.Rp);
    S.d_part_g.alloc(S.sep_energy || S.fast ? 0 : (size_t)B * S.nsub * S.Rp);
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
    if (S.d_rec_states.p) {
        if (filled == cap) {
            CK(cudaMemcpyAsync(S.h_states.data(), S.d_rec_states.p, S.h_states.size(),
                               cudaMemcpyDeviceToHost, st));
        } else {  // only the filled rows of each instance's block
            for (int b = 0; b < B; ++b) {
                const size_t o = (size_t)S.state_off[b] * S.slots * cap;
                CK(cudaMemcpyAsync(S.h_states.data() + o, S.d_rec_states.p + o,
                                   (size_t)filled * S.prep[b].n * S.slots, cudaMemcpyDeviceToHost, st));
            }
        }
    }
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
    NvtxRange nv_("tg: slot/float rounds");
    HostTimer tm_("batch: s2_advance");
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
        if (S.fast) {
            c.sweep_kernel = "slotf_sweep_kernel";
            CK(cudaLaunchCooperativeKernel(slotf_sweep_fn(S.cfg.rule, S.fdeg), dim3(S.grid), dim3(kSlotFThreads),
                                           args, 0, st));
        } else {
            c.sweep_kernel = "slot2_sweep_kernel";
            CK(cudaLaunchCooperativeKernel(slot2_sweep_fn(S.D), dim3(S.grid), dim3(kSlot2Threads), args, 0, st));
        }
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

}  // namespace tgh
