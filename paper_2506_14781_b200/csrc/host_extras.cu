// host_extras.cu -- schedule probes and the adaptive ladder (schedule.cpp:18-163) on the device.
#include "host.cuh"

namespace tgh {


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


}  // namespace tgh
