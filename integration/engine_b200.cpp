// integration/engine_b200.cpp -- the reference-side binding of the B200 engine.
//
// A maintainer of the reference (`tempergrid`, /root/reference/proj) adds this
// one translation unit to proj/src/ and links libtempergrid_b200.so; it
// provides
//
//     Trace tempergrid::run_2dpt_b200(const ConstrainedProblem&, const Schedule&,
//                                     const RunConfig&, const B200Options& = {});
//     BaselineTrace tempergrid::run_jcolumn_pt_b200(const ConstrainedProblem&,
//                                     const std::vector<double>& betas, double p_fixed,
//                                     int j_repeats, const RunConfig&, const B200Options& = {});
//
// with the exact signature, validation, exceptions and Trace contents of
// tempergrid::run_2dpt (include/tempergrid/engine.hpp:62-63, src/engine.cpp:83-219),
// so call sites such as cli.cpp:357 switch by renaming the call.  Everything
// crosses the C ABI of include/tempergrid_b200.h: plain arrays in, records out
// through the sink, status codes mapped back to config_error / resource_error
// (errors.hpp:10-18).
//
// In this repository the file is compiled against the reference headers by
// oracle/Makefile (target `shim`) and exercised by tests/test_integration.py,
// which checks that run_2dpt_b200 and the reference's run_2dpt produce
// byte-identical trace_to_jsonl output when both consume Philox draws.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "tempergrid/engine.hpp"
#include "tempergrid/errors.hpp"
#include "tempergrid_b200.h"

namespace tempergrid {

struct B200Options {
    int device = 0;
    int rule = TG_RULE_METROPOLIS;
    int engine = TG_ENGINE_SLOT;  // SLOT keeps the reference's per-slot RNG association
};

namespace {

[[noreturn]] void raise(tg_ctx* ctx, int code) {
    char buf[512];
    tg_last_error(ctx, buf, sizeof buf);
    if (code == TG_ERR_CONFIG) throw config_error(buf);
    if (code == TG_ERR_RESOURCE) throw resource_error(buf);
    throw std::runtime_error(std::string("tempergrid_b200: ") + buf);
}

struct Collect {
    Trace* trace;
    int n, R;
    bool grid;
    std::vector<std::int64_t> att_p, att_b;  // cumulative attempts (deterministic)
    int I, J;
    std::int64_t last_round = 0;
};

void add_attempts(Collect& c, std::int64_t round) {
    const int even = round % 2 == 0;
    const int direction = ((round - 1) / 2) % 2 == 0 ? 1 : -1;
    bool dp, db;
    if (c.I == 1 && c.J == 1) dp = db = false;
    else if (c.I == 1) { dp = true; db = false; }
    else if (c.J == 1) { dp = false; db = true; }
    else { dp = direction == 1; db = !dp; }
    if (dp) for (int i = 0; i < c.I; ++i) for (int p = even; p + 1 < c.J; p += 2) ++c.att_p[i * (c.J - 1) + p];
    if (db) for (int j = 0; j < c.J; ++j) for (int b = even; b + 1 < c.I; b += 2) ++c.att_b[b * c.J + j];
}

int sink(void* user, const tg_record* recs, std::int64_t n_recs, const std::int8_t* states,
         const std::int64_t* acc_p, const std::int64_t* acc_b) {
    Collect& c = *static_cast<Collect*>(user);
    const std::size_t np = c.att_p.size(), nb = c.att_b.size();
    const std::size_t per = c.grid ? static_cast<std::size_t>(c.R) * c.n : c.n;
    for (std::int64_t k = 0; k < n_recs; ++k) {
        const tg_record& r = recs[k];
        while (c.last_round < r.round) add_attempts(c, ++c.last_round);
        TraceRecord rec;  // engine.cpp:189-214
        rec.round = r.round;
        rec.sweep_count = r.sweep_count;
        rec.f = r.f;
        rec.g = r.g;
        rec.feasible = r.feasible != 0;
        const std::int8_t* s = states + k * per;
        if (c.grid) {
            for (int q = 0; q < c.R; ++q)
                rec.grid.emplace_back(s + static_cast<std::size_t>(q) * c.n,
                                      s + static_cast<std::size_t>(q + 1) * c.n);
            rec.state = rec.grid.back();
        } else {
            rec.state.assign(s, s + c.n);
        }
        rec.acceptance_rates_p.resize(np);
        for (std::size_t q = 0; q < np; ++q)
            rec.acceptance_rates_p[q] =
                c.att_p[q] == 0 ? 0.0 : static_cast<double>(acc_p[k * np + q]) / c.att_p[q];
        rec.acceptance_rates_beta.resize(nb);
        for (std::size_t q = 0; q < nb; ++q)
            rec.acceptance_rates_beta[q] =
                c.att_b[q] == 0 ? 0.0 : static_cast<double>(acc_b[k * nb + q]) / c.att_b[q];
        c.trace->records.push_back(std::move(rec));
    }
    return 0;
}

void set_problem(tg_ctx* ctx, const ConstrainedProblem& problem) {
    const IsingModel& cost = problem.cost;
    std::vector<std::int32_t> ci, cj, pa, pb;
    std::vector<double> w;
    for (const Coupling& c : cost.couplings()) {
        ci.push_back(c.i);
        cj.push_back(c.j);
        w.push_back(c.weight);
    }
    for (const auto& [a, b] : problem.constraints.pairs()) {
        pa.push_back(a);
        pb.push_back(b);
    }
    const int rc = tg_set_problem(ctx, cost.n_spins(), static_cast<int>(ci.size()), ci.data(),
                                  cj.data(), w.data(), cost.fields().data(),
                                  static_cast<int>(pa.size()), pa.data(), pb.data());
    if (rc != TG_OK) raise(ctx, rc);
}

}  // namespace

Trace run_2dpt_b200(const ConstrainedProblem& problem, const Schedule& schedule,
                    const RunConfig& cfg, const B200Options& opt = {}) {
    tg_ctx* ctx = nullptr;
    int rc = tg_create(opt.device, &ctx);
    if (rc != TG_OK) raise(nullptr, rc);
    struct Guard {
        tg_ctx* c;
        ~Guard() { tg_destroy(c); }
    } guard{ctx};

    const IsingModel& cost = problem.cost;
    set_problem(ctx, problem);
    rc = tg_set_schedule(ctx, static_cast<int>(schedule.betas.size()), schedule.betas.data(),
                         static_cast<int>(schedule.penalties.size()), schedule.penalties.data());
    if (rc != TG_OK) raise(ctx, rc);
    if (cfg.threads < 1) throw config_error("run: threads must be >= 1");  // engine.cpp:57

    Trace trace;
    trace.betas = schedule.betas;
    trace.penalties = schedule.penalties;
    trace.sweeps_per_swap = cfg.sweeps_per_swap;
    Collect col;
    col.trace = &trace;
    col.n = cost.n_spins();
    col.I = static_cast<int>(schedule.betas.size());
    col.J = static_cast<int>(schedule.penalties.size());
    col.R = col.I * col.J;
    col.grid = !cfg.store_target_only;
    col.att_p.assign(col.I * std::max(0, col.J - 1), 0);
    col.att_b.assign(std::max(0, col.I - 1) * col.J, 0);

    tg_run_config rc_cfg{};
    rc_cfg.total_sweeps = cfg.total_sweeps;
    rc_cfg.sweeps_per_swap = cfg.sweeps_per_swap;
    rc_cfg.seed = cfg.seed;
    rc_cfg.rule = opt.rule;
    rc_cfg.engine = opt.engine;
    rc_cfg.record_flags = TG_REC_COUNTERS | (col.grid ? TG_REC_GRID : TG_REC_STATE);
    rc_cfg.record_every = 1;
    rc = tg_run(ctx, &rc_cfg, &sink, &col);
    if (rc != TG_OK) raise(ctx, rc);
    return trace;
}

// run_jcolumn_pt (engine.cpp:221-270): all j_repeats columns run as one device
// batch (tg_run_jcolumn), merged per round into the reference's BaselineTrace.
BaselineTrace run_jcolumn_pt_b200(const ConstrainedProblem& problem,
                                  const std::vector<double>& betas, double p_fixed,
                                  int j_repeats, const RunConfig& cfg,
                                  const B200Options& opt = {}) {
    if (p_fixed <= 0.0) throw config_error("baseline: P must be positive");
    if (j_repeats < 1) throw config_error("baseline: repeats must be >= 1");
    tg_ctx* ctx = nullptr;
    int rc = tg_create(opt.device, &ctx);
    if (rc != TG_OK) raise(nullptr, rc);
    struct Guard {
        tg_ctx* c;
        ~Guard() { tg_destroy(c); }
    } guard{ctx};
    set_problem(ctx, problem);
    if (cfg.threads < 1) throw config_error("run: threads must be >= 1");
    tg_run_config rc_cfg{};
    rc_cfg.total_sweeps = cfg.total_sweeps;
    rc_cfg.sweeps_per_swap = cfg.sweeps_per_swap;
    rc_cfg.seed = cfg.seed;
    rc_cfg.rule = opt.rule;
    rc_cfg.engine = TG_ENGINE_SLOT;
    rc_cfg.record_every = 1;
    const std::int64_t rounds =
        cfg.sweeps_per_swap >= 1 ? cfg.total_sweeps / cfg.sweeps_per_swap : 0;
    std::vector<tg_baseline_record> recs(static_cast<std::size_t>(std::max<std::int64_t>(rounds, 1)));
    double ff = 0.0;
    rc = tg_run_jcolumn(ctx, static_cast<int>(betas.size()), betas.data(), p_fixed, j_repeats,
                        &rc_cfg, recs.data(), rounds, &ff);
    if (rc != TG_OK) raise(ctx, rc);
    BaselineTrace out;
    out.betas = betas;
    out.penalty = p_fixed;
    out.sweeps_per_swap = cfg.sweeps_per_swap;
    for (std::int64_t k = 0; k < rounds; ++k) {
        BaselineRecord r;
        r.round = recs[k].round;
        r.sweep_count = recs[k].sweep_count;
        r.best_f = recs[k].best_f;
        r.any_feasible = recs[k].any_feasible != 0;
        r.n_feasible = recs[k].n_feasible;
        r.n_total = recs[k].n_total;
        out.records.push_back(r);
    }
    out.feasible_fraction = ff;
    return out;
}

}  // namespace tempergrid

namespace {
std::string baseline_text(const tempergrid::BaselineTrace& t) {
    std::string s;
    char buf[160];
    for (const auto& r : t.records) {
        std::snprintf(buf, sizeof buf, "%lld %lld %.17g %d %d %d\n", (long long)r.round,
                      (long long)r.sweep_count, r.best_f, r.any_feasible ? 1 : 0, r.n_feasible,
                      r.n_total);
        s += buf;
    }
    std::snprintf(buf, sizeof buf, "fraction %.17g\n", t.feasible_fraction);
    return s + buf;
}
}  // namespace

// C entry for tests: the reference run_jcolumn_pt and run_jcolumn_pt_b200 on
// the same inputs, each serialised record by record (%.17g doubles).
extern "C" int tg_shim_compare_jcolumn(int n, int nc, const int* ci, const int* cj, const double* w,
                                       const double* h, int np, const int* pa, const int* pb,
                                       int I, const double* betas, double p_fixed, int repeats,
                                       std::int64_t total, std::int64_t sps, std::uint64_t seed,
                                       char* ref_out, std::size_t ref_cap, char* gpu_out,
                                       std::size_t gpu_cap, char* err, int errlen) {
    using namespace tempergrid;
    try {
        std::vector<Coupling> cs;
        for (int k = 0; k < nc; ++k) cs.push_back({ci[k], cj[k], w[k]});
        std::vector<std::pair<int, int>> pairs;
        for (int k = 0; k < np; ++k) pairs.emplace_back(pa[k], pb[k]);
        ConstrainedProblem problem{IsingModel(n, cs, std::vector<double>(h, h + n)),
                                   ConstraintSet(n, pairs)};
        std::vector<double> b(betas, betas + I);
        RunConfig cfg;
        cfg.total_sweeps = total;
        cfg.sweeps_per_swap = sps;
        cfg.seed = seed;
        const std::string a = baseline_text(run_jcolumn_pt(problem, b, p_fixed, repeats, cfg));
        const std::string g = baseline_text(run_jcolumn_pt_b200(problem, b, p_fixed, repeats, cfg));
        if (a.size() + 1 > ref_cap || g.size() + 1 > gpu_cap) return -3;
        std::copy(a.begin(), a.end(), ref_out);
        ref_out[a.size()] = '\0';
        std::copy(g.begin(), g.end(), gpu_out);
        gpu_out[g.size()] = '\0';
        return 0;
    } catch (const std::exception& e) {
        std::string m = e.what();
        if (errlen > 0) {
            const std::size_t k = std::min<std::size_t>(m.size(), errlen - 1);
            std::copy(m.begin(), m.begin() + k, err);
            err[k] = '\0';
        }
        return -1;
    }
}

// C entry for tests: run both the reference run_2dpt and run_2dpt_b200 on the
// same inputs and return their trace_to_jsonl texts.
extern "C" int tg_shim_compare(int n, int nc, const int* ci, const int* cj, const double* w,
                               const double* h, int np, const int* pa, const int* pb, int I,
                               const double* betas, int J, const double* pens,
                               std::int64_t total, std::int64_t sps, std::uint64_t seed,
                               int store_grid, char* ref_out, std::size_t ref_cap, char* gpu_out,
                               std::size_t gpu_cap, char* err, int errlen) {
    using namespace tempergrid;
    try {
        std::vector<Coupling> cs;
        for (int k = 0; k < nc; ++k) cs.push_back({ci[k], cj[k], w[k]});
        std::vector<std::pair<int, int>> pairs;
        for (int k = 0; k < np; ++k) pairs.emplace_back(pa[k], pb[k]);
        ConstrainedProblem problem{IsingModel(n, cs, std::vector<double>(h, h + n)),
                                   ConstraintSet(n, pairs)};
        Schedule schedule;
        schedule.betas.assign(betas, betas + I);
        schedule.penalties.assign(pens, pens + J);
        RunConfig cfg;
        cfg.total_sweeps = total;
        cfg.sweeps_per_swap = sps;
        cfg.seed = seed;
        cfg.store_target_only = store_grid == 0;
        const std::string a = trace_to_jsonl(run_2dpt(problem, schedule, cfg));
        const std::string b = trace_to_jsonl(run_2dpt_b200(problem, schedule, cfg));
        if (a.size() + 1 > ref_cap || b.size() + 1 > gpu_cap) return -3;
        std::copy(a.begin(), a.end(), ref_out);
        ref_out[a.size()] = '\0';
        std::copy(b.begin(), b.end(), gpu_out);
        gpu_out[b.size()] = '\0';
        return 0;
    } catch (const std::exception& e) {
        std::string m = e.what();
        if (errlen > 0) {
            const std::size_t k = std::min<std::size_t>(m.size(), errlen - 1);
            std::copy(m.begin(), m.begin() + k, err);
            err[k] = '\0';
        }
        return -1;
    }
}
