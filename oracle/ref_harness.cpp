// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter over the reference library's own entry point,
// tempergrid::run_2dpt (/root/reference/proj/include/tempergrid/engine.hpp:62-63,
// src/engine.cpp:83-219), compiled together with the reference sources into
// oracle/_ref/libtgref_*.so (recipe: oracle/Makefile).  It takes the same
// plain-array structs as the C port (tg_oracle.h) so tests can run the port,
// the reference and the B200 engine on identical inputs.  Exceptions map to
// the CLI's exit codes (cli.cpp:659-668): config_error -> 2, resource_error -> 3.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tempergrid/constraints.hpp"
#include "tempergrid/engine.hpp"
#include "tempergrid/errors.hpp"
#include "tempergrid/ising.hpp"
#include "tempergrid/schedule.hpp"
#ifndef TGREF_NO_SCHEDULE
#include "tempergrid/analysis.hpp"
#include "tempergrid/oracle.hpp"
#endif

#include "philox_ref.h"
#include "tg_oracle.h"

namespace tgref_ctx {
extern thread_local std::uint64_t master;
extern thread_local int n_replicas;
}  // namespace tgref_ctx

#ifdef TGREF_NO_CTX
namespace tgref_ctx {
thread_local std::uint64_t master = 0;
thread_local int n_replicas = 0;
}  // namespace tgref_ctx
#endif

namespace {

void put_err(char* err, int errlen, const std::string& msg) {
    if (!err || errlen <= 0) return;
    std::strncpy(err, msg.c_str(), static_cast<std::size_t>(errlen - 1));
    err[errlen - 1] = '\0';
}

std::uint64_t digest(const tempergrid::SpinState& s) {
    std::uint64_t d = 0;
    for (std::size_t i = 0; i < s.size(); ++i)
        if (s[i] > 0) d += tgo_digest_term(i);
    return d;
}

}  // namespace

extern "C" int tgr_run_2dpt(const tgo_problem* p, const tgo_run_cfg* cfg, tgo_outputs* out,
                            int threads, int store_grid, char* err, int errlen) {
    using namespace tempergrid;
    try {
        std::vector<Coupling> cs;
        for (int k = 0; k < p->n_couplings; ++k) cs.push_back({p->ci[k], p->cj[k], p->cw[k]});
        std::vector<double> h(p->fields, p->fields + p->n);
        IsingModel cost(p->n, std::move(cs), std::move(h));
        std::vector<std::pair<int, int>> pairs;
        for (int k = 0; k < p->n_pairs; ++k) pairs.emplace_back(p->pa[k], p->pb[k]);
        ConstrainedProblem problem{std::move(cost), ConstraintSet(p->n, std::move(pairs))};
        Schedule schedule;
        schedule.betas.assign(cfg->betas, cfg->betas + cfg->n_betas);
        schedule.penalties.assign(cfg->penalties, cfg->penalties + cfg->n_penalties);
        RunConfig rc;
        rc.total_sweeps = cfg->total_sweeps;
        rc.sweeps_per_swap = cfg->sweeps_per_swap;
        rc.seed = cfg->seed;
        rc.threads = threads;
        rc.store_target_only = !(store_grid || out->grid_states || out->final_grid);
        tgref_ctx::master = cfg->seed;
        tgref_ctx::n_replicas = cfg->n_betas * cfg->n_penalties;

        const Trace trace = run_2dpt(problem, schedule, rc);

        const int n = p->n;
        const int R = cfg->n_betas * cfg->n_penalties;
        for (std::size_t k = 0; k < trace.records.size(); ++k) {
            const TraceRecord& r = trace.records[k];
            if (out->f) out->f[k] = r.f;
            if (out->g) out->g[k] = r.g;
            if (out->feasible) out->feasible[k] = r.feasible ? 1 : 0;
            if (out->digest) out->digest[k] = digest(r.state);
            if (out->states) std::memcpy(out->states + k * n, r.state.data(), n);
            if (out->grid_states)
                for (int q = 0; q < R; ++q)
                    std::memcpy(out->grid_states + (k * R + q) * n, r.grid[q].data(), n);
        }
        if (!trace.records.empty()) {
            const TraceRecord& last = trace.records.back();
            if (out->final_grid)
                for (int q = 0; q < R; ++q)
                    std::memcpy(out->final_grid + static_cast<std::size_t>(q) * n,
                                last.grid[q].data(), n);
        }
        // Cumulative acceptance rates are what the reference reports
        // (engine.cpp:197-208); accepts = rate * attempts is exact for the
        // counts involved, so recover integer counters per round.
        const int I = cfg->n_betas, J = cfg->n_penalties;
        std::vector<std::int64_t> att_p(I * std::max(0, J - 1), 0), att_b(std::max(0, I - 1) * J, 0);
        {
            // attempts are a deterministic function of the round schedule
            int direction = 1;
            for (std::size_t k = 0; k < trace.records.size(); ++k) {
                const std::int64_t rn = static_cast<std::int64_t>(k) + 1;
                const int even = rn % 2 == 0;
                bool dp, db;
                if (I == 1 && J == 1) dp = db = false;
                else if (I == 1) { dp = true; db = false; }
                else if (J == 1) { dp = false; db = true; }
                else { dp = direction == 1; db = !dp; }
                if (dp) for (int i = 0; i < I; ++i) for (int q = even; q + 1 < J; q += 2) ++att_p[i * (J - 1) + q];
                if (db) for (int j = 0; j < J; ++j) for (int b = even; b + 1 < I; b += 2) ++att_b[b * J + j];
                const TraceRecord& r = trace.records[k];
                if (out->round_acc_p)
                    for (std::size_t q = 0; q < att_p.size(); ++q)
                        out->round_acc_p[k * att_p.size() + q] =
                            static_cast<std::int64_t>(r.acceptance_rates_p[q] * att_p[q] + 0.5);
                if (out->round_acc_b)
                    for (std::size_t q = 0; q < att_b.size(); ++q)
                        out->round_acc_b[k * att_b.size() + q] =
                            static_cast<std::int64_t>(r.acceptance_rates_beta[q] * att_b[q] + 0.5);
                if (even) direction = -direction;
            }
            if (!trace.records.empty()) {
                const TraceRecord& r = trace.records.back();
                for (std::size_t q = 0; q < att_p.size(); ++q) {
                    if (out->attempts_p) out->attempts_p[q] = att_p[q];
                    if (out->accepts_p) out->accepts_p[q] = static_cast<std::int64_t>(r.acceptance_rates_p[q] * att_p[q] + 0.5);
                }
                for (std::size_t q = 0; q < att_b.size(); ++q) {
                    if (out->attempts_b) out->attempts_b[q] = att_b[q];
                    if (out->accepts_b) out->accepts_b[q] = static_cast<std::int64_t>(r.acceptance_rates_beta[q] * att_b[q] + 0.5);
                }
            }
        }
        return 0;
    } catch (const tempergrid::config_error& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const tempergrid::resource_error& e) {
        put_err(err, errlen, e.what());
        return 3;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

// Timing entry for bench.py's reference arm: run_2dpt on the given inputs,
// discarding the trace (the reference still builds it in RAM, engine.cpp:189-214).
extern "C" int tgr_run_2dpt_timed(const tgo_problem* p, const tgo_run_cfg* cfg, int threads,
                                  double* f_last, char* err, int errlen) {
    using namespace tempergrid;
    try {
        std::vector<Coupling> cs;
        for (int k = 0; k < p->n_couplings; ++k) cs.push_back({p->ci[k], p->cj[k], p->cw[k]});
        std::vector<double> h(p->fields, p->fields + p->n);
        IsingModel cost(p->n, std::move(cs), std::move(h));
        std::vector<std::pair<int, int>> pairs;
        for (int k = 0; k < p->n_pairs; ++k) pairs.emplace_back(p->pa[k], p->pb[k]);
        ConstrainedProblem problem{std::move(cost), ConstraintSet(p->n, std::move(pairs))};
        Schedule schedule;
        schedule.betas.assign(cfg->betas, cfg->betas + cfg->n_betas);
        schedule.penalties.assign(cfg->penalties, cfg->penalties + cfg->n_penalties);
        RunConfig rc;
        rc.total_sweeps = cfg->total_sweeps;
        rc.sweeps_per_swap = cfg->sweeps_per_swap;
        rc.seed = cfg->seed;
        rc.threads = threads;
        tgref_ctx::master = cfg->seed;
        tgref_ctx::n_replicas = cfg->n_betas * cfg->n_penalties;
        const Trace trace = run_2dpt(problem, schedule, rc);
        if (f_last) *f_last = trace.records.empty() ? 0.0 : trace.records.back().f;
        return 0;
    } catch (const tempergrid::config_error& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

// tempergrid::run_jcolumn_pt (engine.cpp:221-270) on the same plain arrays;
// cfg's penalties are ignored (the column runs at p_fixed).
extern "C" int tgr_run_jcolumn(const tgo_problem* p, const tgo_run_cfg* cfg, double p_fixed,
                               int j_repeats, int threads, tgo_baseline_out* out, char* err,
                               int errlen) {
    using namespace tempergrid;
    try {
        std::vector<Coupling> cs;
        for (int k = 0; k < p->n_couplings; ++k) cs.push_back({p->ci[k], p->cj[k], p->cw[k]});
        std::vector<double> h(p->fields, p->fields + p->n);
        IsingModel cost(p->n, std::move(cs), std::move(h));
        std::vector<std::pair<int, int>> pairs;
        for (int k = 0; k < p->n_pairs; ++k) pairs.emplace_back(p->pa[k], p->pb[k]);
        ConstrainedProblem problem{std::move(cost), ConstraintSet(p->n, std::move(pairs))};
        std::vector<double> betas(cfg->betas, cfg->betas + cfg->n_betas);
        RunConfig rc;
        rc.total_sweeps = cfg->total_sweeps;
        rc.sweeps_per_swap = cfg->sweeps_per_swap;
        rc.seed = cfg->seed;
        rc.threads = threads;
        tgref_ctx::master = cfg->seed;
        tgref_ctx::n_replicas = cfg->n_betas;
        const BaselineTrace t = run_jcolumn_pt(problem, betas, p_fixed, j_repeats, rc);
        for (std::size_t k = 0; k < t.records.size(); ++k) {
            const BaselineRecord& r = t.records[k];
            if (out->round) out->round[k] = r.round;
            if (out->sweep_count) out->sweep_count[k] = r.sweep_count;
            if (out->best_f) out->best_f[k] = r.best_f;
            if (out->any_feasible) out->any_feasible[k] = r.any_feasible ? 1 : 0;
            if (out->n_feasible) out->n_feasible[k] = r.n_feasible;
            if (out->n_total) out->n_total[k] = r.n_total;
        }
        if (out->feasible_fraction) *out->feasible_fraction = t.feasible_fraction;
        return 0;
    } catch (const tempergrid::config_error& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const tempergrid::resource_error& e) {
        put_err(err, errlen, e.what());
        return 3;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

#ifndef TGREF_NO_SCHEDULE
namespace {
tempergrid::ConstrainedProblem make_problem(const tgo_problem* p) {
    using namespace tempergrid;
    std::vector<Coupling> cs;
    for (int k = 0; k < p->n_couplings; ++k) cs.push_back({p->ci[k], p->cj[k], p->cw[k]});
    std::vector<double> h(p->fields, p->fields + p->n);
    IsingModel cost(p->n, std::move(cs), std::move(h));
    std::vector<std::pair<int, int>> pairs;
    for (int k = 0; k < p->n_pairs; ++k) pairs.emplace_back(p->pa[k], p->pb[k]);
    return ConstrainedProblem{std::move(cost), ConstraintSet(p->n, std::move(pairs))};
}

void put_stats(const tempergrid::ProbeStats& s, tgo_probe_stats* o) {
    o->row = s.row;
    o->column = s.column;
    o->beta = s.beta;
    o->penalty = s.penalty;
    o->sigma_e = s.sigma_e;
    o->sigma_g = s.sigma_g;
    o->mean_g = s.mean_g;
}
}  // namespace

// tempergrid::probe_population (schedule.cpp:18-52).
extern "C" int tgr_probe_population(const tgo_problem* p, double beta, double penalty,
                                    int n_chains, int sweeps, std::uint64_t seed,
                                    tgo_probe_stats* out, char* err, int errlen) {
    try {
        put_stats(tempergrid::probe_population(make_problem(p), beta, penalty, n_chains, sweeps,
                                               seed),
                  out);
        return 0;
    } catch (const tempergrid::config_error& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

// tempergrid::build_schedule (schedule.cpp:77-163).
extern "C" int tgr_build_schedule(const tgo_problem* p, const tgo_schedule_cfg* c, double* betas,
                                  int* n_betas, double* penalties, int* n_penalties,
                                  tgo_probe_stats* stats, int stats_cap, int* n_stats,
                                  int* budget_exhausted, char* err, int errlen) {
    try {
        tempergrid::ScheduleConfig cfg;
        cfg.beta0 = c->beta0;
        cfg.p0 = c->p0;
        cfg.i_max = c->i_max;
        cfg.j_max = c->j_max;
        cfg.sigma_min = c->sigma_min;
        cfg.alpha_beta = c->alpha_beta;
        cfg.alpha_p = c->alpha_p;
        cfg.n_chains = c->n_chains;
        cfg.sweeps_per_probe = c->sweeps_per_probe;
        cfg.replica_budget = c->replica_budget;
        cfg.seed = c->seed;
        const tempergrid::Schedule s = tempergrid::build_schedule(make_problem(p), cfg);
        *n_betas = static_cast<int>(s.betas.size());
        *n_penalties = static_cast<int>(s.penalties.size());
        std::copy(s.betas.begin(), s.betas.end(), betas);
        std::copy(s.penalties.begin(), s.penalties.end(), penalties);
        *n_stats = static_cast<int>(s.probe_stats.size());
        for (int k = 0; k < *n_stats && k < stats_cap; ++k) put_stats(s.probe_stats[k], stats + k);
        *budget_exhausted = s.budget_exhausted ? 1 : 0;
        return 0;
    } catch (const tempergrid::config_error& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}
// run_2dpt + tempergrid::kl_curve (analysis.cpp:215-241) with the reference's
// own decode (constraints.cpp:149-162) and enumerate_boltzmann (oracle.cpp).
extern "C" int tgr_kl_curve(const tgo_problem* p, const tgo_run_cfg* cfg, const tgo_decoder* dec,
                            double beta, int discard, int threads, std::int64_t* t,
                            std::int64_t* samples, double* kl, char* err, int errlen) {
    using namespace tempergrid;
    try {
        const ConstrainedProblem problem = make_problem(p);
        Schedule schedule;
        schedule.betas.assign(cfg->betas, cfg->betas + cfg->n_betas);
        schedule.penalties.assign(cfg->penalties, cfg->penalties + cfg->n_penalties);
        RunConfig rc;
        rc.total_sweeps = cfg->total_sweeps;
        rc.sweeps_per_swap = cfg->sweeps_per_swap;
        rc.seed = cfg->seed;
        rc.threads = threads;
        const Trace trace = run_2dpt(problem, schedule, rc);
        const ConstrainedProblem lp = make_problem(dec->logical);
        SparsificationMap map;
        map.n_logical = dec->logical->n;
        map.n_physical = p->n;
        for (int u = 0; u < map.n_logical; ++u)
            map.copies.emplace_back(dec->copies + dec->copy_off[u], dec->copies + dec->copy_off[u + 1]);
        const auto pts = kl_curve(trace, map, lp.cost, beta, discard != 0);
        for (std::size_t k = 0; k < pts.size(); ++k) {
            t[k] = pts[k].t;
            samples[k] = pts[k].samples;
            kl[k] = pts[k].kl;
        }
        return 0;
    } catch (const tempergrid::config_error& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const tempergrid::resource_error& e) {
        put_err(err, errlen, e.what());
        return 3;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}
#endif

// tempergrid::sparsify (constraints.cpp:50-120) on a logical model; writes the
// physical couplings (canonical order) and chain pairs.  Returns the number
// of physical spins, or -code on error.  Capacities are the caller's.
extern "C" int tgr_sparsify(int n, int n_couplings, const int* ci, const int* cj, const double* cw,
                            const double* fields, int copies, int max_degree, int* out_ci,
                            int* out_cj, double* out_w, int* out_nc, double* out_h, int* out_pa,
                            int* out_pb, int* out_np, char* err, int errlen) {
    using namespace tempergrid;
    try {
        std::vector<Coupling> cs;
        for (int k = 0; k < n_couplings; ++k) cs.push_back({ci[k], cj[k], cw[k]});
        IsingModel logical(n, std::move(cs), std::vector<double>(fields, fields + n));
        const SparsifyResult r = sparsify(logical, copies, max_degree);
        const auto& pc = r.problem.cost.couplings();
        for (std::size_t k = 0; k < pc.size(); ++k) {
            out_ci[k] = pc[k].i;
            out_cj[k] = pc[k].j;
            out_w[k] = pc[k].weight;
        }
        *out_nc = static_cast<int>(pc.size());
        for (int i = 0; i < r.problem.cost.n_spins(); ++i) out_h[i] = r.problem.cost.fields()[i];
        const auto& pp = r.problem.constraints.pairs();
        for (std::size_t k = 0; k < pp.size(); ++k) {
            out_pa[k] = pp[k].first;
            out_pb[k] = pp[k].second;
        }
        *out_np = static_cast<int>(pp.size());
        return r.problem.cost.n_spins();
    } catch (const tempergrid::config_error& e) {
        put_err(err, errlen, e.what());
        return -2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return -1;
    }
}

#ifndef TGREF_NO_SCHEDULE
// ---- trace reports (analysis.cpp), pinned for paper_2506_14781_b200/reports.py

// time_to_residual (analysis.cpp:260-270) over a flat (t, f, feasible) series;
// *out = -1 when the threshold is never reached.
extern "C" int tgr_time_to_residual(int n, const std::int64_t* t, const double* f, const int* feasible,
                                    double e_gs, int n_logical, double rho_max, std::int64_t* out) {
    try {
        std::vector<tempergrid::EnergySample> s(n);
        for (int i = 0; i < n; ++i) s[i] = tempergrid::EnergySample{t[i], f[i], feasible[i] != 0};
        const auto r = tempergrid::time_to_residual(s, e_gs, n_logical, rho_max);
        *out = r ? *r : -1;
        return 0;
    } catch (const tempergrid::config_error&) {
        return 2;
    } catch (...) {
        return 4;
    }
}

// residual_curve (analysis.cpp:38-96): runs x rounds target records (f,
// feasible, state), the sparsification map (copy chains) and the logical
// model; outputs t, rho_E and ci95 per round.
extern "C" int tgr_residual_curve(int n_runs, int n_rounds, int n_phys, const std::int64_t* t,
                                  const double* f, const int* feasible, const std::int8_t* states,
                                  const double* e_gs, const int* instance_id, int n_logical,
                                  const int* chain_off, const int* chain, int n_lc, const int* lci,
                                  const int* lcj, const double* lw, const double* lh, int strict,
                                  int resamples, std::uint64_t seed, std::int64_t* out_t,
                                  double* out_rho, double* out_ci) {
    try {
        std::vector<tempergrid::Trace> traces(n_runs);
        for (int r = 0; r < n_runs; ++r) {
            traces[r].records.resize(n_rounds);
            for (int k = 0; k < n_rounds; ++k) {
                auto& rec = traces[r].records[k];
                const size_t q = (size_t)r * n_rounds + k;
                rec.sweep_count = t[k];
                rec.f = f[q];
                rec.feasible = feasible[q] != 0;
                rec.state.assign(states + q * n_phys, states + (q + 1) * n_phys);
            }
        }
        std::vector<tempergrid::ResidualInput> runs(n_runs);
        for (int r = 0; r < n_runs; ++r) runs[r] = {&traces[r], e_gs[r], instance_id[r]};
        tempergrid::SparsificationMap map;
        map.n_logical = n_logical;
        map.n_physical = n_phys;
        map.copies.resize(n_logical);
        for (int u = 0; u < n_logical; ++u) map.copies[u].assign(chain + chain_off[u], chain + chain_off[u + 1]);
        std::vector<tempergrid::Coupling> cpl(n_lc);
        for (int e = 0; e < n_lc; ++e) cpl[e] = {lci[e], lcj[e], lw[e]};
        tempergrid::IsingModel logical(n_logical, cpl, std::vector<double>(lh, lh + n_logical));
        const auto curve = tempergrid::residual_curve(runs, map, logical, n_logical, strict != 0,
                                                      resamples, seed);
        for (int k = 0; k < n_rounds; ++k) {
            out_t[k] = curve.points[k].t;
            out_rho[k] = curve.points[k].rho_e;
            out_ci[k] = curve.points[k].ci95;
        }
        return 0;
    } catch (const tempergrid::config_error&) {
        return 2;
    } catch (...) {
        return 4;
    }
}
#endif
