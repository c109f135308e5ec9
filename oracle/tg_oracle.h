/*
 * oracle/tg_oracle.h -- TEST INFRASTRUCTURE ONLY.  C restatement ("port") of
 * the reference 2D-PT hot path, used by tests/ and by bench.py's cpu_baseline
 * leg as the parity checker.  Nothing in paper_2506_14781_b200/ links it.
 *
 * Restates (file:line under /root/reference/proj):
 *   IsingModel ctor / CSR / energy / local_fields / apply_flip   src/ising.cpp:21-96
 *   ConstraintSet ctor / evaluate / delta_flip                   src/constraints.cpp:16-48,
 *                                                                include/tempergrid/constraints.hpp:32-37
 *   build_effective / energy_breakdown                           src/constraints.cpp:122-147
 *   make_sweep_state / refresh_sweep_state / metropolis_sweep    src/mc.cpp:7-35
 *   swap probabilities, validation, run_2dpt round loop          src/engine.cpp:18-219
 *   encode_state                                                 src/oracle.cpp:17-22
 */
#ifndef TG_ORACLE_H
#define TG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TGO_OK = 0, TGO_CONFIG_ERROR = 2, TGO_RESOURCE_ERROR = 3 };
enum { TGO_RULE_METROPOLIS = 0, TGO_RULE_HEAT_BATH = 1 };
/* RNG association: SLOT = reference (stream stays with the grid slot,
 * engine.cpp:36-39,160,182); PLANE = bit-plane draws keyed by physical state. */
enum { TGO_RNG_SLOT = 0, TGO_RNG_PLANE = 1, TGO_RNG_PACK = 2 };

typedef struct {
    int n;
    int n_couplings;
    const int* ci;
    const int* cj;
    const double* cw;
    const double* fields; /* length n */
    int n_pairs;
    const int* pa;
    const int* pb;
} tgo_problem;

typedef struct {
    int n_betas;
    const double* betas;
    int n_penalties;
    const double* penalties;
    int64_t total_sweeps;
    int64_t sweeps_per_swap;
    uint64_t seed;
    int rule;
    int rng_mode;
} tgo_run_cfg;

/* Caller-allocated outputs; any pointer may be NULL. */
typedef struct {
    double* f;              /* [rounds] target f */
    double* g;              /* [rounds] target g */
    uint8_t* feasible;      /* [rounds] */
    uint64_t* digest;       /* [rounds] target-state digest */
    int8_t* states;         /* [rounds * n] target states */
    int8_t* grid_states;    /* [rounds * R * n] every slot's state (store_target_only=false) */
    int64_t* round_acc_p;   /* [rounds * I*(J-1)] cumulative P accepts */
    int64_t* round_acc_b;   /* [rounds * (I-1)*J] cumulative beta accepts */
    int64_t* attempts_p;    /* [I*(J-1)] final */
    int64_t* accepts_p;
    int64_t* attempts_b;    /* [(I-1)*J] final */
    int64_t* accepts_b;
    int8_t* final_grid;     /* [R * n] final state at each slot */
    double* final_f;        /* [R] per slot */
    double* final_g;        /* [R] per slot */
    int32_t* final_state_id;/* [R] physical state id (initial slot) now at each slot */
} tgo_outputs;

int tgo_run_2dpt(const tgo_problem* prob, const tgo_run_cfg* cfg, tgo_outputs* out,
                 char* err, int errlen);

/* Resource-matched J-column baseline, run_jcolumn_pt (engine.cpp:221-270):
 * j_repeats single-column runs (betas, {p_fixed}) with seeds
 * derive_seed(cfg->seed, repeat=5, rep), merged round by round.  cfg's
 * n_penalties/penalties are ignored.  Outputs are [rounds]; best_f is NaN
 * where no repeat was feasible. */
typedef struct {
    int64_t* round;
    int64_t* sweep_count;
    double* best_f;
    uint8_t* any_feasible;
    int32_t* n_feasible;
    int32_t* n_total;
    double* feasible_fraction; /* scalar */
} tgo_baseline_out;

int tgo_run_jcolumn(const tgo_problem* prob, const tgo_run_cfg* cfg, double p_fixed,
                    int j_repeats, tgo_baseline_out* out, char* err, int errlen);

/* Schedule probes and the adaptive ladder (schedule.cpp:18-163,
 * schedule.hpp:10-60).  rule selects the sweep the probes run (the reference
 * calls metropolis_sweep; the heat-bath build links the alt sweep). */
typedef struct {
    int row, column;
    double beta, penalty, sigma_e, sigma_g, mean_g;
} tgo_probe_stats;

typedef struct {
    double beta0, p0;
    int i_max, j_max;
    double sigma_min, alpha_beta, alpha_p;
    int n_chains, sweeps_per_probe, replica_budget;
    uint64_t seed;
} tgo_schedule_cfg;

int tgo_probe_population(const tgo_problem* prob, double beta, double penalty, int n_chains,
                         int sweeps, uint64_t seed, int rule, tgo_probe_stats* out, char* err,
                         int errlen);
/* betas[cap i_max], penalties[cap j_max], stats[cap stats_cap]; counts out. */
int tgo_build_schedule(const tgo_problem* prob, const tgo_schedule_cfg* cfg, int rule,
                       double* betas, int* n_betas, double* penalties, int* n_penalties,
                       tgo_probe_stats* stats, int stats_cap, int* n_stats, int* budget_exhausted,
                       char* err, int errlen);

/* Decoded-sample KL (analysis.cpp:215-241, decode constraints.cpp:149-162,
 * enumerate_boltzmann oracle.cpp:105-165, kl_divergence oracle.cpp:178-195).
 * logical: the logical model; copy_off[n_logical+1] / copies: physical spins
 * of each logical spin in chain order. */
typedef struct {
    const tgo_problem* logical; /* only n, couplings, fields are used */
    const int* copy_off;
    const int* copies;
} tgo_decoder;

/* probs[2^n] (guard: n <= 24, resource error beyond); log_partition optional */
int tgo_enumerate_boltzmann(const tgo_problem* logical, double beta, double* probs,
                            double* log_partition, char* err, int errlen);
/* run_2dpt (cfg) + kl_curve: t/samples/kl per round (kl NaN while empty). */
int tgo_kl_curve(const tgo_problem* prob, const tgo_run_cfg* cfg, const tgo_decoder* dec,
                 double beta, int discard_infeasible, int64_t* t, int64_t* samples, double* kl,
                 char* err, int errlen);

/* engine.cpp:18-32 */
double tgo_p_swap_probability(double beta, double d_penalty, double dg);
double tgo_beta_swap_probability(double d_beta, double d_energy);
double tgo_general_swap_probability(double beta_a, double beta_b, double de_a, double de_b);

/* Cost energy f, constraint g, and effective total of one state (ising.cpp:70-77,
 * constraints.cpp:41-48,142-147). */
int tgo_energy_breakdown(const tgo_problem* prob, double penalty, const int8_t* s,
                         double* f, double* g);
uint64_t tgo_digest(const int8_t* s, int n);
uint64_t tgo_encode_state(const int8_t* s, int n);

/* Greedy index-order colouring of the cost+chain graph and the canonical
 * site order (stable sort by colour, chain degree, cost degree). */
int tgo_canonical_order(const tgo_problem* prob, int32_t* color, int32_t* order,
                        int32_t* n_colors);

/* Philox helpers for KAT tests. */
void tgo_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t tgo_derive(uint64_t master, uint64_t purpose, uint64_t index);
uint64_t tgo_bits(uint64_t seed, uint64_t n);
uint64_t tgo_plane(uint64_t pkey, uint32_t grp, uint64_t t, uint32_t site, int lane);
/* lazy MSB-first decision u < T on the bit-plane uniform (tests only) */
int tgo_plane_less(uint64_t pkey, uint32_t grp, uint64_t t, uint32_t site, int lane, double T);
/* packed-draw 53-bit uniform (engine "float"; philox_ref.h tgo_pack_u53) */
uint64_t tgo_pack(uint64_t pkey, uint32_t m, uint64_t t, uint32_t site);

#ifdef __cplusplus
}
#endif

#endif
