/*
 * tempergrid_b200.h -- C ABI of the B200-native 2D parallel-tempering engine.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `tempergrid` (arXiv 2506.14781): the RNG, sweep, swap and observable
 * machinery under
 *     Trace tempergrid::run_2dpt(const ConstrainedProblem&, const Schedule&,
 *                                const RunConfig&)
 *   (/root/reference/proj/include/tempergrid/engine.hpp:62-63,
 *    /root/reference/proj/src/engine.cpp:83-219).
 * The reference has no FFI of its own; these entry points are what a
 * reference-side binding needs to replace run_2dpt (INTEGRATION.md shows the
 * C++ shim and a ctypes stub).  Plain pointers and sizes only; no exceptions
 * cross the boundary.  Status codes mirror the reference CLI's exit codes
 * (cli.cpp:659-668): config_error -> 2, resource_error -> 3.
 *
 * Ownership: the caller owns every host buffer (copied in or written out);
 * the context owns all device memory.  One context is driven by one host
 * thread.  Multi-GPU: one context per GPU/process, joined by
 * tg_create_distributed with an NCCL unique id.
 */
#ifndef TEMPERGRID_B200_H
#define TEMPERGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 1

typedef struct tg_ctx tg_ctx;

enum tg_status {
    TG_OK = 0,
    TG_ERR_INTERNAL = 1,
    TG_ERR_CONFIG = 2,   /* reference config_error   (errors.hpp:10-12)  */
    TG_ERR_RESOURCE = 3, /* reference resource_error (errors.hpp:16-18)  */
    TG_ERR_CUDA = 4,     /* no device / CUDA or NCCL failure              */
    TG_ERR_SINK = 5      /* the record sink asked to stop                 */
};

/* Update rule. METROPOLIS restates metropolis_sweep (mc.cpp:21-35);
 * HEAT_BATH is the north-star p-bit rule s_i = +1 iff u < sigma(2 beta h_i). */
enum tg_rule { TG_RULE_METROPOLIS = 0, TG_RULE_HEAT_BATH = 1 };

/* Engine.  SLOT: int8 spins, one CTA per replica, FP64 fields, draws from the
 * reference's per-slot streams (bit-exact vs the reference fed Philox draws).
 * PLANE: multi-spin-coded bit planes (32 replicas per word), threshold tables,
 * lazily consumed bit-plane draws keyed by physical replica; requires J = +-1,
 * h = 0 (the integer-coupling instances).  AUTO picks PLANE when eligible. */
enum tg_engine { TG_ENGINE_AUTO = 0, TG_ENGINE_SLOT = 1, TG_ENGINE_PLANE = 2, TG_ENGINE_FLOAT = 3 };

/* What each round record carries beyond (f, g, feasible). */
enum tg_record_flags {
    TG_REC_DIGEST = 1,   /* 64-bit digest of the target state (every round) */
    TG_REC_STATE = 2,    /* target state, int8 in caller spin order          */
    TG_REC_GRID = 4,     /* every slot's state (store_target_only = false)   */
    TG_REC_COUNTERS = 8  /* cumulative per-pair accept counters              */
};

typedef struct {
    int64_t total_sweeps;    /* RunConfig::total_sweeps   (engine.hpp:27) */
    int64_t sweeps_per_swap; /* RunConfig::sweeps_per_swap (engine.hpp:28) */
    uint64_t seed;           /* RunConfig::seed            (engine.hpp:29) */
    int32_t rule;            /* tg_rule */
    int32_t engine;          /* tg_engine */
    int32_t record_flags;    /* tg_record_flags bitmask */
    int32_t record_every;    /* deliver a record every k rounds (1 = every round, as the reference) */
} tg_run_config;

typedef struct {
    int64_t round;        /* 1-based (TraceRecord::round) */
    int64_t sweep_count;  /* round * sweeps_per_swap */
    double f;             /* target replica cost energy */
    double g;             /* target replica constraint value, reference units sum (s_a-s_b)^2 */
    int32_t feasible;     /* g == 0 */
    int32_t target_state; /* physical replica id currently at slot I*J-1 */
    uint64_t digest;      /* sum over +1 spins of mix64(i+1) (caller order), if TG_REC_DIGEST */
} tg_record;

/* Record sink, called on the thread that called tg_run/tg_advance, in round
 * order.  states: n_recs x n int8 (TG_REC_STATE) or n_recs x R x n (TG_REC_GRID),
 * else NULL.  acc_p: n_recs x I*(J-1), acc_b: n_recs x (I-1)*J cumulative accept
 * counts (TG_REC_COUNTERS), else NULL.  Return nonzero to stop (TG_ERR_SINK). */
typedef int (*tg_sink_fn)(void* user, const tg_record* recs, int64_t n_recs,
                          const int8_t* states, const int64_t* acc_p, const int64_t* acc_b);

int tg_abi_version(void);

/* Context on CUDA device `device` (single-GPU: rank 0 of 1). */
int tg_create(int device, tg_ctx** out);
/* Context for rank `rank` of `world_size`, one per GPU/process.  nccl_id is
 * the 128-byte ncclUniqueId created by rank 0 and broadcast by the caller. */
int tg_create_distributed(int device, int rank, int world_size, const void* nccl_id, tg_ctx** out);
/* Create a fresh NCCL unique id (128 bytes) on rank 0. */
int tg_nccl_unique_id(void* out128);
void tg_destroy(tg_ctx* ctx);
/* Last error message of ctx (or of the failed create when ctx == NULL). */
size_t tg_last_error(const tg_ctx* ctx, char* buf, size_t len);

/* ConstrainedProblem (constraints.hpp:44-48): n spins, cost couplings
 * (ci[k], cj[k], w[k]) with any order and i != j, fields[n], and chain
 * constraint pairs (pa[k], pb[k]).  Validated like IsingModel /
 * ConstraintSet (ising.cpp:21-46, constraints.cpp:16-26). */
int tg_set_problem(tg_ctx* ctx, int n, int n_couplings, const int32_t* ci, const int32_t* cj,
                   const double* w, const double* fields, int n_pairs, const int32_t* pa,
                   const int32_t* pb);
/* Schedule (schedule.hpp:35-42): strictly increasing finite betas[I] and
 * penalties[J] >= 0 (engine.cpp:41-52, constraints.cpp:123-124). */
int tg_set_schedule(tg_ctx* ctx, int n_betas, const double* betas, int n_penalties,
                    const double* penalties);

/* run_2dpt: tg_init + tg_advance(total_sweeps / sweeps_per_swap rounds). */
int tg_run(tg_ctx* ctx, const tg_run_config* cfg, tg_sink_fn sink, void* user);
/* Initialise replicas (engine.cpp:98-107) and the round counter. */
int tg_init(tg_ctx* ctx, const tg_run_config* cfg);
/* Continue for n_rounds rounds from the current state (resume-capable). */
int tg_advance(tg_ctx* ctx, int64_t n_rounds, tg_sink_fn sink, void* user);

/* Current configuration at grid slot `slot` (row-major i*J+j), caller order. */
int tg_get_state(tg_ctx* ctx, int slot, int8_t* out);
/* Cumulative attempt/accept counters (engine.cpp:109-112 layouts). */
int tg_get_counters(tg_ctx* ctx, int64_t* attempts_p, int64_t* accepts_p, int64_t* attempts_b,
                    int64_t* accepts_b);
/* Per-slot f and g after the last completed round. */
int tg_get_energies(tg_ctx* ctx, double* f, double* g);

/* ---- Checkpoint / resume (single-GPU contexts, not batches) ----
 * The reference keeps a run only in RAM (engine.hpp:39-56, engine.cpp:119,214)
 * and has no resume; a checkpoint here is everything a run's continuation
 * depends on: every physical state's spins (caller order), the slot labels,
 * the cumulative accept counters, the round counter and the swap-stream
 * position.  The Philox draws are pure functions of (seed, counters), so no
 * RNG state is saved.  tg_restore needs a context initialised (tg_init) with
 * the same problem, schedule and config; the resumed run then continues bit
 * for bit as if it had never stopped.  Layout: tg_checkpoint_header, int8
 * states [R][n], int32 slot_state [R], int64 accepts_p [I(J-1)], int64
 * accepts_b [(I-1)J]. */
typedef struct {
    uint32_t magic;        /* 'TGCP' */
    uint32_t version;      /* 1 */
    int32_t engine, rule, n, I, J, pad;
    int64_t rounds_done;
    uint64_t swap_base;    /* swap-stream draws consumed */
    uint64_t seed;
} tg_checkpoint_header;
int tg_checkpoint_size(tg_ctx* ctx, size_t* bytes);
int tg_checkpoint(tg_ctx* ctx, void* buf, size_t bytes);
int tg_restore(tg_ctx* ctx, const void* buf, size_t bytes);

typedef struct {
    int32_t engine;        /* engine actually selected */
    int32_t n_colors;      /* colour classes of the canonical order */
    int32_t n_replicas;    /* I*J (whole grid) */
    int32_t local_replicas;/* replicas swept by this rank */
    int32_t words;         /* plane engine: 32-replica words per site on this rank */
    int32_t device_sms;
    int64_t rounds_done;
    double last_sweep_ms;  /* device time of the sweep kernels of the last tg_advance */
    double last_swap_ms;   /* device time of the swap/record kernels of the last tg_advance */
    int64_t sweep_launches;
    int64_t other_launches;
    char sweep_kernel[48]; /* name of the sweep kernel the last tg_advance launched ("" before) */
} tg_info;
int tg_get_info(tg_ctx* ctx, tg_info* info);
/* cudaStream_t the context launches on (for external CUDA-event timing). */
void* tg_stream(tg_ctx* ctx);
/* Enable per-kernel CUDA-event timing inside tg_advance (default off). */
int tg_set_profiling(tg_ctx* ctx, int on);

/* ---------------------------------------------------------------- batches
 * Independent instances in one launch (config 3: 64 Wishart instances, each
 * with its own 16x16 grid).  Every instance has its own problem, schedule
 * (same I x J shape across the batch) and seed; results equal independent
 * tg_run / run_2dpt calls instance by instance.  SLOT engine
 * semantics (per-slot reference streams).  The sink receives records per
 * instance, in round order within each instance. */
typedef int (*tg_batch_sink_fn)(void* user, int32_t instance, const tg_record* recs,
                                int64_t n_recs, const int8_t* states, const int64_t* acc_p,
                                const int64_t* acc_b);
int tg_batch_clear(tg_ctx* ctx);
int tg_batch_add(tg_ctx* ctx, int n, int n_couplings, const int32_t* ci, const int32_t* cj,
                 const double* w, const double* fields, int n_pairs, const int32_t* pa,
                 const int32_t* pb, int n_betas, const double* betas, int n_penalties,
                 const double* penalties, uint64_t seed, int32_t* index);
/* cfg->seed is ignored (per-instance seeds); engine must be AUTO or SLOT. */
int tg_batch_run(tg_ctx* ctx, const tg_run_config* cfg, tg_batch_sink_fn sink, void* user);
/* tg_batch_run split in two (resume / timing): build + initial states, then
 * n_rounds more rounds of every instance per call. */
int tg_batch_init(tg_ctx* ctx, const tg_run_config* cfg);
int tg_batch_advance(tg_ctx* ctx, int64_t n_rounds, tg_batch_sink_fn sink, void* user);
int tg_batch_get_state(tg_ctx* ctx, int instance, int slot, int8_t* out);
int tg_batch_get_counters(tg_ctx* ctx, int instance, int64_t* attempts_p, int64_t* accepts_p,
                          int64_t* attempts_b, int64_t* accepts_b);

/* ---- Resource-matched J-column baseline (run_jcolumn_pt, engine.cpp:221-270) ----
 * j_repeats independent single-column runs of the context's problem
 * (tg_set_problem) with schedule (betas, {p_fixed}) and seeds
 * derive_seed(cfg->seed, repeat = 5, rep) (rng.hpp:28, engine.cpp:238),
 * executed as ONE batch on the device (SLOT engine) and merged per round:
 * out[k] for rounds k+1 = 1..total_sweeps/sweeps_per_swap (out_cap must hold
 * them).  best_f is NaN where no repeat was feasible.  cfg->engine must be
 * AUTO or SLOT; record_flags / record_every are ignored.  Errors as the
 * reference: p_fixed <= 0 or j_repeats < 1 -> TG_ERR_CONFIG. */
typedef struct {
    int64_t round;
    int64_t sweep_count;
    double best_f;
    int32_t any_feasible;
    int32_t n_feasible;
    int32_t n_total;
    int32_t reserved;
} tg_baseline_record;

int tg_run_jcolumn(tg_ctx* ctx, int n_betas, const double* betas, double p_fixed, int j_repeats,
                   const tg_run_config* cfg, tg_baseline_record* out, int64_t out_cap,
                   double* feasible_fraction);

/* ---- Decoded-sample KL curve on the device (kl_curve, analysis.cpp:215-241) ----
 * Attach a decoder to the context's following SLOT-engine runs on one GPU
 * (tg_run, tg_init + tg_advance, tg_batch_run -- one curve per instance; AUTO
 * picks SLOT while a decoder is set): after every round the target replica of
 * each instance is decoded on the device
 * through the copy map (decode, constraints.cpp:149-162: majority vote over the
 * logical spin's copies, ties to the first copy; infeasible when chain-adjacent
 * copies differ), added to a device histogram (skipped when infeasible and
 * discard_infeasible), and the KL divergence of the accumulated histogram
 * against the exact Boltzmann distribution of the logical model at beta
 * (enumerate_boltzmann, oracle.cpp:154-165, computed once on the host) is
 * evaluated (kl_divergence, oracle.cpp:178-195).  copy_offsets[n_logical+1],
 * copies[]: physical spins (caller order) of logical spin u in chain order.
 * Read the curve with tg_get_kl_curve (rounds are 1-based; kl is NaN while the
 * histogram is empty).  n_logical <= 20. */
int tg_set_kl_decoder(tg_ctx* ctx, int n_logical, int n_couplings, const int32_t* li,
                      const int32_t* lj, const double* lw, const double* lh, double beta,
                      const int32_t* copy_offsets, const int32_t* copies, int discard_infeasible);
int tg_clear_kl_decoder(tg_ctx* ctx);
int tg_get_kl_curve(tg_ctx* ctx, int instance, int64_t first_round, int64_t n, double* kl,
                    int64_t* samples);

/* ---- Schedule probes and the adaptive ladder (schedule.cpp:18-163) ----
 * tg_probe_population = probe_population (schedule.hpp:44-48) over the
 * context's problem: n_chains independent chains at (beta, penalty), chain c
 * on the Philox stream derive_seed(seed, probe = 4, c) (initial state from
 * draw 0, then one draw per spin per sweep), all chains in one device launch;
 * the second half of the sweeps is pooled on the device.  rule selects the
 * sweep (the reference probes with metropolis_sweep).
 * tg_build_schedule = build_schedule (schedule.hpp:57-58) with every probe on
 * the device; the ladder logic runs on the host between probes. */
typedef struct {
    int32_t row, column;
    double beta, penalty, sigma_e, sigma_g, mean_g;
} tg_probe_stats;

typedef struct {               /* ScheduleConfig, schedule.hpp:10-22 (+ rule) */
    double beta0;              /* 0.3 */
    double p0;                 /* 0.5 */
    int32_t i_max, j_max;      /* 20, 20 */
    double sigma_min;          /* <= 0: 0.5 sqrt(n) */
    double alpha_beta;         /* 1.0 */
    double alpha_p;            /* 1.2 */
    int32_t n_chains;          /* 32 */
    int32_t sweeps_per_probe;  /* 1000 */
    int32_t replica_budget;    /* 400 */
    int32_t rule;              /* TG_RULE_METROPOLIS */
    uint64_t seed;             /* 1 */
} tg_schedule_config;

int tg_probe_population(tg_ctx* ctx, double beta, double penalty, int n_chains, int sweeps,
                        uint64_t seed, int rule, tg_probe_stats* out);
int tg_build_schedule(tg_ctx* ctx, const tg_schedule_config* cfg, double* betas, int betas_cap,
                      int* n_betas, double* penalties, int penalties_cap, int* n_penalties,
                      tg_probe_stats* stats, int stats_cap, int* n_stats, int* budget_exhausted);

/* Host-only helper (no device needed): greedy colouring of cost+chain edges
 * and the canonical sweep order (stable sort by colour, chain degree, cost
 * degree); order[k] = caller spin at internal position k. */
int tg_canonical_order(int n, int n_couplings, const int32_t* ci, const int32_t* cj, int n_pairs,
                       const int32_t* pa, const int32_t* pb, int32_t* order, int32_t* color,
                       int32_t* n_colors);

/* Swap-probability helpers of the reference (engine.hpp:15-24). */
double tg_p_swap_probability(double beta, double d_penalty, double dg);
double tg_beta_swap_probability(double d_beta, double d_energy);
double tg_general_swap_probability(double beta_a, double beta_b, double de_a, double de_b);

/* Replica partition of a multi-GPU run (host-only): rank `rank` of `world`
 * sweeps physical replicas [*state0, *state0 + *count) of the I*J grid
 * (engine TG_ENGINE_PLANE needs count % 32 == 0 when world > 1). */
int tg_partition(int n_replicas, int rank, int world, int engine, int32_t* state0, int32_t* count);

/* Host replay of one swap phase over gathered per-replica (f, g) -- the
 * exact routine the device swap kernel runs, exported so the multi-rank
 * exchange logic can be tested without a GPU.  slot_state[R] (state id at
 * each slot) and the counters are updated in place. */
int tg_swap_phase_host(int n_betas, const double* betas, int n_penalties, const double* penalties,
                       int64_t round, int direction, uint64_t seed, uint64_t swap_base,
                       const double* f_state, const double* g_state, int32_t* slot_state,
                       int64_t* accepts_p, int64_t* accepts_b);

#ifdef __cplusplus
}
#endif

#endif /* TEMPERGRID_B200_H */
