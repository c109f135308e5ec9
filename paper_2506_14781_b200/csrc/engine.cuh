// engine.cuh -- device data layout shared by the sweep, swap and record
// kernels (kernels.cu) and the host driver (capi.cu).
//
// Two sweep engines implement the reference sweep (mc.cpp:21-35) over the
// canonical colour order, in which the reference's sequential index-order
// pass is a chromatic pass:
//   * SLOT  -- int8 spins, one CTA per replica with its configuration in
//              shared memory, FP64 fields, 64-bit draws from the replica's
//              grid-slot stream (the reference's RNG association).
//   * PLANE -- multi-spin coding: bit l of word w at site i is the spin of
//              physical replica 32w+l; 32 replicas per 32-bit lane op, threshold
//              planes instead of exp(), lazily consumed bit-plane draws.
// Swaps permute grid labels (slot_state / state_slot); spin states never move.
#pragma once

#include <stdint.h>

#include "philox.cuh"

namespace tg {

constexpr int kKPlanes = 53;              // planes of a 53-bit threshold
constexpr int kKWords = kKPlanes + 1;     // + the "always" word
constexpr int kMaxDC = 7;                 // plane engine: cost degree bound
constexpr int kMaxDQ = 3;                 // plane engine: chain degree bound
constexpr int kVPlanes = 8;               // vertical counter planes
constexpr int kMaxTypes = 16;
constexpr int kMaxWordsArg = 32;       // plane engine: <= 1024 replicas per rank

// Round counters of the unfused round loop, kept on the device so that a
// captured CUDA graph of rounds can be replayed unchanged: the sweep, swap
// and extract kernels read them, round_tick_kernel advances them.
struct RoundState {
    int64_t round;       // rounds completed
    uint64_t swap_base;  // swap-stream draws consumed
    int32_t filled;      // records in the current chunk
    int32_t pad;
};

// One (cost degree, chain degree) class of sites in the plane engine.
struct PlaneType {
    int dc, dq;      // cost / chain degree of every site of this type
    int ncb, nqb;    // bits of the n_c / n_q bit-sliced counters
    int ncl;         // classes = 1 << (ncb+nqb), padded to >= 4
    int kp_off;      // word offset of this type's [54][ncl] block inside one word block
    int ktab_off;    // offset of this type's classes inside one slot row of ktab
    int pad;
};

// A run of <= 32 consecutive sites of one colour and one type.
struct Chunk {
    int start;       // first internal site
    int len;         // 1..32
    int type;        // PlaneType index
    int nbr_base;    // offset into nbr[] of site `start`
};

struct PlaneArgs {
    int n;                // sites
    int W;                // 32-replica words per site row (padded to the pass width)
    int n_colors;
    int local_states;     // replicas on this rank (<= 32*W)
    int rule;
    int n_types;
    int kpw;              // words per word-block of kp
    int m_cost;           // number of cost couplings (whole instance)
    uint32_t* spins;      // [n][W]
    const int32_t* nbr;   // per site: dc cost neighbours (bit31 = J<0), dq chain partners
    const int4* nbr4;     // tpw config-5 path: per site {3 cost neighbours, chain partner} as
                          // row offsets (index << log2 W), bit 31 = J<0 (cost) / no partner (4th)
    const Chunk* chunks;  // all colours, concatenated
    const int* chunk_off; // [n_colors+1]
    const int* color_start; // [n_colors+1] internal site ranges
    const uint32_t* kp;   // [W][kpw] threshold planes for the current labels
    const uint32_t* kpc;  // [W][n_types][2][64] class-major planes of classes 2,3 (pruned Metropolis types)
    PlaneType ty[kMaxTypes];     // by value: constant bank
    const int32_t* state_slot;   // [R] slot of each physical state (tail thresholds)
    const uint64_t* ktab;        // [R][ktab_row] 53-bit thresholds
    int ktab_row;
    uint32_t pks[20];            // plane-draw Philox key schedule (run key, 10 rounds)
    int w_global0;               // global index of this rank's first 32-replica group
    uint32_t active[kMaxWordsArg]; // lane masks of real replicas (0 for padding words)
    int32_t* cnt_c;       // [32W] unsatisfied cost bonds (accumulated)
    int32_t* cnt_q;       // [32W] unsatisfied chain bonds
    double* f_loc;        // [local_states]
    double* g_loc;
    const RoundState* rs; // unfused loop: sweep index t0 = rs->round * n_sweeps (else the argument)
};

struct SlotArgs {
    int n;
    int n_colors;
    int local_states;
    int state0;           // global id of local state 0
    int rule;
    int I, J;
    int8_t* spins;        // [local_states][n]
    const int* off;       // merged CSR [n+1], neighbours in increasing index order
    const int32_t* nbr;
    const double* w;      // cost weight J (0 for pure chain entries)
    const int8_t* cm;     // chain multiplicity of the entry
    const double* h;      // fields
    const int2* ent;      // FP32 fast path: {j | cm<<28, float bits of J}
    const int2* entp;     // padded [n][D] copy of ent; bit 27 = forward edge (j > i); pads point at i with w = 0
    const double* wp;     // padded [n][D] FP64 cost weights (energy pass)
    int D;                // padded degree (0: general CSR kernel)
    const float* h32;
    float eps_local;      // bound on |local_fp32 - local_fp64| over all sites
    float beta_max;
    const int* color_start;
    const double* betas;
    const double* pens;
    const int32_t* state_slot; // [R] slot of each physical state
    const uint64_t* slot_key;  // [R] derive_seed(seed, replica, slot)
    double* f_loc;
    double* g_loc;
    const RoundState* rs;      // unfused loop: t0 = rs->round * n_sweeps (else the argument)
};

// Fused single-GPU round loop (plane engine).
struct RoundArgs {
    int I, J, R, sps;
    int64_t round0;        // first round (1-based) of this launch
    int n_rounds;
    int rec_flags;         // 1 digest, 2 target state, 8 counters
    uint64_t swap_base0;   // swap-stream draws consumed before round0
    uint64_t swap_seed;
    const double* betas;
    const double* pens;
    int32_t* slot_state;   // [R] global labels (read at start, published per round)
    int32_t* state_slot;
    int64_t* acc_p;
    int64_t* acc_b;
    double* f_all;
    double* g_all;
    int32_t* cnt;          // [2 parities][2 (cost, chain)][cnt_stride]
    int* work;             // [2 parities][n_colors][passes] chunk counters (dynamic distribution)
    int cnt_stride;
    int flush_every;       // tpw kernel: items between vertical-counter flushes (host: <= 255 / max bonds)
    int n_warps;           // tpw kernel: warps of the launch
    int log_w;             // tpw kernel: log2 of the words per site
    int c5_nfree[2];       // c5 kernel: chain-free sites of colours 0, 1 (they precede the chain sites)
    int cl_stage;          // cluster kernel: neighbour entries staged in shared memory (TMA)
    int cl_size;           // cluster kernel: CTAs per cluster the host launched with
    int cl_ktab;           // cluster kernel: ktab staged in shared memory
    unsigned int* cl_bar;  // cluster kernel, group mode: per-word barrier counters [W][32] (one line each)
    int32_t* cl_gtot;      // cluster kernel, group mode: word totals [2 parities][W][64]
    unsigned long long* cl_x;  // cluster kernel: (f, g) exchange words [2 parities][32 W], each
                           // {round tag : 16 | chain count : 24 | cost count : 24}; [2 * 32 W] = error word
    const uint64_t* ktab;
    int ktab_row;
    uint32_t* kp;
    uint32_t* kpc;
    void* rec;             // TgRecordDev[n_rounds], digests pre-zeroed
    int64_t* rec_acc;
    int8_t* rec_states;    // [n_rounds][n] or null
    const int32_t* perm;
};

struct SwapArgs {
    int I, J, R;
    const double* betas;
    const double* pens;
    const double* f_all;   // [R] per physical state
    const double* g_all;
    int32_t* slot_state;   // [R]
    int32_t* state_slot;   // [R]
    int64_t* acc_p;        // [I*(J-1)]
    int64_t* acc_b;        // [(I-1)*J]
    uint64_t swap_seed;
    // record
    void* rec;             // tg_record ring
    int rec_cap;
    int64_t* rec_acc;      // [cap][np+nb] or null
    // plane-engine label tables
    int plane;
    int W, state0, local_states, n_types, kpw;
    const PlaneType* types;
    const uint64_t* ktab;  // [R][ktab_row]: 53-bit thresholds (>= 2^53: always)
    int ktab_row;
    uint32_t* kp;
    uint32_t* kpc;
    const RoundState* rs;  // round = rs->round + 1, swap_base, record index from it (else arguments)
    RoundState* tick;      // unfused loop: advance the round state once the record is written (else null)
};

// ------------------------------------------------- SLOT engine v2 (batched)

struct SInst {              // one instance of a batch (device table)
    int n, D, n_colors, color_off;
    long long spin_off;     // into spins: n * Rp int8
    int entp_off;           // into entp / wp: n * D
    int csr_off;            // into off: n + 1
    int nbr_off;            // into nbr / w / cm
    int h_off;              // into h / h32 / perm (also the instance's site offset)
    int chunk_off;          // into part_f / part_g rows: ceil(n / 32) chunks
    int n_chunks;
    int state_off;          // sum of n over earlier instances (record snapshots)
    float eps, beta_max;    // FP32 fast-path error bound, max |beta|
    unsigned long long pkey; // FLOAT engine: packed-draw key derive_seed(seed, PACK, 0)
};

struct S2Args {
    int B, I, J, R, Rp, G, rule, max_colors;
    const SInst* inst;
    int8_t* spins;                 // [b][site][Rp]
    const int2* entp;              // padded degree-D entries {j | cm<<28 | fwd<<27, float J}
    const double* wp;              // padded FP64 J (energy)
    const int* off;                // merged CSR per instance (FP64 fallback)
    const int32_t* nbr;
    const double* w;
    const int8_t* cm;
    const double* h;
    const float* h32;
    const int* color_start;        // per instance n_colors + 1
    const int* item_pref;          // [max_colors][B+1] prefix sums of sweep-item upper bounds
    const int* energy_pref;        // [B+1] prefix sums of energy items
    const double* betas;           // [B][I]
    const double* pens;            // [B][J]
    const int32_t* state_slot;     // [B][R]
    const uint64_t* slot_key;      // [B][R]
    double* part_f;                // [B][nsub][Rp] per-warp energy partials (fixed order)
    double* part_g;
    double* f;                     // [B][R]
    double* g;
    const double* sbeta;           // [B][Rp] beta of the slot each physical replica occupies
    const double* stwop;           // [B][Rp] 2P of that slot
    const uint64_t* skey;          // [B][Rp] Philox key of that slot's stream
    int nsub;                      // warps per replica group
    // FLOAT engine (slot_fast.cu)
    const float2* lab;             // [B][Rp] (beta, 2P) of the slot each physical replica occupies
    long long* fx;                 // [B][Rp] cost energy, 2^-40 fixed point (zeroed after use)
    int* gx;                       // [B][Rp] unsatisfied chain bonds x multiplicity
    const int* fitem_pref;         // [max_colors][B+1] prefix sums of warp items
    int flps, fspw, fngs;          // lanes per site, sites per warp item, 256-replica group sets
    double* hist_f;                // probes: per-sweep (f, g) of every replica,
    double* hist_g;                //   [t - hist_t0][B*R], for sweeps t >= hist_t0
    int64_t hist_t0;
};

struct S2Swap {
    int R, I, J, rec_cap;
    const double* betas;
    const double* pens;
    const double* f;
    const double* g;
    int32_t* slot_state;           // [B][R]
    int32_t* state_slot;
    int64_t* acc_p;                // [B][I(J-1)]
    int64_t* acc_b;                // [B][(I-1)J]
    const uint64_t* swap_seed;     // [B]
    void* rec;                     // TgRecordDev [B][rec_cap]
    int64_t* rec_acc;              // [B][rec_cap][np+nb]
    int8_t* rec_states;            // snapshots, or null
    const int32_t* perm;           // internal -> caller index, per instance (offset h_off)
    double* sbeta;                 // per-state label tables refreshed after the swaps
    double* stwop;
    uint64_t* skey;
    const uint64_t* slot_key;      // [B][R]
    int Rp;
    float2* lab;                   // FLOAT engine label table (or null)
};

// Decoded-sample histogram + KL per round (analysis.cpp:215-241).
struct KLArgs {
    int n_logical, K, discard, ncopies;
    const int* map_off;            // [n_logical + 1]
    const int* map;                // [B][ncopies] internal spin index of each copy
    const double* p;               // [K] exact logical Boltzmann probabilities
    uint32_t* hist;                // [B][K]
    unsigned long long* total;     // [B]
    double* kl;                    // [B][cap]
    int64_t* samples;              // [B][cap]
    int64_t cap;
    int* error;                    // set when an observed state has zero target mass
};

// ---------------------------------------------------------------- swaps

// Reference round schedule (engine.cpp:121-146,216): parity alternates every
// round; the direction (P first) flips after every even round.
TG_HD void round_phase(int I, int J, int64_t round, int& even, int& do_p, int& do_b) {
    even = (round % 2 == 0) ? 1 : 0;
    const int direction = (((round - 1) / 2) % 2 == 0) ? 1 : -1;
    if (I == 1 && J == 1) { do_p = do_b = 0; }
    else if (I == 1) { do_p = 1; do_b = 0; }
    else if (J == 1) { do_p = 0; do_b = 1; }
    else { do_p = direction == 1; do_b = !do_p; }
}

TG_HD int pairs_in(int len, int even) { return len - even >= 2 ? (len - even) / 2 : 0; }

TG_HD int64_t round_attempts(int I, int J, int64_t round) {
    int even, dp, db;
    round_phase(I, J, round, even, dp, db);
    return dp ? (int64_t)I * pairs_in(J, even) : (db ? (int64_t)J * pairs_in(I, even) : 0);
}

TG_HD double dadd_mul(double f, double p, double g) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(f, __dmul_rn(p, g));  // no FMA contraction: match the reference
#else
    return f + p * g;
#endif
}

TG_HD double dexp(double x) {
#if defined(__CUDA_ARCH__)
    return exp(x);
#else
    return __builtin_exp(x);
#endif
}

// Attempt k of the round: P phase rows i ascending, pairs p = even, even+2..
// (engine.cpp:148-167); beta phase columns j ascending, pairs b = even, ..
// (engine.cpp:168-187).  One swap-stream draw per attempt in that order (u).
// Split in two so that the fused kernels can do everything that does not
// depend on this round's energies (slots, labels, coefficients, the draw)
// before the energies arrive: swap_prepare, then swap_decide.
struct SwapPrep {
    int slot_a, slot_b, counter, is_p;
    int sa, sb;      // states in the two slots before the attempt
    double c;        // P phase: beta_i (P_{p+1} - P_p); beta phase: beta_{b+1} - beta_b
    double pj;       // beta phase: the column's penalty
    double u;
};

TG_HD SwapPrep swap_prepare(int I, int J, const double* betas, const double* pens, int64_t round, int k,
                            const int32_t* slot_state, double u) {
    SwapPrep p;
    int even, dp, db;
    round_phase(I, J, round, even, dp, db);
    p.u = u;
    if (dp) {
        const int per = pairs_in(J, even);
        const int i = k / per;
        const int q = even + 2 * (k % per);
        p.slot_a = i * J + q;
        p.slot_b = p.slot_a + 1;
        p.c = betas[i] * (pens[q + 1] - pens[q]);
        p.pj = 0.0;
        p.counter = i * (J - 1) + q;
        p.is_p = 1;
    } else {
        const int per = pairs_in(I, even);
        const int j = k / per;
        const int b = even + 2 * (k % per);
        p.slot_a = b * J + j;
        p.slot_b = (b + 1) * J + j;
        p.pj = pens[j];
        p.c = betas[b + 1] - betas[b];
        p.counter = b * J + j;
        p.is_p = 0;
    }
    p.sa = slot_state[p.slot_a];
    p.sb = slot_state[p.slot_b];
    return p;
}

// Accept (1) or reject (0): x >= 0 or u < exp(x), the reference expressions
// in the reference's operation order.
TG_HD int swap_decide(const SwapPrep& p, const double* f_all, const double* g_all) {
    double x;
    if (p.is_p) {
        x = p.c * (g_all[p.sb] - g_all[p.sa]);
    } else {
        const double e_lo = dadd_mul(f_all[p.sa], p.pj, g_all[p.sa]);
        const double e_hi = dadd_mul(f_all[p.sb], p.pj, g_all[p.sb]);
        x = p.c * (e_hi - e_lo);
    }
    const double u = p.u;
#if defined(__CUDA_ARCH__)
    // Certified shortcut around the FP64 exp (a long dependent chain in a
    // phase that is one attempt per thread): an FP32 exp bounds exp(x) within
    // 1e-4 relative for x in [-100, 0) (input rounding |x| 2^-24, ex2.approx
    // 2^-22); only a uniform inside that band (probability ~2e-4) takes the
    // FP64 expression, so the decisions are the FP64 ones.
    if (x >= 0.0) return 1;
    if (x < -100.0) return (u > 0.0) ? 0 : (u < dexp(x) ? 1 : 0);  // exp(x) < 2^-53 <= every u > 0
    const double e32 = (double)__expf((float)x);
    if (u < e32 * (1.0 - 1e-4)) return 1;
    if (u > e32 * (1.0 + 1e-4)) return 0;
    return u < dexp(x) ? 1 : 0;
#else
    return (x >= 0.0 || u < dexp(x)) ? 1 : 0;
#endif
}

TG_HD int swap_attempt_u(int I, int J, const double* betas, const double* pens, int64_t round,
                         int k, const double* f_all, const double* g_all, const int32_t* slot_state,
                         double u, int& slot_a, int& slot_b, int& counter, int& is_p) {
    const SwapPrep p = swap_prepare(I, J, betas, pens, round, k, slot_state, u);
    slot_a = p.slot_a;
    slot_b = p.slot_b;
    counter = p.counter;
    is_p = p.is_p;
    return swap_decide(p, f_all, g_all);
}

// The attempt's uniform: draw swap_base + k of the swap stream.
TG_HD double swap_uniform(uint64_t swap_seed, uint64_t swap_base, int k) {
    return (double)(stream_bits(swap_seed, swap_base + (uint64_t)k) >> 11) * 0x1.0p-53;
}

TG_HD int swap_attempt(int I, int J, const double* betas, const double* pens, int64_t round,
                       int k, const double* f_all, const double* g_all, const int32_t* slot_state,
                       uint64_t swap_seed, uint64_t swap_base, int& slot_a, int& slot_b,
                       int& counter, int& is_p) {
    return swap_attempt_u(I, J, betas, pens, round, k, f_all, g_all, slot_state,
                          swap_uniform(swap_seed, swap_base, k), slot_a, slot_b, counter, is_p);
}

}  // namespace tg
