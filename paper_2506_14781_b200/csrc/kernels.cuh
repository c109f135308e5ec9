// kernels.cuh -- launch interface of kernels.cu for the host driver.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "engine.cuh"

namespace tg {

constexpr int kPlaneThreads = 512;
constexpr int kPlaneThreadsFast = 512;
constexpr int kPlaneMinBlocksFast = 1;
#ifndef TG_TPW_THREADS
#define TG_TPW_THREADS 512
#endif
constexpr int kTpwThreads = TG_TPW_THREADS;  // thread-per-(site, word) fused kernel (plane_tpw.cu)
#ifndef TG_TPW_MINB
#define TG_TPW_MINB 1
#endif
constexpr int kTpwMinBlocks = TG_TPW_MINB;
constexpr int kTpwVB = 8;               // planes of its vertical bond counters
constexpr int kTpwQCap = 64;            // per-warp deferred-tail queue entries (>= 31 + 32)
constexpr int kTpwQFields = 7;          // words per queue entry
constexpr int kTpwHbWords = 9 * 32 * 4; // heat-bath threshold stage: [9 planes][<= 32 words] uint4
// Dynamic shared memory of plane_tpw_rounds_kernel: tail queues
// [warps][kTpwQFields][kTpwQCap], chain vertical counters [kTpwVB][threads],
// the heat-bath threshold stage, per-replica counters [2][32W], labels and
// energies (plane_round.cuh).
inline size_t tpw_smem_bytes(int R, int W, int threads) {
    return (size_t)R * (2 * sizeof(double) + 2 * sizeof(int32_t)) + 8 + (size_t)2 * W * 32 * sizeof(int) +
           (size_t)kTpwVB * threads * sizeof(int) + (size_t)kTpwHbWords * sizeof(int) +
           (size_t)(threads / 32) * kTpwQCap * kTpwQFields * sizeof(int);
}
// config-5 fused round kernel (plane_c5.cu): threads per CTA, per-warp tail
// queue entries (>= 31 + 2 words x 32 lanes), dynamic shared memory = queues
// [warps][kC5QCap] int4, staged thresholds [32 words][36], per-replica
// counters [2][32W], labels and energies.
#ifndef TG_C5_THREADS
#define TG_C5_THREADS 512
#endif
#ifndef TG_C5_MINB
#define TG_C5_MINB 1
#endif
constexpr int kC5Threads = TG_C5_THREADS;
constexpr int kC5MinBlocks = TG_C5_MINB;
constexpr int kC5QCap = 96;
inline size_t c5_smem_bytes(int R, int W) {
    return (size_t)(kC5Threads / 32) * kC5QCap * 16 + (size_t)kMaxWordsArg * 36 * sizeof(int) +
           (size_t)2 * W * 32 * sizeof(int) +
           (size_t)R * (2 * sizeof(double) + 2 * sizeof(int32_t)) + 8;
}
void* plane_c5_fn(int rule);
void* plane_c5_sweep_fn(int rule);  // sweep-only (unfused round loop)
// cluster-per-word fused round kernel (plane_cl.cu): threads per CTA, per-warp
// tail queue entries (>= 31 + 32), dynamic shared memory = queues | the word's
// kp / kpc planes | counts | mbarrier | labels and energies | staged entries.
constexpr int kClThreads = 512;
constexpr int kClQCap = 64;
inline size_t cl_smem_bytes(int R, int I, int J, int kpw, int n_types, size_t ktab_words,
                            size_t stage_entries, int wpt) {
    return (size_t)(kClThreads / 32) * kClQCap * 16 + (size_t)wpt * ((kpw + 3) & ~3) * 4 +
           (size_t)wpt * n_types * 128 * 4 + 24 * 4 + (size_t)wpt * 128 * 4 + 16 +
           (size_t)((I + 1) & ~1) * 8 + (size_t)((J + 1) & ~1) * 8 +
           (size_t)((I * (J > 1 ? J - 1 : 0) + (I > 1 ? I - 1 : 0) * J + 3) & ~3) * 4 +
           ((size_t)R * (2 * sizeof(double) + 2 * sizeof(int32_t)) + 8 + 15) / 16 * 16 +
           ((2 * ktab_words + 3) & ~(size_t)3) * 4 + stage_entries * 16;
}
// small: <= 5 sites per thread and phase (4-plane counters); group: software word barrier (no
// clusters); pair: two words per thread (group mode)
void* plane_cl_fn(int rule, int small, int group, int pair);
constexpr int kSlotThreads = 256;
constexpr int kSwapThreads = 1024;

// Device image of tg_record (same layout as the C-ABI struct).
struct TgRecordDev {
    int64_t round;
    int64_t sweep_count;
    double f;
    double g;
    int32_t feasible;
    int32_t target_state;
    uint64_t digest;
};

struct ExtractArgs {
    int n, R, W, plane, all_slots, local_states, state0;
    const int32_t* slot_state;
    const uint32_t* spins32;
    const int8_t* spins8;
    const int32_t* perm;  // internal -> caller index
    int8_t* states;       // [1 or R][n] caller order, or null
    uint64_t* digest;     // record digest slot, or null
    // unfused loop: the chunk's state ring / digest array, indexed by rs->filled
    const RoundState* rs;
    int rs_back;          // 1: the record slot is rs->filled - 1 (swap_kernel advanced the state already)
    size_t per_state;
};
__global__ void round_tick_kernel(RoundState* rs, int I, int J);

void* plane_sweep_fn(int rule, int wv);
void* plane_rounds_fn(int rule, int wv, int fast);
void* plane_tpw_fn(int rule, int fast);
void* plane_tpw_sweep_fn(int rule, int fast);
struct TypeDq { int dq[kMaxTypes]; };
cudaError_t tpw_build_nbr4(const Chunk* chunks, int n_chunks, TypeDq tdq, const int32_t* nbr, int logW,
                           int4* out, cudaStream_t st);
int plane_words_per_pass(int W);
void* slot_sweep_fn();
void* slot_sweep_fn_d(int D);  // padded-degree variant, D in {4, 8}

constexpr int kSlot2Threads = 512;
constexpr int kSlotFThreads = 512;   // FLOAT engine sweep kernel (slot_fast.cu)
void* slotf_sweep_fn(int rule, int deg);
void* slot2_sweep_fn(int D, bool hist = false);
__global__ void slot2_swap_kernel(const __grid_constant__ S2Swap s, int64_t round, uint64_t swap_base,
                                  int rec_idx, int rec_flags);
__global__ void slot2_extract_kernel(const __grid_constant__ S2Args a, const __grid_constant__ S2Swap s,
                                     int rec_idx, int all_slots);
__global__ void slot2_init_kernel(const __grid_constant__ S2Args a, const uint64_t* init_keys);
__global__ void slot2_energy_kernel(const __grid_constant__ S2Args a, int n_slices, double* part);
__global__ void slot2_energy_sum_kernel(const __grid_constant__ S2Args a, int n_slices, const double* part);
__global__ void slot2_kl_kernel(const __grid_constant__ S2Args a, const int32_t* slot_state,
                                const __grid_constant__ KLArgs k, int64_t round);
// ---- device instance preprocessing for the PLANE engine (prep.cu)
enum : unsigned {
    kPrepBadCoupling = 1u, kPrepBadPair = 2u, kPrepBadField = 4u, kPrepDuplicate = 8u,
    kPrepErrors = 15u,
    kPrepNotPM1 = 16u, kPrepNonzeroField = 32u  // plane-engine eligibility (not errors)
};
constexpr int kPrepColourRounds = 4096;
// largest (colour, dq, dc) run list read back together with the run count
constexpr size_t kPrepEagerRuns = 1 << 16;
struct PrepIn {             // device arrays, caller order
    int n, m, np;
    const int* ci;
    const int* cj;
    const double* w;
    const double* h;
    const int* pa;
    const int* pb;
};
struct PrepOut {            // caller-allocated device outputs
    int* order;             // [n] internal -> caller
    int* inv;               // [n] caller -> internal
    int* base;              // [n + 1] internal row offsets
    int* nbr;               // [2 (m + np)] internal rows (cost | sign, then chain)
};
struct PrepSummary {        // host
    unsigned bad = 0;       // kPrep* error flags: invalid instance (host re-validates for the message)
    unsigned info = 0;      // kPrepNotPM1 / kPrepNonzeroField
    bool colour_incomplete = false;
    int colour_rounds = 0, n_colors = 0, max_dc = 0, max_dq = 0;
    std::vector<unsigned> run_keys;   // sorted (colour, dq, dc) keys, one per run
    std::vector<int> run_counts;
};
cudaError_t plane_prep_device(const PrepIn& in, const PrepOut& o, PrepSummary& r, cudaStream_t st,
                              int sms);
cudaError_t plane_chunk_bases(Chunk* chunks, int n_chunks, const int* base, cudaStream_t st, int sms);
// Chunks of <= 32 sites per run of one (colour, site type), generated on the
// device from the run table (kernels.cu); nbr_base is filled by plane_chunk_bases.
constexpr int kMaxRuns = 64;
struct RunTable {
    int n;
    int start[kMaxRuns], cnt[kMaxRuns], type[kMaxRuns];
    int cpref[kMaxRuns + 1];  // first chunk of each run
};
cudaError_t plane_gen_chunks(const RunTable& rt, Chunk* chunks, cudaStream_t st);

__global__ void probe_moments_kernel(const double* hist_f, const double* hist_g, int R, int kept,
                                     double penalty, double* out);

__global__ void plane_rebuild_kernel(SwapArgs a);
__global__ void swap_kernel(SwapArgs a, int64_t round, uint64_t swap_base, int rec_idx,
                            int rec_flags);
__global__ void extract_kernel(ExtractArgs e);
__global__ void plane_init_kernel(uint32_t* spins, int n, int W, int local_states, int state0,
                                  uint64_t seed);
__global__ void slot_init_kernel(int8_t* spins, int n, int local_states, int state0, uint64_t seed);

}  // namespace tg
