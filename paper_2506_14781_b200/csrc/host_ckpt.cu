// host_ckpt.cu -- checkpoint / resume of a single-GPU run (tg_checkpoint,
// tg_restore; include/tempergrid_b200.h).  The reference has no resume (its
// Trace lives in RAM, engine.hpp:39-56); here a run's continuation depends
// only on the spins of every physical state, the slot labels, the cumulative
// accept counters, the round counter and the swap-stream position -- the
// Philox draws are functions of (seed, counters) -- so that is the snapshot.
#include "host.cuh"

namespace tgh {

namespace {

constexpr uint32_t kCkptMagic = 0x50434754u;  // "TGCP"

struct CkptView {
    tg_checkpoint_header* h;
    int8_t* states;      // [R][n] caller order
    int32_t* slot_state; // [R]
    int64_t* acc_p;      // [I(J-1)]
    int64_t* acc_b;      // [(I-1)J]
};

size_t ckpt_bytes(int n, int I, int J) {
    const size_t R = (size_t)I * J, np = (size_t)I * std::max(0, J - 1), nb = (size_t)std::max(0, I - 1) * J;
    return sizeof(tg_checkpoint_header) + R * n + 4 * R + 8 * (np + nb);
}

CkptView view(void* buf, int n, int I, int J) {
    CkptView v;
    char* p = static_cast<char*>(buf);
    const size_t R = (size_t)I * J, np = (size_t)I * std::max(0, J - 1);
    v.h = reinterpret_cast<tg_checkpoint_header*>(p);
    p += sizeof(tg_checkpoint_header);
    v.states = reinterpret_cast<int8_t*>(p);
    p += R * n;
    v.slot_state = reinterpret_cast<int32_t*>(p);
    p += 4 * R;
    v.acc_p = reinterpret_cast<int64_t*>(p);
    p += 8 * np;
    v.acc_b = reinterpret_cast<int64_t*>(p);
    return v;
}

void check_ctx(const tg_ctx& c) {
    if (!c.initialised) fail(TG_ERR_CONFIG, "checkpoint: context not initialised (tg_init)");
    if (c.world != 1) fail(TG_ERR_CONFIG, "checkpoint: single-GPU contexts only");
    if (c.use_s2 && c.s2.B != 1) fail(TG_ERR_CONFIG, "checkpoint: batches are not supported");
}

}  // namespace

size_t checkpoint_size(tg_ctx& c) {
    check_ctx(c);
    return ckpt_bytes(c.n, c.I, c.J);
}

void checkpoint(tg_ctx& c, void* buf, size_t bytes) {
    check_ctx(c);
    if (bytes < ckpt_bytes(c.n, c.I, c.J)) fail(TG_ERR_CONFIG, "checkpoint: buffer too small");
    cudaStream_t st = c.stream;
    const int n = c.n, R = c.R, np = c.I * std::max(0, c.J - 1), nb = std::max(0, c.I - 1) * c.J;
    CkptView v = view(buf, n, c.I, c.J);
    tg_checkpoint_header& h = *v.h;
    h = tg_checkpoint_header{};
    h.magic = kCkptMagic;
    h.version = 1;
    h.engine = c.engine;
    h.rule = c.cfg.rule;
    h.n = n;
    h.I = c.I;
    h.J = c.J;
    h.seed = c.cfg.seed;
    if (c.use_s2) {
        Slot2& S = c.s2;
        h.rounds_done = S.rounds_done;
        h.swap_base = S.swap_base;
        std::vector<int8_t> sp((size_t)n * S.Rp);
        CK(cudaMemcpyAsync(sp.data(), S.d_spins.p, sp.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(v.slot_state, S.d_slot_state.p, 4 * (size_t)R, cudaMemcpyDeviceToHost, st));
        if (np) CK(cudaMemcpyAsync(v.acc_p, S.d_acc_p.p, 8 * (size_t)np, cudaMemcpyDeviceToHost, st));
        if (nb) CK(cudaMemcpyAsync(v.acc_b, S.d_acc_b.p, 8 * (size_t)nb, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const std::vector<int>& order = S.prep[0].order;  // internal -> caller
        for (int i = 0; i < n; ++i)
            for (int m = 0; m < R; ++m) v.states[(size_t)m * n + order[i]] = sp[(size_t)i * S.Rp + m];
        return;
    }
    if (c.engine != TG_ENGINE_PLANE) fail(TG_ERR_CONFIG, "checkpoint: engine not supported");
    h.rounds_done = c.rounds_done;
    h.swap_base = c.swap_base;
    std::vector<uint32_t> sp((size_t)n * c.W);
    std::vector<int32_t> perm(n);
    CK(cudaMemcpyAsync(sp.data(), c.d_spins32.p, 4 * sp.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(perm.data(), c.d_perm.p, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(v.slot_state, c.d_slot_state.p, 4 * (size_t)R, cudaMemcpyDeviceToHost, st));
    if (np) CK(cudaMemcpyAsync(v.acc_p, c.d_acc_p.p, 8 * (size_t)np, cudaMemcpyDeviceToHost, st));
    if (nb) CK(cudaMemcpyAsync(v.acc_b, c.d_acc_b.p, 8 * (size_t)nb, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i)
        for (int m = 0; m < R; ++m)
            v.states[(size_t)m * n + perm[i]] = ((sp[(size_t)i * c.W + (m >> 5)] >> (m & 31)) & 1u) ? 1 : -1;
}

void restore(tg_ctx& c, const void* buf, size_t bytes) {
    check_ctx(c);
    const int n = c.n, R = c.R, np = c.I * std::max(0, c.J - 1), nb = std::max(0, c.I - 1) * c.J;
    if (bytes < sizeof(tg_checkpoint_header) || bytes < ckpt_bytes(n, c.I, c.J))
        fail(TG_ERR_CONFIG, "restore: buffer too small");
    CkptView v = view(const_cast<void*>(buf), n, c.I, c.J);
    const tg_checkpoint_header& h = *v.h;
    if (h.magic != kCkptMagic || h.version != 1) fail(TG_ERR_CONFIG, "restore: not a tempergrid checkpoint");
    if (h.engine != c.engine || h.rule != c.cfg.rule || h.n != n || h.I != c.I || h.J != c.J ||
        h.seed != c.cfg.seed)
        fail(TG_ERR_CONFIG, "restore: checkpoint of another engine / problem / schedule / seed");
    if (h.rounds_done < 0) fail(TG_ERR_CONFIG, "restore: bad round counter");
    std::vector<int32_t> state_slot(R, -1);
    for (int s = 0; s < R; ++s) {
        const int m = v.slot_state[s];
        if (m < 0 || m >= R || state_slot[m] >= 0) fail(TG_ERR_CONFIG, "restore: labels are not a permutation");
        state_slot[m] = s;
    }
    for (size_t q = 0; q < (size_t)R * n; ++q)
        if (v.states[q] != 1 && v.states[q] != -1) fail(TG_ERR_CONFIG, "restore: spins must be +-1");
    cudaStream_t st = c.stream;
    if (c.use_s2) {
        Slot2& S = c.s2;
        const std::vector<int>& order = S.prep[0].order;
        std::vector<int8_t> sp((size_t)n * S.Rp, 1);
        for (int i = 0; i < n; ++i)
            for (int m = 0; m < R; ++m) sp[(size_t)i * S.Rp + m] = v.states[(size_t)m * n + order[i]];
        CK(cudaMemcpyAsync(S.d_spins.p, sp.data(), sp.size(), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(S.d_slot_state.p, v.slot_state, 4 * (size_t)R, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(S.d_state_slot.p, state_slot.data(), 4 * (size_t)R, cudaMemcpyHostToDevice, st));
        if (np) CK(cudaMemcpyAsync(S.d_acc_p.p, v.acc_p, 8 * (size_t)np, cudaMemcpyHostToDevice, st));
        if (nb) CK(cudaMemcpyAsync(S.d_acc_b.p, v.acc_b, 8 * (size_t)nb, cudaMemcpyHostToDevice, st));
        // per-physical-replica label tables (slot2_swap_kernel's refresh)
        const BatchInst& bi = c.batch[0];
        std::vector<double> sb(S.Rp, 0.0), stp(S.Rp, 0.0);
        std::vector<uint64_t> sk(S.Rp, 0);
        std::vector<float2> lab(S.Rp, make_float2(0.f, 0.f));
        for (int m = 0; m < R; ++m) {
            const int sl = state_slot[m];
            sb[m] = bi.betas[sl / S.J];
            stp[m] = 2.0 * bi.pens[sl % S.J];
            sk[m] = derive_seed(bi.seed, kPurposeReplica, (uint64_t)sl);
            lab[m] = make_float2((float)sb[m], (float)stp[m]);
        }
        CK(cudaMemcpyAsync(S.d_sbeta.p, sb.data(), 8 * (size_t)S.Rp, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(S.d_stwop.p, stp.data(), 8 * (size_t)S.Rp, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(S.d_skey.p, sk.data(), 8 * (size_t)S.Rp, cudaMemcpyHostToDevice, st));
        if (S.fast) CK(cudaMemcpyAsync(S.d_lab.p, lab.data(), sizeof(float2) * S.Rp, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        S.rounds_done = h.rounds_done;
        S.swap_base = h.swap_base;
        c.rounds_done = h.rounds_done;
        return;
    }
    if (c.engine != TG_ENGINE_PLANE) fail(TG_ERR_CONFIG, "restore: engine not supported");
    std::vector<int32_t> perm(n);
    CK(cudaMemcpyAsync(perm.data(), c.d_perm.p, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<uint32_t> sp((size_t)n * c.W, 0u);
    for (int i = 0; i < n; ++i)
        for (int m = 0; m < R; ++m)
            if (v.states[(size_t)m * n + perm[i]] > 0) sp[(size_t)i * c.W + (m >> 5)] |= 1u << (m & 31);
    CK(cudaMemcpyAsync(c.d_spins32.p, sp.data(), 4 * sp.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(c.d_slot_state.p, v.slot_state, 4 * (size_t)R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(c.d_state_slot.p, state_slot.data(), 4 * (size_t)R, cudaMemcpyHostToDevice, st));
    if (np) CK(cudaMemcpyAsync(c.d_acc_p.p, v.acc_p, 8 * (size_t)np, cudaMemcpyHostToDevice, st));
    if (nb) CK(cudaMemcpyAsync(c.d_acc_b.p, v.acc_b, 8 * (size_t)nb, cudaMemcpyHostToDevice, st));
    rebuild_planes(c);  // threshold planes of the restored labels
    CK(cudaStreamSynchronize(st));
    c.rounds_done = h.rounds_done;
    c.swap_base = h.swap_base;
}

}  // namespace tgh

using namespace tgh;

extern "C" int tg_checkpoint_size(tg_ctx* ctx, size_t* bytes) {
    if (!ctx || !bytes) return TG_ERR_CONFIG;
    return guard(ctx, [&] { *bytes = checkpoint_size(*ctx); });
}

extern "C" int tg_checkpoint(tg_ctx* ctx, void* buf, size_t bytes) {
    if (!ctx || !buf) return TG_ERR_CONFIG;
    return guard(ctx, [&] { checkpoint(*ctx, buf, bytes); });
}

extern "C" int tg_restore(tg_ctx* ctx, const void* buf, size_t bytes) {
    if (!ctx || !buf) return TG_ERR_CONFIG;
    return guard(ctx, [&] { restore(*ctx, buf, bytes); });
}
