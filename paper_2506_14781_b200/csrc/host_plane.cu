// host_plane.cu -- PLANE engine host driver: eligibility, structure from the device prep (or the host), threshold tables, launch arguments, the fused round loop.
#include "host.cuh"
#include "plane_round.cuh"

namespace tgh {

// Launch bound and co-resident blocks per SM of a kernel at `smem` dynamic
// bytes (raising its dynamic shared-memory limit when needed), cached per
// (device, kernel, threads, smem): the queries cost tens of microseconds and
// set_problem runs once per e2e step.
struct KernelFit {
    int max_threads = 0, blocks_per_sm = 0;
};
static KernelFit kernel_fit(const void* fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, size_t>, KernelFit> cache;
    static std::map<std::pair<int, const void*>, size_t> smem_set;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, fn, threads, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    KernelFit f;
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, fn));
    f.max_threads = fa.maxThreadsPerBlock;
    if (threads <= 0) threads = f.max_threads;
    size_t& have = smem_set[std::make_pair(dev, fn)];
    if (smem > 48 * 1024 && smem > have) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        have = smem;
    }
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f.blocks_per_sm, fn, threads, smem));
    cache[key] = f;
    return f;
}

bool plane_eligible(tg_ctx& c, std::string* why) {
    if (c.dev_prep) {
        if (c.prep.info & kPrepNotPM1) { if (why) *why = "couplings must be +-1"; return false; }
        if (c.prep.info & kPrepNonzeroField) { if (why) *why = "fields must be 0"; return false; }
        if (c.prep.max_dc > kMaxDC || c.prep.max_dq > kMaxDQ) { if (why) *why = "degree bound exceeded"; return false; }
        return true;
    }
    ensure_host_arrays(c);
    for (double w : c.cw) if (!(w == 1.0 || w == -1.0)) { if (why) *why = "couplings must be +-1"; return false; }
    for (double x : c.h) if (x != 0.0) { if (why) *why = "fields must be 0"; return false; }
    std::vector<int> dc(c.n, 0), dq(c.n, 0);
    for (size_t k = 0; k < c.ci.size(); ++k) { dc[c.ci[k]]++; dc[c.cj[k]]++; }
    for (size_t k = 0; k < c.pa.size(); ++k) { dq[c.pa[k]]++; dq[c.pb[k]]++; }
    for (int i = 0; i < c.n; ++i)
        if (dc[i] > kMaxDC || dq[i] > kMaxDQ) { if (why) *why = "degree bound exceeded"; return false; }
    return true;
}

void build_plane_structure_device(tg_ctx& c, std::vector<PlaneType>& types, std::vector<Chunk>& chunks,
                                  std::vector<int>& chunk_off) {
    const PrepSummary& P = c.prep;
    const int mq1 = P.max_dq + 1, mc1 = P.max_dc + 1;
    std::vector<int> tid_of((kMaxDC + 1) * (kMaxDQ + 1), -1);
    chunk_off.assign(c.n_colors + 1, 0);
    int start = 0, cur_col = -1;
    for (size_t q = 0; q < P.run_keys.size(); ++q) {
        const unsigned key = P.run_keys[q];
        const int cnt = P.run_counts[q];
        const int dc = (int)(key % mc1), dq = (int)((key / mc1) % mq1), col = (int)(key / ((unsigned)mc1 * mq1));
        while (cur_col < col) chunk_off[++cur_col] = (int)chunks.size();
        const int tkey = dc * (kMaxDQ + 1) + dq;
        if (tid_of[tkey] < 0) {
            PlaneType t{};
            t.dc = dc;
            t.dq = dq;
            t.ncb = nbits(dc);
            t.nqb = nbits(dq);
            t.ncl = std::max(4, 1 << (t.ncb + t.nqb));
            tid_of[tkey] = (int)types.size();
            types.push_back(t);
        }
        for (int s0 = start; s0 < start + cnt; s0 += 32)
            chunks.push_back(Chunk{s0, std::min(32, start + cnt - s0), tid_of[tkey], 0});
        start += cnt;
    }
    while (cur_col < c.n_colors) chunk_off[++cur_col] = (int)chunks.size();
    chunk_off[c.n_colors] = (int)chunks.size();
}

// Site types, per-colour chunk offsets and the run table of the device prep's
// runs (same chunk order as build_plane_structure_device).
void build_plane_types_device(tg_ctx& c, std::vector<PlaneType>& types, std::vector<int>& chunk_off,
                              RunTable& rt) {
    const PrepSummary& P = c.prep;
    const int mq1 = P.max_dq + 1, mc1 = P.max_dc + 1;
    std::vector<int> tid_of((kMaxDC + 1) * (kMaxDQ + 1), -1);
    chunk_off.assign(c.n_colors + 1, 0);
    int start = 0, cur_col = -1, nch = 0;
    c.c5_nfree[0] = c.c5_nfree[1] = 0;
    rt.n = (int)P.run_keys.size();
    for (int q = 0; q < rt.n; ++q) {
        const unsigned key = P.run_keys[q];
        const int cnt = P.run_counts[q];
        const int dc = (int)(key % mc1), dq = (int)((key / mc1) % mq1), col = (int)(key / ((unsigned)mc1 * mq1));
        while (cur_col < col) chunk_off[++cur_col] = nch;
        const int tkey = dc * (kMaxDQ + 1) + dq;
        if (tid_of[tkey] < 0) {
            PlaneType t{};
            t.dc = dc;
            t.dq = dq;
            t.ncb = nbits(dc);
            t.nqb = nbits(dq);
            t.ncl = std::max(4, 1 << (t.ncb + t.nqb));
            tid_of[tkey] = (int)types.size();
            types.push_back(t);
        }
        if (dq == 0 && col < 2) c.c5_nfree[col] += cnt;
        rt.start[q] = start;
        rt.cnt[q] = cnt;
        rt.type[q] = tid_of[tkey];
        rt.cpref[q] = nch;
        nch += (cnt + 31) / 32;
        start += cnt;
    }
    rt.cpref[rt.n] = nch;
    while (cur_col < c.n_colors) chunk_off[++cur_col] = nch;
    chunk_off[c.n_colors] = nch;
}

void build_plane(tg_ctx& c) {
    HostTimer tm_("build_plane");
    cudaStream_t st = c.stream;
    const int n = c.n;
    if (c.dev_prep) {
        std::vector<PlaneType> types;
        std::vector<Chunk> chunks;
        std::vector<int> chunk_off;
        c.d_nbr.copy_from(c.d_nbr_dev, st);
        if (c.prep.run_keys.size() <= (size_t)kMaxRuns) {
            // the chunk list is a function of the few (colour, type) runs:
            // generate it on the device (a host list of ~n/32 chunks costs
            // first-touch page faults on every set_problem)
            RunTable rt{};
            build_plane_types_device(c, types, chunk_off, rt);
            c.d_chunks.alloc((size_t)rt.cpref[rt.n]);
            CK(plane_gen_chunks(rt, c.d_chunks.p, st));
            CK(plane_chunk_bases(c.d_chunks.p, rt.cpref[rt.n], c.d_base_dev.p, st, c.sms));
        } else {
            build_plane_structure_device(c, types, chunks, chunk_off);
            c.c5_nfree[0] = c.c5_nfree[1] = 0;
            for (int col = 0; col < std::min(2, c.n_colors); ++col)
                for (int q = chunk_off[col]; q < chunk_off[col + 1]; ++q)
                    if (types[chunks[q].type].dq == 0) c.c5_nfree[col] += chunks[q].len;
            c.d_chunks.upload(chunks, st);
            CK(plane_chunk_bases(c.d_chunks.p, (int)chunks.size(), c.d_base_dev.p, st, c.sms));
        }
        build_plane_rest(c, types, chunk_off);
        return;
    }
    ensure_host_arrays(c);
    ensure_host_canonical(c);
    // internal adjacency as flat CSR (cost entries carry the J<0 sign bit)
    std::vector<int> dcv(n, 0), dqv(n, 0);
    for (size_t k = 0; k < c.ci.size(); ++k) { dcv[c.inv[c.ci[k]]]++; dcv[c.inv[c.cj[k]]]++; }
    for (size_t k = 0; k < c.pa.size(); ++k) { dqv[c.inv[c.pa[k]]]++; dqv[c.inv[c.pb[k]]]++; }
    std::vector<int> base(n + 1, 0);
    for (int i = 0; i < n; ++i) base[i + 1] = base[i] + dcv[i] + dqv[i];
    std::vector<int32_t> nbr(base[n]);
    {
        std::vector<int> cc(n), cq(n);
        for (int i = 0; i < n; ++i) { cc[i] = base[i]; cq[i] = base[i] + dcv[i]; }
        for (size_t k = 0; k < c.ci.size(); ++k) {
            const int x = c.inv[c.ci[k]], y = c.inv[c.cj[k]];
            const int32_t sgn = c.cw[k] < 0 ? (int32_t)0x80000000u : 0;
            nbr[cc[x]++] = y | sgn;
            nbr[cc[y]++] = x | sgn;
        }
        for (size_t k = 0; k < c.pa.size(); ++k) {
            const int x = c.inv[c.pa[k]], y = c.inv[c.pb[k]];
            nbr[cq[x]++] = y;
            nbr[cq[y]++] = x;
        }
    }
    // site types (cost degree, chain degree)
    std::vector<int> tid_of((kMaxDC + 1) * (kMaxDQ + 1), -1);
    std::vector<int> site_type(n);
    std::vector<PlaneType> types;
    for (int i = 0; i < n; ++i) {
        const int key = dcv[i] * (kMaxDQ + 1) + dqv[i];
        if (tid_of[key] < 0) {
            PlaneType t{};
            t.dc = dcv[i];
            t.dq = dqv[i];
            t.ncb = nbits(t.dc);
            t.nqb = nbits(t.dq);
            t.ncl = std::max(4, 1 << (t.ncb + t.nqb));
            tid_of[key] = (int)types.size();
            types.push_back(t);
        }
        site_type[i] = tid_of[key];
    }
    // chunks (colour-major; the canonical order keeps types contiguous)
    std::vector<Chunk> chunks;
    std::vector<int> chunk_off(c.n_colors + 1, 0);
    for (int col = 0; col < c.n_colors; ++col) {
        chunk_off[col] = (int)chunks.size();
        int i = c.color_start[col];
        const int end = c.color_start[col + 1];
        while (i < end) {
            const int ty = site_type[i];
            int j = i;
            while (j < end && j - i < 32 && site_type[j] == ty) ++j;
            chunks.push_back(Chunk{i, j - i, ty, base[i]});
            i = j;
        }
    }
    chunk_off[c.n_colors] = (int)chunks.size();
    c.c5_nfree[0] = c.c5_nfree[1] = 0;
    for (int col = 0; col < std::min(2, c.n_colors); ++col)
        for (int q = chunk_off[col]; q < chunk_off[col + 1]; ++q)
            if (types[chunks[q].type].dq == 0) c.c5_nfree[col] += chunks[q].len;
    c.d_nbr.upload(nbr, st);
    c.d_chunks.upload(chunks, st);
    build_plane_rest(c, types, chunk_off);
}

// Everything after the site types and chunks: threshold tables, words, keys,
// masks, buffers and the cooperative grids.
void build_plane_rest(tg_ctx& c, std::vector<PlaneType>& types, const std::vector<int>& chunk_off) {
    cudaStream_t st = c.stream;
    const int n = c.n;
    if ((int)types.size() > kMaxTypes) fail(TG_ERR_RESOURCE, "plane engine: too many site types");
    int kpw = 0, krow = 0;
    for (auto& t : types) {
        t.kp_off = kpw;
        t.ktab_off = krow;
        kpw += kKWords * t.ncl;
        krow += t.ncl;
    }
    c.kpw = kpw;
    c.ktab_row = krow;
    c.n_types = (int)types.size();
    // words, keys, masks: rows padded to a whole number of WV-word passes
    const int w_log = (c.R_local + 31) / 32;
    c.WV = w_log > 2 ? 4 : w_log;
    if (const char* e = std::getenv("TG_PLANE_WV")) {  // tuning override: 1, 2 or 4
        const int v = std::atoi(e);
        if (v == 1 || v == 2 || v == 4) c.WV = std::min(v, w_log > 2 ? 4 : (w_log > 1 ? 2 : 1));
    }
    c.W = (w_log + c.WV - 1) / c.WV * c.WV;
    if (c.W > kMaxWordsArg) fail(TG_ERR_RESOURCE, "plane engine: %d replicas per rank exceed %d", c.R_local, 32 * kMaxWordsArg);
    std::vector<uint32_t> active(c.W, 0u);
    std::vector<uint2> wkey(c.W);
    for (int w = 0; w < c.W; ++w) {
        for (int l = 0; l < 32; ++l) if (w * 32 + l < c.R_local) active[w] |= 1u << l;
        const uint64_t k = derive_seed(c.cfg.seed, kPurposePlane, (uint64_t)(c.state0 / 32 + w));
        wkey[w] = make_uint2((uint32_t)k, (uint32_t)(k >> 32));
    }
    // thresholds per (slot, type, class)
    std::vector<uint64_t> ktab((size_t)c.R * krow, 0ull);
    for (int slot = 0; slot < c.R; ++slot) {
        const double beta = c.betas[slot / c.J], P = c.pens[slot % c.J];
        for (const auto& t : types) {
            for (int cl = 0; cl < t.ncl; ++cl) {
                const int ncnt = cl & ((1 << t.ncb) - 1);
                const int qcnt = cl >> t.ncb;
                uint64_t K = 0;
                if (ncnt <= t.dc && qcnt <= t.dq) {
                    // s_i * local_i (Metropolis, counts of satisfied bonds) or
                    // local_i (heat bath, counts of +1 contributions)
                    const double v = (double)(2 * ncnt - t.dc) + 2.0 * P * (double)(2 * qcnt - t.dq);
                    K = c.cfg.rule == TG_RULE_METROPOLIS ? threshold_metropolis(beta, 2.0 * v)
                                                         : threshold_heat_bath(beta, v);
                }
                ktab[(size_t)slot * krow + t.ktab_off + cl] = K;
            }
        }
    }
    // Metropolis, cost degree 3, no chain partner: flag bit 0 = classes 2 and
    // 3 (de > 0) are never "always" under any label, so a lane is undecided
    // iff its class is 2 or 3 (plane_tpw.cu's single-select compare)
    for (auto& t : types) {
        t.pad = 0;
        if (c.cfg.rule != TG_RULE_METROPOLIS || t.dc != 3 || t.dq != 0 || t.ncb != 2) continue;
        bool ok = true;
        for (int slot = 0; slot < c.R && ok; ++slot)
            for (int cl = 2; cl < 4; ++cl)
                if (ktab[(size_t)slot * krow + t.ktab_off + cl] >= (1ull << 53)) ok = false;
        t.pad = ok ? 1 : 0;
    }
    c.m_cost = c.m;
    c.d_chunk_off.upload(chunk_off, st);
    c.d_color_start.upload(c.color_start, st);
    c.d_types.upload(types, st);
    c.h_types = types;
    c.h_active = active;
    c.h_wkey = wkey;
    c.d_ktab.upload(ktab, st);
    c.d_kp.alloc((size_t)c.W * kpw);
    c.d_kp.zero(st);
    c.d_kpc.alloc((size_t)c.W * c.n_types * 128);
    c.d_kpc.zero(st);
    c.d_spins32.alloc((size_t)n * c.W);
    c.d_cnt_c.alloc((size_t)c.W * 32);
    c.d_cnt_q.alloc((size_t)c.W * 32);
    c.d_cnt_c.zero(st);
    c.d_cnt_q.zero(st);
    c.d_cnt2.alloc((size_t)4 * c.W * 32);
    c.d_cnt2.zero(st);
    c.d_work.alloc((size_t)2 * c.n_colors * std::max(1, c.W));
    c.d_work.zero(st);
    // cooperative grid: a multiple of W warps, all blocks co-resident
    const int per_sm = kernel_fit((const void*)plane_sweep_fn(c.cfg.rule, c.WV), kPlaneThreads, 0).blocks_per_sm;
    if (per_sm < 1) fail(TG_ERR_RESOURCE, "plane engine: kernel does not fit on an SM");
    int blocks = per_sm * c.sms;
    const int passes = c.W / c.WV;
    blocks -= blocks % passes;  // each block owns one pass of WV words
    if (blocks < passes) fail(TG_ERR_RESOURCE, "plane engine: cannot tile %d words", c.W);
    c.plane_grid = blocks;
    // fused round-loop kernel (single GPU)
    c.fused_fast = 1;
    for (const auto& t : types) if (t.ncb > 2 || t.nqb > 1) c.fused_fast = 0;
    // FAST: specialised kernel for site types with cost degree <= 3 and chain
    // degree <= 1 (config 5), cp.async row prefetch; TG_PLANE_FAST=0 disables.
    if (const char* e = std::getenv("TG_PLANE_FAST")) c.fused_fast = c.fused_fast && std::atoi(e) != 0;
    c.fused_grid = 0;
    c.fused_tpw = 0;
    // tpw FAST variant (c5_site): every site of cost degree 3 and chain
    // degree 0 / 1; Metropolis: chain-free types with flag bit 0
    // (heat bath: any labels, its chain-free classes staged per phase)
    c.tpw_fast = 1;
    for (const auto& t : types) {
        const bool metro_ok = t.dq == 1 || (t.dq == 0 && (t.pad & 1));
        if (!(t.dc == 3 && t.dq <= 1 && (c.cfg.rule != TG_RULE_METROPOLIS || metro_ok))) c.tpw_fast = 0;
    }
    if (const char* e = std::getenv("TG_PLANE_FAST")) c.tpw_fast = c.tpw_fast && std::atoi(e) != 0;
    // the config-5 path's per-site padded neighbour table (row offsets)
    c.d_nbr4.release();
    if (c.tpw_fast && (c.W & (c.W - 1)) == 0 && c.W <= 32) {
        TypeDq tdq{};
        for (int q = 0; q < c.n_types; ++q) tdq.dq[q] = types[q].dq;
        int logW = 0;
        while ((1 << logW) < c.W) ++logW;
        c.d_nbr4.alloc((size_t)n);
        CK(tpw_build_nbr4(c.d_chunks.p, (int)c.d_chunks.n, tdq, c.d_nbr.p, logW, c.d_nbr4.p, st));
    }
    // thread-per-(site, word) kernels (rows of a power-of-two number of
    // words): by default only on their config-5 path, where they are faster
    // (r1: 1.60e12 vs 1.39e12 flips/s); on generic site types and heat bath
    // the thread-per-site kernels measured faster (1.34e12 vs 1.08e12).
    // TG_PLANE_TPW = 0 never, 2 always (generic path included), else auto.
    int tpw_mode = 1;
    if (const char* e = std::getenv("TG_PLANE_TPW")) tpw_mode = std::atoi(e);
    const bool tpw_ok = (c.W & (c.W - 1)) == 0 && c.W <= 32 &&
                        (tpw_mode == 2 || (tpw_mode == 1 && c.tpw_fast));
    if (c.world == 1 && c.R <= 2048 && tpw_ok) c.fused_tpw = 1;
    // sweep-only tpw kernel (multi-GPU rounds, full-grid records)
    c.tpw_sweep_grid = 0;
    if (tpw_ok) {
        const void* fn = plane_tpw_sweep_fn(c.cfg.rule, c.tpw_fast);
        c.tpw_sweep_smem = tpw_smem_bytes(0, c.W, kernel_fit(fn, 0, 0).max_threads);
        const int fb = kernel_fit(fn, 0, c.tpw_sweep_smem).blocks_per_sm;
        if (fb >= 1) c.tpw_sweep_grid = fb * c.sms;
    }
    // config-5 kernel (plane_c5.cu): either rule on the tpw config-5 path with
    // a 2-colouring, at least two words per site row; TG_PLANE_C5=0 disables
    c.fused_c5 = 0;
    c.c5_sweep_grid = 0;
    {
        bool elig = tpw_ok && c.tpw_fast && c.n_colors == 2 &&
                    c.W >= 2 && c.n_types <= 2 && c.d_nbr4.p != nullptr &&
                    (long long)n * c.W < (1ll << 30);  // 32-bit byte offsets of the rows
        int nfree_type = 0;
        for (const auto& t : types) nfree_type += t.dq == 0;
        elig = elig && nfree_type <= 1;
        if (const char* e = std::getenv("TG_PLANE_C5")) elig = elig && std::atoi(e) != 0;
        if (elig) {  // its sweep-only form for the unfused round loop (multi-GPU ranks, full-grid records)
            const size_t smem = c5_smem_bytes(c.R, c.W);
            const int fb = kernel_fit(plane_c5_sweep_fn(c.cfg.rule), kC5Threads, smem).blocks_per_sm;
            if (fb >= 1) {
                c.c5_sweep_grid = fb * c.sms;
                c.c5_sweep_smem = smem;
            }
        }
        const bool ok = elig && c.fused_tpw;
        if (ok) {
            const size_t smem = c5_smem_bytes(c.R, c.W);
            const int fb = kernel_fit(plane_c5_fn(c.cfg.rule), kC5Threads, smem).blocks_per_sm;
            if (fb >= 1) {
                c.fused_c5 = 1;
                c.fused_grid = fb * c.sms;
                c.fused_block = kC5Threads;
                c.fused_smem = smem;
            }
        }
    }
    // word-local kernel (plane_cl.cu): the same config-5 path with the CTAs
    // partitioned by 32-replica word (or word pair), so that a colour phase
    // ends with a barrier among the word's CTAs only, one tagged-word (f, g)
    // exchange per round replaces the other grid barriers, and neighbour
    // entries, ktab and threshold planes live in shared memory (entries staged
    // by TMA).  Two launch modes: hardware thread-block clusters (cluster
    // barrier, DSMEM count reduction; on B200 at most 10 CTAs per word when 8
    // words are needed, i.e. 80 SMs) and "group": an ordinary cooperative
    // launch with G = SMs / groups CTAs per word behind a software barrier.
    // Measured on B200 (profiles/r2/c5_sizes_r2.json) group mode is the faster
    // from 2^14 sites up, with one word per thread up to 2^15 sites and a word
    // pair per thread up to 2^18; above that plane_c5 (all words of a row in
    // adjacent lanes: full 32-byte sectors) wins.  TG_PLANE_CL = 0 never, 1
    // whenever eligible; TG_PLANE_CL_MODE = cluster | group; TG_PLANE_CL_PAIR
    // = 0 | 1; TG_PLANE_CL_SIZE caps the CTAs per word.
    c.fused_cl = 0;
    {
        bool ok = c.world == 1 && c.R <= 2048 && c.tpw_fast && c.n_colors == 2 && c.n_types <= 2 &&
                  c.d_nbr4.p != nullptr && c.W <= kMaxWordsArg;
        int nfree_type = 0;
        for (const auto& t : types) nfree_type += t.dq == 0;
        ok = ok && nfree_type <= 1;
        int mode = -1;
        if (const char* e = std::getenv("TG_PLANE_CL")) mode = std::atoi(e);
        if (mode == 0 || (mode < 0 && n > (1 << 18))) ok = false;
        int cmax = 1 << 20;  // cap on the CTAs per word (cluster mode: <= 16 anyway)
        if (const char* e = std::getenv("TG_PLANE_CL_SIZE")) cmax = std::max(1, std::atoi(e));
        // the exchange words carry 24-bit bond counts
        ok = ok && c.m_cost < (1 << 24) && c.np < (1 << 24);
        int gmode = 1;
        if (const char* e = std::getenv("TG_PLANE_CL_MODE")) gmode = std::string(e) == "group";
        if (ok) {
            int dev = 0, smem_max = 0;
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            struct Plan { size_t smem; int stage, kt, small; const void* fn; };
            auto plan = [&](int C, int group, int wpt, Plan& P) -> bool {
                // entries of the largest slice set (rank 0) and its sites per thread and phase
                size_t total = 0;
                int items[2] = {0, 0};
                for (int q = 0; q < 4; ++q) {
                    const int col = q >> 1;
                    const int cs = c.color_start[col], ce = c.color_start[col + 1], cf = cs + c.c5_nfree[col];
                    const int len = (q & 1) ? ce - cf : cf - cs;
                    int per = (len + C - 1) / C;
                    per = (per + 31) & ~31;
                    total += (size_t)std::min(per, len);
                    items[col] += (std::min(per, len) + kClThreads - 1) / kClThreads;
                }
                P.small = std::max(items[0], items[1]) <= 5 && !std::getenv("TG_PLANE_CL_BIGCNT");
                P.fn = plane_cl_fn(c.cfg.rule, P.small, group, wpt == 2);
                // staged in shared memory when they fit: ktab first (24 KB at 16x16), then the entries
                const size_t ktw = (size_t)c.R * c.ktab_row;
                P.kt = 1;
                P.stage = std::getenv("TG_PLANE_CL_NOSTAGE") ? 0 : 1;
                if (cl_smem_bytes(c.R, c.I, c.J, c.kpw, c.n_types, ktw, 0, wpt) > (size_t)smem_max || ktw * 8 > 64 * 1024)
                    P.kt = 0;
                if (cl_smem_bytes(c.R, c.I, c.J, c.kpw, c.n_types, P.kt ? ktw : 0, total, wpt) > (size_t)smem_max)
                    P.stage = 0;
                P.smem = cl_smem_bytes(c.R, c.I, c.J, c.kpw, c.n_types, P.kt ? ktw : 0, P.stage ? total : 0, wpt);
                if (P.smem > (size_t)smem_max) return false;
                CK(cudaFuncSetAttribute(P.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
                return true;
            };
            auto take = [&](int C, int group, int wpt, const Plan& P) {
                c.fused_cl = 1;
                c.cl_group = group;
                c.cl_pair = wpt == 2;
                c.cl_size = C;
                c.cl_stage = P.stage;
                c.cl_ktab = P.kt;
                c.cl_small = P.small;
                c.fused_grid = c.W / wpt * C;
                c.fused_block = kClThreads;
                c.fused_smem = P.smem;
                // exchange words [2][32 W] | error word | barrier lines [W][16] | group totals [2][W][32]
                c.d_clx.alloc((size_t)2 * c.W * 32 + 1 + (size_t)16 * c.W + (size_t)64 * c.W);
            };
            if (gmode) {  // G CTAs per word (or word pair) of an ordinary cooperative launch
                // two words per thread when the row has an even number of words: the pair shares the
                // site's Philox products and row sectors (plane_c5.cu); TG_PLANE_CL_PAIR=0 disables
                int wpt = (c.W % 2 == 0 && n > (1 << 15)) ? 2 : 1;
                if (const char* e = std::getenv("TG_PLANE_CL_PAIR")) wpt = std::atoi(e) != 0 && c.W % 2 == 0 ? 2 : 1;
                const int G = std::min(c.sms / (c.W / wpt), cmax);
                Plan P;
                if (G >= 1 && plan(G, 1, wpt, P)) {
                    int per_sm = 0;
                    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, P.fn, kClThreads, P.smem));
                    if (std::getenv("TG_PLANE_CL_VERBOSE"))
                        std::fprintf(stderr, "plane_cl: group G=%d wpt=%d smem=%zu stage=%d ktab=%d small=%d blocks/SM=%d\n",
                                     G, wpt, P.smem, P.stage, P.kt, P.small, per_sm);
                    if (per_sm >= 1) take(G, 1, wpt, P);
                }
            }
            for (int C = 16; C >= 1 && !c.fused_cl; --C) {  // any size: GPCs differ in SM count
                if (C > cmax || c.W * C > c.sms) continue;
                Plan P;
                if (!plan(C, 0, 1, P)) continue;
                CK(cudaFuncSetAttribute(P.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3(c.W * C);
                lc.blockDim = dim3(kClThreads);
                lc.dynamicSmemBytes = P.smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = C;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                int nact = 0;
                if (cudaOccupancyMaxActiveClusters(&nact, P.fn, &lc) != cudaSuccess) {
                    cudaGetLastError();
                    continue;
                }
                if (std::getenv("TG_PLANE_CL_VERBOSE"))
                    std::fprintf(stderr, "plane_cl: C=%d smem=%zu stage=%d ktab=%d small=%d active clusters=%d (need %d)\n",
                                 C, P.smem, P.stage, P.kt, P.small, nact, c.W);
                if (nact >= c.W) take(C, 0, 1, P);
            }
        }
        if (c.fused_cl) c.fused_c5 = 0;
    }
    if (c.fused_tpw && !c.fused_c5 && !c.fused_cl) {
        const void* fn = plane_tpw_fn(c.cfg.rule, c.tpw_fast);
        c.fused_block = kernel_fit(fn, 0, 0).max_threads;  // the kernel's launch bound
        c.fused_smem = tpw_smem_bytes(c.R, c.W, c.fused_block);
        const int fb = kernel_fit(fn, c.fused_block, c.fused_smem).blocks_per_sm;
        if (fb >= 1) c.fused_grid = fb * c.sms;
        else c.fused_tpw = 0;
    }
    if (!c.fused_tpw && !c.fused_cl && c.world == 1 && c.R <= 2048) {
        c.fused_wv = c.WV;
        const void* fn = plane_rounds_fn(c.cfg.rule, c.fused_wv, c.fused_fast);
        c.fused_block = c.fused_fast ? kPlaneThreadsFast : kPlaneThreads;
        const size_t pf_words = c.fused_fast && (c.fused_wv == 4 || c.fused_wv == 2)
                                    ? (size_t)2 * (5 * 32 * c.fused_wv + 4 * 32) : 0;
        c.fused_smem = (size_t)c.R * (2 * sizeof(double) + 2 * sizeof(int32_t)) + 8 +
                       (size_t)(c.fused_block / 32) * pf_words * sizeof(int32_t);
        const int fb = kernel_fit(fn, c.fused_block, c.fused_smem).blocks_per_sm;
        if (fb >= 1) {
            int g = fb * c.sms;
            const int fp = c.fused_wv ? passes : 1;
            g -= g % fp;
            if (g >= fp) c.fused_grid = g;
        }
    }
}

PlaneArgs plane_args(tg_ctx& c) {
    PlaneArgs a{};
    a.n = c.n;
    a.W = c.W;
    a.n_colors = c.n_colors;
    a.local_states = c.R_local;
    a.rule = c.cfg.rule;
    a.n_types = c.n_types;
    a.kpw = c.kpw;
    a.m_cost = c.m_cost;
    a.spins = c.d_spins32.p;
    a.nbr = c.d_nbr.p;
    a.nbr4 = c.d_nbr4.p;
    a.chunks = c.d_chunks.p;
    a.chunk_off = c.d_chunk_off.p;
    a.color_start = c.d_color_start.p;
    for (int q = 0; q < c.n_types && q < kMaxTypes; ++q) a.ty[q] = c.h_types[q];
    for (int w = 0; w < c.W && w < kMaxWordsArg; ++w) a.active[w] = c.h_active[w];
    philox_key_schedule(derive_seed(c.cfg.seed, kPurposePlane, 0), a.pks);
    a.state_slot = c.d_state_slot.p;
    a.ktab = c.d_ktab.p;
    a.ktab_row = c.ktab_row;
    a.w_global0 = c.state0 / 32;
    a.kp = c.d_kp.p;
    a.kpc = c.d_kpc.p;
    a.cnt_c = c.d_cnt_c.p;
    a.cnt_q = c.d_cnt_q.p;
    a.f_loc = c.d_f.p + c.state0;
    a.g_loc = c.d_g.p + c.state0;
    return a;
}

void rebuild_planes(tg_ctx& c) {
    if (c.engine != TG_ENGINE_PLANE) return;
    SwapArgs a = swap_args(c);
    // round 1 of a 1x1-like schedule attempts nothing: fake I=J=1 for the swap part
    a.I = 1;
    a.J = 1;
    swap_kernel<<<1, kSwapThreads, 0, c.stream>>>(a, 1, 0, c.rec_cap, 0);
    CK(cudaGetLastError());
}

void s2_build(tg_ctx& c, const tg_run_config* cfg);

void do_advance_fused(tg_ctx& c, int64_t n_rounds, const SinkCtx& sink) {
    NvtxRange nv_("tg: fused rounds (sweeps + swaps + records)");
    cudaStream_t st = c.stream;
    const int flags = c.cfg.record_flags;
    if (c.profiling && c.ev.size() < 2) {
        for (auto e : c.ev) cudaEventDestroy(e);
        c.ev.assign(2, nullptr);
        for (auto& e : c.ev) CK(cudaEventCreate(&e));
    }
    double sweep_ms = 0;
    int64_t left = n_rounds;
    while (left > 0) {
        const int n = (int)std::min<int64_t>(left, c.rec_cap);
        CK(cudaMemsetAsync(c.d_rec.p, 0, sizeof(TgRecordDev) * n, st));
        PlaneArgs a = plane_args(c);
        RoundArgs r{};
        r.I = c.I; r.J = c.J; r.R = c.R; r.sps = (int)c.cfg.sweeps_per_swap;
        r.round0 = c.rounds_done + 1;
        r.n_rounds = n;
        r.rec_flags = flags & (TG_REC_DIGEST | TG_REC_STATE | TG_REC_COUNTERS);
        r.swap_base0 = c.swap_base;
        r.swap_seed = derive_seed(c.cfg.seed, kPurposeSwap, 0);
        r.betas = c.d_betas.p; r.pens = c.d_pens.p;
        r.slot_state = c.d_slot_state.p; r.state_slot = c.d_state_slot.p;
        r.acc_p = c.d_acc_p.p; r.acc_b = c.d_acc_b.p;
        r.f_all = c.d_f.p; r.g_all = c.d_g.p;
        r.cnt = c.d_cnt2.p; r.cnt_stride = c.W * 32;
        // tpw kernel: 8-bit vertical counters take <= 255 / (max bonds per item)
        // items between flushes (config-5 path: 3, generic: 7); testing knob
        // TG_TPW_FLUSH_EVERY flushes more often
        r.flush_every = c.tpw_fast ? 255 / 3 : 255 / 7;
        if (const char* e = std::getenv("TG_TPW_FLUSH_EVERY")) {
            const int v = std::atoi(e);
            if (v > 0 && v < r.flush_every) r.flush_every = v;
        }
        r.n_warps = c.fused_grid * (c.fused_block / 32);
        r.log_w = 0;
        while ((1 << r.log_w) < c.W) ++r.log_w;
        // tpw kernel: the last ~item per warp of each colour phase is handed
        // out dynamically ([2 parities][colours][sps] counters)
        r.work = nullptr;
        r.c5_nfree[0] = c.c5_nfree[0];
        r.c5_nfree[1] = c.c5_nfree[1];
        if (c.fused_tpw && c.tpw_fast && !c.fused_c5 && !c.fused_cl) {
            const size_t need = (size_t)2 * c.n_colors * c.cfg.sweeps_per_swap;
            if (c.d_work.n < need) { c.d_work.alloc(need); c.d_work.zero(st); }
            r.work = std::getenv("TG_TPW_STATIC") ? nullptr : c.d_work.p;
        }
        r.ktab = c.d_ktab.p; r.ktab_row = c.ktab_row; r.kp = c.d_kp.p; r.kpc = c.d_kpc.p;
        r.rec = c.d_rec.p; r.rec_acc = c.d_rec_acc.p;
        r.rec_states = (flags & TG_REC_STATE) ? c.d_rec_states.p : nullptr;
        r.perm = c.d_perm.p;
        if (c.fused_cl) {
            r.cl_stage = c.cl_stage;
            r.cl_size = c.cl_size;
            r.cl_ktab = c.cl_ktab;
            r.cl_x = c.d_clx.p;
            r.cl_bar = reinterpret_cast<unsigned int*>(c.d_clx.p + (size_t)2 * c.W * 32 + 1);
            r.cl_gtot = reinterpret_cast<int32_t*>(c.d_clx.p + (size_t)2 * c.W * 32 + 1 + (size_t)16 * c.W);
            CK(cudaMemsetAsync(c.d_clx.p, 0, sizeof(unsigned long long) * c.d_clx.n, st));
        }
        void* args[] = {&a, &r};
        if (c.profiling) CK(cudaEventRecord(c.ev[0], st));
        c.sweep_kernel = c.fused_cl ? "plane_cl_rounds_kernel"
                         : c.fused_c5 ? "plane_c5_rounds_kernel"
                                      : c.fused_tpw ? "plane_tpw_rounds_kernel" : "plane_rounds_kernel";
        const void* fn = c.fused_cl ? plane_cl_fn(c.cfg.rule, c.cl_small, c.cl_group, c.cl_pair)
                         : c.fused_c5 ? plane_c5_fn(c.cfg.rule)
                                      : c.fused_tpw ? plane_tpw_fn(c.cfg.rule, c.tpw_fast)
                                                    : plane_rounds_fn(c.cfg.rule, c.fused_wv, c.fused_fast);
        if (c.fused_cl && !c.cl_group) {
            // W clusters of cl_size CTAs, all co-resident (cooperative launch)
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(c.fused_grid);
            lc.blockDim = dim3(c.fused_block);
            lc.dynamicSmemBytes = c.fused_smem;
            lc.stream = st;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c.cl_size;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeCooperative;
            at[1].val.cooperative = 1;
            lc.attrs = at;
            lc.numAttrs = std::getenv("TG_PLANE_CL_NOCOOP") ? 1 : 2;
            CK(cudaLaunchKernelExC(&lc, fn, args));
        } else {
            CK(cudaLaunchCooperativeKernel(fn, dim3(c.fused_grid), dim3(c.fused_block), args, c.fused_smem, st));
        }
        if (c.profiling) CK(cudaEventRecord(c.ev[1], st));
        c.sweep_launches++;
        const int64_t first = c.rounds_done + 1;
        for (int k = 0; k < n; ++k) c.swap_base += (uint64_t)round_attempts(c.I, c.J, first + k);
        c.rounds_done += n;
        left -= n;
        {
            NvtxRange nr_("tg: drain records");
            drain(c, n, first, sink);
        }
        if (c.profiling) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
            sweep_ms += ms;
        }
    }
    unsigned long long cl_err = 0;
    if (c.fused_cl)
        CK(cudaMemcpyAsync(&cl_err, c.d_clx.p + (size_t)2 * c.W * 32, sizeof(cl_err), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (cl_err)
        fail(TG_ERR_CUDA, "plane_cl_rounds_kernel ran without its cluster dimension (profilers drop it from "
                          "cooperative launches: set TG_PLANE_CL_NOCOOP=1)");
    c.last_sweep_ms = sweep_ms;
    c.last_swap_ms = 0;
}


}  // namespace tgh
