// capi.cpp — host runtime behind include/csattn_b200.h.
//
// Owns device memory per session (one KV head: prefill rows shared across
// forks, appended-row tails, centroids, index-sorted tables), validates every
// call on the host in the reference's order and with the reference's error
// classes/messages, assembles per-launch problem descriptors and launches the
// sm_100a kernels (csrc/*.cu). No computation of the hot path happens here;
// there is no CPU fallback: every compute entry point launches a kernel or fails.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "csattn_b200.h"
#include "kernels.h"
#include "kmeans.h"
#include "errors.hpp"
#include "csat.h"
#include <random>

namespace csa_host {
thread_local std::string g_err;
}  // namespace csa_host

namespace {

using csa_host::Fail;
using csa_host::fail;
using csa_host::g_err;
using csa_host::guard;

// a nested C-ABI call's failure, re-raised with its status and message
void check_status(csattn_status st) {
    if (st != CSATTN_OK) fail(st, g_err);
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(CSATTN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}


// set while a decode graph is being captured (run_graph): every buffer was sized
// by the preceding sizing pass, so a growth here would leave the graph pointing
// at freed memory
thread_local bool g_no_alloc = false;

struct DevMem {
    void* p = nullptr;
    size_t n = 0;
    bool host = false;  // mapped pinned host memory (KV offload), device-addressable through UVA
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() { release(); }
    void release() {
        if (p) host ? cudaFreeHost(p) : cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t bytes) {
        if (g_no_alloc) fail(CSATTN_ERR_GENERIC, "internal: buffer growth while capturing a decode graph");
        static const bool prof = std::getenv("CSATTN_HOST_PROF") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        release();
        host = false;
        if (bytes == 0) bytes = 16;
        ck(cudaMalloc(&p, bytes), "cudaMalloc");
        n = bytes;
        if (prof) {
            const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            if (us > 1000.0) std::fprintf(stderr, "[csattn] slow device alloc: %zu bytes in %.1f us\n", bytes, us);
        }
    }
    // pinned host memory the kernels read and write over the host link
    void alloc_host(size_t bytes) {
        if (g_no_alloc) fail(CSATTN_ERR_GENERIC, "internal: buffer growth while capturing a decode graph");
        release();
        host = true;
        if (bytes == 0) bytes = 16;
        ck(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc");
        n = bytes;
    }
    void alloc_on(bool on_host, size_t bytes) { on_host ? alloc_host(bytes) : alloc(bytes); }
    void ensure(size_t bytes) {
        if (bytes > n) alloc(bytes + bytes / 2);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ceil_ratio (util.hpp:77-81)
uint64_t ceil_ratio(double ratio, uint64_t n) {
    const double v = ratio * static_cast<double>(n);
    const double c = std::ceil(v - 1e-9);
    return c <= 0.0 ? 0 : static_cast<uint64_t>(c);
}

// keep_count (retrieval.cpp:34-38)
uint64_t keep_count(double rho, uint64_t n) {
    if (!(rho > 0.0 && rho <= 1.0)) fail(CSATTN_ERR_PARAMETER, "keep ratio must lie in (0, 1]");
    return std::max<uint64_t>(1, ceil_ratio(rho, n));
}

void require_finite(const float* v, size_t n, const char* what) {
    // exponent all ones = inf or nan; branch-free so the scan vectorizes
    uint32_t bad = 0;
    for (size_t i = 0; i < n; ++i) {
        uint32_t b;
        std::memcpy(&b, v + i, 4);
        bad |= static_cast<uint32_t>((b & 0x7f800000u) == 0x7f800000u);
    }
    if (bad) fail(CSATTN_ERR_DATA, std::string(what) + " contains a non-finite value");
}

// The mixed-select work plan of the last step (run_step), reused while the
// grid and every problem's tile count stay the same.
struct MixedPlan {
    bool valid = false;
    uint64_t G = 0, log = 0;
    std::vector<uint32_t> tiles;
    std::vector<uint4> items;
    std::vector<uint32_t> cta;
    std::vector<uint2> pinfo, slot;
    void clear() {
        valid = false;
        G = 0;
        log = 0;
        tiles.clear();
        items.clear();
        cta.clear();
        pinfo.clear();
        slot.clear();
    }
};

struct SharedRows {
    DevMem k, v;
};

struct HeadState {
    bool has_cache = false;
    uint64_t n_cache = 0;
    double worst = 1.0;
};

}  // namespace

struct csattn_ctx_s {
    int device = 0;
    int refs = 1;  // the handle + one per live session
    cudaStream_t stream = nullptr;
    bool own = false;
    uint64_t launches = 0;
    DevMem probs, iprobs, stage;
    std::vector<csa::DecodeProblem> hprobs;
    std::vector<csa::InsertProblem> hiprobs;
    // Per-step descriptor ring: pinned host staging + device copy + an event
    // marking the step's kernels done, so the host never waits on the GPU
    // before reusing a slot that is still in flight.
    struct Slot {
        void* host = nullptr;
        DevMem dev;
        size_t cap = 0;
        cudaEvent_t done = nullptr;
        bool used = false;
    };
    static constexpr int kSlots = 4;
    Slot ring[kSlots];
    int next_slot = 0;
    // whole-run decode graphs (csattn_decode_run): 0 = off, 1 = sizing pass
    // (buffers grown, no stream work), 2 = capturing. Each captured step gets its
    // own descriptor copy in one arena (a ring slot would be overwritten before
    // the graph runs).
    int capture = 0;
    std::vector<size_t> cap_need, cap_off;
    size_t cap_step = 0, cap_bytes = 0;
    void* cap_host = nullptr;
    DevMem cap_dev, run_stage;
    // side stream for the attention work-list upload (runs beside select)
    cudaStream_t side = nullptr;
    cudaEvent_t side_ev = nullptr;
    // append + insert beside the attention (CSATTN_INSERT_OVERLAP=0: after it)
    cudaEvent_t ins_fork = nullptr, ins_join = nullptr;
    // select launched as a programmatic dependent of route (CSATTN_PDL=0: off)
    // (CSATTN_PDL=1/2/3: route's trigger at its start / once its lists are
    // known / at its exit; default: at its start when route leaves SMs idle
    // (nq <= SMs, c4: -127 us per 32 layers), else at its exit (c3: an early
    // start cost +9 us, the exit trigger saves 3 us))
    int pdl = std::getenv("CSATTN_PDL") ? std::atoi(std::getenv("CSATTN_PDL")) : 4;
    bool insert_overlap = !(std::getenv("CSATTN_INSERT_OVERLAP") && std::atoi(std::getenv("CSATTN_INSERT_OVERLAP")) == 0);
    ~csattn_ctx_s() {
        if (side) cudaStreamDestroy(side);
        if (side_ev) cudaEventDestroy(side_ev);
        if (ins_fork) cudaEventDestroy(ins_fork);
        if (ins_join) cudaEventDestroy(ins_join);
        for (Slot& s : ring) {
            if (s.host) cudaFreeHost(s.host);
            if (s.done) cudaEventDestroy(s.done);
        }
        if (cap_host) cudaFreeHost(cap_host);
        for (uint32_t* pg : bad_pages) cudaFreeHost(pg);
    }
    std::vector<unsigned char> hrep;
    // kernel timing (csattn_ctx_profile)
    bool profile = false;
    std::vector<std::array<cudaEvent_t, 4>> ev_steps;  // select | attend | insert
    DevMem part, counters;  // attention partials + per-problem merge counters
    DevMem plans;           // route.cu -> select.cu routing plans
    DevMem log_idx, log_sc; // select.cu candidate logs: log_rows x log_cap
    DevMem retry;           // select.cu retry list (speculative cut too high)
    DevMem ulog_idx, ulog_sc, umeta;  // split select: per part-unit logs + histograms
    // mixed (tail-split) select: piece logs + histograms, per-problem piece
    // counters (zero between steps: the finalising CTA resets its problem's)
    DevMem mlog_idx, mlog_sc, mumeta, pdone;
    MixedPlan mplan;
    std::vector<uint32_t> tiles_scratch;
    std::vector<uint64_t> Ks_scratch;  // run_step: per-problem K
    uint64_t pdone_n = 0;
    bool tail_split = !(std::getenv("CSATTN_TAIL_SPLIT") && std::atoi(std::getenv("CSATTN_TAIL_SPLIT")) == 0);
    // small batches through the mixed pieces too (CSATTN_SMALL_MIXED=0: part
    // units + select_merge_kernel)
    bool small_mixed = !(std::getenv("CSATTN_SMALL_MIXED") && std::atoi(std::getenv("CSATTN_SMALL_MIXED")) == 0);
    // mixed select: half the CTAs take their pieces before their whole
    // problems (CSATTN_ORDER_SWAP=0: all whole problems first)
    bool order_swap = !(std::getenv("CSATTN_ORDER_SWAP") && std::atoi(std::getenv("CSATTN_ORDER_SWAP")) == 0);
    // GQA warp-per-head attention, opt-in (CSATTN_ATT_GQA=1): measured slower
    // at c3 (attend 252 -> 275 us: 4x the partials, little L1 reuse)
    bool att_gqa = std::getenv("CSATTN_ATT_GQA") && std::atoi(std::getenv("CSATTN_ATT_GQA")) == 1;
    // sharded steps (csattn_shard_step): descriptors + scratch kept across phases
    DevMem sh_desc, sh_pstate, sh_bitmap, sh_kdev, sh_ulog_idx, sh_ulog_sc, sh_umeta, sh_chunks;
    std::vector<csa::DecodeProblem> sh_hprobs;
    std::vector<csa::InsertProblem> sh_hiprobs;
    std::vector<uint32_t> sh_chunk_host;
    std::vector<uint64_t> sh_Ks;
    uint64_t sh_nq = 0, sh_ns = 0, sh_ucap = 0, sh_bm_words = 0, sh_nchunks = 0;
    uint32_t sh_split = 1;
    double sh_spec = 0.0;
    bool sh_scanned = false;
    bool no_split = std::getenv("CSATTN_NO_SPLIT") != nullptr;
    bool shard_split = std::getenv("CSATTN_SHARD_SPLIT") != nullptr;
    // union attend (attend_union.cu) for problems sharing a prefill: opt-in
    // with CSATTN_UNION=1 (read every step); CSATTN_UNION_MIN sets the minimum
    // number of problems on one prefill for it to engage (default 16)
    uint64_t union_min = std::getenv("CSATTN_UNION_MIN") ? std::strtoull(std::getenv("CSATTN_UNION_MIN"), nullptr, 10) : 16;
    DevMem un_row, un_mask, un_count, un_parts, un_tails;
    DevMem dense;  // dense oracle scratch (dense.cu)
    // KV placement of sessions created from now on (csattn_ctx_set_kv_placement)
    bool kv_host = false;
    // table builds through the tcgen05 screen, and those rebuilt by the fp64 path
    uint64_t build_tc = 0, build_fallback = 0;
    bool host_prof = std::getenv("CSATTN_HOST_PROF") != nullptr;
    double host_sum[4] = {0, 0, 0, 0}, host_sub[4] = {0, 0, 0, 0}, host_sub2[3] = {0, 0, 0};
    uint64_t host_n = 0;
    // union-kernel timeline (CSATTN_UNION_PROF=1; diagnostics only): per CTA
    // [16 items][4 stamps] + [16] tile counts, summarised at teardown
    bool union_prof = std::getenv("CSATTN_UNION_PROF") != nullptr;
    DevMem un_prof;
    double un_sum[4] = {0, 0, 0, 0};
    uint64_t un_items = 0, un_tiles = 0, un_launches = 0;
    uint64_t log_cap = 0, log_rows = 0;
    int num_sms = 148;
    // SMs the decode-step select grid assumes (CSATTN_SELECT_SMS: a test hook
    // that shrinks the grid so small batches exercise the round/tail logic)
    int sel_sms = std::getenv("CSATTN_SELECT_SMS") ? std::max(1, std::atoi(std::getenv("CSATTN_SELECT_SMS"))) : 0;
    // select speculation margin (CSATTN_SPEC_KEEP; 0 disables, > 1 forces the
    // retry pass — used by the tests to exercise it). c3: 0.9 logs 10.3K
    // candidates per problem, 0.95 8.6K with 0 of 18,432 problems retried,
    // 0.97 8.1K with 2 retried (each retry is a second pass for its problem)
    double spec_keep = std::getenv("CSATTN_SPEC_KEEP") ? std::atof(std::getenv("CSATTN_SPEC_KEEP")) : 0.95;
    // one-cluster-per-problem fused step for small batches (fused.cu):
    // CSATTN_FUSED=0 never, 1 whenever it fits, default: when the batch's
    // clusters fit the GPU a couple of times over (the latency-bound regime)
    int fused_mode = std::getenv("CSATTN_FUSED") ? std::atoi(std::getenv("CSATTN_FUSED")) : 2;
    uint64_t counters_n = 0;
    // select-kernel phase timestamps (env CSATTN_PHASE_PROF=1; diagnostics only)
    bool phase_prof = std::getenv("CSATTN_PHASE_PROF") != nullptr;
    DevMem phase;
    double phase_sum[6] = {0, 0, 0, 0, 0, 0};
    double phase_dbg[3] = {0, 0, 0};
    uint64_t phase_retry = 0, phase_probs = 0;
    uint64_t phase_n = 0;
    // non-finite append flags (insert.cu sets a session's flag instead of
    // appending a non-finite row): pinned host words the kernel writes
    // directly, one per session, handed out from 4096-word pages
    std::vector<uint32_t*> bad_pages;
    std::vector<uint32_t*> bad_free;
    uint32_t* take_bad_flag() {
        if (bad_free.empty()) {
            void* pg = nullptr;
            ck(cudaMallocHost(&pg, 4096 * sizeof(uint32_t)), "cudaMallocHost");
            bad_pages.push_back(static_cast<uint32_t*>(pg));
            for (int i = 4095; i >= 0; --i) bad_free.push_back(static_cast<uint32_t*>(pg) + i);
        }
        uint32_t* f = bad_free.back();
        bad_free.pop_back();
        *f = 0;
        return f;
    }
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t take_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        return e;
    }
};

struct csattn_session_s {
    csattn_ctx ctx = nullptr;
    csa::SessionDev h{};
    DevMem dev;
    std::shared_ptr<SharedRows> pre;
    DevMem ktail, vtail, cent, ent, n_used, live, blk_off, low, low_cnt, refill, tmm;
    DevMem cache, cbounds, sel, drep, irep, live_g;
    uint64_t group = 1, N = 0, step = 0, max_steps = 0;
    uint64_t index_prefill = 0;  // CsIndex::prefill_len (0: = h.P); differs after loading an image with appended keys
    double alpha = 0.0;
    int32_t score_bits = 32;
    csattn_retrieval_config rc{};
    std::vector<double> weights;
    std::vector<HeadState> hs;
    std::vector<uint64_t> widths;
    // non-finite appended row seen by insert.cu (pinned word from the ctx pool);
    // `poisoned`: such a row was found only after later steps were queued
    // (CSATTN_NO_SYNC), so the host's context length ran ahead of the store
    uint32_t* bad = nullptr;
    bool poisoned = false;

    ~csattn_session_s();
    uint64_t T() const { return static_cast<uint64_t>(h.m) * h.C; }
    size_t device_bytes() const {
        return ktail.n + vtail.n + cent.n + ent.n + n_used.n + live.n + blk_off.n + low.n +
               low_cnt.n + refill.n + tmm.n + cache.n + cbounds.n + sel.n + drep.n + irep.n +
               (pre ? pre->k.n + pre->v.n : 0);
    }
};

namespace {

// SubspaceLayout (core.cpp:35-41 constructor checks)
void validate_layout(const uint64_t* widths, uint64_t m, uint64_t d) {
    if (m == 0) fail(CSATTN_ERR_PARAMETER, "subspace layout needs m >= 1");
    uint64_t sum = 0;
    for (uint64_t b = 0; b < m; ++b) {
        if (widths[b] == 0)
            fail(CSATTN_ERR_PARAMETER,
                 "subspace width must be >= 1 (subspace " + std::to_string(b) + ")");
        sum += widths[b];
    }
    if (sum != d) fail(CSATTN_ERR_DIMENSION, "layout dimension does not match KV dimension");
    if (m > static_cast<uint64_t>(csa::MAXM))
        fail(CSATTN_ERR_PARAMETER, "B200 path supports m <= " + std::to_string(csa::MAXM));
    for (uint64_t b = 0; b < m; ++b)
        if (widths[b] > static_cast<uint64_t>(csa::WMAX))
            fail(CSATTN_ERR_PARAMETER,
                 "B200 path supports subspace widths <= " + std::to_string(csa::WMAX));
    if (d > static_cast<uint64_t>(csa::DMAX))
        fail(CSATTN_ERR_PARAMETER, "B200 path supports d <= " + std::to_string(csa::DMAX));
}

// validate_retrieval_config (session.cpp:10-21)
void validate_retrieval(const csattn_retrieval_config* cfg, uint64_t m) {
    if (!(cfg->keep_ratio > 0.0 && cfg->keep_ratio <= 1.0))
        fail(CSATTN_ERR_PARAMETER, "keep ratio must lie in (0, 1]");
    if (cfg->search_period == 0) fail(CSATTN_ERR_PARAMETER, "search period must be >= 1");
    if (cfg->backoff_tau == 0) fail(CSATTN_ERR_PARAMETER, "backoff tau must be >= 1");
    if (cfg->weights && cfg->n_weights && cfg->n_weights != m)
        fail(CSATTN_ERR_DIMENSION, "need one weight per subspace");
    if (cfg->weights)
        for (uint64_t b = 0; b < cfg->n_weights; ++b)
            if (!(cfg->weights[b] > 0.0))
                fail(CSATTN_ERR_PARAMETER, "subspace weights must be positive");
    if (cfg->backoff_tau > static_cast<uint64_t>(csa::MAXTAU))
        fail(CSATTN_ERR_PARAMETER, "B200 path supports backoff tau <= " +
                                       std::to_string(csa::MAXTAU));
    if (m * std::min<uint64_t>(cfg->backoff_tau, 1u << 20) > static_cast<uint64_t>(csa::MAXL))
        fail(CSATTN_ERR_PARAMETER, "B200 path supports m * tau <= " + std::to_string(csa::MAXL));
}

// validate_index_config (index.cpp:95-103)
void validate_index(const csattn_index_config* c) {
    if (c->list_capacity == 0 && !(c->alpha > 0.0 && c->alpha <= 1.0))
        fail(CSATTN_ERR_PARAMETER, "alpha must lie in (0, 1]");
    if (c->score_bits != 16 && c->score_bits != 32)
        fail(CSATTN_ERR_PARAMETER, "score width must be 16 or 32 bits");
    if (c->centroids == 0) fail(CSATTN_ERR_PARAMETER, "centroid count must be >= 1");
}

void set_retrieval(csattn_session_s* s, const csattn_retrieval_config* rc) {
    s->rc = *rc;
    s->weights.assign(s->h.m, 1.0);
    if (rc->weights && rc->n_weights)
        for (uint32_t b = 0; b < s->h.m; ++b) s->weights[b] = rc->weights[b];
    s->rc.weights = nullptr;
    s->rc.n_weights = 0;
    for (uint32_t b = 0; b < s->h.m; ++b) s->h.weights[b] = s->weights[b];
    s->h.tau = static_cast<uint32_t>(rc->backoff_tau);
    s->h.threshold = rc->backoff_threshold;
    s->h.window = static_cast<uint32_t>(std::min<uint64_t>(rc->recent_window, 0xffffffffu));
    s->h.passthrough = rc->recent_passthrough ? 1u : 0u;
}

void push_dev(csattn_session_s* s) {
    ck(cudaMemcpyAsync(s->dev.p, &s->h, sizeof(csa::SessionDev), cudaMemcpyHostToDevice,
                       s->ctx->stream),
       "upload session");
}

// Allocate everything except prefill rows / centroid contents.
std::unique_ptr<csattn_session_s> new_session(csattn_ctx ctx, uint64_t d, const uint64_t* widths,
                                              uint64_t m, uint64_t c, uint64_t L, uint64_t p,
                                              uint64_t group, uint64_t max_steps,
                                              const csattn_retrieval_config* rc) {
    if (group == 0) fail(CSATTN_ERR_PARAMETER, "group must be >= 1");
    if (m * c > static_cast<uint64_t>(csa::MAX_TABLES))
        fail(CSATTN_ERR_PARAMETER,
             "B200 path supports m * C <= " + std::to_string(csa::MAX_TABLES));
    if (p + max_steps >= static_cast<uint64_t>(csa::MAX_CONTEXT))
        fail(CSATTN_ERR_PARAMETER, "context exceeds 2^31 positions");
    if (L > 0x7fffffffull) fail(CSATTN_ERR_PARAMETER, "list capacity too large");
    auto s = std::make_unique<csattn_session_s>();
    s->ctx = ctx;
    ctx->refs += 1;
    s->group = group;
    s->max_steps = max_steps;
    s->N = p;
    s->widths.assign(widths, widths + m);
    csa::SessionDev& h = s->h;
    h.d = static_cast<uint32_t>(d);
    h.m = static_cast<uint32_t>(m);
    h.C = static_cast<uint32_t>(c);
    h.L = static_cast<uint32_t>(L);
    uint64_t keep = std::min<uint64_t>(L, p);
    uint64_t cap2 = std::max<uint64_t>(L, keep) + csa::LOW_Q;
    cap2 += cap2 & 1;  // even: 16-byte aligned table rows
    h.cap2 = static_cast<uint32_t>(cap2);
    h.P = static_cast<uint32_t>(p);
    h.max_ctx = static_cast<uint32_t>(p + max_steps);
    h.nb_stride = (h.max_ctx >> csa::KEY_BLOCK_SHIFT) + 2;
    uint32_t off = 0;
    for (uint64_t b = 0; b < m; ++b) {
        h.widths[b] = static_cast<uint32_t>(widths[b]);
        h.offs[b] = off;
        off += static_cast<uint32_t>(widths[b]);
    }
    set_retrieval(s.get(), rc);
    const uint64_t T = m * c;
    s->ktail.alloc_on(s->ctx->kv_host, std::max<uint64_t>(max_steps, 1) * d * sizeof(float));
    s->vtail.alloc_on(s->ctx->kv_host, std::max<uint64_t>(max_steps, 1) * d * sizeof(float));
    s->cent.alloc(c * d * sizeof(float));
    s->ent.alloc(T * cap2 * sizeof(uint2));
    s->n_used.alloc(T * 4);
    s->live.alloc(T * 4);
    s->blk_off.alloc(T * h.nb_stride * 4);
    s->low.alloc(T * csa::LOW_Q * sizeof(csa::LowEnt));
    s->low_cnt.alloc(T * 4);
    s->refill.alloc(T * 4);
    s->tmm.alloc(T * sizeof(float2));
    s->sel.alloc(group * (p + max_steps) * 4);
    if (rc->search_period > 1) s->cache.alloc(group * (p + max_steps) * sizeof(double));
    s->cbounds.alloc(group * 4 * sizeof(double));
    ck(cudaMemsetAsync(s->cbounds.p, 0, group * 4 * sizeof(double), ctx->stream), "memset");
    s->drep.alloc(group * sizeof(csa::DecodeReport));
    s->irep.alloc(4 + ((T + 15) & ~15ull));
    s->dev.alloc(sizeof(csa::SessionDev));
    h.ktail = s->ktail.as<float>();
    h.vtail = s->vtail.as<float>();
    h.cent = s->cent.as<float>();
    h.ent = s->ent.as<uint2>();
    h.n_used = s->n_used.as<uint32_t>();
    h.live = s->live.as<uint32_t>();
    h.blk_off = s->blk_off.as<uint32_t>();
    h.low = s->low.as<csa::LowEnt>();
    h.low_cnt = s->low_cnt.as<uint32_t>();
    h.refill = s->refill.as<uint32_t>();
    h.tmm = s->tmm.as<float2>();
    h.key_lo = 0;
    h.key_hi = h.P;
    h.owner = 1;
    h.sharded = 0;
    h.live_g = h.live;  // unsharded: the global count is the local one
    s->hs.assign(group, HeadState{});
    s->bad = ctx->take_bad_flag();
    return s;
}

void upload(csattn_ctx ctx, void* dst, const void* src, size_t bytes, bool host) {
    (void)host;  // UVA: the runtime resolves device, mapped-host and pageable pointers
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream), "copy in");
}

void attach_rows(csattn_session_s* s, const float* keys, const float* values, bool host) {
    s->pre = std::make_shared<SharedRows>();
    const size_t bytes = static_cast<size_t>(s->h.P) * s->h.d * sizeof(float);
    s->pre->k.alloc_on(s->ctx->kv_host, bytes);
    s->pre->v.alloc_on(s->ctx->kv_host, bytes);
    upload(s->ctx, s->pre->k.p, keys, bytes, host);
    upload(s->ctx, s->pre->v.p, values, bytes, host);
    s->h.kpre = s->pre->k.as<float>();
    s->h.vpre = s->pre->v.as<float>();
}

// assemble_index on the device (index.cpp:107-141)
void build_tables(csattn_session_s* s) {
    push_dev(s);
    csattn_ctx ctx = s->ctx;
    // the tcgen05 screen + exact fp64 rescore (build_tc.cu); CSATTN_BUILD=fp64
    // forces the plain fp64 kernels. Mapped-host KV rows stay on the fp64 path.
    const char* mode = std::getenv("CSATTN_BUILD");
    const bool force_fp64 = mode && std::strcmp(mode, "fp64") == 0;
    if (!force_fp64 && !s->pre->k.host && csa::build_tc_eligible(s->h)) {
        const char* qm = std::getenv("CSATTN_BUILD_QMARGIN");  // test hook
        const float qmargin = qm ? static_cast<float>(std::atof(qm)) : 0.0f;
        DevMem scratch, fail;
        scratch.alloc(csa::build_tc_scratch_bytes(s->h, nullptr));
        fail.alloc(4);
        ck(csa::launch_build_tc(s->dev.as<csa::SessionDev>(), s->h, scratch.p, qmargin, fail.as<uint32_t>(),
                                ctx->stream),
           "build_tc launch");
        ctx->launches += 4;
        uint32_t nfail = 0;
        ck(cudaMemcpyAsync(&nfail, fail.p, 4, cudaMemcpyDeviceToHost, ctx->stream), "build_tc flag");
        ck(cudaStreamSynchronize(ctx->stream), "build_tc");
        ctx->build_tc += 1;
        if (nfail == 0) return;
        ctx->build_fallback += 1;  // a table's screen was inconclusive: rebuild exactly
    }
    DevMem scores;
    scores.alloc(s->T() * s->h.P * sizeof(float));
    ck(csa::launch_build_scores(s->dev.as<csa::SessionDev>(), s->h, scores.as<float>(),
                                s->ctx->stream),
       "build_scores launch");
    ck(csa::launch_build_lists(s->dev.as<csa::SessionDev>(), s->h, scores.as<float>(),
                               s->ctx->stream),
       "build_lists launch");
    s->ctx->launches += 2;
    ck(cudaStreamSynchronize(s->ctx->stream), "build");
}

uint64_t list_capacity_of(const csattn_index_config* icfg, uint64_t p, double* alpha) {
    const uint64_t L = icfg->list_capacity ? icfg->list_capacity : ceil_ratio(icfg->alpha, p);
    if (L == 0) fail(CSATTN_ERR_PARAMETER, "list capacity came out as zero");
    *alpha = icfg->list_capacity ? static_cast<double>(L) / static_cast<double>(p) : icfg->alpha;
    return L;
}

void check_rows(const float* keys, const float* values, uint64_t p, uint64_t d, bool host) {
    if (d == 0) fail(CSATTN_ERR_PARAMETER, "head dimension must be >= 1");
    if (host) {
        require_finite(keys, p * d, "prefill keys");
        require_finite(values, p * d, "prefill values");
    }
}

// A session whose insert kernel refused a non-finite row (KvStore::append,
// core.cpp:71-79) after the host had queued later steps on it: its context
// length ran ahead of its store, so it only reports the error from then on.
void check_not_poisoned(csattn_session s) {
    if (!s->poisoned && s->bad && *reinterpret_cast<volatile uint32_t*>(s->bad)) s->poisoned = true;
    if (s->poisoned)
        fail(CSATTN_ERR_DATA,
             "appended row contains a non-finite value (found after later steps were queued; "
             "the session is unusable)");
}

// After a synchronised step: a session whose appended row was non-finite kept
// its KV rows and tables (the kernel skipped the append and the insert), so its
// context length goes back; the search state advanced, as decode_search's does
// before KvStore::append throws (session.cpp:57-81). Raises DataError.
void check_appended(const csattn_session* ss, uint64_t ns) {
    uint32_t first = 0;
    for (uint64_t i = 0; i < ns; ++i) {
        volatile uint32_t* f = ss[i]->bad;
        if (f && *f) {
            if (!first) first = *f;
            *f = 0;
            ss[i]->N -= 1;
        }
    }
    if (first)
        fail(CSATTN_ERR_DATA, first == 1 ? "appended key contains a non-finite value"
                                         : "appended value contains a non-finite value");
}

// one session twice in a batch would append and insert twice at one N
void check_distinct(const csattn_session* ss, uint64_t ns) {
    static thread_local std::vector<csattn_session> u;
    u.assign(ss, ss + ns);
    std::sort(u.begin(), u.end());
    if (std::adjacent_find(u.begin(), u.end()) != u.end())
        fail(CSATTN_ERR_PARAMETER, "a session appears twice in one decode batch");
}

struct Outs {
    float* out;
    uint32_t* sel;
    float* weights;
};

// One decode step for a set of sessions (decode_step, session.cpp:46-99).
void run_step(csattn_ctx ctx, uint64_t ns, const csattn_session* ss, const float* q,
              const float* keys, const float* values, float* out, uint32_t* selected,
              float* weights, uint64_t sel_stride, csattn_step_report* reports,
              const uint64_t* k_override, uint32_t flags) {
    const auto ht0 = std::chrono::steady_clock::now();
    const bool host = flags & CSATTN_HOST_BUFFERS;
    if (ns == 0) fail(CSATTN_ERR_PARAMETER, "no sessions");
    const uint32_t d = ss[0]->h.d;
    uint64_t nq = 0, maxN = 0, maxK = 0;
    std::vector<uint64_t>& Ks = ctx->Ks_scratch;
    Ks.clear();
    check_distinct(ss, ns);
    for (uint64_t i = 0; i < ns; ++i) {
        csattn_session s = ss[i];
        if (s->ctx != ctx) fail(CSATTN_ERR_PARAMETER, "sessions belong to another context");
        if (!ctx->capture) check_not_poisoned(s);
        if (s->h.d != d) fail(CSATTN_ERR_DIMENSION, "sessions differ in head dimension");
        if (s->step >= s->max_steps)
            fail(CSATTN_ERR_CAPACITY, "session is full: max_decode_steps = " +
                                          std::to_string(s->max_steps));
        const uint64_t Ks_ = keep_count(s->rc.keep_ratio, s->N);  // the session's heads share N
        for (uint64_t h = 0; h < s->group; ++h) {
            const uint64_t ko = k_override ? k_override[nq + h] : 0;
            const uint64_t K = ko ? std::min<uint64_t>(ko, s->N) : Ks_;
            Ks.push_back(K);
            maxK = std::max(maxK, K);
        }
        nq += s->group;
        maxN = std::max<uint64_t>(maxN, s->N);
    }
    if ((selected || weights) && sel_stride < maxK)
        fail(CSATTN_ERR_PARAMETER, "selected/weights stride " + std::to_string(sel_stride) +
                                       " is below K = " + std::to_string(maxK));
    const auto hta = std::chrono::steady_clock::now();
    const auto htb = std::chrono::steady_clock::now();
    if (maxN > csa::SELECT_MAX_CONTEXT)
        fail(CSATTN_ERR_CAPACITY, "context of " + std::to_string(maxN) +
                                      " keys exceeds one GPU's decode search (" +
                                      std::to_string(csa::SELECT_MAX_CONTEXT) +
                                      "); shard the sequence");

    // device views of inputs / outputs
    const float *dq = q, *dk = keys, *dv = values;
    float *dout = out, *dw = weights;
    uint32_t* dsel = selected;
    size_t o_q = 0, o_k = 0, o_v = 0, o_out = 0, o_sel = 0, o_w = 0, total = 0;
    auto carve = [&](size_t bytes) {
        const size_t at = total;
        total += (bytes + 255) & ~size_t(255);
        return at;
    };
    if (host) {
        o_q = carve(nq * d * 4);
        o_k = carve(ns * d * 4);
        o_v = carve(ns * d * 4);
        o_out = carve(nq * d * 4);
        if (selected) o_sel = carve(nq * sel_stride * 4);
        if (weights) o_w = carve(nq * sel_stride * 4);
        ctx->stage.ensure(total);
        char* base = ctx->stage.as<char>();
        // copies first (scratch staging: harmless if the scan below refuses),
        // so the DMA overlaps the scan
        // host-buffer calls: the inputs are host memory by contract (an
        // explicit direction skips the runtime's pointer lookup)
        ck(cudaMemcpyAsync(base + o_q, q, nq * d * 4, cudaMemcpyHostToDevice, ctx->stream), "copy in");
        ck(cudaMemcpyAsync(base + o_k, keys, ns * d * 4, cudaMemcpyHostToDevice, ctx->stream), "copy in");
        ck(cudaMemcpyAsync(base + o_v, values, ns * d * 4, cudaMemcpyHostToDevice, ctx->stream), "copy in");
        // a non-finite appended row is refused on the device (insert.cu: the
        // append + insert of that session are skipped, its flag is read after
        // the synchronised step and raises DataError with the search state
        // advanced, as decode_search runs before KvStore::append throws,
        // session.cpp:57-81) -- no host scan of the rows on the critical path
        dq = reinterpret_cast<float*>(base + o_q);
        dk = reinterpret_cast<float*>(base + o_k);
        dv = reinterpret_cast<float*>(base + o_v);
        dout = out ? reinterpret_cast<float*>(base + o_out) : nullptr;
        dsel = selected ? reinterpret_cast<uint32_t*>(base + o_sel) : nullptr;
        dw = weights ? reinterpret_cast<float*>(base + o_w) : nullptr;
    }
    const auto htc = std::chrono::steady_clock::now();
    ctx->hprobs.resize(nq);
    if (ctx->phase_prof) {
        ctx->phase.ensure(nq * 8 * sizeof(unsigned long long));
        ck(cudaMemsetAsync(ctx->phase.p, 0, nq * 8 * 8, ctx->stream), "memset");
    }
    ctx->hiprobs.resize(ns);
    uint64_t qi = 0;
    std::vector<uint32_t> searched(nq);
    std::vector<const float*> pre_of(nq);  // each problem's prefill rows (attend chunk order)
    for (uint64_t i = 0; i < ns; ++i) {
        csattn_session s = ss[i];
        const uint64_t n = s->N;
        for (uint64_t h = 0; h < s->group; ++h, ++qi) {
            pre_of[qi] = s->h.kpre;
            HeadState& hs = s->hs[h];
            csa::DecodeProblem& P = ctx->hprobs[qi];
            const bool srch = !hs.has_cache || (s->step % s->rc.search_period) == 0;
            searched[qi] = srch;
            P.s = s->dev.as<csa::SessionDev>();
            P.q = dq + qi * d;
            P.out = dout ? dout + qi * d : nullptr;
            P.weights = dw ? dw + qi * sel_stride : nullptr;
            P.sel = dsel ? dsel + qi * sel_stride : s->sel.as<uint32_t>() + h * s->h.max_ctx;
            P.cache = s->cache.p ? s->cache.as<double>() + h * s->h.max_ctx : nullptr;
            P.rep = reinterpret_cast<uint32_t*>(s->drep.as<csa::DecodeReport>() + h);
            P.N = static_cast<uint32_t>(n);
            P.K = static_cast<uint32_t>(Ks[qi]);
            P.n_cache = static_cast<uint32_t>(hs.n_cache);
            P.mode = (srch ? csa::MODE_SEARCH : 0u) |
                     ((srch && P.cache) ? csa::MODE_STORE_CACHE : 0u) |
                     (dw ? csa::MODE_WEIGHTS : 0u);
            P.cbounds = s->cbounds.as<double>() + h * 4;
            P.prof = ctx->phase_prof ? ctx->phase.as<unsigned long long>() + qi * 8 : nullptr;
        }
        csa::InsertProblem& I = ctx->hiprobs[i];
        I.s = s->dev.as<csa::SessionDev>();
        I.key = dk + i * d;
        I.value = dv + i * d;
        I.rep = s->irep.as<uint32_t>();
        I.N = static_cast<uint32_t>(n);
        I.bad = s->bad;
        I.pad = 0;
    }
    const auto ht1 = std::chrono::steady_clock::now();
    // stage both descriptor arrays through one pinned ring slot (a graph
    // capture stages through its own arena instead; see run_graph)
    const int cap = ctx->capture;
    const bool live = cap != 1;  // sizing pass: no stream work
    csattn_ctx_s::Slot* slot = nullptr;
    if (!cap) {
        slot = &ctx->ring[ctx->next_slot];
        ctx->next_slot = (ctx->next_slot + 1) % csattn_ctx_s::kSlots;
        if (slot->used) ck(cudaEventSynchronize(slot->done), "descriptor slot");
    }
    // union attend groups: problems on one prefill, in first-appearance order,
    // cut into groups of <= UN_GROUP (attend_union.cu)
    std::vector<uint32_t> ugP, ugmem, umem, umgrp;
    std::vector<char> in_union(nq, 0);
    uint32_t u_maxP = 0;
    const char* uenv = std::getenv("CSATTN_UNION");
    if (!cap && uenv && uenv[0] == '1' && !dw && d == 128) {
        std::vector<std::pair<const float*, std::vector<uint32_t>>> by_pre;
        std::vector<uint32_t> prob_sess(nq);
        qi = 0;
        for (uint64_t i = 0; i < ns; ++i)
            for (uint64_t h = 0; h < ss[i]->group; ++h, ++qi) {
                prob_sess[qi] = static_cast<uint32_t>(i);
                const float* key = ss[i]->h.kpre;
                auto it = std::find_if(by_pre.begin(), by_pre.end(),
                                       [&](const auto& e) { return e.first == key; });
                if (it == by_pre.end()) {
                    by_pre.emplace_back(key, std::vector<uint32_t>{});
                    it = by_pre.end() - 1;
                }
                it->second.push_back(static_cast<uint32_t>(qi));
            }
        for (auto& [key, list] : by_pre) {
            if (list.size() < std::max<uint64_t>(ctx->union_min, 1)) continue;
            const uint64_t ng = (list.size() + csa::UN_GROUP - 1) / csa::UN_GROUP;
            const uint64_t per = (list.size() + ng - 1) / ng;
            for (uint64_t g0 = 0; g0 < list.size(); g0 += per) {
                const uint32_t g = static_cast<uint32_t>(ugP.size());
                const uint32_t Pg = static_cast<uint32_t>(ss[prob_sess[list[g0]]]->h.P);
                ugP.push_back(Pg);
                u_maxP = std::max(u_maxP, Pg);
                ugmem.resize(ugmem.size() + csa::UN_GROUP, 0xffffffffu);
                for (uint64_t b = 0; g0 + b < list.size() && b < per; ++b) {
                    const uint32_t p = list[g0 + b];
                    ugmem[g * csa::UN_GROUP + b] = static_cast<uint32_t>(umem.size());
                    umem.push_back(p);
                    umgrp.push_back(g);
                    in_union[p] = 1;
                }
            }
        }
    }
    const uint64_t ngroups = ugP.size(), nmem = umem.size();
    // the fused cluster step: every problem's search + attention in one
    // cluster; the append + insert stays a separate launch
    int fz_cl = 0, fz_nr = 0;
    // auto: 8-CTA clusters that all fit the GPU at once (c2: 32 problems at
    // 32K keys, search + attention 76 -> ~50 us); 16-CTA clusters (up to 256K
    // keys) measured slower than the multi-kernel path at c4 and are only
    // taken with CSATTN_FUSED=1
    const bool fused = ctx->fused_mode != 0 && !dw && ngroups == 0 &&
                       csa::fused_fits(static_cast<uint32_t>(maxN), d, fz_cl, fz_nr) &&
                       (ctx->fused_mode == 1 ||
                        (fz_cl == 8 && nq * 8ull <= 2ull * static_cast<uint64_t>(ctx->num_sms)));
    const uint32_t u_nrange = (u_maxP + csa::UN_RANGE - 1) / csa::UN_RANGE;
    if (ngroups) {
        ctx->un_row.ensure(ngroups * u_nrange * csa::UN_RANGE * 2);
        ctx->un_mask.ensure(ngroups * u_nrange * csa::UN_RANGE * 8);
        ctx->un_count.ensure(ngroups * u_nrange * 4);
        ctx->un_parts.ensure(nmem * u_nrange * csa::UN_PART_WORDS * 4);
        ctx->un_tails.ensure(nmem * csa::UN_PART_WORDS * 4);
    }
    const auto htd = std::chrono::steady_clock::now();
    // attention work list: ceil(K / ATT_ROWS) chunk-CTAs per problem
    // (cbase = first chunk of each problem; the per-chunk problem ids are written
    // straight into the pinned slot below)
    std::vector<uint32_t> cbase(nq + 1);
    uint64_t n256 = 0;
    for (uint64_t i = 0; i < nq; ++i)
        if (!in_union[i]) n256 += (Ks[i] + csa::ATT_ROWS - 1) / csa::ATT_ROWS;
    uint32_t arows = csa::attend_rows(n256);  // c3: 512 (attend 262 -> 251 us)
    if (const char* ar = std::getenv("CSATTN_ATT_ROWS")) {  // tests: force 128 / 256 / 512
        const int v = std::atoi(ar);
        arows = v == 512 ? csa::ATT_ROWS_BIG : (v == 128 ? csa::ATT_ROWS_SMALL : csa::ATT_ROWS);
    }
    // GQA sessions of 4 query heads (d = 128, no union groups): one CTA per
    // (session, chunk), warp h = head h over arows / 4 rows (attend.cu WARP:
    // the heads' shared rows come from L1); cbase then counts per-warp
    // partials, and the CTA entries are one per (session, chunk)
    bool att_warp = ctx->att_gqa && d == 128 && ngroups == 0 && arows >= 128;
    for (uint64_t i = 0; i < ns && att_warp; ++i) att_warp = ss[i]->group == 4;
    const uint32_t prow = att_warp ? arows / 4 : arows;  // rows per partial
    uint64_t nchunks = 0;  // partials
    for (uint64_t i = 0; i < nq; ++i) {
        cbase[i] = static_cast<uint32_t>(nchunks);
        if (!in_union[i]) nchunks += (Ks[i] + prow - 1) / prow;
    }
    cbase[nq] = static_cast<uint32_t>(nchunks);
    uint64_t ncta = nchunks;  // attention CTAs
    if (att_warp) {
        ncta = 0;
        for (uint64_t i = 0; i < nq; i += 4) ncta = ncta + cbase[i + 1] - cbase[i];
    }
    if (nq > ctx->counters_n) {
        ctx->counters.alloc(nq * 4);
        ck(cudaMemsetAsync(ctx->counters.p, 0, nq * 4, ctx->stream), "memset");
        ctx->counters_n = nq;
    }
    ctx->part.ensure(nchunks * (d + 2) * sizeof(float));
    // Mixed select plan: problems beyond whole rounds of the select grid are
    // cut into contiguous tile pieces spread over the CTAs (one piece range
    // per CTA), instead of a second, partly idle round. The
    // plan depends only on the grid and the problems' tile counts, which
    // change once per 4096 appended keys: it is rebuilt only then.
    MixedPlan& mp = ctx->mplan;
    {
        // small batches (fewer problems than CTA slots): every problem is
        // cut into pieces over all slots, finalised in-kernel by its last
        // piece (instead of part units + select_merge_kernel)
        const int sms = ctx->sel_sms ? ctx->sel_sms : ctx->num_sms;
        const uint64_t slots = static_cast<uint64_t>(csa::select_ctas_per_sm()) * sms;
        const bool small = nq < slots;
        const uint64_t G = small ? slots : csa::select_grid(static_cast<uint32_t>(nq), sms);
        const uint64_t tile = csa::select_tile_keys();
        const bool want = !fused && ctx->tail_split &&
                          ((nq > G && nq % G != 0) || (small && ctx->small_mixed && !ctx->no_split));
        ctx->tiles_scratch.resize(nq);
        for (uint64_t i = 0; i < nq; ++i)
            ctx->tiles_scratch[i] = static_cast<uint32_t>((ctx->hprobs[i].N + tile - 1) / tile);
        if (!want) {
            mp.clear();
        } else if (!(mp.valid && mp.G == G && mp.tiles == ctx->tiles_scratch)) {
            mp.clear();
            mp.valid = true;
            mp.G = G;
            mp.tiles = ctx->tiles_scratch;
            const std::vector<uint32_t>& tl = mp.tiles;
            const uint64_t W = nq / G * G;
            std::vector<uint64_t> tpre(1, 0);  // tail tile prefix
            uint64_t tmax = 1;
            for (uint64_t i = W; i < nq; ++i) {
                tpre.push_back(tpre.back() + tl[i]);
                tmax = std::max<uint64_t>(tmax, tl[i]);
            }
            const uint64_t TT = tpre.back();
            // piece ranges of >= 1 tile and <= MAXPART pieces per problem
            const uint64_t Gp = std::max<uint64_t>(1, std::min<uint64_t>({G, TT, 15 * TT / tmax}));
            mp.cta.assign(G + 1, 0);
            mp.pinfo.assign(nq, make_uint2(0, 0));
            bool ok = true;
            uint64_t q = 0;  // tail problem cursor (relative to W)
            for (uint64_t c = 0; c < G; ++c) {
                mp.cta[c] = static_cast<uint32_t>(mp.items.size());
                // the two CTAs of an SM (c, c + G/2) take their whole problems
                // and their pieces in opposite orders, so one streams while
                // the other runs a final selection
                const bool pieces_first = ctx->order_swap && c >= G / 2;
                auto whole = [&]() {
                    for (uint64_t pw = c; pw < W; pw += G)
                        mp.items.push_back(make_uint4(static_cast<uint32_t>(pw), 0u, tl[pw], csa::NO_SLOT));
                };
                if (!pieces_first) whole();
                if (c >= Gp) {
                    if (pieces_first) whole();
                    continue;
                }
                uint64_t a = c * TT / Gp;
                const uint64_t b = (c + 1) * TT / Gp;
                while (a < b) {
                    while (tpre[q + 1] <= a) ++q;
                    const uint64_t e = std::min(b, tpre[q + 1]);
                    const uint32_t pr = static_cast<uint32_t>(W + q);
                    const uint32_t sl = static_cast<uint32_t>(mp.slot.size());
                    if (mp.pinfo[pr].y == 0) mp.pinfo[pr].x = sl;
                    if (++mp.pinfo[pr].y > csa::SELECT_MAX_PART) ok = false;
                    const uint64_t nt = e - a;
                    mp.slot.push_back(make_uint2(static_cast<uint32_t>(mp.log),
                                                 static_cast<uint32_t>(nt * tile / csa::SELECT_CONSUMER_WARPS)));
                    mp.log += nt * tile;
                    mp.items.push_back(make_uint4(pr, static_cast<uint32_t>(a - tpre[q]),
                                                  static_cast<uint32_t>(e - tpre[q]), sl));
                    a = e;
                }
                if (pieces_first) whole();
            }
            mp.cta[G] = static_cast<uint32_t>(mp.items.size());
            if (!ok || mp.log > 0xffffffffull) {  // no plan: plain rounds / part units
                const std::vector<uint32_t> keep = mp.tiles;
                mp.clear();
                mp.valid = true;
                mp.G = G;
                mp.tiles = keep;
            }
        }
    }
    const std::vector<uint4>& m_items = mp.items;
    const std::vector<uint32_t>& m_cta = mp.cta;
    const std::vector<uint2>& m_pinfo = mp.pinfo;
    const std::vector<uint2>& m_slot = mp.slot;
    const uint64_t m_log = mp.log, m_grid = mp.G;
    const bool mixed_sel = !m_items.empty();
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    // descriptor layout, in two parts uploaded separately: A (problems,
    // inserts, mixed-select tables) before the route/select launches, B (the
    // attention work list and union tables) built and uploaded while select
    // runs on the GPU
    const size_t dbytes = nq * sizeof(csa::DecodeProblem);
    const size_t ibytes = ns * sizeof(csa::InsertProblem);
    const size_t ioff = al(dbytes);
    const size_t m_it = ioff + al(ibytes);  // mixed select: items | cta_items | pinfo | slotinfo
    const size_t m_ct = m_it + al(m_items.size() * 16), m_pi = m_ct + al(m_cta.size() * 4);
    const size_t m_si = m_pi + al(m_pinfo.size() * 8);
    const size_t boff = m_si + al(m_slot.size() * 8);  // part B
    const size_t poff = boff + al((nq + 1) * 4);
    const size_t uoff = poff + al(ncta * 4);  // union tables: gP | gmember | members | mgroup
    const size_t u_gm = uoff + al(ngroups * 4), u_m = u_gm + al(ugmem.size() * 4);
    const size_t u_mg = u_m + al(nmem * 4);
    const size_t need = u_mg + nmem * 4;
    char *hb = nullptr, *db = nullptr;
    if (slot) {
        if (need > slot->cap) {
            if (slot->host) ck(cudaFreeHost(slot->host), "cudaFreeHost");
            slot->cap = need + need / 2;
            ck(cudaMallocHost(&slot->host, slot->cap), "cudaMallocHost");
            slot->dev.alloc(slot->cap);
        }
        if (!slot->done) ck(cudaEventCreateWithFlags(&slot->done, cudaEventDisableTiming), "event");
        hb = static_cast<char*>(slot->host);
        db = slot->dev.as<char>();
    } else if (cap == 1) {
        ctx->cap_need.push_back(need);
    } else {
        const size_t t = ctx->cap_step++;
        if (t >= ctx->cap_need.size() || need > ctx->cap_need[t])
            fail(CSATTN_ERR_GENERIC, "internal: decode graph step differs from its sizing pass");
        hb = static_cast<char*>(ctx->cap_host) + ctx->cap_off[t];
        db = ctx->cap_dev.as<char>() + ctx->cap_off[t];
    }
    if (live) {
        std::memcpy(hb, ctx->hprobs.data(), dbytes);
        std::memcpy(hb + ioff, ctx->hiprobs.data(), ibytes);
        if (mixed_sel) {
            std::memcpy(hb + m_it, m_items.data(), m_items.size() * 16);
            std::memcpy(hb + m_ct, m_cta.data(), m_cta.size() * 4);
            std::memcpy(hb + m_pi, m_pinfo.data(), m_pinfo.size() * 8);
            std::memcpy(hb + m_si, m_slot.data(), m_slot.size() * 8);
        }
        if (!cap)  // a captured step's descriptors go up with its chunk (run_graph)
            ck(cudaMemcpyAsync(db, hb, boff, cudaMemcpyHostToDevice, ctx->stream), "descriptor upload");
    }
    bool staged_b = false;
    auto stage_b = [&]() {  // part B: the attention work list (+ union tables)
    if (!live || staged_b) return;
    staged_b = true;
    std::memcpy(hb + boff, cbase.data(), (nq + 1) * 4);
    {
        // chunk entries (problem | chunk index << 20). Problems on one prefill
        // (a KV head's sequences x query heads) go chunk-major, so the CTAs in
        // flight work on similar key ranges of the shared rows (L2 reuse);
        // CSATTN_ATT_ORDER=problem keeps problem-major order
        uint32_t* cp = reinterpret_cast<uint32_t*>(hb + poff);
        static const bool pmajor = [] {
            const char* o = std::getenv("CSATTN_ATT_ORDER");
            return o && std::strcmp(o, "problem") == 0;
        }();
        uint64_t at = 0;
        const uint64_t step = att_warp ? 4 : 1;  // entries per session (WARP) or per problem
        if (pmajor) {
            for (uint64_t i = 0; i < nq; i += step)
                for (uint32_t j = 0; j < cbase[i + 1] - cbase[i]; ++j)
                    cp[at++] = static_cast<uint32_t>(i) | (j << 20);
        } else {
            uint64_t g0 = 0;
            while (g0 < nq) {  // runs of consecutive problems on the same prefill
                uint64_t g1 = g0 + 1;
                while (g1 < nq && pre_of[g1] == pre_of[g0]) ++g1;
                uint32_t mx = 0;
                for (uint64_t i = g0; i < g1; i += step) mx = std::max(mx, cbase[i + 1] - cbase[i]);
                for (uint32_t j = 0; j < mx; ++j)
                    for (uint64_t i = g0; i < g1; i += step)
                        if (j < cbase[i + 1] - cbase[i]) cp[at++] = static_cast<uint32_t>(i) | (j << 20);
                g0 = g1;
            }
        }
    }
    if (ngroups) {
        std::memcpy(hb + uoff, ugP.data(), ngroups * 4);
        std::memcpy(hb + u_gm, ugmem.data(), ugmem.size() * 4);
        std::memcpy(hb + u_m, umem.data(), nmem * 4);
        std::memcpy(hb + u_mg, umgrp.data(), nmem * 4);
    }
    if (!cap) {
        // on a side stream, joined to the step's stream by an event before
        // attend: the copy overlaps the select kernel instead of sitting
        // between the two. (The slot's earlier use finished: the host waited
        // on slot->done before reusing it.)
        ck(cudaMemcpyAsync(db + boff, hb + boff, need - boff, cudaMemcpyHostToDevice, ctx->side),
           "work list upload");
        ck(cudaEventRecord(ctx->side_ev, ctx->side), "event");
        ck(cudaStreamWaitEvent(ctx->stream, ctx->side_ev, 0), "work list wait");
    }
    };
    const csa::DecodeProblem* dprobs = reinterpret_cast<const csa::DecodeProblem*>(db);
    const csa::InsertProblem* diprobs = reinterpret_cast<const csa::InsertProblem*>(db + ioff);
    const uint32_t* dcbase = reinterpret_cast<const uint32_t*>(db + boff);
    const uint32_t* dcprob = reinterpret_cast<const uint32_t*>(db + poff);
    const auto hte = std::chrono::steady_clock::now();
    std::array<cudaEvent_t, 4> ev{};
    if (ctx->profile) {
        for (auto& e : ev) e = ctx->take_event();
        ck(cudaEventRecord(ev[0], ctx->stream), "event");
    }
    bool ins_forked = false;  // insert launched on the side stream (joined below)
    if (fused) {
        if (live)
            ck(csa::launch_fused_step(dprobs, static_cast<uint32_t>(nq), fz_cl, fz_nr, ctx->stream),
               "fused step launch");
        if (ctx->profile) ck(cudaEventRecord(ev[1], ctx->stream), "event");
    } else {
    ctx->plans.ensure(nq * sizeof(csa::RoutePlan));
    // retry list of problems whose speculative cut proved too high: [count, ids...]
    // (cleared before route: nothing may sit between route and the
    // programmatically launched select)
    ctx->retry.ensure((nq + 1) * 4);
    if (live) ck(cudaMemsetAsync(ctx->retry.p, 0, 4, ctx->stream), "memset");
    if (live)
    ck(csa::launch_route(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq),
                         ctx->stream,
                         ctx->pdl == 4 ? (nq <= static_cast<uint64_t>(ctx->num_sms) ? 1 : 0)
                                       : (ctx->pdl == 1 || ctx->pdl == 2 ? ctx->pdl : 0)),
       "route launch");
    const int sel_sms = ctx->sel_sms ? ctx->sel_sms : ctx->num_sms;
    const uint32_t sgrid = csa::select_grid(static_cast<uint32_t>(nq), sel_sms);
    // Split select for small batches: with fewer problems than CTA slots, each
    // problem's key range is cut into `split` part units (>= one tile each)
    // that run in parallel, then merged (select_merge_kernel).
    const uint64_t tile = csa::select_tile_keys();
    uint64_t min_tiles = ~0ull, max_tiles = 0;
    for (uint64_t i = 0; i < ns; ++i) {
        const uint64_t nt = (ss[i]->N + tile - 1) / tile;
        min_tiles = std::min(min_tiles, nt);
        max_tiles = std::max(max_tiles, nt);
    }
    uint32_t split = 1;
    const uint64_t slots = static_cast<uint64_t>(csa::select_ctas_per_sm()) * sel_sms;  // resident
    if (nq < slots && !ctx->no_split) {
        split = static_cast<uint32_t>((slots + nq - 1) / nq);
        split = static_cast<uint32_t>(std::min<uint64_t>(std::min<uint64_t>(split, 16), min_tiles));
        split = std::max<uint32_t>(split, 1);
    }
    if (const char* fs = std::getenv("CSATTN_FORCE_SPLIT")) {  // experiments only
        split = static_cast<uint32_t>(std::min<uint64_t>(
            std::max<uint64_t>(std::strtoull(fs, nullptr, 10), 1), std::min<uint64_t>(16, min_tiles)));
    }
    if (mixed_sel) split = 1;  // the mixed pieces replace part units
    uint32_t* const rcount = ctx->retry.as<uint32_t>();
    if (maxN > ctx->log_cap || sgrid > ctx->log_rows) {  // non-split / retry-pass logs
        // sized for the sessions' full capacity, so it is not re-grown every step
        uint64_t cap = maxN;
        for (uint64_t i = 0; i < ns; ++i) cap = std::max<uint64_t>(cap, ss[i]->h.max_ctx);
        cap = (cap + csa::SELECT_LOG_ALIGN - 1) / csa::SELECT_LOG_ALIGN * csa::SELECT_LOG_ALIGN;
        ctx->log_cap = std::max<uint64_t>(cap, ctx->log_cap);
        ctx->log_rows = std::max<uint64_t>(sgrid, ctx->log_rows);
        ctx->log_idx.alloc(ctx->log_rows * ctx->log_cap * 4);
        ctx->log_sc.alloc(ctx->log_rows * ctx->log_cap * 8);
    }
    csa::SelMixed smx;
    if (mixed_sel) {
        ctx->mlog_idx.ensure(m_log * 4);
        ctx->mlog_sc.ensure(m_log * 8);
        ctx->mumeta.ensure(m_slot.size() * csa::select_unit_meta_words() * 4);
        if (nq > ctx->pdone_n) {
            ctx->pdone.alloc(nq * 4);
            ck(cudaMemsetAsync(ctx->pdone.p, 0, nq * 4, ctx->stream), "memset");
            ctx->pdone_n = nq;
        }
        smx.items = reinterpret_cast<const uint4*>(db + m_it);
        smx.cta_items = reinterpret_cast<const uint32_t*>(db + m_ct);
        smx.pinfo = reinterpret_cast<const uint2*>(db + m_pi);
        smx.slotinfo = reinterpret_cast<const uint2*>(db + m_si);
        smx.pdone = ctx->pdone.as<uint32_t>();
        smx.plog_idx = ctx->mlog_idx.as<uint32_t>();
        smx.plog_sc = ctx->mlog_sc.as<double>();
        smx.umeta = ctx->mumeta.as<uint32_t>();
    }
    if (!live) {
        if (split > 1) {  // grow the split buffers only
            const uint64_t ucap = (max_tiles + split - 1) / split * tile;
            const uint64_t units = nq * split;
            ctx->ulog_idx.ensure(units * ucap * 4);
            ctx->ulog_sc.ensure(units * ucap * 8);
            ctx->umeta.ensure(units * csa::select_unit_meta_words() * 4);
        }
    } else if (split == 1) {
        ck(csa::launch_select(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq),
                              mixed_sel ? static_cast<uint32_t>(m_grid) : sgrid, ctx->log_idx.as<uint32_t>(), ctx->log_sc.as<double>(),
                              static_cast<uint32_t>(ctx->log_cap), nullptr, nullptr, rcount + 1,
                              rcount, ctx->spec_keep, 1, nullptr, ctx->stream, mixed_sel ? &smx : nullptr,
                              ctx->pdl != 0 && !ctx->profile),
           "select launch");
    } else {
        // per-unit logs: a unit has at most ceil(max_tiles / split) tiles
        const uint64_t ucap = (max_tiles + split - 1) / split * tile;
        const uint64_t units = nq * split;
        ctx->ulog_idx.ensure(units * ucap * 4);
        ctx->ulog_sc.ensure(units * ucap * 8);
        ctx->umeta.ensure(units * csa::select_unit_meta_words() * 4);
        const uint32_t ugrid = static_cast<uint32_t>(std::min<uint64_t>(units, slots));
        ck(csa::launch_select(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq),
                              ugrid, ctx->ulog_idx.as<uint32_t>(), ctx->ulog_sc.as<double>(),
                              static_cast<uint32_t>(ucap), nullptr, nullptr, nullptr, nullptr,
                              ctx->spec_keep, split, ctx->umeta.as<uint32_t>(), ctx->stream),
           "select (split) launch");
        ck(csa::launch_select_merge(dprobs, ctx->plans.as<csa::RoutePlan>(),
                                    static_cast<uint32_t>(nq), split, ctx->umeta.as<uint32_t>(),
                                    ctx->ulog_idx.as<uint32_t>(), ctx->ulog_sc.as<double>(),
                                    static_cast<uint32_t>(ucap), ctx->spec_keep, rcount + 1,
                                    rcount, ctx->stream),
           "select merge launch");
    }
    // second pass over the (usually empty) retry list, without speculation
    if (live)
    ck(csa::launch_select(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq), sgrid,
                          ctx->log_idx.as<uint32_t>(), ctx->log_sc.as<double>(),
                          static_cast<uint32_t>(ctx->log_cap), rcount + 1, rcount, nullptr, nullptr,
                          0.0, 1, nullptr, ctx->stream, nullptr, ctx->pdl != 0 && !ctx->profile),
       "select retry launch");
    stage_b();  // built while route / select run (its upload goes first on the side stream)
    // The append + streaming insert touches the tables and the appended KV
    // row only: it runs beside the attention of this step (which reads rows
    // [0, N) and the selection) once the search has read the tables.
    // (not inside a captured graph: a forked insert branch measured slower
    // there, 761 -> 885 us per c3 step)
    if (live && !cap && ctx->insert_overlap) {
        ck(cudaEventRecord(ctx->ins_fork, ctx->stream), "event");
        ck(cudaStreamWaitEvent(ctx->side, ctx->ins_fork, 0), "insert fork");
        ck(csa::launch_insert(diprobs, static_cast<uint32_t>(ns), ctx->side), "insert launch");
        ck(cudaEventRecord(ctx->ins_join, ctx->side), "event");
        ins_forked = true;
    }
    if (ctx->profile) ck(cudaEventRecord(ev[1], ctx->stream), "event");
    if (nchunks && live)
        ck(csa::launch_attend(dprobs, dcprob, dcbase, static_cast<uint32_t>(ncta),
                              ctx->part.as<float>(), ctx->counters.as<uint32_t>(), d, ctx->stream,
                              false, arows, att_warp),
           "attend launch");
    }
    if (ngroups) {
        stage_b();
        auto u32 = [&](size_t off) { return reinterpret_cast<const uint32_t*>(db + off); };
        if (ctx->union_prof) {
            ctx->un_prof.ensure(static_cast<size_t>(ctx->num_sms) * 160 * 8);
            ck(cudaMemsetAsync(ctx->un_prof.p, 0, static_cast<size_t>(ctx->num_sms) * 160 * 8, ctx->stream), "memset");
        }
        ck(csa::launch_attend_union(dprobs, static_cast<uint32_t>(ngroups), u32(uoff), u32(u_gm),
                                    u32(u_m), u32(u_mg), static_cast<uint32_t>(nmem), u_nrange,
                                    ctx->un_row.as<uint16_t>(), ctx->un_mask.as<unsigned long long>(),
                                    ctx->un_count.as<uint32_t>(), ctx->un_parts.as<float>(),
                                    ctx->un_tails.as<float>(), ctx->num_sms,
                                    ctx->union_prof ? ctx->un_prof.as<unsigned long long>() : nullptr,
                                    ctx->stream),
           "union attend launch");
        ctx->launches += 4;
        if (ctx->union_prof) {
            std::vector<unsigned long long> h(static_cast<size_t>(ctx->num_sms) * 160);
            ck(cudaMemcpyAsync(h.data(), ctx->un_prof.p, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream), "prof");
            ck(cudaStreamSynchronize(ctx->stream), "prof");
            unsigned long long t0 = ~0ull, t1 = 0;
            for (int c = 0; c < ctx->num_sms; ++c)
                for (int i = 0; i < 16; ++i) {
                    const unsigned long long* q = &h[static_cast<size_t>(c) * 160 + i * 4];
                    if (!q[0] || !q[3]) continue;
                    t0 = std::min(t0, q[0]);
                    t1 = std::max(t1, q[3]);
                    ctx->un_sum[0] += double(q[1] - q[0]);
                    if (q[2]) ctx->un_sum[1] += double(q[2] - q[1]);
                    ctx->un_sum[2] += double(q[3] - (q[2] ? q[2] : q[1]));
                    ctx->un_items += 1;
                    ctx->un_tiles += h[static_cast<size_t>(c) * 160 + 64 + i];
                }
            if (t1 > t0) ctx->un_sum[3] += double(t1 - t0);
            if (ctx->un_launches == 3) {  // CTA 0, first item, per tile: relative to item prologue end
                const unsigned long long* q = &h[0];
                const unsigned long long b = q[1];
                for (int t = 0; t < 10 && q[80 + t * 8 + 4]; ++t) {
                    const unsigned long long* z = q + 80 + t * 8;
                    std::fprintf(stderr, "[csattn] tile %d: QK start %.2f issued %.2f  S seen %.2f  P done %.2f  PV start %.2f issued %.2f | K stored %.2f  V stored %.2f us\n", t, (double)(z[7] - b) / 1e3,
                                 (double)(z[0] - b) / 1e3, (double)(z[1] - b) / 1e3, (double)(z[2] - b) / 1e3,
                                 (double)(z[6] - b) / 1e3, (double)(z[3] - b) / 1e3, (double)(z[4] - b) / 1e3,
                                 (double)(z[5] - b) / 1e3);
                }
            }
            ctx->un_launches += 1;
        }
    }
    if (ctx->profile) ck(cudaEventRecord(ev[2], ctx->stream), "event");
    if (ins_forked)
        ck(cudaStreamWaitEvent(ctx->stream, ctx->ins_join, 0), "insert join");
    else if (live)  // after the fused step: a programmatic dependent of it
        ck(csa::launch_insert(diprobs, static_cast<uint32_t>(ns), ctx->stream, nullptr,
                              fused && ctx->pdl != 0 && !ctx->profile),
           "insert launch");
    if (slot) {
        ck(cudaEventRecord(slot->done, ctx->stream), "event");
        slot->used = true;
    }
    if (ctx->profile) {
        ck(cudaEventRecord(ev[3], ctx->stream), "event");
        ctx->ev_steps.push_back(ev);
    }
    ctx->launches += fused ? 2 : (nchunks ? 5 : 4);
    const auto ht2 = std::chrono::steady_clock::now();
    if (ctx->phase_prof) {
        // per problem: streaming (gather + log) and final-selection time,
        // logged candidates, threshold-bin size; printed at context teardown
        std::vector<unsigned long long> ph(nq * 8);
        ck(cudaMemcpyAsync(ph.data(), ctx->phase.p, ph.size() * 8, cudaMemcpyDeviceToHost,
                           ctx->stream), "phase copy");
        ck(cudaStreamSynchronize(ctx->stream), "phase sync");
        double sum[6] = {0, 0, 0, 0, 0, 0};
        uint64_t n = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            const unsigned long long* t = &ph[i * 8];
            if (!t[0] || !t[2]) continue;
            sum[0] += double(t[1] - t[0]);
            sum[1] += double(t[2] - t[1]);
            sum[2] += double(t[3]);
            sum[3] += double(t[4]);
            sum[4] = std::max(sum[4], double(t[4]));
            ++n;
        }
        {
            uint32_t nretry = 0;
            ck(cudaMemcpy(&nretry, ctx->retry.p, 4, cudaMemcpyDeviceToHost), "retry count");
            ctx->phase_retry += nretry;
            ctx->phase_probs += nq;
        }
        if (nq) {
            double lo, hi;
            std::memcpy(&lo, &ph[5], 8);
            std::memcpy(&hi, &ph[6], 8);
            ctx->phase_dbg[0] = lo;
            ctx->phase_dbg[1] = hi;
            ctx->phase_dbg[2] = static_cast<double>(ph[7]);
        }
        {  // select CTA timeline of this step: start / end spread relative to the first start
            const uint32_t nc = static_cast<uint32_t>(std::min<uint64_t>(2 * ctx->num_sms, 1024));
            std::vector<unsigned long long> ts(10 * nc);
            ck(csa::select_cta_times(ts.data(), nc, ctx->stream), "cta times");
            ck(cudaStreamSynchronize(ctx->stream), "cta times");
            std::vector<double> st_, en_;
            unsigned long long t0 = ~0ull;
            for (uint32_t c = 0; c < nc; ++c) if (ts[2 * c]) t0 = std::min(t0, ts[2 * c]);
            for (uint32_t c = 0; c < nc; ++c)
                if (ts[2 * c] && ts[2 * c + 1] > ts[2 * c]) {
                    st_.push_back((ts[2 * c] - t0) / 1e3);
                    en_.push_back((ts[2 * c + 1] - t0) / 1e3);
                }
            if (!en_.empty()) {
                std::sort(st_.begin(), st_.end());
                std::sort(en_.begin(), en_.end());
                auto qv = [](const std::vector<double>& v, double f) { return v[std::min(v.size() - 1, size_t(f * v.size()))]; };
                std::fprintf(stderr, "[cta] n=%zu start q50 %.1f max %.1f | end min %.1f q10 %.1f q50 %.1f q90 %.1f max %.1f us\n",
                             en_.size(), qv(st_, 0.5), st_.back(), en_.front(), qv(en_, 0.1), qv(en_, 0.5), qv(en_, 0.9), en_.back());
                // item-end events: per event index, count by type (1 piece, 2 piece+finalise,
                // 3 whole problem) and the mean time
                {  // mean item duration by type (from the previous event / the CTA start)
                    double dsum[4] = {0, 0, 0, 0};
                    uint32_t dn[4] = {0, 0, 0, 0};
                    for (uint32_t c = 0; c < nc; ++c) {
                        if (!ts[2 * c]) continue;
                        unsigned long long prev = ts[2 * c];
                        for (uint32_t j = 0; j < 8; ++j) {
                            const unsigned long long e = ts[2 * nc + c * 8 + j];
                            const unsigned long long t = e >> 2;
                            if (!e || t < prev || t > ts[2 * c + 1]) break;
                            dsum[e & 3] += (t - prev) / 1e3;
                            dn[e & 3]++;
                            prev = t;
                        }
                    }
                    std::fprintf(stderr, "[cta]   mean item time: piece %.1f us (n=%u), piece+finalise %.1f us (n=%u), whole %.1f us (n=%u)\n",
                                 dn[1] ? dsum[1] / dn[1] : 0.0, dn[1], dn[2] ? dsum[2] / dn[2] : 0.0, dn[2],
                                 dn[3] ? dsum[3] / dn[3] : 0.0, dn[3]);
                }
                for (uint32_t j = 0; j < 8; ++j) {
                    double sum = 0;
                    uint32_t cnt[4] = {0, 0, 0, 0}, n = 0;
                    for (uint32_t c = 0; c < nc; ++c) {
                        const unsigned long long e = ts[2 * nc + c * 8 + j];
                        if (!e || !ts[2 * c]) continue;
                        const unsigned long long t = e >> 2;
                        if (t < ts[2 * c] || t > ts[2 * c + 1]) continue;  // stale (earlier launch)
                        sum += (t - t0) / 1e3;
                        cnt[e & 3]++;
                        ++n;
                    }
                    if (n) std::fprintf(stderr, "[cta]   event %u: n=%u (piece %u, piece+fin %u, whole %u) mean t %.1f us\n",
                                        j, n, cnt[1], cnt[2], cnt[3], sum / n);
                }
            }
        }
        {
            unsigned long long fd[8];
            ck(csa::select_fin_debug(fd, ctx->stream), "fin debug");
            ck(cudaStreamSynchronize(ctx->stream), "fin debug");
            static double acc[8] = {};
            for (int k = 0; k < 8; ++k) acc[k] += double(fd[k]);
            if (acc[6] > 0)
                std::fprintf(stderr, "[fin] per problem us: head %.2f scan %.2f rank %.2f count %.2f pad+scan %.2f emit %.2f (n=%.0f)\n",
                             acc[0] / acc[6] / 1e3, acc[1] / acc[6] / 1e3, acc[2] / acc[6] / 1e3, acc[3] / acc[6] / 1e3,
                             acc[4] / acc[6] / 1e3, acc[5] / acc[6] / 1e3, acc[6]);
        }
        if (n) {
            for (int k = 0; k < 4; ++k) ctx->phase_sum[k] += sum[k] / n;
            ctx->phase_sum[4] = std::max(ctx->phase_sum[4], sum[4]);
            ctx->phase_n += 1;
        }
    }

    // host bookkeeping: SearchState + Session counters
    std::vector<uint64_t> n_before(ns);
    qi = 0;
    for (uint64_t i = 0; i < ns; ++i) {
        csattn_session s = ss[i];
        n_before[i] = s->N;
        for (uint64_t h = 0; h < s->group; ++h, ++qi)
            if (searched[qi]) {
                s->hs[h].has_cache = true;
                s->hs[h].n_cache = s->N;
            }
        s->N += 1;
        s->step += 1;
    }

    if (host) {
        char* base = ctx->stage.as<char>();
        if (out)
            ck(cudaMemcpyAsync(out, base + o_out, nq * d * 4, cudaMemcpyDeviceToHost, ctx->stream),
               "copy out");
        if (selected)
            ck(cudaMemcpyAsync(selected, base + o_sel, nq * sel_stride * 4,
                               cudaMemcpyDeviceToHost, ctx->stream),
               "copy selected");
        if (weights)
            ck(cudaMemcpyAsync(weights, base + o_w, nq * sel_stride * 4, cudaMemcpyDeviceToHost,
                               ctx->stream),
               "copy weights");
    }
    if (reports) {
        qi = 0;
        for (uint64_t i = 0; i < ns; ++i) {
            csattn_session s = ss[i];
            const uint64_t T = s->T();
            std::vector<csa::DecodeReport> dr(s->group);
            uint32_t applied = 0;
            ck(cudaMemcpyAsync(dr.data(), s->drep.p, s->group * sizeof(csa::DecodeReport),
                               cudaMemcpyDeviceToHost, ctx->stream),
               "copy report");
            ck(cudaMemcpyAsync(&applied, s->irep.p, 4, cudaMemcpyDeviceToHost, ctx->stream),
               "copy insert report");
            ck(cudaStreamSynchronize(ctx->stream), "decode step");
            for (uint64_t h = 0; h < s->group; ++h, ++qi) {
                csattn_step_report& r = reports[qi];
                std::memset(&r, 0, sizeof(r));
                r.k = Ks[qi];
                r.searched = searched[qi] ? 1 : 0;
                if (searched[qi]) {
                    r.centroid_dot_ops =
                        dr[h].dot_ops_lo | (static_cast<uint64_t>(dr[h].dot_ops_hi) << 32);
                    r.gathered_entries =
                        dr[h].gathered_lo | (static_cast<uint64_t>(dr[h].gathered_hi) << 32);
                    r.reduce_ops = r.gathered_entries;
                    r.searches = 1;
                    double worst = 1.0;
                    for (uint32_t b = 0; b < s->h.m; ++b) worst = std::min(worst, dr[h].best_cos[b]);
                    s->hs[h].worst = worst;
                }
                r.worst_best_cosine = s->hs[h].worst;
                r.attention_key_ops = Ks[qi] * d;
                r.h2d_bytes_model = 2.0 * s->rc.keep_ratio * static_cast<double>(n_before[i]) *
                                    static_cast<double>(d) * 2.0 /
                                    static_cast<double>(s->rc.search_period);
                r.inserts_attempted = T;
                r.inserts_applied = applied;
                r.insert_dot_ops = static_cast<uint64_t>(s->h.C) * d;
            }
        }
    }
    const auto ht3 = std::chrono::steady_clock::now();
    if (host || !(flags & CSATTN_NO_SYNC)) {
        ck(cudaStreamSynchronize(ctx->stream), "decode step");
        check_appended(ss, ns);
    }
    if (ctx->host_prof && host) {  // host-buffer calls: phases (CSATTN_HOST_PROF=1; diagnostics only)
        const auto ht4 = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        ctx->host_sum[0] += us(ht0, ht1);
        ctx->host_sum[1] += us(ht1, ht2);
        ctx->host_sum[2] += us(ht2, ht3);
        ctx->host_sum[3] += us(ht3, ht4);
        ctx->host_sub[0] += us(ht0, hta);
        ctx->host_sub[1] += us(hta, htb);
        ctx->host_sub[2] += us(htb, htc);
        ctx->host_sub[3] += us(htc, ht1);
        ctx->host_sub2[0] += us(ht1, htd);
        ctx->host_sub2[1] += us(htd, hte);
        ctx->host_sub2[2] += us(hte, ht2);
        ctx->host_n += 1;
    }
}

// ---- host <-> device table images ----

void import_tables(csattn_session_s* s, const uint32_t* lens, const uint32_t* indices,
                   const float* scores, uint64_t stride) {
    const uint64_t T = s->T();
    const uint32_t cap2 = s->h.cap2, nb = s->h.nb_stride, P = s->h.P;
    const uint32_t last_blk = (P - 1) >> csa::KEY_BLOCK_SHIFT;
    std::vector<uint2> ent(T * cap2, make_uint2(0, 0));
    std::vector<uint32_t> nused(T), live(T), bo(T * nb, 0), lcnt(T);
    std::vector<csa::LowEnt> low(T * csa::LOW_Q);
    std::vector<float2> tmm(T, make_float2(0.0f, 0.0f));
    std::vector<uint32_t> order;
    for (uint64_t t = 0; t < T; ++t) {
        const uint32_t n = lens[t];
        if (n > s->h.L) fail(CSATTN_ERR_CORRUPT, "list longer than its capacity");
        const uint32_t* ix = indices + t * stride;
        const float* sc = scores + t * stride;
        order.resize(n);
        for (uint32_t r = 0; r < n; ++r) {
            if (ix[r] >= P) fail(CSATTN_ERR_CORRUPT, "list entry index out of range");
            order[r] = r;
        }
        std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return ix[a] < ix[b]; });
        for (uint32_t r = 1; r < n; ++r)
            if (ix[order[r]] == ix[order[r - 1]]) fail(CSATTN_ERR_CORRUPT, "duplicate key in a list");
        std::vector<uint32_t> pos_of(n);
        for (uint32_t p = 0; p < n; ++p) {
            ent[t * cap2 + p] = make_uint2(ix[order[p]], 0);
            // the stored bits stay as given (a -0.0f score is kept, so an
            // export is byte-identical); select.cu canonicalises at accumulation
            std::memcpy(&ent[t * cap2 + p].y, &sc[order[p]], 4);
            pos_of[order[p]] = p;
        }
        nused[t] = n;
        live[t] = n;
        // key-block offsets
        uint32_t p = 0;
        for (uint32_t kb = 0; kb <= last_blk; ++kb) {
            while (p < n && (ix[order[p]] >> csa::KEY_BLOCK_SHIFT) < kb) ++p;
            bo[t * nb + kb] = p;
        }
        // low buffer: the TopList tail is the eviction order reversed; store
        // descending eviction order = TopList order of the last min(Q, n)
        const uint32_t q = std::min<uint32_t>(n, csa::LOW_Q);
        for (uint32_t r = 0; r < q; ++r) {
            const uint32_t src = n - q + r;  // TopList rank
            csa::LowEnt le{sc[src], ix[src], pos_of[src], 0};
            low[t * csa::LOW_Q + r] = le;
        }
        lcnt[t] = q;
        for (uint32_t r = 0; r < n; ++r) {
            tmm[t].x = r ? std::min(tmm[t].x, sc[r]) : sc[r];
            tmm[t].y = r ? std::max(tmm[t].y, sc[r]) : sc[r];
        }
    }
    cudaStream_t st = s->ctx->stream;
    ck(cudaMemcpyAsync(s->ent.p, ent.data(), ent.size() * sizeof(uint2), cudaMemcpyHostToDevice, st), "import");
    ck(cudaMemcpyAsync(s->n_used.p, nused.data(), T * 4, cudaMemcpyHostToDevice, st), "import");
    ck(cudaMemcpyAsync(s->live.p, live.data(), T * 4, cudaMemcpyHostToDevice, st), "import");
    ck(cudaMemcpyAsync(s->blk_off.p, bo.data(), bo.size() * 4, cudaMemcpyHostToDevice, st), "import");
    ck(cudaMemcpyAsync(s->low.p, low.data(), low.size() * sizeof(csa::LowEnt), cudaMemcpyHostToDevice, st), "import");
    ck(cudaMemcpyAsync(s->low_cnt.p, lcnt.data(), T * 4, cudaMemcpyHostToDevice, st), "import");
    ck(cudaMemcpyAsync(s->tmm.p, tmm.data(), T * sizeof(float2), cudaMemcpyHostToDevice, st), "import");
    ck(cudaStreamSynchronize(st), "import");
}

}  // namespace

extern "C" {

void csattn_index_config_default(csattn_index_config* c) {
    c->alpha = 0.2;
    c->list_capacity = 0;
    c->normalize_keys = 0;
    c->score_bits = 16;
    c->centroids = 64;
    c->iterations = 10;
    c->batch_size = 0;
    c->seed = 0;
    c->tolerance = 1e-7;
}

void csattn_retrieval_config_default(csattn_retrieval_config* c) {
    c->keep_ratio = 0.05;
    c->search_period = 1;
    c->recent_window = 32;
    c->weights = nullptr;
    c->n_weights = 0;
    c->backoff_tau = 1;
    c->backoff_threshold = -std::numeric_limits<double>::infinity();
    c->recent_passthrough = 1;
    c->reserved = 0;
}

void csattn_synthetic_spec_default(csattn_synthetic_spec* s) {
    s->rows = 0;
    s->dim = 64;
    s->clusters = 8;
    s->seed = 0;
    s->plant_fraction = 0.08;
    s->plant_scale = 6.0;
    s->query_noise = 0.05;
    s->dwell = 32;
}

csattn_status csattn_keep_count(double rho, uint64_t n, uint64_t* out) {
    return guard([&] { *out = keep_count(rho, n); });
}

// parse_schedule (retrieval.cpp:10-32)
csattn_status csattn_parse_schedule(const char* cname, double* rho, uint64_t* period) {
    return guard([&] {
        const std::string name = cname ? cname : "";
        const std::string sep = "-step-";
        const auto at = name.find(sep);
        if (at == std::string::npos || at == 0 || at + sep.size() >= name.size())
            fail(CSATTN_ERR_PARAMETER, "schedule must look like \"<rho>-step-<P>\": " + name);
        double r = 0.0;
        unsigned long pp = 0;
        bool bad = false;
        try {
            std::size_t used = 0;
            r = std::stod(name.substr(0, at), &used);
            if (used != at) bad = true;
            const std::string tail = name.substr(at + sep.size());
            if (!bad) {
                pp = std::stoul(tail, &used);
                if (used != tail.size()) bad = true;
            }
        } catch (const std::exception&) {
            bad = true;
        }
        if (bad) fail(CSATTN_ERR_PARAMETER, "cannot parse schedule \"" + name + "\"");
        if (!(r > 0.0 && r <= 1.0))
            fail(CSATTN_ERR_PARAMETER, "schedule keep ratio must lie in (0, 1]");
        if (pp == 0) fail(CSATTN_ERR_PARAMETER, "schedule period must be >= 1");
        *rho = r;
        *period = pp;
    });
}

// h2d_bytes (metrics.cpp:32-38)
csattn_status csattn_h2d_bytes(double rho, uint64_t n, uint64_t d, uint64_t b, uint64_t period,
                               double* out) {
    return guard([&] {
        if (!(rho > 0.0) || n == 0 || d == 0 || b == 0 || period == 0)
            fail(CSATTN_ERR_PARAMETER, "transfer model needs positive parameters");
        *out = 2.0 * rho * static_cast<double>(n) * static_cast<double>(d) *
               static_cast<double>(b) / static_cast<double>(period);
    });
}

const char* csattn_last_error(void) { return g_err.c_str(); }

const char* csattn_status_name(csattn_status s) {
    switch (s) {
        case CSATTN_OK: return "ok";
        case CSATTN_ERR_GENERIC: return "Error";
        case CSATTN_ERR_DIMENSION: return "DimensionError";
        case CSATTN_ERR_PARAMETER: return "ParameterError";
        case CSATTN_ERR_DATA: return "DataError";
        case CSATTN_ERR_BAD_MAGIC: return "BadMagicError";
        case CSATTN_ERR_VERSION: return "VersionError";
        case CSATTN_ERR_TRUNCATED: return "TruncatedError";
        case CSATTN_ERR_CORRUPT: return "CorruptError";
        case CSATTN_ERR_PROPERTY: return "PropertyError";
        case CSATTN_ERR_STREAM_EXHAUSTED: return "StreamExhaustedError";
        case CSATTN_ERR_CUDA: return "CudaError";
        case CSATTN_ERR_CAPACITY: return "CapacityError";
    }
    return "unknown";
}

csattn_status csattn_ctx_create(int device, void* stream, csattn_ctx* out) {
    return guard([&] {
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) fail(CSATTN_ERR_PARAMETER, "no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        int major = 0, minor = 0;
        ck(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device), "attr");
        ck(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device), "attr");
        if (major != 10)
            fail(CSATTN_ERR_CUDA, "this build targets sm_100a (B200); device is sm_" +
                                      std::to_string(major) + std::to_string(minor));
        auto c = std::make_unique<csattn_ctx_s>();
        c->device = device;
        ck(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
        if (stream) {
            c->stream = static_cast<cudaStream_t>(stream);
        } else {
            ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
            c->own = true;
        }
        // the side stream + its events exist before any graph capture
        ck(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream");
        ck(cudaEventCreateWithFlags(&c->side_ev, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->ins_fork, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->ins_join, cudaEventDisableTiming), "event");
        *out = c.release();
    });
}

}  // extern "C"

// A context lives until its handle AND every session created on it are gone
// (sessions keep a reference), so destruction order never matters.
static void ctx_release(csattn_ctx ctx) {
    if (--ctx->refs > 0) return;
    if (ctx->phase_n) {
        const double n = static_cast<double>(ctx->phase_n);
        std::fprintf(stderr,
                     "[csattn] select per problem (mean over %llu steps): stream=%.2fus "
                     "final=%.2fus logged=%.0f bin_members=%.1f (max %.0f)\n",
                     static_cast<unsigned long long>(ctx->phase_n), ctx->phase_sum[0] / n / 1e3,
                     ctx->phase_sum[1] / n / 1e3, ctx->phase_sum[2] / n, ctx->phase_sum[3] / n,
                     ctx->phase_sum[4]);
        std::fprintf(stderr, "[csattn] problem 0 of the last step: bounds [%g, %g] take_all|bin<<1=%g\n",
                     ctx->phase_dbg[0], ctx->phase_dbg[1], ctx->phase_dbg[2]);
        std::fprintf(stderr, "[csattn] speculative cut: %llu of %llu problems retried\n",
                     static_cast<unsigned long long>(ctx->phase_retry),
                     static_cast<unsigned long long>(ctx->phase_probs));
    }
    if (ctx->host_n) {
        const double n = static_cast<double>(ctx->host_n);
        std::fprintf(stderr,
                     "[csattn] run_step host (mean over %llu calls): prepare %.1f us, stage+launch %.1f us, "
                     "bookkeeping+copies %.1f us, sync wait %.1f us\n",
                     static_cast<unsigned long long>(ctx->host_n), ctx->host_sum[0] / n, ctx->host_sum[1] / n,
                     ctx->host_sum[2] / n, ctx->host_sum[3] / n);
        std::fprintf(stderr, "[csattn]   prepare = sizes %.1f + finite checks %.1f + uploads %.1f + descriptors %.1f us\n",
                     ctx->host_sub[0] / n, ctx->host_sub[1] / n, ctx->host_sub[2] / n, ctx->host_sub[3] / n);
        std::fprintf(stderr, "[csattn]   stage+launch = slot wait %.1f + work list/staging %.1f + launches %.1f us\n",
                     ctx->host_sub2[0] / n, ctx->host_sub2[1] / n, ctx->host_sub2[2] / n);
    }
    if (ctx->un_items) {
        const double n = static_cast<double>(ctx->un_items);
        std::fprintf(stderr,
                     "[csattn] union kernel: %llu launches, %.1f items/launch, %.1f tiles/item; per item "
                     "prologue=%.2fus tiles=%.2fus epilogue=%.2fus; kernel span %.1fus\n",
                     static_cast<unsigned long long>(ctx->un_launches), n / ctx->un_launches,
                     static_cast<double>(ctx->un_tiles) / n, ctx->un_sum[0] / n / 1e3,
                     ctx->un_sum[1] / n / 1e3, ctx->un_sum[2] / n / 1e3,
                     ctx->un_sum[3] / ctx->un_launches / 1e3);
    }
    cudaStreamSynchronize(ctx->stream);
    for (auto& ev : ctx->ev_steps)
        for (cudaEvent_t e : ev) ctx->ev_pool.push_back(e);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->own) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

extern "C" {

csattn_status csattn_ctx_destroy(csattn_ctx ctx) {
    return guard([&] {
        if (!ctx) return;
        ctx_release(ctx);
    });
}

}  // extern "C"

csattn_session_s::~csattn_session_s() {
    if (ctx) {
        cudaStreamSynchronize(ctx->stream);
        if (bad) ctx->bad_free.push_back(bad);
        ctx_release(ctx);
    }
}

extern "C" {

csattn_status csattn_ctx_set_kv_placement(csattn_ctx ctx, int32_t placement) {
    return guard([&] {
        if (placement != CSATTN_KV_DEVICE && placement != CSATTN_KV_HOST)
            fail(CSATTN_ERR_PARAMETER, "KV placement must be CSATTN_KV_DEVICE or CSATTN_KV_HOST");
        ctx->kv_host = placement == CSATTN_KV_HOST;
    });
}

csattn_status csattn_ctx_synchronize(csattn_ctx ctx) {
    return guard([&] { ck(cudaStreamSynchronize(ctx->stream), "synchronize"); });
}

uint64_t csattn_ctx_launch_count(csattn_ctx ctx) { return ctx ? ctx->launches : 0; }

csattn_status csattn_ctx_build_stats(csattn_ctx ctx, uint64_t* tc_builds, uint64_t* fallbacks) {
    return guard([&] {
        if (!ctx) fail(CSATTN_ERR_PARAMETER, "null context");
        if (tc_builds) *tc_builds = ctx->build_tc;
        if (fallbacks) *fallbacks = ctx->build_fallback;
    });
}

csattn_status csattn_ctx_profile(csattn_ctx ctx, int32_t enable) {
    return guard([&] { ctx->profile = enable != 0; });
}

csattn_status csattn_ctx_profile_read(csattn_ctx ctx, double* ms, uint64_t* steps,
                                      int32_t reset) {
    return guard([&] {
        ck(cudaStreamSynchronize(ctx->stream), "profile sync");
        ms[0] = ms[1] = ms[2] = 0.0;
        for (auto& ev : ctx->ev_steps)
            for (int k = 0; k < 3; ++k) {
                float x = 0.0f;
                ck(cudaEventElapsedTime(&x, ev[k], ev[k + 1]), "elapsed");
                ms[k] += x;
            }
        *steps = ctx->ev_steps.size();
        if (reset) {
            for (auto& ev : ctx->ev_steps)
                for (cudaEvent_t e : ev) ctx->ev_pool.push_back(e);
            ctx->ev_steps.clear();
        }
    });
}

// prefill (session.cpp:25-44) -> build_index (index.cpp:145-177) on the GPU.
}  // extern "C"

namespace {

// One session's prefill (prefill, session.cpp:25-44): validation, session,
// rows and the per-subspace k-means jobs (setup), then the status check and
// the table build (finish). csattn_prefill runs one; csattn_prefill_batch runs
// a layer's sessions with ONE k-means launch of n x m CTAs (the jobs, and so
// the tables, are identical to n single prefills).
struct PrefillWork {
    std::unique_ptr<csattn_session_s> s;
    DevMem dq, drng, train, best, run, assign, sums, counts, status, info;
    std::vector<csa::KmeansJob> hj;
    bool full_batch = false;
};

void prefill_setup(PrefillWork& W, csattn_ctx ctx, const float* queries, uint64_t nq,
                   const float* keys, const float* values, uint64_t p, uint64_t d,
                   const uint64_t* widths, uint64_t m, const csattn_index_config* icfg,
                   const csattn_retrieval_config* rcfg, uint64_t group, uint64_t max_steps,
                   bool host) {
    validate_layout(widths, m, d);
    if (nq == 0) fail(CSATTN_ERR_PARAMETER, "prefill must be non-empty");
    validate_retrieval(rcfg, m);
    check_rows(keys, values, p, d, host);
    validate_index(icfg);
    if (p == 0) fail(CSATTN_ERR_PARAMETER, "cannot build over an empty prefill");
    const uint64_t C = icfg->centroids;
    for (uint64_t b = 0; b < m; ++b)
        if (C * widths[b] > csa::KM_MAX_KW)
            fail(CSATTN_ERR_PARAMETER, "B200 build supports C * width <= " +
                                           std::to_string(csa::KM_MAX_KW));
    if (nq >= 0x7fffffffull) fail(CSATTN_ERR_PARAMETER, "too many query rows");
    double alpha;
    const uint64_t L = list_capacity_of(icfg, p, &alpha);
    W.s = new_session(ctx, d, widths, m, C, L, p, group, max_steps, rcfg);
    csattn_session_s* s = W.s.get();
    s->alpha = alpha;
    s->h.normalize_keys = icfg->normalize_keys ? 1u : 0u;
    s->score_bits = icfg->score_bits;
    attach_rows(s, keys, values, host);
    cudaStream_t st = ctx->stream;
    // ---- per-subspace exact k-means, one CTA per subspace ----
    W.dq.alloc(nq * d * sizeof(float));
    upload(ctx, W.dq.p, queries, nq * d * sizeof(float), host);
    const uint32_t iters = static_cast<uint32_t>(icfg->iterations);
    const uint32_t bcfg = static_cast<uint32_t>(std::min<uint64_t>(icfg->batch_size, 0xffffffffu));
    const size_t ndraw = csa::kmeans_rng_draws(static_cast<uint32_t>(C), iters,
                                               static_cast<uint32_t>(nq), bcfg);
    std::vector<unsigned long long> draws(m * ndraw);
    for (uint64_t b = 0; b < m; ++b) {
        // cc.seed = mix_seed(seed, b) (index.cpp:170); Rng = mt19937_64
        uint64_t z = icfg->seed + 0x9e3779b97f4a7c15ULL * (b + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        std::mt19937_64 gen(z ^ (z >> 31));
        for (size_t i = 0; i < ndraw; ++i) draws[b * ndraw + i] = gen();
    }
    W.drng.alloc(draws.size() * 8);
    // synchronous: `draws` is a host temporary
    ck(cudaMemcpyAsync(W.drng.p, draws.data(), draws.size() * 8, cudaMemcpyDefault, st), "copy in");
    ck(cudaStreamSynchronize(st), "rng upload");
    uint64_t wsum = 0;
    for (uint64_t b = 0; b < m; ++b) wsum += widths[b];
    W.train.alloc(nq * wsum * sizeof(float));
    W.best.alloc(m * nq * sizeof(double));
    W.run.alloc(m * nq * sizeof(double));
    W.assign.alloc(m * 2 * nq * sizeof(uint32_t));
    W.sums.alloc(C * wsum * sizeof(double));
    W.counts.alloc(m * C * sizeof(uint32_t));
    W.status.alloc(m * sizeof(int));
    W.info.alloc(m * 2 * sizeof(uint32_t));
    ck(cudaMemsetAsync(W.status.p, 0, m * sizeof(int), st), "memset");
    ck(cudaMemsetAsync(W.info.p, 0, m * 2 * sizeof(uint32_t), st), "memset");
    W.hj.resize(m);
    for (uint64_t b = 0; b < m; ++b) {
        csa::KmeansJob& J = W.hj[b];
        const uint32_t off = s->h.offs[b];
        J.q = W.dq.as<float>();
        J.n_total = static_cast<uint32_t>(nq);
        J.d = static_cast<uint32_t>(d);
        J.off = off;
        J.w = static_cast<uint32_t>(widths[b]);
        J.k = static_cast<uint32_t>(C);
        J.iters = iters;
        J.batch_cfg = bcfg;
        J.pad = 0;
        J.tol = icfg->tolerance;
        J.rng = W.drng.as<unsigned long long>() + b * ndraw;
        J.train = W.train.as<float>() + nq * off;
        J.best = W.best.as<double>() + b * nq;
        J.run = W.run.as<double>() + b * nq;
        J.assign = W.assign.as<uint32_t>() + b * 2 * nq;
        J.sums = W.sums.as<double>() + C * off;
        J.counts = W.counts.as<uint32_t>() + b * C;
        J.cent = s->cent.as<float>() + C * off;
        J.status = W.status.as<int>() + b;
        J.info = W.info.as<uint32_t>() + 2 * b;
    }
    const uint64_t bt = bcfg == 0 ? std::min<uint64_t>(4096, nq) : std::min<uint64_t>(bcfg, nq);
    W.full_batch = bt >= nq;
}

// one k-means launch over every job of `works`, then each session's checks + build
void prefill_run(csattn_ctx ctx, std::vector<PrefillWork>& works) {
    cudaStream_t st = ctx->stream;
    std::vector<csa::KmeansJob> all;
    for (auto& W : works) all.insert(all.end(), W.hj.begin(), W.hj.end());
    DevMem jobs;
    jobs.alloc(all.size() * sizeof(csa::KmeansJob));
    upload(ctx, jobs.p, all.data(), all.size() * sizeof(csa::KmeansJob), true);
    ck(csa::launch_kmeans(jobs.as<csa::KmeansJob>(), static_cast<uint32_t>(all.size()), st),
       "kmeans launch");
    ctx->launches += 1;
    std::vector<std::vector<int>> hs(works.size());
    for (size_t i = 0; i < works.size(); ++i) {
        hs[i].resize(works[i].hj.size());
        ck(cudaMemcpyAsync(hs[i].data(), works[i].status.p, hs[i].size() * sizeof(int),
                           cudaMemcpyDeviceToHost, st),
           "status");
    }
    ck(cudaStreamSynchronize(st), "kmeans");
    for (size_t i = 0; i < works.size(); ++i)
        for (int v : hs[i]) {
            if (v == 4) fail(CSATTN_ERR_DATA, "every training row is zero");
            if (v == 9)
                fail(CSATTN_ERR_PROPERTY, works[i].full_batch
                                              ? "clustering objective increased in a full-batch iteration"
                                              : "mini-batch clustering objective diverged");
        }
    for (auto& W : works) build_tables(W.s.get());
}

}  // namespace

extern "C" {

csattn_status csattn_prefill(csattn_ctx ctx, const float* queries, uint64_t nq, const float* keys,
                             const float* values, uint64_t p, uint64_t d, const uint64_t* widths,
                             uint64_t m, const csattn_index_config* icfg,
                             const csattn_retrieval_config* rcfg, uint64_t group,
                             uint64_t max_steps, uint32_t flags, csattn_session* out) {
    return guard([&] {
        std::vector<PrefillWork> works(1);
        prefill_setup(works[0], ctx, queries, nq, keys, values, p, d, widths, m, icfg, rcfg, group,
                      max_steps, flags & CSATTN_HOST_BUFFERS);
        prefill_run(ctx, works);
        *out = works[0].s.release();
    });
}

csattn_status csattn_prefill_batch(csattn_ctx ctx, uint64_t n, const csattn_prefill_rows* rows,
                                   uint64_t d, const uint64_t* widths, uint64_t m,
                                   const csattn_index_config* icfgs,
                                   const csattn_retrieval_config* rcfg, uint64_t group,
                                   uint64_t max_steps, uint32_t flags, csattn_session* out) {
    return guard([&] {
        if (n == 0) fail(CSATTN_ERR_PARAMETER, "no sessions");
        std::vector<PrefillWork> works(n);
        for (uint64_t i = 0; i < n; ++i)
            prefill_setup(works[i], ctx, rows[i].queries, rows[i].n_queries, rows[i].keys,
                          rows[i].values, rows[i].n_rows, d, widths, m, icfgs + i, rcfg, group, max_steps,
                          flags & CSATTN_HOST_BUFFERS);
        prefill_run(ctx, works);
        for (uint64_t i = 0; i < n; ++i) out[i] = works[i].s.release();
    });
}

csattn_status csattn_prefill_from_centroids(csattn_ctx ctx, const float* centroids, uint64_t c,
                                            const float* keys, const float* values, uint64_t p,
                                            uint64_t d, const uint64_t* widths, uint64_t m,
                                            const csattn_index_config* icfg,
                                            const csattn_retrieval_config* rcfg, uint64_t group,
                                            uint64_t max_steps, uint32_t flags,
                                            csattn_session* out) {
    return guard([&] {
        const bool host = flags & CSATTN_HOST_BUFFERS;
        validate_layout(widths, m, d);
        validate_retrieval(rcfg, m);
        check_rows(keys, values, p, d, host);
        validate_index(icfg);
        if (p == 0) fail(CSATTN_ERR_PARAMETER, "cannot build over an empty prefill");
        if (c == 0) fail(CSATTN_ERR_PARAMETER, "centroid sets are empty");
        double alpha;
        const uint64_t L = list_capacity_of(icfg, p, &alpha);
        auto s = new_session(ctx, d, widths, m, c, L, p, group, max_steps, rcfg);
        s->alpha = alpha;
        s->h.normalize_keys = icfg->normalize_keys ? 1u : 0u;
        s->score_bits = icfg->score_bits;
        attach_rows(s.get(), keys, values, host);
        upload(ctx, s->cent.p, centroids, c * d * sizeof(float), true);
        build_tables(s.get());
        *out = s.release();
    });
}

csattn_status csattn_session_import(csattn_ctx ctx, const float* centroids, uint64_t c,
                                    const uint32_t* lens, const uint32_t* indices,
                                    const float* scores, uint64_t stride,
                                    uint64_t list_capacity, double alpha, int32_t normalize_keys,
                                    int32_t score_bits, const float* keys, const float* values,
                                    uint64_t p, uint64_t d, const uint64_t* widths, uint64_t m,
                                    const csattn_retrieval_config* rcfg, uint64_t group,
                                    uint64_t max_steps, csattn_session* out) {
    return guard([&] {
        validate_layout(widths, m, d);
        validate_retrieval(rcfg, m);
        check_rows(keys, values, p, d, true);
        if (p == 0) fail(CSATTN_ERR_PARAMETER, "cannot build over an empty prefill");
        if (c == 0) fail(CSATTN_ERR_PARAMETER, "centroid sets are empty");
        if (list_capacity == 0) fail(CSATTN_ERR_PARAMETER, "list capacity came out as zero");
        auto s = new_session(ctx, d, widths, m, c, list_capacity, p, group, max_steps, rcfg);
        s->alpha = alpha;
        s->h.normalize_keys = normalize_keys ? 1u : 0u;
        s->score_bits = score_bits;
        attach_rows(s.get(), keys, values, true);
        upload(ctx, s->cent.p, centroids, c * d * sizeof(float), true);
        push_dev(s.get());
        import_tables(s.get(), lens, indices, scores, stride);
        *out = s.release();
    });
}

csattn_status csattn_session_export(csattn_session s, uint32_t* lens, uint32_t* indices,
                                    float* scores, uint64_t stride, float* centroids) {
    return guard([&] {
        const uint64_t T = s->T();
        const uint32_t cap2 = s->h.cap2;
        std::vector<uint2> ent(T * cap2);
        std::vector<uint32_t> nused(T), live(T);
        cudaStream_t st = s->ctx->stream;
        ck(cudaMemcpyAsync(ent.data(), s->ent.p, ent.size() * sizeof(uint2), cudaMemcpyDeviceToHost, st), "export");
        ck(cudaMemcpyAsync(nused.data(), s->n_used.p, T * 4, cudaMemcpyDeviceToHost, st), "export");
        ck(cudaMemcpyAsync(live.data(), s->live.p, T * 4, cudaMemcpyDeviceToHost, st), "export");
        if (centroids)
            ck(cudaMemcpyAsync(centroids, s->cent.p, static_cast<size_t>(s->h.C) * s->h.d * 4,
                               cudaMemcpyDeviceToHost, st),
               "export");
        ck(cudaStreamSynchronize(st), "export");
        std::vector<std::pair<float, uint32_t>> v;
        for (uint64_t t = 0; t < T; ++t) {
            v.clear();
            for (uint32_t p = 0; p < nused[t]; ++p) {
                const uint2 e = ent[t * cap2 + p];
                if (e.x & csa::TOMB) continue;
                float f;
                std::memcpy(&f, &e.y, 4);
                v.emplace_back(f, e.x);
            }
            if (v.size() != live[t]) fail(CSATTN_ERR_CORRUPT, "table live count mismatch");
            if (v.size() > stride) fail(CSATTN_ERR_PARAMETER, "export stride too small");
            std::sort(v.begin(), v.end(), [](const auto& a, const auto& b) {
                if (a.first != b.first) return a.first > b.first;
                return a.second < b.second;
            });
            lens[t] = static_cast<uint32_t>(v.size());
            for (size_t r = 0; r < v.size(); ++r) {
                indices[t * stride + r] = v[r].second;
                scores[t * stride + r] = v[r].first;
            }
        }
    });
}

// ---- CSAT v1 image of a session (serialize_index / load_index, index.cpp:289-433) ----

csattn_status csattn_session_serialize(csattn_session s, uint8_t* out, uint64_t capacity,
                                       uint64_t* size) {
    return guard([&] {
        if (!size) fail(CSATTN_ERR_PARAMETER, "size must not be null");
        const uint64_t T = s->T();
        const uint32_t cap2 = s->h.cap2;
        cudaStream_t st = s->ctx->stream;
        csattn_csat_header h{};
        h.m = s->h.m;
        h.centroids = s->h.C;
        h.list_capacity = s->h.L;
        h.dim = s->h.d;
        h.prefill_len = s->index_prefill ? s->index_prefill : s->h.P;
        h.score_bits = s->score_bits == 16 ? 16 : 32;
        h.normalize_keys = s->h.normalize_keys ? 1 : 0;
        for (uint64_t b = 0; b < h.m; ++b) h.widths[b] = s->h.widths[b];
        std::vector<float> cent(static_cast<size_t>(h.centroids) * h.dim);
        std::vector<uint32_t> live(T);
        ck(cudaMemcpyAsync(cent.data(), s->cent.p, cent.size() * 4, cudaMemcpyDeviceToHost, st), "serialize");
        ck(cudaMemcpyAsync(live.data(), s->live.p, T * 4, cudaMemcpyDeviceToHost, st), "serialize");
        ck(cudaStreamSynchronize(st), "serialize");
        const uint64_t pre = csa_host::csat_prefix(&h, cent.data(), nullptr);
        const uint64_t sb = h.score_bits == 16 ? 2 : 4;
        std::vector<unsigned long long> off(T);
        std::vector<int> seg_b(T), seg_e(T);
        uint64_t tb = 0;
        std::vector<uint32_t> nused(T);
        ck(cudaMemcpy(nused.data(), s->n_used.p, T * 4, cudaMemcpyDeviceToHost), "serialize");
        for (uint64_t t = 0; t < T; ++t) {
            off[t] = tb;
            tb += 4 + static_cast<uint64_t>(live[t]) * (4 + sb);
            seg_b[t] = static_cast<int>(t * cap2);
            seg_e[t] = static_cast<int>(t * cap2 + nused[t]);
        }
        *size = pre + tb;
        if (!out) return;
        if (capacity < *size)
            fail(CSATTN_ERR_PARAMETER, "serialize: buffer holds " + std::to_string(capacity) +
                                           " bytes, image needs " + std::to_string(*size));
        if (T * cap2 > static_cast<uint64_t>(std::numeric_limits<int>::max()))
            fail(CSATTN_ERR_CAPACITY, "serialize: table image too large for one sort");
        csa_host::csat_prefix(&h, cent.data(), out);
        DevMem keys, sorted, temp, segs, offs, img;
        keys.alloc(T * cap2 * 8);
        sorted.alloc(T * cap2 * 8);
        const size_t tbytes = csa::csat_sort_temp_bytes(static_cast<uint32_t>(T), cap2);
        temp.alloc(tbytes);
        segs.alloc(T * 8);
        offs.alloc(T * 8);
        img.alloc(tb);
        ck(cudaMemcpyAsync(segs.p, seg_b.data(), T * 4, cudaMemcpyHostToDevice, st), "serialize");
        ck(cudaMemcpyAsync(segs.as<int>() + T, seg_e.data(), T * 4, cudaMemcpyHostToDevice, st), "serialize");
        ck(cudaMemcpyAsync(offs.p, off.data(), T * 8, cudaMemcpyHostToDevice, st), "serialize");
        ck(csa::launch_csat_tables(s->ent.as<uint2>(), s->n_used.as<uint32_t>(), s->live.as<uint32_t>(),
                                   static_cast<uint32_t>(T), cap2, segs.as<int>(), segs.as<int>() + T,
                                   offs.as<unsigned long long>(), h.score_bits == 16 ? 1 : 0,
                                   keys.as<unsigned long long>(), sorted.as<unsigned long long>(), temp.p,
                                   tbytes, img.as<unsigned char>(), st),
           "serialize launch");
        ck(cudaMemcpyAsync(out + pre, img.p, tb, cudaMemcpyDeviceToHost, st), "serialize");
        ck(cudaStreamSynchronize(st), "serialize");
        s->ctx->launches += 3;
    });
}

csattn_status csattn_session_deserialize(csattn_ctx ctx, const uint8_t* bytes, uint64_t n,
                                         const float* keys, const float* values, uint64_t n_rows,
                                         const csattn_retrieval_config* rcfg, uint64_t group,
                                         uint64_t max_decode_steps, csattn_session* out) {
    return guard([&] {
        csattn_csat_header h{};
        check_status(csattn_csat_read_header(bytes, n, &h));
        const uint64_t T = h.m * h.centroids, L = h.list_capacity;
        std::vector<float> cent(h.centroids * h.dim), sc(T * L);
        std::vector<uint32_t> lens(T), ix(T * L);
        check_status(csattn_csat_decode(bytes, n, &h, cent.data(), lens.data(), ix.data(), sc.data(), L));
        // A session's image can index keys appended after the prefill
        // (streaming inserts); the KV rows must cover every indexed key. All
        // n_rows rows become the session's resident rows; prefill_len stays the
        // index's metadata (written back by serialize).
        if (n_rows < h.prefill_len)
            fail(CSATTN_ERR_PARAMETER, "the image indexes " + std::to_string(h.prefill_len) +
                                           " prefill rows, got " + std::to_string(n_rows) + " KV rows");
        const double alpha = static_cast<double>(L) / static_cast<double>(h.prefill_len);
        check_status(csattn_session_import(ctx, cent.data(), h.centroids, lens.data(), ix.data(), sc.data(), L, L,
                                           alpha, h.normalize_keys, h.score_bits, keys, values,
                                           n_rows, h.dim, h.widths, h.m, rcfg, group,
                                           max_decode_steps, out));
        (*out)->index_prefill = h.prefill_len;
    });
}

csattn_status csattn_session_gather_stats(csattn_session s, uint64_t* unique_entries,
                                          uint64_t* total_entries) {
    return guard([&] {
        std::vector<csa::DecodeReport> dr(s->group);
        std::vector<uint32_t> live(s->T());
        ck(cudaMemcpyAsync(dr.data(), s->drep.p, s->group * sizeof(csa::DecodeReport),
                           cudaMemcpyDeviceToHost, s->ctx->stream),
           "copy report");
        ck(cudaMemcpyAsync(live.data(), s->live.p, live.size() * 4, cudaMemcpyDeviceToHost,
                           s->ctx->stream),
           "copy live");
        ck(cudaStreamSynchronize(s->ctx->stream), "gather stats");
        std::vector<char> seen(s->T(), 0);
        uint64_t u = 0, t = 0;
        for (uint64_t h = 0; h < s->group; ++h)
            for (uint32_t l = 0; l < dr[h].nl && l < static_cast<uint32_t>(csa::MAXL); ++l) {
                const uint32_t tb = dr[h].lists[l];
                if (tb >= s->T()) continue;
                t += live[tb];
                if (!seen[tb]) {
                    seen[tb] = 1;
                    u += live[tb];
                }
            }
        *unique_entries = u;
        *total_entries = t;
    });
}


// ---------------------------------------------------------------------------
// sequence sharding
// ---------------------------------------------------------------------------
csattn_status csattn_shard_create(csattn_ctx ctx, csattn_session full, uint64_t key_lo,
                                  uint64_t key_hi, int32_t owner, uint64_t max_steps,
                                  csattn_session* out) {
    return guard([&] {
        const uint64_t P = full->h.P, d = full->h.d, tile = csa::select_tile_keys();
        if (full->step != 0) fail(CSATTN_ERR_PARAMETER, "shard a session before its first decode step");
        if (key_lo % tile || (!owner && key_hi % tile) || key_lo >= key_hi || key_hi > P)
            fail(CSATTN_ERR_PARAMETER, "shard bounds must be multiples of " + std::to_string(tile) +
                                           " keys inside the prefill");
        if (full->rc.search_period != 1)
            fail(CSATTN_ERR_PARAMETER, "sharded decoding needs search period 1");
        const uint64_t T = full->T(), L = full->h.L;
        if (full->ctx->device != ctx->device)
            fail(CSATTN_ERR_PARAMETER, "shard and source session must share a device");
        csattn_retrieval_config rc = full->rc;
        rc.weights = full->weights.data();
        rc.n_weights = full->weights.size();
        ck(cudaStreamSynchronize(full->ctx->stream), "shard source");
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        auto s = new_session(ctx, d, full->widths.data(), full->h.m, full->h.C, L, P, full->group,
                             max_steps, &rc);
        s->alpha = full->alpha;
        s->score_bits = full->score_bits;
        s->h.normalize_keys = full->h.normalize_keys;
        // KV rows [key_lo, key_hi); kpre/vpre offset so that row i is at kpre[i*d]
        s->pre = std::make_shared<SharedRows>();
        const size_t rows = (key_hi - key_lo) * d * sizeof(float);
        s->pre->k.alloc(rows);
        s->pre->v.alloc(rows);
        ck(cudaMemcpy(s->pre->k.p, full->h.kpre + key_lo * d, rows, cudaMemcpyDefault), "shard rows");
        ck(cudaMemcpy(s->pre->v.p, full->h.vpre + key_lo * d, rows, cudaMemcpyDefault), "shard rows");
        s->h.kpre = s->pre->k.as<float>() - key_lo * d;
        s->h.vpre = s->pre->v.as<float>() - key_lo * d;
        ck(cudaMemcpy(s->cent.p, full->cent.p, static_cast<size_t>(full->h.C) * d * 4, cudaMemcpyDefault),
           "shard centroids");
        s->live_g.alloc(T * 4);
        s->h.live_g = s->live_g.as<uint32_t>();
        s->h.key_lo = static_cast<uint32_t>(key_lo);
        s->h.key_hi = static_cast<uint32_t>(key_hi);
        s->h.owner = owner ? 1u : 0u;
        s->h.sharded = 1;
        push_dev(s.get());
        // the shard's part of every list, extracted and re-indexed on the device
        ck(cudaStreamSynchronize(ctx->stream), "shard setup");
        ck(csa::launch_shard_extract(full->dev.as<csa::SessionDev>(), s->dev.as<csa::SessionDev>(),
                                     static_cast<uint32_t>(T), static_cast<uint32_t>(key_lo),
                                     static_cast<uint32_t>(key_hi), ctx->stream),
           "shard extract launch");
        ck(cudaStreamSynchronize(ctx->stream), "shard extract");
        *out = s.release();
    });
}

csattn_status csattn_shard_buffer_words(csattn_session s, uint64_t* hist_words,
                                        uint64_t* bucket_words, uint64_t* partial_floats,
                                        uint64_t* victim_words) {
    return guard([&] {
        *hist_words = csa::shard_hist_words();
        *bucket_words = csa::shard_bucket_words();
        *partial_floats = s->h.d + 2;
        *victim_words = s->T();
    });
}

csattn_status csattn_shard_step(csattn_ctx ctx, uint64_t ns, const csattn_session* ss,
                                int32_t phase, const csattn_shard_io* io) {
    return guard([&] {
        if (ns == 0) fail(CSATTN_ERR_PARAMETER, "no sessions");
        if (!io) fail(CSATTN_ERR_PARAMETER, "null io");
        for (uint64_t i = 0; i < ns; ++i)
            if (!ss[i]->h.sharded) fail(CSATTN_ERR_PARAMETER, "not a shard session (csattn_shard_create)");
        const uint32_t d = ss[0]->h.d;
        cudaStream_t st = ctx->stream;
        const uint64_t tile = csa::select_tile_keys();
        if (phase == CSATTN_SHARD_SCAN || phase == CSATTN_SHARD_RESCAN) {
            ctx->sh_spec = phase == CSATTN_SHARD_SCAN ? ctx->spec_keep : 0.0;
            uint64_t nq = 0, maxtiles = 0, maxrange = 0;
            ctx->sh_Ks.clear();
            for (uint64_t i = 0; i < ns; ++i) {
                csattn_session s = ss[i];
                if (s->ctx != ctx) fail(CSATTN_ERR_PARAMETER, "sessions belong to another context");
                if (s->h.d != d) fail(CSATTN_ERR_DIMENSION, "sessions differ in head dimension");
                check_not_poisoned(s);  // a non-finite row refused by an earlier INSERT phase
                if (s->step >= s->max_steps)
                    fail(CSATTN_ERR_CAPACITY, "session is full: max_decode_steps = " +
                                                  std::to_string(s->max_steps));
                for (uint64_t h = 0; h < s->group; ++h) ctx->sh_Ks.push_back(keep_count(s->rc.keep_ratio, s->N));
                nq += s->group;
                const uint64_t khi = s->h.owner ? s->N : s->h.key_hi;
                maxtiles = std::max(maxtiles, (khi - s->h.key_lo + tile - 1) / tile);
                maxrange = std::max<uint64_t>(maxrange, (s->h.owner ? s->h.max_ctx : s->h.key_hi) - s->h.key_lo);
            }
            if (io->selected && io->sel_stride < *std::max_element(ctx->sh_Ks.begin(), ctx->sh_Ks.end()))
                fail(CSATTN_ERR_PARAMETER, "selected stride is below K");
            // part units over the shard's tiles so a small batch fills the GPU
            uint64_t mintiles = ~0ull;
            for (uint64_t i = 0; i < ns; ++i) {
                const uint64_t khi = ss[i]->h.owner ? ss[i]->N : ss[i]->h.key_hi;
                mintiles = std::min(mintiles, (khi - ss[i]->h.key_lo + tile - 1) / tile);
            }
            const uint64_t slots = static_cast<uint64_t>(csa::select_ctas_per_sm()) * ctx->num_sms;
            // (default 1: the shard phases after the scan walk every part's log;
            // CSATTN_SHARD_SPLIT=1 enables part units here)
            uint64_t split = (nq < slots && ctx->shard_split) ? (slots + nq - 1) / nq : 1;
            split = std::max<uint64_t>(1, std::min<uint64_t>(std::min<uint64_t>(split, 16), mintiles));
            ctx->sh_split = static_cast<uint32_t>(split);
            ctx->sh_nq = nq;
            ctx->sh_ns = ns;
            ctx->sh_ucap = (maxtiles + split - 1) / split * tile;
            ctx->sh_bm_words = (maxrange + 31) / 32;
            ctx->sh_umeta.ensure(nq * split * csa::select_unit_meta_words() * 4);
            ctx->sh_ulog_idx.ensure(nq * split * ctx->sh_ucap * 4);
            ctx->sh_ulog_sc.ensure(nq * split * ctx->sh_ucap * 8);
            ctx->sh_pstate.ensure(nq * csa::shard_pstate_bytes());
            ctx->sh_bitmap.ensure(nq * ctx->sh_bm_words * 4);
            ctx->sh_kdev.ensure(nq * 4);
            ctx->sh_hprobs.resize(nq);
            ctx->sh_hiprobs.resize(ns);
            uint64_t qi = 0;
            for (uint64_t i = 0; i < ns; ++i) {
                csattn_session s = ss[i];
                const uint64_t khi = s->h.owner ? s->N : s->h.key_hi;
                for (uint64_t h = 0; h < s->group; ++h, ++qi) {
                    csa::DecodeProblem& P = ctx->sh_hprobs[qi];
                    P = csa::DecodeProblem{};
                    P.s = s->dev.as<csa::SessionDev>();
                    P.q = io->q + qi * d;
                    P.out = io->partial + qi * (d + 2);
                    P.weights = nullptr;
                    P.sel = io->selected ? io->selected + qi * io->sel_stride
                                         : s->sel.as<uint32_t>() + h * s->h.max_ctx;
                    P.cache = nullptr;
                    P.cbounds = s->cbounds.as<double>() + h * 4;
                    P.rep = reinterpret_cast<uint32_t*>(s->drep.as<csa::DecodeReport>() + h);
                    P.N = static_cast<uint32_t>(s->N);
                    P.K = static_cast<uint32_t>(ctx->sh_Ks[qi]);
                    P.mode = csa::MODE_SEARCH | csa::MODE_PARTIAL;
                    P.tile_lo = static_cast<uint32_t>(s->h.key_lo / tile);
                    P.tile_hi = static_cast<uint32_t>((khi + tile - 1) / tile);
                    P.kdev = ctx->sh_kdev.as<uint32_t>();
                }
                csa::InsertProblem& I = ctx->sh_hiprobs[i];
                I.s = s->dev.as<csa::SessionDev>();
                I.key = io->new_keys + i * d;
                I.value = io->new_values + i * d;
                I.rep = s->irep.as<uint32_t>();
                I.N = static_cast<uint32_t>(s->N);
                I.bad = s->bad;
                I.pad = 0;
            }
            // attention work list: ceil(K / ATT_ROWS) chunk-CTAs per problem (global K:
            // the shard's own share is read on the device, excess chunks idle)
            std::vector<uint32_t> cbase(nq + 1), cprob;
            for (uint64_t i = 0; i < nq; ++i) {
                cbase[i] = static_cast<uint32_t>(cprob.size());
                const uint64_t nc = (ctx->sh_Ks[i] + csa::ATT_ROWS - 1) / csa::ATT_ROWS;
                for (uint32_t j = 0; j < nc; ++j) cprob.push_back(static_cast<uint32_t>(i) | (j << 20));
            }
            cbase[nq] = static_cast<uint32_t>(cprob.size());
            ctx->sh_nchunks = cprob.size();
            ctx->sh_chunk_host.assign(cbase.begin(), cbase.end());
            ctx->sh_chunk_host.insert(ctx->sh_chunk_host.end(), cprob.begin(), cprob.end());
            const size_t dbytes = nq * sizeof(csa::DecodeProblem), ibytes = ns * sizeof(csa::InsertProblem);
            const size_t ioff = (dbytes + 255) & ~size_t(255);
            ctx->sh_desc.ensure(ioff + ibytes);
            ck(cudaMemcpyAsync(ctx->sh_desc.p, ctx->sh_hprobs.data(), dbytes, cudaMemcpyHostToDevice, st), "desc");
            ck(cudaMemcpyAsync(ctx->sh_desc.as<char>() + ioff, ctx->sh_hiprobs.data(), ibytes,
                               cudaMemcpyHostToDevice, st), "desc");
            ctx->sh_chunks.ensure(ctx->sh_chunk_host.size() * 4);
            ck(cudaMemcpyAsync(ctx->sh_chunks.p, ctx->sh_chunk_host.data(), ctx->sh_chunk_host.size() * 4,
                               cudaMemcpyHostToDevice, st), "chunks");
            if (nq > ctx->counters_n) {
                ctx->counters.alloc(nq * 4);
                ck(cudaMemsetAsync(ctx->counters.p, 0, nq * 4, st), "memset");
                ctx->counters_n = nq;
            }
            ctx->part.ensure(ctx->sh_nchunks * (d + 2) * sizeof(float));
            ctx->plans.ensure(nq * sizeof(csa::RoutePlan));
            const csa::DecodeProblem* dprobs = ctx->sh_desc.as<csa::DecodeProblem>();
            ck(csa::launch_route(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq), st),
               "route launch");
            const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(nq * split, slots));
            ck(csa::launch_select(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq), grid,
                                  ctx->sh_ulog_idx.as<uint32_t>(), ctx->sh_ulog_sc.as<double>(),
                                  static_cast<uint32_t>(ctx->sh_ucap), nullptr, nullptr, nullptr,
                                  nullptr, ctx->sh_spec, static_cast<uint32_t>(split),
                                  ctx->sh_umeta.as<uint32_t>(), st),
               "select (shard scan) launch");
            ck(csa::launch_shard_hist_sum(ctx->sh_umeta.as<uint32_t>(), static_cast<uint32_t>(nq),
                                          static_cast<uint32_t>(split), io->ghist, st),
               "histograms");
            ctx->launches += 2;
            ctx->sh_scanned = true;
            return;
        }
        if (!ctx->sh_scanned || ns != ctx->sh_ns) fail(CSATTN_ERR_PARAMETER, "shard phases out of order");
        const uint64_t nq = ctx->sh_nq;
        const csa::DecodeProblem* dprobs = ctx->sh_desc.as<csa::DecodeProblem>();
        const size_t ioff = (nq * sizeof(csa::DecodeProblem) + 255) & ~size_t(255);
        const csa::InsertProblem* diprobs =
            reinterpret_cast<const csa::InsertProblem*>(ctx->sh_desc.as<char>() + ioff);
        switch (phase) {
            case CSATTN_SHARD_BUCKET:
                ck(csa::launch_shard_bucket(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq),
                                            io->ghist, ctx->sh_umeta.as<uint32_t>(),
                                            ctx->sh_ulog_idx.as<uint32_t>(), ctx->sh_ulog_sc.as<double>(),
                                            static_cast<uint32_t>(ctx->sh_ucap), ctx->sh_split,
                                            io->bucket, ctx->sh_pstate.p, ctx->sh_spec,
                                            io->spec_fail, st),
                   "shard bucket launch");
                break;
            case CSATTN_SHARD_MARK:
                ck(csa::launch_shard_mark(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq),
                                          ctx->sh_pstate.p, io->bucket_all, io->n_shards,
                                          ctx->sh_umeta.as<uint32_t>(), ctx->sh_ulog_idx.as<uint32_t>(),
                                          ctx->sh_ulog_sc.as<double>(), static_cast<uint32_t>(ctx->sh_ucap),
                                          ctx->sh_split, ctx->sh_bitmap.as<uint32_t>(),
                                          static_cast<uint32_t>(ctx->sh_bm_words), io->counts, st),
                   "shard mark launch");
                break;
            case CSATTN_SHARD_EMIT: {
                ck(csa::launch_shard_emit(dprobs, ctx->plans.as<csa::RoutePlan>(), static_cast<uint32_t>(nq),
                                          io->counts_all, io->n_shards, io->shard_index,
                                          ctx->sh_bitmap.as<uint32_t>(),
                                          static_cast<uint32_t>(ctx->sh_bm_words), ctx->sh_kdev.as<uint32_t>(), st),
                   "shard emit launch");
                if (io->n_selected)
                    ck(cudaMemcpyAsync(io->n_selected, ctx->sh_kdev.p, nq * 4, cudaMemcpyDeviceToDevice, st),
                       "n_selected");
                const uint32_t* ch = ctx->sh_chunks.as<uint32_t>();
                ck(csa::launch_attend(dprobs, ch + nq + 1, ch, static_cast<uint32_t>(ctx->sh_nchunks),
                                      ctx->part.as<float>(), ctx->counters.as<uint32_t>(), d, st, true),
                   "attend launch");
                ctx->launches += 2;
                break;
            }
            case CSATTN_SHARD_MERGE:
                ck(csa::launch_shard_merge(io->partial_all, io->n_shards, static_cast<uint32_t>(nq), d,
                                           io->out, st),
                   "shard merge launch");
                break;
            case CSATTN_SHARD_VICTIM:
                ck(csa::launch_shard_victim(diprobs, static_cast<uint32_t>(ns), io->victim, st),
                   "shard victim launch");
                break;
            case CSATTN_SHARD_INSERT:
                ck(csa::launch_insert(diprobs, static_cast<uint32_t>(ns), st, io->victim), "insert launch");
                for (uint64_t i = 0; i < ns; ++i) {
                    csattn_session s = ss[i];
                    for (uint64_t h = 0; h < s->group; ++h) {
                        s->hs[h].has_cache = true;
                        s->hs[h].n_cache = s->N;
                    }
                    s->N += 1;
                    s->step += 1;
                }
                ctx->sh_scanned = false;
                // no stream sync: the next step's descriptor copies are stream-
                // ordered after these kernels (pageable sources are staged before
                // cudaMemcpyAsync returns), and the collectives run on this stream
                break;
            default:
                fail(CSATTN_ERR_PARAMETER, "unknown shard phase");
        }
        ctx->launches += 1;
    });
}

csattn_status csattn_session_centroids(csattn_session s, float* centroids) {
    return guard([&] {
        if (!centroids) fail(CSATTN_ERR_PARAMETER, "null output");
        ck(cudaMemcpyAsync(centroids, s->cent.p, static_cast<size_t>(s->h.C) * s->h.d * 4,
                           cudaMemcpyDeviceToHost, s->ctx->stream),
           "copy centroids");
        ck(cudaStreamSynchronize(s->ctx->stream), "centroids");
    });
}

csattn_status csattn_session_fork(csattn_session src, uint64_t max_steps, csattn_session* out) {
    return guard([&] {
        if (max_steps < src->step) fail(CSATTN_ERR_PARAMETER, "fork capacity below steps taken");
        csattn_retrieval_config rc = src->rc;
        rc.weights = src->weights.data();
        rc.n_weights = src->weights.size();
        auto s = new_session(src->ctx, src->h.d, src->widths.data(), src->h.m, src->h.C, src->h.L,
                             src->h.P, src->group, max_steps, &rc);
        s->alpha = src->alpha;
        s->score_bits = src->score_bits;
        s->index_prefill = src->index_prefill;
        s->h.normalize_keys = src->h.normalize_keys;
        s->pre = src->pre;
        s->h.kpre = src->h.kpre;
        s->h.vpre = src->h.vpre;
        s->N = src->N;
        s->step = src->step;
        s->hs = src->hs;
        cudaStream_t st = src->ctx->stream;
        const uint64_t T = s->T();
        auto d2d = [&](DevMem& dst, const DevMem& from, size_t bytes) {
            ck(cudaMemcpyAsync(dst.p, from.p, bytes, cudaMemcpyDefault, st), "fork copy");
        };
        const size_t rows = (src->N - src->h.P) * src->h.d * 4;
        if (rows) {
            d2d(s->ktail, src->ktail, rows);
            d2d(s->vtail, src->vtail, rows);
        }
        d2d(s->cent, src->cent, static_cast<size_t>(src->h.C) * src->h.d * 4);
        // tables: capacities are identical (same L, P)
        d2d(s->ent, src->ent, T * src->h.cap2 * sizeof(uint2));
        d2d(s->n_used, src->n_used, T * 4);
        d2d(s->live, src->live, T * 4);
        const uint32_t nbs = std::min(s->h.nb_stride, src->h.nb_stride);
        ck(cudaMemcpy2DAsync(s->blk_off.p, s->h.nb_stride * 4, src->blk_off.p,
                             src->h.nb_stride * 4, nbs * 4, T, cudaMemcpyDeviceToDevice, st),
           "fork blk_off");
        d2d(s->low, src->low, T * csa::LOW_Q * sizeof(csa::LowEnt));
        d2d(s->low_cnt, src->low_cnt, T * 4);
        d2d(s->tmm, src->tmm, T * sizeof(float2));
        d2d(s->cbounds, src->cbounds, s->group * 4 * sizeof(double));
        if (s->cache.p && src->cache.p)
            for (uint64_t h = 0; h < s->group; ++h)
                ck(cudaMemcpyAsync(s->cache.as<double>() + h * s->h.max_ctx,
                                   src->cache.as<double>() + h * src->h.max_ctx,
                                   src->N * sizeof(double), cudaMemcpyDeviceToDevice, st),
                   "fork cache");
        push_dev(s.get());
        ck(cudaStreamSynchronize(st), "fork");
        *out = s.release();
    });
}

csattn_status csattn_session_destroy(csattn_session s) {
    return guard([&] { delete s; });
}

csattn_status csattn_session_info_get(csattn_session s, csattn_session_info* o) {
    return guard([&] {
        o->dim = s->h.d;
        o->subspaces = s->h.m;
        o->centroids = s->h.C;
        o->list_capacity = s->h.L;
        o->prefill_len = s->index_prefill ? s->index_prefill : s->h.P;
        o->context_len = s->N;
        o->steps = s->step;
        o->max_context = s->h.max_ctx;
        o->group = s->group;
        o->alpha = s->alpha;
        o->normalize_keys = static_cast<int32_t>(s->h.normalize_keys);
        o->score_bits = s->score_bits;
        o->device_bytes = s->device_bytes();
    });
}

csattn_status csattn_session_set_retrieval(csattn_session s, const csattn_retrieval_config* rc) {
    return guard([&] {
        validate_retrieval(rc, s->h.m);
        if (rc->search_period > 1 && !s->cache.p) {
            // decode_search would reuse state.cached from the last search on
            // the next off-period step (retrieval.cpp:237-238); without a kept
            // candidate cache that set is gone, so refuse instead of diverging
            for (const HeadState& h : s->hs)
                if (h.has_cache)
                    fail(CSATTN_ERR_PARAMETER,
                         "B200 path: raising search_period above 1 after decode steps needs "
                         "csattn_session_keep_candidates(1) before those steps");
            s->cache.alloc(s->group * s->h.max_ctx * sizeof(double));
        }
        set_retrieval(s, rc);
        push_dev(s);
        ck(cudaStreamSynchronize(s->ctx->stream), "set_retrieval");
    });
}

csattn_status csattn_session_keep_candidates(csattn_session s, int32_t enable) {
    return guard([&] {
        if (enable && !s->cache.p) {
            s->cache.alloc(s->group * s->h.max_ctx * sizeof(double));
        } else if (!enable && s->cache.p && s->rc.search_period <= 1) {
            cudaStreamSynchronize(s->ctx->stream);
            cudaFree(s->cache.p);
            s->cache.p = nullptr;
            s->cache.n = 0;
        }
    });
}

csattn_status csattn_session_candidates(csattn_session s, uint64_t head, uint32_t* indices,
                                        double* scores, uint64_t cap, uint64_t* n) {
    return guard([&] {
        if (head >= s->group) fail(CSATTN_ERR_PARAMETER, "query head out of range");
        if (!s->cache.p) fail(CSATTN_ERR_PARAMETER, "candidates are not kept (keep_candidates)");
        *n = 0;
        const HeadState& hs = s->hs[head];
        if (!hs.has_cache) return;
        std::vector<double> c(hs.n_cache);
        ck(cudaMemcpyAsync(c.data(), s->cache.as<double>() + head * s->h.max_ctx,
                           hs.n_cache * sizeof(double), cudaMemcpyDeviceToHost, s->ctx->stream),
           "copy candidates");
        ck(cudaStreamSynchronize(s->ctx->stream), "candidates");
        uint64_t k = 0;
        for (uint64_t i = 0; i < hs.n_cache; ++i) {
            uint64_t bits;
            std::memcpy(&bits, &c[i], 8);
            if (bits == 0x7ff4deadbeef0000ull) continue;  // absent (select.cu ABSENT)
            if (k < cap) {
                indices[k] = static_cast<uint32_t>(i);
                scores[k] = c[i];
            }
            ++k;
        }
        if (k > cap) fail(CSATTN_ERR_PARAMETER, "candidate buffer too small");
        *n = k;
    });
}

csattn_status csattn_session_read_kv(csattn_session s, uint64_t first, uint64_t count,
                                     float* keys, float* values) {
    return guard([&] {
        if (first + count > s->N) fail(CSATTN_ERR_PARAMETER, "row range out of bounds");
        const uint64_t d = s->h.d, P = s->h.P;
        cudaStream_t st = s->ctx->stream;
        for (uint64_t i = first; i < first + count;) {
            const bool pre = i < P;
            const uint64_t lim = pre ? std::min(P, first + count) : first + count;
            const uint64_t n = lim - i;
            const float* kb = pre ? s->h.kpre + i * d : s->h.ktail + (i - P) * d;
            const float* vb = pre ? s->h.vpre + i * d : s->h.vtail + (i - P) * d;
            if (keys)
                ck(cudaMemcpyAsync(keys + (i - first) * d, kb, n * d * 4, cudaMemcpyDefault, st), "read kv");
            if (values)
                ck(cudaMemcpyAsync(values + (i - first) * d, vb, n * d * 4, cudaMemcpyDefault, st), "read kv");
            i = lim;
        }
        ck(cudaStreamSynchronize(st), "read kv");
    });
}

csattn_status csattn_decode_step(csattn_session s, const float* q, const float* new_key,
                                 const float* new_value, float* out, uint32_t* selected,
                                 float* weights, uint64_t sel_stride,
                                 csattn_step_report* reports, const uint64_t* k_override,
                                 uint32_t flags) {
    return guard([&] {
        if (!s) fail(CSATTN_ERR_PARAMETER, "null session");
        csattn_session one[1] = {s};
        run_step(s->ctx, 1, one, q, new_key, new_value, out, selected, weights, sel_stride,
                 reports, k_override, flags);
    });
}

csattn_status csattn_decode_batch(csattn_ctx ctx, uint64_t n, const csattn_session* ss,
                                  const float* q, const float* keys, const float* values,
                                  float* out, uint32_t* selected, uint64_t sel_stride,
                                  uint32_t flags) {
    return guard([&] {
        run_step(ctx, n, ss, q, keys, values, out, selected, nullptr, sel_stride, nullptr,
                 nullptr, flags);
    });
}

}  // extern "C"

// ---- whole-run decode as one CUDA graph ----

namespace {

// T consecutive decode steps of a session set (run_decode, session.cpp:101-126,
// without the per-step reports) captured into one CUDA graph and launched once:
// no per-step host round trip, launch or descriptor wait. Pass 1 runs the host
// side of every step without stream work, so every buffer reaches its final
// size and each step's descriptor bytes are known; the session counters are
// then rewound and pass 2 captures the same steps, each staging its descriptors
// in its own slice of one pinned arena.
void run_graph(csattn_ctx ctx, uint64_t ns, const csattn_session* ss, uint64_t T, const float* q,
               const float* keys, const float* values, float* out, uint32_t* selected,
               uint64_t sel_stride, const uint64_t* k_override, uint32_t flags) {
    if (ns == 0) fail(CSATTN_ERR_PARAMETER, "no sessions");
    if (T == 0) return;
    const bool host = flags & CSATTN_HOST_BUFFERS;
    const uint64_t d = ss[0]->h.d;
    uint64_t nq = 0;
    check_distinct(ss, ns);
    for (uint64_t i = 0; i < ns; ++i) {
        if (ss[i]->ctx != ctx) fail(CSATTN_ERR_PARAMETER, "sessions belong to another context");
        check_not_poisoned(ss[i]);
        if (ss[i]->step + T > ss[i]->max_steps)
            fail(CSATTN_ERR_CAPACITY, "session is full: max_decode_steps = " +
                                          std::to_string(ss[i]->max_steps));
        nq += ss[i]->group;
    }
    const auto hs0 = std::chrono::steady_clock::now();
    const float *dq = q, *dk = keys, *dv = values;
    float* dout = out;
    uint32_t* dsel = selected;
    size_t o_out = 0, o_sel = 0;
    if (host) {
        require_finite(keys, T * ns * d, "appended key");
        require_finite(values, T * ns * d, "appended value");
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        const size_t o_k = al(T * nq * d * 4), o_v = o_k + al(T * ns * d * 4);
        o_out = o_v + al(T * ns * d * 4);
        o_sel = o_out + (out ? al(T * nq * d * 4) : 0);
        const size_t total = o_sel + (selected ? T * nq * sel_stride * 4 : 0);
        ctx->run_stage.ensure(total);
        char* b = ctx->run_stage.as<char>();
        upload(ctx, b, q, T * nq * d * 4, true);
        upload(ctx, b + o_k, keys, T * ns * d * 4, true);
        upload(ctx, b + o_v, values, T * ns * d * 4, true);
        dq = reinterpret_cast<const float*>(b);
        dk = reinterpret_cast<const float*>(b + o_k);
        dv = reinterpret_cast<const float*>(b + o_v);
        dout = out ? reinterpret_cast<float*>(b + o_out) : nullptr;
        dsel = selected ? reinterpret_cast<uint32_t*>(b + o_sel) : nullptr;
    }
    struct Saved {
        uint64_t N, step;
        std::vector<HeadState> hs;
    };
    std::vector<Saved> saved;
    for (uint64_t i = 0; i < ns; ++i) saved.push_back({ss[i]->N, ss[i]->step, ss[i]->hs});
    const uint64_t launches0 = ctx->launches;
    const bool prof[3] = {ctx->profile, ctx->phase_prof, ctx->union_prof};
    auto reset = [&] {
        for (uint64_t i = 0; i < ns; ++i) {
            ss[i]->N = saved[i].N;
            ss[i]->step = saved[i].step;
            ss[i]->hs = saved[i].hs;
        }
        ctx->launches = launches0;
    };
    auto leave = [&] {
        g_no_alloc = false;
        ctx->capture = 0;
        ctx->profile = prof[0];
        ctx->phase_prof = prof[1];
        ctx->union_prof = prof[2];
    };
    auto steps = [&](uint64_t t0, uint64_t t1) {
        for (uint64_t t = t0; t < t1; ++t)
            run_step(ctx, ns, ss, dq + t * nq * d, dk + t * ns * d, dv + t * ns * d,
                     dout ? dout + t * nq * d : nullptr,
                     dsel ? dsel + t * nq * sel_stride : nullptr, nullptr, sel_stride, nullptr,
                     k_override ? k_override + t * nq : nullptr, CSATTN_NO_SYNC);
    };
    const auto h0 = std::chrono::steady_clock::now();
    ctx->profile = ctx->phase_prof = ctx->union_prof = false;
    // chunks of kChunk steps: chunk c+1 is captured and instantiated while
    // chunk c runs, so only the sizing pass and the first capture are exposed
    constexpr uint64_t kChunk = 4;
    std::vector<cudaGraph_t> graphs;
    std::vector<cudaGraphExec_t> execs;
    auto release = [&] {
        for (auto x : execs) cudaGraphExecDestroy(x);
        for (auto g : graphs) cudaGraphDestroy(g);
    };
    uint64_t launched = 0;  // steps whose graph was launched
    std::chrono::steady_clock::time_point h1, h2;
    try {
        ctx->capture = 1;  // pass 1: sizes
        ctx->cap_need.clear();
        steps(0, T);
        reset();
        ctx->cap_off.assign(T, 0);
        size_t total = 0;
        for (uint64_t t = 0; t < T; ++t) {
            ctx->cap_off[t] = total;
            total += (ctx->cap_need[t] + 255) & ~size_t(255);
        }
        if (total > ctx->cap_bytes) {
            // the previous run (if any) finished: run_graph synchronizes
            if (ctx->cap_host) ck(cudaFreeHost(ctx->cap_host), "cudaFreeHost");
            ctx->cap_host = nullptr;
            ctx->cap_bytes = 0;
            ck(cudaMallocHost(&ctx->cap_host, total + total / 4), "cudaMallocHost");
            ctx->cap_dev.alloc(total + total / 4);
            ctx->cap_bytes = total + total / 4;
        }
        h1 = std::chrono::steady_clock::now();
        ctx->capture = 2;  // pass 2: capture chunk by chunk
        ctx->cap_step = 0;
        for (uint64_t c0 = 0; c0 < T; c0 += kChunk) {
            const uint64_t c1 = std::min(T, c0 + kChunk);
            cudaGraph_t g = nullptr;
            ck(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
            g_no_alloc = true;
            try {
                steps(c0, c1);
            } catch (...) {
                g_no_alloc = false;
                cudaStreamEndCapture(ctx->stream, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            g_no_alloc = false;
            ck(cudaStreamEndCapture(ctx->stream, &g), "end capture");
            graphs.push_back(g);
            cudaGraphExec_t x = nullptr;
            ck(cudaGraphInstantiate(&x, g, 0), "graph instantiate");
            execs.push_back(x);
            // the chunk's descriptors in one copy, then its kernels
            const size_t a = ctx->cap_off[c0], z = ctx->cap_off[c1 - 1] + ctx->cap_need[c1 - 1];
            ck(cudaMemcpyAsync(ctx->cap_dev.as<char>() + a, static_cast<char*>(ctx->cap_host) + a, z - a,
                               cudaMemcpyHostToDevice, ctx->stream),
               "descriptor upload");
            ck(cudaGraphLaunch(x, ctx->stream), "graph launch");
            launched = c1;
            if (c0 == 0) h2 = std::chrono::steady_clock::now();
        }
        leave();
    } catch (...) {
        leave();
        // host counters back to the last launched step: rewind, then replay the
        // host side of the launched steps without stream work
        reset();
        if (launched) {
            ctx->capture = 1;
            ctx->cap_need.clear();
            try {
                steps(0, launched);
            } catch (...) {
            }
            ctx->capture = 0;
        }
        cudaStreamSynchronize(ctx->stream);
        release();
        throw;
    }
    if (host) {
        const char* b = ctx->run_stage.as<char>();
        if (out)
            ck(cudaMemcpyAsync(out, b + o_out, T * nq * d * 4, cudaMemcpyDeviceToHost, ctx->stream),
               "copy out");
        if (selected)
            ck(cudaMemcpyAsync(selected, b + o_sel, T * nq * sel_stride * 4,
                               cudaMemcpyDeviceToHost, ctx->stream),
               "copy selected");
    }
    const auto h3 = std::chrono::steady_clock::now();
    // the arena and the graphs are released once the run is done
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    release();
    if (ctx->host_prof) {
        const auto h4 = std::chrono::steady_clock::now();
        auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
        std::fprintf(stderr, "[csattn] decode_run %llu steps: inputs %.1f us, sizing %.1f, first chunk capture+launch %.1f, "
                     "remaining captures %.1f, wait %.1f us\n", static_cast<unsigned long long>(T),
                     us(hs0, h0), us(h0, h1), us(h1, h2), us(h2, h3), us(h3, h4));
    }
    ck(e, "decode run");
    // a non-finite row inside a graph run: later steps already ran on it
    for (uint64_t i = 0; i < ns; ++i) check_not_poisoned(ss[i]);
}

}  // namespace

extern "C" {

csattn_status csattn_decode_run(csattn_ctx ctx, uint64_t n_sessions, const csattn_session* sessions,
                                uint64_t n_steps, const float* q, const float* new_keys,
                                const float* new_values, float* out, uint32_t* selected,
                                uint64_t sel_stride, const uint64_t* k_override, uint32_t flags) {
    return guard([&] {
        run_graph(ctx, n_sessions, sessions, n_steps, q, new_keys, new_values, out, selected,
                  sel_stride, k_override, flags);
    });
}

// ---- the dense oracle on the device (core.cpp:118-192) ----

csattn_status csattn_dense_attention(csattn_session s, const float* q, const uint32_t* mask,
                                     uint64_t n_mask, float* out, float* weights,
                                     uint32_t flags) {
    return guard([&] {
        const bool host = flags & CSATTN_HOST_BUFFERS;
        const uint64_t N = s->N, d = s->h.d;
        if (N == 0) fail(CSATTN_ERR_PARAMETER, "attention over an empty KV store");
        uint64_t n = N;
        std::vector<uint32_t> hm;
        if (mask) {
            if (n_mask == 0) fail(CSATTN_ERR_PARAMETER, "attention over an empty index set");
            hm.resize(n_mask);
            if (host)
                std::memcpy(hm.data(), mask, n_mask * 4);
            else
                ck(cudaMemcpy(hm.data(), mask, n_mask * 4, cudaMemcpyDeviceToHost), "dense mask");
            for (uint32_t i : hm)
                if (i >= N) fail(CSATTN_ERR_PARAMETER, "mask index " + std::to_string(i) + " out of range");
            n = n_mask;
        }
        csattn_ctx ctx = s->ctx;
        cudaStream_t st = ctx->stream;
        ctx->dense.ensure(csa::dense_scratch_bytes(static_cast<uint32_t>(n), static_cast<uint32_t>(d)) +
                          n * 8 + d * 8 + n * 4 + 1024);
        char* base = ctx->dense.as<char>();
        const size_t scratch = csa::dense_scratch_bytes(static_cast<uint32_t>(n), static_cast<uint32_t>(d));
        float* dq = reinterpret_cast<float*>(base + scratch);
        uint32_t* dmask = reinterpret_cast<uint32_t*>(base + scratch + ((d * 4 + 255) & ~size_t(255)));
        float* dout = reinterpret_cast<float*>(reinterpret_cast<char*>(dmask) + ((n * 4 + 255) & ~size_t(255)));
        float* dw = dout + ((d + 63) & ~uint64_t(63));
        ck(cudaMemcpyAsync(dq, q, d * 4, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st), "dense q");
        if (mask) ck(cudaMemcpyAsync(dmask, hm.data(), n * 4, cudaMemcpyHostToDevice, st), "dense mask");
        ck(csa::launch_dense_attention(dq, s->h.kpre, s->h.ktail, s->h.vpre, s->h.vtail, s->h.P,
                                       mask ? dmask : nullptr, static_cast<uint32_t>(n),
                                       static_cast<uint32_t>(d), dout, weights ? dw : nullptr, base, st),
           "dense attention launch");
        const cudaMemcpyKind kind = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (out) ck(cudaMemcpyAsync(out, dout, d * 4, kind, st), "dense out");
        if (weights) ck(cudaMemcpyAsync(weights, dw, n * 4, kind, st), "dense weights");
        ck(cudaStreamSynchronize(st), "dense attention");
        ctx->launches += 5;
    });
}

csattn_status csattn_dense_topk(csattn_session s, const float* q, uint64_t k, uint32_t* out,
                                uint32_t flags) {
    return guard([&] {
        const bool host = flags & CSATTN_HOST_BUFFERS;
        const uint64_t N = s->N, d = s->h.d;
        if (k < 1 || k > N) fail(CSATTN_ERR_PARAMETER, "top-k count out of range: " + std::to_string(k));
        csattn_ctx ctx = s->ctx;
        cudaStream_t st = ctx->stream;
        const size_t scratch = csa::dense_scratch_bytes(static_cast<uint32_t>(N), static_cast<uint32_t>(d));
        ctx->dense.ensure(scratch + d * 4 + k * 4 + 1024);
        char* base = ctx->dense.as<char>();
        float* dq = reinterpret_cast<float*>(base + scratch);
        uint32_t* dout = reinterpret_cast<uint32_t*>(base + scratch + ((d * 4 + 255) & ~size_t(255)));
        ck(cudaMemcpyAsync(dq, q, d * 4, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st), "topk q");
        ck(csa::launch_dense_topk(dq, s->h.kpre, s->h.ktail, s->h.P, static_cast<uint32_t>(N),
                                  static_cast<uint32_t>(d), static_cast<uint32_t>(k), dout, base, scratch, st),
           "dense topk launch");
        ck(cudaMemcpyAsync(out, dout, k * 4, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st),
           "topk out");
        ck(cudaStreamSynchronize(st), "dense topk");
        ctx->launches += 4;
    });
}

// ---------------------------------------------------------------------------
// Function-level API (the reference's free functions on host values,
// index.hpp / retrieval.hpp / core.hpp): inputs are uploaded, the work runs on
// the device with the hot path's arithmetic, results are copied back.
// ---------------------------------------------------------------------------

csattn_status csattn_score_keys(csattn_ctx ctx, const float* centroids, uint64_t n_centroids,
                                const uint64_t* offsets, const uint64_t* widths, const float* keys,
                                uint64_t n, uint64_t d, int32_t normalize, float* out, double* out64) {
    return guard([&] {
        if (normalize < 0 || normalize > 2) fail(CSATTN_ERR_PARAMETER, "normalize mode must be 0, 1 or 2");
        if (n_centroids == 0 || n == 0) return;
        std::vector<uint32_t> coff(n_centroids), kof(n_centroids), wid(n_centroids);
        uint64_t cn = 0;
        for (uint64_t j = 0; j < n_centroids; ++j) {
            if (widths[j] == 0 || offsets[j] + widths[j] > d)
                fail(CSATTN_ERR_DIMENSION, "centroid " + std::to_string(j) + " does not fit the key width");
            coff[j] = static_cast<uint32_t>(cn);
            kof[j] = static_cast<uint32_t>(offsets[j]);
            wid[j] = static_cast<uint32_t>(widths[j]);
            cn += widths[j];
        }
        cudaStream_t st = ctx->stream;
        DevMem dc, dk, dm, dout;
        dc.alloc(cn * 4);
        dk.alloc(n * d * 4);
        dm.alloc(n_centroids * 12);
        dout.alloc(n_centroids * n * (out64 ? 8 : 4));
        uint32_t* m = dm.as<uint32_t>();
        ck(cudaMemcpyAsync(dc.p, centroids, cn * 4, cudaMemcpyHostToDevice, st), "score centroids");
        ck(cudaMemcpyAsync(dk.p, keys, n * d * 4, cudaMemcpyHostToDevice, st), "score keys");
        ck(cudaMemcpyAsync(m, coff.data(), n_centroids * 4, cudaMemcpyHostToDevice, st), "score meta");
        ck(cudaMemcpyAsync(m + n_centroids, kof.data(), n_centroids * 4, cudaMemcpyHostToDevice, st), "score meta");
        ck(cudaMemcpyAsync(m + 2 * n_centroids, wid.data(), n_centroids * 4, cudaMemcpyHostToDevice, st), "score meta");
        ck(csa::launch_score_multi(dc.as<float>(), m, m + n_centroids, m + 2 * n_centroids,
                                   static_cast<uint32_t>(n_centroids), dk.as<float>(), static_cast<uint32_t>(n),
                                   static_cast<uint32_t>(d), normalize, out64 ? nullptr : dout.as<float>(),
                                   out64 ? dout.as<double>() : nullptr, st),
           "score launch");
        if (out64)
            ck(cudaMemcpyAsync(out64, dout.p, n_centroids * n * 8, cudaMemcpyDeviceToHost, st), "score out");
        else
            ck(cudaMemcpyAsync(out, dout.p, n_centroids * n * 4, cudaMemcpyDeviceToHost, st), "score out");
        ck(cudaStreamSynchronize(st), "score keys");
        ctx->launches += 1;
    });
}

csattn_status csattn_toplist_from_scores(csattn_ctx ctx, const float* scores, uint64_t n,
                                         uint64_t capacity, uint32_t* out_indices, float* out_scores,
                                         uint64_t* out_len) {
    return guard([&] {
        const uint64_t keep = std::min(capacity, n);
        *out_len = keep;
        if (keep == 0) return;
        if (n >= 0x7fffffffull) fail(CSATTN_ERR_PARAMETER, "too many scores");
        cudaStream_t st = ctx->stream;
        const size_t sb = csa::toplist_scratch_bytes(static_cast<uint32_t>(n));
        DevMem ds, dsort, scratch;
        ds.alloc(n * 4);
        dsort.alloc(n * 8);
        scratch.alloc(sb);
        ck(cudaMemcpyAsync(ds.p, scores, n * 4, cudaMemcpyHostToDevice, st), "toplist scores");
        ck(csa::launch_toplist(ds.as<float>(), static_cast<uint32_t>(n), dsort.as<unsigned long long>(),
                               scratch.p, sb, st),
           "toplist sort");
        std::vector<unsigned long long> keys(keep);
        ck(cudaMemcpyAsync(keys.data(), dsort.p, keep * 8, cudaMemcpyDeviceToHost, st), "toplist out");
        ck(cudaStreamSynchronize(st), "toplist");
        for (uint64_t r = 0; r < keep; ++r) {
            const uint32_t i = ~static_cast<uint32_t>(keys[r]);
            out_indices[r] = i;
            out_scores[r] = scores[i];
        }
        ctx->launches += 2;
    });
}

csattn_status csattn_select_centroids(csattn_ctx ctx, const float* centroids, uint64_t c,
                                      const uint64_t* widths, uint64_t m, const float* q,
                                      uint64_t tau, double threshold, uint32_t* ids, uint32_t* counts,
                                      double* best_cosine, uint64_t* dot_ops) {
    return guard([&] {
        uint64_t d = 0;
        for (uint64_t b = 0; b < m; ++b) d += widths[b];
        validate_layout(widths, m, d);
        if (c == 0 || c * m > csa::MAX_TABLES) fail(CSATTN_ERR_PARAMETER, "centroid count out of range");
        if (tau == 0) fail(CSATTN_ERR_PARAMETER, "backoff tau must be >= 1");
        const uint64_t take = std::min<uint64_t>(tau, c);
        if (take > static_cast<uint64_t>(csa::MAXTAU))
            fail(CSATTN_ERR_CAPACITY, "backoff tau above " + std::to_string(csa::MAXTAU) + " centroids");
        cudaStream_t st = ctx->stream;
        csa::SessionDev h{};
        h.d = static_cast<uint32_t>(d);
        h.m = static_cast<uint32_t>(m);
        h.C = static_cast<uint32_t>(c);
        uint64_t off = 0;
        for (uint64_t b = 0; b < m; ++b) {
            h.widths[b] = static_cast<uint32_t>(widths[b]);
            h.offs[b] = static_cast<uint32_t>(off);
            h.weights[b] = 1.0;
            off += widths[b];
        }
        h.tau = static_cast<uint32_t>(take);
        h.threshold = threshold;
        h.passthrough = 1;
        const uint64_t T = c * m;
        DevMem dcent, dmeta, dsd, dprob, dplan, drep, dq;
        dcent.alloc(c * d * 4);
        dmeta.alloc(T * 12);  // tmm (float2) + live_g: zero (no tables)
        dsd.alloc(sizeof(csa::SessionDev));
        dprob.alloc(sizeof(csa::DecodeProblem));
        dplan.alloc(sizeof(csa::RoutePlan));
        drep.alloc(sizeof(csa::DecodeReport));
        dq.alloc(d * 4);
        ck(cudaMemsetAsync(dmeta.p, 0, T * 12, st), "route meta");
        h.cent = dcent.as<float>();
        h.tmm = dmeta.as<float2>();
        h.live_g = reinterpret_cast<uint32_t*>(dmeta.as<char>() + T * 8);
        csa::DecodeProblem P{};
        P.s = dsd.as<csa::SessionDev>();
        P.q = dq.as<float>();
        P.rep = drep.as<uint32_t>();
        P.mode = csa::MODE_SEARCH;
        ck(cudaMemcpyAsync(dcent.p, centroids, c * d * 4, cudaMemcpyHostToDevice, st), "route centroids");
        ck(cudaMemcpyAsync(dq.p, q, d * 4, cudaMemcpyHostToDevice, st), "route q");
        ck(cudaMemcpyAsync(dsd.p, &h, sizeof(h), cudaMemcpyHostToDevice, st), "route session");
        ck(cudaMemcpyAsync(dprob.p, &P, sizeof(P), cudaMemcpyHostToDevice, st), "route problem");
        ck(csa::launch_route(dprob.as<csa::DecodeProblem>(), dplan.as<csa::RoutePlan>(), 1, st), "route launch");
        csa::RoutePlan plan;
        csa::DecodeReport rep;
        ck(cudaMemcpyAsync(&plan, dplan.p, sizeof(plan), cudaMemcpyDeviceToHost, st), "route plan");
        ck(cudaMemcpyAsync(&rep, drep.p, sizeof(rep), cudaMemcpyDeviceToHost, st), "route report");
        ck(cudaStreamSynchronize(st), "route");
        for (uint64_t b = 0; b < m; ++b) counts[b] = 0;
        for (uint32_t l = 0; l < plan.nl; ++l) {
            const uint32_t b = plan.lsub[l];
            ids[b * tau + counts[b]] = plan.lists[l] - b * static_cast<uint32_t>(c);
            counts[b] += 1;
        }
        for (uint64_t b = 0; b < m; ++b) best_cosine[b] = rep.best_cos[b];
        *dot_ops = (static_cast<uint64_t>(rep.dot_ops_hi) << 32) | rep.dot_ops_lo;
        ctx->launches += 1;
    });
}

csattn_status csattn_reduce_by_key(csattn_ctx ctx, uint64_t n_lists, const uint64_t* lens,
                                   const uint32_t* const* indices, const float* const* scores,
                                   const double* weights, uint32_t* out_indices, double* out_scores,
                                   uint32_t* out_counts, uint64_t capacity, uint64_t* out_n) {
    return guard([&] {
        std::vector<uint64_t> off(n_lists + 1, 0);
        uint32_t nkeys = 0;
        for (uint64_t l = 0; l < n_lists; ++l) {
            off[l + 1] = off[l] + lens[l];
            for (uint64_t r = 0; r < lens[l]; ++r) nkeys = std::max(nkeys, indices[l][r] + 1);
        }
        const uint64_t E = off[n_lists];
        *out_n = 0;
        if (E == 0) return;
        std::vector<uint32_t> hidx(E);
        std::vector<float> hsc(E);
        for (uint64_t l = 0; l < n_lists; ++l) {
            std::copy(indices[l], indices[l] + lens[l], hidx.begin() + off[l]);
            std::copy(scores[l], scores[l] + lens[l], hsc.begin() + off[l]);
        }
        cudaStream_t st = ctx->stream;
        DevMem doff, didx, dsc, dw, dacc, dcnt;
        doff.alloc(off.size() * 8);
        didx.alloc(E * 4);
        dsc.alloc(E * 4);
        dw.alloc(std::max<uint64_t>(n_lists, 1) * 8);
        dacc.alloc(static_cast<size_t>(nkeys) * 8);
        dcnt.alloc(static_cast<size_t>(nkeys) * 4);
        ck(cudaMemcpyAsync(doff.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st), "reduce offsets");
        ck(cudaMemcpyAsync(didx.p, hidx.data(), E * 4, cudaMemcpyHostToDevice, st), "reduce indices");
        ck(cudaMemcpyAsync(dsc.p, hsc.data(), E * 4, cudaMemcpyHostToDevice, st), "reduce scores");
        ck(cudaMemcpyAsync(dw.p, weights, n_lists * 8, cudaMemcpyHostToDevice, st), "reduce weights");
        ck(csa::launch_reduce_lists(static_cast<uint32_t>(n_lists), doff.as<uint64_t>(), didx.as<uint32_t>(),
                                    dsc.as<float>(), dw.as<double>(), dacc.as<double>(), dcnt.as<uint32_t>(),
                                    nkeys, st),
           "reduce launch");
        std::vector<double> acc(nkeys);
        std::vector<uint32_t> cnt(nkeys);
        ck(cudaMemcpyAsync(acc.data(), dacc.p, nkeys * 8, cudaMemcpyDeviceToHost, st), "reduce out");
        ck(cudaMemcpyAsync(cnt.data(), dcnt.p, nkeys * 4, cudaMemcpyDeviceToHost, st), "reduce counts");
        ck(cudaStreamSynchronize(st), "reduce");
        uint64_t n = 0;
        for (uint32_t i = 0; i < nkeys; ++i) {
            if (!cnt[i]) continue;
            if (n >= capacity) fail(CSATTN_ERR_PARAMETER, "candidate capacity exceeded");
            out_indices[n] = i;
            out_scores[n] = acc[i];
            out_counts[n] = cnt[i];
            ++n;
        }
        *out_n = n;
        ctx->launches += 1;
    });
}

csattn_status csattn_select_topk(csattn_ctx ctx, const uint32_t* cand_indices, const double* cand_scores,
                                 uint64_t n_cand, uint64_t n, const csattn_retrieval_config* rcfg,
                                 uint64_t k_override, uint32_t* out, uint64_t* out_k) {
    return guard([&] {
        if (n == 0) fail(CSATTN_ERR_PARAMETER, "cannot select from an empty context");
        if (n > csa::SELECT_MAX_CONTEXT)
            fail(CSATTN_ERR_CAPACITY, "context of " + std::to_string(n) + " keys exceeds one GPU's decode search");
        const uint64_t K = k_override ? std::min<uint64_t>(k_override, n) : keep_count(rcfg->keep_ratio, n);
        *out_k = K;
        const bool pt = rcfg->recent_passthrough != 0;
        // the dense candidate-score array the select kernel reads in its
        // cached-score mode (search_period reuse), absent keys NaN-boxed
        std::vector<double> dense(n);
        const unsigned long long absent = 0x7ff4deadbeef0000ull;
        double absent_d;
        std::memcpy(&absent_d, &absent, 8);
        std::fill(dense.begin(), dense.end(), absent_d);
        double lo = 0.0, hi = 0.0;
        bool any = false;
        for (uint64_t c = 0; c < n_cand; ++c) {
            if (cand_indices[c] >= n) continue;
            const double v = cand_scores[c];
            dense[cand_indices[c]] = v;
            lo = any ? std::min(lo, v) : v;
            hi = any ? std::max(hi, v) : v;
            any = true;
        }
        if (!pt) {  // window keys compete at 0 when absent
            lo = std::min(lo, 0.0);
            hi = std::max(hi, 0.0);
        }
        cudaStream_t st = ctx->stream;
        csa::SessionDev h{};
        h.window = static_cast<uint32_t>(std::min<uint64_t>(rcfg->recent_window, 0xffffffffull));
        h.passthrough = pt ? 1 : 0;
        const uint64_t log_cap = (n + csa::SELECT_LOG_ALIGN - 1) / csa::SELECT_LOG_ALIGN * csa::SELECT_LOG_ALIGN;
        DevMem dsd, dprob, dplan, drep, dcache, dcb, dsel, dlog_i, dlog_s, dretry;
        dsd.alloc(sizeof(csa::SessionDev));
        dprob.alloc(sizeof(csa::DecodeProblem));
        dplan.alloc(sizeof(csa::RoutePlan));
        drep.alloc(sizeof(csa::DecodeReport));
        dcache.alloc(n * 8);
        dcb.alloc(4 * 8);
        dsel.alloc(K * 4);
        dlog_i.alloc(log_cap * 4);
        dlog_s.alloc(log_cap * 8);
        dretry.alloc(8);
        const double cb[4] = {lo, hi, 0.0, 0.0};  // no speculation hint
        csa::DecodeProblem P{};
        P.s = dsd.as<csa::SessionDev>();
        P.sel = dsel.as<uint32_t>();
        P.cache = dcache.as<double>();
        P.cbounds = dcb.as<double>();
        P.rep = drep.as<uint32_t>();
        P.N = static_cast<uint32_t>(n);
        P.K = static_cast<uint32_t>(K);
        P.n_cache = static_cast<uint32_t>(n);
        P.mode = 0;  // no search: the cached (given) candidate scores
        ck(cudaMemcpyAsync(dsd.p, &h, sizeof(h), cudaMemcpyHostToDevice, st), "topk session");
        ck(cudaMemcpyAsync(dprob.p, &P, sizeof(P), cudaMemcpyHostToDevice, st), "topk problem");
        ck(cudaMemcpyAsync(dcache.p, dense.data(), n * 8, cudaMemcpyHostToDevice, st), "topk candidates");
        ck(cudaMemcpyAsync(dcb.p, cb, sizeof(cb), cudaMemcpyHostToDevice, st), "topk bounds");
        ck(cudaMemsetAsync(dretry.p, 0, 8, st), "topk retry");
        uint32_t* rc = dretry.as<uint32_t>();
        ck(csa::launch_select(dprob.as<csa::DecodeProblem>(), dplan.as<csa::RoutePlan>(), 1, 1,
                              dlog_i.as<uint32_t>(), dlog_s.as<double>(), static_cast<uint32_t>(log_cap),
                              nullptr, nullptr, rc + 1, rc, 0.0, 1, nullptr, st),
           "topk select launch");
        ck(cudaMemcpyAsync(out, dsel.p, K * 4, cudaMemcpyDeviceToHost, st), "topk out");
        ck(cudaStreamSynchronize(st), "select topk");
        ctx->launches += 1;
    });
}

csattn_status csattn_dense_attention_rows(csattn_ctx ctx, const float* q, const float* keys,
                                          const float* values, uint64_t n, uint64_t d,
                                          const uint32_t* mask, uint64_t n_mask, float* out,
                                          float* weights) {
    return guard([&] {
        if (n == 0) fail(CSATTN_ERR_PARAMETER, "attention over an empty KV store");
        uint64_t rows = n;
        if (mask) {
            if (n_mask == 0) fail(CSATTN_ERR_PARAMETER, "attention over an empty index set");
            for (uint64_t r = 0; r < n_mask; ++r)
                if (mask[r] >= n) fail(CSATTN_ERR_PARAMETER, "mask index " + std::to_string(mask[r]) + " out of range");
            rows = n_mask;
        }
        cudaStream_t st = ctx->stream;
        const size_t scratch = csa::dense_scratch_bytes(static_cast<uint32_t>(rows), static_cast<uint32_t>(d));
        DevMem dk, dv, dq, dm, dout, dw, ds;
        dk.alloc(n * d * 4);
        dv.alloc(n * d * 4);
        dq.alloc(d * 4);
        dm.alloc(rows * 4);
        dout.alloc(d * 4);
        dw.alloc(rows * 4);
        ds.alloc(scratch);
        ck(cudaMemcpyAsync(dk.p, keys, n * d * 4, cudaMemcpyHostToDevice, st), "dense keys");
        ck(cudaMemcpyAsync(dv.p, values, n * d * 4, cudaMemcpyHostToDevice, st), "dense values");
        ck(cudaMemcpyAsync(dq.p, q, d * 4, cudaMemcpyHostToDevice, st), "dense q");
        if (mask) ck(cudaMemcpyAsync(dm.p, mask, n_mask * 4, cudaMemcpyHostToDevice, st), "dense mask");
        ck(csa::launch_dense_attention(dq.as<float>(), dk.as<float>(), nullptr, dv.as<float>(), nullptr,
                                       static_cast<uint32_t>(n), mask ? dm.as<uint32_t>() : nullptr,
                                       static_cast<uint32_t>(rows), static_cast<uint32_t>(d), dout.as<float>(),
                                       weights ? dw.as<float>() : nullptr, ds.p, st),
           "dense attention launch");
        if (out) ck(cudaMemcpyAsync(out, dout.p, d * 4, cudaMemcpyDeviceToHost, st), "dense out");
        if (weights) ck(cudaMemcpyAsync(weights, dw.p, rows * 4, cudaMemcpyDeviceToHost, st), "dense weights");
        ck(cudaStreamSynchronize(st), "dense attention");
        ctx->launches += 5;
    });
}

csattn_status csattn_dense_topk_rows(csattn_ctx ctx, const float* q, const float* keys, uint64_t n,
                                     uint64_t d, uint64_t k, uint32_t* out) {
    return guard([&] {
        if (k < 1 || k > n) fail(CSATTN_ERR_PARAMETER, "top-k count out of range: " + std::to_string(k));
        cudaStream_t st = ctx->stream;
        const size_t scratch = csa::dense_scratch_bytes(static_cast<uint32_t>(n), static_cast<uint32_t>(d));
        DevMem dk, dq, dout, ds;
        dk.alloc(n * d * 4);
        dq.alloc(d * 4);
        dout.alloc(k * 4);
        ds.alloc(scratch);
        ck(cudaMemcpyAsync(dk.p, keys, n * d * 4, cudaMemcpyHostToDevice, st), "topk keys");
        ck(cudaMemcpyAsync(dq.p, q, d * 4, cudaMemcpyHostToDevice, st), "topk q");
        ck(csa::launch_dense_topk(dq.as<float>(), dk.as<float>(), nullptr, static_cast<uint32_t>(n),
                                  static_cast<uint32_t>(n), static_cast<uint32_t>(d), static_cast<uint32_t>(k),
                                  dout.as<uint32_t>(), ds.p, scratch, st),
           "dense topk launch");
        ck(cudaMemcpyAsync(out, dout.p, k * 4, cudaMemcpyDeviceToHost, st), "topk out");
        ck(cudaStreamSynchronize(st), "dense topk");
        ctx->launches += 4;
    });
}

void* csattn_ctx_stream(csattn_ctx ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

csattn_status csattn_buffer_add_u32(csattn_ctx ctx, uint32_t* dst, const uint32_t* src, uint64_t count) {
    return guard([&] {
        ck(csa::launch_buf_add_u32(dst, src, count, ctx->stream), "buffer add");
        ctx->launches += count ? 1 : 0;
    });
}

csattn_status csattn_buffer_min_u64(csattn_ctx ctx, uint64_t* dst, const uint64_t* src, uint64_t count) {
    return guard([&] {
        ck(csa::launch_buf_min_u64(reinterpret_cast<unsigned long long*>(dst),
                                   reinterpret_cast<const unsigned long long*>(src), count, ctx->stream),
           "buffer min");
        ctx->launches += count ? 1 : 0;
    });
}

}  // extern "C"
