// common.cuh — device-side data layout of one CSAttention session (one KV head)
// and the per-launch problem descriptors. See DESIGN.md §3 for the HBM layout.
//
// Tables (reference TopList m x C grid, index.hpp:19-68) are stored
// INDEX-SORTED instead of score-sorted, so the decode gather is a coalesced
// range read per key block and the fp64 accumulation is a conflict-free
// shared-memory RMW in a fixed list order:
//   ent[t][0 .. n_used[t])      (key index, f32 score) pairs, ascending key;
//                               evicted entries keep their key with TOMB set
//   blk_off[t][k]               first position with key >= k*KEY_BLOCK
//   low[t][0 .. low_cnt[t])     the lowest live entries in eviction order
//                               (score asc, key desc) = the TopList tail
//                               reversed; eviction pops low[t][0]
//   live[t]                     live entries (= TopList::indices.size())
//   tmm[t]                      (lower bound, upper bound) of the live scores:
//                               the min at build time (evictions only raise
//                               the min) and the running max (inserts raise it)
// A list holds at most L live entries plus LOW_Q tombstones: when the low
// buffer runs dry the list is compacted and the buffer refilled.
#pragma once
#include <cstdint>

namespace csa {

constexpr int KEY_BLOCK_SHIFT = 8;   // blk_off granularity: 256 keys
constexpr int KEY_BLOCK = 1 << KEY_BLOCK_SHIFT;
constexpr int MAXM = 32;             // subspaces
constexpr int MAXTAU = 8;            // backoff centroids per subspace
constexpr int MAXL = 64;             // gathered lists per query (m * tau)
constexpr int DMAX = 512;            // head dim
constexpr int WMAX = 64;             // subspace width
constexpr int LOW_Q = 256;           // low-buffer depth = tombstone slack
constexpr int MAX_TABLES = 2048;     // m * C
constexpr uint32_t TOMB = 0x80000000u;
constexpr uint32_t MAX_CONTEXT = 0x7fffffffu;

struct LowEnt {
    float score;
    uint32_t key;
    uint32_t pos;  // position in ent[t]
    uint32_t pad;
};

// Device-resident constants and buffers of one session (KV head).
struct SessionDev {
    uint32_t d, m, C, L;
    uint32_t cap2;       // per-list entry capacity = L + LOW_Q
    uint32_t nb_stride;  // blk_off entries per list
    uint32_t P, max_ctx;
    uint32_t widths[MAXM];
    uint32_t offs[MAXM];
    uint32_t normalize_keys;
    uint32_t tau;
    uint32_t window;
    uint32_t passthrough;
    double weights[MAXM];
    double threshold;
    // KV rows: [0, P) in kpre/vpre (shared across forks), [P, max_ctx) in tails
    const float* kpre;
    const float* vpre;
    float* ktail;
    float* vtail;
    const float* cent;  // C*d, packed per subspace: (b, j) at C*offs[b] + j*widths[b]
    uint2* ent;         // [T][cap2] {key, f32 bits}
    uint32_t* n_used;   // [T]
    uint32_t* live;     // [T]
    uint32_t* blk_off;  // [T][nb_stride]
    LowEnt* low;        // [T][LOW_Q]
    uint32_t* low_cnt;  // [T]
    uint32_t* refill;   // [T] scratch flags for the insert kernel
    float2* tmm;        // [T] live score bounds (min lower bound, max) of the GLOBAL list
    // Sequence sharding: a shard holds the keys [key_lo, key_hi)
    // of the global lists (global indices kept) and of the prefill KV rows;
    // `owner` shards also hold appended keys (index >= P). live_g[t] is the
    // global live count of list t, replicated on every shard (== live when the
    // session is not sharded). kpre/vpre are offset so row i is kpre[i*d].
    uint32_t key_lo, key_hi, owner, sharded;
    uint32_t* live_g;   // [T]
};

// Per-(session, query head) decode-step descriptor.
struct DecodeProblem {
    const SessionDev* s;
    const float* q;
    float* out;        // d floats
    float* weights;    // K floats (nullable)
    uint32_t* sel;     // K entries (scratch or caller buffer)
    double* cache;     // candidate-score cache for search_period > 1 (nullable)
    double* cbounds;   // [lo, hi] of the cached search, [threshold hint, hint valid]
    uint32_t* rep;     // DecodeReport (device)
    uint32_t N;        // context this step attends to (pre-append)
    uint32_t K;        // selected-set size
    uint32_t n_cache;  // context length when the cache was filled
    uint32_t mode;     // MODE_* bits
    unsigned long long* prof;  // phase timestamps [cs][8] (CSATTN_PHASE_PROF) or null
    uint32_t tile_lo, tile_hi;  // select tiles of this shard (tile_hi == 0: all)
    const uint32_t* kdev;       // sharded steps: this shard's selection sizes (emit output)
};
constexpr uint32_t MODE_SEARCH = 1u;       // route + gather + accumulate
constexpr uint32_t MODE_STORE_CACHE = 2u;  // persist candidate scores
constexpr uint32_t MODE_WEIGHTS = 4u;      // emit softmax weights
constexpr uint32_t MODE_PARTIAL = 8u;      // attend writes (max, sum, acc[d]) unnormalised

// Device report written by CTA 0 of a problem (uint32 words).
struct DecodeReport {
    uint32_t k;
    uint32_t nl;                 // gathered lists
    uint32_t dot_ops_lo, dot_ops_hi;
    uint32_t gathered_lo, gathered_hi;
    uint32_t pad[2];
    double best_cos[MAXM];
    uint32_t lists[MAXL];        // table ids gathered, in order
};

// Routing result of one problem (route.cu -> select.cu): the gathered lists
// and bounds [lo, hi] on every accumulated candidate score (from the lists'
// score bounds), which fix the selection histogram before the gather starts.
struct RoutePlan {
    uint32_t nl;
    uint32_t pad[3];
    double lo, hi;
    uint32_t lists[MAXL];               // table ids, gathered order
    uint32_t lsub[MAXL];                // their subspaces
};

// Per-session append + insert descriptor.
struct InsertProblem {
    const SessionDev* s;
    const float* key;
    const float* value;
    uint32_t* rep;     // InsertReport: applied count + mask (T bytes)
    uint32_t* bad;     // set to 1 when the row is non-finite (KvStore::append's
                       // DataError, core.cpp:71-79): nothing is appended or inserted
    uint32_t N;        // key index of the appended row (= pre-append N)
    uint32_t pad;
};

__host__ __device__ inline uint32_t div_up(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

}  // namespace csa
