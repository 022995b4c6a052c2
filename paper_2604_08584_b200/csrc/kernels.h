// kernels.h — host-callable launchers of the sm_100a kernels (csrc/*.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace csa {

// route.cu: centroid routing + score bounds, one CTA per problem
// trig: where a programmatically launched select may start (1: at the CTA's
// start, 2: once its lists are known, 0: at its exit)
cudaError_t launch_route(const DecodeProblem* probs, RoutePlan* plans, uint32_t nprob,
                         cudaStream_t st, int trig = 0);

// select.cu: streaming gather + top-K, persistent (one CTA per SM, problems
// strided over the grid). log_idx/log_sc: grid x log_cap candidate-log slots.
constexpr uint32_t SELECT_MAX_CONTEXT = 4096u * 64u;  // bitmap aliases the tile accumulator
constexpr uint32_t SELECT_LOG_ALIGN = 4096u;           // log_cap multiple (per-warp regions)
uint32_t select_grid(uint32_t nprob, int num_sms);
//   retry_in/retry_in_count: when non-null, process only the listed problems,
//   without speculation (the second pass); retry_out/retry_out_count: where the
//   first pass lists problems whose speculative cut proved too high.
// Mixed mode (tail split): when the problems do not fill whole rounds of
// the grid, every CTA takes its whole problems and then a contiguous piece
// of the remaining problems' tiles. items[i] = (problem, tile_lo, tile_hi,
// slot), slot = NO_SLOT for a whole problem; CTA c owns items
// [cta_items[c], cta_items[c+1]). A piece dumps its histogram + per-warp log
// lengths to umeta[slot] and its log to plog at slotinfo[slot] = (offset,
// per-warp stride); pinfo[p] = (first slot, pieces) of a split problem; the
// CTA whose atomicAdd on pdone[p] completes the count merges and finalises
// it (pdone must start at zero; the finaliser resets it).
constexpr uint32_t NO_SLOT = 0xffffffffu;
constexpr uint32_t SELECT_MAX_PART = 16;      // pieces per problem (seg tables)
constexpr uint32_t SELECT_CONSUMER_WARPS = 8;  // per-warp log regions
struct SelMixed {
    const uint4* items = nullptr;
    const uint32_t* cta_items = nullptr;
    const uint2* pinfo = nullptr;
    const uint2* slotinfo = nullptr;
    uint32_t* pdone = nullptr;
    uint32_t* plog_idx = nullptr;
    double* plog_sc = nullptr;
    uint32_t* umeta = nullptr;
};
cudaError_t launch_select(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                          uint32_t grid, uint32_t* log_idx, double* log_sc, uint32_t log_cap,
                          const uint32_t* retry_in, const uint32_t* retry_in_count,
                          uint32_t* retry_out, uint32_t* retry_out_count, double spec_keep,
                          uint32_t split, uint32_t* unit_meta, cudaStream_t st,
                          const SelMixed* mixed = nullptr, bool pdl = false);
// pdl: launched as a programmatic dependent of the previous kernel in the
// stream (the route launch): its CTAs start, and run their shared-memory
// prologue, while route finishes; they wait (griddepcontrol.wait) before the
// first read of the route plans.
// split > 1: each problem's tiles are cut into `split` part units (logs of
// log_cap entries each, unit_meta: select_unit_meta_words() per unit) and
// finalised by the merge kernel (one CTA per problem).
uint32_t select_unit_meta_words();
uint32_t select_ctas_per_sm();  // resident select CTAs per SM (grid = this x SMs)
// CSATTN_PHASE_PROF only: the final-selection stage times (ns, summed over
// problems; [6] = problem count) accumulated since the library loaded.
// CSATTN_PHASE_PROF: per select CTA (start, end) globaltimer stamps of the last launch
cudaError_t select_cta_times(unsigned long long* out, uint32_t n, cudaStream_t st);
cudaError_t select_fin_debug(unsigned long long* out8, cudaStream_t st);
uint32_t select_tile_keys();
cudaError_t launch_select_merge(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                                uint32_t split, const uint32_t* unit_meta, const uint32_t* log_idx,
                                const double* log_sc, uint32_t log_cap, double spec_keep,
                                uint32_t* retry_out, uint32_t* retry_out_count, cudaStream_t st);

// select.cu, sequence-sharded decode phases (see select.cu)
uint32_t shard_bucket_words();  // per problem, uint32 words of a bucket record
uint32_t shard_hist_words();    // per problem histogram words (all-reduced)
uint32_t shard_pstate_bytes();
cudaError_t launch_shard_hist_sum(const uint32_t* unit_meta, uint32_t nprob, uint32_t split,
                                  uint32_t* ghist, cudaStream_t st);
cudaError_t launch_shard_bucket(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                                const uint32_t* ghist, const uint32_t* unit_meta,
                                const uint32_t* log_idx, const double* log_sc, uint32_t log_cap,
                                uint32_t split, void* bucket, void* pstate, double spec_keep,
                                uint32_t* spec_fail, cudaStream_t st);
cudaError_t launch_shard_mark(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                              const void* pstate, const void* bucket_all, uint32_t nshard,
                              const uint32_t* unit_meta, const uint32_t* log_idx,
                              const double* log_sc, uint32_t log_cap, uint32_t split,
                              uint32_t* bitmap, uint32_t bm_words, uint32_t* counts,
                              cudaStream_t st);
cudaError_t launch_shard_emit(const DecodeProblem* probs, const RoutePlan* plans, uint32_t nprob,
                              const uint32_t* counts_all, uint32_t nshard, uint32_t shard,
                              uint32_t* bitmap, uint32_t bm_words, uint32_t* kdev, cudaStream_t st);

// fused.cu: the whole decode search + attention of a problem in one CTA
// cluster (small batches); fused_fits picks the cluster size and the 512-key
// ranges per CTA for N keys
bool fused_fits(uint32_t N, uint32_t d, int& cl, int& nr);
cudaError_t launch_fused_step(const DecodeProblem* probs, uint32_t nprob, int cl, int nr, cudaStream_t st);

// attend.cu: split-K sparse attention over the selected rows, ATT_ROWS per CTA
constexpr uint32_t ATT_ROWS = 256;      // rows per chunk-CTA (mid-size launches)
constexpr uint32_t ATT_ROWS_BIG = 512;  // from ~7 CTAs per SM of 256-row chunks (c3; c3 on 4 / 8 GPUs)
constexpr uint32_t ATT_ROWS_SMALL = 128;  // when they would give < 2 CTAs per SM (c2)
// rows per chunk-CTA for a launch whose 256-row chunking has n256 chunks
// (measured with GR = 8 at 7 CTAs/SM: c3 on 8 GPUs' share, 1664 chunks, 51 ->
// 43 us with 512 rows; c4's 832 chunks per layer stay faster at 256)
inline uint32_t attend_rows(uint64_t n256) {
    return n256 > 148ull * 7 ? ATT_ROWS_BIG : (n256 < 148ull * 2 ? ATT_ROWS_SMALL : ATT_ROWS);
}
cudaError_t launch_attend(const DecodeProblem* probs, const uint32_t* chunk_prob,
                          const uint32_t* chunk_base, uint32_t nchunks, float* part,
                          uint32_t* counters, uint32_t d, cudaStream_t st, bool partial = false,
                          uint32_t rows = ATT_ROWS, bool warp_heads = false);

// attend_union.cu: problems sharing a prefill (groups of <= UN_GROUP
// members), by prefill row range: each union row is read once per group
constexpr uint32_t UN_GROUP = 64;
constexpr uint32_t UN_RANGE = 2048;
constexpr uint32_t UN_MAX_RANGES = SELECT_MAX_CONTEXT / UN_RANGE;
constexpr uint32_t UN_PART_WORDS = 132;  // max, sum, 2 pad, acc[128] (16-byte aligned)
cudaError_t launch_attend_union(const DecodeProblem* probs, uint32_t ngroups, const uint32_t* gP,
                                const uint32_t* gmember, const uint32_t* members,
                                const uint32_t* mgroup, uint32_t nmembers, uint32_t nrange,
                                uint16_t* urow, unsigned long long* umask, uint32_t* ucount,
                                float* parts, float* tails, int num_sms, unsigned long long* tprof,
                                cudaStream_t st);

// dense.cu: the dense oracle (masked/full dense_attention, dense_topk)
size_t dense_scratch_bytes(uint32_t n, uint32_t d);
cudaError_t launch_dense_attention(const float* q, const float* kpre, const float* ktail, const float* vpre,
                                   const float* vtail, uint32_t P, const uint32_t* mask, uint32_t n,
                                   uint32_t d, float* out, float* weights, void* scratch, cudaStream_t st);
cudaError_t launch_dense_topk(const float* q, const float* kpre, const float* ktail, uint32_t P, uint32_t n,
                              uint32_t d, uint32_t k, uint32_t* out, void* scratch, size_t scratch_bytes,
                              cudaStream_t st);

// csat_dev.cu: the tables section of a CSAT v1 image, written on the device
size_t csat_sort_temp_bytes(uint32_t ntables, uint32_t cap2);
cudaError_t launch_csat_tables(const uint2* ent, const uint32_t* n_used, const uint32_t* live,
                               uint32_t ntables, uint32_t cap2, const int* seg_begin, const int* seg_end,
                               const unsigned long long* off, int half, unsigned long long* keys,
                               unsigned long long* sorted, void* temp, size_t temp_bytes,
                               unsigned char* out, cudaStream_t st);

cudaError_t launch_shard_merge(const float* parts, uint32_t nshard, uint32_t nprob, uint32_t d,
                               float* out, cudaStream_t st);

// insert.cu: append + streaming insert, one CTA per session
//   gvk: sharded sessions only, per session x table the global victim key
//   pdl: a programmatic dependent of the previous kernel (the fused step): the
//   key's scores and the table state are read while that kernel finishes; the
//   table writes wait for it (griddepcontrol.wait)
cudaError_t launch_insert(const InsertProblem* probs, uint32_t nprob, cudaStream_t st,
                          const unsigned long long* gvk = nullptr, bool pdl = false);
cudaError_t launch_shard_victim(const InsertProblem* probs, uint32_t nprob,
                                unsigned long long* vk, cudaStream_t st);

// build.cu: exact fp64 centroid x key scores and top-L tables
//   scores: T x P floats scratch
cudaError_t launch_build_scores(const SessionDev* s_dev, const SessionDev& s_host, float* scores,
                                cudaStream_t st);
cudaError_t launch_shard_extract(const SessionDev* full_dev, const SessionDev* shard_dev,
                                 uint32_t tables, uint32_t key_lo, uint32_t key_hi, cudaStream_t st);
cudaError_t launch_build_lists(const SessionDev* s_dev, const SessionDev& s_host,
                               const float* scores, cudaStream_t st);
// tcgen05 screen + exact rescore build (build_tc.cu): eligibility (layout,
// sizes, driver entry point), scratch size, and the 4-kernel launch; fail_dev
// counts tables whose screen was inconclusive (the host then rebuilds with
// build_scores/build_lists).
bool build_tc_eligible(const SessionDev& sh);
size_t build_tc_scratch_bytes(const SessionDev& sh, uint32_t* cap_out);
cudaError_t launch_build_tc(const SessionDev* s_dev, const SessionDev& sh, void* scratch, float qmargin,
                            uint32_t* fail_dev, cudaStream_t st);


// fnapi.cu: the function-level API kernels (score_keys / streaming_insert
// scoring, reduce_by_key, TopList::from_scores)
cudaError_t launch_score_multi(const float* cent, const uint32_t* coff, const uint32_t* kof,
                               const uint32_t* wid, uint32_t ncent, const float* keys, uint32_t n,
                               uint32_t d, int mode, float* out, double* out64, cudaStream_t st);
cudaError_t launch_reduce_lists(uint32_t nl, const uint64_t* off, const uint32_t* idx, const float* sc,
                                const double* w, double* acc, uint32_t* cnt, uint32_t nkeys,
                                cudaStream_t st);
size_t toplist_scratch_bytes(uint32_t n);
// shard collectives' local combine steps (csattn_buffer_add_u32 / _min_u64)
cudaError_t launch_buf_add_u32(uint32_t* dst, const uint32_t* src, uint64_t n, cudaStream_t st);
// up to 4 copies in one kernel (device-accessible sources, e.g. pinned host memory)
cudaError_t launch_copy_segs(const void* const* src, void* const* dst, const uint64_t* bytes, uint32_t n,
                             cudaStream_t st);
cudaError_t launch_buf_min_u64(unsigned long long* dst, const unsigned long long* src, uint64_t n, cudaStream_t st);
cudaError_t launch_toplist(const float* scores, uint32_t n, unsigned long long* sorted, void* scratch,
                           size_t scratch_bytes, cudaStream_t st);

}  // namespace csa
