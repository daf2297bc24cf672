// kernels.cuh -- host-side launchers of the device kernels (internal).
#pragma once

#include "common.cuh"

namespace cafs {

constexpr u32 kSmallSortMax = 8192;  // single-CTA sort capacity (keys or pairs)
constexpr u32 kBitonicMax = 2048;    // below this a bitonic network replaces the radix passes
constexpr u64 kExpectCtlN = ~0ull - 1;  // pair-sort `expect`: the sharded column's N (ctl)

// estimate.cu
// `kk`: key kind (common.cuh): 0 = 64-bit, 1 = int32, 2 = uint32
// opts: kEstHp (the partitioned count may run), kEstNoWindow (no dense window),
// kEstForceMain (a tiny route becomes MAIN with the same estimate: the re-entry
// after a tiny miss, sorter.py:378-385)
enum : int { kEstHp = 1, kEstNoWindow = 2, kEstForceMain = 4 };
void launch_estimate(const void* x, u64 n, u64 flip, int check_prefix, DevCtl* ctl,
                     cudaStream_t st, int kk = 0, int opts = 0);
void launch_monotone_scan(const void* x, u64 n, u64 flip, DevCtl* ctl, int num_sms,
                          cudaStream_t st, int kk = 0);
void launch_estimate_sharded(const u64* samples, const u64* ghdr, int world, DevCtl* ctl,
                             cudaStream_t st, int opts = 0);
// shard.cu: the stream-ordered sharded pipeline's own kernels
void launch_shard_header(const void* x, u64 n, u64 flip, u64* hdr, int num_sms, cudaStream_t st,
                         int kk = 0);
void launch_shard_samples(const void* x, u64 n, u64 flip, const u64* ghdr, int world, int rank,
                          u64* samples, DevCtl* ctl, cudaStream_t st, int kk = 0);
void launch_shard_tiny_pack(const DevCtl* ctl, u64* out, cudaStream_t st);
void launch_shard_pack_pairs(DevCtl* ctl, const u64* keys, const u64* cnts, u64* send,
                             u64 cap, cudaStream_t st, int from_local = 0);
void launch_shard_merge_check(DevCtl* ctl, const u64* recv, int world, u64 cap, u64 row,
                              cudaStream_t st);
void launch_shard_tiny_finish(DevCtl* ctl, const u64* tiny_sum, u64* pkeys, u64* pcnt, u64* poffs,
                              cudaStream_t st);
void launch_shard_merge(DevCtl* ctl, const u64* recv, int world, u64 cap, u64 row, u64* gkeys,
                        u64* gcnt, u32* glist, int num_sms, cudaStream_t st);
void launch_shard_tiny_gather(const u64* recv, int world, u64 row, u64 tiny_off, u64* tiny_sum,
                              cudaStream_t st);
// tiny.cu
// with pkeys != null the count's last CTA also writes the tiny route's pairs
// and offsets (or flags the miss): the finalize of sorter.py:367-385
void launch_tiny_count(const void* x, u64 n, u64 flip, DevCtl* ctl, int num_sms, cudaStream_t st,
                       int gate, int kk = 0, u64* pkeys = nullptr, u64* pcnt = nullptr,
                       u64* poffs = nullptr);
// hashcount.cu
cudaError_t launch_hash_count(const void* x, u64 n, u64 flip, u64 mult, DevCtl* ctl, u64* gkeys,
                              u64* gcnt, u32* glist, int use_range, int num_sms, cudaStream_t st,
                              int variant, int gate, u64* dense, int kk = 0);
void launch_dense_pairs(DevCtl* ctl, u64* dense, u64* pkeys, u64* pcnt, u64* skeys, u64* scnt,
                        u64* soffs, u64 n_expect, cudaStream_t st, int gate);
size_t dense_window_len();
void launch_insert_pairs(const u64* keys, const u64* cnts, u64 m, u64 mult, DevCtl* ctl,
                         u64* gkeys, u64* gcnt, u32* glist, int num_sms, cudaStream_t st);
void launch_compact(DevCtl* ctl, u64* gkeys, u64* gcnt, const u32* glist, u64* pkeys, u64* pcnt,
                    int num_sms, cudaStream_t st, int gate);
// hashpart.cu: the partitioned count (no dense window) -> sorted pairs
struct HpBufs {
  void* part;     // partitioned spill: n keys of the column's type
  void* scratch;  // hp_scratch_bytes(num_sms): cells, segment tables, partition totals
  u64* pk_stage;  // kHpParts x 4097 staged pairs (keys, counts)
  u64* pc_stage;
};
size_t hp_scratch_bytes(int num_sms);
// tile_pair: the emit's tile -> pair map for the whole column (null: not written)
cudaError_t launch_hp_count(const HpBufs& b, const void* x, u64 n, u64 flip, DevCtl* ctl, u64* pk,
                            u64* pc, u64* poffs, int num_sms, cudaStream_t st, int gate, int kk,
                            u32* tile_pair = nullptr);
cudaError_t launch_hp_shard_merge(const HpBufs& b, const u64* recv, int world, u64 cap, u64 row,
                                  DevCtl* ctl, u64* pk, u64* pc, u64* poffs, cudaStream_t st);
void launch_hp_restore(const HpBufs& b, void* x, u64 n, u64 flip, int num_sms, cudaStream_t st,
                       int kk);
// emit.cu
void launch_emit(const u64* keys, const u64* offs, u64 npairs, const DevCtl* ctl, void* out,
                 u64 begin, u64 end, u64 flip, int num_sms, cudaStream_t st, u64 npairs_bound,
                 int kk = 0, bool ctl_slice = false, const u32* tile_pair = nullptr);
u64 emit_tiles(u64 L, int kk);
void launch_emit_map(const u64* offs, const DevCtl* ctl, const void* out, u64 begin, u64 end,
                     u32* tile_pair, u64 npairs_bound, int num_sms, cudaStream_t st, int kk);
// radix.cu
size_t onesweep_smem(bool has_val);
u64 onesweep_tiles(u64 n);
void launch_radix_hist(const u64* keys, u64 n, u64 flip, u32* ghist, int num_sms,
                       cudaStream_t st);
void launch_radix_prep(const u32* ghist, u64 n, u32* gbase, int* trivial, cudaStream_t st);
cudaError_t launch_onesweep(const u64* src, const u64* srcv, u64* dst, u64* dstv, u64 n, int pass,
                            u64 flip_in, u64 flip_out, const u32* gbase, u64* tile_state,
                            u32* tile_counter, u32 epoch, cudaStream_t st);
size_t small_sort_smem();
cudaError_t launch_small_sort_keys(u64* keys, u64 n, u64 flip, cudaStream_t st);
cudaError_t launch_small_sort_pairs(u64* keys, const u64* cnt, u64 n, DevCtl* ctl, u64 expect,
                                    u64* out_keys, u64* out_cnt, u64* out_offs, cudaStream_t st,
                                    int gate, u64* gkeys = nullptr, u64* gcnt = nullptr,
                                    const u32* glist = nullptr);  // table given: gather mode (no
                                                                  // compaction kernel before it)
void launch_scan(const u64* in, u64 n, u64* bsum, u64* out_offs, DevCtl* ctl, u64 expect,
                 cudaStream_t st);
// msd.cu
size_t msd_state_bytes();
u32 msd_bucket_cap();
size_t msd_maxb_offset();
size_t msd_overflow_offset();
size_t msd_span_offset();
size_t msd_hist_offset();
void launch_msd_span(const u64* keys, u64 n, u64 flip, void* state, int num_sms, cudaStream_t st);
void launch_msd_partition(const u64* keys, u64 n, u64 flip, void* state, u64 kmin, u64 kmax,
                          u64* out, int num_sms, cudaStream_t st);
bool launch_msd_count(const u64* keys, u64 n, u64 flip, void* state, int num_sms, cudaStream_t st);
void launch_msd_sort(const u64* keys, const u64* vals, u64 n, u64 flip, void* state, u64* tk,
                     u64* tv, u64* dk, u64* dv, u32 maxb, int num_sms, cudaStream_t st);
// telemetry.cu
size_t tel_accum_bytes();
void launch_tel_build(const u64* keys, u64 np, u64* tkeys, u32* tidx, int log2s, u32* first,
                      u32* runs, void* acc, int num_sms, cudaStream_t st);
void launch_tel_runs(const void* x, u64 n, u64 flip, const u64* tkeys, const u32* tidx, int log2s,
                     u32* first, u32* runs, void* acc, int num_sms, cudaStream_t st, int kk = 0);
void launch_tel_comp(const u64* keys, u64 np, const u32* first, u64 mult, int m_log2, int dom,
                     u64* comp, u64* cidx, int num_sms, cudaStream_t st);
void launch_tel_classify(const u64* comp, const u64* cidx, u64 np, int cap, const u64* counts,
                         const u32* runs, void* acc, int num_sms, cudaStream_t st);
// convert (gen.cu): 32-bit keys <-> their int64 widening, for the host-driven
// fallback routes of a 32-bit column
void launch_widen(const void* x, u64 n, int kk, u64* out, int num_sms, cudaStream_t st);
void launch_narrow(const u64* x, u64 n, int kk, void* out, int num_sms, cudaStream_t st);
// gen.cu
void launch_gen_mix(u64* out, u64 count, u64 seed, u64 skip, int num_sms, cudaStream_t st);
void launch_gen_draw(u64* out, u64 n, u64 start, u64 seed, const u64* palette, u64 k,
                     const double* cdf, int num_sms, cudaStream_t st);

}  // namespace cafs
