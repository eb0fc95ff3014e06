// Kernel argument blocks and launchers of the training step.
#pragma once
#include "internal.cuh"
#include "rng.cuh"

namespace slide {

struct SelectArgs {
  TablesDev tab;
  const uint32_t* qkeys;  // (B, L) query keys
  const uint8_t* order;   // (B, L) vanilla probe order
  const int32_t* y_ptr;
  const int32_t* y_idx;
  int b, l, strategy, beta, min_freq, sort_bits;
  int64_t cap_max;
  int32_t* act;
  int32_t* cnt;
  int32_t* empty;
  unsigned long long* cand_ctr;  // optional: total probed bucket slots
  // column-sharded tables: a rank's buckets hold only its own
  // ids, so the sampler's global quantities are sums over ranks.  Phase 1
  // (hist_out set): write per sample (L + 1) counts -- [p] distinct ids
  // first seen at probe position p (vanilla), [L] ids the rule selects
  // without a global threshold (vanilla / full union: every distinct id;
  // hard_threshold: freq >= min_freq) -- and stop.  Phase 2 (ghist set):
  // the all-reduced counts decide vanilla's stop position and emptiness.
  int32_t* hist_out = nullptr;
  const int32_t* ghist = nullptr;
  // two-pass selection (launch_select): 1 = small-capacity pass flagging the
  // samples it cannot hold in big[], 2 = full-size pass over the flagged ones
  int tier = 0;
  int32_t* big = nullptr;
};

struct FallbackArgs {
  const int32_t* empty;
  uint64_t* states;
  int states_ready;  // 0: derive default_rng((seed, iteration, slot)) (+ permutation(L) if vanilla)
  uint64_t seed;
  int64_t iteration, slot_offset;
  const int64_t* iter_dev;  // when set, overrides iteration (graph replays)
  int l, vanilla;
  int64_t n, want;
  int64_t* fb_ids;
  int64_t* scratch;
  int64_t scratch_per_slot;
  int smem_scratch;
  uint32_t* bitmap;
  int64_t words;
  const int32_t* y_ptr;
  const int32_t* y_idx;
  int64_t cap_max;
  int32_t* act;
  int32_t* cnt;
  // the slot stream's outputs made in parallel (rng.cuh PcgBuf): rng_n per
  // slot; in shared memory when rng_n <= kFbSmemOutputs, else rng_buf + i * rng_n
  uint64_t* rng_buf;
  int rng_n;
  const u128* jump;  // pcg_jump_table()
};
constexpr int kFbSmemOutputs = 1024;

void launch_slot_rng(int b, uint64_t seed, int64_t it, const int64_t* it_dev, int64_t off, int l, int vanilla,
                     const uint64_t* ext, uint64_t* states, uint8_t* order, cudaStream_t s);
void launch_select(const SelectArgs& a, int max_candidates, cudaStream_t s, int64_t expected = 1 << 30,
                   int32_t* big = nullptr);
// full-union selection through a shared-memory id bitmap; false if N is too wide
bool launch_select_union(const SelectArgs& a, int64_t n_out, cudaStream_t s);
void launch_fallback(const FallbackArgs& a, int b, cudaStream_t s);
void launch_sample_lists(const int32_t* ptr, const int32_t* ids, int n_tables, int width, int strategy, int beta,
                         int min_freq, const int32_t* order, int32_t* freq, uint32_t* seen, int32_t* out,
                         int32_t* result, cudaStream_t s);
void launch_explicit_active(int b, int64_t n, const int32_t* fptr, const int32_t* fidx, const int32_t* y_ptr,
                            const int32_t* y_idx, int64_t cap_max, int32_t* act, int32_t* cnt, int32_t* empty,
                            cudaStream_t s);
// pair lists from the per-slot active sets; also writes offs (B + 1) from cnt
// mark (optional, unsharded dense row grouping): the pairs' bits in the row
// slot masks and the scan tiles reset -- the grouping's first pass fused in
void launch_pairs(int b, const int32_t* act, int64_t cap_max, const int32_t* cnt, int32_t* offs, int shard_count,
                  int32_t* prow, int32_t* pslot, uint8_t* plab, cudaStream_t s, uint32_t* mark_mask = nullptr,
                  int mark_wpk = 0, unsigned long long* mark_status = nullptr, int32_t* mark_ctr = nullptr,
                  int64_t mark_tiles = 0, uint32_t* mark_lmask = nullptr);
void launch_counts_to_f64(int b, const int32_t* cnt, double* out, cudaStream_t s);
void launch_own_filter(int b, int32_t* act, int64_t cap_max, int g, int G, int32_t* cnt, int32_t* cnt_all,
                       cudaStream_t s);
// sharded softmax phases (per sample over the owned pairs)
void launch_softmax_max(int b, const int32_t* offs, const float* z, float* out, cudaStream_t s);
void launch_softmax_sum(int b, const int32_t* offs, const float* z, const float* gmax, float* out, cudaStream_t s);
void launch_softmax_finish(int b, const int32_t* offs, const uint8_t* plab, const int32_t* y_ptr, const float* z,
                           const float* gmax, const float* gsum, float* prob, float* delta, double* loss_part,
                           const int32_t* inv, float* dsort, cudaStream_t s);

// Stable (key, slot) group-by with device-side sizes (group.cu).
// the group-by result a kernel walks (device pointers)
struct GroupView {
  const int32_t *n_uniq, *uniq, *seg_off, *seg_cnt, *order;
  const uint32_t* mask;  // slot masks: row u (bitmap mode) or row uniq[u] (dense mode)
  int wpk;
  int64_t u_max;
  int mask_by_key;
  const int32_t* sslot;  // slot of each sorted position (placed groupings), else null
  // dense groupings: key_rank[key] = the key's first sorted position, so an
  // item's position follows from its key's mask (place-free consumers)
  const int32_t* key_rank;
  __device__ __forceinline__ const uint32_t* mask_of(int64_t u) const {
    return mask + (mask_by_key ? (int64_t)uniq[u] : u) * wpk;
  }
  // sorted position of item (key, slot), dense mode
  __device__ __forceinline__ int pos_of(int key, int slot) const {
    const uint32_t* mk = mask + (int64_t)key * wpk;
    const int w = slot >> 5;
    const uint32_t lo = (1u << (slot & 31)) - 1u;
    const int base = __ldg(key_rank + key);
    if (wpk == 4) {  // B <= 128: the key's whole mask in one 16-byte load
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(mk));
      return base + (w > 0 ? __popc(v.x) : __popc(v.x & lo)) + (w > 1 ? __popc(v.y) : w == 1 ? __popc(v.y & lo) : 0) +
             (w > 2 ? __popc(v.z) : w == 2 ? __popc(v.z & lo) : 0) + (w == 3 ? __popc(v.w & lo) : 0);
    }
    int r = __popc(__ldg(mk + w) & lo);
    for (int q = 0; q < w; ++q) r += __popc(__ldg(mk + q));
    return base + r;
  }
};

struct LongList {
  int32_t* list;
  int32_t* n;
  int min_len;
};

struct GroupBy {
  DBuf bits, key_rank, uniq, seg_cnt, seg_off, n_uniq, mask, order, status, ctrs;
  // long_min >= 0: run() also lists the segments with more than long_min
  // items (long_list[0 .. *n_long), unordered)
  int long_min = -1;
  DBuf long_list, n_long;
  // want_inv: also inv[q] = sorted position of item q and sslot[pos] = its slot
  bool want_inv = false;
  // dense mode only: premarked -- the caller filled the masks and reset the
  // scan tiles (mark_args()); place = false -- no placement pass, the
  // consumers derive positions from the masks (GroupView::pos_of)
  bool premarked = false, place = true;
  // expected item count (0: use the bound): the dense mode scans every key's
  // mask, worth it only when the items are not much sparser than the keys
  int64_t items_hint = 0;
  // dense mode: a second mask per key marking the items that are labels
  // (the lazy softmax, see capi.cu); filled by the caller's marking pass
  bool want_lmask = false;
  DBuf lmask;
  int64_t lmask_words = 0;
  DBuf inv, sslot;
  int64_t K = 0, nwords = 0, u_max = 0, bits_words = 0, mask_words = 0, tiles_bits = 0, tiles_seg = 0;
  int wpk = 1;
  bool dense = false, mask_dense = false;  // dense: one mask per key of the whole key space
  void prepare(int64_t key_space, int64_t slots, int64_t items_max);
  // items q < n (n = *n_dev if given, else n_host), keys[q] / slots[q]
  void run(const int32_t* keys, const int32_t* slots, const int32_t* n_dev, int64_t n_host, int64_t n_max,
           cudaStream_t s);
  void clear(cudaStream_t s);
  void release();
  GroupView view() {
    return GroupView{n_uniq.as<int32_t>(), uniq.as<int32_t>(), seg_off.as<int32_t>(), seg_cnt.as<int32_t>(),
                     place ? order.as<int32_t>() : nullptr, mask.as<uint32_t>(), wpk, u_max, dense ? 1 : 0,
                     want_inv && place ? sslot.as<int32_t>() : nullptr, key_rank.as<int32_t>()};
  }
  // what a fused marking pass needs (dense mode): masks, words per key, the
  // scan's tile status / counter to reset and their number
  struct MarkArgs {
    uint32_t* mask;
    int wpk;
    unsigned long long* status;
    int32_t* ctr;
    int64_t n_tiles;
    uint32_t* lmask;
  };
  MarkArgs mark_args() {
    return MarkArgs{mask.as<uint32_t>(), wpk, status.as<unsigned long long>(), ctrs.as<int32_t>(), tiles_bits,
                    want_lmask && lmask_words ? lmask.as<uint32_t>() : nullptr};
  }
};

// ------------------------------------------------------------------ layers
struct AdamParams {
  float lr, b1, b2, eps;
  double b1d, b2d;
  const float2* table;  // (lr / (1 - b1^t), 1 / (1 - b2^t)) for t < table_n
  int64_t table_n;
  int table_exact;      // beyond the table both factors are exactly (lr, 1) in fp32
};

// h = relu(x W1 + b1); hmask (b x hp/32) = per-sample nonzero bits; the last
// CTA writes live (1 + hp ints): the number of units nonzero anywhere in the
// batch, then the live units ascending followed by the dead ones.  ticket:
// one zero-initialised int (self-resetting).
// SimHash query keys fused into the hidden forward (per-sample queries)
constexpr int kQhMaxBits = 2048;
struct QueryHash {
  const uint16_t* packed_t = nullptr;  // (c, K*L) terms: idx | (sign < 0) << 15
  int k = 0, l = 0, c = 0;
  uint32_t* keys = nullptr;            // (b, L)
};
void launch_hidden_forward(int hp, int b, const int32_t* x_ptr, const int32_t* x_idx, const float* x_val,
                           const float* w1t, const float* b1, float* h, uint32_t* hmask, int32_t* live,
                           int32_t* ticket, cudaStream_t s, const QueryHash* qh = nullptr);
// the same live-unit list from an h written by other means
void launch_live_cols_from_h(int hp, int b, const float* h, uint32_t* hmask, int32_t* live, cudaStream_t s);

// s_rows: the stream of the per-row (sparse tile) kernel, concurrent with
// the dense tiles on s (the caller joins it)
// sparse sets: z[p] = W2[prow[p]] . h[pslot[p]] + b2[prow[p]], p < *n_dev (sample-major)
void launch_logits_pairs(int hp, const int32_t* n_dev, int64_t n_max, const int32_t* prow, const int32_t* pslot,
                         const float* w2, const float* b2, const float* h, const int32_t* live, float* z,
                         cudaStream_t s);
void launch_logits_rows(int hp, int b, const GroupView& g, const int32_t* pslot, const float* w2, const float* b2,
                        const float* h, const int32_t* live, float* z, cudaStream_t s, cudaStream_t s_rows);

// rows != null: z is in the row grouping's order (place-free dense
// grouping); each pair's position comes from its row's slot mask, and the
// kernel also writes sslot[pos] = slot for the W2 Adam
void launch_softmax(int b, const int32_t* offs, const uint8_t* plab, const int32_t* y_ptr, const float* z,
                    float* prob, float* delta, double* loss, const int32_t* inv, float* dsort, cudaStream_t s,
                    const int32_t* prow = nullptr, const GroupView* rows = nullptr, int32_t* sslot = nullptr,
                    bool small_sets = false);
// lazy softmax of a training step under the place-free grouping: per-tile
// partials (part: softmax_lazy_parts(u_max, b) float2), per sample stat =
// (M, 1/S, 1/|Y|) and the loss; pairs' errors are made where they are read
void launch_softmax_lazy(int b, const GroupView& g, const uint32_t* lmask, const float* z, const int32_t* y_ptr,
                         const int32_t* y_idx, float2* part, float* stat, double* loss, cudaStream_t s);
int64_t softmax_lazy_parts(int64_t u_max, int b);
// p (want_delta = false) or delta per pair, sample-major, of a lazy step
void launch_lazy_pairs(int b, const int32_t* offs, const int32_t* prow, const uint8_t* plab, const GroupView& g,
                       const float* z, const float* stat, float* out, bool want_delta, cudaStream_t s);
// place-free row grouping: out[pair] = rows_src[pos(pair)] (to_pairs) or
// rows_dst[pos(pair)] = src[pair] (to_rows), pairs in sample-major order
void launch_rows_pairs(int b, const int32_t* offs, const int32_t* prow, const GroupView& g, const float* src,
                       float* dst, bool to_pairs, cudaStream_t s);
// dst[inv[q]] = src[q] for q < *n_dev
void launch_scatter_sorted(const int32_t* n_dev, int64_t n_max, const int32_t* inv, const float* src, float* dst,
                           cudaStream_t s);
// hidden gradient from the row grouping (single-GPU step; errors in
// row-grouped order, dsort); scratch floats: hidden_grad_rows_scratch
size_t hidden_grad_rows_scratch(int b, int hp);
void launch_hidden_grad_rows(int hp, int b, const GroupView& g, const float* dsort, const float* w2, const float* h,
                             const int32_t* live, float* dh, float* part, int32_t* work_reset, cudaStream_t s,
                             const float* z = nullptr, const float* stat = nullptr, const uint32_t* lmask = nullptr);
// floats of scratch launch_hidden_grad needs
size_t hidden_grad_scratch(int b, int hp);
// done: b zero-initialised ints (self-resetting); work_reset (optional): the
// W2 Adam's row counter, zeroed here
void launch_hidden_grad(int hp, int b, const int32_t* offs, const int32_t* prow, const float* delta, const float* w2,
                        const float* h, const int32_t* live, float* dh, float* part, int32_t* done,
                        int32_t* work_reset, cudaStream_t s);
// sparse-set steps: the rows held by very many samples run in their own
// kernel (stream != null: beside the persistent kernel, forked / joined with
// the two events)
struct AdamVlong {
  cudaStream_t stream;
  cudaEvent_t fork, join;
};
void launch_adam_rows(int hp, int b, const AdamParams& ap, const int32_t* n_uniq, int64_t max_uniq,
                      const int32_t* uniq, const int32_t* seg_off, const int32_t* seg_cnt,
                      const int32_t* sslot, const float* dsort, const float* h, const int32_t* live, float* w2,
                      float* m2, float* v2, float* b2, float* mb2, float* vb2, int64_t* steps2,
                      unsigned long long* touched, int32_t* work, bool work_zeroed, cudaStream_t s,
                      const float* z = nullptr, const float* stat = nullptr, const uint32_t* mask = nullptr,
                      const uint32_t* lmask = nullptr, int wpk = 0, const AdamVlong* vl = nullptr);
void launch_accumulate(unsigned long long* dst, const int32_t* src, cudaStream_t s);
// per slot: the k best active ids by probability (ties: lower id), -1 padded
void launch_topk(int b, const int32_t* offs, const int32_t* rows, int shard_count, int shard_rank, const float* prob,
                 int k, int32_t* out, int32_t* cnt, cudaStream_t s);
void launch_x_slots(int b, const int32_t* x_ptr, int32_t* x_slot, cudaStream_t s);
void launch_hidden_counts(int hp, int b, const AdamParams& ap, const float* h, const int64_t* steps1, int32_t* tc,
                          float2* bc, cudaStream_t s);
void launch_adam_features(int hp, const AdamParams& ap, const int32_t* n_uniq, int64_t max_uniq,
                          const int32_t* uniq, const int32_t* seg_off, const int32_t* seg_cnt,
                          const int32_t* sorted_k, const int32_t* x_slot, const float* x_val, int64_t x_base,
                          const float* h, const float* dh, const float2* bc, const int32_t* live, float* w1t,
                          float* m1t, float* v1t, unsigned long long* touched, const int32_t* long_list,
                          const int32_t* n_long, cudaStream_t s, cudaStream_t s_long, int b);
// chains longer than this go to the segmented long-chain kernel
constexpr int kW1LongChain = 16;
void launch_hidden_prep_bias(int hp, int b, const AdamParams& ap, const float* h, const float* dh, int64_t* steps1,
                             int32_t* tc, float2* bc, float* b1, float* mb1, float* vb1, cudaStream_t s);
void launch_adam_hidden_bias(int hp, int b, const AdamParams& ap, const float* h, const float* dh, const int32_t* tc,
                             const float2* bc, float* b1, float* mb1, float* vb1, int64_t* steps1, cudaStream_t s);

// hidden layer sharded by units; see layers.cu
void launch_shard_hidden(int hp, int hg, int b, const int32_t* x_ptr, const int32_t* x_idx, const float* x_val,
                         const float* w1s, float* part, cudaStream_t s);
void launch_shard_assemble(int hp, int hidden, int hg, int b, const float* parts, const float* b1, float* h,
                           uint32_t* hmask, int32_t* live, int32_t* ticket, cudaStream_t s);
void launch_adam_w1_shard(int hp, int hg, int c0, const AdamParams& ap, const int32_t* n_uniq, int64_t max_uniq,
                          const int32_t* uniq, const int32_t* seg_off, const int32_t* seg_cnt, const int32_t* sorted_k,
                          const int32_t* x_slot, const float* x_val, int64_t x_base, const float* h, const float* dh,
                          const float2* bc, float* w1s, float* m1s, float* v1s, unsigned long long* touched,
                          cudaStream_t s);

}  // namespace slide
