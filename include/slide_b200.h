/*
 * slide_b200.h -- C ABI of the B200-native SLIDE adaptive-sparsity step.
 *
 * The reference (the pure-Python `slide` 0.1.0 package) has no FFI; its
 * hot path is a set of Python methods.  Each entry point below replaces one
 * of them (reference file:line under /root/reference/pkg/src/slide) and is
 * what a binding for that method would call (INTEGRATION.md shows the
 * ctypes stubs the Python mirror in paper_1903_03129_b200/ uses).
 *
 * Conventions
 *   - plain pointers and sizes only; "dev" pointers are CUDA device memory,
 *     "host" pointers are host memory;
 *   - every call returns 0 on success, else a status code (1 ValueError,
 *     2 IndexError, 3 CUDA/RuntimeError, 4 NotImplementedError,
 *     5 internal) with the message in slide_last_error() (thread-local);
 *   - work is queued on the stream given at slide_create (or
 *     slide_set_stream); calls that must report host-visible sizes
 *     synchronise that stream.
 */
#ifndef SLIDE_B200_H
#define SLIDE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct slide_ctx slide_ctx;

/* Network + LSH description.  All integers are int64 so the struct has no
 * padding (ctypes-friendly).  Mirrors SlideNetwork(input_dim, [hidden,
 * n_out], TrainConfig, lsh_layers={1: LshLayerConfig}) (network.py:172-221). */
typedef struct slide_net_desc {
  int64_t input_dim;   /* D */
  int64_t hidden;      /* H = widths[0] */
  int64_t hidden_pad;  /* row stride of every weight row, multiple of 128 >= H */
  int64_t n_out;       /* N = widths[1] */
  int64_t max_batch;   /* TrainConfig.batch_size */
  int64_t family;      /* 0 none (dense output), 1 simhash, 2 dwta, 3 wta */
  int64_t k, l;        /* LshLayerConfig.k / .l */
  int64_t key_bits;    /* K (simhash) or K*ceil(log2 m) (wta/dwta); <= 32 */
  int64_t capacity;    /* bucket cap */
  int64_t policy;      /* 0 fifo, 1 reservoir */
  int64_t strategy;    /* 0 vanilla, 1 topk, 2 hard_threshold */
  int64_t beta;
  int64_t min_freq;
  /* simhash: c entries per projection, (K*L, c) uint16 idx|(sign<0)<<15 */
  int64_t sh_c;
  const uint16_t* sh_packed_host;
  /* wta/dwta */
  int64_t bin_size, bins_per_perm, n_perms, bits;
  const int16_t* dw_perms_host;  /* (n_perms, H) */
  const int16_t* dw_donors_host; /* (K*L, 100): mix(salt, g, a) % KL, a=1..100 */
  /* Adam (TrainConfig, network.py:36-48) */
  double lr, beta1, beta2, eps;
  uint64_t seed;
  /* parameters, device, row stride hidden_pad; W1 stored transposed (D, hp)
   * -- sharded (shard_count > 1): this rank's units only, (D, H / G) */
  float *w1t, *m1t, *v1t, *b1, *mb1, *vb1;
  int64_t* steps1;
  float *w2, *m2, *v2, *b2, *mb2, *vb2;
  int64_t* steps2;
  /* column sharding of the output layer: this context owns
   * the rows id with id % shard_count == shard_rank, stored at local row
   * id / shard_count (W2 and its state hold only those rows).  0 / 1 =
   * unsharded. */
  int64_t shard_rank, shard_count;
} slide_net_desc;

/* One batch as device CSR (int32 offsets are absolute into idx/val).  The
 * host copies of the offsets let sub-batch steps size their work without a
 * device read. */
typedef struct slide_batch {
  int64_t batch;
  const int32_t* x_ptr;      /* dev (batch+1) */
  const int32_t* x_idx;      /* dev, sorted per row */
  const float* x_val;        /* dev */
  const int32_t* y_ptr;      /* dev (batch+1) */
  const int32_t* y_idx;      /* dev, sorted unique per row */
  const int32_t* x_ptr_host; /* host (batch+1) */
  const int32_t* y_ptr_host; /* host (batch+1) */
  uint64_t* rng_states;      /* dev (batch, 6) PCG64 states in/out, or NULL:
                                default_rng((seed, iteration, slot)) */
  const int32_t* forced_ptr; /* dev (batch+1) or NULL: explicit output active sets */
  const int32_t* forced_idx; /* dev, sorted unique per row */
  const int32_t* forced_ptr_host;
} slide_batch;

/* -- lifecycle ------------------------------------------------------- */
const char* slide_version(void);
const char* slide_last_error(void);
int slide_create(const slide_net_desc* desc, void* stream, slide_ctx** out);
int slide_destroy(slide_ctx* ctx);
int slide_set_stream(slide_ctx* ctx, void* stream);

/* -- hashing: HashFamily.hash / .hash_batch (hashing.py:112-118,172-178,
 *    265-287).  x: dev (n, ld) float32, dim <= ld; keys: dev (n, L) uint32. */
int slide_simhash_keys(const float* x, int64_t n, int64_t ld, int64_t dim, int64_t k, int64_t l, int64_t c,
                       const uint16_t* packed_dev, uint32_t* keys, void* stream);
int slide_dwta_keys(const float* x, int64_t n, int64_t ld, int64_t dim, int64_t k, int64_t l, int64_t m,
                    int64_t bins_per_perm, int64_t n_perms, int64_t bits, int64_t dense_mode,
                    const int16_t* perms_dev, const int16_t* donors_dev, uint32_t* keys, void* stream);

/* -- tables: LshTables.build / insert_codes / maybe_rebuild
 *    (tables.py:105-161, 180-196) -------------------------------------- */
/* hash the ctx's W2 rows and rebuild all L tables; mt_state: host 625 words
 * of random.Random(table_seed).getstate()[1], updated in place (reservoir) */
int slide_rebuild_tables(slide_ctx* ctx, uint64_t* mt_state);
/* Renumber the hidden units in place: new unit p takes the state of old unit
 * src[p] (host, a permutation of [0, hidden)) -- the columns of W1^T / W2 and
 * their Adam moments, the hidden biases, moments and step counters, and the
 * input indices of the ctx's hash functions move together, so the net computes
 * the same function; callers map their own unit order through the
 * permutation.  A layout operation with no reference counterpart: it keeps
 * the units that are live (nonzero somewhere in a batch) adjacent so the row
 * kernels' gathers of W[row, live units] (network.py:266,322-332) are
 * contiguous.  Unsharded contexts only. */
int slide_relabel_units(slide_ctx* ctx, const int32_t* src);
/* build from precomputed keys (dev (n, L) uint32) */
int slide_build_tables_from_keys(slide_ctx* ctx, const uint32_t* keys, int64_t n, uint64_t* mt_state);
/* clear every bucket (LshTables._clear, tables.py:123-125) */
int slide_clear_tables(slide_ctx* ctx);
/* sizes of the built index: distinct (table, key) buckets, stored id slots */
int slide_tables_info(slide_ctx* ctx, int64_t* n_buckets, int64_t* n_slots, int64_t* n_items);
/* host export: per bucket (table<<key_bits|key, insert count, first slot,
 * occupancy) and the slot array (FIFO: ascending ids of the kept tail). */
int slide_tables_export(slide_ctx* ctx, uint32_t* skeys, int32_t* counts, int32_t* starts, int32_t* lens,
                        int32_t* ids);
/* load host-built buckets (the reference's tests plant Bucket objects,
 * tests/test_network.py:347-360): n_buckets (skey, count, start, len) rows
 * over a slot array of n_slots ids; n_items = width of the id space */
int slide_tables_load(slide_ctx* ctx, const uint32_t* skeys, const int32_t* counts, const int32_t* starts,
                      const int32_t* lens, int64_t n_buckets, const int32_t* ids, int64_t n_slots,
                      int64_t n_items);
/* disable individual tables (bit t set = table t reads as empty), e.g.
 * after LshTables.tables[t].clear() */
int slide_tables_mask(slide_ctx* ctx, uint64_t disabled);
/* query_codes (tables.py:171-176): dev keys (b, L) -> dev (b, L) first slot
 * and occupancy of each probed bucket (0 when the key is absent) */
int slide_tables_probe(slide_ctx* ctx, const uint32_t* keys, int64_t b, int32_t* starts, int32_t* lens);
/* query_codes with bucket contents (tables.py:171-176), host in/out,
 * synchronous: keys (b, L) -> per probe the occupancy, the insert count and
 * the kept ids ascending at ids[q * capacity ..] (ids: b * L * capacity) */
int slide_tables_probe_ids(slide_ctx* ctx, const uint32_t* keys_host, int64_t b, int32_t* lens_host,
                           int32_t* counts_host, int32_t* ids_host);

/* Query + union (rebuild microbenchmark): hash n query rows
 * (device, stride hidden_pad) and write per query the ascending union of its
 * L buckets -- hard_threshold(min_freq=1), reference samplers.py:109-112.
 * cnt_out: device (n) int32; ids_out: device (n x cap_stride) int32,
 * cap_stride >= L * capacity; n_ids bounds the ids (rows in the tables). */
int slide_query_union(slide_ctx* ctx, const float* q_dev, int64_t n, int64_t n_ids, int64_t cap_stride,
                      int32_t* cnt_out, int32_t* ids_out);

/* samplers.sample on explicit candidate lists (RawCandidates; reference
 * samplers.py:57-120), for callers holding probed buckets.  Host arrays:
 * ptr (n_tables + 1) offsets into ids; order (n_tables) the vanilla probe
 * order (the caller's rng.permutation(L)); ids_out must hold ptr[n_tables]
 * ids (vanilla: fresh ids in probe order; topk: by frequency desc, id asc,
 * at most beta; hard_threshold: ascending); freq_out (width) or NULL. */
int slide_sample_lists(const int32_t* ptr_host, const int32_t* ids_host, int64_t n_tables, int64_t width,
                       int64_t strategy, int64_t beta, int64_t min_freq, const int32_t* order_host,
                       int32_t* ids_out, int64_t* n_out, int64_t* probed, int32_t* freq_out, void* stream);

/* -- the step --------------------------------------------------------- */
/* forward of a (sub-)batch (network.py:241-286, 225-239): hidden layer,
 * query hash, per-slot rng, sampler, fallback, label union, logits,
 * softmax, loss.  *n_pairs = total active (slot, row) pairs.
 * Synchronises the stream once (pair count). */
int slide_forward(slide_ctx* ctx, const slide_batch* batch, int64_t iteration, int64_t slot_offset,
                  int64_t* n_pairs);
/* backward of the last forward (network.py:290-336): output error, hidden
 * error from the pre-update W2, then (update != 0) Adam on every touched
 * row in slot order (network.py:428-451). */
int slide_backward(slide_ctx* ctx, int64_t update);
/* train_batch (network.py:340-379) without the rebuild barrier: slots run
 * in sub-batches of `sub_batch` samples (1 = the reference's sequential
 * workers=1 schedule, batch = the snapshot schedule).  loss_host: per-slot
 * loss (batch doubles); active_host: per-slot active count (batch int64). */
int slide_train_batch(slide_ctx* ctx, const slide_batch* batch, int64_t iteration, int64_t sub_batch,
                      double* loss_host, int64_t* active_host);

/* train_batch (snapshot schedule) as one CUDA graph: the batch (host or
 * device CSR, absolute offsets) is copied into context buffers sized by
 * capacities; the first call with new shapes runs eagerly, the second
 * captures, later calls replay.  A batch above a capacity re-captures.
 * Same outputs as slide_train_batch with sub_batch = batch. */
int slide_graph_step(slide_ctx* ctx, const slide_batch* batch, int64_t iteration, double* loss_host,
                     int64_t* active_host);
/* The same step split for pipelining (train_batches_csr): _async enqueues
 * the H2D copies, the step and the D2H of losses / set sizes without a host
 * wait (the batch's host buffers must stay untouched until that step's
 * _wait returns); _wait blocks for the OLDEST step in flight and fills
 * loss_host / active_host.  Up to two steps in flight per context, so step
 * k+1 is queued behind step k before the host waits for k; anything a
 * barrier enqueues on the context stream between the two (a table rebuild)
 * runs after step k and before step k+1.  slide_graph_step needs none in
 * flight.
 * Host batch arrays and the rebased offsets are staged per in-flight slot
 * on a context copy stream (beside the step in flight); a device batch is
 * read by the step's copy-in kernel after the caller's stream.  The D2H of
 * the results runs on the copy stream too; the caller's stream continues
 * after the step's device work. */
int slide_graph_step_async(slide_ctx* ctx, const slide_batch* batch, int64_t iteration);
int slide_graph_step_wait(slide_ctx* ctx, double* loss_host, int64_t* active_host);

/* stage readout of the last forward/backward (host copy), for parity:
 * 0 h (B, hp) f32 | 1 query keys (B, L) u32 | 2 offsets (B+1) i32 |
 * 3 pair rows (P) i32 | 4 pair label flag (P) u8 | 5 probs (P) f32 |
 * 6 delta (P) f32 | 7 loss (B) f64 | 8 dh (B, hp) f32 | 9 empty (B) i32 |
 * 10 rng states (B, 6) u64 | 11 logits (P) f32 (before softmax) |
 * 12 global active-set size per slot (B) i32 | 13 live hidden units (1 + hp) i32:
 * the count, then the units nonzero in some sample ascending, then the rest */
int slide_read(slide_ctx* ctx, int64_t what, void* host_dst, int64_t max_bytes, int64_t* bytes);

/* Ranked sampled inference for the last forward (reference network.py:383-391,
 * estimator.py:203-223): per slot the k best active ids by probability,
 * ties to the lower id (np.argsort(-p, kind="stable")), -1 padded; counts =
 * min(k, |A_i|).  ids_out: host (B x k) int32, counts_out: host (B) int32. */
int slide_topk(slide_ctx* ctx, int64_t k, int32_t* ids_out, int32_t* counts_out);
/* overwrite stage 0 (h) or 6 (delta) of the last forward with host values
 * (exact size): backward(trace) replays a trace's forward-time activations
 * and errors, as the reference's backward reads them from the trace
 * (network.py:303-313). */
int slide_write(slide_ctx* ctx, int64_t what, const void* host_src, int64_t bytes);

/* -- column-sharded step (shard_count > 1).  Rank g owns the
 *    output rows id % G == g (W2, its Adam state, its tables over those rows,
 *    global ids in the buckets) and the hidden units [g H/G, (g+1) H/G)
 *    (W1^T is a (D, H/G) array; b1 and its moments are replicated).  The
 *    caller runs the collectives over its process group between the stages
 *    (torch.distributed: NCCL on B200s); no stage synchronises the host.
 *    Replaces the per-layer passes of network.py:262-336 and the table
 *    build of tables.py:105-161 for one shard. ------------------------------ */
/* tables: hash this rank's rows and build its tables; *max_count = largest
 * local bucket (host).  all-reduce MAX; if G * max > cap (FIFO): pack every
 * rank's runs (pack_size / pack, int32), all-gather (padded to the largest
 * pack) and reconcile -- each rank keeps its members of every bucket's
 * global last-cap ids.  Reservoir tables must not overflow (checked). */
int slide_shard_build_local(slide_ctx* ctx, int64_t* max_count);
int slide_shard_tables_pack_size(slide_ctx* ctx, int64_t* n);
int slide_shard_tables_pack(slide_ctx* ctx, int32_t* out);
int slide_shard_tables_reconcile(slide_ctx* ctx, const int32_t* packs, int64_t stride);
/* keys (dev, local_rows x L) of this rank's W2 rows */
int slide_shard_hash_rows(slide_ctx* ctx, uint32_t* keys);
/* 1. part_out (dev, B x H/G): this rank's hidden pre-activations (no bias)
 *    -> all-gather into (G, B, H/G) */
int slide_shard_hidden(slide_ctx* ctx, const slide_batch* batch, float* part_out);
/* 2. h = relu(gathered + b1), nonzero masks, live units */
int slide_shard_assemble(slide_ctx* ctx, int64_t b, const float* parts);
/* 3. query keys, slot streams and this rank's sampler counts: hist_out
 *    (dev, B x (L+1) int32) -> all-reduce SUM */
int slide_shard_select(slide_ctx* ctx, const slide_batch* batch, int64_t iteration, int32_t* hist_out);
/* 4. the sampler rule with the global counts, fallback, label union, the
 *    owned (sample, row) pairs and their logits; max_out (dev, B): per-sample
 *    max over owned pairs (-inf when none) -> all-reduce MAX */
int slide_shard_forward(slide_ctx* ctx, const slide_batch* batch, int64_t iteration, const int32_t* ghist,
                        float* max_out);
/* 5. sum_out (dev, B): sum of exp(z - gmax) over owned pairs -> all-reduce SUM */
int slide_shard_softmax_sum(slide_ctx* ctx, const float* gmax, float* sum_out);
/* 6. p, delta on owned pairs; loss_out (dev, 2B f64): [i] sum over owned
 *    labels of min(-log p, 690.78), [B + i] owned active-set size ->
 *    all-reduce SUM (loss_i = [i] / |Y_i|, |A_i| = [B + i]) */
int slide_shard_softmax_finish(slide_ctx* ctx, const float* gmax, const float* gsum, double* loss_out);
/* 7. dh_out (dev, B x hidden_pad): W2_local^T delta (pre-update) -> all-reduce SUM */
int slide_shard_hidden_grad(slide_ctx* ctx, float* dh_out);
/* 8. Adam on the owned W2 rows, the replicated hidden biases / step
 *    counters, and this rank's W1 units, with the all-reduced dh */
int slide_shard_update(slide_ctx* ctx, const float* dh);

/* -- measurement -------------------------------------------------------- */
/* on != 0: time every stage with CUDA events on the ctx stream and count the
 * realised sets; resets the accumulators either way */
int slide_profile(slide_ctx* ctx, int64_t on);
/* stage_ms[32]: accumulated ms per stage (0 hidden fwd, 1 query hash,
 * 2 slot rng, 3 select, 4 fallback, 5 compaction, 6 logits, 7 softmax,
 * 8 hidden grad, 9 group rows, 10 adam W2, 11 hidden counts, 12 group
 * features, 13 adam W1, 14 hidden bias, 15 rebuild hash, 16 rebuild build);
 * counts[16]: 0 touched W2 coords, 1 touched W1 coords, 2 unique rows,
 * 3 unique features (sums over sub-steps), 4 probed bucket slots,
 * 8 pairs, 9 input nonzeros, 10 samples, 11 rebuilds */
int slide_profile_read(slide_ctx* ctx, double* stage_ms, int64_t* counts);
/* process-wide number of hand-written kernel launches so far */
int slide_launch_count(uint64_t* out);

/* -- host-side random streams (the same code the kernels run) ---------- */
/* default_rng(entropy).bit_generator state -> 6 words */
int slide_pcg64_seed(const uint64_t* entropy, int64_t n_entropy, uint64_t* state6);
int slide_pcg64_permutation(uint64_t* state6, int64_t n, int64_t* out);
int slide_pcg64_choice(uint64_t* state6, int64_t pop, int64_t size, int64_t* out);
/* random.Random: state 625 words in/out, n draws of random() */
int slide_mt19937_random(uint64_t* state625, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif
