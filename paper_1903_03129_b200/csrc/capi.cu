// extern "C" boundary (include/slide_b200.h) and the step orchestration.
#include "../../include/slide_b200.h"
#include "internal.cuh"
#include "kernels.cuh"
#include <cub/cub.cuh>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <cmath>

using namespace slide;

namespace slide {
unsigned long long g_slide_launches = 0;
unsigned long long g_slide_realloc_gen = 0;
}

// Per-stage CUDA-event timing (slide_profile): consecutive marks on the
// stream, the interval ending at a mark is charged to that mark's stage.
struct StageTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<int> stage_of;
  size_t used = 0;
  double acc[32] = {0};
  void mark(cudaStream_t s, int stage) {
    if (!on) return;
    if (used == pool.size()) {
      cudaEvent_t e;
      SLIDE_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    SLIDE_CUDA(cudaEventRecord(pool[used], s));
    if (stage_of.size() <= used) stage_of.resize(used + 1);
    stage_of[used++] = stage;
  }
  void collect() {
    if (!used) return;
    SLIDE_CUDA(cudaEventSynchronize(pool[used - 1]));
    for (size_t k = 1; k < used; ++k) {
      float ms = 0.f;
      SLIDE_CUDA(cudaEventElapsedTime(&ms, pool[k - 1], pool[k]));
      if (stage_of[k] >= 0) acc[stage_of[k]] += ms;
    }
    used = 0;
  }
};

enum Stage {
  kStStart = -1, kStHidden = 0, kStQueryHash, kStSlotRng, kStSelect, kStFallback, kStCompact, kStLogits,
  kStSoftmax, kStHiddenGrad, kStGroupRows, kStAdamRows, kStHiddenCounts, kStGroupFeat, kStAdamFeat,
  kStHiddenBias, kStRebuildHash, kStRebuildBuild
};

struct slide_ctx {
  StageTimer timer;
  DBuf counters;  // u64: 0 touched W2 coords, 1 touched W1 coords, 2 unique rows, 3 unique features
  int64_t host_counts[8] = {0};  // 0 pairs, 1 nnz, 2 samples, 3 rebuilds, 4 fallback slots, 5 graph re-captures
  slide_net_desc d{};
  cudaStream_t s = nullptr;
  // side stream of the backward pass (W1 grouping and W1 Adam run beside
  // the W2 path); forked from and joined back into `s` with events, so a
  // captured step is one graph with two branches
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_dh = nullptr, ev_join = nullptr, ev_pre = nullptr;
  // third stream: the per-row logits beside the dense-tile logits
  cudaStream_t s3 = nullptr;
  cudaEvent_t ev_lg = nullptr, ev_lg_join = nullptr, ev_w1l = nullptr, ev_hg = nullptr;
  cudaEvent_t ev_rng = nullptr, ev_rng_join = nullptr;  // slot streams beside the hidden forward
  // fourth stream: the W2 Adam's hot rows beside its persistent kernel (sparse-set steps)
  cudaStream_t s4 = nullptr;
  cudaEvent_t ev_vl = nullptr, ev_vl_join = nullptr;
  DBuf hg_done;  // per-sample slice tickets of the hidden gradient (self-resetting)
  int64_t hg_done_n = 0;
  // set by the fused step callers: forward already queues the W1 grouping
  // on the side stream (it needs only the inputs)
  bool w1_prefork = false, w1_grouped = false;
  int hp = 0;
  TablesHost tab;
  DBuf sh_packed, sh_packed_t, dw_perms, dw_donors, rowkeys;
  // forward workspace
  DBuf h, qkeys, order, states, act, cnt, empty, offs, prow, pslot, plab, z, prob, delta, loss, dh, dsort;
  // live hidden units of the last forward (see launch_hidden_forward)
  DBuf hmask, live, live_ticket;
  DBuf fb_ids, fb_scratch, fb_bitmap, fb_rng;
  // backward workspace
  GroupBy grow, gfeat;
  bool grow_pending = false;  // grow holds a forward's grouping not yet cleared
  // output-layer sharding: rank g of G owns ids with id % G == g
  int g = 0, G = 1;
  int64_t n_local = 0;
  // hidden layer sharded by units: this rank's W1^T holds units [c0, c0 + hg)
  int hg = 0, c0 = 0;
  // sharded selection phases (slide_shard_select / slide_shard_forward):
  // 1 = stop after the per-rank sampler counts, 2 = finish with the
  // all-reduced counts; 0 = unsharded
  int shard_phase = 0;
  // the last forward's row grouping ran place-free (see forward_impl)
  bool rows_mode = false;
  // ... and its softmax was lazy (training steps: per-tile partials, the
  // errors made by the hidden gradient / W2 Adam from the logits)
  bool lazy = false;
  DBuf prob_tmp, sm_part, sm_stat;
  const int32_t* shard_ghist = nullptr;
  int32_t* shard_hist = nullptr;
  DBuf shard_pack;
  DBuf cnt_all;  // per-slot global active-set size (sharded statistics)
  // CUDA-graph step (slide_graph_step): static shapes + context-owned batch
  struct {
    bool on = false;
    int64_t batch = 0, nnz_cap = 0, lab_cap = 0, ylab_cap = 0;
  } st;
  bool st_active = false;  // forward/backward run with the static shapes above
  DBuf iter_dev, gx_ptr, gx_idx, gx_val, gy_ptr, gy_idx;
  int64_t g_last_pmax = 0;  // host bookkeeping of the captured step
  unsigned long long g_kernels = 0;  // hand-written kernels per replay
  // Graph steps in flight (async API): up to two, each with its own pinned
  // staging (rebased x_ptr | y_ptr, iteration) and result slots and an
  // event after its last copy; a slot is reused two launches later, after
  // its results were taken.
  // Inputs are staged per slot on the copy stream (pinned header H2D, host
  // arrays H2D into gin) while the previous step runs; one copy-in kernel on
  // the graph stream moves them into the graph's buffers.  Results are
  // packed per slot (gout) on the graph stream and read back on the copy
  // stream beside the next step.
  struct GSlot {
    int32_t* ptrs = nullptr;  // pinned header: x_ptr | y_ptr (rebased), then the iteration (int64)
    int64_t ptrs_n = 0;
    int64_t* iter = nullptr;  // inside the header
    double* loss = nullptr;   // pinned results: loss (B doubles) | cnt (B int32)
    int32_t* cnt = nullptr;
    int64_t res_n = 0;
    DBuf gin, gout;
    cudaEvent_t ev = nullptr;  // results in pinned memory (copy stream)
    cudaEvent_t ev_staged = nullptr, ev_consumed = nullptr, ev_dev = nullptr;
    bool used = false;
  } gslot[2];
  cudaStream_t cstream = nullptr;
  // results read back on their own stream: the next step's staging (cstream)
  // must not queue behind this step's device-to-host copy, which waits for
  // the step to finish -- it would put the staging on the critical path
  cudaStream_t ostream = nullptr;
  int g_next = 0;      // slot of the next launch
  int g_q[2] = {0, 0};  // pending slots, oldest first
  int64_t g_qb[2] = {0, 0};
  int g_qn = 0;
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev_in = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int graph_state = 0;  // 0: shapes new (run eagerly), 1: capture next, 2: replay
  unsigned long long graph_gen = 0;  // g_slide_realloc_gen the graph was captured under
  DBuf bias_table;
  int64_t bias_n = 0;
  int bias_exact = 1;
  DBuf xslot, tc, bc, partial, tc_scratch, long_list, n_long, work, topk_out, topk_cnt, relabel, sel_big;
  int64_t fb_bitmap_words = 0;
  double* pinned_loss = nullptr;
  int32_t* pinned_cnt = nullptr;
  int64_t pinned_n = 0;
  // last forward
  bool have_forward = false;
  int last_b = 0;
  int64_t last_P = 0, last_Pmax = 0, last_nnz = 0, last_xbase = 0;
  const int32_t* last_xptr = nullptr;
  const int32_t* last_xidx = nullptr;
  const float* last_xval = nullptr;
  const int32_t* last_yptr = nullptr;
  std::vector<int32_t> h_offs;
};

static thread_local std::string g_err;

static bool getenv_flag(const char* name) {  // experiments only
  const char* e = getenv(name);
  return e && *e && *e != '0';
}

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kInternal;
  }
}

static int bits_for(int64_t n) {
  int b = 1;
  while (b < 62 && ((int64_t)1 << b) < n) ++b;
  return b;
}

// Bias-correction table (fp64 math, fp32 entries): (lr / (1 - b1^t),
// 1 / (1 - b2^t)) up to the step where both become (lr, 1) in fp32.
static void build_bias_table(slide_ctx* c);

static AdamParams adam_of(slide_ctx* c) {
  const slide_net_desc& d = c->d;
  AdamParams ap;
  ap.lr = (float)d.lr;
  ap.b1 = (float)d.beta1;
  ap.b2 = (float)d.beta2;
  ap.eps = (float)d.eps;
  ap.b1d = d.beta1;
  ap.b2d = d.beta2;
  if (!c->bias_table.p) build_bias_table(c);
  ap.table = c->bias_table.as<float2>();
  ap.table_n = c->bias_n;
  ap.table_exact = c->bias_exact;
  return ap;
}

static void build_bias_table(slide_ctx* c) {
  const double b1 = c->d.beta1, b2 = c->d.beta2, lr = c->d.lr;
  const double bmax = std::max(b1, b2);
  // b^t < 2^-40 makes 1 - b^t == 1 in fp32 (and its reciprocal exactly 1)
  int64_t need = bmax <= 0.0 ? 2 : (int64_t)std::ceil(40.0 * std::log(2.0) / -std::log(bmax)) + 2;
  const int64_t cap = (int64_t)1 << 24;
  c->bias_exact = need <= cap;
  c->bias_n = std::min(need, cap);
  std::vector<float2> tab((size_t)c->bias_n);
  tab[0] = make_float2((float)lr, 1.f);
  double p1 = 1.0, p2 = 1.0;
  for (int64_t t = 1; t < c->bias_n; ++t) {
    p1 = std::pow(b1, (double)t);
    p2 = std::pow(b2, (double)t);
    tab[(size_t)t] = make_float2((float)(lr / (1.0 - p1)), (float)(1.0 / (1.0 - p2)));
  }
  SLIDE_CUDA(cudaMemcpy(c->bias_table.ensure<float2>(c->bias_n), tab.data(), c->bias_n * sizeof(float2),
                        cudaMemcpyHostToDevice));
}

static SimHashDev simhash_of(slide_ctx* c) {
  SimHashDev f;
  f.dim = (int)c->d.hidden;
  f.k = (int)c->d.k;
  f.l = (int)c->d.l;
  f.c = (int)c->d.sh_c;
  f.packed = c->sh_packed.as<uint16_t>();
  f.packed_t = c->sh_packed_t.as<uint16_t>();
  return f;
}

static DwtaDev dwta_of(slide_ctx* c) {
  DwtaDev f;
  f.dim = (int)c->d.hidden;
  f.k = (int)c->d.k;
  f.l = (int)c->d.l;
  f.m = (int)c->d.bin_size;
  f.bins_per_perm = (int)c->d.bins_per_perm;
  f.n_perms = (int)c->d.n_perms;
  f.bits = (int)c->d.bits;
  f.dense_mode = c->d.family == 3;
  f.perms = c->dw_perms.as<int16_t>();
  f.donors = c->dw_donors.as<int16_t>();
  return f;
}

// pair count of the last forward (synchronises; API / test paths only)
static int64_t host_pairs(slide_ctx* c) {
  if (c->last_P < 0) {
    int32_t p = 0;
    SLIDE_CUDA(cudaMemcpyAsync(&p, c->offs.as<int32_t>() + c->last_b, 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
    c->last_P = p;
  }
  return c->last_P;
}

static void hash_rows(slide_ctx* c, const float* x, int64_t n, uint32_t* keys) {
  if (c->d.family == 1) launch_simhash_keys(simhash_of(c), x, n, c->hp, keys, c->s, &c->tc_scratch);
  else launch_dwta_keys(dwta_of(c), x, n, c->hp, keys, c->s);
}

extern "C" {

const char* slide_version(void) { return "slide_b200 0.1.0 (sm_100a)"; }
const char* slide_last_error(void) { return g_err.c_str(); }

int slide_create(const slide_net_desc* desc, void* stream, slide_ctx** out) {
  return guarded([&] {
    SLIDE_CHECK(desc && out, kValueError, "null argument");
    const slide_net_desc& d = *desc;
    SLIDE_CHECK(d.hidden >= 1 && d.hidden_pad >= d.hidden && d.hidden_pad % 128 == 0, kValueError,
                "hidden_pad must be a multiple of 128 >= hidden");
    SLIDE_CHECK(d.n_out >= 1 && d.input_dim >= 1 && d.max_batch >= 1, kValueError, "dims must be positive");
    SLIDE_CHECK(d.n_out < (1ll << 25), kNotSupported, "output width must be < 2^25 on the device path");
    SLIDE_CHECK(d.family >= 0 && d.family <= 3, kValueError, "unknown hash family");
    if (d.family) {
      SLIDE_CHECK(d.key_bits >= 1 && d.key_bits <= 32, kNotSupported, "device keys are at most 32 bits");
      SLIDE_CHECK(d.l >= 1 && d.l <= 64, kNotSupported, "at most 64 tables on the device path");
    }
    const int64_t G = d.shard_count < 1 ? 1 : d.shard_count;
    SLIDE_CHECK(d.shard_rank >= 0 && d.shard_rank < G, kValueError, "shard_rank must lie in [0, shard_count)");
    pcg_jump_table();  // the RNG jump table, allocated outside any graph capture
    slide_ctx* c = new slide_ctx();
    c->d = d;
    c->s = (cudaStream_t)stream;
    c->hp = (int)d.hidden_pad;
    c->g = (int)d.shard_rank;
    c->G = (int)G;
    c->n_local = (d.n_out - d.shard_rank + G - 1) / G;
    if (G > 1) {
      SLIDE_CHECK(d.hidden % G == 0 && (d.hidden / G) % 4 == 0 && d.hidden / G <= 128, kNotSupported,
                  "sharded hidden layer: hidden / shard_count must be a multiple of 4 and <= 128");
      SLIDE_CHECK(d.strategy != 1, kNotSupported, "the topk sampler is not supported on a sharded output layer");
      c->hg = (int)(d.hidden / G);
      c->c0 = (int)(d.shard_rank * c->hg);
    }
    try {
      if (d.family == 1) {
        size_t n = (size_t)d.k * d.l * d.sh_c;
        SLIDE_CHECK(d.sh_packed_host != nullptr, kValueError, "simhash projections missing");
        SLIDE_CUDA(cudaMemcpy(c->sh_packed.ensure<uint16_t>(n), d.sh_packed_host, n * 2, cudaMemcpyHostToDevice));
        // (c, K*L) transposed copy for the per-sample query kernel
        const int64_t KL = d.k * d.l;
        std::vector<uint16_t> tr(n);
        for (int64_t p = 0; p < KL; ++p)
          for (int64_t j = 0; j < d.sh_c; ++j) tr[j * KL + p] = d.sh_packed_host[p * d.sh_c + j];
        SLIDE_CUDA(cudaMemcpy(c->sh_packed_t.ensure<uint16_t>(n), tr.data(), n * 2, cudaMemcpyHostToDevice));
      } else if (d.family >= 2) {
        size_t np = (size_t)d.n_perms * d.hidden, nd = (size_t)d.k * d.l * 100;
        SLIDE_CHECK(d.dw_perms_host && d.dw_donors_host, kValueError, "dwta permutations missing");
        SLIDE_CUDA(cudaMemcpy(c->dw_perms.ensure<int16_t>(np), d.dw_perms_host, np * 2, cudaMemcpyHostToDevice));
        SLIDE_CUDA(cudaMemcpy(c->dw_donors.ensure<int16_t>(nd), d.dw_donors_host, nd * 2, cudaMemcpyHostToDevice));
      }
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int slide_destroy(slide_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaStreamSynchronize(c->s);
    c->tab.release();
    for (DBuf* b : {&c->sh_packed, &c->sh_packed_t, &c->dw_perms, &c->dw_donors, &c->rowkeys, &c->h, &c->dsort, &c->hmask, &c->live, &c->live_ticket, &c->qkeys, &c->order,
                    &c->states, &c->act, &c->cnt, &c->empty, &c->offs, &c->prow, &c->pslot, &c->plab, &c->z,
                    &c->prob, &c->delta, &c->loss, &c->dh, &c->fb_ids, &c->fb_scratch, &c->fb_bitmap, &c->xslot,
                    &c->tc, &c->bc, &c->counters, &c->partial, &c->relabel, &c->sel_big, &c->long_list, &c->n_long, &c->work, &c->topk_out, &c->topk_cnt, &c->tc_scratch, &c->bias_table, &c->cnt_all, &c->prob_tmp, &c->shard_pack, &c->fb_rng, &c->sm_part, &c->sm_stat})
      b->release();
    c->grow.release();
    c->gfeat.release();
    if (c->s2) cudaStreamSynchronize(c->s2);
    if (c->s3) cudaStreamSynchronize(c->s3);
    for (cudaEvent_t e : {c->ev_fork, c->ev_dh, c->ev_join, c->ev_pre, c->ev_lg, c->ev_lg_join, c->ev_w1l, c->ev_hg,
                          c->ev_rng, c->ev_rng_join})
      if (e) cudaEventDestroy(e);
    if (c->s2) cudaStreamDestroy(c->s2);
    if (c->s3) cudaStreamDestroy(c->s3);
    if (c->s4) {
      cudaStreamSynchronize(c->s4);
      cudaEventDestroy(c->ev_vl);
      cudaEventDestroy(c->ev_vl_join);
      cudaStreamDestroy(c->s4);
    }
    c->hg_done.release();
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->graph) cudaGraphDestroy(c->graph);
    for (DBuf* b : {&c->iter_dev, &c->gx_ptr, &c->gx_idx, &c->gx_val, &c->gy_ptr, &c->gy_idx}) b->release();
    if (c->gstream) cudaStreamSynchronize(c->gstream);
    if (c->cstream) cudaStreamSynchronize(c->cstream);
    if (c->ostream) cudaStreamSynchronize(c->ostream);
    for (auto& g : c->gslot) {
      if (g.ptrs) cudaFreeHost(g.ptrs);
      if (g.loss) cudaFreeHost(g.loss);
      for (cudaEvent_t e : {g.ev, g.ev_staged, g.ev_consumed, g.ev_dev})
        if (e) cudaEventDestroy(e);
      g.gin.release();
      g.gout.release();
    }
    if (c->gev_in) cudaEventDestroy(c->gev_in);
    if (c->gstream) cudaStreamDestroy(c->gstream);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->ostream) cudaStreamDestroy(c->ostream);
    if (c->pinned_loss) cudaFreeHost(c->pinned_loss);
    if (c->pinned_cnt) cudaFreeHost(c->pinned_cnt);
    for (cudaEvent_t e : c->timer.pool) cudaEventDestroy(e);
    delete c;
  });
}

int slide_set_stream(slide_ctx* c, void* stream) {
  return guarded([&] { c->s = (cudaStream_t)stream; });
}

// ------------------------------------------------------------------ hashing
int slide_simhash_keys(const float* x, int64_t n, int64_t ld, int64_t dim, int64_t k, int64_t l, int64_t c,
                       const uint16_t* packed_dev, uint32_t* keys, void* stream) {
  return guarded([&] {
    SLIDE_CHECK(k * 1 <= 32, kNotSupported, "device keys are at most 32 bits");
    SLIDE_CHECK(dim <= 32767 && dim <= ld, kValueError, "simhash dim must be <= 32767 and <= ld");
    SimHashDev f{(int)dim, (int)k, (int)l, (int)c, packed_dev};
    // large batches take the tensor-core path (its fix-up list is shared scratch)
    static std::mutex mu;
    static DBuf scratch;
    std::lock_guard<std::mutex> lock(mu);
    launch_simhash_keys(f, x, n, (int)ld, keys, (cudaStream_t)stream, &scratch);
  });
}

int slide_dwta_keys(const float* x, int64_t n, int64_t ld, int64_t dim, int64_t k, int64_t l, int64_t m,
                    int64_t bins_per_perm, int64_t n_perms, int64_t bits, int64_t dense_mode,
                    const int16_t* perms_dev, const int16_t* donors_dev, uint32_t* keys, void* stream) {
  return guarded([&] {
    SLIDE_CHECK(k * bits <= 32, kNotSupported, "device keys are at most 32 bits");
    SLIDE_CHECK(dim <= 32767 && dim <= ld && m <= 256, kValueError, "dwta dim must be <= 32767, bin <= 256");
    DwtaDev f{(int)dim, (int)k, (int)l, (int)m, (int)bins_per_perm, (int)n_perms, (int)bits, (int)dense_mode,
              perms_dev, donors_dev};
    launch_dwta_keys(f, x, n, (int)ld, keys, (cudaStream_t)stream);
  });
}

// ------------------------------------------------------------------- tables
static void build_from_keys(slide_ctx* c, const uint32_t* keys, int64_t n, uint64_t* mt) {
  SLIDE_CHECK(c->d.family != 0, kValueError, "layer has no LSH tables");
  tables_build(c->tab, keys, n, (int)c->d.l, (int)c->d.key_bits, (int)c->d.capacity, (int)c->d.policy, mt, c->s);
}

int slide_rebuild_tables(slide_ctx* c, uint64_t* mt_state) {
  return guarded([&] {
    SLIDE_CHECK(c->d.family != 0, kValueError, "layer has no LSH tables");
    SLIDE_CHECK(c->G == 1, kValueError, "sharded contexts rebuild from all-gathered keys (slide_shard_hash_rows)");
    const int64_t n = c->d.n_out;
    uint32_t* keys = c->rowkeys.ensure<uint32_t>((size_t)n * c->d.l);
    c->timer.mark(c->s, kStStart);
    hash_rows(c, c->d.w2, n, keys);
    c->timer.mark(c->s, kStRebuildHash);
    build_from_keys(c, keys, n, mt_state);
    c->timer.mark(c->s, kStRebuildBuild);
    c->host_counts[3] += 1;
  });
}

}  // extern "C"

// ---------------------------------------------------------- unit relabel
// Physical hidden-unit order (ref: none -- a layout choice below the API).
// After the first steps only ~30 of the hidden units are nonzero anywhere in
// a batch, scattered over the hidden width, so every row kernel's gathers of
// W[row, live units] pull one 32-byte sector per 4-byte value.  Renumbering
// the units so that the live ones are adjacent makes those gathers
// contiguous.  The renumbering is a consistent relabelling of the whole net:
// the columns of W1^T / W2 and their moments, the hidden bias state and step
// counters, and the hash functions' input indices all move together, so
// every kernel runs unchanged; the host views map back to the caller's order.
__global__ void __launch_bounds__(256) relabel_cols_kernel(float* __restrict__ a, int64_t rows, int ld, int hn,
                                                           const int32_t* __restrict__ src) {
  extern __shared__ float rl_row[];  // [8][hn]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* buf = rl_row + (size_t)w * hn;
  for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < rows; r += (int64_t)gridDim.x * 8) {
    float* row = a + r * ld;
    for (int p = lane; p < hn; p += 32) buf[p] = row[p];
    __syncwarp();
    for (int p = lane; p < hn; p += 32) row[p] = buf[__ldg(src + p)];
    __syncwarp();
  }
}

template <typename T>
__global__ void relabel_vec_kernel(T* __restrict__ a, int hn, const int32_t* __restrict__ src) {
  extern __shared__ unsigned char rl_vec[];
  T* buf = reinterpret_cast<T*>(rl_vec);
  for (int p = threadIdx.x; p < hn; p += blockDim.x) buf[p] = a[p];
  __syncthreads();
  for (int p = threadIdx.x; p < hn; p += blockDim.x) a[p] = buf[src[p]];
}

// hash parameters: dimension indices (low 15 bits; bit 15 = a SimHash sign)
__global__ void relabel_index_kernel(uint16_t* __restrict__ a, int64_t n, const int32_t* __restrict__ inv) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const uint16_t e = a[q];
    a[q] = (uint16_t)((e & 0x8000u) | (uint16_t)inv[e & 0x7fffu]);
  }
}

extern "C" {

int slide_relabel_units(slide_ctx* c, const int32_t* src_host) {
  return guarded([&] {
    SLIDE_CHECK(c->G == 1, kNotSupported, "a sharded hidden layer keeps its unit order");
    const slide_net_desc& d = c->d;
    const int hn = (int)d.hidden, hp = c->hp;
    std::vector<int32_t> both((size_t)2 * hn, -1);
    for (int p = 0; p < hn; ++p) {
      const int32_t o = src_host[p];
      SLIDE_CHECK(o >= 0 && o < hn && both[hn + o] < 0, kValueError, "src must be a permutation of the hidden units");
      both[p] = o;
      both[hn + o] = p;
    }
    cudaStream_t s = c->s;
    int32_t* dev = c->relabel.ensure<int32_t>((size_t)2 * hn);
    SLIDE_CUDA(cudaMemcpyAsync(dev, both.data(), both.size() * 4, cudaMemcpyHostToDevice, s));
    const int32_t *src = dev, *inv = dev + hn;
    const size_t smem = (size_t)8 * hn * 4;
    SLIDE_CHECK(smem <= 200 * 1024, kNotSupported, "hidden layer too wide to relabel");
    if (smem > 48 * 1024)
      SLIDE_CUDA(cudaFuncSetAttribute(relabel_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto cols = [&](float* a, int64_t rows) {
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 8), (int64_t)kSms * 8));
      relabel_cols_kernel<<<grid, 256, smem, s>>>(a, rows, hp, hn, src);
      SLIDE_LAUNCH_CHECK();
    };
    for (float* a : {d.w1t, d.m1t, d.v1t}) cols(a, d.input_dim);
    for (float* a : {d.w2, d.m2, d.v2}) cols(a, c->n_local);
    for (float* a : {d.b1, d.mb1, d.vb1}) {
      relabel_vec_kernel<float><<<1, 256, (size_t)hn * 4, s>>>(a, hn, src);
      SLIDE_LAUNCH_CHECK();
    }
    relabel_vec_kernel<int64_t><<<1, 256, (size_t)hn * 8, s>>>(d.steps1, hn, src);
    SLIDE_LAUNCH_CHECK();
    auto index = [&](DBuf& b, int64_t n) {
      if (!b.p || n <= 0) return;
      relabel_index_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, s>>>(b.as<uint16_t>(), n, inv);
      SLIDE_LAUNCH_CHECK();
    };
    if (d.family == 1) {
      index(c->sh_packed, d.k * d.l * d.sh_c);
      index(c->sh_packed_t, d.k * d.l * d.sh_c);
    } else if (d.family >= 2) {
      index(c->dw_perms, d.n_perms * d.hidden);
    }
    SLIDE_CUDA(cudaStreamSynchronize(s));  // `both` is read by the copy
  });
}

int slide_build_tables_from_keys(slide_ctx* c, const uint32_t* keys, int64_t n, uint64_t* mt_state) {
  return guarded([&] { build_from_keys(c, keys, n, mt_state); });
}

int slide_clear_tables(slide_ctx* c) {
  return guarded([&] {
    c->tab.dev.empty = 1;
    c->tab.dev.n_runs = 0;
    c->tab.n_items = 0;
    c->tab.built = false;
  });
}

int slide_tables_info(slide_ctx* c, int64_t* n_buckets, int64_t* n_slots, int64_t* n_items) {
  return guarded([&] {
    *n_buckets = c->tab.dev.empty ? 0 : c->tab.dev.n_runs;
    *n_slots = c->tab.dev.empty ? 0 : c->tab.n_slots;
    *n_items = c->tab.n_items;
  });
}

int slide_tables_load(slide_ctx* c, const uint32_t* skeys, const int32_t* counts, const int32_t* starts,
                      const int32_t* lens, int64_t n_buckets, const int32_t* ids, int64_t n_slots, int64_t n_items) {
  return guarded([&] {
    SLIDE_CHECK(c->d.family != 0, kValueError, "layer has no LSH tables");
    tables_load(c->tab, skeys, counts, starts, lens, n_buckets, ids, n_slots, n_items, (int)c->d.l,
                (int)c->d.key_bits, (int)c->d.capacity, c->s);
    c->tab.n_slots = n_slots;
  });
}

int slide_tables_mask(slide_ctx* c, uint64_t disabled) {
  return guarded([&] { c->tab.dev.disabled = disabled; });
}

int slide_tables_export(slide_ctx* c, uint32_t* skeys, int32_t* counts, int32_t* starts, int32_t* lens,
                        int32_t* ids) {
  return guarded([&] {
    if (c->tab.dev.empty) return;
    const int64_t r = c->tab.dev.n_runs, ns = c->tab.n_slots;
    SLIDE_CUDA(cudaMemcpyAsync(skeys, c->tab.uniq.p, r * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaMemcpyAsync(counts, c->tab.dev.bcount, r * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaMemcpyAsync(starts, c->tab.dev.bstart, r * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaMemcpyAsync(lens, c->tab.dev.blen, r * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaMemcpyAsync(ids, c->tab.dev.ids, ns * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
  });
}

__global__ void probe_kernel(TablesDev t, const uint32_t* keys, int64_t b, int32_t* starts, int32_t* lens) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= b * t.l) return;
  int tt = (int)(q % t.l);
  int run = tables_lookup(t, ((uint32_t)tt << t.key_bits) | keys[q]);
  starts[q] = run >= 0 ? t.bstart[run] : 0;
  lens[q] = run >= 0 ? t.blen[run] : 0;
}

int slide_tables_probe(slide_ctx* c, const uint32_t* keys, int64_t b, int32_t* starts, int32_t* lens) {
  return guarded([&] {
    TablesDev t = c->tab.dev;
    t.l = (int)c->d.l;
    t.key_bits = (int)c->d.key_bits;
    int64_t n = b * t.l;
    if (n <= 0) return;
    probe_kernel<<<(int)ceil_div(n, 256), 256, 0, c->s>>>(t, keys, b, starts, lens);
    SLIDE_LAUNCH_CHECK();
  });
}

// query_codes with contents (reference tables.py:171-176): per probe q of
// (b, L) the bucket's occupancy, insert count and kept ids (ascending) at
// ids[q * cap ..]; the caller rotates FIFO rings from the insert count.
__global__ void probe_ids_kernel(TablesDev t, const uint32_t* keys, int64_t b, int32_t* lens, int32_t* counts,
                                 int32_t* ids) {
  const int64_t q = blockIdx.x;
  if (q >= b * t.l) return;
  const int tt = (int)(q % t.l);
  const int run = tables_lookup(t, ((uint32_t)tt << t.key_bits) | keys[q]);
  const int len = run >= 0 ? t.blen[run] : 0;
  if (threadIdx.x == 0) {
    lens[q] = len;
    counts[q] = run >= 0 ? t.bcount[run] : 0;
  }
  for (int j = threadIdx.x; j < len; j += blockDim.x) ids[q * t.cap + j] = t.ids[t.bstart[run] + j];
}

int slide_tables_probe_ids(slide_ctx* c, const uint32_t* keys_host, int64_t b, int32_t* lens_host,
                           int32_t* counts_host, int32_t* ids_host) {
  return guarded([&] {
    TablesDev t = c->tab.dev;
    t.l = (int)c->d.l;
    t.key_bits = (int)c->d.key_bits;
    t.cap = (int)c->d.capacity;
    const int64_t n = b * t.l;
    if (n <= 0) return;
    char* base = nullptr;
    const size_t bytes = (size_t)n * (4 + 4 + 4 + 4 * (size_t)t.cap);
    SLIDE_CUDA(cudaMalloc(&base, bytes));
    struct Free {
      char* p;
      ~Free() { cudaFree(p); }
    } free_base{base};
    uint32_t* d_keys = reinterpret_cast<uint32_t*>(base);
    int32_t* d_lens = reinterpret_cast<int32_t*>(d_keys + n);
    int32_t* d_counts = d_lens + n;
    int32_t* d_ids = d_counts + n;
    SLIDE_CUDA(cudaMemcpyAsync(d_keys, keys_host, n * 4, cudaMemcpyHostToDevice, c->s));
    probe_ids_kernel<<<(int)n, 128, 0, c->s>>>(t, d_keys, b, d_lens, d_counts, d_ids);
    SLIDE_LAUNCH_CHECK();
    SLIDE_CUDA(cudaMemcpyAsync(lens_host, d_lens, n * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaMemcpyAsync(counts_host, d_counts, n * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaMemcpyAsync(ids_host, d_ids, n * t.cap * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
  });
}

// Query + union (the rebuild microbenchmark's second half):
// hash n query rows (device, row stride ld = hidden_pad) and return, per
// query, the ascending union of its L buckets -- hard_threshold(min_freq=1)
// (reference samplers.py:109-112).  cnt_out (n) and ids_out (n x cap_stride)
// are device arrays; cap_stride >= L * capacity.
int slide_query_union(slide_ctx* c, const float* q, int64_t n, int64_t n_ids, int64_t cap_stride, int32_t* cnt_out,
                      int32_t* ids_out) {
  return guarded([&] {
    SLIDE_CHECK(c->d.family != 0, kValueError, "layer has no LSH tables");
    SLIDE_CHECK(c->tab.built, kValueError, "tables are not built");
    const int L = (int)c->d.l;
    SLIDE_CHECK(cap_stride >= (int64_t)L * c->d.capacity, kValueError, "cap_stride must be >= L * capacity");
    cudaStream_t s = c->s;
    const int chunk = 1024;
    uint32_t* keys = c->qkeys.ensure<uint32_t>((size_t)chunk * L);
    int32_t* yp = c->cnt_all.ensure<int32_t>(chunk + 1);
    int32_t* empty = c->empty.ensure<int32_t>(chunk);
    SLIDE_CUDA(cudaMemsetAsync(yp, 0, (chunk + 1) * 4, s));
    for (int64_t o = 0; o < n; o += chunk) {
      const int nb = (int)std::min<int64_t>(chunk, n - o);
      hash_rows(c, q + o * c->hp, nb, keys);
      SelectArgs a;
      a.tab = c->tab.dev;
      a.tab.l = L;
      a.tab.key_bits = (int)c->d.key_bits;
      a.qkeys = keys;
      a.order = nullptr;
      a.y_ptr = yp;
      a.y_idx = nullptr;
      a.b = nb;
      a.l = L;
      a.strategy = 3;  // union of every probed bucket
      a.beta = INT32_MAX;
      a.min_freq = 1;
      a.sort_bits = bits_for(n_ids) + 7;
      a.cap_max = cap_stride;
      a.act = ids_out + o * cap_stride;
      a.cnt = cnt_out + o;
      a.empty = empty;
      a.cand_ctr = nullptr;
      if (!launch_select_union(a, n_ids, s)) {
        a.strategy = 2;  // hard_threshold(min_freq = 1) through the sort path
        launch_select(a, (int)((int64_t)L * c->d.capacity), s);
      }
    }
  });
}

// --------------------------------------------------------------------- step
static void side_stream_init(slide_ctx* c) {
  if (c->s2) return;
  // the side branches (W1 grouping / Adam, per-row logits, long chains) at
  // the highest priority: their CTAs go first when the persistent W2 Adam
  // frees a slot, so the shorter W1 branch is not starved behind it
  int lo = 0, hi = 0;
  SLIDE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  SLIDE_CUDA(cudaStreamCreateWithPriority(&c->s2, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
  SLIDE_CUDA(cudaStreamCreateWithPriority(&c->s3, cudaStreamNonBlocking, hi));
  for (cudaEvent_t* e : {&c->ev_fork, &c->ev_dh, &c->ev_join, &c->ev_pre, &c->ev_lg, &c->ev_lg_join, &c->ev_w1l,
                         &c->ev_hg, &c->ev_rng, &c->ev_rng_join})
    SLIDE_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

static int32_t* live_ticket(slide_ctx* c) {
  if (c->live_ticket.bytes == 0) {
    SLIDE_CUDA(cudaMemset(c->live_ticket.ensure<int32_t>(1), 0, 4));
  }
  return c->live_ticket.as<int32_t>();
}

static int32_t* hg_tickets(slide_ctx* c, int b) {
  if (c->hg_done_n < b) {
    int32_t* p = c->hg_done.ensure<int32_t>(b);
    SLIDE_CUDA(cudaMemset(p, 0, (size_t)b * 4));
    c->hg_done_n = b;
  }
  return c->hg_done.as<int32_t>();
}

// Expected regime of the step's active sets from the configuration: sparse
// when the batch's (sample, row) pairs are few against the output width --
// a sample's set is ~min(beta, L * cap) ids (wide-out, scaled: ~1 sample per
// active row), dense when the full union of L buckets is taken for every
// sample (wide-in: ~45 samples per active row).
static int64_t expected_pairs(const slide_ctx* c, int b) {
  const slide_net_desc& d = c->d;
  if (d.family == 0) return 0;
  const int64_t lcap = d.l * d.capacity;
  const int64_t per = (d.strategy == 0 && d.beta >= lcap) ? lcap : std::min<int64_t>(d.beta, lcap);
  return (int64_t)b * per / std::max(c->G, 1);
}
static bool sparse_sets(const slide_ctx* c, int b) {
  return c->d.family != 0 && expected_pairs(c, b) * 4 < c->n_local;
}

static void forward_impl(slide_ctx* c, const slide_batch* bt, int64_t iteration, int64_t slot_offset,
                         int64_t* n_pairs) {
  const slide_net_desc& d = c->d;
  SLIDE_CHECK(d.w1t && d.w2, kValueError, "context has no network state");
  const int b = (int)bt->batch;
  SLIDE_CHECK(b >= 1 && b <= 1024, kValueError, "batch must hold 1..1024 slots");
  const int hp = c->hp, L = (int)d.l;
  cudaStream_t s = c->s;
  // static shapes (graph capture): capacities instead of this batch's sizes,
  // the batch sits in the context's own buffers (offsets start at 0)
  SLIDE_CHECK(c->G == 1 || c->shard_phase != 0, kValueError,
              "a sharded context runs the slide_shard_* stages (sharded.sharded_step)");
  const bool stat = c->st_active;
  int64_t x_base, nnz;
  int max_labels = 0;
  if (stat) {
    x_base = 0;
    nnz = c->st.nnz_cap;
    max_labels = (int)c->st.lab_cap;
  } else {
    x_base = bt->x_ptr_host[0];
    nnz = bt->x_ptr_host[b] - x_base;
    for (int i = 0; i < b; ++i) max_labels = std::max(max_labels, bt->y_ptr_host[i + 1] - bt->y_ptr_host[i]);
    c->host_counts[1] += nnz;
  }
  const int64_t* iter_dev = stat ? c->iter_dev.as<int64_t>() : nullptr;

  // fused step: the W1 feature grouping needs only the inputs -- queue it on
  // the side stream now, beside the whole forward pass (backward joins it)
  c->w1_grouped = false;
  if (c->w1_prefork && !c->timer.on && nnz > 0 && c->G == 1) {
    side_stream_init(c);
    SLIDE_CUDA(cudaEventRecord(c->ev_pre, s));
    SLIDE_CUDA(cudaStreamWaitEvent(c->s2, c->ev_pre, 0));
    int32_t* xs = c->xslot.ensure<int32_t>(nnz);
    c->gfeat.long_min = kW1LongChain;
    c->gfeat.prepare(d.input_dim, b, nnz);
    launch_x_slots(b, bt->x_ptr, xs, c->s2);
    c->gfeat.run(bt->x_idx + x_base, xs, stat ? bt->x_ptr + b : nullptr, nnz, nnz, c->s2);
    c->w1_grouped = true;
  }

  float* h = c->h.ensure<float>((size_t)b * hp);
  uint32_t* hmask = c->hmask.ensure<uint32_t>((size_t)b * (hp / 32));
  int32_t* live = c->live.ensure<int32_t>(1 + hp);
  c->timer.mark(s, kStStart);
  // SimHash query keys computed by the hidden forward itself when the
  // per-sample query kernel would run (the same arithmetic)
  QueryHash qh;
  const bool fuse_qh = c->G == 1 && !bt->forced_ptr && d.family == 1 && c->sh_packed_t.p != nullptr && b <= kSms * 8 &&
                       (int64_t)d.k * d.l <= kQhMaxBits;
  if (fuse_qh) {
    const SimHashDev f = simhash_of(c);
    qh.packed_t = f.packed_t;
    qh.k = f.k;
    qh.l = f.l;
    qh.c = f.c;
    qh.keys = c->qkeys.ensure<uint32_t>((size_t)b * L);
  }
  // the slot streams need only (seed, iteration, slot): drawn on the third
  // stream beside the hidden forward / query hash, joined before selection
  const bool lsh_sel = !bt->forced_ptr && d.family != 0;
  const bool early_vanilla = d.strategy == 0;
  const bool early_full_union = early_vanilla && d.beta >= (int64_t)L * d.capacity;
  const bool early_rng = lsh_sel && !c->timer.on && (!early_full_union || bt->rng_states) && c->shard_phase != 2;
  if (early_rng) {
    side_stream_init(c);
    uint64_t* states0 = c->states.ensure<uint64_t>((size_t)b * 6);
    uint8_t* order0 = c->order.ensure<uint8_t>((size_t)b * L);
    SLIDE_CUDA(cudaEventRecord(c->ev_rng, s));
    SLIDE_CUDA(cudaStreamWaitEvent(c->s3, c->ev_rng, 0));
    launch_slot_rng(b, d.seed, iteration, iter_dev, slot_offset, L, early_vanilla, bt->rng_states, states0, order0,
                    c->s3);
    SLIDE_CUDA(cudaEventRecord(c->ev_rng_join, c->s3));
  }
  // sharded: h was assembled from the all-gathered unit shards (slide_shard_assemble)
  if (c->G == 1)
    launch_hidden_forward(hp, b, bt->x_ptr, bt->x_idx, bt->x_val, d.w1t, d.b1, h, hmask, live, live_ticket(c), s,
                          fuse_qh ? &qh : nullptr);
  c->timer.mark(s, kStHidden);
  c->host_counts[2] += b;

  int32_t* cnt = c->cnt.ensure<int32_t>(b);
  int32_t* empty = c->empty.ensure<int32_t>(b);
  int64_t cap_max;
  int32_t* act;
  SLIDE_CHECK(!(stat && bt->forced_ptr), kValueError, "forced active sets are not graph-captured");
  if (bt->forced_ptr || d.family == 0) {
    int64_t m = d.n_out;
    if (bt->forced_ptr) {
      m = 0;
      for (int i = 0; i < b; ++i) m = std::max<int64_t>(m, bt->forced_ptr_host[i + 1] - bt->forced_ptr_host[i]);
    }
    cap_max = std::max<int64_t>(m, 1);
    act = c->act.ensure<int32_t>((size_t)b * cap_max);
    launch_explicit_active(b, d.n_out, bt->forced_ptr, bt->forced_idx, bt->y_ptr, bt->y_idx, cap_max, act, cnt,
                           empty, s);
    c->timer.mark(s, kStSelect);
  } else {
    uint32_t* qk = c->qkeys.ensure<uint32_t>((size_t)b * L);
    if (!fuse_qh && c->shard_phase != 2) hash_rows(c, h, b, qk);
    c->timer.mark(s, kStQueryHash);
    uint64_t* states = c->states.ensure<uint64_t>((size_t)b * 6);
    uint8_t* order = c->order.ensure<uint8_t>((size_t)b * L);
    const int vanilla = d.strategy == 0;
    const int64_t want = std::min<int64_t>(d.beta, d.n_out);
    const int64_t lcap = (int64_t)L * d.capacity;
    // vanilla with beta >= L*cap probes every table whatever the order: the
    // slot stream is only needed by the (rare) fallback, which derives it
    const bool full_union = vanilla && d.beta >= lcap;
    const bool rng_first = !full_union || bt->rng_states;
    if (early_rng)
      SLIDE_CUDA(cudaStreamWaitEvent(s, c->ev_rng_join, 0));
    else if (rng_first && c->shard_phase != 2)
      launch_slot_rng(b, d.seed, iteration, iter_dev, slot_offset, L, vanilla, bt->rng_states, states, order, s);
    c->timer.mark(s, kStSlotRng);
    cap_max = std::max<int64_t>(lcap, want) + max_labels;
    act = c->act.ensure<int32_t>((size_t)b * cap_max);
    SelectArgs a;
    a.tab = c->tab.dev;
    if (!c->tab.built) a.tab.empty = 1;
    a.tab.l = L;
    a.tab.key_bits = (int)d.key_bits;
    a.qkeys = qk;
    a.order = order;
    a.y_ptr = bt->y_ptr;
    a.y_idx = bt->y_idx;
    a.b = b;
    a.l = L;
    a.strategy = full_union ? 3 : (int)d.strategy;
    a.beta = (int)std::min<int64_t>(d.beta, INT32_MAX);
    a.min_freq = (int)d.min_freq;
    a.sort_bits = bits_for(d.n_out) + 7;
    a.cap_max = cap_max;
    a.act = act;
    a.cnt = cnt;
    a.empty = empty;
    a.cand_ctr = c->timer.on && c->shard_phase != 1 ? c->counters.as<unsigned long long>() + 4 : nullptr;
    a.hist_out = c->shard_phase == 1 ? c->shard_hist : nullptr;
    a.ghist = c->shard_phase == 2 ? c->shard_ghist : nullptr;
    if (!(full_union && launch_select_union(a, d.n_out, s))) {
      // candidates a sample is likely to gather: L probes of mean-sized buckets
      const int64_t runs = std::max<int64_t>(c->tab.dev.n_runs, 1);
      const int64_t mean_bucket = std::min<int64_t>(d.capacity, ceil_div(c->tab.n_items * d.l, runs));
      launch_select(a, (int)(lcap + max_labels), s, 2 * d.l * mean_bucket + max_labels,
                    c->sel_big.ensure<int32_t>(b));
    }
    c->timer.mark(s, kStSelect);
    if (c->shard_phase == 1) return;  // the caller all-reduces the counts
    // fallback for slots whose sampler returned nothing
    FallbackArgs f;
    f.empty = empty;
    f.states = states;
    f.states_ready = rng_first;
    f.seed = d.seed;
    f.iteration = iteration;
    f.slot_offset = slot_offset;
    f.iter_dev = iter_dev;
    f.l = L;
    f.vanilla = vanilla;
    f.n = d.n_out;
    f.want = want;
    f.fb_ids = c->fb_ids.ensure<int64_t>((size_t)b * want);
    f.scratch_per_slot = choice_scratch_entries(d.n_out, want);
    f.smem_scratch = f.scratch_per_slot * 8 <= 96 * 1024;
    f.scratch = f.smem_scratch ? nullptr : c->fb_scratch.ensure<int64_t>((size_t)b * f.scratch_per_slot);
    f.words = ceil_div(d.n_out, 32);
    if (c->fb_bitmap_words < (int64_t)b * f.words) {
      uint32_t* bm = c->fb_bitmap.ensure<uint32_t>((size_t)b * f.words);
      SLIDE_CUDA(cudaMemsetAsync(bm, 0, (size_t)b * f.words * 4, s));
      c->fb_bitmap_words = (int64_t)b * f.words;
    }
    f.bitmap = c->fb_bitmap.as<uint32_t>();
    f.y_ptr = bt->y_ptr;
    f.y_idx = bt->y_idx;
    f.cap_max = cap_max;
    f.act = act;
    f.cnt = cnt;
    // the choice's draws come from a run of its stream's outputs made in
    // parallel: ~want 64-bit outputs (two 32-bit draws per id, Floyd + shuffle)
    f.rng_n = (int)std::min<int64_t>(kPcgJump, want + 64);
    f.rng_buf = f.rng_n > kFbSmemOutputs ? c->fb_rng.ensure<uint64_t>((size_t)b * f.rng_n) : nullptr;
    f.jump = pcg_jump_table();
    launch_fallback(f, b, s);
    if (bt->rng_states)
      SLIDE_CUDA(cudaMemcpyAsync(bt->rng_states, states, (size_t)b * 48, cudaMemcpyDeviceToDevice, s));
    c->timer.mark(s, kStFallback);
  }
  // sharded: every rank selected the global active sets; keep the owned ids
  if (c->G > 1)
    launch_own_filter(b, act, cap_max, c->g, c->G, cnt, c->cnt_all.ensure<int32_t>(b), s);
  // pair count stays on the device (offs[b]); buffers are sized by the bound
  int32_t* offs = c->offs.ensure<int32_t>(b + 1);
  const int64_t P_max = (int64_t)b * cap_max;
  int32_t* prow = c->prow.ensure<int32_t>(P_max);
  int32_t* pslot = c->pslot.ensure<int32_t>(P_max);
  uint8_t* plab = c->plab.ensure<uint8_t>(P_max);
  // group the pairs by output row (slot order inside a row): the row-major
  // logits, hidden gradient and W2 Adam all walk this structure
  GroupBy& gr = c->grow;
  if (c->grow_pending) gr.clear(s);
  gr.want_inv = true;  // the softmax scatters the errors into row-grouped order
  gr.items_hint = expected_pairs(c, b);
  gr.want_lmask = c->G == 1 && c->w1_prefork;
  gr.prepare(c->n_local, b, P_max);
  // unsharded dense grouping: the pairs kernel fills the row slot masks
  // itself and no placement pass runs -- the logits are written in row order
  // and the softmax finds each pair's row position from the masks
  c->rows_mode = c->G == 1 && gr.dense && !getenv_flag("SLIDE_PLACED_GROUPING");
  gr.premarked = c->rows_mode;
  gr.place = !c->rows_mode;
  // lazy when the samples' sets are large (full unions: thousands of pairs per
  // sample, where the per-pair position lookups dominate the softmax)
  c->lazy = c->rows_mode && c->w1_prefork && gr.lmask_words > 0 && !getenv_flag("SLIDE_EAGER_SOFTMAX") &&
            (expected_pairs(c, b) >= (int64_t)b * 1024 || getenv_flag("SLIDE_LAZY_SOFTMAX"));
  if (c->rows_mode) {
    const GroupBy::MarkArgs m = gr.mark_args();
    launch_pairs(b, act, cap_max, cnt, offs, c->G, prow, pslot, plab, s, m.mask, m.wpk, m.status, m.ctr, m.n_tiles,
                 c->lazy ? m.lmask : nullptr);
  } else {
    launch_pairs(b, act, cap_max, cnt, offs, c->G, prow, pslot, plab, s);
  }
  c->timer.mark(s, kStCompact);
  float* z = c->z.ensure<float>(P_max);
  float* prob = c->prob.ensure<float>(P_max);
  float* delta = c->delta.ensure<float>(P_max);
  double* loss = c->loss.ensure<double>(b);
  float* dsort = c->dsort.ensure<float>(P_max);
  gr.run(prow, pslot, offs + b, 0, P_max, s);
  c->grow_pending = true;
  c->timer.mark(s, kStGroupRows);
  if (sparse_sets(c, b) && !c->rows_mode) {
    // ~one sample per active row: pair by pair, sample-major
    launch_logits_pairs(hp, offs + b, P_max, prow, pslot, d.w2, d.b2, h, live, z, s);
  } else {
    // per-row logits of the sparse tiles beside the dense tiles (third stream)
    const bool fork = !c->timer.on;
    cudaStream_t sr = s;
    if (fork) {
      side_stream_init(c);
      sr = c->s3;
      SLIDE_CUDA(cudaEventRecord(c->ev_lg, s));
      SLIDE_CUDA(cudaStreamWaitEvent(sr, c->ev_lg, 0));
    }
    launch_logits_rows(hp, b, gr.view(), pslot, d.w2, d.b2, h, live, z, s, sr);
    if (fork) {
      SLIDE_CUDA(cudaEventRecord(c->ev_lg_join, sr));
      SLIDE_CUDA(cudaStreamWaitEvent(s, c->ev_lg_join, 0));
    }
  }
  c->timer.mark(s, kStLogits);
  // sharded: the softmax is completed by the slide_shard_softmax_* stages
  if (c->G == 1 && c->lazy) {
    launch_softmax_lazy(b, gr.view(), gr.lmask.as<uint32_t>(), z, bt->y_ptr, bt->y_idx,
                        c->sm_part.ensure<float2>(softmax_lazy_parts(gr.u_max, b)),
                        c->sm_stat.ensure<float>((size_t)3 * b), loss, s);
  } else if (c->G == 1) {
    const GroupView rv = gr.view();
    launch_softmax(b, offs, plab, bt->y_ptr, z, prob, delta, loss, gr.inv.as<int32_t>(), dsort, s,
                   c->rows_mode ? prow : nullptr, c->rows_mode ? &rv : nullptr,
                   c->rows_mode ? gr.sslot.as<int32_t>() : nullptr,
                   /*small_sets=*/d.family != 0 && expected_pairs(c, b) / std::max(b, 1) + max_labels <= 1024);
  }
  c->timer.mark(s, kStSoftmax);
  c->have_forward = true;
  c->last_b = b;
  c->last_P = -1;  // on the device; host_pairs() reads it when needed
  c->last_Pmax = P_max;
  c->last_nnz = nnz;
  c->last_xbase = x_base;
  c->last_xptr = bt->x_ptr;
  c->last_xidx = bt->x_idx;
  c->last_xval = bt->x_val;
  c->last_yptr = bt->y_ptr;
  if (n_pairs) *n_pairs = host_pairs(c);
}

// ext_dh: the hidden gradient already computed (sharded step: all-reduced
// partials); otherwise it is computed here from this context's W2.
static void backward_impl(slide_ctx* c, int64_t update, const float* ext_dh = nullptr) {
  SLIDE_CHECK(c->have_forward, kValueError, "backward needs a forward first");
  const slide_net_desc& d = c->d;
  const int b = c->last_b, hp = c->hp;
  const int64_t P_max = c->last_Pmax;
  cudaStream_t s = c->s;
  GroupBy& gr = c->grow;
  GroupBy& gf = c->gfeat;
  const int64_t nnz = c->last_nnz;
  // W1 branch on the side stream: its grouping needs only the inputs, its
  // Adam only dh -- both overlap the hidden gradient and the W2 Adam.  The
  // profiled pass keeps one stream so the stage timers stay serial.
  const bool fork = update && !c->timer.on;
  cudaStream_t sw = s;
  if (fork) {
    side_stream_init(c);
    sw = c->s2;
    SLIDE_CUDA(cudaEventRecord(c->ev_fork, s));
    SLIDE_CUDA(cudaStreamWaitEvent(sw, c->ev_fork, 0));
  }
  int32_t* xs = nnz > 0 ? c->xslot.ensure<int32_t>(nnz) : nullptr;
  gf.long_min = kW1LongChain;  // the grouping lists the long chains for the W1 Adam
  if (nnz > 0) gf.prepare(d.input_dim, b, nnz);  // host-side sizing before any branch launches
  auto group_features = [&](cudaStream_t st) {
    if (nnz <= 0) return;
    launch_x_slots(b, c->last_xptr, xs, st);
    // static shapes: nnz is a capacity, the live count is x_ptr[b] (x_ptr[0] = 0)
    gf.run(c->last_xidx + c->last_xbase, xs, c->st_active ? c->last_xptr + b : nullptr, nnz, nnz, st);
  };
  if (fork && !c->w1_grouped) group_features(sw);
  const float* dh = ext_dh;
  if (!dh) {
    float* out = c->dh.ensure<float>((size_t)b * hp);
    // by rows (each W2 row read once per 32-slot window) when rows are shared
    // by many samples; by samples when the active sets barely overlap (then
    // every window would walk every row for ~one pair)
    const bool hg_rows = !getenv_flag("SLIDE_HG_SAMPLES") && (getenv_flag("SLIDE_HG_ROWS") || !sparse_sets(c, b));
    if (P_max > 0 && b <= 1024 && hg_rows)  // the errors in row-grouped order (dsort) and the grouping
      launch_hidden_grad_rows(hp, b, gr.view(), c->dsort.as<float>(), d.w2, c->h.as<float>(), c->live.as<int32_t>(),
                              out, c->partial.ensure<float>(hidden_grad_rows_scratch(b, hp)), update ? c->work.ensure<int32_t>(4) : nullptr, s,
                              c->lazy ? c->z.as<float>() : nullptr, c->lazy ? c->sm_stat.as<float>() : nullptr,
                              c->lazy ? gr.lmask.as<uint32_t>() : nullptr);
    else
      launch_hidden_grad(hp, b, c->offs.as<int32_t>(), c->prow.as<int32_t>(), c->delta.as<float>(), d.w2,
                         c->h.as<float>(), c->live.as<int32_t>(), out,
                         c->partial.ensure<float>(hidden_grad_scratch(b, hp)),
                         hg_tickets(c, b), update ? c->work.ensure<int32_t>(4) : nullptr, s);
    dh = out;
  }
  c->timer.mark(s, kStHiddenGrad);
  if (fork && c->grow_pending && !c->lazy) {
    // the row grouping's masks were last read by the hidden gradient: clear
    // them on the third stream beside the rest of the backward pass (a lazy
    // softmax's W2 Adam still reads them: cleared after it, below)
    SLIDE_CUDA(cudaEventRecord(c->ev_hg, s));
    SLIDE_CUDA(cudaStreamWaitEvent(c->s3, c->ev_hg, 0));
    gr.clear(c->s3);
    c->grow_pending = false;
  }
  if (!update) {
    if (c->w1_grouped) {  // a pre-forked grouping must still be joined
      side_stream_init(c);
      SLIDE_CUDA(cudaEventRecord(c->ev_join, c->s2));
      SLIDE_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
      c->w1_grouped = false;
    }
    return;
  }
  const AdamParams ap = adam_of(c);
  unsigned long long* ctr = c->timer.on ? c->counters.as<unsigned long long>() : nullptr;
  int32_t* tc = c->tc.ensure<int32_t>((size_t)b * hp);
  float2* bc = c->bc.ensure<float2>((size_t)b * hp);
  int32_t* work = c->work.ensure<int32_t>(4);
  // W1 branch: per-unit step counts + bias corrections and the hidden biases
  // (one fused pass), then the W1 Adam over the feature grouping
  auto w1_update = [&](cudaStream_t st) {
    launch_hidden_prep_bias(hp, b, ap, c->h.as<float>(), dh, d.steps1, tc, bc, d.b1, d.mb1, d.vb1, st);
    c->timer.mark(st, kStHiddenCounts);
    if (nnz <= 0) return;
    if (!fork) {
      group_features(st);
      c->timer.mark(st, kStGroupFeat);
    }
    c->w1_grouped = false;
    // the long chains on the third stream, beside the short ones
    cudaStream_t sl = st;
    if (fork) {
      sl = c->s3;
      SLIDE_CUDA(cudaEventRecord(c->ev_w1l, st));
      SLIDE_CUDA(cudaStreamWaitEvent(sl, c->ev_w1l, 0));
    }
    if (c->G > 1)  // this rank's hidden units only (W1^T sharded by units)
      launch_adam_w1_shard(hp, c->hg, c->c0, ap, gf.n_uniq.as<int32_t>(), gf.u_max, gf.uniq.as<int32_t>(),
                           gf.seg_off.as<int32_t>(), gf.seg_cnt.as<int32_t>(), gf.order.as<int32_t>(), xs,
                           c->last_xval, c->last_xbase, c->h.as<float>(), dh, bc, d.w1t, d.m1t, d.v1t,
                           ctr ? ctr + 1 : nullptr, st);
    else
      launch_adam_features(hp, ap, gf.n_uniq.as<int32_t>(), gf.u_max, gf.uniq.as<int32_t>(), gf.seg_off.as<int32_t>(),
                           gf.seg_cnt.as<int32_t>(), gf.order.as<int32_t>(), xs, c->last_xval, c->last_xbase,
                           c->h.as<float>(), dh, bc, c->live.as<int32_t>(), d.w1t, d.m1t, d.v1t,
                           ctr ? ctr + 1 : nullptr, gf.long_list.as<int32_t>(), gf.n_long.as<int32_t>(), st, sl, b);
    c->timer.mark(st, kStAdamFeat);
    gf.clear(st);
  };
  if (fork) {
    SLIDE_CUDA(cudaEventRecord(c->ev_dh, s));
    SLIDE_CUDA(cudaStreamWaitEvent(sw, c->ev_dh, 0));
    w1_update(sw);
  }
  // W2: rows in ascending order, each row's samples in slot order
  AdamVlong vl{nullptr, nullptr, nullptr};
  const AdamVlong* vlp = nullptr;
  if (sparse_sets(c, b) && !c->lazy && !getenv_flag("SLIDE_ADAM_ONE_KERNEL")) {
    if (fork) {
      if (!c->s4) {
        int lo = 0, hi = 0;
        SLIDE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        SLIDE_CUDA(cudaStreamCreateWithPriority(&c->s4, cudaStreamNonBlocking, hi));
        SLIDE_CUDA(cudaEventCreateWithFlags(&c->ev_vl, cudaEventDisableTiming));
        SLIDE_CUDA(cudaEventCreateWithFlags(&c->ev_vl_join, cudaEventDisableTiming));
      }
      vl = AdamVlong{c->s4, c->ev_vl, c->ev_vl_join};
    }
    vlp = &vl;
  }
  if (P_max > 0) {
    launch_adam_rows(hp, b, ap, gr.n_uniq.as<int32_t>(), gr.u_max, gr.uniq.as<int32_t>(), gr.seg_off.as<int32_t>(),
                     gr.seg_cnt.as<int32_t>(), gr.sslot.as<int32_t>(), c->dsort.as<float>(),
                     c->h.as<float>(), c->live.as<int32_t>(), d.w2, d.m2, d.v2, d.b2, d.mb2, d.vb2, d.steps2, ctr,
                     work,
                     /*work_zeroed=*/ext_dh == nullptr, s, c->lazy ? c->z.as<float>() : nullptr,
                     c->lazy ? c->sm_stat.as<float>() : nullptr, c->lazy ? gr.mask.as<uint32_t>() : nullptr,
                     c->lazy ? gr.lmask.as<uint32_t>() : nullptr, gr.wpk, vlp);
    c->timer.mark(s, kStAdamRows);
  }
  if (!fork) w1_update(s);
  c->timer.mark(s, kStHiddenBias);
  if (ctr) {
    launch_accumulate(ctr + 2, P_max > 0 ? gr.n_uniq.as<int32_t>() : nullptr, s);
    launch_accumulate(ctr + 3, nnz > 0 ? gf.n_uniq.as<int32_t>() : nullptr, s);
    launch_accumulate(ctr + 5, c->offs.as<int32_t>() + b, s);
  }
  if (c->grow_pending) {
    if (!(c->lazy && P_max > 0)) gr.clear(s);  // (a lazy step's W2 Adam cleared the masks it walked)
    c->grow_pending = false;
  }
  if (fork) {  // join: the next step reads W1, h and the side streams' buffers
    SLIDE_CUDA(cudaEventRecord(c->ev_join, sw));
    SLIDE_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
    SLIDE_CUDA(cudaEventRecord(c->ev_lg_join, c->s3));
    SLIDE_CUDA(cudaStreamWaitEvent(s, c->ev_lg_join, 0));
  }
}

int slide_forward(slide_ctx* c, const slide_batch* bt, int64_t iteration, int64_t slot_offset, int64_t* n_pairs) {
  return guarded([&] { forward_impl(c, bt, iteration, slot_offset, n_pairs); });
}

int slide_backward(slide_ctx* c, int64_t update) {
  return guarded([&] { backward_impl(c, update); });
}

int slide_train_batch(slide_ctx* c, const slide_batch* bt, int64_t iteration, int64_t sub_batch, double* loss_host,
                      int64_t* active_host) {
  return guarded([&] {
    const int64_t B = bt->batch;
    SLIDE_CHECK(B >= 1, kValueError, "batch is empty");
    SLIDE_CHECK(sub_batch >= 1, kValueError, "sub_batch must be >= 1");
    SLIDE_CHECK(c->G == 1, kValueError, "sharded contexts step through slide_shard_*");
    if (c->pinned_n < B) {
      if (c->pinned_loss) cudaFreeHost(c->pinned_loss);
      if (c->pinned_cnt) cudaFreeHost(c->pinned_cnt);
      SLIDE_CUDA(cudaHostAlloc((void**)&c->pinned_loss, B * 8, cudaHostAllocDefault));
      SLIDE_CUDA(cudaHostAlloc((void**)&c->pinned_cnt, B * 4, cudaHostAllocDefault));
      c->pinned_n = B;
    }
    for (int64_t s0 = 0; s0 < B; s0 += sub_batch) {
      const int64_t nb = std::min<int64_t>(sub_batch, B - s0);
      slide_batch v = *bt;
      v.batch = nb;
      v.x_ptr = bt->x_ptr + s0;
      v.y_ptr = bt->y_ptr + s0;
      v.x_ptr_host = bt->x_ptr_host + s0;
      v.y_ptr_host = bt->y_ptr_host + s0;
      if (bt->rng_states) v.rng_states = bt->rng_states + 6 * s0;
      if (bt->forced_ptr) {
        v.forced_ptr = bt->forced_ptr + s0;
        v.forced_ptr_host = bt->forced_ptr_host + s0;
      }
      c->w1_prefork = true;
      forward_impl(c, &v, iteration, s0, nullptr);
      c->w1_prefork = false;
      backward_impl(c, 1);
      // results ride back asynchronously; one host sync per call
      SLIDE_CUDA(cudaMemcpyAsync(c->pinned_loss + s0, c->loss.p, nb * 8, cudaMemcpyDeviceToHost, c->s));
      SLIDE_CUDA(cudaMemcpyAsync(c->pinned_cnt + s0, c->cnt.p, nb * 4, cudaMemcpyDeviceToHost, c->s));
    }
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
    for (int64_t i = 0; i < B; ++i) {
      if (loss_host) loss_host[i] = c->pinned_loss[i];
      if (active_host) active_host[i] = c->pinned_cnt[i];
      c->host_counts[0] += c->pinned_cnt[i];
    }
  });
}

// Word copies of up to 8 segments in one launch (graph-step staging in and
// results out).
struct CopyIn {
  uint32_t* dst[8];
  const uint32_t* src[8];
  int64_t words[8];
  int n = 0;
  void add(void* d, const void* s, int64_t w) {
    if (w <= 0) return;
    dst[n] = static_cast<uint32_t*>(d);
    src[n] = static_cast<const uint32_t*>(s);
    words[n] = w;
    ++n;
  }
};

__global__ void copy_in_kernel(CopyIn a) {
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int k = 0; k < a.n; ++k) {
    uint32_t* __restrict__ d = a.dst[k];
    const uint32_t* __restrict__ s = a.src[k];
    for (int64_t q = t0; q < a.words[k]; q += nt) d[q] = __ldcs(s + q);
  }
}

static void launch_copy_in(const CopyIn& a, cudaStream_t s) {
  if (a.n == 0) return;
  int64_t w = 0;
  for (int k = 0; k < a.n; ++k) w = std::max(w, a.words[k]);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(w, 256 * 2), kSms * 4));
  copy_in_kernel<<<grid, 256, 0, s>>>(a);
  SLIDE_LAUNCH_CHECK();
}

// One snapshot step as a CUDA graph (see header).  The first call with new
// shapes runs eagerly (and sizes every buffer), the second captures, the
// rest replay: no host work between the kernels, one sync per step.
// Enqueue one graph step: H2D of the batch, the step, D2H of the per-slot
// losses and set sizes into pinned memory; no host wait.
static void graph_step_launch(slide_ctx* c, const slide_batch* bt, int64_t iteration) {
    const int64_t B = bt->batch;
    SLIDE_CHECK(B >= 1 && B <= 1024, kValueError, "batch must hold 1..1024 slots");
    SLIDE_CHECK(!bt->forced_ptr && !bt->rng_states, kValueError, "graph steps take plain training batches");
    SLIDE_CHECK(c->G == 1, kValueError, "sharded contexts step through slide_shard_*");
    const int64_t x0 = bt->x_ptr_host[0], nnz = bt->x_ptr_host[B] - x0;
    const int64_t y0 = bt->y_ptr_host[0], nlab = bt->y_ptr_host[B] - y0;
    int64_t max_lab = 0;
    for (int64_t i = 0; i < B; ++i) max_lab = std::max<int64_t>(max_lab, bt->y_ptr_host[i + 1] - bt->y_ptr_host[i]);
    SLIDE_CHECK(c->g_qn < 2, kValueError, "two graph steps are already in flight");
    if (!c->gstream) {
      SLIDE_CUDA(cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
      SLIDE_CUDA(cudaEventCreateWithFlags(&c->gev_in, cudaEventDisableTiming));
      SLIDE_CUDA(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
      SLIDE_CUDA(cudaStreamCreateWithFlags(&c->ostream, cudaStreamNonBlocking));
      for (auto& g : c->gslot)
        for (cudaEvent_t* e : {&g.ev, &g.ev_staged, &g.ev_consumed, &g.ev_dev})
          SLIDE_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    const int slot = c->g_next;
    auto& gsl = c->gslot[slot];
    // the launch two steps back used this staging: its copies are done once
    // its event fired (its results were taken already: g_qn < 2)
    if (gsl.used) SLIDE_CUDA(cudaEventSynchronize(gsl.ev));
    auto& st = c->st;
    if (!st.on || st.batch != B || nnz > st.nnz_cap || max_lab > st.lab_cap || nlab > st.ylab_cap) {
      if (c->gexec) cudaGraphExecDestroy(c->gexec);
      if (c->graph) cudaGraphDestroy(c->graph);
      c->gexec = nullptr;
      c->graph = nullptr;
      st.on = true;
      st.batch = B;
      st.nnz_cap = std::max<int64_t>(nnz + nnz / 4, st.nnz_cap);
      st.lab_cap = std::max<int64_t>(max_lab + max_lab / 4 + 4, st.lab_cap);
      st.ylab_cap = std::max<int64_t>(nlab + nlab / 4 + 8, st.ylab_cap);
      c->gx_ptr.ensure<int32_t>(B + 1);
      c->gy_ptr.ensure<int32_t>(B + 1);
      c->gx_idx.ensure<int32_t>(st.nnz_cap);
      c->gx_val.ensure<float>(st.nnz_cap);
      c->gy_idx.ensure<int32_t>(st.ylab_cap);
      c->iter_dev.ensure<int64_t>(1);
      c->graph_state = 0;
    }
    const int64_t pw = (2 * (B + 1) + 1) & ~(int64_t)1;  // header words before the iteration (8-aligned)
    if (gsl.ptrs_n < pw + 2) {
      if (gsl.ptrs) cudaFreeHost(gsl.ptrs);
      SLIDE_CUDA(cudaHostAlloc((void**)&gsl.ptrs, (pw + 2) * 4, cudaHostAllocDefault));
      gsl.ptrs_n = pw + 2;
    }
    gsl.iter = reinterpret_cast<int64_t*>(gsl.ptrs + pw);
    if (gsl.res_n < B) {
      if (gsl.loss) cudaFreeHost(gsl.loss);
      SLIDE_CUDA(cudaHostAlloc((void**)&gsl.loss, B * 12, cudaHostAllocDefault));
      gsl.res_n = B;
    }
    gsl.cnt = reinterpret_cast<int32_t*>(gsl.loss + B);
    // per-slot device staging: header | x_idx | x_val | y_idx at the capacities
    const int64_t o_xi = (pw + 2) * 4, o_xv = o_xi + st.nnz_cap * 4, o_yi = o_xv + st.nnz_cap * 4;
    char* gin = gsl.gin.ensure<char>(o_yi + st.ylab_cap * 4);
    char* gout = gsl.gout.ensure<char>(B * 12);
    cudaStream_t user = c->s, gs = c->gstream, cs = c->cstream;
    // eager runs and captures read host-side sizes: nothing may be in flight
    if (c->graph_state < 2 || c->graph_gen != g_slide_realloc_gen) SLIDE_CUDA(cudaStreamSynchronize(gs));
    for (int64_t i = 0; i <= B; ++i) {
      gsl.ptrs[i] = (int32_t)(bt->x_ptr_host[i] - x0);
      gsl.ptrs[B + 1 + i] = (int32_t)(bt->y_ptr_host[i] - y0);
    }
    *gsl.iter = iteration;
    // staging on the copy stream, beside the step in flight: the copy-in two
    // steps back has read this slot's staging; host arrays are ready by
    // program order (device arrays are read by the copy-in kernel itself,
    // after the caller's stream)
    const void* probe = nnz ? (const void*)bt->x_idx : (const void*)bt->y_idx;
    cudaPointerAttributes pa{};
    const bool dev_src = (nnz || nlab) && cudaPointerGetAttributes(&pa, probe) == cudaSuccess &&
                         (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
    cudaGetLastError();  // unregistered host memory reports an error on some drivers
    if (gsl.used) SLIDE_CUDA(cudaStreamWaitEvent(cs, gsl.ev_consumed, 0));
    SLIDE_CUDA(cudaMemcpyAsync(gin, gsl.ptrs, (pw + 2) * 4, cudaMemcpyHostToDevice, cs));
    if (!dev_src) {
      if (nnz) {
        SLIDE_CUDA(cudaMemcpyAsync(gin + o_xi, bt->x_idx + x0, nnz * 4, cudaMemcpyDefault, cs));
        SLIDE_CUDA(cudaMemcpyAsync(gin + o_xv, bt->x_val + x0, nnz * 4, cudaMemcpyDefault, cs));
      }
      if (nlab) SLIDE_CUDA(cudaMemcpyAsync(gin + o_yi, bt->y_idx + y0, nlab * 4, cudaMemcpyDefault, cs));
    }
    SLIDE_CUDA(cudaEventRecord(gsl.ev_staged, cs));
    SLIDE_CUDA(cudaEventRecord(c->gev_in, user));
    SLIDE_CUDA(cudaStreamWaitEvent(gs, c->gev_in, 0));
    SLIDE_CUDA(cudaStreamWaitEvent(gs, gsl.ev_staged, 0));
    {
      CopyIn ci{};
      ci.add(c->gx_ptr.p, gin, B + 1);
      ci.add(c->gy_ptr.p, gin + (B + 1) * 4, B + 1);
      ci.add(c->iter_dev.p, gin + pw * 4, 2);
      ci.add(c->gx_idx.p, dev_src ? (const void*)(bt->x_idx + x0) : gin + o_xi, nnz);
      ci.add(c->gx_val.p, dev_src ? (const void*)(bt->x_val + x0) : gin + o_xv, nnz);
      ci.add(c->gy_idx.p, dev_src ? (const void*)(bt->y_idx + y0) : gin + o_yi, nlab);
      launch_copy_in(ci, gs);
    }
    SLIDE_CUDA(cudaEventRecord(gsl.ev_consumed, gs));
    slide_batch v{};
    v.batch = B;
    v.x_ptr = c->gx_ptr.as<int32_t>();
    v.x_idx = c->gx_idx.as<int32_t>();
    v.x_val = c->gx_val.as<float>();
    v.y_ptr = c->gy_ptr.as<int32_t>();
    v.y_idx = c->gy_idx.as<int32_t>();
    v.x_ptr_host = gsl.ptrs;
    v.y_ptr_host = gsl.ptrs + B + 1;
    c->s = gs;
    const bool timing = c->timer.on;
    c->st_active = true;
    try {
      if (c->grow_pending) {  // a single-sample forward left its grouping behind
        c->grow.clear(gs);
        c->grow_pending = false;
      }
      // a buffer the graph points into moved (e.g. a table rebuild with more
      // bucket runs than before): one eager step re-sizes every buffer for
      // the new tables (a capture must not allocate), then capture again
      if (c->graph_state == 2 && c->graph_gen != g_slide_realloc_gen) {
        c->graph_state = 0;
        ++c->host_counts[5];
      }
      if (c->graph_state < 2) c->timer.on = c->graph_state == 0 && timing;
      if (c->graph_state == 0) {
        c->w1_prefork = true;
        forward_impl(c, &v, iteration, 0, nullptr);
        c->w1_prefork = false;
        backward_impl(c, 1);
        c->graph_state = 1;
      } else if (c->graph_state == 1) {
        c->timer.on = false;
        const unsigned long long lc0 = g_slide_launches;
        if (c->gexec) {  // the previous graph's last replay is complete (stream synchronised above)
          cudaGraphExecDestroy(c->gexec);
          cudaGraphDestroy(c->graph);
          c->gexec = nullptr;
          c->graph = nullptr;
        }
        SLIDE_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        try {
          c->w1_prefork = true;
          forward_impl(c, &v, iteration, 0, nullptr);
          c->w1_prefork = false;
          backward_impl(c, 1);
        } catch (...) {
          c->w1_prefork = false;
          cudaGraph_t g;
          cudaStreamEndCapture(gs, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        SLIDE_CUDA(cudaStreamEndCapture(gs, &c->graph));
        c->graph_gen = g_slide_realloc_gen;
        // captured launches were counted once; every replay runs them again
        c->g_kernels = g_slide_launches - lc0;
        SLIDE_CUDA(cudaGraphInstantiate(&c->gexec, c->graph, 0));
        SLIDE_CUDA(cudaGraphLaunch(c->gexec, gs));
        c->g_last_pmax = c->last_Pmax;
        c->graph_state = 2;
      } else {
        SLIDE_CUDA(cudaGraphLaunch(c->gexec, gs));
        g_slide_launches += c->g_kernels;
        // host bookkeeping as if this step had run eagerly
        c->have_forward = true;
        c->last_b = (int)B;
        c->last_P = -1;
        c->last_Pmax = c->g_last_pmax;
        c->last_nnz = st.nnz_cap;
        c->last_xbase = 0;
        c->last_xptr = v.x_ptr;
        c->last_xidx = v.x_idx;
        c->last_xval = v.x_val;
        c->last_yptr = v.y_ptr;
      }
    } catch (...) {
      c->s = user;
      c->timer.on = timing;
      c->st_active = false;
      throw;
    }
    c->s = user;
    c->timer.on = timing;
    c->st_active = false;
    // results: packed into the slot's device buffer on the graph stream, read
    // back on the copy stream (beside the next step); the caller's stream
    // continues after the device work
    {
      CopyIn co{};
      co.add(gout, c->loss.p, 2 * B);
      co.add(gout + B * 8, c->cnt.p, B);
      launch_copy_in(co, gs);
    }
    SLIDE_CUDA(cudaEventRecord(gsl.ev_dev, gs));
    SLIDE_CUDA(cudaStreamWaitEvent(c->ostream, gsl.ev_dev, 0));
    SLIDE_CUDA(cudaMemcpyAsync(gsl.loss, gout, B * 12, cudaMemcpyDeviceToHost, c->ostream));
    SLIDE_CUDA(cudaEventRecord(gsl.ev, c->ostream));
    SLIDE_CUDA(cudaStreamWaitEvent(user, gsl.ev_dev, 0));
    gsl.used = true;
    c->g_q[c->g_qn] = slot;
    c->g_qb[c->g_qn] = B;
    ++c->g_qn;
    c->g_next = slot ^ 1;
}

// results of the oldest graph step in flight
static void graph_step_finish(slide_ctx* c, double* loss_host, int64_t* active_host) {
  SLIDE_CHECK(c->g_qn > 0, kValueError, "no graph step in flight");
  auto& gsl = c->gslot[c->g_q[0]];
  const int64_t B = c->g_qb[0];
  c->g_q[0] = c->g_q[1];
  c->g_qb[0] = c->g_qb[1];
  --c->g_qn;
  SLIDE_CUDA(cudaEventSynchronize(gsl.ev));
  for (int64_t i = 0; i < B; ++i) {
    if (loss_host) loss_host[i] = gsl.loss[i];
    if (active_host) active_host[i] = gsl.cnt[i];
    c->host_counts[0] += gsl.cnt[i];
  }
}

int slide_graph_step(slide_ctx* c, const slide_batch* bt, int64_t iteration, double* loss_host,
                     int64_t* active_host) {
  return guarded([&] {
    SLIDE_CHECK(c->g_qn == 0, kValueError, "collect the asynchronous graph steps in flight first");
    graph_step_launch(c, bt, iteration);
    graph_step_finish(c, loss_host, active_host);
  });
}

int slide_graph_step_async(slide_ctx* c, const slide_batch* bt, int64_t iteration) {
  return guarded([&] {
    graph_step_launch(c, bt, iteration);
  });
}

int slide_graph_step_wait(slide_ctx* c, double* loss_host, int64_t* active_host) {
  return guarded([&] { graph_step_finish(c, loss_host, active_host); });
}

int slide_read(slide_ctx* c, int64_t what, void* dst, int64_t max_bytes, int64_t* bytes) {
  return guarded([&] {
    SLIDE_CHECK(c->have_forward, kValueError, "nothing to read before a forward");
    const int64_t b = c->last_b, P = host_pairs(c), hp = c->hp, L = c->d.l;
    const void* src = nullptr;
    int64_t n = 0;
    switch (what) {
      case 0: src = c->h.p; n = b * hp * 4; break;
      case 1: src = c->qkeys.p; n = b * L * 4; break;
      case 2: src = c->offs.p; n = (b + 1) * 4; break;
      case 3: src = c->prow.p; n = P * 4; break;
      case 4: src = c->plab.p; n = P; break;
      case 5:
      case 6:  // probabilities / errors per pair (made from the logits after a lazy softmax)
        if (c->lazy) {
          float* tmp = c->prob_tmp.ensure<float>(std::max<int64_t>(P, 1));
          launch_lazy_pairs((int)b, c->offs.as<int32_t>(), c->prow.as<int32_t>(), c->plab.as<uint8_t>(),
                            c->grow.view(), c->z.as<float>(), c->sm_stat.as<float>(), tmp, what == 6, c->s);
          src = tmp;
        } else {
          src = what == 5 ? c->prob.p : c->delta.p;
        }
        n = P * 4;
        break;
      case 7: src = c->loss.p; n = b * 8; break;
      case 8: src = c->dh.p; n = b * hp * 4; break;
      case 9: src = c->empty.p; n = b * 4; break;
      case 10: src = c->states.p; n = b * 48; break;
      case 11:  // logits per pair, sample-major (row order under the place-free grouping)
        if (c->rows_mode) {
          float* tmp = c->prob_tmp.ensure<float>(std::max<int64_t>(P, 1));
          launch_rows_pairs((int)b, c->offs.as<int32_t>(), c->prow.as<int32_t>(), c->grow.view(), c->z.as<float>(),
                            tmp, true, c->s);
          src = tmp;
        } else {
          src = c->z.p;
        }
        n = P * 4;
        break;
      case 12: src = c->G > 1 ? c->cnt_all.p : c->cnt.p; n = b * 4; break;
      case 13: src = c->live.p; n = (1 + hp) * 4; break;
      default: throw Error(kValueError, "unknown stage");
    }
    SLIDE_CHECK(src != nullptr || n == 0, kValueError, "stage not computed");
    SLIDE_CHECK(n <= max_bytes, kValueError, "destination too small");
    if (n) SLIDE_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
    if (bytes) *bytes = n;
  });
}

int slide_topk(slide_ctx* c, int64_t k, int32_t* ids_out, int32_t* counts_out) {
  return guarded([&] {
    SLIDE_CHECK(c->have_forward, kValueError, "ranking needs a forward first");
    SLIDE_CHECK(k >= 1 && k <= 4096, kValueError, "k must be in 1..4096");
    SLIDE_CHECK(c->G == 1, kNotSupported, "ranking a sharded layer needs the gathered probabilities");
    const int b = c->last_b;
    int32_t* out = c->topk_out.ensure<int32_t>((size_t)b * k);
    int32_t* cnt = c->topk_cnt.ensure<int32_t>(b);
    launch_topk(b, c->offs.as<int32_t>(), c->prow.as<int32_t>(), c->G, c->g, c->prob.as<float>(), (int)k, out, cnt,
                c->s);
    SLIDE_CUDA(cudaMemcpyAsync(ids_out, out, (size_t)b * k * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaMemcpyAsync(counts_out, cnt, (size_t)b * 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
  });
}

// ------------------------------------------------------------- sharded step
int slide_shard_hash_rows(slide_ctx* c, uint32_t* keys) {
  return guarded([&] {
    SLIDE_CHECK(c->d.family != 0, kValueError, "layer has no LSH tables");
    c->timer.mark(c->s, kStStart);
    hash_rows(c, c->d.w2, c->n_local, keys);
    c->timer.mark(c->s, kStRebuildHash);
  });
}

__global__ void max_count_kernel(const int32_t* __restrict__ counts, int64_t n, int32_t* out) {
  int m = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    m = max(m, counts[r]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Column-sharded tables: hash this rank's W2 rows and build
// its tables over them, ids stored as global ids (local r -> r G + g).
// *max_count: the largest local bucket insert count; the caller all-reduces
// it (MAX): while G * max <= cap no global bucket can overflow and the local
// tables are exact, else the runs are exchanged (pack / reconcile).
int slide_shard_build_local(slide_ctx* c, int64_t* max_count) {
  return guarded([&] {
    SLIDE_CHECK(c->G > 1 && c->d.family != 0, kValueError, "slide_shard_* needs a sharded context with tables");
    const int64_t n = c->n_local;
    uint32_t* keys = c->rowkeys.ensure<uint32_t>((size_t)std::max<int64_t>(n, 1) * c->d.l);
    c->timer.mark(c->s, kStStart);
    hash_rows(c, c->d.w2, n, keys);
    c->timer.mark(c->s, kStRebuildHash);
    tables_build(c->tab, keys, n, (int)c->d.l, (int)c->d.key_bits, (int)c->d.capacity, (int)c->d.policy, nullptr,
                 c->s, c->G, c->g);
    int32_t* mx = c->work.ensure<int32_t>(4) + 2;
    SLIDE_CUDA(cudaMemsetAsync(mx, 0, 4, c->s));
    if (c->tab.dev.n_runs > 0) {
      max_count_kernel<<<(int)std::min<int64_t>(ceil_div(c->tab.dev.n_runs, 256), kSms * 4), 256, 0, c->s>>>(
          c->tab.dev.bcount, c->tab.dev.n_runs, mx);
      SLIDE_LAUNCH_CHECK();
    }
    int32_t h = 0;
    SLIDE_CUDA(cudaMemcpyAsync(&h, mx, 4, cudaMemcpyDeviceToHost, c->s));
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
    c->tab.n_items = c->d.n_out;
    c->timer.mark(c->s, kStRebuildBuild);
    c->host_counts[3] += 1;
    *max_count = h;
  });
}

int slide_shard_tables_pack_size(slide_ctx* c, int64_t* n) {
  return guarded([&] { *n = tables_pack_size(c->tab); });
}

int slide_shard_tables_pack(slide_ctx* c, int32_t* out) {
  return guarded([&] { tables_pack(c->tab, out, c->s); });
}

// packs: the all-gathered (G, stride) int32 packs of every rank (FIFO only)
int slide_shard_tables_reconcile(slide_ctx* c, const int32_t* packs, int64_t stride) {
  return guarded([&] {
    SLIDE_CHECK(c->G > 1, kValueError, "slide_shard_* needs a sharded context");
    SLIDE_CHECK(c->d.policy == 0, kNotSupported,
                "sharded reservoir tables need every bucket within capacity (shard_count * max bucket <= cap)");
    tables_reconcile(c->tab, packs, stride, c->G, c->g, (int)c->d.capacity, c->s);
  });
}

int slide_shard_hidden(slide_ctx* c, const slide_batch* bt, float* part_out) {
  return guarded([&] {
    SLIDE_CHECK(c->G > 1, kValueError, "slide_shard_* needs a sharded context");
    const int b = (int)bt->batch;
    SLIDE_CHECK(b >= 1 && b <= 1024, kValueError, "batch must hold 1..1024 slots");
    c->timer.mark(c->s, kStStart);
    launch_shard_hidden(c->hp, c->hg, b, bt->x_ptr, bt->x_idx, bt->x_val, c->d.w1t, part_out, c->s);
  });
}

int slide_shard_assemble(slide_ctx* c, int64_t b, const float* parts) {
  return guarded([&] {
    SLIDE_CHECK(c->G > 1, kValueError, "slide_shard_* needs a sharded context");
    SLIDE_CHECK(b >= 1 && b <= 1024, kValueError, "batch must hold 1..1024 slots");
    const int hp = c->hp;
    float* h = c->h.ensure<float>((size_t)b * hp);
    uint32_t* hmask = c->hmask.ensure<uint32_t>((size_t)b * (hp / 32));
    int32_t* live = c->live.ensure<int32_t>(1 + hp);
    launch_shard_assemble(hp, (int)c->d.hidden, c->hg, (int)b, parts, c->d.b1, h, hmask, live, live_ticket(c), c->s);
    c->timer.mark(c->s, kStHidden);
  });
}

int slide_shard_select(slide_ctx* c, const slide_batch* bt, int64_t iteration, int32_t* hist_out) {
  return guarded([&] {
    SLIDE_CHECK(c->G > 1, kValueError, "slide_shard_* needs a sharded context");
    SLIDE_CHECK(c->d.family != 0 && !bt->forced_ptr, kNotSupported, "sharded selection needs LSH tables");
    c->shard_phase = 1;
    c->shard_hist = hist_out;
    struct Reset {
      slide_ctx* c;
      ~Reset() { c->shard_phase = 0; }
    } reset{c};
    forward_impl(c, bt, iteration, 0, nullptr);
  });
}

int slide_shard_forward(slide_ctx* c, const slide_batch* bt, int64_t iteration, const int32_t* ghist,
                        float* max_out) {
  return guarded([&] {
    SLIDE_CHECK(c->G > 1, kValueError, "slide_shard_* needs a sharded context");
    c->shard_phase = 2;
    c->shard_ghist = ghist;
    struct Reset {
      slide_ctx* c;
      ~Reset() { c->shard_phase = 0; }
    } reset{c};
    forward_impl(c, bt, iteration, 0, nullptr);
    launch_softmax_max(c->last_b, c->offs.as<int32_t>(), c->z.as<float>(), max_out, c->s);
  });
}

int slide_shard_softmax_sum(slide_ctx* c, const float* gmax, float* sum_out) {
  return guarded([&] {
    SLIDE_CHECK(c->have_forward, kValueError, "no forward");
    launch_softmax_sum(c->last_b, c->offs.as<int32_t>(), c->z.as<float>(), gmax, sum_out, c->s);
  });
}

int slide_shard_softmax_finish(slide_ctx* c, const float* gmax, const float* gsum, double* loss_out) {
  return guarded([&] {
    SLIDE_CHECK(c->have_forward, kValueError, "no forward");
    const int b = c->last_b;
    launch_softmax_finish(b, c->offs.as<int32_t>(), c->plab.as<uint8_t>(), c->last_yptr, c->z.as<float>(), gmax,
                          gsum, c->prob.as<float>(), c->delta.as<float>(), loss_out, c->grow.inv.as<int32_t>(),
                          c->dsort.as<float>(), c->s);
    // loss_out[b + i] = the rank's owned active-set size of slot i (summed over ranks: |A_i|)
    launch_counts_to_f64(b, c->cnt.as<int32_t>(), loss_out + b, c->s);
  });
}

int slide_shard_hidden_grad(slide_ctx* c, float* dh_out) {
  return guarded([&] {
    SLIDE_CHECK(c->have_forward, kValueError, "no forward");
    const int b = c->last_b, hp = c->hp;
    // unmasked partial (h = null): masking commutes with the all-reduce
    launch_hidden_grad(hp, b, c->offs.as<int32_t>(), c->prow.as<int32_t>(), c->delta.as<float>(), c->d.w2, nullptr,
                       c->live.as<int32_t>(), dh_out, c->partial.ensure<float>(hidden_grad_scratch(b, hp)),
                       hg_tickets(c, b), nullptr, c->s);
  });
}

int slide_shard_update(slide_ctx* c, const float* dh) {
  return guarded([&] { backward_impl(c, 1, dh); });
}

int slide_sample_lists(const int32_t* ptr_host, const int32_t* ids_host, int64_t n_tables, int64_t width,
                       int64_t strategy, int64_t beta, int64_t min_freq, const int32_t* order_host,
                       int32_t* ids_out, int64_t* n_out, int64_t* probed, int32_t* freq_out, void* stream) {
  return guarded([&] {
    SLIDE_CHECK(n_tables >= 1 && n_tables <= 4096, kValueError, "need 1..4096 candidate lists");
    SLIDE_CHECK(width >= 1 && width < INT32_MAX, kValueError, "width must be positive");
    SLIDE_CHECK(strategy >= 0 && strategy <= 2, kValueError, "unknown sampling strategy");
    SLIDE_CHECK(beta >= 1 && min_freq >= 1, kValueError, "beta and min_freq must be positive");
    const int64_t n_ids = ptr_host[n_tables];
    for (int64_t q = 0; q < n_ids; ++q)
      SLIDE_CHECK(ids_host[q] >= 0 && ids_host[q] < width, kIndexError, "candidate id outside [0, width)");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t words = ceil_div(width, 32);
    // scratch outside the DBuf pool: no step graph needs re-capturing for it
    char* base = nullptr;
    SLIDE_CUDA(cudaMalloc(&base, (n_tables + 1 + n_tables + 2) * 4 + (n_ids + width + 1) * 4 + words * 4 +
                                     (n_ids + 1) * 4 + 64));
    struct Free {
      char* p;
      ~Free() { cudaFree(p); }
    } free_base{base};
    int32_t* d_ptr = reinterpret_cast<int32_t*>(base);
    int32_t* d_order = d_ptr + n_tables + 1;
    int32_t* d_res = d_order + n_tables;
    int32_t* d_ids = d_res + 2;
    int32_t* d_freq = d_ids + n_ids + 1;
    uint32_t* d_seen = reinterpret_cast<uint32_t*>(d_freq + width);
    int32_t* d_out = reinterpret_cast<int32_t*>(d_seen + words);
    SLIDE_CUDA(cudaMemcpyAsync(d_ptr, ptr_host, (n_tables + 1) * 4, cudaMemcpyHostToDevice, s));
    if (strategy == 0) SLIDE_CUDA(cudaMemcpyAsync(d_order, order_host, n_tables * 4, cudaMemcpyHostToDevice, s));
    if (n_ids) SLIDE_CUDA(cudaMemcpyAsync(d_ids, ids_host, n_ids * 4, cudaMemcpyHostToDevice, s));
    SLIDE_CUDA(cudaMemsetAsync(d_freq, 0, (width + words) * 4, s));
    launch_sample_lists(d_ptr, d_ids, (int)n_tables, (int)width, (int)strategy, (int)std::min<int64_t>(beta, INT32_MAX),
                        (int)min_freq, d_order, d_freq, d_seen, d_out, d_res, s);
    int32_t res[2];
    SLIDE_CUDA(cudaMemcpyAsync(res, d_res, 8, cudaMemcpyDeviceToHost, s));
    SLIDE_CUDA(cudaStreamSynchronize(s));
    if (res[0]) SLIDE_CUDA(cudaMemcpy(ids_out, d_out, (size_t)res[0] * 4, cudaMemcpyDeviceToHost));
    if (freq_out) SLIDE_CUDA(cudaMemcpy(freq_out, d_freq, (size_t)width * 4, cudaMemcpyDeviceToHost));
    *n_out = res[0];
    *probed = res[1];
  });
}

int slide_launch_count(uint64_t* out) {
  return guarded([&] { *out = g_slide_launches; });
}

int slide_profile(slide_ctx* c, int64_t on) {
  return guarded([&] {
    c->timer.collect();
    c->timer.on = on != 0;
    for (double& a : c->timer.acc) a = 0.0;
    for (int64_t& h : c->host_counts) h = 0;
    unsigned long long* ctr = c->counters.ensure<unsigned long long>(8);
    SLIDE_CUDA(cudaMemsetAsync(ctr, 0, 64, c->s));
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
  });
}

int slide_profile_read(slide_ctx* c, double* stage_ms, int64_t* counts) {
  return guarded([&] {
    c->timer.collect();
    for (int k = 0; k < 32; ++k) stage_ms[k] = c->timer.acc[k];
    unsigned long long dev[8] = {0};
    if (c->counters.p) SLIDE_CUDA(cudaMemcpy(dev, c->counters.p, 64, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 8; ++k) counts[k] = (int64_t)dev[k];
    for (int k = 0; k < 8; ++k) counts[8 + k] = c->host_counts[k];
  });
}

int slide_write(slide_ctx* c, int64_t what, const void* src, int64_t bytes) {
  return guarded([&] {
    SLIDE_CHECK(c->have_forward, kValueError, "nothing to overwrite before a forward");
    void* dst = nullptr;
    int64_t n = 0;
    if (what == 0) {
      dst = c->h.p;
      n = (int64_t)c->last_b * c->hp * 4;
    } else if (what == 6) {
      dst = c->delta.p;
      n = host_pairs(c) * 4;
    } else {
      throw Error(kValueError, "only h (0) and delta (6) can be written");
    }
    SLIDE_CHECK(bytes == n, kValueError, "size mismatch for stage write");
    if (n) SLIDE_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, c->s));
    // replayed errors in the W2 Adam's row-grouped order
    if (what == 6) {
      if (c->rows_mode)
        launch_rows_pairs(c->last_b, c->offs.as<int32_t>(), c->prow.as<int32_t>(), c->grow.view(),
                          c->delta.as<float>(), c->dsort.as<float>(), false, c->s);
      else
        launch_scatter_sorted(c->offs.as<int32_t>() + c->last_b, c->last_Pmax, c->grow.inv.as<int32_t>(),
                              c->delta.as<float>(), c->dsort.as<float>(), c->s);
    }
    // a replayed h has its own live units
    if (what == 0)
      launch_live_cols_from_h(c->hp, c->last_b, c->h.as<float>(), c->hmask.as<uint32_t>(), c->live.as<int32_t>(), c->s);
    SLIDE_CUDA(cudaStreamSynchronize(c->s));
  });
}

// ------------------------------------------------------------ host streams
int slide_pcg64_seed(const uint64_t* ent, int64_t n_ent, uint64_t* state6) {
  return guarded([&] {
    SLIDE_CHECK(n_ent >= 1 && n_ent <= 8, kValueError, "1..8 entropy words");
    Pcg64 g;
    g.seed_from(ent, (int)n_ent);
    g.store(state6);
  });
}

int slide_pcg64_permutation(uint64_t* state6, int64_t n, int64_t* out) {
  return guarded([&] {
    Pcg64 g;
    g.load(state6);
    pcg_permutation(g, out, (int)n);
    g.store(state6);
  });
}

int slide_pcg64_choice(uint64_t* state6, int64_t pop, int64_t size, int64_t* out) {
  return guarded([&] {
    SLIDE_CHECK(size >= 0 && size <= pop, kValueError,
                "Cannot take a larger sample than population when replace is False");
    Pcg64 g;
    g.load(state6);
    std::vector<int64_t> scratch((size_t)std::max<int64_t>(choice_scratch_entries(pop, size), 1));
    pcg_choice(g, pop, size, out, scratch.data());
    g.store(state6);
  });
}

int slide_mt19937_random(uint64_t* state625, int64_t n, double* out) {
  return guarded([&] {
    Mt19937 mt;
    mt.load(state625);
    for (int64_t q = 0; q < n; ++q) out[q] = mt.random();
    mt.store(state625);
  });
}

}  // extern "C"
