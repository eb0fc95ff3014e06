// Output-layer active-set selection: query -> sample -> fallback -> union
// with labels (reference network.py:225-239, samplers.py:57-120,
// tables.py:165-176).
//
// One CTA per sample.  Candidates are the ids of the L probed buckets, each
// tagged with its probe position (vanilla) or table index, plus the labels
// tagged 127; a block-wide sort of (id << 7 | tag) groups an id's
// occurrences, which gives for every distinct id its frequency (topk /
// hard_threshold), its first probe position (vanilla: the union of the
// first tau probes, tau = first prefix reaching beta distinct ids) and
// whether it is a label.  The output list is sorted ascending, label bit 31.
#include "internal.cuh"
#include "kernels.cuh"
#include <cub/cub.cuh>
#include <climits>
#include <vector>

namespace slide {

// ------------------------------------------------------------ per-slot rng
// The jump table of rng.cuh (A_k, S_k for k = 0..kPcgJump), built once.
const u128* pcg_jump_table() {
  static const u128* table = [] {
    std::vector<u128> h(2 * (size_t)(kPcgJump + 1));
    u128 A = 1, S = 0;
    for (int k = 0; k <= kPcgJump; ++k) {
      h[2 * k] = A;
      h[2 * k + 1] = S;
      S = S * Pcg64::mult() + 1;
      A = A * Pcg64::mult();
    }
    u128* d = nullptr;
    SLIDE_CUDA(cudaMalloc(&d, h.size() * sizeof(u128)));
    SLIDE_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(u128), cudaMemcpyHostToDevice));
    return (const u128*)d;
  }();
  return table;
}

// default_rng((seed, iteration, slot)) (network.py:353) or an explicit
// Generator state; vanilla draws permutation(L) first (samplers.py:69).
// One warp per slot: every lane seeds (the same arithmetic), the warp makes
// the stream's first kSlotRngOut outputs in parallel (jump-ahead), lane 0
// walks them through the permutation's rejection draws.
constexpr int kSlotRngOut = 128;
constexpr int kSlotRngWarps = 8;

__global__ void __launch_bounds__(kSlotRngWarps * 32) slot_rng_kernel(int b, uint64_t seed, int64_t iteration,
                                                                      const int64_t* iter_dev, int64_t slot_offset,
                                                                      int l, int vanilla,
                                                                      const uint64_t* __restrict__ ext,
                                                                      uint64_t* __restrict__ states,
                                                                      uint8_t* __restrict__ order, const u128* jump) {
  __shared__ uint64_t buf[kSlotRngWarps][kSlotRngOut];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSlotRngWarps + warp;
  if (i >= b) return;
  if (iter_dev) iteration = *iter_dev;  // graph replays read the step number from memory
  Pcg64 g;
  if (ext) {
    g.load(ext + 6 * i);
  } else {
    uint64_t ent[3] = {seed, (uint64_t)iteration, (uint64_t)(slot_offset + i)};
    g.seed_from(ent, 3);
  }
  if (vanilla) {
    __shared__ uint8_t perm_s[kSlotRngWarps][64];
    pcg_fill(g, buf[warp], kSlotRngOut, lane, 32, jump);
    for (int p = lane; p < l; p += 32) perm_s[warp][p] = (uint8_t)p;
    __syncwarp();
    if (lane == 0) {
      // permutation(L): Fisher-Yates with random_interval's masked
      // rejection, walked directly over the buffered 32-bit values
      const uint64_t* bw = buf[warp];
      const uint32_t h0 = g.has32 ? 1u : 0u;
      const int avail = 2 * kSlotRngOut + (int)h0;
      int t = 0;
      bool ok = true;
      for (int p = l - 1; p >= 1 && ok; --p) {
        uint32_t mask = (uint32_t)p;
        mask |= mask >> 1;
        mask |= mask >> 2;
        mask |= mask >> 4;
        mask |= mask >> 8;
        mask |= mask >> 16;
        uint32_t v;
        do {
          if (t >= avail) {
            ok = false;
            break;
          }
          int64_t q = t++;
          uint32_t u;
          if (h0 && q == 0) {
            u = g.u32;
          } else {
            q -= h0;
            u = (q & 1) ? (uint32_t)(bw[q >> 1] >> 32) : (uint32_t)bw[q >> 1];
          }
          v = u & mask;
        } while (v > (uint32_t)p);
        if (!ok) break;
        const uint8_t x = perm_s[warp][p];
        perm_s[warp][p] = perm_s[warp][v];
        perm_s[warp][v] = x;
      }
      if (ok) {  // the generator after t values
        const int64_t tt = t - (int64_t)h0;
        const int64_t n64 = tt > 0 ? (tt + 1) >> 1 : 0;
        Pcg64 e = g;
        const u128 A = jump[2 * n64], S = jump[2 * n64 + 1];
        e.state = A * g.state + S * g.inc;
        if (tt > 0) {
          e.has32 = (uint32_t)(tt & 1);
          e.u32 = (uint32_t)(bw[n64 - 1] >> 32);
        } else {
          e.has32 = t == 0 ? g.has32 : 0u;  // only the buffered value (if any) was used
        }
        g = e;
      } else {  // more rejections than buffered values: the serial walk
        PcgBuf pb(g, bw, kSlotRngOut, jump);
        uint8_t a[64];
        pcg_permutation(pb, a, l);
        pb.finish(g);
        for (int p = 0; p < l; ++p) perm_s[warp][p] = a[p];
      }
      for (int p = 0; p < l; ++p) order[(int64_t)i * l + p] = perm_s[warp][p];
    }
  }
  if (lane == 0) g.store(states + 6 * i);
}

void launch_slot_rng(int b, uint64_t seed, int64_t it, const int64_t* it_dev, int64_t off, int l, int vanilla,
                     const uint64_t* ext, uint64_t* states, uint8_t* order, cudaStream_t s) {
  slot_rng_kernel<<<(int)ceil_div(b, kSlotRngWarps), kSlotRngWarps * 32, 0, s>>>(b, seed, it, it_dev, off, l,
                                                                                 vanilla, ext, states, order,
                                                                                 pcg_jump_table());
  SLIDE_LAUNCH_CHECK();
}

// ----------------------------------------------------------------- select
constexpr int kSelThreads = 256;
constexpr uint32_t kLabelTag = 127;

template <int ITEMS>
struct SelSmem {
  using Sort = cub::BlockRadixSort<uint32_t, kSelThreads, ITEMS>;
  static constexpr int CAP = kSelThreads * ITEMS;
  static constexpr size_t kA = sizeof(typename Sort::TempStorage), kB = (size_t)CAP * 4;
  static constexpr size_t kRegion2 = ((kA > kB ? kA : kB) + 15) & ~(size_t)15;
  __host__ __device__ static constexpr size_t region2() { return kRegion2; }
  __host__ __device__ static constexpr size_t bytes() { return (size_t)CAP * 4 + kRegion2 + CAP; }
};

template <int ITEMS>
__global__ void __launch_bounds__(kSelThreads) select_kernel(SelectArgs a) {
  using S = SelSmem<ITEMS>;
  using Scan = cub::BlockScan<int, kSelThreads>;
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* cand = reinterpret_cast<uint32_t*>(sm);
  uint8_t* region2 = sm + (size_t)S::CAP * 4;
  uint32_t* uid = reinterpret_cast<uint32_t*>(region2);
  uint8_t* ufreq = region2 + S::region2();
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int s_start[64], s_len[64], s_off[65], s_tag[64], s_hist[130];
  __shared__ int s_misc[4];

  const int i = blockIdx.x, tid = threadIdx.x, L = a.l;
  if (a.tier == 2 && !a.big[i]) return;  // taken by the small-capacity pass
  const int y0 = a.y_ptr[i], ny = a.y_ptr[i + 1] - y0;
  // 1. probe the L tables (exactly L lookups, tables.py:171-176)
  if (tid < L) {
    uint32_t skey = ((uint32_t)tid << a.tab.key_bits) | a.qkeys[(int64_t)i * L + tid];
    int run = tables_lookup(a.tab, skey);
    s_start[tid] = run >= 0 ? a.tab.bstart[run] : 0;
    s_len[tid] = run >= 0 ? a.tab.blen[run] : 0;
    if (a.strategy != 0) s_tag[tid] = tid;
    else s_tag[a.order[(int64_t)i * L + tid]] = tid;  // probe position of table order[p] is p
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int t = 0; t < L; ++t) {
      s_off[t] = acc;
      acc += s_len[t];
    }
    s_off[L] = acc;
  }
  for (int q = tid; q < 130; q += kSelThreads) s_hist[q] = 0;
  __syncthreads();
  const int C = s_off[L] + ny;
  if (a.tier == 1) {  // small-capacity pass: samples that do not fit are left to the second pass
    const bool over = C > S::CAP;
    if (tid == 0) a.big[i] = over;
    if (over) return;
  }
  if (tid == 0 && a.cand_ctr) atomicAdd(a.cand_ctr, (unsigned long long)s_off[L]);
  // 2. gather (id << 7 | tag); labels carry tag 127
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int t = warp; t < L; t += kSelThreads / 32) {
      const int32_t* src = a.tab.ids + s_start[t];
      uint32_t tag = (uint32_t)s_tag[t];
      for (int j = lane; j < s_len[t]; j += 32) cand[s_off[t] + j] = ((uint32_t)src[j] << 7) | tag;
    }
    for (int j = tid; j < ny; j += kSelThreads)
      cand[s_off[L] + j] = ((uint32_t)a.y_idx[y0 + j] << 7) | kLabelTag;
  }
  __syncthreads();
  // 3. sort
  if (C <= kSelThreads) {
    uint32_t key = tid < C ? cand[tid] : 0u;
    int rank = 0;
    if (tid < C)
      for (int s2 = 0; s2 < C; ++s2) rank += cand[s2] < key;
    __syncthreads();
    if (tid < C) cand[rank] = key;  // keys are unique
    __syncthreads();
  } else {
    uint32_t keys[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      int k = tid * ITEMS + q;
      keys[q] = k < C ? cand[k] : 0xffffffffu;
    }
    typename S::Sort(*reinterpret_cast<typename S::Sort::TempStorage*>(region2)).Sort(keys, 0, a.sort_bits);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      int k = tid * ITEMS + q;
      if (k < C) cand[k] = keys[q];
    }
    __syncthreads();
  }
  // 4. distinct ids: first tag (min probe position), frequency, label flag
  const int ch = (C + kSelThreads - 1) / kSelThreads;
  const int k0 = min(tid * ch, C), k1 = min(k0 + ch, C);
  int nh = 0;
  for (int k = k0; k < k1; ++k) nh += (k == 0 || (cand[k - 1] >> 7) != (cand[k] >> 7));
  int hofs, U;
  Scan(scan_tmp).ExclusiveSum(nh, hofs, U);
  __syncthreads();
  for (int k = k0; k < k1; ++k) {
    uint32_t id = cand[k] >> 7;
    if (k != 0 && (cand[k - 1] >> 7) == id) continue;
    int e = k + 1;
    while (e < C && (cand[e] >> 7) == id) ++e;
    int lab = (cand[e - 1] & 127u) == kLabelTag;
    int freq = e - k - lab;
    uid[hofs] = cand[k];
    ufreq[hofs] = (uint8_t)(freq | (lab << 7));
    ++hofs;
  }
  __syncthreads();
  // 5. sampler rule on the non-label occurrences
  const int uch = (U + kSelThreads - 1) / kSelThreads;
  const int u0 = min(tid * uch, U), u1 = min(u0 + uch, U);
  if (a.strategy == 0) {  // vanilla
    for (int u = u0; u < u1; ++u)
      if (ufreq[u] & 127) atomicAdd(&s_hist[uid[u] & 127u], 1);
  } else if (a.strategy == 1) {  // topk
    for (int u = u0; u < u1; ++u)
      if (ufreq[u] & 127) atomicAdd(&s_hist[ufreq[u] & 127], 1);
  }
  __syncthreads();
  if (a.hist_out) {  // sharded phase 1: this rank's counts, summed over ranks by the caller
    int nsel_local = 0;
    if (a.strategy == 2)
      for (int u = u0; u < u1; ++u) nsel_local += (ufreq[u] & 127) >= a.min_freq;
    else
      for (int u = u0; u < u1; ++u) nsel_local += (ufreq[u] & 127) > 0;
    int before, all;
    Scan(scan_tmp).ExclusiveSum(nsel_local, before, all);
    int32_t* ho = a.hist_out + (int64_t)i * (L + 1);
    for (int p = tid; p < L; p += kSelThreads) ho[p] = a.strategy == 0 ? s_hist[p] : 0;
    if (tid == 0) ho[L] = all;
    return;
  }
  const int32_t* gh = a.ghist ? a.ghist + (int64_t)i * (L + 1) : nullptr;
  if (tid == 0) {
    if (a.strategy == 0) {
      int acc = 0, tau = L;
      for (int p = 0; p < L; ++p) {
        acc += gh ? gh[p] : s_hist[p];
        if (acc >= a.beta) {
          tau = p + 1;
          break;
        }
      }
      s_misc[0] = tau;
    } else if (a.strategy == 1) {
      int total = 0;
      for (int f = 1; f <= 127; ++f) total += s_hist[f];
      int F = 1, need = 1 << 30;
      if (total > a.beta) {
        int cum = 0;
        for (int f = 127; f >= 1; --f) {
          if (cum + s_hist[f] >= a.beta) {
            F = f;
            need = a.beta - cum;
            break;
          }
          cum += s_hist[f];
        }
      }
      s_misc[0] = F;
      s_misc[1] = need;
    }
  }
  __syncthreads();
  int eq_before = 0;
  if (a.strategy == 1) {
    int F = s_misc[0], neq = 0;
    for (int u = u0; u < u1; ++u) neq += (ufreq[u] & 127) == F;
    int tot;
    Scan(scan_tmp).ExclusiveSum(neq, eq_before, tot);
    __syncthreads();
  }
  int nkeep = 0, nsel = 0;
  const int tau = s_misc[0], F = s_misc[0], need = s_misc[1];
  // selected flag computed twice (count, then write) to avoid a smem array
  auto selected = [&](int u, int& eqc) -> bool {
    int f = ufreq[u] & 127;
    if (f == 0) return false;
    if (a.strategy == 0) return (int)(uid[u] & 127u) < tau;
    if (a.strategy == 1) {
      if (f > F) return true;
      if (f == F) return eqc++ < need;
      return false;
    }
    if (a.strategy == 3) return true;  // vanilla with beta >= L*cap: every table is probed
    return f >= a.min_freq;
  };
  {
    int eqc = eq_before;
    for (int u = u0; u < u1; ++u) {
      bool sl = selected(u, eqc);
      nsel += sl;
      nkeep += sl || (ufreq[u] >> 7);
    }
  }
  int any = __syncthreads_or(nsel > 0);
  if (gh) any = gh[L] > 0;  // sharded: empty only when every rank's rule selects nothing
  if (!any) {
    if (tid == 0) {
      a.empty[i] = 1;
      a.cnt[i] = 0;
    }
    return;
  }
  int kofs, K;
  Scan(scan_tmp).ExclusiveSum(nkeep, kofs, K);
  int32_t* out = a.act + (int64_t)i * a.cap_max;
  {
    int eqc = eq_before;
    for (int u = u0; u < u1; ++u) {
      bool sl = selected(u, eqc);
      int lab = ufreq[u] >> 7;
      if (sl || lab) out[kofs++] = (int32_t)((uid[u] >> 7) | ((uint32_t)lab << 31));
    }
  }
  if (tid == 0) {
    a.empty[i] = 0;
    a.cnt[i] = K;
  }
}

template <int ITEMS>
static void launch_select_t(const SelectArgs& a, cudaStream_t s) {
  size_t smem = SelSmem<ITEMS>::bytes();
  SLIDE_CUDA(cudaFuncSetAttribute(select_kernel<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  select_kernel<ITEMS><<<a.b, kSelThreads, smem, s>>>(a);
  SLIDE_LAUNCH_CHECK();
}

void launch_select(const SelectArgs& a0, int max_candidates, cudaStream_t s, int64_t expected, int32_t* big) {
  SLIDE_CHECK(a0.l <= 64, kNotSupported, "at most 64 tables supported on the device path");
  SelectArgs a = a0;
  // The kernel's shared memory is sized by the BOUND on a sample's candidates
  // (L x capacity + labels: 150 KB, one CTA per SM at L = 64, capacity 128)
  // while sparse buckets hold a handful of ids: a first pass with room for
  // 1,024 candidates (8+ CTAs per SM) takes every sample that fits and flags
  // the others for the full-size pass, whose CTAs otherwise exit at once.
  if (big && max_candidates > kSelThreads * 16 && expected <= kSelThreads * 2) {
    a.big = big;
    a.tier = 1;
    launch_select_t<4>(a, s);
    a.tier = 2;
  }
  if (max_candidates <= kSelThreads * 16) launch_select_t<16>(a, s);
  else if (max_candidates <= kSelThreads * 32) launch_select_t<32>(a, s);
  else if (max_candidates <= kSelThreads * 64) launch_select_t<64>(a, s);
  else throw Error(kNotSupported, "L*capacity + labels exceeds 16384 candidates per sample");
}

// Full-union selection (vanilla with beta >= L*cap: every table is probed and
// every id kept, samplers.py:57-87): a shared-memory bitmap over the N output
// ids replaces the sort.  The sampler result is empty exactly when all L
// probed buckets are empty.
constexpr int kUnionThreads = 1024;

__global__ void __launch_bounds__(kUnionThreads) select_union_kernel(SelectArgs a, int words) {
  using Scan = cub::BlockScan<int, kUnionThreads>;
  extern __shared__ __align__(16) uint32_t bm[];  // [words] ids, then [words] labels
  uint32_t* lb = bm + words;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int s_start[64], s_len[64], s_tot;
  const int i = blockIdx.x, tid = threadIdx.x, L = a.l;
  const int y0 = a.y_ptr[i], ny = a.y_ptr[i + 1] - y0;
  for (int w = tid; w < 2 * words; w += kUnionThreads) bm[w] = 0u;
  if (tid < L) {
    const uint32_t skey = ((uint32_t)tid << a.tab.key_bits) | a.qkeys[(int64_t)i * L + tid];
    const int run = tables_lookup(a.tab, skey);
    s_start[tid] = run >= 0 ? a.tab.bstart[run] : 0;
    s_len[tid] = run >= 0 ? a.tab.blen[run] : 0;
  }
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int q = 0; q < L; ++q) t += s_len[q];
    s_tot = t;
    if (a.cand_ctr) atomicAdd(a.cand_ctr, (unsigned long long)t);
  }
  __syncthreads();
  if (a.hist_out) {  // sharded phase 1: this rank's retrieved count (ids are disjoint across ranks)
    int32_t* ho = a.hist_out + (int64_t)i * (L + 1);
    for (int p = tid; p <= L; p += kUnionThreads) ho[p] = p == L ? s_tot : 0;
    return;
  }
  if (a.ghist ? a.ghist[(int64_t)i * (L + 1) + L] == 0 : s_tot == 0) {
    // nothing retrieved (on any rank): the fallback kernel takes this slot
    if (tid == 0) {
      a.empty[i] = 1;
      a.cnt[i] = 0;
    }
    return;
  }
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int t = warp; t < L; t += kUnionThreads / 32) {
      const int32_t* src = a.tab.ids + s_start[t];
      for (int j = lane; j < s_len[t]; j += 32) {
        const uint32_t id = (uint32_t)src[j];
        atomicOr(&bm[id >> 5], 1u << (id & 31));
      }
    }
    for (int j = tid; j < ny; j += kUnionThreads) {
      const uint32_t id = (uint32_t)a.y_idx[y0 + j];
      atomicOr(&bm[id >> 5], 1u << (id & 31));
      atomicOr(&lb[id >> 5], 1u << (id & 31));
    }
  }
  __syncthreads();
  const int ch = (words + kUnionThreads - 1) / kUnionThreads;
  const int w0 = min(tid * ch, words), w1 = min(w0 + ch, words);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
  int ofs, total;
  Scan(scan_tmp).ExclusiveSum(cnt, ofs, total);
  int32_t* out = a.act + (int64_t)i * a.cap_max;
  for (int w = w0; w < w1; ++w) {
    uint32_t bits = bm[w];
    const uint32_t labs = lb[w];
    while (bits) {
      const int bit = __ffs(bits) - 1;
      bits &= bits - 1;
      out[ofs++] = (int32_t)((uint32_t)(w * 32 + bit) | (((labs >> bit) & 1u) << 31));
    }
  }
  if (tid == 0) {
    a.empty[i] = 0;
    a.cnt[i] = total;
  }
}

bool launch_select_union(const SelectArgs& a, int64_t n_out, cudaStream_t s) {
  const int words = (int)ceil_div(n_out, 32);
  const size_t smem = (size_t)words * 8;
  if (smem > 200 * 1024) return false;
  if (smem > 48 * 1024)
    SLIDE_CUDA(cudaFuncSetAttribute(select_union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  select_union_kernel<<<a.b, kUnionThreads, smem, s>>>(a, words);
  SLIDE_LAUNCH_CHECK();
  return true;
}

// --------------------------------------------------------------- fallback
// Empty sampler result: beta uniform ids without replacement from the slot's
// generator (network.py:229-231), union labels, sorted (network.py:236-238).
// Thread 0 replays numpy's choice() serially; the CTA then emits the id set
// in ascending order from a per-slot bitmap.
constexpr int kFbSortItems = 4;  // sets of <= 1024 ids (beta + labels) are sorted in the block

__global__ void __launch_bounds__(256) fallback_kernel(FallbackArgs a) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage scan_tmp;
  extern __shared__ __align__(16) int64_t fb_smem[];
  const int i = blockIdx.x, tid = threadIdx.x;
  if (!a.empty[i]) return;
  int64_t* ids = a.fb_ids + (int64_t)i * a.want;
  // the slot's stream: every thread derives the same base state; its
  // outputs are made in parallel (jump-ahead) and thread 0 walks them
  // through the draws (rng.cuh PcgBuf) -- the serial part is the hash-set /
  // shuffle bookkeeping, not the 128-bit generator steps
  __shared__ uint64_t rbuf_s[kFbSmemOutputs];
  __shared__ uint64_t g_s[6];
  Pcg64 g;
  if (a.states_ready) {
    g.load(a.states + 6 * i);
  } else {  // slot stream not drawn yet (full-union vanilla): seed + probe order first
    const int64_t it = a.iter_dev ? *a.iter_dev : a.iteration;
    uint64_t ent[3] = {a.seed, (uint64_t)it, (uint64_t)(a.slot_offset + i)};
    g.seed_from(ent, 3);
    if (a.vanilla) {
      pcg_fill(g, rbuf_s, 128, tid, 256, a.jump);
      __syncthreads();
      if (tid == 0) {
        PcgBuf pb(g, rbuf_s, 128, a.jump);
        uint8_t perm[64];
        pcg_permutation(pb, perm, a.l);
        pb.finish(g);
        g.store(g_s);
      }
      __syncthreads();
      g.load(g_s);
    }
  }
  uint64_t* rbuf = a.rng_n <= kFbSmemOutputs ? rbuf_s : a.rng_buf + (int64_t)i * a.rng_n;
  pcg_fill(g, rbuf, a.rng_n, tid, 256, a.jump);
  __syncthreads();
  // Floyd's choice in parallel.  The draws (Floyd's `size`, then the
  // final shuffle's size - 1) are Lemire bounded draws on the stream's
  // 32-bit values; draw k takes value k + (values rejected before it).  All
  // draws are evaluated at once; the first draw that lands in its rejection
  // zone (p ~ range / 2^32) shifts every later draw by one value and the
  // remainder is re-evaluated -- one extra round per rejection.  Floyd then
  // keeps val_j unless an earlier id equals it (then j): collisions are
  // resolved against the earlier values and verified against the earlier
  // outputs; anything else (a substitution colliding again, too few buffered
  // values) takes thread 0's serial replay below.
  __shared__ int fl_bad, fl_first, fl_shift;
  __shared__ uint32_t fl_val[256 * kFbSortItems];
  const int64_t size = a.want, base = a.n - a.want;
  const bool try_fast = !choice_uses_tail(a.n, size) && size <= 256 * kFbSortItems && a.n <= 0xffffffffll &&
                        base >= 1;
  if (try_fast) {
    const uint32_t h0 = g.has32 ? 1u : 0u;
    const int64_t avail = 2 * (int64_t)a.rng_n + h0;  // buffered 32-bit values
    auto u32_at = [&](int64_t t) -> uint32_t {  // the stream's t-th 32-bit value (numpy's buffered halves)
      if (h0) {
        if (t == 0) return g.u32;
        t -= 1;
      }
      const uint64_t v = rbuf[t >> 1];
      return (t & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
    };
    const int D = (int)(2 * size - 1);
    if (tid == 0) {
      fl_bad = 0;
      fl_shift = 0;
    }
    int start = 0;
    while (true) {
      if (tid == 0) fl_first = INT_MAX;
      __syncthreads();
      const int shift = fl_shift;
      for (int k = start + tid; k < D; k += 256) {
        const int64_t idx = k + shift;
        if (idx >= avail) {
          atomicOr(&fl_bad, 1);
          continue;
        }
        const uint32_t rng = k < size ? (uint32_t)(base + k) : (uint32_t)(2 * size - 1 - k);
        const uint32_t rx = rng + 1u;
        const uint64_t m = (uint64_t)u32_at(idx) * rx;
        const uint32_t left = (uint32_t)m;
        if (left < rx && left < (0xffffffffu - rng) % rx) atomicMin(&fl_first, k);
        if (k < size) fl_val[k] = (uint32_t)(m >> 32);
      }
      __syncthreads();
      const int first = fl_first;
      if (first == INT_MAX || fl_bad) break;
      start = first;  // draw `first` retries on the next value; the rest move up by one
      __syncthreads();
      if (tid == 0) fl_shift = shift + 1;
    }
    __syncthreads();
    // Floyd's set: val_j, or j when an earlier id equals val_j
    if (!fl_bad) {
      for (int j = tid; j < size; j += 256) {
        const uint32_t v = fl_val[j];
        bool coll = false;
        for (int k = 0; k < j; ++k) coll |= fl_val[k] == v;
        ids[j] = coll ? (int64_t)(base + j) : (int64_t)v;
      }
      __syncthreads();
      for (int j = tid; j < size; j += 256) {  // verify against the outputs themselves
        const uint32_t v = fl_val[j];
        bool in = false, coll = false;
        for (int k = 0; k < j; ++k) {
          in |= (uint32_t)ids[k] == v;
          coll |= fl_val[k] == v;
        }
        if (in != coll) atomicOr(&fl_bad, 2);
      }
      __syncthreads();
    }
    if (fl_bad == 0 && tid == 0) {  // the generator after the consumed values
      const int64_t t = (int64_t)D + fl_shift - h0;
      const int64_t n64 = (t + 1) >> 1;
      Pcg64 e = g;
      const u128 A = a.jump[2 * n64], S = a.jump[2 * n64 + 1];
      e.state = A * g.state + S * g.inc;
      e.has32 = (uint32_t)(t & 1);
      // numpy keeps the last 64-bit value's high half as `uinteger` (stale once used)
      e.u32 = n64 > 0 ? (uint32_t)(rbuf[n64 - 1] >> 32) : g.u32;
      e.store(a.states + 6 * i);
    }
  }
  if (!try_fast || fl_bad != 0) if (tid == 0) {
    PcgBuf pb(g, rbuf, a.rng_n, a.jump);
    int64_t* scratch = a.smem_scratch ? fb_smem : a.scratch + (int64_t)i * a.scratch_per_slot;
    pcg_choice(pb, a.n, a.want, ids, scratch, /*keep_order=*/false);  // the ids go into a bitmap
    pb.finish(g);
    g.store(a.states + 6 * i);
  }
  __syncthreads();
  const int y0 = a.y_ptr[i], ny = a.y_ptr[i + 1] - y0;
  const int n = (int)a.want + ny;
  auto key_at = [&](int k) -> uint32_t {
    return k < a.want ? (uint32_t)ids[k] << 1 : ((uint32_t)a.y_idx[y0 + k - a.want] << 1) | 1u;
  };
  int32_t* out = a.act + (int64_t)i * a.cap_max;
  if (n <= 256) {
    // the usual case (beta + labels <= 256): keys (id << 1 | label) are
    // distinct, so each one's rank is the count of smaller keys; keep the
    // last of each id's run (a label sorts after the same id drawn)
    __shared__ uint32_t kin[256], ks[256];
    if (tid < n) kin[tid] = key_at(tid);
    __syncthreads();
    if (tid < n) {
      const uint32_t me = kin[tid];
      int r = 0;
      for (int q = 0; q < n; ++q) r += kin[q] < me;
      ks[r] = me;
    }
    __syncthreads();
    const bool keep = tid < n && (tid + 1 == n || (ks[tid + 1] >> 1) != (ks[tid] >> 1));
    int ofs, total;
    Scan(scan_tmp).ExclusiveSum(keep ? 1 : 0, ofs, total);
    if (keep) out[ofs] = (int32_t)((ks[tid] >> 1) | ((ks[tid] & 1u) << 31));
    if (tid == 0) a.cnt[i] = total;
    return;
  }
  if (n <= 256 * kFbSortItems) {
    using Sort = cub::BlockRadixSort<uint32_t, 256, kFbSortItems>;
    __shared__ typename Sort::TempStorage sort_tmp;
    int end_bit = 2;
    while (((int64_t)1 << (end_bit - 1)) < a.n) ++end_bit;  // id bits + the label bit
    uint32_t key[kFbSortItems];
#pragma unroll
    for (int q = 0; q < kFbSortItems; ++q) {
      const int k = tid * kFbSortItems + q;
      key[q] = k < n ? key_at(k) : 0xffffffffu;
    }
    Sort(sort_tmp).Sort(key, 0, end_bit);  // blocked: thread t holds sorted items [t * kFbSortItems, ...)
    __shared__ uint32_t last_s[256];
    last_s[tid] = key[0];
    __syncthreads();
    const uint32_t nxt0 = tid + 1 < 256 ? last_s[tid + 1] : 0xffffffffu;  // first item of the next thread
    int keep[kFbSortItems], m = 0;
#pragma unroll
    for (int q = 0; q < kFbSortItems; ++q) {
      const uint32_t nx = q + 1 < kFbSortItems ? key[q + 1] : nxt0;
      keep[q] = key[q] != 0xffffffffu && (nx == 0xffffffffu || (nx >> 1) != (key[q] >> 1));
      m += keep[q];
    }
    int ofs, total;
    __syncthreads();  // last_s reads done before the scan storage is reused
    Scan(scan_tmp).ExclusiveSum(m, ofs, total);
#pragma unroll
    for (int q = 0; q < kFbSortItems; ++q)
      if (keep[q]) out[ofs++] = (int32_t)((key[q] >> 1) | ((key[q] & 1u) << 31));
    if (tid == 0) a.cnt[i] = total;
    return;
  }
  uint32_t* bm = a.bitmap + (int64_t)i * a.words;
  for (int64_t k = tid; k < a.want; k += 256) {
    int64_t id = ids[k];
    atomicOr(&bm[id >> 5], 1u << (id & 31));
  }
  for (int k = tid; k < ny; k += 256) {
    int id = a.y_idx[y0 + k];
    atomicOr(&bm[id >> 5], 1u << (id & 31));
  }
  __syncthreads();
  const int64_t ch = (a.words + 255) / 256;
  const int64_t w0 = tid * ch < a.words ? tid * ch : a.words;
  const int64_t w1 = w0 + ch < a.words ? w0 + ch : a.words;
  int cnt = 0;
  for (int64_t w = w0; w < w1; ++w) cnt += __popc(bm[w]);
  int ofs, total;
  Scan(scan_tmp).ExclusiveSum(cnt, ofs, total);
  // (out: the slot's active list, above)
  const int32_t* lab = a.y_idx + y0;
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t bits = bm[w];
    while (bits) {
      int bpos = __ffs(bits) - 1;
      bits &= bits - 1;
      int id = (int)(w * 32 + bpos);
      int lo = 0, hi = ny;  // labels sorted: binary search
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (lab[mid] < id) lo = mid + 1;
        else hi = mid;
      }
      int is_lab = lo < ny && lab[lo] == id;
      out[ofs++] = (int32_t)((uint32_t)id | ((uint32_t)is_lab << 31));
    }
    bm[w] = 0u;
  }
  if (tid == 0) a.cnt[i] = total;
}

void launch_fallback(const FallbackArgs& a, int b, cudaStream_t s) {
  size_t smem = a.smem_scratch ? (size_t)a.scratch_per_slot * 8 : 0;
  if (smem > 48 * 1024)
    SLIDE_CUDA(cudaFuncSetAttribute(fallback_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fallback_kernel<<<b, 256, smem, s>>>(a);
  SLIDE_LAUNCH_CHECK();
}

// ------------------------------------------- dense / forced active sets
// No LSH on the layer: every neuron is active (network.py:234-235).  Forced
// sets (forward(forced_active=...), network.py:258-259) replace selection.
__global__ void explicit_active_kernel(int b, int64_t n, const int32_t* __restrict__ fptr,
                                       const int32_t* __restrict__ fidx, const int32_t* __restrict__ y_ptr,
                                       const int32_t* __restrict__ y_idx, int64_t cap_max,
                                       int32_t* __restrict__ act, int32_t* __restrict__ cnt,
                                       int32_t* __restrict__ empty) {
  const int i = blockIdx.x;
  const int y0 = y_ptr[i], ny = y_ptr[i + 1] - y0;
  int64_t m = fptr ? (int64_t)(fptr[i + 1] - fptr[i]) : n;
  int32_t* out = act + (int64_t)i * cap_max;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    int id = fptr ? fidx[fptr[i] + k] : (int)k;
    int lo = 0, hi = ny;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (y_idx[y0 + mid] < id) lo = mid + 1;
      else hi = mid;
    }
    int is_lab = lo < ny && y_idx[y0 + lo] == id;
    out[k] = (int32_t)((uint32_t)id | ((uint32_t)is_lab << 31));
  }
  if (threadIdx.x == 0) {
    cnt[i] = (int32_t)m;
    empty[i] = 0;
  }
}

void launch_explicit_active(int b, int64_t n, const int32_t* fptr, const int32_t* fidx, const int32_t* y_ptr,
                            const int32_t* y_idx, int64_t cap_max, int32_t* act, int32_t* cnt, int32_t* empty,
                            cudaStream_t s) {
  explicit_active_kernel<<<b, 256, 0, s>>>(b, n, fptr, fidx, y_ptr, y_idx, cap_max, act, cnt, empty);
  SLIDE_LAUNCH_CHECK();
}

// ------------------------------------------------------------- compaction
// Exclusive scan of per-slot counts (B <= 1024) and the sample-major pair
// list: row id, slot, label flag.
// Pair rows are local W2 rows: id / shard_count (identity when unsharded).
// Each CTA (one sample) sums the counts of the samples before it itself --
// no separate offsets pass; CTA 0 also writes every offset for the later
// stages (the counts are B <= 1024 ints).
__global__ void __launch_bounds__(1024) pairs_kernel(int b, const int32_t* __restrict__ act, int64_t cap_max,
                                                     const int32_t* __restrict__ cnt, int shard_count,
                                                     int32_t* __restrict__ offs, int32_t* __restrict__ prow,
                                                     int32_t* __restrict__ pslot, uint8_t* __restrict__ plab,
                                                     uint32_t* __restrict__ mask, int wpk,
                                                     unsigned long long* __restrict__ status, int32_t* ctr,
                                                     int64_t n_tiles, uint32_t* __restrict__ lmask) {
  if (mask) {  // the row grouping's scan tiles, reset for its scan kernel
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_tiles; q += (int64_t)gridDim.x * blockDim.x)
      status[q] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) *ctr = 0;
  }
  using Red = cub::BlockReduce<int, 1024>;
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ union {
    typename Red::TempStorage r;
    typename Scan::TempStorage s;
  } tmp;
  __shared__ int s_o;
  const int i = blockIdx.x;
  const int c = threadIdx.x < b ? cnt[threadIdx.x] : 0;
  if (i == 0) {
    int o, total;
    Scan(tmp.s).ExclusiveSum(c, o, total);
    if (threadIdx.x < b) offs[threadIdx.x] = o;
    if (threadIdx.x == 0) {
      offs[b] = total;
      s_o = 0;
    }
  } else {
    const int o = Red(tmp.r).Sum(threadIdx.x < i ? c : 0);
    if (threadIdx.x == 0) s_o = o;
  }
  __syncthreads();
  const int o = s_o, n = cnt[i];
  const int32_t* src = act + (int64_t)i * cap_max;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    uint32_t v = (uint32_t)src[k];
    const uint32_t id = v & 0x7fffffffu;
    const uint32_t row = shard_count == 1 ? id : id / (uint32_t)shard_count;
    prow[o + k] = (int32_t)row;
    pslot[o + k] = i;
    plab[o + k] = (uint8_t)(v >> 31);
    if (mask) atomicOr(&mask[(int64_t)row * wpk + (i >> 5)], 1u << (i & 31));  // the row's slot mask
    if (lmask && (v >> 31)) atomicOr(&lmask[(int64_t)row * wpk + (i >> 5)], 1u << (i & 31));  // a label pair
  }
}

void launch_pairs(int b, const int32_t* act, int64_t cap_max, const int32_t* cnt, int32_t* offs, int shard_count,
                  int32_t* prow, int32_t* pslot, uint8_t* plab, cudaStream_t s, uint32_t* mark_mask, int mark_wpk,
                  unsigned long long* mark_status, int32_t* mark_ctr, int64_t mark_tiles, uint32_t* mark_lmask) {
  SLIDE_CHECK(b <= 1024, kNotSupported, "batch size above 1024 not supported on the device path");
  pairs_kernel<<<b, 1024, 0, s>>>(b, act, cap_max, cnt, shard_count, offs, prow, pslot, plab, mark_mask, mark_wpk,
                                  mark_status, mark_ctr, mark_tiles, mark_lmask);
  SLIDE_LAUNCH_CHECK();
}

// Sharded step: keep only the ids this rank owns (id % G == g), in order,
// in place; cnt_all keeps the global active-set size for the statistics.
constexpr int kOwnThreads = 1024;
constexpr int kOwnPer = 64;  // cap_max <= 65536

__global__ void __launch_bounds__(kOwnThreads) own_filter_kernel(int32_t* __restrict__ act, int64_t cap_max,
                                                                 int g, int G, int32_t* __restrict__ cnt,
                                                                 int32_t* __restrict__ cnt_all) {
  using Scan = cub::BlockScan<int, kOwnThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int i = blockIdx.x;
  const int n = cnt[i];
  int32_t* a = act + (int64_t)i * cap_max;
  const int ch = (n + kOwnThreads - 1) / kOwnThreads;
  const int k0 = min((int)threadIdx.x * ch, n), k1 = min(k0 + ch, n);
  int32_t mine[kOwnPer];
  int m = 0;
  for (int k = k0; k < k1; ++k) {
    const int32_t v = a[k];
    if ((int)((uint32_t)(v & 0x7fffffff) % (uint32_t)G) == g) mine[m++] = v;
  }
  int ofs, total;
  Scan(tmp).ExclusiveSum(m, ofs, total);  // block-wide barrier: every read is done
  for (int q = 0; q < m; ++q) a[ofs + q] = mine[q];
  if (threadIdx.x == 0) {
    cnt_all[i] = n;
    cnt[i] = total;
  }
}

__global__ void counts_to_f64_kernel(int b, const int32_t* __restrict__ cnt, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < b) out[i] = (double)cnt[i];
}

void launch_counts_to_f64(int b, const int32_t* cnt, double* out, cudaStream_t s) {
  if (b <= 0) return;
  counts_to_f64_kernel<<<(b + 255) / 256, 256, 0, s>>>(b, cnt, out);
  SLIDE_LAUNCH_CHECK();
}

void launch_own_filter(int b, int32_t* act, int64_t cap_max, int g, int G, int32_t* cnt, int32_t* cnt_all,
                       cudaStream_t s) {
  SLIDE_CHECK(cap_max <= (int64_t)kOwnThreads * kOwnPer, kNotSupported, "active sets above 65536 ids per sample");
  own_filter_kernel<<<b, kOwnThreads, 0, s>>>(act, cap_max, g, G, cnt, cnt_all);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide

namespace slide {

// ----------------------------------------------------------- ranked top-k
// Sampled inference ranking (network.py:383-391): per slot, the active ids
// (ascending) ordered by descending probability, ties to the earlier (lower)
// id -- np.argsort(-p, kind="stable") -- truncated to k.  One CTA per slot,
// k rounds of a block argmax over (p, -position).
constexpr int kTopThreads = 256;

__global__ void __launch_bounds__(kTopThreads) topk_kernel(const int32_t* __restrict__ offs,
                                                          const int32_t* __restrict__ rows, int shard_count,
                                                          int shard_rank, const float* __restrict__ prob, int k,
                                                          int32_t* __restrict__ out, int32_t* __restrict__ cnt_out) {
  using Red = cub::BlockReduce<unsigned long long, kTopThreads>;
  __shared__ typename Red::TempStorage tmp;
  __shared__ unsigned long long s_best;
  const int i = blockIdx.x;
  const int o = offs[i], n = offs[i + 1] - o;
  const int kk = min(k, n);
  int prev = -1;  // position taken in the previous round
  float prev_p = 0.f;
  for (int r = 0; r < kk; ++r) {
    // key: p (non-negative, so its bits order like the float) high, then
    // the complement of the position (earlier wins ties); positions already
    // taken are excluded by (p, position) <= (prev_p, prev) ordering
    unsigned long long best = 0ull;
    for (int q = threadIdx.x; q < n; q += kTopThreads) {
      const float p = prob[o + q];
      const bool after = r == 0 || p < prev_p || (p == prev_p && q > prev);
      if (!after) continue;
      const unsigned long long key = ((unsigned long long)__float_as_uint(p) << 32) | (uint32_t)(0x7fffffff - q);
      best = key > best ? key : best;
    }
    best = Red(tmp).Reduce(best, cub::Max());
    if (threadIdx.x == 0) s_best = best;
    __syncthreads();
    const unsigned long long b = s_best;
    prev = 0x7fffffff - (int)(uint32_t)b;
    prev_p = __uint_as_float((uint32_t)(b >> 32));
    if (threadIdx.x == 0) {
      const int row = rows[o + prev];
      out[(int64_t)i * k + r] = row * shard_count + shard_rank;  // global id
    }
    __syncthreads();
  }
  for (int r = kk + threadIdx.x; r < k; r += kTopThreads) out[(int64_t)i * k + r] = -1;
  if (threadIdx.x == 0) cnt_out[i] = kk;
}

void launch_topk(int b, const int32_t* offs, const int32_t* rows, int shard_count, int shard_rank, const float* prob,
                 int k, int32_t* out, int32_t* cnt, cudaStream_t s) {
  if (b <= 0 || k <= 0) return;
  topk_kernel<<<b, kTopThreads, 0, s>>>(offs, rows, shard_count, shard_rank, prob, k, out, cnt);
  SLIDE_LAUNCH_CHECK();
}

// ------------------------------------------------- sampler on explicit lists
// samplers.sample (reference samplers.py:57-120) on caller-held candidate
// lists (RawCandidates): one CTA walks the L lists.  vanilla: the lists in
// `order` (the caller's rng.permutation(L)), whole lists, fresh ids appended
// in list order (a block scan keeps it), stop once >= beta distinct ids
// (checked after every list, empty ones included); freq counts the probed
// lists.  topk: freq over all lists, ids by (freq desc, id asc), first beta.
// hard_threshold: ids with freq >= min_freq ascending.  freq / seen are
// zeroed by the caller.
constexpr int kSampleThreads = 1024;

__global__ void __launch_bounds__(kSampleThreads) sample_lists_kernel(
    const int32_t* __restrict__ ptr, const int32_t* __restrict__ ids, int n_tables, int width, int strategy,
    int beta, int min_freq, const int32_t* __restrict__ order, int32_t* __restrict__ freq,
    uint32_t* __restrict__ seen, int32_t* __restrict__ out, int32_t* __restrict__ result) {
  using Scan = cub::BlockScan<int, kSampleThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_n;
  const int tid = threadIdx.x;
  if (tid == 0) s_n = 0;
  __syncthreads();
  if (strategy == 0) {
    int probed = 0;
    for (int k = 0; k < n_tables; ++k) {
      const int t = order[k];
      ++probed;
      const int a = ptr[t], e = ptr[t + 1];
      for (int q0 = a; q0 < e; q0 += kSampleThreads) {
        const int q = q0 + tid;
        int fresh = 0, id = 0;
        if (q < e) {
          id = ids[q];
          atomicAdd(&freq[id], 1);
          const uint32_t bit = 1u << (id & 31);
          fresh = (atomicOr(&seen[id >> 5], bit) & bit) == 0;
        }
        int pos, total;
        Scan(tmp).ExclusiveSum(fresh, pos, total);
        if (fresh) out[s_n + pos] = id;
        __syncthreads();
        if (tid == 0) s_n += total;
        __syncthreads();
      }
      if (s_n >= beta) break;
    }
    if (tid == 0) {
      result[0] = s_n;
      result[1] = probed;
    }
    return;
  }
  for (int t = 0; t < n_tables; ++t)
    for (int q = ptr[t] + tid; q < ptr[t + 1]; q += kSampleThreads) atomicAdd(&freq[ids[q]], 1);
  __syncthreads();
  // ordered compaction of the ids whose freq satisfies `pred`, ascending
  auto compact = [&](int lo, int hi, int limit) {
    for (int c0 = 0; c0 < width; c0 += kSampleThreads) {
      const int c = c0 + tid;
      const int f = c < width ? freq[c] : 0;
      const int take = f >= lo && f <= hi;
      int pos, total;
      Scan(tmp).ExclusiveSum(take, pos, total);
      if (take && s_n + pos < limit) out[s_n + pos] = c;
      __syncthreads();
      if (tid == 0) s_n = min(limit, s_n + total);
      __syncthreads();
      if (s_n >= limit) break;
    }
  };
  if (strategy == 2) {
    compact(min_freq, n_tables, width);
  } else {
    for (int f = n_tables; f >= 1 && s_n < beta; --f) compact(f, f, beta);
  }
  if (tid == 0) {
    result[0] = s_n;
    result[1] = n_tables;
  }
}

void launch_sample_lists(const int32_t* ptr, const int32_t* ids, int n_tables, int width, int strategy, int beta,
                         int min_freq, const int32_t* order, int32_t* freq, uint32_t* seen, int32_t* out,
                         int32_t* result, cudaStream_t s) {
  sample_lists_kernel<<<1, kSampleThreads, 0, s>>>(ptr, ids, n_tables, width, strategy, beta, min_freq, order, freq,
                                                   seen, out, result);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide
