// Stable group-by of (key, slot) items without a sort and without host
// round trips (every count stays on the device).
//
// Items are (key in [0, K), slot in [0, B)), each pair unique: the active
// (output row, sample) pairs of a step (W2 Adam) or the (feature, sample)
// input nonzeros (W1 Adam).  The Adam kernels need, per distinct key in
// ascending order, its items in slot order -- the order the reference
// applies per-sample updates (network.py:351-361).
//
//   1. mark   : bit `key` of a K-bit bitmap
//   2. rank   : popc prefix of the bitmap (single-pass scan) -> unique keys
//               ascending, key->rank
//   3. mask   : per unique key a B-bit slot mask
//   4. seg    : segment sizes (popc of the mask) -> offsets (single-pass scan)
//   5. place  : item goes to seg_off[u] + popc(mask bits below its slot)
//
// Five launches, sized by static maxima with device-side bounds; nothing to
// clear afterwards.
#include "internal.cuh"
#include "kernels.cuh"
#include <cub/cub.cuh>
#include <algorithm>

namespace slide {

__device__ __forceinline__ int64_t dev_count(const int32_t* n_dev, int64_t n_host) {
  return n_dev ? (int64_t)*n_dev : n_host;
}

// ---- single-pass tile scan (decoupled look-back).  Tiles are taken in
// order from a device counter, so a tile only ever waits on tiles already
// running.  status[t] = flag << 32 | value (flag 1: tile aggregate, 2:
// inclusive prefix); the kernel before each scan zeroes status and counter.
constexpr int kGT = 256;  // threads (= items) per tile

// The status word carries its value itself (flag and prefix in one aligned
// 64-bit word), so relaxed gpu-scope accesses suffice: no other data is
// published through it.  (ld.acquire compiles to an L1 invalidation per
// load -- CCTL.IVALL -- which dominated the scan's stall samples.)
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// warp 0: publish this tile's aggregate and resolve its exclusive prefix,
// reading 32 predecessors per round
__device__ __forceinline__ int tile_lookback(int tile, int agg, unsigned long long* status) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_status(status, (2ull << 32) | (uint32_t)agg);
    return 0;
  }
  if (lane == 0) st_status(status + tile, (1ull << 32) | (uint32_t)agg);
  int acc = 0;
  for (int top = tile - 1;;) {
    const int idx = top - lane;
    const unsigned long long v = idx >= 0 ? ld_status(status + idx) : (2ull << 32);
    const uint32_t flag = (uint32_t)(v >> 32);
    const unsigned inc = __ballot_sync(0xffffffffu, flag == 2), none = __ballot_sync(0xffffffffu, flag == 0);
    const unsigned need = inc ? (inc & (0u - inc)) * 2u - 1u : 0xffffffffu;  // lanes up to the closest prefix
    if (none & need) continue;  // a predecessor has not published yet
    int x = (need >> lane) & 1u ? (int)(uint32_t)v : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    acc += x;
    if (inc) break;
    top -= 32;
  }
  if (lane == 0) st_status(status + tile, (2ull << 32) | (uint32_t)(acc + agg));
  return acc;
}

struct TileCtl {
  unsigned long long* status;
  int32_t* ctr;
};

__device__ __forceinline__ void tile_reset(TileCtl t, int64_t n_tiles) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_tiles; q += (int64_t)gridDim.x * blockDim.x)
    t.status[q] = 0ull;
  if (blockIdx.x == 0 && threadIdx.x == 0) *t.ctr = 0;
}

__global__ void g_mark_kernel(const int32_t* __restrict__ keys, const int32_t* n_dev, int64_t n_host,
                              uint32_t* __restrict__ bits, TileCtl next, int64_t next_tiles) {
  tile_reset(next, next_tiles);
  const int64_t n = dev_count(n_dev, n_host);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = (uint32_t)keys[q];
    atomicOr(&bits[k >> 5], 1u << (k & 31));
  }
}

using GScan = cub::BlockScan<int, kGT>;

// popc prefix of the key bitmap -> unique keys ascending + key -> rank; the
// bitmap words are zeroed as they are consumed and each assigned rank's mask
// row is zeroed for the mask pass (no separate clear).
__global__ void __launch_bounds__(kGT) g_scan_rank_kernel(uint32_t* __restrict__ bits, int64_t nwords,
                                                          uint32_t* __restrict__ mask, int wpk,
                                                          int32_t* __restrict__ uniq, int32_t* __restrict__ key_rank,
                                                          int32_t* __restrict__ n_uniq, TileCtl tc) {
  __shared__ typename GScan::TempStorage tmp;
  __shared__ int s_tile, s_base;
  if (threadIdx.x == 0) s_tile = atomicAdd(tc.ctr, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t w = (int64_t)tile * kGT + threadIdx.x;  // bitmap padded to whole tiles
  uint32_t x = bits[w];
  const int c = __popc(x);
  int off, agg;
  GScan(tmp).ExclusiveSum(c, off, agg);
  if (threadIdx.x < 32) {
    const int base = tile_lookback(tile, agg, tc.status);
    if (threadIdx.x == 0) s_base = base;
  }
  __syncthreads();
  int r = s_base + off;
  if (x) bits[w] = 0u;
  while (x) {
    const int pos = __ffs(x) - 1;
    x &= x - 1;
    const int key = (int)(w * 32 + pos);
    uniq[r] = key;
    key_rank[key] = r;
    for (int q = 0; q < wpk; ++q) mask[(int64_t)r * wpk + q] = 0u;
    ++r;
  }
  if (w == nwords - 1) *n_uniq = r;
}

__global__ void g_mask_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ slots, const int32_t* n_dev,
                              int64_t n_host, const int32_t* __restrict__ key_rank, int words_per_key,
                              uint32_t* __restrict__ mask, TileCtl next, int64_t next_tiles) {
  tile_reset(next, next_tiles);
  const int64_t n = dev_count(n_dev, n_host);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int u = key_rank[keys[q]];
    const int s = slots[q];
    atomicOr(&mask[(int64_t)u * words_per_key + (s >> 5)], 1u << (s & 31));
  }
}

// segment sizes (popc of each unique key's slot mask) -> exclusive offsets
__global__ void __launch_bounds__(kGT) g_seg_kernel(const uint32_t* __restrict__ mask, int wpk,
                                                    const int32_t* __restrict__ n_uniq, int32_t* __restrict__ seg_off,
                                                    int32_t* __restrict__ seg_cnt, TileCtl tc, LongList ll) {
  __shared__ typename GScan::TempStorage tmp;
  __shared__ int s_tile, s_base;
  const int64_t nu = *n_uniq;
  // only the first ceil(nu / kGT) CTAs take tiles (static grid for graphs)
  if ((int64_t)blockIdx.x * kGT >= nu) return;
  if (threadIdx.x == 0) s_tile = atomicAdd(tc.ctr, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t u = (int64_t)tile * kGT + threadIdx.x;
  int c = 0;
  if (u < nu)
    for (int q = 0; q < wpk; ++q) c += __popc(mask[u * wpk + q]);
  int off, agg;
  GScan(tmp).ExclusiveSum(c, off, agg);
  if (threadIdx.x < 32) {
    const int base = tile_lookback(tile, agg, tc.status);
    if (threadIdx.x == 0) s_base = base;
  }
  __syncthreads();
  if (u < nu) {
    seg_off[u] = s_base + off;
    seg_cnt[u] = c;
    if (ll.list && c > ll.min_len) ll.list[atomicAdd(ll.n, 1)] = (int32_t)u;
  }
}

__global__ void g_place_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ slots, const int32_t* n_dev,
                               int64_t n_host, const int32_t* __restrict__ key_rank, int words_per_key,
                               const uint32_t* __restrict__ mask, const int32_t* __restrict__ seg_off,
                               int32_t* __restrict__ order, int32_t* __restrict__ inv, int32_t* __restrict__ sslot) {
  const int64_t n = dev_count(n_dev, n_host);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int u = key_rank[keys[q]];
    const int s = slots[q];
    const uint32_t* m = mask + (int64_t)u * words_per_key;
    int r = 0;
    for (int w = 0; w < (s >> 5); ++w) r += __popc(m[w]);
    r += __popc(m[s >> 5] & ((1u << (s & 31)) - 1u));
    const int pos = seg_off[u] + r;
    order[pos] = (int32_t)q;
    if (inv) {
      inv[q] = pos;
      sslot[pos] = s;
    }
  }
}

// ---- dense-mask mode: one B-bit slot mask per key of the whole key space
// (used when K x B bits is small: W2 rows, W1 features at the BASELINE
// sizes).  mark + mask are one atomicOr pass, the unique-key ranks and the
// segment offsets come out of one two-value look-back scan over the keys
// (rank in the high half, pair offset in the low half of the status word),
// and the masks of the used keys are cleared after the consumers ran.
__global__ void gd_mask_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ slots, const int32_t* n_dev,
                               int64_t n_host, int wpk, uint32_t* __restrict__ mask, TileCtl next, int64_t next_tiles) {
  tile_reset(next, next_tiles);
  const int64_t n = dev_count(n_dev, n_host);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int s = slots[q];
    atomicOr(&mask[(int64_t)keys[q] * wpk + (s >> 5)], 1u << (s & 31));
  }
}

// warp 0 of a tile: publish (rank count, pair count) and resolve the
// exclusive prefix of both; values packed rank << 31 | pairs (each < 2^31)
__device__ __forceinline__ unsigned long long tile_lookback2(int tile, unsigned long long agg,
                                                             unsigned long long* status) {
  const int lane = threadIdx.x & 31;
  // flag in the top 2 bits would collide with the values: keep it in a
  // separate bit pattern -- status = value + 1 (aggregate) or value + 1 with
  // bit 63 set (inclusive); 0 = not yet published
  constexpr unsigned long long kInc = 1ull << 63;
  if (tile == 0) {
    if (lane == 0) st_status(status, kInc | (agg + 1));
    return 0;
  }
  if (lane == 0) st_status(status + tile, agg + 1);
  unsigned long long acc = 0;
  for (int top = tile - 1;;) {
    const int idx = top - lane;
    const unsigned long long v = idx >= 0 ? ld_status(status + idx) : (kInc | 1ull);
    const unsigned inc = __ballot_sync(0xffffffffu, (v & kInc) != 0), none = __ballot_sync(0xffffffffu, v == 0);
    const unsigned need = inc ? (inc & (0u - inc)) * 2u - 1u : 0xffffffffu;
    if (none & need) continue;
    unsigned long long x = (need >> lane) & 1u ? ((v & ~kInc) - 1) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    acc += x;
    if (inc) break;
    top -= 32;
  }
  if (lane == 0) st_status(status + tile, kInc | (acc + agg + 1));
  return acc;
}

// Block-wide look-back for the two-value scan: every thread of the tile
// reads one predecessor's status (kGT per round instead of 32), so a tile
// whose predecessors have only published aggregates resolves in one round
// trip instead of one per 32 tiles.  Called by all threads; returns the
// exclusive prefix.
__device__ __forceinline__ unsigned long long tile_lookback2_block(int tile, unsigned long long agg,
                                                                   unsigned long long* status) {
  using Red = cub::BlockReduce<unsigned long long, kGT>;
  __shared__ typename Red::TempStorage red;
  __shared__ int s_lim;
  __shared__ unsigned long long s_acc;
  constexpr unsigned long long kInc = 1ull << 63;
  if (tile == 0) {
    if (threadIdx.x == 0) st_status(status, kInc | (agg + 1));
    return 0;
  }
  if (threadIdx.x == 0) {
    st_status(status + tile, agg + 1);
    s_acc = 0;
  }
  unsigned long long acc = 0;
  for (int top = tile - 1;; top -= kGT) {
    if (threadIdx.x == 0) s_lim = top - kGT;  // no inclusive prefix in this window yet
    __syncthreads();
    const int idx = top - (int)threadIdx.x;
    unsigned long long v = 0;
    if (idx >= 0) {
      do v = ld_status(status + idx);
      while (v == 0);
      if (v & kInc) atomicMax(&s_lim, idx);
    } else {
      atomicMax(&s_lim, -1);  // before tile 0: an inclusive prefix of 0
    }
    __syncthreads();
    const int lim = s_lim;
    const unsigned long long x = idx >= 0 && idx >= lim ? (v & ~kInc) - 1 : 0ull;
    const unsigned long long sum = Red(red).Sum(x);
    if (threadIdx.x == 0) s_acc += sum;
    __syncthreads();
    if (lim > top - kGT) break;
  }
  acc = s_acc;
  if (threadIdx.x == 0) st_status(status + tile, kInc | (acc + agg + 1));
  return acc;
}

// kKPT keys per thread: every mask word of the thread's keys is loaded at
// once (the scan is latency-bound), a tile covers kGT * kKPT keys
constexpr int kKPT = 4;

template <int MAXW>
__device__ __forceinline__ void load_masks(const uint32_t* __restrict__ mask, int64_t k0, int64_t K, int wpk,
                                           uint32_t (&m)[kKPT][MAXW == 0 ? 1 : MAXW], int (&c)[kKPT]) {
  if constexpr (MAXW == 4) {
    if (wpk == 4) {  // one 16-byte row per key
#pragma unroll
      for (int j = 0; j < kKPT; ++j) {
        const uint4 v = k0 + j < K ? __ldcg(reinterpret_cast<const uint4*>(mask) + k0 + j) : make_uint4(0, 0, 0, 0);
        m[j][0] = v.x, m[j][1] = v.y, m[j][2] = v.z, m[j][3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < kKPT; ++j) c[j] = __popc(m[j][0]) + __popc(m[j][1]) + __popc(m[j][2]) + __popc(m[j][3]);
      return;
    }
  }
  if constexpr (MAXW > 0) {
#pragma unroll
    for (int j = 0; j < kKPT; ++j)
#pragma unroll
      for (int w = 0; w < MAXW; ++w) m[j][w] = k0 + j < K && w < wpk ? __ldcg(mask + (k0 + j) * wpk + w) : 0u;
#pragma unroll
    for (int j = 0; j < kKPT; ++j) {
      c[j] = 0;
#pragma unroll
      for (int w = 0; w < MAXW; ++w) c[j] += __popc(m[j][w]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kKPT; ++j) {
      c[j] = 0;
      if (k0 + j < K)
        for (int w = 0; w < wpk; ++w) c[j] += __popc(__ldcg(mask + (k0 + j) * wpk + w));
    }
  }
}

template <int MAXW>
__global__ void __launch_bounds__(kGT) gd_scan_kernel(int64_t K, int wpk, const uint32_t* __restrict__ mask,
                                                      int32_t* __restrict__ uniq, int32_t* __restrict__ key_rank,
                                                      int32_t* __restrict__ seg_off, int32_t* __restrict__ seg_cnt,
                                                      int32_t* __restrict__ n_uniq, TileCtl tc, LongList ll) {
  using Scan2 = cub::BlockScan<unsigned long long, kGT>;
  __shared__ typename Scan2::TempStorage tmp;
  __shared__ int s_tile;
  __shared__ unsigned long long s_base;
  if (threadIdx.x == 0) s_tile = atomicAdd(tc.ctr, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t k0 = ((int64_t)tile * kGT + threadIdx.x) * kKPT;
  uint32_t m[kKPT][MAXW == 0 ? 1 : MAXW];
  int c[kKPT];
  load_masks<MAXW>(mask, k0, K, wpk, m, c);
  unsigned long long nk = 0, np = 0;
#pragma unroll
  for (int j = 0; j < kKPT; ++j) nk += c[j] ? 1 : 0, np += (unsigned)c[j];
  const unsigned long long mine = (nk << 31) | np;
  unsigned long long off, agg;
  Scan2(tmp).ExclusiveSum(mine, off, agg);
  const unsigned long long pre = tile_lookback2_block(tile, agg, tc.status) + off;
  int r = (int)(pre >> 31), po = (int)(pre & 0x7fffffffull);
#pragma unroll
  for (int j = 0; j < kKPT; ++j) {
    if (c[j]) {
      const int64_t key = k0 + j;
      uniq[r] = (int32_t)key;
      key_rank[key] = po;  // dense mode: the key's segment offset (all the placement needs)
      seg_off[r] = po;
      seg_cnt[r] = c[j];
      if (ll.list && c[j] > ll.min_len) ll.list[atomicAdd(ll.n, 1)] = r;
      ++r;
      po += c[j];
    }
  }
  if (k0 <= K - 1 && K - 1 < k0 + kKPT) *n_uniq = r;
}

// kPPT pairs per thread, every load of the group issued before any store
constexpr int kPPT = 4;

__global__ void __launch_bounds__(256) gd_place_kernel(const int32_t* __restrict__ keys,
                                                       const int32_t* __restrict__ slots, const int32_t* n_dev,
                                                       int64_t n_host, const int32_t* __restrict__ key_rank, int wpk,
                                                       const uint32_t* __restrict__ mask,
                                                       const int32_t* __restrict__ seg_off,
                                                       int32_t* __restrict__ order, int32_t* __restrict__ inv,
                                                       int32_t* __restrict__ sslot) {
  const int64_t n = dev_count(n_dev, n_host);
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < n; q0 += T * kPPT) {
    int key[kPPT], s[kPPT];
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
      const int64_t q = q0 + j * T;
      key[j] = q < n ? __ldcs(keys + q) : -1;
      s[j] = q < n ? __ldcs(slots + q) : 0;
    }
    int base[kPPT], r[kPPT];
    if (wpk == 4) {  // the whole 16-byte mask row
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        uint4 v = make_uint4(0, 0, 0, 0);
        base[j] = 0;
        if (key[j] >= 0) {
          v = __ldcg(reinterpret_cast<const uint4*>(mask) + key[j]);
          base[j] = __ldcg(key_rank + key[j]);
        }
        const int w = s[j] >> 5;
        const uint32_t lo = (1u << (s[j] & 31)) - 1u;
        r[j] = (w > 0 ? __popc(v.x) : __popc(v.x & lo)) + (w > 1 ? __popc(v.y) : w == 1 ? __popc(v.y & lo) : 0) +
               (w > 2 ? __popc(v.z) : w == 2 ? __popc(v.z & lo) : 0) + (w == 3 ? __popc(v.w & lo) : 0);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPPT; ++j) {
        base[j] = key[j] >= 0 ? __ldcg(key_rank + key[j]) : 0;
        r[j] = 0;
        if (key[j] >= 0) {
          const uint32_t* mk = mask + (int64_t)key[j] * wpk;
          for (int w = 0; w < (s[j] >> 5); ++w) r[j] += __popc(__ldcg(mk + w));
          r[j] += __popc(__ldcg(mk + (s[j] >> 5)) & ((1u << (s[j] & 31)) - 1u));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kPPT; ++j) {
      if (key[j] < 0) continue;
      const int64_t q = q0 + j * T;
      const int pos = base[j] + r[j];  // (dense mode: key_rank holds the segment offset)
      order[pos] = (int32_t)q;
      if (inv) {
        inv[q] = pos;
        sslot[pos] = s[j];
      }
    }
  }
}

__global__ void gd_clear_kernel(const int32_t* __restrict__ uniq, const int32_t* __restrict__ n_uniq, int wpk,
                                uint32_t* __restrict__ mask, uint32_t* __restrict__ lmask) {
  const int64_t n = (int64_t)*n_uniq * wpk;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)uniq[q / wpk] * wpk + q % wpk;
    mask[o] = 0u;
    if (lmask) lmask[o] = 0u;
  }
}

static int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), kSms * 8)); }

void GroupBy::prepare(int64_t key_space, int64_t slots, int64_t items_max) {
  K = key_space;
  nwords = ceil_div(key_space, 32);
  wpk = (int)ceil_div(slots, 32);
  u_max = std::min<int64_t>(key_space, std::max<int64_t>(items_max, 1));
  // dense-mask mode when the whole key space's masks are small (<= 32 MB)
  // and the scan over the key space is not much longer than the item list
  const int64_t items_est = items_hint > 0 ? std::min(items_hint, items_max) : items_max;
  dense = key_space * wpk * 4 <= ((int64_t)32 << 20) && key_space <= 4 * std::max<int64_t>(items_est, 1);
  key_rank.ensure<int32_t>(key_space);
  uniq.ensure<int32_t>(u_max);
  seg_cnt.ensure<int32_t>(u_max);
  seg_off.ensure<int32_t>(u_max);
  n_uniq.ensure<int32_t>(1);
  order.ensure<int32_t>(std::max<int64_t>(items_max, 1));
  if (want_inv) {
    inv.ensure<int32_t>(std::max<int64_t>(items_max, 1));
    sslot.ensure<int32_t>(std::max<int64_t>(items_max, 1));
  }
  ctrs.ensure<int32_t>(2);
  if (dense) {
    const int64_t need = key_space * wpk;
    if (want_lmask && lmask_words < need) {
      SLIDE_CUDA(cudaMemset(lmask.ensure<uint32_t>(need), 0, need * 4));  // kept zero between runs by clear()
      lmask_words = need;
    }
    if (mask_words < need || !mask_dense) {
      uint32_t* m = mask.ensure<uint32_t>(need);
      SLIDE_CUDA(cudaMemset(m, 0, need * 4));  // kept zero between runs by clear()
      mask_words = need;
      mask_dense = true;
    }
    tiles_bits = ceil_div(key_space, (int64_t)kGT * kKPT);
    tiles_seg = 0;
    status.ensure<unsigned long long>(tiles_bits);
    return;
  }
  mask_dense = false;
  const int64_t words_pad = ceil_div(nwords, kGT) * kGT;  // whole scan tiles
  if (bits_words < words_pad) {
    uint32_t* b = bits.ensure<uint32_t>(words_pad);
    SLIDE_CUDA(cudaMemset(b, 0, words_pad * 4));
    bits_words = words_pad;
  }
  const int64_t need_mask = u_max * wpk;
  if (mask_words < need_mask) mask.ensure<uint32_t>(need_mask), mask_words = need_mask;  // rows zeroed on use
  tiles_bits = words_pad / kGT;
  tiles_seg = ceil_div(u_max, kGT);
  status.ensure<unsigned long long>(tiles_bits + tiles_seg);
}

void GroupBy::run(const int32_t* keys, const int32_t* slots, const int32_t* n_dev, int64_t n_host, int64_t n_max,
                  cudaStream_t s) {
  // optional list of the segments longer than long_min (in no fixed order)
  LongList long_out{nullptr, nullptr, long_min};
  if (long_min >= 0) {
    long_out.list = long_list.ensure<int32_t>(std::max<int64_t>(u_max, 1));
    long_out.n = n_long.ensure<int32_t>(1);
    SLIDE_CUDA(cudaMemsetAsync(long_out.n, 0, 4, s));
  }
  if (dense) {
    const TileCtl t{status.as<unsigned long long>(), ctrs.as<int32_t>()};
    const int grid_place = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_max, 256 * kPPT), kSms * 8));
    if (!premarked) {
      gd_mask_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, slots, n_dev, n_host, wpk, mask.as<uint32_t>(), t,
                                                    tiles_bits);
      SLIDE_LAUNCH_CHECK();
    }
#define SLIDE_GDS(W)                                                                                   \
  gd_scan_kernel<W><<<(int)tiles_bits, kGT, 0, s>>>(K, wpk, mask.as<uint32_t>(), uniq.as<int32_t>(),           \
                                                    key_rank.as<int32_t>(), seg_off.as<int32_t>(),             \
                                                    seg_cnt.as<int32_t>(), n_uniq.as<int32_t>(), t, long_out)
    if (wpk <= 1) SLIDE_GDS(1);
    else if (wpk <= 2) SLIDE_GDS(2);
    else if (wpk <= 4) SLIDE_GDS(4);
    else if (wpk <= 8) SLIDE_GDS(8);
    else SLIDE_GDS(0);
#undef SLIDE_GDS
    SLIDE_LAUNCH_CHECK();
    if (place) {
      gd_place_kernel<<<grid_place, 256, 0, s>>>(keys, slots, n_dev, n_host, key_rank.as<int32_t>(), wpk,
                                                     mask.as<uint32_t>(), seg_off.as<int32_t>(), order.as<int32_t>(),
                                                     want_inv ? inv.as<int32_t>() : nullptr, sslot.as<int32_t>());
      SLIDE_LAUNCH_CHECK();
    }
    return;
  }
  uint32_t* b = bits.as<uint32_t>();
  const TileCtl t1{status.as<unsigned long long>(), ctrs.as<int32_t>()};
  const TileCtl t2{status.as<unsigned long long>() + tiles_bits, ctrs.as<int32_t>() + 1};
  g_mark_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, n_dev, n_host, b, t1, tiles_bits);
  SLIDE_LAUNCH_CHECK();
  g_scan_rank_kernel<<<(int)tiles_bits, kGT, 0, s>>>(b, nwords, mask.as<uint32_t>(), wpk, uniq.as<int32_t>(),
                                                     key_rank.as<int32_t>(), n_uniq.as<int32_t>(), t1);
  SLIDE_LAUNCH_CHECK();
  g_mask_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, slots, n_dev, n_host, key_rank.as<int32_t>(), wpk,
                                                mask.as<uint32_t>(), t2, tiles_seg);
  SLIDE_LAUNCH_CHECK();
  g_seg_kernel<<<(int)tiles_seg, kGT, 0, s>>>(mask.as<uint32_t>(), wpk, n_uniq.as<int32_t>(), seg_off.as<int32_t>(),
                                              seg_cnt.as<int32_t>(), t2, long_out);
  SLIDE_LAUNCH_CHECK();
  g_place_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, slots, n_dev, n_host, key_rank.as<int32_t>(), wpk,
                                                 mask.as<uint32_t>(), seg_off.as<int32_t>(), order.as<int32_t>(),
                                                 want_inv ? inv.as<int32_t>() : nullptr, sslot.as<int32_t>());
  SLIDE_LAUNCH_CHECK();
}

// Bitmap mode: every buffer is reset by the next run itself (bitmap words as
// they are scanned, mask rows as ranks are assigned, scan status by the
// kernel before).  Dense mode: the used keys' masks are zeroed here, after
// the last consumer.
void GroupBy::clear(cudaStream_t s) {
  if (!dense) return;
  gd_clear_kernel<<<grid_of(u_max * wpk), 256, 0, s>>>(uniq.as<int32_t>(), n_uniq.as<int32_t>(), wpk,
                                                       mask.as<uint32_t>(), lmask_words ? lmask.as<uint32_t>() : nullptr);
  SLIDE_LAUNCH_CHECK();
}

void GroupBy::release() {
  for (DBuf* b : {&bits, &key_rank, &uniq, &seg_cnt, &seg_off, &n_uniq, &mask, &order, &inv, &sslot, &status, &ctrs,
                  &long_list, &n_long})
    b->release();
  bits_words = mask_words = lmask_words = 0;
  lmask.release();
  mask_dense = false;
}

}  // namespace slide
