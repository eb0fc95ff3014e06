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

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// warp 0: publish this tile's aggregate and resolve its exclusive prefix,
// reading 32 predecessors per round
__device__ __forceinline__ int tile_lookback(int tile, int agg, unsigned long long* status) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_release(status, (2ull << 32) | (uint32_t)agg);
    return 0;
  }
  if (lane == 0) st_release(status + tile, (1ull << 32) | (uint32_t)agg);
  int acc = 0;
  for (int top = tile - 1;;) {
    const int idx = top - lane;
    const unsigned long long v = idx >= 0 ? ld_acquire(status + idx) : (2ull << 32);
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
  if (lane == 0) st_release(status + tile, (2ull << 32) | (uint32_t)(acc + agg));
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
                                                    int32_t* __restrict__ seg_cnt, TileCtl tc) {
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
  }
}

__global__ void g_place_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ slots, const int32_t* n_dev,
                               int64_t n_host, const int32_t* __restrict__ key_rank, int words_per_key,
                               const uint32_t* __restrict__ mask, const int32_t* __restrict__ seg_off,
                               int32_t* __restrict__ order) {
  const int64_t n = dev_count(n_dev, n_host);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int u = key_rank[keys[q]];
    const int s = slots[q];
    const uint32_t* m = mask + (int64_t)u * words_per_key;
    int r = 0;
    for (int w = 0; w < (s >> 5); ++w) r += __popc(m[w]);
    r += __popc(m[s >> 5] & ((1u << (s & 31)) - 1u));
    order[seg_off[u] + r] = (int32_t)q;
  }
}

static int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), kSms * 8)); }

void GroupBy::prepare(int64_t key_space, int64_t slots, int64_t items_max) {
  K = key_space;
  nwords = ceil_div(key_space, 32);
  wpk = (int)ceil_div(slots, 32);
  u_max = std::min<int64_t>(key_space, std::max<int64_t>(items_max, 1));
  const int64_t words_pad = ceil_div(nwords, kGT) * kGT;  // whole scan tiles
  if (bits_words < words_pad) {
    uint32_t* b = bits.ensure<uint32_t>(words_pad);
    SLIDE_CUDA(cudaMemset(b, 0, words_pad * 4));
    bits_words = words_pad;
  }
  const int64_t need_mask = u_max * wpk;
  if (mask_words < need_mask) mask.ensure<uint32_t>(need_mask), mask_words = need_mask;  // rows zeroed on use
  key_rank.ensure<int32_t>(key_space);
  uniq.ensure<int32_t>(u_max);
  seg_cnt.ensure<int32_t>(u_max);
  seg_off.ensure<int32_t>(u_max);
  n_uniq.ensure<int32_t>(1);
  order.ensure<int32_t>(std::max<int64_t>(items_max, 1));
  tiles_bits = words_pad / kGT;
  tiles_seg = ceil_div(u_max, kGT);
  status.ensure<unsigned long long>(tiles_bits + tiles_seg);
  ctrs.ensure<int32_t>(2);
}

void GroupBy::run(const int32_t* keys, const int32_t* slots, const int32_t* n_dev, int64_t n_host, int64_t n_max,
                  cudaStream_t s) {
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
                                              seg_cnt.as<int32_t>(), t2);
  SLIDE_LAUNCH_CHECK();
  g_place_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, slots, n_dev, n_host, key_rank.as<int32_t>(), wpk,
                                                 mask.as<uint32_t>(), seg_off.as<int32_t>(), order.as<int32_t>());
  SLIDE_LAUNCH_CHECK();
}

// Every buffer is reset by the next run itself (bitmap words as they are
// scanned, mask rows as ranks are assigned, scan status by the kernel before).
void GroupBy::clear(cudaStream_t) {}

void GroupBy::release() {
  for (DBuf* b : {&bits, &key_rank, &uniq, &seg_cnt, &seg_off, &n_uniq, &mask, &order, &status, &ctrs}) b->release();
  bits_words = mask_words = 0;
}

}  // namespace slide
