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
//   2. rank   : popc prefix of the bitmap -> unique keys ascending, key->rank
//   3. mask   : per unique key a B-bit slot mask
//   4. count  : segment sizes (popc of the mask) -> exclusive scan
//   5. place  : item goes to seg_off[u] + popc(mask bits below its slot)
//
// All launches are sized by static maxima with device-side bounds.
#include "internal.cuh"
#include "kernels.cuh"
#include <cub/cub.cuh>
#include <algorithm>

namespace slide {

__device__ __forceinline__ int64_t dev_count(const int32_t* n_dev, int64_t n_host) {
  return n_dev ? (int64_t)*n_dev : n_host;
}

__global__ void g_mark_kernel(const int32_t* __restrict__ keys, const int32_t* n_dev, int64_t n_host,
                              uint32_t* __restrict__ bits) {
  const int64_t n = dev_count(n_dev, n_host);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = (uint32_t)keys[q];
    atomicOr(&bits[k >> 5], 1u << (k & 31));
  }
}

__global__ void g_popc_kernel(const uint32_t* __restrict__ bits, int64_t nwords, int32_t* __restrict__ wcnt) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x)
    wcnt[w] = __popc(bits[w]);
}

__global__ void g_rank_kernel(const uint32_t* __restrict__ bits, int64_t nwords, const int32_t* __restrict__ woff,
                              int32_t* __restrict__ uniq, int32_t* __restrict__ key_rank, int32_t* __restrict__ n_uniq) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = bits[w];
    int r = woff[w];
    while (b) {
      const int pos = __ffs(b) - 1;
      b &= b - 1;
      const int key = (int)(w * 32 + pos);
      uniq[r] = key;
      key_rank[key] = r;
      ++r;
    }
    if (w == nwords - 1) *n_uniq = r;
  }
}

__global__ void g_mask_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ slots, const int32_t* n_dev,
                              int64_t n_host, const int32_t* __restrict__ key_rank, int words_per_key,
                              uint32_t* __restrict__ mask) {
  const int64_t n = dev_count(n_dev, n_host);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int u = key_rank[keys[q]];
    const int s = slots[q];
    atomicOr(&mask[(int64_t)u * words_per_key + (s >> 5)], 1u << (s & 31));
  }
}

__global__ void g_count_kernel(const uint32_t* __restrict__ mask, int words_per_key, const int32_t* __restrict__ n_uniq,
                               int64_t u_max, int32_t* __restrict__ cnt) {
  const int64_t nu = *n_uniq;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < u_max; u += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    if (u < nu)
      for (int w = 0; w < words_per_key; ++w) c += __popc(mask[u * words_per_key + w]);
    cnt[u] = c;
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

__global__ void g_clear_kernel(uint32_t* __restrict__ mask, int words_per_key, const int32_t* __restrict__ n_uniq) {
  const int64_t n = (int64_t)*n_uniq * words_per_key;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    mask[q] = 0u;
}

static int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), kSms * 8)); }

void GroupBy::prepare(int64_t key_space, int64_t slots, int64_t items_max) {
  K = key_space;
  nwords = ceil_div(key_space, 32);
  wpk = (int)ceil_div(slots, 32);
  u_max = std::min<int64_t>(key_space, std::max<int64_t>(items_max, 1));
  if (bits_words < nwords) {
    uint32_t* b = bits.ensure<uint32_t>(nwords);
    SLIDE_CUDA(cudaMemset(b, 0, nwords * 4));
    bits_words = nwords;
  }
  const int64_t need_mask = u_max * wpk;
  if (mask_words < need_mask) {
    uint32_t* m = mask.ensure<uint32_t>(need_mask);
    SLIDE_CUDA(cudaMemset(m, 0, need_mask * 4));
    mask_words = need_mask;
  }
  key_rank.ensure<int32_t>(key_space);
  woff.ensure<int32_t>(nwords + 1);
  uniq.ensure<int32_t>(u_max);
  seg_cnt.ensure<int32_t>(u_max + 1);
  seg_off.ensure<int32_t>(u_max + 1);
  n_uniq.ensure<int32_t>(1);
  order.ensure<int32_t>(std::max<int64_t>(items_max, 1));
  size_t t1 = 0, t2 = 0;
  SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, woff.as<int32_t>(), woff.as<int32_t>(), (int)nwords + 1));
  SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, seg_cnt.as<int32_t>(), seg_off.as<int32_t>(), (int)u_max + 1));
  temp_bytes = std::max(t1, t2);
  temp.ensure<uint8_t>(temp_bytes);
}

void GroupBy::run(const int32_t* keys, const int32_t* slots, const int32_t* n_dev, int64_t n_host, int64_t n_max,
                  cudaStream_t s) {
  uint32_t* b = bits.as<uint32_t>();
  int32_t* wo = woff.as<int32_t>();
  g_mark_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, n_dev, n_host, b);
  SLIDE_LAUNCH_CHECK();
  g_popc_kernel<<<grid_of(nwords), 256, 0, s>>>(b, nwords, wo);
  SLIDE_LAUNCH_CHECK();
  // a trailing zero makes the exclusive scan's last entry the total
  SLIDE_CUDA(cudaMemsetAsync(wo + nwords, 0, 4, s));
  SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, temp_bytes, wo, wo, (int)nwords + 1, s));
  g_rank_kernel<<<grid_of(nwords), 256, 0, s>>>(b, nwords, wo, uniq.as<int32_t>(), key_rank.as<int32_t>(),
                                                 n_uniq.as<int32_t>());
  SLIDE_LAUNCH_CHECK();
  g_mask_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, slots, n_dev, n_host, key_rank.as<int32_t>(), wpk,
                                                mask.as<uint32_t>());
  SLIDE_LAUNCH_CHECK();
  g_count_kernel<<<grid_of(u_max + 1), 256, 0, s>>>(mask.as<uint32_t>(), wpk, n_uniq.as<int32_t>(), u_max + 1,
                                                     seg_cnt.as<int32_t>());
  SLIDE_LAUNCH_CHECK();
  SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, temp_bytes, seg_cnt.as<int32_t>(), seg_off.as<int32_t>(),
                                           (int)u_max + 1, s));
  g_place_kernel<<<grid_of(n_max), 256, 0, s>>>(keys, slots, n_dev, n_host, key_rank.as<int32_t>(), wpk,
                                                 mask.as<uint32_t>(), seg_off.as<int32_t>(), order.as<int32_t>());
  SLIDE_LAUNCH_CHECK();
}

void GroupBy::clear(cudaStream_t s) {
  // bitmap: clear all words (static size); masks: only the rows used
  SLIDE_CUDA(cudaMemsetAsync(bits.p, 0, nwords * 4, s));
  g_clear_kernel<<<grid_of(u_max * wpk), 256, 0, s>>>(mask.as<uint32_t>(), wpk, n_uniq.as<int32_t>());
  SLIDE_LAUNCH_CHECK();
}

void GroupBy::release() {
  for (DBuf* b : {&bits, &key_rank, &woff, &uniq, &seg_cnt, &seg_off, &n_uniq, &mask, &order, &temp}) b->release();
  bits_words = mask_words = 0;
}

}  // namespace slide
