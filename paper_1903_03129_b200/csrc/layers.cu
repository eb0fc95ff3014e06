#include <cstdlib>
// Sparse forward / backward / Adam kernels (reference network.py:241-336,
// 428-451).  Row layout: every weight row (a W1^T feature row, a W2 output
// row) is hp floats, hp a multiple of 128, so one warp moves a row with one
// 128-bit load per lane per 128 columns (NV = hp / 128).
#include "internal.cuh"
#include "kernels.cuh"
#include <cub/cub.cuh>
#include <type_traits>

namespace slide {

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4_cg(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float& comp(float4& v, int q) { return reinterpret_cast<float*>(&v)[q]; }
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#define SLIDE_NV_DISPATCH(hp, KERNEL_CALL)                                                        \
  switch ((hp) / 128) {                                                                           \
    case 1: { constexpr int NV = 1; KERNEL_CALL; } break;                                         \
    case 2: { constexpr int NV = 2; KERNEL_CALL; } break;                                         \
    case 4: { constexpr int NV = 4; KERNEL_CALL; } break;                                         \
    case 8: { constexpr int NV = 8; KERNEL_CALL; } break;                                         \
    default: throw Error(kNotSupported, "padded hidden width must be 128, 256, 512 or 1024");     \
  }

// ------------------------------------------------------------ hidden forward
// z1 = sum_f x_f W1^T[f, :] + b1, h = max(z1, 0) (network.py:262-280).  One
// CTA of 32 warps per sample (a sample has ~75-300 nonzeros: enough rows in
// flight per SM), warp w owns every 32nd nonzero; partial sums are added in
// warp order (deterministic).
template <int NV>
struct FwdWarps {
  static constexpr int value = NV <= 2 ? 32 : 8;  // static smem: warps x hp floats <= 32 KB
};

// ------------------------------------------------------------ live columns
// The hidden units that are nonzero in at least one sample of the batch.  A
// unit c with h_i[c] = 0 for every i moves nothing downstream: its logit
// terms are exact zeros, its hidden-error entries are masked, its W1 / W2
// Adam coordinates stay frozen -- the reference itself only touches
// W[A, nz(h)] (network.py:266, 322-332).  live[0] = n live units,
// live[1..hp] = a permutation of the units: the live ones ascending, then the
// dead ones ascending.  Row kernels map lane l of 32-column group g to unit
// live[1 + 32 g + l] and walk only the ceil(n / 32) groups that hold live
// units; the tail lanes of the last group land on dead units (h = 0
// everywhere), so they need no predicate.  After the first step of the
// BASELINE workloads ~26 of 128 units stay live batch-wide.
// Whole CTA; hmask (b x hp/32 words, bit = h > 0) written by other CTAs.
__device__ void build_live_cols(int hp, int b, const uint32_t* hmask, int32_t* __restrict__ live) {
  __shared__ uint32_t words[32];
  const int mw = hp >> 5;
  for (int w = threadIdx.x; w < mw; w += blockDim.x) words[w] = 0u;
  __syncthreads();
  for (int q = threadIdx.x; q < b * mw; q += blockDim.x) {
    const uint32_t v = __ldcg(hmask + q);
    if (v) atomicOr(&words[q % mw], v);
  }
  __syncthreads();
  int n = 0;
  for (int w = 0; w < mw; ++w) n += __popc(words[w]);
  for (int c = threadIdx.x; c < hp; c += blockDim.x) {
    const int w = c >> 5;
    int before = 0;  // live units below c
    for (int k = 0; k < w; ++k) before += __popc(words[k]);
    before += __popc(words[w] & ((1u << (c & 31)) - 1u));
    const bool on = (words[w] >> (c & 31)) & 1u;
    live[1 + (on ? before : n + (c - before))] = c;
  }
  if (threadIdx.x == 0) live[0] = n;
}

__global__ void __launch_bounds__(1024) live_cols_from_h_kernel(int hp, int b, const float* __restrict__ h,
                                                                uint32_t* __restrict__ hmask, int32_t* __restrict__ live) {
  const int mw = hp >> 5;
  for (int q = threadIdx.x; q < b * hp; q += blockDim.x) {  // hp % 32 == 0: warps stay inside one word
    const unsigned bal = __ballot_sync(0xffffffffu, h[q] > 0.f);
    if ((threadIdx.x & 31) == 0) hmask[(q / hp) * mw + (q % hp) / 32] = bal;
  }
  __threadfence_block();
  __syncthreads();
  build_live_cols(hp, b, hmask, live);
}

void launch_live_cols_from_h(int hp, int b, const float* h, uint32_t* hmask, int32_t* live, cudaStream_t s) {
  if (b <= 0) return;
  live_cols_from_h_kernel<<<1, 1024, 0, s>>>(hp, b, h, hmask, live);
  SLIDE_LAUNCH_CHECK();
}

// QH: the sample's SimHash query keys are computed by the same CTA from its
// h row in shared memory (simhash_query_kernel's arithmetic: fp64 sums in
// the packed term order, bit = sum > 0) -- one launch and one dependent
// round trip fewer on the forward path.
template <int NV, bool QH = false, int kFwdWarps = FwdWarps<NV>::value>
__global__ void __launch_bounds__(kFwdWarps * 32) hidden_fwd_kernel(int hp, const int32_t* __restrict__ x_ptr,
                                                                    const int32_t* __restrict__ x_idx,
                                                                    const float* __restrict__ x_val,
                                                                    const float* __restrict__ w1t,
                                                                    const float* __restrict__ b1,
                                                                    float* __restrict__ h, uint32_t* __restrict__ hmask,
                                                                    int32_t* __restrict__ live,
                                                                    int32_t* __restrict__ ticket, QueryHash qh) {
  __shared__ float red[kFwdWarps][NV * 128];
  const int i = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = x_ptr[i], e = x_ptr[i + 1];
  float4 acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = a + warp;
  for (; k + kFwdWarps < e; k += 2 * kFwdWarps) {
    float4 r[2][NV];
    float v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int f = x_idx[k + kFwdWarps * u];
      v[u] = x_val[k + kFwdWarps * u];
      const float* row = w1t + (int64_t)f * hp + lane * 4;
#pragma unroll
      for (int q = 0; q < NV; ++q) r[u][q] = ld4(row + q * 128);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        acc[q].x = fmaf(v[u], r[u][q].x, acc[q].x);
        acc[q].y = fmaf(v[u], r[u][q].y, acc[q].y);
        acc[q].z = fmaf(v[u], r[u][q].z, acc[q].z);
        acc[q].w = fmaf(v[u], r[u][q].w, acc[q].w);
      }
  }
  for (; k < e; k += kFwdWarps) {
    const int f = x_idx[k];
    const float v = x_val[k];
    const float* row = w1t + (int64_t)f * hp + lane * 4;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      float4 r = ld4(row + q * 128);
      acc[q].x = fmaf(v, r.x, acc[q].x);
      acc[q].y = fmaf(v, r.y, acc[q].y);
      acc[q].z = fmaf(v, r.z, acc[q].z);
      acc[q].w = fmaf(v, r.w, acc[q].w);
    }
  }
#pragma unroll
  for (int q = 0; q < NV; ++q) *reinterpret_cast<float4*>(&red[warp][q * 128 + lane * 4]) = acc[q];
  __syncthreads();
  for (int c = threadIdx.x; c < hp; c += kFwdWarps * 32) {
    float s = red[0][c];
#pragma unroll 8
    for (int w = 1; w < kFwdWarps; ++w) s += red[w][c];
    s += b1[c];
    const float hv = s > 0.f ? s : 0.f;
    h[(int64_t)i * hp + c] = hv;
    if (QH) red[0][c] = hv;  // column c is read by this thread only
    // warps cover 32 consecutive units (hp % 32 == 0): one mask word each
    const unsigned bal = __ballot_sync(0xffffffffu, hv > 0.f);
    if (lane == 0) hmask[(int64_t)i * (hp >> 5) + (c >> 5)] = bal;
  }
  if constexpr (QH) {
    __shared__ uint8_t qbits[kQhMaxBits];
    __syncthreads();
    const int KL = qh.k * qh.l;
    const float* hs = &red[0][0];
    for (int p = threadIdx.x; p < KL; p += kFwdWarps * 32) {
      double acc = 0.0;
      // the terms come from L2: 8 loads in flight, summed in term order
      int j = 0;
      for (; j + 8 <= qh.c; j += 8) {
        uint16_t t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = __ldg(qh.packed_t + (j + u) * KL + p);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double v = (double)hs[t[u] & 0x7fff];
          acc += (t[u] >> 15) ? -v : v;
        }
      }
      for (; j < qh.c; ++j) {
        const uint16_t t = __ldg(qh.packed_t + j * KL + p);
        const double v = (double)hs[t & 0x7fff];
        acc += (t >> 15) ? -v : v;
      }
      qbits[p] = acc > 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < qh.l; t += kFwdWarps * 32) {
      uint32_t key = 0;
      for (int kk = 0; kk < qh.k; ++kk) key |= (uint32_t)qbits[t * qh.k + kk] << kk;
      qh.keys[(int64_t)i * qh.l + t] = key;
    }
  }
  // the batch's last CTA to finish builds the live-unit permutation
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  build_live_cols(hp, gridDim.x, hmask, live);
  if (threadIdx.x == 0) *ticket = 0;  // self-resetting
}

void launch_hidden_forward(int hp, int b, const int32_t* x_ptr, const int32_t* x_idx, const float* x_val,
                           const float* w1t, const float* b1, float* h, uint32_t* hmask, int32_t* live,
                           int32_t* ticket, cudaStream_t s, const QueryHash* qh) {
  if (b <= 0) return;
  if (qh) {
    SLIDE_NV_DISPATCH(hp, (hidden_fwd_kernel<NV, true><<<b, FwdWarps<NV>::value * 32, 0, s>>>(
                              hp, x_ptr, x_idx, x_val, w1t, b1, h, hmask, live, ticket, *qh)));
  } else {
    SLIDE_NV_DISPATCH(hp, (hidden_fwd_kernel<NV><<<b, FwdWarps<NV>::value * 32, 0, s>>>(
                              hp, x_ptr, x_idx, x_val, w1t, b1, h, hmask, live, ticket, QueryHash{})));
  }
  SLIDE_LAUNCH_CHECK();
}

// lane's unit in each of the G = hp / 32 groups (see build_live_cols); returns
// the number of groups that hold live units
template <int G>
__device__ __forceinline__ int live_lanes(const int32_t* __restrict__ live, int (&col)[G]) {
  const int lane = threadIdx.x & 31;
  const int n = __ldg(live);
#pragma unroll
  for (int g = 0; g < G; ++g) col[g] = __ldg(live + 1 + g * 32 + lane);
  return (n + 31) >> 5;
}

// Device-side dispatch on the live group count ng (read on the device, so
// graph replays adapt): FN<NG>(...) with NG >= max(ng, 1) from a short list.
#define SLIDE_NG_DISPATCH(NV, ng, FN, ...)                                  \
  do {                                                                      \
    if ((ng) <= 1) FN<1>(__VA_ARGS__);                                      \
    else if ((ng) == 2) FN<2>(__VA_ARGS__);                                 \
    else if ((NV) == 1) FN<4>(__VA_ARGS__);                                 \
    else if ((ng) <= 4) FN<4>(__VA_ARGS__);                                 \
    else if ((NV) == 2) FN<(NV) * 4>(__VA_ARGS__);                          \
    else if ((ng) <= 8) FN<8>(__VA_ARGS__);                                 \
    else FN<(NV) * 4>(__VA_ARGS__);                                         \
  } while (0)

// ------------------------------------------------------------ output logits
// z[p] = W2[row_p] . h[slot_p] + b2[row_p] for every (slot, active row)
// pair (network.py:266).
// Row-major logits.  The distinct active rows (ascending, the stable group-by)
// are cut into 64-row tiles; each tile picks its path from its own pair
// density:
//  * dense (>= 1/8 of the tile's rows x B cells are pairs): a register-tiled
//    fp32 product of the tile's W2 rows with all of h (64 x 128 outputs per
//    CTA, k in chunks of 32 through shared memory), then the pairs are picked
//    out through the slot masks -- wide-in rows are held by ~half the batch;
//  * sparse: one warp per row, the row in registers, dotted with each of its
//    samples; 4 pairs share one butterfly (6 shuffles instead of 20).
__device__ __forceinline__ float reduce4(float v0, float v1, float v2, float v3, int lane) {
  const bool hi16 = lane & 16;
  float k0 = hi16 ? v2 : v0, k1 = hi16 ? v3 : v1;
  k0 += __shfl_xor_sync(0xffffffffu, hi16 ? v0 : v2, 16);
  k1 += __shfl_xor_sync(0xffffffffu, hi16 ? v1 : v3, 16);
  const bool hi8 = lane & 8;
  float k = hi8 ? k1 : k0;
  k += __shfl_xor_sync(0xffffffffu, hi8 ? k0 : k1, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;  // the sum for pair ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1)
}

// position of the r-th (0-based) set bit of w
__device__ __forceinline__ int select_bit(uint32_t w, int r) {
  int pos = 0;
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {
    const int c = __popc(w & ((1u << sh) - 1u));
    if (c <= r) {
      r -= c;
      pos += sh;
      w >>= sh;
    }
  }
  return pos;
}

// slot of the t-th item of a key's mask (lane-held words wd, their
// inclusive popcount prefix incl; wpk <= 32 words)
__device__ __forceinline__ int mask_select(uint32_t wd, int incl, int wpk, int t) {
  int lo = 0, hi = wpk - 1;  // first word whose inclusive count exceeds t
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__shfl_sync(0xffffffffu, incl, mid) > t) hi = mid;
    else lo = mid + 1;
  }
  const uint32_t w = __shfl_sync(0xffffffffu, wd, lo);
  const int before = __shfl_sync(0xffffffffu, incl, lo) - __popc(w);
  return 32 * lo + select_bit(w, t - before);
}

template <int NV>
__device__ __forceinline__ void logits_row_warp(int hp, int64_t u, const GroupView& g, const int32_t* __restrict__ pslot,
                                                const float* __restrict__ w2, const float* __restrict__ b2,
                                                const float* __restrict__ h, float* __restrict__ z,
                                                const int (&col)[NV * 4], int ng) {
  constexpr int G = NV * 4;
  const int lane = threadIdx.x & 31;
  const int mine = ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
  const int r = g.uniq[u];
  const int s0 = g.seg_off[u], len = g.seg_cnt[u];
  const float bias = b2[r];
  float w[G];
#pragma unroll
  for (int q = 0; q < G; ++q) w[q] = q < ng ? __ldg(w2 + (int64_t)r * hp + col[q]) : 0.f;
  // place-free grouping: slots from the row's mask, logits in row order
  const bool rows_mode = g.order == nullptr;
  uint32_t wd = 0;
  int incl = 0;
  if (rows_mode) {
    wd = lane < g.wpk ? __ldg(g.mask_of(u) + lane) : 0u;
    incl = __popc(wd);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
  }
  for (int j0 = 0; j0 < len; j0 += 32) {
    int pl, sl;
    if (rows_mode) {
      const int t = min(j0 + lane, len - 1);
      if (g.wpk == 4) {  // the row's four words are in every lane (wd / incl of lanes 0..3)
        const int c0 = __shfl_sync(0xffffffffu, incl, 0), c1 = __shfl_sync(0xffffffffu, incl, 1),
                  c2 = __shfl_sync(0xffffffffu, incl, 2);
        const int w = (t >= c0) + (t >= c1) + (t >= c2);
        const uint32_t wv = __shfl_sync(0xffffffffu, wd, w);
        const int before = w == 0 ? 0 : w == 1 ? c0 : w == 2 ? c1 : c2;
        sl = 32 * w + select_bit(wv, t - before);
      } else {
        sl = mask_select(wd, incl, g.wpk, t);
      }
      pl = s0 + j0 + lane;
    } else {
      pl = j0 + lane < len ? g.order[s0 + j0 + lane] : 0;
      sl = j0 + lane < len ? pslot[pl] : 0;
    }
    const int nc = min(32, len - j0);
    for (int q2 = 0; q2 < nc; q2 += 4) {
      float v[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int slot = __shfl_sync(0xffffffffu, sl, min(q2 + t, nc - 1));
        const float* hr = h + (int64_t)slot * hp;
        float d = 0.f;
#pragma unroll
        for (int q = 0; q < G; ++q)
          if (q < ng) d = fmaf(w[q], __ldg(hr + col[q]), d);
        v[t] = d;
      }
      const float sum = reduce4(v[0], v[1], v[2], v[3], lane);
      const int p = __shfl_sync(0xffffffffu, pl, min(q2 + mine, nc - 1));
      if ((lane & 7) == 0 && q2 + mine < nc) z[p] = sum + bias;
    }
  }
}

constexpr int kTM = 64;         // rows per tile
constexpr int kTN = 64;         // samples per tile
constexpr int kKC = 32;         // k (live units) per shared-memory stage
constexpr int kLd = kKC + 4;    // padded row stride (conflict-free float4 reads)
constexpr int kMaskWords = 32;  // B <= 1024
constexpr int kZLd = kTN + 1;  // the 64 x 64 logit tile in shared memory (reuses the staging area)
static_assert(kTM * kZLd <= 2 * kTM * kLd, "logit tile must fit the staging area");
constexpr int kTileSmem = (2 * kTM * kLd) * 4 + kTM * 16;

// dense work item = (64-row tile, 64-sample block).  A row tile goes dense
// unless its pairs cover < 1/64 of its rows x B cells (then the per-row
// kernel is cheaper); wide-in tiles are 10-50% full.
__device__ __forceinline__ bool tile_is_dense(const GroupView& g, int64_t u0, int nrow, int b) {
  const int64_t last = u0 + nrow - 1;
  const int64_t npairs = (int64_t)g.seg_off[last] + g.seg_cnt[last] - g.seg_off[u0];
  return npairs * 64 >= (int64_t)nrow * b;
}

template <int NV>
__global__ void __launch_bounds__(256, 3) logits_tiles_kernel(int hp, int b, GroupView g,
                                                              const int32_t* __restrict__ pslot,
                                                              const float* __restrict__ w2,
                                                              const float* __restrict__ b2,
                                                              const float* __restrict__ h,
                                                              const int32_t* __restrict__ live,
                                                              float* __restrict__ z) {
  extern __shared__ __align__(16) float tsm[];
  float* ws = tsm;                                   // [kTM][kLd]
  float* hs = ws + kTM * kLd;                        // [kTN][kLd]
  float* zt = tsm;                                   // [kTM][kZLd] after the product
  int* base_s = reinterpret_cast<int*>(hs + kTN * kLd);  // [kTM] first sorted position of each row
  int* len_s = base_s + kTM;                         // [kTM] its pair count
  float* bias_s = reinterpret_cast<float*>(len_s + kTM);
  int* wrow_s = reinterpret_cast<int*>(bias_s + kTM);  // [kTM] W2 row of each tile row
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t nu = *g.n_uniq;
  const int64_t tiles = (nu + kTM - 1) / kTM;
  const int nsb = (b + kTN - 1) / kTN;
  // k runs over the live units only (32 per stage, the last stage's tail on
  // dead units, whose h is 0): the lane's unit of every stage
  const int kn = ((__ldg(live) + 31) >> 5) * 32;
  for (int64_t item = blockIdx.x; item < tiles * nsb; item += gridDim.x) {
    const int64_t tile = item / nsb;
    const int s0 = (int)(item - tile * nsb) * kTN;
    const int64_t u0 = tile * kTM;
    const int nrow = (int)min((int64_t)kTM, nu - u0);
    if (!tile_is_dense(g, u0, nrow, b)) continue;  // sparse tile: logits_rows_kernel
    if (tid < nrow) {
      const int64_t u = u0 + tid;
      base_s[tid] = g.seg_off[u];
      len_s[tid] = g.seg_cnt[u];
      const int r = g.uniq[u];
      bias_s[tid] = b2[r];
      wrow_s[tid] = r;
    }
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[j][jj] = 0.f;
    for (int k0 = 0; k0 < kn; k0 += kKC) {
      // stage 64 W rows and 64 h rows of these 32 units: 16 loads in flight
      const int c = __ldg(live + 1 + k0 + lane);
      float lw[8], lh[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int row = warp + q * 8;
        lw[q] = row < nrow ? __ldg(w2 + (int64_t)wrow_s[row] * hp + c) : 0.f;
        lh[q] = s0 + row < b ? __ldg(h + (int64_t)(s0 + row) * hp + c) : 0.f;
      }
      __syncthreads();  // previous readers of ws / hs are done
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int row = warp + q * 8;
        ws[row * kLd + lane] = lw[q];
        hs[row * kLd + lane] = lh[q];
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kKC; kk += 4) {
        float4 wv[4], hv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) wv[j] = *reinterpret_cast<const float4*>(&ws[(ty + 16 * j) * kLd + kk]);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) hv[jj] = *reinterpret_cast<const float4*>(&hs[(tx + 16 * jj) * kLd + kk]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[j][jj] = fmaf(wv[j].x, hv[jj].x, acc[j][jj]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[j][jj] = fmaf(wv[j].y, hv[jj].y, acc[j][jj]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[j][jj] = fmaf(wv[j].z, hv[jj].z, acc[j][jj]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[j][jj] = fmaf(wv[j].w, hv[jj].w, acc[j][jj]);
      }
    }
    // the 64 x 64 block to shared memory; then the tile's pairs -- one
    // contiguous range of the grouping, each row's slot-ascending -- are
    // walked flat by the whole CTA (coalesced slots and pair ids, 4
    // positions in flight per thread) and those of this sample block pick
    // their logit
    __syncthreads();  // readers of ws / hs are done
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) zt[(ty + 16 * j) * kZLd + tx + 16 * jj] = acc[j][jj];
    __syncthreads();
    // each row's pairs are slot-ascending, so this sample block's pairs of
    // a row are one sub-range of its segment, found from the row's slot
    // mask: lane r < 8 of warp w sizes row w + 8 r, then the warp walks
    // those rows' sub-ranges (coalesced slots and pair ids)
    {
      int lo_l = 0, n_l = 0;
      const int rr = warp + 8 * lane;
      if (lane < 8 && rr < nrow) {
        const uint32_t* mk = g.mask_of(u0 + rr);
        const int wa = s0 >> 5, wb = (s0 + kTN) >> 5;  // kTN = 64: whole words
        int below = 0, in = 0;
        for (int w = 0; w < g.wpk; ++w) {
          const int c = __popc(__ldg(mk + w));
          if (w < wa) below += c;
          else if (w < wb) in += c;
        }
        lo_l = base_s[rr] + below;
        n_l = in;
      }
#pragma unroll 2
      for (int r = 0; r < 8; ++r) {
        const int row = warp + 8 * r;
        if (row >= nrow) break;
        const int lo = __shfl_sync(0xffffffffu, lo_l, r), n = __shfl_sync(0xffffffffu, n_l, r);
        if (g.order == nullptr) {
          // place-free grouping: the block's 64 slots are mask words s0/32
          // and s0/32 + 1; lane l takes slots s0 + l and s0 + 32 + l, the
          // logits go to their row-order positions
          const uint32_t* mk = g.mask_of(u0 + row);
          const int wa = s0 >> 5;
          const uint32_t m0 = wa < g.wpk ? __ldg(mk + wa) : 0u, m1 = wa + 1 < g.wpk ? __ldg(mk + wa + 1) : 0u;
          const uint32_t lt = (1u << lane) - 1u;
          if ((m0 >> lane) & 1u) z[lo + __popc(m0 & lt)] = zt[row * kZLd + lane] + bias_s[row];
          if ((m1 >> lane) & 1u) z[lo + __popc(m0) + __popc(m1 & lt)] = zt[row * kZLd + 32 + lane] + bias_s[row];
          continue;
        }
        for (int j = lane; j < n; j += 32) {
          const int pos = lo + j;
          const int sl = g.sslot[pos] - s0;
          z[g.order[pos]] = zt[row * kZLd + sl] + bias_s[row];
        }
      }
    }
    __syncthreads();  // zt / base / len / bias / wrow reuse by the next item
  }
}

// rows of the sparse tiles: one warp per row
template <int NV>
__global__ void __launch_bounds__(256) logits_rows_kernel(int hp, int b, GroupView g, const int32_t* __restrict__ pslot,
                                                          const float* __restrict__ w2, const float* __restrict__ b2,
                                                          const float* __restrict__ h,
                                                          const int32_t* __restrict__ live, float* __restrict__ z,
                                                          int dense_ok) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nu = *g.n_uniq;
  int col[NV * 4];
  const int ng = live_lanes<NV * 4>(live, col);
  for (int64_t u = gw; u < nu; u += nw) {
    const int64_t u0 = u / kTM * kTM;
    if (dense_ok && tile_is_dense(g, u0, (int)min((int64_t)kTM, nu - u0), b)) continue;  // logits_tiles_kernel
    logits_row_warp<NV>(hp, u, g, pslot, w2, b2, h, z, col, ng);
  }
}

// Sparse active sets (wide-out, scaled: ~1 sample per active row): the
// logits pair by pair in sample-major order, no row grouping -- 8 lanes per
// pair, each lane 4 live units of every live group, an 8-lane butterfly.
__global__ void __launch_bounds__(256) logits_pairs_kernel(int hp, const int32_t* __restrict__ n_dev,
                                                           const int32_t* __restrict__ prow,
                                                           const int32_t* __restrict__ pslot,
                                                           const float* __restrict__ w2, const float* __restrict__ b2,
                                                           const float* __restrict__ h,
                                                           const int32_t* __restrict__ live, float* __restrict__ z) {
  const int lane = threadIdx.x & 31, g8 = lane & 7;
  const int64_t n = *n_dev;
  const int ng = max(1, (__ldg(live) + 31) >> 5);
  const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int64_t np = ((int64_t)gridDim.x * blockDim.x) >> 3;
  for (int64_t p = p0; p - (lane >> 3) < n; p += np) {  // the warp's 4 pairs stay together for the butterfly
    const bool ok = p < n;
    const int r = ok ? prow[p] : 0, sl = ok ? pslot[p] : 0;
    const float* wr = w2 + (int64_t)r * hp;
    const float* hr = h + (int64_t)sl * hp;
    float acc = 0.f;
    for (int q = 0; q < ng; ++q) {
      int c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] = __ldg(live + 1 + 32 * q + 4 * g8 + k);
#pragma unroll
      for (int k = 0; k < 4; ++k) acc = fmaf(__ldg(wr + c[k]), __ldg(hr + c[k]), acc);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (ok && g8 == 0) z[p] = acc + b2[r];
  }
}

void launch_logits_pairs(int hp, const int32_t* n_dev, int64_t n_max, const int32_t* prow, const int32_t* pslot,
                         const float* w2, const float* b2, const float* h, const int32_t* live, float* z,
                         cudaStream_t s) {
  if (n_max <= 0) return;
  const int grid = (int)std::min<int64_t>(ceil_div(n_max, 32), (int64_t)kSms * 16);
  logits_pairs_kernel<<<grid, 256, 0, s>>>(hp, n_dev, prow, pslot, w2, b2, h, live, z);
  SLIDE_LAUNCH_CHECK();
}

void launch_logits_rows(int hp, int b, const GroupView& g, const int32_t* pslot, const float* w2, const float* b2,
                        const float* h, const int32_t* live, float* z, cudaStream_t s, cudaStream_t s_rows) {
  if (g.u_max <= 0) return;
  // dense tiles need the whole batch's slot masks in 32 words
  const int dense_ok = b <= 32 * kMaskWords;
  if (dense_ok) {
    const int grid = (int)std::min<int64_t>(ceil_div(g.u_max, kTM) * ceil_div(b, kTN), (int64_t)kSms * 3);
    SLIDE_NV_DISPATCH(hp, ({
      SLIDE_CUDA(cudaFuncSetAttribute(logits_tiles_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kTileSmem));
      logits_tiles_kernel<NV><<<grid, 256, kTileSmem, s>>>(hp, b, g, pslot, w2, b2, h, live, z);
    }));
    SLIDE_LAUNCH_CHECK();
  }
  const int rgrid = (int)std::min<int64_t>(ceil_div(g.u_max, 8), (int64_t)kSms * 8);
  SLIDE_NV_DISPATCH(hp, (logits_rows_kernel<NV><<<rgrid, 256, 0, s_rows>>>(hp, b, g, pslot, w2, b2, h, live, z,
                                                                            dense_ok)));
  SLIDE_LAUNCH_CHECK();
}

// ---------------------------------------------------- softmax + CE + delta
// p = softmax over the active set (max-shifted, network.py:282-285);
// delta = p - [label]/|Y| (network.py:308-309); loss = mean over labels of
// -log(max(p_y, 1e-300)) (network.py:154-158), taken as a log-softmax.
// ROWS: z is in the place-free row grouping's order; a pair's position is
// read off its row's slot mask (g.pos_of), its error and slot go to dsort /
// sslot at that position
// T threads per sample: 1,024 for large active sets, 128 when a sample holds
// at most ~1,000 pairs (the block-wide reductions of 32 warps cost more than
// the set's arithmetic there; B = 1,024 samples: 23 -> a few us).
template <bool ROWS, int T>
__global__ void __launch_bounds__(T) softmax_kernel(const int32_t* __restrict__ offs,
                                                      const uint8_t* __restrict__ plab,
                                                      const int32_t* __restrict__ y_ptr, const float* __restrict__ z,
                                                      float* __restrict__ prob, float* __restrict__ delta,
                                                      double* __restrict__ loss, const int32_t* __restrict__ inv,
                                                      float* __restrict__ dsort, const int32_t* __restrict__ prow,
                                                      GroupView g, int32_t* __restrict__ sslot) {
  using RF = cub::BlockReduce<float, T>;
  using RD = cub::BlockReduce<double, T>;
  __shared__ union {
    typename RF::TempStorage f;
    typename RD::TempStorage d;
  } tmp;
  __shared__ float s_max, s_sum;
  const int i = blockIdx.x, tid = threadIdx.x;
  const int o = offs[i], n = offs[i + 1] - o;
  const int ny = y_ptr[i + 1] - y_ptr[i];
  // the first kSmC logits per thread stay in registers (with their
  // exponentials) across the three passes; a longer set re-reads the rest
  constexpr int kSmC = 8;
  float zr[kSmC], er[kSmC];
  int pr[kSmC];  // ROWS: the pair's row-order position
  auto pos_of = [&](int k) { return ROWS ? g.pos_of(prow[o + k], i) : o + k; };
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < kSmC; ++j) {
    const int k = tid + j * T;
    pr[j] = k < n ? pos_of(k) : 0;
    zr[j] = k < n ? z[pr[j]] : -INFINITY;
    mx = fmaxf(mx, zr[j]);
  }
  for (int k = tid + kSmC * T; k < n; k += T) mx = fmaxf(mx, z[pos_of(k)]);
  mx = RF(tmp.f).Reduce(mx, cub::Max());
  if (tid == 0) s_max = n > 0 ? mx : 0.f;
  __syncthreads();
  mx = s_max;
  float se = 0.f;
#pragma unroll
  for (int j = 0; j < kSmC; ++j) {
    er[j] = tid + j * T < n ? expf(zr[j] - mx) : 0.f;
    se += er[j];
  }
  for (int k = tid + kSmC * T; k < n; k += T) se += expf(z[pos_of(k)] - mx);
  se = RF(tmp.f).Sum(se);
  if (tid == 0) s_sum = se;
  __syncthreads();
  se = s_sum;
  const float lse = logf(se);
  const float inv_ny = ny > 0 ? 1.f / (float)ny : 0.f;
  double lsum = 0.0;
#pragma unroll
  for (int j = 0; j < kSmC; ++j) {
    const int k = tid + j * T;
    if (k >= n) break;
    const float zz = zr[j] - mx;
    const float p = er[j] / se;
    const int lab = plab[o + k];
    prob[o + k] = p;
    const float dl = lab ? p - inv_ny : p;
    delta[o + k] = dl;
    if (ROWS) {
      dsort[pr[j]] = dl;
      sslot[pr[j]] = i;
    } else if (inv) {
      dsort[inv[o + k]] = dl;
    }
    if (lab) {
      double nl = -((double)zz - (double)lse);
      lsum += (nl < 690.7755278982137 || nl != nl) ? nl : 690.7755278982137;  // NaN propagates (np.maximum)
    }
  }
  for (int k = tid + kSmC * T; k < n; k += T) {
    const int pk = pos_of(k);
    const float zz = z[pk] - mx;
    const float p = expf(zz) / se;
    const int lab = plab[o + k];
    prob[o + k] = p;
    const float dl = lab ? p - inv_ny : p;
    delta[o + k] = dl;
    if (ROWS) {  // the W2 Adam reads the errors and slots in row-grouped order
      dsort[pk] = dl;
      sslot[pk] = i;
    } else if (inv) {
      dsort[inv[o + k]] = dl;
    }
    if (lab) {
      double nl = -((double)zz - (double)lse);
      lsum += (nl < 690.7755278982137 || nl != nl) ? nl : 690.7755278982137;  // NaN propagates (np.maximum)
    }
  }
  lsum = RD(tmp.d).Sum(lsum);
  if (tid == 0) loss[i] = ny > 0 ? lsum / ny : (double)NAN;
}

__global__ void scatter_sorted_kernel(const int32_t* __restrict__ n_dev, const int32_t* __restrict__ inv,
                                      const float* __restrict__ src, float* __restrict__ dst) {
  const int n = *n_dev;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) dst[inv[q]] = src[q];
}

void launch_scatter_sorted(const int32_t* n_dev, int64_t n_max, const int32_t* inv, const float* src, float* dst,
                           cudaStream_t s) {
  if (n_max <= 0) return;
  scatter_sorted_kernel<<<(int)std::min<int64_t>(ceil_div(n_max, 256), (int64_t)kSms * 8), 256, 0, s>>>(n_dev, inv, src,
                                                                                                       dst);
  SLIDE_LAUNCH_CHECK();
}

void launch_softmax(int b, const int32_t* offs, const uint8_t* plab, const int32_t* y_ptr, const float* z,
                    float* prob, float* delta, double* loss, const int32_t* inv, float* dsort, cudaStream_t s,
                    const int32_t* prow, const GroupView* rows, int32_t* sslot, bool small_sets) {
  if (b <= 0) return;
  if (rows) {
    if (small_sets)
      softmax_kernel<true, 128><<<b, 128, 0, s>>>(offs, plab, y_ptr, z, prob, delta, loss, nullptr, dsort, prow,
                                                  *rows, sslot);
    else
      softmax_kernel<true, 1024><<<b, 1024, 0, s>>>(offs, plab, y_ptr, z, prob, delta, loss, nullptr, dsort, prow,
                                                    *rows, sslot);
  } else if (small_sets) {
    softmax_kernel<false, 128><<<b, 128, 0, s>>>(offs, plab, y_ptr, z, prob, delta, loss, inv, dsort, nullptr,
                                                 GroupView{}, nullptr);
  } else {
    softmax_kernel<false, 1024><<<b, 1024, 0, s>>>(offs, plab, y_ptr, z, prob, delta, loss, inv, dsort, nullptr,
                                                   GroupView{}, nullptr);
  }
  SLIDE_LAUNCH_CHECK();
}

// ------------------------------------------------ lazy softmax (rows mode)
// Training steps under the place-free grouping do not materialise p / delta
// per pair: per 64-row tile of the grouping and per slot, the online (max,
// sum exp) of the slot's logits in those rows; per sample, the tiles
// combined (max, then sum) and the label loss terms; the hidden gradient and
// the W2 Adam then compute each pair's error from its logit where they read
// it (row order, coalesced): delta = exp(z - M_i) / S_i - [label] / |Y_i|.
constexpr int kLzRows = 16;  // rows per tile: every slot's loads of a tile in flight at once

__global__ void __launch_bounds__(256) softmax_partials_kernel(GroupView g, const uint32_t* __restrict__ lmask,
                                                               const float* __restrict__ z, int b,
                                                               float2* __restrict__ part) {
  __shared__ int s_off[kLzRows];
  __shared__ uint32_t s_mk[kLzRows][32], s_pre[kLzRows][32];
  const int64_t nu = *g.n_uniq;
  const int64_t tiles = (nu + kLzRows - 1) / kLzRows;
  const int wpk = g.wpk;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int nr = (int)min((int64_t)kLzRows, nu - t * kLzRows);
    __syncthreads();  // the previous tile's readers are done
    for (int q = threadIdx.x; q < nr * wpk; q += blockDim.x) {
      const int r = q / wpk, w = q - r * wpk;
      const int64_t u = t * kLzRows + r;
      s_mk[r][w] = __ldg(g.mask_of(u) + w);
      if (w == 0) s_off[r] = __ldg(g.seg_off + u);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {  // exclusive popcount prefix per row
      uint32_t acc = 0;
      for (int w = 0; w < wpk; ++w) {
        s_pre[r][w] = acc;
        acc += __popc(s_mk[r][w]);
      }
    }
    __syncthreads();
    for (int slot = threadIdx.x; slot < b; slot += blockDim.x) {
      const int w = slot >> 5;
      const uint32_t bit = 1u << (slot & 31), lo = bit - 1u;
      float zv[kLzRows];
#pragma unroll
      for (int r = 0; r < kLzRows; ++r) {  // the slot's logits of the tile, all loads in flight
        const uint32_t word = r < nr ? s_mk[r][w] : 0u;
        zv[r] = (word & bit) ? __ldg(z + s_off[r] + s_pre[r][w] + __popc(word & lo)) : -INFINITY;
      }
      float m = -INFINITY;
#pragma unroll
      for (int r = 0; r < kLzRows; ++r) m = fmaxf(m, zv[r]);
      float sum = 0.f;
#pragma unroll
      for (int r = 0; r < kLzRows; ++r) sum += zv[r] == -INFINITY ? 0.f : expf(zv[r] - m);
      part[t * b + slot] = make_float2(m, sum);
    }
  }
}

// per sample: M, 1 / S, 1 / |Y| and the loss (reference network.py:154-158,
// 282-285: -log p_y = M + log S - z_y per label, clamped at -log 1e-300)
__global__ void __launch_bounds__(256) softmax_combine_kernel(GroupView g, const float2* __restrict__ part, int b,
                                                              const int32_t* __restrict__ y_ptr,
                                                              const int32_t* __restrict__ y_idx,
                                                              const float* __restrict__ z, float* __restrict__ stat,
                                                              double* __restrict__ loss) {
  using RF = cub::BlockReduce<float, 256>;
  using RD = cub::BlockReduce<double, 256>;
  __shared__ union {
    typename RF::TempStorage f;
    typename RD::TempStorage d;
  } tmp;
  __shared__ float s_m, s_s;
  const int i = blockIdx.x;
  const int64_t tiles = (*g.n_uniq + kLzRows - 1) / kLzRows;
  float m = -INFINITY;
  for (int64_t t = threadIdx.x; t < tiles; t += blockDim.x) m = fmaxf(m, part[t * b + i].x);
  m = RF(tmp.f).Reduce(m, cub::Max());
  if (threadIdx.x == 0) s_m = m;
  __syncthreads();
  m = s_m;
  float sum = 0.f;
  for (int64_t t = threadIdx.x; t < tiles; t += blockDim.x) {
    const float2 pt = part[t * b + i];
    if (pt.y > 0.f) sum += pt.y * expf(pt.x - m);
  }
  __syncthreads();
  sum = RF(tmp.f).Sum(sum);
  if (threadIdx.x == 0) s_s = sum;
  __syncthreads();
  sum = s_s;
  const int y0 = y_ptr[i], ny = y_ptr[i + 1] - y0;
  const float lse = logf(sum);
  double lsum = 0.0;
  for (int k = threadIdx.x; k < ny; k += blockDim.x) {
    const int row = y_idx[y0 + k];
    const float zz = __ldg(z + g.pos_of(row, i)) - m;
    const double nl = -((double)zz - (double)lse);
    lsum += (nl < 690.7755278982137 || nl != nl) ? nl : 690.7755278982137;  // NaN propagates (np.maximum)
  }
  __syncthreads();
  lsum = RD(tmp.d).Sum(lsum);
  if (threadIdx.x == 0) {
    loss[i] = ny > 0 ? lsum / ny : (double)NAN;
    stat[3 * i] = m;
    stat[3 * i + 1] = sum > 0.f ? 1.f / sum : 0.f;
    stat[3 * i + 2] = ny > 0 ? 1.f / (float)ny : 0.f;
  }
}

__device__ __forceinline__ float lazy_delta(float zz, const float* __restrict__ stat, int slot, bool lab) {
  const float p = expf(zz - __ldg(stat + 3 * slot)) * __ldg(stat + 3 * slot + 1);
  return lab ? p - __ldg(stat + 3 * slot + 2) : p;
}

void launch_softmax_lazy(int b, const GroupView& g, const uint32_t* lmask, const float* z, const int32_t* y_ptr,
                         const int32_t* y_idx, float2* part, float* stat, double* loss, cudaStream_t s) {
  if (b <= 0) return;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(g.u_max, kLzRows), (int64_t)kSms * 4));
  softmax_partials_kernel<<<grid, 256, 0, s>>>(g, lmask, z, b, part);
  SLIDE_LAUNCH_CHECK();
  softmax_combine_kernel<<<b, 256, 0, s>>>(g, part, b, y_ptr, y_idx, z, stat, loss);
  SLIDE_LAUNCH_CHECK();
}

int64_t softmax_lazy_parts(int64_t u_max, int b) { return std::max<int64_t>(1, ceil_div(u_max, kLzRows)) * b; }

// readouts of a lazy step: per pair (sample-major) its p (what 5) or delta (6)
__global__ void lazy_pairs_kernel(const int32_t* __restrict__ offs, const int32_t* __restrict__ prow,
                                  const uint8_t* __restrict__ plab, GroupView g, const float* __restrict__ z,
                                  const float* __restrict__ stat, float* __restrict__ out, int want_delta) {
  const int i = blockIdx.x;
  const int o = offs[i], n = offs[i + 1] - o;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const float zz = z[g.pos_of(prow[o + k], i)];
    const float p = expf(zz - stat[3 * i]) * stat[3 * i + 1];
    out[o + k] = want_delta && plab[o + k] ? p - stat[3 * i + 2] : p;
  }
}

void launch_lazy_pairs(int b, const int32_t* offs, const int32_t* prow, const uint8_t* plab, const GroupView& g,
                       const float* z, const float* stat, float* out, bool want_delta, cudaStream_t s) {
  if (b <= 0) return;
  lazy_pairs_kernel<<<b, 256, 0, s>>>(offs, prow, plab, g, z, stat, out, want_delta ? 1 : 0);
  SLIDE_LAUNCH_CHECK();
}

__global__ void rows_pairs_kernel(const int32_t* __restrict__ offs, const int32_t* __restrict__ prow, GroupView g,
                                  const float* __restrict__ src, float* __restrict__ dst, int to_pairs) {
  const int i = blockIdx.x;
  const int o = offs[i], n = offs[i + 1] - o;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int pos = g.pos_of(prow[o + k], i);
    if (to_pairs) dst[o + k] = src[pos];
    else dst[pos] = src[o + k];
  }
}

void launch_rows_pairs(int b, const int32_t* offs, const int32_t* prow, const GroupView& g, const float* src,
                       float* dst, bool to_pairs, cudaStream_t s) {
  if (b <= 0) return;
  rows_pairs_kernel<<<b, 256, 0, s>>>(offs, prow, g, src, dst, to_pairs ? 1 : 0);
  SLIDE_LAUNCH_CHECK();
}

// -------------------------------------------------------- hidden gradient
// dh_i = W2[A_i, :]^T delta_i with the pre-update W2, kept on nz(h_i)
// (network.py:328-332).  Sample i's pairs are cut into S slices, one CTA
// each (B*S CTAs fill the GPU); every slice sums in a fixed order, the
// slices are added in slice order -- deterministic.  Used for the sharded
// partials; the single-GPU step uses hidden_grad_rows_kernel below (each W2
// row read once per 32-slot window from the row grouping, 28 -> 15 us at
// wide-in).
struct HiddenGradArgs {
  int hp, b, slices;
  const int32_t *offs, *prow;
  const float *delta, *w2, *h;
  const int32_t* live;
  float *part, *dh;
  int32_t *done, *work_reset;
};

// the sample's slice [beg, e) of pairs: acc[q] = sum_k delta_k W2[row_k, col[q]]
template <int NG>
__device__ __forceinline__ void hidden_grad_acc(const HiddenGradArgs& A, int beg, int e, float* red_w) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int col[NG];
#pragma unroll
  for (int q = 0; q < NG; ++q) col[q] = __ldg(A.live + 1 + q * 32 + lane);
  float acc[NG];
#pragma unroll
  for (int q = 0; q < NG; ++q) acc[q] = 0.f;
  int k = beg + warp;
  constexpr int U = NG <= 2 ? 8 : 4;  // rows in flight per warp
  for (; k + 8 * (U - 1) < e; k += 8 * U) {
    float r[U][NG];
    float d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      d[u] = A.delta[k + 8 * u];
      const float* rp = A.w2 + (int64_t)A.prow[k + 8 * u] * A.hp;
#pragma unroll
      for (int q = 0; q < NG; ++q) r[u][q] = __ldg(rp + col[q]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NG; ++q) acc[q] = fmaf(d[u], r[u][q], acc[q]);
  }
  for (; k < e; k += 8) {
    const float d = A.delta[k];
    const float* rp = A.w2 + (int64_t)A.prow[k] * A.hp;
#pragma unroll
    for (int q = 0; q < NG; ++q) acc[q] = fmaf(d, __ldg(rp + col[q]), acc[q]);
  }
#pragma unroll
  for (int q = 0; q < NG; ++q) red_w[warp * (NG * 32) + q * 32 + lane] = acc[q];
}

template <int NV>
__global__ void __launch_bounds__(256) hidden_grad_kernel(HiddenGradArgs A) {
  constexpr int G = NV * 4;
  __shared__ float red[8 * G * 32];
  __shared__ int s_last;
  const int hp = A.hp, b = A.b, slices = A.slices;
  // the W2 Adam's row counter: its previous use is over, its next comes after
  if (A.work_reset && blockIdx.x == 0 && threadIdx.x == 0) *A.work_reset = 0;
  const int i = blockIdx.x / slices, sl = blockIdx.x - i * slices;
  const int o = A.offs[i], n = A.offs[i + 1] - o;
  const int beg = o + (int)((int64_t)n * sl / slices), e = o + (int)((int64_t)n * (sl + 1) / slices);
  // only the live units' columns of W2 are read (dh is masked by h > 0)
  const int ng = (__ldg(A.live) + 31) >> 5;
  const int ngp = ng <= 2 ? (ng < 1 ? 1 : ng) : (NV == 1 || ng <= 4 ? 4 : (NV == 2 || ng > 8 ? G : 8));
  SLIDE_NG_DISPATCH(NV, ng, hidden_grad_acc, A, beg, e, red);
  __syncthreads();
  const int kn = ngp * 32;  // red holds [8][kn]
  // column k of the compact order is unit live[1 + k]; the units past the
  // live groups are dead (dh = 0), and so is h on the live groups' tail
  const float* __restrict__ h = A.h;
  for (int kk = threadIdx.x; kk < hp; kk += 256) {
    float sum = 0.f;
    if (kk < kn) {
      sum = red[kk];
#pragma unroll
      for (int w = 1; w < 8; ++w) sum += red[w * kn + kk];
    }
    if (slices == 1) {
      const int64_t q = (int64_t)i * hp + __ldg(A.live + 1 + kk);
      A.dh[q] = (h == nullptr || h[q] > 0.f) ? sum : 0.f;  // h == null: unmasked partial
    } else if (kk < kn) {
      A.part[(int64_t)sl * b * hp + (int64_t)i * hp + kk] = sum;
    }
  }
  if (slices == 1) return;
  // the sample's last slice to finish adds the slices in slice order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(A.done + i, 1) == slices - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int kk = threadIdx.x; kk < hp; kk += 256) {
    float sum = 0.f;
    if (kk < kn) {
      const int64_t q = (int64_t)i * hp + kk;
      sum = __ldcg(A.part + q);
      for (int t = 1; t < slices; ++t) sum += __ldcg(A.part + (int64_t)t * b * hp + q);
    }
    const int64_t q = (int64_t)i * hp + __ldg(A.live + 1 + kk);
    A.dh[q] = (h == nullptr || h[q] > 0.f) ? sum : 0.f;
  }
  if (threadIdx.x == 0) A.done[i] = 0;  // self-resetting
}

int hidden_grad_slices(int b) { return std::max(1, std::min(8, (int)ceil_div((int64_t)kSms * 4, b))); }

size_t hidden_grad_scratch(int b, int hp) { return (size_t)hidden_grad_slices(b) * b * hp; }

void launch_hidden_grad(int hp, int b, const int32_t* offs, const int32_t* prow, const float* delta, const float* w2,
                        const float* h, const int32_t* live, float* dh, float* part, int32_t* done, int32_t* work_reset,
                        cudaStream_t s) {
  if (b <= 0) return;
  const int S = hidden_grad_slices(b);
  HiddenGradArgs A{hp, b, S, offs, prow, delta, w2, h, live, part, dh, done, work_reset};
  SLIDE_NV_DISPATCH(hp, (hidden_grad_kernel<NV><<<b * S, 256, 0, s>>>(A)));
  SLIDE_LAUNCH_CHECK();
}

// Hidden gradient by rows (single-GPU step): the row-major grouping gives,
// per distinct active row, its slots (mask) and errors (dsort, slot order).
// CTA (window, chunk) takes 32 slots and a contiguous chunk of distinct
// rows; each warp reads its rows' grouping entries and masks at once (one
// row per lane), then walks the rows with the next row's errors and live
// W2 columns in flight, adding the errors of the window's slots into 32 x
// (32 NG) register accumulators.  The warps are summed in warp order into
// the chunk's partial; hidden_grad_reduce_kernel sums the chunks in a fixed
// order -- deterministic.  Each W2 row is read once per window instead of
// once per (sample, row) pair.
constexpr int kHgWin = 32;

struct HiddenGradRowsArgs {
  int hp, b, nwin, nchunk;
  GroupView g;
  const float *dsort, *w2, *h;
  const int32_t* live;
  float *part, *dh;
  int32_t* work_reset;
  // lazy softmax (z != null): errors made from the row-order logits, the
  // per-sample stat (M, 1/S, 1/|Y|) and the label masks, instead of dsort
  const float *z = nullptr, *stat = nullptr;
  const uint32_t* lmask = nullptr;
};

// one pass per live group g0 (32 live columns).  Lane t holds slot
// s_lo + t's error of the current row (0 where the row is not active for
// it) and its 32 accumulators (one per live column); the row's live W2
// columns go through a per-warp shared-memory line and are read back as
// broadcast float4s: 8 loads + 32 FMAs per (row, window).
__device__ __forceinline__ void hg_rows_body(const HiddenGradRowsArgs& A, float* red, float* wsm, int g0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int win = blockIdx.x % A.nwin, chunk = blockIdx.x / A.nwin;
  const int64_t nu = *A.g.n_uniq;
  const int64_t u_beg = nu * chunk / A.nchunk, u_end = nu * (chunk + 1) / A.nchunk;
  const int col = __ldg(A.live + 1 + g0 * 32 + lane);
  const unsigned below = (1u << lane) - 1u;
  float* ws = wsm + warp * 32;
  float acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.f;
  for (int64_t ub = u_beg + warp; ub < u_end; ub += 8 * 32) {
    // lane j: row ub + 8 j -- its W2 row, first sorted position, window bits
    const int64_t uj = ub + 8 * lane;
    const bool ok = uj < u_end;
    const int row_l = ok ? __ldg(A.g.uniq + uj) : 0;
    int p0_l = ok ? __ldg(A.g.seg_off + uj) : 0;
    uint32_t bits_l = 0, lbits_l = 0;
    if (ok) {
      const int64_t mo = (A.g.mask_by_key ? (int64_t)row_l : uj) * A.g.wpk;
      const uint32_t* mk = A.g.mask + mo;
      bits_l = __ldg(mk + win);
      if (A.z) lbits_l = __ldg(A.lmask + mo + win);
      for (int w = 0; w < win; ++w) p0_l += __popc(__ldg(mk + w));
    }
    const int nr = (int)min((int64_t)32, (u_end - ub + 7) / 8);
    // two-stage pipeline over the rows: errors + W2 columns of row j + 1
    // are loaded while row j is added
    auto fetch = [&](int j, float& e, float& w) {
      const uint32_t bits = __shfl_sync(0xffffffffu, bits_l, j);
      const uint32_t lbits = __shfl_sync(0xffffffffu, lbits_l, j);
      const int p0 = __shfl_sync(0xffffffffu, p0_l, j);
      const int r = __shfl_sync(0xffffffffu, row_l, j);
      if ((bits >> lane) & 1u) {
        const int pos = p0 + __popc(bits & below);
        e = A.z ? lazy_delta(__ldg(A.z + pos), A.stat, win * kHgWin + lane, (lbits >> lane) & 1u)
                : __ldg(A.dsort + pos);
      } else {
        e = 0.f;
      }
      w = bits ? __ldg(A.w2 + (int64_t)r * A.hp + col) : 0.f;
    };
    float e, w;
    fetch(0, e, w);
    for (int j = 0; j < nr; ++j) {
      float e_n = 0.f, w_n = 0.f;
      if (j + 1 < nr) fetch(j + 1, e_n, w_n);
      __syncwarp();
      ws[lane] = w;
      __syncwarp();
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const float4 w4 = *reinterpret_cast<const float4*>(ws + 4 * k4);
        acc[4 * k4 + 0] = fmaf(e, w4.x, acc[4 * k4 + 0]);
        acc[4 * k4 + 1] = fmaf(e, w4.y, acc[4 * k4 + 1]);
        acc[4 * k4 + 2] = fmaf(e, w4.z, acc[4 * k4 + 2]);
        acc[4 * k4 + 3] = fmaf(e, w4.w, acc[4 * k4 + 3]);
      }
      e = e_n;
      w = w_n;
    }
  }
  // every warp's accumulators into its own [32 slots][33] slab, then the
  // chunk's partial as the sum over the warps in warp order (the same order,
  // bit for bit, as accumulating warp after warp -- whose eight barrier-
  // separated turns were 28% of this kernel's stall samples)
  float* slab = red + warp * (kHgWin * 33);
#pragma unroll
  for (int k = 0; k < 32; ++k) slab[lane * 33 + k] = acc[k];
  __syncthreads();
  const int s_lo = win * kHgWin;
  for (int idx = threadIdx.x; idx < kHgWin * 32; idx += 256) {
    const int t = idx >> 5, k = idx & 31;
    float sum = red[t * 33 + k];
#pragma unroll
    for (int wp = 1; wp < 8; ++wp) sum += red[wp * (kHgWin * 33) + t * 33 + k];
    if (s_lo + t < A.b) A.part[((int64_t)chunk * A.b + s_lo + t) * A.hp + g0 * 32 + k] = sum;
  }
  __syncthreads();  // red is reused by the next pass
}

__global__ void __launch_bounds__(256, 4) hidden_grad_rows_kernel(HiddenGradRowsArgs A) {
  __shared__ __align__(16) float hg_red[8 * kHgWin * 33];
  __shared__ __align__(16) float hg_w[8 * 32];
  if (A.work_reset && blockIdx.x == 0 && threadIdx.x == 0) *A.work_reset = 0;
  const int ng = max(1, (__ldg(A.live) + 31) >> 5);
  for (int g0 = 0; g0 < ng; ++g0) hg_rows_body(A, hg_red, hg_w, g0);
}

// one CTA per sample: warp w sums chunks w, w + 8, ... (lane = live column),
// the warps are added in warp order; dh = sum on h > 0, dead units 0
__global__ void __launch_bounds__(256) hidden_grad_reduce_kernel(HiddenGradRowsArgs A) {
  extern __shared__ __align__(16) float hg_sum[];  // [8][hp]
  const int i = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kn = ((__ldg(A.live) + 31) >> 5) * 32;
  for (int kk = lane; kk < kn; kk += 32) {
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
    int c = warp;
    for (; c + 24 < A.nchunk; c += 32) {
#pragma unroll
      for (int j = 0; j < 4; ++j) s4[j] += __ldcg(A.part + ((int64_t)(c + 8 * j) * A.b + i) * A.hp + kk);
    }
    float sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    for (; c < A.nchunk; c += 8) sum += __ldcg(A.part + ((int64_t)c * A.b + i) * A.hp + kk);
    hg_sum[warp * A.hp + kk] = sum;
  }
  __syncthreads();
  for (int kk = threadIdx.x; kk < A.hp; kk += 256) {
    float sum = 0.f;
    if (kk < kn)
      for (int w = 0; w < 8; ++w) sum += hg_sum[w * A.hp + kk];
    const int64_t q = (int64_t)i * A.hp + __ldg(A.live + 1 + kk);
    A.dh[q] = (A.h == nullptr || A.h[q] > 0.f) ? sum : 0.f;
  }
}

static int hg_rows_chunks(int b) {
  const int nwin = (int)ceil_div(b, kHgWin);
  return std::max(1, kSms * 4 / nwin);  // one wave at 4 CTAs per SM
}

size_t hidden_grad_rows_scratch(int b, int hp) { return (size_t)hg_rows_chunks(b) * b * hp; }

void launch_hidden_grad_rows(int hp, int b, const GroupView& g, const float* dsort, const float* w2, const float* h,
                             const int32_t* live, float* dh, float* part, int32_t* work_reset, cudaStream_t s,
                             const float* z, const float* stat, const uint32_t* lmask) {
  if (b <= 0) return;
  const int nwin = (int)ceil_div(b, kHgWin), nchunk = hg_rows_chunks(b);
  HiddenGradRowsArgs A{hp, b, nwin, nchunk, g, dsort, w2, h, live, part, dh, work_reset, z, stat, lmask};
  hidden_grad_rows_kernel<<<nwin * nchunk, 256, 0, s>>>(A);
  SLIDE_LAUNCH_CHECK();
  hidden_grad_reduce_kernel<<<b, 256, 8 * hp * 4, s>>>(A);
  SLIDE_LAUNCH_CHECK();
}

// ----------------------------------------------------------- Adam, W2 rows
// Per active output row r, the samples that hold it are applied in slot
// order (the snapshot schedule): t = steps[r] + j + 1 for the
// row's j-th sample; moments move only where h_i > 0; the bias always moves
// (network.py:428-451).
// c1 = lr / (1 - b1^t), c2 = 1 / (1 - b2^t) (bias corrections in fp64, then
// fp32): w -= c1 m / (sqrt(c2 v) + eps).  Approximate sqrt / divide (<= 2 ulp)
// keep the update far inside the 1e-4 weight tolerance.
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Hoisted optimizer constants (registers, not constant-bank reloads).
struct AdamK {
  float b1, omb1, b2, omb2, eps;
  __device__ __forceinline__ explicit AdamK(const AdamParams& ap)
      : b1(ap.b1), omb1(1.f - ap.b1), b2(ap.b2), omb2(1.f - ap.b2), eps(ap.eps) {}
};

__device__ __forceinline__ void adam_coord(float& w, float& m, float& v, float g, float c1, float c2,
                                           const AdamK& k) {
  m = fmaf(k.b1, m, k.omb1 * g);
  v = fmaf(k.b2, v, k.omb2 * (g * g));
  w -= (c1 * m) * rcp_approx(sqrt_approx(v * c2) + k.eps);
}

// predicated form: moments and weight move only when `on` (frozen otherwise)
__device__ __forceinline__ void adam_coord_if(bool on, float& w, float& m, float& v, float g, float c1, float c2,
                                              const AdamK& k) {
  const float mn = fmaf(k.b1, m, k.omb1 * g);
  const float vn = fmaf(k.b2, v, k.omb2 * (g * g));
  const float wn = w - (c1 * mn) * rcp_approx(sqrt_approx(vn * c2) + k.eps);
  m = on ? mn : m;
  v = on ? vn : v;
  w = on ? wn : w;
}

// (c1, c2) for step t: a host-built fp64 table up to the point where both
// corrections are exactly (lr, 1) in fp32; pow beyond only if the table was
// capped (betas extremely close to 1).
__device__ __forceinline__ float2 bias_corr(const AdamParams& ap, int64_t t) {
  if (t < ap.table_n) return __ldg(ap.table + t);
  if (ap.table_exact) return make_float2(ap.lr, 1.f);
  const double td = (double)t;
  return make_float2((float)((double)ap.lr / (1.0 - pow(ap.b1d, td))), (float)(1.0 / (1.0 - pow(ap.b2d, td))));
}

// predicated Adam step with the per-pair factors folded in:
// e1 = (1-b1) d, e2 = (1-b2) d^2, coordinate gradient g = d h.
__device__ __forceinline__ void adam_coord_h(bool on, float& w, float& m, float& v, float hc, float e1, float e2,
                                             float c1, float c2, const AdamK& k) {
  const float mn = fmaf(k.b1, m, e1 * hc);
  const float vn = fmaf(k.b2, v, e2 * (hc * hc));
  const float wn = fmaf(-(c1 * mn), rcp_approx(sqrt_approx(vn * c2) + k.eps), w);
  m = on ? mn : m;
  v = on ? vn : v;
  w = on ? wn : w;
}

// as adam_coord_h with sqrt(c2) hoisted per pair: den = sqrt(v) sqrt(c2) + eps
__device__ __forceinline__ void adam_coord_hs(bool on, float& w, float& m, float& v, float hc, float e1, float e2,
                                              float c1, float s2, const AdamK& k) {
  const float mn = fmaf(k.b1, m, e1 * hc);
  const float vn = fmaf(k.b2, v, e2 * (hc * hc));
  const float wn = fmaf(-(c1 * mn), rcp_approx(fmaf(sqrt_approx(vn), s2, k.eps)), w);
  m = on ? mn : m;
  v = on ? vn : v;
  w = on ? wn : w;
}

struct AdamRowsArgs {
  int hp;
  AdamParams ap;
  // sslot / dsort: each pair's slot and output error in row-grouped order
  const int32_t *n_uniq, *uniq, *seg_off, *seg_cnt, *sslot;
  const float *dsort, *h;
  const int32_t* live;
  float *w2, *m2, *v2, *b2, *mb2, *vb2;
  int64_t* steps2;
  unsigned long long* touched;
  int32_t* work;
  // lazy softmax (z != null): each pair's slot from its row's slot mask and
  // its error from the row-order logit (see softmax_partials_kernel)
  const float *z = nullptr, *stat = nullptr;
  const uint32_t *mask = nullptr, *lmask = nullptr;
  int wpk = 0;
  int vlong = 0;  // > 0: rows held by more samples than this belong to adam_rows_vlong_kernel
};

// pairs whose activations are loaded ahead of their updates (8 / NG)
template <int NG>
struct AdamPf {
  static constexpr int value = NG >= 4 ? 2 : 8 / NG;
};
constexpr int kAdamExtra = 8;  // live units past whole groups taken in scan form
constexpr int kAdamSmallLive = 64 + kAdamExtra;  // hidden_pad > 128: up to two live groups + extras run in adam_rows_small_kernel

// The persistent row loop for NG live 32-unit groups (compile-time, so the
// per-pair body has no group guards and the next kAdamPf pairs' activations
// are in flight before their updates start).
// EX > 0: besides the NG full groups, up to EX further live units (the
// count ne is read on the device) go through the scan form of the
// recurrences -- lanes = the chunk's pairs, one unit at a time, like the
// bias -- instead of a whole extra group of lanes (a batch with 33 live
// units would otherwise pay a second 32-unit group for one unit).  Lane e
// keeps extra unit e's (w, m, v).
template <int NG, int EX, bool COUNT>
__device__ __forceinline__ void adam_rows_loop(const AdamRowsArgs& A, const int (&col)[NG], float4 (*pq)[32],
                                               int (*poff)[32]) {
  constexpr int kAdamPf = AdamPf<NG>::value;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int hp = A.hp;
  int ne = 0, xc = 0;
  if (EX > 0) {
    ne = min(EX, max(0, __ldg(A.live) - NG * 32));
    xc = __ldg(A.live + 1 + NG * 32 + (lane < ne ? lane : 0));
  }
  const int nu = *A.n_uniq;
  const AdamK ak(A.ap);
  // persistent warps take rows from a counter: a CTA's slot is never held
  // by idle warps waiting on one long row; the next row is claimed while
  // this one is updated
  // (the first row of every warp is its own index: no burst of claims on
  // the counter at launch; later rows come from the counter past them)
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  int u = blockIdx.x * (blockDim.x >> 5) + wid;
  while (u < nu) {
    int u_next = 0;
    if (lane == 0) u_next = nwarps + atomicAdd(A.work, 1);
    uint32_t tmask = 0;
    const int r = A.uniq[u];
    const int s0 = A.seg_off[u], len = A.seg_cnt[u];
    if (A.vlong && len > A.vlong) {
      u = __shfl_sync(0xffffffffu, u_next, 0);
      continue;
    }
    float* wr = A.w2 + (int64_t)r * hp;
    float* mr = A.m2 + (int64_t)r * hp;
    float* vr = A.v2 + (int64_t)r * hp;
    float w[NG], m[NG], v[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      w[q] = wr[col[q]];
      m[q] = mr[col[q]];
      v[q] = vr[col[q]];
    }
    float xw = 0.f, xm = 0.f, xv = 0.f;  // lane e < ne: extra unit e
    if (EX > 0 && lane < ne) {
      xw = wr[xc];
      xm = mr[xc];
      xv = vr[xc];
    }
    float bb = A.b2[r], mb = A.mb2[r], vb = A.vb2[r];
    const int64_t st = A.steps2[r];
    // lane j holds the j-th pair of a chunk; the next chunk's slot and error
    // are loaded while this one updates
    uint32_t wd = 0, lwd = 0;
    int incl = 0;
    if (A.z) {  // lazy: the row's slot / label masks in lanes, their popcount prefix
      wd = lane < A.wpk ? __ldg(A.mask + (int64_t)r * A.wpk + lane) : 0u;
      lwd = lane < A.wpk ? __ldg(A.lmask + (int64_t)r * A.wpk + lane) : 0u;
      incl = __popc(wd);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
    }
    auto fetch = [&](int jj, int& sl, float& d) {  // every lane calls it (shuffles inside)
      if (!A.z) {
        if (jj < len) {
          sl = A.sslot[s0 + jj];
          d = A.dsort[s0 + jj];
        }
        return;
      }
      const int slot = mask_select(wd, incl, A.wpk, min(jj, len - 1));
      const bool lab = (__shfl_sync(0xffffffffu, lwd, slot >> 5) >> (slot & 31)) & 1u;
      if (jj < len) {
        sl = slot;
        d = lazy_delta(__ldg(A.z + s0 + jj), A.stat, slot, lab);
      }
    };
    int slot_n = 0;
    float d_n = 0.f;
    fetch(lane, slot_n, d_n);
    for (int c0 = 0; c0 < len; c0 += 32) {
      const int j = c0 + lane;
      const bool valid = j < len;
      const int slot_l = valid ? slot_n : 0;
      const float d_l = valid ? d_n : 0.f;
      float2 bc_l = make_float2(0.f, 1.f);
      if (valid) bc_l = bias_corr(A.ap, st + j + 1);
      if (c0 + 32 < len) fetch(j + 32, slot_n, d_n);
      const float e1_l = ak.omb1 * d_l, e2_l = ak.omb2 * d_l * d_l;
      const float s2_l = sqrt_approx(bc_l.y);
      __syncwarp();
      pq[wid][lane] = make_float4(e1_l, e2_l, bc_l.x, s2_l);
      poff[wid][lane] = slot_l * hp;
      __syncwarp();
      // Bias (gradient d, always moves): its moments are linear recurrences
      // in the chunk's pairs -> two warp scans; the weight update does not
      // feed back, so the chunk's bias steps are summed.
      {
        float a1 = valid ? ak.b1 : 1.f, x1 = e1_l, a2 = valid ? ak.b2 : 1.f, x2 = e2_l;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float pa1 = __shfl_up_sync(0xffffffffu, a1, o), px1 = __shfl_up_sync(0xffffffffu, x1, o);
          const float pa2 = __shfl_up_sync(0xffffffffu, a2, o), px2 = __shfl_up_sync(0xffffffffu, x2, o);
          if (lane >= o) {
            x1 = fmaf(a1, px1, x1);
            a1 *= pa1;
            x2 = fmaf(a2, px2, x2);
            a2 *= pa2;
          }
        }
        const float mj = fmaf(a1, mb, x1), vj = fmaf(a2, vb, x2);
        float upd = valid ? (bc_l.x * mj) * rcp_approx(fmaf(sqrt_approx(vj), s2_l, ak.eps)) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) upd += __shfl_xor_sync(0xffffffffu, upd, o);
        bb -= upd;
        mb = __shfl_sync(0xffffffffu, mj, 31);
        vb = __shfl_sync(0xffffffffu, vj, 31);
      }
      // extra units: the same scans with the pair's activation as a factor
      for (int e = 0; e < ne; ++e) {
        const int c = __shfl_sync(0xffffffffu, xc, e);
        const float hc = valid ? __ldg(A.h + ((unsigned)(slot_l * hp) + (unsigned)c)) : 0.f;
        const bool on = hc > 0.f;
        float a1 = on ? ak.b1 : 1.f, x1 = on ? e1_l * hc : 0.f;
        float a2 = on ? ak.b2 : 1.f, x2 = on ? e2_l * (hc * hc) : 0.f;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float pa1 = __shfl_up_sync(0xffffffffu, a1, o), px1 = __shfl_up_sync(0xffffffffu, x1, o);
          const float pa2 = __shfl_up_sync(0xffffffffu, a2, o), px2 = __shfl_up_sync(0xffffffffu, x2, o);
          if (lane >= o) {
            x1 = fmaf(a1, px1, x1);
            a1 *= pa1;
            x2 = fmaf(a2, px2, x2);
            a2 *= pa2;
          }
        }
        const float mj = fmaf(a1, __shfl_sync(0xffffffffu, xm, e), x1);
        const float vj = fmaf(a2, __shfl_sync(0xffffffffu, xv, e), x2);
        float upd = on ? (bc_l.x * mj) * rcp_approx(fmaf(sqrt_approx(vj), s2_l, ak.eps)) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) upd += __shfl_xor_sync(0xffffffffu, upd, o);
        const float ml = __shfl_sync(0xffffffffu, mj, 31), vl = __shfl_sync(0xffffffffu, vj, 31);
        const unsigned moved = __ballot_sync(0xffffffffu, on);
        if (lane == e) {
          xw -= upd;
          xm = ml;
          xv = vl;
          if (COUNT) tmask |= (moved ? 1u : 0u) << 31;  // (a distinct bit per lane: summed by popc below)
        }
      }
      const int nc = min(32, len - c0);
      // kAdamPf pairs at a time: their activations are loaded before the
      // first of their updates; in the chunk's tail batch the pairs past nc
      // are off
      auto batch = [&](int q0, auto tail) {
        float hv[kAdamPf][NG];
#pragma unroll
        for (int t = 0; t < kAdamPf; ++t) {
          const unsigned off = (unsigned)poff[wid][(q0 + t) & 31];
#pragma unroll
          for (int q = 0; q < NG; ++q) hv[t][q] = __ldg(A.h + (off + (unsigned)col[q]));
        }
#pragma unroll
        for (int t = 0; t < kAdamPf; ++t) {
          const float4 P = pq[wid][(q0 + t) & 31];
          const bool in = !decltype(tail)::value || q0 + t < nc;
#pragma unroll
          for (int q = 0; q < NG; ++q) {
            const bool on = in && hv[t][q] > 0.f;
            adam_coord_hs(on, w[q], m[q], v[q], hv[t][q], P.x, P.y, P.z, P.w, ak);
            if (COUNT) tmask |= (on ? 1u : 0u) << q;
          }
        }
      };
      int q0 = 0;
      for (; q0 + kAdamPf <= nc; q0 += kAdamPf) batch(q0, std::false_type{});
      if (q0 < nc) batch(q0, std::true_type{});
    }
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      wr[col[q]] = w[q];
      mr[col[q]] = m[q];
      vr[col[q]] = v[q];
    }
    if (EX > 0 && lane < ne) {
      wr[xc] = xw;
      mr[xc] = xm;
      vr[xc] = xv;
    }
    if (lane == 0) {
      A.b2[r] = bb;
      A.mb2[r] = mb;
      A.vb2[r] = vb;
      A.steps2[r] = st + len;
    }
    if (A.z && lane < A.wpk) {  // lazy: the last reader of the row's masks clears them for the next step
      const_cast<uint32_t*>(A.mask)[(int64_t)r * A.wpk + lane] = 0u;
      const_cast<uint32_t*>(A.lmask)[(int64_t)r * A.wpk + lane] = 0u;
    }
    if (COUNT) {
      int tc = __popc(tmask);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tc += __shfl_xor_sync(0xffffffffu, tc, o);
      if (lane == 0) atomicAdd(A.touched, (unsigned long long)tc);
    }
    u = __shfl_sync(0xffffffffu, u_next, 0);
  }
}

template <int NG, bool COUNT, int EX = 0>
__device__ __forceinline__ void adam_rows_ng(const AdamRowsArgs& A, float4 (*pq)[32], int (*poff)[32]) {
  int col[NG];
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NG; ++q) col[q] = __ldg(A.live + 1 + q * 32 + lane);
  adam_rows_loop<NG, EX, COUNT>(A, col, pq, poff);
}

// lane l owns unit live[1 + 32 q + l] of live group q: only the groups
// holding live units are walked (dead units' coordinates never move).  The
// group count is read on the device (graph replays); one loop body per count.
template <int NV, bool COUNT>
__global__ void __launch_bounds__(256, NV == 1 ? 4 : 2) adam_rows_kernel(AdamRowsArgs A) {
  // per-warp broadcast of the current chunk's pair scalars: (e1, e2, c1,
  // sqrt(c2)) and the h row offset; h itself is read through L1
  __shared__ float4 pq[8][32];
  __shared__ int poff[8][32];
  const int nl = __ldg(A.live);
  const int ng = (nl + 31) >> 5;
  // wide hidden layers: the steady regime (at most one live group + extras)
  // runs in adam_rows_small_kernel, launched before this one
  if (NV >= 2 && nl <= kAdamSmallLive) return;
  // a few units past a whole group: the group plus scan-form extras
  if (nl > 32 && nl <= 32 + kAdamExtra) {
    adam_rows_ng<1, COUNT, kAdamExtra>(A, pq, poff);
    return;
  }
  if (NV >= 2 && nl > 64 && nl <= 64 + kAdamExtra) {
    adam_rows_ng<2, COUNT, kAdamExtra>(A, pq, poff);
    return;
  }
  if (NV == 1) {
    // (4 CTAs/SM: the 3- and 4-group bodies spill a little; they run only
    // while most units are live, i.e. the first step)
    switch (ng) {
      case 0:  // no live unit: group 0's lanes sit on dead units, nothing moves
      case 1: adam_rows_ng<1, COUNT>(A, pq, poff); break;
      case 2: adam_rows_ng<2, COUNT>(A, pq, poff); break;
      default: adam_rows_ng<4, COUNT>(A, pq, poff); break;
    }
  } else if (NV == 2) {
    switch (ng) {
      case 0:
      case 1: adam_rows_ng<1, COUNT>(A, pq, poff); break;
      case 2: adam_rows_ng<2, COUNT>(A, pq, poff); break;
      case 3: case 4: adam_rows_ng<4, COUNT>(A, pq, poff); break;
      default: adam_rows_ng<8, COUNT>(A, pq, poff); break;
    }
  } else {
    // wide hidden layers: the live groups rounded up to a power of two
    if (ng <= 1) adam_rows_ng<1, COUNT>(A, pq, poff);
    else if (ng <= 2) adam_rows_ng<2, COUNT>(A, pq, poff);
    else if (ng <= 4) adam_rows_ng<4, COUNT>(A, pq, poff);
    else if (ng <= 8) adam_rows_ng<8, COUNT>(A, pq, poff);
    else if (NV == 4 || ng <= 16) adam_rows_ng<NV * 4 < 16 ? NV * 4 : 16, COUNT>(A, pq, poff);
    else adam_rows_ng<NV * 4, COUNT>(A, pq, poff);
  }
}

// hidden_pad > 128: the kernel above carries the register budget of its
// 4- and 8-group bodies (126 registers, 2 CTAs per SM), but after the first
// steps at most ~40 units are live and a row's update is a chain of dependent
// loads -- bound by the rows in flight.  The one-group bodies alone fit 64
// registers: twice the resident warps.  Exactly one of the two kernels works
// on a given step (the live count is read on the device).
template <bool COUNT>
__global__ void __launch_bounds__(256, 3) adam_rows_small_kernel(AdamRowsArgs A) {
  __shared__ float4 pq[8][32];
  __shared__ int poff[8][32];
  const int nl = __ldg(A.live);
  if (nl > kAdamSmallLive) return;
  if (nl <= 32) adam_rows_ng<1, COUNT>(A, pq, poff);
  else if (nl <= 32 + kAdamExtra) adam_rows_ng<1, COUNT, kAdamExtra>(A, pq, poff);
  else if (nl <= 64) adam_rows_ng<2, COUNT>(A, pq, poff);
  else adam_rows_ng<2, COUNT, kAdamExtra>(A, pq, poff);
}

// Sparse-set steps (wide-out, scaled): a few hot rows (Zipf labels) are held
// by hundreds of samples while every other row has one or two.  The
// persistent kernel gives a row to one warp; ncu at the scaled shape: 138 us
// at 12% active warps and 2.5M instructions -- the whole launch is one warp
// walking a 1,024-pair row (~0.13 us a pair: an L2 round trip per 8-pair
// batch, then dependent FMA / MUFU chains with nothing else to issue).  So
// those rows get a CTA each, as the W1 long chains do
// (adam_features_long_kernel): lane = live unit, the row's pairs cut into 16
// consecutive segments; the moments are linear recurrences, so every warp
// folds its segment into (A1, X1, A2, X2), the segments' start moments follow
// from the earlier coefficients, every warp replays its segment with the real
// bias corrections summing its weight steps, and the steps are subtracted in
// segment order.  Two unit groups and the bias (activation 1) share a walk.
// Runs on a side stream beside the persistent kernel, which skips these rows;
// the grouping's entries are dealt round-robin to the CTAs (hot labels have
// neighbouring ids).
constexpr int kAdamVeryLong = 64;
constexpr int kVlWarps = 16;

template <bool COUNT>
__global__ void __launch_bounds__(kVlWarps * 32) adam_rows_vlong_kernel(AdamRowsArgs A) {
  // per warp and lane: (A1, X1, A2, X2) of two unit groups and the bias
  __shared__ float4 coef[kVlWarps][3][32];
  __shared__ float part[kVlWarps][3][32];
  __shared__ uint32_t movedw[kVlWarps][2];
  __shared__ int s_rows[kVlWarps * 32];
  __shared__ int s_n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hp = A.hp;
  const int ng = max(1, (__ldg(A.live) + 31) >> 5);
  const int nu = *A.n_uniq;
  const AdamK ak(A.ap);
  for (int base = 0; base < nu; base += gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int idx = base + threadIdx.x * gridDim.x + blockIdx.x;
    if (idx < nu && A.seg_cnt[idx] > kAdamVeryLong) s_rows[atomicAdd(&s_n, 1)] = idx;
    __syncthreads();
    const int n_rows = s_n;
    for (int ri = 0; ri < n_rows; ++ri) {
      const int uu = s_rows[ri];
      const int r = A.uniq[uu], s0 = A.seg_off[uu], len = A.seg_cnt[uu];
      const int64_t st = A.steps2[r];
      const int j0 = len * warp / kVlWarps, j1 = len * (warp + 1) / kVlWarps;
      // two unit groups per walk (the steady regime has one or two); the bias
      // rides with the first walk (activation 1, every lane the same value)
      for (int q0 = 0; q0 < ng; q0 += 2) {
        const bool bias = q0 == 0, two = q0 + 1 < ng;
        const int c0 = __ldg(A.live + 1 + q0 * 32 + lane);
        const int c1 = two ? __ldg(A.live + 1 + (q0 + 1) * 32 + lane) : 0;
        const int64_t ro0 = (int64_t)r * hp + c0, ro1 = (int64_t)r * hp + c1;
        // moments at the row's start, read before the last warp writes them back
        float m[3], v[3];
        m[0] = __ldcg(A.m2 + ro0), v[0] = __ldcg(A.v2 + ro0);
        m[1] = two ? __ldcg(A.m2 + ro1) : 0.f, v[1] = two ? __ldcg(A.v2 + ro1) : 0.f;
        m[2] = bias ? __ldcg(A.mb2 + r) : 0.f, v[2] = bias ? __ldcg(A.vb2 + r) : 0.f;
        // walk this warp's segment: fn(pair is inside, error, h0, h1, c1, sqrt(c2))
        auto walk = [&](auto fn, auto with_bc) {
          for (int jb = j0; jb < j1; jb += 32) {
            int off_l = 0;
            float d_l = 0.f, c1_l = 0.f, s2_l = 1.f;
            if (jb + lane < j1) {
              off_l = A.sslot[s0 + jb + lane] * hp;
              d_l = A.dsort[s0 + jb + lane];
              if (decltype(with_bc)::value) {
                const float2 bc = bias_corr(A.ap, st + jb + lane + 1);
                c1_l = bc.x;
                s2_l = sqrt_approx(bc.y);
              }
            }
            const int nc = min(32, j1 - jb);
            for (int t0 = 0; t0 < nc; t0 += 8) {
              float h0[8], h1[8];
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                const unsigned off = (unsigned)__shfl_sync(0xffffffffu, off_l, (t0 + t) & 31);
                h0[t] = __ldg(A.h + (off + (unsigned)c0));
                h1[t] = two ? __ldg(A.h + (off + (unsigned)c1)) : 0.f;
              }
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                const float d = __shfl_sync(0xffffffffu, d_l, (t0 + t) & 31);
                const float cc1 = __shfl_sync(0xffffffffu, c1_l, (t0 + t) & 31);
                const float s2 = __shfl_sync(0xffffffffu, s2_l, (t0 + t) & 31);
                fn(t0 + t < nc, d, h0[t], h1[t], cc1, s2);
              }
            }
          }
        };
        // phase 1: the segment's moment recurrences as (A1, X1, A2, X2)
        float a1[3] = {1.f, 1.f, 1.f}, x1[3] = {0.f, 0.f, 0.f}, a2[3] = {1.f, 1.f, 1.f}, x2[3] = {0.f, 0.f, 0.f};
        walk([&](bool in, float d, float h0, float h1, float, float) {
          const float hh[3] = {h0, h1, 1.f};
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            const bool on = in && (e == 2 ? bias : hh[e] > 0.f);
            const float g = d * hh[e];
            const float nx1 = fmaf(ak.b1, x1[e], ak.omb1 * g), nx2 = fmaf(ak.b2, x2[e], ak.omb2 * (g * g));
            x1[e] = on ? nx1 : x1[e];
            x2[e] = on ? nx2 : x2[e];
            a1[e] = on ? a1[e] * ak.b1 : a1[e];
            a2[e] = on ? a2[e] * ak.b2 : a2[e];
          }
        }, std::false_type{});
#pragma unroll
        for (int e = 0; e < 3; ++e) coef[warp][e][lane] = make_float4(a1[e], x1[e], a2[e], x2[e]);
        __syncthreads();
        for (int k = 0; k < warp; ++k) {
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            const float4 cf = coef[k][e][lane];
            m[e] = fmaf(cf.x, m[e], cf.y);
            v[e] = fmaf(cf.z, v[e], cf.w);
          }
        }
        // phase 2: replay with the bias corrections, sum the weight steps
        float psum[3] = {0.f, 0.f, 0.f};
        bool moved[2] = {false, false};
        walk([&](bool in, float d, float h0, float h1, float cc1, float s2) {
          const float hh[3] = {h0, h1, 1.f};
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            const bool on = in && (e == 2 ? bias : hh[e] > 0.f);
            const float g = d * hh[e];
            const float mn = fmaf(ak.b1, m[e], ak.omb1 * g), vn = fmaf(ak.b2, v[e], ak.omb2 * (g * g));
            const float stp = (cc1 * mn) * rcp_approx(fmaf(sqrt_approx(vn), s2, ak.eps));
            m[e] = on ? mn : m[e];
            v[e] = on ? vn : v[e];
            psum[e] += on ? stp : 0.f;
            if (e < 2) moved[e] |= on;
          }
        }, std::true_type{});
#pragma unroll
        for (int e = 0; e < 3; ++e) part[warp][e][lane] = psum[e];
        const uint32_t mv0 = __ballot_sync(0xffffffffu, moved[0]), mv1 = __ballot_sync(0xffffffffu, moved[1]);
        if (lane == 0) movedw[warp][0] = mv0, movedw[warp][1] = mv1;
        if (warp == kVlWarps - 1) {  // the chain's end state
          A.m2[ro0] = m[0];
          A.v2[ro0] = v[0];
          if (two) {
            A.m2[ro1] = m[1];
            A.v2[ro1] = v[1];
          }
          if (bias && lane == 0) {
            A.mb2[r] = m[2];
            A.vb2[r] = v[2];
          }
        }
        __syncthreads();
        if (warp == 0 || (warp == 1 && two) || (warp == 2 && bias)) {
          // warp e finishes entry e: the steps are subtracted in segment order
          const int e = warp;
          float* dst = e == 0 ? A.w2 + ro0 : e == 1 ? A.w2 + ro1 : A.b2 + r;
          float w = __ldcg(dst);
#pragma unroll
          for (int k = 0; k < kVlWarps; ++k) w -= part[k][e][lane];
          if (e < 2 || lane == 0) *dst = w;
          if (COUNT && e < 2 && lane == 0) {
            uint32_t any = 0;
#pragma unroll
            for (int k = 0; k < kVlWarps; ++k) any |= movedw[k][e];
            atomicAdd(A.touched, (unsigned long long)__popc(any));
          }
        }
        __syncthreads();  // coef / part / movedw reuse
      }
      if (threadIdx.x == 0) A.steps2[r] = st + len;
    }
    __syncthreads();  // s_rows / s_n reuse
  }
}

__global__ void accumulate_kernel(unsigned long long* dst, const int32_t* src) {
  if (src) *dst += (unsigned long long)*src;
}

void launch_accumulate(unsigned long long* dst, const int32_t* src, cudaStream_t s) {
  if (!src) return;
  accumulate_kernel<<<1, 1, 0, s>>>(dst, src);
  SLIDE_LAUNCH_CHECK();
}

void launch_adam_rows(int hp, int b, const AdamParams& ap, const int32_t* n_uniq, int64_t max_uniq,
                      const int32_t* uniq, const int32_t* seg_off, const int32_t* seg_cnt,
                      const int32_t* sslot, const float* dsort, const float* h, const int32_t* live, float* w2,
                      float* m2, float* v2, float* b2, float* mb2, float* vb2, int64_t* steps2,
                      unsigned long long* touched, int32_t* work, bool work_zeroed, cudaStream_t s,
                      const float* z, const float* stat, const uint32_t* mask, const uint32_t* lmask, int wpk,
                      const AdamVlong* vl) {
  if (max_uniq <= 0) return;
  if (!work_zeroed) SLIDE_CUDA(cudaMemsetAsync(work, 0, 4, s));
  // persistent: as many CTAs as are resident at once
  static const int env_per_sm = [] {
    const char* e = getenv("SLIDE_ADAM_ROWS_PER_SM");  // experiments only
    return e ? atoi(e) : 0;
  }();
  // one CTA slot per SM stays free for the W1 branch running beside it
  const int per_sm = env_per_sm > 0 ? env_per_sm : (hp <= 128 ? 3 : 2);
  const int grid = (int)std::min<int64_t>(ceil_div(max_uniq, 8), (int64_t)kSms * per_sm);
  AdamRowsArgs A{hp, ap, n_uniq, uniq, seg_off, seg_cnt, sslot, dsort, h, live,
                 w2, m2, v2, b2, mb2, vb2, steps2, touched, work, z, stat, mask, lmask, wpk};
  if (vl && !z) {
    // the hot rows first, on their own stream: their CTAs are placed before
    // the persistent kernel's, which skips them
    cudaStream_t sv = vl->stream ? vl->stream : s;
    if (vl->stream) {
      SLIDE_CUDA(cudaEventRecord(vl->fork, s));
      SLIDE_CUDA(cudaStreamWaitEvent(sv, vl->fork, 0));
    }
    const int vgrid = (int)std::min<int64_t>(ceil_div(max_uniq, kAdamVeryLong), (int64_t)kSms * 2);
    if (touched) adam_rows_vlong_kernel<true><<<vgrid, kVlWarps * 32, 0, sv>>>(A);
    else adam_rows_vlong_kernel<false><<<vgrid, kVlWarps * 32, 0, sv>>>(A);
    SLIDE_LAUNCH_CHECK();
    if (vl->stream) SLIDE_CUDA(cudaEventRecord(vl->join, sv));
    A.vlong = kAdamVeryLong;
  }
  if (hp > 128) {
    const int sgrid = (int)std::min<int64_t>(ceil_div(max_uniq, 8), (int64_t)kSms * (env_per_sm > 0 ? env_per_sm : 3));
    if (touched) adam_rows_small_kernel<true><<<sgrid, 256, 0, s>>>(A);
    else adam_rows_small_kernel<false><<<sgrid, 256, 0, s>>>(A);
    SLIDE_LAUNCH_CHECK();
  }
  if (touched) {
    SLIDE_NV_DISPATCH(hp, (adam_rows_kernel<NV, true><<<grid, 256, 0, s>>>(A)));
  } else {
    SLIDE_NV_DISPATCH(hp, (adam_rows_kernel<NV, false><<<grid, 256, 0, s>>>(A)));
  }
  SLIDE_LAUNCH_CHECK();
  if (vl && !z && vl->stream) SLIDE_CUDA(cudaStreamWaitEvent(s, vl->join, 0));
}

// ------------------------------------------------------- Adam, W1 features
__global__ void x_slots_kernel(const int32_t* __restrict__ x_ptr, int32_t* __restrict__ x_slot) {
  const int i = blockIdx.x;
  const int base = x_ptr[0];
  for (int k = x_ptr[i] + threadIdx.x; k < x_ptr[i + 1]; k += blockDim.x) x_slot[k - base] = i;
}

void launch_x_slots(int b, const int32_t* x_ptr, int32_t* x_slot, cudaStream_t s) {
  if (b <= 0) return;
  x_slots_kernel<<<b, 128, 0, s>>>(x_ptr, x_slot);
  SLIDE_LAUNCH_CHECK();
}

// tc[i][c] = #{i' <= i : h_i'[c] > 0}; hidden unit c's step for sample i is
// steps1[c] + tc[i][c] (each sample bumps the counter of its nz(h) rows,
// network.py:436-437).  bc holds the two bias corrections.
// One warp per hidden unit: ballot + popc prefix over the samples.
__global__ void hidden_counts_kernel(int hp, int b, AdamParams ap, const float* __restrict__ h,
                                     const int64_t* __restrict__ steps1, int32_t* __restrict__ tc,
                                     float2* __restrict__ bc) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= hp) return;
  const int64_t st = steps1[c];
  int run = 0;
  for (int i0 = 0; i0 < b; i0 += 32) {
    const int i = i0 + lane;
    const int64_t q = (int64_t)i * hp + c;
    const bool act = i < b && h[q] > 0.f;
    const unsigned mask = __ballot_sync(0xffffffffu, act);
    const int cnt = run + __popc(mask & ((1u << lane) - 1u)) + (act ? 1 : 0);
    if (i < b) {
      tc[q] = cnt;
      if (act) bc[q] = bias_corr(ap, st + cnt);
    }
    run += __popc(mask);
  }
}

void launch_hidden_counts(int hp, int b, const AdamParams& ap, const float* h, const int64_t* steps1, int32_t* tc,
                          float2* bc, cudaStream_t s) {
  hidden_counts_kernel<<<(int)ceil_div((int64_t)hp * 32, 256), 256, 0, s>>>(hp, b, ap, h, steps1, tc, bc);
  SLIDE_LAUNCH_CHECK();
}

constexpr int kColGroup = 8;  // pairs per prefetch group of the column path

struct AdamFeatArgs {
  int hp;
  AdamParams ap;
  const int32_t *n_uniq, *uniq, *seg_off, *seg_cnt, *sorted_k, *x_slot;
  const float* x_val;
  int64_t x_base;
  const float *h, *dh;
  const float2* bc;
  const int32_t* live;
  float *w1t, *m1t, *v1t;
  unsigned long long* touched;
  const int32_t *long_list, *n_long;  // the grouping's chains longer than kW1LongChain
};

// Short chains (<= kW1LongChain samples hold the feature), one warp per
// feature row, lane l on unit live[1 + 32 q + l] of live group q; every
// pair's (h, dh, bias corrections) loads are issued before its updates.
template <int NG>
__device__ __forceinline__ void adam_features_loop(const AdamFeatArgs& A) {
  constexpr int PF = NG >= 4 ? 2 : 8 / NG;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nu = *A.n_uniq;
  const int hp = A.hp;
  const AdamK ak(A.ap);
  int col[NG];
#pragma unroll
  for (int q = 0; q < NG; ++q) col[q] = __ldg(A.live + 1 + q * 32 + lane);
  // a long chain (a hot feature held by many samples) is the long-chain
  // kernel's (the grouping listed it)
  for (int64_t u = gw; u < nu; u += nw) {
    const int len = A.seg_cnt[u];
    if (len > kW1LongChain) continue;
    uint32_t tmask = 0;
    const int f = A.uniq[u];
    const int s0 = A.seg_off[u];
    float* wr = A.w1t + (int64_t)f * hp;
    float* mr = A.m1t + (int64_t)f * hp;
    float* vr = A.v1t + (int64_t)f * hp;
    // lane j < len: pair j's h row offset and input value
    int off_l = 0;
    float xv_l = 0.f;
    if (lane < len) {
      const int k = A.sorted_k[s0 + lane];
      off_l = A.x_slot[k] * hp;
      xv_l = A.x_val[A.x_base + k];
    }
    float w[NG], m[NG], v[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      w[q] = wr[col[q]];
      m[q] = mr[col[q]];
      v[q] = vr[col[q]];
    }
    for (int t0 = 0; t0 < len; t0 += PF) {
      float hv[PF][NG], gv[PF][NG];
      float2 bv[PF][NG];
#pragma unroll
      for (int t = 0; t < PF; ++t) {
        const int off = __shfl_sync(0xffffffffu, off_l, (t0 + t) & 31);  // past len: lane's 0 offset, off below
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          hv[t][q] = __ldg(A.h + off + col[q]);
          gv[t][q] = __ldg(A.dh + off + col[q]);
          bv[t][q] = __ldg(A.bc + off + col[q]);
        }
      }
#pragma unroll
      for (int t = 0; t < PF; ++t) {
        const float xv = __shfl_sync(0xffffffffu, xv_l, (t0 + t) & 31);
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          // the hidden error already carries the h > 0 mask; h decides which
          // coordinates move
          const bool on = t0 + t < len && hv[t][q] > 0.f;
          adam_coord_if(on, w[q], m[q], v[q], gv[t][q] * xv, bv[t][q].x, bv[t][q].y, ak);
          tmask |= (on ? 1u : 0u) << q;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      wr[col[q]] = w[q];
      mr[col[q]] = m[q];
      vr[col[q]] = v[q];
    }
    if (A.touched) {
      int tc = __popc(tmask);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tc += __shfl_xor_sync(0xffffffffu, tc, o);
      if (lane == 0) atomicAdd(A.touched, (unsigned long long)tc);
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(256, NV == 1 ? 4 : 2) adam_features_kernel(AdamFeatArgs A) {
  const int ng = (__ldg(A.live) + 31) >> 5;
  SLIDE_NG_DISPATCH(NV, ng, adam_features_loop, A);
}

// Long chains (a hot feature held by > kW1LongChain samples): work item =
// (feature, live 32-unit group), one CTA of kLongWarps warps, lane = unit.
// The feature's pairs are cut into kLongWarps consecutive segments.  The
// moments are linear recurrences, so each warp first folds its segment into
// (A1, X1, A2, X2) with m_end = A1 m_start + X1 (v alike); the segments'
// start moments follow from the earlier segments' coefficients, every warp
// then replays its segment with the real bias corrections and sums its
// weight steps, and the steps are subtracted in segment order.  The
// sequential chain of the reference (network.py:428-451, one Adam step per
// sample in slot order) becomes kLongWarps chains 1 / kLongWarps as long.
// kLongWarps: 4 for batches up to 128 slots, 8 beyond (the chains are as
// long as the batch).
template <int kLongWarps>
__global__ void __launch_bounds__(kLongWarps * 32) adam_features_long_kernel(AdamFeatArgs A) {
  __shared__ float4 coef[kLongWarps][32];
  __shared__ float part[kLongWarps][32];
  __shared__ uint32_t movedw[kLongWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hp = A.hp;
  const int G = (__ldg(A.live) + 31) >> 5;
  const int64_t items = (int64_t)*A.n_long * G;
  const AdamK ak(A.ap);
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int u = A.long_list[item / G];
    const int grp = (int)(item % G);
    const int c = __ldg(A.live + 1 + grp * 32 + lane);
    const int f = A.uniq[u], s0 = A.seg_off[u], len = A.seg_cnt[u];
    const int j0 = len * warp / kLongWarps, j1 = len * (warp + 1) / kLongWarps;
    const int64_t ro = (int64_t)f * hp + c;
    float m = __ldcg(A.m1t + ro), v = __ldcg(A.v1t + ro);  // read before the last warp writes them back
    // walk this warp's segment: fn(j, on, gd, bias corrections)
    auto walk = [&](auto fn, auto with_bc) {
      for (int jb = j0; jb < j1; jb += 32) {
        int off_l = 0;
        float xv_l = 0.f;
        if (jb + lane < j1) {
          const int k = A.sorted_k[s0 + jb + lane];
          off_l = A.x_slot[k] * hp;
          xv_l = A.x_val[A.x_base + k];
        }
        const int nc = min(32, j1 - jb);
        for (int t0 = 0; t0 < nc; t0 += kColGroup) {
          float hv[kColGroup], gv[kColGroup];
          float2 bv[kColGroup];
#pragma unroll
          for (int t = 0; t < kColGroup; ++t) {
            const unsigned off = (unsigned)__shfl_sync(0xffffffffu, off_l, (t0 + t) & 31) + (unsigned)c;
            hv[t] = __ldg(A.h + off);
            gv[t] = __ldg(A.dh + off);
            if (decltype(with_bc)::value) bv[t] = __ldg(A.bc + off);
          }
#pragma unroll
          for (int t = 0; t < kColGroup; ++t) {
            const float xv = __shfl_sync(0xffffffffu, xv_l, (t0 + t) & 31);
            const bool on = t0 + t < nc && hv[t] > 0.f;
            fn(on, gv[t] * xv, bv[t]);
          }
        }
      }
    };
    // phase 1: the segment's moment recurrences as (A1, X1, A2, X2)
    float a1 = 1.f, x1 = 0.f, a2 = 1.f, x2 = 0.f;
    walk([&](bool on, float g, float2) {
      const float nx1 = fmaf(ak.b1, x1, ak.omb1 * g), nx2 = fmaf(ak.b2, x2, ak.omb2 * (g * g));
      x1 = on ? nx1 : x1;
      x2 = on ? nx2 : x2;
      a1 = on ? a1 * ak.b1 : a1;
      a2 = on ? a2 * ak.b2 : a2;
    }, std::false_type{});
    coef[warp][lane] = make_float4(a1, x1, a2, x2);
    __syncthreads();
    for (int k = 0; k < warp; ++k) {
      const float4 cf = coef[k][lane];
      m = fmaf(cf.x, m, cf.y);
      v = fmaf(cf.z, v, cf.w);
    }
    // phase 2: replay with the bias corrections, sum the weight steps
    float psum = 0.f;
    bool moved = false;
    walk([&](bool on, float g, float2 cc) {
      const float mn = fmaf(ak.b1, m, ak.omb1 * g), vn = fmaf(ak.b2, v, ak.omb2 * (g * g));
      const float st = (cc.x * mn) * rcp_approx(sqrt_approx(vn * cc.y) + ak.eps);
      m = on ? mn : m;
      v = on ? vn : v;
      psum += on ? st : 0.f;
      moved |= on;
    }, std::true_type{});
    part[warp][lane] = psum;
    const uint32_t mv = __ballot_sync(0xffffffffu, moved);
    if (lane == 0) movedw[warp] = mv;
    if (warp == kLongWarps - 1) {  // the chain's end state
      A.m1t[ro] = m;
      A.v1t[ro] = v;
    }
    __syncthreads();
    if (warp == 0) {
      float w = __ldcg(A.w1t + ro);
#pragma unroll
      for (int k = 0; k < kLongWarps; ++k) w -= part[k][lane];
      A.w1t[ro] = w;
      if (A.touched && lane == 0) {
        uint32_t any = 0;
#pragma unroll
        for (int k = 0; k < kLongWarps; ++k) any |= movedw[k];
        atomicAdd(A.touched, (unsigned long long)__popc(any));
      }
    }
    __syncthreads();  // coef / part / movedw reuse
  }
}

void launch_adam_features(int hp, const AdamParams& ap, const int32_t* n_uniq, int64_t max_uniq,
                          const int32_t* uniq, const int32_t* seg_off, const int32_t* seg_cnt,
                          const int32_t* sorted_k, const int32_t* x_slot, const float* x_val, int64_t x_base,
                          const float* h, const float* dh, const float2* bc, const int32_t* live, float* w1t,
                          float* m1t, float* v1t, unsigned long long* touched, const int32_t* long_list,
                          const int32_t* n_long, cudaStream_t s, cudaStream_t s_long, int b) {
  if (max_uniq <= 0) return;
  int grid = (int)std::min<int64_t>(ceil_div(max_uniq, 8), (int64_t)kSms * 16);
  AdamFeatArgs A{hp, ap, n_uniq, uniq, seg_off, seg_cnt, sorted_k, x_slot, x_val, x_base, h, dh, bc, live,
                 w1t, m1t, v1t, touched, long_list, n_long};
  // long chains first (on s_long, beside the short ones; they are the
  // branch's tail): at most max_uniq / (kW1LongChain + 1) of them
  const int64_t max_long = std::min<int64_t>(max_uniq, ceil_div(max_uniq, kW1LongChain)) * (hp / 32);
  const int lgrid = (int)std::min<int64_t>(std::max<int64_t>(max_long, 1), (int64_t)kSms * 16);
  // (16 warps were tried for B = 1,024: a 512-thread CTA only finds room once
  // the short-chain kernel's 256-thread CTAs have drained, so the long chains
  // started when the short ones ended; 8 warps run beside them)
  if (b <= 128) adam_features_long_kernel<4><<<lgrid, 4 * 32, 0, s_long>>>(A);
  else adam_features_long_kernel<8><<<lgrid, 8 * 32, 0, s_long>>>(A);
  SLIDE_LAUNCH_CHECK();
  SLIDE_NV_DISPATCH(hp, (adam_features_kernel<NV><<<grid, 256, 0, s>>>(A)));
  SLIDE_LAUNCH_CHECK();
}

// hidden biases: rows nz(h_i) of every sample in slot order, g = dh_i
__global__ void adam_hidden_bias_kernel(int hp, int b, AdamParams ap, const float* __restrict__ h,
                                        const float* __restrict__ dh, const int32_t* __restrict__ tc,
                                        const float2* __restrict__ bc, float* __restrict__ b1,
                                        float* __restrict__ mb1, float* __restrict__ vb1,
                                        int64_t* __restrict__ steps1) {
  // one warp per hidden unit: 32 samples' inputs loaded at once, the Adam
  // recurrence then walks them in slot order (all lanes redundantly)
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= hp || b <= 0) return;
  const AdamK ak(ap);
  float bb = b1[c], mb = mb1[c], vb = vb1[c];
  for (int i0 = 0; i0 < b; i0 += 32) {
    const int i = i0 + lane;
    const int64_t q = (int64_t)i * hp + c;
    const bool act = i < b && h[q] > 0.f;
    const float g = act ? dh[q] : 0.f;
    const float2 cc = act ? bc[q] : make_float2(0.f, 1.f);
    unsigned mask = __ballot_sync(0xffffffffu, act);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      adam_coord(bb, mb, vb, __shfl_sync(0xffffffffu, g, src), __shfl_sync(0xffffffffu, cc.x, src),
                 __shfl_sync(0xffffffffu, cc.y, src), ak);
    }
  }
  if (lane == 0) {
    b1[c] = bb;
    mb1[c] = mb;
    vb1[c] = vb;
    steps1[c] += tc[(int64_t)(b - 1) * hp + c];
  }
}

void launch_adam_hidden_bias(int hp, int b, const AdamParams& ap, const float* h, const float* dh, const int32_t* tc,
                             const float2* bc, float* b1, float* mb1, float* vb1, int64_t* steps1, cudaStream_t s) {
  adam_hidden_bias_kernel<<<(int)ceil_div((int64_t)hp * 32, 256), 256, 0, s>>>(hp, b, ap, h, dh, tc, bc, b1, mb1,
                                                                               vb1, steps1);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide

namespace slide {

// Hidden-unit bookkeeping and bias update in one pass, one warp per hidden
// unit c: tc[i][c] = #{i' <= i : h_i'[c] > 0} (unit c's step for sample i is
// steps1[c] + tc[i][c], network.py:436-437), the two bias corrections for the
// W1 Adam, then the bias recurrence over those samples in slot order
// (g = dh_i[c]) and the step counter.  Runs after the hidden gradient and
// before the W1 Adam (which reads tc / bc, not steps1).
// One CTA per hidden unit, one warp per 32 samples: the chunks' active counts
// and their folded moment recurrences (A, X per chunk: m_end = A m_start + X)
// are exchanged through shared memory, every warp chains the earlier chunks'
// coefficients in order -- the same operations in the same order as walking
// the chunks one after another (bit-identical), without the serial walk
// (B = 1,024: 32 dependent chunks of scattered loads, 46 us -> a few).
__global__ void __launch_bounds__(1024) hidden_prep_bias_kernel(int hp, int b, AdamParams ap,
                                                                const float* __restrict__ h,
                                                                const float* __restrict__ dh,
                                                                int64_t* __restrict__ steps1, int32_t* __restrict__ tc,
                                                                float2* __restrict__ bc, float* __restrict__ b1,
                                                                float* __restrict__ mb1, float* __restrict__ vb1) {
  __shared__ int wcnt[32];
  __shared__ float4 agg[32];
  __shared__ float usum[32];
  const int c = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const AdamK ak(ap);
  const int i = w * 32 + lane;
  const int64_t q = (int64_t)i * hp + c;
  const bool act = i < b && h[q] > 0.f;
  const unsigned mask = __ballot_sync(0xffffffffu, act);
  if (lane == 0) wcnt[w] = __popc(mask);
  __syncthreads();
  int run = 0, total = 0;
  for (int k = 0; k < nw; ++k) {
    const int n = wcnt[k];
    run += k < w ? n : 0;
    total += n;
  }
  const int cnt = run + __popc(mask & ((1u << lane) - 1u)) + (act ? 1 : 0);
  if (i < b) tc[q] = cnt;
  if (total == 0) return;  // a dead unit: nothing moves (uniform over the CTA)
  const int64_t st = steps1[c];
  float g = 0.f;
  float2 cc = make_float2(0.f, 1.f);
  if (act) {
    cc = bias_corr(ap, st + cnt);
    bc[q] = cc;
    g = dh[q];
  }
  // the bias moments are linear recurrences over the active samples (slot
  // order): a warp scan inside the chunk, the chunks' coefficients chained
  float a1 = act ? ak.b1 : 1.f, x1 = act ? ak.omb1 * g : 0.f;
  float a2 = act ? ak.b2 : 1.f, x2 = act ? ak.omb2 * (g * g) : 0.f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float pa1 = __shfl_up_sync(0xffffffffu, a1, o), px1 = __shfl_up_sync(0xffffffffu, x1, o);
    const float pa2 = __shfl_up_sync(0xffffffffu, a2, o), px2 = __shfl_up_sync(0xffffffffu, x2, o);
    if (lane >= o) {
      x1 = fmaf(a1, px1, x1);
      a1 *= pa1;
      x2 = fmaf(a2, px2, x2);
      a2 *= pa2;
    }
  }
  if (lane == 31) agg[w] = make_float4(a1, x1, a2, x2);
  __syncthreads();
  float mb = mb1[c], vb = vb1[c];
  for (int k = 0; k < w; ++k) {
    if (wcnt[k] == 0) continue;  // (an all-inactive chunk leaves the moments alone)
    const float4 cf = agg[k];
    mb = fmaf(cf.x, mb, cf.y);
    vb = fmaf(cf.z, vb, cf.w);
  }
  const float mj = fmaf(a1, mb, x1), vj = fmaf(a2, vb, x2);
  float upd = act ? (cc.x * mj) * rcp_approx(sqrt_approx(vj * cc.y) + ak.eps) : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_xor_sync(0xffffffffu, upd, o);
  if (lane == 0) usum[w] = upd;
  __syncthreads();
  if (w == nw - 1 && lane == 31) {
    float bb = b1[c];
    for (int k = 0; k < nw; ++k)
      if (wcnt[k]) bb -= usum[k];
    b1[c] = bb;
    mb1[c] = wcnt[w] ? mj : mb;
    vb1[c] = wcnt[w] ? vj : vb;
    steps1[c] = st + total;
  }
}

void launch_hidden_prep_bias(int hp, int b, const AdamParams& ap, const float* h, const float* dh, int64_t* steps1,
                             int32_t* tc, float2* bc, float* b1, float* mb1, float* vb1, cudaStream_t s) {
  if (b <= 0) return;
  SLIDE_CHECK(b <= 1024, kNotSupported, "hidden bias update: at most 1,024 slots");
  hidden_prep_bias_kernel<<<hp, (int)ceil_div(b, 32) * 32, 0, s>>>(hp, b, ap, h, dh, steps1, tc, bc, b1, mb1, vb1);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide

namespace slide {

// ---------------------------------------------- sharded softmax (3 phases)
// The active set of a sample is split across ranks; the max and the sum of
// exponentials are combined by the caller's all-reduces between phases.
__global__ void __launch_bounds__(1024) softmax_max_kernel(const int32_t* __restrict__ offs, const float* __restrict__ z,
                                                          float* __restrict__ out) {
  using RF = cub::BlockReduce<float, 1024>;
  __shared__ typename RF::TempStorage tmp;
  const int i = blockIdx.x;
  const int o = offs[i], n = offs[i + 1] - o;
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < n; k += 1024) mx = fmaxf(mx, z[o + k]);
  mx = RF(tmp).Reduce(mx, cub::Max());
  if (threadIdx.x == 0) out[i] = mx;
}

__global__ void __launch_bounds__(1024) softmax_sum_kernel(const int32_t* __restrict__ offs, const float* __restrict__ z,
                                                          const float* __restrict__ gmax, float* __restrict__ out) {
  using RF = cub::BlockReduce<float, 1024>;
  __shared__ typename RF::TempStorage tmp;
  const int i = blockIdx.x;
  const int o = offs[i], n = offs[i + 1] - o;
  const float mx = gmax[i];
  float se = 0.f;
  for (int k = threadIdx.x; k < n; k += 1024) se += expf(z[o + k] - mx);
  se = RF(tmp).Sum(se);
  if (threadIdx.x == 0) out[i] = se;
}

__global__ void __launch_bounds__(1024) softmax_finish_kernel(const int32_t* __restrict__ offs,
                                                             const uint8_t* __restrict__ plab,
                                                             const int32_t* __restrict__ y_ptr,
                                                             const float* __restrict__ z,
                                                             const float* __restrict__ gmax,
                                                             const float* __restrict__ gsum, float* __restrict__ prob,
                                                             float* __restrict__ delta, double* __restrict__ loss,
                                                             const int32_t* __restrict__ inv,
                                                             float* __restrict__ dsort) {
  using RD = cub::BlockReduce<double, 1024>;
  __shared__ typename RD::TempStorage tmp;
  const int i = blockIdx.x;
  const int o = offs[i], n = offs[i + 1] - o;
  const int ny = y_ptr[i + 1] - y_ptr[i];
  const float mx = gmax[i], se = gsum[i], lse = logf(se);
  const float inv_ny = ny > 0 ? 1.f / (float)ny : 0.f;
  double lsum = 0.0;
  for (int k = threadIdx.x; k < n; k += 1024) {
    const float zz = z[o + k] - mx;
    const float p = expf(zz) / se;
    const int lab = plab[o + k];
    prob[o + k] = p;
    const float dl = lab ? p - inv_ny : p;
    delta[o + k] = dl;
    if (inv) dsort[inv[o + k]] = dl;
    if (lab) {
      const double nl = -((double)zz - (double)lse);
      lsum += (nl < 690.7755278982137 || nl != nl) ? nl : 690.7755278982137;  // NaN propagates (np.maximum)
    }
  }
  lsum = RD(tmp).Sum(lsum);
  if (threadIdx.x == 0) loss[i] = lsum;  // sum over this rank's labels; / |Y| after the all-reduce
}

void launch_softmax_max(int b, const int32_t* offs, const float* z, float* out, cudaStream_t s) {
  softmax_max_kernel<<<b, 1024, 0, s>>>(offs, z, out);
  SLIDE_LAUNCH_CHECK();
}

void launch_softmax_sum(int b, const int32_t* offs, const float* z, const float* gmax, float* out, cudaStream_t s) {
  softmax_sum_kernel<<<b, 1024, 0, s>>>(offs, z, gmax, out);
  SLIDE_LAUNCH_CHECK();
}

void launch_softmax_finish(int b, const int32_t* offs, const uint8_t* plab, const int32_t* y_ptr, const float* z,
                           const float* gmax, const float* gsum, float* prob, float* delta, double* loss_part,
                           const int32_t* inv, float* dsort, cudaStream_t s) {
  softmax_finish_kernel<<<b, 1024, 0, s>>>(offs, plab, y_ptr, z, gmax, gsum, prob, delta, loss_part, inv, dsort);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide

namespace slide {

// ------------------------------------------ hidden layer sharded by units
// W1^T is split by hidden units -- rank g holds the hg columns
// [g hg, (g + 1) hg) as a (D, hg) array.  Phase 1 (shard_hidden_kernel):
// the rank's pre-activation partial sums for every sample, in the exact
// term order of hidden_fwd_kernel (KW partial chains over the nonzeros
// k = w, w + KW, ... then the chains summed in chain order), so the
// all-gathered row equals the unsharded one bit for bit.  Phase 2
// (shard_assemble_kernel, after the all-gather): h = relu(row + b1), the
// per-sample nonzero masks and, by the last CTA, the live-unit list.
template <int KW>
__global__ void shard_hidden_kernel(int hg, const int32_t* __restrict__ x_ptr, const int32_t* __restrict__ x_idx,
                                    const float* __restrict__ x_val, const float* __restrict__ w1s,
                                    float* __restrict__ part) {
  extern __shared__ float red[];  // [KW][hg]
  const int i = blockIdx.x;
  const int nq = hg >> 2;
  const int w = threadIdx.x / nq, q = threadIdx.x % nq;
  const int a = x_ptr[i], e = x_ptr[i + 1];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = a + w; k < e; k += KW) {
    const float v = x_val[k];
    const float4 r = ld4(w1s + (int64_t)x_idx[k] * hg + 4 * q);
    acc.x = fmaf(v, r.x, acc.x);
    acc.y = fmaf(v, r.y, acc.y);
    acc.z = fmaf(v, r.z, acc.z);
    acc.w = fmaf(v, r.w, acc.w);
  }
  *reinterpret_cast<float4*>(&red[w * hg + 4 * q]) = acc;
  __syncthreads();
  for (int c = threadIdx.x; c < hg; c += blockDim.x) {
    float s = red[c];
    for (int k = 1; k < KW; ++k) s += red[k * hg + c];
    part[(int64_t)i * hg + c] = s;
  }
}

void launch_shard_hidden(int hp, int hg, int b, const int32_t* x_ptr, const int32_t* x_idx, const float* x_val,
                         const float* w1s, float* part, cudaStream_t s) {
  if (b <= 0) return;
  SLIDE_CHECK(hg % 4 == 0 && hg <= 128, kNotSupported, "hidden units per shard must be a multiple of 4, <= 128");
  // the unsharded kernel's chain count for this padded width
  const int kw = hp / 128 <= 2 ? 32 : 8;
  const int threads = kw * (hg / 4);
  const size_t smem = (size_t)kw * hg * 4;
  if (kw == 32)
    shard_hidden_kernel<32><<<b, threads, smem, s>>>(hg, x_ptr, x_idx, x_val, w1s, part);
  else
    shard_hidden_kernel<8><<<b, threads, smem, s>>>(hg, x_ptr, x_idx, x_val, w1s, part);
  SLIDE_LAUNCH_CHECK();
}

// parts: the all-gathered (G, b, hg) partial rows; unit c = g hg + j
__global__ void __launch_bounds__(256) shard_assemble_kernel(int hp, int hidden, int hg, int b,
                                                             const float* __restrict__ parts,
                                                             const float* __restrict__ b1, float* __restrict__ h,
                                                             uint32_t* __restrict__ hmask, int32_t* __restrict__ live,
                                                             int32_t* __restrict__ ticket) {
  const int i = blockIdx.x, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < hp; c += blockDim.x) {
    float s = 0.f;
    if (c < hidden) s = parts[((int64_t)(c / hg) * b + i) * hg + c % hg];
    s += b1[c];
    const float hv = s > 0.f ? s : 0.f;
    h[(int64_t)i * hp + c] = hv;
    const unsigned bal = __ballot_sync(0xffffffffu, hv > 0.f);
    if (lane == 0) hmask[(int64_t)i * (hp >> 5) + (c >> 5)] = bal;
  }
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  build_live_cols(hp, gridDim.x, hmask, live);
  if (threadIdx.x == 0) *ticket = 0;
}

void launch_shard_assemble(int hp, int hidden, int hg, int b, const float* parts, const float* b1, float* h,
                           uint32_t* hmask, int32_t* live, int32_t* ticket, cudaStream_t s) {
  if (b <= 0) return;
  shard_assemble_kernel<<<b, 256, 0, s>>>(hp, hidden, hg, b, parts, b1, h, hmask, live, ticket);
  SLIDE_LAUNCH_CHECK();
}

// W1 Adam on this rank's hg hidden units (reference network.py:428-451 for
// layer 0): one warp per distinct input feature of the batch, lanes on the
// shard's columns, the feature's samples walked in slot order; unit c moves
// for sample i iff h_i[c] > 0, with its bias corrections bc[i][c] (the
// replicated hidden_prep_bias_kernel's) and gradient dh_i[c] x_i[f].
__global__ void __launch_bounds__(256) adam_w1_shard_kernel(int hp, int hg, int c0, AdamParams ap,
                                                            const int32_t* __restrict__ n_uniq,
                                                            const int32_t* __restrict__ uniq,
                                                            const int32_t* __restrict__ seg_off,
                                                            const int32_t* __restrict__ seg_cnt,
                                                            const int32_t* __restrict__ sorted_k,
                                                            const int32_t* __restrict__ x_slot,
                                                            const float* __restrict__ x_val, int64_t x_base,
                                                            const float* __restrict__ h, const float* __restrict__ dh,
                                                            const float2* __restrict__ bc, float* __restrict__ w1s,
                                                            float* __restrict__ m1s, float* __restrict__ v1s,
                                                            unsigned long long* touched) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nu = *n_uniq;
  const AdamK ak(ap);
  for (int64_t u = gw; u < nu; u += nw) {
    const int f = uniq[u], s0 = seg_off[u], len = seg_cnt[u];
    int moved = 0;
    for (int j0 = 0; j0 < hg; j0 += 32) {
      const int j = j0 + lane;
      const bool mine = j < hg;
      const int c = c0 + (mine ? j : 0);
      const int64_t ro = (int64_t)f * hg + (mine ? j : 0);
      float w = mine ? w1s[ro] : 0.f, m = mine ? m1s[ro] : 0.f, v = mine ? v1s[ro] : 0.f;
      for (int t = 0; t < len; ++t) {
        const int k = sorted_k[s0 + t];
        const unsigned off = (unsigned)(x_slot[k] * hp + c);
        const float xv = x_val[x_base + k];
        const float hv = __ldg(h + off);
        const bool on = mine && hv > 0.f;
        const float2 cc = on ? __ldg(bc + off) : make_float2(0.f, 1.f);
        adam_coord_if(on, w, m, v, __ldg(dh + off) * xv, cc.x, cc.y, ak);
        moved |= on;
      }
      if (mine) {
        w1s[ro] = w;
        m1s[ro] = m;
        v1s[ro] = v;
      }
    }
    if (touched) {
      const int tc = __popc(__ballot_sync(0xffffffffu, moved));
      if (lane == 0) atomicAdd(touched, (unsigned long long)tc);
    }
  }
}

void launch_adam_w1_shard(int hp, int hg, int c0, const AdamParams& ap, const int32_t* n_uniq, int64_t max_uniq,
                          const int32_t* uniq, const int32_t* seg_off, const int32_t* seg_cnt, const int32_t* sorted_k,
                          const int32_t* x_slot, const float* x_val, int64_t x_base, const float* h, const float* dh,
                          const float2* bc, float* w1s, float* m1s, float* v1s, unsigned long long* touched,
                          cudaStream_t s) {
  if (max_uniq <= 0) return;
  const int grid = (int)std::min<int64_t>(ceil_div(max_uniq, 8), (int64_t)kSms * 16);
  adam_w1_shard_kernel<<<grid, 256, 0, s>>>(hp, hg, c0, ap, n_uniq, uniq, seg_off, seg_cnt, sorted_k, x_slot, x_val,
                                            x_base, h, dh, bc, w1s, m1s, v1s, touched);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide
